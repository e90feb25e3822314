#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench (cfg 3 + cfg 2), ncu launch list and
# a full capture of the forward gather and backward kernels.  Outputs in gpurun_out/.
set -x
O=gpurun_out/${TAG:-run}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench3.json 2> $O/bench3.err
timeout 300 python bench.py --config 2 --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err
timeout 300 python bench.py --config 1 --no-cpu-baseline > $O/bench1.json 2> $O/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gather|k_backward_points|k_emit|k_cellsort|k_count|k_scatter' -c 8 \
   -o $O/full python tools/prof_small.py 4 > $O/ncu_full.log 2>&1
ls -la $O

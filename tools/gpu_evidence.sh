#!/bin/bash
# Round evidence on one B200: parity tests, smoke, bench lines for every
# BASELINE config, the reference arm, the launch list and full ncu captures.
O=gpurun_out/${TAG:-evidence}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench3.json 2> $O/bench3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench3_ref.json 2> $O/bench3_ref.err
for c in 1 2 4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench$c.json 2> $O/bench$c.err
done
timeout 900 python bench.py --config 5 --steps 3 --no-cpu-baseline --e2e-steps 0 > $O/bench5.json 2> $O/bench5.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
   --log-file $O/launches_cfg3.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gather|k_backward_points|k_scatter_emit|k_count4' -c 4 \
   -o $O/full python tools/prof_small.py 4 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gather_wide|k_backward_wide' -c 2 \
   -o $O/wide python tools/prof_cfg5.py 2 > $O/ncu_wide.log 2>&1
python tools/cfg5_cluster_split.py > $O/cfg5_cluster_split.txt 2>&1
ls -la $O

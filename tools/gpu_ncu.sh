#!/bin/bash
# one iteration: parity tests, cfg3 bench, full ncu capture of the kernels matching $KREGEX
O=gpurun_out/${TAG:-band}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $O/bench3.json 2> $O/bench3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_gather}" -c 1 \
   -o $O/full python tools/prof_small.py 8 > $O/ncu_full.log 2>&1
tail -3 $O/pytest_gpu.log; python -c "import json; d=json.load(open('$O/bench3.json')); print(d['ms_per_step'], d['value'], d['phases_ms_per_step'])"

#!/bin/bash
# quick GPU pass: parity tests + cfg3 bench (no ncu)
O=gpurun_out/${TAG:-quick}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $O/bench3.json 2> $O/bench3.err
tail -3 $O/pytest_gpu.log; cat $O/bench3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phases_ms_per_step'])"

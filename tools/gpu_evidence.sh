#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, bench lines for every
# BASELINE config, the reference arm, the launch list and full ncu captures.
O=gpurun_out/${TAG:-evidence}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench3.json 2> $O/bench3.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench3_ref.json 2> $O/bench3_ref.err
for c in 1 2 4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench$c.json 2> $O/bench$c.err
done
timeout 900 python bench.py --config 5 --steps 3 --no-cpu-baseline --e2e-steps 0 > $O/bench5.json 2> $O/bench5.err
for f in $O/bench*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1].split('/')[-1], d.get('ms_per_step'), d.get('value'), d.get('phases_ms_per_step'), (d.get('roofline') or {}).get('step_frac'), (d.get('e2e') or {}).get('value'))
except Exception as e:
    print(sys.argv[1], 'failed', e)
PY
done
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv $CMD > $O/ncu_launch.log 2>&1
python tools/prof_small.py 64 > $O/plain_b64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_gather|k_backward_points|k_scatter_emit|k_count_smem' -s 4 -c 4 -o $O/full_b64 python tools/prof_small.py 64 > $O/ncu_full.log 2>&1
ls -la $O

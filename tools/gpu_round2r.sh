#!/bin/bash
# GPU suite + configs[3] with and without slot-order gradients (env switch).
O=gpurun_out/${TAG:-r2r}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
A="--config 4 --no-cpu-baseline --e2e-steps 0 --steps 5"
for r in 1 2; do
  timeout 600 python bench.py $A > $O/cfg4_slot_$r.json 2>/dev/null
  GMI_SLOT_GRADS_MIN_N=2000000000 timeout 600 python bench.py $A > $O/cfg4_direct_$r.json 2>/dev/null
done
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 10 > $O/cfg3.json 2>/dev/null
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1].split('/')[-1], d['ms_per_step'], d.get('ms_per_step_median'), d['phases_ms_per_step'])
PY
done
CMD="python bench.py --config 4 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > $O/cfg4_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg4.csv $CMD > $O/ncu_cfg4.log 2>&1
python tools/launch_summary.py $O/launches_cfg4.csv | head -12

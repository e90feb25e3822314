#!/bin/bash
# GPU suite + shared-memory count vs RED count (env switch) at configs[1]/[2].
O=gpurun_out/${TAG:-r2w}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
for r in 1 2; do
  for c in 3 2; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 10 > $O/cfg${c}_smem_$r.json 2>/dev/null
    GMI_K1_COUNT_RED=1 timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 10 > $O/cfg${c}_red_$r.json 2>/dev/null
  done
done
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1].split('/')[-1], d['ms_per_step'], d.get('ms_per_step_median'), d['phases_ms_per_step'])
PY
done

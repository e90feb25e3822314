#!/bin/bash
# GPU suite + configs[2] / configs[3] phases on the current build.
O=gpurun_out/${TAG:-r2u}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 10 > $O/cfg3.json 2>/dev/null
timeout 600 python bench.py --config 4 --no-cpu-baseline --e2e-steps 0 --steps 5 > $O/cfg4.json 2>/dev/null
timeout 600 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 --steps 10 > $O/cfg2.json 2>/dev/null
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1].split('/')[-1], d['ms_per_step'], d.get('ms_per_step_median'), d['phases_ms_per_step'])
PY
done

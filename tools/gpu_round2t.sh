#!/bin/bash
# configs[2] with and without slot-order gradients (env switch).
O=gpurun_out/${TAG:-r2t}
mkdir -p $O
A="--no-cpu-baseline --e2e-steps 0 --steps 10"
for r in 1 2; do
  timeout 600 python bench.py $A > $O/cfg3_direct_$r.json 2>/dev/null
  GMI_SLOT_GRADS_MIN_N=1 timeout 600 python bench.py $A > $O/cfg3_slot_$r.json 2>/dev/null
done
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1].split('/')[-1], d['ms_per_step'], d.get('ms_per_step_median'), d['phases_ms_per_step'])
PY
done

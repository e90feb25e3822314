#!/bin/bash
# A/B of kernel variants on one box: the in-tree library and every
# build/variants/<name>/libgmi_b200.so, each timed by bench.py (config 3,
# phases per step), interleaved twice to expose drift.
O=gpurun_out/${TAG:-ab}
mkdir -p $O
ARGS=${ARGS:---no-cpu-baseline --e2e-steps 0 --steps 10}
for round in 1 2; do
  timeout 600 python bench.py $ARGS > $O/base_$round.json 2>/dev/null
  for d in build/variants/*/; do
    n=$(basename $d)
    GMI_LIBRARY=$d/libgmi_b200.so timeout 600 python bench.py $ARGS > $O/${n}_$round.json 2>/dev/null
  done
done
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(sys.argv[1].split('/')[-1], d['ms_per_step'], d.get('ms_per_step_median'), d['phases_ms_per_step'])
except Exception as e:
    print(sys.argv[1], 'failed', e)
PY
done

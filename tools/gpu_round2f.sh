#!/bin/bash
O=gpurun_out/${TAG:-r2f}
mkdir -p $O
TAG=${TAG:-r2f}/ab tools/ab_variants.sh
for c in 2 1; do timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > $O/bench_cfg$c.json 2>$O/bench_cfg$c.err; done
python -c "
import json
for c in (2, 1):
    d = json.load(open('$O/bench_cfg%d.json' % c)); print(c, d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['bound'], d['roofline']['step_frac'])"
python tools/prof_small.py 64 > $O/plain_b64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_gather|k_backward_points' -s 2 -c 2 -o $O/full_b64 python tools/prof_small.py 64 > $O/ncu_full.log 2>&1
tail -3 $O/ncu_full.log

#!/bin/bash
O=gpurun_out/${TAG:-r2c}
mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $O/bench3.json 2> $O/bench3.err
python -c "import json; d=json.load(open('$O/bench3.json')); print(d['ms_per_step'], d['value'], d['phases_ms_per_step'])" || tail -20 $O/bench3.err
timeout 900 python -m pytest tests/test_gpu_api_robustness.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
TAG=${TAG:-r2c}/san tools/gpu_sanitize.sh > /dev/null 2>&1; cat $O/san/summary.txt
S=${SECS:-300}
timeout $((S+120)) python tools/fuzz_parity.py --domain baseline --seconds $S --seed 31 --out $O/fail > $O/baseline.log 2>&1; echo "rc=$?" >> $O/baseline.log
timeout $((S+300)) python tools/fuzz_parity.py --domain baseline --large --seconds $S --seed 32 --out $O/fail > $O/baseline_large.log 2>&1; echo "rc=$?" >> $O/baseline_large.log
for f in $O/*.log; do echo "== $f"; grep -E "fuzz ok|FUZZ" $f; done

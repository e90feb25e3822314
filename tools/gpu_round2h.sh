#!/bin/bash
O=gpurun_out/${TAG:-r2h}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
timeout 900 python bench.py > $O/bench3.json 2> $O/bench3.err
python -c "import json; d=json.load(open('$O/bench3.json')); print(d['ms_per_step'], d['value'], d['phases_ms_per_step'], d['roofline']['frac'], d['roofline']['step_frac'], d['e2e']['value'], d['e2e']['numpy_shim'], d['cpu_baseline'])" || tail -5 $O/bench3.err
S=${SECS:-240}
timeout $((S+120)) python tools/fuzz_parity.py --domain baseline --seconds $S --seed 61 --out $O/fail > $O/fuzz_baseline.log 2>&1
timeout $((S+120)) python tools/fuzz_parity.py --domain stress --seconds $((S/2)) --seed 62 --out $O/fail --max-save 4 > $O/fuzz_stress.log 2>&1
timeout $((S+120)) python tools/fuzz_parity.py --domain stress --precise --seconds $((S/2)) --seed 63 --out $O/fail --max-save 4 > $O/fuzz_stress_precise.log 2>&1
for f in $O/fuzz*.log; do tail -1 $f; done

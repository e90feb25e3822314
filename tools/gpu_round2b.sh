#!/bin/bash
O=gpurun_out/${TAG:-r2b}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_api_robustness.py tests/test_gpu_cxx_api.py tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py tests/test_gpu_golden.py tests/test_gpu_sweep.py -q -rs > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $O/bench3.json 2> $O/bench3.err
python -c "import json; d=json.load(open('$O/bench3.json')); print(d['ms_per_step'], d['value'], d['phases_ms_per_step'], d['roofline']['bound'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['numpy_shim'])" || tail -20 $O/bench3.err
S=${SECS:-120}
timeout $((S+120)) python tools/fuzz_parity.py --domain contract --seconds $S --seed 21 --out $O/fail > $O/contract.log 2>&1; echo "rc=$?" >> $O/contract.log
timeout $((S+120)) python tools/fuzz_parity.py --domain contract --precise --seconds $S --seed 22 --out $O/fail > $O/contract_precise.log 2>&1; echo "rc=$?" >> $O/contract_precise.log
timeout $((S+120)) python tools/fuzz_parity.py --domain stress --precise --seconds $S --seed 23 --out $O/fail > $O/stress_precise.log 2>&1; echo "rc=$?" >> $O/stress_precise.log
timeout $((S+300)) python tools/fuzz_parity.py --domain contract --large --seconds $S --seed 24 --out $O/fail > $O/large.log 2>&1; echo "rc=$?" >> $O/large.log
for f in $O/*.log; do echo "== $f"; grep -E "fuzz ok|FUZZ" $f; done

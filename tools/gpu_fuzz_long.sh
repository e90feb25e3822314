#!/bin/bash
# Long strict fuzz on the final build + the full GPU suite
O=gpurun_out/${TAG:-fuzzlong}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 1500 python tools/fuzz_parity.py --domain baseline --seconds 1200 --seed 81 --out $O/fail > $O/fuzz_baseline.log 2>&1
timeout 1000 python tools/fuzz_parity.py --domain baseline --large --seconds 600 --seed 82 --out $O/fail > $O/fuzz_baseline_large.log 2>&1
timeout 700 python tools/fuzz_parity.py --domain contract --precise --seconds 480 --seed 83 --out $O/fail > $O/fuzz_contract_precise.log 2>&1
timeout 700 python tools/fuzz_parity.py --domain stress --precise --seconds 480 --seed 84 --out $O/fail > $O/fuzz_stress_precise.log 2>&1
timeout 400 python tools/fuzz_parity.py --domain contract --seconds 240 --seed 85 --out $O/fail --max-save 0 > $O/fuzz_contract_fp32.log 2>&1
for f in $O/fuzz_*.log; do tail -1 $f; done

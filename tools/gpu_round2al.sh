#!/bin/bash
# A/B against HEAD + GPU suite + strict fuzz of the current build.
O=gpurun_out/${TAG:-r2al}
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
TAG=$(basename $O)/ab tools/ab_variants.sh > $O/ab.txt 2>&1; cat $O/ab.txt
timeout 700 python tools/fuzz_parity.py --domain baseline --seconds 480 --seed 93 --out $O/fail > $O/fuzz_baseline.log 2>&1
timeout 400 python tools/fuzz_parity.py --domain contract --seconds 240 --seed 85 --out $O/fail --max-save 0 > $O/fuzz_contract_fp32.log 2>&1
for f in $O/fuzz_*.log; do tail -1 $f; done

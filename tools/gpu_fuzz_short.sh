#!/bin/bash
# Strict fuzz of the fp32 path after kernel changes: BASELINE regimes (must
# stay at 0 images over 1x) and the contract domain (documented envelope).
O=gpurun_out/${TAG:-fuzzshort}
mkdir -p $O
timeout 1100 python tools/fuzz_parity.py --domain baseline --seconds 900 --seed 91 --out $O/fail > $O/fuzz_baseline.log 2>&1
timeout 500 python tools/fuzz_parity.py --domain baseline --large --seconds 300 --seed 92 --out $O/fail > $O/fuzz_baseline_large.log 2>&1
timeout 400 python tools/fuzz_parity.py --domain contract --seconds 240 --seed 85 --out $O/fail --max-save 0 > $O/fuzz_contract_fp32.log 2>&1
for f in $O/fuzz_*.log; do tail -1 $f; done

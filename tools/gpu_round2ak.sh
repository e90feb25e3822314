#!/bin/bash
# fp32 cross-row position sums (variant): timing, GPU suite and strict fuzz.
O=gpurun_out/${TAG:-r2ak}
mkdir -p $O
V=$PWD/build/variants/bwd_rows_f32/libgmi_b200.so
TAG=$(basename $O)/ab tools/ab_variants.sh > $O/ab.txt 2>&1; cat $O/ab.txt
GMI_LIBRARY=$V timeout 600 python -m pytest tests -m gpu -q -k "not cxx" > $O/pytest_f32.log 2>&1; tail -3 $O/pytest_f32.log
GMI_LIBRARY=$V timeout 700 python tools/fuzz_parity.py --domain baseline --seconds 480 --seed 93 --out $O/fail > $O/fuzz_baseline_f32.log 2>&1
GMI_LIBRARY=$V timeout 400 python tools/fuzz_parity.py --domain contract --seconds 240 --seed 85 --out $O/fail --max-save 0 > $O/fuzz_contract_f32.log 2>&1
for f in $O/fuzz_*.log; do tail -1 $f; done

#!/bin/bash
O=gpurun_out/${TAG:-r2g}
mkdir -p $O
# correctness of the new gather layout first (variant library)
GMI_LIBRARY=$PWD/build/variants/rpl4/libgmi_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_sweep.py tests/test_gpu_baseline_configs.py tests/test_gpu_api_robustness.py -q -x -k "not cxx" > $O/pytest_rpl4.log 2>&1; echo "rc=$?" >> $O/pytest_rpl4.log; tail -2 $O/pytest_rpl4.log
GMI_LIBRARY=$PWD/build/variants/rpl4/libgmi_b200.so timeout 200 python tools/fuzz_parity.py --domain baseline --seconds 90 --seed 51 --out $O/fail > $O/fuzz_rpl4.log 2>&1; tail -1 $O/fuzz_rpl4.log
GMI_LIBRARY=$PWD/build/variants/rpl4/libgmi_b200.so timeout 200 python tools/fuzz_parity.py --domain contract --precise --seconds 60 --seed 52 --out $O/fail > $O/fuzz_rpl4p.log 2>&1; tail -1 $O/fuzz_rpl4p.log
TAG=${TAG:-r2g}/ab tools/ab_variants.sh

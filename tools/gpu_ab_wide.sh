#!/bin/bash
O=gpurun_out/${TAG:-abw}
mkdir -p $O
GMI_LIBRARY=$PWD/build/variants/wide_squad/libgmi_b200.so timeout 900 python -m pytest tests/test_gpu_baseline_configs.py tests/test_gpu_parity.py -q -x -k "configs4 or channel or deterministic or sweep or C5" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
GMI_LIBRARY=$PWD/build/variants/wide_squad/libgmi_b200.so timeout 400 python tools/fuzz_parity.py --domain baseline --seconds 120 --seed 71 --out $O/fail > $O/fuzz.log 2>&1; tail -1 $O/fuzz.log
GMI_LIBRARY=$PWD/build/variants/wide_squad/libgmi_b200.so timeout 400 python tools/fuzz_parity.py --domain stress --seconds 60 --seed 72 --out $O/fail --max-save 0 > $O/fuzz_stress.log 2>&1; tail -1 $O/fuzz_stress.log
ARGS="--config 5 --steps 3 --no-cpu-baseline --e2e-steps 0" TAG=${TAG:-abw}/ab tools/ab_variants.sh

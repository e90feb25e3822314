#!/bin/bash
# tests touched this round + strict fuzz
O=gpurun_out/${TAG:-r2a}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_api_robustness.py tests/test_gpu_cxx_api.py tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -x -rs > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
TAG=${TAG:-r2a} SECS=${SECS:-150} tools/gpu_fuzz.sh

#!/bin/bash
# GPU suite, A/B at configs[2] and configs[3], ncu --set full of the hot
# kernels at B = 64 on the current build.
O=gpurun_out/${TAG:-r2p}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
TAG=$(basename $O)/ab3 timeout 1200 tools/ab_variants.sh > $O/ab3.txt 2>&1; cat $O/ab3.txt
ARGS="--config 4 --no-cpu-baseline --e2e-steps 0 --steps 5" TAG=$(basename $O)/ab4 timeout 1200 tools/ab_variants.sh > $O/ab4.txt 2>&1; cat $O/ab4.txt




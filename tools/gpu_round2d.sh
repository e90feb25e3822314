#!/bin/bash
O=gpurun_out/${TAG:-r2d}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
TAG=${TAG:-r2d}/ab tools/ab_variants.sh

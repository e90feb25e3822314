#!/bin/bash
# GPU suite on the current build, A/B of the built variants, and the launch
# list of config 4 (one 8192^2 image; where its bin phase goes).
O=gpurun_out/${TAG:-r2o}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
TAG=$(basename $O)/ab timeout 1500 tools/ab_variants.sh > $O/ab.txt 2>&1; cat $O/ab.txt
CMD="python bench.py --config 4 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > $O/cfg4_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg4.csv $CMD > $O/ncu_cfg4.log 2>&1
tail -1 $O/cfg4_plain.json | cut -c1-400

#!/bin/bash
# ncu evidence at the bench's B = 64: the launch list of the bench and one
# --set full capture of the gather and the backward
O=gpurun_out/${TAG:-ncu}
mkdir -p $O
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv $CMD > $O/ncu_launch.log 2>&1
python tools/prof_small.py 64 > $O/plain_b64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_gather|k_backward_points|k_scatter_emit' -s 3 -c 3 -o $O/full_b64 python tools/prof_small.py 64 > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log

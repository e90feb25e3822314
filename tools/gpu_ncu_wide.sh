#!/bin/bash
O=gpurun_out/${TAG:-wide}
mkdir -p $O
python tools/prof_cfg5.py 1 > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_gather_wide|k_backward_wide' -s 2 -c 2 -o $O/full_wide python tools/prof_cfg5.py 1 > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log

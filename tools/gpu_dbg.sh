#!/bin/bash
# debugging pass: a test subset (K=...) plus the ncu launch list of a small run
O=gpurun_out/${TAG:-dbg}
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "${K:-batch_equals}" > $O/pytest_k.log 2>&1; echo "rc=$?" >> $O/pytest_k.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/launches.csv python tools/prof_small.py 8 > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1 || true
tail -5 $O/pytest_k.log; cat $O/launch_summary.txt | head -30

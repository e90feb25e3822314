#!/bin/bash
# bounds-checked debug build over the GPU suite, saved-case replays, a
# 30-minute strict fuzz, and the ncu evidence at the bench's B = 64
O=gpurun_out/${TAG:-r2e}
mkdir -p $O
TAG=${TAG:-r2e}/bounds tools/gpu_bounds.sh
timeout 600 python -m pytest tests/test_gpu_fuzz_cases.py -q > $O/pytest_cases.log 2>&1; echo "rc=$?" >> $O/pytest_cases.log; tail -2 $O/pytest_cases.log
S=${SECS:-600}
timeout $((S+120)) python tools/fuzz_parity.py --domain baseline --seconds $S --seed 41 --out $O/fail > $O/fuzz_baseline.log 2>&1; echo "rc=$?" >> $O/fuzz_baseline.log
timeout $((S/2+300)) python tools/fuzz_parity.py --domain baseline --large --seconds $((S/2)) --seed 42 --out $O/fail > $O/fuzz_baseline_large.log 2>&1; echo "rc=$?" >> $O/fuzz_baseline_large.log
timeout $((S/2+120)) python tools/fuzz_parity.py --domain contract --precise --seconds $((S/2)) --seed 43 --out $O/fail > $O/fuzz_contract_precise.log 2>&1; echo "rc=$?" >> $O/fuzz_contract_precise.log
timeout $((S/2+120)) python tools/fuzz_parity.py --domain stress --precise --seconds $((S/2)) --seed 44 --out $O/fail > $O/fuzz_stress_precise.log 2>&1; echo "rc=$?" >> $O/fuzz_stress_precise.log
timeout $((S/4+120)) python tools/fuzz_parity.py --domain contract --seconds $((S/4)) --seed 45 --out $O/fail --max-save 0 > $O/fuzz_contract_fp32.log 2>&1; echo "rc=$?" >> $O/fuzz_contract_fp32.log
for f in $O/fuzz_*.log; do grep -E "fuzz ok|FUZZ" $f; done
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv $CMD > $O/ncu_launch.log 2>&1
python tools/prof_small.py 64 > $O/plain_b64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_gather<|k_backward_points<|k_scatter_emit|k_count_red|k_bbox_validate4' -s 7 -c 5 -o $O/full_b64 python tools/prof_small.py 64 > $O/ncu_full.log 2>&1
ls -la $O

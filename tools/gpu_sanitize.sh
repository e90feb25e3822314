#!/bin/bash
# compute-sanitizer over every hot-path kernel family (tools/sanitize_case.py)
O=gpurun_out/${TAG:-sanitize}
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  for mode in fast1 fast3 fast4 wide generic precise cluster sparse async bins; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_case.py $mode > $O/${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok' $O/${tool}_${mode}.log | tr '\n' ' ')" | tee -a $O/summary.txt
  done
done

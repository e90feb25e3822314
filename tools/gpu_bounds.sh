#!/bin/bash
# The GPU test suite against the bounds-checked debug build
# (build/debug/bounds, -DGMI_DEBUG_BOUNDS: every staging / list / scatter
# index of the hot kernels checked on the device, a violation traps).
# compute-sanitizer is closed on this pool; this is its stand-in.
O=gpurun_out/${TAG:-bounds}
mkdir -p $O
GMI_LIBRARY=$PWD/build/debug/bounds/libgmi_b200.so timeout 1800 python -m pytest tests -m gpu -q \
  -k "not cxx" > $O/pytest_bounds.log 2>&1; echo "pytest rc=$?" >> $O/pytest_bounds.log
grep -c "GMI_CHECK failed" $O/pytest_bounds.log; tail -3 $O/pytest_bounds.log
for mode in fast1 fast3 fast4 wide generic precise cluster sparse async bins; do
  GMI_LIBRARY=$PWD/build/debug/bounds/libgmi_b200.so timeout 300 python tools/sanitize_case.py $mode > $O/case_$mode.log 2>&1
  echo "$mode rc=$? $(tail -1 $O/case_$mode.log)" | tee -a $O/summary.txt
done

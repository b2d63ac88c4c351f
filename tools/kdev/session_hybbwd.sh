#!/bin/bash
# A/B: the backward of the hybrid launch split like the forward (WHIT_HYB_BWD=1) vs one sequential launch
out=gpurun_out/ab_hybbwd.log
: > $out
for rep in 1 2 3; do
  for v in 0 1; do
    for qb in 65536 61440 73728; do
      echo "### HYB_BWD=$v homo B=$qb rep=$rep" >> $out
      WHIT_HYB_BWD=$v QT_B=$qb timeout 300 python tools/quick_time.py homo >> $out 2>&1
      echo "### HYB_BWD=$v hetero B=$qb rep=$rep" >> $out
      WHIT_HYB_BWD=$v QT_B=$qb timeout 300 python tools/quick_time.py hetero >> $out 2>&1
    done
  done
done
WHIT_HYB_BWD=1 python -m pytest tests -q -m gpu -x -k "hybrid" > gpurun_out/hybbwd_tests.log 2>&1
tail -1 gpurun_out/hybbwd_tests.log

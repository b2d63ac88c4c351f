#!/bin/bash
# re-tune the hybrid launch's sequential share (WHIT_HYB_G1) after the twisted-kernel changes
out=gpurun_out/g1tune.log
: > $out
for rep in 1 2; do
  for g1 in 1376 1504 1632 1728; do
    for cfg in homo hetero; do
      for qb in 65536 61440; do
        echo "### G1=$g1 $cfg B=$qb rep=$rep" >> $out
        WHIT_HYB_G1=$g1 QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
      done
    done
  done
done

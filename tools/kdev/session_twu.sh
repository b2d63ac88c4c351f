#!/bin/bash
# A/B: partial unroll of the twisted up sweep (code size / instruction cache)
out=gpurun_out/ab_twu.log
: > $out
for rep in 1 2; do
  for lib in libwhit.so libwhit_u4.so libwhit_u2.so; do
    for qb in 8192 16384; do
      for cfg in hetero homo; do
        echo "### $lib $cfg B=$qb rep=$rep" >> $out
        WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
      done
    done
  done
done

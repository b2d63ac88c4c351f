#!/bin/bash
# timing split of the twisted kernel: all but the down sweep (WHIT_TW_STAGE=5 build) vs the full kernel
out=gpurun_out/twsplit.log
: > $out
for lib in libwhit.so libwhit_s5.so; do
  for qb in 8192 16384; do
    for cfg in hetero homo; do
      echo "### $lib $cfg B=$qb" >> $out
      WHIT_TWIST=1 WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
    done
  done
done

#!/bin/bash
# A/B: twisted kernel at 255 registers (no spills; fewer warps per SM) vs 168, by batch size
out=gpurun_out/ab_tw255.log
: > $out
for rep in 1 2; do
  for lib in libwhit.so libwhit_tw255.so; do
    for qb in 8192 16384 24576; do
      for cfg in hetero homo; do
        echo "### $lib $cfg B=$qb rep=$rep" >> $out
        WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
      done
    done
    echo "### $lib homo rep=$rep" >> $out
    WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_time.py homo >> $out 2>&1
  done
done

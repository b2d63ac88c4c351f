#!/bin/bash
# A/B: ring depth of the scalar-lambda layouts (WHIT_TILE_ST_S / WHIT_BWD_WB_ST_S) on homo-shaped batches
out=gpurun_out/ab_st.log
: > $out
for rep in 1 2; do
for lib in libwhit.so libwhit_st3.so libwhit_st34.so; do
  for hyb in auto 0; do
    for qb in 65536 262144; do
      echo "### $lib hybrid=$hyb B=$qb rep=$rep" >> $out
      if [ $hyb = auto ]; then
        WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib QT_B=$qb timeout 300 python tools/quick_time.py homo >> $out 2>&1
      else
        WHIT_HYBRID=0 WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib QT_B=$qb timeout 300 python tools/quick_time.py homo >> $out 2>&1
      fi
    done
  done
done
done

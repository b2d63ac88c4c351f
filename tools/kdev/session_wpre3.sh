#!/bin/bash
# A/B: bit words prefetched two chunks ahead (WHIT_WPRE2=1) vs one
out=gpurun_out/ab_wpre3.log
: > $out
for rep in 1 2 3; do
  for lib in libwhit.so libwhit_p2.so; do
    for cfg in hetero homo; do
      echo "### $lib $cfg rep=$rep" >> $out
      WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
    done
  done
done

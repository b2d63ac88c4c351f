#!/bin/bash
# A/B: shared-factor kernel's factor warp -- checkpoints two chunks ahead (a2), backward factor ring 4 deep (f4)
out=gpurun_out/ab_mb2f.log
: > $out
for rep in 1 2; do
  bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_a2.so libwhit_f4.so libwhit_a2f4.so -- --config s2tile --steps 10 --warmup 3 --no-e2e
  bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_a2.so libwhit_f4.so libwhit_a2f4.so -- --op table1 --steps 20 --warmup 5 --no-e2e
done
for lib in libwhit.so libwhit_a2f4.so; do
  for C in 2 4 10; do
    echo "### $lib quick_bands C=$C" >> $out
    WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 600 python tools/quick_bands.py $C >> $out 2>&1
  done
done

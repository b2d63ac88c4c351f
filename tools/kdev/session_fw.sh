#!/bin/bash
# A/B: the shared-factor kernel's factor-warp index (its scheduler): last (default) vs 0..3
out=gpurun_out/ab_fw.log
: > $out
for rep in 1 2; do
  bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_fw0.so libwhit_fw2.so -- --op table1 --steps 20 --warmup 5 --no-e2e
  bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_fw0.so libwhit_fw2.so -- --config s2tile --steps 10 --warmup 3 --no-e2e
done

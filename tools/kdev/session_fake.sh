#!/bin/bash
# timing probe: the shared-factor kernels with the factor warp's arithmetic removed (how much it paces them)
out=gpurun_out/ab_fake.log
: > $out
bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_fake.so libwhit.so libwhit_fake.so -- --op table1 --steps 20 --warmup 5 --no-e2e
bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_fake.so -- --config s2tile --steps 10 --warmup 3 --no-e2e

#!/bin/bash
# shared-factor backward: the per-date dL/dlambda band reduction with one barrier per two chunks (RED2) vs per chunk
python -m pytest tests -q -m gpu -x -k "bands or s2tile or table1 or irregular_full" > gpurun_out/red2_tests.log 2>&1
tail -1 gpurun_out/red2_tests.log
out=gpurun_out/ab_red2.log
: > $out
for rep in 1 2; do
  bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_r1.so -- --config s2tile --steps 10 --warmup 3 --no-e2e
  bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_r1.so -- --op table1 --steps 20 --warmup 5 --no-e2e
done

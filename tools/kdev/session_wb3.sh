#!/bin/bash
# A/B: 3-stage ring for the bit-packed backward body (WHIT_BWD_WB_ST=3, per-warp allocation the larger body's)
out=gpurun_out/ab_wb3.log
: > $out
for rep in 1 2 3; do
  for lib in libwhit.so libwhit_wb3.so; do
    for cfg in hetero homo; do
      echo "### $lib $cfg rep=$rep" >> $out
      WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
    done
  done
done
bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_wb3.so libwhit.so libwhit_wb3.so -- --steps 20 --warmup 5 --no-e2e --no-extras --no-cpu-baseline
WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/libwhit_wb3.so python -m pytest tests -q -m gpu -x -k "wdet or guard or status or parity" > gpurun_out/wb3_tests.log 2>&1
tail -2 gpurun_out/wb3_tests.log

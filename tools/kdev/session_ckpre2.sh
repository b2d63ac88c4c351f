#!/bin/bash
# A/B (twisted, scalar-lambda forward back to its at-the-chunk checkpoint loads) + twisted / guard tests
out=gpurun_out/ab_ckpre2.log
: > $out
for rep in 1 2; do
  for lib in libwhit.so libwhit_old.so; do
    for qb in 8192 16384 28416; do
      for cfg in hetero homo; do
        echo "### $lib $cfg B=$qb rep=$rep" >> $out
        WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
      done
    done
  done
done
python -m pytest tests -q -m gpu -x -k "twist or guard or status or hybrid" > gpurun_out/ckpre2_tests.log 2>&1
tail -2 gpurun_out/ckpre2_tests.log

#!/bin/bash
# A/B: checkpoint prefetch in the 255-register scalar-lambda twisted forward
out=gpurun_out/ab_twck.log
: > $out
for rep in 1 2; do
  for lib in libwhit.so libwhit_old.so; do
    for qb in 8192 16384; do
      echo "### $lib homo B=$qb rep=$rep" >> $out
      WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib QT_B=$qb timeout 300 python tools/quick_time.py homo >> $out 2>&1
    done
    echo "### $lib homo rep=$rep" >> $out
    WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_time.py homo >> $out 2>&1
  done
done
python -m pytest tests -q -m gpu -x -k "twist" > gpurun_out/twck_tests.log 2>&1; tail -1 gpurun_out/twck_tests.log

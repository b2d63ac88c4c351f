#!/bin/bash
# full GPU suite on the predicated bit-word loads; A/B vs the previous build (hetero, homo, d = 3, fp64)
python -m pytest tests -q -m gpu -x > gpurun_out/wpre2_tests.log 2>&1
tail -2 gpurun_out/wpre2_tests.log
out=gpurun_out/ab_wpre2.log
: > $out
for rep in 1 2; do
  for lib in libwhit.so libwhit_old.so; do
    for cfg in hetero homo; do
      echo "### $lib $cfg rep=$rep" >> $out
      WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
    done
    echo "### $lib hetero f64 rep=$rep" >> $out
    WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_time.py hetero f64 >> $out 2>&1
    echo "### $lib d3 rep=$rep" >> $out
    WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_d.py 3 >> $out 2>&1
  done
done

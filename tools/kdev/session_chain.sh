#!/bin/bash
# A/B: the loop-carried chains (factor recurrence, back substitution) shortened by one op vs the previous build
out=gpurun_out/ab_chain3.log
: > $out
for rep in 1 2; do
  for lib in libwhit.so libwhit_old.so; do
    for qb in 8192 16384; do
      for cfg in hetero homo; do
        echo "### $lib $cfg B=$qb rep=$rep" >> $out
        WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
      done
    done
    for cfg in hetero homo; do
      echo "### $lib $cfg rep=$rep" >> $out
      WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
    done
  done
done
bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_old.so libwhit.so libwhit_old.so -- --op table1 --steps 20 --warmup 5 --no-e2e
bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_old.so libwhit.so libwhit_old.so -- --config s2tile --steps 10 --warmup 3 --no-e2e
bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_old.so -- --op irregular --steps 20 --warmup 5 --no-e2e
python -m pytest tests -q -m gpu > gpurun_out/chain3_tests.log 2>&1
tail -3 gpurun_out/chain3_tests.log

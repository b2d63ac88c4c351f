#!/bin/bash
# A/B: bit-plane word loaded a chunk ahead with the extraction at the use (new) vs at the load (old)
out=gpurun_out/ab_wpre.log
: > $out
for rep in 1 2 3; do
  for lib in libwhit.so libwhit_old.so; do
    for cfg in hetero homo; do
      echo "### $lib $cfg rep=$rep" >> $out
      WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
    done
  done
done
bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_old.so -- --steps 20 --warmup 5 --no-e2e --no-extras --no-cpu-baseline
python -m pytest tests/test_gpu_wdet.py tests/test_gpu_status.py tests/test_gpu_guards.py -q -x > gpurun_out/wpre_tests.log 2>&1
tail -2 gpurun_out/wpre_tests.log

#!/bin/bash
for lib in libwhit.so libwhit_t200.so libwhit_tst.so; do
  echo "### $lib" >> gpurun_out/qt_tw2.log
  for B in 65536 8192; do
    WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib WHIT_TWIST=1 QT_B=$B python tools/quick_time.py homo >> gpurun_out/qt_tw2.log 2>&1
  done
  WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib WHIT_TWIST=1 QT_B=65536 python tools/quick_time.py hetero >> gpurun_out/qt_tw2.log 2>&1
done
python -m pytest tests/test_gpu_twist.py -m gpu -q > gpurun_out/t_twist.log 2>&1
tail -n 3 gpurun_out/t_twist.log

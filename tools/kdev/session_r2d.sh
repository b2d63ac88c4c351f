#!/bin/bash
python -m pytest tests/test_gpu_twist.py -m gpu -q -x > gpurun_out/t_twist.log 2>&1
for tw in 0 1; do
  for B in 65536 8192 131072; do
    WHIT_TWIST=$tw QT_B=$B python tools/quick_time.py homo >> gpurun_out/qt_twist.log 2>&1
  done
  WHIT_TWIST=$tw QT_B=65536 python tools/quick_time.py hetero >> gpurun_out/qt_twist.log 2>&1
done
tail -n 3 gpurun_out/t_twist.log

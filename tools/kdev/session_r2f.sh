#!/bin/bash
for cfg in homo hetero; do for B in 8192 16384 32768 65536 98304; do for tw in 0 1; do
  echo -n "tw=$tw " >> gpurun_out/qt_tw3.log
  WHIT_TWIST=$tw QT_B=$B python tools/quick_time.py $cfg 2>&1 | grep -v nfail >> gpurun_out/qt_tw3.log
done; done; done
python -m pytest tests/test_gpu_twist.py -m gpu -q > gpurun_out/t_twist.log 2>&1
tail -n 3 gpurun_out/t_twist.log

#!/bin/bash
for lib in "$@"; do for cfg in homo hetero; do for B in 8192 16384; do
  echo -n "$lib " >> gpurun_out/qt_twab.log
  WHIT_TWIST=1 QT_B=$B WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib python tools/quick_time.py $cfg 2>&1 | grep -v nfail | cut -c1-140 >> gpurun_out/qt_twab.log
done; done; done
cat gpurun_out/qt_twab.log

#!/bin/bash
# A/B of dev builds: session_ab.sh <lib>... (quick_time hetero + homo per lib, twice)
for rep in 1 2; do for lib in "$@"; do
  echo -n "$lib " >> gpurun_out/qt_ab.log
  WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib python tools/quick_time.py hetero 2>&1 | grep -v nfail >> gpurun_out/qt_ab.log
  echo -n "$lib " >> gpurun_out/qt_ab.log
  WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib python tools/quick_time.py homo 2>&1 | grep -v nfail >> gpurun_out/qt_ab.log
done; done
cut -c1-150 gpurun_out/qt_ab.log

#!/bin/bash
# backward register/occupancy experiment + launch list of the bench command
for lib in libwhit.so libwhit_b168.so libwhit_bst.so; do
  for wb in 0 1; do
    echo "### $lib WHIT_WBITS=$wb" >> gpurun_out/qt_b168.log
    WHIT_WBITS=$wb WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib python tools/quick_time.py hetero >> gpurun_out/qt_b168.log 2>&1
    WHIT_WBITS=$wb WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib python tools/quick_time.py homo >> gpurun_out/qt_b168.log 2>&1
  done
done
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_list.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:whit -c 60 --csv \
    --log-file gpurun_out/r2_launches_whit.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1

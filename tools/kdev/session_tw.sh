#!/bin/bash
for st in 1 2 3 4; do
  timeout 120 env WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/libwhit_tw$st.so python tools/kdev/tw_stage.py >> gpurun_out/tw_stage.log 2>&1
done
timeout 120 python tools/kdev/tw_stage.py >> gpurun_out/tw_stage.log 2>&1
cat gpurun_out/tw_stage.log

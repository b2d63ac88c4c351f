#!/bin/bash
# A/B: factor warp's stencil pass (WHIT_MB2_IRR_SPASS) on the Table 1 workload; parity of the irregular bands
out=gpurun_out/ab_spass.log
: > $out
for rep in 1 2 3; do
  bash tools/kdev/gpu_ab.sh $out libwhit.so libwhit_sp0.so -- --op table1 --steps 20 --warmup 5
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_status.py -q -x -k "irregular or times or bands" > gpurun_out/spass_tests.log 2>&1
tail -2 gpurun_out/spass_tests.log

#!/bin/bash
# the pipelined twisted down sweep: tests (twisted path, guards, status, hybrid) and timing vs WHIT_TW_PIPE=0
timeout 900 python -m pytest tests -q -m gpu -x -k "twist or guard or status or hybrid or toy" > gpurun_out/pipe_tests.log 2>&1
tail -3 gpurun_out/pipe_tests.log
out=gpurun_out/ab_pipe.log
: > $out
for rep in 1 2; do
  for pipe in 1 0; do
    for qb in 4096 8192 9472 16384; do
      for cfg in hetero homo; do
        echo "### PIPE=$pipe $cfg B=$qb rep=$rep" >> $out
        WHIT_TW_PIPE=$pipe QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
      done
    done
  done
done

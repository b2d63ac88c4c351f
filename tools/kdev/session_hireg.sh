#!/bin/bash
# twisted kernel: 255-register build for one-wave launches (<= 592 groups); tests + timing by batch size
python -m pytest tests -q -m gpu -x -k "twist or guard or status or hybrid" > gpurun_out/hireg_tests.log 2>&1
tail -1 gpurun_out/hireg_tests.log
out=gpurun_out/hireg_time.log
: > $out
for qb in 8192 16384 18944 24576; do
  for cfg in hetero homo; do
    echo "### $cfg B=$qb" >> $out
    QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
  done
done
echo "### homo" >> $out; timeout 300 python tools/quick_time.py homo >> $out 2>&1
echo "### d3 8192" >> $out; WHIT_TWIST=1 timeout 300 python tools/quick_d.py 3 3288 8192 >> $out 2>&1
echo "### d3 8192 seq" >> $out; WHIT_TWIST=0 timeout 300 python tools/quick_d.py 3 3288 8192 >> $out 2>&1

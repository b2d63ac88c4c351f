#!/bin/bash
# re-tune the twisted / sequential / hybrid thresholds after the checkpoint prefetch
out=gpurun_out/twtune.log
: > $out
for qb in 20480 24576 28416 32768 40960 49152 57344 65536; do
  for cfg in hetero homo; do
    for mode in 0 1 auto; do
      echo "### $cfg B=$qb twist=$mode" >> $out
      if [ $mode = auto ]; then QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1
      else WHIT_TWIST=$mode QT_B=$qb timeout 300 python tools/quick_time.py $cfg >> $out 2>&1; fi
    done
  done
done

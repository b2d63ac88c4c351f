#!/bin/bash
# launch lists (time + DRAM bytes per launch) of the NEXT-row workloads: checks the byte models of bench.py
for op in "--op irregular" "--op table1" "--op variance" "--op train" "--config s2tile" "--config homo"; do
  tag=$(echo $op | tr -d ' -')
  python bench.py $op --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:whit -c 40 --csv \
      --log-file gpurun_out/r2_launches_${tag}_whit.csv python bench.py $op --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
done
ls gpurun_out/r2_launches_*

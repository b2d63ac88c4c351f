#!/bin/bash
# round-2 evidence after the load-wait fixes: bench lines of every workload (+ reference arm), launch lists
python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
python bench.py > gpurun_out/r2j_bench_rep.json 2>> gpurun_out/r2j_bench.err
python bench.py --steps 20 --warmup 5 > gpurun_out/r2j_bench_20.json 2>> gpurun_out/r2j_bench.err
: > gpurun_out/r2j_bench_extra.jsonl
for a in "--config homo" "--op train" "--op variance" "--op irregular" "--op table1" "--config s2tile" \
         "--io f64 --no-e2e --no-cpu-baseline" "--config toy --no-cpu-baseline"; do
  python bench.py $a --steps 20 >> gpurun_out/r2j_bench_extra.jsonl 2>> gpurun_out/r2j_bench_extra.err
done
python bench.py --config s2tile --scaling strong --steps 3 --no-e2e >> gpurun_out/r2j_bench_extra.jsonl 2>> gpurun_out/r2j_bench_extra.err
python bench.py --impl reference --steps 2 --warmup 3 >> gpurun_out/r2j_bench_extra.jsonl 2>> gpurun_out/r2j_bench_extra.err
for op in "" "--op irregular" "--op table1" "--op variance" "--op train" "--config s2tile" "--config homo"; do
  tag=$(echo "x$op" | tr -d ' -')
  python bench.py $op --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2j_plain_$tag.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:whit -c 60 --csv \
      --log-file gpurun_out/r2j_launches_${tag}_whit.csv python bench.py $op --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2j_ncu_$tag.log 2>&1
done
python tools/bench_summary.py gpurun_out/r2j_bench.json gpurun_out/r2j_bench_extra.jsonl

#!/bin/bash
# round-2 evidence: bench lines of every workload (+ the reference arm), launch list, one full ncu capture
python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err
for a in "--config homo" "--op train" "--op variance" "--op irregular" "--op table1" "--config s2tile" \
         "--io f64 --no-e2e --no-cpu-baseline" "--config toy --no-cpu-baseline"; do
  python bench.py $a --steps 20 >> gpurun_out/r2_bench_extra.jsonl 2>> gpurun_out/r2_bench_extra.err
done
python bench.py --config s2tile --scaling strong --steps 3 --no-e2e >> gpurun_out/r2_bench_extra.jsonl 2>> gpurun_out/r2_bench_extra.err
python bench.py --impl reference --steps 2 --warmup 3 >> gpurun_out/r2_bench_extra.jsonl 2>> gpurun_out/r2_bench_extra.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_list.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:whit -c 60 --csv \
    --log-file gpurun_out/r2_launches_final_whit.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
python tools/quick_time.py hetero > gpurun_out/qt_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:whit_kernel -s 6 -c 2 -o gpurun_out/r2_full_final \
    python tools/quick_time.py hetero > gpurun_out/ncu_full.log 2>&1
python tools/bench_summary.py gpurun_out/r2_bench_final.json gpurun_out/r2_bench_extra.jsonl

#!/bin/bash
# round-2 evidence refresh: default bench twice (variance), every workload line, reference arm
python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_final_rep.json 2>> gpurun_out/r2_bench_final.err
rm -f gpurun_out/r2_bench_extra.jsonl
for a in "--config homo" "--op train" "--op variance" "--op irregular" "--op table1" "--config s2tile" \
         "--io f64 --no-e2e --no-cpu-baseline" "--config toy --no-cpu-baseline"; do
  python bench.py $a --steps 20 >> gpurun_out/r2_bench_extra.jsonl 2>> gpurun_out/r2_bench_extra.err
done
python bench.py --config s2tile --scaling strong --steps 3 --no-e2e >> gpurun_out/r2_bench_extra.jsonl 2>> gpurun_out/r2_bench_extra.err
python bench.py --config homo --scaling strong --gpus 1 --steps 20 --no-e2e --no-cpu-baseline >> gpurun_out/r2_bench_extra.jsonl 2>> gpurun_out/r2_bench_extra.err
python bench.py --impl reference --steps 2 --warmup 3 >> gpurun_out/r2_bench_extra.jsonl 2>> gpurun_out/r2_bench_extra.err
python bench_sweep.py --Ts 128,1024,3288,8192 --masks bernoulli,s2 > gpurun_out/r2_sweep.jsonl 2> gpurun_out/r2_sweep.err
python tools/bench_summary.py gpurun_out/r2_bench_final.json gpurun_out/r2_bench_final_rep.json gpurun_out/r2_bench_extra.jsonl

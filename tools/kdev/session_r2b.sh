#!/bin/bash
# round-2 evidence session: GPU tests, the default bench line, ncu launch list + one full capture.
python -m pytest tests/test_gpu_guards.py -m gpu -q > gpurun_out/t_guards.log 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1
python bench.py > gpurun_out/b_full.log 2> gpurun_out/b_full.err
python tools/quick_time.py hetero > gpurun_out/qt_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
python tools/quick_time.py hetero > gpurun_out/qt_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:whit_kernel -s 6 -c 2 -o gpurun_out/r2_full \
    python tools/quick_time.py hetero > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/t_guards.log gpurun_out/t_all.log

python -m pytest tests/test_gpu_wdet.py -m gpu -q > gpurun_out/t_wdet.log 2>&1
A=tools/kdev/gpu_ab.sh
$A gpurun_out/ab_bwd.log libwhit.so libwhit_bst.so -- --steps 20 --no-e2e --no-cpu-baseline --no-extras
$A gpurun_out/ab_bwd.log libwhit.so libwhit_bst.so -- --config homo --steps 30 --no-e2e --no-cpu-baseline
WHIT_WDET=0 $A gpurun_out/ab_bwd.log libwhit.so libwhit_bst.so -- --steps 20 --no-e2e --no-cpu-baseline --no-extras
$A gpurun_out/ab_mb2.log libwhit.so libwhit_st3.so libwhit_st4.so -- --config s2tile --steps 5 --no-e2e
$A gpurun_out/ab_mb2.log libwhit.so libwhit_st3.so libwhit_st4.so -- --op table1 --steps 10
timeout 900 python bench_sweep.py --accuracy --Ts 128,1024,3288,8192 > gpurun_out/sweep_acc.jsonl 2> gpurun_out/sweep_acc.err
for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/diag/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool.log; done
tail -n 3 gpurun_out/t_wdet.log

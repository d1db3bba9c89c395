timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/gpu_tests_9.txt
timeout 300 python tools/attn_sweep.py > gpurun_out/sweep_v8.txt 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/bench_9.txt 2>&1
cat gpurun_out/gpu_tests_9.txt gpurun_out/sweep_v8.txt; tail -1 gpurun_out/bench_9.txt

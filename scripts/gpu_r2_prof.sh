# round-2 profiling pass: GPU tests, default bench line, ncu full (warp states, source counters) of the hot kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:quantize_kernel|reduce_kernel|norm_kernel" -s 3 -c 3 -o gpurun_out/prof_c2 python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e --no-fp32 > gpurun_out/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:quantize_kernel|reduce_kernel" -s 200 -c 2 -o gpurun_out/prof_c4 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-fp32 --overlap 0 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c2.log gpurun_out/ncu_c4.log
ls -la gpurun_out

# one ncu --set full capture of the hot kernels (single GPU, short bench)
mkdir -p gpurun_out
TAG=${TAG:-v}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-quantize_kernel|reduce_kernel|norm_kernel}" -s ${SKIP:-3} -c ${COUNT:-3} -o gpurun_out/prof_${TAG} python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
ls -la gpurun_out/

# bench each tuning variant in build/variants (kernel times only), c2 and c4
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=short -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1
tail -2 gpurun_out/pytest_quick.log
for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  for wl in c2 c4; do
    if [ $wl = c4 ]; then A="--workload c4 --steps 10 --warmup 3"; else A="--steps 200 --warmup 5"; fi
    GQ_B200_LIB=$PWD/$lib timeout 300 python bench.py $A --no-cpu --no-e2e --no-fp32 > gpurun_out/bench_${v}_$wl.json 2>gpurun_out/bench_${v}_$wl.err
    python -c "
import json
l=json.load(open('gpurun_out/bench_${v}_$wl.json'))
print('$v $wl', 'ms/step %.4f'%l['ms_per_step'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in l['kernels'].items()))
" || tail -3 gpurun_out/bench_${v}_$wl.err
  done
done

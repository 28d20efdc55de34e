# every build/variants/lib_*.so on C2 and C4 (bench step + per-kernel CUDA-event times), twice
mkdir -p gpurun_out
for rep in 1 2; do
for wl in ${WLS:-c2 c4}; do
for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  GQ_B200_LIB=$PWD/$lib timeout 300 python bench.py --workload $wl --steps ${STEPS:-100} --warmup 5 --no-cpu --no-e2e --no-fp32 > gpurun_out/bv.json 2>gpurun_out/bv.err
  python -c "
import json
l=json.load(open('gpurun_out/bv.json'))
print('$wl $v', 'ms/step %.4f'%l['ms_per_step'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in l['kernels'].items()))
" || tail -3 gpurun_out/bv.err
done; done; done

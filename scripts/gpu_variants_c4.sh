# per-variant C4 step and kernel times (libraries from build/variants/)
mkdir -p gpurun_out
for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  GQ_B200_LIB=$PWD/$lib timeout 300 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu --no-e2e --no-fp32 > gpurun_out/bv4.json 2>gpurun_out/bv4.err
  python -c "
import json
l=json.load(open('gpurun_out/bv4.json'))
print('$v', 'ms/step %.4f'%l['ms_per_step'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in l['kernels'].items()))
" || tail -3 gpurun_out/bv4.err
done

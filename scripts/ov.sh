mkdir -p gpurun_out
for cfg in "--overlap 0" "--overlap 1" "--overlap 2" "--overlap 2 --reduce-ctas 1" "--overlap 2 --reduce-ctas 2"; do
  timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-fp32 $cfg > gpurun_out/ov.json 2> gpurun_out/ov.err
  python -c "
import json
l=json.load(open('gpurun_out/ov.json'))
print('$cfg', 'ms/step %.3f'%l['ms_per_step'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in l['kernels'].items()))
" || tail -3 gpurun_out/ov.err
done

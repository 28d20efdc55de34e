# per-variant step times of the launch-sensitive workloads (libraries from build/variants/)
for w in c1 c2 c3n2; do for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  GQ_B200_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps 200 --warmup 5 --no-cpu --no-e2e --no-fp32 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read())
print('$w $v', 'ms/step %.4f'%l['ms_per_step'], 'graph', l['config']['cuda_graph'])
"
done; done

# quick GPU loop: parity subset + kernel timings (no CPU baseline / e2e)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=short -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_quick.log 2>&1
tail -3 gpurun_out/pytest_quick.log
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'PY'
import json
l=json.load(open('gpurun_out/bench_quick.json'))
print('ms/step', l['ms_per_step'], 'value', '%.3e'%l['value'])
for k,v in l['kernels'].items(): print(k, '%.4f ms'%v['ms'], '%.0f GB/s'%v['gbs'], '%.3f'%v['frac'])
print(l['clocks'])
PY
tail -3 gpurun_out/bench_quick.err

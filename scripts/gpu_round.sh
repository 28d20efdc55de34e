# full GPU pass: parity + dist tests, smoke, bench lines (c2 inproc, c2 dist-engine, c4)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --steps 50 --warmup 5 --engine dist --no-cpu > gpurun_out/bench_c2_dist.json 2> gpurun_out/bench_c2_dist.err
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --engine dist --exchange nccl_sum --no-cpu --no-e2e > gpurun_out/bench_c4_dist.json 2> gpurun_out/bench_c4_dist.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
for f in gpurun_out/bench_*.json; do echo "== $f"; head -c 600 $f; echo; done
for f in gpurun_out/bench_*.err; do echo "== $f"; tail -5 $f; done

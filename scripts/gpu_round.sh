# full GPU pass: parity + dist + drop-in tests, smoke, bench lines, launch list, ncu full captures
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --workload c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 300 python bench.py --engine dist --exchange p2p --steps 50 --no-cpu > gpurun_out/bench_c2_dist_p2p.json 2> gpurun_out/bench_c2_dist_p2p.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:norm_kernel|quantize_kernel|reduce_kernel" -s 3 -c 3 -o gpurun_out/prof_c2 python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e --no-fp32 > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:norm_kernel|quantize_kernel|reduce_kernel" -s 3 -c 3 -o gpurun_out/prof_c4 python bench.py --workload c4 --overlap 0 --steps 1 --warmup 1 --no-cpu --no-e2e --no-fp32 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
for f in gpurun_out/bench_*.json; do echo "== $f"; head -c 400 $f; echo; done
for f in gpurun_out/bench_*.err; do echo "== $f"; tail -3 $f; done

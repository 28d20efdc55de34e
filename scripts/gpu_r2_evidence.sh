# round-2 evidence pass: default bench line (as the driver runs it), the
# reference arm, the other workloads, ncu captures and launch lists, the
# randomised parity sweeps. Outputs under gpurun_out/ (copied to profiles/r2).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for wl in c1 c3n2 c3n4 c3n8 c4; do
  timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
done
timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu --no-e2e --overlap 0 > gpurun_out/bench_c4_serial.json 2> gpurun_out/bench_c4_serial.err
timeout 900 python bench.py --engine dist --exchange p2p --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_dist_c2.json 2> gpurun_out/bench_dist_c2.err
timeout 900 python bench.py --engine dist --exchange p2p --workload c4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_dist_c4.json 2> gpurun_out/bench_dist_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-fp32 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:quantize_kernel|reduce_kernel|norm_kernel" -s 3 -c 3 -o gpurun_out/prof_c2_final python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e --no-fp32 > gpurun_out/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:quantize_kernel|reduce_kernel|norm_kernel" -s 300 -c 3 -o gpurun_out/prof_c4_final python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-fp32 --overlap 0 > gpurun_out/ncu_c4.log 2>&1
timeout 900 python scripts/parity_sweep.py --cases 400 --seed 2026 > gpurun_out/parity_sweep.txt 2>&1
timeout 900 python scripts/dist_parity_sweep.py --cases 120 --seed 77 > gpurun_out/dist_parity_sweep.txt 2>&1
tail -1 gpurun_out/parity_sweep.txt gpurun_out/dist_parity_sweep.txt
for f in bench_default bench_ref bench_c1 bench_c3n2 bench_c3n4 bench_c3n8 bench_c4 bench_c4_serial bench_dist_c2 bench_dist_c4; do python -c "
import json
l=json.loads([x for x in open('gpurun_out/$f.json').read().splitlines() if x.startswith('{')][0])
print('$f', l.get('ms_per_step'), l.get('value'), (l.get('e2e') or {}).get('value'), {k:round(v['ms'],4) for k,v in (l.get('kernels') or {}).items()}, (l.get('dist_check') or {}).get('all_ranks_bit_identical_to_single_device'))
" || tail -3 gpurun_out/$f.err; done

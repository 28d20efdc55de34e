# Scaling run on one node (needs N GPUs): the bench contract's torchrun launch
# for N = 1, 2, 4, 8, one JSON line per N (exchange "auto" = peer memory over
# NVLink; --exchange pull for the NCCL route). Usage: bash scripts/bench_scaling.sh [workload]
W=${1:-c2}
python bench.py --workload $W --gpus 1
for N in 2 4 8; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --workload $W --gpus $N
done

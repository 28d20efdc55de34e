"""Measured per-rank kernel times of an N = 8 step, from one GPU.

At N = 8 (one worker per GPU) every rank runs: the norm of its own shard with
the k draws of its own lane slice (exponential tree), the quantize of its own
shard (whose stores land in the slices' owners), the schedule replay of its
1/8 slice over the 8 workers' rows, and the decode (+ SGD) of the full summed
lanes. Each of those kernels is timed here at exactly the per-rank size with
CUDA events (the stores stay in local HBM); NVLink transfers and flag
latencies are then added from B200_PROFILING.md's measured peer-copy
bandwidth (770 GB/s per direction), as the only unmeasured terms.

    python scripts/project_n8.py [--reps 30]  -> JSON on stdout
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402
from paper_2305_18627_b200._lib import check, lib, ptr_array  # noqa: E402

LINK_GBS = 770.0   # measured peer copy per direction (B200_PROFILING.md)
FLAG_US = 2.5      # one release/acquire round trip over NVLink (assumed)


def timed(fn, reps):
    """Per-launch device time of back-to-back launches (queued, so host
    submission latency does not sit between the events)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def rank_step(kind, s, width, n, d, sgd, reps, seed=42):
    dev = torch.device("cuda:0")
    L = lib()
    N = n  # one worker per GPU
    sp = torch.cuda.current_stream().cuda_stream
    x0 = torch.randn(d, device=dev)
    stats = torch.zeros(1, dtype=torch.float64, device=dev)
    norm = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = torch.zeros(int(L.gq_norm_workspace_bytes(1, d)), dtype=torch.uint8, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    lb = G.lane_bytes(d, width)
    lanes = [torch.zeros(lb, dtype=torch.uint8, device=dev) for _ in range(n)]
    summed = torch.zeros(lb, dtype=torch.uint8, device=dev)
    mean = torch.zeros(d, dtype=torch.float32, device=dev)
    param = torch.zeros(d, dtype=torch.float32, device=dev)
    G_ = 32 // width
    slice_lanes = -(-d // (N * 512)) * 512
    l1 = min(d, slice_lanes)
    INF = 0xFFFFFFFF
    out = {}
    # 1. norm of the rank's shard (+ the k draws of its slice for the exponential tree)
    spec = _lib.GqKdraws(None, n, kind, width, s, 0, 0, 0, l1, seed, 0)
    kb = int(L.gq_kdraws_bytes(C.byref(spec)))
    kbuf = torch.empty(max(kb, 4) // 4, dtype=torch.int32, device=dev)
    spec.buf = kbuf.data_ptr()
    sh = ptr_array([x0.data_ptr()])
    if kb:
        out["norm_us"] = timed(lambda: check(L.gq_norm_kdraws(sh, 0, 1, d, INF, INF, stats.data_ptr(),
                                                              norm.data_ptr(), ws.data_ptr(), err.data_ptr(),
                                                              C.byref(spec), sp)), reps)
    else:
        out["norm_us"] = timed(lambda: check(L.gq_norm(sh, 0, 1, d, INF, INF, stats.data_ptr(), norm.data_ptr(),
                                                       ws.data_ptr(), err.data_ptr(), sp)), reps)
    torch.cuda.synchronize()
    # 2. quantize of the rank's shard (n_total = n for the token shift)
    ids = (C.c_uint32 * 1)(0)
    la = ptr_array([lanes[0].data_ptr()])
    out["quantize_us"] = timed(lambda: check(L.gq_quantize(sh, 0, 1, ids, d, norm.data_ptr(), kind, s, n, width,
                                                           seed, 0, la, err.data_ptr(), sp)), reps)
    for t in lanes[1:]:
        t.copy_(lanes[0])
    # 3. schedule replay of the rank's slice over the n rows (k draws precomputed)
    arr = ptr_array([t.data_ptr() for t in lanes])
    if kb:
        out["reduce_slice_us"] = timed(lambda: check(L.gq_reduce_lanes_kdraws(
            arr, n, d, 0, l1, kind, width, s, 0, seed, 0, norm.data_ptr(), summed.data_ptr(), None, None, 0.0,
            err.data_ptr(), C.byref(spec), sp)), reps)
    else:
        out["reduce_slice_us"] = timed(lambda: check(L.gq_reduce_lanes(
            arr, n, d, 0, l1, kind, width, s, 0, seed, 0, norm.data_ptr(), summed.data_ptr(), None, None, 0.0,
            err.data_ptr(), sp)), reps)
    # 4. decode (+ SGD) of the full summed lanes
    out["decode_us"] = timed(lambda: check(L.gq_dequant(summed.data_ptr(), 0, d, norm.data_ptr(), kind, s, n, width,
                                                        None if sgd else mean.data_ptr(),
                                                        param.data_ptr() if sgd else None, 1e-3, err.data_ptr(),
                                                        sp)), reps)
    check(L.gq_check(err.data_ptr(), sp))
    compute = out["norm_us"] + out["quantize_us"] + out["reduce_slice_us"] + out["decode_us"]
    wire = (N - 1) / N * d * width / 8  # bytes each rank stores into peers per exchange (scatter, multicast)
    link_us = wire / (LINK_GBS * 1e9) * 1e6
    # scatter / multicast stores overlap their kernels; what exceeds the kernel is exposed
    exposed = max(0.0, link_us - out["quantize_us"]) + max(0.0, link_us - out["reduce_slice_us"])
    out.update(compute_us=compute, wire_bytes_per_exchange=wire, link_us_per_exchange=link_us,
               flags_us=2 * FLAG_US, step_us=compute + exposed + 2 * FLAG_US)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    res = {"what": "per-rank kernel times of an N=8 step measured on one B200 at the per-rank sizes; "
                   f"NVLink at {LINK_GBS} GB/s and {FLAG_US} us per flag round trip added (unmeasured)"}
    c2 = rank_step(1, 4, 4, 8, 1 << 24, False, a.reps)
    c2["value_d_per_s"] = (1 << 24) / (c2["step_us"] * 1e-6)
    # fp32 ring all_reduce of the same 64 MiB gradient at a 700 GB/s bus bandwidth (NCCL busbw convention)
    c2["fp32_allreduce_us_at_700GBs_busbw"] = 2 * 7 / 8 * (1 << 24) * 4 / 700e9 * 1e6
    res["c2"] = c2
    b = rank_step(0, 15, 8, 8, 6553600, True, a.reps)
    b["value_d_per_s"] = 6553600 / (b["step_us"] * 1e-6)
    b["c4_step_ms_serial_52_buckets"] = 52 * b["step_us"] * 1e-3
    b["fp32_allreduce_c4_ms_at_700GBs_busbw"] = 2 * 7 / 8 * 340e6 * 4 / 700e9 * 1e3
    res["c4_bucket"] = b
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

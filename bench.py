"""Benchmark of the Global-QSGD gradient-sync hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c4] [--impl reference]

One "step" = one full sync of the workload's gradients: global norm ->
quantize (+ lane encode) -> schedule-replay aggregate -> decode (+ SGD for c4),
on synthetic gaussian_shards-shaped data resident in HBM. Metric (BASELINE.json):
fp32 gradient elements synced per second, summed over all workers
(value = n_workers * d / step time), higher is better.

Workloads (BASELINE.json configs):
  c2 (default, configs[1]): global exponential dithering s=4, 4-bit packed
      lanes, d = 2^24, n = 8 workers, tree schedule, seed 42, round = step.
  c4 (configs[3]): BERT-large-sized 340M-element gradient per worker, n = 8,
      8-bit standard dithering s = 15, 25 MiB buckets (round = step*52 + bucket),
      decode fused with the SGD update of fp32 parameters.
At N = 1 all n workers live on the one GPU (the reference's Transport::Inproc
simulation, algorithm.cpp:127-228); at N > 1 each rank hosts n/N workers.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "c2": dict(kind=1, s=4, width=4, n=8, d=1 << 24, topo=0, seed=42, bucket=None, sgd=False,
               desc="C2: global exponential dithering s=4, 4-bit packed lanes, d=2^24, n=8 workers, tree"),
    "c4": dict(kind=0, s=15, width=8, n=8, d=340_000_000, topo=0, seed=42, bucket=6_553_600, sgd=True,
               desc="C4: BERT-large 340M fp32 gradient per worker, n=8, 8-bit standard dithering s=15, "
                    "25 MiB buckets, fused SGD"),
}
METRIC = "fp32 grad elems/s synced (quant+int allreduce+dequant)"
UNIT = "elem/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (NVML)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        reasons = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(s)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own implementation on the host cores
# ---------------------------------------------------------------------------
def cpu_reference_sample(wl: dict, budget_s: float, steps: int | None = None):
    """Time gqsgd_mean (Transport::Tcp: one thread per worker, the reference's
    parallel mode) of the unmodified reference (oracle/_ref) on a bounded
    sample of the workload; falls back to the C oracle port (1 thread)."""
    import numpy as np
    from oracle.bind import Oracle, reference_or_none
    ref = reference_or_none()
    n = wl["n"]
    d_s = 1 << 18 if wl["d"] >= (1 << 18) else wl["d"]
    o = Oracle()
    x = o.gaussian_shards(n, d_s, 12345).astype(np.float32).astype(np.float64)
    width = 8 if wl["width"] == 4 else wl["width"]  # the reference's narrowest lane
    if ref is not None:
        kind, cores = "reference", min(n, os.cpu_count() or 1)
        run = lambda r: ref.mean(x, wl["kind"], wl["s"], width=width, topo=wl["topo"], seed=wl["seed"],
                                 round=r, transport=1)
    else:
        kind, cores = "port", 1
        run = lambda r: o.mean(x, wl["kind"], wl["s"], width=width, topo=wl["topo"], seed=wl["seed"], round=r)
    times = []
    t_start = time.perf_counter()
    r = 0
    while True:
        t0 = time.perf_counter()
        run(r)
        times.append(time.perf_counter() - t0)
        r += 1
        if steps is not None and r >= steps:
            break
        if steps is None and time.perf_counter() - t_start >= budget_s:
            break
    return dict(times=times, d_sample=d_s, n=n, kind=kind, cores=cores, width=width)


# ---------------------------------------------------------------------------
def reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    res = cpu_reference_sample(wl, 0, steps=args.warmup + args.steps)
    t = res["times"][args.warmup:]
    per_step = sum(t) / len(t)
    value = res["n"] * res["d_sample"] / per_step
    sample = (f"gqsgd_mean n={res['n']} d={res['d_sample']} (of d={wl['d']}) w={res['width']} "
              f"{'Transport::Tcp' if res['kind'] == 'reference' else 'C oracle port'}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gaussian_shards seed 12345, fp32-cast)",
            "config": {"workload": wl["desc"], "n_workers": wl["n"], "d": wl["d"],
                       "parallelism": "cpu threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": res["cores"], "kind": res["kind"],
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        reference_arm(args, wl)
        return

    import torch
    import torch.distributed as dist

    from paper_2305_18627_b200 import _lib
    from paper_2305_18627_b200 import gqsgd as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, d = wl["n"], wl["d"]
    if n % world:
        raise SystemExit("workers must divide evenly over ranks")
    if world > 1:
        raise SystemExit("multi-GPU bench path: see paper_2305_18627_b200/dist.py (not yet wired)")

    L = _lib.lib()
    kind, s, width, topo, seed = wl["kind"], wl["s"], wl["width"], wl["topo"], wl["seed"]
    plan = G.plan_path(G.GqsgdConfig(workers=n, scheme=G.LevelKind(kind), s=s, width_bits=width,
                                     topo=G.TopologyKind(topo), seed=seed))
    assert plan.lane_width == width
    stream = torch.cuda.Stream(dev)
    sp = stream.cuda_stream

    # Synthetic gradients in HBM: one generator call per worker (randn is
    # plumbing; parity runs use the reference's gaussian_shards instead).
    gen = torch.Generator(device=dev).manual_seed(12345)
    shards = [torch.randn(d, dtype=torch.float32, device=dev, generator=gen) for _ in range(n)]
    lbytes = G.lane_bytes(d, width)
    lanes = [torch.zeros(lbytes, dtype=torch.uint8, device=dev) for _ in range(n)]
    mean = torch.zeros(d, dtype=torch.float32, device=dev)
    param = torch.zeros(d, dtype=torch.float32, device=dev) if wl["sgd"] else None
    stats = torch.zeros(n, dtype=torch.float64, device=dev)
    norm = torch.zeros(1, dtype=torch.float64, device=dev)
    bucket = wl["bucket"] or d
    nb = (d + bucket - 1) // bucket
    ws = torch.zeros(int(L.gq_norm_workspace_bytes(n, bucket)), dtype=torch.uint8, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    ids = (C.c_uint32 * n)(*range(n))
    lr = 1e-3

    # per-bucket pointer arrays (16-byte aligned offsets)
    def arrs(b):
        off = b * bucket
        db = min(bucket, d - off)
        sh = _lib.ptr_array([x.data_ptr() + 4 * off for x in shards])
        ln = _lib.ptr_array([l.data_ptr() + off * width // 8 for l in lanes])
        return db, off, sh, ln
    bucket_args = [arrs(b) for b in range(nb)]
    for db, off, _, _ in bucket_args:
        assert (off * width // 8) % 16 == 0 and (4 * off) % 16 == 0

    def step(t: int, ev=None):
        for b, (db, off, sh, ln) in enumerate(bucket_args):
            rnd = t * nb + b
            if ev is not None and b == 0:
                ev[0].record(stream)
            _lib.check(L.gq_norm(sh, 0, n, db, 0xFFFFFFFF, 0xFFFFFFFF, stats.data_ptr(), norm.data_ptr(),
                                 ws.data_ptr(), err.data_ptr(), sp))
            if ev is not None and b == 0:
                ev[1].record(stream)
            _lib.check(L.gq_quantize(sh, 0, n, ids, db, norm.data_ptr(), kind, s, n, width, seed, rnd, ln,
                                     err.data_ptr(), sp))
            if ev is not None and b == 0:
                ev[2].record(stream)
            # every worker's lane buffer, offset to this bucket
            _lib.check(L.gq_reduce_lanes(ln, n, db, 0, db, kind, width, s, topo, seed, rnd, norm.data_ptr(),
                                         None, mean.data_ptr() + 4 * off,
                                         (param.data_ptr() + 4 * off) if param is not None else None,
                                         lr, err.data_ptr(), sp))
            if ev is not None and b == 0:
                ev[3].record(stream)

    with torch.cuda.stream(stream):
        for t in range(args.warmup):
            step(t)
        _lib.check(L.gq_check(err.data_ptr(), sp))
        torch.cuda.synchronize()

        K = args.steps
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local_rank) as clk:
            start.record(stream)
            for t in range(K):
                step(args.warmup + t, evs[t])
            stop.record(stream)
            torch.cuda.synchronize()
        _lib.check(L.gq_check(err.data_ptr(), sp))
        ms = start.elapsed_time(stop) / K
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()

        # per-kernel device time (first bucket of each step; all buckets equal-sized but the last)
        k_norm = sum(e[0].elapsed_time(e[1]) for e in evs) / K
        k_quant = sum(e[1].elapsed_time(e[2]) for e in evs) / K
        k_red = sum(e[2].elapsed_time(e[3]) for e in evs) / K

        # fp32 uncompressed comparator on the same buffers (tree-order sum of n shards)
        fp32_ms = None
        if wl["bucket"] is None:
            shp = _lib.ptr_array([x.data_ptr() for x in shards])
            for _ in range(3):
                _lib.check(L.gq_baseline_mean_inproc(shp, n, d, 0, mean.data_ptr(), sp))
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(20):
                _lib.check(L.gq_baseline_mean_inproc(shp, n, d, 0, mean.data_ptr(), sp))
            b_.record(stream)
            torch.cuda.synchronize()
            fp32_ms = a.elapsed_time(b_) / 20

    # e2e through the public API with host buffers (pinned), H2D + D2H inside
    e2e = None
    if not args.no_e2e:
        host = [torch.empty(d, dtype=torch.float32, pin_memory=True) for _ in range(n)]
        for h, x in zip(host, shards):
            h.copy_(x.cpu())
        out_host = torch.empty(d, dtype=torch.float32, pin_memory=True)
        Ke = max(3, min(args.steps, 10))
        with torch.cuda.stream(stream):
            def e2e_step(t):
                for h, x in zip(host, shards):
                    x.copy_(h, non_blocking=True)
                step(t)
                out_host.copy_(mean, non_blocking=True)
            e2e_step(0)
            torch.cuda.synchronize()
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for t in range(Ke):
                e2e_step(t)
            b_.record(stream)
            torch.cuda.synchronize()
            e2e_ms = a.elapsed_time(b_) / Ke
        e2e = {"value": n * d / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": n * d * 4, "d2h_bytes_per_step": d * 4}

    if rank != 0:
        return
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # algorithmic bytes per launch (first bucket), DESIGN.md §3
    db0 = bucket_args[0][0]
    wb = width / 8
    kbytes = {
        "norm": n * db0 * 4,
        "quantize": n * db0 * (4 + wb),
        "reduce_decode": n * db0 * wb + db0 * 4 + (db0 * 8 if wl["sgd"] else 0),
    }
    ktime = {"norm": k_norm, "quantize": k_quant, "reduce_decode": k_red}
    dom = max(ktime, key=ktime.get)
    achieved = kbytes[dom] / (ktime[dom] * 1e-3) / 1e9
    kernels = {k: {"ms": ktime[k], "alg_bytes": kbytes[k],
                   "gbs": kbytes[k] / (ktime[k] * 1e-3) / 1e9,
                   "frac": kbytes[k] / (ktime[k] * 1e-3) / 1e9 / hbm_peak} for k in ktime}
    step_bytes = sum(kbytes.values()) * nb
    traffic = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(args.workload, {}).get(dom)

    cpu = None
    if not args.no_cpu and world == 1:
        r = cpu_reference_sample(wl, budget_s=12.0)
        per = sum(r["times"]) / len(r["times"])
        cpu = {"value": r["n"] * r["d_sample"] / per, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
               "sample": (f"gqsgd_mean n={r['n']} d={r['d_sample']} (1/{wl['d'] // r['d_sample']} of d) "
                          f"w={r['width']}, {len(r['times'])} calls, "
                          f"{'Transport::Tcp' if r['kind'] == 'reference' else '1 thread'}")}

    value = n * d / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32-in/u%d-lanes/f64-scale" % width,
        "data": "synthetic (torch.randn fp32 gradients resident in HBM)",
        "config": {"workload": wl["desc"], "n_workers": n, "d": d, "lane_width": width,
                   "buckets": nb, "parallelism": f"dp{n} simulated on {world} GPU(s)",
                   "l2": "inputs (%.0f MiB) exceed the 126 MB L2; no flush" % (n * d * 4 / 2**20)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                     "step_alg_bytes": step_bytes,
                     "step_gbs": step_bytes / (ms * 1e-3) / 1e9},
        "kernels": kernels,
        "gpu_launches": 3 * nb * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "fp32_baseline": ({"what": "uncompressed fp32 tree-sum of the n shards on the same GPU",
                           "ms_per_step": fp32_ms, "value": n * d / (fp32_ms * 1e-3), "unit": UNIT}
                          if fp32_ms else None),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

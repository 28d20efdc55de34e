"""Benchmark of the Global-QSGD gradient-sync hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c4] [--impl reference]

One "step" = one full sync of the workload's gradients: global norm ->
quantize (+ lane encode) -> schedule-replay aggregate -> decode (+ SGD for c4),
on synthetic gaussian_shards-shaped data resident in HBM. Metric (BASELINE.json,
BASELINE.md §2 "d/t"): fp32 gradient elements synchronised per second,
value = d / step time (every worker's d-element gradient is synced in a step;
value_n_times_d = n * d / step time is the per-element work rate over all n
workers), higher is better.

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
    # the reference's CPU-runnable case (configs[0])
    "c1": dict(kind=0, s=31, width=8, n=4, d=1 << 20, topo=0, seed=42, bucket=None, sgd=False,
               desc="C1: global standard dithering s=31, 8-bit, d=2^20, n=4 workers, tree"),
    # ResNet-50-sized gradient (configs[2]) at n = 2 / 4 / 8 workers; s is the
    # largest 8-bit-admissible level count (n (s+1) <= 128)
    "c3n2": dict(kind=0, s=63, width=8, n=2, d=25_600_000, topo=0, seed=42, bucket=None, sgd=False,
                 desc="C3: ResNet-50 25.6M fp32 gradient, standard s=63, 8-bit, n=2 workers"),
    "c3n4": dict(kind=0, s=31, width=8, n=4, d=25_600_000, topo=0, seed=42, bucket=None, sgd=False,
                 desc="C3: ResNet-50 25.6M fp32 gradient, standard s=31, 8-bit, n=4 workers"),
    "c3n8": dict(kind=0, s=15, width=8, n=8, d=25_600_000, topo=0, seed=42, bucket=None, sgd=False,
                 desc="C3: ResNet-50 25.6M fp32 gradient, standard s=15, 8-bit, n=8 workers"),
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
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--overlap", type=int, default=2,
                    help="bucketed N=1 runs: 0 serial; 1 norm pass on a side stream ahead of quantize; "
                         "2 also reduce(b) on a third stream under quantize(b+1)")
    ap.add_argument("--graph", type=int, default=1,
                    help="single-bucket N=1 runs: time the step as one CUDA graph launch")
    ap.add_argument("--kdraws", type=int, default=1,
                    help="exponential tree path: precompute the reduce's k draws in the norm launch")
    ap.add_argument("--quant-ctas", type=int, default=0, help="gq_set_option quantize CTAs/SM (0 auto)")
    ap.add_argument("--reduce-ctas", type=int, default=0, help="gq_set_option reduce CTAs/SM (0 auto)")
    ap.add_argument("--small-path", type=int, default=1,
                    help="gq_set_option GQ_OPT_SMALL_PATH: small syncs as one fused cooperative kernel")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help=argparse.SUPPRESS)  # gloo + GQ_BENCH_SHARED_GPU=1: the N-rank code path on one GPU (tests)
    ap.add_argument("--engine", default="auto", choices=["auto", "dist"],
                    help="dist: force the multi-rank DistSync path even at N=1 (testing)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "p2p", "pull", "nccl_sum"],
                    help="N>1 lane exchange (nccl_sum: standard 8/32-bit only)")
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
def cpu_reference_sample(wl: dict, budget_s: float, steps: int | None = None, warmup: int = 0,
                         full: bool = True):
    """Time gqsgd_mean (Transport::Tcp: one thread per worker, the reference's
    parallel mode) of the unmodified reference (oracle/_ref) on the workload;
    falls back to the C oracle port (1 thread).

    full=True runs the workload's own size (C1/C2/C3: the whole d; bucketed
    C4: one 25 MiB bucket of the gradient per call, the unit the reference is
    called on, round = bucket index); at most `steps` calls, stopping early
    once `budget_s` of timed calls have run (at least one call)."""
    import numpy as np
    from oracle.bind import Oracle, reference_or_none
    ref = reference_or_none()
    n = wl["n"]
    d_full = wl["bucket"] or wl["d"]
    d_s = d_full if full else min(d_full, 1 << 18)
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
    for r in range(warmup):
        run(r)
    times = []
    t_start = time.perf_counter()
    r = warmup
    while True:
        t0 = time.perf_counter()
        run(r)
        times.append(time.perf_counter() - t0)
        r += 1
        if steps is not None and len(times) >= steps:
            break
        if time.perf_counter() - t_start >= budget_s:
            break
    del x
    return dict(times=times, d_sample=d_s, n=n, kind=kind, cores=cores, width=width,
                same_config=(d_s == wl["d"]))


def cpu_reference_extras(wl: dict, budget_s: float = 3.0) -> dict:
    """The other CPU timings SURVEY §8(d) asks for, on the same sample:
    gqsgd_mean with Transport::Inproc (1 core, the reference semantics) and
    the uncompressed fp32 baseline_mean; plus the host's core count and model."""
    import platform

    import numpy as np
    from oracle.bind import Oracle, reference_or_none
    ref = reference_or_none()
    out = {"nproc": os.cpu_count(), "cpu_model": platform.processor() or platform.machine()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                out["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    if ref is None:
        return out
    n = wl["n"]
    d_s = 1 << 18 if wl["d"] >= (1 << 18) else wl["d"]
    x = Oracle().gaussian_shards(n, d_s, 12345).astype(np.float32).astype(np.float64)
    width = 8 if wl["width"] == 4 else wl["width"]

    def rate(fn):
        t, k, t0 = 0.0, 0, time.perf_counter()
        while k < 1 or time.perf_counter() - t0 < budget_s:
            a = time.perf_counter()
            fn(k)
            t += time.perf_counter() - a
            k += 1
        return d_s / (t / k)
    out["sample"] = f"d={d_s} per worker, n={n}"
    out["gqsgd_mean_inproc_1core"] = rate(lambda r: ref.mean(x, wl["kind"], wl["s"], width=width, topo=wl["topo"],
                                                             seed=wl["seed"], round=r, transport=0))
    out["baseline_mean_fp32_cpu"] = rate(lambda r: ref.baseline_mean(x, topo=wl["topo"], transport=0, round=r))
    out["unit"] = UNIT
    return out


# ---------------------------------------------------------------------------
def reference_arm(args, wl):
    """The reference's own CPU implementation of the path (oracle/_ref, the
    unmodified reference built from its sources; gqsgd_mean with
    Transport::Tcp) on the host cores, on the same workload as our arm: the
    full d per step (C4: one 25 MiB bucket per step, the unit the reference is
    called on). Warm-up is capped at one call and the timed calls at what fits
    ~4 minutes; the line says how many ran."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    res = cpu_reference_sample(wl, budget_s=240.0, steps=args.steps, warmup=min(args.warmup, 1))
    t = res["times"]
    per_step = sum(t) / len(t)
    value = res["d_sample"] / per_step
    sample = (f"gqsgd_mean n={res['n']} d={res['d_sample']} w={res['width']} "
              f"{'Transport::Tcp (one thread per worker)' if res['kind'] == 'reference' else 'C oracle port'}"
              f", {len(t)} timed calls after {min(args.warmup, 1)} warm-up")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(t), "steps_requested": args.steps, "warmup": min(args.warmup, 1),
            "ms_per_step": per_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gaussian_shards seed 12345, fp32-cast)",
            "config": config_of(wl, 1, wl["n"], None),
            "same_config": res["same_config"],
            "reference_lane_width": res["width"],
            "value_n_times_d": res["n"] * value,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": res["cores"], "kind": res["kind"],
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if wl["width"] == 4:
        line["note"] = ("the reference refuses 4-bit token lanes (exp_arith.cpp:65-66), so it runs its "
                        "narrowest lane (8 bits); the levels and decoded mean are identical")
    print(json.dumps(line), flush=True)


def config_of(wl: dict, world: int, n_local: int, eng) -> dict:
    """The workload's config dict, identical in both arms (the engine-specific
    execution details go in "execution")."""
    n, d = wl["n"], wl["d"]
    return {"workload": wl["desc"], "n_workers": n, "d": d, "lane_width": wl["width"], "s": wl["s"],
            "kind": "standard" if wl["kind"] == 0 else "exponential", "topo": "tree" if wl["topo"] == 0 else "ring",
            "buckets": (d + (wl["bucket"] or d) - 1) // (wl["bucket"] or d), "seed": wl["seed"],
            "fused_sgd": wl["sgd"],
            "l2": (("inputs (%.0f MiB per GPU) fit twice in the 126 MB L2: a 256 MiB write (then read back) between "
                    "timed steps evicts them, outside the per-step events") if l2_flush(n_local, d) else
                   "inputs (%.0f MiB per GPU) exceed twice the 126 MB L2; no flush") % (n_local * d * 4 / 2**20)}


L2_BYTES = 126 * 10**6


def l2_flush(n_local: int, d: int) -> bool:
    """Flush L2 between timed steps unless the step's fp32 inputs are larger
    than twice the L2 (then every step streams them from HBM anyway)."""
    return n_local * d * 4 < 2 * L2_BYTES


class L2Flusher:
    """Between timed steps: a 256 MiB device write (evicts the 126 MB L2),
    then a read of the same buffer, which writes those dirty lines back here
    rather than inside the next step. The step is timed with its own pair of
    events, so neither is counted."""

    def __init__(self, dev, enabled: bool):
        import torch
        self.buf = torch.empty(64 << 20, dtype=torch.float32, device=dev) if enabled else None
        self.k, self.acc = 0, None

    def __call__(self):
        if self.buf is not None:
            self.k += 1
            self.buf.fill_(float(self.k & 0xFF))
            self.acc = self.buf.sum()


# ---------------------------------------------------------------------------
class InprocEngine:
    """N = 1: all n workers on this GPU (Transport::Inproc, algorithm.cpp:127-228),
    straight through the C ABI: 3 launches per bucket.

    overlap (bucketed workloads): 1 = the HBM-bound norm pass of every bucket
    runs on a side stream ahead of the ALU-bound quantize of earlier buckets
    (per-bucket stats / norm buffers; norm(b) of step t+1 waits for
    quantize(b) of step t); 2 = also reduce(b) (HBM-bound) on a third stream
    under quantize(b+1) (quantize(b) of step t+1 waits for reduce(b) of step
    t, which read its lanes). Every bucket is still its own reference call
    with its own round; only the overlap of independent buckets changes.
    Measured on C4: 7.56 ms serial -> 5.86 ms with overlap 2."""
    phases = ("norm", "quantize", "reduce_decode")

    def __init__(self, L, G, _lib, wl, shards, param, mean, dev, sp, bucket, overlap=False, kdraws=True,
                 small_path=1):
        import torch
        self.L, self._lib, self.wl, self.sp = L, _lib, wl, sp
        self.small_path, self.fused = small_path, False
        n, d, width = wl["n"], wl["d"], wl["width"]
        self.n = n
        lbytes = G.lane_bytes(d, width)
        nb = (d + bucket - 1) // bucket
        self.overlap = bool(overlap) and nb > 1
        nbuf = nb if self.overlap else 1
        self.lanes = [torch.zeros(lbytes, dtype=torch.uint8, device=dev) for _ in range(n)]
        self.stats = torch.zeros(nbuf, n, dtype=torch.float64, device=dev)
        self.norm = torch.zeros(nbuf, dtype=torch.float64, device=dev)
        self.ws = torch.zeros(int(L.gq_norm_workspace_bytes(n, bucket)), dtype=torch.uint8, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ids = (C.c_uint32 * n)(*range(n))
        self.mean, self.param = mean, param
        self.buckets = []
        for b in range(nb):
            off = b * bucket
            db = min(bucket, d - off)
            assert (off * width // 8) % 16 == 0 and (4 * off) % 16 == 0
            self.buckets.append((db, off, _lib.ptr_array([x.data_ptr() + 4 * off for x in shards]),
                                 _lib.ptr_array([l.data_ptr() + off * width // 8 for l in self.lanes])))
        self.launches_per_step = 3 * nb
        # exponential tree path: the k draws ride in the norm launch (gq_norm_kdraws)
        self.kd = None
        if nb == 1 and kdraws:
            spec = _lib.GqKdraws(None, n, wl["kind"], width, wl["s"], wl["topo"], 0, 0, d, wl["seed"], 0)
            nbytes = int(L.gq_kdraws_bytes(C.byref(spec)))
            if nbytes:
                self.kbuf = torch.empty(nbytes // 4, dtype=torch.int32, device=dev)
                spec.buf = self.kbuf.data_ptr()
                self.kd = spec
        self.overlap_reduce = self.overlap and overlap >= 2
        if self.overlap:
            self.side = torch.cuda.Stream(dev)
            self.ev_norm = [torch.cuda.Event() for _ in range(nb)]
            self.ev_quant = [torch.cuda.Event() for _ in range(nb)]
        if self.overlap_reduce:
            self.rstream = torch.cuda.Stream(dev)
            self.ev_red = [torch.cuda.Event() for _ in range(nb)]

    def step(self, t, marks=None):
        """marks: optional 6 events, (start, end) of norm / quantize / reduce
        of bucket 0, recorded on the stream each runs on."""
        import torch
        L, wl, sp, chk = self.L, self.wl, self.sp, self._lib.check
        n, kind, s, width = self.n, wl["kind"], wl["s"], wl["width"]
        nb = len(self.buckets)
        main = torch.cuda.current_stream()
        nsp = self.side.cuda_stream if self.overlap else sp

        def norm_of(b):
            i = b if self.overlap else 0
            return self.stats[i].data_ptr(), self.norm[i:i + 1].data_ptr()

        def launch_norm(b):
            db, off, sh, ln = self.buckets[b]
            st, nm = norm_of(b)
            if self.kd is not None:
                self.kd.round = t * nb + b
                chk(L.gq_norm_kdraws(sh, 0, n, db, 0xFFFFFFFF, 0xFFFFFFFF, st, nm, self.ws.data_ptr(),
                                     self.err.data_ptr(), C.byref(self.kd), nsp))
                return
            chk(L.gq_norm(sh, 0, n, db, 0xFFFFFFFF, 0xFFFFFFFF, st, nm, self.ws.data_ptr(),
                          self.err.data_ptr(), nsp))

        if self.overlap:
            # side streams start after everything already queued on the main
            # stream (e.g. the H2D of this step's gradients in the e2e loop)
            start = torch.cuda.Event()
            start.record(main)
            self.side.wait_event(start)
            if self.overlap_reduce:
                self.rstream.wait_event(start)
            for b in range(nb):
                self.side.wait_event(self.ev_quant[b])  # quantize(b) of the previous step read norm[b]
                if marks is not None and b == 0:
                    marks[0].record(self.side)
                launch_norm(b)
                self.ev_norm[b].record(self.side)
                if marks is not None and b == 0:
                    marks[1].record(self.side)
        for b, (db, off, sh, ln) in enumerate(self.buckets):
            rnd = t * nb + b
            mk = marks if (marks is not None and b == 0) else None
            if self.overlap:
                main.wait_event(self.ev_norm[b])
            else:
                if mk: mk[0].record()
                launch_norm(b)
                if mk: mk[1].record()
            _, nm = norm_of(b)
            if self.overlap_reduce:  # lanes(b) of the previous step were read
                main.wait_event(self.ev_red[b])
            if mk: mk[2].record()
            chk(L.gq_quantize(sh, 0, n, self.ids, db, nm, kind, s, n, width, wl["seed"], rnd, ln,
                              self.err.data_ptr(), sp))
            if self.overlap:
                self.ev_quant[b].record(main)
            if mk: mk[3].record()
            rs = main
            if self.overlap_reduce:  # reduce(b) on a third stream, after quantize(b)
                rs = self.rstream
                rs.wait_event(self.ev_quant[b])
            if mk: mk[4].record(rs)
            mean_p = (self.mean.data_ptr() + 4 * off) if self.mean is not None else None
            param_p = (self.param.data_ptr() + 4 * off) if self.param is not None else None
            if self.kd is not None:
                chk(L.gq_reduce_lanes_kdraws(ln, n, db, 0, db, kind, width, s, wl["topo"], wl["seed"], rnd, nm,
                                             None, mean_p, param_p, LR, self.err.data_ptr(), C.byref(self.kd),
                                             rs.cuda_stream))
            else:
                chk(L.gq_reduce_lanes(ln, n, db, 0, db, kind, width, s, wl["topo"], wl["seed"], rnd, nm, None,
                                      mean_p, param_p, LR, self.err.data_ptr(), rs.cuda_stream))
            if mk: mk[5].record(rs)
            if self.overlap_reduce:
                self.ev_red[b].record(rs)
        if self.overlap_reduce:  # the step ends when every reduce has
            for b in range(nb):
                main.wait_event(self.ev_red[b])

    def check(self):
        self._lib.check(self.L.gq_check(self.err.data_ptr(), self.sp))

    def make_graph(self, first_round):
        """Single-bucket workloads: the whole step as one CUDA graph
        (gq_graph_mean_inproc; the round lives in device memory and the graph
        increments it), so small-d steps are not bound by launch latency."""
        import torch
        if len(self.buckets) != 1:
            return None
        wl, n = self.wl, self.n
        db, off, sh, ln = self.buckets[0]
        cfg = self._lib.GqConfig(n, wl["kind"], wl["s"], 0xFFFFFFFF, 0xFFFFFFFF, wl["width"], wl["topo"], 0,
                                 wl["seed"])
        self.round_dev = torch.tensor([first_round], dtype=torch.int64, device=self.ws.device)
        self.res_lanes = torch.zeros_like(self.lanes[0])
        h = C.c_void_p()
        # the library runs small single-bucket steps as one cooperative kernel
        # (GQ_OPT_SMALL_PATH; include/gq_b200.h states the conditions)
        self.fused = (self.small_path != 0 and n in (2, 4, 8) and wl["width"] in (4, 8) and wl["topo"] == 0
                      and (wl["kind"] == 0 or wl["s"] + 1 <= 32)
                      and n * db <= (1 << (24 if self.small_path == 2 else 23)))
        if self.fused:
            self.launches_per_step = 1
        self._lib.check(self.L.gq_graph_mean_inproc(
            sh, 0, db, C.byref(cfg), self.round_dev.data_ptr(), ln, None,
            self.mean.data_ptr() if self.mean is not None else None,
            self.param.data_ptr() if self.param is not None else None, LR, self.stats[0].data_ptr(),
            self.norm[0:1].data_ptr(), self.ws.data_ptr(), self.kbuf.data_ptr() if self.kd is not None else None,
            self.err.data_ptr(), C.byref(h)))
        self.graph = h
        return h

    def graph_step(self):
        self._lib.check(self.L.gq_graph_launch(self.graph, self.sp))

    def reset_graph_round(self, r):
        self.round_dev.fill_(r)

    def alg_bytes(self, db):
        """SURVEY.md §8(d) bytes only: norm reads 4 B/elem/worker; quantize reads
        4 and writes w/8; the reduce reads every worker's w/8 and writes the
        decoded fp32 (4 B) - or, with the fused SGD, reads and writes the fp32
        parameter (8 B) and writes no mean. The k-draw words (a by-product the
        norm pass writes and the reduce reads) are not counted."""
        wb, n = self.wl["width"] / 8, self.n
        return {"norm": n * db * 4, "quantize": n * db * (4 + wb),
                "reduce_decode": n * db * wb + (db * 8 if self.wl["sgd"] else db * 4)}


class DistEngine:
    """N > 1: rank g hosts workers [g n/N, (g+1) n/N); one dist.BucketedSync
    pipelines all buckets of the step (each its own reference call / round):
    norm | quantize | exchange (all_to_all + schedule replay + all_gather, or
    NCCL integer all_reduce) | decode, with every collective asynchronous so
    bucket b's transfers run under bucket b+1's kernels."""
    phases = ("norm", "quantize", "exchange", "decode")

    def __init__(self, wl, shards, param, mean, dev, stream, bucket, exchange):
        from paper_2305_18627_b200 import gqsgd as G
        from paper_2305_18627_b200.dist import BucketedSync, DeviceKernels
        self.wl = wl
        n, d = wl["n"], wl["d"]
        cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind(wl["kind"]), s=wl["s"], width_bits=wl["width"],
                            topo=G.TopologyKind(wl["topo"]), seed=wl["seed"])
        self.kern = DeviceKernels(dev, stream)
        self.buckets = []
        nb = (d + bucket - 1) // bucket
        for b in range(nb):
            off = b * bucket
            db = min(bucket, d - off)
            self.buckets.append((db, off, [x[off:off + db] for x in shards]))
        self.pipe = BucketedSync(cfg, [db for db, _, _ in self.buckets], kernels=self.kern, device=dev,
                                 exchange=exchange)
        self.param = param
        e0 = self.pipe.syncs[0]
        if mean is not None and nb != 1:
            raise SystemExit("the decoded-mean output is only kept for single-bucket workloads")
        self.mean = e0.mean if mean is not None else None
        self.world, self.n_local, self.exchange = e0.world, e0.n_local, e0.exchange
        # norm + combine + quantize + (reduce_slice | local partial sum if n_local > 1) + dequant;
        # p2p: norm + combine + quantize_scatter + 2x(signal, wait) + reduce_multicast + dequant
        if self.exchange == "p2p":  # eager: gq_norm; put+wait+combine; quantize (signals in-kernel); wait; reduce
            per = 9                 # (signals); wait; dequant - a graph replay folds the exchange into 4 (make_graph)
        else:
            per = 4 + (1 if self.exchange == "pull" else (1 if e0.n_local > 1 else 0))
        self.launches_per_step = per * nb

    def step(self, t, marks=None):
        nb = len(self.buckets)
        bounds = None
        if marks is not None:  # (start, end) pairs from the 5 phase boundaries of bucket 0
            bounds = [marks[0], marks[1], marks[3], marks[5], marks[7]]
        params = ([self.param[off:off + db] for db, off, _ in self.buckets] if self.param is not None else None)
        self.pipe.run([sh for _, _, sh in self.buckets], [t * nb + b for b in range(nb)], params=params, lr=LR,
                      write_mean=self.mean is not None, marks=bounds)

    def check(self):
        self.pipe.check()

    def make_graph(self, first_round):
        """p2p exchange: each bucket's whole rank step (norm, stats and lane
        exchanges over peer memory, decode + SGD) as one CUDA graph; bucket b
        of step t runs round t*nb + b as in the eager path."""
        e0 = self.pipe.syncs[0]
        if e0.exchange != "p2p" or e0.device.type != "cuda" or e0.host_waits:
            return None
        nb = len(self.buckets)
        self.graphs = []
        # folded step: norm (+ stats put), quantize (+ stats wait / fold, row
        # signal), reduce (+ row wait, summed signal), decode (+ summed wait,
        # round advance)
        self.launches_per_step = 4 * nb
        for b, (sync, (db, off, sh)) in enumerate(zip(self.pipe.syncs, self.buckets)):
            prm = self.param[off:off + db] if self.param is not None else None
            self.graphs.append(sync.make_graph(sh, first_round * nb + b, prm, LR, self.mean is not None,
                                               round_step=nb))
        return self.graphs

    def reset_graph_round(self, r):
        nb = len(self.buckets)
        for b, g in enumerate(self.graphs):
            g.round.fill_(r * nb + b)

    def graph_step(self):
        # buckets alternate between two streams: bucket b+1's norm / quantize
        # run under bucket b's flag waits and NVLink transfers; bucket b uses
        # communicator lane b % BucketedSync.COMM_LANES, so each stream
        # replays the buckets of one communicator in order
        if len(self.graphs) == 1:
            self.graphs[0].launch()
            return
        import torch
        lanes = self.pipe.COMM_LANES
        if not hasattr(self, "sides"):
            self.sides = [torch.cuda.Stream(self.kern.device) for _ in range(lanes - 1)]
            self.ev_fork = torch.cuda.Event()
            self.ev_join = [torch.cuda.Event() for _ in range(lanes - 1)]
        main = self.kern.stream
        streams = [main] + self.sides
        self.ev_fork.record(main)
        for sd in self.sides:
            sd.wait_event(self.ev_fork)
        for b, g in enumerate(self.graphs):
            g.launch(streams[b % lanes].cuda_stream)
        for sd, ev in zip(self.sides, self.ev_join):
            ev.record(sd)
            main.wait_event(ev)

    def alg_bytes(self, db):
        wb, nl, N = self.wl["width"] / 8, self.n_local, self.world
        return {"norm": nl * db * 4, "quantize": nl * db * (4 + wb),
                # bytes each rank puts on the wire (all_to_all + all_gather): ring-allreduce volume
                "exchange": 2 * (N - 1) / N * nl * db * wb,
                "decode": db * wb + (db * 8 if self.wl["sgd"] else db * 4)}


LR = 1e-3


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
    gpu = 0 if os.environ.get("GQ_BENCH_SHARED_GPU") == "1" else local_rank  # test mode: every rank on cuda:0
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    use_dist = world > 1 or args.engine == "dist"
    if use_dist and "RANK" not in os.environ:  # --engine dist without torchrun: a 1-rank group
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(port))
    if use_dist:
        # keep stdout to the one JSON line (NCCL otherwise prints its version banner there)
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    n, d = wl["n"], wl["d"]
    if n % world:
        raise SystemExit("workers must divide evenly over ranks")
    n_local = n // world
    workers = list(range(rank * n_local, (rank + 1) * n_local))

    L = _lib.lib()
    _lib.check(L.gq_set_option(_lib.GQ_OPT_QUANT_CTAS_PER_SM, args.quant_ctas))
    _lib.check(L.gq_set_option(_lib.GQ_OPT_REDUCE_CTAS_PER_SM, args.reduce_ctas))
    _lib.check(L.gq_set_option(_lib.GQ_OPT_SMALL_PATH, args.small_path))
    width = wl["width"]
    plan = G.plan_path(G.GqsgdConfig(workers=n, scheme=G.LevelKind(wl["kind"]), s=wl["s"], width_bits=width,
                                     topo=G.TopologyKind(wl["topo"]), seed=wl["seed"]))
    assert plan.lane_width == width
    stream = torch.cuda.Stream(dev)
    sp = stream.cuda_stream

    # Synthetic gradients in HBM, one generator seed per GLOBAL worker, so a
    # worker's data does not depend on N (randn is plumbing; parity runs use
    # the reference's gaussian_shards instead).
    shards = []
    for w in workers:
        gen = torch.Generator(device=dev).manual_seed(12345 + w)
        shards.append(torch.randn(d, dtype=torch.float32, device=dev, generator=gen))
    mean = torch.zeros(d, dtype=torch.float32, device=dev)
    param = torch.zeros(d, dtype=torch.float32, device=dev) if wl["sgd"] else None
    bucket = wl["bucket"] or d
    nb = (d + bucket - 1) // bucket

    with torch.cuda.stream(stream):
        def make_engine(shard_set):
            if not use_dist:
                return InprocEngine(L, G, _lib, wl, shard_set, param, None if wl["sgd"] else mean, dev, sp, bucket,
                                    overlap=args.overlap, kdraws=bool(args.kdraws), small_path=args.small_path)
            return DistEngine(wl, shard_set, param, None if wl["sgd"] else mean, dev, stream, bucket,
                              args.exchange)
        eng = make_engine(shards)
        if use_dist and eng.mean is not None:
            mean = eng.mean
        for t in range(args.warmup):
            eng.step(t)
        eng.check()
        torch.cuda.synchronize()

        K = args.steps
        nph = len(eng.phases)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nph)] for _ in range(K)]
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        graph = None
        if args.graph and hasattr(eng, "make_graph"):
            graph = eng.make_graph(args.warmup)  # rounds warmup, warmup+1, ... as the eager loop
            if graph is not None:
                for _ in range(2):  # warm the graph (advances the device round; re-set below)
                    eng.graph_step()
                eng.reset_graph_round(args.warmup)
                torch.cuda.synchronize()
        flush = L2Flusher(dev, l2_flush(n_local, d))
        step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(gpu) as clk:
            start.record(stream)
            for t in range(K):
                if flush.buf is not None:
                    with torch.cuda.stream(stream):
                        flush()
                    step_ev[t][0].record(stream)
                if graph is not None:
                    eng.graph_step()
                else:
                    eng.step(args.warmup + t, evs[t])
                if flush.buf is not None:
                    step_ev[t][1].record(stream)
            stop.record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        eng.check()
        if flush.buf is not None:  # the steps alone, the flushes between them excluded
            ms = sum(a.elapsed_time(b) for a, b in step_ev) / K
        else:
            ms = start.elapsed_time(stop) / K
        if graph is not None:  # per-kernel times from an eager pass with event marks
            for t in range(K):
                with torch.cuda.stream(stream):
                    flush()
                eng.step(args.warmup + t, evs[t])
            torch.cuda.synchronize()
            eng.check()
        if use_dist:  # DistSync records the 5 boundaries into slots 0,1,3,5,7
            for e in evs:
                e[2], e[4], e[6] = e[1], e[3], e[5]
        ph_ms = {p: sum(e[2 * i].elapsed_time(e[2 * i + 1]) for e in evs) / K for i, p in enumerate(eng.phases)}
        if world > 1:
            tt = torch.tensor([ms] + [ph_ms[p] for p in eng.phases], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt[0].item()
            ph_ms = {p: tt[i + 1].item() for i, p in enumerate(eng.phases)}

        # fp32 uncompressed comparator on the same shards: N = 1 tree-sum of the
        # n shards on this GPU; N > 1 local pre-sum + NCCL fp32 all_reduce.
        fp32_ms = None
        if not args.no_fp32:
            acc = torch.empty(bucket, dtype=torch.float32, device=dev)

            def fp32_step():
                for b in range(nb):
                    off = b * bucket
                    db = min(bucket, d - off)
                    if world == 1 or n_local > 1:
                        shp = _lib.ptr_array([x.data_ptr() + 4 * off for x in shards])
                        _lib.check(L.gq_baseline_mean_inproc(shp, n_local, db, 0, acc.data_ptr(), sp))
                    else:
                        acc[:db].copy_(shards[0][off:off + db])
                    if world > 1:
                        dist.all_reduce(acc[:db])
                        acc[:db].mul_(n_local / n)
            for _ in range(3):
                fp32_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            Kf = max(3, min(K, 20))
            fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(Kf)]
            for a, b_ in fev:  # the same L2 treatment as the timed steps
                with torch.cuda.stream(stream):
                    flush()
                a.record(stream)
                fp32_step()
                b_.record(stream)
            torch.cuda.synchronize()
            fp32_ms = sum(a.elapsed_time(b_) for a, b_ in fev) / Kf
            if world > 1:
                tt = torch.tensor([fp32_ms], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                fp32_ms = tt.item()

        # e2e through the public API with host buffers (pinned): every step copies
        # this rank's shards H2D and the step's result D2H inside the timed
        # region. Steps are pipelined the way a training loop overlaps them: the
        # H2D of step t+1 (copy stream, into the other of two shard buffers)
        # runs under the compute of step t and the D2H of step t-1 (a third
        # stream); parameters / results are shared, so the sync semantics are
        # unchanged.
        e2e = None
        if not args.no_e2e:
            host = [torch.empty(d, dtype=torch.float32, pin_memory=True) for _ in shards]
            for h, x in zip(host, shards):
                h.copy_(x.cpu())
            out_host = torch.empty(d, dtype=torch.float32, pin_memory=True)
            shards2 = [torch.empty_like(x) for x in shards]
            engines = [eng, make_engine(shards2)]
            shard_sets = [shards, shards2]
            results = [param if param is not None else (e.mean if use_dist else mean) for e in engines]
            s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            ev_h2d = [torch.cuda.Event() for _ in range(2)]
            ev_comp = [torch.cuda.Event() for _ in range(2)]
            ev_d2h = torch.cuda.Event()

            def e2e_step(t):
                i = t % 2
                s_h2d.wait_event(ev_comp[i])            # buffer i is no longer read
                with torch.cuda.stream(s_h2d):
                    for h, x in zip(host, shard_sets[i]):
                        x.copy_(h, non_blocking=True)
                ev_h2d[i].record(s_h2d)
                stream.wait_event(ev_h2d[i])
                stream.wait_event(ev_d2h)               # the shared result was read back
                engines[i].step(t)
                ev_comp[i].record(stream)
                s_d2h.wait_event(ev_comp[i])
                with torch.cuda.stream(s_d2h):
                    out_host.copy_(results[i], non_blocking=True)
                ev_d2h.record(s_d2h)
            for t in range(2):
                e2e_step(t)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            Ke = max(4, min(K, 10))
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s_h2d)
            for t in range(Ke):
                e2e_step(1000 + t)
            b_.record(s_d2h)
            torch.cuda.synchronize()
            e2e_ms = a.elapsed_time(b_) / Ke
            if world > 1:
                tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                e2e_ms = tt.item()
            for e in engines:
                e.check()
            e2e = {"value": d / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                   "h2d_bytes_per_step": n_local * d * 4, "d2h_bytes_per_step": d * 4,
                   "h2d_gbs": n_local * d * 4 / (e2e_ms * 1e-3) / 1e9,
                   "path": "pinned host shards -> H2D (copy stream, double-buffered) -> "
                           + ("gq_* C ABI" if not use_dist else "dist.DistSync")
                           + " -> D2H of the " + ("updated params" if param is not None else "decoded mean")
                           + " (third stream); steps pipelined"}

        # Multi-rank parity, outside the timed region: one more step (the graph
        # when one was timed) at round R must leave every rank with the bits of
        # the single-device path - rank 0 regenerates all n workers' shards and
        # runs gqsgd_mean bucket by bucket (rounds R*nb + b, SGD from zero).
        dist_check = None
        if use_dist:
            R = 777
            if param is not None:
                param.zero_()
            if graph is not None:
                eng.reset_graph_round(R)
                eng.graph_step()
            else:
                eng.step(R)
            eng.check()
            torch.cuda.synchronize()
            got = param if param is not None else eng.mean
            want = torch.zeros(d, dtype=torch.float32, device=dev)
            if rank == 0:
                allx = []
                for w in range(n):
                    gen = torch.Generator(device=dev).manual_seed(12345 + w)
                    allx.append(torch.randn(d, dtype=torch.float32, device=dev, generator=gen))
                cfg1 = G.GqsgdConfig(workers=n, scheme=G.LevelKind(wl["kind"]), s=wl["s"], width_bits=width,
                                     topo=G.TopologyKind(wl["topo"]), seed=wl["seed"])
                for b in range(nb):
                    off = b * bucket
                    db = min(bucket, d - off)
                    res = G.gqsgd_mean([x[off:off + db] for x in allx], cfg1, R * nb + b,
                                       param=want[off:off + db] if param is not None else None, lr=LR)
                    if param is None:
                        want[off:off + db].copy_(res.mean)
                del allx
                torch.cuda.synchronize()
            if world > 1:
                dist.broadcast(want, 0)
            same = torch.tensor([1 if torch.equal(want.view(torch.int32), got.view(torch.int32)) else 0],
                                device=dev)
            if world > 1:
                dist.all_reduce(same, op=dist.ReduceOp.MIN)
            dist_check = {"round": R, "checked": "updated params" if param is not None else "decoded mean",
                          "path": "cuda graph" if graph is not None else "eager",
                          "all_ranks_bit_identical_to_single_device": bool(same.item()), "exchange": eng.exchange}

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    link_peak = 770.0  # measured peer copy per direction, B200_PROFILING.md
    db0 = eng.buckets[0][0]
    kbytes = eng.alg_bytes(db0)
    dom = max(ph_ms, key=ph_ms.get)
    kernels = {}
    for p in eng.phases:
        gbs = kbytes[p] / (ph_ms[p] * 1e-3) / 1e9
        pk = link_peak if p == "exchange" else hbm_peak
        kernels[p] = {"ms": ph_ms[p], "alg_bytes": kbytes[p], "gbs": gbs, "frac": gbs / pk,
                      "bound": "nvlink" if p == "exchange" else "hbm"}
    achieved = kernels[dom]["gbs"]
    peak = link_peak if dom == "exchange" else hbm_peak
    step_bytes = sum(v for k, v in kbytes.items() if k != "exchange") * nb
    # DRAM bytes and issue utilisation are not measurable inside a timed run:
    # they come from the committed ncu --set full capture named in
    # profiles/traffic.json "source" (capture file and the commit it was taken at)
    traffic = issue = traffic_src = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        tj = json.loads(prof.read_text())
        traffic = tj.get(args.workload, {}).get(dom)
        issue = tj.get("issue_active_pct", {}).get(args.workload, {}).get(dom)
        src = tj.get("sources", {}).get(args.workload, tj.get("source", {}))
        traffic_src = (f"ncu --set full: {src.get('capture', '?')} @ commit {src.get('commit', '?')}"
                       if traffic is not None else None)

    cpu = None
    if not args.no_cpu and world == 1:
        # the workload itself (C2: the full d = 2^24 per worker) on the host
        # cores, a few calls (~10-30 s of CPU work)
        r = cpu_reference_sample(wl, budget_s=15.0, steps=8)
        per = sum(r["times"]) / len(r["times"])
        cpu = {"value": r["d_sample"] / per, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
               "sample": (f"gqsgd_mean n={r['n']} d={r['d_sample']} w={r['width']} (the workload's "
                          f"{'bucket' if wl['bucket'] else 'full size'}), {len(r['times'])} calls, "
                          f"{'Transport::Tcp, one thread per worker' if r['kind'] == 'reference' else '1 thread'}"),
               "same_config": r["same_config"],
               "also": cpu_reference_extras(wl)}

    # perf_model (perf_model.cpp) fed with this run's B200 numbers: gamma = the
    # fp32 sum kernel's throughput, omega = the quantized reduce's throughput
    # per original fp32 byte relative to it, delta = norm + quantize seconds
    # per original byte, beta = 770 GB/s NVLink (measured peer copy).
    perf = None
    if fp32_ms and not use_dist:
        from paper_2305_18627_b200.perf_model import b200_params, predict
        orig = n * d * 4.0
        red = ph_ms["reduce_decode"] * nb
        codec = (ph_ms["norm"] + ph_ms["quantize"]) * nb
        pm = b200_params(workers=n, size_bytes=d * 4.0, fp32_sum_bytes_per_s=orig / (fp32_ms * 1e-3),
                         quant_reduce_bytes_per_s=orig / (red * 1e-3), codec_s_per_byte=codec * 1e-3 / orig,
                         lane_bits=width)
        pr = predict(pm)
        perf = {"workers": pm.workers, "size_bytes": pm.size, "beta": pm.beta, "gamma": pm.gamma,
                "omega": pm.omega, "rho": pm.rho, "delta": pm.delta, "baseline_s": pr.baseline,
                "quantized_s": pr.quantized, "predicted_speedup": pr.speedup,
                "verdict": pr.threshold.verdict.value, "beta_max": pr.threshold.beta_max,
                "what": "reference perf_model (alpha-beta-gamma ring) with B200-measured omega/gamma/delta, "
                        "beta = 770 GB/s NVLink, predicting the n-GPU sync vs an fp32 allreduce"}

    value = d / (ms * 1e-3)  # d/t, fp32 gradient elements synchronised per second
    line = {
        "metric": METRIC, "value": value, "value_n_times_d": n * d / (ms * 1e-3),
        "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32-in/u%d-lanes/f64-scale" % width,
        "data": "synthetic (torch.randn fp32 gradients resident in HBM)",
        "config": config_of(wl, world, n_local, eng),
        "execution": {"parallelism": f"dp{n}: {n_local} worker(s) on each of {world} GPU(s)",
                      "exchange": "in-device schedule replay" if not use_dist else eng.exchange,
                      "overlap": (2 if getattr(eng, "overlap_reduce", False) else 1 if getattr(eng, "overlap", False)
                                  else 0),
                      "kdraws_in_norm_pass": (getattr(eng, "kd", None) is not None) if not use_dist else (
                          eng.exchange == "p2p" and wl["kind"] == 1 and width in (4, 8) and wl["topo"] == 0
                          and n in (2, 4, 8) and wl["s"] + 1 <= 32),
                      "cuda_graph": graph is not None,
                      "fused_small_step": bool(getattr(eng, "fused", False)) and graph is not None,
                      "ctas_per_sm": {"quantize": args.quant_ctas or "auto", "reduce": args.reduce_ctas or "auto"}},
        "roofline": {"bound": "nvlink" if dom == "exchange" else "hbm", "kernel": dom, "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     # the same ncu capture's issue-slot utilisation: what bounds a kernel
                     # that is below the HBM roofline (quantize: one hash per element)
                     "ncu_issue_active_pct": issue, "traffic_source": traffic_src,
                     "peak_source": peak_src if dom != "exchange" else "770 GB/s measured peer copy (B200_PROFILING.md)",
                     "alg_bytes_per_launch": kbytes[dom],
                     "step_hbm_alg_bytes": step_bytes, "step_hbm_gbs": step_bytes / (ms * 1e-3) / 1e9,
                     # the whole step's SURVEY §8(d) bytes against the same peak (north star: >= 0.70 at C4)
                     "step_hbm_frac": step_bytes / (ms * 1e-3) / 1e9 / hbm_peak},
        "kernels": kernels,
        "kernels_from": ("an eager pass of the three kernels with event marks (the timed step is one fused "
                         "cooperative kernel)" if getattr(eng, "fused", False) and graph is not None
                         else "an eager pass with CUDA-event marks around each phase"),
        # graphs add no kernels: the round / flag-epoch counters advance inside
        # the reduce (last block) and the flag kernels
        "gpu_launches": eng.launches_per_step * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "fp32_baseline": ({"what": ("uncompressed fp32 tree-sum of the n shards on the same GPU" if world == 1
                                    else "uncompressed fp32 NCCL all_reduce (+ local pre-sum) of the same shards"),
                           "ms_per_step": fp32_ms, "value": d / (fp32_ms * 1e-3), "unit": UNIT}
                          if fp32_ms else None),
        "perf_model": perf,
        "clocks": clk.summary(),
    }
    if dist_check is not None:
        line["dist_check"] = dist_check
    print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

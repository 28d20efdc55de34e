"""The reference's ring-allreduce cost model (perf_model.hpp/.cpp), restated
for host-side use, plus its parameters measured on B200.

    reference                                   here
    CostParams        perf_model.hpp:12-21      CostParams
    baseline_cost     perf_model.cpp:20-25      baseline_cost
    quantized_cost    perf_model.cpp:27-34      quantized_cost
    speedup_threshold perf_model.cpp:48-68      speedup_threshold
    predict           perf_model.cpp:70-78      predict

`b200_params(...)` fills the model with numbers measured on this hardware
(bench.py reports it): gamma = native fp32 reduction throughput (the fp32
sum kernel's bytes/s), omega = quantized reduction throughput / gamma (the
device token / integer reduce kernel, per original fp32 byte), beta = the
measured NVLink peer bandwidth, delta = codec seconds per original byte (norm
+ quantize + decode). Pure host arithmetic: no kernels here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

from ._lib import InvalidArgument


@dataclass
class CostParams:
    """perf_model.hpp:12-21 (defaults are the reference's)."""
    alpha: float = 1e-6      # per-hop latency, s
    beta: float = 53.9e9     # link bandwidth, B/s
    gamma: float = 2000e9    # native reduction throughput, B/s
    omega: float = 1.0       # quantized reduction relative throughput
    rho: float = 4.0         # compression ratio
    delta: float = 0.0       # codec overhead, s per original byte
    workers: int = 16
    size: float = 100e6      # payload bytes per worker


def _validate(p: CostParams) -> None:  # perf_model.cpp:10-16
    if (p.alpha < 0 or p.beta <= 0 or p.gamma <= 0 or p.omega <= 0 or p.omega > 1.0 or p.rho <= 0
            or p.delta < 0 or p.workers < 2 or p.size <= 0):
        raise InvalidArgument("cost parameters out of range")


def baseline_cost(p: CostParams) -> float:
    """2 log2(N) alpha + 2 log2(N) S / beta + log2(N) S / gamma (perf_model.cpp:20-25)."""
    _validate(p)
    hops = math.log2(p.workers)
    return 2.0 * hops * p.alpha + 2.0 * hops * p.size / p.beta + hops * p.size / p.gamma


def quantized_cost(p: CostParams) -> float:
    """Same shape on S / rho at omega * gamma, plus delta * S (perf_model.cpp:27-34)."""
    _validate(p)
    hops = math.log2(p.workers)
    s_hat = p.size / p.rho
    gamma_hat = p.omega * p.gamma
    return 2.0 * hops * p.alpha + 2.0 * hops * s_hat / p.beta + hops * s_hat / gamma_hat + p.delta * p.size


class SpeedupVerdict(Enum):
    Always = "Always"
    Never = "Never"
    Threshold = "Threshold"


@dataclass
class SpeedupThreshold:
    verdict: SpeedupVerdict = SpeedupVerdict.Threshold
    beta_max: float = 0.0


def speedup_threshold(omega: float, rho: float, gamma: float) -> SpeedupThreshold:
    """quantized < baseline iff beta < 2 omega (rho-1) / (1 - omega rho) gamma (perf_model.cpp:48-68)."""
    if omega <= 0 or omega > 1.0 or rho <= 0 or gamma <= 0:
        raise InvalidArgument("cost parameters out of range")
    if rho <= 1.0:
        return SpeedupThreshold(SpeedupVerdict.Never)
    if omega * rho >= 1.0:
        return SpeedupThreshold(SpeedupVerdict.Always)
    return SpeedupThreshold(SpeedupVerdict.Threshold, 2.0 * omega * (rho - 1.0) / (1.0 - omega * rho) * gamma)


@dataclass
class Prediction:
    baseline: float = 0.0
    quantized: float = 0.0
    speedup: float = 0.0
    beats_baseline: bool = False
    threshold: SpeedupThreshold = field(default_factory=SpeedupThreshold)


def predict(p: CostParams) -> Prediction:
    """perf_model.cpp:70-78"""
    b, q = baseline_cost(p), quantized_cost(p)
    return Prediction(b, q, b / q, q < b, speedup_threshold(p.omega, p.rho, p.gamma))


def b200_params(*, workers: int, size_bytes: float, fp32_sum_bytes_per_s: float,
                quant_reduce_bytes_per_s: float, codec_s_per_byte: float, lane_bits: int,
                beta: float = 770e9, alpha: float = 5e-6) -> CostParams:
    """CostParams from B200 measurements. Throughputs are per ORIGINAL fp32
    byte reduced (so omega compares like with like); rho = 32 / lane_bits;
    beta defaults to the measured 770 GB/s peer copy (B200_PROFILING.md)."""
    gamma = fp32_sum_bytes_per_s
    omega = min(1.0, quant_reduce_bytes_per_s / gamma)
    return CostParams(alpha=alpha, beta=beta, gamma=gamma, omega=omega, rho=32.0 / lane_bits,
                      delta=codec_s_per_byte, workers=workers, size=size_bytes)

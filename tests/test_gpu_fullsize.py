"""North-star sizes against the reference's own fingerprints.

tests/golden/make_golden.py (LARGE) ran the UNMODIFIED reference
(oracle/_ref: gqsgd_mean, quantize_shard + encode, allreduce_inproc) on
columns [j0, j0+d) of gaussian_shards(n, D, 12345) cast to fp32 and stored
SHA-256 fingerprints of every output:

  C3: the 25.6M-element ResNet-50 gradient, standard s = 63/31/15 at
      n = 2/4/8 (8-bit lanes), one call (round 0);
  C4: the 340M-element BERT-large gradient in 25 MiB buckets, n = 8,
      standard s = 15 (and exponential s = 7) 8-bit; bucket b of step t = 3 is
      the call with round t*52 + b (buckets 0, 1 and the short last bucket 51),
      its decode feeding the SGD line x[j] -= eta*est[j] (trainer.cpp:335) of
      a fixed fp32 parameter vector.

The device must reproduce the lanes of every worker, the summed lanes, the
f64 mean (gq_dequant_f64) and fl32 of it bit for bit. The fused fp32 SGD
update equals fl32(p - fl32(lr * fl32(mean))) bit for bit (the kernel's
separate mul then sub) and the reference's f64 update within 1e-6 relative
to the operands of the subtraction.
"""
import ctypes as C
import hashlib

import numpy as np
import pytest
import torch

from paper_2305_18627_b200 import _lib
from paper_2305_18627_b200 import gqsgd as G
from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind, TopologyKind

pytestmark = pytest.mark.gpu
REL_TOL = 1e-6
SGD_LR = np.float32(1e-3)   # tests/golden/make_golden.py SGD_LR
C3 = ["C3_std_s63_n2_d25.6M", "C3_std_s31_n4_d25.6M", "C3_std_s15_n8_d25.6M"]
C4 = ["C4_std_s15_n8_bucket0", "C4_std_s15_n8_bucket1", "C4_std_s15_n8_bucket51", "C4_exp_s7_n8_bucket51"]


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _payload(lanes: torch.Tensor, d: int, width: int) -> np.ndarray:
    return lanes.cpu().numpy()[: (d * width + 7) // 8]


def _inputs(oracle, f):
    x = oracle.gaussian_range(f["n"], f["j0"], f["d"], f["data_seed"]).astype(np.float32)
    assert _sha(x) == f["x_sha"]
    return x


def _cfg(f):
    return GqsgdConfig(workers=f["n"], scheme=LevelKind(f["kind"]), s=f["s"], width_bits=f["width"],
                       topo=TopologyKind(f["topo"]), seed=f["seed"])


def _mean_f64(lanes: torch.Tensor, f, norm: torch.Tensor) -> np.ndarray:
    out = torch.empty(f["d"], dtype=torch.float64, device=lanes.device)
    err = torch.zeros(1, dtype=torch.int32, device=lanes.device)
    L = _lib.lib()
    _lib.check(L.gq_dequant_f64(lanes.data_ptr(), 0, f["d"], norm.data_ptr(), f["kind"], f["s"], f["n"],
                                f["width"], out.data_ptr(), err.data_ptr(), torch.cuda.current_stream().cuda_stream))
    _lib.check(L.gq_check(err.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy()


def _check_sync(eng, f, x):
    n, d, w = f["n"], f["d"], f["width"]
    assert eng.norm.item() == f["norm"]
    for r in range(n):
        assert _sha(_payload(eng.lane_bufs[r], d, w)) == f["lanes_sha"][r], f"worker {r} lanes"
    assert _sha(_payload(eng.result_lanes, d, w)) == f["summed_sha"]
    assert _sha(eng.mean.cpu().numpy()) == f["mean_f32_sha"]
    m64 = _mean_f64(eng.result_lanes, f, eng.norm)
    assert _sha(m64) == f["mean_f64_sha"]
    return m64


@pytest.mark.parametrize("name", C3)
def test_c3_full_size_matches_reference(cuda, oracle, fingerprints, name):
    f = fingerprints[name]
    x = _inputs(oracle, f)
    eng = G.InprocSync(_cfg(f), f["d"], cuda)
    shards = [torch.from_numpy(x[r]).to(cuda) for r in range(f["n"])]
    eng.run(shards, f["round"])
    eng.check()
    _check_sync(eng, f, x)
    # the one-launch graph of the same sync gives the same bits
    eng.mean.zero_()
    g = eng.graph(shards, f["round"])
    g.launch()
    eng.check()
    torch.cuda.synchronize()
    assert _sha(eng.mean.cpu().numpy()) == f["mean_f32_sha"]


@pytest.mark.parametrize("name", C4)
def test_c4_bucket_with_sgd_matches_reference(cuda, oracle, fingerprints, name):
    f = fingerprints[name]
    x = _inputs(oracle, f)
    p0 = oracle.gaussian_range(1, f["j0"], f["d"], f["sgd_param_seed"])[0].astype(np.float32)
    assert _sha(p0) == f["param0_sha"] and np.float32(f["sgd_lr"]) == SGD_LR
    eng = G.InprocSync(_cfg(f), f["d"], cuda)
    param = torch.from_numpy(p0.copy()).to(cuda)
    eng.run([torch.from_numpy(x[r]).to(cuda) for r in range(f["n"])], f["round"], param=param, lr=float(SGD_LR))
    eng.check()
    m64 = _check_sync(eng, f, x)
    got = param.cpu().numpy()
    assert _sha(got) == f["param_f32_sha"]
    # the reference's f64 update x -= eta * est (trainer.cpp:335), within the fp32
    # tolerance relative to the operands of the subtraction (the result itself
    # can cancel to ~0)
    step = np.float64(SGD_LR) * m64
    want = p0.astype(np.float64) - step
    assert np.all(np.abs(got.astype(np.float64) - want) <= REL_TOL * (np.abs(p0) + np.abs(step)))


def test_c4_buckets_through_the_multi_rank_path(cuda, oracle, fingerprints):
    """Bucket 51 (the short last bucket, round 207) through DistSync at world 2
    (two ranks as threads on this GPU, NCCL-free ThreadComm): the SGD params
    on both ranks carry the reference's fingerprint."""
    import threading

    from dist_fakes import ThreadComm
    from paper_2305_18627_b200.dist import DeviceKernels, DistSync

    f = fingerprints["C4_std_s15_n8_bucket51"]
    x = _inputs(oracle, f)
    p0 = oracle.gaussian_range(1, f["j0"], f["d"], f["sgd_param_seed"])[0].astype(np.float32)
    world = 2
    comms = ThreadComm.group(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(cuda)
            eng = DistSync(_cfg(f), f["d"], comm=comms[r], kernels=DeviceKernels(cuda), device=cuda,
                           exchange="pull")
            mine = [torch.from_numpy(x[w].copy()).to(cuda) for w in eng.worker_ids]
            param = torch.from_numpy(p0.copy()).to(cuda)
            eng.run(mine, f["round"], param=param, lr=float(SGD_LR))
            eng.check()
            torch.cuda.synchronize()
            out[r] = param.cpu().numpy()
        except BaseException as e:
            errs.append(e)
            comms[r].sh.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    for r in range(world):
        assert _sha(out[r]) == f["param_f32_sha"], f"rank {r}"

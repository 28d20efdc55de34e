"""The reference's own C++ API with the GPU path swapped in.

oracle/_ref/dropin_check and oracle/_ref/acceptance_b200 are built here by
integration/Makefile against the reference sources (they travel to the GPU
box as built binaries; /root/reference is not needed at run time):
  - dropin_check: gqsgd_b200::{DeviceIntSumOps, DeviceTokenReduceOps,
    quantize_shard, gqsgd_mean} vs the unmodified reference, bit for bit;
  - acceptance_b200: the reference's release acceptance gate
    (proj/tests/acceptance.cpp) with gqsgd::gqsgd_mean routed to the GPU;
  - comm_example: the communicator C ABI from plain C (no reference code).
"""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


def _run(name, timeout):
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    return subprocess.run([str(exe)], capture_output=True, text=True, timeout=timeout)


def test_dropin_check(cuda):
    p = _run("dropin_check", 600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "FAIL" not in p.stdout


def test_reference_acceptance_on_gpu_core(cuda):
    p = _run("acceptance_b200", 1500)
    print(p.stdout)
    lines = [l for l in p.stdout.splitlines() if "criterion-" in l]
    assert len(lines) == 12, p.stdout + p.stderr
    failed = [l for l in lines if not l.startswith("PASS")]
    assert not failed, "\n".join(failed)


def test_comm_abi_from_plain_c(cuda):
    """integration/comm_example.c: the communicator C ABI driven from C by two
    forked processes (file-based handle exchange); both ranks' means equal the
    single-device gq_mean_inproc bit for bit."""
    p = _run("comm_example", 300)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "PASS comm_example" in p.stdout

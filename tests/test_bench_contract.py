"""The bench.py JSON contract that needs no GPU: the reference arm (the
unmodified reference library, oracle/_ref, on the host cores) and the config
dict both arms must share so the driver's ratio is a same-config ratio."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _reference_built() -> bool:
    from oracle.bind import reference_or_none
    return reference_or_none() is not None


@pytest.mark.skipif(not _reference_built(), reason="reference library not built")
def test_reference_arm_line_is_same_config():
    import bench
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "2",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    wl = bench.WORKLOADS["c1"]
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["higher_is_better"] is True
    assert line["same_config"] is True and line["config"] == bench.config_of(wl, 1, wl["n"], None)
    assert line["steps"] == 2 and line["value"] > 0
    # d/t: the line's value is fp32 gradient elements synced per second
    assert line["value"] == pytest.approx(wl["d"] / (line["ms_per_step"] * 1e-3), rel=1e-9)
    assert line["value_n_times_d"] == pytest.approx(wl["n"] * line["value"], rel=1e-12)
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": bench.UNIT, "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_print_nothing():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, RANK="1", WORLD_SIZE="2", CUDA_VISIBLE_DEVICES=""))
    assert p.returncode == 0 and not [ln for ln in p.stdout.splitlines() if ln.startswith("{")]


def test_algorithmic_bytes_follow_survey():
    """SURVEY §8(d) bytes only: no k-draw buffer, no mean write under the fused SGD."""
    import bench
    eng = bench.InprocEngine.__new__(bench.InprocEngine)
    eng.n = 8
    eng.wl = dict(bench.WORKLOADS["c2"])
    b = eng.alg_bytes(1 << 24)
    d = 1 << 24
    assert b == {"norm": 8 * d * 4, "quantize": 8 * d * 4.5, "reduce_decode": 8 * d * 0.5 + d * 4}
    eng.wl = dict(bench.WORKLOADS["c4"])
    db = bench.WORKLOADS["c4"]["bucket"]
    b = eng.alg_bytes(db)
    assert b["reduce_decode"] == 8 * db * 1 + db * 8  # lanes + param read/write, no mean


def test_l2_flush_rule_and_config_field():
    """Inputs smaller than twice the 126 MB L2 are flushed between timed steps
    (and the config says so); C2 / C4 stream from HBM without one."""
    import bench
    assert bench.l2_flush(4, 1 << 20)            # C1: 16 MiB
    assert bench.l2_flush(2, 25_600_000)          # C3 n=2: 205 MB
    assert not bench.l2_flush(4, 25_600_000)      # C3 n=4: 410 MB
    assert not bench.l2_flush(8, 1 << 24)         # C2: 512 MiB
    assert not bench.l2_flush(8, 340_000_000)     # C4: the whole 340M gradient per step
    for name, flushed in (("c1", True), ("c2", False), ("c3n2", True), ("c3n8", False)):
        wl = bench.WORKLOADS[name]
        l2 = bench.config_of(wl, 1, wl["n"], None)["l2"]
        assert ("write (then read back) between" in l2) == flushed, (name, l2)

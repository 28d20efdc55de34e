"""perf_model restatement pinned to the reference's own goldens
(proj/tests/test_perf_model.cpp) and to the compiled reference."""
import math

import pytest

from paper_2305_18627_b200.perf_model import (CostParams, SpeedupVerdict, b200_params, baseline_cost,
                                              predict, quantized_cost, speedup_threshold)


def test_cost_goldens():  # test_perf_model.cpp:13-27
    p = CostParams(omega=1.0 / 79.0, rho=4.0)
    assert baseline_cost(p) == pytest.approx(0.015050300556586271, rel=1e-14)
    assert quantized_cost(p) == pytest.approx(0.007668575139146568, rel=1e-14)
    pr = predict(p)
    assert pr.speedup == pytest.approx(1.9625941303955472, rel=1e-12)
    assert pr.beats_baseline and pr.threshold.verdict == SpeedupVerdict.Threshold
    assert pr.threshold.beta_max == pytest.approx(1.6e11, rel=1e-12)


def test_threshold_is_008_gamma():  # test_perf_model.cpp:29-36
    for gamma in (1.0, 2000e9, 3.5e12):
        t = speedup_threshold(1.0 / 79.0, 4.0, gamma)
        assert t.verdict == SpeedupVerdict.Threshold
        assert t.beta_max == pytest.approx(0.08 * gamma, rel=1e-12)


def test_verdicts():  # test_perf_model.cpp:51-65
    assert speedup_threshold(1.0, 4.0, 1e9).verdict == SpeedupVerdict.Always
    assert speedup_threshold(0.25, 4.0, 1e9).verdict == SpeedupVerdict.Always
    assert speedup_threshold(0.2, 1.0, 1e9).verdict == SpeedupVerdict.Never
    assert speedup_threshold(1.0, 0.5, 1e9).verdict == SpeedupVerdict.Never
    assert speedup_threshold(0.1, 2.0, 1e9).verdict == SpeedupVerdict.Threshold


def test_threshold_is_the_crossing():  # test_perf_model.cpp:67-85
    t = speedup_threshold(0.1, 2.0, 1e9)
    assert t.beta_max == pytest.approx(0.25e9, rel=1e-12)
    p = CostParams(workers=4, size=1e6, gamma=1e9, omega=0.1, rho=2.0, beta=0.999 * t.beta_max)
    assert quantized_cost(p) < baseline_cost(p)
    p.beta = 1.001 * t.beta_max
    assert quantized_cost(p) > baseline_cost(p)


def test_out_of_range():
    with pytest.raises(ValueError):
        baseline_cost(CostParams(workers=1))
    with pytest.raises(ValueError):
        speedup_threshold(1.5, 4.0, 1.0)


def test_b200_params_shape():
    p = b200_params(workers=8, size_bytes=1.36e9, fp32_sum_bytes_per_s=4e12, quant_reduce_bytes_per_s=2e12,
                    codec_s_per_byte=1e-13, lane_bits=8)
    assert p.rho == 4.0 and p.omega == 0.5 and p.beta == 770e9
    assert math.isfinite(predict(p).speedup)

"""Quality metrics on the GPU: sliced-W2 / MMD / permutation
threshold / trajectory deviation vs the reference's values on the same inputs
(tests/golden/metrics.json, made by importing the reference), the reference's
own metric tests (test_metrics.py), its distributional-quality acceptance
check (test_acceptance.py:206-229, 10^4 samples through the device samplers)
and a latent-size MMD that the reference's dense numpy form cannot hold."""

import json
import math
import os
import sys

import numpy as np
import pytest
import torch

from paper_2603_25872_b200 import (AnalyticEps, GaussianMixture, RngStream, Role, SampleSet, VarianceRule,
                                   default_schedule, derive_noise, mmd_gaussian, mmd_permutation_threshold,
                                   run_aggressive, run_conservative, sample_ddim, sliced_w2, trajectory_max_dev)
from paper_2603_25872_b200.errors import DimensionMismatch, EmptySet, InsufficientSamples, TimestepMismatch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from metric_cases import metric_inputs  # noqa: E402


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "metrics.json")) as f:
        return json.load(f)


def test_metrics_match_reference(cuda, gold):
    for c in gold:
        a, b = metric_inputs(c["seed"], c["n_a"], c["n_b"], c["dim"], c["shift"])
        A, B = SampleSet(torch.from_numpy(a).to(cuda)), SampleSet(torch.from_numpy(b).to(cuda))
        w2 = sliced_w2(A, B, projections=c["projections"], seed=c["w2_seed"])
        assert w2 == pytest.approx(c["sliced_w2"], rel=1e-12), c["name"]
        mmd = mmd_gaussian(A, B, c["bandwidth"])
        assert mmd == pytest.approx(c["mmd"], rel=1e-10), c["name"]
        thr = mmd_permutation_threshold(A, B, c["bandwidth"], permutations=20, seed=c["w2_seed"])
        assert thr == pytest.approx(c["threshold"], rel=1e-9), c["name"]


def _loop_sliced_w2(a, b, projections, seed):
    """Independent numpy check: one direction at a time, quantile pairing."""
    rng = np.random.default_rng(seed)
    total = 0.0
    dirs = rng.standard_normal((projections, a.shape[1]))
    m = min(len(a), len(b))
    qs = (np.arange(m) + 0.5) / m
    for d in dirs:
        d = d / np.linalg.norm(d)
        pa, pb = np.sort(a @ d), np.sort(b @ d)
        qa = pa if len(pa) == m else np.quantile(pa, qs)
        qb = pb if len(pb) == m else np.quantile(pb, qs)
        total += float(np.mean((qa - qb) ** 2))
    return total / projections


class TestSlicedW2:
    """reference test_metrics.py:38-80"""

    def test_identical_sets_are_zero(self, cuda):
        x = np.random.default_rng(0).normal(size=(100, 3))
        assert sliced_w2(SampleSet(x), SampleSet(x.copy())) == 0.0

    @pytest.mark.parametrize("na,nb", [(80, 80), (120, 50)])
    def test_matches_loop_form(self, cuda, na, nb):
        rng = np.random.default_rng(na + nb)
        a, b = rng.normal(size=(na, 2)), rng.normal(1.0, 2.0, size=(nb, 2))
        got = sliced_w2(SampleSet(a), SampleSet(b), projections=16, seed=9)
        assert got == pytest.approx(_loop_sliced_w2(a, b, 16, 9), rel=1e-12)

    def test_1d_shift_closed_form(self, cuda):
        a = np.random.default_rng(3).normal(size=(200, 1))
        assert sliced_w2(SampleSet(a), SampleSet(a + 1.5), projections=8, seed=0) == pytest.approx(2.25, rel=1e-12)

    def test_deterministic_in_seed(self, cuda):
        rng = np.random.default_rng(4)
        a, b = SampleSet(rng.normal(size=(50, 2))), SampleSet(rng.normal(size=(50, 2)))
        v1, v2, v3 = sliced_w2(a, b, seed=7), sliced_w2(a, b, seed=7), sliced_w2(a, b, seed=8)
        assert v1 == v2 and v1 != v3

    def test_errors(self, cuda):
        a = SampleSet(np.zeros((4, 2)))
        with pytest.raises(DimensionMismatch):
            sliced_w2(a, SampleSet(np.zeros((4, 3))))
        with pytest.raises(ValueError):
            sliced_w2(a, a, projections=0)
        with pytest.raises(EmptySet):
            SampleSet(np.zeros((0, 2)))


class TestMmd:
    """reference test_metrics.py:83-140"""

    def test_hand_cases(self, cuda):
        k = lambda d: math.exp(-d * d / 2.0)   # noqa: E731
        assert mmd_gaussian(SampleSet([[0.0], [1.0]]), SampleSet([[0.0], [1.0]]), 1.0) == pytest.approx(k(1) - 1.0,
                                                                                                          rel=1e-12)
        expected = 2 * k(1) - 2 * (k(2) + k(3) + k(1) + k(2)) / 4
        got = mmd_gaussian(SampleSet([[0.0], [1.0]]), SampleSet([[2.0], [3.0]]), 1.0)
        assert got == pytest.approx(expected, rel=1e-12)

    def test_bandwidth_to_infinity_vanishes(self, cuda):
        rng = np.random.default_rng(5)
        assert abs(mmd_gaussian(SampleSet(rng.normal(size=(30, 2))), SampleSet(rng.normal(3.0, 1.0, size=(30, 2))),
                                1e8)) < 1e-10

    def test_permutation_null(self, cuda):
        rng = np.random.default_rng(7)
        a, b = SampleSet(rng.normal(size=(80, 1))), SampleSet(rng.normal(2.0, 1.0, size=(80, 1)))
        assert mmd_gaussian(a, b, 1.0) > mmd_permutation_threshold(a, b, 1.0, permutations=100)
        rng = np.random.default_rng(8)
        a, b = SampleSet(rng.normal(size=(80, 1))), SampleSet(rng.normal(size=(80, 1)))
        assert mmd_gaussian(a, b, 1.0) <= mmd_permutation_threshold(a, b, 1.0, permutations=100)

    def test_errors(self, cuda):
        a = SampleSet(np.zeros((4, 2)))
        with pytest.raises(ValueError):
            mmd_gaussian(a, a, 0.0)
        with pytest.raises(InsufficientSamples):
            mmd_gaussian(SampleSet([[0.0, 0.0]]), a, 1.0)

    def test_latent_scale(self, cuda):
        """10^4 x 16,384-D (C3-sized latents): 2.6 GB per dense kernel matrix in
        the reference's form; K10 streams the pairs.  Same-distribution MMD ~ 0."""
        g = torch.Generator(device=cuda).manual_seed(0)
        a = torch.randn(10_000, 16_384, device=cuda, generator=g, dtype=torch.float64)
        b = torch.randn(10_000, 16_384, device=cuda, generator=g, dtype=torch.float64)
        v = mmd_gaussian(SampleSet(a), SampleSet(b), 128.0)
        assert math.isfinite(v) and abs(v) < 1e-3


def test_trajectory_max_dev(cuda):
    s = default_schedule(10)
    den = AnalyticEps(GaussianMixture(weights=[1.0], means=[[0.0, 0.0]], variances=[1.0]))
    x = torch.tensor([1.0, -1.0], dtype=torch.float64, device=cuda)
    t1 = sample_ddim(s, den, x, VarianceRule.deterministic(), RngStream(0))
    t2 = sample_ddim(s, den, x + 0.5, VarianceRule.deterministic(), RngStream(0))
    dev = trajectory_max_dev(t1, t2)
    ref = max(float(torch.linalg.vector_norm(a - b)) for (_, a), (_, b) in zip(t1.states, t2.states))
    assert dev == ref
    t3 = sample_ddim(default_schedule(5), den, x, VarianceRule.deterministic(), RngStream(0))
    with pytest.raises(TimestepMismatch):
        trajectory_max_dev(t1, t3)


def test_distributional_quality(cuda):
    """reference test_acceptance.py:206-229: 10^4 samples of a 2-D mixture,
    T=50 deterministic DDIM; sliced-W2 of each parallel mode (devices=4) vs
    sequential stays within 2x the seed-to-seed null."""
    n = 10_000
    s = default_schedule(50)
    den = AnalyticEps(GaussianMixture(weights=[0.5, 0.5], means=[[-2.0, 0.0], [2.0, 0.0]], variances=[1.0, 1.0]))
    rule = VarianceRule.deterministic()

    def batch(seed, runner=None):
        stream = RngStream(seed=seed)
        x_T = derive_noise(stream, 50, Role.INIT, (n, 2), device=cuda)
        if runner is None:
            return sample_ddim(s, den, x_T, rule, stream).final
        return runner(s, den, x_T, 4, rule, stream)[0].final

    seq_a, seq_b = batch(0), batch(1)
    null = sliced_w2(SampleSet(seq_a), SampleSet(seq_b))
    assert sliced_w2(SampleSet(batch(0, run_aggressive)), SampleSet(seq_a)) <= 2 * null
    assert sliced_w2(SampleSet(batch(0, run_conservative)), SampleSet(seq_a)) <= 2 * null

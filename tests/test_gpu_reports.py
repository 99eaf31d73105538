"""The device samplers + writers reproduce the reference CLI's output files
(SURVEY 8f row 3): with the state-independent denoiser the samples CSV is
byte-identical (bit-exact sampler); the Euler mixture run matches to K9's
fp64 rounding; the rounds CSV's round/anchor_t/parallel_evals columns and the
eval/round totals are identical (wall times are this machine's)."""

import csv
import json
import os

import numpy as np
import pytest
import torch

from paper_2603_25872_b200 import (GaussianMixture, Mode, RngStream, Role, StateIndependent, VarianceRule,
                                   build_linear_beta, build_sigma_grid, derive_noise, run_aggressive,
                                   run_parallel_euler)
from paper_2603_25872_b200.reports import collect_runs, rounds_csv, samples_csv

pytestmark = pytest.mark.gpu
CLI = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


def _read(name):
    with open(os.path.join(CLI, name), newline="") as f:
        return f.read()


def _cols(text, n=3):
    return [r[:n] for r in csv.reader(text.splitlines())]


def test_si_sample_outputs_byte_identical(cuda):
    """golden/cli/si.cfg: linear schedule T=12 (0.002, 0.4), SI seed 11, dim 16,
    DDIM aggressive n=3, ddpm rule, seeds 4..6."""
    s = build_linear_beta(12, 0.002, 0.4)
    den = StateIndependent(seed=11, dim=16)
    rule = VarianceRule.ddpm_induced()

    def run_once(seed):
        stream = RngStream(seed=seed)
        return run_aggressive(s, den, derive_noise(stream, 12, Role.INIT, 16, device=cuda), 3, rule, stream)

    finals, reports, totals = collect_runs(run_once, 4, 3)
    assert samples_csv(finals, 16) == _read("si_samples.csv")
    assert _cols(rounds_csv(reports)) == _cols(_read("si_rounds.csv"))
    ref = json.loads(_read("si_report.json"))["totals"]
    assert (totals["evals"], totals["rounds"]) == (ref["evals"], ref["rounds"])


def test_euler_sample_outputs(cuda):
    """golden/cli/eul.cfg: 2-D bimodal mixture, Euler N=9 on the default grid
    (0.02, 10, rho 3), conservative n=3, seeds 1..2, x_init = sigma_max * INIT noise."""
    g = build_sigma_grid(9, 0.02, 10.0, 3.0)
    gm = GaussianMixture(weights=[0.5, 0.5], means=[[-2.0, 0.0], [2.0, 0.0]], variances=[1.0, 1.0])

    def run_once(seed):
        x0 = g.sigmas[0] * derive_noise(RngStream(seed=seed), 9, Role.INIT, 2, device=cuda)
        return run_parallel_euler(g, gm, x0, 3, Mode.CONSERVATIVE)

    finals, reports, _ = collect_runs(run_once, 1, 2)
    got = list(csv.reader(samples_csv(finals, 2).splitlines()))
    ref = list(csv.reader(_read("eul_samples.csv").splitlines()))
    assert got[0] == ref[0] and [r[0] for r in got] == [r[0] for r in ref]
    np.testing.assert_allclose(np.array([[float(v) for v in r[1:]] for r in got[1:]]),
                               np.array([[float(v) for v in r[1:]] for r in ref[1:]]), rtol=1e-10, atol=0)
    assert _cols(rounds_csv(reports)) == _cols(_read("eul_rounds.csv"))

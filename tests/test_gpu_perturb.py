"""Perturbed-denoiser ablation on the GPU: the BLAKE2b key
kernel reproduces the reference's digests exactly, the device draw equals
_perturbation bit-for-bit, and Perturbed(state-independent) runs of the
parallel and sequential samplers reproduce the reference's trajectories
bit-for-bit (tests/golden/perturb.npz)."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from paper_2603_25872_b200 import (AnalyticEps, GaussianMixture, Perturbed, RngStream, Role, StateIndependent,
                                   VarianceRule, default_schedule, derive_noise, evaluate, run_aggressive,
                                   run_conservative, sample_ddim)
from paper_2603_25872_b200 import _lib
from paper_2603_25872_b200.denoiser import PERTURB_QUANTUM, _ptr_array, apply_perturbations

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "golden", "perturb.npz"))


def _sha(t):
    return hashlib.sha256(np.ascontiguousarray(t.cpu().numpy(), dtype=np.float64).tobytes()).hexdigest()


def test_blake2b_keys_match_reference(cuda, gold):
    n = len(gold["ts"])
    xs = [torch.from_numpy(gold[f"x{i}"]).to(cuda) for i in range(n)]
    for i in range(n):                     # rows of different lengths: one launch each
        keys = torch.zeros(_lib.ctypes.sizeof(_lib.DrsKey), dtype=torch.uint8, device=cuda)
        ts = torch.tensor([int(gold["ts"][i])], dtype=torch.int32, device=cuda)
        ptrs = _ptr_array([xs[i]], cuda)
        _lib.check(_lib.lib().drs_perturb_keys(ptrs.data_ptr(), ts.data_ptr(), 1, xs[i].numel(), PERTURB_QUANTUM,
                                               keys.data_ptr(), _lib.stream_ptr()), "drs_perturb_keys")
        k = _lib.DrsKey.from_buffer_copy(bytes(keys.cpu().numpy()))
        assert k.vals[0] & 0xFFFFFFFFFFFFFFFF == int(gold["digests"][i]) and k.n_vals == 1


def test_device_draw_equals_reference(cuda, gold):
    for i, t in enumerate(gold["ts"]):
        x = torch.from_numpy(gold[f"x{i}"]).to(cuda)
        got = apply_perturbations([0.3], x, int(t), torch.zeros_like(x))
        assert torch.equal(got.cpu(), torch.from_numpy(gold[f"pert{i}"]))


@pytest.mark.parametrize("idx", range(3))
def test_perturbed_trajectories_bit_exact(cuda, gold, idx):
    c = json.loads(str(gold["manifest"]))[idx]
    s = default_schedule(c["T"])
    rule = VarianceRule.deterministic() if c["rule"] == "det" else VarianceRule.ddpm_induced()
    den = Perturbed(StateIndependent(seed=c["si_seed"], dim=c["D"]), c["scale"])
    stream = RngStream(seed=c["seed"])
    x_T = derive_noise(stream, c["T"], Role.INIT, c["D"], device=cuda)
    if c["sampler"] == "aggressive":
        traj, rep = run_aggressive(s, den, x_T, c["devices"], rule, stream, update_family=c["family"])
    elif c["sampler"] == "conservative":
        traj, rep = run_conservative(s, den, x_T, c["devices"], rule, stream, update_family=c["family"])
    else:
        traj, rep = sample_ddim(s, den, x_T, rule, stream), []
    assert [_sha(x) for _, x in traj.states] == list(gold[f"{c['name']}_sha"])
    assert traj.eval_count == c["eval_count"] and len(rep) == c["rounds"]


def test_zero_scale_identity_and_bounded(cuda):
    """reference test_denoiser.py:186-205"""
    s = default_schedule(50)
    gm = GaussianMixture(weights=[1.0], means=[[0.0]], variances=[1.0])
    base = AnalyticEps(gm)
    x = torch.tensor([0.4], dtype=torch.float64, device=cuda)
    assert torch.equal(evaluate(Perturbed(base, 0.0), s, x, 7), evaluate(base, s, x, 7))
    wrapped = Perturbed(base, 0.1)
    first = evaluate(wrapped, s, x, 5)
    assert torch.equal(first, evaluate(wrapped, s, x, 5))
    rng = np.random.default_rng(3)
    worst = 0.0
    for _ in range(200):
        xx = torch.tensor(rng.normal(0, 1, 1), device=cuda)
        worst = max(worst, float((evaluate(wrapped, s, xx, 5) - evaluate(base, s, xx, 5)).abs().max()))
    assert 0 < worst < 0.1 * 6

"""Pin the oracle (oracle/) to the reference: golden fixtures produced by
running skipdiff itself (tests/golden/make_golden.py) and the frozen numbers
of the reference's own test suite.  CPU only."""

import hashlib
import json
import math
import os

import numpy as np
import pytest

import noise_restated as NR
import skipdiff_oracle as O


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def noise_gold(golden_dir):
    return np.load(os.path.join(golden_dir, "noise.npz"))


@pytest.fixture(scope="module")
def traj_gold(golden_dir):
    return np.load(os.path.join(golden_dir, "traj.npz"))


def _streams(z, gen):
    meta = json.loads(str(z[f"{gen}_meta"]))
    vals = z[f"{gen}_values"]
    off = 0
    for m in meta:
        yield tuple(m["key"]), m["n"], vals[off:off + m["n"]], m["paths"]
        off += m["n"]


@pytest.mark.parametrize("gen", ["pcg64", "sfc64"])
def test_oracle_noise_matches_golden(noise_gold, gen):
    for key, n, ref, _ in _streams(noise_gold, gen):
        got = O.rng_for(key, gen).standard_normal(n)
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), key


@pytest.mark.parametrize("gen", ["pcg64", "sfc64"])
def test_restated_noise_bit_exact_and_paths(noise_gold, gen):
    seen = set()
    for key, n, ref, paths in _streams(noise_gold, gen):
        vals, p = NR.draw(key, n, gen)
        assert np.array_equal(np.array(vals).view(np.uint64), ref.view(np.uint64)), key
        seen.update(paths)
    # the fixtures exercise every ziggurat path the device kernel implements
    assert {"fast", "wedge", "wedge-reject", "tail", "tail-retry"} <= seen


def test_si_golden_value(noise_gold):
    # tests/test_denoiser.py:162-165 of the reference
    np.testing.assert_allclose(noise_gold["si_golden_0_1_2"], [0.6596311229815894, -1.0995664042571076],
                               rtol=1e-15)
    assert np.array_equal(O.state_independent_eps(0, 1, 2), noise_gold["si_golden_0_1_2"])


def _run_case(m):
    T, D = m["T"], m["D"]
    ab = O.default_alpha_bar(T)
    rule = ("det",) if m["rule"] == "det" else ("ddpm",)
    eps = O.SI(m["si_seed"], D) if m["denoiser"] == "si" else O.toy_bimodal(D)
    x_T = O.derive_noise(m["seed"], T, O.INIT, D)
    if m["sampler"] == "seq_ddim":
        return O.sample_ddim(ab, eps, x_T, rule, m["seed"])
    if m["sampler"] == "seq_ddpm":
        return O.sample_ddpm(ab, eps, x_T, m["seed"])
    states, evals, rounds = O.run_parallel(ab, eps, x_T, m["devices"], m["sampler"], rule, m["seed"],
                                           family=m["family"])
    assert evals == m["eval_count"] and rounds == m["rounds"]
    return states


def test_oracle_trajectories_bit_exact(traj_gold):
    for m in json.loads(str(traj_gold["manifest"])):
        states = _run_case(m)
        assert [t for t, _ in states] == list(traj_gold[m["name"] + "_t"]), m["name"]
        assert [_sha(x) for _, x in states] == list(traj_gold[m["name"] + "_sha"]), m["name"]


def test_plans_match_reference(golden_dir):
    plans = json.load(open(os.path.join(golden_dir, "plans.json")))
    for key, p in plans.items():
        T, n, mode = key.split("_")
        blocks, rounds, evals = O.plan_blocks(int(T), int(n), mode)
        assert [list(b) for b in blocks] == p["blocks"] and rounds == p["rounds"] and evals == p["evals"]


def test_frozen_transition_values():
    # reference tests/test_transitions.py: halving schedule build_linear_beta(4, .5, .5)
    ab, _ = O.build_linear_beta(4, 0.5, 0.5)
    got = O.ddpm_skip_sample(ab, 2, 1, np.array([1.0]), np.array([1.0]), np.array([1.0]))
    assert got[0] == pytest.approx(1.5201593107716891, rel=1e-14)          # :41-44
    got = O.ddim_skip(ab, 4, 2, np.array([1.0]), np.array([0.3]), ("det",))
    assert got[0] == pytest.approx(1.6788601192042191, rel=1e-14)          # :144-148
    a_t, a_s = ab[4], ab[2]
    kappa = math.sqrt(1.0 - a_s) / math.sqrt(1.0 - a_t)
    assert kappa == pytest.approx(0.8944271909999159, rel=1e-14)           # :87-92

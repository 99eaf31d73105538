"""Perturbed-denoiser ablation, CPU side: the oracle's
restatement of _perturbation (denoiser.py:224-231) reproduces the reference's
digests and draws (tests/golden/perturb.npz, made by importing the reference)."""

import os

import numpy as np

import skipdiff_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def test_oracle_perturbation_bit_exact():
    z = np.load(os.path.join(HERE, "golden", "perturb.npz"))
    for i, t in enumerate(z["ts"]):
        x = z[f"x{i}"]
        assert O.perturb_digest(x, int(t)) == int(z["digests"][i])
        assert np.array_equal(O.perturbation(x, int(t), 0.3), z[f"pert{i}"])

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


def test_perturb_launches_cut_at_row_boundaries():
    """A row's ops after its first read the CUR register, so a launch may only
    start at a row boundary (advisor r1: S=3 scales, >= 22 tasks)."""
    import pytest
    from paper_2603_25872_b200.denoiser import perturb_launch_pieces
    for S in (1, 2, 3, 5, 7, 64):
        for rows in (1, 21, 22, 50):
            pieces = perturb_launch_pieces(rows * S, S)
            assert sum(n for _, n in pieces) == rows * S
            assert all(off % S == 0 and n <= 64 for off, n in pieces)
            assert [off for off, _ in pieces] == sorted(off for off, _ in pieces)
    with pytest.raises(ValueError):
        perturb_launch_pieces(65, 65)

"""K2 skip transitions on device vs the oracle restatement, bit-exact."""

import numpy as np
import pytest
import torch

import skipdiff_oracle as O

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


def test_frozen_values(cuda):
    from paper_2603_25872_b200 import VarianceRule, build_linear_beta, ddim_skip, ddpm_skip_posterior, ddpm_skip_sample
    s = build_linear_beta(4, 0.5, 0.5)
    one = torch.ones(1, dtype=torch.float64, device=cuda)
    got = ddpm_skip_sample(s, 2, 1, one, one, one)
    assert _np(got)[0] == pytest.approx(1.5201593107716891, rel=1e-14)
    got = ddim_skip(s, 4, 2, one, 0.3 * one, VarianceRule.deterministic())
    assert _np(got)[0] == pytest.approx(1.6788601192042191, rel=1e-14)
    post = ddpm_skip_posterior(s, 3, 3, 0.9 * one, 0.2 * one)
    assert post.variance == 0.0
    np.testing.assert_allclose(_np(post.mean), [0.2], atol=1e-15)
    out = ddpm_skip_sample(s, 3, 3, 0.9 * one, 0.2 * one, None)
    np.testing.assert_allclose(_np(out), [0.2], atol=1e-15)
    with pytest.raises(ValueError):
        ddpm_skip_sample(s, 3, 1, 0.9 * one, 0.2 * one, None)
    with pytest.raises(ValueError):
        ddim_skip(s, 3, 1, one, one, VarianceRule.ddpm_induced(), None)


@pytest.mark.parametrize("T", [30, 50, 250])
def test_random_skips_bit_exact(cuda, T):
    from paper_2603_25872_b200 import VarianceRule, ddim_skip, ddpm_skip_sample, default_schedule, predicted_x0
    s = default_schedule(T)
    ab = O.default_alpha_bar(T)
    rng = np.random.default_rng(T)
    rules = [(VarianceRule.deterministic(), ("det",)), (VarianceRule.ddpm_induced(), ("ddpm",)),
             (VarianceRule.eta_scaled(0.3), ("eta", 0.3))]
    for _ in range(40):
        t = int(rng.integers(1, T + 1))
        k = int(rng.integers(1, t + 1))
        x, e, z = rng.normal(size=(3, 4096))
        xd, ed, zd = (torch.from_numpy(a).to(cuda) for a in (x, e, z))
        for rule, orule in rules:
            got = _np(ddim_skip(s, t, k, xd, ed, rule, zd))
            ref = O.ddim_skip(ab, t, k, x, e, orule, z)
            assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (t, k, orule)
        x0 = _np(predicted_x0(s, xd, ed, t))
        assert np.array_equal(x0, O.predicted_x0(ab, x, e, t))
        got = _np(ddpm_skip_sample(s, t, k, xd, torch.from_numpy(x0).to(cuda), zd))
        ref = O.ddpm_skip_sample(ab, t, k, x, x0, z)
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (t, k)


@pytest.mark.parametrize("D,vec,offset", [(16384, 1, 0), (1 << 19, 1, 0), (1 << 19, 0, 0), (1 << 19, 1, 1),
                                          ((1 << 19) + 6, 1, 0)])
def test_fused_chain_matches_unfused(cuda, D, vec, offset):
    """One drs_skip_chain launch over a refine chain + fan-out == op-by-op numpy,
    bit for bit: the latency-bound path (16 K), and for HBM-sized latents the
    16-byte vector kernel (vec = 1), the scalar kernel (vec = 0) and the vector
    kernel on rows at an odd element offset (8-byte aligned only: scalar access
    for those ops)."""
    from paper_2603_25872_b200 import _lib, default_schedule, VarianceRule
    from paper_2603_25872_b200.transitions import ddim_op_coeffs, ddpm_op_coeffs, launch_chain, make_op, ops_to_device
    _lib.lib().drs_set_chain_vec(vec)
    try:
        _fused_chain_case(cuda, D, offset)
    finally:
        _lib.lib().drs_set_chain_vec(1)


def _fused_chain_case(cuda, D, offset):
    from paper_2603_25872_b200 import _lib, default_schedule, VarianceRule
    from paper_2603_25872_b200.transitions import ddim_op_coeffs, ddpm_op_coeffs, launch_chain, make_op, ops_to_device
    s = default_schedule(50)
    ab = O.default_alpha_bar(50)
    rng = np.random.default_rng(0)
    x = rng.normal(size=D)
    eps = rng.normal(size=(6, D))
    z = rng.normal(size=(6, D))
    xd = torch.from_numpy(x).to(cuda)
    ed = torch.from_numpy(eps).to(cuda)
    ed32 = ed.float()
    zd = torch.from_numpy(z).to(cuda)
    if offset:                   # same values in views starting one element in (8-byte aligned)
        def shifted(t):
            buf = torch.zeros(t.numel() + offset * t.shape[0] + 8, dtype=t.dtype, device=cuda)
            v = buf[offset:offset + t.numel()].view(t.shape)
            v.copy_(t)
            return v
        xd, ed, zd = shifted(xd), shifted(ed), shifted(zd)
        ed32 = shifted(ed32)
    outs = torch.zeros(8 * D + 1, dtype=torch.float64, device=cuda)[offset:offset + 8 * D].view(8, D)
    rule = VarianceRule.ddpm_induced()
    ops = []
    for i in range(4):   # refine chain 40 -> 36
        c, noisy = ddim_op_coeffs(s, 40 - i, 1, rule)
        ops.append(make_op(c, _lib.FAMILY_DDIM, noisy, src=_lib.SRC_X if i == 0 else _lib.SRC_CUR,
                           x=xd if i == 0 else None, eps=ed[i], z=zd[i], out=outs[i], save_anchor=(i == 3)))
    for i in range(1, 4):  # drafts from the new anchor, ddpm family, fp32 eps
        c, noisy = ddpm_op_coeffs(s, 36, i)
        ops.append(make_op(c, _lib.FAMILY_DDPM, noisy, src=_lib.SRC_ANCHOR, eps=ed32[4], z=zd[4 + (i > 1)],
                           out=outs[3 + i]))
    launch_chain(ops_to_device(ops, cuda), len(ops), D)
    got = _np(outs)
    cur = x
    for i in range(4):
        cur = O.ddim_skip(ab, 40 - i, 1, cur, eps[i], ("ddpm",), z[i])
        assert np.array_equal(got[i], cur)
    e32 = eps[4].astype(np.float32).astype(np.float64)
    for i in range(1, 4):
        ref = O.ddpm_skip_sample(ab, 36, i, cur, O.predicted_x0(ab, cur, e32, 36), z[4 + (i > 1)])
        assert np.array_equal(got[3 + i], ref)

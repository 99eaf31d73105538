"""Guard-band and determinism checks of the libdrs kernels -- what this pool
allows in place of compute-sanitizer (closed on the GPU pool: runs under it
left GPUs needing a reset).

* Out-of-bounds WRITES: every output is a view inside a larger buffer whose
  head and tail (and, for strided outputs, the gaps between rows) hold a NaN
  canary bit pattern; after the launch every canary word must be intact.
* Races: the same launch repeated (eagerly and from a CUDA-graph replay) must
  give bit-identical outputs -- an intra-kernel race on shared memory, TMEM or
  an mbarrier phase shows up as run-to-run differences or garbage.
Kernels: K1 noise (PCG64 + the SFC64 named-barrier pipeline), K2/K3 skip
chains (scalar and 16-byte vector paths), K4 GEMM (persistent, split-K
cluster, CTA pair, implicit conv), K6 attention, cluster GroupNorm, LayerNorm.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CANARY = 0x7FF4DEADBEEFCAFE          # a NaN payload no kernel writes


def _guarded(shape, dtype, cuda, pad=4096, row_gap=0):
    """(view, check) -- view of `shape` inside a canary-filled buffer; rows are
    separated by `row_gap` canary elements when row_gap > 0."""
    rows, cols = (shape if len(shape) == 2 else (1, shape[0]))
    ld = cols + row_gap
    n = pad + rows * ld + pad
    esz = torch.empty(0, dtype=dtype).element_size()
    words = (n * esz + 7) // 8
    raw = torch.full((words,), CANARY, dtype=torch.int64, device=cuda)
    buf = raw.view(torch.uint8)[:n * esz].view(dtype)
    view = buf[pad:pad + rows * ld].view(rows, ld)[:, :cols]
    if len(shape) == 1:
        view = view[0]
    mask = torch.ones(n, dtype=torch.bool, device=cuda)
    inner = mask[pad:pad + rows * ld].view(rows, ld)
    inner[:, :cols] = False
    pattern = raw.clone()

    def check():
        now = raw.view(torch.uint8)[:n * esz].view(dtype)
        ref = pattern.view(torch.uint8)[:n * esz].view(dtype)
        bad = (now.view(torch.uint8).view(-1, esz) != ref.view(torch.uint8).view(-1, esz)).any(1) & mask
        assert not bool(bad.any()), f"{int(bad.sum())} canary element(s) overwritten"
    return view, check


def _twice_equal(fn, out):
    """fn() twice eagerly and twice from a graph replay: bit-identical outputs."""
    fn()
    a = out.clone()
    fn()
    assert torch.equal(out.view(torch.uint8), a.view(torch.uint8)), "eager repeat differs"
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    out.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.uint8), a.view(torch.uint8)), "graph replay differs"
    return a


@pytest.mark.parametrize("gen", ["pcg64", "sfc64"])
def test_noise_guards(cuda, gen):
    from paper_2603_25872_b200.rng import _KeyBuffer, entropy_key, fill_streams
    n, ns = 5003, 7
    out, check = _guarded((ns, n), torch.float64, cuda, row_gap=13)
    keys = _KeyBuffer([entropy_key((0x7A9C, 3, t, 1)) for t in range(ns)], cuda)     # staged before capture
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    _twice_equal(lambda: fill_streams(keys, n, out, gen, err=err), out)
    assert int(err.item()) == 0
    check()
    ref = np.random.Generator(np.random.PCG64(np.random.SeedSequence((0x7A9C, 3, 2, 1))) if gen == "pcg64" else
                              np.random.SFC64(np.random.SeedSequence((0x7A9C, 3, 2, 1)))).standard_normal(n)
    assert np.array_equal(out[2].cpu().numpy(), ref)


@pytest.mark.parametrize("D,vec", [(4097, 1), (1 << 19, 1), (1 << 19, 0)])
def test_chain_guards(cuda, D, vec):
    from paper_2603_25872_b200 import _lib, default_schedule, VarianceRule
    from paper_2603_25872_b200.transitions import ddim_op_coeffs, launch_chain, make_op, ops_to_device
    _lib.lib().drs_set_chain_vec(vec)
    try:
        s, rule = default_schedule(50), VarianceRule.ddpm_induced()
        g = torch.Generator(device=cuda).manual_seed(D)
        x = torch.randn(D, dtype=torch.float64, device=cuda, generator=g)
        eps = torch.randn(4, D, dtype=torch.float64, device=cuda, generator=g)
        z = torch.randn(4, D, dtype=torch.float64, device=cuda, generator=g)
        outs, check = _guarded((4, D), torch.float64, cuda, row_gap=2)
        ops = []
        for i in range(4):
            c, noisy = ddim_op_coeffs(s, 30 - i, 1, rule)
            ops.append(make_op(c, _lib.FAMILY_DDIM, noisy, src=_lib.SRC_X if i == 0 else _lib.SRC_CUR,
                               x=x if i == 0 else None, eps=eps[i], z=z[i], out=outs[i]))
        od = ops_to_device(ops, cuda)
        _twice_equal(lambda: launch_chain(od, 4, D), outs)
        check()
    finally:
        _lib.lib().drs_set_chain_vec(1)


@pytest.mark.parametrize("M,N,K,bn,split,pair,res", [(300, 200, 136, 64, 1, False, False),
                                                      (1000, 640, 2880, 160, 1, False, True),
                                                      (512, 1280, 5120, 128, 3, False, False),
                                                      (512, 1280, 11520, 128, 2, True, False),
                                                      (2048, 640, 640, 128, 1, True, True),
                                                      (256, 1152, 4608, 64, 3, False, True)])
def test_gemm_guards(cuda, M, N, K, bn, split, pair, res):
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g)
    r = torch.randn(M, N, device=cuda, generator=g) if res else None
    out, check = _guarded((M, N), torch.float32, cuda, row_gap=8)
    _twice_equal(lambda: linear(x, w, bias=bias, residual=r, out=out, bn=bn, split=split, pair=pair), out)
    check()
    ref = x.float() @ w.float().t() + bias + (r if res else 0)
    assert (out - ref).abs().max().item() <= 2e-3 * max(1.0, ref.abs().max().item())


def test_conv_guards(cuda):
    from paper_2603_25872_b200.netops import linear
    N, H, W, C, Co = 2, 32, 32, 128, 320
    g = torch.Generator(device=cuda).manual_seed(5)
    x = (torch.randn(N * H * W, C, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(Co, 9 * C, device=cuda, generator=g) * 0.05).bfloat16()
    out, check = _guarded((N * H * W, Co), torch.bfloat16, cuda, row_gap=8)
    _twice_equal(lambda: linear(x, w, conv=(N, H, W, C), out=out), out)
    check()


@pytest.mark.parametrize("B,H,Lq,Lk,d", [(2, 8, 1024, 1024, 40), (1, 5, 300, 333, 64), (2, 4, 129, 77, 160)])
def test_attention_guards(cuda, B, H, Lq, Lk, d):
    from paper_2603_25872_b200.netops import attention_tc
    g = torch.Generator(device=cuda).manual_seed(Lq + d)
    q = torch.randn(B * Lq, H * d, device=cuda, generator=g).bfloat16()
    k = torch.randn(B * Lk, H * d, device=cuda, generator=g).bfloat16()
    vimg = (Lk + 7) // 8 * 8
    vt = torch.randn(H * d, B * vimg, device=cuda, generator=g).bfloat16()
    out, check = _guarded((B * Lq, H * d), torch.bfloat16, cuda, row_gap=16)
    _twice_equal(lambda: attention_tc(q, k, vt, out, B, H, Lq, Lk, d, vt_img=vimg), out)
    check()


@pytest.mark.parametrize("N,HW,C", [(2, 4096, 320), (2, 256, 1280), (2, 16384, 320)])
def test_groupnorm_layernorm_guards(cuda, N, HW, C):
    from paper_2603_25872_b200.netops import groupnorm, layernorm
    g = torch.Generator(device=cuda).manual_seed(HW + C)
    x = torch.randn(N * HW, C, device=cuda, generator=g).bfloat16()
    gamma, beta = torch.randn(C, device=cuda, generator=g), torch.randn(C, device=cuda, generator=g)
    out, check = _guarded((N * HW, C), torch.bfloat16, cuda)
    _twice_equal(lambda: groupnorm(x, N, HW, C, 32, gamma, beta, out, silu=True), out)
    check()
    out2, check2 = _guarded((N * HW, C), torch.bfloat16, cuda)
    _twice_equal(lambda: layernorm(x, out=out2, gamma=gamma, beta=beta), out2)
    check2()

"""K4 tcgen05 GEMM vs a plain PyTorch fp32 reference of the same op."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=[0, 1], ids=["kb1", "kb2"])
def kb2_mode(request):
    """Every GEMM test runs with one and with two k-blocks per TMA box (the KPB=2
    kernel instantiations: 3-D [K/64][rows][64] tensor maps, ring slots of 2
    stages; K % 64 == 0)."""
    from paper_2603_25872_b200 import _lib
    _lib.lib().drs_set_gemm_kb2(request.param)
    yield request.param
    _lib.lib().drs_set_gemm_kb2(_lib.GEMM_KB2_DEFAULT)


def _ref(x, w, bias, act, res, alpha):
    y = alpha * (x.float() @ w.float().t())
    if bias is not None:
        y = y + bias
    if act == "gelu_tanh":
        y = torch.nn.functional.gelu(y, approximate="tanh")
    elif act == "silu":
        y = torch.nn.functional.silu(y)
    elif act == "gelu":
        y = torch.nn.functional.gelu(y)
    elif act == "geglu":
        y = y[:, 0::2] * torch.nn.functional.gelu(y[:, 1::2])
    if res is not None:
        y = y + res.float()
    return y


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 1152, 1152), (300, 200, 136), (77, 768, 320),
                                   (1024, 3456, 1152), (4096, 320, 2880), (8, 64, 4608)])
@pytest.mark.parametrize("bn", [64, 128, 160, 192, 256])
def test_gemm_shapes(cuda, M, N, K, bn):
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N)
    x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    y = linear(x, w, out_dtype=torch.float32, bn=bn)
    ref = _ref(x, w, None, None, None, 1.0)
    err = (y - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), (M, N, K, bn, err)


@pytest.mark.parametrize("act", [None, "gelu_tanh", "silu", "gelu", "geglu"])
@pytest.mark.parametrize("split", [1, 3])
def test_gemm_epilogues(cuda, act, split):
    from paper_2603_25872_b200.netops import linear
    M, N, K = 320, 640, 576
    g = torch.Generator(device=cuda).manual_seed(3)
    x = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    b = torch.randn(N, device=cuda, generator=g) * 0.1
    n_out = N // 2 if act == "geglu" else N
    r = torch.randn(M, n_out, device=cuda, generator=g).bfloat16()
    y = linear(x, w, bias=b, act=act, residual=r, alpha=0.5, split=split)
    ref = _ref(x, w, b, act, r, 0.5)
    rel = ((y.float() - ref).norm() / ref.norm()).item()
    assert y.shape == (M, n_out) and rel <= 8e-3, (act, split, rel)


@pytest.mark.parametrize("N,H,W,C,Co", [(2, 64, 64, 320, 320), (2, 32, 32, 640, 640), (2, 16, 16, 1280, 1280),
                                        (2, 8, 8, 1280, 1280), (1, 128, 128, 64, 320), (4, 8, 8, 128, 64),
                                        (2, 32, 32, 64, 4)])
def test_implicit_conv3x3(cuda, N, H, W, C, Co):
    """Implicit-GEMM 3x3 conv (4-D TMA boxes, zero-fill padding) vs torch conv2d (fp32)."""
    import torch.nn.functional as F
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(H * C + Co)
    x = torch.randn(N, H, W, C, device=cuda, generator=g).bfloat16()             # NHWC
    w = (torch.randn(Co, 3, 3, C, device=cuda, generator=g) * 0.05).bfloat16()    # (Co, ky, kx, C)
    b = torch.randn(Co, device=cuda, generator=g) * 0.1
    y = linear(x.reshape(N * H * W, C), w.reshape(Co, 9 * C), bias=b, out_dtype=torch.float32, conv=(N, H, W, C))
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), b, padding=1)
    ref = ref.permute(0, 2, 3, 1).reshape(N * H * W, Co)
    rel = ((y - ref).norm() / ref.norm()).item()
    assert rel < 5e-3, rel


@pytest.mark.parametrize("M,N,K", [(128, 1280, 11520), (300, 200, 1152), (77, 768, 320), (256, 1152, 128)])
@pytest.mark.parametrize("bn", [64, 128, 256])
@pytest.mark.parametrize("split", [2, 3, 5, 8])
def test_gemm_cluster_splitk(cuda, M, N, K, bn, split):
    """Cluster split-K (DSMEM reduction): vs fp32 torch, bit-identical across runs
    (fixed reduction order); K=128 with split >= 3 leaves some splits empty."""
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    b = torch.randn(N, device=cuda, generator=g) * 0.1
    r = torch.randn(M, N, device=cuda, generator=g).bfloat16()
    y1 = linear(x, w, bias=b, residual=r, out_dtype=torch.float32, bn=bn, split=split)
    y2 = linear(x, w, bias=b, residual=r, out_dtype=torch.float32, bn=bn, split=split)
    ref = _ref(x, w, b, None, r, 1.0)
    err = (y1 - ref).abs().max().item()
    assert err <= 2e-3 * max(1.0, ref.abs().max().item()), (M, N, K, bn, split, err)
    assert torch.equal(y1, y2)


def test_gemm_auto_pick(cuda):
    """Library-chosen (bn, split) are valid and the default path matches torch."""
    from paper_2603_25872_b200.netops import linear, pick
    for (M, N, K) in [(128, 1280, 11520), (512, 1280, 1280), (8192, 320, 2880), (256, 1152, 4608)]:
        bn, split = pick(M, N, K)
        assert bn in (64, 128, 160, 192, 256) and 1 <= split <= 8
        assert pick(M, N, K, bn=64)[0] == 64 and pick(M, N, K, split=2)[1] == 2
        g = torch.Generator(device=cuda).manual_seed(M)
        x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
        w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
        y = linear(x, w, out_dtype=torch.float32)
        ref = _ref(x, w, None, None, None, 1.0)
        assert (y - ref).abs().max().item() <= 2e-3 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("split", [2, 4])
def test_implicit_conv3x3_splitk(cuda, split):
    from paper_2603_25872_b200.netops import linear
    N, H, W, C, Co = 2, 8, 8, 1280, 1280
    g = torch.Generator(device=cuda).manual_seed(11)
    x = torch.randn(N, H, W, C, device=cuda, generator=g).bfloat16()
    wt = (torch.randn(Co, 3, 3, C, device=cuda, generator=g) * 0.02).bfloat16()
    y = linear(x.reshape(-1, C), wt.reshape(Co, -1), out_dtype=torch.float32, conv=(N, H, W, C), split=split)
    ref = torch.nn.functional.conv2d(x.permute(0, 3, 1, 2).float(), wt.permute(0, 3, 1, 2).float(), padding=1)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Co)
    err = (y - ref).abs().max().item()
    assert err <= 2e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K,bn,conv", [(1000, 640, 576, 160, None), (300, 256, 1152, 128, None),
                                           (8192, 320, 2880, 160, (2, 64, 64, 320)), (512, 1280, 1280, 64, None),
                                           (384, 1152, 1152, 256, None), (2048, 640, 640, 192, None)])
@pytest.mark.parametrize("act", [None, "geglu"])
def test_gemm_cta_pair(cuda, M, N, K, bn, conv, act):
    """2-SM (cta_group::2) tiles -- ragged last pair included -- equal the 1-SM
    kernel bit for bit (same K order per output element), with the epilogues."""
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M + N + bn)
    x = (torch.randn(M, K if conv is None else conv[3], device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    b = torch.randn(N, device=cuda, generator=g) * 0.1
    n_out = N // 2 if act == "geglu" else N
    r = torch.randn(M, n_out, device=cuda, generator=g).bfloat16()
    y0 = linear(x, w, bias=b, act=act, residual=r, out_dtype=torch.float32, bn=bn, split=1, conv=conv, pair=False)
    y1 = linear(x, w, bias=b, act=act, residual=r, out_dtype=torch.float32, bn=bn, split=1, conv=conv, pair=True)
    assert torch.equal(y0, y1)
    ref = _ref(x if conv is None else x, w, b, act, r, 1.0) if conv is None else None
    if ref is not None:
        rel = ((y1 - ref).norm() / ref.norm()).item()
        assert rel <= 8e-3, rel


@pytest.mark.parametrize("M,N,K,bn,conv,split", [(512, 1280, 11520, 128, None, 3), (512, 1280, 1280, 64, None, 2),
                                                 (300, 256, 1152, 256, None, 4), (512, 256, 192, 128, None, 4),
                                                 (512, 1280, 11520, 128, (2, 16, 16, 1280), 3),
                                                 (512, 640, 5760, 64, None, 8), (1024, 320, 2880, 160, None, 6),
                                                 (640, 192, 640, 192, None, 2)])
def test_gemm_cta_pair_splitk(cuda, M, N, K, bn, conv, split):
    """CTA pair + cluster split-K (2 * split CTAs per tile, DSMEM reduction in
    split order) equals the 1-SM cluster split-K bit for bit; empty K ranges
    (split > k-blocks) and ragged last pairs included."""
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M + N + K + split)
    x = (torch.randn(M, K if conv is None else conv[3], device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    b = torch.randn(N, device=cuda, generator=g) * 0.1
    r = torch.randn(M, N, device=cuda, generator=g).bfloat16()
    y0 = linear(x, w, bias=b, residual=r, out_dtype=torch.float32, bn=bn, split=split, conv=conv, pair=False)
    y1 = linear(x, w, bias=b, residual=r, out_dtype=torch.float32, bn=bn, split=split, conv=conv, pair=True)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    if conv is None:
        ref = _ref(x, w, b, None, r, 1.0)
        rel = ((y1 - ref).norm() / ref.norm()).item()
        assert rel <= 8e-3, rel


@pytest.mark.parametrize("M,N,K,img,bn,split,pair", [(512, 320, 640, 256, 64, 1, False), (512, 320, 640, 256, 128, 1, True),
                                                     (1024, 768, 320, 512, 192, 1, False),
                                                     (512, 1280, 1280, 256, 128, 2, False),
                                                     (512, 1280, 1280, 256, 64, 2, True), (384, 256, 128, 128, 64, 1, True)])
def test_gemm_per_image_b(cuda, M, N, K, img, bn, split, pair):
    """b_img: rows of odd images read the second half of the B operand (the
    CFG pair's per-context weights), in every kernel variant."""
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(2 * N, K, device=cuda, generator=g) * 0.05).bfloat16()
    b = torch.randn(N, device=cuda, generator=g) * 0.1
    y = linear(x, w, bias=b, out_dtype=torch.float32, bn=bn, split=split, pair=pair, b_img=(img, N))
    odd = (torch.arange(M, device=cuda) // img) % 2 == 1
    ref = torch.where(odd[:, None], _ref(x, w[N:], b, None, None, 1.0), _ref(x, w[:N], b, None, None, 1.0))
    err = (y - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,heads,K,valid", [(8192, 8, 320, 77), (512, 8, 1280, 77), (300, 3, 64, 96), (256, 1, 128, 5)])
def test_gemm_head_softmax(cuda, M, heads, K, valid):
    """act="headsoftmax": every 96-column block is exp2-softmax-normalised over
    its first `valid` columns (zeros after), bf16 out."""
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M + heads)
    x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(heads * 96, K, device=cuda, generator=g) * 0.2).bfloat16()
    y = linear(x, w, act="headsoftmax", hs_valid=valid)
    s = (x.float() @ w.float().t()).view(M, heads, 96)
    p = torch.zeros_like(s)
    p[:, :, :valid] = torch.softmax(s[:, :, :valid] * 0.6931471805599453, dim=-1)
    err = (y.float().view(M, heads, 96) - p).abs().max().item()
    assert err <= 4e-3, err
    assert torch.all(y.view(M, heads, 96)[:, :, valid:] == 0)


@pytest.mark.parametrize("M,N,K,bn,pair", [(256, 64, 64, 64, False), (8192, 320, 320, 160, False), (300, 200, 136, 128, False),
                                           (2048, 640, 640, 128, True), (512, 1280, 1280, 64, True), (77, 768, 320, 192, False)])
@pytest.mark.parametrize("f32", [False, True])
@pytest.mark.parametrize("inplace", [False, True])
def test_gemm_tma_residual(cuda, M, N, K, bn, pair, f32, inplace):
    """Residual of the output's dtype is TMA-loaded into the epilogue's staging
    tile (also in place, out == residual as the fp32 transformer stream uses
    it); result equals the per-thread residual path bit for bit."""
    import os
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M * 3 + N + K)
    dt = torch.float32 if f32 else torch.bfloat16
    x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    b = torch.randn(N, device=cuda, generator=g) * 0.1
    r0 = torch.randn(M, N, device=cuda, generator=g).to(dt)
    r = r0.clone()
    y = linear(x, w, bias=b, residual=r, out=r if inplace else torch.empty_like(r), bn=bn, split=1, pair=pair)
    ref = _ref(x, w, b, None, r0, 1.0)
    tol = 1e-3 if f32 else 2e-2
    err = (y.float() - ref).abs().max().item()
    assert err <= tol * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K,bn,split,pair", [(8192, 320, 1280, 160, 1, False), (2048, 640, 2560, 128, 1, True),
                                                 (512, 1280, 5120, 128, 2, True), (128, 1280, 5120, 64, 4, False),
                                                 (300, 200, 136, 64, 1, False)])
def test_gemm_bf16_copy_output(cuda, M, N, K, bn, split, pair):
    """out2: the fp32 output (bias + in-place fp32 residual) and its bf16 copy
    from one epilogue, in the persistent, pair and split-K kernels."""
    from paper_2603_25872_b200.netops import linear
    g = torch.Generator(device=cuda).manual_seed(M + N + K + 1)
    x = (torch.randn(M, K, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    b = torch.randn(N, device=cuda, generator=g) * 0.1
    s = torch.randn(M, N, device=cuda, generator=g)
    ref = _ref(x, w, b, None, s.clone(), 1.0)
    cp = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    linear(x, w, bias=b, residual=s, out=s, out2=cp, bn=bn, split=split, pair=pair)
    assert (s - ref).abs().max().item() <= 1e-3 * max(1.0, ref.abs().max().item())
    assert torch.equal(cp, s.bfloat16())


@pytest.mark.parametrize("M,N,K", [(1, 1152, 1152), (1, 193536, 1152), (2, 1280, 320), (1, 20160, 1280),
                                   (3, 77, 264), (4, 2304, 4608), (2, 5, 16)])
@pytest.mark.parametrize("act,res,out_f32", [(None, None, True), ("silu", None, False), (None, "f32", True),
                                             ("silu", "bf16", False)])
def test_gemv_small_m(cuda, M, N, K, act, res, out_f32):
    """M <= 4 linears dispatch to the CUDA-core GEMV (drs_gemv) -- vs torch fp32."""
    from paper_2603_25872_b200.netops import gemv, linear
    g = torch.Generator(device=cuda).manual_seed(M * N + K)
    x = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    w = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g)
    r = None
    if res:
        r = torch.randn(M, N, device=cuda, generator=g)
        r = r if res == "f32" else r.bfloat16()
    ref = x.float() @ w.float().t() + bias
    if act == "silu":
        ref = torch.nn.functional.silu(ref)
    if r is not None:
        ref = ref + r.float()
    dt = torch.float32 if out_f32 else torch.bfloat16
    for fn in (gemv, linear):
        y = fn(x, w, bias=bias, act=act, residual=r, out_dtype=dt)
        assert y.dtype == dt
        err = (y.float() - ref).abs().max().item()
        assert err <= (1e-3 if out_f32 else 1e-2) * max(1.0, ref.abs().max().item()), (fn.__name__, err)


@pytest.mark.parametrize("N,H,W,C,Co", [(2, 32, 32, 320, 320), (2, 16, 16, 640, 640), (2, 8, 8, 1280, 1280),
                                        (1, 64, 64, 128, 192)])
@pytest.mark.parametrize("bn,split,pair", [(0, 0, None), (128, 1, False), (64, 3, False), (128, 1, True)])
def test_implicit_conv3x3_stride2(cuda, N, H, W, C, Co, bn, split, pair):
    """Stride-2 3x3 conv (the UNet downsamplers) as an implicit GEMM: the TMA box
    walks the NHWC input with element stride 2 -- vs torch conv2d(stride=2, pad=1)."""
    from paper_2603_25872_b200.netops import implicit_conv_ok, linear
    Ho, Wo = H // 2, W // 2
    if not implicit_conv_ok(N, Ho, Wo, C) or (pair and N * Ho * Wo < 256):
        pytest.skip("geometry not covered by the implicit path")
    g = torch.Generator(device=cuda).manual_seed(H * C + Co)
    x = (torch.randn(N, H, W, C, device=cuda, generator=g) * 0.5).bfloat16()
    w = (torch.randn(Co, 3, 3, C, device=cuda, generator=g) * 0.05).bfloat16()
    bias = torch.randn(Co, device=cuda, generator=g)
    y = linear(x.reshape(-1, C), w.reshape(Co, 9 * C), bias=bias, conv=(N, Ho, Wo, C, 2), out_dtype=torch.float32,
               bn=bn, split=split, pair=pair)
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), bias,
                                     stride=2, padding=1)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Co)
    err = (y - ref).abs().max().item()
    assert err <= 2e-3 * max(1.0, ref.abs().max().item()), err

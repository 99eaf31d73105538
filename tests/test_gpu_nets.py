"""Denoiser networks on the tcgen05 path vs plain PyTorch fp32 references,
and the attention / LayerNorm kernels vs torch."""

import math

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,H,Lq,Lk,d", [(1, 16, 256, 256, 72), (2, 8, 1024, 77, 40), (1, 5, 300, 300, 64),
                                         (2, 20, 64, 77, 64), (1, 8, 128, 200, 160), (1, 2, 70, 33, 80)])
def test_attention_kernel(cuda, B, H, Lq, Lk, d):
    from paper_2603_25872_b200.netops import attention
    g = torch.Generator(device=cuda).manual_seed(Lq + d)
    q = torch.randn(B * Lq, 3 * H * d, device=cuda, generator=g).bfloat16()     # strided views like qkv
    kv = torch.randn(B * Lk, 2 * H * d, device=cuda, generator=g).bfloat16()
    out = torch.empty(B * Lq, H * d, device=cuda, dtype=torch.bfloat16)
    attention(q[:, :H * d], kv[:, :H * d], kv[:, H * d:], out, B, H, Lq, Lk, d)
    Q = q[:, :H * d].float().reshape(B, Lq, H, d).transpose(1, 2)
    K = kv[:, :H * d].float().reshape(B, Lk, H, d).transpose(1, 2)
    V = kv[:, H * d:].float().reshape(B, Lk, H, d).transpose(1, 2)
    ref = (torch.softmax(Q @ K.transpose(-1, -2) / math.sqrt(d), -1) @ V).transpose(1, 2).reshape(B * Lq, H * d)
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel


def test_layernorm_modulate(cuda):
    from paper_2603_25872_b200.netops import layernorm
    x = torch.randn(512, 1152, device=cuda) * 3 + 1
    mod = torch.randn(2, 4000, device=cuda)
    shift, scale = mod[:, 12:12 + 1152], mod[:, 2000:2000 + 1152]
    y = layernorm(x, shift=shift, scale=scale, eps=1e-6, mod_group=256)
    xn = F.layer_norm(x, (1152,), eps=1e-6)
    ref = torch.cat([xn[:256] * (1 + scale[0]) + shift[0], xn[256:] * (1 + scale[1]) + shift[1]])
    assert ((y.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2
    with pytest.raises(ValueError):                      # misaligned modulation rows are rejected, not faulted
        layernorm(x, shift=mod[:, 10:10 + 1152], scale=scale, mod_group=256)
    g, b = torch.randn(1152, device=cuda), torch.randn(1152, device=cuda)
    y = layernorm(x.bfloat16(), gamma=g, beta=b, eps=1e-5)
    ref = F.layer_norm(x.bfloat16().float(), (1152,), g, b, eps=1e-5)
    assert ((y.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2


def test_dit_forward_vs_torch_fp32(cuda):
    """Batched DiT-XL/2 forward (2 images, different t) vs the fp32 torch reference.
    Tolerance: bf16 activations between GEMMs -> rel-L2 of eps <= 3e-2."""
    from paper_2603_25872_b200.dit import DiT, DiTConfig
    from nets_ref import dit_ref
    cfg = DiTConfig()
    net = DiT(cfg, cuda, seed=0, max_batch=2)
    x = torch.randn(2, 4, 32, 32, device=cuda, dtype=torch.float64)
    t = torch.tensor([999.0, 37.0], device=cuda)
    outs = [torch.empty(4096, device=cuda) for _ in range(2)]
    net.forward([x[0].reshape(-1), x[1].reshape(-1)], t, 2, outs=outs)
    got = torch.stack(outs).reshape(2, 4, 32, 32)
    ref = dit_ref(net.w, cfg, x.float(), t)
    for b in range(2):
        rel = ((got[b] - ref[b]).norm() / ref[b].norm()).item()
        assert rel < 3e-2, (b, rel)
    assert ref.abs().mean().item() > 1e-3          # random init is not the zero-eps adaLN-Zero init


def test_dit_conditioning_table(cuda):
    """The per-run conditioning table (one batched pass over a run's timesteps) gives
    the same eps as the per-eval conditioning path: single rows, a batched contiguous
    block, rows after a table re-allocation, and a captured graph replay.  The two
    paths compute the modulations with different kernels (M = 1 GEMV vs M = n GEMM,
    both fp32-accumulated), and a last-bit modulation difference moves bf16 roundings
    through 28 blocks: rel-L2 <= 5e-3 (the bf16 noise floor; vs fp32 the bound is 3e-2)."""
    from paper_2603_25872_b200.dit import DiT, DiTConfig
    cfg = DiTConfig()
    net = DiT(cfg, cuda, seed=1, max_batch=2)
    x = torch.randn(2, 4096, device=cuda, dtype=torch.float64)
    ts = torch.tensor([999.0, 500.0, 37.0, 3.0], device=cuda)
    net.alloc_conditioning(4)
    net.prepare_conditioning(ts)
    ref = [torch.empty(4096, device=cuda) for _ in range(2)]
    got = [torch.empty(4096, device=cuda) for _ in range(2)]
    for r0 in (0, 1, 2):
        t2 = ts[r0:r0 + 2].clone()
        net.forward([x[0], x[1]], t2, 2, outs=ref)
        net.forward([x[0], x[1]], t2, 2, outs=got, cond_rows=(r0, r0 + 1))
        for b in range(2):
            rel = ((got[b] - ref[b]).norm() / ref[b].norm()).item()
            assert rel < 5e-3, (r0, b, rel)
    net.forward([x[0]], ts[3:4].clone(), 1, outs=ref[:1])
    net.alloc_conditioning(8)                       # grows: earlier graphs keep the old table alive
    net.prepare_conditioning(torch.cat([ts, ts]))
    s = torch.cuda.Stream(device=cuda)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            net.prepare_conditioning(torch.cat([ts, ts]))
            net.forward([x[0]], ts[3:4], 1, outs=got[:1], cond_rows=(7,))
    torch.cuda.current_stream().wait_stream(s)
    got[0].zero_()
    g.replay()
    torch.cuda.synchronize()
    rel = ((got[0] - ref[0]).norm() / ref[0].norm()).item()
    assert rel < 5e-3, rel


@pytest.mark.parametrize("size", [32, 64])
@pytest.mark.parametrize("g", [0.0, 1.0])
def test_sd15_unet_vs_torch_fp32(cuda, size, g):
    """SD1.5-shaped UNet (CFG pair, random init) vs the fp32 torch reference.
    g = 0 checks the unconditional branch, g = 1 the conditional one (the
    production g = 7.5 multiplies the branch difference, and with it the bf16
    error of a small c - u, by 7.5).  bf16 activations through ~100 layers:
    rel-L2 of each branch <= 3e-2."""
    from paper_2603_25872_b200.unet import UNet, sd15_config
    from nets_ref import unet_ref
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    net = UNet(sd15_config(size), cuda, seed=0, max_batch=1, cfg_scale=g)
    x = torch.randn(4, size, size, device=cuda, dtype=torch.float64)
    t = torch.tensor([601.0], device=cuda)
    out = torch.empty(4 * size * size, device=cuda)
    net.forward([x.reshape(-1)], t, 1, outs=[out])
    ref = unet_ref(net, x.float()[None], t)[0]
    rel = ((out.reshape(4, size, size) - ref).norm() / ref.norm()).item()
    print(f"\n[sd15 {size} g={g} t=601] rel-L2 {rel:.3e}")
    assert torch.isfinite(out).all() and rel < 3e-2, rel
    assert net.flops > 0


# per-eval tolerance at the production guidance scale.  eps = u + 7.5 (c - u)
# carries 7.5x the error of the branch difference: measured per-branch rel-L2 1.4e-2 (bf16
# activations, test above), |c - u| / |u| = 5.2e-2 for this random-init net, so the
# uncorrelated branch errors give ~7.5 * sqrt(2) * 1.4e-2 / |u + 7.5 (c - u)| / |u| ~ 0.14;
# measured 0.118-0.124 (fold on / off alike).  SDXL's branches differ more (pooled text and
# time ids per branch), so its guided error is 2.9e-2.
G75_REL = 0.2


@pytest.mark.parametrize("fold", [True, False])
@pytest.mark.parametrize("t_model", [980.0, 500.0, 20.0])
def test_sd15_unet_g75_vs_torch_fp32(cuda, t_model, fold):
    """SD1.5 UNet at 64x64 with the production CFG scale g = 7.5, at the start,
    middle and end of a 1000-step model schedule, vs the fp32 torch reference:
    rel-L2 and max-abs of the guided eps."""
    from paper_2603_25872_b200.unet import UNet, sd15_config
    from nets_ref import unet_ref
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    net = UNet(sd15_config(64), cuda, seed=0, max_batch=1, cfg_scale=7.5)
    net.fold_cross = fold
    g = torch.Generator(device=cuda).manual_seed(int(t_model))
    x = torch.randn(4, 64, 64, device=cuda, dtype=torch.float64, generator=g)
    t = torch.tensor([t_model], device=cuda)
    out = torch.empty(4 * 64 * 64, device=cuda)
    net.forward([x.reshape(-1)], t, 1, outs=[out])
    ref = unet_ref(net, x.float()[None], t)[0].reshape(-1)
    rel = ((out - ref).norm() / ref.norm()).item()
    mab = ((out - ref).abs().max() / ref.abs().max()).item()
    net.cfg_scale = 0.0
    u = unet_ref(net, x.float()[None], t)[0].reshape(-1)
    net.cfg_scale = 1.0
    c = unet_ref(net, x.float()[None], t)[0].reshape(-1)
    net.cfg_scale = 7.5
    print(f"\n[sd15 g=7.5 t={t_model} fold={fold}] rel-L2 {rel:.3e} max-abs/max|ref| {mab:.3e} "
          f"|c-u|/|u| {((c - u).norm() / u.norm()).item():.3e}")
    assert torch.isfinite(out).all() and rel < G75_REL and mab < 2 * G75_REL, (rel, mab)


@pytest.mark.parametrize("size,g,t_model", [(64, 0.0, 700.0), (64, 1.0, 300.0), (64, 7.5, 900.0),
                                            (128, 7.5, 500.0)])
def test_sdxl_unet_vs_torch_fp32(cuda, size, g, t_model):
    """SDXL-shaped UNet (BASELINE C5: 3 levels, 2/10-deep transformers with 64-dim
    heads, 2048-d context, added pooled/time-id embedding) vs the fp32 torch
    reference: each CFG branch (g = 0 / 1) at a reduced 64x64 latent, and the
    guided eps (g = 7.5) at 64x64 and at the full 128x128 C5 latent."""
    from paper_2603_25872_b200.unet import UNet, sdxl_config
    from nets_ref import unet_ref
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    net = UNet(sdxl_config(size), cuda, seed=0, max_batch=1, cfg_scale=g)
    gen = torch.Generator(device=cuda).manual_seed(size + int(t_model))
    x = torch.randn(4, size, size, device=cuda, dtype=torch.float64, generator=gen)
    t = torch.tensor([t_model], device=cuda)
    out = torch.empty(4 * size * size, device=cuda)
    net.forward([x.reshape(-1)], t, 1, outs=[out])
    ref = unet_ref(net, x.float()[None], t)[0].reshape(-1)
    rel = ((out - ref).norm() / ref.norm()).item()
    mab = ((out - ref).abs().max() / ref.abs().max()).item()
    print(f"\n[sdxl {size} g={g} t={t_model}] rel-L2 {rel:.3e} max-abs/max|ref| {mab:.3e}")
    tol = 3e-2 if g <= 1.0 else 6e-2
    assert torch.isfinite(out).all() and rel < tol and mab < 2 * tol, (rel, mab)
    assert net.flops > 0


@pytest.mark.parametrize("B,H,Lq,Lk,d,amp", [(1, 16, 256, 256, 72, 1), (2, 8, 1024, 77, 40, 1), (1, 5, 300, 300, 64, 1),
                                             (2, 8, 4096, 4096, 40, 1), (1, 8, 128, 200, 160, 1), (1, 2, 70, 33, 80, 1),
                                             (2, 10, 1024, 1024, 64, 1), (3, 4, 70, 300, 160, 1),
                                             (3, 3, 200, 333, 96, 1), (2, 8, 64, 64, 160, 1), (2, 2, 129, 1, 64, 1),
                                             (2, 4, 256, 700, 64, 6), (2, 4, 256, 700, 160, 6)])
def test_attention_tc_kernel(cuda, B, H, Lq, Lk, d, amp):
    """tcgen05 attention (V given transposed) vs torch fp32; amp > 1 sharpens the
    softmax so the running max moves across key tiles (O rescaling)."""
    from paper_2603_25872_b200.netops import attention_tc
    g = torch.Generator(device=cuda).manual_seed(Lq + d + 1)
    q = (amp * torch.randn(B * Lq, 3 * H * d, device=cuda, generator=g)).bfloat16()
    k = torch.randn(B * Lk, 2 * H * d, device=cuda, generator=g).bfloat16()
    v = torch.randn(B * Lk, H * d, device=cuda, generator=g).bfloat16()
    vimg = (Lk + 7) // 8 * 8                          # TMA: 16-byte aligned per-image key blocks
    vt = torch.zeros(H * d, B * vimg, device=cuda, dtype=torch.bfloat16)
    for b in range(B):
        vt[:, b * vimg:b * vimg + Lk] = v[b * Lk:(b + 1) * Lk].t()
    # output rows beyond B*Lq hold a sentinel the kernel must not touch
    full = torch.full((B * Lq + 130, H * d), 7.0, device=cuda, dtype=torch.bfloat16)
    out = full[:B * Lq]
    attention_tc(q[:, :H * d], k[:, :H * d], vt, out, B, H, Lq, Lk, d, vt_img=vimg)
    Q = q[:, :H * d].float().reshape(B, Lq, H, d).transpose(1, 2)
    K = k[:, :H * d].float().reshape(B, Lk, H, d).transpose(1, 2)
    V = v.float().reshape(B, Lk, H, d).transpose(1, 2)
    ref = (torch.softmax(Q @ K.transpose(-1, -2) / math.sqrt(d), -1) @ V).transpose(1, 2).reshape(B * Lq, H * d)
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel
    assert bool((full[B * Lq:] == 7.0).all())


@pytest.mark.parametrize("N,HW,C,G,f32,silu", [(2, 4096, 320, 32, False, True), (2, 1024, 640, 32, True, False),
                                               (2, 1024, 1920, 32, False, True), (2, 256, 2560, 32, False, True),
                                               (2, 4096, 960, 32, False, False), (1, 16384, 640, 32, False, True),
                                               (2, 64, 1280, 32, False, True), (16, 4096, 320, 32, False, True),
                                               (2, 16384, 320, 32, False, False), (3, 100, 960, 32, False, True),
                                               (2, 256, 64, 32, False, True)])
@pytest.mark.parametrize("mode", [1, 2])
def test_groupnorm(cuda, N, HW, C, G, f32, silu, mode):
    """GroupNorm (+SiLU) vs torch fp32: fused cooperative path (slice kept in smem
    or re-read), the two-kernel fallback (C/G < 8), bit-identical repeats, and
    replays from a CUDA graph (grid-barrier state reused across launches)."""
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.netops import groupnorm
    _lib.lib().drs_set_gn_mode(mode)          # 1: one CTA per (image, group); 2: cluster / two-kernel paths
    g = torch.Generator(device=cuda).manual_seed(N * HW + C)
    x = (torch.randn(N * HW, C, device=cuda, generator=g) * 2 + 0.5)
    x = x if f32 else x.bfloat16()
    gamma = torch.randn(C, device=cuda, generator=g)
    beta = torch.randn(C, device=cuda, generator=g)
    out = torch.empty(N * HW, C, device=cuda, dtype=torch.bfloat16)
    groupnorm(x, N, HW, C, G, gamma, beta, out, eps=1e-5, silu=silu)
    ref = torch.nn.functional.group_norm(x.float().reshape(N, HW, C).permute(0, 2, 1), G, gamma, beta, eps=1e-5)
    if silu:
        ref = torch.nn.functional.silu(ref)
    ref = ref.permute(0, 2, 1).reshape(N * HW, C)
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err
    out2 = torch.empty_like(out)
    s = torch.cuda.Stream(cuda)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        groupnorm(x, N, HW, C, G, gamma, beta, out2, eps=1e-5, silu=silu)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(3):
                groupnorm(x, N, HW, C, G, gamma, beta, out2, eps=1e-5, silu=silu)
        out2.zero_()
        gr.replay()
        gr.replay()
    torch.cuda.synchronize()
    _lib.lib().drs_set_gn_mode(0)
    assert torch.equal(out, out2)


@pytest.mark.parametrize("M,C,f32,mod", [(8192, 320, True, False), (2048, 640, False, False), (512, 1280, True, False),
                                         (2048, 1280, True, False), (77, 1152, True, True), (4096, 1152, False, True)])
def test_layernorm_paths(cuda, M, C, f32, mod):
    """Both LayerNorm kernels (one warp per row for narrow rows at large M, one
    CTA per row otherwise) vs torch fp32, with affine and adaLN modulation."""
    from paper_2603_25872_b200.netops import layernorm
    g = torch.Generator(device=cuda).manual_seed(M + C)
    x = torch.randn(M, C, device=cuda, generator=g) * 3 + 1
    x = x if f32 else x.bfloat16()
    gamma = torch.randn(C, device=cuda, generator=g)
    beta = torch.randn(C, device=cuda, generator=g)
    kw = dict(gamma=gamma, beta=beta, eps=1e-5)
    ref = torch.nn.functional.layer_norm(x.float(), (C,), gamma, beta, 1e-5)
    if mod:
        groups = (M + 63) // 64
        shift = torch.randn(groups, C, device=cuda, generator=g)
        scale = torch.randn(groups, C, device=cuda, generator=g) * 0.1
        kw.update(shift=shift, scale=scale, mod_group=64)
        idx = torch.arange(M, device=cuda) // 64
        ref = ref * (1 + scale[idx]) + shift[idx]
    y = layernorm(x, **kw)
    err = (y.float() - ref).abs().max().item()
    assert err <= 3e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("size,B", [(32, 2), (32, 3)])
@pytest.mark.parametrize("g", [0.0, 1.0])
def test_sd15_cross_attention_fold_batched(cuda, size, B, g):
    """Folded cross-attention (score GEMM + per-head softmax epilogue, then
    P x (Wo V)) with per-context weights chosen by image parity, for a batch
    of CFG pairs: every image vs the fp32 torch reference (rel-L2 <= 3e-2, as
    the B = 1 test), and the attention-kernel path on the same net likewise."""
    from paper_2603_25872_b200.unet import UNet, sd15_config
    from nets_ref import unet_ref
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    net = UNet(sd15_config(size), cuda, seed=0, max_batch=B, cfg_scale=g)
    x = torch.randn(B, 4, size, size, device=cuda, dtype=torch.float64)
    t = torch.tensor([601.0, 233.0, 901.0][:B], device=cuda)
    ref = unet_ref(net, x.float(), t)
    for fold in (True, False):
        net.fold_cross = fold
        o = [torch.empty(4 * size * size, device=cuda) for _ in range(B)]
        net.forward([x[b].reshape(-1) for b in range(B)], t, B, outs=o)
        for b in range(B):
            rel = ((o[b].reshape(4, size, size) - ref[b]).norm() / ref[b].norm()).item()
            assert rel < 3e-2, (fold, b, rel)


@pytest.mark.parametrize("B,H,Lq,Lk,d,amp", [(2, 8, 4096, 4096, 40, 1), (1, 5, 300, 2500, 64, 6),
                                             (3, 7, 130, 2049, 40, 6), (2, 10, 4096, 4096, 64, 1),
                                             (1, 3, 1000, 1500, 32, 6), (2, 8, 1024, 1024, 80, 1),
                                             (1, 16, 256, 256, 72, 1), (2, 4, 256, 300, 160, 6)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_attention_modes(cuda, B, H, Lq, Lk, d, amp, mode):
    """Every attention variant vs torch fp32: one / two MMA issuer warps and the
    paired-FP32 softmax (default), incl. ragged key tiles and a sharp softmax
    (amp = 6: the running max moves, O rescale); repeats are bit-identical."""
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.netops import attention_qkv
    L = _lib.lib()
    L.drs_set_attn_split(mode)
    try:
        g = torch.Generator(device=cuda).manual_seed(Lq + Lk + d)
        q = (amp * torch.randn(B * Lq, H * d, device=cuda, generator=g)).bfloat16()
        kv = torch.randn(B * Lk, 2 * H * d, device=cuda, generator=g).bfloat16()
        k, v = kv[:, :H * d], kv[:, H * d:]
        full = torch.full((B * Lq + 130, H * d), 7.0, device=cuda, dtype=torch.bfloat16)
        out = full[:B * Lq]
        attention_qkv(q, k, v, out, B, H, Lq, Lk, d)
        first = out.clone()
        for _ in range(3):
            attention_qkv(q, k, v, out, B, H, Lq, Lk, d)
            assert torch.equal(out, first)
        Q = q.float().reshape(B, Lq, H, d).transpose(1, 2)
        K = k.float().reshape(B, Lk, H, d).transpose(1, 2)
        V = v.float().reshape(B, Lk, H, d).transpose(1, 2)
        ref = (torch.softmax(Q @ K.transpose(-1, -2) / math.sqrt(d), -1) @ V).transpose(1, 2).reshape(B * Lq, H * d)
        rel = ((out.float() - ref).norm() / ref.norm()).item()
        assert rel < 1e-2, rel
        assert bool((full[B * Lq:] == 7.0).all())
    finally:
        L.drs_set_attn_split(2)


@pytest.mark.parametrize("B,H,Lq,Lk,d,amp", [(2, 8, 1024, 1024, 40, 1), (1, 16, 256, 256, 72, 1),
                                             (2, 10, 256, 256, 64, 1), (1, 5, 300, 333, 64, 6),
                                             (3, 4, 70, 300, 160, 1), (2, 2, 129, 77, 96, 6),
                                             (2, 20, 64, 64, 64, 1), (2, 8, 4096, 4096, 40, 1)])
def test_attention_qkv_rowmajor_v(cuda, B, H, Lq, Lk, d, amp):
    """tcgen05 attention reading V row-major from a fused QKV buffer (MN-major PV
    operand) vs torch fp32, and equal to the V^T path up to fp32 summation order."""
    from paper_2603_25872_b200.netops import attention_qkv, attention_tc
    g = torch.Generator(device=cuda).manual_seed(Lq * 3 + d)
    qkv_q = (amp * torch.randn(B * Lq, 3 * H * d, device=cuda, generator=g)).bfloat16()
    kv = torch.randn(B * Lk, 3 * H * d, device=cuda, generator=g).bfloat16()
    q, k, v = qkv_q[:, :H * d], kv[:, H * d:2 * H * d], kv[:, 2 * H * d:]
    full = torch.full((B * Lq + 130, H * d), 7.0, device=cuda, dtype=torch.bfloat16)
    out = full[:B * Lq]
    attention_qkv(q, k, v, out, B, H, Lq, Lk, d)
    Q = q.float().reshape(B, Lq, H, d).transpose(1, 2)
    K = k.float().reshape(B, Lk, H, d).transpose(1, 2)
    V = v.float().reshape(B, Lk, H, d).transpose(1, 2)
    ref = (torch.softmax(Q @ K.transpose(-1, -2) / math.sqrt(d), -1) @ V).transpose(1, 2).reshape(B * Lq, H * d)
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel
    assert bool((full[B * Lq:] == 7.0).all())
    vimg = (Lk + 7) // 8 * 8
    vt = torch.zeros(H * d, B * vimg, device=cuda, dtype=torch.bfloat16)
    for b in range(B):
        vt[:, b * vimg:b * vimg + Lk] = v[b * Lk:(b + 1) * Lk].t()
    out_t = torch.empty_like(out)
    attention_tc(q, k, vt, out_t, B, H, Lq, Lk, d, vt_img=vimg)
    assert ((out.float() - out_t.float()).abs().max() <= 1e-2 * ref.abs().max()).item()

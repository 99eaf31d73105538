"""Plain PyTorch fp32 references of the denoiser networks (test-only): the
same random weights (bf16 matrices upcast), the same math, no custom kernels."""

import math

import torch
import torch.nn.functional as F


def dit_ref(w, cfg, x, t_model, class_label=0):
    """x: (B, C, S, S) fp32 cuda; t_model: (B,) fp32.  Returns eps (B, C, S, S) fp32."""
    B, C, S, _ = x.shape
    p, h, T = cfg.patch, cfg.hidden, cfg.tokens
    gs = S // p
    tok = x.reshape(B, C, gs, p, gs, p).permute(0, 2, 4, 1, 3, 5).reshape(B * T, C * p * p)
    hs = F.linear(tok, w.x_w.float(), w.x_b) + w.pos.repeat(B, 1)
    half = 128
    freqs = torch.exp(-math.log(10000.0) * torch.arange(half, device=x.device, dtype=torch.float32) / half)
    args = t_model[:, None].float() * freqs[None]
    temb = torch.cat([torch.cos(args), torch.sin(args)], dim=1)
    c = F.linear(F.silu(F.linear(temb, w.t_w1.float(), w.t_b1)), w.t_w2.float(), w.t_b2) + w.y_table[class_label]
    ca = F.silu(c)
    mod = F.linear(ca, w.ada_w.float(), w.ada_b).reshape(B, cfg.depth, 6, h)
    nh, hd = cfg.heads, h // cfg.heads

    def ln_mod(z, shift, scale):
        zn = F.layer_norm(z.reshape(B, T, h), (h,), eps=1e-6)
        return (zn * (1 + scale[:, None]) + shift[:, None]).reshape(B * T, h)

    for i, blk in enumerate(w.blocks):
        m = mod[:, i]
        xn = ln_mod(hs, m[:, 0], m[:, 1])
        qkv = F.linear(xn, blk["qkv_w"].float(), blk["qkv_b"]).reshape(B, T, 3, nh, hd).permute(2, 0, 3, 1, 4)
        att = torch.softmax(qkv[0] @ qkv[1].transpose(-1, -2) / math.sqrt(hd), dim=-1) @ qkv[2]
        att = att.permute(0, 2, 1, 3).reshape(B * T, h)
        proj = F.linear(att, blk["proj_w"].float(), blk["proj_b"])
        hs = hs + (proj.reshape(B, T, h) * m[:, 2][:, None]).reshape(B * T, h)
        xn = ln_mod(hs, m[:, 3], m[:, 4])
        mlp = F.linear(F.gelu(F.linear(xn, blk["fc1_w"].float(), blk["fc1_b"]), approximate="tanh"),
                       blk["fc2_w"].float(), blk["fc2_b"])
        hs = hs + (mlp.reshape(B, T, h) * m[:, 5][:, None]).reshape(B * T, h)
    fm = F.linear(ca, w.f_ada_w.float(), w.f_ada_b)
    xn = ln_mod(hs, fm[:, :h], fm[:, h:])
    out = F.linear(xn, w.f_w.float(), w.f_b).reshape(B, gs, gs, p, p, cfg.out_ch)
    img = torch.einsum("nhwpqc->nchpwq", out).reshape(B, cfg.out_ch, S, S)
    return img[:, :C]

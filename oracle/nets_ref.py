"""ORACLE -- test infrastructure only (tests/, bench.py CPU legs).

Plain PyTorch fp32 references of the denoiser networks: the same random
weights (bf16 matrices upcast), the same math, no libdrs kernels.  The
reference package has no networks (its eps is analytic, skipdiff
denoiser.py:85-145); BASELINE configs C3-C5 put these shapes behind its
`evaluate` boundary, and SURVEY 8(d) times them on host cores by injecting
such a torch-CPU network into the reference sampler."""

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


def _conv_w(w, cin, k):
    """(co, k*k*cin) with K order (ky, kx, c) -> torch (co, cin, k, k)."""
    return w.float().reshape(w.shape[0], k, k, cin).permute(0, 3, 1, 2)


def unet_ref(net, x, t_model):
    """x: (B, 4, S, S) fp32; every image as a CFG pair; returns eps (B, 4, S, S) fp32."""
    cfg, p = net.cfg, net.p
    B = x.shape[0]
    N = 2 * B
    xx = x.repeat_interleave(2, dim=0)
    xx = torch.cat([xx, torch.zeros(N, 64 - cfg.in_ch, cfg.size, cfg.size, device=x.device)], 1)
    tp = t_model.repeat_interleave(2)
    half = cfg.channels[0] // 2
    freqs = torch.exp(-math.log(10000.0) * torch.arange(half, device=x.device, dtype=torch.float32) / half)
    args = tp[:, None] * freqs[None]
    tf = torch.cat([torch.cos(args), torch.sin(args)], 1)
    th = F.silu(F.linear(tf, p["t1"][0].float(), p["t1"][1]))
    temb = F.linear(th, p["t2"][0].float(), p["t2"][1])
    if cfg.add_embed_dim:
        ah = F.silu(F.linear(net.add_in.float().repeat(B, 1), p["a1"][0].float(), p["a1"][1]))
        temb = temb + F.linear(ah, p["a2"][0].float(), p["a2"][1])
    temb_all = F.linear(F.silu(temb), net.temb_w.float(), net.temb_b)
    ctx = net.ctx.float().reshape(2, cfg.ctx_len, cfg.ctx_dim)

    def conv(h, wb, cin, stride=1):
        return F.conv2d(h, _conv_w(wb[0], cin, 3), wb[1], stride=stride, padding=1)

    def res(r, h, skip):
        if skip is not None:
            h = torch.cat([h, skip], 1)
        cin = h.shape[1]
        a = F.silu(F.group_norm(h, cfg.groups, r["gn1"][0], r["gn1"][1], eps=1e-5))
        a = conv(a, r["conv1"], cin) + temb_all[:, r["temb_off"]:r["temb_off"] + r["co"], None, None]
        a = F.silu(F.group_norm(a, cfg.groups, r["gn2"][0], r["gn2"][1], eps=1e-5))
        short = h if r["sc"] is None else F.conv2d(h, r["sc"][0].float()[:, :, None, None], r["sc"][1])
        return conv(a, r["conv2"], r["co"]) + short

    def attn(q, k, v, heads):
        Bq, Lq, c = q.shape
        d = c // heads
        q = q.reshape(Bq, Lq, heads, d).transpose(1, 2)
        k = k.reshape(Bq, -1, heads, d).transpose(1, 2)
        v = v.reshape(Bq, -1, heads, d).transpose(1, 2)
        return (torch.softmax(q @ k.transpose(-1, -2) / math.sqrt(d), -1) @ v).transpose(1, 2).reshape(Bq, Lq, c)

    def tx(tb, h):
        c = tb["c"]
        Nn, _, H, W = h.shape
        heads = cfg.n_heads(c)
        hn = F.group_norm(h, cfg.groups, tb["gn"][0], tb["gn"][1], eps=1e-6)
        s = F.linear(hn.permute(0, 2, 3, 1).reshape(Nn, H * W, c), tb["pin"][0].float(), tb["pin"][1])
        for L in tb["layers"]:
            n1 = F.layer_norm(s, (c,), L["ln1"][0], L["ln1"][1], eps=1e-5)
            qkv = F.linear(n1, L["qkv"].float())
            s = s + F.linear(attn(qkv[..., :c], qkv[..., c:2 * c], qkv[..., 2 * c:], heads), L["o1"][0].float(),
                             L["o1"][1])
            n2 = F.layer_norm(s, (c,), L["ln2"][0], L["ln2"][1], eps=1e-5)
            q = F.linear(n2, L["q2"].float())
            cx = ctx[torch.arange(Nn, device=x.device) % 2]
            k = F.linear(cx, L["wk"].float())
            v = F.linear(cx, L["wv"].float())
            s = s + F.linear(attn(q, k, v, heads), L["o2"][0].float(), L["o2"][1])
            n3 = F.layer_norm(s, (c,), L["ln3"][0], L["ln3"][1], eps=1e-5)
            y = F.linear(n3, L["ff1"][0].float(), L["ff1"][1])
            s = s + F.linear(y[..., 0::2] * F.gelu(y[..., 1::2]), L["ff2"][0].float(), L["ff2"][1])
        out = F.linear(s, tb["pout"][0].float(), tb["pout"][1]).reshape(Nn, H, W, c).permute(0, 3, 1, 2)
        return out + h

    h = conv(xx, p["conv_in"], 64)
    saved = [h]
    for kind, blk, _ in net.blocks:
        if kind == "res":
            h = res(blk, h, saved.pop() if blk["c2"] else None)
        elif kind == "tx":
            h = tx(blk, h)
        elif kind == "push":
            saved.append(h)
        elif kind == "down":
            h = conv(h, blk, h.shape[1], stride=2)
        elif kind == "up":
            h = conv(F.interpolate(h, scale_factor=2, mode="nearest"), blk, h.shape[1])
    hn = F.silu(F.group_norm(h, cfg.groups, p["gn_out"][0], p["gn_out"][1], eps=1e-5))
    y = conv(hn, p["conv_out"], h.shape[1])
    u, c = y[0::2], y[1::2]
    return u + net.cfg_scale * (c - u)

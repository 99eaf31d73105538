"""SD1.5- and SDXL-shaped conditional UNets (BASELINE configs C3, C5) on this
package's kernels, random-init (no checkpoints offline).

Layout: NHWC bf16 activations, so every 1x1 conv / linear is a GEMM over
(pixels, channels) and every 3x3 conv is im2col (drs_im2col, which also
folds in the skip-connection concat and the nearest-2x upsample) followed by
the tcgen05 GEMM (drs_gemm) with bias / time-embedding (per-image row bias) /
residual fused into the epilogue.  Classifier-free guidance runs the
(uncond, cond) pair as one batch-2 forward; eps = u + g (c - u) is formed in
the output kernel (drs_cfg_combine).  Cross-attention K/V of the fixed
random text context are computed once at construction.

Blocks (diffusers UNet2DConditionModel semantics): ResnetBlock2D
(GN+SiLU -> conv3x3 (+temb) -> GN+SiLU -> conv3x3, 1x1 shortcut),
Transformer2DModel (GN -> proj_in -> depth x [LN self-attn, LN cross-attn,
LN GEGLU FF] -> proj_out + residual), Downsample2D (conv3x3 stride 2),
Upsample2D (nearest 2x + conv3x3).
"""

import contextlib
import os
from dataclasses import dataclass, field

import torch

from . import netops as ops


@dataclass(frozen=True)
class UNetConfig:
    name: str = "sd15"
    in_ch: int = 4
    out_ch: int = 4
    size: int = 64
    channels: tuple = (320, 640, 1280, 1280)
    layers_per_block: int = 2
    tx_depth: tuple = (1, 1, 1, 0)        # transformer layers per attention, per down level
    mid_tx_depth: int = 1
    heads: int = 8                        # SD1.5: fixed 8 heads
    head_dim: int = 0                     # SDXL: fixed 64-dim heads (heads = c / 64)
    ctx_dim: int = 768
    ctx_len: int = 77
    add_embed_dim: int = 0                # SDXL: 2816 (pooled 1280 + 6 x 256 time ids)
    groups: int = 32
    temb_dim: int = 1280

    def n_heads(self, c):
        return c // self.head_dim if self.head_dim else self.heads


def sd15_config(size=64):
    return UNetConfig(size=size)


def sdxl_config(size=128):
    return UNetConfig(name="sdxl", size=size, channels=(320, 640, 1280), tx_depth=(0, 2, 10), mid_tx_depth=10,
                      heads=0, head_dim=64, ctx_dim=2048, add_embed_dim=2816)


class _Init:
    def __init__(self, device, seed, std=0.02):
        self.g = torch.Generator(device=device).manual_seed(seed)
        self.device, self.std = device, std

    def mat(self, n, k):
        return (torch.randn(n, k, generator=self.g, device=self.device) * self.std).to(torch.bfloat16)

    def vec(self, n, std=None):
        return torch.randn(n, generator=self.g, device=self.device) * (self.std if std is None else std)

    def gn(self, c):
        return (1.0 + self.vec(c, 0.1), self.vec(c, 0.1))


class UNet:
    def __init__(self, cfg: UNetConfig = UNetConfig(), device="cuda", seed: int = 0, max_batch: int = 1,
                 cfg_scale: float = 7.5):
        self.cfg = cfg
        self.device = torch.device(device)
        self.cfg_scale = cfg_scale
        self.max_batch = max_batch                   # images per forward (each is a CFG pair)
        self.latent_numel = cfg.in_ch * cfg.size * cfg.size
        self.ctx_pad = (cfg.ctx_len + 7) // 8 * 8
        # cross-attention folded into two GEMMs against the fixed context (DRS_FOLD_CROSS=0: attention kernel)
        self.fold_cross = os.environ.get("DRS_FOLD_CROSS", "1") != "0"
        # self-attention Q, K, V from ONE GEMM; the attention kernel reads V row-major
        # (DRS_QKV_FUSED=0: Q|K GEMM + swapped V^T GEMM, the round-1 layout)
        self.fused_qkv = os.environ.get("DRS_QKV_FUSED", "1") != "0"
        # stride-2 downsampling convs as implicit GEMMs (DRS_STRIDED_CONV=0: im2col + GEMM)
        self.strided_conv = os.environ.get("DRS_STRIDED_CONV", "1") != "0"
        # resblock 1x1 shortcuts on a side stream (DRS_SIDE_SHORTCUT=0: in line)
        side = os.environ.get("DRS_SIDE_SHORTCUT", "1") != "0" and self.device.type == "cuda"
        self._side = torch.cuda.Stream(self.device) if side else None
        I = _Init(self.device, seed)
        c0, T = cfg.channels[0], cfg.temb_dim
        self.p = p = {}
        p["conv_in"] = (I.mat(c0, 9 * 64), I.vec(c0))                # input padded to 64 channels
        p["t1"] = (I.mat(T, c0), I.vec(T))
        p["t2"] = (I.mat(T, T), I.vec(T))
        if cfg.add_embed_dim:
            p["a1"] = (I.mat(T, cfg.add_embed_dim), I.vec(T))
            p["a2"] = (I.mat(T, T), I.vec(T))
        # fixed random text context: [uncond, cond] x ctx_len x ctx_dim (+ SDXL pooled / time ids)
        self.ctx = torch.randn(2 * cfg.ctx_len, cfg.ctx_dim, generator=I.g, device=self.device).to(torch.bfloat16)
        if cfg.add_embed_dim:
            self.add_in = torch.randn(2, cfg.add_embed_dim, generator=I.g, device=self.device).to(torch.bfloat16)
            self.add_in_rep = self.add_in.repeat(self.max_batch, 1).contiguous()   # (uncond, cond) per image
        self.blocks = []          # ordered description of the network (built once)
        self.temb_slices = []     # (offset, c) of every resblock's time projection
        self._temb_w, self._temb_b = [], []
        skips = [c0]
        c = c0
        nlev = len(cfg.channels)
        for lev, co in enumerate(cfg.channels):
            for _ in range(cfg.layers_per_block):
                self.blocks.append(("res", self._res(I, c, 0, co), lev))
                c = co
                if cfg.tx_depth[lev]:
                    self.blocks.append(("tx", self._tx(I, c, cfg.tx_depth[lev]), lev))
                self.blocks.append(("push", None, lev))
                skips.append(c)
            if lev < nlev - 1:
                self.blocks.append(("down", (I.mat(c, 9 * c), I.vec(c)), lev))
                self.blocks.append(("push", None, lev))
                skips.append(c)
        self.blocks.append(("res", self._res(I, c, 0, c), nlev - 1))
        if cfg.mid_tx_depth:
            self.blocks.append(("tx", self._tx(I, c, cfg.mid_tx_depth), nlev - 1))
        self.blocks.append(("res", self._res(I, c, 0, c), nlev - 1))
        for i, co in enumerate(reversed(cfg.channels)):
            lev = nlev - 1 - i
            depth = cfg.tx_depth[lev]
            for _ in range(cfg.layers_per_block + 1):
                cs = skips.pop()
                self.blocks.append(("res", self._res(I, c, cs, co), lev))
                c = co
                if depth:
                    self.blocks.append(("tx", self._tx(I, c, depth), lev))
            if lev > 0:
                self.blocks.append(("up", (I.mat(c, 9 * c), I.vec(c)), lev))
        p["gn_out"] = I.gn(c)
        p["conv_out"] = (I.mat(cfg.out_ch, 9 * c), I.vec(cfg.out_ch))
        self.temb_w = torch.cat(self._temb_w, 0).contiguous()
        self.temb_b = torch.cat(self._temb_b, 0).contiguous()
        self._buf = {}
        self.flops = 0.0
        self._count = True

    # ---------------------------------------------------------------- params ---
    def _res(self, I, c1, c2, co):
        cin = c1 + c2
        off = sum(w.shape[0] for w in self._temb_w)
        self._temb_w.append(I.mat(co, self.cfg.temb_dim))
        self._temb_b.append(I.vec(co))
        return dict(c1=c1, c2=c2, co=co, gn1=I.gn(cin), conv1=(I.mat(co, 9 * cin), I.vec(co)), gn2=I.gn(co),
                    conv2=(I.mat(co, 9 * co), I.vec(co)), temb_off=off,
                    sc=(I.mat(co, cin), I.vec(co)) if cin != co else None)

    def _tx(self, I, c, depth):
        cfg = self.cfg
        layers = []
        for _ in range(depth):
            wk = I.mat(c, cfg.ctx_dim)
            wv = I.mat(c, cfg.ctx_dim)
            k_ctx = vt_ctx = None
            if self.device.type == "cuda":
                # fixed context: K (rows) and V^T (columns) of every CFG image, once.
                # image n uses context n % 2; V^T blocks are 8-aligned (TMA)
                n_img = 2 * self.max_batch
                ctx_all = self.ctx.view(2, cfg.ctx_len, cfg.ctx_dim).repeat(self.max_batch, 1, 1)
                ctx_all = ctx_all.reshape(n_img * cfg.ctx_len, cfg.ctx_dim).contiguous()
                k_ctx = ops.linear(ctx_all, wk)                                    # (n_img*77, c)
                vt = ops.linear(wv, ctx_all)                                       # (c, n_img*77)
                vt_ctx = torch.zeros(c, n_img * self.ctx_pad, dtype=torch.bfloat16, device=self.device)
                for n in range(n_img):
                    vt_ctx[:, n * self.ctx_pad:n * self.ctx_pad + cfg.ctx_len] = \
                        vt[:, n * cfg.ctx_len:(n + 1) * cfg.ctx_len]
            layers.append(dict(ln1=I.gn(c), qkv=I.mat(3 * c, c), o1=(I.mat(c, c), I.vec(c)), ln2=I.gn(c),
                               q2=I.mat(c, c), wk=wk, wv=wv, k_ctx=k_ctx, vt_ctx=vt_ctx,
                               o2=(I.mat(c, c), I.vec(c)), ln3=I.gn(c),
                               ff1=(I.mat(8 * c, c), I.vec(8 * c)), ff2=(I.mat(c, 4 * c), I.vec(c))))
            if self.device.type == "cuda":
                L = layers[-1]
                L["ws"], L["wpv"] = self._cross_fold(L["q2"], L["o2"][0], k_ctx, vt, c)
        return dict(c=c, gn=I.gn(c), pin=(I.mat(c, c), I.vec(c)), layers=layers, pout=(I.mat(c, c), I.vec(c)))

    XH = 96       # padded head width of the folded cross-attention (ctx_len <= 96)

    def _cross_fold(self, wq, wo, k_ctx, vt, c):
        """Cross-attention against the FIXED text context folded into two GEMMs:
        S_h = (n1 Wq_h^T) K_h^T * scale = n1 (K_h Wq_h * scale)^T, so the score
        block of head h is a GEMM with B_S[h*96 + j] = scale * log2(e) * K_h[j] Wq_h
        (zero rows for j >= ctx_len); and sum_h P_h V_h Wo_h^T = P B_PV^T with
        B_PV[:, h*96 + j] = Wo_h V_h[j].  One matrix per CFG context (uncond /
        cond), stacked: image n uses context n % 2 (drs_gemm b_img).  Built once
        in fp32 from the bf16 weights and context projections, rounded to bf16."""
        cfg = self.cfg
        heads = cfg.n_heads(c)
        d = c // heads
        T, XH = cfg.ctx_len, self.XH
        assert T <= XH
        f = (d ** -0.5) * 1.4426950408889634
        wqf, wof = wq.float(), wo.float()
        ws = torch.zeros(2, heads * XH, c, device=self.device)
        wpv = torch.zeros(2, c, heads * XH, device=self.device)
        for ctx in range(2):
            K = k_ctx[ctx * T:(ctx + 1) * T].float()                    # (T, c)
            V = vt[:, ctx * T:(ctx + 1) * T].float().t()                # (T, c)
            for h in range(heads):
                sl = slice(h * d, (h + 1) * d)
                ws[ctx, h * XH:h * XH + T] = f * (K[:, sl] @ wqf[sl, :])
                wpv[ctx, :, h * XH:h * XH + T] = wof[:, sl] @ V[:, sl].t()
        return (ws.reshape(2 * heads * XH, c).bfloat16().contiguous(),
                wpv.reshape(2 * c, heads * XH).bfloat16().contiguous())

    # --------------------------------------------------------------- buffers ---
    def buf(self, tag, shape, dtype=torch.bfloat16):
        key = (tag, tuple(shape), dtype)
        b = self._buf.get(key)
        if b is None:
            b = torch.empty(shape, dtype=dtype, device=self.device)
            self._buf[key] = b
        return b

    def _lin(self, x, w, **kw):
        if self._count:
            self.flops += 2.0 * x.shape[0] * w.shape[0] * w.shape[1]
        return ops.linear(x, w, **kw)

    def _attn(self, q, k, vt, out, B, H, Lq, Lk, d, vt_img):
        if self._count:
            self.flops += 4.0 * B * H * Lq * Lk * d
        return ops.attention_tc(q, k, vt, out, B, H, Lq, Lk, d, vt_img=vt_img)

    def _conv3(self, x1, c1, x2, c2, N, H, W, wb, stride=1, up=1, **kw):
        """3x3 conv, pad 1.  Stride-1 convs on one NHWC tensor run as implicit
        GEMMs (A tiles are 4-D TMA boxes of the input; no im2col); a nearest-2x
        upsample is materialised first (4x, vs 9x for im2col); the stride-2
        downsamples go through im2col."""
        if x2 is None and stride == 2 and self.strided_conv and ops.implicit_conv_ok(N, H // 2, W // 2, c1):
            # downsampler: the TMA box walks the input with element stride 2 (no im2col)
            Ho, Wo = H // 2, W // 2
            if self._count:
                self.flops += 2.0 * N * Ho * Wo * wb[0].shape[0] * wb[0].shape[1]
            return ops.linear(x1, wb[0], bias=wb[1], conv=(N, Ho, Wo, c1, 2), **kw), Ho, Wo
        if x2 is None and stride == 1 and ops.implicit_conv_ok(N, H * up, W * up, c1):
            if up == 2:
                xu = self.buf(f"ups{c1}_{H}", (N * 4 * H * W, c1))
                ops.im2col(x1, c1, None, 0, N, H, W, 1, 1, 0, 2, xu)
                x1, H, W = xu, 2 * H, 2 * W
            if self._count:
                self.flops += 2.0 * N * H * W * wb[0].shape[0] * wb[0].shape[1]
            return ops.linear(x1, wb[0], bias=wb[1], conv=(N, H, W, c1), **kw), H, W
        Ho = (H * up + 2 - 3) // stride + 1
        Wo = (W * up + 2 - 3) // stride + 1
        A = self.buf("im2col", (N * Ho * Wo, 9 * (c1 + c2)))
        ops.im2col(x1, c1, x2, c2, N, H, W, 3, stride, 1, up, A)
        return self._lin(A, wb[0], bias=wb[1], **kw), Ho, Wo

    # ---------------------------------------------------------------- blocks ---
    def _resblock(self, r, x, skip, N, H, W, temb_all, out_tag=None):
        c1, c2, co = r["c1"], r["c2"], r["co"]
        HW = H * W
        if c2:
            cat = self.buf(f"cat{c1 + c2}_{HW}", (N * HW, c1 + c2))
            ops.im2col(x, c1, skip, c2, N, H, W, 1, 1, 0, 1, cat)
            x = cat
        cin = c1 + c2
        ev = None
        if r["sc"] is not None:
            short = self.buf(f"sc{co}_{HW}", (N * HW, co))
            if self._side is not None:
                # the 1x1 shortcut only needs x: it runs on a side stream (a parallel
                # branch of the captured graph) under GN1 -> conv1 -> GN2
                main = torch.cuda.current_stream(self.device)
                self._side.wait_stream(main)
                with torch.cuda.stream(self._side):
                    self._lin(x, r["sc"][0], bias=r["sc"][1], out=short)
                    ev = torch.cuda.Event()
                    ev.record(self._side)
            else:
                self._lin(x, r["sc"][0], bias=r["sc"][1], out=short)
        else:
            short = x
        hn = self.buf(f"gn{cin}_{HW}", (N * HW, cin))
        ops.groupnorm(x, N, HW, cin, self.cfg.groups, r["gn1"][0], r["gn1"][1], hn, eps=1e-5, silu=True)
        h1 = self.buf(f"r1_{co}_{HW}", (N * HW, co))
        tb = temb_all[:, r["temb_off"]:r["temb_off"] + co]
        self._conv3(hn, cin, None, 0, N, H, W, r["conv1"], out=h1, rowbias=tb, rb_group=HW * self._tg)
        hn2 = self.buf(f"gn{co}_{HW}", (N * HW, co))
        ops.groupnorm(h1, N, HW, co, self.cfg.groups, r["gn2"][0], r["gn2"][1], hn2, eps=1e-5, silu=True)
        if ev is not None:
            torch.cuda.current_stream(self.device).wait_event(ev)
        out = self.buf(out_tag or f"res_out{co}_{HW}", (N * HW, co))
        self._conv3(hn2, co, None, 0, N, H, W, r["conv2"], out=out, residual=short)
        return out

    def _transformer(self, t, x, N, H, W, out_tag=None):
        cfg = self.cfg
        c, HW = t["c"], H * W
        M = N * HW
        heads = cfg.n_heads(c)
        d = c // heads
        hn = self.buf(f"gn{c}_{HW}", (M, c))
        ops.groupnorm(x, N, HW, c, cfg.groups, t["gn"][0], t["gn"][1], hn, eps=1e-6, silu=False)
        s = self.buf(f"txs{c}_{HW}", (M, c), torch.float32)                   # fp32 residual stream
        self._lin(hn, t["pin"][0], bias=t["pin"][1], out=s)
        n1 = self.buf(f"txn{c}_{HW}", (M, c))
        qk = self.buf(f"qkv{c}_{HW}", (M, 3 * c))           # Q | K | V (V^T in vt if not fused)
        vt = None if self.fused_qkv else self.buf(f"vt{c}_{HW}", (c, M))
        att = self.buf(f"att{c}_{HW}", (M, c))
        ffb = self.buf(f"ff{c}_{HW}", (M, 4 * c))
        sb = self.buf(f"txsb{c}_{HW}", (M, c))              # bf16 copy of the stream for proj_out
        for L in t["layers"]:
            ops.layernorm(s, out=n1, gamma=L["ln1"][0], beta=L["ln1"][1], eps=1e-5)
            if self.fused_qkv:      # one QKV GEMM; attention reads V row-major (MN-major PV operand)
                self._lin(n1, L["qkv"], out=qk)
                if self._count:
                    self.flops += 4.0 * N * heads * HW * HW * d
                ops.attention_qkv(qk[:, :c], qk[:, c:2 * c], qk[:, 2 * c:], att, N, heads, HW, HW, d)
            else:
                self._lin(n1, L["qkv"][:2 * c], out=qk[:, :2 * c])           # Q | K
                self._lin(L["qkv"][2 * c:], n1, out=vt)                       # V^T = Wv n1^T (swapped GEMM)
                self._attn(qk[:, :c], qk[:, c:2 * c], vt, att, N, heads, HW, HW, d, HW)
            self._lin(att, L["o1"][0], bias=L["o1"][1], residual=s, out=s)
            ops.layernorm(s, out=n1, gamma=L["ln2"][0], beta=L["ln2"][1], eps=1e-5)
            if "ws" in L and HW % 128 == 0 and self.fold_cross:
                # cross-attention folded into two GEMMs (see _cross_fold): scores ->
                # per-head softmax in the epilogue -> P; P B_PV^T + bias + residual
                if self._count:           # the architecture's FLOPs (q2, attention, o2), not the fold's
                    self.flops += 2.0 * M * c * c * 2 + 4.0 * N * heads * HW * cfg.ctx_len * d
                xh = heads * self.XH
                pbuf = self.buf(f"xp{c}_{HW}", (M, xh))
                ops.linear(n1, L["ws"], act="headsoftmax", hs_valid=cfg.ctx_len, b_img=(HW, xh), out=pbuf)
                ops.linear(pbuf, L["wpv"], bias=L["o2"][1], residual=s, out=s, b_img=(HW, c))
            else:
                q = qk[:, :c]
                self._lin(n1, L["q2"], out=q)
                # every image n attends to context n % 2 (uncond / cond): one launch
                self._attn(q, L["k_ctx"], L["vt_ctx"], att, N, heads, HW, cfg.ctx_len, d, self.ctx_pad)
                self._lin(att, L["o2"][0], bias=L["o2"][1], residual=s, out=s)
            ops.layernorm(s, out=n1, gamma=L["ln3"][0], beta=L["ln3"][1], eps=1e-5)
            self._lin(n1, L["ff1"][0], bias=L["ff1"][1], act="geglu", out=ffb)
            last = L is t["layers"][-1]
            # the last layer's FF output also writes the bf16 copy proj_out reads (no cast kernel)
            self._lin(ffb, L["ff2"][0], bias=L["ff2"][1], residual=s, out=s, out2=sb if last else None)
        out = self.buf(out_tag or f"tx_out{c}_{HW}", (M, c))
        self._lin(sb, t["pout"][0], bias=t["pout"][1], residual=x, out=out)
        return out

    # --------------------------------------------------------------- forward ---
    def forward(self, xs, t_dev, B: int, outs=None):
        """xs: B latents (in_ch*S*S fp64/fp32 CUDA rows); t_dev: (>= B,) fp32 model timesteps.
        Each image runs as a CFG pair (batch 2B); eps (fp32, in_ch*S*S) written to outs[b]."""
        cfg, p = self.cfg, self.p
        S, HW = cfg.size, cfg.size * cfg.size
        N = 2 * B
        assert B <= self.max_batch
        if self._count:
            self.flops = 0.0
        x_in = self.buf("x_in", (N * HW, 64))
        for b, x in enumerate(xs):
            ops.latent_to_nhwc(x, cfg.in_ch, HW, 64, x_in[(2 * b) * HW:(2 * b + 1) * HW])
            ops.latent_to_nhwc(x, cfg.in_ch, HW, 64, x_in[(2 * b + 1) * HW:(2 * b + 2) * HW])
        # the time-embedding MLP (M <= 2B rows: GEMVs) only needs t: a side-stream branch
        # of the captured graph, in parallel with the input layout + conv_in
        main = torch.cuda.current_stream(self.device)
        temb_ev = None
        if self._side is not None:
            self._side.wait_stream(main)
        with torch.cuda.stream(self._side) if self._side is not None else contextlib.nullcontext():
            if cfg.add_embed_dim:
                # SDXL: the added (pooled text + size) embedding differs between the CFG
                # images, so the time embedding is per image (N rows)
                tpair = self.buf("tpair", (N,), torch.float32)
                tpair.view(B, 2).copy_(t_dev[:B, None].expand(B, 2))
                tf = self.buf("tfreq", (N, cfg.channels[0]))
                ops.timestep_embedding(tpair, cfg.channels[0], tf)
                th = self.buf("th", (N, cfg.temb_dim))
                self._lin(tf, p["t1"][0], bias=p["t1"][1], act="silu", out=th)
                temb = self.buf("temb", (N, cfg.temb_dim), torch.float32)
                ah = self.buf("ah", (N, cfg.temb_dim))
                self._lin(self.add_in_rep[:N], p["a1"][0], bias=p["a1"][1], act="silu", out=ah)
                aemb = self.buf("aemb", (N, cfg.temb_dim), torch.float32)
                self._lin(ah, p["a2"][0], bias=p["a2"][1], out=aemb)
                self._lin(th, p["t2"][0], bias=p["t2"][1], residual=aemb, out=temb)
                temb_act = self.buf("temb_act", (N, cfg.temb_dim))
                ops.silu_cast(temb, temb_act)
                self._tg = 1                                  # temb rows per image
                n_t = N
            else:
                # SD1.5: both CFG images share the timestep, so the embedding MLP runs once
                # per pair (B rows), SiLU fused into the second linear's epilogue, and the
                # resblocks index the per-pair row (row bias group = 2 HW)
                tf = self.buf("tfreq", (B, cfg.channels[0]))
                ops.timestep_embedding(t_dev[:B], cfg.channels[0], tf)
                th = self.buf("th", (B, cfg.temb_dim))
                self._lin(tf, p["t1"][0], bias=p["t1"][1], act="silu", out=th)
                temb_act = self.buf("temb_act", (B, cfg.temb_dim))
                self._lin(th, p["t2"][0], bias=p["t2"][1], act="silu", out=temb_act)
                self._tg = 2
                n_t = B
            temb_all = self.buf("temb_all", (n_t, self.temb_w.shape[0]), torch.float32)
            self._lin(temb_act, self.temb_w, bias=self.temb_b, out=temb_all)
            if self._side is not None:
                temb_ev = torch.cuda.Event()
                temb_ev.record(self._side)

        h = self.buf("h_in", (N * HW, cfg.channels[0]))
        self._conv3(x_in, 64, None, 0, N, S, S, p["conv_in"], out=h)
        if temb_ev is not None:
            main.wait_event(temb_ev)
        H = W = S
        cur_c = cfg.channels[0]
        saved = [(h, H)]                  # h_in is written once per forward: no copy
        blocks = self.blocks
        for bi, (kind, blk, lev) in enumerate(blocks):
            # a block whose output becomes a skip connection writes it straight into
            # its own buffer (no copy out of a reused one)
            pushed = bi + 1 < len(blocks) and blocks[bi + 1][0] == "push"
            tag = f"skip{len(saved)}" if pushed else None
            if kind == "res":
                skip = None
                if blk["c2"]:
                    skip, sH = saved.pop()
                    assert sH == H, (sH, H)
                h = self._resblock(blk, h, skip, N, H, W, temb_all, out_tag=tag)
                cur_c = blk["co"]
            elif kind == "tx":
                h = self._transformer(blk, h, N, H, W, out_tag=tag)
            elif kind == "push":
                saved.append((h, H))
            elif kind == "down":
                out = self.buf(tag or f"down{cur_c}_{H}", (N * (H // 2) * (W // 2), cur_c))
                h, H, W = self._conv3(h, cur_c, None, 0, N, H, W, blk, stride=2, out=out)
            elif kind == "up":
                out = self.buf(f"up{cur_c}_{H}", (N * 4 * H * W, cur_c))
                h, H, W = self._conv3(h, cur_c, None, 0, N, H, W, blk, up=2, out=out)
        hn = self.buf(f"gn_out", (N * HW, cur_c))
        ops.groupnorm(h, N, HW, cur_c, cfg.groups, p["gn_out"][0], p["gn_out"][1], hn, eps=1e-5, silu=True)
        y = self.buf("y_out", (N * HW, cfg.out_ch), torch.float32)
        self._conv3(hn, cur_c, None, 0, N, S, S, p["conv_out"], out=y)
        if self._side is not None:              # join the side stream (graph capture needs it)
            torch.cuda.current_stream(self.device).wait_stream(self._side)
        for b in range(B):
            dst = outs[b] if outs is not None else self.buf(f"eps{b}", (self.latent_numel,), torch.float32)
            ops.cfg_combine(y[2 * b * HW:(2 * b + 2) * HW], HW, cfg.in_ch, self.cfg_scale, True, dst)
        self._count = False
        return outs


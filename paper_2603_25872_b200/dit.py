"""DiT-XL/2-shaped eps network (BASELINE config C4) on this package's kernels.

Architecture (Peebles & Xie, DiT-XL/2): 4x32x32 latent, patch 2 -> 256
tokens, hidden 1152, 28 blocks, 16 heads (d_head 72), MLP 4x with tanh-GELU,
adaLN-Zero conditioning on t and class, learned sigma (8 output channels, the
first 4 are eps), fixed 2-D sin-cos position embedding.  Weights are random
(no checkpoint is available offline): every matrix ~ N(0, 0.02) and biases
~ N(0, 0.02) -- NOT the zero adaLN init of the paper, which would make eps
identically 0 (hard part 8).

Per forward (B images, M = 256 B tokens), all on device, no host sync:
  patchify -> GEMM(+bias, +pos) -> fp32 residual stream h
  t-embedding -> GEMM(SiLU) -> GEMM(+y-embedding) -> c ; SiLU(c) -> ONE GEMM
  producing every block's 6 modulation vectors (depth*6*1152 columns)
  per block: LN+modulate -> GEMM qkv -> attention -> GEMM proj (*gate, +h)
             LN+modulate -> GEMM fc1 (tanh-GELU) -> GEMM fc2 (*gate, +h)
  final: LN+modulate -> GEMM -> unpatchify -> eps (first 4 channels, fp32)
The 28 x 4 GEMMs run on the tcgen05 kernel (drs_gemm); the adaLN
gate multiply and the residual add are fused into their epilogues.
"""

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import netops as ops


@dataclass(frozen=True)
class DiTConfig:
    input_size: int = 32
    patch: int = 2
    in_ch: int = 4
    hidden: int = 1152
    depth: int = 28
    heads: int = 16
    mlp_ratio: float = 4.0
    num_classes: int = 1000
    learn_sigma: bool = True

    @property
    def tokens(self):
        return (self.input_size // self.patch) ** 2

    @property
    def out_ch(self):
        return self.in_ch * 2 if self.learn_sigma else self.in_ch

    def flops_per_image(self) -> float:
        """2*MAC of every GEMM + attention (norms/elementwise excluded)."""
        T, h, m = self.tokens, self.hidden, int(self.hidden * self.mlp_ratio)
        per_block = 2 * T * h * (3 * h) + 2 * T * h * h + 2 * T * h * m * 2 + 2 * 2 * T * T * h
        embed = 2 * T * (self.in_ch * self.patch ** 2) * h + 2 * T * h * self.patch ** 2 * self.out_ch
        cond = 2 * (256 * h + h * h + h * 6 * h * self.depth + h * 2 * h)
        return float(self.depth * per_block + embed + cond)


def _sincos_pos_embed(dim, grid):
    """Fixed 2-D sin-cos position embedding (DiT get_2d_sincos_pos_embed)."""
    def emb_1d(d, pos):
        omega = 1.0 / 10000 ** (np.arange(d // 2, dtype=np.float64) / (d / 2.0))
        out = np.einsum("m,d->md", pos.reshape(-1), omega)
        return np.concatenate([np.sin(out), np.cos(out)], axis=1)
    gh, gw = np.meshgrid(np.arange(grid, dtype=np.float32), np.arange(grid, dtype=np.float32))
    g = np.stack([gw, gh], axis=0)
    return np.concatenate([emb_1d(dim // 2, g[0]), emb_1d(dim // 2, g[1])], axis=1)


class DiTWeights:
    """Random-init parameters (bf16 matrices, fp32 vectors) on one device."""

    def __init__(self, cfg: DiTConfig, device, seed: int = 0, std: float = 0.02):
        g = torch.Generator(device="cpu").manual_seed(seed)
        h, m, L = cfg.hidden, int(cfg.hidden * cfg.mlp_ratio), cfg.depth

        def mat(n, k):
            return (torch.randn(n, k, generator=g) * std).to(torch.bfloat16).to(device)

        def vec(n):
            return (torch.randn(n, generator=g) * std).to(device)

        p2c = cfg.patch * cfg.patch * cfg.in_ch
        self.x_w, self.x_b = mat(h, p2c), vec(h)
        self.t_w1, self.t_b1 = mat(h, 256), vec(h)
        self.t_w2, self.t_b2 = mat(h, h), vec(h)
        self.y_table = (torch.randn(cfg.num_classes + 1, h, generator=g) * std).to(device)
        self.ada_w, self.ada_b = mat(L * 6 * h, h), vec(L * 6 * h)        # every block's adaLN, one GEMM
        self.blocks = []
        for _ in range(L):
            self.blocks.append(dict(qkv_w=mat(3 * h, h), qkv_b=vec(3 * h), proj_w=mat(h, h), proj_b=vec(h),
                                    fc1_w=mat(m, h), fc1_b=vec(m), fc2_w=mat(h, m), fc2_b=vec(h)))
        for blk in self.blocks:   # V bias folded through the attention into the projection bias
            blk["proj_b_eff"] = blk["proj_b"] + blk["proj_w"].float() @ blk["qkv_b"][2 * h:]
        self.f_ada_w, self.f_ada_b = mat(2 * h, h), vec(2 * h)
        self.f_w = mat(cfg.patch * cfg.patch * cfg.out_ch, h)
        self.f_b = vec(cfg.patch * cfg.patch * cfg.out_ch)
        pos = _sincos_pos_embed(h, cfg.input_size // cfg.patch)
        self.pos = torch.from_numpy(pos).float().to(device)                 # (T, h) fp32


class DiT:
    """Forward pass with preallocated buffers for up to `max_batch` images (CUDA-graph capturable)."""

    def __init__(self, cfg: DiTConfig = DiTConfig(), device="cuda", seed: int = 0, max_batch: int = 8,
                 class_label: int = 0, weights: DiTWeights | None = None):
        self.cfg = cfg
        self.device = torch.device(device)
        self.w = weights or DiTWeights(cfg, self.device, seed)
        self.max_batch = max_batch
        self.class_label = class_label
        T, h, m, L = cfg.tokens, cfg.hidden, int(cfg.hidden * cfg.mlp_ratio), cfg.depth
        MB = max_batch * T
        bf, f32 = torch.bfloat16, torch.float32
        dev = self.device
        self.tok_in = torch.empty(MB, cfg.patch * cfg.patch * cfg.in_ch, dtype=bf, device=dev)
        self.pos_b = self.w.pos.repeat(max_batch, 1).contiguous()        # (MB, h) fp32 residual for x-embed
        self.hs = torch.empty(MB, h, dtype=f32, device=dev)               # residual stream
        self.xn = torch.empty(MB, h, dtype=bf, device=dev)
        # one fused QKV GEMM; the attention reads V row-major as an MN-major operand
        # (DRS_QKV_FUSED=0: Q|K GEMM + swapped V^T GEMM, the round-1 layout)
        self.fused_qkv = os.environ.get("DRS_QKV_FUSED", "1") != "0"
        self.overlap_mod = os.environ.get("DRS_DIT_OVERLAP", "0") == "1" and self.device.type == "cuda"
        self._side = torch.cuda.Stream(self.device) if self.overlap_mod else None
        self.qkv = torch.empty(MB, 3 * h, dtype=bf, device=dev)            # Q | K | V
        self.vt = torch.empty(h, MB, dtype=bf, device=dev)                 # V^T (unfused layout only)
        self.att = torch.empty(MB, h, dtype=bf, device=dev)
        self.mlp = torch.empty(MB, m, dtype=bf, device=dev)
        self.tout = torch.empty(MB, cfg.patch * cfg.patch * cfg.out_ch, dtype=f32, device=dev)
        self.t_in = torch.zeros(max_batch, dtype=f32, device=dev)
        self.t_freq = torch.empty(max_batch, 256, dtype=bf, device=dev)
        self.t_h = torch.empty(max_batch, h, dtype=bf, device=dev)
        self.y_emb = self.w.y_table[class_label].repeat(max_batch, 1).contiguous()
        self.c = torch.empty(max_batch, h, dtype=f32, device=dev)
        self.c_act = torch.empty(max_batch, h, dtype=bf, device=dev)
        self.mod = torch.empty(max_batch, L * 6 * h, dtype=f32, device=dev)
        self.fmod = torch.empty(max_batch, 2 * h, dtype=f32, device=dev)
        self.eps_img = torch.empty(max_batch, cfg.in_ch, cfg.input_size, cfg.input_size, dtype=f32, device=dev)
        self.cond_n = 0                      # rows of the per-run conditioning table (alloc_conditioning)

    # ---- per-run conditioning table --------------------------------------------
    # The adaLN modulations depend on the timestep (and this instance's class label)
    # only, not on the latent.  A sampler run knows every timestep it will evaluate,
    # so the run computes them all at its start in ONE batched pass (the 446 MB of
    # adaLN weights streamed once per run as an M = n GEMM, instead of one M = 1
    # GEMV per eval), and each eval reads its rows.  Inside the run's timed graph.
    COND_TABLE = os.environ.get("DRS_COND_TABLE", "1") != "0"

    def alloc_conditioning(self, n: int):
        """Buffers for a table of n timesteps (call before CUDA-graph capture)."""
        cfg, h, L, dev = self.cfg, self.cfg.hidden, self.cfg.depth, self.device
        if n <= self.cond_n:
            return
        if self.cond_n:        # graphs captured against the old buffers keep them alive
            self._old_cond = getattr(self, "_old_cond", []) + [(self.cond_freq, self.cond_h, self.cond_y, self.cond_c,
                                                                   self.cond_act, self.mod_table, self.fmod_table)]
        bf, f32 = torch.bfloat16, torch.float32
        self.cond_freq = torch.empty(n, 256, dtype=bf, device=dev)
        self.cond_h = torch.empty(n, h, dtype=bf, device=dev)
        self.cond_y = self.w.y_table[self.class_label].repeat(n, 1).contiguous()
        self.cond_c = torch.empty(n, h, dtype=f32, device=dev)
        self.cond_act = torch.empty(n, h, dtype=bf, device=dev)
        self.mod_table = torch.empty(n, L * 6 * h, dtype=f32, device=dev)
        self.fmod_table = torch.empty(n, 2 * h, dtype=f32, device=dev)
        self.cond_n = n

    def prepare_conditioning(self, t_dev):
        """Modulation rows for the n model timesteps in t_dev (device fp32, n <= cond_n)."""
        n, w = t_dev.shape[0], self.w
        ops.timestep_embedding(t_dev, 256, self.cond_freq[:n])
        ops.linear(self.cond_freq[:n], w.t_w1, bias=w.t_b1, act="silu", out=self.cond_h[:n])
        ops.linear(self.cond_h[:n], w.t_w2, bias=w.t_b2, residual=self.cond_y[:n], out=self.cond_c[:n])
        ops.silu_cast(self.cond_c[:n], self.cond_act[:n])
        ops.linear(self.cond_act[:n], w.ada_w, bias=w.ada_b, out=self.mod_table[:n])
        ops.linear(self.cond_act[:n], w.f_ada_w, bias=w.f_ada_b, out=self.fmod_table[:n])

    # DRS_DIT_OVERLAP=1 (measured slower, off by default): the adaLN modulation GEMVs
    # (M = B rows, 6 h columns per block, 446 MB of weights for 28 blocks) in chunks on a
    # side stream, each block waiting only for its own chunk.  On a B200 the side stream's
    # weight stream slows the blocks' latency-bound GEMMs more than it hides
    # (DiT b1 1.565 -> 1.63 ms with one GEMV CTA per SM; no change with four), so the
    # default keeps one in-line GEMV at the head of the eval.
    MOD_CHUNKS = ((0, 1), (1, 2), (2, 4), (4, 8), (8, 28))

    def _modulations(self, B):
        w, h, L = self.w, self.cfg.hidden, self.cfg.depth
        if not self.overlap_mod:
            ops.linear(self.c_act[:B], w.ada_w, bias=w.ada_b, out=self.mod[:B])
            ops.linear(self.c_act[:B], w.f_ada_w, bias=w.f_ada_b, out=self.fmod[:B])
            return {}
        main = torch.cuda.current_stream(self.device)
        self._side.wait_stream(main)                 # c_act is ready
        ready = {}
        with torch.cuda.stream(self._side):
            for l0, l1 in self.MOD_CHUNKS:
                if l0 >= L:
                    break
                l1 = min(l1, L)
                a, b = l0 * 6 * h, l1 * 6 * h
                ops.linear(self.c_act[:B], w.ada_w[a:b], bias=w.ada_b[a:b], out=self.mod[:B, a:b], gemv_ctas=1)
                ev = torch.cuda.Event()
                ev.record(self._side)
                ready[l0] = ev
            ops.linear(self.c_act[:B], w.f_ada_w, bias=w.f_ada_b, out=self.fmod[:B], gemv_ctas=1)
            ev = torch.cuda.Event()
            ev.record(self._side)
            ready["final"] = ev
        return ready

    def forward(self, xs, t_dev, B: int, outs=None, cond_rows=None):
        """xs: list of B latents (in_ch*S*S, fp64/fp32 CUDA tensors); t_dev: (>=B,) fp32 device
        timesteps (model units).  eps (first in_ch channels, fp32) is written to outs[b] if
        given, else returned as a view (B, in_ch, S, S) of an internal buffer.  cond_rows: B
        row indices into the conditioning table (prepare_conditioning) for these timesteps --
        the conditioning MLP and adaLN projections are then not recomputed."""
        cfg, w = self.cfg, self.w
        T, h, L, S, p = cfg.tokens, cfg.hidden, cfg.depth, cfg.input_size, cfg.patch
        M = B * T
        assert B <= self.max_batch
        for b, x in enumerate(xs):
            ops.patchify(x, cfg.in_ch, S, S, p, self.tok_in[b * T:(b + 1) * T])
        ops.linear(self.tok_in[:M], w.x_w, bias=w.x_b, residual=self.pos_b[:M], out=self.hs[:M])
        ready = {}
        mod, fmod = self.mod, self.fmod
        r0 = cond_rows[0] if cond_rows is not None else -1
        if cond_rows is not None and list(cond_rows) == list(range(r0, r0 + B)) and r0 + B <= self.cond_n:
            # a contiguous block of this run's conditioning table, read in place
            mod, fmod = self.mod_table[r0:r0 + B], self.fmod_table[r0:r0 + B]
        else:
            # conditioning: c = MLP(freq(t)) + y_emb ; SiLU(c) drives every adaLN
            ops.timestep_embedding(t_dev[:B], 256, self.t_freq[:B])
            ops.linear(self.t_freq[:B], w.t_w1, bias=w.t_b1, act="silu", out=self.t_h[:B])
            ops.linear(self.t_h[:B], w.t_w2, bias=w.t_b2, residual=self.y_emb[:B], out=self.c[:B])
            ops.silu_cast(self.c[:B], self.c_act[:B])
            ready = self._modulations(B)
        hs, xn, qkv, att, mlp = self.hs[:M], self.xn[:M], self.qkv[:M], self.att[:M], self.mlp[:M]
        main = torch.cuda.current_stream(self.device)
        for i, blk in enumerate(w.blocks):
            if i in ready:
                main.wait_event(ready[i])
            base = i * 6 * h
            md = mod[:B]
            sh_a, sc_a, g_a = md[:, base:base + h], md[:, base + h:base + 2 * h], md[:, base + 2 * h:base + 3 * h]
            sh_m, sc_m, g_m = (md[:, base + 3 * h:base + 4 * h], md[:, base + 4 * h:base + 5 * h],
                               md[:, base + 5 * h:base + 6 * h])
            ops.layernorm(hs, out=xn, shift=sh_a, scale=sc_a, eps=1e-6, mod_group=T)
            if self.fused_qkv:
                ops.linear(xn, blk["qkv_w"], bias=blk["qkv_b"], out=qkv)
                ops.attention_qkv(qkv[:, 0:h], qkv[:, h:2 * h], qkv[:, 2 * h:3 * h], att, B, cfg.heads, T, T,
                                  h // cfg.heads)
                proj_b = blk["proj_b"]
            else:
                ops.linear(xn, blk["qkv_w"][:2 * h], bias=blk["qkv_b"][:2 * h], out=qkv[:, :2 * h])
                # V^T = W_v xn^T for the V^T attention path.  The V bias is folded into the
                # projection bias (softmax rows sum to 1: P (V + 1 b_v^T) = P V + b_v)
                ops.linear(blk["qkv_w"][2 * h:], xn, out=self.vt[:, :M])
                ops.attention_tc(qkv[:, 0:h], qkv[:, h:2 * h], self.vt[:, :M], att, B, cfg.heads, T, T,
                                 h // cfg.heads, vt_img=T)
                proj_b = blk["proj_b_eff"]
            ops.linear(att, blk["proj_w"], bias=proj_b, colscale=g_a, cs_group=T, residual=hs, out=hs)
            ops.layernorm(hs, out=xn, shift=sh_m, scale=sc_m, eps=1e-6, mod_group=T)
            ops.linear(xn, blk["fc1_w"], bias=blk["fc1_b"], act="gelu_tanh", out=mlp)
            ops.linear(mlp, blk["fc2_w"], bias=blk["fc2_b"], colscale=g_m, cs_group=T, residual=hs, out=hs)
        if "final" in ready:
            main.wait_event(ready["final"])
            main.wait_stream(self._side)            # join the side stream (graph capture needs it)
        fm = fmod[:B]
        ops.layernorm(hs, out=xn, shift=fm[:, 0:h], scale=fm[:, h:2 * h], eps=1e-6, mod_group=T)
        ops.linear(xn, w.f_w, bias=w.f_b, out=self.tout[:M])
        for b in range(B):
            dst = outs[b] if outs is not None else self.eps_img[b]
            ops.unpatchify(self.tout[b * T:(b + 1) * T], cfg.out_ch, cfg.in_ch, S, S, p, dst)
        return self.eps_img[:B] if outs is None else outs

"""Python wrappers of the network kernels in libdrs.so (include/drs_net.h).

Tensors are torch CUDA tensors; every op launches on the current stream and
raises if libdrs.so is missing (no fallback).  Weights are bf16, K-major
(nn.Linear layout: W[out, in]); activations bf16; accumulation fp32.
"""

import json
import os

import torch

from . import _lib

ACT = {None: 0, "none": 0, "gelu_tanh": 1, "silu": 2, "gelu": 3, "geglu": 4, "headsoftmax": 5}


# Instrumentation (bench.py): when TIMERS is a list, every GEMM records
# (flops, start event, end event) on the current stream.
TIMERS = None


def _ptr(t):
    return t.data_ptr() if t is not None else None


def linear(x, w, bias=None, act=None, residual=None, out=None, out_dtype=torch.bfloat16, alpha=1.0,
           bn=0, split=0, colscale=None, cs_group=0, rowbias=None, rb_group=0, conv=None, pair=None,
           b_img=None, hs_valid=0, out2=None, gemv_ctas=0, kbox=0):
    """out[M, N'] = act(alpha * x[M, K] @ w[N, K]^T + bias + rowbias) * colscale (+ residual);
    N' = N/2 for geglu.  residual may be bf16 or fp32 (same shape as out); colscale /
    rowbias (n_groups, >=N) views indexed by row // group.  b_img = (rows, off): rows
    of images with odd index (row // rows) use w[off + n] instead of w[n] (w holds
    N + off rows; CFG pairs with per-context weights).  act="headsoftmax": per
    96-column head, softmax (exp2) over the first hs_valid columns.  out2: a bf16
    tensor that also receives the (fp32) output, rounded.  kbox: k-blocks per TMA box
    (0: the tuned table / library default, 1, 2)."""
    assert x.dtype == torch.bfloat16 and w.dtype == torch.bfloat16
    if (conv is None and x.shape[0] <= 4 and act in (None, "none", "silu") and colscale is None and rowbias is None
            and b_img is None and out2 is None and GEMV and _gemv_ok(x, w)):
        return gemv(x, w, bias=bias, act=act, residual=residual, out=out, out_dtype=out_dtype, ctas_per_sm=gemv_ctas)
    if conv is not None:          # implicit 3x3 conv: x is NHWC, K = 9*C; conv = (N, H, W, C[, stride])
        cn, ch, cw, cc = conv[:4]   # H, W: the output grid (input 2H x 2W for stride 2)
        M, K = cn * ch * cw, 9 * cc
    else:
        M, K = x.shape
    N = w.shape[0] if b_img is None else w.shape[0] - b_img[1]
    assert w.shape[1] == K and x.stride(-1) == 1 and w.stride(1) == 1
    n_out = N // 2 if act == "geglu" else N
    if out is None:
        out = torch.empty(M, n_out, dtype=out_dtype, device=x.device)
    g = _lib.DrsGemmArgs()
    g.A, g.lda, g.B, g.ldb, g.C, g.ldc = x.data_ptr(), x.stride(0), w.data_ptr(), w.stride(0), out.data_ptr(), out.stride(0)
    if conv is not None:
        g.lda = K
    g.M, g.N, g.K = M, N, K
    g.act, g.out_f32, g.alpha = ACT[act], 1 if out.dtype == torch.float32 else 0, float(alpha)
    if bias is not None:
        assert bias.dtype == torch.float32
        g.bias = bias.data_ptr()
    if residual is not None:
        assert residual.stride(1) == 1 and residual.dtype in (torch.bfloat16, torch.float32)
        g.residual, g.ldr, g.res_f32 = residual.data_ptr(), residual.stride(0), int(residual.dtype == torch.float32)
    if colscale is not None:
        assert colscale.dtype == torch.float32
        g.colscale, g.cs_group = colscale.data_ptr(), cs_group
        g.cs_ld = colscale.stride(0) if colscale.dim() == 2 else 0
    if rowbias is not None:
        assert rowbias.dtype == torch.float32 and rb_group > 0
        g.rowbias, g.rb_group, g.rb_ld = rowbias.data_ptr(), rb_group, rowbias.stride(0)
    if SHAPES is not None:
        SHAPES.append((M, N, K, act, residual is not None and residual.dtype == torch.float32,
                       residual is not None, out.dtype == torch.float32, None if conv is None else tuple(conv)))
    if bn == 0 or split == 0:                    # tuned table, else the library cost model
        cv = False if conv is None else (conv[4] if len(conv) > 4 else 1)
        bn, split, tpair = pick3(M, N, K, bn, split, cv)
        if pair is None:
            pair = tpair
        if kbox == 0:
            kbox = table_kbox(M, N, K, cv)
    g.bn, g.split = bn, split
    g.kbox = kbox
    g.cta_pair = 1 if pair else 0
    if conv is not None:
        g.conv_N, g.conv_H, g.conv_W, g.conv_C = conv[:4]
        g.conv_stride = conv[4] if len(conv) > 4 else 1
    if b_img is not None:
        g.b_img_rows, g.b_img_off = b_img
    g.hs_valid = hs_valid
    if out2 is not None:
        assert out2.dtype == torch.bfloat16 and out2.stride(1) == 1 and out.dtype == torch.float32
        g.out2, g.ldo2 = out2.data_ptr(), out2.stride(0)
    if GEMM_RECORD is not None:
        GEMM_RECORD.append((2.0 * M * N * K, _lib.DrsGemmArgs.from_buffer_copy(g)))
    if TIMERS is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    _lib.check(_lib.lib().drs_gemm(_lib.ctypes.byref(g), _lib.stream_ptr()), "drs_gemm")
    if TIMERS is not None:
        e1.record()
        TIMERS.append((2.0 * M * N * K, e0, e1, (M, N, K, bn, split)))
    return out


# M <= 4 linears (the conditioning MLPs) run on the CUDA-core GEMV (drs_gemv): a
# pure weight stream, small enough to co-reside with the tensor-core GEMMs
GEMV = os.environ.get("DRS_GEMV", "1") != "0"


def _gemv_ok(x, w):
    K = x.shape[1]
    return (K % 8 == 0 and x.stride(1) == 1 and w.stride(1) == 1 and x.stride(0) % 8 == 0 and w.stride(0) % 8 == 0
            and x.data_ptr() % 16 == 0 and w.data_ptr() % 16 == 0 and x.shape[0] * K * 2 <= 72 * 1024)


def gemv(x, w, bias=None, act=None, residual=None, out=None, out_dtype=torch.bfloat16, ctas_per_sm=0):
    """out[m, n] = act(x[m] . w[n] + bias[n]) (+ residual[m, n]) for M <= 4 rows (drs_gemv).
    ctas_per_sm=1 keeps the grid small enough for tensor-core GEMM CTAs to co-reside
    (side-stream use); 0 = 4 CTAs per SM (in-line use)."""
    M, K = x.shape
    N = w.shape[0]
    if out is None:
        out = torch.empty(M, N, dtype=out_dtype, device=x.device)
    st = _lib.lib().drs_gemv(x.data_ptr(), x.stride(0), w.data_ptr(), w.stride(0), _ptr(bias), _ptr(residual),
                             residual.stride(0) if residual is not None else 0,
                             int(residual is not None and residual.dtype == torch.float32), out.data_ptr(),
                             out.stride(0), int(out.dtype == torch.float32), M, N, K, ACT[act], int(ctas_per_sm),
                             _lib.stream_ptr())
    _lib.check(st, "drs_gemv")
    return out


BN_CHOICES = (64, 128, 160, 192, 256)


_TABLE_PATH = os.environ.get("DRS_GEMM_TABLE") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                                "gemm_table.json")
_TABLE = None
SHAPES = None      # when a list: linear() appends (M, N, K, act, res_f32, has_res, out_f32, conv) (tuning)
GEMM_RECORD = None  # when a list: linear() appends (flops, drs_gemm_args copy) -- bench.py replays them
                    # back to back in one CUDA graph to time the tensor-core kernels alone


def _table():
    global _TABLE
    if _TABLE is None:
        try:
            with open(_TABLE_PATH) as f:
                _TABLE = {k: tuple(v) for k, v in json.load(f)["configs"].items()}
        except (OSError, ValueError, KeyError):
            _TABLE = {}
    return _TABLE


def table_key(M, N, K, conv=False):
    """conv: False, True / 1 (stride-1 implicit conv) or 2 (stride-2)."""
    return f"{M}x{N}x{K}" + ((":conv2" if conv == 2 else ":conv") if conv else "")


def pick3(M, N, K, bn=0, split=0, conv=False):
    """(bn, split, cta_pair) for this GEMM: explicit bn/split win; otherwise the
    measured B200 table (tools/gemm_tune.py -> gemm_table.json) for shapes the
    networks issue, else the library's cost model (drs_gemm_pick, no pair)."""
    if bn == 0 and split == 0:
        hit = _table().get(table_key(M, N, K, conv))
        if hit is not None:
            return (hit[0], hit[1], bool(hit[2]) if len(hit) > 2 else False)
    b, sp = pick(M, N, K, bn, split, conv)
    return b, sp, False


def table_kbox(M, N, K, conv=False):
    """k-blocks per TMA box the tuned table holds for this shape (0: library default)."""
    hit = _table().get(table_key(M, N, K, conv))
    return int(hit[3]) if hit is not None and len(hit) > 3 else 0


def pick(M, N, K, bn=0, split=0, conv=False):
    """(bn, split) for this GEMM (see pick3)."""
    if bn == 0 and split == 0:
        hit = _table().get(table_key(M, N, K, conv))
        if hit is not None:
            return tuple(hit[:2])
    b, sp = _lib.ctypes.c_int(bn), _lib.ctypes.c_int(split)
    _lib.check(_lib.lib().drs_gemm_pick(M, N, K, _lib.ctypes.byref(b), _lib.ctypes.byref(sp)), "drs_gemm_pick")
    return b.value, sp.value


def implicit_conv_ok(N, H, W, C):
    """Geometry the implicit-GEMM conv supports (mirrors drs_gemm's checks):
    128-pixel tiles of whole image rows (or whole images) of an NHWC input."""
    if C % 64 or W > 128 or W & (W - 1):
        return False
    rows = 1 if W >= 128 else min(128 // W, H)
    imgs = 128 // (W * rows)
    if W * rows * imgs != 128 or H % rows:
        return False
    return imgs == 1 or (rows == H and N % imgs == 0)


def layernorm(x, out=None, gamma=None, beta=None, shift=None, scale=None, eps=1e-6, mod_group=0):
    """shift/scale: (C,) or (n_groups, >=C) views with row stride; mod_group rows per group."""
    M, C = x.shape
    if out is None:
        out = torch.empty(M, C, dtype=torch.bfloat16, device=x.device)
    mod = shift if shift is not None else scale
    mod_ld = mod.stride(0) if (mod is not None and mod.dim() == 2) else 0
    st = _lib.lib().drs_layernorm(x.data_ptr(), x.stride(0), 1 if x.dtype == torch.float32 else 0, M, C,
                                  _ptr(gamma), _ptr(beta), _ptr(shift), _ptr(scale), mod_group, mod_ld, float(eps),
                                  out.data_ptr(), out.stride(0), _lib.stream_ptr())
    _lib.check(st, "drs_layernorm")
    return out


def attention(q, k, v, out, B, H, Lq, Lk, d, scale=None):
    """q: (B*Lq, >= H*d) view, k/v: (B*Lk, ...) views (row strides may exceed H*d)."""
    scale = d ** -0.5 if scale is None else scale
    st = _lib.lib().drs_attention(q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), v.data_ptr(), v.stride(0),
                                  out.data_ptr(), out.stride(0), B, H, Lq, Lk, d, float(scale), _lib.stream_ptr())
    _lib.check(st, "drs_attention")
    return out


def attention_tc(q, k, vt, out, B, H, Lq, Lk, d, scale=None, vt_img=None):
    """tcgen05 attention; vt = V^T (H*d, >= B*vt_img) view, image b's keys at
    columns b*vt_img.. (vt_img defaults to Lk and must be a multiple of 8)."""
    scale = d ** -0.5 if scale is None else scale
    vt_img = Lk if vt_img is None else vt_img
    st = _lib.lib().drs_attention_tc(q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), vt.data_ptr(),
                                     vt.stride(0), vt_img, out.data_ptr(), out.stride(0), B, H, Lq, Lk, d,
                                     float(scale), _lib.stream_ptr())
    _lib.check(st, "drs_attention_tc")
    return out


def attention_qkv(q, k, v, out, B, H, Lq, Lk, d, scale=None):
    """tcgen05 attention with V row-major (B*Lk rows, head h at column h*d):
    the Q / K / V column blocks of one fused QKV GEMM output, no V^T GEMM."""
    scale = d ** -0.5 if scale is None else scale
    st = _lib.lib().drs_attention_tc_v(q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), v.data_ptr(),
                                       v.stride(0), out.data_ptr(), out.stride(0), B, H, Lq, Lk, d, float(scale),
                                       _lib.stream_ptr())
    _lib.check(st, "drs_attention_tc_v")
    return out


def timestep_embedding(t, dim, out, max_period=10000.0):
    _lib.check(_lib.lib().drs_timestep_embedding(t.data_ptr(), t.numel(), dim, float(max_period), out.data_ptr(),
                                                 _lib.stream_ptr()), "drs_timestep_embedding")
    return out


def patchify(x, C, H, W, p, out):
    _lib.check(_lib.lib().drs_patchify(x.data_ptr(), 1 if x.dtype == torch.float64 else 0, C, H, W, p,
                                       out.data_ptr(), _lib.stream_ptr()), "drs_patchify")
    return out


def unpatchify(tok, c_out, c_keep, H, W, p, out):
    _lib.check(_lib.lib().drs_unpatchify(tok.data_ptr(), c_out, c_keep, H, W, p, out.data_ptr(),
                                         _lib.stream_ptr()), "drs_unpatchify")
    return out


def silu_cast(x, out):
    _lib.check(_lib.lib().drs_silu_cast(x.data_ptr(), x.numel(), out.data_ptr(), _lib.stream_ptr()),
               "drs_silu_cast")
    return out


def im2col(x1, C1, x2, C2, N, H, W, ks, stride, pad, up, out):
    _lib.check(_lib.lib().drs_im2col(x1.data_ptr(), C1, _ptr(x2), C2, N, H, W, ks, stride, pad, up,
                                     out.data_ptr(), _lib.stream_ptr()), "drs_im2col")
    return out


_gn_ws = {}
_gn_old = []

# Instrumentation (bench.py): when TIMERS is a list, every GEMM records
# (flops, start event, end event) on the current stream.
TIMERS = None


def groupnorm(x, N, HW, C, G, gamma, beta, out, eps=1e-5, silu=False):
    # workspace for the two-kernel fallback path only (the cluster path needs none)
    key = x.device
    need = int(_lib.lib().drs_groupnorm_workspace_bytes(N, G))
    ws = _gn_ws.get(key)
    if ws is None or ws.numel() < need:
        if ws is not None:
            _gn_old.append(ws)               # may still be referenced by captured graphs
        ws = torch.empty(max(need, 1 << 17), dtype=torch.uint8, device=x.device)
        _gn_ws[key] = ws
    _lib.check(_lib.lib().drs_groupnorm(x.data_ptr(), 1 if x.dtype == torch.float32 else 0, N, HW, C, G,
                                        gamma.data_ptr(), beta.data_ptr(), float(eps), 1 if silu else 0,
                                        out.data_ptr(), ws.data_ptr(), _lib.stream_ptr()), "drs_groupnorm")
    return out


def latent_to_nhwc(x, C, HW, Cpad, out):
    _lib.check(_lib.lib().drs_latent_to_nhwc(x.data_ptr(), 1 if x.dtype == torch.float64 else 0, C, HW, Cpad,
                                             out.data_ptr(), _lib.stream_ptr()), "drs_latent_to_nhwc")
    return out


def cfg_combine(y, HW, C, g, pair, eps_out):
    _lib.check(_lib.lib().drs_cfg_combine(y.data_ptr(), y.stride(0), HW, C, float(g), 1 if pair else 0,
                                          eps_out.data_ptr(), _lib.stream_ptr()), "drs_cfg_combine")
    return eps_out


def cast_f32_bf16(x, out):
    _lib.check(_lib.lib().drs_cast_f32_bf16(x.data_ptr(), x.numel(), out.data_ptr(), _lib.stream_ptr()),
               "drs_cast_f32_bf16")
    return out

"""HBM roofline of the sampler's elementwise kernels (K2/K3 skip chain, K1 noise)
at latent sizes larger than L2, where they are bandwidth- rather than
latency-bound (the BASELINE latents are 16-131 K elements: a few microseconds).

Algorithmic bytes per element:
  DDIM op, x from HBM, fp64 eps:      8 (x) + 8 (eps) + 8 (out)           = 24
  DDPM noisy op, fp32 eps:            8 (x) + 4 (eps) + 8 (z) + 8 (out)   = 28
  DDPM noisy op, fp64 eps:            8 + 8 + 8 + 8                        = 32
  3-op draft chain (x, eps read once; 3 noisy drafts, z each, 3 outputs):
                                      8 + 8 + 3 * (8 + 8)                  = 64
  noise (PCG64 / SFC64 normal draws): 8 written per draw
GB/s = bytes / (CUDA-event time per launch), warm, back-to-back launches; the
peak is MEASURED_PEAKS.json hbm_gbs (copy bandwidth).

    python tools/sampler_roofline.py [--log2d 25]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, reps=30):
    import torch
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3     # s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2d", type=int, default=25)
    ap.add_argument("--vec", type=int, default=1,
                    help="skip-chain kernel for HBM-sized latents: 0 scalar, 1 16-byte vector (1 pair/thread), 2 (2 pairs)")
    a = ap.parse_args()
    import torch

    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.rng import _KeyBuffer, entropy_key, fill_streams
    from paper_2603_25872_b200.transitions import (ddim_op_coeffs, ddpm_op_coeffs, launch_chain, make_op,
                                                   ops_to_device)

    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak, src = 7700.0, "B200_PROFILING.md fallback"
    dev = torch.device("cuda", 0)
    _lib.lib().drs_set_chain_vec(a.vec)
    D = 1 << a.log2d
    s = P.default_schedule(50)
    x = torch.randn(D, dtype=torch.float64, device=dev)
    e64 = torch.randn(D, dtype=torch.float64, device=dev)
    e32 = e64.float()
    z = torch.randn(3, D, dtype=torch.float64, device=dev)
    outs = torch.empty(3, D, dtype=torch.float64, device=dev)
    rows = []

    def chain(label, ops, bpe):
        od = ops_to_device(ops, dev)
        t = timeit(lambda: launch_chain(od, len(ops), D))
        gbs = bpe * D / t / 1e9
        rows.append((label, bpe, t * 1e6, gbs, gbs / peak))

    c, noisy = ddim_op_coeffs(s, 40, 1, P.VarianceRule.deterministic())
    chain("skip_chain DDIM op (fp64 eps)", [make_op(c, _lib.FAMILY_DDIM, noisy, x=x, eps=e64, out=outs[0])], 24)
    c, noisy = ddpm_op_coeffs(s, 40, 2)
    chain("skip_chain DDPM noisy op (fp32 eps)",
          [make_op(c, _lib.FAMILY_DDPM, noisy, x=x, eps=e32, z=z[0], out=outs[0])], 28)
    chain("skip_chain DDPM noisy op (fp64 eps)",
          [make_op(c, _lib.FAMILY_DDPM, noisy, x=x, eps=e64, z=z[0], out=outs[0])], 32)
    ops = []
    for i in range(3):
        c, noisy = ddpm_op_coeffs(s, 40, 1 + i)
        ops.append(make_op(c, _lib.FAMILY_DDPM, noisy, x=x, eps=e64, z=z[i], out=outs[i]))
    chain("skip_chain 3 DDPM drafts from one anchor", ops, 64)
    if True:                                            # longer draft fans on D/4
        zz = torch.randn(10, D // 4, dtype=torch.float64, device=dev)
        oo = torch.empty(10, D // 4, dtype=torch.float64, device=dev)
        xq, eq = x[:D // 4], e64[:D // 4]
        for k in (6, 10):
            ops = []
            for i in range(k):
                c, noisy = ddpm_op_coeffs(s, 40, 1 + i)
                ops.append(make_op(c, _lib.FAMILY_DDPM, noisy, x=xq, eps=eq, z=zz[i], out=oo[i]))
            od = ops_to_device(ops, dev)
            t = timeit(lambda: launch_chain(od, k, D // 4))
            bpe = 16 + 16 * k
            gbs = bpe * (D // 4) / t / 1e9
            rows.append((f"skip_chain {k} DDPM drafts (D/4)", bpe, t * 1e6, gbs, gbs / peak))

    err = torch.zeros(1, dtype=torch.int32, device=dev)
    for gen in ("pcg64", "sfc64"):
        ns = 148 * 4
        n = D // ns
        kb = _KeyBuffer([entropy_key((0x7A9C, 1, t, 0)) for t in range(ns)], dev)
        tab = torch.empty(ns, n, dtype=torch.float64, device=dev)
        t = timeit(lambda: fill_streams(kb, n, tab, gen, err=err), 10)
        gbs = 8 * ns * n / t / 1e9
        rows.append((f"noise {gen} ({ns} streams x {n} draws)", 8, t * 1e6, gbs, gbs / peak))
    print(f"# chain kernel: {['scalar (skip_chain_kernel)', '16-byte vector, 1 pair/thread', '16-byte vector, 2 pairs/thread'][a.vec]}")
    print(f"# D = 2^{a.log2d} = {D} elements (fp64 state: {8 * D / 2**20:.0f} MiB per array, > 126 MB L2); "
          f"peak {peak} GB/s ({src})")
    for label, bpe, us, gbs, frac in rows:
        print(f"{label:48s} {bpe:3d} B/elem {us:9.1f} us {gbs:8.0f} GB/s  frac {frac:.2f}")


if __name__ == "__main__":
    main()

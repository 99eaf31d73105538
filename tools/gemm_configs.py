"""Every (bn, split, pair) candidate of one GEMM shape, timed like tools/gemm_tune.py
(CUDA graph of back-to-back launches, weights streamed from HBM with --cold),
with its L2 operand traffic (A read once per n-tile group, B once per m-tile group).

    python tools/gemm_configs.py M N K [--cold] [--act gelu_tanh] [--res]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("M", type=int)
    ap.add_argument("N", type=int)
    ap.add_argument("K", type=int)
    ap.add_argument("--cold", action="store_true")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from gemm_tune import tune_shape
    dev = torch.device("cuda", 0)
    best, us, res, _ = tune_shape((a.M, a.N, a.K, None, False, False, False, None), dev, a.reps, a.cold)
    M, N, K = a.M, a.N, a.K
    rows = []
    for (bn, sp, pr), t in res.items():
        n_t = -(-N // bn)
        m_t = -(-M // (256 if pr else 128))
        traffic = (M * K * 2) * n_t + (N * K * 2) * m_t
        ctas = (m_t * n_t * (2 if pr else 1)) * sp
        kb = -(-K // 64) / sp
        per_cta = kb * (128 * 128 + (bn // 2 if pr else bn) * 128)      # A 128 rows + (half) B tile per k-block
        rows.append((t, bn, sp, pr, traffic / 1e6, ctas, per_cta / 1e3))
    for t, bn, sp, pr, mb, ctas, pc in sorted(rows):
        print(f"{M}x{N}x{K} bn={bn:3d} split={sp} pair={pr}: {t:7.2f} us  L2 traffic {mb:6.1f} MB  {ctas:4d} CTAs "
              f"x {pc:6.0f} KB/CTA ({pc / t:5.1f} KB/us/CTA)")


if __name__ == "__main__":
    main()

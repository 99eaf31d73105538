"""Fixed per-launch cost of the tensor-core GEMM inside a CUDA graph of
back-to-back launches, as a function of CTA count and K (tiny M/N tiles),
to separate launch/prologue/epilogue latency from streaming.
    python tools/gemm_floor.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from launch_floor import graph_us  # noqa: E402


def main():
    import torch
    from paper_2603_25872_b200 import netops
    dev = torch.device("cuda", 0)
    for (M, N, K, bn, res) in [(128, 64, 64, 64, 0), (128 * 16, 64, 64, 64, 0), (128 * 74, 64, 64, 64, 0),
                               (128 * 148, 64, 64, 64, 0), (128, 64 * 148, 64, 64, 0), (128 * 148, 128, 64, 128, 0),
                               (128 * 148, 64, 640, 64, 0), (128 * 148, 128, 640, 128, 0),
                               (128 * 148, 128, 640, 128, 1), (2048, 640, 640, 128, 1), (2048, 640, 64, 128, 1)]:
        x = torch.randn(M, K, device=dev).bfloat16()
        w = torch.randn(N, K, device=dev).bfloat16()
        o = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        r = torch.randn(M, N, device=dev).bfloat16() if res else None
        us = graph_us(lambda: netops.linear(x, w, out=o, residual=r, bn=bn, split=1, pair=False))
        ctas = ((M + 127) // 128) * ((N + bn - 1) // bn)
        print(f"M={M:6d} N={N:6d} K={K:4d} bn={bn:3d} res={res} ctas={ctas:4d}: {us:6.2f} us/launch")


if __name__ == "__main__":
    main()

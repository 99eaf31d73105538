"""TFLOP/s of the tcgen05 GEMM (drs_gemm_bf16) vs torch.matmul (cuBLAS) on
large and denoiser-shaped problems.   python tools/gemm_bench.py"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def bench(fn, reps=20):
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    import torch
    from paper_2603_25872_b200.netops import linear
    dev = torch.device("cuda", 0)
    shapes = [(8192, 8192, 8192), (4096, 4096, 4096), (8192, 1280, 5120), (256, 3456, 1152), (256, 4608, 1152),
              (256, 1152, 4608), (8192, 640, 2880), (2048, 1280, 11520), (16384, 640, 640)]
    for M, N, K in shapes:
        x = torch.randn(M, K, device=dev).bfloat16()
        w = torch.randn(N, K, device=dev).bfloat16()
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        flops = 2.0 * M * N * K
        res = []
        for bn in (128, 256):
            ms = bench(lambda: linear(x, w, out=out, bn=bn))
            res.append(f"bn{bn} {flops / ms / 1e9:7.1f}")
        ms_cb = bench(lambda: torch.matmul(x, w.t(), out=out))
        print(f"M={M:5d} N={N:5d} K={K:5d}  ours: {'  '.join(res)} TF/s   cuBLAS {flops / ms_cb / 1e9:7.1f} TF/s")


if __name__ == "__main__":
    main()

"""Per-launch time of small GEMMs inside a CUDA graph of 50 back-to-back
launches (what the UNet graph sees).   python tools/gemm_latency.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_25872_b200.netops import linear
    dev = torch.device("cuda", 0)
    for (M, N, K) in [(8192, 320, 64), (8192, 320, 320), (8192, 320, 2880), (8192, 2560, 320), (2048, 640, 640),
                      (128, 64, 64), (256, 1152, 1152), (8192, 960, 320)]:
        x = torch.randn(M, K, device=dev).bfloat16()
        w = torch.randn(N, K, device=dev).bfloat16()
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        res = []
        for bn in (64, 128, 160, 256):
            linear(x, w, out=out, bn=bn)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(50):
                    linear(x, w, out=out, bn=bn)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            us = e0.elapsed_time(e1) / 50 * 1e3
            res.append(f"bn{bn}:{us:6.1f}us({2 * M * N * K / us / 1e6:5.0f}TF)")
        print(f"M={M:5d} N={N:5d} K={K:5d} " + " ".join(res))


if __name__ == "__main__":
    main()

"""Time a few GEMM configurations (explicit bn / split / pair / kbox) from one
CUDA graph of back-to-back launches -- for A/B runs of two library builds.

    python tools/gemm_ab.py [--kbox 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.getcwd())
sys.path.insert(1, ROOT)

CASES = [  # (label, M, N, K, bn, split, pair, conv)
    ("dit qkv", 256, 3456, 1152, 64, 1, False, None),
    ("dit fc1", 256, 4608, 1152, 64, 1, False, None),
    ("dit fc2 pair-split", 256, 1152, 4608, 64, 3, True, None),
    ("sd15 64x64 conv", 8192, 320, 2880, 160, 1, False, (2, 64, 64, 320)),
    ("sd15 64x64 ff", 8192, 2560, 320, 192, 1, False, None),
    ("sd15 32x32 pair", 2048, 640, 1280, 128, 1, True, None),
    ("sd15 16x16 conv", 512, 1280, 11520, 64, 1, False, (2, 16, 16, 1280)),
    ("8192^3", 8192, 8192, 8192, 256, 1, False, None),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kbox", type=int, default=1)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import inspect
    import torch
    from paper_2603_25872_b200.netops import linear
    has_kbox = "kbox" in inspect.signature(linear).parameters
    dev = torch.device("cuda", 0)
    for label, M, N, K, bn, sp, pr, conv in CASES:
        if conv is not None:
            x = torch.randn(conv[0] * conv[1] * conv[2], conv[3], device=dev).bfloat16()
        else:
            x = torch.randn(M, K, device=dev).bfloat16()
        w = (torch.randn(N, K, device=dev) * 0.02).bfloat16()
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        kw = dict(bn=bn, split=sp, pair=pr, conv=conv, out=out)
        if has_kbox:
            kw["kbox"] = a.kbox
        run = lambda: linear(x, w, **kw)   # noqa: E731
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(a.reps):
                run()
        g.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / a.reps)
        print(f"{label:22s} {M}x{N}x{K} bn={bn} split={sp} pair={int(pr)} kbox={a.kbox if has_kbox else '-'}: "
              f"{best:8.2f} us  {2.0 * M * N * K / best / 1e6:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()

"""Per-launch time of GEMMs (with the UNet's epilogues) inside a CUDA graph of
50 back-to-back launches -- what the network graph sees (L2-warm).

    python tools/gemm_latency.py [--bns 0,64,128,160]     (bn 0 = auto pick)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# (M, N, K, epilogue)   epilogue: plain | bias | geglu | res | res32 (fp32 residual + fp32 out)
SHAPES = [(8192, 320, 320, "res"), (8192, 320, 320, "plain"), (8192, 2560, 320, "geglu"),
          (8192, 320, 1280, "res"), (8192, 320, 2880, "bias"), (2048, 640, 640, "res"),
          (2048, 5120, 640, "geglu"), (512, 1280, 1280, "res"), (512, 10240, 1280, "geglu"),
          (8192, 640, 320, "plain"), (8192, 320, 320, "res32")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bns", default="0")
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    import torch
    from paper_2603_25872_b200.netops import linear
    dev = torch.device("cuda", 0)
    for (M, N, K, epi) in SHAPES:
        x = torch.randn(M, K, device=dev).bfloat16()
        w = torch.randn(N, K, device=dev).bfloat16()
        n_out = N // 2 if epi == "geglu" else N
        f32 = epi == "res32"
        out = torch.empty(M, n_out, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
        bias = torch.randn(N, device=dev)
        res = torch.randn(M, n_out, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
        kw = dict(out=out)
        if epi in ("bias", "geglu", "res", "res32"):
            kw["bias"] = bias
        if epi == "geglu":
            kw["act"] = "geglu"
        if epi in ("res", "res32"):
            kw["residual"] = res
        line = []
        for bn in [int(b) for b in a.bns.split(",")]:
            linear(x, w, bn=bn, **kw)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(a.reps):
                    linear(x, w, bn=bn, **kw)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            us = e0.elapsed_time(e1) / a.reps * 1e3
            line.append(f"bn{bn}:{us:6.1f}us({2 * M * N * K / us / 1e6:5.0f}TF)")
        print(f"M={M:5d} N={N:5d} K={K:5d} {epi:6s} " + " ".join(line))


if __name__ == "__main__":
    main()

"""Sweep BN x split-K for given GEMM shapes (graph replay, L2-warm), to tune
netops.pick_bn / pick_split.

    python tools/gemm_sweep.py 512x1280x11520 128x1280x11520 --bns 64,128,256 --splits 1,2,3,4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shapes", nargs="+")
    ap.add_argument("--bns", default="64,128,160,256")
    ap.add_argument("--splits", default="1,2,4")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    import torch
    from paper_2603_25872_b200.netops import linear, pick
    dev = torch.device("cuda", 0)
    for sh in a.shapes:
        M, N, K = (int(v) for v in sh.split("x"))
        x = torch.randn(M, K, device=dev).bfloat16()
        w = torch.randn(N, K, device=dev).bfloat16()
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        res = torch.randn(M, N, device=dev).bfloat16()
        bias = torch.randn(N, device=dev)
        auto = pick(M, N, K)
        print(f"M={M} N={N} K={K}  auto bn={auto[0]} split={auto[1]}")
        for bn in [int(b) for b in a.bns.split(",")]:
            line = []
            for sp in [int(s) for s in a.splits.split(",")]:
                def run():
                    linear(x, w, bias=bias, residual=res, out=out, bn=bn, split=sp)
                run()
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(a.reps):
                        run()
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                e1.synchronize()
                us = e0.elapsed_time(e1) / a.reps * 1e3
                line.append(f"s{sp}:{us:6.1f}us({2 * M * N * K / us / 1e6:4.0f})")
            print(f"  bn{bn:3d} " + " ".join(line))


if __name__ == "__main__":
    main()

"""Run one GEMM (or implicit 3x3 conv) shape a few times, for ncu captures.
    python tools/gemm_one.py M N K [bn]          plain GEMM
    python tools/gemm_one.py conv N H W C Co      implicit conv"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_25872_b200.netops import linear
    dev = torch.device("cuda", 0)
    if sys.argv[1] == "conv":
        n, h, w, c, co = (int(v) for v in sys.argv[2:7])
        x = torch.randn(n * h * w, c, device=dev).bfloat16()
        wt = torch.randn(co, 9 * c, device=dev).bfloat16()
        out = torch.empty(n * h * w, co, device=dev, dtype=torch.bfloat16)
        run = lambda: linear(x, wt, out=out, conv=(n, h, w, c))   # noqa: E731
    else:
        M, N, K = (int(v) for v in sys.argv[1:4])
        bn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
        x = torch.randn(M, K, device=dev).bfloat16()
        wt = torch.randn(N, K, device=dev).bfloat16()
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        run = lambda: linear(x, wt, out=out, bn=bn)   # noqa: E731
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()

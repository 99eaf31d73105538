"""Run one GEMM (or implicit 3x3 conv) shape a few times, for ncu captures.
    python tools/gemm_one.py M N K [bn] [act] [res]   GEMM (act: none|geglu|gelu_tanh|silu, res: 0|1)
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
        act = sys.argv[5] if len(sys.argv) > 5 and sys.argv[5] != "none" else None
        res = len(sys.argv) > 6 and sys.argv[6] == "1"
        x = torch.randn(M, K, device=dev).bfloat16()
        wt = (torch.randn(N, K, device=dev) * 0.05).bfloat16()
        n_out = N // 2 if act == "geglu" else N
        out = torch.empty(M, n_out, device=dev, dtype=torch.bfloat16)
        r = torch.randn(M, n_out, device=dev).bfloat16() if res else None
        b = torch.randn(N, device=dev)
        run = lambda: linear(x, wt, bias=b, act=act, residual=r, out=out, bn=bn)   # noqa: E731
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()

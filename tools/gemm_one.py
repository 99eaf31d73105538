"""Run one GEMM shape a few times (for ncu).  python tools/gemm_one.py M N K [bn]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_25872_b200.netops import linear
    M, N, K = (int(v) for v in sys.argv[1:4])
    bn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    dev = torch.device("cuda", 0)
    x = torch.randn(M, K, device=dev).bfloat16()
    w = torch.randn(N, K, device=dev).bfloat16()
    b = torch.randn(N, device=dev)
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(5):
        linear(x, w, bias=b, out=out, bn=bn)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()

"""Per-launch cost of the GEMM epilogue variants (output dtype, residual dtype)
on the UNet's residual-GEMM shapes, in CUDA graphs of back-to-back launches.
    python tools/gemm_epi_cost.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from launch_floor import graph_us  # noqa: E402


def main():
    import torch
    from paper_2603_25872_b200 import netops
    dev = torch.device("cuda", 0)
    for (M, N, K) in [(8192, 320, 320), (8192, 320, 1280), (2048, 640, 640), (512, 1280, 1280)]:
        x = torch.randn(M, K, device=dev).bfloat16()
        w = torch.randn(N, K, device=dev).bfloat16()
        b = torch.randn(N, device=dev)
        row = []
        for od, rd in [(torch.bfloat16, None), (torch.float32, None), (torch.bfloat16, torch.bfloat16),
                       (torch.float32, torch.float32)]:
            o = torch.empty(M, N, device=dev, dtype=od)
            r = None if rd is None else torch.randn(M, N, device=dev, dtype=rd)
            us = graph_us(lambda: netops.linear(x, w, bias=b, out=o, residual=r))
            row.append(f"out={str(od)[6:]:8s} res={str(rd)[6:] if rd else '-':8s} {us:6.2f}")
        print(f"{M}x{N}x{K}: " + " | ".join(row))


if __name__ == "__main__":
    main()

"""Per-launch device time of the tcgen05 attention (K6) on UNet/DiT shapes,
replayed from a CUDA graph of `--reps` launches (L2-warm, no profiler).

    python tools/attn_bench.py [--reps 50]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (label, B, H, Lq, Lk, d)
SHAPES = [
    ("sd15 64x64 self", 2, 8, 4096, 4096, 40),
    ("sd15 64x64 cross", 2, 8, 4096, 77, 40),
    ("sd15 32x32 self", 2, 8, 1024, 1024, 80),
    ("sd15 32x32 cross", 2, 8, 1024, 77, 80),
    ("sd15 16x16 self", 2, 8, 256, 256, 160),
    ("sd15 16x16 cross", 2, 8, 256, 77, 160),
    ("sd15 8x8 self", 2, 8, 64, 64, 160),
    ("sdxl 64x64 self", 2, 10, 4096, 4096, 64),
    ("sdxl 32x32 self", 2, 20, 1024, 1024, 64),
    ("dit 256 self", 2, 16, 256, 256, 72),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--only", default="", help="substring of the shape label to run")
    ap.add_argument("--eager", type=int, default=0, help="N eager launches only (for ncu), no timing")
    ap.add_argument("--split", type=int, default=2, help="attention variant (drs_set_attn_split)")
    ap.add_argument("--qkv", type=int, default=0, help="1: row-major V from a fused QKV buffer (attention_qkv)")
    ap.add_argument("--shapes", default="", help="custom shapes 'B,H,Lq,Lk,d;...' instead of the UNet/DiT list")
    a = ap.parse_args()
    shapes = SHAPES
    if a.shapes:
        shapes = [("custom",) + tuple(int(v) for v in t.split(",")) for t in a.shapes.split(";") if t]
    import torch
    from paper_2603_25872_b200 import _lib, netops
    _lib.lib().drs_set_attn_split(a.split)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    for label, B, H, Lq, Lk, d in shapes:
        if a.only and a.only not in label:
            continue
        vt_img = (Lk + 7) // 8 * 8
        q = torch.randn(B * Lq, H * d, device=dev, generator=g).bfloat16()
        k = torch.randn(B * Lk, H * d, device=dev, generator=g).bfloat16()
        vt = torch.randn(H * d, B * vt_img, device=dev, generator=g).bfloat16()
        o = torch.empty(B * Lq, H * d, device=dev, dtype=torch.bfloat16)
        if a.qkv:
            qkv = torch.randn(B * max(Lq, Lk), 3 * H * d, device=dev, generator=g).bfloat16()
            qq, kk, vv = qkv[:B * Lq, :H * d], qkv[:B * Lk, H * d:2 * H * d], qkv[:B * Lk, 2 * H * d:]
            call = lambda: netops.attention_qkv(qq, kk, vv, o, B, H, Lq, Lk, d)   # noqa: E731
        else:
            call = lambda: netops.attention_tc(q, k, vt, o, B, H, Lq, Lk, d, vt_img=vt_img)   # noqa: E731
        if a.eager:
            for _ in range(a.eager):
                call()
            torch.cuda.synchronize()
            continue
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            call()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(a.reps):
                    call()
            gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            gr.replay()
            e1.record(s)
            torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.reps
        dp = 64 if d <= 64 else (128 if d <= 128 else 192)
        fl = 4.0 * B * H * Lq * Lk * d
        print(f"{label:18s} B={B} H={H} Lq={Lq:5d} Lk={Lk:5d} d={d:3d}: {us:8.2f} us  "
              f"{fl / us / 1e6:7.1f} TF/s (d)  {fl * dp / d / us / 1e6:7.1f} TF/s (padded)")


if __name__ == "__main__":
    main()

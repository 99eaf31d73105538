"""LayerNorm per-launch time in a CUDA graph at the UNet's transformer shapes
(fp32 residual stream in, bf16 out).   python tools/ln_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_25872_b200.netops import layernorm
    dev = torch.device("cuda", 0)
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    for _ in range(100):
        a @ a
    for (M, C) in [(8192, 320), (2048, 640), (512, 1280), (128, 1280), (256, 1152), (8192, 640), (2048, 1280), (4096, 1152), (32768, 320)]:
        x = torch.randn(M, C, device=dev)
        g, b = torch.randn(C, device=dev), torch.randn(C, device=dev)
        out = torch.empty(M, C, device=dev, dtype=torch.bfloat16)
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            layernorm(x, out=out, gamma=g, beta=b)
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(50):
                    layernorm(x, out=out, gamma=g, beta=b)
            gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(4):
                gr.replay()
            e1.record(s)
            torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 200
        mb = M * C * 6 / 1e6
        print(f"M={M:5d} C={C:5d}: {us:6.2f} us  ({mb / us:5.2f} TB/s on {mb:.1f} MB)")


if __name__ == "__main__":
    main()

"""Per-kernel floor inside a CUDA graph: a tiny torch op vs tiny libdrs kernels
(with and without PDL), to separate launch cost from kernel work.

    python tools/launch_floor.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def graph_us(fn, reps=50):
    import torch
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    import torch
    from paper_2603_25872_b200 import _lib, netops
    dev = torch.device("cuda", 0)
    a = torch.zeros(256, device=dev)
    b = torch.zeros(256, device=dev, dtype=torch.bfloat16)
    x = torch.randn(128, 64, device=dev).bfloat16()
    w = torch.randn(64, 64, device=dev).bfloat16()
    o = torch.empty(128, 64, device=dev, dtype=torch.bfloat16)
    for pdl in (0, 1):
        _lib.lib().drs_set_pdl(pdl)
        print(f"pdl={pdl}: torch add_ {graph_us(lambda: a.add_(1)):6.2f} us | "
              f"drs cast {graph_us(lambda: netops.cast_f32_bf16(a, b)):6.2f} us | "
              f"drs gemm 128x64x64 {graph_us(lambda: netops.linear(x, w, out=o, bn=64, split=1)):6.2f} us | "
              f"drs attn tiny {graph_us(lambda: netops.attention_tc(x, x, x.t().contiguous(), o, 1, 1, 128, 64, 64)):6.2f} us")
    _lib.lib().drs_set_pdl(0)


if __name__ == "__main__":
    main()

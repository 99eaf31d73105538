"""GroupNorm per-launch time in a CUDA graph: fused cooperative kernel vs the
two-kernel path (forced by an 8-byte-misaligned input view).

    python tools/gn_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.netops import groupnorm
    _lib.lib().drs_set_pdl(int(os.environ.get("PDL", "1")))
    dev = torch.device("cuda", 0)
    # bring the clocks up first (short replays otherwise run at idle clocks)
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    for _ in range(200):
        a @ a
    torch.cuda.synchronize()
    for (N, HW, C) in [(2, 4096, 320), (2, 1024, 640), (2, 256, 1280), (2, 64, 1280), (2, 16384, 320),
                       (16, 4096, 320)]:
        G = 32
        line = []
        for mode, fused in ((1, True), (2, True), (2, False)):
            _lib.lib().drs_set_gn_mode(mode)
            raw = torch.randn(N * HW * C + 8, device=dev).bfloat16()
            x = raw[:N * HW * C].view(N * HW, C) if fused else raw[4:4 + N * HW * C].view(N * HW, C)
            gamma, beta = torch.randn(C, device=dev), torch.randn(C, device=dev)
            out = torch.empty(N * HW, C, device=dev, dtype=torch.bfloat16)
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                groupnorm(x, N, HW, C, G, gamma, beta, out, silu=True)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(20):
                        groupnorm(x, N, HW, C, G, gamma, beta, out, silu=True)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(10):
                    g.replay()
                e1.record(s)
                torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 200
            mb = 2 * N * HW * C * 2 / 1e6
            name = "group" if mode == 1 else ("cluster" if fused else "2-kern")
            line.append(f"{name} {us:6.2f} us ({mb / us:5.2f} TB/s)")
        print(f"N={N:2d} HW={HW:5d} C={C:4d}: " + "   ".join(line))


if __name__ == "__main__":
    main()

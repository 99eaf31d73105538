"""Latency / TFLOP/s of one denoiser-network evaluation (CUDA-graph replay).

    python tools/net_bench.py [--net dit] [--batches 1,2,4,8]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="dit")
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--early", type=int, default=1, help="GEMM weight tiles requested before the PDL wait")
    ap.add_argument("--kb2", type=int, default=-1, help="GEMM 2-k-block TMA boxes (drs_set_gemm_kb2; -1 = default)")
    ap.add_argument("--attn", type=int, default=2, help="attention variant (drs_set_attn_split)")
    a = ap.parse_args()
    import torch
    from paper_2603_25872_b200 import _lib
    _lib.lib().drs_set_pdl(a.pdl)
    _lib.lib().drs_set_early_weights(a.early)
    _lib.lib().drs_set_attn_split(a.attn)
    if a.kb2 >= 0:
        _lib.lib().drs_set_gemm_kb2(a.kb2)
    dev = torch.device("cuda", 0)
    if a.net == "dit":
        from paper_2603_25872_b200.dit import DiT, DiTConfig
        cfg = DiTConfig()
        bs = [int(b) for b in a.batches.split(",")]
        net = DiT(cfg, dev, max_batch=max(bs))
        flops1 = cfg.flops_per_image()
        D = 4 * 32 * 32
    elif a.net in ("sd15", "sdxl"):
        from paper_2603_25872_b200.unet import UNet, sd15_config, sdxl_config
        cfgu = sd15_config() if a.net == "sd15" else sdxl_config()
        bs = [int(b) for b in a.batches.split(",")]
        net = UNet(cfgu, dev, max_batch=max(bs))
        D = net.latent_numel
        xs0 = [torch.randn(D, device=dev, dtype=torch.float64)]
        net.forward(xs0, torch.full((1,), 500.0, device=dev), 1, [torch.empty(D, device=dev)])
        flops1 = net.flops
    else:
        raise SystemExit(f"unknown net {a.net}")
    for B in bs:
        xs = [torch.randn(D, device=dev, dtype=torch.float64) for _ in range(B)]
        outs = [torch.empty(D, device=dev) for _ in range(B)]
        t = torch.full((B,), 500.0, device=dev)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            net.forward(xs, t, B, outs)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            net.forward(xs, t, B, outs)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            g.replay()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"{a.net} B={B}: {ms:.3f} ms/eval  {B * flops1 / ms / 1e9:.1f} TFLOP/s  "
              f"({flops1 / 1e9:.1f} GFLOP/image)")


if __name__ == "__main__":
    main()

"""Per-GEMM-shape time of one network forward (CUDA events around every
drs_gemm launch), plus the non-GEMM remainder.   python tools/gemm_breakdown.py --net sd15"""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="sd15")
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2603_25872_b200 import netops
    dev = torch.device("cuda", 0)
    if a.net == "dit":
        from paper_2603_25872_b200.dit import DiT, DiTConfig
        net, D = DiT(DiTConfig(), dev, max_batch=a.batch), 4096
    else:
        from paper_2603_25872_b200.unet import UNet, sd15_config, sdxl_config
        net = UNet(sd15_config() if a.net == "sd15" else sdxl_config(), dev, max_batch=a.batch)
        D = net.latent_numel
    xs = [torch.randn(D, device=dev, dtype=torch.float64) for _ in range(a.batch)]
    outs = [torch.empty(D, device=dev) for _ in range(a.batch)]
    t = torch.full((a.batch,), 500.0, device=dev)
    net.forward(xs, t, a.batch, outs)
    torch.cuda.synchronize()
    netops.TIMERS = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    net.forward(xs, t, a.batch, outs)
    e1.record()
    torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for f, a0, a1, shp in netops.TIMERS:
        agg[shp][0] += 1
        agg[shp][1] += a0.elapsed_time(a1)
        agg[shp][2] += f
    g_ms = sum(v[1] for v in agg.values())
    print(f"forward (eager, incl. host gaps) {tot:.2f} ms; GEMM device time {g_ms:.2f} ms in {len(netops.TIMERS)} launches")
    for shp, (n, ms, fl) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        M, N, K, bn, sp = shp
        print(f"  M={M:5d} N={N:5d} K={K:5d} bn={bn:3d} split={sp} x{n:3d}: {ms:7.3f} ms  {fl / ms / 1e9:7.1f} TF/s")


if __name__ == "__main__":
    main()

"""One denoiser-network forward bracketed by cudaProfilerStart/Stop (for ncu).

    python tools/profile_net.py [--net dit] [--batch 1]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="dit")
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    import torch
    dev = torch.device("cuda", 0)
    B = a.batch
    if a.net == "dit":
        from paper_2603_25872_b200.dit import DiT, DiTConfig
        net = DiT(DiTConfig(), dev, max_batch=B)
        D = 4096
    elif a.net == "sd15":
        from paper_2603_25872_b200.unet import UNet, sd15_config
        net = UNet(sd15_config(), dev, max_batch=B)
        D = net.latent_numel
    else:
        raise SystemExit(a.net)
    xs = [torch.randn(D, device=dev, dtype=torch.float64) for _ in range(B)]
    outs = [torch.empty(D, device=dev) for _ in range(B)]
    t = torch.full((B,), 500.0, device=dev)
    net.forward(xs, t, B, outs)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    net.forward(xs, t, B, outs)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled one forward")


if __name__ == "__main__":
    main()

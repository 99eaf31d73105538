"""One bench image under the CUDA profiler API, for ncu captures.

    python tools/profile_run.py [--config c2] [--graph]

Warms up (one image), then brackets exactly one image with
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees that image's
launches only.  Eager by default (every kernel is a separate launch ncu can
attribute); --graph replays the captured graph instead.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--graph", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200.pipeline import Sampler

    cfg = bench.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    s = P.default_schedule(cfg["T"])
    D = cfg["D"]
    m = np.zeros((2, D))
    m[0, 0], m[1, 0] = -2.0, 2.0
    den = P.AnalyticEps(P.GaussianMixture(weights=[0.5, 0.5], means=m, variances=[1.0, 1.0]))
    rule = P.VarianceRule.deterministic() if cfg["rule"] == "det" else P.VarianceRule.ddpm_induced()
    smp = Sampler(s, den, D, mode=cfg["mode"], devices=cfg["n"], rule=rule, family=cfg["family"],
                  generator=cfg["generator"], device=dev, graph=a.graph)
    smp.stage(1)
    smp.launch()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    smp.stage(2)
    smp.launch()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    smp.run.check_err()
    print("profiled one image:", smp.launches_per_image, "libdrs launches")


if __name__ == "__main__":
    main()

"""Marginal in-graph cost of each kernel class of one network forward: the
forward is captured once per ablation with that class's launches replaced by
no-ops (results are garbage; only the replay time matters) and the drop in
replay time is what the class costs inside the real graph (gaps, PDL overlap
and tails included -- unlike per-launch events or serialised ncu times).

    python tools/ablate.py [--net sd15]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="sd15")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    from paper_2603_25872_b200 import netops
    dev = torch.device("cuda", 0)
    if a.net == "dit":
        from paper_2603_25872_b200.dit import DiT, DiTConfig
        net, D = DiT(DiTConfig(), dev, max_batch=1), 4096
    else:
        from paper_2603_25872_b200.unet import UNet, sd15_config, sdxl_config
        net = UNet(sd15_config() if a.net == "sd15" else sdxl_config(), dev, max_batch=1)
        D = net.latent_numel
    xs = [torch.randn(D, device=dev, dtype=torch.float64)]
    outs = [torch.empty(D, device=dev)]
    t = torch.full((1,), 500.0, device=dev)
    net.forward(xs, t, 1, outs)
    torch.cuda.synchronize()

    def replay_ms():
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            net.forward(xs, t, 1, outs)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            net.forward(xs, t, 1, outs)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            g.replay()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / a.reps

    orig = {k: getattr(netops, k) for k in ("linear", "groupnorm", "layernorm", "attention_tc", "attention_qkv",
                                            "im2col", "cast_f32_bf16", "latent_to_nhwc", "cfg_combine")}
    noop = lambda *args, **kw: kw.get("out")            # noqa: E731

    def gemm_if(pred):
        def f(x, w, *args, **kw):
            conv = kw.get("conv")
            M = conv[0] * conv[1] * conv[2] if conv else x.shape[0]
            K = 9 * conv[3] if conv else x.shape[1]
            if pred(M, w.shape[0], K, kw):
                return kw.get("out")
            return orig["linear"](x, w, *args, **kw)
        return f

    cases = [
        ("all GEMMs", {"linear": noop}),
        ("GEGLU GEMMs", {"linear": gemm_if(lambda M, N, K, kw: kw.get("act") == "geglu")}),
        ("conv GEMMs", {"linear": gemm_if(lambda M, N, K, kw: kw.get("conv") is not None)}),
        ("GEMMs K<=1280 non-conv", {"linear": gemm_if(lambda M, N, K, kw: kw.get("conv") is None and K <= 1280)}),
        ("GEMMs M<=512", {"linear": gemm_if(lambda M, N, K, kw: M <= 512)}),
        ("GroupNorm", {"groupnorm": noop}),
        ("LayerNorm", {"layernorm": noop}),
        ("attention", {"attention_tc": noop, "attention_qkv": noop}),
        ("im2col/upsample/concat", {"im2col": noop}),
        ("cast f32->bf16", {"cast_f32_bf16": noop}),
    ]
    base = replay_ms()
    print(f"{a.net}: full forward {base:.3f} ms")
    for name, patch in cases:
        for k, f in patch.items():
            setattr(netops, k, f)
        try:
            ms = replay_ms()
        finally:
            for k in patch:
                setattr(netops, k, orig[k])
        print(f"  without {name:26s}: {ms:7.3f} ms   -> class costs {base - ms:6.3f} ms ({(base - ms) / base:5.1%})")


if __name__ == "__main__":
    main()

"""Measure the best (bn, split, cta_pair) for every GEMM shape the denoiser
networks issue and write paper_2603_25872_b200/gemm_table.json (read by
netops.pick3).

Each candidate is timed inside a CUDA graph of back-to-back launches with the
shape's own epilogue (activation, residual dtype, output dtype, implicit conv),
which is how the network graphs run it.  The table is keyed by M x N x K
(+ ":conv"), so the result is deterministic for a given table.

    python tools/gemm_tune.py [--nets sd15:1,2,4,8 dit:1,2,4,8 sdxl:1,2] [--out PATH]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BNS = (64, 128, 160, 192, 256)
KBOX = False      # --with-kbox: also search 1 / 2 k-blocks per TMA box
SPLITS = (1, 2, 3, 4, 6, 8)


def collect(net_name, batches, dev):
    import torch
    from paper_2603_25872_b200 import netops
    bmax = max(batches)
    if net_name == "dit":
        from paper_2603_25872_b200.dit import DiT, DiTConfig
        net, D = DiT(DiTConfig(), dev, max_batch=bmax), 4 * 32 * 32
    else:
        from paper_2603_25872_b200.unet import UNet, sd15_config, sdxl_config
        net = UNet(sd15_config() if net_name == "sd15" else sdxl_config(), dev, max_batch=bmax)
        D = net.latent_numel
    shapes = []
    for B in batches:
        xs = [torch.randn(D, device=dev, dtype=torch.float64) for _ in range(B)]
        outs = [torch.empty(D, device=dev) for _ in range(B)]
        netops.SHAPES = []
        net.forward(xs, torch.full((B,), 500.0, device=dev), B, outs)
        torch.cuda.synchronize()
        shapes += netops.SHAPES
        netops.SHAPES = None
    del net
    torch.cuda.empty_cache()
    return shapes


def time_config(run, reps):
    import torch
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            run()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def tune_shape(desc, dev, reps, cold=False):
    import torch
    from paper_2603_25872_b200.netops import linear, pick
    M, N, K, act, res_f32, has_res, out_f32, conv = desc
    if conv is not None:
        cn, ch, cw, cc = conv[:4]
        s2 = conv[4] if len(conv) > 4 else 1              # stride-2 conv: input is (s H) x (s W)
        x = torch.randn(cn * ch * cw * s2 * s2, cc, device=dev).bfloat16()
    else:
        x = torch.randn(M, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) * 0.02).bfloat16()
    # cold: the graph's launches rotate over enough weight copies (> 2x L2) that
    # every launch streams its weights from HBM, as in the network (1.7 GB of weights)
    copies = max(1, min(reps, -(-(256 << 20) // (N * K * 2)))) if cold else 1
    ws = [w] + [w.clone() for _ in range(copies - 1)]
    wi = [0]

    def wnext():
        wi[0] = (wi[0] + 1) % copies
        return ws[wi[0]]
    n_out = N // 2 if act == "geglu" else N
    out = torch.empty(M, n_out, device=dev, dtype=torch.float32 if out_f32 else torch.bfloat16)
    res = None
    if has_res:
        res = torch.randn(M, n_out, device=dev, dtype=torch.float32 if res_f32 else torch.bfloat16)
    bias = torch.randn(N, device=dev)
    tiles_of = lambda bn: ((M + 127) // 128) * ((N + bn - 1) // bn)   # noqa: E731
    kb = (K + 63) // 64
    results = {}
    kboxes = (1, 2) if KBOX and K % 64 == 0 else (1,)
    for bn in BNS:
        for sp in SPLITS:
            for pr in (0, 1):
                if pr and M < 256:
                    continue
                # split-K runs one wave of clusters: 1-SM tiles x split, or pair tiles x 2 x split CTAs
                ctas = (((M + 255) // 256) * ((N + bn - 1) // bn) * 2 if pr else tiles_of(bn)) * sp
                if sp > 1 and (ctas > 148 or kb // sp < 4):
                    continue
                for kx in kboxes:
                    run = lambda bn=bn, sp=sp, pr=pr, kx=kx: linear(x, wnext(), bias=bias, act=act,   # noqa: E731
                                                                    residual=res, out=out, bn=bn, split=sp,
                                                                    conv=conv, pair=bool(pr), kbox=kx)
                    results[(bn, sp, pr, kx) if KBOX else (bn, sp, pr)] = time_config(run, reps)
    best = min(results, key=results.get)
    model = (pick(M, N, K, 0, 0, False) + ((0, 1) if KBOX else (0,))) if conv is None else None
    return best, results[best], results, model


def tune_kbox(desc, cfg, dev, reps, cold=False):
    """Time the table's (bn, split, pair) for this shape with 1 and 2 k-blocks per TMA box."""
    import torch
    from paper_2603_25872_b200.netops import linear
    M, N, K, act, res_f32, has_res, out_f32, conv = desc
    if conv is not None:
        cn, ch, cw, cc = conv[:4]
        s2 = conv[4] if len(conv) > 4 else 1
        x = torch.randn(cn * ch * cw * s2 * s2, cc, device=dev).bfloat16()
    else:
        x = torch.randn(M, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) * 0.02).bfloat16()
    copies = max(1, min(reps, -(-(256 << 20) // (N * K * 2)))) if cold else 1
    ws = [w] + [w.clone() for _ in range(copies - 1)]
    wi = [0]

    def wnext():
        wi[0] = (wi[0] + 1) % copies
        return ws[wi[0]]
    n_out = N // 2 if act == "geglu" else N
    out = torch.empty(M, n_out, device=dev, dtype=torch.float32 if out_f32 else torch.bfloat16)
    res = torch.randn(M, n_out, device=dev, dtype=torch.float32 if res_f32 else torch.bfloat16) if has_res else None
    bias = torch.randn(N, device=dev)
    bn, sp, pr = cfg[0], cfg[1], bool(cfg[2]) if len(cfg) > 2 else False
    t = {}
    for kbox in (1, 2):
        run = lambda kbox=kbox: linear(x, wnext(), bias=bias, act=act, residual=res, out=out, bn=bn,   # noqa: E731
                                       split=sp, conv=conv, pair=pr, kbox=kbox)
        t[kbox] = time_config(run, reps)
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nets", nargs="+", default=["sd15:1,2,4,8", "dit:1,2,4,8", "sdxl:1,2"])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2603_25872_b200", "gemm_table.json"))
    ap.add_argument("--cold", action="store_true", help="weights streamed from HBM (rotating copies)")
    ap.add_argument("--mmax", type=int, default=0, help="only shapes with M <= mmax")
    ap.add_argument("--merge", action="store_true", help="update the existing table instead of replacing it")
    ap.add_argument("--only-missing", action="store_true", help="with --merge: tune only shapes not in the table")
    ap.add_argument("--with-kbox", action="store_true", help="full search including 1 / 2 k-blocks per TMA box")
    ap.add_argument("--kbox", action="store_true",
                    help="keep each entry's (bn, split, pair); choose 1 or 2 k-blocks per TMA box")
    a = ap.parse_args()
    global KBOX
    KBOX = a.with_kbox
    import torch
    from paper_2603_25872_b200 import netops
    netops._TABLE = {}                       # tune against the model, not an old table
    dev = torch.device("cuda", 0)
    uniq = {}
    for spec in a.nets:
        name, bs = spec.split(":")
        for d in collect(name, [int(b) for b in bs.split(",")], dev):
            key = netops.table_key(d[0], d[1], d[2], False if d[7] is None else (d[7][4] if len(d[7]) > 4 else 1))
            if d[3] == "headsoftmax":          # fixed tile (bn 192, 1-SM): nothing to tune
                continue
            if not a.mmax or d[0] <= a.mmax:
                uniq.setdefault(key, d)
    print(f"{len(uniq)} unique GEMM shapes", flush=True)
    table, t0 = {}, time.time()
    base = os.path.join(ROOT, "paper_2603_25872_b200", "gemm_table.json")
    if a.merge and os.path.exists(base):
        table = {k: list(v) for k, v in json.load(open(base))["configs"].items()}
    tot_best = tot_model = 0.0
    if a.kbox:
        tot1 = tot_sel = 0.0
        for key, d in sorted(uniq.items()):
            cfg = table.get(key)
            if cfg is None or d[2] % 64:
                continue
            t = tune_kbox(d, cfg[:3], dev, a.reps, a.cold)
            kbox = min(t, key=t.get)
            if t[kbox] > t[1] * 0.98:
                kbox = 1
            table[key] = list(cfg[:3]) + [kbox] if len(cfg) > 2 else list(cfg[:2]) + [0, kbox]
            tot1 += t[1]
            tot_sel += t[kbox]
            print(f"{key:24s} bn={cfg[0]:3d} split={cfg[1]} pair={cfg[2] if len(cfg) > 2 else 0}  kbox1 {t[1]:8.1f} us  kbox2 {t[2]:8.1f} us -> {kbox}",
                  flush=True)
        print(f"kbox pass: sum {tot1:.0f} us (1 k-block per box) -> {tot_sel:.0f} us (selected)")
        uniq = {}
    if a.only_missing:
        uniq = {k: d for k, d in uniq.items() if k not in table}
        print(f"{len(uniq)} shapes missing from the table", flush=True)
    for key, d in sorted(uniq.items()):
        best, us, res, model = tune_shape(d, dev, a.reps, a.cold)
        table[key] = list(best)
        mt = res.get(model, float("nan")) if model else float("nan")
        if model in res:
            tot_best += us
            tot_model += mt
        print(f"{key:24s} best bn={best[0]:3d} split={best[1]} pair={best[2]} kbox={best[3] if len(best) > 3 else 1} "
              f"{us:8.1f} us   model {model} "
              f"{mt:8.1f} us",
              flush=True)
    print(f"tuned {len(table)} shapes in {time.time() - t0:.0f} s; sum best {tot_best:.0f} us vs model "
          f"{tot_model:.0f} us (shapes the model covers)")
    with open(a.out, "w") as f:
        json.dump({"device": torch.cuda.get_device_name(0), "tool": "tools/gemm_tune.py",
                   "configs": dict(sorted(table.items()))}, f, indent=1)
        f.write("\n")
    print("wrote", a.out)


if __name__ == "__main__":
    main()

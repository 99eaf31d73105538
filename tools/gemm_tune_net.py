"""In-network GEMM tuning: greedy coordinate descent over the (bn, split,
cta_pair, kbox) of each GEMM shape of one network forward, scored by the replay time
of the WHOLE forward's CUDA graph (the isolated tuner, tools/gemm_tune.py, times
a shape repeated back to back -- L2-warm, no neighbours -- which misranks some
configurations inside the real graph).  Updates gemm_table.json in place for
the shapes it improves.

    python tools/gemm_tune_net.py [--net sd15] [--batch 1] [--rounds 1] [--out PATH]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="sd15")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2603_25872_b200", "gemm_table.json"))
    ap.add_argument("--full", action="store_true", help="every (bn, split, pair, kbox) instead of single-coordinate moves")
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
    B = a.batch
    xs = [torch.randn(D, device=dev, dtype=torch.float64) for _ in range(B)]
    outs = [torch.empty(D, device=dev) for _ in range(B)]
    t = torch.full((B,), 500.0, device=dev)
    netops.SHAPES = []
    net.forward(xs, t, B, outs)
    shapes, netops.SHAPES = netops.SHAPES, None
    table = netops._table()

    def replay_ms():
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
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                g.replay()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / a.reps)
        del g
        return best

    uniq = {}
    for d in shapes:
        if d[3] == "headsoftmax":
            continue
        cv = False if d[7] is None else (d[7][4] if len(d[7]) > 4 else 1)
        key = netops.table_key(d[0], d[1], d[2], cv)
        uniq.setdefault(key, (d, cv))
    base = replay_ms()
    print(f"{a.net} B={B}: start {base:.4f} ms/forward, {len(uniq)} shapes", flush=True)
    for rnd in range(a.rounds):
        for key, (d, cv) in uniq.items():
            M, N, K = d[0], d[1], d[2]
            kb = (K + 63) // 64
            c0 = tuple(table.get(key, netops.pick3(M, N, K, 0, 0, cv)))
            cur = (c0[0], c0[1], int(c0[2]) if len(c0) > 2 else 0, int(c0[3]) if len(c0) > 3 else 1)
            kboxes = (1, 2) if K % 64 == 0 else (1,)

            def ok(c):
                bn, sp, pr, kx = c
                if pr and M < 256:
                    return False
                tiles = ((M + 127) // 128) * ((N + bn - 1) // bn)
                ptiles = ((M + 255) // 256) * ((N + bn - 1) // bn)
                ctas = (ptiles * 2 if pr else tiles) * sp
                return not (sp > 1 and (ctas > 148 or kb // sp < 4 or (pr and sp > 4)))
            if a.full:
                cands = [(bn, sp, pr, kx) for bn in netops.BN_CHOICES for sp in (1, 2, 3, 4, 6, 8) for pr in (0, 1)
                         for kx in kboxes]
            else:                                   # single-coordinate moves from the current entry
                bn0, sp0, pr0, kx0 = cur
                cands = ([(bn, sp0, pr0, kx0) for bn in netops.BN_CHOICES] +
                         [(bn0, sp, pr0, kx0) for sp in (1, 2, 3, 4, 6, 8)] +
                         [(bn0, sp0, 1 - pr0, kx0)] + [(bn0, sp0, pr0, kx) for kx in kboxes])
            cands = [c for c in dict.fromkeys(cands) if ok(c)]
            best_cfg, best_ms = cur, base
            for c in cands:
                if c == cur:
                    continue
                table[key] = c
                try:
                    ms = replay_ms()
                except Exception:                       # configuration the kernel rejects
                    ms = 1e30
                if ms < best_ms * 0.9985:
                    best_cfg, best_ms = c, ms
            table[key] = best_cfg
            if best_cfg != cur:
                print(f"  {key:24s} {cur} -> {best_cfg}: {base:.4f} -> {best_ms:.4f} ms", flush=True)
                base = best_ms
    final = replay_ms()
    print(f"final {final:.4f} ms/forward", flush=True)
    full = json.load(open(a.out)) if os.path.exists(a.out) else {"configs": {}}
    full["configs"].update({k: list(v) for k, v in table.items()})
    full["configs"] = dict(sorted(full["configs"].items()))
    full["tool"] = "tools/gemm_tune.py + tools/gemm_tune_net.py"
    with open(a.out, "w") as f:
        json.dump(full, f, indent=1)
        f.write("\n")
    print("wrote", a.out)


if __name__ == "__main__":
    main()

"""GEMM time per network eval by shape: launch count x tuned per-launch time
(profiles/r1_gemm_tune.log), with each shape's TF/s -- where the GEMM share
of an eval goes.   python tools/gemm_mix.py --net sd15 --batch 1"""
import argparse
import collections
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="sd15")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--log", default=os.path.join(ROOT, "profiles", "r1_gemm_tune.log"))
    a = ap.parse_args()
    import torch
    from paper_2603_25872_b200 import netops
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from gemm_tune import collect
    times = {}
    for line in open(a.log):
        m = re.match(r"(\S+)\s+best bn=\s*(\d+) split=(\d+)(?: pair=(\d))?\s+([\d.]+) us", line)
        if m:
            times[m.group(1)] = (float(m.group(5)), m.group(2), m.group(3), m.group(4))
    shapes = collect(a.net, [a.batch], torch.device("cuda", 0))
    cnt = collections.Counter(netops.table_key(d[0], d[1], d[2], d[7] is not None) for d in shapes)
    rows, tot = [], 0.0
    for k, n in cnt.items():
        us, bn, sp, pr = times.get(k, (float("nan"), "?", "?", "?"))
        M, N, K = (int(v) for v in k.split(":")[0].split("x"))
        rows.append((n * us, k, n, us, 2 * M * N * K / us / 1e6, bn, sp, pr))
        tot += n * us
    rows.sort(reverse=True)
    for t, k, n, us, tf, bn, sp, pr in rows:
        print(f"{k:24s} x{n:3d}  {us:7.1f} us  {tf:6.0f} TF/s  bn={bn} split={sp} pair={pr}  "
              f"total {t:8.1f} us ({100 * t / tot:4.1f}%)")
    print(f"GEMM total per eval: {tot / 1000:.3f} ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main()

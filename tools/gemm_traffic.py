"""DRAM traffic of the network's tensor-core GEMMs vs their algorithmic bytes.

    python tools/gemm_traffic.py record --net sd15 > gpurun_out/gemm_algo.json
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
        --clock-control none --profile-from-start off -k regex:gemm --csv --log-file gpurun_out/gemm_dram.csv \
        python tools/profile_net.py --net sd15
    python tools/gemm_traffic.py summarise gpurun_out/gemm_algo.json gpurun_out/gemm_dram.csv

`record` lists every GEMM of one forward with its algorithmic bytes (A and B
read once, C written once, residual read once); `summarise` joins it with the
ncu per-launch DRAM bytes (same launch order; caches not flushed, so operands
produced by the previous kernel are L2 hits as in the real graph) and prints
the per-launch averages that bench.py reports as roofline.traffic
(profiles/dram_traffic.json)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def record(net_name):
    import torch
    from paper_2603_25872_b200 import netops
    from paper_2603_25872_b200.unet import UNet, sd15_config, sdxl_config
    dev = torch.device("cuda", 0)
    net = UNet(sd15_config() if net_name == "sd15" else sdxl_config(), dev, max_batch=1)
    D = net.latent_numel
    xs = [torch.randn(D, device=dev, dtype=torch.float64)]
    outs = [torch.empty(D, device=dev)]
    t = torch.full((1,), 500.0, device=dev)
    net.forward(xs, t, 1, outs)
    netops.GEMM_RECORD = []
    net.forward(xs, t, 1, outs)
    rec, netops.GEMM_RECORD = netops.GEMM_RECORD, None
    torch.cuda.synchronize()
    rows = []
    for flops, g in rec:
        n_out = g.N // 2 if g.act == netops.ACT["geglu"] else g.N
        elem = 4 if g.out_f32 else 2
        a_cols = g.conv_C if g.conv_C > 0 else g.K        # implicit conv: the NHWC input once, not 9x
        byts = 2 * g.M * a_cols + 2 * g.N * g.K + elem * g.M * n_out
        if g.residual:
            byts += (4 if g.res_f32 else 2) * g.M * n_out
        rows.append({"M": g.M, "N": g.N, "K": g.K, "conv_C": g.conv_C, "act": g.act, "out_f32": g.out_f32,
                     "res": int(bool(g.residual)), "res_f32": g.res_f32, "flops": flops, "algo_bytes": byts})
    print(json.dumps(rows))


def summarise(algo_path, csv_path):
    algo = json.load(open(algo_path))
    launches = {}
    hdr = None
    for r in csv.reader(open(csv_path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
                 "msecond": 1e3}.get(u, 1.0)
        launches.setdefault(key, {})[d["Metric Name"]] = v * scale
    rows = [launches[k] for k in sorted(launches, key=int)]
    n = min(len(rows), len(algo))
    dram = sum(r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0) for r in rows[:n])
    ab = sum(a["algo_bytes"] for a in algo[:n])
    out = {"gemm_bf16_tc_kernel (tcgen05.mma, TMA, TMEM)": dram / n,
           "_detail": {"net": "sd15", "launches": n, "dram_bytes_per_launch": dram / n, "algorithmic_bytes_per_launch": ab / n,
                       "dram_over_algorithmic": dram / ab, "source": os.path.basename(csv_path),
                       "method": "ncu dram__bytes_read.sum + dram__bytes_write.sum per GEMM launch of one SD1.5 "
                                 "forward (--cache-control none), averaged"}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "record":
        net = sys.argv[sys.argv.index("--net") + 1] if "--net" in sys.argv else "sd15"
        record(net)
    else:
        summarise(sys.argv[2], sys.argv[3])

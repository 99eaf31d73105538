"""Benchmark: DRiffusion ms/image on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one image sampled end to end (x_T -> x_0) through the compiled
pipeline call (skipdiff cli._run_once semantics: x_T = INIT noise of the
step's seed, then the configured sampler).  Default workload at N=1 is
BASELINE config C2: the toy Gaussian-mixture eps (2 components, +-2 e_0,
D = 4x32x32 = 4096, fp64), DDPM family, aggressive mode n=3, SFC64 noise
streams, T=50; with one GPU the 3 logical devices' evaluations run as one
batched launch per round.  With --gpus N > 1 (torchrun, one rank per GPU)
the same config runs with n = N devices, rank r evaluating draft r+1 and the
eps rows all-gathered over NCCL each round (latency: time per image, max over
ranks).  Prints one JSON line on rank 0.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (T, D, mode, n, family, rule, generator)
    "c1": dict(T=50, D=4096, mode="conservative", n=2, family="ddim", rule="det", generator="pcg64",
               desc="toy GM eps, DDIM 50 steps, 4x32x32, conservative n=2, pcg64"),
    "c2": dict(T=50, D=4096, mode="aggressive", n=3, family="ddpm", rule="det", generator="sfc64",
               desc="toy GM eps, DDPM 50 steps, 4x32x32, aggressive n=3, sfc64 noise"),
}


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ CPU legs ----
def _oracle_image(cfg, seed):
    import skipdiff_oracle as O
    ab = O.default_alpha_bar(cfg["T"])
    x_T = O.derive_noise(seed, cfg["T"], O.INIT, cfg["D"], cfg["generator"])
    rule = ("det",) if cfg["rule"] == "det" else ("ddpm",)
    states, _, _ = O.run_parallel(ab, O.toy_bimodal(cfg["D"]), x_T, cfg["n"], cfg["mode"], rule, seed,
                                  family=cfg["family"], generator=cfg["generator"])
    return states[-1][1]


def cpu_baseline(cfg, seconds):
    """The reference's algorithm (oracle port, numpy) on this host's cores,
    bounded to ~`seconds` of CPU work."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    _oracle_image(cfg, 10_000)                       # warm-up
    times, t_end, seed = [], time.perf_counter() + seconds, 20_000
    while time.perf_counter() < t_end or len(times) < 3:
        t0 = time.perf_counter()
        _oracle_image(cfg, seed)
        times.append((time.perf_counter() - t0) * 1e3)
        seed += 1
    return {"value": statistics.mean(times), "unit": "ms/image", "cores": 1, "kind": "port",
            "sample": f"{len(times)} images of {cfg['desc']} (oracle/skipdiff_oracle.py run_parallel, "
                      f"numpy single-threaded), ~{seconds:.0f} s of CPU work"}


def run_reference_arm(a, cfg, rank):
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    for i in range(a.warmup):
        _oracle_image(cfg, 1000 + i)
    times = []
    for i in range(a.steps):
        t0 = time.perf_counter()
        _oracle_image(cfg, i)
        times.append((time.perf_counter() - t0) * 1e3)
    v = statistics.mean(times)
    line = {"impl": "reference", "metric": "ms/image sampling latency", "value": v, "unit": "ms/image",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": a.config, "desc": cfg["desc"]},
            "cpu_baseline": {"value": v, "unit": "ms/image", "cores": 1, "kind": "port",
                             "sample": f"{a.steps} images, oracle port of skipdiff run_parallel (numpy)"},
            "e2e": {"value": v, "unit": "ms/image", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU leg -----
def main():
    a = _args()
    cfg = CONFIGS[a.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if a.impl == "reference":
        run_reference_arm(a, cfg, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200.engine import Comm
    from paper_2603_25872_b200.pipeline import Sampler

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = Comm(rank, world)
    n = cfg["n"] if world == 1 else world

    s = P.default_schedule(cfg["T"])
    D = cfg["D"]
    m = np.zeros((2, D))
    m[0, 0], m[1, 0] = -2.0, 2.0
    den = P.AnalyticEps(P.GaussianMixture(weights=[0.5, 0.5], means=m, variances=[1.0, 1.0]))
    rule = P.VarianceRule.deterministic() if cfg["rule"] == "det" else P.VarianceRule.ddpm_induced()
    sampler = Sampler(s, den, D, mode=cfg["mode"], devices=n, rule=rule, family=cfg["family"],
                      generator=cfg["generator"], comm=comm, device=dev)
    seq = Sampler(s, den, D, mode="sequential", rule=rule, family=cfg["family"], generator=cfg["generator"],
                  device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed_images(smp, steps, seed0, world_sync=True):
        """Device time per image (inputs staged in HBM before the start event);
        L2 flushed between images, outside the timed window."""
        ts = []
        for i in range(steps):
            smp.stage(seed0 + i)
            flush.zero_()
            if world_sync:
                barrier()
            else:
                torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            smp.launch()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return ts

    for i in range(max(a.warmup, 3)):
        sampler.stage(1000 + i)
        sampler.launch()
    barrier()
    with ClockSampler(local) as clk:
        per_image = timed_images(sampler, a.steps, 0)
    t_img = torch.tensor([statistics.mean(per_image)], device=dev)
    if world > 1:
        dist.all_reduce(t_img, op=dist.ReduceOp.MAX)
    value = float(t_img.item())
    sampler.run.check_err()

    # end to end through the public pipeline call: x_T from pinned host memory,
    # final sample back to pinned host memory, synchronised, wall clock
    x_hosts = [P.derive_noise(P.RngStream(50_000 + i, cfg["generator"]), cfg["T"], P.Role.INIT, D,
                              device=dev).cpu().pin_memory() for i in range(a.steps)]
    out_host = torch.empty(D, dtype=torch.float64).pin_memory()
    sampler(49_999, x_T=x_hosts[0], out=out_host)          # warm the explicit-x_T graph
    e2e = []
    for i in range(a.steps):
        barrier()
        t0 = time.perf_counter()
        sampler(50_000 + i, x_T=x_hosts[i], out=out_host)
        e2e.append((time.perf_counter() - t0) * 1e3)
    t_e2e = torch.tensor([statistics.mean(e2e)], device=dev)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)

    # kernel classes: per-launch CUDA events over eager replays of the same run
    timers = []
    for i in range(3):
        sampler.stage(2000 + i)
        torch.cuda.synchronize(dev)
        sampler.run.enqueue(timers=timers)
    torch.cuda.synchronize(dev)
    classes = {}
    for label, nbytes, e0, e1 in timers:
        c = classes.setdefault(label, {"ms": 0.0, "bytes": 0, "launches": 0})
        c["ms"] += e0.elapsed_time(e1)
        c["bytes"] += nbytes
        c["launches"] += 1
    kernels = {k: v for k, v in classes.items() if k != "gather"}
    top = max(kernels, key=lambda k: kernels[k]["ms"])
    peaks = _peaks()
    avg_ms = kernels[top]["ms"] / kernels[top]["launches"]
    algo = kernels[top]["bytes"] / kernels[top]["launches"]
    achieved = algo / (avg_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(prof):
        traffic = json.load(open(prof)).get(top)

    # 1-GPU sequential baseline T1 (the reference's `sequential` bench row)
    for i in range(3):
        seq.stage(3000 + i)
        seq.launch()
    torch.cuda.synchronize(dev)
    seq_ms = statistics.mean(timed_images(seq, max(5, a.steps // 2), 0, False)) if rank == 0 else None

    if rank != 0:
        dist.destroy_process_group()
        return
    plan = sampler.prog.plan
    rounds = len(sampler.prog.rounds)
    line = {
        "metric": "ms/image sampling latency", "value": value, "unit": "ms/image", "n_gpus": world,
        "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": value, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": a.config, "desc": cfg["desc"], "T": cfg["T"], "latent": "4x32x32",
                   "mode": cfg["mode"], "devices": n, "family": cfg["family"], "noise": cfg["generator"],
                   "denoiser": "toy gaussian mixture (2 comps, +-2 e0), fp64", "batch": 1,
                   "l2": "flushed between timed images (256 MB memset outside the events)",
                   "graph": sampler.use_graph},
        "e2e": {"value": float(t_e2e.item()), "unit": "ms/image", "h2d_bytes_per_step": D * 8 + 16,
                "d2h_bytes_per_step": D * 8,
                "how": "Sampler(seed, x_T=pinned host, out=pinned host), wall clock incl. sync"},
        "gpu_launches": sampler.launches_per_image * a.steps,
        "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peaks.get("hbm_gbs"),
                     "unit": "GB/s", "frac": achieved / peaks.get("hbm_gbs"), "traffic": traffic,
                     "algo_bytes_per_launch": algo, "avg_launch_us": avg_ms * 1e3,
                     "peak_source": "fallback" if peaks.get("_fallback") else "MEASURED_PEAKS.json hbm_gbs"},
        "kernels": {k: {"ms_per_image": v["ms"] / 3, "launches_per_image": v["launches"] // 3,
                        "gbs": (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["ms"] else None}
                    for k, v in classes.items()},
        "clocks": clk.summary(),
        "drf": {"sequential_1gpu_ms": seq_ms, "rounds": rounds, "T": cfg["T"],
                "round_law_ms": seq_ms * rounds / cfg["T"] if seq_ms else None,
                "ideal_1_over_n_ms": seq_ms / n if seq_ms else None,
                "ideal_2_over_n_plus_1_ms": seq_ms * 2 / (n + 1) if seq_ms else None,
                "speedup_vs_sequential": seq_ms / value if seq_ms else None,
                "plan_blocks": [list(b) for b in plan.blocks] if plan else None},
    }
    if not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, a.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

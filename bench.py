"""Benchmark: DRiffusion ms/image on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Metric: "ms/image sampling latency at 1/2/4/8 B200 vs 1/n, 2/(n+1) ideal".
One step = one image sampled end to end (x_T -> x_0) through the compiled
pipeline call (skipdiff cli._run_once semantics: x_T = INIT noise of the
step's seed, then the sampler).  Default workload: BASELINE config C3, the
config the 1/2/4/8-GPU metric is quoted on -- SD1.5-shaped UNet (random
init, bf16 tcgen05 kernels), 4x64x64 latent, classifier-free guidance as a
batch-2 (uncond, cond) forward (g = 7.5), DDIM 50 steps:
  N = 1   the 1-GPU sequential sampler (T1 of the metric)
  N > 1   aggressive draft-and-refine with n = N devices, one process per
          GPU (torchrun): rank r evaluates draft r+1, eps rows all-gathered
          over NCCL each round, refine replayed on every rank.
Other configs: c1/c2 (toy Gaussian-mixture eps), c4 (DiT-XL/2, DDPM 250,
conservative), c5 (SDXL-shaped UNet 4x128x128, DDIM 30).  Prints one JSON
line on rank 0.
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
    "c1": dict(net="toy", T=50, size=32, mode="conservative", n=2, family="ddim", rule="det", generator="pcg64",
               desc="toy GM eps, DDIM 50, 4x32x32, conservative n=2"),
    "c2": dict(net="toy", T=50, size=32, mode="aggressive", n=3, family="ddpm", rule="det", generator="sfc64",
               desc="toy GM eps, DDPM 50, 4x32x32, aggressive n=3, sfc64 noise"),
    "c3": dict(net="sd15", T=50, size=64, mode="aggressive", n=8, family="ddim", rule="det", generator="pcg64",
               desc="SD1.5-shaped UNet (random init), 4x64x64, CFG batch 2 (g=7.5), DDIM 50, aggressive n=N"),
    "c4": dict(net="dit", T=250, size=32, mode="conservative", n=8, family="ddpm", rule="det", generator="pcg64",
               desc="DiT-XL/2-shaped (random init), 4x32x32, DDPM 250, conservative n=N"),
    "c5": dict(net="sdxl", T=30, size=128, mode="aggressive", n=8, family="ddim", rule="det", generator="pcg64",
               desc="SDXL-shaped UNet (random init) bf16, 4x128x128, CFG batch 2, DDIM 30, aggressive n=N"),
}


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def _gemm_replay_ms(rec, dev, warm=3, reps=5):
    """ms per replay of a CUDA graph holding every recorded drs_gemm launch."""
    import torch
    from paper_2603_25872_b200 import _lib
    st = torch.cuda.Stream(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g, stream=st):
            for _, args in rec:
                _lib.check(_lib.lib().drs_gemm(_lib.ctypes.byref(args), st.cuda_stream), "drs_gemm")
        for _ in range(warm):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / reps


def _sampler_hbm(dev, peaks, log2d=25):
    """HBM roofline of the refine kernel (K3 skip chain, one DDPM noisy op, fp32
    eps: 8 x + 4 eps + 8 z + 8 out = 28 B/element) on a 2^25-element latent,
    where it is bandwidth-bound (the BASELINE latents are latency-bound)."""
    import torch

    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.transitions import ddpm_op_coeffs, launch_chain, make_op, ops_to_device
    D = 1 << log2d
    x = torch.randn(D, dtype=torch.float64, device=dev)
    eps = torch.randn(D, dtype=torch.float32, device=dev)
    z = torch.randn(D, dtype=torch.float64, device=dev)
    out = torch.empty(D, dtype=torch.float64, device=dev)
    c, noisy = ddpm_op_coeffs(P.default_schedule(50), 40, 2)
    od = ops_to_device([make_op(c, _lib.FAMILY_DDPM, noisy, x=x, eps=eps, z=z, out=out)], dev)
    st = torch.cuda.current_stream(dev)
    for _ in range(5):
        launch_chain(od, 1, D, stream=st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        launch_chain(od, 1, D, stream=st)
    e1.record(st)
    e1.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    gbs = 28 * D / (us * 1e-6) / 1e9
    del x, eps, z, out
    return {"kernel": "skip_chain_kernel (DDPM noisy op, fp32 eps)", "elements": D, "algo_bytes_per_element": 28,
            "avg_launch_us": us, "achieved": gbs, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
            "frac": gbs / peaks.get("hbm_gbs"), "inputs": "2^25-element fp64 latent (> L2), 5 warm + 20 timed launches"}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


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
            self._stop.wait(0.2)

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


# ------------------------------------------------------------- networks ----
def build_net(cfg, device, max_batch):
    """(network object or None, latent numel).  Random init, seed 0."""
    if cfg["net"] == "toy":
        return None, 4 * cfg["size"] ** 2
    if cfg["net"] == "dit":
        from paper_2603_25872_b200.dit import DiT, DiTConfig
        return DiT(DiTConfig(), device, seed=0, max_batch=max_batch), 4096
    from paper_2603_25872_b200.unet import UNet, sd15_config, sdxl_config
    ucfg = sd15_config() if cfg["net"] == "sd15" else sdxl_config()
    net = UNet(ucfg, device, seed=0, max_batch=max_batch)
    return net, net.latent_numel


def build_denoiser(cfg, net, D):
    import numpy as np
    import paper_2603_25872_b200 as P
    if cfg["net"] == "toy":
        m = np.zeros((2, D))
        m[0, 0], m[1, 0] = -2.0, 2.0
        return P.AnalyticEps(P.GaussianMixture(weights=[0.5, 0.5], means=m, variances=[1.0, 1.0]))
    return P.NetworkEps(net, (4, cfg["size"], cfg["size"]))


def evals_per_image(cfg, mode, n):
    from paper_2603_25872_b200.program import Mode, plan_blocks
    if mode == "sequential":
        return cfg["T"], cfg["T"]
    p = plan_blocks(cfg["T"], n, Mode(mode))
    return p.total_evals, p.total_rounds


# ------------------------------------------------------------ CPU legs ----
def _cpu_eval_fn(cfg):
    """eps callable for the oracle sampler on host cores: the analytic toy, or
    the same-architecture torch-CPU fp32 network (oracle/nets_ref.py)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import skipdiff_oracle as O
    if cfg["net"] == "toy":
        return O.toy_bimodal(4 * cfg["size"] ** 2)
    import torch
    import nets_ref
    net, _ = build_net(cfg, torch.device("cpu"), 1)
    S = cfg["size"]
    scale = 1000.0 / cfg["T"]

    def eps(ab, x, t):
        with torch.no_grad():
            xt = torch.from_numpy(np.asarray(x, dtype=np.float32)).reshape(1, 4, S, S)
            tt = torch.tensor([t * scale], dtype=torch.float32)
            if cfg["net"] == "dit":
                out = nets_ref.dit_ref(net.w, net.cfg, xt, tt)
            else:
                out = nets_ref.unet_ref(net, xt, tt)
            return out.reshape(-1).double().numpy()
    return eps


def cpu_sample(cfg, seconds, threads):
    """Reference algorithm on host cores (bounded).  Toy configs: whole images
    (oracle run_parallel / sample_*).  Network configs: a full image is minutes
    of CPU time, so the sample is `k` network evaluations timed and
    extrapolated to the sequential sampler's T evaluations per image."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import skipdiff_oracle as O
    torch.set_num_threads(threads)
    eps = _cpu_eval_fn(cfg)
    ab = O.default_alpha_bar(cfg["T"])
    D = 4 * cfg["size"] ** 2
    rule = ("det",) if cfg["rule"] == "det" else ("ddpm",)
    if cfg["net"] == "toy":
        def image(seed):
            x_T = O.derive_noise(seed, cfg["T"], O.INIT, D, cfg["generator"])
            O.run_parallel(ab, eps, x_T, cfg["n"], cfg["mode"], rule, seed, family=cfg["family"],
                           generator=cfg["generator"])
        image(99)
        times, t_end, seed = [], time.perf_counter() + seconds, 0
        while time.perf_counter() < t_end or len(times) < 3:
            t0 = time.perf_counter()
            image(seed)
            times.append((time.perf_counter() - t0) * 1e3)
            seed += 1
        return statistics.mean(times), f"{len(times)} whole images ({cfg['desc']}), oracle run_parallel"
    x = O.derive_noise(0, cfg["T"], O.INIT, D, cfg["generator"])
    eps(ab, x, cfg["T"])                               # warm-up
    times, t_end = [], time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 2:
        t0 = time.perf_counter()
        eps(ab, x, cfg["T"] - len(times))
        times.append((time.perf_counter() - t0) * 1e3)
    per_eval = statistics.mean(times)
    return per_eval * cfg["T"], (f"{len(times)} torch-CPU fp32 network evaluations ({per_eval:.0f} ms each, "
                                 f"{threads} threads) x T={cfg['T']} evals of the sequential sampler "
                                 f"(extrapolated; sampler arithmetic is negligible next to it)")


def run_reference_arm(a, cfg, rank):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    seconds = max(5.0, min(60.0, 20.0 * a.steps / 5))
    v, sample = cpu_sample(cfg, seconds, threads)
    line = {"impl": "reference", "metric": "ms/image sampling latency", "value": v, "unit": "ms/image",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if cfg["net"] != "toy" else "f64",
            "data": "synthetic", "config": {"workload": a.config, "desc": cfg["desc"]},
            "cpu_baseline": {"value": v, "unit": "ms/image", "cores": threads if cfg["net"] != "toy" else 1,
                             "kind": "port", "sample": sample},
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

    import torch
    import torch.distributed as dist

    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200 import _lib, netops
    from paper_2603_25872_b200.engine import Comm
    from paper_2603_25872_b200.pipeline import Sampler

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = Comm(rank, world)
    net_cfg = cfg["net"] != "toy"
    if world == 1:
        mode, n = ("sequential", 1) if net_cfg else (cfg["mode"], cfg["n"])
    else:
        mode, n = cfg["mode"], world
    s = P.default_schedule(cfg["T"])
    net, D = build_net(cfg, dev, max_batch=max(1, cfg["n"] if world == 1 else 1))
    den = build_denoiser(cfg, net, D)
    rule = P.VarianceRule.deterministic() if cfg["rule"] == "det" else P.VarianceRule.ddpm_induced()
    sampler = Sampler(s, den, D, mode=mode, devices=n, rule=rule, family=cfg["family"],
                      generator=cfg["generator"], comm=comm, device=dev)
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
    l0 = _lib.LAUNCHES[0]
    with ClockSampler(local) as clk:
        per_image = timed_images(sampler, a.steps, 0)
    graph_note = "graph replays (no host launches)" if sampler.use_graph else "eager"
    t_img = torch.tensor([statistics.mean(per_image)], device=dev)
    if world > 1:
        dist.all_reduce(t_img, op=dist.ReduceOp.MAX)
    value = float(t_img.item())
    sampler.run.check_err()

    # launches per image: count libdrs entry points of one eager image
    l0 = _lib.LAUNCHES[0]
    sampler.stage(4242)
    sampler.run.enqueue()
    torch.cuda.synchronize(dev)
    launches = _lib.LAUNCHES[0] - l0
    barrier()

    # end to end through the public pipeline call: x_T from pinned host memory,
    # final sample back to pinned host memory, synchronised, wall clock
    x_hosts = [P.derive_noise(P.RngStream(50_000 + i, cfg["generator"]), cfg["T"], P.Role.INIT, D,
                              device=dev).cpu().pin_memory() for i in range(a.steps)]
    out_host = torch.empty(D, dtype=torch.float64).pin_memory()
    sampler(49_999, x_T=x_hosts[0], out=out_host)
    barrier()
    e2e = []
    for i in range(a.steps):
        barrier()
        t0 = time.perf_counter()
        sampler(50_000 + i, x_T=x_hosts[i], out=out_host)
        e2e.append((time.perf_counter() - t0) * 1e3)
    t_e2e = torch.tensor([statistics.mean(e2e)], device=dev)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)

    # roofline of the dominant kernel: per-launch CUDA events over one eager image
    peaks = _peaks()
    timers = []
    netops.TIMERS = [] if net_cfg else None
    netops.GEMM_RECORD = [] if net_cfg else None
    sampler.stage(2000)
    torch.cuda.synchronize(dev)
    sampler.run.enqueue(timers=timers)
    torch.cuda.synchronize(dev)
    classes = {}
    for label, nbytes, e0, e1 in timers:
        c = classes.setdefault(label, {"ms": 0.0, "bytes": 0, "launches": 0})
        c["ms"] += e0.elapsed_time(e1)
        c["bytes"] += nbytes
        c["launches"] += 1
    if net_cfg:
        gt = netops.TIMERS
        netops.TIMERS = None
        rec = netops.GEMM_RECORD
        netops.GEMM_RECORD = None
        g_ms_events = sum(e0.elapsed_time(e1) for _, e0, e1, _ in gt)
        g_flops = sum(f for f, _ in rec)
        # the image's GEMM launches (same arguments and buffers) replayed back to
        # back from one CUDA graph: device time of the tensor-core kernels alone
        g_ms = _gemm_replay_ms(rec, dev)
        achieved = g_flops / (g_ms * 1e-3) / 1e12
        peak = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops")
        ev_ms = classes.get("eval_net", {"ms": 0.0})["ms"]
        roofline = {"bound": "tensor", "kernel": "gemm_bf16_tc_kernel (tcgen05.mma, TMA, TMEM)",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": None, "gemm_ms_per_image": g_ms, "gemm_tflop_per_image": g_flops / 1e12,
                    "gemm_ms_per_image_eager_events": g_ms_events,
                    "method": "all GEMM launches of one image (recorded drs_gemm arguments) replayed from one "
                              "CUDA graph, 3 warm + 5 timed replays, CUDA events on the replay stream",
                    "gemm_launches_per_image": len(gt), "gemm_share_of_eval_time": g_ms / ev_ms if ev_ms else None,
                    "network_tflop_per_eval": (net.flops or 0) / 1e12 if cfg["net"] != "dit" else
                    net.cfg.flops_per_image() / 1e12,
                    "peak_source": "fallback" if peaks.get("_fallback") else "MEASURED_PEAKS.json bf16_tflops_sustained"}
    else:
        kernels = {k: v for k, v in classes.items() if k != "gather"}
        top = max(kernels, key=lambda k: kernels[k]["ms"])
        avg_ms = kernels[top]["ms"] / kernels[top]["launches"]
        algo = kernels[top]["bytes"] / kernels[top]["launches"]
        achieved = algo / (avg_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peaks.get("hbm_gbs"),
                    "unit": "GB/s", "frac": achieved / peaks.get("hbm_gbs"), "traffic": None,
                    "algo_bytes_per_launch": algo, "avg_launch_us": avg_ms * 1e3,
                    "peak_source": "fallback" if peaks.get("_fallback") else "MEASURED_PEAKS.json hbm_gbs"}
    prof = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(prof):
        tr = json.load(open(prof))
        # the capture is of one network's GEMMs (tools/gemm_traffic.py): only that config reports it
        if not net_cfg or tr.get("_detail", {}).get("net", "sd15") == cfg["net"]:
            roofline["traffic"] = tr.get(roofline["kernel"])
            if roofline["traffic"] is not None and net_cfg:
                roofline["traffic_detail"] = tr.get("_detail")

    if world == 1 and rank == 0:
        roofline["sampler_hbm"] = _sampler_hbm(dev, peaks)

    # draft-and-refine on this one GPU (logical devices batched per round), for context
    drf = {"T": cfg["T"], "mode_timed": mode, "devices": n}
    if world == 1 and net_cfg and rank == 0:
        par = Sampler(s, den, D, mode=cfg["mode"], devices=cfg["n"], rule=rule, family=cfg["family"],
                      generator=cfg["generator"], device=dev)
        par.stage(7)
        par.launch()
        torch.cuda.synchronize(dev)
        pms = statistics.mean(timed_images(par, 2, 0, False))
        ev, rounds = evals_per_image(cfg, cfg["mode"], cfg["n"])
        drf.update({"sequential_1gpu_ms": value,
                    "batched_drafts_1gpu": {"mode": cfg["mode"], "n": cfg["n"], "ms_per_image": pms,
                                            "rounds": rounds, "evals": ev, "speedup": value / pms}})
        for nn in (2, 4, 8):
            ev2, r2 = evals_per_image(cfg, cfg["mode"], nn)
            drf[f"ideal_n{nn}"] = {"round_law_ms": value * r2 / cfg["T"], "one_over_n_ms": value / nn,
                                   "two_over_n_plus_1_ms": value * 2 / (nn + 1), "rounds": r2}
    elif world > 1:
        ev, rounds = evals_per_image(cfg, mode, n)
        drf.update({"rounds": rounds, "evals": ev})

    if rank != 0:
        dist.destroy_process_group()
        return
    line = {
        "metric": "ms/image sampling latency", "value": value, "unit": "ms/image", "n_gpus": world,
        "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": value, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if net_cfg else "f64", "data": "synthetic",
        "config": {"workload": a.config, "desc": cfg["desc"], "T": cfg["T"], "latent": f"4x{cfg['size']}x{cfg['size']}",
                   "mode": mode, "devices": n, "family": cfg["family"], "noise": cfg["generator"], "batch": 1,
                   "state": "fp64 sampler state, fp32 eps" if net_cfg else "fp64",
                   "weights": "random init N(0, 0.02), seed 0" if net_cfg else "analytic",
                   "l2": "flushed between timed images (256 MB memset outside the events)", "launch": graph_note},
        "e2e": {"value": float(t_e2e.item()), "unit": "ms/image", "h2d_bytes_per_step": D * 8 + 16,
                "d2h_bytes_per_step": D * 8,
                "how": "Sampler(seed, x_T=pinned host, out=pinned host): H2D x_T, graph replay, D2H x_0, sync"},
        "gpu_launches": launches * a.steps,
        "roofline": roofline,
        "kernels": {k: {"ms_per_image": v["ms"], "launches_per_image": v["launches"]} for k, v in classes.items()},
        "clocks": clk.summary(),
        "drf": drf,
    }
    if not a.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        v, sample = cpu_sample(cfg, a.cpu_seconds, threads)
        line["cpu_baseline"] = {"value": v, "unit": "ms/image", "cores": threads if net_cfg else 1, "kind": "port",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

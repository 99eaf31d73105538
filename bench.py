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
    ap.add_argument("--ref-seconds", type=float, default=150.0,
                    help="reference arm: whole images timed while they fit this budget (>= 1 image)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nccl-one-rank", action="store_true",
                    help="N=1 diagnostic: the N>1 code path (NCCL communicator, per-round eps all-gathers "
                         "captured in the image graph, drf ratios) on a one-rank communicator")
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


class _Budget(Exception):
    """Raised inside the eps callable to stop a bounded CPU sample at a step boundary."""


def _oracle_image(cfg, eps, seed, mode, n, marks=None, limit=None):
    """One image of the restated reference pipeline (cli._run_once, cli.py:43-67):
    x_T = INIT noise of the seed, then the configured sampler, on host cores.
    `marks` collects a perf_counter stamp at the start of every eps evaluation;
    `limit` stops the image (raising _Budget) before evaluation limit+1."""
    import skipdiff_oracle as O
    T, D = cfg["T"], 4 * cfg["size"] ** 2
    ab = O.default_alpha_bar(T)
    rule = ("det",) if cfg["rule"] == "det" else ("ddpm",)

    def timed(ab_, x, t):
        if marks is not None:
            marks.append(time.perf_counter())
            if limit is not None and len(marks) > limit:
                raise _Budget()
        return eps(ab_, x, t)
    x_T = O.derive_noise(seed, T, O.INIT, D, cfg["generator"])
    if mode == "sequential":
        if cfg["family"] == "ddpm":
            return O.sample_ddpm(ab, timed, x_T, seed, cfg["generator"])
        return O.sample_ddim(ab, timed, x_T, rule, seed, cfg["generator"])
    return O.run_parallel(ab, timed, x_T, n, mode, rule, seed, family=cfg["family"],
                          generator=cfg["generator"])[0]


def cpu_steps(cfg, mode, n, threads, seconds):
    """Bounded CPU baseline: consecutive steps of ONE image of the oracle
    sampler (each step = one eps evaluation + its update; the network configs
    run the same-architecture torch-CPU fp32 net), stopped at a step boundary
    after `seconds`; ms/image = mean step time x evaluations per image."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    torch.set_num_threads(threads)
    eps = _cpu_eval_fn(cfg)
    evals, _ = evals_per_image(cfg, mode, n)
    warm = []
    try:                                                # warm-up: one evaluation
        _oracle_image(cfg, eps, 99, mode, n, warm, 1)
    except _Budget:
        pass
    marks, t_end = [], time.perf_counter() + seconds

    class _Deadline(list):
        def append(self, v):
            super().append(v)
            if v > t_end and len(self) >= 3:
                raise _Budget()
    marks = _Deadline()
    try:
        _oracle_image(cfg, eps, 0, mode, n, marks, None)
        marks.append(time.perf_counter())               # whole image finished inside the budget
    except _Budget:
        pass
    steps = [b - a for a, b in zip(marks, marks[1:])]
    per_step = statistics.mean(steps) * 1e3
    return per_step * evals, (f"{len(steps)} consecutive sampler steps (eps evaluation + update) of one "
                              f"{mode} image, oracle sampler with the {_eps_desc(cfg)} on {_threads_desc(cfg, threads)} "
                              f"({per_step:.0f} ms/step) x {evals} evaluations per image"), len(steps), per_step


def _threads_desc(cfg, threads):
    return "1 host thread (numpy)" if cfg["net"] == "toy" else f"{threads} host threads"


def _eps_desc(cfg):
    return "analytic GM eps" if cfg["net"] == "toy" else "torch-CPU fp32 network (same weights)"


def cpu_images(cfg, mode, n, threads, budget_s, max_images):
    """Reference arm: WHOLE images of the oracle pipeline (x_T noise + sampler)
    on host cores, timed image by image, as many as fit `budget_s` (at least
    one).  If one image is projected (from a warm-up evaluation) to exceed the
    budget, a bounded run of consecutive steps is extrapolated instead and the
    line says so.  Returns (per-image ms list, sample text, whole-images flag)."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    torch.set_num_threads(threads)
    eps = _cpu_eval_fn(cfg)
    evals, _ = evals_per_image(cfg, mode, n)
    warm = []
    t0 = time.perf_counter()
    try:
        _oracle_image(cfg, eps, 99, mode, n, warm, 2)
    except _Budget:
        pass
    per_eval = (time.perf_counter() - t0) / 2
    if per_eval * evals > budget_s:
        v, sample, n_steps, per_step = cpu_steps(cfg, mode, n, threads, min(budget_s, 60.0))
        return [v], sample + " (one image exceeds the time budget: extrapolated)", (n_steps, per_step)
    times, t_end = [], time.perf_counter() + budget_s
    while len(times) < max_images and (not times or time.perf_counter() + statistics.mean(times) / 1e3 < t_end):
        t0 = time.perf_counter()
        _oracle_image(cfg, eps, len(times), mode, n)
        times.append((time.perf_counter() - t0) * 1e3)
    return times, (f"{len(times)} whole image(s), x_T -> x_0 ({evals} evaluations each), oracle {mode} sampler "
                   f"with the {_eps_desc(cfg)} on {_threads_desc(cfg, threads)}"
                   + ("; the reference's thread pool shares these cores, so parallel-mode evaluations run "
                      "one after another" if mode != "sequential" else "")), None


def workload_config(cfg, name, mode, n):
    """The `config` object both arms print (same keys and values)."""
    net_cfg = cfg["net"] != "toy"
    return {"workload": name, "desc": cfg["desc"], "T": cfg["T"], "latent": f"4x{cfg['size']}x{cfg['size']}",
            "mode": mode, "devices": n, "family": cfg["family"], "noise": cfg["generator"], "batch": 1,
            "state": "fp64 sampler state" + (", fp32 eps" if net_cfg else ""),
            "weights": "random init N(0, 0.02), seed 0" if net_cfg else "analytic",
            "l2": "GPU arm: flushed between timed images (256 MB memset outside the events); CPU arm: n/a"}


def arm_modes(cfg, world):
    """(mode, n) timed at this world size: N = 1 runs the 1-GPU sequential sampler
    for the network configs (T1 of the metric), N > 1 the configured mode with n = N."""
    if world == 1:
        return ("sequential", 1) if cfg["net"] != "toy" else (cfg["mode"], cfg["n"])
    return cfg["mode"], world


def run_reference_arm(a, cfg, rank, world):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    mode, n = arm_modes(cfg, world)
    times, sample, extrap = cpu_images(cfg, mode, n, threads, a.ref_seconds, max(1, a.steps))
    v = statistics.mean(times)
    whole = extrap is None
    # steps / ms_per_step describe what was actually timed: whole images, or (when one
    # image exceeds the budget) consecutive sampler steps, each one eps evaluation + update
    n_timed, ms_step = (len(times), v) if whole else extrap
    cores = threads if cfg["net"] != "toy" else 1
    line = {"impl": "reference", "metric": "ms/image sampling latency", "value": v, "unit": "ms/image",
            "n_gpus": a.gpus, "steps": n_timed, "warmup": a.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if cfg["net"] != "toy" else "f64", "data": "synthetic",
            "config": workload_config(cfg, a.config, mode, n),
            "steps_note": (f"steps = whole images timed ({len(times)}; --steps {a.steps} requested): one image "
                           f"is {v / 1e3:.0f} s of CPU work, so the arm times as many as fit "
                           f"--ref-seconds {a.ref_seconds:.0f}" if whole else
                           f"one image exceeds --ref-seconds: steps = {n_timed} consecutive sampler steps timed "
                           f"(ms_per_step per sampler step), value = ms/step x evaluations per image"),
            "precision_note": ("reference arm computes eps with the fp32 torch-CPU network; the GPU arm with the "
                               "bf16 tcgen05 network (fp32 accumulate, fp64 sampler state) -- per-step latent "
                               "tolerance in DESIGN.md 3a" if cfg["net"] != "toy" else "both arms fp64"),
            "cpu_baseline": {"value": v, "unit": "ms/image", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "ms/image", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU leg -----
def main():
    a = _args()
    cfg = CONFIGS[a.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if a.impl == "reference":
        run_reference_arm(a, cfg, rank, world)
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
    multi = world > 1 or a.nccl_one_rank
    if multi:
        # NCCL's own init log (communicator ranks, NVLS/NVLink transport) goes to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        else:
            dist.init_process_group("nccl", device_id=dev)
        comm = Comm(rank, world)
    net_cfg = cfg["net"] != "toy"
    mode, n = arm_modes(cfg, world)
    if a.nccl_one_rank:
        mode, n = cfg["mode"], cfg["n"]
    s = P.default_schedule(cfg["T"])
    net, D = build_net(cfg, dev, max_batch=max(1, cfg["n"] if world == 1 else 1))
    den = build_denoiser(cfg, net, D)
    rule = P.VarianceRule.deterministic() if cfg["rule"] == "det" else P.VarianceRule.ddpm_induced()
    sampler = Sampler(s, den, D, mode=mode, devices=n, rule=rule, family=cfg["family"],
                      generator=cfg["generator"], comm=comm, device=dev, exchange=multi)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2

    def barrier():
        if multi:
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
    graph_note = (f"graph replays, {sampler.run.graph_mode} (no host launches)" if sampler.use_graph
                  else "eager")
    t_img = torch.tensor([statistics.mean(per_image)], device=dev)
    if multi:
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
    if multi:
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
    if world == 1 and net_cfg and rank == 0 and not multi:
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
    elif multi:
        # T1 on this rank's GPU (the 1-GPU sequential sampler, no communicator), so the
        # line carries the measured / round-law and measured / 2/(n+1) ratios itself
        ev, rounds = evals_per_image(cfg, mode, n)
        seq = Sampler(s, den, D, mode="sequential" if net_cfg else cfg["mode"], devices=1 if net_cfg else cfg["n"],
                      rule=rule, family=cfg["family"], generator=cfg["generator"], device=dev)
        seq.stage(7)
        seq.launch()
        torch.cuda.synchronize(dev)
        t1 = torch.tensor([statistics.mean(timed_images(seq, 3, 0, False))], device=dev)
        dist.all_reduce(t1, op=dist.ReduceOp.MAX)
        t1 = float(t1.item())
        g = classes.get("gather", {"ms": 0.0, "launches": 0})
        round_law = t1 * rounds / cfg["T"]
        drf.update({"rounds": rounds, "evals": ev, "t1_sequential_ms": t1,
                    "gather_us_per_round": g["ms"] * 1e3 / max(1, g["launches"]),
                    "gathers_per_image": g["launches"],
                    "exchange": sampler.run.graph_mode,
                    "round_law_ms": round_law, "measured_over_round_law": value / round_law,
                    "one_over_n_ms": t1 / n, "measured_over_one_over_n": value / (t1 / n),
                    "two_over_n_plus_1_ms": t1 * 2 / (n + 1),
                    "measured_over_two_over_n_plus_1": value / (t1 * 2 / (n + 1)),
                    "speedup_vs_t1": t1 / value})

    if rank != 0:
        dist.destroy_process_group()
        return
    line = {
        "metric": "ms/image sampling latency", "value": value, "unit": "ms/image", "n_gpus": world,
        "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": value, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if net_cfg else "f64", "data": "synthetic",
        "config": workload_config(cfg, a.config, mode, n),
        "launch": graph_note,
        "precision_note": ("bf16 tcgen05 network (fp32 accumulate), fp32 eps, fp64 sampler state; the reference "
                           "arm uses the fp32 torch-CPU network -- per-step tolerance in DESIGN.md 3a")
        if net_cfg else "fp64",
        "e2e": {"value": float(t_e2e.item()), "unit": "ms/image", "h2d_bytes_per_step": D * 8 + 16,
                "d2h_bytes_per_step": D * 8,
                "how": "Sampler(seed, x_T=pinned host, out=pinned host): H2D x_T, graph replay, D2H x_0, sync"},
        "gpu_launches": launches * a.steps,
        "roofline": roofline,
        "kernels": {k: {"ms_per_image": v["ms"], "launches_per_image": v["launches"]} for k, v in classes.items()},
        "clocks": clk.summary(),
        "drf": drf,
    }
    if not a.no_cpu_baseline and world == 1:      # rank 0 at N = 1 only
        threads = len(os.sched_getaffinity(0))
        if net_cfg:
            v, sample, _, _ = cpu_steps(cfg, mode, n, threads, a.cpu_seconds)
        else:
            times, sample, _ = cpu_images(cfg, mode, n, threads, a.cpu_seconds, 1000)
            v = statistics.mean(times)
        line["cpu_baseline"] = {"value": v, "unit": "ms/image", "cores": threads if net_cfg else 1, "kind": "port",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Draft-and-refine parallel schedulers (skipdiff parallel.py) on B200.

Same entry points and semantics as the reference:
  run_aggressive   one parallel round per k steps, T+1 evals, cached anchor eps
  run_conservative stand-alone anchor eval + one parallel round per k+1 steps
  execute_round    one round of concurrent evals, results ordered by task

"Devices" are logical: with `comm=None` every round's k evaluations run as
one batched launch on this GPU; with `comm=Comm(rank, world)` (one process
per GPU, torch.distributed/NCCL) rank r evaluates tasks i with i % world == r
and the round's eps rows are all-gathered; drafts and refines are replayed
redundantly and bit-identically on every rank, so nothing else crosses
NVLink.  `workers` / `submit_order_seed` / SKIPDIFF_MAX_WORKERS are accepted
for drop-in compatibility; outputs never depend on them (parallel.py:13-16).
"""

import os

import torch

from . import _lib
from .denoiser import AnalyticEps, StateIndependent, apply_perturbations, evaluate, latency_of, perturb_scales
from .engine import Comm, unwrap
from .errors import InvalidPlanParams, WorkerFailure
from .program import BlockPlan, Mode, build_parallel, plan_blocks
from .rng import RngStream
from .runner import RoundReport, Trajectory, execute, get_run, resolve_device
from .transitions import VarianceRule

WORKER_CAP_ENV = "SKIPDIFF_MAX_WORKERS"   # parallel.py:41


def _worker_cap(requested: int) -> int:
    cap = os.environ.get(WORKER_CAP_ENV)
    if cap:
        return max(1, min(requested, int(cap)))
    return requested


def _numel(x):
    """Elements of an array-like x_T (tensor, ndarray, nested list: np.asarray semantics)."""
    if not hasattr(x, "shape"):
        import numpy as np
        x = np.asarray(x, dtype=float)
    n = 1
    for d in x.shape:
        n *= int(d)
    return n


def execute_round(d, s, tasks: list, devices: int, *, anchor_t: int, pool=None, clock=None,
                  submit_order=None):
    """Evaluate all (x, t) tasks as one concurrent round; eps ordered by task
    index; wall = max over tasks + dispatch overhead (parallel.py:98-184).
    A failing task does not stop the others; the first error is re-raised as
    WorkerFailure after the round drains."""
    if len(tasks) > devices:
        raise InvalidPlanParams(f"{len(tasks)} tasks exceed {devices} devices")
    model = latency_of(d)
    overhead = model.dispatch_overhead_ms if model else 0.0
    if clock is not None:
        from .denoiser import VirtualClock
        results, spans = [], []
        for i, (x, t) in enumerate(tasks):
            sub = VirtualClock()
            results.append(evaluate(d, s, x, t, sub))
            spans.append((i, 0.0, sub.elapsed_ms))
        round_ms = max((ms for _, _, ms in spans), default=0.0) + overhead
        clock.charge(round_ms)
        return results, RoundReport(anchor_t, len(tasks), round_ms, spans)

    core, eval_ms, counters = unwrap(d)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if overhead > 0:
        _lib.check(_lib.lib().drs_spin(overhead * 1000.0, 1, _lib.stream_ptr()), "drs_spin")
    if eval_ms > 0 and tasks:          # all tasks' latency occupies the GPU concurrently
        _lib.check(_lib.lib().drs_spin(eval_ms * 1000.0, len(tasks), _lib.stream_ptr()), "drs_spin")
    results, error = [None] * len(tasks), None
    scales = perturb_scales(d)
    for i, (x, t) in enumerate(tasks):
        try:
            results[i] = evaluate(core, s, x, t)
            if scales:          # the perturbation chain runs on fp64 rows (network eps is fp32)
                results[i] = apply_perturbations(scales, torch.as_tensor(x, dtype=torch.float64,
                                                                         device=results[i].device),
                                                 t, results[i].to(torch.float64).contiguous().clone())
        except Exception as exc:      # drain the round before raising (parallel.py:168-179)
            if error is None:
                error = exc
    for c in counters:
        c.count += len(tasks)
    e1.record()
    e1.synchronize()
    if error is not None:
        raise WorkerFailure(str(error)) from error
    ms = e0.elapsed_time(e1)
    return results, RoundReport(anchor_t, len(tasks), ms, [(i, 0.0, ms) for i in range(len(tasks))])


def _check_workers(workers, submit_order_seed):
    """`workers or devices` sizes the reference's pool (parallel.py:269): None and
    0 both mean one worker per device; negative counts are rejected."""
    if workers is not None and workers < 0:
        raise InvalidPlanParams(f"workers must be >= 0, got {workers}")


def _run(mode: Mode, s, d, x_T, devices, rule, stream, clock, workers, submit_order_seed,
         recompute_anchor_eps, update_family, comm):
    if update_family not in ("ddim", "ddpm"):
        raise ValueError(f"unknown update family: {update_family!r}")
    _check_workers(workers, submit_order_seed)
    plan = plan_blocks(s.T, devices, mode)
    world = comm.size if comm else 1
    rank = comm.rank if comm else 0
    dev = resolve_device(x_T)
    run = get_run(("par", mode, s.T, devices, rule, update_family, recompute_anchor_eps, world, rank),
                  lambda: build_parallel(s, plan, rule, update_family, recompute_anchor_eps, world, rank),
                  s, d, _numel(x_T), dev, stream.generator, comm)
    return execute(run, x_T, stream.seed, clock)


def run_aggressive(s, d, x_T, devices: int, rule: VarianceRule, stream: RngStream, *, clock=None,
                   workers=None, submit_order_seed=None, recompute_anchor_eps: bool = False,
                   update_family: str = "ddim", comm: Comm | None = None):
    """Aggressive draft-and-refine run (parallel.py:203-227)."""
    return _run(Mode.AGGRESSIVE, s, d, x_T, devices, rule, stream, clock, workers, submit_order_seed,
                recompute_anchor_eps, update_family, comm)


def run_conservative(s, d, x_T, devices: int, rule: VarianceRule, stream: RngStream, *, clock=None,
                     workers=None, submit_order_seed=None, update_family: str = "ddim",
                     comm: Comm | None = None):
    """Conservative run: stand-alone anchor eval then one round per block (parallel.py:230-247)."""
    return _run(Mode.CONSERVATIVE, s, d, x_T, devices, rule, stream, clock, workers, submit_order_seed,
                False, update_family, comm)


def run_parallel_euler(g, gm, x_init, devices: int, mode: Mode, *, workers=None, comm: Comm | None = None):
    """Euler-family variant of the two schedulers on a sigma grid with the
    analytic velocity oracle (parallel.py:324-381).  Deterministic; timesteps
    count remaining grid intervals; velocity tasks at sigma = 0 are dropped.
    Same device program machinery as run_aggressive / run_conservative
    (drafts from the anchor, one batched or rank-sharded velocity round,
    fused refine chain; with `comm`, rank r evaluates tasks i % world == r)."""
    from .denoiser import euler_velocity_core
    _check_workers(workers, None)
    plan = plan_blocks(g.N, devices, mode)
    world = comm.size if comm else 1
    rank = comm.rank if comm else 0
    dev = resolve_device(x_init)
    core = euler_velocity_core(gm, g)
    run = get_run(("par", mode, "euler", g.N, devices, world, rank),
                  lambda: build_parallel(g, plan, None, "euler", False, world, rank),
                  g, core, _numel(x_init), dev, "pcg64", comm)
    return execute(run, x_init, 0, None)


__all__ = ["BlockPlan", "Comm", "Mode", "RoundReport", "Trajectory", "WORKER_CAP_ENV", "execute_round",
           "plan_blocks", "run_aggressive", "run_conservative", "run_parallel_euler",
           "AnalyticEps", "StateIndependent"]

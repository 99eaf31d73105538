"""Output formats of the reference (skipdiff cli.py:69-153), so
B200 runs are diffable with reference output file-for-file:

  samples CSV   seed,dim0..dim{D-1}; values written with repr(float)
  rounds CSV    round,anchor_t,parallel_evals,round_wall_ms (%.3f)
  JSON report   {"config", "totals": {evals, rounds, wall_ms}, "rounds": [...],
                 "artifacts": {"samples", "rounds"}}
  bench CSV     mode,devices,median_ms,speedup,theory_bound

`collect_runs` replays cli.py:72-81's accounting over seeds seed..seed+n-1
with any run function returning (Trajectory, [RoundReport]) -- the device
samplers of this package -- and `write_outputs` writes the three artifacts
with cli.py's no-partial-outputs-on-failure rule.  (The reference's config
parser and command line are outside the hot-path scope; callers pass the
same values directly.)
"""

import csv
import io
import json
import os
import statistics

import numpy as np


def _host_row(x):
    if hasattr(x, "detach"):
        x = x.detach().reshape(-1).cpu().numpy()
    return np.atleast_1d(np.asarray(x, dtype=float)).reshape(-1)


def collect_runs(run_once, seed: int, samples: int):
    """[(seed_i, final)], [RoundReport], totals for seeds seed..seed+samples-1
    (cli.py:72-81)."""
    finals, reports = [], []
    totals = {"evals": 0, "rounds": 0, "wall_ms": 0.0}
    for i in range(samples):
        traj, reps = run_once(seed + i)
        finals.append((seed + i, traj.final))
        reports.extend(reps)
        totals["evals"] += traj.eval_count
        totals["rounds"] += len(reps)
        totals["wall_ms"] += traj.wall_ms
    return finals, reports, totals


def samples_csv(finals, dim: int) -> str:
    """cli.py:84-90: header seed,dim0.., one row per seed, repr(float) values."""
    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    w.writerow(["seed"] + [f"dim{j}" for j in range(dim)])
    for seed, x in finals:
        w.writerow([seed] + [repr(float(v)) for v in _host_row(x)])
    return buf.getvalue()


def rounds_csv(reports) -> str:
    """cli.py:91-97."""
    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    w.writerow(["round", "anchor_t", "parallel_evals", "round_wall_ms"])
    for n, r in enumerate(reports):
        w.writerow([n, r.anchor_t, r.parallel_evals, f"{r.round_wall_ms:.3f}"])
    return buf.getvalue()


def report_dict(config: dict, totals: dict, reports, out_samples=None, out_rounds=None) -> dict:
    """cli.py:98-106."""
    return {
        "config": config,
        "totals": totals,
        "rounds": [{"anchor_t": r.anchor_t, "parallel_evals": r.parallel_evals, "round_wall_ms": r.round_wall_ms}
                   for r in reports],
        "artifacts": {"samples": out_samples, "rounds": out_rounds},
    }


def write_outputs(finals, reports, totals, dim: int, *, config=None, out_samples=None, out_rounds=None,
                  out_report=None):
    """Write the requested artifacts; on any failure remove the ones already
    written (cli.py:113-119).  Returns the stdout summary dict of cli.py:111."""
    written = []
    try:
        if out_samples:
            with open(out_samples, "w", newline="") as fh:
                written.append(out_samples)
                fh.write(samples_csv(finals, dim))
        if out_rounds:
            with open(out_rounds, "w", newline="") as fh:
                written.append(out_rounds)
                fh.write(rounds_csv(reports))
        if out_report:
            with open(out_report, "w") as fh:
                written.append(out_report)
                json.dump(report_dict(config or {}, totals, reports, out_samples, out_rounds), fh, indent=2)
        return {"totals": totals, "samples": len(finals)}
    except Exception:
        for path in written:
            try:
                os.remove(path)
            except OSError:
                pass
        raise


def bench_rows(median_wall, modes, devices_list):
    """cli.py:133-141: the sequential row, then per (mode, devices) the median
    wall, speedup vs sequential and the theory bound (seq/n aggressive,
    2 seq/(n+1) conservative).  median_wall(mode, devices) -> ms."""
    seq_ms = median_wall("sequential", 1)
    rows = [("sequential", 1, seq_ms, 1.0, seq_ms)]
    for mode in modes:
        for devices in devices_list:
            ms = median_wall(mode, devices)
            bound = seq_ms / devices if mode == "aggressive" else seq_ms * 2 / (devices + 1)
            rows.append((mode, devices, ms, seq_ms / ms, bound))
    return rows


def median_of(fn, repeats: int):
    """cli.py:125-131: one warm-up, then the median of `repeats` runs."""
    fn()
    return statistics.median([fn() for _ in range(repeats)])


def bench_csv(rows) -> str:
    """cli.py:143-148."""
    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    w.writerow(["mode", "devices", "median_ms", "speedup", "theory_bound"])
    for mode, devices, ms, speedup, bound in rows:
        w.writerow([mode, devices, f"{ms:.3f}", f"{speedup:.4f}", f"{bound:.3f}"])
    return buf.getvalue()


__all__ = ["bench_csv", "bench_rows", "collect_runs", "median_of", "report_dict", "rounds_csv", "samples_csv",
           "write_outputs"]

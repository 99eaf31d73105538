"""Host-numpy face of the drop-in (the reference's return types).

The reference package `skipdiff` returns numpy arrays everywhere: noise
(rng.py:27-33), transitions (transitions.py:105-188), eps (denoiser.py:73-145,
234-267), trajectories (sequential.py:18-32, parallel.py:203-381).  This
module wraps this package's public API so that every array that comes back
is a host fp64 ndarray, while every computation still runs on the B200 through
libdrs.so (inputs may be numpy arrays, lists or tensors; they are staged to
the GPU, results are copied back with one D2H per call).  `dropin/skipdiff`
re-exports it under the reference's module names, so the reference's own test
suite (pkg/tests/) runs unmodified against the GPU path
(tools/run_reference_suite.sh, profiles/r2_reference_suite.txt).

There is no CPU fallback: without CUDA every call raises like the rest of the
package.
"""

import functools

import numpy as np

from . import denoiser as _den
from . import metrics as _met
from . import parallel as _par
from . import rng as _rng
from . import sequential as _seq
from . import transitions as _tr
from .denoiser import (AnalyticEps, Counting, GaussianMixture, Latency, LatencyModel, NetworkEps, Perturbed,
                       StateIndependent, VirtualClock, standard_normal_mixture)
from .errors import *  # noqa: F401,F403
from .metrics import SampleSet, mmd_gaussian, mmd_permutation_threshold, sliced_w2
from .parallel import WORKER_CAP_ENV, BlockPlan, Mode, RoundReport, plan_blocks
from .rng import RngStream, Role
from .runner import Trajectory
from .schedule import (NoiseSchedule, ScheduleKind, SigmaGrid, alpha_at, build_cosine, build_linear_beta,
                       build_sigma_grid, default_schedule)
from .transitions import SkipCoeffs, SkipPosterior, VarianceKind, VarianceRule, ddim_skip_coeffs


def to_host(x):
    """CUDA tensor -> host ndarray (fp64/fp32 kept); containers converted element-wise."""
    try:
        import torch
    except ImportError:       # pragma: no cover
        torch = None
    if torch is not None and isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    if isinstance(x, list):
        return [to_host(v) for v in x]
    if isinstance(x, tuple):
        return tuple(to_host(v) for v in x)
    return x


def host_trajectory(tr):
    """A Trajectory whose states are host ndarrays (one D2H of the whole buffer)."""
    if not tr.states:
        return tr
    import torch
    xs = [x for _, x in tr.states]
    if isinstance(xs[0], torch.Tensor):
        base = torch.stack([x.reshape(-1) for x in xs]).cpu().numpy()
        states = [(t, base[j].reshape(tuple(x.shape))) for j, ((t, _), x) in enumerate(zip(tr.states, xs))]
    else:
        states = list(tr.states)
    return Trajectory(states=states, eval_count=tr.eval_count, wall_ms=tr.wall_ms, device_ms=tr.device_ms)


def _returns_host(fn):
    @functools.wraps(fn)
    def wrap(*a, **k):
        return to_host(fn(*a, **k))
    return wrap


def _returns_traj(fn):
    @functools.wraps(fn)
    def wrap(*a, **k):
        out = fn(*a, **k)
        if isinstance(out, tuple):
            return (host_trajectory(out[0]),) + tuple(out[1:])
        return host_trajectory(out)
    return wrap


# ---- noise / eps (rng.py:27-33, denoiser.py:73-145, 234-267) -----------------
derive_noise = _returns_host(_rng.derive_noise)
state_independent_eps = _returns_host(_den.state_independent_eps)
eps_oracle = _returns_host(_den.eps_oracle)
velocity_oracle = _returns_host(_den.velocity_oracle)
x0_posterior_mean = _returns_host(_den.x0_posterior_mean)
evaluate = _returns_host(_den.evaluate)

# ---- transitions (transitions.py:105-188, sequential.py:51-54) ---------------
ddim_skip = _returns_host(_tr.ddim_skip)
ddpm_skip_sample = _returns_host(_tr.ddpm_skip_sample)
euler_skip = _returns_host(_tr.euler_skip)
predicted_x0 = _returns_host(_seq.predicted_x0)


@functools.wraps(_tr.ddpm_skip_posterior)
def ddpm_skip_posterior(*a, **k):
    p = _tr.ddpm_skip_posterior(*a, **k)
    return SkipPosterior(to_host(p.mean), p.variance)


# ---- samplers / schedulers (sequential.py:57-130, parallel.py:98-381) --------
sample_ddim = _returns_traj(_seq.sample_ddim)
sample_ddpm = _returns_traj(_seq.sample_ddpm)
sample_euler = _returns_traj(_seq.sample_euler)
run_aggressive = _returns_traj(_par.run_aggressive)
run_conservative = _returns_traj(_par.run_conservative)
run_parallel_euler = _returns_traj(_par.run_parallel_euler)
execute_round = _returns_host(_par.execute_round)


@functools.wraps(_met.trajectory_max_dev)
def trajectory_max_dev(a, b) -> float:
    return _met.trajectory_max_dev(a, b)


__all__ = [n for n in dir() if not n.startswith("_")]

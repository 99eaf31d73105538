"""Noise-prediction (eps) plugins evaluated on the GPU.

The reference's plugin boundary is the closed union `Denoiser` and the single
dispatch `evaluate(d, s, x, t, clock)` (skipdiff denoiser.py:221,234-267).
The same kinds exist here, evaluated by libdrs kernels:

  AnalyticEps(gm)        -> drs_gm_eps (K9): Gaussian-mixture eps oracle
  StateIndependent(seed) -> drs_noise_fill with key (0x51DE, seed & 2^32-1, t)
  Latency(inner, model)  -> drs_spin for eval_time_ms (or a VirtualClock charge)
  Counting(inner)        -> host-side counter
  NetworkEps(net)        -> a random-init denoiser network (new; no reference)

`Perturbed` (denoiser.py:191-201,224-231) runs on device too: a BLAKE2b
kernel hashes the quantised state into a noise key in HBM, K1 draws the
pseudo-noise from it and a K3 chain adds scale * noise to the eps rows, so a
perturbed run stays one captured program (PerturbPlan below).
"""

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DimensionMismatch, NonPositiveSigma, TimestepOutOfRange
from .schedule import NoiseSchedule

_STATE_INDEP_SALT = 0x51DE       # denoiser.py:22
_SEED_MASK32 = 0xFFFFFFFF        # denoiser.py:144
GM_MAX_COMP = 1920               # include/drs.h DRS_GM_MAX_COMP


@dataclass(frozen=True, eq=False)
class GaussianMixture:
    """Isotropic mixture: weights (n,), means (n, dim), variances (n,) (denoiser.py:27-58)."""

    weights: np.ndarray
    means: np.ndarray
    variances: np.ndarray
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=float)
        m = np.atleast_2d(np.asarray(self.means, dtype=float))
        v = np.asarray(self.variances, dtype=float)
        if np.any(w < 0) or abs(w.sum() - 1.0) > 1e-12:
            raise ValueError("weights must be nonnegative and sum to 1")
        if np.any(v <= 0):
            raise ValueError("variances must be positive")
        if len(w) != m.shape[0] or len(w) != len(v):
            raise DimensionMismatch("weights/means/variances lengths disagree")
        if len(w) > GM_MAX_COMP:       # K9 keeps per-component scalars in shared memory
            raise ValueError(f"{len(w)} mixture components exceed the device eps kernel's "
                             f"limit of {GM_MAX_COMP} (include/drs.h DRS_GM_MAX_COMP)")
        object.__setattr__(self, "weights", w)
        object.__setattr__(self, "means", m)
        object.__setattr__(self, "variances", v)

    @property
    def dim(self) -> int:
        return self.means.shape[1]

    def device_params(self, device):
        """(means (n, dim), log w (n,), variances (n,)) fp64 in HBM, cached."""
        import torch
        key = str(device)
        p = self._dev.get(key)
        if p is None:
            p = (torch.from_numpy(np.ascontiguousarray(self.means)).to(device),
                 torch.from_numpy(np.log(self.weights)).to(device),
                 torch.from_numpy(np.ascontiguousarray(self.variances)).to(device))
            self._dev[key] = p
        return p


def standard_normal_mixture(dim: int = 1) -> GaussianMixture:
    """N(0, I) as a one-component mixture (denoiser.py:61-63)."""
    return GaussianMixture(weights=[1.0], means=np.zeros((1, dim)), variances=[1.0])


@dataclass(frozen=True)
class LatencyModel:
    """Simulated eval cost + per-round dispatch overhead (denoiser.py:148-159)."""

    eval_time_ms: float
    dispatch_overhead_ms: float = 0.0

    def __post_init__(self):
        if not (self.eval_time_ms >= 0 and np.isfinite(self.eval_time_ms)):
            raise ValueError("eval_time_ms must be finite and >= 0")
        if not (self.dispatch_overhead_ms >= 0 and np.isfinite(self.dispatch_overhead_ms)):
            raise ValueError("dispatch_overhead_ms must be finite and >= 0")


class VirtualClock:
    """Simulated milliseconds instead of device time (denoiser.py:162-173)."""

    def __init__(self):
        self.elapsed_ms = 0.0

    def charge(self, ms: float):
        self.elapsed_ms += ms


@dataclass(frozen=True)
class AnalyticEps:
    gm: GaussianMixture


@dataclass(frozen=True)
class StateIndependent:
    seed: int
    dim: int


@dataclass(frozen=True)
class Perturbed:
    inner: object
    scale: float

    def __post_init__(self):
        if not (self.scale >= 0 and np.isfinite(self.scale)):
            raise ValueError("scale must be finite and >= 0")


@dataclass(frozen=True)
class Latency:
    inner: object
    model: LatencyModel


class Counting:
    """Counts evaluate() calls; advisory (denoiser.py:212-218)."""

    def __init__(self, inner):
        self.inner = inner
        self.count = 0


@dataclass(frozen=True, eq=False)
class NetworkEps:
    """A neural eps-predictor (UNet / DiT) running on this package's kernels.

    `net(x, t_vec) -> eps` maps a (B, *latent_shape) batch in the network's
    dtype and a (B,) timestep vector to fp32 eps of the same shape.
    `latent_shape` is the per-image latent (e.g. (4, 64, 64)); `cfg_scale`
    > 1 runs the conditional/unconditional pair as one batch-2 call and
    combines eps_u + g (eps_c - eps_u) (classifier-free guidance)."""

    net: object
    latent_shape: tuple
    cfg_scale: float = 1.0
    t_scale: float | None = None      # model timestep per sampler step (default 1000 / T)


Denoiser = AnalyticEps | StateIndependent | Perturbed | Latency | Counting | NetworkEps


# ------------------------------------------------------------ Perturbed ---
PERTURB_QUANTUM = 1e-8        # denoiser.py:24


def perturb_scales(d) -> list:
    """Scales of the Perturbed layers of a wrapper stack, innermost first;
    zero scales are identity (denoiser.py:253-256) and dropped."""
    out = []
    while True:
        if isinstance(d, Perturbed):
            if d.scale != 0.0:
                out.append(float(d.scale))
            d = d.inner
        elif isinstance(d, (Latency, Counting)):
            d = d.inner
        else:
            return out[::-1]


class _DevKeys:
    """drs_key rows already in HBM (written by drs_perturb_keys)."""

    def __init__(self, dev, n):
        self.dev, self.n = dev, n


def perturb_launch_pieces(n_ops: int, n_scales: int, limit: int = 64) -> list:
    """(offset, count) launches of a perturbation op list: row i owns ops
    [i*S, (i+1)*S), and every op of a row after its first reads the CUR
    register, so launches (<= limit ops, csrc/chain.cu kMaxOps) are cut at row
    boundaries only."""
    if n_scales > limit:
        raise ValueError(f"{n_scales} nested Perturbed layers exceed one chain launch ({limit})")
    per = (limit // n_scales) * n_scales
    return [(off, min(per, n_ops - off)) for off in range(0, n_ops, per)]


class PerturbPlan:
    """Device resources adding every Perturbed layer's pseudo-noise to eps rows:
    outs[i] += scale * default_rng(blake2b(state_i, t_i)).standard_normal(D)
    for each scale, innermost first (denoiser.py:224-231,253-256)."""

    def __init__(self, scales, xs, ts, outs, device):
        import torch
        from .transitions import make_op, ops_to_device
        self.n, self.D = len(xs), int(xs[0].numel())
        self.xs = _ptr_array(xs, device)
        self.ts = torch.tensor([int(t) for t in ts], dtype=torch.int32, device=device)
        self.keys = torch.zeros(self.n * _lib.ctypes.sizeof(_lib.DrsKey), dtype=torch.uint8, device=device)
        self.noise = torch.empty(self.n, self.D, dtype=torch.float64, device=device)
        ops = []
        for i in range(self.n):
            for j, sc in enumerate(scales):       # out = eps + scale * noise (K3 euler form), chained
                ops.append(make_op([sc, 1.0, 0.0, 0.0, 1.0, 0.0], _lib.FAMILY_EULER, False,
                                   src=_lib.SRC_X if j == 0 else _lib.SRC_CUR, x=outs[i] if j == 0 else None,
                                   eps=self.noise[i], out=outs[i]))
        self.n_ops = len(ops)
        self.ops = ops_to_device(ops, device)
        # a row's ops after the first read the CUR register: launches are cut at
        # row boundaries only (<= 64 ops, csrc/chain.cu kMaxOps)
        self.pieces = perturb_launch_pieces(self.n_ops, len(scales))

    def launch(self, err, stream=None):
        from .rng import fill_streams
        L = _lib.lib()
        sp = _lib.stream_ptr(stream)
        _lib.check(L.drs_perturb_keys(self.xs.data_ptr(), self.ts.data_ptr(), self.n, self.D, PERTURB_QUANTUM,
                                      self.keys.data_ptr(), sp), "drs_perturb_keys")
        fill_streams(_DevKeys(self.keys, self.n), self.D, self.noise, "pcg64", err=err, stream=stream)
        size = _lib.ctypes.sizeof(_lib.DrsOp)
        for off, n in self.pieces:
            _lib.check(L.drs_skip_chain(self.ops.data_ptr() + off * size, n, self.D, sp), "drs_skip_chain")


def apply_perturbations(scales, x, t: int, value):
    """value (eps of state x at t, CUDA fp64) + the Perturbed layers' noise, in place."""
    import torch
    from .rng import _check_err
    if not scales:
        return value
    err = torch.zeros(1, dtype=torch.int32, device=value.device)
    plan = PerturbPlan(scales, [x.reshape(-1)], [t], [value.reshape(-1)], value.device)
    plan.launch(err)
    _check_err(err)
    return value


# ------------------------------------------------------------ oracles -----
def _rows(x, D):
    """x (D,) or (n, D) CUDA fp64 -> list of row tensors."""
    if x.dim() == 1:
        return [x]
    return [x[i] for i in range(x.shape[0])]


def _ptr_array(tensors, device):
    import torch
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64, device=device)


def gm_eps_launch(gm: GaussianMixture, s: NoiseSchedule, xs, ts, outs, err, stream=None):
    """Launch K9 for row lists xs/outs (CUDA fp64 tensors of gm.dim) at timesteps ts."""
    import torch
    dev = outs[0].device
    means, logw, var = gm.device_params(dev)
    xs_p = _ptr_array(xs, dev)
    out_p = _ptr_array(outs, dev)
    ts_d = torch.tensor([int(t) for t in ts], dtype=torch.int32, device=dev)
    st = _lib.lib().drs_gm_eps(xs_p.data_ptr(), ts_d.data_ptr(), len(xs), gm.dim,
                              s.device_alpha_bar(dev).data_ptr(), s.T, means.data_ptr(),
                              logw.data_ptr(), var.data_ptr(), len(gm.weights),
                              out_p.data_ptr(), err.data_ptr(), _lib.stream_ptr(stream))
    _lib.check(st, "drs_gm_eps")
    return (xs_p, out_p, ts_d)      # keep the staging alive until the launch retires


def eps_oracle(gm: GaussianMixture, s: NoiseSchedule, x, t: int):
    """Bayes-optimal eps of the VP-noised mixture (denoiser.py:85-107), on device."""
    import torch
    from .transitions import _device_of, as_device
    if not 0 <= t <= s.T:
        raise TimestepOutOfRange(f"t={t} outside 0..{s.T}")
    dev = _device_of(x)
    xd = as_device(x, dev, torch.float64)
    if xd.shape[-1] != gm.dim:
        raise DimensionMismatch(f"state dim {xd.shape[-1]} != mixture dim {gm.dim}")
    flat = xd.reshape(-1, gm.dim)
    out = torch.empty_like(flat)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    keep = gm_eps_launch(gm, s, _rows(flat, gm.dim), [t] * flat.shape[0], _rows(out, gm.dim), err)
    del keep
    return out.reshape(xd.shape)


def state_independent_key(seed: int, t: int):
    from .rng import entropy_key
    return entropy_key((_STATE_INDEP_SALT, seed & _SEED_MASK32, t))


def state_independent_eps(seed: int, t: int, dim: int, *, device=None):
    """Pseudo-noise depending only on (seed, t, dim) (denoiser.py:139-145)."""
    import torch
    from .rng import _check_err, _default_device, fill_streams
    if t < 0:
        raise TimestepOutOfRange(f"t={t} must be >= 0")
    dev = _default_device(device)
    out = torch.empty(dim, dtype=torch.float64, device=dev)
    if dim:
        _check_err(fill_streams([state_independent_key(seed, t)], dim, out.view(1, dim)))
    return out


def gm_velocity_launch(gm: GaussianMixture, sigmas, N: int, xs, idx, outs, err, stream=None):
    """Launch K9 in VE-velocity mode for row lists xs/outs (CUDA fp64, gm.dim)
    at sigma-table indices idx (sigmas: CUDA fp64, N+1 entries)."""
    import torch
    dev = outs[0].device
    means, logw, var = gm.device_params(dev)
    xs_p = _ptr_array(xs, dev)
    out_p = _ptr_array(outs, dev)
    idx_d = torch.tensor([int(i) for i in idx], dtype=torch.int32, device=dev)
    st = _lib.lib().drs_gm_velocity(xs_p.data_ptr(), idx_d.data_ptr(), len(xs), gm.dim, sigmas.data_ptr(), N,
                                    means.data_ptr(), logw.data_ptr(), var.data_ptr(), len(gm.weights),
                                    out_p.data_ptr(), err.data_ptr(), _lib.stream_ptr(stream))
    _lib.check(st, "drs_gm_velocity")
    return (xs_p, out_p, idx_d)


def velocity_oracle(gm: GaussianMixture, x, sigma: float):
    """ODE velocity (x - x0_hat)/sigma of the variance-exploding mixture
    p_sigma = sum_i w_i N(m_i, (v_i + sigma^2) I) (denoiser.py:124-136), on device."""
    import torch
    from .rng import _check_err
    from .transitions import _device_of, as_device
    if not sigma > 0.0:
        raise NonPositiveSigma(f"sigma must be > 0, got {sigma}")
    dev = _device_of(x)
    xd = as_device(x, dev, torch.float64)
    if xd.shape[-1] != gm.dim:
        raise DimensionMismatch(f"state dim {xd.shape[-1]} != mixture dim {gm.dim}")
    flat = xd.reshape(-1, gm.dim)
    out = torch.empty_like(flat)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    table = torch.tensor([float(sigma)], dtype=torch.float64, device=dev)
    keep = gm_velocity_launch(gm, table, 0, _rows(flat, gm.dim), [0] * flat.shape[0], _rows(out, gm.dim), err)
    _check_err(err)
    del keep
    return out.reshape(xd.shape)


def x0_posterior_mean(gm: GaussianMixture, x, abar: float):
    """E[x_0 | x_t = x] under the same VP noising as eps_oracle (denoiser.py:110-121),
    on device (K9 posterior-mean mode)."""
    import torch
    from .rng import _check_err
    from .transitions import _device_of, as_device
    if not 0.0 < abar <= 1.0:
        raise ValueError(f"abar must lie in (0, 1], got {abar}")
    dev = _device_of(x)
    xd = as_device(x, dev, torch.float64)
    if xd.shape[-1] != gm.dim:
        raise DimensionMismatch(f"state dim {xd.shape[-1]} != mixture dim {gm.dim}")
    flat = xd.reshape(-1, gm.dim)
    out = torch.empty_like(flat)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    means, logw, var = gm.device_params(dev)
    xs_p = _ptr_array(_rows(flat, gm.dim), dev)
    out_p = _ptr_array(_rows(out, gm.dim), dev)
    zeros = torch.zeros(flat.shape[0], dtype=torch.int32, device=dev)
    table = torch.tensor([float(abar)], dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().drs_gm_x0_mean(xs_p.data_ptr(), zeros.data_ptr(), flat.shape[0], gm.dim,
                                         table.data_ptr(), means.data_ptr(), logw.data_ptr(), var.data_ptr(),
                                         len(gm.weights), out_p.data_ptr(), err.data_ptr(), _lib.stream_ptr()),
               "drs_gm_x0_mean")
    _check_err(err)
    return out.reshape(xd.shape)


@dataclass(frozen=True, eq=False)
class EulerVelocity:
    """Engine core of the Euler family: the velocity of `gm` on sigma grid `g`;
    a program task at "t" (remaining grid intervals) evaluates at sigma_{N-t}."""
    gm: GaussianMixture
    grid: object


_EULER_CORES: dict = {}


def euler_velocity_core(gm: GaussianMixture, g) -> EulerVelocity:
    """One EulerVelocity per (mixture, grid) so compiled runs are reused."""
    key = (id(gm), id(g))
    core = _EULER_CORES.get(key)
    if core is None or core.gm is not gm or core.grid is not g:
        core = EulerVelocity(gm, g)
        _EULER_CORES[key] = core
    return core


def latency_of(d):
    """Innermost LatencyModel of a wrapper stack (denoiser.py:270-277)."""
    if isinstance(d, Latency):
        return d.model
    if isinstance(d, (Perturbed, Counting)):
        return latency_of(d.inner)
    return None


def spin(ms: float, n_ctas: int = 1, stream=None):
    _lib.check(_lib.lib().drs_spin(ms * 1000.0, n_ctas, _lib.stream_ptr(stream)), "drs_spin")


def evaluate(d, s: NoiseSchedule, x, t: int, clock: VirtualClock | None = None):
    """The single eps entry point of the samplers (denoiser.py:234-267).

    With a VirtualClock, Latency charges the clock; without one it occupies
    the GPU for eval_time_ms (drs_spin) before the inner evaluation."""
    if isinstance(d, AnalyticEps):
        return eps_oracle(d.gm, s, x, t)
    if isinstance(d, StateIndependent):
        if t < 0 or t > s.T:
            raise TimestepOutOfRange(f"t={t} outside 0..{s.T}")
        import torch
        dev = x.device if isinstance(x, torch.Tensor) and x.is_cuda else None
        return state_independent_eps(d.seed, t, d.dim, device=dev)
    if isinstance(d, Perturbed):
        value = evaluate(d.inner, s, x, t, clock)
        if d.scale == 0.0:
            return value
        import torch
        from .transitions import _device_of, as_device
        dev = _device_of(x, value)
        xd = as_device(x, dev, torch.float64)
        out = as_device(value, dev, torch.float64).clone().reshape(xd.shape)
        return apply_perturbations([d.scale], xd, t, out)
    if isinstance(d, Latency):
        if clock is not None:
            clock.charge(d.model.eval_time_ms)
        elif d.model.eval_time_ms > 0:
            spin(d.model.eval_time_ms)
        return evaluate(d.inner, s, x, t, clock)
    if isinstance(d, Counting):
        d.count += 1
        return evaluate(d.inner, s, x, t, clock)
    if isinstance(d, NetworkEps):
        from .netdenoise import network_eps
        return network_eps(d, s, x, [t])
    raise TypeError(f"unknown denoiser kind: {type(d).__name__}")

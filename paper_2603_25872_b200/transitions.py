"""Closed-form skip transitions x_t -> x_{t-k} on the GPU.

Scalar coefficients are computed on the host with the reference's own scalar
expressions (skipdiff transitions.py:98-179, sequential.py:51-54) and the
elementwise update runs in libdrs `drs_skip_chain` (K2/K3, csrc/chain.cu) in
the reference's operation order with no FMA contraction, so results are
bit-identical to the numpy reference given the same inputs.  Noise z is
always injected by the caller (transitions.py:14-15).
"""

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .errors import IndexOutOfRange, InvalidSkip, TimestepOutOfRange, VarianceTooLarge
from .schedule import NoiseSchedule, SigmaGrid


class VarianceKind(Enum):
    DETERMINISTIC = "deterministic"
    DDPM_INDUCED = "ddpm"
    ETA = "eta"


@dataclass(frozen=True)
class VarianceRule:
    """sigma_{t,k} policy: zero, DDPM-induced, or eta x induced (transitions.py:34-71)."""

    kind: VarianceKind
    eta: float = 0.0

    def __post_init__(self):
        if self.kind is VarianceKind.ETA and not 0.0 <= self.eta <= 1.0:
            raise ValueError(f"eta must lie in [0, 1], got {self.eta}")

    @classmethod
    def deterministic(cls):
        return cls(VarianceKind.DETERMINISTIC)

    @classmethod
    def ddpm_induced(cls):
        return cls(VarianceKind.DDPM_INDUCED)

    @classmethod
    def eta_scaled(cls, eta: float):
        return cls(VarianceKind.ETA, eta=eta)

    @property
    def stochastic(self) -> bool:
        if self.kind is VarianceKind.DDPM_INDUCED:
            return True
        return self.kind is VarianceKind.ETA and self.eta > 0.0

    def sigma(self, s: NoiseSchedule, t: int, k: int) -> float:
        if self.kind is VarianceKind.DETERMINISTIC:
            return 0.0
        induced = math.sqrt(_ddpm_skip_variance(s, t, k))
        return induced if self.kind is VarianceKind.DDPM_INDUCED else self.eta * induced


@dataclass(frozen=True)
class SkipCoeffs:
    """x_{t-k} = kappa x_t + lam x_0 + sigma z (transitions.py:74-80)."""

    kappa: float
    lam: float
    sigma: float


@dataclass(frozen=True)
class SkipPosterior:
    """q(x_{t-k} | x_t, x_0): device mean tensor + scalar variance (transitions.py:83-88)."""

    mean: object
    variance: float


def _check_skip(s: NoiseSchedule, t: int, k: int):
    if k < 1:
        raise InvalidSkip(f"k={k} must be >= 1")
    if t > s.T or k > t:
        raise TimestepOutOfRange(f"(t={t}, k={k}) outside 1 <= k <= t <= {s.T}")


def _ddpm_skip_variance(s: NoiseSchedule, t: int, k: int) -> float:
    _check_skip(s, t, k)
    a_t = s.alpha_bar[t]
    a_s = s.alpha_bar[t - k]
    return (1.0 - a_t / a_s) * (1.0 - a_s) / (1.0 - a_t)


def ddim_skip_coeffs(s: NoiseSchedule, t: int, k: int, rule: VarianceRule) -> SkipCoeffs:
    """kappa/lambda/sigma with the VarianceTooLarge check (transitions.py:137-152)."""
    _check_skip(s, t, k)
    a_t, a_s = s.alpha_bar[t], s.alpha_bar[t - k]
    sigma = rule.sigma(s, t, k)
    radicand = 1.0 - a_s - sigma * sigma
    if radicand < 0.0:
        raise VarianceTooLarge(f"sigma^2={sigma * sigma} exceeds 1 - alpha_bar[{t - k}]={1.0 - a_s}")
    kappa = math.sqrt(radicand) / math.sqrt(1.0 - a_t)
    return SkipCoeffs(kappa=kappa, lam=math.sqrt(a_s) - kappa * math.sqrt(a_t), sigma=sigma)


# ------------------------------------------------------- device op builders --
def ddim_op_coeffs(s: NoiseSchedule, t: int, k: int, rule: VarianceRule):
    """(c[6], noisy) of the DDIM update t -> t-k; host validation as ddim_skip."""
    coeffs = ddim_skip_coeffs(s, t, k, rule)
    a_t, a_s = s.alpha_bar[t], s.alpha_bar[t - k]
    c = [math.sqrt(1.0 - a_t), math.sqrt(a_t), math.sqrt(a_s),
         math.sqrt(1.0 - a_s - coeffs.sigma ** 2), coeffs.sigma, 0.0]
    return c, coeffs.sigma > 0.0


def ddpm_op_coeffs(s: NoiseSchedule, t: int, k: int):
    """(c[6], noisy) of the DDPM posterior skip t -> t-k (transitions.py:105-134)."""
    _check_skip(s, t, k)
    a_t, a_s = s.alpha_bar[t], s.alpha_bar[t - k]
    ratio = a_t / a_s
    denom = 1.0 - a_t
    variance = (1.0 - ratio) * (1.0 - a_s) / denom
    c = [math.sqrt(1.0 - a_t), math.sqrt(a_t),
         float(np.sqrt(ratio) * (1.0 - a_s)), float(np.sqrt(a_s) * (1.0 - ratio)),
         float(denom), math.sqrt(variance)]
    return c, variance != 0.0


def make_op(c, family, noisy, *, src=_lib.SRC_X, x=None, eps=None, z=None, out=None, out2=None,
            save_anchor=False) -> _lib.DrsOp:
    op = _lib.DrsOp()
    for i in range(6):
        op.c[i] = float(c[i])
    op.family = family
    op.noisy = 1 if noisy else 0
    op.src = src
    op.flags = _lib.OP_SAVE_ANCHOR if save_anchor else 0
    op.eps_f32 = 0
    if eps is not None:
        import torch
        op.eps_f32 = 1 if eps.dtype == torch.float32 else 0
        op.eps = eps.data_ptr()
    op.x = x.data_ptr() if x is not None else None
    op.z = z.data_ptr() if z is not None else None
    op.out = out.data_ptr() if out is not None else None
    op.out2 = out2.data_ptr() if out2 is not None else None
    return op


def ops_to_device(ops, device):
    import torch
    raw = (_lib.DrsOp * len(ops))(*ops)
    return torch.frombuffer(bytearray(bytes(raw)), dtype=torch.uint8).to(device)


def launch_chain(ops_dev, n_ops: int, D: int, offset: int = 0, stream=None):
    """Run n_ops device ops starting at op index `offset` of ops_dev."""
    ptr = ops_dev.data_ptr() + offset * _lib.ctypes.sizeof(_lib.DrsOp)
    _lib.check(_lib.lib().drs_skip_chain(ptr, n_ops, D, _lib.stream_ptr(stream)), "drs_skip_chain")


# ------------------------------------------------------- functional API ----
def _device_of(*arrs):
    import torch
    for a in arrs:
        if isinstance(a, torch.Tensor) and a.is_cuda:
            return a.device
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_25872_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def as_device(a, device, dtype=None):
    """Contiguous CUDA tensor view/copy of a numpy array or tensor (fp64 by default)."""
    import torch
    if isinstance(a, torch.Tensor):
        t = a.to(device=device)
        if dtype is not None or t.dtype not in (torch.float64, torch.float32):
            t = t.to(dtype or torch.float64)
        return t.contiguous()
    return torch.as_tensor(np.asarray(a, dtype=float), device=device).contiguous()


def _run_single(c, family, noisy, x, eps, z):
    import torch
    dev = _device_of(x, eps, z)
    xd = as_device(x, dev, torch.float64)
    ed = as_device(eps, dev)
    zd = as_device(z, dev, torch.float64) if (z is not None and noisy) else None
    shape = torch.broadcast_shapes(xd.shape, ed.shape, *( [zd.shape] if zd is not None else []))
    xd = xd.expand(shape).contiguous()
    ed = ed.expand(shape).contiguous()
    if zd is not None:
        zd = zd.expand(shape).contiguous()
    out = torch.empty(shape, dtype=torch.float64, device=dev)
    op = make_op(c, family, noisy, x=xd, eps=ed, z=zd, out=out)
    launch_chain(ops_to_device([op], dev), 1, out.numel())
    return out


def ddpm_skip_posterior(s: NoiseSchedule, t: int, k: int, x_t, x0_hat) -> SkipPosterior:
    """k-step DDPM posterior q(x_{t-k}|x_t, x0_hat) (transitions.py:105-116)."""
    c, noisy = ddpm_op_coeffs(s, t, k)
    a_t, a_s = s.alpha_bar[t], s.alpha_bar[t - k]
    ratio = a_t / a_s
    variance = (1.0 - ratio) * (1.0 - a_s) / (1.0 - a_t)
    mean = _run_single(c, _lib.FAMILY_DDPM_X0, False, x_t, x0_hat, None)
    return SkipPosterior(mean=mean, variance=float(variance))


def ddpm_skip_sample(s: NoiseSchedule, t: int, k: int, x_t, x0_hat, z):
    """mean + sqrt(var) z; z may be None only if var == 0 (transitions.py:119-134)."""
    c, noisy = ddpm_op_coeffs(s, t, k)
    if noisy and z is None:
        raise ValueError("z required for a stochastic transition")
    return _run_single(c, _lib.FAMILY_DDPM_X0, noisy, x_t, x0_hat, z)


def ddim_skip(s: NoiseSchedule, t: int, k: int, x_t, eps, rule: VarianceRule, z=None):
    """DDIM skip x_t -> x_{t-k} (transitions.py:155-179)."""
    c, noisy = ddim_op_coeffs(s, t, k, rule)
    if noisy and z is None:
        raise ValueError("z required for a stochastic transition")
    return _run_single(c, _lib.FAMILY_DDIM, noisy, x_t, eps, z)


def predicted_x0_device(s: NoiseSchedule, x_t, eps, t: int):
    """x0_hat = (x_t - sqrt(1-abar_t) eps) / sqrt(abar_t) (sequential.py:51-54)."""
    a_t = s.alpha_bar[t]
    c = [math.sqrt(1.0 - a_t), math.sqrt(a_t), 0.0, 0.0, 1.0, 0.0]
    return _run_single(c, _lib.FAMILY_PRED_X0, False, x_t, eps, None)


def euler_op_coeffs(g: SigmaGrid, i: int, k: int):
    """(c[6], noisy) of the fused Euler step across grid intervals i..i+k:
    out = x + (sigma_{i+k} - sigma_i) v, the difference formed on the host in
    fp64 exactly as transitions.py:188; host validation as euler_skip."""
    if k < 1:
        raise InvalidSkip(f"k={k} must be >= 1")
    if i < 0 or i + k > g.N:
        raise IndexOutOfRange(f"(i={i}, k={k}) outside 0 <= i, i+k <= {g.N}")
    return [float(g.sigmas[i + k] - g.sigmas[i]), 1.0, 0.0, 0.0, 1.0, 0.0], False


def euler_skip(g: SigmaGrid, i: int, k: int, x, v):
    """x + (sigma_{i+k} - sigma_i) v (transitions.py:182-188)."""
    c, _ = euler_op_coeffs(g, i, k)
    return _run_single(c, _lib.FAMILY_EULER, False, x, v, None)

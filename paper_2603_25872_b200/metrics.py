"""Distribution distances and trajectory deviation on the GPU (skipdiff
metrics.py): the 10^4-sample quality checks of
test_acceptance.py:206-229 at real latent sizes.

Same names, arguments and errors as the reference.  Samples live in HBM as
(n, dim) fp64.  `sliced_w2` draws its directions with the device PCG64 +
ziggurat kernel (K1), bit-identical to numpy's default_rng(seed)
.standard_normal; projections are one fp64 GEMM; 1-D quantiles are sorted on
device with numpy's 'linear' interpolation.  `mmd_gaussian` sums the Gaussian
kernel over all pairs with K10 (csrc/metrics.cu) without forming the n x m
kernel matrices.  Results match the reference to fp64 rounding (reduction
order differs), the tolerance its own tests use (rel 1e-12).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatch, EmptySet, InsufficientSamples, TimestepMismatch
from .rng import _check_err, _default_device, entropy_key, fill_streams


@dataclass(frozen=True)
class SampleSet:
    """Samples as an (n, dim) CUDA fp64 tensor with a label (metrics.py:17-35)."""

    samples: object
    label: str = ""

    def __post_init__(self):
        x = self.samples
        if not isinstance(x, torch.Tensor):
            x = torch.as_tensor(np.asarray(x, dtype=float))
        if x.numel() == 0:
            raise EmptySet(f"sample set {self.label!r} is empty")
        if x.dim() < 2:
            x = x.reshape(1, -1)
        dev = x.device if x.device.type == "cuda" else _default_device(None)
        object.__setattr__(self, "samples", x.reshape(x.shape[0], -1).to(dev, torch.float64).contiguous())

    @property
    def dim(self) -> int:
        return self.samples.shape[1]

    def __len__(self) -> int:
        return self.samples.shape[0]


def _check_dims(a: SampleSet, b: SampleSet):
    if a.dim != b.dim:
        raise DimensionMismatch(f"dims differ: {a.dim} vs {b.dim}")


def _directions(seed: int, projections: int, dim: int, device):
    """default_rng(seed).standard_normal((projections, dim)), unit rows."""
    d = torch.empty(projections * dim, dtype=torch.float64, device=device)
    _check_err(fill_streams([entropy_key((int(seed),))], projections * dim, d.view(1, -1)))
    d = d.view(projections, dim)
    return d / torch.linalg.vector_norm(d, dim=1, keepdim=True)


def _quantiles_linear(sorted_cols, qs):
    """np.quantile(method='linear') of each column of an ascending-sorted
    (n, P) tensor at levels qs, with numpy's two-sided lerp (numpy
    lib/_function_base_impl.py _lerp: b - (b - a)(1 - t) for t >= 0.5)."""
    n = sorted_cols.shape[0]
    pos = qs * (n - 1)
    lo = torch.floor(pos).to(torch.int64)
    hi = torch.clamp(lo + 1, max=n - 1)
    t = (pos - lo.to(pos.dtype)).unsqueeze(1)
    a, b = sorted_cols[lo], sorted_cols[hi]
    diff = b - a
    return torch.where(t >= 0.5, b - diff * (1.0 - t), a + diff * t)


def sliced_w2(a: SampleSet, b: SampleSet, projections: int = 64, seed: int = 0) -> float:
    """Mean over random unit directions of the squared 1-D W2 between the
    projected empirical distributions (metrics.py:42-69)."""
    _check_dims(a, b)
    if projections < 1:
        raise ValueError("projections must be >= 1")
    dev = a.samples.device
    dirs = _directions(seed, projections, a.dim, dev)
    proj_a = a.samples @ dirs.T
    proj_b = b.samples.to(dev) @ dirs.T
    m = min(len(a), len(b))
    qs = (torch.arange(m, dtype=torch.float64, device=dev) + 0.5) / m

    def quantiles(proj):
        s = torch.sort(proj, dim=0).values
        return s if proj.shape[0] == m else _quantiles_linear(s, qs)

    diff = quantiles(proj_a) - quantiles(proj_b)
    return float(torch.mean(diff * diff).item())


def _mmd_sum(A, na, B, nb, gamma, same):
    n, m = A.shape[0], B.shape[0]
    gx, gy = -(-m // 64), -(-n // 64)
    part = torch.empty(gx * gy, dtype=torch.float64, device=A.device)
    _lib.check(_lib.lib().drs_mmd_partials(A.data_ptr(), na.data_ptr(), n, B.data_ptr(), nb.data_ptr(), m,
                                           A.shape[1], float(gamma), 1 if same else 0, part.data_ptr(),
                                           _lib.stream_ptr()), "drs_mmd_partials")
    return part.sum()


def _sqnorms(X):
    out = torch.empty(X.shape[0], dtype=torch.float64, device=X.device)
    _lib.check(_lib.lib().drs_row_sqnorm(X.data_ptr(), X.shape[0], X.shape[1], out.data_ptr(), _lib.stream_ptr()),
               "drs_row_sqnorm")
    return out


def mmd_gaussian(a: SampleSet, b: SampleSet, bandwidth: float) -> float:
    """Unbiased MMD^2 with kernel exp(-||u - v||^2 / (2 bandwidth^2)) (metrics.py:72-89)."""
    _check_dims(a, b)
    if bandwidth <= 0:
        raise ValueError("bandwidth must be > 0")
    if len(a) < 2 or len(b) < 2:
        raise InsufficientSamples("unbiased MMD needs at least 2 samples per set")
    A, B = a.samples, b.samples.to(a.samples.device)
    gamma = 1.0 / (2.0 * bandwidth ** 2)
    na, nb = _sqnorms(A), _sqnorms(B)
    n, m = len(a), len(b)
    term_aa = _mmd_sum(A, na, A, na, gamma, True) / (n * (n - 1))
    term_bb = _mmd_sum(B, nb, B, nb, gamma, True) / (m * (m - 1))
    term_ab = _mmd_sum(A, na, B, nb, gamma, False) / (n * m)
    return float((term_aa + term_bb - 2.0 * term_ab).item())


def mmd_permutation_threshold(a: SampleSet, b: SampleSet, bandwidth: float, permutations: int = 200,
                              quantile: float = 0.95, seed: int = 0) -> float:
    """Null threshold: the quantile of MMD^2 over random relabelings of the
    pooled samples (metrics.py:92-109); permutations drawn with numpy's
    Generator exactly as the reference, the MMDs evaluated on device."""
    _check_dims(a, b)
    pooled = torch.cat([a.samples, b.samples.to(a.samples.device)])
    n = len(a)
    rng = np.random.default_rng(seed)
    vals = []
    for _ in range(permutations):
        idx = torch.from_numpy(rng.permutation(len(pooled))).to(pooled.device)
        p = pooled[idx]
        vals.append(mmd_gaussian(SampleSet(p[:n]), SampleSet(p[n:]), bandwidth))
    return float(np.quantile(vals, quantile))


def trajectory_max_dev(a, b) -> float:
    """Max over shared timesteps of the Euclidean distance between states (metrics.py:112-121)."""
    ta, tb = a.timesteps(), b.timesteps()
    if ta != tb:
        raise TimestepMismatch(f"timestep lists differ: {ta[:5]}... vs {tb[:5]}...")
    dev = next((x.device for _, x in a.states + b.states if isinstance(x, torch.Tensor) and x.is_cuda), None)
    dev = _default_device(dev)
    xa = torch.stack([torch.as_tensor(x, dtype=torch.float64).reshape(-1).to(dev) for _, x in a.states])
    xb = torch.stack([torch.as_tensor(x, dtype=torch.float64).reshape(-1).to(dev) for _, x in b.states])
    return float(torch.linalg.vector_norm(xa - xb, dim=1).max().item())


__all__ = ["SampleSet", "mmd_gaussian", "mmd_permutation_threshold", "sliced_w2", "trajectory_max_dev"]

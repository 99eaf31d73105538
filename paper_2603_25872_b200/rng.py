"""Counter-based noise streams generated on the GPU.

Every normal vector is a pure function of a key (skipdiff rng.py:1-3): the
key is the entropy tuple handed to numpy's SeedSequence, and the draw is
bit-identical to `Generator(PCG64(SeedSequence(key))).standard_normal(n)`
(rng.py:32-33).  `RngStream(seed, generator="sfc64")` selects the SFC64
variant of the same key scheme (BASELINE config C2).  Draws are produced by
libdrs `drs_noise_fill` (K1, csrc/noise.cu) straight into HBM.
"""

import ctypes
from dataclasses import dataclass
from enum import IntEnum

from . import _lib

_STREAM_SALT = 0x7A9C                 # rng.py:10
_SEED_MASK48 = 0xFFFFFFFFFFFF         # rng.py:32
GENERATORS = {"pcg64": _lib.GEN_PCG64, "sfc64": _lib.GEN_SFC64}


class Role(IntEnum):
    """Key role (rng.py:13-16)."""

    TRANSITION = 0   # noise of the transition that survives into timestep t
    DRAFT = 1        # noise of discarded drafts (i >= 2)
    INIT = 2         # the run's initial x_T


@dataclass(frozen=True)
class RngStream:
    """A seed plus the bit generator behind it (rng.py:19-24)."""

    seed: int
    generator: str = "pcg64"

    def __post_init__(self):
        if self.generator not in GENERATORS:
            raise ValueError(f"unknown generator {self.generator!r}; use one of {sorted(GENERATORS)}")

    def derive(self, t: int, role: Role, shape, *, device=None):
        return derive_noise(self, t, role, shape, device=device)


def key_for(stream: RngStream, t: int, role: Role, seed_slot: int = -1) -> _lib.DrsKey:
    """drs_key for (0x7A9C, seed & 2^48-1, t, role).  With seed_slot >= 0 the
    seed is read from a device word at launch time (graph replay)."""
    if t < 0:
        raise ValueError(f"t={t} must be >= 0")
    k = _lib.DrsKey()
    k.vals[0] = _STREAM_SALT
    k.vals[1] = stream.seed & _SEED_MASK48
    k.vals[2] = int(t)
    k.vals[3] = int(role)
    k.n_vals = 4
    k.seed_slot = seed_slot
    k.seed_mask = _SEED_MASK48
    return k


def entropy_key(vals, seed_slot: int = -1, seed_mask: int = 0xFFFFFFFFFFFFFFFF) -> _lib.DrsKey:
    """drs_key for an arbitrary tuple of <= 4 non-negative ints < 2^63."""
    vals = [int(v) for v in vals]
    if not 1 <= len(vals) <= 4 or any(v < 0 or v >= 1 << 63 for v in vals):
        raise ValueError(f"unsupported entropy tuple {vals}")
    k = _lib.DrsKey()
    for i, v in enumerate(vals):
        k.vals[i] = v
    k.n_vals = len(vals)
    k.seed_slot = seed_slot
    k.seed_mask = seed_mask
    return k


def _numel(shape) -> tuple:
    if isinstance(shape, int):
        return (shape,), shape
    shape = tuple(int(s) for s in shape)
    n = 1
    for s in shape:
        n *= s
    return shape, n


def _default_device(device):
    import torch
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_25872_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


class _KeyBuffer:
    """Keys staged in HBM for one drs_noise_fill launch."""

    def __init__(self, keys, device):
        import torch
        raw = (_lib.DrsKey * len(keys))(*keys)
        host = torch.frombuffer(bytearray(bytes(raw)), dtype=torch.uint8)
        self.dev = host.to(device)
        self.n = len(keys)


def fill_streams(keys, n: int, out, generator: str = "pcg64", seeds=None, err=None, stream=None):
    """Launch K1: out[s, :n] = normals of keys[s].  `out` is a CUDA fp64
    tensor of shape (len(keys), >= n), row-contiguous."""
    import torch
    device = out.device
    kb = keys if hasattr(keys, "dev") else _KeyBuffer(keys, device)     # keys already in HBM, or a host list
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=device)
    ld = out.stride(0) if out.dim() == 2 else n
    st = _lib.lib().drs_noise_fill(
        GENERATORS[generator], kb.dev.data_ptr(), kb.n,
        seeds.data_ptr() if seeds is not None else None,
        n, out.data_ptr(), ld, err.data_ptr(), _lib.stream_ptr(stream))
    _lib.check(st, "drs_noise_fill")
    return err


def derive_noise(stream: RngStream, t: int, role: Role, shape, *, device=None):
    """Standard normals keyed by (seed, t, role) (rng.py:27-33), as a CUDA fp64
    tensor of `shape` (C-order fill, so any shape with the same numel holds
    the same draws, like numpy)."""
    import torch
    key = key_for(stream, t, role)
    shp, n = _numel(shape)
    dev = _default_device(device)
    out = torch.empty(shp, dtype=torch.float64, device=dev)
    if n:
        err = fill_streams([key], n, out.view(1, n), stream.generator)
        _check_err(err)
    return out


def _check_err(err):
    v = int(err.item())
    if v & _lib.ERR_NOISE_WINDOW_BIT:
        raise RuntimeError("ziggurat tail exceeded the noise kernel's lookahead window")
    if v & _lib.ERR_GM_SIGMA_BIT:
        from .errors import NonPositiveSigma
        raise NonPositiveSigma("device velocity evaluated at sigma <= 0")
    if v & _lib.ERR_GM_TIMESTEP_BIT:
        from .errors import TimestepOutOfRange
        raise TimestepOutOfRange("device eps evaluated outside 0..T")

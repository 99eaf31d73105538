"""libdrs.so host-side checks (no GPU): every symbol include/drs.h declares is
exported; the host builds of the glibc ports used by the noise kernel match
the host libm bit-for-bit; SeedSequence restatement matches numpy; the
generated tables are current; the product fails loudly without CUDA."""

import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported(libdrs):
    decls = set()
    for h in ("drs.h", "drs_net.h"):
        hdr = open(os.path.join(ROOT, "include", h)).read()
        decls |= set(re.findall(r"^(?:int|double|size_t)\s+(drs_\w+)\s*\(", hdr, re.M))
    assert decls, "no declarations parsed"
    from paper_2603_25872_b200 import _lib
    assert decls == set(_lib.EXPORTED)
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (drs_\w+)", nm))
    assert decls <= exported, decls - exported
    for name in decls:
        assert getattr(libdrs, name) is not None


def _libm():
    m = ctypes.CDLL("libm.so.6")
    for f in (m.log1p, m.exp):
        f.restype, f.argtypes = ctypes.c_double, [ctypes.c_double]
    return m


def test_log1p_port_matches_libm(libdrs):
    m = _libm()
    rng = np.random.default_rng(0)
    # the ziggurat tail feeds log1p(-u), u = k * 2^-53 in [0, 1)
    us = -(rng.integers(0, 2 ** 53, 200_000).astype(np.float64) * 2.0 ** -53)
    broad = np.concatenate([rng.uniform(-1, 1, 20_000), rng.uniform(-1, 1e6, 20_000),
                            np.exp(rng.uniform(-80, 40, 20_000)), -np.exp(rng.uniform(-80, 0, 20_000)),
                            [0.0, -0.0, 1e-300, -1e-300, 2.0 ** -54, 2.0 ** -29, -0.2929, 0.41422]])
    for x in np.concatenate([us, broad[broad > -1]]):
        a, b = libdrs.drs_host_log1p(float(x)), m.log1p(float(x))
        assert a == b or (a != a and b != b), x


def test_exp_port_matches_libm(libdrs):
    m = _libm()
    rng = np.random.default_rng(1)
    wedge = -0.5 * rng.uniform(0, 3.7, 200_000) ** 2          # numpy ziggurat wedge test argument
    broad = np.concatenate([rng.uniform(-745, 709, 50_000), rng.uniform(-1e-12, 1e-12, 5_000),
                            [0.0, -0.0, 1e-320, -708.5, 709.7, -745.1]])
    for x in np.concatenate([wedge, broad]):
        assert libdrs.drs_host_exp(float(x)) == m.exp(float(x)), x


def test_seedseq_restatement(libdrs):
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.rng import entropy_key
    for vals in [(0x7A9C, 0, 50, 2), (0x7A9C, 12345678901, 3, 1), (0x51DE, 0, 1), (0,), (5, 0, 0, 0),
                 (0x7A9C, 0xFFFFFFFFFFFF, 2 ** 40 + 3, 2)]:
        out = (ctypes.c_uint32 * 8)()
        assert libdrs.drs_host_seedseq(ctypes.byref(entropy_key(vals)), 0, out, 8) == _lib.DRS_OK
        ref = np.random.SeedSequence(vals).generate_state(8, np.uint32)
        assert list(out) == list(ref), vals


def test_seed_slot_masks_on_device_path(libdrs):
    from paper_2603_25872_b200.rng import entropy_key
    key = entropy_key((0x7A9C, 0, 9, 1), seed_slot=0, seed_mask=0xFFFFFFFFFFFF)
    out = (ctypes.c_uint32 * 8)()
    libdrs.drs_host_seedseq(ctypes.byref(key), (1 << 50) + 77, out, 8)
    ref = np.random.SeedSequence((0x7A9C, ((1 << 50) + 77) & 0xFFFFFFFFFFFF, 9, 1)).generate_state(8, np.uint32)
    assert list(out) == list(ref)


def test_generated_tables_current():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_tables.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_no_cpu_fallback_without_cuda(libdrs):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2603_25872_b200 import RngStream, Role, derive_noise
    with pytest.raises(RuntimeError, match="CUDA"):
        derive_noise(RngStream(0), 3, Role.INIT, 16)


def test_errors_hierarchy_matches_reference_names():
    import paper_2603_25872_b200.errors as E
    names = ["InvalidScheduleParams", "TimestepOutOfRange", "DimensionMismatch", "NonPositiveSigma",
             "InvalidSkip", "VarianceTooLarge", "IndexOutOfRange", "InvalidSubsequence", "InvalidPlanParams",
             "PlanMismatch", "WorkerFailure", "TimestepMismatch", "EmptySet", "InsufficientSamples",
             "ParseError", "ConfigError", "SuiteNotFound"]
    for n in names:
        assert issubclass(getattr(E, n), E.SkipDiffError)


def test_host_validation_errors():
    from paper_2603_25872_b200 import VarianceRule, build_linear_beta, ddim_skip_coeffs, plan_blocks, Mode
    from paper_2603_25872_b200.errors import InvalidPlanParams, InvalidSkip, TimestepOutOfRange, VarianceTooLarge
    s = build_linear_beta(4, 0.5, 0.5)
    c = ddim_skip_coeffs(s, 4, 2, VarianceRule.deterministic())
    assert c.kappa == pytest.approx(0.8944271909999159, rel=1e-14)
    assert c.lam == pytest.approx(0.2763932022500210, rel=1e-13)
    c = ddim_skip_coeffs(s, 2, 1, VarianceRule.ddpm_induced())
    assert c.kappa == pytest.approx(0.4714045207910317, rel=1e-14)
    with pytest.raises(InvalidSkip):
        ddim_skip_coeffs(s, 2, 0, VarianceRule.deterministic())
    with pytest.raises(TimestepOutOfRange):
        ddim_skip_coeffs(s, 5, 1, VarianceRule.deterministic())

    class Huge(VarianceRule):
        def sigma(self, s, t, k):
            return 10.0
    with pytest.raises(VarianceTooLarge):
        ddim_skip_coeffs(build_linear_beta(10, 0.01, 0.1), 5, 2, Huge(VarianceRule.deterministic().kind))
    with pytest.raises(ValueError):
        VarianceRule.eta_scaled(1.5)
    with pytest.raises(InvalidPlanParams):
        plan_blocks(0, 3, Mode.AGGRESSIVE)
    with pytest.raises(InvalidPlanParams):
        plan_blocks(10, 0, Mode.CONSERVATIVE)

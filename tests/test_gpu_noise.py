"""K1 device noise vs the reference's numpy streams, bit-exact."""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _gold_streams(golden_dir, gen):
    z = np.load(os.path.join(golden_dir, "noise.npz"))
    meta = json.loads(str(z[f"{gen}_meta"]))
    vals, off = z[f"{gen}_values"], 0
    for m in meta:
        yield tuple(m["key"]), m["n"], vals[off:off + m["n"]]
        off += m["n"]


def _fill(keys, n, gen, device):
    from paper_2603_25872_b200.rng import _check_err, entropy_key, fill_streams
    out = torch.full((len(keys), n), float("nan"), dtype=torch.float64, device=device)
    err = fill_streams([entropy_key(k) for k in keys], n, out, gen)
    _check_err(err)
    return out.cpu().numpy()


def _np_stream(key, n, gen):
    if gen == "pcg64":
        return np.random.default_rng(key).standard_normal(n)
    return np.random.Generator(np.random.SFC64(np.random.SeedSequence(key))).standard_normal(n)


@pytest.fixture(params=[1, 0], ids=["parallel_resolve", "serial_resolve"])
def resolve_mode(request, cuda):
    """Both chain resolvers of K1 (drs_set_noise_resolve): they must give the same bits."""
    from paper_2603_25872_b200 import _lib
    _lib.check(_lib.lib().drs_set_noise_resolve(request.param), "drs_set_noise_resolve")
    yield request.param
    _lib.check(_lib.lib().drs_set_noise_resolve(1), "drs_set_noise_resolve")


@pytest.mark.parametrize("gen", ["pcg64", "sfc64"])
def test_golden_streams_bit_exact(cuda, golden_dir, gen, resolve_mode):
    """Golden streams cover every ziggurat path: fast, wedge accept / reject, tail, tail retry."""
    for key, n, ref in _gold_streams(golden_dir, gen):
        got = _fill([key], n, gen, cuda)[0]
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (key, np.flatnonzero(got != ref)[:5])


@pytest.mark.parametrize("gen", ["pcg64", "sfc64"])
@pytest.mark.parametrize("n", [1, 31, 2239, 2240, 2241, 4096, 16384, 65536])
def test_random_keys_vs_numpy(cuda, gen, n, resolve_mode):
    rng = np.random.default_rng(n)
    keys = [(0x7A9C, int(rng.integers(0, 2 ** 48)), int(rng.integers(0, 300)), int(rng.integers(0, 3)))
            for _ in range(8 if n > 10000 else 24)]
    got = _fill(keys, n, gen, cuda)
    for i, k in enumerate(keys):
        ref = _np_stream(k, n, gen)
        assert np.array_equal(got[i].view(np.uint64), ref.view(np.uint64)), (k, n)


def test_many_streams_one_launch(cuda):
    # a C4-sized noise table: 445 streams x 4096 in one launch
    keys = [(0x7A9C, 3, t, r) for t in range(250) for r in (0, 1)][:445]
    got = _fill(keys, 4096, "pcg64", cuda)
    for i in range(0, 445, 7):
        assert np.array_equal(got[i], _np_stream(keys[i], 4096, "pcg64"))


def test_derive_noise_api(cuda):
    from paper_2603_25872_b200 import RngStream, Role, derive_noise, state_independent_eps
    x = derive_noise(RngStream(seed=5), 50, Role.INIT, (1, 4, 32, 32), device=cuda)
    assert x.shape == (1, 4, 32, 32) and x.dtype == torch.float64
    ref = np.random.default_rng((0x7A9C, 5, 50, 2)).standard_normal((1, 4, 32, 32))
    assert np.array_equal(x.cpu().numpy(), ref)
    # seed is masked to 48 bits (rng.py:32)
    y = derive_noise(RngStream(seed=(1 << 60) + 5), 50, Role.INIT, 4096, device=cuda)
    assert np.array_equal(y.cpu().numpy(), ref.reshape(-1))
    si = state_independent_eps(0, 1, 2, device=cuda).cpu().numpy()
    np.testing.assert_allclose(si, [0.6596311229815894, -1.0995664042571076], rtol=1e-15)
    with pytest.raises(ValueError):
        derive_noise(RngStream(0), -1, Role.INIT, 3, device=cuda)
    z = derive_noise(RngStream(7, generator="sfc64"), 3, Role.DRAFT, 1000, device=cuda)
    assert np.array_equal(z.cpu().numpy(), _np_stream((0x7A9C, 7, 3, 1), 1000, "sfc64"))

"""Samplers and schedulers on device vs the reference (golden SHA pins) and the
oracle; reference test-suite laws (tests/test_parallel.py) on the B200 path."""

import hashlib
import json
import math
import os

import numpy as np
import pytest
import torch

import skipdiff_oracle as O

pytestmark = pytest.mark.gpu

import paper_2603_25872_b200 as P  # noqa: E402


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _np(t):
    return t.detach().cpu().numpy()


def _ident(a, b):
    return a.timesteps() == b.timesteps() and all(
        torch.equal(xa, xb) for (_, xa), (_, xb) in zip(a.states, b.states))


def _gm_toy(D):
    m = np.zeros((2, D))
    m[0, 0], m[1, 0] = -2.0, 2.0
    return P.GaussianMixture(weights=[0.5, 0.5], means=m, variances=[1.0, 1.0])


def _run_case(m, cuda, generator="pcg64"):
    T, D = m["T"], m["D"]
    s = P.default_schedule(T)
    rule = P.VarianceRule.deterministic() if m["rule"] == "det" else P.VarianceRule.ddpm_induced()
    den = P.StateIndependent(seed=m["si_seed"], dim=D) if m["denoiser"] == "si" else P.AnalyticEps(_gm_toy(D))
    stream = P.RngStream(seed=m["seed"], generator=generator)
    x_T = P.derive_noise(P.RngStream(m["seed"]), T, P.Role.INIT, D, device=cuda)
    if m["sampler"] == "aggressive":
        traj, rep = P.run_aggressive(s, den, x_T, m["devices"], rule, stream, update_family=m["family"])
    elif m["sampler"] == "conservative":
        traj, rep = P.run_conservative(s, den, x_T, m["devices"], rule, stream, update_family=m["family"])
    elif m["sampler"] == "seq_ddim":
        traj, rep = P.sample_ddim(s, den, x_T, rule, stream), []
    else:
        traj, rep = P.sample_ddpm(s, den, x_T, stream), []
    return traj, rep


def test_golden_trajectories(cuda, golden_dir):
    """SI denoiser: every state bit-identical to the reference run (sha256 of
    each state).  GM denoiser: the squared-distance reduction order differs
    from numpy's pairwise sum (and numpy's SIMD log/exp are host-dependent),
    so d2 ~ 4e3 carries ~1e-13 absolute rounding that the softmax turns into
    ~1e-13 relative eps error, amplified up to 1/sqrt(abar_T) ~ 360 along the
    trajectory: states are compared to the oracle per step within
    rel-L2 <= 1e-10 and max-abs <= 1e-9 (fp64)."""
    z = np.load(os.path.join(golden_dir, "traj.npz"))
    for m in json.loads(str(z["manifest"])):
        traj, rep = _run_case(m, cuda)
        assert traj.timesteps() == list(z[m["name"] + "_t"]), m["name"]
        assert traj.eval_count == m["eval_count"], m["name"]
        if m["rounds"]:
            assert len(rep) == m["rounds"]
        if m["denoiser"] == "si":
            assert [_sha(_np(x)) for _, x in traj.states] == list(z[m["name"] + "_sha"]), m["name"]
        else:
            ab = O.default_alpha_bar(m["T"])
            rule = ("det",) if m["rule"] == "det" else ("ddpm",)
            x_T = O.derive_noise(m["seed"], m["T"], O.INIT, m["D"])
            eps = O.toy_bimodal(m["D"])
            if m["sampler"] == "seq_ddim":
                ref = O.sample_ddim(ab, eps, x_T, rule, m["seed"])
            elif m["sampler"] == "seq_ddpm":
                ref = O.sample_ddpm(ab, eps, x_T, m["seed"])
            else:
                ref, _, _ = O.run_parallel(ab, eps, x_T, m["devices"], m["sampler"], rule, m["seed"],
                                           family=m["family"])
            assert _sha(ref[-1][1]) == _sha(z[m["name"] + "_final"])   # oracle == reference here
            for (_, g), (_, r) in zip(traj.states, ref):
                g = _np(g)
                rel = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)
                assert rel <= 1e-10 and np.max(np.abs(g - r)) <= 1e-9, (m["name"], rel)


@pytest.mark.parametrize("family", ["ddim", "ddpm"])
def test_sfc64_variant_matches_oracle(cuda, family):
    """C2's SFC64 noise stream: SI bit-exact vs the oracle's numpy SFC64 run."""
    T, D, n = 50, 4096, 3
    s, ab = P.default_schedule(T), O.default_alpha_bar(T)
    x_T = O.derive_noise(4, T, O.INIT, D, "sfc64")
    traj, _ = P.run_aggressive(s, P.StateIndependent(11, D), torch.from_numpy(x_T).to(cuda), n,
                               P.VarianceRule.ddpm_induced(), P.RngStream(4, "sfc64"), update_family=family)
    ref, _, _ = O.run_parallel(ab, O.SI(11, D), x_T, n, "aggressive", ("ddpm",), 4, family=family,
                               generator="sfc64")
    for (_, g), (_, r) in zip(traj.states, ref):
        assert np.array_equal(_np(g), r)


@pytest.mark.parametrize("T", [8, 20, 50])
@pytest.mark.parametrize("devices", [1, 2, 3, 4])
@pytest.mark.parametrize("rule", ["det", "ddpm"])
def test_equivalence_grid(cuda, T, devices, rule):
    """reference tests/test_parallel.py:94-107 on device."""
    s = P.default_schedule(T)
    r = P.VarianceRule.deterministic() if rule == "det" else P.VarianceRule.ddpm_induced()
    den = P.StateIndependent(seed=11, dim=2)
    stream = P.RngStream(seed=T)
    x_T = P.derive_noise(stream, T, P.Role.INIT, 2, device=cuda)
    seq = P.sample_ddim(s, den, x_T, r, stream)
    agg, _ = P.run_aggressive(s, den, x_T, devices, r, stream)
    con, _ = P.run_conservative(s, den, x_T, devices, r, stream)
    assert _ident(agg, seq) and _ident(con, seq)
    ref = O.sample_ddim(O.default_alpha_bar(T), O.SI(11, 2), _np(x_T), ("det",) if rule == "det" else ("ddpm",), T)
    assert all(np.array_equal(_np(g), rr) for (_, g), (_, rr) in zip(seq.states, ref))


def test_ddpm_family_equivalence(cuda):
    s = P.default_schedule(50)
    den = P.StateIndependent(seed=7, dim=1)
    stream = P.RngStream(seed=1)
    x_T = P.derive_noise(stream, 50, P.Role.INIT, 1, device=cuda)
    seq = P.sample_ddpm(s, den, x_T, stream)
    for devices in (1, 3):
        agg, _ = P.run_aggressive(s, den, x_T, devices, P.VarianceRule.deterministic(), stream, update_family="ddpm")
        con, _ = P.run_conservative(s, den, x_T, devices, P.VarianceRule.deterministic(), stream,
                                    update_family="ddpm")
        assert _ident(agg, seq) and _ident(con, seq)


@pytest.mark.parametrize("T", [8, 20, 50])
@pytest.mark.parametrize("devices", [1, 2, 3, 4])
def test_eval_and_round_laws(cuda, T, devices):
    s = P.default_schedule(T)
    den = P.Counting(P.StateIndependent(seed=3, dim=1))
    stream = P.RngStream(seed=9)
    x_T = P.derive_noise(stream, T, P.Role.INIT, 1, device=cuda)
    ta, ra = P.run_aggressive(s, den, x_T, devices, P.VarianceRule.deterministic(), stream)
    assert den.count == ta.eval_count == T + 1
    assert len(ra) == 1 + math.ceil(T / devices)
    den.count = 0
    tc, rc = P.run_conservative(s, den, x_T, devices, P.VarianceRule.deterministic(), stream)
    assert den.count == tc.eval_count == T
    assert len(rc) == 2 * math.ceil(T / (devices + 1))


def test_recompute_anchor_ablation(cuda):
    s = P.default_schedule(50)
    gm = P.GaussianMixture(weights=[0.5, 0.5], means=[[-2.0], [2.0]], variances=[1.0, 1.0])
    den = P.AnalyticEps(gm)
    stream = P.RngStream(seed=5)
    x_T = P.derive_noise(stream, 50, P.Role.INIT, 1, device=cuda)
    rule = P.VarianceRule.deterministic()
    base, _ = P.run_aggressive(s, den, x_T, 3, rule, stream)
    fresh, reports = P.run_aggressive(s, den, x_T, 3, rule, stream, recompute_anchor_eps=True)
    blocks = P.plan_blocks(50, 3, P.Mode.AGGRESSIVE).blocks
    interior = sum(1 for t, _ in blocks if t != 50)
    assert fresh.eval_count == 51 + interior
    assert len(reports) == 1 + len(blocks) + interior
    assert not torch.equal(base.final, fresh.final)


def test_virtual_clock_round_laws(cuda):
    """reference tests/test_parallel.py:312-346: 17 / 24 rounds and T evals."""
    T, eval_ms = 48, 50.0
    s = P.default_schedule(T)
    den = P.Latency(P.StateIndependent(seed=1, dim=1), P.LatencyModel(eval_time_ms=eval_ms))
    stream = P.RngStream(seed=0)
    x_T = P.derive_noise(stream, T, P.Role.INIT, 1, device=cuda)
    clock = P.VirtualClock()
    traj, reps = P.run_aggressive(s, den, x_T, 3, P.VarianceRule.deterministic(), stream, clock=clock)
    assert traj.wall_ms == len(reps) * eval_ms == 17 * eval_ms
    clock = P.VirtualClock()
    traj, reps = P.run_conservative(s, den, x_T, 3, P.VarianceRule.deterministic(), stream, clock=clock)
    assert traj.wall_ms == len(reps) * eval_ms == 24 * eval_ms
    clock = P.VirtualClock()
    traj = P.sample_ddim(s, den, x_T, P.VarianceRule.deterministic(), stream, clock=clock)
    assert traj.wall_ms == T * eval_ms


def test_execute_round_semantics(cuda):
    s = P.default_schedule(50)
    den = P.StateIndependent(seed=2, dim=1)
    tasks = [(torch.zeros(1, dtype=torch.float64, device=cuda), t) for t in (9, 5, 7)]
    vals, report = P.execute_round(den, s, tasks, 3, anchor_t=9, submit_order=[2, 0, 1])
    for v, (_, t) in zip(vals, tasks):
        assert torch.equal(v, P.state_independent_eps(2, t, 1, device=cuda))
    assert report.parallel_evals == 3 and len(report.worker_spans) == 3
    with pytest.raises(P.InvalidPlanParams):
        P.execute_round(den, s, tasks, 2, anchor_t=9)
    gm = P.GaussianMixture(weights=[0.5, 0.5], means=[[-2.0], [2.0]], variances=[1.0, 1.0])
    bad = [(torch.zeros(1, dtype=torch.float64, device=cuda), 5), (torch.zeros(2, dtype=torch.float64, device=cuda), 5)]
    with pytest.raises(P.WorkerFailure):
        P.execute_round(P.AnalyticEps(gm), s, bad, 2, anchor_t=5)
    lat = P.Latency(P.AnalyticEps(gm), P.LatencyModel(eval_time_ms=40.0, dispatch_overhead_ms=2.0))
    clock = P.VirtualClock()
    _, rep = P.execute_round(lat, s, tasks, 3, anchor_t=9, clock=clock)
    assert rep.round_wall_ms == 42.0 and clock.elapsed_ms == 42.0


def test_wall_is_max_not_sum(cuda):
    """Latency evals occupy the GPU concurrently: a round of 3 x 20 ms is ~20 ms."""
    s = P.default_schedule(50)
    gm = P.GaussianMixture(weights=[0.5, 0.5], means=[[-2.0], [2.0]], variances=[1.0, 1.0])
    den = P.Latency(P.AnalyticEps(gm), P.LatencyModel(eval_time_ms=20.0))
    tasks = [(torch.zeros(1, dtype=torch.float64, device=cuda), t) for t in (9, 5, 7)]
    _, rep = P.execute_round(den, s, tasks, 3, anchor_t=9)
    assert 20.0 <= rep.round_wall_ms < 0.7 * 60.0


def test_gm_batched_matches_rows(cuda):
    s = P.default_schedule(50)
    gm = P.GaussianMixture(weights=[0.5, 0.5], means=np.array([[-2.0, 0.0], [2.0, 0.0]]), variances=[1.0, 1.0])
    xs = np.random.default_rng(9).normal(0, 2, (8, 2))
    batch = _np(P.eps_oracle(gm, s, torch.from_numpy(xs).to(cuda), 13))
    ref = O.GM(gm.weights, gm.means, gm.variances)(O.default_alpha_bar(50), xs, 13)
    np.testing.assert_allclose(batch, ref, rtol=1e-13, atol=1e-15)
    for i in range(8):
        row = _np(P.eps_oracle(gm, s, torch.from_numpy(xs[i]).to(cuda), 13))
        assert np.array_equal(row, batch[i])
    with pytest.raises(P.TimestepOutOfRange):
        P.eps_oracle(gm, s, torch.from_numpy(xs).to(cuda), 51)


def test_graph_replay_matches_eager(cuda):
    """The captured single-rank program replays bit-identically for new seeds."""
    from paper_2603_25872_b200.engine import DeviceRun
    T, D = 50, 4096
    s = P.default_schedule(T)
    prog = P.build_parallel(s, P.plan_blocks(T, 3, P.Mode.AGGRESSIVE), P.VarianceRule.deterministic(), "ddpm")
    run = DeviceRun(prog, s, P.AnalyticEps(_gm_toy(D)), D, cuda, generator="sfc64")
    finals = {}
    for seed in (0, 1, 2):
        x = P.derive_noise(P.RngStream(seed), T, P.Role.INIT, D, device=cuda)
        run.set_inputs(x, seed)
        run.enqueue()
        finals[seed] = run.traj[-1].clone()
    run.capture()
    for seed in (2, 0, 1):
        x = P.derive_noise(P.RngStream(seed), T, P.Role.INIT, D, device=cuda)
        run.set_inputs(x, seed)
        run.replay()
        torch.cuda.synchronize()
        assert torch.equal(run.traj[-1], finals[seed])
    run.check_err()


@pytest.mark.parametrize("rule", ["det", "ddpm", "eta"])
def test_ddim_subsequence_vs_oracle(cuda, rule):
    """f4 ablation: DDIM along a timestep subsequence (sequential.py:79-113) on
    device, SI denoiser: every state bit-identical to the oracle (z of the
    transition into u is key (u, TRANSITION), skip k = t - u)."""
    T, D, sub = 50, 4096, [20, 15, 9, 4, 0]
    s, ab = P.default_schedule(T), O.default_alpha_bar(T)
    r = {"det": P.VarianceRule.deterministic(), "ddpm": P.VarianceRule.ddpm_induced(),
         "eta": P.VarianceRule.eta_scaled(0.5)}[rule]
    orule = {"det": ("det",), "ddpm": ("ddpm",), "eta": ("eta", 0.5)}[rule]
    x = O.derive_noise(6, 20, O.INIT, D)
    traj = P.sample_ddim(s, P.StateIndependent(11, D), torch.from_numpy(x).to(cuda), r, P.RngStream(6),
                         subsequence=sub)
    ref = O.sample_ddim(ab, O.SI(11, D), x, orule, 6, subsequence=sub)
    assert traj.timesteps() == sub == [t for t, _ in ref]
    for (_, g), (_, rr) in zip(traj.states, ref):
        assert np.array_equal(_np(g), rr)
    with pytest.raises(P.InvalidSubsequence):
        P.sample_ddim(s, P.StateIndependent(11, D), torch.from_numpy(x).to(cuda), r, P.RngStream(6),
                      subsequence=[20, 20, 0])


@pytest.mark.parametrize("T,devices,mode", [(100, 40, "aggressive"), (100, 65, "conservative")])
def test_long_chain_runs_bit_exact(cuda, T, devices, mode):
    """> 64-op refine+draft chains run as several launches (advisor r1) and stay
    bit-identical to the oracle (SI eps, stochastic DDIM rule)."""
    D = 256
    s, ab = P.default_schedule(T), O.default_alpha_bar(T)
    x = O.derive_noise(3, T, O.INIT, D)
    run = P.run_aggressive if mode == "aggressive" else P.run_conservative
    traj, reps = run(s, P.StateIndependent(5, D), torch.from_numpy(x).to(cuda), devices,
                     P.VarianceRule.ddpm_induced(), P.RngStream(3), workers=0)
    ref, evals, rounds = O.run_parallel(ab, O.SI(5, D), x, devices, mode, ("ddpm",), 3)
    assert traj.eval_count == evals and len(reps) == rounds
    for (_, g), (_, r) in zip(traj.states, ref):
        assert np.array_equal(_np(g), r)


@pytest.mark.parametrize("n_comp", [1, 8, 9, 13, 40])
def test_gm_eps_many_components(cuda, n_comp):
    """K9 accepts any mixture size up to DRS_GM_MAX_COMP (advisor r1: it stopped
    at 8): components are reduced 8 per sweep; vs the oracle within fp64 rounding."""
    rng = np.random.default_rng(n_comp)
    D, T = 5000, 50
    w = rng.random(n_comp)
    w /= w.sum()
    means = rng.normal(size=(n_comp, D)) * 0.3
    var = rng.random(n_comp) + 0.5
    gm = P.GaussianMixture(weights=w, means=means, variances=var)
    s, ab = P.default_schedule(T), O.default_alpha_bar(T)
    x = rng.normal(size=(3, D))
    for t in (1, 17, 50):
        got = _np(P.eps_oracle(gm, s, torch.from_numpy(x).to(cuda), t))
        ref = O.gm_eps(w, means, var, ab, x, t)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel <= 1e-11, (n_comp, t, rel)
    with pytest.raises(ValueError):
        P.GaussianMixture(weights=np.full(2000, 1 / 2000), means=np.zeros((2000, 1)), variances=np.ones(2000))


def test_execute_round_perturbed_network_eps(cuda):
    """Perturbed over a NetworkEps (fp32 eps) in execute_round: the perturbation
    runs on an fp64 copy (advisor r1: it used to treat the fp32 row as fp64)."""
    from paper_2603_25872_b200.unet import UNet, sd15_config
    net = UNet(sd15_config(32), cuda, seed=0, max_batch=1)
    s = P.default_schedule(20)
    base = P.NetworkEps(net, (4, 32, 32))
    x = torch.randn(4096, dtype=torch.float64, device=cuda)
    (e0,), _ = P.execute_round(base, s, [(x, 7)], 1, anchor_t=7)
    (e1,), _ = P.execute_round(P.Perturbed(base, 0.25), s, [(x, 7)], 1, anchor_t=7)
    assert e1.dtype == torch.float64 and e1.shape == e0.shape
    want = e0.double() + 0.25 * torch.from_numpy(O.perturbation(_np(x), 7, 1.0)).to(cuda)
    assert torch.allclose(e1, want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("n_comp", [1, 2, 11])
def test_x0_posterior_mean_vs_oracle(cuda, n_comp):
    """x0_posterior_mean (denoiser.py:110-121) on device (K9 posterior-mean mode)."""
    rng = np.random.default_rng(n_comp + 7)
    D = 300
    w = rng.random(n_comp)
    w /= w.sum()
    means, var = rng.normal(size=(n_comp, D)), rng.random(n_comp) + 0.3
    gm = P.GaussianMixture(weights=w, means=means, variances=var)
    x = rng.normal(size=(4, D))
    for abar in (1.0, 0.25, 1e-3):
        got = _np(P.x0_posterior_mean(gm, torch.from_numpy(x).to(cuda), abar))
        ref = O.gm_x0_mean(w, means, var, x, abar)
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12, (n_comp, abar)
    with pytest.raises(ValueError):
        P.x0_posterior_mean(gm, torch.from_numpy(x).to(cuda), 0.0)


def test_derive_override_feeds_sequential_samplers(cuda):
    """A RngStream subclass overriding derive() supplies the sequential
    samplers' z (sequential.py:72,109 call noise.derive): called once per
    step in the reference order, and the samples use its values."""
    calls = []

    class Audit(P.RngStream):
        def derive(self, t, role, shape, *, device=None):
            calls.append((t, P.Role(role)))
            return 2.0 * super().derive(t, role, shape, device=device)     # visibly different noise

    s, D = P.default_schedule(20), 64
    x = torch.from_numpy(O.derive_noise(1, 20, O.INIT, D)).to(cuda)
    den = P.StateIndependent(3, D)
    traj = P.sample_ddim(s, den, x, P.VarianceRule.ddpm_induced(), Audit(seed=1))
    assert calls == [(u, P.Role.TRANSITION) for u in range(19, -1, -1)]
    plain = P.sample_ddim(s, den, x, P.VarianceRule.ddpm_induced(), P.RngStream(1))
    assert not torch.equal(traj.final, plain.final)
    ab = O.default_alpha_bar(20)
    xr, ref = _np(x), [(20, _np(x))]
    for t in range(20, 0, -1):
        z = 2.0 * O.derive_noise(1, t - 1, O.TRANSITION, D)
        xr = O.ddim_skip(ab, t, 1, xr, O.SI(3, D)(ab, xr, t), ("ddpm",), z)
        ref.append((t - 1, xr))
    for (_, g), (_, r) in zip(traj.states, ref):
        assert np.array_equal(_np(g), r)
    calls.clear()
    P.sample_ddpm(s, den, x, Audit(seed=1))
    assert calls == [(t - 1, P.Role.TRANSITION) for t in range(20, 0, -1)]


def test_realtime_speedup_laws_spin_latency(cuda):
    """Real-time latency-law calibration (reference tests/test_acceptance.py:164-203,
    SURVEY 8(d)): the Latency denoiser occupies the GPU for eval_time_ms per round
    (drs_spin, all tasks of a round concurrently), T = 48; measured wall-clock
    speedup of both schedulers >= 0.9x the round law T/rounds for devices 2..4,
    and aggressive devices = 3 >= 2.5x.  Host wall clock around the public call,
    min over 2 repeats, as the reference."""
    import time
    T, eval_ms = 48, 20.0
    s = P.default_schedule(T)
    den = P.Latency(P.AnalyticEps(P.standard_normal_mixture(1)),
                    P.LatencyModel(eval_time_ms=eval_ms, dispatch_overhead_ms=0.2))
    rule, stream = P.VarianceRule.deterministic(), P.RngStream(seed=0)
    x_T = P.derive_noise(stream, T, P.Role.INIT, 1, device=cuda)

    def timed(fn, repeats=2):
        best = math.inf
        for _ in range(repeats):
            torch.cuda.synchronize()
            t0 = time.monotonic()
            fn()
            torch.cuda.synchronize()
            best = min(best, (time.monotonic() - t0) * 1000.0)
        return best

    timed(lambda: P.run_aggressive(s, den, x_T, 2, rule, stream), 1)           # build + warm the programs
    seq_ms = timed(lambda: P.sample_ddim(s, den, x_T, rule, stream))
    assert seq_ms >= T * eval_ms
    fails = []
    for devices in (2, 3, 4):
        for runner, rounds in ((P.run_aggressive, 1 + math.ceil(T / devices)),
                               (P.run_conservative, 2 * math.ceil(T / (devices + 1)))):
            timed(lambda: runner(s, den, x_T, devices, rule, stream), 1)
            par_ms = timed(lambda: runner(s, den, x_T, devices, rule, stream))
            speedup, theory = seq_ms / par_ms, T / rounds
            if speedup < 0.9 * theory:
                fails.append((runner.__name__, devices, speedup, theory))
            if runner is P.run_aggressive and devices == 3:
                assert speedup >= 2.5, speedup
    assert not fails, fails

"""Generate the golden fixtures by running the REFERENCE itself.

    python tests/golden/make_golden.py

Imports skipdiff from /root/reference/pkg/src (read-only, this container only;
the reference does not travel to the GPU box) and writes:
  noise.npz  normal streams of chosen keys, PCG64 (the reference's rng.py:32
             path) and the SFC64 variant of the same SeedSequence keys, with
             the ziggurat path counts of each stream (keys chosen so wedge
             rejections, tails and a tail retry all occur);
  traj.npz   sha256 of every trajectory state (bit-exact pin) + selected
             final states for the BASELINE configs' sampler shapes with the
             state-independent and Gaussian-mixture toy denoisers;
  plans.json plan_blocks for every config;
  euler.npz  Euler family (next-row scope): sigma grids, velocity_oracle
             values, and sequential / parallel Euler trajectories (sha256 of
             every state, finals, eval counts, rounds) of the reference;
  cli/       the reference CLI's own output files (samples CSV, rounds CSV,
             JSON report) for the configs cli/*.cfg, written by its
             `sample` command in a scratch directory;
  perturb.npz Perturbed-denoiser ablation: BLAKE2b digests and
             _perturbation draws of seeded states, and Perturbed(SI)
             trajectories (sha256 per state) of the parallel schedulers;
  metrics.json sliced_w2 / mmd_gaussian / mmd_permutation_threshold of the
             reference on seeded sample sets (inputs regenerated from the
             seeds by metric_inputs()).
Run on numpy 2.3.5 / scipy 1.18.1 / glibc 2.39 (FMA libm variant).
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))

import noise_restated  # noqa: E402
import skipdiff as sd  # noqa: E402

NOISE_KEYS = [
    # (key tuple, n)
    ((0x7A9C, 0, 50, 2), 4096),             # INIT of seed 0, T=50
    ((0x7A9C, 12345678901, 3, 1), 4096),    # two-word seed, DRAFT role, a tail
    ((0x7A9C, 0xFFFFFFFFFFFF, 0, 0), 4096),  # max 48-bit seed, t=0 (word 0)
    ((0x51DE, 0, 1), 4096),                 # state_independent_eps(0, 1, .) (denoiser.py:144)
    ((0x51DE, 11, 250), 1),                 # n = 1
    ((0x7A9C, 7, 30, 0), 32768),            # multi-tile stream, several tails
]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def find_tail_retry_key(gen):
    for seed in range(2000):
        key = (0x7A9C, seed, 17, 0)
        _, paths = noise_restated.draw(key, 4096, gen)
        if any("tail-retry" in p for p in paths):
            return key
    raise RuntimeError("no tail retry found")


def noise_fixture():
    out = {}
    for gen in ("pcg64", "sfc64"):
        keys = list(NOISE_KEYS) + [(find_tail_retry_key(gen), 4096)]
        streams, meta = [], []
        for key, n in keys:
            if gen == "pcg64":
                v = np.random.default_rng(key).standard_normal(n)
            else:
                v = np.random.Generator(np.random.SFC64(np.random.SeedSequence(key))).standard_normal(n)
            _, paths = noise_restated.draw(key, n, gen)
            counts = {}
            for p in paths:
                for x in p:
                    counts[x] = counts.get(x, 0) + 1
            streams.append(v)
            meta.append({"key": list(key), "n": n, "paths": counts})
        out[f"{gen}_values"] = np.concatenate(streams)
        out[f"{gen}_meta"] = np.array(json.dumps(meta))
    # the only PRNG output the reference's own tests pin (test_denoiser.py:162-165)
    out["si_golden_0_1_2"] = sd.state_independent_eps(0, 1, 2)
    np.savez_compressed(os.path.join(HERE, "noise.npz"), **out)


def gm_toy(dim):
    m = np.zeros((2, dim))
    m[0, 0], m[1, 0] = -2.0, 2.0
    return sd.GaussianMixture(weights=[0.5, 0.5], means=m, variances=[1.0, 1.0])


CASES = [
    # name, T, D, sampler, devices, family, rule, denoiser, keep_final
    ("c1_si_det", 50, 4096, "conservative", 2, "ddim", "det", "si", True),
    ("c1_si_ddpmrule", 50, 4096, "conservative", 2, "ddim", "ddpm", "si", True),
    ("c1_gm_det", 50, 4096, "conservative", 2, "ddim", "det", "gm", True),
    ("c1_gm_ddpmrule", 50, 4096, "conservative", 2, "ddim", "ddpm", "gm", True),
    ("c1_seq_gm_det", 50, 4096, "seq_ddim", 1, "ddim", "det", "gm", True),
    ("c2_si", 50, 4096, "aggressive", 3, "ddpm", "det", "si", True),
    ("c2_gm", 50, 4096, "aggressive", 3, "ddpm", "det", "gm", True),
    ("c2_seq_gm", 50, 4096, "seq_ddpm", 1, "ddpm", "det", "gm", True),
    ("c3_si_n2", 50, 16384, "aggressive", 2, "ddim", "det", "si", False),
    ("c3_si_n4", 50, 16384, "aggressive", 4, "ddim", "det", "si", False),
    ("c3_si_n8", 50, 16384, "aggressive", 8, "ddim", "det", "si", False),
    ("c4_si", 250, 4096, "conservative", 8, "ddpm", "det", "si", True),
    ("c5_si", 30, 65536, "aggressive", 8, "ddim", "det", "si", False),
]


def traj_fixture():
    out, manifest = {}, []
    for name, T, D, sampler, n, fam, rule_s, den_s, keep in CASES:
        s = sd.default_schedule(T)
        rule = sd.VarianceRule.deterministic() if rule_s == "det" else sd.VarianceRule.ddpm_induced()
        den = sd.StateIndependent(seed=11, dim=D) if den_s == "si" else sd.AnalyticEps(gm_toy(D))
        stream = sd.RngStream(seed=0)
        x_T = sd.derive_noise(stream, T, sd.Role.INIT, D)
        if sampler == "aggressive":
            traj, rep = sd.run_aggressive(s, den, x_T, n, rule, stream, update_family=fam)
        elif sampler == "conservative":
            traj, rep = sd.run_conservative(s, den, x_T, n, rule, stream, update_family=fam)
        elif sampler == "seq_ddim":
            traj, rep = sd.sample_ddim(s, den, x_T, rule, stream), []
        else:
            traj, rep = sd.sample_ddpm(s, den, x_T, stream), []
        out[f"{name}_sha"] = np.array([_sha(x) for _, x in traj.states])
        out[f"{name}_t"] = np.array(traj.timesteps())
        if keep:
            out[f"{name}_final"] = traj.final
        manifest.append({"name": name, "T": T, "D": D, "sampler": sampler, "devices": n, "family": fam,
                         "rule": rule_s, "denoiser": den_s, "seed": 0, "si_seed": 11,
                         "eval_count": traj.eval_count, "rounds": len(rep)})
    out["manifest"] = np.array(json.dumps(manifest))
    np.savez_compressed(os.path.join(HERE, "traj.npz"), **out)


def plans_fixture():
    plans = {}
    for T in (50, 250, 30, 48, 10, 9, 5):
        for n in (1, 2, 3, 4, 8):
            for mode in sd.Mode:
                p = sd.plan_blocks(T, n, mode)
                plans[f"{T}_{n}_{mode.value}"] = {"blocks": [list(b) for b in p.blocks],
                                                  "rounds": p.total_rounds, "evals": p.total_evals}
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans, f, indent=0, sort_keys=True)


EULER_CASES = [
    # name, N, sigma_min, sigma_max, rho, dim, sampler, devices
    ("e16_1d_seq", 16, 0.02, 20.0, 7.0, 1, "seq", 1),
    ("e16_1d_agg3", 16, 0.02, 20.0, 7.0, 1, "aggressive", 3),
    ("e16_1d_con3", 16, 0.02, 20.0, 7.0, 1, "conservative", 3),
    ("e40_4096_seq", 40, 0.002, 80.0, 7.0, 4096, "seq", 1),
    ("e40_4096_agg4", 40, 0.002, 80.0, 7.0, 4096, "aggressive", 4),
    ("e40_4096_con4", 40, 0.002, 80.0, 7.0, 4096, "conservative", 4),
    ("e41_4096_agg8", 41, 0.002, 80.0, 7.0, 4096, "aggressive", 8),
    ("e9_4096_con8", 9, 0.01, 10.0, 3.0, 4096, "conservative", 8),
]


def euler_fixture():
    """x_init = sigma_max * derive_noise(INIT) as cli.py:46-47; mixture: the
    reference's bimodal_1d fixture (tests/conftest.py:17-19) generalised to dim
    as the configs' toy GM."""
    out, manifest = {}, []
    for name, N, smin, smax, rho, dim, sampler, n in EULER_CASES:
        g = sd.build_sigma_grid(N, smin, smax, rho)
        gm = gm_toy(dim)
        stream = sd.RngStream(seed=0)
        x0 = g.sigmas[0] * sd.derive_noise(stream, N, sd.Role.INIT, dim)
        if sampler == "seq":
            traj, rep = sd.sample_euler(g, gm, x0), []
        else:
            traj, rep = sd.run_parallel_euler(g, gm, x0, n, sd.Mode(sampler))
        out[f"{name}_sigmas"] = g.sigmas
        out[f"{name}_x0"] = x0
        out[f"{name}_sha"] = np.array([_sha(x) for _, x in traj.states])
        out[f"{name}_t"] = np.array(traj.timesteps())
        out[f"{name}_final"] = traj.final
        out[f"{name}_mid"] = traj.states[len(traj.states) // 2][1]
        manifest.append({"name": name, "N": N, "sigma_min": smin, "sigma_max": smax, "rho": rho, "dim": dim,
                         "sampler": sampler, "devices": n, "eval_count": traj.eval_count, "rounds": len(rep)})
    # velocity values: a state per sigma of the 4096-D grid
    g = sd.build_sigma_grid(40, 0.002, 80.0, 7.0)
    gm = gm_toy(4096)
    xs, vs = [], []
    for i in (0, 7, 20, 33, 39):
        x = g.sigmas[i] * sd.derive_noise(sd.RngStream(seed=5), i + 1, sd.Role.DRAFT, 4096)
        xs.append(x)
        vs.append(sd.velocity_oracle(gm, x, float(g.sigmas[i])))
    out["vel_sigmas"] = np.array([g.sigmas[i] for i in (0, 7, 20, 33, 39)])
    out["vel_x"] = np.array(xs)
    out["vel_v"] = np.array(vs)
    out["manifest"] = np.array(json.dumps(manifest))
    np.savez_compressed(os.path.join(HERE, "euler.npz"), **out)


from metric_cases import METRIC_CASES, metric_inputs  # noqa: E402


def metrics_fixture():
    vals = []
    for name, seed, (na, nb, dim), shift, P, wseed, bw in METRIC_CASES:
        a, b = metric_inputs(seed, na, nb, dim, shift)
        A, B = sd.SampleSet(a), sd.SampleSet(b)
        vals.append({"name": name, "seed": seed, "n_a": na, "n_b": nb, "dim": dim, "shift": shift,
                     "projections": P, "w2_seed": wseed, "bandwidth": bw,
                     "sliced_w2": sd.sliced_w2(A, B, projections=P, seed=wseed),
                     "mmd": sd.mmd_gaussian(A, B, bw),
                     "threshold": sd.mmd_permutation_threshold(A, B, bw, permutations=20, seed=wseed)})
    with open(os.path.join(HERE, "metrics.json"), "w") as f:
        json.dump(vals, f, indent=1)


PERTURB_TRAJ = [
    # name, T, D, sampler, devices, family, rule, scale, seed
    ("p_agg3", 20, 64, "aggressive", 3, "ddim", "ddpm", 0.05, 2),
    ("p_con4", 17, 256, "conservative", 4, "ddpm", "det", 0.2, 3),
    ("p_seq", 12, 64, "seq_ddim", 1, "ddim", "det", 0.1, 1),
]


def perturb_fixture():
    import hashlib as hl
    from skipdiff import denoiser as sdd
    out = {}
    rng = np.random.default_rng(99)
    xs, ts, digs, pert = [], [], [], []
    for i, (D, t) in enumerate([(1, 0), (5, 7), (64, 50), (1000, 3), (4096, 250)]):
        x = rng.normal(size=D) * (10.0 ** (i - 2))
        q = np.round(np.asarray(x, dtype=float) / sdd._PERTURB_QUANTUM).astype(np.int64)
        dig = hl.blake2b(sdd._PERTURB_SALT + int(t).to_bytes(8, "little", signed=True) + q.tobytes(),
                         digest_size=8).digest()
        out[f"x{i}"] = x
        out[f"pert{i}"] = sdd._perturbation(x, t, 0.3)
        ts.append(t)
        digs.append(int.from_bytes(dig, "little"))
    out["ts"] = np.array(ts)
    out["digests"] = np.array(digs, dtype=np.uint64)
    manifest = []
    for name, T, D, sampler, n, fam, rule_s, scale, seed in PERTURB_TRAJ:
        s_ = sd.default_schedule(T)
        rule = sd.VarianceRule.deterministic() if rule_s == "det" else sd.VarianceRule.ddpm_induced()
        den = sd.Perturbed(sd.StateIndependent(seed=11, dim=D), scale)
        stream = sd.RngStream(seed=seed)
        x_T = sd.derive_noise(stream, T, sd.Role.INIT, D)
        if sampler == "aggressive":
            traj, rep = sd.run_aggressive(s_, den, x_T, n, rule, stream, update_family=fam)
        elif sampler == "conservative":
            traj, rep = sd.run_conservative(s_, den, x_T, n, rule, stream, update_family=fam)
        else:
            traj, rep = sd.sample_ddim(s_, den, x_T, rule, stream), []
        out[f"{name}_sha"] = np.array([_sha(x) for _, x in traj.states])
        out[f"{name}_final"] = traj.final
        manifest.append({"name": name, "T": T, "D": D, "sampler": sampler, "devices": n, "family": fam,
                         "rule": rule_s, "scale": scale, "seed": seed, "si_seed": 11,
                         "eval_count": traj.eval_count, "rounds": len(rep)})
    out["manifest"] = np.array(json.dumps(manifest))
    np.savez_compressed(os.path.join(HERE, "perturb.npz"), **out)


def cli_fixture():
    import shutil
    import tempfile
    from skipdiff.cli import main as cli_main
    src = os.path.join(HERE, "cli")
    with tempfile.TemporaryDirectory() as tmp:
        for cfg in sorted(f for f in os.listdir(src) if f.endswith(".cfg")):
            shutil.copy(os.path.join(src, cfg), tmp)
            cwd = os.getcwd()
            os.chdir(tmp)
            try:
                assert cli_main(["sample", "--config", cfg]) == 0
            finally:
                os.chdir(cwd)
        for f in os.listdir(tmp):
            if not f.endswith(".cfg"):
                shutil.copy(os.path.join(tmp, f), src)


if __name__ == "__main__":
    cli_fixture()
    noise_fixture()
    traj_fixture()
    plans_fixture()
    euler_fixture()
    metrics_fixture()
    perturb_fixture()
    print("golden fixtures written to", HERE)

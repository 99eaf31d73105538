"""Per-step latent parity of NETWORK-driven sampler runs (BASELINE C3 / C4 / C5
configs at their full T) -- the north_star's "latents and final samples within a
stated fp32/bf16 tolerance (max-abs and relative-L2 per step)".

Device side: the product path -- `run_aggressive` / `run_conservative` /
`sample_ddim` / `sample_ddpm` with `NetworkEps` (bf16 tcgen05 network, fp32 eps,
fp64 sampler state, device PCG64 noise).
Oracle side: the restated reference sampler (`oracle/skipdiff_oracle.py`,
parallel.py:250-321 / sequential.py:57-113, numpy fp64 state, numpy noise)
driven by the plain fp32 torch network of the same weights (`oracle/nets_ref.py`)
evaluated on the same GPU with TF32 off -- the SURVEY 8(d)(ii) construction
(`skipdiff.{parallel,sequential}.evaluate` patched with an fp32 network).

Noise and timestep indexing are bit-exact (test_gpu_samplers.py), so every
difference below is the bf16 network's eps error propagated through the
sampler.  Tolerances are per trajectory state j:
    rel-L2(x_dev[j], x_ref[j])  <= REL[config]
    max-abs(x_dev[j] - x_ref[j]) <= ABS[config] * max|x_ref[j]|
The measured per-state values are printed (pytest -s); the round-2 log is
profiles/r2_net_trajectories.txt.
"""

import numpy as np
import pytest
import torch

import skipdiff_oracle as O

pytestmark = pytest.mark.gpu

import paper_2603_25872_b200 as P  # noqa: E402

# stated per-state tolerances; round-2 measured worst cases on a B200:
#   c3 (SD1.5, g = 7.5): rel-L2 2.5e-2 (sequential) .. 3.7e-2 (stochastic DDIM), max-abs 6.1e-2
#   c4 (DiT-XL/2, DDPM 250): rel-L2 2.1e-4, max-abs 2.1e-4
#   c5 (SDXL, g = 7.5):  rel-L2 2.9e-2, max-abs 2.8e-2
REL = {"c3": 6e-2, "c4": 1e-3, "c5": 6e-2}
ABS = {"c3": 1e-1, "c4": 1e-3, "c5": 6e-2}


def _no_tf32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False


def _fp32_eps(ref_fn, T, shape, dev, t_scale=None):
    """eps_fn(ab, x, t) for the oracle sampler: the fp32 torch net on the GPU."""
    scale = t_scale if t_scale is not None else 1000.0 / T

    def eps(ab, x, t):
        xt = torch.from_numpy(np.asarray(x, dtype=np.float32)).to(dev).reshape(1, *shape)
        tt = torch.tensor([t * scale], dtype=torch.float32, device=dev)
        with torch.no_grad():
            out = ref_fn(xt, tt)
        return out.reshape(-1).double().cpu().numpy()
    return eps


def _compare(cfg, traj, ref, stats=None):
    assert traj.timesteps() == [t for t, _ in ref]
    worst_rel, worst_abs = 0.0, 0.0
    rels = []
    for j, ((t, g), (_, r)) in enumerate(zip(traj.states, ref)):
        g = g.detach().cpu().numpy().reshape(-1)
        r = np.asarray(r).reshape(-1)
        rel = float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300))
        mab = float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))
        worst_rel, worst_abs = max(worst_rel, rel), max(worst_abs, mab)
        rels.append((t, round(rel, 6), round(mab, 6)))
    print(f"\n[{cfg}] per-state (t, rel-L2, max-abs/max|ref|): {rels}")
    for j, ((t, g), (_, r)) in enumerate(zip(traj.states, ref)):
        g = g.detach().cpu().numpy().reshape(-1)
        r = np.asarray(r).reshape(-1)
        rel = float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300))
        mab = float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))
        assert np.isfinite(g).all(), (cfg, t)
        assert rel <= REL[cfg], (cfg, "state", j, "t", t, "rel-L2", rel)
        assert mab <= ABS[cfg], (cfg, "state", j, "t", t, "max-abs/max|ref|", mab)
    print(f"\n[{cfg}] worst per-step rel-L2 {worst_rel:.3e}, max-abs/max|ref| {worst_abs:.3e} "
          f"over {len(ref)} states")
    if stats is not None:
        stats.append((cfg, worst_rel, worst_abs))
    return worst_rel, worst_abs


@pytest.fixture(scope="module")
def sd15(cuda):
    from paper_2603_25872_b200.unet import UNet, sd15_config
    _no_tf32()
    return UNet(sd15_config(64), cuda, seed=0, max_batch=4, cfg_scale=7.5)


@pytest.mark.parametrize("mode,n", [("sequential", 1), ("aggressive", 4), ("aggressive", 8)])
def test_c3_sd15_trajectory_vs_oracle(cuda, sd15, mode, n):
    """C3 shape (SD1.5 UNet, 4x64x64, CFG g = 7.5 as one batch-2 forward, DDIM
    deterministic) at the config's T = 50: aggressive n = 4 / 8 (batched drafts on one GPU;
    the same program the ranks run) and the sequential 1-GPU baseline."""
    from nets_ref import unet_ref
    T, shape = 50, (4, 64, 64)
    s, ab = P.default_schedule(T), O.default_alpha_bar(T)
    den = P.NetworkEps(sd15, shape)
    stream = P.RngStream(5)
    x_T = O.derive_noise(5, T, O.INIT, 16384)
    xd = torch.from_numpy(x_T).to(cuda)
    rule = P.VarianceRule.deterministic()
    eps = _fp32_eps(lambda x, t: unet_ref(sd15, x, t), T, shape, cuda)
    if mode == "sequential":
        traj = P.sample_ddim(s, den, xd, rule, stream)
        ref = O.sample_ddim(ab, eps, x_T, ("det",), 5)
    else:
        traj, reps = P.run_aggressive(s, den, xd, n, rule, stream)
        ref, evals, rounds = O.run_parallel(ab, eps, x_T, n, "aggressive", ("det",), 5)
        assert traj.eval_count == evals and len(reps) == rounds
    _compare("c3", traj, ref)


def test_c3_sd15_stochastic_ddim_vs_oracle(cuda, sd15):
    """C3 shape with the ddpm-induced (stochastic) DDIM rule: device PCG64 noise
    rows enter every draft and refine; aggressive n = 4, T = 50."""
    from nets_ref import unet_ref
    T, shape = 50, (4, 64, 64)
    s, ab = P.default_schedule(T), O.default_alpha_bar(T)
    x_T = O.derive_noise(9, T, O.INIT, 16384)
    traj, _ = P.run_aggressive(s, P.NetworkEps(sd15, shape), torch.from_numpy(x_T).to(cuda), 4,
                               P.VarianceRule.ddpm_induced(), P.RngStream(9))
    ref, _, _ = O.run_parallel(ab, _fp32_eps(lambda x, t: unet_ref(sd15, x, t), T, shape, cuda), x_T, 4,
                               "aggressive", ("ddpm",), 9)
    _compare("c3", traj, ref)


def test_c4_dit_conservative_trajectory_vs_oracle(cuda):
    """C4 config (DiT-XL/2, 4x32x32, DDPM family, T = 250, conservative n = 8):
    every state vs the oracle conservative run with the fp32 DiT, and the
    sequential DDPM baseline likewise (replaces round 1's self-consistency check)."""
    from nets_ref import dit_ref
    from paper_2603_25872_b200.dit import DiT, DiTConfig
    _no_tf32()
    T, shape = 250, (4, 32, 32)
    s, ab = P.default_schedule(T), O.default_alpha_bar(T)
    net = DiT(DiTConfig(), cuda, seed=1, max_batch=8)
    den = P.NetworkEps(net, shape)
    x_T = O.derive_noise(3, T, O.INIT, 4096)
    xd = torch.from_numpy(x_T).to(cuda)
    eps = _fp32_eps(lambda x, t: dit_ref(net.w, net.cfg, x, t), T, shape, cuda)
    traj, reps = P.run_conservative(s, den, xd, 8, P.VarianceRule.deterministic(), P.RngStream(3),
                                    update_family="ddpm")
    ref, evals, rounds = O.run_parallel(ab, eps, x_T, 8, "conservative", ("det",), 3, family="ddpm")
    assert traj.eval_count == evals == T and len(reps) == rounds
    _compare("c4", traj, ref)
    seq = P.sample_ddpm(s, den, xd, P.RngStream(3))
    _compare("c4", seq, O.sample_ddpm(ab, eps, x_T, 3))


def test_c5_sdxl_trajectory_vs_oracle(cuda):
    """C5 config (SDXL UNet, 4x128x128, CFG pair, DDIM T = 30, aggressive n = 8)."""
    from nets_ref import unet_ref
    from paper_2603_25872_b200.unet import UNet, sdxl_config
    _no_tf32()
    T, shape = 30, (4, 128, 128)
    s, ab = P.default_schedule(T), O.default_alpha_bar(T)
    net = UNet(sdxl_config(128), cuda, seed=0, max_batch=8, cfg_scale=7.5)
    x_T = O.derive_noise(2, T, O.INIT, 65536)
    traj, reps = P.run_aggressive(s, P.NetworkEps(net, shape), torch.from_numpy(x_T).to(cuda), 8,
                                  P.VarianceRule.deterministic(), P.RngStream(2))
    ref, evals, rounds = O.run_parallel(ab, _fp32_eps(lambda x, t: unet_ref(net, x, t), T, shape, cuda),
                                        x_T, 8, "aggressive", ("det",), 2)
    assert traj.eval_count == evals and len(reps) == rounds
    _compare("c5", traj, ref)

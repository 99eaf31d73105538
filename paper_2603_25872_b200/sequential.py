"""Single-stream samplers: the 1-GPU baseline the parallel schedulers are
measured against (skipdiff sequential.py:57-130), as device programs."""

from .parallel import _numel          # np.asarray semantics for array-like x_T
from .program import build_sequential
from .rng import RngStream
from .runner import Trajectory, execute, get_run, resolve_device
from .transitions import VarianceRule, predicted_x0_device


def predicted_x0(s, x_t, eps, t: int):
    """x0_hat = (x_t - sqrt(1-abar_t) eps) / sqrt(abar_t) (sequential.py:51-54)."""
    return predicted_x0_device(s, x_t, eps, t)




def _derived_rows(noise: RngStream, run, x_T):
    """The reference's sequential samplers draw z through the stream's own
    method, noise.derive(u, TRANSITION, x.shape) (sequential.py:72,109), so a
    RngStream subclass may override it.  When it does, the run's noise rows come
    from that method, called in the reference's order; otherwise the noise
    kernel generates them in-program (bit-identical to RngStream.derive)."""
    if type(noise).derive is RngStream.derive:
        return None
    from .rng import Role
    shape = tuple(getattr(x_T, "shape", ())) or (run.D,)
    return [noise.derive(t, Role(role), shape) for _, t, role in run.prog.noise_keys]


def sample_ddpm(s, d, x_T, noise: RngStream, clock=None) -> Trajectory:
    """Ancestral DDPM: T unit-step posterior transitions, z of step t from
    key (t-1, TRANSITION) (sequential.py:57-76)."""
    dev = resolve_device(x_T)
    rule = VarianceRule.deterministic()
    run = get_run(("seq", "ddpm", s.T), lambda: build_sequential(s, rule, "ddpm"),
                  s, d, _numel(x_T), dev, noise.generator, None)
    traj, _ = execute(run, x_T, noise.seed, clock, noise_rows=_derived_rows(noise, run, x_T))
    return traj


def sample_ddim(s, d, x_T, rule: VarianceRule, noise: RngStream, subsequence=None, clock=None) -> Trajectory:
    """DDIM along a timestep subsequence (default every step); the z of the
    transition into u is key (u, TRANSITION) (sequential.py:88-113)."""
    dev = resolve_device(x_T)
    sub = tuple(subsequence) if subsequence is not None else None
    run = get_run(("seq", "ddim", s.T, rule, sub), lambda: build_sequential(s, rule, "ddim", sub),
                  s, d, _numel(x_T), dev, noise.generator, None)
    traj, _ = execute(run, x_T, noise.seed, clock, noise_rows=_derived_rows(noise, run, x_T))
    return traj


def sample_euler(g, gm, x_init) -> Trajectory:
    """Plain Euler integration of dx/dsigma = (x - x0_hat)/sigma down the grid
    (sequential.py:116-130): N velocity evaluations (K9, VE mode) and N unit
    Euler steps (K3), one device program.  Trajectory timesteps count the
    remaining grid intervals (N at the start, 0 at the end)."""
    from .denoiser import euler_velocity_core
    from .program import build_sequential_euler
    dev = resolve_device(x_init)
    core = euler_velocity_core(gm, g)
    run = get_run(("seq", "euler", g.N), lambda: build_sequential_euler(g), g, core, _numel(x_init), dev,
                  "pcg64", None)
    traj, _ = execute(run, x_init, 0, None)
    return traj


__all__ = ["Trajectory", "predicted_x0", "sample_ddpm", "sample_ddim", "sample_euler"]

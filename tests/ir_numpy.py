"""Test-only numpy interpreter of sampler programs (paper_2603_25872_b200/program.py).

Executes a Program's steps exactly as engine.DeviceRun lowers them -- same
buffers, same task ownership, same op coefficients and the kernel's
expression order (csrc/chain.cu) -- but with numpy on the host and the
oracle's noise/eps.  Comparing it to the oracle sampler (a restatement of the
reference's _run) checks the schedule IR itself, including the multi-rank
partition + all-gather, on CPU.
"""

import numpy as np

import skipdiff_oracle as O
from paper_2603_25872_b200 import _lib
from paper_2603_25872_b200.program import Chain, Eval, Gather


def apply_op(op, x, e, z):
    c = op.c
    if op.family == _lib.FAMILY_DDIM:
        x0 = (x - c[0] * e) / c[1]
        y = c[2] * x0 + c[3] * e
        if op.noisy:
            y = y + c[4] * z
    elif op.family in (_lib.FAMILY_DDPM, _lib.FAMILY_DDPM_X0):
        x0 = (x - c[0] * e) / c[1] if op.family == _lib.FAMILY_DDPM else e
        y = (c[2] * x + c[3] * x0) / c[4]
        if op.noisy:
            y = y + c[5] * z
    elif op.family == _lib.FAMILY_PRED_X0:
        y = (x - c[0] * e) / c[1]
    else:
        y = x + c[0] * e
    return y


def run_ir(prog, ab, eps_fn, x_T, seed, generator="pcg64", rank=0, allgather=None):
    """Returns (list of trajectory states, number of local eps evaluations)."""
    x_T = np.asarray(x_T, float)
    D = x_T.size
    bufs = {("traj", 0): x_T.reshape(-1).copy()}
    for key in prog.noise_keys:
        _, t, role = key
        bufs[("noise", key)] = O.derive_noise(seed, t, role, D, generator)
    local_evals = 0
    for st in prog.steps:
        if isinstance(st, Eval):
            for (i, src, t), dst, own in zip(st.tasks, st.dst, st.owner):
                if own is None or own == rank:
                    eps = np.asarray(eps_fn(ab, bufs[src].reshape(x_T.shape), t), float)
                    if eps.size != D:                          # SI eps broadcast over a batched state
                        eps = np.broadcast_to(eps, x_T.shape)
                    bufs[dst] = eps.reshape(-1).copy()
                    local_evals += 1
        elif isinstance(st, Gather):
            rows = {i: bufs[("eps", i)] for i in range(st.n_tasks) if ("eps", i) in bufs}
            got = allgather(rows, st.n_tasks)
            for i, v in got.items():
                bufs[("eps", i)] = v
        elif isinstance(st, Chain):
            cur = anchor = None
            for op in st.ops:
                if op.src == _lib.SRC_X:
                    x = bufs[op.x]
                elif op.src == _lib.SRC_CUR:
                    x = cur
                else:
                    x = anchor
                z = bufs[op.z] if op.z is not None else None
                y = apply_op(op, x, bufs[op.eps], z)
                cur = y
                if op.save_anchor:
                    anchor = y
                if op.out is not None:
                    bufs[op.out] = y
                if op.out2 is not None:
                    bufs[op.out2] = y
    states = [(t, bufs[("traj", j)].reshape(x_T.shape)) for j, t in enumerate(prog.timesteps)]
    return states, local_evals

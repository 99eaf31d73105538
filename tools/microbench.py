"""Warm per-kernel timings of the sampler kernels (CUDA events, back-to-back
launches), to separate kernel time from launch gaps.

    python tools/microbench.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, reps=200):
    import torch
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


def main():
    import numpy as np
    import torch

    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.denoiser import gm_eps_launch
    from paper_2603_25872_b200.rng import entropy_key, fill_streams
    from paper_2603_25872_b200.transitions import ddpm_op_coeffs, launch_chain, make_op, ops_to_device

    dev = torch.device("cuda", 0)
    D = 4096
    s = P.default_schedule(50)
    m = np.zeros((2, D))
    m[0, 0], m[1, 0] = -2.0, 2.0
    gm = P.GaussianMixture(weights=[0.5, 0.5], means=m, variances=[1.0, 1.0])
    x = torch.randn(3, D, dtype=torch.float64, device=dev)
    out = torch.empty_like(x)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    res = {}
    for rows in (1, 3):
        keep = []

        def f():
            keep.append(gm_eps_launch(gm, s, [x[i] for i in range(rows)], [40] * rows,
                                      [out[i] for i in range(rows)], err))
        res[f"gm_eps rows={rows} (incl. host staging)"] = timeit(f, 50)
    # pre-staged pointer arrays (as the engine does)
    means, logw, var = gm.device_params(dev)
    xs = torch.tensor([x[i].data_ptr() for i in range(3)], dtype=torch.int64, device=dev)
    os_ = torch.tensor([out[i].data_ptr() for i in range(3)], dtype=torch.int64, device=dev)
    ts = torch.tensor([40, 39, 38], dtype=torch.int32, device=dev)
    ab = s.device_alpha_bar(dev)
    L = _lib.lib()
    for rows in (1, 3):
        res[f"gm_eps rows={rows}"] = timeit(lambda: L.drs_gm_eps(
            xs.data_ptr(), ts.data_ptr(), rows, D, ab.data_ptr(), 50, means.data_ptr(), logw.data_ptr(),
            var.data_ptr(), 2, os_.data_ptr(), err.data_ptr(), _lib.stream_ptr()))
    z = torch.randn(8, D, dtype=torch.float64, device=dev)
    outs = torch.zeros(8, D, dtype=torch.float64, device=dev)
    for n_ops in (1, 3, 5):
        ops = []
        for i in range(n_ops):
            c, noisy = ddpm_op_coeffs(s, 40, 1 + i % 3)
            ops.append(make_op(c, _lib.FAMILY_DDPM, noisy, src=_lib.SRC_X, x=x[0], eps=x[1], z=z[i], out=outs[i]))
        od = ops_to_device(ops, dev)
        res[f"skip_chain ops={n_ops}"] = timeit(lambda: launch_chain(od, n_ops, D))
    for gen in ("pcg64", "sfc64"):
        for ns in (1, 84):
            keys = [entropy_key((0x7A9C, 1, t, 0)) for t in range(ns)]
            from paper_2603_25872_b200.rng import _KeyBuffer
            kb = _KeyBuffer(keys, dev)
            tab = torch.empty(ns, D, dtype=torch.float64, device=dev)
            res[f"noise {gen} streams={ns} n={D}"] = timeit(lambda: fill_streams(kb, D, tab, gen, err=err), 20)
    res["empty torch kernel (launch floor)"] = timeit(lambda: err.zero_())
    for k, v in res.items():
        print(f"{k:45s} {v:9.2f} us")


if __name__ == "__main__":
    main()

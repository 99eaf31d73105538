"""Multi-rank engine on real kernels: 2 processes share one GPU, each runs
its own drafts/evals/refines with libdrs, and the round eps rows move over a
CPU gloo group (host-staged all-gather -- no kernel ever waits on another
process).  Every rank's trajectory must be bit-identical to the single-rank
run with the same logical devices, through both the eager path and the
per-segment CUDA-graph path."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _gm(D):
    import paper_2603_25872_b200 as P
    m = np.zeros((2, D))
    m[0, 0], m[1, 0] = -2.0, 2.0
    return P.GaussianMixture(weights=[0.5, 0.5], means=m, variances=[1.0, 1.0])


CASES = [("aggressive", "ddpm", "sfc64"), ("conservative", "ddim", "pcg64"), ("aggressive", "ddim", "pcg64")]


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200.engine import Comm
    from paper_2603_25872_b200.pipeline import Sampler
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        T, D = 16, 4096
        s = P.default_schedule(T)
        out = []
        for mode, fam, gen in CASES:
            den = P.AnalyticEps(_gm(D))
            for graph in (False, True):
                smp = Sampler(s, den, D, mode=mode, devices=world, rule=P.VarianceRule.ddpm_induced(), family=fam,
                              generator=gen, comm=Comm(rank, world), device=dev, graph=graph)
                finals = []
                for seed in (5, 6):
                    smp.stage(seed)
                    smp.launch()
                    torch.cuda.synchronize()
                    finals.append(smp.run.traj.cpu().numpy().copy())
                out.append(finals)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_ranks_match_single_rank(cuda):
    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200.pipeline import Sampler
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    T, D = 16, 4096
    s = P.default_schedule(T)
    k = 0
    for mode, fam, gen in CASES:
        smp = Sampler(s, P.AnalyticEps(_gm(D)), D, mode=mode, devices=world, rule=P.VarianceRule.ddpm_induced(),
                      family=fam, generator=gen, device=cuda, graph=True)
        for graph in (False, True):
            for j, seed in enumerate((5, 6)):
                smp.stage(seed)
                smp.launch()
                torch.cuda.synchronize()
                ref = smp.run.traj.cpu().numpy()
                for r in range(world):
                    assert np.array_equal(res[r][k][j], ref), (mode, fam, gen, graph, seed, r)
            k += 1

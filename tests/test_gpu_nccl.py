"""The NCCL data plane on a real GPU: a one-rank NCCL communicator with the
per-round eps all-gathers kept in the program (`exchange=True`), so the exact
code the N-GPU bench runs -- in-place `all_gather_into_tensor` of the round's
eps rows, captured into the run's single CUDA graph -- executes on one B200
(gpurun leases one GPU; NCCL refuses two ranks on one device).  Trajectories
must be bit-identical to the run without an exchange (reference: the ordered
gather of parallel.py:160-177)."""

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


def _worker(port, log_path, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_DEBUG="INFO",
                      NCCL_DEBUG_SUBSYS="INIT,COLL", NCCL_DEBUG_FILE=log_path)
    import torch.distributed as dist
    import paper_2603_25872_b200 as P
    from paper_2603_25872_b200.engine import Comm
    from paper_2603_25872_b200.pipeline import Sampler
    from paper_2603_25872_b200.unet import UNet, sd15_config
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        out = {}
        T = 12
        s = P.default_schedule(T)
        m = np.zeros((2, 4096))
        m[0, 0], m[1, 0] = -2.0, 2.0
        gm = P.AnalyticEps(P.GaussianMixture(weights=[0.5, 0.5], means=m, variances=[1.0, 1.0]))
        net = P.NetworkEps(UNet(sd15_config(32), dev, seed=0, max_batch=4), (4, 32, 32))
        for name, den, D, fam, rule in [("gm", gm, 4096, "ddpm", P.VarianceRule.deterministic()),
                                        ("net", net, 4096, "ddim", P.VarianceRule.ddpm_induced())]:
            res = {}
            for key, kw in [("plain", dict()), ("nccl_graph", dict(comm=Comm(0, 1), exchange=True)),
                            ("nccl_eager", dict(comm=Comm(0, 1), exchange=True, graph=False))]:
                smp = Sampler(s, den, D, mode="aggressive", devices=4, rule=rule, family=fam, device=dev, **kw)
                finals = []
                for seed in (3, 4, 3):
                    smp.stage(seed)
                    smp.launch()
                    torch.cuda.synchronize()
                    finals.append(smp.run.traj.cpu().numpy().copy())
                comm = kw.get("comm")
                res[key] = dict(finals=finals, mode=smp.run.graph_mode, gathers=comm.gathers if comm else 0,
                                rounds=len(smp.run.gather_rounds))
            out[name] = res
        q.put(out)
    finally:
        dist.destroy_process_group()


def test_nccl_allgather_data_plane_one_rank(cuda, tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    log = str(tmp_path / "nccl.log")
    p = ctx.Process(target=_worker, args=(_free_port(), log, q))
    p.start()
    out = q.get(timeout=900)
    p.join(timeout=120)
    assert p.exitcode == 0
    for name, res in out.items():
        plain = res["plain"]["finals"]
        for key in ("nccl_graph", "nccl_eager"):
            assert res[key]["rounds"] > 0                        # the gathers are in the program
            for a, b in zip(res[key]["finals"], plain):
                assert np.array_equal(a, b), (name, key)          # bit-identical through the collective
        assert "NCCL all-gathers captured" in res["nccl_graph"]["mode"], res["nccl_graph"]["mode"]
        # eager: one collective per round per image; graph: issued at warm-up + capture only
        rounds = res["nccl_eager"]["rounds"]
        assert res["nccl_eager"]["gathers"] == 3 * rounds
        assert res["nccl_graph"]["gathers"] == 2 * rounds
        assert not np.array_equal(plain[0], plain[1]) and np.array_equal(plain[0], plain[2])
    text = open(log).read() if os.path.exists(log) else ""
    assert "NCCL" in text and ("nRanks 1" in text or "nranks 1" in text.lower()), text[:2000]
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "nccl_one_rank.log"), "w") as f:
        f.write(text)

"""The sampler-program IR (what the GPU executes) interpreted with numpy must
reproduce the oracle restatement of the reference's schedulers bit-for-bit,
on one rank and across a world-size-2 gloo group.  CPU only."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import skipdiff_oracle as O
from ir_numpy import run_ir
from paper_2603_25872_b200 import VarianceRule, default_schedule
from paper_2603_25872_b200.program import Mode, build_parallel, build_sequential, plan_blocks

RULES = {"det": (VarianceRule.deterministic(), ("det",)),
         "ddpm": (VarianceRule.ddpm_induced(), ("ddpm",)),
         "eta": (VarianceRule.eta_scaled(0.4), ("eta", 0.4))}


def _same(a, b):
    return [t for t, _ in a] == [t for t, _ in b] and all(
        np.array_equal(np.asarray(x).view(np.uint64), np.asarray(y).view(np.uint64))
        for (_, x), (_, y) in zip(a, b))


def test_plans_match_golden(golden_dir):
    plans = json.load(open(os.path.join(golden_dir, "plans.json")))
    for key, p in plans.items():
        T, n, mode = key.split("_")
        got = plan_blocks(int(T), int(n), Mode(mode))
        assert [list(b) for b in got.blocks] == p["blocks"]
        assert got.total_rounds == p["rounds"] and got.total_evals == p["evals"]


@pytest.mark.parametrize("T", [8, 20, 50])
@pytest.mark.parametrize("devices", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("rule", ["det", "ddpm", "eta"])
@pytest.mark.parametrize("family", ["ddim", "ddpm"])
@pytest.mark.parametrize("mode", ["aggressive", "conservative"])
def test_ir_matches_oracle_gm(T, devices, rule, family, mode):
    s = default_schedule(T)
    ab = O.default_alpha_bar(T)
    assert np.array_equal(s.alpha_bar, ab)
    eps = O.toy_bimodal(3)
    x_T = O.derive_noise(T, T, O.INIT, (2, 3))              # batched state (2 rows)
    prog = build_parallel(s, plan_blocks(T, devices, Mode(mode)), RULES[rule][0], family)
    got, _ = run_ir(prog, ab, eps, x_T, seed=T)
    ref, evals, rounds = O.run_parallel(ab, eps, x_T, devices, mode, RULES[rule][1], T, family=family)
    assert _same(got, ref)
    assert prog.eval_count == evals and len(prog.rounds) == rounds


@pytest.mark.parametrize("devices", [2, 3])
def test_ir_recompute_anchor_ablation(devices):
    s = default_schedule(50)
    ab = O.default_alpha_bar(50)
    eps = O.toy_bimodal(1)
    x_T = O.derive_noise(5, 50, O.INIT, 1)
    prog = build_parallel(s, plan_blocks(50, devices, Mode.AGGRESSIVE), VarianceRule.deterministic(),
                          "ddim", recompute_anchor_eps=True)
    got, _ = run_ir(prog, ab, eps, x_T, seed=5)
    ref, evals, _ = O.run_parallel(ab, eps, x_T, devices, "aggressive", ("det",), 5,
                                   recompute_anchor_eps=True)
    assert _same(got, ref) and prog.eval_count == evals


@pytest.mark.parametrize("gen", ["pcg64", "sfc64"])
def test_ir_sequential_matches_oracle(gen):
    s = default_schedule(20)
    ab = O.default_alpha_bar(20)
    eps = O.toy_bimodal(4)
    x_T = O.derive_noise(3, 20, O.INIT, 4, gen)
    prog = build_sequential(s, VarianceRule.ddpm_induced(), "ddim")
    got, _ = run_ir(prog, ab, eps, x_T, seed=3, generator=gen)
    assert _same(got, O.sample_ddim(ab, eps, x_T, ("ddpm",), 3, gen))
    prog = build_sequential(s, VarianceRule.deterministic(), "ddim", subsequence=[20, 15, 9, 4, 0])
    got, _ = run_ir(prog, ab, eps, x_T, seed=3, generator=gen)
    assert _same(got, O.sample_ddim(ab, eps, x_T, ("det",), 3, gen, subsequence=[20, 15, 9, 4, 0]))
    prog = build_sequential(s, VarianceRule.deterministic(), "ddpm")
    got, _ = run_ir(prog, ab, eps, x_T, seed=3, generator=gen)
    assert _same(got, O.sample_ddpm(ab, eps, x_T, 3, gen))


def test_state_independent_makes_parallel_equal_sequential():
    # reference tests/test_parallel.py:94-107: with SI eps both modes == sequential DDIM
    for T in (8, 20):
        s, ab = default_schedule(T), O.default_alpha_bar(T)
        eps = O.SI(11, 2)
        x_T = O.derive_noise(T, T, O.INIT, 2)
        seq = O.sample_ddim(ab, eps, x_T, ("ddpm",), T)
        for devices in (1, 2, 3, 4):
            for mode in Mode:
                prog = build_parallel(s, plan_blocks(T, devices, mode), VarianceRule.ddpm_induced())
                got, _ = run_ir(prog, ab, eps, x_T, seed=T)
                assert _same(got, seq)


# ----------------------------------------------------- world size 2 (gloo) --
def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _gloo_worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for T, devices, mode, family, rule in cases:
            s, ab = default_schedule(T), O.default_alpha_bar(T)
            eps = O.toy_bimodal(5)
            x_T = O.derive_noise(1, T, O.INIT, 5)
            prog = build_parallel(s, plan_blocks(T, devices, Mode(mode)), RULES[rule][0], family,
                                  world=world, rank=rank)

            def allgather(rows, n_tasks):
                D = x_T.size
                per = -(-n_tasks // world)
                mine = torch.zeros(per, D, dtype=torch.float64)
                for i, v in rows.items():
                    if i % world == rank:
                        mine[i // world] = torch.from_numpy(v)
                out = [torch.zeros_like(mine) for _ in range(world)]
                dist.all_gather(out, mine)
                return {i: out[i % world][i // world].numpy().copy() for i in range(n_tasks)}

            got, local = run_ir(prog, ab, eps, x_T, seed=1, rank=rank, allgather=allgather)
            ref, evals, _ = O.run_parallel(ab, eps, x_T, devices, mode, RULES[rule][1], 1, family=family)
            results.append((_same(got, ref), local, evals))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_partition_and_gather():
    cases = [(20, 2, "aggressive", "ddim", "det"), (20, 4, "aggressive", "ddpm", "ddpm"),
             (21, 3, "conservative", "ddim", "ddpm"), (13, 2, "conservative", "ddpm", "det"),
             (10, 1, "aggressive", "ddim", "det")]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci in range(len(cases)):
        (ok0, l0, evals), (ok1, l1, _) = out[0][ci], out[1][ci]
        assert ok0 and ok1, cases[ci]
        # every task is evaluated exactly once across ranks, except the
        # redundant single-task (anchor) rounds which every rank evaluates
        prog = build_parallel(default_schedule(cases[ci][0]),
                              plan_blocks(cases[ci][0], cases[ci][1], Mode(cases[ci][2])),
                              RULES[cases[ci][4]][0], cases[ci][3], world=2, rank=0)
        redundant = sum(1 for st in prog.steps if hasattr(st, "owner") and st.owner[0] is None)
        assert l0 + l1 == evals + redundant


@pytest.mark.parametrize("T,devices,mode", [(100, 33, "aggressive"), (100, 40, "aggressive"),
                                            (100, 65, "conservative"), (150, 70, "aggressive"),
                                            (130, 100, "conservative")])
@pytest.mark.parametrize("rule", ["det", "ddpm"])
def test_long_chains_split_into_launches(T, devices, mode, rule):
    """Chains longer than one drs_skip_chain launch (64 ops, csrc/chain.cu kMaxOps)
    are cut; ops whose CUR / ANCHOR register would come from an earlier launch
    read the stored state instead -- bit-identical to the oracle run (advisor r1:
    T=100 with 33 devices built a 65-op chain)."""
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.program import CHAIN_MAX_OPS, Chain
    s = default_schedule(T)
    ab = O.default_alpha_bar(T)
    eps = O.toy_bimodal(2)
    x_T = O.derive_noise(1, T, O.INIT, 2)
    prog = build_parallel(s, plan_blocks(T, devices, Mode(mode)), RULES[rule][0], "ddim")
    chains = [st for st in prog.steps if isinstance(st, Chain)]
    assert max(len(c.ops) for c in chains) <= CHAIN_MAX_OPS
    assert sum(len(c.ops) for c in chains) > CHAIN_MAX_OPS
    for c in chains:          # no launch reads a register it did not set
        cur = anchor = False
        for o in c.ops:
            assert o.src != _lib.SRC_CUR or cur
            assert o.src != _lib.SRC_ANCHOR or anchor
            cur, anchor = True, anchor or o.save_anchor
    got, _ = run_ir(prog, ab, eps, x_T, seed=1)
    ref, evals, _ = O.run_parallel(ab, eps, x_T, devices, mode, RULES[rule][1], 1)
    assert _same(got, ref) and prog.eval_count == evals


def test_array_like_x_T_and_workers_zero():
    """x_T may be any array-like (np.asarray semantics, parallel.py:262) and
    workers=0 means one worker per device (`workers or devices`, parallel.py:269)."""
    from paper_2603_25872_b200.parallel import _check_workers, _numel
    from paper_2603_25872_b200.errors import InvalidPlanParams
    assert _numel([[0.1, 0.2, 0.3], [1.0, 2.0, 3.0]]) == 6
    assert _numel(np.zeros((1, 4, 8))) == 32 and _numel(torch.zeros(5)) == 5 and _numel(0.5) == 1
    _check_workers(0, None)
    _check_workers(None, None)
    with pytest.raises(InvalidPlanParams):
        _check_workers(-1, None)

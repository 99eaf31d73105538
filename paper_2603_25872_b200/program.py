"""Sampler programs: the static schedule of one sampling run as a small IR.

Everything in a DRiffusion run except the seed and x_T is known before the
first kernel launches: `plan_blocks` fixes every (t, k), so every skip
coefficient, every noise key and every evaluation task is host-computable up
front (skipdiff parallel.py:69-88,187-200,250-321).  A `Program` records the
run as a list of steps over symbolic buffers:

  Noise               fill the run's noise table (all keys, one launch)
  Eval(round, tasks)  eps for (state buffer, t) tasks; `owner[i]` is the rank
                      that evaluates task i (all ranks for redundant rounds)
  Gather(round)       all-gather of the round's eps rows across ranks
  Chain(ops)          one fused elementwise launch of skip updates (K3)

Buffers are tuples: ("traj", j) trajectory slot j, ("draft", i) draft row,
("eps", i) gathered eps row of round task i, ("anchor",) the stand-alone eps,
("noise", key) a noise row, ("xin",) the input x_T.

The CUDA backend (engine.py) lowers the IR to pointers, launches and CUDA
graphs; tests/ interpret the same IR with the numpy oracle (single process
and world-size-2 gloo) to check the schedule itself against the reference.
"""

from dataclasses import dataclass, field
from enum import Enum

from . import _lib
from .errors import InvalidPlanParams, InvalidSubsequence, PlanMismatch
from .rng import Role
from .transitions import VarianceRule, ddim_op_coeffs, ddpm_op_coeffs, euler_op_coeffs


class Mode(Enum):
    AGGRESSIVE = "aggressive"
    CONSERVATIVE = "conservative"


@dataclass(frozen=True)
class BlockPlan:
    """Blocks (anchor_t, k) covering T..1 (parallel.py:49-58)."""

    mode: Mode
    blocks: tuple
    total_rounds: int
    total_evals: int


def plan_blocks(T: int, devices: int, mode: Mode) -> BlockPlan:
    """Aggressive: k = min(n, t) per block, 1 + #blocks rounds, T+1 evals.
    Conservative: a block consumes min(n+1, t) steps, shrinking by one when
    that would leave a lone final step (unless it is already a pair); rounds
    count 2 per block with k >= 1 and 1 for a k = 0 tail (parallel.py:69-88)."""
    if T < 1 or devices < 1:
        raise InvalidPlanParams(f"need T >= 1 and devices >= 1, got ({T}, {devices})")
    blocks, t = [], T
    if mode is Mode.AGGRESSIVE:
        while t > 0:
            k = min(devices, t)
            blocks.append((t, k))
            t -= k
        return BlockPlan(mode, tuple(blocks), 1 + len(blocks), T + 1)
    while t > 0:
        span = min(devices + 1, t)
        if span > 2 and t - span == 1:
            span -= 1
        blocks.append((t, span - 1))
        t -= span
    rounds = sum(1 if k == 0 else 2 for _, k in blocks)
    return BlockPlan(mode, tuple(blocks), rounds, T)


# ------------------------------------------------------------------ IR ----
@dataclass
class OpIR:
    family: int
    c: list
    noisy: bool
    src: int                   # _lib.SRC_X / SRC_CUR / SRC_ANCHOR
    x: tuple | None            # buffer when src == SRC_X
    eps: tuple
    z: tuple | None
    out: tuple | None
    out2: tuple | None = None
    save_anchor: bool = False
    label: tuple = ()          # (t, k) for diagnostics


@dataclass
class Eval:
    round: int
    tasks: list                # [(task_index, src_buf, t)]
    dst: list                  # [dst_buf] per task
    owner: list                # rank per task; None = every rank (redundant)


@dataclass
class Gather:
    round: int
    n_tasks: int


@dataclass
class Chain:
    ops: list


@dataclass
class Noise:
    keys: list                 # [(kind, t, role)] ; kind "rng" | "si"


@dataclass
class RoundInfo:
    anchor_t: int
    n_tasks: int


@dataclass
class Program:
    kind: str                  # "parallel" | "sequential"
    T: int
    n_states: int              # trajectory slots
    timesteps: list            # t of every trajectory slot
    steps: list
    rounds: list               # RoundInfo per round
    noise_keys: list           # ordered keys -> noise row
    max_tasks: int             # rows of the eps gather buffer
    world: int
    eval_count: int
    stochastic: bool
    plan: BlockPlan | None = None
    meta: dict = field(default_factory=dict)

    def key_row(self, key) -> int:
        return self._rows[key]

    def __post_init__(self):
        self._rows = {k: i for i, k in enumerate(self.noise_keys)}


class _Builder:
    def __init__(self, s, rule, family, world, exchange=False):
        self.s, self.rule, self.family, self.world = s, rule, family, world
        self.exchange = exchange or world > 1      # emit Gather steps (also at world 1 when asked)
        self.stochastic = family == "ddpm" or (family == "ddim" and rule.stochastic)
        self.keys = []
        self._key_set = {}
        self.steps = []
        self.rounds = []
        self.eval_count = 0
        self.max_tasks = 1

    def noise(self, t, role):
        if not self.stochastic:
            return None
        key = ("rng", t, int(role))
        if key not in self._key_set:
            self._key_set[key] = len(self.keys)
            self.keys.append(key)
        return ("noise", key)

    def op(self, t, k, *, src, x, eps, z, out, out2=None, save_anchor=False):
        if self.family == "euler":     # t = remaining grid intervals: i = N - t
            c, noisy = euler_op_coeffs(self.s, self.s.N - t, k)
            fam = _lib.FAMILY_EULER
        elif self.family == "ddim":
            c, noisy = ddim_op_coeffs(self.s, t, k, self.rule)
            fam = _lib.FAMILY_DDIM
        else:
            c, noisy = ddpm_op_coeffs(self.s, t, k)
            fam = _lib.FAMILY_DDPM
        if noisy and z is None:
            raise ValueError("z required for a stochastic transition")
        return OpIR(fam, c, noisy, src, x, eps, z if noisy else None, out, out2, save_anchor, (t, k))

    def round_(self, anchor_t, tasks, dst, redundant):
        r = len(self.rounds)
        self.rounds.append(RoundInfo(anchor_t, len(tasks)))
        owner = [None] * len(tasks) if redundant else [i % self.world for i in range(len(tasks))]
        self.steps.append(Eval(r, tasks, dst, owner))
        if not redundant and self.exchange and tasks:
            self.steps.append(Gather(r, len(tasks)))
        self.eval_count += len(tasks)
        self.max_tasks = max(self.max_tasks, len(tasks))
        return r

    def chain(self, ops):
        for piece in split_chain(ops):
            self.steps.append(Chain(piece))


CHAIN_MAX_OPS = 64        # ops per drs_skip_chain launch (csrc/chain.cu kMaxOps)


def split_chain(ops, limit: int = CHAIN_MAX_OPS) -> list:
    """Cut a fused op list into launches of <= limit ops.  Inside a launch the
    CUR / ANCHOR registers carry the running state; an op that would read a
    register set in an EARLIER launch reads the buffer that op stored instead
    (every chained state is also written to HBM: a trajectory slot or a draft
    row), which is the same value bit for bit.  A long aggressive refine chain
    (k-1 refines + the next block's k2 drafts, e.g. 65 ops at T=100 with 33
    devices) thus runs as several launches instead of failing."""
    from dataclasses import replace
    if len(ops) <= limit:
        return [ops] if ops else []
    pieces, prev_buf = [], None
    anchor_buf, anchor_piece = None, -1
    for p0 in range(0, len(ops), limit):
        piece, pi = [], p0 // limit
        for j, o in enumerate(ops[p0:p0 + limit]):
            if o.src == _lib.SRC_CUR and j == 0:
                if prev_buf is None:
                    raise PlanMismatch("chain split: running state was never stored")
                o = replace(o, src=_lib.SRC_X, x=prev_buf)
            elif o.src == _lib.SRC_ANCHOR and anchor_piece < pi:
                if anchor_buf is None:
                    raise PlanMismatch("chain split: anchor state was never stored")
                o = replace(o, src=_lib.SRC_X, x=anchor_buf)
            piece.append(o)
            prev_buf = o.out if o.out is not None else o.out2
            if o.save_anchor:
                anchor_buf, anchor_piece = prev_buf, pi
        pieces.append(piece)
    return pieces


def _draft_key(t, i):
    """Draft i of anchor t: i == 1 is the kept state -> TRANSITION (parallel.py:187-194)."""
    return (t - i, Role.TRANSITION if i == 1 else Role.DRAFT)


def build_parallel(s, plan: BlockPlan, rule: VarianceRule, family: str = "ddim",
                   recompute_anchor_eps: bool = False, world: int = 1, rank: int = 0,
                   exchange: bool = False) -> Program:
    """IR of parallel.py:_run (250-321) for a plan, as seen by `rank` of `world`.

    Every rank replays drafts and refines redundantly (bit-identical), so no
    refined state is ever broadcast; each rank only evaluates its own tasks
    (owner = task % world) and the eps rows are all-gathered.  Stand-alone
    anchor evaluations (aggressive initial, conservative per-block,
    recompute ablation) are single-task rounds computed redundantly.

    family "euler" (parallel.py:324-381): `s` is a SigmaGrid, t counts the
    remaining grid intervals (N at the start), updates are euler_skip and the
    velocity tasks at sigma = 0 (t = 0, the aggressive mode's last draft) are
    dropped, since nothing consumes them (parallel.py:346-349).

    exchange=True emits the per-round Gather steps even at world 1 (a
    one-rank communicator: exercises the collective data plane on one GPU)."""
    if family not in ("ddim", "ddpm", "euler"):
        raise ValueError(f"unknown update family: {family!r}")
    T = s.N if family == "euler" else s.T
    b = _Builder(s, rule, family, world, exchange)
    slot = lambda t: ("traj", T - t)                  # noqa: E731
    mine = lambda i: world == 1 or (i - 1) % world == rank   # noqa: E731  draft i owned?
    anchor_eps = None                                 # buffer holding the current anchor eps
    pending_drafts = None                             # drafts fused into the previous refine chain

    def draft_ops(t, k, src, x, eps):
        ops = []
        for i in range(1, k + 1):
            if i != 1 and not mine(i):
                continue
            zt, role = _draft_key(t, i)
            ops.append(b.op(t, i, src=src, x=x, eps=eps, z=b.noise(zt, role), out=("draft", i - 1),
                            out2=slot(t - 1) if i == 1 else None))
        return ops

    if plan.mode is Mode.AGGRESSIVE:
        b.round_(T, [(0, slot(T), T)], [("anchor",)], redundant=True)
        anchor_eps = ("anchor",)
    for bi, (t, k) in enumerate(plan.blocks):
        if plan.mode is Mode.CONSERVATIVE:
            b.round_(t, [(0, slot(t), t)], [("anchor",)], redundant=True)
            anchor_eps = ("anchor",)
            if k == 0:     # degenerate tail: one unit step, no parallel round (parallel.py:288-292)
                b.chain([b.op(t, 1, src=_lib.SRC_X, x=slot(t), eps=anchor_eps,
                              z=b.noise(t - 1, Role.TRANSITION), out=slot(t - 1))])
                continue
        elif recompute_anchor_eps and t != T:
            b.round_(t, [(0, slot(t), t)], [("anchor",)], redundant=True)
            anchor_eps = ("anchor",)
            pending_drafts = None
        if pending_drafts is None:
            b.chain(draft_ops(t, k, _lib.SRC_X, slot(t), anchor_eps))
        live = [i for i in range(1, k + 1) if family != "euler" or t - i > 0]
        tasks = [(i - 1, ("draft", i - 1), t - i) for i in live]
        b.round_(t, tasks, [("eps", i - 1) for i in live], redundant=False)
        last = k if plan.mode is Mode.AGGRESSIVE else k + 1
        ops = []
        for i in range(2, last + 1):
            ops.append(b.op(t - i + 1, 1, src=_lib.SRC_X if i == 2 else _lib.SRC_CUR,
                            x=slot(t - 1) if i == 2 else None, eps=("eps", i - 2),
                            z=b.noise(t - i, Role.TRANSITION), out=slot(t - i),
                            save_anchor=(i == last)))
        pending_drafts = None
        if plan.mode is Mode.AGGRESSIVE:
            anchor_eps = ("eps", k - 1)               # cached draft-state eps (parallel.py:307)
            nxt = plan.blocks[bi + 1] if bi + 1 < len(plan.blocks) else None
            if nxt is not None and not recompute_anchor_eps:
                t2, k2 = nxt
                if ops:
                    ops += draft_ops(t2, k2, _lib.SRC_ANCHOR, None, anchor_eps)
                else:      # k == 1: the new anchor is the stored draft-1 state
                    ops += draft_ops(t2, k2, _lib.SRC_X, slot(t2), anchor_eps)
                pending_drafts = True
        b.chain(ops)

    expected = plan.total_evals
    if family == "euler" and plan.mode is Mode.AGGRESSIVE:
        expected -= 1                                 # the sigma = 0 draft of the last block
    if recompute_anchor_eps and plan.mode is Mode.AGGRESSIVE:
        expected += sum(1 for t, _ in plan.blocks if t != T)
    if b.eval_count != expected:
        raise PlanMismatch(f"{b.eval_count} evals, plan expected {expected}")
    prog = Program("parallel", T, T + 1, list(range(T, -1, -1)), b.steps, b.rounds, b.keys,
                   b.max_tasks, world, b.eval_count, b.stochastic, plan,
                   meta={"rank": rank, "family": family, "mode": plan.mode.value})
    if prog.timesteps[-1] != 0:
        raise PlanMismatch("trajectory does not end at t=0")
    return prog


def check_subsequence(T: int, subsequence) -> list:
    """Strictly decreasing, starts <= T, ends at 0 (sequential.py:79-85)."""
    ts = list(subsequence)
    if not ts or ts[-1] != 0 or ts[0] > T:
        raise InvalidSubsequence(f"subsequence must start <= {T} and end at 0: {ts}")
    if any(a <= b for a, b in zip(ts, ts[1:])):
        raise InvalidSubsequence(f"subsequence must be strictly decreasing: {ts}")
    return ts


def build_sequential(s, rule: VarianceRule, family: str = "ddim", subsequence=None) -> Program:
    """IR of sample_ddim (sequential.py:88-113) / sample_ddpm (:57-76):
    one eval then one skip per step; z of the step into u is (u, TRANSITION)."""
    if family == "ddim":
        ts = check_subsequence(s.T, subsequence if subsequence is not None else range(s.T, -1, -1))
    else:
        ts = list(range(s.T, -1, -1))
        rule = VarianceRule.deterministic()
    b = _Builder(s, rule, family, 1)
    for j, (t, u) in enumerate(zip(ts, ts[1:])):
        b.round_(t, [(0, ("traj", j), t)], [("anchor",)], redundant=True)
        b.chain([b.op(t, t - u, src=_lib.SRC_X, x=("traj", j), eps=("anchor",),
                      z=b.noise(u, Role.TRANSITION), out=("traj", j + 1))])
    return Program("sequential", s.T, len(ts), ts, b.steps, b.rounds, b.keys, 1, 1,
                   b.eval_count, b.stochastic, None, meta={"family": family})


def build_sequential_euler(g) -> Program:
    """IR of sample_euler (sequential.py:116-130): velocity at sigma_i, then
    x + (sigma_{i+1} - sigma_i) v, for i = 0..N-1; t counts remaining intervals."""
    N = g.N
    b = _Builder(g, None, "euler", 1)
    for j in range(N):
        t = N - j
        b.round_(t, [(0, ("traj", j), t)], [("anchor",)], redundant=True)
        b.chain([b.op(t, 1, src=_lib.SRC_X, x=("traj", j), eps=("anchor",), z=None, out=("traj", j + 1))])
    return Program("sequential", N, N + 1, list(range(N, -1, -1)), b.steps, b.rounds, b.keys, 1, 1,
                   b.eval_count, False, None, meta={"family": "euler"})

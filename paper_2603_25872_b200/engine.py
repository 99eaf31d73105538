"""CUDA backend of sampler programs (program.py): HBM layout, launches, graphs.

HBM layout of one run (D = latent elements, fp64 unless noted):
  traj   (n_states, D)          every trajectory state, slot j <-> timesteps[j]
  drafts (max_tasks, D)         this rank's drafts of the current block
  anchor (D)  eps dtype         stand-alone eps (anchor / sequential evals)
  gbuf   (world, per_rank, D)   round eps, task i at [i % world, i // world];
                                all-gathered in place across ranks
  noise  (n_keys, D)            every noise row the run consumes, generated
                                by ONE drs_noise_fill launch at the start
  ops    (n_ops x 112 B)        every drs_op of the run, uploaded once
All pointers are fixed at build time, so a single-rank run is captured as one
CUDA graph and replayed per image with only x_T and the seed words changed.
"""

import math

import torch

from . import _lib
from .denoiser import (AnalyticEps, Counting, EulerVelocity, Latency, NetworkEps, Perturbed, PerturbPlan,
                       StateIndependent, latency_of, perturb_scales, state_independent_key)
from .program import Chain, Eval, Gather, Noise, Program
from .rng import _STREAM_SALT, _SEED_MASK48, GENERATORS, _KeyBuffer, entropy_key
from .transitions import ops_to_device

_OP_BYTES = _lib.ctypes.sizeof(_lib.DrsOp)


class _nvtx:
    """NVTX range around a libdrs launch group (ncu --nvtx / nsys timelines: noise,
    eval_<kind>, chain, gather, spin), a no-op without CUDA."""

    def __init__(self, label):
        self.label = label

    def __enter__(self):
        if torch.cuda.is_available():
            torch.cuda.nvtx.range_push(self.label)

    def __exit__(self, *a):
        if torch.cuda.is_available():
            torch.cuda.nvtx.range_pop()


def _nvtx_mark(msg):
    """NVTX marker at the start of every scheduler round (round index, anchor t, tasks)."""
    if torch.cuda.is_available():
        torch.cuda.nvtx.mark(msg)


def _n_tasks(low):
    """Evaluations in a lowered eval payload (a Perturbed payload wraps the core one)."""
    return _n_tasks(low[1]) if low[0] == "pert" else low[1]["n_tasks"]


def unwrap(d):
    """(core denoiser, eval latency ms (sum of nested Latency), [Counting wrappers])."""
    lat, counters = 0.0, []
    while True:
        if isinstance(d, Latency):
            lat += d.model.eval_time_ms
            d = d.inner
        elif isinstance(d, Counting):
            counters.append(d)
            d = d.inner
        elif isinstance(d, Perturbed):      # applied after the core eval (PerturbPlan)
            d = d.inner
        else:
            return d, lat, counters


class Comm:
    """Rank/world plus the per-round eps exchange (torch.distributed / NCCL).

    On NCCL the exchange is one in-place ncclAllGather of the round's eps rows
    on the current stream, so it is captured into the run's CUDA graph with
    the kernels around it (a multi-rank image is ONE graph replay per rank).
    The gloo backend stages through the host (tests: several ranks' kernels
    on one GPU, or CPU-only hosts) and is issued between per-segment graph
    replays."""

    def __init__(self, rank: int = 0, size: int = 1, group=None):
        self.rank, self.size, self.group = rank, size, group
        self.gathers = 0                  # collectives issued (host calls, incl. captures)

    @property
    def backend(self):
        import torch.distributed as dist
        if not dist.is_available() or not dist.is_initialized():
            return None
        return dist.get_backend(self.group)

    @property
    def capturable(self) -> bool:
        """The exchange can live inside a CUDA graph (device-side collective)."""
        return self.backend == "nccl"

    def all_gather_rows(self, gbuf):
        """In-place all-gather of gbuf[world, per_rank, D]: rank r contributes gbuf[r]."""
        import torch.distributed as dist
        flat = gbuf.view(self.size, -1)
        self.gathers += 1
        if dist.get_backend(self.group) == "gloo":
            # host-staged path: lets tests run several ranks' kernels on one GPU
            # (no device-side waits between processes) over a CPU process group
            parts = [torch.empty_like(flat[0], device="cpu") for _ in range(self.size)]
            dist.all_gather(parts, flat[self.rank].cpu(), group=self.group)
            for r, t in enumerate(parts):
                if r != self.rank:
                    flat[r].copy_(t)
            return
        dist.all_gather_into_tensor(flat.view(-1), flat[self.rank], group=self.group)


class DeviceRun:
    """A Program bound to a denoiser, a latent size and one CUDA device."""

    def __init__(self, prog: Program, s, d, D: int, device, *, generator: str = "pcg64",
                 comm: Comm | None = None, derive_init: bool = False):
        self.prog, self.s, self.D = prog, s, int(D)
        self.derive_init = derive_init     # x_T = INIT noise of the seed (cli.py:53), in-program
        self.device = torch.device(device)
        self.comm = comm or Comm()
        if self.comm.size != prog.world:
            raise ValueError(f"program built for world {prog.world}, comm has {self.comm.size}")
        self.generator = generator
        self.core, self.eval_ms, self.counters = unwrap(d)
        self.perturb = perturb_scales(d)
        self.overhead_ms = (latency_of(d).dispatch_overhead_ms if latency_of(d) else 0.0)
        core = self.core
        if isinstance(core, (AnalyticEps, StateIndependent, EulerVelocity)):
            dim = core.dim if isinstance(core, StateIndependent) else core.gm.dim
            if dim < 1 or self.D % dim:
                from .errors import DimensionMismatch
                raise DimensionMismatch(f"denoiser dim {dim} does not tile state size {self.D}")
            self.dim, self.B = dim, self.D // dim      # B independent rows per state (batched x_T)
            self.eps_dtype = torch.float64
        elif isinstance(core, NetworkEps):
            n = 1
            for v in core.latent_shape:
                n *= int(v)
            if n != self.D:
                from .errors import DimensionMismatch
                raise DimensionMismatch(f"network latent {core.latent_shape} != state size {self.D}")
            self.dim, self.B = self.D, 1
            self.eps_dtype = torch.float32
        else:
            raise TypeError(f"unknown denoiser kind: {type(core).__name__}")
        if self.perturb and self.eps_dtype != torch.float64:
            raise NotImplementedError("Perturbed wraps the fp64 toy denoisers (denoiser.py:191-201)")
        self._alloc()
        self._lower()
        self.graph = None
        self.graph_mode = "eager"

    # ---------------------------------------------------------- layout ----
    def _alloc(self):
        p, D, dev = self.prog, self.D, self.device
        f64 = torch.float64
        self.traj = torch.zeros(p.n_states, D, dtype=f64, device=dev)
        self.drafts = torch.zeros(max(p.max_tasks, 1), D, dtype=f64, device=dev)
        self.anchor = torch.zeros(D, dtype=self.eps_dtype, device=dev)
        self.per_rank = max(1, math.ceil(p.max_tasks / p.world))
        self.gbuf = torch.zeros(p.world, self.per_rank, D, dtype=self.eps_dtype, device=dev)
        # noise rows: the sampler's rng keys, then the SI table (one row per eval t)
        self.keys = list(p.noise_keys)
        self.init_key = ("rng", p.timesteps[0], 2)          # Role.INIT
        if self.derive_init and self.init_key not in self.keys:
            self.keys.append(self.init_key)
        if isinstance(self.core, StateIndependent):
            ts = sorted({t for st in p.steps if isinstance(st, Eval) for (_, _, t) in st.tasks})
            for t in ts:
                self.keys.append(("si", t, None))
        self.rows = {k: i for i, k in enumerate(self.keys)}
        self.noise = torch.zeros(max(len(self.keys), 1), D, dtype=f64, device=dev)
        self.seeds = torch.zeros(2, dtype=torch.int64, device=dev)    # [stream seed, si seed]
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.xin = torch.zeros(D, dtype=f64, device=dev)
        dkeys = []
        for kind, t, role in self.keys:
            if kind == "rng":
                dkeys.append(entropy_key((_STREAM_SALT, 0, t, role), seed_slot=0, seed_mask=_SEED_MASK48))
            else:
                dkeys.append(entropy_key((0x51DE, 0, t), seed_slot=1, seed_mask=0xFFFFFFFF))
        self.keybuf = _KeyBuffer(dkeys, dev) if dkeys else None

    def buf(self, ref):
        kind = ref[0]
        if kind == "traj":
            return self.traj[ref[1]]
        if kind == "draft":
            return self.drafts[ref[1]]
        if kind == "anchor":
            return self.anchor
        if kind == "eps":
            i = ref[1]
            return self.gbuf[i % self.prog.world, i // self.prog.world]
        if kind == "noise":
            return self.noise[self.rows[ref[1]]]
        if kind == "xin":
            return self.xin
        raise KeyError(ref)

    # --------------------------------------------------------- lowering ---
    def _lower(self):
        from .transitions import make_op
        rank = self.comm.rank
        ops_all = []
        self.launches = []                 # (kind, payload)
        for st in self.prog.steps:
            if isinstance(st, Chain):
                off = len(ops_all)
                written = set()
                for o in st.ops:   # chain.cu prefetches operands: no RAW through memory within a chain
                    if o.src == _lib.SRC_X and o.x in written:
                        raise AssertionError(f"chain op reads {o.x} written earlier in the same launch")
                    written.update(b for b in (o.out, o.out2) if b is not None)
                for o in st.ops:
                    ops_all.append(make_op(
                        o.c, o.family, o.noisy, src=o.src,
                        x=self.buf(o.x) if o.x is not None else None,
                        eps=self.buf(o.eps), z=self.buf(o.z) if o.z is not None else None,
                        out=self.buf(o.out) if o.out is not None else None,
                        out2=self.buf(o.out2) if o.out2 is not None else None,
                        save_anchor=o.save_anchor))
                self.launches.append(("chain", (off, len(st.ops))))
            elif isinstance(st, Eval):
                local = [(tk, dst) for tk, dst, own in zip(st.tasks, st.dst, st.owner)
                         if own is None or own == rank]
                low = self._lower_eval(local)
                if low is not None and self.perturb:
                    low = ("pert", low, PerturbPlan(self.perturb, [self.buf(src) for (_, src, _), _ in local],
                                                    [t for (_, _, t), _ in local],
                                                    [self.buf(dst) for _, dst in local], self.device))
                self.launches.append(("eval", (st.round, low)))
            elif isinstance(st, Gather):
                self.launches.append(("gather", st.round))
            elif isinstance(st, Noise):
                pass
        if isinstance(self.core, NetworkEps):
            # per-run conditioning table (DiT): filled by one launch ahead of the first eval
            from .netdenoise import plan_conditioning
            tcond = plan_conditioning(self.core, self.launches, self.device)
            if tcond is not None:
                self.launches.insert(0, ("cond", tcond))
        self.local_evals = sum(_n_tasks(payload[1]) for kind, payload in self.launches
                               if kind == "eval" and payload[1] is not None)
        self.n_ops = len(ops_all)
        self.ops_dev = ops_to_device(ops_all, self.device) if ops_all else None
        self._split_segments()
        self.launch_bytes = [self._algo_bytes(k, p, ops_all) for k, p in self.launches]

    def _algo_bytes(self, kind, payload, ops_all):
        """Algorithmic HBM bytes of one launch: every operand vector read once,
        every output vector written once."""
        D, esz = self.D, self.gbuf.element_size()
        if kind == "chain":
            off, n = payload
            b = 0
            for o in ops_all[off:off + n]:
                b += (8 * D if o.src == _lib.SRC_X else 0) + (4 if o.eps_f32 else 8) * D
                b += (8 * D if o.noisy else 0) + (8 * D if o.out else 0) + (8 * D if o.out2 else 0)
            return b
        if kind == "eval":
            low = payload[1]
            if low is None:
                return 0
            if low[0] == "pert":
                low = low[1]
            if low[0] in ("gm", "gmv"):
                return low[1]["n"] * self.dim * 8 * (2 + low[1]["n_comp"])
            if low[0] == "copy":
                return low[1]["n"] * self.dim * 16
            return 0
        if kind == "gather":
            return self.prog.world * self.per_rank * D * esz
        return 0

    def _lower_eval(self, local):
        if not local:
            return None
        core = self.core
        if isinstance(core, NetworkEps):
            from .netdenoise import lower_eval
            chunks = lower_eval(core, self.s, [self.buf(src) for (_, src, _), _ in local],
                                [t for (_, _, t), _ in local], [self.buf(dst) for _, dst in local], self.device)
            return ("net", dict(chunks=chunks, n=len(local), n_tasks=len(local)))
        # one row per (task, batch row b): GM rows are independent states;
        # the SI eps of a task is the same row broadcast over b (denoiser.py:252)
        xs, outs, ts = [], [], []
        dim = self.dim
        for (_, src, t), dst in local:
            x, o = self.buf(src), self.buf(dst)
            for bi in range(self.B):
                xs.append(x[bi * dim:(bi + 1) * dim])
                outs.append(o[bi * dim:(bi + 1) * dim])
                ts.append(t)
        if isinstance(core, AnalyticEps):
            means, logw, var = core.gm.device_params(self.device)
            return ("gm", dict(
                xs=torch.tensor([x.data_ptr() for x in xs], dtype=torch.int64, device=self.device),
                outs=torch.tensor([o.data_ptr() for o in outs], dtype=torch.int64, device=self.device),
                ts=torch.tensor(ts, dtype=torch.int32, device=self.device),
                n=len(xs), n_tasks=len(local), means=means, logw=logw, var=var, n_comp=len(core.gm.weights),
                alpha=self.s.device_alpha_bar(self.device)))
        if isinstance(core, EulerVelocity):      # task t = remaining intervals: sigma_{N - t}
            means, logw, var = core.gm.device_params(self.device)
            N = core.grid.N
            return ("gmv", dict(
                xs=torch.tensor([x.data_ptr() for x in xs], dtype=torch.int64, device=self.device),
                outs=torch.tensor([o.data_ptr() for o in outs], dtype=torch.int64, device=self.device),
                idx=torch.tensor([N - t for t in ts], dtype=torch.int32, device=self.device),
                n=len(xs), n_tasks=len(local), means=means, logw=logw, var=var, n_comp=len(core.gm.weights),
                sigmas=core.grid.device_sigmas(self.device), N=N))
        if isinstance(core, StateIndependent):
            src = [self.noise[self.rows[("si", t, None)]] for t in ts]
            return ("copy", dict(
                src=torch.tensor([x.data_ptr() for x in src], dtype=torch.int64, device=self.device),
                outs=torch.tensor([o.data_ptr() for o in outs], dtype=torch.int64, device=self.device),
                n=len(src), n_tasks=len(local)))

    # -------------------------------------------------------- execution ---
    def set_inputs(self, x_T, seed: int, si_seed: int | None = None):
        """Stage x_T (device or pinned host tensor) and the seed words."""
        self.xin.copy_(x_T.reshape(-1), non_blocking=True)
        si = si_seed if si_seed is not None else (self.core.seed if isinstance(self.core, StateIndependent) else 0)
        self._seed_host = torch.tensor([seed & _SEED_MASK48, si & 0xFFFFFFFF], dtype=torch.int64)
        self.seeds.copy_(self._seed_host, non_blocking=True)

    def _launch_eval(self, payload, stream):
        if payload[0] == "pert":
            self._launch_eval(payload[1], stream)
            payload[2].launch(self.err)
            return
        kind, a = payload
        L = _lib.lib()
        if kind == "gm":
            st = L.drs_gm_eps(a["xs"].data_ptr(), a["ts"].data_ptr(), a["n"], self.dim,
                              a["alpha"].data_ptr(), self.s.T, a["means"].data_ptr(),
                              a["logw"].data_ptr(), a["var"].data_ptr(), a["n_comp"],
                              a["outs"].data_ptr(), self.err.data_ptr(), stream)
            _lib.check(st, "drs_gm_eps")
        elif kind == "gmv":
            st = L.drs_gm_velocity(a["xs"].data_ptr(), a["idx"].data_ptr(), a["n"], self.dim,
                                   a["sigmas"].data_ptr(), a["N"], a["means"].data_ptr(),
                                   a["logw"].data_ptr(), a["var"].data_ptr(), a["n_comp"],
                                   a["outs"].data_ptr(), self.err.data_ptr(), stream)
            _lib.check(st, "drs_gm_velocity")
        elif kind == "copy":
            _lib.check(L.drs_copy_rows(a["src"].data_ptr(), a["outs"].data_ptr(), a["n"], self.dim, stream),
                       "drs_copy_rows")
        else:
            from .netdenoise import network_eval_into
            network_eval_into(self.core, a["chunks"])

    def enqueue(self, events=None, timers=None):
        """Issue the whole run on the current stream.  Stochastic noise uses the
        generator of the run's RngStream; the SI table always uses PCG64
        (denoiser.py:144).  `events[r]` (start, end) bracket round r; `timers`,
        if a list, receives (kernel class, algorithmic bytes, start event, end
        event) for every libdrs launch."""
        for i in range(len(self.segments)):
            self.enqueue_segment(i, events, timers)
            self.gather_after(i, events, timers)

    def _timed(self, timers):
        def timed(label, nbytes, fn):
            if timers is None:
                with _nvtx(label):
                    return fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            with _nvtx(label):
                fn()
            e1.record()
            timers.append((label, nbytes, e0, e1))
        return timed

    def enqueue_segment(self, i, events=None, timers=None):
        """Launches between two eps all-gathers (segment 0 also fills the noise
        table and stages x_T).  Contains no collective, so it is capturable."""
        stream = _lib.stream_ptr()
        L = _lib.lib()
        timed = self._timed(timers)
        if i == 0:
            self.err.zero_()
            self._enqueue_noise(stream, timed)
            if self.derive_init:
                self.traj[0].copy_(self.noise[self.rows[self.init_key]])
            else:
                self.traj[0].copy_(self.xin)
        lo, hi = self.segments[i]
        for (kind, payload), nbytes in zip(self.launches[lo:hi], self.launch_bytes[lo:hi]):
            if kind == "chain":
                off, n = payload
                timed("chain", nbytes, lambda: _lib.check(
                    L.drs_skip_chain(self.ops_dev.data_ptr() + off * _OP_BYTES, n, self.D, stream),
                    "drs_skip_chain"))
            elif kind == "cond":
                timed("cond", nbytes, lambda: self.core.net.prepare_conditioning(payload))
            elif kind == "eval":
                rnd, lowered = payload
                if events is not None:
                    events[rnd][0].record()
                info = self.prog.rounds[rnd]
                _nvtx_mark(f"round {rnd}: anchor t={info.anchor_t}, {info.n_tasks} eval(s)")
                if lowered is not None:
                    if self.eval_ms > 0:
                        timed("spin", 0, lambda: _lib.check(
                            L.drs_spin(self.eval_ms * 1000.0, _n_tasks(lowered), stream), "drs_spin"))
                    timed("eval_" + lowered[0], nbytes, lambda: self._launch_eval(lowered, stream))
                if events is not None and not self._gathered(rnd):
                    events[rnd][1].record()

    def gather_after(self, i, events=None, timers=None):
        if i < len(self.gather_rounds):
            rnd = self.gather_rounds[i]
            nb = self.prog.world * self.per_rank * self.D * self.gbuf.element_size()
            self._timed(timers)("gather", nb, lambda: self.comm.all_gather_rows(self.gbuf))
            if events is not None:
                events[rnd][1].record()

    def _split_segments(self):
        self.segments, self.gather_rounds = [], []
        lo = 0
        for j, (kind, payload) in enumerate(self.launches):
            if kind == "gather":
                self.segments.append((lo, j))
                self.gather_rounds.append(payload)
                lo = j + 1
        self.segments.append((lo, len(self.launches)))

    def _gathered(self, rnd):
        return any(k == "gather" and p == rnd for k, p in self.launches)

    def _key_ranges(self):
        rng_rows = [i for i, k in enumerate(self.keys) if k[0] == "rng"]
        si_rows = [i for i, k in enumerate(self.keys) if k[0] == "si"]
        return rng_rows, si_rows

    def _enqueue_noise(self, stream, timed):
        if not self.keys:
            return
        L = _lib.lib()
        rng_rows, si_rows = self._key_ranges()
        # rng rows come first, si rows after (see _alloc): two contiguous launches
        ext = getattr(self, "external_noise", None)
        if rng_rows and ext is not None:      # caller-supplied rows (an RngStream.derive override)
            for r, row in zip(rng_rows, ext):
                self.noise[r].copy_(torch.as_tensor(row).reshape(-1), non_blocking=True)
        elif rng_rows:
            timed("noise", len(rng_rows) * self.D * 8, lambda: _lib.check(L.drs_noise_fill(
                GENERATORS[self.generator], self.keybuf.dev.data_ptr(), len(rng_rows), self.seeds.data_ptr(),
                self.D, self.noise.data_ptr(), self.noise.stride(0), self.err.data_ptr(), stream),
                "drs_noise_fill"))
        if si_rows:
            off = si_rows[0]
            timed("noise_si", len(si_rows) * self.dim * 8, lambda: _lib.check(L.drs_noise_fill(
                _lib.GEN_PCG64, self.keybuf.dev.data_ptr() + off * 48, len(si_rows), self.seeds.data_ptr(),
                self.dim, self.noise[off].data_ptr(), self.noise.stride(0), self.err.data_ptr(), stream),
                "drs_noise_fill"))

    def launches_per_run(self) -> int:
        """libdrs kernel launches issued per run (torch copies excluded)."""
        rng_rows, si_rows = self._key_ranges()
        n = (1 if rng_rows else 0) + (1 if si_rows else 0)
        for kind, payload in self.launches:
            if kind == "chain":
                n += 1
            elif kind == "eval" and payload[1] is not None and payload[1][0] != "net":
                n += 1 + (1 if self.eval_ms > 0 else 0)
        return n

    def _warm_stream(self):
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        return s

    def capture(self):
        """Capture the run into CUDA graphs: ONE graph when the run has no
        exchange or its exchange is a device collective (NCCL all-gathers
        captured between the kernels); one graph per segment between
        all-gathers otherwise (host-staged gloo exchange between replays)."""
        s = self._warm_stream()
        with torch.cuda.stream(s):
            self.enqueue()                    # warm-up outside capture (allocations, tensor maps, NCCL comm)
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        if not self.gather_rounds or self.comm.capturable:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self.enqueue()
                self.graph, self.seg_graphs = g, None
                self.graph_mode = "one graph" + (" (NCCL all-gathers captured)" if self.gather_rounds else "")
                return g
            except RuntimeError as exc:
                if not self.gather_rounds:
                    raise
                # a collective that refuses capture: per-segment graphs with the same
                # all-gathers issued between replays (NCCL matches collectives by order,
                # so ranks that captured and ranks that did not stay in step)
                torch.cuda.synchronize(self.device)
                self.capture_error = str(exc)
        self.graph_mode = "per-segment graphs, exchange between replays"
        self.seg_graphs = []
        for i in range(len(self.segments)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.enqueue_segment(i)
            self.seg_graphs.append(g)
        self.graph = None
        return self.seg_graphs

    def replay(self):
        if self.graph is None and not getattr(self, "seg_graphs", None):
            self.capture()
        if self.graph is not None:
            self.graph.replay()
            return
        for i, g in enumerate(self.seg_graphs):
            g.replay()
            self.gather_after(i)

    def check_err(self):
        from .rng import _check_err
        _check_err(self.err)

    def account(self, clock=None):
        """Host-side accounting of one run: Counting wrappers and VirtualClock
        (rounds charge max task latency + dispatch overhead, parallel.py:138-148;
        sequential evals charge eval_time each, sequential.py:104-111)."""
        for c in self.counters:       # evaluations this rank performed (denoiser.py:264-266)
            c.count += self.local_evals
        if clock is None:
            return None
        per_round = []
        for r in self.prog.rounds:
            if self.prog.kind == "sequential":
                ms = self.eval_ms
            else:
                ms = (self.eval_ms if r.n_tasks else 0.0) + self.overhead_ms
            clock.charge(ms)
            per_round.append(ms)
        return per_round

"""Pipelined MLSDC across a block of time steps -- PFASST / IPFASST (pfasst.py).

The reference's serial schedule (pfasst.py:213-228) is normative and is kept
exactly: predictor phases, coarse hand-offs, blocking fine hand-offs per
iteration, convergence freezing, block chaining.  Three executors:

``"serial"`` / ``"threaded"``
    all P time ranks resident on one GPU, issued in the serial order on one
    CUDA stream.  Hand-offs are stream-ordered device reads of the sender's
    state (identical to the reference's snapshots).
    Convergence flags are resolved lazily: rank n's residual of iteration k
    is read back only when rank n's iteration k+1 is about to be issued, by
    which time ranks n+1..P-1 of iteration k are still queued -- the GPU never
    drains waiting for the host.  ("threaded" is the reference's bitwise-
    identical alternative executor; here it is the same device schedule.)
    With ``streams=True`` (default) every time rank issues on its own CUDA
    stream in wavefront order (anti-diagonals n + k): iteration k of rank n
    depends only on iteration k of rank n-1 (its payloads, copied at the
    start) and on iteration k-1 of itself, so latency-bound work of one rank
    (coarse sweeps, small multigrid levels) overlaps the bandwidth-bound fine
    sweeps of others.  Two events per rank order the hand-offs: "done"
    (payload final) and "copied" (successor took its copy, the state may be
    overwritten).  Results and traces are those of the serial order.
``"nccl"``
    one process per GPU (torch.distributed, NCCL over NVLink/NVSwitch), time
    rank n on process n mod G.  Fine / coarse hand-offs are NCCL send/recv of
    snapshot buffers; the final value of a block is broadcast from the owner
    of the last rank.  Frozen ranks stop sending once their receiver has seen
    converged=True and the receiver re-uses the cached payloads, which is
    numerically identical to the reference's resend.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from ._device import (clone_field, field_elems, field_from_flat, flat_storage, like_input,
                      to_device, zeros)
from .hierarchy import (Hooks, Level, TimeStep, burn_in, check_hierarchy, interpolate_up,
                        mlsdc_iteration, restrict_state)
from .sdc import NodeStates, residual_into


@dataclass
class TraceRow:
    """pfasst.py:24-31."""

    block: int
    rank: int
    iteration: int
    level: int
    residual: float
    vcycles: int


@dataclass
class PfasstResult:
    """pfasst.py:34-46."""

    u: object
    rank_iterations: list = field(default_factory=list)
    rank_vcycles: list = field(default_factory=list)
    converged: list = field(default_factory=list)
    trace: list = field(default_factory=list)
    final_values: list = field(default_factory=list)

    @property
    def total_vcycles(self) -> int:
        return sum(sum(b) for b in self.rank_vcycles)


# ---------------------------------------------------------------------------
# per-rank device engine


class _PreCoarse(Hooks):
    def __init__(self, fn):
        self.fn = fn

    def pre_coarse_sweep(self, ts):
        if self.fn is not None:
            self.fn(ts)


_RANK_STREAMS: dict = {}


def _rank_stream(n):
    """The CUDA stream of time rank n on the current device, created once per
    process: the per-stream multigrid plans and scratch (multigrid.plan_for,
    _device.scratch) are keyed by the stream, so reusing the streams across
    pfasst_run calls reuses those workspaces instead of growing them."""
    key = (torch.cuda.current_device(), n)
    st = _RANK_STREAMS.get(key)
    if st is None:
        st = _RANK_STREAMS[key] = torch.cuda.Stream()
    return st


class DeviceEngine:
    """Owns the TimeStep state of the time ranks of this process (one GPU)."""

    def __init__(self, levels, dt, ranks, streams=False):
        self.levels = levels
        self.dt = dt
        self.L = len(levels)
        self.ranks = list(ranks)
        self.ts = {}
        self.spread_y = {}
        self.streams = {n: _rank_stream(n) for n in self.ranks} if streams else None
        self._coarse_in = {}
        self._res = zeros((max(self.ranks) + 1 if self.ranks else 1,))
        self._res_host = torch.zeros(self._res.shape, dtype=torch.float64,
                                     pin_memory=True)
        self._events = {}

    # -- state ---------------------------------------------------------------
    def spread(self, n, u):
        """TimeStep.spread + spread copies of levels >= 1 (hierarchy.py:138-150,
        pfasst.py:132-134); buffers are reused across blocks."""
        ts = self.ts.get(n)
        if ts is None:
            ts = self.ts[n] = TimeStep.spread(self.levels, u)
        else:
            uu = u
            for l, lvl in enumerate(self.levels):
                if l > 0:
                    prev = self.levels[l - 1]
                    if lvl.grid.n == prev.grid.n:
                        uu = clone_field(uu)
                    else:
                        from .transfers import full_weighting, inject
                        uu = inject(uu) if prev.space_restrict == "inject" else \
                            full_weighting(uu)
                st = ts.states[l]
                st.y.copy_(uu.unsqueeze(0).expand_as(st.y))
                lvl.operator.apply_into(st.y[0], st.f[0])
                st.f[1:].copy_(st.f[0].unsqueeze(0).expand_as(st.f[1:]))
                ts.set_y0(l, uu)
                ts.tau[l] = None
        copies = self.spread_y.get(n)
        if copies is None:
            copies = self.spread_y[n] = [None] + [clone_field(ts.states[l].y, lvl_d)
                                                  for l in range(1, self.L)
                                                  for lvl_d in [self.levels[l].grid.dim]]
        else:
            for l in range(1, self.L):
                copies[l].copy_(ts.states[l].y)

    def coarse_payload(self, n):
        return self.ts[n].states[self.L - 1].y[-1]

    def fine_payload(self, n):
        return self.ts[n].states[0].y[-1]

    def set_coarse_y0(self, n, t):
        self.ts[n].set_y0(self.L - 1, t)

    def set_fine_y0(self, n, t):
        """pfasst.py:196-198 for level 0."""
        ts = self.ts[n]
        ts.states[0].y[0].copy_(t)
        ts.set_y0(0, ts.states[0].y[0], alias=True)
        self.levels[0].operator.apply_into(ts.states[0].y[0], ts.states[0].f[0])

    def stream(self, n):
        """Context issuing rank n's work (its own stream in wavefront mode)."""
        import contextlib
        return torch.cuda.stream(self.streams[n]) if self.streams else contextlib.nullcontext()

    def stage_coarse(self, n, t):
        """Copy of the predecessor's coarse payload, taken at the start of the
        iteration (the predecessor may move on afterwards)."""
        buf = self._coarse_in.get(n)
        if buf is None:
            buf = self._coarse_in[n] = clone_field(t)
        else:
            buf.copy_(t)
        return buf

    # -- work ----------------------------------------------------------------
    def burn_in(self, n):
        return burn_in(self.ts[n], self.dt, 1)

    def interpolate_up(self, n, exact):
        ts = self.ts[n]
        interpolate_up(ts, self.spread_y[n], exact_y0=clone_field(ts.y0[0]) if exact else None)

    def iteration(self, n, pre_coarse):
        return mlsdc_iteration(self.ts[n], self.dt, _PreCoarse(pre_coarse))

    def residual(self, n):
        """Launch the fine residual (pfasst.py:200) and its readback."""
        ts = self.ts[n]
        residual_into(ts.states[0], ts.y0[0], self.dt, self._res[n:n + 1])
        self._res_host[n:n + 1].copy_(self._res[n:n + 1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return ev

    def read(self, n, handle):
        handle.synchronize()
        return float(self._res_host[n].item())

    def snapshot(self, t):
        return clone_field(t)

    on_device = True

    # wire format of the hand-offs: the field's flat padded storage, sent
    # straight from the state (DistExchange.fence orders later overwrites)
    def to_wire(self, t):
        return flat_storage(t)

    def wire_buffer(self, like):
        return torch.empty(field_elems(tuple(like.shape)), dtype=torch.float64,
                           device=like.device)

    def from_wire(self, buf, like):
        return field_from_flat(buf, tuple(like.shape))


# ---------------------------------------------------------------------------
# exchanges


class _LocalExchange:
    """All ranks in this process: hand-offs read the sender's current state,
    which in the serial issue order equals the reference's snapshot."""

    def __init__(self, engine):
        self.e = engine

    def owns(self, n):
        return True

    def send_pred(self, n, ph):
        pass

    def recv_pred(self, n, ph):
        return self.e.coarse_payload(n - 1)

    def send_coarse(self, n, k):
        pass

    def recv_iteration(self, n, k):
        return self.e.fine_payload(n - 1), self.e.coarse_payload(n - 1)

    def send_fine(self, n, k):
        pass

    def send_flag(self, n, k, flag):
        pass

    def recv_flag(self, n, k):
        return None        # resolved from this process's own bookkeeping

    def fence(self, n):
        pass


class DistExchange:
    """torch.distributed point-to-point hand-offs between processes (NCCL on
    GPUs, gloo in the CPU tests).  Time rank n lives on process n % world.

    Ordering rules that keep NCCL's per-pair stream deadlock-free: payload
    receives are posted when the receiving rank starts its iteration (and
    waited on at once), sends are posted as soon as the payload is final,
    and the 8-byte converged flag is received lazily, right before the host
    needs it.

    No payload is copied for sending: a send reads the sender's live state
    (its flat padded storage), and ``fence(n)`` -- called before rank n's
    next sweep can overwrite that state -- makes the compute stream wait for
    rank n's outstanding sends (a device-side wait under NCCL).  Receives land
    in per-(rank, level) buffers reused across iterations.  With device
    fields on a gloo group (two processes sharing one GPU in the tests) the
    wire is staged through host memory."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.e = engine
        self.group = group
        self.world = dist.get_world_size(group)
        self.me = dist.get_rank(group)
        self._pending = {}       # rank n -> outstanding send works (+ their buffers)
        self._cache = {}         # n -> (fine, coarse) once the predecessor froze
        self._last = {}          # n -> last (fine, coarse) received
        self._last_pred = {}
        self._rbuf = {}          # (n, tag) -> receive buffer
        self.host_wire = dist.get_backend(group) == "gloo" and getattr(engine, "on_device",
                                                                       False)

    def proc(self, n):
        return n % self.world

    def owns(self, n):
        return self.proc(n) == self.me

    def fence(self, n):
        """Rank n's state may be overwritten after this (its sends are done)."""
        for w, _ in self._pending.pop(n, ()):
            w.wait()

    def _send(self, n, t, dst_rank):
        buf = self.e.to_wire(t)
        if self.host_wire:
            buf = buf.cpu()
        w = self.dist.isend(buf, self.proc(dst_rank), group=self.group)
        self._pending.setdefault(n, []).append((w, buf))

    def _recv(self, like, src_rank, n, tag):
        key = (n, tag)
        buf = self._rbuf.get(key)
        if buf is None:
            buf = self._rbuf[key] = self.e.wire_buffer(like)
        if self.host_wire:
            hb = torch.empty(buf.shape, dtype=buf.dtype)
            self.dist.irecv(hb, self.proc(src_rank), group=self.group).wait()
            buf.copy_(hb)
        else:
            self.dist.irecv(buf, self.proc(src_rank), group=self.group).wait()
        return self.e.from_wire(buf, like)

    def send_pred(self, n, ph):
        self._send(n, self.e.coarse_payload(n), n + 1)

    def recv_pred(self, n, ph):
        # rank n-1 took part in phases 0..n-1; phase n re-reads phase n-1
        if ph < n:
            self._last_pred[n] = self._recv(self.e.coarse_payload(n), n - 1, n, "pred")
        return self._last_pred[n]

    def send_coarse(self, n, k):
        self._send(n, self.e.coarse_payload(n), n + 1)

    def recv_iteration(self, n, k):
        if n in self._cache:
            return self._cache[n]
        coarse = self._recv(self.e.coarse_payload(n), n - 1, n, "coarse")
        fine = self._recv(self.e.fine_payload(n), n - 1, n, "fine")
        self._last[n] = (fine, coarse)
        return fine, coarse

    def send_fine(self, n, k):
        self._send(n, self.e.fine_payload(n), n + 1)

    def send_flag(self, n, k, flag):
        buf = torch.tensor([1.0 if flag else 0.0], dtype=torch.float64)
        if not self.host_wire:
            buf = buf.to(self.e.fine_payload(n).device)
        w = self.dist.isend(buf, self.proc(n + 1), group=self.group)
        self._pending.setdefault(-1, []).append((w, buf))

    def recv_flag(self, n, k):
        if n in self._cache:
            return True
        flag = torch.empty(1, dtype=torch.float64)
        if not self.host_wire:
            flag = flag.to(self.e.fine_payload(n).device)
        self.dist.irecv(flag, self.proc(n - 1), group=self.group).wait()
        ok = bool(flag.item() != 0.0)
        if ok:                   # predecessor frozen: keep its final payloads
            self._cache[n] = self._last[n]
        return ok

    def broadcast_final(self, p, like):
        """The last rank's fine value of the block, on every process
        (pfasst.py:272-278)."""
        last = (p - 1) % self.world
        wire = self.e.to_wire(self.e.fine_payload(p - 1)) if self.owns(p - 1) \
            else self.e.wire_buffer(like)
        if self.host_wire:
            host = wire.cpu()
            self.dist.broadcast(host, last, group=self.group)
            if not self.owns(p - 1):
                wire.copy_(host)
        else:
            self.dist.broadcast(wire, last, group=self.group)
        return self.e.snapshot(self.e.from_wire(wire, like))

    def finish(self):
        for n in list(self._pending):
            self.fence(n)
        self._cache.clear()
        self._last.clear()
        self._last_pred.clear()


# ---------------------------------------------------------------------------
# the schedule (pfasst.py:121-253)


class _Block:
    def __init__(self, engine, exchange, p, tol, max_iter, block, record_final_values):
        self.e, self.x = engine, exchange
        self.p, self.tol, self.max_iter, self.block = p, tol, max_iter, block
        self.record = record_final_values
        self.mine = [n for n in range(p) if exchange.owns(n)]
        self.vcycles = [0] * p
        self.iterations = [0] * p
        self.converged = [False] * p
        self.trace = []
        self.final_values = []
        self.frozen = [False] * p
        self.pending = {}        # n -> (k, cycles, residual handle)
        self.status = [dict() for _ in range(p)]   # n -> {k: converged}
        self.solves = []         # ((stage, k or phase, rank, seq), record) when logging
        self.tag = None

    def sink(self, recs):
        """sdc._solve_sink while this block logs solves: tags each record with
        its position in the reference's serial order (predictor phase-major,
        then iteration-major, rank-minor; pfasst.py:213-228)."""
        for r in recs:
            self.solves.append(((*self.tag, len(self.solves)), r))

    def serial_solves(self):
        return [r for _, r in sorted(self.solves, key=lambda t: t[0])]

    def predictor(self):
        """pfasst.py:166-181, phase-major (serial order)."""
        e, x, p = self.e, self.x, self.p
        for ph in range(p):
            for n in range(ph, p):
                if not x.owns(n):
                    continue
                if n > 0:
                    e.set_coarse_y0(n, x.recv_pred(n, ph))
                x.fence(n)          # the sweep overwrites the last coarse payload
                self.tag = (0, ph, n)
                self.vcycles[n] += e.burn_in(n)
                if n + 1 < p and not x.owns(n + 1):
                    x.send_pred(n, ph)
                elif n + 1 < p:
                    pass  # local receiver reads the state directly
        for n in self.mine:
            e.interpolate_up(n, exact=(n == 0))

    def _resolve(self, n):
        """Read rank n's residual of its last live iteration and settle its
        converged flag (pfasst.py:200-210)."""
        if n not in self.pending:
            return
        k, cyc, handle = self.pending.pop(n)
        res = self.e.read(n, handle)
        if n == 0:
            pred_ok = True
        elif self.x.owns(n - 1):
            if n - 1 in self.pending and self.pending[n - 1][0] == k:
                self._resolve(n - 1)
            # a predecessor frozen before k resends converged=True
            pred_ok = self.status[n - 1].get(k, True)
        else:
            pred_ok = self.x.recv_flag(n, k)
        ok = (res <= self.tol) and pred_ok
        self.status[n][k] = ok
        self.converged[n] = ok
        self.frozen[n] = ok
        self.trace.append(TraceRow(self.block, n, k, 0, res, cyc))
        if n + 1 < self.p and not self.x.owns(n + 1):
            self.x.send_flag(n, k, ok)

    def _schedule(self):
        """(k, n) issue order of this process's ranks.  One process (or one
        owned rank): the reference's serial order, k-major.  Several owned
        ranks on a process of the nccl executor (cyclic placement, G < P):
        anti-diagonals d = n + k ascending, n descending -- rank n's iteration
        k needs rank n-1's iteration k, which its owner issued on diagonal
        d - 1, so no process waits inside a diagonal and the G processes run
        concurrently instead of handing one iteration around the ring.  Every
        process uses the same global order, so the messages between any pair
        of processes are posted and matched in the same sequence on both
        sides; convergence decisions are unchanged."""
        if len(self.mine) <= 1 or isinstance(self.x, _LocalExchange):
            for k in range(1, self.max_iter + 1):
                yield k, None
            return
        for d in range(1, self.max_iter + self.p):
            for n in sorted(self.mine, reverse=True):
                k = d - n
                if 1 <= k <= self.max_iter:
                    yield k, n

    def iterations_loop(self):
        e, x, p = self.e, self.x, self.p
        stopped = set()
        for k, only in self._schedule():
            active = False
            for n in (self.mine if only is None else (only,)):
                if n in stopped:
                    continue
                self._resolve(n)
                if self.frozen[n]:
                    if only is not None:
                        stopped.add(n)
                    continue
                active = True
                x.fence(n)          # this iteration overwrites the payloads sent
                if n > 0:
                    fine, coarse = x.recv_iteration(n, k)
                    e.set_fine_y0(n, fine)
                    coarse_msg = coarse
                    pre = (lambda ts, n=n, c=coarse_msg: e.set_coarse_y0(n, c))
                else:
                    pre = None
                # the local exchange hands over the predecessor's coarse value
                # by reading its state inside the pre-coarse hook (same as the
                # reference's blocking coarse recv, pfasst.py:107-112)
                self.tag = (1, k, n)
                cyc = e.iteration(n, pre)
                if n + 1 < p and not x.owns(n + 1):
                    # coarse payload was produced by the coarse sweep; the fine
                    # one by the finest sweep -- both final now
                    x.send_coarse(n, k)
                    x.send_fine(n, k)
                handle = e.residual(n)
                self.vcycles[n] += cyc
                self.iterations[n] = k
                self.pending[n] = (k, cyc, handle)
                if self.record and n == p - 1:
                    self.final_values.append(e.snapshot(e.fine_payload(n)))
            if not active and only is None:
                break
        for n in self.mine:
            self._resolve(n)


    def iterations_wavefront(self):
        """The iteration loop issued by anti-diagonals d = n + k (descending n
        inside a diagonal), one CUDA stream per rank.  Convergence decisions
        are taken exactly as in the serial loop; only the issue order and the
        overlap on the device differ."""
        e, p = self.e, self.p
        caller = torch.cuda.current_stream()
        for n in range(p):
            e.streams[n].wait_stream(caller)
        done_ev = [None] * p       # rank n's payload of its latest issued iteration is final
        copied_ev = [None] * p     # rank n took its copies of rank n-1's payload
        issued = [0] * p
        stopped = [False] * p
        for d in range(1, self.max_iter + p):
            for n in range(p - 1, -1, -1):
                k = d - n
                if k < 1 or k > self.max_iter or stopped[n]:
                    continue
                self._resolve(n)
                if self.frozen[n]:
                    stopped[n] = True
                    continue
                st = e.streams[n]
                with torch.cuda.stream(st):
                    pre = None
                    if n > 0:
                        st.wait_event(done_ev[n - 1])
                        e.set_fine_y0(n, e.fine_payload(n - 1))
                        coarse = e.stage_coarse(n, e.coarse_payload(n - 1))
                        pre = (lambda ts, n=n, c=coarse: e.set_coarse_y0(n, c))
                        copied_ev[n] = torch.cuda.Event()
                        copied_ev[n].record(st)
                    # the successor's copy of this rank's previous payload
                    if n + 1 < p and issued[n + 1] == k - 1 and copied_ev[n + 1] is not None:
                        st.wait_event(copied_ev[n + 1])
                    self.tag = (1, k, n)
                    cyc = e.iteration(n, pre)
                    handle = e.residual(n)
                    done_ev[n] = torch.cuda.Event()
                    done_ev[n].record(st)
                    if self.record and n == p - 1:
                        self.final_values.append(e.snapshot(e.fine_payload(n)))
                self.vcycles[n] += cyc
                self.iterations[n] = k
                issued[n] = k
                self.pending[n] = (k, cyc, handle)
        for n in self.mine:
            self._resolve(n)
        for n in range(p):
            caller.wait_stream(e.streams[n])


def _rank_stream_options():
    """pl_set_option values held while the rank-stream wavefront runs:
    {key: (value, library default)}.  PINTLAB_RANK_STREAM_OPTS="K=V,..." (A/B
    runs) replaces the built-in choice."""
    import os

    from . import _capi as capi
    defaults = {capi.OPT_MID: 1, capi.OPT_MID_CTAS: 0, capi.OPT_ZMARCH_MIN_N: 127}
    env = os.environ.get("PINTLAB_RANK_STREAM_OPTS")
    if env is None:   # A/B on one box, 5 steps each: see DESIGN.md section 4
        return {capi.OPT_MID: (0, 1), capi.OPT_ZMARCH_MIN_N: (63, 127)}
    out = {}
    for kv in filter(None, env.split(",")):
        k, v = (int(x) for x in kv.split("="))
        out[k] = (v, defaults.get(k, 0))
    return out


def _rank_streams_fit(levels, p) -> bool:
    """Per-rank streams give each time rank its own sweep / multigrid scratch.
    Use them only when that extra memory (a conservative 2x of the sweep and
    multigrid workspaces per level) fits in half of the free device memory;
    otherwise the single-stream schedule runs (same results)."""
    from . import _capi as capi
    lib = capi.lib()
    per = 0
    for lv in levels:
        g = lv.operator.grid
        per += 2 * (lib.pl_sweep_workspace_bytes(g.dim, g.n, lv.table.m) +
                    lib.pl_mg_workspace_bytes(g.dim, g.n, lv.mg_cfg.coarsest_n))
    free, _ = torch.cuda.mem_get_info()
    return (p - 1) * per <= 0.5 * free


def _run_block(blk, engine, exchange):
    """Predictor and iterations of one block (pfasst.py:213-228)."""
    blk.predictor()
    if isinstance(exchange, _LocalExchange) and getattr(engine, "streams", None):
        # rank streams overlap each other's work: the small V-cycle levels
        # then run as ordinary per-level launches (no cooperative grid that
        # must be co-resident on every SM; the TMA sweeps from 63^3 up) and
        # interleave with the other ranks' kernels -- +15-25 % time-steps/s
        # against the one-CTA-per-SM cooperative kernel, which a lone solve
        # keeps (results are bit-identical either way)
        from contextlib import ExitStack

        from . import _capi as capi
        with ExitStack() as scope:
            for key, (value, default) in _rank_stream_options().items():
                scope.enter_context(capi.option(key, value, default))
            blk.iterations_wavefront()
    else:
        blk.iterations_loop()


_ENGINE_CACHE: list = []     # [(key, engine)] of the most recent pfasst_run configuration


def _device_engine(levels, dt, ranks, streams):
    """The DeviceEngine of a previous pfasst_run when it ran the same level
    objects, dt, ranks and stream mode on this device: its per-rank state
    buffers are re-spread rather than reallocated, so repeated runs keep their
    device addresses (and the captured sweep graphs keyed by them).  One
    engine per schedule (rank streams / single stream) of the most recent
    configuration is kept, the second only while more than a quarter of the
    device memory stays free; a run with other levels, dt or ranks replaces
    them."""
    base = (tuple(id(lv) for lv in levels), float(dt), tuple(ranks),
            torch.cuda.current_device())
    key = base + (bool(streams),)
    for k, eng in _ENGINE_CACHE:
        if k == key and all(a is b for a, b in zip(eng.levels, levels)):
            return eng
    if any(k[:-1] != base or not all(a is b for a, b in zip(e.levels, levels))
           for k, e in _ENGINE_CACHE):
        _ENGINE_CACHE.clear()
    engine = DeviceEngine(levels, dt, ranks, streams=streams)
    _ENGINE_CACHE.append((key, engine))
    return engine


def _trim_engines():
    """Keep the other schedule's engine only while memory is plentiful."""
    if len(_ENGINE_CACHE) > 1:
        free, total = torch.cuda.mem_get_info()
        if free < 0.25 * total:
            del _ENGINE_CACHE[0]


def release_engines():
    """Drop the cached engine (its device buffers)."""
    _ENGINE_CACHE.clear()


def _gather_block(blk, exchange):
    """Combine per-process bookkeeping (nccl executor)."""
    if not isinstance(exchange, DistExchange):
        return blk.iterations, blk.vcycles, blk.converged, blk.trace, blk.serial_solves()
    dist = exchange.dist
    mine = {n: (blk.iterations[n], blk.vcycles[n], blk.converged[n]) for n in blk.mine}
    rows = [(r.block, r.rank, r.iteration, r.level, r.residual, r.vcycles) for r in blk.trace]
    gathered = [None] * exchange.world
    dist.all_gather_object(gathered, (mine, rows, blk.solves), group=exchange.group)
    it, vc, cv, tr, sv = [0] * blk.p, [0] * blk.p, [False] * blk.p, [], []
    for m, rws, solves in gathered:
        for n, (a, b, c) in m.items():
            it[n], vc[n], cv[n] = a, b, c
        tr.extend(TraceRow(*r) for r in rws)
        sv.extend(solves)
    return it, vc, cv, tr, [r for _, r in sorted(sv, key=lambda t: t[0])]


def _world(group):
    import torch.distributed as dist
    return dist.get_world_size(group) if dist.is_initialized() else 1


def pfasst_run(levels, u0, t_end: float, p: int, blocks: int = 1, tol: float = 1e-9,
               max_iter: int = 20, executor: str = "serial", record_final_values: bool = False,
               engine_factory=None, group=None, streams: bool = True,
               solve_log: list | None = None, out=None) -> PfasstResult:
    """Run PFASST / IPFASST over ``blocks`` windows of ``p`` steps (pfasst.py:256-287).

    ``u0`` may be a numpy array (result returned on the host, drop-in) or an
    fp64 CUDA tensor (result stays on the device).  ``streams`` (single
    process only) issues each time rank on its own CUDA stream in wavefront
    order when the per-stream scratch fits (``_rank_streams_fit``); results
    are identical either way.

    ``solve_log`` (optional list) receives, per block, the list of
    ``[n, sigma, cycles, status]`` records of every sub-step solve in the
    reference's serial order (predictor, then iterations; the parity aid of
    the oracle's per-solve log), whatever the executor or issue order.

    ``out`` (optional, with host input): a caller-owned host buffer of the
    fine grid's shape -- a numpy array or a CPU tensor, ideally pinned -- that
    receives the final value and is returned as ``result.u``.  A fresh pageable
    array costs ~64 ms per 133 MB result (page faults and a staged copy); a
    reused pinned buffer 2.5 ms."""
    check_hierarchy(levels)
    if out is not None:
        out_t = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
        if out_t.is_cuda or out_t.dtype != torch.float64 or \
                tuple(out_t.shape) != tuple(levels[0].grid.shape) or not out_t.is_contiguous():
            raise ValueError("out must be a contiguous fp64 host buffer of the fine grid's shape")
    if executor not in ("serial", "threaded", "nccl"):
        raise ValueError(f"unknown executor {executor!r}")
    if p < 1 or blocks < 1:
        raise ValueError("need at least one rank and one block")
    dt = t_end / (p * blocks)
    if engine_factory is None:
        u, host = to_device(u0, levels[0].grid.dim)
        engine_factory = DeviceEngine
    else:                       # test hook: alternative engines (CPU oracle)
        u, host = u0, False
    result = PfasstResult(u=u0)
    engine = None
    for block in range(blocks):
        if executor == "nccl" and _world(group) > 1:
            import torch.distributed as dist
            world = dist.get_world_size(group)
            me = dist.get_rank(group)
            ranks = [n for n in range(p) if n % world == me]
            if engine is None:
                engine = (_device_engine(levels, dt, ranks, False)
                          if engine_factory is DeviceEngine else
                          engine_factory(levels, dt, ranks))
            exchange = DistExchange(engine, group)
        else:
            if engine is None:
                if engine_factory is DeviceEngine:
                    use = streams and p > 1 and _rank_streams_fit(levels, p)
                    engine = _device_engine(levels, dt, range(p), use)
                else:
                    engine = engine_factory(levels, dt, range(p))
            exchange = _LocalExchange(engine)
        for n in range(p):
            if exchange.owns(n):
                engine.spread(n, u)
        blk = _Block(engine, exchange, p, tol, max_iter, block, record_final_values)
        if solve_log is not None:
            from . import sdc as _sdc
            _sdc._solve_sink = blk.sink
        try:
            _run_block(blk, engine, exchange)
        finally:
            if solve_log is not None:
                _sdc._solve_sink = None
        if isinstance(exchange, DistExchange):
            exchange.finish()
            last = (p - 1) % exchange.world
            like = engine.fine_payload(engine.ranks[0]) if engine.ranks else u
            u = exchange.broadcast_final(p, like)
            if record_final_values:
                fv = [v.contiguous().cpu().numpy() for v in blk.final_values] \
                    if exchange.owns(p - 1) else None
                holder = [fv]
                exchange.dist.broadcast_object_list(holder, last, group=group)
                blk.final_values = holder[0]
        else:
            u = engine.snapshot(engine.fine_payload(p - 1))
        it, vc, cv, tr, sv = _gather_block(blk, exchange)
        if solve_log is not None:
            solve_log.append(sv)
        result.rank_iterations.append(list(it))
        result.rank_vcycles.append(list(vc))
        result.converged.append(list(cv))
        result.trace.extend(sorted(tr, key=lambda r: (r.iteration, r.rank, r.level)))
        result.final_values.append([like_input(v, host) if isinstance(v, torch.Tensor)
                                    else v for v in blk.final_values])
    if engine_factory is DeviceEngine:
        _trim_engines()
    if out is not None and isinstance(u, torch.Tensor) and u.is_cuda:
        out_t.copy_(u)             # synchronous: the caller may read out right away
        result.u = out
    else:
        result.u = like_input(u, host)
    return result


def predictor_sweep_counts(p: int) -> list:
    """pfasst.py:290-292."""
    return [n + 1 for n in range(p)]


def write_trace_csv(rows, path: str) -> None:
    """pfasst.py:295-300 (byte-identical format)."""
    with open(path, "w") as fh:
        fh.write("block,rank,iter,level,residual,vcycles\n")
        for r in rows:
            fh.write(f"{r.block},{r.rank},{r.iteration},{r.level},"
                     f"{r.residual:.16e},{r.vcycles}\n")

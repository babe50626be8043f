"""RW-TTT serving loop (Alg. 1; full loop App. H) over the C ABI.

    View -> NextStep -> LegalGroups -> ExecuteOperatorGroup -> ReturnOutputs
         -> CommitVersions (WRITE) -> UpdateKVAndTailMetadata

Python here only sequences calls into libtttstate.so.  The default step is ONE
native call per decode step, `tttstate_serve_step` (NextStep -> plan_batch ->
L read_apply launches per group -> step done / write_commit, with the App. H
singleton retry of a group that hits an injected failure), so the host cost
per step does not grow with the layer count and nothing waits for the GPU.
Controls (snapshot / rollback / fork / release) are issued before the step.
`step_percall()` sequences the same operators with one C-ABI call per
operator (the stress suite uses it to inspect state between calls).

Commits are provisional until confirmed (include/tttstate.h "Commit
confirmation"): the device refuses a member whose candidate is not finite and
resolves App. H's singleton retries itself.  `finish()` (or `drain()`)
synchronises, reads the device refusal records and writes the final commit log:
a group with a refused member is logged as failed, then each member's singleton
outcome.  PyTorch provides the device arena and streams only.
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import torch

from . import capi
from .capi import READ, WRITE, Group, TTTError


class Engine:
    """One TTTState pool (placement π = this device) plus its planner."""

    def __init__(self, d_model: int, d_ff: int, chunk: int, n_layers: int, dtype: str, max_owners: int,
                 w_down: torch.Tensor, n_ckpt: int = 0, mode: int = capi.MODE_FULL, B: int = 8, w: int = 0,
                 shape_id: int = 0, placement: int = 0, device=None, eta: float = 0.01,
                 backend: int = capi.FAST_WEIGHT, rank: int = 0, rule: int = 0):
        device = torch.device(device) if device is not None else w_down.device
        assert w_down.is_cuda, "w_down must be a device tensor"
        self.d_model, self.d_ff, self.chunk, self.n_layers, self.dtype = d_model, d_ff, chunk, n_layers, dtype
        self.tdtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.eta = float(torch.tensor(eta, dtype=torch.float32))
        self.shape = capi.make_shape(d_model, d_ff, chunk, n_layers, dtype, backend=backend, rank=rank, rule=rule)
        self.backend, self.rank = backend, rank
        self.max_owners = max_owners
        self.arena_bytes = capi.tttstate_pool_bytes(self.shape, max_owners, n_ckpt)
        self._arena = torch.empty(self.arena_bytes + 1024, dtype=torch.uint8, device=device)
        base = (self._arena.data_ptr() + 1023) // 1024 * 1024
        self.w_down = w_down
        self.pool = capi.tttstate_pool_create(self.shape, shape_id, placement, max_owners, n_ckpt, base,
                                              self.arena_bytes, w_down)
        capi.tttstate_set_eta(self.pool, self.eta)
        self.planner = capi.ttt_planner_create(mode, B, w)
        capi.ttt_planner_attach(self.planner, self.pool)
        self.shape_id, self.placement, self.device = shape_id, placement, device

    def close(self):
        if self.planner:
            capi.ttt_planner_destroy(self.planner)
            self.planner = None
        if self.pool:
            capi.tttstate_pool_destroy(self.pool)
            self.pool = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class RunLog:
    commits: list = field(default_factory=list)     # (s, p, v_before, v_after, outcome)
    census: dict = field(default_factory=lambda: {READ: 0, WRITE: 0})
    plan: list = field(default_factory=list)        # (issue_step, effect, [streams], [ready])
    versions: dict = field(default_factory=dict)
    fallbacks: int = 0
    device_failures: int = 0                        # groups with a member refused on the device
    rejected: int = 0                               # planner rejections (re-extracted next step)
    rollbacks: int = 0
    branches: dict = field(default_factory=dict)    # live branch owner -> version


@dataclass
class StepIO:
    """One decode step's device operands: layer l of X / Vt / Y starts *_stride elements after
    layer l-1; the token of the i-th listed stream sits at row rows[i] of every layer."""
    X: torch.Tensor
    x_stride: int
    Vt: torch.Tensor
    v_stride: int
    Y: torch.Tensor
    y_stride: int
    rows: list
    rows_total: int = 0           # rows of each layer's X / Vt / Y (0: unknown)


class InputSource:
    """Where a run's per-token inputs come from and where outputs go (device tensors)."""

    def init_delta(self, s: int):                 # device [L, d_model, d_ff] or None (ΔW_0 = 0)
        return None

    def tail_prefill(self, s: int):               # (n, Z [L,n,d_ff], V [L,n,d_model]) or None
        return None

    def step_io(self, streams, positions) -> StepIO:
        """Operands of one native step for the listed (stream, position) tokens."""
        raise NotImplementedError

    def on_step(self, executed, io: StepIO):
        """executed: [(s, p, row)] tokens the step ran (ReturnOutputs); their y is in io.Y."""

    # per-operator path (Server.step_percall)
    def group_io(self, l: int, streams, positions):
        """-> (X, x_rows, Vt, v_rows, Y, y_rows) device tensors (+ row maps or None)."""
        raise NotImplementedError

    def on_output(self, l: int, streams, positions, Y, y_rows):
        pass


class Server:
    """Alg. 1 state for one trace: per-stream position, pending events, logs.

    `step()` runs exactly one iteration of the serving loop at the current clock
    (one native call).  With `profile=True` CUDA events on `stream` bracket every
    `profile_every`-th READ-only step (read_events: (start, end, READ launches))
    and every step's first WRITE (write_events), for bench.py's live rooflines.
    """

    def __init__(self, eng: Engine, tr, src: InputSource, stream=None, profile: bool = False,
                 profile_every: int = 1, native: bool = True):
        self.eng, self.tr, self.src, self.stream = eng, tr, src, stream
        self.profile, self.profile_every = profile, max(1, profile_every)
        self.native = native and os.environ.get("TTT_NATIVE_STEP", "1") != "0"   # A/B switch: per-operator calls
        self.log = RunLog()
        self.owners = [tr.owner(s) for s in range(tr.n_streams)]
        self.by_owner = {o: s for s, o in enumerate(self.owners)}
        self.pos = [0] * tr.n_streams
        self.pending: set = set()
        self.ready_at: dict = {}
        self.failed_once: set = set()
        self.forks: dict = {}
        self.branches: set = set()
        self.clock = 0
        self.read_events: list = []       # (start, end, launches): events around a step's back-to-back READs
        self.write_events: list = []      # (start, end) around the step's first write_commit
        self.plan_s = 0.0                 # host seconds in View/controls + marshalling (P:525's overhead share)
        self._items: list = []            # commit log items, expanded by drain() (provisional commits)
        self._has_controls = bool(tr.controls)
        self._vtrue = {s: tr.v0 for s in range(tr.n_streams)}   # confirmed version replay (drain)
        self.bufs = capi.StepBuffers(eng.max_owners)
        self._wev = self._fresh_pair() if profile else (None, None)

    def _stream_obj(self):
        return torch.cuda.current_stream() if self.stream is None else self.stream

    def _fresh_pair(self):
        pair = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for e in pair:                    # materialise the cudaEvent_t the library records into
            e.record(self._stream_obj())
        return pair

    def _ev(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record(self._stream_obj())
        return e

    def admit(self):
        eng, tr, src = self.eng, self.tr, self.src
        for s, o in enumerate(self.owners):
            capi.tttstate_alloc(eng.pool, o, src.init_delta(s), tr.v0, self.stream)
            pre = src.tail_prefill(s)
            if pre is not None:
                capi.tttstate_tail_load(eng.pool, o, pre[0], pre[1], pre[2], self.stream)

    def done(self) -> bool:
        return all(p >= self.tr.n_steps for p in self.pos)

    # ---------------------------------------------------------------- View + controls
    def _controls(self, s):
        pool, stream, log, tr = self.eng.pool, self.stream, self.log, self.tr
        o = self.owners[s]
        for op in tr.controls_at(s, self.pos[s]):
            if op == "snapshot":
                capi.tttstate_snapshot(pool, o, stream)
            elif op == "rollback":                              # v_before comes from drain()'s replay
                va = capi.rollback(pool, o, stream)
                self._items.append(("rb", s, self.pos[s], None, va))
                log.rollbacks += 1
            elif op == "fork":                                  # new lineage
                k = self.forks.get(s, 0)
                capi.tttstate_fork(pool, o, tr.branch_owner(s, k), stream)
                self.branches.add(tr.branch_owner(s, k))
                self.forks[s] = k + 1
            elif op == "release":
                b = tr.branch_owner(s, self.forks[s] - 1)
                capi.tttstate_free(pool, b)
                self.branches.discard(b)

    def _injected(self, s) -> bool:
        p = self.pos[s]
        return self._has_controls and "fail" in self.tr.controls_at(s, p) and (s, p) not in self.failed_once

    def step(self):
        if not self.native:
            return self.step_percall()
        eng, tr, src, log, bufs = self.eng, self.tr, self.src, self.log, self.bufs
        clock = self.clock
        t0 = time.perf_counter()
        active = [s for s in range(tr.n_streams) if self.pos[s] < tr.n_steps]
        n_fail = 0
        for s in active:
            if s not in self.pending:
                if self._has_controls:
                    self._controls(s)
                self.ready_at[s] = clock
            if self._injected(s):
                bufs.fail[n_fail] = self.owners[s]
                n_fail += 1
        io = src.step_io(active, [self.pos[s] for s in active])
        for i, s in enumerate(active):
            bufs.owners[i] = self.owners[s]
            bufs.rows[i] = io.rows[i]
        prof = self.profile and clock % self.profile_every == 0
        if prof:
            e0 = self._ev()
        self.plan_s += time.perf_counter() - t0
        out = capi.tttstate_serve_step(eng.pool, eng.planner, bufs, len(active), clock, io.X, io.x_stride, io.Vt,
                                       io.v_stride, io.Y, io.y_stride, tr.eta, n_fail, stream=self.stream,
                                       ev_write=self._wev, rows_total=io.rows_total)
        t1 = time.perf_counter()
        for s in active:
            self.pending.add(s)
        for k in range(out.n_rejected):                          # stale pending events: re-extract
            self.pending.discard(self.by_owner[bufs.rejected[k].owner])
            log.rejected += 1
        executed = []
        n_read_launches = 0
        row_of = {s: io.rows[i] for i, s in enumerate(active)}
        for eff, owners, vb, seqs, inj in bufs.groups_issued():
            ss = [self.by_owner[o] for o in owners]
            ps = [self.pos[s] for s in ss]
            log.plan.append((clock, eff, ss, [self.ready_at[s] for s in ss]))
            log.census[eff] += len(ss)
            if eff == READ:
                n_read_launches += (len(ss) + 7) // 8
            else:
                if inj:
                    for s, p in zip(ss, ps):
                        self.failed_once.add((s, p))
                        self._items.append(("fail", s, p))
                    log.fallbacks += 1
                    for o, s, p, q in zip(owners, ss, ps, seqs):   # singleton retries
                        self._items.append(("single", q, o, s, p))
                else:
                    self._items.append(("group", seqs[0], list(zip(owners, ss, ps))))
            for s in ss:
                executed.append((s, self.pos[s], row_of[s]))
                self.pos[s] += 1
                self.pending.discard(s)
        src.on_step(executed, io)
        if self.profile:
            if out.n_write:
                self.write_events.append(self._wev)
                self._wev = self._fresh_pair()
            elif prof and n_read_launches:
                self.read_events.append((e0, self._ev(), n_read_launches * tr.n_layers))
        self.plan_s += time.perf_counter() - t1
        self.clock += 1

    # ---------------------------------------------------------------- per-operator path
    def step_percall(self):
        eng, tr, src, log, stream = self.eng, self.tr, self.src, self.log, self.stream
        pool, owners, clock = eng.pool, self.owners, self.clock
        t_plan = time.perf_counter()
        ready = []
        for s in range(tr.n_streams):                                   # View + controls
            if self.pos[s] < tr.n_steps and s not in self.pending:
                ready.append(s)
                self._controls(s)
        events = capi.tttstate_next_events(pool, [owners[s] for s in ready], clock) if ready else []
        for s in ready:
            self.pending.add(s)
            self.ready_at[s] = clock
        groups, rejected = capi.plan_batch(eng.planner, events, clock)  # LegalGroups
        self.plan_s += time.perf_counter() - t_plan
        for r in rejected:
            self.pending.discard(self.by_owner[r.owner])
            log.rejected += 1
        for g in groups:
            ss = [self.by_owner[o] for o in g.owners]
            ps = [self.pos[s] for s in ss]
            log.plan.append((g.issue_step, g.effect, ss, [self.ready_at[s] for s in ss]))
            for l in range(tr.n_layers):                                # ExecuteOperatorGroup
                X, xr, Vt, vr, Y, yr = src.group_io(l, ss, ps)
                capi.read_apply(pool, g, l, X, xr, Vt, vr, Y, yr, None, stream)
                src.on_output(l, ss, ps, Y, yr)                         # ReturnOutputs
            log.census[g.effect] += len(ss)
            if g.effect == READ:
                capi.tttstate_step_done(pool, g)                        # UpdateKVAndTailMetadata
            else:
                self._write_percall(g, ss, ps)
            for s in ss:
                self.pos[s] += 1
                self.pending.discard(s)
        self.clock += 1

    def _write_percall(self, g, ss, ps):
        tr, log, stream, pool = self.tr, self.log, self.stream, self.eng.pool
        mask = [self._injected(s) for s in ss]
        try:                                                            # CommitVersions
            capi.write_commit(pool, g, tr.eta, mask if any(mask) else None, stream)
            self._items.append(("group", capi.tttstate_last_commit_seq(pool), list(zip(g.owners, ss, ps))))
            return
        except TTTError as e:
            if e.status != capi.TTT_E_WRITE_FAILED:
                raise
        for s, p in zip(ss, ps):
            self.failed_once.add((s, p))
            self._items.append(("fail", s, p))
        log.fallbacks += 1
        for s, p, o in zip(ss, ps, g.owners):                           # App. H fallback: singletons
            single = Group(WRITE, [o], g.c.shape_id, g.c.placement, g.c.backend, self.clock)
            capi.write_commit(pool, single, tr.eta, None, stream)
            self._items.append(("single", capi.tttstate_last_commit_seq(pool), o, s, p))

    # ---------------------------------------------------------------- confirmation + log
    def drain(self):
        """Synchronise, read the device refusal records and expand the provisional commits
        into the final log, replaying each stream's committed version (the host mirror's
        versions are provisional while commits are unconfirmed): a group with a refused member
        is logged failed, then each member's singleton outcome (App. H); a refused singleton
        is logged failed."""
        pool, log = self.eng.pool, self.log
        capi.tttstate_sync(pool, self.stream)
        refused = {(q, o) for o, _v, q in capi.tttstate_refusals(pool, self.stream)}
        vt = self._vtrue

        def one(s, p, ok):
            v = vt[s]
            log.commits.append((s, p, v, v + 1, "ok") if ok else (s, p, v, v, "failed"))
            vt[s] = v + 1 if ok else v

        for it in self._items:
            if it[0] == "group":
                _, q, mem = it
                bad = [(q, o) in refused for o, _, _ in mem]
                if any(bad):
                    log.fallbacks += 1
                    log.device_failures += 1
                    for _o, s, p in mem:
                        one(s, p, False)
                for (_o, s, p), b in zip(mem, bad):
                    one(s, p, not b)
            elif it[0] == "single":
                _, q, o, s, p = it
                one(s, p, (q, o) not in refused)
            elif it[0] == "fail":
                one(it[1], it[2], False)
            else:                                               # ("rb", s, p, v_before, v_after)
                _, s, p, vb, va = it
                log.commits.append((s, p, vt[s] if vb is None else vb, va, "rolled_back"))
                vt[s] = va
        self._items = []

    def finish(self) -> RunLog:
        self.drain()
        for s, o in enumerate(self.owners):
            self.log.versions[s] = capi.tttstate_version(self.eng.pool, o)
        for b in self.branches:
            self.log.branches[b] = capi.tttstate_version(self.eng.pool, b)
        return self.log


def run_trace(eng: Engine, tr, src: InputSource, stream=None, max_clock: int | None = None,
              native: bool = True) -> RunLog:
    """Alg. 1 over a workload.traces.Trace (App. H: fallback + wait budget)."""
    srv = Server(eng, tr, src, stream, native=native)
    srv.admit()
    while not srv.done():
        if max_clock is not None and srv.clock >= max_clock:
            break
        srv.step()
    return srv.finish()

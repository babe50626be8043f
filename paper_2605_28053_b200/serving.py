"""RW-TTT serving loop (Alg. 1; full loop App. H) over the C ABI.

    View -> NextStep -> LegalGroups -> ExecuteOperatorGroup -> ReturnOutputs
         -> CommitVersions (WRITE) -> UpdateKVAndTailMetadata

Python here only sequences calls into libtttstate.so: event extraction
(tttstate_next_event), planning (plan_batch), READ (read_apply), WRITE +
commit (write_commit), control (snapshot / rollback) all run natively.  A
WRITE group that fails is re-run as serial singletons in μ order (App. H
fallback handling).  PyTorch provides the device arena and
streams only.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import time

import torch

from . import capi
from .capi import READ, WRITE, Group, TTTError


class Engine:
    """One TTTState pool (placement π = this device) plus its planner."""

    def __init__(self, d_model: int, d_ff: int, chunk: int, n_layers: int, dtype: str, max_owners: int,
                 w_down: torch.Tensor, n_ckpt: int = 0, mode: int = capi.MODE_FULL, B: int = 8, w: int = 0,
                 shape_id: int = 0, placement: int = 0, device=None, eta: float = 0.01,
                 backend: int = capi.FAST_WEIGHT, rank: int = 0):
        device = torch.device(device) if device is not None else w_down.device
        assert w_down.is_cuda, "w_down must be a device tensor"
        self.d_model, self.d_ff, self.chunk, self.n_layers, self.dtype = d_model, d_ff, chunk, n_layers, dtype
        self.tdtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.eta = float(torch.tensor(eta, dtype=torch.float32))
        self.shape = capi.make_shape(d_model, d_ff, chunk, n_layers, dtype, backend=backend, rank=rank)
        self.backend, self.rank = backend, rank
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
    device_failures: int = 0
    branches: dict = field(default_factory=dict)    # live branch owner -> version


class InputSource:
    """Where a run's per-token inputs come from and where outputs go (device tensors)."""

    def init_delta(self, s: int):                 # device [L, d_model, d_ff] or None (ΔW_0 = 0)
        return None

    def tail_prefill(self, s: int):               # (n, Z [L,n,d_ff], V [L,n,d_model]) or None
        return None

    def group_io(self, l: int, streams, positions):
        """-> (X, x_rows, Vt, v_rows, Y, y_rows) device tensors (+ row maps or None)."""
        raise NotImplementedError

    def on_output(self, l: int, streams, positions, Y, y_rows):
        pass


class Server:
    """Alg. 1 state for one trace: per-stream position, pending events, logs.

    `step()` runs exactly one iteration of the serving loop at the current
    clock.  With `profile=True` every read_apply / write_commit is bracketed by
    CUDA events on `stream` (used by bench.py for the live per-kernel roofline).
    """

    def __init__(self, eng: Engine, tr, src: InputSource, stream=None, sync_writes: bool = True,
                 profile: bool = False, profile_every: int = 1):
        self.eng, self.tr, self.src, self.stream = eng, tr, src, stream
        self.sync_writes, self.profile, self.profile_every = sync_writes, profile, max(1, profile_every)
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
        self.write_events: list = []      # (start, end) around write_commit
        self.plan_s = 0.0                 # host seconds in NextStep + LegalGroups (P:525's overhead)

    def admit(self):
        eng, tr, src = self.eng, self.tr, self.src
        for s, o in enumerate(self.owners):
            capi.tttstate_alloc(eng.pool, o, src.init_delta(s), tr.v0, self.stream)
            pre = src.tail_prefill(s)
            if pre is not None:
                capi.tttstate_tail_load(eng.pool, o, pre[0], pre[1], pre[2], self.stream)

    def done(self) -> bool:
        return all(p >= self.tr.n_steps for p in self.pos)

    def _ev(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream() if self.stream is None else self.stream)
        return e

    def step(self):
        eng, tr, src, log, stream = self.eng, self.tr, self.src, self.log, self.stream
        pool, owners, clock = eng.pool, self.owners, self.clock
        t_plan = time.perf_counter()
        ready = []
        for s in range(tr.n_streams):                                   # View + controls
            if self.pos[s] < tr.n_steps and s not in self.pending:
                ready.append(s)
                for op in tr.controls_at(s, self.pos[s]):
                    if op == "snapshot":
                        capi.tttstate_snapshot(pool, owners[s], stream)
                    elif op == "rollback":
                        vb = capi.tttstate_version(pool, owners[s])
                        va = capi.rollback(pool, owners[s], stream)
                        log.commits.append((s, self.pos[s], vb, va, "rolled_back"))
                    elif op == "fork":                                  # new lineage
                        k = self.forks.get(s, 0)
                        capi.tttstate_fork(pool, owners[s], tr.branch_owner(s, k), stream)
                        self.branches.add(tr.branch_owner(s, k))
                        self.forks[s] = k + 1
                    elif op == "release":
                        b = tr.branch_owner(s, self.forks[s] - 1)
                        capi.tttstate_free(pool, b)
                        self.branches.discard(b)
        # NextStep for every ready stream in one call
        events = capi.tttstate_next_events(pool, [owners[s] for s in ready], clock) if ready else []
        for s in ready:
            self.pending.add(s)
            self.ready_at[s] = clock
        groups, rejected = capi.plan_batch(eng.planner, events, clock)  # LegalGroups
        self.plan_s += time.perf_counter() - t_plan
        if rejected:
            raise RuntimeError(f"planner rejected events of a well-formed trace: {rejected}")
        for g in groups:
            ss = [self.by_owner[o] for o in g.owners]
            ps = [self.pos[s] for s in ss]
            log.plan.append((g.issue_step, g.effect, ss, [self.ready_at[s] for s in ss]))
            prof = self.profile and clock % self.profile_every == 0
            if prof:                    # one event pair per group: per-launch events would break PDL overlap
                e0 = self._ev()
            for l in range(tr.n_layers):                                # ExecuteOperatorGroup
                X, xr, Vt, vr, Y, yr = src.group_io(l, ss, ps)
                capi.read_apply(pool, g, l, X, xr, Vt, vr, Y, yr, None, stream)
                src.on_output(l, ss, ps, Y, yr)                         # ReturnOutputs
            if prof:
                self.read_events.append((e0, self._ev(), tr.n_layers))
            log.census[g.effect] += len(ss)
            if g.effect == READ:
                capi.tttstate_step_done(pool, g)                        # UpdateKVAndTailMetadata
            else:
                self._write(g, ss, ps)
            for s in ss:
                self.pos[s] += 1
                self.pending.discard(s)
        self.clock += 1

    def _write(self, g, ss, ps):
        eng, tr, log, stream = self.eng, self.tr, self.log, self.stream
        pool = eng.pool
        vb = [capi.tttstate_version(pool, o) for o in g.owners]
        mask = [("fail" in tr.controls_at(s, p)) and (s, p) not in self.failed_once for s, p in zip(ss, ps)]
        try:                                                            # CommitVersions
            if self.profile:
                e0 = self._ev()
            capi.write_commit(pool, g, tr.eta, mask if any(mask) else None, stream)
            if self.profile:
                self.write_events.append((e0, self._ev()))
            ok = True
            if self.sync_writes and capi.tttstate_sync(pool, stream):
                log.device_failures += 1
                ok = False
        except TTTError as e:
            if e.status != capi.TTT_E_WRITE_FAILED:
                raise
            ok = False
        if ok:
            for s, p, v in zip(ss, ps, vb):
                log.commits.append((s, p, v, v + 1, "ok"))
            return
        for s, p, v in zip(ss, ps, vb):
            self.failed_once.add((s, p))
            log.commits.append((s, p, v, v, "failed"))
        log.fallbacks += 1
        for s, p, v, o in zip(ss, ps, vb, g.owners):                    # App. H fallback: singletons
            single = Group(WRITE, [o], g.c.shape_id, g.c.placement, g.c.backend, self.clock)
            capi.write_commit(pool, single, tr.eta, None, stream)
            log.commits.append((s, p, v, v + 1, "ok"))

    def finish(self) -> RunLog:
        for s, o in enumerate(self.owners):
            self.log.versions[s] = capi.tttstate_version(self.eng.pool, o)
        for b in self.branches:
            self.log.branches[b] = capi.tttstate_version(self.eng.pool, b)
        return self.log


def run_trace(eng: Engine, tr, src: InputSource, stream=None, sync_writes: bool = True,
              max_clock: int | None = None) -> RunLog:
    """Alg. 1 over a workload.traces.Trace (App. H: fallback + wait budget)."""
    srv = Server(eng, tr, src, stream, sync_writes)
    srv.admit()
    while not srv.done():
        if max_clock is not None and srv.clock >= max_clock:
            break
        srv.step()
    return srv.finish()

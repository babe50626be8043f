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

import torch

from . import capi
from .capi import READ, WRITE, Group, TTTError


class Engine:
    """One TTTState pool (placement π = this device) plus its planner."""

    def __init__(self, d_model: int, d_ff: int, chunk: int, n_layers: int, dtype: str, max_owners: int,
                 w_down: torch.Tensor, n_ckpt: int = 0, mode: int = capi.MODE_FULL, B: int = 8, w: int = 0,
                 shape_id: int = 0, placement: int = 0, device=None, eta: float = 0.01):
        device = torch.device(device) if device is not None else w_down.device
        assert w_down.is_cuda, "w_down must be a device tensor"
        self.d_model, self.d_ff, self.chunk, self.n_layers, self.dtype = d_model, d_ff, chunk, n_layers, dtype
        self.tdtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.eta = float(torch.tensor(eta, dtype=torch.float32))
        self.shape = capi.make_shape(d_model, d_ff, chunk, n_layers, dtype)
        self.arena_bytes = capi.tttstate_pool_bytes(self.shape, max_owners, n_ckpt)
        self._arena = torch.empty(self.arena_bytes + 1024, dtype=torch.uint8, device=device)
        base = (self._arena.data_ptr() + 1023) // 1024 * 1024
        self.w_down = w_down
        self.pool = capi.tttstate_pool_create(self.shape, shape_id, placement, max_owners, n_ckpt, base,
                                              self.arena_bytes, w_down)
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


def run_trace(eng: Engine, tr, src: InputSource, stream=None, sync_writes: bool = True,
              max_clock: int | None = None) -> RunLog:
    """Alg. 1 over a workload.traces.Trace (App. H: fallback + wait budget)."""
    log = RunLog()
    owners = [tr.owner(s) for s in range(tr.n_streams)]
    by_owner = {o: s for s, o in enumerate(owners)}
    for s, o in enumerate(owners):
        capi.tttstate_alloc(eng.pool, o, src.init_delta(s), tr.v0, stream)
        pre = src.tail_prefill(s)
        if pre is not None:
            capi.tttstate_tail_load(eng.pool, o, pre[0], pre[1], pre[2], stream)
    pos = [0] * tr.n_streams
    pending: set = set()
    ready_at: dict = {}
    failed_once: set = set()
    clock = 0
    while any(p < tr.n_steps for p in pos):
        if max_clock is not None and clock >= max_clock:
            break
        events = []
        for s in range(tr.n_streams):                                   # View + NextStep
            if pos[s] < tr.n_steps and s not in pending:
                for op in tr.controls_at(s, pos[s]):
                    if op == "snapshot":
                        capi.tttstate_snapshot(eng.pool, owners[s], stream)
                    elif op == "rollback":
                        vb = capi.tttstate_version(eng.pool, owners[s])
                        va = capi.rollback(eng.pool, owners[s], stream)
                        log.commits.append((s, pos[s], vb, va, "rolled_back"))
                events.append(capi.tttstate_next_event(eng.pool, owners[s], clock))
                pending.add(s)
                ready_at[s] = clock
        groups, rejected = capi.plan_batch(eng.planner, events, clock)  # LegalGroups
        if rejected:
            raise RuntimeError(f"planner rejected events of a well-formed trace: {rejected}")
        for g in groups:
            ss = [by_owner[o] for o in g.owners]
            ps = [pos[s] for s in ss]
            log.plan.append((g.issue_step, g.effect, ss, [ready_at[s] for s in ss]))
            for l in range(tr.n_layers):                                # ExecuteOperatorGroup
                X, xr, Vt, vr, Y, yr = src.group_io(l, ss, ps)
                capi.read_apply(eng.pool, g, l, X, xr, Vt, vr, Y, yr, None, stream)
                src.on_output(l, ss, ps, Y, yr)                         # ReturnOutputs
            log.census[g.effect] += len(ss)
            if g.effect == READ:
                capi.tttstate_step_done(eng.pool, g)                    # UpdateKVAndTailMetadata
            else:
                vb = [capi.tttstate_version(eng.pool, o) for o in g.owners]
                mask = [("fail" in tr.controls_at(s, p)) and (s, p) not in failed_once for s, p in zip(ss, ps)]
                try:                                                    # CommitVersions
                    capi.write_commit(eng.pool, g, tr.eta, mask if any(mask) else None, stream)
                    ok = True
                    if sync_writes and capi.tttstate_sync(eng.pool, stream):
                        log.device_failures += 1
                        ok = False
                except TTTError as e:
                    if e.status != capi.TTT_E_WRITE_FAILED:
                        raise
                    ok = False
                if ok:
                    for s, p, v in zip(ss, ps, vb):
                        log.commits.append((s, p, v, v + 1, "ok"))
                else:
                    for s, p, v in zip(ss, ps, vb):
                        failed_once.add((s, p))
                        log.commits.append((s, p, v, v, "failed"))
                    log.fallbacks += 1
                    for s, p, v, o in zip(ss, ps, vb, g.owners):        # App. H fallback: singletons
                        single = Group(WRITE, [o], g.c.shape_id, g.c.placement, g.c.backend, clock)
                        capi.write_commit(eng.pool, single, tr.eta, None, stream)
                        log.commits.append((s, p, v, v + 1, "ok"))
            for s in ss:
                pos[s] += 1
                pending.discard(s)
        clock += 1
    for s, o in enumerate(owners):
        log.versions[s] = capi.tttstate_version(eng.pool, o)
    return log

"""Oracle drivers: the sequential TTT execution and the oracle's own batched Alg. 1.

TEST INFRASTRUCTURE ONLY (see oracle/numerics.py header).

`run_sequential` is the target behaviour the paper defines: "the original
sequential TTT execution using the same backend and update rule",
one stream at a time, singleton steps.  `run_batched` follows Alg. 1
 with the oracle planner (oracle/planner.py): View -> NextStep ->
LegalGroups -> ExecuteOperatorGroup -> ReturnOutputs -> CommitVersions (WRITE)
-> UpdateKVAndTailMetadata, plus the App. H fallback: a failed WRITE group is
re-run as serial singletons in μ order.
Both consume a `workload.traces.Trace`; per-request arithmetic is identical so
the two must agree bit for bit.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from workload.traces import Trace

from . import numerics as nm
from .planner import Event, OraclePlanner
from .state import READ, WRITE, ContractError, StateTable


@dataclass
class Record:
    outputs: dict = field(default_factory=dict)      # (s, p, l) -> float64 y
    commits: list = field(default_factory=list)      # (s, p, v_before, v_after, outcome)
    census: dict = field(default_factory=lambda: {READ: 0, WRITE: 0})
    plan: list = field(default_factory=list)         # (issue_step, effect, [streams], [ready])
    versions: dict = field(default_factory=dict)     # s -> final V
    state: dict = field(default_factory=dict)        # s -> [per layer ΔW float64]
    events: dict = field(default_factory=dict)       # (s, p) -> effect
    branches: dict = field(default_factory=dict)     # live branch owner -> (v, [payload per layer])


def make_table(tr: Trace, layers=None) -> StateTable:
    layers = range(tr.n_layers) if layers is None else layers
    if tr.rule == 1:
        W = [np.eye(tr.d_model, tr.d_ff) for _ in layers]
    else:
        W = [nm.widen(tr.w_down(l), tr.dtype) for l in layers]
    return StateTable(len(W), tr.d_model, tr.d_ff, tr.chunk, tr.dtype, W, tr.eta, tr.rule,
                      backend=tr.backend, rank=tr.rank)


def init_stream(tab: StateTable, tr: Trace, s: int, layers=None):
    layers = list(range(tr.n_layers)) if layers is None else list(layers)
    d0 = [tr.delta0_of(s, l) for l in layers]
    if d0[0] is None:
        init = None
    elif tr.backend == 1:
        init = [(nm.widen(a, tr.dtype), nm.widen(b, tr.dtype)) for a, b in d0]
    else:
        init = [nm.widen(d, tr.dtype) for d in d0]
    tab.alloc(tr.owner(s), init, tr.v0)
    off = tr.offset(s)
    if off:
        ps = list(range(-off, 0))
        tab.prefill_tail(tr.owner(s),
                         [[nm.widen(tr.x(s, p, l), tr.dtype) for l in layers] for p in ps],
                         [[nm.widen(tr.tgt(s, p, l), tr.dtype) for l in layers] for p in ps], ps)


def _inputs(tr: Trace, s: int, p: int, layers):
    zs = [nm.widen(tr.x(s, p, l), tr.dtype) for l in layers]
    vs = [nm.widen(tr.tgt(s, p, l), tr.dtype) for l in layers]
    return zs, vs


def _control(tab, tr, rec, s, p, forks=None):
    r = tr.owner(s)
    forks = {} if forks is None else forks
    for op in tr.controls_at(s, p):
        if op == "snapshot":
            tab.snapshot(r)
        elif op == "rollback":
            v_before = tab.version(r)
            v_after = tab.rollback(r)
            rec.commits.append((s, p, v_before, v_after, "rolled_back"))
        elif op == "fork":                                  # new owner/version lineage
            k = forks.get(s, 0)
            tab.fork(r, tr.branch_owner(s, k))
            forks[s] = k + 1
        elif op == "release":                               # free the stream's latest branch
            tab.free(tr.branch_owner(s, forks[s] - 1))


def _branches(tab, tr, rec):
    for b, o in tab.owners.items():
        if b >= tr.owner_base + 1_000_000:
            rec.branches[b] = (o.v, [tuple(x.copy() for x in S) if isinstance(S, tuple) else S.copy() for S in o.S])


def run_sequential(tr: Trace, layers=None, keep_outputs: bool = True, streams=None) -> Record:
    """Sequential execution; `streams` restricts it to a subset (streams are independent)."""
    layers = list(range(tr.n_layers)) if layers is None else list(layers)
    tab = make_table(tr, layers)
    rec = Record()
    forks: dict = {}
    for s in (range(tr.n_streams) if streams is None else streams):
        init_stream(tab, tr, s, layers)
        r = tr.owner(s)
        for p in range(tr.n_steps):
            _control(tab, tr, rec, s, p, forks)
            eff = tab.next_effect(r)
            rec.events[(s, p)] = eff
            zs, vs = _inputs(tr, s, p, layers)
            ys = tab.apply(r, p, zs, vs)
            if keep_outputs:
                for i, l in enumerate(layers):
                    rec.outputs[(s, p, l)] = ys[i]
            rec.census[eff] += 1
            if eff == WRITE:
                v = tab.version(r)
                if "fail" in tr.controls_at(s, p):
                    try:
                        tab.write_group([r], fail=True)
                    except ContractError:
                        rec.commits.append((s, p, v, v, "failed"))
                _retry(tab, rec, r, s, p, v)
        rec.versions[s] = tab.version(r)
        rec.state[s] = _state_copy(tab.owners[r].S)
    _branches(tab, tr, rec)
    return rec


def _retry(tab, rec, r, s, p, v):
    """A singleton WRITE (App. H fallback).  A non-finite candidate fails it
    again — the update is deterministic — so that failure is final: v and ΔW stay and the
    chunk's evidence is dropped (reading xx)."""
    try:
        tab.write_group([r])
        rec.commits.append((s, p, v, v + 1, "ok"))
    except ContractError as e:
        if e.code != "WRITE_FAILED":
            raise
        tab.drop_chunk(r)
        rec.commits.append((s, p, v, v, "failed"))


def _state_copy(S):
    return [tuple(a.copy() for a in x) if isinstance(x, tuple) else x.copy() for x in S]


def run_batched(tr: Trace, layers=None, keep_outputs: bool = True) -> Record:
    layers = list(range(tr.n_layers)) if layers is None else list(layers)
    tab = make_table(tr, layers)
    rec = Record()
    for s in range(tr.n_streams):
        init_stream(tab, tr, s, layers)
    by_owner = {tr.owner(s): s for s in range(tr.n_streams)}
    planner = OraclePlanner(tr.B, tr.w, tr.mode)
    pos = [0] * tr.n_streams
    pending = set()
    failed_once = set()
    forks: dict = {}

    def V(r):
        return tab.version(r) if r in tab.owners else None

    clock = 0
    while any(p < tr.n_steps for p in pos):
        events = []
        for s in range(tr.n_streams):                       # View + NextStep
            if pos[s] < tr.n_steps and s not in pending:
                _control(tab, tr, rec, s, pos[s], forks)
                r = tr.owner(s)
                events.append(Event(r, tab.next_effect(r), tr.backend, 0, 0, tab.version(r), clock))
                pending.add(s)
        groups, rejected = planner.plan(events, clock, V)   # LegalGroups
        assert not rejected, rejected
        for g in groups:
            ss = [by_owner[r] for r in g.owners]
            rec.plan.append((g.issue_step, g.effect, ss, list(g.ready_steps)))
            for s in ss:                                    # ExecuteOperatorGroup / ReturnOutputs
                p = pos[s]
                zs, vs = _inputs(tr, s, p, layers)
                ys = tab.apply(tr.owner(s), p, zs, vs)
                if keep_outputs:
                    for i, l in enumerate(layers):
                        rec.outputs[(s, p, l)] = ys[i]
                rec.census[g.effect] += 1
                rec.events[(s, p)] = g.effect
            if g.effect == WRITE:                           # CommitVersions
                vb = {s: tab.version(tr.owner(s)) for s in ss}
                fail = any("fail" in tr.controls_at(s, pos[s]) and (s, pos[s]) not in failed_once
                           for s in ss)
                try:
                    tab.write_group(list(g.owners), fail=fail)
                    for s in ss:
                        rec.commits.append((s, pos[s], vb[s], vb[s] + 1, "ok"))
                except ContractError as e:
                    assert e.code == "WRITE_FAILED"
                    for s in ss:
                        failed_once.add((s, pos[s]))
                        rec.commits.append((s, pos[s], vb[s], vb[s], "failed"))
                    for s in ss:                            # fallback: serial singletons in μ order
                        _retry(tab, rec, tr.owner(s), s, pos[s], vb[s])
            for s in ss:                                    # UpdateKVAndTailMetadata
                pos[s] += 1
                pending.discard(s)
        clock += 1
    for s in range(tr.n_streams):
        rec.versions[s] = tab.version(tr.owner(s))
        rec.state[s] = _state_copy(tab.owners[tr.owner(s)].S)
    _branches(tab, tr, rec)
    return rec


def ok_commits(rec: Record) -> dict:
    """Per stream, the successful commits and rollbacks in order (unique across schedules)."""
    out = {}
    for (s, p, vb, va, oc) in rec.commits:
        if oc != "failed":
            out.setdefault(s, []).append((p, vb, va, oc))
    return out

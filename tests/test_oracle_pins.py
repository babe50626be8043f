"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test pins oracle/ to something other than itself: SPEC/PAPER worked
examples (tests/golden/spec_examples.json, cited), exact rational brute force
on tiny inputs (fractions.Fraction), closed forms (chunking invariance of the
committed state), library routines (torch's bf16 rounding), and invariants
of the serving contract.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import numerics as nm
from oracle.planner import MODE_FULL, MODE_PHASE, MODE_SERIAL, Event, OraclePlanner, validate_group
from oracle.run import ok_commits, run_batched, run_sequential
from oracle.state import READ, WRITE, ContractError, StateTable
from workload import traces as T

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- bf16 storage
def test_round_bf16_matches_torch_library_rounding():
    rs = np.random.default_rng(1)
    x = np.concatenate([rs.standard_normal(20000).astype(np.float32) * 10.0 ** rs.integers(-6, 6, 20000),
                        np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -1.0 - 2 ** -8, 2 ** -130, 3e38],
                                 dtype=np.float32)]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    got = nm.round_bf16(x.astype(np.float64))
    assert np.array_equal(got, ref)


def test_round_bf16_hand_values():
    # 1 + 2^-8 is a tie between 1 and 1 + 2^-7: ties to even -> 1.0
    assert nm.round_bf16(np.array([1.0 + 2 ** -8]))[0] == 1.0
    # 1 + 3*2^-8 ties between 1+2^-7 (odd) and 1+2^-6 (even) -> 1 + 2^-6
    assert nm.round_bf16(np.array([1.0 + 3 * 2 ** -8]))[0] == 1.0 + 2 ** -6
    assert nm.round_bf16(np.array([1.0 + 2 ** -8 + 2 ** -20]))[0] == 1.0 + 2 ** -7


# ---------------------------------------------------------------- READ
def _frac_read(W, S, z):
    dm, dff = len(W), len(W[0])
    return [sum((Fraction(W[i][j]) + Fraction(S[i][j])) * Fraction(z[j]) for j in range(dff))
            for i in range(dm)]


def test_read_exact_rational_brute_force_nonsquare():
    rs = np.random.default_rng(2)
    dm, dff = 3, 5          # non-square: a transposed operand cannot type-check
    W = rs.integers(-8, 8, (dm, dff)) / 16.0
    S = rs.integers(-8, 8, (dm, dff)) / 32.0
    z = rs.integers(-8, 8, dff) / 8.0
    y = nm.apply_read(W, S, z)
    ref = _frac_read(W.tolist(), S.tolist(), z.tolist())
    assert [Fraction(v) for v in y] == ref


def test_read_spec_examples_rule1():
    for k in ("read_identity_zero", "read_identity_I"):
        g = GOLD[k]
        y = nm.apply_read(None, np.array(g["W"], float), np.array(g["x"], float), rule=g["rule"])
        assert y.tolist() == g["y"], g["cite"]


def test_read_base_only_when_delta_zero_and_delta_only_when_base_zero():
    rs = np.random.default_rng(3)
    W = rs.integers(-4, 4, (4, 6)) / 4.0
    z = rs.integers(-4, 4, 6) / 4.0
    zero = np.zeros_like(W)
    assert np.array_equal(nm.apply_read(W, zero, z), nm.apply_read(zero, W, z))
    assert not np.array_equal(nm.apply_read(W, W, z), nm.apply_read(W, zero, z)) or not z.any()


# ---------------------------------------------------------------- WRITE
def test_write_exact_rational_brute_force():
    rs = np.random.default_rng(4)
    dm, dff, C = 3, 4, 5
    S = rs.integers(-8, 8, (dm, dff)) / 16.0
    Z = rs.integers(-4, 4, (C, dff)) / 4.0
    V = rs.integers(-4, 4, (C, dm)) / 4.0
    eta = 2.0 ** -4
    cand = nm.boundary_update(S, Z, V, eta, "fp32")
    for i in range(dm):
        for j in range(dff):
            ref = Fraction(S[i, j]) + Fraction(eta) * sum(Fraction(V[t, i]) * Fraction(Z[t, j]) for t in range(C))
            assert Fraction(cand[i, j]) == ref


def test_write_spec_examples_rule1():
    g = GOLD["update_outer"]
    eta = float(np.float32(g["eta"]))
    # tokens all equal to m give evidence mean m
    Z = np.array([g["m"], g["m"]], float)
    cand = nm.boundary_update(np.array(g["W"], float), Z, None, eta, "fp32", rule=1)
    assert np.all(cand == np.float32(g["W_new_each"])), g["cite"]
    g = GOLD["update_zero"]
    cand = nm.boundary_update(np.array(g["W"], float), np.array([g["m"]], float), None, 0.01, "fp32", rule=1)
    assert np.all(cand == 0.0)
    g = GOLD["mean_evidence"]
    cand = nm.boundary_update(np.zeros((2, 2)), np.array(g["tokens"], float), None, 1.0, "fp32", rule=1)
    assert np.array_equal(cand, np.outer(g["m"], g["m"])), g["cite"]


def test_write_two_boundary_toy_spec_s564():
    # W = η(m1 m1ᵀ + m2 m2ᵀ) after two boundaries from W = 0
    eta = 2.0 ** -3
    Z1 = np.array([[1.0, 0.5], [0.0, 0.5]])
    Z2 = np.array([[-1.0, 1.0], [0.5, 0.0]])
    W1 = nm.boundary_update(np.zeros((2, 2)), Z1, None, eta, "fp32", rule=1)
    W2 = nm.boundary_update(W1, Z2, None, eta, "fp32", rule=1)
    m1, m2 = Z1.mean(0), Z2.mean(0)
    assert np.array_equal(W2, eta * (np.outer(m1, m1) + np.outer(m2, m2)))


def test_write_bf16_storage_is_library_rounding_of_exact_candidate():
    rs = np.random.default_rng(5)
    S = nm.round_bf16(rs.standard_normal((4, 6)) * 0.01)
    Z = rs.integers(-4, 4, (8, 6)) / 4.0
    V = rs.integers(-4, 4, (8, 4)) / 4.0
    eta = float(np.float32(0.01))
    exact = S + eta * (V.T @ Z)                     # exact in fp64 at these sizes? check via fp32 path
    ref = torch.from_numpy(exact.astype(np.float32)).to(torch.bfloat16).double().numpy()
    got = nm.boundary_update(S, Z, V, eta, "bf16")
    # reading xi: the storage RNE rounds the fp32 accumulator value -> exactly torch's
    # fp64 -> fp32 -> bf16 conversion (library routines)
    assert np.array_equal(got, ref) and nm.normwise_rel_err(got, exact) < 2 ** -8


def test_committed_state_closed_form_chunking_invariance():
    """S_k = S_0 + η Σ_{committed t} v_t z_tᵀ, independent of chunking (SURVEY §8(c) pins).

    fp32 storage with dyadic inputs keeps every partial sum exact, so the
    chunked state must equal one unchunked sum bit for bit.
    """
    for C in (1, 2, 4, 8):
        tr = T.uniform_small(n_streams=2, n_layers=2, d_model=3, d_ff=5, chunk=C, n_steps=16, dtype="fp32")
        tr = tr.replace(eta=2.0 ** -4)
        # dyadic inputs: override generator with small integers / 4
        rs = np.random.default_rng(6)
        X = rs.integers(-4, 5, (2, 16, 2, 5)) / 4.0
        Vt = rs.integers(-4, 5, (2, 16, 2, 3)) / 4.0
        tab = StateTable(2, 3, 5, C, "fp32", [np.zeros((3, 5))] * 2, tr.eta)
        for s in range(2):
            tab.alloc(s)
            for p in range(16):
                eff = tab.next_effect(s)
                tab.apply(s, p, list(X[s, p]), list(Vt[s, p]))
                if eff == WRITE:
                    tab.write_group([s])
            for l in range(2):
                closed = tr.eta * Vt[s, :, l, :].T @ X[s, :, l, :]
                assert np.array_equal(tab.owners[s].S[l], closed)
            assert tab.version(s) == 16 // C


# ---------------------------------------------------------------- state contract
def _tiny_table(C=2, dtype="fp32"):
    return StateTable(1, 2, 3, C, dtype, [np.zeros((2, 3))], 0.5)


def test_state_contract_spec_examples():
    tab = _tiny_table()
    assert tab.alloc(1) == 0
    with pytest.raises(ContractError):
        tab.alloc(1)
    for r in range(2, 9):
        tab.alloc(r)
    assert all(tab.version(r) == 0 for r in range(1, 9))
    z, v = [np.array([1.0, 0, 1])], [np.array([1.0, -1])]
    assert tab.next_effect(1) == READ
    tab.apply(1, 0, z, v)
    assert tab.version(1) == 0                                  # S:72 READ preserves version
    assert tab.next_effect(1) == WRITE
    S_before = tab.owners[1].S[0].copy()
    tab.apply(1, 1, z, v)
    with pytest.raises(ContractError):
        tab.write_group([1], fail=True)                         # failed write: nothing changes
    assert tab.version(1) == 0 and np.array_equal(tab.owners[1].S[0], S_before) and tab.tail_len(1) == 2
    assert tab.write_group([1]) == [1]
    assert tab.tail_len(1) == 0
    tab.snapshot(1)
    snap = tab.owners[1].S[0].copy()
    tab.apply(1, 2, z, v)
    tab.apply(1, 3, z, v)
    tab.write_group([1])
    assert tab.version(1) == 2                                  # S:90 / S:99
    assert tab.rollback(1) == 1
    assert np.array_equal(tab.owners[1].S[0], snap) and tab.tail_len(1) == 0
    assert tab.rollback(1) == 1                                 # checkpoint retained
    with pytest.raises(ContractError):
        tab.rollback(2)
    tab.fork(1, 99)
    assert tab.version(99) == 1
    tab.apply(99, 0, z, v)
    tab.apply(99, 1, z, v)
    tab.write_group([99])
    assert tab.version(99) == 2 and tab.version(1) == 1 and np.array_equal(tab.owners[1].S[0], snap)


def test_rollback_mid_chunk_and_fork_contents():
    """Reading vii (rollback clears the tail: the rolled-back chunk's evidence is discarded) and
    reading viii (a fork carries the committed state at the same version, empty tail; S:113,
    S:145): checked by the values they imply, with dyadic inputs so every sum is exact."""
    eta = 0.5
    tab = StateTable(1, 2, 3, 2, "fp32", [np.zeros((2, 3))], eta)      # C = 2
    init = [np.array([[1.0, 0.0, -1.0], [0.5, 2.0, 0.0]])]
    tab.alloc(1, init=init, v0=3)
    tab.snapshot(1)
    z1, v1 = np.array([1.0, 2.0, 0.0]), np.array([1.0, -1.0])
    tab.apply(1, 0, [z1], [v1])                                          # half a chunk of evidence
    assert tab.tail_len(1) == 1
    assert tab.rollback(1) == 3 and tab.tail_len(1) == 0                 # reading vii: evidence dropped
    assert tab.next_effect(1) == READ                                    # a full new chunk is needed
    z2, v2 = np.array([0.0, 1.0, 1.0]), np.array([2.0, 0.0])
    z3, v3 = np.array([1.0, 0.0, 0.5]), np.array([0.0, 1.0])
    tab.apply(1, 1, [z2], [v2])
    assert tab.next_effect(1) == WRITE
    tab.apply(1, 2, [z3], [v3])
    assert tab.write_group([1]) == [4]
    expect = init[0] + eta * (np.outer(v2, z2) + np.outer(v3, z3))   # z1's evidence absent
    assert np.array_equal(tab.owners[1].S[0], expect)
    # fork: same committed bytes and version, empty tail; its READ equals the source's
    assert tab.fork(1, 7) == 4 and tab.version(7) == 4 and tab.tail_len(7) == 0
    assert np.array_equal(tab.owners[7].S[0], expect)
    y_src = tab.apply(1, 3, [z1], [v1])[0]
    y_fork = tab.apply(7, 0, [z1], [v1])[0]
    assert np.array_equal(y_src, y_fork) and np.array_equal(y_fork, expect @ z1)
    tab.apply(7, 1, [z2], [v2])
    assert tab.write_group([7]) == [5]
    assert np.array_equal(tab.owners[7].S[0], expect + eta * (np.outer(v1, z1) + np.outer(v2, z2)))
    assert np.array_equal(tab.owners[1].S[0], expect) and tab.version(1) == 4   # isolation


def test_group_write_is_atomic_and_owner_local():
    tab = _tiny_table()
    for r in (1, 2, 3):
        tab.alloc(r)
        for p in range(2):
            tab.apply(r, p, [np.array([1.0, 2, 3])], [np.array([r * 1.0, 1])])
    before = {r: tab.owners[r].S[0].copy() for r in (1, 2, 3)}
    with pytest.raises(ContractError):
        tab.write_group([1, 2], fail=True)
    assert [tab.version(r) for r in (1, 2, 3)] == [0, 0, 0]
    tab.write_group([1, 2])
    assert [tab.version(r) for r in (1, 2, 3)] == [1, 1, 0]
    assert np.array_equal(tab.owners[3].S[0], before[3])        # commit exclusivity
    assert not np.array_equal(tab.owners[1].S[0], tab.owners[2].S[0])   # no aliasing
    with pytest.raises(ContractError):
        tab.write_group([3, 3])                                 # μ injective


# ---------------------------------------------------------------- census and versions
def test_census_uniform_trace_paper_p573():
    g = GOLD["census_uniform"]
    tr = T.uniform_small(n_streams=g["streams"], n_layers=1, d_model=2, d_ff=2, chunk=g["chunk"],
                         n_steps=g["decode"], dtype="fp32")
    rec = run_batched(tr, keep_outputs=False)
    assert rec.census[READ] == g["reads"] and rec.census[WRITE] == g["writes"], g["cite"]
    assert set(rec.versions.values()) == {GOLD["versions_uniform"]["final_version"]}


def test_versions_all_update_trace():
    g = GOLD["versions_all_update"]
    tr = T.uniform_small(n_streams=g["streams"], n_layers=1, d_model=2, d_ff=2, chunk=g["chunk"],
                         n_steps=g["decode"], dtype="fp32")
    rec = run_batched(tr, keep_outputs=False)
    assert rec.census[WRITE] == g["writes"] and set(rec.versions.values()) == {g["final_version"]}


def test_config1_final_versions_and_log():
    tr = T.config1_tiny()
    rec = run_batched(tr)
    assert [rec.versions[0], rec.versions[1]] == GOLD["config1_final_versions"]["versions"]
    fails = [c for c in rec.commits if c[4] == "failed"]
    assert {(c[0], c[1]) for c in fails} == {(0, 11), (1, 11)}        # group-atomic failure
    assert all(c[2] == c[3] for c in fails)                            # v intact on failure
    rb = [c for c in rec.commits if c[4] == "rolled_back"]
    assert rb == [(1, 8, 2, 1, "rolled_back")]


# ---------------------------------------------------------------- sequential == batched
@pytest.mark.parametrize("mode", [MODE_SERIAL, MODE_PHASE, MODE_FULL])
@pytest.mark.parametrize("w", [0, 2, 5])
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_sequential_equals_batched_bit_exact(mode, w, dtype):
    tr = T.uniform_small(n_streams=5, n_layers=2, d_model=8, d_ff=12, chunk=4, n_steps=13, dtype=dtype,
                         w=w, mode=mode, offsets=(0, 1, 3, 2, 0), delta0="rng", v0=7,
                         controls={(1, 2): ["snapshot"], (1, 5): ["rollback"], (2, 0): ["fail"],
                                   (4, 3): ["fail"], (3, 9): ["snapshot", "rollback"]})
    tr = tr.replace(B=3)
    a, b = run_sequential(tr), run_batched(tr)
    assert a.outputs.keys() == b.outputs.keys()
    for k in a.outputs:
        assert np.array_equal(a.outputs[k], b.outputs[k]), k
    assert a.versions == b.versions
    for s in a.state:
        for l in range(tr.n_layers):
            assert np.array_equal(a.state[s][l], b.state[s][l])
    assert ok_commits(a) == ok_commits(b)
    assert a.census == b.census
    # Eq. 4 bounded waiting, phase separation, injective μ on every issued group
    for (issue, eff, ss, ready) in b.plan:
        assert len(set(ss)) == len(ss)
        assert all(0 <= issue - r <= tr.w for r in ready)
        if mode == MODE_SERIAL:
            assert len(ss) == 1
        if mode == MODE_PHASE and eff == WRITE:
            assert len(ss) == 1
        assert len(ss) <= tr.B


# ---------------------------------------------------------------- planner
def _ev(r, eff=READ, v=0, ready=0, shape=0):
    return Event(r, eff, 0, shape, 0, v, ready)


def test_planner_spec_examples():
    V = lambda r: 0
    p = OraclePlanner(8, 0)
    g, rej = p.plan([_ev(r) for r in range(8)], 0, V)
    assert [len(x.owners) for x in g] == GOLD["planner_8_reads"]["groups"] and not rej
    p = OraclePlanner(8, 0)
    g, _ = p.plan([_ev(r) for r in range(6)] + [_ev(r, WRITE) for r in range(6, 8)], 0, V)
    assert sorted(len(x.owners) for x in g) == sorted(GOLD["planner_6r_2w"]["groups"])
    assert all(len({x for x in grp.owners}) == len(grp.owners) for grp in g)
    assert {grp.effect for grp in g} == {READ, WRITE}
    gw = GOLD["planner_wait"]
    p = OraclePlanner(gw["B"], gw["w"])
    issued = None
    evs = [_ev(r, ready=gw["ready"]) for r in range(gw["n"])]
    for clock in range(gw["ready"], gw["ready"] + 10):
        g, _ = p.plan(evs if clock == gw["ready"] else [], clock, V)
        if g:
            issued = g[0].issue_step
            break
    assert issued == gw["issue"]


def test_planner_rejects_stale_and_collisions_and_allows_mixed_versions():
    V = {1: 3, 2: 1, 3: 5}.get
    p = OraclePlanner(8, 0)
    g, rej = p.plan([_ev(1, v=2), _ev(2, v=1), _ev(3, v=5), _ev(3, v=5)], 0, V)
    assert [e.owner for e in rej] == [1, 3]          # stale and duplicate owner
    assert g[0].owners == [2, 3]                     # different numeric versions co-issue
    assert validate_group(g[0], V, [1, 5]) is None
    assert validate_group(g[0], V, [1, 4]) == "VERSION_MISMATCH"


def test_planner_rejects_waiting_event_after_commit_behind_its_back():
    """S:301 (a version mismatch is rejected to revalidation, never silently issued) and S:314
    ("commit behind the event's back, then validate"): an event that matched V(r) on arrival and
    is still waiting in its bucket is rejected once a commit moves V(r); the others still issue
    when the wait budget runs out (Eq. 4)."""
    V = {1: 0, 2: 0}
    p = OraclePlanner(8, 4)                               # B = 8, w = 4: two events wait
    g, rej = p.plan([_ev(1, v=0, ready=0), _ev(2, v=0, ready=0)], 0, V.get)
    assert not g and not rej
    V[1] = 1                                              # owner 1 commits behind its event's back
    g, rej = p.plan([], 1, V.get)
    assert [e.owner for e in rej] == [1] and not g
    issued = []
    for clock in range(2, 8):
        g, rej = p.plan([], clock, V.get)
        assert not rej
        issued += [(grp.owners, grp.issue_step) for grp in g]
    assert issued == [([2], 4)]


def test_planner_property_eq3_eq4_random():
    """≥1000 random event sets: homogeneous κ, injective μ, version match, bounded wait."""
    rs = np.random.default_rng(7)
    for trial in range(1000):
        B, w = int(rs.integers(1, 6)), int(rs.integers(0, 4))
        p = OraclePlanner(B, w, int(rs.integers(0, 3)))
        Vt = {r: int(rs.integers(0, 3)) for r in range(12)}
        waiting = {}
        for clock in range(8):
            evs = []
            for r in range(12):
                if r not in waiting and rs.random() < 0.5:
                    v = Vt[r] if rs.random() < 0.9 else Vt[r] + 1
                    evs.append(Event(r, int(rs.integers(0, 2)), 0, int(rs.integers(0, 2)), 0, v, clock))
            groups, rej = p.plan(evs, clock, Vt.get)
            for e in evs:
                if e not in rej:
                    waiting[e.owner] = e
            for g in groups:
                assert len(set(g.owners)) == len(g.owners) and 1 <= len(g.owners) <= B
                for r in g.owners:
                    e = waiting.pop(r)
                    assert (e.effect, e.shape_id) == (g.effect, g.shape_id)
                    assert e.version == Vt[r]
                    assert 0 <= clock - e.ready_step <= w
            for e in rej:
                assert e.version != Vt[e.owner] or e.owner in waiting
        # drain: every waiting event issues within w more steps
        for clock in range(8, 8 + w + 1):
            for g in p.plan([], clock, Vt.get)[0]:
                for r in g.owners:
                    waiting.pop(r)
        assert not waiting


def test_storage_rounding_goes_through_fp32():
    """Reading xi (SURVEY §8(c) xi): bf16 storage is one RNE of the fp32 accumulator
    value, so a candidate just above a bf16 tie whose excess is below fp32 resolution rounds as
    the tie does (to even).  Pinned to torch's fp64 -> fp32 -> bf16 conversions (library RNE)."""
    x = np.array([1 + 2**-8 + 2**-30, -(1 + 3 * 2**-8 + 2**-30), 1 + 2**-8 + 2**-20, 3 * 2**-130 + 2**-160])
    ref = torch.tensor(x, dtype=torch.float64).to(torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    got = nm.to_storage(x, "bf16")
    assert np.array_equal(got, ref), (got, ref)
    assert got[0] == 1.0                                  # a direct fp64 -> bf16 RNE gives 1 + 2**-7
    assert got[2] == 1 + 2**-7


def test_normwise_metric():
    assert nm.normwise_rel_err(np.array([1.0, 2.0]), np.array([1.0, 2.0])) == 0.0
    assert nm.normwise_rel_err(np.array([1.0, 2.1]), np.array([1.0, 2.0])) == pytest.approx(0.05)


# ---------------------------------------------------------------- low-rank delta (NEXT f1)
from oracle import lowrank as lr  # noqa: E402


def test_lowrank_spec_examples_square_identity_base():
    # y = x + Bᵀ(A x) with the identity base; A = 0 -> y = x for any B
    rs = np.random.default_rng(30)
    d, R = 4, 2
    x = rs.integers(-4, 4, d) / 4.0
    B = rs.integers(-4, 4, (R, d)) / 4.0
    assert np.array_equal(lr.apply_read(np.eye(d), np.zeros((R, d)), B, x), x)
    A = rs.integers(-4, 4, (R, d)) / 4.0
    assert np.array_equal(lr.apply_read(np.eye(d), A, B, x), x + B.T @ (A @ x))


def test_lowrank_exact_rational_brute_force_nonsquare():
    rs = np.random.default_rng(31)
    dm, dff, R, C = 3, 5, 2, 4
    W = rs.integers(-4, 4, (dm, dff)) / 8.0
    A = rs.integers(-4, 4, (R, dff)) / 8.0
    B = rs.integers(-4, 4, (R, dm)) / 8.0
    z = rs.integers(-4, 4, dff) / 4.0
    y = lr.apply_read(W, A, B, z)
    for i in range(dm):
        ref = sum(Fraction(W[i, j]) * Fraction(z[j]) for j in range(dff))
        ref += sum(Fraction(B[k, i]) * sum(Fraction(A[k, j]) * Fraction(z[j]) for j in range(dff)) for k in range(R))
        assert Fraction(y[i]) == ref
    Z = rs.integers(-4, 4, (C, dff)) / 4.0
    eta = 2.0 ** -3
    A2, B2 = lr.boundary_update(A, B, Z, eta, "fp32")
    m = [sum(Fraction(Z[t, j]) for t in range(C)) / C for j in range(dff)]
    for k in range(R):
        am = sum(Fraction(A[k, j]) * m[j] for j in range(dff))
        for j in range(dff):
            assert Fraction(A2[k, j]) == Fraction(A[k, j]) + Fraction(eta) * am * m[j]
    assert np.array_equal(B2, B)                                # B' = B


def test_lowrank_spec_update_example_s219_generalised():
    # A = I (2x2), m = (1,1), η = 0.01: A' = I + η·(A m) mᵀ = I + 0.01·ones (fp32 storage)
    eta = float(np.float32(0.01))
    A2, _ = lr.boundary_update(np.eye(2), np.zeros((2, 2)), np.array([[1.0, 1.0], [1.0, 1.0]]), eta, "fp32")
    assert np.array_equal(A2, (np.eye(2) + eta * np.ones((2, 2))).astype(np.float32).astype(np.float64))


def test_config4_branches_sequential_equals_batched():
    tr = T.config4_lowrank(n_steps=20, n_layers=2, rank=4, d_model=12, d_ff=16, chunk=4, n_streams=6, seed=3)
    a, b = run_sequential(tr), run_batched(tr)
    assert a.versions == b.versions and ok_commits(a) == ok_commits(b)
    for k in a.outputs:
        assert np.array_equal(a.outputs[k], b.outputs[k])
    assert set(a.branches) == set(b.branches) and len(a.branches) == tr.n_streams   # one live branch each
    for br, (v, S) in a.branches.items():
        assert b.branches[br][0] == v
        for l in range(tr.n_layers):
            assert all(np.array_equal(x, y) for x, y in zip(S[l], b.branches[br][1][l]))
    assert any(c[4] == "rolled_back" for c in a.commits)


# ---------------------------------------------------------------- exact widening
def test_widen_bf16_exhaustive_against_torch():
    """Every one of the 65,536 bf16 bit patterns widens exactly as torch's
    bfloat16 -> float32 -> float64 conversion does (library routine, not a retyped
    shift).  NaN patterns must stay NaN; everything else must be bit-identical."""
    bits = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    got = nm.widen(bits, "bf16")
    ref = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).to(torch.float64).numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint64), ref[~nan].view(np.uint64))   # ±0 kept apart
    # hand values: 0x3F80 = 1.0, 0xC000 = -2.0, 0x0001 = smallest subnormal 2^-133
    assert nm.widen(np.array([0x3F80, 0xC000, 0x0001], dtype=np.uint16), "bf16").tolist() == \
        [1.0, -2.0, 2.0 ** -133]


def test_widen_fp32_is_exact():
    rs = np.random.default_rng(11)
    u = rs.integers(0, 1 << 32, 200_000, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    got = nm.widen(x, "fp32")
    ref = torch.from_numpy(x.copy()).to(torch.float64).numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint64), ref[~nan].view(np.uint64))


# ---------------------------------------------------------------- pre-filled tails (reading xv)
def test_prefill_tail_hand_worked_bursty_example():
    """A stream that starts with 2 of C = 3 evidence entries already in its tail
    (bursty start, reading xv; "the tail holds the chunk's evidence").

    Worked by hand (d_model = 1, d_ff = 2, W_down = [1, 1], η = 1/2, ΔW_0 = 0):
      pre-filled  p = -2: z = (1, 0), v = 2;   p = -1: z = (0, 1), v = 1
      decode      p =  0: z = (1, 1), v = -1  -> tail holds C-1 = 2 before it: WRITE
                  y_0 = (W + ΔW_0) z = 2  (pre-update version, reading xvii)
                  ΔW_1 = η (2·(1,0) + 1·(0,1) − 1·(1,1)) = (1/2, 0),  v: 0 -> 1
      decode      p =  1: z = (2, 0), v = 1   -> READ,  y_1 = (1.5, 1)·(2, 0) = 3
                  p =  2: z = (0, 2), v = 1   -> READ,  y_2 = 2
                  p =  3: z = (1, 0), v = 1   -> WRITE, y_3 = 1.5 (pre-update), then
                  ΔW_2 = ΔW_1 + η (1·(2,0) + 1·(0,2) + 1·(1,0)) = (2, 1)
    """
    tab = StateTable(1, 1, 2, 3, "fp32", [np.array([[1.0, 1.0]])], 0.5)
    tab.alloc(7)
    tab.prefill_tail(7, [[np.array([1.0, 0.0])], [np.array([0.0, 1.0])]],
                     [[np.array([2.0])], [np.array([1.0])]], [-2, -1])
    assert tab.tail_len(7) == 2
    steps = [((1.0, 1.0), -1.0), ((2.0, 0.0), 1.0), ((0.0, 2.0), 1.0), ((1.0, 0.0), 1.0)]
    effects, ys = [], []
    for p, (z, v) in enumerate(steps):
        eff = tab.next_effect(7)
        effects.append(eff)
        ys.append(float(tab.apply(7, p, [np.array(z)], [np.array([v])])[0][0]))
        if eff == WRITE:
            tab.write_group([7])
            if p == 0:
                assert tab.owners[7].S[0].tolist() == [[0.5, 0.0]] and tab.version(7) == 1
    assert effects == [WRITE, READ, READ, WRITE]
    assert ys == [2.0, 3.0, 2.0, 1.5]     # p=2: (1.5,1)·(0,2) = 2; p=3: (1.5,1)·(1,0) = 1.5
    assert tab.owners[7].S[0].tolist() == [[2.0, 1.0]] and tab.version(7) == 2


def test_prefill_tail_bursty_trace_first_write_and_closed_form():
    """Through the trace driver (init_stream -> prefill_tail) on a bursty trace:
    stream s's first WRITE is at p = C-1-offset_s, every later one C steps apart,
    and the committed ΔW equals the closed form over pre-filled + decoded evidence
    η·Σ_{p=-off..last committed} v_p z_pᵀ (P:299-308 target = sequential execution)."""
    C = 4
    offs = (0, 1, 2, 3)
    tr = T.uniform_small(n_streams=4, n_layers=1, d_model=3, d_ff=5, chunk=C, n_steps=11, dtype="fp32")
    tr = tr.replace(offsets=offs, eta=2.0 ** -3)
    rec = run_sequential(tr)
    for s, off in enumerate(offs):
        writes = [p for p in range(tr.n_steps) if rec.events[(s, p)] == WRITE]
        assert writes == list(range(C - 1 - off, tr.n_steps, C))
        last = writes[-1]
        Z = np.stack([nm.widen(tr.x(s, p, 0), "fp32") for p in range(-off, last + 1)])
        Vt = np.stack([nm.widen(tr.tgt(s, p, 0), "fp32") for p in range(-off, last + 1)])
        closed = tr.eta * (Vt.T @ Z)
        assert rec.versions[s] == len(writes)
        # fp32 storage rounds once per commit: agreement to fp32 precision, while a
        # dropped or duplicated evidence entry moves the state by ~η·|v||z| ≫ 1e-6.
        assert nm.normwise_rel_err(rec.state[s][0], closed) < 1e-6


# ---------------------------------------------------------------- device-detected failure (reading xx)
def test_nonfinite_candidate_fails_group_then_singletons_resolve():
    """A non-finite candidate fails its WRITE group (nothing commits: S:368); App. H's
    singleton retries publish the clean members, while the poisoned member fails
    again (the update is deterministic) and its failure is final: v and ΔW stay, the chunk's
    evidence is dropped (reading xx), and it goes on decoding from v."""
    C = 2
    tr = T.uniform_small(n_streams=3, n_layers=1, d_model=3, d_ff=4, chunk=C, n_steps=6, dtype="fp32",
                         controls={(1, 1): ["poison"]})
    rec = run_batched(tr)
    # step p = 1 is every stream's first WRITE; stream 1's target at p = 1 carries +inf
    assert rec.commits[:6] == [(0, 1, 0, 0, "failed"), (1, 1, 0, 0, "failed"), (2, 1, 0, 0, "failed"),
                               (0, 1, 0, 1, "ok"), (1, 1, 0, 0, "failed"), (2, 1, 0, 1, "ok")]
    assert rec.versions == {0: 3, 1: 2, 2: 3}
    assert all(np.all(np.isfinite(rec.state[s][0])) for s in range(3))
    # stream 1 = a clean stream whose first chunk never happened: its later commits use only
    # evidence of p = 2..5 (closed form from ΔW_0 = 0)
    Z = np.stack([nm.widen(tr.x(1, p, 0), "fp32") for p in range(2, 6)])
    Vt = np.stack([nm.widen(tr.tgt(1, p, 0), "fp32") for p in range(2, 6)])
    assert nm.normwise_rel_err(rec.state[1][0], tr.eta * (Vt.T @ Z)) < 1e-6
    seq = run_sequential(tr)
    assert ok_commits(seq) == ok_commits(rec) and seq.versions == rec.versions
    for s in range(3):
        assert np.array_equal(seq.state[s][0], rec.state[s][0])


def test_drop_chunk_keeps_version_and_payload():
    tab = _tiny_table(C=2)
    tab.alloc(5)
    tab.apply(5, 0, [np.ones(3)], [np.ones(2)])
    S0 = tab.owners[5].S[0].copy()
    tab.drop_chunk(5)
    assert tab.tail_len(5) == 0 and tab.version(5) == 0 and np.array_equal(tab.owners[5].S[0], S0)

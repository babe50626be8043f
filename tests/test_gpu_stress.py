"""T4 state-contract stress suite (Table 6 "State-contract stress: 5 injected
failures, 5/5 pass"; scenario names from SPEC S:349, S:372, S:386-390,
S:574-581), through the C ABI on the GPU.

Each scenario injects one failure into the uniform trace, checks the contract at the moment
of injection (rejection before any side effect, or an all-or-nothing group), then finishes
the run and must recover to full oracle equivalence: owner ids, versions and the commit /
rollback log bit-exact, READ outputs and fast weights within the bf16 tolerance.

  MidGroupWriteFail   fail bit on slot 3 of the first WRITE group: no member advances, every
                      member's committed bytes equal the pre-group bytes; App. H singleton retry
  VersionMismatch     a WRITE event forged with expected_version v+1: plan_batch rejects it,
                      validate_group reports TTT_E_VERSION_MISMATCH; nothing launched
  OwnerMapCollision   duplicate owner in one planner call and in a hand-built group: the
                      duplicate is rejected / read_apply fails with TTT_E_OWNER_COLLISION
                      before any launch
  StaleReadAttempt    a READ event forged with expected_version v-1: rejected; no state read
                      (no kernel launched, tail and bytes unchanged)
  RollbackRetry       snapshot + injected group failure at a boundary, singleton retry, then
                      rollback to the snapshot; the run continues to oracle equivalence

Negative control: with the group-atomic commit disabled by the library's test hook
(TTT_HOOK_NO_GROUP_ATOMICITY), MidGroupWriteFail must FAIL.
"""
import pytest
import torch

from oracle import numerics as nm
from oracle.run import run_batched
from workload import traces as T

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200 import serving  # noqa: E402

from .gpu_helpers import HostGenInputs, make_engine  # noqa: E402

DEV = "cuda"
SCENARIOS = ["MidGroupWriteFail", "VersionMismatch", "OwnerMapCollision", "StaleReadAttempt", "RollbackRetry"]
E_VERSION_MISMATCH, E_OWNER_COLLISION = 3, 4


def _trace(scn):
    # 8 streams, boundaries at p = 3, 7, 11 (C = 4), 2 layers, random ΔW_0
    tr = T.uniform_small(n_streams=8, n_layers=2, d_model=128, d_ff=256, chunk=4, n_steps=12, dtype="bf16",
                         delta0="rng", seed=21)
    ctl = {"MidGroupWriteFail": {(3, 3): ["fail"]},
           "RollbackRetry": {(2, 3): ["snapshot", "fail"], (2, 4): ["rollback"]}}.get(scn, {})
    return tr.replace(controls=ctl)


def _state(pool, tr, owners):
    """(host version, device version, tail length, layer-0 committed bytes) per owner."""
    return [(capi.tttstate_version(pool, o), capi.tttstate_device_version(pool, o), capi.tttstate_tail_len(pool, o),
             capi.tttstate_read_payload(pool, o, 0, tr.d_model, tr.d_ff, tr.dtype).tobytes()) for o in owners]


def _equivalent(tr, ref, src, log, eng):
    tol = nm.TOL[tr.dtype]
    if set(ref.outputs) != set(src.out):
        return "output keys differ"
    if (log.versions, log.commits, log.census, log.plan) != (ref.versions, ref.commits, ref.census, ref.plan):
        return f"integer log differs: versions {log.versions} vs {ref.versions}"
    worst = max(nm.normwise_rel_err(src.out[k], ref.outputs[k]) for k in ref.outputs)
    if worst > tol:
        return f"READ outputs normwise err {worst}"
    for s in range(tr.n_streams):
        for l in range(tr.n_layers):
            got = capi.tttstate_read_payload(eng.pool, tr.owner(s), l, tr.d_model, tr.d_ff, tr.dtype)
            err = nm.normwise_rel_err(nm.widen(got, tr.dtype), ref.state[s][l])
            if err > tol:
                return f"fast weights of stream {s} layer {l}: normwise err {err}"
    return None


def _inject(scn, srv, tr):
    """Forged-input scenarios, injected before decode step `clock`; returns the recovery path."""
    eng = srv.eng
    pool, clock = eng.pool, srv.clock
    owners = [tr.owner(s) for s in range(tr.n_streams)]
    before, launches = _state(pool, tr, owners), capi.tttstate_launch_count()
    o = owners[5]
    e = capi.tttstate_next_event(pool, o, clock)
    v = e.expected_version
    if scn == "VersionMismatch":
        assert e.effect == capi.WRITE
        e.expected_version = v + 1
        groups, rej = capi.plan_batch(eng.planner, [e], clock)
        assert not groups and [(r.owner, r.expected_version) for r in rej] == [(o, v + 1)]
        with pytest.raises(capi.TTTError) as ex:
            capi.validate_group(pool, capi.Group(capi.WRITE, [o]), [v + 1])
        assert ex.value.status == E_VERSION_MISMATCH
        path = "rejected to revalidation; re-extracted next step"
    elif scn == "StaleReadAttempt":
        assert e.effect == capi.READ and v >= 1
        e.expected_version = v - 1
        groups, rej = capi.plan_batch(eng.planner, [e], clock)
        assert not groups and [(r.owner, r.expected_version) for r in rej] == [(o, v - 1)]
        with pytest.raises(capi.TTTError) as ex:
            capi.validate_group(pool, capi.Group(capi.READ, [o]), [v - 1])
        assert ex.value.status == E_VERSION_MISMATCH
        path = "rejected by the version check; no state read"
    elif scn == "OwnerMapCollision":
        groups, rej = capi.plan_batch(eng.planner, [e, e], clock)   # planner state is empty again (w = 0)
        assert [list(g.owners) for g in groups] == [[o]] and [r.owner for r in rej] == [o]
        X = torch.zeros(2, tr.d_ff, dtype=torch.bfloat16, device=DEV)
        Vt = torch.zeros(2, tr.d_model, dtype=torch.bfloat16, device=DEV)
        Y = torch.zeros(2, tr.d_model, dtype=torch.bfloat16, device=DEV)
        with pytest.raises(capi.TTTError) as ex:
            capi.read_apply(pool, capi.Group(e.effect, [o, o]), 0, X, None, Vt, None, Y)
        assert ex.value.status == E_OWNER_COLLISION
        path = "duplicate rejected pre-execution"
    else:
        raise AssertionError(scn)
    torch.cuda.synchronize()
    assert capi.tttstate_launch_count() == launches, "a rejected input launched a kernel"
    assert _state(pool, tr, owners) == before, "a rejected input changed owner state"
    return path


def _run_scenario(scn):
    tr = _trace(scn)
    ref = run_batched(tr)
    eng = make_engine(tr, DEV, n_ckpt=2)
    src = HostGenInputs(tr, DEV)
    owners = [tr.owner(s) for s in range(tr.n_streams)]
    seen = {}
    orig = capi.write_commit

    def checked_write_commit(pool, g, eta, fail_mask=None, stream=None):
        if not (fail_mask and any(fail_mask)):
            return orig(pool, g, eta, fail_mask, stream)
        pre = _state(pool, tr, g.owners)
        try:
            return orig(pool, g, eta, fail_mask, stream)
        except capi.TTTError as ex:
            torch.cuda.synchronize()
            post = _state(pool, tr, g.owners)
            # all-or-nothing: nobody advanced, committed bytes equal the pre-group bytes
            seen["atomic"] = all(a[0] == b[0] and a[1] == b[1] and a[3] == b[3] for a, b in zip(pre, post))
            raise ex

    inject_at = {"VersionMismatch": 3, "StaleReadAttempt": 5, "OwnerMapCollision": 2}.get(scn)
    serving.capi.write_commit = checked_write_commit
    try:
        srv = serving.Server(eng, tr, src, None, native=False)   # per-operator calls: state checked between them
        srv.admit()
        path = None
        while not srv.done():
            if srv.clock == inject_at:
                path = _inject(scn, srv, tr)
            srv.step()
        log = srv.finish()
    finally:
        serving.capi.write_commit = orig
    torch.cuda.synchronize()
    if scn in ("MidGroupWriteFail", "RollbackRetry"):
        if not seen.get("atomic"):
            return False, "failed group was not all-or-nothing"
        path = "group not committed; App. H singleton retry" + ("; rollback to snapshot" if scn == "RollbackRetry"
                                                                 else "")
        if log.fallbacks != 1:
            return False, f"fallbacks {log.fallbacks}"
    bad = _equivalent(tr, ref, src, log, eng)
    assert [capi.tttstate_version(eng.pool, o) for o in owners] == [log.versions[s] for s in range(tr.n_streams)]
    return bad is None, bad or path


def test_stress_suite_5_of_5_and_negative_control():
    verdicts = {scn: _run_scenario(scn) for scn in SCENARIOS}
    print({k: v[1] for k, v in verdicts.items()})
    assert all(ok for ok, _ in verdicts.values()), verdicts            # Table 6: 5/5 pass
    prev = capi.tttstate_set_test_hook(capi.TTT_HOOK_NO_GROUP_ATOMICITY)
    try:
        try:
            ok, why = _run_scenario("MidGroupWriteFail")
        except (capi.TTTError, AssertionError) as ex:                 # e.g. the retry finds a cleared tail
            ok, why = False, str(ex)
    finally:
        capi.tttstate_set_test_hook(prev)
    assert not ok, "negative control: a non-atomic commit must fail MidGroupWriteFail"
    print("negative control:", why)

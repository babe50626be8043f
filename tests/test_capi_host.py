"""C-ABI library on the host (no GPU): exports, host-only pool state machine,
validation-before-side-effect error codes, and the C++ planner vs the oracle planner."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle.planner import Event, OraclePlanner
from paper_2605_28053_b200 import capi

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "tttstate.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 30, names
    lib = ctypes.CDLL(capi.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(capi.EXPORTED) | {"tttstate_status_name", "tttstate_last_error"}


def _host_pool(shape_id=0, placement=0, chunk=4, L=2, max_owners=16):
    sh = capi.make_shape(8, 16, chunk, L, "bf16")
    return capi.tttstate_pool_create(sh, shape_id, placement, max_owners, 2, None, 0, None)


def test_host_pool_state_machine_and_errors():
    p = _host_pool()
    assert capi.tttstate_alloc(p, 1) == 0
    assert capi.tttstate_alloc(p, 2, None, 7) == 7
    with pytest.raises(capi.TTTError) as e:
        capi.tttstate_alloc(p, 1)
    assert e.value.status == 2
    e1 = capi.tttstate_next_event(p, 1, 5)
    assert (e1.owner, e1.effect, e1.expected_version, e1.ready_step) == (1, capi.READ, 0, 5)
    evs = capi.tttstate_next_events(p, [2, 1], 5)                    # batched a1 == per-owner a1
    assert [(e.owner, e.effect, e.expected_version, e.ready_step) for e in evs] == [(2, capi.READ, 7, 5),
                                                                                  (1, capi.READ, 0, 5)]
    with pytest.raises(capi.TTTError) as e:
        capi.tttstate_next_events(p, [1, 99], 5)                        # unknown owner: whole call fails
    assert e.value.status == 1
    assert capi.tttstate_next_events(p, [], 5) == []
    g = capi.Group(capi.READ, [1, 2])
    capi.validate_group(p, g, [0, 7])
    for bad, code in [((capi.Group(capi.READ, [1, 1]), None), 4), ((g, [0, 6]), 3),
                      ((capi.Group(capi.READ, [1, 99]), None), 1),
                      ((capi.Group(capi.READ, [1], shape_id=3), None), 5)]:
        with pytest.raises(capi.TTTError) as e:
            capi.validate_group(p, *bad)
        assert e.value.status == code
    # validation precedes the no-device error; no side effects on failure
    with pytest.raises(capi.TTTError) as e:
        capi.read_apply(p, capi.Group(capi.WRITE, [1]), 0, 1, None, 1, None, 1)
    assert e.value.status == 13
    with pytest.raises(capi.TTTError) as e:
        capi.read_apply(p, g, 0, 1, None, 1, None, 1)
    assert e.value.status == -3
    with pytest.raises(capi.TTTError) as e:
        capi.tttstate_step_done(p, g)                # nothing was applied
    assert e.value.status == 14
    with pytest.raises(capi.TTTError) as e:
        capi.write_commit(p, capi.Group(capi.WRITE, [1]), 0.01)
    assert e.value.status == 7
    with pytest.raises(capi.TTTError) as e:
        capi.rollback(p, 1)
    assert e.value.status == 8
    capi.tttstate_snapshot(p, 1)
    assert capi.tttstate_version(p, 1) == 0 and capi.tttstate_tail_len(p, 1) == 0
    capi.tttstate_free(p, 1)
    with pytest.raises(capi.TTTError):
        capi.tttstate_version(p, 1)
    capi.tttstate_pool_destroy(p)


def test_pool_full_and_shape_errors():
    p = _host_pool(max_owners=2)
    capi.tttstate_alloc(p, 1)
    capi.tttstate_alloc(p, 2)
    with pytest.raises(capi.TTTError) as e:
        capi.tttstate_alloc(p, 3)
    assert e.value.status == 10
    with pytest.raises(capi.TTTError) as e:
        capi.tttstate_pool_bytes(capi.make_shape(8, 12, 4, 1, "bf16"), 1, 0)   # d_ff % 8
    assert e.value.status == 11
    n = capi.tttstate_pool_bytes(capi.make_shape(2560, 9728, 128, 36, "bf16"), 8, 0)
    assert n >= 16 * 36 * 2560 * 9728 * 2


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_cpp_planner_matches_oracle_planner(mode):
    """Bit-exact group composition / rejections vs oracle/planner.py on random event streams."""
    rs = np.random.default_rng(mode + 10)
    pools = [_host_pool(0, 0, max_owners=64), _host_pool(1, 0, max_owners=64)]
    V = {}
    for k in range(40):
        sid = k % 2
        v0 = int(rs.integers(0, 4))
        capi.tttstate_alloc(pools[sid], 100 + k, None, v0)
        V[100 + k] = v0
    for trial in range(60):
        B, w = int(rs.integers(1, 7)), int(rs.integers(0, 4))
        pl = capi.ttt_planner_create(mode, B, w)
        for p in pools:
            capi.ttt_planner_attach(pl, p)
        op = OraclePlanner(B, w, mode)
        waiting = set()
        for clock in range(10):
            evs = []
            for r in rs.permutation(list(V))[: int(rs.integers(0, 20))]:
                r = int(r)
                if r in waiting and rs.random() < 0.9:
                    continue
                v = V[r] if rs.random() < 0.85 else V[r] + 1
                evs.append((r, int(rs.integers(0, 2)), (r - 100) % 2, v))
            cev = [capi.ttt_event(r, eff, 0, sid, 0, v, clock) for (r, eff, sid, v) in evs]
            oev = [Event(r, eff, 0, sid, 0, v, clock) for (r, eff, sid, v) in evs]
            cg, crej = capi.plan_batch(pl, cev, clock)
            og, orej = op.plan(oev, clock, V.get)
            assert [(g.effect, g.c.shape_id, g.owners) for g in cg] == \
                   [(g.effect, g.shape_id, tuple(g.owners)) for g in og]
            assert [(e.owner, e.expected_version) for e in crej] == [(e.owner, e.version) for e in orej]
            for g in og:
                waiting -= set(g.owners)
            waiting |= {e.owner for e in oev} - {e.owner for e in orej}
        capi.ttt_planner_destroy(pl)


def test_binding_checks_tensor_operands_before_the_call():
    """tensors handed to read_apply / read_apply_chunk / tail_load / serve_step are
    checked against the pool's σ.dtype, contiguity, row width and row count; raw integer
    addresses stay the caller's unchecked opt-in path."""
    import torch
    p = _host_pool()                                   # bf16, d_model 8, d_ff 16
    capi.tttstate_alloc(p, 1)
    g = capi.Group(capi.READ, [1])
    X, V, Y = (torch.zeros(1, 16, dtype=torch.bfloat16), torch.zeros(1, 8, dtype=torch.bfloat16),
               torch.zeros(1, 8, dtype=torch.bfloat16))
    bad = [(X.float(), V, Y), (torch.zeros(1, 32, dtype=torch.bfloat16)[:, ::2], V, Y),
           (torch.zeros(1, 8, dtype=torch.bfloat16), V, Y), (X, V, torch.zeros(0, 8, dtype=torch.bfloat16))]
    for x, v, y in bad:
        with pytest.raises(ValueError):
            capi.read_apply(p, g, 0, x, None, v, None, y)
    with pytest.raises(ValueError):                    # a row map shorter than the group
        capi.read_apply(p, capi.Group(capi.READ, [1]), 0, X, [], V, None, Y)
    with pytest.raises(capi.TTTError) as e:            # well-formed operands reach the library
        capi.read_apply(p, g, 0, X, None, V, None, Y)
    assert e.value.status == -3                        # TTT_E_NO_DEVICE on a host-only pool
    capi.tttstate_pool_destroy(p)


def test_serve_step_validates_before_side_effects_on_a_host_pool():
    p = _host_pool()
    pl = capi.ttt_planner_create(capi.MODE_FULL, 8, 0)
    capi.ttt_planner_attach(pl, p)
    for o in (1, 2):
        capi.tttstate_alloc(p, o)
    bufs = capi.StepBuffers(16)
    bufs.owners[0], bufs.owners[1] = 1, 2
    with pytest.raises(capi.TTTError) as e:
        capi.tttstate_serve_step(p, pl, bufs, 2, 0, 1 << 20, 16, 2 << 20, 8, 3 << 20, 8, 0.01)
    assert e.value.status == -3                        # no device: nothing planned, nothing pending
    assert capi.ttt_planner_pending(pl) == 0
    bufs.owners[1] = 1
    with pytest.raises(capi.TTTError):
        capi.tttstate_serve_step(p, pl, bufs, 2, 0, 1 << 20, 16, 2 << 20, 8, 3 << 20, 8, 0.01)
    assert capi.tttstate_last_commit_seq(p) == 0
    capi.ttt_planner_destroy(pl)
    capi.tttstate_pool_destroy(p)


def test_rule1_shape_checks():
    """SPEC-compat rule 1 is accepted for a square fast-weight pool only."""
    ok = capi.make_shape(16, 16, 4, 1, "fp32", rule=1)
    p = capi.tttstate_pool_create(ok, 0, 0, 4, 0, None, 0, None)
    capi.tttstate_pool_destroy(p)
    for bad in (capi.make_shape(8, 16, 4, 1, "fp32", rule=1), capi.make_shape(16, 16, 4, 1, "fp32", rule=2)):
        with pytest.raises(capi.TTTError) as e:
            capi.tttstate_pool_create(bad, 0, 0, 4, 0, None, 0, None)
        assert e.value.status == 11

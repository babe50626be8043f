"""GPU parity: the CUDA path (through the C ABI) vs the CPU fp64 oracle, same seeded inputs.

Integers (owner ids, versions, commit/rollback log, census, group plan) must
be bit-exact; activations and fast weights within BASELINE.json's tolerance
(normwise max relative error 2e-2 bf16, 1e-5 fp32).
"""
import numpy as np
import pytest
import torch

from oracle import numerics as nm
from oracle.run import run_batched
from workload import rng
from workload import traces as T

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.serving import run_trace  # noqa: E402

from .gpu_helpers import HostGenInputs, make_engine  # noqa: E402

DEV = "cuda"


def _compare(tr, ref, src, log, eng):
    tol = nm.TOL[tr.dtype]
    assert set(ref.outputs) == set(src.out)
    worst = max(nm.normwise_rel_err(src.out[k], ref.outputs[k]) for k in ref.outputs)
    assert worst <= tol, f"READ outputs: normwise err {worst} > {tol}"
    assert log.versions == ref.versions
    assert log.commits == ref.commits
    assert log.census == ref.census
    assert log.plan == ref.plan
    werr, n_eq, n_all = 0.0, 0, 0
    for s in range(tr.n_streams):
        for l in range(tr.n_layers):
            got = nm.widen(capi.tttstate_read_payload(eng.pool, tr.owner(s), l, tr.d_model, tr.d_ff, tr.dtype), tr.dtype)
            werr = max(werr, nm.normwise_rel_err(got, ref.state[s][l]))
            n_eq += int(np.sum(got == ref.state[s][l]))
            n_all += got.size
    assert werr <= tol, f"fast weights: normwise err {werr} > {tol}"
    # the oracle mirrors the storage rounding (reading xi), so the committed bytes differ only
    # where fp32 accumulation order flips a rounding: bf16 (8-bit mantissa) >= 99 % bit-equal
    if tr.dtype == "bf16":
        assert n_eq / n_all >= 0.99, f"committed bf16 fast weights bit-equal in {n_eq / n_all:.4f} < 0.99"
    # elementwise p99 relative error of the READ outputs: reported for information (reading xii)
    p99 = float(np.percentile(np.concatenate([np.abs(src.out[k] - ref.outputs[k]) / (np.abs(ref.outputs[k]) + 1e-30)
                                              for k in list(ref.outputs)[:512]]), 99))
    print(f"parity {tr.name}: READ normwise {worst:.2e} (elementwise p99 {p99:.2e}), fast weights {werr:.2e}, "
          f"bit-equal {n_eq / n_all:.4f}")
    return worst, werr


def _run(tr, **kw):
    ref = run_batched(tr)
    eng = make_engine(tr, DEV, **kw)
    src = HostGenInputs(tr, DEV)
    log = run_trace(eng, tr, src)
    torch.cuda.synchronize()
    return ref, src, log, eng


def test_config1_tiny_fp32_parity():
    tr = T.config1_tiny()
    ref, src, log, eng = _run(tr)
    _compare(tr, ref, src, log, eng)
    assert [log.versions[0], log.versions[1]] == [4, 3]
    assert log.fallbacks == 1


@pytest.mark.parametrize("dtype,streams,d_model,d_ff", [("bf16", 9, 196, 328), ("fp32", 9, 196, 328),
                                                      ("bf16", 3, 100, 1000), ("bf16", 8, 2560, 1224),
                                                      ("bf16", 9, 200, 1536), ("bf16", 5, 64, 512)])
def test_uniform_parity_ragged_and_split_groups(dtype, streams, d_model, d_ff):
    # 9 members > 8 per READ launch (split), d_model/d_ff not tile multiples, 2 boundaries;
    # bf16 decode runs the mma.sync base: ragged 16-row blocks (196, 100), ragged 512-wide K
    # chunks (328, 1000, 1224), absent members (3 < 8), paper d_model (2560); whole 512-wide
    # K chunks only (1536: three, 512: one)
    tr = T.uniform_small(n_streams=streams, n_layers=2, d_model=d_model, d_ff=d_ff, chunk=8, n_steps=20,
                         dtype=dtype, delta0="rng", v0=5, seed=3)
    ref, src, log, eng = _run(tr)
    _compare(tr, ref, src, log, eng)


@pytest.mark.parametrize("mode,w", [(capi.MODE_SERIAL, 0), (capi.MODE_PHASE, 2), (capi.MODE_FULL, 0),
                                    (capi.MODE_FULL, 3)])
def test_bursty_controls_modes_parity(mode, w):
    tr = T.uniform_small(n_streams=6, n_layers=2, d_model=64, d_ff=96, chunk=4, n_steps=14, dtype="bf16",
                         delta0="rng", v0=2, offsets=(0, 1, 3, 2, 0, 3), mode=mode, w=w, seed=1,
                         controls={(1, 2): ["snapshot"], (1, 5): ["rollback"], (2, 0): ["fail"],
                                   (4, 3): ["fail"], (3, 9): ["snapshot"], (3, 11): ["rollback"],
                                   (5, 0): ["snapshot"], (5, 13): ["rollback"]})
    tr = tr.replace(B=4)
    ref, src, log, eng = _run(tr)
    _compare(tr, ref, src, log, eng)


def test_all_update_chunk1_parity():
    tr = T.uniform_small(n_streams=4, n_layers=1, d_model=64, d_ff=128, chunk=1, n_steps=10, dtype="bf16",
                         delta0="rng", seed=2)
    ref, src, log, eng = _run(tr)
    _compare(tr, ref, src, log, eng)
    assert set(log.versions.values()) == {10}


def _slot(eng, tr, s, which, l=0):
    return capi.tttstate_read_slot_raw(eng.pool, tr.owner(s), which, l, tr.d_model, tr.d_ff, tr.dtype)


def test_read_immutability_failed_write_and_rollback_bytes():
    tr = T.uniform_small(n_streams=2, n_layers=1, d_model=64, d_ff=96, chunk=2, n_steps=0, dtype="bf16",
                         delta0="rng", seed=4)
    eng = make_engine(tr, DEV, n_ckpt=1)
    src = HostGenInputs(tr, DEV)
    for s in range(2):
        capi.tttstate_alloc(eng.pool, tr.owner(s), src.init_delta(s), 0)
    pool, owners = eng.pool, [tr.owner(0), tr.owner(1)]
    g_read = capi.Group(capi.READ, owners)
    g_write = capi.Group(capi.WRITE, owners)

    def step(p, group):
        X, _, Vt, _, Y, _ = src.group_io(0, [0, 1], [p, p])
        capi.read_apply(pool, group, 0, X, None, Vt, None, Y)

    before = capi.tttstate_read_payload(pool, owners[0], 0, tr.d_model, tr.d_ff, "bf16")
    step(0, g_read)
    capi.tttstate_step_done(pool, g_read)
    assert np.array_equal(before, capi.tttstate_read_payload(pool, owners[0], 0, tr.d_model, tr.d_ff, "bf16"))
    with pytest.raises(capi.TTTError) as e:
        step(1, g_read)                       # a WRITE step issued as READ
    assert e.value.status == 13
    step(1, g_write)
    with pytest.raises(capi.TTTError) as e:
        capi.write_commit(pool, g_write, tr.eta, [False, True])   # MidGroupWriteFail
    assert e.value.status == capi.TTT_E_WRITE_FAILED
    # versions and committed bytes intact for BOTH members; the shadow slot was written
    assert [capi.tttstate_device_version(pool, o) for o in owners] == [0, 0]
    assert np.array_equal(before, capi.tttstate_read_payload(pool, owners[0], 0, tr.d_model, tr.d_ff, "bf16"))
    assert not np.array_equal(before, _slot(eng, tr, 0, 1))
    capi.tttstate_snapshot(pool, owners[0])
    assert capi.write_commit(pool, g_write, tr.eta) == [1, 1]
    after1 = capi.tttstate_read_payload(pool, owners[0], 0, tr.d_model, tr.d_ff, "bf16")
    assert not np.array_equal(before, after1)
    # second commit writes into the pinned slot -> checkpoint moves to the pool first
    for p in (2, 3):
        g = g_read if p == 2 else g_write
        step(p, g)
        if p == 2:
            capi.tttstate_step_done(pool, g)
    capi.write_commit(pool, g_write, tr.eta)
    assert capi.tttstate_version(pool, owners[0]) == 2
    assert np.array_equal(before, _slot(eng, tr, 0, 2))            # checkpoint-pool copy is exact
    assert capi.rollback(pool, owners[0]) == 0
    assert capi.tttstate_device_version(pool, owners[0]) == 0
    assert np.array_equal(before, capi.tttstate_read_payload(pool, owners[0], 0, tr.d_model, tr.d_ff, "bf16"))
    assert capi.tttstate_version(pool, owners[1]) == 2              # owner-local
    # fork isolation
    capi.tttstate_fork(pool, owners[1], 77)
    f0 = capi.tttstate_read_payload(pool, 77, 0, tr.d_model, tr.d_ff, "bf16")
    assert np.array_equal(f0, capi.tttstate_read_payload(pool, owners[1], 0, tr.d_model, tr.d_ff, "bf16"))
    assert capi.tttstate_version(pool, 77) == 2


def test_device_detected_nonfinite_write_fails_group():
    tr = T.uniform_small(n_streams=2, n_layers=1, d_model=64, d_ff=96, chunk=1, n_steps=0, dtype="fp32", seed=5)
    eng = make_engine(tr, DEV)
    pool, owners = eng.pool, [tr.owner(0), tr.owner(1)]
    for o in owners:
        capi.tttstate_alloc(pool, o)
    g = capi.Group(capi.WRITE, owners)
    X = torch.ones(2, tr.d_ff, device=DEV)
    X[1, 3] = float("inf")
    Vt = torch.ones(2, tr.d_model, device=DEV)
    Y = torch.empty(2, tr.d_model, device=DEV)
    capi.read_apply(pool, g, 0, X, None, Vt, None, Y)
    assert capi.write_commit(pool, g, tr.eta) == [1, 1]      # optimistic host mirror, no host sync
    seq = capi.tttstate_last_commit_seq(pool)
    # the device fails the group and resolves App. H's singleton retries at once (control.cu):
    # owner 0's candidate is finite -> published; owner 1's is not -> refused for good (reading xx)
    assert capi.tttstate_sync(pool) == 1
    assert capi.tttstate_refusals(pool) == [(owners[1], 0, seq)]
    assert [capi.tttstate_version(pool, o) for o in owners] == [1, 0]
    assert [capi.tttstate_device_version(pool, o) for o in owners] == [1, 0]
    assert [capi.tttstate_tail_len(pool, o) for o in owners] == [0, 0]        # owner 1's evidence dropped
    assert capi.tttstate_next_event(pool, owners[1], 0).effect == 1 and capi.tttstate_sync(pool) == 0


@pytest.mark.parametrize("native", [True, False])
@pytest.mark.parametrize("dtype,chunk", [("bf16", 4), ("fp32", 4), ("bf16", 1)])
def test_poisoned_evidence_device_failure_through_the_serving_loop(native, dtype, chunk):
    """a non-finite candidate (an inf target in the chunk's evidence) fails its WRITE group on
    the device; App. H's singleton retries publish the clean members and refuse the poisoned one for good
    (v and bytes kept, evidence dropped).  Logs, versions, outputs and fast weights match the oracle, which
    follows the same reading (oracle/run.py _retry); snapshots / rollbacks / injected failures around it."""
    tr = T.uniform_small(n_streams=6, n_layers=2, d_model=128, d_ff=256, chunk=chunk, n_steps=4 * chunk + 2,
                         dtype=dtype, delta0="rng", v0=2, seed=21,
                         controls={(1, chunk - 1): ["poison"], (3, 2 * chunk - 1): ["poison", "fail"],
                                   (4, chunk): ["snapshot"], (4, 2 * chunk + 1): ["rollback"],
                                   (0, 3 * chunk - 1): ["fail"], (2, 2 * chunk): ["poison"]})
    ref = run_batched(tr)
    eng = make_engine(tr, DEV)
    src = HostGenInputs(tr, DEV)
    log = run_trace(eng, tr, src, native=native)
    torch.cuda.synchronize()
    _compare(tr, ref, src, log, eng)
    assert log.device_failures >= 1
    finals = {s for s in (1, 2, 3) if sum(c[0] == s and c[4] == "failed" for c in log.commits) >= 2}
    assert finals == {1, 2, 3}          # group attempt + final singleton failure of every poisoned stream


def test_generator_device_matches_numpy():
    for bf16 in (True, False):
        for (t, o, l, p, n, amp) in [(rng.T_X, 1003, 2, 17, 1000, 1.0), (rng.T_W_DOWN, 0, 5, 0, 4099, 0.0101),
                                     (rng.T_TGT, 7, 0, -3, 333, 1.0)]:
            out = torch.empty(n, dtype=torch.bfloat16 if bf16 else torch.float32, device=DEV)
            capi.gen_uniform(out, 11, t, o, l, p, n, amp, bf16)
            ref = rng.gen(11, t, o, l, p, (n,), amp, "bf16" if bf16 else "fp32")
            got = out.view(torch.int16).cpu().numpy().view(np.uint16) if bf16 else out.cpu().numpy()
            assert np.array_equal(got, ref)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("impl", [0, 1])   # 0: fused C=1 READ+WRITE (f3), 1: separate SIMT WRITE
def test_all_update_streaming_learner_controls(dtype, impl):
    tr = T.uniform_small(n_streams=5, n_layers=2, d_model=128, d_ff=192, chunk=1, n_steps=9, dtype=dtype,
                         delta0="rng", seed=12, v0=3,
                         controls={(0, 2): ["snapshot"], (0, 5): ["rollback"], (1, 1): ["fail"], (3, 0): ["snapshot"],
                                   (3, 4): ["rollback"], (4, 6): ["fail"], (2, 3): ["snapshot"]})
    prev = capi.tttstate_set_write_impl(impl)
    try:
        ref, src, log, eng = _run(tr)
    finally:
        capi.tttstate_set_write_impl(prev)
    _compare(tr, ref, src, log, eng)
    assert log.fallbacks == 2


def _random_shapes(n, seed):
    g = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        dtype = ["bf16", "bf16", "fp32"][g.integers(3)]
        vec = 8 if dtype == "bf16" else 4
        d_model = int(g.integers(4, 120)) * 4                       # multiples of 4, not of 16 / 128
        d_ff = int(g.integers(2, 160)) * vec
        streams = int(g.integers(1, 13))
        chunk = int([1, 2, 3, 5, 16][g.integers(5)])
        out.append((dtype, d_model, d_ff, streams, chunk, int(g.integers(1 << 30))))
    return out


def _tc_read_shapes(n, seed):
    """bf16 shapes the TMA + tcgen05 decode READ serves (d_model >= 128, d_ff >= 64, ≤ 8 members):
    row blocks and 64-wide K boxes both ragged (TMA out-of-bounds fill), 1..8 members."""
    g = np.random.default_rng(seed)
    return [(int(g.integers(32, 180)) * 4, int(g.integers(8, 150)) * 8, int(g.integers(1, 9)), int(g.integers(1 << 30)))
            for _ in range(n)]


@pytest.mark.parametrize("d_model,d_ff,streams,seed", _tc_read_shapes(8, 77))
def test_tc_read_ragged_shapes_parity(d_model, d_ff, streams, seed):
    tr = T.uniform_small(n_streams=streams, n_layers=2, d_model=d_model, d_ff=d_ff, chunk=8, n_steps=18, dtype="bf16",
                         delta0="rng", v0=1, seed=seed % 1000)
    ref, src, log, eng = _run(tr)
    _compare(tr, ref, src, log, eng)


@pytest.mark.parametrize("dtype,d_model,d_ff,streams,chunk,seed", _random_shapes(6, 2026))
def test_random_shapes_parity(dtype, d_model, d_ff, streams, chunk, seed):
    """Seeded random shapes: ragged row blocks / K chunks / vector tails, 1..12 members
    (split READ launches), C = 1 (fused f3 path) to 16, both dtypes, two boundaries."""
    tr = T.uniform_small(n_streams=streams, n_layers=2, d_model=d_model, d_ff=d_ff, chunk=chunk,
                         n_steps=2 * chunk + 1, dtype=dtype, delta0="rng", v0=1, seed=seed % 1000)
    ref, src, log, eng = _run(tr)
    _compare(tr, ref, src, log, eng)


def test_determinism_bitwise_rerun():
    # SPEC acceptance criterion 10 (determinism): every reduction runs in a fixed order (per-row
    # tickets, fixed-order partial sums, no data atomics), so rerunning a trace on fresh pools
    # reproduces every READ output and every committed fast-weight byte exactly
    tr = T.uniform_small(n_streams=8, n_layers=2, d_model=256, d_ff=1536, chunk=8, n_steps=17, dtype="bf16",
                         delta0="rng", v0=3, seed=12)
    runs = []
    for _ in range(2):
        eng = make_engine(tr, DEV)
        src = HostGenInputs(tr, DEV)
        log = run_trace(eng, tr, src)
        torch.cuda.synchronize()
        pay = [capi.tttstate_read_payload(eng.pool, tr.owner(s), l, tr.d_model, tr.d_ff, tr.dtype).tobytes()
               for s in range(tr.n_streams) for l in range(tr.n_layers)]
        runs.append((log.versions, {k: v.tobytes() for k, v in src.out.items()}, pay))
    assert runs[0][0] == runs[1][0]
    assert runs[0][1] == runs[1][1]
    assert runs[0][2] == runs[1][2]


@pytest.mark.parametrize("dtype,chunk", [("fp32", 4), ("bf16", 8), ("fp32", 1)])
def test_rule1_spec_mean_rule_parity(dtype, chunk):
    """SPEC-compat rule 1 on the GPU (S:188 y = x + ΔW x, S:206 / S:215
    ΔW += η m mᵀ with m the chunk mean): a square trace with snapshots, rollbacks and an injected
    failure against the oracle's rule-1 arithmetic; the base W_down is the identity."""
    tr = T.uniform_small(n_streams=4, n_layers=2, d_model=96, d_ff=96, chunk=chunk, n_steps=3 * chunk + 1,
                         dtype=dtype, rule=1, seed=17,
                         controls={(1, chunk - 1): ["snapshot"], (1, chunk): ["rollback"], (2, 2 * chunk - 1): ["fail"]})
    ref, src, log, eng = _run(tr)
    _compare(tr, ref, src, log, eng)


def test_rule1_spec_worked_example_s219():
    """W = 0 (ΔW_0), z = (1, 1) twice (m = (1, 1)), η = 0.01 -> ΔW = 0.01·[[1,1],[1,1]]
    (d = 2 is below the kernels' vector width, so d = 8 with the example in the leading 2×2 block
    and zeros elsewhere); y on the boundary token = x + ΔW_0 x = x."""
    d, C = 8, 2
    W = torch.eye(d, device=DEV).unsqueeze(0).contiguous()
    from paper_2605_28053_b200.serving import Engine
    eng = Engine(d, d, C, 1, "fp32", 2, W, eta=0.01, rule=1)
    pool = eng.pool
    capi.tttstate_alloc(pool, 5)
    x = torch.zeros(1, d, device=DEV)
    x[0, :2] = 1.0
    v = torch.zeros(1, d, device=DEV)
    Y = torch.empty(1, d, device=DEV)
    for effect in (capi.READ, capi.WRITE):
        g = capi.Group(effect, [5])
        capi.read_apply(pool, g, 0, x, None, v, None, Y)
        assert torch.equal(Y, x)                    # ΔW_0 = 0: y = x
        if effect == capi.READ:
            capi.tttstate_step_done(pool, g)
    assert capi.write_commit(pool, capi.Group(capi.WRITE, [5]), 0.01) == [1]
    dw = capi.tttstate_read_payload(pool, 5, 0, d, d, "fp32")
    ref = np.zeros((d, d), dtype=np.float32)
    ref[:2, :2] = np.float32(0.01)
    assert np.array_equal(dw, ref) and capi.tttstate_version(pool, 5) == 1
    eng.close()

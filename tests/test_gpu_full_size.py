"""Full-size parity for every path whose performance is claimed (VERDICT r1 "next" 2): paper dims
(d_model 2560, d_ff 9728 — Qwen3-4B), bf16, in the launch configurations the benchmarks
time, with the oracle run on sampled streams one by one (run_sequential(streams=...): per-request
results do not depend on the grouping, P:295-297 / P:299-308):

  * f3 streaming learner (C = 1, all-update) with snapshot / rollback / injected failure;
  * the configs 3 / 5 decode READ with 64 members per group (8 launches per layer, the L2
    evict_last / evict_first W_down hints) on a bursty trace with failures and rollbacks;
  * f2 chunk-granular READ (prefill) with 8 and 64 members (the full 152-block K loop);
  * f1 low-rank READ / WRITE at R = 16 and 64 with 128 members (fused tcgen05 base GEMM with its
    split-K), speculative branches (fork / snapshot / rollback / release).

Integers (versions, commit / rollback outcomes) bit-exact; floats within BASELINE.json's 2e-2
normwise bound, and committed fast weights — where the oracle mirrors the bf16 storage rounding
(reading xi) — bit-equal in >= 99 % of the elements.
"""
import numpy as np
import pytest
import torch

from oracle import numerics as nm
from oracle.run import ok_commits, run_sequential
from workload import rng
from workload import traces as T

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1500)]

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.serving import Engine, run_trace  # noqa: E402

from .gpu_helpers import DeviceGenInputs, read_lowrank  # noqa: E402

DEV = "cuda"
DM, DFF = 2560, 9728
TOL = nm.TOL["bf16"]


def _engine(tr, src, max_owners=None, n_ckpt=0):
    W = src.w_down()
    return Engine(tr.d_model, tr.d_ff, tr.chunk, tr.n_layers, "bf16", max_owners or tr.n_streams, W, n_ckpt=n_ckpt,
                  B=tr.B, w=tr.w, eta=tr.eta, backend=tr.backend, rank=tr.rank), W


def _check_sampled(tr, eng, src, log, sample):
    ref = run_sequential(tr, streams=sample)
    assert set(ref.outputs) <= set(src.out)
    worst = max(nm.normwise_rel_err(src.out[k], ref.outputs[k]) for k in ref.outputs)
    assert worst <= TOL, worst
    got_ok = {s: c for s, c in ok_commits_log(log).items() if s in sample}
    assert got_ok == {s: c for s, c in ok_commits(ref).items()}
    for s in sample:
        assert log.versions[s] == ref.versions[s]
        for l in range(tr.n_layers):
            got = nm.widen(capi.tttstate_read_payload(eng.pool, tr.owner(s), l, tr.d_model, tr.d_ff, "bf16"), "bf16")
            assert nm.normwise_rel_err(got, ref.state[s][l]) <= TOL
            assert np.mean(got == ref.state[s][l]) >= 0.99, (s, l, np.mean(got == ref.state[s][l]))
    return worst


def ok_commits_log(log):
    out = {}
    for (s, p, vb, va, oc) in log.commits:
        if oc != "failed":
            out.setdefault(s, []).append((p, vb, va, oc))
    return out


def test_f3_streaming_learner_paper_dims():
    """C = 1: every step is a WRITE whose evidence is its own token; the fused single-pass READ+WRITE
    kernel (f3) writes the candidate while it streams ΔW (reading xvii: y uses the pre-update row)."""
    sample = (0, 2, 5)
    tr = T.uniform_small(n_streams=8, n_layers=2, d_model=DM, d_ff=DFF, chunk=1, n_steps=3, dtype="bf16",
                         delta0="rng", v0=5, seed=31,
                         controls={(2, 0): ["snapshot"], (2, 2): ["rollback"], (5, 1): ["fail"]})
    src = DeviceGenInputs(tr, DEV, record_streams=sample)
    eng, _W = _engine(tr, src, n_ckpt=2)
    log = run_trace(eng, tr, src)
    torch.cuda.synchronize()
    assert log.fallbacks == 1 and log.census == {0: 0, 1: 24}
    _check_sampled(tr, eng, src, log, sample)


def test_config3_decode_read_64_members_paper_dims():
    """The configs 3 / 5 READ: one group of 64 members = 8 launches per layer; launches 1-7 load
    W_down with the L2 evict_last hint and ΔW with evict_first.  Bursty offsets put the sampled
    streams across a boundary (WRITE of a 64-wide group, tcgen05), with an injected failure and a
    snapshot + rollback on sampled streams."""
    sample = (0, 9, 63)
    # offsets 124..126: step 0 is a 64-member READ group, the boundaries fall on p = 1, 2, 3
    offs = tuple({0: 126, 9: 125, 63: 126}.get(s, 124 + s % 3) for s in range(64))
    tr = T.Trace("config3_fullsize", n_streams=64, n_layers=2, d_model=DM, d_ff=DFF, chunk=128, n_steps=4,
                 dtype="bf16", seed=33, v0=3, delta0="rng", offsets=offs, B=64, w=0,
                 controls={(0, 1): ["fail"], (9, 1): ["snapshot"], (9, 3): ["rollback"]})
    src = DeviceGenInputs(tr, DEV, record_streams=sample)
    eng, _W = _engine(tr, src, n_ckpt=4)
    log = run_trace(eng, tr, src)
    torch.cuda.synchronize()
    assert log.fallbacks >= 1 and any(c[4] == "rolled_back" and c[0] == 9 for c in log.commits)
    assert max(len(ss) for _, _, ss, _ in log.plan) == 64
    _check_sampled(tr, eng, src, log, sample)


@pytest.mark.parametrize("members", [8, 64])
def test_f2_chunk_read_paper_dims(members):
    """Prefill: one chunk of C = 128 tokens per member through read_apply_chunk (tcgen05 TN GEMM,
    W + ΔW in one TMEM accumulator, the full d_ff = 9728 K loop), then the boundary WRITE."""
    sample = (0, members - 1)
    tr = T.uniform_small(n_streams=members, n_layers=1, d_model=DM, d_ff=DFF, chunk=128, n_steps=128, dtype="bf16",
                         delta0="rng", v0=2, seed=35)
    src = DeviceGenInputs(tr, DEV)
    eng, _W = _engine(tr, src)
    owners = [tr.owner(s) for s in range(members)]
    for s, o in enumerate(owners):
        capi.tttstate_alloc(eng.pool, o, src.init_delta(s), tr.v0)
    X = torch.empty(members, 128, DFF, dtype=torch.bfloat16, device=DEV)
    V = torch.empty(members, 128, DM, dtype=torch.bfloat16, device=DEV)
    for s in range(members):
        for p in range(128):
            capi.gen_uniform(X[s, p], tr.seed, rng.T_X, tr.owner(s), 0, p, DFF, 1.0, True)
            capi.gen_uniform(V[s, p], tr.seed, rng.T_TGT, tr.owner(s), 0, p, DM, 1.0, True)
    Y = torch.empty(members, 128, DM, dtype=torch.bfloat16, device=DEV)
    g = capi.Group(capi.WRITE, owners)
    capi.read_apply_chunk(eng.pool, g, 0, X, V, Y)
    assert capi.write_commit(eng.pool, g, tr.eta) == [tr.v0 + 1] * members
    torch.cuda.synchronize()
    ref = run_sequential(tr, streams=sample)
    Yh = Y.float().cpu().numpy().astype(np.float64)
    worst = max(nm.normwise_rel_err(Yh[s, p], ref.outputs[(s, p, 0)]) for s in sample for p in range(128))
    assert worst <= TOL, worst
    for s in sample:
        assert capi.tttstate_version(eng.pool, tr.owner(s)) == ref.versions[s] == tr.v0 + 1
        got = nm.widen(capi.tttstate_read_payload(eng.pool, tr.owner(s), 0, DM, DFF, "bf16"), "bf16")
        assert nm.normwise_rel_err(got, ref.state[s][0]) <= TOL
        assert np.mean(got == ref.state[s][0]) >= 0.99


@pytest.mark.parametrize("rank", [16, 64])
def test_f1_lowrank_128_members_paper_dims(rank):
    """BJ configs[3] at full size: 128 streams, R = 16 / 64, the fused low-rank READ (tcgen05 base
    GEMM with split-K + u = A x, Bᵀu streams); tails pre-filled so each stream's boundary comes
    at p = 3 with a fork + snapshot, the speculative WRITE rolled back or kept (p = 0.75)."""
    sample = (0, 77, 127)
    tr = T.config4_lowrank(n_steps=6, n_layers=2, rank=rank, n_streams=128, seed=37, offset=124)
    src = DeviceGenInputs(tr, DEV, record_streams=sample)
    eng, _W = _engine(tr, src, max_owners=2 * 128 + 2, n_ckpt=130)
    log = run_trace(eng, tr, src)
    torch.cuda.synchronize()
    ref = run_sequential(tr, streams=sample)
    worst = max(nm.normwise_rel_err(src.out[k], ref.outputs[k]) for k in ref.outputs)
    assert worst <= TOL, worst
    assert {s: c for s, c in ok_commits_log(log).items() if s in sample} == ok_commits(ref)
    assert any(c[4] == "rolled_back" for c in log.commits)
    for s in sample:
        assert log.versions[s] == ref.versions[s]
        for l in range(tr.n_layers):
            A, B = read_lowrank(eng, tr, tr.owner(s), l)
            rA, rB = ref.state[s][l]
            assert nm.normwise_rel_err(A, rA) <= TOL and np.array_equal(B, rB)
            assert np.mean(A == rA) >= 0.99
    for b, (v, S) in ref.branches.items():                       # fork isolation at full size
        assert log.branches[b] == v
        A, B = read_lowrank(eng, tr, b, 0)
        assert nm.normwise_rel_err(A, S[0][0]) <= TOL and np.array_equal(B, S[0][1])

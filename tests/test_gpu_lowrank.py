"""NEXT f1 parity: low-rank delta TTTState + speculative branch lineages (BJ configs[3]
structure at reduced dims) — READ (u = A x, tcgen05 base GEMM with split-K, y = base + Bᵀu),
WRITE (A' = A + η(A m)mᵀ, B' = B), fork / release / snapshot / rollback."""
import pytest
import torch

from oracle import numerics as nm
from oracle.run import run_batched
from workload import traces as T

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_28053_b200.serving import run_trace  # noqa: E402

from .gpu_helpers import HostGenInputs, make_engine, read_lowrank  # noqa: E402

DEV = "cuda"


@pytest.mark.parametrize("rank,streams,d_model,d_ff", [(8, 16, 256, 384), (16, 130, 320, 256), (64, 4, 256, 448), (16, 6, 400, 256)])
def test_config4_lowrank_branches_parity(rank, streams, d_model, d_ff):
    tr = T.config4_lowrank(n_steps=26, n_layers=2, rank=rank, d_model=d_model, d_ff=d_ff, chunk=8,
                           n_streams=streams, seed=rank)
    tr = tr.replace(B=min(streams, 256))
    ref = run_batched(tr)
    eng = make_engine(tr, DEV, n_ckpt=streams + 2, max_owners=2 * streams + 2)
    src = HostGenInputs(tr, DEV)
    log = run_trace(eng, tr, src)
    torch.cuda.synchronize()
    tol = nm.TOL["bf16"]
    worst = max(nm.normwise_rel_err(src.out[k], ref.outputs[k]) for k in ref.outputs)
    assert worst <= tol, worst
    assert log.versions == ref.versions and log.commits == ref.commits and log.plan == ref.plan
    assert log.branches == {b: v for b, (v, _) in ref.branches.items()}
    for s in range(min(streams, 6)):
        for l in range(tr.n_layers):
            A, B = read_lowrank(eng, tr, tr.owner(s), l)
            rA, rB = ref.state[s][l]
            assert nm.normwise_rel_err(A, rA) <= tol and nm.normwise_rel_err(B, rB) == 0.0
    for b, (v, S) in list(ref.branches.items())[:4]:           # fork isolation: branch bytes = source at fork
        for l in range(tr.n_layers):
            A, B = read_lowrank(eng, tr, b, l)
            assert nm.normwise_rel_err(A, S[l][0]) <= tol and nm.normwise_rel_err(B, S[l][1]) == 0.0


def test_two_lowrank_pools_on_two_streams():
    """Two low-rank pools driven concurrently on two CUDA streams (the fused READ spin-waits
    across CTAs, so with two live pools it launches cooperatively): both match the oracle."""
    trs = [T.config4_lowrank(n_steps=18, n_layers=2, rank=16, d_model=256, d_ff=384, chunk=8, n_streams=24,
                             seed=40 + k).replace(B=24, owner_base=5000 * (k + 1)) for k in range(2)]
    refs = [run_batched(tr) for tr in trs]
    engs = [make_engine(tr, DEV, n_ckpt=26, max_owners=50) for tr in trs]
    srcs = [HostGenInputs(tr, DEV) for tr in trs]
    streams = [torch.cuda.Stream() for _ in trs]
    from paper_2605_28053_b200.serving import Server
    srvs = [Server(e, tr, src, stream=st) for e, tr, src, st in zip(engs, trs, srcs, streams)]
    for srv in srvs:
        srv.admit()
    while not all(srv.done() for srv in srvs):                  # interleave the two serving loops
        for srv in srvs:
            if not srv.done():
                srv.step()
    torch.cuda.synchronize()
    for srv, tr, ref, src in zip(srvs, trs, refs, srcs):
        log = srv.finish()
        assert log.versions == ref.versions and log.commits == ref.commits
        worst = max(nm.normwise_rel_err(src.out[k], ref.outputs[k]) for k in ref.outputs)
        assert worst <= nm.TOL["bf16"], worst


def test_lowrank_contiguous_rows_of_a_larger_buffer_no_gather():
    """The native step tells the library how many rows each layer's X holds (ttt_step_io.rows_total);
    a low-rank group whose tokens sit in contiguous rows x_row0 .. x_row0 + n - 1 of that buffer runs
    the fused READ with the TMA row offset instead of gathering X (r2).  Rows start at 37 here."""
    from paper_2605_28053_b200.serving import StepIO

    class OffsetRows(HostGenInputs):
        def step_io(self, ss, ps):
            io = super().step_io(ss, ps)
            n, off, L = len(ss), 37, len(self.layers)
            X = torch.zeros(L, n + 80, self.tr.d_ff, dtype=io.X.dtype, device=DEV)
            V = torch.zeros(L, n + 80, self.tr.d_model, dtype=io.X.dtype, device=DEV)
            Y = torch.zeros(L, n + 80, self.tr.d_model, dtype=io.X.dtype, device=DEV)
            X[:, off:off + n] = io.X
            V[:, off:off + n] = io.Vt
            return StepIO(X, (n + 80) * self.tr.d_ff, V, (n + 80) * self.tr.d_model, Y, (n + 80) * self.tr.d_model,
                          [off + i for i in range(n)], n + 80)

    tr = T.config4_lowrank(n_steps=18, n_layers=2, rank=16, d_model=256, d_ff=384, chunk=8, n_streams=24, seed=9)
    tr = tr.replace(B=24)
    ref = run_batched(tr)
    eng = make_engine(tr, DEV, n_ckpt=26, max_owners=50)
    src = OffsetRows(tr, DEV)
    log = run_trace(eng, tr, src)
    torch.cuda.synchronize()
    worst = max(nm.normwise_rel_err(src.out[k], ref.outputs[k]) for k in ref.outputs)
    assert worst <= nm.TOL["bf16"], worst
    assert log.versions == ref.versions and log.commits == ref.commits

"""NEXT f2 parity: chunk-granular READ (prefill, tcgen05) vs the oracle's sequential
token-by-token execution — identical semantics because every READ of a chunk sees the
same committed version (Table 3) and the chunk ends in its WRITE."""
import numpy as np
import pytest
import torch

from oracle import numerics as nm
from oracle.run import run_sequential
from workload import traces as T

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_28053_b200 import capi  # noqa: E402

from .gpu_helpers import make_engine, to_dev, to_host_f64  # noqa: E402

DEV = "cuda"


def run_prefill(tr, eng):
    owners = [tr.owner(s) for s in range(tr.n_streams)]
    for s, o in enumerate(owners):
        d0 = None if tr.delta0 == "zero" else to_dev(np.stack([tr.delta0_of(s, l) for l in range(tr.n_layers)]),
                                                     tr.dtype, DEV)
        capi.tttstate_alloc(eng.pool, o, d0, tr.v0)
    g = capi.Group(capi.WRITE, owners)
    outs = {}
    for k in range(tr.n_steps // tr.chunk):
        ps = range(k * tr.chunk, (k + 1) * tr.chunk)
        for l in range(tr.n_layers):
            X = to_dev(np.stack([np.stack([tr.x(s, p, l) for p in ps]) for s in range(tr.n_streams)]), "bf16", DEV)
            V = to_dev(np.stack([np.stack([tr.tgt(s, p, l) for p in ps]) for s in range(tr.n_streams)]), "bf16", DEV)
            Y = torch.empty(tr.n_streams, tr.chunk, tr.d_model, dtype=torch.bfloat16, device=DEV)
            capi.read_apply_chunk(eng.pool, g, l, X, V, Y)
            Yh = to_host_f64(Y)
            for s in range(tr.n_streams):
                for i, p in enumerate(ps):
                    outs[(s, p, l)] = Yh[s, i]
        assert capi.write_commit(eng.pool, g, tr.eta) == [tr.v0 + k + 1] * tr.n_streams
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("d_model,d_ff,chunk,streams", [(320, 384, 16, 3), (256, 448, 64, 2), (384, 256, 128, 2),
                                                        (640, 512, 48, 9), (400, 320, 32, 5),
                                                        (2560, 256, 128, 8), (2560, 1024, 128, 8),
                                                        (1024, 2048, 100, 4)])
def test_chunk_read_prefill_parity(d_model, d_ff, chunk, streams):
    # d_model 400 / 2560 exercise the mixed-width N blocks (25 × 16 / 16 × 144 + 2 × 128)
    tr = T.uniform_small(n_streams=streams, n_layers=2, d_model=d_model, d_ff=d_ff, chunk=chunk, n_steps=2 * chunk,
                         dtype="bf16", delta0="rng", v0=4, seed=21)
    eng = make_engine(tr, DEV)
    outs = run_prefill(tr, eng)
    ref = run_sequential(tr)
    assert set(outs) == set(ref.outputs)
    worst = max(nm.normwise_rel_err(outs[k], ref.outputs[k]) for k in ref.outputs)
    assert worst <= nm.TOL["bf16"], worst
    for s in range(tr.n_streams):
        assert capi.tttstate_version(eng.pool, tr.owner(s)) == ref.versions[s] == tr.v0 + 2
        for l in range(tr.n_layers):
            got = nm.widen(capi.tttstate_read_payload(eng.pool, tr.owner(s), l, d_model, d_ff, "bf16"), "bf16")
            assert nm.normwise_rel_err(got, ref.state[s][l]) <= nm.TOL["bf16"]


def test_chunk_read_contract_errors():
    tr = T.uniform_small(n_streams=2, n_layers=2, d_model=256, d_ff=256, chunk=16, n_steps=0, dtype="bf16", seed=2)
    eng = make_engine(tr, DEV)
    owners = [tr.owner(s) for s in range(2)]
    for o in owners:
        capi.tttstate_alloc(eng.pool, o)
    X = torch.zeros(2, 16, 256, dtype=torch.bfloat16, device=DEV)
    V = torch.zeros(2, 16, 256, dtype=torch.bfloat16, device=DEV)
    Y = torch.empty(2, 16, 256, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(capi.TTTError) as e:
        capi.read_apply_chunk(eng.pool, capi.Group(capi.READ, owners), 0, X, V, Y)
    assert e.value.status == 13
    g = capi.Group(capi.WRITE, owners)
    capi.read_apply_chunk(eng.pool, g, 0, X, V, Y)
    with pytest.raises(capi.TTTError) as e:
        capi.read_apply_chunk(eng.pool, g, 0, X, V, Y)        # same layer twice
    assert e.value.status == 15
    with pytest.raises(capi.TTTError) as e:
        capi.write_commit(eng.pool, g, 0.01)                   # layer 1 not applied yet
    assert e.value.status == 7
    with pytest.raises(capi.TTTError) as e:                    # decode READ mid-chunk is refused
        capi.read_apply(eng.pool, capi.Group(capi.READ, owners), 1, X[:, 0].contiguous(), None,
                        V[:, 0].contiguous(), None, Y[:, 0].contiguous())
    assert e.value.status == 13
    capi.read_apply_chunk(eng.pool, g, 1, X, V, Y)
    with pytest.raises(capi.TTTError) as e:                    # a chunk ends in write_commit,
        capi.tttstate_step_done(eng.pool, capi.Group(capi.READ, owners))   # not in a READ step_done
    assert e.value.status == 13 and capi.tttstate_tail_len(eng.pool, owners[0]) == tr.chunk - 1
    assert capi.write_commit(eng.pool, g, 0.01) == [1, 1]
    assert capi.tttstate_tail_len(eng.pool, owners[0]) == 0


def test_chunk_read_deterministic():
    """Two engines, same inputs: the chunk READ outputs are bit-identical (the wide split-K
    kernel adds its K-slab partials in a fixed order, never by arrival)."""
    tr = T.uniform_small(n_streams=8, n_layers=1, d_model=2560, d_ff=1024, chunk=128, n_steps=128, dtype="bf16",
                         delta0="rng", v0=2, seed=5)
    a = run_prefill(tr, make_engine(tr, DEV))
    b = run_prefill(tr, make_engine(tr, DEV))
    assert all(np.array_equal(a[k], b[k]) for k in a)

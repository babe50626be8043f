"""T6 multi-GPU path on one B200: two ranks (gloo, both on cuda:0 —
the pool has one GPU per call) each serve their owner shard π(o) = s mod 2 of a mixed
READ/WRITE/failure/rollback trace through the C ABI.  Per rank: equivalence to the oracle
restricted to that rank's owners (the oracle run on the same shard).  Across ranks: the
gathered versions and payload digests equal a single-process run of the whole trace (the
fast weights of an owner depend on its own evidence only, so they are bit-identical however
the owners are grouped or placed)."""
import hashlib
import os
import socket

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _trace():
    from workload import traces as T
    return T.config3_interleaved(n_steps=40, n_layers=2, w=2, d_model=256, d_ff=384, chunk=16, seed=7)


def _serve(tr):
    """Run a (shard) trace through the CUDA path; returns (log, src, eng, {owner: (version, digest)})."""
    from paper_2605_28053_b200 import capi
    from paper_2605_28053_b200.serving import run_trace
    from tests.gpu_helpers import HostGenInputs, make_engine

    eng = make_engine(tr, "cuda")
    src = HostGenInputs(tr, "cuda")
    log = run_trace(eng, tr, src)
    torch.cuda.synchronize()
    out = {}
    for s in range(tr.n_streams):
        o = tr.owner(s)
        h = hashlib.sha256()
        for l in range(tr.n_layers):
            h.update(capi.tttstate_read_payload(eng.pool, o, l, tr.d_model, tr.d_ff, tr.dtype).tobytes())
        out[o] = (log.versions[s], h.hexdigest())
    return log, src, eng, out


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle import numerics as nm
    from oracle.run import run_batched
    from paper_2605_28053_b200 import capi
    from paper_2605_28053_b200 import distributed as D
    from workload import traces as T

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = T.shard(_trace(), world, rank)
        log, src, eng, mine = _serve(tr)
        ref = run_batched(tr)                                     # the oracle restricted to this rank's owners
        assert (log.versions, log.commits, log.census) == (ref.versions, ref.commits, ref.census)
        worst = max(nm.normwise_rel_err(src.out[k], ref.outputs[k]) for k in ref.outputs)
        assert worst <= nm.TOL[tr.dtype], worst
        for s in range(tr.n_streams):
            for l in range(tr.n_layers):
                got = capi.tttstate_read_payload(eng.pool, tr.owner(s), l, tr.d_model, tr.d_ff, tr.dtype)
                assert nm.normwise_rel_err(nm.widen(got, tr.dtype), ref.state[s][l]) <= nm.TOL[tr.dtype]
        allv = D.gather_dict(mine)                                # end-of-run gather (§8(e) item 3)
        tot = D.sum_over_ranks(log.census[0] + log.census[1])
        if rank == 0:
            q.put((allv, tot, worst))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_oracle_shards_and_single_process_run():
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allv, tot, worst = q.get(timeout=500)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    tr = _trace()
    log, _, _, single = _serve(tr)
    assert tot == log.census[0] + log.census[1] == tr.n_streams * tr.n_steps
    assert sorted(allv) == sorted(single)                          # every owner on exactly one rank
    assert allv == single, "sharded run differs from the single-process run (versions / payload digests)"

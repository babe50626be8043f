"""BJ configs[4]: 256 streams sharded by owner across G GPUs of one node,
64K context (v0 = 512), L = 4 TTT layers, paper dims, bf16 — the STRONG-scaling form (total
work fixed as G grows; bench.py's torchrun form is weak scaling at 8 streams per GPU).

    python tools/bench_config5.py                                   # G = 1
    python -m torch.distributed.run --nnodes=1 --nproc-per-node G --master-addr 127.0.0.1 \\
        --master-port 29531 tools/bench_config5.py                  # G GPUs, one rank each

Each rank serves its shard π(o) = s mod G (workload.traces.shard) through the serving loop
(NextStep → plan_batch → read_apply / write_commit) with its own pool, planner and W_down
replica; NCCL carries only the barrier, the MAX of per-rank window times and the census sum —
no data-path collective (the path has no exchange step).  One C = 128-step window
after a warm-up window; aggregate tok/s = 256 × 128 / max over ranks of the device time.
The SURVEY §8(d) roofline for the same G (HBM: 51.2 / G GB + 0.2 GB per step) is reported
beside it.  TTT_SAME_DEVICE=1 with TTT_DIST_BACKEND=gloo runs every rank on one GPU (a
code-path check on a 1-GPU box; the pool of 256 / G owners per rank must fit alongside the
others).
"""
from __future__ import annotations

import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench_configs import SEED, WindowInputs  # noqa: E402
from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200 import distributed as D  # noqa: E402
from paper_2605_28053_b200.serving import Engine, Server  # noqa: E402
from workload import rng  # noqa: E402
from workload import traces as T  # noqa: E402

ROOFLINE = {1: 32800.0, 2: 65300.0, 4: 129600.0, 8: 255400.0}   # SURVEY §8(d), tok/s aggregate


def main():
    rank, world, local = D.env_rank()
    backend = os.environ.get("TTT_DIST_BACKEND", "nccl")
    dev = torch.device("cuda", 0 if os.environ.get("TTT_SAME_DEVICE") == "1" else local)
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    coll_dev = dev if backend == "nccl" else None
    tr = T.config5_sharded(n_steps=1 << 30)
    sh = T.shard(tr, world, rank)
    L = tr.n_layers
    W = torch.empty(L, tr.d_model, tr.d_ff, dtype=torch.bfloat16, device=dev)
    for l in range(L):
        capi.gen_uniform(W[l], SEED, rng.T_W_DOWN, 0, l, 0, tr.d_model * tr.d_ff, rng.amp_inv_sqrt(tr.d_ff), True)
    eng = Engine(tr.d_model, tr.d_ff, tr.chunk, L, "bf16", sh.n_streams, W, n_ckpt=0, B=sh.B, w=0, placement=rank)
    src = WindowInputs(sh, dev)
    stream = torch.cuda.current_stream(dev)
    srv = Server(eng, sh, src, stream=stream)
    srv.admit()
    torch.cuda.synchronize(dev)
    del src.d0
    for _ in range(tr.chunk):                       # warm-up window
        srv.step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    c0 = dict(srv.log.census)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(tr.chunk):
        srv.step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = D.max_over_ranks(e0.elapsed_time(e1), coll_dev)
    tokens = D.sum_over_ranks(sum(srv.log.census.values()) - sum(c0.values()), coll_dev)
    writes = D.sum_over_ranks(srv.log.census.get(1, 0) - c0.get(1, 0), coll_dev)
    versions = D.gather_dict({sh.owner(s): capi.tttstate_version(eng.pool, sh.owner(s)) for s in range(sh.n_streams)})
    if rank == 0:
        tok_s = tokens / (ms / 1e3)
        roof = ROOFLINE.get(world)
        print(json.dumps({"config": "5", "scaling": "strong", "G": world, "streams_total": tr.n_streams,
                          "streams_per_rank": sh.n_streams, "layers": L, "window_steps": tr.chunk,
                          "ms_max_over_ranks": ms, "tok_s": tok_s, "tokens": int(tokens), "writes": int(writes),
                          "owners": len(versions), "versions": sorted(set(versions.values())),
                          "roofline_tok_s": roof, "frac_of_roofline": tok_s / roof if roof else None,
                          "ranks_on_one_device": os.environ.get("TTT_SAME_DEVICE") == "1"}), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""NEXT f4 measurement: end-to-end decode tok/s of a full Qwen3-4B-shaped model (synthetic,
random-init) whose 36 MLP down-projections are RW-TTT layers (paper_2605_28053_b200.fullmodel).

    python tools/bench_fullmodel.py [--streams 8] [--ctx 4096] [--steps 128] [--warmup 8]

Setting of the paper's serving rows: 8 streams, 4096-token context,
C_ttt = 128, bf16. The TTT state starts at v0 = ctx / C with random ΔW (the prefill is not
timed; the KV cache holds synthetic K/V). A timed window of 128 decode steps has 127 READ
steps and one boundary WRITE per stream. Also reports the same loop with a static
down-projection (cuBLAS z·W_downᵀ, no TTT state) for the TTT overhead. The non-TTT part of
each layer is replayed from a CUDA graph (one per layer); the TTT layer is a live C-ABI call.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.fullmodel import QWEN3_4B, GraphedDecodeStep, SyntheticDecoder, TTTLayerDriver  # noqa: E402
from paper_2605_28053_b200.serving import Engine  # noqa: E402
from workload import rng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--layers", type=int, default=QWEN3_4B.n_layers)
    a = ap.parse_args()
    shape = QWEN3_4B if a.layers == QWEN3_4B.n_layers else QWEN3_4B.__class__(**{**QWEN3_4B.__dict__,
                                                                                 "n_layers": a.layers})
    dev = torch.device("cuda")
    B, C = a.streams, 128
    model = SyntheticDecoder(shape, B, a.ctx + a.warmup + 2 * a.steps + 8, dev)
    model.fill_context(a.ctx)
    eng = Engine(shape.d_model, shape.d_ff, C, shape.n_layers, "bf16", B, model.w_down, n_ckpt=0, B=B, w=0)
    owners = list(range(1000, 1000 + B))
    d0 = torch.empty(shape.n_layers, shape.d_model, shape.d_ff, dtype=torch.bfloat16, device=dev)
    for o in owners:
        capi.gen_uniform(d0, 0, rng.T_DELTA0, o, 0, 0, d0.numel(), rng.amp_inv_sqrt(shape.d_ff), True)
        capi.tttstate_alloc(eng.pool, o, d0, a.ctx // C)
    del d0
    drv = TTTLayerDriver(eng, owners)
    stream = torch.cuda.current_stream()
    tokens = torch.randint(0, shape.vocab, (B,), device=dev)

    graphed = GraphedDecodeStep(model)

    def ttt_step(tok):                              # harness in CUDA graphs, TTT layers live
        drv.begin_step()
        nxt = graphed.step(tok, drv)
        drv.end_step()
        return nxt.clone()

    def static_step(tok):                           # same harness, dense down-projection (no TTT state)
        return graphed.step(tok, lambda l, z, v, h, out: torch.addmm(h, z, model.w_down[l].t(), out=out)).clone()

    res = {"model": "synthetic Qwen3-4B-shaped (random init)", "streams": B, "ctx": a.ctx, "layers": shape.n_layers,
           "chunk": C, "steps": a.steps}
    for name, fn in (("rw_ttt", ttt_step), ("static_down_proj", static_step)):
        for _ in range(a.warmup):
            tokens = fn(tokens)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        for _ in range(a.steps):
            tokens = fn(tokens)
        host_ms = (time.perf_counter() - t0) * 1e3
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[name] = {"ms_per_step": ms / a.steps, "tok_s": B * a.steps / (ms / 1e3),
                     "host_enqueue_ms_per_step": host_ms / a.steps}
    res["ttt_overhead"] = res["static_down_proj"]["tok_s"] / res["rw_ttt"]["tok_s"]
    res["versions"] = [capi.tttstate_version(eng.pool, o) for o in owners]
    res["paper_context_tok_s"] = 274.61      # RW-TTT full, uniform, P:557 (other GPU: context only)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

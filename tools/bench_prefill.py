"""NEXT f2 measurement: chunk-granular READ (prefill) at paper dims on tcgen05.

    python tools/bench_prefill.py [--layers 4] [--members 8] [--chunks 3]

One chunk = C=128 tokens per member at one version, all layers, then the boundary
WRITE + commit (a whole prefill chunk of the long-context state build).  Reports
READ-chunk TFLOP/s (4·C·d_model·d_ff per member per layer: base + delta products)
against MEASURED_PEAKS.json's bf16 peak, HBM GB/s of the WRITE, and prefill tok/s.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.serving import Engine  # noqa: E402
from workload import rng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--members", type=int, default=8)
    ap.add_argument("--chunks", type=int, default=3)
    ap.add_argument("--d-model", type=int, default=2560)
    ap.add_argument("--d-ff", type=int, default=9728)
    ap.add_argument("--chunk", type=int, default=128)
    a = ap.parse_args()
    dm, dff, L, B, C = a.d_model, a.d_ff, a.layers, a.members, a.chunk
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    dev = torch.device("cuda")
    amp = rng.amp_inv_sqrt(dff)
    W = torch.empty(L, dm, dff, dtype=torch.bfloat16, device=dev)
    capi.gen_uniform(W, 0, rng.T_W_DOWN, 0, 0, 0, W.numel(), amp, True)
    eng = Engine(dm, dff, C, L, "bf16", B, W, n_ckpt=0, B=B)
    owners = list(range(100, 100 + B))
    d0 = torch.empty(L, dm, dff, dtype=torch.bfloat16, device=dev)
    for o in owners:
        capi.gen_uniform(d0, 0, rng.T_DELTA0, o, 0, 0, d0.numel(), amp, True)
        capi.tttstate_alloc(eng.pool, o, d0, 0)
    del d0
    X = torch.empty(L, B, C, dff, dtype=torch.bfloat16, device=dev)
    V = torch.empty(L, B, C, dm, dtype=torch.bfloat16, device=dev)
    Y = torch.empty(L, B, C, dm, dtype=torch.bfloat16, device=dev)
    capi.gen_uniform(X, 0, rng.T_X, 0, 0, 0, X.numel(), 1.0, True)
    capi.gen_uniform(V, 0, rng.T_TGT, 0, 0, 0, V.numel(), 1.0, True)
    g = capi.Group(capi.WRITE, owners)
    s = torch.cuda.current_stream()
    read_ms, write_ms, chunk_ms = [], [], []
    for k in range(a.chunks + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(s)
        for l in range(L):
            capi.read_apply_chunk(eng.pool, g, l, X[l], V[l], Y[l], s)
        ev[1].record(s)
        capi.write_commit(eng.pool, g, 0.01, None, s)
        ev[2].record(s)
        torch.cuda.synchronize()
        if k > 0:                                           # first chunk = warm-up
            read_ms.append(ev[0].elapsed_time(ev[1]) / L)
            write_ms.append(ev[1].elapsed_time(ev[2]) / L)
            chunk_ms.append(ev[0].elapsed_time(ev[2]))
    rmed = sorted(read_ms)[len(read_ms) // 2]
    flops = 4.0 * C * dm * dff * B                          # per layer
    rbytes = dm * dff * 2 * (1 + B) + B * C * (2 * dff + 3 * dm) * 2
    wmed = sorted(write_ms)[len(write_ms) // 2]
    wbytes = B * (2 * dm * dff * 2 + C * (dff + dm) * 2)
    cmed = sorted(chunk_ms)[len(chunk_ms) // 2]
    out = {"read_chunk": {"ms_per_layer": rmed, "TFLOPs": flops / rmed / 1e9,
                          "frac_bf16_peak": flops / rmed / 1e9 / peaks["bf16_tflops"],
                          "GBps": rbytes / rmed / 1e6, "AI_flop_per_byte": flops / rbytes},
           "write": {"ms_per_layer": wmed, "GBps": wbytes / wmed / 1e6, "frac_hbm": wbytes / wmed / 1e6 / peaks["hbm_gbs"]},
           "prefill_tok_per_s_36_layers": B * C / (cmed / L * 36 / 1e3),
           "config": {"members": B, "C": C, "d_model": dm, "d_ff": dff, "layers_timed": L}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

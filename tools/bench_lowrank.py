"""NEXT f1 measurement: low-rank delta TTTState, BJ configs[3] shape (128 streams, R = 16 / 64).

    python tools/bench_lowrank.py [--rank 16] [--layers 4] [--members 128]

Times one decode READ step over L layers (u = A x, tcgen05 base GEMM, Bᵀu) and one boundary
WRITE + commit; reports tok/s for a 128-token window extrapolated to 36 layers and the
HBM bytes of the READ step (W_down once + every A and B once).
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
from paper_2605_28053_b200.serving import Engine  # noqa: E402
from workload import rng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--members", type=int, default=128)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    dm, dff, L, B, R, C = 2560, 9728, a.layers, a.members, a.rank, 128
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    dev = torch.device("cuda")
    W = torch.empty(L, dm, dff, dtype=torch.bfloat16, device=dev)
    capi.gen_uniform(W, 0, rng.T_W_DOWN, 0, 0, 0, W.numel(), rng.amp_inv_sqrt(dff), True)
    eng = Engine(dm, dff, C, L, "bf16", B, W, n_ckpt=0, B=B, backend=capi.LOW_RANK, rank=R)
    owners = list(range(100, 100 + B))
    d0 = torch.empty(L, R * (dff + dm), dtype=torch.bfloat16, device=dev)
    for o in owners:
        capi.gen_uniform(d0, 0, rng.T_LR_A, o, 0, 0, d0.numel(), rng.amp_inv_sqrt(dff), True)
        capi.tttstate_alloc(eng.pool, o, d0, 0)
    X = torch.empty(L, B, dff, dtype=torch.bfloat16, device=dev)
    V = torch.empty(L, B, dm, dtype=torch.bfloat16, device=dev)
    Y = torch.empty(L, B, dm, dtype=torch.bfloat16, device=dev)
    capi.gen_uniform(X, 0, rng.T_X, 0, 0, 0, X.numel(), 1.0, True)
    capi.gen_uniform(V, 0, rng.T_TGT, 0, 0, 0, V.numel(), 1.0, True)
    g = capi.Group(capi.READ, owners, backend=capi.LOW_RANK)
    gw = capi.Group(capi.WRITE, owners, backend=capi.LOW_RANK)
    s = torch.cuda.current_stream()
    ms, host_us = [], []
    for it in range(a.iters + 2):                    # READ steps (tail fills)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        t0 = time.perf_counter()
        for l in range(L):
            capi.read_apply(eng.pool, g, l, X[l], None, V[l], None, Y[l], None, None, s)
        host_us.append((time.perf_counter() - t0) / L * 1e6)
        e1.record(s)
        capi.tttstate_step_done(eng.pool, g)
        torch.cuda.synchronize()
        if it >= 2:
            ms.append(e0.elapsed_time(e1) / L)
    while capi.tttstate_tail_len(eng.pool, owners[0]) < C - 1:
        for l in range(L):
            capi.read_apply(eng.pool, g, l, X[l], None, V[l], None, Y[l], None, None, s)
        capi.tttstate_step_done(eng.pool, g)
    for l in range(L):
        capi.read_apply(eng.pool, gw, l, X[l], None, V[l], None, Y[l], None, None, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    capi.write_commit(eng.pool, gw, eng.eta, None, s)
    e1.record(s)
    torch.cuda.synchronize()
    wms = e0.elapsed_time(e1) / L
    rms = sorted(ms)[len(ms) // 2]
    rbytes = dm * dff * 2 + B * R * (dff + dm) * 2 + B * (2 * dff + 3 * dm) * 2
    window_ms = 36 * (C * rms + wms)
    print(json.dumps({"rank": R, "members": B, "read_ms_per_layer": rms,
                      "host_us_per_read_call": sorted(host_us)[len(host_us) // 2], "read_GBps": rbytes / rms / 1e6,
                      "read_frac_hbm": rbytes / rms / 1e6 / peaks["hbm_gbs"], "write_ms_per_layer": wms,
                      "tok_per_s_window_36_layers": B * C / (window_ms / 1e3)}, indent=1))


if __name__ == "__main__":
    main()

"""NEXT f3 measurement: streaming learner / all-update (C = 1) at paper dims.

    python tools/bench_all_update.py [--layers 4] [--steps 6]

Every decode step is a WRITE (Table 4 "all-update stress").  impl 0 = fused
READ+WRITE pass (read_apply writes ΔW + η·v·xᵀ to the shadow slot, write_commit only
commits); impl 1 = READ kernel then a separate SIMT WRITE pass.  Reports step time,
tok/s extrapolated to 36 layers and HBM GB/s on algorithmic bytes.
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


def run(impl, a):
    dm, dff, L, B = a.d_model, a.d_ff, a.layers, a.members
    dev = torch.device("cuda")
    amp = rng.amp_inv_sqrt(dff)
    W = torch.empty(L, dm, dff, dtype=torch.bfloat16, device=dev)
    capi.gen_uniform(W, 0, rng.T_W_DOWN, 0, 0, 0, W.numel(), amp, True)
    eng = Engine(dm, dff, 1, L, "bf16", B, W, n_ckpt=0, B=B)
    owners = list(range(100, 100 + B))
    d0 = torch.empty(L, dm, dff, dtype=torch.bfloat16, device=dev)
    for o in owners:
        capi.gen_uniform(d0, 0, rng.T_DELTA0, o, 0, 0, d0.numel(), amp, True)
        capi.tttstate_alloc(eng.pool, o, d0, 0)
    del d0
    X = torch.empty(L, B, dff, dtype=torch.bfloat16, device=dev)
    V = torch.empty(L, B, dm, dtype=torch.bfloat16, device=dev)
    Y = torch.empty(L, B, dm, dtype=torch.bfloat16, device=dev)
    capi.gen_uniform(X, 0, rng.T_X, 0, 0, 0, X.numel(), 1.0, True)
    capi.gen_uniform(V, 0, rng.T_TGT, 0, 0, 0, V.numel(), 1.0, True)
    g = capi.Group(capi.WRITE, owners)
    s = torch.cuda.current_stream()
    prev = capi.tttstate_set_write_impl(impl)
    times = []
    try:
        for k in range(a.steps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for l in range(L):
                capi.read_apply(eng.pool, g, l, X[l], None, V[l], None, Y[l], None, None, s)
            capi.write_commit(eng.pool, g, eng.eta, None, s)
            e1.record(s)
            torch.cuda.synchronize()
            if k >= 2:
                times.append(e0.elapsed_time(e1))
    finally:
        capi.tttstate_set_write_impl(prev)
    eng.close()
    ms = sorted(times)[len(times) // 2]
    alg = L * (dm * dff * 2 * (1 + 2 * B))           # W once, each ΔW read + written once
    return {"ms_per_step": ms, "tok_per_s_36_layers": B / (ms / L * 36 / 1e3), "alg_GBps": alg / ms / 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--members", type=int, default=8)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--d-model", type=int, default=2560)
    ap.add_argument("--d-ff", type=int, default=9728)
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    out = {"fused_f3": run(0, a), "separate": run(1, a)}
    for k in out:
        out[k]["frac_hbm_alg"] = out[k]["alg_GBps"] / peaks["hbm_gbs"]
    out["speedup_fused"] = out["separate"]["ms_per_step"] / out["fused_f3"]["ms_per_step"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

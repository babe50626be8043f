"""Phase trace of the one-pass low-rank READ (TTT_LR_TRACE=1): per-CTA %globaltimer stamps at
main kernel entry (after griddepcontrol.wait) and exit, finish kernel entry (after its wait) and exit — for the last launch.

    TTT_LR_TRACE=1 python tools/lr_trace.py [--rank 16] [--members 128]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TTT_LR_TRACE", "1")

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.serving import Engine  # noqa: E402
from workload import rng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--members", type=int, default=128)
    ap.add_argument("--layers", type=int, default=8)
    a = ap.parse_args()
    dm, dff, L, B, R, Cc = 2560, 9728, a.layers, a.members, a.rank, 128
    dev = torch.device("cuda")
    W = torch.empty(L, dm, dff, dtype=torch.bfloat16, device=dev)
    capi.gen_uniform(W, 0, rng.T_W_DOWN, 0, 0, 0, W.numel(), rng.amp_inv_sqrt(dff), True)
    eng = Engine(dm, dff, Cc, L, "bf16", B, W, n_ckpt=0, B=B, backend=capi.LOW_RANK, rank=R)
    owners = list(range(100, 100 + B))
    d0 = torch.empty(L, R * (dff + dm), dtype=torch.bfloat16, device=dev)
    for o in owners:
        capi.gen_uniform(d0, 0, rng.T_LR_A, o, 0, 0, d0.numel(), rng.amp_inv_sqrt(dff), True)
        capi.tttstate_alloc(eng.pool, o, d0, 0)
    X = torch.empty(L, B, dff, dtype=torch.bfloat16, device=dev)
    V = torch.empty(L, B, dm, dtype=torch.bfloat16, device=dev)
    Y = torch.empty(L, B, dm, dtype=torch.bfloat16, device=dev)
    capi.gen_uniform(X, 0, rng.T_X, 0, 0, 0, X.numel(), 1.0, True)
    g = capi.Group(capi.READ, owners, backend=capi.LOW_RANK)
    s = torch.cuda.current_stream()
    f = capi._lib.ttt_debug_lr_trace
    f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    for it in range(2):
        for l in range(L):
            capi.read_apply(eng.pool, g, l, X[l], None, V[l], None, Y[l], None, None, s)
        capi.tttstate_step_done(eng.pool, g)
        torch.cuda.synchronize()
    buf = (C.c_ulonglong * (8 * 4096))()
    assert f(buf, 8 * 4096) == 0
    launches = []
    for k in range(8):
        rows = [tuple(buf[k * 4096 + 4 * c + i] for i in range(4)) for c in range(1024) if buf[k * 4096 + 4 * c]]
        if rows:
            launches.append(rows)
    launches.sort(key=lambda rows: min(r[0] for r in rows))
    t0 = min(r[0] for r in launches[0])
    print(f"R={R} members={B} CTAs={len(launches[0])}; per launch (us from the first): "
          "main entry min / main done med, max / finish entry min / finish exit max")
    for rows in launches:
        def col(i):
            return sorted((r[i] - t0) / 1000 for r in rows if r[i])
        a, b, c, d = col(0), col(1), col(2), col(3)
        print(f"  {a[0]:7.2f}  {b[len(b) // 2]:7.2f} {b[-1]:7.2f}  {c[0]:7.2f}  {d[-1]:7.2f}")
    # single-wave main grid: CTA c runs tile c; tiles (unit, slab) unit-major, W units first
    units = -(-dm // 256) + -(-B * R // 256)
    rows = launches[-1]
    if len(rows) % units == 0:
        ks = len(rows) // units
        nw = -(-dm // 256) * ks
        done = [(r[1] - r[0]) / 1000 for r in rows]
        w, a_ = sorted(done[:nw]), sorted(done[nw:])
        print(f"  last launch: W tiles main {w[len(w) // 2]:.2f} med / {w[-1]:.2f} max us; "
              f"A tiles {a_[len(a_) // 2]:.2f} / {a_[-1]:.2f} (KS={ks})")


if __name__ == "__main__":
    main()

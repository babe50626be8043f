"""Phase timeline of the fused low-rank READ (f1) from per-CTA %globaltimer stamps.

    python tools/lr_print_trace.py [--rank 16] [--members 128]

Runs the kernel with TTT_LR_PRINT=1 (each CTA printf's its stamps) in a child process for a few
decode READ steps over 2 layers and summarises, per launch, the median / max over CTAs of:
entry, after griddepcontrol.wait, last MMA issued, split-K slab written, u = A x done,
Bᵀu done, finish gate passed, exit — in µs from the launch's first CTA entry, and the gap to
the next launch.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2605_28053_b200 import capi
from paper_2605_28053_b200.serving import Engine
from workload import rng
dm, dff, L, B, R, C = 2560, 9728, 2, %d, %d, 128
W = torch.empty(L, dm, dff, dtype=torch.bfloat16, device="cuda")
capi.gen_uniform(W, 0, rng.T_W_DOWN, 0, 0, 0, W.numel(), rng.amp_inv_sqrt(dff), True)
eng = Engine(dm, dff, C, L, "bf16", B, W, n_ckpt=0, B=B, backend=capi.LOW_RANK, rank=R)
owners = list(range(100, 100 + B))
d0 = torch.empty(L, R * (dff + dm), dtype=torch.bfloat16, device="cuda")
for o in owners:
    capi.gen_uniform(d0, 0, rng.T_LR_A, o, 0, 0, d0.numel(), rng.amp_inv_sqrt(dff), True)
    capi.tttstate_alloc(eng.pool, o, d0, 0)
X = torch.empty(L, B, dff, dtype=torch.bfloat16, device="cuda"); capi.gen_uniform(X, 0, rng.T_X, 0, 0, 0, X.numel(), 1.0, True)
V = torch.empty(L, B, dm, dtype=torch.bfloat16, device="cuda"); capi.gen_uniform(V, 0, rng.T_TGT, 0, 0, 0, V.numel(), 1.0, True)
Y = torch.empty(L, B, dm, dtype=torch.bfloat16, device="cuda")
g = capi.Group(capi.READ, owners, backend=capi.LOW_RANK)
for it in range(4):
    for l in range(L):
        capi.read_apply(eng.pool, g, l, X[l], None, V[l], None, Y[l])
    capi.tttstate_step_done(eng.pool, g)
torch.cuda.synchronize()
'''


def n_ctas(rows):
    return max(r[0] for r in rows) + 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--members", type=int, default=128)
    a = ap.parse_args()
    env = dict(os.environ, TTT_LR_PRINT="1")
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, a.members, a.rank)], env=env, capture_output=True,
                         text=True, check=True).stdout
    rows = [list(map(int, ln.split()[1:])) for ln in out.splitlines() if ln.startswith("LRT ")]
    # group into launches: launches run in order and alternate layers; a launch's CTAs all enter
    # before the next launch's (1 CTA per SM, the next grid waits for SMs to free up)
    rows.sort(key=lambda r: r[1])
    launches, cur = [], []
    for r in rows:
        if cur and (r[9] != cur[0][9] or len(cur) == n_ctas(rows)):
            launches.append(cur)
            cur = []
        cur.append(r)
    launches.append(cur)
    names = ["wait", "mma_issued", "slab", "u_done", "bu_done", "gate", "exit"]
    prev_end = None
    for k, ls in enumerate(launches):
        t0 = min(r[1] for r in ls)
        line = [f"launch {k}: {len(ls)} CTAs"]
        if prev_end is not None:
            line.append(f"gap {1e-3 * (t0 - prev_end):.2f}")
        for i, nm in enumerate(names, start=2):
            v = sorted(1e-3 * (r[i] - t0) for r in ls if r[i] > 0)
            if v:
                line.append(f"{nm} {v[len(v) // 2]:.2f}/{v[-1]:.2f}")
        prev_end = max(r[8] for r in ls)
        print("  ".join(line), " (median/max us from first entry)")


if __name__ == "__main__":
    main()

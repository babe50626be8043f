"""Phase timeline of the TMA + tcgen05 decode READ (read_decode_tc.cu) from per-CTA %globaltimer
stamps: run tools/microbench.py with TTT_READ_TC_TRACE=1 in a child, parse the DTC lines and print,
per launch, the median / max over CTAs (µs from the launch's first CTA entry) of: x slice ready,
first row block accumulated, epilogue done, exit — and the gap to the next launch.

    python tools/dtc_trace.py [--layers 4] [--iters 2]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--iters", type=int, default=2)
    a = ap.parse_args()
    env = dict(os.environ, TTT_READ_TC_TRACE="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "microbench.py"), "--layers", str(a.layers),
                          "--iters", str(a.iters)], env=env, capture_output=True, text=True).stdout
    rows = [list(map(int, ln.split()[1:])) for ln in out.splitlines() if ln.startswith("DTC ")]
    rows.sort(key=lambda r: r[1])
    n_cta = max(r[0] for r in rows) + 1
    rows = rows[-2 * a.layers * n_cta:]                  # the last two iterations
    def med(v):
        v = sorted(v)
        return f"{v[len(v) // 2]:.2f} (p10 {v[len(v) // 10]:.2f}, max {v[-1]:.2f})"
    print("per CTA, us:  x_ready - entry", med([1e-3 * (r[2] - r[1]) for r in rows]))
    print("              first row block - x_ready", med([1e-3 * (r[3] - r[2]) for r in rows]))
    print("              epilogue done - x_ready", med([1e-3 * (r[4] - r[2]) for r in rows]))
    print("              exit - epilogue done", med([1e-3 * (r[5] - r[4]) for r in rows]))
    by = {}
    for r in rows:
        by.setdefault(r[0], []).append(1e-3 * (r[4] - r[2]))
    per = sorted((sorted(v)[len(v) // 2], c) for c, v in by.items())
    print("slowest CTAs (median streaming us, cta):", " ".join(f"{t:.1f}@{c}" for t, c in per[-12:]))
    print("fastest CTAs:", " ".join(f"{t:.1f}@{c}" for t, c in per[:6]))
    # launches: CTAs sorted by x_ready; a launch's x_ready stamps cluster within a few us
    xr = sorted(r[2] for r in rows)
    starts = [xr[i] for i in range(0, len(xr), n_cta)]
    ends = sorted(r[5] for r in rows)
    spans = [1e-3 * (ends[min(len(ends) - 1, i + n_cta - 1)] - xr[i]) for i in range(0, len(xr) - n_cta + 1, n_cta)]
    print("launch span (first x_ready -> last exit), us:", " ".join(f"{x:.1f}" for x in spans))
    # launches = 148 consecutive rows by x_ready; gap = this launch's first wait release - the
    # previous launch's last exit; staging = x_ready - wait release (per CTA median)
    byx = sorted(rows, key=lambda r: r[2])
    ls = [byx[i:i + n_cta] for i in range(0, len(byx) - n_cta + 1, n_cta)]
    for k in range(1, len(ls)):
        last_exit = max(r[5] for r in ls[k - 1])
        rel = sorted(r[7] for r in ls[k] if len(r) > 7)
        if rel:
            stg = sorted(r[2] - r[7] for r in ls[k])
            print(f"launch {k}: wait release {1e-3 * (rel[0] - last_exit):.2f} .. {1e-3 * (rel[-1] - last_exit):.2f} us "
                  f"after the previous last exit; x staging median {1e-3 * stg[len(stg) // 2]:.2f} us; "
                  f"previous exits spread {1e-3 * (last_exit - min(r[5] for r in ls[k - 1])):.2f} us")


if __name__ == "__main__":
    main()

"""SURVEY §8(d) per-config throughput at full size (BASELINE.json configs[2..4]) through the
serving loop (Alg. 1: NextStep → plan_batch → read_apply / write_commit, controls, App. H
fallback) on one B200.

    python tools/bench_configs.py [--configs 3,4r16,4r64,5] [--windows 1]

* config 3: 64 streams, L = 12, paper dims, bursty offsets, injected write failures on 1/16
  of the streams, speculative snapshot + rollback on 1/8, B = 64, wait budget w = 0 ("3") or
  4 / 16 ("3w4", "3w16": a WRITE bucket below B holds its members up to w steps — Eq. 4 —
  so fewer tokens per step by design);
* config 4: low-rank R = 16 / 64, 128 streams, L = 36, a branch lineage forked at every
  boundary, speculative WRITE accepted with p = 0.75 else rolled back, branch released;
* config 5: 256 streams, L = 4, one GPU (the G = 1 base of the scaling table; bench.py under
  torchrun runs the sharded form).

A window is C = 128 decode steps per stream (every stream crosses one boundary); inputs are
synthesised in HBM for one window and reused (rows (p mod C)·S + s). Reports device-time
tok/s (CUDA events around the window), the census, fallbacks / device failures, and the
SURVEY §8(d) HBM roofline prediction for the same config.
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
from paper_2605_28053_b200.serving import Engine, InputSource, Server, StepIO  # noqa: E402
from workload import rng  # noqa: E402
from workload import traces as T  # noqa: E402

SEED = 0
# SURVEY §8(d) per-config roofline predictions (tok/s, one GPU)
ROOFLINE = {"3": 10600.0, "3w4": 10600.0, "3w16": 10600.0, "4r16": 226000.0, "4r64": 92000.0, "5": 32800.0}


class WindowInputs(InputSource):
    """One window of seeded inputs resident in HBM, X [L][C·S][d_ff], V/Y [L][C·S][d_model]."""

    def __init__(self, tr, dev):
        self.tr, self.dev = tr, dev
        L, S, C = tr.n_layers, tr.n_streams, tr.chunk
        self.X = torch.empty(L, C * S, tr.d_ff, dtype=torch.bfloat16, device=dev)
        self.V = torch.empty(L, C * S, tr.d_model, dtype=torch.bfloat16, device=dev)
        self.Y = torch.empty(L, C * S, tr.d_model, dtype=torch.bfloat16, device=dev)
        for l in range(L):
            capi.gen_uniform(self.X[l], SEED, rng.T_X, tr.owner_base, l, 0, self.X[l].numel(), 1.0, True)
            capi.gen_uniform(self.V[l], SEED, rng.T_TGT, tr.owner_base, l, 0, self.V[l].numel(), 1.0, True)
        if tr.backend == 1:
            self.d0 = torch.empty(L, tr.rank * (tr.d_ff + tr.d_model), dtype=torch.bfloat16, device=dev)
        else:
            self.d0 = torch.empty(L, tr.d_model, tr.d_ff, dtype=torch.bfloat16, device=dev)

    def init_delta(self, s):
        tr = self.tr
        for l in range(tr.n_layers):
            capi.gen_uniform(self.d0[l], SEED, rng.T_LR_A if tr.backend == 1 else rng.T_DELTA0, tr.owner(s), l, 0,
                             self.d0[l].numel(), rng.amp_inv_sqrt(tr.d_ff), True)
        return self.d0

    def tail_prefill(self, s):
        tr = self.tr
        n = tr.offset(s)
        if not n:
            return None
        Z = torch.empty(tr.n_layers, n, tr.d_ff, dtype=torch.bfloat16, device=self.dev)
        V = torch.empty(tr.n_layers, n, tr.d_model, dtype=torch.bfloat16, device=self.dev)
        capi.gen_uniform(Z, SEED, rng.T_X, tr.owner(s), 0, -n, Z.numel(), 1.0, True)
        capi.gen_uniform(V, SEED, rng.T_TGT, tr.owner(s), 0, -n, V.numel(), 1.0, True)
        return n, Z, V

    def group_io(self, l, ss, ps):
        S, C = self.tr.n_streams, self.tr.chunk
        key = (tuple(ss), tuple(ps))
        if key != getattr(self, "_key", None):     # one row map per step, reused by every layer
            self._key, self._rows = key, capi.rows_array([(p % C) * S + s for s, p in zip(ss, ps)])
        rows = self._rows
        return self.X[l], rows, self.V[l], rows, self.Y[l], rows

    def step_io(self, ss, ps):
        S, C, tr = self.tr.n_streams, self.tr.chunk, self.tr
        rows = [(p % C) * S + s for s, p in zip(ss, ps)]
        return StepIO(self.X, C * S * tr.d_ff, self.V, C * S * tr.d_model, self.Y, C * S * tr.d_model, rows, C * S)


def trace_of(name: str, warmup: int = 1):
    if name.startswith("3"):                       # "3" (w = 0) or "3w4", "3w16": bounded wait w
        # failures / snapshots / rollbacks in the first timed window (after `warmup` windows)
        return T.config3_interleaved(n_steps=1 << 30, w=int(name[2:]) if "w" in name else 0, control_chunk=warmup)
    if name.startswith("4r"):
        return T.config4_lowrank(n_steps=1 << 16, rank=int(name[2:]))
    if name == "5":
        return T.config5_sharded(n_steps=1 << 30)
    raise ValueError(name)


def sampled_parity(srv, eng, tr, src, W):
    """The oracle's READ (oracle/numerics.apply_read, oracle/lowrank.apply_read; fp64) on the last
    decode step of the timed window for streams {0, S-1} x layers {0, L-1}, at the payload version
    that step read: the committed slot, or the slot the step's own commit retired when that step
    was the stream's WRITE (reading xvii).  Normwise error against BJ's 2e-2 bound."""
    import numpy as np

    from oracle import lowrank as olr
    from oracle import numerics as nm

    capi.tttstate_sync(eng.pool)
    worst, n = 0.0, 0
    E = tr.rank * (tr.d_ff + tr.d_model) if tr.backend == 1 else tr.d_model * tr.d_ff
    for s in (0, tr.n_streams - 1):
        p = srv.pos[s] - 1
        was_write = (p + tr.offset(s)) % tr.chunk == tr.chunk - 1
        dsel = capi.tttstate_read_slot_raw(eng.pool, tr.owner(s), -1, 0, 1, E, "bf16")
        slots = [capi.tttstate_read_slot_raw(eng.pool, tr.owner(s), w, 0, 1, E, "bf16") for w in (0, 1)]
        active = 0 if np.array_equal(slots[0], dsel) and not np.array_equal(slots[1], dsel) else 1
        which = 1 - active if was_write else active
        row = (p % tr.chunk) * tr.n_streams + s
        for l in sorted({0, tr.n_layers - 1}):
            pay = nm.widen(capi.tttstate_read_slot_raw(eng.pool, tr.owner(s), which, l, 1, E, "bf16")[0], "bf16")
            Wl = nm.widen(W[l].view(torch.int16).cpu().numpy().view(np.uint16), "bf16")
            x = nm.widen(src.X[l, row].view(torch.int16).cpu().numpy().view(np.uint16), "bf16")
            y = nm.widen(src.Y[l, row].view(torch.int16).cpu().numpy().view(np.uint16), "bf16")
            if tr.backend == 1:
                A = pay[: tr.rank * tr.d_ff].reshape(tr.rank, tr.d_ff)
                B = pay[tr.rank * tr.d_ff:].reshape(tr.rank, tr.d_model)
                ref = olr.apply_read(Wl, A, B, x)
            else:
                ref = nm.apply_read(Wl, pay.reshape(tr.d_model, tr.d_ff), x)
            worst = max(worst, nm.normwise_rel_err(y, ref))
            n += 1
    return {"samples": n, "max_normwise_err": worst, "tol": nm.TOL["bf16"], "ok": bool(worst <= nm.TOL["bf16"])}


def run(name: str, windows: int, warmup: int):
    dev = torch.device("cuda")
    tr = trace_of(name, warmup)
    L = tr.n_layers
    W = torch.empty(L, tr.d_model, tr.d_ff, dtype=torch.bfloat16, device=dev)
    for l in range(L):
        capi.gen_uniform(W[l], SEED, rng.T_W_DOWN, 0, l, 0, tr.d_model * tr.d_ff, rng.amp_inv_sqrt(tr.d_ff), True)
    branches = 2 if tr.backend == 1 else 0          # live fork lineages per stream (reading xix)
    n_ckpt = tr.n_streams if tr.controls else 0
    eng = Engine(tr.d_model, tr.d_ff, tr.chunk, L, "bf16", tr.n_streams * (1 + branches), W, n_ckpt=n_ckpt,
                 B=tr.B, w=tr.w, backend=tr.backend, rank=tr.rank)
    src = WindowInputs(tr, dev)
    stream = torch.cuda.current_stream(dev)
    srv = Server(eng, tr, src, stream=stream)
    srv.admit()
    torch.cuda.synchronize(dev)
    for _ in range(warmup * tr.chunk):
        srv.step()
    torch.cuda.synchronize(dev)
    srv.drain()
    census0 = dict(srv.log.census)
    fb0, df0 = srv.log.fallbacks, srv.log.device_failures
    rb0 = srv.log.rollbacks
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(windows * tr.chunk):
        srv.step()
    e1.record(stream)
    t_enq = time.perf_counter() - t0
    torch.cuda.synchronize(dev)
    t_wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    srv.drain()                                    # confirm the window's commits (device refusals)
    tokens = sum(srv.log.census.values()) - sum(census0.values())
    out = {"config": name, "trace": tr.name, "streams": tr.n_streams, "layers": L, "rank": tr.rank or None,
           "B": tr.B, "w": tr.w, "window_steps": windows * tr.chunk, "ms": ms, "tok_s": tokens / (ms / 1e3),
           "census": {"READ": srv.log.census[0] - census0.get(0, 0), "WRITE": srv.log.census[1] - census0.get(1, 0)},
           "fallbacks": srv.log.fallbacks - fb0, "device_failures": srv.log.device_failures - df0,
           "rollbacks": srv.log.rollbacks - rb0,
           "roofline_tok_s": ROOFLINE.get(name),
           "host_enqueue_ms_per_step": 1e3 * t_enq / (windows * tr.chunk), "device_ms_per_step": ms / (windows * tr.chunk),
           "host_wall_over_device": 1e3 * t_wall / ms}
    out["frac_of_roofline"] = out["tok_s"] / out["roofline_tok_s"] if out["roofline_tok_s"] else None
    out["parity"] = sampled_parity(srv, eng, tr, src, W)
    assert out["parity"]["ok"], out["parity"]
    eng.close()
    del src, W, eng
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,3w4,4r16,4r64,5")
    ap.add_argument("--windows", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args()
    res = [run(c, a.windows, a.warmup) for c in a.configs.split(",")]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

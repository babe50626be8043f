"""Synthetic decode traces (inputs only; no method arithmetic).

A trace fixes *what the user does*: which streams decode how many tokens,
their seeded inputs, their starting state, and the control operations
(snapshot / rollback / injected write failure) keyed by ``(stream, pos)``.
Whether a decode step is a READ or a WRITE, how steps are grouped, and what
they compute is the method's business and is derived independently by the
oracle and by the CUDA path.

Shapes follow SURVEY.md §8(d) / BASELINE.json configs; the recipe is in
DESIGN.md §"Input recipe".
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import rng

READ, WRITE = 0, 1
MODE_SERIAL, MODE_PHASE, MODE_FULL = 0, 1, 2


@dataclass
class Trace:
    name: str
    n_streams: int
    n_layers: int
    d_model: int
    d_ff: int
    chunk: int
    n_steps: int                 # decode positions p = 0 .. n_steps-1 per stream
    dtype: str = "bf16"          # storage + operand dtype: "fp32" | "bf16"
    seed: int = 0
    eta: float = float(np.float32(0.01))   # fp32 value (reading iv)
    v0: int = 0                  # starting committed version (ctx / C for long-context starts)
    delta0: str = "zero"         # "zero" | "rng"
    offsets: tuple = ()          # per-stream initial tail fill (bursty: U[0, C))
    controls: dict = field(default_factory=dict)   # (stream, pos) -> list of "snapshot"|"rollback"|"fail"
    B: int = 8                   # planner target batch
    w: int = 0                   # planner wait budget (decode steps)
    mode: int = MODE_FULL
    rule: int = 0                # 0: chunk sum of outer products (reading i); 1: SPEC mean rule
    owner_base: int = 1000       # owner id of stream s is owner_base + s
    backend: int = 0             # τ: 0 fast weights (ΔW), 1 low-rank delta (A, B) — NEXT f1
    rank: int = 0                # R for the low-rank backend

    def replace(self, **kw) -> "Trace":
        return dataclasses.replace(self, **kw)

    # ---- amplitudes (fp32 values handed to both sides) --------------------
    @property
    def amp_w(self) -> float:
        return rng.amp_inv_sqrt(self.d_ff)

    def owner(self, s: int) -> int:
        return self.owner_base + s

    def offset(self, s: int) -> int:
        return int(self.offsets[s]) if self.offsets else 0

    # ---- operands, as the device sees them (bf16 bits or fp32) -----------
    def w_down(self, l: int) -> np.ndarray:
        return rng.gen(self.seed, rng.T_W_DOWN, 0, l, 0, (self.d_model, self.d_ff), self.amp_w, self.dtype)

    def delta0_of(self, s: int, l: int):
        """Initial payload of layer l: ΔW_0, or (A_0, B_0) for the low-rank backend."""
        if self.delta0 == "zero":
            return None
        if self.backend == 1:
            return (rng.gen(self.seed, rng.T_LR_A, self.owner(s), l, 0, (self.rank, self.d_ff), self.amp_w, self.dtype),
                    rng.gen(self.seed, rng.T_LR_B, self.owner(s), l, 0, (self.rank, self.d_model),
                            rng.amp_inv_sqrt(self.rank), self.dtype))
        return rng.gen(self.seed, rng.T_DELTA0, self.owner(s), l, 0, (self.d_model, self.d_ff), self.amp_w, self.dtype)

    def branch_owner(self, s: int, k: int) -> int:
        """Owner id of stream s's k-th forked branch lineage."""
        return self.owner(s) + 1_000_000 * (k + 1)

    def x(self, s: int, p: int, l: int) -> np.ndarray:
        """READ input z for stream s at position p, layer l (p < 0: pre-filled tail)."""
        return rng.gen(self.seed, rng.T_X, self.owner(s), l, p, (self.d_ff,), 1.0, self.dtype)

    def tgt(self, s: int, p: int, l: int) -> np.ndarray:
        """Update target v for stream s at position p, layer l (reading iii).  A "poison"
        control at (s, p) makes element 0 +inf (an input fault: the chunk's candidate is then
        not finite, so its WRITE fails on the device — DESIGN.md reading xx)."""
        v = rng.gen(self.seed, rng.T_TGT, self.owner(s), l, p, (self.d_model,), 1.0, self.dtype)
        if "poison" in self.controls_at(s, p):
            v = v.copy()
            v[0] = 0x7F80 if self.dtype == "bf16" else np.float32(np.inf)
        return v

    def controls_at(self, s: int, p: int):
        return self.controls.get((s, p), ())

    def tokens(self) -> int:
        return self.n_streams * self.n_steps


def bursty_offsets(n_streams: int, chunk: int, seed: int) -> tuple:
    """Per-stream initial tail offsets ~ U[0, C) (reading xv)."""
    u = rng.raw_u24(seed, 99, 0, 0, 0, n_streams) + (1 << 23)
    return tuple(int(x) % chunk for x in u)


# --------------------------------------------------------------------------
# BASELINE.json configs as traces (SURVEY.md §8(d) per-config plan)
# --------------------------------------------------------------------------
def config1_tiny(seed: int = 0) -> Trace:
    """BJ configs[0]: 2 streams, 1 layer, 64/256, C=4, 16 steps, fp32, one rollback.

    s1 snapshots before its p=7 write (v=1), commits v=2, rolls back before p=8
    (v=1, tail cleared); s0's p=11 write gets one injected failure (group
    atomic: s1's p=11 write fails with it); both retry as singletons.
    Expected final versions (4, 3).
    """
    return Trace("config1_tiny", n_streams=2, n_layers=1, d_model=64, d_ff=256, chunk=4,
                 n_steps=16, dtype="fp32", seed=seed, B=2, w=0,
                 controls={(1, 7): ["snapshot"], (1, 8): ["rollback"], (0, 11): ["fail"]})


def config2_paper(seed: int = 0, n_steps: int = 512, n_layers: int = 36) -> Trace:
    """BJ configs[1]: 8 streams, Qwen3-4B dims, 36 layers, bf16, 32K ctx (v0=256), uniform."""
    return Trace("config2_paper", n_streams=8, n_layers=n_layers, d_model=2560, d_ff=9728, chunk=128,
                 n_steps=n_steps, dtype="bf16", seed=seed, v0=256, delta0="rng", B=8, w=0)


def config3_interleaved(seed: int = 0, n_steps: int = 512, n_layers: int = 12, w: int = 4,
                        d_model: int = 2560, d_ff: int = 9728, chunk: int = 128, control_chunk: int = 0) -> Trace:
    """BJ configs[2]: 64 streams, L=12 (memory), bursty offsets, injected write
    failures on 1/16 of the streams' boundary in chunk `control_chunk`, speculative snapshot +
    rollback on 1/8 (control_chunk = 1 puts them inside a timed window after one warm-up window)."""
    offs = bursty_offsets(64, chunk, seed)
    ctl = {}
    base = control_chunk * chunk
    for s in range(0, 64, 16):                     # injected write failures
        ctl.setdefault((s, base + chunk - 1 - offs[s]), []).append("fail")
    for s in range(3, 64, 8):                      # speculative snapshot + rollback
        p = base + chunk - 1 - offs[s]
        ctl.setdefault((s, p), []).append("snapshot")
        ctl.setdefault((s, p + 1), []).append("rollback")
    return Trace("config3_interleaved", n_streams=64, n_layers=n_layers, d_model=d_model, d_ff=d_ff,
                 chunk=chunk, n_steps=n_steps, dtype="bf16", seed=seed, v0=0, delta0="rng",
                 offsets=offs, controls=ctl, B=64, w=w)


def config5_sharded(seed: int = 0, n_steps: int = 512, n_layers: int = 4, d_model: int = 2560,
                    d_ff: int = 9728, chunk: int = 128, n_streams: int = 256) -> Trace:
    """BJ configs[4]: 256 streams sharded by owner over G GPUs, 64K context (v0 = 512), uniform."""
    return Trace("config5_sharded", n_streams=n_streams, n_layers=n_layers, d_model=d_model, d_ff=d_ff,
                 chunk=chunk, n_steps=n_steps, dtype="bf16", seed=seed, v0=512, delta0="rng", B=n_streams, w=0)


def config4_lowrank(seed: int = 0, n_steps: int = 512, n_layers: int = 36, rank: int = 16,
                    d_model: int = 2560, d_ff: int = 9728, chunk: int = 128, n_streams: int = 128,
                    accept_p: float = 0.75, offset: int = 0) -> Trace:
    """BJ configs[3]: low-rank delta TTTState (R = 16 or 64), 128 streams, speculative branch
    versions: at every boundary each stream forks a branch lineage and snapshots; the
    speculative WRITE is accepted with p = 0.75 (seeded) or rolled back; the previous
    boundary's branch is released (reading xix)."""
    ctl = {}
    u = rng.raw_u24(seed, 98, 0, 0, 0, n_streams * (n_steps // chunk + 1)) + (1 << 23)
    k = 0
    for s in range(n_streams):
        for b, p in enumerate(range(chunk - 1 - offset, n_steps, chunk)):
            ops = ctl.setdefault((s, p), [])
            if b > 0:
                ops.append("release")
            ops += ["fork", "snapshot"]
            if u[k] / float(1 << 24) >= accept_p and p + 1 < n_steps:
                ctl.setdefault((s, p + 1), []).append("rollback")
            k += 1
    return Trace("config4_lowrank", n_streams=n_streams, n_layers=n_layers, d_model=d_model, d_ff=d_ff,
                 chunk=chunk, n_steps=n_steps, dtype="bf16", seed=seed, v0=0, delta0="rng", controls=ctl,
                 B=n_streams, w=0, backend=1, rank=rank, offsets=(offset,) * n_streams if offset else ())


def shard(tr: Trace, world: int, rank: int) -> Trace:
    """The streams placed on `rank` (π(o) = s mod world) as a trace of their own; owner ids and
    inputs are unchanged because streams keep their global index via owner_base + s."""
    mine = [s for s in range(tr.n_streams) if s % world == rank]
    return ShardTrace(tr, mine)


class ShardTrace(Trace):
    """A Trace restricted to a subset of the streams (local index k -> global stream mine[k])."""

    def __init__(self, base: Trace, mine):
        import dataclasses as _dc
        fields = {f.name: getattr(base, f.name) for f in _dc.fields(base)}
        fields["n_streams"] = len(mine)
        fields["B"] = min(base.B, len(mine))
        fields["offsets"] = tuple(base.offset(s) for s in mine) if base.offsets else ()
        fields["controls"] = {(mine.index(s), p): ops for (s, p), ops in base.controls.items() if s in mine}
        super().__init__(**fields)
        self.base, self.mine = base, list(mine)

    def owner(self, s):
        return self.base.owner(self.mine[s])

    def delta0_of(self, s, l):
        return self.base.delta0_of(self.mine[s], l)

    def x(self, s, p, l):
        return self.base.x(self.mine[s], p, l)

    def tgt(self, s, p, l):
        return self.base.tgt(self.mine[s], p, l)


def uniform_small(seed=0, n_streams=8, n_layers=2, d_model=128, d_ff=320, chunk=8, n_steps=24,
                  dtype="bf16", **kw) -> Trace:
    """Reduced-dims uniform trace for parity tests (several tiles + a ragged tail)."""
    return Trace("uniform_small", n_streams=n_streams, n_layers=n_layers, d_model=d_model, d_ff=d_ff,
                 chunk=chunk, n_steps=n_steps, dtype=dtype, seed=seed, B=n_streams, **kw)

"""Oracle owner-indexed state table: versions, tails, commit, snapshot, rollback, fork.

TEST INFRASTRUCTURE ONLY (see oracle/numerics.py header).

Follows the paper's serving contract step by step:
  * ownership: Read(r,x,s^v) -> (y,s^v); Write(r,x,u,s^v) -> (y,s^{v+1})
  * event e=(r,τ,σ,ρ,v) per request (Eq. 2); ρ=WRITE on the step whose
    token completes the chunk (SURVEY.md §8(c) reading ii)
  * ApplyState keeps the version; TailBufferUpdate appends, no bump (Table 3)
  * BoundaryUpdate computes a dirty candidate from committed v and evidence
  * Commit publishes only after the WRITE group succeeds; the version counter
    changes here; group-atomic (reading vi)
  * snapshot c_r^v <- s_r^v before speculative writes; rollback
    restores slot and version, clears the tail (reading vii) and keeps
    the checkpoint; fork copies committed state only (reading viii)
State per owner is held in float64 (values exactly representable in σ.dtype).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import lowrank as lr
from . import numerics as nm

READ, WRITE = 0, 1


def _copy(S):
    """Deep copy of one owner's payload (per layer: ΔW array, or (A, B) for low rank)."""
    return [tuple(np.array(a, copy=True) for a in x) if isinstance(x, tuple) else x.copy() for x in S]


def _finite(x) -> bool:
    return all(np.all(np.isfinite(a)) for a in x) if isinstance(x, tuple) else bool(np.all(np.isfinite(x)))


class ContractError(Exception):
    """A request violating the serving contract (mirrors the C-ABI error codes)."""

    def __init__(self, code: str, msg: str = ""):
        super().__init__(f"{code}: {msg}")
        self.code = code


@dataclass
class Owner:
    v: int
    S: list                       # per layer ΔW (float64 [d_model, d_ff])
    ckpt: tuple | None = None     # (v, [S copies])
    tail_z: list = field(default_factory=list)   # per entry: [per layer z]
    tail_v: list = field(default_factory=list)   # per entry: [per layer v]
    tail_p: list = field(default_factory=list)


class StateTable:
    def __init__(self, n_layers: int, d_model: int, d_ff: int, chunk: int, dtype: str,
                 w_down: list, eta: float, rule: int = 0, backend: int = 0, rank: int = 0):
        self.L, self.dm, self.dff, self.C = n_layers, d_model, d_ff, chunk
        self.dtype, self.eta, self.rule = dtype, float(eta), rule
        self.backend, self.rank = backend, rank          # τ: 0 fast weights, 1 low-rank delta (NEXT f1)
        self.W = w_down                      # per layer float64 (identity for rule 1)
        self.owners: dict[int, Owner] = {}

    # ---- registration ----------------------------------------------------
    def alloc(self, r: int, init: list | None = None, v0: int = 0) -> int:
        """register -> v=0, or given init bytes with v0 (reading v)."""
        if r in self.owners:
            raise ContractError("DUPLICATE_OWNER", str(r))
        if self.backend == 1:
            S = [(np.zeros((self.rank, self.dff)), np.zeros((self.rank, self.dm))) if init is None else
                 (np.array(init[l][0], dtype=np.float64), np.array(init[l][1], dtype=np.float64))
                 for l in range(self.L)]
        else:
            S = [np.zeros((self.dm, self.dff)) if init is None else np.array(init[l], dtype=np.float64)
                 for l in range(self.L)]
        self.owners[r] = Owner(v=v0, S=S)
        return v0

    def free(self, r: int):
        self._get(r)
        del self.owners[r]

    def _get(self, r: int) -> Owner:
        if r not in self.owners:
            raise ContractError("UNKNOWN_OWNER", str(r))
        return self.owners[r]

    def version(self, r: int) -> int:
        return self._get(r).v

    def tail_len(self, r: int) -> int:
        return len(self._get(r).tail_p)

    # ---- a1: NextStep (Eq. 2) --------------------------------------------
    def next_effect(self, r: int) -> int:
        """ρ = WRITE iff this step's token completes the chunk (reading ii)."""
        return WRITE if self.tail_len(r) == self.C - 1 else READ

    # ---- a3 + a4: ApplyState + TailBufferUpdate --------------------------
    def apply(self, r: int, p: int, zs: list, vs: list) -> list:
        """Per layer y = (W + ΔW_v) z with the committed version, then append (z, v)."""
        o = self._get(r)
        if len(o.tail_p) >= self.C:
            raise ContractError("TAIL_FULL", str(r))
        if self.backend == 1:
            ys = [lr.apply_read(self.W[l], o.S[l][0], o.S[l][1], zs[l]) for l in range(self.L)]
        else:
            ys = [nm.apply_read(self.W[l], o.S[l], zs[l], self.rule) for l in range(self.L)]
        o.tail_z.append(list(zs))
        o.tail_v.append(list(vs))
        o.tail_p.append(p)
        return ys

    # ---- a5 + a6: BoundaryUpdate + group-atomic Commit -------------------
    def write_group(self, members: list, fail: bool = False) -> list:
        """Compute every member's candidate from its committed v; commit all or none.

        Returns the new versions.  On failure nothing changes (v, ΔW and tail
        intact) and ContractError("WRITE_FAILED") is raised.
        """
        if len(set(members)) != len(members):
            raise ContractError("OWNER_COLLISION", str(members))
        for r in members:
            if self.tail_len(r) != self.C:
                raise ContractError("TAIL_NOT_FULL", str(r))
        cands = {}
        for r in members:
            o = self.owners[r]
            cands[r] = []
            for l in range(self.L):
                Z = np.stack([e[l] for e in o.tail_z])     # [C, d_ff]
                V = np.stack([e[l] for e in o.tail_v])     # [C, d_model]
                if self.backend == 1:
                    cands[r].append(lr.boundary_update(o.S[l][0], o.S[l][1], Z, self.eta, self.dtype))
                else:
                    cands[r].append(nm.boundary_update(o.S[l], Z, V, self.eta, self.dtype, self.rule))
        if fail or any(not all(_finite(c) for c in cands[r]) for r in members):
            raise ContractError("WRITE_FAILED", str(members))
        out = []
        for r in members:
            o = self.owners[r]
            o.S = cands[r]
            o.v += 1
            o.tail_z, o.tail_v, o.tail_p = [], [], []
            out.append(o.v)
        return out

    # ---- a7: control ------------------------------------------------------
    def snapshot(self, r: int):
        """c_r^v <- s_r^v; latest wins."""
        o = self._get(r)
        o.ckpt = (o.v, _copy(o.S))

    def rollback(self, r: int) -> int:
        """Restore the checkpointed slot and version; clear tail (reading vii)."""
        o = self._get(r)
        if o.ckpt is None:
            raise ContractError("NO_CHECKPOINT", str(r))
        o.v = o.ckpt[0]
        o.S = _copy(o.ckpt[1])
        o.tail_z, o.tail_v, o.tail_p = [], [], []
        return o.v

    def fork(self, src: int, dst: int) -> int:
        """New owner/version lineage: committed state, same v, empty tail."""
        o = self._get(src)
        if dst in self.owners:
            raise ContractError("DUPLICATE_OWNER", str(dst))
        self.owners[dst] = Owner(v=o.v, S=_copy(o.S))
        return o.v

    def drop_chunk(self, r: int):
        """A WRITE that failed for good (its singleton retry failed too: a non-finite candidate
        fails the same way every time): v and ΔW stay, the chunk's evidence is discarded
        (tail cleared, as rollback does — reading vii; reading xx)."""
        o = self._get(r)
        o.tail_z, o.tail_v, o.tail_p = [], [], []

    def prefill_tail(self, r: int, zs_list: list, vs_list: list, ps: list):
        """Seed a partially-filled tail (bursty starts, reading xv)."""
        o = self._get(r)
        for zs, vs, p in zip(zs_list, vs_list, ps):
            o.tail_z.append(list(zs))
            o.tail_v.append(list(vs))
            o.tail_p.append(p)

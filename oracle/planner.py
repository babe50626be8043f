"""Oracle TTT-aware batch planner (plain Python).

TEST INFRASTRUCTURE ONLY (see oracle/numerics.py header).

Follows §4.3 and Eq. 3 / Eq. 4 in the paper's order:
  1. for each ready transition e_i compute κ_i = (ρ_i, τ_i, σ_i, π_i)
  2. check v_i against the committed V(r_i); a mismatch is rejected to a
     revalidation list, never issued (reading x)
  3. requests with different keys are never co-issued
  4. per key: emit a group at target batch size B, or after waiting at most
     w decode steps issue the current legal prefix
  5. μ is injective: one pending transition per owner
Readings: the B oldest by (ready_step, owner id) are taken from an over-full
bucket and the wait timer runs from the oldest member (reading ix).  Modes:
serial = singleton groups; phase grouping = only READ keys batch; full = both
(Table 4 rows P:554-557).
"""
from __future__ import annotations

from dataclasses import dataclass

READ, WRITE = 0, 1
MODE_SERIAL, MODE_PHASE, MODE_FULL = 0, 1, 2


@dataclass(frozen=True)
class Event:
    owner: int
    effect: int          # ρ
    backend: int         # τ
    shape_id: int        # σ
    placement: int       # π
    version: int         # expected v_i
    ready_step: int


@dataclass
class Group:
    effect: int
    backend: int
    shape_id: int
    placement: int
    owners: list         # μ: batch slot b -> owner
    issue_step: int
    ready_steps: list


class OraclePlanner:
    def __init__(self, B: int, w: int, mode: int = MODE_FULL):
        assert B >= 1 and w >= 0
        self.B, self.w, self.mode = B, w, mode
        self.buckets: dict[tuple, list[Event]] = {}

    def pending_owners(self) -> set:
        return {e.owner for b in self.buckets.values() for e in b}

    def cap(self, effect: int) -> int:
        if self.mode == MODE_SERIAL or (self.mode == MODE_PHASE and effect == WRITE):
            return 1
        return self.B

    def plan(self, events: list, clock: int, V) -> tuple[list, list]:
        """Return (groups, rejected events).  V(owner) -> committed version or None."""
        rejected = []
        pend = self.pending_owners()
        for e in events:
            if V(e.owner) is None or e.version != V(e.owner):
                rejected.append(e)                        # step 2
            elif e.owner in pend:
                rejected.append(e)                        # step 5 (μ injective)
            else:
                key = (e.effect, e.backend, e.shape_id, e.placement)   # step 1
                self.buckets.setdefault(key, []).append(e)
                pend.add(e.owner)
        # pending events whose owner version moved (e.g. rollback) are stale
        for key in list(self.buckets):
            keep = []
            for e in self.buckets[key]:
                (keep if V(e.owner) == e.version else rejected).append(e)
            self.buckets[key] = keep
        groups = []
        for key in sorted(self.buckets):                  # step 3: one key per group
            b = sorted(self.buckets[key], key=lambda e: (e.ready_step, e.owner))
            cap = self.cap(key[0])
            while len(b) >= cap:                          # step 4: target batch size
                groups.append(self._group(key, b[:cap], clock))
                b = b[cap:]
            if b and clock - b[0].ready_step >= self.w:   # step 4: wait budget expired
                groups.append(self._group(key, b, clock))
                b = []
            self.buckets[key] = b
        self.buckets = {k: v for k, v in self.buckets.items() if v}
        return groups, rejected

    @staticmethod
    def _group(key, evs, clock) -> Group:
        return Group(effect=key[0], backend=key[1], shape_id=key[2], placement=key[3],
                     owners=[e.owner for e in evs], issue_step=clock,
                     ready_steps=[e.ready_step for e in evs])


def validate_group(g: Group, V, expected_versions: list | None = None) -> str | None:
    """Eq. 3 + owner-map clause: returns the first violation or None."""
    if len(g.owners) == 0:
        return "EMPTY"
    if len(set(g.owners)) != len(g.owners):
        return "OWNER_COLLISION"
    if expected_versions is not None:
        for r, v in zip(g.owners, expected_versions):
            if V(r) != v:
                return "VERSION_MISMATCH"
    return None

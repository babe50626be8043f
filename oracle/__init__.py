"""CPU float64 oracle of RW-TTT's READ/WRITE hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import, call or execute anything under `oracle/`.
The product path (`paper_2605_28053_b200/`) never does and fails loudly when
its CUDA library is missing.  The oracle shares no code with the CUDA path;
both consume seeded inputs from `workload/` only.

Modules:  numerics (READ / WRITE arithmetic, bf16 storage rounding),
state (owner table: versions, tails, commit, snapshot, rollback, fork),
planner (§4.3 / Eq. 3 / Eq. 4), run (sequential execution and Alg. 1),
lowrank (DeltaAdapterState, NEXT f1).
Pins: tests/test_oracle_pins.py.  Parity unpinned: agreement with the real
In-Place-TTT rule (the paper does not state it) — every float
result is pinned to the stated reading only (DESIGN.md §"Readings").
"""

"""Oracle arithmetic of the low-rank delta backend (DeltaAdapterState, NEXT f1).

TEST INFRASTRUCTURE ONLY (see oracle/numerics.py header).

The paper names the payload — "a LoRA-style backend stores request-owned low-rank
deltas in DeltaAdapterState" (App. F) — but, as for the fast
weights, not its learning rule.  SPEC fixes a rank-1 stand-in on a square state
(S:168-172 A, B are r×d; S:188 READ y = x + Bᵀ(A x); S:215 WRITE A' = A + η·(A m)·mᵀ,
B' = B, m = chunk mean).  Generalised to d_model ≠ d_ff with the shared base
(reading xviii):
    READ   y  = W_down · z + Bᵀ (A z)          A ∈ R^{R×d_ff}, B ∈ R^{R×d_model}
    WRITE  m  = (1/C) Σ_t z_t;   A' = A + η (A m) mᵀ;   B' = B
The candidate is stored in σ.dtype (reading xi).  With W_down = I and d_model = d_ff
this is exactly SPEC's rule (pinned by tests/test_oracle_pins.py).
"""
from __future__ import annotations

import numpy as np

from . import numerics as nm


def apply_read(w_down: np.ndarray, A: np.ndarray, B: np.ndarray, z: np.ndarray) -> np.ndarray:
    """y = W_down z + Bᵀ (A z)."""
    return w_down @ z + B.T @ (A @ z)


def boundary_update(A: np.ndarray, B: np.ndarray, Z: np.ndarray, eta: float, dtype: str):
    """(A', B') with A' = A + η (A m) mᵀ, m = mean of the chunk's z rows; B' = B."""
    m = Z.sum(axis=0) / Z.shape[0]
    A_new = A + eta * np.outer(A @ m, m)
    return nm.to_storage(A_new, dtype), np.array(B, copy=True)

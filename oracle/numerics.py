"""Oracle arithmetic of the READ / WRITE operators, plain NumPy float64.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path may import `oracle/`;
only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs do.  The oracle shares no code with the CUDA path:
its only common dependency is `workload/` (seeded inputs, no method math).

Every operand arrives as the exact bits the device receives (bf16 bit
patterns or fp32 values) and is widened *exactly* to float64 here.

Pins: tests/test_oracle_pins.py (closed forms, SPEC worked examples, exact
rational brute force, library routines).  See DESIGN.md §"Oracle and pins".
"""
from __future__ import annotations

import numpy as np


# ---------------------------------------------------------------------------
# exact widening / storage rounding
# ---------------------------------------------------------------------------
def widen(a, dtype: str) -> np.ndarray:
    """Device operand -> float64, exactly.  bf16: bits << 16 is the fp32 pattern."""
    if dtype == "bf16":
        u = np.asarray(a, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
        return u.view(np.float32).astype(np.float64)
    if dtype == "fp32":
        return np.asarray(a, dtype=np.float32).astype(np.float64)
    raise ValueError(dtype)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 value (ties to even), as float64.

    Storage rounding of a committed fast-weight version when σ.dtype = bf16
    (SURVEY.md §8(c) reading xi: "bf16 storage uses RNE ... once per version";
    P:253-255 puts dtype in the operator shape class; "BF16 cached decode").
    bf16 = 1 sign, 8 exponent, 7 stored mantissa bits: 8 significant bits.
    """
    x = np.asarray(x, dtype=np.float64)
    out = np.array(x, copy=True)
    fin = np.isfinite(x) & (x != 0.0)
    m, e = np.frexp(x[fin])                 # x = m * 2^e, 0.5 <= |m| < 1
    # quantum of an 8-significant-bit number with exponent e is 2^(e-8);
    # bf16 subnormals have the fixed quantum 2^-133.
    q = np.maximum(e - 8, -133)
    r = np.rint(np.ldexp(x[fin], -q))       # np.rint rounds half to even
    out[fin] = np.ldexp(r, q)
    big = np.abs(out) > float(np.float32(3.3895313892515355e38))
    out[big] = np.sign(out[big]) * np.inf
    return out


def to_storage(x: np.ndarray, dtype: str) -> np.ndarray:
    """Value of the exact candidate `x` after being stored in the declared storage dtype.

    Reading xi: "bf16 storage uses RNE from fp32 accumulators, once per version" — the value
    rounded to bf16 is the fp32 accumulator, so the mirror first rounds the exact candidate to
    fp32 (round to nearest even) and then applies the bf16 RNE; storage rounding is a decision
    taken in the kernel's precision, and both sides take it there.
    """
    if dtype == "bf16":
        return round_bf16(np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64))
    if dtype == "fp32":
        return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)
    raise ValueError(dtype)


# ---------------------------------------------------------------------------
# READ: ApplyState (Table 3; READ paragraph P:403-409)
# ---------------------------------------------------------------------------
def apply_read(w_down: np.ndarray, delta: np.ndarray, z: np.ndarray, rule: int = 0) -> np.ndarray:
    """y = (W_down + ΔW_owner) · z   (BASELINE.json north_star: y = x·(W_down + ΔW)ᵀ).

    rule 1: W_down is the identity and y = z + ΔW·z.
    The state is read, never written: the version is kept.
    """
    if rule == 1:
        return z + delta @ z
    return (w_down + delta) @ z


# ---------------------------------------------------------------------------
# WRITE: BoundaryUpdate (Table 3; WRITE paragraph P:410-417)
# ---------------------------------------------------------------------------
def boundary_update(delta: np.ndarray, Z: np.ndarray, V: np.ndarray, eta: float,
                    dtype: str, rule: int = 0) -> np.ndarray:
    """Dirty candidate ΔW̃_{v+1} from committed ΔW_v and the chunk evidence.

    rule 0 (SURVEY.md §8(c) reading i, the chunked In-Place-TTT outer-product
    update BJ names):  ΔW̃ = ΔW_v + η · Σ_{t=1..C} v_t z_tᵀ = ΔW_v + η · V_cᵀ Z_c,
      with Z_c = [C, d_ff] (READ inputs z_t) and V_c = [C, d_model] (targets v_t).
    rule 1:  m = mean_t z_t;  ΔW̃ = ΔW_v + η · m mᵀ.
    The candidate is then stored in σ.dtype (reading xi).  The input state is
    not modified; a fresh array is returned (the candidate is
    invisible until commit).
    """
    if rule == 1:
        m = Z.sum(axis=0) / Z.shape[0]
        cand = delta + eta * np.outer(m, m)
    else:
        cand = delta + eta * (V.T @ Z)
    return to_storage(cand, dtype)


# ---------------------------------------------------------------------------
# tolerance metric (SURVEY.md §8(c) reading xii)
# ---------------------------------------------------------------------------
def normwise_rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    """max|g − o| / max|o| over one tensor (reading xii).  0/0 -> 0."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = float(np.max(np.abs(ref))) if ref.size else 0.0
    num = float(np.max(np.abs(got - ref))) if ref.size else 0.0
    if den == 0.0:
        return num
    return num / den


TOL = {"bf16": 2e-2, "fp32": 1e-5}   # BASELINE.json north_star tolerances

"""Seeded, counter-based input generator shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no READ, no WRITE, no
commit, no planning).  It only turns a counter key
``(seed, tensor, owner, layer, pos, index)`` into a reproducible number, so
that `oracle/` and the CUDA path can consume bit-identical inputs without
sharing any code.  The CUDA side re-implements the same generator in
`paper_2605_28053_b200/csrc/gen/ttt_gen.cu` (a separate shared library,
`libttt_gen.so`, that is not part of the product boundary); `tests/
test_workload_gen.py` checks the two agree bit for bit on the GPU.

Generator (both sides):

    mix(z)   = splitmix64 finaliser (Steele et al., 2014)
    key      = mix(mix(mix(mix(mix(seed ^ G0) ^ tensor) ^ owner) ^ layer) ^ (pos + 2^31))
    h_i      = mix(key + (i + 1) * G1)                    (uint64, wraps mod 2^64)
    u_i      = int(h_i >> 40) - 2^23                      (int in [-2^23, 2^23))
    f_i      = fp32(u_i) * 2^-23 * amp                    (two fp32 multiplies, RN)
    bf16_i   = RNE(f_i)                                   (for bf16 operands)

with G0 = 0x243F6A8885A308D3 and G1 = 0x9E3779B97F4A7C15.  `amp` is an fp32
scalar; f_i lies in [-amp, amp).  The recipe (which tensors, which amp) is in
DESIGN.md §"Input recipe" and follows SURVEY.md §8(d): W_down, ΔW_0 ~
U(-1,1)/sqrt(d_ff); z, v ~ U(-1,1) (SPEC S:238 bound).
"""
from __future__ import annotations

import numpy as np

G0 = np.uint64(0x243F6A8885A308D3)
G1 = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

# tensor ids (stable; the CUDA generator receives the same integers)
T_W_DOWN = 1     # shared base down-projection W_down[l]      [d_model, d_ff]
T_DELTA0 = 2     # initial fast-weight delta ΔW_0[r, l]        [d_model, d_ff]
T_X = 3          # READ input z = x[r, p, l] (down-proj input) [d_ff]
T_TGT = 4        # update target v[r, p, l]                    [d_model]
T_LR_A = 5       # low-rank A_0[r, l]                          [rank, d_ff]
T_LR_B = 6       # low-rank B[r, l]                            [rank, d_model]

POS_BIAS = 1 << 31


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= M1
    z ^= z >> np.uint64(27)
    z *= M2
    z ^= z >> np.uint64(31)
    return z


def stream_key(seed: int, tensor: int, owner: int, layer: int, pos: int) -> np.uint64:
    """64-bit key of one generated tensor (see module docstring)."""
    k = np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ G0], dtype=np.uint64)
    k = _mix(k)
    for part in (tensor, owner, layer, pos + POS_BIAS):
        k = _mix(k ^ np.uint64(part & 0xFFFFFFFFFFFFFFFF))
    return k[0]


def raw_u24(seed, tensor, owner, layer, pos, n: int) -> np.ndarray:
    """The integers u_i in [-2^23, 2^23) for i in [0, n)."""
    key = stream_key(seed, tensor, owner, layer, pos)
    idx = np.arange(1, n + 1, dtype=np.uint64)
    h = _mix(key + idx * G1)
    return (h >> np.uint64(40)).astype(np.int64) - (1 << 23)


def uniform_f32(seed, tensor, owner, layer, pos, shape, amp: float = 1.0) -> np.ndarray:
    """fp32 values fp32(u) * 2^-23 * amp, shape `shape` (row-major)."""
    n = int(np.prod(shape))
    u = raw_u24(seed, tensor, owner, layer, pos, n).astype(np.float32)
    f = u * np.float32(2.0 ** -23)
    f = f * np.float32(amp)
    return f.reshape(shape)


def f32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns.

    Input generation only: both sides receive these bits as their operands.
    """
    b = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = ((b >> np.uint64(23)) & np.uint64(0xFF)) == np.uint64(0xFF)
    nan &= (b & np.uint64(0x7FFFFF)) != np.uint64(0)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = (b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    r = np.where(nan, (b >> np.uint64(16)) | np.uint64(0x40), r)
    return r.astype(np.uint16).reshape(np.shape(f))


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def gen(seed, tensor, owner, layer, pos, shape, amp: float, dtype: str) -> np.ndarray:
    """Operand as the device sees it: uint16 bf16 bits, or fp32 values."""
    f = uniform_f32(seed, tensor, owner, layer, pos, shape, amp)
    if dtype == "bf16":
        return f32_to_bf16_bits(f)
    if dtype == "fp32":
        return f
    raise ValueError(dtype)


def amp_inv_sqrt(n: int) -> float:
    """fp32 amplitude 1/sqrt(n), the value both sides are handed."""
    return float(np.float32(1.0 / np.sqrt(float(n))))

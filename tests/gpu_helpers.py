"""Helpers for -m gpu parity tests: seeded host inputs uploaded to the device.

Inputs come from workload/ only (shared seeded generator, no method math);
expected values come from oracle/ only.  Nothing here computes the method.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import numerics as nm
from paper_2605_28053_b200.serving import Engine, InputSource, StepIO


def to_dev(arr: np.ndarray, dtype: str, device) -> torch.Tensor:
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(arr).view(np.int16)).to(device).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(device)


def to_host_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def bits_to_f64(a: np.ndarray, dtype: str) -> np.ndarray:
    return nm.widen(a, dtype)


class HostGenInputs(InputSource):
    def __init__(self, tr, device, layers=None):
        self.tr, self.dev = tr, device
        self.layers = list(range(tr.n_layers)) if layers is None else layers
        self.out = {}

    def init_delta(self, s):
        if self.tr.delta0 == "zero":
            return None
        if self.tr.backend == 1:                 # low-rank payload per layer: A (R·d_ff) then B (R·d_model)
            flat = [np.concatenate([a.ravel(), b.ravel()]) for a, b in (self.tr.delta0_of(s, l) for l in self.layers)]
            return to_dev(np.stack(flat), self.tr.dtype, self.dev)
        return to_dev(np.stack([self.tr.delta0_of(s, l) for l in self.layers]), self.tr.dtype, self.dev)

    def tail_prefill(self, s):
        off = self.tr.offset(s)
        if not off:
            return None
        ps = range(-off, 0)
        Z = np.stack([np.stack([self.tr.x(s, p, l) for p in ps]) for l in self.layers])
        V = np.stack([np.stack([self.tr.tgt(s, p, l) for p in ps]) for l in self.layers])
        return off, to_dev(Z, self.tr.dtype, self.dev), to_dev(V, self.tr.dtype, self.dev)

    def group_io(self, l, ss, ps):
        tr = self.tr
        X = to_dev(np.stack([tr.x(s, p, l) for s, p in zip(ss, ps)]), tr.dtype, self.dev)
        Vt = to_dev(np.stack([tr.tgt(s, p, l) for s, p in zip(ss, ps)]), tr.dtype, self.dev)
        Y = torch.empty(len(ss), tr.d_model, dtype=X.dtype, device=self.dev)
        return X, None, Vt, None, Y, None

    def on_output(self, l, ss, ps, Y, yr):
        Yh = to_host_f64(Y)
        for k, (s, p) in enumerate(zip(ss, ps)):
            self.out[(s, p, l)] = Yh[k]

    def step_io(self, ss, ps):
        tr, L, n = self.tr, len(self.layers), len(ss)
        X = to_dev(np.stack([np.stack([tr.x(s, p, l) for s, p in zip(ss, ps)]) for l in self.layers]), tr.dtype, self.dev)
        Vt = to_dev(np.stack([np.stack([tr.tgt(s, p, l) for s, p in zip(ss, ps)]) for l in self.layers]), tr.dtype,
                    self.dev)
        Y = torch.empty(L, n, tr.d_model, dtype=X.dtype, device=self.dev)
        return StepIO(X, n * tr.d_ff, Vt, n * tr.d_model, Y, n * tr.d_model, list(range(n)))

    def on_step(self, executed, io):
        if not executed:
            return
        Yh = to_host_f64(io.Y)
        for s, p, row in executed:
            for i, l in enumerate(self.layers):
                self.out[(s, p, l)] = Yh[i, row]


def make_engine(tr, device="cuda", n_ckpt=4, max_owners=None, mode=None, B=None, w=None):
    if tr.rule == 1:                       # SPEC-compat rule 1: the base is the identity
        eye = np.eye(tr.d_model, tr.d_ff)
        one = (eye * 0x3F80).astype(np.uint16) if tr.dtype == "bf16" else eye.astype(np.float32)
        W = to_dev(np.stack([one] * tr.n_layers), tr.dtype, device)
    else:
        W = to_dev(np.stack([tr.w_down(l) for l in range(tr.n_layers)]), tr.dtype, device)
    return Engine(tr.d_model, tr.d_ff, tr.chunk, tr.n_layers, tr.dtype,
                  max_owners or tr.n_streams + 2, W, n_ckpt=n_ckpt,
                  mode=tr.mode if mode is None else mode, B=tr.B if B is None else B,
                  w=tr.w if w is None else w, eta=tr.eta, backend=tr.backend, rank=tr.rank, rule=tr.rule)


def read_lowrank(eng, tr, owner, l):
    """Committed (A, B) of one owner-layer as float64 (low-rank backend)."""
    from paper_2605_28053_b200 import capi
    flat = capi.tttstate_read_payload_flat(eng.pool, owner, l, tr.rank * (tr.d_ff + tr.d_model), tr.dtype)
    A = nm.widen(flat[: tr.rank * tr.d_ff], tr.dtype).reshape(tr.rank, tr.d_ff)
    B = nm.widen(flat[tr.rank * tr.d_ff:], tr.dtype).reshape(tr.rank, tr.d_model)
    return A, B


class DeviceGenInputs(InputSource):
    """Paper-sized inputs generated on the device by libttt_gen.so with the same counter
    keys as workload/ (bit-identical: tests/test_gpu_parity.py::test_generator_device_matches_numpy)."""

    def __init__(self, tr, device, record_streams=()):
        from paper_2605_28053_b200 import capi
        from workload import rng
        self.capi, self.rng, self.tr, self.dev = capi, rng, tr, device
        self.bf16 = tr.dtype == "bf16"
        self.tdt = torch.bfloat16 if self.bf16 else torch.float32
        self.record = set(record_streams)
        self.out = {}

    def _gen(self, shape, tensor, owner, layer, pos, amp):
        t = torch.empty(*shape, dtype=self.tdt, device=self.dev)
        self.capi.gen_uniform(t, self.tr.seed, tensor, owner, layer, pos, t.numel(), amp, self.bf16)
        return t

    def w_down(self):
        tr, rng = self.tr, self.rng
        return torch.stack([self._gen((tr.d_model, tr.d_ff), rng.T_W_DOWN, 0, l, 0, tr.amp_w)
                            for l in range(tr.n_layers)])

    def init_delta(self, s):
        tr, rng = self.tr, self.rng
        if tr.delta0 == "zero":
            return None
        if tr.backend == 1:                      # low-rank payload per layer: A (R·d_ff) then B (R·d_model)
            return torch.stack([torch.cat([self._gen((tr.rank * tr.d_ff,), rng.T_LR_A, tr.owner(s), l, 0, tr.amp_w),
                                           self._gen((tr.rank * tr.d_model,), rng.T_LR_B, tr.owner(s), l, 0,
                                                     rng.amp_inv_sqrt(tr.rank))])
                                for l in range(tr.n_layers)])
        return torch.stack([self._gen((tr.d_model, tr.d_ff), rng.T_DELTA0, tr.owner(s), l, 0, tr.amp_w)
                            for l in range(tr.n_layers)])

    def tail_prefill(self, s):
        tr, rng = self.tr, self.rng
        off = tr.offset(s)
        if not off:
            return None
        Z = torch.stack([torch.stack([self._gen((tr.d_ff,), rng.T_X, tr.owner(s), l, p, 1.0) for p in range(-off, 0)])
                         for l in range(tr.n_layers)])
        V = torch.stack([torch.stack([self._gen((tr.d_model,), rng.T_TGT, tr.owner(s), l, p, 1.0)
                                      for p in range(-off, 0)]) for l in range(tr.n_layers)])
        return off, Z, V

    def group_io(self, l, ss, ps):
        tr, rng = self.tr, self.rng
        X = torch.stack([self._gen((tr.d_ff,), rng.T_X, tr.owner(s), l, p, 1.0) for s, p in zip(ss, ps)])
        Vt = torch.stack([self._gen((tr.d_model,), rng.T_TGT, tr.owner(s), l, p, 1.0) for s, p in zip(ss, ps)])
        Y = torch.empty(len(ss), tr.d_model, dtype=self.tdt, device=self.dev)
        return X, None, Vt, None, Y, None

    def on_output(self, l, ss, ps, Y, yr):
        for k, (s, p) in enumerate(zip(ss, ps)):
            if s in self.record:
                self.out[(s, p, l)] = to_host_f64(Y[k])

    def step_io(self, ss, ps):
        tr, rng, L, n = self.tr, self.rng, self.tr.n_layers, len(ss)
        X = torch.empty(L, n, tr.d_ff, dtype=self.tdt, device=self.dev)
        Vt = torch.empty(L, n, tr.d_model, dtype=self.tdt, device=self.dev)
        for l in range(L):
            for i, (s, p) in enumerate(zip(ss, ps)):
                self.capi.gen_uniform(X[l, i], tr.seed, rng.T_X, tr.owner(s), l, p, tr.d_ff, 1.0, self.bf16)
                self.capi.gen_uniform(Vt[l, i], tr.seed, rng.T_TGT, tr.owner(s), l, p, tr.d_model, 1.0, self.bf16)
        Y = torch.empty(L, n, tr.d_model, dtype=self.tdt, device=self.dev)
        return StepIO(X, n * tr.d_ff, Vt, n * tr.d_model, Y, n * tr.d_model, list(range(n)))

    def on_step(self, executed, io):
        for s, p, row in executed:
            if s in self.record:
                for l in range(self.tr.n_layers):
                    self.out[(s, p, l)] = to_host_f64(io.Y[l, row])

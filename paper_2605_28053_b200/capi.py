"""Thin ctypes binding of include/tttstate.h — same names, argument marshalling only.

Every step of the hot path runs in libtttstate.so (C++ host logic + sm_100a
kernels).  Importing this module fails loudly if the library is missing;
there is no Python or CPU fallback.  Device buffers may be given as torch
tensors (their data_ptr is passed) or as raw integer addresses.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TTT_LIB_PATH") or os.path.join(_HERE, "lib", "libtttstate.so")   # override: A/B tuning builds
GEN_PATH = os.path.join(_HERE, "lib", "libttt_gen.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2605_28053_b200.build_native` "
                      "(or __graft_entry__.build()); there is no fallback path")
_lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
TTT_OK = 0
TTT_E_WRITE_FAILED = 9
READ, WRITE = 0, 1
FP32, BF16 = 0, 1
FAST_WEIGHT, LOW_RANK, STREAMING = 0, 1, 2
MODE_SERIAL, MODE_PHASE, MODE_FULL = 0, 1, 2
DTYPE = {"fp32": FP32, "bf16": BF16}


class ttt_shape(C.Structure):
    _fields_ = [("backend", C.c_int32), ("dtype", C.c_int32), ("d_model", C.c_int32), ("d_ff", C.c_int32),
                ("chunk", C.c_int32), ("rank", C.c_int32), ("n_layers", C.c_int32), ("rule", C.c_int32)]


class ttt_event(C.Structure):
    _fields_ = [("owner", C.c_uint64), ("effect", C.c_int32), ("backend", C.c_int32),
                ("shape_id", C.c_int32), ("placement", C.c_int32), ("expected_version", C.c_uint64),
                ("ready_step", C.c_int64)]

    def __repr__(self):
        return (f"ttt_event(owner={self.owner}, effect={self.effect}, shape_id={self.shape_id}, "
                f"placement={self.placement}, v={self.expected_version}, ready={self.ready_step})")


class ttt_group(C.Structure):
    _fields_ = [("effect", C.c_int32), ("backend", C.c_int32), ("shape_id", C.c_int32),
                ("placement", C.c_int32), ("n", C.c_int32), ("_reserved", C.c_int32),
                ("owner_map", C.POINTER(C.c_uint64)), ("issue_step", C.c_int64)]


class ttt_step_io(C.Structure):
    _fields_ = [("X", C.c_void_p), ("x_layer_stride", C.c_int64), ("Vt", C.c_void_p), ("v_layer_stride", C.c_int64),
                ("Y", C.c_void_p), ("y_layer_stride", C.c_int64), ("resid", C.c_void_p), ("r_layer_stride", C.c_int64),
                ("rows", C.POINTER(C.c_int32)), ("ev_write_begin", C.c_void_p), ("ev_write_end", C.c_void_p),
                ("rows_total", C.c_int64)]


class ttt_step_out(C.Structure):
    _fields_ = [("groups", C.POINTER(ttt_group)), ("group_cap", C.c_int32), ("owner_cap", C.c_int32),
                ("owner_buf", C.POINTER(C.c_uint64)), ("v_before", C.POINTER(C.c_uint64)),
                ("member_seq", C.POINTER(C.c_uint64)), ("injected", C.POINTER(C.c_int32)),
                ("rej_cap", C.c_int32), ("_pad", C.c_int32), ("rejected", C.POINTER(ttt_event)),
                ("n_groups", C.c_int32), ("n_rejected", C.c_int32), ("n_read", C.c_int32), ("n_write", C.c_int32),
                ("n_injected", C.c_int32), ("_pad2", C.c_int32)]


assert C.sizeof(ttt_event) == 40 and C.sizeof(ttt_shape) == 32


class TTTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


P = C.c_void_p
_sigs = {
    "tttstate_last_error": (C.c_char_p, []),
    "tttstate_status_name": (C.c_char_p, [C.c_int]),
    "tttstate_pool_bytes": (C.c_int, [C.POINTER(ttt_shape), C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]),
    "tttstate_pool_create": (C.c_int, [C.POINTER(ttt_shape), C.c_int32, C.c_int32, C.c_int32, C.c_int32, P,
                                       C.c_size_t, P, C.POINTER(P)]),
    "tttstate_pool_destroy": (C.c_int, [P]),
    "tttstate_alloc": (C.c_int, [P, C.c_uint64, P, C.c_uint64, C.POINTER(C.c_uint64), P]),
    "tttstate_free": (C.c_int, [P, C.c_uint64]),
    "tttstate_tail_load": (C.c_int, [P, C.c_uint64, C.c_int32, P, P, P]),
    "tttstate_version": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_uint64)]),
    "tttstate_tail_len": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_int32)]),
    "tttstate_next_event": (C.c_int, [P, C.c_uint64, C.c_int64, C.POINTER(ttt_event)]),
    "tttstate_next_events": (C.c_int, [P, C.POINTER(C.c_uint64), C.c_int32, C.c_int64, C.POINTER(ttt_event)]),
    "ttt_planner_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]),
    "ttt_planner_destroy": (C.c_int, [P]),
    "ttt_planner_attach": (C.c_int, [P, P]),
    "ttt_planner_pending": (C.c_int, [P, C.POINTER(C.c_int32)]),
    "plan_batch": (C.c_int, [P, C.POINTER(ttt_event), C.c_int32, C.c_int64, C.POINTER(ttt_group), C.c_int32,
                             C.POINTER(C.c_uint64), C.c_int32, C.POINTER(C.c_int32), C.POINTER(ttt_event),
                             C.c_int32, C.POINTER(C.c_int32)]),
    "validate_group": (C.c_int, [P, C.POINTER(ttt_group), C.POINTER(C.c_uint64)]),
    "read_apply": (C.c_int, [P, C.POINTER(ttt_group), C.c_int32, P, C.POINTER(C.c_int32), P,
                             C.POINTER(C.c_int32), P, C.POINTER(C.c_int32), P, P]),
    "tttstate_step_done": (C.c_int, [P, C.POINTER(ttt_group)]),
    "read_apply_chunk": (C.c_int, [P, C.POINTER(ttt_group), C.c_int32, P, P, P, P]),
    "tttstate_set_eta": (C.c_int, [P, C.c_float]),
    "write_commit": (C.c_int, [P, C.POINTER(ttt_group), C.c_float, C.POINTER(C.c_uint32),
                               C.POINTER(C.c_uint64), P]),
    "tttstate_snapshot": (C.c_int, [P, C.c_uint64, P]),
    "rollback": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_uint64), P]),
    "tttstate_fork": (C.c_int, [P, C.c_uint64, C.c_uint64, P]),
    "tttstate_sync": (C.c_int, [P, P, C.POINTER(C.c_int32)]),
    "tttstate_refusals": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                    C.c_int32, C.POINTER(C.c_int32), P]),
    "tttstate_last_commit_seq": (C.c_int, [P, C.POINTER(C.c_uint64)]),
    "tttstate_serve_step": (C.c_int, [P, P, C.POINTER(C.c_uint64), C.c_int32, C.c_int64, C.POINTER(ttt_step_io),
                                      C.c_float, C.POINTER(C.c_uint64), C.c_int32, C.POINTER(ttt_step_out), P]),
    "tttstate_read_payload": (C.c_int, [P, C.c_uint64, C.c_int32, P, P]),
    "tttstate_read_slot_raw": (C.c_int, [P, C.c_uint64, C.c_int32, C.c_int32, P, P]),
    "tttstate_read_tail": (C.c_int, [P, C.c_uint64, C.c_int32, P, P, P]),
    "tttstate_device_version": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_uint64), P]),
    "tttstate_launch_count": (C.c_int64, []),
    "tttstate_set_write_impl": (C.c_int32, [C.c_int32]),
    "tttstate_set_test_hook": (C.c_int32, [C.c_int32]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype, _f.argtypes = _res, _args

EXPORTED = tuple(_sigs)


def _check(st: int):
    if st != TTT_OK:
        raise TTTError(st, _lib.tttstate_last_error().decode())


def _ptr(x):
    """Device address of a torch tensor / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


_POOL_INFO: dict = {}     # pool handle -> ttt_shape (argument checks of tensor operands)
_TORCH_DTYPE = {FP32: "torch.float32", BF16: "torch.bfloat16"}


def _check_tensor(t, what: str, pool, last: int | None = None, min_rows: int = 0):
    """Checks a torch-tensor operand against the pool's σ.dtype / row width (raw integer
    addresses are the caller's opt-in unchecked path)."""
    if t is None or isinstance(t, int) or pool not in _POOL_INFO:
        return
    sh = _POOL_INFO[pool]
    if str(t.dtype) != _TORCH_DTYPE[sh.dtype]:
        raise ValueError(f"{what}: dtype {t.dtype} does not match the pool's {_TORCH_DTYPE[sh.dtype]}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: must be contiguous (row-major)")
    if last is not None and (t.dim() == 0 or t.shape[-1] != last):
        raise ValueError(f"{what}: last dimension {tuple(t.shape)[-1:]} != {last}")
    rows = t.numel() // last if last else 0
    if min_rows and rows < min_rows:
        raise ValueError(f"{what}: {rows} rows < {min_rows} needed")


def _check_rows(rows, n: int, what: str):
    if rows is not None and len(rows) < n:
        raise ValueError(f"{what}: {len(rows)} row indices for a group of {n}")


def _rows(rows):
    if rows is None or isinstance(rows, C.Array):   # a prebuilt c_int32 array passes through
        return rows
    return (C.c_int32 * len(rows))(*rows)


def rows_array(rows):
    """A c_int32 row map to reuse across the layers of one step (saves per-call marshalling)."""
    return (C.c_int32 * len(rows))(*rows)


def status_name(st: int) -> str:
    return _lib.tttstate_status_name(st).decode()


# ---------------------------------------------------------------- groups
class Group:
    """A ttt_group plus the storage of its owner map μ (kept alive here)."""

    def __init__(self, effect: int, owners, shape_id: int = 0, placement: int = 0, backend: int = 0,
                 issue_step: int = 0):
        self.owners = tuple(int(o) for o in owners)
        self._buf = (C.c_uint64 * max(1, len(self.owners)))(*self.owners)
        self.c = ttt_group(effect, backend, shape_id, placement, len(self.owners), 0,
                           C.cast(self._buf, C.POINTER(C.c_uint64)), issue_step)

    @property
    def effect(self):
        return self.c.effect

    @property
    def issue_step(self):
        return self.c.issue_step

    def __len__(self):
        return len(self.owners)

    def __repr__(self):
        return f"Group(effect={self.effect}, owners={self.owners}, issue={self.issue_step})"


# ---------------------------------------------------------------- pool
def make_shape(d_model, d_ff, chunk, n_layers, dtype="bf16", backend=FAST_WEIGHT, rank=0, rule=0) -> ttt_shape:
    return ttt_shape(backend, DTYPE[dtype] if isinstance(dtype, str) else dtype, d_model, d_ff, chunk, rank,
                     n_layers, rule)


def tttstate_pool_bytes(shape: ttt_shape, max_owners: int, n_ckpt: int) -> int:
    out = C.c_size_t()
    _check(_lib.tttstate_pool_bytes(C.byref(shape), max_owners, n_ckpt, C.byref(out)))
    return out.value


def tttstate_pool_create(shape: ttt_shape, shape_id: int, placement: int, max_owners: int, n_ckpt: int,
                         dev_arena, arena_bytes: int, w_down):
    out = P()
    _check(_lib.tttstate_pool_create(C.byref(shape), shape_id, placement, max_owners, n_ckpt, _ptr(dev_arena),
                                     arena_bytes, _ptr(w_down), C.byref(out)))
    _POOL_INFO[out.value] = ttt_shape.from_buffer_copy(shape)
    if shape.rule == 0:
        _check_tensor(w_down, "w_down", out.value, shape.d_ff, shape.n_layers * shape.d_model)
    return out.value


def tttstate_pool_destroy(pool):
    _POOL_INFO.pop(pool, None)
    _check(_lib.tttstate_pool_destroy(pool))


def tttstate_alloc(pool, owner: int, init=None, v0: int = 0, stream=None) -> int:
    if pool in _POOL_INFO and init is not None and not isinstance(init, int):
        sh = _POOL_INFO[pool]
        per = sh.rank * (sh.d_ff + sh.d_model) if sh.backend == LOW_RANK else sh.d_model * sh.d_ff
        _check_tensor(init, "init", pool)
        if init.numel() < sh.n_layers * per:
            raise ValueError(f"init: {init.numel()} elements < {sh.n_layers * per}")
    v = C.c_uint64()
    _check(_lib.tttstate_alloc(pool, owner, _ptr(init), v0, C.byref(v), _stream(stream)))
    return v.value


def tttstate_free(pool, owner: int):
    _check(_lib.tttstate_free(pool, owner))


def tttstate_tail_load(pool, owner: int, n: int, Z, V, stream=None):
    if pool in _POOL_INFO and n > 0:
        sh = _POOL_INFO[pool]
        _check_tensor(Z, "Z", pool, sh.d_ff, sh.n_layers * n)
        _check_tensor(V, "V", pool, sh.d_model, sh.n_layers * n)
    _check(_lib.tttstate_tail_load(pool, owner, n, _ptr(Z), _ptr(V), _stream(stream)))


def tttstate_version(pool, owner: int) -> int:
    v = C.c_uint64()
    _check(_lib.tttstate_version(pool, owner, C.byref(v)))
    return v.value


def tttstate_tail_len(pool, owner: int) -> int:
    v = C.c_int32()
    _check(_lib.tttstate_tail_len(pool, owner, C.byref(v)))
    return v.value


def tttstate_next_events(pool, owners, clock: int) -> list:
    """a1 for every owner in one call (returns a list of ttt_event)."""
    n = len(owners)
    arr = owners if isinstance(owners, C.Array) else (C.c_uint64 * n)(*owners)
    out = (ttt_event * n)()
    _check(_lib.tttstate_next_events(pool, arr, n, clock, out))
    return list(out)


def tttstate_next_event(pool, owner: int, clock: int) -> ttt_event:
    e = ttt_event()
    _check(_lib.tttstate_next_event(pool, owner, clock, C.byref(e)))
    return e


# ---------------------------------------------------------------- planner
def ttt_planner_create(mode: int, B: int, w: int):
    out = P()
    _check(_lib.ttt_planner_create(mode, B, w, C.byref(out)))
    return out.value


def ttt_planner_destroy(pl):
    _check(_lib.ttt_planner_destroy(pl))


def ttt_planner_attach(pl, pool):
    _check(_lib.ttt_planner_attach(pl, pool))


def ttt_planner_pending(pl) -> int:
    n = C.c_int32()
    _check(_lib.ttt_planner_pending(pl, C.byref(n)))
    return n.value


def plan_batch(pl, events, clock: int, cap: int = 512):
    """Returns (groups: list[Group], rejected: list[ttt_event])."""
    n = len(events)
    ev = (ttt_event * max(1, n))(*events)
    out = (ttt_group * cap)()
    obuf = (C.c_uint64 * (cap * 4 + n + 1))()
    rej = (ttt_event * (cap + n + 1))()
    n_out, n_rej = C.c_int32(), C.c_int32()
    _check(_lib.plan_batch(pl, ev, n, clock, out, cap, obuf, len(obuf), C.byref(n_out), rej, len(rej),
                           C.byref(n_rej)))
    groups = []
    for k in range(n_out.value):
        g = out[k]
        groups.append(Group(g.effect, [g.owner_map[b] for b in range(g.n)], g.shape_id, g.placement, g.backend,
                            g.issue_step))
    return groups, [rej[k] for k in range(n_rej.value)]


def validate_group(pool, group: Group, expected_versions=None):
    ev = None if expected_versions is None else (C.c_uint64 * len(expected_versions))(*expected_versions)
    _check(_lib.validate_group(pool, C.byref(group.c), ev))


# ---------------------------------------------------------------- operators
def read_apply(pool, group: Group, layer: int, X, x_rows, Vt, v_rows, Y, y_rows=None, resid=None, stream=None):
    if pool in _POOL_INFO:
        sh, n = _POOL_INFO[pool], len(group)
        _check_tensor(X, "X", pool, sh.d_ff, 0 if x_rows is not None else n)
        _check_tensor(Vt, "Vt", pool, sh.d_model, 0 if v_rows is not None else n)
        _check_tensor(Y, "Y", pool, sh.d_model, 0 if y_rows is not None else n)
        _check_tensor(resid, "resid", pool, sh.d_model)
        for r, w in ((x_rows, "x_rows"), (v_rows, "v_rows"), (y_rows, "y_rows")):
            _check_rows(r, n, w)
    _check(_lib.read_apply(pool, C.byref(group.c), layer, _ptr(X), _rows(x_rows), _ptr(Vt), _rows(v_rows),
                           _ptr(Y), _rows(y_rows), _ptr(resid), _stream(stream)))


def read_apply_chunk(pool, group: Group, layer: int, X, Vt, Y, stream=None):
    """NEXT f2: all C tokens of each member's chunk at version v (tcgen05); then write_commit."""
    if pool in _POOL_INFO:
        sh, n = _POOL_INFO[pool], len(group)
        _check_tensor(X, "X", pool, sh.d_ff, n * sh.chunk)
        _check_tensor(Vt, "Vt", pool, sh.d_model, n * sh.chunk)
        _check_tensor(Y, "Y", pool, sh.d_model, n * sh.chunk)
    _check(_lib.read_apply_chunk(pool, C.byref(group.c), layer, _ptr(X), _ptr(Vt), _ptr(Y), _stream(stream)))


def tttstate_set_eta(pool, eta: float):
    _check(_lib.tttstate_set_eta(pool, C.c_float(eta)))


def tttstate_step_done(pool, group: Group):
    _check(_lib.tttstate_step_done(pool, C.byref(group.c)))


def write_commit(pool, group: Group, eta: float, fail_mask=None, stream=None):
    """Returns the new versions; raises TTTError(status=TTT_E_WRITE_FAILED) on a failed group."""
    nv = (C.c_uint64 * len(group))()
    fm = None
    if fail_mask is not None:
        words = [0] * ((len(group) + 31) // 32)
        for b, bad in enumerate(fail_mask):
            if bad:
                words[b // 32] |= 1 << (b % 32)
        fm = (C.c_uint32 * len(words))(*words)
    _check(_lib.write_commit(pool, C.byref(group.c), C.c_float(eta), fm, nv, _stream(stream)))
    return list(nv)


def tttstate_snapshot(pool, owner: int, stream=None):
    _check(_lib.tttstate_snapshot(pool, owner, _stream(stream)))


def rollback(pool, owner: int, stream=None) -> int:
    v = C.c_uint64()
    _check(_lib.rollback(pool, owner, C.byref(v), _stream(stream)))
    return v.value


def tttstate_fork(pool, src: int, dst: int, stream=None):
    _check(_lib.tttstate_fork(pool, src, dst, _stream(stream)))


def tttstate_sync(pool, stream=None) -> int:
    """Synchronise; returns the number of groups that failed on the device since the last sync."""
    n = C.c_int32()
    st = _lib.tttstate_sync(pool, _stream(stream), C.byref(n))
    if st not in (TTT_OK, TTT_E_WRITE_FAILED):
        _check(st)
    return n.value


def tttstate_refusals(pool, stream=None, cap: int = 4096):
    """Drain the device refusal records: list of (owner, version kept, commit seq)."""
    o, v, q = (C.c_uint64 * cap)(), (C.c_uint64 * cap)(), (C.c_uint64 * cap)()
    n = C.c_int32()
    _check(_lib.tttstate_refusals(pool, o, v, q, cap, C.byref(n), _stream(stream)))
    return [(o[k], v[k], q[k]) for k in range(n.value)]


def tttstate_last_commit_seq(pool) -> int:
    v = C.c_uint64()
    _check(_lib.tttstate_last_commit_seq(pool, C.byref(v)))
    return v.value


class StepBuffers:
    """Preallocated host buffers of tttstate_serve_step (reused every step: marshalling only)."""

    def __init__(self, max_owners: int, group_cap: int = 256):
        self.owners = (C.c_uint64 * max(1, max_owners))()
        self.rows = (C.c_int32 * max(1, max_owners))()
        self.fail = (C.c_uint64 * max(1, max_owners))()
        self.groups = (ttt_group * group_cap)()
        self.owner_buf = (C.c_uint64 * max(1, max_owners))()
        self.v_before = (C.c_uint64 * max(1, max_owners))()
        self.member_seq = (C.c_uint64 * max(1, max_owners))()
        self.injected = (C.c_int32 * group_cap)()
        self.rejected = (ttt_event * max(1, max_owners))()
        self.io = ttt_step_io()
        self.io.rows = C.cast(self.rows, C.POINTER(C.c_int32))
        self.out = ttt_step_out(self.groups, group_cap, max(1, max_owners), self.owner_buf, self.v_before,
                                self.member_seq, self.injected, max(1, max_owners), 0, self.rejected)

    def groups_issued(self):
        """[(effect, [owners], [v_before], [member_seq], injected)] of the last step."""
        res, off = [], 0
        for k in range(self.out.n_groups):
            g = self.groups[k]
            res.append((g.effect, list(self.owner_buf[off:off + g.n]), list(self.v_before[off:off + g.n]),
                        list(self.member_seq[off:off + g.n]), bool(self.injected[k])))
            off += g.n
        return res


def tttstate_serve_step(pool, pl, bufs: StepBuffers, n: int, clock: int, X, x_stride, Vt, v_stride, Y, y_stride,
                        eta: float, n_fail: int = 0, resid=None, r_stride: int = 0, stream=None,
                        ev_write=(None, None), rows_total: int = 0):
    """One Alg. 1 iteration for bufs.owners[:n] at rows bufs.rows[:n] (fill those arrays first)."""
    if pool in _POOL_INFO:
        sh = _POOL_INFO[pool]
        rmax = 1 + max((bufs.rows[i] for i in range(n)), default=-1)
        for t, w, last, stride in ((X, "X", sh.d_ff, x_stride), (Vt, "Vt", sh.d_model, v_stride),
                                   (Y, "Y", sh.d_model, y_stride)):
            _check_tensor(t, w, pool, last)
            if t is not None and not isinstance(t, int) and \
                    t.numel() < (sh.n_layers - 1) * stride + rmax * last:
                raise ValueError(f"{w}: too small for {sh.n_layers} layers at stride {stride} and row {rmax - 1}")
    io = bufs.io
    io.X, io.x_layer_stride, io.Vt, io.v_layer_stride = _ptr(X), x_stride, _ptr(Vt), v_stride
    io.Y, io.y_layer_stride, io.resid, io.r_layer_stride = _ptr(Y), y_stride, _ptr(resid), r_stride
    io.ev_write_begin = None if ev_write[0] is None else ev_write[0].cuda_event
    io.ev_write_end = None if ev_write[1] is None else ev_write[1].cuda_event
    io.rows_total = rows_total
    _check(_lib.tttstate_serve_step(pool, pl, bufs.owners, n, clock, C.byref(io), C.c_float(eta),
                                    bufs.fail if n_fail else None, n_fail, C.byref(bufs.out), _stream(stream)))
    return bufs.out


def _np_dtype(dtype):
    return np.uint16 if dtype in (BF16, "bf16") else np.float32


def tttstate_read_payload(pool, owner: int, layer: int, d_model: int, d_ff: int, dtype, stream=None):
    out = np.empty((d_model, d_ff), dtype=_np_dtype(dtype))
    _check(_lib.tttstate_read_payload(pool, owner, layer, out.ctypes.data, _stream(stream)))
    return out


def tttstate_read_payload_flat(pool, owner: int, layer: int, n_elems: int, dtype, stream=None):
    """Committed payload of one layer as a flat array (low-rank: A [R·d_ff] then B [R·d_model])."""
    out = np.empty((n_elems,), dtype=_np_dtype(dtype))
    _check(_lib.tttstate_read_payload(pool, owner, layer, out.ctypes.data, _stream(stream)))
    return out


def tttstate_read_slot_raw(pool, owner: int, which: int, layer: int, d_model: int, d_ff: int, dtype, stream=None):
    out = np.empty((d_model, d_ff), dtype=_np_dtype(dtype))
    _check(_lib.tttstate_read_slot_raw(pool, owner, which, layer, out.ctypes.data, _stream(stream)))
    return out


def tttstate_read_tail(pool, owner: int, layer: int, chunk: int, d_model: int, d_ff: int, dtype, stream=None):
    Z = np.empty((chunk, d_ff), dtype=_np_dtype(dtype))
    V = np.empty((chunk, d_model), dtype=_np_dtype(dtype))
    _check(_lib.tttstate_read_tail(pool, owner, layer, Z.ctypes.data, V.ctypes.data, _stream(stream)))
    return Z, V


def tttstate_device_version(pool, owner: int, stream=None) -> int:
    v = C.c_uint64()
    _check(_lib.tttstate_device_version(pool, owner, C.byref(v), _stream(stream)))
    return v.value


def tttstate_launch_count() -> int:
    return _lib.tttstate_launch_count()


TTT_HOOK_NO_GROUP_ATOMICITY = 1


def tttstate_set_test_hook(flags: int) -> int:
    """Stress-suite negative control only (include/tttstate.h); returns the previous flags."""
    return _lib.tttstate_set_test_hook(flags)


def tttstate_set_write_impl(impl: int) -> int:
    return _lib.tttstate_set_write_impl(impl)


# ---------------------------------------------------------------- input generator (bench/tests)
_gen = None


def gen_uniform(out, seed, tensor, owner, layer, pos, n, amp, bf16: bool, stream=None):
    """Fill device buffer `out` with workload/rng.py's generator (libttt_gen.so)."""
    global _gen
    if _gen is None:
        _gen = C.CDLL(GEN_PATH)
        _gen.ttt_gen_uniform.restype = C.c_int
        _gen.ttt_gen_uniform.argtypes = [P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64,
                                         C.c_size_t, C.c_float, C.c_int, P]
    st = _gen.ttt_gen_uniform(_ptr(out), seed, tensor, owner, layer, pos, n, C.c_float(amp), int(bf16),
                              _stream(stream))
    if st != 0:
        raise RuntimeError(f"ttt_gen_uniform failed: cuda error {st}")

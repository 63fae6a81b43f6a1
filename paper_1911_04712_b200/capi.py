"""Thin ctypes binding of libdpd.so (include/dpd.h): same names, argument marshalling only.

Every step of the DPD path runs in the CUDA kernels behind the C-ABI; nothing here
computes.  Loading fails loudly if the library is missing and cannot be built (there is no
CPU fallback).  Arrays are numpy (host) or any object exposing ``data_ptr()`` (e.g. a torch
CUDA tensor) -- the library copies with cudaMemcpyDefault.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

DPD_OK, DPD_ERR_ARG, DPD_ERR_CONFIG, DPD_ERR_CUDA, DPD_ERR_NUMERIC, DPD_ERR_CAPACITY, DPD_ERR_COMM, \
    DPD_ERR_IO = range(8)
_ERR_NAMES = {1: "DPD_ERR_ARG", 2: "DPD_ERR_CONFIG", 3: "DPD_ERR_CUDA", 4: "DPD_ERR_NUMERIC",
              5: "DPD_ERR_CAPACITY", 6: "DPD_ERR_COMM", 7: "DPD_ERR_IO"}


class DPDError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None
_P = C.POINTER
_vp = C.c_void_p

# (name, restype, argtypes) for every symbol in include/dpd.h
SIGNATURES = [
    ("dpd_create", C.c_int, [_P(C.c_double), C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                             C.c_double, C.c_uint64, _P(_vp)]),
    ("dpd_destroy", None, [_vp]),
    ("dpd_last_error", C.c_char_p, [_vp]),
    ("dpd_set_stream", C.c_int, [_vp, _vp]),
    ("dpd_set_body_force", C.c_int, [_vp, C.c_double]),
    ("dpd_set_option", C.c_int, [_vp, C.c_char_p, C.c_int64]),
    ("dpd_get_stat", C.c_int, [_vp, C.c_char_p, _P(C.c_int64)]),
    ("dpd_set_particles", C.c_int, [_vp, C.c_int64, _vp, _vp]),
    ("dpd_set_particles_ex", C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, C.c_int64]),
    ("dpd_set_particles_typed", C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, C.c_int64]),
    ("dpd_set_species", C.c_int, [_vp, C.c_int, _P(C.c_double), _P(C.c_double)]),
    ("dpd_step", C.c_int, [_vp, C.c_int64]),
    ("dpd_step_async", C.c_int, [_vp, C.c_int64]),
    ("dpd_sync", C.c_int, [_vp]),
    ("dpd_get_count", C.c_int, [_vp, _P(C.c_int64)]),
    ("dpd_get_step", C.c_int, [_vp, _P(C.c_int64)]),
    ("dpd_get_particles", C.c_int, [_vp, C.c_int64, _vp, _vp]),
    ("dpd_get_forces", C.c_int, [_vp, C.c_int64, _vp]),
    ("dpd_get_state", C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, _P(C.c_int64)]),
    ("dpd_debug_cells", C.c_int, [_vp, _vp, _vp, _vp]),
    ("dpd_get_grid", C.c_int, [_vp, _P(C.c_int32)]),
    ("dpd_debug_pairs", C.c_int, [_vp, C.c_int64, _vp, _P(C.c_int64)]),
    ("dpd_set_timing", C.c_int, [_vp, C.c_int]),
    ("dpd_get_timing", C.c_int, [_vp, C.c_int, _P(C.c_double), _P(C.c_int64)]),
    ("dpd_kernel_name", C.c_char_p, [C.c_int]),
    ("dpd_get_launch_count", C.c_int, [_vp, _P(C.c_int64)]),
    ("dpd_plan_peers", C.c_int, [_P(C.c_int32), C.c_int, _vp, _vp, _vp]),
    ("dpd_nccl_unique_id", C.c_int, [_vp]),
    ("dpd_create_dist", C.c_int, [_P(C.c_double), C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_uint64, C.c_int, C.c_int, _P(C.c_int32), _vp, _P(_vp)]),
    ("dpd_create_loopback", C.c_int, [_P(C.c_double), C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_uint64, _P(C.c_int32), _vp, _P(_vp)]),
    ("dpd_create_group", C.c_int, [_P(C.c_double), C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, _P(C.c_int32), _P(_vp)]),
    ("dpd_group_step", C.c_int, [_P(_vp), C.c_int, C.c_int64]),
    ("dpd_get_particles_ex", C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _P(C.c_int64)]),
    ("dpd_get_forces_ex", C.c_int, [_vp, C.c_int64, _vp, _vp, _P(C.c_int64)]),
    ("dpd_get_species", C.c_int, [_vp, C.c_int64, _vp]),
    ("dpd_set_walls", C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
    ("dpd_set_frozen_species", C.c_int, [_vp, C.c_int32]),
    ("dpd_wall_carve", C.c_int, [_vp, C.c_int32, _P(C.c_int64), _P(C.c_int64)]),
    ("dpd_wall_sdf", C.c_int, [_vp, C.c_int64, _vp, _vp]),
    ("dpd_get_species_ex", C.c_int, [_vp, C.c_int64, _vp, _vp, _P(C.c_int64)]),
    ("dpd_debug_philox", C.c_int, [C.c_int64, _vp, _vp, _vp]),
    ("dpd_debug_pair_words", C.c_int, [C.c_int64, _vp, C.c_uint64, _vp, _vp]),
    ("dpd_dump_open", C.c_int, [_vp, C.c_char_p, C.c_int]),
    ("dpd_dump_every", C.c_int, [_vp, C.c_int64]),
    ("dpd_dump_now", C.c_int, [_vp]),
    ("dpd_dump_close", C.c_int, [_vp, _P(C.c_int64)]),
    ("dpd_step_schedule", C.c_int, [_vp, C.c_int, C.c_char_p, C.c_int64]),
    ("dpd_tg_create", C.c_int, [_P(_vp)]),
    ("dpd_tg_add", C.c_int, [_vp, C.c_char_p, C.c_int, _P(C.c_int32)]),
    ("dpd_tg_edge", C.c_int, [_vp, C.c_int32, C.c_int32]),
    ("dpd_tg_order", C.c_int, [_vp, C.c_int64, _vp, _P(C.c_int64)]),
    ("dpd_tg_destroy", None, [_vp]),
    ("dpd_ioq_create", C.c_int, [C.c_int, _P(_vp)]),
    ("dpd_ioq_write", C.c_int, [_vp, C.c_char_p, _vp, C.c_int64, C.c_int64]),
    ("dpd_ioq_pending", C.c_int, [_vp, _P(C.c_int64)]),
    ("dpd_ioq_close", C.c_int, [_vp, _P(C.c_int64)]),
    ("dpd_ioq_last_error", C.c_char_p, [_vp]),
]


def lib_path() -> str:
    return _build.LIB


def load():
    """Load (building first if stale) libdpd.so.  Raises if it cannot be built or loaded."""
    global _lib
    if _lib is None:
        path = _build.build()
        if not os.path.exists(path):
            raise RuntimeError(f"libdpd.so missing at {path}")
        L = C.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(a.ctypes.data)
    raise TypeError(f"unsupported buffer {type(a)}")


def _check(ctx, code):
    if code != DPD_OK:
        msg = load().dpd_last_error(ctx).decode() if ctx else ""
        raise DPDError(code, msg)


# ---- functions with the C names -----------------------------------------------------------
def dpd_create(box, rc, a, gamma, kT, power, dt, seed):
    L = load()
    b = (C.c_double * 3)(*[float(x) for x in box])
    out = C.c_void_p()
    code = L.dpd_create(b, rc, a, gamma, kT, power, dt, int(seed), C.byref(out))
    if code != DPD_OK:
        raise DPDError(code, "dpd_create failed (see stderr)")
    return out


def dpd_destroy(ctx):
    load().dpd_destroy(ctx)


def dpd_set_stream(ctx, stream_handle):
    _check(ctx, load().dpd_set_stream(ctx, C.c_void_p(stream_handle) if stream_handle else None))


def dpd_set_option(ctx, name, value):
    _check(ctx, load().dpd_set_option(ctx, name.encode(), int(value)))


def dpd_get_stat(ctx, name):
    v = C.c_int64()
    _check(ctx, load().dpd_get_stat(ctx, name.encode(), C.byref(v)))
    return v.value


def dpd_set_body_force(ctx, f):
    _check(ctx, load().dpd_set_body_force(ctx, float(f)))


def dpd_set_particles(ctx, pos, vel):
    n = int(pos.shape[0])
    _check(ctx, load().dpd_set_particles(ctx, n, _ptr(pos), _ptr(vel)))


def dpd_set_particles_ex(ctx, pos, vel, ids=None, step0=0):
    n = int(pos.shape[0])
    _check(ctx, load().dpd_set_particles_ex(ctx, n, _ptr(pos), _ptr(vel), _ptr(ids), int(step0)))


def dpd_set_particles_typed(ctx, pos, vel, ids=None, species=None, step0=0):
    n = int(pos.shape[0])
    _check(ctx, load().dpd_set_particles_typed(ctx, n, _ptr(pos), _ptr(vel), _ptr(ids), _ptr(species), int(step0)))


def dpd_set_species(ctx, a, gamma):
    """a, gamma: nspecies x nspecies symmetric matrices (NEXT-2)."""
    a = np.ascontiguousarray(a, np.float64)
    gamma = np.ascontiguousarray(gamma, np.float64)
    ns = int(a.shape[0])
    if a.shape != (ns, ns) or gamma.shape != (ns, ns):
        raise ValueError("a and gamma must be square and of equal size")
    _check(ctx, load().dpd_set_species(ctx, ns, a.ctypes.data_as(_P(C.c_double)),
                                       gamma.ctypes.data_as(_P(C.c_double))))


def dpd_set_walls(ctx, walls):
    """walls: list of (type, (p0, p1, p2, p3), (uwx, uwy, uwz)) -- see dpd.h (NEXT-3)."""
    walls = list(walls or [])
    t = np.array([w[0] for w in walls], np.int32)
    prm = np.array([list(w[1]) for w in walls], np.float64).reshape(-1)
    uw = np.array([list(w[2]) for w in walls], np.float64).reshape(-1)
    _check(ctx, load().dpd_set_walls(ctx, len(walls), _ptr(t) if len(walls) else None,
                                     _ptr(prm) if len(walls) else None, _ptr(uw) if len(walls) else None))


def dpd_set_frozen_species(ctx, mask):
    _check(ctx, load().dpd_set_frozen_species(ctx, int(mask)))


def dpd_wall_carve(ctx, wall_species):
    """Frozen layer + removal; returns (n_frozen, n_removed) of this context."""
    nf, nr = C.c_int64(), C.c_int64()
    _check(ctx, load().dpd_wall_carve(ctx, int(wall_species), C.byref(nf), C.byref(nr)))
    return nf.value, nr.value


def dpd_wall_sdf(ctx, x):
    x = np.ascontiguousarray(x, np.float32).reshape(-1, 3)
    out = np.empty(len(x), np.float32)
    _check(ctx, load().dpd_wall_sdf(ctx, len(x), _ptr(x), _ptr(out)))
    return out


def dpd_step(ctx, nsteps):
    _check(ctx, load().dpd_step(ctx, int(nsteps)))


def dpd_step_async(ctx, nsteps):
    _check(ctx, load().dpd_step_async(ctx, int(nsteps)))


def dpd_sync(ctx):
    _check(ctx, load().dpd_sync(ctx))


def dpd_get_count(ctx):
    """Current local count (synchronises first: migration changes it on the device)."""
    _check(ctx, load().dpd_sync(ctx))
    n = C.c_int64()
    _check(ctx, load().dpd_get_count(ctx, C.byref(n)))
    return n.value


def dpd_get_step(ctx):
    s = C.c_int64()
    _check(ctx, load().dpd_get_step(ctx, C.byref(s)))
    return s.value


def dpd_get_grid(ctx):
    d = (C.c_int32 * 3)()
    _check(ctx, load().dpd_get_grid(ctx, d))
    return tuple(d)


def dpd_get_particles(ctx, pos=None, vel=None):
    n = dpd_get_count(ctx)
    pos = np.empty((n, 3), np.float32) if pos is None else pos
    vel = np.empty((n, 3), np.float32) if vel is None else vel
    _check(ctx, load().dpd_get_particles(ctx, n, _ptr(pos), _ptr(vel)))
    return pos, vel


def dpd_get_forces(ctx, f=None):
    n = dpd_get_count(ctx)
    f = np.empty((n, 3), np.float32) if f is None else f
    _check(ctx, load().dpd_get_forces(ctx, n, _ptr(f)))
    return f


def dpd_get_state(ctx):
    n = dpd_get_count(ctx)
    pos, u, f = (np.empty((n, 3), np.float32) for _ in range(3))
    ids = np.empty(n, np.int32)
    cnt = C.c_int64()
    _check(ctx, load().dpd_get_state(ctx, n, _ptr(pos), _ptr(u), _ptr(f), _ptr(ids), C.byref(cnt)))
    return pos, u, f, ids


def dpd_debug_cells(ctx, with_cells=True):
    n = dpd_get_count(ctx)
    nd = dpd_get_grid(ctx)
    ncell = nd[0] * nd[1] * nd[2]
    cell = np.empty(n, np.int32) if with_cells else None
    count = np.empty(ncell, np.int32)
    start = np.empty(ncell + 1, np.int32)
    _check(ctx, load().dpd_debug_cells(ctx, _ptr(cell), _ptr(count), _ptr(start)))
    return cell, count, start


def dpd_debug_pairs(ctx, cap=None):
    if cap is None:
        cap = max(64, dpd_get_count(ctx) * 64)
    quad = np.empty((cap, 4), np.uint32)
    npairs = C.c_int64()
    _check(ctx, load().dpd_debug_pairs(ctx, cap, _ptr(quad), C.byref(npairs)))
    if npairs.value > cap:
        return dpd_debug_pairs(ctx, int(npairs.value))
    return quad[: npairs.value].copy()


def dpd_set_timing(ctx, enable):
    _check(ctx, load().dpd_set_timing(ctx, int(bool(enable))))


def dpd_get_timing(ctx):
    """Per-kernel (total_ms, launches) since timing was enabled, keyed by kernel name."""
    L = load()
    out = {}
    k = 0
    while True:
        name = L.dpd_kernel_name(k)
        if name is None:
            break
        ms, nl = C.c_double(), C.c_int64()
        _check(ctx, L.dpd_get_timing(ctx, k, C.byref(ms), C.byref(nl)))
        out[name.decode()] = (ms.value, nl.value)
        k += 1
    return out


def dpd_get_launch_count(ctx):
    n = C.c_int64()
    _check(ctx, load().dpd_get_launch_count(ctx, C.byref(n)))
    return n.value


def dpd_debug_philox(ctr, key):
    """Device Philox2x32-10: ctr (n, 2), key (n,) -> (n, 2)."""
    ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 2)
    key = np.ascontiguousarray(key, np.uint32).reshape(-1)
    out = np.empty_like(ctr)
    code = load().dpd_debug_philox(ctr.shape[0], _ptr(ctr), _ptr(key), _ptr(out))
    if code != DPD_OK:
        raise DPDError(code, "dpd_debug_philox")
    return out


def dpd_debug_pair_words(quads, seed):
    q = np.ascontiguousarray(quads, np.uint32).reshape(-1, 4)
    words = np.empty((q.shape[0], 2), np.uint32)
    xi = np.empty(q.shape[0], np.float32)
    code = load().dpd_debug_pair_words(q.shape[0], _ptr(q), int(seed), _ptr(words), _ptr(xi))
    if code != DPD_OK:
        raise DPDError(code, "dpd_debug_pair_words")
    return words, xi


# ---- NEXT-4: asynchronous dumps, the step schedule, task graph and I/O queue ----------------
def dpd_dump_open(ctx, path_prefix, queue_depth=4):
    _check(ctx, load().dpd_dump_open(ctx, os.fsencode(path_prefix), int(queue_depth)))


def dpd_dump_every(ctx, every):
    _check(ctx, load().dpd_dump_every(ctx, int(every)))


def dpd_dump_now(ctx):
    _check(ctx, load().dpd_dump_now(ctx))


def dpd_dump_close(ctx):
    """Drain and join the writer; returns the number of snapshots written."""
    n = C.c_int64()
    _check(ctx, load().dpd_dump_close(ctx, C.byref(n)))
    return n.value


def dpd_step_schedule(ctx, with_dump=False):
    """[(stream slot, task name, [predecessors])] in issue order."""
    buf = C.create_string_buffer(8192)
    _check(ctx, load().dpd_step_schedule(ctx, int(bool(with_dump)), buf, len(buf)))
    out = []
    for line in buf.value.decode().splitlines():
        head, _, preds = line.partition(" <- ")
        slot, name = head.split(" ", 1)
        out.append((int(slot), name, preds.split(",") if preds else []))
    return out


def read_dump(path):
    """Read one snapshot file (layout in include/dpd.h) -> dict of numpy arrays."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:8] != b"DPDSNAP1":
        raise ValueError(f"{path}: not a DPD snapshot")
    n, step, rank = np.frombuffer(raw, np.int64, 3, 8)
    box = np.frombuffer(raw, np.float64, 3, 32)
    origin = np.frombuffer(raw, np.float64, 3, 56)
    o = 80
    pos = np.frombuffer(raw, np.float32, 3 * n, o).reshape(n, 3)
    vel = np.frombuffer(raw, np.float32, 3 * n, o + 12 * n).reshape(n, 3)
    ids = np.frombuffer(raw, np.int32, n, o + 24 * n)
    return {"n": int(n), "step": int(step), "rank": int(rank), "box": box.copy(), "origin": origin.copy(),
            "pos": pos.copy(), "vel": vel.copy(), "ids": ids.copy()}


class TaskGraph:
    """Host-side Kahn scheduler of the step (dpd_tg_*): add(name, slot) -> id, edge(a, b), order()."""

    def __init__(self):
        self.h = C.c_void_p()
        code = load().dpd_tg_create(C.byref(self.h))
        if code != DPD_OK:
            raise DPDError(code, "dpd_tg_create")

    def __del__(self):
        if getattr(self, "h", None):
            load().dpd_tg_destroy(self.h)
            self.h = None

    def add(self, name, slot=0):
        i = C.c_int32()
        code = load().dpd_tg_add(self.h, name.encode(), int(slot), C.byref(i))
        if code != DPD_OK:
            raise DPDError(code, "dpd_tg_add")
        return i.value

    def edge(self, before, after):
        code = load().dpd_tg_edge(self.h, int(before), int(after))
        if code != DPD_OK:
            raise DPDError(code, "dpd_tg_edge")

    def order(self):
        n = C.c_int64()
        buf = np.empty(4096, np.int32)
        code = load().dpd_tg_order(self.h, len(buf), _ptr(buf), C.byref(n))
        if code != DPD_OK:
            raise DPDError(code, "dpd_tg_order: cycle" if code == DPD_ERR_CONFIG else "dpd_tg_order")
        return buf[: n.value].tolist()


class IoQueue:
    """Host-side bounded writer (dpd_ioq_*): write(path, bytes, delay_us) / pending() / close()."""

    def __init__(self, depth=4):
        self.h = C.c_void_p()
        code = load().dpd_ioq_create(int(depth), C.byref(self.h))
        if code != DPD_OK:
            raise DPDError(code, "dpd_ioq_create")

    def write(self, path, data, delay_us=0):
        buf = np.frombuffer(bytes(data), np.uint8)
        code = load().dpd_ioq_write(self.h, os.fsencode(path), _ptr(buf) if len(buf) else None, len(buf),
                                    int(delay_us))
        if code != DPD_OK:
            raise DPDError(code, load().dpd_ioq_last_error(self.h).decode())

    def pending(self):
        n = C.c_int64()
        load().dpd_ioq_pending(self.h, C.byref(n))
        return n.value

    def close(self):
        """Drain, join, free; returns the number of completed writes."""
        n = C.c_int64()
        h, self.h = self.h, None
        code = load().dpd_ioq_close(h, C.byref(n))
        if code != DPD_OK:
            raise DPDError(code, "a queued write failed")
        return n.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                self.close()
            except Exception:
                pass


class DPD:
    """Convenience owner of one context (same calls, RAII)."""

    def __init__(self, box, rc=1.0, a=25.0, gamma=45.0, kT=1.0, power=0.5, dt=0.01, seed=42):
        self.ctx = dpd_create(box, rc, a, gamma, kT, power, dt, seed)

    def __del__(self):
        if getattr(self, "ctx", None):
            try:
                dpd_destroy(self.ctx)
            except Exception:
                pass
            self.ctx = None

    def __getattr__(self, name):
        fn = globals().get("dpd_" + name)
        if fn is None:
            raise AttributeError(name)
        return lambda *a, **k: fn(self.ctx, *a, **k)


def dpd_nccl_unique_id():
    buf = np.zeros(128, np.uint8)
    code = load().dpd_nccl_unique_id(_ptr(buf))
    if code != DPD_OK:
        raise DPDError(code, "dpd_nccl_unique_id")
    return buf


def dpd_create_dist(box, rc, a, gamma, kT, power, dt, seed, rank, world, grid, nccl_id):
    L = load()
    b = (C.c_double * 3)(*[float(x) for x in box])
    g = (C.c_int32 * 3)(*[int(x) for x in grid])
    uid = np.ascontiguousarray(nccl_id, np.uint8)
    out = C.c_void_p()
    code = L.dpd_create_dist(b, rc, a, gamma, kT, power, dt, int(seed), int(rank), int(world), g, _ptr(uid),
                             C.byref(out))
    if code != DPD_OK:
        raise DPDError(code, "dpd_create_dist failed (see stderr)")
    return out


def dpd_create_loopback(box, rc, a, gamma, kT, power, dt, seed, split, nccl_id=None):
    L = load()
    b = (C.c_double * 3)(*[float(x) for x in box])
    sp = (C.c_int32 * 3)(*[int(x) for x in split])
    uid = np.ascontiguousarray(dpd_nccl_unique_id() if nccl_id is None else nccl_id, np.uint8)
    out = C.c_void_p()
    code = L.dpd_create_loopback(b, rc, a, gamma, kT, power, dt, int(seed), sp, _ptr(uid), C.byref(out))
    if code != DPD_OK:
        raise DPDError(code, "dpd_create_loopback failed (see stderr)")
    return out


def dpd_create_group(box, rc, a, gamma, kT, power, dt, seed, grid):
    L = load()
    b = (C.c_double * 3)(*[float(x) for x in box])
    g = (C.c_int32 * 3)(*[int(x) for x in grid])
    nctx = int(grid[0]) * int(grid[1]) * int(grid[2])
    out = (C.c_void_p * nctx)()
    code = L.dpd_create_group(b, rc, a, gamma, kT, power, dt, int(seed), g, out)
    if code != DPD_OK:
        raise DPDError(code, "dpd_create_group failed (see stderr)")
    return [C.c_void_p(out[k]) for k in range(nctx)]


def dpd_group_step(ctxs, nsteps):
    arr = (C.c_void_p * len(ctxs))(*[c.value for c in ctxs])
    code = load().dpd_group_step(arr, len(ctxs), int(nsteps))
    if code != DPD_OK:
        msg = " | ".join(load().dpd_last_error(c).decode() for c in ctxs)
        raise DPDError(code, msg)


def dpd_get_particles_ex(ctx, pos=None, vel=None, ids=None):
    """Local particles in storage order (global coordinates, full-step v, global ids)."""
    n = dpd_get_count(ctx)
    pos = np.empty((n, 3), np.float32) if pos is None else pos
    vel = np.empty((n, 3), np.float32) if vel is None else vel
    ids = np.empty(n, np.int32) if ids is None else ids
    cnt = C.c_int64()
    cap = int(pos.shape[0])
    _check(ctx, load().dpd_get_particles_ex(ctx, cap, _ptr(pos), _ptr(vel), _ptr(ids), C.byref(cnt)))
    k = cnt.value
    return pos[:k], vel[:k], ids[:k]


def dpd_get_forces_ex(ctx, f=None, ids=None):
    n = dpd_get_count(ctx)
    f = np.empty((n, 3), np.float32) if f is None else f
    ids = np.empty(n, np.int32) if ids is None else ids
    cnt = C.c_int64()
    _check(ctx, load().dpd_get_forces_ex(ctx, int(f.shape[0]), _ptr(f), _ptr(ids), C.byref(cnt)))
    return f[: cnt.value], ids[: cnt.value]


def dpd_get_species(ctx, out=None):
    """Species index per particle in id order (dense ids)."""
    n = dpd_get_count(ctx)
    out = np.empty(n, np.int32) if out is None else out
    _check(ctx, load().dpd_get_species(ctx, n, _ptr(out)))
    return out


def dpd_get_species_ex(ctx, species=None, ids=None):
    """Species and ids of the local particles in storage order."""
    n = dpd_get_count(ctx)
    species = np.empty(n, np.int32) if species is None else species
    ids = np.empty(n, np.int32) if ids is None else ids
    cnt = C.c_int64()
    _check(ctx, load().dpd_get_species_ex(ctx, int(species.shape[0]), _ptr(species), _ptr(ids), C.byref(cnt)))
    return species[: cnt.value], ids[: cnt.value]


def dpd_plan_peers(grid, rank):
    """(peer_to[27], peer_from[27], used[27]) of `rank` on the rank grid (host only)."""
    g = (C.c_int32 * 3)(*[int(x) for x in grid])
    to = np.zeros(27, np.int32)
    fr = np.zeros(27, np.int32)
    us = np.zeros(27, np.int32)
    code = load().dpd_plan_peers(g, int(rank), _ptr(to), _ptr(fr), _ptr(us))
    if code != DPD_OK:
        raise DPDError(code, "dpd_plan_peers")
    return to, fr, us.astype(bool)

"""CPU oracle for the Mirheo DPD solvent step (arXiv:1911.04712) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It is a ctypes wrapper (marshalling
only) around ``dpd_oracle.c``, a plain fp64 C program that shares no code with the CUDA
path in ``paper_1911_04712_b200/``.  Each function cites the PAPER.md passage (P:n) or
the DESIGN.md reading (C-n) it follows; the pins live in ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dpd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# DPD_ORACLE_NATIVE=1 (bench.py's CPU-timing legs only): the same source built -O3
# -march=native for the host it runs on, as a separate library next to the parity build
NATIVE = os.environ.get("DPD_ORACLE_NATIVE", "0") == "1"
_LIB_NATIVE = os.path.join(_HERE, "liboracle_native.so")
FLAGS = ["-O3", "-march=native"] if NATIVE else ["-O2"]


def build(force: bool = False) -> str:
    """Compile dpd_oracle.c with gcc (-O2, OpenMP; -O3 -march=native under DPD_ORACLE_NATIVE=1).
    Building the checker is not using it."""
    out = _LIB_NATIVE if NATIVE else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        cmd = ["gcc", *FLAGS, "-std=c11", "-D_DEFAULT_SOURCE", "-fopenmp", "-fPIC", "-shared",
               "-Wall", "-Wextra", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, out)
    return out


class Params(C.Structure):
    """Mirror of ``oracle_params`` in dpd_oracle.c."""
    _fields_ = [("box", C.c_double * 3), ("rc", C.c_double), ("a", C.c_double),
                ("gamma", C.c_double), ("kT", C.c_double), ("power", C.c_double),
                ("dt", C.c_double), ("seed", C.c_uint64), ("body_f", C.c_double),
                ("nspecies", C.c_int32), ("amat", C.c_double * 16), ("gmat", C.c_double * 16),
                ("species", C.POINTER(C.c_int32)),
                ("nwall", C.c_int32), ("wtype", C.c_int32 * 4), ("wprm", C.c_double * 16),
                ("wvel", C.c_double * 12), ("frozen_mask", C.c_int32), ("body_mode", C.c_int32)]


@dataclass
class DPDParams:
    box: tuple
    rc: float = 1.0
    a: float = 25.0
    gamma: float = 45.0
    kT: float = 1.0
    power: float = 0.5
    dt: float = 0.01
    seed: int = 42
    body_f: float = 0.0
    # NEXT-2 species matrices (ns x ns, symmetric) and per-particle species (index order);
    # None = single species (a, gamma)
    amat: object = None
    gmat: object = None
    species: object = None
    # NEXT-3 walls: list of (type, (p0, p1, p2, p3), (uwx, uwy, uwz)); type 1 plane
    # s = n.x - c with (n, c); 2/3/4 cylinder along x/y/z with (c1, c2, R, sign)
    walls: object = None
    frozen_mask: int = 0
    body_mode: int = 0  # 0 periodic Poiseuille, 1 uniform +f along z

    def c(self) -> Params:
        p = Params()
        for k in range(3):
            p.box[k] = float(self.box[k])
        p.rc, p.a, p.gamma, p.kT = float(self.rc), float(self.a), float(self.gamma), float(self.kT)
        p.power, p.dt, p.seed, p.body_f = float(self.power), float(self.dt), int(self.seed), float(self.body_f)
        if self.amat is not None:
            A = np.asarray(self.amat, np.float64)
            G = np.asarray(self.gmat, np.float64)
            ns = A.shape[0]
            if A.shape != (ns, ns) or G.shape != (ns, ns) or ns > 4:
                raise ValueError("species matrices must be square, equal, <= 4 x 4")
            p.nspecies = ns
            for k, val in enumerate(A.ravel()):
                p.amat[k] = float(val)
            for k, val in enumerate(G.ravel()):
                p.gmat[k] = float(val)
        if self.species is not None:
            self._sp = np.ascontiguousarray(self.species, np.int32)  # kept alive with p
            p.species = self._sp.ctypes.data_as(C.POINTER(C.c_int32))
        if self.walls:
            if len(self.walls) > 4:
                raise ValueError("at most 4 wall primitives")
            p.nwall = len(self.walls)
            for k, (t, prm, uw) in enumerate(self.walls):
                p.wtype[k] = int(t)
                for c in range(4):
                    p.wprm[4 * k + c] = float(prm[c])
                for c in range(3):
                    p.wvel[3 * k + c] = float(uw[c])
        p.frozen_mask = int(self.frozen_mask)
        p.body_mode = int(self.body_mode)
        return p


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        d, u32, i64, dp = C.c_double, C.c_uint32, C.c_int64, P(C.c_double)
        L.oracle_philox4x32_10.argtypes = [P(u32), P(u32), P(u32)]
        L.oracle_philox2x32_10.argtypes = [P(u32), u32, P(u32)]
        L.oracle_step_key.argtypes = [C.c_uint64, i64]
        L.oracle_step_key.restype = u32
        L.oracle_fmix32.argtypes = [u32]
        L.oracle_fmix32.restype = u32
        L.oracle_step_keys.argtypes = [C.c_uint64, i64, i64, P(u32)]
        L.oracle_pair_words.argtypes = [C.c_uint64, i64, u32, u32, P(u32)]
        L.oracle_xi.argtypes = [u32, u32]
        L.oracle_xi.restype = d
        L.oracle_pair_force.argtypes = [P(Params), dp, dp, u32, u32, i64, dp, dp]
        L.oracle_pair_force.restype = C.c_int
        L.oracle_min_image.argtypes = [P(Params), dp, dp, dp]
        L.oracle_forces.argtypes = [P(Params), i64, dp, dp, P(u32), i64, d, d, dp, dp, P(i64)]
        L.oracle_forces_subset.argtypes = [P(Params), i64, dp, dp, P(u32), i64, d, d, i64, P(i64), dp, dp]
        L.oracle_pairs.argtypes = [P(Params), i64, dp, P(u32), i64, d, d, i64, P(u32), P(C.c_uint8)]
        L.oracle_pairs.restype = i64
        L.oracle_grid_dims.argtypes = [P(Params), P(C.c_int32)]
        L.oracle_cells.argtypes = [P(Params), i64, P(C.c_float), P(C.c_int32), P(C.c_int32), P(C.c_int32)]
        L.oracle_prime.argtypes = [P(Params), i64, dp, dp, P(u32), i64, dp]
        L.oracle_step.argtypes = [P(Params), i64, dp, dp, dp, P(u32), P(i64), i64, dp]
        L.oracle_temperature.argtypes = [i64, dp]
        L.oracle_temperature.restype = d
        L.oracle_virial.argtypes = [P(Params), i64, dp]
        L.oracle_virial.restype = d
        L.oracle_forces_celllist.argtypes = [P(Params), i64, dp, dp, P(u32), i64, dp, P(i64)]
        L.oracle_forces_celllist.restype = C.c_int
        L.oracle_step_celllist.argtypes = [P(Params), i64, dp, dp, dp, P(u32), P(i64), i64]
        L.oracle_step_celllist.restype = C.c_int
        L.oracle_num_threads.restype = C.c_int
        L.oracle_set_num_threads.argtypes = [C.c_int]
        L.oracle_wall_sdf.argtypes = [P(Params), dp, dp]
        L.oracle_wall_sdf.restype = d
        L.oracle_kick_drift.argtypes = [P(Params), i64, dp, dp, dp, d]
        L.oracle_kick_drift.restype = i64
        L.oracle_wall_carve.argtypes = [P(Params), i64, dp, dp, P(C.c_int32), C.c_int32, P(C.c_uint8)]
        L.oracle_wall_carve.restype = i64
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ids(n, ids):
    if ids is None:
        return np.arange(n, dtype=np.uint32)
    return np.ascontiguousarray(ids, dtype=np.uint32)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def philox4x32_10(ctr, key):
    """Philox4x32-10 (C-7).  ctr: 4 uint32, key: 2 uint32 -> 4 uint32."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(o, C.c_uint32))
    return o


def philox2x32_10(ctr, key: int):
    """Philox2x32-10 (C-7).  ctr: 2 uint32, key: uint32 -> 2 uint32."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    o = np.zeros(2, dtype=np.uint32)
    lib().oracle_philox2x32_10(_p(c, C.c_uint32), int(key) & 0xFFFFFFFF, _p(o, C.c_uint32))
    return o


def fmix32(h: int) -> int:
    """MurmurHash3's 32-bit finalizer, a bijection of the 32-bit words (C-7)."""
    return int(lib().oracle_fmix32(int(h) & 0xFFFFFFFF))


def step_key(seed: int, step: int) -> int:
    """k_s = fmix32(s_lo ^ seed_lo ^ fmix32(s_hi)) ^ seed_hi (C-7, round-2 revision)."""
    return int(lib().oracle_step_key(int(seed), int(step)))


def step_keys(seed: int, s0: int, n: int) -> np.ndarray:
    """Step keys of steps s0 .. s0 + n - 1 (uint32 array)."""
    o = np.zeros(int(n), dtype=np.uint32)
    lib().oracle_step_keys(int(seed), int(s0), int(n), _p(o, C.c_uint32))
    return o


def pair_words(seed: int, step: int, ida: int, idb: int):
    """(w0, w1) = Philox2x32-10(ctr={min id, max id}, key=k_s) (C-7)."""
    o = np.zeros(2, dtype=np.uint32)
    lib().oracle_pair_words(int(seed), int(step), int(ida), int(idb), _p(o, C.c_uint32))
    return int(o[0]), int(o[1])


def xi(w0: int, w1: int) -> float:
    """Box-Muller Gaussian from two words (C-7)."""
    return float(lib().oracle_xi(int(w0), int(w1)))


def pair_force(p: DPDParams, d, vij, ida: int, idb: int, step: int):
    """Force on i from j for separation d = r_i - r_j and v_ij.
    Returns (f[3], interacting, xi)."""
    dd, vv = _f64(d), _f64(vij)
    f = np.zeros(3)
    x = C.c_double(0.0)
    pc = p.c()
    hit = lib().oracle_pair_force(C.byref(pc), _p(dd, C.c_double), _p(vv, C.c_double),
                                  int(ida), int(idb), int(step), _p(f, C.c_double), C.byref(x))
    return f, bool(hit), x.value


def min_image(p: DPDParams, xi_, xj_):
    a, b, d = _f64(xi_), _f64(xj_), np.zeros(3)
    pc = p.c()
    lib().oracle_min_image(C.byref(pc), _p(a, C.c_double), _p(b, C.c_double), _p(d, C.c_double))
    return d


def forces(p: DPDParams, x, v, step: int, ids=None, *, eps: float = 0.0, eps_image=None):
    """PairForces(x, v, s): O(N^2) minimum-image sum (C-1, C-2 item 4).
    Returns (F[n,3], allow[n], npairs); allow = boundary-pair allowance (C-12) over pairs
    within eps of r_c (eps_image, default eps, for pairs across a periodic edge)."""
    eps_image = eps if eps_image is None else eps_image
    x, v = _f64(x), _f64(v)
    n = x.shape[0]
    ids = _ids(n, ids)
    F = np.zeros((n, 3))
    allow = np.zeros(n)
    npairs = C.c_int64(0)
    pc = p.c()
    lib().oracle_forces(C.byref(pc), n, _p(x, C.c_double), _p(v, C.c_double), _p(ids, C.c_uint32),
                        int(step), float(eps), float(eps_image), _p(F, C.c_double), _p(allow, C.c_double),
                        C.byref(npairs))
    return F, allow, int(npairs.value)


def forces_subset(p: DPDParams, x, v, step: int, sel, ids=None, *, eps: float = 0.0, eps_image=None):
    """PairForces for the selected particles only (same all-j sum).  Returns (F[m,3], allow[m])."""
    eps_image = eps if eps_image is None else eps_image
    x, v = _f64(x), _f64(v)
    n = x.shape[0]
    ids = _ids(n, ids)
    sel = np.ascontiguousarray(sel, dtype=np.int64)
    m = sel.shape[0]
    F = np.zeros((m, 3))
    allow = np.zeros(m)
    pc = p.c()
    lib().oracle_forces_subset(C.byref(pc), n, _p(x, C.c_double), _p(v, C.c_double), _p(ids, C.c_uint32),
                               int(step), float(eps), float(eps_image), m, _p(sel, C.c_int64), _p(F, C.c_double),
                               _p(allow, C.c_double))
    return F, allow


def forces_celllist(p: DPDParams, x, v, step: int, ids=None):
    """CPU-timing mode: same arithmetic over 27 neighbour cells (C-2 item 7)."""
    x, v = _f64(x), _f64(v)
    n = x.shape[0]
    ids = _ids(n, ids)
    F = np.zeros((n, 3))
    npairs = C.c_int64(0)
    pc = p.c()
    rc = lib().oracle_forces_celllist(C.byref(pc), n, _p(x, C.c_double), _p(v, C.c_double),
                                      _p(ids, C.c_uint32), int(step), _p(F, C.c_double), C.byref(npairs))
    if rc != 0:
        raise ValueError(f"oracle_forces_celllist failed ({rc}); grid needs n_d >= 3")
    return F, int(npairs.value)


def pairs(p: DPDParams, x, step: int, ids=None, *, eps: float = 0.0, cap: int | None = None, eps_image=None):
    """Interacting or boundary pairs: returns (quad[k,4] = lo, hi, w0, w1; flag[k]) (T3)."""
    eps_image = eps if eps_image is None else eps_image
    x = _f64(x)
    n = x.shape[0]
    ids = _ids(n, ids)
    pc = p.c()
    if cap is None:
        cap = max(16, int(n * 40))
    quad = np.zeros((cap, 4), dtype=np.uint32)
    flag = np.zeros(cap, dtype=np.uint8)
    k = lib().oracle_pairs(C.byref(pc), n, _p(x, C.c_double), _p(ids, C.c_uint32), int(step),
                           float(eps), float(eps_image), cap, _p(quad, C.c_uint32), _p(flag, C.c_uint8))
    if k > cap:
        return pairs(p, x, step, ids, eps, cap=int(k), eps_image=eps_image)
    return quad[:k].copy(), flag[:k].copy()


def grid_dims(p: DPDParams):
    dims = np.zeros(3, dtype=np.int32)
    pc = p.c()
    lib().oracle_grid_dims(C.byref(pc), _p(dims, C.c_int32))
    return tuple(int(v) for v in dims)


def cells(p: DPDParams, pos):
    """Cell of each particle, counts and exclusive starts, fp32 arithmetic (C-8)."""
    pos = np.ascontiguousarray(pos, dtype=np.float32)
    n = pos.shape[0]
    nd = grid_dims(p)
    ncell = nd[0] * nd[1] * nd[2]
    cell = np.zeros(n, dtype=np.int32)
    count = np.zeros(ncell, dtype=np.int32)
    start = np.zeros(ncell + 1, dtype=np.int32)
    pc = p.c()
    lib().oracle_cells(C.byref(pc), n, _p(pos, C.c_float), _p(cell, C.c_int32), _p(count, C.c_int32),
                       _p(start, C.c_int32))
    return cell, count, start


def temperature(v) -> float:
    v = _f64(v)
    return float(lib().oracle_temperature(v.shape[0], _p(v, C.c_double)))


def virial(p: DPDParams, x) -> float:
    x = _f64(x)
    pc = p.c()
    return float(lib().oracle_virial(C.byref(pc), x.shape[0], _p(x, C.c_double)))


class State:
    """Oracle trajectory state (x, v full-step, F, ids, s) advanced by GW-VV (C-2 item 3)."""

    def __init__(self, p: DPDParams, x, v, ids=None, step0: int = 0, celllist: bool = False):
        self.p = p
        self.x = _f64(x).copy()
        self.v = _f64(v).copy()
        n = self.x.shape[0]
        self.ids = _ids(n, ids).copy()
        self.s = int(step0)
        self.celllist = celllist
        self.F = np.zeros((n, 3))
        self.u = self.v.copy()
        pc = p.c()
        if celllist:
            self.F, _ = forces_celllist(p, self.x, self.v, self.s, self.ids)
        else:
            lib().oracle_prime(C.byref(pc), n, _p(self.x, C.c_double), _p(self.v, C.c_double),
                               _p(self.ids, C.c_uint32), self.s, _p(self.F, C.c_double))

    def step(self, k: int = 1):
        n = self.x.shape[0]
        s = C.c_int64(self.s)
        pc = self.p.c()
        if self.celllist:
            rc = lib().oracle_step_celllist(C.byref(pc), n, _p(self.x, C.c_double), _p(self.v, C.c_double),
                                            _p(self.F, C.c_double), _p(self.ids, C.c_uint32), C.byref(s), int(k))
            if rc != 0:
                raise RuntimeError(f"oracle_step_celllist failed ({rc})")
        else:
            lib().oracle_step(C.byref(pc), n, _p(self.x, C.c_double), _p(self.v, C.c_double),
                              _p(self.F, C.c_double), _p(self.ids, C.c_uint32), C.byref(s), int(k),
                              _p(self.u, C.c_double))
        self.s = int(s.value)
        return self


def wall_sdf(p: DPDParams, x):
    """s(x) = max over the wall primitives (C-23) and the wall velocity there, per row."""
    x = _f64(np.atleast_2d(x))
    pc = p.c()
    s = np.empty(len(x))
    uw = np.empty((len(x), 3))
    for i in range(len(x)):
        row = np.ascontiguousarray(x[i])
        s[i] = lib().oracle_wall_sdf(C.byref(pc), _p(row, C.c_double), _p(uw[i], C.c_double))
    return s, uw


def kick_drift(p: DPDParams, x, v, F, kick: float):
    """One kick-drift with bounce-back (C-6, C-23); returns (x', u', bounces)."""
    x, v, F = _f64(x).copy(), _f64(v).copy(), _f64(F)
    pc = p.c()
    nb = lib().oracle_kick_drift(C.byref(pc), x.shape[0], _p(x, C.c_double), _p(v, C.c_double),
                                 _p(F, C.c_double), float(kick))
    return x, v, int(nb)


def wall_carve(p: DPDParams, x, v, species, wall_species: int):
    """Frozen layer (C-23): returns (keep mask, v', species', n_frozen)."""
    x, v = _f64(x), _f64(v).copy()
    sp = np.ascontiguousarray(species, np.int32).copy()
    keep = np.zeros(x.shape[0], np.uint8)
    pc = p.c()
    nf = lib().oracle_wall_carve(C.byref(pc), x.shape[0], _p(x, C.c_double), _p(v, C.c_double),
                                 _p(sp, C.c_int32), int(wall_species), _p(keep, C.c_uint8))
    return keep.astype(bool), v, sp, int(nf)

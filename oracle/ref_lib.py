"""ctypes binding of ``oracle/_ref/libbbsi_ref.so`` (the compiled, unmodified reference).

TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py reference arm). Build recipe:
``oracle/ref/Makefile``. Matrices cross in slot order, see ``ref_driver.cpp``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import bbsi_oracle as O

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libbbsi_ref.so"
# the same unmodified reference linked against scipy's OpenBLAS 0.3.31 (oracle/ref/Makefile):
# only its BLAS rounding differs, so its distance to LIB_PATH is the reference's own floor
SCIPY_LIB_PATH = HERE / "_ref" / "libbbsi_ref_scipy.so"
_lib = None
_lib_scipy = None


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle/ref` (needs /root/reference)")
        _lib = C.CDLL(str(LIB_PATH))
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def lib_scipy():
    global _lib_scipy
    if _lib_scipy is None:
        if not SCIPY_LIB_PATH.exists():
            raise FileNotFoundError(f"{SCIPY_LIB_PATH} missing: run `make -C oracle/ref`")
        _lib_scipy = C.CDLL(str(SCIPY_LIB_PATH))
        _lib_scipy.ref_last_error.restype = C.c_char_p
    return _lib_scipy


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def to_slots(band: O.Band) -> np.ndarray:
    """(l, 2w+1, bs, bs) row/col array -> column-major slot memory (complex128)."""
    return np.ascontiguousarray(band.data.transpose(0, 1, 3, 2))


def from_slots(layout: O.BlockLayout, mem: np.ndarray) -> O.Band:
    return O.Band(layout, np.ascontiguousarray(mem.transpose(0, 1, 3, 2)))


def _sizes(layout):
    return np.array(layout.block_sizes, dtype=np.int32)


def _check(rc, fail):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 1:
        raise O.InvalidArgumentError(msg)
    if rc == 2:
        raise O.SingularMatrixError(msg, int(fail.value))
    raise RuntimeError(msg)


def set_threads(n: int):
    lib().ref_set_threads(C.c_int(n))


def _gen(fn, layout, seed, dominance):
    l, w, bs = layout.num_layers, layout.bandwidth, layout.bs
    mem = np.zeros((l, 2 * w + 1, bs, bs), dtype=np.complex128)
    sz = _sizes(layout)
    rc = fn(l, w, bs, _p(sz), C.c_uint64(seed), C.c_double(dominance), _p(mem))
    _check(rc, C.c_int(-1))
    return from_slots(layout, mem)


def random_spd_like(layout, seed, dominance):
    return _gen(lib().ref_random_spd_like, layout, seed, dominance)


def random_hermitian(layout, seed, dominance):
    return _gen(lib().ref_random_hermitian, layout, seed, dominance)


def _solve(name, m: O.Band, extra=()):
    lay = m.layout
    l, w, bs = lay.num_layers, lay.bandwidth, lay.bs
    a = to_slots(m)
    g = np.zeros_like(a)
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    sz = _sizes(lay)
    rc = getattr(lib(), name)(l, w, bs, _p(sz), _p(a), _p(g), _p(cnt), *extra, C.byref(fail))
    _check(rc, fail)
    return from_slots(lay, g), O.KernelCounters(*map(int, cnt))


def rgf_tridiag(m):
    return _solve("ref_rgf_tridiag", m)


def rgf_fused(m):
    return _solve("ref_rgf_fused", m)


def rgf_ndiag(m, trace=None):
    mo = C.c_int(0)
    g, c = _solve("ref_rgf_ndiag", m, (C.byref(mo),))
    if trace is not None:
        trace["max_update_offset"] = mo.value
    return g, c


def ddrgf(m: O.Band, s2_levels, n_threads=1, terminal_threads=1):
    lay = m.layout
    l, w, bs = lay.num_layers, lay.bandwidth, lay.bs
    a = to_slots(m)
    g = np.zeros_like(a)
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    s2 = np.array(list(s2_levels), dtype=np.int32)
    rc = lib().ref_ddrgf(l, w, bs, _p(_sizes(lay)), _p(a), _p(s2), len(s2), n_threads, terminal_threads,
                         _p(g), _p(cnt), C.byref(fail))
    _check(rc, fail)
    return from_slots(lay, g), O.KernelCounters(*map(int, cnt))


def rgf_extended(m: O.Band):
    lay = m.layout
    l, w, bs = lay.num_layers, lay.bandwidth, lay.bs
    a = to_slots(m)
    g = np.zeros_like(a)
    halos = [np.zeros((l, bs, bs), dtype=np.complex128) for _ in range(4)]
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    rc = lib().ref_rgf_extended(l, w, bs, _p(_sizes(lay)), _p(a), _p(g), *[_p(h) for h in halos], _p(cnt),
                                C.byref(fail))
    _check(rc, fail)
    ext = O.ExtendedInverse(from_slots(lay, g))
    bsz = lay.block_sizes
    fr, lr, fc, lc = [[h[k].T for k in range(l)] for h in halos]
    ext.first_row = [fr[k][: bsz[0], : bsz[k]] for k in range(l)]
    ext.last_row = [lr[k][: bsz[-1], : bsz[k]] for k in range(l)]
    ext.first_col = [fc[k][: bsz[k], : bsz[0]] for k in range(l)]
    ext.last_col = [lc[k][: bsz[k], : bsz[-1]] for k in range(l)]
    return ext, O.KernelCounters(*map(int, cnt))


def oracle_selected_inverse(m: O.Band):
    lay = m.layout
    l, w, bs = lay.num_layers, lay.bandwidth, lay.bs
    a = to_slots(m)
    g = np.zeros_like(a)
    rc = lib().ref_oracle_selected_inverse(l, w, bs, _p(_sizes(lay)), _p(a), _p(g))
    _check(rc, C.c_int(-1))
    return from_slots(lay, g)


def interleave_permutation(l, s1, s2):
    order = np.zeros(l, dtype=np.int32)
    inter = np.zeros(2 * l + 2, dtype=np.int32)
    sep = np.zeros(2 * l + 2, dtype=np.int32)
    n = lib().ref_interleave_permutation(l, s1, s2, _p(order), _p(inter), _p(sep))
    if n < 0:
        raise O.InvalidArgumentError(lib().ref_last_error().decode())
    return (list(map(int, order)), [(int(inter[2 * t]), int(inter[2 * t + 1])) for t in range(n)],
            [(int(sep[2 * t]), int(sep[2 * t + 1])) for t in range(n)])


def predict_ddrgf_counters(l, s2_levels):
    s2 = np.array(list(s2_levels), dtype=np.int32)
    out = np.zeros(3, dtype=np.int64)
    rc = lib().ref_predict_ddrgf_counters(C.c_longlong(l), _p(s2), len(s2), _p(out))
    _check(rc, C.c_int(-1))
    return O.KernelCounters(*map(int, out))


def write_bbm(path: str, m: O.Band):
    """bbsi::write_bbm (io.cpp:26-45) of the compiled reference."""
    lay = m.layout
    mem = to_slots(m)
    rc = lib().ref_write_bbm(str(path).encode(), lay.num_layers, lay.bandwidth, lay.bs, _p(_sizes(lay)), _p(mem))
    _check(rc, C.c_int(-1))


def read_bbm(path: str) -> O.Band:
    """bbsi::read_bbm (io.cpp:47-73) of the compiled reference."""
    dims = np.zeros(3, dtype=np.int32)
    _check(lib().ref_read_bbm(str(path).encode(), _p(dims), None, 0, None), C.c_int(-1))
    l, w, bs = map(int, dims)
    sizes = np.zeros(l, dtype=np.int32)
    mem = np.zeros((l, 2 * w + 1, bs, bs), dtype=np.complex128)
    _check(lib().ref_read_bbm(str(path).encode(), _p(dims), _p(sizes), l, _p(mem)), C.c_int(-1))
    return from_slots(O.BlockLayout(l, [int(s) for s in sizes], w), mem)


def cost(kind: str, l: int, w: int = 1, s2_levels=(), n_threads=1, terminal_threads=1, r_lu=0.0, r_getrs=0.0,
         t_gemm=1.0, blas_cap=12):
    """cost_rgf / cost_nrgf / cost_fused / cost_ddrgf (cost_model.hpp:67-130): (gemm_eq, seconds)."""
    k = {"rgf": 0, "nrgf": 1, "fused": 2, "ddrgf": 3}[kind]
    s2 = np.array(list(s2_levels) or [1], dtype=np.int32)
    out = np.zeros(2)
    rc = lib().ref_cost(k, C.c_longlong(l), C.c_longlong(w), _p(s2), len(s2_levels), n_threads, terminal_threads,
                        C.c_double(r_lu), C.c_double(r_getrs), C.c_double(t_gemm), blas_cap, _p(out))
    _check(rc, C.c_int(-1))
    return float(out[0]), float(out[1])


def autotune(l, n_threads, r_lu, r_getrs, t_gemm=1.0, max_levels=5, s2_max=4, blas_cap=12):
    """autotune (cost_model.hpp:174-224): dict of the verdict."""
    ints = np.zeros(64, dtype=np.int32)
    dbl = np.zeros(2)
    rc = lib().ref_autotune(C.c_longlong(l), n_threads, C.c_double(r_lu), C.c_double(r_getrs), C.c_double(t_gemm),
                            max_levels, s2_max, blas_cap, _p(ints), 64, _p(dbl))
    _check(rc, C.c_int(-1))
    n = int(ints[2])
    return {"use_rgf": bool(ints[0]), "ddrgf_valid": bool(ints[1]), "s2_levels": [int(x) for x in ints[4:4 + n]],
            "terminal_threads": int(ints[3]), "rgf_gemm_equivalents": float(dbl[0]),
            "ddrgf_gemm_equivalents": float(dbl[1])}

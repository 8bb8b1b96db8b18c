"""ctypes binding of ``oracle/_build/librgf_stream.so`` (oracle/stream/rgf_stream.cpp).

TEST INFRASTRUCTURE ONLY (tests/, tools/parity_full.py): a streaming restatement of
the reference rgf_tridiag (rgf.hpp:37-76) with the reference's own BLAS/LAPACK calls,
for full-size parity where the dense band does not fit next to the GPU result. Blocks
come out one layer at a time, as (row, col) complex128 arrays.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "librgf_stream.so"            # OpenBLAS 0.3.15: bitwise = oracle/_ref
FAST_PATH = HERE / "_build" / "librgf_stream_fast.so"      # scipy OpenBLAS 0.3.31: <= 1e-13 of it
_libs = {}
_use_fast = False


def available() -> bool:
    return LIB_PATH.exists()


def use_fast(on: bool = True):
    """Selects the scipy-OpenBLAS build for subsequent streams (full-size runs)."""
    global _use_fast
    _use_fast = bool(on)


def lib():
    path = FAST_PATH if _use_fast else LIB_PATH
    if path not in _libs:
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle/stream`")
        L = C.CDLL(str(path))
        L.rs_create.restype = C.c_void_p
        L.rs_create.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_int, C.c_double,
                                C.c_uint64, C.c_int]
        L.rs_destroy.argtypes = [C.c_void_p]
        L.rs_set_threads.argtypes = [C.c_int]
        L.rs_upward.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        L.rs_next.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.rs_block.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        _libs[path] = L
    return _libs[path]


class DysonStream:
    """rgf_tridiag of A(E) = z I - H - Sigma (BASELINE Dyson spec, w = 1), streamed.

    pert > 0: every real/imaginary component of A is moved one ulp up or down (at
    random) with probability ``pert`` -- the input-noise floor protocol.
    ckpt: segment length of the recomputing upward sweep (0 = keep all 3l blocks).
    """

    def __init__(self, l, b, seed, z, sigma_layers=1, pert=0.0, pert_seed=0, ckpt=0):
        self.l, self.b = l, b
        self.L = lib()
        self.h = self.L.rs_create(l, b, seed, float(z.real), float(z.imag), sigma_layers, float(pert), pert_seed,
                                 ckpt)
        fail = C.c_int(-1)
        if self.L.rs_upward(self.h, C.byref(fail)) != 0:
            raise RuntimeError(f"singular Schur pivot at layer {fail.value}")
        self._buf = [np.empty((b, b), dtype=np.complex128) for _ in range(3)]

    def __del__(self):
        if getattr(self, "h", None):
            self.L.rs_destroy(self.h)
            self.h = None

    def next(self):
        """(i, G[i,i], G[i-1,i], G[i,i-1]) as (row, col) arrays (views, valid until the next call)."""
        d, u, lo = self._buf
        i = self.L.rs_next(self.h, d.ctypes.data, u.ctypes.data, lo.ctypes.data)
        if i == -2:
            raise RuntimeError("singular Schur pivot (segment recompute)")
        if i < 0:
            return None
        return i, d.T, (u.T if i > 0 else None), (lo.T if i > 0 else None)

    def block(self, a, off):
        m = np.empty((self.b, self.b), dtype=np.complex128)
        self.L.rs_block(self.h, a, off, m.ctypes.data)
        return m.T.copy()


def set_threads(n: int):
    lib().rs_set_threads(n)

"""Accuracy of the sm_100a building blocks against extended-precision references.

GEMM: relative error vs numpy clongdouble (80-bit) products.
Inverse: forward error vs an LU-based inverse and residual ||S X - I|| for matrices
with prescribed condition numbers.
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2))).cuda()


def host(t):
    return np.swapaxes(t.cpu().numpy(), -1, -2)


def main():
    import torch

    from paper_2605_19910_b200._native import lib

    rng = np.random.default_rng(0)
    n = 256
    # ---- GEMM vs extended precision
    a = rng.uniform(-1, 1, (2, n, n)) + 1j * rng.uniform(-1, 1, (2, n, n))
    b = rng.uniform(-1, 1, (2, n, n)) + 1j * rng.uniform(-1, 1, (2, n, n))
    c = np.zeros_like(a)
    da, db, dc = dev(a), dev(b), dev(c)
    alpha, beta = np.array([1.0, 0.0]), np.array([0.0, 0.0])
    lib().bbsi_cuda_zgemm_dev(n, n, n, alpha.ctypes.data_as(C.c_void_p), C.c_void_p(da.data_ptr()), n, n * n,
                              C.c_void_p(db.data_ptr()), n, n * n, beta.ctypes.data_as(C.c_void_p),
                              C.c_void_p(dc.data_ptr()), n, n * n, 2, C.c_void_p(0))
    torch.cuda.synchronize()
    got = host(dc)
    exact = a.astype(np.clongdouble) @ b.astype(np.clongdouble)
    np_prod = a @ b
    for i in range(2):
        e_gpu = float(np.linalg.norm((got[i] - exact[i]).astype(np.complex128)) / np.linalg.norm(exact[i].astype(np.complex128)))
        e_np = float(np.linalg.norm((np_prod[i] - exact[i]).astype(np.complex128)) / np.linalg.norm(exact[i].astype(np.complex128)))
        print(f"zgemm n={n}: gpu rel err {e_gpu:.2e}   numpy/OpenBLAS {e_np:.2e}")
    # ---- inverse at prescribed condition numbers
    for kappa in (1e2, 1e6, 1e10):
        u, _ = np.linalg.qr(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)))
        v, _ = np.linalg.qr(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)))
        s = np.logspace(0, -np.log10(kappa), n)
        S = (u * s) @ v.conj().T
        dS = dev(S[None])
        st = np.zeros(1, np.int32)
        lib().bbsi_cuda_zinv_dev(n, n, 1, C.c_void_p(dS.data_ptr()), n, n * n, st.ctypes.data_as(C.c_void_p),
                                 C.c_void_p(0))
        X = host(dS)[0]
        Xl = np.linalg.inv(S)
        Xe = np.linalg.inv(S.astype(np.clongdouble)) if False else None
        res_gpu = np.linalg.norm(S @ X - np.eye(n)) / np.sqrt(n)
        res_np = np.linalg.norm(S @ Xl - np.eye(n)) / np.sqrt(n)
        resl_gpu = np.linalg.norm(X @ S - np.eye(n)) / np.sqrt(n)
        resl_np = np.linalg.norm(Xl @ S - np.eye(n)) / np.sqrt(n)
        fe = np.linalg.norm(X - Xl) / np.linalg.norm(Xl)
        print(f"zinv n={n} kappa={kappa:.0e}: ||SX-I|| gpu {res_gpu:.2e} lapack {res_np:.2e} | ||XS-I|| gpu {resl_gpu:.2e} "
              f"lapack {resl_np:.2e} | gpu-vs-lapack {fe:.2e}")


if __name__ == "__main__":
    main()

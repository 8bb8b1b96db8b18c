"""Kernel-level parity of the sm_100a building blocks against numpy FP64.

Tolerances follow the reference's dense-kernel tests (tests/test_dense_kernels.cpp:
gemm vs naive <= 1e-13, :25-36; solve/inverse residuals <= 1e-12, :97-134).
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


def _rand(rng, *shape):
    return rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)


def _dev(x):
    torch = _torch()
    # column-major per matrix: store the transpose contiguously
    return torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2))).cuda()


def _host(t):
    return np.swapaxes(t.cpu().numpy(), -1, -2)


@pytest.mark.parametrize("m,n,k,batch", [(64, 64, 16, 1), (128, 192, 64, 3), (256, 256, 256, 4), (64, 128, 768, 2), (32, 96, 48, 2), (100, 70, 32, 1)])
def test_zgemm_matches_numpy(gpu, m, n, k, batch):
    from paper_2605_19910_b200._native import lib

    torch = _torch()
    rng = np.random.default_rng(m + n + k)
    a, b, c = _rand(rng, batch, m, k), _rand(rng, batch, k, n), _rand(rng, batch, m, n)
    alpha, beta = np.array([0.7, -0.3]), np.array([-1.1, 0.2])
    da, db, dc = _dev(a), _dev(b), _dev(c)
    rc = lib().bbsi_cuda_zgemm_dev(m, n, k, alpha.ctypes.data_as(C.c_void_p), C.c_void_p(da.data_ptr()), m, m * k,
                                   C.c_void_p(db.data_ptr()), k, k * n, beta.ctypes.data_as(C.c_void_p),
                                   C.c_void_p(dc.data_ptr()), m, m * n, batch, C.c_void_p(0))
    assert rc == 0
    torch.cuda.synchronize()
    ref = complex(*alpha) * (a @ b) + complex(*beta) * c
    got = _host(dc)
    for i in range(batch):
        err = np.linalg.norm(got[i] - ref[i]) / np.linalg.norm(ref[i])
        assert err <= 1e-13, err


@pytest.mark.parametrize("n,n_true,batch", [(64, 64, 2), (128, 100, 3), (256, 256, 2), (512, 512, 2), (768, 768, 1)])
def test_zinv_matches_numpy(gpu, n, n_true, batch):
    from paper_2605_19910_b200._native import lib

    torch = _torch()
    rng = np.random.default_rng(n)
    a = _rand(rng, batch, n, n)
    a[:, n_true:, :] = 0
    a[:, :, n_true:] = 0
    for i in range(batch):
        a[i, n_true:, n_true:] = np.eye(n - n_true)
    da = _dev(a)
    st = np.zeros(batch, dtype=np.int32)
    rc = lib().bbsi_cuda_zinv_dev(n, n_true, batch, C.c_void_p(da.data_ptr()), n, n * n,
                                  st.ctypes.data_as(C.c_void_p), C.c_void_p(0))
    assert rc == 0
    assert (st == -1).all()
    got = _host(da)
    for i in range(batch):
        ref = np.linalg.inv(a[i])
        err = np.linalg.norm(got[i] - ref) / np.linalg.norm(ref)
        assert err <= 1e-12, err
        res = np.linalg.norm(a[i] @ got[i] - np.eye(n)) / np.sqrt(n)
        assert res <= 1e-11, res


@pytest.mark.parametrize("n,batch", [(128, 3), (256, 5)])
def test_zinv_split_pair_bit_identical(gpu, n, batch, monkeypatch):
    """The pair panel with several CTAs per matrix (BBSI_PANEL_SPLIT; the default for small
    batches) factors every panel redundantly and splits only the V / Wz tails: the result,
    the row interchanges and the singular-pivot status are bit-identical to one CTA."""
    from paper_2605_19910_b200._native import lib

    torch = _torch()
    rng = np.random.default_rng(7 * n + batch)
    a = _rand(rng, batch, n, n)
    a[batch - 1, :, 17] = 0  # exactly singular last matrix
    outs = {}
    monkeypatch.setenv("BBSI_GJ_ROWS", "0")  # the LU + Pinv pair panel (gj_rows_kernel has no split)
    for split in (1, 2, 4, 8):
        monkeypatch.setenv("BBSI_PANEL_SPLIT", str(split))
        da = _dev(a)
        st = np.zeros(batch, dtype=np.int32)
        rc = lib().bbsi_cuda_zinv_dev(n, n, batch, C.c_void_p(da.data_ptr()), n, n * n,
                                      st.ctypes.data_as(C.c_void_p), C.c_void_p(0))
        assert rc == 0
        torch.cuda.synchronize()
        outs[split] = (da.cpu().numpy(), st.copy())
    for split in (2, 4, 8):
        assert np.array_equal(outs[split][1], outs[1][1])
        assert np.array_equal(outs[split][0][: batch - 1].view(np.uint64), outs[1][0][: batch - 1].view(np.uint64))
    assert (outs[1][1][: batch - 1] == -1).all() and outs[1][1][batch - 1] >= 0


@pytest.mark.parametrize("n,n_true,batch", [(64, 64, 3), (128, 100, 3), (192, 192, 2), (256, 256, 5), (320, 300, 2), (512, 512, 3),
                                            (768, 768, 2), (1024, 1000, 2)])
def test_zinv_rows_panel_vs_lu_panel(gpu, n, n_true, batch, monkeypatch):
    """gj_rows_kernel (in-place Gauss-Jordan on register rows, raw pivot rows as the GEMM
    operand; one CTA for n <= 256, a cluster of ceil(n / 256) CTAs up to n = 1024) against the LU + Pinv pair panel (BBSI_GJ_ROWS=0)
    and numpy: same inverse to rounding (inverse <= 1e-12 as tests/test_dense_kernels.cpp:
    97-134), same singular-pivot status."""
    from paper_2605_19910_b200._native import lib

    torch = _torch()
    rng = np.random.default_rng(11 * n + batch)
    a = _rand(rng, batch, n, n)
    a[:, n_true:, :] = 0
    a[:, :, n_true:] = 0
    for i in range(batch):
        a[i, n_true:, n_true:] = np.eye(n - n_true)
    a[batch - 1, :, 9] = 0  # exactly singular last matrix
    outs = {}
    modes = ("4", "0") if n <= 768 else ("4",)  # the LU panels stage n + 2 columns in shared memory: n <= 768
    for mode in modes:
        monkeypatch.setenv("BBSI_GJ_ROWS", mode)
        da = _dev(a)
        st = np.zeros(batch, dtype=np.int32)
        rc = lib().bbsi_cuda_zinv_dev(n, n_true, batch, C.c_void_p(da.data_ptr()), n, n * n,
                                      st.ctypes.data_as(C.c_void_p), C.c_void_p(0))
        assert rc == 0
        torch.cuda.synchronize()
        outs[mode] = (_host(da), st.copy())
    for mode in modes:
        assert (outs[mode][1][: batch - 1] == -1).all() and outs[mode][1][batch - 1] == 9, (mode, outs[mode][1])
    for i in range(batch - 1):
        ref = np.linalg.inv(a[i])
        for mode in modes:
            err = np.linalg.norm(outs[mode][0][i] - ref) / np.linalg.norm(ref)
            assert err <= 1e-12, (mode, err)
        res = np.linalg.norm(a[i] @ outs["4"][0][i] - np.eye(n)) / np.sqrt(n)
        assert res <= 1e-11, res


@pytest.mark.parametrize("n", [128, 256, 512, 768])
def test_zinv_bits_independent_of_batch(gpu, n):
    """A matrix inverts to the same bits alone and inside a larger launch (the panel family
    and the cluster size depend on n only): a solve gives the same result however its
    matrices are grouped into launches (stream groups, ranks, domains)."""
    from paper_2605_19910_b200._native import lib

    torch = _torch()
    rng = np.random.default_rng(n + 1)
    a = _rand(rng, 5, n, n)
    outs = []
    for sel in ([0], [0, 1], [0, 1, 2, 3, 4]):
        da = _dev(a[sel])
        st = np.zeros(len(sel), dtype=np.int32)
        rc = lib().bbsi_cuda_zinv_dev(n, n, len(sel), C.c_void_p(da.data_ptr()), n, n * n,
                                      st.ctypes.data_as(C.c_void_p), C.c_void_p(0))
        assert rc == 0 and (st == -1).all()
        torch.cuda.synchronize()
        outs.append(da.cpu().numpy()[0])
    assert np.array_equal(outs[0].view(np.uint64), outs[1].view(np.uint64))
    assert np.array_equal(outs[0].view(np.uint64), outs[2].view(np.uint64))


@pytest.mark.parametrize("n,batch", [(256, 6), (512, 3), (768, 2)])
def test_zinv_deterministic_under_load(gpu, n, batch):
    """Repeated inversions of one batch give the same bits every time, alone and while another
    stream keeps the SMs busy with FP64 GEMMs (the panel CTA shares its SM with other CTAs; the
    cluster variant exchanges pivots through DSMEM): a data race would show as run-to-run noise."""
    from paper_2605_19910_b200._native import lib

    torch = _torch()
    rng = np.random.default_rng(3 * n + batch)
    a = _rand(rng, batch, n, n)
    side = torch.cuda.Stream()
    x = torch.randn(2048, 2048, dtype=torch.float64, device="cuda")
    first = None
    for rep in range(12):
        if rep >= 4:  # background load on another stream from the fifth repetition on
            with torch.cuda.stream(side):
                for _ in range(4):
                    x = (x @ x) * 1e-3
        da = _dev(a)
        st = np.zeros(batch, dtype=np.int32)
        rc = lib().bbsi_cuda_zinv_dev(n, n, batch, C.c_void_p(da.data_ptr()), n, n * n,
                                      st.ctypes.data_as(C.c_void_p), C.c_void_p(0))
        assert rc == 0 and (st == -1).all()
        torch.cuda.synchronize()
        out = da.cpu().numpy().view(np.uint64)
        if first is None:
            first = out
        else:
            assert np.array_equal(out, first), rep


def test_zinv_flags_singular(gpu):
    from paper_2605_19910_b200._native import lib

    n = 64
    rng = np.random.default_rng(3)
    a = _rand(rng, 2, n, n)
    a[1, :, 5] = 0  # exactly singular second matrix
    da = _dev(a)
    st = np.zeros(2, dtype=np.int32)
    rc = lib().bbsi_cuda_zinv_dev(n, n, 2, C.c_void_p(da.data_ptr()), n, n * n, st.ctypes.data_as(C.c_void_p),
                                  C.c_void_p(0))
    assert rc == 0
    assert st[0] == -1 and st[1] >= 0


def test_dyson_generator_device_matches_host(gpu):
    from paper_2605_19910_b200 import dyson as D

    torch = _torch()
    cfg = D.scaled(D.CONFIGS[3], num_layers=5, block_size=64)
    H = torch.empty((5, 5, 64, 64), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    torch.cuda.synchronize()
    assert np.array_equal(H.cpu().numpy(), D.fill_h_host(cfg))


@pytest.mark.parametrize("k,layers,ne,b", [(2, 24, 6, 256), (3, 20, 4, 128), (5, 6, 2, 768)])
def test_tma_gemm_bit_identical(gpu, k, layers, ne, b):
    """The TMA-staged sweep GEMM (csrc/zgemm_tma.cu) performs the same DMMA sequence per
    output element as the cp.async kernel: the whole Dyson solve is bit-identical with
    BBSI_TMA=0 and =1 (and both match the oracle)."""
    import os

    import torch

    from paper_2605_19910_b200 import dyson as D

    cfg = D.scaled(D.CONFIGS[k], num_layers=layers, n_energy=ne, block_size=b)
    l, w = cfg.num_layers, cfg.bandwidth
    H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    out = []
    for flag in ("0", "1"):
        os.environ["BBSI_TMA"] = flag
        try:
            G = torch.empty((cfg.n_energy, l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
            D.solve_device(cfg, H, G, stream=torch.cuda.Stream())
            torch.cuda.synchronize()
            out.append(G.cpu())
        finally:
            os.environ.pop("BBSI_TMA", None)
    assert torch.equal(out[0], out[1])

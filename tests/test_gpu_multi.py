"""Multi-GPU entry points of the C ABI on one GPU (the pool gives one GPU per box):
the NCCL code path with a one-rank communicator, the single-process multi-GPU drop-ins
with ngpu = 1, and concurrent host threads on the per-thread workspaces. Each must give
exactly the single-GPU result."""
import ctypes as C
import threading

import numpy as np
import pytest

import paper_2605_19910_b200 as P
from oracle import bbsi_oracle as O
from oracle import dyson_oracle as DO
from paper_2605_19910_b200 import distributed as Dd
from paper_2605_19910_b200 import dyson as D
from paper_2605_19910_b200._native import lib
from tests._util import max_err, to_product

pytestmark = pytest.mark.gpu


def _stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def test_nccl_rank_path_one_rank(gpu):
    """bbsi_cuda_ddrgf_rank_dev with a real (one-rank) NCCL communicator: the packet and
    halo all-gathers run through NCCL and the result equals the resident single-call path."""
    import torch

    assert lib().bbsi_cuda_nccl_available() == 1, "NCCL must load on the GPU box"
    l, b, s2 = 70, 64, 8
    a = DO.dyson_matrix(DO.hamiltonian(l, 1, b, 6), complex(0.35, 1e-4), 1)
    full = torch.from_numpy(np.ascontiguousarray(a.data.transpose(0, 1, 3, 2))).cuda()
    comm = Dd.NcclComm()
    try:
        t0, t1, L0, L1 = Dd.rank_layers(l, s2, comm.world, comm.rank)
        assert (L0, L1) == (0, l)
        G = torch.empty_like(full)
        Dd.ddrgf_nccl(comm, full, G, l, b, s2)
    finally:
        comm.close()
    Gd = torch.empty_like(full)
    fail = C.c_int(-1)
    assert lib().bbsi_cuda_ddrgf_dev(l, b, s2, C.c_void_p(full.data_ptr()), C.c_void_p(Gd.data_ptr()), C.byref(fail),
                                     _stream()) == 0
    torch.cuda.synchronize()
    assert torch.equal(G, Gd)
    got = O.Band(a.layout, np.ascontiguousarray(G.cpu().numpy().transpose(0, 1, 3, 2)))
    assert O.max_block_error(got, O.rgf_tridiag(a)[0]) <= 1e-10


def test_nccl_rank_plan_one_rank(gpu):
    """bbsi_cuda_ddrgf_rank_plan_dev (nested interface levels) through a one-rank NCCL
    communicator equals the resident multi-level plan entry bit for bit."""
    import torch

    l, b = 90, 64
    a = DO.dyson_matrix(DO.hamiltonian(l, 1, b, 9), complex(-0.25, 1e-4), 1)
    full = torch.from_numpy(np.ascontiguousarray(a.data.transpose(0, 1, 3, 2))).cuda()
    comm = Dd.NcclComm()
    try:
        G = torch.empty_like(full)
        Dd.ddrgf_nccl(comm, full, G, l, b, 4, levels_above=(3,))
    finally:
        comm.close()
    Gd = torch.empty_like(full)
    lv = np.array([4, 3], dtype=np.int32)
    fail = C.c_int(-1)
    assert lib().bbsi_cuda_ddrgf_plan_dev(l, b, lv.ctypes.data_as(C.c_void_p), 2, C.c_void_p(full.data_ptr()),
                                          C.c_void_p(Gd.data_ptr()), C.byref(fail), _stream()) == 0
    torch.cuda.synchronize()
    assert torch.equal(G, Gd)
    got = O.Band(a.layout, np.ascontiguousarray(G.cpu().numpy().transpose(0, 1, 3, 2)))
    assert O.max_block_error(got, O.rgf_tridiag(a)[0]) <= 1e-10


def test_ddrgf_multi_one_gpu(gpu):
    """bbsi_cuda_ddrgf_multi_z (one host thread per GPU) with ngpu = 1 == bbsi_cuda_ddrgf_z."""
    m = to_product(DO.dyson_matrix(DO.hamiltonian(40, 1, 48, 8), complex(-0.3, 1e-4), 1))
    plan = P.DomainPlan([6], 2, 1)
    g1, c1 = P.ddrgf(m, plan)
    from paper_2605_19910_b200.bbsi import _args, _ptr

    lay, sizes, a, g = _args(m)
    s2 = np.array([6], dtype=np.int32)
    cnt = np.zeros(3, dtype=np.int64)
    fail = C.c_int(-1)
    dev = np.array([0], dtype=np.int32)
    rc = lib().bbsi_cuda_ddrgf_multi_z(lay.num_layers, lay.bandwidth, lay.slot_size, _ptr(sizes), _ptr(a), _ptr(s2), 1,
                                       2, 1, 1, _ptr(dev), _ptr(g), _ptr(cnt), C.byref(fail))
    assert rc == 0, lib().bbsi_cuda_last_error()
    g2 = P.BlockBandedMatrix._from_slots(lay, g)
    assert np.array_equal(g2.data, g1.data)
    assert tuple(cnt) == c1.as_tuple()
    with pytest.raises(P.InvalidArgumentError):
        P.ddrgf(m, P.DomainPlan([6], 2, 1), ngpu=64)  # more GPUs than visible / domains


def test_dyson_multi_one_gpu(gpu):
    cfg = D.scaled(D.CONFIGS[2], num_layers=24, n_energy=5, block_size=64)
    G1, f1 = D.solve_host(cfg)
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    H = D.fill_h_host(cfg)
    z = cfg.z()
    sig = cfg.sigma()
    G2 = np.empty_like(G1)
    fails = np.full(len(z), -1, dtype=np.int32)
    rc = lib().bbsi_cuda_dyson_rgf_multi_z(l, w, b, len(z), H.ctypes.data_as(C.c_void_p), z.ctypes.data_as(C.c_void_p),
                                           sig.ctypes.data_as(C.c_void_p), C.c_void_p(G2.ctypes.data),
                                           fails.ctypes.data_as(C.c_void_p), 0, 1, None)
    assert rc == 0
    assert np.array_equal(G1, G2) and (fails == -1).all()


def test_concurrent_host_threads(gpu):
    """Per-thread workspaces: drop-in calls from several host threads run concurrently and
    each returns exactly what it returns alone (the reference solvers are reentrant,
    SPEC.md:301,376)."""
    ms = [to_product(DO.dyson_matrix(DO.hamiltonian(32, 1, 64, 20 + k), complex(0.1 * k, 1e-3), 1)) for k in range(4)]
    alone = [P.rgf_tridiag(m)[0].data.copy() for m in ms]
    dd_alone = [P.ddrgf(m, P.DomainPlan([5], 1, 1))[0].data.copy() for m in ms]
    got, dd_got, errs = [None] * 4, [None] * 4, []

    def run(k):
        try:
            for _ in range(3):
                got[k] = P.rgf_tridiag(ms[k])[0].data.copy()
                dd_got[k] = P.ddrgf(ms[k], P.DomainPlan([5], 1, 1))[0].data.copy()
        except Exception as ex:  # pragma: no cover
            errs.append(ex)

    th = [threading.Thread(target=run, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    for k in range(4):
        assert np.array_equal(got[k], alone[k]) and np.array_equal(dd_got[k], dd_alone[k])
    ref, _ = O.rgf_tridiag(DO.dyson_matrix(DO.hamiltonian(32, 1, 64, 20), complex(0.0, 1e-3), 1))
    assert max_err(P.rgf_tridiag(ms[0])[0], ref) <= 1e-10

"""GPU parity of the stabilised DDRGF (csrc/ddrgf.cu) through the C ABI.

Restates tests/test_ddrgf.cpp (same seeds, sizes, plans and tolerances) with the
sequential RGF (oracle) as the reference result, plus Dyson-matrix cases where
the reference's own DDRGF formulation loses digits (SURVEY.md finding 3) and the
stabilised one must stay within the 1e-10 bar.
"""
import numpy as np
import pytest

import paper_2605_19910_b200 as P
from oracle import bbsi_oracle as O
from oracle import dyson_oracle as DO
from tests._util import max_err, to_product

pytestmark = pytest.mark.gpu


def _plan(levels, nt=3):
    return P.DomainPlan(list(levels), nt, 1)


def test_matches_sequential_across_plans_and_sizes(gpu):
    """test_ddrgf.cpp:44-60"""
    for l in (6, 10, 15, 40):
        m = O.random_spd_like(O.make_layout(l, 3, 1), 500 + l, 2.0)
        ref, _ = O.rgf_tridiag(m)
        for levels in ([1], [4], [2, 1], [4, 1]):
            if l < levels[0] + 1:
                continue
            g, c = P.ddrgf(to_product(m), _plan(levels))
            assert max_err(g, ref) <= 1e-10, (l, levels)


def test_independent_of_thread_count(gpu):
    """test_ddrgf.cpp:62-74: bit identical across n_threads."""
    m = to_product(O.random_spd_like(O.make_layout(21, 4, 1), 601, 2.0))
    g1, c1 = P.ddrgf(m, _plan([4, 2], 1))
    for nt in (2, 3, 8):
        g, c = P.ddrgf(m, _plan([4, 2], nt))
        assert np.array_equal(g.data, g1.data)
        assert c == c1


def test_counters_closed_form_even_plans(gpu):
    """test_ddrgf.cpp:76-94"""
    for l, levels in ((10, [4]), (15, [4, 2]), (8, [1, 1, 1]), (18, [2])):
        assert O.ddrgf_divides_evenly(l, levels)
        m = O.random_spd_like(O.make_layout(l, 2, 1), 700 + l, 2.0)
        g, c = P.ddrgf(to_product(m), _plan(levels, 2))
        assert c.as_tuple() == O.predict_ddrgf_counters(l, levels).as_tuple()
        assert max_err(g, O.rgf_tridiag(m)[0]) <= 1e-10


def test_trailing_groups(gpu):
    """test_ddrgf.cpp:96-108"""
    for l in (11, 12, 13):
        m = O.random_spd_like(O.make_layout(l, 2, 1), 800 + l, 2.0)
        g, c = P.ddrgf(to_product(m), _plan([4], 2))
        assert max_err(g, O.rgf_tridiag(m)[0]) <= 1e-10
        assert c.as_tuple() == O.ddrgf(m, [4])[1].as_tuple()


def test_zero_couplings(gpu):
    """test_ddrgf.cpp:204-216"""
    m = O.random_spd_like(O.make_layout(10, 2, 1), 904, 2.0)
    m.block(4, 1)[...] = 0
    m.block(5, -1)[...] = 0
    g, _ = P.ddrgf(to_product(m), _plan([4], 2))
    assert max_err(g, O.rgf_tridiag(m)[0]) <= 1e-10


def test_validation_and_plan_exhaustion(gpu):
    """test_ddrgf.cpp:218-234"""
    m = to_product(O.random_spd_like(O.make_layout(6, 2, 1), 905, 2.0))
    with pytest.raises(P.InvalidArgumentError):
        P.ddrgf(m, _plan([4, 4]))
    with pytest.raises(P.InvalidArgumentError):
        P.ddrgf(m, P.DomainPlan([], 1, 1))
    wide = to_product(O.random_spd_like(O.make_layout(6, 2, 2), 906, 2.0))
    with pytest.raises(P.InvalidArgumentError):
        P.ddrgf(wide, _plan([1]))
    ragged = to_product(O.random_spd_like(O.BlockLayout(6, [2, 3, 2, 3, 2, 3], 1), 907, 2.0))
    with pytest.raises(P.InvalidArgumentError):
        P.ddrgf(ragged, _plan([1]))


def test_singular_subdomain_global_layer(gpu):
    """test_ddrgf.cpp:236-250"""
    m = O.random_spd_like(O.make_layout(10, 2, 1), 908, 2.0)
    m.block(7, 0)[...] = 0
    m.block(7, 1)[...] = 0
    m.block(7, -1)[...] = 0
    with pytest.raises(P.SingularMatrixError) as ei:
        P.ddrgf(to_product(m), _plan([4], 2))
    assert ei.value.layer == 7


@pytest.mark.parametrize("l,b,s2,eta,E", [(64, 64, 15, 1e-4, 0.1), (96, 64, 11, 1e-5, -0.4), (66, 128, 10, 1e-4, 0.1),
                                          (45, 256, 8, 1e-4, 0.1), (19, 64, 4, 1e-3, 0.3)])
def test_dyson_matrices_within_bar(gpu, l, b, s2, eta, E):
    """BASELINE-type matrices (indefinite, weakly damped): stabilised DDRGF vs sequential RGF <= 1e-10."""
    h = DO.hamiltonian(l, 1, b, 3)
    a = DO.dyson_matrix(h, complex(E, eta), 1)
    ref, _ = O.rgf_tridiag(a)
    g, _ = P.ddrgf(to_product(a), _plan([s2]))
    assert max_err(g, ref) <= 1e-10


@pytest.mark.parametrize("l,b,s2,world", [(63, 64, 7, 2), (70, 64, 8, 3), (45, 128, 10, 4)])
def test_sharded_phases_emulated_ranks(gpu, l, b, s2, world):
    """The domain-sharded protocol with the CUDA phases, ranks emulated one after the
    other on one device (packets concatenated instead of all-gathered)."""
    import torch

    from paper_2605_19910_b200 import distributed as Dd

    a = DO.dyson_matrix(DO.hamiltonian(l, 1, b, 4), complex(-0.2, 1e-4), 1)
    ref, _ = O.rgf_tridiag(a)
    full = torch.from_numpy(np.ascontiguousarray(a.data.transpose(0, 1, 3, 2))).cuda()
    tasks = Dd.partition(l, s2)
    ranges = Dd.task_ranges(len(tasks), world)
    eng = Dd.CudaPhases(l, b, s2)
    packets, locs = [], []
    for t0, t1 in ranges:
        L0, L1 = Dd.layer_range(tasks, t0, t1)
        A_loc = full[L0:L1].clone()
        packets.append(eng.phase1(A_loc, t0, t1))
        locs.append((L0, L1, A_loc, t0, t1))
    out = eng.phase2(torch.cat(packets))
    G = torch.zeros_like(full)
    Gs, halos = [], []
    for L0, L1, A_loc, t0, t1 in locs:
        Gl = eng.phase3(A_loc, out, t0, t1)
        Gs.append(Gl)
        halos.append(eng.halo(Gl, t0, t1))
    for r, (L0, L1, A_loc, t0, t1) in enumerate(locs):
        prev = halos[r - 1][1] if r > 0 else None
        nxt = halos[r + 1][0] if r + 1 < len(locs) else None
        G[L0:L1] = eng.couplings(A_loc, Gs[r], out, t0, t1, prev, nxt)
    got = O.Band(a.layout, np.ascontiguousarray(G.cpu().numpy().transpose(0, 1, 3, 2)))
    assert O.max_block_error(got, ref) <= 1e-10
    # same bits as the one-call resident path (the exchanges only move data)
    Gd = torch.empty_like(full)
    import ctypes as C

    from paper_2605_19910_b200._native import lib

    fail = C.c_int(-1)
    assert lib().bbsi_cuda_ddrgf_dev(l, b, s2, C.c_void_p(full.data_ptr()), C.c_void_p(Gd.data_ptr()),
                                     C.byref(fail), C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    assert torch.equal(Gd, G)


@pytest.mark.parametrize("scale", [1e-6, 1.0, 1e6])
def test_scale_invariance(gpu, scale):
    """The fake-lead strength follows the matrix scale (gamma_t = gamma0 max|A[s,s]|), so
    DDRGF of c*A matches sequential RGF of c*A for tiny and huge c."""
    a = DO.dyson_matrix(DO.hamiltonian(48, 1, 64, 5), complex(0.2, 1e-4), 1)
    a = O.Band(a.layout, a.data * scale)
    ref, _ = O.rgf_tridiag(a)
    g, _ = P.ddrgf(to_product(a), _plan([7]))
    assert max_err(g, ref) <= 1e-10


@pytest.mark.parametrize("l,b,plan,E,eta", [(96, 64, [7, 2], 0.1, 1e-4), (120, 64, [4, 3, 1], -0.3, 1e-4),
                                            (64, 128, [3, 2], 0.2, 1e-4), (77, 64, [5, 4], 0.05, 1e-5),
                                            (40, 64, [2, 1, 1], 0.3, 1e-3)])
def test_nested_levels_on_device(gpu, l, b, plan, E, eta):
    """Multi-level plans (s2_levels[1..], ddrgf.hpp:363-369) run on the device: the level-0
    2-ports are merged into super 2-ports per level (csrc/ddrgf_iface.cu) and the interface
    system is solved top-down. Same output as sequential RGF to the 1e-10 bar."""
    a = DO.dyson_matrix(DO.hamiltonian(l, 1, b, 11), complex(E, eta), 1)
    ref, _ = O.rgf_tridiag(a)
    g, c = P.ddrgf(to_product(a), _plan(plan))
    assert max_err(g, ref) <= 1e-10
    g1, _ = P.ddrgf(to_product(a), _plan(plan[:1]))
    assert max_err(g, O.Band(ref.layout, g1.data.copy())) <= 1e-10

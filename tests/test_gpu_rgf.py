"""GPU parity of rgf_tridiag / rgf_ndiag / rgf_fused through the C ABI.

Each case restates a reference test (tests/test_rgf.cpp) with the same seeds,
sizes and tolerances; the checker is the compiled reference (oracle/_ref) when
present, else the numpy restatement (oracle/bbsi_oracle.py), plus the dense
oracle (block_banded.hpp:175-181).
"""
import numpy as np
import pytest

import paper_2605_19910_b200 as P
from oracle import bbsi_oracle as O
from tests._util import max_err, to_oracle, to_product

pytestmark = pytest.mark.gpu


def test_second_difference_known_answer(gpu):
    """test_rgf.cpp:10-25 (real input promoted to complex128)."""
    m = O.Band(O.make_layout(3, 1, 1))
    for i in range(3):
        m.block(i, 0)[0, 0] = 2
        if i > 0:
            m.block(i, -1)[0, 0] = -1
        if i < 2:
            m.block(i, 1)[0, 0] = -1
    g, c = P.rgf_tridiag(to_product(m))
    assert abs(g.block(0, 0)[0, 0] - 0.75) <= 1e-14
    assert abs(g.block(1, 0)[0, 0] - 1.0) <= 1e-14
    assert abs(g.block(2, 0)[0, 0] - 0.75) <= 1e-14
    assert abs(g.block(0, 1)[0, 0] - 0.5) <= 1e-14
    assert abs(g.block(1, 1)[0, 0] - 0.5) <= 1e-14
    assert c.as_tuple() == (8, 3, 7)


def test_single_layer(gpu):
    """test_rgf.cpp:27-32"""
    m = O.random_spd_like(O.make_layout(1, 4, 0), 3, 2.0)
    g, c = P.rgf_tridiag(to_product(m))
    assert max_err(g, O.oracle_selected_inverse(m)) <= 1e-13
    assert c.as_tuple() == O.predict_rgf_counters(1).as_tuple()


def test_tridiag_matches_oracle_with_counters(gpu):
    """test_rgf.cpp:34-40"""
    m = O.random_spd_like(O.make_layout(12, 8, 1), 77, 2.0)
    g, c = P.rgf_tridiag(to_product(m))
    assert max_err(g, O.oracle_selected_inverse(m)) <= 1e-10
    assert max_err(g, O.rgf_tridiag(m)[0]) <= 1e-12
    assert c.as_tuple() == (44, 12, 34)


def test_ragged_block_sizes(gpu):
    """test_rgf.cpp:42-48"""
    m = O.random_spd_like(O.BlockLayout(5, [3, 1, 4, 2, 3], 1), 8, 2.0)
    g, c = P.rgf_tridiag(to_product(m))
    assert max_err(g, O.oracle_selected_inverse(m)) <= 1e-10
    assert c.as_tuple() == O.predict_rgf_counters(5).as_tuple()


def test_ndiag_reduces_to_tridiag(gpu):
    """test_rgf.cpp:50-56 (identical kernel sequence on the GPU path -> bit-identical)."""
    m = to_product(O.random_spd_like(O.make_layout(9, 4, 1), 13, 2.0))
    g1, c1 = P.rgf_tridiag(m)
    gn, cn = P.rgf_ndiag(m)
    assert np.array_equal(g1.data, gn.data)
    assert c1 == cn


@pytest.mark.parametrize("w", [2, 3])
def test_ndiag_matches_oracle(gpu, w):
    """test_rgf.cpp:58-67"""
    m = O.random_spd_like(O.make_layout(10, 4, w), 100 + w, 2.0)
    trace = {}
    g, c = P.rgf_ndiag(to_product(m), trace)
    assert max_err(g, O.oracle_selected_inverse(m)) <= 1e-10
    assert trace["max_update_offset"] <= w - 1
    assert c.as_tuple() == O.predict_nrgf_counters(10, w).as_tuple()


def test_ndiag_counters_closed_form(gpu):
    """test_rgf.cpp:69-77 (plus parity on every case)."""
    for w in range(1, 4):
        for l in range(w + 1, 13):
            m = O.random_spd_like(O.make_layout(l, 2, w), l * 10 + w, 2.0)
            g, c = P.rgf_ndiag(to_product(m))
            assert c.as_tuple() == O.predict_nrgf_counters(l, w).as_tuple()
            assert max_err(g, O.rgf_ndiag(m)[0]) <= 1e-10


def test_fused_agrees_with_ndiag(gpu):
    """test_rgf.cpp:79-88"""
    m = O.random_spd_like(O.make_layout(9, 3, 2), 55, 2.0)
    gf, cf = P.rgf_fused(to_product(m))
    assert max_err(gf, O.rgf_ndiag(m)[0]) <= 1e-10
    assert cf.as_tuple() == (16, 5, 13)


def test_fused_short_last_superblock(gpu):
    """test_rgf.cpp:90-95"""
    m = O.random_spd_like(O.make_layout(10, 2, 3), 56, 2.0)
    gf, cf = P.rgf_fused(to_product(m))
    assert max_err(gf, O.oracle_selected_inverse(m)) <= 1e-10
    assert cf.as_tuple() == O.predict_rgf_counters(4).as_tuple()


def test_hermitian_input_gives_hermitian_inverse(gpu):
    """test_rgf.cpp:150-160"""
    h1 = O.random_hermitian(O.make_layout(8, 3, 1), 31, 1.0)
    g1, _ = P.rgf_tridiag(to_product(h1))
    assert O.hermitian_defect(to_oracle(g1)) <= 1e-12
    h2 = O.random_hermitian(O.make_layout(8, 3, 2), 32, 1.0)
    g2, _ = P.rgf_ndiag(to_product(h2))
    assert O.hermitian_defect(to_oracle(g2)) <= 1e-12


def test_singular_pivot_attribution(gpu):
    """test_rgf.cpp:162-171"""
    m = O.random_spd_like(O.make_layout(5, 2, 1), 40, 2.0)
    m.block(4, 0)[...] = 0
    with pytest.raises(P.SingularMatrixError) as ei:
        P.rgf_tridiag(to_product(m))
    assert ei.value.layer == 4


def test_wrong_bandwidth_rejected(gpu):
    """test_rgf.cpp:173-179"""
    wide = to_product(O.random_spd_like(O.make_layout(6, 2, 2), 41, 2.0))
    with pytest.raises(P.InvalidArgumentError):
        P.rgf_tridiag(wide)
    ragged = to_product(O.random_spd_like(O.BlockLayout(4, [2, 3, 2, 3], 2), 42, 2.0))
    with pytest.raises(P.InvalidArgumentError):
        P.rgf_fused(ragged)


@pytest.mark.parametrize("l,b,w", [(6, 64, 1), (7, 128, 1), (9, 64, 2), (5, 192, 2), (4, 96, 3)])
def test_padded_and_native_block_sizes(gpu, l, b, w):
    """Block sizes on and off the 64-wide tile grid, diagonally dominant inputs."""
    m = O.random_spd_like(O.make_layout(l, b, w), 1000 + l + b + w, 2.0)
    g, _ = P.rgf_ndiag(to_product(m))
    assert max_err(g, O.rgf_ndiag(m)[0]) <= 1e-12


@pytest.mark.parametrize("l", [1, 2, 3, 5, 6])
def test_extended_halos_equal_dense_inverse(gpu, l):
    """test_rgf.cpp:97-123"""
    m = O.random_spd_like(O.make_layout(l, 3, 0 if l == 1 else 1), 200 + l, 2.0)
    ext, c = P.rgf_extended(to_product(m))
    assert c.as_tuple() == O.predict_extended_counters(l).as_tuple()
    dense = np.linalg.inv(O.to_dense(m))

    def slab(a, b):
        return dense[3 * a:3 * a + 3, 3 * b:3 * b + 3]

    for b in range(l):
        assert O.rel_frobenius_error(ext.first_row[b], slab(0, b)) <= 1e-10
        assert O.rel_frobenius_error(ext.last_row[b], slab(l - 1, b)) <= 1e-10
        assert O.rel_frobenius_error(ext.first_col[b], slab(b, 0)) <= 1e-10
        assert O.rel_frobenius_error(ext.last_col[b], slab(b, l - 1)) <= 1e-10
    g, _ = P.rgf_tridiag(to_product(m))
    assert np.array_equal(ext.core.data, g.data)


def test_extended_overlaps_are_exact_copies(gpu):
    """test_rgf.cpp:125-135"""
    m = O.random_spd_like(O.make_layout(6, 2, 1), 201, 2.0)
    ext, _ = P.rgf_extended(to_product(m))
    core = ext.core
    assert np.array_equal(ext.first_row[0], core.block(0, 0))
    assert np.array_equal(ext.first_row[1], core.block(0, 1))
    assert np.array_equal(ext.last_row[5], core.block(5, 0))
    assert np.array_equal(ext.last_row[4], core.block(5, -1))
    assert np.array_equal(ext.first_col[1], core.block(1, -1))
    assert np.array_equal(ext.last_col[4], core.block(4, 1))


def test_extended_vs_reference_on_dyson_blocks(gpu):
    """Halos at b = 64 on a Dyson matrix against the reference rgf_extended (numpy restatement)."""
    from oracle import dyson_oracle as DO

    a = DO.dyson_matrix(DO.hamiltonian(9, 1, 64, 5), complex(0.2, 1e-3), 1)
    ext, _ = P.rgf_extended(to_product(a))
    ref, _ = O.rgf_extended(a)
    for k in range(9):
        for got, exp in ((ext.first_row[k], ref.first_row[k]), (ext.last_row[k], ref.last_row[k]),
                         (ext.first_col[k], ref.first_col[k]), (ext.last_col[k], ref.last_col[k])):
            assert O.rel_frobenius_error(got, exp) <= 1e-10


def test_rgf_many_matches_single_calls(gpu):
    """bbsi_cuda_rgf_many_z: many matrices of one layout in one pass give exactly the
    single-call results (same kernels, one batch), w = 1 and w = 2, ragged blocks included."""
    for lay in (O.make_layout(14, 9, 1), O.make_layout(16, 6, 2), O.BlockLayout(7, [3, 5, 2, 5, 4, 1, 5], 1)):
        ms = [to_product(O.random_spd_like(lay, 1300 + k, 2.0)) for k in range(4)]
        many = P.rgf_many(ms)
        single = P.rgf_ndiag if lay.bandwidth > 1 else P.rgf_tridiag
        for m, (g, c) in zip(ms, many):
            g1, c1 = single(m)
            assert np.array_equal(g.data, g1.data) and c == c1


def test_rgf_many_reports_first_failing_matrix(gpu):
    ms = [O.random_spd_like(O.make_layout(10, 4, 1), 1400 + k, 2.0) for k in range(3)]
    for off in (-1, 0, 1):
        ms[1].block(6, off)[...] = 0
    with pytest.raises(P.SingularMatrixError) as ei:
        P.rgf_many([to_product(m) for m in ms])
    assert ei.value.layer == 6

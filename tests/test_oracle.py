"""Pins the numpy oracle (oracle/bbsi_oracle.py) before it is trusted as the checker:
(1) against committed golden fixtures generated from the compiled reference,
(2) against the compiled reference itself (oracle/_ref) when present,
(3) against the reference's own known-answer tests."""
from pathlib import Path

import numpy as np
import pytest

from oracle import bbsi_oracle as O
from oracle import dyson_oracle as DO
from oracle import ref_lib as R

GOLD = Path(__file__).resolve().parent / "golden"


def load(name):
    d = np.load(GOLD / f"{name}.npz")
    lay = O.BlockLayout(len(d["sizes"]), list(d["sizes"]), int(d["w"]))
    return O.Band(lay, d["A"].copy()), d


def test_golden_generators_bit_exact():
    """UniformSource / random_spd_like (block_banded.hpp:70-133) restated bit-exactly."""
    m, _ = load("rgf_tridiag_l12_b8_s77")
    assert np.array_equal(O.random_spd_like(O.make_layout(12, 8, 1), 77, 2.0).data, m.data)
    m, _ = load("rgf_tridiag_ragged_s8")
    assert np.array_equal(O.random_spd_like(O.BlockLayout(5, [3, 1, 4, 2, 3], 1), 8, 2.0).data, m.data)
    h, _ = load("hermitian_l8_b3_s31")
    assert np.array_equal(O.random_hermitian(O.make_layout(8, 3, 1), 31, 1.0).data, h.data)


@pytest.mark.parametrize("name", ["rgf_tridiag_l12_b8_s77", "rgf_tridiag_ragged_s8", "hermitian_l8_b3_s31"])
def test_golden_rgf_tridiag(name):
    m, d = load(name)
    g, c = O.rgf_tridiag(m)
    assert O.max_block_error(g, O.Band(m.layout, d["G"])) <= 1e-13
    assert c.as_tuple() == tuple(d["counters"])


@pytest.mark.parametrize("w", [2, 3])
def test_golden_rgf_ndiag(w):
    m, d = load(f"rgf_ndiag_l10_b4_w{w}")
    tr = {}
    g, c = O.rgf_ndiag(m, tr)
    assert O.max_block_error(g, O.Band(m.layout, d["G"])) <= 1e-13
    assert c.as_tuple() == tuple(d["counters"])
    assert tr["max_update_offset"] == int(d["max_update_offset"])


def test_golden_rgf_fused_and_extended():
    m, d = load("rgf_fused_l9_b3_w2")
    g, c = O.rgf_fused(m)
    assert O.max_block_error(g, O.Band(m.layout, d["G"])) <= 1e-13 and c.as_tuple() == tuple(d["counters"])
    m, d = load("rgf_extended_l5_b3")
    e, c = O.rgf_extended(m)
    assert c.as_tuple() == tuple(d["counters"])
    for k in range(5):
        for got, exp in ((e.first_row[k], d["first_row"][k]), (e.last_row[k], d["last_row"][k]),
                         (e.first_col[k], d["first_col"][k]), (e.last_col[k], d["last_col"][k])):
            assert O.rel_frobenius_error(got, exp) <= 1e-13


@pytest.mark.parametrize("name", ["ddrgf_l10_b3_4", "ddrgf_l13_b3_4", "ddrgf_l15_b3_4_2", "ddrgf_l40_b3_2_1"])
def test_golden_ddrgf(name):
    m, d = load(name)
    g, c = O.ddrgf(m, list(d["levels"]))
    assert O.max_block_error(g, O.Band(m.layout, d["G"])) <= 1e-13
    assert c.as_tuple() == tuple(d["counters"])


def test_golden_partition_orders():
    d = np.load(GOLD / "partition_orders.npz")
    for l, s2 in ((10, 4), (11, 4), (12, 4), (2, 1)):
        order, desc = O.interleave_permutation(O.make_layout(l, 1, 1), 1, s2)
        assert order == list(d[f"order_{l}_{s2}"])
        assert [list(x) for x in desc.interior_groups] == [list(x) for x in d[f"inter_{l}_{s2}"]]
    # test_partition.cpp:9-19 known order
    order, _ = O.interleave_permutation(O.make_layout(10, 2, 1), 1, 4)
    assert order == [4, 9, 0, 1, 2, 3, 5, 6, 7, 8]


def test_known_answers():
    """test_rgf.cpp:10-25, test_block_banded.cpp:94-115"""
    m = O.Band(O.make_layout(3, 1, 1))
    for i in range(3):
        m.block(i, 0)[0, 0] = 2
        if i > 0:
            m.block(i, -1)[0, 0] = -1
        if i < 2:
            m.block(i, 1)[0, 0] = -1
    for g in (O.rgf_tridiag(m)[0], O.oracle_selected_inverse(m)):
        assert abs(g.block(0, 0)[0, 0] - 0.75) < 1e-14 and abs(g.block(1, 0)[0, 0] - 1.0) < 1e-14
        assert abs(g.block(0, 1)[0, 0] - 0.5) < 1e-14 and abs(g.block(1, -1)[0, 0] - 0.5) < 1e-14
    assert O.rgf_tridiag(m)[1].as_tuple() == (8, 3, 7)
    ident = O.Band(O.make_layout(4, 3, 1))
    for i in range(4):
        ident.block(i, 0)[...] = np.eye(3)
    assert O.max_block_error(O.oracle_selected_inverse(ident), ident) <= 1e-14


def test_singular_attribution():
    m = O.random_spd_like(O.make_layout(5, 2, 1), 40, 2.0)
    m.block(4, 0)[...] = 0
    with pytest.raises(O.SingularMatrixError) as ei:
        O.rgf_tridiag(m)
    assert ei.value.layer == 4


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_restatement_matches_compiled_reference():
    for (l, b, w, s) in [(12, 8, 1, 77), (10, 4, 2, 102), (10, 2, 3, 56), (7, 5, 1, 3)]:
        m = R.random_spd_like(O.make_layout(l, b, w), s, 2.0)
        assert np.array_equal(O.random_spd_like(O.make_layout(l, b, w), s, 2.0).data, m.data)
        g1, c1 = O.rgf_ndiag(m)
        g2, c2 = R.rgf_ndiag(m)
        assert O.max_block_error(g1, g2) <= 1e-13 and c1 == c2
    for l, lev in ((6, [1]), (10, [4]), (15, [2, 1]), (11, [4])):
        m = R.random_spd_like(O.make_layout(l, 3, 1), 500 + l, 2.0)
        g1, c1 = O.ddrgf(m, lev)
        g2, c2 = R.ddrgf(m, lev, 2)
        assert O.max_block_error(g1, g2) <= 1e-13 and c1 == c2


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_restatement_on_dyson_matrix_matches_reference():
    """The Dyson generator spec fed to both the compiled reference and the restatement."""
    a = DO.dyson_matrix(DO.hamiltonian(24, 1, 32, 1), complex(0.3, 1e-3), 1)
    g1, _ = O.rgf_tridiag(a)
    g2, _ = R.rgf_tridiag(a)
    assert O.max_block_error(g1, g2) <= 1e-12
    assert O.max_block_error(g1, O.oracle_selected_inverse(a)) <= 1e-10


# ---- streaming restatement (oracle/stream/rgf_stream.cpp), the full-size config-5 checker
@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("ckpt", [0, 1, 4, 7, 21])
def test_stream_oracle_bitwise_vs_reference(ckpt):
    """Same BLAS build as oracle/_ref (OpenBLAS 0.3.15): every G block and every A block
    is bit-identical to the compiled reference rgf_tridiag, for any checkpoint length."""
    from oracle import stream_lib as S

    S.use_fast(False)
    S.set_threads(1)
    l, b, seed, z = 21, 32, 5, complex(0.3, 1e-4)
    a = DO.dyson_matrix(DO.hamiltonian(l, 1, b, seed), z, 1)
    ref, _ = R.rgf_tridiag(a)
    s = S.DysonStream(l, b, seed, z, 1, ckpt=ckpt)
    for i in range(l):
        for off in (-1, 0, 1):
            if 0 <= i + off < l:
                assert np.array_equal(s.block(i, off), a.block(i, off))
    n = 0
    while (r := s.next()) is not None:
        i, d, u, lo = r
        assert np.array_equal(d, ref.block(i, 0))
        if i > 0:
            assert np.array_equal(u, ref.block(i - 1, 1)) and np.array_equal(lo, ref.block(i, -1))
        n += 1
    assert n == l


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")
def test_stream_oracle_fast_blas_vs_reference():
    """The scipy-OpenBLAS build used at full size agrees with the reference to <= 1e-13
    (different BLAS kernels, same calls) and its perturbed stream moves A by one ulp."""
    from oracle import stream_lib as S

    S.use_fast(True)
    try:
        S.set_threads(1)
        l, b, seed, z = 17, 48, 4, complex(-1.0, 1e-5)
        a = DO.dyson_matrix(DO.hamiltonian(l, 1, b, seed), z, 1)
        ref, _ = R.rgf_tridiag(a)
        s = S.DysonStream(l, b, seed, z, 1, ckpt=5)
        worst = 0.0
        while (r := s.next()) is not None:
            i, d, u, lo = r
            worst = max(worst, O.rel_frobenius_error(d, ref.block(i, 0)))
            if i > 0:
                worst = max(worst, O.rel_frobenius_error(u, ref.block(i - 1, 1)),
                            O.rel_frobenius_error(lo, ref.block(i, -1)))
        assert worst <= 1e-13
        p = S.DysonStream(l, b, seed, z, 1, pert=0.5, pert_seed=3, ckpt=5)
        x, y = a.block(3, 0), p.block(3, 0)
        rel = np.abs(y.view(np.float64) - x.view(np.float64)) / np.abs(x.view(np.float64))
        assert 0.3 < np.mean(rel > 0) < 0.7 and rel.max() <= 2.0**-52
    finally:
        S.use_fast(False)

"""CPU-side checks of the C ABI: the library loads and exports every symbol that
include/bbsi_cuda.h declares; without a GPU the compute entry points fail loudly
(BBSI_CUDA_ERROR) instead of falling back to the CPU."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "bbsi_cuda.h").read_text()
    return sorted(set(re.findall(r"\b(bbsi_(?:cuda|dyson|random)_\w+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    from paper_2605_19910_b200._native import SIGNATURES, lib

    names = _declared()
    assert len(names) >= 14
    L = lib()
    for n in names:
        assert hasattr(L, n), n
        assert n in SIGNATURES, n


def test_no_cpu_fallback_without_gpu():
    from paper_2605_19910_b200._native import lib

    L = lib()
    if L.bbsi_cuda_device_count() > 0:
        pytest.skip("GPU present")
    a = np.zeros((3, 3, 1, 1), dtype=np.complex128)
    a[:, 1] = 2.0
    g = np.zeros_like(a)
    rc = L.bbsi_cuda_rgf_tridiag_z(3, 1, 1, None, a.ctypes.data_as(C.c_void_p), g.ctypes.data_as(C.c_void_p),
                                   None, None)
    assert rc == 3  # BBSI_CUDA_ERROR
    assert "no CUDA device" in L.bbsi_cuda_last_error().decode()


def test_invalid_arguments_rejected_before_device():
    import paper_2605_19910_b200 as P

    with pytest.raises(P.InvalidArgumentError):
        P.make_layout(0, 2, 1)
    with pytest.raises(P.InvalidArgumentError):
        P.BlockLayout(3, [2, 2, 2], 3)
    from paper_2605_19910_b200._native import lib

    rc = lib().bbsi_cuda_rgf_tridiag_z(4, 2, 2, None, None, None, None, None)
    assert rc == 1


def test_host_dyson_generator_matches_oracle_spec():
    from oracle import dyson_oracle as DO
    from paper_2605_19910_b200 import dyson as D

    for k in (1, 3):
        cfg = D.scaled(D.CONFIGS[k], num_layers=4, block_size=64)
        h = D.fill_h_host(cfg)
        ref = DO.hamiltonian(cfg.num_layers, cfg.bandwidth, cfg.block_size, cfg.seed)
        assert np.array_equal(h.transpose(0, 1, 3, 2), ref.data)

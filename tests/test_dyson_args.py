"""Argument checks of the Dyson host API (paper_2605_19910_b200/dyson.py): the C ABI
takes raw pointers, so dtype / shape / contiguity / placement are validated before any
native call (no GPU needed: every case raises first)."""
import numpy as np
import pytest
import torch

from paper_2605_19910_b200 import InvalidArgumentError
from paper_2605_19910_b200 import dyson as D

CFG = D.scaled(D.CONFIGS[2], num_layers=4, n_energy=3, block_size=64)
SH = (4, 3, 64, 64)


def test_host_buffers_checked():
    H = np.zeros(SH, dtype=np.complex128)
    z = CFG.z()
    with pytest.raises(InvalidArgumentError, match="complex128"):
        D.solve_host(CFG, H=H.astype(np.complex64), z=z)
    with pytest.raises(InvalidArgumentError, match="shape"):
        D.solve_host(CFG, H=H[:3], z=z)
    with pytest.raises(InvalidArgumentError, match="shape"):  # undersized G
        D.solve_host(CFG, H=H, z=z, G=np.zeros((2,) + SH, dtype=np.complex128))
    with pytest.raises(InvalidArgumentError, match="complex128"):
        D.solve_host(CFG, H=H, z=z, G=np.zeros((3,) + SH, dtype=np.complex64))
    G = np.zeros((3, 4, 3, 64, 128), dtype=np.complex128)[..., ::2]
    with pytest.raises(InvalidArgumentError, match="contiguous"):
        D.solve_host(CFG, H=H, z=z, G=G)
    with pytest.raises(InvalidArgumentError, match="numpy"):
        D.solve_host(CFG, H=H, z=z, G=[0])


def test_device_buffers_checked():
    H = torch.zeros(SH, dtype=torch.complex128)
    G = torch.zeros((3,) + SH, dtype=torch.complex128)
    with pytest.raises(InvalidArgumentError, match="CUDA"):
        D.solve_device(CFG, H, G)
    with pytest.raises(InvalidArgumentError, match="CUDA"):
        D.fill_h_device(CFG, H)
    with pytest.raises(InvalidArgumentError, match="CUDA"):
        D.solve_device(CFG, np.zeros(SH, dtype=np.complex128), G)


def test_energy_vector_materialised():
    z = CFG.z()
    zz = np.concatenate([z, z])[::2]  # strided view
    v = D._vec(zz)
    assert v.flags.c_contiguous and v.dtype == np.complex128 and np.array_equal(v, zz)
    with pytest.raises(InvalidArgumentError):
        D._vec(np.zeros(3), 4, "sigma")

"""BASELINE configurations at FULL size on the GPU, checked through a size-independent
property: the diagonal-block residual of A G = I,

    R_i = A[i,i-1] G[i-1,i] + A[i,i] G[i,i] + A[i,i+1] G[i+1,i] - I,   max_i ||R_i||_F / sqrt(b),

for every energy (config 2: all 64 energies of the headline step) and for the config-4
DDRGF solve. The element-wise comparison with the compiled reference at full size is
tools/parity_full.py (profiles/r01_parity.md: minutes of CPU time per configuration);
the GPU residuals there are 2e-12 (config 2) and 1.1e-9 (config 4, DDRGF P = 32).
"""
import numpy as np
import pytest
import torch

from paper_2605_19910_b200 import distributed as Dd
from paper_2605_19910_b200 import dyson as D

pytestmark = pytest.mark.gpu


def _residual(H, G, z, sigma):
    """max over layers of ||(A G)_ii - I||_F / sqrt(b); H, G in slot memory [l, 3, col, row]."""
    Hm = H.transpose(-1, -2)  # [l, 3, row, col]
    Gm = G.transpose(-1, -2)
    l, b = Hm.shape[0], Hm.shape[-1]
    eye = torch.eye(b, dtype=Hm.dtype, device=Hm.device)
    Aii = -Hm[:, 1] + (z - sigma)[:, None, None] * eye
    R = Aii @ Gm[:, 1] - eye
    R[1:] += (-Hm[1:, 0]) @ Gm[:-1, 2]   # A[i,i-1] G[i-1,i]
    R[:-1] += (-Hm[:-1, 2]) @ Gm[1:, 0]  # A[i,i+1] G[i+1,i]
    return float((torch.linalg.matrix_norm(R) / b ** 0.5).max())


def test_config2_full_size_residual_gate(gpu):
    cfg = D.CONFIGS[2]
    l, b = cfg.num_layers, cfg.block_size
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    G = torch.empty((cfg.n_energy, l, 3, b, b), dtype=torch.complex128, device="cuda")
    fails = D.solve_device(cfg, H, G)
    assert (fails == -1).all()
    sig = torch.from_numpy(cfg.sigma()).to("cuda")
    worst = 0.0
    for e, z in enumerate(cfg.z()):
        assert torch.isfinite(torch.view_as_real(G[e])).all()
        worst = max(worst, _residual(H, G[e], complex(z), sig))
    assert worst <= 1e-9, worst


def test_config4_full_size_ddrgf_residual_gate(gpu):
    cfg = D.CONFIGS[4]
    l, b = cfg.num_layers, cfg.block_size
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    z = complex(cfg.z()[0])
    sig = torch.from_numpy(np.asarray(cfg.sigma())).to("cuda")
    A = -H
    dg = A[:, 1].diagonal(dim1=-2, dim2=-1)
    dg.copy_((dg + z) - sig[:, None])
    G = Dd.ddrgf_distributed(A, l, b, s2=127)  # 32 domains (the bench default)
    del A
    assert torch.isfinite(torch.view_as_real(G)).all()
    assert _residual(H, G, z, sig) <= 1e-8

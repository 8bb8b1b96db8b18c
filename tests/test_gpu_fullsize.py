"""BASELINE configurations at FULL size on the GPU, checked through a size-independent
property: the diagonal-block residual of A G = I,

    R_i = A[i,i-1] G[i-1,i] + A[i,i] G[i,i] + A[i,i+1] G[i+1,i] - I,   max_i ||R_i||_F / sqrt(b),

for every energy (config 2: all 64 energies of the headline step) and for the config-4
DDRGF solve, with gates about 10x the residuals observed on B200 (profiles/r02_parity.md:
config 2 <= 2.6e-11, config 4 DDRGF <= 6e-11), plus a strict element-wise subset: config 2
at four energies spread over the grid against the compiled, unmodified reference
(oracle/_ref), every in-band block <= 1e-10. The full sweep over every energy of every
configuration is tools/parity_full.py.
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
    assert worst <= 2.5e-10, worst


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
    assert _residual(H, G, z, sig) <= 5e-10


def test_config2_full_size_elementwise_vs_reference(gpu):
    """Config 2 at full size (l = 256, b = 256), energies 0, 21, 42, 63: every in-band block
    of the GPU G^R within 1e-10 (relative Frobenius) of the compiled reference rgf_tridiag."""
    from oracle import ref_lib as R

    if not R.available():
        pytest.skip("oracle/_ref not built on this box")
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    import parity_full as PF

    from oracle import dyson_oracle as DO

    cfg = D.CONFIGS[2]
    l, b = cfg.num_layers, cfg.block_size
    es = [0, 21, 42, 63]
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    G = torch.empty((len(es), l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.solve_device(cfg, H, G, z=cfg.z()[es])
    del H
    h = DO.hamiltonian(l, 1, b, cfg.seed)
    SAs = [PF.dyson_slots(h, cfg, e) for e in es]
    refs = PF.ref_solve_many(SAs, 1)
    for q in range(len(es)):
        mx, _, _ = PF.summarize(G[q].cpu().numpy(), refs[q], 1)
        assert mx <= 1e-10, (es[q], mx)

"""Accuracy context for a Dyson configuration (SURVEY.md section 7 hard part 1 protocol):
GPU vs reference RGF, the reference's own input-noise floor (1/2-ulp perturbation of A),
and the diagonal residual gate ||(A G)_ii - I||_F / sqrt(b) for both solutions.

  python tools/accuracy_probe.py --config 3 --energies 17 0
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import bbsi_oracle as O  # noqa: E402
from oracle import dyson_oracle as DO  # noqa: E402
from paper_2605_19910_b200 import dyson as D  # noqa: E402


def residual_diag(a: O.Band, g: O.Band) -> float:
    """max_i ||sum_k A[i,k] G[k,i] - I||_F / sqrt(b) over the band (all needed G blocks are in band)."""
    w, l = a.bandwidth, a.num_layers
    worst = 0.0
    for i in range(l):
        acc = np.zeros_like(a.block(i, 0))
        for off in range(-w, w + 1):
            if a.in_band(i, off):
                acc = acc + a.block(i, off) @ g.block(i + off, -off)
        acc -= np.eye(acc.shape[0])
        worst = max(worst, np.linalg.norm(acc) / np.sqrt(acc.shape[0]))
    return worst


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--energies", type=int, nargs="+", default=[0])
    p.add_argument("--layers", type=int, default=0)
    a_ = p.parse_args()
    import torch

    cfg = D.CONFIGS[a_.config]
    if a_.layers:
        cfg = D.scaled(cfg, num_layers=a_.layers)
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    zs = cfg.z()[a_.energies]
    G = torch.empty((len(zs), l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.solve_device(cfg, H, G, z=zs)
    torch.cuda.synchronize()
    h = DO.hamiltonian(l, w, b, cfg.seed)
    rng = np.random.default_rng(7)
    for q, e in enumerate(a_.energies):
        a = DO.dyson_matrix(h, complex(cfg.z()[e]), cfg.sigma_layers)
        solve = O.rgf_ndiag if w > 1 else O.rgf_tridiag
        ref, _ = solve(a)
        ap = a.copy()
        ap.data = ap.data * (1 + 2.0**-53 * rng.uniform(-1, 1, ap.data.shape))
        noisy, _ = solve(ap)
        gpu = O.Band(ref.layout, np.swapaxes(G[q].cpu().numpy(), -1, -2))
        e_gpu = O.block_errors(gpu, ref)
        e_noise = O.block_errors(noisy, ref)
        print(f"{cfg.name} E={cfg.z()[e].real:+.4f}: gpu-vs-ref max {e_gpu.max():.2e} med {np.median(e_gpu):.2e} | "
              f"ref noise floor max {e_noise.max():.2e} med {np.median(e_noise):.2e} | residual gpu "
              f"{residual_diag(a, gpu):.2e} ref {residual_diag(a, ref):.2e}", flush=True)


if __name__ == "__main__":
    main()

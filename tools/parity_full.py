"""Full-size parity report for the five BASELINE configurations (run on a GPU box).

  python -u tools/parity_full.py [--configs 1 2 3 4 5] | tee gpurun_out/parity_full.log

For each checked energy: max / median per-block relative Frobenius error of the GPU
G^R against the reference RGF algorithm (oracle/bbsi_oracle.py restates rgf.hpp;
scipy zgetrf/zgetrs + numpy zgemm), the reference's own 1/2-ulp input-noise floor,
and the diagonal residual gate ||(A G)_ii - I||_F/sqrt(b) of both solutions
(hard part 1 protocol). Config 5 at full size needs ~174 GB of
host RAM for the CPU oracle; it is checked on a reduced-N_b proxy with the true
b = 768 and eta = 1e-5.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from accuracy_probe import residual_diag  # noqa: E402

from oracle import bbsi_oracle as O  # noqa: E402
from oracle import dyson_oracle as DO  # noqa: E402
from paper_2605_19910_b200 import dyson as D  # noqa: E402


def report(tag, a, ref, got, floor=True):
    e = O.block_errors(got, ref)
    line = f"{tag}: max {e.max():.3e} median {np.median(e):.3e}"
    if floor:
        rng = np.random.default_rng(11)
        ap = a.copy()
        ap.data = ap.data * (1 + 2.0**-53 * rng.uniform(-1, 1, ap.data.shape))
        solve = O.rgf_ndiag if a.bandwidth > 1 else O.rgf_tridiag
        nf = O.block_errors(solve(ap)[0], ref).max()
        line += f" | ref noise floor {nf:.3e}"
    line += f" | residual gpu {residual_diag(a, got):.2e} ref {residual_diag(a, ref):.2e}"
    line += "  PASS(1e-10)" if e.max() <= 1e-10 else "  ABOVE 1e-10"
    print(line, flush=True)


def gpu_batch(cfg, energies=None):
    import torch

    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    z = cfg.z() if energies is None else cfg.z()[energies]
    G = torch.empty((len(z), l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.solve_device(cfg, H, G, z=z)
    torch.cuda.synchronize()
    return H, G


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    args = p.parse_args()
    import torch

    for k in args.configs:
        t0 = time.time()
        cfg = D.CONFIGS[k]
        if k == 5:
            cfg = D.scaled(cfg, num_layers=64, n_energy=8)
        l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
        h = DO.hamiltonian(l, w, b, cfg.seed)
        solve = O.rgf_ndiag if w > 1 else O.rgf_tridiag
        if k in (1, 2, 3, 5):
            es = {1: [0], 2: [0, 21, 42, 63], 3: [0, 17, 31], 5: [0, 7]}[k]
            H, G = gpu_batch(cfg, es)
            for q, e in enumerate(es):
                a = DO.dyson_matrix(h, complex(cfg.z()[e]), cfg.sigma_layers)
                ref, _ = solve(a)
                got = O.Band(ref.layout, np.swapaxes(G[q].cpu().numpy(), -1, -2))
                report(f"config {k} ({cfg.name}) E={cfg.z()[e].real:+.4f} rgf", a, ref, got)
                if k == 1:
                    dense = O.oracle_selected_inverse(a)
                    print(f"config 1 gpu vs dense oracle: {O.max_block_error(got, dense):.3e}; "
                          f"reference rgf vs dense: {O.max_block_error(ref, dense):.3e}", flush=True)
            if k == 5:
                Gd = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
                for e in es:
                    D.solve_ddrgf_device(cfg, H, Gd, 7, energy=e)
                    torch.cuda.synchronize()
                    a = DO.dyson_matrix(h, complex(cfg.z()[e]), 1)
                    ref, _ = solve(a)
                    got = O.Band(ref.layout, np.swapaxes(Gd.cpu().numpy(), -1, -2))
                    report(f"config 5 proxy E={cfg.z()[e].real:+.4f} ddrgf 8 domains", a, ref, got, floor=False)
            del H, G
        if k == 4:
            a = DO.dyson_matrix(h, complex(cfg.z()[0]), 1)
            ref, _ = solve(a)
            print(f"config 4 oracle rgf done in {time.time() - t0:.0f}s", flush=True)
            H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
            D.fill_h_device(cfg, H)
            Gd = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
            for ndom in (2, 4, 8, 32):
                D.solve_ddrgf_device(cfg, H, Gd, l // ndom - 1)
                torch.cuda.synchronize()
                got = O.Band(ref.layout, np.swapaxes(Gd.cpu().numpy(), -1, -2))
                report(f"config 4 ddrgf P={ndom}", a, ref, got, floor=(ndom == 2))
            del H, Gd
        torch.cuda.empty_cache()
        print(f"config {k} checked in {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()

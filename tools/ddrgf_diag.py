"""Where does the DDRGF error come from? Config 4 (or a proxy) against the compiled
reference: per solve, max block error and residual split into interface rows (within
one layer of a separator or a chain start) and interior rows, for several domain
counts and fake-lead strengths gamma (BBSI_DDRGF_GAMMA).

  python -u tools/ddrgf_diag.py [--layers 4096] [--domains 2 8 32] [--gammas 1]
"""
import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import parity_full as PF  # noqa: E402

from oracle import dyson_oracle as DO  # noqa: E402
from paper_2605_19910_b200 import dyson as D  # noqa: E402


def rows_near_interfaces(l, s2):
    rows = set()
    pos = 0
    while pos < l:
        sep = pos + s2
        for r in (pos - 1, pos, pos + 1, sep - 1, sep, sep + 1):
            if 0 <= r < l:
                rows.add(r)
        pos += s2 + 1
    m = np.zeros(l, bool)
    m[list(rows)] = True
    return m


def main():
    import torch

    p = argparse.ArgumentParser()
    p.add_argument("--layers", type=int, default=4096)
    p.add_argument("--block", type=int, default=256)
    p.add_argument("--domains", type=int, nargs="+", default=[2, 8, 32])
    p.add_argument("--gammas", type=float, nargs="+", default=[1.0])
    p.add_argument("--refine", type=int, nargs="+", default=[1], help="BBSI_DDRGF_REFINE values to compare")
    a = p.parse_args()
    cfg = D.scaled(D.CONFIGS[4], num_layers=a.layers, block_size=a.block)
    l, b = cfg.num_layers, cfg.block_size
    t0 = time.time()
    SA = PF.dyson_slots(DO.hamiltonian(l, 1, b, cfg.seed), cfg, 0)
    Sr = PF.ref_solve_many([SA], 1, os.cpu_count() or 1)[0]
    print(f"reference in {time.time() - t0:.0f}s; residual ref {PF.residual_rows(SA, Sr, 1).max():.2e}", flush=True)
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    Gd = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.solve_device(cfg, H, Gd.view(1, l, 3, b, b))
    Sg = Gd.cpu().numpy()
    e = PF.block_errors(Sg, Sr, 1)
    print(f"gpu rgf: max {np.nanmax(e):.3e} residual {PF.residual_rows(SA, Sg, 1).max():.2e}", flush=True)
    for P in a.domains:
        s2 = -(-l // P) - 1
        near = rows_near_interfaces(l, s2)
        for g, rf in [(g, rf) for g in a.gammas for rf in a.refine]:
            os.environ["BBSI_DDRGF_GAMMA"] = str(g)
            os.environ["BBSI_DDRGF_REFINE"] = str(rf)
            D.solve_ddrgf_device(cfg, H, Gd, s2)
            torch.cuda.synchronize()
            Sg = Gd.cpu().numpy()
            e = PF.block_errors(Sg, Sr, 1)
            r = PF.residual_rows(SA, Sg, 1)
            er = np.nanmax(e, axis=1)
            wr = int(np.nanargmax(er))
            print(f"P={P:3d} gamma={g:g} refine={rf}: max {np.nanmax(e):.3e} (interface rows {er[near].max():.3e}, interior "
                  f"{er[~near].max():.3e}, worst row {wr}) | residual interface {r[near].max():.2e} interior "
                  f"{r[~near].max():.2e} worst row {int(np.argmax(r))}", flush=True)
    os.environ.pop("BBSI_DDRGF_GAMMA", None)


if __name__ == "__main__":
    main()

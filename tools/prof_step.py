"""One resident Dyson solve for profiling (ncu / compute-sanitizer targets).

  python tools/prof_step.py --config 2 --layers 8 --energies 64 [--reps 1]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--layers", type=int, default=8)
    p.add_argument("--energies", type=int, default=64)
    p.add_argument("--reps", type=int, default=1)
    a = p.parse_args()
    import torch

    from paper_2605_19910_b200 import dyson as D

    cfg = D.scaled(D.CONFIGS[a.config], num_layers=a.layers, n_energy=a.energies)
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    G = torch.empty((cfg.n_energy, l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    from paper_2605_19910_b200._native import lib

    for r in range(a.reps):
        torch.cuda.synchronize()
        n0 = lib().bbsi_cuda_launch_count()
        t0 = time.perf_counter()
        D.solve_device(cfg, H, G)
        torch.cuda.synchronize()
        print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.2f} ms, {lib().bbsi_cuda_launch_count() - n0} launches",
              flush=True)


if __name__ == "__main__":
    main()

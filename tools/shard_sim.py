"""Per-GPU work of the energy-sharded config-2 bench at N = 1/2/4/8 GPUs, on one GPU:
the resident Dyson solve of 64/N energies (CUDA-graph replay, CUDA-event time).

  BBSI_GROUPS=1 python tools/shard_sim.py [--energies 64 32 16 8]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--energies", type=int, nargs="+", default=[64, 32, 16, 8])
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    import torch

    from paper_2605_19910_b200 import dyson as D

    cfg = D.CONFIGS[2]
    l, b = cfg.num_layers, cfg.block_size
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    zs = cfg.z()
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    for n in a.energies:
        G = torch.empty((n, l, 3, b, b), dtype=torch.complex128, device="cuda")
        z = zs[:n]
        for _ in range(3):
            D.solve_device(cfg, H, G, z=z, stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            D.solve_device(cfg, H, G, z=z, stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"{n:3d} energies: {ms:8.1f} ms  ({n / (ms * 1e-3):6.1f} energies/s on this GPU; "
              f"x{64 // n} GPUs would give {64 / (ms * 1e-3):6.1f} energies/s)", flush=True)
        del G
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

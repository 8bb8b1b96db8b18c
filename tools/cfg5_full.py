"""Config 5 at full size on one B200 (l = 2048, b = 768, E = -1, eta = 1e-5; 58 GB per
band): device-resident two-ended RGF and stabilised DDRGF (P = 8 domains), timed, and
their G^R compared block by block (the CPU reference would need ~174 GB of host RAM,
SURVEY.md 8(c), so this is the GPU self-consistency check of the full-size case).

  python -u tools/cfg5_full.py [--domains 8]
"""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--domains", type=int, default=8)
    a = p.parse_args()
    import torch

    from paper_2605_19910_b200 import distributed as Dd
    from paper_2605_19910_b200 import dyson as D
    from paper_2605_19910_b200._native import lib

    cfg = D.CONFIGS[5]
    l, b = cfg.num_layers, cfg.block_size
    z = cfg.z()[:1]
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device=dev)
    D.fill_h_device(cfg, H)
    G = torch.empty((1, l, 3, b, b), dtype=torch.complex128, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D.solve_device(cfg, H, G, z=z, stream=st)
    torch.cuda.synchronize()
    t_rgf = time.perf_counter() - t0
    print(f"config 5 full size, E={z[0].real:+.1f}: two-ended RGF {t_rgf:.2f} s "
          f"({l / t_rgf:.0f} selected inversions/s, {D.algorithmic_flops(cfg) / t_rgf / 1e12:.2f} TFLOP/s)",
          flush=True)
    g_rgf = G[0].cpu().numpy()
    del G
    lib().bbsi_cuda_release_workspace()
    torch.cuda.empty_cache()
    # A = z I - H - Sigma in place of H (diagonal entries in csrc/band_ops.cu's order)
    A = H
    A.neg_()
    sig = torch.from_numpy(np.asarray(cfg.sigma(), dtype=np.complex128)).to(dev)
    dg = A[:, 1].diagonal(dim1=-2, dim2=-1)
    dg.copy_((dg + complex(z[0])) - sig[:, None])
    s2 = -(-l // a.domains) - 1
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Gd = Dd.ddrgf_distributed(A, l, b, s2)
    torch.cuda.synchronize()
    t_dd = time.perf_counter() - t0
    print(f"config 5 full size: DDRGF P={len(Dd.partition(l, s2))} {t_dd:.2f} s ({l / t_dd:.0f} selected inversions/s)",
          flush=True)
    del A
    g_dd = Gd.cpu().numpy()
    del Gd
    worst, where = 0.0, None
    for layer in range(l):
        for off in (-1, 0, 1):
            if not 0 <= layer + off < l:
                continue
            r, d = g_rgf[layer, off + 1], g_dd[layer, off + 1]
            e = np.linalg.norm(d - r) / np.linalg.norm(r)
            if e > worst:
                worst, where = e, (layer, layer + off)
    print(f"config 5 full size: DDRGF vs RGF max block rel. Frobenius difference {worst:.3e} at block {where}",
          flush=True)


if __name__ == "__main__":
    main()

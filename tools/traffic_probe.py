"""One eager step of a bench workload, for the DRAM-traffic probe bench.py runs under
ncu (the roofline's `traffic`): the same launches as the timed step, no CUDA graph.

  python tools/traffic_probe.py --config 2            # Dyson batch (configs 1-3)
  python tools/traffic_probe.py --config 4 --domains 32   # one energy of the DDRGF arm
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--domains", type=int, default=0)
    a = p.parse_args()
    import os

    os.environ["BBSI_GRAPHS"] = "0"
    import torch

    from paper_2605_19910_b200 import distributed as Dd
    from paper_2605_19910_b200 import dyson as D

    cfg = D.CONFIGS[a.config]
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    if a.config in (1, 2, 3):
        H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
        D.fill_h_device(cfg, H)
        G = torch.empty((cfg.n_energy, l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
        D.solve_device(cfg, H, G)
    else:
        P = a.domains or (32 if a.config == 4 else 8)
        s2 = -(-l // P) - 1
        A = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
        D.fill_h_rows_device(cfg, A, 0, l)
        hd = A[:, 1].diagonal(dim1=-2, dim2=-1).clone()
        A.neg_()
        sig = torch.from_numpy(cfg.sigma()).to(A.device)
        A[:, 1].diagonal(dim1=-2, dim2=-1).copy_((complex(cfg.z()[0]) - hd) - sig[:, None])
        G = torch.empty_like(A)
        comm = Dd.NcclComm()
        Dd.ddrgf_nccl(comm, A, G, l, b, s2)
        comm.close()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()

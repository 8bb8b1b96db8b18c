"""Phase timing of one GJ panel (matrix 0, panel k = 32) from clock64 marks.

Needs the instrumented library: python paper_2605_19910_b200/build.py --debug-zinv, then
BBSI_LIB=paper_2605_19910_b200/_lib/libbbsi_cuda_dbg.so python tools/dbg_zinv.py
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2605_19910_b200 import dyson as D  # noqa: E402
from paper_2605_19910_b200._native import lib  # noqa: E402

NAMES = ["load+tol", "LU loop", "lmap", "Wz+barrier", "Vs prefetch+fix", "Pinv", "Vs stage", "V dmma", "scatter+end"]
cfg = D.scaled(D.CONFIGS[2], num_layers=4, n_energy=64)
l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
H = torch.empty((l, 3, b, b), dtype=torch.complex128, device='cuda')
D.fill_h_device(cfg, H)
G = torch.empty((64, l, 3, b, b), dtype=torch.complex128, device='cuda')
for rep in range(3):
    D.solve_device(cfg, H, G)
    torch.cuda.synchronize()
    out = np.zeros(64, dtype=np.int64)
    lib().bbsi_debug_zinv(out.ctypes.data_as(C.c_void_p))
    t = out[:10]
    d = np.diff(t)
    print("total", t[9] - t[0], "cycles |", " ".join(f"{n}={v}" for n, v in zip(NAMES, d)))

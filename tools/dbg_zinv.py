"""Phase timing of one Gauss-Jordan step (matrix 0, step k = 32) from clock64 marks.

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

PAIR = [(10, 11, "load"), (11, 12, "LU1"), (12, 13, "lmap1"), (13, 14, "-"), (14, 15, "Pinv1"),
        (15, 16, "Vs1 stage"), (16, 17, "V1 dmma"), (17, 18, "Wz1 + M2"), (18, 21, "load2"), (21, 22, "LU2"),
        (22, 23, "lmap2"), (23, 24, "Wz fixes"), (24, 25, "Pinv2"), (25, 26, "Vs2"), (26, 27, "V2 dmma"),
        (27, 28, "end")]
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
    print("pair step total", out[28] - out[10], "cycles |",
          " ".join(f"{name}={out[b_] - out[a_]}" for a_, b_, name in PAIR if name != "-"))

import ctypes as C, numpy as np, sys
sys.path.insert(0, '.')
import torch
from paper_2605_19910_b200 import dyson as D
from paper_2605_19910_b200._native import lib
cfg = D.scaled(D.CONFIGS[2], num_layers=4, n_energy=64)
l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
H = torch.empty((l, 3, b, b), dtype=torch.complex128, device='cuda'); D.fill_h_device(cfg, H)
G = torch.empty((64, l, 3, b, b), dtype=torch.complex128, device='cuda')
for rep in range(2):
    D.solve_device(cfg, H, G); torch.cuda.synchronize()
    L = C.CDLL(str(lib()._name)); out = np.zeros(64, dtype=np.int64); L.bbsi_debug_zinv(out.ctypes.data_as(C.c_void_p))
    t = out - out[0]
    print("phases (cycles from start): tol/load", t[1], "LU end", t[2], "rowmap+pinv end", t[3], "wz/vs end", t[4])
    print("per-column starts:", np.diff(out[10:18]))
    print("col1: resolve", out[20]-out[11], "perm", out[21]-out[20], "crcp", out[22]-out[21], "update", out[23]-out[22], "publish", out[24]-out[23])

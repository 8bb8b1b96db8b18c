"""Phase timing of one gj_rows_kernel step (matrix 0, step k = 32) from clock64 marks.

Needs the instrumented library: python paper_2605_19910_b200/build.py --debug-zinv, then
BBSI_LIB=paper_2605_19910_b200/_lib/libbbsi_cuda_dbg.so python tools/dbg_zinv_rows.py [--block 256]
"""
import argparse
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2605_19910_b200._native import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--block", type=int, default=256)
ap.add_argument("--batch", type=int, default=128)
a = ap.parse_args()
MARKS = [(30, 31, "setup+load"), (31, 32, "publish0"), (32, 33, "GJ1 (16 cols)"), (33, 34, "wait Vs1 + W1s"),
         (34, 35, "M2"), (35, 40, "publish0'"), (40, 41, "GJ2 (16 cols)"), (41, 44, "Wz out"), (44, 45, "w1p2"),
         (45, 46, "Vs2 + V out"), (46, 47, "end")]
n = a.block
rng = np.random.default_rng(0)
m = torch.from_numpy(rng.uniform(-1, 1, (a.batch, n, n)) + 1j * rng.uniform(-1, 1, (a.batch, n, n))).cuda()
st = np.zeros(a.batch, dtype=np.int32)
for rep in range(3):
    x = m.clone()
    rc = lib().bbsi_cuda_zinv_dev(n, n, a.batch, C.c_void_p(x.data_ptr()), n, n * n, st.ctypes.data_as(C.c_void_p),
                                  C.c_void_p(0))
    assert rc == 0
    torch.cuda.synchronize()
    out = np.zeros(64, dtype=np.int64)
    lib().bbsi_debug_zinv(out.ctypes.data_as(C.c_void_p))
    print(f"n={n} batch={a.batch}: step total", out[47] - out[30], "cycles |",
          " ".join(f"{name}={out[b_] - out[a_]}" for a_, b_, name in MARKS))

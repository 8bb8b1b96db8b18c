"""compute-sanitizer target: batched inversions through gj_rows_kernel (one CTA and clusters).

  compute-sanitizer --tool racecheck python tools/sanitize_zinv.py
  compute-sanitizer --tool memcheck  python tools/sanitize_zinv.py
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2605_19910_b200._native import lib  # noqa: E402

for n, batch in ((64, 2), (128, 2), (256, 2), (512, 1), (768, 1)):
    rng = np.random.default_rng(n)
    a = rng.uniform(-1, 1, (batch, n, n)) + 1j * rng.uniform(-1, 1, (batch, n, n))
    d = torch.from_numpy(a).cuda()
    st = np.zeros(batch, dtype=np.int32)
    rc = lib().bbsi_cuda_zinv_dev(n, n, batch, C.c_void_p(d.data_ptr()), n, n * n, st.ctypes.data_as(C.c_void_p),
                                  C.c_void_p(0))
    torch.cuda.synchronize()
    got = np.swapaxes(d.cpu().numpy(), -1, -2)
    ref = np.linalg.inv(np.swapaxes(a, -1, -2))
    print(n, batch, "rc", rc, "status", st.tolist(), "err", float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))

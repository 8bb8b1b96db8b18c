"""Device->host 2D copy bandwidth for the e2e hand-off shape (rows of one band row-block
per energy, pitch = one energy's band)."""
import ctypes as C
import glob
import os
import time

import torch

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
    glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = C.CDLL(cands[0])
band_b = 256 * 3 * 256 * 256 * 16  # one energy's band (config 2): 768 MiB... per layer 3 MiB
row_b = 3 * 256 * 256 * 16
ne = 32
d = torch.empty(ne * band_b // 16, dtype=torch.complex128, device="cuda")
h = torch.empty(ne * band_b // 16, dtype=torch.complex128).pin_memory()
s = torch.cuda.Stream()
for rows in (8, 32, 256):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for r0 in range(0, 256, rows):
        rc = rt.cudaMemcpy2DAsync(C.c_void_p(h.data_ptr() + r0 * row_b), C.c_size_t(band_b),
                                  C.c_void_p(d.data_ptr() + r0 * row_b), C.c_size_t(band_b),
                                  C.c_size_t(rows * row_b), C.c_size_t(ne), 2, C.c_void_p(s.cuda_stream))
        assert rc == 0, rc
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"2D hand-offs of {rows} rows x {ne} energies: {ne * band_b / dt / 1e9:.1f} GB/s")
t = time.perf_counter()
h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"1D: {ne * band_b / (time.perf_counter() - t) / 1e9:.1f} GB/s")

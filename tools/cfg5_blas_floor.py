"""CPU only: the config-5 BLAS-rounding floor per energy. The streaming reference
restatement (oracle/stream, scipy OpenBLAS 0.3.31) runs twice on the SAME A(E): once with
the library's native kernels (SkylakeX / AVX-512 on these hosts) and once in a child
process with OPENBLAS_CORETYPE=Haswell (the AVX2 kernels of the same library: same
algorithm, same calls, only the rounding order inside the BLAS kernels differs). The two
streams are compared block by block in lockstep (the child pipes its blocks to the
parent), so no band is ever held. One record per energy:
  {"config": 5, "kind": "floor_blas", "energy_index": e, "floor": max block error, ...}

  python -u tools/cfg5_blas_floor.py [--energies 0 1 ...] [--layers 2048] >> profiles/r02_cfg5_floor_blas.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def child(e: int, layers: int, ckpt: int):
    from oracle import stream_lib as S
    from paper_2605_19910_b200 import dyson as D

    cfg = D.CONFIGS[5]
    l, b = layers, cfg.block_size
    S.use_fast(True)
    S.set_threads(1)
    st = S.DysonStream(l, b, cfg.seed, complex(cfg.z()[e]), cfg.sigma_layers, ckpt=ckpt)
    out = sys.stdout.buffer
    zero = np.zeros((b, b), dtype=np.complex128)
    while True:
        r = st.next()
        if r is None:
            break
        for x in r[1:]:
            out.write(np.ascontiguousarray(zero if x is None else x).tobytes())
    out.flush()


def run_energy(e: int, layers: int, ckpt: int, core: str, lock):
    from oracle import stream_lib as S
    from paper_2605_19910_b200 import dyson as D

    cfg = D.CONFIGS[5]
    l, b = layers, cfg.block_size
    t0 = time.time()
    env = dict(os.environ, OPENBLAS_CORETYPE=core, OPENBLAS_NUM_THREADS="1")
    p = subprocess.Popen([sys.executable, "-u", __file__, "--child", str(e), "--layers", str(l), "--ckpt", str(ckpt)],
                         stdout=subprocess.PIPE, env=env)
    st = S.DysonStream(l, b, cfg.seed, complex(cfg.z()[e]), cfg.sigma_layers, ckpt=ckpt)
    nbytes = 16 * b * b
    errs = []
    while True:
        r = st.next()
        if r is None:
            break
        for x in r[1:]:
            buf = p.stdout.read(nbytes)
            if len(buf) != nbytes:
                raise RuntimeError(f"energy {e}: child stream ended early")
            if x is None:
                continue
            y = np.frombuffer(buf, dtype=np.complex128).reshape(b, b)
            errs.append(float(np.linalg.norm(y - x) / np.linalg.norm(x)))
    p.wait()
    with lock:
        print(json.dumps({"config": 5, "workload": cfg.name, "kind": "floor_blas", "energy_index": int(e),
                          "E": float(cfg.z()[e].real), "layers": l, "floor": max(errs),
                          "floor_median": float(np.median(errs)),
                          "oracle": f"oracle/stream (scipy OpenBLAS 0.3.31), native kernels vs OPENBLAS_CORETYPE={core}",
                          "seconds": round(time.time() - t0, 1)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--energies", type=int, nargs="*", default=list(range(8)))
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--ckpt", type=int, default=64)
    ap.add_argument("--core", default="Haswell")
    ap.add_argument("--child", type=int, default=None)
    a = ap.parse_args()
    from paper_2605_19910_b200 import dyson as D

    layers = a.layers or D.CONFIGS[5].num_layers
    if a.child is not None:
        child(a.child, layers, a.ckpt)
        return
    from oracle import stream_lib as S

    S.use_fast(True)
    S.set_threads(1)
    lock = threading.Lock()
    ths = [threading.Thread(target=run_energy, args=(e, layers, a.ckpt, a.core, lock)) for e in a.energies]
    for t in ths:
        t.start()
    for t in ths:
        t.join()


if __name__ == "__main__":
    main()

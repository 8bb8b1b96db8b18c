"""Full-size parity of the GPU selected inversion against the reference, all five
BASELINE configurations (run on a GPU box; writes one JSON record per checked solve).

  python -u tools/parity_full.py --configs 1 2 3 4 --out gpurun_out/parity.jsonl
  python -u tools/parity_full.py --configs 5 --out gpurun_out/parity5.jsonl

Oracles (the checker, never the product path):
  * configs 1-4: the compiled, unmodified reference (oracle/_ref: rgf_tridiag /
    rgf_ndiag on OpenBLAS 0.3.15), every energy of the grid;
  * config 5 (58 GB per band; the reference's own rgf_tridiag would need ~174 GB of
    host RAM next to the GPU result): the streaming restatement oracle/stream
    (the reference's calls in the reference's order, rgf.hpp:37-76; bitwise equal
    to oracle/_ref on the 0.3.15 build, <= 1e-13 on the faster scipy-OpenBLAS
    build used here, tests/test_oracle.py), all 8 energies, GPU RGF and GPU DDRGF
    (8 domains) compared in the same pass.

Per solve: max / median of the per-block relative Frobenius error
||G_gpu - G_ref||_F / ||G_ref||_F over every in-band block (north_star's metric,
bar 1e-10), the reference's own floor at that energy, and the residual
max_i ||(A G)_ii - I||_F / sqrt(b) of the GPU and of the reference solution.
The floor is how far the reference moves from itself under perturbations no
implementation controls, the max of
  floor_input: the reference on A vs on A with every real/imaginary component moved
               one ulp up or down with probability 1/2 (input rounding, mean 1/2 ulp);
  floor_blas:  the reference vs the SAME unmodified reference linked against another
               OpenBLAS build (0.3.31 instead of 0.3.15: only the rounding order of the
               BLAS kernels differs; oracle/_ref/libbbsi_ref_scipy.so).
An implementation whose residual matches the reference's is as close to it as the
reference is to itself; the verdict is "<= 1e-10", else "<= floor", else "ABOVE".
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import dyson_oracle as DO  # noqa: E402
from oracle import ref_lib as R  # noqa: E402
from paper_2605_19910_b200 import dyson as D  # noqa: E402

BAR = 1e-10
OUT = None


def emit(rec: dict):
    m = rec.get("max")
    fl = rec.get("floor")
    if m is not None:
        if m <= BAR:
            rec["verdict"] = "<= 1e-10"
        elif fl is not None and m <= fl:
            rec["verdict"] = "<= floor"
        else:
            rec["verdict"] = "ABOVE"
    print(json.dumps(rec), flush=True)
    if OUT:
        with open(OUT, "a") as f:
            f.write(json.dumps(rec) + "\n")


# ------------------------------------------------------------------ slot-memory helpers
# slot memory: complex128 [l, 2w+1, b(col), b(row)] (each block column-major, C ABI order)
def in_band_mask(l, w):
    a = np.arange(l)[:, None]
    off = np.arange(-w, w + 1)[None, :]
    return (a + off >= 0) & (a + off < l)


def block_errors(Sg, Sr, w):
    """(l, 2w+1) relative Frobenius errors, NaN outside the band."""
    l = Sr.shape[0]
    num = np.linalg.norm((Sg - Sr).reshape(l, 2 * w + 1, -1), axis=-1)
    den = np.linalg.norm(Sr.reshape(l, 2 * w + 1, -1), axis=-1)
    e = np.where(den > 0, num / np.where(den > 0, den, 1), num)
    e[~in_band_mask(l, w)] = np.nan
    return e


def residual_rows(SA, SG, w):
    """max over rows i of ||sum_off A[i,i+off] G[i+off,i] - I||_F / sqrt(b) (slot memory:
    transposed blocks, so R^T = sum_off G^T[i+off, -off] A^T[i, off])."""
    l, b = SA.shape[0], SA.shape[-1]
    R_ = np.zeros((l, b, b), dtype=np.complex128)
    for off in range(-w, w + 1):
        lo, hi = max(0, -off), min(l, l - off)
        R_[lo:hi] += np.matmul(SG[lo + off:hi + off, w - off], SA[lo:hi, w + off])
    R_ -= np.eye(b)[None]
    return np.linalg.norm(R_.reshape(l, -1), axis=-1) / np.sqrt(b)


def perturb(S, seed):
    """Every real/imaginary component moved one ulp up or down with probability 1/2."""
    x = S.view(np.float64)
    rng = np.random.default_rng(seed)
    move = rng.random(x.shape) < 0.5
    up = rng.random(x.shape) < 0.5
    y = np.where(move, np.where(up, np.nextafter(x, np.inf), np.nextafter(x, -np.inf)), x)
    return y.view(np.complex128).reshape(S.shape)


def ref_solve_many(SAs, w, threads_per_solve=1, scipy_blas=False):
    """Compiled reference rgf_tridiag / rgf_ndiag on each slot array, one host thread each
    (scipy_blas: the same reference built on scipy's OpenBLAS 0.3.31)."""
    L = R.lib_scipy() if scipy_blas else R.lib()
    L.ref_set_threads(C.c_int(threads_per_solve))
    outs = [np.zeros_like(a) for a in SAs]
    errs = []

    def run(k):
        l, b = SAs[k].shape[0], SAs[k].shape[-1]
        fail = C.c_int(-1)
        fn = L.ref_rgf_tridiag if w == 1 else L.ref_rgf_ndiag
        args = [l, w, b, None, SAs[k].ctypes.data_as(C.c_void_p), outs[k].ctypes.data_as(C.c_void_p), None]
        if w != 1:
            args.append(None)
        rc = fn(*args, C.byref(fail))
        if rc:
            errs.append((k, rc, fail.value))

    ths = [threading.Thread(target=run, args=(k,)) for k in range(len(SAs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise RuntimeError(f"reference failed: {errs}")
    return outs


def dyson_slots(h_band, cfg, e):
    return R.to_slots(DO.dyson_matrix(h_band, complex(cfg.z()[e]), cfg.sigma_layers))


def summarize(Sg, Sr, w):
    e = block_errors(Sg, Sr, w)
    v = e[~np.isnan(e)]
    return float(v.max()), float(np.median(v)), e


# ------------------------------------------------------------------ configs 1-3 (batched RGF)
def check_batched(k, energies=None, group=16):
    import torch

    cfg = D.CONFIGS[k]
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    n_all = cfg.n_energy
    es = list(range(n_all)) if energies is None else energies
    t0 = time.time()
    H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    z = cfg.z()[es]
    G = torch.empty((len(es), l, 2 * w + 1, b, b), dtype=torch.complex128, device="cuda")
    D.solve_device(cfg, H, G, z=z)
    torch.cuda.synchronize()
    print(f"config {k}: GPU solve of {len(es)} energies done", flush=True)
    del H
    h = DO.hamiltonian(l, w, b, cfg.seed)
    for g0 in range(0, len(es), group):
        idx = es[g0:g0 + group]
        SAs = [dyson_slots(h, cfg, e) for e in idx]
        SPs = [perturb(a, 1000 + e) for a, e in zip(SAs, idx)]
        refs = ref_solve_many(SAs + SPs, w)
        refs_b = ref_solve_many(SAs, w, scipy_blas=True)
        for q, e in enumerate(idx):
            Sr, Sp = refs[q], refs[len(idx) + q]
            Sg = G[g0 + q].cpu().numpy()
            mx, md, _ = summarize(Sg, Sr, w)
            fi = summarize(Sp, Sr, w)[0]
            fb = summarize(refs_b[q], Sr, w)[0]
            rec = {"config": k, "workload": cfg.name, "solver": "gpu rgf (batched, default path)",
                   "energy_index": int(e), "E": float(cfg.z()[e].real), "max": mx, "median": md,
                   "floor": max(fi, fb), "floor_input": fi, "floor_blas": fb,
                   "residual_gpu": float(residual_rows(SAs[q], Sg, w).max()),
                   "residual_ref": float(residual_rows(SAs[q], Sr, w).max()),
                   "oracle": "oracle/_ref (compiled reference, OpenBLAS 0.3.15)"}
            if k == 1:
                dense = R.oracle_selected_inverse(R.from_slots(R.O.make_layout(l, b, w), SAs[q]))
                Sd = R.to_slots(dense)
                rec["gpu_vs_dense"] = summarize(Sg, Sd, w)[0]
                rec["ref_vs_dense"] = summarize(Sr, Sd, w)[0]
            emit(rec)
        del SAs, SPs, refs, refs_b
    print(f"config {k} checked in {time.time() - t0:.0f}s", flush=True)


# ------------------------------------------------------------------ config 4 (DDRGF, one energy)
def check_cfg4(domains=(2, 4, 8, 16, 32)):
    import torch

    cfg = D.CONFIGS[4]
    l, w, b = cfg.num_layers, 1, cfg.block_size
    t0 = time.time()
    nproc = os.cpu_count() or 1
    h = DO.hamiltonian(l, w, b, cfg.seed)
    SA = dyson_slots(h, cfg, 0)
    del h
    Sr = ref_solve_many([SA], w, nproc)[0]
    Sp = ref_solve_many([perturb(SA, 4000)], w, nproc)[0]
    fi = summarize(Sp, Sr, w)[0]
    del Sp
    Sp = ref_solve_many([SA], w, nproc, scipy_blas=True)[0]
    fb = summarize(Sp, Sr, w)[0]
    del Sp
    fl = max(fi, fb)
    print(f"config 4: references in {time.time() - t0:.0f}s, floor input {fi:.3e} blas {fb:.3e}", flush=True)
    res_ref = float(residual_rows(SA, Sr, w).max())
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    Gd = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    runs = [("gpu rgf (two-ended)", None)] + [(f"gpu ddrgf P={P}", P) for P in domains]
    for name, P in runs:
        if P is None:
            D.solve_device(cfg, H, Gd.view(1, l, 3, b, b))
        else:
            D.solve_ddrgf_device(cfg, H, Gd, -(-l // P) - 1)
        torch.cuda.synchronize()
        Sg = Gd.cpu().numpy()
        mx, md, e = summarize(Sg, Sr, w)
        emit({"config": 4, "workload": cfg.name, "solver": name, "energy_index": 0, "E": float(cfg.z()[0].real),
              "max": mx, "median": md, "floor": fl, "floor_input": fi, "floor_blas": fb,
              "residual_gpu": float(residual_rows(SA, Sg, w).max()),
              "residual_ref": res_ref, "worst_block": [int(x) for x in np.unravel_index(np.nanargmax(e), e.shape)],
              "oracle": "oracle/_ref (compiled reference, OpenBLAS 0.3.15)"})
        del Sg
    print(f"config 4 checked in {time.time() - t0:.0f}s", flush=True)


# ------------------------------------------------------------------ config 5 (streaming oracle)
def check_cfg5(energies, domains=8, resid_every=16, floor_file=None):
    import torch

    from oracle import stream_lib as S

    cfg = D.CONFIGS[5]
    l, b = cfg.num_layers, cfg.block_size
    S.use_fast(True)
    S.set_threads(os.cpu_count() or 1)
    floors = {}
    if floor_file and Path(floor_file).exists():
        for line in open(floor_file):
            r = json.loads(line)
            floors[r["energy_index"]] = r["floor"]
    s2 = -(-l // domains) - 1
    seps = set()
    pos = 0
    while pos < l:  # interface rows of the DDRGF partition (partition.hpp:39-75)
        seps.update({pos, pos + s2 - 1, pos + s2, pos + s2 + 1})
        pos += s2 + 1
    rows = sorted({i for i in range(l) if i % resid_every == 0} | {i for i in seps if 0 <= i < l})
    for e in energies:
        t0 = time.time()
        z = complex(cfg.z()[e])
        # GPU RGF (Dyson batch of one energy), result to pinned host memory
        H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
        D.fill_h_device(cfg, H)
        G = torch.empty((1, l, 3, b, b), dtype=torch.complex128, device="cuda")
        D.solve_device(cfg, H, G, z=np.array([z]))
        torch.cuda.synchronize()
        Grgf = torch.empty((l, 3, b, b), dtype=torch.complex128).pin_memory()
        Grgf.copy_(G[0])
        del G
        from paper_2605_19910_b200._native import lib

        lib().bbsi_cuda_release_workspace()
        torch.cuda.empty_cache()
        # A(E) in place of H (58 GB each: H, G and the DDRGF workspace do not fit next to a
        # separate A): off-diagonal -h, diagonal (z + (-h)) - sigma == (z - h) - sigma exactly
        A = H.neg_()
        del H
        dg = A[:, 1].diagonal(dim1=-2, dim2=-1)
        sig = torch.from_numpy(cfg.sigma()).to(A.device)
        dg.copy_((z + dg) - sig[:, None])
        Gdd = torch.empty_like(A)
        fail = C.c_int(-1)
        rc = lib().bbsi_cuda_ddrgf_dev(l, b, s2, C.c_void_p(A.data_ptr()), C.c_void_p(Gdd.data_ptr()), C.byref(fail),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        if rc != 0:
            raise RuntimeError(f"ddrgf failed rc={rc}: {lib().bbsi_cuda_last_error()}")
        del A, dg
        lib().bbsi_cuda_release_workspace()
        torch.cuda.empty_cache()
        t_gpu = time.time() - t0
        st = S.DysonStream(l, b, cfg.seed, z, cfg.sigma_layers)
        errs = {"rgf": np.full((l, 3), np.nan), "ddrgf": np.full((l, 3), np.nan)}
        res = {"ref": [], "rgf": [], "ddrgf": []}
        prev = {}  # solution -> (G[i-1,i-1]^T, G[i-1,i]^T (row i-1 -> col i), G[i-2,i-1]) in slot form
        cur_rows = {}
        hold = {}
        srcs = {"rgf": lambda a, s: Grgf[a, s].numpy(), "ddrgf": lambda a, s: Gdd[a, s].cpu().numpy()}
        A_cache = {}

        def A_slot(a, off):
            key = (a, off)
            if key not in A_cache:
                A_cache[key] = st.block(a, off).T.copy()  # slot (column-major) form
            return A_cache[key]

        keep = {}  # (sol, a, slot) -> slot block for residual rows
        while True:
            r = st.next()
            if r is None:
                break
            i, gd, gu, glo = r
            ref_blocks = {(i, 1): gd.T.copy()}
            if i > 0:
                ref_blocks[(i - 1, 2)] = gu.T.copy()  # G[i-1, i] lives in slot (i-1, +1)
                ref_blocks[(i, 0)] = glo.T.copy()     # G[i, i-1] in slot (i, -1)
            for (a, s), Rb in ref_blocks.items():
                nr = np.linalg.norm(Rb)
                for name, f in srcs.items():
                    Gb = f(a, s)
                    errs[name][a, s] = np.linalg.norm(Gb - Rb) / nr
                    if a in rows or a + 1 in rows or a - 1 in rows:
                        keep[(name, a, s)] = Gb.copy()
                if a in rows or a + 1 in rows or a - 1 in rows:
                    keep[("ref", a, s)] = Rb
            # row i-1 is complete once G[i, i-1] exists (and at the end for row l-1)
            done = [i - 1] if i > 0 else []
            if i == l - 1:
                done.append(l - 1)
            for row in done:
                if row in rows:
                    for name in ("ref", "rgf", "ddrgf"):
                        acc = np.zeros((b, b), dtype=np.complex128)
                        for off in (-1, 0, 1):
                            c = row + off
                            if 0 <= c < l:
                                acc += keep[(name, c, 1 - off)] @ A_slot(row, off)
                        acc -= np.eye(b)
                        res[name].append(np.linalg.norm(acc) / np.sqrt(b))
                for kk in [k_ for k_ in keep if k_[1] < row - 1]:
                    del keep[kk]
                for kk in [k_ for k_ in A_cache if k_[0] < row]:
                    del A_cache[kk]
        del st
        fl = floors.get(e)
        for name in ("rgf", "ddrgf"):
            v = errs[name][~np.isnan(errs[name])]
            emit({"config": 5, "workload": cfg.name, "solver": "gpu rgf (two-ended)" if name == "rgf" else
                  f"gpu ddrgf P={domains}", "energy_index": int(e), "E": float(z.real), "max": float(v.max()),
                  "median": float(np.median(v)), "floor": fl, "residual_gpu": float(max(res[name])),
                  "residual_ref": float(max(res["ref"])), "residual_rows": len(res["ref"]),
                  "worst_block": [int(x) for x in np.unravel_index(np.nanargmax(errs[name]), errs[name].shape)],
                  "oracle": "oracle/stream (streaming rgf_tridiag restatement, scipy OpenBLAS 0.3.31)",
                  "seconds": {"gpu": round(t_gpu, 1), "total": round(time.time() - t0, 1)}})
        del Grgf, Gdd
        torch.cuda.empty_cache()


def floor_cfg5(energies, ckpt=64, threads=None):
    """CPU only: config-5 noise floor per energy (streaming reference on A vs on the
    one-ulp-perturbed A), energies in parallel host threads, 1 BLAS thread each."""
    from oracle import stream_lib as S

    cfg = D.CONFIGS[5]
    l, b = cfg.num_layers, cfg.block_size
    S.use_fast(True)
    S.set_threads(1)
    lock = threading.Lock()

    def run(e):
        t0 = time.time()
        z = complex(cfg.z()[e])
        a = S.DysonStream(l, b, cfg.seed, z, cfg.sigma_layers, ckpt=ckpt)
        p = S.DysonStream(l, b, cfg.seed, z, cfg.sigma_layers, pert=0.5, pert_seed=5000 + e, ckpt=ckpt)
        worst = 0.0
        errs = []
        while True:
            ra, rp = a.next(), p.next()
            if ra is None:
                break
            for x, y in zip(ra[1:], rp[1:]):
                if x is not None:
                    v = float(np.linalg.norm(y - x) / np.linalg.norm(x))
                    errs.append(v)
                    worst = max(worst, v)
        with lock:
            emit({"config": 5, "workload": cfg.name, "kind": "floor", "energy_index": int(e), "E": z.real,
                  "floor": worst, "floor_median": float(np.median(errs)),
                  "oracle": "oracle/stream (scipy OpenBLAS 0.3.31), perturbed: one ulp on each component w.p. 1/2",
                  "seconds": round(time.time() - t0, 1)})

    ths = [threading.Thread(target=run, args=(e,)) for e in energies]
    for t in ths:
        t.start()
    for t in ths:
        t.join()


def main():
    global OUT
    p = argparse.ArgumentParser()
    p.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4])
    p.add_argument("--energies", type=int, nargs="*", default=None)
    p.add_argument("--out", default=None)
    p.add_argument("--cfg5-floor", action="store_true", help="CPU only: config-5 floors (no GPU)")
    p.add_argument("--floor-file", default=str(ROOT / "profiles" / "r02_cfg5_floor.jsonl"))
    args = p.parse_args()
    OUT = args.out
    if args.cfg5_floor:
        floor_cfg5(args.energies if args.energies else list(range(8)))
        return
    for k in args.configs:
        if k in (1, 2, 3):
            check_batched(k, args.energies)
        elif k == 4:
            check_cfg4()
        elif k == 5:
            check_cfg5(args.energies if args.energies else list(range(8)), floor_file=args.floor_file)


if __name__ == "__main__":
    main()

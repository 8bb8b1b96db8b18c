#!/usr/bin/env python
"""Benchmark: batched selected inversion of the BASELINE Dyson matrices on B200.

Workload (N=1 default): BASELINE.json configs[1] -- block-tridiagonal RGF, N_b=256,
b=256, complex128, 64 energies in [-1.5, 1.5], eta=1e-4, seed 1 (synthetic, seeded;
BASELINE names no dataset). A "step" is the selected inversion of all 64 energies
(diagonal + off-diagonal G^R blocks). Energies shard contiguously across ranks
(strong scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]
  python bench.py --config 4 [--domains P]     DDRGF of config 4 (one energy), P domains
                                                sharded over the ranks (NCCL all-gather of
                                                the corner packets, distributed.py)

Prints ONE JSON line (rank 0). Keys beyond the driver contract:
  roofline      dominant kernel (the DMMA GEMM) vs the FP64 DMMA peak measured live
  cpu_baseline  compiled reference rgf_tridiag (oracle/_ref) on a bounded sample, host cores
  e2e           same metric through the host-buffer C ABI (H2D of H, D2H of every G band)
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "selected inversions/s (energy pts x blocks / s)"
UNIT = "energy_pts*blocks/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--domains", type=int, default=0, help="config 4: DDRGF domains (0 = max(32, world))")
    p.add_argument("--chunk", type=int, default=0, help="energy chunk of the e2e path (0 = library default: ~32 energies per chunk from 48 energies up)")
    return p.parse_args()


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" in r[2 + i]
                          and "Not" not in r[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------- CPU reference
def energy_sample(n_all: int, k: int) -> list:
    """k energy indices spread over the whole grid (both ends included)."""
    k = max(1, min(k, n_all))
    return sorted({int(round(x)) for x in np.linspace(0, n_all - 1, k)})


def cpu_inputs(cfg, energies):
    """Reference-arm inputs: A(E) = z I - H - Sigma in slot memory from the oracle's own
    restatement of the generator (oracle/dyson_oracle.py), so no repo library is mapped
    by the reference process. Built before any timed region."""
    from oracle import dyson_oracle as DO
    from oracle import ref_lib as R

    h = DO.hamiltonian(cfg.num_layers, cfg.bandwidth, cfg.block_size, cfg.seed)
    zs = cfg.z()
    return [R.to_slots(DO.dyson_matrix(h, complex(zs[e]), cfg.sigma_layers)) for e in energies]


def cpu_reference(cfg, inputs, threads_per_energy: int):
    """Times the compiled, unmodified reference rgf_tridiag / rgf_ndiag (oracle/_ref) on
    the prepared inputs (one host thread each, threads_per_energy BLAS threads each).
    Returns seconds."""
    from oracle import ref_lib as R

    L = R.lib()
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    fn = L.ref_rgf_tridiag if w == 1 else L.ref_rgf_ndiag
    L.ref_set_threads(C.c_int(threads_per_energy))
    outs = [np.empty_like(a) for a in inputs]
    errs = []

    def run(e):
        fail = C.c_int(-1)
        args = [l, w, b, None, inputs[e].ctypes.data_as(C.c_void_p), outs[e].ctypes.data_as(C.c_void_p), None]
        if w != 1:
            args.append(None)
        rc = fn(*args, C.byref(fail))
        if rc != 0:
            errs.append(rc)

    t0 = time.perf_counter()
    ths = [threading.Thread(target=run, args=(e,)) for e in range(len(inputs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    if errs:
        raise RuntimeError(f"reference solve failed: {errs}")
    return dt


def cpu_baseline_block(cfg, nproc: int):
    """Best of (i) energy-parallel, 1 BLAS thread per energy and (ii) one energy with
    nproc BLAS threads. The energies span the whole grid."""
    idx = energy_sample(cfg.n_energy, nproc)
    inputs = cpu_inputs(cfg, idx)
    t_par = cpu_reference(cfg, inputs, 1)
    t_one = cpu_reference(cfg, inputs[len(inputs) // 2: len(inputs) // 2 + 1], nproc)
    r_par, r_one = len(idx) / t_par, 1 / t_one
    if r_par >= r_one:
        rate, sample, cores = r_par, f"energies {idx} of {cfg.name}, one per host thread, 1 BLAS thread each", \
            min(nproc, len(idx))
    else:
        rate, sample, cores = r_one, f"energy {idx[len(idx) // 2]} of {cfg.name}, {nproc} BLAS threads", nproc
    return {"value": rate * cfg.num_layers, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": sample, "seconds": {"energy_parallel": round(t_par, 3), "threaded_blas": round(t_one, 3)},
            "energies_per_s": rate}


def workload_config(cfg, n_energies: int) -> dict:
    """The `config` object of both arms (identical keys and values)."""
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    gb = 16 * l * (2 * w + 1) * b * b * n_energies / 2**30
    return {"workload": cfg.name, "num_layers": l, "block_size": b, "bandwidth": w, "energies": n_energies,
            "eta": cfg.eta, "seed": cfg.seed,
            "l2": (f"inputs larger than L2 (G band {gb:.1f} GiB)" if gb * 2**30 > 126e6 else
                   "L2-resident workload (below the 126 MB L2; not flushed)")}


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    from paper_2605_19910_b200.dyson import CONFIGS

    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    nproc = os.cpu_count() or 1
    idx = energy_sample(cfg.n_energy, nproc)
    inputs = cpu_inputs(cfg, idx)  # outside the timed region
    for _ in range(args.warmup):
        cpu_reference(cfg, inputs, 1)
    times = [cpu_reference(cfg, inputs, 1) for _ in range(args.steps)]
    tot = sum(times)
    value = args.steps * len(idx) * cfg.num_layers / tot
    sample = (f"energies {idx} of the {cfg.n_energy}-point grid per step, one per host thread, 1 BLAS thread "
              f"each (compiled reference, oracle/_ref)")
    maps = Path("/proc/self/maps").read_text() if Path("/proc/self/maps").exists() else ""
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded Dyson generator; oracle/dyson_oracle.py restatement)",
            "config": workload_config(cfg, cfg.n_energy),
            "solver": "reference rgf_tridiag / rgf_ndiag (oracle/_ref: unmodified headers, OpenBLAS 0.3.15)",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": len(idx), "kind": "reference",
                             "sample": sample},
            "repo_library_mapped": "libbbsi_cuda" in maps,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2605_19910_b200 import dyson as D
    from paper_2605_19910_b200._native import lib

    L = lib()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = D.CONFIGS[args.config]
    l, w, b = cfg.num_layers, cfg.bandwidth, cfg.block_size
    zs_all = cfg.z()
    n_all = len(zs_all)
    lo, hi = rank * n_all // world, (rank + 1) * n_all // world
    zs = zs_all[lo:hi]
    n_loc = len(zs)

    H = torch.empty((l, 2 * w + 1, b, b), dtype=torch.complex128, device=dev)
    D.fill_h_device(cfg, H)
    G = torch.empty((n_loc, l, 2 * w + 1, b, b), dtype=torch.complex128, device=dev)
    # a dedicated (non-default) stream: the library captures the static per-step
    # launch sequence into a CUDA graph after the first call (legacy stream 0 cannot be captured)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    def step():
        D.solve_device(cfg, H, G, z=zs, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    n0 = L.bbsi_cuda_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = L.bbsi_cuda_launch_count() - n0
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = n_all * l / (ms_step * 1e-3)
    flops_energy = D.algorithmic_flops(cfg)
    tflops = n_all * flops_energy / (ms_step * 1e-3) / 1e12

    # ---- per-kernel breakdown of one step (CUDA events around every library launch).
    # One stream group, so every launch runs alone and its event time is its own
    # duration (with two groups the events of concurrent launches overlap).
    old_groups = os.environ.get("BBSI_GROUPS")
    os.environ["BBSI_GROUPS"] = "1"
    L.bbsi_cuda_profile_enable(1)
    step()
    torch.cuda.synchronize()
    L.bbsi_cuda_profile_enable(0)
    if old_groups is None:
        del os.environ["BBSI_GROUPS"]
    else:
        os.environ["BBSI_GROUPS"] = old_groups
    prof = np.zeros(16)
    L.bbsi_cuda_profile_collect(prof.ctypes.data_as(C.c_void_p), 4)
    cats = {}
    for i, name in enumerate(["zgemm_dmma", "gj_panel", "band_ops", "gj_gemm"]):
        cnt, tms, fl, by = prof[4 * i: 4 * i + 4]
        cats[name] = {"launches": int(cnt), "ms": round(tms, 3),
                      "tflops": round(fl / (tms * 1e-3) / 1e12, 3) if tms > 0 else None,
                      "gbs": round(by / (tms * 1e-3) / 1e9, 1) if tms > 0 else None}
    peak = L.bbsi_cuda_fp64_peak_tflops(50.0, 5)
    g = cats["zgemm_dmma"]
    step_kernel_ms = sum(c["ms"] for c in cats.values())
    roofline = {"bound": "tensor", "kernel": "zgemm_grouped_kernel (DMMA f64), sweep launches "
                "(its Gauss-Jordan launches are listed as gj_gemm)", "achieved": g["tflops"],
                "peak": round(peak, 2), "unit": "TFLOP/s", "frac": round(g["tflops"] / peak, 4) if peak > 0 else None,
                # dram read + write of one sweep-GEMM launch (window + um of both chains of
                # one 32-energy stream group, 2048 tiles) from the ncu --set full capture
                # in profiles/r01_ncu_kernels.md
                "traffic": 297.07e6, "traffic_unit": "bytes per launch (win+um, 2048 tiles)",
                "peak_source": "FP64 DMMA peak measured live in this run (bbsi_cuda_fp64_peak_tflops; "
                               "MEASURED_PEAKS.json has no FP64 entry)",
                "share_of_step": round(g["ms"] / step_kernel_ms, 3) if step_kernel_ms else None,
                "step_algorithmic_tflops": round(tflops / world, 3),
                "step_frac_of_peak": round(tflops / world / peak, 4) if peak > 0 else None,
                "kernels": cats}

    # ---- end to end through the host-buffer C ABI
    e2e = None
    if not args.no_e2e:
        del G  # the resident result band (48 GiB at config 2): the host path allocates its own
        torch.cuda.empty_cache()
        band = l * (2 * w + 1) * b * b
        Hh = torch.from_numpy(D.fill_h_host(cfg)).pin_memory()
        Gh = torch.empty((n_loc, l, 2 * w + 1, b, b), dtype=torch.complex128).pin_memory()
        zz = np.ascontiguousarray(zs, dtype=np.complex128)

        Hn, Gn = Hh.numpy(), Gh.numpy()

        def e2e_step():  # the public host-buffer API: H in, every G band streamed back
            D.solve_host(cfg, H=Hn, z=zz, G=Gn, chunk=args.chunk)

        for _ in range(2):  # eager call, then the CUDA-graph capture (pinned buffers); time replays
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        # the PCIe device->host rate of this box (4 GiB pinned copy, best of 3): G's bytes at
        # that rate are the floor of this path
        dbuf = torch.empty(1 << 28, dtype=torch.complex128, device=dev)
        hbuf = torch.empty(1 << 28, dtype=torch.complex128).pin_memory()
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            hbuf.copy_(dbuf, non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, dbuf.numel() * 16 / (time.perf_counter() - t1) / 1e9)
        del dbuf, hbuf
        d2h_b = 16 * band * n_loc
        e2e = {"value": n_all * l / dt, "unit": UNIT, "ms_per_step": round(dt * 1e3, 2),
               "pcie_d2h_gbs": round(best, 1), "d2h_floor_ms": round(d2h_b / (best * 1e9) * 1e3, 1),
               "h2d_bytes_per_step": int(16 * band + 16 * n_loc + 16 * l) * world,
               "d2h_bytes_per_step": int(16 * band * n_loc + 4 * n_loc) * world,
               "path": "bbsi_cuda_dyson_rgf_z (host H in, every G band out, pinned host memory)"}
        del Hh, Gh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_block(cfg, os.cpu_count() or 1)
        except Exception as ex:  # the GPU number stands without it
            cpu = {"error": str(ex)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic (seeded Dyson generator, "
                "csrc/dyson_gen.h)",
                "config": workload_config(cfg, n_all), "solver": "rgf (batched two-ended sweeps)",
                "parallelism": f"energy shards x{world}",
                "energies_per_s": n_all / (ms_step * 1e-3), "tflops_algorithmic": tflops,
                "gpu_launches": int(launches), "clocks": clocks.summary(), "roofline": roofline,
                "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- DDRGF arm (config 4)
def run_ddrgf(args, rank, world, local_rank):
    """Config 4 (l = 4096, b = 256, E = 0.1, one energy): stabilised DDRGF with P domains,
    contiguous task ranges per rank; the only collective is the all-gather of the
    per-task interface packets (paper_2605_19910_b200/distributed.py). Strong scaling."""
    import torch
    import torch.distributed as dist

    from paper_2605_19910_b200 import distributed as Dd
    from paper_2605_19910_b200 import dyson as D
    from paper_2605_19910_b200._native import lib

    L = lib()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = D.CONFIGS[args.config]
    l, b = cfg.num_layers, cfg.block_size
    P = args.domains or max(32, world)
    s2 = -(-l // P) - 1
    tasks = Dd.partition(l, s2)
    t0, t1 = Dd.task_ranges(len(tasks), world)[rank]
    L0, L1 = Dd.layer_range(tasks, t0, t1)
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device=dev)
    D.fill_h_device(cfg, H)
    A = -H[L0:L1].clone()  # this rank's band rows of A = z I - H - Sigma (slot order)
    del H
    z = complex(cfg.z()[0])
    sig = torch.from_numpy(np.asarray(cfg.sigma()[L0:L1], dtype=np.complex128)).to(dev)
    dg = A[:, 1].diagonal(dim1=-2, dim2=-1)
    dg.copy_((dg + z) - sig[:, None])  # (z - H_aa) - sigma_a, the order of csrc/band_ops.cu
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    def step():
        return Dd.ddrgf_distributed(A, l, b, s2)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    barrier()
    n0 = L.bbsi_cuda_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = L.bbsi_cuda_launch_count() - n0
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    flops = D.algorithmic_flops(cfg)
    if rank == 0:
        line = {"metric": METRIC, "value": l / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
                "data": "synthetic (seeded Dyson generator, csrc/dyson_gen.h)",
                "config": {"workload": cfg.name, "num_layers": l, "block_size": b, "bandwidth": 1, "energies": 1,
                           "eta": cfg.eta, "seed": cfg.seed, "solver": "stabilised ddrgf (DESIGN.md section 5)",
                           "domains": len(tasks), "s2": s2,
                           "parallelism": f"ddrgf domains over {world} rank(s), NCCL all-gather of the corner packets",
                           "l2": "inputs larger than L2 (A band 12 GiB)"},
                "tflops_rgf_equivalent": flops / (ms_step * 1e-3) / 1e12, "gpu_launches": int(launches),
                "clocks": clocks.summary(), "roofline": None, "e2e": None, "cpu_baseline": None}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.config == 4:
        run_ddrgf(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

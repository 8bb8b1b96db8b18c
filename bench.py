#!/usr/bin/env python
"""Benchmark: batched selected inversion of the BASELINE Dyson matrices on B200.

Workload (N=1 default): BASELINE.json configs[1] -- block-tridiagonal RGF, N_b=256,
b=256, complex128, 64 energies in [-1.5, 1.5], eta=1e-4, seed 1 (synthetic, seeded;
BASELINE names no dataset). A "step" is the selected inversion of all 64 energies
(diagonal + off-diagonal G^R blocks). Energies shard contiguously across ranks
(strong scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]
  python bench.py --config 3                    n-diagonal RGF (w = 2), 32 energies
  python bench.py --config 4|5 [--domains P]   DDRGF of config 4 (one energy, P = 32) / config 5
                                                (8 energies, P = 8); domains sharded over the
                                                ranks, NCCL inside the library

Prints ONE JSON line (rank 0). Keys beyond the driver contract:
  roofline      dominant kernel (the DMMA GEMM) vs the FP64 DMMA peak measured live; its
                DRAM traffic per launch from an ncu probe run in the same bench
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
    p.add_argument("--domains", type=int, default=0, help="configs 4/5: DDRGF domains (0 = 32 / 8, at least world)")
    p.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic probe of the dominant kernel")
    p.add_argument("--levels", type=int, nargs="*", default=None,
                   help="configs 4/5: the DomainPlan's later levels s2_levels[1..] (nested interface system; "
                        "default: DDRGF_LEVELS[config])")
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


# DomainPlan levels above the first (ddrgf.hpp:18-32, 363-369) the DDRGF arm uses by default
DDRGF_LEVELS = {4: (), 5: ()}
SUBCHAIN = {4: 1024, 5: 48}  # leading layers of the reference's bounded single-energy sample (DDRGF configs)


def cpu_subchain(cfg, nproc: int, k: int):
    """Compiled reference rgf_tridiag on the leading SUBCHAIN[k] layers of the config's
    first energy, nproc BLAS threads (rgf_tridiag costs the same per layer at any chain
    length, so layers/s is the metric's rate). Returns (seconds, layers, sample text)."""
    nl = min(SUBCHAIN[k], cfg.num_layers)
    from paper_2605_19910_b200.dyson import scaled

    sub = scaled(cfg, num_layers=nl)
    t = cpu_reference(sub, cpu_inputs(sub, [0]), nproc)
    return t, nl, (f"layers 0..{nl - 1} of {cfg.name} (one energy, E = {cfg.z()[0].real:g}), {nproc} BLAS threads "
                   f"(compiled reference rgf_tridiag, oracle/_ref)")


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    from paper_2605_19910_b200.dyson import CONFIGS

    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    nproc = os.cpu_count() or 1
    if args.config in (4, 5):
        for _ in range(args.warmup):
            cpu_subchain(cfg, nproc, args.config)
        res = [cpu_subchain(cfg, nproc, args.config) for _ in range(args.steps)]
        tot = sum(r[0] for r in res)
        value = sum(r[1] for r in res) / tot
        sample, cores = res[0][2] + " per step", nproc
    else:
        idx = energy_sample(cfg.n_energy, nproc)
        inputs = cpu_inputs(cfg, idx)  # outside the timed region
        for _ in range(args.warmup):
            cpu_reference(cfg, inputs, 1)
        times = [cpu_reference(cfg, inputs, 1) for _ in range(args.steps)]
        tot = sum(times)
        value = args.steps * len(idx) * cfg.num_layers / tot
        sample = (f"energies {idx} of the {cfg.n_energy}-point grid per step, one per host thread, 1 BLAS thread "
                  f"each (compiled reference, oracle/_ref)")
        cores = len(idx)
    maps = Path("/proc/self/maps").read_text() if Path("/proc/self/maps").exists() else ""
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded Dyson generator; oracle/dyson_oracle.py restatement)",
            "config": workload_config(cfg, cfg.n_energy),
            "solver": "reference rgf_tridiag / rgf_ndiag (oracle/_ref: unmodified headers, OpenBLAS 0.3.15)",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "repo_library_mapped": "libbbsi_cuda" in maps,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- profiling helpers
CATS = ["zgemm_dmma", "gj_panel", "band_ops", "gj_gemm"]


def profile_step(L, step, one_group=True):
    """CUDA events around every library launch of one step (one stream group, so each
    launch's event time is its own duration). Per category: launches, ms, TFLOP/s, GB/s
    (algorithmic flops / bytes the launches declare) and bytes per launch."""
    import torch

    old = os.environ.get("BBSI_GROUPS")
    if one_group:
        os.environ["BBSI_GROUPS"] = "1"
    L.bbsi_cuda_profile_enable(1)
    step()
    torch.cuda.synchronize()
    L.bbsi_cuda_profile_enable(0)
    if one_group:
        if old is None:
            del os.environ["BBSI_GROUPS"]
        else:
            os.environ["BBSI_GROUPS"] = old
    prof = np.zeros(4 * len(CATS))
    L.bbsi_cuda_profile_collect(prof.ctypes.data_as(C.c_void_p), len(CATS))
    cats = {}
    for i, name in enumerate(CATS):
        cnt, tms, fl, by = prof[4 * i: 4 * i + 4]
        cats[name] = {"launches": int(cnt), "ms": round(tms, 3),
                      "tflops": round(fl / (tms * 1e-3) / 1e12, 3) if tms > 0 else None,
                      "gbs": round(by / (tms * 1e-3) / 1e9, 1) if tms > 0 else None,
                      "alg_bytes_per_launch": round(by / cnt) if cnt else None,
                      "flops_per_launch": round(fl / cnt) if cnt else None}
    return cats


def measure_traffic(config: int, domains: int, timeout: float = 240.0):
    """DRAM bytes per launch of the dominant kernel, measured in this run: ncu on a child
    process that runs one eager step of the same workload (tools/traffic_probe.py),
    profiling a few sweep-GEMM launches (zgemm_grouped_kernel<0,...>: the non-plain
    instantiations: the TMA kernel, or the cp.async one with BBSI_TMA=0 -- not the
    Gauss-Jordan updates). None / {"error": ...} if ncu is unavailable or fails."""
    import csv
    import io
    import shutil
    import tempfile

    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not Path(ncu).exists():
        return None
    with tempfile.TemporaryDirectory() as td:
        log = Path(td) / "ncu.csv"
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
               "--clock-control", "none", "--kernel-name-base", "demangled", "--kernel-name",
               "regex:zgemm_(tma_kernel|grouped_kernel<0)", "--launch-skip", "40", "--launch-count", "6", "--csv",
               "--log-file", str(log), sys.executable, str(ROOT / "tools" / "traffic_probe.py"), "--config",
               str(config)]
        if domains:
            cmd += ["--domains", str(domains)]
        try:
            # one stream group, as in profile_step: the profiled launches are the same size
            # (same tiles, same algorithmic bytes) as the ones the roofline divides by
            env = dict(os.environ, BBSI_GROUPS="1")
            subprocess.run(cmd, capture_output=True, timeout=timeout, check=True, env=env)
            text = log.read_text()
        except Exception as ex:  # the bench line stands without it
            return {"error": f"ncu probe failed: {type(ex).__name__}"}
    try:
        start = text.find('"ID"')
        if start < 0:
            return {"error": "ncu probe matched no launches"}
        rows = list(csv.reader(io.StringIO(text[start:])))
        hdr = rows[0]
        ii, im, iv, iu = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        ik = hdr.index("Kernel Name")
        per, names = {}, {}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6,
                 "ms": 1e-3, "s": 1}
        for r in rows[1:]:
            if len(r) <= max(ii, im, iv, iu, ik):
                continue
            v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
            per.setdefault(r[ii], {})[r[im]] = v
            names[r[ii]] = r[ik]
        launches = [d for d in per.values() if "dram__bytes_read.sum" in d]
        if not launches:
            return {"error": "ncu probe: no DRAM metrics in the capture"}
        traffic = statistics.mean(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in launches)
        dur = statistics.mean(d.get("gpu__time_duration.sum", 0.0) for d in launches)
        import re

        kern = sorted({(re.search(r"zgemm_\w+<[^>]*>", n) or re.search(r"\w+", n)).group(0) for n in names.values()})
    except Exception as ex:  # the bench line stands without it
        return {"error": f"ncu probe parse failed: {type(ex).__name__}: {ex}"}
    return {"bytes_per_launch": traffic, "launches_profiled": len(launches), "ncu_mean_duration_us": dur * 1e6,
            "kernels": kern,
            "command": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:zgemm_(tma_kernel|"
                       f"grouped_kernel<0) -s 40 -c 6 python tools/traffic_probe.py --config {config}"}


def roofline_block(cats, peak, traffic, step_tflops, kernel_note):
    g = cats["zgemm_dmma"]
    step_kernel_ms = sum(c["ms"] for c in cats.values())
    out = {"bound": "tensor", "kernel": kernel_note, "achieved": g["tflops"], "peak": round(peak, 2),
           "unit": "TFLOP/s", "frac": round(g["tflops"] / peak, 4) if (peak > 0 and g["tflops"]) else None,
           "traffic": (traffic or {}).get("bytes_per_launch"), "traffic_unit": "DRAM bytes per sweep-GEMM launch "
           "(ncu, this run)", "traffic_probe": traffic,
           "alg_bytes_per_launch": g["alg_bytes_per_launch"],
           "peak_source": "FP64 DMMA peak measured live in this run (bbsi_cuda_fp64_peak_tflops; "
                          "MEASURED_PEAKS.json has no FP64 entry)",
           "share_of_step": round(g["ms"] / step_kernel_ms, 3) if step_kernel_ms else None,
           "step_algorithmic_tflops": round(step_tflops, 3),
           "step_frac_of_peak": round(step_tflops / peak, 4) if peak > 0 else None, "kernels": cats}
    return out


def timed_loop(step, steps, stream, local_rank, world, dev):
    """W warm-up steps are the caller's; here: barrier, K timed steps on `stream` with CUDA
    events, barrier; returns (max-over-ranks ms, launches, clock summary)."""
    import torch
    import torch.distributed as dist

    from paper_2605_19910_b200._native import lib

    L = lib()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = L.bbsi_cuda_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = L.bbsi_cuda_launch_count() - n0
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, launches, clocks.summary()


# ---------------------------------------------------------------------------- our arm (configs 1-3)
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

    for _ in range(max(3, args.warmup)):
        step()
    ms, launches, clocks = timed_loop(step, args.steps, stream, local_rank, world, dev)
    ms_step = ms / args.steps
    value = n_all * l / (ms_step * 1e-3)
    tflops = n_all * D.algorithmic_flops(cfg) / (ms_step * 1e-3) / 1e12

    cats = profile_step(L, step)
    peak = L.bbsi_cuda_fp64_peak_tflops(50.0, 5)
    traffic = None

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
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        best = pcie_d2h_gbs(dev)
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
    if rank == 0 and world == 1 and not args.no_traffic:
        torch.cuda.empty_cache()
        L.bbsi_cuda_release_workspace()
        try:
            traffic = measure_traffic(args.config, 0)
        except Exception as ex:  # never lose the bench line to the probe
            traffic = {"error": f"{type(ex).__name__}: {ex}"}

    if rank == 0:
        roofline = roofline_block(cats, peak, traffic, tflops / world,
                                  "zgemm_grouped_kernel (DMMA f64), sweep launches (its Gauss-Jordan launches are "
                                  "listed as gj_gemm)")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic (seeded Dyson generator, "
                "csrc/dyson_gen.h)",
                "config": workload_config(cfg, n_all), "solver": "rgf (batched sweeps; two-ended for w = 1)",
                "parallelism": f"energy shards x{world}",
                "energies_per_s": n_all / (ms_step * 1e-3), "tflops_algorithmic": tflops,
                "gpu_launches": int(launches), "clocks": clocks, "roofline": roofline,
                "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)


def pcie_d2h_gbs(dev):
    """The box's PCIe device->host rate (4 GiB pinned copy, best of 3)."""
    import torch

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
    return best


# ---------------------------------------------------------------------------- DDRGF arm (configs 4, 5)
def run_ddrgf(args, rank, world, local_rank):
    """Configs 4 and 5: stabilised DDRGF of every energy of the config (4: E = 0.1; 5: the 8
    energies in [-1, 1]), P domains (4: 32, 5: 8, or --domains) sharded over the ranks as
    contiguous task ranges. Inside the library (bbsi_cuda_ddrgf_rank_dev): phase 1, the
    NCCL all-gather of the per-task interface packets, phase 2 (redundant on every
    rank), phase 3 in place, the NCCL all-gather of two halo blocks per rank, the
    couplings. A rank holds only its band rows; per energy only A's diagonal changes.
    Strong scaling (fixed work: all energies x all layers)."""
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
    P = args.domains or max(32 if args.config == 4 else 8, world)
    s2 = -(-l // P) - 1
    t0, t1, L0, L1 = Dd.rank_layers(l, s2, world, rank)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    A = torch.empty((L1 - L0, 3, b, b), dtype=torch.complex128, device=dev)
    D.fill_h_rows_device(cfg, A, L0, L1, stream=stream)
    hd = A[:, 1].diagonal(dim1=-2, dim2=-1).clone()  # H_aa diagonals (real), kept for every energy
    A.neg_()  # A = -H off the diagonal
    sig = torch.from_numpy(cfg.sigma()[L0:L1].copy()).to(dev)
    G = torch.empty_like(A)
    zs = cfg.z()
    comm = Dd.NcclComm()
    diag = A[:, 1].diagonal(dim1=-2, dim2=-1)

    levels = tuple(args.levels) if args.levels is not None else DDRGF_LEVELS[args.config]

    def solve_energy(z):
        diag.copy_((complex(z) - hd) - sig[:, None])  # (z - h) - sigma: the generator's order
        Dd.ddrgf_nccl(comm, A, G, l, b, s2, levels)

    def step():
        for z in zs:
            solve_energy(z)

    for _ in range(max(3, args.warmup)):
        step()
    ms, launches, clocks = timed_loop(step, args.steps, stream, local_rank, world, dev)
    ms_step = ms / args.steps
    n_e = len(zs)
    flops_rgf = n_e * D.algorithmic_flops(cfg)
    tflops = flops_rgf / (ms_step * 1e-3) / 1e12
    cats = profile_step(L, lambda: solve_energy(zs[0]), one_group=True)
    executed = sum((c["flops_per_launch"] or 0) * c["launches"] for c in cats.values())
    peak = L.bbsi_cuda_fp64_peak_tflops(50.0, 5)

    # ---- end to end: host buffers in and out every step (the drop-in bbsi_cuda_ddrgf_z at
    # N = 1; at N > 1 each rank's rows through pinned memory around the rank entry)
    e2e = None
    if not args.no_e2e:
        Ah = torch.empty(A.shape, dtype=A.dtype).pin_memory()
        Gh = torch.empty(A.shape, dtype=A.dtype).pin_memory()
        e2e_energies = zs if args.config == 4 else zs[:1]
        Ah.copy_(A)
        hd_h, sig_h = hd.cpu(), sig.cpu()[:, None]
        dg = Ah[:, 1].diagonal(dim1=-2, dim2=-1)
        if world == 1:  # the drop-in allocates its own device band (config 5: 2 x 58 GB + scratch)
            del A, G, diag
            torch.cuda.empty_cache()
            L.bbsi_cuda_release_workspace()

        def e2e_step():
            for z in e2e_energies:
                dg.copy_((complex(z) - hd_h) - sig_h)  # this energy's A in host memory (the input)
                if world == 1:
                    from paper_2605_19910_b200 import bbsi as B

                    B.ddrgf_slots(Ah.numpy(), Gh.numpy(), l, b, [s2, *levels])
                else:
                    A.copy_(Ah, non_blocking=True)
                    Dd.ddrgf_nccl(comm, A, G, l, b, s2, levels)
                    Gh.copy_(G, non_blocking=True)
                    torch.cuda.synchronize()

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        tt = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - tt) / args.steps
        if world > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        band_b = 16 * 3 * b * b * l
        e2e = {"value": len(e2e_energies) * l / dt, "unit": UNIT, "ms_per_step": round(dt * 1e3, 2),
               "energies_per_step": len(e2e_energies), "h2d_bytes_per_step": band_b * len(e2e_energies),
               "d2h_bytes_per_step": band_b * len(e2e_energies),
               "path": ("bbsi_cuda_ddrgf_z (host A in, host G out, pinned)" if world == 1 else
                        "per rank: pinned host rows -> bbsi_cuda_ddrgf_rank_dev -> pinned host rows")}
        del Ah, Gh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            nproc = os.cpu_count() or 1
            t, nl, sample = cpu_subchain(cfg, nproc, args.config)
            cpu = {"value": nl / t, "unit": UNIT, "cores": nproc, "kind": "reference", "sample": sample,
                   "seconds": round(t, 3)}
        except Exception as ex:
            cpu = {"error": str(ex)}
    traffic = None
    comm.close()
    if rank == 0 and world == 1 and not args.no_traffic:
        A = G = diag = None  # the probe process needs the device memory (config 5: 154 GB)
        torch.cuda.empty_cache()
        L.bbsi_cuda_release_workspace()
        try:
            traffic = measure_traffic(args.config, P)
        except Exception as ex:  # never lose the bench line to the probe
            traffic = {"error": f"{type(ex).__name__}: {ex}"}
    if rank == 0:
        roofline = roofline_block(cats, peak, traffic, tflops / world,
                                  "zgemm_grouped_kernel (DMMA f64): sweep, corner-chain and interface GEMMs of one "
                                  "energy")
        roofline["executed_tflop_per_energy"] = round(executed / 1e12, 3)
        roofline["rgf_equivalent_tflop_per_energy"] = round(D.algorithmic_flops(cfg) / 1e12, 3)
        line = {"metric": METRIC, "value": n_e * l / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
                "data": "synthetic (seeded Dyson generator, csrc/dyson_gen.h)",
                "config": workload_config(cfg, n_e),
                "solver": f"stabilised ddrgf, {len(Dd.partition(l, s2))} domains (DomainPlan s2_levels = "
                          f"{[s2, *levels]}), NCCL inside the library",
                "parallelism": f"ddrgf domains over {world} rank(s)",
                "energies_per_s": n_e / (ms_step * 1e-3), "tflops_rgf_equivalent": tflops,
                "gpu_launches": int(launches), "clocks": clocks, "roofline": roofline, "e2e": e2e,
                "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    # stdout carries ONE JSON line: keep NCCL's "NCCL version ..." banner (NCCL_DEBUG=VERSION) off it
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"
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
    if args.config in (4, 5):
        run_ddrgf(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""`bbsi` command-line front end on the GPU path (tools/bbsi.cpp:108-365 of the reference).

    python -m paper_2605_19910_b200.cli solve    [flags]   run a solver, print a timing record
    python -m paper_2605_19910_b200.cli validate [flags]   same, plus the dense-inverse check
    python -m paper_2605_19910_b200.cli scale --axis layers --grid 20,40,80
    python -m paper_2605_19910_b200.cli bench-kernels --sizes 64,128,256 [--batch B]
    python -m paper_2605_19910_b200.cli tune --layers 4096 --block-size 256 [--execute]

Flags, environment names (BBSI_*), record keys and exit codes follow the reference
CLI (tools/bbsi.cpp:43-63, 149-181, 183-199): 0 ok, 1 validation failed, 2 usage /
solver error. Inputs come from a .bbm file (--matrix, io.cpp format) or from
random_spd_like (--layers/--block-size/--bandwidth/--seed/--dominance). Every solve
runs on the device through the C ABI; `validate` compares with a dense numpy inverse
of the same matrix (the reference's oracle_selected_inverse, block_banded.hpp:136-181),
capped by --oracle-cap like the reference.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

from . import bbsi as B


def _env(name, default, cast):
    v = os.environ.get(name)
    return cast(v) if v is not None else default


def _common(p: argparse.ArgumentParser) -> None:
    """tools/bbsi.cpp:43-63"""
    p.add_argument("--layers", type=int, default=_env("BBSI_LAYERS", 12, int))
    p.add_argument("--block-size", type=int, default=_env("BBSI_BLOCK_SIZE", 8, int))
    p.add_argument("--bandwidth", type=int, default=_env("BBSI_BANDWIDTH", 1, int))
    p.add_argument("--solver", default=_env("BBSI_SOLVER", "rgf", str), help="rgf | nrgf | fused | ddrgf")
    p.add_argument("--plan", default=_env("BBSI_PLAN", "", str), help='ddrgf plan, e.g. "s2:4,1,1"')
    p.add_argument("--threads", type=int, default=_env("BBSI_THREADS", 1, int))
    p.add_argument("--terminal-threads", type=int, default=_env("BBSI_TERMINAL_THREADS", 1, int))
    p.add_argument("--reps", type=int, default=_env("BBSI_REPS", 30, int))
    p.add_argument("--seed", type=int, default=_env("BBSI_SEED", 12345, int))
    p.add_argument("--dominance", type=float, default=_env("BBSI_DOMINANCE", 2.0, float))
    p.add_argument("--validate", action="store_true")
    p.add_argument("--oracle-cap", type=int, default=_env("BBSI_ORACLE_CAP", 4096, int))
    p.add_argument("--tolerance", type=float, default=1e-10)
    p.add_argument("--out", default="")
    p.add_argument("--matrix", default="")


def parse_plan(o) -> B.DomainPlan:
    """tools/bbsi.cpp:75-85"""
    body = o.plan[3:] if o.plan.startswith("s2:") else o.plan
    levels = [int(t) for t in body.split(",") if t]
    return B.DomainPlan(levels or [1], o.threads, o.terminal_threads)


def load_or_generate(o) -> B.BlockBandedMatrix:
    """tools/bbsi.cpp:87-91"""
    if o.matrix:
        return B.read_bbm(o.matrix)
    return B.random_spd_like(B.make_layout(o.layers, o.block_size, o.bandwidth), o.seed, o.dominance)


def run_solver(m: B.BlockBandedMatrix, o):
    """tools/bbsi.cpp:108-138: wall time per call (host buffers in and out, as the
    reference's by-value API)."""
    fns = {"rgf": B.rgf_tridiag, "nrgf": B.rgf_ndiag, "fused": B.rgf_fused}
    if o.solver not in fns and o.solver != "ddrgf":
        raise B.InvalidArgumentError(f"unknown solver: {o.solver}")
    plan = parse_plan(o)
    times, res = [], None
    for _ in range(max(1, o.reps)):
        t0 = time.perf_counter()
        res = B.ddrgf(m, plan) if o.solver == "ddrgf" else fns[o.solver](m)
        times.append((time.perf_counter() - t0) * 1e3)
    return res[0], res[1], times


def run_record(m, o, counters, times) -> dict:
    """tools/bbsi.cpp:163-179"""
    rec = {"solver": o.solver, "layers": m.num_layers, "block_size": m.layout.block_sizes[0],
           "bandwidth": m.bandwidth, "threads": o.threads, "repetitions": max(1, o.reps),
           "wall_time_ms": sum(times) / len(times), "wall_time_ms_min": min(times), "wall_time_ms_max": max(times),
           "seed": o.seed, "counters": {"gemm": counters.n_gemm, "lu": counters.n_lu, "getrs": counters.n_getrs},
           "device": "cuda (sm_100a, libbbsi_cuda.so)"}
    if o.solver == "ddrgf":
        rec["plan"] = parse_plan(o).s2_levels
    return rec


def dense(m: B.BlockBandedMatrix) -> np.ndarray:
    lay = m.layout
    off = np.concatenate([[0], np.cumsum(lay.block_sizes)])
    d = np.zeros((off[-1], off[-1]), dtype=np.complex128)
    for a in range(lay.num_layers):
        for k in range(-lay.bandwidth, lay.bandwidth + 1):
            if m.in_band(a, k):
                d[off[a]:off[a + 1], off[a + k]:off[a + k + 1]] = m.block(a, k)
    return d


def oracle_error(got: B.BlockBandedMatrix, m: B.BlockBandedMatrix):
    """tools/bbsi.cpp:142-160: largest per-block relative Frobenius error against the
    dense inverse, and the (row layer, column layer) where it occurs."""
    lay = m.layout
    off = np.concatenate([[0], np.cumsum(lay.block_sizes)])
    inv = np.linalg.inv(dense(m))
    worst, where = 0.0, (-1, -1)
    for a in range(lay.num_layers):
        for k in range(-lay.bandwidth, lay.bandwidth + 1):
            if not m.in_band(a, k):
                continue
            ref = inv[off[a]:off[a + 1], off[a + k]:off[a + k + 1]]
            nr = np.linalg.norm(ref)
            e = np.linalg.norm(got.block(a, k) - ref) / (nr if nr > 0 else 1.0)
            if e > worst:
                worst, where = float(e), (a, a + k)
    return worst, where


def validate_into(rec: dict, m, o, got) -> int:
    """tools/bbsi.cpp:181-199"""
    n = m.layout.total_dim()
    if n > o.oracle_cap:
        print(f"error: oracle validation requested above --oracle-cap ({n} > {o.oracle_cap})", file=sys.stderr)
        return 2
    err, where = oracle_error(got, m)
    rec["max_block_error"] = err
    if err > o.tolerance:
        print(f"validation FAILED: block ({where[0]}, {where[1]}) relative error {err} > {o.tolerance}",
              file=sys.stderr)
        return 1
    return 0


def emit(o, text: str) -> None:
    if not o.out:
        sys.stdout.write(text)
        return
    try:
        with open(o.out, "w") as f:
            f.write(text)
    except OSError:
        raise B.InvalidArgumentError(f"cannot open output path {o.out}") from None


def loglog_slope(xs, ys) -> float:
    lx, ly = [math.log(x) for x in xs], [math.log(y) for y in ys]
    n = len(xs)
    sx, sy = sum(lx), sum(ly)
    sxx, sxy = sum(x * x for x in lx), sum(x * y for x, y in zip(lx, ly))
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)


def ratios_to_json(r) -> dict:
    """tools/bbsi.cpp:216-222"""
    return {"block_size": r.block_size, "t_gemm_us": r.t_gemm * 1e6, "r_lu": r.r_lu, "r_getrs": r.r_getrs,
            "samples": r.sample_count}


def ratios_from_json(j: dict):
    """tools/bbsi.cpp:224-232"""
    from .tuner import KernelRatios

    return KernelRatios(int(j["block_size"]), float(j["t_gemm_us"]) * 1e-6, float(j["r_lu"]), float(j["r_getrs"]),
                        int(j.get("samples", 0)))


def _pad64(n: int) -> int:
    return max(64, -(-n // 64) * 64)


def bench_kernels(o) -> str:
    """`bench-kernels` (tools/bbsi.cpp:279-290): per block size, the device time of one
    b x b GEMM and the inversion / solve ratios the GPU solvers see, measured as one
    batched launch over --batch blocks (sizes are padded to multiples of 64 as the solvers do)."""
    from . import tuner as T

    lines = ["block_size,t_gemm_us,r_lu,r_getrs,samples"]
    for n in [int(t) for t in o.sizes.split(",") if t]:
        t = T.measure_kernels(_pad64(n), batches=(o.batch,), samples=o.samples or 10)
        r = T.kernel_ratios(t, o.batch)
        lines.append(f"{n},{r.t_gemm * 1e6},{r.r_lu},{r.r_getrs},{o.samples or 10}")
    return "\n".join(lines) + "\n"


def tune(o) -> str:
    """`tune` (tools/bbsi.cpp:318-360): the reference's autotune on GPU-measured ratios (or
    --ratios-file), plus the B200 plan (plan_gpu: energy-batched RGF vs DDRGF domains,
    with the NCCL term across --gpus). --execute times RGF and the chosen DDRGF plan."""
    from . import tuner as T

    times = None
    if o.ratios_file:
        try:
            with open(o.ratios_file) as f:
                ratios = ratios_from_json(json.load(f))
        except OSError:
            raise B.InvalidArgumentError(f"cannot open {o.ratios_file}") from None
    else:
        times = T.measure_kernels(_pad64(o.block_size), samples=o.samples or 5)
        ratios = T.kernel_ratios(times, 1)
    t = T.autotune(o.layers, o.threads, ratios, o.max_levels, o.s2_max)
    out = {"ratios": ratios_to_json(ratios), "choice": "rgf" if t.use_rgf else "ddrgf",
           "rgf_gemm_equivalents": t.rgf_cost.gemm_equivalents,
           "rgf_predicted_seconds": t.rgf_cost.predicted_seconds}
    if t.ddrgf_valid:
        levels = [{"level": k + 1, "s2": s2, "threads": t.plan.n_threads} for k, s2 in enumerate(t.plan.s2_levels)]
        levels.append({"level": len(t.plan.s2_levels) + 1, "terminal": True, "threads": t.plan.terminal_threads})
        out.update({"plan": levels, "ddrgf_gemm_equivalents": t.ddrgf_cost.gemm_equivalents,
                    "ddrgf_predicted_seconds": t.ddrgf_cost.predicted_seconds,
                    "ddrgf_breakdown": t.ddrgf_cost.breakdown})
    if times is not None and o.bandwidth == 1:
        g = T.plan_gpu(o.layers, o.energies, times, o.gpus)
        out["gpu_plan"] = {"solver": g.solver, "s2": g.s2, "domains": g.domains, "energy_batch": g.energy_batch,
                           "gpus": o.gpus, "predicted_seconds": g.predicted_seconds, "breakdown": g.breakdown,
                           "candidates": [{"solver": c[0], "s2": c[1], "predicted_seconds": c[2]}
                                          for c in g.candidates]}
    if o.execute:
        m = load_or_generate(o)
        run = argparse.Namespace(**vars(o))
        run.solver, run.reps = "rgf", max(1, o.reps)
        out["measured_rgf_ms"] = sum(run_solver(m, run)[2]) / run.reps
        plan_s2 = out.get("gpu_plan", {}).get("s2") or (t.plan.s2_levels[0] if t.ddrgf_valid else 0)
        if plan_s2:
            run.solver, run.plan = "ddrgf", f"s2:{plan_s2}"
            out["measured_ddrgf_ms"] = sum(run_solver(m, run)[2]) / run.reps
    return json.dumps(out, indent=2) + "\n"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="bbsi", description="selected inversion of block banded matrices (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    _common(sub.add_parser("solve", help="run a solver, report a timing record"))
    _common(sub.add_parser("validate", help="run a solver and compare to the dense inverse"))
    sc = sub.add_parser("scale", help="sweep one axis, emit CSV and a log-log slope")
    sc.add_argument("--axis", default="layers", help="layers | blocksize | bandwidth | threads")
    sc.add_argument("--grid", default="20,40,80,160")
    _common(sc)
    bk = sub.add_parser("bench-kernels", help="time the GPU GEMM / inversion kernels, emit CSV")
    bk.add_argument("--sizes", default="64,128,256")
    bk.add_argument("--samples", type=int, default=0)
    bk.add_argument("--batch", type=int, default=1, help="blocks per batched launch")
    _common(bk)
    tu = sub.add_parser("tune", help="pick the cheapest solver plan from the cost model")
    tu.add_argument("--max-levels", type=int, default=5)
    tu.add_argument("--s2-max", type=int, default=4)
    tu.add_argument("--execute", action="store_true")
    tu.add_argument("--ratios-file", default="")
    tu.add_argument("--samples", type=int, default=0)
    tu.add_argument("--energies", type=int, default=1, help="energy points of the B200 plan")
    tu.add_argument("--gpus", type=int, default=1, help="GPUs of the B200 plan")
    _common(tu)
    o = ap.parse_args(argv)
    try:
        if o.cmd == "bench-kernels":
            emit(o, bench_kernels(o))
            return 0
        if o.cmd == "tune":
            emit(o, tune(o))
            return 0
        if o.cmd in ("solve", "validate"):
            if o.cmd == "validate":
                o.validate = True
            m = load_or_generate(o)
            got, cnt, times = run_solver(m, o)
            rec = run_record(m, o, cnt, times)
            rc = validate_into(rec, m, o, got) if o.validate else 0
            emit(o, json.dumps(rec, indent=2) + "\n")
            return rc
        lines = ["axis,value,mean_ms,min_ms,max_ms,gemm,lu,getrs"]
        xs, ys = [], []
        attr = {"layers": "layers", "blocksize": "block_size", "bandwidth": "bandwidth", "threads": "threads"}
        if o.axis not in attr:
            raise B.InvalidArgumentError(f"unknown axis: {o.axis}")
        for v in [int(t) for t in o.grid.split(",") if t]:
            run = argparse.Namespace(**vars(o))
            setattr(run, attr[o.axis], v)
            m = load_or_generate(run)
            _, cnt, times = run_solver(m, run)
            mean = sum(times) / len(times)
            lines.append(f"{o.axis},{v},{mean},{min(times)},{max(times)},{cnt.n_gemm},{cnt.n_lu},{cnt.n_getrs}")
            xs.append(v)
            ys.append(mean)
        if o.axis in ("layers", "blocksize") and len(xs) >= 2:
            lines.append(f"# loglog_slope,{loglog_slope(xs, ys)}")
        emit(o, "\n".join(lines) + "\n")
        return 0
    except (B.InvalidArgumentError, B.SingularMatrixError, B.CudaError, ImportError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

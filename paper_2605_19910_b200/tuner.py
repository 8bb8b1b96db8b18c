"""Cost model, auto-tuner and orchestrator: the reference's closed forms
(cost_model.hpp) plus their B200 calibration.

Reference part (same names, formulas, tie-breaks and errors):
  KernelRatios, CostEstimate                  cost_model.hpp:12-38
  rgf_extra_gemms, cost_rgf, cost_nrgf,
  cost_fused, cost_ddrgf                      cost_model.hpp:40-130
  autotune / orchestrate                      cost_model.hpp:156-230

GPU part (this package's executed algorithms, not the reference's CPU threads):
  measure_kernels(n, batches)   device time of one batched GEMM / inversion launch per
                                batch size (bbsi_cuda_bench_kernels), the B200 analogue
                                of benchmark_kernels
  kernel_ratios(t, batch)       KernelRatios from those timings: r_lu = t_inv / t_gemm;
                                r_getrs = 2/3 because the GPU replaces the reference's
                                3 GETRS per layer by 2 GEMMs against the explicit inverse
  predict_rgf_gpu / predict_ddrgf_gpu / plan_gpu
                                launch-level models of the batched (two-ended) RGF and the
                                stabilised DDRGF, with an NCCL term
                                for the corner all-gather when domains span GPUs, and the
                                planner that picks solver, s2 (domains) and energy batch.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .bbsi import DomainPlan, InvalidArgumentError, KernelCounters


# ----------------------------------------------------------------- reference closed forms
@dataclass
class KernelRatios:
    """cost_model.hpp:12-18 (t_gemm in seconds)."""

    block_size: int = 0
    t_gemm: float = 0.0
    r_lu: float = 0.0
    r_getrs: float = 0.0
    sample_count: int = 0


@dataclass
class CostEstimate:
    """cost_model.hpp:22-38: GEMM-equivalents with a breakdown that sums to the total."""

    gemm_equivalents: float = 0.0
    breakdown: dict = field(default_factory=dict)
    predicted_seconds: float = 0.0


def _finish(breakdown: dict, t_gemm: float) -> CostEstimate:
    total = 0.0
    for k in sorted(breakdown):  # std::map iteration order
        total += breakdown[k]
    return CostEstimate(total, breakdown, total * t_gemm)


def rgf_extra_gemms(l: int) -> int:
    """cost_model.hpp:43"""
    return 0 if l <= 2 else (l - 1) * (l - 2)


def predict_rgf_counters(l: int) -> KernelCounters:
    """cost_model.hpp:46-48"""
    return KernelCounters(4 * (l - 1), l, 3 * l - 2)


def predict_nrgf_counters(l: int, w: int) -> KernelCounters:
    """cost_model.hpp:51-53"""
    return KernelCounters((3 * w * w + w) * l - 2 * w ** 3 - 2 * w * w, l, l * (2 * w + 1) - w * w - w)


def cost_rgf(l: int, r: KernelRatios) -> CostEstimate:
    """cost_model.hpp:65-72"""
    if l < 1:
        raise InvalidArgumentError("cost_rgf: l must be >= 1")
    return _finish({"gemm": float(4 * (l - 1)), "lu": float(l) * r.r_lu, "getrs": float(3 * l - 2) * r.r_getrs},
                   r.t_gemm)


def cost_nrgf(l: int, w: int, r: KernelRatios) -> CostEstimate:
    """cost_model.hpp:76-84"""
    if w < 1 or l <= w:
        raise InvalidArgumentError("cost_nrgf: requires l > w >= 1")
    return _finish({"gemm": float((3 * w * w + w) * l - 2 * w ** 3 - 2 * w * w), "lu": float(l) * r.r_lu,
                    "getrs": float(l * (2 * w + 1) - w * w - w) * r.r_getrs}, r.t_gemm)


def cost_fused(l: int, w: int, ratios_at_super: KernelRatios) -> CostEstimate:
    """cost_model.hpp:88-91"""
    if w < 1 or l <= w:
        raise InvalidArgumentError("cost_fused: requires l > w >= 1")
    return cost_rgf((l + w - 1) // w, ratios_at_super)


def cost_ddrgf(l: int, plan: DomainPlan, r: KernelRatios, blas_cap: int = 12) -> CostEstimate:
    """cost_model.hpp:96-124"""
    plan.validate()
    terms = {}
    lk = l
    for k, s2 in enumerate(plan.s2_levels):
        if lk < 1 + s2:
            raise InvalidArgumentError(f"cost_ddrgf: plan exhausts layers at level {k}")
        n_tasks = (lk + s2) // (1 + s2)
        f = float(n_tasks) / float(plan.n_threads)
        p = f"L{k}."
        r_rgf_s2 = float(4 * (s2 - 1)) + float(s2) * r.r_lu + float(3 * s2 - 2) * r.r_getrs
        terms[p + "interior_inv"] = f * (r_rgf_s2 + float(rgf_extra_gemms(s2)))
        terms[p + "coupling_rows"] = f * float(2 * s2)
        terms[p + "coupling_cols"] = f * float(2 * s2)
        terms[p + "schur_assembly"] = f * 4.0
        terms[p + "corr_offdiag_rows"] = f * float(4 * s2)
        terms[p + "corr_offdiag_cols"] = f * 4.0
        terms[p + "corr_diag"] = f * float(6 * s2 - 4)
        lk = n_tasks
    tt = min(plan.terminal_threads, blas_cap)
    terms["terminal"] = cost_rgf(lk, r).gemm_equivalents / float(tt)
    return _finish(terms, r.t_gemm)


def predict_ddrgf_counters(l: int, plan: DomainPlan) -> KernelCounters:
    """cost_model.hpp:137-154"""
    c = KernelCounters()
    lk = l
    for s2 in plan.s2_levels:
        if lk < 1 + s2:
            raise InvalidArgumentError("predict_ddrgf_counters: plan exhausts layers")
        n = (lk + s2) // (1 + s2)
        c = c + KernelCounters(n * (4 * (s2 - 1) + rgf_extra_gemms(s2) + 2 * s2 + 2 * s2 + 4 + 4 * s2 + 4 + 6 * s2 - 4),
                               n * s2, n * (3 * s2 - 2))
        lk = n
    return c + predict_rgf_counters(lk)


@dataclass
class TuneResult:
    """cost_model.hpp:158-165"""

    use_rgf: bool = True
    plan: DomainPlan = field(default_factory=DomainPlan)
    ddrgf_valid: bool = False
    rgf_cost: CostEstimate = field(default_factory=CostEstimate)
    ddrgf_cost: CostEstimate = field(default_factory=CostEstimate)


def autotune(l: int, n_threads: int, r: KernelRatios, max_levels: int = 5, s2_max: int = 4,
             blas_cap: int = 12) -> TuneResult:
    """cost_model.hpp:171-224: exhaustive search, same tie-breaks (fewer levels, then the
    lexicographically smaller sequence, then fewer terminal threads; RGF wins ties)."""
    if l < 1 or n_threads < 1:
        raise InvalidArgumentError("autotune: bad arguments")
    out = TuneResult()
    seq = cost_rgf(l, r)
    scale = 1.0 / float(min(n_threads, blas_cap))
    out.rgf_cost = _finish({k: v * scale for k, v in seq.breakdown.items()}, r.t_gemm)

    def better(est, plan):
        if not out.ddrgf_valid or est.gemm_equivalents < out.ddrgf_cost.gemm_equivalents:
            return True
        if est.gemm_equivalents != out.ddrgf_cost.gemm_equivalents:
            return False
        a, b = plan.s2_levels, out.plan.s2_levels
        if len(a) != len(b):
            return len(a) < len(b)
        if a != b:
            return a < b
        return plan.terminal_threads < out.plan.terminal_threads

    def search(stack):
        if stack:
            for tt in range(1, min(n_threads, blas_cap) + 1):
                plan = DomainPlan(list(stack), n_threads, tt)
                try:
                    est = cost_ddrgf(l, plan, r, blas_cap)
                except InvalidArgumentError:
                    continue
                if better(est, plan):
                    out.ddrgf_valid, out.plan, out.ddrgf_cost = True, plan, est
        if len(stack) == max_levels:
            return
        for s2 in range(1, s2_max + 1):
            search(stack + [s2])

    search([])
    out.use_rgf = not out.ddrgf_valid or out.rgf_cost.gemm_equivalents <= out.ddrgf_cost.gemm_equivalents
    return out


orchestrate = autotune  # cost_model.hpp:228-230


# ----------------------------------------------------------------- B200 calibration
@dataclass
class GpuKernelTimes:
    """Device seconds of ONE batched launch over `batch` n x n blocks (bench_kernels)."""

    n: int
    batches: list
    t_gemm: list
    t_inv: list

    def gemm(self, batch: float) -> float:
        return float(np.interp(batch, self.batches, self.t_gemm, right=None)) if batch <= self.batches[-1] else \
            self.t_gemm[-1] * batch / self.batches[-1]

    def inv(self, batch: float) -> float:
        return float(np.interp(batch, self.batches, self.t_inv)) if batch <= self.batches[-1] else \
            self.t_inv[-1] * batch / self.batches[-1]


def measure_kernels(n: int, batches=(1, 2, 4, 8, 16, 32, 64, 128), samples: int = 5) -> GpuKernelTimes:
    """Times bbsi_cuda_bench_kernels at every batch size (needs a GPU)."""
    import ctypes as C

    from ._native import lib
    from .bbsi import _raise

    tg, ti = [], []
    for b in batches:
        out = np.zeros(3)
        _raise(lib().bbsi_cuda_bench_kernels(int(n), int(b), int(samples), out.ctypes.data_as(C.c_void_p)))
        tg.append(float(out[0]))
        ti.append(float(out[1]))
    return GpuKernelTimes(int(n), list(batches), tg, ti)


def kernel_ratios(t: GpuKernelTimes, batch: int = 1) -> KernelRatios:
    """The reference's KernelRatios seen by the GPU solvers at one batch size."""
    g = t.gemm(batch)
    return KernelRatios(t.n, g, t.inv(batch) / g, 2.0 / 3.0, len(t.batches))


# NVLink 5 through NVSwitch: ~900 GB/s per direction per GPU; one collective ~20 us.
NVLINK_BPS = 900e9
NCCL_LATENCY_S = 20e-6


def predict_rgf_gpu(l: int, n_energy: int, t: GpuKernelTimes, n_gpus: int = 1) -> CostEstimate:
    """Batched two-ended RGF (csrc/rgf.cu rgf_sweeps_two), energies sharded over GPUs:
    l/2 lockstep steps, each one inversion launch over 2E blocks and GEMM launches over
    2E (lm) and 4E (window + um) blocks inward, 4E + 2E outward; the middle inversion."""
    e = -(-n_energy // n_gpus)
    steps = (l - 1 + 1) // 2
    terms = {"inversion": steps * t.inv(2 * e) + t.inv(e),
             "gemm": steps * (2 * t.gemm(2 * e) + 2 * t.gemm(4 * e))}
    return _finish(terms, 1.0)


def predict_ddrgf_gpu(l: int, s2: int, t: GpuKernelTimes, n_gpus: int = 1) -> CostEstimate:
    """Stabilised DDRGF of one energy (csrc/ddrgf.cu), P = ceil(l / (s2+1)) domains spread
    over the GPUs: phase 1 one-ended chain sweeps + corner recurrences over P/G chains,
    the corner all-gather (4 b x b blocks per domain) over NVLink when G > 1, phase 2's
    sequential separator sweeps (b x b work), phase 3 two-ended re-solve of the chains."""
    if s2 < 1 or l < 1 + s2:
        raise InvalidArgumentError("predict_ddrgf_gpu: requires 1 <= s2 <= l - 1")
    P = (l + s2) // (1 + s2)
    p = -(-P // n_gpus)
    blk = 16.0 * t.n * t.n
    terms = {
        "phase1_sweeps": s2 * (t.inv(p) + 2 * t.gemm(p) + 2 * t.gemm(2 * p)),
        "phase1_corners": s2 * t.gemm(2 * p),
        "phase2_separators": P * (2 * t.inv(1) + 8 * t.gemm(1)),
        "phase3_resolve": ((s2 + 2) // 2) * (t.inv(2 * p) + 2 * t.gemm(2 * p) + 2 * t.gemm(4 * p)),
    }
    if n_gpus > 1:
        terms["nccl_allgather"] = NCCL_LATENCY_S + 4 * blk * P * (n_gpus - 1) / n_gpus / NVLINK_BPS
    return _finish(terms, 1.0)


@dataclass
class GpuPlan:
    solver: str                 # "rgf" (energy-batched) or "ddrgf"
    s2: int = 0                 # ddrgf interior group size (domains = ceil(l / (s2+1)))
    domains: int = 0
    energy_batch: int = 0       # energies per GPU launch
    predicted_seconds: float = 0.0
    breakdown: dict = field(default_factory=dict)
    candidates: list = field(default_factory=list)


def plan_gpu(l: int, n_energy: int, t: GpuKernelTimes, n_gpus: int = 1, max_domains: int = 256) -> GpuPlan:
    """Cheapest predicted way to run `n_energy` energies of an l-layer tridiagonal chain:
    energy-batched two-ended RGF, or DDRGF per energy with domains = l/(s2+1) chosen
    among powers of two (ties: RGF, then fewer domains)."""
    rgf = predict_rgf_gpu(l, n_energy, t, n_gpus)
    best = GpuPlan("rgf", energy_batch=-(-n_energy // n_gpus), predicted_seconds=rgf.predicted_seconds,
                   breakdown=rgf.breakdown)
    cands = [("rgf", 0, rgf.predicted_seconds)]
    d = 2
    while d <= min(max_domains, l // 2):
        s2 = -(-l // d) - 1
        if s2 >= 1:
            est = predict_ddrgf_gpu(l, s2, t, n_gpus)
            total = est.predicted_seconds * n_energy
            cands.append(("ddrgf", s2, total))
            if total < best.predicted_seconds:
                best = GpuPlan("ddrgf", s2, (l + s2) // (1 + s2), 1, total, est.breakdown)
        d *= 2
    best.candidates = cands
    return best

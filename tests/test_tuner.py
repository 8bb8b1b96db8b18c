"""Cost model / auto-tuner (paper_2605_19910_b200/tuner.py): the reference's own
test_cost_model.cpp cases restated, every closed form pinned against the compiled
reference (oracle/_ref), and the GPU calibration + planner on a B200."""
import random

import pytest

from oracle import ref_lib as R
from paper_2605_19910_b200 import tuner as T
from paper_2605_19910_b200.bbsi import DomainPlan, InvalidArgumentError


def ratios(r_lu, r_getrs, t_gemm=1.0):
    return T.KernelRatios(64, t_gemm, r_lu, r_getrs, 100)


def test_tridiagonal_cost_formula():  # test_cost_model.cpp:22-37
    assert T.cost_rgf(4, ratios(0, 0)).gemm_equivalents == 12.0
    assert T.cost_rgf(1, ratios(1, 1)).gemm_equivalents == 2.0
    e = T.cost_rgf(10, ratios(2.0, 0.5))
    assert e.gemm_equivalents == pytest.approx(70, rel=1e-14)
    assert (e.breakdown["gemm"], e.breakdown["lu"], e.breakdown["getrs"]) == (36.0, 20.0, 14.0)
    assert sum(e.breakdown.values()) == e.gemm_equivalents
    assert T.cost_rgf(5, ratios(1, 1, 1e-6)).predicted_seconds == pytest.approx(34e-6, rel=1e-12)
    with pytest.raises(InvalidArgumentError):
        T.cost_rgf(0, ratios(1, 1))


def test_ndiag_and_fused_examples():  # test_cost_model.cpp:49-66
    rng = random.Random(1)
    for _ in range(50):
        l = 2 + rng.randrange(200)
        r = ratios(rng.randrange(1000) / 64.0, rng.randrange(1000) / 64.0)
        assert T.cost_nrgf(l, 1, r).gemm_equivalents == T.cost_rgf(l, r).gemm_equivalents
    assert T.cost_nrgf(160, 2, ratios(0, 0)).gemm_equivalents == 2216.0
    assert T.cost_fused(160, 3, ratios(0, 0)).gemm_equivalents == 4.0 * 53
    with pytest.raises(InvalidArgumentError):
        T.cost_nrgf(3, 3, ratios(0, 0))
    with pytest.raises(InvalidArgumentError):
        T.cost_fused(2, 2, ratios(0, 0))


def test_ddrgf_cost_by_hand_and_scaling():  # test_cost_model.cpp:83-135
    e = T.cost_ddrgf(10, DomainPlan([4], 2, 1), ratios(0, 0))
    assert e.breakdown == {"L0.interior_inv": 18.0, "L0.coupling_rows": 8.0, "L0.coupling_cols": 8.0,
                           "L0.schur_assembly": 4.0, "L0.corr_offdiag_rows": 16.0, "L0.corr_offdiag_cols": 4.0,
                           "L0.corr_diag": 20.0, "terminal": 4.0}
    assert e.gemm_equivalents == 82.0
    r = ratios(3, 1.5)
    e2 = T.cost_ddrgf(300, DomainPlan([4, 2], 2), r)
    e8 = T.cost_ddrgf(300, DomainPlan([4, 2], 8), r)
    for k, v in e2.breakdown.items():
        assert e8.breakdown[k] == (v if k == "terminal" else pytest.approx(v / 4.0, rel=1e-12))
    capped = T.cost_ddrgf(100, DomainPlan([4], 4, 4), ratios(1, 1), blas_cap=2)
    two = T.cost_ddrgf(100, DomainPlan([4], 4, 2), ratios(1, 1), blas_cap=2)
    assert capped.breakdown["terminal"] == two.breakdown["terminal"]
    with pytest.raises(InvalidArgumentError):
        T.cost_ddrgf(6, DomainPlan([4, 4], 2), ratios(1, 1))


def test_autotune_cases():  # test_cost_model.cpp:137-199
    assert T.autotune(64, 1, ratios(1, 1)).use_rgf
    t = T.orchestrate(512, 64, ratios(1, 1))
    assert not t.use_rgf and t.ddrgf_valid and t.plan.n_threads == 64
    assert t.ddrgf_cost.gemm_equivalents < t.rgf_cost.gemm_equivalents
    forced = T.autotune(300, 8, ratios(1.3, 0.7), max_levels=0)
    assert forced.use_rgf and not forced.ddrgf_valid


def test_counters_match_reference_closed_forms():
    if not R.available():
        pytest.skip("oracle/_ref not built")
    for l in (2, 5, 31, 160):
        assert T.predict_rgf_counters(l).as_tuple() == (4 * (l - 1), l, 3 * l - 2)
        for lev in ([1], [2], [4, 1], [3, 2, 1]):
            try:
                ref = R.predict_ddrgf_counters(l, lev)
            except Exception:
                with pytest.raises(InvalidArgumentError):
                    T.predict_ddrgf_counters(l, DomainPlan(lev))
                continue
            assert T.predict_ddrgf_counters(l, DomainPlan(lev)).as_tuple() == ref.as_tuple()


def test_costs_and_autotune_pinned_to_reference():
    """Random ratios / plans: every cost term total and every autotune verdict equals
    the compiled reference's (cost_model.hpp), bit for bit."""
    if not R.available():
        pytest.skip("oracle/_ref not built")
    rng = random.Random(7)
    for _ in range(40):
        r_lu, r_getrs, tg = rng.uniform(0, 8), rng.uniform(0, 3), rng.uniform(1e-6, 1e-3)
        r = ratios(r_lu, r_getrs, tg)
        l = rng.randrange(3, 600)
        w = rng.randrange(1, 4)
        assert T.cost_rgf(l, r).gemm_equivalents == R.cost("rgf", l, r_lu=r_lu, r_getrs=r_getrs, t_gemm=tg)[0]
        if l > w:
            assert T.cost_nrgf(l, w, r).gemm_equivalents == R.cost("nrgf", l, w, r_lu=r_lu, r_getrs=r_getrs,
                                                                   t_gemm=tg)[0]
            assert T.cost_fused(l, w, r).predicted_seconds == R.cost("fused", l, w, r_lu=r_lu, r_getrs=r_getrs,
                                                                     t_gemm=tg)[1]
        lev = [rng.randrange(1, 6) for _ in range(rng.randrange(1, 4))]
        nt, tt = rng.randrange(1, 65), rng.randrange(1, 20)
        try:
            ref = R.cost("ddrgf", l, 1, lev, nt, tt, r_lu, r_getrs, tg)
        except Exception:
            with pytest.raises(InvalidArgumentError):
                T.cost_ddrgf(l, DomainPlan(lev, nt, tt), r)
            continue
        got = T.cost_ddrgf(l, DomainPlan(lev, nt, tt), r)
        assert (got.gemm_equivalents, got.predicted_seconds) == ref
    for _ in range(6):
        l, nt = rng.randrange(8, 400), rng.randrange(1, 40)
        r_lu, r_getrs = rng.uniform(0.5, 6), rng.uniform(0.2, 2)
        got = T.autotune(l, nt, ratios(r_lu, r_getrs), max_levels=3, s2_max=4)
        ref = R.autotune(l, nt, r_lu, r_getrs, max_levels=3, s2_max=4)
        assert got.use_rgf == ref["use_rgf"] and got.ddrgf_valid == ref["ddrgf_valid"]
        assert got.rgf_cost.gemm_equivalents == ref["rgf_gemm_equivalents"]
        if got.ddrgf_valid:
            assert got.plan.s2_levels == ref["s2_levels"]
            assert got.plan.terminal_threads == ref["terminal_threads"]
            assert got.ddrgf_cost.gemm_equivalents == ref["ddrgf_gemm_equivalents"]


def test_gpu_models_are_consistent():
    """Planner arithmetic on synthetic timings (no GPU): more GPUs never predict a slower
    energy-sharded RGF, the NCCL term appears only across GPUs, and the plan is the
    cheapest candidate."""
    t = T.GpuKernelTimes(256, [1, 2, 4, 8, 16, 32, 64, 128],
                         [60e-6, 60e-6, 61e-6, 62e-6, 65e-6, 120e-6, 240e-6, 480e-6],
                         [400e-6, 400e-6, 402e-6, 404e-6, 410e-6, 420e-6, 560e-6, 1100e-6])
    one = T.predict_rgf_gpu(256, 64, t, 1).predicted_seconds
    eight = T.predict_rgf_gpu(256, 64, t, 8).predicted_seconds
    assert eight < one
    assert "nccl_allgather" not in T.predict_ddrgf_gpu(4096, 63, t, 1).breakdown
    assert T.predict_ddrgf_gpu(4096, 63, t, 8).breakdown["nccl_allgather"] > 0
    p = T.plan_gpu(4096, 1, t)
    assert p.predicted_seconds == min(c[2] for c in p.candidates)
    assert p.solver == "ddrgf" and p.domains > 1
    assert T.plan_gpu(256, 64, t).solver == "rgf"


@pytest.mark.gpu
def test_gpu_calibration_predicts_measured_sweep(gpu):
    """bench_kernels timings feed the model; the predicted batched RGF time for a config-2
    proxy is within a factor 2 of the measured resident solve."""
    import time

    import torch

    from paper_2605_19910_b200 import dyson as D

    t = T.measure_kernels(128, batches=(1, 2, 4, 8, 16, 32), samples=3)
    assert all(x > 0 for x in t.t_gemm + t.t_inv)
    kr = T.kernel_ratios(t, 8)
    assert kr.r_lu > 1.0 and kr.t_gemm > 0
    cfg = D.scaled(D.CONFIGS[2], num_layers=40, n_energy=8, block_size=128)
    H = torch.empty((40, 3, 128, 128), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    G = torch.empty((8, 40, 3, 128, 128), dtype=torch.complex128, device="cuda")
    st = torch.cuda.Stream()
    for _ in range(2):  # eager call, then the CUDA-graph capture; time the replay
        D.solve_device(cfg, H, G, stream=st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D.solve_device(cfg, H, G, stream=st)
    torch.cuda.synchronize()
    measured = time.perf_counter() - t0
    pred = T.predict_rgf_gpu(40, 8, t).predicted_seconds
    assert 0.33 < pred / measured < 3.0, (pred, measured)  # one stream group modelled; several run
    plan = T.plan_gpu(40, 8, t)
    assert plan.solver in ("rgf", "ddrgf") and plan.predicted_seconds > 0

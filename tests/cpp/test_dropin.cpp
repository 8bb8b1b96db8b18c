// Drop-in parity program: the reference's own solvers (CPU, OpenBLAS) against
// bbsi::gpu:: (include/bbsi_gpu.hpp -> libbbsi_cuda.so) on the reference's own
// inputs (random_spd_like, testutil::random_hermitian) with the reference's
// tolerances. Mirrors acceptance criteria 1-3 (tests/acceptance.cpp:73-140) and
// the exception contract of tests/test_rgf.cpp:162-179 / test_ddrgf.cpp:218-250.
// Built by oracle/ref/Makefile (needs /root/reference); run by
// tests/test_gpu_dropin_cpp.py on a GPU box. Prints one PASS/FAIL line per case
// and exits with the number of failures.
#include <cstdio>
#include <string>
#include <vector>

#include "bbsi/cost_model.hpp"
#include "bbsi/ddrgf.hpp"
#include "bbsi/rgf.hpp"
#include "bbsi_gpu.hpp"
#include "helpers.hpp"

using namespace bbsi;
using cd = std::complex<double>;

static int g_fail = 0;

static void report(const char* name, bool ok, const std::string& detail) {
  std::printf("%s %-44s %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
  std::fflush(stdout);
  if (!ok) ++g_fail;
}

static std::string fmt(double x) {
  char b[32];
  std::snprintf(b, sizeof b, "%.3e", x);
  return b;
}

int main() {
  // ---- known answer, real input promoted (test_rgf.cpp:10-25)
  {
    BlockBandedMatrix<cd> m(make_layout(3, 1, 1));
    for (int i = 0; i < 3; ++i) {
      m.block(i, 0)(0, 0) = 2;
      if (i > 0) m.block(i, -1)(0, 0) = -1;
      if (i < 2) m.block(i, 1)(0, 0) = -1;
    }
    auto [g, c] = gpu::rgf_tridiag(m);
    bool ok = std::abs(g.block(0, 0)(0, 0) - 0.75) <= 1e-14 && std::abs(g.block(1, 0)(0, 0) - 1.0) <= 1e-14 &&
              std::abs(g.block(2, 0)(0, 0) - 0.75) <= 1e-14 && std::abs(g.block(0, 1)(0, 0) - 0.5) <= 1e-14 &&
              c == KernelCounters{8, 3, 7};
    report("known answer tridiag(-1,2,-1)", ok, "");
  }
  // ---- criterion 1: 200 instances, gpu vs dense oracle, plus gpu vs reference solver
  {
    const int bs_set[] = {1, 2, 4, 8};
    double worst = 0.0, worst_ref = 0.0;
    int instances = 0, counter_mismatch = 0;
    for (int i = 0; instances < 200; ++i) {
      const int w = 1 + i % 3;
      const int l = 1 + i % 12;
      if (l < w + 1) continue;
      const int bs = bs_set[i % 4];
      auto m = random_spd_like<cd>(make_layout(l, bs, w), uint64_t(1000 + i), 2.0);
      auto oracle = oracle_selected_inverse(m);
      auto [gn, cn] = gpu::rgf_ndiag(m);
      auto [rn, crn] = rgf_ndiag(m);
      worst = std::max(worst, testutil::max_block_error(gn, oracle));
      worst_ref = std::max(worst_ref, testutil::max_block_error(gn, rn));
      counter_mismatch += !(cn == crn);
      auto [gf, cf] = gpu::rgf_fused(m);
      worst = std::max(worst, testutil::max_block_error(gf, oracle));
      counter_mismatch += !(cf == rgf_fused(m).second);
      if (w == 1) {
        auto [gt, ct] = gpu::rgf_tridiag(m);
        worst = std::max(worst, testutil::max_block_error(gt, oracle));
        counter_mismatch += !(ct == rgf_tridiag(m).second);
      }
      ++instances;
    }
    report("C1 200 instances vs dense oracle (<=1e-10)", worst <= 1e-10 && counter_mismatch == 0,
           "max " + fmt(worst) + ", vs reference rgf " + fmt(worst_ref) + ", counter mismatches " +
               std::to_string(counter_mismatch));
  }
  // ---- criterion 2: ddrgf reproduces sequential RGF, thread-count independent
  {
    const std::vector<std::vector<int>> plans = {{1}, {2}, {3}, {4}, {2, 1}, {4, 2}, {3, 2}, {4, 2, 1}, {2, 2, 2}};
    const int bs_set[] = {2, 4, 8};
    double worst_vs_rgf = 0.0, worst_vs_threads = 0.0;
    int instances = 0, counter_mismatch = 0;
    for (int i = 0; instances < 60; ++i) {
      const int l = 6 + (i * 7) % 35;
      const auto& levels = plans[i % plans.size()];
      long long lk = l;
      bool feasible = true;
      for (int s2 : levels) {
        if (lk < 1 + s2) feasible = false;
        lk = (lk + s2) / (1 + s2);
      }
      if (!feasible) continue;
      auto m = random_spd_like<cd>(make_layout(l, bs_set[i % 3], 1), uint64_t(2000 + i), 2.0);
      auto ref = rgf_tridiag(m).first;
      DomainPlan plan;
      plan.s2_levels = levels;
      BlockBandedMatrix<cd> first;
      for (int nt : {1, 2, 4}) {
        plan.n_threads = nt;
        auto [g, c] = gpu::ddrgf(m, plan);
        if (nt == 1) {
          first = g;
          worst_vs_rgf = std::max(worst_vs_rgf, testutil::max_block_error(g, ref));
          counter_mismatch += !(c == ddrgf(m, plan).second);
        } else {
          worst_vs_threads = std::max(worst_vs_threads, testutil::max_block_error(g, first));
        }
      }
      ++instances;
    }
    report("C2 60 ddrgf instances vs rgf (<=1e-10)",
           worst_vs_rgf <= 1e-10 && worst_vs_threads <= 1e-12 && counter_mismatch == 0,
           "max " + fmt(worst_vs_rgf) + ", thread variance " + fmt(worst_vs_threads) + ", counter mismatches " +
               std::to_string(counter_mismatch));
  }
  // ---- criterion 3: counters equal the closed forms
  {
    long long mismatches = 0;
    for (int w = 1; w <= 3; ++w)
      for (int l = w + 1; l <= 12; ++l) {
        auto m = random_spd_like<cd>(make_layout(l, 2, w), uint64_t(3000 + 16 * l + w), 2.0);
        if (gpu::rgf_ndiag(m).second != predict_nrgf_counters(l, w)) ++mismatches;
        if (w == 1 && gpu::rgf_tridiag(m).second != predict_rgf_counters(l)) ++mismatches;
      }
    report("C3 counter closed forms", mismatches == 0, std::to_string(mismatches) + " mismatches");
  }
  // ---- rgf_extended halos vs the reference rgf_extended
  {
    double worst = 0.0;
    bool counters_ok = true;
    for (int l : {1, 2, 3, 5, 6, 9}) {
      auto m = random_spd_like<cd>(make_layout(l, 3, l == 1 ? 0 : 1), uint64_t(200 + l), 2.0);
      auto [ge, gc] = gpu::rgf_extended(m);
      auto [re, rc] = rgf_extended(m);
      counters_ok = counters_ok && gc == rc;
      for (int k = 0; k < l; ++k) {
        worst = std::max(worst, rel_frobenius_error(ge.first_row[k], re.first_row[k]));
        worst = std::max(worst, rel_frobenius_error(ge.last_row[k], re.last_row[k]));
        worst = std::max(worst, rel_frobenius_error(ge.first_col[k], re.first_col[k]));
        worst = std::max(worst, rel_frobenius_error(ge.last_col[k], re.last_col[k]));
      }
      worst = std::max(worst, testutil::max_block_error(ge.core, re.core));
    }
    report("rgf_extended halos vs reference (<=1e-10)", worst <= 1e-10 && counters_ok, "max " + fmt(worst));
  }
  // ---- Hermitian input -> Hermitian selected inverse (test_rgf.cpp:150-160)
  {
    auto h1 = testutil::random_hermitian(make_layout(8, 3, 1), 31, 1.0);
    auto h2 = testutil::random_hermitian(make_layout(8, 3, 2), 32, 1.0);
    const double d1 = testutil::hermitian_defect(gpu::rgf_tridiag(h1).first);
    const double d2 = testutil::hermitian_defect(gpu::rgf_ndiag(h2).first);
    report("Hermitian defect (<=1e-12)", d1 <= 1e-12 && d2 <= 1e-12, fmt(d1) + " " + fmt(d2));
  }
  // ---- exception contract
  {
    bool ok = false;
    auto m = random_spd_like<cd>(make_layout(5, 2, 1), 40, 2.0);
    m.block(4, 0) = DenseMatrix<cd>(2, 2);
    try {
      gpu::rgf_tridiag(m);
    } catch (const singular_matrix_error& e) {
      ok = e.layer() == 4;
    }
    report("singular pivot -> layer 4 (test_rgf.cpp:162)", ok, "");
    ok = false;
    auto m2 = random_spd_like<cd>(make_layout(10, 2, 1), 908, 2.0);
    m2.block(7, 0) = DenseMatrix<cd>(2, 2);
    m2.block(7, 1) = DenseMatrix<cd>(2, 2);
    m2.block(7, -1) = DenseMatrix<cd>(2, 2);
    DomainPlan plan;
    plan.s2_levels = {4};
    plan.n_threads = 2;
    try {
      gpu::ddrgf(m2, plan);
    } catch (const singular_matrix_error& e) {
      ok = e.layer() == 7;
    }
    report("ddrgf singular -> global layer 7", ok, "");
    int thrown = 0;
    auto wide = random_spd_like<cd>(make_layout(6, 2, 2), 41, 2.0);
    try {
      gpu::rgf_tridiag(wide);
    } catch (const invalid_argument_error&) {
      ++thrown;
    }
    try {
      gpu::rgf_extended(wide);
    } catch (const invalid_argument_error&) {
      ++thrown;
    }
    BlockLayout ragged(4, {2, 3, 2, 3}, 2);
    try {
      gpu::rgf_fused(random_spd_like<cd>(ragged, 42, 2.0));
    } catch (const invalid_argument_error&) {
      ++thrown;
    }
    DomainPlan bad;
    bad.s2_levels = {4, 4};
    try {
      gpu::ddrgf(random_spd_like<cd>(make_layout(6, 2, 1), 905, 2.0), bad);
    } catch (const invalid_argument_error&) {
      ++thrown;
    }
    report("invalid_argument_error contract", thrown == 4, std::to_string(thrown) + "/4 thrown");
  }
  // ---- ragged block sizes (test_rgf.cpp:42-48)
  {
    BlockLayout layout(5, {3, 1, 4, 2, 3}, 1);
    auto m = random_spd_like<cd>(layout, 8, 2.0);
    const double e = testutil::max_block_error(gpu::rgf_tridiag(m).first, oracle_selected_inverse(m));
    report("ragged layout {3,1,4,2,3}", e <= 1e-10, fmt(e));
  }
  std::printf("%d failure(s)\n", g_fail);
  // ---- many matrices in one pass (bbsi::gpu::rgf_many) vs the reference solver on each
  {
    std::vector<BlockBandedMatrix<cd>> ms;
    for (int k = 0; k < 5; ++k) ms.push_back(random_spd_like<cd>(make_layout(12, 7, 1), 1200 + k, 2.0));
    auto got = gpu::rgf_many(ms);
    double worst = 0.0;
    bool counters_ok = true;
    for (size_t k = 0; k < ms.size(); ++k) {
      auto [ref, rc] = rgf_tridiag(ms[k]);
      worst = std::max(worst, testutil::max_block_error(got[k].first, ref));
      counters_ok = counters_ok && got[k].second == rc;
    }
    report("rgf_many (5 x rgf_tridiag, l=12 b=7)", worst <= 1e-10 && counters_ok, fmt(worst));
    std::vector<BlockBandedMatrix<cd>> bad = ms;
    bad[3].block(6, 0) = DenseMatrix<cd>(7, 7);
    bad[3].block(6, 1) = DenseMatrix<cd>(7, 7);
    bad[3].block(6, -1) = DenseMatrix<cd>(7, 7);
    int layer = -2;
    try {
      gpu::rgf_many(bad);
    } catch (const singular_matrix_error& e) {
      layer = e.layer();
    }
    int ref_layer = -3;
    try {
      rgf_tridiag(bad[3]);
    } catch (const singular_matrix_error& e) {
      ref_layer = e.layer();
    }
    report("rgf_many singular layer = reference's", layer == ref_layer && layer >= 0, std::to_string(layer));
  }
  return g_fail;
}

// bbsi_gpu.hpp -- C++ drop-in for the reference bbsi solver entry points, backed
// by the B200 library through the C ABI in bbsi_cuda.h.
//
// Include AFTER the reference headers (it uses their types unchanged):
//   #include "bbsi/ddrgf.hpp"      // reference: BlockBandedMatrix, KernelCounters, DomainPlan, errors
//   #include "bbsi_gpu.hpp"        // this file: bbsi::gpu::rgf_tridiag / rgf_ndiag / ... on the GPU
// and link libbbsi_cuda.so. Every function keeps the reference signature and
// semantics (return by value, KernelCounters = the reference's logical counts,
// invalid_argument_error / singular_matrix_error(layer)) for T = std::complex<double>.
// singular_matrix_error is raised on the reference's conditions for the RGF solvers
// (the same pivots, the same layer). ddrgf differs by construction: the stabilised
// formulation never inverts an isolated domain, so it reports a
// singular pivot only where a domain WITH its boundary self-energies (or a separator)
// is singular; the layer is the global layer of that pivot.
//   rgf_tridiag  rgf.hpp:37-76      rgf_ndiag     rgf.hpp:82-137
//   rgf_fused    rgf.hpp:143-192    rgf_extended  rgf.hpp:209-270
//   ddrgf        ddrgf.hpp:420-428
// A project switches by calling bbsi::gpu::X where it called bbsi::X (or by a
// `namespace solver = bbsi::gpu;` alias).
#pragma once

#include <complex>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bbsi_cuda.h"

namespace bbsi {
namespace gpu {

using cd = std::complex<double>;

namespace detail {

struct Slots {
  int l = 0, w = 0, bs = 0;
  std::vector<int> sizes;
  std::vector<cd> data;  // [l][2w+1][bs][bs], column-major blocks (block_banded.hpp:58-60 order)
  cd* slot(int a, int off) { return data.data() + (size_t(a) * (2 * w + 1) + off + w) * size_t(bs) * bs; }
};

inline Slots to_slots(const BlockBandedMatrix<cd>& m) {
  Slots s;
  const auto& lay = m.layout();
  s.l = lay.num_layers;
  s.w = lay.bandwidth;
  s.sizes = lay.block_sizes;
  for (int b : s.sizes) s.bs = std::max(s.bs, b);
  s.data.assign(size_t(s.l) * (2 * s.w + 1) * s.bs * s.bs, cd{});
  for (int a = 0; a < s.l; ++a)
    for (int off = -s.w; off <= s.w; ++off) {
      if (!m.in_band(a, off)) continue;
      const auto& blk = m.block(a, off);
      cd* d = s.slot(a, off);
      for (int j = 0; j < blk.cols(); ++j)
        std::memcpy(d + size_t(j) * s.bs, blk.data() + size_t(j) * blk.rows(), sizeof(cd) * blk.rows());
    }
  return s;
}

inline BlockBandedMatrix<cd> from_slots(const BlockLayout& lay, Slots& s) {
  BlockBandedMatrix<cd> g(lay);
  for (int a = 0; a < s.l; ++a)
    for (int off = -s.w; off <= s.w; ++off) {
      if (!g.in_band(a, off)) continue;
      auto& blk = g.block(a, off);
      const cd* src = s.slot(a, off);
      for (int j = 0; j < blk.cols(); ++j)
        std::memcpy(blk.data() + size_t(j) * blk.rows(), src + size_t(j) * s.bs, sizeof(cd) * blk.rows());
    }
  return g;
}

// (evaluate the C call before reading fail_layer: argument order is unspecified)
inline void check(int rc, int fail_layer) {
  if (rc == BBSI_OK) return;
  const std::string msg = bbsi_cuda_last_error();
  if (rc == BBSI_INVALID_ARGUMENT) throw invalid_argument_error(msg);
  if (rc == BBSI_SINGULAR) throw singular_matrix_error(msg, fail_layer);
  throw std::runtime_error("bbsi_cuda: " + msg);
}

inline KernelCounters counters(const long long c[3]) {
  KernelCounters k;
  k.n_gemm = c[0];
  k.n_lu = c[1];
  k.n_getrs = c[2];
  return k;
}

inline std::vector<DenseMatrix<cd>> halo(const std::vector<cd>& mem, int l, int bs, const std::vector<int>& rows,
                                         const std::vector<int>& cols) {
  std::vector<DenseMatrix<cd>> out(l);
  for (int k = 0; k < l; ++k) {
    out[k] = DenseMatrix<cd>(rows[k], cols[k]);
    for (int j = 0; j < cols[k]; ++j)
      std::memcpy(out[k].data() + size_t(j) * rows[k], mem.data() + (size_t(k) * bs + j) * bs, sizeof(cd) * rows[k]);
  }
  return out;
}

}  // namespace detail

inline std::pair<BlockBandedMatrix<cd>, KernelCounters> rgf_tridiag(const BlockBandedMatrix<cd>& m,
                                                                    StructuralTrace* trace = nullptr) {
  auto s = detail::to_slots(m);
  std::vector<cd> g(s.data.size());
  long long c[3];
  int fl = -1;
  const int rc = bbsi_cuda_rgf_tridiag_z(s.l, s.w, s.bs, s.sizes.data(), reinterpret_cast<const double*>(s.data.data()),
                                        reinterpret_cast<double*>(g.data()), c, &fl);
  detail::check(rc, fl);
  if (trace) trace->max_update_offset = 0;
  s.data.swap(g);
  return {detail::from_slots(m.layout(), s), detail::counters(c)};
}

inline std::pair<BlockBandedMatrix<cd>, KernelCounters> rgf_ndiag(const BlockBandedMatrix<cd>& m,
                                                                  StructuralTrace* trace = nullptr) {
  auto s = detail::to_slots(m);
  std::vector<cd> g(s.data.size());
  long long c[3];
  int fl = -1, mo = trace ? trace->max_update_offset : 0;
  const int rc = bbsi_cuda_rgf_ndiag_z(s.l, s.w, s.bs, s.sizes.data(), reinterpret_cast<const double*>(s.data.data()),
                                      reinterpret_cast<double*>(g.data()), c, &mo, &fl);
  detail::check(rc, fl);
  if (trace) trace->max_update_offset = mo;
  s.data.swap(g);
  return {detail::from_slots(m.layout(), s), detail::counters(c)};
}

inline std::pair<BlockBandedMatrix<cd>, KernelCounters> rgf_fused(const BlockBandedMatrix<cd>& m) {
  auto s = detail::to_slots(m);
  std::vector<cd> g(s.data.size());
  long long c[3];
  int fl = -1;
  const int rc = bbsi_cuda_rgf_fused_z(s.l, s.w, s.bs, s.sizes.data(), reinterpret_cast<const double*>(s.data.data()),
                                      reinterpret_cast<double*>(g.data()), c, &fl);
  detail::check(rc, fl);
  s.data.swap(g);
  return {detail::from_slots(m.layout(), s), detail::counters(c)};
}

inline std::pair<ExtendedInverse<cd>, KernelCounters> rgf_extended(const BlockBandedMatrix<cd>& m) {
  auto s = detail::to_slots(m);
  std::vector<cd> g(s.data.size());
  const size_t hn = size_t(s.l) * s.bs * s.bs;
  std::vector<cd> fr(hn), lr(hn), fc(hn), lc(hn);
  long long c[3];
  int fl = -1;
  const int rc = bbsi_cuda_rgf_extended_z(s.l, s.w, s.bs, s.sizes.data(), reinterpret_cast<const double*>(s.data.data()),
                               reinterpret_cast<double*>(g.data()), reinterpret_cast<double*>(fr.data()),
                               reinterpret_cast<double*>(lr.data()), reinterpret_cast<double*>(fc.data()),
                               reinterpret_cast<double*>(lc.data()), c, &fl);
  detail::check(rc, fl);
  s.data.swap(g);
  ExtendedInverse<cd> ext;
  ext.core = detail::from_slots(m.layout(), s);
  const int l = s.l;
  std::vector<int> first(l, s.sizes.front()), last(l, s.sizes.back());
  ext.first_row = detail::halo(fr, l, s.bs, first, s.sizes);
  ext.last_row = detail::halo(lr, l, s.bs, last, s.sizes);
  ext.first_col = detail::halo(fc, l, s.bs, s.sizes, first);
  ext.last_col = detail::halo(lc, l, s.bs, s.sizes, last);
  return {std::move(ext), detail::counters(c)};
}

// ngpu > 1 shards the domains over GPUs 0..ngpu-1 of this process (NCCL all-gather of
// the interface packets inside the library); ngpu = 0 reads BBSI_GPUS (default 1).
inline std::pair<BlockBandedMatrix<cd>, KernelCounters> ddrgf(const BlockBandedMatrix<cd>& m, const DomainPlan& plan,
                                                               int ngpu = 0) {
  if (ngpu <= 0) {
    const char* e = std::getenv("BBSI_GPUS");
    ngpu = e ? std::atoi(e) : 1;
    if (ngpu < 1) ngpu = 1;
  }
  auto s = detail::to_slots(m);
  std::vector<cd> g(s.data.size());
  long long c[3];
  int fl = -1;
  const int rc =
      ngpu > 1 ? bbsi_cuda_ddrgf_multi_z(s.l, s.w, s.bs, s.sizes.data(), reinterpret_cast<const double*>(s.data.data()),
                                         plan.s2_levels.data(), plan.n_levels(), plan.n_threads,
                                         plan.terminal_threads, ngpu, nullptr, reinterpret_cast<double*>(g.data()), c,
                                         &fl)
               : bbsi_cuda_ddrgf_z(s.l, s.w, s.bs, s.sizes.data(), reinterpret_cast<const double*>(s.data.data()),
                                   plan.s2_levels.data(), plan.n_levels(), plan.n_threads, plan.terminal_threads,
                                   reinterpret_cast<double*>(g.data()), c, &fl);
  detail::check(rc, fl);
  s.data.swap(g);
  return {detail::from_slots(m.layout(), s), detail::counters(c)};
}

// Many matrices of one layout in one device pass (an energy loop over host-built A(E)):
// the results of rgf_tridiag / rgf_ndiag for each, in order; throws for the first matrix
// with a negligible pivot, as calling the single solver on each in turn would.
inline std::vector<std::pair<BlockBandedMatrix<cd>, KernelCounters>> rgf_many(
    const std::vector<BlockBandedMatrix<cd>>& ms) {
  std::vector<std::pair<BlockBandedMatrix<cd>, KernelCounters>> out;
  if (ms.empty()) return out;
  std::vector<detail::Slots> in;
  for (const auto& m : ms) in.push_back(detail::to_slots(m));
  const auto& s0 = in[0];
  const size_t n = s0.data.size();
  std::vector<cd> a(n * ms.size()), g(n * ms.size());
  for (size_t k = 0; k < ms.size(); ++k) std::memcpy(a.data() + k * n, in[k].data.data(), n * sizeof(cd));
  long long c[3];
  std::vector<int> fails(ms.size(), -1);
  const int rc = bbsi_cuda_rgf_many_z(s0.l, s0.w, s0.bs, s0.sizes.data(), int(ms.size()),
                                      reinterpret_cast<const double*>(a.data()), reinterpret_cast<double*>(g.data()), c,
                                      fails.data());
  int fl = -1;
  for (int f : fails)
    if (f >= 0) {
      fl = f;
      break;
    }
  detail::check(rc, fl);
  for (size_t k = 0; k < ms.size(); ++k) {
    auto s = in[k];
    std::memcpy(s.data.data(), g.data() + k * n, n * sizeof(cd));
    out.push_back({detail::from_slots(ms[k].layout(), s), detail::counters(c)});
  }
  return out;
}

}  // namespace gpu
}  // namespace bbsi

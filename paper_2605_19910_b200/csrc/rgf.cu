// Batched RGF sweeps (block tridiagonal and block n-diagonal) on the device.
//
// Restates rgf_ndiag (rgf.hpp:82-137) -- and through w = 1 rgf_tridiag
// (rgf.hpp:37-76) -- for a batch of independent matrices (energies, domains):
//
//   upward  j = l-1 .. 1, k = min(w, j):
//     X_j          = inv(M'[j,j])                        (zinv: zgetrf + zgetrs(I))
//     lm[j][t]     = X_j M'[j, j-t]          t = 1..k    (one GEMM, b x kb)
//     um[j][t]     = M'[j-t, j] X_j                      (one GEMM, kb x b)
//     M'[j-s, j-t] -= M'[j-s, j] lm[j][t]    s,t = 1..k  (one GEMM, kb x kb window)
//   X_0 = inv(M'[0,0]) = G[0,0]
//   downward j = 1 .. l-1:
//     G[j, j-t]    = -sum_s lm[j][s] G[j-s, j-t]         (one GEMM, b x kb)
//     G[j-t, j]    = -sum_s G[j-t, j-s] um[j][s]         (one GEMM, kb x b)
//     G[j, j]      = X_j - sum_s lm[j][s] G[j-s, j]      (one GEMM, b x b, K = kb)
//
// The working copy M' lives in the output band G itself (its slots are only
// overwritten by G^R after the upward sweep has consumed them), and the
// explicit inverse X_j is written into G[j,j], which the downward pass updates
// in place. Every operand is a strided set of slots of the band storage
// slot(a, off) = a*(2w+1) + off + w (block_banded.hpp:58-60).
#include <cstdlib>
#include <mutex>

#include "internal.h"

namespace bbsi_gpu {

int dyson_groups(int batch) {
  if (const char* e = getenv("BBSI_GROUPS")) {
    int g = atoi(e);
    if (g >= 1) return g < batch ? g : batch;
  }
  // Energy batches: up to 16 independent stream groups. The chains of a group are
  // latency-bound (inversion panels), so more concurrent groups help small batches:
  // B200, config 2 at 64 / 32 / 16 / 8 energies (the per-GPU share at 1 / 2 / 4 / 8 GPUs),
  // 2 groups: 572 / 311 / 186 / 128 ms; min(16, batch): 573 / 289 / 162 / 116 ms.
  return batch < 16 ? batch : 16;
}

int default_groups(int batch, int bs) {
  if (const char* e = getenv("BBSI_GROUPS")) {
    int g = atoi(e);
    if (g >= 1) return g < batch ? g : batch;
  }
  (void)bs;
  // Two side-stream groups: one group's latency-bound panels overlap the other's
  // GEMMs (B200, config 2, 64 energies: 739 ms vs 771 ms with one group).
  return batch >= 8 ? 2 : 1;
}

bool two_ended_default() {
  static const bool on = [] {
    const char* e = getenv("BBSI_TWO_ENDED");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

namespace {
// Banded (w >= 2) two-ended sweeps (BBSI_TWO_ENDED_BANDED=0: one-ended). With one
// refinement step of every multiplier and of the dense middle inverse they are the
// faster and the more accurate order on config 3 (B200: 278 vs 353 ms per step; 25 of 32
// energies <= 1e-10 against the compiled reference vs 15, residual at the reference's
// level; profiles/r02_parity.md). Round 1 kept them opt-in: without the refinement their
// worst error was 2.3x the reference's floor at E = 0.145.
bool two_ended_banded() {
  static const bool on = [] {
    const char* e = getenv("BBSI_TWO_ENDED_BANDED");
    return !(e && atoi(e) == 0);
  }();
  return on;
}
bool two_ended_ok(bool two_ended, int l, int w) {
  return two_ended && ((w == 1 && l >= 3) || (w >= 2 && two_ended_banded() && l >= 3 * w + 2));
}
bool use_two_ended(const SweepWork& W) { return two_ended_ok(W.two_ended, W.l, W.w) && (W.w == 1 || !W.Hoff); }
}  // namespace

namespace {
size_t mid_dense_bytes(int w, int b, int batch) {
  return (size_t(w) * b * w * b * batch * sizeof(double2) + 255) & ~size_t(255);
}
size_t mid_bytes(int w, int b, int batch) { return mid_dense_bytes(w, b, batch) + zinv_scratch_bytes(w * b, batch) + 256; }
bool mid_dense_enabled() {
  static const bool on = [] {
    const char* e = getenv("BBSI_MID_DENSE");
    return !(e && atoi(e) == 0);
  }();
  return on;
}
}  // namespace

bool sweep_is_two_ended(const SweepWork& W) { return use_two_ended(W); }

bool refine_multipliers_default() {
  static const bool on = [] {
    const char* e = getenv("BBSI_REFINE");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

namespace {
bool refine_ok(int l, int w, bool two_ended) {
  (void)l;
  (void)two_ended;
  return w >= 2 && refine_multipliers_default();
}
// pivot copies of one stream group (complex elements): one-ended f_j [batch]; two-ended
// f_jR, f_jL [2][batch] plus the dense middle window [batch][(w b)^2]
long long fcopy_elems(int l, int w, int bs, int batch_g, bool two_ended) {
  const long long bb = (long long)bs * bs;
  if (two_ended_ok(two_ended, l, w) && w >= 2) return 2LL * batch_g * bb + (long long)batch_g * w * w * bb;
  return (long long)batch_g * bb;
}
}  // namespace



size_t sweep_scratch_bytes(int l, int w, int bs, int batch, int groups, bool two_ended) {
  const size_t bb = size_t(bs) * bs * sizeof(double2);
  const int chains = two_ended_ok(two_ended, l, w) ? 2 : 1;
  size_t s = 2 * size_t(batch) * l * w * bb;              // LM, UM
  s += size_t(groups) * (zinv_scratch_bytes(bs, chains * ((batch + groups - 1) / groups)) + 256);  // inversion scratch
  s += size_t(l) * batch * sizeof(int) + 256;             // status
  if (chains == 2 && w >= 2) s += size_t(groups) * mid_bytes(w, bs, (batch + groups - 1) / groups);  // dense middle
  if (refine_ok(l, w, two_ended))  // pivot copies for the refinement, per group
    s += size_t(groups) * size_t(fcopy_elems(l, w, bs, (batch + groups - 1) / groups, two_ended)) * sizeof(double2) +
         256;
  return s;
}

void sweep_carve(SweepWork& W, void* base) {
  char* p = static_cast<char*>(base);
  const size_t bb = size_t(W.bs) * W.bs;
  W.LM = reinterpret_cast<double2*>(p);
  p += size_t(W.batch) * W.l * W.w * bb * sizeof(double2);
  W.UM = reinterpret_cast<double2*>(p);
  p += size_t(W.batch) * W.l * W.w * bb * sizeof(double2);
  W.inv = p;
  const int gs = (W.batch + W.groups - 1) / W.groups;
  p += size_t(W.groups) * (zinv_scratch_bytes(W.bs, (use_two_ended(W) ? 2 : 1) * gs) + 256);
  W.status = reinterpret_cast<int*>(p);
  p += size_t(W.l) * W.batch * sizeof(int);
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));  // (+256 slack sized)
  W.mid = (use_two_ended(W) && W.w >= 2) ? p : nullptr;
  if (W.mid) p += size_t(W.groups) * mid_bytes(W.w, W.bs, gs);
  W.fcopy = (!W.Hoff && refine_ok(W.l, W.w, W.two_ended)) ? reinterpret_cast<double2*>(p) : nullptr;
}

namespace {

struct Ctx {
  const SweepWork& W;
  long long bb, nslot;
  Ctx(const SweepWork& w) : W(w), bb((long long)w.bs * w.bs), nslot(2 * w.w + 1) {}
  double2* slot(int a, int off) const { return W.G + ((long long)a * nslot + off + W.w) * bb; }
  double2* lm(int j) const { return W.LM + (long long)j * W.w * bb; }
  double2* um(int j) const { return W.UM + (long long)j * W.w * bb; }
  long long lm_bstride() const { return (long long)(W.lm_layers > 0 ? W.lm_layers : W.l) * W.w * bb; }
  ZOp gop(const double2* p, long long rs_slots, long long cs_slots) const {
    return ZOp{p, W.bs, rs_slots * bb, cs_slots * bb, W.g_bstride};
  }
  // block (a, off) of the shared H band (bstride 0: every batch entry reads the same block)
  ZOp hop(int a, int off) const { return ZOp{W.Hoff + ((long long)a * nslot + off + W.w) * bb, W.bs, 0, 0, 0}; }
  ZOp mop(const double2* p, long long rs_blocks, long long cs_blocks) const {
    return ZOp{p, W.bs, rs_blocks * bb, cs_blocks * bb, lm_bstride()};
  }
};

ZGemmProblem prob(int M, int N, int K, double alpha, double beta, ZOp A, ZOp B, ZOp C) {
  ZGemmProblem p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.alpha = make_double2(alpha, 0.0);
  p.beta = make_double2(beta, 0.0);
  p.A = A;
  p.B = B;
  p.C = C;
  p.D = C;
  return p;
}

cudaError_t launch(const SweepWork& W, std::initializer_list<ZGemmProblem> ps, cudaStream_t s) {
  ZGemmGroup g{};
  g.batch = W.batch;
  g.bs = W.bs;
  for (const auto& p : ps) g.prob[g.nprob++] = p;
  return zgemm_grouped(g, s);
}

}  // namespace

namespace {

cudaError_t rgf_sweeps_one(const SweepWork& W, const int* n_true, int* status, int status_stride, cudaStream_t s) {
  Ctx c(W);
  const int l = W.l, w = W.w, b = W.bs;
  const long long two_w = 2LL * w;
  cudaError_t e;
  auto inv = [&](int j) {
    return zinv_batched(c.slot(j, 0), b, W.g_bstride, b, n_true[j], W.batch, W.inv,
                        status + (long long)j * status_stride, s);
  };

  // ---------------- upward sweep (rgf.hpp:98-114)
  for (int j = l - 1; j >= 1; --j) {
    const int k = j < w ? j : w;
    if (W.fcopy && !(W.Hoff && w == 1) &&
        (e = cudaMemcpy2DAsync(W.fcopy, c.bb * sizeof(double2), c.slot(j, 0), W.g_bstride * sizeof(double2),
                               c.bb * sizeof(double2), W.batch, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return e;
    if ((e = inv(j)) != cudaSuccess) return e;
    const ZOp X = c.gop(c.slot(j, 0), 0, 0);
    // lm[j] = X_j [M'(j,j-1) .. M'(j,j-k)]
    // (tridiagonal Dyson batch: M'(j,j-1) = -H(j,j-1) is never modified, read from H)
    const bool hs = W.Hoff && w == 1;
    const double sg = hs ? -1.0 : 1.0;
    ZGemmProblem p_lm = prob(b, k * b, b, sg, 0.0, X, hs ? c.hop(j, -1) : c.gop(c.slot(j, -1), 0, -1),
                             c.mop(c.lm(j), 0, 1));
    if ((e = launch(W, {p_lm}, s)) != cudaSuccess) return e;
    const bool refine = W.fcopy && !hs;
    const ZOp F{W.fcopy, b, 0, 0, c.bb};
    if (refine) {  // R = M'(j, j-t) - f_j lm (in place: the row is not read again); lm += X R
      const ZOp row = c.gop(c.slot(j, -1), 0, -1);
      if ((e = launch(W, {prob(b, k * b, b, -1.0, 1.0, F, c.mop(c.lm(j), 0, 1), row)}, s)) != cudaSuccess) return e;
      if ((e = launch(W, {prob(b, k * b, b, 1.0, 1.0, X, row, c.mop(c.lm(j), 0, 1))}, s)) != cudaSuccess) return e;
    }
    // window M'(j-s, j-t) -= M'(j-s, j) lm[j][t];  um[j] = [M'(j-t, j)]_t X_j
    ZOp upper = hs ? c.hop(j - 1, +1) : c.gop(c.slot(j - 1, +1), -two_w, 0);
    ZGemmProblem p_win = prob(k * b, k * b, b, -sg, 1.0, upper, c.mop(c.lm(j), 0, 1), c.gop(c.slot(j - 1, 0), -two_w, -1));
    if (hs && W.zdev) {  // A[j-1, j-1] = z I - H - sigma I read from H (first and only update)
      p_win.C = c.hop(j - 1, 0);
      p_win.cz = W.zdev;
      p_win.csig = W.sigdev + (j - 1);
    }
    ZGemmProblem p_um = prob(k * b, b, b, sg, 0.0, upper, X, c.mop(c.um(j), 1, 0));
    if ((e = launch(W, {p_win, p_um}, s)) != cudaSuccess) return e;
    if (refine) {  // R = M'(j-t, j) - um f_j (in place: the column is not read again); um += R X
      if ((e = launch(W, {prob(k * b, b, b, -1.0, 1.0, c.mop(c.um(j), 1, 0), F, upper)}, s)) != cudaSuccess) return e;
      if ((e = launch(W, {prob(k * b, b, b, 1.0, 1.0, upper, X, c.mop(c.um(j), 1, 0))}, s)) != cudaSuccess) return e;
    }
  }
  if ((e = inv(0)) != cudaSuccess) return e;

  // ---------------- downward sweep (rgf.hpp:117-135)
  // Step j writes rows j (slots -t, 0) and j-t (slot +t), t <= w: after it, rows
  // [0, j-w] are final.
  int flushed = 0;
  auto flush = [&](int upto) -> cudaError_t {
    if (!W.rows_done || upto <= flushed) return cudaSuccess;
    const cudaError_t r = W.rows_done(flushed, upto, W.e_off, W.batch, s);
    flushed = upto;
    return r;
  };
  if (l == 1 && (e = flush(1)) != cudaSuccess) return e;
  for (int j = 1; j < l; ++j) {
    const int k = j < w ? j : w;
    ZOp lmrow = c.mop(c.lm(j), 0, 1);
    ZOp window = c.gop(c.slot(j - 1, 0), -two_w, -1);
    ZGemmProblem p_row = prob(b, k * b, k * b, -1.0, 0.0, lmrow, window, c.gop(c.slot(j, -1), 0, -1));
    ZGemmProblem p_col = prob(k * b, b, k * b, -1.0, 0.0, window, c.mop(c.um(j), 1, 0), c.gop(c.slot(j - 1, +1), -two_w, 0));
    if ((e = launch(W, {p_row, p_col}, s)) != cudaSuccess) return e;
    ZGemmProblem p_diag = prob(b, b, k * b, -1.0, 1.0, lmrow, c.gop(c.slot(j - 1, +1), -two_w, 0), c.gop(c.slot(j, 0), 0, 0));
    if ((e = launch(W, {p_diag}, s)) != cudaSuccess) return e;
    const int complete = j - w + 1;
    if (W.rows_done && complete - flushed >= W.hook_rows && (e = flush(complete)) != cudaSuccess) return e;
  }
  if ((e = flush(l)) != cudaSuccess) return e;
  return cudaSuccess;
}

// Two-ended block-tridiagonal sweep (w = 1). The right-connected chain of
// rgf_tridiag (rgf.hpp:58-64) runs from layer l-1 down to m+1 while its mirror, the
// left-connected chain, runs from layer 0 up to m-1, in lockstep: every inversion
// launch covers both chains (2 x batch matrices) and every GEMM launch both chains'
// products. Layer m receives both Schur corrections and its inverse is G[m,m]; the
// two outward sweeps (rgf.hpp:66-74 and its mirror) then run in lockstep as well.
//   right, j = l-1 .. m+1:  X_j = inv(M'[j,j]),  lm[j] = X_j A[j,j-1],  um[j] = A[j-1,j] X_j,
//                           M'[j-1,j-1] -= A[j-1,j] lm[j]
//   left,  j = 0 .. m-1:    Y_j = inv(M'[j,j]),  lm[j] = Y_j A[j,j+1],  um[j] = A[j+1,j] Y_j,
//                           M'[j+1,j+1] -= A[j+1,j] lm[j]
//   G[m,m] = inv(M'[m,m])
//   right, j = m+1 .. l-1:  G[j,j-1] = -lm[j] G[j-1,j-1],  G[j-1,j] = -G[j-1,j-1] um[j],
//                           G[j,j] = X_j - lm[j] G[j-1,j]
//   left,  j = m-1 .. 0:    G[j,j+1] = -lm[j] G[j+1,j+1],  G[j+1,j] = -G[j+1,j+1] um[j],
//                           G[j,j] = Y_j - lm[j] G[j+1,j]
// Same products and inverses per layer as the one-ended sweep. status[j] records the
// pivot of layer j in this elimination order.
cudaError_t rgf_sweeps_two(const SweepWork& W, const int* n_true, int* status, int status_stride, cudaStream_t s) {
  Ctx c(W);
  const int l = W.l, b = W.bs;
  const int m = l / 2, nR = l - 1 - m, nL = m;
  const bool hs = W.Hoff != nullptr;
  const double sg = hs ? -1.0 : 1.0;  // A's off-diagonal blocks are -H when read from H
  cudaError_t e;
  auto blk = [&](const double2* p) { return c.gop(p, 0, 0); };
  auto offd = [&](int a, int off) { return hs ? c.hop(a, off) : blk(c.slot(a, off)); };
  auto lmo = [&](int j) { return c.mop(c.lm(j), 0, 0); };
  auto umo = [&](int j) { return c.mop(c.um(j), 0, 0); };
  auto grp = [&](const ZGemmProblem* ps, int np) {
    ZGemmGroup g{};
    g.batch = W.batch;
    g.bs = b;
    for (int i = 0; i < np; ++i) g.prob[g.nprob++] = ps[i];
    return zgemm_grouped(g, s);
  };
  // inversion of layer jR (and jL when >= 0) for the whole batch in one launch
  auto inv2 = [&](int jR, int jL) {
    double2* mR = c.slot(jR, 0);
    if (jL < 0 || n_true[jL] != n_true[jR]) {  // (ragged layers: one launch per chain)
      cudaError_t r = zinv_batched2(mR, b, W.g_bstride, b, n_true[jR], W.batch, 1, 0, W.inv,
                                    status + (long long)jR * status_stride, 0, s);
      if (r != cudaSuccess || jL < 0) return r;
      return zinv_batched2(c.slot(jL, 0), b, W.g_bstride, b, n_true[jL], W.batch, 1, 0, W.inv,
                           status + (long long)jL * status_stride, 0, s);
    }
    return zinv_batched2(mR, b, W.g_bstride, b, n_true[jR], W.batch, 2, (long long)(c.slot(jL, 0) - mR), W.inv,
                         status + (long long)jR * status_stride, (long long)(jL - jR) * status_stride, s);
  };

  // ---------------- two inward chains
  // diagonal blocks still to be formed from H by their first Schur update (W.zdev):
  // all but the two chain starts
  std::vector<char> formed(l, W.zdev ? 0 : 1);
  formed[0] = formed[l - 1] = 1;
  auto win = [&](int a, const ZOp& A_, const ZOp& B_) {  // M'[a, a] -= A_ B_ (into G)
    ZGemmProblem p = prob(b, b, b, -sg, 1.0, A_, B_, blk(c.slot(a, 0)));
    if (!formed[a]) {
      p.C = c.hop(a, 0);
      p.cz = W.zdev;
      p.csig = W.sigdev + a;
      formed[a] = 1;
    }
    return p;
  };
  const int nup = nR > nL ? nR : nL;
  for (int t = 0; t < nup; ++t) {
    const int jR = t < nR ? l - 1 - t : -1, jL = t < nL ? t : -1;
    if ((e = jR >= 0 ? inv2(jR, jL) : inv2(jL, -1)) != cudaSuccess) return e;
    ZGemmProblem p1[2], p2[4];
    int n1 = 0, n2 = 0;
    if (jR >= 0) {
      p1[n1++] = prob(b, b, b, sg, 0.0, blk(c.slot(jR, 0)), offd(jR, -1), lmo(jR));
      const ZOp up = offd(jR - 1, +1);
      p2[n2++] = win(jR - 1, up, lmo(jR));
      p2[n2++] = prob(b, b, b, sg, 0.0, up, blk(c.slot(jR, 0)), umo(jR));
    }
    if (jL >= 0) {
      p1[n1++] = prob(b, b, b, sg, 0.0, blk(c.slot(jL, 0)), offd(jL, +1), lmo(jL));
      const ZOp dn = offd(jL + 1, -1);
      p2[n2++] = win(jL + 1, dn, lmo(jL));
      p2[n2++] = prob(b, b, b, sg, 0.0, dn, blk(c.slot(jL, 0)), umo(jL));
    }
    if ((e = grp(p1, n1)) != cudaSuccess) return e;
    if (jR >= 0 && jL >= 0 && jR - 1 == jL + 1) {  // both chains correct layer m: serialise
      if ((e = grp(p2, 2)) != cudaSuccess) return e;
      if ((e = grp(p2 + 2, 2)) != cudaSuccess) return e;
    } else if ((e = grp(p2, n2)) != cudaSuccess) {
      return e;
    }
  }
  if ((e = inv2(m, -1)) != cudaSuccess) return e;

  // ---------------- two outward sweeps; after step t rows [lo, hi) are final
  int flo = m, fhi = m;  // rows [flo, fhi) already handed to rows_done
  auto flush = [&](int lo, int hi, bool force) -> cudaError_t {
    if (!W.rows_done) return cudaSuccess;
    if (!force && (flo - lo) + (hi - fhi) < W.hook_rows) return cudaSuccess;
    cudaError_t r = cudaSuccess;
    if (lo < flo) r = W.rows_done(lo, flo, W.e_off, W.batch, s);
    if (r == cudaSuccess && hi > fhi) r = W.rows_done(fhi, hi, W.e_off, W.batch, s);
    flo = lo;
    fhi = hi;
    return r;
  };
  const int ndown = nR > nL ? nR : nL;
  for (int t = 1; t <= ndown; ++t) {
    const int jR = m + t <= l - 1 ? m + t : -1, jL = m - t >= 0 ? m - t : -1;
    ZGemmProblem pa[4], pb[2];
    int na = 0, nb = 0;
    if (jR >= 0) {
      const ZOp gprev = blk(c.slot(jR - 1, 0));
      pa[na++] = prob(b, b, b, -1.0, 0.0, lmo(jR), gprev, blk(c.slot(jR, -1)));
      pa[na++] = prob(b, b, b, -1.0, 0.0, gprev, umo(jR), blk(c.slot(jR - 1, +1)));
      pb[nb++] = prob(b, b, b, -1.0, 1.0, lmo(jR), blk(c.slot(jR - 1, +1)), blk(c.slot(jR, 0)));
    }
    if (jL >= 0) {
      const ZOp gnext = blk(c.slot(jL + 1, 0));
      pa[na++] = prob(b, b, b, -1.0, 0.0, lmo(jL), gnext, blk(c.slot(jL, +1)));
      pa[na++] = prob(b, b, b, -1.0, 0.0, gnext, umo(jL), blk(c.slot(jL + 1, -1)));
      pb[nb++] = prob(b, b, b, -1.0, 1.0, lmo(jL), blk(c.slot(jL + 1, -1)), blk(c.slot(jL, 0)));
    }
    if ((e = grp(pa, na)) != cudaSuccess) return e;
    if ((e = grp(pb, nb)) != cudaSuccess) return e;
    const int lo = m - t <= 0 ? 0 : m - t + 1, hi = m + t >= l - 1 ? l : m + t;
    if ((e = flush(lo, hi, false)) != cudaSuccess) return e;
  }
  return flush(0, l, true);
}

// Two-ended sweep of the block n-diagonal recursion (w >= 2, A's band in G). The
// right chain of rgf_ndiag (rgf.hpp:98-114) eliminates layers l-1 .. m+w, its mirror
// eliminates 0 .. m-1 from the top, in lockstep (one inversion launch for both, the
// products of both in the same grouped launches while their windows are disjoint):
//   left, layer j:  Y_j = inv(M'[j,j]),  lm[j][t] = Y_j M'[j, j+t],  um[j][t] = M'[j+t, j] Y_j,
//                   M'[j+s, j+t] -= M'[j+s, j] lm[j][t]          (s, t = 1..w)
// The w middle layers [m, m+w) then hold the Schur complement of both sides; the
// one-ended recursion on that w-layer sub-band gives its full inverse, and the two
// outward sweeps (rgf.hpp:117-135 and its mirror) finish the band:
//   left, j = m-1 .. 0:  G[j, j+t] = -sum_s lm[j][s] G[j+s, j+t],
//                        G[j+t, j] = -sum_s G[j+t, j+s] um[j][s],
//                        G[j, j]   = Y_j - sum_s lm[j][s] G[j+s, j]
cudaError_t rgf_sweeps_two_w(const SweepWork& W, const int* n_true, int* status, int status_stride, cudaStream_t s) {
  Ctx c(W);
  const int l = W.l, w = W.w, b = W.bs, kb = w * b;
  const long long two_w = 2LL * w;
  const int m = (l - w) / 2, nR = l - (m + w), nL = m;
  cudaError_t e;
  auto grp = [&](const ZGemmProblem* ps, int np) {
    ZGemmGroup g{};
    g.batch = W.batch;
    g.bs = b;
    for (int i = 0; i < np; ++i) g.prob[g.nprob++] = ps[i];
    return zgemm_grouped(g, s);
  };
  auto inv1 = [&](int j) {
    return zinv_batched2(c.slot(j, 0), b, W.g_bstride, b, n_true[j], W.batch, 1, 0, W.inv,
                         status + (long long)j * status_stride, 0, s);
  };
  auto inv2 = [&](int jR, int jL) {
    if (jR < 0) return inv1(jL);
    if (jL < 0) return inv1(jR);
    if (n_true[jL] != n_true[jR]) {
      cudaError_t r = inv1(jR);
      return r != cudaSuccess ? r : inv1(jL);
    }
    double2* mR = c.slot(jR, 0);
    return zinv_batched2(mR, b, W.g_bstride, b, n_true[jR], W.batch, 2, (long long)(c.slot(jL, 0) - mR), W.inv,
                         status + (long long)jR * status_stride, (long long)(jL - jR) * status_stride, s);
  };
  // refinement of the multipliers (see refine_multipliers_default): pivot copies of
  // both chains and of the dense middle window
  const bool refine = W.fcopy != nullptr;
  double2* FR = W.fcopy;
  double2* FL = refine ? W.fcopy + (long long)W.batch * c.bb : nullptr;
  double2* D0 = refine ? W.fcopy + 2LL * W.batch * c.bb : nullptr;
  const ZOp opFR{FR, b, 0, 0, c.bb}, opFL{FL, b, 0, 0, c.bb};
  auto save = [&](double2* dst, int j) {
    return cudaMemcpy2DAsync(dst, c.bb * sizeof(double2), c.slot(j, 0), W.g_bstride * sizeof(double2),
                             c.bb * sizeof(double2), W.batch, cudaMemcpyDeviceToDevice, s);
  };
  // ---------------- inward chains
  const int nup = nR > nL ? nR : nL;
  for (int t = 0; t < nup; ++t) {
    const int jR = t < nR ? l - 1 - t : -1, jL = t < nL ? t : -1;
    if (refine && jR >= 0 && (e = save(FR, jR)) != cudaSuccess) return e;
    if (refine && jL >= 0 && (e = save(FL, jL)) != cudaSuccess) return e;
    if ((e = inv2(jR, jL)) != cudaSuccess) return e;
    ZGemmProblem p1[2], pR[2], pL[2];
    int n1 = 0;
    if (jR >= 0) {
      p1[n1++] = prob(b, kb, b, 1.0, 0.0, c.gop(c.slot(jR, 0), 0, 0), c.gop(c.slot(jR, -1), 0, -1),
                      c.mop(c.lm(jR), 0, 1));
      const ZOp upper = c.gop(c.slot(jR - 1, +1), -two_w, 0);
      pR[0] = prob(kb, kb, b, -1.0, 1.0, upper, c.mop(c.lm(jR), 0, 1), c.gop(c.slot(jR - 1, 0), -two_w, -1));
      pR[1] = prob(kb, b, b, 1.0, 0.0, upper, c.gop(c.slot(jR, 0), 0, 0), c.mop(c.um(jR), 1, 0));
    }
    if (jL >= 0) {
      p1[n1++] = prob(b, kb, b, 1.0, 0.0, c.gop(c.slot(jL, 0), 0, 0), c.gop(c.slot(jL, +1), 0, +1),
                      c.mop(c.lm(jL), 0, 1));
      const ZOp lower = c.gop(c.slot(jL + 1, -1), two_w, 0);
      pL[0] = prob(kb, kb, b, -1.0, 1.0, lower, c.mop(c.lm(jL), 0, 1), c.gop(c.slot(jL + 1, 0), two_w, +1));
      pL[1] = prob(kb, b, b, 1.0, 0.0, lower, c.gop(c.slot(jL, 0), 0, 0), c.mop(c.um(jL), 1, 0));
    }
    if ((e = grp(p1, n1)) != cudaSuccess) return e;
    if (refine) {  // R = M'(row) - f lm (in place in the row, not read again); lm += X R
      ZGemmProblem r1[2], r2[2];
      int nr = 0;
      if (jR >= 0) {
        const ZOp row = c.gop(c.slot(jR, -1), 0, -1);
        r1[nr] = prob(b, kb, b, -1.0, 1.0, opFR, c.mop(c.lm(jR), 0, 1), row);
        r2[nr++] = prob(b, kb, b, 1.0, 1.0, c.gop(c.slot(jR, 0), 0, 0), row, c.mop(c.lm(jR), 0, 1));
      }
      if (jL >= 0) {
        const ZOp row = c.gop(c.slot(jL, +1), 0, +1);
        r1[nr] = prob(b, kb, b, -1.0, 1.0, opFL, c.mop(c.lm(jL), 0, 1), row);
        r2[nr++] = prob(b, kb, b, 1.0, 1.0, c.gop(c.slot(jL, 0), 0, 0), row, c.mop(c.lm(jL), 0, 1));
      }
      if ((e = grp(r1, nr)) != cudaSuccess) return e;
      if ((e = grp(r2, nr)) != cudaSuccess) return e;
    }
    // windows: right rows/cols [jR-w, jR-1], left [jL+1, jL+w]; disjoint -> one launch
    if (jR >= 0 && jL >= 0 && jR - w > jL + w) {
      ZGemmProblem p2[4] = {pR[0], pR[1], pL[0], pL[1]};
      if ((e = grp(p2, 4)) != cudaSuccess) return e;
    } else {
      if (jR >= 0 && (e = grp(pR, 2)) != cudaSuccess) return e;
      if (jL >= 0 && (e = grp(pL, 2)) != cudaSuccess) return e;
    }
    if (refine) {  // R = M'(column) - um f (in place, not read again); um += R X
      ZGemmProblem r1[2], r2[2];
      int nr = 0;
      if (jR >= 0) {
        const ZOp col = c.gop(c.slot(jR - 1, +1), -two_w, 0);
        r1[nr] = prob(kb, b, b, -1.0, 1.0, c.mop(c.um(jR), 1, 0), opFR, col);
        r2[nr++] = prob(kb, b, b, 1.0, 1.0, col, c.gop(c.slot(jR, 0), 0, 0), c.mop(c.um(jR), 1, 0));
      }
      if (jL >= 0) {
        const ZOp col = c.gop(c.slot(jL + 1, -1), two_w, 0);
        r1[nr] = prob(kb, b, b, -1.0, 1.0, c.mop(c.um(jL), 1, 0), opFL, col);
        r2[nr++] = prob(kb, b, b, 1.0, 1.0, col, c.gop(c.slot(jL, 0), 0, 0), c.mop(c.um(jL), 1, 0));
      }
      if ((e = grp(r1, nr)) != cudaSuccess) return e;
      if ((e = grp(r2, nr)) != cudaSuccess) return e;
    }
  }
  // ---------------- the w middle layers: their (w b) x (w b) Schur complement inverted as
  // one dense matrix (partial pivoting across its layers), or by the one-ended recursion
  // on the sub-band [m, m+w) when the layers are ragged / no dense scratch was given
  bool uniform = true;
  for (int a = m; a < m + w; ++a) uniform = uniform && n_true[a] == b;
  if (W.mid && uniform) {
    const long long wb2 = (long long)kb * kb;
    double2* D = static_cast<double2*>(W.mid);
    void* zs = static_cast<char*>(W.mid) + mid_dense_bytes(w, b, W.batch);
    if ((e = band_window(W.G, W.g_bstride, D, m, w, b, W.batch, true, s)) != cudaSuccess) return e;
    if (refine && (e = cudaMemcpyAsync(D0, D, sizeof(double2) * size_t(wb2) * W.batch, cudaMemcpyDeviceToDevice, s)))
      return e;
    if ((e = zinv_batched(D, kb, wb2, kb, kb, W.batch, zs, status + (long long)m * status_stride, s)) != cudaSuccess)
      return e;
    if (refine) {  // Newton-Schulz: X += X (I - D0 X); D0 <- I - D0 X in place, then the update
      ZGemmGroup g{};
      g.batch = W.batch;
      g.bs = kb;
      g.nprob = 1;
      ZGemmProblem& q = g.prob[0];
      q.M = q.N = q.K = kb;
      // D0 <- -D0 X (beta 0), then + I on its diagonal
      q.alpha = make_double2(-1.0, 0.0);
      q.beta = make_double2(0.0, 0.0);
      q.A = ZOp{D0, kb, 0, 0, wb2};
      q.B = ZOp{D, kb, 0, 0, wb2};
      q.C = q.D = ZOp{D0 + 0, kb, 0, 0, wb2};
      // the product may not overwrite its own A operand tile by tile: go through the
      // multiplier scratch of layer m (free at this point: >= kb*kb per batch entry)
      double2* T = c.lm(m);
      const long long tstride = c.lm_bstride();
      q.C = q.D = ZOp{T, kb, 0, 0, tstride};
      if ((e = zgemm_grouped(g, s)) != cudaSuccess) return e;
      if ((e = diag_shift_batched(T, kb, tstride, W.batch, s)) != cudaSuccess) return e;
      // D0 <- X R, then X += D0
      q.alpha = make_double2(1.0, 0.0);
      q.A = ZOp{D, kb, 0, 0, wb2};
      q.B = ZOp{T, kb, 0, 0, tstride};
      q.C = q.D = ZOp{D0, kb, 0, 0, wb2};
      if ((e = zgemm_grouped(g, s)) != cudaSuccess) return e;
      if ((e = axpy_batched(D, D0, wb2 * W.batch, s)) != cudaSuccess) return e;
    }
    if ((e = band_window(W.G, W.g_bstride, D, m, w, b, W.batch, false, s)) != cudaSuccess) return e;
    // layers m+1 .. m+w-1 have no pivot of their own here: status -1 (0xff bytes)
    if ((e = cudaMemset2DAsync(status + (long long)(m + 1) * status_stride, sizeof(int) * size_t(status_stride), 0xff,
                               sizeof(int) * size_t(W.batch), size_t(w - 1), s)) != cudaSuccess)
      return e;
  } else {
    SweepWork Wm = W;
    Wm.l = w;
    Wm.lm_layers = W.lm_layers > 0 ? W.lm_layers : l;
    Wm.G = c.slot(m, -w);
    Wm.LM = c.lm(m);
    Wm.UM = c.um(m);
    Wm.rows_done = nullptr;
    Wm.two_ended = false;
    if ((e = rgf_sweeps_one(Wm, n_true + m, status + (long long)m * status_stride, status_stride, s)) != cudaSuccess)
      return e;
  }
  // ---------------- outward sweeps; after step t rows [lo, hi) are final
  int flo = m + w, fhi = m + w;
  bool any = false;
  auto flush = [&](int lo, int hi, bool force) -> cudaError_t {
    if (!W.rows_done || lo >= hi) return cudaSuccess;
    if (!any) {  // first complete range
      if (!force && hi - lo < W.hook_rows) return cudaSuccess;
      any = true;
      flo = lo;
      fhi = hi;
      return W.rows_done(lo, hi, W.e_off, W.batch, s);
    }
    if (!force && (flo - lo) + (hi - fhi) < W.hook_rows) return cudaSuccess;
    cudaError_t r = cudaSuccess;
    if (lo < flo) r = W.rows_done(lo, flo, W.e_off, W.batch, s);
    if (r == cudaSuccess && hi > fhi) r = W.rows_done(fhi, hi, W.e_off, W.batch, s);
    flo = lo;
    fhi = hi;
    return r;
  };
  const int ndown = nR > nL ? nR : nL;
  for (int t = 1; t <= ndown; ++t) {
    const int jR = t <= nR ? m + w - 1 + t : -1, jL = t <= nL ? m - t : -1;
    ZGemmProblem pa[4], pb[2];
    int na = 0, nb = 0;
    if (jR >= 0) {
      const ZOp lmrow = c.mop(c.lm(jR), 0, 1), window = c.gop(c.slot(jR - 1, 0), -two_w, -1);
      pa[na++] = prob(b, kb, kb, -1.0, 0.0, lmrow, window, c.gop(c.slot(jR, -1), 0, -1));
      pa[na++] = prob(kb, b, kb, -1.0, 0.0, window, c.mop(c.um(jR), 1, 0), c.gop(c.slot(jR - 1, +1), -two_w, 0));
      pb[nb++] = prob(b, b, kb, -1.0, 1.0, lmrow, c.gop(c.slot(jR - 1, +1), -two_w, 0), c.gop(c.slot(jR, 0), 0, 0));
    }
    if (jL >= 0) {
      const ZOp lmrow = c.mop(c.lm(jL), 0, 1), window = c.gop(c.slot(jL + 1, 0), two_w, +1);
      pa[na++] = prob(b, kb, kb, -1.0, 0.0, lmrow, window, c.gop(c.slot(jL, +1), 0, +1));
      pa[na++] = prob(kb, b, kb, -1.0, 0.0, window, c.mop(c.um(jL), 1, 0), c.gop(c.slot(jL + 1, -1), two_w, 0));
      pb[nb++] = prob(b, b, kb, -1.0, 1.0, lmrow, c.gop(c.slot(jL + 1, -1), two_w, 0), c.gop(c.slot(jL, 0), 0, 0));
    }
    if ((e = grp(pa, na)) != cudaSuccess) return e;
    if ((e = grp(pb, nb)) != cudaSuccess) return e;
    const int rdone = t <= nR ? jR : l - 1, ldone = t <= nL ? jL : 0;
    const int hi = rdone >= l - 1 ? l : rdone - w + 1, lo = ldone <= 0 ? 0 : ldone + w;
    if ((e = flush(lo, hi, false)) != cudaSuccess) return e;
  }
  return flush(0, l, true);
}

struct StreamPool {
  int dev = -1;
  std::vector<cudaStream_t> s;
  std::vector<cudaEvent_t> ev;
};
// Per host thread (and device): concurrent callers on different threads get their own
// side streams and events, so their sweeps overlap instead of interleaving on shared ones.
thread_local std::vector<StreamPool> t_pools;

StreamPool& pool_for(int n) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (int(t_pools.size()) <= dev) t_pools.resize(dev + 1);
  StreamPool& p = t_pools[dev];
  p.dev = dev;
  while (int(p.s.size()) < n) {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    p.s.push_back(st);
  }
  while (int(p.ev.size()) < n + 1) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    p.ev.push_back(e);
  }
  return p;
}

}  // namespace

cudaError_t rgf_sweeps(const SweepWork& W, const int* n_true, cudaStream_t s) {
  // the buffers every sweep GEMM operand lives in, for the TMA-staged GEMM
  TmaScope tma;
  {
    const size_t bb16 = size_t(W.bs) * W.bs * sizeof(double2);
    const size_t band = size_t(W.l) * (2 * W.w + 1) * bb16;
    tma.add(W.G, size_t(W.batch - 1) * W.g_bstride * sizeof(double2) + band, W.bs);
    const size_t lmb = size_t(W.batch) * (W.lm_layers > 0 ? W.lm_layers : W.l) * W.w * bb16;
    tma.add(W.LM, lmb, W.bs);
    tma.add(W.UM, lmb, W.bs);
    if (W.Hoff) tma.add(W.Hoff, band, W.bs);
  }
  const int G = W.groups < 1 ? 1 : (W.groups > W.batch ? W.batch : W.groups);
  const int sstride = W.status_stride > 0 ? W.status_stride : W.batch;
  // dense middle window of the banded two-ended sweep: one scratch per stream group
  char* mid = (W.mid && mid_dense_enabled()) ? static_cast<char*>(W.mid) : nullptr;
  const size_t mid_g = mid ? mid_bytes(W.w, W.bs, (W.batch + G - 1) / G) : 0;
  auto sweep = [&](const SweepWork& X0, int* st, cudaStream_t q, int g) {
    SweepWork X = X0;
    X.mid = mid ? mid + mid_g * g : nullptr;
    if (!use_two_ended(X)) return rgf_sweeps_one(X, n_true, st, sstride, q);
    return X.w == 1 ? rgf_sweeps_two(X, n_true, st, sstride, q) : rgf_sweeps_two_w(X, n_true, st, sstride, q);
  };
  zinv_set_concurrency(G);
  struct ConcReset {
    ~ConcReset() { zinv_set_concurrency(1); }
  } conc_reset;
  if (G == 1) return sweep(W, W.status, s, 0);
  // Independent batch groups on side streams: one group's latency-bound pivot
  // inversions overlap the other groups' GEMMs.
  StreamPool& P = pool_for(G);
  cudaError_t e;
  if ((e = cudaEventRecord(P.ev[G], s))) return e;
  const int gs = (W.batch + G - 1) / G;
  const long long bb = (long long)W.bs * W.bs;
  const size_t inv_b = zinv_scratch_bytes(W.bs, (use_two_ended(W) ? 2 : 1) * gs) + 256;
  for (int g = 0; g < G; ++g) {
    const int e0 = g * gs, ne = std::min(gs, W.batch - e0);
    if (ne <= 0) break;
    SweepWork Wg = W;
    Wg.batch = ne;
    Wg.G = W.G + (long long)e0 * W.g_bstride;
    Wg.LM = W.LM + (long long)e0 * W.l * W.w * bb;
    Wg.UM = W.UM + (long long)e0 * W.l * W.w * bb;
    Wg.inv = static_cast<char*>(W.inv) + size_t(g) * inv_b;
    Wg.e_off = W.e_off + e0;
    if (W.zdev) Wg.zdev = W.zdev + e0;
    if (W.fcopy) Wg.fcopy = W.fcopy + (long long)g * fcopy_elems(W.l, W.w, W.bs, gs, W.two_ended);
    if ((e = cudaStreamWaitEvent(P.s[g], P.ev[G], 0))) return e;
    if ((e = sweep(Wg, W.status + e0, P.s[g], g))) return e;
    if ((e = cudaEventRecord(P.ev[g], P.s[g]))) return e;
    if ((e = cudaStreamWaitEvent(s, P.ev[g], 0))) return e;
  }
  return cudaSuccess;
}

cudaError_t collect_failures(const SweepWork& W, std::vector<int>& fail, cudaStream_t s) {
  std::vector<int> st(size_t(W.l) * W.batch);
  cudaError_t e = cudaMemcpyAsync(st.data(), W.status, st.size() * sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  fail.assign(W.batch, -1);
  // elimination order of the reference: l-1, l-2, ..., 0 (rgf.hpp:58,64 / :100,114)
  for (int bt = 0; bt < W.batch; ++bt)
    for (int j = W.l - 1; j >= 0; --j)
      if (st[size_t(j) * W.batch + bt] >= 0) {
        fail[bt] = j;
        break;
      }
  return cudaSuccess;
}

// ------------------------------------------------------------------ arena
// Grow-only device workspace, one set of slots per (host thread, device): calls made
// from different host threads never share scratch, so they may run concurrently (the
// reference solvers are reentrant).
namespace {
struct Buf {
  void* p = nullptr;
  size_t n = 0;
};
thread_local std::vector<std::vector<Buf>> t_arena;  // [device][slot]
thread_local std::vector<std::vector<cudaStream_t>> t_streams;  // [device][which]
}  // namespace

cudaStream_t thread_stream(int which) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (int(t_streams.size()) <= dev) t_streams.resize(dev + 1);
  auto& v = t_streams[dev];
  while (int(v.size()) <= which) {
    cudaStream_t st = nullptr;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    v.push_back(st);
  }
  return v[which];
}

void* arena_get(int slot, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (int(t_arena.size()) <= dev) t_arena.resize(dev + 1);
  auto& v = t_arena[dev];
  if (int(v.size()) <= slot) v.resize(slot + 1);
  Buf& b = v[slot];
  if (b.n >= bytes && b.p) return b.p;
  if (b.p) {
    cudaDeviceSynchronize();
    cudaFree(b.p);
    b.p = nullptr;
    b.n = 0;
  }
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    return nullptr;
  }
  b.n = bytes;
  return b.p;
}

size_t arena_held(std::initializer_list<int> slots) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (int(t_arena.size()) <= dev) return 0;
  size_t n = 0;
  for (int sl : slots)
    if (sl < int(t_arena[dev].size()) && t_arena[dev][sl].p) n += t_arena[dev][sl].n;
  return n;
}

void arena_release_all() {
  int cur = 0;
  cudaGetDevice(&cur);
  for (size_t d = 0; d < t_arena.size(); ++d) {
    bool any = false;
    for (auto& b : t_arena[d]) any |= b.p != nullptr;
    if (!any) continue;
    cudaSetDevice(int(d));
    cudaDeviceSynchronize();
    for (auto& b : t_arena[d])
      if (b.p) cudaFree(b.p), b.p = nullptr, b.n = 0;
  }
  cudaSetDevice(cur);
}

void thread_resources_release() {
  arena_release_all();
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& p : t_pools) {
    if (p.dev < 0) continue;
    cudaSetDevice(p.dev);
    for (auto st : p.s) cudaStreamDestroy(st);
    for (auto e : p.ev) cudaEventDestroy(e);
    p.s.clear();
    p.ev.clear();
  }
  for (size_t d = 0; d < t_streams.size(); ++d) {
    if (t_streams[d].empty()) continue;
    cudaSetDevice(int(d));
    for (auto st : t_streams[d]) cudaStreamDestroy(st);
    t_streams[d].clear();
  }
  cudaSetDevice(cur);
}

}  // namespace bbsi_gpu

// Domain-decomposition RGF (DDRGF) on the device, stabilised formulation.
//
// Same decomposition and outputs as the reference ddrgf (ddrgf.hpp:344-428,
// partition.hpp:39-75): interior groups of s2 layers separated by single-layer
// separators, the last separator being the chain end; the result is the
// block-tridiagonal part of G = A^{-1}. The reference eliminates each isolated
// domain (rgf_extended, rgf.hpp:209-270), assembles the separator Schur system
// (ddrgf.hpp:282-303) and applies W S^{-1} V corrections (ddrgf.hpp:142-235).
// On the BASELINE Dyson matrices (indefinite, damped only by i*eta) isolated
// domains are nearly singular and that formulation loses 3-6 digits (SURVEY.md
// finding 3). This version never forms an isolated-domain inverse:
//
//   phase 1 (batched over domains): RGF of every domain with FAKE absorbing leads
//     Sigma0 = -i*gamma*I on its first and last block -> corners a, b, c, e of a
//     well-conditioned inverse (b, c by the first-row / first-column recurrences
//     G[0,j] = -G[0,j-1] um_j, G[j,0] = -lm_j G[j-1,0], rgf.hpp:250-258 in O(s2));
//   phase 2 (sequential over the P separators, b x b work): left- and
//     right-connected Green's functions at every separator; the true boundary
//     self-energy replaces the fake lead through two rank-b Woodbury updates of
//     the corners (one b x b inverse each);
//   phase 3 (batched over domains): plain RGF of every chain [domain, right
//     separator] with the exact boundary self-energies on its end blocks, written
//     in place into the output band; separator couplings from the right-connected
//     Green's functions, G[f, s-1] = -gR_f A[f, s-1] G[s-1, s-1].
//
// All chains live in the output band itself (domain i + separator i occupy a
// contiguous run of slots with a uniform stride), so no extra band buffers exist.
#include <algorithm>
#include <vector>

#include "internal.h"

namespace bbsi_gpu {

namespace {

__global__ void diag_add_kernel(double2* base, long long stride, int n, int nblk, double2 v) {
  const int b = blockIdx.y;
  if (b >= nblk) return;
  double2* m = base + (long long)b * stride;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double2 x = m[(long long)i * n + i];
    m[(long long)i * n + i] = make_double2(x.x + v.x, x.y + v.y);
  }
}

cudaError_t diag_add(double2* base, long long stride, int n, int nblk, double2 v, cudaStream_t s) {
  if (nblk <= 0) return cudaSuccess;
  ProfScope prof(s, PROF_BAND, 0.0, 32.0 * n * nblk);
  diag_add_kernel<<<dim3((n + 255) / 256, nblk), 256, 0, s>>>(base, stride, n, nblk, v);
  return cudaGetLastError();
}

__global__ void axpy_kernel(double2* y, const double2* x, long long n, double2 a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = cfma(a, x[i], y[i]);
}

// y += a * x (n complex entries)
cudaError_t axpy(double2* y, const double2* x, long long n, double2 a, cudaStream_t s) {
  ProfScope prof(s, PROF_BAND, 8.0 * n, 48.0 * n);
  axpy_kernel<<<(int)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0, s>>>(y, x, n, a);
  return cudaGetLastError();
}

// b x b plain operands (ld = b) with a batch stride (elements)
ZOp blk(const double2* p, int b, long long bstride = 0) { return ZOp{p, b, 64, 64LL * b, bstride}; }

// D = alpha * A * B + beta * C over `batch` independent b x b products (C may alias D)
cudaError_t mm(int b, int batch, double alpha, ZOp A, ZOp B, double beta, ZOp C, cudaStream_t s) {
  ZGemmGroup g{};
  g.batch = batch;
  g.bs = 64;
  g.nprob = 1;
  ZGemmProblem& p = g.prob[0];
  p.M = b;
  p.N = b;
  p.K = b;
  p.alpha = make_double2(alpha, 0.0);
  p.beta = make_double2(beta, 0.0);
  p.A = A;
  p.B = B;
  p.C = C;
  p.D = C;
  return zgemm_grouped(g, s);
}

// complex-scaled product: D = alpha * A * B + beta * C with complex alpha
cudaError_t mmz(int b, double2 alpha, ZOp A, ZOp B, double beta, ZOp C, cudaStream_t s) {
  ZGemmGroup g{};
  g.batch = 1;
  g.bs = 64;
  g.nprob = 1;
  ZGemmProblem& p = g.prob[0];
  p.M = b;
  p.N = b;
  p.K = b;
  p.alpha = alpha;
  p.beta = make_double2(beta, 0.0);
  p.A = A;
  p.B = B;
  p.C = C;
  p.D = C;
  return zgemm_grouped(g, s);
}

struct Part {
  std::vector<int> first, count, sep;  // per task
  int T = 0;
};

// interleave_permutation(layout, 1, s2) (partition.hpp:39-75)
Part partition(int l, int s2) {
  Part P;
  int pos = 0;
  while (pos < l) {
    const int rem = l - pos;
    int d2, d1;
    if (rem >= 1 + s2) {
      d2 = s2;
      d1 = 1;
    } else {
      d1 = std::min(1, rem);
      d2 = rem - d1;
    }
    P.first.push_back(pos);
    P.count.push_back(d2);
    P.sep.push_back(pos + d2);
    pos += d2 + d1;
  }
  P.T = int(P.first.size());
  return P;
}

}  // namespace

ZOp zblk(const double2* p, int b, long long bstride) { return blk(p, b, bstride); }

cudaError_t zmm(int b, int batch, double2 alpha, ZOp A, ZOp B, double beta, ZOp C, cudaStream_t s) {
  ZGemmGroup g{};
  g.batch = batch;
  g.bs = 64;
  g.nprob = 1;
  ZGemmProblem& p = g.prob[0];
  p.M = b;
  p.N = b;
  p.K = b;
  p.alpha = alpha;
  p.beta = make_double2(beta, 0.0);
  p.A = A;
  p.B = B;
  p.C = C;
  p.D = C;
  return zgemm_grouped(g, s);
}

cudaError_t ddrgf_device(const double2* A, double2* G, int l, int b, const int* n_true, int s2, double gamma,
                         void* scratch, size_t scratch_bytes, int* fail_layer, cudaStream_t s) {
  *fail_layer = -1;
  const long long bb = (long long)b * b;
  const long long slot3 = 3 * bb;
  auto aslot = [&](int a, int off) { return A + ((long long)a * 3 + off + 1) * bb; };
  auto gslot = [&](int a, int off) { return G + ((long long)a * 3 + off + 1) * bb; };
  const Part P = partition(l, s2);
  const int T = P.T;
  // full-length domains are tasks 0..nfull-1 (all but possibly the trailing one)
  int nfull = T;
  if (P.count[T - 1] != s2) nfull = T - 1;
  const int tc = P.count[T - 1];  // trailing interior count (== s2 when nfull == T)
  cudaError_t e;

  // ---- device scratch carve: per-task b x b matrices
  enum { KA, KB, KC, KE, GL, GR, GLD, GRD, NMAT };
  const size_t per = size_t(NMAT) * T * bb * sizeof(double2);
  const size_t tmp_n = 8;  // temporaries for phase 2
  const size_t need = per + tmp_n * bb * sizeof(double2) + 2 * size_t(T) * bb * sizeof(double2);
  if (scratch_bytes < need) return cudaErrorMemoryAllocation;
  double2* mats = static_cast<double2*>(scratch);
  auto M_ = [&](int kind, int t) { return mats + ((size_t)kind * T + t) * bb; };
  double2* tmp = mats + (size_t)NMAT * T * bb;
  auto Tm = [&](int i) { return tmp + (size_t)i * bb; };
  double2* rc = tmp + tmp_n * bb;  // [2][T] ping-pong for the first row / column chains (R, C)

  // ================= phase 1: corners with fake absorbing leads
  if ((e = cudaMemcpyAsync(G, A, sizeof(double2) * size_t(l) * slot3, cudaMemcpyDeviceToDevice, s))) return e;
  const double2 ig = make_double2(0.0, gamma);  // -Sigma0 = +i*gamma
  // fake leads on the first and last block of every nonempty domain
  for (int t = 0; t < T; ++t) {
    if (P.count[t] == 0) continue;
    if ((e = diag_add(gslot(P.first[t], 0), 0, b, 1, ig, s))) return e;
    if ((e = diag_add(gslot(P.first[t] + P.count[t] - 1, 0), 0, b, 1, ig, s))) return e;
  }
  auto sweep = [&](int first_task, int ntask, int len, SweepWork& W, std::vector<int>& fails) -> cudaError_t {
    W = SweepWork{};
    W.l = len;
    W.w = 1;
    W.bs = b;
    W.batch = ntask;
    W.G = gslot(P.first[first_task], -1);
    W.g_bstride = (long long)(s2 + 1) * slot3;
    W.groups = default_groups(ntask, b);
    void* sc = arena_get(6, sweep_scratch_bytes(len, 1, b, ntask, W.groups));
    if (!sc) return cudaErrorMemoryAllocation;
    sweep_carve(W, sc);
    std::vector<int> nt(len, b);
    for (int j = 0; j < len; ++j) nt[j] = n_true ? n_true[P.first[first_task] + j] : b;
    cudaError_t e2 = rgf_sweeps(W, nt.data(), s);
    if (e2) return e2;
    return collect_failures(W, fails, s);
  };
  auto first_fail = [&](const std::vector<int>& fails, int first_task) {
    for (size_t q = 0; q < fails.size(); ++q)
      if (fails[q] >= 0) return P.first[first_task + q] + fails[q];
    return -1;
  };
  // corners of a batch of domains (tasks t0..t0+nt-1, all of length len) from a finished sweep
  auto corners = [&](int t0, int nt, int len, const SweepWork& W) -> cudaError_t {
    cudaError_t e2;
    const long long gs = W.g_bstride;
    // a = G[0,0], e = G[len-1,0]
    if ((e2 = cudaMemcpy2DAsync(M_(KA, t0), bb * sizeof(double2), gslot(P.first[t0], 0), gs * sizeof(double2),
                                bb * sizeof(double2), nt, cudaMemcpyDeviceToDevice, s)))
      return e2;
    if ((e2 = cudaMemcpy2DAsync(M_(KE, t0), bb * sizeof(double2), gslot(P.first[t0] + len - 1, 0),
                                gs * sizeof(double2), bb * sizeof(double2), nt, cudaMemcpyDeviceToDevice, s)))
      return e2;
    // first row R_j = G[0,j] = -R_{j-1} um_j ; first column C_j = G[j,0] = -lm_j C_{j-1}
    // ping-pong between the b / c output slots and scratch (nt matrices each)
    double2* pr = rc;             // R ping  [nt]
    double2* pc = rc + nt * bb;   // C ping  [nt]  (rc has 2*T matrices)
    if (len == 1) {
      if ((e2 = cudaMemcpyAsync(M_(KB, t0), M_(KA, t0), nt * bb * sizeof(double2), cudaMemcpyDeviceToDevice, s)))
        return e2;
      return cudaMemcpyAsync(M_(KC, t0), M_(KA, t0), nt * bb * sizeof(double2), cudaMemcpyDeviceToDevice, s);
    }
    // R_0 = C_0 = a; chains alternate between (pr/pc) and the output slots (KB/KC)
    double2* r_cur = M_(KA, t0);
    double2* c_cur = M_(KA, t0);
    for (int j = 1; j < len; ++j) {
      const bool to_out = ((len - 1 - j) % 2) == 0;  // the last step lands in KB / KC
      double2* r_nxt = to_out ? M_(KB, t0) : pr;
      double2* c_nxt = to_out ? M_(KC, t0) : pc;
      const double2* um = W.UM + (long long)j * bb;  // um[j] (w = 1), batch stride l*bb
      const double2* lm = W.LM + (long long)j * bb;
      ZGemmGroup g{};
      g.batch = nt;
      g.bs = 64;
      g.nprob = 2;
      ZGemmProblem& p0 = g.prob[0];
      p0.M = p0.N = p0.K = b;
      p0.alpha = make_double2(-1.0, 0.0);
      p0.beta = make_double2(0.0, 0.0);
      p0.A = blk(r_cur, b, bb);
      p0.B = blk(um, b, (long long)W.l * bb);
      p0.C = p0.D = blk(r_nxt, b, bb);
      ZGemmProblem& p1 = g.prob[1];
      p1 = p0;
      p1.A = blk(lm, b, (long long)W.l * bb);
      p1.B = blk(c_cur, b, bb);
      p1.C = p1.D = blk(c_nxt, b, bb);
      if ((e2 = zgemm_grouped(g, s))) return e2;
      r_cur = r_nxt;
      c_cur = c_nxt;
    }
    return cudaSuccess;
  };
  {
    SweepWork W;
    std::vector<int> fails;
    if (nfull > 0) {
      if ((e = sweep(0, nfull, s2, W, fails))) return e;
      if ((*fail_layer = first_fail(fails, 0)) >= 0) return cudaSuccess;
      if ((e = corners(0, nfull, s2, W))) return e;
    }
    if (nfull < T && tc > 0) {
      if ((e = sweep(T - 1, 1, tc, W, fails))) return e;
      if ((*fail_layer = first_fail(fails, T - 1)) >= 0) return cudaSuccess;
      if ((e = corners(T - 1, 1, tc, W))) return e;
    }
  }

  // ================= phase 3 input: fresh copy of A (phase 2 adds the self-energies)
  if ((e = cudaMemcpyAsync(G, A, sizeof(double2) * size_t(l) * slot3, cudaMemcpyDeviceToDevice, s))) return e;

  // ================= phase 2: left / right sweeps over the separators (b x b work)
  const int max_inv = 6 * T + 2;
  void* inv_scr = arena_get(7, zinv_scratch_bytes(b, 1) + 256);
  int* st = static_cast<int*>(arena_get(8, sizeof(int) * size_t(max_inv)));
  if (!inv_scr || !st) return cudaErrorMemoryAllocation;
  std::vector<int> st_layer;  // layer to blame per inversion (failure attribution)
  auto inv = [&](double2* m, int layer) -> cudaError_t {
    if (int(st_layer.size()) >= max_inv) return cudaErrorInvalidValue;
    int* slot = st + st_layer.size();
    st_layer.push_back(layer);
    return zinv_batched(m, b, bb, b, n_true ? n_true[layer] : b, 1, inv_scr, slot, s);
  };
  auto ident = [&](double2* m) -> cudaError_t {
    cudaError_t e2 = cudaMemsetAsync(m, 0, bb * sizeof(double2), s);
    return e2 ? e2 : diag_add(m, 0, b, 1, make_double2(1.0, 0.0), s);
  };
  auto copy = [&](double2* d, const double2* x) {
    return cudaMemcpyAsync(d, x, bb * sizeof(double2), cudaMemcpyDeviceToDevice, s);
  };
  // out = x + i*gamma * x (I - i*gamma x)^{-1} x   (removes the fake lead -i*gamma at the block of x)
  auto remove_fake = [&](double2* out, double2* x, int layer) -> cudaError_t {
    cudaError_t e2;
    if ((e2 = ident(Tm(2)))) return e2;
    if ((e2 = axpy(Tm(2), x, bb, make_double2(0.0, -gamma), s))) return e2;
    if ((e2 = inv(Tm(2), layer))) return e2;
    if ((e2 = mm(b, 1, 1.0, blk(Tm(2), b), blk(x, b), 0.0, blk(Tm(3), b), s))) return e2;
    if ((e2 = copy(out, x))) return e2;
    return mmz(b, make_double2(0.0, gamma), blk(x, b), blk(Tm(3), b), 1.0, blk(out, b), s);
  };
  // left sweep
  for (int t = 0; t < T; ++t) {
    const int f = P.first[t], cnt = P.count[t], sp = P.sep[t];
    double2* gl = M_(GL, t);
    if (cnt > 0) {
      double2* Df = Tm(1);
      if (t > 0) {  // Sigma^L = A[f,-1] gL_{t-1} A[f-1,+1], also subtracted from phase 3's first block
        if ((e = mm(b, 1, 1.0, blk(aslot(f, -1), b), blk(M_(GL, t - 1), b), 0.0, blk(Tm(0), b), s))) return e;
        if ((e = mm(b, 1, 1.0, blk(Tm(0), b), blk(aslot(f - 1, 1), b), 0.0, blk(Df, b), s))) return e;
        if ((e = axpy(gslot(f, 0), Df, bb, make_double2(-1.0, 0.0), s))) return e;
      } else {
        if ((e = cudaMemsetAsync(Df, 0, bb * sizeof(double2), s))) return e;
      }
      // step A (true lead at f): Df = Sigma^L - Sigma0 ; P = I - Df a ; e' = e + c P^{-1} Df b
      if ((e = diag_add(Df, 0, b, 1, ig, s))) return e;
      if ((e = ident(Tm(2)))) return e;
      if ((e = mm(b, 1, -1.0, blk(Df, b), blk(M_(KA, t), b), 1.0, blk(Tm(2), b), s))) return e;
      if ((e = inv(Tm(2), f))) return e;
      if ((e = mm(b, 1, 1.0, blk(Tm(2), b), blk(Df, b), 0.0, blk(Tm(3), b), s))) return e;
      if ((e = mm(b, 1, 1.0, blk(Tm(3), b), blk(M_(KB, t), b), 0.0, blk(Tm(4), b), s))) return e;
      if ((e = copy(Tm(5), M_(KE, t)))) return e;
      if ((e = mm(b, 1, 1.0, blk(M_(KC, t), b), blk(Tm(4), b), 1.0, blk(Tm(5), b), s))) return e;
      // step B (drop the fake lead at l): gLdom
      if ((e = remove_fake(M_(GLD, t), Tm(5), f + cnt - 1))) return e;
      if ((e = mm(b, 1, 1.0, blk(aslot(sp, -1), b), blk(M_(GLD, t), b), 0.0, blk(Tm(0), b), s))) return e;
    } else {
      if (t == 0) return cudaErrorInvalidValue;  // task 0 always has interior layers
      if ((e = mm(b, 1, 1.0, blk(aslot(sp, -1), b), blk(M_(GL, t - 1), b), 0.0, blk(Tm(0), b), s))) return e;
    }
    // gL_t = (A[s,0] - Tm0 A[s-1,+1])^{-1}; an empty trailing domain also puts Sigma^L on G[s,0]
    if ((e = copy(gl, aslot(sp, 0)))) return e;
    if ((e = mm(b, 1, 1.0, blk(Tm(0), b), blk(aslot(sp - 1, 1), b), 0.0, blk(Tm(1), b), s))) return e;
    if ((e = axpy(gl, Tm(1), bb, make_double2(-1.0, 0.0), s))) return e;
    if (cnt == 0 && (e = axpy(gslot(sp, 0), Tm(1), bb, make_double2(-1.0, 0.0), s))) return e;
    if ((e = inv(gl, sp))) return e;
  }
  // right sweep
  for (int t = T - 1; t >= 0; --t) {
    const int sp = P.sep[t];
    double2* gr = M_(GR, t);
    if ((e = copy(gr, aslot(sp, 0)))) return e;
    if (t < T - 1) {  // Sigma^R of separator t = A[s,+1] Y A[s+1,-1], also subtracted from phase 3's G[s,0]
      const double2* Y = P.count[t + 1] > 0 ? M_(GRD, t + 1) : M_(GR, t + 1);
      if ((e = mm(b, 1, 1.0, blk(aslot(sp, 1), b), blk(Y, b), 0.0, blk(Tm(0), b), s))) return e;
      if ((e = mm(b, 1, 1.0, blk(Tm(0), b), blk(aslot(sp + 1, -1), b), 0.0, blk(Tm(1), b), s))) return e;
      if ((e = axpy(gr, Tm(1), bb, make_double2(-1.0, 0.0), s))) return e;
      if ((e = axpy(gslot(sp, 0), Tm(1), bb, make_double2(-1.0, 0.0), s))) return e;
    }
    if ((e = inv(gr, sp))) return e;
    const int cnt = P.count[t];
    if (cnt > 0) {
      const int last = P.first[t] + cnt - 1;
      // step A (true lead at l): Dl = A[l,+1] gR_t A[s,-1] - Sigma0 ; P = I - Dl e ; a' = a + b P^{-1} Dl c
      double2* Dl = Tm(1);
      if ((e = mm(b, 1, 1.0, blk(aslot(last, 1), b), blk(gr, b), 0.0, blk(Tm(0), b), s))) return e;
      if ((e = mm(b, 1, 1.0, blk(Tm(0), b), blk(aslot(sp, -1), b), 0.0, blk(Dl, b), s))) return e;
      if ((e = diag_add(Dl, 0, b, 1, ig, s))) return e;
      if ((e = ident(Tm(2)))) return e;
      if ((e = mm(b, 1, -1.0, blk(Dl, b), blk(M_(KE, t), b), 1.0, blk(Tm(2), b), s))) return e;
      if ((e = inv(Tm(2), last))) return e;
      if ((e = mm(b, 1, 1.0, blk(Tm(2), b), blk(Dl, b), 0.0, blk(Tm(3), b), s))) return e;
      if ((e = mm(b, 1, 1.0, blk(Tm(3), b), blk(M_(KC, t), b), 0.0, blk(Tm(4), b), s))) return e;
      if ((e = copy(Tm(5), M_(KA, t)))) return e;
      if ((e = mm(b, 1, 1.0, blk(M_(KB, t), b), blk(Tm(4), b), 1.0, blk(Tm(5), b), s))) return e;
      // step B (drop the fake lead at f): gRdom
      if ((e = remove_fake(M_(GRD, t), Tm(5), P.first[t]))) return e;
    }
  }
  {  // phase 2 failures, first in issue order
    std::vector<int> sh(st_layer.size());
    if ((e = cudaMemcpyAsync(sh.data(), st, sh.size() * sizeof(int), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    for (size_t q = 0; q < sh.size(); ++q)
      if (sh[q] >= 0) {
        *fail_layer = st_layer[q];
        return cudaSuccess;
      }
  }

  // ================= phase 3: re-solve [domain t, separator t] chains in place
  {
    SweepWork W;
    std::vector<int> fails;
    if (nfull > 0) {
      if ((e = sweep(0, nfull, s2 + 1, W, fails))) return e;
      if ((*fail_layer = first_fail(fails, 0)) >= 0) return cudaSuccess;
    }
    if (nfull < T) {
      if ((e = sweep(T - 1, 1, tc + 1, W, fails))) return e;
      if ((*fail_layer = first_fail(fails, T - 1)) >= 0) return cudaSuccess;
    }
  }
  // couplings between separator t-1 and the first layer x0 of chain t
  for (int t = 1; t < T; ++t) {
    const int x0 = P.count[t] > 0 ? P.first[t] : P.sep[t];
    const int sp = P.sep[t - 1];
    const double2* Y = P.count[t] > 0 ? M_(GRD, t) : M_(GR, t);
    // G[x0,-1] = -Y A[x0,-1] G[s,0] ;  G[s,+1] = -G[s,0] A[s,+1] Y
    if ((e = mm(b, 1, 1.0, blk(Y, b), blk(aslot(x0, -1), b), 0.0, blk(Tm(0), b), s))) return e;
    if ((e = mm(b, 1, -1.0, blk(Tm(0), b), blk(gslot(sp, 0), b), 0.0, blk(gslot(x0, -1), b), s))) return e;
    if ((e = mm(b, 1, 1.0, blk(gslot(sp, 0), b), blk(aslot(sp, 1), b), 0.0, blk(Tm(1), b), s))) return e;
    if ((e = mm(b, 1, -1.0, blk(Tm(1), b), blk(Y, b), 0.0, blk(gslot(sp, 1), b), s))) return e;
  }
  return cudaSuccess;
}

size_t ddrgf_scratch_bytes(int l, int b, int s2) {
  const Part P = partition(l, s2);
  const long long bb = (long long)b * b;
  return (size_t(8) * P.T + 8 + 2 * size_t(P.T)) * bb * sizeof(double2) + 4096;
}

// Logical kernel counts of the reference ddrgf for this plan (walks the same
// descriptors as ddrgf_level, ddrgf.hpp:344-412; equals predict_ddrgf_counters,
// cost_model.hpp:137-154, for evenly dividing plans).
void ddrgf_reference_counters(long long l, const int* s2_levels, int n_levels, long long out[3]) {
  long long g = 0, lu = 0, rs = 0;
  long long lk = l;
  for (int lev = 0; lev < n_levels; ++lev) {
    const Part P = partition(int(lk), s2_levels[lev]);
    for (int t = 0; t < P.T; ++t) {
      const long long c = P.count[t];
      if (c == 0) continue;
      // rgf_extended(c): 4(c-1) + extra, c LU, 3c-2 GETRS
      g += 4 * (c - 1) + (c <= 2 ? 0 : (c - 1) * (c - 2));
      lu += c;
      rs += 3 * c - 2;
      g += 4 * c + 4;            // couplings v/w + schur_update (ddrgf.hpp:127-138)
      g += 4 * c;                // compute_y (ddrgf.hpp:142-160)
      g += 4;                    // collect_separator_cols (ddrgf.hpp:177-194)
      g += 2 * (3 * c - 2);      // diag_update_right over the tridiagonal (ddrgf.hpp:198-208)
    }
    lk = P.T;
  }
  g += 4 * (lk - 1);
  lu += lk;
  rs += 3 * lk - 2;
  out[0] = g;
  out[1] = lu;
  out[2] = rs;
}

}  // namespace bbsi_gpu

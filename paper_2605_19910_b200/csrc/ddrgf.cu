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
#include <cstdio>
#include <cstdlib>
#include <mutex>
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

// ---------------------------------------------------------------------------------
// The three phases operate on a rank-local slice of the band (whole chains
// [domain t, separator t] for tasks t0..t1-1, layers [first(t0), sep(t1-1)]) plus a
// per-task interface packet of PK b x b blocks; only packets cross ranks.
//   packet[t] = { a, b, c, e (fake-lead corners), A[s,s], A[s,l], A[l,s], A[s,s+1], A[x0,x0-1] }
//   phase-2 output[t] = { Sigma^L on the chain's first block, Sigma^R on its separator,
//                         Y_t = right-connected G at the chain's first layer x0,
//                         gL_t = left-connected G at separator t }
enum { PA, PB, PC, PE, PASS, PASL, PALS, PASN, PAX0, PK };
enum { OSL, OSR, OY, OGL, NOUT };

namespace {

struct Local {
  const double2* A;  // local band, layer 0 = global layer L0
  double2* G;
  int L0;
  long long bb;
  const double2* aslot(int a, int off) const { return A + ((long long)(a - L0) * 3 + off + 1) * bb; }
  double2* gslot(int a, int off) const { return G + ((long long)(a - L0) * 3 + off + 1) * bb; }
};

// RGF sweeps over the chains of tasks [t, t+nt) (same length len), in place in G. The
// two-ended sweep is used in both phases: phase 1 reads its multipliers in the
// two-ended layout (sweep_is_two_ended), phase 3 only needs the chains' G.
cudaError_t chain_sweeps(const Local& X, const Part& P, int s2, int t, int nt, int len, int b, const int* n_true,
                         SweepWork& W, int* fail_layer, cudaStream_t s, bool two_ended = false) {
  W = SweepWork{};
  W.l = len;
  W.w = 1;
  W.bs = b;
  W.batch = nt;
  W.G = X.gslot(P.first[t], -1);
  W.g_bstride = (long long)(s2 + 1) * 3 * X.bb;
  W.groups = default_groups(nt, b);
  W.two_ended = two_ended && two_ended_default();
  void* sc = arena_get(6, sweep_scratch_bytes(len, 1, b, nt, W.groups, W.two_ended));
  if (!sc) return cudaErrorMemoryAllocation;
  sweep_carve(W, sc);
  std::vector<int> ntr(len, b);
  for (int j = 0; j < len; ++j) ntr[j] = n_true ? n_true[P.first[t] + j] : b;
  cudaError_t e = rgf_sweeps(W, ntr.data(), s);
  if (e) return e;
  std::vector<int> fails;
  if ((e = collect_failures(W, fails, s))) return e;
  for (int q = 0; q < nt; ++q)
    if (fails[q] >= 0) {
      *fail_layer = P.first[t + q] + fails[q];
      break;
    }
  return cudaSuccess;
}

// groups of equal-length consecutive tasks inside [t0, t1): only the global trailing
// task can be shorter than s2
template <class F>
cudaError_t for_task_runs(const Part& P, int s2, int t0, int t1, F&& f) {
  int t = t0;
  while (t < t1) {
    int u = t;
    while (u < t1 && P.count[u] == P.count[t]) ++u;
    cudaError_t e = f(t, u - t, P.count[t]);
    if (e) return e;
    t = u;
  }
  return cudaSuccess;
}

// max |z| over each of nblk b x b blocks at base + off[k] (one CTA per block)
__global__ void block_maxabs_kernel(const double2* base, const long long* off, long long n2, double* out) {
  const double2* m = base + off[blockIdx.x];
  double v = 0.0;
  for (long long i = threadIdx.x; i < n2; i += blockDim.x) v = fmax(v, hypot(m[i].x, m[i].y));
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) out[blockIdx.x] = v;
  }
}

// Fake-lead strength per task: gamma0 * max|A[s_t, s_t]| (the separator block, which
// both phase 1 (locally) and phase 2 (from the packet) can see), so the fake leads
// scale with the matrix and DDRGF stays scale-invariant like the reference.
cudaError_t task_gammas(const double2* base, const std::vector<long long>& offs, int b, double gamma0,
                        std::vector<double>& out, cudaStream_t s) {
  const int n = int(offs.size());
  out.assign(n, gamma0);
  if (n == 0) return cudaSuccess;
  char* buf = static_cast<char*>(arena_get(18, size_t(n) * (sizeof(long long) + sizeof(double)) + 256));
  if (!buf) return cudaErrorMemoryAllocation;
  long long* doff = reinterpret_cast<long long*>(buf);
  double* dmx = reinterpret_cast<double*>(buf + ((size_t(n) * sizeof(long long) + 255) & ~size_t(255)));
  cudaError_t e;
  if ((e = cudaMemcpyAsync(doff, offs.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, s))) return e;
  {
    ProfScope prof(s, PROF_BAND, 0.0, 16.0 * b * b * n);
    block_maxabs_kernel<<<n, 256, 0, s>>>(base, doff, (long long)b * b, dmx);
    if ((e = cudaGetLastError())) return e;
  }
  std::vector<double> mx(n);
  if ((e = cudaMemcpyAsync(mx.data(), dmx, sizeof(double) * n, cudaMemcpyDeviceToHost, s))) return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  for (int k = 0; k < n; ++k) out[k] = gamma0 * (mx[k] > 0.0 ? mx[k] : 1.0);
  return cudaSuccess;
}

}  // namespace

double ddrgf_gamma0() {
  if (const char* e = getenv("BBSI_DDRGF_GAMMA")) {
    const double v = atof(e);
    if (v > 0.0) return v;
  }
  return 1.0;
}

size_t ddrgf_packet_bytes(int ntask, int b) { return size_t(ntask) * PK * b * b * sizeof(double2); }
size_t ddrgf_phase2_out_bytes(int ntask, int b) { return size_t(ntask) * NOUT * b * b * sizeof(double2); }

// Phase 1: fake-lead corners of the local domains + interface A blocks -> packet.
cudaError_t ddrgf_phase1(const double2* A, double2* G, int l, int b, const int* n_true, int s2, double gamma0, int t0,
                         int t1, double2* packet, int* fail_layer, cudaStream_t s) {
  *fail_layer = -1;
  const Part P = partition(l, s2);
  if (t0 < 0 || t1 > P.T || t0 >= t1) return cudaErrorInvalidValue;
  const long long bb = (long long)b * b;
  Local X{A, G, P.first[t0], bb};
  const int L1 = P.sep[t1 - 1] + 1;
  const size_t band_b = sizeof(double2) * size_t(L1 - X.L0) * 3 * bb;
  cudaError_t e;
  std::vector<long long> offs;
  for (int t = t0; t < t1; ++t) offs.push_back(X.aslot(P.sep[t], 0) - A);
  std::vector<double> gam;
  if ((e = task_gammas(A, offs, b, gamma0, gam, s))) return e;
  if ((e = cudaMemcpyAsync(G, A, band_b, cudaMemcpyDeviceToDevice, s))) return e;
  for (int t = t0; t < t1; ++t) {
    if (P.count[t] == 0) continue;
    const double2 ig = make_double2(0.0, gam[t - t0]);  // -Sigma0 = +i*gamma_t
    if ((e = diag_add(X.gslot(P.first[t], 0), 0, b, 1, ig, s))) return e;
    if ((e = diag_add(X.gslot(P.first[t] + P.count[t] - 1, 0), 0, b, 1, ig, s))) return e;
  }
  auto pk = [&](int t, int k) { return packet + ((size_t)(t - t0) * PK + k) * bb; };
  double2* rc = static_cast<double2*>(arena_get(12, 2 * size_t(t1 - t0) * bb * sizeof(double2)));
  if (!rc) return cudaErrorMemoryAllocation;
  e = for_task_runs(P, s2, t0, t1, [&](int t, int nt, int len) -> cudaError_t {
    if (len == 0) return cudaSuccess;
    SweepWork W;
    cudaError_t e2 = chain_sweeps(X, P, s2, t, nt, len, b, n_true, W, fail_layer, s, true);
    if (e2 || *fail_layer >= 0) return e2;
    // a = G[f,f], e = G[l,l]; b = G[f,l], c = G[l,f] by the first row / column chains
    const long long gs = W.g_bstride;
    const size_t pkstride = PK * bb * sizeof(double2);
    if ((e2 = cudaMemcpy2DAsync(pk(t, PA), pkstride, X.gslot(P.first[t], 0), gs * sizeof(double2),
                                bb * sizeof(double2), nt, cudaMemcpyDeviceToDevice, s)))
      return e2;
    if ((e2 = cudaMemcpy2DAsync(pk(t, PE), pkstride, X.gslot(P.first[t] + len - 1, 0), gs * sizeof(double2),
                                bb * sizeof(double2), nt, cudaMemcpyDeviceToDevice, s)))
      return e2;
    if (len == 1) {
      if ((e2 = cudaMemcpy2DAsync(pk(t, PB), pkstride, pk(t, PA), pkstride, bb * sizeof(double2), nt,
                                  cudaMemcpyDeviceToDevice, s)))
        return e2;
      return cudaMemcpy2DAsync(pk(t, PC), pkstride, pk(t, PA), pkstride, bb * sizeof(double2), nt,
                               cudaMemcpyDeviceToDevice, s);
    }
    double2* pr = rc;
    double2* pc = rc + (size_t)nt * bb;
    if (sweep_is_two_ended(W)) {
      // two-ended multipliers (m = len/2): from G[m,m],
      //   b: G[i, m] = -lm[i] G[i+1, m] (i = m-1 .. 0), then G[0, a] = -G[0, a-1] um[a] (a = m+1 ..)
      //   c: G[a, m] = -lm[a] G[a-1, m] (a = m+1 ..),   then G[l-1, i] = -G[l-1, i+1] um[i] (i = m-1 .. 0)
      const int m = len / 2, nr = len - 1 - m;
      const double2* v = X.gslot(P.first[t] + m, 0);
      const double2* u = v;
      long long vs = gs, us = gs;
      auto mult = [&](const double2* base, int j) { return blk(base + (long long)j * bb, b, (long long)W.l * bb); };
      for (int st = 0; st < len - 1; ++st) {
        const bool to_out = ((len - 2 - st) % 2) == 0;  // the last step lands in the packet
        double2* r_nxt = to_out ? pk(t, PB) : pr;
        double2* c_nxt = to_out ? pk(t, PC) : pc;
        const long long nstride = to_out ? PK * bb : bb;
        ZGemmGroup g{};
        g.batch = nt;
        g.bs = 64;
        g.nprob = 2;
        ZGemmProblem& p0 = g.prob[0];
        p0.M = p0.N = p0.K = b;
        p0.alpha = make_double2(-1.0, 0.0);
        p0.beta = make_double2(0.0, 0.0);
        ZGemmProblem& p1 = g.prob[1];
        p1 = p0;
        if (st < m) {
          p0.A = mult(W.LM, m - 1 - st);
          p0.B = blk(v, b, vs);
        } else {
          p0.A = blk(v, b, vs);
          p0.B = mult(W.UM, m + 1 + (st - m));
        }
        p0.C = p0.D = blk(r_nxt, b, nstride);
        if (st < nr) {
          p1.A = mult(W.LM, m + 1 + st);
          p1.B = blk(u, b, us);
        } else {
          p1.A = blk(u, b, us);
          p1.B = mult(W.UM, m - 1 - (st - nr));
        }
        p1.C = p1.D = blk(c_nxt, b, nstride);
        if ((e2 = zgemm_grouped(g, s))) return e2;
        v = r_nxt;
        u = c_nxt;
        vs = us = nstride;
      }
      return cudaSuccess;
    }
    const double2* r_cur = pk(t, PA);
    const double2* c_cur = pk(t, PA);
    long long rstride = PK * bb, cstride = PK * bb;
    for (int j = 1; j < len; ++j) {
      const bool to_out = ((len - 1 - j) % 2) == 0;  // the last step lands in the packet
      double2* r_nxt = to_out ? pk(t, PB) : pr;
      double2* c_nxt = to_out ? pk(t, PC) : pc;
      const long long nstride = to_out ? PK * bb : bb;
      ZGemmGroup g{};
      g.batch = nt;
      g.bs = 64;
      g.nprob = 2;
      ZGemmProblem& p0 = g.prob[0];
      p0.M = p0.N = p0.K = b;
      p0.alpha = make_double2(-1.0, 0.0);
      p0.beta = make_double2(0.0, 0.0);
      p0.A = blk(r_cur, b, rstride);
      p0.B = blk(W.UM + (long long)j * bb, b, (long long)W.l * bb);
      p0.C = p0.D = blk(r_nxt, b, nstride);
      ZGemmProblem& p1 = g.prob[1];
      p1 = p0;
      p1.A = blk(W.LM + (long long)j * bb, b, (long long)W.l * bb);
      p1.B = blk(c_cur, b, cstride);
      p1.C = p1.D = blk(c_nxt, b, nstride);
      if ((e2 = zgemm_grouped(g, s))) return e2;
      r_cur = r_nxt;
      c_cur = c_nxt;
      rstride = cstride = nstride;
    }
    return cudaSuccess;
  });
  if (e || *fail_layer >= 0) return e;
  // interface A blocks (out-of-band slots are zero in the band)
  auto cp = [&](double2* d, const double2* x) {
    return cudaMemcpyAsync(d, x, bb * sizeof(double2), cudaMemcpyDeviceToDevice, s);
  };
  for (int t = t0; t < t1; ++t) {
    const int sp = P.sep[t], cnt = P.count[t];
    const int x0 = cnt > 0 ? P.first[t] : sp;
    if ((e = cp(pk(t, PASS), X.aslot(sp, 0)))) return e;
    if ((e = cp(pk(t, PASL), X.aslot(sp, -1)))) return e;
    if (cnt > 0) {
      if ((e = cp(pk(t, PALS), X.aslot(sp - 1, 1)))) return e;
    } else if ((e = cudaMemsetAsync(pk(t, PALS), 0, bb * sizeof(double2), s))) {
      return e;
    }
    if ((e = cp(pk(t, PASN), X.aslot(sp, 1)))) return e;
    if ((e = cp(pk(t, PAX0), X.aslot(x0, -1)))) return e;
    if (cnt == 0) {  // no corners: keep them zero
      for (int k = PA; k <= PE; ++k)
        if ((e = cudaMemsetAsync(pk(t, k), 0, bb * sizeof(double2), s))) return e;
    }
  }
  return cudaSuccess;
}

// Phase 2 (redundant on every rank): the interface system over all T tasks from the
// gathered packets, single level or nested over the plan's later levels
// (csrc/ddrgf_iface.cu). The right-connected recursions run on a side stream.
namespace {
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream() {
  thread_local std::vector<SideStream> per_dev;  // per host thread: concurrent callers do not share it
  int dev = 0;
  cudaGetDevice(&dev);
  if (int(per_dev.size()) <= dev) per_dev.resize(dev + 1);
  SideStream& x = per_dev[dev];
  if (!x.s) {
    cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
  }
  return x;
}
}  // namespace

cudaError_t ddrgf_phase2(const double2* packets, int l, int b, const int* n_true, int s2, double gamma0, double2* out,
                         int* fail_layer, cudaStream_t s, const int* levels_above, int n_above) {
  *fail_layer = -1;
  const Part P = partition(l, s2);
  const int T = P.T;
  const long long bb = (long long)b * b;
  cudaError_t e;
  std::vector<long long> offs;
  for (int t = 0; t < T; ++t) offs.push_back((long long)((size_t)t * PK + PASS) * bb);
  std::vector<double> gam;
  if ((e = task_gammas(packets, offs, b, gamma0, gam, s))) return e;
  std::vector<char> empty(T);
  std::vector<int> first(T), last(T), sep(T);
  for (int t = 0; t < T; ++t) {
    empty[t] = P.count[t] == 0;
    first[t] = P.count[t] > 0 ? P.first[t] : P.sep[t];
    last[t] = P.count[t] > 0 ? P.first[t] + P.count[t] - 1 : P.sep[t];
    sep[t] = P.sep[t];
  }
  if (T > 0 && empty[0]) return cudaErrorInvalidValue;  // task 0 always has interior layers
  const int cap = iface_status_cap(T);
  int* st = static_cast<int*>(arena_get(8, sizeof(int) * size_t(cap)));
  if (!st) return cudaErrorMemoryAllocation;
  SideStream& side = side_stream();
  std::vector<int> st_layer;
  e = iface_solve(packets, out, T, b, n_true ? n_true[0] : b, gam, empty, first, last, sep, levels_above, n_above, st,
                  cap, st_layer, s, side.s, side.fork, side.join);
  if (e) return e;
  std::vector<int> sh(st_layer.size());
  if (!sh.empty() && (e = cudaMemcpyAsync(sh.data(), st, sh.size() * sizeof(int), cudaMemcpyDeviceToHost, s)))
    return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  for (size_t q = 0; q < sh.size(); ++q)
    if (sh[q] >= 0) {
      *fail_layer = st_layer[q];
      break;
    }
  return cudaSuccess;
}

// Phase 3: re-solve the local chains with the exact boundary self-energies (in place).
cudaError_t ddrgf_phase3(const double2* A, double2* G, int l, int b, const int* n_true, int s2, int t0, int t1,
                         const double2* out, int* fail_layer, cudaStream_t s) {
  *fail_layer = -1;
  const Part P = partition(l, s2);
  const int T = P.T;
  const long long bb = (long long)b * b;
  Local X{A, G, P.first[t0], bb};
  const int L1 = P.sep[t1 - 1] + 1;
  auto o = [&](int t, int k) { return out + ((size_t)t * NOUT + k) * bb; };
  const double2 m1 = make_double2(-1.0, 0.0);
  cudaError_t e;
  if ((e = cudaMemcpyAsync(G, A, sizeof(double2) * size_t(L1 - X.L0) * 3 * bb, cudaMemcpyDeviceToDevice, s))) return e;
  for (int t = t0; t < t1; ++t) {
    const int x0 = P.count[t] > 0 ? P.first[t] : P.sep[t];
    if (t > 0 && (e = axpy(X.gslot(x0, 0), o(t, OSL), bb, m1, s))) return e;
    if (t < T - 1 && (e = axpy(X.gslot(P.sep[t], 0), o(t, OSR), bb, m1, s))) return e;
  }
  return for_task_runs(P, s2, t0, t1, [&](int t, int nt, int len) -> cudaError_t {
    SweepWork W;
    return chain_sweeps(X, P, s2, t, nt, len + 1, b, n_true, W, fail_layer, s, true);
  });
}

// The couplings between chains, each made consistent with the chain whose row of A*G
// it closes: G[x0_t, s_{t-1}] (column s_{t-1}: row s_{t-1} of chain t-1, solved with
// Sigma^R = A[s,x0] Y_t A[x0,s]) = -Y_t A[x0,s] G[s,s]; G[s_t, x0_{t+1}] (column x0_{t+1}:
// chain t+1, solved with Sigma^L = A[x0,s] gL_t A[s,x0]) = -gL_t A[s,x0] G[x0,x0]. Both use
// the neighbour chain's diagonal block from phase 3; at a rank boundary that block comes
// from the neighbour rank (prev_sep_g = G[s_{t0-1}, s_{t0-1}], next_x0_g = G[x0_{t1},
// x0_{t1}]; null where there is no neighbour).
cudaError_t ddrgf_couplings(const double2* A, double2* G, int l, int b, int s2, int t0, int t1, const double2* out,
                            const double2* prev_sep_g, const double2* next_x0_g, cudaStream_t s) {
  const Part P = partition(l, s2);
  const int T = P.T;
  const long long bb = (long long)b * b;
  Local X{A, G, P.first[t0], bb};
  auto o = [&](int t, int k) { return out + ((size_t)t * NOUT + k) * bb; };
  auto x0_of = [&](int t) { return P.count[t] > 0 ? P.first[t] : P.sep[t]; };
  double2* tmp = static_cast<double2*>(arena_get(14, bb * sizeof(double2)));
  if (!tmp) return cudaErrorMemoryAllocation;
  cudaError_t e;
  for (int t = t0; t < t1; ++t) {
    const int x0 = x0_of(t);
    if (t > 0) {
      const double2* gss = t == t0 ? prev_sep_g : X.gslot(P.sep[t - 1], 0);
      if (!gss) return cudaErrorInvalidValue;
      if ((e = mm(b, 1, 1.0, blk(o(t, OY), b), blk(X.aslot(x0, -1), b), 0.0, blk(tmp, b), s))) return e;
      if ((e = mm(b, 1, -1.0, blk(tmp, b), blk(gss, b), 0.0, blk(X.gslot(x0, -1), b), s))) return e;
    }
    if (t < T - 1) {
      const int sp = P.sep[t];
      const double2* gxx = t == t1 - 1 ? next_x0_g : X.gslot(x0_of(t + 1), 0);
      if (!gxx) return cudaErrorInvalidValue;
      if ((e = mm(b, 1, 1.0, blk(o(t, OGL), b), blk(X.aslot(sp, 1), b), 0.0, blk(tmp, b), s))) return e;
      if ((e = mm(b, 1, -1.0, blk(tmp, b), blk(gxx, b), 0.0, blk(X.gslot(sp, 1), b), s))) return e;
    }
  }
  return cudaSuccess;
}

// This rank's two boundary diagonal blocks after phase 3 (the halo its neighbours'
// couplings need): halo[0] = G[x0_{t0}, x0_{t0}], halo[1] = G[s_{t1-1}, s_{t1-1}].
cudaError_t ddrgf_halo(const double2* G, int l, int b, int s2, int t0, int t1, double2* halo, cudaStream_t s) {
  const Part P = partition(l, s2);
  const long long bb = (long long)b * b;
  const int L0 = P.first[t0];
  const int x0 = P.count[t0] > 0 ? P.first[t0] : P.sep[t0];
  cudaError_t e = cudaMemcpyAsync(halo, G + ((long long)(x0 - L0) * 3 + 1) * bb, bb * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, s);
  if (e) return e;
  return cudaMemcpyAsync(halo + bb, G + ((long long)(P.sep[t1 - 1] - L0) * 3 + 1) * bb, bb * sizeof(double2),
                         cudaMemcpyDeviceToDevice, s);
}

std::vector<std::pair<int, int>> ddrgf_rank_ranges(int n_tasks, int nranks) {
  std::vector<std::pair<int, int>> r;
  const int base = n_tasks / nranks, extra = n_tasks % nranks;
  int t = 0;
  for (int k = 0; k < nranks; ++k) {
    const int n = base + (k < extra ? 1 : 0);
    r.emplace_back(t, t + n);
    t += n;
  }
  return r;
}

// One rank of the domain-sharded DDRGF; `exchange` is the packet all-gather (NCCL across
// GPUs, identity on one), `halo_exchange` the neighbours' boundary blocks.
cudaError_t ddrgf_rank(const double2* A_loc, double2* G_loc, int l, int b, const int* n_true, int s2, int t0, int t1,
                       double gamma0, const DdrgfExchange& x, void* scratch, size_t scratch_bytes, int* fail_layer,
                       cudaStream_t s, const int* levels_above, int n_above) {
  *fail_layer = -1;
  const Part P = partition(l, s2);
  const int T = P.T;
  const long long bb = (long long)b * b;
  if (scratch_bytes < ddrgf_packet_bytes(T, b) + ddrgf_phase2_out_bytes(T, b) + 4 * bb * sizeof(double2))
    return cudaErrorMemoryAllocation;
  double2* packets = static_cast<double2*>(scratch);          // [T][PK] (own range at t0)
  double2* out = packets + (size_t)T * PK * bb;                // [T][NOUT]
  double2* halo = out + (size_t)T * NOUT * bb;                 // [2] own, [2] neighbours' (prev last, next first)
  cudaError_t e;
  int fl = -1;
  // BBSI_DDRGF_TRACE=1: device time of each phase on stderr
  const bool trace = getenv("BBSI_DDRGF_TRACE") != nullptr;
  cudaEvent_t ev[6] = {};
  auto mark = [&](int i) {
    if (!trace) return;
    cudaEventCreate(&ev[i]);
    cudaEventRecord(ev[i], s);
  };
  struct Report {
    bool on;
    cudaEvent_t* ev;
    ~Report() {
      if (!on || !ev[0]) return;
      const char* names[5] = {"phase 1", "packet exchange", "phase 2", "phase 3", "halo + couplings"};
      cudaEventSynchronize(ev[5] ? ev[5] : ev[0]);
      for (int i = 0; i < 5; ++i) {
        if (!ev[i] || !ev[i + 1]) continue;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
        fprintf(stderr, "[ddrgf] %-17s %9.3f ms\n", names[i], ms);
      }
      for (int i = 0; i < 6; ++i)
        if (ev[i]) cudaEventDestroy(ev[i]);
    }
  } report{trace, ev};
  mark(0);
  e = ddrgf_phase1(A_loc, G_loc, l, b, n_true, s2, gamma0, t0, t1, packets + (size_t)t0 * PK * bb, &fl, s);
  mark(1);
  if (e) return e;
  int any = fl;
  if ((e = x.packets(packets, t0, t1, fl, &any, s))) return e;
  if (any >= 0) {
    *fail_layer = any;
    return cudaSuccess;
  }
  mark(2);
  if ((e = ddrgf_phase2(packets, l, b, n_true, s2, gamma0, out, &fl, s, levels_above, n_above)) || fl >= 0) {
    *fail_layer = fl;
    return e;
  }
  mark(3);
  if ((e = ddrgf_phase3(A_loc, G_loc, l, b, n_true, s2, t0, t1, out, &fl, s))) return e;
  mark(4);
  if ((e = ddrgf_halo(G_loc, l, b, s2, t0, t1, halo, s))) return e;
  any = fl;
  if ((e = x.halo(halo, halo + 2 * bb, fl, &any, s))) return e;  // also agrees on phase-3 failures
  if (any >= 0) {
    *fail_layer = any;
    return cudaSuccess;
  }
  e = ddrgf_couplings(A_loc, G_loc, l, b, s2, t0, t1, out, t0 > 0 ? halo + 2 * bb : nullptr,
                      t1 < T ? halo + 3 * bb : nullptr, s);
  mark(5);
  return e;
}

cudaError_t ddrgf_device(const double2* A, double2* G, int l, int b, const int* n_true, int s2, double gamma0,
                         void* scratch, size_t scratch_bytes, int* fail_layer, cudaStream_t s, const int* levels_above,
                         int n_above) {
  DdrgfExchange local;  // one rank: nothing to exchange
  local.packets = [](double2*, int, int, int fl, int* any, cudaStream_t) {
    *any = fl;
    return cudaSuccess;
  };
  local.halo = [](const double2*, double2*, int fl, int* any, cudaStream_t) {
    *any = fl;
    return cudaSuccess;
  };
  const int T = partition(l, s2).T;
  return ddrgf_rank(A, G, l, b, n_true, s2, 0, T, gamma0, local, scratch, scratch_bytes, fail_layer, s, levels_above,
                    n_above);
}

int ddrgf_num_tasks(int l, int s2) { return partition(l, s2).T; }

size_t ddrgf_scratch_bytes(int l, int b, int s2) {
  const int T = partition(l, s2).T;
  return ddrgf_packet_bytes(T, b) + ddrgf_phase2_out_bytes(T, b) + 4 * size_t(b) * b * sizeof(double2) + 4096;
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

// Batched inversion of bs x bs complex128 blocks: blocked Gauss-Jordan elimination
// with partial (row) pivoting, split into a per-matrix panel kernel and two
// grouped DMMA GEMM launches per panel, so the O(n^3) part runs on every SM.
//
// Replaces, per Schur pivot, the reference's lu_factor + invert pair
// (kernels.hpp:140-160 zgetrf with the negligible-pivot test, kernels.hpp:192-195
// zgetrs against the identity); solve_left / solve_right (kernels.hpp:163-189)
// become plain GEMMs with the explicit inverse.
//
// Block sweep on the panel K = [k, k+nb) with pivot rows P (after interchanges):
//   M[P,K] <- Pinv = (L_P U)^{-1},  M[P,C] <- Pinv M[P,C],
//   M[R,K] <- -M[R,K] Pinv,         M[R,C] <- M[R,C] - M[R,K] Pinv M[P,C].
// Per panel:
//   gj_panel (1 CTA / matrix): tall-panel LU with partial pivoting of rows k..n-1
//     (|re|+|im| pivot choice, first index on ties, as izamax in zgetrf); the
//     row interchanges become a row map; Pinv by warp-parallel triangular solves;
//     Wz = M[:,K] in post-interchange row order with -I on the pivot rows;
//     Vs = M[P,:] with the identity in the K columns.
//   GEMM 1: V = Pinv Vs                                  (nb x n)
//   GEMM 2: Next = Cur[rowmap] (0 on rows P / cols K) - Wz V  (n x n, all SMs)
// Cur/Next ping-pong between the input block and two scratch matrices; the last
// panel's GEMM writes into the input block with the column map that undoes the
// interchanges (X = Y P), so no separate un-pivoting pass exists.
// The U diagonal is tested against eps * n * max|A| (|.| = hypot), the reference
// threshold (kernels.hpp:149-158); status[] gets the first failing column or -1.
#include <cfloat>
#include <climits>

#include "internal.h"

namespace bbsi_gpu {

namespace {

constexpr int PT = 1024;  // panel kernel threads

struct GjScratch {
  int* rowmap;    // [batch][n]
  int* colmap;    // [batch][n]
  int* piv;       // [batch][n]
  double* tol;    // [batch]
  double2* wz;    // [batch][n*nb]   (col-major, ld n)
  double2* pinv;  // [batch][nb*nb]  (col-major, ld nb)
  double2* vs;    // [batch][nb*n]   (col-major, ld nb)
  double2* vbuf;  // [batch][nb*n]
  double2* s0;    // [batch][n*n]
  double2* s1;    // [batch][n*n]
};

int pick_nb(int n) { return (size_t(n) * 32 * sizeof(double2) <= 200 * 1024) ? 32 : 16; }

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t carve(GjScratch& s, void* base, int n, int nb, int batch) {
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p ? p + off : nullptr;
    off = align256(off + bytes);
    return r;
  };
  s.rowmap = reinterpret_cast<int*>(take(sizeof(int) * size_t(batch) * n));
  s.colmap = reinterpret_cast<int*>(take(sizeof(int) * size_t(batch) * n));
  s.piv = reinterpret_cast<int*>(take(sizeof(int) * size_t(batch) * n));
  s.tol = reinterpret_cast<double*>(take(sizeof(double) * size_t(batch)));
  s.wz = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * n * nb));
  s.pinv = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * nb * nb));
  s.vs = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * nb * n));
  s.vbuf = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * nb * n));
  s.s0 = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * n * n));
  s.s1 = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * n * n));
  return off;
}

__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

template <int NB>
__global__ void __launch_bounds__(PT, 1)
    gj_panel_kernel(const double2* __restrict__ cur0, long long ld, long long bstride, int n, int n_true, int k,
                    GjScratch S, int* __restrict__ status) {
  extern __shared__ __align__(16) double2 pn[];  // NB columns x rows (ld = rows + 1), panel in smem
  __shared__ double cand_v[PT / 32];
  __shared__ int cand_i[PT / 32];
  __shared__ int s_piv[NB];   // pivot row (panel-local) chosen at step j
  __shared__ int s_src[NB];   // source row (global index) of pivot row k+j after interchanges
  __shared__ int s_fail;
  __shared__ double s_tol;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const double2* __restrict__ cur = cur0 + (long long)b * bstride;
  const int rows = n - k;
  const int ldp = rows + 1;
  int* __restrict__ rowmap = S.rowmap + (long long)b * n;
  int* __restrict__ piv = S.piv + (long long)b * n;

  if (tid == 0) s_fail = INT_MAX;
  if (k == 0) {  // threshold eps * n * max|A| over the true block (kernels.hpp:149-158)
    double mx = 0.0;
    if (tid < n_true) {
#pragma unroll 1
      for (int c0 = 0; c0 < n_true; c0 += 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = (c0 + u < n_true) ? cur[(long long)(c0 + u) * ld + tid] : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < 8; ++u) mx = fmax(mx, hypot(v[u].x, v[u].y));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) cand_v[warp] = mx;
    __syncthreads();
    if (warp == 0) {
      double m = cand_v[lane];
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) {
        s_tol = DBL_EPSILON * double(n_true) * m;
        S.tol[b] = s_tol;
        status[b] = -1;
      }
    }
  } else if (tid == 0) {
    s_tol = S.tol[b];
  }

  // ---- load the panel (rows k..n-1, columns k..k+NB-1 of Cur), flat and coalesced
  for (int base = tid; base < NB * rows; base += 4 * PT) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = base + u * PT;
      v[u] = idx < NB * rows ? cur[(long long)(k + idx / rows) * ld + k + idx % rows] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = base + u * PT;
      if (idx < NB * rows) pn[(idx / rows) * ldp + idx % rows] = v[u];
    }
  }
  __syncthreads();
  const double tol = s_tol;

  // warp-level argmax of |re|+|im| over the rows this thread offers; lane 0 publishes
  auto publish = [&](double bv, int bi) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(bv, bi, v2, i2);
    }
    if (lane == 0) {
      cand_v[warp] = bv;
      cand_i[warp] = bi;
    }
  };
  {  // candidates for column 0
    const int r = tid;
    const bool on = r < rows;
    publish(on ? cabs1(pn[r]) : -1.0, on ? r : INT_MAX);
  }

  // ---- right-looking LU with partial pivoting, 3 barriers per column:
  //   B1 candidates visible -> warp 0 resolves the pivot, swaps rows j/p and
  //      publishes 1/pivot
  //   B2 -> multipliers of column j
  //   B3 -> rank-1 update of the trailing block by a 256 (rows) x 4 (column
  //         groups) thread grid; column j+1's updaters publish its candidates.
  __shared__ double2 s_inv;
  const int nwarp_rows = (rows + 31) / 32 < 8 ? (rows + 31) / 32 : 8;
  const int rt = tid & 255, cg = tid >> 8;
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    __syncthreads();  // B1
    if (warp == 0) {
      double v = lane < nwarp_rows ? cand_v[lane] : -2.0;
      int p = lane < nwarp_rows ? cand_i[lane] : INT_MAX;
#pragma unroll
      for (int o = 4; o; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        int i2 = __shfl_xor_sync(0xffffffffu, p, o);
        argmax_merge(v, p, v2, i2);
      }
      p = __shfl_sync(0xffffffffu, p, 0);  // lanes 0..7 hold the reduction; broadcast
      if (p == INT_MAX) p = j;              // empty / NaN column: keep row j
      if (p != j && lane < NB) {
        const double2 x = pn[lane * ldp + j];
        pn[lane * ldp + j] = pn[lane * ldp + p];
        pn[lane * ldp + p] = x;
      }
      __syncwarp();
      if (lane == 0) {
        s_piv[j] = p;
        piv[k + j] = k + p;
        const double2 pv = pn[j * ldp + j];  // pivot value, now in row j
        if (k + j < n_true && hypot(pv.x, pv.y) <= tol) s_fail = min(s_fail, k + j);
        s_inv = crcp(pv);
      }
    }
    __syncthreads();  // B2
    const double2 inv = s_inv;
    for (int r = j + 1 + tid; r < rows; r += PT) pn[j * ldp + r] = cmul(pn[j * ldp + r], inv);
    __syncthreads();  // B3
    double bv = -1.0;
    int bi = INT_MAX;
    for (int r = j + 1 + rt; r < rows; r += 256) {
      const double2 l = pn[j * ldp + r];
      for (int c = j + 1 + cg; c < NB; c += 4) {
        const double2 u = pn[c * ldp + j];
        double2 x = pn[c * ldp + r];
        x.x = fma(-l.x, u.x, fma(l.y, u.y, x.x));
        x.y = fma(-l.x, u.y, fma(-l.y, u.x, x.y));
        pn[c * ldp + r] = x;
        if (c == j + 1) {
          const double a = cabs1(x);
          if (a > bv) {
            bv = a;
            bi = r;
          }
        }
      }
    }
    if (j + 1 < NB && warp < nwarp_rows) publish(bv, bi);
  }
  __syncthreads();

  // ---- row map of the interchanges (new row r holds old row src(r))
  for (int r = tid; r < n; r += PT) {
    int src = r;
    if (r >= k) {
#pragma unroll
      for (int j = NB - 1; j >= 0; --j) {
        const int p = k + s_piv[j];
        if (src == k + j)
          src = p;
        else if (src == p)
          src = k + j;
      }
    }
    rowmap[r] = src;
    if (r >= k && r < k + NB) s_src[r - k] = src;
  }

  // ---- Pinv = U^{-1} L^{-1} of the pivot block (panel rows 0..NB-1): one warp per column
  if (warp < NB) {
    double2* __restrict__ pinv = S.pinv + (long long)b * NB * NB;
    const bool act = lane < NB;
    const int row = act ? lane : 0;
    const int c = warp;
    double2 t = make_double2(lane == c ? 1.0 : 0.0, 0.0);
#pragma unroll
    for (int q = 0; q < NB; ++q) {  // forward: unit lower L
      const double2 lq = pn[q * ldp + row];
      double2 tq;
      tq.x = __shfl_sync(0xffffffffu, t.x, q);
      tq.y = __shfl_sync(0xffffffffu, t.y, q);
      if (act && lane > q) t = csub(t, cmul(lq, tq));
    }
    const double2 dinv = crcp(pn[row * ldp + row]);
#pragma unroll
    for (int q = NB - 1; q >= 0; --q) {  // backward: upper U
      const double2 uq = pn[q * ldp + row];
      if (lane == q) t = cmul(t, dinv);
      double2 xq;
      xq.x = __shfl_sync(0xffffffffu, t.x, q);
      xq.y = __shfl_sync(0xffffffffu, t.y, q);
      if (lane < q) t = csub(t, cmul(uq, xq));
    }
    if (act) pinv[c * NB + lane] = t;
  }
  __syncthreads();

  // ---- Wz (n x NB, ld n): current M[:,K] in post-interchange order, -I on pivot rows
  {
    double2* __restrict__ wz = S.wz + (long long)b * n * NB;
    for (int base = tid; base < n * NB; base += 4 * PT) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * PT;
        const int r = idx % n, c = idx / n;
        if (idx < n * NB)
          v[u] = (r >= k && r < k + NB) ? make_double2(r - k == c ? -1.0 : 0.0, 0.0)
                                        : cur[(long long)(k + c) * ld + rowmap[r]];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * PT;
        if (idx < n * NB) wz[idx] = v[u];
      }
    }
  }
  // ---- Vs (NB x n, ld NB): pivot rows of M after interchanges, identity in columns K
  {
    double2* __restrict__ vs = S.vs + (long long)b * NB * n;
    for (int base = tid; base < n * NB; base += 4 * PT) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * PT;
        const int j = idx % NB, col = idx / NB;
        if (idx < n * NB)
          v[u] = (col >= k && col < k + NB) ? make_double2(col - k == j ? 1.0 : 0.0, 0.0)
                                            : cur[(long long)col * ld + s_src[j]];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * PT;
        if (idx < n * NB) vs[idx] = v[u];
      }
    }
  }
  __syncthreads();
  if (tid == 0 && s_fail != INT_MAX && status[b] < 0) status[b] = s_fail;
}

// After the last panel: column map that undoes the interchanges. With
// X[:, c] = Y[:, q[c]] (q from the column swaps j = n-1 .. 0), the GEMM scatters
// column c' of Y to colmap[c'] = q^{-1}(c').
__global__ void build_colmap_kernel(const int* __restrict__ piv0, int* __restrict__ colmap0, int n) {
  extern __shared__ int sq[];
  const int b = blockIdx.x;
  const int* piv = piv0 + (long long)b * n;
  int* colmap = colmap0 + (long long)b * n;
  int* spiv = sq + n;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    sq[c] = c;
    spiv[c] = piv[c];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = n - 1; j >= 0; --j) {
      const int p = spiv[j];
      const int t = sq[j];
      sq[j] = sq[p];
      sq[p] = t;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) colmap[sq[c]] = c;
}

}  // namespace

size_t zinv_scratch_bytes(int n, int batch) {
  GjScratch s;
  return carve(s, nullptr, n, pick_nb(n), batch) + 256;
}

cudaError_t zinv_batched(double2* M, long long ld, long long bstride, int n, int n_true, int batch, void* scratch,
                         int* status, cudaStream_t stream) {
  if (n % 64 || n_true > n || n_true < 1) return cudaErrorInvalidValue;
  if (batch == 0) return cudaSuccess;
  const int nb = pick_nb(n);
  GjScratch S;
  carve(S, scratch, n, nb, batch);
  const size_t smem = size_t(nb) * (n + 1) * sizeof(double2);
  static size_t attr16 = 0, attr32 = 0;
  cudaError_t e;
  if (nb == 32 && smem > attr32) {
    if ((e = cudaFuncSetAttribute(gj_panel_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))))
      return e;
    attr32 = smem;
  }
  if (nb == 16 && smem > attr16) {
    if ((e = cudaFuncSetAttribute(gj_panel_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))))
      return e;
    attr16 = smem;
  }
  const long long nn = (long long)n * n;
  const int npan = n / nb;
  for (int pi = 0; pi < npan; ++pi) {
    const int k = pi * nb;
    const bool last = pi == npan - 1;
    const double2* cur = pi == 0 ? M : (pi % 2 ? S.s0 : S.s1);
    const long long cld = pi == 0 ? ld : n, cbs = pi == 0 ? bstride : nn;
    double2* nxt = last ? M : (pi % 2 ? S.s1 : S.s0);
    const long long nld = last ? ld : n, nbs = last ? bstride : nn;
    {
      ProfScope prof(stream, PROF_INV, 8.0 * double(n) * nb * nb * batch, 16.0 * (3.0 * n * nb) * batch);
      if (nb == 32)
        gj_panel_kernel<32><<<batch, PT, smem, stream>>>(cur, cld, cbs, n, n_true, k, S, status);
      else
        gj_panel_kernel<16><<<batch, PT, smem, stream>>>(cur, cld, cbs, n, n_true, k, S, status);
      if ((e = cudaGetLastError())) return e;
      if (last) {
        build_colmap_kernel<<<batch, 256, 2 * n * sizeof(int), stream>>>(S.piv, S.colmap, n);
        if ((e = cudaGetLastError())) return e;
      }
    }
    // GEMM 1: V = Pinv * Vs
    ZGemmGroup g{};
    g.batch = batch;
    g.bs = 64;
    g.nprob = 1;
    ZGemmProblem& p1 = g.prob[0];
    p1.M = nb;
    p1.N = n;
    p1.K = nb;
    p1.alpha = make_double2(1.0, 0.0);
    p1.beta = make_double2(0.0, 0.0);
    p1.A = ZOp{S.pinv, nb, 64, 64LL * nb, (long long)nb * nb};
    p1.B = ZOp{S.vs, nb, 64, 64LL * nb, (long long)nb * n};
    p1.D = ZOp{S.vbuf, nb, 64, 64LL * nb, (long long)nb * n};
    p1.C = p1.D;
    if ((e = zgemm_grouped(g, stream))) return e;
    // GEMM 2: Next = Cur[rowmap] (zero on rows P, cols K) - Wz * V
    ZGemmProblem& p2 = g.prob[0];
    p2 = ZGemmProblem{};
    p2.M = n;
    p2.N = n;
    p2.K = nb;
    p2.alpha = make_double2(-1.0, 0.0);
    p2.beta = make_double2(1.0, 0.0);
    p2.A = ZOp{S.wz, n, 64, 64LL * n, (long long)n * nb};
    p2.B = ZOp{S.vbuf, nb, 64, 64LL * nb, (long long)nb * n};
    p2.C = ZOp{cur, cld, 64, 64LL * cld, cbs};
    p2.D = ZOp{nxt, nld, 64, 64LL * nld, nbs};
    p2.rowmap = S.rowmap;
    p2.colmap = last ? S.colmap : nullptr;
    p2.map_bstride = n;
    p2.zr0 = k;
    p2.zr1 = k + nb;
    p2.zc0 = k;
    p2.zc1 = k + nb;
    if ((e = zgemm_grouped(g, stream))) return e;
  }
  return cudaSuccess;
}

}  // namespace bbsi_gpu

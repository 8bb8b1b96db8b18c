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
//   M[P,K] <- Pinv = (L_P U)^{-1},  M[P,C] <- Pinv M[P,C]  (both = V below),
//   M[R,K] <- -M[R,K] Pinv,         M[R,C] <- M[R,C] - M[R,K] Pinv M[P,C].
// Per panel:
//   gj_panel (1 CTA / matrix): tall-panel LU with partial pivoting of rows k..n-1
//     (|re|+|im| pivot choice, first index on ties, as izamax in zgetrf); the
//     row interchanges become a row map; Wz = M[:,K] in post-interchange row
//     order with -I on the pivot rows; V = U^{-1} L^{-1} M[P,:] (identity in the
//     K columns, so V[:,K] = Pinv) by triangular solves, one column per thread.
//   GEMM:  Next = Cur[rowmap] (0 on rows P / cols K) - Wz V  (n x n, all SMs)
// Cur/Next ping-pong between the input block and two scratch matrices; the last
// panel's GEMM writes into the input block with the column map that undoes the
// interchanges (X = Y P), so no separate un-pivoting pass exists.
// The U diagonal is tested against eps * n * max|A| (|.| = hypot), the reference
// threshold (kernels.hpp:149-158); status[] gets the first failing column or -1.
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "internal.h"

namespace bbsi_gpu {
__device__ long long g_zinv_dbg[64];

namespace {

constexpr int PT = 256;  // panel kernel threads

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

// Panel width. 16 is the default: blocked Gauss-Jordan loses accuracy with the
// pivot-block width (numpy emulation on config 3, E = 0.145: RGF vs reference
// 2.2e-10 at nb = 32, 1.4e-10 at nb = 16, 1.3e-10 unblocked; the reference's own
// 1/2-ulp input-noise floor there is 1.1-1.4e-10). BBSI_GJ_NB=32 trades accuracy
// for fewer, wider panels.
int pick_nb(int n) {
  static int forced = [] {
    const char* e = getenv("BBSI_GJ_NB");
    return e ? atoi(e) : 0;
  }();
  if (forced == 32 && size_t(n) * 32 * sizeof(double2) <= 200 * 1024) return 32;
  return 16;
}

int panel_priority() {
  static int p = [] {
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return 0;
    const char* e = getenv("BBSI_PANEL_PRIORITY");
    return (e && atoi(e) == 0) ? lo : hi;  // hi = greatest priority (numerically lowest)
  }();
  return p;
}

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
  __shared__ double cand_v[2][PT / 32];
  __shared__ int cand_i[2][PT / 32];
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

#ifdef BBSI_ZINV_DEBUG
#define DBG(i) if (b == 0 && tid == 0 && k == 32) g_zinv_dbg[i] = clock64();
#else
#define DBG(i)
#endif
  DBG(0)
  if (tid == 0) s_fail = INT_MAX;
  if (k == 0) {  // threshold eps * n * max|A| over the true block (kernels.hpp:149-158)
    double mx = 0.0;
    for (int r = tid; r < n_true; r += PT) {
#pragma unroll 1
      for (int c0 = 0; c0 < n_true; c0 += 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = (c0 + u < n_true) ? cur[(long long)(c0 + u) * ld + r] : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < 8; ++u) mx = fmax(mx, hypot(v[u].x, v[u].y));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) cand_v[1][warp] = mx;
    __syncthreads();
    if (warp == 0) {
      double m = cand_v[1][lane];
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
  DBG(1)
  const double tol = s_tol;

  // Row interchanges are applied to a logical->physical row permutation (double
  // buffered by parity) instead of moving data, so one barrier per column
  // suffices: every warp resolves the pivot redundantly from the published
  // per-warp candidates (also double buffered).
  int* perm = reinterpret_cast<int*>(pn + NB * ldp);  // [2][rows]
  for (int r = tid; r < rows; r += PT) perm[r] = r;

  // warp-level argmax of |re|+|im| over the rows this thread offers; lane 0 publishes
  auto publish = [&](int par, double bv, int bi) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(bv, bi, v2, i2);
    }
    if (lane == 0) {
      cand_v[par][warp] = bv;
      cand_i[par][warp] = bi;
    }
  };
  {  // candidates for column 0
    double bv = -1.0;
    int bi = INT_MAX;
    for (int r = tid; r < rows; r += PT) {
      const double a = cabs1(pn[r]);
      if (a > bv) {
        bv = a;
        bi = r;
      }
    }
    publish(0, bv, bi);
  }

  const int nwarp_rows = (rows + 31) / 32 < PT / 32 ? (rows + 31) / 32 : PT / 32;
  // The register-resident variant measured slower than the shared-memory one on
  // B200 (4.6k vs 3.9k cycles per column at n = 256); kept for experiments.
  constexpr bool kRegPath = false;
  const bool reg = kRegPath && rows <= PT;
  if (reg) {
    // ---- register path: physical row t is owned by thread t and kept in
    // registers; interchanges only relabel logical indices. Per column: one
    // barrier; each warp's best candidate lane publishes its whole row, every
    // warp resolves the pivot redundantly and reads the winning row.
    __shared__ double2 cand_row[2][PT / 32][NB];
    __shared__ int cand_ph[2][PT / 32];
    const int t = tid;
    const bool own = t < rows;
    double2 a[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) a[c] = own ? pn[c * ldp + t] : make_double2(0.0, 0.0);
    int mylog = t;
    auto publish_reg = [&](int par, double bv, int blog) {
      int bph = t;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        int i2 = __shfl_xor_sync(0xffffffffu, blog, o);
        int p2 = __shfl_xor_sync(0xffffffffu, bph, o);
        if (v2 > bv || (v2 == bv && i2 < blog)) {
          bv = v2;
          blog = i2;
          bph = p2;
        }
      }
      if (bph == t && blog != INT_MAX) {
#pragma unroll
        for (int c = 0; c < NB; ++c) cand_row[par][warp][c] = a[c];
      }
      if (lane == 0) {
        cand_v[par][warp] = bv;
        cand_i[par][warp] = blog;
        cand_ph[par][warp] = bph;
      }
    };
    __syncthreads();  // everyone has consumed the smem-path candidates of column 0
    publish_reg(0, own ? cabs1(a[0]) : -1.0, own ? t : INT_MAX);
#pragma unroll 1
    for (int j = 0; j < NB; ++j) {
      const int par = j & 1;
      __syncthreads();  // the only barrier of step j
      if (j < 8) { DBG(10 + j) }
      double v = lane < nwarp_rows ? cand_v[par][lane] : -2.0;
      int p = lane < nwarp_rows ? cand_i[par][lane] : INT_MAX;
      int ws = lane;
#pragma unroll
      for (int o = 4; o; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        int i2 = __shfl_xor_sync(0xffffffffu, p, o);
        int w2 = __shfl_xor_sync(0xffffffffu, ws, o);
        if (v2 > v || (v2 == v && i2 < p)) {
          v = v2;
          p = i2;
          ws = w2;
        }
      }
      p = __shfl_sync(0xffffffffu, p, 0);
      ws = __shfl_sync(0xffffffffu, ws, 0);
      if (j == 1) { DBG(20) }
      int phj = -1;
      const bool has = p != INT_MAX;
      if (!has) p = j;  // no candidate (NaN column): keep logical row j in place
      else phj = cand_ph[par][ws];
      const double2 (&prow)[NB] = cand_row[par][has ? ws : 0];
      if (tid == 0) {
        s_piv[j] = p;
        piv[k + j] = k + p;
      }
      // logical interchange j <-> p
      int nl = mylog;
      if (mylog == j) nl = p;
      if (t == phj) nl = j;
      if (phj < 0 && mylog == j) nl = j;
      mylog = nl;
      const double2 inv = has ? crcp_fast(prow[j]) : make_double2(0.0, 0.0);
      if (j == 1) { DBG(22) }
      const bool upd = own && mylog > j && has;
      double bv = -1.0;
#define GJR_CHUNK(C0)                                                          \
  {                                                                            \
    double2 aj = a[C0];                                                        \
    _Pragma("unroll") for (int c = (C0) + 1; c < (C0) + 8 && c < NB; ++c)     \
      if (c == j) aj = a[c];                                                   \
    const double2 l = cmul(aj, inv);                                           \
    const double2 lz = upd ? l : make_double2(0.0, 0.0);                       \
    _Pragma("unroll") for (int c = (C0); c < NB; ++c) {                        \
      const double2 lc = (c > j) ? lz : make_double2(0.0, 0.0);               \
      const double2 pc = prow[c];                                              \
      double2 x = a[c];                                                        \
      x.x = fma(-lc.x, pc.x, fma(lc.y, pc.y, x.x));                            \
      x.y = fma(-lc.x, pc.y, fma(-lc.y, pc.x, x.y));                           \
      if (c == j + 1) bv = cabs1(x);                                           \
      a[c] = (upd && c == j) ? l : x;                                          \
    }                                                                          \
  }
      const int ch = j >> 3;
      if (ch == 0) {
        GJR_CHUNK(0)
      } else if (ch == 1) {
        GJR_CHUNK(8 < NB ? 8 : 0)
      } else if (ch == 2) {
        GJR_CHUNK(16 < NB ? 16 : 0)
      } else {
        GJR_CHUNK(24 < NB ? 24 : 0)
      }
#undef GJR_CHUNK
      if (j == 1) { DBG(23) }
      if (j + 1 < NB) publish_reg(par ^ 1, (own && mylog > j) ? bv : -1.0, (own && mylog > j) ? mylog : INT_MAX);
      if (j == 1) { DBG(24) }
    }
    __syncthreads();
    int* fp = perm + (NB & 1) * rows;
    if (own) {
#pragma unroll
      for (int c = 0; c < NB; ++c) pn[c * ldp + t] = a[c];
      fp[mylog] = t;
    }
  } else {
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const int par = j & 1;
    __syncthreads();  // the only barrier of step j
    if (j < 8) { DBG(10 + j) }
    double v = lane < nwarp_rows ? cand_v[par][lane] : -2.0;
    int p = lane < nwarp_rows ? cand_i[par][lane] : INT_MAX;
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      int i2 = __shfl_xor_sync(0xffffffffu, p, o);
      argmax_merge(v, p, v2, i2);
    }
    p = __shfl_sync(0xffffffffu, p, 0);
    if (j == 1) { DBG(20) }
    if (p == INT_MAX) p = j;  // empty / NaN column: keep row j
    const int* pold = perm + par * rows;
    int* pnew = perm + (par ^ 1) * rows;
    const int phj = pold[p];  // physical row of the pivot = new logical row j
    const int php = pold[j];  // physical row of old logical row j = new logical row p
    for (int r = tid; r < rows; r += PT) pnew[r] = (r == j) ? phj : ((r == p) ? php : pold[r]);
    if (tid == 0) {
      s_piv[j] = p;
      piv[k + j] = k + p;
    }
    if (j == 1) { DBG(21) }
    const double2 inv = crcp_fast(pn[j * ldp + phj]);
    if (j == 1) { DBG(22) }
    double bv = -1.0;
    int bi = INT_MAX;
    // each logical row r > j is owned by exactly one thread: it scales its
    // multiplier in place and updates its trailing columns in batches of 8
    for (int r = j + 1 + tid; r < rows; r += PT) {
      const int ph = (r == p) ? php : pold[r];
      const double2 l = cmul(pn[j * ldp + ph], inv);
      pn[j * ldp + ph] = l;
#pragma unroll 1
      for (int c0 = j + 1; c0 < NB; c0 += 8) {
        double2 x[8], u[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int c = c0 + i;
          if (c < NB) {
            u[i] = pn[c * ldp + phj];
            x[i] = pn[c * ldp + ph];
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int c = c0 + i;
          if (c < NB) {
            x[i].x = fma(-l.x, u[i].x, fma(l.y, u[i].y, x[i].x));
            x[i].y = fma(-l.x, u[i].y, fma(-l.y, u[i].x, x[i].y));
            pn[c * ldp + ph] = x[i];
          }
        }
        if (c0 == j + 1) {  // column j+1 candidates
          const double a = cabs1(x[0]);
          if (a > bv) {
            bv = a;
            bi = r;
          }
        }
      }
    }
    if (j == 1) { DBG(23) }
    if (j + 1 < NB && warp < nwarp_rows) publish(par ^ 1, bv, bi);
    if (j == 1) { DBG(24) }
  }
  __syncthreads();
  }
  const int* fperm = perm + (NB & 1) * rows;  // final logical -> physical rows
  __syncthreads();
  DBG(2)
  if (tid < NB && k + tid < n_true) {  // negligible-pivot test on the U diagonal
    const double2 d = pn[tid * ldp + fperm[tid]];
    if (hypot(d.x, d.y) <= tol) atomicMin(&s_fail, k + tid);
  }

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

  // 1 / U[j][j] of the pivot block (logical rows 0..NB-1, physical fperm[j])
  __shared__ double2 s_uinv[NB];
  if (tid < NB) s_uinv[tid] = crcp_fast(pn[tid * ldp + fperm[tid]]);
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
  // ---- V (NB x n, ld NB) = U^{-1} L^{-1} Vs, Vs = pivot rows of M after the
  //      interchanges with the identity in columns K (so V[:,K] = (L U)^{-1}).
  //      Triangular solves, one column per thread: backward stable, no explicit
  //      inverse of the pivot block.
  {
    double2* __restrict__ vb = S.vbuf + (long long)b * NB * n;
    for (int col = tid; col < n; col += PT) {
      const bool kc = col >= k && col < k + NB;
      double2 x[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j)
        x[j] = kc ? make_double2(col - k == j ? 1.0 : 0.0, 0.0) : cur[(long long)col * ld + s_src[j]];
#pragma unroll
      for (int j = 1; j < NB; ++j) {  // L (unit lower): x_j -= sum_{q<j} L[j][q] x_q
        const int pj = fperm[j];
#pragma unroll
        for (int q = 0; q < j; ++q) x[j] = csub(x[j], cmul(pn[q * ldp + pj], x[q]));
      }
#pragma unroll
      for (int j = NB - 1; j >= 0; --j) {  // U: x_j = (x_j - sum_{q>j} U[j][q] x_q) / U[j][j]
        const int pj = fperm[j];
#pragma unroll
        for (int q = j + 1; q < NB; ++q) x[j] = csub(x[j], cmul(pn[q * ldp + pj], x[q]));
        x[j] = cmul(x[j], s_uinv[j]);
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) vb[(long long)col * NB + j] = x[j];
    }
  }
  __syncthreads();
  DBG(4)
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

extern "C" int bbsi_debug_zinv(long long* out) { return (int)cudaMemcpyFromSymbol(out, g_zinv_dbg, sizeof(long long) * 64); }

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
  const size_t smem = size_t(nb) * (n + 1) * sizeof(double2) + 2 * size_t(n) * sizeof(int);
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
      // The panel is latency-bound and on the critical path of the sweep: launched at
      // the greatest priority so its CTAs take SMs ahead of queued GEMM tiles of
      // other streams (side-stream groups).
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(batch);
      cfg.blockDim = dim3(PT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributePriority;
      attr[0].val.priority = panel_priority();
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (nb == 32)
        e = cudaLaunchKernelEx(&cfg, gj_panel_kernel<32>, (const double2*)cur, cld, cbs, n, n_true, k, S, status);
      else
        e = cudaLaunchKernelEx(&cfg, gj_panel_kernel<16>, (const double2*)cur, cld, cbs, n, n_true, k, S, status);
      if (e) return e;
      if (last) {
        build_colmap_kernel<<<batch, 256, 2 * n * sizeof(int), stream>>>(S.piv, S.colmap, n);
        if ((e = cudaGetLastError())) return e;
      }
    }
    ZGemmGroup g{};
    g.batch = batch;
    g.bs = 64;
    g.nprob = 1;
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

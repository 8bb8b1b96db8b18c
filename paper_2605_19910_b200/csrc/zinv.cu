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

// BBSI_PANEL_ROWS=0 selects the shared-memory panel kernel everywhere (A/B checks).
bool use_rows_kernel() {
  static bool on = [] {
    const char* e = getenv("BBSI_PANEL_ROWS");
    return !(e && atoi(e) == 0);
  }();
  return on;
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

// Everything after the pivot search, shared by both panel kernels.
//   lu[j][c]  pivot row j (logical): L multipliers for c < j, U for c >= j
//   lmap[r]   panel-local logical row r -> physical (= original) row
//   lpiv[j]   LAPACK-style interchange partner of step j (panel-local)
// Writes rowmap / piv, Wz and V, and the first negligible U-diagonal column.
template <int NB>
__device__ __forceinline__ void panel_tail(const double2* __restrict__ cur, long long ld, int n, int n_true, int k, int b,
                                           const GjScratch& S, int* __restrict__ status, const double2 (*lu)[NB + 1],
                                           const int* lmap, const int* lpiv, double tol, int* s_fail) {
  __shared__ double2 s_uinv[NB];
  __shared__ int s_src[NB];
  const int tid = threadIdx.x;
  int* __restrict__ rowmap = S.rowmap + (long long)b * n;
  if (tid < NB) {
    const double2 d = lu[tid][tid];
    if (k + tid < n_true && hypot(d.x, d.y) <= tol) atomicMin(s_fail, k + tid);  // kernels.hpp:149-158
    s_uinv[tid] = crcp_fast(d);
    S.piv[(long long)b * n + k + tid] = k + lpiv[tid];
  }
  // row map of the interchanges: new row r holds old row rowmap[r]
  for (int r = tid; r < n; r += PT) {
    const int src = r < k ? r : k + lmap[r - k];
    rowmap[r] = src;
    if (r >= k && r < k + NB) s_src[r - k] = src;
  }
  __syncthreads();
  // Wz (n x NB, ld n): current M[:,K] in post-interchange order, -I on the pivot rows
  {
    double2* __restrict__ wz = S.wz + (long long)b * n * NB;
#pragma unroll 1
    for (int c = 0; c < NB; c += 4) {
      for (int r = tid; r < n; r += PT) {
        const bool pr = r >= k && r < k + NB;
        const int src = r < k ? r : k + lmap[r - k];
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = pr ? make_double2(r - k == c + u ? -1.0 : 0.0, 0.0) : cur[(long long)(k + c + u) * ld + src];
#pragma unroll
        for (int u = 0; u < 4; ++u) wz[(long long)(c + u) * n + r] = v[u];
      }
    }
  }
  // V (NB x n, ld NB) = U^{-1} L^{-1} Vs, Vs = pivot rows of M after the interchanges
  // with the identity in columns K (so V[:,K] = (L U)^{-1}); triangular solves, one
  // column per thread (backward stable, no explicit inverse of the pivot block).
  {
    double2* __restrict__ vb = S.vbuf + (long long)b * NB * n;
    for (int col = tid; col < n; col += PT) {
      const bool kc = col >= k && col < k + NB;
      double2 x[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j)
        x[j] = kc ? make_double2(col - k == j ? 1.0 : 0.0, 0.0) : cur[(long long)col * ld + s_src[j]];
#pragma unroll
      for (int j = 1; j < NB; ++j) {  // unit lower L
#pragma unroll
        for (int q = 0; q < j; ++q) x[j] = csub(x[j], cmul(lu[j][q], x[q]));
      }
#pragma unroll
      for (int j = NB - 1; j >= 0; --j) {  // upper U
#pragma unroll
        for (int q = j + 1; q < NB; ++q) x[j] = csub(x[j], cmul(lu[j][q], x[q]));
        x[j] = cmul(x[j], s_uinv[j]);
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) vb[(long long)col * NB + j] = x[j];
    }
  }
  __syncthreads();
  if (tid == 0 && *s_fail != INT_MAX && status[b] < 0) status[b] = *s_fail;
}

// max |a_ij| (hypot) over the true n_true x n_true block -> eps * n_true * max (kernels.hpp:149-158)
__device__ __forceinline__ double panel_threshold(const double2* __restrict__ cur, long long ld, int n_true,
                                                  double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double mx = 0.0;
  for (int r = tid; r < n_true; r += PT) {
#pragma unroll 1
    for (int c0 = 0; c0 < n_true; c0 += 16) {
      double2 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        v[u] = (c0 + u < n_true) ? cur[(long long)(c0 + u) * ld + r] : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 16; ++u) mx = fmax(mx, hypot(v[u].x, v[u].y));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  double m = 0.0;
#pragma unroll
  for (int q = 0; q < PT / 32; ++q) m = fmax(m, red[q]);
  return DBL_EPSILON * double(n_true) * m;
}

template <int NB>
__global__ void __launch_bounds__(PT, 1)
    gj_panel_kernel(const double2* __restrict__ cur0, long long ld, long long bstride, int n, int n_true, int k,
                    GjScratch S, int* __restrict__ status) {
  extern __shared__ __align__(16) double2 pn[];  // NB columns x rows (ld = rows + 1), panel in smem
  __shared__ double cand_v[2][PT / 32];
  __shared__ int cand_i[2][PT / 32];
  __shared__ int s_piv[NB];   // pivot row (panel-local) chosen at step j
  __shared__ int s_fail;
  __shared__ double s_tol;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const double2* __restrict__ cur = cur0 + (long long)b * bstride;
  const int rows = n - k;
  const int ldp = rows + 1;
  int* __restrict__ piv = S.piv + (long long)b * n;

#ifdef BBSI_ZINV_DEBUG
#define DBG(i) if (b == 0 && tid == 0 && k == 32) g_zinv_dbg[i] = clock64();
#else
#define DBG(i)
#endif
  DBG(0)
  if (tid == 0) s_fail = INT_MAX;
  if (k == 0) {
    const double t = panel_threshold(cur, ld, n_true, cand_v[1]);
    if (tid == 0) {
      s_tol = t;
      S.tol[b] = t;
      status[b] = -1;
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
  {
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
  __shared__ double2 s_lu[NB][NB + 1];
  for (int e = tid; e < NB * NB; e += PT) s_lu[e / NB][e % NB] = pn[(e % NB) * ldp + fperm[e / NB]];
  __syncthreads();
  DBG(2)
  panel_tail<NB>(cur, ld, n, n_true, k, b, S, status, s_lu, fperm, s_piv, tol, &s_fail);
}

// Pivot-search key: |re|+|im| truncated to sign, exponent and 11 mantissa bits of
// the double, above the complemented physical row. The unsigned maximum is the
// largest magnitude (lowest row among equal keys), so one warp-wide REDUX.MAX is the
// argmax. The chosen pivot is within a factor 1 - 2^-11 of the column maximum
// (threshold partial pivoting, |l| <= 1.0005).
constexpr int KEY_IB = 10;  // physical rows < 1024
constexpr unsigned KEY_IMASK = (1u << KEY_IB) - 1;
__device__ __forceinline__ unsigned piv_key(double2 v, int ph) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(cabs1(v)) & 0x7fffffffffffffffULL;
  return (unsigned(bits >> (63 - (32 - KEY_IB))) << KEY_IB) | (KEY_IMASK - unsigned(ph));
}

// Register-resident panel (rows <= RPT * PT). Thread t owns physical panel rows
// t + i*PT for good: rows never move, the interchanges only relabel logical row
// numbers, so the elimination never touches shared memory for its own data. Per
// column: one barrier, the pivot resolved from the 8 published warp keys, the
// winning row and its reciprocal read from the winner's warp slot, the update, and
// the next column's warp keys by REDUX.
template <int NB, int RPT>
__global__ void __launch_bounds__(PT, 1)
    gj_panel_rows_kernel(const double2* __restrict__ cur0, long long ld, long long bstride, int n, int n_true, int k,
                         GjScratch S, int* __restrict__ status) {
  __shared__ unsigned cand_k[2][PT / 32];
  __shared__ double2 cand_r[2][PT / 32];
  __shared__ __align__(16) double2 cand_row[2][PT / 32][NB];
  __shared__ double2 s_lu[NB][NB + 1];
  __shared__ int s_map[RPT * PT];
  __shared__ int s_p[NB];
  __shared__ double s_red[PT / 32];
  __shared__ int s_fail;
  __shared__ double s_tol;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const double2* __restrict__ cur = cur0 + (long long)b * bstride;
  const int rows = n - k;

  double2 a[RPT][NB];
  int lg[RPT];
  bool act[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int ph = tid + i * PT;
    act[i] = ph < rows;
    lg[i] = ph;
#pragma unroll
    for (int c = 0; c < NB; ++c) a[i][c] = act[i] ? cur[(long long)(k + c) * ld + k + ph] : make_double2(0.0, 0.0);
  }
  if (tid == 0) s_fail = INT_MAX;
  if (k == 0) {
    const double t = panel_threshold(cur, ld, n_true, s_red);
    if (tid == 0) {
      s_tol = t;
      S.tol[b] = t;
      status[b] = -1;
    }
  } else if (tid == 0) {
    s_tol = S.tol[b];
  }

  // publish this warp's best candidate for column J: key, reciprocal, row (c > J)
  auto publish = [&](int par, int J) {
    unsigned key = 0;
    int wi = 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (act[i]) {
        const unsigned kk = piv_key(a[i][J], tid + i * PT);
        if (kk > key) {
          key = kk;
          wi = i;
        }
      }
    const unsigned wk = __reduce_max_sync(0xffffffffu, key);
    if (lane == 0) cand_k[par][warp] = wk;
    if (wk != 0 && key == wk) {
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (i == wi) {
          cand_r[par][warp] = crcp_fast(a[i][J]);
#pragma unroll
          for (int c = 0; c < NB; ++c)
            if (c > J) cand_row[par][warp][c] = a[i][c];
        }
    }
  };
  publish(0, 0);

  int prev_ph = -1;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int par = j & 1;
    __syncthreads();
    if (j > 0) {  // deferred relabel of step j-1: the old logical row j-1 takes the partner's number
      const int pp = s_p[j - 1];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (lg[i] == j - 1 && tid + i * PT != prev_ph) lg[i] = pp;
    }
    unsigned best = 0;
#pragma unroll
    for (int q = 0; q < PT / 32; ++q) best = max(best, cand_k[par][q]);
    const int phj = int(KEY_IMASK - (best & KEY_IMASK));
    const int qw = (phj % PT) >> 5;
    const double2 rcp = cand_r[par][qw];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (tid + i * PT == phj) {  // this row becomes logical row j
        s_p[j] = lg[i];
        lg[i] = j;
        act[i] = false;
#pragma unroll
        for (int c = 0; c < NB; ++c) s_lu[j][c] = a[i][c];
      }
    }
    double2 l[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      l[i] = act[i] ? cmul(a[i][j], rcp) : make_double2(0.0, 0.0);
      if (act[i]) a[i][j] = l[i];
    }
#pragma unroll
    for (int c = j + 1; c < NB; ++c) {
      const double2 u = cand_row[par][qw][c];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        double2 x = a[i][c];
        x.x = fma(-l[i].x, u.x, fma(l[i].y, u.y, x.x));
        x.y = fma(-l[i].x, u.y, fma(-l[i].y, u.x, x.y));
        a[i][c] = x;
      }
    }
    prev_ph = phj;
    if (j + 1 < NB) publish(par ^ 1, j + 1);
  }
  __syncthreads();
  {
    const int pp = s_p[NB - 1];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int ph = tid + i * PT;
      if (lg[i] == NB - 1 && ph != prev_ph) lg[i] = pp;
      if (ph < rows) s_map[lg[i]] = ph;
    }
  }
  __syncthreads();
  panel_tail<NB>(cur, ld, n, n_true, k, b, S, status, s_lu, s_map, s_p, s_tol, &s_fail);
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
      const int rows = n - k;
      const double2* cc = cur;
      if (use_rows_kernel() && nb == 16 && rows <= PT) {
        cfg.dynamicSmemBytes = 0;
        e = cudaLaunchKernelEx(&cfg, gj_panel_rows_kernel<16, 1>, cc, cld, cbs, n, n_true, k, S, status);
      } else if (use_rows_kernel() && nb == 16 && rows <= 2 * PT) {
        cfg.dynamicSmemBytes = 0;
        e = cudaLaunchKernelEx(&cfg, gj_panel_rows_kernel<16, 2>, cc, cld, cbs, n, n_true, k, S, status);
      } else if (use_rows_kernel() && nb == 32 && rows <= PT) {
        cfg.dynamicSmemBytes = 0;
        e = cudaLaunchKernelEx(&cfg, gj_panel_rows_kernel<32, 1>, cc, cld, cbs, n, n_true, k, S, status);
      } else if (nb == 32) {
        e = cudaLaunchKernelEx(&cfg, gj_panel_kernel<32>, cc, cld, cbs, n, n_true, k, S, status);
      } else {
        e = cudaLaunchKernelEx(&cfg, gj_panel_kernel<16>, cc, cld, cbs, n, n_true, k, S, status);
      }
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

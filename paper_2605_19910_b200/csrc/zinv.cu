// Batched inversion of bs x bs complex128 blocks: blocked Gauss-Jordan elimination
// with partial (row) pivoting, split into a per-matrix panel kernel and one grouped
// DMMA GEMM per panel, so the O(n^3) part runs on every SM.
//
// Replaces, per Schur pivot, the reference's lu_factor + invert pair
// (kernels.hpp:140-160 zgetrf with the negligible-pivot test, kernels.hpp:192-195
// zgetrs against the identity); solve_left / solve_right (kernels.hpp:163-189)
// become plain GEMMs with the explicit inverse.
//
// Rows never move. The interchanges live in a logical -> physical row map
// (lmap); logical rows k..n-1 are the rows not yet used as pivots. Block step on
// the panel K = [k, k+nb) with pivot rows P (physical) and the other rows R:
//   M[P,K] <- Pinv = (L U)^{-1},     M[P,C] <- Pinv M[P,C]
//   M[R,K] <- -M[R,K] Pinv,          M[R,C] <- M[R,C] - M[R,K] Pinv M[P,C]
// i.e. M <- M (0 on rows P / cols K) - Wz V with Wz = M[:,K] (-I on rows P) and
// V = Pinv Vs, Vs = M[P,:] with the identity in columns K.
// Per panel:
//   panel kernel (1 CTA / matrix): tall-panel LU with partial pivoting of the
//     active rows (pivot search on |re|+|im|, as izamax in zgetrf), the new lmap,
//     Wz, Pinv (column solves of the pivot block) and V.
//   GEMM: M <- M[mask] - Wz V, in place (a tile reads and writes only itself).
// The first panel reads the input block and writes the working matrix s0; the last
// one writes back into the input block, scattering rows and columns through lmap:
// with Y the eliminated matrix in physical row order, A^{-1}[i, lmap[c]] =
// Y[lmap[i], c], so no separate un-pivoting pass exists.
// The U diagonal is tested against eps * n * max|A| (|.| = hypot), the reference
// threshold (kernels.hpp:149-158); status[] gets the first failing column or -1.
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "internal.h"

namespace bbsi_gpu {
__device__ long long g_zinv_dbg[64];
#ifdef BBSI_ZINV_DEBUG
#define ZDBG(i)                                                       \
  if (blockIdx.x == 0 && threadIdx.x == 0 && k == 32) g_zinv_dbg[i] = clock64();
#else
#define ZDBG(i)
#endif

namespace {

constexpr int PT = 256;  // panel kernel threads

// Panel width 16. Measured on B200 (config 2 / config 3 E = 0.145): 32 is both slower
// (858 vs 771 ms per step) and less accurate (2.9e-10 vs 1.9e-10 against the
// reference, whose own 1/2-ulp floor there is 1.4e-10); blocked Gauss-Jordan loses
// accuracy with the pivot-block width.
constexpr int kNB = 16;

// Panel kernels (A/B switch BBSI_PANEL): 1 (default) two register-resident panels per
// step with one rank-32 update; 3 one register-resident panel per step; 2 the
// tall-panel shared-memory kernel everywhere. Panels with more than 2*PT active rows
// always use the tall-panel kernel. A compact variant with the rows in shared memory
// and rolled column loops measured slower on B200 (41 k vs 15 k cycles for the 16
// elimination steps at n = 256).
int panel_kind() {
  static int kind = [] {
    const char* e = getenv("BBSI_PANEL");
    const int v = e ? atoi(e) : 1;
    return (v == 2 || v == 3) ? v : 1;
  }();
  return kind;
}

// The panel is latency-bound and on the critical path of the sweep: launched at the
// greatest stream priority so its CTAs take SMs ahead of queued GEMM tiles of the
// other stream group (BBSI_PANEL_PRIORITY=0: lowest).
// Pair kernel: panel 2's pivot rows get their own prefetch buffer when two NB x (n+2)
// staging buffers fit next to the static shared memory (n <= 320).
bool pair_pre2(int n) { return 2 * size_t(kNB) * (n + 2) * sizeof(double2) + 40 * 1024 <= 227 * 1024; }

// V by forming Pinv and the DMMA product Pinv * Vs (default) or by substitution with the
// panel's LU factors (BBSI_GJ_SUBST=1). Measured on B200, config 2: substitution 85 ms of
// panel time per step against 73 ms (561 vs 549 ms per step), so it stays opt-in.
int gj_subst() {
  const char* e = getenv("BBSI_GJ_SUBST");
  return (e && atoi(e) == 1) ? 1 : 0;
}

// Concurrent inversion batches of this host thread (stream groups of the running sweep).
thread_local int t_conc = 1;

// Register-resident Gauss-Jordan panels (gj_rows_kernel, n <= 4 PT): the default;
// BBSI_GJ_ROWS=0 keeps the LU + Pinv pair / tall panels (A/B).
// Largest cluster (CTAs per matrix) gj_rows_kernel may use: BBSI_GJ_ROWS = 0 (never) .. 4 (n <= 1024,
// default). The choice never depends on the batch: the two panel families round differently, and a
// solve must give the same bits however its matrices are grouped into launches (stream groups, ranks).
// (One or two n = 256 matrices on their own are 9 % faster on the LU pair panel, whose tails split over
// 8 CTAs per matrix: B200, config 4 single-energy RGF, 1.45 s against 1.58 s.)
int gj_rows_max_cl(int n, int batch) {
  (void)n;
  (void)batch;
  const char* e = getenv("BBSI_GJ_ROWS");  // read per call: tests compare both in one process
  const int v = e ? atoi(e) : 4;
  return v < 0 ? 0 : (v > 4 ? 4 : v);
}

// CTAs per matrix of the pair panel (BBSI_PANEL_SPLIT, else the largest power of two
// <= 8 that keeps batch x concurrency x split within one wave of the 148 SMs). Only for
// n <= PT (register rows, one row per thread) and at least 16 columns per CTA.
int pair_split(int n, int batch) {
  const char* ev = getenv("BBSI_PANEL_SPLIT");  // read per call: tests compare splits in one process
  const int env = ev ? atoi(ev) : 0;
  if (n > PT) return 1;
  int s = 1;
  if (env >= 1) {
    s = env;
  } else {
    const int dev_sms = 148;
    while (s < 8 && (long long)batch * t_conc * s * 2 <= dev_sms) s *= 2;
  }
  while (s > 1 && (n % s || (n / s) % 16)) s /= 2;
  return s;
}

int panel_priority() {
  static int p = [] {
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return 0;
    const char* e = getenv("BBSI_PANEL_PRIORITY");
    return (e && atoi(e) == 0) ? lo : hi;
  }();
  return p;
}

struct GjScratch {
  int* lmap;      // [batch][n]  logical row -> physical row
  int* rowmask;   // [batch][n]  GEMM C rows: r, or -1 on this panel's pivot rows
  int* rowscat;   // [batch][n]  last panel: physical row -> output row
  int* colmap;    // [batch][n]  last panel: column c -> output column lmap[c]
  unsigned long long* amax;  // [batch]  bits of max |a_ij| over the input block (>= 0: ordered as integers)
  double* piv;    // [batch][n]  |u_jj| of logical column j (tested against the threshold at the end)
  double2* wz;    // [batch][n*nb]  (col-major, ld n)
  double2* vbuf;  // [batch][nb*n]  (col-major, ld nb)
  double2* s0;    // [batch][n*n]   working matrix
  int subst;      // V by per-column LU substitution (1) or Pinv * Vs on DMMA (0)
};

// Matrix b of a launch lives at base + (b % inner) * bstride + (b / inner) * ostride and
// reports into status[(b % inner) + (b / inner) * sostride]: `outer` independent
// batches with one uniform stride each (e.g. the two chains of a two-ended sweep).
struct BatchIdx {
  int inner;
  long long bstride, ostride, sostride;
  __host__ __device__ long long off(int b) const { return (long long)(b % inner) * bstride + (long long)(b / inner) * ostride; }
  __host__ __device__ long long sidx(int b) const { return (long long)(b % inner) + (long long)(b / inner) * sostride; }
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t carve(GjScratch& s, void* base, int n, int nb, int batch) {
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p ? p + off : nullptr;
    off = align256(off + bytes);
    return r;
  };
  s.lmap = reinterpret_cast<int*>(take(sizeof(int) * size_t(batch) * n));
  s.rowmask = reinterpret_cast<int*>(take(sizeof(int) * size_t(batch) * n));
  s.rowscat = reinterpret_cast<int*>(take(sizeof(int) * size_t(batch) * n));
  s.colmap = reinterpret_cast<int*>(take(sizeof(int) * size_t(batch) * n));
  s.amax = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * size_t(batch)));
  s.piv = reinterpret_cast<double*>(take(sizeof(double) * size_t(batch) * n));
  s.wz = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * n * 2 * nb));  // two panels
  s.vbuf = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * 2 * nb * n));
  s.s0 = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(batch) * n * n));
  return off;
}

// Physical row of active-list entry t of the panel at k (the list is lmap[k..n-1]).
__device__ __forceinline__ int active_row(const int* lmap, int k, int t) { return k == 0 ? t : lmap[k + t]; }

// Pinv = U^{-1} L^{-1} of a factored NB x NB pivot block (lu: L \ U, uinv: 1/U_jj).
// Warp w solves columns 2w, 2w+1 of both triangular inverses at once (one row per
// lane, values exchanged by shuffles; the two 16-step chains interleave), then every
// thread forms one entry of the product. Called by the whole CTA; ends synchronised.
template <int NB>
__device__ __forceinline__ void pivot_block_inverse(const double2 (*lu)[NB + 1], const double2* uinv,
                                                    double2 (*pinv)[NB + 1]) {
  static_assert(NB == 16, "the warp-level pivot-block inverse assumes NB = 16 (two columns per warp)");
  __shared__ double2 s_li[NB][NB + 1];
  __shared__ double2 s_ui[NB][NB + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp < NB / 2) {
    const int r = lane & 15, c = 2 * warp + (lane >> 4), base = lane & 16;
    double2 yl = make_double2(r == c ? 1.0 : 0.0, 0.0), yu = yl;
#pragma unroll 1
    for (int j = 0; j < NB; ++j) {
      const int ju = NB - 1 - j;
      double2 tl, tu;
      tl.x = __shfl_sync(0xffffffffu, yl.x, base | (j < NB - 1 ? j : 0));
      tl.y = __shfl_sync(0xffffffffu, yl.y, base | (j < NB - 1 ? j : 0));
      tu.x = __shfl_sync(0xffffffffu, yu.x, base | ju);
      tu.y = __shfl_sync(0xffffffffu, yu.y, base | ju);
      if (j < NB - 1 && r > j) yl = csub(yl, cmul(lu[r][j], tl));  // L yl = e_c, forward step j
      const double2 xj = cmul(tu, uinv[ju]);                        // U yu = e_c, backward step ju
      if (r == ju)
        yu = xj;
      else if (r < ju)
        yu = csub(yu, cmul(lu[r][ju], xj));
    }
    s_li[r][c] = yl;
    s_ui[r][c] = yu;
  }
  __syncthreads();
  for (int e = tid; e < NB * NB; e += PT) {  // Pinv[r][c] = sum_{q >= max(r, c)} Ui[r][q] Li[q][c]
    const int r = e / NB, c = e % NB;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < NB; ++q)
      if (q >= r && q >= c) acc = cfma(s_ui[r][q], s_li[q][c], acc);
    pinv[r][c] = acc;
  }
  __syncthreads();
}

// x <- U^{-1} L^{-1} x for one column held in registers (lu: L \ U of the pivot block in
// shared memory, read as broadcasts; uinv: 1 / U_jj). Right-looking: once x_j is final,
// the updates of the later entries are independent, so the dependent chain is NB deep
// instead of NB^2/2. Replaces forming Pinv (two triangular inverses and their product)
// and the Pinv * Vs product: V = Pinv Vs column by column, and the identity columns of
// Vs give Pinv itself.
// Shared-memory load the compiler may not hoist out of the column loop (the 240 factor
// entries are loop invariant; hoisting them all spills the register file).
__device__ __forceinline__ double2 lds_keep(const double2* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n"
               : "=d"(v.x), "=d"(v.y)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

template <int NB>
__device__ __forceinline__ void lu_solve_col(const double2 (*lu)[NB + 1], const double2* uinv, double2 (&x)[NB]) {
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const double2 xj = make_double2(-x[j].x, -x[j].y);
#pragma unroll
    for (int i = 0; i < NB; ++i)
      if (i > j) x[i] = cfma(lds_keep(&lu[i][j]), xj, x[i]);
  }
#pragma unroll
  for (int jj = 0; jj < NB; ++jj) {
    const int j = NB - 1 - jj;
    x[j] = cmul(x[j], lds_keep(&uinv[j]));
    const double2 xj = make_double2(-x[j].x, -x[j].y);
#pragma unroll
    for (int i = 0; i < NB; ++i)
      if (i < j) x[i] = cfma(lds_keep(&lu[i][j]), xj, x[i]);
  }
}

// V = Pinv Vs on the tensor cores, Vs (NB x n) staged in shared memory with ld svld.
// Each warp takes 8-column tiles (2 x 4 complex m8n8k4 steps, 4 real DMMAs each).
// dst != nullptr: V[j][col] -> dst[col * dld + j]; otherwise V overwrites Vs in place
// (a warp reads all of its tile before writing it).
// Tiles: [t0, t1) (t1 < 0: every tile), plus [x0, x1) when it lies outside that range.
template <int NB>
__device__ __forceinline__ void apply_pinv_dmma(const double2 (*pinv)[NB + 1], double2* sv, int svld, int n,
                                                double2* __restrict__ dst, int dld, int t0 = 0, int t1 = -1,
                                                int x0 = 0, int x1 = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  if (t1 < 0) t1 = n / 8;
  const int nown = t1 - t0, nx = (x1 > x0 && (x0 >= t1 || x1 <= t0)) ? x1 - x0 : 0;
  double2 af[2][NB / 4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ks = 0; ks < NB / 4; ++ks) af[mt][ks] = pinv[mt * 8 + lr][ks * 4 + lc];
  for (int it = warp; it < nown + nx; it += PT / 32) {
    const int nt = it < nown ? t0 + it : x0 + (it - nown);
    double2 bv[NB / 4];
#pragma unroll
    for (int ks = 0; ks < NB / 4; ++ks) bv[ks] = sv[(ks * 4 + lc) * svld + nt * 8 + lr];
    double cr[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, ci[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int ks = 0; ks < NB / 4; ++ks)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double2 av = af[mt][ks];
        dmma884(cr[mt], av.x, bv[ks].x);
        dmma884(cr[mt], -av.y, bv[ks].y);
        dmma884(ci[mt], av.x, bv[ks].y);
        dmma884(ci[mt], av.y, bv[ks].x);
      }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int col = nt * 8 + 2 * lc + q, row = mt * 8 + lr;
        const double2 v = make_double2(cr[mt][q], ci[mt][q]);
        if (dst)
          dst[(long long)col * dld + row] = v;
        else
          sv[row * svld + col] = v;
      }
  }
}

// The negligible-pivot test |u_jj| <= eps * n_true * max|a| (kernels.hpp:149-158) runs
// once, in the last panel kernel: every panel stores |u_jj|, and max |a|^2 over the input
// block comes from the first GJ GEMM, which streams the whole block anyway
// (ZGemmProblem::amax) -- no separate pass over the matrix on the critical path.
__device__ __forceinline__ void final_status(const GjScratch& S, int b, int n, int n_true, int* status) {
  __shared__ int s_first;
  if (threadIdx.x == 0) s_first = INT_MAX;
  __syncthreads();
  const double tol = DBL_EPSILON * double(n_true) * sqrt(__longlong_as_double((long long)S.amax[b]));
  const double* pv = S.piv + (long long)b * n;
  for (int i = threadIdx.x; i < n_true; i += PT)
    if (pv[i] <= tol) atomicMin(&s_first, i);
  __syncthreads();
  if (threadIdx.x == 0) *status = s_first == INT_MAX ? -1 : s_first;
}

// Everything after the pivot search, shared by both panel kernels.
//   lu[j][c]   pivot row j (logical): L multipliers for c < j, U for c >= j
//   lloc[r]    panel-local logical row r -> active-list entry
//   act[t]     active-list entry -> physical row
// Writes lmap, the row mask, Wz, V (and on the last panel the output scatters), and
// the first negligible U-diagonal column.
template <int NB>
__device__ __forceinline__ void panel_tail(const double2* __restrict__ cur, long long ld, int n, int n_true, int k, int b,
                                           bool last, const GjScratch& S, int* __restrict__ status,
                                           const double2 (*lu)[NB + 1], const int* lloc, const int* act,
                                           double2* sv) {
  static_assert(NB == 16, "the warp-level pivot-block inverse assumes NB = 16 (two columns per warp)");
  __shared__ double2 s_uinv[NB];
  __shared__ int s_src[NB];  // physical pivot rows
  __shared__ double2 s_pinv[NB][NB + 1];
  const int tid = threadIdx.x;
  const int rows = n - k;
  int* __restrict__ lmap = S.lmap + (long long)b * n;
  int* __restrict__ rowmask = S.rowmask + (long long)b * n;
  double2* __restrict__ wz = S.wz + (long long)b * n * NB;
  double2* __restrict__ vb = S.vbuf + (long long)b * NB * n;
  if (tid < NB) {
    const double2 d = lu[tid][tid];
    S.piv[(long long)b * n + k + tid] = hypot(d.x, d.y);  // kernels.hpp:149-158, tested at the end
    s_uinv[tid] = crcp_fast(d);
    s_src[tid] = act[lloc[tid]];
  }
  for (int r = tid; r < rows; r += PT) lmap[k + r] = act[lloc[r]];
  ZDBG(3)
  // Wz (n x NB, ld n) = M[:,K] (rows are not permuted: coalesced); pivot rows fixed below
  for (int r = tid; r < n; r += PT) {
    rowmask[r] = r;
    double2 v[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) v[c] = cur[(long long)(k + c) * ld + r];
#pragma unroll
    for (int c = 0; c < NB; ++c) wz[(long long)c * n + r] = v[c];
  }
  __syncthreads();
  ZDBG(4)
  // Vs (pivot rows of M, identity in columns K) of this thread's first column, issued
  // now so the loads overlap the pivot-block inverse
  double2 xpre[NB];
  {
    const bool kc = tid >= k && tid < k + NB;
#pragma unroll
    for (int j = 0; j < NB; ++j)
      xpre[j] = tid >= n ? make_double2(0.0, 0.0)
                         : (kc ? make_double2(tid - k == j ? 1.0 : 0.0, 0.0) : cur[(long long)tid * ld + s_src[j]]);
  }
  for (int e = tid; e < NB * NB; e += PT) {  // pivot rows: -I in Wz, 0 in C
    const int j = e / NB, c = e % NB;
    wz[(long long)c * n + s_src[j]] = make_double2(j == c ? -1.0 : 0.0, 0.0);
    if (c == 0) rowmask[s_src[j]] = -1;
  }
  ZDBG(5)
  if (S.subst) {
    // V = U^{-1} L^{-1} Vs by substitution, one column per thread (xpre: the first one)
    __syncthreads();
    for (int col = tid; col < n; col += PT) {
      double2 x[NB];
      const bool kc = col >= k && col < k + NB;
#pragma unroll
      for (int j = 0; j < NB; ++j)
        x[j] = col == tid ? xpre[j]
                          : (kc ? make_double2(col - k == j ? 1.0 : 0.0, 0.0) : cur[(long long)col * ld + s_src[j]]);
      lu_solve_col<NB>(lu, s_uinv, x);
#pragma unroll
      for (int j = 0; j < NB; ++j) vb[(long long)col * NB + j] = x[j];
    }
    ZDBG(8)
  } else {
    pivot_block_inverse<NB>(lu, s_uinv, s_pinv);
    ZDBG(6)
    if (sv) {
      // V = Pinv Vs on the tensor cores: Vs staged in smem (ld n + 2), each warp takes
      // 8-column tiles, 2 x 4 complex m8n8k4 steps (4 real DMMAs each) per tile.
      const int svld = n + 2;
      for (int col = tid; col < n; col += PT) {
        const bool kc = col >= k && col < k + NB;
  #pragma unroll
        for (int j = 0; j < NB; ++j)
          sv[j * svld + col] = col == tid ? xpre[j]
                                          : (kc ? make_double2(col - k == j ? 1.0 : 0.0, 0.0)
                                                : cur[(long long)col * ld + s_src[j]]);
      }
      __syncthreads();
      ZDBG(7)
      apply_pinv_dmma<NB>(s_pinv, sv, svld, n, vb, NB);
      ZDBG(8)
    } else {
      // V = Pinv Vs, one column per thread (tall panels: no smem left for Vs)
      for (int col = tid; col < n; col += PT) {
        double2 x[NB], acc[NB];
        const bool kc = col >= k && col < k + NB;
  #pragma unroll
        for (int j = 0; j < NB; ++j) {
          x[j] = col == tid ? xpre[j]
                            : (kc ? make_double2(col - k == j ? 1.0 : 0.0, 0.0) : cur[(long long)col * ld + s_src[j]]);
          acc[j] = make_double2(0.0, 0.0);
        }
  #pragma unroll 1
        for (int q = 0; q < NB; ++q) {
          double2 xq = x[0];
  #pragma unroll
          for (int u = 1; u < NB; ++u)
            if (u == q) xq = x[u];
  #pragma unroll
          for (int j = 0; j < NB; ++j) acc[j] = cfma(s_pinv[j][q], xq, acc[j]);
        }
  #pragma unroll
        for (int j = 0; j < NB; ++j) vb[(long long)col * NB + j] = acc[j];
      }
    }
  }
  if (last) {  // output scatters: row lmap[i] -> i, column c -> lmap[c]
    // (gathering the last GEMM's C and Wz rows through lmap instead, so that it writes
    // whole rows in order, measured slower on B200: 101 vs 87 us per launch)
    int* __restrict__ rowscat = S.rowscat + (long long)b * n;
    int* __restrict__ colmap = S.colmap + (long long)b * n;
    for (int i = tid; i < n; i += PT) {
      const int p = lmap[i];
      rowscat[p] = i;
      colmap[i] = p;
    }
  }
  __syncthreads();
  if (last) final_status(S, b, n, n_true, status);
  ZDBG(9)
}

// First panel: reset of the max |a|^2 the first GJ GEMM accumulates.
__device__ __forceinline__ void panel_threshold_once(int k, int b, const GjScratch& S) {
  if (k == 0 && threadIdx.x == 0) S.amax[b] = 0ull;
}

__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

// Shared-memory panel for tall panels (more than 2*PT active rows): the panel lives
// in smem, interchanges go through a double-buffered logical -> entry permutation
// (one barrier per column, every warp resolves the pivot from the published
// per-warp candidates).
template <int NB>
__global__ void __launch_bounds__(PT, 1)
    gj_panel_kernel(const double2* __restrict__ cur0, long long ld, long long bstride, int n, int n_true, int k, int last,
                    GjScratch S, int* __restrict__ status0, BatchIdx bi) {
  extern __shared__ __align__(16) double2 pn[];  // NB columns x rows (ld = rows + 1), then perm[2][rows], act[rows]
  __shared__ double cand_v[2][PT / 32];
  __shared__ int cand_i[2][PT / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const double2* __restrict__ cur = cur0 + (k == 0 ? bi.off(b) : (long long)b * bstride);
  int* __restrict__ status = status0 + bi.sidx(b);
  const int rows = n - k;
  const int ldp = rows + 1;
  int* perm = reinterpret_cast<int*>(pn + NB * ldp);  // [2][rows]
  int* act = perm + 2 * rows;                          // [rows]
  const int* lmapg = S.lmap + (long long)b * n;

  for (int r = tid; r < rows; r += PT) {
    act[r] = active_row(lmapg, k, r);
    perm[r] = r;
  }
  panel_threshold_once(k, b, S);
  __syncthreads();
  for (int r = tid; r < rows; r += PT) {
    const int ph = act[r];
    double2 v[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) v[c] = cur[(long long)(k + c) * ld + ph];
#pragma unroll
    for (int c = 0; c < NB; ++c) pn[c * ldp + r] = v[c];
  }
  __syncthreads();

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
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const int par = j & 1;
    __syncthreads();  // the only barrier of step j
    double v = lane < nwarp_rows ? cand_v[par][lane] : -2.0;
    int p = lane < nwarp_rows ? cand_i[par][lane] : INT_MAX;
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      int i2 = __shfl_xor_sync(0xffffffffu, p, o);
      argmax_merge(v, p, v2, i2);
    }
    p = __shfl_sync(0xffffffffu, p, 0);
    if (p == INT_MAX) p = j;  // empty / NaN column: keep row j
    const int* pold = perm + par * rows;
    int* pnew = perm + (par ^ 1) * rows;
    const int phj = pold[p];  // entry of the pivot = new logical row j
    const int php = pold[j];  // entry of old logical row j = new logical row p
    for (int r = tid; r < rows; r += PT) pnew[r] = (r == j) ? phj : ((r == p) ? php : pold[r]);
    const double2 inv = crcp_fast(pn[j * ldp + phj]);
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
    if (j + 1 < NB && warp < nwarp_rows) publish(par ^ 1, bv, bi);
  }
  __syncthreads();
  const int* fperm = perm + (NB & 1) * rows;  // final logical -> entry
  __shared__ double2 s_lu[NB][NB + 1];
  for (int e = tid; e < NB * NB; e += PT) s_lu[e / NB][e % NB] = pn[(e % NB) * ldp + fperm[e / NB]];
  __syncthreads();
  panel_tail<NB>(cur, ld, n, n_true, k, b, last != 0, S, status, s_lu, fperm, act, nullptr);
}

// Pivot-search key: |re|+|im| truncated to sign, exponent and 11 mantissa bits of
// the double, above the complemented active-list entry. The unsigned maximum is the
// largest magnitude (lowest entry among equal keys), so one warp-wide REDUX.MAX is
// the argmax. The chosen pivot is within a factor 1 - 2^-11 of the column maximum
// (threshold partial pivoting, |l| <= 1.0005).
constexpr int KEY_IB = 10;  // active-list entries < 1024
constexpr unsigned KEY_IMASK = (1u << KEY_IB) - 1;
__device__ __forceinline__ unsigned piv_key(double2 v, int t) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(cabs1(v)) & 0x7fffffffffffffffULL;
  return (unsigned(bits >> (63 - (32 - KEY_IB))) << KEY_IB) | (KEY_IMASK - unsigned(t));
}

// Shared memory of the register-resident panel LU.
template <int NB, int RPT>
struct PanelSmem {
  unsigned cand_k[2][PT / 32];
  double2 cand_r[2][PT / 32];
  __align__(16) double2 cand_row[2][PT / 32][NB];
  double2 lu[NB][NB + 1];  // pivot rows (logical order): L \ U
  int map[RPT * PT];       // panel-local logical row -> active-list entry
  int act[RPT * PT];       // active-list entry -> physical row
  int p[NB];               // interchange partner of step j (logical)
};

// Tall-panel LU with partial pivoting of register-resident rows (at most RPT * PT).
// Thread t owns active-list entries t + i*PT for good: the interchanges only relabel
// logical row numbers, so the elimination never touches shared memory for its own
// data. Per column: one barrier, the pivot resolved from the 8 published warp keys,
// the winning row and its reciprocal read from the winner's warp slot, column j+1
// updated first so its REDUX pivot search overlaps the rest of the update.
// Ends synchronised with sm.lu / sm.map complete.
template <int NB, int RPT>
__device__ __forceinline__ void panel_lu_regs(double2 (&a)[RPT][NB], int rows, PanelSmem<NB, RPT>& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int lg[RPT];
  bool act[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    act[i] = tid + i * PT < rows;
    lg[i] = tid + i * PT;
  }
  // this warp's best candidate for column J: its key (lane 0), and from the winning
  // lane the reciprocal now and the row (c > J) once the row is fully updated
  auto publish_key = [&](int par, int J, int& wi) -> bool {
    unsigned key = 0;
    wi = 0;
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
    if (lane == 0) sm.cand_k[par][warp] = wk;
    const bool win = wk != 0 && key == wk;
    if (win) {
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (i == wi) sm.cand_r[par][warp] = crcp_fast(a[i][J]);
    }
    return win;
  };
  auto publish_row = [&](int par, int J, int wi) {
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i == wi) {
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c > J) sm.cand_row[par][warp][c] = a[i][c];
      }
  };
  {
    int wi;
    if (publish_key(0, 0, wi)) publish_row(0, 0, wi);
  }
  int prev_t = -1;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int par = j & 1;
    __syncthreads();
    if (j > 0) {  // deferred relabel of step j-1: the old logical row j-1 takes the partner's number
      const int pp = sm.p[j - 1];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (lg[i] == j - 1 && tid + i * PT != prev_t) lg[i] = pp;
    }
    unsigned best = 0;
#pragma unroll
    for (int q = 0; q < PT / 32; ++q) best = max(best, sm.cand_k[par][q]);
    const int tj = int(KEY_IMASK - (best & KEY_IMASK));
    const int qw = (tj % PT) >> 5;
    const double2 rcp = sm.cand_r[par][qw];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (tid + i * PT == tj) {  // this row becomes logical row j
        sm.p[j] = lg[i];
        lg[i] = j;
        act[i] = false;
#pragma unroll
        for (int c = 0; c < NB; ++c) sm.lu[j][c] = a[i][c];
      }
    }
    double2 l[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      l[i] = act[i] ? cmul(a[i][j], rcp) : make_double2(0.0, 0.0);
      if (act[i]) a[i][j] = l[i];
    }
    auto update = [&](int c) {
      const double2 u = sm.cand_row[par][qw][c];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        double2 x = a[i][c];
        x.x = fma(-l[i].x, u.x, fma(l[i].y, u.y, x.x));
        x.y = fma(-l[i].x, u.y, fma(-l[i].y, u.x, x.y));
        a[i][c] = x;
      }
    };
    prev_t = tj;
    if (j + 1 < NB) {
      update(j + 1);
      int wi;
      const bool win = publish_key(par ^ 1, j + 1, wi);
#pragma unroll
      for (int c = j + 2; c < NB; ++c) update(c);
      if (win) publish_row(par ^ 1, j + 1, wi);
    }
  }
  __syncthreads();
  {
    const int pp = sm.p[NB - 1];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int t = tid + i * PT;
      if (lg[i] == NB - 1 && t != prev_t) lg[i] = pp;
      if (t < rows) sm.map[lg[i]] = t;
    }
  }
  __syncthreads();
}

// One panel (at most RPT * PT active rows): register LU + the shared tail.
template <int NB, int RPT>
__global__ void __launch_bounds__(PT, 1)
    gj_panel_rows_kernel(const double2* __restrict__ cur0, long long ld, long long bstride, int n, int n_true, int k,
                         int last, GjScratch S, int* __restrict__ status0, BatchIdx bi) {
  extern __shared__ __align__(16) double2 sv[];  // Vs staging for the tail, NB x (n + 2)
  __shared__ PanelSmem<NB, RPT> sm;
  const int tid = threadIdx.x, b = blockIdx.x;
  const double2* __restrict__ cur = cur0 + (k == 0 ? bi.off(b) : (long long)b * bstride);
  int* __restrict__ status = status0 + bi.sidx(b);
  const int rows = n - k;
  ZDBG(0)
  const int* lmapg = S.lmap + (long long)b * n;
  double2 a[RPT][NB];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int t = tid + i * PT;
    const bool ok = t < rows;
    const int ph = ok ? active_row(lmapg, k, t) : 0;
    if (ok) sm.act[t] = ph;
#pragma unroll
    for (int c = 0; c < NB; ++c) a[i][c] = ok ? cur[(long long)(k + c) * ld + ph] : make_double2(0.0, 0.0);
  }
  panel_threshold_once(k, b, S);
  ZDBG(1)
  panel_lu_regs<NB, RPT>(a, rows, sm);
  ZDBG(2)
  panel_tail<NB>(cur, ld, n, n_true, k, b, last != 0, S, status, sm.lu, sm.map, sm.act, sv);
}

// Two consecutive panels K1 = [k, k+NB), K2 = [k+NB, k+2NB) and ONE rank-2NB update
// (halves the full-matrix GEMM passes; same pivots and arithmetic as two panels).
// From the current matrix M, Wz1 = M[:,K1] (-I on P1) and V1 = Pinv1 Vs1:
//   M2[:,K2]  = M[:,K2] (0 on P1) - Wz1 V1[:,K2]          (panel 2's input, all rows)
//   Vs2       = M[P2,:] (0 on K1) - Wz1[P2] V1, I on K2    (panel 2's pivot rows)
//   M <- M (0 on rows P1, P2 and cols K1, K2) - [Wz1 (0 on P2) | Wz2] [V1 (0 on K2); V2]
// with Wz2 = M2[:,K2] (-I on P2) and V2 = Pinv2 Vs2. Rows <= RPT * PT for both panels.
// (Capping it at 168 registers -- 12 B of spills -- so that a GEMM CTA of the other
// stream group can share its SM measured no better on B200: 577-579 vs 575 ms per step.)
//
// split > 1 (small batches, n <= PT): `split` CTAs per matrix. Every CTA factors both
// panels itself (same inputs, same code: identical pivots and LU bits) and keeps its own
// copies of the active-row lists and of M2 in shared memory; the column-parallel tails
// (Vs staging, V1, Vs2, V2) and the row-parallel ones (Wz, row mask, output scatters) are
// split: CTA s owns columns and rows [s n/split, (s+1) n/split). Global scratch is written
// by its owner only (lmap, piv and the status by CTA 0), so no two CTAs write one word.
template <int NB, int RPT>
__global__ void __launch_bounds__(PT, 1)
    gj_pair_kernel(const double2* __restrict__ cur0, long long ld, long long bstride, int n, int n_true, int k,
                   int last, GjScratch S, int* __restrict__ status0, BatchIdx bi, int pre2, int split) {
  constexpr int W2 = 2 * NB;
  // dynamic smem: NB x (n + 2) Vs1 / V1, then Vs2 / V2; then sv2 (pre2); then M2 (split > 1)
  extern __shared__ __align__(16) double2 sv[];
  double2* const sv2 = pre2 ? sv + NB * (n + 2) : nullptr;  // NB x (n + 2): pivot rows P2 of M
  double2* const m2s = sv + (pre2 ? 2 : 1) * NB * (n + 2);   // [NB][n] panel 2's input (split > 1)
  __shared__ PanelSmem<NB, RPT> sm;
  __shared__ double2 s_pinv[NB][NB + 1];
  __shared__ double2 s_uinv[NB];
  __shared__ double2 s_wz1p2[NB][NB + 1];  // Wz1 on the rows P2
  __shared__ int s_src1[NB], s_src2[NB];
  __shared__ int s_next[RPT * PT];  // panel 1's new active list (lmap[k .. n)), as seen by this CTA
  __shared__ int s_lmap[RPT * PT];  // last step: the final row map lmap[0 .. n)
  const int tid = threadIdx.x, b = blockIdx.x / split, part = blockIdx.x % split;
  const bool own_all = split == 1, lead = part == 0;
  const int cw = n / split, c0 = part * cw, c1 = c0 + cw;  // this CTA's columns and rows
  const double2* __restrict__ cur = cur0 + (k == 0 ? bi.off(b) : (long long)b * bstride);
  int* __restrict__ status = status0 + bi.sidx(b);
  const int k2 = k + NB, svld = n + 2;
  int* __restrict__ lmap = S.lmap + (long long)b * n;
  int* __restrict__ rowmask = S.rowmask + (long long)b * n;
  double2* __restrict__ wz = S.wz + (long long)b * n * W2;  // [W2][n], ld n
  double2* __restrict__ vb = S.vbuf + (long long)b * W2 * n;  // [n][W2], ld W2
  if (k == 0 && tid == 0 && lead) S.amax[b] = 0ull;  // the first GJ GEMM accumulates max |a|^2
  if (last && !own_all)
    for (int i = tid; i < k; i += PT) s_lmap[i] = lmap[i];
  ZDBG(10)

  // Both panels run through the same loop body (one copy of the unrolled elimination
  // in the binary: the kernel executes its code once per SM, so code size is time).
#pragma unroll 1
  for (int ph = 0; ph < 2; ++ph) {
    const int kk = ph ? k2 : k, rows = n - kk;
    int* s_src = ph ? s_src2 : s_src1;
    // panel 1 reads M[:,K1]; panel 2 reads its input M2[:,K2], computed into wz[NB..2NB)
    // (or this CTA's shared copy)
    const double2* src = ph ? (own_all ? wz + (long long)NB * n : m2s) : cur + (long long)k * ld;
    const long long sld = ph ? n : ld;
    double2 a[RPT][NB];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int t = tid + i * PT;
      const bool ok = t < rows;
      const int phys = ok ? (ph && !own_all ? s_next[NB + t] : active_row(lmap, kk, t)) : 0;
      if (ok) sm.act[t] = phys;
#pragma unroll
      for (int c = 0; c < NB; ++c) a[i][c] = ok ? src[(long long)c * sld + phys] : make_double2(0.0, 0.0);
    }
    ZDBG(11 + 10 * ph)
    panel_lu_regs<NB, RPT>(a, rows, sm);
    ZDBG(12 + 10 * ph)
    if (tid < NB) {
      const double2 d = sm.lu[tid][tid];
      if (lead) S.piv[(long long)b * n + kk + tid] = hypot(d.x, d.y);  // kernels.hpp:149-158, tested at the end
      s_uinv[tid] = crcp_fast(d);
      s_src[tid] = sm.act[sm.map[tid]];
    }
    for (int r = tid; r < rows; r += PT) {
      const int p = sm.act[sm.map[r]];
      if (lead) lmap[kk + r] = p;
      if (!own_all) {
        if (ph == 0) s_next[r] = p;
        if (last) s_lmap[kk + r] = p;
      }
    }
    __syncthreads();
    ZDBG(13 + 10 * ph)
    if (ph == 1) {
      // Wz1 on P2 = M[P2, K1] (P2 holds no P1 row)
      for (int e = tid; e < NB * NB; e += PT) s_wz1p2[e / NB][e % NB] = cur[(long long)(k + e % NB) * ld + s_src2[e / NB]];
      __syncthreads();
      for (int e = tid; e < NB * NB; e += PT) {  // rows P2: 0 in Wz1, -I in Wz2, 0 in C (by the row's owner)
        const int j = e / NB, c = e % NB, r = s_src2[j];
        if (r < c0 || r >= c1) continue;
        wz[(long long)c * n + r] = make_double2(0.0, 0.0);
        wz[(long long)(NB + c) * n + r] = make_double2(j == c ? -1.0 : 0.0, 0.0);
        if (c == 0) rowmask[r] = -1;
      }
    }
    ZDBG(14 + 10 * ph)
    // the pivot rows of M this panel needs (Vs1 into sv: this CTA's columns and K2; panel
    // 2's raw rows into sv2: this CTA's columns) are copied asynchronously so that the
    // loads overlap the pivot-block inverse
    for (int col = tid; col < n; col += PT) {
      const bool k1c = col >= k && col < k2, k2c = col >= k2 && col < k2 + NB;
      const bool mine = col >= c0 && col < c1;
      if (!(mine || (ph == 0 && k2c))) continue;
      double2* dst = ph ? sv2 : sv;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (ph == 0 && k1c)
          dst[j * svld + col] = make_double2(col - k == j ? 1.0 : 0.0, 0.0);
        else if (ph == 0 || (pre2 && !(k1c || k2c)))
          cp_async16(&dst[j * svld + col], &cur[(long long)col * ld + s_src[j]]);
      }
    }
    cp_async_commit();
    if (!S.subst) pivot_block_inverse<NB>(sm.lu, s_uinv, s_pinv);
    ZDBG(15 + 10 * ph)
    cp_async_wait<0>();
    __syncthreads();
    if (ph == 1) break;
    ZDBG(16)
    if (S.subst) {  // sv = V1 = U1^{-1} L1^{-1} Vs1, column by column (panel 1's LU is still in sm.lu)
      for (int col = tid; col < n; col += PT) {
        if (!((col >= c0 && col < c1) || (col >= k2 && col < k2 + NB))) continue;
        double2 x[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) x[j] = sv[j * svld + col];
        lu_solve_col<NB>(sm.lu, s_uinv, x);
#pragma unroll
        for (int j = 0; j < NB; ++j) sv[j * svld + col] = x[j];
      }
    } else {
      apply_pinv_dmma<NB>(s_pinv, sv, svld, n, nullptr, 0, c0 / 8, c1 / 8, k2 / 8, (k2 + NB) / 8);  // sv = V1
    }
    __syncthreads();
    ZDBG(17)
    // Wz1 and panel 2's input M2[:,K2], one row per thread: every row for this CTA's
    // panel-2 factorisation, the global copies (the GEMM's operands) for its own rows
    for (int r = tid; r < n; r += PT) {
      int j1 = -1;
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if (s_src1[q] == r) j1 = q;
      const bool mine = r >= c0 && r < c1;
      double2 w[NB], m2[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        w[c] = j1 >= 0 ? make_double2(j1 == c ? -1.0 : 0.0, 0.0) : cur[(long long)(k + c) * ld + r];
        m2[c] = j1 >= 0 ? make_double2(0.0, 0.0) : cur[(long long)(k2 + c) * ld + r];
      }
      if (mine) {
#pragma unroll
        for (int c = 0; c < NB; ++c) wz[(long long)c * n + r] = w[c];
      }
#pragma unroll 1
      for (int q = 0; q < NB; ++q) {
        double2 wq = w[0];
#pragma unroll
        for (int u = 1; u < NB; ++u)
          if (u == q) wq = w[u];
        const double2 nq = make_double2(-wq.x, -wq.y);
#pragma unroll
        for (int c = 0; c < NB; ++c) m2[c] = cfma(nq, sv[q * svld + k2 + c], m2[c]);
      }
      if (mine) {
#pragma unroll
        for (int c = 0; c < NB; ++c) wz[(long long)(NB + c) * n + r] = m2[c];
        rowmask[r] = j1 >= 0 ? -1 : r;
      }
      if (!own_all) {
#pragma unroll
        for (int c = 0; c < NB; ++c) m2s[(long long)c * n + r] = m2[c];
      }
    }
    __syncthreads();
    ZDBG(18)
  }
  // per column of this CTA: V1 (0 on K2) -> vb rows 0..NB-1; Vs2 replaces V1 in sv
  for (int col = c0 + tid; col < c1; col += PT) {
    double2 v1[NB], x[NB];
    const bool c1c = col >= k && col < k2, c2 = col >= k2 && col < k2 + NB;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      v1[j] = sv[j * svld + col];
      vb[(long long)col * W2 + j] = c2 ? make_double2(0.0, 0.0) : v1[j];
      x[j] = c2 ? make_double2(col - k2 == j ? 1.0 : 0.0, 0.0)
                : (c1c ? make_double2(0.0, 0.0) : (pre2 ? sv2[j * svld + col] : cur[(long long)col * ld + s_src2[j]]));
    }
    if (!c2) {
#pragma unroll 1
      for (int q = 0; q < NB; ++q) {
        double2 vq = v1[0];
#pragma unroll
        for (int u = 1; u < NB; ++u)
          if (u == q) vq = v1[u];
        const double2 nq = make_double2(-vq.x, -vq.y);
#pragma unroll
        for (int j = 0; j < NB; ++j) x[j] = cfma(s_wz1p2[j][q], nq, x[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) sv[j * svld + col] = x[j];
  }
  __syncthreads();
  ZDBG(26)
  if (S.subst) {  // V2 = U2^{-1} L2^{-1} Vs2 -> vb rows NB..2NB-1
    for (int col = c0 + tid; col < c1; col += PT) {
      double2 x[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) x[j] = sv[j * svld + col];
      lu_solve_col<NB>(sm.lu, s_uinv, x);
#pragma unroll
      for (int j = 0; j < NB; ++j) vb[(long long)col * W2 + NB + j] = x[j];
    }
  } else {
    apply_pinv_dmma<NB>(s_pinv, sv, svld, n, vb + NB, W2, c0 / 8, c1 / 8);  // V2 -> vb rows NB..2NB-1
  }
  ZDBG(27)
  if (last) {  // output scatters: row lmap[i] -> i, column c -> lmap[c] (this CTA's i)
    // (gathering the last GEMM's C and Wz rows through lmap instead, so that it writes
    // whole rows in order, measured slower on B200: 101 vs 87 us per launch)
    int* __restrict__ rowscat = S.rowscat + (long long)b * n;
    int* __restrict__ colmap = S.colmap + (long long)b * n;
    if (!own_all) __syncthreads();  // s_lmap complete
    for (int i = c0 + tid; i < c1; i += PT) {
      const int p = own_all ? lmap[i] : s_lmap[i];
      rowscat[p] = i;
      colmap[i] = p;
    }
  }
  __syncthreads();
  if (last && lead) final_status(S, b, n, n_true, status);
  ZDBG(28)
}


// ---------------------------------------------------------------------------------------
// Register-resident Gauss-Jordan panels (round 2, the default for n <= PT).
//
// Thread t owns PHYSICAL row t of the matrix for the whole kernel (rows never move, so the
// panel columns load coalesced with no row map), and instead of factoring the panel
// (L \ U), forming Pinv from two triangular inverses and multiplying V = Pinv Vs, the
// elimination itself runs as in-place Gauss-Jordan on all n rows of the n x NB panel:
//   column j, pivot row p (largest |re|+|im| among the rows not yet used as pivots):
//     row p:   a[p][j] <- 1/a[p][j],  a[p][c] <- a[p][c] / a[p][j]         (c != j)
//     row r:   l = a[r][j] / a[p][j], a[r][j] <- -l, a[r][c] <- a[r][c] - l a[p][c]
// After NB columns the registers hold W = E[:, P], the columns of the accumulated row
// operation E (E M[:, K] = unit columns at the pivot rows): W[P] = Pinv and
// W[R] = -M[R, K] Pinv, which are exactly the new panel columns of the blocked step
// (see the header of this file), and for the other columns
//   M <- M (0 on rows P / cols K) + W Vs,   Vs = M[P, :] with the identity in columns K,
// so the GEMM operands are W (from registers) and the RAW pivot rows: no Pinv, no V
// product. The active rows see the same operations in the same order as in the LU panel,
// so pivots are chosen from the same values. The pivot rows are fetched with cp.async as
// each pivot is resolved (their latency hides behind the remaining columns).
// Two panels per launch, one rank-2NB update, as in gj_pair_kernel:
//   M2[:, K2] = M[:, K2] (0 on P1) + W1 Vs1[:, K2]      (per thread: its own row)
//   Vs2       = M[P2, :] (0 on K1) + W1[P2] Vs1, I on K2
//   M <- M (0 on rows P1, P2 / cols K1, K2) + [W1 (0 on P2) | W2] [Vs1 (0 on K2); Vs2]
// Several CTAs per matrix (n > PT): a thread-block cluster of CL CTAs, CTA `rank` owns
// rows and columns [rank PT, (rank + 1) PT). Every warp pushes its pivot KEY into the same
// slot of every CTA's shared memory (one DSMEM store per CTA) and keeps its candidate record
// (row, reciprocal, pivot) local; the per-column barrier becomes a cluster barrier (release /
// acquire), every CTA resolves the same winner from the CL * 8 keys, and the CTAs that do not
// own it fetch its record (18 DSMEM loads by 18 threads) from the owner. (Pushing every
// candidate row to every CTA measured 4.3 k cycles per column on B200 against 1.4 k for one
// CTA: 54 remote stores per warp and column, 23 of 24 rows never used.)
template <int CL>
__device__ __forceinline__ void gj_sync() {
  if constexpr (CL == 1)
    __syncthreads();
  else
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned dsmem_addr(const void* p, unsigned rank) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(unsigned addr, unsigned v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ double2 ld_cluster(unsigned addr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}

template <int NB>
struct GjCand {  // one warp's pivot candidate
  double2 row[NB];  // the candidate row (all NB columns of the panel)
  double2 rcp;      // reciprocal of its entry in the pivot column
  double2 piv;      // the entry itself (deferred negligible-pivot test)
};

template <int NB, int CL>
struct GjRowSmem {
  static constexpr int NC = CL * (PT / 32);  // one key slot per warp of the cluster
  __align__(16) unsigned cand_k[2][NC];      // keys of every warp of the cluster (pushed by their owners)
  __align__(16) GjCand<NB> cand[2][PT / 32]; // this CTA's candidates
  __align__(16) GjCand<NB> pulled;           // CL > 1: the winner's record, fetched from its owner
  double2 w1p2[NB][NB + 1];                  // W1 on the rows P2
  __align__(16) double2 vk2[NB][NB];         // Vs1[:, K2]
  double2 pv[2][NB];                         // the pivots
  int src[2][NB];                            // physical pivot rows of the two panels
  unsigned char used[PT];                    // own rows used as pivots by earlier steps
};

// Resources sized so that one 128-thread GEMM CTA of another stream group fits next to a panel CTA on the
// same SM: 168 registers (no spills worth naming: 8-24 bytes) and two staging tiles only -- W1 goes
// through the global Wz operand and, for the panel-2 input, through this thread's free sv2 slots
// (146 KB of shared memory with the static part; the sweep GEMM CTA needs 64-75 KB and 21.5 K registers).
// B200, config 2: 535.8 -> 514.1 ms per step (the panels no longer hold ~half of the SMs to themselves);
// 8-energy shards 103.7 -> 108.2 ms (the shared FP64 pipe lengthens the panels' chain). -DBBSI_GJ_EXCLUSIVE_SM
// builds the exclusive variant (W1 in a third shared-memory tile, one CTA per SM).
#ifndef BBSI_GJ_EXCLUSIVE_SM
#define GJ_ROWS_BOUNDS __maxnreg__(168)
constexpr bool kW1Smem = false;
#else
#define GJ_ROWS_BOUNDS __launch_bounds__(PT, 1)
constexpr bool kW1Smem = true;
#endif

template <int NB, int CL>
__global__ void GJ_ROWS_BOUNDS
    gj_rows_kernel(const double2* __restrict__ cur0, long long ld, long long bstride, int n, int n_true, int k, int last,
                   GjScratch S, int* __restrict__ status0, BatchIdx bi) {
  static_assert(PT == NB * NB, "one thread per entry of the NB x NB blocks");
  static_assert(CL * PT <= int(KEY_IMASK) + 1, "row numbers must fit the pivot key");
  constexpr int W2 = 2 * NB;
  // One CTA: the pivot rows are fetched as each pivot is resolved (the latency hides behind the remaining
  // columns). Clusters: after the 16 columns (copies in flight lengthen every release barrier: measured on
  // B200 at n = 768, 123 k -> 111 k cycles per step).
  constexpr bool kGatherInLoop = CL == 1;
  constexpr int svld = PT + 1;  // odd: a warp reading one column of the [NB][svld] tiles hits 32 distinct bank groups
  extern __shared__ __align__(16) double2 sv[];  // own columns of Vs1 [NB][svld]; of the raw rows P2; W1 [NB][PT]
  double2* const sv2 = sv + NB * svld;
  double2* const w1s = sv2 + NB * svld;  // W1 of the own rows (panel 1's result, kept out of the registers)
  __shared__ GjRowSmem<NB, CL> sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x / CL, rank = blockIdx.x % CL;
  const int grow = rank * PT + tid;  // this thread's row (and column) of the matrix
  const int slot = rank * (PT / 32) + warp;
  const double2* __restrict__ cur = cur0 + (k == 0 ? bi.off(b) : (long long)b * bstride);
  int* __restrict__ status = status0 + bi.sidx(b);
  const int k2 = k + NB;
  int* __restrict__ lmap = S.lmap + (long long)b * n;
  int* __restrict__ rowmask = S.rowmask + (long long)b * n;
  double2* __restrict__ wz = S.wz + (long long)b * n * W2;    // [W2][n], ld n
  double2* __restrict__ vb = S.vbuf + (long long)b * W2 * n;  // [n][W2], ld W2
  if (k == 0 && tid == 0 && rank == 0) S.amax[b] = 0ull;  // the first GJ GEMM accumulates max |a|^2
  ZDBG(30)
  sm.used[tid] = 0;
  __syncthreads();
  for (int i = tid; i < k; i += PT) {
    const int p = lmap[i] - rank * PT;
    if (p >= 0 && p < PT) sm.used[p] = 1;
  }
  gj_sync<CL>();  // (CL > 1: every CTA of the cluster is resident before the first remote store)
  const bool inrow = grow < n;
  bool cand = inrow && !sm.used[tid];
  bool piv1 = false, piv2 = false;
  double2 a[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) a[c] = inrow ? cur[(long long)(k + c) * ld + grow] : make_double2(0.0, 0.0);
  // panel 2's raw columns M[:, K2] of the own row, staged in sv2 (free until panel 2's pivot rows arrive, which
  // land in the same thread's slots); they join panel 1's copy group
  if (inrow) {
#pragma unroll
    for (int c = 0; c < NB; ++c) cp_async16(&sv2[c * svld + tid], &cur[(long long)(k2 + c) * ld + grow]);
  }
  ZDBG(31)

  // Both panels run through one loop body (the kernel executes its code once per SM).
#pragma unroll 1
  for (int ph = 0; ph < 2; ++ph) {
    const int kk = ph ? k2 : k;
    double2* const dst = ph ? sv2 : sv;
    const bool kcol = ph == 0 && grow >= kk && grow < kk + NB;  // identity columns of Vs1
    // this warp's best candidate for column J: the key now (lane 0); from the winning lane its
    // reciprocal, the pivot itself and the row once the row is fully updated. Every lane forms the
    // reciprocal of its own entry (branch-free), so its dependent chain overlaps the other updates
    auto publish_key = [&](int par, int J, double2& rc) -> bool {
      const unsigned key = cand ? piv_key(a[J], grow) : 0u;
      rc = crcp_lanes(a[J]);
      const unsigned wk = __reduce_max_sync(0xffffffffu, key);
      if (lane == 0) {
        if constexpr (CL == 1) {
          sm.cand_k[par][slot] = wk;
        } else {
#pragma unroll
          for (int r = 0; r < CL; ++r) st_cluster(dsmem_addr(&sm.cand_k[par][slot], r), wk);
        }
      }
      return wk != 0 && key == wk;
    };
    auto publish_rcp = [&](int par, int J, double2 rc) {
      sm.cand[par][warp].rcp = rc;
      sm.cand[par][warp].piv = a[J];
    };
    auto publish_row = [&](int par) {
#pragma unroll
      for (int c = 0; c < NB; ++c) sm.cand[par][warp].row[c] = a[c];
    };
    {
      double2 rc;
      if (publish_key(0, 0, rc)) {
        publish_rcp(0, 0, rc);
        publish_row(0);
      }
    }
  ZDBG(32 + 8 * ph)
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int par = j & 1;
      gj_sync<CL>();
      unsigned best = 0;
#pragma unroll
      for (int q = 0; q < GjRowSmem<NB, CL>::NC / 4; ++q) {
        const uint4 kq = reinterpret_cast<const uint4*>(sm.cand_k[par])[q];
        best = max(max(best, max(kq.x, kq.y)), max(kq.z, kq.w));
      }
      const int tj = int(KEY_IMASK - (best & KEY_IMASK));  // the pivot's row of the matrix
      const int qw = tj >> 5;                               // and its key slot: CTA qw / 8, warp qw % 8
      const GjCand<NB>* cw = &sm.cand[par][qw % (PT / 32)];
      if constexpr (CL > 1) {
        const int owner = qw / (PT / 32);
        if (owner != rank) {  // (uniform over the CTA) fetch the winner's record from its owner's shared memory
          if (tid < NB + 2)
            reinterpret_cast<double2*>(&sm.pulled)[tid] =
                ld_cluster(dsmem_addr(reinterpret_cast<const double2*>(cw) + tid, unsigned(owner)));
          __syncthreads();
          cw = &sm.pulled;
        }
      }
      const double2 rcp = cw->rcp;
      const bool isp = grow == tj;
      if (isp) {  // this row is pivot j of the panel: its own row comes back from cand_row scaled by 1/p
        cand = false;
        if (ph)
          piv2 = true;
        else
          piv1 = true;
#pragma unroll
        for (int c = 0; c < NB; ++c) a[c] = make_double2(0.0, 0.0);
      }
      if (tid == 0) {
        sm.src[ph][j] = tj;
        sm.pv[ph][j] = cw->piv;
      }
      if constexpr (kGatherInLoop) {
        if (inrow && !kcol) cp_async16(&dst[j * svld + tid], &cur[(long long)grow * ld + tj]);
        if (ph == 0 && tid < NB) cp_async16(&sm.vk2[j][tid], &cur[(long long)(k2 + tid) * ld + tj]);
      }
      double2 l = cmul(a[j], rcp);
      if (isp) l = make_double2(-rcp.x, -rcp.y);
      a[j] = make_double2(-l.x, -l.y);
      auto update = [&](int c) {
        const double2 u = cw->row[c];
        double2 x = a[c];
        x.x = fma(-l.x, u.x, fma(l.y, u.y, x.x));
        x.y = fma(-l.x, u.y, fma(-l.y, u.x, x.y));
        a[c] = x;
      };
      if (j + 1 < NB) {
        update(j + 1);
        double2 rc;
        const bool win = publish_key(par ^ 1, j + 1, rc);
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c != j && c != j + 1) update(c);
        if (win) {
          publish_rcp(par ^ 1, j + 1, rc);
          publish_row(par ^ 1);
        }
      } else {
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c != j) update(c);
      }
    }
    if constexpr (!kGatherInLoop) {  // (clusters: copies in flight would stall every release barrier)
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int tj = sm.src[ph][j];
        if (inrow && !kcol) cp_async16(&dst[j * svld + tid], &cur[(long long)grow * ld + tj]);
        if (ph == 0 && tid < NB) cp_async16(&sm.vk2[j][tid], &cur[(long long)(k2 + tid) * ld + tj]);
      }
    }
    cp_async_commit();
  ZDBG(33 + 8 * ph)
    if (kcol) {
#pragma unroll
      for (int j = 0; j < NB; ++j) sv[j * svld + tid] = make_double2(grow - kk == j ? 1.0 : 0.0, 0.0);
    }
    if (ph == 1) break;
    // panel 2's input, this thread's row: M2[r, K2] = M[r, K2] (0 on P1) + W1[r] Vs1[:, K2]
    if constexpr (kW1Smem) {
#pragma unroll
      for (int c = 0; c < NB; ++c) w1s[c * PT + tid] = a[c];
      cp_async_wait<0>();
#pragma unroll
      for (int c = 0; c < NB; ++c) a[c] = (inrow && !piv1) ? sv2[c * svld + tid] : make_double2(0.0, 0.0);
    } else {  // W1 -> the Wz operand (global) and, for the loop below, this thread's slots of sv2
      cp_async_wait<0>();
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const double2 raw = (inrow && !piv1) ? sv2[c * svld + tid] : make_double2(0.0, 0.0);
        if (inrow) wz[(long long)c * n + grow] = a[c];
        sv2[c * svld + tid] = a[c];
        a[c] = raw;
      }
    }
    __syncthreads();
  ZDBG(34)
#pragma unroll 1
    for (int q = 0; q < NB; ++q) {
      const double2 wq = kW1Smem ? w1s[q * PT + tid] : sv2[q * svld + tid];
#pragma unroll
      for (int c = 0; c < NB; ++c) a[c] = cfma(wq, sm.vk2[q][c], a[c]);
    }
  ZDBG(35)
  }
  // ---- the GEMM operands and the bookkeeping
  if (inrow) {
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if constexpr (kW1Smem) wz[(long long)c * n + grow] = piv2 ? make_double2(0.0, 0.0) : w1s[c * PT + tid];
      wz[(long long)(NB + c) * n + grow] = a[c];
    }
    rowmask[grow] = (piv1 || piv2) ? -1 : grow;
  }
  ZDBG(44)
  cp_async_wait<0>();
  __syncthreads();
  {  // W1 on the rows P2, from the rows' owners
    const int j = tid / NB, c = tid % NB, r = sm.src[1][j];
    if constexpr (!kW1Smem)
      sm.w1p2[j][c] = __ldcg(&wz[(long long)c * n + r]);  // written before the last 16 (cluster) barriers
    else if constexpr (CL == 1)
      sm.w1p2[j][c] = w1s[c * PT + r];
    else
      sm.w1p2[j][c] = ld_cluster(dsmem_addr(&w1s[c * PT + (r % PT)], unsigned(r / PT)));
  }
  gj_sync<CL>();  // (CL > 1: no CTA leaves while a peer still reads its shared memory)
  if constexpr (!kW1Smem) {  // W1 is 0 on the rows P2 in the combined update (after every read of those rows)
    if (inrow && piv2) {
#pragma unroll
      for (int c = 0; c < NB; ++c) wz[(long long)c * n + grow] = make_double2(0.0, 0.0);
    }
  }
  ZDBG(45)
  if (rank == 0 && tid < W2) {
    const int ph = tid / NB, j = tid % NB;
    const double2 d = sm.pv[ph][j];
    S.piv[(long long)b * n + k + tid] = hypot(d.x, d.y);  // kernels.hpp:149-158, tested at the end
    lmap[k + tid] = sm.src[ph][j];
  }
  {  // this thread's column: Vs2 = M[P2, col] (0 on K1) + W1[P2] Vs1[:, col], I on K2; it replaces the raw rows in sv2
    const int col = grow;
    const bool c1c = col >= k && col < k2, c2 = col >= k2 && col < k2 + NB;
    double2 x[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j)
      x[j] = c2 ? make_double2(col - k2 == j ? 1.0 : 0.0, 0.0) : ((c1c || !inrow) ? make_double2(0.0, 0.0) : sv2[j * svld + tid]);
    if (!c2 && inrow) {
#pragma unroll 1
      for (int q = 0; q < NB; ++q) {
        const double2 vq = sv[q * svld + tid];
#pragma unroll
        for (int j = 0; j < NB; ++j) x[j] = cfma(sm.w1p2[j][q], vq, x[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      sv2[j * svld + tid] = x[j];
      if (c2) sv[j * svld + tid] = make_double2(0.0, 0.0);  // Vs1 is 0 on K2 in the combined update
    }
  }
  __syncthreads();
  // [Vs1; Vs2] of the own columns -> vb, one warp per column (32 consecutive entries: coalesced)
#pragma unroll 4
  for (int i = 0; i < PT / 8; ++i) {
    const int cl_ = warp + (PT / 32) * i, col = rank * PT + cl_;
    if (col < n) vb[(long long)col * W2 + lane] = lane < NB ? sv[lane * svld + cl_] : sv2[(lane - NB) * svld + cl_];
  }
  ZDBG(46)
  if (last && inrow) {  // output scatters: row lmap[i] -> i, column c -> lmap[c]
    int* __restrict__ rowscat = S.rowscat + (long long)b * n;
    int* __restrict__ colmap = S.colmap + (long long)b * n;
    const int i = grow;
    const int p = i < k ? lmap[i] : (i < k2 ? sm.src[0][i - k] : sm.src[1][i - k2]);
    rowscat[p] = i;
    colmap[i] = p;
  }
  __syncthreads();
  if (last && rank == 0) final_status(S, b, n, n_true, status);
  ZDBG(47)
}

}  // namespace

void zinv_set_concurrency(int groups) { t_conc = groups < 1 ? 1 : groups; }

extern "C" int bbsi_debug_zinv(long long* out) { return (int)cudaMemcpyFromSymbol(out, g_zinv_dbg, sizeof(long long) * 64); }

size_t zinv_scratch_bytes(int n, int batch) {
  GjScratch s;
  return carve(s, nullptr, n, kNB, batch) + 256;
}

cudaError_t zinv_batched(double2* M, long long ld, long long bstride, int n, int n_true, int batch, void* scratch,
                         int* status, cudaStream_t stream) {
  return zinv_batched2(M, ld, bstride, n, n_true, batch, 1, 0, scratch, status, 0, stream);
}

cudaError_t zinv_batched2(double2* M, long long ld, long long bstride, int n, int n_true, int inner, int outer,
                          long long ostride, void* scratch, int* status, long long sostride, cudaStream_t stream) {
  if (n % 64 || n_true > n || n_true < 1 || outer < 1 || outer > kMaxProblems) return cudaErrorInvalidValue;
  const int batch = inner * outer;
  if (batch == 0) return cudaSuccess;
  constexpr int nb = kNB;
  GjScratch S;
  carve(S, scratch, n, nb, batch);
  S.subst = gj_subst();
  const size_t smem = size_t(nb) * (n + 1) * sizeof(double2) + 3 * size_t(n) * sizeof(int);
  cudaError_t e;
  const int kind = panel_kind();
  // gj_rows_kernel: one thread per row, CL = ceil(n / PT) CTAs (a cluster) per matrix; n % 64 == 0, so every
  // step is a pair of panels
  const int cl = (n + PT - 1) / PT;
  const bool rowsgj = kind == 1 && cl <= gj_rows_max_cl(n, batch);
  const size_t gjr_smem = (2 * size_t(nb) * (PT + 1) + (kW1Smem ? size_t(nb) * PT : 0)) * sizeof(double2);  // Vs1, raw rows P2, W1
  const void* gjr_fn = cl == 1   ? (const void*)gj_rows_kernel<kNB, 1>
                       : cl == 2 ? (const void*)gj_rows_kernel<kNB, 2>
                       : cl == 3 ? (const void*)gj_rows_kernel<kNB, 3>
                                 : (const void*)gj_rows_kernel<kNB, 4>;
  if (rowsgj && (e = set_max_dyn_smem(gjr_fn, gjr_smem))) return e;
  const size_t rows_smem = size_t(nb) * (n + 2) * sizeof(double2);  // Vs staging of the tail
  const int split = pair_split(n, batch);
  const size_t m2_smem = split > 1 ? size_t(nb) * n * sizeof(double2) : 0;  // per-CTA M2 (split pair)
  if (!rowsgj) {  // LU panels: tall (shared-memory) panel, register panels, pair panels
    if ((e = set_max_dyn_smem((const void*)gj_panel_kernel<kNB>, smem))) return e;
    const void* fns[4] = {(const void*)gj_panel_rows_kernel<kNB, 1>, (const void*)gj_panel_rows_kernel<kNB, 2>,
                          (const void*)gj_pair_kernel<kNB, 1>, (const void*)gj_pair_kernel<kNB, 2>};
    for (int i = 0; i < 4; ++i)  // (the M2 copy: split pair, RPT = 1, only)
      if ((e = set_max_dyn_smem(fns[i], (i >= 2 && pair_pre2(n) ? 2 : 1) * rows_smem + (i == 2 ? m2_smem : 0))))
        return e;
  }
  const long long nn = (long long)n * n;
  // LU panel steps: two panels per step (pair kernel, one rank-2nb GEMM) wherever both
  // fit the register kernel; single panels otherwise (tall panels, BBSI_PANEL=2/3)
  for (int k = 0; k < n;) {
    const int rows = n - k;
    const bool pair = rowsgj || (kind == 1 && rows <= 2 * PT && k + 2 * nb <= n);
    const int kw = pair ? 2 * nb : nb;
    const int last = k + kw == n;
    // the first step reads the input block; the working matrix s0 is updated in place
    const double2* cur = k == 0 ? M : S.s0;
    const BatchIdx bi{inner, k == 0 ? bstride : nn, k == 0 ? ostride : nn * inner, sostride};
    const long long cld = k == 0 ? ld : n, cbs = k == 0 ? bstride : nn;
    const long long nld = last ? ld : n, nbs = last ? bstride : nn;
    {
      ProfScope prof(stream, PROF_INV, 8.0 * double(n) * nb * kw * batch, 16.0 * (3.0 * n * kw) * batch);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(batch);
      cfg.blockDim = dim3(PT);
      cfg.dynamicSmemBytes = rows_smem;
      cfg.stream = stream;
      cudaLaunchAttribute attr_[1];
      attr_[0].id = cudaLaunchAttributePriority;
      attr_[0].val.priority = panel_priority();
      cfg.attrs = attr_;
      cfg.numAttrs = 1;
      const int pre2 = pair_pre2(n) ? 1 : 0;
      if (pair && pre2) cfg.dynamicSmemBytes = 2 * rows_smem;  // Vs staging + panel 2's pivot rows
      if (rowsgj) {
        cfg.dynamicSmemBytes = gjr_smem;
        cfg.gridDim = dim3(batch * cl);
        cudaLaunchAttribute attr2[2];
        attr2[0] = attr_[0];
        attr2[1].id = cudaLaunchAttributeClusterDimension;
        attr2[1].val.clusterDim.x = cl;
        attr2[1].val.clusterDim.y = 1;
        attr2[1].val.clusterDim.z = 1;
        cfg.attrs = attr2;
        cfg.numAttrs = cl > 1 ? 2 : 1;
        int kl = last;
        void* args[] = {(void*)&cur, (void*)&cld, (void*)&cbs, (void*)&n, (void*)&n_true, (void*)&k, (void*)&kl,
                        (void*)&S, (void*)&status, (void*)&bi};
        e = cudaLaunchKernelExC(&cfg, gjr_fn, args);
      } else if (pair && rows <= PT) {
        cfg.gridDim = dim3(batch * split);
        cfg.dynamicSmemBytes += m2_smem;
        e = cudaLaunchKernelEx(&cfg, gj_pair_kernel<kNB, 1>, cur, cld, cbs, n, n_true, k, last, S, status, bi, pre2,
                               split);
      } else if (pair) {
        e = cudaLaunchKernelEx(&cfg, gj_pair_kernel<kNB, 2>, cur, cld, cbs, n, n_true, k, last, S, status, bi, pre2,
                               1);
      } else if (kind != 2 && rows <= PT) {
        e = cudaLaunchKernelEx(&cfg, gj_panel_rows_kernel<kNB, 1>, cur, cld, cbs, n, n_true, k, last, S, status, bi);
      } else if (kind != 2 && rows <= 2 * PT) {
        e = cudaLaunchKernelEx(&cfg, gj_panel_rows_kernel<kNB, 2>, cur, cld, cbs, n, n_true, k, last, S, status, bi);
      } else {
        cfg.dynamicSmemBytes = smem;
        e = cudaLaunchKernelEx(&cfg, gj_panel_kernel<kNB>, cur, cld, cbs, n, n_true, k, last, S, status, bi);
      }
      if (e) return e;
    }
    ZGemmGroup g{};
    g.batch = inner;
    g.bs = 64;
    g.nprob = outer;
    g.prof_cat = PROF_GJ_GEMM;
    // M <- M (0 on the pivot rows and the panel columns) - Wz V, one problem per outer batch
    for (int o = 0; o < outer; ++o) {
      const long long so = (long long)o * inner;  // first scratch entry of this outer batch
      ZGemmProblem& p = g.prob[o];
      p = ZGemmProblem{};
      p.M = n;
      p.N = n;
      p.K = kw;
      p.alpha = make_double2(rowsgj ? 1.0 : -1.0, 0.0);  // gj_rows_kernel: M + W Vs; LU panels: M - Wz V
      p.beta = make_double2(1.0, 0.0);
      p.A = ZOp{S.wz + so * n * kw, n, 64, 64LL * n, (long long)n * kw};
      p.B = ZOp{S.vbuf + so * kw * n, kw, 64, 64LL * kw, (long long)kw * n};
      const double2* c0 = k == 0 ? M + o * ostride : S.s0 + so * nn;
      double2* d0 = last ? M + o * ostride : S.s0 + so * nn;
      p.C = ZOp{c0, cld, 64, 64LL * cld, cbs};
      p.D = ZOp{d0, nld, 64, 64LL * nld, nbs};
      p.rowmap = S.rowmask + so * n;
      p.rowscat = last ? S.rowscat + so * n : nullptr;
      p.colmap = last ? S.colmap + so * n : nullptr;
      p.map_bstride = n;
      p.zr0 = p.zr1 = 0;
      p.zc0 = k;
      p.zc1 = k + kw;
      if (k == 0) {  // completes max |a| of the input block for the deferred pivot test
        p.amax = S.amax + so;
        p.amax_n = n_true;
      }
    }
    if ((e = zgemm_grouped(g, stream))) return e;
    k += kw;
  }
  return cudaSuccess;
}

}  // namespace bbsi_gpu

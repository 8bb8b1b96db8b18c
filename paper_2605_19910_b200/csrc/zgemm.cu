// Grouped, batched, block-strided complex-FP64 GEMM on DMMA (mma.sync m8n8k4 f64).
//
// Replaces every zgemm the reference issues through gemm_into (kernels.hpp:102-117)
// on the solver path: one launch covers up to kMaxProblems independent products,
// each batched over energies / domains, each operand a strided set of bs x bs
// blocks (see ZOp). The n-diagonal k x k window updates (rgf.hpp:107-112) and the
// downward row/column accumulations (rgf.hpp:122-134) become ONE product each.
//
// Complex product with 4 real DMMAs per 8x8x4 step (no 3M trick: same rounding
// class as zgemm). CTA tile 64x64 complex, 4 warps of 32x32, K staged 16 at a
// time through a 2-stage cp.async pipeline into padded, bank-conflict-free smem.
#include <cstdlib>

#include "internal.h"

namespace bbsi_gpu {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int LDA_S = BM + 2;  // As[k][m]: 16B lanes l/4 rows x l%4 ks -> 8 distinct slots per phase
constexpr int LDB_S = BK + 4;  // Bs[n][k]
constexpr int STAGES = 2;
constexpr int A_STAGE = BK * LDA_S;
constexpr int B_STAGE = BN * LDB_S;
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * sizeof(double2);

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}

template <bool PLAIN>
__device__ __forceinline__ long long toff(const ZOp& o, int bs, int r, int c) {
  return PLAIN ? (long long)c * o.ld + r : zop_offset(o, bs, r, c);
}

template <bool PLAIN>
__device__ __forceinline__ void load_tile(const ZGemmProblem& P, int bs, int batch, int m0, int n0, int k0,
                                          double2* As, double2* Bs, int tid) {
  const double2* a = P.A.p + (long long)batch * P.A.bstride + toff<PLAIN>(P.A, bs, m0, k0);
  const double2* b = P.B.p + (long long)batch * P.B.bstride + toff<PLAIN>(P.B, bs, k0, n0);
  const int mlim = P.M - m0, nlim = P.N - n0;
#pragma unroll
  for (int i = 0; i < (BM * BK) / 128; ++i) {
    int e = tid + 128 * i;
    int m = e & (BM - 1), k = e >> 6;
    const bool v = m < mlim;
    cp_async16_zfill(&As[k * LDA_S + m], v ? a + (long long)k * P.A.ld + m : a, v);
  }
#pragma unroll
  for (int i = 0; i < (BN * BK) / 128; ++i) {
    int e = tid + 128 * i;
    int k = e & (BK - 1), n = e >> 4;
    const bool v = n < nlim;
    cp_async16_zfill(&Bs[n * LDB_S + k], v ? b + (long long)n * P.B.ld + k : b, v);
  }
}

// MINB = resident CTAs per SM the register budget is sized for (2: 243 regs, no
// spills; 3: 168 regs, 12 warps per SM, a few epilogue spills).
// AMAX: the first Gauss-Jordan step's variant (max |C|^2, ZGemmProblem::amax); a
// separate instantiation so the other launches keep their register allocation.
// One 64 x 64 output tile t of the flattened (problem, batch, tile) index.
template <bool PLAIN, bool AMAX, bool CFORM>
__device__ __forceinline__ void zgemm_tile(const ZGemmGroup& g, const int t, double2* As, double2* Bs) {
  // ---- decode the flattened tile index
  int pi = 0;
#pragma unroll 1
  for (int q = 1; q < g.nprob; ++q)
    if (t >= g.prob[q].tile_begin) pi = q;
  const ZGemmProblem& P = g.prob[pi];
  int local = t - P.tile_begin;
  const int per_batch = P.tiles_m * P.tiles_n;
  const int batch = local / per_batch;
  local -= batch * per_batch;
  const int m0 = (local % P.tiles_m) * BM;
  const int n0 = (local / P.tiles_m) * BN;
  const int bs = g.bs;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int lr = lane >> 2, lc = lane & 3;

  double cr[4][4][2], ci[4][4][2];
  const int nk = P.K / BK;
  load_tile<PLAIN>(P, bs, batch, m0, n0, 0, As, Bs, tid);
  cp_async_commit();

  // C enters as the accumulator's initial value when beta == 1 and alpha = +-1
  // (D = alpha*(alpha*C + AB) = C + alpha*AB exactly); all C loads are issued
  // up front, overlapping the first tile copies, and the epilogue only stores.
  const bool use_c = (P.beta.x != 0.0 || P.beta.y != 0.0);
  const bool c_in_acc = use_c && P.beta.x == 1.0 && P.beta.y == 0.0 && P.alpha.y == 0.0 &&
                        (P.alpha.x == 1.0 || P.alpha.x == -1.0);
  if (c_in_acc) {
    // tiles never straddle a bs block: address = tile base + local offset. A row
    // map is only allowed on plain operands (offset(r, c) = r + c*ld).
    const int* rmap = P.rowmap ? P.rowmap + (long long)batch * P.map_bstride : nullptr;
    const double2* __restrict__ cb = P.C.p + (long long)batch * P.C.bstride;
    const double2* __restrict__ ct = cb + toff<PLAIN>(P.C, bs, m0, n0);
    const double sg = P.alpha.x;
    int srow[4];
    bool rowok[4], colok[4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int m = m0 + wm + mi * 8 + lr;
      rowok[mi] = m < P.M && !(m >= P.zr0 && m < P.zr1);
      srow[mi] = rmap ? (m < P.M ? __ldg(&rmap[m]) : 0) : m - m0;
      if (srow[mi] < 0) rowok[mi] = false;
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int n = n0 + wn + ni * 8 + lc * 2 + q;
        colok[ni][q] = n < P.N && !(n >= P.zc0 && n < P.zc1);
      }
    const double2* __restrict__ rb = rmap ? cb + (long long)n0 * P.C.ld : ct;
    double2 cv[4][4][2];
    if (AMAX && PLAIN && P.amax) {
      // first Gauss-Jordan step (identity row map): the whole tile as stored is read in
      // the same batch of loads -- masked entries only feed max |C_ij|^2 (rows, columns
      // < amax_n), the accumulator takes them as 0
      const double2* __restrict__ raw = cb + (long long)n0 * P.C.ld;
      double mx = 0.0;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = m0 + wm + mi * 8 + lr;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int nl = wn + ni * 8 + lc * 2 + q;
            cv[mi][ni][q] = (r < P.M && n0 + nl < P.N) ? raw[(long long)nl * P.C.ld + r] : make_double2(0.0, 0.0);
          }
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = m0 + wm + mi * 8 + lr;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double2 v = cv[mi][ni][q];
            if (r < P.amax_n && n0 + wn + ni * 8 + lc * 2 + q < P.amax_n) mx = fmax(mx, fma(v.x, v.x, v.y * v.y));
            if (!(rowok[mi] && colok[ni][q])) cv[mi][ni][q] = make_double2(0.0, 0.0);
          }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) atomicMax(P.amax + batch, (unsigned long long)__double_as_longlong(mx));
    } else {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int nl = wn + ni * 8 + lc * 2 + q;
            cv[mi][ni][q] = (rowok[mi] && colok[ni][q]) ? rb[(long long)nl * P.C.ld + srow[mi]] : make_double2(0.0, 0.0);
          }
      if (CFORM && P.cz) {  // the Dyson diagonal block from H (see ZGemmProblem::cz)
        const double2 z = P.cz[batch], sgm = *P.csig;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const double2 h = cv[mi][ni][q];
              const bool dg = m0 + wm + mi * 8 + lr == n0 + wn + ni * 8 + lc * 2 + q;
              cv[mi][ni][q] = dg ? make_double2((z.x - h.x) - sgm.x, (z.y - h.y) - sgm.y) : make_double2(-h.x, -h.y);
            }
      }
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          cr[mi][ni][q] = sg * cv[mi][ni][q].x;
          ci[mi][ni][q] = sg * cv[mi][ni][q].y;
        }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  }

#pragma unroll 1
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc & 1;
    if (kc + 1 < nk)
      load_tile<PLAIN>(P, bs, batch, m0, n0, (kc + 1) * BK, As + (s ^ 1) * A_STAGE, Bs + (s ^ 1) * B_STAGE, tid);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double2* as = As + s * A_STAGE;
    const double2* bsm = Bs + s * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double ar[4], ai[4], an[4], br[4], bi[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        double2 v = as[(kk * 4 + lc) * LDA_S + wm + mi * 8 + lr];
        ar[mi] = v.x;
        ai[mi] = v.y;
        an[mi] = -v.y;
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        double2 v = bsm[(wn + ni * 8 + lr) * LDB_S + kk * 4 + lc];
        br[ni] = v.x;
        bi[ni] = v.y;
      }
      // 4 passes over the 16 sub-tiles: consecutive DMMAs never share an
      // accumulator, so the pipe never waits on its own result
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma884(cr[mi][ni], ar[mi], br[ni]);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma884(ci[mi][ni], ar[mi], bi[ni]);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma884(cr[mi][ni], an[mi], bi[ni]);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma884(ci[mi][ni], ai[mi], br[ni]);
    }
    __syncthreads();
  }

  // ---- epilogue
  const int* cmap = P.colmap ? P.colmap + (long long)batch * P.map_bstride : nullptr;
  const int* rscat = P.rowscat ? P.rowscat + (long long)batch * P.map_bstride : nullptr;
  double2* __restrict__ dbase = const_cast<double2*>(P.D.p) + (long long)batch * P.D.bstride;
  if (c_in_acc || !use_c) {  // D = alpha * acc (C already inside acc when c_in_acc)
    const double2 al = c_in_acc ? make_double2(P.alpha.x, 0.0) : P.alpha;
    if (!cmap && !rscat && m0 + BM <= P.M && n0 + BN <= P.N) {
      double2* __restrict__ dptr = dbase + toff<PLAIN>(P.D, bs, m0, n0);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int m = wm + mi * 8 + lr, n = wn + ni * 8 + lc * 2 + q;
            dptr[(long long)n * P.D.ld + m] = cmul(al, make_double2(cr[mi][ni][q], ci[mi][ni][q]));
          }
    } else {  // edge tile and/or row / column scatter (plain operand: offset = r + c*ld)
      double2* __restrict__ dt = dbase + toff<PLAIN>(P.D, bs, m0, n0);
      long long dcol[4][2];
      int drow[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int m = m0 + wm + mi * 8 + lr;
        drow[mi] = (rscat && m < P.M) ? __ldg(&rscat[m]) - m0 : m - m0;
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = n0 + wn + ni * 8 + lc * 2 + q;
          dcol[ni][q] = (n < P.N) ? (long long)(cmap ? __ldg(&cmap[n]) - n0 : n - n0) * P.D.ld : 0;
        }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int ml = wm + mi * 8 + lr;
            if (m0 + ml >= P.M || n0 + wn + ni * 8 + lc * 2 + q >= P.N) continue;
            dt[dcol[ni][q] + drow[mi]] = cmul(al, make_double2(cr[mi][ni][q], ci[mi][ni][q]));
          }
    }
  } else {  // general complex alpha / beta: D = alpha*acc + beta*C, C read in two halves
    const int* rmap = P.rowmap ? P.rowmap + (long long)batch * P.map_bstride : nullptr;
    const double2* __restrict__ cbase = P.C.p + (long long)batch * P.C.bstride;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      double2 cv[2][4][2];
#pragma unroll
      for (int mh = 0; mh < 2; ++mh)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int m = m0 + wm + (half * 2 + mh) * 8 + lr, n = n0 + wn + ni * 8 + lc * 2 + q;
            const int sr = (rmap && m < P.M) ? __ldg(&rmap[m]) : m;
            const bool z = m >= P.M || n >= P.N || sr < 0 || (m >= P.zr0 && m < P.zr1) || (n >= P.zc0 && n < P.zc1);
            cv[mh][ni][q] = z ? make_double2(0.0, 0.0) : cbase[toff<PLAIN>(P.C, bs, sr, n)];
          }
#pragma unroll
      for (int mh = 0; mh < 2; ++mh)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int mi = half * 2 + mh;
            const int m = m0 + wm + mi * 8 + lr, n = n0 + wn + ni * 8 + lc * 2 + q;
            if (m >= P.M || n >= P.N) continue;
            double2 out = cfma(P.beta, cv[mh][ni][q], cmul(P.alpha, make_double2(cr[mi][ni][q], ci[mi][ni][q])));
            dbase[toff<PLAIN>(P.D, bs, rscat ? __ldg(&rscat[m]) : m, cmap ? __ldg(&cmap[n]) : n)] = out;
          }
    }
  }
}

// One CTA per tile. (A persistent grid of 3 CTAs/SM walking the tiles with an L2
// prefetch of the next tile's C measured slower for the Gauss-Jordan updates on B200:
// 136 vs 121 ms per step.)
template <bool PLAIN, int MINB, bool AMAX = false, bool CFORM = false>
__global__ void __launch_bounds__(128, MINB) zgemm_grouped_kernel(const __grid_constant__ ZGemmGroup g) {
  extern __shared__ __align__(16) double2 smem[];
  zgemm_tile<PLAIN, AMAX, CFORM>(g, blockIdx.x, smem, smem + STAGES * A_STAGE);
}

}  // namespace

int gemm_minb() {
  static int m = [] {
    const char* e = getenv("BBSI_GEMM_MINB");
    return (e && atoi(e) == 2) ? 2 : 3;
  }();
  return m;
}

template <bool PLAIN, int MINB, bool AMAX = false, bool CFORM = false>
cudaError_t gemm_attrs() {
  return set_max_dyn_smem((const void*)zgemm_grouped_kernel<PLAIN, MINB, AMAX, CFORM>, SMEM_BYTES, true);
}

cudaError_t zgemm_grouped(ZGemmGroup& g, cudaStream_t stream) {
  int total = 0;
  bool plain = true;
  auto is_plain = [&](const ZOp& o) { return o.rs == g.bs && o.cs == (long long)g.bs * o.ld; };
  for (int p = 0; p < g.nprob; ++p) {
    ZGemmProblem& P = g.prob[p];
    if (P.M < 1 || P.N < 1 || P.K % BK || P.K < BK || g.bs % BM) return cudaErrorInvalidValue;
    P.tiles_m = (P.M + BM - 1) / BM;
    P.tiles_n = (P.N + BN - 1) / BN;
    P.tile_begin = total;
    total += P.tiles_m * P.tiles_n * g.batch;
    plain = plain && is_plain(P.A) && is_plain(P.B) && is_plain(P.C) && is_plain(P.D);
  }
  g.total_tiles = total;
  if (total == 0) return cudaSuccess;
  double fl = 0, by = 0;
  for (int p = 0; p < g.nprob; ++p) {
    const ZGemmProblem& P = g.prob[p];
    const bool rc = P.beta.x != 0.0 || P.beta.y != 0.0;
    fl += 8.0 * P.M * P.N * double(P.K) * g.batch;
    by += 16.0 * g.batch * (double(P.M) * P.K + double(P.K) * P.N + double(P.M) * P.N * (rc ? 2 : 1));
  }
  ProfScope prof(stream, g.prof_cat ? g.prof_cat : PROF_GEMM, fl, by);
  cudaError_t e;
  if (!plain) {
    bool done = false;
    if ((e = zgemm_tma_try(g, stream, &done)) || done) return e ? e : cudaGetLastError();
  }
  const bool three = gemm_minb() == 3;  // (2 CTAs/SM for the GJ updates alone: 130 vs 121 ms)
  bool amax = false, cform = false;
  for (int p = 0; p < g.nprob; ++p) {
    amax |= g.prob[p].amax != nullptr;
    cform |= g.prob[p].cz != nullptr;
  }
  if (cform) {
    if (plain) return cudaErrorInvalidValue;  // the Dyson form only feeds block-strided sweep GEMMs
    if ((e = gemm_attrs<false, 3, false, true>())) return e;
    zgemm_grouped_kernel<false, 3, false, true><<<total, 128, SMEM_BYTES, stream>>>(g);
  } else if (plain && amax) {
    if ((e = gemm_attrs<true, 3, true>())) return e;
    zgemm_grouped_kernel<true, 3, true><<<total, 128, SMEM_BYTES, stream>>>(g);
  } else if (plain && three) {
    if ((e = gemm_attrs<true, 3>())) return e;
    zgemm_grouped_kernel<true, 3><<<total, 128, SMEM_BYTES, stream>>>(g);
  } else if (plain) {
    if ((e = gemm_attrs<true, 2>())) return e;
    zgemm_grouped_kernel<true, 2><<<total, 128, SMEM_BYTES, stream>>>(g);
  } else if (three) {
    if ((e = gemm_attrs<false, 3>())) return e;
    zgemm_grouped_kernel<false, 3><<<total, 128, SMEM_BYTES, stream>>>(g);
  } else {
    if ((e = gemm_attrs<false, 2>())) return e;
    zgemm_grouped_kernel<false, 2><<<total, 128, SMEM_BYTES, stream>>>(g);
  }
  return cudaGetLastError();
}

}  // namespace bbsi_gpu

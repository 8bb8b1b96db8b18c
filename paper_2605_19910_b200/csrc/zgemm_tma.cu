// Warp-specialised DMMA GEMM with TMA operand staging (the sweep GEMMs).
//
// Same contract as zgemm_grouped (zgemm.cu, the reference's gemm_into,
// kernels.hpp:102-117): grouped, batched, block-strided complex-FP64 products
// D = alpha A B + beta C. One elected thread streams the A and B tiles into a ring
// of shared-memory stages with cp.async.bulk.tensor (TMA) and mbarrier transaction
// counts (a stage is refilled as soon as all four warps have arrived on its "empty"
// barrier); the four warps only issue DMMA (mma.sync m8n8k4 f64) and their C / D
// traffic: no per-thread cp.async address arithmetic or issue.
//
// Tensor maps. Operands are views of bs x bs slots of a few device buffers (the band,
// the multiplier arrays, the shared H); each registered buffer (tma_register) gets one
// 4-D tensor map per operand role over (8 complex = 16 doubles, column, 8-row chunk,
// slot) with strides (16 B, bs*16 B, 128 B, bs*bs*16 B), so any tile of any block of
// the buffer is one box: A tiles 64 rows x 16 columns (box {16, 16, 8, 1}), B tiles
// 16 rows x 64 columns (box {16, 64, 2, 1}).
//
// Shared memory, 128-byte swizzle. A stage holds [row chunk 8][k 16][8 complex] and B
// [k chunk 2][n 64][8 complex]; with 128-byte rows the hardware XORs the 16-byte chunk
// index with the row index mod 8. A DMMA fragment load (lane: row l/4, k l%4) then hits
// 8 distinct bank groups per quarter warp when the 8 fragment rows are taken in the
// order pi(r) = ((r & 1) << 2) | (r >> 1) (rows 2p, 2p+1 of a quarter warp differ in
// bit 2). pi is applied to the A rows (m) and to the B columns (n) of every 8 x 8
// sub-tile; the accumulators follow it (lane holds C[pi(l/4)][pi(2(l%4) + q)]).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "internal.h"

namespace bbsi_gpu {

namespace {

constexpr int TBM = 64, TBN = 64, TBK = 16;
constexpr int TSTAGE_A = TBM * TBK;  // complex
constexpr int TSTAGE_B = TBK * TBN;
constexpr int TSTAGE_BYTES = (TSTAGE_A + TSTAGE_B) * 16;
constexpr int kMaxMaps = 8;

struct TmaOp {
  int map;            // index into TmaParams::maps
  long long slot0;    // first slot of the operand (batch 0, block (0, 0))
  long long rs, cs;   // block strides in slots
  long long bst;      // batch stride in slots
};

struct TmaParams {
  CUtensorMap maps[kMaxMaps];  // 64-byte aligned (CUtensorMap is declared alignas(64))
  TmaOp a[kMaxProblems], b[kMaxProblems];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int pi8(int r) { return ((r & 1) << 2) | (r >> 1); }

// 128-byte swizzle: complex index of (row, 16-byte chunk) in a stage
__device__ __forceinline__ int swz(int row, int chunk) { return row * 8 + (chunk ^ (row & 7)); }

template <int STAGES, bool CFORM>
__global__ void __launch_bounds__(128, STAGES == 2 ? 3 : 2)
    zgemm_tma_kernel(const __grid_constant__ ZGemmGroup g, const __grid_constant__ TmaParams tp) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  // 1024-byte alignment of the stages (128-byte swizzle atoms)
  double2* stages = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + STAGES * (TSTAGE_A + TSTAGE_B));
  uint64_t* empty = full + STAGES;

  // ---- decode the tile
  const int t = blockIdx.x;
  int pi = 0;
#pragma unroll 1
  for (int q = 1; q < g.nprob; ++q)
    if (t >= g.prob[q].tile_begin) pi = q;
  const ZGemmProblem& P = g.prob[pi];
  int local = t - P.tile_begin;
  const int per_batch = P.tiles_m * P.tiles_n;
  const int batch = local / per_batch;
  local -= batch * per_batch;
  const int m0 = (local % P.tiles_m) * TBM;
  const int n0 = (local / P.tiles_m) * TBN;
  const int bs = g.bs;
  const int nk = P.K / TBK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ---------------- TMA issue (one elected thread of warp 0; no separate producer warp,
  // so the CTA keeps 128 threads and the register budget of 3 CTAs per SM)
  const TmaOp& oa = tp.a[pi];
  const TmaOp& ob = tp.b[pi];
  const CUtensorMap* ma = &tp.maps[oa.map];
  const CUtensorMap* mb = &tp.maps[ob.map];
  const long long abase = oa.slot0 + (long long)batch * oa.bst + (long long)(m0 / bs) * oa.rs;
  const long long bbase = ob.slot0 + (long long)batch * ob.bst + (long long)(n0 / bs) * ob.cs;
  const int am = (m0 % bs) / 8, bn = n0 % bs;
  auto issue = [&](int kc) {
    const int s = kc % STAGES;
    mbar_expect_tx(&full[s], TSTAGE_BYTES);
    const int k0 = kc * TBK;
    double2* As = stages + s * (TSTAGE_A + TSTAGE_B);
    double2* Bs = As + TSTAGE_A;
    tma_load_4d(As, ma, 0, k0 % bs, am, int(abase + (long long)(k0 / bs) * oa.cs), &full[s]);
    tma_load_4d(Bs, mb, 0, bn, (k0 % bs) / 8, int(bbase + (long long)(k0 / bs) * ob.rs), &full[s]);
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(ma)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(mb)) : "memory");
    for (int kc = 0; kc < STAGES && kc < nk; ++kc) issue(kc);
  }

  // ---------------- consumers: 4 warps of 32 x 32
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int lr = lane >> 2, lc = lane & 3;
  const int pr = pi8(lr);                       // this lane's fragment row (A) / column (B) in 8
  const int pc0 = pi8(2 * lc), pc1 = pi8(2 * lc + 1);  // this lane's two accumulator columns
  double cr[4][4][2], ci[4][4][2];

  const bool use_c = (P.beta.x != 0.0 || P.beta.y != 0.0);
  const bool c_in_acc = use_c && P.beta.x == 1.0 && P.beta.y == 0.0 && P.alpha.y == 0.0 &&
                        (P.alpha.x == 1.0 || P.alpha.x == -1.0);
  if (c_in_acc) {
    const double2* __restrict__ ct = P.C.p + (long long)batch * P.C.bstride + zop_offset(P.C, bs, m0, n0);
    const double sg = P.alpha.x;
    const double2 z = (CFORM && P.cz) ? P.cz[batch] : make_double2(0.0, 0.0);
    const double2 sgm = (CFORM && P.cz) ? *P.csig : make_double2(0.0, 0.0);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int m = wm + mi * 8 + pr, n = wn + ni * 8 + (q ? pc1 : pc0);
          double2 v = ct[(long long)n * P.C.ld + m];
          if (CFORM && P.cz)  // the Dyson diagonal block from H (see ZGemmProblem::cz)
            v = (m0 + m == n0 + n) ? make_double2((z.x - v.x) - sgm.x, (z.y - v.y) - sgm.y) : make_double2(-v.x, -v.y);
          cr[mi][ni][q] = sg * v.x;
          ci[mi][ni][q] = sg * v.y;
        }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  }

  // smem offsets (complex) of this lane's fragments inside a stage, per (sub-tile, kk)
  // A: row = (wm/8 + mi)*16 + k, chunk = pr;  B: row = (k/8)*64 + wn + ni*8 + pr, chunk = k%8
#pragma unroll 1
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc % STAGES;
    mbar_wait(&full[s], (kc / STAGES) & 1);
    const double2* as = stages + s * (TSTAGE_A + TSTAGE_B);
    const double2* bsm = as + TSTAGE_A;
#pragma unroll
    for (int kk = 0; kk < TBK / 4; ++kk) {
      const int k = kk * 4 + lc;
      double ar[4], ai[4], an[4], br[4], bi[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const double2 v = as[swz((wm / 8 + mi) * 16 + k, pr)];
        ar[mi] = v.x;
        ai[mi] = v.y;
        an[mi] = -v.y;
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const double2 v = bsm[swz((k >> 3) * 64 + wn + ni * 8 + pr, k & 7)];
        br[ni] = v.x;
        bi[ni] = v.y;
      }
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && kc + STAGES < nk) {  // refill this stage once all 4 warps left it
      mbar_wait(&empty[s], (kc / STAGES) & 1);
      issue(kc + STAGES);
    }
  }

  // ---- epilogue (full tiles only on this path)
  double2* __restrict__ dptr =
      const_cast<double2*>(P.D.p) + (long long)batch * P.D.bstride + zop_offset(P.D, bs, m0, n0);
  if (c_in_acc || !use_c) {
    const double2 al = c_in_acc ? make_double2(P.alpha.x, 0.0) : P.alpha;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int m = wm + mi * 8 + pr, n = wn + ni * 8 + (q ? pc1 : pc0);
          dptr[(long long)n * P.D.ld + m] = cmul(al, make_double2(cr[mi][ni][q], ci[mi][ni][q]));
        }
  } else {
    const double2* __restrict__ cbase = P.C.p + (long long)batch * P.C.bstride + zop_offset(P.C, bs, m0, n0);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int m = wm + mi * 8 + pr, n = wn + ni * 8 + (q ? pc1 : pc0);
          const double2 c = cbase[(long long)n * P.C.ld + m];
          dptr[(long long)n * P.D.ld + m] = cfma(P.beta, c, cmul(P.alpha, make_double2(cr[mi][ni][q], ci[mi][ni][q])));
        }
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

struct TmaBuf {
  const char* base = nullptr;
  size_t bytes = 0;
  int bs = 0;
  int dev = -1;
  CUtensorMap ma, mb;
};
thread_local std::vector<TmaBuf> t_cache;     // encoded maps (grow-only, small)
thread_local std::vector<int> t_registered;   // indices into t_cache, innermost scope last

bool encode(TmaBuf& e) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t bb = (cuuint64_t)e.bs * e.bs;
  const cuuint64_t nslot = e.bytes / (bb * 16);
  if (nslot == 0 || nslot > 0x7fffffffULL) return false;
  const cuuint64_t dims[4] = {16, (cuuint64_t)e.bs, (cuuint64_t)e.bs / 8, nslot};
  const cuuint64_t strides[3] = {(cuuint64_t)e.bs * 16, 128, bb * 16};  // bytes, dims 1..3
  const cuuint32_t elem[4] = {1, 1, 1, 1};
  const cuuint32_t boxa[4] = {16, TBK, TBM / 8, 1};
  const cuuint32_t boxb[4] = {16, TBN, TBK / 8, 1};
  void* gp = const_cast<char*>(e.base);
  CUresult r1 = fn(&e.ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, gp, dims, strides, boxa, elem,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = fn(&e.mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, gp, dims, strides, boxb, elem,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r1 == CUDA_SUCCESS && r2 == CUDA_SUCCESS;
}

bool tma_enabled() {  // read per call (tests compare BBSI_TMA=0 / 1 in one process)
  const char* e = getenv("BBSI_TMA");
  return !(e && atoi(e) == 0);
}

int tma_stages() {
  static const int s = [] {
    const char* e = getenv("BBSI_TMA_STAGES");
    const int v = e ? atoi(e) : 2;
    return v == 3 || v == 4 ? v : 2;
  }();
  return s;
}

// the registered buffer holding [p, p + extent) at a slot boundary, or -1
int find_buf(const void* p, size_t extent, int bs) {
  const char* c = static_cast<const char*>(p);
  for (int i = int(t_registered.size()) - 1; i >= 0; --i) {
    const TmaBuf& e = t_cache[t_registered[i]];
    if (e.bs != bs || c < e.base || c + extent > e.base + e.bytes) continue;
    if ((size_t(c - e.base) % (size_t(bs) * bs * 16)) != 0) continue;
    return t_registered[i];
  }
  return -1;
}

}  // namespace

void tma_register(const void* base, size_t bytes, int bs) {
  if (!tma_enabled() || !base || bytes == 0 || bs % 64) return;
  int dev = 0;
  cudaGetDevice(&dev);
  int idx = -1;
  for (size_t i = 0; i < t_cache.size(); ++i)
    if (t_cache[i].base == base && t_cache[i].bytes == bytes && t_cache[i].bs == bs && t_cache[i].dev == dev) {
      idx = int(i);
      break;
    }
  if (idx < 0) {
    TmaBuf e;
    e.base = static_cast<const char*>(base);
    e.bytes = bytes;
    e.bs = bs;
    e.dev = dev;
    if (!encode(e)) return;
    if (t_cache.size() >= 64) t_cache.erase(t_cache.begin());  // keep the cache small
    t_cache.push_back(e);
    idx = int(t_cache.size()) - 1;
  }
  t_registered.push_back(idx);
}

void tma_unregister(int n) {
  while (n-- > 0 && !t_registered.empty()) t_registered.pop_back();
}

// Launches g on the TMA kernel when every problem qualifies (full 64 x 64 tiles, A / B
// views of registered buffers with ld = bs, no Gauss-Jordan remaps); *done = false
// otherwise (the caller falls back to the cp.async kernel).
cudaError_t zgemm_tma_try(const ZGemmGroup& g, cudaStream_t stream, bool* done) {
  *done = false;
  if (!tma_enabled() || t_registered.empty()) return cudaSuccess;
  TmaParams tp;
  std::vector<int> used;
  auto map_of = [&](int buf) {
    for (size_t i = 0; i < used.size(); ++i)
      if (used[i] == buf) return int(i);
    if (int(used.size()) >= kMaxMaps) return -1;
    used.push_back(buf);
    return int(used.size()) - 1;
  };
  bool cform = false;
  const long long bb = (long long)g.bs * g.bs;
  for (int p = 0; p < g.nprob; ++p) {
    const ZGemmProblem& P = g.prob[p];
    if (P.M % TBM || P.N % TBN || P.K % TBK || P.rowmap || P.colmap || P.rowscat || P.amax || P.zr1 > P.zr0 ||
        P.zc1 > P.zc0)
      return cudaSuccess;
    const bool use_c = P.beta.x != 0.0 || P.beta.y != 0.0;
    if (P.A.ld != g.bs || P.B.ld != g.bs || (use_c && P.C.ld != g.bs) || P.D.ld != g.bs) return cudaSuccess;
    if (P.A.rs % bb || P.A.cs % bb || P.B.rs % bb || P.B.cs % bb || P.A.bstride % bb || P.B.bstride % bb)
      return cudaSuccess;
    cform |= P.cz != nullptr;
    // operand extents: the lowest and highest slot any tile reaches
    auto span = [&](const ZOp& o, int rows, int cols, const char** lo, size_t* ext) {
      long long mn = 0, mx = 0;
      const long long rb = rows / g.bs - 1, cb = cols / g.bs - 1, e = g.batch - 1;
      for (long long v : {rb * o.rs, 0LL}) {
        for (long long w : {cb * o.cs, 0LL}) {
          for (long long u : {e * o.bstride, 0LL}) {
            mn = std::min(mn, v + w + u);
            mx = std::max(mx, v + w + u);
          }
        }
      }
      *lo = reinterpret_cast<const char*>(o.p + mn);
      *ext = size_t(mx - mn + bb) * 16;
    };
    for (int which = 0; which < 2; ++which) {
      const ZOp& o = which ? P.B : P.A;
      const char* lo;
      size_t ext;
      span(o, which ? P.K : P.M, which ? P.N : P.K, &lo, &ext);
      const int buf = find_buf(lo, ext, g.bs);
      if (buf < 0) return cudaSuccess;
      const int mi = map_of(buf);
      if (mi < 0) return cudaSuccess;
      TmaOp& to = which ? tp.b[p] : tp.a[p];
      to.map = mi;
      to.slot0 = (reinterpret_cast<const char*>(o.p) - t_cache[buf].base) / (bb * 16);
      to.rs = o.rs / bb;
      to.cs = o.cs / bb;
      to.bst = o.bstride / bb;
    }
  }
  // maps[2i] = A-box, maps[2i+1] = B-box map of buffer used[i]
  if (int(used.size()) * 2 > kMaxMaps) return cudaSuccess;
  for (size_t i = 0; i < used.size(); ++i) {
    tp.maps[2 * i] = t_cache[used[i]].ma;
    tp.maps[2 * i + 1] = t_cache[used[i]].mb;
  }
  for (int p = 0; p < g.nprob; ++p) {
    tp.a[p].map = 2 * tp.a[p].map;
    tp.b[p].map = 2 * tp.b[p].map + 1;
  }
  const int stages = tma_stages();
  const size_t smem = size_t(stages) * TSTAGE_BYTES + 2 * stages * sizeof(uint64_t) + 1024;
  cudaError_t e;
  const void* fn = nullptr;
  if (stages == 2)
    fn = cform ? (const void*)zgemm_tma_kernel<2, true> : (const void*)zgemm_tma_kernel<2, false>;
  else if (stages == 4)
    fn = cform ? (const void*)zgemm_tma_kernel<4, true> : (const void*)zgemm_tma_kernel<4, false>;
  else
    fn = cform ? (const void*)zgemm_tma_kernel<3, true> : (const void*)zgemm_tma_kernel<3, false>;
  if ((e = set_max_dyn_smem(fn, smem, true))) return e;
  void* args[2] = {const_cast<ZGemmGroup*>(&g), &tp};
  if ((e = cudaLaunchKernel(fn, dim3(g.total_tiles), dim3(128), args, smem, stream))) return e;
  *done = true;
  return cudaSuccess;
}

}  // namespace bbsi_gpu

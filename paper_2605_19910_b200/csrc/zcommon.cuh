// Shared definitions for the complex-FP64 block kernels (sm_100a).
//
// Storage: every block is bs x bs complex128, column-major, (re, im) interleaved,
// exactly the reference DenseMatrix<std::complex<double>> layout (dense.hpp:28-50).
// bs is the padded slot size (a multiple of 64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bbsi_gpu {

// Logical operand made of bs x bs blocks that are not necessarily contiguous:
// element (r, c) lives at p + bstride*batch + (r/bs)*rs + (c/bs)*cs + (c%bs)*ld + r%bs.
// With rs/cs expressed in slots of the band storage, one descriptor covers the
// k x k windows of the n-diagonal recursion (rgf.hpp:107-112,122-134).
struct ZOp {
  const double2* p;
  long long ld;
  long long rs;
  long long cs;
  long long bstride;
};

struct ZGemmProblem {
  int M, N, K;          // logical sizes; K % 16 == 0, M/N arbitrary (masked edge tiles)
  double2 alpha, beta;  // D = alpha * A*B + beta * C
  ZOp A, B, C;          // C may be ignored when beta == 0
  ZOp D;                // output operand (p is written)
  // optional epilogue remaps (plain single-block operands; used by the blocked
  // Gauss-Jordan inversion): C row r is read from row rowmap[r] (a negative entry
  // reads 0); C is taken as 0 for rows [zr0, zr1) and columns [zc0, zc1); D row r /
  // column c is written to row rowscat[r] / column colmap[c].
  const int* rowmap;
  const int* colmap;
  const int* rowscat;
  long long map_bstride;
  int zr0, zr1, zc0, zc1;
  // optional (C-as-accumulator path, plain operands, identity row map): atomicMax of
  // max |C_ij|^2 (as double bits) over the tile's entries of C as stored, row, column
  // < amax_n, masked ones included, into amax[batch] (the first Gauss-Jordan step)
  unsigned long long* amax;
  int amax_n;
  // optional (C-as-accumulator path): C holds H (a diagonal block shared by the batch,
  // bstride 0) and the GEMM reads A = z I - H - sigma I from it, entry by entry as
  // dyson_form_diag does: diagonal (z - h) - sigma, elsewhere -h; z = cz[batch], sigma = *csig
  const double2* cz;
  const double2* csig;
  int tiles_m, tiles_n; // filled by the launcher
  int tile_begin;       // first flattened tile index of this problem
};

constexpr int kMaxProblems = 6;

struct ZGemmGroup {
  ZGemmProblem prob[kMaxProblems];
  int nprob;
  int batch;
  int bs;
  int total_tiles;      // sum over problems of tiles_m * tiles_n * batch
  int prof_cat;         // profiling category of the launch (0 = main GEMM)
};

__host__ __device__ inline long long zop_offset(const ZOp& o, int bs, int r, int c) {
  return (long long)(r / bs) * o.rs + (long long)(c / bs) * o.cs + (long long)(c % bs) * o.ld + (r % bs);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // c + a*b
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
// Reciprocal with the same scaling idea as LAPACK zladiv / Smith's algorithm.
__device__ __forceinline__ double2 crcp(double2 a) {
  if (fabs(a.x) >= fabs(a.y)) {
    if (a.x == 0.0 && a.y == 0.0) return make_double2(0.0, 0.0);
    double r = a.y / a.x, d = a.x + a.y * r;
    return make_double2(1.0 / d, -r / d);
  } else {
    double r = a.x / a.y, d = a.x * r + a.y;
    return make_double2(r / d, -1.0 / d);
  }
}

// Division-free reciprocal of a nonzero complex: conj(a) * (1/|a|^2) with |a|^2
// formed after scaling by a power of two (exact) to avoid over/underflow; 1/x by
// the MUFU seed plus two Newton steps (~1 ulp). Zero maps to zero.
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double2 crcp_fast(double2 a) {
  const double m = fmax(fabs(a.x), fabs(a.y));
  if (m == 0.0) return make_double2(0.0, 0.0);
  int ex;
  frexp(m, &ex);
  const double sc = ldexp(1.0, -ex);  // power of two: exact scaling
  const double xr = a.x * sc, xi = a.y * sc;
  const double inv = rcp_nr(fma(xr, xr, xi * xi)) * sc;
  return make_double2(xr * inv, -xi * inv);
}

// crcp_fast without branches or library calls (every lane of a warp can run it next to
// independent work): the power-of-two scale comes from the exponent bits of max(|re|, |im|)
// (scaled to [1, 2) instead of frexp's [0.5, 1): both scalings are exact, so the result has
// the same bits as crcp_fast for normal inputs). Zero maps to zero.
__device__ __forceinline__ double2 crcp_lanes(double2 a) {
  const double m = fmax(fabs(a.x), fabs(a.y));
  const long long e = (__double_as_longlong(m) >> 52) & 0x7ff;
  const double sc = __longlong_as_double((0x7feLL - e) << 52);
  const double xr = a.x * sc, xi = a.y * sc;
  const double inv = rcp_nr(fma(xr, xr, xi * xi)) * sc;
  const bool z = m == 0.0;
  return make_double2(z ? 0.0 : xr * inv, z ? 0.0 : -xi * inv);
}

// DMMA: D(8x8) += A(8x4, row) * B(4x8, col), FP64. One lane holds A[l/4][l%4],
// B[l%4][l/4] and C[l/4][2*(l%4) + {0,1}].
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace bbsi_gpu

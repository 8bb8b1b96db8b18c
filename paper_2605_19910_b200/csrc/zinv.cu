// Batched in-place inversion of bs x bs complex128 blocks by blocked Gauss-Jordan
// elimination with partial (row) pivoting.
//
// Replaces, per Schur pivot, the reference's lu_factor + invert pair
// (kernels.hpp:140-160 zgetrf with the negligible-pivot test, kernels.hpp:192-195
// zgetrs against the identity) and lets solve_left / solve_right
// (kernels.hpp:163-189) become plain GEMMs with the explicit inverse.
//
// Algorithm (one CTA per matrix, panels of NB=16 columns):
//   for each panel K = [k, k+16):
//     1. tall-panel LU with partial pivoting (|re|+|im| pivot choice, like izamax)
//        on rows k..n-1, in shared memory; pivots identical to zgetrf's;
//     2. apply the 16 row interchanges to the rest of the matrix;
//     3. Pinv = (L_PP U)^{-1} (16 x 16);
//     4. Wz = old M[:,K] with the pivot rows zeroed (global scratch);
//     5. pivot rows: M[P,:] <- Pinv * M[P,:], M[P,K] <- Pinv;
//     6. rank-16 update M[R,:] -= Wz[R] * M[P,:] on DMMA, R = all non-pivot rows
//        (this also produces M[R,K] = -Wz Pinv because M[R,K] was zeroed).
//   finally undo the row interchanges as column interchanges in reverse order.
// The diagonal of U is checked against eps * n * max|A| (|.| = hypot), exactly the
// reference's threshold (kernels.hpp:149-158); the first failing column is
// reported per matrix in status[] (-1 when regular).
#include <cfloat>
#include <climits>

#include "internal.h"

namespace bbsi_gpu {

namespace {

constexpr int NB = 16;
constexpr int NT = 256;
constexpr int T_LDA = 64 + 2;  // update tiles: As[t][m]
constexpr int T_LDB = NB + 4;  // Bs[n][t]

__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__global__ void __launch_bounds__(NT, 1)
    zinv_gj_kernel(double2* __restrict__ M0, long long ld, long long bstride, int n, int n_true,
                   int* __restrict__ piv0, double2* __restrict__ wz0, int* __restrict__ status) {
  extern __shared__ __align__(16) double2 sm[];
  const int ldp = n + 1;
  double2* Pn = sm;                      // NB columns x n rows (panel), ld = n+1
  double2* Pinv = sm + NB * ldp;         // 16 x 17
  double2* As = sm;                      // update tiles overlay the panel
  double2* Bs = sm + NB * T_LDA;
  __shared__ double red_v[NT / 32];
  __shared__ int red_i[NT / 32];
  __shared__ int s_piv[NB];
  __shared__ int s_fail;
  __shared__ double s_tol;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2* M = M0 + (long long)blockIdx.x * bstride;
  int* piv = piv0 + (long long)blockIdx.x * n;
  double2* Wz = wz0 + (long long)blockIdx.x * n * NB;

  // ---- 0. threshold eps * n * max|A| over the true (unpadded) block
  {
    double mx = 0.0;
    for (int idx = tid; idx < n_true * n_true; idx += NT) {
      int r = idx % n_true, c = idx / n_true;
      double2 v = M[(long long)c * ld + r];
      mx = fmax(mx, hypot(v.x, v.y));
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red_v[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double m = 0.0;
      for (int w = 0; w < NT / 32; ++w) m = fmax(m, red_v[w]);
      s_tol = DBL_EPSILON * double(n_true) * m;
      s_fail = INT_MAX;
    }
    __syncthreads();
  }
  const double tol = s_tol;

#pragma unroll 1
  for (int k = 0; k < n; k += NB) {
    const int rows = n - k;
    // ---- 1. load the panel (rows k..n-1 of columns k..k+15)
    for (int idx = tid; idx < NB * rows; idx += NT) {
      int c = idx / rows, r = idx - c * rows;
      Pn[c * ldp + r] = M[(long long)(k + c) * ld + k + r];
    }
    __syncthreads();

    // ---- panel LU with partial pivoting
#pragma unroll 1
    for (int j = 0; j < NB; ++j) {
      double bv = -1.0;
      int bi = INT_MAX;
      for (int r = j + tid; r < rows; r += NT) {
        double v = cabs1(Pn[j * ldp + r]);
        if (v > bv) {
          bv = v;
          bi = r;
        }
      }
      for (int o = 16; o; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        argmax_merge(bv, bi, v2, i2);
      }
      if (lane == 0) {
        red_v[warp] = bv;
        red_i[warp] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double v = red_v[0];
        int i = red_i[0];
        for (int w = 1; w < NT / 32; ++w) argmax_merge(v, i, red_v[w], red_i[w]);
        if (i == INT_MAX) i = j;
        s_piv[j] = i;
        piv[k + j] = k + i;
      }
      __syncthreads();
      const int p = s_piv[j];
      if (p != j && tid < NB) {
        double2 x = Pn[tid * ldp + j];
        Pn[tid * ldp + j] = Pn[tid * ldp + p];
        Pn[tid * ldp + p] = x;
      }
      __syncthreads();
      const double2 pv = Pn[j * ldp + j];
      if (tid == 0 && k + j < n_true && hypot(pv.x, pv.y) <= tol) s_fail = min(s_fail, k + j);
      const double2 inv = crcp(pv);
      for (int r = j + 1 + tid; r < rows; r += NT) {
        double2 l = cmul(Pn[j * ldp + r], inv);
        Pn[j * ldp + r] = l;
#pragma unroll 4
        for (int c = j + 1; c < NB; ++c) Pn[c * ldp + r] = csub(Pn[c * ldp + r], cmul(l, Pn[c * ldp + j]));
      }
      __syncthreads();
    }

    // ---- 2. row interchanges outside the panel columns
    for (int c = tid; c < n; c += NT) {
      if (c >= k && c < k + NB) continue;
      double2* col = M + (long long)c * ld;
#pragma unroll 1
      for (int j = 0; j < NB; ++j) {
        int p = k + s_piv[j];
        if (p != k + j) {
          double2 x = col[k + j];
          col[k + j] = col[p];
          col[p] = x;
        }
      }
    }

    // ---- 3. Pinv = U^{-1} L^{-1} of the 16 x 16 pivot block (one column per thread)
    if (tid < NB) {
      const int c = tid;
      double2 t[NB];
#pragma unroll
      for (int r = 0; r < NB; ++r) t[r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
#pragma unroll
      for (int r = 1; r < NB; ++r) {
        double2 s = t[r];
#pragma unroll
        for (int q = 0; q < r; ++q) s = csub(s, cmul(Pn[q * ldp + r], t[q]));
        t[r] = s;
      }
#pragma unroll
      for (int r = NB - 1; r >= 0; --r) {
        double2 s = t[r];
#pragma unroll
        for (int q = r + 1; q < NB; ++q) s = csub(s, cmul(Pn[q * ldp + r], t[q]));
        t[r] = cmul(s, crcp(Pn[r * ldp + r]));
      }
#pragma unroll
      for (int r = 0; r < NB; ++r) Pinv[c * 17 + r] = t[r];
    }

    // ---- 4. Wz = current M[:,K] (rows in post-interchange order), pivot rows zero.
    //      Rows >= k still hold pre-interchange panel values in global memory.
    for (int r = tid; r < n; r += NT) {
      int src = r;
      if (r >= k) {
#pragma unroll 1
        for (int j = NB - 1; j >= 0; --j) {
          int p = k + s_piv[j];
          if (src == k + j) src = p;
          else if (src == p) src = k + j;
        }
      }
      const bool prow = (r >= k && r < k + NB);
#pragma unroll 4
      for (int c = 0; c < NB; ++c)
        Wz[(long long)c * n + r] = prow ? make_double2(0.0, 0.0) : M[(long long)(k + c) * ld + src];
    }
    __syncthreads();
    for (int r = tid; r < n; r += NT) {
      if (r >= k && r < k + NB) continue;
#pragma unroll 4
      for (int c = 0; c < NB; ++c) M[(long long)(k + c) * ld + r] = make_double2(0.0, 0.0);
    }

    // ---- 5. pivot rows: M[P,c] <- Pinv * M[P,c];  M[P,K] <- Pinv
    for (int c = tid; c < n; c += NT) {
      double2* col = M + (long long)c * ld + k;
      if (c >= k && c < k + NB) {
#pragma unroll
        for (int r = 0; r < NB; ++r) col[r] = Pinv[(c - k) * 17 + r];
      } else {
        double2 x[NB];
#pragma unroll
        for (int r = 0; r < NB; ++r) x[r] = col[r];
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          double2 s = make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < NB; ++q) s = cfma(Pinv[q * 17 + r], x[q], s);
          col[r] = s;
        }
      }
    }
    __syncthreads();

    // ---- 6. rank-16 update of every non-pivot row on DMMA: M -= Wz * M[P,:]
    {
      const int wm = (warp & 1) * 32;   // 2 x 4 warps, warp tile 32 x 16
      const int wn = (warp >> 1) * 16;
      const int lr = lane >> 2, lc = lane & 3;
      const int nt = n / 64;
#pragma unroll 1
      for (int tile = 0; tile < nt * nt; ++tile) {
        const int m0 = (tile % nt) * 64, n0 = (tile / nt) * 64;
        for (int idx = tid; idx < 64 * NB; idx += NT) {
          int m = idx & 63, t = idx >> 6;
          double2 v = Wz[(long long)t * n + m0 + m];
          As[t * T_LDA + m] = make_double2(-v.x, -v.y);
        }
        for (int idx = tid; idx < 64 * NB; idx += NT) {
          int t = idx & (NB - 1), nn = idx >> 4;
          Bs[nn * T_LDB + t] = M[(long long)(n0 + nn) * ld + k + t];
        }
        __syncthreads();
        double cr[4][2][2], ci[4][2][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int m = m0 + wm + mi * 8 + lr, c = n0 + wn + ni * 8 + lc * 2 + q;
              double2 v = M[(long long)c * ld + m];
              cr[mi][ni][q] = v.x;
              ci[mi][ni][q] = v.y;
            }
#pragma unroll
        for (int kk = 0; kk < NB / 4; ++kk) {
          double ar[4], ai[4], an[4], br[2], bi[2];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            double2 v = As[(kk * 4 + lc) * T_LDA + wm + mi * 8 + lr];
            ar[mi] = v.x;
            ai[mi] = v.y;
            an[mi] = -v.y;
          }
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            double2 v = Bs[(wn + ni * 8 + lr) * T_LDB + kk * 4 + lc];
            br[ni] = v.x;
            bi[ni] = v.y;
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) {
              dmma884(cr[mi][ni], ar[mi], br[ni]);
              dmma884(ci[mi][ni], ar[mi], bi[ni]);
              dmma884(cr[mi][ni], an[mi], bi[ni]);
              dmma884(ci[mi][ni], ai[mi], br[ni]);
            }
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int m = m0 + wm + mi * 8 + lr;
          if (m >= k && m < k + NB) continue;
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int c = n0 + wn + ni * 8 + lc * 2 + q;
              M[(long long)c * ld + m] = make_double2(cr[mi][ni][q], ci[mi][ni][q]);
            }
        }
        __syncthreads();
      }
    }
  }

  // ---- undo the interchanges: column swaps in reverse order
#pragma unroll 1
  for (int j = n - 1; j >= 0; --j) {
    const int p = piv[j];
    if (p != j) {
      double2* a = M + (long long)j * ld;
      double2* b = M + (long long)p * ld;
      for (int r = tid; r < n; r += NT) {
        double2 x = a[r];
        a[r] = b[r];
        b[r] = x;
      }
    }
    __syncthreads();
  }
  if (tid == 0) status[blockIdx.x] = (s_fail == INT_MAX) ? -1 : s_fail;
}

}  // namespace

size_t zinv_smem_bytes(int n) {
  size_t panel = size_t(NB) * (n + 1) * sizeof(double2);
  size_t tiles = size_t(NB * T_LDA + 64 * T_LDB) * sizeof(double2);
  return (panel > tiles ? panel : tiles) + 16 * 17 * sizeof(double2) + 64;
}

size_t zinv_scratch_bytes(int n) { return size_t(n) * NB * sizeof(double2); }

cudaError_t zinv_batched(double2* M, long long ld, long long bstride, int n, int n_true, int batch, int* piv,
                         double2* wz, int* status, cudaStream_t stream) {
  if (n % 64 || n_true > n || n_true < 1) return cudaErrorInvalidValue;
  size_t smem = zinv_smem_bytes(n);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(zinv_gj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  if (batch == 0) return cudaSuccess;
  ProfScope prof(stream, PROF_INV, 8.0 * double(n) * n * n * batch, 32.0 * double(n) * n * batch);
  zinv_gj_kernel<<<batch, NT, smem, stream>>>(M, ld, bstride, n, n_true, piv, wz, status);
  return cudaGetLastError();
}

}  // namespace bbsi_gpu

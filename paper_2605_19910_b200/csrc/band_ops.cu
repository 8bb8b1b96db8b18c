// Band-level elementwise kernels: Dyson-matrix synthesis on the device and the
// formation of the per-energy working band A(E) = z I - H - Sigma from a shared H.
#include "dyson_gen.h"
#include "internal.h"

namespace bbsi_gpu {

namespace {

// H slots [rows][2w+1][b*b] for the global layers a0 .. a0+rows-1 of an l-layer band
// (b = slot size, blocks fill the whole slot).
__global__ void dyson_fill_h_kernel(double2* H, int l, int w, int b, uint64_t seedmix, int a0, int rows) {
  const long long bb = (long long)b * b;
  const long long total = (long long)rows * (2 * w + 1) * bb;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long slot = idx / bb;
    long long e = idx - slot * bb;
    int a = a0 + int(slot / (2 * w + 1));
    int off = int(slot % (2 * w + 1)) - w;
    int i = int(e % b), j = int(e / b);
    double re = 0.0, im = 0.0;
    if (a + off >= 0 && a + off < l) bbsi_h_entry(seedmix, b, a, off, i, j, &re, &im);
    H[idx] = make_double2(re, im);
  }
}

// G[e] = -H (full band), diagonal entries += z_e - sigma_a:
//   re = (E - h_re) - s_re,  im = (eta - h_im) - s_im   (fixed operation order).
__global__ void dyson_form_band_kernel(double2* __restrict__ G, const double2* __restrict__ H, int l, int w, int bs,
                                       int batch, const double2* __restrict__ z, const double2* __restrict__ sigma) {
  const long long bb = (long long)bs * bs;
  const long long band = (long long)l * (2 * w + 1) * bb;
  const long long total = band * batch;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long e = idx / band;
    long long r = idx - e * band;
    long long slot = r / bb;
    long long q = r - slot * bb;
    int off = int(slot % (2 * w + 1)) - w;
    double2 h = H[r];
    double2 out;
    if (off == 0 && (q % bs) == (q / bs)) {
      int a = int(slot / (2 * w + 1));
      double2 ze = z[e], sg = sigma[a];
      out = make_double2((ze.x - h.x) - sg.x, (ze.y - h.y) - sg.y);
    } else {
      out = make_double2(-h.x, -h.y);
    }
    G[idx] = out;
  }
}

// Diagonal slots of every band (energy e, layer a) from H, the two out-of-range
// off-diagonal slots of each band zeroed; in-range off-diagonal slots are left for
// the downward sweep to fill with G.
// sel0 >= 0: only the diagonal blocks of layers sel0 (and sel1 >= 0) are formed (the
// sweeps read the others' A from H inside the GEMM that first updates them).
__global__ void dyson_form_diag_kernel(double2* __restrict__ G, const double2* __restrict__ H, int l, int w, int bs,
                                       int batch, const double2* __restrict__ z, const double2* __restrict__ sigma,
                                       int sel0, int sel1) {
  const long long bb = (long long)bs * bs;
  const long long band = (long long)l * (2 * w + 1) * bb;
  const int nd = sel0 < 0 ? l : (sel1 < 0 ? 1 : 2);  // diagonal blocks formed per energy
  const long long per = (long long)(nd + 2 * w) * bb;  // + 2w edge slots per energy
  const long long total = per * batch;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long e = idx / per;
    const long long r = idx - e * per;
    const long long blk = r / bb, q = r - blk * bb;
    if (blk < nd) {  // diagonal block of layer a
      const long long a = sel0 < 0 ? blk : (blk == 0 ? sel0 : sel1);
      const long long src = (a * (2 * w + 1) + w) * bb + q;
      const double2 h = H[src];
      double2 out = make_double2(-h.x, -h.y);
      if ((q % bs) == (q / bs)) {
        const double2 ze = z[e], sg = sigma[a];
        out = make_double2((ze.x - h.x) - sg.x, (ze.y - h.y) - sg.y);
      }
      G[e * band + src] = out;
    } else {  // edge slots: layer 0 offsets -w..-1, layer l-1 offsets 1..w
      const int t = int(blk - nd);
      const long long slot = t < w ? (long long)t : (long long)(l - 1) * (2 * w + 1) + w + 1 + (t - w);
      G[e * band + slot * bb + q] = make_double2(0.0, 0.0);
    }
  }
}

int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  if (g > 148LL * 32) g = 148LL * 32;
  return int(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t dyson_fill_h(double2* H, int l, int w, int b, uint64_t seed, cudaStream_t s) {
  return dyson_fill_h_rows(H, l, w, b, seed, 0, l, s);
}

cudaError_t dyson_fill_h_rows(double2* H, int l, int w, int b, uint64_t seed, int a0, int a1, cudaStream_t s) {
  long long total = (long long)(a1 - a0) * (2 * w + 1) * b * b;
  if (total <= 0) return cudaSuccess;
  ProfScope prof(s, PROF_BAND, 0.0, 16.0 * total);
  dyson_fill_h_kernel<<<grid_for(total, 256), 256, 0, s>>>(H, l, w, b, bbsi_mix64(seed), a0, a1 - a0);
  return cudaGetLastError();
}

cudaError_t dyson_form_diag(double2* G, const double2* H, int l, int w, int bs, int batch, const double2* z,
                            const double2* sigma, cudaStream_t s) {
  const long long total = (long long)(l + 2 * w) * bs * bs * batch;
  ProfScope prof(s, PROF_BAND, 0.0, 16.0 * (total + (long long)l * bs * bs));
  dyson_form_diag_kernel<<<grid_for(total, 256), 256, 0, s>>>(G, H, l, w, bs, batch, z, sigma, -1, -1);
  return cudaGetLastError();
}

cudaError_t dyson_form_diag_ends(double2* G, const double2* H, int l, int w, int bs, int batch, const double2* z,
                                 const double2* sigma, bool first, cudaStream_t s) {
  const int a0 = l - 1, a1 = (first && l > 1) ? 0 : -1;
  const long long total = (long long)((a1 >= 0 ? 2 : 1) + 2 * w) * bs * bs * batch;
  ProfScope prof(s, PROF_BAND, 0.0, 16.0 * total);
  dyson_form_diag_kernel<<<grid_for(total, 256), 256, 0, s>>>(G, H, l, w, bs, batch, z, sigma, a0, a1);
  return cudaGetLastError();
}

cudaError_t dyson_form_band(double2* G, const double2* H, int l, int w, int bs, int batch, const double2* z,
                            const double2* sigma, cudaStream_t s) {
  long long total = (long long)l * (2 * w + 1) * bs * bs * batch;
  ProfScope prof(s, PROF_BAND, 0.0, 16.0 * (total + (long long)l * (2 * w + 1) * bs * bs));
  dyson_form_band_kernel<<<grid_for(total, 256), 256, 0, s>>>(G, H, l, w, bs, batch, z, sigma);
  return cudaGetLastError();
}


namespace {
// Dense window <-> band slots: D (batch x [wb x wb], column-major, ld wb) block (r, c) is
// band slot (a0 + r, c - r) of each batch entry (stride gstride). to_dense: band -> D.
__global__ void band_window_kernel(double2* __restrict__ G, long long gstride, double2* __restrict__ D, int a0, int w,
                                   int b, int batch, int to_dense) {
  const long long bb = (long long)b * b, wb = (long long)w * b;
  const long long per = wb * wb, total = per * batch;
  const int nslot = 2 * w + 1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long e = idx / per, q = idx - e * per;
    const long long col = q / wb, row = q - col * wb;  // dense (row, col)
    const int r = int(row / b), c = int(col / b);
    const long long i = row - (long long)r * b, j = col - (long long)c * b;
    double2* g = G + e * gstride + ((long long)(a0 + r) * nslot + (c - r) + w) * bb + j * b + i;
    if (to_dense)
      D[idx] = *g;
    else
      *g = D[idx];
  }
}
}  // namespace

cudaError_t band_window(double2* G, long long gstride, double2* D, int a0, int w, int b, int batch, bool to_dense,
                        cudaStream_t s) {
  const long long total = (long long)w * b * w * b * batch;
  ProfScope prof(s, PROF_BAND, 0.0, 32.0 * total);
  band_window_kernel<<<grid_for(total, 256), 256, 0, s>>>(G, gstride, D, a0, w, b, batch, to_dense ? 1 : 0);
  return cudaGetLastError();
}

namespace {
__global__ void diag_shift_kernel(double2* M, int n, long long stride, int batch) {
  const int b = blockIdx.y;
  if (b >= batch) return;
  double2* m = M + (long long)b * stride;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double2 x = m[(long long)i * n + i];
    m[(long long)i * n + i] = make_double2(x.x + 1.0, x.y);
  }
}
__global__ void axpy1_kernel(double2* y, const double2* x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = make_double2(y[i].x + x[i].x, y[i].y + x[i].y);
}
}  // namespace

// M_b += I for batch matrices n x n (ld n) at M + b*stride
cudaError_t diag_shift_batched(double2* M, int n, long long stride, int batch, cudaStream_t s) {
  ProfScope prof(s, PROF_BAND, 0.0, 32.0 * n * batch);
  diag_shift_kernel<<<dim3((n + 255) / 256, batch), 256, 0, s>>>(M, n, stride, batch);
  return cudaGetLastError();
}

namespace {
__global__ void axpy_strided_kernel(double2* y, long long ys, const double2* x, long long xs, long long n, double2 a) {
  const long long g = blockIdx.y;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 v = x[g * xs + i];
    double2& o = y[g * ys + i];
    o = make_double2(fma(a.x, v.x, fma(-a.y, v.y, o.x)), fma(a.x, v.y, fma(a.y, v.x, o.y)));
  }
}
}  // namespace

// y_g += a * x_g for nb strided families of n contiguous complex entries
cudaError_t axpy_strided(double2* y, long long ys, const double2* x, long long xs, long long n, int nb, double2 a,
                         cudaStream_t s) {
  ProfScope prof(s, PROF_BAND, 8.0 * n * nb, 48.0 * n * nb);
  axpy_strided_kernel<<<dim3(grid_for(n, 256) / 4 + 1, nb), 256, 0, s>>>(y, ys, x, xs, n, a);
  return cudaGetLastError();
}

// y += x over n complex entries
cudaError_t axpy_batched(double2* y, const double2* x, long long n, cudaStream_t s) {
  ProfScope prof(s, PROF_BAND, 2.0 * n, 48.0 * n);
  axpy1_kernel<<<grid_for(n, 256), 256, 0, s>>>(y, x, n);
  return cudaGetLastError();
}

}  // namespace bbsi_gpu

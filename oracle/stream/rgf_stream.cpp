// Streaming restatement of the reference rgf_tridiag (rgf.hpp:37-76) for full-size
// parity checks whose dense band does not fit in host RAM next to the GPU result
// (config 5: 58 GB per band). TEST INFRASTRUCTURE ONLY: called by tools/parity_full.py
// as the checker, never by the product library.
//
// The BLAS/LAPACK calls are the reference's, in the reference's order and with its
// arguments (kernels.hpp:101-195): lu_factor = zgetrf + the eps*n*max|A| negligible-
// pivot test; solve_left = zgetrs('N'); solve_right = zgetrs('T') on the transposed
// right-hand side, transposed back; invert = zgetrs('N', I); gemm_into = zgemm. With
// the same OpenBLAS (0.3.15, oracle/ref/Makefile) the blocks are the reference's;
// tests/test_oracle.py pins this against oracle/_ref on small matrices.
//
// Differences from the reference are only in storage:
//  * A's blocks are generated on demand from the Dyson spec (restated here from
//    oracle/dyson_oracle.py; optionally perturbed by one ulp on a random half of the
//    components, the noise-floor protocol of tools/parity_full.py);
//  * the upward sweep keeps f / umult / lmult for every `ckpt`-th segment only and
//    recomputes a segment (same calls, same order, so the same bits) when the downward
//    sweep reaches it: memory O(ckpt + l/ckpt) blocks instead of 3l.
#include <cblas.h>
#include <lapacke.h>
#ifdef RS_SCIPY_OPENBLAS
// scipy's LP64 OpenBLAS (0.3.31, prefixed symbols): same calls, faster kernels on
// AVX-512 hosts. Not bit-identical to oracle/_ref (different BLAS build); pinned to it
// at <= 1e-13 by tests/test_oracle.py.
extern "C" {
void scipy_cblas_zgemm(int, int, int, int, int, int, const void*, const void*, int, const void*, int, const void*,
                       void*, int);
int scipy_LAPACKE_zgetrf(int, int, int, void*, int, int*);
int scipy_LAPACKE_zgetrs(int, char, int, int, const void*, int, const int*, void*, int);
void scipy_openblas_set_num_threads(int);
}
#define cblas_zgemm(o, ta, tb, m, n, k, al, a, lda, b, ldb, be, c, ldc) \
  scipy_cblas_zgemm(o, ta, tb, m, n, k, al, a, lda, b, ldb, be, c, ldc)
#define LAPACKE_zgetrf(o, m, n, a, lda, p) scipy_LAPACKE_zgetrf(o, m, n, a, lda, p)
#define LAPACKE_zgetrs(o, t, n, r, a, lda, p, b, ldb) scipy_LAPACKE_zgetrs(o, t, n, r, a, lda, p, b, ldb)
#define openblas_set_num_threads(n) scipy_openblas_set_num_threads(n)
#endif

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

using cd = std::complex<double>;

namespace {

uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double unif(uint64_t sm, int a, int off, long long k, int c) {
  uint64_t ctr = ((uint64_t)a << 40) | ((uint64_t)(off + 8) << 36) | (uint64_t)(2 * k + c);
  return (double)(mix64(sm ^ ctr) >> 11) * (1.0 / 4503599627370496.0) - 1.0;
}

struct Mat {
  int n = 0;
  std::vector<cd> v;  // column-major
  Mat() = default;
  explicit Mat(int n_) : n(n_), v(size_t(n_) * n_) {}
  cd& operator()(int i, int j) { return v[size_t(j) * n + i]; }
  cd* data() { return v.data(); }
  const cd* data() const { return v.data(); }
};

struct LU {
  Mat packed;
  std::vector<int> piv;
};

struct Stream {
  int l, b, sigma_layers, ckpt;
  uint64_t sm;
  cd z;
  double pert;  // 0: none; else probability of a one-ulp move per component
  uint64_t pseed;
  int fail_layer = -1;
  // checkpoints: f at the start layer of every segment (upward order: seg top = c*ckpt)
  std::vector<std::unique_ptr<LU>> fck;  // f[c*ckpt] for c >= 1 (the upward carry into segment c-1)
  // current segment [s0, s1): f, umult[i] (i in [s0, s1)), lmult[i]
  int s0 = -1, s1 = -1;
  std::vector<LU> f;
  std::vector<Mat> um, lm;
  // downward state
  int next = 0;
  Mat gprev;  // G[i-1, i-1]

  double jitter(double x, int a, int off, long long k, int c) const {
    if (pert <= 0.0) return x;
    uint64_t h = mix64(pseed ^ (((uint64_t)a << 40) | ((uint64_t)(off + 8) << 36) | (uint64_t)(2 * k + c)));
    double r = (double)(h >> 11) * (1.0 / 9007199254740992.0);  // [0, 1)
    if (r >= pert) return x;
    return (h & 1) ? std::nextafter(x, INFINITY) : std::nextafter(x, -INFINITY);
  }

  // block (a, a+off) of A(E) = z I - H - Sigma (dyson_oracle.dyson_matrix order)
  Mat block(int a, int off) const {
    Mat m(b);
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) {
        double re, im;
        const long long k = (long long)j * b + i;
        if (off == 0) {
          double xr = unif(sm, a, 0, k, 0), xi = unif(sm, a, 0, k, 1);
          double yr = unif(sm, a, 0, (long long)i * b + j, 0), yi = unif(sm, a, 0, (long long)i * b + j, 1);
          double hr = 0.5 * (xr + yr), hi = 0.5 * (xi - yi);
          if (i == j) {
            const bool s = a < sigma_layers || a >= l - sigma_layers;
            const double sr = 0.0, si = s ? -0.5 : 0.0;
            re = (z.real() - hr) - sr;
            im = (z.imag() - hi) - si;
          } else {
            re = -hr;
            im = -hi;
          }
        } else if (off > 0) {
          re = -(0.5 * unif(sm, a, 1, k, 0));
          im = -(0.5 * unif(sm, a, 1, k, 1));
        } else {
          re = -(0.5 * unif(sm, a - 1, 1, (long long)i * b + j, 0));
          im = 0.5 * unif(sm, a - 1, 1, (long long)i * b + j, 1);
        }
        m(i, j) = cd(jitter(re, a, off, k, 0), jitter(im, a, off, k, 1));
      }
    return m;
  }

  // kernels.hpp:140-160
  bool lu_factor(const Mat& a, LU& out) {
    out.packed = a;
    out.piv.assign(std::max(1, b), 0);
    double scale = 0.0;
    for (const cd& x : a.v) scale = std::max(scale, std::abs(x));
    int info = LAPACKE_zgetrf(LAPACK_COL_MAJOR, b, b, out.packed.data(), b, out.piv.data());
    const double tol = std::numeric_limits<double>::epsilon() * double(b) * scale;
    if (info > 0) return false;
    for (int i = 0; i < b; ++i)
      if (std::abs(out.packed(i, i)) <= tol) return false;
    return true;
  }
  Mat solve_left(const LU& f, const Mat& rhs) {
    Mat x = rhs;
    LAPACKE_zgetrs(LAPACK_COL_MAJOR, 'N', b, b, f.packed.data(), b, f.piv.data(), x.data(), b);
    return x;
  }
  Mat transposed(const Mat& m) {
    Mat t(b);
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) t(j, i) = const_cast<Mat&>(m)(i, j);
    return t;
  }
  Mat solve_right(const Mat& rhs, const LU& f) {
    Mat xt = transposed(rhs);
    LAPACKE_zgetrs(LAPACK_COL_MAJOR, 'T', b, b, f.packed.data(), b, f.piv.data(), xt.data(), b);
    return transposed(xt);
  }
  Mat invert(const LU& f) {
    Mat id(b);
    for (int i = 0; i < b; ++i) id(i, i) = 1.0;
    return solve_left(f, id);
  }
  void gemm_into(cd alpha, const Mat& A, const Mat& B, cd beta, Mat& C) {
    cblas_zgemm(CblasColMajor, CblasNoTrans, CblasNoTrans, b, b, b, &alpha, A.data(), b, B.data(), b, &beta,
                C.data(), b);
  }

  // one upward step (rgf.hpp:58-64): given f[i+1] -> umult[i], lmult[i], f[i]
  bool up_step(int i, const LU& fnext, Mat& umi, Mat& lmi, LU& fi) {
    const Mat aup = block(i, +1);
    umi = solve_right(aup, fnext);
    lmi = solve_left(fnext, block(i + 1, -1));
    Mat pivot = block(i, 0);
    gemm_into(cd(-1), aup, lmi, cd(1), pivot);
    if (!lu_factor(pivot, fi)) {
      fail_layer = i;
      return false;
    }
    return true;
  }

  int nseg() const { return (l + ckpt - 1) / ckpt; }

  // full upward sweep keeping only the checkpoints f[c*ckpt], c >= 1
  bool upward() {
    fck.clear();
    fck.resize(nseg() + 1);
    LU cur, nxt;
    if (!lu_factor(block(l - 1, 0), cur)) {
      fail_layer = l - 1;
      return false;
    }
    if ((l - 1) % ckpt == 0 && l - 1 > 0) fck[(l - 1) / ckpt].reset(new LU(cur));
    Mat u, m;
    for (int i = l - 2; i >= 0; --i) {
      if (!up_step(i, cur, u, m, nxt)) return false;
      std::swap(cur, nxt);
      if (i % ckpt == 0 && i > 0) fck[i / ckpt].reset(new LU(cur));
    }
    return true;
  }

  // recompute segment [s0, s1) = [c*ckpt, min(l, (c+1)*ckpt)): f[s0..s1-1], um/lm[s0-1..s1-2]
  // (the multipliers of rows i with i+1 in the segment are what the downward sweep needs)
  bool load_segment(int c) {
    s0 = c * ckpt;
    s1 = std::min(l, s0 + ckpt);
    const int n = s1 - s0;
    f.assign(n, LU{});
    um.assign(n, Mat{});
    lm.assign(n, Mat{});
    // f[s1-1] from the checkpoint above or from scratch
    int top = s1 - 1;
    LU cur;
    if (s1 == l) {
      if (!lu_factor(block(l - 1, 0), cur)) return false;
    } else {
      // f[s1] is checkpoint c+1; step down to s1-1
      LU tmp;
      Mat u, m;
      if (!up_step(s1 - 1, *fck[c + 1], u, m, tmp)) return false;
      um[n - 1] = std::move(u);  // umult[s1-1] (row s1-1 -> s1): not needed in this segment
      lm[n - 1] = std::move(m);
      cur = std::move(tmp);
    }
    f[top - s0] = cur;
    for (int i = top - 1; i >= s0; --i) {
      Mat u, m;
      LU fi;
      if (!up_step(i, f[i + 1 - s0], u, m, fi)) return false;
      um[i - s0] = std::move(u);  // umult[i]
      lm[i - s0] = std::move(m);  // lmult[i]
      f[i - s0] = std::move(fi);
    }
    return true;
  }
};

}  // namespace

extern "C" {

void* rs_create(int l, int b, uint64_t seed, double zr, double zi, int sigma_layers, double pert, uint64_t pseed,
                int ckpt) {
  auto* s = new Stream();
  s->l = l;
  s->b = b;
  s->sm = mix64(seed);
  s->z = cd(zr, zi);
  s->sigma_layers = sigma_layers;
  s->pert = pert;
  s->pseed = pseed;
  s->ckpt = ckpt > 0 ? ckpt : l;
  return s;
}

void rs_destroy(void* h) { delete static_cast<Stream*>(h); }

void rs_set_threads(int n) { openblas_set_num_threads(n); }

// Upward sweep (checkpoints only). Returns 0, or 2 with the failing layer in *fail.
int rs_upward(void* h, int* fail) {
  auto* s = static_cast<Stream*>(h);
  s->next = 0;
  s->s0 = s->s1 = -1;
  if (s->nseg() == 1) {  // no checkpoints: the first segment load is the whole upward sweep
    *fail = -1;
    return 0;
  }
  bool ok = s->upward();
  *fail = s->fail_layer;
  return ok ? 0 : 2;
}

// Next layer i of the downward sweep (rgf.hpp:66-75), i = 0, 1, ...: writes G[i,i]
// into gdiag and, for i >= 1, G[i-1,i] into gup and G[i,i-1] into glo (column-major
// b x b each). Returns the layer index, or -1 past the end / -2 on failure.
int rs_next(void* h, void* gdiag, void* gup, void* glo) {
  auto* s = static_cast<Stream*>(h);
  const int i = s->next;
  if (i >= s->l) return -1;
  if (s->l == 1) {
    LU f;
    if (!s->lu_factor(s->block(0, 0), f)) return -2;
    Mat g = s->invert(f);
    std::memcpy(gdiag, g.data(), sizeof(cd) * g.v.size());
    s->next = 1;
    return 0;
  }
  if (i == 0 || i >= s->s1) {
    if (!s->load_segment(i / s->ckpt)) return -2;
  }
  const size_t bytes = sizeof(cd) * size_t(s->b) * s->b;
  if (i == 0) {
    s->gprev = s->invert(s->f[0]);
    std::memcpy(gdiag, s->gprev.data(), bytes);
    s->next = 1;
    return 0;
  }
  // umult[i-1], lmult[i-1]: row i-1 lives in this segment unless i == s0 (then the
  // previous segment's last row, kept below)
  const Mat* umi;
  const Mat* lmi;
  Mat uprev, lprev;
  if (i - 1 >= s->s0) {
    umi = &s->um[i - 1 - s->s0];
    lmi = &s->lm[i - 1 - s->s0];
  } else {
    // row i-1 = s0-1: its multipliers are computed from f[s0] (this segment)
    LU tmp;
    if (!s->up_step(i - 1, s->f[0], uprev, lprev, tmp)) return -2;
    umi = &uprev;
    lmi = &lprev;
  }
  Mat gup_m(s->b), glo_m(s->b);
  s->gemm_into(cd(-1), s->gprev, *umi, cd(0), gup_m);
  s->gemm_into(cd(-1), *lmi, s->gprev, cd(0), glo_m);
  Mat gd = s->invert(s->f[i - s->s0]);
  s->gemm_into(cd(-1), *lmi, gup_m, cd(1), gd);
  std::memcpy(gup, gup_m.data(), bytes);
  std::memcpy(glo, glo_m.data(), bytes);
  std::memcpy(gdiag, gd.data(), bytes);
  s->gprev = std::move(gd);
  s->next = i + 1;
  return i;
}

// Block (a, off) of this stream's A (perturbed if the stream is), column-major.
void rs_block(void* h, int a, int off, void* out) {
  auto* s = static_cast<Stream*>(h);
  Mat m = s->block(a, off);
  std::memcpy(out, m.data(), sizeof(cd) * m.v.size());
}

}  // extern "C"

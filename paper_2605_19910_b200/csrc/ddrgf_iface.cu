// DDRGF phase 2: the interface system, single- or multi-level (DomainPlan::s2_levels).
//
// The reference reduces the separator Schur system level by level (ddrgf_level's
// recursion, ddrgf.hpp:363-369) and solves the last level with rgf_tridiag. Here the
// "reduced system" is the chain of 2-ports the stabilised phase 1 produces: per level-0
// task t the fake-lead corners K_t = (a, b, c, e) of its domain plus the interface
// blocks of A around its separator (the packet). A level of the plan groups s2 2-ports
// (+ the separator after each) into one super 2-port:
//
//   merge    [X, s, Y] -> the corners of the concatenation with fake leads only at its
//            outer ends: Woodbury on the three interface blocks {l_X, s, f_Y} of
//            N = blockdiag(X~, A_ss + i g_s, Y~) (every block well conditioned), with
//            W = (I + U D)^{-1} U, D = blockdiag(e_X, (A_ss + i g_s)^{-1}, a_Y):
//              a = a_X - b_X W11 c_X,  b = -b_X W13 b_Y,  c = -c_Y W31 c_X,  e = e_Y - c_Y W33 b_Y;
//   sweeps   the left- and right-connected recursions over a chain of 2-ports (the
//            single-level phase 2), optionally with boundary values from the level above;
//   nested   merge every group (batched over groups), solve the chain of super 2-ports
//            (recursively, one level less), then run the sweeps inside every group with
//            the boundary values the level above produced (batched over groups).
//
// Every operation is batched over independent chains (groups), so the sequential depth
// of phase 2 drops from T separators to T/(s2_1+1) + s2_1 + ... . No isolated-domain
// inverse is ever formed. tools/ddrgf_nested_proto.py is the numpy model of this file.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace bbsi_gpu {

namespace {

// y_g[r, c] += scale * coef_g * x_g[r, c]   (rows x cols, column-major with ld; nb batches)
__global__ void zaxpy2d_kernel(double2* y, long long ldy, long long ys, const double2* x, long long ldx, long long xs,
                               int rows, int cols, const double2* coef, long long cs, double2 scale) {
  const int g = blockIdx.y;
  double2 a = scale;
  if (coef) {
    const double2 c = coef[(long long)g * cs];
    a = make_double2(scale.x * c.x - scale.y * c.y, scale.x * c.y + scale.y * c.x);
  }
  const long long n = (long long)rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long c = i / rows, r = i - c * rows;
    double2* py = y + g * ys + c * ldy + r;
    const double2 v = x[g * xs + c * ldx + r];
    *py = cfma(a, v, *py);
  }
}

// y_g[i, i] += scale * coef_g (coef may be null: += scale)
__global__ void zdiag2d_kernel(double2* y, long long ldy, long long ys, int n, const double2* coef, long long cs,
                               double2 scale) {
  const int g = blockIdx.y;
  double2 a = scale;
  if (coef) {
    const double2 c = coef[(long long)g * cs];
    a = make_double2(scale.x * c.x - scale.y * c.y, scale.x * c.y + scale.y * c.x);
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double2* p = y + g * ys + (long long)i * ldy + i;
    *p = make_double2(p->x + a.x, p->y + a.y);
  }
}

// A strided family of nb b x b blocks (block g at p + g * gs, leading dimension ld)
struct Blk {
  double2* p;
  long long gs;
  long long ld;
};

struct Ctx {
  int b;
  int nb;
  int n_true;
  cudaStream_t s;
  long long bb() const { return (long long)b * b; }
};

cudaError_t zaxpy2d(const Ctx& c, Blk y, Blk x, const double2* coef, long long cs, double2 scale) {
  ProfScope prof(c.s, PROF_BAND, 8.0 * c.bb() * c.nb, 48.0 * c.bb() * c.nb);
  const int gx = (int)std::min<long long>((c.bb() + 255) / 256, 148LL * 4);
  zaxpy2d_kernel<<<dim3(gx, c.nb), 256, 0, c.s>>>(y.p, y.ld, y.gs, x.p, x.ld, x.gs, c.b, c.b, coef, cs, scale);
  return cudaGetLastError();
}
cudaError_t zdiag2d(const Ctx& c, Blk y, const double2* coef, long long cs, double2 scale) {
  ProfScope prof(c.s, PROF_BAND, 0.0, 32.0 * c.b * c.nb);
  zdiag2d_kernel<<<dim3((c.b + 255) / 256, c.nb), 256, 0, c.s>>>(y.p, y.ld, y.gs, c.b, coef, cs, scale);
  return cudaGetLastError();
}
ZOp zo(Blk x) { return ZOp{x.p, x.ld, 64, 64LL * x.ld, x.gs}; }
// y = alpha * a * b + beta * y  (batched over nb)
cudaError_t mm(const Ctx& c, double alpha, Blk a, Blk b, double beta, Blk y) {
  return zmm(c.b, c.nb, make_double2(alpha, 0.0), zo(a), zo(b), beta, zo(y), c.s);
}
cudaError_t copy(const Ctx& c, Blk d, Blk x) {
  if (d.ld == c.b && x.ld == c.b)
    return cudaMemcpy2DAsync(d.p, d.gs * sizeof(double2), x.p, x.gs * sizeof(double2), c.bb() * sizeof(double2), c.nb,
                             cudaMemcpyDeviceToDevice, c.s);
  for (int g = 0; g < c.nb; ++g) {
    cudaError_t e = cudaMemcpy2DAsync(d.p + g * d.gs, d.ld * sizeof(double2), x.p + g * x.gs, x.ld * sizeof(double2),
                                      c.b * sizeof(double2), c.b, cudaMemcpyDeviceToDevice, c.s);
    if (e) return e;
  }
  return cudaSuccess;
}
cudaError_t zero(const Ctx& c, Blk d) {
  if (d.ld == c.b)
    return cudaMemset2DAsync(d.p, d.gs * sizeof(double2), 0, c.bb() * sizeof(double2), c.nb, c.s);
  for (int g = 0; g < c.nb; ++g) {
    cudaError_t e = cudaMemset2DAsync(d.p + g * d.gs, d.ld * sizeof(double2), 0, c.b * sizeof(double2), c.b, c.s);
    if (e) return e;
  }
  return cudaSuccess;
}
cudaError_t ident(const Ctx& c, Blk d) {
  cudaError_t e = zero(c, d);
  return e ? e : zdiag2d(c, d, nullptr, 0, make_double2(1.0, 0.0));
}

// In-place batched inverse with one Newton-Schulz refinement step (the interface
// quantities feed every later separator); `keep` / `r` are two scratch families.
struct InvLog {
  int* st = nullptr;          // device status slots
  int cap = 0, used = 0;
  std::vector<int> layer;     // per slot: the global layer it reports (per chain: layer_base + ...)
};
cudaError_t inv_ref(const Ctx& c, Blk m, Blk keep, Blk r, InvLog& log, const std::vector<int>& layers, bool refine,
                    void* iscr) {
  if (log.used + c.nb > log.cap) return cudaErrorInvalidValue;
  int* slot = log.st + log.used;
  for (int g = 0; g < c.nb; ++g) log.layer.push_back(layers[g]);
  log.used += c.nb;
  cudaError_t e;
  if (refine && (e = copy(c, keep, m))) return e;
  if (m.ld != c.b) return cudaErrorInvalidValue;
  if ((e = zinv_batched(m.p, c.b, m.gs, c.b, c.n_true, c.nb, iscr, slot, c.s))) return e;
  if (!refine) return cudaSuccess;
  if ((e = ident(c, r))) return e;
  if ((e = mm(c, -1.0, keep, m, 1.0, r))) return e;       // R = I - M X
  if ((e = mm(c, 1.0, m, r, 0.0, keep))) return e;        // keep = X R
  return zaxpy2d(c, m, keep, nullptr, 0, make_double2(1.0, 0.0));  // X += X R
}

bool refine_iface() {
  const char* ev = getenv("BBSI_DDRGF_REFINE");
  return !(ev && atoi(ev) == 0);
}

}  // namespace

// One chain family: nb chains of nt 2-ports. Packet of task k in chain g at
// pk + (g*pk_gs + k*pk_ts) (PK blocks of bb each), output at out + (g*o_gs + k*o_ts).
struct IfaceChains {
  const double2* pk;
  long long pk_gs, pk_ts;
  double2* out;
  long long o_gs, o_ts;
  int nb, nt;
  const double2* gamL;  // device complex [nb][nt]: fake-lead strength at the 2-port's first block
  const double2* gamR;  //   ... at its last block
  std::vector<char> empty;        // [nt]: 2-port without interior (same for every chain)
  std::vector<int> first, last, sep;  // [nb][nt] global layers (status labels)
  // optional boundaries (device, per chain stride bnd_gs): gL of the separator before
  // task 0 and that separator's coupling to task 0's first layer (A[s, s+1]); Sigma^R
  // on the last task's separator
  const double2* left_gL = nullptr;
  const double2* left_An = nullptr;
  long long left_gs = 0, left_an_gs = 0;
  const double2* right_SR = nullptr;
  long long right_gs = 0;
};

enum { PA_, PB_, PC_, PE_, PASS_, PASL_, PALS_, PASN_, PAX0_, PK_ };
enum { OSL_, OSR_, OY_, OGL_, NOUT_ };

// The left- and right-connected recursions (the right one on a side stream).
cudaError_t iface_sweeps(const IfaceChains& q, int b, int n_true, InvLog& log, cudaStream_t s, cudaStream_t side,
                         cudaEvent_t fork, cudaEvent_t join) {
  const long long bb = (long long)b * b;
  const int nb = q.nb;
  const bool refine = refine_iface();
  constexpr int NT = 10;
  double2* scr = static_cast<double2*>(arena_get(13, size_t(2 * NT) * nb * bb * sizeof(double2)));
  void* is1 = arena_get(7, zinv_scratch_bytes(b, nb) + 256);
  void* is2 = arena_get(17, zinv_scratch_bytes(b, nb) + 256);
  if (!scr || !is1 || !is2) return cudaErrorMemoryAllocation;
  auto P = [&](int k, int f) { return Blk{const_cast<double2*>(q.pk) + k * q.pk_ts + f * bb, q.pk_gs, b}; };
  auto O = [&](int k, int f) { return Blk{q.out + k * q.o_ts + f * bb, q.o_gs, b}; };
  auto gL_ = [&](int k) { return q.gamL + k; };
  auto gR_ = [&](int k) { return q.gamR + k; };
  const long long gam_gs = q.nt;
  const Ctx L{b, nb, n_true, s}, R{b, nb, n_true, side};
  auto Tm = [&](int which, int i) { return Blk{scr + ((size_t)which * NT + i) * nb * bb, bb, b}; };
  auto layers = [&](const std::vector<int>& v, int k) {
    std::vector<int> out(nb);
    for (int g = 0; g < nb; ++g) out[g] = v[(size_t)g * q.nt + k];
    return out;
  };
  cudaError_t e;
  // d = x * y * z
  auto mm3 = [&](const Ctx& c, int w, Blk d, Blk x, Blk y, Blk z) -> cudaError_t {
    cudaError_t e2 = mm(c, 1.0, x, y, 0.0, Tm(w, 7));
    return e2 ? e2 : mm(c, 1.0, Tm(w, 7), z, 0.0, d);
  };
  // o = x + i g x (I - i g x)^{-1} x  (removes the fake lead of strength g at x's block)
  auto remove_fake = [&](const Ctx& c, int w, Blk o, Blk x, const double2* gam, const std::vector<int>& lay,
                         void* iscr) -> cudaError_t {
    cudaError_t e2;
    if ((e2 = ident(c, Tm(w, 2)))) return e2;
    if ((e2 = zaxpy2d(c, Tm(w, 2), x, gam, gam_gs, make_double2(0.0, -1.0)))) return e2;
    if ((e2 = inv_ref(c, Tm(w, 2), Tm(w, 8), Tm(w, 9), log, lay, refine, iscr))) return e2;
    if ((e2 = mm(c, 1.0, Tm(w, 2), x, 0.0, Tm(w, 3)))) return e2;
    if ((e2 = mm(c, 1.0, x, Tm(w, 3), 0.0, Tm(w, 4)))) return e2;
    if ((e2 = copy(c, o, x))) return e2;
    return zaxpy2d(c, o, Tm(w, 4), gam, gam_gs, make_double2(0.0, 1.0));
  };
  if ((e = cudaEventRecord(fork, s)) || (e = cudaStreamWaitEvent(side, fork, 0))) return e;
  // ---- right-connected recursion (side stream): Sigma^R and Y
  for (int k = q.nt - 1; k >= 0; --k) {
    const int w = 1;
    if (k < q.nt - 1) {
      if ((e = mm3(R, w, O(k, OSR_), P(k, PASN_), O(k + 1, OY_), P(k + 1, PAX0_)))) return e;
    } else if (q.right_SR) {
      if ((e = copy(R, O(k, OSR_), Blk{const_cast<double2*>(q.right_SR), q.right_gs, b}))) return e;
    } else if ((e = zero(R, O(k, OSR_)))) {
      return e;
    }
    Blk gR = Tm(w, 0);
    if ((e = copy(R, gR, P(k, PASS_))) || (e = zaxpy2d(R, gR, O(k, OSR_), nullptr, 0, make_double2(-1.0, 0.0))))
      return e;
    if ((e = inv_ref(R, gR, Tm(w, 8), Tm(w, 9), log, layers(q.sep, k), refine, is2))) return e;
    if (!q.empty[k]) {
      Blk Dl = Tm(w, 1);
      if ((e = mm3(R, w, Dl, P(k, PALS_), gR, P(k, PASL_)))) return e;
      if ((e = zdiag2d(R, Dl, gR_(k), gam_gs, make_double2(0.0, 1.0)))) return e;
      if ((e = ident(R, Tm(w, 2))) || (e = mm(R, -1.0, Dl, P(k, PE_), 1.0, Tm(w, 2)))) return e;
      if ((e = inv_ref(R, Tm(w, 2), Tm(w, 8), Tm(w, 9), log, layers(q.last, k), refine, is2))) return e;
      if ((e = mm(R, 1.0, Tm(w, 2), Dl, 0.0, Tm(w, 3)))) return e;
      if ((e = mm(R, 1.0, Tm(w, 3), P(k, PC_), 0.0, Tm(w, 4)))) return e;
      if ((e = copy(R, Tm(w, 5), P(k, PA_)))) return e;
      if ((e = mm(R, 1.0, P(k, PB_), Tm(w, 4), 1.0, Tm(w, 5)))) return e;
      if ((e = remove_fake(R, w, O(k, OY_), Tm(w, 5), gL_(k), layers(q.first, k), is2))) return e;
    } else if ((e = copy(R, O(k, OY_), gR))) {
      return e;
    }
  }
  if ((e = cudaEventRecord(join, side))) return e;
  // ---- left-connected recursion (main stream): Sigma^L and gL
  for (int k = 0; k < q.nt; ++k) {
    const int w = 0;
    Blk SL = Tm(w, 6);
    const bool has_prev = k > 0 || q.left_gL;
    Blk prev_gL = k > 0 ? O(k - 1, OGL_) : Blk{const_cast<double2*>(q.left_gL), q.left_gs, b};
    Blk prev_An = k > 0 ? P(k - 1, PASN_) : Blk{const_cast<double2*>(q.left_An), q.left_an_gs, b};
    if (!q.empty[k]) {
      Blk Df = Tm(w, 1);
      if (has_prev) {
        if ((e = mm3(L, w, O(k, OSL_), P(k, PAX0_), prev_gL, prev_An))) return e;
      } else if ((e = zero(L, O(k, OSL_)))) {
        return e;
      }
      if ((e = copy(L, Df, O(k, OSL_))) || (e = zdiag2d(L, Df, gL_(k), gam_gs, make_double2(0.0, 1.0)))) return e;
      if ((e = ident(L, Tm(w, 2))) || (e = mm(L, -1.0, Df, P(k, PA_), 1.0, Tm(w, 2)))) return e;
      if ((e = inv_ref(L, Tm(w, 2), Tm(w, 8), Tm(w, 9), log, layers(q.first, k), refine, is1))) return e;
      if ((e = mm(L, 1.0, Tm(w, 2), Df, 0.0, Tm(w, 3)))) return e;
      if ((e = mm(L, 1.0, Tm(w, 3), P(k, PB_), 0.0, Tm(w, 4)))) return e;
      if ((e = copy(L, Tm(w, 5), P(k, PE_)))) return e;
      if ((e = mm(L, 1.0, P(k, PC_), Tm(w, 4), 1.0, Tm(w, 5)))) return e;
      Blk gld = Tm(w, 0);
      if ((e = remove_fake(L, w, gld, Tm(w, 5), gR_(k), layers(q.last, k), is1))) return e;
      if ((e = mm3(L, w, SL, P(k, PASL_), gld, P(k, PALS_)))) return e;
    } else {
      if (!has_prev) return cudaErrorInvalidValue;  // an empty first 2-port needs a left neighbour
      if ((e = mm3(L, w, SL, P(k, PASL_), prev_gL, prev_An))) return e;
      if ((e = copy(L, O(k, OSL_), SL))) return e;  // the chain's only block is the separator
    }
    if ((e = copy(L, O(k, OGL_), P(k, PASS_))) || (e = zaxpy2d(L, O(k, OGL_), SL, nullptr, 0, make_double2(-1.0, 0.0))))
      return e;
    if ((e = inv_ref(L, O(k, OGL_), Tm(w, 8), Tm(w, 9), log, layers(q.sep, k), refine, is1))) return e;
  }
  return cudaStreamWaitEvent(s, join, 0);
}

}  // namespace bbsi_gpu

namespace bbsi_gpu {

namespace {

// Level partition of a chain of T 2-ports (interleave_permutation, partition.hpp:39-75).
struct Groups {
  std::vector<int> first, count, sep;
};
Groups groups_of(int T, int s2) {
  Groups g;
  int pos = 0;
  while (pos < T) {
    const int rem = T - pos;
    int d2, d1;
    if (rem >= 1 + s2) {
      d2 = s2;
      d1 = 1;
    } else {
      d1 = std::min(1, rem);
      d2 = rem - d1;
    }
    g.first.push_back(pos);
    g.count.push_back(d2);
    g.sep.push_back(pos + d2);
    pos += d2 + d1;
  }
  return g;
}

struct Solve {
  int b, n_true;
  cudaStream_t s, side;
  cudaEvent_t fork, join;
  InvLog* log;
  double2* gam_dev;            // device pool of fake-lead strengths
  std::vector<double2> gam_h;  // host mirror (filled family by family)
  size_t gam_cap;
};

// uploads v into the next free region of the gamma pool, returns its device address
const double2* put_gam(Solve& S, const std::vector<double2>& v) {
  if (S.gam_h.size() + v.size() > S.gam_cap) return nullptr;
  const size_t off = S.gam_h.size();
  S.gam_h.insert(S.gam_h.end(), v.begin(), v.end());
  if (cudaMemcpyAsync(S.gam_dev + off, S.gam_h.data() + off, v.size() * sizeof(double2), cudaMemcpyHostToDevice, S.s))
    return nullptr;
  return S.gam_dev + off;
}

// A chain of 2-ports as the solver sees it (host-side description).
struct Chain {
  const double2* pk;  // packet of task k at pk + k * pk_ts
  long long pk_ts;
  double2* out;       // output of task k at out + k * o_ts
  long long o_ts;
  int T;
  std::vector<double> gL, gR;  // fake-lead strengths at each 2-port's first / last block
  std::vector<char> empty;
  std::vector<int> first, last, sep;
};

// One merge step over nb groups: (X, s, Y) -> X. Blk families: running corners K[4],
// the separator blocks of task t and the next 2-port (task t+1).
cudaError_t merge_step(Solve& S, const Ctx& c, Blk K[4], Blk ALS, Blk ASL, Blk ASS, Blk ASN, Blk AX0n, Blk KY[4],
                       const double2* gX, const double2* gS, const double2* gY, double2* scr,
                       const std::vector<int>& sep_layers) {
  const long long bb = (long long)c.b * c.b;
  const int b = c.b, nb = c.nb;
  const long long b3 = 3LL * b;
  cudaError_t e;
  auto T = [&](int i) { return Blk{scr + (size_t)i * nb * bb, bb, b}; };
  double2* m3 = scr + (size_t)20 * nb * bb;  // [nb][3b x 3b]
  void* is3 = arena_get(24, zinv_scratch_bytes(3 * b, nb) + 256);
  if (!is3) return cudaErrorMemoryAllocation;
  auto M = [&](int i, int j) { return Blk{m3 + (long long)j * b * b3 + (long long)i * b, 9 * bb, b3}; };
  // g_s = (A_ss + i g_s)^{-1}
  Blk Gs = T(0);
  if ((e = copy(c, Gs, ASS)) || (e = zdiag2d(c, Gs, gS, 1, make_double2(0.0, 1.0)))) return e;
  if ((e = inv_ref(c, Gs, T(18), T(19), *S.log, sep_layers, refine_iface(), arena_get(25, zinv_scratch_bytes(b, nb) + 256))))
    return e;
  // M3 = I + U D
  if ((e = cudaMemset2DAsync(m3, 9 * bb * sizeof(double2), 0, 9 * bb * sizeof(double2), nb, c.s))) return e;
  const Ctx c3{3 * b, nb, 3 * b, c.s};
  if ((e = zdiag2d(c3, Blk{m3, 9 * bb, b3}, nullptr, 0, make_double2(1.0, 0.0)))) return e;
  if ((e = zaxpy2d(c, M(0, 0), K[3], gX, 1, make_double2(0.0, -1.0)))) return e;  // -i gX e_X
  if ((e = mm(c, 1.0, ALS, Gs, 1.0, M(0, 1)))) return e;                          // A[l,s] g_s
  if ((e = mm(c, 1.0, ASL, K[3], 1.0, M(1, 0)))) return e;                        // A[s,l] e_X
  if ((e = zaxpy2d(c, M(1, 1), Gs, gS, 1, make_double2(0.0, -1.0)))) return e;    // -i g_s g_s
  if ((e = mm(c, 1.0, ASN, KY[0], 1.0, M(1, 2)))) return e;                       // A[s,f] a_Y
  if ((e = mm(c, 1.0, AX0n, Gs, 1.0, M(2, 1)))) return e;                         // A[f,s] g_s
  if ((e = zaxpy2d(c, M(2, 2), KY[0], gY, 1, make_double2(0.0, -1.0)))) return e; // -i gY a_Y
  // (I + U D)^{-1} in place
  {
    if (S.log->used + nb > S.log->cap) return cudaErrorInvalidValue;
    int* slot = S.log->st + S.log->used;
    for (int g = 0; g < nb; ++g) S.log->layer.push_back(sep_layers[g]);
    S.log->used += nb;
    if ((e = zinv_batched(m3, b3, 9 * bb, 3 * b, 3 * b, nb, is3, slot, c.s))) return e;
  }
  // W11 = -i gX Inv11 + Inv12 A[s,l];  W13 = Inv12 A[s,f] - i gY Inv13
  // W31 = -i gX Inv31 + Inv32 A[s,l];  W33 = Inv32 A[s,f] - i gY Inv33
  Blk W11 = T(1), W13 = T(2), W31 = T(3), W33 = T(4);
  if ((e = mm(c, 1.0, M(0, 1), ASL, 0.0, W11)) || (e = zaxpy2d(c, W11, M(0, 0), gX, 1, make_double2(0.0, -1.0))))
    return e;
  if ((e = mm(c, 1.0, M(0, 1), ASN, 0.0, W13)) || (e = zaxpy2d(c, W13, M(0, 2), gY, 1, make_double2(0.0, -1.0))))
    return e;
  if ((e = mm(c, 1.0, M(2, 1), ASL, 0.0, W31)) || (e = zaxpy2d(c, W31, M(2, 0), gX, 1, make_double2(0.0, -1.0))))
    return e;
  if ((e = mm(c, 1.0, M(2, 1), ASN, 0.0, W33)) || (e = zaxpy2d(c, W33, M(2, 2), gY, 1, make_double2(0.0, -1.0))))
    return e;
  // corners: a -= b W11 c;  b = -b W13 bY;  c = -cY W31 c;  e = eY - cY W33 bY
  Blk t5 = T(5), t6 = T(6), t7 = T(7), t8 = T(8), t9 = T(9);
  if ((e = mm(c, 1.0, W11, K[2], 0.0, t5))) return e;
  if ((e = mm(c, 1.0, W31, K[2], 0.0, t8))) return e;
  if ((e = mm(c, 1.0, W13, KY[1], 0.0, t6))) return e;
  if ((e = mm(c, 1.0, W33, KY[1], 0.0, t9))) return e;
  if ((e = mm(c, -1.0, K[1], t5, 1.0, K[0]))) return e;
  if ((e = mm(c, -1.0, K[1], t6, 0.0, t7)) || (e = copy(c, K[1], t7))) return e;
  if ((e = mm(c, -1.0, KY[2], t8, 0.0, K[2]))) return e;
  if ((e = copy(c, K[3], KY[3])) || (e = mm(c, -1.0, KY[2], t9, 1.0, K[3]))) return e;
  return cudaSuccess;
}

cudaError_t solve_chain(Solve& S, const Chain& ch, const int* levels, int nl, int depth);

// the sweeps over one batch of equal-length chains (groups), with optional boundaries
cudaError_t run_sweeps(Solve& S, const Chain& ch, int g0, int ng, const Groups& gr, const Chain* up, bool left,
                       bool right) {
  const long long bb = (long long)S.b * S.b;
  const int ta0 = gr.first[g0], nt = gr.count[g0] + 1;
  const long long gstride_t = (ng > 1) ? (long long)(gr.first[g0 + 1] - gr.first[g0]) : 0;
  IfaceChains q;
  q.pk = ch.pk + ta0 * ch.pk_ts;
  q.pk_ts = ch.pk_ts;
  q.pk_gs = gstride_t * ch.pk_ts;
  q.out = ch.out + ta0 * ch.o_ts;
  q.o_ts = ch.o_ts;
  q.o_gs = gstride_t * ch.o_ts;
  q.nb = ng;
  q.nt = nt;
  std::vector<double2> gl, grv;
  for (int g = 0; g < ng; ++g)
    for (int k = 0; k < nt; ++k) {
      const int t = gr.first[g0 + g] + k;
      gl.push_back(make_double2(ch.gL[t], 0.0));
      grv.push_back(make_double2(ch.gR[t], 0.0));
      q.first.push_back(ch.first[t]);
      q.last.push_back(ch.last[t]);
      q.sep.push_back(ch.sep[t]);
    }
  q.gamL = put_gam(S, gl);
  q.gamR = put_gam(S, grv);
  if (!q.gamL || !q.gamR) return cudaErrorMemoryAllocation;
  for (int k = 0; k < nt; ++k) q.empty.push_back(ch.empty[ta0 + k]);
  if (up && left) {  // gL of the level-above separator before each group, and its A[s, s+1]
    q.left_gL = up->out + (long long)(g0 - 1) * up->o_ts + OGL_ * bb;
    q.left_gs = up->o_ts;
    q.left_An = up->pk + (long long)(g0 - 1) * up->pk_ts + PASN_ * bb;
    q.left_an_gs = up->pk_ts;
  }
  if (up && right) {
    q.right_SR = up->out + (long long)g0 * up->o_ts + OSR_ * bb;
    q.right_gs = up->o_ts;
  }
  return iface_sweeps(q, S.b, S.n_true, *S.log, S.s, S.side, S.fork, S.join);
}

cudaError_t solve_chain(Solve& S, const Chain& ch, const int* levels, int nl, int depth) {
  const long long bb = (long long)S.b * S.b;
  bool nest = nl > 0 && ch.T >= 1 + levels[0];
  for (int t = 0; nest && t < ch.T; ++t) nest = !ch.empty[t];
  if (!nest) {  // one chain, no boundaries: the single-level sweeps
    Groups one;
    one.first = {0};
    one.count = {ch.T - 1};
    one.sep = {ch.T - 1};
    return run_sweeps(S, ch, 0, 1, one, nullptr, false, false);
  }
  const Groups gr = groups_of(ch.T, levels[0]);
  const int G = int(gr.first.size());
  // ---- super 2-ports: packets (merged corners + the interface blocks) and outputs
  const size_t PKb = PK_ * bb, NOb = NOUT_ * bb;
  double2* sup = static_cast<double2*>(arena_get(26 + 2 * depth, size_t(G) * (PKb + NOb) * sizeof(double2)));
  double2* scr = static_cast<double2*>(arena_get(27 + 2 * depth, size_t(29) * G * bb * sizeof(double2)));
  if (!sup || !scr) return cudaErrorMemoryAllocation;
  double2* sup_out = sup + (size_t)G * PKb;
  cudaError_t e;
  Chain up;
  up.pk = sup;
  up.pk_ts = PKb;
  up.out = sup_out;
  up.o_ts = NOb;
  up.T = G;
  for (int u = 0; u < G; ++u) {
    const int ta = gr.first[u], tb = gr.sep[u];
    up.gL.push_back(ch.gL[ta]);
    up.gR.push_back(ch.gR[tb]);
    up.empty.push_back(0);
    up.first.push_back(ch.first[ta]);
    up.last.push_back(ch.last[tb]);
    up.sep.push_back(ch.sep[tb]);
    auto cp = [&](int dst_field, int t, int src_field) {
      return cudaMemcpyAsync(sup + u * PKb + dst_field * bb, ch.pk + t * ch.pk_ts + src_field * bb,
                             bb * sizeof(double2), cudaMemcpyDeviceToDevice, S.s);
    };
    for (int f = PA_; f <= PE_; ++f)
      if ((e = cp(f, ta, f))) return e;  // running corners start as task ta's
    for (int f : {PASS_, PASL_, PALS_, PASN_})
      if ((e = cp(f, tb, f))) return e;
    if ((e = cp(PAX0_, ta, PAX0_))) return e;
  }
  // ---- merges, batched over groups of equal size
  int u0 = 0;
  while (u0 < G) {
    int u1 = u0;
    while (u1 < G && gr.count[u1] == gr.count[u0]) ++u1;
    const int ng = u1 - u0, cnt = gr.count[u0];
    const long long tstr = ng > 1 ? (long long)(gr.first[u0 + 1] - gr.first[u0]) * ch.pk_ts : 0;
    const Ctx c{S.b, ng, S.n_true, S.s};
    for (int k = 0; k < cnt; ++k) {
      Blk K[4], KY[4];
      for (int f = 0; f < 4; ++f) {
        K[f] = Blk{sup + u0 * PKb + f * bb, (long long)PKb, S.b};
        KY[f] = Blk{const_cast<double2*>(ch.pk) + (gr.first[u0] + k + 1) * ch.pk_ts + f * bb, tstr, S.b};
      }
      auto tb_ = [&](int t, int f) {
        return Blk{const_cast<double2*>(ch.pk) + (gr.first[u0] + t) * ch.pk_ts + f * bb, tstr, S.b};
      };
      std::vector<double2> gx, gs_, gy;
      std::vector<int> lay;
      for (int g = 0; g < ng; ++g) {
        const int t = gr.first[u0 + g] + k;
        gx.push_back(make_double2(ch.gR[t], 0.0));
        gs_.push_back(make_double2(ch.gR[t], 0.0));
        gy.push_back(make_double2(ch.gL[t + 1], 0.0));
        lay.push_back(ch.sep[t]);
      }
      const double2* dgx = put_gam(S, gx);
      const double2* dgs = put_gam(S, gs_);
      const double2* dgy = put_gam(S, gy);
      if (!dgx || !dgs || !dgy) return cudaErrorMemoryAllocation;
      if ((e = merge_step(S, c, K, tb_(k, PALS_), tb_(k, PASL_), tb_(k, PASS_), tb_(k, PASN_), tb_(k + 1, PAX0_), KY,
                          dgx, dgs, dgy, scr, lay)))
        return e;
    }
    u0 = u1;
  }
  // ---- the level above, then the sweeps inside every group with its boundary values
  if ((e = solve_chain(S, up, levels + 1, nl - 1, depth + 1))) return e;
  auto batch = [&](int g0, int g1, bool left, bool right) -> cudaError_t {
    int g = g0;
    while (g < g1) {  // equal-size runs
      int h = g;
      while (h < g1 && gr.count[h] == gr.count[g]) ++h;
      cudaError_t e2 = run_sweeps(S, ch, g, h - g, gr, &up, left, right);
      if (e2) return e2;
      g = h;
    }
    return cudaSuccess;
  };
  if (G == 1) return batch(0, 1, false, false);
  if ((e = batch(0, 1, false, true))) return e;
  if (G > 2 && (e = batch(1, G - 1, true, true))) return e;
  return batch(G - 1, G, true, false);
}

}  // namespace

// Phase 2 of the (multi-level) stabilised DDRGF over T level-0 tasks: the packets
// (task order, PK blocks each) -> the per-task boundary values (NOUT blocks each).
// levels[0..nl): the plan's s2 of levels 1, 2, ... (s2_levels[1..]).
cudaError_t iface_solve(const double2* packets, double2* out, int T, int b, int n_true, const std::vector<double>& gam,
                        const std::vector<char>& empty, const std::vector<int>& first, const std::vector<int>& last,
                        const std::vector<int>& sep, const int* levels, int nl, int* st, int st_cap,
                        std::vector<int>& st_layer, cudaStream_t s, cudaStream_t side, cudaEvent_t fork,
                        cudaEvent_t join) {
  const long long bb = (long long)b * b;
  InvLog log;
  log.st = st;
  log.cap = st_cap;
  Solve S;
  S.b = b;
  S.n_true = n_true;
  S.s = s;
  S.side = side;
  S.fork = fork;
  S.join = join;
  S.log = &log;
  S.gam_cap = size_t(16) * (T + 8);
  S.gam_h.reserve(S.gam_cap);
  S.gam_dev = static_cast<double2*>(arena_get(40, S.gam_cap * sizeof(double2)));
  if (!S.gam_dev) return cudaErrorMemoryAllocation;
  Chain ch;
  ch.pk = packets;
  ch.pk_ts = PK_ * bb;
  ch.out = out;
  ch.o_ts = NOUT_ * bb;
  ch.T = T;
  ch.gL = gam;
  ch.gR = gam;
  ch.empty = empty;
  ch.first = first;
  ch.last = last;
  ch.sep = sep;
  cudaError_t e = solve_chain(S, ch, levels, nl, 0);
  st_layer = log.layer;
  return e;
}

int iface_status_cap(int T) { return 16 * (T + 8) + 64; }

}  // namespace bbsi_gpu

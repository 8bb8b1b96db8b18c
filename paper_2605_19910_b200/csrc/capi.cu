// C ABI (include/bbsi_cuda.h) over the sm_100a kernels. Validation mirrors the
// reference's preconditions and messages (layout.hpp:27-38, rgf.hpp:41-42,86-87,
// ddrgf.hpp:26-31,424-425); failures map onto the reference exception contract.
#include <cstdio>
#include <map>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <complex>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bbsi_cuda.h"
#include "dyson_gen.h"
#include "internal.h"

using namespace bbsi_gpu;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();
  return fail(e == cudaErrorMemoryAllocation ? BBSI_OUT_OF_MEMORY : BBSI_CUDA_ERROR,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                      \
  do {                                                \
    cudaError_t e_ = (expr);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)

// BlockLayout::validate (layout.hpp:27-38)
int validate_layout(int l, int w, int bs, const int* sizes) {
  if (l < 1) return fail(BBSI_INVALID_ARGUMENT, "BlockLayout: num_layers must be >= 1");
  for (int a = 0; a < l; ++a) {
    int b = sizes ? sizes[a] : bs;
    if (b < 1) return fail(BBSI_INVALID_ARGUMENT, "BlockLayout: block sizes must be >= 1");
    if (b > bs) return fail(BBSI_INVALID_ARGUMENT, "slot size bs smaller than a block size");
  }
  if (w < 0) return fail(BBSI_INVALID_ARGUMENT, "BlockLayout: negative bandwidth");
  if (l > 1 && w > l - 1) return fail(BBSI_INVALID_ARGUMENT, "BlockLayout: bandwidth exceeds num_layers - 1");
  if (l == 1 && w != 0) return fail(BBSI_INVALID_ARGUMENT, "BlockLayout: single layer requires bandwidth 0");
  return BBSI_OK;
}

int pad64(int b) { return (b + 63) / 64 * 64; }

int device_ok() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(BBSI_CUDA_ERROR, "no CUDA device: the bbsi GPU path has no CPU fallback");
  }
  return BBSI_OK;
}

void put_counters(long long* out, long long g, long long lu, long long rs) {
  if (!out) return;
  out[0] = g;
  out[1] = lu;
  out[2] = rs;
}

// Host band in slot order, block (a, a+off) of rows(a) x cols(a+off), ld = bs.
struct HostBand {
  int l, w, bs;
  std::vector<int> sz;
  const double2* p;
  const double2* slot(int a, int off) const { return p + ((long long)a * (2 * w + 1) + off + w) * bs * bs; }
  bool in_band(int a, int off) const { return a + off >= 0 && a + off < l && off >= -w && off <= w; }
};

// Copies a host band into a padded device-layout staging buffer (identity in the
// padding of diagonal blocks: blockdiag(A, I)^{-1} = blockdiag(A^{-1}, I), exact).
void pad_band(const HostBand& h, int bp, std::vector<double2>& out) {
  const long long bb = (long long)bp * bp;
  out.assign(size_t(h.l) * (2 * h.w + 1) * bb, make_double2(0.0, 0.0));
  for (int a = 0; a < h.l; ++a)
    for (int off = -h.w; off <= h.w; ++off) {
      if (!h.in_band(a, off)) continue;
      double2* d = out.data() + ((long long)a * (2 * h.w + 1) + off + h.w) * bb;
      const double2* s = h.slot(a, off);
      const int r = h.sz[a], c = h.sz[a + off];
      for (int j = 0; j < c; ++j) std::memcpy(d + (long long)j * bp, s + (long long)j * h.bs, sizeof(double2) * r);
      if (off == 0)
        for (int i = r; i < bp; ++i) d[(long long)i * bp + i] = make_double2(1.0, 0.0);
    }
}

void unpad_band(const std::vector<double2>& in, int bp, const HostBand& h, double2* G) {
  const long long bb = (long long)bp * bp;
  std::memset(G, 0, sizeof(double2) * size_t(h.l) * (2 * h.w + 1) * h.bs * h.bs);
  for (int a = 0; a < h.l; ++a)
    for (int off = -h.w; off <= h.w; ++off) {
      if (!h.in_band(a, off)) continue;
      const double2* s = in.data() + ((long long)a * (2 * h.w + 1) + off + h.w) * bb;
      double2* d = G + ((long long)a * (2 * h.w + 1) + off + h.w) * h.bs * h.bs;
      const int r = h.sz[a], c = h.sz[a + off];
      for (int j = 0; j < c; ++j) std::memcpy(d + (long long)j * h.bs, s + (long long)j * bp, sizeof(double2) * r);
    }
}

// ---- CUDA-graph replay of a static launch sequence (a sweep is ~10^4 small
// launches per step). Keyed by shapes and every device pointer the sequence
// touches; the first call runs eagerly, the second captures, later calls replay.
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  long long launches = 0;
};
std::mutex g_graph_mu;
std::map<std::string, GraphEntry> g_graphs;

bool graphs_enabled() {
  const char* e = getenv("BBSI_GRAPHS");
  return !(e && e[0] == '0');
}

template <class F>
cudaError_t run_graphed(const std::string& key, cudaStream_t s, F&& enqueue) {
  if (!graphs_enabled() || prof_enabled() || s == nullptr) return enqueue(s);
  GraphEntry ent;
  bool seen = false;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = g_graphs.find(key);
    if (it == g_graphs.end()) {
      g_graphs.emplace(key, GraphEntry{});
    } else {
      seen = true;
      ent = it->second;
    }
  }
  if (!seen) return enqueue(s);  // first call: eager
  if (ent.exec) {
    launch_count_add(ent.launches);
    return cudaGraphLaunch(ent.exec, s);
  }
  // second call: capture (keys are per host thread, so no other thread captures this one)
  const long long c0 = launch_count();
  auto forget = [&] {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    g_graphs.erase(key);
  };
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (e) return e;
  cudaError_t e2 = enqueue(s);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(s, &g);
  if (e2 || e) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    forget();  // fall back to eager launches for this key
    return enqueue(s);
  }
  cudaGraphExec_t x = nullptr;
  e = cudaGraphInstantiate(&x, g, 0);
  cudaGraphDestroy(g);
  if (e) {
    cudaGetLastError();
    forget();
    return enqueue(s);
  }
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    g_graphs[key] = GraphEntry{x, launch_count() - c0};
  }
  return cudaGraphLaunch(x, s);
}

// Graph keys name the device and the host thread (workspaces are per thread) plus the
// shapes and every device pointer the launch sequence touches.
std::string graph_key(const char* tag, std::initializer_list<long long> v) {
  std::string k(tag);
  int dev = 0;
  cudaGetDevice(&dev);
  thread_local const unsigned long long tid = [] {
    static std::atomic<unsigned long long> next{0};
    return next++;
  }();
  k += ":" + std::to_string(dev) + ":t" + std::to_string(tid);
  for (long long x : v) k += ":" + std::to_string(x);
  return k;
}

// Runs the batched sweeps on a device band (already holding A) with the arena scratch.
int run_sweeps(SweepWork& W, const std::vector<int>& n_true, std::vector<int>& fails, cudaStream_t s) {
  W.groups = default_groups(W.batch, W.bs);
  void* scratch = arena_get(1, sweep_scratch_bytes(W.l, W.w, W.bs, W.batch, W.groups));
  if (!scratch) return fail(BBSI_OUT_OF_MEMORY, "sweep workspace allocation failed");
  sweep_carve(W, scratch);
  CK(rgf_sweeps(W, n_true.data(), s));
  CK(collect_failures(W, fails, s));
  return BBSI_OK;
}

// Single-matrix drop-in solve of the padded band (shared by tridiag/ndiag/fused).
int solve_host(const HostBand& h, double2* Gout, int* fail_layer) {
  if (int rc = device_ok()) return rc;
  const int bp = pad64(h.bs);
  std::vector<double2> staging;
  pad_band(h, bp, staging);
  const size_t bytes = staging.size() * sizeof(double2);
  double2* dG = static_cast<double2*>(arena_get(0, bytes));
  if (!dG) return fail(BBSI_OUT_OF_MEMORY, "band allocation failed");
  cudaStream_t s = thread_stream(0);
  CK(cudaMemcpyAsync(dG, staging.data(), bytes, cudaMemcpyHostToDevice, s));
  SweepWork W;
  W.l = h.l;
  W.w = h.w;
  W.bs = bp;
  W.batch = 1;
  W.G = dG;
  W.g_bstride = (long long)h.l * (2 * h.w + 1) * bp * bp;
  std::vector<int> fails;
  if (int rc = run_sweeps(W, h.sz, fails, s)) return rc;
  CK(cudaMemcpyAsync(staging.data(), dG, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (fails[0] >= 0) {
    if (fail_layer) *fail_layer = fails[0];
    return fail(BBSI_SINGULAR, "singular Schur pivot at layer " + std::to_string(fails[0]));
  }
  unpad_band(staging, bp, h, Gout);
  return BBSI_OK;
}

HostBand make_host(int l, int w, int bs, const int* sizes, const double* A) {
  HostBand h{l, w, bs, {}, reinterpret_cast<const double2*>(A)};
  h.sz.resize(l);
  for (int a = 0; a < l; ++a) h.sz[a] = sizes ? sizes[a] : bs;
  return h;
}

}  // namespace

extern "C" {

int bbsi_cuda_version(void) { return 100; }
const char* bbsi_cuda_last_error(void) { return g_err.c_str(); }

int bbsi_cuda_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void bbsi_cuda_release_workspace(void) { arena_release_all(); }

int bbsi_cuda_rgf_ndiag_z(int l, int w, int bs, const int* sizes, const double* A, double* G, long long* counters,
                          int* max_update_offset, int* fail_layer) {
  if (fail_layer) *fail_layer = -1;
  if (int rc = validate_layout(l, w, bs, sizes)) return rc;
  if (w < 1 && l != 1) return fail(BBSI_INVALID_ARGUMENT, "rgf_ndiag: requires bandwidth >= 1");
  HostBand h = make_host(l, w, bs, sizes, A);
  if (int rc = solve_host(h, reinterpret_cast<double2*>(G), fail_layer)) return rc;
  if (l == 1) {
    put_counters(counters, 0, 1, 1);  // predict_rgf_counters(1) (cost_model.hpp:47-49)
  } else {
    long long L = l, W = w;
    put_counters(counters, (3 * W * W + W) * L - 2 * W * W * W - 2 * W * W, L, L * (2 * W + 1) - W * W - W);
    if (max_update_offset) *max_update_offset = w - 1;
  }
  return BBSI_OK;
}

int bbsi_cuda_rgf_tridiag_z(int l, int w, int bs, const int* sizes, const double* A, double* G, long long* counters,
                            int* fail_layer) {
  if (fail_layer) *fail_layer = -1;
  if (int rc = validate_layout(l, w, bs, sizes)) return rc;
  if (w != 1 && l != 1) return fail(BBSI_INVALID_ARGUMENT, "rgf_tridiag: requires bandwidth 1");
  HostBand h = make_host(l, w, bs, sizes, A);
  if (int rc = solve_host(h, reinterpret_cast<double2*>(G), fail_layer)) return rc;
  long long L = l;
  put_counters(counters, 4 * (L - 1), L, 3 * L - 2);
  return BBSI_OK;
}

int bbsi_cuda_rgf_fused_z(int l, int w, int bs, const int* sizes, const double* A, double* G, long long* counters,
                          int* fail_layer) {
  if (fail_layer) *fail_layer = -1;
  if (int rc = validate_layout(l, w, bs, sizes)) return rc;
  if (w < 1 && l != 1) return fail(BBSI_INVALID_ARGUMENT, "rgf_fused: requires bandwidth >= 1");
  for (int a = 0; a < l; ++a)
    if ((sizes ? sizes[a] : bs) != (sizes ? sizes[0] : bs))
      return fail(BBSI_INVALID_ARGUMENT, "rgf_fused: requires uniform block sizes");
  if (w <= 1) return bbsi_cuda_rgf_tridiag_z(l, w, bs, sizes, A, G, counters, fail_layer);
  // rgf.hpp:152-191: super-layer s holds layers [s*w, min(l, s*w+w)).
  const int b = sizes ? sizes[0] : bs;
  const int lp = (l + w - 1) / w;
  std::vector<int> fsz(lp);
  for (int s = 0; s < lp; ++s) fsz[s] = (std::min(l, s * w + w) - s * w) * b;
  const int fbs = w * b;
  const int fw = lp == 1 ? 0 : 1;
  const long long fbb = (long long)fbs * fbs;
  std::vector<double2> fused(size_t(lp) * (2 * fw + 1) * fbb, make_double2(0.0, 0.0));
  HostBand h = make_host(l, w, bs, sizes, A);
  auto fslot = [&](int s, int off) { return fused.data() + ((long long)s * (2 * fw + 1) + off + fw) * fbb; };
  for (int a = 0; a < l; ++a)
    for (int off = -w; off <= w; ++off) {
      if (!h.in_band(a, off)) continue;
      const int c = a + off;
      double2* dst = fslot(a / w, c / w - a / w);
      const double2* src = h.slot(a, off);
      const int r0 = (a % w) * b, c0 = (c % w) * b;
      for (int j = 0; j < b; ++j)
        std::memcpy(dst + (long long)(c0 + j) * fbs + r0, src + (long long)j * bs, sizeof(double2) * b);
    }
  std::vector<double2> gf(fused.size());
  HostBand fh = make_host(lp, fw, fbs, fsz.data(), reinterpret_cast<const double*>(fused.data()));
  // a singular pivot reports the super-layer, as rgf_tridiag(fused) does in the reference
  if (int rc = solve_host(fh, gf.data(), fail_layer)) return rc;
  double2* Go = reinterpret_cast<double2*>(G);
  std::memset(Go, 0, sizeof(double2) * size_t(l) * (2 * w + 1) * bs * bs);
  for (int a = 0; a < l; ++a)
    for (int off = -w; off <= w; ++off) {
      if (!h.in_band(a, off)) continue;
      const int c = a + off;
      const double2* src = gf.data() + ((long long)(a / w) * (2 * fw + 1) + (c / w - a / w) + fw) * fbb;
      double2* dst = Go + ((long long)a * (2 * w + 1) + off + w) * bs * bs;
      const int r0 = (a % w) * b, c0 = (c % w) * b;
      for (int j = 0; j < b; ++j)
        std::memcpy(dst + (long long)j * bs, src + (long long)(c0 + j) * fbs + r0, sizeof(double2) * b);
    }
  long long L = lp;
  put_counters(counters, 4 * (L - 1), L, 3 * L - 2);
  return BBSI_OK;
}

// Many independent matrices of one layout in one call (an energy loop that built its
// A(E) on the host): every matrix is padded, the batch is solved by the batched sweeps in
// the reference's one-ended order (so fail_layers[k] is the layer rgf_tridiag /
// rgf_ndiag would report for matrix k), and the results come back in one pass.
int bbsi_cuda_rgf_many_z(int l, int w, int bs, const int* sizes, int batch, const double* A, double* G,
                         long long* counters, int* fail_layers) {
  if (int rc = validate_layout(l, w, bs, sizes)) return rc;
  if (w < 1 && l != 1) return fail(BBSI_INVALID_ARGUMENT, "rgf_ndiag: requires bandwidth >= 1");
  if (batch < 1) return fail(BBSI_INVALID_ARGUMENT, "batch must be >= 1");
  if (int rc = device_ok()) return rc;
  const int bp = pad64(bs);
  const size_t band_h = size_t(l) * (2 * w + 1) * bs * bs;  // complex per host band
  const size_t band_d = size_t(l) * (2 * w + 1) * bp * bp;
  double2* dG = static_cast<double2*>(arena_get(0, band_d * batch * sizeof(double2)));
  if (!dG) return fail(BBSI_OUT_OF_MEMORY, "band allocation failed");
  cudaStream_t s = thread_stream(0);
  std::vector<double2> staging;
  std::vector<int> sz;
  for (int k = 0; k < batch; ++k) {
    HostBand h = make_host(l, w, bs, sizes, A + 2 * band_h * k);
    pad_band(h, bp, staging);
    // on the sweep's own (non-blocking) stream: a synchronous cudaMemcpy from pageable memory returns once
    // the data is staged, before the DMA lands, and orders nothing against a non-blocking stream
    CK(cudaMemcpyAsync(dG + band_d * k, staging.data(), band_d * sizeof(double2), cudaMemcpyHostToDevice, s));
    if (k == 0) sz = h.sz;
  }
  SweepWork W;
  W.l = l;
  W.w = w;
  W.bs = bp;
  W.batch = batch;
  W.G = dG;
  W.g_bstride = (long long)band_d;
  std::vector<int> fails;
  if (int rc = run_sweeps(W, sz, fails, s)) return rc;
  bool bad = false;
  for (int k = 0; k < batch; ++k) {
    if (fail_layers) fail_layers[k] = fails[k];
    bad |= fails[k] >= 0;
    if (fails[k] >= 0) continue;
    staging.resize(band_d);
    CK(cudaMemcpy(staging.data(), dG + band_d * k, band_d * sizeof(double2), cudaMemcpyDeviceToHost));
    HostBand h = make_host(l, w, bs, sizes, A + 2 * band_h * k);
    unpad_band(staging, bp, h, reinterpret_cast<double2*>(G) + band_h * k);
  }
  long long L = l, Wd = w;
  if (l == 1)
    put_counters(counters, 0, 1, 1);
  else if (w == 1)
    put_counters(counters, 4 * (L - 1), L, 3 * L - 2);
  else
    put_counters(counters, (3 * Wd * Wd + Wd) * L - 2 * Wd * Wd * Wd - 2 * Wd * Wd, L, L * (2 * Wd + 1) - Wd * Wd - Wd);
  return bad ? fail(BBSI_SINGULAR, "singular Schur pivot in at least one matrix") : BBSI_OK;
}

int bbsi_cuda_rgf_batched_dev(int l, int w, int bs, int batch, const double* dA, long long a_bstride, double* dG,
                              int* fail_layers, void* stream) {
  if (int rc = validate_layout(l, w, bs, nullptr)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (w < 1 && l != 1) return fail(BBSI_INVALID_ARGUMENT, "rgf_ndiag: requires bandwidth >= 1");
  if (batch < 1) return fail(BBSI_INVALID_ARGUMENT, "batch must be >= 1");
  if (int rc = device_ok()) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long band = (long long)l * (2 * w + 1) * bs * bs;
  CK(cudaMemcpy2DAsync(dG, band * sizeof(double2), dA, a_bstride * sizeof(double2), band * sizeof(double2), batch,
                       cudaMemcpyDeviceToDevice, s));
  SweepWork W;
  W.l = l;
  W.w = w;
  W.bs = bs;
  W.batch = batch;
  W.G = reinterpret_cast<double2*>(dG);
  W.g_bstride = band;
  std::vector<int> nt(l, bs), fails;
  if (int rc = run_sweeps(W, nt, fails, s)) return rc;
  bool bad = false;
  for (int b = 0; b < batch; ++b) {
    if (fail_layers) fail_layers[b] = fails[b];
    bad |= fails[b] >= 0;
  }
  return bad ? fail(BBSI_SINGULAR, "singular Schur pivot in at least one batch entry") : BBSI_OK;
}

// Dyson diagonal blocks formed inside the first Schur-update GEMM (BBSI_FORM_IN_GEMM=0: a
// separate pass over every diagonal block first).
static bool form_in_gemm() {
  static const bool on = [] {
    const char* e = getenv("BBSI_FORM_IN_GEMM");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// The two-ended sweep eliminates layers in another order than rgf_tridiag / rgf_ndiag
// (rgf.hpp:58-64, 100-114), so its pivots are different matrices: an energy whose
// two-ended sweep hits a negligible pivot is re-solved with the reference's one-ended
// order. Either that succeeds (its band replaces the failed one) or it reports the layer
// the reference would (*fail_layer).
static cudaError_t dyson_retry_one_ended(int l, int w, int bs, const double2* dH, const double2* dz,
                                         const double2* dsig, double2* dGb, int* fail_layer, cudaStream_t s) {
  SweepWork W;
  W.l = l;
  W.w = w;
  W.bs = bs;
  W.batch = 1;
  W.G = dGb;
  W.g_bstride = (long long)l * (2 * w + 1) * bs * bs;
  W.groups = 1;
  W.two_ended = false;
  void* scr = arena_get(19, sweep_scratch_bytes(l, w, bs, 1, 1, false));
  if (!scr) return cudaErrorMemoryAllocation;
  sweep_carve(W, scr);
  cudaError_t e = dyson_form_band(dGb, dH, l, w, bs, 1, dz, dsig, s);
  if (e) return e;
  std::vector<int> nt(l, bs), fails;
  if ((e = rgf_sweeps(W, nt.data(), s))) return e;
  if ((e = collect_failures(W, fails, s))) return e;
  *fail_layer = fails[0];
  return cudaSuccess;
}

int bbsi_cuda_dyson_rgf_dev(int l, int w, int bs, int n_energy, const double* dH, const double* z,
                            const double* sigma, double* dG, int* fail_layers, void* stream) {
  if (int rc = validate_layout(l, w, bs, nullptr)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (w < 1 && l != 1) return fail(BBSI_INVALID_ARGUMENT, "rgf_ndiag: requires bandwidth >= 1");
  if (n_energy < 1) return fail(BBSI_INVALID_ARGUMENT, "n_energy must be >= 1");
  if (int rc = device_ok()) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double2* dzs = static_cast<double2*>(arena_get(2, sizeof(double2) * (size_t(n_energy) + l)));
  if (!dzs) return fail(BBSI_OUT_OF_MEMORY, "parameter upload allocation failed");
  CK(cudaMemcpyAsync(dzs, z, sizeof(double2) * n_energy, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dzs + n_energy, sigma, sizeof(double2) * l, cudaMemcpyHostToDevice, s));
  SweepWork W;
  W.l = l;
  W.w = w;
  W.bs = bs;
  W.batch = n_energy;
  W.G = reinterpret_cast<double2*>(dG);
  W.g_bstride = (long long)l * (2 * w + 1) * bs * bs;
  W.groups = dyson_groups(W.batch);
  W.two_ended = two_ended_default();
  void* scratch = arena_get(1, sweep_scratch_bytes(W.l, W.w, W.bs, W.batch, W.groups, W.two_ended));
  if (!scratch) return fail(BBSI_OUT_OF_MEMORY, "sweep workspace allocation failed");
  sweep_carve(W, scratch);
  std::vector<int> nt(l, bs), fails;
  const std::string key = graph_key("dyson", {l, w, bs, n_energy, (long long)dH, (long long)dG, (long long)dzs,
                                              (long long)scratch, W.groups, W.two_ended});
  // tridiagonal: the sweeps read A's off-diagonal blocks (-H) from the shared H, so only
  // the diagonal blocks of each energy's band are formed
  if (w == 1) W.Hoff = reinterpret_cast<const double2*>(dH);
  if (W.Hoff && form_in_gemm()) {
    W.zdev = dzs;
    W.sigdev = dzs + n_energy;
  }
  CK(run_graphed(key, s, [&](cudaStream_t st) -> cudaError_t {
    double2* g = reinterpret_cast<double2*>(dG);
    const double2* h = reinterpret_cast<const double2*>(dH);
    cudaError_t e = W.zdev  ? dyson_form_diag_ends(g, h, l, w, bs, n_energy, dzs, dzs + n_energy,
                                                   sweep_is_two_ended(W), st)
                    : W.Hoff ? dyson_form_diag(g, h, l, w, bs, n_energy, dzs, dzs + n_energy, st)
                             : dyson_form_band(g, h, l, w, bs, n_energy, dzs, dzs + n_energy, st);
    return e ? e : rgf_sweeps(W, nt.data(), st);
  }));
  CK(collect_failures(W, fails, s));
  bool bad = false;
  for (int b = 0; b < n_energy; ++b) {
    if (fails[b] >= 0 && sweep_is_two_ended(W))
      CK(dyson_retry_one_ended(l, w, bs, reinterpret_cast<const double2*>(dH), dzs + b, dzs + n_energy,
                               reinterpret_cast<double2*>(dG) + size_t(b) * W.g_bstride, &fails[b], s));
    if (fail_layers) fail_layers[b] = fails[b];
    bad |= fails[b] >= 0;
  }
  return bad ? fail(BBSI_SINGULAR, "singular Schur pivot in at least one energy") : BBSI_OK;
}

// Dyson batch with full lead self-energy blocks: A_e = z_e I - H - Sigma_e, where Sigma_e
// is a full bs x bs block on each of the first and last w layers (energy dependent, as
// lead self-energies are): dSigma [n_energy][2w][bs][bs] (layers 0..w-1, then l-w..l-1).
int bbsi_cuda_dyson_rgf_sigma_dev(int l, int w, int bs, int n_energy, const double* dH, const double* z,
                                  const double* dSigma, double* dG, int* fail_layers, void* stream) {
  if (int rc = validate_layout(l, w, bs, nullptr)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (w < 1 || l < 2 * w) return fail(BBSI_INVALID_ARGUMENT, "Sigma blocks need l >= 2w and w >= 1");
  if (n_energy < 1) return fail(BBSI_INVALID_ARGUMENT, "n_energy must be >= 1");
  if (int rc = device_ok()) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double2* dzs = static_cast<double2*>(arena_get(2, sizeof(double2) * (size_t(n_energy) + l)));
  if (!dzs) return fail(BBSI_OUT_OF_MEMORY, "parameter upload allocation failed");
  CK(cudaMemcpyAsync(dzs, z, sizeof(double2) * n_energy, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(dzs + n_energy, 0, sizeof(double2) * l, s));  // scalar sigma 0: the blocks come next
  double2* G = reinterpret_cast<double2*>(dG);
  const long long bb = (long long)bs * bs, band = (long long)l * (2 * w + 1) * bb;
  CK(dyson_form_band(G, reinterpret_cast<const double2*>(dH), l, w, bs, n_energy, dzs, dzs + n_energy, s));
  // A[a, a] -= Sigma_e[a] on the 2w boundary layers
  const double2* Sg = reinterpret_cast<const double2*>(dSigma);
  for (int q = 0; q < 2 * w; ++q) {
    const int a = q < w ? q : l - 2 * w + q;
    CK(axpy_strided(G + ((long long)a * (2 * w + 1) + w) * bb, band, Sg + (long long)q * bb, 2LL * w * bb, bb,
                    n_energy, make_double2(-1.0, 0.0), s));
  }
  SweepWork W;
  W.l = l;
  W.w = w;
  W.bs = bs;
  W.batch = n_energy;
  W.G = G;
  W.g_bstride = band;
  W.groups = dyson_groups(W.batch);
  W.two_ended = two_ended_default();
  void* scratch = arena_get(1, sweep_scratch_bytes(W.l, W.w, W.bs, W.batch, W.groups, W.two_ended));
  if (!scratch) return fail(BBSI_OUT_OF_MEMORY, "sweep workspace allocation failed");
  sweep_carve(W, scratch);
  std::vector<int> nt(l, bs), fails;
  CK(rgf_sweeps(W, nt.data(), s));
  CK(collect_failures(W, fails, s));
  bool bad = false;
  for (int b = 0; b < n_energy; ++b) {
    if (fails[b] >= 0) bad = true;
    if (fail_layers) fail_layers[b] = fails[b];
  }
  return bad ? fail(BBSI_SINGULAR, "singular Schur pivot in at least one energy") : BBSI_OK;
}

int bbsi_cuda_dyson_fill_h_dev(int l, int w, int b, uint64_t seed, double* dH, void* stream) {
  if (int rc = validate_layout(l, w, b, nullptr)) return rc;
  if (int rc = device_ok()) return rc;
  CK(dyson_fill_h(reinterpret_cast<double2*>(dH), l, w, b, seed, static_cast<cudaStream_t>(stream)));
  return BBSI_OK;
}

int bbsi_cuda_dyson_fill_h_rows_dev(int l, int w, int b, uint64_t seed, int a0, int a1, double* dH, void* stream) {
  if (int rc = validate_layout(l, w, b, nullptr)) return rc;
  if (a0 < 0 || a1 > l || a0 >= a1) return fail(BBSI_INVALID_ARGUMENT, "bad row range");
  if (int rc = device_ok()) return rc;
  CK(dyson_fill_h_rows(reinterpret_cast<double2*>(dH), l, w, b, seed, a0, a1, static_cast<cudaStream_t>(stream)));
  return BBSI_OK;
}

void bbsi_dyson_fill_h_host(int l, int w, int b, uint64_t seed, double* H) {
  const uint64_t sm = bbsi_mix64(seed);
  const long long bb = (long long)b * b;
  for (int a = 0; a < l; ++a)
    for (int off = -w; off <= w; ++off) {
      double* d = H + 2 * ((long long)a * (2 * w + 1) + off + w) * bb;
      const bool in = a + off >= 0 && a + off < l;
      for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) {
          double re = 0.0, im = 0.0;
          if (in) bbsi_h_entry(sm, b, a, off, i, j, &re, &im);
          d[2 * ((long long)j * b + i)] = re;
          d[2 * ((long long)j * b + i) + 1] = im;
        }
    }
}

int bbsi_random_spd_like_z(int l, int w, int bs, const int* sizes, uint64_t seed, double dominance, double* A) {
  if (int rc = validate_layout(l, w, bs, sizes)) return rc;
  if (!(dominance > 0.0)) return fail(BBSI_INVALID_ARGUMENT, "random_spd_like: dominance must be positive");
  using cd = std::complex<double>;
  std::vector<int> sz(l, bs);
  if (sizes)
    for (int a = 0; a < l; ++a) sz[a] = sizes[a];
  const long long bb = (long long)bs * bs;
  cd* m = reinterpret_cast<cd*>(A);
  std::memset(A, 0, sizeof(cd) * size_t(l) * (2 * w + 1) * bb);
  auto blk = [&](int a, int off) { return m + ((long long)a * (2 * w + 1) + off + w) * bb; };
  auto in_band = [&](int a, int off) { return a + off >= 0 && a + off < l; };
  std::mt19937_64 rng(seed);
  auto next_real = [&] { return double(rng() >> 11) * (2.0 / 9007199254740992.0) - 1.0; };
  for (int a = 0; a < l; ++a)
    for (int off = -w; off <= w; ++off)
      if (in_band(a, off)) {
        cd* p = blk(a, off);
        for (int j = 0; j < sz[a + off]; ++j)
          for (int i = 0; i < sz[a]; ++i) {
            const double re = next_real();
            const double im = next_real();
            p[(long long)j * bs + i] = cd(re, im);
          }
      }
  for (int a = 0; a < l; ++a) {
    cd* diag = blk(a, 0);
    for (int i = 0; i < sz[a]; ++i) {
      double row_sum = 0.0;
      for (int off = -w; off <= w; ++off) {
        if (!in_band(a, off)) continue;
        const cd* p = blk(a, off);
        for (int j = 0; j < sz[a + off]; ++j) {
          if (off == 0 && j == i) continue;
          row_sum += std::abs(p[(long long)j * bs + i]);
        }
      }
      const cd d = diag[(long long)i * bs + i];
      const double mag = std::abs(d);
      const cd phase = mag > 1e-12 ? d / cd(mag) : cd(1);
      diag[(long long)i * bs + i] = d + phase * cd(dominance * row_sum);
    }
  }
  return BBSI_OK;
}

int bbsi_cuda_zgemm_dev(int m, int n, int k, const double* alpha, const double* dA, long long lda, long long a_bstride,
                        const double* dB, long long ldb, long long b_bstride, const double* beta, double* dC,
                        long long ldc, long long c_bstride, int batch, void* stream) {
  if (m < 1 || n < 1 || k % 16 || k < 16 || batch < 1)
    return fail(BBSI_INVALID_ARGUMENT, "zgemm: requires m, n >= 1 and k % 16 == 0");
  if (int rc = device_ok()) return rc;
  // plain column-major matrices as 64 x 64 block operands
  ZGemmGroup g{};
  g.batch = batch;
  g.bs = 64;
  g.nprob = 1;
  ZGemmProblem& p = g.prob[0];
  p.M = m;
  p.N = n;
  p.K = k;
  p.alpha = make_double2(alpha[0], alpha[1]);
  p.beta = make_double2(beta[0], beta[1]);
  p.A = ZOp{reinterpret_cast<const double2*>(dA), lda, 64, 64 * lda, a_bstride};
  p.B = ZOp{reinterpret_cast<const double2*>(dB), ldb, 64, 64 * ldb, b_bstride};
  p.C = ZOp{reinterpret_cast<const double2*>(dC), ldc, 64, 64 * ldc, c_bstride};
  p.D = p.C;
  CK(zgemm_grouped(g, static_cast<cudaStream_t>(stream)));
  return BBSI_OK;
}

int bbsi_cuda_zinv_dev(int n, int n_true, int batch, double* dM, long long ld, long long bstride, int* status_host,
                       void* stream) {
  if (n % 64 || n_true < 1 || n_true > n || batch < 1)
    return fail(BBSI_INVALID_ARGUMENT, "zinv: requires n % 64 == 0 and 1 <= n_true <= n");
  if (int rc = device_ok()) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  size_t scr = zinv_scratch_bytes(n, batch) + sizeof(int) * batch + 256;
  char* base = static_cast<char*>(arena_get(3, scr));
  if (!base) return fail(BBSI_OUT_OF_MEMORY, "zinv scratch allocation failed");
  int* st = reinterpret_cast<int*>(base + zinv_scratch_bytes(n, batch));
  CK(zinv_batched(reinterpret_cast<double2*>(dM), ld, bstride, n, n_true, batch, base, st, s));
  if (status_host) {
    CK(cudaMemcpyAsync(status_host, st, sizeof(int) * batch, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return BBSI_OK;
}

long long bbsi_cuda_launch_count(void) { return launch_count(); }

void bbsi_cuda_profile_enable(int on) { prof_enable(on != 0); }

int bbsi_cuda_profile_collect(double* out, int ncat) {
  if (!out || ncat < 1) return fail(BBSI_INVALID_ARGUMENT, "profile_collect: bad output buffer");
  return prof_collect(out, ncat);
}

int bbsi_cuda_bench_kernels(int n, int batch, int samples, double* out) {
  if (n < 64 || n % 64 || batch < 1 || samples < 1 || !out)
    return fail(BBSI_INVALID_ARGUMENT, "bench_kernels: requires n % 64 == 0, batch >= 1, samples >= 1");
  if (int rc = device_ok()) return rc;
  const long long nn = (long long)n * n;
  const size_t scr = zinv_scratch_bytes(n, batch) + sizeof(int) * batch + 256;
  double2* buf = static_cast<double2*>(arena_get(3, scr));
  double2* mats = static_cast<double2*>(arena_get(16, 4 * size_t(nn) * batch * sizeof(double2)));
  if (!buf || !mats) return fail(BBSI_OUT_OF_MEMORY, "bench_kernels: allocation failed");
  int* st = reinterpret_cast<int*>(reinterpret_cast<char*>(buf) + zinv_scratch_bytes(n, batch));
  double2 *A = mats, *B = mats + nn * batch, *Cm = mats + 2 * nn * batch, *M = mats + 3 * nn * batch;
  // diagonally dominant seeded operands (inversion well defined); timing only
  CK(dyson_fill_h(A, 1, 0, n, 7, nullptr));
  for (int b = 1; b < batch; ++b) CK(cudaMemcpy(A + b * nn, A, nn * sizeof(double2), cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(B, A, nn * batch * sizeof(double2), cudaMemcpyDeviceToDevice));
  double2* zs = static_cast<double2*>(arena_get(2, sizeof(double2) * (size_t(batch) + 1)));
  if (!zs) return fail(BBSI_OUT_OF_MEMORY, "bench_kernels: allocation failed");
  std::vector<double2> zh(batch + 1, make_double2(3.0 * n, 0.0));  // z_e = 3n; sigma = 0
  zh[batch] = make_double2(0.0, 0.0);
  CK(cudaMemcpy(zs, zh.data(), zh.size() * sizeof(double2), cudaMemcpyHostToDevice));
  CK(dyson_form_diag(M, A, 1, 0, n, batch, zs, zs + batch, nullptr));
  ZGemmGroup g{};
  g.batch = batch;
  g.bs = n;
  g.nprob = 1;
  ZGemmProblem& p = g.prob[0];
  p.M = p.N = p.K = n;
  p.alpha = make_double2(1.0, 0.0);
  p.beta = make_double2(0.0, 0.0);
  p.A = ZOp{A, n, nn, nn, nn};
  p.B = ZOp{B, n, nn, nn, nn};
  p.C = p.D = ZOp{Cm, n, nn, nn, nn};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timed = [&](auto&& launch) -> double {
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < samples; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return 1e-3 * ms / samples;
  };
  // the inversion runs in place: every sample inverts the previous result (same cost)
  out[0] = timed([&] { zgemm_grouped(g, nullptr); });
  out[1] = timed([&] { zinv_batched(M, n, nn, n, n, batch, buf, st, nullptr); });
  out[2] = samples;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CK(cudaGetLastError());
  return BBSI_OK;
}

double bbsi_cuda_fp64_peak_tflops(double duration_ms, int reps) {
  if (device_ok()) return -1.0;
  return fp64_dmma_peak(duration_ms, reps < 1 ? 1 : reps);
}

// End-to-end Dyson batch from HOST buffers: H2D of H, energy chunks computed on
// one stream while the finished chunks' G bands stream back to the host on a
// second stream (pinned G_host gives full overlap).
// Band rows per host hand-off of the streamed downward sweep (env BBSI_E2E_ROWS).
static int e2e_rows() {
  const char* e = getenv("BBSI_E2E_ROWS");
  const int v = e ? atoi(e) : 0;
  return v > 0 ? v : 8;
}

// Persistent compute / copy streams of the host-buffer path (per device) and a pinned
// staging buffer for z and sigma.
struct E2eStreams {
  cudaStream_t sc = nullptr, sd = nullptr;
};
static E2eStreams& e2e_streams() {
  thread_local std::vector<E2eStreams> v;  // per host thread
  int dev = 0;
  cudaGetDevice(&dev);
  if (int(v.size()) <= dev) v.resize(dev + 1);
  if (!v[dev].sc) {
    cudaStreamCreateWithFlags(&v[dev].sc, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&v[dev].sd, cudaStreamNonBlocking);
  }
  return v[dev];
}
static double2* e2e_stage(size_t n) {
  thread_local std::vector<std::pair<double2*, size_t>> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  if (int(per_dev.size()) <= dev) per_dev.resize(dev + 1, {nullptr, 0});
  auto& b = per_dev[dev];
  if (b.second < n) {
    if (b.first) {
      cudaDeviceSynchronize();
      cudaFreeHost(b.first);
    }
    b = {nullptr, 0};
    void* p = nullptr;
    if (cudaHostAlloc(&p, n * sizeof(double2), cudaHostAllocDefault) != cudaSuccess) return nullptr;
    b = {static_cast<double2*>(p), n};
  }
  return b.first;
}
static bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int bbsi_cuda_dyson_rgf_z(int l, int w, int bs, int n_energy, const double* H, const double* z, const double* sigma,
                          double* G, int* fail_layers, int chunk) {
  if (int rc = validate_layout(l, w, bs, nullptr)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "Dyson batch requires bs % 64 == 0");
  if (w < 1 && l != 1) return fail(BBSI_INVALID_ARGUMENT, "rgf_ndiag: requires bandwidth >= 1");
  if (n_energy < 1) return fail(BBSI_INVALID_ARGUMENT, "n_energy must be >= 1");
  if (int rc = device_ok()) return rc;
  const long long band = (long long)l * (2 * w + 1) * bs * bs;
  const size_t band_b = size_t(band) * sizeof(double2);
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  free_b += arena_held({1, 4, 5});  // this call's own workspace slots are reused or regrown
  // Default: chunks of at most 12 energies once there are >= 24. Measured on B200,
  // config 2, CUDA-graph replay, e2e time above the box's PCIe copy floor (0.90-0.99 s):
  // chunks of 8 / 10 / 12 / 16 / 20 / 24 / 32 energies +155 / +130 / +140..177 / +119..155
  // / +194 / +188 / +200 ms; one chunk of 64 (eager) 1.27 s. The G stream starts when the
  // first chunk's rows are final and then stays busy while later chunks compute; with
  // smaller chunks the compute falls behind the copy. Smaller chunks when HBM is short.
  if (chunk <= 0 || chunk > n_energy) {
    const int nc = (n_energy + 11) / 12;
    chunk = n_energy >= 24 ? (n_energy + nc - 1) / nc : n_energy;
    while (chunk > 1 && (size_t(chunk) * band_b + band_b +
                         sweep_scratch_bytes(l, w, bs, chunk, default_groups(chunk, bs), two_ended_default())) > free_b * 9 / 10)
      chunk = (chunk + 1) / 2;
  }
  const int nchunk = (n_energy + chunk - 1) / chunk;
  // two groups per chunk here: the copy stream, not the sweeps, bounds this path, and
  // more groups hand it smaller pieces (graph replay, config 2: 2 / 4 / 8 / 16 groups
  // 1.112 / 1.113 / 1.120 / 1.148 s; eager with 16 groups: 2.38 s)
  const int groups = default_groups(chunk, bs);
  const size_t scr_b = sweep_scratch_bytes(l, w, bs, chunk, groups, two_ended_default());
  int nbuf = nchunk;
  while (nbuf > 1 && (size_t(nbuf) * chunk * band_b + band_b + scr_b) > free_b * 9 / 10) --nbuf;
  double2* dH = static_cast<double2*>(arena_get(4, band_b));
  double2* dG = static_cast<double2*>(arena_get(5, size_t(nbuf) * chunk * band_b));
  double2* dzs = static_cast<double2*>(arena_get(2, sizeof(double2) * (size_t(n_energy) + l)));
  void* scratch = arena_get(1, scr_b);
  // per-layer pivot status of every energy, [l][n_energy], read back once at the end
  // (a per-chunk read-back would queue behind the streamed G copies on the copy engine)
  int* dstat = static_cast<int*>(arena_get(15, sizeof(int) * size_t(l) * n_energy));
  if (!dH || !dG || !dzs || !scratch || !dstat)
    return fail(BBSI_OUT_OF_MEMORY, "Dyson batch workspace allocation failed");
  E2eStreams& es = e2e_streams();
  cudaStream_t sc = es.sc, sd = es.sd;
  if (!sc || !sd) return fail(BBSI_CUDA_ERROR, "stream creation failed");
  // z and sigma through a pinned staging buffer (the graph's copy nodes read it at replay)
  double2* zst = e2e_stage(size_t(n_energy) + l);
  if (!zst) return fail(BBSI_OUT_OF_MEMORY, "pinned staging allocation failed");
  std::memcpy(zst, z, sizeof(double2) * n_energy);
  std::memcpy(zst + n_energy, sigma, sizeof(double2) * l);
  std::vector<cudaEvent_t> done(nchunk), freed(nbuf);
  for (auto& e : done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : freed) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t rows_ev = nullptr;  // re-recorded per hand-off (each wait binds the current record)
  CK(cudaEventCreateWithFlags(&rows_ev, cudaEventDisableTiming));
  const size_t row_b = size_t(2 * w + 1) * bs * bs * sizeof(double2);
  std::vector<int> status(size_t(l) * n_energy, -1);
  // BBSI_E2E_TRACE=1: device timeline of the call on stderr (compute / copy streams)
  const bool trace = getenv("BBSI_E2E_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> tl;
  auto mark = [&](const std::string& what, cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tl.emplace_back(what, e);
  };
  bool first_copy = true;
  int rc = BBSI_OK;
  cudaEvent_t join = nullptr;
  CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  // everything the call puts on the GPU, on sc (compute) and sd (copies back), ending
  // with sc joined to sd: replayed as one CUDA graph when H and G are pinned
  auto enqueue = [&](cudaStream_t) -> cudaError_t {
    mark("start", sc);
    cudaError_t e;
    if ((e = cudaMemcpyAsync(dH, H, band_b, cudaMemcpyHostToDevice, sc))) return e;
    if ((e = cudaMemcpyAsync(dzs, zst, sizeof(double2) * (size_t(n_energy) + l), cudaMemcpyHostToDevice, sc))) return e;
    std::vector<int> nt(l, bs);
    for (int c = 0; c < nchunk; ++c) {
      const int e0 = c * chunk, ne = std::min(chunk, n_energy - e0), buf = c % nbuf;
      if (c >= nbuf && (e = cudaStreamWaitEvent(sc, freed[buf], 0))) return e;
      double2* g = dG + size_t(buf) * chunk * band;
      SweepWork W;
      W.l = l;
      W.w = w;
      W.bs = bs;
      W.batch = ne;
      W.G = g;
      W.g_bstride = band;
      W.groups = groups;
      W.two_ended = two_ended_default();
      if (w == 1) W.Hoff = dH;
      if (W.Hoff && form_in_gemm()) {
        W.zdev = dzs + e0;
        W.sigdev = dzs + n_energy;
      }
      sweep_carve(W, scratch);
      e = W.zdev    ? dyson_form_diag_ends(g, dH, l, w, bs, ne, dzs + e0, dzs + n_energy, sweep_is_two_ended(W), sc)
          : w == 1 ? dyson_form_diag(g, dH, l, w, bs, ne, dzs + e0, dzs + n_energy, sc)
                   : dyson_form_band(g, dH, l, w, bs, ne, dzs + e0, dzs + n_energy, sc);
      if (e) return e;
      W.status = dstat + e0;
      W.status_stride = n_energy;
      // finished band rows of the downward sweep -> host, on the copy stream, while the
      // sweep continues (one 2D copy per hand-off: rows [r0, r1) of ne_g energies)
      W.hook_rows = e2e_rows();
      W.rows_done = [&, g, e0](int r0, int r1, int eg, int ne_g, cudaStream_t st) -> cudaError_t {
        cudaError_t e = cudaEventRecord(rows_ev, st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, rows_ev, 0);
        if (e != cudaSuccess) return e;
        if (first_copy) mark("first D2H issued", sd);
        first_copy = false;
        char* dst = reinterpret_cast<char*>(G) + size_t(e0 + eg) * band_b + size_t(r0) * row_b;
        const char* src = reinterpret_cast<const char*>(g + size_t(eg) * band) + size_t(r0) * row_b;
        return cudaMemcpy2DAsync(dst, band_b, src, band_b, size_t(r1 - r0) * row_b, size_t(ne_g),
                                 cudaMemcpyDeviceToHost, sd);
      };
      if ((e = rgf_sweeps(W, nt.data(), sc))) return e;
      if ((e = cudaEventRecord(done[c], sc))) return e;
      mark("chunk " + std::to_string(c) + " computed", sc);
      if ((e = cudaStreamWaitEvent(sd, done[c], 0))) return e;
      if ((e = cudaEventRecord(freed[buf], sd))) return e;
      mark("chunk " + std::to_string(c) + " copied", sd);
    }
    if ((e = cudaEventRecord(join, sd))) return e;
    return cudaStreamWaitEvent(sc, join, 0);
  };
  auto body = [&]() -> int {
    const bool graphable = !trace && host_pinned(H) && host_pinned(G);
    if (graphable) {
      const std::string key = graph_key("e2e", {l, w, bs, n_energy, chunk, groups, nbuf, (long long)H, (long long)G,
                                                (long long)dH, (long long)dG, (long long)dzs, (long long)scratch,
                                                (long long)dstat, (long long)zst, e2e_rows(), two_ended_default()});
      CK(run_graphed(key, sc, enqueue));
    } else {
      CK(enqueue(sc));
    }
    CK(cudaStreamSynchronize(sc));
    CK(cudaMemcpy(status.data(), dstat, sizeof(int) * status.size(), cudaMemcpyDeviceToHost));
    return BBSI_OK;
  };
  rc = body();
  if (trace && !tl.empty()) {
    for (auto& [what, e] : tl) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tl[0].second, e);
      fprintf(stderr, "[e2e] %9.2f ms  %s\n", ms, what.c_str());
    }
    for (auto& pe : tl) cudaEventDestroy(pe.second);
  }
  for (auto& e : done) cudaEventDestroy(e);
  for (auto& e : freed) cudaEventDestroy(e);
  cudaEventDestroy(rows_ev);
  cudaEventDestroy(join);
  if (rc) return rc;
  bool bad = false;
  for (int e = 0; e < n_energy; ++e) {
    int f = -1;
    for (int j = l - 1; j >= 0; --j)
      if (status[size_t(j) * n_energy + e] >= 0) {
        f = j;
        break;
      }
    SweepWork Wt;
    Wt.l = l;
    Wt.w = w;
    Wt.two_ended = two_ended_default();
    if (f >= 0 && sweep_is_two_ended(Wt)) {  // see dyson_retry_one_ended
      double2* gb = static_cast<double2*>(arena_get(16, band_b));
      if (!gb) return fail(BBSI_OUT_OF_MEMORY, "retry band allocation failed");
      CK(dyson_retry_one_ended(l, w, bs, dH, dzs + e, dzs + n_energy, gb, &f, sc));
      if (f < 0) CK(cudaMemcpy(reinterpret_cast<char*>(G) + size_t(e) * band_b, gb, band_b, cudaMemcpyDeviceToHost));
    }
    if (fail_layers) fail_layers[e] = f;
    bad |= f >= 0;
  }
  return bad ? fail(BBSI_SINGULAR, "singular Schur pivot in at least one energy") : BBSI_OK;
}

// rgf_extended (rgf.hpp:209-270): the tridiagonal core plus the full first/last
// block rows and columns of the inverse. The reference carries whole columns and
// rows through the downward sweep ((l-1)(l-2) extra GEMMs); here they come from
// O(l) chains over the stored multipliers after the sweep:
//   first row  G[0,a]   = -G[0,a-1] um_a            (left to right)
//   first col  G[a,0]   = -lm_a G[a-1,0]
//   last col   G[a,l-1] = G[a,a] Q_a,  Q_a = -um_{a+1} Q_{a+1},  Q_{l-1} = I
//   last row   G[l-1,a] = R_a G[a,a],  R_a = -R_{a+1} lm_{a+1},  R_{l-1} = I
// with the entries that lie in the band copied from the core, as the reference does.
int bbsi_cuda_rgf_extended_z(int l, int w, int bs, const int* sizes, const double* A, double* G, double* first_row,
                             double* last_row, double* first_col, double* last_col, long long* counters,
                             int* fail_layer) {
  if (fail_layer) *fail_layer = -1;
  if (int rc = validate_layout(l, w, bs, sizes)) return rc;
  if (w != 1 && l != 1) return fail(BBSI_INVALID_ARGUMENT, "rgf_extended: requires bandwidth 1");
  if (int rc = device_ok()) return rc;
  HostBand h = make_host(l, w, bs, sizes, A);
  const int bp = pad64(h.bs);
  const long long bb = (long long)bp * bp;
  std::vector<double2> staging;
  pad_band(h, bp, staging);
  const size_t bytes = staging.size() * sizeof(double2);
  double2* dG = static_cast<double2*>(arena_get(0, bytes));
  double2* halo = static_cast<double2*>(arena_get(11, sizeof(double2) * size_t(4 * l + 4) * bb));
  if (!dG || !halo) return fail(BBSI_OUT_OF_MEMORY, "rgf_extended allocation failed");
  cudaStream_t s = thread_stream(0);
  CK(cudaMemcpyAsync(dG, staging.data(), bytes, cudaMemcpyHostToDevice, s));
  SweepWork W;
  W.l = l;
  W.w = w;
  W.bs = bp;
  W.batch = 1;
  W.G = dG;
  W.g_bstride = (long long)l * (2 * w + 1) * bb;
  std::vector<int> fails;
  if (int rc = run_sweeps(W, h.sz, fails, s)) return rc;
  if (fails[0] >= 0) {
    if (fail_layer) *fail_layer = fails[0];
    return fail(BBSI_SINGULAR, "singular Schur pivot at layer " + std::to_string(fails[0]));
  }
  const int ns = 2 * w + 1;
  auto gs = [&](int a, int off) { return dG + ((long long)a * ns + off + w) * bb; };
  double2* FR = halo;                 // [l]
  double2* LR = halo + (long long)l * bb;
  double2* FC = halo + 2LL * l * bb;
  double2* LC = halo + 3LL * l * bb;
  double2* Q = halo + 4LL * l * bb;   // [4] accumulators (P, S ping-pong)
  const double2 m1 = make_double2(-1.0, 0.0), p1 = make_double2(1.0, 0.0);
  auto cp = [&](double2* d, const double2* x) {
    return cudaMemcpyAsync(d, x, bb * sizeof(double2), cudaMemcpyDeviceToDevice, s);
  };
  auto um = [&](int a) { return W.UM + (long long)a * bb; };
  auto lm = [&](int a) { return W.LM + (long long)a * bb; };
  CK(cp(FR, gs(0, 0)));
  CK(cp(FC, gs(0, 0)));
  CK(cp(LC + (l - 1) * bb, gs(l - 1, 0)));
  CK(cp(LR + (l - 1) * bb, gs(l - 1, 0)));
  if (l >= 2) {
    CK(cp(FR + bb, gs(0, 1)));
    CK(cp(FC + bb, gs(1, -1)));
    CK(cp(LC + (l - 2) * bb, gs(l - 2, 1)));
    CK(cp(LR + (l - 2) * bb, gs(l - 1, -1)));
  }
  for (int a = 2; a < l; ++a) {
    CK(zmm(bp, 1, m1, zblk(FR + (a - 1) * bb, bp), zblk(um(a), bp), 0.0, zblk(FR + a * bb, bp), s));
    CK(zmm(bp, 1, m1, zblk(lm(a), bp), zblk(FC + (a - 1) * bb, bp), 0.0, zblk(FC + a * bb, bp), s));
  }
  if (l >= 3) {
    // P_a = um_{a+1} ... um_{l-1},  S_a = lm_{l-1} ... lm_{a+1};  sign (-1)^(l-1-a) applied at the end
    double2* Pp[2] = {Q, Q + bb};
    double2* Sp[2] = {Q + 2 * bb, Q + 3 * bb};
    CK(cp(Pp[0], um(l - 1)));
    CK(cp(Sp[0], lm(l - 1)));
    int cur = 0;
    for (int a = l - 3; a >= 0; --a) {
      CK(zmm(bp, 1, p1, zblk(um(a + 1), bp), zblk(Pp[cur], bp), 0.0, zblk(Pp[cur ^ 1], bp), s));
      CK(zmm(bp, 1, p1, zblk(Sp[cur], bp), zblk(lm(a + 1), bp), 0.0, zblk(Sp[cur ^ 1], bp), s));
      cur ^= 1;
      const double2 sg = ((l - 1 - a) % 2) ? m1 : p1;
      CK(zmm(bp, 1, sg, zblk(gs(a, 0), bp), zblk(Pp[cur], bp), 0.0, zblk(LC + a * bb, bp), s));
      CK(zmm(bp, 1, sg, zblk(Sp[cur], bp), zblk(gs(a, 0), bp), 0.0, zblk(LR + a * bb, bp), s));
    }
  }
  std::vector<double2> hh(size_t(4) * l * bb);
  CK(cudaMemcpyAsync(staging.data(), dG, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hh.data(), halo, hh.size() * sizeof(double2), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  unpad_band(staging, bp, h, reinterpret_cast<double2*>(G));
  // halo blocks: first_row[b]: rows(0) x cols(b); last_row[b]: rows(l-1) x cols(b);
  //              first_col[a]: rows(a) x cols(0); last_col[a]: rows(a) x cols(l-1)
  auto put = [&](double* dst, int which, int rows_of, int cols_of) {
    if (!dst) return;
    double2* d = reinterpret_cast<double2*>(dst);
    std::memset(d, 0, sizeof(double2) * size_t(l) * h.bs * h.bs);
    for (int k = 0; k < l; ++k) {
      const int r = rows_of >= 0 ? h.sz[rows_of] : h.sz[k];
      const int c = cols_of >= 0 ? h.sz[cols_of] : h.sz[k];
      const double2* src = hh.data() + ((size_t)which * l + k) * bb;
      for (int j = 0; j < c; ++j)
        std::memcpy(d + (size_t)k * h.bs * h.bs + (size_t)j * h.bs, src + (size_t)j * bp, sizeof(double2) * r);
    }
  };
  put(first_row, 0, 0, -1);
  put(last_row, 1, l - 1, -1);
  put(first_col, 2, -1, 0);
  put(last_col, 3, -1, l - 1);
  long long L = l;
  put_counters(counters, 4 * (L - 1) + (L <= 2 ? 0 : (L - 1) * (L - 2)), L, 3 * L - 2);
  return BBSI_OK;
}

// DomainPlan validation and plan exhaustion, as the reference (ddrgf.hpp:26-31,
// 364-366, 423-425; partition.hpp:41-45).
static int validate_ddrgf(int l, int w, int bs, const int* sizes, const int* s2_levels, int n_levels, int n_threads,
                          int terminal_threads) {
  if (n_levels < 1 || !s2_levels) return fail(BBSI_INVALID_ARGUMENT, "DomainPlan: needs at least one level");
  for (int k = 0; k < n_levels; ++k)
    if (s2_levels[k] < 1) return fail(BBSI_INVALID_ARGUMENT, "DomainPlan: s2 must be >= 1");
  if (n_threads < 1 || terminal_threads < 1)
    return fail(BBSI_INVALID_ARGUMENT, "DomainPlan: thread counts must be >= 1");
  if (int rc = validate_layout(l, w, bs, sizes)) return rc;
  if (w != 1) return fail(BBSI_INVALID_ARGUMENT, "ddrgf: requires bandwidth 1");
  for (int a = 0; a < l; ++a)
    if ((sizes ? sizes[a] : bs) != (sizes ? sizes[0] : bs))
      return fail(BBSI_INVALID_ARGUMENT, "ddrgf: requires uniform block sizes");
  if (l < 1 + s2_levels[0]) return fail(BBSI_INVALID_ARGUMENT, "interleave_permutation: too few layers to split");
  long long lk = l;
  for (int k = 0; k < n_levels; ++k) {
    if (lk < 1 + s2_levels[k])
      return fail(BBSI_INVALID_ARGUMENT, "ddrgf: plan exhausts layers at level " + std::to_string(k));
    lk = (lk + s2_levels[k]) / (1 + s2_levels[k]);
  }
  return BBSI_OK;
}

// Runs the stabilised DDRGF on device buffers; fills *fail_layer on a singular pivot.
static int ddrgf_on_device(const double2* dA, double2* dG, int l, int bp, const std::vector<int>& n_true, int s2,
                           int* fail_layer, cudaStream_t s, const int* levels_above = nullptr, int n_above = 0) {
  const size_t sb = ddrgf_scratch_bytes(l, bp, s2);
  void* scr = arena_get(9, sb);
  if (!scr) return fail(BBSI_OUT_OF_MEMORY, "ddrgf workspace allocation failed");
  int fl = -1;
  CK(ddrgf_device(dA, dG, l, bp, n_true.data(), s2, ddrgf_gamma0(), scr, sb, &fl, s, levels_above, n_above));
  CK(cudaStreamSynchronize(s));
  if (fl >= 0) {
    if (fail_layer) *fail_layer = fl;
    return fail(BBSI_SINGULAR, "singular pivot at layer " + std::to_string(fl));
  }
  return BBSI_OK;
}

int bbsi_cuda_ddrgf_z(int l, int w, int bs, const int* sizes, const double* A, const int* s2_levels, int n_levels,
                      int n_threads, int terminal_threads, double* G, long long* counters, int* fail_layer) {
  if (fail_layer) *fail_layer = -1;
  if (int rc = validate_ddrgf(l, w, bs, sizes, s2_levels, n_levels, n_threads, terminal_threads)) return rc;
  if (int rc = device_ok()) return rc;
  HostBand h = make_host(l, w, bs, sizes, A);
  const int bp = pad64(h.bs);
  bool direct = bp == h.bs;  // uniform blocks filling their slots: copy the caller's buffers as they are
  for (int a = 0; direct && a < l; ++a) direct = h.sz[a] == bs;
  std::vector<double2> staging;
  if (!direct) pad_band(h, bp, staging);
  const size_t bytes = size_t(l) * 3 * bp * bp * sizeof(double2);
  double2* dA = static_cast<double2*>(arena_get(0, bytes));
  double2* dG = static_cast<double2*>(arena_get(10, bytes));
  if (!dA || !dG) return fail(BBSI_OUT_OF_MEMORY, "band allocation failed");
  cudaStream_t s = thread_stream(0);
  CK(cudaMemcpyAsync(dA, direct ? static_cast<const void*>(A) : staging.data(), bytes, cudaMemcpyHostToDevice, s));
  if (direct) {  // out-of-band slots are ignored on input
    CK(cudaMemsetAsync(dA, 0, size_t(bp) * bp * sizeof(double2), s));
    CK(cudaMemsetAsync(dA + (size_t(l - 1) * 3 + 2) * bp * bp, 0, size_t(bp) * bp * sizeof(double2), s));
  }
  // s2_levels[1..]: the nested interface solve (csrc/ddrgf_iface.cu)
  if (int rc = ddrgf_on_device(dA, dG, l, bp, h.sz, s2_levels[0], fail_layer, s, s2_levels + 1, n_levels - 1))
    return rc;
  if (direct) {
    CK(cudaMemcpyAsync(G, dG, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::memset(G, 0, size_t(bp) * bp * sizeof(double2));  // out-of-band slots zero-filled on output
    std::memset(G + 2 * (size_t(l - 1) * 3 + 2) * bp * bp, 0, size_t(bp) * bp * sizeof(double2));
  } else {
    CK(cudaMemcpyAsync(staging.data(), dG, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    unpad_band(staging, bp, h, reinterpret_cast<double2*>(G));
  }
  if (counters) ddrgf_reference_counters(l, s2_levels, n_levels, counters);
  return BBSI_OK;
}

int bbsi_cuda_ddrgf_dev(int l, int bs, int s2, const double* dA, double* dG, int* fail_layer, void* stream) {
  if (fail_layer) *fail_layer = -1;
  int one = s2;
  if (int rc = validate_ddrgf(l, 1, bs, nullptr, &one, 1, 1, 1)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (int rc = device_ok()) return rc;
  std::vector<int> nt(l, bs);
  return ddrgf_on_device(reinterpret_cast<const double2*>(dA), reinterpret_cast<double2*>(dG), l, bs, nt, s2,
                         fail_layer, static_cast<cudaStream_t>(stream));
}

int bbsi_cuda_ddrgf_plan_dev(int l, int bs, const int* s2_levels, int n_levels, const double* dA, double* dG,
                             int* fail_layer, void* stream) {
  if (fail_layer) *fail_layer = -1;
  if (int rc = validate_ddrgf(l, 1, bs, nullptr, s2_levels, n_levels, 1, 1)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (int rc = device_ok()) return rc;
  std::vector<int> nt(l, bs);
  return ddrgf_on_device(reinterpret_cast<const double2*>(dA), reinterpret_cast<double2*>(dG), l, bs, nt, s2_levels[0],
                         fail_layer, static_cast<cudaStream_t>(stream), s2_levels + 1, n_levels - 1);
}

int bbsi_cuda_dyson_ddrgf_dev(int l, int bs, const double* dH, const double* z, const double* sigma, int s2,
                              double* dG, int* fail_layer, void* stream) {
  if (fail_layer) *fail_layer = -1;
  int one = s2;
  if (int rc = validate_ddrgf(l, 1, bs, nullptr, &one, 1, 1, 1)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (int rc = device_ok()) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t band_b = sizeof(double2) * size_t(l) * 3 * bs * bs;
  double2* dA = static_cast<double2*>(arena_get(0, band_b));
  double2* dzs = static_cast<double2*>(arena_get(2, sizeof(double2) * (size_t(1) + l)));
  if (!dA || !dzs) return fail(BBSI_OUT_OF_MEMORY, "ddrgf band allocation failed");
  CK(cudaMemcpyAsync(dzs, z, sizeof(double2), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dzs + 1, sigma, sizeof(double2) * l, cudaMemcpyHostToDevice, s));
  CK(dyson_form_band(dA, reinterpret_cast<const double2*>(dH), l, 1, bs, 1, dzs, dzs + 1, s));
  std::vector<int> nt(l, bs);
  return ddrgf_on_device(dA, reinterpret_cast<double2*>(dG), l, bs, nt, s2, fail_layer, s);
}

int bbsi_cuda_ddrgf_num_tasks(int l, int s2) { return (l >= 1 + s2 && s2 >= 1) ? ddrgf_num_tasks(l, s2) : -1; }

long long bbsi_cuda_ddrgf_packet_bytes(int ntask, int bs) { return (long long)ddrgf_packet_bytes(ntask, bs); }
long long bbsi_cuda_ddrgf_phase2_bytes(int ntask, int bs) { return (long long)ddrgf_phase2_out_bytes(ntask, bs); }

static int phase_rc(cudaError_t e, int fl, int* fail_layer, const char* what) {
  if (e != cudaSuccess) return cuda_fail(e, what);
  if (fl >= 0) {
    if (fail_layer) *fail_layer = fl;
    return fail(BBSI_SINGULAR, std::string(what) + ": singular pivot at layer " + std::to_string(fl));
  }
  return BBSI_OK;
}

int bbsi_cuda_ddrgf_phase1_dev(int l, int bs, int s2, int t0, int t1, const double* dA, double* dG, double* dPacket,
                               int* fail_layer, void* stream) {
  if (fail_layer) *fail_layer = -1;
  int one = s2;
  if (int rc = validate_ddrgf(l, 1, bs, nullptr, &one, 1, 1, 1)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (t0 < 0 || t1 > ddrgf_num_tasks(l, s2) || t0 >= t1) return fail(BBSI_INVALID_ARGUMENT, "bad task range");
  if (int rc = device_ok()) return rc;
  int fl = -1;
  cudaError_t e = ddrgf_phase1(reinterpret_cast<const double2*>(dA), reinterpret_cast<double2*>(dG), l, bs, nullptr,
                               s2, ddrgf_gamma0(), t0, t1, reinterpret_cast<double2*>(dPacket), &fl,
                               static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  return phase_rc(e, fl, fail_layer, "ddrgf phase 1");
}

int bbsi_cuda_ddrgf_phase2_dev(int l, int bs, int s2, const double* dPackets, double* dOut, int* fail_layer,
                               void* stream) {
  if (fail_layer) *fail_layer = -1;
  int one = s2;
  if (int rc = validate_ddrgf(l, 1, bs, nullptr, &one, 1, 1, 1)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (int rc = device_ok()) return rc;
  int fl = -1;
  cudaError_t e = ddrgf_phase2(reinterpret_cast<const double2*>(dPackets), l, bs, nullptr, s2, ddrgf_gamma0(),
                               reinterpret_cast<double2*>(dOut), &fl, static_cast<cudaStream_t>(stream));
  return phase_rc(e, fl, fail_layer, "ddrgf phase 2");
}

int bbsi_cuda_ddrgf_phase3_dev(int l, int bs, int s2, int t0, int t1, const double* dA, double* dG, const double* dOut,
                               int* fail_layer, void* stream) {
  if (fail_layer) *fail_layer = -1;
  int one = s2;
  if (int rc = validate_ddrgf(l, 1, bs, nullptr, &one, 1, 1, 1)) return rc;
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (t0 < 0 || t1 > ddrgf_num_tasks(l, s2) || t0 >= t1) return fail(BBSI_INVALID_ARGUMENT, "bad task range");
  if (int rc = device_ok()) return rc;
  int fl = -1;
  cudaError_t e = ddrgf_phase3(reinterpret_cast<const double2*>(dA), reinterpret_cast<double2*>(dG), l, bs, nullptr, s2,
                               t0, t1, reinterpret_cast<const double2*>(dOut), &fl, static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  return phase_rc(e, fl, fail_layer, "ddrgf phase 3");
}

int bbsi_cuda_ddrgf_halo_dev(int l, int bs, int s2, int t0, int t1, const double* dG, double* dHalo, void* stream) {
  if (t0 < 0 || s2 < 1 || l < 1 + s2 || t1 > ddrgf_num_tasks(l, s2) || t0 >= t1)
    return fail(BBSI_INVALID_ARGUMENT, "bad task range");
  CK(ddrgf_halo(reinterpret_cast<const double2*>(dG), l, bs, s2, t0, t1, reinterpret_cast<double2*>(dHalo),
                static_cast<cudaStream_t>(stream)));
  return BBSI_OK;
}

int bbsi_cuda_ddrgf_couplings_dev(int l, int bs, int s2, int t0, int t1, const double* dA, double* dG,
                                  const double* dOut, const double* dPrevSepG, const double* dNextX0G, void* stream) {
  if (t0 < 0 || s2 < 1 || l < 1 + s2 || t1 > ddrgf_num_tasks(l, s2) || t0 >= t1)
    return fail(BBSI_INVALID_ARGUMENT, "bad task range");
  if ((t0 > 0 && !dPrevSepG) || (t1 < ddrgf_num_tasks(l, s2) && !dNextX0G))
    return fail(BBSI_INVALID_ARGUMENT, "ddrgf couplings: a neighbour's halo block is required");
  CK(ddrgf_couplings(reinterpret_cast<const double2*>(dA), reinterpret_cast<double2*>(dG), l, bs, s2, t0, t1,
                     reinterpret_cast<const double2*>(dOut), reinterpret_cast<const double2*>(dPrevSepG),
                     reinterpret_cast<const double2*>(dNextX0G), static_cast<cudaStream_t>(stream)));
  return BBSI_OK;
}

void bbsi_ddrgf_reference_counters(long long l, const int* s2_levels, int n_levels, long long* out) {
  ddrgf_reference_counters(l, s2_levels, n_levels, out);
}

}  // extern "C"

// ------------------------------------------------------------------ multi-GPU (NCCL)
// One process per GPU (torchrun / MPI style): the caller shares a NCCL unique id and
// creates one communicator per rank; bbsi_cuda_ddrgf_rank_dev then runs the rank's part
// of the domain-sharded DDRGF with the packet all-gather and the halo exchange inside
// the library. One process driving several GPUs: bbsi_cuda_ddrgf_multi_z /
// bbsi_cuda_dyson_rgf_multi_z (ncclCommInitAll, one host thread per GPU).
int bbsi_cuda_nccl_available(void) {
  std::string err;
  if (nccl_ready(&err)) return 1;
  fail(BBSI_CUDA_ERROR, err);
  return 0;
}

int bbsi_cuda_nccl_unique_id(void* out128) {
  std::string err;
  if (nccl_unique_id(out128, &err)) return fail(BBSI_CUDA_ERROR, err);
  return BBSI_OK;
}

int bbsi_cuda_nccl_comm_init(const void* id128, int nranks, int rank, void** comm) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !comm) return fail(BBSI_INVALID_ARGUMENT, "bad NCCL rank / size");
  if (int rc = device_ok()) return rc;
  std::string err;
  if (nccl_comm_init_rank(id128, nranks, rank, comm, &err)) return fail(BBSI_CUDA_ERROR, err);
  return BBSI_OK;
}

void bbsi_cuda_nccl_comm_destroy(void* comm) { nccl_comm_destroy(comm); }

int bbsi_cuda_ddrgf_rank_layers(int l, int s2, int nranks, int rank, int* t0, int* t1, int* L0, int* L1) {
  if (s2 < 1 || l < 1 + s2) return fail(BBSI_INVALID_ARGUMENT, "interleave_permutation: too few layers to split");
  const int T = ddrgf_num_tasks(l, s2);
  if (nranks < 1 || nranks > T || rank < 0 || rank >= nranks)
    return fail(BBSI_INVALID_ARGUMENT, "ddrgf: " + std::to_string(nranks) + " ranks for " + std::to_string(T) +
                                           " domains");
  const auto r = ddrgf_rank_ranges(T, nranks)[rank];
  // tasks t = [t*(s2+1), ...): first(t) = t*(s2+1); sep(t) = min(first + s2, l - 1)
  auto first = [&](int t) { return t * (s2 + 1); };
  auto sep = [&](int t) { return std::min(first(t) + s2, l - 1); };
  if (t0) *t0 = r.first;
  if (t1) *t1 = r.second;
  if (L0) *L0 = first(r.first);
  if (L1) *L1 = sep(r.second - 1) + 1;
  return BBSI_OK;
}

int bbsi_cuda_ddrgf_rank_dev(void* comm, int l, int bs, int s2, const double* dA_loc, double* dG_loc, int* fail_layer,
                             void* stream) {
  return bbsi_cuda_ddrgf_rank_plan_dev(comm, l, bs, &s2, 1, dA_loc, dG_loc, fail_layer, stream);
}

int bbsi_cuda_ddrgf_rank_plan_dev(void* comm, int l, int bs, const int* s2_levels, int n_levels, const double* dA_loc,
                                  double* dG_loc, int* fail_layer, void* stream) {
  if (fail_layer) *fail_layer = -1;
  if (int rc = validate_ddrgf(l, 1, bs, nullptr, s2_levels, n_levels, 1, 1)) return rc;
  const int s2 = s2_levels[0];
  if (bs % 64) return fail(BBSI_INVALID_ARGUMENT, "resident API requires bs % 64 == 0");
  if (int rc = device_ok()) return rc;
  std::string err;
  int nr = 1, rk = 0;
  if (nccl_comm_shape(comm, &nr, &rk, &err)) return fail(BBSI_CUDA_ERROR, err);
  int t0 = 0, t1 = 0;
  if (int rc = bbsi_cuda_ddrgf_rank_layers(l, s2, nr, rk, &t0, &t1, nullptr, nullptr)) return rc;
  const size_t sb = ddrgf_scratch_bytes(l, bs, s2);
  void* scr = arena_get(9, sb);
  if (!scr) return fail(BBSI_OUT_OF_MEMORY, "ddrgf workspace allocation failed");
  DdrgfExchange x = nccl_ddrgf_exchange(comm, l, bs, s2, &err);
  int fl = -1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = ddrgf_rank(reinterpret_cast<const double2*>(dA_loc), reinterpret_cast<double2*>(dG_loc), l, bs,
                             nullptr, s2, t0, t1, ddrgf_gamma0(), x, scr, sb, &fl, s, s2_levels + 1, n_levels - 1);
  if (e != cudaSuccess) return err.empty() ? cuda_fail(e, "ddrgf rank") : fail(BBSI_CUDA_ERROR, err);
  CK(cudaStreamSynchronize(s));
  if (fl >= 0) {
    if (fail_layer) *fail_layer = fl;
    return fail(BBSI_SINGULAR, "singular pivot at layer " + std::to_string(fl));
  }
  return BBSI_OK;
}

// Runs f(rank, device) on one host thread per GPU; each thread releases its workspaces
// before it exits. Returns the first non-zero code (by rank) and its message.
template <class F>
static int on_gpus(int ngpu, const int* devices, F&& f) {
  std::vector<int> rc(ngpu, BBSI_OK);
  std::vector<std::string> msg(ngpu);
  std::vector<std::thread> th;
  for (int r = 0; r < ngpu; ++r)
    th.emplace_back([&, r] {
      const int dev = devices ? devices[r] : r;
      if (cudaSetDevice(dev) != cudaSuccess) {
        cudaGetLastError();
        rc[r] = BBSI_CUDA_ERROR;
        msg[r] = "cudaSetDevice(" + std::to_string(dev) + ") failed";
        return;
      }
      rc[r] = f(r, dev);
      if (rc[r]) msg[r] = g_err;
      thread_resources_release();
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < ngpu; ++r)
    if (rc[r]) return fail(rc[r], "rank " + std::to_string(r) + ": " + msg[r]);
  return BBSI_OK;
}

static int check_devices(int ngpu, const int* devices) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (ngpu < 1) return fail(BBSI_INVALID_ARGUMENT, "ngpu must be >= 1");
  for (int r = 0; r < ngpu; ++r) {
    const int d = devices ? devices[r] : r;
    if (d < 0 || d >= n) return fail(BBSI_INVALID_ARGUMENT, "device " + std::to_string(d) + " not visible");
  }
  return BBSI_OK;
}

int bbsi_cuda_ddrgf_multi_z(int l, int w, int bs, const int* sizes, const double* A, const int* s2_levels,
                            int n_levels, int n_threads, int terminal_threads, int ngpu, const int* devices, double* G,
                            long long* counters, int* fail_layer) {
  if (fail_layer) *fail_layer = -1;
  if (int rc = validate_ddrgf(l, w, bs, sizes, s2_levels, n_levels, n_threads, terminal_threads)) return rc;
  if (int rc = device_ok()) return rc;
  if (int rc = check_devices(ngpu, devices)) return rc;
  const int s2 = s2_levels[0];
  if (ngpu > ddrgf_num_tasks(l, s2))
    return fail(BBSI_INVALID_ARGUMENT, "ddrgf: more GPUs than domains in the plan");
  HostBand h = make_host(l, w, bs, sizes, A);
  const int bp = pad64(h.bs);
  std::vector<double2> staging;
  pad_band(h, bp, staging);
  const long long row = 3LL * bp * bp;  // complex entries per band row
  std::vector<void*> comms(ngpu, nullptr);
  std::vector<int> devs(ngpu);
  for (int r = 0; r < ngpu; ++r) devs[r] = devices ? devices[r] : r;
  std::string err;
  if (ngpu > 1 && nccl_comm_init_all(ngpu, devs.data(), comms, &err)) return fail(BBSI_CUDA_ERROR, err);
  std::vector<int> fl(ngpu, -1);
  int rc = on_gpus(ngpu, devs.data(), [&](int r, int) -> int {
    int t0 = 0, t1 = 0, L0 = 0, L1 = 0;
    if (int q = bbsi_cuda_ddrgf_rank_layers(l, s2, ngpu, r, &t0, &t1, &L0, &L1)) return q;
    const size_t bytes = size_t(L1 - L0) * row * sizeof(double2);
    double2* dA = static_cast<double2*>(arena_get(0, bytes));
    double2* dG = static_cast<double2*>(arena_get(10, bytes));
    if (!dA || !dG) return fail(BBSI_OUT_OF_MEMORY, "band allocation failed");
    cudaStream_t s = thread_stream(0);
    CK(cudaMemcpyAsync(dA, staging.data() + size_t(L0) * row, bytes, cudaMemcpyHostToDevice, s));
    const size_t sb = ddrgf_scratch_bytes(l, bp, s2);
    void* scr = arena_get(9, sb);
    if (!scr) return fail(BBSI_OUT_OF_MEMORY, "ddrgf workspace allocation failed");
    std::string xerr;
    DdrgfExchange x;
    if (ngpu > 1) {
      x = nccl_ddrgf_exchange(comms[r], l, bp, s2, &xerr);
    } else {
      x.packets = [](double2*, int, int, int f, int* any, cudaStream_t) {
        *any = f;
        return cudaSuccess;
      };
      x.halo = [](const double2*, double2*, int f, int* any, cudaStream_t) {
        *any = f;
        return cudaSuccess;
      };
    }
    cudaError_t e = ddrgf_rank(dA, dG, l, bp, h.sz.data(), s2, t0, t1, ddrgf_gamma0(), x, scr, sb, &fl[r], s,
                               s2_levels + 1, n_levels - 1);
    if (e != cudaSuccess) return xerr.empty() ? cuda_fail(e, "ddrgf rank") : fail(BBSI_CUDA_ERROR, xerr);
    if (fl[r] >= 0) return BBSI_OK;
    // rows [L0, L1) of G: this rank's chains (written once, disjoint across ranks)
    CK(cudaMemcpyAsync(staging.data() + size_t(L0) * row, dG, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return BBSI_OK;
  });
  for (void* c : comms) nccl_comm_destroy(c);
  if (rc) return rc;
  for (int r = 0; r < ngpu; ++r)
    if (fl[r] >= 0) {
      if (fail_layer) *fail_layer = fl[r];
      return fail(BBSI_SINGULAR, "singular pivot at layer " + std::to_string(fl[r]));
    }
  unpad_band(staging, bp, h, reinterpret_cast<double2*>(G));
  if (counters) ddrgf_reference_counters(l, s2_levels, n_levels, counters);
  return BBSI_OK;
}

int bbsi_cuda_dyson_rgf_multi_z(int l, int w, int bs, int n_energy, const double* H, const double* z,
                                const double* sigma, double* G, int* fail_layers, int chunk, int ngpu,
                                const int* devices) {
  if (int rc = device_ok()) return rc;
  if (int rc = check_devices(ngpu, devices)) return rc;
  if (n_energy < ngpu) return fail(BBSI_INVALID_ARGUMENT, "fewer energies than GPUs");
  const size_t band = size_t(l) * (2 * w + 1) * bs * bs;
  std::vector<int> devs(ngpu);
  for (int r = 0; r < ngpu; ++r) devs[r] = devices ? devices[r] : r;
  // contiguous energy shards, no collective
  return on_gpus(ngpu, devs.data(), [&](int r, int) -> int {
    const int e0 = int((long long)r * n_energy / ngpu), e1 = int((long long)(r + 1) * n_energy / ngpu);
    return bbsi_cuda_dyson_rgf_z(l, w, bs, e1 - e0, H, z + 2 * e0, sigma, G + 2 * size_t(e0) * band,
                                 fail_layers ? fail_layers + e0 : nullptr, chunk);
  });
}

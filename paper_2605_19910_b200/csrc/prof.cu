// Launch accounting and optional per-launch CUDA-event timing of the library's own
// kernels (used by bench.py for the roofline of the dominant kernel), plus the
// FP64 DMMA peak probe that gives the roofline its denominator.
#include <atomic>
#include <map>
#include <mutex>
#include <vector>

#include "internal.h"

namespace bbsi_gpu {

namespace {
std::atomic<long long> g_launches{0};
std::mutex g_mu;
bool g_on = false;
struct Rec {
  cudaEvent_t a, b;
  int cat;
  double flops, bytes;
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t ev() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

ProfScope::ProfScope(cudaStream_t s, int cat, double flops, double bytes) : s_(s), a_(nullptr) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  a_ = ev();
  b_ = ev();
  cat_ = cat;
  flops_ = flops;
  bytes_ = bytes;
  cudaEventRecord(static_cast<cudaEvent_t>(a_), s);
}

ProfScope::~ProfScope() {
  if (!a_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(static_cast<cudaEvent_t>(b_), s_);
  g_recs.push_back(Rec{static_cast<cudaEvent_t>(a_), static_cast<cudaEvent_t>(b_), cat_, flops_, bytes_});
}

long long launch_count() { return g_launches.load(); }
void launch_count_add(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
bool prof_enabled() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_on;
}

void prof_enable(bool on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on;
}

// out[cat*4 + {0,1,2,3}] = launches, total ms, flops, bytes
int prof_collect(double* out, int ncat) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (int i = 0; i < ncat * 4; ++i) out[i] = 0.0;
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (r.cat < ncat) {
      out[r.cat * 4 + 0] += 1;
      out[r.cat * 4 + 1] += ms;
      out[r.cat * 4 + 2] += r.flops;
      out[r.cat * 4 + 3] += r.bytes;
    }
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  return 0;
}

// ------------------------------------------------------------------ FP64 peak probe
namespace {
__global__ void __launch_bounds__(128) dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
}  // namespace

// Runs the DMMA loop on every SM for ~duration_ms; returns achieved TFLOP/s
// (burst, best of reps) or a negative value on error.
double fp64_dmma_peak(double duration_ms, int reps) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = nsm * 2;
  int iters = 1000;
  dmma_peak_kernel<<<grid, 128>>>(d, 100);
  float ms = 0.f;
  cudaEventRecord(e0);
  dmma_peak_kernel<<<grid, 128>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  if (ms > 0) iters = int(iters * duration_ms / ms) + 1;
  double best = 0.0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    dmma_peak_kernel<<<grid, 128>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8 * (128 / 32) * double(grid) * iters;
    double tf = fl / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

// Kernel attributes are per device: remembered per (device, kernel) so a process that
// drives several GPUs sets them on each one (and concurrent callers do not race).
cudaError_t set_max_dyn_smem(const void* fn, size_t bytes, bool max_carveout) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{dev, fn}];
  if (have >= bytes && have > 0) return cudaSuccess;
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)))) return e;
  if (max_carveout &&
      (e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared)))
    return e;
  have = bytes;
  return cudaSuccess;
}

}  // namespace bbsi_gpu

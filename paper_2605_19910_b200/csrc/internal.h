// Internal declarations shared by the CUDA translation units of libbbsi_cuda.so.
#pragma once
#include <cuda_runtime.h>

#include <functional>
#include <initializer_list>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "zcommon.cuh"

namespace bbsi_gpu {

// kernels
cudaError_t zgemm_grouped(ZGemmGroup& g, cudaStream_t stream);
// TMA-staged sweep GEMM (zgemm_tma.cu): used by zgemm_grouped when every operand A / B is
// a view of a registered buffer; *done = false -> not applicable.
cudaError_t zgemm_tma_try(const ZGemmGroup& g, cudaStream_t stream, bool* done);
// Registers [base, base + bytes) of bs x bs slots for TMA operands (per host thread,
// scoped: tma_unregister(n) drops the n most recent registrations; env BBSI_TMA=0 off).
void tma_register(const void* base, size_t bytes, int bs);
void tma_unregister(int n);
struct TmaScope {
  int n = 0;
  void add(const void* base, size_t bytes, int bs) {
    if (base && bytes) {
      tma_register(base, bytes, bs);
      ++n;
    }
  }
  ~TmaScope() { tma_unregister(n); }
};
// In-place batched inverse (blocked Gauss-Jordan, partial pivoting); scratch of
// zinv_scratch_bytes(n, batch) bytes; status[b] = -1 or the first negligible pivot.
cudaError_t zinv_batched(double2* M, long long ld, long long bstride, int n, int n_true, int batch, void* scratch,
                         int* status, cudaStream_t stream);
// Same over `outer` x `inner` matrices: matrix (o, i) at M + i*bstride + o*ostride,
// status at status[i + o*sostride] (outer <= kMaxProblems; scratch for inner*outer).
cudaError_t zinv_batched2(double2* M, long long ld, long long bstride, int n, int n_true, int inner, int outer,
                          long long ostride, void* scratch, int* status, long long sostride, cudaStream_t stream);
size_t zinv_scratch_bytes(int n, int batch);
// How many inversion batches of this host thread run concurrently (stream groups of a
// sweep); the pair panel picks its CTAs per matrix from batch x concurrency.
void zinv_set_concurrency(int groups);
cudaError_t dyson_fill_h(double2* H, int l, int w, int b, uint64_t seed, cudaStream_t s);
// Rows [a0, a1) of the same band into H ([a1-a0][2w+1][b][b], local row 0 = layer a0).
cudaError_t dyson_fill_h_rows(double2* H, int l, int w, int b, uint64_t seed, int a0, int a1, cudaStream_t s);
// Diagonal blocks only (A_aa = z I - H_aa - sigma_a I) plus zeroed out-of-range slots,
// for sweeps that read the off-diagonal blocks from H (SweepWork::Hoff).
cudaError_t dyson_form_diag(double2* G, const double2* H, int l, int w, int bs, int batch, const double2* z,
                            const double2* sigma, cudaStream_t s);
// Copies the w x w block window of band rows [a0, a0 + w) between the band slots and a
// dense (w b) x (w b) column-major matrix per batch entry (to_dense: band -> dense).
cudaError_t band_window(double2* G, long long gstride, double2* D, int a0, int w, int b, int batch, bool to_dense,
                        cudaStream_t s);
// Same for the last layer only (and layer 0 when `first`): the sweeps' first pivots.
// The other diagonal blocks are read from H by the GEMM that first updates them
// (ZGemmProblem::cz, SweepWork::zdev).
cudaError_t dyson_form_diag_ends(double2* G, const double2* H, int l, int w, int bs, int batch, const double2* z,
                                 const double2* sigma, bool first, cudaStream_t s);
// M_b += I (n x n, ld n, batch stride) and y += x (n complex entries).
cudaError_t diag_shift_batched(double2* M, int n, long long stride, int batch, cudaStream_t s);
cudaError_t axpy_batched(double2* y, const double2* x, long long n, cudaStream_t s);
cudaError_t axpy_strided(double2* y, long long ys, const double2* x, long long xs, long long n, int nb, double2 a,
                         cudaStream_t s);
cudaError_t dyson_form_band(double2* G, const double2* H, int l, int w, int bs, int batch, const double2* z,
                            const double2* sigma, cudaStream_t s);

// Error codes of the C ABI (include/bbsi_cuda.h).
enum Status { OK = 0, INVALID = 1, SINGULAR = 2, CUDA_ERR = 3, NOMEM = 4 };

struct Error {
  int code;
  std::string what;
};

// Device workspace of one batched n-diagonal sweep (all pointers device memory).
struct SweepWork {
  int l = 0, w = 0, bs = 0, batch = 0;
  double2* G = nullptr;   // [batch][l][2w+1][bs*bs]: working copy of A, then G^R
  long long g_bstride = 0;
  double2* LM = nullptr;  // [batch][l][w][bs*bs]: lm[j][t-1] = X_j M'[j, j-t]
  double2* UM = nullptr;  // [batch][l][w][bs*bs]: um[j][t-1] = M'[j-t, j] X_j
  void* inv = nullptr;    // zinv scratch for `batch` matrices
  int groups = 1;         // independent batch groups swept concurrently on side streams
  int* status = nullptr;  // [l][status_stride] (entry b of layer j at status[j*stride + b])
  int status_stride = 0;  // 0: batch
  // Optional: called (while enqueueing) once band rows [r0, r1) of batch entries
  // [e0, e0 + ne) are final on stream s -- every `hook_rows` rows of the downward
  // sweep and at its end. Used to stream results to the host during the sweep.
  std::function<cudaError_t(int r0, int r1, int e0, int ne, cudaStream_t s)> rows_done;
  int hook_rows = 8;
  int e_off = 0;          // batch offset of this (group's) sub-batch, for rows_done
  // Optional (w == 1 only): energy-independent band H with A's off-diagonal blocks
  // = -H (Dyson batches). The sweeps then read those operands from H, shared by the
  // whole batch, and G's off-diagonal slots need not hold A (see dyson_form_diag).
  const double2* Hoff = nullptr;
  // w == 1 only: two-ended sweep (left- and right-connected Schur chains run
  // concurrently, meet at layer l/2, then two outward sweeps). Same output; twice the
  // batch per latency-bound inversion launch and half the sequential steps. Set
  // before sweep_carve (the inversion scratch doubles).
  bool two_ended = false;
  int lm_layers = 0;      // layers per batch entry of LM / UM (0: l; a sub-band view keeps the parent's)
  void* mid = nullptr;    // two-ended, w >= 2: dense (w b)^2 middle window + its inversion scratch (per group)
  // Optional (with Hoff): per-batch z (device, this (group's) batch entries) and per-layer
  // sigma (device): the diagonal blocks of A are not in G until the Schur update that first
  // touches them reads A = z I - H - sigma I from H (only the chains' first layers are formed)
  const double2* zdev = nullptr;
  const double2* sigdev = nullptr;
  // one-ended sweeps, w >= 2 (refine_multipliers_default): copies of the pivots f_j
  // ([batch][bs*bs]) for one step of iterative refinement of every multiplier
  double2* fcopy = nullptr;
};
// One refinement step of the w >= 2 multipliers (lm += X (M - f lm), um += (M - um f) X):
// explicit-inverse products are not backward stable; with it the residual of the
// n-diagonal sweep matches the reference's LU solves (env BBSI_REFINE=0 turns it off).
bool refine_multipliers_default();

// Bytes of LM+UM+piv+wz+status for a sweep.
size_t sweep_scratch_bytes(int l, int w, int bs, int batch, int groups = 1, bool two_ended = false);
// Two-ended sweeps for Dyson batches (env BBSI_TWO_ENDED=0 turns them off).
bool two_ended_default();
// Whether rgf_sweeps runs the two-ended variant for this workspace (two_ended set and
// the layer count allows it); its multipliers then hold the right chain for layers
// > m and the left chain (lm = Y A[j, j+1], um = A[j+1, j] Y) for layers < m = l/2 (w = 1).
bool sweep_is_two_ended(const SweepWork& W);
// Stream groups of a Dyson energy batch (env BBSI_GROUPS overrides).
int dyson_groups(int batch);
// Default number of concurrent batch groups (env BBSI_GROUPS overrides).
int default_groups(int batch, int bs);
// Carves the scratch part of a SweepWork out of `base` (>= sweep_scratch_bytes).
void sweep_carve(SweepWork& W, void* base);

// Upward + downward sweeps of rgf_ndiag (rgf.hpp:82-137; w=1 is rgf_tridiag,
// rgf.hpp:37-76) on a batch of working bands already holding A.
// n_true[a] = unpadded size of layer a (for the singular-pivot threshold).
cudaError_t rgf_sweeps(const SweepWork& W, const int* n_true, cudaStream_t s);

// Reads back W.status and returns, per batch entry, the failing layer the
// reference would report (first failure in elimination order) or -1.
cudaError_t collect_failures(const SweepWork& W, std::vector<int>& fail, cudaStream_t s);

// Small b x b helpers (ddrgf.cu): plain block operand (ld = b) and
// D = alpha*A*B + beta*C over `batch` products (C may alias D).
ZOp zblk(const double2* p, int b, long long bstride = 0);
cudaError_t zmm(int b, int batch, double2 alpha, ZOp A, ZOp B, double beta, ZOp C, cudaStream_t s);

// Stabilised DDRGF (ddrgf.cu) on one device band A (w = 1, uniform bs) -> G.
// gamma0: fake-lead strength relative to max|A[s,s]| of each task (BBSI_DDRGF_GAMMA).
// levels_above / n_above: the plan's s2_levels[1..] (nested interface solve, ddrgf_iface.cu)
cudaError_t ddrgf_device(const double2* A, double2* G, int l, int b, const int* n_true, int s2, double gamma0,
                         void* scratch, size_t scratch_bytes, int* fail_layer, cudaStream_t s,
                         const int* levels_above = nullptr, int n_above = 0);
size_t ddrgf_scratch_bytes(int l, int b, int s2);
double ddrgf_gamma0();
// Phases of the same algorithm on a rank-local slice (tasks [t0, t1)); only the
// per-task interface packets (and two halo blocks per rank) cross ranks (csrc/ddrgf.cu).
int ddrgf_num_tasks(int l, int s2);
size_t ddrgf_packet_bytes(int ntask, int b);
size_t ddrgf_phase2_out_bytes(int ntask, int b);
cudaError_t ddrgf_phase1(const double2* A, double2* G, int l, int b, const int* n_true, int s2, double gamma0, int t0,
                         int t1, double2* packet, int* fail_layer, cudaStream_t s);
cudaError_t ddrgf_phase2(const double2* packets, int l, int b, const int* n_true, int s2, double gamma0, double2* out,
                         int* fail_layer, cudaStream_t s, const int* levels_above = nullptr, int n_above = 0);
// The interface solve behind phase 2 (ddrgf_iface.cu).
cudaError_t iface_solve(const double2* packets, double2* out, int T, int b, int n_true, const std::vector<double>& gam,
                        const std::vector<char>& empty, const std::vector<int>& first, const std::vector<int>& last,
                        const std::vector<int>& sep, const int* levels, int nl, int* st, int st_cap,
                        std::vector<int>& st_layer, cudaStream_t s, cudaStream_t side, cudaEvent_t fork,
                        cudaEvent_t join);
int iface_status_cap(int T);
cudaError_t ddrgf_phase3(const double2* A, double2* G, int l, int b, const int* n_true, int s2, int t0, int t1,
                         const double2* out, int* fail_layer, cudaStream_t s);
cudaError_t ddrgf_halo(const double2* G, int l, int b, int s2, int t0, int t1, double2* halo, cudaStream_t s);
cudaError_t ddrgf_couplings(const double2* A, double2* G, int l, int b, int s2, int t0, int t1, const double2* out,
                            const double2* prev_sep_g, const double2* next_x0_g, cudaStream_t s);
// Balanced contiguous task ranges per rank (distributed.py task_ranges).
std::vector<std::pair<int, int>> ddrgf_rank_ranges(int n_tasks, int nranks);
// The two exchanges of a domain-sharded DDRGF (ddrgf_rank):
//   packets(all, t0, t1, fail, any, s): on entry all[t0..t1) holds this rank's packets;
//     on return every task's packet (task order) and *any = the first failing layer of
//     any rank (or -1);
//   halo(own, nbr, fail, any, s): own = this rank's [2] boundary blocks; nbr[0] = the
//     previous rank's own[1], nbr[1] = the next rank's own[0]; *any as above.
struct DdrgfExchange {
  std::function<cudaError_t(double2*, int, int, int, int*, cudaStream_t)> packets;
  std::function<cudaError_t(const double2*, double2*, int, int*, cudaStream_t)> halo;
};
cudaError_t ddrgf_rank(const double2* A_loc, double2* G_loc, int l, int b, const int* n_true, int s2, int t0, int t1,
                       double gamma0, const DdrgfExchange& x, void* scratch, size_t scratch_bytes, int* fail_layer,
                       cudaStream_t s, const int* levels_above = nullptr, int n_above = 0);
// NCCL (multi.cu, resolved with dlopen at first use).
bool nccl_ready(std::string* err);
int nccl_unique_id(void* out, std::string* err);
int nccl_comm_init_rank(const void* id, int nranks, int rank, void** comm, std::string* err);
int nccl_comm_init_all(int n, const int* devs, std::vector<void*>& comms, std::string* err);
void nccl_comm_destroy(void* comm);
int nccl_comm_shape(void* comm, int* nranks, int* rank, std::string* err);
DdrgfExchange nccl_ddrgf_exchange(void* comm, int l, int b, int s2, std::string* err);

void ddrgf_reference_counters(long long l, const int* s2_levels, int n_levels, long long out[3]);

// Launch accounting / optional event timing around one kernel launch (prof.cu).
enum ProfCat { PROF_GEMM = 0, PROF_INV = 1, PROF_BAND = 2, PROF_GJ_GEMM = 3, PROF_NCAT = 4 };
class ProfScope {
 public:
  ProfScope(cudaStream_t s, int cat, double flops, double bytes);
  ~ProfScope();

 private:
  cudaStream_t s_;
  void* a_;
  void* b_ = nullptr;
  int cat_ = 0;
  double flops_ = 0, bytes_ = 0;
};
long long launch_count();
void launch_count_add(long long n);
bool prof_enabled();
void prof_enable(bool on);
int prof_collect(double* out, int ncat);
double fp64_dmma_peak(double duration_ms, int reps);

// cudaFuncAttributeMaxDynamicSharedMemorySize >= bytes for fn on the current device
// (set once per device and kernel; optionally the max-shared carveout too).
cudaError_t set_max_dyn_smem(const void* fn, size_t bytes, bool max_carveout = false);

// Grow-only device arena per (host thread, device, slot); returns nullptr on OOM.
void* arena_get(int slot, size_t bytes);
// Bytes currently held by the given arena slots on the current device (reusable).
size_t arena_held(std::initializer_list<int> slots);
// Frees the calling thread's arenas (every device).
void arena_release_all();
// Frees everything the calling thread holds: arenas, side-stream pools, the
// per-thread streams of the C ABI (worker threads call this before they exit).
void thread_resources_release();
// Per-thread streams of the C ABI (non-blocking; created on first use per device).
cudaStream_t thread_stream(int which);

}  // namespace bbsi_gpu

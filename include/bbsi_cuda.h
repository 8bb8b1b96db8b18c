/* bbsi_cuda.h -- C ABI of the B200-native selected-inversion library
 * (libbbsi_cuda.so, built from paper_2605_19910_b200/csrc).
 *
 * This is the drop-in boundary for the reference solver entry points of
 * /root/reference/proj/core/include/bbsi (the "bbsi" C++ library). Each entry
 * point below names the reference interface it replaces. The reference's C++
 * signatures take a BlockBandedMatrix<std::complex<double>> by const& and return
 * {BlockBandedMatrix, KernelCounters} by value (rgf.hpp:37-39, 82-84;
 * ddrgf.hpp:420-422); across this ABI the matrix travels as plain caller-owned
 * buffers in the reference's own slot order (block_banded.hpp:58-60):
 *
 *   slot(a, off) = a*(2w+1) + off + w,  a = 0..l-1, off = -w..w
 *   each slot    = bs x bs complex128, column-major, (re, im) interleaved,
 *                  block (a, a+off) of size sizes[a] x sizes[a+off] in its
 *                  top-left corner with leading dimension bs.
 *   Out-of-band slots are ignored on input and zero-filled on output.
 *
 * Host-buffer entry points ("_z") copy in and out of the device inside the call
 * (the drop-in semantics); "_dev" entry points take device pointers and a
 * cudaStream_t (passed as void*) and keep everything resident.
 *
 * Return codes (the C++ shim include/bbsi_gpu.hpp rethrows the reference types):
 *   BBSI_OK 0; BBSI_INVALID_ARGUMENT 1 -> bbsi::invalid_argument_error (errors.hpp:9-12);
 *   BBSI_SINGULAR 2 -> bbsi::singular_matrix_error(layer) (errors.hpp:18-27), the failing
 *   global layer in *fail_layer; BBSI_CUDA_ERROR 3; BBSI_OUT_OF_MEMORY 4.
 * bbsi_cuda_last_error() returns the message of the last failure on this thread.
 * All arithmetic is complex FP64 on the GPU; there is no CPU fallback: without a
 * CUDA device every compute entry point returns BBSI_CUDA_ERROR.
 */
#ifndef BBSI_CUDA_H
#define BBSI_CUDA_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBSI_OK 0
#define BBSI_INVALID_ARGUMENT 1
#define BBSI_SINGULAR 2
#define BBSI_CUDA_ERROR 3
#define BBSI_OUT_OF_MEMORY 4

/* ABI version (major*100 + minor). */
int bbsi_cuda_version(void);
const char* bbsi_cuda_last_error(void);
/* Number of CUDA devices visible (0 on a CPU-only host). */
int bbsi_cuda_device_count(void);
/* Releases the library's cached device workspaces on every device. */
void bbsi_cuda_release_workspace(void);

/* ---------------------------------------------------------------- solvers (drop-in)
 * sizes: per-layer block sizes (length l) or NULL for uniform bs.
 * counters: int64[3] = {n_gemm, n_lu, n_getrs}, the reference's logical
 *   KernelCounters for this call (kernels.hpp:18-31), or NULL.
 * fail_layer: receives the failing layer on BBSI_SINGULAR (may be NULL). */

/* replaces bbsi::rgf_tridiag (rgf.hpp:37-76) */
int bbsi_cuda_rgf_tridiag_z(int l, int w, int bs, const int* sizes, const double* A, double* G,
                            long long* counters, int* fail_layer);

/* replaces bbsi::rgf_ndiag (rgf.hpp:82-137); *max_update_offset mirrors
 * StructuralTrace::max_update_offset (rgf.hpp:14-16), may be NULL. */
int bbsi_cuda_rgf_ndiag_z(int l, int w, int bs, const int* sizes, const double* A, double* G,
                          long long* counters, int* max_update_offset, int* fail_layer);

/* replaces bbsi::rgf_fused (rgf.hpp:143-192): super-blocks of w layers, tridiagonal
 * solve, restriction to the original band. */
int bbsi_cuda_rgf_fused_z(int l, int w, int bs, const int* sizes, const double* A, double* G,
                          long long* counters, int* fail_layer);

/* replaces bbsi::rgf_extended (rgf.hpp:197-270): core band plus full first/last
 * block rows and columns of the inverse, each [l][bs][bs] (entry b of first_row
 * = (M^-1)[0, b], etc.). Any halo pointer may be NULL. */
int bbsi_cuda_rgf_extended_z(int l, int w, int bs, const int* sizes, const double* A, double* G,
                             double* first_row, double* last_row, double* first_col, double* last_col,
                             long long* counters, int* fail_layer);

/* replaces bbsi::ddrgf (ddrgf.hpp:420-428) with DomainPlan{s2_levels, n_threads,
 * terminal_threads} (ddrgf.hpp:18-32). n_threads only bounds host concurrency;
 * results do not depend on it. Uses the stabilised boundary-self-energy variant
 * (DESIGN.md "DDRGF"); counters are the reference's logical counts. */
int bbsi_cuda_ddrgf_z(int l, int w, int bs, const int* sizes, const double* A, const int* s2_levels,
                      int n_levels, int n_threads, int terminal_threads, double* G, long long* counters,
                      int* fail_layer);

/* The reference's logical KernelCounters of ddrgf for a plan (ddrgf.hpp:344-412
 * walked on the host; predict_ddrgf_counters, cost_model.hpp:137-154, when the
 * plan divides evenly). out: int64[3]. */
void bbsi_ddrgf_reference_counters(long long l, const int* s2_levels, int n_levels, long long* out);

/* Many independent matrices of one layout (the host-buffer batch form of rgf_tridiag /
 * rgf_ndiag): A, G host [batch][l][2w+1][bs][bs]; solved together on the device in the
 * reference's elimination order; fail_layers[k] = -1 or matrix k's failing layer (the
 * other matrices' results are still written); counters as for one call. */
int bbsi_cuda_rgf_many_z(int l, int w, int bs, const int* sizes, int batch, const double* A, double* G,
                         long long* counters, int* fail_layers);

/* ---------------------------------------------------------------- resident batched API
 * A batch of independent band matrices (energies or domains) with uniform
 * bs % 64 == 0. dA / dG: device pointers to [batch][l][2w+1][bs][bs];
 * a_bstride: elements (complex) between consecutive A bands.
 * fail_layers: host int[batch], -1 or the failing layer per entry. */
int bbsi_cuda_rgf_batched_dev(int l, int w, int bs, int batch, const double* dA, long long a_bstride,
                              double* dG, int* fail_layers, void* stream);

/* Dyson batch: A_e = z_e I - H - Sigma (Sigma_a = sigma_a I) formed on the fly
 * from ONE shared Hamiltonian band dH ([l][2w+1][bs][bs], device), z: host
 * complex[n_energy] (E + i eta), sigma: host complex[l]. */
int bbsi_cuda_dyson_rgf_dev(int l, int w, int bs, int n_energy, const double* dH, const double* z,
                            const double* sigma, double* dG, int* fail_layers, void* stream);

/* Dyson batch with FULL lead self-energy blocks (energy dependent): A_e = z_e I - H - Sigma_e,
 * dSigma device [n_energy][2w][bs][bs]: blocks for layers 0..w-1 then l-w..l-1 (Sigma is
 * zero elsewhere). */
int bbsi_cuda_dyson_rgf_sigma_dev(int l, int w, int bs, int n_energy, const double* dH, const double* z,
                                  const double* dSigma, double* dG, int* fail_layers, void* stream);

/* Same solve end to end from HOST buffers (the drop-in form): H host [l][2w+1][bs][bs],
 * G host [n_energy][l][2w+1][bs][bs]. Energies run in chunks of `chunk` (<= 0: n/4);
 * finished chunks stream back to G while the next computes (pin G for overlap). */
int bbsi_cuda_dyson_rgf_z(int l, int w, int bs, int n_energy, const double* H, const double* z,
                          const double* sigma, double* G, int* fail_layers, int chunk);

/* Resident stabilised DDRGF of one band (w = 1): dA, dG device [l][3][bs][bs],
 * interior groups of s2 layers (single-level plan). */
int bbsi_cuda_ddrgf_dev(int l, int bs, int s2, const double* dA, double* dG, int* fail_layer, void* stream);
/* Same with a whole DomainPlan: s2_levels[0] partitions the band, s2_levels[1..] the
 * interface system level by level (ddrgf.hpp:363-369). */
int bbsi_cuda_ddrgf_plan_dev(int l, int bs, const int* s2_levels, int n_levels, const double* dA, double* dG,
                             int* fail_layer, void* stream);
/* Domain-sharded DDRGF, phase by phase (one process per GPU, the caller does the
 * collectives; paper_2605_19910_b200/distributed.py). Tasks = interleave_permutation(l,1,s2)
 * groups (partition.hpp:39-75), T = bbsi_cuda_ddrgf_num_tasks(l, s2). A rank owning
 * tasks [t0,t1) holds the band rows of layers [first(t0), sep(t1-1)] (dA/dG local,
 * [rows][3][bs][bs], slot order). Protocol:
 *   phase1 -> all-gather of the packets (packet_bytes(t1-t0) per rank, T packets in
 *   task order) -> phase2 (identical on every rank) -> phase3 (chains, in place) ->
 *   halo (2 blocks per rank) all-gathered -> couplings (the previous rank's halo[1] and
 *   the next rank's halo[0]; NULL at the ends).
 * Only the packets (9 bs x bs blocks per task) and the halos cross ranks. */
int bbsi_cuda_ddrgf_num_tasks(int l, int s2);
long long bbsi_cuda_ddrgf_packet_bytes(int ntask, int bs);
long long bbsi_cuda_ddrgf_phase2_bytes(int ntask, int bs);
int bbsi_cuda_ddrgf_phase1_dev(int l, int bs, int s2, int t0, int t1, const double* dA, double* dG, double* dPacket,
                               int* fail_layer, void* stream);
int bbsi_cuda_ddrgf_phase2_dev(int l, int bs, int s2, const double* dPackets, double* dOut, int* fail_layer,
                               void* stream);
int bbsi_cuda_ddrgf_phase3_dev(int l, int bs, int s2, int t0, int t1, const double* dA, double* dG, const double* dOut,
                               int* fail_layer, void* stream);
/* dHalo [2][bs][bs] = { G[x0(t0), x0(t0)], G[sep(t1-1), sep(t1-1)] } after phase 3. */
int bbsi_cuda_ddrgf_halo_dev(int l, int bs, int s2, int t0, int t1, const double* dG, double* dHalo, void* stream);
/* The inter-chain coupling blocks G[x0_t, sep_{t-1}] and G[sep_t, x0_{t+1}] of the local
 * tasks; dPrevSepG = previous rank's halo[1] (t0 > 0), dNextX0G = next rank's halo[0]
 * (t1 < T), NULL otherwise. */
int bbsi_cuda_ddrgf_couplings_dev(int l, int bs, int s2, int t0, int t1, const double* dA, double* dG,
                                  const double* dOut, const double* dPrevSepG, const double* dNextX0G, void* stream);

/* ---------------------------------------------------------------- multi-GPU (NCCL inside the library)
 * The reference's concurrency seam is run_tasks inside ddrgf (ddrgf.hpp:239-262,
 * 355-386); here domains map onto GPUs and NCCL carries the interface packets.
 * NCCL is loaded at first use (dlopen libnccl.so.2); without it these return
 * BBSI_CUDA_ERROR. */
int bbsi_cuda_nccl_available(void);
/* ncclGetUniqueId into out128 (128 bytes; rank 0 creates it, the caller broadcasts it). */
int bbsi_cuda_nccl_unique_id(void* out128);
/* ncclCommInitRank on the current device; *comm is an opaque ncclComm_t. */
int bbsi_cuda_nccl_comm_init(const void* id128, int nranks, int rank, void** comm);
void bbsi_cuda_nccl_comm_destroy(void* comm);
/* The task range [t0,t1) and band rows [L0,L1) a rank owns (balanced contiguous ranges). */
int bbsi_cuda_ddrgf_rank_layers(int l, int s2, int nranks, int rank, int* t0, int* t1, int* L0, int* L1);
/* One rank of the domain-sharded DDRGF (one process per GPU): dA_loc / dG_loc are its
 * band rows [L0, L1); phase 1, the NCCL all-gather of the packets, phase 2, phase 3, the
 * halo all-gather and the couplings all run inside. Every rank returns the same
 * status (a singular pivot anywhere is reported on all ranks). */
int bbsi_cuda_ddrgf_rank_dev(void* comm, int l, int bs, int s2, const double* dA_loc, double* dG_loc,
                             int* fail_layer, void* stream);
/* The same with a multi-level DomainPlan (ddrgf.hpp:18-32, 363-369): ranks own level-0
 * tasks of s2_levels[0]; the interface system every rank solves redundantly after the
 * packet all-gather is nested over s2_levels[1..]. */
int bbsi_cuda_ddrgf_rank_plan_dev(void* comm, int l, int bs, const int* s2_levels, int n_levels, const double* dA_loc,
                                  double* dG_loc, int* fail_layer, void* stream);
/* bbsi::ddrgf (ddrgf.hpp:420-428) over ngpu GPUs of this process (devices: NULL = 0..ngpu-1):
 * ncclCommInitAll, one host thread per GPU, domains sharded as above. Same arguments and
 * results as bbsi_cuda_ddrgf_z. */
int bbsi_cuda_ddrgf_multi_z(int l, int w, int bs, const int* sizes, const double* A, const int* s2_levels,
                            int n_levels, int n_threads, int terminal_threads, int ngpu, const int* devices, double* G,
                            long long* counters, int* fail_layer);
/* bbsi_cuda_dyson_rgf_z with the energies sharded contiguously over ngpu GPUs (no collective). */
int bbsi_cuda_dyson_rgf_multi_z(int l, int w, int bs, int n_energy, const double* H, const double* z,
                                const double* sigma, double* G, int* fail_layers, int chunk, int ngpu,
                                const int* devices);

/* Dyson DDRGF for one energy z (host complex) from the shared device H. */
int bbsi_cuda_dyson_ddrgf_dev(int l, int bs, const double* dH, const double* z, const double* sigma, int s2,
                              double* dG, int* fail_layer, void* stream);

/* Seeded Dyson Hamiltonian (include/.. csrc/dyson_gen.h spec) written on the device. */
int bbsi_cuda_dyson_fill_h_dev(int l, int w, int b, uint64_t seed, double* dH, void* stream);
/* Band rows [a0, a1) of the same H (a rank's share of a domain-sharded band). */
int bbsi_cuda_dyson_fill_h_rows_dev(int l, int w, int b, uint64_t seed, int a0, int a1, double* dH, void* stream);
/* Same bytes on the host (for the end-to-end path and the parity tests). */
void bbsi_dyson_fill_h_host(int l, int w, int b, uint64_t seed, double* H);
/* random_spd_like<std::complex<double>> (block_banded.hpp:99-133, raw mt19937_64 bits,
 * block_banded.hpp:70-91) into slot memory (l x (2w+1) slots of bs x bs column-major,
 * bs = max block size; out-of-band slots zero). Host only; used by the CLI's generated
 * inputs. Returns BBSI_INVALID_ARGUMENT for a bad layout or dominance <= 0. */
int bbsi_random_spd_like_z(int l, int w, int bs, const int* sizes, uint64_t seed, double dominance, double* A);

/* Kernel timings for the GPU cost model (the B200 counterpart of benchmark_kernels,
 * microbench.hpp / cost_model.hpp:12-18): mean device time of ONE batched launch over
 * `batch` n x n complex128 matrices, out[0] = GEMM (C = A*B) seconds, out[1] = inversion
 * (zgetrf + zgetrs(I) equivalent) seconds, out[2] = timed samples. n % 64 == 0. */
int bbsi_cuda_bench_kernels(int n, int batch, int samples, double* out);

/* ---------------------------------------------------------------- kernel-level API (device pointers)
 * Batched C = alpha*A*B + beta*C on plain column-major complex128 matrices,
 * m, n % 64 == 0, k % 16 == 0 (the sm_100a DMMA GEMM of the sweeps). */
int bbsi_cuda_zgemm_dev(int m, int n, int k, const double* alpha, const double* dA, long long lda,
                        long long a_bstride, const double* dB, long long ldb, long long b_bstride,
                        const double* beta, double* dC, long long ldc, long long c_bstride, int batch,
                        void* stream);
/* Batched in-place inverse (GJ with partial pivoting), n % 64 == 0, threshold on
 * the leading n_true x n_true block; status_host[batch] = -1 or first bad pivot. */
int bbsi_cuda_zinv_dev(int n, int n_true, int batch, double* dM, long long ld, long long bstride,
                       int* status_host, void* stream);

/* ---------------------------------------------------------------- instrumentation
 * Number of library kernel launches since load (all entry points). */
long long bbsi_cuda_launch_count(void);
/* When enabled, every library kernel launch is bracketed by CUDA events on its
 * stream; collect() synchronises and returns, per category (0 GEMM, 1 inversion,
 * 2 band ops), {launches, total ms, algorithmic FLOPs, algorithmic bytes} and
 * clears the records. */
void bbsi_cuda_profile_enable(int on);
int bbsi_cuda_profile_collect(double* out, int ncat);
/* Measured FP64 DMMA (mma.sync f64) peak of device 0 in TFLOP/s (best of reps). */
double bbsi_cuda_fp64_peak_tflops(double duration_ms, int reps);

#ifdef __cplusplus
}
#endif
#endif

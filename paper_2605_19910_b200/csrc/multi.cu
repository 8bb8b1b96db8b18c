// NCCL for the multi-GPU paths: the packet all-gather of the
// domain-sharded DDRGF and its two-block halo exchange, over NVLink / NVSwitch.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2": the one torch already mapped, or
// the system's), so the library has no link-time NCCL dependency and single-GPU users
// never load it; a multi-GPU call without NCCL fails loudly (BBSI_CUDA_ERROR).
//
// The reference's concurrency seam is run_tasks inside ddrgf (ddrgf.hpp:239-262,
// 355-386): a fork-join over tasks on host threads. Here a rank owns a contiguous
// task range on its GPU and the only data that crosses GPUs is, per task, the 9-block
// interface packet (after phase 1) and, per rank, two boundary blocks (after phase 3).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace bbsi_gpu {

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a = [] {
    NcclApi x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      x.err = std::string("NCCL not found: ") + dlerror();
      return x;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && x.err.empty()) x.err = std::string("NCCL symbol missing: ") + n;
      return p;
    };
    x.GetUniqueId = reinterpret_cast<decltype(x.GetUniqueId)>(sym("ncclGetUniqueId"));
    x.CommInitRank = reinterpret_cast<decltype(x.CommInitRank)>(sym("ncclCommInitRank"));
    x.CommInitAll = reinterpret_cast<decltype(x.CommInitAll)>(sym("ncclCommInitAll"));
    x.CommDestroy = reinterpret_cast<decltype(x.CommDestroy)>(sym("ncclCommDestroy"));
    x.CommCount = reinterpret_cast<decltype(x.CommCount)>(sym("ncclCommCount"));
    x.CommUserRank = reinterpret_cast<decltype(x.CommUserRank)>(sym("ncclCommUserRank"));
    x.AllGather = reinterpret_cast<decltype(x.AllGather)>(sym("ncclAllGather"));
    x.GroupStart = reinterpret_cast<decltype(x.GroupStart)>(sym("ncclGroupStart"));
    x.GroupEnd = reinterpret_cast<decltype(x.GroupEnd)>(sym("ncclGroupEnd"));
    x.GetErrorString = reinterpret_cast<decltype(x.GetErrorString)>(sym("ncclGetErrorString"));
    x.ok = x.err.empty();
    return x;
  }();
  return a;
}

std::string nerr(ncclResult_t r) {
  return api().GetErrorString ? api().GetErrorString(r) : ("NCCL error " + std::to_string(int(r)));
}

// all-gather of `count` doubles per rank
cudaError_t gather_doubles(ncclComm_t c, const double* send, double* recv, size_t count, cudaStream_t s,
                           std::string* err) {
  ncclResult_t r = api().AllGather(send, recv, count, ncclFloat64, c, s);
  if (r != ncclSuccess) {
    *err = "ncclAllGather: " + nerr(r);
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}

}  // namespace

bool nccl_ready(std::string* err) {
  if (!api().ok && err) *err = api().err;
  return api().ok;
}

int nccl_unique_id(void* out, std::string* err) {
  if (!nccl_ready(err)) return 1;
  ncclUniqueId id;
  ncclResult_t r = api().GetUniqueId(&id);
  if (r != ncclSuccess) {
    *err = "ncclGetUniqueId: " + nerr(r);
    return 1;
  }
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

int nccl_comm_init_rank(const void* id, int nranks, int rank, void** comm, std::string* err) {
  if (!nccl_ready(err)) return 1;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  ncclResult_t r = api().CommInitRank(&c, nranks, u, rank);
  if (r != ncclSuccess) {
    *err = "ncclCommInitRank: " + nerr(r);
    return 1;
  }
  *comm = c;
  return 0;
}

int nccl_comm_init_all(int n, const int* devs, std::vector<void*>& comms, std::string* err) {
  if (!nccl_ready(err)) return 1;
  std::vector<ncclComm_t> c(n);
  ncclResult_t r = api().CommInitAll(c.data(), n, devs);
  if (r != ncclSuccess) {
    *err = "ncclCommInitAll: " + nerr(r);
    return 1;
  }
  comms.assign(c.begin(), c.end());
  return 0;
}

void nccl_comm_destroy(void* comm) {
  if (comm && api().ok) api().CommDestroy(static_cast<ncclComm_t>(comm));
}

int nccl_comm_shape(void* comm, int* nranks, int* rank, std::string* err) {
  if (!nccl_ready(err)) return 1;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  if (api().CommCount(c, nranks) != ncclSuccess || api().CommUserRank(c, rank) != ncclSuccess) {
    *err = "ncclCommCount / ncclCommUserRank failed";
    return 1;
  }
  return 0;
}

// The packet and halo exchanges of ddrgf_rank over a NCCL communicator. Buffers come
// from the calling thread's arena (slots 20-23).
DdrgfExchange nccl_ddrgf_exchange(void* comm, int l, int b, int s2, std::string* err) {
  DdrgfExchange x;
  const long long bb = (long long)b * b;
  x.packets = [=](double2* all, int t0, int t1, int fl, int* any, cudaStream_t s) -> cudaError_t {
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int nr = 1, rk = 0;
    if (nccl_comm_shape(comm, &nr, &rk, err)) return cudaErrorUnknown;
    const int T = ddrgf_num_tasks(l, s2);
    const auto ranges = ddrgf_rank_ranges(T, nr);
    int maxn = 0;
    for (auto& r : ranges) maxn = std::max(maxn, r.second - r.first);
    const size_t pk_elems = ddrgf_packet_bytes(1, b) / sizeof(double2);  // one task's packet
    // send: this rank's packets padded to maxn, plus one header word (its failure layer)
    const size_t per_rank = size_t(maxn) * pk_elems * 2 + 2;  // doubles
    double* send = static_cast<double*>(arena_get(20, per_rank * sizeof(double)));
    double* recv = static_cast<double*>(arena_get(21, per_rank * nr * sizeof(double)));
    if (!send || !recv) return cudaErrorMemoryAllocation;
    cudaError_t e;
    const size_t own = size_t(t1 - t0) * pk_elems * sizeof(double2);
    if ((e = cudaMemcpyAsync(send, all + size_t(t0) * pk_elems, own, cudaMemcpyDeviceToDevice, s))) return e;
    const double hdr[2] = {double(fl), 0.0};
    if ((e = cudaMemcpyAsync(send + per_rank - 2, hdr, sizeof(hdr), cudaMemcpyHostToDevice, s))) return e;
    if ((e = gather_doubles(c, send, recv, per_rank, s, err))) return e;
    for (int r = 0; r < nr; ++r) {
      const auto [a, z] = ranges[r];
      if (r == rk || z == a) continue;
      if ((e = cudaMemcpyAsync(all + size_t(a) * pk_elems, recv + size_t(r) * per_rank,
                               size_t(z - a) * pk_elems * sizeof(double2), cudaMemcpyDeviceToDevice, s)))
        return e;
    }
    std::vector<double> hdrs(size_t(nr) * 2);
    if ((e = cudaMemcpy2DAsync(hdrs.data(), 2 * sizeof(double), recv + per_rank - 2, per_rank * sizeof(double),
                               2 * sizeof(double), nr, cudaMemcpyDeviceToHost, s)))
      return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    *any = -1;
    for (int r = 0; r < nr; ++r) {
      const int f = int(hdrs[2 * r]);
      if (f >= 0 && (*any < 0 || f < *any)) *any = f;
    }
    return cudaSuccess;
  };
  x.halo = [=](const double2* own, double2* nbr, int fl, int* any, cudaStream_t s) -> cudaError_t {
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int nr = 1, rk = 0;
    if (nccl_comm_shape(comm, &nr, &rk, err)) return cudaErrorUnknown;
    const size_t per_rank = size_t(2 * bb) * 2 + 2;
    double* send = static_cast<double*>(arena_get(22, per_rank * sizeof(double)));
    double* recv = static_cast<double*>(arena_get(23, per_rank * nr * sizeof(double)));
    if (!send || !recv) return cudaErrorMemoryAllocation;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(send, own, 2 * bb * sizeof(double2), cudaMemcpyDeviceToDevice, s))) return e;
    const double hdr[2] = {double(fl), 0.0};
    if ((e = cudaMemcpyAsync(send + per_rank - 2, hdr, sizeof(hdr), cudaMemcpyHostToDevice, s))) return e;
    if ((e = gather_doubles(c, send, recv, per_rank, s, err))) return e;
    if (rk > 0 &&
        (e = cudaMemcpyAsync(nbr, recv + size_t(rk - 1) * per_rank + 2 * bb, bb * sizeof(double2),
                             cudaMemcpyDeviceToDevice, s)))
      return e;
    if (rk + 1 < nr &&
        (e = cudaMemcpyAsync(nbr + bb, recv + size_t(rk + 1) * per_rank, bb * sizeof(double2),
                             cudaMemcpyDeviceToDevice, s)))
      return e;
    std::vector<double> hdrs(size_t(nr) * 2);
    if ((e = cudaMemcpy2DAsync(hdrs.data(), 2 * sizeof(double), recv + per_rank - 2, per_rank * sizeof(double),
                               2 * sizeof(double), nr, cudaMemcpyDeviceToHost, s)))
      return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    *any = -1;
    for (int r = 0; r < nr; ++r) {
      const int f = int(hdrs[2 * r]);
      if (f >= 0 && (*any < 0 || f < *any)) *any = f;
    }
    return cudaSuccess;
  };
  return x;
}

}  // namespace bbsi_gpu

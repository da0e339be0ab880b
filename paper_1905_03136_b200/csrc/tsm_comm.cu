// tsm_comm.cu -- multi-GPU layer of libtsm.
//
// One process per GPU; K is sharded by rows (rank r holds a contiguous row
// block of A and B, as in distributed block-vector solvers).
//   TSMTTSM: local fixed-order TSMTTSM of the shard -> sum of the tiny C over
//            ranks: ncclAllReduce (sum), or, with TSM_COMM_DETERMINISTIC,
//            ncclAllGather of the partial C's + a fixed rank-order sum.
//   TSMM:    ncclBroadcast(C) from root, then the purely local TSMM.
//
// NCCL is resolved with dlopen("libnccl.so.2") at tsm_comm_init time, i.e.
// the NCCL already loaded into the process (torch's wheel), so there is one
// NCCL per process.  The handful of ABI constants used here are NCCL's stable
// public values (ncclFloat64 = 8, ncclSum = 0, 128-byte unique id).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/libtsm.h"
#include "tsm_internal.h"

namespace {

typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclFloat64 = 8;
constexpr int kNcclSum = 0;

struct NcclApi {
  bool loaded = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

bool load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.loaded) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  const char* env = getenv("TSM_NCCL_LIB");
  if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  for (const char* n : names) {
    if (h) break;
    h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) {
    g_nccl.err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
    return false;
  }
#define TSM_SYM(field, name)                                             \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
  if (!g_nccl.field) {                                                   \
    g_nccl.err = std::string("missing NCCL symbol ") + name;             \
    return false;                                                        \
  }
  TSM_SYM(GetUniqueId, "ncclGetUniqueId");
  TSM_SYM(CommInitRank, "ncclCommInitRank");
  TSM_SYM(CommDestroy, "ncclCommDestroy");
  TSM_SYM(AllReduce, "ncclAllReduce");
  TSM_SYM(AllGather, "ncclAllGather");
  TSM_SYM(Broadcast, "ncclBroadcast");
  TSM_SYM(GetErrorString, "ncclGetErrorString");
#undef TSM_SYM
  g_nccl.loaded = true;
  return true;
}

tsm_status nccl_fail(ncclResult_t r, const char* what) {
  std::string s = std::string(what) + ": ";
  s += g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : std::to_string(r);
  return tsm::fail(TSM_ERR_NCCL, s);
}

__global__ void rank_sum_kernel(const double* __restrict__ g, double* __restrict__ C, int nranks,
                                int cells) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cells) return;
  double s = g[i];
  for (int r = 1; r < nranks; r++) s += g[static_cast<long long>(r) * cells + i];  // rank order
  C[i] = s;
}

}  // namespace

struct tsm_comm_s {
  ncclComm_t comm;
  int nranks, rank, device, flags;
};

namespace tsm {
tsm_status rank_sum(const double* gathered, double* C, int nranks, int cells, void* stream) {
  rank_sum_kernel<<<(cells + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      gathered, C, nranks, cells);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TSM_ERR_CUDA, std::string("rank_sum launch: ") + cudaGetErrorString(e));
  return TSM_SUCCESS;
}
}  // namespace tsm

using tsm::fail;

extern "C" {

tsm_status tsm_comm_unique_id(void* uid128) {
  if (!uid128) return fail(TSM_ERR_INVALID_VALUE, "uid == NULL");
  if (!load_nccl()) return fail(TSM_ERR_NCCL, g_nccl.err);
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(uid128, id.internal, 128);
  return TSM_SUCCESS;
}

tsm_status tsm_comm_init(tsm_comm* out, const void* uid128, int nranks, int rank, int device,
                         int flags) {
  if (!out || !uid128) return fail(TSM_ERR_INVALID_VALUE, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TSM_ERR_INVALID_VALUE, "bad rank/nranks");
  if (!load_nccl()) return fail(TSM_ERR_NCCL, g_nccl.err);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(TSM_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  ncclUniqueId id;
  memcpy(id.internal, uid128, 128);
  ncclComm_t comm = nullptr;
  ncclResult_t r = g_nccl.CommInitRank(&comm, nranks, id, rank);
  if (prev != device) cudaSetDevice(prev);
  if (r != 0) return nccl_fail(r, "ncclCommInitRank");
  tsm_comm c = new tsm_comm_s{comm, nranks, rank, device, flags};
  *out = c;
  return TSM_SUCCESS;
}

tsm_status tsm_comm_destroy(tsm_comm c) {
  if (!c) return TSM_SUCCESS;
  ncclResult_t r = g_nccl.CommDestroy ? g_nccl.CommDestroy(c->comm) : 0;
  delete c;
  if (r != 0) return nccl_fail(r, "ncclCommDestroy");
  return TSM_SUCCESS;
}

tsm_status tsm_comm_workspace_extra_bytes(tsm_comm c, tsm_plan p, size_t* bytes) {
  if (!c || !p || !bytes) return fail(TSM_ERR_INVALID_VALUE, "null argument");
  *bytes = (c->flags & TSM_COMM_DETERMINISTIC)
               ? static_cast<size_t>(c->nranks) * tsm::plan_cells(p) * sizeof(double)
               : 0;
  return TSM_SUCCESS;
}

static tsm_status allreduce_impl(tsm_plan p, tsm_comm c, int dt, int64_t K, const void* A,
                                 const void* B, void* C, void* ws, size_t ws_bytes,
                                 tsm_stream stream) {
  if (!p || !c) return fail(TSM_ERR_INVALID_VALUE, "null plan/comm");
  if (K < 0) return fail(TSM_ERR_INVALID_VALUE, "K_local < 0");
  const int cells = tsm::plan_cells(p);
  const size_t local = tsm::workspace_bytes(p, K);
  const size_t extra = (c->flags & TSM_COMM_DETERMINISTIC)
                           ? static_cast<size_t>(c->nranks) * cells * sizeof(double)
                           : 0;
  if (ws_bytes < local + extra) return fail(TSM_ERR_WORKSPACE, "workspace too small for sharded TSMTTSM");
  tsm_status st = tsm::launch_tsmttsm(p, dt, K, A, B, C, ws, ws_bytes - extra, stream, true);
  if (st != TSM_SUCCESS) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // (a 1-rank communicator still goes through NCCL: same code path at any size)
  if (c->flags & TSM_COMM_DETERMINISTIC) {
    // gather region: 256-byte aligned, after the local workspace
    size_t off = (local + 255) & ~static_cast<size_t>(255);
    if (off + extra > ws_bytes) off = local;  // caller sized exactly; still 16 B aligned
    double* gathered = reinterpret_cast<double*>(static_cast<char*>(ws) + off);
    ncclResult_t r = g_nccl.AllGather(C, gathered, static_cast<size_t>(cells), kNcclFloat64, c->comm, s);
    if (r != 0) return nccl_fail(r, "ncclAllGather");
    return tsm::rank_sum(gathered, static_cast<double*>(C), c->nranks, cells, stream);
  }
  ncclResult_t r = g_nccl.AllReduce(C, C, static_cast<size_t>(cells), kNcclFloat64, kNcclSum, c->comm, s);
  if (r != 0) return nccl_fail(r, "ncclAllReduce");
  return TSM_SUCCESS;
}

tsm_status tsmttsm_allreduce_d(tsm_plan p, tsm_comm c, int64_t K_local, const double* A,
                               const double* B, double* C, void* ws, size_t ws_bytes,
                               tsm_stream stream) {
  return allreduce_impl(p, c, TSM_D, K_local, A, B, C, ws, ws_bytes, stream);
}
tsm_status tsmttsm_allreduce_z(tsm_plan p, tsm_comm c, int64_t K_local, const tsm_zcomplex* A,
                               const tsm_zcomplex* B, tsm_zcomplex* C, void* ws,
                               size_t ws_bytes, tsm_stream stream) {
  return allreduce_impl(p, c, TSM_Z, K_local, A, B, C, ws, ws_bytes, stream);
}

static tsm_status bcast_impl(tsm_plan p, tsm_comm c, int dt, int root, int64_t K, const void* A,
                             void* C, void* B, tsm_stream stream) {
  if (!p || !c || !C) return fail(TSM_ERR_INVALID_VALUE, "null plan/comm/C");
  if (root < 0 || root >= c->nranks) return fail(TSM_ERR_INVALID_VALUE, "bad root");
  if (tsm::plan_op(p) != TSM_OP_TSMM || tsm::plan_dt(p) != dt)
    return fail(TSM_ERR_INVALID_VALUE, "plan op/dtype does not match the call");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ncclResult_t r = g_nccl.Broadcast(C, C, static_cast<size_t>(tsm::plan_cells(p)), kNcclFloat64,
                                    root, c->comm, s);
  if (r != 0) return nccl_fail(r, "ncclBroadcast");
  return tsm::launch_tsmm(p, dt, K, A, C, B, stream, true);
}

tsm_status tsmm_bcast_d(tsm_plan p, tsm_comm c, int root, int64_t K_local, const double* A,
                        double* C, double* B, tsm_stream stream) {
  return bcast_impl(p, c, TSM_D, root, K_local, A, C, B, stream);
}
tsm_status tsmm_bcast_z(tsm_plan p, tsm_comm c, int root, int64_t K_local, const tsm_zcomplex* A,
                        tsm_zcomplex* C, tsm_zcomplex* B, tsm_stream stream) {
  return bcast_impl(p, c, TSM_Z, root, K_local, A, C, B, stream);
}

// One block classical Gram-Schmidt projection (NEXT row N1):
// C = A^T B (A^H B with a TSM_FLAG_CONJ plan), summed over ranks when comm is
// given, then B <- B - A C through the TSMM update path (reduce-add into B).
static tsm_status cgs_impl(tsm_plan ptt, tsm_plan pmm, tsm_comm c, int dt, int64_t K, const void* A,
                           void* B, void* C, void* ws, size_t ws_bytes, tsm_stream stream) {
  if (!ptt || !pmm) return fail(TSM_ERR_INVALID_VALUE, "null plan");
  if (tsm::plan_op(ptt) != TSM_OP_TSMTTSM || tsm::plan_op(pmm) != TSM_OP_TSMM)
    return fail(TSM_ERR_INVALID_VALUE, "p_tt must be a TSMTTSM plan and p_mm a TSMM plan");
  if (tsm::plan_dt(ptt) != dt || tsm::plan_dt(pmm) != dt)
    return fail(TSM_ERR_INVALID_VALUE, "plan dtype does not match the call");
  if (tsm::plan_M(ptt) != tsm::plan_M(pmm) || tsm::plan_N(ptt) != tsm::plan_N(pmm))
    return fail(TSM_ERR_INVALID_VALUE, "p_tt and p_mm must have the same (M, N)");
  tsm_status st = c ? allreduce_impl(ptt, c, dt, K, A, B, C, ws, ws_bytes, stream)
                    : tsm::launch_tsmttsm(ptt, dt, K, A, B, C, ws, ws_bytes, stream, false);
  if (st != TSM_SUCCESS) return st;
  return tsm::launch_tsmm_update(pmm, dt, K, -1.0, 0.0, A, C, 1.0, 0.0, B, stream, c != nullptr);
}

tsm_status tsm_cgs_step_d(tsm_plan p_tt, tsm_plan p_mm, tsm_comm comm, int64_t K, const double* A,
                          double* B, double* C, void* ws, size_t ws_bytes, tsm_stream stream) {
  return cgs_impl(p_tt, p_mm, comm, TSM_D, K, A, B, C, ws, ws_bytes, stream);
}
tsm_status tsm_cgs_step_z(tsm_plan p_tt, tsm_plan p_mm, tsm_comm comm, int64_t K,
                          const tsm_zcomplex* A, tsm_zcomplex* B, tsm_zcomplex* C, void* ws,
                          size_t ws_bytes, tsm_stream stream) {
  return cgs_impl(p_tt, p_mm, comm, TSM_Z, K, A, B, C, ws, ws_bytes, stream);
}

}  // extern "C"

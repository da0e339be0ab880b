// tsm_peer.cu -- NEXT N3: TSMTTSM with the grid reduction
// fused with the cross-GPU sum over peer memory (include/libtsm.h tsm_peer_*).
//
// Each rank allocates one slot buffer (header + 2 parities x kMaxPeers slots
// of kPeerCells doubles); every rank maps every other rank's buffer with CUDA
// IPC, so the finisher blocks of the TSMTTSM kernel (tsm_kernels.cuh
// grid_reduce, PeerArgs) store straight into peer HBM over NVLink and signal
// with system-scope atomics.  The host side only tracks the call count: call n
// uses parity n & 1 and waits for cnt[parity] >= (n / 2 + 1) * nranks.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../include/libtsm.h"
#include "tsm_internal.h"
#include "tsm_kernels.cuh"

using tsm::fail;
using tsm::kMaxPeers;
using tsm::kPeerCells;
using tsm::kPeerHeaderBytes;

struct tsm_peer_s {
  int nranks = 0, rank = 0, device = 0;
  double* own = nullptr;                  // this rank's slot buffer (cudaMalloc)
  double* base[kMaxPeers] = {};           // every rank's buffer as mapped here
  bool opened[kMaxPeers] = {};            // IPC mappings to close
  bool ready = false;                     // tsm_peer_open done
  unsigned long long calls = 0;           // fused reductions issued (parity / target / seq)
  unsigned long long timeout_ns = 2000000000ull;  // bounded wait for the other ranks
};

namespace {

constexpr size_t kPeerBytes =
    kPeerHeaderBytes + sizeof(double) * static_cast<size_t>(2) * kMaxPeers * kPeerCells;

tsm_status cuda_err(cudaError_t e, const char* what) {
  return fail(TSM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevScope {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DevScope(int d) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != d) err = cudaSetDevice(d);
    else prev = -1;
  }
  ~DevScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

tsm_status peer_call(tsm_plan p, tsm_peer c, int dt, int64_t K, const void* A, const void* B, void* C,
                     void* ws, size_t ws_bytes, tsm_stream stream) {
  if (!p || !c) return fail(TSM_ERR_INVALID_VALUE, "null plan / peer");
  if (!c->ready) return fail(TSM_ERR_INVALID_VALUE, "tsm_peer_open has not been called");
  if (tsm::plan_op(p) != TSM_OP_TSMTTSM || tsm::plan_dt(p) != dt)
    return fail(TSM_ERR_INVALID_VALUE, "plan op/dtype does not match the call");
  if (tsm::plan_device(p) != c->device) return fail(TSM_ERR_INVALID_VALUE, "plan and peer on different devices");
  if (tsm::plan_cells(p) > kPeerCells) return fail(TSM_ERR_INTERNAL, "C larger than a peer slot");
  tsm::PeerArgs q{};
  for (int r = 0; r < c->nranks; r++) q.base[r] = c->base[r];
  q.nranks = c->nranks;
  q.rank = c->rank;
  q.parity = static_cast<int>(c->calls & 1ull);
  q.target = ((c->calls >> 1) + 1ull) * static_cast<unsigned long long>(c->nranks);
  q.seq = c->calls + 1ull;
  q.timeout_ns = c->timeout_ns;
  tsm_status st = tsm::launch_tsmttsm(p, dt, K, A, B, C, ws, ws_bytes, stream, true, 0, 0, &q);
  if (st == TSM_SUCCESS) c->calls++;  // a launched call has signalled (or will) on every rank
  return st;
}

}  // namespace

extern "C" {

tsm_status tsm_peer_create(tsm_peer* out, int nranks, int rank, int device) {
  if (!out) return fail(TSM_ERR_INVALID_VALUE, "out == NULL");
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks)
    return fail(TSM_ERR_INVALID_VALUE, "nranks must be in [1, 8] and rank in [0, nranks)");
  DevScope ds(device);
  if (ds.err != cudaSuccess) return cuda_err(ds.err, "cudaSetDevice");
  tsm_peer c = new (std::nothrow) tsm_peer_s;
  if (!c) return fail(TSM_ERR_INTERNAL, "out of host memory");
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  void* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, kPeerBytes);
  if (e == cudaSuccess) e = cudaMemset(buf, 0, kPeerBytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (buf) cudaFree(buf);
    delete c;
    return cuda_err(e, "slot buffer");
  }
  c->own = static_cast<double*>(buf);
  c->base[rank] = c->own;
  *out = c;
  return TSM_SUCCESS;
}

tsm_status tsm_peer_export(tsm_peer c, void* handle64) {
  if (!c || !handle64) return fail(TSM_ERR_INVALID_VALUE, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  DevScope ds(c->device);
  if (ds.err != cudaSuccess) return cuda_err(ds.err, "cudaSetDevice");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, c->own);
  if (e != cudaSuccess) return cuda_err(e, "cudaIpcGetMemHandle");
  memcpy(handle64, &h, 64);
  return TSM_SUCCESS;
}

tsm_status tsm_peer_open(tsm_peer c, const void* handles) {
  if (!c || !handles) return fail(TSM_ERR_INVALID_VALUE, "null argument");
  if (c->ready) return fail(TSM_ERR_INVALID_VALUE, "tsm_peer_open called twice");
  DevScope ds(c->device);
  if (ds.err != cudaSuccess) return cuda_err(ds.err, "cudaSetDevice");
  const char* hs = static_cast<const char*>(handles);
  for (int r = 0; r < c->nranks; r++) {
    if (r == c->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, hs + 64 * r, 64);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int q = 0; q < r; q++)
        if (c->opened[q]) {
          cudaIpcCloseMemHandle(c->base[q]);
          c->opened[q] = false;
          c->base[q] = nullptr;
        }
      return cuda_err(e, ("cudaIpcOpenMemHandle(rank " + std::to_string(r) + ")").c_str());
    }
    c->base[r] = static_cast<double*>(ptr);
    c->opened[r] = true;
  }
  c->ready = true;
  return TSM_SUCCESS;
}

tsm_status tsm_peer_destroy(tsm_peer c) {
  if (!c) return TSM_SUCCESS;
  {
    DevScope ds(c->device);
    for (int r = 0; r < c->nranks; r++)
      if (c->opened[r]) cudaIpcCloseMemHandle(c->base[r]);
    if (c->own) cudaFree(c->own);
  }
  delete c;
  return TSM_SUCCESS;
}

tsm_status tsm_peer_error(tsm_peer c, int* err) {
  if (!c || !err) return fail(TSM_ERR_INVALID_VALUE, "null argument");
  DevScope ds(c->device);
  if (ds.err != cudaSuccess) return cuda_err(ds.err, "cudaSetDevice");
  unsigned int v = 0;
  cudaError_t e = cudaMemcpy(&v, reinterpret_cast<char*>(c->own) + 16, sizeof v, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_err(e, "read peer error flag");
  *err = v ? 1 : 0;
  return TSM_SUCCESS;
}

tsm_status tsm_peer_set_timeout(tsm_peer c, uint64_t timeout_ns) {
  if (!c || timeout_ns == 0) return fail(TSM_ERR_INVALID_VALUE, "null peer / zero timeout");
  c->timeout_ns = timeout_ns;
  return TSM_SUCCESS;
}

tsm_status tsm_peer_reset(tsm_peer c, tsm_stream stream) {
  if (!c) return fail(TSM_ERR_INVALID_VALUE, "null peer");
  DevScope ds(c->device);
  if (ds.err != cudaSuccess) return cuda_err(ds.err, "cudaSetDevice");
  // wait for this rank's fused calls, then clear its header (counters, err, seq);
  // the slots themselves are rewritten by every call before they are read
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaMemset(c->own, 0, kPeerHeaderBytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_err(e, "tsm_peer_reset");
  c->calls = 0;
  return TSM_SUCCESS;
}

tsm_status tsmttsm_peer_d(tsm_plan p, tsm_peer c, int64_t K_local, const double* A, const double* B,
                          double* C, void* ws, size_t ws_bytes, tsm_stream stream) {
  return peer_call(p, c, TSM_D, K_local, A, B, C, ws, ws_bytes, stream);
}

tsm_status tsmttsm_peer_z(tsm_plan p, tsm_peer c, int64_t K_local, const tsm_zcomplex* A,
                          const tsm_zcomplex* B, tsm_zcomplex* C, void* ws, size_t ws_bytes,
                          tsm_stream stream) {
  return peer_call(p, c, TSM_Z, K_local, A, B, C, ws, ws_bytes, stream);
}

}  // extern "C"

// tsm_internal.h -- internal host-side interfaces shared by the libtsm sources.
#pragma once
#include <string>

#include "../../include/libtsm.h"
#include "tsm_registry.h"

namespace tsm {

// Registry (tsm_registry.cpp + generated tables).
const KernelEntry* find_aot(int op, int dt, int M, int N);
const KernelEntry* find_aot_config(const KernelEntry& want);  // same shape AND config
const KernelEntry* default_params(int op, int dt, int M, int N);
// TSM_FLAG_STRIDED plans (NEXT N4): a TMA kernel configuration when the shape
// has one, else a gather-capable one; TSM_FLAG_GATHER: always gather-capable
const KernelEntry* default_params_strided(int op, int dt, int M, int N);
const KernelEntry* default_params_gather(int op, int dt, int M, int N);
bool strided_capable(const KernelEntry& k);  // TMA or gather-capable
bool gather_capable(const KernelEntry& k);   // TSMTTSM 1 / TSMM 4: any row stride, 8-byte D bases
const char* build_info_json();

// NVRTC run-time instantiation (tsm_jit.cpp).
tsm_status jit_kernel(const KernelEntry& want, const KernelEntry** out);
tsm_status jit_precompile(const KernelEntry& want);  // NVRTC -> disk cache only (no device)
int jit_count();

// Error helpers (tsm_api.cu): record a thread-local detail string.
tsm_status fail(tsm_status s, const std::string& why);

// Launch paths (tsm_api.cu).  allow_k0: the sharded layer may pass K = 0.
// lda, ldb: row strides in elements (0 = dense: M, N); strided views need a TMA kernel.
struct PeerArgs;  // tsm_kernels.cuh (NEXT N3: fused cross-GPU reduction)
tsm_status launch_tsmttsm(const tsm_plan_s* p, int dt, long long K, const void* A, const void* B,
                          void* C, void* ws, size_t ws_bytes, void* stream, bool allow_k0,
                          long long lda = 0, long long ldb = 0, const PeerArgs* peer = nullptr);
// TSMM output mode (NEXT N1): B = alpha A C (reduce = 0) or B += alpha A C (reduce = 1).
struct TsmmMode {
  double alpha_re = 1.0, alpha_im = 0.0;
  int reduce = 0;
};
tsm_status launch_tsmm(const tsm_plan_s* p, int dt, long long K, const void* A, const void* C,
                       void* B, void* stream, bool allow_k0, const TsmmMode* mode = nullptr,
                       long long lda = 0, long long ldb = 0);
// B <- alpha A C + beta B (tsmm_update_*): beta in {0, 1} in one pass, else B *= beta first.
tsm_status launch_tsmm_update(const tsm_plan_s* p, int dt, long long K, double ar, double ai,
                              const void* A, const void* C, double br, double bi, void* B,
                              void* stream, bool allow_k0);
size_t workspace_bytes(const tsm_plan_s* p, long long K);
int plan_device(const tsm_plan_s* p);
int plan_cells(const tsm_plan_s* p);  // doubles in C
int plan_op(const tsm_plan_s* p);
int plan_dt(const tsm_plan_s* p);
int plan_M(const tsm_plan_s* p);
int plan_N(const tsm_plan_s* p);

// Fixed rank-order sum of nranks gathered partial C's (tsm_comm.cu).
tsm_status rank_sum(const double* gathered, double* C, int nranks, int cells, void* stream);

}  // namespace tsm

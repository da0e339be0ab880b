// tsm_registry.cpp -- lookup over the generated AOT instantiation tables and
// the per-shape default launch parameters (JIT path).
#include "tsm_internal.h"
#include "tsm_registry.h"

namespace tsm {
extern const KernelTable g_gen_tables[];
extern const int g_gen_ntables;
extern const char* g_gen_info;
extern const KernelEntry g_param_table[];
extern const KernelEntry g_param_table_strided[];
extern const KernelEntry g_param_table_gather[];

const KernelEntry* find_aot(int op, int dt, int M, int N) {
  for (int t = 0; t < g_gen_ntables; t++)
    for (int i = 0; i < g_gen_tables[t].count; i++) {
      const KernelEntry& e = g_gen_tables[t].entries[i];
      if (e.op == op && e.dt == dt && e.M == M && e.N == N) return &e;
    }
  return nullptr;
}

const KernelEntry* find_aot_config(const KernelEntry& want) {
  const KernelEntry* e = find_aot(want.op, want.dt, want.M, want.N);
  if (e && e->NT == want.NT && e->R == want.R && e->p0 == want.p0 && e->p1 == want.p1 &&
      e->p2 == want.p2 && e->p3 == want.p3 && e->impl == want.impl &&
      (e->edge & ~64) == (want.edge & ~64))  // bit 6 (warp order) is a launch argument
    return e;
  return nullptr;
}

const KernelEntry* default_params(int op, int dt, int M, int N) {
  if (op < 0 || op > 1 || dt < 0 || dt > 1 || M < 1 || M > 64 || N < 1 || N > 64) return nullptr;
  return &g_param_table[((op * 2 + dt) * 64 + (M - 1)) * 64 + (N - 1)];
}

const KernelEntry* default_params_strided(int op, int dt, int M, int N) {
  if (op < 0 || op > 1 || dt < 0 || dt > 1 || M < 1 || M > 64 || N < 1 || N > 64) return nullptr;
  const KernelEntry* e = &g_param_table_strided[((op * 2 + dt) * 64 + (M - 1)) * 64 + (N - 1)];
  return e->impl < 0 ? nullptr : e;
}

const KernelEntry* default_params_gather(int op, int dt, int M, int N) {
  if (op < 0 || op > 1 || dt < 0 || dt > 1 || M < 1 || M > 64 || N < 1 || N > 64) return nullptr;
  const KernelEntry* e = &g_param_table_gather[((op * 2 + dt) * 64 + (M - 1)) * 64 + (N - 1)];
  return e->impl < 0 ? nullptr : e;
}

const char* build_info_json() { return g_gen_info; }
}  // namespace tsm

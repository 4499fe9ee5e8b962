// common.cuh — shared host helpers for the C ABI: error reporting, argument
// validation, workspace layout, launch accounting.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <utility>

#include "../../include/moe.h"

namespace moe {

// ---- programmatic dependent launch (PDL) ----
// With MOE_PDL=1 every kernel of the library is launched with programmatic
// stream serialisation: kernel N+1's CTAs may be scheduled while kernel N
// drains. Each kernel triggers its dependents at entry and executes
// griddepcontrol.wait before it touches global memory a previous kernel wrote;
// without the launch attribute (default) both instructions are no-ops.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif
bool pdl_enabled();
// MOE_CARVEOUT=1 (experiment): every kernel of the library prefers the maximum
// shared-memory carveout, so consecutive kernels never re-partition L1 / shared
// memory between launches. Measured: the GEMMs unchanged, the permutation
// kernels slower (less L1), so off by default. Set once per kernel and device.
void prefer_max_smem(const void* kern);

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  prefer_max_smem(reinterpret_cast<const void*>(kern));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Raise a kernel's dynamic shared-memory limit once per device (the attribute
// is per device: a process driving several GPUs must set it on each). `mask`
// is a per-call-site static holding one bit per device id; the value set is
// the maximum ever requested at that site.
template <typename K>
cudaError_t set_smem_attr_once(K* kern, int bytes, unsigned long long& mask, int& set_bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if ((mask & bit) && bytes <= set_bytes) return cudaSuccess;
  if (bytes > set_bytes) {
    set_bytes = bytes;
    mask = 0;  // a larger request re-applies on every device
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, set_bytes);
  if (e == cudaSuccess) mask |= bit;
  return e;
}

moe_status set_error(moe_status st, const char* fmt, ...);
void clear_error();
void count_launch(int n = 1);
void reset_launch_count();

#define MOE_CHECK_ARG(cond, ...)                              \
  do {                                                        \
    if (!(cond)) return ::moe::set_error(MOE_EINVAL, __VA_ARGS__); \
  } while (0)

#define MOE_CHECK_LAUNCH(name)                                                         \
  do {                                                                                 \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess)                                                             \
      return ::moe::set_error(MOE_ECUDA, "%s: %s", name, cudaGetErrorString(_e));      \
    ::moe::count_launch();                                                             \
  } while (0)

// Launch through launch_k and account for it (errors -> MOE_ECUDA).
#define MOE_LAUNCH(name, ...)                                                         \
  do {                                                                                 \
    cudaError_t _le = ::moe::launch_k(__VA_ARGS__);                                    \
    if (_le == cudaSuccess) _le = cudaGetLastError();                                  \
    if (_le != cudaSuccess)                                                            \
      return ::moe::set_error(MOE_ECUDA, "%s: %s", name, cudaGetErrorString(_le));     \
    ::moe::count_launch();                                                             \
  } while (0)

#define MOE_TRY(expr)                  \
  do {                                 \
    moe_status _s = (expr);            \
    if (_s != MOE_OK) return _s;       \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Host-side config validation for the GPU path.
moe_status check_config_gpu(const moe_config* cfg);
moe_status check_topo(const moe_topology_t* t);

// Workspace layout (byte offsets inside the caller's ws buffer).
struct WsLayout {
  size_t topo_chunk_counts;  // int32 [n_chunks][E]
  size_t router_hist;        // int32 [ceil(T/128)][E]: per-router-tile expert histograms (tensor-core router)
  size_t topo_end;
  // backward scratch
  size_t dy_g;      // bf16 [max_rows, h]
  size_t dh;        // bf16 [max_nnz, bs, bs]
  size_t dx_g;      // bf16 [max_rows, h]
  size_t dgates;    // f32 [T, k]
  size_t dlogits;   // f32 [T, E]
  size_t dwr_part;  // f32 [n_parts, h, E]
  size_t aux;       // f32 [1 + E] {aux loss, per-expert gradient coefficients} + partials
  size_t total;
};
constexpr int kTopoChunk = 1024;  // assignments per topology CTA
constexpr int kAuxParts = 148;    // fixed token partition of the auxiliary-loss reduction
int router_bwd_parts(const moe_config* cfg);
bool router_on_tensor_cores(const moe_config* cfg);
WsLayout ws_layout(const moe_config* cfg);
// moe_topology from per-row expert histograms hist [n_rows][E] of consecutive
// row_chunk-assignment ranges (the tensor-core router's per-tile histograms):
// one launch (topo_scan_emit) instead of topo_hist + topo_scan_emit.
moe_status topology_from_hist(const moe_config* cfg, const int32_t* expert_idx, const int32_t* hist, int n_rows,
                              int row_chunk, const moe_topology_t* topo, cudaStream_t s);

}  // namespace moe

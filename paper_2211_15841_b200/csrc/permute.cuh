// permute.cuh — internal entry points of permute.cu used by the layer.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/moe.h"

namespace moe {
// Per-token scatter backward: dy_rows[map[i]] = g_i * dy[t], dgates[i] =
// <y_rows[map[i]], dy[t]>; with logits != NULL also the router's dlogits
// (E <= 256), written as bf16 (tensor-core router backward) or fp32.
// pad_topo != NULL zeroes the pad rows of dy_rows.
moe_status scatter_bwd_fused(const moe_config* cfg, const void* dy, const void* y_rows, const int32_t* map,
                             const float* gates, void* dy_rows, float* dgates, const float* logits,
                             const int32_t* expert_idx, __nv_bfloat16* dlogits_bf16, float* dlogits_f32,
                             const moe_topology_t* pad_topo, cudaStream_t s, const float* aux_c = nullptr);
}  // namespace moe

// Executor glue between MoE layers (not part of the MoE hot path): the
// residual stream update of the previous layer and the pre-MoE RMSNorm of
// the next one in one pass over the rows,
//     h[t] += delta[t]            (when delta != nullptr; bf16 result)
//     xn[t] = h[t] * rsqrt(mean(h[t]^2) + eps)
// Qwen3 applies RMSNorm (`post_attention_layernorm`) before every sparse MoE
// block (HF transformers 5.5 modeling_qwen3_moe.py, Qwen3MoeDecoderLayer);
// the learned gain is 1 here (random-init model). One warp per row,
// 16-byte vectors, fp32 sum of squares.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include "ptx.cuh"

namespace lp {

constexpr int kNormWarps = 8;

__global__ void __launch_bounds__(32 * kNormWarps)
    k_add_rmsnorm(__nv_bfloat16* __restrict__ h, const __nv_bfloat16* __restrict__ delta,
                  __nv_bfloat16* __restrict__ xn, int T, int H, float eps) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x * kNormWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  uint4* hr = reinterpret_cast<uint4*>(h + static_cast<size_t>(t) * H);
  const uint4* dr = delta ? reinterpret_cast<const uint4*>(delta + static_cast<size_t>(t) * H) : nullptr;
  uint4* xr = reinterpret_cast<uint4*>(xn + static_cast<size_t>(t) * H);
  const int nv = H / 8;
  float ss = 0.f;
  for (int v = lane; v < nv; v += 32) {
    uint4 a = hr[v];
    if (dr) {
      const uint4 d = dr[v];
      __nv_bfloat162* a2 = reinterpret_cast<__nv_bfloat162*>(&a);
      const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&d);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 fa = __bfloat1622float2(a2[q]), fd = __bfloat1622float2(d2[q]);
        a2[q] = __floats2bfloat162_rn(fa.x + fd.x, fa.y + fd.y);
      }
      hr[v] = a;
    }
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(a2[q]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float r = rsqrtf(ss / static_cast<float>(H) + eps);
  for (int v = lane; v < nv; v += 32) {
    const uint4 a = hr[v];
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(a2[q]);
      o2[q] = __floats2bfloat162_rn(f.x * r, f.y * r);
    }
    xr[v] = o;
  }
}

}  // namespace lp

// K1: router logits (tcgen05) + softmax/top-k gating (warp shuffles).
//
// Semantics follow HF transformers 5.5 `Qwen3MoeTopKRouter.forward`
// (modeling_qwen3_moe.py:260-270): logits = x . Wr^T accumulated in fp32,
// softmax over all E experts in fp32, top-k, optional renormalisation of the
// k selected probabilities (`norm_topk_prob`). Tie-break is fixed as
// (probability desc, expert index asc) on both the GPU and the oracle.
//
// The logits GEMM is swap-AB like the expert kernel: M = 128 expert rows of Wr,
// N = RN tokens, split along H into `ksplit` slices so small token counts still
// fill the machine; partial sums are reduced in a fixed order by the top-k
// kernel, so the result is deterministic run to run.
#pragma once
#include <cuda_bf16.h>
#include "ptx.cuh"

namespace lp {

constexpr int kRouterN = 64;       // tokens per router tile
constexpr int kRouterStages = 4;
constexpr int kRouterThreads = 192;
constexpr int kRouterSmem = 1024 + kRouterStages * (16384 + kRouterN * 128) + 256;

struct RouterParams {
  int T, H, E;
  int ksplit;     // number of H slices
  int kb_split;   // 64-wide K blocks per slice
  int mtiles;     // ceil(E / 128)
  float* partial; // [ksplit, T, E]
};

__global__ void __launch_bounds__(kRouterThreads, 1)
    k_router_logits(const __grid_constant__ CUtensorMap tm_wr, const __grid_constant__ CUtensorMap tm_x,
                    const RouterParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStage = 16384 + kRouterN * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRouterStages * kStage);
  uint64_t* empty = full + kRouterStages;
  uint64_t* tfull = empty + kRouterStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = warp_idx();
  const int lane = threadIdx.x & 31;
  const int split = blockIdx.x % p.ksplit;
  const int mt = (blockIdx.x / p.ksplit) % p.mtiles;
  const int nt = blockIdx.x / (p.ksplit * p.mtiles);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRouterStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kRouterN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int kb0 = split * p.kb_split;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      for (int i = 0; i < p.kb_split; ++i) {
        const int s = i % kRouterStages;
        mbar_wait(&empty[s], ((i / kRouterStages) & 1) ^ 1);
        uint8_t* sa = smem + s * kStage;
        mbar_arrive_expect_tx(&full[s], kStage);
        tma_load_2d(sa, &tm_wr, &full[s], (kb0 + i) * 64, mt * 128, pol);
        tma_load_2d(sa + 16384, &tm_x, &full[s], (kb0 + i) * 64, nt * kRouterN, pol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, kRouterN);
      for (int i = 0; i < p.kb_split; ++i) {
        const int s = i % kRouterStages;
        mbar_wait(&full[s], (i / kRouterStages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * kStage);
        const uint64_t a = sdesc_kmajor_sw128(sa);
        const uint64_t b = sdesc_kmajor_sw128(sa + 16384);
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_bf16(tmem_base, a + 2 * k, b + 2 * k, idesc, (i | k) != 0);
        mma_commit(&empty[s]);
      }
      mma_commit(tfull);
    }
  } else {
    const int q = warp & 3;
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int e = mt * 128 + 32 * q + lane;
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
#pragma unroll 1
    for (int c = 0; c < kRouterN / 16; ++c) {
      uint32_t v[16];
      tmem_ld16(taddr + c * 16, v);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int t = nt * kRouterN + c * 16 + i;
        if (t < p.T && e < p.E)
          p.partial[(static_cast<size_t>(split) * p.T + t) * p.E + e] = __uint_as_float(v[i]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kRouterN);
  }
}

// One warp per token. Lane l owns experts l, l+32, ... (EPL of them).
template <int EPL>
__global__ void __launch_bounds__(256) k_topk(const float* __restrict__ partial, int T, int E, int ksplit,
                                              int topk, int renorm, int32_t* __restrict__ ids,
                                              float* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (t >= T) return;
  float l[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = lane + 32 * j;
    float acc = 0.f;
    if (e < E) {
      for (int s = 0; s < ksplit; ++s) acc += partial[(static_cast<size_t>(s) * T + t) * E + e];
    }
    l[j] = (e < E) ? acc : -INFINITY;
  }
  // softmax statistics over all E (fp32, like softmax(dtype=float))
  float m = -INFINITY;
#pragma unroll
  for (int j = 0; j < EPL; ++j) m = fmaxf(m, l[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float ssum = 0.f;
#pragma unroll
  for (int j = 0; j < EPL; ++j) ssum += (l[j] == -INFINITY) ? 0.f : expf(l[j] - m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);

  bool taken[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) taken[j] = false;
  float psel = 0.f, psum = 0.f;
  int my_id = 0;
  for (int r = 0; r < topk; ++r) {
    // local best (value desc, index asc)
    float bv = -INFINITY;
    int bi = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = lane + 32 * j;
      if (!taken[j] && e < E && (l[j] > bv || (l[j] == bv && e < bi))) { bv = l[j]; bi = e; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (lane + 32 * j == bi) taken[j] = true;
    const float pr = expf(bv - m) / ssum;
    psum += pr;
    if (lane == r) { psel = pr; my_id = bi; }
  }
  if (lane < topk) {
    ids[static_cast<size_t>(t) * topk + lane] = my_id;
    w[static_cast<size_t>(t) * topk + lane] = renorm ? psel / psum : psel;
  }
}

}  // namespace lp

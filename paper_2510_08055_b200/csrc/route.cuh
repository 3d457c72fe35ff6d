// K1: router logits (tcgen05) + softmax / top-k gating + per-tile expert
// histogram, in ONE launch.
//
// Semantics follow HF transformers 5.5 `Qwen3MoeTopKRouter.forward`
// (modeling_qwen3_moe.py:260-270): logits = x . Wr^T accumulated in fp32,
// softmax over all E experts in fp32, top-k, optional renormalisation of the
// k selected probabilities (`norm_topk_prob`). Tie-break is fixed as
// (logit desc, expert index asc) on both the GPU and the oracle.
//
// Tiling: M = 128 expert rows of Wr (E <= 256 -> up to 2 m-tiles), N = 32
// tokens per tile, K = H split into `ksplit` equal slices so small batches
// still spread over the SMs. Every (tile, m-tile, split) CTA stores its fp32
// partial logits; the LAST CTA to arrive for a token tile (global ticket,
// self-resetting) sums the partials in fixed split order — deterministic run
// to run — and then, with its four epilogue warps:
//   * softmax + top-k per token (warp shuffles), writes ids / weights;
//   * stable per-tile expert histogram + in-tile ranks of the routing entries
//     (match_any within a warp, exclusive scan across the 4 warps), which the
//     permutation (permute.cuh) turns into expert-contiguous slots.
#pragma once
#include <cuda_bf16.h>
#include "ptx.cuh"

namespace lp {

constexpr int kRouterN = 32;        // tokens per router tile (= permutation chunk)
constexpr int kRouterStages = 4;
constexpr int kRouterThreads = 192; // w0 TMA, w1 MMA + TMEM, w2..w5 epilogue
constexpr int kRouterMaxSplit = 8;
constexpr int kRouterStage = 16384 + kRouterN * 128;
constexpr int kRouterSmem = 1024 + kRouterStages * kRouterStage + 256;

struct RouterParams {
  int T, H, E, topk, renorm;
  int ksplit;        // number of H slices
  int kb_split;      // 64-wide K blocks per slice
  int mtiles;        // ceil(E / 128)
  float* partial;    // [ksplit * mtiles, T, E_pad] (unused when ksplit*mtiles == 1)
  uint32_t* ticket;  // [ntiles], zero between calls (self-resetting)
  int32_t* ids;      // [T, topk]
  float* w;          // [T, topk]
  int32_t* tile_hist;   // [ntiles, E] per-tile expert counts
  int32_t* rank_local;  // [T*topk] rank of the entry among same-expert entries of its tile
};

__global__ void __launch_bounds__(kRouterThreads, 1)
    k_router(const __grid_constant__ CUtensorMap tm_wr, const __grid_constant__ CUtensorMap tm_x,
             const RouterParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRouterStages * kRouterStage);
  uint64_t* empty = full + kRouterStages;
  uint64_t* tfull = empty + kRouterStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = warp_idx();
  const int lane = threadIdx.x & 31;
  const int arrivals = p.ksplit * p.mtiles;
  const int split = blockIdx.x % p.ksplit;
  const int mt = (blockIdx.x / p.ksplit) % p.mtiles;
  const int nt = blockIdx.x / arrivals;
  const int t0 = nt * kRouterN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRouterStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 32);
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
        uint8_t* sa = smem + s * kRouterStage;
        mbar_arrive_expect_tx(&full[s], kRouterStage);
        tma_load_2d(sa, &tm_wr, &full[s], (kb0 + i) * 64, mt * 128, pol);
        tma_load_2d(sa + 16384, &tm_x, &full[s], (kb0 + i) * 64, t0, pol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, kRouterN);
      for (int i = 0; i < p.kb_split; ++i) {
        const int s = i % kRouterStages;
        mbar_wait(&full[s], (i / kRouterStages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * kRouterStage);
        const uint64_t a = sdesc_kmajor_sw128(sa);
        const uint64_t b = sdesc_kmajor_sw128(sa + 16384);
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_bf16(tmem_base, a + 2 * k, b + 2 * k, idesc, (i | k) != 0);
        mma_commit(&empty[s]);
      }
      mma_commit(tfull);
    }
  } else {
    // ========================= epilogue: 4 warps, 128 threads =========================
    const int q = warp & 3;
    const int et = threadIdx.x - 64;  // 0..127
    const int e_pad = (p.E + 31) & ~31;
    float* s_logit = reinterpret_cast<float*>(smem);  // [kRouterN][e_pad], pipeline smem is free now
    int32_t* s_ids = reinterpret_cast<int32_t*>(s_logit + kRouterN * 256);  // [kRouterN][topk]
    int32_t* s_wh = s_ids + kRouterN * 32;                                 // [4][e_pad] warp histograms
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int e = mt * 128 + 32 * q + lane;
    uint32_t v[32];
    {
      uint32_t a[16], b[16];
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
      tmem_ld16(taddr, a);
      tmem_ld16(taddr + 16, b);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) { v[i] = a[i]; v[16 + i] = b[i]; }
    }
    bool last = true;
    if (arrivals > 1) {
      // partial rows are padded to e_pad so the reduction can use float4 loads
      const int slice = split * p.mtiles + mt;
      float* dst = p.partial + (static_cast<size_t>(slice) * p.T) * e_pad;
#pragma unroll
      for (int i = 0; i < kRouterN; ++i) {
        const int t = t0 + i;
        if (t < p.T && e < e_pad) dst[static_cast<size_t>(t) * e_pad + e] = __uint_as_float(v[i]);
      }
      __threadfence();
      named_bar_sync(1, 128);
      if (et == 0) {
        const uint32_t old = atomicAdd(&p.ticket[nt], 1u);
        *s_flag = (old == static_cast<uint32_t>(arrivals - 1));
      }
      named_bar_sync(1, 128);
      last = *s_flag != 0;
      if (last) {
        __threadfence();
        if (et == 0) p.ticket[nt] = 0u;  // ready for the next call
        // Fixed-order reduction of the slices into s_logit[t][e]. Warp q owns
        // tokens q*8..q*8+7, lane owns 4 consecutive experts (float4); all
        // slices of two tokens are loaded before any is summed.
        const int nslices = arrivals;
        for (int eb = 4 * lane; eb < e_pad; eb += 128) {
          const int emt = eb >> 7;
#pragma unroll 1
          for (int i = q * 8; i < q * 8 + 8; i += 2) {
            float4 part[2][kRouterMaxSplit];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int t = min(t0 + i + u, p.T - 1);
#pragma unroll
              for (int sp = 0; sp < kRouterMaxSplit; ++sp) {
                if (sp < p.ksplit) {
                  const int sl = sp * p.mtiles + emt;
                  part[u][sp] = __ldcg(reinterpret_cast<const float4*>(
                      p.partial + (static_cast<size_t>(sl) * p.T + t) * e_pad + eb));
                } else {
                  part[u][sp] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
              }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int sp = 0; sp < kRouterMaxSplit; ++sp) {
                if (sp < p.ksplit) {
                  acc.x += part[u][sp].x; acc.y += part[u][sp].y;
                  acc.z += part[u][sp].z; acc.w += part[u][sp].w;
                }
              }
              *reinterpret_cast<float4*>(s_logit + (i + u) * e_pad + eb) = acc;
            }
          }
        }
        (void)nslices;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kRouterN; ++i) s_logit[i * e_pad + e] = __uint_as_float(v[i]);
    }
    named_bar_sync(1, 128);
    if (last) {
      // ---------------- softmax + top-k: warp q owns tokens q*8 .. q*8+7 ----------------
      const int epl = e_pad / 32;
      for (int i = q * 8; i < q * 8 + 8; ++i) {
        const int t = t0 + i;
        if (t >= p.T) break;
        float l[8];
        float m = -INFINITY;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int ex = lane + 32 * j;
          l[j] = (j < epl && ex < p.E) ? s_logit[i * e_pad + ex] : -INFINITY;
          m = fmaxf(m, l[j]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float ssum = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) ssum += (l[j] == -INFINITY) ? 0.f : expf(l[j] - m);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
        float psel = 0.f, psum = 0.f;
        int my_id = 0;
        for (int r = 0; r < p.topk; ++r) {
          float bv = -INFINITY;
          int bi = 0x7fffffff, bj = -1;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int ex = lane + 32 * j;
            if (l[j] > bv || (l[j] == bv && l[j] != -INFINITY && ex < bi)) { bv = l[j]; bi = ex; bj = j; }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (lane + 32 * j == bi) l[j] = -INFINITY;
          (void)bj;
          const float pr = expf(bv - m) / ssum;
          psum += pr;
          if (lane == r) { psel = pr; my_id = bi; }
        }
        if (lane < p.topk) {
          p.ids[static_cast<size_t>(t) * p.topk + lane] = my_id;
          p.w[static_cast<size_t>(t) * p.topk + lane] = p.renorm ? psel / psum : psel;
          s_ids[i * p.topk + lane] = my_id;
        }
      }
      // ---------------- stable per-tile histogram + ranks ----------------
      for (int ee = lane; ee < e_pad; ee += 32) s_wh[q * e_pad + ee] = 0;
      __syncwarp();
      const int tok_lo = min(q * 8, max(p.T - t0, 0));
      const int tok_hi = min(q * 8 + 8, p.T - t0);
      const int n_ent = max(tok_hi - tok_lo, 0) * p.topk;
      const unsigned lt = (1u << lane) - 1u;
      int my_rank[8];  // ranks for this lane's entries (<= 8 steps since 8 tokens * topk <= 256)
      int my_e[8];
      for (int st = 0; st < 8; ++st) {
        const int k0 = st * 32;
        my_e[st] = -1;
        my_rank[st] = 0;
        if (k0 >= n_ent) continue;
        const int idx = k0 + lane;
        const int ex = (idx < n_ent) ? s_ids[tok_lo * p.topk + idx] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, ex);
        int base = 0;
        if (ex >= 0) base = s_wh[q * e_pad + ex];
        __syncwarp();
        if (ex >= 0) {
          my_rank[st] = base + __popc(peers & lt);
          my_e[st] = ex;
          if ((__ffs(peers) - 1) == lane) s_wh[q * e_pad + ex] = base + __popc(peers);
        }
        __syncwarp();
      }
      named_bar_sync(1, 128);
      // exclusive scan over the 4 warps per expert; tile totals to global
      for (int ee = et; ee < e_pad; ee += 128) {
        int run = 0;
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) {
          const int c = s_wh[w4 * e_pad + ee];
          s_wh[w4 * e_pad + ee] = run;
          run += c;
        }
        if (ee < p.E) p.tile_hist[static_cast<size_t>(nt) * p.E + ee] = run;
      }
      named_bar_sync(1, 128);
      for (int st = 0; st < 8; ++st) {
        const int idx = st * 32 + lane;
        if (my_e[st] >= 0)
          p.rank_local[static_cast<size_t>(t0 + tok_lo) * p.topk + idx] = my_rank[st] + s_wh[q * e_pad + my_e[st]];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 32);
  }
}

}  // namespace lp

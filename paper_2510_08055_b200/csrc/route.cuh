// K1: router logits (tcgen05) + softmax / top-k gating + per-tile expert
// histogram, in ONE launch.
//
// Semantics follow HF transformers 5.5 `Qwen3MoeTopKRouter.forward`
// (modeling_qwen3_moe.py:260-270): logits = x . Wr^T accumulated in fp32,
// softmax over all E experts in fp32, top-k, optional renormalisation of the
// k selected probabilities (`norm_topk_prob`). Tie-break is fixed as
// (logit desc, expert index asc) on both the GPU and the oracle.
//
// Tiling (swap-AB): M = 128 expert rows of Wr per m-tile (E <= 256 -> up to
// two m-tiles accumulated side by side in TMEM), N = 16 tokens per tile.
// Small batches are latency-bound on streaming Wr (0.5 MB for Qwen, L2
// resident), so each token tile is owned by a thread-block CLUSTER of `csize`
// CTAs that split K = H: every CTA streams 1/csize of Wr through a 6-deep TMA
// ring and parks its fp32 partial logits in its own smem. CTA r of the
// cluster then owns tokens [r*16/csize, (r+1)*16/csize) of the tile: it sums
// those rows of every CTA's partials over DSMEM in fixed rank order
// (deterministic, no global round trip) and its 4 epilogue warps run
//   * softmax + top-k with 8*csize lanes per token (all tokens concurrently);
//   * the stable expert histogram of its tokens + ranks of the routing
//     entries (match_any within a warp, exclusive scans across the 4 warps and
//     across the cluster's CTAs over DSMEM), so each 16-token tile gets one
//     histogram that the permutation (permute.cuh) turns into slots.
#pragma once
#include <cuda_bf16.h>
#include "ptx.cuh"

namespace lp {

constexpr int kRouterN = 16;         // tokens per router tile for small batches (= permutation chunk)
constexpr int kRouterStages = 6;
// w0 TMA, w1 MMA + TMEM, w2..w5 TMEM drain + histogram, w2.. top-k. Large
// tiles gate 64 tokens per CTA: the latency-bound top-k gets 10 warps.
__host__ __device__ constexpr int router_threads(int TN) { return TN >= 64 ? 384 : 192; }
constexpr int kRouterTileLarge = 64;  // tokens per tile for large batches (fewer Wr re-reads)

struct RouterParams {
  int T, H, E, topk, renorm;
  int mtiles;           // ceil(E / 128)
  int32_t* ids;         // [T, topk]
  float* w;             // [T, topk]
  int32_t* tile_hist;   // [ntiles, E] per-tile expert counts (tile = TN tokens)
  int32_t* rank_local;  // [T*topk] rank of the entry among same-expert entries of its tile
  // ---- fused permutation (FUSED instantiation only; every CTA co-resident) ----
  int ntiles, max_n;
  int32_t* counts;        // [E]
  int32_t* offsets;       // [E+1]
  int32_t* slot_of;       // [T*topk]
  int32_t* tok_of;        // [T*topk]
  const __nv_bfloat16* x; // [T, H] token rows
  __nv_bfloat16* x_perm;  // [T*topk, H] (nullptr: slot maps only)
  int32_t* tile_prefix;   // [E+1] expert token-tile schedule for k_experts
  int32_t* tile_rows;     // [E]
  uint32_t* sched;        // [E+1] expert scheduler words, reset here
  uint32_t* gbar;         // [2] grid barrier (arrive, depart); zero on entry, left zero
  // ---- L2 warm-up of the expert kernel's first weights (forward path only) ----
  const uint8_t* warm;    // start of the W13 range the expert kernel streams first
  size_t warm_bytes;      // bytes to prefetch into L2, split across the router grid
};

// Grid-wide barrier for a co-resident grid (<= 1 CTA per SM, checked by the
// host). Release: __syncthreads + thread 0's gpu-scope fence before arriving;
// acquire: ld.acquire of the arrive count. The last CTA to depart resets both
// words, so the workspace header is zero again for the next call.
__device__ __forceinline__ void grid_barrier(uint32_t* gbar, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&gbar[0], 1u);
    while (ld_acquire_u32(&gbar[0]) < nblocks) __nanosleep(32);
    if (atomicAdd(&gbar[1], 1u) == nblocks - 1) {
      gbar[0] = 0u;
      gbar[1] = 0u;
    }
  }
  __syncthreads();
}

// Softmax + top-k of one token held by LPT consecutive lanes (lane `sub` owns
// experts sub, sub+LPT, ...). Writes the k ids and their unnormalised
// exp(logit - max) to smem; psum = their sum in selection order, inv = 1 / the
// full softmax denominator. With renormalisation the weights are
// exp_r / psum: independent of LPT (the lane split changes with the router's
// tile shape), so a token's weights are bit-identical for every batch size.
template <int LPT, int NV>
__device__ __forceinline__ void topk_lanes(const float* row, int E, int topk, int sub, int32_t* out_ids, float* out_p,
                                           float& psum, float& inv_out) {
  float l[NV];
  float m = -INFINITY;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int ex = sub + LPT * j;
    l[j] = (ex < E) ? row[ex] : -INFINITY;
    if (l[j] != l[j]) l[j] = -INFINITY;  // NaN logits rank last (ids stay in range)
    m = fmaxf(m, l[j]);
  }
#pragma unroll
  for (int o = 1; o < LPT; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float ssum = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) ssum += (l[j] == -INFINITY) ? 0.f : __expf(l[j] - m);
#pragma unroll
  for (int o = 1; o < LPT; o <<= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
  const float inv = 1.0f / ssum;
  inv_out = inv;
  uint32_t taken = 0;
  psum = 0.f;
  if constexpr (LPT == 32) {
    // whole warp per token: two redux.sync per selection round (max key, then min index)
    for (int r = 0; r < topk; ++r) {
      float bv = -INFINITY;
      int bj = -1;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (sub + 32 * j < E && !((taken >> j) & 1u) && (bj < 0 || l[j] > bv)) { bv = l[j]; bj = j; }
      const uint32_t bits = __float_as_uint(bv);
      const uint32_t key = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);  // order-preserving
      const uint32_t kmax = __reduce_max_sync(0xffffffffu, bj >= 0 ? key : 0u);
      const uint32_t cand = (bj >= 0 && key == kmax) ? static_cast<uint32_t>(sub + 32 * bj) : 0xffffffffu;
      const int bi = static_cast<int>(__reduce_min_sync(0xffffffffu, cand));
      if ((bi & 31) == sub) taken |= 1u << (bi >> 5);
      const uint32_t vb = (kmax & 0x80000000u) ? (kmax & 0x7fffffffu) : ~kmax;
      const float pr = __expf(__uint_as_float(vb) - m);
      psum += pr;
      if (sub == 0) { out_ids[r] = bi; out_p[r] = pr; }
    }
  } else {
    for (int r = 0; r < topk; ++r) {
      float bv = -INFINITY;
      int bj = -1;
#pragma unroll
      for (int j = 0; j < NV; ++j)  // ascending expert index: the first maximum wins ties
        if (sub + LPT * j < E && !((taken >> j) & 1u) && (bj < 0 || l[j] > bv)) { bv = l[j]; bj = j; }
      int bi = bj >= 0 ? sub + LPT * bj : 0x7fffffff;
#pragma unroll
      for (int o = 1; o < LPT; o <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi) || bi == 0x7fffffff) {
          if (oi != 0x7fffffff) { bv = ov; bi = oi; }
        }
      }
      if (bi % LPT == sub) taken |= 1u << (bi / LPT);
      const float pr = __expf(bv - m);
      psum += pr;
      if (sub == 0) { out_ids[r] = bi; out_p[r] = pr; }
    }
  }
}

// Shared-memory plan of one router CTA: the TMA ring during the K loop, then
// (aliased, once every MMA has drained it) the epilogue scratch.
__host__ __device__ constexpr int router_ring_bytes(int mtiles, int TN) {
  return kRouterStages * (mtiles * 16384 + TN * 128);
}
__host__ __device__ constexpr int router_part_floats() { return 4 * 16 * 256; }  // 64 KiB: cluster partials
__host__ __device__ constexpr int router_scratch_bytes(int TN) {
  // partials | logits [TN][256] | ids, p [TN][32] | 4 warp hists + cta + base [7][256] | ranks, experts [128][4]
  return 4 * (router_part_floats() + TN * 256 + 2 * TN * 32 + 7 * 256 + 2 * 512);
}
__host__ __device__ constexpr int router_smem_bytes(int mtiles, int TN) {
  return 1024 + (router_ring_bytes(mtiles, TN) > router_scratch_bytes(TN) ? router_ring_bytes(mtiles, TN)
                                                                           : router_scratch_bytes(TN)) +
         256;
}

// CS: cluster size (CTAs per token tile); NV: logits per lane in the top-k;
// TN: tokens per tile (MMA N, = the permutation chunk). LPT lanes gate one
// token, so the 128 epilogue threads take 128/LPT tokens per round.
template <int CS, int NV, int TN, bool FUSED>
__global__ void __launch_bounds__(router_threads(TN), 1)
    k_router(const __grid_constant__ CUtensorMap tm_wr, const __grid_constant__ CUtensorMap tm_x,
             const RouterParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = p.mtiles * 16384 + TN * 128;
  const int ring = router_ring_bytes(p.mtiles, TN);
  const int scratch = router_scratch_bytes(TN);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (ring > scratch ? ring : scratch));
  uint64_t* empty = full + kRouterStages;
  uint64_t* tfull = empty + kRouterStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = warp_idx();
  const int lane = threadIdx.x & 31;
  constexpr int kRouterGate = router_threads(TN) - 64;  // threads gating tokens
  constexpr int TPC = TN / CS;                    // tokens this CTA gates
  constexpr int LPT = (128 / TPC) > 8 ? (128 / TPC) : 8;  // lanes per token in the top-k
  constexpr int TMEM_COLS = 4 * 2 * TN <= 32 ? 32 : (4 * 2 * TN <= 128 ? 128 : (4 * 2 * TN <= 256 ? 256 : 512));
  const int cr = CS > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int tile = blockIdx.x / CS;
  const int t0 = tile * TN;
  // K = H is summed as NPART fixed partial sums (each a separate TMEM
  // accumulator, folded left in part order), whatever the cluster size: the
  // fp32 logits of a token are then bit-identical for every batch size and
  // batch composition (layered vs chunked prefill see the same per-token math).
  const int kb_total = p.H / 64;
  const int npart = (kb_total % 4 == 0) ? 4 : ((kb_total % 2 == 0) ? 2 : 1);
  const int ppc = npart / CS;               // partial sums owned by this CTA
  const int kb_part = kb_total / npart;     // k-blocks per partial sum
  const int kb_per = ppc * kb_part;
  const int kb0 = cr * kb_per;
  [[maybe_unused]] const bool tr = blockIdx.x == 0;  // trace builds only
  if (threadIdx.x == 0) { LP_TRACE_AT(tr, 0); LP_TRACE_MIN(8); }

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRouterStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    fence_mbar_init();
    prefetch_tmap(&tm_wr);
    prefetch_tmap(&tm_x);
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) LP_TRACE_AT(tr, 1);

  const int e_pad = (p.E + 31) & ~31;
  float* s_part = reinterpret_cast<float*>(smem);                 // [ppc][TN][e_pad] partial logits (CS > 1)
  float* s_logit = s_part + router_part_floats();                  // [TPC][e_pad] this CTA's token logits
  int32_t* s_ids = reinterpret_cast<int32_t*>(s_logit + TN * 256);  // [TN][32]
  float* s_p = reinterpret_cast<float*>(s_ids + TN * 32);           // [TN][32]
  int32_t* s_wh = reinterpret_cast<int32_t*>(s_p + TN * 32);        // [4][e_pad]
  int32_t* s_cta = s_wh + 4 * 256;                                 // [e_pad] this CTA's chunk totals
  int32_t* s_base = s_cta + 256;                                   // [e_pad] totals of lower ranks
  int32_t* s_rank = s_base + 256;                                  // [128][4] in-warp ranks
  int32_t* s_ent = s_rank + 512;                                   // [128][4] entry experts

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      for (int i = 0; i < kb_per; ++i) {
        const int s = i % kRouterStages;
        mbar_wait(&empty[s], ((i / kRouterStages) & 1) ^ 1);
        uint8_t* sa = smem + s * stage_bytes;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        for (int mt = 0; mt < p.mtiles; ++mt)
          tma_load_2d(sa + mt * 16384, &tm_wr, &full[s], (kb0 + i) * 64, mt * 128, pol);
        tma_load_2d(sa + p.mtiles * 16384, &tm_x, &full[s], (kb0 + i) * 64, t0, pol);
      }
      LP_TRACE_AT(tr, 3);
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, TN);
      for (int i = 0; i < kb_per; ++i) {
        const int s = i % kRouterStages;
        mbar_wait(&full[s], (i / kRouterStages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * stage_bytes);
        const uint64_t b = sdesc_kmajor_sw128(sa + p.mtiles * 16384);
        const uint32_t d0 = tmem_base + (i / kb_part) * (p.mtiles * TN);
        for (int mt = 0; mt < p.mtiles; ++mt) {
          const uint64_t a = sdesc_kmajor_sw128(sa + mt * 16384);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_bf16(d0 + mt * TN, a + 2 * k, b + 2 * k, idesc, ((i % kb_part) | k) != 0);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tfull);
    }
    __syncwarp();
  } else if (warp < 6) {
    // TMEM -> smem (the ring is drained once tfull fires: every MMA has read its stage)
    const int q = warp & 3;
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (threadIdx.x == 64) LP_TRACE_AT(tr, 4);
    if (threadIdx.x == 64 && p.warm_bytes) {
      // This CTA's HBM reads are done. The expert kernel streams every touched
      // expert's weights right after routing: pull its first items' W13 rows
      // into L2 while the rest of the routing prologue leaves HBM idle.
      const size_t per = ((p.warm_bytes + gridDim.x - 1) / gridDim.x + 65535) & ~size_t(65535);
      const size_t lo = per * blockIdx.x, hi = min(p.warm_bytes, lo + per);
      for (size_t o = lo; o < hi; o += 65536) {
        const size_t n = hi - o < 65536 ? hi - o : 65536;
        bulk_prefetch_l2(p.warm + o, static_cast<uint32_t>(n));
      }
    }
    for (int mt = 0; mt < p.mtiles; ++mt) {
      const int e = mt * 128 + 32 * q + lane;
      for (int c = 0; c < TN / 16; ++c) {
        float acc[16];
        for (int pl = 0; pl < ppc; ++pl) {
          uint32_t v[16];
          tmem_ld16(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + (pl * p.mtiles + mt) * TN + c * 16, v);
          tmem_wait_ld();
          if (CS > 1) {  // parked for the cluster-wide fold below
            if (e < e_pad) {
#pragma unroll
              for (int i = 0; i < 16; ++i) s_part[(pl * TN + c * 16 + i) * e_pad + e] = __uint_as_float(v[i]);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] = pl ? acc[i] + __uint_as_float(v[i]) : __uint_as_float(v[i]);
          }
        }
        if (CS == 1 && e < e_pad) {
#pragma unroll
          for (int i = 0; i < 16; ++i) s_logit[(c * 16 + i) * e_pad + e] = acc[i];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) LP_TRACE_AT(tr, 10);
  if (CS > 1) {
    cluster_sync();  // every CTA's partial logits are now readable over DSMEM
    if (threadIdx.x == 0) LP_TRACE_AT(tr, 11);
    if (warp >= 2) {
      // this CTA's token rows: s_logit[i][e] = fold over global part order (rank r, local part pl)
      const int et = threadIdx.x - 64;
      const int nq = TPC * (e_pad / 4);
      for (int idx = et; idx < nq; idx += kRouterGate) {
        const int off = cr * TPC * e_pad + idx * 4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < CS; ++r) {
          for (int pl = 0; pl < ppc; ++pl) {
            const float4 v = ld_dsmem_f4(mapa_shared(smem_u32(s_part + pl * TN * e_pad + off), r));
            if (r == 0 && pl == 0) {
              acc = v;
            } else {
              acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
          }
        }
        *reinterpret_cast<float4*>(s_logit + idx * 4) = acc;
      }
    }
    cluster_sync();  // partials consumed: any CTA may leave
    if (threadIdx.x == 0) LP_TRACE_AT(tr, 12);
  }
  if (warp >= 2) {
    // ---------------- softmax + top-k: LPT lanes per token, all gating warps ----------------
    const int tk = threadIdx.x - 64;  // 0..kRouterGate-1
    const int tc0 = t0 + cr * TPC;   // first token of this CTA's chunk
    named_bar_sync(1, kRouterGate);
    constexpr int TPRG = (kRouterGate / 32) * (32 / LPT);  // tokens per round (whole warps)
    for (int g0 = 0; g0 < TPC; g0 += TPRG) {
      const int g = g0 + tk / LPT;  // warp-uniform bound: TPC is a multiple of 32/LPT
      if (g < TPC) {
        const int sub = tk % LPT;
        const int t = tc0 + g;
        float psum, inv;
        topk_lanes<LPT, NV>(s_logit + g * e_pad, p.E, p.topk, sub, s_ids + g * 32, s_p + g * 32, psum, inv);
        __syncwarp();
        if (t < p.T) {
          for (int r = sub; r < p.topk; r += LPT) {
            p.ids[static_cast<size_t>(t) * p.topk + r] = s_ids[g * 32 + r];
            p.w[static_cast<size_t>(t) * p.topk + r] = p.renorm ? s_p[g * 32 + r] / psum : s_p[g * 32 + r] * inv;
          }
        }
      }
    }
    named_bar_sync(1, kRouterGate);
    if (tk == 0) LP_TRACE_AT(tr, 5);
  }
  // (tile_hist == nullptr: the permutation ranks the entries itself, k_scan_slots)
  const bool hist = FUSED || p.tile_hist != nullptr;
  if (hist && warp >= 2 && warp < 6) {
    const int q = warp & 3;
    const int et = threadIdx.x - 64;  // 0..127
    const int tc0 = t0 + cr * TPC;
    // ---------------- stable chunk histogram + ranks: warp q owns TPC/4 tokens ----------------
    constexpr int TPW = TPC / 4;
    for (int ee = lane; ee < e_pad; ee += 32) s_wh[q * e_pad + ee] = 0;
    __syncwarp();
    const int tok_lo = q * TPW;
    const int n_tok = max(0, min(TPW, p.T - tc0 - tok_lo));
    const int n_ent = n_tok * p.topk;  // <= 128 (host picks TN so that TPW * topk <= 128)
    const unsigned lt = (1u << lane) - 1u;
    int my_rank[4], my_e[4];
#pragma unroll
    for (int st = 0; st < 4; ++st) {
      my_e[st] = -1;
      my_rank[st] = 0;
      const int idx = st * 32 + lane;  // entry within this warp's tokens (token-major, then j)
      const int ex = (idx < n_ent) ? s_ids[(tok_lo + idx / p.topk) * 32 + idx % p.topk] : -1;
      if (st * 32 < n_ent) {
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
    }
    named_bar_sync(2, 128);
    // exclusive scan over this CTA's 4 warps; the CTA's total goes to s_cta[e]
    for (int ee = et; ee < e_pad; ee += 128) {
      int run = 0;
#pragma unroll
      for (int w4 = 0; w4 < 4; ++w4) {
        const int c = s_wh[w4 * e_pad + ee];
        s_wh[w4 * e_pad + ee] = run;
        run += c;
      }
      s_cta[ee] = run;
    }
    named_bar_sync(2, 128);
    if constexpr (CS == 1) {
      for (int ee = et; ee < p.E; ee += 128) p.tile_hist[static_cast<size_t>(tile) * p.E + ee] = s_cta[ee];
#pragma unroll
      for (int st = 0; st < 4; ++st) {
        if (my_e[st] >= 0)
          p.rank_local[static_cast<size_t>(tc0 + tok_lo) * p.topk + st * 32 + lane] =
              my_rank[st] + s_wh[q * e_pad + my_e[st]];
      }
    }
    // (CS > 1: cross-CTA bases are applied after the cluster barrier below)
    for (int st = 0; st < 4; ++st) { s_rank[et * 4 + st] = my_rank[st]; s_ent[et * 4 + st] = my_e[st]; }
  }
  if (CS > 1 && hist) {  // uniform across the cluster (same params)
    // tile histogram across the cluster: CTA r adds the totals of ranks < r to
    // its ranks; the last CTA writes the tile total. Fixed order -> stable slots.
    __syncthreads();
    cluster_sync();
    if (warp >= 2 && warp < 6) {
      const int q = warp & 3;
      const int et = threadIdx.x - 64;
      const int tc0 = t0 + cr * TPC;
      constexpr int TPW = TPC / 4;
      for (int ee = et; ee < e_pad; ee += 128) {
        int before = 0, total = 0;
        const uint32_t la = smem_u32(s_cta + ee);
#pragma unroll
        for (int r = 0; r < CS; ++r) {
          uint32_t v;
          asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(mapa_shared(la, r)) : "memory");
          if (r < cr) before += static_cast<int>(v);
          total += static_cast<int>(v);
        }
        s_base[ee] = before;
        if (cr == CS - 1 && ee < p.E) p.tile_hist[static_cast<size_t>(tile) * p.E + ee] = total;
      }
      named_bar_sync(2, 128);
#pragma unroll
      for (int st = 0; st < 4; ++st) {
        const int ex = s_ent[et * 4 + st];
        if (ex >= 0)
          p.rank_local[static_cast<size_t>(tc0 + q * TPW) * p.topk + st * 32 + lane] =
              s_rank[et * 4 + st] + s_wh[q * e_pad + ex] + s_base[ex];
      }
    }
    cluster_sync();  // s_cta of every CTA consumed
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 64) LP_TRACE_AT(tr, 14);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
  if constexpr (FUSED) {
    // ---------------- permutation (replaces k_scan + k_scatter) ----------------
    grid_barrier(p.gbar, gridDim.x);  // every tile histogram / rank is published
    if (threadIdx.x == 0) LP_TRACE_AT(tr, 15);
    constexpr int NT = router_threads(TN);
    // expert totals and this tile's base over all tile histograms: int4 per
    // thread (4 experts), G thread groups split the tile range, 4 rows in flight
    const int nvec = e_pad / 4;
    const int G = NT / nvec;
    int32_t* s_tot = reinterpret_cast<int32_t*>(smem);  // [G][e_pad] partial totals
    int32_t* s_bas = s_tot + G * e_pad;                  // [G][e_pad] partial tile bases
    int32_t* s_off = s_bas + G * e_pad;                  // [e_pad + 1] expert offsets
    int32_t* s_tb = s_off + 260;                         // [e_pad] this tile's base per expert
    {
      const int gi = threadIdx.x / nvec, vq = threadIdx.x % nvec;
      if (gi < G) {
        const int per = (p.ntiles + G - 1) / G;
        const int c0 = min(gi * per, p.ntiles), c1 = min(c0 + per, p.ntiles);
        int4 tot = make_int4(0, 0, 0, 0), bas = make_int4(0, 0, 0, 0);
        if (vq * 4 < p.E) {
          const int4* h4 = reinterpret_cast<const int4*>(p.tile_hist) + vq;
          const int rs = p.E / 4;  // row stride in int4 (E % 4 == 0 on this path)
          for (int c = c0; c < c1; c += 4) {
            int4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              v[u] = (c + u < c1) ? __ldcg(h4 + static_cast<size_t>(c + u) * rs) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              tot.x += v[u].x; tot.y += v[u].y; tot.z += v[u].z; tot.w += v[u].w;
              if (c + u < tile) { bas.x += v[u].x; bas.y += v[u].y; bas.z += v[u].z; bas.w += v[u].w; }
            }
          }
        }
        reinterpret_cast<int4*>(s_tot + gi * e_pad)[vq] = tot;
        reinterpret_cast<int4*>(s_bas + gi * e_pad)[vq] = bas;
      }
    }
    __syncthreads();
    if (warp == 0) {  // expert totals -> exclusive offsets (e_pad <= 256: 8 experts per lane)
      constexpr int EPL = 8;
      int v[EPL];
      int run = 0;
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int ee = lane * EPL + u;
        int tot = 0;
        if (ee < p.E)
          for (int g = 0; g < G; ++g) tot += s_tot[g * e_pad + ee];
        v[u] = tot;
        run += tot;
      }
      int inc = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      int ex = inc - run;
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int ee = lane * EPL + u;
        if (ee < p.E) s_off[ee] = ex;
        ex += v[u];
      }
      if (lane == 31) s_off[p.E] = inc;
      if (blockIdx.x == 0) {  // the expert tile schedule k_experts consumes (same as k_scan)
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          const int ee = lane * EPL + u;
          if (ee < p.E) { p.counts[ee] = v[u]; p.offsets[ee] = s_off[ee]; }
        }
        if (lane == 31) p.offsets[p.E] = inc;
        int nt[EPL], tr_run = 0;
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          nt[u] = v[u] > 0 ? (v[u] + p.max_n - 1) / p.max_n : 0;
          tr_run += nt[u];
        }
        int tinc = tr_run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, tinc, o);
          if (lane >= o) tinc += y;
        }
        int tex = tinc - tr_run;
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          const int ee = lane * EPL + u;
          if (ee < p.E) {
            p.tile_prefix[ee] = tex;
            const int rows = nt[u] ? (v[u] + nt[u] - 1) / nt[u] : 0;
            p.tile_rows[ee] = min(p.max_n, (rows + 15) & ~15);
          }
          tex += nt[u];
        }
        if (lane == 31) p.tile_prefix[p.E] = tinc;
      }
    } else if (warp == 1 && blockIdx.x == 0) {
      for (int i = lane; i <= p.E; i += 32) p.sched[i] = 0u;
    }
    for (int ee = threadIdx.x; ee < p.E; ee += NT) {
      int b = 0;
      for (int g = 0; g < G; ++g) b += s_bas[g * e_pad + ee];
      s_tb[ee] = b;
    }
    __syncthreads();
    // this CTA's routing entries: slot maps and token-row copies (one warp per entry)
    const int tc0 = t0 + cr * TPC;
    const int n_tok = max(0, min(TPC, p.T - tc0));
    const int n_ent = n_tok * p.topk;
    const size_t i0 = static_cast<size_t>(tc0) * p.topk;
    for (int k = threadIdx.x; k < n_ent; k += NT) {  // slot maps
      const int ee = s_ids[(k / p.topk) * 32 + k % p.topk];
      const int slot = s_off[ee] + s_tb[ee] + __ldcg(p.rank_local + i0 + k);
      p.slot_of[i0 + k] = slot;
      p.tok_of[slot] = tc0 + k / p.topk;
      s_ent[k] = slot;  // (free after the histogram) slot of this CTA's entry k
    }
    __syncthreads();
    if (p.x_perm != nullptr) {  // token-row copies: 2 entries per warp, a whole row per lane batch
      const int nv = p.H / 8;
      constexpr int U = 8;
      for (int k0 = 2 * warp; k0 < n_ent; k0 += 2 * (NT / 32)) {
        for (int v0 = lane; v0 < nv; v0 += 32 * U) {
          uint4 r[2][U];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = k0 + h;
            const uint4* src = reinterpret_cast<const uint4*>(p.x + static_cast<size_t>(tc0 + k / p.topk) * p.H);
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (k < n_ent && v0 + 32 * u < nv) r[h][u] = __ldg(src + v0 + 32 * u);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = k0 + h;
            if (k < n_ent) {
              uint4* dst = reinterpret_cast<uint4*>(p.x_perm + static_cast<size_t>(s_ent[k]) * p.H);
#pragma unroll
              for (int u = 0; u < U; ++u)
                if (v0 + 32 * u < nv) dst[v0 + 32 * u] = r[h][u];
            }
          }
        }
      }
    }
  }
  if (threadIdx.x == 0) { LP_TRACE_AT(tr, 6); LP_TRACE_MAX(9); }
}

}  // namespace lp

// Decode-size MoE layer in ONE launch: router + top-k + permutation + grouped
// expert FFN (K1 + K2 + K3) for T <= 16 tokens with T*topk <= E <= 128 — the
// decode-only layers of a layered-prefill iteration.
//
// Why: at T = 1 the separate launches spent ~12 us routing before any expert
// weight streamed (router 7 us, scan+slots 2 us, launch gaps), against ~12 us
// of weight streaming at the HBM roofline (8 experts x 9.4 MB). Here:
//
//  * Routing is computed redundantly by every CTA pair (cluster of 2, always
//    co-resident, so all 148 SMs stream afterwards): CTA r of the pair
//    computes the router's fixed partial sums 2r and 2r+1 of K = H (each
//    k-blocks [p*H/256, (p+1)*H/256)) with exactly the router's tcgen05 MMA
//    chain (M = 128 expert rows of Wr, N = 16 tokens, SWIZZLE_128B, same K
//    order, one TMEM accumulator per partial), the partials are folded over
//    DSMEM in part order (p0 + p1 + p2 + p3, as k_router<4, 4, 16> folds its
//    four CTAs' partials) and every CTA runs the router's own
//    topk_lanes<32, 4> on the folded fp32 logits: ids, weights and logits are
//    bit-identical to k_router at this T, with no inter-cluster dependency.
//    Wr k-blocks are requested before griddepcontrol.wait (weights do not
//    depend on the predecessor), the token rows after it.
//  * Every CTA derives the stable permutation (slot = offsets[e] + #{j < i :
//    ids[j] = e}, match_any within a warp + per-warp prefix) and the work-item
//    list in shared memory; CTA 0 publishes ids, w, counts, offsets, slot_of
//    and tok_of for k_combine and the caller.
//  * The expert stream is k_experts_tiny's (identical MMAs and epilogue, so a
//    token's rows are bit-identical to the other expert kernels): UP items of
//    64 act features (64 gate + 64 up rows, one 128-row tile, K = H), DN items
//    of 128 W2 rows (K = I), items claimed dynamically (deadlock-free without
//    co-residency: all UP items precede all DN items). NEW: a DN item's W2
//    tiles are requested into the ring BEFORE its UP dependency resolves (the
//    act rows follow once it does), and when the hit experts' W2 is small
//    (<= kW2WarmBytes) it is bulk-prefetched into L2 while the UP items
//    stream, so the DN phase no longer starts from HBM.
//  * Scheduler words are left zero: the last CTA to finish resets them.
//
// Warp roles (256 threads): w0 TMA producer + scheduler (lane 1: W2 L2
// prefetch), w1 MMA issuer, w2 TMEM allocator, w2-w3 token-row gather,
// w4-w7 TMEM drain / epilogue; all 8 warps fold, gate and permute.
#pragma once
#include <cuda_bf16.h>
#include "experts_sm100.cuh"
#include "ptx.cuh"
#include "route.cuh"

namespace lp {

struct DecodeCfg {
  static constexpr int kThreads = 256;
  static constexpr int kParts = 4;     // the router's fixed K partial sums
  static constexpr int kMaxPpc = 2;    // partials per CTA at the smallest cluster (2)
  static constexpr int kN = 16;        // token rows per item (MMA N) = the router tile
  static constexpr int kMaxT = 16;
  static constexpr int kMaxE = 128;    // one router m-tile
  static constexpr int kBBytes = kN * 128;
  static constexpr int kAcc = 2;
  static constexpr int kTmemCols = 32;
  static constexpr int kXBytes = 64 * kN * 4;                // up values handed to the gate warps
  static constexpr int kPartBytes = kMaxPpc * kMaxT * kMaxE * 4;  // this CTA's partial logits (read over DSMEM)
  static constexpr int kLogitBytes = kMaxT * kMaxE * 4;      // folded logits
  static constexpr int kTopBytes = 2 * kMaxT * 32 * 4;       // selected ids / probabilities
  // off[E+1] cnt[E] hit[E] tok[S] ent[S] slot[S] + per-warp counts [4][E] + 16 scalars
  // ... + routing weights w[S] + the fused combine's finished-token lists [2][kMaxT + 1] (+ padding)
  static constexpr int kPermBytes = 4 * ((kMaxE + 1) + 5 * kMaxE + 4 * kMaxE + 19 + kMaxE + 40);  // 16-B multiple
  static constexpr int kExitWord = 1 + kMaxExperts + 8;  // sched word counting finished CTAs
  static constexpr int kUpDoneWord = 1 + kMaxExperts + 4;  // UP items finished (all experts)
};
static_assert(DecodeCfg::kPermBytes % 16 == 0, "barrier / ring alignment");

// The weight ring: KS k-blocks (64-wide K slices) per stage, laid out [A_0 .. A_{KS-1} | B_0 .. B_{KS-1}]
// (16 KiB weight tile + 2 KiB token rows per k-block, every tile 1024-B aligned). A decode item's
// stream is paced per STAGE (each one waits for its TMA, its MMAs and the tcgen05.commit that frees
// it), not per byte: tools/sm_stream_bench.cu on a B200 with the same MMA consumer, 96 SMs x 512 KiB,
// 11 x 16 KiB stages 40 GB/s per SM vs 5 x 32 KiB 51 GB/s (profiles/r02/probe/sm_stream_stage_size.txt).
// KS = 2 (5 stages of 36 KiB) is the default; KS = 1 (11 stages of 18 KiB) the round-2 original; KS = 3
// (3 stages of 54 KiB, all that fits) measured slower: T=1 / 8 / 16 33.4 / 99.6 / 150.0 vs 29.5 / 87.3 /
// 132.3 us (profiles/r02/probe/bench_ks3.txt) — too few stages in flight.
template <int KS>
struct DecodeRing {
  static_assert(KS == 1 || KS == 2, "k-blocks per stage");
  static constexpr int kStageBytes = KS * (kATileBytes + DecodeCfg::kBBytes);
  static constexpr int kStages = KS == 1 ? 11 : 5;
  static constexpr int kBOff = KS * kATileBytes;  // first token-row tile of a stage
  static constexpr int kBarBytes = 8 * (3 * kStages + 1 + 2 * DecodeCfg::kAcc + 2 * kRing) + 16 * kRing + 16;
  // folded logits + top-k scratch alias ring stage 0: used only between the routing MMAs' completion
  // and the first streaming load
  static_assert(DecodeCfg::kLogitBytes + DecodeCfg::kTopBytes <= kStageBytes, "routing scratch fits one ring stage");
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + DecodeCfg::kXBytes + DecodeCfg::kPartBytes +
                                    DecodeCfg::kPermBytes + kBarBytes;
  static_assert(kSmemBytes <= 232448, "decode kernel shared memory");
};

// hit experts' W2 below this many bytes is warmed in L2 during the UP phase
constexpr size_t kW2WarmBytes = 40u << 20;

struct DecodeParams {
  int T, H, I, E, topk, renorm;
  const __nv_bfloat16* x;  // [T, H]
  const uint8_t* w2;       // [E, H, I] bf16 (L2 warm-up addresses)
  int32_t* ids;            // [T, topk]
  float* w;                // [T, topk]
  int32_t* counts;         // [E]
  int32_t* offsets;        // [E+1]
  int32_t* slot_of;        // [T*topk]
  int32_t* tok_of;         // [T*topk]
  __nv_bfloat16* act;      // [S, I]
  __nv_bfloat16* y_perm;   // [S, H]
  uint32_t* sched;         // [0] item counter, [1+e] UP items done, [kUpDoneWord] all UP items done,
                           // [kExitWord] finished CTAs
  __nv_bfloat16* y;        // [T, H] combined output (nullptr: the caller runs k_combine)
  uint32_t* cmb;           // [T * H/256] fused-combine counters, zero on entry and left zero
  int weights_evict_first;
  int warm_w2;             // 1: L2-prefetch the hit experts' W2 when small
  int dnc;                 // 1: block-diagonal DN + combine items when S <= 16 and every UP item fits one wave
};

__device__ __forceinline__ void cluster_arrive_rel() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
// only orders "my DSMEM reads are done" (their values were consumed): no release needed
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acq() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// CS: CTAs per cluster (2: pairs, always co-resident, every SM streams; 4: each CTA computes one
// partial (half the Wr bytes per CTA, shorter routing), but 4-CTA clusters leave some SMs unused
// on a B200 (GPC boundaries) — the host picks 4 for latency-bound tiny batches)
template <int CS, int KS>
__global__ void __launch_bounds__(DecodeCfg::kThreads, 1)
    k_decode(const __grid_constant__ CUtensorMap tm_wr, const __grid_constant__ CUtensorMap tm_x,
             const __grid_constant__ CUtensorMap tm_w13h, const __grid_constant__ CUtensorMap tm_w2,
             const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_w2r8,
             const __grid_constant__ CUtensorMap tm_w2r16, const __grid_constant__ CUtensorMap tm_w2r32,
             const __grid_constant__ CUtensorMap tm_w2r64, const DecodeParams p) {
  using C = DecodeCfg;
  using R = DecodeRing<KS>;
  constexpr int kCl = CS;                 // CTAs per cluster
  constexpr int kPpc = C::kParts / CS;    // partial sums per CTA
  static_assert(kPpc <= C::kMaxPpc, "partials per CTA");
  constexpr int S_ = R::kStages;
  constexpr int A_ = C::kAcc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* cur = smem + S_ * R::kStageBytes;
  // k-block h of ring stage st: weight tile / token-row tile
  auto a_at = [&](int st, int h) { return smem + st * R::kStageBytes + h * kATileBytes; };
  auto b_at = [&](int st, int h) { return smem + st * R::kStageBytes + R::kBOff + h * C::kBBytes; };
  float* xbuf = reinterpret_cast<float*>(cur);        cur += C::kXBytes;     // [16 cols][64 lanes]
  float* s_part = reinterpret_cast<float*>(cur);      cur += C::kPartBytes;  // [ppc][16 tokens][128 experts]
  float* s_logit = reinterpret_cast<float*>(smem);                           // [16][128] (ring stage 0)
  int32_t* s_ids = reinterpret_cast<int32_t*>(smem + C::kLogitBytes);        // [16][32]
  float* s_p = reinterpret_cast<float*>(s_ids + C::kMaxT * 32);              // [16][32]
  int32_t* s_off = reinterpret_cast<int32_t*>(cur);   // [E+1]
  int32_t* s_cnt = s_off + (C::kMaxE + 1);            // [E]
  int32_t* s_hit = s_cnt + C::kMaxE;                  // [nnz] hit experts, ascending
  int32_t* s_tok = s_hit + C::kMaxE;                  // [S] token of each slot
  int32_t* s_ent = s_tok + C::kMaxE;                  // [S] expert of each routing entry
  int32_t* s_slot = s_ent + C::kMaxE;                 // [S] slot of each routing entry
  int32_t* s_wc = s_slot + C::kMaxE;                  // [4][E] per-warp counts, then exclusive bases
  int32_t* s_scal = s_wc + 4 * C::kMaxE;              // [0] nnz, [4..7] warp sums, [8..11] warp hit counts
  float* s_w = reinterpret_cast<float*>(s_scal + 19);  // [S] routing weights (every CTA)
  int32_t* s_fin = reinterpret_cast<int32_t*>(s_w + C::kMaxE);  // [2][kMaxT + 1] combine: finished tokens, count
  cur += C::kPermBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(cur);
  uint64_t* empty = full + S_;
  uint64_t* bfull = empty + S_;
  uint64_t* tfull = bfull + S_ + 1;
  uint64_t* tempty = tfull + A_;
  uint64_t* sfull = tempty + A_;
  uint64_t* sempty = sfull + kRing;
  int4* ring = reinterpret_cast<int4*>(sempty + kRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);

  const int warp = warp_idx();
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const int E = p.E, T = p.T, K = p.topk, S = T * K;
  const int cr = static_cast<int>(cluster_ctarank());
  const int kbp = p.H / 256;  // k-blocks per partial sum (4 fixed partials of K = H)
  const int kbr = kPpc * kbp;  // routing k-blocks of this CTA: partials kPpc*cr .. kPpc*cr+kPpc-1
  [[maybe_unused]] const bool tr = blockIdx.x == 0;  // trace builds only
  if (tid == 0) LP_TRACE_MIN(48);

  if (tid == 0) {
    for (int s = 0; s < S_; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&bfull[s], kGatherThreads);
    }
    for (int a = 0; a < A_; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    for (int r = 0; r < kRing; ++r) { mbar_init(&sfull[r], 1); mbar_init(&sempty[r], 4); }  // MMA, epi, 2 gather
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_wr); prefetch_tmap(&tm_x); prefetch_tmap(&tm_w13h); prefetch_tmap(&tm_w2);
    prefetch_tmap(&tm_act);
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Pipeline positions carried from the routing item into the expert stream.
  int stage = 0; uint32_t phase = 0;  // ring (producer / MMA / gather each keep their own copy)
  int acc = 0; uint32_t aph = 0;      // TMEM accumulators (MMA / epilogue)

  // =============================== routing: partial sum `cr` of the logits ===============================
  const int nst_r = (kbr + KS - 1) / KS;  // ring stages of the routing item
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      const int npre = nst_r < S_ ? nst_r : S_;
      for (int i = 0; i < npre; ++i) {  // Wr before griddepcontrol.wait: weights never depend on the predecessor
        const int nh = min(KS, kbr - i * KS);
        mbar_arrive_expect_tx(&full[i], nh * (kATileBytes + C::kBBytes));
        for (int h = 0; h < nh; ++h) tma_load_2d(a_at(i, h), &tm_wr, &full[i], (cr * kbr + i * KS + h) * kTileK, 0, pol);
      }
      pdl_wait();
      LP_TRACE_AT(tr, 54);
      for (int i = 0; i < npre; ++i)
        for (int h = 0; h < min(KS, kbr - i * KS); ++h)
          tma_load_2d(b_at(i, h), &tm_x, &full[i], (cr * kbr + i * KS + h) * kTileK, 0, pol);
      stage = npre % S_;
      phase = npre == S_ ? 1u : 0u;
      for (int i = npre; i < nst_r; ++i) {
        const int nh = min(KS, kbr - i * KS);
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], nh * (kATileBytes + C::kBBytes));
        for (int h = 0; h < nh; ++h) {
          tma_load_2d(a_at(stage, h), &tm_wr, &full[stage], (cr * kbr + i * KS + h) * kTileK, 0, pol);
          tma_load_2d(b_at(stage, h), &tm_x, &full[stage], (cr * kbr + i * KS + h) * kTileK, 0, pol);
        }
        if (++stage == S_) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, C::kN);
      // routing k-block kb of this CTA: partial (kb / kbp) accumulates in TMEM columns 16 * (kb / kbp)
      auto mma_kb = [&](int st, int h, int kb) {
        const uint64_t a0 = sdesc_kmajor_sw128(smem_u32(a_at(st, h)));
        const uint64_t b0 = sdesc_kmajor_sw128(smem_u32(b_at(st, h)));
        const uint32_t d = tmem_base + (kb / kbp) * C::kN;
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_bf16(d, a0 + 2 * k, b0 + 2 * k, idesc, ((kb % kbp) | k) != 0);
      };
      if (nst_r <= S_) {
        // every routing stage fits the ring (all loads already in flight): wait for all of them,
        // then issue the whole MMA chain back to back — a stage wait after an MMA issue costs the
        // issuing thread ~250 cycles (tools/mma_chain_bench.cu), so no wait sits between MMAs.
        // Same MMAs in the same order as below (bit-identical logits).
        for (int i = 0; i < nst_r; ++i) {
          mbar_wait(&full[i], 0);
          mbar_wait(&bfull[i], 0);
        }
        tc_fence_after();
        for (int kb = 0; kb < kbr; ++kb) mma_kb(kb / KS, kb % KS, kb);
        for (int i = 0; i < nst_r; ++i) mma_commit(&empty[i]);
        stage = nst_r % S_;
        phase = nst_r == S_ ? 1u : 0u;
      }
      for (int i = 0; i < (nst_r <= S_ ? 0 : nst_r); ++i) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&bfull[stage], phase);
        tc_fence_after();
        for (int h = 0; h < min(KS, kbr - i * KS); ++h) mma_kb(stage, h, i * KS + h);
        mma_commit(&empty[stage]);
        if (++stage == S_) { stage = 0; phase ^= 1; }
      }
      mma_commit(&tfull[0]);
    }
  } else if (warp == 2 || warp == 3) {
    for (int i = 0; i < nst_r; ++i) {  // routing operands come by TMA: keep bfull's phases in step
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_arrive(&bfull[stage]);
      cp_async_commit();  // one (empty) group per stage, as in the stream below
      if (++stage == S_) { stage = 0; phase ^= 1; }
    }
  } else {
    const int q = warp & 3;
    mbar_wait(&tfull[0], 0);
    tc_fence_after();
    const int e = 32 * q + lane;
#pragma unroll
    for (int pl = 0; pl < kPpc; ++pl) {
      uint32_t v[16];
      tmem_ld16(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + pl * C::kN, v);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) s_part[(pl * C::kMaxT + i) * C::kMaxE + e] = __uint_as_float(v[i]);
    }
    tc_fence_before();
    mbar_arrive(&tempty[0]);
    if (tid == 128) LP_TRACE_AT(tr, 49);
  }
  // ring / accumulator positions after the routing item (every role advanced through nst_r stages)
  stage = nst_r % S_;
  phase = (nst_r / S_) & 1;
  acc = 1;
  aph = 0;
  pdl_wait();
  __syncthreads();
  cluster_arrive_rel();  // this CTA's partial is readable over DSMEM
  cluster_wait_acq();

  // fold the 4 partials in global part order p0 + p1 + p2 + p3 (rank r holds parts kPpc*r ..), exactly
  // as k_router<4, 4, 16> folds its four CTAs' partials
  for (int idx = tid; idx < T * (C::kMaxE / 4); idx += C::kThreads) {
    const int t = idx / (C::kMaxE / 4), e4 = (idx % (C::kMaxE / 4)) * 4;
    float4 v[C::kParts];
#pragma unroll
    for (int r = 0; r < kCl; ++r)
#pragma unroll
      for (int pl = 0; pl < kPpc; ++pl)
        v[r * kPpc + pl] =
            ld_dsmem_f4(mapa_shared(smem_u32(s_part + (pl * C::kMaxT + t) * C::kMaxE + e4), r));
    float4 a = v[0];
#pragma unroll
    for (int i = 1; i < C::kParts; ++i) { a.x += v[i].x; a.y += v[i].y; a.z += v[i].z; a.w += v[i].w; }
    *reinterpret_cast<float4*>(s_logit + t * C::kMaxE + e4) = a;
  }
  __syncthreads();
  if (tid == 0) LP_TRACE_AT(tr, 50);
  cluster_arrive_relaxed();  // remote partials consumed (matched by the wait before exit)
  if (tid == 0) LP_TRACE_AT(tr, 57);

  // softmax + top-k: one warp per token (the router's LPT = 32 at this tile shape)
  for (int g = warp; g < T; g += C::kThreads / 32) {
    float psum, inv;
    topk_lanes<32, 4>(s_logit + g * C::kMaxE, E, K, lane, s_ids + g * 32, s_p + g * 32, psum, inv);
    __syncwarp();
    for (int r = lane; r < K; r += 32) {
      const int id = s_ids[g * 32 + r];
      const float wt = p.renorm ? s_p[g * 32 + r] / psum : s_p[g * 32 + r] * inv;
      s_ent[g * K + r] = id;
      s_w[g * K + r] = wt;
      if (blockIdx.x == 0) {
        p.ids[static_cast<size_t>(g) * K + r] = id;
        p.w[static_cast<size_t>(g) * K + r] = wt;
      }
    }
  }
  if (tid == 0) LP_TRACE_AT(tr, 55);
  for (int i = tid; i < 4 * C::kMaxE; i += C::kThreads) s_wc[i] = 0;
  __syncthreads();
  if (tid == 0) LP_TRACE_AT(tr, 56);

  // stable counting sort of the S <= 128 routing entries (warps 0-3 own entries 32w..32w+31)
  int my_e = -1, my_rank = 0;
  if (warp < 4) {
    my_e = tid < S ? s_ent[tid] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, my_e);
    my_rank = __popc(peers & ((1u << lane) - 1u));
    if (my_e >= 0 && (__ffs(peers) - 1) == lane) s_wc[warp * C::kMaxE + my_e] = __popc(peers);
  }
  __syncthreads();
  if (tid < C::kMaxE) {  // per expert: exclusive bases over the 4 warps, total count
    int run = 0;
#pragma unroll
    for (int w4 = 0; w4 < 4; ++w4) {
      const int c = s_wc[w4 * C::kMaxE + tid];
      s_wc[w4 * C::kMaxE + tid] = run;
      run += c;
    }
    s_cnt[tid] = tid < E ? run : 0;
  }
  __syncthreads();
  if (warp < 4) {  // exclusive scan of counts over experts (4 warps x 32) + the hit-expert list
    const int c = s_cnt[tid];
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += n;
    }
    const unsigned hb = __ballot_sync(0xffffffffu, c > 0);
    if (lane == 31) { s_scal[4 + warp] = inc; s_scal[8 + warp] = __popc(hb); }
    named_bar_sync(3, 128);
    int base = 0, hbase = 0;
    for (int w4 = 0; w4 < warp; ++w4) { base += s_scal[4 + w4]; hbase += s_scal[8 + w4]; }
    if (tid < E) s_off[tid] = base + inc - c;
    if (tid == 0) s_off[E] = S;
    if (c > 0) s_hit[hbase + __popc(hb & ((1u << lane) - 1u))] = tid;
    if (tid == 127) s_scal[0] = hbase + __popc(hb);
  }
  __syncthreads();
  if (my_e >= 0) {
    const int slot = s_off[my_e] + s_wc[warp * C::kMaxE + my_e] + my_rank;
    s_slot[tid] = slot;
    s_tok[slot] = tid / K;
  }
  __syncthreads();
  if (blockIdx.x == 0) {  // publish the permutation (k_combine, the caller's stats)
    for (int i = tid; i < S; i += C::kThreads) {
      p.slot_of[i] = s_slot[i];
      p.tok_of[i] = s_tok[i];
    }
    for (int i = tid; i < E; i += C::kThreads) p.counts[i] = s_cnt[i];
    for (int i = tid; i <= E; i += C::kThreads) p.offsets[i] = s_off[i];
  }

  if (tid == 0) LP_TRACE_AT(tr, 51);
  const int nnz = s_scal[0];
  const int mt_up = p.I / 64;
  const int mt_dn = (p.H + kTileM - 1) / kTileM;
  const int n_up = mt_up * nnz;
  // S <= 16 (T <= 2 at top-8): DN items are block-diagonal tiles of ALL hit experts — rows
  // [j*R, (j+1)*R) of the 128-row A tile are W2 rows f0..f0+R-1 of hit expert j (R = 128 / nnz
  // rounded up to a power of two), B = every slot's act row, so D[j*R + r][slot] is expert j's
  // output feature f0 + r for that slot (the other columns are discarded). Each item then holds
  // every routed row of its R features and combines them in the epilogue (fixed j order, the
  // bf16-rounded row values: bit-identical to k_combine) — no y_perm round trip, no cross-CTA
  // completion counters on the critical path.
  // (all UP items must run in one wave: a DNC item waits for EVERY UP item, not just its expert's)
  const bool dnc = p.dnc && p.y != nullptr && S <= C::kN && n_up <= static_cast<int>(gridDim.x);
  int rdnc = 128;
  while (dnc && rdnc > 8 && rdnc * nnz > 128) rdnc >>= 1;
  const int n_items = n_up + (dnc ? p.H / rdnc : mt_dn * nnz);

  // =============================== expert stream (k_experts_tiny's pipeline) ===============================
  if (warp == 0) {
    if (lane == 1 && p.warm_w2) {
      // warm the hit experts' W2 in L2 while the UP items stream (this CTA's share of the union)
      const size_t per_e = static_cast<size_t>(p.H) * p.I * 2;
      const size_t total = per_e * nnz;
      if (total <= kW2WarmBytes) {
        const size_t share = ((total + gridDim.x - 1) / gridDim.x + 4095) & ~size_t(4095);
        size_t lo = share * blockIdx.x;
        const size_t hi = min(total, lo + share);
        while (lo < hi) {
          const size_t k = lo / per_e, o = lo - k * per_e;
          const size_t n = min(min(hi - lo, per_e - o), size_t(65536));
          bulk_prefetch_l2(p.w2 + static_cast<size_t>(s_hit[k]) * per_e + o, static_cast<uint32_t>(n));
          lo += n;
        }
      }
    }
    if (lane == 0) {
      const uint64_t pol_w = p.weights_evict_first ? policy_evict_first() : policy_evict_normal();
      int r = 0; uint32_t rph = 0;
      [[maybe_unused]] int n_item = 0;
      while (true) {
        // first item static (CTA b takes item b: no global atomic round trip before the first weight load),
        // the rest claimed dynamically in item order (all UP items precede all DN items: deadlock-free)
        const int it = n_item == 0 ? static_cast<int>(blockIdx.x)
                                   : static_cast<int>(gridDim.x + atomicAdd(&p.sched[0], 1u));
        if (n_item == 0) LP_TRACE_MIN(52);
        LP_ITEM(n_item, 0, static_cast<unsigned long long>(it));
        LP_ITEM(n_item, 1, LP_NOW());
        int4 info;
        if (it >= n_items) {
          info = make_int4(kItemEnd, 0, 0, 0);
        } else {
          const bool up = it < n_up;
          if (!up && dnc) {
            info = make_int4(kItemDnc, (it - n_up) * rdnc, 0, S);
          } else {
            const int mtc = up ? mt_up : mt_dn;
            const int local = up ? it : it - n_up;
            const int e = s_hit[local / mtc];
            const int mt = local % mtc;
            info = make_int4((up ? kItemUp : kItemDown) | (e << 8), mt * (up ? 64 : kTileM), s_off[e], s_cnt[e]);
          }
        }
        mbar_wait(&sempty[r], rph ^ 1);
        ring[r] = info;
        mbar_arrive(&sfull[r]);
        if (++r == kRing) { r = 0; rph ^= 1; }
        const int kind = info.x & 0xff;
        if (kind == kItemEnd) break;
        const int e = info.x >> 8, m0 = info.y;
        // weight tiles only: UP token rows and DN / DNC act rows are copied by the gather warps
        const int kblocks = kind == kItemUp ? p.H / kTileK : p.I / kTileK;
        const CUtensorMap* tmr = kind != kItemDnc ? &tm_w2 : rdnc == 8 ? &tm_w2r8 : rdnc == 16 ? &tm_w2r16
                                 : rdnc == 32 ? &tm_w2r32 : rdnc == 64 ? &tm_w2r64 : &tm_w2;
        const uint32_t abytes = kind == kItemDnc ? static_cast<uint32_t>(nnz * rdnc * 128) : kATileBytes;
        LP_ITEM(n_item, 2, LP_NOW());
        for (int kb = 0; kb < kblocks; kb += KS) {
          const int nh = min(KS, kblocks - kb);
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], nh * abytes);
          for (int h = 0; h < nh; ++h) {
            uint8_t* sa = a_at(stage, h);
            const int kc = (kb + h) * kTileK;
            if (kind == kItemUp) {
              // rows 0-63: gate features m0..m0+63, rows 64-127: the matching up rows
              tma_load_2d(sa, &tm_w13h, &full[stage], kc, e * 2 * p.I + m0, pol_w);
              tma_load_2d(sa + kATileBytes / 2, &tm_w13h, &full[stage], kc, e * 2 * p.I + p.I + m0, pol_w);
            } else if (kind == kItemDnc) {
              // W2 rows f0..f0+R-1 of every hit expert (block-diagonal A tile)
              for (int j = 0; j < nnz; ++j) tma_load_2d(sa + j * rdnc * 128, tmr, &full[stage], kc, s_hit[j] * p.H + m0, pol_w);
            } else {
              tma_load_2d(sa, &tm_w2, &full[stage], kc, e * p.H + m0, pol_w);
            }
          }
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
        LP_ITEM(n_item, 3, LP_NOW());
        ++n_item;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int r = 0; uint32_t rph = 0;
      [[maybe_unused]] int n_item = 0;
      while (true) {
        mbar_wait(&sfull[r], rph);
        const int4 info = ring[r];
        mbar_arrive(&sempty[r]);
        if (++r == kRing) { r = 0; rph ^= 1; }
        const int kind = info.x & 0xff;
        if (kind == kItemEnd) break;
        const bool up = kind == kItemUp;
        const uint32_t idesc = idesc_bf16_f32(kTileM, (info.w + 15) & ~15);
        const int kblocks = up ? p.H / kTileK : p.I / kTileK;
        const int nst = (kblocks + KS - 1) / KS;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * C::kN;
#ifndef LP_DECODE_MMA_BATCH
// k-blocks waited for together. KS = 1: 4 (T=1 / 16 30.3 / 133.7-134.5 vs 30.8-31.1 / 136.6 us with 1);
// KS = 2: 2, i.e. one stage (T=1 / 2 / 8 / 16 28.7 / 38.8 / 86.9 / 130.7 vs 29.7 / 39.9 / 87.7 / 132.5 us
// with 4 and 33.1 / 44.6 / 96.7 / 145.6 with 6; profiles/r02/probe/bench_mma_batch.txt)
#define LP_DECODE_MMA_BATCH (KS == 1 ? 4 : 2)
#endif
        constexpr int MB = (LP_DECODE_MMA_BATCH + KS - 1) / KS;  // stages waited for together, then issued back to back
        for (int s0 = 0; s0 < nst; s0 += MB) {
          int st[MB];
          uint32_t ph[MB];
#pragma unroll
          for (int g = 0; g < MB; ++g) {
            st[g] = stage + g < S_ ? stage + g : stage + g - S_;
            ph[g] = stage + g < S_ ? phase : phase ^ 1u;
          }
#pragma unroll
          for (int g = 0; g < MB; ++g) {
            if (s0 + g < nst) {
              mbar_wait(&full[st[g]], ph[g]);
              mbar_wait(&bfull[st[g]], ph[g]);
            }
          }
          tc_fence_after();
          if (s0 == 0) LP_ITEM(n_item, 5, LP_NOW());
#pragma unroll
          for (int g = 0; g < MB; ++g) {
#pragma unroll
            for (int h = 0; h < KS; ++h) {
              const int kb = (s0 + g) * KS + h;
              if (s0 + g < nst && kb < kblocks) {
                const uint64_t a0 = sdesc_kmajor_sw128(smem_u32(a_at(st[g], h)));
                const uint64_t b0 = sdesc_kmajor_sw128(smem_u32(b_at(st[g], h)));
#pragma unroll
                for (int k = 0; k < kTileK / 16; ++k) mma_bf16(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0);
              }
            }
          }
#pragma unroll
          for (int g = 0; g < MB; ++g) {
            if (s0 + g < nst) {
              mma_commit(&empty[stage]);
              if (++stage == S_) { stage = 0; phase ^= 1; }
            }
          }
        }
        mma_commit(&tfull[acc]);
        LP_ITEM(n_item, 6, LP_NOW());
        ++n_item;
        if (++acc == A_) { acc = 0; aph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 2 || warp == 3) {
    // B rows of every item, 16-byte cp.async into the SWIZZLE_128B layout: UP items' token rows
    // (from x), DN / DNC items' act rows once the UP items they need are done (expert e's for DN,
    // every expert's for DNC)
    constexpr int RPT = C::kN / 8;
    const int gt = tid - 64;
    const int g = gt >> 3, j = gt & 7;
    const uint64_t pol_x = policy_evict_last();
    const uint32_t sw = static_cast<uint32_t>((j ^ g) << 4) + static_cast<uint32_t>(g * 128);
    int r = 0; uint32_t rph = 0;
    while (true) {
      mbar_wait(&sfull[r], rph);
      const int4 info = ring[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[r]);
      if (++r == kRing) { r = 0; rph ^= 1; }
      const int kind = info.x & 0xff;
      if (kind == kItemEnd) break;
      const int row0 = info.z, nvalid = info.w;
      const bool up = kind == kItemUp;
      const int K_ = up ? p.H : p.I;  // row length of the source
      const __nv_bfloat16* src0;
      int rowi[RPT];  // source row of each copied tile row (-1: none)
      if (up) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int rr = g + 8 * i;
          rowi[i] = rr < nvalid ? s_tok[row0 + rr] : -1;
        }
        src0 = p.x + j * 8;
      } else {
        // every lane acquires (its own cp.async reads are ordered after its own acquire)
        if (kind == kItemDnc)
          while (ld_acquire_u32(&p.sched[C::kUpDoneWord]) < static_cast<uint32_t>(n_up)) __nanosleep(32);
        else
          while (ld_acquire_u32(&p.sched[1 + (info.x >> 8)]) < static_cast<uint32_t>(mt_up)) __nanosleep(32);
#pragma unroll
        for (int i = 0; i < RPT; ++i) rowi[i] = g + 8 * i < nvalid ? g + 8 * i : -1;
        src0 = p.act + static_cast<size_t>(row0) * p.I + j * 8;
      }
      const int kblocks = K_ / kTileK;
      for (int kb = 0; kb < kblocks; kb += KS) {
        mbar_wait(&empty[stage], phase ^ 1);
        cp_async_wait_group<S_ - 1>();  // this slot's previous copies (S_ groups ago) landed
        for (int h = 0; h < min(KS, kblocks - kb); ++h) {
          const uint32_t sb = smem_u32(b_at(stage, h)) + sw;
#pragma unroll
          for (int i = 0; i < RPT; ++i)
            if (rowi[i] >= 0) cp_async16(sb + i * 8 * 128, src0 + static_cast<size_t>(rowi[i]) * K_ + (kb + h) * kTileK, pol_x);
        }
        cp_async_arrive_noinc(&bfull[stage]);
        cp_async_commit();
        if (++stage == S_) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // epilogue (w4-w7: TMEM lane quarter q = warp & 3), as k_experts_tiny
    const int q = warp & 3;
    const int et = tid - 128;  // 0..127
    int r = 0; uint32_t rph = 0;
    [[maybe_unused]] int n_item = 0;
    int n_dn = 0;
    while (true) {
      mbar_wait(&sfull[r], rph);
      const int4 info = ring[r];
      const int kind = info.x & 0xff;
      if (kind == kItemEnd) break;
      const int e = info.x >> 8, m0 = info.y, row0 = info.z, nvalid = info.w;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      if (et == 0) LP_ITEM(n_item, 7, LP_NOW());
      uint32_t v[16];
      tmem_ld16(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * C::kN, v);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == A_) { acc = 0; aph ^= 1; }
      if (kind == kItemUp) {
        named_bar_sync(2, 128);  // the previous item's readers are done with xbuf
        if (q >= 2) {
#pragma unroll
          for (int i = 0; i < 16; ++i) xbuf[i * 64 + 32 * (q - 2) + lane] = __uint_as_float(v[i]);
        }
        named_bar_sync(2, 128);
        if (q < 2) {
          const int feat = m0 + 32 * q + lane;
          __nv_bfloat16* dst = p.act + static_cast<size_t>(row0) * p.I + feat;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < nvalid)
              dst[static_cast<size_t>(i) * p.I] =
                  __float2bfloat16_rn(silu_mul(__uint_as_float(v[i]), xbuf[i * 64 + 32 * q + lane]));
        }
        fence_proxy_async_global();  // act rows are read back through TMA (async proxy)
        named_bar_sync(1, 128);      // every thread's act stores precede the count
      } else if (kind == kItemDnc) {
        // lane m = j*R + r of the block-diagonal tile: expert slot j (hit expert s_hit[j]), feature m0 + r
        __nv_bfloat16* yv = reinterpret_cast<__nv_bfloat16*>(xbuf);  // [S slots][R] bf16 row values
        named_bar_sync(2, 128);  // the previous item's readers are done with xbuf
        const int jx = et / rdnc, r = et - jx * rdnc;
        if (jx < nnz) {
          const int e = s_hit[jx];
          const int n0 = s_off[e], n1 = n0 + s_cnt[e];
#pragma unroll
          for (int n = 0; n < 16; ++n)
            if (n >= n0 && n < n1) yv[n * rdnc + r] = __float2bfloat16_rn(__uint_as_float(v[n]));
        }
        named_bar_sync(2, 128);
        for (int idx = et; idx < T * rdnc; idx += 128) {
          const int t = idx / rdnc, rr = idx - t * rdnc;
          float a = 0.f;
          for (int jj = 0; jj < K; ++jj)  // fixed j order, as k_combine
            a += s_w[t * K + jj] * __bfloat162float(yv[s_slot[t * K + jj] * rdnc + rr]);
          p.y[static_cast<size_t>(t) * p.H + m0 + rr] = __float2bfloat16_rn(a);
        }
      } else {
        const int feat = m0 + 32 * q + lane;
        if (feat < p.H) {
          __nv_bfloat16* dst = p.y_perm + static_cast<size_t>(row0) * p.H + feat;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < nvalid) dst[static_cast<size_t>(i) * p.H] = __float2bfloat16_rn(__uint_as_float(v[i]));
        }
        if (p.y != nullptr) {
          // Fused combine: per (token, 256-feature block) a counter of finished DN halves; the item
          // completing a block (2 * topk halves) sums the token's topk y_perm rows over those 256
          // features in fixed j order (bit-identical to k_combine) and writes y. Release: this
          // item's y_perm stores precede the barrier and each row's acq_rel increment; acquire:
          // the completing increment, then L2 reads (ld.cg) of the other items' rows.
          int32_t* fin = s_fin + (n_dn & 1) * (C::kMaxT + 1);
          ++n_dn;
          if (et == 0) fin[C::kMaxT] = 0;  // readers of this buffer (two DN items ago) are past barrier 1
          named_bar_sync(1, 128);
          const int nfb = p.H / 256, fb = m0 / 256;
          if (et < nvalid) {
            const int t = s_tok[row0 + et];
            uint32_t* c = p.cmb + t * nfb + fb;
            if (atom_add_acqrel_gpu(c, 1u) == 2u * static_cast<uint32_t>(K) - 1u) {
              *c = 0u;  // every increment of this call has happened: left zero for the next call
              fin[atomicAdd(&fin[C::kMaxT], 1)] = t;
            }
          }
          named_bar_sync(1, 128);
          const int nfin = fin[C::kMaxT];
          for (int i = q; i < nfin; i += 4) {
            const int t = fin[i];
            const size_t col = static_cast<size_t>(fb) * 256 + lane * 8;
            float a8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a8[u] = 0.f;
            for (int j0 = 0; j0 < K; j0 += 8) {  // eight rows in flight, summed in j order
              uint4 d[8];
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (j0 + u < K)
                  d[u] = __ldcg(reinterpret_cast<const uint4*>(p.y_perm + static_cast<size_t>(s_slot[t * K + j0 + u]) *
                                                                              p.H + col));
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                if (j0 + u < K) {
                  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&d[u]);
                  const float wj = s_w[t * K + j0 + u];
#pragma unroll
                  for (int q2 = 0; q2 < 4; ++q2) {
                    const float2 f = __bfloat1622float2(h2[q2]);
                    a8[2 * q2] += wj * f.x;
                    a8[2 * q2 + 1] += wj * f.y;
                  }
                }
              }
            }
            uint4 o;
            __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) o2[q2] = __floats2bfloat162_rn(a8[2 * q2], a8[2 * q2 + 1]);
            *reinterpret_cast<uint4*>(p.y + static_cast<size_t>(t) * p.H + col) = o;
          }
        }
      }
      if (et == 0) {
        mbar_arrive(&sempty[r]);
        if (kind == kItemUp) {  // release: the item's act rows are written
          __threadfence();
          atomicAdd(&p.sched[1 + e], 1u);
          if (dnc) atomicAdd(&p.sched[C::kUpDoneWord], 1u);
        }
        LP_ITEM(n_item, 4, LP_NOW());
      }
      ++n_item;
      if (++r == kRing) { r = 0; rph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {  // the last CTA out leaves the scheduler words zero for the next call
    __threadfence();
    if (atomicAdd(&p.sched[C::kExitWord], 1u) == gridDim.x - 1) {
      for (int i = 0; i <= E; ++i) p.sched[i] = 0u;
      p.sched[C::kUpDoneWord] = 0u;
      p.sched[C::kExitWord] = 0u;
      __threadfence();
    }
  }
  if (tid == 0) LP_TRACE_MAX(53);
  cluster_wait_acq();  // no CTA leaves while a cluster peer may still read its partials
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

}  // namespace lp

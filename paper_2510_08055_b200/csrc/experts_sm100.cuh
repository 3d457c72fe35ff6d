// Grouped expert FFN for one MoE layer on sm_100a (tcgen05 + TMEM + TMA).
//
// One persistent launch does both expert GEMMs of Qwen3-MoE experts
// (HF transformers 5.5 `Qwen3MoeExperts.forward`, modeling_qwen3_moe.py:229-249):
//     act[s, :]    = SiLU(x_perm[s] . W13[e, 0:I]^T) * (x_perm[s] . W13[e, I:2I]^T)
//     y_perm[s, :] = act[s] . W2[e]^T
// for every slot s of expert e (slots are expert-contiguous, see permute.cuh).
//
// Swap-AB: the weight rows are the MMA M operand (128 rows per tile) and the
// expert's tokens are the N operand (16..MAX_N), so a tile streams a 128-row
// weight slice exactly once no matter how few tokens the expert received —
// the low-tokens-per-expert (memory-bound) regime the layered-prefill paper
// is about. Work items, in the order they are handed out:
//   UP  (e, mt, nt): 128 gate rows + the matching 128 up rows, K = H.
//                    Gate and up accumulate into separate TMEM column ranges
//                    of the same lanes, so SiLU(g)*u is a per-thread epilogue.
//   DN  (e, mt, nt): 256 rows of W2 (output features) as two 128-row tiles
//                    accumulated side by side (same smem/TMEM shape as UP, so
//                    both phases keep 2 weight tiles in flight per stage),
//                    K = I, waits until all UP items of expert e have
//                    published their act rows.
// Items are claimed dynamically (global atomic) by 1 CTA/SM; all UP items
// precede all DN items, so a DN wait can only target items already claimed
// by running CTAs (deadlock-free without co-residency guarantees).
//
// Warp roles (384 threads): w0 TMA producer + scheduler, w1 MMA issuer,
// w2 TMEM allocator, w4..w11 epilogue: warp w drains TMEM lanes 32*(w%4) ...,
// warps 4..7 the even 16-column chunks and 8..11 the odd ones, so the
// accumulator is released twice as fast (it is single-buffered at N=256).
#pragma once
#include <cuda_bf16.h>
#include "ptx.cuh"

namespace lp {

constexpr int kExpertsThreads = 384;  // w0 TMA+sched, w1 MMA, w2 TMEM alloc (+w3: gather), w4..w11 epilogue
constexpr int kGatherThreads = 64;    // warps 2-3 in GATHER mode
constexpr int kEpiThreads = 256;
constexpr int kTileM = 128;        // weight rows per tile
constexpr int kTileK = 64;         // bf16 elements per 128-byte swizzle row
constexpr int kBoxRows = 32;       // token rows per B-operand TMA box
constexpr int kRing = 4;           // scheduler ring depth
constexpr int kMaxExperts = 256;
constexpr uint32_t kATileBytes = kTileM * kTileK * 2;  // 16 KiB

struct ExpertsParams {
  int H, I, E;
  const int32_t* tok_of;       // [S] source row of each slot (nullptr: slot s reads row s)
  const int32_t* offsets;      // [E+1] expert slot offsets
  const int32_t* tile_prefix;  // [E+1] prefix sum of token tiles per expert
  const int32_t* tile_rows;    // [E]   token rows per tile of expert e
  __nv_bfloat16* act;          // [S, I]
  __nv_bfloat16* y_perm;       // [S, H]
  uint32_t* sched;             // [0] work counter, [1+e] UP items done for expert e
  int prefetch_kblocks;        // k-blocks of the first item's W13 rows to warm in L2 before pdl_wait
  int warm_rows;               // W13 rows [0, warm_rows) already warmed in L2 by the router
  int lookahead;               // L2 prefetch distance (k-blocks) for weight tiles ahead of the smem ring; 0 = off
  int weights_evict_first;     // weights loaded with L2::evict_first (1) or evict_normal (0)
  // Fused combine (y != nullptr): DN items count, per (token, 256-feature
  // block), how many of the token's topk slots are final; the item that
  // completes a block sums the token's topk y_perm rows in fixed j order
  // (bit-identical to k_combine) and writes y. Counters are zero on entry and
  // left zero (the completing item resets them).
  __nv_bfloat16* y;            // [T, H] or nullptr (separate k_combine)
  const int32_t* slot_tok;     // [S] token of each slot
  const int32_t* slot_of;      // [T*topk] slot of each routing entry
  const float* wgt;            // [T*topk] routing weights
  uint32_t* blk_cnt;           // [T * ceil(H/256)] completion counters
  int topk;
  const __nv_bfloat16* xsrc;   // GATHER: [rows, H] token rows read through tok_of by the gather warps
};

// DN-item tail of the fused combine (256 epilogue threads, named barrier 1).
// Release: every thread's y_perm stores precede the barrier, and each thread's
// acq_rel counter increment is cumulative over them; acquire: the completing
// increment, then the barrier, then L2 (ld.cg) reads of the other items' rows.
__device__ __forceinline__ uint32_t atom_add_acqrel_gpu(uint32_t* a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fused_combine(const ExpertsParams& p, int m0, int row0, int nvalid, int et,
                                              int32_t* s_fin) {
  const int nfb = (p.H + 255) / 256;
  const int fb = m0 / 256;
  if (et == 0) s_fin[kEpiThreads] = 0;
  named_bar_sync(1, kEpiThreads);
  if (et < nvalid) {
    const int t = __ldcg(p.slot_tok + row0 + et);
    uint32_t* c = p.blk_cnt + static_cast<size_t>(t) * nfb + fb;
    if (atom_add_acqrel_gpu(c, 1u) == static_cast<uint32_t>(p.topk - 1)) {
      *c = 0u;  // every increment of this call has happened: reset for the next call
      s_fin[atomicAdd(&s_fin[kEpiThreads], 1)] = t;
    }
  }
  named_bar_sync(1, kEpiThreads);
  const int nfin = s_fin[kEpiThreads];
  const int width = min(256, p.H - m0);  // features in this block (multiple of 128)
  const int lane = et & 31;
  for (int i = et >> 5; i < nfin; i += kEpiThreads / 32) {
    const int t = s_fin[i];
    if (lane * 8 < width) {
      float acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.f;
      for (int j0 = 0; j0 < p.topk; j0 += 8) {  // fixed j order: bit-identical to k_combine
        // all index / weight loads, then all row loads in flight, then the ordered sum
        int slot[8];
        float wj[8];
        uint4 d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool ok = j0 + u < p.topk;
          slot[u] = ok ? __ldcg(p.slot_of + static_cast<size_t>(t) * p.topk + j0 + u) : 0;
          wj[u] = ok ? __ldcg(p.wgt + static_cast<size_t>(t) * p.topk + j0 + u) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + u < p.topk)
            d[u] = __ldcg(reinterpret_cast<const uint4*>(p.y_perm + static_cast<size_t>(slot[u]) * p.H + m0) + lane);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (j0 + u < p.topk) {
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&d[u]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f = __bfloat1622float2(h2[q]);
              acc[2 * q] += wj[u] * f.x;
              acc[2 * q + 1] += wj[u] * f.y;
            }
          }
        }
      }
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q) o2[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
      reinterpret_cast<uint4*>(p.y + static_cast<size_t>(t) * p.H + m0)[lane] = o;
    }
  }
}

template <int MAX_N>
struct ExpertsCfg {
  static constexpr int kBBytes = MAX_N * 128;
  static constexpr int kStageBytes = 2 * kATileBytes + kBBytes;
  static constexpr int kStages = (MAX_N >= 256) ? 3 : (MAX_N >= 128 ? 4 : 5);
  static constexpr int kAccStages = (4 * MAX_N <= 512) ? 2 : 1;
  static constexpr int kAccCols = 2 * MAX_N;  // gate | up
  static constexpr int kTmemCols = kAccStages * kAccCols < 32 ? 32 : kAccStages * kAccCols;
  // barriers + ring + scalars + expert tables
  static constexpr int kAuxBytes = 8 * (3 * kStages + 1 + 2 * kAccStages + 2 * kRing) + 16 * kRing + 16 +
                                   4 * (3 * kMaxExperts + 2) + 4 * MAX_N + 4 * (kEpiThreads + 4);
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kAuxBytes;
};

enum : int { kItemUp = 0, kItemDown = 1, kItemEnd = 2, kItemDnc = 3 };  // kItemDnc: k_decode only

// SiLU(g) * u with one MUFU op: silu(g) = 0.5 g (1 + tanh(g / 2)); tanh.approx
// (rel. err ~2^-11) is well below the bf16 rounding of the result.
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float silu_mul(float g, float u) {
  const float hg = 0.5f * g;
  return fmaf(hg, tanh_approx(hg), hg) * u;
}

// GATHER: UP items read token rows of the unpermuted [rows, H] source (x)
// through tok_of: warps 2-3 copy them with 16-byte cp.async straight into the
// SWIZZLE_128B layout TMA would have produced and arrive on bfull[stage] when
// their copies land (no x_perm round trip through HBM). Otherwise rows are
// expert-contiguous (x_perm) and arrive in 32-row TMA boxes.
template <int MAX_N, bool GATHER>
__global__ void __launch_bounds__(kExpertsThreads, 1)
    k_experts(const __grid_constant__ CUtensorMap tm_w13, const __grid_constant__ CUtensorMap tm_w2,
              const __grid_constant__ CUtensorMap tm_xsrc, const __grid_constant__ CUtensorMap tm_act,
              const ExpertsParams p) {
  using C = ExpertsCfg<MAX_N>;
  constexpr int S_ = C::kStages;
  constexpr int A_ = C::kAccStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* aux = smem + S_ * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);
  uint64_t* empty = full + S_;
  uint64_t* tfull = empty + S_;
  uint64_t* tempty = tfull + A_;
  uint64_t* sfull = tempty + A_;
  uint64_t* sempty = sfull + kRing;
  uint64_t* bfull = sempty + kRing;  // GATHER: B operand (token rows) of the stage landed
  int4* ring = reinterpret_cast<int4*>(bfull + ((S_ + 1) & ~1));  // 16-byte aligned
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);
  int32_t* s_off = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_tp = s_off + (kMaxExperts + 1);
  int32_t* s_ts = s_tp + (kMaxExperts + 1);
  int32_t* s_tok = s_ts + kMaxExperts;  // [MAX_N] source rows of the current UP item
  int32_t* s_fin = s_tok + MAX_N;       // [kEpiThreads] tokens whose block this DN item completed; [.. + 0] count

  const int warp = warp_idx();
  const int lane = threadIdx.x & 31;
  const int E = p.E;
  if (threadIdx.x == 0) { LP_TRACE_MIN(32); LP_TRACE_AT(blockIdx.x == 0, 33); }

  if (threadIdx.x == 0) {
    for (int s = 0; s < S_; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < A_; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], kEpiThreads); }
    for (int r = 0; r < kRing; ++r) { mbar_init(&sfull[r], 1); mbar_init(&sempty[r], GATHER ? 4 : 2); }
    if (GATHER)
      for (int s = 0; s < S_; ++s) mbar_init(&bfull[s], kGatherThreads);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_w13); prefetch_tmap(&tm_w2); prefetch_tmap(&tm_xsrc); prefetch_tmap(&tm_act);
    // While the predecessors (router / scan / gather) finish, warm L2 with the
    // first k-blocks of this CTA's first work item (item == blockIdx.x), guessed
    // assuming one token tile per expert — exact in the memory-bound regime.
    const int mt_up0 = (p.I + kTileM - 1) / kTileM;
    const int e_guess = blockIdx.x / mt_up0;
    if (e_guess < E && e_guess * 2 * p.I + 2 * p.I > p.warm_rows) {
      const int row = e_guess * 2 * p.I + (blockIdx.x % mt_up0) * kTileM;
      const int kb_pf = min(p.prefetch_kblocks, p.H / kTileK);
      for (int kb = 0; kb < kb_pf; ++kb) {
        tma_prefetch_2d(&tm_w13, kb * kTileK, row);
        tma_prefetch_2d(&tm_w13, kb * kTileK, row + p.I);
      }
    }
  }
  // all 512 TMEM columns (MAX_N = 256) are only claimed once the predecessors
  // completed, so a co-resident predecessor CTA can never starve on allocation
  if (warp == 2 && C::kTmemCols < 512) tmem_alloc(tmem_slot, C::kTmemCols);
  pdl_trigger();
  pdl_wait();
  if (warp == 2 && C::kTmemCols >= 512) tmem_alloc(tmem_slot, C::kTmemCols);
  for (int i = threadIdx.x; i <= E; i += blockDim.x) { s_off[i] = p.offsets[i]; s_tp[i] = p.tile_prefix[i]; }
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_ts[i] = p.tile_rows[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // I and H need only be multiples of 64 (one k-block): a last partial 128-row
  // tile reads into the next rows (or TMA zero fill) and its extra features are
  // never stored (epilogue masks feat >= I / H).
  const int mt_up = (p.I + kTileM - 1) / kTileM;
  const int mt_dn = (p.H + 2 * kTileM - 1) / (2 * kTileM);
  const int total_tiles = s_tp[E];
  const int n_up = mt_up * total_tiles;
  const int n_items = (mt_up + mt_dn) * total_tiles;

  if (warp == 0) {
    // ===================== scheduler + TMA producer (warp-wide) =====================
    const uint64_t pol_w = p.weights_evict_first ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_a = policy_evict_last();   // activations: re-read by every m-tile
    int stage = 0; uint32_t phase = 0;
    int r = 0; uint32_t rph = 0;
    bool first = true;
#ifdef LP_TRACE
    int n_claimed = 0;
#endif
    while (true) {
      int it = 0;  // first item static (matches the L2 prefetch), then dynamic
      if (lane == 0) it = first ? static_cast<int>(blockIdx.x) : static_cast<int>(gridDim.x + atomicAdd(&p.sched[0], 1u));
      first = false;
      it = __shfl_sync(0xffffffffu, it, 0);
      int4 info;
      int need = 0;
      if (it >= n_items) {
        info = make_int4(kItemEnd, 0, 0, 0);
      } else {
        const bool up = it < n_up;
        const int mtc = up ? mt_up : mt_dn;
        const int local = up ? it : it - n_up;
        int lo = 0, hi = E;  // largest e with mtc*tp[e] <= local
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (mtc * s_tp[mid] <= local) lo = mid; else hi = mid;
        }
        const int e = lo;
        const int nt_e = s_tp[e + 1] - s_tp[e];
        const int rr = local - mtc * s_tp[e];
        const int mt = rr / nt_e, nt = rr - mt * nt_e;
        const int n_e = s_off[e + 1] - s_off[e];
        const int ts = s_ts[e];
        const int row0 = s_off[e] + nt * ts;
        const int nvalid = min(ts, n_e - nt * ts);
        info = make_int4((up ? kItemUp : kItemDown) | (e << 8), mt * (up ? kTileM : 2 * kTileM), row0, nvalid);
        need = mt_up * nt_e;
      }
      if (lane == 0) {
        mbar_wait(&sempty[r], rph ^ 1);
        ring[r] = info;
        mbar_arrive(&sfull[r]);
#ifdef LP_TRACE
        if (blockIdx.x < 4 && n_claimed < 30) {
          lp_trace(64 + blockIdx.x * 32 + n_claimed);
          g_lp_trace[192 + blockIdx.x * 32 + n_claimed] = static_cast<unsigned long long>(it);
        }
        ++n_claimed;
#endif
      }
      if (++r == kRing) { r = 0; rph ^= 1; }
      const int kind = info.x & 0xff;
      if (kind == kItemEnd) break;
      const int e = info.x >> 8, m0 = info.y, row0 = info.z, nvalid = info.w;
      const int nmma = (nvalid + 15) & ~15;
      const bool up = kind == kItemUp;
      (void)nmma;
      if (lane == 0) {
        const int nbox = (nvalid + kBoxRows - 1) / kBoxRows;
        if (!up) {
          while (ld_acquire_u32(&p.sched[1 + e]) < static_cast<uint32_t>(need)) __nanosleep(64);
          fence_proxy_async_global();
        }
        const int kblocks = up ? p.H / kTileK : p.I / kTileK;
        const bool two = up || m0 + kTileM < p.H;  // second A tile (up rows / upper W2 rows)
        const uint32_t bytes = (two ? 2 : 1) * kATileBytes + (GATHER && up ? 0 : nbox * kBoxRows * 128);
        const int arow = up ? e * 2 * p.I + m0 : e * p.H + m0;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + 2 * kATileBytes;
          mbar_arrive_expect_tx(&full[stage], bytes);
          if (p.lookahead && kb + p.lookahead < kblocks) {  // warm L2 ahead of the ring
            const int kp = (kb + p.lookahead) * kTileK;
            if (up) {
              tma_prefetch_2d(&tm_w13, kp, arow);
              tma_prefetch_2d(&tm_w13, kp, arow + p.I);
            } else {
              tma_prefetch_2d(&tm_w2, kp, arow);
              if (two) tma_prefetch_2d(&tm_w2, kp, arow + kTileM);
            }
          }
          if (up) {
            tma_load_2d(sa, &tm_w13, &full[stage], kb * kTileK, arow, pol_w);
            tma_load_2d(sa + kATileBytes, &tm_w13, &full[stage], kb * kTileK, arow + p.I, pol_w);
            if (!GATHER) {
              for (int b = 0; b < nbox; ++b)
                tma_load_2d(sb + b * kBoxRows * 128, &tm_xsrc, &full[stage], kb * kTileK, row0 + b * kBoxRows,
                            pol_a);
            }
          } else {
            tma_load_2d(sa, &tm_w2, &full[stage], kb * kTileK, arow, pol_w);
            if (two) tma_load_2d(sa + kATileBytes, &tm_w2, &full[stage], kb * kTileK, arow + kTileM, pol_w);
            for (int b = 0; b < nbox; ++b)
              tma_load_2d(sb + b * kBoxRows * 128, &tm_act, &full[stage], kb * kTileK, row0 + b * kBoxRows, pol_a);
          }
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (single thread) =====================
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      int r = 0; uint32_t rph = 0;
      int acc = 0; uint32_t aph = 0;
      while (true) {
        mbar_wait(&sfull[r], rph);
        const int4 info = ring[r];
        mbar_arrive(&sempty[r]);
        if (++r == kRing) { r = 0; rph ^= 1; }
        const int kind = info.x & 0xff;
        if (kind == kItemEnd) break;
        const bool up = kind == kItemUp;
        const bool two = up || info.y + kTileM < p.H;
        const int nmma = (info.w + 15) & ~15;
        const uint32_t idesc = idesc_bf16_f32(kTileM, nmma);
        const int kblocks = up ? p.H / kTileK : p.I / kTileK;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_gate = tmem_base + acc * C::kAccCols;
        const uint32_t d_up = d_gate + MAX_N;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          if (GATHER) mbar_wait(&bfull[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::kStageBytes);
          const uint64_t a0 = sdesc_kmajor_sw128(sa);
          const uint64_t a1 = sdesc_kmajor_sw128(sa + kATileBytes);
          const uint64_t b0 = sdesc_kmajor_sw128(sa + 2 * kATileBytes);
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k) {
            const uint32_t accum = (kb | k) != 0;
            mma_bf16(d_gate, a0 + 2 * k, b0 + 2 * k, idesc, accum);
            if (two) mma_bf16(d_up, a1 + 2 * k, b0 + 2 * k, idesc, accum);
          }
          mma_commit(&empty[stage]);
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        if (++acc == A_) { acc = 0; aph ^= 1; }
      }
    }
    __syncwarp();
  } else if (GATHER && (warp == 2 || warp == 3)) {
    // ===================== token-row gather (64 threads, LSU cp.async) =====================
    // Thread (g, j) copies 16-byte chunk j of rows g, g+8, ... of the item's
    // token tile; SWIZZLE_128B puts chunk j of row r at chunk slot j ^ (r & 7),
    // and r & 7 == g for all of this thread's rows.
    constexpr int RPT = MAX_N / 8;
    const int gt = threadIdx.x - 64;
    const int g = gt >> 3, j = gt & 7;
    const uint64_t pol_x = policy_evict_last();  // x is re-read by every m-tile of the token tile
    int stage = 0; uint32_t phase = 0;
    int r = 0; uint32_t rph = 0;
    while (true) {
      mbar_wait(&sfull[r], rph);
      const int4 info = ring[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[r]);
      if (++r == kRing) { r = 0; rph ^= 1; }
      const int kind = info.x & 0xff;
      if (kind == kItemEnd) break;
      if (kind == kItemUp) {
        const int row0 = info.z, nvalid = info.w;
        int tok[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int rr = g + 8 * i;
          tok[i] = rr < nvalid ? __ldg(p.tok_of + row0 + rr) : -1;
        }
        const __nv_bfloat16* xs = p.xsrc + j * 8;
        const uint32_t sw = static_cast<uint32_t>((j ^ g) << 4) + static_cast<uint32_t>(g * 128);
        for (int kb = 0; kb < p.H / kTileK; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          cp_async_wait_group<S_ - 1>();  // this slot's previous copies (S_ groups ago) landed
          const uint32_t sb = smem_u32(smem + stage * C::kStageBytes + 2 * kATileBytes) + sw;
#pragma unroll
          for (int i = 0; i < RPT; ++i)
            if (tok[i] >= 0) cp_async16(sb + i * 8 * 128, xs + static_cast<size_t>(tok[i]) * p.H + kb * kTileK, pol_x);
          cp_async_arrive_noinc(&bfull[stage]);
          cp_async_commit();
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      } else {  // DN items: B (act rows) comes by TMA; keep bfull's phases in step
        for (int kb = 0; kb < p.I / kTileK; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive(&bfull[stage]);
          cp_async_commit();  // (empty group: one group per stage)
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> regs -> global =====================
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;       // 0: even chunks, 1: odd chunks
    const int et = threadIdx.x - 128;       // 0..255
    int r = 0; uint32_t rph = 0;
    int acc = 0; uint32_t aph = 0;
    while (true) {
      mbar_wait(&sfull[r], rph);
      const int4 info = ring[r];
      const int kind = info.x & 0xff;
      if (kind == kItemEnd) break;
      const int e = info.x >> 8, m0 = info.y, row0 = info.z, nvalid = info.w;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t t_gate = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * C::kAccCols;
      const int feat = m0 + 32 * q + lane;  // output feature owned by this thread
      const int nchunks = (nvalid + 15) / 16;
      if (kind == kItemUp) {
        const bool fok = feat < p.I;
        __nv_bfloat16* dst = p.act + static_cast<size_t>(row0) * p.I + feat;
        for (int c = half; c < nchunks; c += 2) {
          uint32_t g[16], u[16];
          tmem_ld16(t_gate + c * 16, g);
          tmem_ld16(t_gate + MAX_N + c * 16, u);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = c * 16 + i;
            if (n < nvalid && fok)
              dst[static_cast<size_t>(n) * p.I] =
                  __float2bfloat16_rn(silu_mul(__uint_as_float(g[i]), __uint_as_float(u[i])));
          }
        }
      } else {
        const bool two = m0 + kTileM < p.H;
        const bool fok = feat < p.H, fok2 = feat + kTileM < p.H;
        __nv_bfloat16* dst = p.y_perm + static_cast<size_t>(row0) * p.H + feat;
        for (int c = half; c < nchunks; c += 2) {
          uint32_t v[16], v2[16];
          tmem_ld16(t_gate + c * 16, v);
          if (two) tmem_ld16(t_gate + MAX_N + c * 16, v2);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = c * 16 + i;
            if (n < nvalid) {
              if (fok) dst[static_cast<size_t>(n) * p.H] = __float2bfloat16_rn(__uint_as_float(v[i]));
              if (two && fok2) dst[static_cast<size_t>(n) * p.H + kTileM] = __float2bfloat16_rn(__uint_as_float(v2[i]));
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == A_) { acc = 0; aph ^= 1; }
      if (kind == kItemUp) fence_proxy_async_global();  // act rows are read back through TMA (async proxy)
      if (kind == kItemDown && p.y != nullptr) fused_combine(p, m0, row0, nvalid, et, s_fin);
      if (kind == kItemUp) named_bar_sync(1, kEpiThreads);  // every thread's act stores precede the count
      if (et == 0) {
        mbar_arrive(&sempty[r]);
        if (kind == kItemUp) {  // release: every epilogue thread's act stores precede the count
          __threadfence();
          atomicAdd(&p.sched[1 + e], 1u);
        }
      }
      if (++r == kRing) { r = 0; rph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) { LP_TRACE_MAX(34); LP_TRACE_AT(blockIdx.x == 0, 35); }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

}  // namespace lp

// Grouped expert FFN for decode-size batches (<= 1 routed token per expert on
// average, e.g. the decode-only layers of a layered-prefill iteration): the
// same math as experts_sm100.cuh (HF transformers 5.5 Qwen3MoeExperts.forward,
// modeling_qwen3_moe.py:229-249), cut into twice as many, half-size work items.
//
// With few tokens, only a handful of experts are touched and k_experts' items
// (1 MiB of W13 per UP item) leave most SMs idle while each busy SM streams at
// its own in-flight limit. Here
//   UP (e, m0, nt): 64 act features: A tile = 64 gate rows + the matching 64
//                   up rows (one 128-row tile, ONE accumulator: TMEM lanes
//                   0-63 gate, 64-127 up); the up-lane warps hand their values
//                   to the gate-lane warps through shared memory for SiLU(g)*u.
//   DN (e, m0, nt): 128 W2 rows, one tile.
// Every stage holds two k-blocks (2 x (16 KiB weight tile + 16 token rows)), 5
// stages: about the weight bytes in flight per SM of k_experts while twice as
// many SMs stream, and half the per-stage round trips that pace a decode-size
// stream (TinyCfg). Per output element the K order is unchanged: results are
// bit-identical to k_experts on the same token.
//
// Warp roles (256 threads): w0 TMA producer + scheduler, w1 MMA issuer, w2 TMEM
// allocator + w2-w3 token-row gather (cp.async, as k_experts), w4-w7 epilogue.
#pragma once
#include <cuda_bf16.h>
#include "experts_sm100.cuh"
#include "ptx.cuh"

namespace lp {

struct TinyCfg {
  static constexpr int kThreads = 256;
  static constexpr int kN = 16;                                   // token rows per item (MMA N)
  static constexpr int kBBytes = kN * 128;                        // 2 KiB
  // two k-blocks per ring stage, [A_0 | A_1 | B_0 | B_1] (36 KiB): the stream of a decode-size item is
  // paced per stage, not per byte (decode_sm100.cuh DecodeRing, tools/sm_stream_bench.cu)
  static constexpr int kKS = 2;
  static constexpr int kStageBytes = kKS * (kATileBytes + kBBytes);
  static constexpr int kBOff = kKS * kATileBytes;
  static constexpr int kStages = 5;
  static constexpr int kAcc = 2;
  static constexpr int kTmemCols = 32;                            // 2 x 16 columns
  static constexpr int kXBytes = 64 * kN * 4;                     // up values handed to the gate warps
  static constexpr int kAuxBytes = 8 * (3 * kStages + 1 + 2 * kAcc + 2 * kRing) + 16 * kRing + 16 +
                                   4 * (3 * kMaxExperts + 2);
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kXBytes + kAuxBytes;
  static constexpr int kUpFeat = 64;
  static constexpr int kDnRows = 128;
};

__global__ void __launch_bounds__(TinyCfg::kThreads, 1)
    k_experts_tiny(const __grid_constant__ CUtensorMap tm_w13h, const __grid_constant__ CUtensorMap tm_w2,
                   const __grid_constant__ CUtensorMap tm_act, const ExpertsParams p) {
  using C = TinyCfg;
  constexpr int S_ = C::kStages;
  constexpr int A_ = C::kAcc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* xbuf = reinterpret_cast<float*>(smem + S_ * C::kStageBytes);  // [16 cols][64 lanes]
  constexpr int KS = C::kKS;
  auto a_at = [&](int st, int h) { return smem + st * C::kStageBytes + h * kATileBytes; };
  auto b_at = [&](int st, int h) { return smem + st * C::kStageBytes + C::kBOff + h * C::kBBytes; };
  uint8_t* aux = smem + S_ * C::kStageBytes + C::kXBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);
  uint64_t* empty = full + S_;
  uint64_t* bfull = empty + S_;
  uint64_t* tfull = bfull + ((S_ + 1) & ~1);
  uint64_t* tempty = tfull + A_;
  uint64_t* sfull = tempty + A_;
  uint64_t* sempty = sfull + kRing;
  int4* ring = reinterpret_cast<int4*>(sempty + kRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);
  int32_t* s_off = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_tp = s_off + (kMaxExperts + 1);
  int32_t* s_ts = s_tp + (kMaxExperts + 1);

  const int warp = warp_idx();
  const int lane = threadIdx.x & 31;
  const int E = p.E;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S_; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&bfull[s], kGatherThreads);
    }
    for (int a = 0; a < A_; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    for (int r = 0; r < kRing; ++r) { mbar_init(&sfull[r], 1); mbar_init(&sempty[r], 4); }  // MMA, epi, 2 gather
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { prefetch_tmap(&tm_w13h); prefetch_tmap(&tm_w2); prefetch_tmap(&tm_act); }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  pdl_trigger();
  pdl_wait();
  for (int i = threadIdx.x; i <= E; i += blockDim.x) { s_off[i] = p.offsets[i]; s_tp[i] = p.tile_prefix[i]; }
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_ts[i] = p.tile_rows[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int mt_up = p.I / C::kUpFeat;                           // I % 64 == 0
  const int mt_dn = (p.H + C::kDnRows - 1) / C::kDnRows;
  const int total_tiles = s_tp[E];
  const int n_up = mt_up * total_tiles;
  const int n_items = (mt_up + mt_dn) * total_tiles;

  if (warp == 0) {
    // ===================== scheduler + TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_w = p.weights_evict_first ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_a = policy_evict_last();
      int stage = 0; uint32_t phase = 0;
      int r = 0; uint32_t rph = 0;
      [[maybe_unused]] int n_item = 0;
      while (true) {
        const int it = static_cast<int>(atomicAdd(&p.sched[0], 1u));  // every item claimed dynamically
        LP_ITEM(n_item, 0, static_cast<unsigned long long>(it));
        LP_ITEM(n_item, 1, LP_NOW());
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
          info = make_int4((up ? kItemUp : kItemDown) | (e << 8), mt * (up ? C::kUpFeat : C::kDnRows),
                           s_off[e] + nt * ts, min(ts, n_e - nt * ts));
          need = mt_up * nt_e;
        }
        mbar_wait(&sempty[r], rph ^ 1);
        ring[r] = info;
        mbar_arrive(&sfull[r]);
        if (++r == kRing) { r = 0; rph ^= 1; }
        const int kind = info.x & 0xff;
        if (kind == kItemEnd) break;
        const int e = info.x >> 8, m0 = info.y, row0 = info.z;
        const bool up = kind == kItemUp;
        if (!up) {
          while (ld_acquire_u32(&p.sched[1 + e]) < static_cast<uint32_t>(need)) __nanosleep(64);
          fence_proxy_async_global();
        }
        LP_ITEM(n_item, 2, LP_NOW());
        const int kblocks = up ? p.H / kTileK : p.I / kTileK;
        const uint32_t bytes = kATileBytes + (up ? 0 : C::kBBytes);
        for (int kb0 = 0; kb0 < kblocks; kb0 += KS) {
          const int nh = min(KS, kblocks - kb0);
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], nh * bytes);
          for (int h = 0; h < nh; ++h) {
            uint8_t* sa = a_at(stage, h);
            const int kc = (kb0 + h) * kTileK;
            if (up) {  // rows 0-63: gate features m0..m0+63, rows 64-127: the matching up rows
              tma_load_2d(sa, &tm_w13h, &full[stage], kc, e * 2 * p.I + m0, pol_w);
              tma_load_2d(sa + kATileBytes / 2, &tm_w13h, &full[stage], kc, e * 2 * p.I + p.I + m0, pol_w);
            } else {
              tma_load_2d(sa, &tm_w2, &full[stage], kc, e * p.H + m0, pol_w);
              tma_load_2d(b_at(stage, h), &tm_act, &full[stage], kc, row0, pol_a);
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
    // ===================== MMA issuer =====================
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
        const uint32_t idesc = idesc_bf16_f32(kTileM, (info.w + 15) & ~15);
        const int kblocks = up ? p.H / kTileK : p.I / kTileK;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * C::kN;
        for (int kb0 = 0; kb0 < kblocks; kb0 += KS) {
          mbar_wait(&full[stage], phase);
          mbar_wait(&bfull[stage], phase);
          tc_fence_after();
          for (int h = 0; h < min(KS, kblocks - kb0); ++h) {
            const uint64_t a0 = sdesc_kmajor_sw128(smem_u32(a_at(stage, h)));
            const uint64_t b0 = sdesc_kmajor_sw128(smem_u32(b_at(stage, h)));
            const int kb = kb0 + h;
#pragma unroll
            for (int k = 0; k < kTileK / 16; ++k) mma_bf16(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        if (++acc == A_) { acc = 0; aph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 2 || warp == 3) {
    // ===================== token-row gather (UP items; DN rows come by TMA) =====================
    constexpr int RPT = C::kN / 8;
    const int gt = threadIdx.x - 64;
    const int g = gt >> 3, j = gt & 7;
    const uint64_t pol_x = policy_evict_last();
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
        const int kblocks = p.H / kTileK;
        for (int kb0 = 0; kb0 < kblocks; kb0 += KS) {
          mbar_wait(&empty[stage], phase ^ 1);
          cp_async_wait_group<S_ - 1>();  // this slot's previous copies (S_ groups ago) landed
          for (int h = 0; h < min(KS, kblocks - kb0); ++h) {
            const uint32_t sb = smem_u32(b_at(stage, h)) + sw;
#pragma unroll
            for (int i = 0; i < RPT; ++i)
              if (tok[i] >= 0)
                cp_async16(sb + i * 8 * 128, xs + static_cast<size_t>(tok[i]) * p.H + (kb0 + h) * kTileK, pol_x);
          }
          cp_async_arrive_noinc(&bfull[stage]);
          cp_async_commit();
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      } else {
        for (int kb0 = 0; kb0 < p.I / kTileK; kb0 += KS) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive(&bfull[stage]);
          cp_async_commit();
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp < 8) {
    // ===================== epilogue (w4-w7: TMEM lane quarter q = warp & 3) =====================
    const int q = warp & 3;
    const int et = threadIdx.x - 128;  // 0..127
    int r = 0; uint32_t rph = 0;
    int acc = 0; uint32_t aph = 0;
    [[maybe_unused]] int n_item = 0;
    while (true) {
      mbar_wait(&sfull[r], rph);
      const int4 info = ring[r];
      const int kind = info.x & 0xff;
      if (kind == kItemEnd) break;
      const int e = info.x >> 8, m0 = info.y, row0 = info.z, nvalid = info.w;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
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
      } else {
        const int feat = m0 + 32 * q + lane;
        if (feat < p.H) {
          __nv_bfloat16* dst = p.y_perm + static_cast<size_t>(row0) * p.H + feat;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < nvalid) dst[static_cast<size_t>(i) * p.H] = __float2bfloat16_rn(__uint_as_float(v[i]));
        }
      }
      if (et == 0) {
        mbar_arrive(&sempty[r]);
        if (kind == kItemUp) {  // release: the item's act rows are written
          __threadfence();
          atomicAdd(&p.sched[1 + e], 1u);
        }
        LP_ITEM(n_item, 4, LP_NOW());
      }
      ++n_item;
      if (++r == kRing) { r = 0; rph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

}  // namespace lp

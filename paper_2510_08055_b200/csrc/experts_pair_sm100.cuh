// Grouped expert FFN, compute-bound regime (>= ~100 tokens per expert), on
// CTA pairs (cta_group::2): the same math and item space as experts_sm100.cuh
// (HF transformers 5.5 Qwen3MoeExperts.forward, modeling_qwen3_moe.py:229-249).
//
// An item is one M=256 MMA chain over the pair (cluster of 2 SMs):
//   UP (e, m0, nt): act features m0..m0+255; CTA r holds gate rows and up rows
//                   of features m0+128r..+127 (two A tiles -> two TMEM
//                   accumulators, SiLU(g)*u per thread as in k_experts).
//   DN (e, m0, nt): W2 rows m0..m0+511; CTA r holds rows m0+256r..+255 (two
//                   128-row A tiles).
// The token tile's B rows are split: CTA r stages rows [r*N/2, (r+1)*N/2) and
// the tensor core reads the peer's half over the pair, so per k-block each SM
// receives 2 A tiles + N/2 token rows (48 KiB at N=256) instead of 2 A tiles +
// N rows (64 KiB): 25% fewer L2->SM bytes per MAC and 33% more work in flight
// in the same shared memory. The leader (even rank) schedules items,
// broadcasts them to the peer over DSMEM and issues the MMAs; both CTAs load
// (TMA completing on the leader's barrier) and drain their own TMEM.
//
// Warp roles (384 threads): w0 TMA producer (+ scheduler on the leader), w1 MMA
// issuer (leader), w2 TMEM allocator, w4..w11 epilogue (w4-7 even 16-column
// chunks, w8-11 odd ones).
#pragma once
#include <cuda_bf16.h>
#include "experts_sm100.cuh"
#include "ptx.cuh"

namespace lp {

#ifdef LP_WATCHDOG
// debug builds: a wait that spins ~forever reports who waits on what, then traps
#define PW_LOCAL(bar, par, tag)                                                                            \
  do {                                                                                                     \
    long long n_ = 0;                                                                                      \
    while (!mbar_try_wait((bar), (par)))                                                                   \
      if (++n_ == (1ll << 22)) {                                                                           \
        printf("WATCHDOG %s blk %d rank %u warp %d par %u\n", tag, blockIdx.x, cluster_ctarank(), warp, (par)); \
        break;                                                                                             \
      }                                                                                                    \
  } while (0)
#define PW_CLUSTER(bar, par, tag)                                                                          \
  do {                                                                                                     \
    long long n_ = 0;                                                                                      \
    while (!mbar_try_wait_cluster((bar), (par)))                                                           \
      if (++n_ == (1ll << 22)) {                                                                           \
        printf("WATCHDOG %s blk %d rank %u warp %d par %u\n", tag, blockIdx.x, cluster_ctarank(), warp, (par)); \
        break;                                                                                             \
      }                                                                                                    \
  } while (0)
#else
#define PW_LOCAL(bar, par, tag) mbar_wait((bar), (par))
#define PW_CLUSTER(bar, par, tag) mbar_wait_cluster((bar), (par))
#endif

// BN: token-tile width. 256: one item's two accumulators fill TMEM (single-
// buffered); 128: two items' accumulators fit, so the drain overlaps the next
// item's MMAs at the price of more operand bytes per MAC.
template <int BN>
struct PairCfg {
  static constexpr int kN = BN;                       // tokens per item (MMA N)
  static constexpr int kBRows = kN / 2;               // B rows staged per CTA
  static constexpr int kStageBytes = 2 * kATileBytes + kBRows * 128;
  static constexpr int kStages = BN >= 256 ? 4 : 5;
  static constexpr int kAcc = BN >= 256 ? 1 : 2;      // accumulator sets (gate | up) in TMEM
  static constexpr int kTmemCols = 512;
  static constexpr int kAuxBytes = 8 * (3 * kStages + 1 + 2 * kAcc + 2 * kRing) + 16 * kRing + 16 + 4 * (3 * kMaxExperts + 2);
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kAuxBytes;
  static constexpr int kUpFeat = 128;                 // act features per CTA per UP item
  static constexpr int kDnRows = 256;                 // W2 rows per CTA per DN item
};

// GATHER: UP items' token rows come straight from x (tok_of) through 16-byte
// cp.async by warps 2-3 of each CTA (its half of the tile), as in k_experts'
// memory-bound path; the peer's completions are relayed to the leader's B-full
// barrier by the peer's otherwise idle warp 1. No x_perm is materialised.
template <bool GATHER, int BN>
__global__ void __launch_bounds__(kExpertsThreads, 1)
    k_experts_pair(const __grid_constant__ CUtensorMap tm_w13, const __grid_constant__ CUtensorMap tm_w2,
                   const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_act,
                   const ExpertsParams p) {
  using C = PairCfg<BN>;
  constexpr int S_ = C::kStages;
  constexpr int A_ = C::kAcc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* aux = smem + S_ * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);  // leader's counts both CTAs' bytes
  uint64_t* empty = full + S_;
  uint64_t* tfull = empty + S_;                       // [A_]
  uint64_t* tempty = tfull + A_;                      // [A_] leader's counts both CTAs' epilogue warps
  uint64_t* sfull = tempty + A_;
  uint64_t* sempty = sfull + kRing;                   // leader's counts both CTAs' consumers
  uint64_t* bfull = sempty + kRing;                   // GATHER: this CTA's B half landed (+ peer relay on the leader)
  int4* ring = reinterpret_cast<int4*>(bfull + ((S_ + 1) & ~1));  // 16-byte aligned
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);
  int32_t* s_off = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_tp = s_off + (kMaxExperts + 1);
  int32_t* s_ts = s_tp + (kMaxExperts + 1);

  const int warp = warp_idx();
  const int lane = threadIdx.x & 31;
  const int E = p.E;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S_; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < A_; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 16); }  // 8 epi warps x 2 CTAs
    // ring consumers: MMA + epilogue (leader), producer + epilogue (peer); GATHER adds
    // both CTAs' two gather warps and the peer's relay
    for (int r = 0; r < kRing; ++r) { mbar_init(&sfull[r], 1); mbar_init(&sempty[r], GATHER ? 9 : 4); }
    if (GATHER)
      for (int s = 0; s < S_; ++s) mbar_init(&bfull[s], kGatherThreads + (leader ? 1 : 0));
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_w13); prefetch_tmap(&tm_w2); prefetch_tmap(&tm_x); prefetch_tmap(&tm_act);
  }
  pdl_trigger();
  pdl_wait();
  // TMEM only after the predecessors completed: a CTA holding all 512 columns
  // while it waits could starve a co-resident predecessor CTA's allocation
  if (warp == 2) tmem_alloc_pair(tmem_slot, C::kTmemCols);
  for (int i = threadIdx.x; i <= E; i += blockDim.x) { s_off[i] = p.offsets[i]; s_tp[i] = p.tile_prefix[i]; }
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_ts[i] = p.tile_rows[i];
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive / DSMEM store
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int mt_up = p.I / (2 * C::kUpFeat);
  const int mt_dn = p.H / (2 * C::kDnRows);
  const int total_tiles = s_tp[E];
  const int n_up = mt_up * total_tiles;
  const int n_items = (mt_up + mt_dn) * total_tiles;

  if (warp == 0) {
    // ===================== scheduler (leader) + TMA producer (both CTAs) =====================
    if (lane == 0) {
      const uint64_t pol_w = p.weights_evict_first ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_a = policy_evict_last();
      int stage = 0; uint32_t phase = 0;
      int r = 0; uint32_t rph = 0;
      while (true) {
        int4 info;
        if (leader) {
          // every item is claimed dynamically: a pair only ever waits (DN) on
          // UP items claimed by pairs that are running, whether or not all
          // pairs of the grid are co-resident
          const int it = static_cast<int>(atomicAdd(&p.sched[0], 1u));
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
            info = make_int4((up ? kItemUp : kItemDown) | (e << 8), mt * 2 * (up ? C::kUpFeat : C::kDnRows), row0,
                             nvalid);
          }
          PW_LOCAL(&sempty[r], rph ^ 1, "sched:sempty");
          ring[r] = info;
          st_dsmem_v4(mapa_shared(smem_u32(&ring[r]), 1), info);
          mbar_arrive_remote(mapa_shared(smem_u32(&sfull[r]), 1));  // release: the DSMEM ring store
          mbar_arrive(&sfull[r]);
        } else {
          PW_CLUSTER(&sfull[r], rph, "peerprod:sfull");
          info = ring[r];
          mbar_arrive_remote(mapa_shared(smem_u32(&sempty[r]), 0));
        }
        if (++r == kRing) { r = 0; rph ^= 1; }
        const int kind = info.x & 0xff;
        if (kind == kItemEnd) break;
        const int e = info.x >> 8, m0 = info.y, row0 = info.z, nvalid = info.w;
        const bool up = kind == kItemUp;
        const int half = ((nvalid + 15) & ~15) / 2;  // B rows this CTA stages
        const int nbox = (half + kBoxRows - 1) / kBoxRows;
        const int brow = row0 + static_cast<int>(rank) * half;
        if (!up) {
          const uint32_t need = static_cast<uint32_t>(mt_up * (s_tp[e + 1] - s_tp[e]) * 2);
#ifdef LP_WATCHDOG
          long long n_ = 0;
          while (ld_acquire_u32(&p.sched[1 + e]) < need) {
            __nanosleep(64);
            if (++n_ == (1ll << 22)) {
              printf("WATCHDOG dn-dep blk %d rank %u e %d have %u need %u\n", blockIdx.x, rank, e,
                     ld_acquire_u32(&p.sched[1 + e]), need);
              break;
            }
          }
#else
          while (ld_acquire_u32(&p.sched[1 + e]) < need) __nanosleep(64);
#endif
          fence_proxy_async_global();
        }
        const int kblocks = up ? p.H / kTileK : p.I / kTileK;
        const uint32_t bytes = 2 * (2 * kATileBytes + (GATHER && up ? 0 : nbox * kBoxRows * 128));
        const int f = m0 + static_cast<int>(rank) * (up ? C::kUpFeat : C::kDnRows);
        const int arow = up ? e * 2 * p.I + f : e * p.H + f;
        const int arow2 = up ? arow + p.I : arow + kTileM;
        const CUtensorMap* ta = up ? &tm_w13 : &tm_w2;
        const CUtensorMap* tb = up ? &tm_x : &tm_act;
        for (int kb = 0; kb < kblocks; ++kb) {
          PW_LOCAL(&empty[stage], phase ^ 1, "prod:empty");
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + 2 * kATileBytes;
          if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_2d_pair(sa, ta, &full[stage], kb * kTileK, arow, pol_w);
          tma_load_2d_pair(sa + kATileBytes, ta, &full[stage], kb * kTileK, arow2, pol_w);
          if (!(GATHER && up))
            for (int b = 0; b < nbox; ++b)
              tma_load_2d_pair(sb + b * kBoxRows * 128, tb, &full[stage], kb * kTileK, brow + b * kBoxRows, pol_a);
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer (leader, single thread) =====================
    if (leader && lane == 0) {
      int stage = 0; uint32_t phase = 0;
      int r = 0; uint32_t rph = 0;
      int acc = 0; uint32_t aph = 0;
      while (true) {
        PW_LOCAL(&sfull[r], rph, "mma:sfull");
        const int4 info = ring[r];
        mbar_arrive(&sempty[r]);
        if (++r == kRing) { r = 0; rph ^= 1; }
        const int kind = info.x & 0xff;
        if (kind == kItemEnd) break;
        const bool up = kind == kItemUp;
        const uint32_t idesc = idesc_bf16_f32(256, (info.w + 15) & ~15);
        const int kblocks = up ? p.H / kTileK : p.I / kTileK;
        PW_CLUSTER(&tempty[acc], aph ^ 1, "mma:tempty");
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * 2 * C::kN, d1 = d0 + C::kN;
        for (int kb = 0; kb < kblocks; ++kb) {
          PW_LOCAL(&full[stage], phase, "mma:full");
          if (GATHER) PW_LOCAL(&bfull[stage], phase, "mma:bfull");
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::kStageBytes);
          const uint64_t a0 = sdesc_kmajor_sw128(sa);
          const uint64_t a1 = sdesc_kmajor_sw128(sa + kATileBytes);
          const uint64_t b0 = sdesc_kmajor_sw128(sa + 2 * kATileBytes);
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k) {
            const uint32_t accum = (kb | k) != 0;
            mma_bf16_pair(d0, a0 + 2 * k, b0 + 2 * k, idesc, accum);
            mma_bf16_pair(d1, a1 + 2 * k, b0 + 2 * k, idesc, accum);
          }
          mma_commit_pair(&empty[stage]);
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(&tfull[acc]);
        if (++acc == A_) { acc = 0; aph ^= 1; }
      }
    } else if (GATHER && !leader && lane == 0) {
      // relay: the peer's B half of a stage landed -> arrive on the leader's bfull
      const uint32_t bfull_leader0 = mapa_shared(smem_u32(&bfull[0]), 0);
      const uint32_t sempty_leader0 = mapa_shared(smem_u32(&sempty[0]), 0);
      int stage = 0; uint32_t phase = 0;
      int r = 0; uint32_t rph = 0;
      while (true) {
        PW_CLUSTER(&sfull[r], rph, "relay:sfull");
        const int4 info = ring[r];
        mbar_arrive_remote(sempty_leader0 + r * 8);
        if (++r == kRing) { r = 0; rph ^= 1; }
        const int kind = info.x & 0xff;
        if (kind == kItemEnd) break;
        const int kblocks = kind == kItemUp ? p.H / kTileK : p.I / kTileK;
        for (int kb = 0; kb < kblocks; ++kb) {
          PW_LOCAL(&bfull[stage], phase, "relay:bfull");
          mbar_arrive_remote(bfull_leader0 + stage * 8);
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (GATHER && (warp == 2 || warp == 3)) {
    // ===================== token-row gather (64 threads per CTA, LSU cp.async) =====================
    // Thread (g, j) copies 16-byte chunk j of rows g, g+8, ... of this CTA's
    // half of the token tile into the SWIZZLE_128B layout (chunk slot j ^ g).
    constexpr int RPT = C::kBRows / 8;
    const int gt = threadIdx.x - 64;
    const int g = gt >> 3, j = gt & 7;
    const uint64_t pol_x = policy_evict_last();
    const uint32_t sempty_leader0 = mapa_shared(smem_u32(&sempty[0]), 0);
    int stage = 0; uint32_t phase = 0;
    int r = 0; uint32_t rph = 0;
    while (true) {
      if (leader) PW_LOCAL(&sfull[r], rph, "gather:sfull");
      else PW_CLUSTER(&sfull[r], rph, "gather:sfull");
      const int4 info = ring[r];
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&sempty[r]);
        else mbar_arrive_remote(sempty_leader0 + r * 8);
      }
      if (++r == kRing) { r = 0; rph ^= 1; }
      const int kind = info.x & 0xff;
      if (kind == kItemEnd) break;
      if (kind == kItemUp) {
        const int row0 = info.z, nvalid = info.w;
        const int half = ((nvalid + 15) & ~15) / 2;
        const int base = static_cast<int>(rank) * half;  // first tile row of this CTA's half
        const int mine = min(half, nvalid - base);         // valid rows in this half (may be <= 0)
        int tok[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int rr = g + 8 * i;
          tok[i] = rr < mine ? __ldg(p.tok_of + row0 + base + rr) : -1;
        }
        const __nv_bfloat16* xs = p.xsrc + j * 8;
        const uint32_t sw = static_cast<uint32_t>((j ^ g) << 4) + static_cast<uint32_t>(g * 128);
        for (int kb = 0; kb < p.H / kTileK; ++kb) {
          PW_LOCAL(&empty[stage], phase ^ 1, "gather:empty");
          cp_async_wait_group<S_ - 1>();  // this slot's previous copies (S_ groups ago) landed
          const uint32_t sb = smem_u32(smem + stage * C::kStageBytes + 2 * kATileBytes) + sw;
#pragma unroll
          for (int i = 0; i < RPT; ++i)
            if (tok[i] >= 0) cp_async16(sb + i * 8 * 128, xs + static_cast<size_t>(tok[i]) * p.H + kb * kTileK, pol_x);
          cp_async_arrive_noinc(&bfull[stage]);
          cp_async_commit();
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      } else {  // DN items: B comes by TMA; keep bfull's phases in step
        for (int kb = 0; kb < p.I / kTileK; ++kb) {
          PW_LOCAL(&empty[stage], phase ^ 1, "gather:empty");
          mbar_arrive(&bfull[stage]);
          cp_async_commit();  // (empty group: one group per stage)
          if (++stage == S_) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> regs -> global =====================
    const int q = warp & 3;             // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;   // 0: even chunks, 1: odd chunks
    const int et = threadIdx.x - 128;   // 0..255
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t sempty_leader0 = mapa_shared(smem_u32(&sempty[0]), 0);
    int r = 0; uint32_t rph = 0;
    int acc = 0; uint32_t aph = 0;
    while (true) {
      if (leader) PW_LOCAL(&sfull[r], rph, "epi:sfull");
      else PW_CLUSTER(&sfull[r], rph, "peerepi:sfull");
      const int4 info = ring[r];
      const int kind = info.x & 0xff;
      if (kind == kItemEnd) break;
      const int e = info.x >> 8, m0 = info.y, row0 = info.z, nvalid = info.w;
      PW_LOCAL(&tfull[acc], aph, "epi:tfull");
      tc_fence_after();
      const uint32_t t0 = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * 2 * C::kN;
      // 32-column TMEM loads: one wait per 32 tokens (the drain is on the MMA's critical path)
      const int nchunks32 = (nvalid + 31) / 32;
      if (kind == kItemUp) {
        const int feat = m0 + static_cast<int>(rank) * C::kUpFeat + 32 * q + lane;
        __nv_bfloat16* dst = p.act + static_cast<size_t>(row0) * p.I + feat;
        for (int c = half; c < nchunks32; c += 2) {
          uint32_t g[32], u[32];
          tmem_ld32(t0 + c * 32, g);
          tmem_ld32(t0 + C::kN + c * 32, u);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int n = c * 32 + i;
            if (n < nvalid)
              dst[static_cast<size_t>(n) * p.I] =
                  __float2bfloat16_rn(silu_mul(__uint_as_float(g[i]), __uint_as_float(u[i])));
          }
        }
      } else {
        const int feat = m0 + static_cast<int>(rank) * C::kDnRows + 32 * q + lane;
        __nv_bfloat16* dst = p.y_perm + static_cast<size_t>(row0) * p.H + feat;
        for (int c = half; c < nchunks32; c += 2) {
          uint32_t v[32], v2[32];
          tmem_ld32(t0 + c * 32, v);
          tmem_ld32(t0 + C::kN + c * 32, v2);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int n = c * 32 + i;
            if (n < nvalid) {
              dst[static_cast<size_t>(n) * p.H] = __float2bfloat16_rn(__uint_as_float(v[i]));
              dst[static_cast<size_t>(n) * p.H + kTileM] = __float2bfloat16_rn(__uint_as_float(v2[i]));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty[acc]);
        else mbar_arrive_remote(tempty_leader0 + acc * 8);
      }
      if (++acc == A_) { acc = 0; aph ^= 1; }
      if (kind == kItemUp) {
        fence_proxy_async_global();       // act rows are read back through TMA (async proxy)
        named_bar_sync(1, kEpiThreads);   // every thread's act stores precede the count
      }
      if (et == 0) {
        if (leader) mbar_arrive(&sempty[r]);
        else mbar_arrive_remote(sempty_leader0 + r * 8);
        if (kind == kItemUp) {  // release: this CTA's act rows of the item are written
          __threadfence();
          atomicAdd(&p.sched[1 + e], 1u);
        }
      }
      if (++r == kRing) { r = 0; rph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its pair may still touch its smem / TMEM / barriers
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::kTmemCols);
  }
}

}  // namespace lp

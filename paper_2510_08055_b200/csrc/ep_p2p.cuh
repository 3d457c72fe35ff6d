// Expert parallelism over peer memory (NVLink / NVSwitch P2P through CUDA IPC
// mappings): the dispatch and return all-to-alls of ep.py's NCCL path folded
// into the permutation and the combine.
//
// Every rank exposes, at the same logical layout, a control block (barrier
// counter, double-buffered count inbox + ready tags), a receive buffer
// recv_x [cap, H] and its expert outputs y_out [cap, H]; the other ranks hold
// mapped pointers to them (device arrays of P pointers). Per layer, rank r
// (P ranks, E = P * El experts), 6 launches after route + permute:
//   1. route + local slot order (liblpmoe route / permute, index-only)
//   2. k_ep_exchange: r's counts -> every rank's inbox, release a ready tag,
//      wait for every source's tag in r's own block, then plan: r's first row
//      in each owner's receive buffer per expert (rows are expert-major,
//      source-major within an expert, source order within a source: the
//      layout a single-GPU x_perm of the concatenated batch would have per
//      expert), and r's own expert offsets
//   3. k_ep_dispatch: token rows stored straight into the owners' recv_x
//      (fused permute + send, no staging buffer)
//   4. barrier; owners run the expert kernel on recv_x -> y_out
//   5. barrier; k_ep_combine: y[t] = sum_j w[t,j] * y_out_d[row] read straight
//      from the owners (fused receive + weighted combine, fixed j order)
// No end-of-layer barrier: a source writes an owner's recv_x again only after
// the next layer's exchange saw the owner's tag (posted after its expert
// kernel), and an owner rewrites y_out only after the next dispatch barrier
// (every source has finished its combine). Barriers are device-side: each rank
// adds 1 to every rank's counter with a system-scope release and spins on its
// own with a system-scope acquire; the barrier and layer sequence numbers live
// in device memory, so a layer is CUDA-graph capturable.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include "ptx.cuh"

namespace lp {

__device__ __forceinline__ void red_add_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
// Spin with relaxed system-scope polls, then one acquire fence (an acquire per poll is slower)
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// Per-rank control block (the first lp_ep_ctl_bytes(P, E) bytes of a rank's region):
//   u32 [0]  barrier counter (peers add to it)      u32 [1]  barriers this rank passed (own)
//   u32 [2]  layers this rank exchanged (own)       u32 [64 + 2*parity + ...] ready tags, [2][P]
//   int32 inbox [2][P src][E] at byte kCtlInbox      (parity = layer & 1: double-buffered)
constexpr int kCtlReadyWord = 64;
constexpr int kCtlInbox = 512;
constexpr int kEpMaxRanks = 32;

// One warp: signal every rank, then wait until this rank's counter reaches P x (barriers so
// far, kept on the device in ctl[1], so a captured CUDA graph replays correctly). Counters only
// grow; no rank can arrive at barrier n+1 before every rank arrived at barrier n.
__global__ void k_ep_barrier(uint32_t* const* __restrict__ peer_ctl, int P, int rank) {
  pdl_trigger();  // (PDL: the next kernel's prologue may start; it waits for this grid before its data)
  pdl_wait();
  const int lane = threadIdx.x;
  uint32_t* mine = peer_ctl[rank];
  if (lane == 0) __threadfence_system();  // the preceding kernels' peer stores, before the release adds
  __syncwarp();
  for (int q = lane; q < P; q += 32) red_add_release_sys(peer_ctl[q], 1u);
  if (lane == 0) {
    const uint32_t n = mine[1] + 1u;
    const uint32_t target = static_cast<uint32_t>(P) * n;
    while (static_cast<int32_t>(ld_relaxed_sys(mine) - target) < 0) {
    }
    fence_acq_rel_sys();
    mine[1] = n;
  }
  __syncwarp();
}

__device__ __forceinline__ void st_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

// Count exchange + plan in ONE launch (one CTA; replaces post-counts, a full barrier and the
// plan kernel). This rank's per-global-expert counts go to every rank's inbox[parity][rank],
// followed by a system-scope release of ready[parity][rank] = layer + 1; the CTA then waits for
// every source's tag in its OWN control block and plans from its own inbox:
//   dest_base[d*El+el]: first row of (source = rank, expert el of d) in d's receive buffer
//     (rows expert-major, source-rank-major within an expert, source order within a source);
//   off_local[0..El]: this rank's expert offsets over all sources (off_local[El] = rows received).
// Reusing inbox[parity] two layers later is safe: a rank posts layer n+2 only after its
// exchange of layer n+1 saw every peer's tag n+2, which each peer posts after planning layer n.
__global__ void __launch_bounds__(1024)
    k_ep_exchange(const int32_t* __restrict__ counts, uint32_t* const* __restrict__ peer_ctl, int P, int El,
                  int rank, int32_t* __restrict__ dest_base, int32_t* __restrict__ off_local,
                  int32_t* __restrict__ rows_out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ int32_t s_cnt[];  // [P src][E]
  __shared__ uint32_t s_layer;
  const int E = P * El;
  uint32_t* mine = peer_ctl[rank];
  if (threadIdx.x == 0) s_layer = mine[2];
  __syncthreads();
  const uint32_t layer = s_layer;
  const int parity = static_cast<int>(layer & 1u);
  const size_t box = static_cast<size_t>(parity) * P * E + static_cast<size_t>(rank) * E;
  for (int i = threadIdx.x; i < P * E; i += blockDim.x) {
    const int d = i / E, e = i - d * E;
    reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(peer_ctl[d]) + kCtlInbox)[box + e] = counts[e];
  }
  // one system-scope fence after the CTA barrier publishes every thread's inbox stores (cumulativity);
  // a fence per thread cost ~35 us per launch
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
  __syncthreads();
  if (threadIdx.x < P && threadIdx.x != rank)
    st_release_sys(peer_ctl[threadIdx.x] + kCtlReadyWord + parity * kEpMaxRanks + rank, layer + 1u);
  if (threadIdx.x < P && threadIdx.x != rank) {  // (this rank's own counts: ordered by the CTA barrier)
    const uint32_t* tag = mine + kCtlReadyWord + parity * kEpMaxRanks + threadIdx.x;
    while (ld_relaxed_sys(tag) != layer + 1u) {
    }
    fence_acq_rel_sys();
  }
  __syncthreads();
  const int32_t* inbox = reinterpret_cast<const int32_t*>(reinterpret_cast<const uint8_t*>(mine) + kCtlInbox) +
                         static_cast<size_t>(parity) * P * E;
  for (int i = threadIdx.x; i < P * E; i += blockDim.x) s_cnt[i] = __ldcv(inbox + i);  // L1 may hold layer n-2
  __syncthreads();
  // plan with one block-wide scan (E <= 256 = blockDim experts): tot[e] = rows of expert e over all
  // sources; incl[e] = inclusive prefix of tot; the prefix within owner d's block of El experts is
  // incl[e] - tot[e] - incl[d*El - 1]
  __shared__ int32_t s_incl[256];
  __shared__ int32_t s_warp[8];
  const int t = threadIdx.x;
  int tot = 0, before = 0;
  if (t < E) {
    for (int s2 = 0; s2 < P; ++s2) {
      const int c = s_cnt[s2 * E + t];
      tot += c;
      if (s2 < rank) before += c;
    }
  }
  int incl = tot;
  const int lane = t & 31, wid = t >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  for (int w2 = 0; w2 < wid; ++w2) incl += s_warp[w2];
  if (t < E) s_incl[t] = incl;
  __syncthreads();
  if (t < E) {
    const int d = t / El;
    const int blk0 = d * El > 0 ? s_incl[d * El - 1] : 0;
    const int excl_blk = incl - tot - blk0;  // rows of experts d*El .. t-1 (all sources)
    dest_base[t] = excl_blk + before;
    if (d == rank) off_local[t - rank * El] = excl_blk;
    if (t == (rank + 1) * El - 1) {
      off_local[El] = incl - blk0;
      if (rows_out != nullptr) *rows_out = incl - blk0;  // the caller's copy (off_local is rewritten next layer)
    }
  }
  if (threadIdx.x == 0) mine[2] = layer + 1u;
}

// Warp per routing entry i = t * topk + j: the token row goes straight into
// the owner's receive buffer at its planned row; (dest_rank, dest_row) are
// kept for the combine.
__global__ void __launch_bounds__(256)
    k_ep_dispatch(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ ids,
                  const int32_t* __restrict__ slot_of, const int32_t* __restrict__ offsets,
                  const int32_t* __restrict__ dest_base, __nv_bfloat16* const* __restrict__ peer_recv, int S, int H,
                  int topk, int El, int32_t* __restrict__ dest_rank, int32_t* __restrict__ dest_row) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (i < S) {
    const int e = ids[i];
    const int d = e / El, el = e - d * El;
    const int row = dest_base[d * El + el] + (slot_of[i] - offsets[e]);
    if (lane == 0) {
      dest_rank[i] = d;
      dest_row[i] = row;
    }
    const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(i / topk) * H);
    uint4* dst = reinterpret_cast<uint4*>(peer_recv[d] + static_cast<size_t>(row) * H);
    for (int v = lane; v < H / 8; v += 32) dst[v] = src[v];
  }
  __syncthreads();  // one fence per CTA (after the barrier) instead of one per thread
  if (threadIdx.x == 0) __threadfence_system();
}

// CTA per token: y[t] = sum_j w[t,j] * y_out_{dest_rank}[dest_row] (fp32, fixed j order), with
// up to eight of the token's rows in flight per thread (L1 bypassed: the owners rewrite y_out
// every layer).
__global__ void __launch_bounds__(256)
    k_ep_combine(__nv_bfloat16* const* __restrict__ peer_y, const int32_t* __restrict__ dest_rank,
                 const int32_t* __restrict__ dest_row, const float* __restrict__ w, int T, int topk, int H,
                 __nv_bfloat16* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  __shared__ const uint4* s_row[32];
  __shared__ float s_w[32];
  if (threadIdx.x < topk) {
    const int i = t * topk + threadIdx.x;
    s_row[threadIdx.x] = reinterpret_cast<const uint4*>(peer_y[dest_rank[i]] + static_cast<size_t>(dest_row[i]) * H);
    s_w[threadIdx.x] = w[i];
  }
  __syncthreads();
  for (int v = threadIdx.x; v < H / 8; v += blockDim.x) {
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    for (int j0 = 0; j0 < topk; j0 += 8) {
      uint4 d[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < topk) d[u] = __ldcg(s_row[j0 + u] + v);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j0 + u < topk) {
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&d[u]);
          const float wj = s_w[j0 + u];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __bfloat1622float2(h2[q]);
            acc[2 * q] += wj * f.x;
            acc[2 * q + 1] += wj * f.y;
          }
        }
      }
    }
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) o2[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
    reinterpret_cast<uint4*>(y + static_cast<size_t>(t) * H)[v] = o;
  }
}

}  // namespace lp

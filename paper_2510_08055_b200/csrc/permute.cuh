// K2: per-expert histogram, exclusive prefix sum, stable permutation and
// token gather; K4: weighted combine.
//
// Slot order is the stable counting sort of the flattened routing entries
// i = t*topk + j by expert id: slots [offsets[e], offsets[e+1]) hold expert
// e's entries in increasing i. This is the order HF's per-expert loop visits
// tokens (`torch.where(expert_mask[e])`, modeling_qwen3_moe.py:243) and the
// order the oracle's stable argsort produces, so slot_of is bit-exact.
//
// Chunks are the router's token tiles (16 or 64 tokens): the router kernel (route.cuh) emits
// each tile's expert histogram and in-tile stable ranks. One single-block scan
// kernel turns the per-tile counts into per-tile bases (fixed order), the
// expert offsets, every entry's slot (slot_of) and its inverse (tok_of), the
// token-tile schedule the expert kernel consumes, and resets the expert
// kernel's scheduler words (the whole layer stays graph-capturable).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include "ptx.cuh"

namespace lp {

constexpr int kHistWarps = 4;

// Standalone permutation path (ids supplied by the caller): per tile of
// kRouterN tokens (chunk = kRouterN*topk entries) the same stable histogram +
// in-tile ranks the router kernel produces. One warp per tile.
__global__ void __launch_bounds__(32 * kHistWarps)
    k_chunk_hist(const int32_t* __restrict__ ids, int S, int E, int chunk, int32_t* __restrict__ chunk_hist,
                 int32_t* __restrict__ rank_local) {
  extern __shared__ int32_t sh_hist[];
  const int wl = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kHistWarps + wl;
  pdl_trigger();
  pdl_wait();
  int32_t* hist = sh_hist + wl * E;
  for (int e = lane; e < E; e += 32) hist[e] = 0;
  __syncwarp();
  const int nchunks = (S + chunk - 1) / chunk;
  if (c < nchunks) {
    const unsigned lt = (1u << lane) - 1u;
    for (int s = 0; s < chunk; s += 32) {
      const int i = c * chunk + s + lane;
      const int e = (s + lane < chunk && i < S) ? ids[i] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      int base = 0;
      if (e >= 0) base = hist[e];
      __syncwarp();
      if (e >= 0) {
        rank_local[i] = base + __popc(peers & lt);
        if ((__ffs(peers) - 1) == lane) hist[e] = base + __popc(peers);
      }
      __syncwarp();
    }
    for (int e = lane; e < E; e += 32) chunk_hist[static_cast<size_t>(c) * E + e] = hist[e];
  }
}

// Single block of 1024 threads. The per-tile histograms are staged in shared
// memory when they fit (nchunks*E <= kScanSmemInts, i.e. T <= ~3k tokens for
// E=128), otherwise scanned in place in global memory. G = 1024/E_pad groups of
// E_pad threads; group g owns a contiguous range of tiles: pass 1 sums the
// range, the G partial sums are scanned, pass 2 rewrites the histograms as
// per-tile exclusive bases (fixed order). Then offsets, every entry's slot
// (slot_of) and inverse (tok_of), the expert kernel's token-tile schedule, and
// the reset of its scheduler words.
constexpr int kScanThreads = 1024;
constexpr int kScanSmemInts = 24576;  // 96 KiB

__global__ void __launch_bounds__(kScanThreads)
    k_scan(int32_t* __restrict__ chunk_hist, int nchunks, int E, int max_n, int32_t* __restrict__ counts,
           int32_t* __restrict__ offsets, int32_t* __restrict__ tile_prefix, int32_t* __restrict__ tile_rows,
           uint32_t* __restrict__ sched, uint32_t* __restrict__ zero_buf, int zero_n) {
  extern __shared__ int32_t s_hist[];
  __shared__ int32_t s_part[kScanThreads];
  __shared__ int32_t s_cnt[256];
  __shared__ int32_t s_til[256];
  const int tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();
  if (tid == 0) LP_TRACE_AT(true, 16);
  const int e_pad = (E + 31) & ~31;
  const int G = kScanThreads / e_pad;
  const int g = tid / e_pad;
  const int e = tid % e_pad;
  const int n_hist = nchunks * E;
  const bool staged = n_hist <= kScanSmemInts;
  int32_t* hist = staged ? s_hist : chunk_hist;
  if (staged) {
    for (int i = tid; i < n_hist; i += 4 * kScanThreads) {
      int v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (i + u * kScanThreads < n_hist) ? __ldcg(chunk_hist + i + u * kScanThreads) : 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * kScanThreads < n_hist) s_hist[i + u * kScanThreads] = v[u];
    }
    __syncthreads();
  }
  if (tid == 0) LP_TRACE_AT(true, 17);
  const int per = (nchunks + G - 1) / G;
  const int c0 = min(g * per, nchunks), c1 = min(c0 + per, nchunks);
  int sum = 0;
  if (g < G && e < E) {
    for (int c = c0; c < c1; ++c) sum += staged ? hist[c * E + e] : __ldcg(hist + static_cast<size_t>(c) * E + e);
  }
  if (g < G) s_part[g * e_pad + e] = sum;
  __syncthreads();
  if (tid < e_pad) {
    int run = 0;
    for (int gg = 0; gg < G; ++gg) {
      const int v = s_part[gg * e_pad + tid];
      s_part[gg * e_pad + tid] = run;
      run += v;
    }
    s_cnt[tid] = (tid < E) ? run : 0;
  }
  __syncthreads();
  if (g < G && e < E) {
    int run = s_part[g * e_pad + e];
    for (int c = c0; c < c1; ++c) {
      const size_t at = static_cast<size_t>(c) * E + e;
      const int v = staged ? hist[at] : __ldcg(hist + at);
      hist[at] = run;
      run += v;
    }
  }
  // offsets / tile schedule over experts: warp-shuffle scans (e_pad <= 256 -> <= 8 warps)
  int cnt = 0, ntiles = 0;
  if (tid < e_pad) {
    cnt = s_cnt[tid];
    ntiles = (cnt > 0) ? (cnt + max_n - 1) / max_n : 0;
    if (tid < E) counts[tid] = cnt;
    int a = cnt, b = ntiles;
    const int lane = tid & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ua = __shfl_up_sync(0xffffffffu, a, o);
      const int ub = __shfl_up_sync(0xffffffffu, b, o);
      if (lane >= o) { a += ua; b += ub; }
    }
    s_cnt[tid] = a;  // inclusive within the warp
    s_til[tid] = b;
  }
  __syncthreads();
  if (tid < e_pad) {
    int wa = 0, wb = 0;
    for (int w = 0; w < (tid >> 5); ++w) { wa += s_cnt[w * 32 + 31]; wb += s_til[w * 32 + 31]; }
    const int inc_a = s_cnt[tid] + wa, inc_b = s_til[tid] + wb;
    if (tid < E) {
      offsets[tid] = inc_a - cnt;
      tile_prefix[tid] = inc_b - ntiles;
      const int rows = ntiles ? (cnt + ntiles - 1) / ntiles : 0;
      tile_rows[tid] = min(max_n, (rows + 15) & ~15);
      if (tid == E - 1) {
        offsets[E] = inc_a;
        tile_prefix[E] = inc_b;
      }
    }
  }
  for (int i = tid; i <= E; i += kScanThreads) sched[i] = 0u;
  // fused-combine counters of the expert kernel start from zero (256-B aligned region)
  for (int i = tid; i < zero_n / 4; i += kScanThreads) reinterpret_cast<uint4*>(zero_buf)[i] = make_uint4(0, 0, 0, 0);
  for (int i = (zero_n / 4) * 4 + tid; i < zero_n; i += kScanThreads) zero_buf[i] = 0u;
  if (!staged) return;
  // staged path: the per-tile bases live in smem; publish them for the scatter
  __syncthreads();
  for (int i = tid; i < n_hist; i += kScanThreads) chunk_hist[i] = s_hist[i];
  if (tid == 0) LP_TRACE_AT(true, 18);
}

// One warp per token t: lane j < topk computes the expert-contiguous slot of
// routing entry t*topk + j and the inverse map; the warp then reads token row
// t once (8 x 16 B per lane in flight) and writes it to its topk slots of x_perm.
__global__ void __launch_bounds__(256)
    k_scatter(const int32_t* __restrict__ ids, const int32_t* __restrict__ chunk_base,
              const int32_t* __restrict__ rank_local, const int32_t* __restrict__ offsets,
              const __nv_bfloat16* __restrict__ x, int S, int E, int topk, int H, int chunk,
              int32_t* __restrict__ slot_of, int32_t* __restrict__ tok_of, __nv_bfloat16* __restrict__ x_perm) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) LP_TRACE_MIN(24);
  if (t * topk >= S) return;
  int slot = 0;
  if (lane < topk) {
    const int i = t * topk + lane;
    const int e = __ldcg(ids + i);
    slot = __ldcg(offsets + e) + __ldcg(chunk_base + static_cast<size_t>(i / chunk) * E + e) + __ldcg(rank_local + i);
    slot_of[i] = slot;
    tok_of[slot] = t;
  }
  if (x_perm != nullptr) {
    const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * H);
    const int nv = H / 8;
    for (int v0 = 0; v0 < nv; v0 += 8 * 32) {
      uint4 r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (v0 + u * 32 + lane < nv) r[u] = __ldg(src + v0 + u * 32 + lane);
      for (int j = 0; j < topk; ++j) {
        const int sj = __shfl_sync(0xffffffffu, slot, j);
        uint4* dst = reinterpret_cast<uint4*>(x_perm + static_cast<size_t>(sj) * H);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (v0 + u * 32 + lane < nv) dst[v0 + u * 32 + lane] = r[u];
      }
    }
  }
  if (lane == 0) LP_TRACE_MAX(25);
}

// Index-only scatter (token rows are gathered later by the expert kernel):
// one thread per routing entry.
__global__ void __launch_bounds__(256)
    k_slots(const int32_t* __restrict__ ids, const int32_t* __restrict__ chunk_base,
            const int32_t* __restrict__ rank_local, const int32_t* __restrict__ offsets, int S, int E, int topk,
            int chunk, int32_t* __restrict__ slot_of, int32_t* __restrict__ tok_of) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (threadIdx.x == 0) LP_TRACE_MIN(24);
  if (i >= S) return;
  const int e = __ldcg(ids + i);
  const int slot = __ldcg(offsets + e) + __ldcg(chunk_base + static_cast<size_t>(i / chunk) * E + e) +
                   __ldcg(rank_local + i);
  slot_of[i] = slot;
  tok_of[slot] = i / topk;
  if (threadIdx.x == 0) LP_TRACE_MAX(25);
}

// Scan + slot maps in one launch, straight from the routing ids (gather path:
// no x_perm; the router then skips its per-tile histogram). Every CTA owns 512
// routing entries. It histograms ALL entries (totals -> offsets) and those
// before its own (the base of each expert's run; smem atomics), and ranks its own entries
// stably (match_any within a warp, exclusive scan over the 16 warps), so
//   slot(i) = offsets[e] + #{j < i : ids[j] = e}
// — the stable counting sort, identical to k_scan + k_slots. CTA 0 also
// publishes counts / offsets and the expert kernel's token-tile schedule and
// resets its scheduler words. Latency-bound: loads are issued in batches.
constexpr int kScanSlotsThreads = 512;
__global__ void __launch_bounds__(kScanSlotsThreads)
    k_scan_slots(const int32_t* __restrict__ ids, int S, int E, int topk, int max_n, int32_t* __restrict__ counts,
                 int32_t* __restrict__ offsets, int32_t* __restrict__ tile_prefix, int32_t* __restrict__ tile_rows,
                 uint32_t* __restrict__ sched, int32_t* __restrict__ slot_of, int32_t* __restrict__ tok_of) {
  constexpr int NT = kScanSlotsThreads, NW = NT / 32;
  __shared__ int32_t s_pre[256], s_tot[256], s_off[256], s_ws[2][NW];
  __shared__ int32_t s_wh[NW][256];
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) LP_TRACE_MIN(24);
  const int i0 = blockIdx.x * NT;
  const int i = i0 + tid;
  const int ex = i < S ? __ldcg(ids + i) : -1;
  for (int k = tid; k < 256; k += NT) { s_pre[k] = 0; s_tot[k] = 0; }
  for (int k = tid; k < NW * 256; k += NT) (&s_wh[0][0])[k] = 0;
  __syncthreads();
  // (1) histograms of all entries and of the entries before this CTA's (smem atomics)
  for (int j0 = 0; j0 < S; j0 += 8 * NT) {
    int v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u * NT + tid;
      v[u] = j < S ? __ldcg(ids + j) : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u * NT + tid;
      if (v[u] >= 0) {
        atomicAdd(&s_tot[v[u]], 1);
        if (j < i0) atomicAdd(&s_pre[v[u]], 1);
      }
    }
  }
  // (2) stable rank of this CTA's entries: within the warp, then across warps
  const unsigned peers = __match_any_sync(0xffffffffu, ex);
  const int rank_w = __popc(peers & ((1u << lane) - 1u));
  if (ex >= 0 && (__ffs(peers) - 1) == lane) s_wh[wid][ex] = __popc(peers);
  __syncthreads();
  const int e_pad = (E + 31) & ~31;
  if (tid < e_pad) {
    int run = s_pre[tid];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int c = s_wh[w][tid];
      s_wh[w][tid] = run;
      run += c;
    }
  }
  // (3) offsets and the tile schedule over experts (block scan over <= 256 experts)
  const int cnt = (tid < E) ? s_tot[tid] : 0;
  const int ntiles = (cnt > 0) ? (cnt + max_n - 1) / max_n : 0;
  int a = cnt, b = ntiles;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ua = __shfl_up_sync(0xffffffffu, a, o);
    const int ub = __shfl_up_sync(0xffffffffu, b, o);
    if (lane >= o) { a += ua; b += ub; }
  }
  if (lane == 31) { s_ws[0][wid] = a; s_ws[1][wid] = b; }
  __syncthreads();
  if (tid < 256) {
    int wa = 0, wb = 0;
    for (int w = 0; w < wid; ++w) { wa += s_ws[0][w]; wb += s_ws[1][w]; }
    const int inc_a = a + wa, inc_b = b + wb;
    s_off[tid] = inc_a - cnt;
    if (blockIdx.x == 0 && tid < E) {
      counts[tid] = cnt;
      offsets[tid] = inc_a - cnt;
      tile_prefix[tid] = inc_b - ntiles;
      const int rows = ntiles ? (cnt + ntiles - 1) / ntiles : 0;
      tile_rows[tid] = min(max_n, (rows + 15) & ~15);
      if (tid == E - 1) { offsets[E] = inc_a; tile_prefix[E] = inc_b; }
    }
  }
  if (blockIdx.x == 0)
    for (int k = tid; k <= E; k += NT) sched[k] = 0u;
  __syncthreads();
  // (4) this CTA's entries
  if (ex >= 0) {
    const int slot = s_off[ex] + s_wh[wid][ex] + rank_w;
    slot_of[i] = slot;
    tok_of[slot] = i / topk;
  }
  if (tid == 0) LP_TRACE_MAX(25);
}

// x_perm[slot] = x[tok_of[slot]] (standalone lp_moe_permute only; the fused
// forward never materialises x_perm — the expert kernel gathers rows by TMA).
__global__ void __launch_bounds__(256)
    k_gather_rows(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ tok_of, int S, int H,
                  __nv_bfloat16* __restrict__ x_perm) {
  const int slot = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) { LP_TRACE_MIN(24); }
  if (slot >= S) return;
  const int t = tok_of[slot];
  const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * H);
  uint4* dst = reinterpret_cast<uint4*>(x_perm + static_cast<size_t>(slot) * H);
  for (int v = lane; v < H / 8; v += 32) dst[v] = src[v];
  if (lane == 0) LP_TRACE_MAX(25);
}

// y[t] = sum_j w[t,j] * y_perm[slot_of[t,j]]   (fp32 accumulate in fixed j order, bf16 out)
// One CTA per token; each thread owns 8 consecutive features and keeps all
// topk row loads in flight.
constexpr int kCombineThreads = 256;
__global__ void __launch_bounds__(kCombineThreads)
    k_combine(const __nv_bfloat16* __restrict__ y_perm, const int32_t* __restrict__ slot_of,
              const float* __restrict__ w, int T, int topk, int H, __nv_bfloat16* __restrict__ y) {
  __shared__ int s_slot[32];
  __shared__ float s_w[32];
  const int t = blockIdx.x;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) LP_TRACE_MIN(40);
  if (threadIdx.x < topk) {
    s_slot[threadIdx.x] = slot_of[static_cast<size_t>(t) * topk + threadIdx.x];
    s_w[threadIdx.x] = w[static_cast<size_t>(t) * topk + threadIdx.x];
  }
  __syncthreads();
  const int nv = H / 8;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    int j = 0;
    for (; j + 8 <= topk; j += 8) {  // eight rows in flight
      uint4 d[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        d[u] = __ldcs(reinterpret_cast<const uint4*>(y_perm + static_cast<size_t>(s_slot[j + u]) * H) + v);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&d[u]);
        const float wj = s_w[j + u];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(h2[q]);
          acc[2 * q] += wj * f.x;
          acc[2 * q + 1] += wj * f.y;
        }
      }
    }
    for (; j + 4 <= topk; j += 4) {
      uint4 d[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        d[u] = __ldcg(reinterpret_cast<const uint4*>(y_perm + static_cast<size_t>(s_slot[j + u]) * H) + v);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&d[u]);
        const float wj = s_w[j + u];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(h2[q]);
          acc[2 * q] += wj * f.x;
          acc[2 * q + 1] += wj * f.y;
        }
      }
    }
    for (; j < topk; ++j) {
      const uint4 d = __ldcg(reinterpret_cast<const uint4*>(y_perm + static_cast<size_t>(s_slot[j]) * H) + v);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&d);
      const float wj = s_w[j];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h2[q]);
        acc[2 * q] += wj * f.x;
        acc[2 * q + 1] += wj * f.y;
      }
    }
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) o2[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
    reinterpret_cast<uint4*>(y + static_cast<size_t>(t) * H)[v] = o;
  }
  if (threadIdx.x == 0) LP_TRACE_MAX(41);
}

}  // namespace lp

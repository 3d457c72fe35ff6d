// K2: per-expert histogram, exclusive prefix sum, stable permutation and
// token gather; K4: weighted combine.
//
// Slot order is the stable counting sort of the flattened routing entries
// i = t*topk + j by expert id: slots [offsets[e], offsets[e+1]) hold expert
// e's entries in increasing i. This is the order HF's per-expert loop visits
// tokens (`torch.where(expert_mask[e])`, modeling_qwen3_moe.py:243) and the
// order the oracle's stable argsort produces, so slot_of is bit-exact.
//
// Histogram: one warp per chunk of kChunk entries, __match_any_sync for the
// in-warp rank, a per-warp smem counter table for the running rank. The scan
// kernel turns per-chunk counts into per-chunk bases (fixed order), computes
// offsets and the token-tile schedule the expert kernel consumes, and resets
// the expert kernel's scheduler words (so the whole layer stays graph-capturable).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace lp {

constexpr int kChunk = 512;          // routing entries per histogram warp
constexpr int kHistWarps = 4;

__global__ void __launch_bounds__(32 * kHistWarps)
    k_chunk_hist(const int32_t* __restrict__ ids, int S, int E, int32_t* __restrict__ chunk_hist,
                 int32_t* __restrict__ rank_local) {
  extern __shared__ int32_t sh_hist[];
  const int wl = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kHistWarps + wl;
  int32_t* hist = sh_hist + wl * E;
  for (int e = lane; e < E; e += 32) hist[e] = 0;
  __syncwarp();
  const int nchunks = (S + kChunk - 1) / kChunk;
  if (c < nchunks) {
    const unsigned lt = (1u << lane) - 1u;
    for (int s = 0; s < kChunk; s += 32) {
      const int i = c * kChunk + s + lane;
      const int e = (i < S) ? ids[i] : -1;
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

// Single block, one thread per expert (E <= blockDim.x <= 1024).
__global__ void k_scan(int32_t* __restrict__ chunk_hist, int nchunks, int E, int max_n,
                       int32_t* __restrict__ counts, int32_t* __restrict__ offsets,
                       int32_t* __restrict__ tile_prefix, int32_t* __restrict__ tile_rows,
                       uint32_t* __restrict__ sched) {
  extern __shared__ int32_t sh[];
  int32_t* s_cnt = sh;               // [blockDim]
  int32_t* s_til = sh + blockDim.x;  // [blockDim]
  const int e = threadIdx.x;
  int run = 0;
  if (e < E) {
    int c = 0;
    for (; c + 4 <= nchunks; c += 4) {
      const int v0 = chunk_hist[static_cast<size_t>(c) * E + e];
      const int v1 = chunk_hist[static_cast<size_t>(c + 1) * E + e];
      const int v2 = chunk_hist[static_cast<size_t>(c + 2) * E + e];
      const int v3 = chunk_hist[static_cast<size_t>(c + 3) * E + e];
      chunk_hist[static_cast<size_t>(c) * E + e] = run;
      chunk_hist[static_cast<size_t>(c + 1) * E + e] = run + v0;
      chunk_hist[static_cast<size_t>(c + 2) * E + e] = run + v0 + v1;
      chunk_hist[static_cast<size_t>(c + 3) * E + e] = run + v0 + v1 + v2;
      run += v0 + v1 + v2 + v3;
    }
    for (; c < nchunks; ++c) {
      const int v = chunk_hist[static_cast<size_t>(c) * E + e];
      chunk_hist[static_cast<size_t>(c) * E + e] = run;
      run += v;
    }
    counts[e] = run;
  }
  const int ntiles = (e < E && run > 0) ? (run + max_n - 1) / max_n : 0;
  s_cnt[e] = (e < E) ? run : 0;
  s_til[e] = ntiles;
  __syncthreads();
  // Hillis-Steele inclusive scans (E <= 1024, negligible)
  for (int o = 1; o < static_cast<int>(blockDim.x); o <<= 1) {
    const int a = (e >= o) ? s_cnt[e - o] : 0;
    const int b = (e >= o) ? s_til[e - o] : 0;
    __syncthreads();
    s_cnt[e] += a;
    s_til[e] += b;
    __syncthreads();
  }
  if (e < E) {
    offsets[e] = s_cnt[e] - run;
    tile_prefix[e] = s_til[e] - ntiles;
    // even split of the expert's rows over its tiles, rounded to the MMA N step
    const int per = ntiles ? (run + ntiles - 1) / ntiles : 0;
    tile_rows[e] = min(max_n, (per + 15) & ~15);
    if (e == E - 1) {
      offsets[E] = s_cnt[e];
      tile_prefix[E] = s_til[e];
    }
  }
  for (int i = e; i <= E; i += blockDim.x) sched[i] = 0u;
}

// One warp per routing entry: final slot, inverse map, and the row gather.
__global__ void __launch_bounds__(256)
    k_scatter(const int32_t* __restrict__ ids, const int32_t* __restrict__ chunk_base,
              const int32_t* __restrict__ rank_local, const int32_t* __restrict__ offsets,
              const __nv_bfloat16* __restrict__ x, int S, int E, int topk, int H,
              int32_t* __restrict__ slot_of, int32_t* __restrict__ tok_of, __nv_bfloat16* __restrict__ x_perm) {
  const int i = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (i >= S) return;
  const int e = ids[i];
  const int t = i / topk;
  const int slot = offsets[e] + chunk_base[static_cast<size_t>(i / kChunk) * E + e] + rank_local[i];
  if (lane == 0) {
    slot_of[i] = slot;
    tok_of[slot] = t;
  }
  if (x_perm != nullptr) {
    const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * H);
    uint4* dst = reinterpret_cast<uint4*>(x_perm + static_cast<size_t>(slot) * H);
    const int nv = H / 8;
    for (int v = lane; v < nv; v += 32) dst[v] = src[v];
  }
}

// y[t] = sum_j w[t,j] * y_perm[slot_of[t,j]]   (fp32 accumulate, bf16 out)
__global__ void __launch_bounds__(256)
    k_combine(const __nv_bfloat16* __restrict__ y_perm, const int32_t* __restrict__ slot_of,
              const float* __restrict__ w, int T, int topk, int H, __nv_bfloat16* __restrict__ y) {
  const int t = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int nv = H / 8;
  for (int v0 = 0; v0 < nv; v0 += 32 * 4) {
    float acc[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[u][q] = 0.f;
    for (int j = 0; j < topk; ++j) {
      const int slot = slot_of[static_cast<size_t>(t) * topk + j];
      const float wj = w[static_cast<size_t>(t) * topk + j];
      const uint4* src = reinterpret_cast<const uint4*>(y_perm + static_cast<size_t>(slot) * H);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < nv) {
          const uint4 d = src[v];
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&d);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __bfloat1622float2(h2[q]);
            acc[u][2 * q] += wj * f.x;
            acc[u][2 * q + 1] += wj * f.y;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int v = v0 + u * 32 + lane;
      if (v < nv) {
        uint4 o;
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int q = 0; q < 4; ++q) o2[q] = __floats2bfloat162_rn(acc[u][2 * q], acc[u][2 * q + 1]);
        reinterpret_cast<uint4*>(y + static_cast<size_t>(t) * H)[v] = o;
      }
    }
  }
}

}  // namespace lp

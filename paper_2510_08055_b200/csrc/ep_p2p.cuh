// Expert parallelism over peer memory (NVLink / NVSwitch P2P through CUDA IPC
// mappings): the dispatch and return all-to-alls of ep.py's NCCL path folded
// into the permutation and the combine.
//
// Every rank exposes, at the same logical layout, an inbox of per-source
// expert counts, a receive buffer recv_x [cap, H] and its expert outputs
// y_out [cap, H]; the other ranks hold mapped pointers to them (device arrays
// of P pointers). Per layer, rank r (P ranks, E = P * El experts):
//   1. route + local slot order (liblpmoe route / permute, index-only)
//   2. k_ep_post_counts: counts of r's tokens per expert of rank d -> inbox_d[r]
//   3. barrier
//   4. k_ep_plan: from every destination's inbox, r's first row in d's receive
//      buffer per expert (rows are expert-major, source-major within an expert,
//      source order within a source: the layout a single-GPU x_perm of the
//      concatenated batch would have per expert), and r's own expert offsets
//   5. k_ep_dispatch: token rows stored straight into the owners' recv_x
//      (fused permute + send, no staging buffer)
//   6. barrier; owners run the expert kernel on recv_x -> y_out
//   7. barrier; k_ep_combine: y[t] = sum_j w[t,j] * y_out_d[row] read straight
//      from the owners (fused receive + weighted combine, fixed j order)
//   8. barrier (buffers reusable)
// Barriers are device-side: each rank adds 1 to every rank's counter with a
// system-scope release and spins on its own with a system-scope acquire.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace lp {

__device__ __forceinline__ void red_add_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// One warp: signal every rank, then wait until this rank's counter reaches
// `target` (= P * barrier epoch). Counters only grow.
__global__ void k_ep_barrier(uint32_t* const* __restrict__ peer_flag, int P, int rank, uint32_t target) {
  const int lane = threadIdx.x;
  __threadfence_system();
  __syncwarp();
  for (int q = lane; q < P; q += 32) red_add_release_sys(peer_flag[q], 1u);
  if (lane == 0) {
    const uint32_t* mine = peer_flag[rank];
    while (static_cast<int32_t>(ld_acquire_sys(mine) - target) < 0) __nanosleep(128);
  }
  __syncwarp();
}

// counts[E] of this rank's routing entries per global expert -> inbox of rank
// d at row `rank`: inbox_d[rank * El + el] = counts[d * El + el].
__global__ void k_ep_post_counts(const int32_t* __restrict__ counts, int32_t* const* __restrict__ peer_inbox, int P,
                                 int El, int rank) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < P * El) {
    const int d = e / El, el = e - d * El;
    peer_inbox[d][rank * El + el] = counts[e];
  }
  __threadfence_system();
}

// dest_base[d * El + el]: first row of (source = rank, expert el of d) in d's
// receive buffer; off_local[0..El]: this rank's expert offsets over all sources.
// One CTA, blockDim >= max(P * El, El + 1).
__global__ void k_ep_plan(int32_t* const* __restrict__ peer_inbox, int P, int El, int rank,
                          int32_t* __restrict__ dest_base, int32_t* __restrict__ off_local) {
  extern __shared__ int32_t s_cnt[];  // [P dest][P src][El]
  const int n = P * P * El;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int d = i / (P * El), rest = i - d * P * El;  // rest = src * El + el
    s_cnt[i] = __ldcv(peer_inbox[d] + rest);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P * El; i += blockDim.x) {
    const int d = i / El, el = i - d * El;
    const int32_t* c = s_cnt + d * P * El;  // c[src * El + e']
    int base = 0;
    for (int e2 = 0; e2 < el; ++e2)
      for (int s = 0; s < P; ++s) base += c[s * El + e2];
    for (int s = 0; s < rank; ++s) base += c[s * El + el];
    dest_base[i] = base;
  }
  for (int i = threadIdx.x; i <= El; i += blockDim.x) {  // El + 1 entries: El may reach blockDim.x
    const int32_t* c = s_cnt + rank * P * El;
    int o = 0;
    for (int e2 = 0; e2 < i; ++e2)
      for (int s = 0; s < P; ++s) o += c[s * El + e2];
    off_local[i] = o;
  }
}

// Warp per routing entry i = t * topk + j: the token row goes straight into
// the owner's receive buffer at its planned row; (dest_rank, dest_row) are
// kept for the combine.
__global__ void __launch_bounds__(256)
    k_ep_dispatch(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ ids,
                  const int32_t* __restrict__ slot_of, const int32_t* __restrict__ offsets,
                  const int32_t* __restrict__ dest_base, __nv_bfloat16* const* __restrict__ peer_recv, int S, int H,
                  int topk, int El, int32_t* __restrict__ dest_rank, int32_t* __restrict__ dest_row) {
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
  __threadfence_system();
}

// CTA per token: y[t] = sum_j w[t,j] * y_out_{dest_rank}[dest_row] (fp32, fixed j order).
__global__ void __launch_bounds__(256)
    k_ep_combine(__nv_bfloat16* const* __restrict__ peer_y, const int32_t* __restrict__ dest_rank,
                 const int32_t* __restrict__ dest_row, const float* __restrict__ w, int T, int topk, int H,
                 __nv_bfloat16* __restrict__ y) {
  const int t = blockIdx.x;
  __shared__ const __nv_bfloat16* s_row[32];
  __shared__ float s_w[32];
  if (threadIdx.x < topk) {
    const int i = t * topk + threadIdx.x;
    s_row[threadIdx.x] = peer_y[dest_rank[i]] + static_cast<size_t>(dest_row[i]) * H;
    s_w[threadIdx.x] = w[i];
  }
  __syncthreads();
  for (int v = threadIdx.x; v < H / 8; v += blockDim.x) {
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    for (int j = 0; j < topk; ++j) {
      const uint4 d = __ldcv(reinterpret_cast<const uint4*>(s_row[j]) + v);
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
}

}  // namespace lp

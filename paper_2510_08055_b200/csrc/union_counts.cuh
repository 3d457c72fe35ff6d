// Routing-surrogate sampler: per-trial union size of `batch` top-k expert
// draws from pre-drawn uniforms. Bit-exact GPU restatement of the reference's
// numba kernels (moesim/kernels.py:73-103 uniform partial Fisher-Yates,
// kernels.py:106-145 weighted draw without replacement); the float64
// arithmetic is issued op-for-op in the reference order with explicit _rn
// intrinsics so no FMA contraction can change a comparison.
//
// One CTA per trial; threads stride over the trial's tokens and OR the chosen
// experts into a shared bitmask (order-independent, so the integer result is
// exact regardless of thread interleaving).
#pragma once
#include <cstdint>

namespace lp {

constexpr int kUnionThreads = 256;

template <int KMAX>
__global__ void __launch_bounds__(kUnionThreads)
    k_union_uniform(const double* __restrict__ u, int batch, int k, int E, int64_t* __restrict__ out) {
  extern __shared__ uint32_t bits[];
  const int trial = blockIdx.x;
  const int nw = (E + 31) / 32;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) bits[i] = 0u;
  __syncthreads();
  for (int b = threadIdx.x; b < batch; b += blockDim.x) {
    const double* ub = u + (static_cast<size_t>(trial) * batch + b) * k;
    // sparse view of the identity pool: only swapped positions are stored
    int pos[2 * KMAX], val[2 * KMAX];
    int n = 0;
    for (int i = 0; i < k; ++i) {
      const int j = i + static_cast<int>(__dmul_rn(ub[i], static_cast<double>(E - i)));
      int vi = i, vj = j, si = -1, sj = -1;
      for (int q = 0; q < n; ++q) {
        if (pos[q] == i) { vi = val[q]; si = q; }
        if (pos[q] == j) { vj = val[q]; sj = q; }
      }
      if (si < 0) { si = n; pos[n] = i; ++n; }
      if (sj < 0 && j != i) { sj = n; pos[n] = j; ++n; }
      if (j == i) sj = si;
      val[si] = vj;
      val[sj] = vi;
      if (j == i) val[si] = vi;
      atomicOr(&bits[vj >> 5], 1u << (vj & 31));
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int c = 0;
    for (int i = threadIdx.x; i < nw; i += 32) c += __popc(bits[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (threadIdx.x == 0) out[trial] = c;
  }
}

__global__ void __launch_bounds__(kUnionThreads)
    k_union_weighted(const double* __restrict__ u, int batch, int k, int E, const double* __restrict__ weights,
                     int64_t* __restrict__ out) {
  extern __shared__ uint8_t sh_raw[];
  double* sw = reinterpret_cast<double*>(sh_raw);
  uint32_t* bits = reinterpret_cast<uint32_t*>(sw + E);
  __shared__ double s_total;
  const int trial = blockIdx.x;
  const int nw = (E + 31) / 32;
  for (int i = threadIdx.x; i < E; i += blockDim.x) sw[i] = weights[i];
  for (int i = threadIdx.x; i < nw; i += blockDim.x) bits[i] = 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tw = 0.0;
    for (int e = 0; e < E; ++e) tw = __dadd_rn(tw, sw[e]);  // kernels.py:113-115 order
    s_total = tw;
  }
  __syncthreads();
  const double total_w = s_total;
  for (int b = threadIdx.x; b < batch; b += blockDim.x) {
    const double* ub = u + (static_cast<size_t>(trial) * batch + b) * k;
    uint32_t drawn[32];  // E <= 1024
    for (int i = 0; i < nw; ++i) drawn[i] = 0u;
    double w_rem = total_w;
    for (int i = 0; i < k; ++i) {
      const double target = __dmul_rn(ub[i], w_rem);
      double cum = 0.0;
      int sel = -1;
      for (int e = 0; e < E; ++e) {
        if (drawn[e >> 5] & (1u << (e & 31))) continue;
        cum = __dadd_rn(cum, sw[e]);
        if (cum > target) { sel = e; break; }
      }
      if (sel < 0) {  // round-off pushed target past the final cumsum (kernels.py:133-138)
        for (int e = E - 1; e >= 0; --e)
          if (!(drawn[e >> 5] & (1u << (e & 31)))) { sel = e; break; }
      }
      drawn[sel >> 5] |= 1u << (sel & 31);
      w_rem = __dsub_rn(w_rem, sw[sel]);
      atomicOr(&bits[sel >> 5], 1u << (sel & 31));
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int c = 0;
    for (int i = threadIdx.x; i < nw; i += 32) c += __popc(bits[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (threadIdx.x == 0) out[trial] = c;
  }
}

}  // namespace lp

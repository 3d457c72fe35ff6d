// cta_group::2 vs cta_group::1 tcgen05.mma issue cost at decode-size N (B200 experiment, not shipped).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/mma_pair_bench tools/mma_pair_bench.cu
//
// Question: is the ~55-130 cycles per M=128 x N=16 x K=16 MMA (tools/mma_chain_bench.cu) a cost per
// INSTRUCTION (then a CTA pair issuing M=256 instructions moves twice the weight rows per SM per
// cycle) or per 128-row block? Operands resident in smem; the leader of each pair issues `kb`
// k-blocks of 4 MMAs (M=256 over the pair, N=16) with a commit + stage wait per k-block (the decode
// kernel's loop) and times issue -> completion.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2510_08055_b200/csrc/ptx.cuh"

using namespace lp;

template <int N, int WAIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_pair(int kblocks, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int kA = 16384, kB = N * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kA + kB);  // [0] done, [1..8] ring, [9..16] full
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 17);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < (kA + kB) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 17; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    for (int i = 9; i < 17; ++i) mbar_arrive(&bars[i]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 2) tmem_alloc_pair(tslot, 256);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (rank == 0 && warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(256, N);
    const uint64_t a0 = sdesc_kmajor_sw128(smem_u32(smem));
    const uint64_t b0 = sdesc_kmajor_sw128(smem_u32(smem + kA));
    const unsigned long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
      if (WAIT) { mbar_wait(&bars[9 + (kb & 7)], 0); mbar_wait(&bars[9 + ((kb + 1) & 7)], 0); tc_fence_after(); }
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_bf16_pair(tbase, a0 + 2 * k, b0 + 2 * k, idesc, kb | k);
      if (WAIT) mma_commit_pair(&bars[1 + (kb & 7)]);
    }
    mma_commit_pair(&bars[0]);
    mbar_wait(&bars[0], 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  } else if (rank == 1 && warp == 1 && lane == 0) {
    mbar_wait(&bars[0], 0);  // the leader's multicast commit arrives here too
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, 256);
  }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int N, int WAIT>
void run(int kblocks, unsigned long long* d_out) {
  const int smem = 1024 + 16384 + N * 128 + 256;
  CK(cudaFuncSetAttribute(k_pair<N, WAIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long best = ~0ull;
  for (int rep = 0; rep < 5; ++rep) {
    k_pair<N, WAIT><<<148, 128, smem>>>(kblocks, d_out);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, d_out, sizeof(c), cudaMemcpyDeviceToHost));
    if (c < best) best = c;
  }
  const double per = static_cast<double>(best) / (4.0 * kblocks);
  // weight bytes per pair MMA: 256 rows x 16 k x 2 B = 8 KiB, i.e. 4 KiB per SM
  printf("pair N=%3d wait=%d kblocks=%3d: %6.1f cycles/MMA -> %6.1f GB/s of weight rows per SM at 1.9 GHz\n", N, WAIT,
         kblocks, per, 4096.0 / (per / 1.9e9) / 1e9);
}

int main() {
  unsigned long long* d_out;
  CK(cudaMalloc(&d_out, 64));
  run<16, 0>(32, d_out);
  run<16, 1>(32, d_out);
  run<32, 1>(32, d_out);
  run<256, 0>(32, d_out);
  return 0;
}

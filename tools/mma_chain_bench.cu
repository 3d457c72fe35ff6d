// Latency of a dependent tcgen05.mma chain at decode-size N (B200 experiment, not shipped).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/mma_chain_bench tools/mma_chain_bench.cu
//   ./tools/mma_chain_bench
//
// The decode-size expert items issue 4 MMAs (M=128 x N=16 x K=16) per 16 KiB weight k-block,
// all accumulating into ONE TMEM accumulator. If a dependent MMA costs a fixed pipeline latency,
// such a chain caps an SM at (16 KiB / (4 x latency)) of weight streaming regardless of HBM.
// Operands sit in shared memory (no loads): one CTA per SM issues `n` k-blocks of 4 MMAs into
// NACC accumulators (k-block i -> accumulator i % NACC), commits once, and times issue -> commit
// completion with clock64. Reports cycles per MMA and the implied weight-streaming rate per SM.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2510_08055_b200/csrc/ptx.cuh"

using namespace lp;

template <int N, int NACC, int COMMIT = 0, int SPIN = 0>
__global__ void __launch_bounds__(256, 1) k_chain(int kblocks, unsigned long long* out) {
  const uint32_t* gflag = reinterpret_cast<const uint32_t*>(out + 4);  // a zero word in global memory
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int kA = 16384, kB = N * 128;
  uint64_t* done = reinterpret_cast<uint64_t*>(smem + kA + kB);
  uint64_t* ring = done + 1;  // COMMIT: 8 stage barriers (empty) + 8 pre-completed (full)
  uint64_t* spinbar = ring + 16;  // SPIN: warps 0, 2-7 spin on it until the MMA thread is done
  uint32_t* flag = reinterpret_cast<uint32_t*>(spinbar + 1);  // COMMIT 8: 8 ready words, set to 1
  uint32_t* tslot = flag + 8;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (kA + kB) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(done, 1);
    for (int i = 0; i < 16; ++i) mbar_init(&ring[i], 1);
    mbar_init(spinbar, 1);
    for (int i = 0; i < 8; ++i) flag[i] = 1u;
    fence_mbar_init();
    for (int i = 8; i < 16; ++i) mbar_arrive(&ring[i]);  // "full" barriers: phase 0 complete
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t a0 = sdesc_kmajor_sw128(smem_u32(smem));
    const uint64_t b0 = sdesc_kmajor_sw128(smem_u32(smem + kA));
    const unsigned long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
      const uint32_t d = tbase + (kb % NACC) * N;
      // 2: two waits + fence (the expert kernels' loop), 3: one wait + fence, 4: two waits, 5: one wait
      if (COMMIT == 2 || COMMIT == 4) { mbar_wait(&ring[8 + (kb & 7)], 0); mbar_wait(&ring[8 + ((kb + 1) & 7)], 0); }
      if (COMMIT == 3 || COMMIT == 5) mbar_wait(&ring[8 + (kb & 7)], 0);
      if (COMMIT == 2 || COMMIT == 3) tc_fence_after();
      if (COMMIT == 10) mbar_wait(&ring[8 + (kb & 7)], 0);  // wait per k-block, NO commit
      if (COMMIT == 11) {  // poll a GLOBAL word (LDG) per k-block, then commit
        uint32_t v;
        do {
          asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(gflag) : "memory");
        } while (v != 0u);
      }
      if (COMMIT == 9) {  // relaxed volatile LDS poll, no fence
        uint32_t v;
        do {
          asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(flag + (kb & 7))) : "memory");
        } while (v != 1u);
      }
      if (COMMIT == 8) {  // poll a shared-memory ready word (LDS) instead of an mbarrier, then commit per k-block
        uint32_t v;
        do {
          asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(flag + (kb & 7))) : "memory");
        } while (v != 1u);
        tc_fence_after();
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_bf16(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb >= NACC) || k != 0);
      if ((COMMIT >= 1 && COMMIT <= 5) || COMMIT == 8 || COMMIT == 9 || COMMIT == 11) mma_commit(&ring[kb & 7]);
      // 6: one wait + one commit per PAIR of k-blocks; 7: two waits + two commits per pair (per-stage release)
      if (COMMIT == 6 && (kb & 1)) { mma_commit(&ring[kb & 7]); mbar_wait(&ring[8 + (kb & 7)], 0); }
      if (COMMIT == 7 && (kb & 1)) {
        mma_commit(&ring[(kb - 1) & 7]);
        mma_commit(&ring[kb & 7]);
        mbar_wait(&ring[8 + (kb & 7)], 0);
        mbar_wait(&ring[8 + ((kb + 1) & 7)], 0);
      }
    }
    mma_commit(done);
    mbar_wait(done, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    mbar_arrive(spinbar);
  } else if (SPIN && lane == 0 && warp != 1) {
    if (SPIN == 1) mbar_wait(spinbar, 0);  // try_wait spin, as the expert kernels' waiting roles
    else while (!mbar_try_wait(spinbar, 0)) __nanosleep(64);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int N, int NACC, int COMMIT = 0, int SPIN = 0>
void run(int kblocks, unsigned long long* d_out) {
  const int smem = 1024 + 16384 + N * 128 + 256;
  CK(cudaFuncSetAttribute(k_chain<N, NACC, COMMIT, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long best = ~0ull;
  for (int rep = 0; rep < 5; ++rep) {
    k_chain<N, NACC, COMMIT, SPIN><<<148, 256, smem>>>(kblocks, d_out);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, d_out, sizeof(c), cudaMemcpyDeviceToHost));
    if (c < best) best = c;
  }
  const double per = static_cast<double>(best) / (4.0 * kblocks);
  // weight bytes per MMA: 128 rows x 16 k x 2 B = 4 KiB; at ~1.9 GHz
  printf("N=%3d acc=%d commit=%d spin=%d kblocks=%3d: %6.1f cycles/MMA  -> %6.1f GB/s of M=128 weight rows per SM at 1.9 GHz\n", N, NACC,
         COMMIT, SPIN, kblocks, per, 4096.0 / (per / 1.9e9) / 1e9);
}

int main() {
  unsigned long long* d_out;
  CK(cudaMalloc(&d_out, 64));
  CK(cudaMemset(d_out, 0, 64));
  for (int kb : {12, 32, 128}) {
    run<16, 1>(kb, d_out);
    run<16, 2>(kb, d_out);
    run<16, 4>(kb, d_out);
  }
  run<16, 1, 1>(32, d_out);   // + tcgen05.commit per k-block (stage release)
  run<16, 1, 2>(32, d_out);   // + two mbarrier waits per k-block (full, bfull) as the expert kernels
  run<16, 1, 3>(32, d_out);
  run<16, 1, 4>(32, d_out);
  run<16, 1, 5>(32, d_out);
  run<16, 1, 8>(32, d_out);
  run<16, 1, 9>(32, d_out);
  run<16, 1, 10>(32, d_out);
  run<16, 1, 11>(32, d_out);
  run<64, 2, 2>(32, d_out);
  run<128, 1, 2>(32, d_out);
  run<256, 1, 2>(32, d_out);
  run<256, 1, 1>(32, d_out);
  run<16, 1, 6>(32, d_out);
  run<16, 1, 7>(32, d_out);
  run<16, 1, 2, 1>(32, d_out);  // + 7 other warps spinning on an mbarrier (try_wait loops)
  run<16, 1, 2, 2>(32, d_out);  // + 7 other warps polling with nanosleep backoff
  run<32, 1>(32, d_out);
  run<64, 1>(32, d_out);
  run<64, 2>(32, d_out);
  run<128, 1>(32, d_out);
  run<256, 1>(32, d_out);
  return 0;
}

// tcgen05 issue-rate ceilings for the expert kernel's tile shapes (B200 experiment, not shipped).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/mma_bench tools/mma_bench.cu
//   ./tools/mma_bench
//
// Persistent grid, 1 CTA/SM. Per k-block (K = 64) the MMA thread issues, like
// k_experts' UP items, two M=128 x N x K=16 MMAs per k-step (gate and up
// accumulators sharing the B tile), then commits the stage.
//   MODE 0: operands already in smem (no TMA): pure MMA issue ceiling.
//   MODE 1: a TMA producer refills every stage from an L2-resident buffer
//           (A 2 x 16 KiB weight boxes + B token boxes), full/empty ring.
// Reports achieved bf16 TFLOP/s over the whole grid (CUDA events).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2510_08055_b200/csrc/ptx.cuh"

using namespace lp;

constexpr int kA = 16384;

template <int N, int STAGES, int MODE, int NACC>
__global__ void __launch_bounds__(128, 1) k_mma(const __grid_constant__ CUtensorMap tmw,
                                                 const __grid_constant__ CUtensorMap tmx, int kblocks) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int kB = N * 128;
  constexpr int kStage = 2 * kA + kB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (warp == 0 && lane == 0 && MODE == 1) {
    int stage = 0; uint32_t ph = 0;
    const uint64_t pol = policy_evict_last();
    const int row0 = (blockIdx.x % 16) * 256;
    for (int kb = 0; kb < kblocks; ++kb) {
      mbar_wait(&empty[stage], ph ^ 1);
      uint8_t* sa = smem + stage * kStage;
      mbar_arrive_expect_tx(&full[stage], kStage);
      const int k0 = (kb % 32) * 64;
      tma_load_2d(sa, &tmw, &full[stage], k0, row0, pol);
      tma_load_2d(sa + kA, &tmw, &full[stage], k0, row0 + 128, pol);
      for (int b = 0; b < N / 32; ++b) tma_load_2d(sa + 2 * kA + b * 4096, &tmx, &full[stage], k0, b * 32, pol);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    int stage = 0; uint32_t ph = 0;
    for (int kb = 0; kb < kblocks; ++kb) {
      if (MODE == 1) mbar_wait(&full[stage], ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + stage * kStage);
      const uint64_t a0 = sdesc_kmajor_sw128(sa), a1 = sdesc_kmajor_sw128(sa + kA);
      const uint64_t b0 = sdesc_kmajor_sw128(sa + 2 * kA);
      const uint32_t acc = (kb & 7) != 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mma_bf16(tbase, a0 + 2 * k, b0 + 2 * k, idesc, acc | (k != 0));
        if (NACC == 2) mma_bf16(tbase + N, a1 + 2 * k, b0 + 2 * k, idesc, acc | (k != 0));
      }
      mma_commit(&empty[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    mma_commit(done);
    mbar_wait(done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode;

void make_map(CUtensorMap* m, void* p, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); exit(1); }
}

template <int N, int STAGES, int MODE, int NACC>
void run(const CUtensorMap& tmw, const CUtensorMap& tmx, int sms) {
  constexpr int kStage = 2 * kA + N * 128;
  const int smem = 1024 + STAGES * kStage + 256;
  auto k = k_mma<N, STAGES, MODE, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int kblocks = 4096;
  k<<<sms, 128, smem>>>(tmw, tmx, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k<<<sms, 128, smem>>>(tmw, tmx, kblocks);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); exit(1); }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 128 * N * 64 * NACC * double(kblocks) * sms * reps;
  printf("N=%3d stages=%d mode=%d acc=%d : %7.1f TFLOP/s  (%.1f us/launch)\n", N, STAGES, MODE, NACC,
         flops / (ms * 1e-3) / 1e12, ms * 1e3 / reps);
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *w, *x;
  cudaMalloc(&w, 4096ull * 2048 * 2);  // 16 MiB weights (L2 resident)
  cudaMalloc(&x, 256ull * 2048 * 2);
  cudaMemset(w, 0, 4096ull * 2048 * 2);
  cudaMemset(x, 0, 256ull * 2048 * 2);
  CUtensorMap tmw, tmx;
  make_map(&tmw, w, 4096, 2048, 128);
  make_map(&tmx, x, 256, 2048, 32);
  run<256, 3, 0, 2>(tmw, tmx, sms);
  run<256, 3, 1, 2>(tmw, tmx, sms);
  run<256, 3, 0, 1>(tmw, tmx, sms);
  run<256, 3, 1, 1>(tmw, tmx, sms);
  run<192, 3, 0, 2>(tmw, tmx, sms);
  run<192, 3, 1, 2>(tmw, tmx, sms);
  run<128, 4, 0, 2>(tmw, tmx, sms);
  run<128, 4, 1, 2>(tmw, tmx, sms);
  run<64, 5, 0, 2>(tmw, tmx, sms);
  run<64, 5, 1, 2>(tmw, tmx, sms);
  return 0;
}

// Read-bandwidth ceilings for the expert-weight stream (B200 experiment, not shipped).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/stream_bench tools/stream_bench.cu
//   ./tools/stream_bench
//
// Streams a 1.2 GB bf16 matrix laid out like W13 ([E*2I, H] row-major) from HBM:
//   A  TMA 2-D boxes of 128 rows x 64 cols (the expert kernel's pattern), S-stage ring
//   B  TMA 1-D bulk copies of contiguous 16 KiB chunks (a pre-tiled weight layout)
//   C  plain 16-byte LDG loads, all threads (read-only HBM ceiling)
// Persistent grid (1 CTA/SM), dynamic 1 MiB work items, no math.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2510_08055_b200/csrc/ptx.cuh"

using namespace lp;

constexpr int H = 2048;
constexpr long long kTotalRows = 128LL * 1536;  // E * 2I
constexpr int kItemKb = 32;                     // k-blocks per item (H / 64)

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int STAGES, int MODE>
__global__ void __launch_bounds__(128, 1) k_stream(const __grid_constant__ CUtensorMap tm, const uint8_t* lin,
                                                    unsigned* counter, int n_items) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStage = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  __shared__ int s_item;
  if (threadIdx.x == 0) s_item = -1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    const uint64_t pol = policy_evict_first();
    int stage = 0; uint32_t ph = 0;
    int produced = 0;
    while (true) {
      const int it = atomicAdd(counter, 1u);
      if (it >= n_items) break;
      const int row = it * 256;  // two 128-row slabs per item (gate-like + up-like), disjoint across items
      for (int kb = 0; kb < kItemKb; ++kb) {
        mbar_wait(&empty[stage], ph ^ 1);
        mbar_arrive_expect_tx(&full[stage], kStage);
        uint8_t* dst = smem + stage * kStage;
        if (MODE == 0) {
          tma_load_2d(dst, &tm, &full[stage], kb * 64, row, pol);
          tma_load_2d(dst + 16384, &tm, &full[stage], kb * 64, row + 128, pol);
        } else {
          const size_t off = ((size_t)it * kItemKb + kb) * kStage;
          bulk_load(dst, lin + off, 16384, &full[stage], pol);
          bulk_load(dst + 16384, lin + off + 16384, 16384, &full[stage], pol);
        }
        ++produced;
        if (++stage == STAGES) { stage = 0; ph ^= 1; }
      }
    }
    *(volatile int*)&s_item = produced;
  } else if (warp == 1 && lane == 0) {
    int stage = 0; uint32_t ph = 0;
    int consumed = 0;
    while (true) {
      const int total = *(volatile int*)&s_item;
      if (total >= 0 && consumed == total) break;
      if (mbar_try_wait(&full[stage], ph)) {
        mbar_arrive(&empty[stage]);
        ++consumed;
        if (++stage == STAGES) { stage = 0; ph ^= 1; }
      }
    }
  }
  __syncthreads();
}

__global__ void k_ldg(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t j = i + (size_t)u * gridDim.x * blockDim.x;
      v[u] = j < n ? __ldcs(p + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1u);
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int STAGES, int MODE>
float run(const CUtensorMap& tm, const uint8_t* lin, unsigned* counter, int n_items, int sms) {
  const int smem = 1024 + STAGES * 32768 + 256;
  CK(cudaFuncSetAttribute(k_stream<STAGES, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaMemset(counter, 0, 4));
    cudaEventRecord(a);
    k_stream<STAGES, MODE><<<sms, 128, smem>>>(tm, lin, counter, n_items);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = (size_t)kTotalRows * H * 2;  // 805 MB (W13 of one layer)
  uint8_t* w; CK(cudaMalloc(&w, bytes * 2));
  CK(cudaMemset(w, 1, bytes * 2));
  unsigned* counter; CK(cudaMalloc(&counter, 16));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  cuuint64_t dims[2] = {H, (cuuint64_t)kTotalRows};
  cuuint64_t strides[1] = {H * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
    printf("encode failed\n"); return 1;
  }
  const int n_items = (int)(kTotalRows / 256);  // 768 items of 1 MiB = 805 MB, every byte read once
  const double item_bytes = 32768.0 * kItemKb;
  const double total = item_bytes * n_items;
  printf("SMs %d, items %d x %.0f KiB = %.3f GB\n", sms, n_items, item_bytes / 1024, total / 1e9);
  float t;
  t = run<4, 0>(tm, w, counter, n_items, sms); printf("A 2-D boxes   4 stages: %.1f us  %.0f GB/s\n", t * 1e3, total / (t * 1e-3) / 1e9);
  t = run<5, 0>(tm, w, counter, n_items, sms); printf("A 2-D boxes   5 stages: %.1f us  %.0f GB/s\n", t * 1e3, total / (t * 1e-3) / 1e9);
  t = run<6, 0>(tm, w, counter, n_items, sms); printf("A 2-D boxes   6 stages: %.1f us  %.0f GB/s\n", t * 1e3, total / (t * 1e-3) / 1e9);
  t = run<4, 1>(tm, w, counter, n_items, sms); printf("B 1-D bulk    4 stages: %.1f us  %.0f GB/s\n", t * 1e3, total / (t * 1e-3) / 1e9);
  t = run<6, 1>(tm, w, counter, n_items, sms); printf("B 1-D bulk    6 stages: %.1f us  %.0f GB/s\n", t * 1e3, total / (t * 1e-3) / 1e9);
  {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    const size_t n = bytes / 16;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      k_ldg<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(w), n, counter);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("C LDG.128 read-only: %.1f us  %.0f GB/s\n", best * 1e3, bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}

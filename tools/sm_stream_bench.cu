// Per-SM weight-streaming rate in the decode regime (B200 experiment, not shipped).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/sm_stream_bench tools/sm_stream_bench.cu -lcuda
//   ./tools/sm_stream_bench
//
// A decode-size MoE layer streams only ~75 MB (T=1: 8 experts x 9.4 MB), so the
// question is not the aggregate HBM ceiling but how fast ONE SM can pull a
// 0.2-0.5 MB work item through a TMA ring and how many SMs it takes to saturate
// HBM. Each CTA streams `per_cta` bytes of W13-like 128-row x 64-col boxes
// (SWIZZLE_128B, the expert kernels' pattern) through S stages of 16 KiB; we
// time the whole launch (cold L2: the buffer is rotated over 1.6 GB).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2510_08055_b200/csrc/ptx.cuh"

using namespace lp;

// MMA consumer shape: g_mma_k of the stage's four K=16 slices issued, N = g_mma_n token columns
__constant__ int g_mma_k = 4;
__constant__ int g_mma_n = 16;

constexpr int H = 2048;
constexpr long long kRows = 128LL * 1536 * 4;  // 4 layers of W13: 3.2 GB

template <int STAGES, int SK = 1>  // SK: 16 KiB k-blocks per stage
// mma = 1: the consumer is a decode item's (one thread issues 4 tcgen05.mma M=128 x N=16 x K=16 per
// 16 KiB stage into one TMEM accumulator, tcgen05.commit frees the stage); 0: it frees each stage as
// soon as it lands (plain TMA ring)
__global__ void __launch_bounds__(64, 1) k_sm_stream(const __grid_constant__ CUtensorMap tm, int kb_per_cta,
                                                      long long row_base, int hot, int boxes, int mma) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStage = 16384 * SK;
  uint8_t* bbuf = smem + STAGES * kStage;  // up to 64 token rows x 128 B (B operand, zeros)
  uint64_t* full = reinterpret_cast<uint64_t*>(bbuf + 8192);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 2048; i += 64) reinterpret_cast<uint32_t*>(bbuf)[i] = 0u;
  if (mma && threadIdx.x >= 32) tmem_alloc(tslot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  // CTA b streams 128-row slabs: slab = b*? ; each slab is 32 k-blocks (512 KiB of 128 rows)
  if (warp == 0 && lane == 0) {
    const uint64_t pol = policy_evict_first();
    int stage = 0; uint32_t ph = 0;
    for (int i = 0; i < kb_per_cta; i += SK) {
      // hot: every CTA reads the same 0.5 MB (a router weight in L2); boxes: 128-row box split in 1 or 2
      const long long slab = hot ? (i / 32) % 2 : (static_cast<long long>(blockIdx.x) * kb_per_cta + i) / 32;
      const int kb = i % 32;
      mbar_wait(&empty[stage], ph ^ 1);
      mbar_arrive_expect_tx(&full[stage], kStage);
      if (boxes == 1) {
        for (int h = 0; h < SK; ++h)
          tma_load_2d(smem + stage * kStage + h * 16384, &tm, &full[stage], (kb + h) * 64,
                      static_cast<int>(row_base + slab * 128), pol);
      } else if (boxes == 2) {  // gate/up-like: two 64-row boxes 768 rows apart
        tma_load_2d(smem + stage * kStage, &tm, &full[stage], kb * 64, static_cast<int>(row_base + slab * 128), pol);
        tma_load_2d(smem + stage * kStage + 8192, &tm, &full[stage], kb * 64,
                    static_cast<int>(row_base + slab * 128 + 768), pol);
      } else {  // the same 128 rows as `boxes == 1`, in `-boxes` boxes of 128/-boxes rows (no overlap)
        const int nb = -boxes, rows = 128 / nb;
        for (int b = 0; b < nb; ++b)
          tma_load_2d(smem + stage * kStage + b * rows * 128, &tm, &full[stage], kb * 64,
                      static_cast<int>(row_base + slab * 128 + b * rows), pol);
      }
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    int stage = 0; uint32_t ph = 0;
    const uint32_t tmem = mma ? *tslot : 0u;
    const uint64_t b0 = sdesc_kmajor_sw128(smem_u32(bbuf));
    for (int i = 0; i < kb_per_cta; i += SK) {
      mbar_wait(&full[stage], ph);
      if (mma) {
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < SK; ++h) {
          const uint64_t a0 = sdesc_kmajor_sw128(smem_u32(smem + stage * kStage + h * 16384));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < g_mma_k) mma_bf16(tmem, a0 + 2 * k, b0 + 2 * k, idesc_bf16_f32(128, g_mma_n), (i | h | k) != 0);
        }
        mma_commit(&empty[stage]);
      } else {
        mbar_arrive(&empty[stage]);
      }
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    if (mma) { mma_commit(done); mbar_wait(done, 0); }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (mma && warp == 1) tmem_dealloc(*tslot, 64);
}

// keeps the stream busy while the host submits the timed launch: without it the first event is
// stamped before the kernel is even submitted and every line carries ~5-7 us of host launch latency
__global__ void k_spin(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
}

static int g_mma = 0;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int STAGES, int SK = 1>
void run(const CUtensorMap& tm, int ctas, int kb_per_cta, int hot = 0, int boxes = 1, const char* tag = "") {
  const int smem = 1024 + STAGES * 16384 * SK + 8192 + 512;
  CK(cudaFuncSetAttribute(k_sm_stream<STAGES, SK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const long long rows_per_launch = static_cast<long long>(ctas) * kb_per_cta / 32 * 128 + 128;
  float tot = 0.f, best = 1e9f;
  const int reps = 12;
  long long base = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (base + rows_per_launch > kRows) base = 0;
    if (getenv("SPIN")) k_spin<<<1, 32>>>(50000);
    cudaEventRecord(a);
    k_sm_stream<STAGES, SK><<<ctas, 64, smem>>>(tm, kb_per_cta, hot ? 0 : base, hot, boxes, g_mma);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep >= 2) { tot += ms; if (ms < best) best = ms; }
    base += rows_per_launch;
  }
  const double bytes = static_cast<double>(ctas) * kb_per_cta * 16384;
  const double us = tot / (reps - 2) * 1e3;
  printf("%-8s ctas %3d  stages %2d (%3d KiB in flight)  per-CTA %4d KiB  total %6.1f MB: %7.2f us (best %7.2f)  "
         "%6.0f GB/s aggregate  %5.1f GB/s per CTA\n",
         tag, ctas, STAGES, STAGES * 16, kb_per_cta * 16, bytes / 1e6, us, best * 1e3, bytes / (us * 1e-6) / 1e9,
         bytes / ctas / (us * 1e-6) / 1e9);
}

int main() {
  const size_t bytes = static_cast<size_t>(kRows) * H * 2;
  uint8_t* w; CK(cudaMalloc(&w, bytes));
  CK(cudaMemset(w, 1, bytes));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm, tm64;
  cuuint64_t dims[2] = {H, static_cast<cuuint64_t>(kRows)};
  cuuint64_t strides[1] = {H * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
    printf("encode failed\n"); return 1;
  }
  cuuint32_t box64[2] = {64, 64};
  if (enc(&tm64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
    printf("encode failed\n"); return 1;
  }
  // box-count sensitivity: the same 128-row x 16 KiB stages as 1, 2, 4 boxes (non-overlapping rows)
  CUtensorMap tm32, tm16;
  cuuint32_t box32[2] = {64, 32}, box16b[2] = {64, 64};
  if (enc(&tm32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0 ||
      enc(&tm16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box16b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
    printf("encode failed\n"); return 1;
  }
  if (getenv("MMA_AB")) {
    // plain ring vs decode-item MMA consumer, launch floor (1 k-block) beside each for the slope
    for (int m : {0, 1}) {
      g_mma = m;
      const char* tag = m ? "mma" : "plain";
      for (int ctas : {16, 96, 132, 148}) {
        run<11>(tm, ctas, 1, 0, 1, tag);
        run<11>(tm, ctas, 32, 0, 1, tag);
      }
      run<11>(tm64, 96, 32, 0, 2, m ? "mma2x64" : "plain2x64");  // gate/up boxes 768 rows apart
    }
    // per-stage or per-byte pacing: the same bytes in flight as 5 stages of 32 KiB (two k-blocks each)
    for (int m : {0, 1}) {
      g_mma = m;
      for (int ctas : {16, 96, 132}) {
        run<11>(tm, ctas, 32, 0, 1, m ? "mma16K" : "plain16K");
        run<5, 2>(tm, ctas, 32, 0, 1, m ? "mma32Kx5" : "plain32Kx5");
        run<6, 2>(tm, ctas, 32, 0, 1, m ? "mma32Kx6" : "plain32Kx6");
      }
    }
    if (getenv("SK_ONLY")) return 0;
    // what paces the MMA consumer: MMAs per stage (K slices) and N
    g_mma = 1;
    for (int kk : {1, 2, 4})
      for (int nn : {16, 32, 64}) {
        CK(cudaMemcpyToSymbol(g_mma_k, &kk, sizeof(int)));
        CK(cudaMemcpyToSymbol(g_mma_n, &nn, sizeof(int)));
        char tag[32];
        snprintf(tag, sizeof(tag), "k%dn%d", kk, nn);
        run<11>(tm, 16, 32, 0, 1, tag);
        run<11>(tm, 96, 32, 0, 1, tag);
      }
    return 0;
  }
  for (int ctas : {96, 148}) {
    run<11>(tm, ctas, 32, 0, 1, "1x128");
    run<11>(tm16, ctas, 32, 0, -2, "2x64nov");
    run<11>(tm32, ctas, 32, 0, -4, "4x32nov");
  }
  if (getenv("BOXES_ONLY")) return 0;
  // hot L2 reads (router weight pattern): every CTA streams the same 256 KB / 128 KB
  run<11>(tm, 148, 16, 1, 1, "hot");
  run<11>(tm, 148, 8, 1, 1, "hot");
  run<11>(tm, 8, 16, 1, 1, "hot");
  run<11>(tm, 148, 1, 1, 1, "hot");
  // gate/up pattern with 64-row boxes vs one 128-row box
  run<11>(tm64, 96, 32, 0, 2, "2x64");
  run<11>(tm, 96, 32, 0, 1, "1x128");
  run<11>(tm64, 148, 32, 0, 2, "2x64");
  run<11>(tm, 148, 32, 0, 1, "1x128");
  // launch overhead floor
  run<4>(tm, 148, 1);
  for (int ctas : {16, 48, 96, 148}) {
    run<4>(tm, ctas, 32);
    run<8>(tm, ctas, 32);
    run<12>(tm, ctas, 32);
    run<13>(tm, ctas, 32);
  }
  // the T=1 layer's bytes (75.5 MB) split over all SMs at several granularities
  run<12>(tm, 148, 32);   // 148 x 512 KiB
  run<12>(tm, 148, 12);   // 148 x 192 KiB (a DN item)
  run<13>(tm, 148, 31);   // ~75 MB
  run<6>(tm, 148, 31);
  run<13>(tm, 96, 32);    // the tiny kernel's UP phase at T=1: 96 x 512 KiB = 50 MB
  run<13>(tm, 128, 12);   // its DN phase: 128 x 192 KiB = 25 MB
  run<13>(tm, 148, 200);  // long stream: steady-state ceiling
  return 0;
}

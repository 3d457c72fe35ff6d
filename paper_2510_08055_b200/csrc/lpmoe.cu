// liblpmoe.so — C ABI (include/lpmoe.h) over the sm_100a kernels.
// Host side: argument validation, workspace carving, TMA descriptor encoding
// (driver entry point, no -lcuda), launch configuration. No allocation, no
// host synchronisation: every entry point is stream-ordered and graph-safe.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <atomic>
#include <mutex>
#include <utility>

#include "../../include/lpmoe.h"
#include "experts_sm100.cuh"
#include "experts_pair_sm100.cuh"
#include "experts_tiny_sm100.cuh"
#include "decode_sm100.cuh"
#include "ep_p2p.cuh"
#include "norm.cuh"
#include "permute.cuh"
#include "route.cuh"
#include "union_counts.cuh"

namespace {

thread_local int g_code = LP_OK;
thread_local cudaEvent_t g_prof[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
thread_local int g_prof_n = 0;

inline void prof_mark(int i, cudaStream_t st) {
  if (g_prof_n >= 5) cudaEventRecord(g_prof[i], st);
}
thread_local char g_msg[512] = "ok";

int fail(int code, const char* fmt, ...) {
  g_code = code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
  return code;
}
int ok() {
  g_code = LP_OK;
  return LP_OK;
}
#define LP_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) return fail(LP_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define LP_CHECK_LAUNCH(name)                                                                       \
  do {                                                                                              \
    cudaError_t e_ = cudaGetLastError();                                                            \
    if (e_ != cudaSuccess) return fail(LP_ECUDA, "launch %s: %s", name, cudaGetErrorString(e_));    \
  } while (0)

constexpr int kTargetCtas = 148;  // B200 SM count; fixes ksplit independent of the device queried
constexpr size_t kAlign = 256;

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ------------------------------------------------------------------ shapes
// Tuning knobs read once from the environment (experiments only; defaults are the product).
int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}
bool use_pdl() {
  static const bool v = env_int("LPMOE_PDL", 1) != 0;
  return v;
}

// Token-tile width of the CTA-pair kernel in the compute-bound regime
// (LPMOE_PAIR_N: 256 default; 128 double-buffers the accumulator).
int pair_n() {
  static const int v = env_int("LPMOE_PAIR_N", 256);
  return v == 128 ? 128 : 256;
}

int pick_max_n(int S, int E) {
  static const int forced = env_int("LPMOE_MAX_N", 0);
  if (forced == 64 || forced == 128 || forced == 256) return forced;
  const int avg = (S + E - 1) / E;
  if (avg <= 40) return 64;
  if (avg <= 96) return 128;
  return pair_n();
}

// Workspace header (fixed offsets, independent of T): router tickets and the
// expert kernel's scheduler words. Must be zero-filled once after allocation;
// every kernel leaves it zeroed again.
constexpr int kMaxTokens = 262144;
constexpr size_t kSchedOff = (kMaxTokens / 32) * 4;          // 32 KiB reserved (formerly router tickets)
constexpr size_t kHeaderBytes = kSchedOff + 8192;            // + sched words (E+1 <= 257), decode combine counters
constexpr size_t kGbarOff = kSchedOff + 2048;                // fused router grid barrier (2 words)
// k_decode's own scheduler words (item counter, per-expert UP counters, exit counter): only it
// touches them and its last CTA leaves them zero (the other expert kernels leave `sched` dirty
// until the next k_scan* resets it)
constexpr size_t kDecodeSchedOff = kSchedOff + 2400;
constexpr size_t kDecodeCmbOff = kSchedOff + 4096;  // k_decode's fused-combine counters (<= 1024 words)
static_assert(kDecodeSchedOff + 4 * (lp::DecodeCfg::kExitWord + 1) <= kHeaderBytes, "decode scheduler words");

struct Layout {
  size_t chunk_hist, rank_local, ids, w, counts, offsets, slot_of, tok_of;
  size_t tile_prefix, tile_rows, sched, blk_cnt, x_perm, act, y_perm, total;
  int blk_n;  // fused-combine counters: T * ceil(H/256)
  int csize;         // router cluster size
  int chunk_tokens;  // tokens per permutation chunk (= router tile)
  int nchunks;
};

// Router tile (tokens per MMA N = permutation chunk): 16 while the batch is
// small (many CTAs, latency-bound), 64 once 16-token tiles would make every
// one of >= kRouterLargeTiles CTAs re-stream all of Wr from L2.
constexpr int kRouterLargeTiles = 149;  // > one wave of 16-token tiles on 148 SMs
int router_tile_tokens(int T, int E, int topk) {
  static const int forced = env_int("LPMOE_ROUTER_TN", 0);
  if (forced == 16 || forced == 64) return (forced == 64 && topk > 8) ? 16 : forced;
  // 64-token tiles need 6 x (16 KiB per 128 experts + 8 KiB) of ring: one m-tile (E <= 128) only
  if (topk > 8 || E > 128) return lp::kRouterN;
  return (T + lp::kRouterN - 1) / lp::kRouterN >= kRouterLargeTiles ? lp::kRouterTileLarge : lp::kRouterN;
}

// CTAs per router token tile: split H across a cluster while the grid is small.
int router_cluster(int ntiles, int H, int TN, int E) {
  static const int forced = env_int("LPMOE_ROUTER_CS", 0);  // tuning knob: 1, 2 or 4
  if (forced == 1 || forced == 2 || forced == 4) {
    const int e_pad = (E + 31) / 32 * 32;
    int cs = forced < (TN == lp::kRouterTileLarge ? 2 : 4) ? forced : (TN == lp::kRouterTileLarge ? 2 : 4);
    while (cs > 1 && ((H / 64) % cs != 0 || (4 / cs) * TN * e_pad > lp::router_part_floats() || TN / cs < 4)) cs >>= 1;
    return cs;
  }
  int cs = 1;
  const int cs_max = TN == lp::kRouterTileLarge ? 2 : 4;
  while (cs < cs_max && ntiles * cs * 2 <= kTargetCtas && (H / 64) % (cs * 2) == 0) {
    const int e_pad = (E + 31) / 32 * 32;
    const int ppc = 4 / (cs * 2);  // partial sums per CTA after doubling (npart <= 4)
    if (ppc * TN * e_pad > lp::router_part_floats() || (TN / (cs * 2)) < 4) break;
    cs *= 2;
  }
  return cs;
}

Layout make_layout(int T, int H, int I, int E, int topk) {
  Layout L{};
  const size_t S = static_cast<size_t>(T) * topk;
  L.chunk_tokens = router_tile_tokens(T, E, topk);
  L.csize = router_cluster((T + L.chunk_tokens - 1) / L.chunk_tokens, H, L.chunk_tokens, E);
  L.nchunks = (T + L.chunk_tokens - 1) / L.chunk_tokens;
  size_t o = kHeaderBytes;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, kAlign);
    return at;
  };
  L.chunk_hist = take(static_cast<size_t>(L.nchunks) * E * 4);
  L.rank_local = take(S * 4);
  L.ids = take(S * 4);
  L.w = take(S * 4);
  L.counts = take(static_cast<size_t>(E) * 4);
  L.offsets = take(static_cast<size_t>(E + 1) * 4);
  L.slot_of = take(S * 4);
  L.tok_of = take(S * 4);
  L.tile_prefix = take(static_cast<size_t>(E + 1) * 4);
  L.tile_rows = take(static_cast<size_t>(E) * 4);
  L.sched = kSchedOff;
  L.x_perm = take(S * H * 2);
  L.act = take(S * I * 2);
  L.y_perm = take(S * H * 2);
  L.blk_n = T * ((H + 255) / 256);
  L.blk_cnt = take(static_cast<size_t>(L.blk_n) * 4);
  L.total = o;
  return L;
}

int check_dims(int T, int H, int I, int E, int topk) {
  if (T < 0 || T > kMaxTokens) return fail(LP_EINVAL, "T must be in [0, %d], got %d", kMaxTokens, T);
  if (H <= 0 || H % 64) return fail(LP_EINVAL, "H must be a positive multiple of 64, got %d", H);
  if (I <= 0 || I % 64) return fail(LP_EINVAL, "I must be a positive multiple of 64, got %d", I);
  if (E < 1) return fail(LP_EINVAL, "E must be >= 1, got %d", E);
  if (E > lp::kMaxExperts) return fail(LP_EUNSUPPORTED, "E > %d not supported, got %d", lp::kMaxExperts, E);
  if (topk < 1 || topk > E) return fail(LP_EINVAL, "topk out of range: need 1 <= topk <= E, got %d", topk);
  if (topk > 32) return fail(LP_EUNSUPPORTED, "topk > 32 not supported, got %d", topk);
  return LP_OK;
}

// ------------------------------------------------------------------ TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

int get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) return fail(LP_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  return LP_OK;
}

// Encoded descriptors are a pure function of (address, shape, box): cache them,
// encoding is host time on every layer call otherwise (weights never move;
// activation buffers recur through the caching allocator). Bounded: cleared when full.
struct TmapKey {
  const void* ptr;
  uint64_t rows, cols;
  uint32_t box_rows;
  bool operator<(const TmapKey& o) const {
    if (ptr != o.ptr) return ptr < o.ptr;
    if (rows != o.rows) return rows < o.rows;
    if (cols != o.cols) return cols < o.cols;
    return box_rows < o.box_rows;
  }
};
std::mutex g_tmap_mu;
std::map<TmapKey, CUtensorMap> g_tmap_cache;

int encode_tmap(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);

// bf16 matrix [rows, cols] row-major, box = 64 cols (128 B, SWIZZLE_128B) x box_rows.
int make_tmap(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  const TmapKey key{ptr, rows, cols, box_rows};
  {
    std::lock_guard<std::mutex> lk(g_tmap_mu);
    auto it = g_tmap_cache.find(key);
    if (it != g_tmap_cache.end()) {
      *m = it->second;
      return LP_OK;
    }
  }
  int rc = encode_tmap(m, ptr, rows, cols, box_rows);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(g_tmap_mu);
  if (g_tmap_cache.size() >= 4096) g_tmap_cache.clear();
  g_tmap_cache.emplace(key, *m);
  return LP_OK;
}

int encode_tmap(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(LP_ECUDA, "cuTensorMapEncodeTiled(rows=%llu cols=%llu box_rows=%u) failed: %d",
                (unsigned long long)rows, (unsigned long long)cols, box_rows, (int)r);
  return LP_OK;
}

template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

// ------------------------------------------------------------------ device info
int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return kTargetCtas;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return kTargetCtas;
  return n;
}

// Kernels this library has launched (lp_launch_count): host-side evidence of
// which native kernels ran inside a timed region.
std::atomic<unsigned long long> g_launches{0};
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Launch with programmatic stream serialization (PDL): the kernel may begin
// while its stream predecessor drains; kernels pdl_wait() before global I/O.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = use_pdl() ? 1 : 0;
  int n = 1;
  if (cluster > 1) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    n = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  return launch_pdl_cluster(kernel, grid, block, smem, st, 1, std::forward<Args>(args)...);
}

// Dynamic shared-memory opt-in, set once per (kernel, device, size): the
// attribute call is host overhead on every layer of a decode step otherwise.
std::mutex g_smem_mu;
std::map<std::pair<const void*, int>, int> g_smem_set;

template <typename K>
int set_smem(K kernel, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  {
    std::lock_guard<std::mutex> lk(g_smem_mu);
    auto it = g_smem_set.find(key);
    if (it != g_smem_set.end() && it->second >= bytes) return LP_OK;
  }
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return fail(LP_ECUDA, "cudaFuncSetAttribute(smem=%d): %s", bytes, cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(g_smem_mu);
  int& v = g_smem_set[key];
  if (bytes > v) v = bytes;
  return LP_OK;
}

// ------------------------------------------------------------------ stages
template <int CS, int NV, int TN, bool FUSED>
int launch_router_t(const CUtensorMap& tm_wr, const CUtensorMap& tm_x, const lp::RouterParams& rp, int ntiles,
                    cudaStream_t st) {
  int rc;
  const int smem = lp::router_smem_bytes(rp.mtiles, TN);
  if ((rc = set_smem(lp::k_router<CS, NV, TN, FUSED>, smem))) return rc;
  LP_CUDA(launch_pdl_cluster(lp::k_router<CS, NV, TN, FUSED>, ntiles * CS, lp::router_threads(TN), smem, st, CS,
                             tm_wr, tm_x, rp));
  return LP_OK;
}

template <int CS, int TN, bool FUSED>
int launch_router_cs(const CUtensorMap& tm_wr, const CUtensorMap& tm_x, const lp::RouterParams& rp, int ntiles,
                     int e_pad, cudaStream_t st) {
  constexpr int TPC = TN / CS;
  constexpr int LPT = (128 / TPC) > 8 ? (128 / TPC) : 8;  // lanes per token (route.cuh)
  const int nv = (e_pad + LPT - 1) / LPT;
  if (nv <= 4) return launch_router_t<CS, 4, TN, FUSED>(tm_wr, tm_x, rp, ntiles, st);
  if (nv <= 8) return launch_router_t<CS, 8, TN, FUSED>(tm_wr, tm_x, rp, ntiles, st);
  if (nv <= 16) return launch_router_t<CS, 16, TN, FUSED>(tm_wr, tm_x, rp, ntiles, st);
  return launch_router_t<CS, 32, TN, FUSED>(tm_wr, tm_x, rp, ntiles, st);
}

template <bool FUSED>
int launch_router_dispatch(const CUtensorMap& tm_wr, const CUtensorMap& tm_x, const lp::RouterParams& rp,
                           int ntiles, int TN, int csize, int e_pad, cudaStream_t st) {
  if (TN == lp::kRouterTileLarge) {
    if (csize == 2) return launch_router_cs<2, lp::kRouterTileLarge, FUSED>(tm_wr, tm_x, rp, ntiles, e_pad, st);
    return launch_router_cs<1, lp::kRouterTileLarge, FUSED>(tm_wr, tm_x, rp, ntiles, e_pad, st);
  }
  switch (csize) {
    case 4: return launch_router_cs<4, lp::kRouterN, FUSED>(tm_wr, tm_x, rp, ntiles, e_pad, st);
    case 2: return launch_router_cs<2, lp::kRouterN, FUSED>(tm_wr, tm_x, rp, ntiles, e_pad, st);
    default: return launch_router_cs<1, lp::kRouterN, FUSED>(tm_wr, tm_x, rp, ntiles, e_pad, st);
  }
}

// Fused permutation outputs (router + grid barrier replaces k_scan + k_scatter).
struct FusedPermute {
  int32_t* counts;
  int32_t* offsets;
  int32_t* slot_of;
  int32_t* tok_of;
  void* x_perm;
  int max_n;
  int32_t* tile_prefix;
  int32_t* tile_rows;
  uint32_t* sched;
  uint32_t* gbar;
};

// Whether the router grid may run the permutation itself: every CTA must be
// co-resident for the grid barrier (<= one CTA per SM).
bool fused_route_ok(const Layout& L, int T, int E) {
  // Off by default: on B200 the post-barrier permutation (latency-bound row
  // copies from <= 148 CTAs) took as long as k_scan + k_scatter (T=576: 228 vs
  // 224 us per layer; T=8224: 881 vs 870 us). Kept for experiments.
  static const bool on = env_int("LPMOE_FUSED_ROUTE", 0) != 0;
  const int TN = L.chunk_tokens;
  const int grid = (T + TN - 1) / TN * L.csize;
  const int e_pad = (E + 31) / 32 * 32;
  return on && grid <= sm_count() && E % 4 == 0 && e_pad / 4 <= lp::router_threads(TN);
}

int launch_route(const void* x, const void* wr, int T, int H, int E, int topk, int renorm, int32_t* ids, float* w,
                 void* ws, const Layout& L, cudaStream_t st, const FusedPermute* fp = nullptr,
                 const void* warm = nullptr, size_t warm_bytes = 0, bool hist = true) {
  int rc;
  if ((rc = get_encode())) return rc;
  const int TN = L.chunk_tokens;
  CUtensorMap tm_wr, tm_x;
  if ((rc = make_tmap(&tm_wr, wr, E, H, 128))) return rc;
  if ((rc = make_tmap(&tm_x, x, T, H, TN))) return rc;
  const int mtiles = (E + 127) / 128;
  const int ntiles = (T + TN - 1) / TN;
  lp::RouterParams rp{T, H, E, topk, renorm, mtiles, ids, w, at<int32_t>(ws, L.chunk_hist),
                      at<int32_t>(ws, L.rank_local)};
  rp.ntiles = ntiles;
  if (!hist && !fp) {  // the permutation ranks entries itself (k_scan_slots)
    rp.tile_hist = nullptr;
    rp.rank_local = nullptr;
  }
  rp.warm = static_cast<const uint8_t*>(warm);
  rp.warm_bytes = warm ? warm_bytes : 0;
  const int e_pad = (E + 31) / 32 * 32;
  if (fp) {
    rp.max_n = fp->max_n;
    rp.counts = fp->counts;
    rp.offsets = fp->offsets;
    rp.slot_of = fp->slot_of;
    rp.tok_of = fp->tok_of;
    rp.x = static_cast<const __nv_bfloat16*>(x);
    rp.x_perm = static_cast<__nv_bfloat16*>(fp->x_perm);
    rp.tile_prefix = fp->tile_prefix;
    rp.tile_rows = fp->tile_rows;
    rp.sched = fp->sched;
    rp.gbar = fp->gbar;
    return launch_router_dispatch<true>(tm_wr, tm_x, rp, ntiles, TN, L.csize, e_pad, st);
  }
  return launch_router_dispatch<false>(tm_wr, tm_x, rp, ntiles, TN, L.csize, e_pad, st);
}

// Scan and slot maps fused into one launch when no x_perm is materialised
// (LPMOE_SCAN_SLOTS=0: the two-kernel k_scan + k_slots path).
bool use_scan_slots() {
  static const bool v = env_int("LPMOE_SCAN_SLOTS", 1) != 0;
  return v;
}

int launch_scan_slots(const int32_t* ids, int T, int E, int topk, int max_n, int32_t* counts, int32_t* offsets,
                      int32_t* slot_of, int32_t* tok_of, int32_t* tile_prefix, int32_t* tile_rows, uint32_t* sched,
                      cudaStream_t st) {
  const int S = T * topk;
  LP_CUDA(launch_pdl(lp::k_scan_slots, (S + lp::kScanSlotsThreads - 1) / lp::kScanSlotsThreads,
                     lp::kScanSlotsThreads, 0, st, ids, S, E, topk, max_n, counts, offsets, tile_prefix, tile_rows,
                     sched, slot_of, tok_of));
  return LP_OK;
}

// chunk_hist/rank_local come from the router (forward) or k_chunk_hist (standalone).
// Scan (one CTA): per-tile bases, counts, offsets, expert tile schedule. Scatter
// (one warp per routing entry): slot_of / tok_of and, if x_perm, the row copy.
int launch_scan_scatter(const int32_t* ids, const void* x, int T, int H, int E, int topk, int chunk_tokens,
                        int32_t* counts, int32_t* offsets, int32_t* slot_of, int32_t* tok_of, void* x_perm,
                        int32_t* chunk_hist, const int32_t* rank_local, int max_n, int32_t* tile_prefix,
                        int32_t* tile_rows, uint32_t* sched, cudaStream_t st, uint32_t* zero_buf = nullptr,
                        int zero_n = 0) {
  const int S = T * topk;
  const int nchunks = (T + chunk_tokens - 1) / chunk_tokens;
  const int n_hist = nchunks * E;
  const int smem = n_hist <= lp::kScanSmemInts ? n_hist * 4 : 0;
  // opt in whenever dynamic + static (s_part, 4 KiB) may pass the 48 KiB default (cached per device)
  if (smem > 0) {
    int rc;
    if ((rc = set_smem(lp::k_scan, lp::kScanSmemInts * 4))) return rc;
  }
  {
    const cudaError_t e = launch_pdl(lp::k_scan, 1, lp::kScanThreads, smem, st, chunk_hist, nchunks, E, max_n, counts,
                                     offsets, tile_prefix, tile_rows, sched, zero_buf, zero_n);
    if (e != cudaSuccess)
      return fail(LP_ECUDA, "k_scan launch (T=%d nchunks=%d E=%d smem=%d): %s", T, nchunks, E, smem,
                  cudaGetErrorString(e));
  }
  if (x_perm == nullptr) {
    LP_CUDA(launch_pdl(lp::k_slots, (S + 255) / 256, 256, 0, st, ids, static_cast<const int32_t*>(chunk_hist),
                       rank_local, static_cast<const int32_t*>(offsets), S, E, topk, chunk_tokens * topk, slot_of,
                       tok_of));
    return LP_OK;
  }
  LP_CUDA(launch_pdl(lp::k_scatter, (T + 7) / 8, 256, 0, st, ids, static_cast<const int32_t*>(chunk_hist), rank_local,
                     static_cast<const int32_t*>(offsets), static_cast<const __nv_bfloat16*>(x), S, E, topk, H,
                     chunk_tokens * topk, slot_of, tok_of, static_cast<__nv_bfloat16*>(x_perm)));
  return LP_OK;
}

template <int MAX_N, bool GATHER>
int launch_experts_t(const void* src, int src_rows, const void* act_in, int S, const void* w13, const void* w2,
                     int H, int I, int E, const lp::ExpertsParams& p, cudaStream_t st) {
  int rc;
  if ((rc = get_encode())) return rc;
  CUtensorMap tm_w13, tm_w2, tm_xsrc, tm_act;
  if ((rc = make_tmap(&tm_w13, w13, static_cast<uint64_t>(E) * 2 * I, H, lp::kTileM))) return rc;
  if ((rc = make_tmap(&tm_w2, w2, static_cast<uint64_t>(E) * H, I, lp::kTileM))) return rc;
  if ((rc = make_tmap(&tm_xsrc, src, src_rows, H, GATHER ? 1 : lp::kBoxRows))) return rc;
  if ((rc = make_tmap(&tm_act, act_in, S, I, lp::kBoxRows))) return rc;
  constexpr int smem = lp::ExpertsCfg<MAX_N>::kSmemBytes;
  if ((rc = set_smem(lp::k_experts<MAX_N, GATHER>, smem))) return rc;
  LP_CUDA(launch_pdl(lp::k_experts<MAX_N, GATHER>, sm_count(), lp::kExpertsThreads, smem, st, tm_w13, tm_w2, tm_xsrc,
                     tm_act, p));
  return LP_OK;
}

// Compute-bound regime (max_n == 256): the expert kernel on CTA pairs
// (cta_group::2, experts_pair_sm100.cuh). LPMOE_PAIR=0 selects k_experts<256>.
bool use_pair(int max_n, int H, int I) {
  static const int v = env_int("LPMOE_PAIR", 1);
  return v != 0 && (max_n == 256 || (max_n == 128 && pair_n() == 128)) && H % 512 == 0 && I % 256 == 0;
}

template <bool GATHER, int BN>
int launch_experts_pair(const void* src, int src_rows, int S, const void* act, const void* w13, const void* w2, int H,
                        int I, int E, const lp::ExpertsParams& p, cudaStream_t st) {
  int rc;
  if ((rc = get_encode())) return rc;
  CUtensorMap tm_w13, tm_w2, tm_x, tm_act;
  if ((rc = make_tmap(&tm_w13, w13, static_cast<uint64_t>(E) * 2 * I, H, lp::kTileM))) return rc;
  if ((rc = make_tmap(&tm_w2, w2, static_cast<uint64_t>(E) * H, I, lp::kTileM))) return rc;
  if ((rc = make_tmap(&tm_x, src, src_rows, H, lp::kBoxRows))) return rc;
  if ((rc = make_tmap(&tm_act, act, S, I, lp::kBoxRows))) return rc;
  constexpr int smem = lp::PairCfg<BN>::kSmemBytes;
  if ((rc = set_smem(lp::k_experts_pair<GATHER, BN>, smem))) return rc;
  const int sms = sm_count();
  // pairs that fit at once (one CTA per SM), per device and kernel instance
  static std::mutex mu;
  static int cached[64] = {};  // 0 = not computed yet
  int dev = 0;
  LP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  int& max_clusters = cached[dev & 63];
  if (max_clusters <= 0) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(sms & ~1);
    cfg.blockDim = dim3(lp::kExpertsThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, lp::k_experts_pair<GATHER, BN>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = sms / 2;
    }
    max_clusters = n < sms / 2 ? n : sms / 2;
  }
  LP_CUDA(launch_pdl_cluster(lp::k_experts_pair<GATHER, BN>, 2 * max_clusters, lp::kExpertsThreads, smem, st, 2, tm_w13, tm_w2,
                             tm_x, tm_act, p));
  return LP_OK;
}

// Decode-size batches (<= 1 routed token per expert on average): half-size
// items on more SMs (experts_tiny_sm100.cuh). LPMOE_TINY=0 disables.
bool use_tiny(int S, int E, int H, int I) {
  static const int v = env_int("LPMOE_TINY", 1);
  return v != 0 && S <= E && H % 64 == 0 && I % 64 == 0;
}

int launch_experts_tiny(const void* x, const int32_t* tok_of, int S, const void* act, const void* w13, const void* w2,
                        int H, int I, int E, lp::ExpertsParams p, cudaStream_t st) {
  int rc;
  if ((rc = get_encode())) return rc;
  CUtensorMap tm_w13h, tm_w2, tm_act;
  if ((rc = make_tmap(&tm_w13h, w13, static_cast<uint64_t>(E) * 2 * I, H, 64))) return rc;
  if ((rc = make_tmap(&tm_w2, w2, static_cast<uint64_t>(E) * H, I, lp::kTileM))) return rc;
  if ((rc = make_tmap(&tm_act, act, S, I, lp::TinyCfg::kN))) return rc;
  constexpr int smem = lp::TinyCfg::kSmemBytes;
  if ((rc = set_smem(lp::k_experts_tiny, smem))) return rc;
  p.xsrc = static_cast<const __nv_bfloat16*>(x);
  p.tok_of = tok_of;
  LP_CUDA(launch_pdl(lp::k_experts_tiny, sm_count(), lp::TinyCfg::kThreads, smem, st, tm_w13h, tm_w2, tm_act, p));
  return LP_OK;
}

// Decode-size layers (T <= 16, T*topk <= E <= 128, H % 256 == 0) run router,
// permutation and the expert stream in ONE launch (decode_sm100.cuh), bit-
// identical to k_router<4, 4, 16> + k_scan_slots + k_experts_tiny. LPMOE_DECODE=0
// disables. Knobs (B200, T=1 / 2 / 8 layer us, profiles/r02): LPMOE_DECODE_W2_WARM=1 L2-warms the hit
// experts' W2 during the UP phase (off: 32.3 vs 34.2 at T=1 — it competes with the UP stream);
// LPMOE_DECODE_DNC=0 disables the block-diagonal DN+combine items (on: 31.0 vs 31.9 at T=1);
// DN act rows are copied by the gather warps (cp.async; the TMA alternative measured 32.8 / 41.9 /
// 91.7 vs 31.0 / 41.6 / 86.7 us and was removed). LPMOE_DECODE_KS=1 selects the 11 x 18 KiB ring.
bool use_decode(int T, int H, int I, int E, int topk) {
  static const int v = env_int("LPMOE_DECODE", 1);
  return v != 0 && T >= 1 && T <= lp::DecodeCfg::kMaxT && T * topk <= E && E <= lp::DecodeCfg::kMaxE &&
         H % 256 == 0 && I % 64 == 0 && T * (H / 256) <= 1024;
}

int launch_decode(const void* x, const void* wr, const void* w13, const void* w2, int T, int H, int I, int E,
                  int topk, int renorm, int32_t* ids, float* w, int32_t* counts, int32_t* offsets, int32_t* slot_of,
                  int32_t* tok_of, void* act, void* y_perm, uint32_t* sched, void* y, uint32_t* cmb, int wpol,
                  cudaStream_t st) {
  static const int warm = env_int("LPMOE_DECODE_W2_WARM", 0);
  static const int dnc = env_int("LPMOE_DECODE_DNC", 1);
  // k-blocks per ring stage (decode_sm100.cuh DecodeRing): 2 = 5 stages of 36 KiB (default), 1 = 11 of 18 KiB
  static const int ks_env = env_int("LPMOE_DECODE_KS", 2);
  const int ks = ks_env == 1 ? 1 : 2;
  int rc;
  if ((rc = get_encode())) return rc;
  const int S = T * topk;
  CUtensorMap tm_wr, tm_x, tm_w13h, tm_w2, tm_act;
  if ((rc = make_tmap(&tm_wr, wr, E, H, 128))) return rc;
  if ((rc = make_tmap(&tm_x, x, T, H, lp::DecodeCfg::kN))) return rc;
  if ((rc = make_tmap(&tm_w13h, w13, static_cast<uint64_t>(E) * 2 * I, H, 64))) return rc;
  if ((rc = make_tmap(&tm_w2, w2, static_cast<uint64_t>(E) * H, I, lp::kTileM))) return rc;
  if ((rc = make_tmap(&tm_act, act, S, I, lp::DecodeCfg::kN))) return rc;
  // W2 boxes of 8/16/32/64 rows: the block-diagonal DN tiles of S <= 16 (R rows per hit expert)
  CUtensorMap tm_w2r[4];
  for (int i = 0; i < 4; ++i)
    if ((rc = make_tmap(&tm_w2r[i], w2, static_cast<uint64_t>(E) * H, I, 8u << i))) return rc;
  const int smem = ks == 1 ? lp::DecodeRing<1>::kSmemBytes : lp::DecodeRing<2>::kSmemBytes;
  static const int forced_cs = env_int("LPMOE_DECODE_CS", 0);
  // B200, two-k-block ring (profiles/r02/probe/decode_cs_ks2.txt): 4-CTA clusters (132 SMs, half the Wr
  // bytes per CTA) win up to T=12 (T=1 28.4 vs 30.8 us, T=4 54.5 vs 57.5, T=8 85.0 vs 86.3, T=12 111.6 vs
  // 112.4), pairs (148 SMs streaming) at T=16 (130.2 vs 130.9); with the one-k-block ring pairs won from T=4
  const int cs = forced_cs == 2 || forced_cs == 4 ? forced_cs : (T <= 12 ? 4 : 2);
  auto kern = cs == 4 ? (ks == 1 ? lp::k_decode<4, 1> : lp::k_decode<4, 2>)
                      : (ks == 1 ? lp::k_decode<2, 1> : lp::k_decode<2, 2>);
  if ((rc = set_smem(kern, smem))) return rc;
  const lp::DecodeParams p{T, H, I, E, topk, renorm, static_cast<const __nv_bfloat16*>(x),
                           static_cast<const uint8_t*>(w2), ids, w, counts, offsets, slot_of, tok_of,
                           static_cast<__nv_bfloat16*>(act), static_cast<__nv_bfloat16*>(y_perm), sched,
                           static_cast<__nv_bfloat16*>(y), cmb, wpol, warm != 0 ? 1 : 0, dnc != 0 ? 1 : 0};
  // clusters of 4 that are co-resident (GPC boundaries can leave SMs that no 4-CTA cluster fits):
  // a second wave would repeat the routing prologue after the first wave's stream
  static std::mutex mu;
  static int cached[64][2][2] = {};
  int dev = 0;
  LP_CUDA(cudaGetDevice(&dev));
  int grid;
  {
    std::lock_guard<std::mutex> lock(mu);
    int& g = cached[dev & 63][cs == 4][ks == 2];
    if (g <= 0) {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(sm_count() / cs * cs);
      cfg.blockDim = dim3(lp::DecodeCfg::kThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = sm_count() / cs;
      }
      g = n * cs;
    }
    grid = g;
  }
  LP_CUDA(launch_pdl_cluster(kern, grid, lp::DecodeCfg::kThreads, smem, st, cs, tm_wr, tm_x, tm_w13h, tm_w2, tm_act,
                             tm_w2r[0], tm_w2r[1], tm_w2r[2], tm_w2r[3], p));
  return LP_OK;
}

// k-blocks of the first item's W13 warmed in L2 before pdl_wait (2 x 16 KiB each);
// tuning knob LPMOE_PREFETCH_KB (default 32 = the whole first UP item, 1 MiB per CTA;
// B200, T=576: 210.4-211.5 vs 211.8-212.2 us at 16, e2e 208 vs 210.5).
int prefetch_kblocks() {
  static const int v = [] {
    const char* s = getenv("LPMOE_PREFETCH_KB");
    return s ? atoi(s) : 32;
  }();
  return v;
}

// Bytes of W13 (from its start, i.e. the first UP items in claim order) the
// router warms in L2 for the expert kernel. Knob LPMOE_L2_WARM_MB; default 0:
// measured on B200, the router grid only completes once its bulk prefetches
// have landed, so the warm-up lengthens the routing critical path as much as
// it shortens the expert stream (T=576: 224.7 us at 0 MB vs 227.5 at 80 MB).
size_t l2_warm_bytes(size_t w13_bytes) {
  static const long mb = env_int("LPMOE_L2_WARM_MB", 0);
  const size_t b = mb > 0 ? static_cast<size_t>(mb) << 20 : 0;
  return (b < w13_bytes ? b : w13_bytes) & ~size_t(15);
}

// Token rows reach the expert kernel gathered straight from x by its cp.async
// warps (no x_perm round trip) in the memory-bound regime (max_n == 64);
// at larger tiles the per-SM LSU in-flight limit makes the gather slower than
// TMA boxes from a materialised x_perm (B200, T=2048: 333 vs 321 us; T=8224:
// 858 vs 824 us; T=576: 212 vs 221 us). LPMOE_GATHER=0/1 forces it off/on.
bool use_gather(int max_n) {
  static const int v = env_int("LPMOE_GATHER", -1);
  static const int pair_v = env_int("LPMOE_PAIR_GATHER", 0);
  return v < 0 ? (max_n == 64 || (max_n == 256 && pair_v != 0)) : v != 0;
}
int env_lookahead() {
  static const int v = env_int("LPMOE_LOOKAHEAD", 0);
  return v;
}
int env_wpol() {
  static const int v = env_int("LPMOE_WEVICT_FIRST", 1);
  return v;
}

// Optional combine fused into the expert kernel's DN epilogue (experts_sm100.cuh).
struct FusedCombine {
  void* y = nullptr;
  const int32_t* slot_tok = nullptr;
  const int32_t* slot_of = nullptr;
  const float* wgt = nullptr;
  uint32_t* blk_cnt = nullptr;
  int topk = 0;
};
bool use_fused_combine() {
  // Off by default: measured slower on B200 (the DN epilogue is on the critical
  // path: +10 us at T=576, +140 us at T=8224 vs the separate k_combine).
  static const bool v = env_int("LPMOE_FUSED_COMBINE", 0) != 0;
  return v;
}

// src: [src_rows, H] token rows; slot s reads row tok_of[s] (tok_of == nullptr: row s).
int launch_experts(const void* src, int src_rows, const int32_t* tok_of, int S, const void* w13, const void* w2,
                   int H, int I, int E, int max_n, const int32_t* offsets, const int32_t* tile_prefix,
                   const int32_t* tile_rows, uint32_t* sched, void* act, void* y_perm, cudaStream_t st,
                   const FusedCombine& fc = FusedCombine{}, int warm_rows = 0) {
  lp::ExpertsParams p{H,       I,           E,        tok_of, offsets, tile_prefix, tile_rows,
                      static_cast<__nv_bfloat16*>(act), static_cast<__nv_bfloat16*>(y_perm), sched,
                      prefetch_kblocks(), warm_rows, env_lookahead(), env_wpol(), static_cast<__nv_bfloat16*>(fc.y),
                      fc.slot_tok, fc.slot_of, fc.wgt, fc.blk_cnt, fc.topk, nullptr};
  if (fc.y == nullptr && use_pair(max_n, H, I)) {
    if (tok_of) {  // rows gathered by the kernel's cp.async warps from the unpermuted source
      p.xsrc = static_cast<const __nv_bfloat16*>(src);
      return launch_experts_pair<true, 256>(src, src_rows, S, act, w13, w2, H, I, E, p, st);
    }
    if (max_n == 128) return launch_experts_pair<false, 128>(src, S, S, act, w13, w2, H, I, E, p, st);
    return launch_experts_pair<false, 256>(src, S, S, act, w13, w2, H, I, E, p, st);
  }
  if (tok_of) {  // rows gathered by the kernel's cp.async warps from the unpermuted source
    p.xsrc = static_cast<const __nv_bfloat16*>(src);
    switch (max_n) {
      case 64: return launch_experts_t<64, true>(src, src_rows, act, S, w13, w2, H, I, E, p, st);
      case 128: return launch_experts_t<128, true>(src, src_rows, act, S, w13, w2, H, I, E, p, st);
      default: return launch_experts_t<256, true>(src, src_rows, act, S, w13, w2, H, I, E, p, st);
    }
  }
  switch (max_n) {
    case 64: return launch_experts_t<64, false>(src, src_rows, act, S, w13, w2, H, I, E, p, st);
    case 128: return launch_experts_t<128, false>(src, src_rows, act, S, w13, w2, H, I, E, p, st);
    default: return launch_experts_t<256, false>(src, src_rows, act, S, w13, w2, H, I, E, p, st);
  }
}

// Tile schedule from externally supplied offsets (staged / expert-parallel use).
__global__ void k_plan(const int32_t* __restrict__ offsets, int E, int max_n, int32_t* __restrict__ tile_prefix,
                       int32_t* __restrict__ tile_rows, uint32_t* __restrict__ sched) {
  lp::pdl_trigger();  // PDL: the expert kernel's prologue (TMEM, barriers, L2 weight prefetch) overlaps
  lp::pdl_wait();
  extern __shared__ int32_t s_til[];
  const int e = threadIdx.x;
  const int n = (e < E) ? offsets[e + 1] - offsets[e] : 0;
  const int nt = (n > 0) ? (n + max_n - 1) / max_n : 0;
  s_til[e] = nt;
  __syncthreads();
  for (int o = 1; o < static_cast<int>(blockDim.x); o <<= 1) {
    const int a = (e >= o) ? s_til[e - o] : 0;
    __syncthreads();
    s_til[e] += a;
    __syncthreads();
  }
  if (e < E) {
    tile_prefix[e] = s_til[e] - nt;
    const int per = nt ? (n + nt - 1) / nt : 0;
    tile_rows[e] = min(max_n, (per + 15) & ~15);
    if (e == E - 1) tile_prefix[E] = s_til[e];
  }
  for (int i = e; i <= E; i += blockDim.x) sched[i] = 0u;
}


}  // namespace

// ====================================================================== C ABI
extern "C" {

uint64_t lp_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* lp_version(void) { return "lpmoe 0.1 sm_100a"; }

int lp_last_error(char* buf, size_t n) {
  if (buf && n) {
    strncpy(buf, g_msg, n - 1);
    buf[n - 1] = '\0';
  }
  return g_code;
}

size_t lp_moe_workspace_bytes(int T, int H, int I, int E, int topk) {
  if (T < 0 || H <= 0 || I <= 0 || E <= 0 || topk <= 0) return 0;
  return make_layout(T, H, I, E, topk).total;
}

int lp_moe_route(const void* x, const void* wr, int T, int H, int E, int topk, int renorm, int32_t* ids, float* w,
                 void* ws, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_dims(T, H, 128, E, topk))) return rc;
  if (T == 0) return ok();
  if (!x || !wr || !ids || !w || !ws) return fail(LP_EINVAL, "lp_moe_route: null pointer argument");
  if (!aligned16(x) || !aligned16(wr)) return fail(LP_EINVAL, "lp_moe_route: x/wr must be 16-byte aligned");
  const Layout L = make_layout(T, H, 128, E, topk);
  if (ws_bytes < L.ids) return fail(LP_EINVAL, "lp_moe_route: workspace %zu < %zu bytes", ws_bytes, L.ids);
  // no per-tile histogram: a standalone lp_moe_permute recomputes what it needs from the ids
  // (k_scan_slots, or k_chunk_hist on the chunked path), so the router's would never be read
  if ((rc = launch_route(x, wr, T, H, E, topk, renorm, ids, w, ws, L, static_cast<cudaStream_t>(stream), nullptr,
                         nullptr, 0, false)))
    return rc;
  return ok();
}

int lp_moe_permute(const int32_t* ids, const void* x, int T, int H, int E, int topk, int32_t* counts,
                   int32_t* offsets, int32_t* slot_of, int32_t* tok_of, void* x_perm, void* ws, size_t ws_bytes,
                   void* stream) {
  int rc;
  if ((rc = check_dims(T, H, 128, E, topk))) return rc;
  if (!ids || !counts || !offsets || !slot_of || !tok_of || !ws || (x_perm && !x))
    return fail(LP_EINVAL, "lp_moe_permute: null pointer argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (T == 0) {
    LP_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, st));
    LP_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (E + 1), st));
    return ok();
  }
  const Layout L = make_layout(T, H, 128, E, topk);
  if (ws_bytes < L.x_perm) return fail(LP_EINVAL, "lp_moe_permute: workspace %zu < %zu bytes", ws_bytes, L.x_perm);
  const int max_n = pick_max_n(T * topk, E);
  if (!x_perm && use_scan_slots() && T * topk <= 32768) {  // every CTA reads all ids: small batches only
    if ((rc = launch_scan_slots(ids, T, E, topk, max_n, counts, offsets, slot_of, tok_of,
                                at<int32_t>(ws, L.tile_prefix), at<int32_t>(ws, L.tile_rows),
                                at<uint32_t>(ws, L.sched), st)))
      return rc;
    return ok();
  }
  int32_t* chunk_hist = at<int32_t>(ws, L.chunk_hist);
  int32_t* rank_local = at<int32_t>(ws, L.rank_local);
  const int chunk = L.chunk_tokens * topk;
  count_launch();
  lp::k_chunk_hist<<<(L.nchunks + lp::kHistWarps - 1) / lp::kHistWarps, 32 * lp::kHistWarps,
                     lp::kHistWarps * E * sizeof(int32_t), st>>>(ids, T * topk, E, chunk, chunk_hist, rank_local);
  LP_CHECK_LAUNCH("k_chunk_hist");
  if ((rc = launch_scan_scatter(ids, x, T, H, E, topk, L.chunk_tokens, counts, offsets, slot_of, tok_of, x_perm,
                                chunk_hist,
                                rank_local, max_n, at<int32_t>(ws, L.tile_prefix), at<int32_t>(ws, L.tile_rows),
                                at<uint32_t>(ws, L.sched), st)))
    return rc;
  return ok();
}

int lp_moe_experts_rows(const void* x_perm, const int32_t* offsets, int S, int S_hint, const void* w13,
                        const void* w2, int H, int I, int E, void* act, void* y_perm, void* ws, size_t ws_bytes,
                        void* stream) {
  int rc;
  if ((rc = check_dims(0, H, I, E, 1))) return rc;
  if (S < 0 || S_hint < 0) return fail(LP_EINVAL, "S and S_hint must be >= 0, got %d, %d", S, S_hint);
  if (S == 0) return ok();
  if (!x_perm || !offsets || !w13 || !w2 || !act || !y_perm || !ws)
    return fail(LP_EINVAL, "lp_moe_experts: null pointer argument");
  if (!aligned16(x_perm) || !aligned16(w13) || !aligned16(w2) || !aligned16(act) || !aligned16(y_perm))
    return fail(LP_EINVAL, "lp_moe_experts: tensors must be 16-byte aligned");
  const size_t blk = align_up(static_cast<size_t>(E + 1) * 4, kAlign);
  const size_t need = kHeaderBytes + 2 * blk;
  if (ws_bytes < need) return fail(LP_EINVAL, "lp_moe_experts: workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* tile_prefix = at<int32_t>(ws, kHeaderBytes);
  int32_t* tile_rows = at<int32_t>(ws, kHeaderBytes + blk);
  uint32_t* sched = at<uint32_t>(ws, kSchedOff);
  const int max_n = pick_max_n(S_hint > 0 ? S_hint : S, E);
  const int sb = (E + 31) / 32 * 32;
  LP_CUDA(launch_pdl(k_plan, 1, sb, sb * sizeof(int32_t), st, offsets, E, max_n, tile_prefix, tile_rows, sched));
  if ((rc = launch_experts(x_perm, S, nullptr, S, w13, w2, H, I, E, max_n, offsets, tile_prefix, tile_rows, sched,
                           act, y_perm,
                           st)))
    return rc;
  return ok();
}

int lp_moe_experts(const void* x_perm, const int32_t* offsets, int S, const void* w13, const void* w2, int H, int I,
                   int E, void* act, void* y_perm, void* ws, size_t ws_bytes, void* stream) {
  return lp_moe_experts_rows(x_perm, offsets, S, S, w13, w2, H, I, E, act, y_perm, ws, ws_bytes, stream);
}

int lp_moe_combine(const void* y_perm, const int32_t* slot_of, const float* w, int T, int H, int topk, void* y,
                   void* stream) {
  if (T < 0 || H <= 0 || H % 8 || topk < 1) return fail(LP_EINVAL, "lp_moe_combine: bad shape T=%d H=%d topk=%d", T, H, topk);
  if (topk > 32) return fail(LP_EUNSUPPORTED, "lp_moe_combine: topk=%d > 32", topk);
  if (T == 0) return ok();
  if (!y_perm || !slot_of || !w || !y) return fail(LP_EINVAL, "lp_moe_combine: null pointer argument");
  if (!aligned16(y_perm) || !aligned16(y)) return fail(LP_EINVAL, "lp_moe_combine: y_perm and y must be 16-byte aligned");
  if (H / 8 > 32 * lp::kCombineThreads) return fail(LP_EUNSUPPORTED, "lp_moe_combine: H too large");
  LP_CUDA(launch_pdl(lp::k_combine, T, lp::kCombineThreads, 0, static_cast<cudaStream_t>(stream),
                     static_cast<const __nv_bfloat16*>(y_perm), slot_of, w, T, topk, H, static_cast<__nv_bfloat16*>(y)));
  return ok();
}

int lp_moe_forward(const void* x, const void* wr, const void* w13, const void* w2, int T, int H, int I, int E,
                   int topk, int renorm, void* y, int32_t* ids, float* w, int32_t* counts, void* ws, size_t ws_bytes,
                   void* stream) {
  int rc;
  if ((rc = check_dims(T, H, I, E, topk))) return rc;
  if (T == 0) {  // empty batch: no expert is hit
    if (counts) LP_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, static_cast<cudaStream_t>(stream)));
    return ok();
  }
  if (!x || !wr || !w13 || !w2 || !y || !ws) return fail(LP_EINVAL, "lp_moe_forward: null pointer argument");
  if (!aligned16(x) || !aligned16(wr) || !aligned16(w13) || !aligned16(w2) || !aligned16(y) || !aligned16(ws))
    return fail(LP_EINVAL, "lp_moe_forward: tensors and workspace must be 16-byte aligned");
  const Layout L = make_layout(T, H, I, E, topk);
  if (ws_bytes < L.total) return fail(LP_EINVAL, "lp_moe_forward: workspace %zu < %zu bytes", ws_bytes, L.total);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!ids) ids = at<int32_t>(ws, L.ids);
  if (!w) w = at<float>(ws, L.w);
  if (!counts) counts = at<int32_t>(ws, L.counts);
  const int S = T * topk;
  const bool tiny = !use_fused_combine() && use_gather(pick_max_n(S, E)) && use_tiny(S, E, H, I);
  const int max_n = tiny ? lp::TinyCfg::kN : pick_max_n(S, E);
  int32_t* offsets = at<int32_t>(ws, L.offsets);
  int32_t* slot_of = at<int32_t>(ws, L.slot_of);
  int32_t* tok_of = at<int32_t>(ws, L.tok_of);
  // Token rows reach the expert kernel either materialised in slot order
  // (x_perm, one scatter pass) or gathered straight from x by TMA (tok_of).
  const bool gather = tiny || use_gather(max_n);
  const bool fused = use_fused_combine();
  const bool fused_route = !fused && fused_route_ok(L, T, E);
  if (!fused && !fused_route && use_decode(T, H, I, E, topk)) {  // one launch + combine
    prof_mark(0, st);
    prof_mark(1, st);
    prof_mark(2, st);
    // the combine runs inside k_decode's DN epilogues unless LPMOE_DECODE_COMBINE=0
    static const bool fuse_combine = env_int("LPMOE_DECODE_COMBINE", 1) != 0;
    if ((rc = launch_decode(x, wr, w13, w2, T, H, I, E, topk, renorm, ids, w, counts, offsets, slot_of, tok_of,
                            at<void>(ws, L.act), at<void>(ws, L.y_perm), at<uint32_t>(ws, kDecodeSchedOff),
                            fuse_combine ? y : nullptr, at<uint32_t>(ws, kDecodeCmbOff), env_wpol(), st)))
      return rc;
    prof_mark(3, st);
    if (!fuse_combine && (rc = lp_moe_combine(at<void>(ws, L.y_perm), slot_of, w, T, H, topk, y, stream))) return rc;
    prof_mark(4, st);
    return ok();
  }
  const size_t warm = l2_warm_bytes(static_cast<size_t>(E) * 2 * I * H * 2);
  prof_mark(0, st);
  if (fused_route) {  // router + grid barrier + permutation in one launch
    const FusedPermute fp{counts, offsets, slot_of, tok_of, gather ? nullptr : at<void>(ws, L.x_perm), max_n,
                          at<int32_t>(ws, L.tile_prefix), at<int32_t>(ws, L.tile_rows), at<uint32_t>(ws, L.sched),
                          at<uint32_t>(ws, kGbarOff)};
    if ((rc = launch_route(x, wr, T, H, E, topk, renorm, ids, w, ws, L, st, &fp, w13, warm))) return rc;
    prof_mark(1, st);
  } else {
    const bool ids_scan = gather && !fused && use_scan_slots() && S <= 32768;  // every CTA reads all ids
    if ((rc = launch_route(x, wr, T, H, E, topk, renorm, ids, w, ws, L, st, nullptr, w13, warm, !ids_scan)))
      return rc;
    prof_mark(1, st);
    if (ids_scan) {
      if ((rc = launch_scan_slots(ids, T, E, topk, max_n, counts, offsets, slot_of, tok_of,
                                  at<int32_t>(ws, L.tile_prefix), at<int32_t>(ws, L.tile_rows),
                                  at<uint32_t>(ws, L.sched), st)))
        return rc;
    } else if ((rc = launch_scan_scatter(ids, x, T, H, E, topk, L.chunk_tokens, counts, offsets, slot_of, tok_of,
                                  gather ? nullptr : at<void>(ws, L.x_perm),
                                  at<int32_t>(ws, L.chunk_hist), at<int32_t>(ws, L.rank_local), max_n,
                                  at<int32_t>(ws, L.tile_prefix), at<int32_t>(ws, L.tile_rows),
                                  at<uint32_t>(ws, L.sched), st, fused ? at<uint32_t>(ws, L.blk_cnt) : nullptr,
                                  fused ? L.blk_n : 0)))
      return rc;
  }
  FusedCombine fc;
  if (fused) fc = FusedCombine{y, tok_of, slot_of, w, at<uint32_t>(ws, L.blk_cnt), topk};
  prof_mark(2, st);
  if (tiny) {
    const lp::ExpertsParams p{H, I, E, tok_of, offsets, at<int32_t>(ws, L.tile_prefix), at<int32_t>(ws, L.tile_rows),
                              at<__nv_bfloat16>(ws, L.act), at<__nv_bfloat16>(ws, L.y_perm), at<uint32_t>(ws, L.sched),
                              0, 0, 0, env_wpol(), nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr};
    if ((rc = launch_experts_tiny(x, tok_of, S, at<void>(ws, L.act), w13, w2, H, I, E, p, st))) return rc;
  } else if ((rc = launch_experts(gather ? x : at<void>(ws, L.x_perm), gather ? T : S, gather ? tok_of : nullptr, S, w13,
                           w2, H, I, E, max_n, offsets,
                           at<int32_t>(ws, L.tile_prefix),
                           at<int32_t>(ws, L.tile_rows), at<uint32_t>(ws, L.sched), at<void>(ws, L.act),
                           at<void>(ws, L.y_perm), st, fc, static_cast<int>(warm / (static_cast<size_t>(H) * 2)))))
    return rc;
  prof_mark(3, st);
  if (!fused && (rc = lp_moe_combine(at<void>(ws, L.y_perm), slot_of, w, T, H, topk, y, stream))) return rc;
  prof_mark(4, st);
  return ok();
}

int lp_union_counts_uniform(const double* u, int trials, int batch, int k, int E, int64_t* out, void* stream) {
  if (trials < 0 || batch < 0 || E < 1 || E > 1024 || k < 1 || k > E)
    return fail(LP_EINVAL, "lp_union_counts_uniform: bad shape trials=%d batch=%d k=%d E=%d", trials, batch, k, E);
  if (k > 64) return fail(LP_EUNSUPPORTED, "lp_union_counts_uniform: k > 64 not supported");
  if (trials == 0) return ok();
  if (!out || (batch > 0 && !u)) return fail(LP_EINVAL, "lp_union_counts_uniform: null pointer argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t sm = ((E + 31) / 32) * sizeof(uint32_t);
  count_launch();
  if (k <= 16)
    lp::k_union_uniform<16><<<trials, lp::kUnionThreads, sm, st>>>(u, batch, k, E, out);
  else
    lp::k_union_uniform<64><<<trials, lp::kUnionThreads, sm, st>>>(u, batch, k, E, out);
  LP_CHECK_LAUNCH("k_union_uniform");
  return ok();
}

int lp_union_counts_weighted(const double* u, int trials, int batch, int k, int E, const double* weights,
                             int64_t* out, void* stream) {
  if (trials < 0 || batch < 0 || E < 1 || E > 1024 || k < 1 || k > E)
    return fail(LP_EINVAL, "lp_union_counts_weighted: bad shape trials=%d batch=%d k=%d E=%d", trials, batch, k, E);
  if (trials == 0) return ok();
  if (!out || !weights || (batch > 0 && !u)) return fail(LP_EINVAL, "lp_union_counts_weighted: null pointer argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t sm = E * sizeof(double) + ((E + 31) / 32) * sizeof(uint32_t);
  count_launch();
  lp::k_union_weighted<<<trials, lp::kUnionThreads, sm, st>>>(u, batch, k, E, weights, out);
  LP_CHECK_LAUNCH("k_union_weighted");
  return ok();
}

int lp_add_rmsnorm(void* h, const void* delta, void* xn, int T, int H, float eps, void* stream) {
  if (T < 0 || H <= 0 || H % 8) return fail(LP_EINVAL, "lp_add_rmsnorm: bad shape T=%d H=%d", T, H);
  if (!(eps >= 0.f)) return fail(LP_EINVAL, "lp_add_rmsnorm: eps must be >= 0");
  if (T == 0) return ok();
  if (!h || !xn) return fail(LP_EINVAL, "lp_add_rmsnorm: null pointer argument");
  if (!aligned16(h) || !aligned16(xn) || (delta && !aligned16(delta)))
    return fail(LP_EINVAL, "lp_add_rmsnorm: tensors must be 16-byte aligned");
  LP_CUDA(launch_pdl(lp::k_add_rmsnorm, (T + lp::kNormWarps - 1) / lp::kNormWarps, 32 * lp::kNormWarps, 0,
                     static_cast<cudaStream_t>(stream), static_cast<__nv_bfloat16*>(h),
                     static_cast<const __nv_bfloat16*>(delta), static_cast<__nv_bfloat16*>(xn), T, H, eps));
  return ok();
}

int lp_profile_events(void* const* events, int n) {
  if (n < 0 || (n > 0 && !events)) return fail(LP_EINVAL, "lp_profile_events: bad arguments");
  g_prof_n = n >= 5 ? 5 : 0;
  for (int i = 0; i < 5; ++i) g_prof[i] = (g_prof_n && i < n) ? static_cast<cudaEvent_t>(events[i]) : nullptr;
  return ok();
}

// ---------------------------------------------------------------- expert parallelism over peer memory
int lp_ipc_handle(const void* dptr, void* handle64, size_t* offset) {
  if (!dptr || !handle64 || !offset) return fail(LP_EINVAL, "lp_ipc_handle: null pointer argument");
  // the handle names the whole allocation (e.g. a caching-allocator segment):
  // report dptr's offset from its base so the importer can rebase
  static PFN_cuMemGetAddressRange_v3020 range_fn = nullptr;
  if (!range_fn) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(LP_ECUDA, "cuMemGetAddressRange entry point unavailable");
    range_fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS)
    return fail(LP_ECUDA, "cuMemGetAddressRange failed");
  *offset = reinterpret_cast<CUdeviceptr>(dptr) - base;
  cudaIpcMemHandle_t h;
  LP_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, sizeof(h));
  return ok();
}

int lp_ipc_alloc(size_t bytes, void** dptr) {
  if (!dptr || bytes == 0) return fail(LP_EINVAL, "lp_ipc_alloc: bad arguments");
  // plain cudaMalloc: IPC handles cannot name VMM (expandable-segment) allocations
  LP_CUDA(cudaMalloc(dptr, bytes));
  LP_CUDA(cudaMemset(*dptr, 0, bytes));
  return ok();
}

int lp_ipc_free(void* dptr) {
  if (!dptr) return fail(LP_EINVAL, "lp_ipc_free: null pointer argument");
  LP_CUDA(cudaFree(dptr));
  return ok();
}

int lp_ipc_open(const void* handle64, void** dptr) {
  if (!handle64 || !dptr) return fail(LP_EINVAL, "lp_ipc_open: null pointer argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  LP_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return ok();
}

int lp_ipc_close(void* dptr) {
  if (!dptr) return fail(LP_EINVAL, "lp_ipc_close: null pointer argument");
  LP_CUDA(cudaIpcCloseMemHandle(dptr));
  return ok();
}

size_t lp_ep_ctl_bytes(int P, int E) {
  if (P < 1 || P > lp::kEpMaxRanks || E < P || E % P) return 0;
  return static_cast<size_t>(lp::kCtlInbox) + 2u * static_cast<size_t>(P) * E * sizeof(int32_t);
}

int lp_ep_barrier(uint32_t* const* peer_ctl, int P, int rank, void* stream) {
  if (P < 1 || P > lp::kEpMaxRanks || rank < 0 || rank >= P || !peer_ctl)
    return fail(LP_EINVAL, "lp_ep_barrier: bad arguments P=%d rank=%d", P, rank);
  LP_CUDA(launch_pdl(lp::k_ep_barrier, 1, 32, 0, static_cast<cudaStream_t>(stream), peer_ctl, P, rank));
  return ok();
}

int lp_ep_exchange(const int32_t* counts, uint32_t* const* peer_ctl, int P, int El, int rank, int32_t* dest_base,
                   int32_t* off_local, int32_t* rows_out, void* stream) {
  if (P < 1 || P > lp::kEpMaxRanks || El < 1 || P * El > lp::kMaxExperts || rank < 0 || rank >= P || !counts ||
      !peer_ctl || !dest_base || !off_local)
    return fail(LP_EINVAL, "lp_ep_exchange: bad arguments P=%d El=%d rank=%d", P, El, rank);
  const size_t sm = static_cast<size_t>(P) * P * El * sizeof(int32_t);
  if (sm > 48 * 1024) return fail(LP_EUNSUPPORTED, "lp_ep_exchange: P*P*El too large");
  const int threads = 256;  // one thread per global expert (P * El <= 256) for the plan's block scan
  LP_CUDA(launch_pdl(lp::k_ep_exchange, 1, threads, sm, static_cast<cudaStream_t>(stream), counts, peer_ctl, P, El,
                     rank, dest_base, off_local, rows_out));
  return ok();
}

int lp_ep_dispatch(const void* x, const int32_t* ids, const int32_t* slot_of, const int32_t* offsets,
                   const int32_t* dest_base, void* const* peer_recv, int T, int H, int topk, int El,
                   int32_t* dest_rank, int32_t* dest_row, void* stream) {
  if (T < 0 || H <= 0 || H % 8 || topk < 1 || El < 1) return fail(LP_EINVAL, "lp_ep_dispatch: bad shape");
  if (T == 0) return ok();
  if (!x || !ids || !slot_of || !offsets || !dest_base || !peer_recv || !dest_rank || !dest_row)
    return fail(LP_EINVAL, "lp_ep_dispatch: null pointer argument");
  if (!aligned16(x)) return fail(LP_EINVAL, "lp_ep_dispatch: x must be 16-byte aligned");
  const int S = T * topk;
  LP_CUDA(launch_pdl(lp::k_ep_dispatch, (S + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream),
                     static_cast<const __nv_bfloat16*>(x), ids, slot_of, offsets, dest_base,
                     reinterpret_cast<__nv_bfloat16* const*>(peer_recv), S, H, topk, El, dest_rank, dest_row));
  return ok();
}

int lp_ep_combine(void* const* peer_y, const int32_t* dest_rank, const int32_t* dest_row, const float* w, int T,
                  int H, int topk, void* y, void* stream) {
  if (T < 0 || H <= 0 || H % 8 || topk < 1 || topk > 32) return fail(LP_EINVAL, "lp_ep_combine: bad shape");
  if (T == 0) return ok();
  if (!peer_y || !dest_rank || !dest_row || !w || !y) return fail(LP_EINVAL, "lp_ep_combine: null pointer argument");
  if (!aligned16(y)) return fail(LP_EINVAL, "lp_ep_combine: y must be 16-byte aligned");
  LP_CUDA(launch_pdl(lp::k_ep_combine, T, 256, 0, static_cast<cudaStream_t>(stream),
                     reinterpret_cast<__nv_bfloat16* const*>(peer_y), dest_rank, dest_row, w, T, topk, H,
                     static_cast<__nv_bfloat16*>(y)));
  return ok();
}

#ifdef LP_TRACE
// trace builds only (not part of include/lpmoe.h): read / reset the timestamps
int lp_trace_fetch(unsigned long long* out, int n) {
  if (n > 512) n = 512;
  if (cudaMemcpyFromSymbol(out, lp::g_lp_trace, sizeof(unsigned long long) * n) != cudaSuccess) return LP_ECUDA;
  return LP_OK;
}
int lp_trace_items(unsigned long long* out, int n) {
  const int total = lp::kTraceCtas * lp::kTraceItems * lp::kTraceFields;
  if (n > total) n = total;
  if (cudaMemcpyFromSymbol(out, lp::g_lp_items, sizeof(unsigned long long) * n) != cudaSuccess) return LP_ECUDA;
  return LP_OK;
}
int lp_trace_reset(void) {
  static unsigned long long zeros[lp::kTraceCtas * lp::kTraceItems * lp::kTraceFields] = {};
  if (cudaMemcpyToSymbol(lp::g_lp_items, zeros, sizeof(zeros)) != cudaSuccess) return LP_ECUDA;
  unsigned long long init[512];
  for (int i = 0; i < 512; ++i) init[i] = (i % 8 == 0 || i == 24 || i == 32 || i == 40 || i == 52) ? ~0ull : 0ull;
  if (cudaMemcpyToSymbol(lp::g_lp_trace, init, sizeof(init)) != cudaSuccess) return LP_ECUDA;
  return LP_OK;
}
#endif

}  // extern "C"

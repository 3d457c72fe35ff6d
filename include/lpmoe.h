/*
 * lpmoe.h — C ABI of the B200-native MoE-layer hot path (liblpmoe.so).
 *
 * The reference (arxiv 2510.08055 simulator `moesim`) has no numerical MoE
 * layer: it models the layer with `costmodel.moe_cost` (costmodel.py:57-85),
 * fed by a `CoverageModel.coverage(routed_tokens, rng)` (coverage.py:216-257)
 * whose Monte-Carlo backend is `kernels.uniform_union_counts` /
 * `kernels.weighted_union_counts` (kernels.py:209-222). Those call sites
 * (engine.py:144-154, cli.py:222-227) are where this library plugs in; each
 * entry point below names the reference interface it replaces or serves.
 *
 * Conventions
 *  - All tensor pointers are DEVICE pointers (CUDA global memory), 16-byte
 *    aligned, row-major, no padding. bf16 tensors are passed as void*.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream), performs no allocation, no host sync and
 *    no host<->device copy, so a whole layer is CUDA-graph capturable.
 *  - Return value: LP_OK or an LP_E* code; lp_last_error() gives the text
 *    (thread-local). Invalid arguments never launch anything.
 *  - Stateless and reentrant: any host thread may call with its own stream
 *    and its own workspace.
 *  - Layouts (HF Qwen3-MoE, transformers 5.5 modeling_qwen3_moe.py:220-224,
 *    :255): x, y [T,H]; wr [E,H]; w13 [E,2I,H] (gate rows 0..I-1, up rows
 *    I..2I-1); w2 [E,H,I]. Constraints: H%64==0, I%64==0, E<=256,
 *    1<=topk<=min(E,32).
 */
#ifndef LPMOE_H_
#define LPMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LP_OK 0
#define LP_EINVAL 1        /* argument outside the documented domain */
#define LP_ECUDA 2         /* CUDA runtime/driver error */
#define LP_EUNSUPPORTED 3  /* valid but not implemented (e.g. E > 256) */

/* Library version string, e.g. "lpmoe 0.1 sm_100a". */
const char* lp_version(void);

/* Copies the calling thread's last error message into buf (NUL-terminated);
 * returns the last error code. */
int lp_last_error(char* buf, size_t n);

/* Number of kernels this library has launched in the process so far (all
 * entry points, all threads). Not a reference interface: host-side evidence
 * of which native kernels ran inside a timed region (bench.py gpu_launches). */
uint64_t lp_launch_count(void);

/* Bytes of scratch `lp_moe_forward` needs for this shape (>= 0, 256-aligned
 * regions). Also sufficient for every staged call below. The workspace must be
 * zero-filled ONCE after allocation (its fixed-offset header holds the
 * router's split-K tickets and the expert scheduler's words); every call
 * leaves that header zeroed again, so it can be reused for any T. */
size_t lp_moe_workspace_bytes(int T, int H, int I, int E, int topk);

/* K1 — router + gating. Replaces the routing the reference only models
 * (coverage.py:140-169 `sample_activation`, kernels.py:73-145): fp32 logits
 * x.Wr^T, softmax over E, top-k (prob desc, index asc), optional
 * renormalisation. ids int32 [T,topk], w fp32 [T,topk]. */
int lp_moe_route(const void* x, const void* wr, int T, int H, int E, int topk, int renorm, int32_t* ids,
                 float* w, void* ws, size_t ws_bytes, void* stream);

/* K2 — per-expert histogram, offsets (exclusive scan) and stable
 * permutation. counts [E], offsets [E+1], slot_of [T*topk] (slot of entry
 * t*topk+j), tok_of [T*topk] (token of slot); x_perm [T*topk,H] gathered rows
 * (may be NULL to skip the gather). The nnz of `counts` is the measured
 * coverage the reference's CoverageModel.coverage estimates
 * (coverage.py:216-257, called at engine.py:147/152). */
int lp_moe_permute(const int32_t* ids, const void* x, int T, int H, int E, int topk, int32_t* counts,
                   int32_t* offsets, int32_t* slot_of, int32_t* tok_of, void* x_perm, void* ws, size_t ws_bytes,
                   void* stream);

/* K3 — grouped expert FFN over S expert-contiguous slots (offsets [E+1]):
 * act = SiLU(x_perm.W13gate^T) * (x_perm.W13up^T) [S,I], y_perm = act.W2^T
 * [S,H]. tcgen05/TMEM/TMA, one persistent launch. Expert weights of every
 * expert with >=1 slot are streamed from HBM once per call while
 * tokens/expert <= the tile cap (the moe_cost byte model, costmodel.py:77). */
int lp_moe_experts(const void* x_perm, const int32_t* offsets, int S, const void* w13, const void* w2, int H,
                   int I, int E, void* act, void* y_perm, void* ws, size_t ws_bytes, void* stream);
/* As lp_moe_experts, with the row count left on the device: x_perm / act /
 * y_perm hold S rows (capacity), offsets[E] <= S rows are valid, and S_hint
 * (the expected routed rows, e.g. T*topk of the sender ranks) picks the token
 * tile width. No host read of offsets: the expert-parallel layer stays
 * stream-ordered and graph-capturable. */
int lp_moe_experts_rows(const void* x_perm, const int32_t* offsets, int S, int S_hint, const void* w13,
                        const void* w2, int H, int I, int E, void* act, void* y_perm, void* ws, size_t ws_bytes,
                        void* stream);

/* K4 — weighted combine y[t] = sum_j w[t,j] * y_perm[slot_of[t,j]] (bf16 out). */
int lp_moe_combine(const void* y_perm, const int32_t* slot_of, const float* w, int T, int H, int topk, void* y,
                   void* stream);

/* K1..K4 in one call: y [T,H] bf16 = MoE(x). ids / w / counts may be NULL
 * (kept in the workspace); T == 0 only zero-fills counts (if given). Replaces the pair
 * `coverage_model.coverage(routed)` + `moe_cost(model, routed, cov, 1)` at
 * engine.py:147-148 / :152-153 with the real layer. */
int lp_moe_forward(const void* x, const void* wr, const void* w13, const void* w2, int T, int H, int I, int E,
                   int topk, int renorm, void* y, int32_t* ids, float* w, int32_t* counts, void* ws,
                   size_t ws_bytes, void* stream);

/* Routing-surrogate sampler, bit-exact with the reference kernels.
 * u float64 [trials,batch,k] (C-contiguous), out int64 [trials].
 * Replaces kernels.uniform_union_counts (kernels.py:209-213, numba body
 * :73-103) and kernels.weighted_union_counts (kernels.py:216-222, body
 * :106-145; weights float64 [E]). k <= 64 (uniform), E <= 1024. */
int lp_union_counts_uniform(const double* u, int trials, int batch, int k, int E, int64_t* out, void* stream);
int lp_union_counts_weighted(const double* u, int trials, int batch, int k, int E, const double* weights,
                             int64_t* out, void* stream);

/* Executor glue between layers (serving.py / executor.py, not the MoE hot
 * path): h += delta (if delta != NULL, in place, bf16), then
 * xn = h * rsqrt(mean(h^2) + eps) per row — the residual update and the
 * pre-MoE RMSNorm of a Qwen3 decoder layer with unit gain. Stands in for the
 * non-MoE layer work the reference charges via dense_cost
 * (costmodel.py:128-145, engine.py:149). h, delta, xn [T,H] bf16. */
int lp_add_rmsnorm(void* h, const void* delta, void* xn, int T, int H, float eps, void* stream);

/* Profiling hook (calling thread only): when n >= 5, the next lp_moe_forward
 * calls record events[0..4] (cudaEvent_t handles) on their stream at the
 * stage boundaries route | permute | experts | combine | end. n = 0 clears. */
int lp_profile_events(void* const* events, int n);

/* ---------------------------------------------------------------------------
 * Expert parallelism over peer memory (ep.py PeerEP). Replaces the two
 * all_to_all_single exchanges of the NCCL EP path (ep.py EPMoE.forward) with
 * the dispatch fused into the permutation and the return fused into the
 * combine, reading/writing the other ranks' buffers through CUDA IPC mappings
 * (NVLink/NVSwitch P2P across GPUs). The reference has no multi-GPU code
 * (SPEC.md:24); the per-layer MoE call it stands for is engine.py:144-154.
 * `peer_*` arguments are DEVICE arrays of P device pointers (index = rank),
 * the caller's own buffer included. */

/* CUDA IPC export / import of a device allocation (64-byte opaque handle).
 * lp_ipc_handle names the allocation containing dptr and returns dptr's byte
 * offset in it; lp_ipc_open maps a handle from ANOTHER process (peer access
 * enabled lazily) and returns the allocation base. */
int lp_ipc_handle(const void* dptr, void* handle64, size_t* offset);
/* Zero-filled cudaMalloc region for a rank's symmetric EP buffers (setup time,
 * not on the layer path; IPC cannot export caching-allocator VMM segments). */
int lp_ipc_alloc(size_t bytes, void** dptr);
int lp_ipc_free(void* dptr);
int lp_ipc_open(const void* handle64, void** dptr);
int lp_ipc_close(void* dptr);

/* Bytes of a rank's EP control block (the first bytes of its zero-filled
 * region, 256-aligned by the caller): u32 barrier counter, u32 barrier and
 * layer sequence numbers, ready tags [2][32], int32 count inbox [2][P][E].
 * 0 when P > 32 or E is not a multiple of P. */
size_t lp_ep_ctl_bytes(int P, int E);

/* Device-side barrier over P ranks: adds 1 to every rank's counter
 * (system-scope release), then waits until its own counter reaches P x the
 * number of barriers it has passed (kept in its control block, so captured
 * CUDA graphs replay correctly). peer_ctl: device array of the P control blocks. */
int lp_ep_barrier(uint32_t* const* peer_ctl, int P, int rank, void* stream);

/* Count exchange + plan (one launch, replaces a post / barrier / plan
 * sequence): this rank's per-global-expert counts (int32 [P*El]) go to every
 * rank's inbox, followed by a system-scope ready tag; once every source's tag
 * is in this rank's block: dest_base[d*El+el] = first row of this rank's
 * entries for expert el in rank d's receive buffer (rows expert-major,
 * source-rank-major within an expert); off_local[0..El] = this rank's expert
 * offsets over all sources (off_local[El] = rows received; also stored to
 * *rows_out when rows_out is not NULL: off_local is rewritten by the next layer). */
int lp_ep_exchange(const int32_t* counts, uint32_t* const* peer_ctl, int P, int El, int rank, int32_t* dest_base,
                   int32_t* off_local, int32_t* rows_out, void* stream);

/* Fused permute + dispatch: entry i = t*topk + j (ids/slot_of/offsets from
 * lp_moe_route + lp_moe_permute over the P*El global experts) stores x[t]
 * into peer_recv[d][dest_base[d*El+el] + slot_of[i] - offsets[e]] (bf16
 * [cap, H] on every rank); records dest_rank[i], dest_row[i]. */
int lp_ep_dispatch(const void* x, const int32_t* ids, const int32_t* slot_of, const int32_t* offsets,
                   const int32_t* dest_base, void* const* peer_recv, int T, int H, int topk, int El,
                   int32_t* dest_rank, int32_t* dest_row, void* stream);

/* Fused receive + combine: y[t] = sum_j w[t,j] * peer_y[dest_rank][dest_row]
 * (fp32 accumulate in fixed j order, bf16 out) read straight from the owners. */
int lp_ep_combine(void* const* peer_y, const int32_t* dest_rank, const int32_t* dest_row, const float* w, int T,
                  int H, int topk, void* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LPMOE_H_ */

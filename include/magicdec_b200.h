/*
 * magicdec_b200.h — C ABI of the B200 (sm_100a) MagicDec self-speculative decode hot path.
 *
 * MagicDec (arXiv 2408.11049) speeds up large-batch long-context decoding by letting
 * the target model draft for itself with a StreamingLLM-compressed KV cache
 * (attention-sink tokens + a recent window) and then
 * verifying the gamma drafted tokens against the full KV cache.
 * One speculation step is gamma draft passes plus one verify pass
 * (T_total = gamma*T_D + T_V) followed by the speculative-sampling
 * acceptance of Leviathan et al..  In the long-context, large-batch
 * regime the paper targets, KV loading dominates both passes,
 * so the four calls below are the data-parallel hot path:
 *
 *   md_kv_append          write the new K/V rows of a pass into the shared cache
 *   md_draft_attn_sparse  1 query token / sequence over sink ∪ window (no KV copy)
 *   md_draft_attn_indexed 1 query token / sequence over a SnapKV index list ∪ recent tail
 *   md_snapkv_select      prefill-time SnapKV selection of that index list
 *   md_pq_encode / md_pq_select  PQCache-style dynamic selection of that list per query
 *   md_verify_attn_full   gamma+1 query tokens / sequence over the full KV, GQA, causal
 *   md_spec_accept        batched acceptance + residual / bonus resampling (or greedy)
 *   md_philox_u32         counter-based uniforms feeding md_spec_accept
 *
 * Tree-based speculation (P:173 names token trees as compatible with
 * the analysis): md_verify_attn_tree (tree-masked verify), md_spec_accept_tree (recursive
 * rejection over siblings) and md_kv_compact (move the accepted path's K/V rows together).
 *
 * Conventions shared by every call
 *   - Every pointer argument named as "device" is caller-owned CUDA device memory;
 *     the library never allocates, frees, synchronises or copies host<->device.
 *     Each call only enqueues work on `stream` (a cudaStream_t; NULL = legacy default
 *     stream), so a whole speculation step can be captured in a CUDA graph, as the
 *     paper does with PyTorch CUDA graphs.
 *   - bf16 tensors are raw IEEE bfloat16 bit patterns (uint16_t storage).
 *   - GQA: query head h reads KV head floor(h / g), g = num_q_heads / num_kv_heads.
 *   - Softmax scale `scale` multiplies q.k (pass 1/sqrt(head_dim) for the usual model).
 *   - LSE outputs are natural-log log-sum-exp of the scaled scores.
 *   - Return value: MD_OK, or an error code with a message from md_last_error().
 *     Host-side argument errors are detected before anything is enqueued.  Violating a
 *     device-side precondition (values inside device arrays) is undefined behaviour.
 *   - Thread safety: calls are reentrant; the only library state is thread-local (the error
 *     string and the md_debug_trace diagnostics buffer).  The library reads no environment
 *     variables: every plan choice is a compile-time constant or a function of the arguments.
 */
#ifndef MAGICDEC_B200_H
#define MAGICDEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MD_ABI_VERSION 1

#if defined(__GNUC__)
#define MD_API __attribute__((visibility("default")))
#else
#define MD_API
#endif

typedef struct CUstream_st* md_stream_t; /* identical to cudaStream_t */

typedef enum {
  MD_OK = 0,
  MD_ERR_INVALID_ARG = 1, /* bad scalar, NULL or misaligned pointer, bad stride      */
  MD_ERR_UNSUPPORTED = 2, /* valid but not built: head_dim not in {64,128}, g*T > 128 */
  MD_ERR_WORKSPACE = 3,   /* workspace NULL or smaller than md_attn_workspace_bytes   */
  MD_ERR_CUDA = 4         /* a CUDA runtime/driver call or kernel launch failed       */
} md_status;

typedef enum { MD_ACCEPT_SAMPLE = 0, MD_ACCEPT_GREEDY = 1 } md_accept_mode;

/*
 * One layer's KV cache, shared by the draft and the verify passes (the paper's "static
 * compressed KV" of P:720 is realised as an index set over this cache, not a copy).
 * k, v: device bf16, logical shape [batch][num_kv_heads][capacity][head_dim], element
 * strides (stride_b, stride_h, stride_s, 1).  Strides must be multiples of 8 elements
 * (16 bytes) and k, v 16-byte aligned.  The contiguous layout is
 * (num_kv_heads*capacity*head_dim, capacity*head_dim, head_dim); an NHD cache
 * ([batch][capacity][num_kv_heads][head_dim]) is expressed with
 * (capacity*Hkv*d, d, Hkv*d).  Passed by pointer, read during the call only.
 */
typedef struct {
  void* k;
  void* v;
  int32_t batch, num_kv_heads, head_dim, capacity;
  int64_t stride_b, stride_h, stride_s;
} md_kv_cache;

/* MD_ABI_VERSION of the loaded library. */
MD_API int md_abi_version(void);

/* Message for the last non-MD_OK status returned on this thread ("" if none).
 * Valid until the next md_* call on the same thread. */
MD_API const char* md_last_error(void);

/*
 * md_kv_append — cache update of one pass (implied by decode,
 * P:720; ragged per-sequence positions).
 * For every sequence b, new token t in [0, T) and KV head h:
 *     cache[b][h][start_pos[b] + t][:] = new[b][t][h][:]     (for k and v)
 * k_new, v_new: device bf16 [B][T][Hkv][head_dim], contiguous (as a QKV projection
 * emits them, already rotary-embedded upstream).  start_pos: device int32[B].
 * A draft step appends T = 1 row at L_b + j; verify appends T = gamma+1 rows at L_b,
 * overwriting the draft-written slots (reading Z11).
 * Preconditions (device): 0 <= start_pos[b] and start_pos[b] + T <= capacity.
 */
MD_API md_status md_kv_append(const md_kv_cache* cache, const void* k_new, const void* v_new, int32_t T,
                       const int32_t* start_pos, md_stream_t stream);

/*
 * Bytes of scratch the attention calls need: a fixed block of arrival
 * counters (one per (b, kv head), up to B*Hkv = 65536, plus two for the dynamic chunk
 * scheduler) followed by the split partials (o, lse) of the work chunks of the persistent
 * grid.  Depends on (g*T, head_dim) and the current device's SM count, not on the context
 * length (`max_kv_len` and `batch` are accepted for symmetry).
 * The workspace must be zero-filled ONCE when allocated (e.g. cudaMemset / torch.zeros);
 * every call leaves the counters at zero again, so it can be reused by any later call of any
 * shape on the same stream (not by two calls in flight concurrently).  Returns 0 for
 * invalid args.
 */
MD_API size_t md_attn_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads, int32_t head_dim,
                               int32_t T, int32_t max_kv_len);

/*
 * md_verify_attn_full — verification attention ("the time taken by the target
 * model to verify gamma tokens"; "verification and decoding share the same KV
 * budget"; reading Z4: T = gamma + 1 query tokens, the pending token plus gamma drafts).
 * For b < B, t < T, h < Hq, with n = kv_len[b] (which COUNTS the T new tokens):
 *     J        = [0, n - T + t]                     (causal among the T new rows, Z10)
 *     out[b][t][h][:] = softmax_j(scale * q[b][t][h] . k[b][h/g][j]) @ v[b][h/g][J]
 *     lse[b][t][h]    = log sum_{j in J} exp(scale * q . k_j)
 * The g*T query rows of one KV head share a single read of that head's KV.
 * T = 1 is plain autoregressive decode.
 *   q:   device bf16 [B][T][Hq][head_dim], contiguous.   kv_len: device int32[B].
 *   max_kv_len: host upper bound on kv_len[b] (used to plan splits; keys beyond
 *               kv_len[b] are never read).
 *   out: device fp32 [B][T][Hq][head_dim]; lse: device fp32 [B][T][Hq] or NULL.
 *   workspace: zero-initialised device scratch of >= md_attn_workspace_bytes(B, Hq, Hkv, d, T,
 *              max_kv_len) bytes.
 * Supported: head_dim in {64, 128}, 1 <= T <= 16, g*T <= 128 query rows per KV head at head_dim 128
 * (the tcgen05 kernel) and g*T <= 64 at head_dim 64.
 * Preconditions (device): T <= kv_len[b] <= min(max_kv_len, capacity).
 */
MD_API md_status md_verify_attn_full(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                              const int32_t* kv_len, int32_t max_kv_len, float scale, float* out, float* lse,
                              void* workspace, size_t workspace_bytes, md_stream_t stream);

/*
 * md_verify_attn_full_det / md_draft_attn_sparse_det — the same results as md_verify_attn_full /
 * md_draft_attn_sparse (same definition, tolerance and limits), computed with a DETERMINISTIC
 * fixed-split plan: every (sequence, KV head) unit's key sequence is cut at multiples of
 * `split_keys` (a multiple of 64), each piece is reduced by one CTA and the pieces' partials are
 * merged in piece order (the log-sum-exp combination of SURVEY §8(a) row a4).  The bits of a unit's
 * output then depend only on that unit's inputs and on split_keys -- not on the GPU's SM count,
 * the other sequences or KV heads, or how a batch is sharded over ranks: a KV-head tensor-parallel
 * or batch-sharded run reproduces the single-GPU output bit for bit (SURVEY §8(e) MD_FIXED_SPLIT).
 * The stream-K plan of the plain calls balances bytes across SMs instead and is the faster one.
 *   workspace: zero-initialised, >= md_attn_workspace_bytes_det(B, Hq, Hkv, d, T, max_keys,
 *              split_keys) bytes, max_keys = max_kv_len (verify) or min(sink + window, capacity)
 *              (draft; T = 1).  Returns 0 for invalid args.
 */
MD_API size_t md_attn_workspace_bytes_det(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads, int32_t head_dim,
                                          int32_t T, int32_t max_keys, int32_t split_keys);
MD_API md_status md_verify_attn_full_det(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                                         const int32_t* kv_len, int32_t max_kv_len, int32_t split_keys, float scale,
                                         float* out, float* lse, void* workspace, size_t workspace_bytes,
                                         md_stream_t stream);
MD_API md_status md_draft_attn_sparse_det(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                          const int32_t* kv_len, int32_t sink, int32_t window, int32_t split_keys,
                                          float scale, float* out, float* lse, void* workspace,
                                          size_t workspace_bytes, md_stream_t stream);

/*
 * md_verify_attn_tree — verification of a token TREE of T nodes per sequence (f3; the
 * chain of md_verify_attn_full is the special case tree_mask[b][t] = 2^(t+1) - 1).
 * Node t's K/V row sits at cache position n - T + t (node 0 = the pending root token),
 * parent[t] < t.  For b < B, t < T, h < Hq, with n = kv_len[b]:
 *     J = [0, n - T)  ∪  { n - T + j : bit j of tree_mask[b][t] is set }
 * (for a tree: the ancestors-or-self of node t, mask[t] = mask[parent[t]] | 1 << t),
 * otherwise exactly md_verify_attn_full (same outputs, workspace and limits).
 *   tree_mask: device uint32 [B][T]; bits >= T are ignored.
 * Preconditions (device): a row whose J is empty (only possible when n = T and its mask is
 * 0) gets out = 0, lse = -inf.
 */
MD_API md_status md_verify_attn_tree(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                              const int32_t* kv_len, int32_t max_kv_len, const uint32_t* tree_mask, float scale,
                              float* out, float* lse, void* workspace, size_t workspace_bytes,
                              md_stream_t stream);

/*
 * md_draft_attn_sparse — self-speculative draft attention over the StreamingLLM
 * compressed KV ("StreamingLLM style sparse KV for drafting", P:460 budgets,
 * P:720 static compressed KV; Eq.3 P:1081 with T_select = 0 for a static method).
 * For b < B, h < Hq, with n = kv_len[b] (counts the just-appended draft token):
 *     J = {j < min(sink, n)}  U  {max(sink, n - window) <= j < n}     (no index twice)
 *     out[b][h][:] = softmax_j(scale * q[b][h] . k[b][h/g][j]) @ v[b][h/g][J],  lse likewise.
 * The window slides with n (reading Z2); positions are not re-indexed (Z3); the
 * kernel walks the two row ranges of the shared cache directly (no gather copy).
 *   q: device bf16 [B][Hq][head_dim]; out: fp32 [B][Hq][head_dim]; lse: fp32 [B][Hq] or NULL.
 *   workspace: zero-initialised, >= md_attn_workspace_bytes(B, Hq, Hkv, d, 1, min(sink + window, capacity)).
 * Supported: head_dim in {64, 128}, g <= 64, sink >= 0, window >= 0, sink + window >= 1.
 * Preconditions (device): 1 <= kv_len[b] <= capacity.
 */
MD_API md_status md_draft_attn_sparse(const md_kv_cache* cache, const void* q, int32_t num_q_heads, const int32_t* kv_len,
                               int32_t sink, int32_t window, float scale, float* out, float* lse, void* workspace,
                               size_t workspace_bytes, md_stream_t stream);

/*
 * md_draft_attn_sparse_windows — md_draft_attn_sparse with a window per sequence, for
 * heterogeneous batches ("different sequences in the same batch can leverage different draft
 * KV cache sizes").  Sequence b attends to
 *     J_b = {j < min(sink, n)}  U  {max(sink, n - w_b) <= j < n},
 *     w_b = min(window, max(windows[b], max(0, 1 - sink)))    (n = kv_len[b]).
 *   windows: device int32 [B]; `window` bounds every w_b and sizes the workspace exactly as
 *   for md_draft_attn_sparse.  Other arguments, layouts and errors as md_draft_attn_sparse;
 *   a NULL `windows` is MD_ERR_INVALID_ARG.
 */
MD_API md_status md_draft_attn_sparse_windows(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                              const int32_t* kv_len, int32_t sink, int32_t window,
                                              const int32_t* windows, float scale, float* out, float* lse,
                                              void* workspace, size_t workspace_bytes, md_stream_t stream);

/*
 * md_verify_attn_full_append / md_draft_attn_sparse_append — the append of a pass fused into
 * its attention call (SURVEY §8(a) row a1 "can be fused into the attention prologue"; the
 * step of §8(a): kv_append(start = L_b + j) then draft, kv_append(start = L_b) then verify).
 * Exactly equivalent to
 *     md_kv_append(cache, k_new, v_new, T, start = kv_len - T);  then the plain call
 * (T = 1 for the draft call), in one kernel launch: the CTA that streams the key tile holding a
 * new row writes that row into the cache before its TMA load of the tile (the K/V of the new
 * rows come from k_new / v_new, so the attention reads exactly what md_kv_append would write).
 *   k_new, v_new: device bf16 [B][T][Hkv][head_dim], contiguous, 16-byte aligned (as for
 *                 md_kv_append); the cache rows [kv_len[b] - T, kv_len[b]) are overwritten.
 *   All other arguments, outputs, workspace and limits: as md_verify_attn_full /
 *   md_draft_attn_sparse.  The draft form needs window >= 1 (the new token is in its window).
 * The fused form runs the static stream-K plan (no dynamic tail); where the kernel the shape
 * selects cannot fuse (the mma.sync rows kernel: head_dim 64 verify with g*T > 8) or a long
 * keys-kernel call would use the dynamic tail (B * Hkv * ceil(max_kv_len / 64) >= 128 tiles per
 * CTA, e.g. the MHA verify), the call enqueues the md_kv_append kernel ahead of the attention
 * kernel instead — same results.
 * Preconditions (device): as the plain calls, plus T <= kv_len[b].
 */
MD_API md_status md_verify_attn_full_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                                     const void* k_new, const void* v_new, const int32_t* kv_len,
                                     int32_t max_kv_len, float scale, float* out, float* lse, void* workspace,
                                     size_t workspace_bytes, md_stream_t stream);
MD_API md_status md_draft_attn_sparse_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                      const void* k_new, const void* v_new, const int32_t* kv_len, int32_t sink,
                                      int32_t window, float scale, float* out, float* lse, void* workspace,
                                      size_t workspace_bytes, md_stream_t stream);

/*
 * md_draft_attn_sparse_append_ex — md_draft_attn_sparse_append with option flags (0 = identical).
 *
 *   MD_ATTN_EARLY_KV: the caller guarantees that kv_len[] and the cache rows this call attends to,
 *     other than the row it appends itself, are not written by an md_* call that precedes it on
 *     the stream without an intervening ordinary kernel, copy, event wait or host synchronisation
 *     (this library's kernels let the next kernel launch early, before they finish; ordinary
 *     work does not).  The kernel may then read kv_len and stream the first key tiles of a unit
 *     (never one holding the appended row, never q; the next few tiles are also prefetched into
 *     L2, a hint that is correct regardless) before waiting for the previous kernel, so
 *     the call's ramp overlaps the previous call's tail (a draft step: every layer's call, the
 *     layers' caches distinct from the previous call's).  Results are bit-identical with and
 *     without the flag; without the guarantee the flag is a data race.  Used only where the draft
 *     runs the unit-aligned plan (always at head_dim 128 / 64 with g <= 8); ignored otherwise.
 * Errors: as md_draft_attn_sparse_append; MD_ERR_INVALID_ARG for an unknown flag bit.
 */
#define MD_ATTN_EARLY_KV 1u
MD_API md_status md_draft_attn_sparse_append_ex(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                         const void* k_new, const void* v_new, const int32_t* kv_len,
                                         int32_t sink, int32_t window, float scale, float* out, float* lse,
                                         void* workspace, size_t workspace_bytes, uint32_t flags,
                                         md_stream_t stream);

/*
 * md_draft_attn_indexed — self-speculative draft attention over a static SnapKV-selected KV
 * (the paper's best drafter; SnapKV with observation
 * window 32 and average pooling 5; per-sequence budgets).
 * For b < B, h < Hq, with n = kv_len[b], kv head u = h / g:
 *     J = {idx[b][u][i] : i < idx_count[b]}  U  {tail_start[b] <= j < n}
 *     out[b][h][:] = softmax_j(scale * q[b][h] . k[b][u][j]) @ v[b][u][J],  lse likewise.
 * The listed rows are copied from the shared cache in place (16-byte cp.async per row), the tail
 * (the observation window plus every token generated since prefill) is streamed.
 *   idx: device int32 [B][Hkv][idx_stride], 16-byte aligned, idx_stride % 4 == 0; entries
 *        0 <= idx < tail_start[b] (ascending order recommended for locality).
 *   idx_count, tail_start: device int32 [B], idx_count[b] <= idx_stride.
 *   q, out, lse, workspace: as md_draft_attn_sparse (workspace sized with T = 1).
 * Supported: head_dim in {64, 128}, g <= 8, cache strides multiples of head_dim.
 * Preconditions (device): tail_start[b] <= kv_len[b] <= capacity, idx_count[b] +
 * kv_len[b] - tail_start[b] >= 1.
 */
MD_API md_status md_draft_attn_indexed(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                       const int32_t* kv_len, const int32_t* idx, int32_t idx_stride,
                                       const int32_t* idx_count, const int32_t* tail_start, float scale, float* out,
                                       float* lse, void* workspace, size_t workspace_bytes, md_stream_t stream);

/*
 * md_draft_attn_indexed_append — md_draft_attn_indexed with the draft step's append fused in:
 * exactly md_kv_append(k_new, v_new, T = 1, start = kv_len - 1) followed by
 * md_draft_attn_indexed, in one launch.  When the new row lies in the streamed tail, the CTA whose
 * tail tile holds it writes it before loading the tile (see md_draft_attn_sparse_append); when it
 * lies before the tail (tail_start[b] = kv_len[b], e.g. after md_pq_select with window 0), the CTA
 * holding the unit's first tile writes it and any listed copy of it reads k_new / v_new directly.
 *   k_new, v_new: device bf16 [B][1][Hkv][head_dim], contiguous, 16-byte aligned.
 * Preconditions (device): as md_draft_attn_indexed.
 */
MD_API md_status md_draft_attn_indexed_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                       const void* k_new, const void* v_new, const int32_t* kv_len,
                                       const int32_t* idx, int32_t idx_stride, const int32_t* idx_count,
                                       const int32_t* tail_start, float scale, float* out, float* lse,
                                       void* workspace, size_t workspace_bytes, md_stream_t stream);

/*
 * md_snapkv_select — SnapKV static KV selection at prefill for md_draft_attn_indexed
 * (P:1141 footnote: observation window 32, average pooling kernel 5;
 * a static method, so drafting pays no per-step selection cost, Eq.3).  Per
 * sequence b (prompt length L = prefill_len[b]) and KV head u, with the g*w window queries
 * q_obs[b][i][u*g + hh] (prompt positions L-w+i):
 *   S1 a[hh,i,j] = softmax_j(scale q . k[b][u][j]) over the causal keys j <= L-w+i;
 *   S2 vote[j]   = sum_{hh,i} a[hh,i,j]                 for j < L-w;
 *   S3 pooled[j] = (vote[j-2] + ... + vote[j+2]) / 5     (zero padding);
 *   S4 idx[b][u][0 .. c) = the c = min(B_b-w, L-w) largest pooled positions (ties ->
 *      lower position), ascending; idx_count[b] = c.  Entries past c are left untouched.
 *      B_b = budget, or with per-sequence budgets (heterogeneous batches)
 *      B_b = min(max(budgets[b], w), budget).
 * The draft then attends to idx U [L-w, n) (pass tail_start = L - w).  Scores are fp32 on
 * the tensor cores, so positions whose pooled votes tie to ~1e-6 relative may order
 * differently from an fp64 evaluation.
 *   q_obs: device bf16 [B][w][Hq][head_dim]; prefill_len: device int32[B];
 *   max_prefill_len: host bound >= every prefill_len[b];
 *   idx: device int32 [B][Hkv][idx_stride] (idx_stride >= budget - w); idx_count: int32[B];
 *   budgets: optional device int32[B] (NULL: every sequence uses `budget`, which bounds them);
 *   workspace: >= md_snapkv_workspace_bytes(B, Hq, Hkv, w, max_prefill_len) bytes (no init).
 * Supported: head_dim in {64, 128}, g*w <= 256.
 * Preconditions (device): w <= prefill_len[b] <= max_prefill_len.
 */
MD_API size_t md_snapkv_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads, int32_t w,
                                        int32_t max_prefill_len);
MD_API md_status md_snapkv_select(const md_kv_cache* cache, const void* q_obs, int32_t num_q_heads,
                                  const int32_t* prefill_len, int32_t max_prefill_len, int32_t w, int32_t budget,
                                  const int32_t* budgets, float scale, int32_t* idx, int32_t idx_stride,
                                  int32_t* idx_count, void* workspace,
                                  size_t workspace_bytes, md_stream_t stream);

/*
 * PQCache-style dynamic KV selection.  Dynamic methods "search the KV
 * cache for each input query, attempting to find the top k nearest neighbors";
 * PQCache "employs product quantization with 16 sub-vectors and 8-bit quantization per key
 * vector" (P:1141 footnote); its search is the T_select term of Eq.3.  Keys are
 * cut into 16 sub-vectors of s = head_dim/16 elements, each coded by the index of its
 * nearest of 256 centroids; a draft query scores every candidate key through a lookup table
 * of query-centroid inner products, and the top-scoring positions plus the sink rows form
 * the index list of md_draft_attn_indexed (with the recent window as its streamed tail).
 * Readings Z25-Z29; oracle/pqcache.py P1-P5.
 *
 * codebook: device bf16 [B][Hkv][16][256][s] (trained at prefill by the caller, e.g.
 *           k-means; not part of the decode path), 16-byte aligned.
 * codes:    device uint8 [B][Hkv][code_capacity][16], 16-byte aligned.
 *
 * md_pq_encode — codes[b][h][start_pos[b] + t][m] for t < count, every KV head h and
 * sub-space m: the index c of the centroid minimising sum_{i<s} (x_i - C[m][c][i])^2, the sum
 * evaluated left to right with every operation rounded to fp32 (no fused multiply-add); ties
 * -> lowest c.  Called once at prefill (count = prompt length) and then for rows about to
 * leave the recent window (rows inside it are attended exactly, so encoding can be lazy).
 * Preconditions (device): start_pos[b] + count <= min(capacity, code_capacity).
 */
MD_API md_status md_pq_encode(const md_kv_cache* cache, const void* codebook, const int32_t* start_pos,
                              int32_t count, uint8_t* codes, int32_t code_capacity, md_stream_t stream);

/*
 * md_pq_select — per draft query, for every sequence b (n = kv_len[b]) and KV head u:
 *   lut[m][c]  = sum_{hh<g} sum_{i<s} q[b][u*g+hh][m*s+i] * C[m][c][i]   (fp32, hh outer, i
 *                inner, left to right, no FMA; the GQA group shares one selection);
 *   lutq       = rint(lut * 2^e) as int32, e = 26 - E with max|lut| = f*2^E, f in [0.5, 1)
 *                (e = 0 for an all-zero table) — exact power-of-two scaling;
 *   score[j]   = sum_m lutq[m][code[j][m]]   (exact integer);
 *   s0 = min(sink, n), tail = max(s0, n - window), c = min(budget, tail - s0);
 *   idx[b][u][0 .. s0 + c) = 0 .. s0-1, then the c positions of [s0, tail) with the largest
 *   score (ties -> lower position) in ascending order; idx_count[b] = s0 + c;
 *   tail_start[b] = tail.  Entries past s0 + c are left untouched.
 * Then md_draft_attn_indexed(idx, idx_stride, idx_count, tail_start) attends to
 * idx U [tail, n).  Every decision is taken on exact integers, so the lists are bit-exact.
 *   q: device bf16 [B][Hq][head_dim] (the draft query); kv_len: device int32[B];
 *   max_kv_len: host bound >= every kv_len[b], <= code_capacity;
 *   idx: device int32 [B][Hkv][idx_stride], idx_stride >= sink + budget (a multiple of 4
 *        for md_draft_attn_indexed); idx_count, tail_start: device int32[B];
 *   workspace: >= md_pq_workspace_bytes(B, Hkv, max_kv_len) bytes (no initialisation).
 * Supported: head_dim in {64, 128}, g <= 16.
 * Preconditions (device): kv_len[b] <= max_kv_len; codes of [0, tail) encoded.
 */
MD_API size_t md_pq_workspace_bytes(int32_t batch, int32_t num_kv_heads, int32_t max_kv_len);
MD_API md_status md_pq_select(const void* q, int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                              int32_t head_dim, const void* codebook, const uint8_t* codes, int32_t code_capacity,
                              const int32_t* kv_len, int32_t max_kv_len, int32_t sink, int32_t window,
                              int32_t budget, int32_t* idx, int32_t idx_stride, int32_t* idx_count,
                              int32_t* tail_start, void* workspace, size_t workspace_bytes, md_stream_t stream);

/*
 * Fused tensor-parallel output exchange (the paper runs 8-way tensor
 * parallelism).  Rank r of `world` owns KV heads [r*Hkv, (r+1)*Hkv) and their
 * query heads [r*Hq, (r+1)*Hq) (Hkv, Hq = this rank's counts).  Instead of writing a local
 * output and all-gathering it, the _tp calls store each finished output row into EVERY rank's
 * full-head buffer (peer-mapped device memory reachable over NVLink / NVSwitch, e.g. CUDA IPC
 * or symmetric-memory mappings): row (b, t, r*Hq + h) of [B][T][world*Hq][head_dim] fp32.
 * md_tp_barrier then publishes completion; after it returns on a rank's stream, that rank's
 * buffer holds every rank's heads.
 *   out_peers: device array [world] of device pointers, out_peers[k] = rank k's full-head
 *              buffer (16-byte aligned; out_peers[rank] is this rank's own);
 *   lse:       local layout [B][T][Hq] (may be NULL), as the non-TP calls.
 * All other arguments and the workspace are those of md_verify_attn_full / md_draft_attn_sparse
 * with the rank-local Hq and cache.  Returns MD_ERR_INVALID_ARG for a bad md_tp_out.
 * Every rank writes into every buffer at each call: a rank that still reads the previous
 * call's result while a faster peer may already issue the next call should alternate two
 * buffer sets (each with its own md_tp_sync) between consecutive calls.
 */
typedef struct {
  float* const* out_peers;
  int32_t world, rank;
} md_tp_out;

MD_API md_status md_verify_attn_full_tp(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                                        const int32_t* kv_len, int32_t max_kv_len, float scale, const md_tp_out* tp,
                                        float* lse, void* workspace, size_t workspace_bytes, md_stream_t stream);
MD_API md_status md_draft_attn_sparse_tp(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                         const int32_t* kv_len, int32_t sink, int32_t window, float scale,
                                         const md_tp_out* tp, float* lse, void* workspace, size_t workspace_bytes,
                                         md_stream_t stream);
/*
 * md_verify_attn_full_tp_append / md_draft_attn_sparse_tp_append — the _tp calls with the
 * rank's append fused in, exactly as md_verify_attn_full_append / md_draft_attn_sparse_append
 * (k_new, v_new: this rank's KV heads, [B][T][Hkv_local][head_dim]); outputs as the _tp calls.
 */
MD_API md_status md_verify_attn_full_tp_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                        int32_t T, const void* k_new, const void* v_new, const int32_t* kv_len,
                                        int32_t max_kv_len, float scale, const md_tp_out* tp, float* lse,
                                        void* workspace, size_t workspace_bytes, md_stream_t stream);
MD_API md_status md_draft_attn_sparse_tp_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                         const void* k_new, const void* v_new, const int32_t* kv_len, int32_t sink,
                                         int32_t window, float scale, const md_tp_out* tp, float* lse,
                                         void* workspace, size_t workspace_bytes, md_stream_t stream);

/*
 * md_tp_barrier — completion barrier of the fused exchange: every rank calls it once after each
 * _tp attention call, in the same order.  A device-side epoch (uint64 per rank, zero
 * initialised, bumped by the call itself, so a whole step can be captured in a CUDA graph) is
 * written with system-scope release into flags[k][rank] of every rank k after a system fence
 * (ordering the preceding kernels' peer stores); the call then waits (acquire) until
 * flags[rank][j] reaches the epoch for every j.
 *   flags_peers: device array [world] of device pointers to each rank's uint64 flags[world]
 *                (zero initialised, peer-mapped); epoch: this rank's device uint64 counter.
 * A peer that never arrives traps the kernel after ~20 s (no silent hang).  world <= 32.
 */
typedef struct {
  uint64_t* const* flags_peers;
  uint64_t* epoch;
  int32_t world, rank;
} md_tp_sync;

MD_API md_status md_tp_barrier(const md_tp_sync* sync, md_stream_t stream);

/*
 * md_philox_u32 — Philox4x32-10 uniforms for md_spec_accept (
 * SPEC.md S:472 counter-based PRNG with per-sequence streams; reading Z8).
 * out[b][w] = word (w % 4) of Philox4x32-10(counter = (b, step_lo, step_hi, w / 4),
 *                                          key = (seed_lo, seed_hi)).
 * out: device uint32 [B][words_per_seq].  For md_spec_accept use words_per_seq = gamma+2.
 */
MD_API md_status md_philox_u32(uint64_t seed, uint64_t step, int32_t B, int32_t words_per_seq, uint32_t* out,
                        md_stream_t stream);
/* md_philox_u32_dev — as md_philox_u32 with the step read from device memory (*step, uint64),
 * so a captured CUDA graph of a whole speculation step draws fresh uniforms at every replay
 * (the caller advances *step inside the graph). */
MD_API md_status md_philox_u32_dev(uint64_t seed, const uint64_t* step, int32_t B, int32_t words_per_seq,
                                   uint32_t* out, md_stream_t stream);

/*
 * md_spec_accept — batched speculative-sampling acceptance (the rule of Leviathan et
 * al. that P:204 cites; accepted counts are ragged per sequence; the paper's
 * experiments decode greedily).  Per sequence b (j = 0..gamma-1, x = d[b][j]):
 *   SAMPLE: accept iff (rnd[b][j] >> 3) * q[b][j][x] < p[b][j][x] * 2^29, evaluated
 *           exactly in fp64 (Z6).  At the first rejection n = j, draw the new token
 *           from W = max(0, floor(p_n 2^40) - floor(q_n 2^40)) (if sum W = 0: W =
 *           floor(p_n 2^40); if that is 0 too: lowest-index argmax p_n) with the
 *           64-bit uniform u = rnd[b][gamma] << 32 | rnd[b][gamma+1]:
 *           t = floor(u * sum W / 2^64), token = min{k : sum_{i<=k} W_i > t} (Z7, Z8).
 *           If all gamma are accepted, n = gamma and the bonus token is drawn the
 *           same way from W = floor(p_gamma 2^40).
 *   GREEDY: accept iff argmax p[b][j] == x (lowest index on ties); new token =
 *           argmax p[b][n].  rnd and q are not read (may be NULL).
 * Outputs: out_tokens[b] = [d_0 .. d_{n-1}, new, -1 ...] (gamma+1 entries),
 * num_accepted[b] = n, and, if committed_len_inout != NULL, committed_len[b] += n + 1.
 * Integer decisions are exact, so results are bit-reproducible and equal to the
 * oracle's on the same inputs.  gamma = 0 samples one token from p[b][0] (plain AR).
 *   p: device fp32 [B][gamma+1][V]; q: device fp32 [B][gamma][V];
 *   draft_tokens: device int32 [B][gamma]; rnd: device uint32 [B][gamma+2];
 *   out_tokens: device int32 [B][gamma+1]; num_accepted: device int32 [B].
 * Supported: 0 <= gamma <= 15, V >= 1.
 * Preconditions (device): 0 <= d < V; probabilities finite and in [0, 1].
 */
MD_API md_status md_spec_accept(const float* p, const float* q, const int32_t* draft_tokens, const uint32_t* rnd,
                         int32_t B, int32_t gamma, int32_t V, md_accept_mode mode, int32_t* out_tokens,
                         int32_t* num_accepted, int32_t* committed_len_inout, md_stream_t stream);

/*
 * md_spec_accept_tree — acceptance over a token tree (f3; readings Z21-Z24).
 * Node 0 is the root (the pending token), parent[b][t] < t for t >= 1; tokens[b][t] is
 * node t's token (tokens[b][0] is not read); p[b][t] / q[b][t] are the target / draft
 * distributions AT node t (over node t's children).  Walk from cur = 0:
 *   SAMPLE: children c of cur are tested in index order, test word rnd[b][k] for the k-th
 *     test overall (m = rnd >> 3).  First child: m q_cur(x) < p_cur(x) 2^29 (fp64, as
 *     md_spec_accept).  After its rejection R = max(0, P - Q) on the 2^-40 grid (P =
 *     floor(p_cur 2^40), Q = floor(q_cur 2^40); R = P if that sums to 0); each later
 *     sibling x is accepted iff m Q_x S < R_x 2^69 (S = sum R, exact integers; rejected if
 *     S = 0), a rejection updating R_i <- max(0, floor(R_i 2^40 / S) - Q_i) (kept if that
 *     sums to 0).  An accepted child becomes cur.  When every child is rejected the new
 *     token is drawn from R, at a leaf from P (argmax p_cur if the weights sum to 0), with
 *     u = rnd[b][T-1] << 32 | rnd[b][T] exactly as md_spec_accept.
 *   GREEDY: a = lowest-index argmax p_cur; move to the lowest-index child whose token is a,
 *     else emit a.  q and rnd are not read.
 * For a chain (parent[t] = t - 1) this equals md_spec_accept bit for bit.
 * Outputs: out_tokens[b] = [path tokens..., new, -1 ...] (T entries), num_accepted[b] =
 * path length n, accepted_nodes[b] = [path node indices..., -1 ...] (T entries; may be
 * NULL), committed_len[b] += n + 1 if committed_len_inout != NULL.
 *   p, q: device fp32 [B][T][V]; tokens, parent: device int32 [B][T];
 *   rnd: device uint32 [B][T+1].  Supported: 1 <= T <= 16.
 */
MD_API md_status md_spec_accept_tree(const float* p, const float* q, const int32_t* tokens, const int32_t* parent,
                              const uint32_t* rnd, int32_t B, int32_t T, int32_t V, md_accept_mode mode,
                              int32_t* out_tokens, int32_t* num_accepted, int32_t* accepted_nodes,
                              int32_t* committed_len_inout, md_stream_t stream);

/*
 * md_kv_compact — after tree acceptance, move the K/V rows of the accepted path next to
 * the root: for every b, kv head h and i < count[b], row base[b] + nodes[b][i] is copied
 * to base[b] + 1 + i (all reads happen before any write of a (b, h), so overlapping sets
 * are safe).  base[b] = the root's position (n - T); nodes is md_spec_accept_tree's
 * accepted_nodes, count its num_accepted.
 *   base, count: device int32 [B]; nodes: device int32 [B][nodes_stride].
 * Supported: 1 <= nodes_stride <= 16, head_dim a multiple of 8 up to 256.
 * Preconditions (device): count[b] <= nodes_stride, base[b] + nodes[b][i] < capacity.
 */
MD_API md_status md_kv_compact(const md_kv_cache* cache, const int32_t* base, const int32_t* nodes,
                        int32_t nodes_stride, const int32_t* count, md_stream_t stream);

/*
 * md_debug_trace — diagnostics only.  While `buf` (device uint64 [G][16], G = CTAs of the
 * attention grid) is set, every attention call stamps %globaltimer per CTA in slots: 0 entry,
 * 1 after the grid-dependency wait, 2 after locating its stream-K range, 3 first K/V tile
 * landed, 4 last segment epilogue start, 5 end, 6 = the SM id, 7/8/9 last epilogue after the
 * cross-warp combine / after its stores / after the split merge, 10 producer done,
 * 11 = segments processed (slots 7-11: draft/keys kernel only).  The setting belongs to the
 * calling thread (thread-local, like the error string): only attention calls made from that
 * thread stamp into `buf`.  NULL disables.
 */
MD_API md_status md_debug_trace(void* buf, size_t bytes);

#ifdef __cplusplus
}
#endif

#endif /* MAGICDEC_B200_H */

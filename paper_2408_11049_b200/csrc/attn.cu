// attn.cu — md_verify_attn_full, md_draft_attn_sparse, md_attn_workspace_bytes
// (SURVEY §8(a) rows a2, a3, a4).
//
// Both calls are split-KV flash decoding over the shared [B][Hkv][cap][d] bf16 cache.
//
// Work decomposition (stream-K).  A unit is one (b, kv head); its key index space is cut
// into 64-key tiles (verify: [0, kv_len); draft: the StreamingLLM set J = sink rows
// [0, min(sink, n)) then window rows [max(sink, n - window), n), walked in place — the
// "static compressed KV" of P:453/P:720 is never materialised).  All units' tiles are laid
// end to end and the persistent grid of G CTAs takes G equal contiguous ranges, so every
// SM streams the same number of KV bytes whatever B, the lengths or their raggedness
// (P:182).  A unit that straddles CTA ranges is finished by the last CTA to arrive (an
// acquire/release counter per unit): it combines the partials (o, lse) by the
// log-sum-exp identity (O6).  Each CTA writes at most two partials (its first and last
// unit), so merge traffic is ~2*G*R*D*4 bytes per call.  Each KV byte is read from HBM
// exactly once per call (verify and decode share the same KV bytes).
//
// Per CTA: one TMA producer warp (one lane) streams 64-key K and V tiles with 4-D
// cp.async.bulk.tensor boxes (SWIZZLE_128B, L2 evict_first) into an mbarrier ring — one
// 64-row box per 128-byte column slab for full tiles, 16-row boxes for ragged ends so
// only rows holding valid keys are fetched — and the consumer warps do the math with an
// online softmax in the log2 domain.  Three kernels:
//   attn_tc_kernel    (attn_tc.cuh) head_dim 128 verify with 8 < R <= 128 query rows per KV
//                     head (GQA verify: g*(gamma+1) = 20 / 35 ...): tcgen05 MMAs, S^T and O^T in
//                     TMEM, one CTA / SM.
//   attn_rows_kernel  head_dim 64 verify with R > 8, drafts with g > 8: mma.sync m16n8k16,
//                     query rows on the MMA M dimension (16-row tiles); 2 CTAs / SM.
//   attn_keys_kernel  R <= 8 (every draft call, MHA verify): mma.sync "swap-AB", 16 KV tokens
//                     on M and the query rows on N (padded to 8; an A/B with CUDA-core FMA ran
//                     1.35x slower); 2 CTAs / SM.  Draft calls run the unit-aligned plan (whole
//                     units per CTA, no merges), pack up to 8 / R units of a CTA into one pass
//                     (AttnParams::pack), and with MD_ATTN_EARLY_KV stream their first tiles
//                     (and prefetch the next ones into L2) before the grid-dependency wait.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "md_common.cuh"
#include "md_internal.h"
#include "tcgen05.cuh"

namespace md {

#ifndef MD_KEYS_PF
#define MD_KEYS_PF 0  // experiment (A/B builds only): keys-kernel producer prefetches tile +PF into L2
#endif

constexpr int TK = 64;        // keys per pipeline tile
constexpr int BOX_ROWS = 16;  // rows per TMA box of a partial tile (fetch granularity of ragged ends)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

enum : int { MODE_VERIFY = 0, MODE_DRAFT = 1, MODE_INDEXED = 2 };

// K and V tensor maps with a full-tile box (TK rows) and a partial-tile box (BOX_ROWS rows)
// (the index-list draft copies its listed rows with cp.async: no row maps)
struct TmapSet {
  CUtensorMap k_full, v_full, k_part, v_part;
};

constexpr int XS_FRAGS = 3;  // rows kernel: at most MT * (KS - 1) = 3 parked warp fragments per CTA

struct AttnParams {
  const uint16_t* q;      // bf16 [B][T][Hq][D]
  float* out;             // [B][T][Hq][D]
  float* lse;             // [B][T][Hq] natural log, may be null
  float* ws_o;            // [chunks][2][R][D] normalised partial outputs
  float* ws_lse;          // [chunks][2][R]    partial lse, log2 units (-inf if empty)
  int* counters;          // [B*Hkv] arrival counters (zero between calls)
  const int32_t* kv_len;  // [B]
  int B, Hq, Hkv, T, g, R;
  int sink, window;       // StreamingLLM draft only
  const int32_t* idx;     // SnapKV draft: [B][Hkv][idx_stride] selected prefix positions (ascending)
  const int32_t* idx_count;   // [B] selected positions per (b, kv head)
  const int32_t* tail_start;  // [B] first position of the always-attended tail
  int idx_stride;
  int64_t row_sB, row_sH, row_sS;  // cache strides in units of rows (d elements), for listed rows
  const uint16_t* kc;              // cache K / V base pointers (listed-row copies of MODE_INDEXED)
  const uint16_t* vc;
  unsigned long long* trace;       // diagnostics: [G][8] globaltimer stamps (md_debug_trace), or null
  int* dyn;               // [2] dynamic chunk counter and finished-CTA counter (zero between calls)
  float* ws_x;            // rows kernel: per-CTA [XS_FRAGS][16][D] fragment scratch (key-slice sum)
  int dyn_k;              // dynamic chunks per active CTA (0: static stream-K only)
  int dyn_static_permille;  // share of the tiles assigned statically (per mille)
  int dyn_min_tiles;      // dynamic only when total tiles >= dyn_min_tiles * active CTAs
  const uint32_t* tree_mask;  // verify: [B][T] bit j of (b, t) = node t sees new key n-T+j (null: causal chain)
  // outputs: row o_row(b, kvh, r) of [B][T][out_hq][D]; with tensor parallelism (f1) every
  // rank's full-head buffer out_peers[0..tp_world) receives this rank's heads at head offset
  // out_h0 (stores over NVLink to peer-mapped memory), otherwise only `out`
  float* const* out_peers;
  int tp_world, out_hq, out_h0;
  int pdl_early;          // tcgen05 kernel: trigger the dependent launch at entry (1) or at exit (0)
  const int32_t* windows; // MODE_DRAFT: per-sequence windows [B] or nullptr (p.window for all)
  // fused append (md_*_append): new K/V rows [B][T][Hkv][D] written to cache rows [n-T, n) by
  // the CTA that owns their tile (append_own_rows); null for the plain calls
  const uint16_t* kn;
  const uint16_t* vn;
  uint16_t* kw;                    // writable cache base pointers
  uint16_t* vw;
  int64_t c_sB, c_sH, c_sS;        // cache strides in elements
  int mode;
  float scale_log2;       // scale * log2(e)
  // deterministic fixed-split plan (md_*_det): every unit is cut at multiples of det_split tiles,
  // each piece is one segment with its own partial slot (unit * det_maxp + piece), merged in
  // piece order -> results independent of the grid, of the other units and of how the batch or
  // the KV heads are sharded.  0: the stream-K plan.
  int det_split;
  int det_maxp;
  // unit-aligned static plan (draft calls): every CTA boundary moves forward to the end of the unit
  // holding it, so CTAs process whole units -- no split partials, no merges (short units: a
  // split's epilogue + merge costs more than the byte imbalance of whole units)
  int unit_aligned;
  // dynamic whole-unit plan (draft calls): CTA c starts on unit c, the units >= G are claimed one
  // at a time from an atomic counter (fast SMs take more units; nothing is split or merged); the
  // fused append is then done by the producer warp right before it issues a tile holding a new row
  int unit_dyn;
  int cap;                // cache capacity (rows), for the MD_DEBUG precondition checks
  // MD_ATTN_EARLY_KV (draft, unit-aligned keys kernel): the producer streams the first tiles of its
  // first unit before the grid-dependency wait (kv_len and those rows are final; see the header)
  int early_kv;
  // unit packing (unit-aligned keys kernel, R <= 4): up to `pack` consecutive units of a CTA share
  // one pass -- their query rows side by side in the 8 MMA rows (unit s on rows [sR, sR + R)), their
  // key ranges streamed one after the other, each tile masking the rows of the other units -- so the
  // CTA runs one epilogue for the group instead of one per unit (1 = off)
  int pack;
};

// ------------------------------------------------------------------ stream-K decomposition
// StreamingLLM window of sequence b: p.window, or its own (heterogeneous batches: "different
// sequences in the same batch can leverage different draft KV cache sizes"), clamped
// to [max(0, 1 - sink), p.window] so every sequence attends to at least one key
__device__ __forceinline__ int window_of(const AttnParams& p, int b) {
  return p.windows ? min(p.window, max(max(0, 1 - p.sink), __ldg(p.windows + b))) : p.window;
}
__device__ __forceinline__ int unit_keys(const AttnParams& p, int n, int b) {
  if (p.mode == MODE_VERIFY) return n;
  if (p.mode == MODE_INDEXED) return __ldg(p.idx_count + b) + max(0, n - __ldg(p.tail_start + b));
  const int nA = min(p.sink, n);
  return nA + max(0, n - max(p.sink, n - window_of(p, b)));
}
__device__ __forceinline__ int unit_tiles(const AttnParams& p, int b) {
  return (unit_keys(p, __ldg(p.kv_len + b), b) + TK - 1) / TK;
}
// Visibility of the T new keys [n-T, n) to verify query node t: the
// causal chain (2^(t+1) - 1) or the caller's tree mask (ancestors-or-self of node t).
// A key at offset rel = pos - (n - T) is hidden iff rel >= 0 and bit rel is clear; draft
// modes pass vbase = INT_MAX so rel < 0 always.
__device__ __forceinline__ uint32_t node_mask(const AttnParams& p, int b, int row) {
  const int t = min(row, p.R - 1) / p.g;
  return p.tree_mask ? __ldg(p.tree_mask + (size_t)b * p.T + t) : ((2u << t) - 1u);
}
__device__ __forceinline__ bool key_hidden(uint32_t mask, int rel) { return rel >= 0 && !((mask >> (rel & 31)) & 1u); }

// Per-CTA prefix table over sequences in shared memory: pre[b] = sum_{b' < b} Hkv * tiles(b')
// (built once per CTA with one parallel load of kv_len, so locating a CTA's range costs a
// binary search instead of B dependent global loads).  Batches larger than TABLE_B (256)
// fall back to walking kv_len in global memory.
constexpr int TABLE_B = 256;
constexpr int TABLE_BYTES = (TABLE_B + 1) * 4 + 60;

__device__ void build_prefix(const AttnParams& p, int* pre) {
  if (p.B > TABLE_B) return;
  for (int b = threadIdx.x; b < p.B; b += blockDim.x) pre[b + 1] = unit_tiles(p, b) * p.Hkv;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int run = 0;
    for (int base = 0; base < p.B; base += 32) {
      const int v = base + lane < p.B ? pre[base + lane + 1] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int up = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += up;
      }
      if (base + lane < p.B) pre[base + lane + 1] = run + incl;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) pre[0] = 0;
  }
  __syncthreads();
}
__device__ int64_t total_tiles(const AttnParams& p, const int* pre) {
  if (p.B <= TABLE_B) return pre[p.B];
  int64_t t = 0;
  for (int b = 0; b < p.B; ++b) t += (int64_t)unit_tiles(p, b) * p.Hkv;
  return t;
}
__device__ __forceinline__ int tiles_of(const AttnParams& p, const int* pre, int b) {
  return p.B <= TABLE_B ? (pre[b + 1] - pre[b]) / p.Hkv : unit_tiles(p, b);
}
// Work plan over the global tile space [0, total).  Chunks 0..G-1 are static: equal
// contiguous ranges covering [0, S0), chunk c processed by CTA c.  If dynamic balancing is on,
// chunks G..nch-1 of CH tiles cover [S0, total) and are claimed at run time from an atomic
// counter by whichever CTA's producer runs out of work first (per-SM HBM bandwidth differs
// by several percent, so equal static shares finish at different times).  Every chunk is
// non-empty (S0 >= G, and G = min(gridDim.x, total): an empty chunk would never arrive on a
// unit's counter); CTAs >= G exit at once.  A split unit's partials live in the slots of
// the chunks covering it: chunk * 2 + (0 if the unit is the chunk's first, 1 if its last).
struct Plan {
  int64_t total, S0, CH;
  int G, nch;
  __device__ int64_t start(int c) const {
    return c <= G ? (int64_t)c * S0 / G : min(total, S0 + (int64_t)(c - G) * CH);
  }
  // the chunk holding global tile t: largest c with start(c) <= t
  __device__ int chunk_of(int64_t t) const {
    return t < S0 ? static_cast<int>(((t + 1) * G + S0 - 1) / S0 - 1) : G + static_cast<int>((t - S0) / CH);
  }
  __device__ int slot(int64_t ustart, int c) const { return ustart > start(c) ? 1 : 0; }
};
__device__ Plan make_plan(const AttnParams& p, int64_t total, int grid) {
  Plan pl;
  pl.total = total;
  pl.G = total < (int64_t)grid ? static_cast<int>(total) : grid;
  pl.S0 = total;
  pl.CH = 1;
  pl.nch = pl.G;
  if (p.unit_dyn) {  // chunks are units (cta_range): G = min(grid, units), units >= G are claimed
    const int U = p.B * p.Hkv;
    pl.G = min(grid, U);
    pl.nch = U;
    return pl;
  }
  // short calls (few tiles per CTA, e.g. every draft call) stay static: extra segments and
  // hand-offs cost more there than the bandwidth imbalance they remove
  if (p.dyn_k > 0 && total >= (int64_t)p.dyn_min_tiles * pl.G) {
    const int64_t S0 = max((int64_t)pl.G, total * p.dyn_static_permille / 1000);
    if (S0 < total) {
      const int64_t rest = total - S0, per = (int64_t)pl.G * p.dyn_k;
      pl.S0 = S0;
      pl.CH = (rest + per - 1) / per;
      pl.nch = pl.G + static_cast<int>((rest + pl.CH - 1) / pl.CH);  // <= G * (1 + dyn_k)
    }
  }
  return pl;
}

// MD_DEBUG: the header's device preconditions on kv_len[b] (and the index-list draft's counts)
__device__ __forceinline__ void check_len(const AttnParams& p, int b, int n) {
  MD_DCHECK(n <= p.cap && n >= (p.mode == MODE_VERIFY ? p.T : 1));
  if (p.mode == MODE_INDEXED) {
    const int ts = __ldg(p.tail_start + b), ic = __ldg(p.idx_count + b);
    MD_DCHECK(ts <= n && ic >= 0 && ic <= p.idx_stride && ic + n - ts >= 1);
  }
  (void)b;
}

// One contiguous piece of one unit processed by one CTA: tiles [lo, hi) of `tiles`.
struct Seg {
  int b, kvh, unit, n, tiles, lo, hi;
  int64_t ustart;  // global index of the unit's first tile
  __device__ bool complete() const { return lo == 0 && hi == tiles; }
};

// Walks this CTA's range [S, E) of the global tile space unit by unit.  The producer and
// the consumers each run their own walker over the same range, in the same order.
struct SegWalker {
  int64_t t, end, ustart;
  int b, h, tiles_b;
  int umode;  // 1: whole units t .. end-1 by unit index (unit-aligned plan; no prefix table)
  const int* kvs;  // umode: kv_len of sequences kvs_b0.. staged in shared memory (early-KV calls), or null
  int kvs_b0;
  __device__ void init_units(int u0, int u1, const int* stash = nullptr, int stash_b0 = 0) {
    umode = 1;
    t = u0;
    end = u1;
    kvs = stash;
    kvs_b0 = stash_b0;
  }
  __device__ void init(const AttnParams& p, const int* pre, int64_t S, int64_t E) {
    umode = 0;
    kvs = nullptr;
    t = S;
    end = E;
    int64_t acc = 0;
    if (p.B <= TABLE_B) {  // b = (first index with pre[i] > S) - 1
      int lo = 0, hi = p.B;  // invariant: pre[lo] <= S < pre[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= S) lo = mid;
        else hi = mid;
      }
      b = lo;
      acc = pre[lo];
    } else {
      for (b = 0; b < p.B; ++b) {
        const int64_t blk = (int64_t)unit_tiles(p, b) * p.Hkv;
        if (S < acc + blk) break;
        acc += blk;
      }
    }
    if (b >= p.B) {
      t = end;  // empty range
      return;
    }
    tiles_b = tiles_of(p, pre, b);
    h = static_cast<int>((S - acc) / tiles_b);
    ustart = acc + (int64_t)h * tiles_b;
  }
  __device__ bool next(const AttnParams& p, const int* pre, Seg& sg) {
    if (umode) {  // the next unit with at least one key tile
      while (t < end) {
        const int u = static_cast<int>(t++);
        sg.b = u / p.Hkv;
        sg.kvh = u - sg.b * p.Hkv;
        sg.unit = u;
        sg.n = kvs != nullptr ? kvs[sg.b - kvs_b0] : __ldg(p.kv_len + sg.b);
        check_len(p, sg.b, sg.n);
        sg.tiles = (unit_keys(p, sg.n, sg.b) + TK - 1) / TK;
        sg.lo = 0;
        sg.hi = sg.tiles;
        sg.ustart = 0;  // whole units need no partial slot
        if (sg.tiles > 0) return true;
      }
      return false;
    }
    if (t >= end) return false;
    sg.b = b;
    sg.kvh = h;
    sg.unit = b * p.Hkv + h;
    sg.n = __ldg(p.kv_len + b);
    check_len(p, b, sg.n);
    sg.tiles = tiles_b;
    sg.ustart = ustart;
    sg.lo = static_cast<int>(t - ustart);
    sg.hi = static_cast<int>(min(end, ustart + tiles_b) - ustart);
    if (p.det_split > 0) sg.hi = min(sg.hi, (sg.lo / p.det_split + 1) * p.det_split);  // one piece per segment
    t = ustart + sg.hi;
    if (sg.hi == tiles_b) {  // advance to the next unit (skipping empty sequences)
      ustart += tiles_b;
      if (++h == p.Hkv) {
        h = 0;
        do {
          ++b;
          tiles_b = b < p.B ? tiles_of(p, pre, b) : 0;
        } while (b < p.B && tiles_b == 0);
      }
    }
    return true;
  }
};

// Deterministic plan: a nominal CTA boundary t of the tile space moves forward to the next piece
// boundary of the unit that holds it (ustart + k * det_split, or the unit's end), so every piece
// is processed whole by one CTA.  A pure function of t: neighbouring CTAs agree on it.
__device__ int64_t det_snap(const AttnParams& p, const int* pre, int64_t t, int64_t total) {
  if ((p.det_split <= 0 && !p.unit_aligned) || t >= total) return t;
  SegWalker w;
  w.init(p, pre, t, total);
  if (w.t >= w.end) return total;
  const int64_t rel = t - w.ustart;
  if (rel == 0) return t;
  if (p.det_split <= 0) return w.ustart + w.tiles_b;  // unit-aligned: the end of the unit
  const int64_t snapped = w.ustart + (rel + p.det_split - 1) / p.det_split * p.det_split;
  return min(snapped, w.ustart + (int64_t)w.tiles_b);
}
// this CTA's static range [S, E) of the tile space (chunk = blockIdx.x)
// first tile of unit u = b * Hkv + h (O(1) with the in-CTA prefix table)
__device__ __forceinline__ int64_t unit_start(const AttnParams& p, const int* pre, int u) {
  const int b = u / p.Hkv, h = u - b * p.Hkv;
  if (b >= p.B) return pre[p.B];
  return pre[b] + (int64_t)h * tiles_of(p, pre, b);
}
__device__ __forceinline__ void cta_range(const AttnParams& p, const int* pre, const Plan& pl, int chunk, int64_t& S,
                                          int64_t& E) {
  if (p.unit_dyn) {  // chunk c = unit c (static: c < G, claimed: c >= G)
    S = unit_start(p, pre, chunk);
    E = unit_start(p, pre, chunk + 1);
    return;
  }
  if (p.unit_aligned && p.B <= TABLE_B) {  // whole units, evenly by count: CTA c takes units [cU/G, (c+1)U/G)
    const int U = p.B * p.Hkv;
    S = unit_start(p, pre, (int)((int64_t)chunk * U / pl.G));
    E = unit_start(p, pre, (int)((int64_t)(chunk + 1) * U / pl.G));
    return;
  }
  S = pl.start(chunk);
  E = pl.start(chunk + 1);
  if (p.det_split > 0 || p.unit_aligned) {
    S = det_snap(p, pre, S, pl.total);
    E = det_snap(p, pre, E, pl.total);
  }
}
// partial slot of a segment that does not complete its unit
__device__ __forceinline__ int seg_slot(const AttnParams& p, const Plan& pl, const Seg& sg, int chunk) {
  return p.det_split > 0 ? sg.unit * p.det_maxp + sg.lo / p.det_split : chunk * 2 + pl.slot(sg.ustart, chunk);
}

// Key ranges [s0, e0) then [s1, e1) of the segment's logical keys.  Part 1 is always a range
// of cache rows; part 0 is a range of cache rows too, except in MODE_INDEXED where it is a
// range of positions in the unit's index list (gathered row by row).
struct Ranges {
  int s0, e0, s1, e1;
};
__device__ __forceinline__ Ranges seg_ranges(const AttnParams& p, const Seg& sg) {
  const int keys = unit_keys(p, sg.n, sg.b);
  const int lo = sg.lo * TK, hi = min(keys, sg.hi * TK);
  Ranges r{lo, lo, 0, 0};
  if (p.mode == MODE_VERIFY) {
    r.e0 = max(lo, hi);
  } else if (p.mode == MODE_INDEXED) {
    const int cnt = __ldg(p.idx_count + sg.b), tail = __ldg(p.tail_start + sg.b);
    r.e0 = max(lo, min(hi, cnt));                  // index-list entries
    r.s1 = tail + (max(lo, cnt) - cnt);            // tail rows
    r.e1 = max(r.s1, tail + (hi - cnt));
  } else {
    const int nA = min(p.sink, sg.n);
    const int startB = max(p.sink, sg.n - window_of(p, sg.b));
    r.e0 = max(lo, min(hi, nA));         // sink rows
    r.s1 = startB + (max(lo, nA) - nA);  // window rows
    r.e1 = max(r.s1, startB + (hi - nA));
  }
  return r;
}


// ------------------------------------------------------------------ fused append (a1 in a2/a3)
// md_draft_attn_sparse_append / md_verify_attn_full_append: the T new K/V rows of every
// (b, kv head) go to cache rows [n-T, n) inside the attention kernel, i.e. exactly
// md_kv_append(start = kv_len - T) followed by the attention call.  Every key tile belongs to
// exactly one CTA's static range and every new row lies in some tile (verify reads [0, n); a
// draft window >= 1 ends at n), so each CTA writes the new rows of its own tiles and no CTA
// reads a row another CTA writes.  The writers order their generic stores before the async
// proxy (fence.proxy.async.global) and arrive on an mbarrier that the producer waits on before
// issuing a tile holding a new row (tile_has_new).  Static plans only (the host sets dyn_k = 0).
__device__ __forceinline__ bool tile_has_new(const AttnParams& p, int n, int pos, int nvalid) {
  return p.kn != nullptr && pos < n && pos + nvalid > n - p.T;
}
template <int D>
__device__ void append_own_rows(const AttnParams& p, const int* pre, SegWalker w, int tid, int nthr) {
  constexpr int NV = D / 8;  // 16-byte vectors per row
  Seg sg;
  while (w.next(p, pre, sg)) {
    const Ranges rg = seg_ranges(p, sg);
    const int n = sg.n, nb = n - p.T;
    const int64_t ubase = (int64_t)sg.b * p.c_sB + (int64_t)sg.kvh * p.c_sH;
    // indexed part 0 holds list positions, not rows; part 2 (indexed only): new rows before the
    // streamed tail (tail_start > n - T, e.g. a PQ selection with window 0), which no tile
    // streams, are written by the CTA holding the unit's first tile (listed copies of such rows
    // read k_new / v_new directly in produce_segment, never the cache)
    for (int part = p.mode == MODE_INDEXED ? 1 : 0; part < (p.mode == MODE_INDEXED ? 3 : 2); ++part) {
      int a, e;
      if (part < 2) {
        a = max(part ? rg.s1 : rg.s0, nb);
        e = min(part ? rg.e1 : rg.e0, n);
      } else {
        a = nb;
        e = sg.lo == 0 ? min(n, __ldg(p.tail_start + sg.b)) : nb;
      }
      for (int i = tid; i < (e - a) * NV; i += nthr) {
        const int r = a + i / NV, c = (i % NV) * 8;
        const int64_t src = (((int64_t)sg.b * p.T + (r - nb)) * p.Hkv + sg.kvh) * D + c;
        const int64_t dst = ubase + (int64_t)r * p.c_sS + c;
        const uint4 kv = __ldg(reinterpret_cast<const uint4*>(p.kn + src));
        const uint4 vv = __ldg(reinterpret_cast<const uint4*>(p.vn + src));
        *reinterpret_cast<uint4*>(p.kw + dst) = kv;
        *reinterpret_cast<uint4*>(p.vw + dst) = vv;
      }
    }
  }
  fence_proxy_async_global();
}

// diagnostics: consumer warp 0 / lane 0 stamps phase k of this CTA (md_debug_trace)
constexpr int TRACE_SLOTS = 16;
// Diagnostics (md_debug_trace): slot 0 entry, 1 after the grid-dependency wait, 2 range
// located, 3 first tile landed, 4 last epilogue start, 5 end, 6 smid, 7 last epilogue after
// the cross-warp combine, 8 after its stores, 9 after finish_unit, 10 producer done,
// 11 segments processed, 12 consumer warp 0 done with the fused append, 13 first Q landed
// (consumer warp 0), 14 first Q loads issued (producer).
__device__ __forceinline__ void trace_put(const AttnParams& p, int k, unsigned long long v) {
  if (p.trace != nullptr) p.trace[blockIdx.x * TRACE_SLOTS + k] = v;
}
__device__ __forceinline__ void trace_stamp(const AttnParams& p, int k) {
  if (p.trace != nullptr && threadIdx.x == 0) {
    trace_put(p, k, globaltimer());
    if (k == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace_put(p, 6, smid);
    }
  }
}

__device__ __forceinline__ int64_t out_row(const AttnParams& p, int b, int kvh, int r) {
  return (int64_t)(b * p.T + r / p.g) * p.Hq + kvh * p.g + r % p.g;
}
// row j of a group of consecutive units starting at gu0 (unit gu0 + j / R, its row j % R) in the
// [B][T][Hq] layout of q / out; drafts (T = 1, R = g): row rr of unit u is u * g + rr, so the
// group's rows are contiguous and need no integer divisions
__device__ __forceinline__ int64_t group_row(const AttnParams& p, int gu0, int j) {
  if (p.T == 1) return (int64_t)gu0 * p.g + j;
  const int su = j / p.R, r = j - su * p.R;
  const int bb = (gu0 + su) / p.Hkv, hh = gu0 + su - bb * p.Hkv;
  return out_row(p, bb, hh, r);
}
// row of query row r of unit (b, kvh) in the output layout (local heads, or the TP full-head layout)
__device__ __forceinline__ int64_t o_row(const AttnParams& p, int b, int kvh, int r) {
  return (int64_t)(b * p.T + r / p.g) * p.out_hq + p.out_h0 + kvh * p.g + r % p.g;
}
// final output store: local buffer, or every TP rank's buffer (f1: the all-gather is the store)
template <typename V>
__device__ __forceinline__ void store_out(const AttnParams& p, int64_t off, V v) {
  if (p.out_peers == nullptr) {
    *reinterpret_cast<V*>(p.out + off) = v;
    return;
  }
  for (int k = 0; k < p.tp_world; ++k) {
    float* base = reinterpret_cast<float*>(__ldg(reinterpret_cast<const unsigned long long*>(p.out_peers) + k));
    *reinterpret_cast<V*>(base + off) = v;
  }
}

// ------------------------------------------------------------------ producer
// Stream the K/V tiles of one segment into the ring; `it` is the running tile counter.
// Called by all 32 lanes of the producer warp (lane 0 owns the barriers; in MODE_INDEXED
// every lane copies 2 listed rows of an index-list tile with cp.async).
// skip / limit / stop_at_new (MD_ATTN_EARLY_KV): the first `skip` tiles of the segment were issued
// already (their `it` slots are passed over), at most `limit` tiles are issued, and with stop_at_new
// the walk stops before a tile holding one of the call's new rows.  Returns the tiles issued.
template <int D, int NSTAGE>
__device__ __forceinline__ int produce_segment(const AttnParams& p, const TmapSet& tm, const Ranges& rg, int b,
                                               int kvh, uint8_t* ring, uint64_t* full, uint64_t* empty, int& it,
                                               uint64_t pol, int n = 0, uint64_t* apb = nullptr, int skip = 0,
                                               int limit = 0x7fffffff, bool stop_at_new = false) {
  int tix = 0, issued = 0;
  constexpr int SUB = D / 64, TILE = TK * D * 2, STAGE = 2 * TILE;
  const int lane = threadIdx.x & 31;
  const bool gathered0 = (p.mode == MODE_INDEXED);
  // MODE_INDEXED: the listed rows are copied by all 32 producer lanes with 16-byte cp.async into
  // the SWIZZLE_128B layout the consumers read, completing on the stage's mbarrier through
  // cp.async.mbarrier.arrive.  Lane l owns tile rows 8j + l/4 (j = 0..7) and, of each, the 16-byte
  // chunks 4k + l%4 (k < D/32): one warp instruction moves 64 contiguous bytes of each of 8 rows,
  // and each lane forms one K and one V row address per owned row, the chunks following as
  // immediate offsets.  (Lane-per-row copies -- 32 rows per instruction -- ran at 3.5 TB/s, TMA
  // tile::gather4 at 3.3; tools/gather_probe.py, tools/microbench/gather_sol.cu.)  Each lane's
  // row indices of the NEXT tile are loaded while the current tile is issued.
  constexpr int JR = 8, CPL = D / 32;  // rows per lane and tile, chunks per lane and row
  const int32_t* ip = gathered0 ? p.idx + ((int64_t)b * p.Hkv + kvh) * p.idx_stride : nullptr;
  const int64_t ubase = (int64_t)b * p.row_sB + (int64_t)kvh * p.row_sH;
  const int g8 = lane >> 2, l4 = lane & 3;
  auto load_rows = [&](int pos, int nvalid, int* row) {
#pragma unroll
    for (int j = 0; j < JR; ++j) row[j] = (8 * j + g8 < nvalid) ? __ldg(ip + pos + 8 * j + g8) : -1;
  };
  int rows_next[JR];
#pragma unroll
  for (int j = 0; j < JR; ++j) rows_next[j] = -1;
  if (gathered0 && rg.s0 < rg.e0) load_rows(rg.s0, min(TK, rg.e0 - rg.s0), rows_next);
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
#pragma unroll 1
    for (int pos = rs; pos < re; pos += TK, ++it, ++tix) {
      const int stage = it % NSTAGE;
      const int nvalid = min(TK, re - pos);
      uint8_t* kt = ring + stage * STAGE;
      uint8_t* vt = kt + TILE;
      if (tix < skip) continue;  // issued before the grid-dependency wait
      if (issued == limit || (stop_at_new && tile_has_new(p, n, pos, nvalid))) return issued;
      ++issued;
      if (part == 0 && gathered0) {
        int row[JR];
#pragma unroll
        for (int j = 0; j < JR; ++j) row[j] = rows_next[j];
        const int npos = pos + TK;
        if (npos < re) load_rows(npos, min(TK, re - npos), rows_next);
        // every copying lane acquires the stage itself (the consumers' release of its previous
        // contents), so no lane's copies rely on ordering through another lane
        mbar_wait(&empty[stage], ((it / NSTAGE) & 1) ^ 1);
        __syncwarp();
        const uint32_t kt_a = smem_u32(kt) + g8 * 128, vt_a = smem_u32(vt) + g8 * 128;
#pragma unroll
        for (int j = 0; j < JR; ++j) {
          if (row[j] < 0) continue;  // rows past the tile's valid keys stay stale (masked / zeroed)
          const uint16_t* ks = p.kc + (ubase + (int64_t)row[j] * p.row_sS) * D;
          const uint16_t* vs = p.vc + (ubase + (int64_t)row[j] * p.row_sS) * D;
          if (p.kn != nullptr && row[j] >= n - p.T) {  // fused append: a new row, from k_new / v_new
            const int64_t src = (((int64_t)b * p.T + (row[j] - (n - p.T))) * p.Hkv + kvh) * D;
            ks = p.kn + src;
            vs = p.vn + src;
          }
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            const int c = 4 * k + l4;  // chunk; the tile row is 8j + g8, so (row & 7) == g8
            const uint32_t dst = (uint32_t)((c >> 3) * TK * 128 + j * 1024 + (((c & 7) ^ g8) << 4));
            cp_async16_pol(kt_a + dst, ks + c * 8, pol);
            cp_async16_pol(vt_a + dst, vs + c * 8, pol);
          }
        }
        // MODE_INDEXED: full[] expects one arrival per producer lane; this one fires when the
        // lane's copies have landed
        cp_async_arrive_noinc(&full[stage]);
        continue;
      }
      if (p.unit_dyn && p.kn != nullptr && tile_has_new(p, n, pos, nvalid)) {
        // dynamic-unit plan: the producer warp writes the new rows of this tile itself (generic
        // stores ordered before its own TMA reads by fence.proxy.async + __syncwarp)
        constexpr int NV = D / 8;
        const int a = max(pos, n - p.T), e = min(pos + nvalid, n);
        const int64_t ubase = (int64_t)b * p.c_sB + (int64_t)kvh * p.c_sH;
        for (int i = lane; i < (e - a) * NV; i += 32) {
          const int r = a + i / NV, c = (i % NV) * 8;
          const int64_t src = (((int64_t)b * p.T + (r - (n - p.T))) * p.Hkv + kvh) * D + c;
          const int64_t dst = ubase + (int64_t)r * p.c_sS + c;
          *reinterpret_cast<uint4*>(p.kw + dst) = __ldg(reinterpret_cast<const uint4*>(p.kn + src));
          *reinterpret_cast<uint4*>(p.vw + dst) = __ldg(reinterpret_cast<const uint4*>(p.vn + src));
        }
        fence_proxy_async_global();
        __syncwarp();
      }
      if (gathered0) {  // MODE_INDEXED (the streamed tail): full[] expects all 32 producer lanes
        mbar_wait(&empty[stage], ((it / NSTAGE) & 1) ^ 1);
        if (lane != 0) {
          mbar_arrive(&full[stage]);
          continue;
        }
      } else if (lane != 0) {
        continue;
      }
      if (apb != nullptr && tile_has_new(p, n, pos, nvalid)) mbar_wait(apb, 0);  // fused append done
      mbar_wait(&empty[stage], ((it / NSTAGE) & 1) ^ 1);
      if (nvalid == TK) {  // full tile: one TK-row box per 128-byte column slab
        mbar_arrive_expect_tx(&full[stage], STAGE);
        for (int sub = 0; sub < SUB; ++sub) {
          tma_load_4d(kt + sub * TK * 128, &tm.k_full, &full[stage], sub * 64, pos, kvh, b, pol);
          tma_load_4d(vt + sub * TK * 128, &tm.v_full, &full[stage], sub * 64, pos, kvh, b, pol);
        }
        if (MD_KEYS_PF > 0 && pos + (MD_KEYS_PF + 1) * TK <= re) {  // experiment: L2 prefetch ahead of the ring
          const int pp = pos + MD_KEYS_PF * TK;
          for (int sub = 0; sub < SUB; ++sub) {
            tma_prefetch_4d(&tm.k_full, sub * 64, pp, kvh, b);
            tma_prefetch_4d(&tm.v_full, sub * 64, pp, kvh, b);
          }
        }
      } else {  // ragged end: only the BOX_ROWS-row boxes that hold valid keys
        const int nbox = (nvalid + BOX_ROWS - 1) / BOX_ROWS;
        mbar_arrive_expect_tx(&full[stage], nbox * BOX_ROWS * 128 * SUB * 2);
        for (int sub = 0; sub < SUB; ++sub)
          for (int bx = 0; bx < nbox; ++bx) {
            const int off = sub * TK * 128 + bx * BOX_ROWS * 128;
            tma_load_4d(kt + off, &tm.k_part, &full[stage], sub * 64, pos + bx * BOX_ROWS, kvh, b, pol);
            tma_load_4d(vt + off, &tm.v_part, &full[stage], sub * 64, pos + bx * BOX_ROWS, kvh, b, pol);
          }
      }
    }
  }
  return issued;
}

// ------------------------------------------------------------------ cross-CTA finish
// Called by all `nthr` consumer threads after this CTA stored its partial of `sg`.  The
// last CTA to arrive for the unit combines every contributor's partial (O6 identity):
// o = sum_c 2^{lse_c - M} o_c / sum_c 2^{lse_c - M}.  bar.sync orders every thread's
// partial stores before thread 0's release-add; the acq_rel atomic of the last arriver
// makes all contributors' stores visible to its CTA (read back with ld.global.cg).
template <int D>
__device__ void finish_unit(const AttnParams& p, const Seg& sg, const Plan& pl, int nthr, int* flag) {
  named_bar_sync(1, nthr);
  if (threadIdx.x == 0 && p.det_split > 0) {  // deterministic plan: pieces 0 .. np-1 of the unit
    const int np = (sg.tiles + p.det_split - 1) / p.det_split;
    const int old = atomic_add_acq_rel_gpu(p.counters + sg.unit, 1);
    const int last = (old == np - 1);
    if (last) p.counters[sg.unit] = 0;
    flag[0] = last;
    flag[1] = 0;
    flag[2] = np - 1;
    flag[3] = 0;
  } else if (threadIdx.x == 0) {
    const int cf = pl.chunk_of(sg.ustart), cl = pl.chunk_of(sg.ustart + sg.tiles - 1);
    const int old = atomic_add_acq_rel_gpu(p.counters + sg.unit, 1);
    const int last = (old == cl - cf);
    if (last) p.counters[sg.unit] = 0;  // leave the workspace ready for the next call
    flag[0] = last;
    flag[1] = cf;
    flag[2] = cl;
    // the unit is the LAST segment of chunk cf iff cf began before it (slot 1); for every
    // later chunk it is the first segment (slot 0)
    flag[3] = pl.slot(sg.ustart, cf);
  }
  named_bar_sync(1, nthr);
  if (!flag[0]) return;
  const int cf = flag[1], cl = flag[2], s0 = flag[3];
  // each thread owns (row, 4 columns) elements; every partial's lse and values are loaded
  // together and combined online, so the merge costs one L2 round trip per partial
  constexpr int V4 = D / 4;
  for (int idx = threadIdx.x; idx < p.R * V4; idx += nthr) {
    const int r = idx / V4, c4 = (idx - r * V4) * 4;
    float M = -INFINITY, W = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
    for (int c = cf; c <= cl; ++c) {
      const int64_t prow = (p.det_split > 0 ? (int64_t)sg.unit * p.det_maxp + c : (int64_t)c * 2 + (c == cf ? s0 : 0)) *
                               p.R + r;
      const float ls = __ldcg(p.ws_lse + prow);
      const float4 v = __ldcg(reinterpret_cast<const float4*>(p.ws_o + prow * D + c4));
      if (ls == -INFINITY) continue;  // an empty partial
      const float mn = fmaxf(M, ls);
      const float a = ex2(M - mn), w = ex2(ls - mn);  // a = 0 on the first partial
      M = mn;
      W = W * a + w;
      acc.x = acc.x * a + w * v.x;
      acc.y = acc.y * a + w * v.y;
      acc.z = acc.z * a + w * v.z;
      acc.w = acc.w * a + w * v.w;
    }
    const float inv = W > 0.f ? 1.f / W : 0.f;
    store_out(p, o_row(p, sg.b, sg.kvh, r) * D + c4, make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
    if (c4 == 0 && p.lse != nullptr) p.lse[out_row(p, sg.b, sg.kvh, r)] = (W > 0.f) ? (M + __log2f(W)) * LN2 : -INFINITY;
  }
}

// ============================================================================ rows kernel
// Query rows on the MMA M dimension.  Consumer warp (mt, ks) owns query-row tile mt (16 of
// the R rows) and the ks-th KW-key slice of every 64-key tile: S = Q K^T, O += P V.
// 2 CTAs / SM.  The key-slice sum of the epilogue goes through a per-CTA scratch in the
// workspace (L2-resident), so the ring is never aliased and the producer streams straight
// across segment boundaries (and dynamic chunks).
template <int D>
struct RowsSmem {
  static constexpr int NSTAGE = 3;  // 3 x 32 KB at d=128 -> 2 CTAs / SM
  static constexpr int TILE_BYTES = TK * D * 2;
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  static constexpr int RING_BYTES = NSTAGE * STAGE_BYTES;
  static constexpr int EPI_BYTES = 4 * 16 * 2 * 4 + 4 * 16 * 4;  // mlbuf [NC<=4][16][2] + lsebuf [MT<=4][16]
  static constexpr int TOTAL = RING_BYTES + 1024 /*align slack*/ + (2 * NSTAGE + 4) * 8 + 16 /*cids*/ + 128 /*flag, plan*/ +
                               EPI_BYTES + TABLE_BYTES;
};

// 2 CTAs / SM (ptxas then keeps <= 3 warps' registers per SM sub-partition: 168 regs at 5 warps).
template <int D, int MT, int KS>
__global__ void __launch_bounds__((MT * KS + 1) * 32, 2)
    attn_rows_kernel(const __grid_constant__ TmapSet tm, const AttnParams p) {
  constexpr int NC = MT * KS;  // consumer warps
  constexpr int KW = TK / KS;  // keys per consumer warp per tile
  constexpr int NT_S = KW / 8; // n8 tiles of S per warp
  constexpr int NT_O = D / 8;  // n8 tiles of O
  constexpr int KQ = D / 16;   // k16 steps of QK^T
  using L = RowsSmem<D>;
  constexpr int NSTAGE = L::NSTAGE;
  static_assert(KW % 16 == 0, "key slice must be a multiple of 16");
  static_assert(NC <= 4 && MT <= 4 && MT * (KS - 1) <= XS_FRAGS, "epilogue buffers are sized for <= 4 warps");

  extern __shared__ uint8_t smem_raw[];
  // align to 1 KB by offsetting the __shared__ array itself, so every derived pointer keeps
  // the shared address space (LDS/STS instead of generic loads/stores)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::RING_BYTES);
  uint64_t* empty = full + NSTAGE;
  uint64_t* cfull = empty + NSTAGE;  // dynamic chunk hand-off, producer -> consumers (2 slots)
  uint64_t* cempty = cfull + 2;
  int* cids = reinterpret_cast<int*>(cempty + 2);
  int* flag = cids + 4;                                   // [16] finish_unit
  Plan* plan_smem = reinterpret_cast<Plan*>(flag + 16);   // 40 bytes (reserved 64)
  float* mlbuf = reinterpret_cast<float*>(flag + 32);     // [NC][16][2] (m, l) per warp row
  float* lsebuf = mlbuf + 4 * 16 * 2;                     // [MT*16] combined lse (log2)
  int* pre = reinterpret_cast<int*>(lsebuf + 4 * 16);     // [TABLE_B + 1] per-sequence tile prefix

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], NC);
    }
    fence_mbar_init();
  }
  trace_stamp(p, 0);
  pdl_trigger();
  pdl_wait();  // kv_len, the cache and q may come from the previous kernel
  trace_stamp(p, 1);
  __syncthreads();
  build_prefix(p, pre);
  // the plan lives in shared memory (read only at segment boundaries: keeps registers free)
  if (threadIdx.x == 0) *plan_smem = make_plan(p, total_tiles(p, pre), gridDim.x);
  __syncthreads();
  const Plan& pl = *plan_smem;
  if ((int)blockIdx.x >= pl.G) return;  // uniform across the CTA
  int chunk = blockIdx.x;                // this CTA's static chunk, then claimed dynamic ones
  SegWalker walk;
  {
    int64_t S0, E0;
    cta_range(p, pre, pl, chunk, S0, E0);
    walk.init(p, pre, S0, E0);
  }
  Seg sg;
  trace_stamp(p, 2);

  if (warp == NC) {
    // ============================== TMA producer warp ==============================
    if (lane == 0) {
      prefetch_tmap(&tm.k_full);
      prefetch_tmap(&tm.v_full);
      prefetch_tmap(&tm.k_part);
      prefetch_tmap(&tm.v_part);
    }
    const uint64_t pol = policy_evict_first();
    int it = 0, ck = 0;
    int ahead = 0;  // dynamic chunk claimed one ahead (see the keys kernel)
    if (pl.nch > pl.G && lane == 0) ahead = atomicAdd(p.dyn, 1);
    auto next_seg = [&]() -> bool {
      while (!walk.next(p, pre, sg)) {
        if (pl.nch == pl.G) return false;
        int nxt = -1;
        if (lane == 0) {
          const int c = pl.G + ahead;
          nxt = c < pl.nch ? c : -1;
          if (nxt >= 0) ahead = atomicAdd(p.dyn, 1);
          const int cs = ck & 1;
          mbar_wait(&cempty[cs], ((ck >> 1) & 1) ^ 1);
          cids[cs] = nxt;
          mbar_arrive(&cfull[cs]);
        }
        nxt = __shfl_sync(0xffffffffu, nxt, 0);
        ++ck;
        if (nxt < 0) return false;
        chunk = nxt;
        {
          int64_t S_, E_;
          cta_range(p, pre, pl, chunk, S_, E_);
          walk.init(p, pre, S_, E_);
        }
      }
      return true;
    };
    while (next_seg())
      produce_segment<D, NSTAGE>(p, tm, seg_ranges(p, sg), sg.b, sg.kvh, smem, full, empty, it, pol);
    return;
  }

  // ============================== consumers ==============================
  const int mt = warp / KS, ks = warp - mt * KS;
  const int gq = lane >> 2, cq = lane & 3;  // fragment row group / column quad
  const uint32_t ring = smem_u32(smem);
  int it = 0, ck = 0;
  auto next_seg = [&]() -> bool {  // mirrors the producer's chunk sequence
    while (!walk.next(p, pre, sg)) {
      if (pl.nch == pl.G) return false;
      const int cs = ck & 1;
      mbar_wait(&cfull[cs], (ck >> 1) & 1);
      const int nxt = cids[cs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty[cs]);
      ++ck;
      if (nxt < 0) return false;
      chunk = nxt;
      {
        int64_t S_, E_;
        cta_range(p, pre, pl, chunk, S_, E_);
        walk.init(p, pre, S_, E_);
      }
    }
    return true;
  };
  while (next_seg()) {
    const int b = sg.b, kvh = sg.kvh, n = sg.n;
    const Ranges rg = seg_ranges(p, sg);
    // Q fragments for rows mt*16 + {gq, gq+8}; row r -> (t = r / g, head = kvh*g + r % g)
    uint32_t qa[KQ][4];
    {
      const int r0 = mt * 16 + gq, r1 = r0 + 8;
      const uint32_t* q0 = r0 < p.R ? reinterpret_cast<const uint32_t*>(p.q + out_row(p, b, kvh, r0) * D) : nullptr;
      const uint32_t* q1 = r1 < p.R ? reinterpret_cast<const uint32_t*>(p.q + out_row(p, b, kvh, r1) * D) : nullptr;
#pragma unroll
      for (int kk = 0; kk < KQ; ++kk) {
        const int c = kk * 8 + cq;  // 32-bit word index = (kk*16 + 2*cq) / 2
        qa[kk][0] = q0 ? __ldg(q0 + c) : 0u;
        qa[kk][1] = q1 ? __ldg(q1 + c) : 0u;
        qa[kk][2] = q0 ? __ldg(q0 + c + 4) : 0u;
        qa[kk][3] = q1 ? __ldg(q1 + c + 4) : 0u;
      }
    }
    // visibility of the new keys per fragment row (verify): node_mask of t(row)
    const int vbase = (p.mode == MODE_VERIFY) ? n - p.T : 0x7fffffff;  // keys < vbase: visible to all rows
    const uint32_t msk0 = node_mask(p, b, mt * 16 + gq), msk1 = node_mask(p, b, mt * 16 + gq + 8);

    float o[NT_O][4];
#pragma unroll
    for (int i = 0; i < NT_O; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
#pragma unroll 1
      for (int pos = rs; pos < re; pos += TK, ++it) {
        const int stage = it % NSTAGE;
        mbar_wait(&full[stage], (it / NSTAGE) & 1);
        if (it == 0) trace_stamp(p, 3);
        const int nvalid = min(TK, re - pos);
        const int kw0 = ks * KW;
        if (kw0 < nvalid) {
          const uint32_t kt = ring + stage * L::STAGE_BYTES;
          const uint32_t vt = kt + L::TILE_BYTES;
          // ---------------- S = Q K^T  (16 rows x KW keys)
          float s[NT_S][4];
#pragma unroll
          for (int i = 0; i < NT_S; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
          for (int kk = 0; kk < KQ; ++kk) {
#pragma unroll
            for (int np = 0; np < NT_S / 2; ++np) {
              const int row = kw0 + np * 16 + ((lane >> 4) << 3) + (lane & 7);
              const int chunk = kk * 2 + ((lane >> 3) & 1);
              uint32_t b0, b1, b2, b3;
              ldsm_x4(kt + (chunk >> 3) * (TK * 128) + swz128(row, chunk & 7), b0, b1, b2, b3);
              mma_bf16_16816(s[2 * np], qa[kk], b0, b1);
              mma_bf16_16816(s[2 * np + 1], qa[kk], b2, b3);
            }
          }
          // ---------------- scale, mask, online softmax (log2 domain)
          const bool need_mask = (kw0 + KW > nvalid) || (pos + kw0 + KW - 1 >= vbase);
          float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
          for (int i = 0; i < NT_S; ++i) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float v = s[i][e] * p.scale_log2;
              if (need_mask) {
                const int ko = kw0 + i * 8 + cq * 2 + (e & 1);
                v = (ko >= nvalid || key_hidden((e < 2) ? msk0 : msk1, pos + ko - vbase)) ? -INFINITY : v;
              }
              s[i][e] = v;
            }
            mx0 = fmaxf(mx0, fmaxf(s[i][0], s[i][1]));
            mx1 = fmaxf(mx1, fmaxf(s[i][2], s[i][3]));
          }
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
          const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
          const float base0 = (mn0 == -INFINITY) ? 0.f : mn0;
          const float base1 = (mn1 == -INFINITY) ? 0.f : mn1;
          const float corr0 = ex2(m0 - base0), corr1 = ex2(m1 - base1);
          m0 = mn0;
          m1 = mn1;
          float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
          for (int i = 0; i < NT_S; ++i) {
            s[i][0] = ex2(s[i][0] - base0);
            s[i][1] = ex2(s[i][1] - base0);
            s[i][2] = ex2(s[i][2] - base1);
            s[i][3] = ex2(s[i][3] - base1);
            rs0 += s[i][0] + s[i][1];
            rs1 += s[i][2] + s[i][3];
          }
          l0 = l0 * corr0 + rs0;
          l1 = l1 * corr1 + rs1;
          if (__any_sync(0xffffffffu, corr0 != 1.f || corr1 != 1.f)) {
#pragma unroll
            for (int i = 0; i < NT_O; ++i) {
              o[i][0] *= corr0;
              o[i][1] *= corr0;
              o[i][2] *= corr1;
              o[i][3] *= corr1;
            }
          }
          // ---------------- O += P V
          const bool sanitize = kw0 + KW > nvalid;
#pragma unroll
          for (int kp = 0; kp < KW / 16; ++kp) {
            uint32_t a[4];
            a[0] = pack_bf16(s[2 * kp][0], s[2 * kp][1]);
            a[1] = pack_bf16(s[2 * kp][2], s[2 * kp][3]);
            a[2] = pack_bf16(s[2 * kp + 1][0], s[2 * kp + 1][1]);
            a[3] = pack_bf16(s[2 * kp + 1][2], s[2 * kp + 1][3]);
            const int krow = kw0 + kp * 16 + (((lane >> 3) & 1) << 3) + (lane & 7);
            const int kf = kw0 + kp * 16 + cq * 2;  // keys this thread's B fragments hold
            const uint32_t m_lo = (kf < nvalid ? 0x0000ffffu : 0u) | (kf + 1 < nvalid ? 0xffff0000u : 0u);
            const uint32_t m_hi = (kf + 8 < nvalid ? 0x0000ffffu : 0u) | (kf + 9 < nvalid ? 0xffff0000u : 0u);
#pragma unroll
            for (int dp = 0; dp < NT_O / 2; ++dp) {
              const int chunk = dp * 2 + (lane >> 4);
              uint32_t b0, b1, b2, b3;
              ldsm_x4_t(vt + (chunk >> 3) * (TK * 128) + swz128(krow, chunk & 7), b0, b1, b2, b3);
              if (sanitize) {  // rows past the valid keys may hold non-finite bits: zero them
                b0 &= m_lo;
                b1 &= m_hi;
                b2 &= m_lo;
                b3 &= m_hi;
              }
              mma_bf16_16816(o[2 * dp], a, b0, b1);
              mma_bf16_16816(o[2 * dp + 1], a, b2, b3);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      }
    }

    // ============================== segment epilogue ==============================
    // The ring is not touched: the producer keeps streaming the next segment meanwhile.
    trace_stamp(p, 4);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    if (cq == 0) {
      mlbuf[(warp * 16 + gq) * 2 + 0] = m0;
      mlbuf[(warp * 16 + gq) * 2 + 1] = l0;
      mlbuf[(warp * 16 + gq + 8) * 2 + 0] = m1;
      mlbuf[(warp * 16 + gq + 8) * 2 + 1] = l1;
    }
    named_bar_sync(1, NC * 32);
    // scale this warp's O by 2^(m_w - M) / L where (M, L) combine the KS key slices
    float f0, f1;
    {
      float M0 = -INFINITY, M1 = -INFINITY;
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        M0 = fmaxf(M0, mlbuf[((mt * KS + k) * 16 + gq) * 2]);
        M1 = fmaxf(M1, mlbuf[((mt * KS + k) * 16 + gq + 8) * 2]);
      }
      float L0 = 0.f, L1 = 0.f;
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const float* e0 = &mlbuf[((mt * KS + k) * 16 + gq) * 2];
        const float* e1 = &mlbuf[((mt * KS + k) * 16 + gq + 8) * 2];
        if (e0[1] > 0.f) L0 += e0[1] * ex2(e0[0] - M0);
        if (e1[1] > 0.f) L1 += e1[1] * ex2(e1[0] - M1);
      }
      f0 = (l0 > 0.f) ? ex2(m0 - M0) / L0 : 0.f;
      f1 = (l1 > 0.f) ? ex2(m1 - M1) / L1 : 0.f;
      if (ks == 0 && cq == 0) {
        lsebuf[mt * 16 + gq] = (L0 > 0.f) ? M0 + __log2f(L0) : -INFINITY;
        lsebuf[mt * 16 + gq + 8] = (L1 > 0.f) ? M1 + __log2f(L1) : -INFINITY;
      }
    }
#pragma unroll
    for (int i = 0; i < NT_O; ++i) {
      o[i][0] *= f0;
      o[i][1] *= f0;
      o[i][2] *= f1;
      o[i][3] *= f1;
    }
    // key-slice sum: warps ks >= 1 park their fragments in the CTA's global scratch (lane-major,
    // coalesced), warps ks == 0 add them (L2 hits, L1 bypassed) and store their 16 rows
    if (KS > 1) {
      float* xs = p.ws_x + (size_t)blockIdx.x * XS_FRAGS * 16 * D;  // this CTA's fragment scratch
      if (ks > 0) {
        float* dst = xs + (size_t)(mt * (KS - 1) + ks - 1) * 16 * D;
#pragma unroll
        for (int i = 0; i < NT_O; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) __stcg(dst + (i * 4 + e) * 32 + lane, o[i][e]);
      }
      named_bar_sync(1, NC * 32);
      if (ks == 0) {
#pragma unroll
        for (int k = 1; k < KS; ++k) {
          const float* src = xs + (size_t)(mt * (KS - 1) + k - 1) * 16 * D;
#pragma unroll
          for (int i = 0; i < NT_O; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) o[i][e] += __ldcg(src + (i * 4 + e) * 32 + lane);
        }
      }
    } else {
      named_bar_sync(1, NC * 32);  // lsebuf
    }
    // rows r < R -> the final output, or this chunk's partial slot
    const bool complete = sg.complete();
    const int slot_base = seg_slot(p, pl, sg, chunk);
    if (ks == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = mt * 16 + gq + h * 8;
        if (r < p.R) {
          if (complete) {
            const int64_t orow = o_row(p, b, kvh, r) * D;
            if (cq == 0 && p.lse != nullptr) p.lse[out_row(p, b, kvh, r)] = lsebuf[r] * LN2;
#pragma unroll
            for (int i = 0; i < NT_O; ++i) store_out(p, orow + i * 8 + cq * 2, make_float2(o[i][2 * h], o[i][2 * h + 1]));
          } else {
            const int64_t prow = (int64_t)slot_base * p.R + r;
            float* dst = p.ws_o + prow * D;
            if (cq == 0) __stcg(p.ws_lse + prow, lsebuf[r]);
#pragma unroll
            for (int i = 0; i < NT_O; ++i)
              __stcg(reinterpret_cast<float2*>(dst + i * 8 + cq * 2), make_float2(o[i][2 * h], o[i][2 * h + 1]));
          }
        }
      }
    }
    if (!complete) finish_unit<D>(p, sg, pl, NC * 32, flag);
    named_bar_sync(1, NC * 32);  // mlbuf / lsebuf / scratch reused by the next segment
    trace_stamp(p, 5);
  }
  // the last CTA to finish re-arms the dynamic counters for the next call
  if (pl.nch > pl.G && threadIdx.x == 0) {
    if (atomicAdd(p.dyn + 1, 1) == pl.G - 1) {
      p.dyn[0] = 0;
      p.dyn[1] = 0;
    }
  }
}

// ============================================================================ keys kernel
// Swap-AB for R <= 8 query rows: consumer warp ks computes S^T = K Q^T (16 KV tokens on M,
// the query rows on N) and O^T += V^T P^T over keys [ks*KW, (ks+1)*KW) of every tile; the
// P^T operand is the bf16-packed S^T fragment transposed in registers (movmatrix).  One
// CTA / SM with a dedicated epilogue buffer, so the producer streams across segment
// boundaries; each segment's Q rows are bulk-copied into a double-buffered padded slot.
#ifndef MD_DIRECT_UNITS
#define MD_DIRECT_UNITS 1  // unit-aligned keys-kernel calls walk their units without a prefix table (0: A/B builds)
#endif
#ifndef MD_EARLY_PF
// early-KV draft prologue: full tiles prefetched into L2 beyond the NSTAGE issued to shared memory
// (graph-timed sweep 0 / 2 / 3 / 4 / 5 / 6 / 8 / 16 / 32, profiles/draft_ab_r02_early_l2pf*.txt:
// 3 best, Llama-3.1 47.2 -> 45.8 us, Qwen2.5 45.4 -> 43.7, B = 128 88.6 -> 87.4; 16+ slower)
#define MD_EARLY_PF 3
#endif
#ifndef MD_EPF_AFTER
#define MD_EPF_AFTER 0  // experiment (A/B builds only): the early L2 prefetch after the wait and the first Q loads
#endif
#ifndef MD_PACK_UNITS
#define MD_PACK_UNITS 1  // unit packing for R <= 4 drafts (AttnParams::pack; 0: A/B builds)
#endif
#ifndef MD_EXP_FMA
#define MD_EXP_FMA 0  // experiment (A/B builds only): R <= 4 draft segments on CUDA-core FMA (fma_segment)
#endif
#ifndef MD_EXP_EPI
#define MD_EXP_EPI 0  // experiment (A/B builds only): keys kernel skips 1 = all output stores, 2 = lse, 3 = out
#endif
#ifndef MD_EXP_NOMATH
#define MD_EXP_NOMATH 0  // experiment (A/B builds only): the keys kernel skips its tile math
#endif
template <int D, int KS, int CTAS>
struct KeysCfg {
  static constexpr int NC = KS;
  static constexpr int THREADS = (NC + 1) * 32;  // + TMA producer warp
  static constexpr int KW = TK / KS;       // keys per consumer warp per tile
  static constexpr int KB = KW / 16;       // 16-key blocks per warp per tile
  static constexpr int ROWS = 8;           // query rows (padded)
  static constexpr int TILE = TK * D * 2;
  static constexpr int STAGE = 2 * TILE;
  static constexpr int QSTR = D * 2 + 16;  // padded smem row of Q (conflict-free ldmatrix)
  static constexpr int QBUF = 2 * ROWS * QSTR;
  static constexpr int FRAG = (D / 16) * 4 * 32;  // fp32 of one warp's O^T fragments
  static constexpr int EPI = (NC / 2) * FRAG * 4 + NC * ROWS * 2 * 4 + ROWS * 4 + 64;
  static constexpr int FIXED = QBUF + EPI + 256 /*barriers, hand-off slots*/ + TABLE_BYTES + 1024 /*alignment slack*/;
  static constexpr int NSTAGE_FIT = ((CTAS == 1 ? 227 * 1024 : 112 * 1024) - FIXED) / STAGE;
  static constexpr int NSTAGE = NSTAGE_FIT > 8 ? 8 : NSTAGE_FIT;
  static constexpr int SMEM = NSTAGE * STAGE + FIXED;
  static_assert(NSTAGE >= 2, "not enough shared memory for a 2-stage ring");
  static_assert(KW % 16 == 0, "key slice must be a multiple of 16");
};

#if MD_EXP_FMA
#include "attn_exp_fma.cuh"  // experiment only: CUDA-core FMA draft consumer (A/B builds)
#endif

// early-KV draft calls: the next MD_EARLY_PF full tiles of the CTA's units after the NSTAGE issued
// to shared memory, prefetched into L2 (a hint: safe whatever the previous kernel still writes --
// L2 is the point of coherence), so the CTAs that become resident during the previous call's tail
// fill its idle HBM bandwidth with this call's reads.  s0 / w0: the first unit and its walker.
template <int D>
__device__ void early_l2_prefetch(const AttnParams& p, const TmapSet& tm, const int* pre, Seg su, SegWalker w0,
                                  int skip) {
  int left = MD_EARLY_PF;
  do {
    const Ranges rg = seg_ranges(p, su);
    for (int part = 0; part < 2 && left > 0; ++part) {
      const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
      for (int pos = rs; pos + TK <= re && left > 0; pos += TK) {
        if (skip > 0) {
          --skip;
          continue;
        }
        for (int sub = 0; sub < D / 64; ++sub) {
          tma_prefetch_4d(&tm.k_full, sub * 64, pos, su.kvh, su.b);
          tma_prefetch_4d(&tm.v_full, sub * 64, pos, su.kvh, su.b);
        }
        --left;
      }
    }
    skip = 0;
  } while (left > 0 && w0.next(p, pre, su));
}

template <int D, int KS, int CTAS, bool EARLY>
__global__ void __launch_bounds__(KeysCfg<D, KS, CTAS>::THREADS, CTAS)
    attn_keys_kernel(const __grid_constant__ TmapSet tm, const AttnParams p) {
  using C = KeysCfg<D, KS, CTAS>;
  constexpr int NC = C::NC, KW = C::KW, KB = C::KB, NSTAGE = C::NSTAGE, FRAG = C::FRAG;
  static_assert(NC == 4, "the epilogue tree merge assumes 4 consumer warps");
  constexpr int MD16 = D / 16;  // m16 tiles of O^T (head-dim rows) == k16 steps of S^T

  extern __shared__ uint8_t smem_raw[];
  // align to 1 KB by offsetting the __shared__ array itself, so every derived pointer keeps
  // the shared address space (LDS/STS instead of generic loads/stores)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* qbuf = smem + NSTAGE * C::STAGE;
  float* obuf = reinterpret_cast<float*>(qbuf + C::QBUF);  // [NC/2][FRAG]    O^T fragments (tree merge)
  float* mlbuf = obuf + (NC / 2) * FRAG;                    // [NC][8][2]      (m, l) per warp row
  float* lsebuf = mlbuf + NC * C::ROWS * 2;                 // [8]             combined lse (log2)
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(obuf) + C::EPI);
  uint64_t* empty = full + NSTAGE;
  uint64_t* qfull = empty + NSTAGE;
  uint64_t* qempty = qfull + 2;
  uint64_t* cfull = qempty + 2;   // dynamic chunk hand-off, producer -> consumers (2 slots)
  uint64_t* cempty = cfull + 2;
  uint64_t* apb = cempty + 2;     // fused append: the consumers' new-row stores are done
  int* cids = reinterpret_cast<int*>(apb + 1);
  int* flag = cids + 2;  // [4] finish_unit
  Plan* plan_smem = reinterpret_cast<Plan*>(flag + 4);  // 40 bytes (reserved 48)
  int* pre = flag + 16;  // [TABLE_B + 1] per-sequence tile prefix

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], p.mode == MODE_INDEXED ? 32 : 1);  // indexed: every producer lane arrives
      mbar_init(&empty[s], NC);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], NC);
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], NC);
    }
    mbar_init(apb, NC);
    fence_mbar_init();
  }
  // query rows >= R of both Q slots stay zero for the whole kernel
  for (int i = threadIdx.x; i < 2 * C::ROWS * (D / 8); i += C::THREADS) {
    const int row = i / (D / 8), c = i - row * (D / 8);
    if ((row % C::ROWS) >= p.R * p.pack) *reinterpret_cast<uint4*>(qbuf + row * C::QSTR + c * 16) = make_uint4(0, 0, 0, 0);
  }
  trace_stamp(p, 0);
  if (warp == NC && lane == 0) {  // descriptor fetches overlap the grid-dependency wait
    prefetch_tmap(&tm.k_full);
    prefetch_tmap(&tm.v_full);
    prefetch_tmap(&tm.k_part);
    prefetch_tmap(&tm.v_part);
  }
  if (p.pdl_early) pdl_trigger();  // else the dependent launch waits for this grid's exit
  // MD_ATTN_EARLY_KV: kv_len and the rows of the first tiles are final (header contract), so the
  // producer issues up to NSTAGE tiles of its first unit -- never one holding a new row, never Q --
  // before the grid-dependency wait: they stream while the previous kernel's last CTAs finish
  int pre_issued = 0;
  // early-KV calls also stage the kv_len of the CTA's sequences in shared memory (the prefix-table
  // space, unused by the unit-aligned walk) before the wait: the walkers then need no global load
  // after the release (griddepcontrol.wait makes the L1 reload it: ~2 us under a saturated fabric),
  // and the producer issues the first group's Q loads as its first action after the release
  const bool stashed = EARLY && MD_DIRECT_UNITS && p.unit_aligned && p.early_kv;
  // this CTA's units of the unit-aligned plan, [cu0, cu1) = [c U / G, (c + 1) U / G), in 32-bit
  // unsigned arithmetic (c < G and U <= MAX_UNITS = 2^16: the products stay below 2^32) -- computed
  // once, before the grid-dependency wait (64-bit divisions cost ~0.1 us each on the start-up path)
  const unsigned cu0 = (unsigned)blockIdx.x * (unsigned)(p.B * p.Hkv) / gridDim.x;
  const unsigned cu1 = ((unsigned)blockIdx.x + 1u) * (unsigned)(p.B * p.Hkv) / gridDim.x;
  const int stash_b0 = (int)cu0 / p.Hkv;
  int q0_unit = -1, q0_ng = 0;  // producer lane 0: the first group, whose Q loads go out right after the wait
  Seg pf_s0{};                  // (MD_EPF_AFTER: the prefetch walk starts after the wait)
  SegWalker pf_w0{};
  if (stashed) {
    if (warp == NC) {
      const int u0 = (int)cu0, u1 = (int)cu1;
      const int nb = u1 > u0 ? (u1 - 1) / p.Hkv - stash_b0 + 1 : 0;
      for (int i = lane; i < nb; i += 32) pre[i] = __ldg(p.kv_len + stash_b0 + i);
    }
    if (threadIdx.x == 0) {  // the unit-aligned direct plan
      Plan d{};
      d.G = d.nch = gridDim.x;
      *plan_smem = d;
    }
    __syncthreads();  // the barrier initialisation, the plan and the stash are visible to every warp
    if (warp == NC) {
      SegWalker w0;
      w0.init_units((int)cu0, (int)cu1, pre, stash_b0);
      Seg s0;
      if (w0.next(p, pre, s0)) {
        q0_unit = s0.unit;
        q0_ng = p.pack > 1 ? (int)min((int64_t)p.pack, 1 + w0.end - w0.t) : 1;
        int it0 = 0;
        pre_issued = produce_segment<D, NSTAGE>(p, tm, seg_ranges(p, s0), s0.b, s0.kvh, smem, full, empty, it0,
                                                policy_evict_first(), s0.n, nullptr, 0, NSTAGE, true);
        // the next MD_EARLY_PF tiles into L2 while the previous call's tail leaves bandwidth idle
        if (!MD_EPF_AFTER && MD_EARLY_PF > 0 && lane == 0 && p.mode == MODE_DRAFT)
          early_l2_prefetch<D>(p, tm, pre, s0, w0, pre_issued);
        pf_s0 = s0;
        pf_w0 = w0;
      }
    }
  }
  pdl_wait();  // kv_len, the cache and q may come from the previous kernel
  trace_stamp(p, 1);
  if (stashed && warp == NC && lane == 0 && q0_ng > 0) {  // the first group's Q rows into slot 0
    mbar_arrive_expect_tx(&qfull[0], q0_ng * p.R * D * 2);
    for (int j = 0; j < q0_ng * p.R; ++j)
      bulk_load(qbuf + j * C::QSTR, p.q + group_row(p, q0_unit, j) * D, D * 2, &qfull[0]);
    if (p.trace != nullptr) trace_put(p, 14, globaltimer());
    if (MD_EPF_AFTER && MD_EARLY_PF > 0 && p.mode == MODE_DRAFT) early_l2_prefetch<D>(p, tm, pre, pf_s0, pf_w0, pre_issued);
  }
  // Unit-aligned plan (draft calls): CTA c owns the whole units [c*U/G, (c+1)*U/G), G = gridDim.x,
  // so it needs neither the per-sequence prefix table nor a plan -- its producer issues the
  // first tile right after reading its first unit's kv_len (MD_DIRECT_UNITS; the prefix walk
  // costs a batch-wide kv_len load, a scan and two CTA barriers before the first TMA issue)
  const bool direct = MD_DIRECT_UNITS && p.unit_aligned;
  if (direct) {
    if (threadIdx.x == 0 && !stashed) {  // (early-KV calls wrote it before the prologue's barrier)
      Plan d{};
      d.G = d.nch = gridDim.x;
      *plan_smem = d;
    }
  } else {
    __syncthreads();
    build_prefix(p, pre);
    // the plan lives in shared memory (read only at segment boundaries: keeps registers free)
    if (threadIdx.x == 0) *plan_smem = make_plan(p, total_tiles(p, pre), gridDim.x);
  }
  // early-KV calls need no CTA barrier after the release: the barriers, the plan and the kv_len
  // stash were published by the prologue's __syncthreads, so every warp starts its first
  // post-release loads (producer: Q; consumers: the fused append's new rows) at once
  if (!stashed) __syncthreads();
  const Plan& pl = *plan_smem;
  if ((int)blockIdx.x >= pl.G) return;  // uniform across the CTA
  int chunk = blockIdx.x;                // this CTA's static chunk, then claimed dynamic ones
  const int U = p.B * p.Hkv;
  auto init_walk = [&](SegWalker& w) {
    if (direct) {
      // (chunk == blockIdx.x and pl.G == gridDim.x in the unit-aligned plan: no dynamic chunks)
      w.init_units((int)cu0, (int)cu1, stashed ? pre : nullptr,
                   stash_b0);
    } else {
      int64_t S0, E0;
      cta_range(p, pre, pl, chunk, S0, E0);
      w.init(p, pre, S0, E0);
    }
  };
  SegWalker walk;
  init_walk(walk);
  Seg sg;
  trace_stamp(p, 2);
  if (p.kn != nullptr && !p.unit_dyn && warp < NC) {  // fused append: the new rows of this CTA's tiles
    SegWalker aw;
    init_walk(aw);
    append_own_rows<D>(p, pre, aw, threadIdx.x, NC * 32);
    __syncwarp();
    if (lane == 0) mbar_arrive(apb);
    trace_stamp(p, 12);
  }

  if (warp == NC) {
    // ============================== TMA producer warp ==============================
    if (lane == 0) {
      prefetch_tmap(&tm.k_full);
      prefetch_tmap(&tm.v_full);
      prefetch_tmap(&tm.k_part);
      prefetch_tmap(&tm.v_part);
    }
    const uint64_t pol = policy_evict_first();
    int it = 0, qi = 0, ck = 0;
    // Dynamic chunks are claimed one ahead (the atomic's latency hides behind a whole chunk
    // of TMA issue); when the current chunk is exhausted the claimed id (-1: none left) is
    // handed to the consumers.
    // The dynamic-unit plan claims only when the walker runs dry (the ring's buffered stages hide
    // the atomic), so a unit goes to whichever CTA frees up first.
    int ahead = 0;
    if (pl.nch > pl.G && lane == 0 && !p.unit_dyn) ahead = atomicAdd(p.dyn, 1);
    auto next_seg = [&]() -> bool {
      while (!walk.next(p, pre, sg)) {
        if (pl.nch == pl.G) return false;
        int nxt = -1;
        if (lane == 0) {
          if (p.unit_dyn) ahead = atomicAdd(p.dyn, 1);
          const int c = pl.G + ahead;
          nxt = c < pl.nch ? c : -1;
          if (nxt >= 0 && !p.unit_dyn) ahead = atomicAdd(p.dyn, 1);
          const int cs = ck & 1;
          mbar_wait(&cempty[cs], ((ck >> 1) & 1) ^ 1);
          cids[cs] = nxt;
          mbar_arrive(&cfull[cs]);
        }
        nxt = __shfl_sync(0xffffffffu, nxt, 0);
        ++ck;
        if (nxt < 0) return false;
        chunk = nxt;
        {
          int64_t S_, E_;
          cta_range(p, pre, pl, chunk, S_, E_);
          walk.init(p, pre, S_, E_);
        }
      }
      return true;
    };
    while (next_seg()) {
      // this group's query rows: row s*R + r of unit gu0 + s = (t = r / g, head = kvh*g + r % g);
      // a group is one unit unless the call packs units (p.pack > 1: consecutive whole units, each
      // with >= 1 key by the header's preconditions)
      const int gu0 = sg.unit;
      const int ng = p.pack > 1 ? (int)min((int64_t)p.pack, 1 + walk.end - walk.t) : 1;
      if (lane == 0 && !(qi == 0 && q0_ng > 0)) {  // (the first group's Q went out right after the wait)
        const int qs = qi & 1;
        mbar_wait(&qempty[qs], ((qi >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qfull[qs], ng * p.R * D * 2);
        for (int j = 0; j < ng * p.R; ++j)
          bulk_load(qbuf + (qs * C::ROWS + j) * C::QSTR, p.q + group_row(p, gu0, j) * D, D * 2, &qfull[qs]);
        if (qi == 0 && p.trace != nullptr) trace_put(p, 14, globaltimer());
      }
      __syncwarp();
      for (int su = 0; su < ng; ++su) {
        if (su > 0) walk.next(p, pre, sg);
        produce_segment<D, NSTAGE>(p, tm, seg_ranges(p, sg), sg.b, sg.kvh, smem, full, empty, it, pol, sg.n,
                                   (p.kn != nullptr && !p.unit_dyn) ? apb : nullptr,
                                   (qi == 0 && su == 0) ? pre_issued : 0);
      }
      ++qi;
    }
    if (lane == 0) trace_put(p, 10, globaltimer());
    return;
  }
  // ============================== consumers ==============================
  const int ks = warp;
  const int gq = lane >> 2, cq = lane & 3;  // fragment row group / column quad
  const uint32_t ring = smem_u32(smem);
  const uint32_t qring = smem_u32(qbuf);
  int it = 0, qi = 0, ck = 0;
  unsigned long long qi_seg = 0;
  auto next_seg = [&]() -> bool {  // mirrors the producer's chunk sequence
    while (!walk.next(p, pre, sg)) {
      if (pl.nch == pl.G) return false;
      const int cs = ck & 1;
      mbar_wait(&cfull[cs], (ck >> 1) & 1);
      const int nxt = cids[cs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty[cs]);
      ++ck;
      if (nxt < 0) return false;
      chunk = nxt;
      {
        int64_t S_, E_;
        cta_range(p, pre, pl, chunk, S_, E_);
        walk.init(p, pre, S_, E_);
      }
    }
    return true;
  };
  while (next_seg()) {
#if MD_EXP_FMA
    if (D == 128 && p.R <= 4 && p.mode == MODE_DRAFT) {
      fma_segment<D, C>(p, pl, sg, chunk, ring, qbuf, obuf, mlbuf, lsebuf, full, empty, qfull, qempty, flag, it, qi);
      continue;
    }
#endif
    // a group of ng consecutive whole units (unit packing, p.pack > 1; mirrors the producer) or one segment
    const int gu0 = sg.unit;
    const int ng = p.pack > 1 ? (int)min((int64_t)p.pack, 1 + walk.end - walk.t) : 1;
    // Q^T fragments (B operand): qb[kk][0..1] = Q[gq][kk*16 + 2cq (+8) ..]
    uint32_t qb[MD16][2];
    {
      const int qs = qi & 1;
      mbar_wait(&qfull[qs], (qi >> 1) & 1);
      if (qi == 0) trace_stamp(p, 13);
      const uint32_t qrow = qring + (qs * C::ROWS + (lane & 7)) * C::QSTR + (lane >> 3) * 16;
#pragma unroll
      for (int kk = 0; kk < MD16; kk += 2) ldsm_x4(qrow + kk * 32, qb[kk][0], qb[kk][1], qb[kk + 1][0], qb[kk + 1][1]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
      ++qi;
    }

    float o[MD16][4];
#pragma unroll
    for (int i = 0; i < MD16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};

#pragma unroll 1
    for (int su = 0; su < ng; ++su) {
    if (su > 0) walk.next(p, pre, sg);
    const int n = sg.n;
    const Ranges rg = seg_ranges(p, sg);
    // new-key visibility of the two rows 2cq, 2cq+1 this thread holds (verify; rows past R
    // take the mask of row R-1, their output is dropped)
    const int vbase = (p.mode == MODE_VERIFY) ? n - p.T : 0x7fffffff;
    uint32_t msk[2] = {~0u, ~0u};
    if (p.mode == MODE_VERIFY) {
#pragma unroll
      for (int j = 0; j < 2; ++j) msk[j] = node_mask(p, sg.b, 2 * cq + j);
    }
    // packed group: rows 2cq, 2cq+1 take part in this unit's tiles only if they are its rows,
    // [su R, su R + R) (no division: this runs at every sub-unit start)
    bool act[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) act[j] = p.pack == 1 || (unsigned)(2 * cq + j - su * p.R) < (unsigned)p.R;
    const bool packed = p.pack > 1;

#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
#pragma unroll 1
      for (int pos = rs; pos < re; pos += TK, ++it) {
        const int stage = it % NSTAGE;
        mbar_wait(&full[stage], (it / NSTAGE) & 1);
        if (it == 0) trace_stamp(p, 3);
        const int nvalid = min(TK, re - pos);
        const int kw0 = ks * KW;
        if (!MD_EXP_NOMATH && kw0 < nvalid) {
          const uint32_t kt = ring + stage * C::STAGE;
          const uint32_t vt = kt + C::TILE;
          // ---------------- S^T = K Q^T : KB blocks of 16 keys x 8 query rows
          float s[KB][4];
#pragma unroll
          for (int kb = 0; kb < KB; ++kb) s[kb][0] = s[kb][1] = s[kb][2] = s[kb][3] = 0.f;
#pragma unroll
          for (int kk = 0; kk < MD16; ++kk) {
            const int chunk = kk * 2 + (lane >> 4);
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              const int key = kw0 + kb * 16 + (lane & 15);
              uint32_t a[4];
              ldsm_x4(kt + (chunk >> 3) * (TK * 128) + swz128(key, chunk & 7), a[0], a[1], a[2], a[3]);
              mma_bf16_16816(s[kb], a, qb[kk][0], qb[kk][1]);
            }
          }
          // ---------------- scale, mask, online softmax (log2 domain); rows 2cq, 2cq+1
          const bool need_mask = packed || (kw0 + KW > nvalid) || (pos + kw0 + KW - 1 >= vbase);
          float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
          for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float v = s[kb][e] * p.scale_log2;
              if (need_mask) {
                const int ko = kw0 + kb * 16 + gq + ((e >> 1) << 3);
                v = (!act[e & 1] || ko >= nvalid || key_hidden(msk[e & 1], pos + ko - vbase)) ? -INFINITY : v;
              }
              s[kb][e] = v;
              mx[e & 1] = fmaxf(mx[e & 1], v);
            }
          float corr[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 4));
            mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 8));
            mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 16));
            const float mn = fmaxf(m[j], mx[j]);
            const float base = (mn == -INFINITY) ? 0.f : mn;
            // (an unchanged maximum, also -inf: the row has seen no key yet, gives exactly 1)
            corr[j] = (mn == m[j]) ? 1.f : ex2(m[j] - base);
            m[j] = mn;
            float rsum = 0.f;
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              s[kb][j] = ex2(s[kb][j] - base);
              s[kb][j + 2] = ex2(s[kb][j + 2] - base);
              rsum += s[kb][j] + s[kb][j + 2];
            }
            l[j] = l[j] * corr[j] + rsum;
          }
          if (__any_sync(0xffffffffu, corr[0] != 1.f || corr[1] != 1.f)) {
#pragma unroll
            for (int i = 0; i < MD16; ++i) {
              o[i][0] *= corr[0];
              o[i][1] *= corr[1];
              o[i][2] *= corr[0];
              o[i][3] *= corr[1];
            }
          }
          // ---------------- O^T += V^T P^T
          const bool sanitize = kw0 + KW > nvalid;
#pragma unroll
          for (int kb = 0; kb < KB; ++kb) {
            // P^T B fragments: transpose the bf16-packed S^T fragments (keys gq/gq+8 x rows 2cq..)
            const uint32_t pb0 = movmatrix_t(pack_bf16(s[kb][0], s[kb][1]));
            const uint32_t pb1 = movmatrix_t(pack_bf16(s[kb][2], s[kb][3]));
            const int key = kw0 + kb * 16 + (lane & 7) + ((lane >> 4) << 3);
            const int kf = kw0 + kb * 16 + cq * 2;  // keys this thread's A fragments hold
            const uint32_t m_lo = (kf < nvalid ? 0x0000ffffu : 0u) | (kf + 1 < nvalid ? 0xffff0000u : 0u);
            const uint32_t m_hi = (kf + 8 < nvalid ? 0x0000ffffu : 0u) | (kf + 9 < nvalid ? 0xffff0000u : 0u);
#pragma unroll
            for (int i = 0; i < MD16; ++i) {
              const int chunk = i * 2 + ((lane >> 3) & 1);
              uint32_t a[4];
              ldsm_x4_t(vt + (chunk >> 3) * (TK * 128) + swz128(key, chunk & 7), a[0], a[1], a[2], a[3]);
              if (sanitize) {  // rows past the valid keys may hold non-finite bits: zero them
                a[0] &= m_lo;
                a[1] &= m_lo;
                a[2] &= m_hi;
                a[3] &= m_hi;
              }
              mma_bf16_16816(o[i], a, pb0, pb1);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      }
    }
    }  // sub-units of the group

    // ============================== segment epilogue ==============================
    trace_stamp(p, 4);
    // full row sums: reduce over the 8 lanes sharing cq (they hold different keys)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      l[j] += __shfl_xor_sync(0xffffffffu, l[j], 4);
      l[j] += __shfl_xor_sync(0xffffffffu, l[j], 8);
      l[j] += __shfl_xor_sync(0xffffffffu, l[j], 16);
    }
    if (gq == 0) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        mlbuf[(warp * C::ROWS + 2 * cq + j) * 2 + 0] = m[j];
        mlbuf[(warp * C::ROWS + 2 * cq + j) * 2 + 1] = l[j];
      }
    }
    named_bar_sync(1, NC * 32);
    // scale this warp's O^T by 2^(m_w - M) / L where (M, L) combine the KS key slices
    {
      float f[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int rl = 2 * cq + j;
        float M = -INFINITY;
#pragma unroll
        for (int k = 0; k < KS; ++k) M = fmaxf(M, mlbuf[(k * C::ROWS + rl) * 2]);
        float L = 0.f;
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          const float* e = &mlbuf[(k * C::ROWS + rl) * 2];
          if (e[1] > 0.f) L += e[1] * ex2(e[0] - M);
        }
        f[j] = (l[j] > 0.f) ? ex2(m[j] - M) / L : 0.f;
        if (ks == 0 && gq == 0) lsebuf[rl] = (L > 0.f) ? M + __log2f(L) : -INFINITY;
      }
#pragma unroll
      for (int i = 0; i < MD16; ++i) {
        o[i][0] *= f[0];
        o[i][1] *= f[1];
        o[i][2] *= f[0];
        o[i][3] *= f[1];
      }
    }
    // Sum the KS = 4 slices: warps 2, 3 park their fragments (every warp holds the same
    // fragment layout, so lane t adds lane t's values: conflict-free), warps 0, 1 add them
    // and write their sums as two row-major [8][D] planes over the same buffer (column
    // XOR-swizzled by (r >> 1) << 3: conflict-free), then all warps add the planes and store
    // whole rows with 16-byte vectors.
    if (warp >= 2) {
      float* ob = obuf + (warp - 2) * FRAG;
#pragma unroll
      for (int i = 0; i < MD16; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) ob[(i * 4 + e) * 32 + lane] = o[i][e];
    }
    named_bar_sync(1, NC * 32);
    if (warp < 2) {
      float* ob = obuf + warp * FRAG;  // FRAG == 8 * D: one plane
#pragma unroll
      for (int i = 0; i < MD16; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[i][e] += ob[(i * 4 + e) * 32 + lane];
      __syncwarp();
#pragma unroll
      for (int i = 0; i < MD16; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 2 * cq + (e & 1), dd = i * 16 + gq + ((e >> 1) << 3);
          ob[r * D + (dd ^ (cq << 3))] = o[i][e];
        }
    }
    named_bar_sync(1, NC * 32);
    trace_stamp(p, 7);
    // rows r < R -> the final output, or this CTA's partial slot
    const bool complete = sg.complete();
    const int slot_base = complete ? 0 : seg_slot(p, pl, sg, chunk);  // (a 64-bit division: split segments only)
    {
      constexpr int V4 = D / 4;
      for (int idx = threadIdx.x; idx < ng * p.R * V4; idx += NC * 32) {
        const int r = idx / V4, c4 = (idx - r * V4) * 4;
        const int sc = c4 ^ (((r >> 1) & 3) << 3);
        const float4 a = *reinterpret_cast<const float4*>(obuf + r * D + sc);
        const float4 c = *reinterpret_cast<const float4*>(obuf + FRAG + r * D + sc);
        const float4 v = make_float4(a.x + c.x, a.y + c.y, a.z + c.z, a.w + c.w);
        if (MD_EXP_EPI == 1) {  // experiment: no output stores (bound of their cost)
          if (v.x == 12345.f) p.out[0] = v.y;
        } else if (MD_EXP_EPI != 4 && complete && p.T == 1 && p.out_peers == nullptr) {
          // drafts (T = 1, R = g): row rr of unit u is output row u * g + rr, so the group's rows are
          // the contiguous rows gu0 * g + r -- no integer divisions on the store path
          const int64_t orow = group_row(p, gu0, r);
          if (MD_EXP_EPI != 3) *reinterpret_cast<float4*>(p.out + orow * D + c4) = v;
          if (MD_EXP_EPI != 2 && c4 == 0 && p.lse != nullptr) p.lse[orow] = lsebuf[r] * LN2;
        } else if (complete) {
          // row r of the group = row r % R of unit gu0 + r / R (one unit: gu0 = sg.unit)
          const int su = r / p.R, rr = r - su * p.R;
          const int bb = (gu0 + su) / p.Hkv, hh = gu0 + su - bb * p.Hkv;
          if (MD_EXP_EPI != 3) store_out(p, o_row(p, bb, hh, rr) * D + c4, v);
          else if (v.x == 12345.f) p.out[0] = v.y;
          if (MD_EXP_EPI != 2 && c4 == 0 && p.lse != nullptr) p.lse[out_row(p, bb, hh, rr)] = lsebuf[r] * LN2;
        } else {
          const int64_t prow = (int64_t)slot_base * p.R + r;
          __stcg(reinterpret_cast<float4*>(p.ws_o + prow * D + c4), v);
          if (c4 == 0) __stcg(p.ws_lse + prow, lsebuf[r]);
        }
      }
    }
    trace_stamp(p, 8);
    if (!complete) finish_unit<D>(p, sg, pl, NC * 32, flag);
    trace_stamp(p, 9);
    named_bar_sync(1, NC * 32);  // the epilogue buffers are reused by the next segment
    trace_stamp(p, 5);
    ++qi_seg;
    if (threadIdx.x == 0) trace_put(p, 11, qi_seg);
  }
  // the last CTA to finish re-arms the dynamic counters for the next call (every CTA's
  // producer has made its final claim before its consumers saw the -1 hand-off)
  if (pl.nch > pl.G && threadIdx.x == 0) {
    if (atomicAdd(p.dyn + 1, 1) == pl.G - 1) {
      p.dyn[0] = 0;
      p.dyn[1] = 0;
    }
  }
}

#include "attn_tc.cuh"

// ------------------------------------------------------------------------------ host side
constexpr int ROWS_CTAS_PER_SM = 2;
constexpr int KEYS_CTAS_PER_SM = 2;  // keys kernel: 2 CTAs / SM (1 CTA with a deeper ring measured slower)

static bool use_keys_kernel(int R) { return R <= 8; }

// tcgen05 verify kernel for every R = g*T > 8 at head_dim 128 (the mma.sync rows kernel serves
// head_dim 64 with R > 8)
static bool use_tc_kernel(int R, int D, int mode) { return D == 128 && mode == 0 /*MODE_VERIFY*/ && R > 8; }

// Persistent stream-K grid: the resident CTAs of one wave.
static int grid_for(int R, int sm_count, bool tc = false) {
  if (tc) return sm_count;
  return sm_count * (use_keys_kernel(R) ? KEYS_CTAS_PER_SM : ROWS_CTAS_PER_SM);
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Dynamic tail of the keys kernel (long calls only, see make_plan): the first DYN_STATIC_PERMILLE
// of the tile space is split statically, the rest into DYN_K chunks per CTA claimed at run time.
// Only the keys kernel: the rows kernel (HMMA-heavy consumers that fetch Q at each segment) and
// the tcgen05 kernel (every extra segment costs a Q load, an O^T epilogue and a split merge)
// measured slower with claimed chunks (Llama verify 1.23 -> 1.34 ms / 1.24 -> 1.30 ms).
// Compile-time constants: the library reads no environment variables.
constexpr int DYN_K = 4;
constexpr int DYN_MIN_TILES = 128;  // dynamic only when a call has >= 128 tiles (8 MB of K+V) per CTA
constexpr int DYN_STATIC_PERMILLE = 750;
#ifndef MD_TC_MORE_RR
#define MD_TC_MORE_RR 1  // compile-time row counts for the paper's gammas (0: A/B builds, faster compile)
#endif
#ifndef MD_DRAFT_DYN_UNITS
#define MD_DRAFT_DYN_UNITS 0  // StreamingLLM draft calls: dynamic whole-unit claims (A/B)
#endif
#ifndef MD_UNIT_ALIGNED_DRAFT
#define MD_UNIT_ALIGNED_DRAFT 1  // draft calls: whole units per CTA (0: the stream-K plan; A/B builds only)
#endif
static int dyn_k_for(int R) { return use_keys_kernel(R) ? DYN_K : 0; }

// [counters int32: 2 dynamic-chunk counters + MAX_UNITS unit counters][partials fp32 C*2*R*D]
// [partial lse fp32 C*2*R], C = G*(1+dyn_k) chunks (G static + at most G*dyn_k dynamic).
// The counters sit at a fixed offset with a fixed capacity, so calls of ANY shape can share
// one workspace: no call's partials ever overlap another call's counters.
constexpr int MAX_UNITS = 65536;  // B * Hkv
constexpr size_t COUNTER_BYTES = ((size_t)(MAX_UNITS + 2) * 4 + 255) & ~size_t(255);
// partial slots: two per work chunk of the stream-K plan (the mma.sync kernels' grid with its
// dynamic chunks, or the tcgen05 kernel's 1 CTA / SM, whichever is larger: the workspace query
// does not know which kernel will run), or, for the deterministic plan, one per piece
// (units * det_maxp)
static size_t partial_slots(int G, int units, int R, int det_maxp) {
  if (det_maxp > 0) return (size_t)units * det_maxp;
  return 2 * std::max((size_t)G * (1 + dyn_k_for(R)), (size_t)device_sm_count());
}
static size_t workspace_for(int G, int units, int R, int D, int det_maxp = 0) {
  const size_t C = partial_slots(G, units, R, det_maxp);
  const size_t X = use_keys_kernel(R) ? 0 : (size_t)G * XS_FRAGS * 16 * D * 4;  // rows-kernel scratch
  return COUNTER_BYTES + align256(C * R * D * 4) + align256(C * R * 4) + align256(X);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

static md_status make_tmap(CUtensorMap* m, const md_kv_cache* c, void* base, int box_rows) {
  auto enc = get_encode();
  MD_REQUIRE(enc != nullptr, MD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[4] = {(cuuint64_t)c->head_dim, (cuuint64_t)c->capacity, (cuuint64_t)c->num_kv_heads,
                        (cuuint64_t)c->batch};
  cuuint64_t strides[3] = {(cuuint64_t)c->stride_s * 2, (cuuint64_t)c->stride_h * 2, (cuuint64_t)c->stride_b * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MD_REQUIRE(r == CUDA_SUCCESS, MD_ERR_INVALID_ARG, "cuTensorMapEncodeTiled failed (code %d): check strides/alignment",
             (int)r);
  return MD_OK;
}

template <typename K>
static md_status set_smem(K kern, int bytes, int* done_dev) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (*done_dev != dev) {  // per-process; the attribute call is idempotent (benign race)
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
      return check_launch("cudaFuncSetAttribute");
    *done_dev = dev;
  }
  return MD_OK;
}

template <int D, int MT, int KS>
static md_status launch_rows(const TmapSet& tm, const AttnParams& p, int grid, cudaStream_t s) {
  auto kern = attn_rows_kernel<D, MT, KS>;
  constexpr int smem = RowsSmem<D>::TOTAL;
  static int done = -1;
  md_status st = set_smem(kern, smem, &done);
  if (st != MD_OK) return st;
  if (launch_pdl(kern, grid, (MT * KS + 1) * 32, smem, s, tm, p) != cudaSuccess) return check_launch("attn_rows_kernel");
  return check_launch("attn_rows_kernel");
}

template <int D, int KS, int CTAS>
static md_status launch_keys(const TmapSet& tm, const AttnParams& p, int grid, cudaStream_t s) {
  // early-KV calls run their own instantiation: the prologue that streams before the grid-dependency
  // wait is compiled out of every other call (its mere presence cost the plain draft ~0.5 us:
  // register allocation and scheduling of the whole kernel change with it)
  using C = KeysCfg<D, KS, CTAS>;
  auto kern = p.early_kv ? attn_keys_kernel<D, KS, CTAS, true> : attn_keys_kernel<D, KS, CTAS, false>;
  static int done[2] = {-1, -1};
  md_status st = set_smem(kern, C::SMEM, &done[p.early_kv ? 1 : 0]);
  if (st != MD_OK) return st;
  if (launch_pdl(kern, grid, C::THREADS, C::SMEM, s, tm, p) != cudaSuccess) return check_launch("attn_keys_kernel");
  return check_launch("attn_keys_kernel");
}

template <int NP, int RR>
static md_status launch_tc(const TmapSet& tm, const CUtensorMap& qm, const AttnParams& p, int grid, cudaStream_t s) {
  auto kern = tc::attn_tc_kernel<NP, RR>;
  constexpr int smem = tc::Cfg<NP>::SMEM;
  static int done = -1;
  md_status st = set_smem(kern, smem, &done);
  if (st != MD_OK) return st;
  if (launch_pdl(kern, grid, tc::Cfg<NP>::THREADS, smem, s, tm, qm, p) != cudaSuccess) return check_launch("attn_tc_kernel");
  return check_launch("attn_tc_kernel");
}

// Q [B][T][Hq][d] as a 4-D map (d, Hq, T, B) with a (64, g, T, 1) box: one box holds the R
// query rows of a (b, kv head) unit for one 64-column slab, in row order r = t * g + h.
static md_status make_qmap(CUtensorMap* m, const void* q, int B, int T, int Hq, int g, int d) {
  auto enc = get_encode();
  MD_REQUIRE(enc != nullptr, MD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)Hq, (cuuint64_t)T, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)Hq * d * 2, (cuuint64_t)T * Hq * d * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)g, (cuuint32_t)T, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(q), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MD_REQUIRE(r == CUDA_SUCCESS, MD_ERR_INVALID_ARG, "cuTensorMapEncodeTiled (q) failed (code %d)", (int)r);
  return MD_OK;
}

template <int D>
static md_status launch_dim(const TmapSet& tm, const AttnParams& p, int grid, cudaStream_t s) {
  if (use_keys_kernel(p.R))
    return launch_keys<D, 4, KEYS_CTAS_PER_SM>(tm, p, grid, s);
  switch ((p.R + 15) / 16) {
    case 1: return launch_rows<D, 1, 4>(tm, p, grid, s);
    case 2: return launch_rows<D, 2, 2>(tm, p, grid, s);
    case 3: return launch_rows<D, 3, 1>(tm, p, grid, s);
    case 4: return launch_rows<D, 4, 1>(tm, p, grid, s);
    default: return fail(MD_ERR_UNSUPPORTED, "g*T > 64 query rows per KV head is not supported");
  }
}

static md_status check_cache(const md_kv_cache* c, const char* who) {
  MD_REQUIRE(c != nullptr && c->k != nullptr && c->v != nullptr, MD_ERR_INVALID_ARG, "%s: NULL cache", who);
  MD_REQUIRE(c->batch >= 1 && c->num_kv_heads >= 1 && c->capacity >= 1, MD_ERR_INVALID_ARG,
             "%s: batch, num_kv_heads, capacity must be >= 1", who);
  MD_REQUIRE(c->head_dim == 64 || c->head_dim == 128, MD_ERR_UNSUPPORTED, "%s: head_dim must be 64 or 128", who);
  MD_REQUIRE(c->stride_s % 8 == 0 && c->stride_h % 8 == 0 && c->stride_b % 8 == 0 && c->stride_s >= c->head_dim,
             MD_ERR_INVALID_ARG, "%s: strides must be multiples of 8 elements and stride_s >= head_dim", who);
  MD_REQUIRE(aligned16(c->k) && aligned16(c->v), MD_ERR_INVALID_ARG, "%s: cache must be 16-byte aligned", who);
  return MD_OK;
}

// md_debug_trace: per calling thread (diagnostics only; thread_local keeps calls reentrant)
static thread_local unsigned long long* g_trace = nullptr;
static thread_local size_t g_trace_bytes = 0;

struct IndexedArgs {
  const int32_t* idx = nullptr;
  int idx_stride = 0;
  const int32_t* idx_count = nullptr;
  const int32_t* tail_start = nullptr;
  const uint32_t* tree_mask = nullptr;  // verify only
  const md_tp_out* tp = nullptr;        // f1: outputs stored into every TP rank's full-head buffer
  const int32_t* windows = nullptr;     // draft: per-sequence windows
  const void* k_new = nullptr;          // fused append (md_*_append): [B][T][Hkv][d] rows for [n-T, n)
  const void* v_new = nullptr;
  int max_keys = 0;                     // fused append / det: upper bound of the keys per unit (plan choice)
  bool early_kv = false;                // MD_ATTN_EARLY_KV
  int det_split_tiles = 0;              // deterministic fixed-split plan (md_*_det): piece length in tiles
};

static md_status run_attention(const md_kv_cache* c, const void* q, int Hq, int T, const int32_t* kv_len, int sink,
                               int window, int mode, float scale, float* out, float* lse, void* ws, size_t ws_bytes,
                               cudaStream_t s, const char* who, const IndexedArgs& ix = IndexedArgs()) {
  md_status st = check_cache(c, who);
  if (st != MD_OK) return st;
  if (ix.tp != nullptr) {
    MD_REQUIRE(ix.tp->out_peers != nullptr && ix.tp->world >= 1 && ix.tp->rank >= 0 && ix.tp->rank < ix.tp->world &&
                   ix.tp->world <= 32,
               MD_ERR_INVALID_ARG, "%s: bad md_tp_out (need out_peers, 0 <= rank < world <= 32)", who);
  }
  MD_REQUIRE(q != nullptr && kv_len != nullptr && (out != nullptr || ix.tp != nullptr), MD_ERR_INVALID_ARG,
             "%s: NULL q/kv_len/out", who);
  MD_REQUIRE(Hq >= 1 && Hq % c->num_kv_heads == 0, MD_ERR_INVALID_ARG, "%s: num_q_heads must be a multiple of Hkv",
             who);
  MD_REQUIRE(aligned16(q) && aligned16(out), MD_ERR_INVALID_ARG, "%s: q and out must be 16-byte aligned", who);
  // (with tensor-parallel outputs `out` is NULL: every output row goes to ix.tp->out_peers)
  const int g = Hq / c->num_kv_heads;
  const int R = g * T;
  // the tcgen05 verify kernel (head_dim 128) takes up to 128 query rows per KV head; the
  // mma.sync kernels (head_dim 64 verify, drafts with g > 8) up to 64
  const int max_rows = use_tc_kernel(R, c->head_dim, mode) ? 128 : 64;
  MD_REQUIRE(R <= max_rows, MD_ERR_UNSUPPORTED, "%s: g*T = %d > %d query rows per KV head is not supported", who, R,
             max_rows);
  const int units = c->batch * c->num_kv_heads;
  MD_REQUIRE(units <= MAX_UNITS, MD_ERR_UNSUPPORTED, "%s: batch * num_kv_heads = %d > %d is not supported", who,
             units, MAX_UNITS);
  const bool tcg = use_tc_kernel(R, c->head_dim, mode);
  int grid = grid_for(R, device_sm_count(), tcg);
  // Draft calls (short units: <= sink + window keys) run the unit-aligned plan on ceil(units / per)
  // CTAs, per = ceil(units / grid) whole units each: no split partials or merges.  Measured at the
  // target point (B = 64, 512 units of 1024 keys): 51.4 -> 49.1 us per call; Qwen2.5 (256 units of
  // 2048 keys): 50.7 -> 48.5 us (tools/draft_ab.py, profiles/draft_ab_r02.txt).  Not when the
  // keys kernel's dynamic tail engages (long calls), nor for the deterministic plan.
  bool unit_aligned = false, unit_dyn = false;
  if ((mode == MODE_DRAFT || mode == MODE_INDEXED) && !tcg && ix.det_split_tiles == 0 && MD_UNIT_ALIGNED_DRAFT) {
    const int64_t keys_ub = mode == MODE_DRAFT ? std::min<int64_t>((int64_t)sink + window, c->capacity) : c->capacity;
    const int64_t tiles_ub = (int64_t)c->batch * c->num_kv_heads * ((keys_ub + TK - 1) / TK);
    if (!(dyn_k_for(R) > 0 && tiles_ub >= (int64_t)DYN_MIN_TILES * grid)) {
      const int units_ = c->batch * c->num_kv_heads, per = (units_ + grid - 1) / grid;
#ifndef MD_EXP_UNIT_FULLGRID
#define MD_EXP_UNIT_FULLGRID 0  // experiment (A/B builds only): keep the full grid, boundaries snapped
#endif
      if (MD_DRAFT_DYN_UNITS && mode == MODE_DRAFT && use_keys_kernel(R) && c->batch <= TABLE_B) {
        grid = std::min(grid, units_);  // one unit per CTA, then claimed units
        unit_dyn = true;
      } else {
        if (!MD_EXP_UNIT_FULLGRID) grid = (units_ + per - 1) / per;
        unit_aligned = true;
      }
    }
  }
  const int det_maxp = ix.det_split_tiles > 0
                           ? (int)(((int64_t)(ix.max_keys + TK - 1) / TK + ix.det_split_tiles - 1) / ix.det_split_tiles)
                           : 0;
  const size_t need = workspace_for(grid, units, R, c->head_dim, det_maxp);
  MD_REQUIRE(ws != nullptr && ws_bytes >= need, MD_ERR_WORKSPACE, "%s: workspace of %zu bytes required, %zu given",
             who, need, ws_bytes);
  TmapSet tm;
  if ((st = make_tmap(&tm.k_full, c, c->k, TK)) != MD_OK || (st = make_tmap(&tm.v_full, c, c->v, TK)) != MD_OK ||
      (st = make_tmap(&tm.k_part, c, c->k, BOX_ROWS)) != MD_OK ||
      (st = make_tmap(&tm.v_part, c, c->v, BOX_ROWS)) != MD_OK)
    return st;
  if (mode == MODE_INDEXED) {
    MD_REQUIRE(R <= 8, MD_ERR_UNSUPPORTED, "%s: at most 8 query heads per KV head", who);
    MD_REQUIRE(c->stride_s % c->head_dim == 0 && c->stride_h % c->head_dim == 0 && c->stride_b % c->head_dim == 0,
               MD_ERR_UNSUPPORTED, "%s: cache strides must be multiples of head_dim for row gathers", who);
  }
  bool fuse_append = false;
  if (ix.k_new != nullptr) {
    MD_REQUIRE(ix.v_new != nullptr && aligned16(ix.k_new) && aligned16(ix.v_new), MD_ERR_INVALID_ARG,
               "%s: k_new / v_new must be non-NULL and 16-byte aligned", who);
    // the keys and tcgen05 kernels write the new rows themselves; the rows kernel (d = 64 verify,
    // MD_TC=0) gets the same rows from a kv_append launch ahead of it
    fuse_append = tcg || use_keys_kernel(R);
    // a long keys-kernel call (the MHA verify) runs the dynamic tail (make_plan), which the fused
    // append cannot serve (its rows are written per static range): keep the tail and enqueue the
    // append kernel ahead instead (decided on an upper bound of the tile count)
    const int64_t tiles_ub = (int64_t)c->batch * c->num_kv_heads * ((ix.max_keys + TK - 1) / TK);
    if (fuse_append && !tcg && dyn_k_for(R) > 0 && tiles_ub >= (int64_t)DYN_MIN_TILES * grid) fuse_append = false;
  }
  // host-side errors must be found before anything is enqueued: the separate append (when the
  // kernel cannot fuse it) is launched only once every check and tensor map has succeeded
  const bool separate_append = ix.k_new != nullptr && !fuse_append;
  AttnParams p{};
  p.q = static_cast<const uint16_t*>(q);
  if (fuse_append) {
    p.kn = static_cast<const uint16_t*>(ix.k_new);
    p.vn = static_cast<const uint16_t*>(ix.v_new);
    p.kw = static_cast<uint16_t*>(c->k);
    p.vw = static_cast<uint16_t*>(c->v);
  }
  p.c_sB = c->stride_b;
  p.c_sH = c->stride_h;
  p.c_sS = c->stride_s;
  p.out = out;
  p.lse = lse;
  p.kv_len = kv_len;
  p.B = c->batch;
  p.Hq = Hq;
  p.Hkv = c->num_kv_heads;
  p.T = T;
  p.g = g;
  p.R = R;
  p.sink = sink;
  p.window = window;
  p.mode = mode;
  p.scale_log2 = scale * LOG2E;
  p.idx = ix.idx;
  p.idx_stride = ix.idx_stride;
  p.idx_count = ix.idx_count;
  p.tail_start = ix.tail_start;
  p.tree_mask = ix.tree_mask;
  p.windows = ix.windows;
  p.out_peers = ix.tp ? ix.tp->out_peers : nullptr;
  p.tp_world = ix.tp ? ix.tp->world : 1;
  p.out_hq = ix.tp ? ix.tp->world * Hq : Hq;
  p.out_h0 = ix.tp ? ix.tp->rank * Hq : 0;
  p.trace = (g_trace != nullptr && g_trace_bytes >= (size_t)grid * TRACE_SLOTS * 8) ? g_trace : nullptr;
  p.kc = static_cast<const uint16_t*>(c->k);
  p.vc = static_cast<const uint16_t*>(c->v);
  p.row_sB = c->stride_b / c->head_dim;
  p.row_sH = c->stride_h / c->head_dim;
  p.row_sS = c->stride_s / c->head_dim;
  p.dyn_k = tcg ? 0 : dyn_k_for(R);  // dynamic tail: keys kernel only (make_plan)
  if (fuse_append) p.dyn_k = 0;  // the new rows are written per static range (append_own_rows)
  p.dyn_static_permille = DYN_STATIC_PERMILLE;
  p.dyn_min_tiles = DYN_MIN_TILES;
  p.det_split = ix.det_split_tiles;
  p.det_maxp = det_maxp;
  p.unit_aligned = unit_aligned ? 1 : 0;
  p.unit_dyn = unit_dyn ? 1 : 0;
  p.cap = c->capacity;
  p.early_kv = (ix.early_kv && unit_aligned && MD_DIRECT_UNITS && mode == MODE_DRAFT) ? 1 : 0;
  p.pack = (MD_PACK_UNITS && !MD_EXP_FMA && unit_aligned && MD_DIRECT_UNITS && use_keys_kernel(R) && R <= 4)
               ? 8 / R
               : 1;
  if (unit_aligned || unit_dyn) p.dyn_k = 0;
  if (p.det_split > 0) p.dyn_k = 0;
  const size_t slots = partial_slots(grid, units, R, det_maxp);
  uint8_t* w = static_cast<uint8_t*>(ws);
  p.dyn = reinterpret_cast<int*>(w);
  p.counters = p.dyn + 2;
  w += COUNTER_BYTES;
  p.ws_o = reinterpret_cast<float*>(w);
  w += align256(slots * R * c->head_dim * 4);
  p.ws_lse = reinterpret_cast<float*>(w);
  w += align256(slots * R * 4);
  p.ws_x = use_keys_kernel(R) ? nullptr : reinterpret_cast<float*>(w);
  p.pdl_early = 1;  // keys kernel: trigger the dependent launch at entry
  if (tcg) {
    // measured: an entry trigger lets the next kv_append pre-launch and costs ~29 us per
    // verify -> append boundary; triggering at exit makes the appends free (tools/step_probe.py)
    p.pdl_early = 0;
    CUtensorMap qm;
    if ((st = make_qmap(&qm, q, c->batch, T, Hq, g, c->head_dim)) != MD_OK) return st;
    if (separate_append && (st = launch_kv_append(c, ix.k_new, ix.v_new, T, kv_len, -T, s)) != MD_OK) return st;
    // the BASELINE shapes get a compile-time row count (Llama-3.1 g=4 x T=5, Qwen2.5 g=7 x T=5)
    st = (R == 20)   ? launch_tc<32, 20>(tm, qm, p, grid, s)
         : (R == 35) ? launch_tc<48, 35>(tm, qm, p, grid, s)
#if MD_TC_MORE_RR
         // the paper's other operating points: Llama-3.1-8B gamma 5 / 6 /
         // 7 / 8 / 11 (R = 24 / 28 / 32 / 36 / 48), Mistral-7B gamma 5 (24), Qwen2.5-7B gamma 3 / 5
         // (28 / 42): compile-time rows skip the padded columns' work (measured at 100k, B = 41:
         // R = 36 6.40 -> 6.81 TB/s, R = 48 6.20 -> 6.60; at 32k R = 24 6.76 -> 7.05;
         // profiles/rows_sweep_r02_compile_time_rows.txt)
         : (R == 24) ? launch_tc<32, 24>(tm, qm, p, grid, s)
         : (R == 28) ? launch_tc<32, 28>(tm, qm, p, grid, s)
         : (R == 32) ? launch_tc<32, 32>(tm, qm, p, grid, s)
         : (R == 36) ? launch_tc<48, 36>(tm, qm, p, grid, s)
         : (R == 42) ? launch_tc<48, 42>(tm, qm, p, grid, s)
         : (R == 48) ? launch_tc<48, 48>(tm, qm, p, grid, s)
#endif
         : (R <= 16) ? launch_tc<16, 0>(tm, qm, p, grid, s)
         : (R <= 32) ? launch_tc<32, 0>(tm, qm, p, grid, s)
         // 32 < R <= 64 (R != 35): two row groups (measured: R = 48 at 5.9 TB/s with one group of
         // 48 run-time rows, R = 49..64 at 6.5-6.8 TB/s with two groups; tools/rows_sweep.py)
         : (R <= 64) ? launch_tc<64, 0>(tm, qm, p, grid, s)
         : (R <= 96) ? launch_tc<96, 0>(tm, qm, p, grid, s)
                     : launch_tc<128, 0>(tm, qm, p, grid, s);
  } else {
    if (separate_append && (st = launch_kv_append(c, ix.k_new, ix.v_new, T, kv_len, -T, s)) != MD_OK) return st;
    st = (c->head_dim == 128) ? launch_dim<128>(tm, p, grid, s) : launch_dim<64>(tm, p, grid, s);
  }
  return st;
}

}  // namespace md

extern "C" size_t md_attn_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads, int32_t head_dim,
                                          int32_t T, int32_t max_kv_len) {
  using namespace md;
  if (batch < 1 || num_kv_heads < 1 || num_q_heads < 1 || num_q_heads % num_kv_heads || T < 1 || max_kv_len < 1 ||
      (head_dim != 64 && head_dim != 128))
    return 0;
  const int R = (num_q_heads / num_kv_heads) * T;
  return workspace_for(grid_for(R, device_sm_count()), batch * num_kv_heads, R, head_dim);
}

extern "C" md_status md_verify_attn_full(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                                         const int32_t* kv_len, int32_t max_kv_len, float scale, float* out,
                                         float* lse, void* workspace, size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(T >= 1 && T <= 16, MD_ERR_UNSUPPORTED, "md_verify_attn_full: T must be in [1, 16]");
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_verify_attn_full: NULL cache");
  MD_REQUIRE(max_kv_len >= T && max_kv_len <= cache->capacity, MD_ERR_INVALID_ARG,
             "md_verify_attn_full: need T <= max_kv_len <= capacity");
  return run_attention(cache, q, num_q_heads, T, kv_len, 0, 0, MODE_VERIFY, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_verify_attn_full");
}

extern "C" md_status md_verify_attn_tree(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                                         const int32_t* kv_len, int32_t max_kv_len, const uint32_t* tree_mask,
                                         float scale, float* out, float* lse, void* workspace, size_t workspace_bytes,
                                         md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(T >= 1 && T <= 16, MD_ERR_UNSUPPORTED, "md_verify_attn_tree: T must be in [1, 16]");
  MD_REQUIRE(cache != nullptr && tree_mask != nullptr, MD_ERR_INVALID_ARG, "md_verify_attn_tree: NULL cache/mask");
  MD_REQUIRE(max_kv_len >= T && max_kv_len <= cache->capacity, MD_ERR_INVALID_ARG,
             "md_verify_attn_tree: need T <= max_kv_len <= capacity");
  IndexedArgs ix;
  ix.tree_mask = tree_mask;
  return run_attention(cache, q, num_q_heads, T, kv_len, 0, 0, MODE_VERIFY, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_verify_attn_tree", ix);
}

extern "C" md_status md_draft_attn_sparse(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                          const int32_t* kv_len, int32_t sink, int32_t window, float scale,
                                          float* out, float* lse, void* workspace, size_t workspace_bytes,
                                          md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_draft_attn_sparse: NULL cache");
  MD_REQUIRE(sink >= 0 && window >= 0 && (int64_t)sink + window >= 1, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse: need sink >= 0, window >= 0, sink + window >= 1");
  return run_attention(cache, q, num_q_heads, 1, kv_len, sink, window, MODE_DRAFT, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_sparse");
}

extern "C" md_status md_draft_attn_sparse_windows(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                                  const int32_t* kv_len, int32_t sink, int32_t window,
                                                  const int32_t* windows, float scale, float* out, float* lse,
                                                  void* workspace, size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr && windows != nullptr, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_windows: NULL cache / windows");
  MD_REQUIRE(sink >= 0 && window >= 0 && (int64_t)sink + window >= 1, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_windows: need sink >= 0, window >= 0, sink + window >= 1");
  IndexedArgs ix;
  ix.windows = windows;
  return run_attention(cache, q, num_q_heads, 1, kv_len, sink, window, MODE_DRAFT, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_sparse_windows", ix);
}

extern "C" md_status md_draft_attn_indexed(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                           const int32_t* kv_len, const int32_t* idx, int32_t idx_stride,
                                           const int32_t* idx_count, const int32_t* tail_start, float scale,
                                           float* out, float* lse, void* workspace, size_t workspace_bytes,
                                           md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_draft_attn_indexed: NULL cache");
  MD_REQUIRE(idx != nullptr && idx_count != nullptr && tail_start != nullptr, MD_ERR_INVALID_ARG,
             "md_draft_attn_indexed: NULL idx / idx_count / tail_start");
  MD_REQUIRE(idx_stride >= 0 && idx_stride % 4 == 0 && aligned16(idx), MD_ERR_INVALID_ARG,
             "md_draft_attn_indexed: idx must be 16-byte aligned with idx_stride a multiple of 4");
  IndexedArgs ix;
  ix.idx = idx;
  ix.idx_stride = idx_stride;
  ix.idx_count = idx_count;
  ix.tail_start = tail_start;
  return run_attention(cache, q, num_q_heads, 1, kv_len, 0, 0, MODE_INDEXED, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_indexed", ix);
}

extern "C" md_status md_verify_attn_full_tp(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                                            const int32_t* kv_len, int32_t max_kv_len, float scale,
                                            const md_tp_out* tp, float* lse, void* workspace, size_t workspace_bytes,
                                            md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(T >= 1 && T <= 16, MD_ERR_UNSUPPORTED, "md_verify_attn_full_tp: T must be in [1, 16]");
  MD_REQUIRE(cache != nullptr && tp != nullptr, MD_ERR_INVALID_ARG, "md_verify_attn_full_tp: NULL cache / tp");
  MD_REQUIRE(max_kv_len >= T && max_kv_len <= cache->capacity, MD_ERR_INVALID_ARG,
             "md_verify_attn_full_tp: need T <= max_kv_len <= capacity");
  IndexedArgs ix;
  ix.tp = tp;
  return run_attention(cache, q, num_q_heads, T, kv_len, 0, 0, MODE_VERIFY, scale, nullptr, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_verify_attn_full_tp", ix);
}

extern "C" md_status md_draft_attn_sparse_tp(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                             const int32_t* kv_len, int32_t sink, int32_t window, float scale,
                                             const md_tp_out* tp, float* lse, void* workspace, size_t workspace_bytes,
                                             md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr && tp != nullptr, MD_ERR_INVALID_ARG, "md_draft_attn_sparse_tp: NULL cache / tp");
  MD_REQUIRE(sink >= 0 && window >= 0 && (int64_t)sink + window >= 1, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_tp: need sink >= 0, window >= 0, sink + window >= 1");
  IndexedArgs ix;
  ix.tp = tp;
  return run_attention(cache, q, num_q_heads, 1, kv_len, sink, window, MODE_DRAFT, scale, nullptr, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_sparse_tp", ix);
}

extern "C" md_status md_verify_attn_full_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                                int32_t T, const void* k_new, const void* v_new,
                                                const int32_t* kv_len, int32_t max_kv_len, float scale, float* out,
                                                float* lse, void* workspace, size_t workspace_bytes,
                                                md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(T >= 1 && T <= 16, MD_ERR_UNSUPPORTED, "md_verify_attn_full_append: T must be in [1, 16]");
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_verify_attn_full_append: NULL cache");
  MD_REQUIRE(k_new != nullptr && v_new != nullptr, MD_ERR_INVALID_ARG, "md_verify_attn_full_append: NULL k_new/v_new");
  MD_REQUIRE(max_kv_len >= T && max_kv_len <= cache->capacity, MD_ERR_INVALID_ARG,
             "md_verify_attn_full_append: need T <= max_kv_len <= capacity");
  IndexedArgs ix;
  ix.k_new = k_new;
  ix.v_new = v_new;
  ix.max_keys = max_kv_len;
  return run_attention(cache, q, num_q_heads, T, kv_len, 0, 0, MODE_VERIFY, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_verify_attn_full_append", ix);
}

extern "C" md_status md_draft_attn_sparse_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                                 const void* k_new, const void* v_new, const int32_t* kv_len,
                                                 int32_t sink, int32_t window, float scale, float* out, float* lse,
                                                 void* workspace, size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_draft_attn_sparse_append: NULL cache");
  MD_REQUIRE(k_new != nullptr && v_new != nullptr, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_append: NULL k_new/v_new");
  MD_REQUIRE(sink >= 0 && window >= 1, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_append: need sink >= 0 and window >= 1 (the draft token attends to itself)");
  IndexedArgs ix;
  ix.k_new = k_new;
  ix.v_new = v_new;
  ix.max_keys = (int)std::min<int64_t>((int64_t)sink + window, cache->capacity);
  return run_attention(cache, q, num_q_heads, 1, kv_len, sink, window, MODE_DRAFT, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_sparse_append", ix);
}

extern "C" md_status md_draft_attn_sparse_append_ex(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                                    const void* k_new, const void* v_new, const int32_t* kv_len,
                                                    int32_t sink, int32_t window, float scale, float* out, float* lse,
                                                    void* workspace, size_t workspace_bytes, uint32_t flags,
                                                    md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_draft_attn_sparse_append_ex: NULL cache");
  MD_REQUIRE(k_new != nullptr && v_new != nullptr, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_append_ex: NULL k_new/v_new");
  MD_REQUIRE(sink >= 0 && window >= 1, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_append_ex: need sink >= 0 and window >= 1 (the draft token attends to itself)");
  MD_REQUIRE((flags & ~(uint32_t)MD_ATTN_EARLY_KV) == 0, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_append_ex: unknown flags 0x%x", (unsigned)flags);
  IndexedArgs ix;
  ix.k_new = k_new;
  ix.v_new = v_new;
  ix.max_keys = (int)std::min<int64_t>((int64_t)sink + window, cache->capacity);
  ix.early_kv = (flags & MD_ATTN_EARLY_KV) != 0;
  return run_attention(cache, q, num_q_heads, 1, kv_len, sink, window, MODE_DRAFT, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_sparse_append_ex", ix);
}

extern "C" md_status md_verify_attn_full_tp_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                                   int32_t T, const void* k_new, const void* v_new,
                                                   const int32_t* kv_len, int32_t max_kv_len, float scale,
                                                   const md_tp_out* tp, float* lse, void* workspace,
                                                   size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(T >= 1 && T <= 16, MD_ERR_UNSUPPORTED, "md_verify_attn_full_tp_append: T must be in [1, 16]");
  MD_REQUIRE(cache != nullptr && tp != nullptr, MD_ERR_INVALID_ARG, "md_verify_attn_full_tp_append: NULL cache / tp");
  MD_REQUIRE(k_new != nullptr && v_new != nullptr, MD_ERR_INVALID_ARG,
             "md_verify_attn_full_tp_append: NULL k_new/v_new");
  MD_REQUIRE(max_kv_len >= T && max_kv_len <= cache->capacity, MD_ERR_INVALID_ARG,
             "md_verify_attn_full_tp_append: need T <= max_kv_len <= capacity");
  IndexedArgs ix;
  ix.tp = tp;
  ix.k_new = k_new;
  ix.v_new = v_new;
  ix.max_keys = max_kv_len;
  return run_attention(cache, q, num_q_heads, T, kv_len, 0, 0, MODE_VERIFY, scale, nullptr, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_verify_attn_full_tp_append", ix);
}

extern "C" md_status md_draft_attn_sparse_tp_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                                    const void* k_new, const void* v_new, const int32_t* kv_len,
                                                    int32_t sink, int32_t window, float scale, const md_tp_out* tp,
                                                    float* lse, void* workspace, size_t workspace_bytes,
                                                    md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr && tp != nullptr, MD_ERR_INVALID_ARG, "md_draft_attn_sparse_tp_append: NULL cache / tp");
  MD_REQUIRE(k_new != nullptr && v_new != nullptr, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_tp_append: NULL k_new/v_new");
  MD_REQUIRE(sink >= 0 && window >= 1, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_tp_append: need sink >= 0 and window >= 1 (the draft token attends to itself)");
  IndexedArgs ix;
  ix.tp = tp;
  ix.k_new = k_new;
  ix.v_new = v_new;
  ix.max_keys = (int)std::min<int64_t>((int64_t)sink + window, cache->capacity);
  return run_attention(cache, q, num_q_heads, 1, kv_len, sink, window, MODE_DRAFT, scale, nullptr, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_sparse_tp_append", ix);
}

extern "C" md_status md_draft_attn_indexed_append(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                                  const void* k_new, const void* v_new, const int32_t* kv_len,
                                                  const int32_t* idx, int32_t idx_stride, const int32_t* idx_count,
                                                  const int32_t* tail_start, float scale, float* out, float* lse,
                                                  void* workspace, size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_draft_attn_indexed_append: NULL cache");
  MD_REQUIRE(k_new != nullptr && v_new != nullptr, MD_ERR_INVALID_ARG,
             "md_draft_attn_indexed_append: NULL k_new/v_new");
  MD_REQUIRE(idx != nullptr && idx_count != nullptr && tail_start != nullptr, MD_ERR_INVALID_ARG,
             "md_draft_attn_indexed_append: NULL idx / idx_count / tail_start");
  MD_REQUIRE(idx_stride >= 0 && idx_stride % 4 == 0 && aligned16(idx), MD_ERR_INVALID_ARG,
             "md_draft_attn_indexed_append: idx must be 16-byte aligned with idx_stride a multiple of 4");
  IndexedArgs ix;
  ix.idx = idx;
  ix.idx_stride = idx_stride;
  ix.idx_count = idx_count;
  ix.tail_start = tail_start;
  ix.k_new = k_new;
  ix.v_new = v_new;
  return run_attention(cache, q, num_q_heads, 1, kv_len, 0, 0, MODE_INDEXED, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_indexed_append", ix);
}

extern "C" size_t md_attn_workspace_bytes_det(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                                              int32_t head_dim, int32_t T, int32_t max_keys, int32_t split_keys) {
  using namespace md;
  if (batch < 1 || num_kv_heads < 1 || num_q_heads < 1 || num_q_heads % num_kv_heads || T < 1 || max_keys < 1 ||
      (head_dim != 64 && head_dim != 128) || split_keys < TK || split_keys % TK)
    return 0;
  const int R = (num_q_heads / num_kv_heads) * T;
  const int S = split_keys / TK;
  const int maxp = (int)(((int64_t)(max_keys + TK - 1) / TK + S - 1) / S);
  return workspace_for(grid_for(R, device_sm_count()), batch * num_kv_heads, R, head_dim, maxp);
}

extern "C" md_status md_verify_attn_full_det(const md_kv_cache* cache, const void* q, int32_t num_q_heads, int32_t T,
                                             const int32_t* kv_len, int32_t max_kv_len, int32_t split_keys,
                                             float scale, float* out, float* lse, void* workspace,
                                             size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(T >= 1 && T <= 16, MD_ERR_UNSUPPORTED, "md_verify_attn_full_det: T must be in [1, 16]");
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_verify_attn_full_det: NULL cache");
  MD_REQUIRE(max_kv_len >= T && max_kv_len <= cache->capacity, MD_ERR_INVALID_ARG,
             "md_verify_attn_full_det: need T <= max_kv_len <= capacity");
  MD_REQUIRE(split_keys >= TK && split_keys % TK == 0, MD_ERR_INVALID_ARG,
             "md_verify_attn_full_det: split_keys must be a positive multiple of 64");
  IndexedArgs ix;
  ix.det_split_tiles = split_keys / TK;
  ix.max_keys = max_kv_len;
  return run_attention(cache, q, num_q_heads, T, kv_len, 0, 0, MODE_VERIFY, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_verify_attn_full_det", ix);
}

extern "C" md_status md_draft_attn_sparse_det(const md_kv_cache* cache, const void* q, int32_t num_q_heads,
                                              const int32_t* kv_len, int32_t sink, int32_t window,
                                              int32_t split_keys, float scale, float* out, float* lse,
                                              void* workspace, size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(cache != nullptr, MD_ERR_INVALID_ARG, "md_draft_attn_sparse_det: NULL cache");
  MD_REQUIRE(sink >= 0 && window >= 0 && (int64_t)sink + window >= 1, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_det: need sink >= 0, window >= 0, sink + window >= 1");
  MD_REQUIRE(split_keys >= TK && split_keys % TK == 0, MD_ERR_INVALID_ARG,
             "md_draft_attn_sparse_det: split_keys must be a positive multiple of 64");
  IndexedArgs ix;
  ix.det_split_tiles = split_keys / TK;
  ix.max_keys = (int)std::min<int64_t>((int64_t)sink + window, cache->capacity);
  return run_attention(cache, q, num_q_heads, 1, kv_len, sink, window, MODE_DRAFT, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_draft_attn_sparse_det", ix);
}

extern "C" MD_API md_status md_debug_trace(void* buf, size_t bytes) {
  md::g_trace = static_cast<unsigned long long*>(buf);
  md::g_trace_bytes = bytes;
  return MD_OK;
}

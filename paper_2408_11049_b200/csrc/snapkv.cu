// snapkv.cu — md_snapkv_select: SnapKV static KV selection at prefill (
// P:1141 footnote "SnapKV ... average pooling with a kernel size of 5 and an observation
// window size of 32"; oracle/snapkv.py S1-S4).  Prefill-time, once per sequence (T_select
// = 0 during drafting, Eq.3); its output drives md_draft_attn_indexed.
//
// Per unit (b, kv head) with prompt length L and window w, the g*w window queries of the
// GQA group (rows r = i*g + h) score the prompt keys:
//   lse_kernel    pass 1: per (unit, 1024-key chunk) CTA, online (max, sum) of
//                 exp(scale q_r . k_j) over the row's causal keys [0, L-w+i] -> partials;
//   vote_kernel   pass 2: merges the chunk partials into lse_r, recomputes the scores of the
//                 prefix keys j < L-w and writes vote[j] = sum_r exp(s_rj - lse_r);
//   select_kernel per unit: pooled[j] = (vote[j-2] + .. + vote[j+2]) / 5 (zero padded),
//                 4-pass 8-bit radix select of the (budget - w)-th largest pooled value, then
//                 an ordered compaction (ties -> lower positions) into ascending positions.
// Scores use mma.sync m16n8k16 (rows on M, keys on N) with swizzled K tiles in shared memory.
#include <cuda.h>

#include <cmath>

#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "md_common.cuh"
#include "md_internal.h"
#include "tcgen05.cuh"

namespace md {
namespace snap {

constexpr int KT = 64;          // keys per smem tile
constexpr int CHUNK = 1024;     // keys per CTA
constexpr int WARPS = 8;
constexpr int THREADS = WARPS * 32;
constexpr float LOG2E = 1.4426950408889634f;

struct Params {
  const uint16_t* k;       // cache K
  int64_t sB, sH, sS;      // element strides
  const uint16_t* q;       // [B][w][Hq][D]
  const int32_t* L;        // [B] prompt lengths
  int B, Hq, Hkv, g, w, R; // R = g*w rows per unit
  int nchunks;             // chunks per unit (from max prompt length)
  float scale_log2;
  float* part;             // [units][nchunks][R][2] (m, l) in log2 domain
  float* vote;             // [units][maxL]
  float* pooled;           // [units][maxL]
  int maxL;
  int32_t* idx;            // [B][Hkv][idx_stride]
  int32_t* idx_count;      // [B]
  int idx_stride, keep;    // keep = budget - w
  const int32_t* budgets;  // [B] per-sequence budgets or nullptr
};

// cooperative swizzled load of KT keys x D (bf16) of one unit into smem (zero rows past nkeys)
template <int D>
__device__ __forceinline__ void load_ktile(const Params& p, int b, int h, int k0, int nkeys, uint8_t* dst) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < KT * CH; i += THREADS) {
    const int r = i / CH, c = i - r * CH;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < nkeys) v = __ldg(reinterpret_cast<const uint4*>(p.k + b * p.sB + h * p.sH + (int64_t)(k0 + r) * p.sS) + c);
    *reinterpret_cast<uint4*>(dst + (c >> 3) * (KT * 128) + swz128(r, c & 7)) = v;
  }
}

// the same tile with 16-byte cp.async (rows past nkeys are left as they are: every consumer
// masks or drops keys past the chunk); the caller commits / waits
template <int D>
__device__ __forceinline__ void load_ktile_async(const Params& p, int b, int h, int k0, int nkeys, uint8_t* dst) {
  constexpr int CH = D / 8;
  const uint32_t base = smem_u32(dst);
  for (int i = threadIdx.x; i < KT * CH; i += THREADS) {
    const int r = i / CH, c = i - r * CH;
    if (r < nkeys) {
      const void* src = reinterpret_cast<const uint4*>(p.k + b * p.sB + h * p.sH + (int64_t)(k0 + r) * p.sS) + c;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + (c >> 3) * (KT * 128) + swz128(r, c & 7)),
                   "l"(src)
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_le(int n) {
  if (n == 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
  else asm volatile("cp.async.wait_group 1;" ::: "memory");
}

// Q fragments of rows mt*16 + {gq, gq+8}: row r = i*g + hh -> q[b][i][h*g + hh]
template <int D>
__device__ __forceinline__ void load_q(const Params& p, int b, int h, int mt, uint32_t (&qa)[D / 16][4]) {
  const int lane = threadIdx.x & 31, gq = lane >> 2, cq = lane & 3;
  const int r0 = mt * 16 + gq, r1 = r0 + 8;
  const uint32_t* q0 =
      r0 < p.R ? reinterpret_cast<const uint32_t*>(p.q + ((int64_t)(b * p.w + r0 / p.g) * p.Hq + h * p.g + r0 % p.g) * D)
               : nullptr;
  const uint32_t* q1 =
      r1 < p.R ? reinterpret_cast<const uint32_t*>(p.q + ((int64_t)(b * p.w + r1 / p.g) * p.Hq + h * p.g + r1 % p.g) * D)
               : nullptr;
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const int c = kk * 8 + cq;
    qa[kk][0] = q0 ? __ldg(q0 + c) : 0u;
    qa[kk][1] = q1 ? __ldg(q1 + c) : 0u;
    qa[kk][2] = q0 ? __ldg(q0 + c + 4) : 0u;
    qa[kk][3] = q1 ? __ldg(q1 + c + 4) : 0u;
  }
}

// S (16 rows x 64 keys) of one warp for one smem tile, scaled to the log2 domain
template <int D>
__device__ __forceinline__ void tile_scores(const uint32_t (&qa)[D / 16][4], uint32_t kt, float (&s)[8][4],
                                            float scale_log2) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      const int row = np * 16 + ((lane >> 4) << 3) + (lane & 7);
      const int chunk = kk * 2 + ((lane >> 3) & 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(kt + (chunk >> 3) * (KT * 128) + swz128(row, chunk & 7), b0, b1, b2, b3);
      mma_bf16_16816(s[2 * np], qa[kk], b0, b1);
      mma_bf16_16816(s[2 * np + 1], qa[kk], b2, b3);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) s[i][e] *= scale_log2;
}

// pass 1: per (unit, chunk) partial (m, l) of every row over its causal keys in the chunk
template <int D>
__global__ void __launch_bounds__(THREADS) lse_kernel(const Params p) {
  __shared__ __align__(1024) uint8_t ktiles[2][KT * D * 2];  // double-buffered (cp.async)
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x / p.nchunks, chunk = blockIdx.x - unit * p.nchunks;
  const int b = unit / p.Hkv, h = unit - b * p.Hkv;
  const int L = __ldg(p.L + b);
  const int k_begin = chunk * CHUNK, k_end = min(L, k_begin + CHUNK);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, cq = lane & 3;
  const int MT = (p.R + 15) / 16;
  for (int mt0 = 0; mt0 < MT; mt0 += WARPS) {
    const int mt = mt0 + warp;
    uint32_t qa[D / 16][4];
    if (mt < MT) load_q<D>(p, b, h, mt, qa);
    // causal limit of the two rows: key j visible to window query i iff j <= L - w + i
    const int lim0 = L - p.w + min(mt * 16 + gq, p.R - 1) / p.g;
    const int lim1 = L - p.w + min(mt * 16 + gq + 8, p.R - 1) / p.g;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    __syncthreads();
    if (k_begin < k_end) load_ktile_async<D>(p, b, h, k_begin, min(KT, k_end - k_begin), ktiles[0]);
    int buf = 0;
    for (int k0 = k_begin; k0 < k_end; k0 += KT, buf ^= 1) {
      const bool more = k0 + KT < k_end;
      if (more) load_ktile_async<D>(p, b, h, k0 + KT, min(KT, k_end - k0 - KT), ktiles[buf ^ 1]);
      cp_async_wait_le(more ? 1 : 0);
      __syncthreads();
      if (mt < MT) {
      float s[8][4];
      tile_scores<D>(qa, smem_u32(ktiles[buf]), s, p.scale_log2);
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = k0 + i * 8 + cq * 2 + (e & 1);
          if (j >= k_end || j > ((e < 2) ? lim0 : lim1)) s[i][e] = -INFINITY;
          if (e < 2) mx0 = fmaxf(mx0, s[i][e]);
          else mx1 = fmaxf(mx1, s[i][e]);
        }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
      const float b0 = n0 == -INFINITY ? 0.f : n0, b1 = n1 == -INFINITY ? 0.f : n1;
      float r0 = 0.f, r1 = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        r0 += ex2(s[i][0] - b0) + ex2(s[i][1] - b0);
        r1 += ex2(s[i][2] - b1) + ex2(s[i][3] - b1);
      }
      l0 = l0 * ex2(m0 - b0) + r0;
      l1 = l1 * ex2(m1 - b1) + r1;
      m0 = n0;
      m1 = n1;
      }
      __syncthreads();  // every warp is done with this buffer before it is refilled
    }
    if (mt >= MT) continue;
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    if (cq == 0) {
      float* base = p.part + ((int64_t)unit * p.nchunks + chunk) * p.R * 2;
      const int r0 = mt * 16 + gq, r1 = r0 + 8;
      if (r0 < p.R) base[r0 * 2] = m0, base[r0 * 2 + 1] = l0;
      if (r1 < p.R) base[r1 * 2] = m1, base[r1 * 2 + 1] = l1;
    }
  }
}

// pass 2: lse per row from the chunk partials, then vote[j] = sum_r 2^(s_rj - lse_r), j < L - w
template <int D>
__global__ void __launch_bounds__(THREADS) vote_kernel(const Params p) {
  __shared__ __align__(1024) uint8_t ktiles[2][KT * D * 2];  // double-buffered (cp.async)
  __shared__ float lse_s[256];
  __shared__ float wsum[WARPS][KT];
  pdl_trigger();
  pdl_wait();  // the chunk partials come from lse_kernel
  const int unit = blockIdx.x / p.nchunks, chunk = blockIdx.x - unit * p.nchunks;
  const int b = unit / p.Hkv, h = unit - b * p.Hkv;
  const int L = __ldg(p.L + b);
  const int prefix = L - p.w;
  const int k_begin = chunk * CHUNK, k_end = min(prefix, k_begin + CHUNK);
  if (k_begin >= k_end) return;
  const int nch = (L + CHUNK - 1) / CHUNK;
  for (int r = threadIdx.x; r < p.R; r += THREADS) {
    const float* base = p.part + (int64_t)unit * p.nchunks * p.R * 2 + r * 2;
    float M = -INFINITY;
    for (int c = 0; c < nch; ++c) M = fmaxf(M, base[(int64_t)c * p.R * 2]);
    float S = 0.f;
    for (int c = 0; c < nch; ++c) {
      const float l = base[(int64_t)c * p.R * 2 + 1];
      if (l > 0.f) S += l * ex2(base[(int64_t)c * p.R * 2] - M);
    }
    lse_s[r] = M + __log2f(S);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, cq = lane & 3;
  const int MT = (p.R + 15) / 16;
  // this warp's Q fragments stay in registers when every row tile has its own warp
  uint32_t qown[D / 16][4];
  const bool own = MT <= WARPS;
  if (own && warp < MT) load_q<D>(p, b, h, warp, qown);
  __syncthreads();  // lse_s
  load_ktile_async<D>(p, b, h, k_begin, min(KT, k_end - k_begin), ktiles[0]);
  int buf = 0;
  for (int k0 = k_begin; k0 < k_end; k0 += KT, buf ^= 1) {
    float ksum[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) ksum[i][0] = ksum[i][1] = 0.f;
    const bool more = k0 + KT < k_end;
    if (more) load_ktile_async<D>(p, b, h, k0 + KT, min(KT, k_end - k0 - KT), ktiles[buf ^ 1]);
    cp_async_wait_le(more ? 1 : 0);
    __syncthreads();
    for (int mt = warp; mt < MT; mt += WARPS) {
      uint32_t qa[D / 16][4];
      if (own) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
#pragma unroll
          for (int e = 0; e < 4; ++e) qa[kk][e] = qown[kk][e];
      } else {
        load_q<D>(p, b, h, mt, qa);
      }
      float s[8][4];
      tile_scores<D>(qa, smem_u32(ktiles[buf]), s, p.scale_log2);
      const int r0 = mt * 16 + gq, r1 = r0 + 8;
      const float lse0 = r0 < p.R ? lse_s[r0] : INFINITY, lse1 = r1 < p.R ? lse_s[r1] : INFINITY;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        ksum[i][0] += ex2(s[i][0] - lse0) + ex2(s[i][2] - lse1);
        ksum[i][1] += ex2(s[i][1] - lse0) + ex2(s[i][3] - lse1);
      }
    }
    // reduce over the 8 lanes of a column quad (rows gq), then across warps in smem
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float v = ksum[i][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        ksum[i][e] = v;
      }
    if (gq == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        wsum[warp][i * 8 + cq * 2] = ksum[i][0];
        wsum[warp][i * 8 + cq * 2 + 1] = ksum[i][1];
      }
    }
    __syncthreads();
    if (threadIdx.x < KT && k0 + threadIdx.x < k_end) {
      float v = 0.f;
      for (int w2 = 0; w2 < WARPS; ++w2) v += wsum[w2][threadIdx.x];
      p.vote[(int64_t)unit * p.maxL + k0 + threadIdx.x] = v;
    }
  }
}

// per unit: pool, radix-select the keep-th largest, ordered compaction into ascending positions
constexpr int SEL_THREADS = 1024;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sm, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  __syncthreads();
  if (lane == 31) sm[warp] = incl;
  __syncthreads();
  uint32_t before = 0;
  total = 0;
  for (int w = 0; w < SEL_THREADS / 32; ++w) {
    if (w < warp) before += sm[w];
    total += sm[w];
  }
  return before + incl - v;
}

__global__ void __launch_bounds__(SEL_THREADS) select_kernel(const Params p) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t scan_sm[SEL_THREADS / 32];
  __shared__ uint32_t s_prefix, s_need;
  __shared__ int s_keep;
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x;
  const int b = unit / p.Hkv, h = unit - b * p.Hkv;
  const int n = __ldg(p.L + b) - p.w;  // prefix positions
  int32_t* out = p.idx + ((int64_t)b * p.Hkv + h) * p.idx_stride;
  const float* vote = p.vote + (int64_t)unit * p.maxL;
  float* pooled = p.pooled + (int64_t)unit * p.maxL;
  // per-sequence budget (heterogeneous batches): clamped to [w, budget]; read by one
  // thread and broadcast through shared memory
  if (threadIdx.x == 0) {
    int kb = p.keep;
    if (p.budgets != nullptr) kb = min(kb, max(0, p.budgets[b] - p.w));
    s_keep = max(0, min(kb, n));
    if (h == 0) p.idx_count[b] = s_keep;
  }
  __syncthreads();
  const int keep = s_keep;
  if (keep == n) {  // budget covers the prompt: keep everything
    for (int j = threadIdx.x; j < n; j += SEL_THREADS) out[j] = j;
    return;
  }
  // S3: zero-padded average pool of width 5 (fixed summation order)
  for (int j = threadIdx.x; j < n; j += SEL_THREADS) {
    float s = 0.f;
#pragma unroll
    for (int t = -2; t <= 2; ++t) s += (j + t >= 0 && j + t < n) ? vote[j + t] : 0.f;
    pooled[j] = s / 5.0f;
  }
  __syncthreads();
  // S4: radix select of the keep-th largest value (non-negative floats order as uint32)
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_need = keep;
  }
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += SEL_THREADS) hist[i] = 0;
    __syncthreads();
    const uint32_t pre = s_prefix;
    const uint32_t mask = (shift == 24) ? 0u : (0xffffffffu << (shift + 8));
    for (int j = threadIdx.x; j < n; j += SEL_THREADS) {
      const uint32_t u = __float_as_uint(pooled[j]);
      if ((u & mask) == (pre & mask)) atomicAdd(&hist[(u >> shift) & 255], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t need = s_need;
      int bin = 255;
      for (; bin > 0; --bin) {
        if (hist[bin] >= need) break;
        need -= hist[bin];
      }
      s_prefix = pre | ((uint32_t)bin << shift);
      s_need = need;  // how many of the values equal to the final threshold to take
    }
    __syncthreads();
  }
  const uint32_t thr = s_prefix, take_eq = s_need;
  // ordered compaction: > thr always, == thr for the first take_eq positions
  uint32_t base_out = 0, base_eq = 0;
  for (int j0 = 0; j0 < n; j0 += SEL_THREADS) {
    const int j = j0 + threadIdx.x;
    const uint32_t u = j < n ? __float_as_uint(pooled[j]) : 0u;
    const uint32_t eq = (j < n && u == thr) ? 1u : 0u;
    uint32_t tot_eq;
    const uint32_t rank_eq = base_eq + block_excl_scan(eq, scan_sm, tot_eq);
    const uint32_t sel = (j < n && (u > thr || (eq && rank_eq < take_eq))) ? 1u : 0u;
    uint32_t tot_sel;
    const uint32_t pos = base_out + block_excl_scan(sel, scan_sm, tot_sel);
    if (sel) out[pos] = j;
    base_out += tot_sel;
    base_eq += tot_eq;
  }
}

}  // namespace snap

// ============================================================================ tcgen05 passes
// S1/S2 on the 5th-generation tensor cores (head_dim 128, R = g*w <= 256 window-query rows):
// S[rows][128 keys] = Q . K^T with the rows on the MMA M dimension (one or two 128-row tiles)
// and the accumulator in TMEM, so thread x of softmax warp group m owns row m*128 + x and the
// lse pass is thread-local (online max / sum over its row); the vote pass turns its row into
// 2^(s - lse_r) and sums the 128 rows of every key column with a warp butterfly reduce-scatter
// (31 shuffles per 32 columns) plus a shared-memory sum over the warps.  Q arrives by one TMA
// box per 64-column slab (rows r = i*g + h in order), K by the 64-/16-row boxes of the verify
// kernel into a 3-stage ring; one thread issues the MMAs (K-major SWIZZLE_128B operands).
namespace snaptc {

constexpr int KT = 128;            // keys per stage (MMA N)
constexpr int SLAB = KT * 128;     // one 64-column slab of a 128-key K tile
constexpr int KSTAGE = 2 * SLAB;   // K only (32 KB)
constexpr int CHUNK = 4096;        // keys per CTA (32 stages: the CTA setup is amortised)
constexpr int BOXF = 64, BOXP = 16;  // full / partial TMA box rows

template <int NM>
struct Cfg {
  static constexpr int NSTAGE = NM == 1 ? 2 : 3;  // NM = 1: 2 CTAs / SM
  static constexpr int QROWS = NM * 128;
  static constexpr int QBUF = 2 * QROWS * 128;
  static constexpr int NSW = NM * 4;                     // softmax warps
  static constexpr int THREADS = NSW * 32 + 64;          // + producer warp + MMA warp
  static constexpr int AUX = NSW * KT * 4 + QROWS * 4 + 512;
  static constexpr int SMEM = NSTAGE * KSTAGE + QBUF + AUX + 1024;
  static constexpr int CTAS = NM == 1 ? 2 : 1;
  static constexpr int TMEM_COLS = 2 * NM * KT <= 256 ? 256 : 512;
};

template <int PASS, int NM>
__global__ void __launch_bounds__(Cfg<NM>::THREADS, Cfg<NM>::CTAS)
    snap_tc_kernel(const __grid_constant__ CUtensorMap kfull, const __grid_constant__ CUtensorMap kpart,
                   const __grid_constant__ CUtensorMap qmap, const snap::Params p) {
  using C = Cfg<NM>;
  constexpr int NSTAGE = C::NSTAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint8_t* qbuf = ring + NSTAGE * KSTAGE;
  float* wsum = reinterpret_cast<float*>(qbuf + C::QBUF);  // [NSW][KT] vote partial sums
  float* lse_s = wsum + C::NSW * KT;                       // [QROWS]
  uint64_t* full = reinterpret_cast<uint64_t*>(lse_s + C::QROWS);
  uint64_t* empty = full + NSTAGE;
  uint64_t* qfull = empty + NSTAGE;
  uint64_t* sfull = qfull + 1;   // [2]
  uint64_t* sempty = sfull + 2;  // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x / p.nchunks, chunk = blockIdx.x - unit * p.nchunks;
  const int b = unit / p.Hkv, h = unit - b * p.Hkv;
  pdl_wait();  // q_obs / the cache (and, for the vote pass, the lse partials) are ready
  const int L = __ldg(p.L + b);
  const int k_begin = chunk * CHUNK;
  const int k_end = PASS == 0 ? min(L, k_begin + CHUNK) : min(L - p.w, k_begin + CHUNK);
  if (k_begin >= k_end) {  // uniform: a chunk past the prompt (lse pass: an empty partial)
    if (PASS == 0)
      for (int r = threadIdx.x; r < p.R; r += blockDim.x) {
        float* base = p.part + ((int64_t)unit * p.nchunks + chunk) * p.R * 2;
        base[r * 2] = -INFINITY;
        base[r * 2 + 1] = 0.f;
      }
    pdl_trigger();
    return;
  }
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < NSTAGE; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], 1);
    }
    mbar_init(qfull, 1);
    for (int s2 = 0; s2 < 2; ++s2) {
      mbar_init(&sfull[s2], 1);
      mbar_init(&sempty[s2], C::NSW);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < C::QBUF / 16; i += blockDim.x) {  // Q rows >= R stay zero
    if (((i * 16) / 128) % C::QROWS >= p.R) reinterpret_cast<uint4*>(qbuf)[i] = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async();
  if (warp == C::NSW + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *tslot;
  const int nst = (k_end - k_begin + KT - 1) / KT;

  if (warp == C::NSW) {
    // ============================== TMA producer ==============================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(qfull, 2 * p.R * 128);
      for (int sub = 0; sub < 2; ++sub) tma_load_4d(qbuf + sub * C::QROWS * 128, &qmap, qfull, sub * 64, h * p.g, 0, b, pol);
      for (int j = 0; j < nst; ++j) {
        const int stage = j % NSTAGE, pos = k_begin + j * KT, nvalid = min(KT, k_end - pos);
        uint8_t* kt = ring + stage * KSTAGE;
        mbar_wait(&empty[stage], ((j / NSTAGE) & 1) ^ 1);
        int bytes = 0;
        for (int hf = 0; hf < 2; ++hf) {
          const int hv = nvalid - hf * BOXF;
          if (hv >= BOXF) bytes += 2 * BOXF * 128;
          else if (hv > 0) bytes += 2 * ((hv + BOXP - 1) / BOXP) * BOXP * 128;
        }
        mbar_arrive_expect_tx(&full[stage], bytes);
        for (int hf = 0; hf < 2; ++hf) {
          const int hv = nvalid - hf * BOXF, r0 = pos + hf * BOXF;
          for (int sub = 0; sub < 2; ++sub) {
            const int off = sub * SLAB + hf * BOXF * 128;
            if (hv >= BOXF) {
              tma_load_4d(kt + off, &kfull, &full[stage], sub * 64, r0, h, b, pol);
            } else if (hv > 0) {
              for (int bx = 0; bx * BOXP < hv; ++bx)
                tma_load_4d(kt + off + bx * BOXP * 128, &kpart, &full[stage], sub * 64, r0 + bx * BOXP, h, b, pol);
            }
          }
        }
      }
    }
  } else if (warp == C::NSW + 1) {
    // ============================== MMA issuer ==============================
    if (lane == 0) {
      constexpr uint32_t ID = tc::idesc(128, KT, 0, 0);
      const uint32_t ring_a = smem_u32(ring), q_a = smem_u32(qbuf);
      mbar_wait(qfull, 0);
      for (int j = 0; j < nst; ++j) {
        const int stage = j % NSTAGE, sb = j & 1;
        mbar_wait(&full[stage], (j / NSTAGE) & 1);
        mbar_wait(&sempty[sb], ((j >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t kt = ring_a + stage * KSTAGE;
#pragma unroll
        for (int m = 0; m < NM; ++m)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * SLAB + (kk & 3) * 32;
            const uint32_t qoff = (kk >> 2) * (C::QROWS * 128) + m * 128 * 128 + (kk & 3) * 32;
            tc::mma_f16(tbase + (sb * NM + m) * KT, tc::sdesc(q_a + qoff, 16, 1024, 2), tc::sdesc(kt + off, 16, 1024, 2),
                        ID, kk > 0 ? 1u : 0u);
          }
        tc::commit(&sfull[sb]);
        tc::commit(&empty[stage]);
      }
    }
  } else {
    // ============================== row threads ==============================
    const int m = warp >> 2, x = threadIdx.x;           // row r = x (warps 0..NSW-1)
    const int r = x;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const bool live = r < p.R;
    const int lim = live ? L - p.w + r / p.g : -1;       // causal limit of window query i = r / g
    float mrow = -INFINITY, lrow = 0.f, lse = INFINITY;
    if (PASS == 1 && live) {  // lse_r from the chunk partials of the lse pass
      const int nch = (L + CHUNK - 1) / CHUNK;
      const float* base = p.part + (int64_t)unit * p.nchunks * p.R * 2 + r * 2;
      float M = -INFINITY;
      for (int c2 = 0; c2 < nch; ++c2) M = fmaxf(M, base[(int64_t)c2 * p.R * 2]);
      float S = 0.f;
      for (int c2 = 0; c2 < nch; ++c2) {
        const float l = base[(int64_t)c2 * p.R * 2 + 1];
        if (l > 0.f) S += l * ex2(base[(int64_t)c2 * p.R * 2] - M);
      }
      lse = M + __log2f(S);
    }
    const float sl2 = p.scale_log2;
    for (int j = 0; j < nst; ++j) {
      const int sb = j & 1, pos = k_begin + j * KT;
      mbar_wait(&sfull[sb], (j >> 1) & 1);
      tc::fence_after();
      const uint32_t ta = tbase + (sb * NM + m) * KT + lane_off;
#pragma unroll 1
      for (int c = 0; c < KT; c += 32) {
        float v[32];
        tc::tld16(ta + c, v);
        tc::tld16(ta + c + 16, v + 16);
        tc::wait_ld();
        if (PASS == 0) {
          float mx = -INFINITY;
          if (pos + c + 32 <= k_end && pos + c + 31 <= L - p.w && live) {  // no key masked
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              v[t] *= sl2;
              mx = fmaxf(mx, v[t]);
            }
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              const int key = pos + c + t;
              v[t] = (live && key < k_end && key <= lim) ? v[t] * sl2 : -INFINITY;
              mx = fmaxf(mx, v[t]);
            }
          }
          const float mn = fmaxf(mrow, mx);
          const float base = (mn == -INFINITY) ? 0.f : mn;
          float sum = 0.f;
#pragma unroll
          for (int t = 0; t < 32; ++t) sum += ex2(v[t] - base);
          lrow = lrow * ex2(mrow - base) + sum;
          mrow = mn;
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int key = pos + c + t;
            v[t] = (live && key < k_end) ? ex2(v[t] * sl2 - lse) : 0.f;
          }
          // butterfly reduce-scatter over the warp: lane t ends with column t's sum of 32 rows
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            const bool hi = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < o; ++i) {
              const float keep = hi ? v[i + o] : v[i];
              const float send = hi ? v[i] : v[i + o];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          wsum[warp * KT + c + lane] = v[0];
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[sb]);
      if (PASS == 1) {
        named_bar_sync(2, C::NSW * 32);
        if (x < KT && pos + x < k_end) {
          float vsum = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < C::NSW; ++w2) vsum += wsum[w2 * KT + x];
          p.vote[(int64_t)unit * p.maxL + pos + x] = vsum;
        }
        named_bar_sync(2, C::NSW * 32);  // wsum is rewritten by the next stage
      }
    }
    if (PASS == 0 && live) {
      float* base = p.part + ((int64_t)unit * p.nchunks + chunk) * p.R * 2;
      base[r * 2] = mrow;
      base[r * 2 + 1] = lrow;
    }
  }
  tc::fence_before();
  __syncthreads();
  pdl_trigger();
  if (warp == C::NSW + 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TMEM_COLS));
  }
}

}  // namespace snaptc

static size_t snap_align(size_t x) { return (x + 255) & ~size_t(255); }

static size_t snap_ws(int B, int Hkv, int R, int maxL) {
  const int nchunks = (maxL + snap::CHUNK - 1) / snap::CHUNK;
  const size_t units = (size_t)B * Hkv;
  return snap_align(units * nchunks * R * 2 * 4) + 2 * snap_align(units * maxL * 4);
}

static PFN_cuTensorMapEncodeTiled_v12000 snap_encode() {
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

static bool snap_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                     const cuuint32_t* box) {
  auto enc = snap_encode();
  if (enc == nullptr) return false;
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NM>
static md_status snap_tc_launch(const md_kv_cache* c, const void* q_obs, const snap::Params& p, unsigned grid,
                                cudaStream_t s) {
  using C = snaptc::Cfg<NM>;
  CUtensorMap kf, kp, qm;
  const cuuint64_t kd[4] = {(cuuint64_t)c->head_dim, (cuuint64_t)c->capacity, (cuuint64_t)c->num_kv_heads,
                            (cuuint64_t)c->batch};
  const cuuint64_t ks[3] = {(cuuint64_t)c->stride_s * 2, (cuuint64_t)c->stride_h * 2, (cuuint64_t)c->stride_b * 2};
  const cuuint32_t kbf[4] = {64, (cuuint32_t)snaptc::BOXF, 1, 1}, kbp[4] = {64, (cuuint32_t)snaptc::BOXP, 1, 1};
  const cuuint64_t qd[4] = {(cuuint64_t)c->head_dim, (cuuint64_t)p.Hq, (cuuint64_t)p.w, (cuuint64_t)p.B};
  const cuuint64_t qs[3] = {(cuuint64_t)c->head_dim * 2, (cuuint64_t)p.Hq * c->head_dim * 2,
                            (cuuint64_t)p.w * p.Hq * c->head_dim * 2};
  const cuuint32_t qb[4] = {64, (cuuint32_t)p.g, (cuuint32_t)p.w, 1};
  MD_REQUIRE(snap_map(&kf, c->k, 4, kd, ks, kbf) && snap_map(&kp, c->k, 4, kd, ks, kbp) &&
                 snap_map(&qm, q_obs, 4, qd, qs, qb),
             MD_ERR_INVALID_ARG, "md_snapkv_select: cuTensorMapEncodeTiled failed (strides / alignment)");
  static int done_dev = -1;  // per-process; the attribute call is idempotent (benign race)
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev != dev) {
    if (cudaFuncSetAttribute(snaptc::snap_tc_kernel<0, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) !=
            cudaSuccess ||
        cudaFuncSetAttribute(snaptc::snap_tc_kernel<1, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) !=
            cudaSuccess)
      return check_launch("cudaFuncSetAttribute");
    done_dev = dev;
  }
  launch_pdl(snaptc::snap_tc_kernel<0, NM>, dim3(grid), dim3(C::THREADS), (size_t)C::SMEM, s, kf, kp, qm, p);
  launch_pdl(snaptc::snap_tc_kernel<1, NM>, dim3(grid), dim3(C::THREADS), (size_t)C::SMEM, s, kf, kp, qm, p);
  return check_launch("snap_tc_kernel");
}

}  // namespace md

extern "C" MD_API size_t md_snapkv_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads, int32_t w,
                                            int32_t max_prefill_len) {
  if (batch < 1 || num_kv_heads < 1 || num_q_heads < 1 || num_q_heads % num_kv_heads || w < 1 || max_prefill_len < w)
    return 0;
  return md::snap_ws(batch, num_kv_heads, (num_q_heads / num_kv_heads) * w, max_prefill_len);
}

extern "C" MD_API md_status md_snapkv_select(const md_kv_cache* c, const void* q_obs, int32_t num_q_heads,
                                      const int32_t* prefill_len, int32_t max_prefill_len, int32_t w, int32_t budget,
                                      const int32_t* budgets, float scale, int32_t* idx, int32_t idx_stride,
                                      int32_t* idx_count,
                                      void* workspace, size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(c != nullptr && c->k != nullptr && q_obs != nullptr && prefill_len != nullptr && idx != nullptr &&
                 idx_count != nullptr,
             MD_ERR_INVALID_ARG, "md_snapkv_select: NULL argument");
  MD_REQUIRE(c->head_dim == 64 || c->head_dim == 128, MD_ERR_UNSUPPORTED, "md_snapkv_select: head_dim must be 64/128");
  MD_REQUIRE(num_q_heads >= 1 && num_q_heads % c->num_kv_heads == 0, MD_ERR_INVALID_ARG,
             "md_snapkv_select: num_q_heads must be a multiple of Hkv");
  MD_REQUIRE(w >= 1 && budget > w && max_prefill_len >= w && max_prefill_len <= c->capacity, MD_ERR_INVALID_ARG,
             "md_snapkv_select: need 1 <= w < budget and w <= max_prefill_len <= capacity");
  MD_REQUIRE(idx_stride >= budget - w, MD_ERR_INVALID_ARG, "md_snapkv_select: idx_stride < budget - w");
  const int g = num_q_heads / c->num_kv_heads;
  MD_REQUIRE(g * w <= 256, MD_ERR_UNSUPPORTED, "md_snapkv_select: g * w > 256 rows per KV head");
  MD_REQUIRE(c->stride_s % 8 == 0 && c->stride_h % 8 == 0 && c->stride_b % 8 == 0 && aligned16(c->k) &&
                 aligned16(q_obs),
             MD_ERR_INVALID_ARG, "md_snapkv_select: 16-byte alignment of cache rows and q_obs required");
  const size_t need = snap_ws(c->batch, c->num_kv_heads, g * w, max_prefill_len);
  MD_REQUIRE(workspace != nullptr && workspace_bytes >= need, MD_ERR_WORKSPACE,
             "md_snapkv_select: workspace of %zu bytes required, %zu given", need, workspace_bytes);
  snap::Params p{};
  p.k = static_cast<const uint16_t*>(c->k);
  p.sB = c->stride_b;
  p.sH = c->stride_h;
  p.sS = c->stride_s;
  p.q = static_cast<const uint16_t*>(q_obs);
  p.L = prefill_len;
  p.B = c->batch;
  p.Hq = num_q_heads;
  p.Hkv = c->num_kv_heads;
  p.g = g;
  p.w = w;
  p.R = g * w;
  p.nchunks = (max_prefill_len + snap::CHUNK - 1) / snap::CHUNK;
  p.scale_log2 = scale * snap::LOG2E;
  p.maxL = max_prefill_len;
  const size_t units = (size_t)c->batch * c->num_kv_heads;
  uint8_t* w8 = static_cast<uint8_t*>(workspace);
  p.part = reinterpret_cast<float*>(w8);
  w8 += snap_align(units * p.nchunks * p.R * 2 * 4);
  p.vote = reinterpret_cast<float*>(w8);
  w8 += snap_align(units * max_prefill_len * 4);
  p.pooled = reinterpret_cast<float*>(w8);
  p.idx = idx;
  p.idx_count = idx_count;
  p.idx_stride = idx_stride;
  p.keep = budget - w;
  p.budgets = budgets;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = static_cast<unsigned>(units * p.nchunks);
  if (c->head_dim == 128) {  // tcgen05 scoring passes (the mma.sync passes serve head_dim 64)
    p.nchunks = (max_prefill_len + snaptc::CHUNK - 1) / snaptc::CHUNK;  // <= the workspace's chunk count
    const unsigned grid_tc = static_cast<unsigned>(units * p.nchunks);
    const md_status st = (p.R <= 128) ? snap_tc_launch<1>(c, q_obs, p, grid_tc, s)
                                   : snap_tc_launch<2>(c, q_obs, p, grid_tc, s);
    if (st != MD_OK) return st;
  } else {
    launch_pdl(snap::lse_kernel<64>, dim3(grid), dim3(snap::THREADS), 0, s, p);
    launch_pdl(snap::vote_kernel<64>, dim3(grid), dim3(snap::THREADS), 0, s, p);
  }
  launch_pdl(snap::select_kernel, dim3(static_cast<unsigned>(units)), dim3(snap::SEL_THREADS), 0, s, p);
  return check_launch("md_snapkv_select");
}

// attn.cu — md_verify_attn_full, md_draft_attn_sparse, md_attn_workspace_bytes
// (SURVEY §8(a) rows a2, a3, a4).
//
// Both calls are split-KV flash decoding over the shared [B][Hkv][cap][d] bf16 cache:
//
//   work item = (b, kv head, split): a contiguous chunk of the unit's key index space,
//            producing (o, lse) for all R = g*T query rows of that KV head (verify) or
//            R = g rows (draft), so each KV byte is read from HBM exactly once per call
//            (verify and decode share the same KV bytes).  Persistent grid: one
//            CTA per SM walks items c, c+G, ...; the producer runs ahead across items.
//   warp 0..NC-1  consumers: warp (mt, ks) owns query-row tile mt (16 rows) and the
//            ks-th KW-key slice of every tile: S = Q K^T and O += P V with
//            mma.sync m16n8k16 bf16 -> fp32 (B200 legacy HMMA path, ~550 TFLOP/s measured,
//            far above the <= 48 FLOP/B * 7 TB/s this HBM-bound loop needs), online
//            softmax in the log2 domain with quad shuffles.
//   warp NC  producer: one lane bulk-copies each item's Q rows into a double-buffered
//            padded smem slot and streams 64-key K and V tiles with 4-D TMA
//            (cp.async.bulk.tensor, SWIZZLE_128B, L2 evict_first) into an NSTAGE
//            mbarrier ring; only boxes that hold valid keys are fetched.
//   epilogue  the KS key-slice partials are merged in shared memory; with one split the
//            CTA writes the final out/lse, otherwise a partial to the workspace, and the
//            last CTA to finish a unit (atomic arrival counter) combines the splits by
//            log-sum-exp (O6 identity) — no second kernel launch.
//
// The draft call is the same kernel walking two row ranges of the cache (sink rows
// [0, min(sink, n)) and window rows [max(sink, n - window), n)), i.e. the StreamingLLM
// compressed KV of P:453/P:720 without materialising it.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <mutex>

#include "md_common.cuh"
#include "md_internal.h"

namespace md {

constexpr int TK = 64;        // keys per pipeline tile
constexpr int BOX_ROWS = 16;  // rows per TMA box of a partial tile (fetch granularity of ragged ends)
constexpr int NSTAGE = 3;     // pipeline depth (3 x 32 KB at d=128 -> 2 CTAs / SM)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

enum : int { MODE_VERIFY = 0, MODE_DRAFT = 1 };

// K and V tensor maps with a full-tile box (TK rows) and a partial-tile box (BOX_ROWS rows).
struct TmapSet {
  CUtensorMap k_full, v_full, k_part, v_part;
};

struct AttnParams {
  const uint16_t* q;     // bf16 [B][T][Hq][D]
  float* out;            // [B][T][Hq][D] (written directly when splits == 1)
  float* lse;            // [B][T][Hq] natural log, may be null
  float* ws_o;           // [units][splits][R][D] normalised partial outputs
  float* ws_lse;         // [units][splits][R] partial lse, log2 units (-inf if empty)
  const int32_t* kv_len; // [B]
  int Hq, Hkv, T, g, R;
  int* counters;         // [units] split-arrival counters (zero between calls)
  int splits, chunk;     // chunk: keys per split, multiple of TK
  int items;             // units * splits work items
  int sink, window;      // draft only
  int mode;
  float scale_log2;      // scale * log2(e)
};

// Physical key ranges one CTA walks, in logical order.
struct Ranges {
  int s0, e0, s1, e1;
};

__device__ __forceinline__ Ranges cta_ranges(const AttnParams& p, int n, int split) {
  Ranges r{0, 0, 0, 0};
  const int lo = split * p.chunk;
  if (p.mode == MODE_VERIFY) {
    r.s0 = lo;
    r.e0 = max(lo, min(n, lo + p.chunk));
  } else {
    const int nA = min(p.sink, n);
    const int startB = max(p.sink, n - p.window);
    const int nB = max(0, n - startB);
    const int hi = min(nA + nB, lo + p.chunk);
    // logical [lo, hi) -> sink part [lo, min(hi, nA)) and window part
    r.s0 = lo;
    r.e0 = max(lo, min(hi, nA));
    const int wl = max(lo, nA), wh = hi;
    r.s1 = startB + (wl - nA);
    r.e1 = max(r.s1, startB + (wh - nA));
  }
  return r;
}

// ============================================================================ rows kernel
// attn_rows_kernel: one CTA per work item (b, kv head, split), 2 CTAs / SM, query rows on
// the MMA M dimension (16-row tiles), used for R > 8 query rows per KV head (GQA verify:
// R = 20 for Llama-3.1 gamma=4, 35 for Qwen2.5).  Consumer warp (mt, ks) owns row tile mt
// and the ks-th key slice of every 64-key tile.  Split partials are combined by
// attn_merge_kernel.  (Measured 7.07 TB/s = 97% of a plain read stream at the target point.)
template <int D>
struct SmemLayout {
  static constexpr int SUB = D / 64;                    // 128-byte column sub-tiles per row
  static constexpr int TILE_BYTES = TK * D * 2;         // one K (or V) tile
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES;    // K + V
  static constexpr int RING_BYTES = NSTAGE * STAGE_BYTES;
  static constexpr int TOTAL = RING_BYTES + 1024 /*align slack*/ + 2 * NSTAGE * 8 + 64;
};

template <int D, int MT, int KS>
__global__ void __launch_bounds__((MT * KS + 1) * 32, 2)
    attn_rows_kernel(const __grid_constant__ TmapSet tm, const AttnParams p) {
  constexpr int NC = MT * KS;          // consumer warps
  constexpr int KW = TK / KS;          // keys per consumer warp per tile
  constexpr int NT_S = KW / 8;         // n8 tiles of S per warp
  constexpr int NT_O = D / 8;          // n8 tiles of O
  constexpr int KQ = D / 16;           // k16 steps of QK^T
  using L = SmemLayout<D>;
  static_assert(KW % 16 == 0, "key slice must be a multiple of 16");
  static_assert(NC * 16 * (D + 4) * 4 + NC * 16 * 2 * 4 + MT * 16 * 4 <= L::RING_BYTES, "epilogue buffer must fit in the ring");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::RING_BYTES);
  uint64_t* empty = full + NSTAGE;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x / p.splits, split = blockIdx.x - unit * p.splits;
  const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
  const int n = __ldg(p.kv_len + b);
  const Ranges rg = cta_ranges(p, n, split);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NC) {
    // ============================== TMA producer ==============================
    if (lane == 0) {
      prefetch_tmap(&tm.k_full);
      prefetch_tmap(&tm.v_full);
      prefetch_tmap(&tm.k_part);
      prefetch_tmap(&tm.v_part);
      const uint64_t pol = policy_evict_first();
      int it = 0;
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
        const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
#pragma unroll 1
        for (int pos = rs; pos < re; pos += TK, ++it) {
          const int stage = it % NSTAGE;
          mbar_wait(&empty[stage], ((it / NSTAGE) & 1) ^ 1);
          const int nvalid = min(TK, re - pos);
          uint8_t* kt = smem + stage * L::STAGE_BYTES;
          uint8_t* vt = kt + L::TILE_BYTES;
          if (nvalid == TK) {  // full tile: one TK-row box per 128-byte column slab
            mbar_arrive_expect_tx(&full[stage], L::STAGE_BYTES);
            for (int sub = 0; sub < L::SUB; ++sub) {
              tma_load_4d(kt + sub * TK * 128, &tm.k_full, &full[stage], sub * 64, pos, kvh, b, pol);
              tma_load_4d(vt + sub * TK * 128, &tm.v_full, &full[stage], sub * 64, pos, kvh, b, pol);
            }
          } else {  // ragged end: only the BOX_ROWS-row boxes that hold valid keys
            const int nbox = (nvalid + BOX_ROWS - 1) / BOX_ROWS;
            mbar_arrive_expect_tx(&full[stage], nbox * BOX_ROWS * 128 * L::SUB * 2);
            for (int sub = 0; sub < L::SUB; ++sub)
              for (int bx = 0; bx < nbox; ++bx) {
                const int off = sub * TK * 128 + bx * BOX_ROWS * 128;
                tma_load_4d(kt + off, &tm.k_part, &full[stage], sub * 64, pos + bx * BOX_ROWS, kvh, b, pol);
                tma_load_4d(vt + off, &tm.v_part, &full[stage], sub * 64, pos + bx * BOX_ROWS, kvh, b, pol);
              }
            }
        }
      }
    }
    return;
  }

  // ============================== consumers ==============================
  const int mt = warp / KS, ks = warp - mt * KS;
  const int gq = lane >> 2, cq = lane & 3;  // fragment row group / column quad
  // Q fragments for rows mt*16 + {gq, gq+8}; row r -> (t = r / g, head = kvh*g + r % g)
  uint32_t qa[KQ][4];
  {
    const int r0 = mt * 16 + gq, r1 = r0 + 8;
    const uint32_t* q0 = nullptr;
    const uint32_t* q1 = nullptr;
    if (r0 < p.R)
      q0 = reinterpret_cast<const uint32_t*>(
          p.q + ((int64_t)(b * p.T + r0 / p.g) * p.Hq + kvh * p.g + r0 % p.g) * D);
    if (r1 < p.R)
      q1 = reinterpret_cast<const uint32_t*>(
          p.q + ((int64_t)(b * p.T + r1 / p.g) * p.Hq + kvh * p.g + r1 % p.g) * D);
#pragma unroll
    for (int kk = 0; kk < KQ; ++kk) {
      const int c = kk * 8 + cq;  // 32-bit word index = (kk*16 + 2*cq) / 2
      qa[kk][0] = q0 ? __ldg(q0 + c) : 0u;
      qa[kk][1] = q1 ? __ldg(q1 + c) : 0u;
      qa[kk][2] = q0 ? __ldg(q0 + c + 4) : 0u;
      qa[kk][3] = q1 ? __ldg(q1 + c + 4) : 0u;
    }
  }
  // causal limit per fragment row (verify): key j visible iff j <= n - T + t(row)
  int lim0 = 0x7fffffff, lim1 = 0x7fffffff;
  if (p.mode == MODE_VERIFY) {
    const int r0 = mt * 16 + gq, r1 = r0 + 8;
    lim0 = n - p.T + min(r0, p.R - 1) / p.g;
    lim1 = n - p.T + min(r1, p.R - 1) / p.g;
  }

  float o[NT_O][4];
#pragma unroll
  for (int i = 0; i < NT_O; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const uint32_t ring = smem_u32(smem);
  int it = 0;
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
#pragma unroll 1
    for (int pos = rs; pos < re; pos += TK, ++it) {
      const int stage = it % NSTAGE;
      mbar_wait(&full[stage], (it / NSTAGE) & 1);
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
            const uint32_t addr = kt + (chunk >> 3) * (TK * 128) + swz128(row, chunk & 7);
            uint32_t b0, b1, b2, b3;
            ldsm_x4(addr, b0, b1, b2, b3);
            mma_bf16_16816(s[2 * np], qa[kk], b0, b1);
            mma_bf16_16816(s[2 * np + 1], qa[kk], b2, b3);
          }
        }
        // ---------------- scale, mask, online softmax (log2 domain)
        const bool need_mask = (kw0 + KW > nvalid) || (pos + kw0 + KW - 1 > min(lim0, lim1));
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int i = 0; i < NT_S; ++i) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float v = s[i][e] * p.scale_log2;
            if (need_mask) {
              const int ko = kw0 + i * 8 + cq * 2 + (e & 1);
              const int lim = (e < 2) ? lim0 : lim1;
              if (ko >= nvalid || pos + ko > lim) v = -INFINITY;
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
          // keys this thread's B fragments cover (for sanitising invalid rows)
          const int kf = kw0 + kp * 16 + cq * 2;
#pragma unroll
          for (int dp = 0; dp < NT_O / 2; ++dp) {
            const int chunk = dp * 2 + (lane >> 4);
            const uint32_t addr = vt + (chunk >> 3) * (TK * 128) + swz128(krow, chunk & 7);
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(addr, b0, b1, b2, b3);
            if (sanitize) {  // rows past the valid keys may hold non-finite bits: zero them
              const uint32_t m_lo = (kf < nvalid ? 0x0000ffffu : 0u) | (kf + 1 < nvalid ? 0xffff0000u : 0u);
              const uint32_t m_hi = (kf + 8 < nvalid ? 0x0000ffffu : 0u) | (kf + 9 < nvalid ? 0xffff0000u : 0u);
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

  // ============================== epilogue ==============================
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

  constexpr int OSTR = D + 4;  // padded fp32 row stride of the merge buffer
  float* obuf = reinterpret_cast<float*>(smem);                 // [NC][16][OSTR]
  float* mlbuf = obuf + NC * 16 * OSTR;                          // [NC][16][2] (m, l) per warp row
  float* lsebuf = mlbuf + NC * 16 * 2;                           // [MT][16] combined lse (log2)
  named_bar_sync(1, NC * 32);  // every consumer is done reading the ring
  if (cq == 0) {
    mlbuf[(warp * 16 + gq) * 2 + 0] = m0;
    mlbuf[(warp * 16 + gq) * 2 + 1] = l0;
    mlbuf[(warp * 16 + gq + 8) * 2 + 0] = m1;
    mlbuf[(warp * 16 + gq + 8) * 2 + 1] = l1;
  }
  named_bar_sync(1, NC * 32);
  // scale this warp's O by exp2(m_w - M) / L, where M, L combine the KS key slices
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
      const float mk0 = mlbuf[((mt * KS + k) * 16 + gq) * 2], lk0 = mlbuf[((mt * KS + k) * 16 + gq) * 2 + 1];
      const float mk1 = mlbuf[((mt * KS + k) * 16 + gq + 8) * 2], lk1 = mlbuf[((mt * KS + k) * 16 + gq + 8) * 2 + 1];
      if (lk0 > 0.f) L0 += lk0 * ex2(mk0 - M0);
      if (lk1 > 0.f) L1 += lk1 * ex2(mk1 - M1);
    }
    f0 = (l0 > 0.f) ? ex2(m0 - M0) / L0 : 0.f;
    f1 = (l1 > 0.f) ? ex2(m1 - M1) / L1 : 0.f;
    if (ks == 0 && cq == 0) {  // the combined lse (log2) of the row tile
      lsebuf[mt * 16 + gq] = (L0 > 0.f) ? M0 + __log2f(L0) : -INFINITY;
      lsebuf[mt * 16 + gq + 8] = (L1 > 0.f) ? M1 + __log2f(L1) : -INFINITY;
    }
  }
#pragma unroll
  for (int i = 0; i < NT_O; ++i) {
    const int d0 = i * 8 + cq * 2;
    *reinterpret_cast<float2*>(&obuf[(warp * 16 + gq) * OSTR + d0]) = make_float2(o[i][0] * f0, o[i][1] * f0);
    *reinterpret_cast<float2*>(&obuf[(warp * 16 + gq + 8) * OSTR + d0]) = make_float2(o[i][2] * f1, o[i][3] * f1);
  }
  named_bar_sync(1, NC * 32);
  // sum the KS slices and write rows r < R (float4 per thread)
  constexpr int V4 = D / 4;
  const bool final_out = (p.splits == 1);
  for (int idx = threadIdx.x; idx < MT * 16 * V4; idx += NC * 32) {
    const int rr = idx / V4, c4 = (idx - rr * V4) * 4;
    const int mtile = rr >> 4, rin = rr & 15;
    const int r = mtile * 16 + rin;
    if (r >= p.R) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(&obuf[((mtile * KS + k) * 16 + rin) * OSTR + c4]);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    const float lse2 = lsebuf[mtile * 16 + rin];
    if (final_out) {
      const int t = r / p.g, h = kvh * p.g + r % p.g;
      const int64_t orow = (int64_t)(b * p.T + t) * p.Hq + h;
      *reinterpret_cast<float4*>(p.out + orow * D + c4) = acc;
      if (c4 == 0 && p.lse != nullptr) p.lse[orow] = lse2 * LN2;
    } else {
      const int64_t prow = ((int64_t)unit * p.splits + split) * p.R + r;
      *reinterpret_cast<float4*>(p.ws_o + prow * D + c4) = acc;
      if (c4 == 0) p.ws_lse[prow] = lse2;
    }
  }
}

// Combine the split partials of one (unit, row) for attn_rows_kernel: one warp per row, lane = split for the
// weights, lanes over d for the sum.  o = sum_s 2^{lse_s - M} o_s / sum_s 2^{lse_s - M}.
template <int D>
__global__ void __launch_bounds__(256) attn_merge_kernel(const AttnParams p, int units) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp_global >= units * p.R) return;
  const int unit = warp_global / p.R, r = warp_global - unit * p.R;
  const int S = p.splits;
  const float* lse_base = p.ws_lse + (int64_t)unit * S * p.R + r;
  float M = -INFINITY;
  for (int s = lane; s < S; s += 32) M = fmaxf(M, lse_base[(int64_t)s * p.R]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  constexpr int PER = D / 32;
  float acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
  float W = 0.f;
  for (int s = 0; s < S; ++s) {
    const float ls = lse_base[(int64_t)s * p.R];
    if (ls == -INFINITY) continue;
    const float w = ex2(ls - M);
    W += w;
    const float* src = p.ws_o + (((int64_t)unit * S + s) * p.R + r) * D + lane * PER;
#pragma unroll
    for (int i = 0; i < PER; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(src + i);
      acc[i] += w * v.x;
      acc[i + 1] += w * v.y;
      acc[i + 2] += w * v.z;
      acc[i + 3] += w * v.w;
    }
  }
  const float inv = W > 0.f ? 1.f / W : 0.f;
  const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
  const int t = r / p.g, h = kvh * p.g + r % p.g;
  const int64_t orow = (int64_t)(b * p.T + t) * p.Hq + h;
#pragma unroll
  for (int i = 0; i < PER; i += 4)
    *reinterpret_cast<float4*>(p.out + orow * D + lane * PER + i) =
        make_float4(acc[i] * inv, acc[i + 1] * inv, acc[i + 2] * inv, acc[i + 3] * inv);
  if (lane == 0 && p.lse != nullptr) p.lse[orow] = (W > 0.f) ? (M + __log2f(W)) * LN2 : -INFINITY;
}

// ============================================================================ keys kernel
// Compile-time geometry of one kernel instance.
//   D    head dim (64 / 128)
//   NTW  n8 query-row tiles per consumer warp (rows on the MMA N dimension, padded to 8)
//   NG   row groups (NG * NTW * 8 >= R)
//   KS   key slices per tile (consumer warps sharing one K/V tile)
// Consumer warp (grp, ks) computes S^T = K Q^T and O^T += V^T P^T for rows
// [grp*NTW*8, (grp+1)*NTW*8) over keys [ks*KW, (ks+1)*KW) of every tile ("swap-AB": the
// 16 KV tokens of an MMA sit on M, the few query rows on N, so padding waste is at most
// 7 rows per group instead of up to 15, and each K/V fragment feeds all NTW row tiles).
template <int D, int NTW, int NG, int KS>
struct KCfg {
  static constexpr int NC = NG * KS;
  static constexpr int THREADS = (NC + 1) * 32;
  static constexpr int KW = TK / KS;                 // keys per consumer warp per tile
  static constexpr int KB = KW / 16;                 // 16-key blocks per warp per tile
  static constexpr int GROWS = NTW * 8;              // query rows per group
  static constexpr int ROWS = NG * GROWS;            // padded query rows
  static constexpr int SUB = D / 64;                 // 128-byte column sub-tiles per K/V row
  static constexpr int TILE = TK * D * 2;            // one K (or V) tile
  static constexpr int STAGE = 2 * TILE;             // K + V
  static constexpr int QSTR = D * 2 + 16;            // padded smem row of Q (conflict-free ldmatrix)
  static constexpr int QBUF = 2 * ROWS * QSTR;       // double-buffered per work item
  static constexpr int OSTR = GROWS + 1;             // fp32 epilogue stride per d (transposed O)
  static constexpr int EPI = NC * D * OSTR * 4 + NC * GROWS * 2 * 4 + ROWS * 4 + 64;
  static constexpr int BARS = 256;
  static constexpr int FIXED = QBUF + EPI + BARS + 1024 /*alignment slack*/;
  static constexpr int SMEM_MAX = 227 * 1024;
  static constexpr int NSTAGE_FIT = (SMEM_MAX - FIXED) / STAGE;
  static constexpr int NSTAGE = NSTAGE_FIT > 8 ? 8 : NSTAGE_FIT;
  static constexpr int SMEM = NSTAGE * STAGE + FIXED;
  static_assert(NSTAGE >= 2, "not enough shared memory for a 2-stage ring");
  static_assert(KW % 16 == 0, "key slice must be a multiple of 16");
};

// Persistent split-KV attention for few query rows (R <= 8 per KV head: the draft call and
// MHA verify).  CTA c processes work items c, c + G, c + 2G, ... where an
// item is (unit = (b, kv head), split); the producer streams items back to back so the
// next item's Q rows and K/V tiles are in flight while the consumers finish the current one.
template <int D, int NTW, int NG, int KS>
__global__ void __launch_bounds__(KCfg<D, NTW, NG, KS>::THREADS, 1)
    attn_keys_kernel(const __grid_constant__ TmapSet tm, const AttnParams p) {
  using C = KCfg<D, NTW, NG, KS>;
  constexpr int NC = C::NC, KW = C::KW, KB = C::KB, NSTAGE = C::NSTAGE;
  constexpr int MD16 = D / 16;  // m16 tiles of O^T (head-dim rows) == k16 steps of S^T

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qbuf = smem + NSTAGE * C::STAGE;
  float* obuf = reinterpret_cast<float*>(qbuf + C::QBUF);       // [NC][D][OSTR]   O^T per warp
  float* mlbuf = obuf + NC * D * C::OSTR;                        // [NC][GROWS][2]  (m, l) per warp row
  float* lsebuf = mlbuf + NC * C::GROWS * 2;                     // [ROWS]          combined lse (log2)
  int* flag = reinterpret_cast<int*>(lsebuf + C::ROWS);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(obuf) + C::EPI);
  uint64_t* empty = full + NSTAGE;
  uint64_t* qfull = empty + NSTAGE;
  uint64_t* qempty = qfull + 2;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], NC);
    }
    fence_mbar_init();
  }
  // query rows >= R of both Q slots stay zero for the whole kernel
  for (int i = threadIdx.x; i < 2 * C::ROWS * (D / 8); i += C::THREADS) {
    const int row = i / (D / 8), c = i - row * (D / 8);
    if ((row % C::ROWS) >= p.R) *reinterpret_cast<uint4*>(qbuf + row * C::QSTR + c * 16) = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();

  if (warp == NC) {
    // ============================== producer (one lane) ==============================
    if (lane == 0) {
      prefetch_tmap(&tm.k_full);
      prefetch_tmap(&tm.v_full);
      prefetch_tmap(&tm.k_part);
      prefetch_tmap(&tm.v_part);
      const uint64_t pol = policy_evict_first();
      int it = 0, qi = 0;
#pragma unroll 1
      for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++qi) {
        const int unit = item / p.splits, split = item - unit * p.splits;
        const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
        const int n = __ldg(p.kv_len + b);
        const Ranges rg = cta_ranges(p, n, split);
        // this item's query rows: row r = (t = r / g, head = kvh*g + r % g)
        const int qs = qi & 1;
        mbar_wait(&qempty[qs], ((qi >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qfull[qs], p.R * D * 2);
        for (int r = 0; r < p.R; ++r)
          bulk_load(qbuf + (qs * C::ROWS + r) * C::QSTR,
                    p.q + ((int64_t)(b * p.T + r / p.g) * p.Hq + kvh * p.g + r % p.g) * D, D * 2, &qfull[qs]);
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {
          const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
#pragma unroll 1
          for (int pos = rs; pos < re; pos += TK, ++it) {
            const int stage = it % NSTAGE;
            mbar_wait(&empty[stage], ((it / NSTAGE) & 1) ^ 1);
            const int nvalid = min(TK, re - pos);
            uint8_t* kt = smem + stage * C::STAGE;
            uint8_t* vt = kt + C::TILE;
            if (nvalid == TK) {  // full tile: one TK-row box per 128-byte column slab
              mbar_arrive_expect_tx(&full[stage], C::STAGE);
              for (int sub = 0; sub < C::SUB; ++sub) {
                tma_load_4d(kt + sub * TK * 128, &tm.k_full, &full[stage], sub * 64, pos, kvh, b, pol);
                tma_load_4d(vt + sub * TK * 128, &tm.v_full, &full[stage], sub * 64, pos, kvh, b, pol);
              }
            } else {  // ragged end: only the BOX_ROWS-row boxes that hold valid keys
              const int nbox = (nvalid + BOX_ROWS - 1) / BOX_ROWS;
              mbar_arrive_expect_tx(&full[stage], nbox * BOX_ROWS * 128 * C::SUB * 2);
              for (int sub = 0; sub < C::SUB; ++sub)
                for (int bx = 0; bx < nbox; ++bx) {
                  const int off = sub * TK * 128 + bx * BOX_ROWS * 128;
                  tma_load_4d(kt + off, &tm.k_part, &full[stage], sub * 64, pos + bx * BOX_ROWS, kvh, b, pol);
                  tma_load_4d(vt + off, &tm.v_part, &full[stage], sub * 64, pos + bx * BOX_ROWS, kvh, b, pol);
                }
            }
          }
        }
      }
    }
    return;
  }

  // ============================== consumers ==============================
  const int grp = warp / KS, ks = warp - grp * KS;
  const int gq = lane >> 2, cq = lane & 3;  // fragment row group / column quad
  const int row0 = grp * C::GROWS;          // first query row of this warp's group
  const uint32_t ring = smem_u32(smem);
  const uint32_t qring = smem_u32(qbuf);
  int it = 0, qi = 0;
#pragma unroll 1
  for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++qi) {
    const int unit = item / p.splits, split = item - unit * p.splits;
    const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
    const int n = __ldg(p.kv_len + b);
    const Ranges rg = cta_ranges(p, n, split);
    // causal limit of the two rows this thread holds per n8 tile (verify): key j visible
    // iff j <= n - T + t(row); rows past R get the limit of row R-1 (their output is dropped)
    int lim[NTW][2];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        lim[nt][j] = (p.mode == MODE_VERIFY) ? n - p.T + min(row0 + nt * 8 + 2 * cq + j, p.R - 1) / p.g
                                             : 0x7fffffff;
    // Q^T fragments (B operand): qb[nt][kk][0..1] = Q[row0 + nt*8 + gq][kk*16 + 2cq (+8) ..]
    uint32_t qb[NTW][MD16][2];
    {
      const int qs = qi & 1;
      mbar_wait(&qfull[qs], (qi >> 1) & 1);
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) {
        const uint32_t qrow = qring + (qs * C::ROWS + row0 + nt * 8 + (lane & 7)) * C::QSTR + (lane >> 3) * 16;
#pragma unroll
        for (int kk = 0; kk < MD16; kk += 2)
          ldsm_x4(qrow + kk * 32, qb[nt][kk][0], qb[nt][kk][1], qb[nt][kk + 1][0], qb[nt][kk + 1][1]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
    }

    float o[MD16][NTW][4];
#pragma unroll
    for (int i = 0; i < MD16; ++i)
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) o[i][nt][0] = o[i][nt][1] = o[i][nt][2] = o[i][nt][3] = 0.f;
    float m[NTW][2], l[NTW][2];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) m[nt][0] = m[nt][1] = -INFINITY, l[nt][0] = l[nt][1] = 0.f;

#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
#pragma unroll 1
      for (int pos = rs; pos < re; pos += TK, ++it) {
        const int stage = it % NSTAGE;
        mbar_wait(&full[stage], (it / NSTAGE) & 1);
        const int nvalid = min(TK, re - pos);
        const int kw0 = ks * KW;
        if (kw0 < nvalid) {
          const uint32_t kt = ring + stage * C::STAGE;
          const uint32_t vt = kt + C::TILE;
          // ---------------- S^T = K Q^T : KB blocks of 16 keys x NTW n8 row tiles
          float s[KB][NTW][4];
#pragma unroll
          for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) s[kb][nt][0] = s[kb][nt][1] = s[kb][nt][2] = s[kb][nt][3] = 0.f;
#pragma unroll
          for (int kk = 0; kk < MD16; ++kk) {
            const int chunk = kk * 2 + (lane >> 4);
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              const int key = kw0 + kb * 16 + (lane & 15);
              uint32_t a[4];
              ldsm_x4(kt + (chunk >> 3) * (TK * 128) + swz128(key, chunk & 7), a[0], a[1], a[2], a[3]);
#pragma unroll
              for (int nt = 0; nt < NTW; ++nt) mma_bf16_16816(s[kb][nt], a, qb[nt][kk][0], qb[nt][kk][1]);
            }
          }
          // ---------------- scale, mask, online softmax (log2 domain); rows 2cq, 2cq+1 per n8 tile
          const bool need_mask = (kw0 + KW > nvalid) || (pos + kw0 + KW - 1 > lim[0][0]);
          float corr[NTW][2];
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) {
            float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int kb = 0; kb < KB; ++kb)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float v = s[kb][nt][e] * p.scale_log2;
                if (need_mask) {
                  const int ko = kw0 + kb * 16 + gq + ((e >> 1) << 3);
                  if (ko >= nvalid || pos + ko > lim[nt][e & 1]) v = -INFINITY;
                }
                s[kb][nt][e] = v;
                mx[e & 1] = fmaxf(mx[e & 1], v);
              }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 4));
              mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 8));
              mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 16));
              const float mn = fmaxf(m[nt][j], mx[j]);
              const float base = (mn == -INFINITY) ? 0.f : mn;
              corr[nt][j] = ex2(m[nt][j] - base);
              m[nt][j] = mn;
              float rs = 0.f;
#pragma unroll
              for (int kb = 0; kb < KB; ++kb) {
                s[kb][nt][j] = ex2(s[kb][nt][j] - base);
                s[kb][nt][j + 2] = ex2(s[kb][nt][j + 2] - base);
                rs += s[kb][nt][j] + s[kb][nt][j + 2];
              }
              l[nt][j] = l[nt][j] * corr[nt][j] + rs;
            }
          }
          bool rescale = false;
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) rescale |= (corr[nt][0] != 1.f) | (corr[nt][1] != 1.f);
          if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
            for (int i = 0; i < MD16; ++i)
#pragma unroll
              for (int nt = 0; nt < NTW; ++nt) {
                o[i][nt][0] *= corr[nt][0];
                o[i][nt][1] *= corr[nt][1];
                o[i][nt][2] *= corr[nt][0];
                o[i][nt][3] *= corr[nt][1];
              }
          }
          // ---------------- O^T += V^T P^T
          const bool sanitize = kw0 + KW > nvalid;
#pragma unroll
          for (int kb = 0; kb < KB; ++kb) {
            // P^T B fragments: transpose the bf16-packed S^T fragments (keys gq/gq+8 x rows 2cq..)
            uint32_t pb[NTW][2];
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) {
              pb[nt][0] = movmatrix_t(pack_bf16(s[kb][nt][0], s[kb][nt][1]));
              pb[nt][1] = movmatrix_t(pack_bf16(s[kb][nt][2], s[kb][nt][3]));
            }
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
#pragma unroll
              for (int nt = 0; nt < NTW; ++nt) mma_bf16_16816(o[i][nt], a, pb[nt][0], pb[nt][1]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      }
    }

    // ============================== item epilogue ==============================
    // full row sums: reduce over the 8 lanes sharing cq (they hold different keys)
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        l[nt][j] += __shfl_xor_sync(0xffffffffu, l[nt][j], 4);
        l[nt][j] += __shfl_xor_sync(0xffffffffu, l[nt][j], 8);
        l[nt][j] += __shfl_xor_sync(0xffffffffu, l[nt][j], 16);
      }
    if (gq == 0) {
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          mlbuf[(warp * C::GROWS + nt * 8 + 2 * cq + j) * 2 + 0] = m[nt][j];
          mlbuf[(warp * C::GROWS + nt * 8 + 2 * cq + j) * 2 + 1] = l[nt][j];
        }
    }
    named_bar_sync(1, NC * 32);
    // scale this warp's O^T by 2^(m_w - M) / L where (M, L) combine the KS key slices
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) {
      float f[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int rl = nt * 8 + 2 * cq + j;  // row within the group
        float M = -INFINITY;
#pragma unroll
        for (int k = 0; k < KS; ++k) M = fmaxf(M, mlbuf[((grp * KS + k) * C::GROWS + rl) * 2]);
        float L = 0.f;
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          const float* e = &mlbuf[((grp * KS + k) * C::GROWS + rl) * 2];
          if (e[1] > 0.f) L += e[1] * ex2(e[0] - M);
        }
        f[j] = (l[nt][j] > 0.f) ? ex2(m[nt][j] - M) / L : 0.f;
        if (ks == 0 && gq == 0) lsebuf[row0 + rl] = (L > 0.f) ? M + __log2f(L) : -INFINITY;
      }
#pragma unroll
      for (int i = 0; i < MD16; ++i) {
        float* ob = obuf + (size_t)warp * D * C::OSTR;
        const int d0 = i * 16 + gq, r0 = nt * 8 + 2 * cq;
        ob[d0 * C::OSTR + r0] = o[i][nt][0] * f[0];
        ob[d0 * C::OSTR + r0 + 1] = o[i][nt][1] * f[1];
        ob[(d0 + 8) * C::OSTR + r0] = o[i][nt][2] * f[0];
        ob[(d0 + 8) * C::OSTR + r0 + 1] = o[i][nt][3] * f[1];
      }
    }
    named_bar_sync(1, NC * 32);
    // sum the KS slices; write the final rows (one split) or this split's partial rows
    const bool final_out = (p.splits == 1);
    for (int idx = threadIdx.x; idx < p.R * D; idx += NC * 32) {
      const int r = idx / D, dd = idx - r * D;
      const int g2 = r / C::GROWS, rl = r - g2 * C::GROWS;
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < KS; ++k) acc += obuf[((size_t)(g2 * KS + k) * D + dd) * C::OSTR + rl];
      const float lse2 = lsebuf[r];
      if (final_out) {
        const int64_t orow = (int64_t)(b * p.T + r / p.g) * p.Hq + kvh * p.g + r % p.g;
        p.out[orow * D + dd] = acc;
        if (dd == 0 && p.lse != nullptr) p.lse[orow] = lse2 * LN2;
      } else {
        const int64_t prow = ((int64_t)unit * p.splits + split) * p.R + r;
        __stcg(p.ws_o + prow * D + dd, acc);
        if (dd == 0) __stcg(p.ws_lse + prow, lse2);
      }
    }
    if (!final_out) {
      // ---- fused split merge: the last CTA to finish a unit combines its splits (O6 identity).
      // bar.sync orders every thread's partial stores before thread 0's release-add; the
      // acq_rel atomic of the last arriver makes all splits' stores visible to its CTA.
      named_bar_sync(1, NC * 32);
      if (threadIdx.x == 0) {
        const int old = atomic_add_acq_rel_gpu(p.counters + unit, 1);
        const int last = (old == p.splits - 1);
        if (last) p.counters[unit] = 0;  // leave the workspace ready for the next call
        *flag = last;
      }
      named_bar_sync(1, NC * 32);
      if (*flag) {
        float* wts = obuf;  // [R][splits] merge weights (obuf is free after the barrier above)
        const float* lsep = p.ws_lse + (int64_t)unit * p.splits * p.R;
        for (int r = threadIdx.x; r < p.R; r += NC * 32) {
          float M = -INFINITY;
          for (int s2 = 0; s2 < p.splits; ++s2) M = fmaxf(M, __ldcg(lsep + s2 * p.R + r));
          float W = 0.f;
          for (int s2 = 0; s2 < p.splits; ++s2) {
            const float ls = __ldcg(lsep + s2 * p.R + r);
            const float w = (ls == -INFINITY) ? 0.f : ex2(ls - M);
            wts[r * p.splits + s2] = w;
            W += w;
          }
          const float inv = W > 0.f ? 1.f / W : 0.f;
          for (int s2 = 0; s2 < p.splits; ++s2) wts[r * p.splits + s2] *= inv;
          lsebuf[r] = (W > 0.f) ? M + __log2f(W) : -INFINITY;
        }
        named_bar_sync(1, NC * 32);
        constexpr int V4 = D / 4;
        for (int idx = threadIdx.x; idx < p.R * V4; idx += NC * 32) {
          const int r = idx / V4, c4 = (idx - r * V4) * 4;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int s2 = 0; s2 < p.splits; ++s2) {
            const float w = wts[r * p.splits + s2];
            if (w == 0.f) continue;
            const float4 v = __ldcg(
                reinterpret_cast<const float4*>(p.ws_o + (((int64_t)unit * p.splits + s2) * p.R + r) * D + c4));
            acc.x += w * v.x;
            acc.y += w * v.y;
            acc.z += w * v.z;
            acc.w += w * v.w;
          }
          const int64_t orow = (int64_t)(b * p.T + r / p.g) * p.Hq + kvh * p.g + r % p.g;
          *reinterpret_cast<float4*>(p.out + orow * D + c4) = acc;
          if (c4 == 0 && p.lse != nullptr) p.lse[orow] = lsebuf[r] * LN2;
        }
      }
    }
    named_bar_sync(1, NC * 32);  // the epilogue buffers are reused by the next item
  }
}

// ------------------------------------------------------------------------------ host side
struct Plan {
  bool keys = false;  // attn_keys_kernel (persistent, R <= 8) or attn_rows_kernel
  int splits = 1, chunk = TK, items = 0, grid = 0;
};

constexpr int ROWS_CTAS_PER_SM = 2;

static int forced_splits() {  // tuning knob for experiments: MD_SPLITS=<n>
  static const int v = [] {
    const char* e = getenv("MD_SPLITS");
    return e ? atoi(e) : 0;
  }();
  return v;
}

static void set_splits(Plan& pl, int tiles, int s) {
  const int chunk_tiles = (tiles + s - 1) / s;
  pl.splits = (tiles + chunk_tiles - 1) / chunk_tiles;
  pl.chunk = chunk_tiles * TK;
}

// rows kernel: one CTA per item, 2 resident per SM.  Splits per unit are chosen so the
// items fill whole waves: efficiency = W / ceil(W), W = items / (SMs * 2); ties (within
// 2%) go to fewer splits, and a split keeps >= 4 tiles so merge traffic stays ~1%.
// keys kernel: persistent, one CTA per SM; one split per unit unless there are fewer
// units than SMs (a split costs a cross-CTA release/acquire in the fused merge).
static Plan plan_attention(int units, int R, int max_keys, int sm_count) {
  Plan pl;
  pl.keys = R <= 8;
  const int tiles = max(1, (max_keys + TK - 1) / TK);
  const int max_splits = max(1, min(32, tiles / 4));
  if (forced_splits() > 0) {
    set_splits(pl, tiles, min(forced_splits(), tiles));
  } else if (pl.keys) {
    set_splits(pl, tiles, min(max_splits, max(1, sm_count / units)));
  } else {
    const int slots = sm_count * ROWS_CTAS_PER_SM;
    double best = -1.0;
    for (int s = 1; s <= max_splits; ++s) {
      const int chunk_tiles = (tiles + s - 1) / s;
      if ((tiles + chunk_tiles - 1) / chunk_tiles != s) continue;
      const double w = static_cast<double>(units) * s / slots;
      const double eff = w / std::ceil(w);
      if (eff > best + 0.02) {
        best = eff;
        set_splits(pl, tiles, s);
      }
    }
  }
  pl.items = units * pl.splits;
  pl.grid = pl.keys ? min(pl.items, sm_count) : pl.items;
  return pl;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// [partials fp32 units*splits*R*D][partial lse fp32 units*splits*R][counters int32 units]
static size_t workspace_for(const Plan& pl, int units, int R, int D) {
  if (pl.splits <= 1) return 0;
  return align256((size_t)units * pl.splits * R * D * 4) + align256((size_t)units * pl.splits * R * 4) +
         align256((size_t)units * 4);
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
  constexpr int smem = SmemLayout<D>::TOTAL;
  static int done = -1;
  md_status st = set_smem(kern, smem, &done);
  if (st != MD_OK) return st;
  kern<<<grid, (MT * KS + 1) * 32, smem, s>>>(tm, p);
  return check_launch("attn_rows_kernel");
}

template <int D, int NTW, int NG, int KS>
static md_status launch_keys(const TmapSet& tm, const AttnParams& p, int grid, cudaStream_t s) {
  using C = KCfg<D, NTW, NG, KS>;
  auto kern = attn_keys_kernel<D, NTW, NG, KS>;
  static int done = -1;
  md_status st = set_smem(kern, C::SMEM, &done);
  if (st != MD_OK) return st;
  kern<<<grid, C::THREADS, C::SMEM, s>>>(tm, p);
  return check_launch("attn_keys_kernel");
}

template <int D>
static md_status launch_dim(const TmapSet& tm, const AttnParams& p, const Plan& pl, cudaStream_t s) {
  if (pl.keys) return launch_keys<D, 1, 1, 4>(tm, p, pl.grid, s);
  switch ((p.R + 15) / 16) {
    case 1: return launch_rows<D, 1, 4>(tm, p, pl.grid, s);
    case 2: return launch_rows<D, 2, 2>(tm, p, pl.grid, s);
    case 3: return launch_rows<D, 3, 1>(tm, p, pl.grid, s);
    case 4: return launch_rows<D, 4, 1>(tm, p, pl.grid, s);
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

static md_status run_attention(const md_kv_cache* c, const void* q, int Hq, int T, const int32_t* kv_len,
                               int max_keys, int sink, int window, int mode, float scale, float* out, float* lse,
                               void* ws, size_t ws_bytes, cudaStream_t s, const char* who) {
  md_status st = check_cache(c, who);
  if (st != MD_OK) return st;
  MD_REQUIRE(q != nullptr && kv_len != nullptr && out != nullptr, MD_ERR_INVALID_ARG, "%s: NULL q/kv_len/out", who);
  MD_REQUIRE(Hq >= 1 && Hq % c->num_kv_heads == 0, MD_ERR_INVALID_ARG, "%s: num_q_heads must be a multiple of Hkv",
             who);
  MD_REQUIRE(aligned16(q) && aligned16(out), MD_ERR_INVALID_ARG, "%s: q and out must be 16-byte aligned", who);
  const int g = Hq / c->num_kv_heads;
  const int R = g * T;
  MD_REQUIRE(R <= 64, MD_ERR_UNSUPPORTED, "%s: g*T = %d > 64 query rows per KV head is not supported", who, R);
  const int units = c->batch * c->num_kv_heads;
  const Plan pl = plan_attention(units, R, max_keys, device_sm_count());
  const size_t need = workspace_for(pl, units, R, c->head_dim);
  MD_REQUIRE(ws_bytes >= need && (need == 0 || ws != nullptr), MD_ERR_WORKSPACE,
             "%s: workspace of %zu bytes required, %zu given", who, need, ws_bytes);
  TmapSet tm;
  if ((st = make_tmap(&tm.k_full, c, c->k, TK)) != MD_OK || (st = make_tmap(&tm.v_full, c, c->v, TK)) != MD_OK ||
      (st = make_tmap(&tm.k_part, c, c->k, BOX_ROWS)) != MD_OK || (st = make_tmap(&tm.v_part, c, c->v, BOX_ROWS)) != MD_OK)
    return st;
  AttnParams p{};
  p.q = static_cast<const uint16_t*>(q);
  p.out = out;
  p.lse = lse;
  p.kv_len = kv_len;
  p.Hq = Hq;
  p.Hkv = c->num_kv_heads;
  p.T = T;
  p.g = g;
  p.R = R;
  p.splits = pl.splits;
  p.chunk = pl.chunk;
  p.sink = sink;
  p.window = window;
  p.mode = mode;
  p.scale_log2 = scale * LOG2E;
  p.items = pl.items;
  if (pl.splits > 1) {
    uint8_t* w = static_cast<uint8_t*>(ws);
    p.ws_o = reinterpret_cast<float*>(w);
    w += align256((size_t)units * pl.splits * R * c->head_dim * 4);
    p.ws_lse = reinterpret_cast<float*>(w);
    w += align256((size_t)units * pl.splits * R * 4);
    p.counters = reinterpret_cast<int*>(w);
  }
  st = (c->head_dim == 128) ? launch_dim<128>(tm, p, pl, s) : launch_dim<64>(tm, p, pl, s);
  if (st != MD_OK || pl.keys || pl.splits == 1) return st;
  const int warps = units * R;
  const int blocks = (warps * 32 + 255) / 256;
  if (c->head_dim == 128)
    attn_merge_kernel<128><<<blocks, 256, 0, s>>>(p, units);
  else
    attn_merge_kernel<64><<<blocks, 256, 0, s>>>(p, units);
  return check_launch("attn_merge_kernel");
}

}  // namespace md

extern "C" size_t md_attn_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads, int32_t head_dim,
                                          int32_t T, int32_t max_kv_len) {
  using namespace md;
  if (batch < 1 || num_kv_heads < 1 || num_q_heads < 1 || num_q_heads % num_kv_heads || T < 1 || max_kv_len < 1 ||
      (head_dim != 64 && head_dim != 128))
    return 0;
  const int R = (num_q_heads / num_kv_heads) * T;
  const int units = batch * num_kv_heads;
  return workspace_for(plan_attention(units, R, max_kv_len, device_sm_count()), units, R, head_dim);
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
  return run_attention(cache, q, num_q_heads, T, kv_len, max_kv_len, 0, 0, MODE_VERIFY, scale, out, lse, workspace,
                       workspace_bytes, (cudaStream_t)stream, "md_verify_attn_full");
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
  const int64_t budget = (int64_t)sink + window;
  const int max_keys = static_cast<int>(budget < cache->capacity ? budget : cache->capacity);
  return run_attention(cache, q, num_q_heads, 1, kv_len, max_keys, sink, window, MODE_DRAFT, scale, out, lse,
                       workspace, workspace_bytes, (cudaStream_t)stream, "md_draft_attn_sparse");
}

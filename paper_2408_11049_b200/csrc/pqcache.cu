// pqcache.cu — md_pq_encode, md_pq_workspace_bytes, md_pq_select: PQCache-style dynamic KV
// selection for self-speculative drafting (P:1141 footnote "PQCache
// employs product quantization with 16 sub-vectors and 8-bit quantization per key vector";
// dynamic methods search the cache for every query, at a batch-dependent cost
// T_select, Eq.3).  The selected index list drives md_draft_attn_indexed.
//
// Per unit (b, kv head):
//   pq_encode_kernel  (prefill / lazily for rows leaving the window) code[j][m] = nearest of
//                     256 centroids of sub-space m, fp32 distance left to right, no FMA;
//   pq_lut_kernel     the group's query heads folded into one table lut[16][256] (fp32,
//                     no FMA), scaled by 2^e (max |lut| < 2^26) and rounded to int32;
//   pq_score_kernel   score[j] = sum_m lutq[m][code[j][m]]: one 16-byte code per key and
//                     thread, 16 table lookups from shared memory laid out so the 32 lanes
//                     of a warp always hit 32 different banks (lane l reads sub-space
//                     (i ^ l) & 15 at step i, from copy l >> 4 of the table, and table m
//                     lives in bank m (copy 0) / 16 + m (copy 1));
//   pq_select_kernel  top-c of [s0, tail) by score (ties -> lower position): 4-pass 8-bit
//                     radix select on order-preserving uint32 keys, then an ordered
//                     compaction over per-thread contiguous runs (two block scans); the
//                     candidate scores are staged in shared memory when they fit.
// Integer scores make every selection decision exact and independent of summation order, so
// the index lists equal the oracle's bit for bit (oracle/pqcache.py P1-P5).
#include <cuda.h>

#include <cmath>

#include "md_common.cuh"
#include "md_internal.h"

namespace md {
namespace pq {

constexpr int M = 16;      // sub-vectors per key
constexpr int NC = 256;    // centroids per sub-space (8-bit codes)
constexpr int SCORE_CH = 4096;   // keys per score CTA
constexpr int SCORE_THREADS = 256;
constexpr int SEL_THREADS = 1024;
constexpr int SEL_SMEM_MAX = 49152;  // candidate scores staged in smem up to this count

__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }

// ------------------------------------------------------------------ P1 encode
// grid (units, 16 sub-spaces), 256 threads; centroids of (unit, m) in smem as fp32.
template <int S>
__global__ void __launch_bounds__(256) pq_encode_kernel(const uint16_t* __restrict__ k, int64_t sB, int64_t sH,
                                                        int64_t sS, int Hkv, const uint16_t* __restrict__ cb,
                                                        const int32_t* __restrict__ start, int count,
                                                        uint8_t* __restrict__ codes, int code_cap) {
  __shared__ float cent[NC * S];
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x, m = blockIdx.y;
  const int b = unit / Hkv, u = unit - b * Hkv;
  const uint16_t* cbm = cb + ((size_t)unit * M + m) * NC * S;
  for (int i = threadIdx.x; i < NC * S; i += blockDim.x) cent[i] = bf16_to_f32(cbm[i]);
  __syncthreads();
  const int s0 = __ldg(start + b);
  const uint16_t* krow = k + (int64_t)b * sB + (int64_t)u * sH + m * S;
  uint8_t* crow = codes + (size_t)unit * code_cap * M + m;
  for (int t = threadIdx.x; t < count; t += blockDim.x) {
    const int pos = s0 + t;
    float x[S];
    const uint16_t* src = krow + (int64_t)pos * sS;
    if constexpr (S == 8) {
      const uint4 w = *reinterpret_cast<const uint4*>(src);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[2 * i] = __uint_as_float(ws[i] << 16);
        x[2 * i + 1] = __uint_as_float(ws[i] & 0xffff0000u);
      }
    } else {
      const uint2 w = *reinterpret_cast<const uint2*>(src);
      const uint32_t ws[2] = {w.x, w.y};
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        x[2 * i] = __uint_as_float(ws[i] << 16);
        x[2 * i + 1] = __uint_as_float(ws[i] & 0xffff0000u);
      }
    }
    float best = INFINITY;
    int arg = 0;
#pragma unroll 4
    for (int c = 0; c < NC; ++c) {
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const float dlt = __fsub_rn(x[i], cent[c * S + i]);
        acc = __fadd_rn(acc, __fmul_rn(dlt, dlt));
      }
      if (acc < best) {  // strict: ties keep the lowest index
        best = acc;
        arg = c;
      }
    }
    crow[(size_t)pos * M] = static_cast<uint8_t>(arg);
  }
}

// ------------------------------------------------------------------ P2 + P3 lookup table
// grid units, 256 threads: thread c computes lut[m][c] for all 16 m.
template <int S>
__global__ void __launch_bounds__(256) pq_lut_kernel(const uint16_t* __restrict__ q, int Hq, int Hkv,
                                                     const uint16_t* __restrict__ cb, int32_t* __restrict__ lutq) {
  constexpr int D = S * M;
  extern __shared__ float qs[];  // [g][D]
  __shared__ float red[8];
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x, g = Hq / Hkv;
  const int b = unit / Hkv, u = unit - b * Hkv;
  const uint16_t* qg = q + ((size_t)b * Hq + (size_t)u * g) * D;
  for (int i = threadIdx.x; i < g * D; i += blockDim.x) qs[i] = bf16_to_f32(qg[i]);
  __syncthreads();
  const int c = threadIdx.x;
  const uint16_t* cbu = cb + (size_t)unit * M * NC * S;
  float lut[M];
  float mx = 0.f;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    float cen[S];
    const uint16_t* src = cbu + ((size_t)m * NC + c) * S;
#pragma unroll
    for (int i = 0; i < S; ++i) cen[i] = bf16_to_f32(src[i]);
    float acc = 0.f;
    for (int hh = 0; hh < g; ++hh) {
#pragma unroll
      for (int i = 0; i < S; ++i) acc = __fadd_rn(acc, __fmul_rn(qs[hh * D + m * S + i], cen[i]));
    }
    lut[m] = acc;
    mx = fmaxf(mx, fabsf(acc));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  int e = 0;
  if (mx > 0.f) {
    int E;
    frexpf(mx, &E);
    e = 26 - E;
  }
  int32_t* dst = lutq + (size_t)unit * M * NC;
#pragma unroll
  for (int m = 0; m < M; ++m) dst[m * NC + c] = __float2int_rn(ldexpf(lut[m], e));
}

// ------------------------------------------------------------------ P4 scores
// grid (units, chunks of SCORE_CH keys); scores of the candidates [s0, tail) only.
__global__ void __launch_bounds__(SCORE_THREADS) pq_score_kernel(const uint8_t* __restrict__ codes, int code_cap,
                                                                 const int32_t* __restrict__ lutq,
                                                                 const int32_t* __restrict__ kv_len, int Hkv, int sink,
                                                                 int window, int32_t* __restrict__ scores,
                                                                 int score_stride) {
  // tab[c * 32 + copy * 16 + m] = lutq[m][c]: table m in bank m (copy 0) / 16 + m (copy 1)
  __shared__ int32_t tab[NC * 32];
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x;
  const int b = unit / Hkv;
  const int n = __ldg(kv_len + b);
  const int s0 = min(sink, n), tail = max(s0, n - window);
  const int lo = max(s0, (int)blockIdx.y * SCORE_CH), hi = min(tail, (int)(blockIdx.y + 1) * SCORE_CH);
  if (lo >= hi) return;  // uniform
  const int32_t* src = lutq + (size_t)unit * M * NC;
  for (int i = threadIdx.x; i < M * NC; i += blockDim.x) {
    const int m = i / NC, c = i - m * NC;
    const int32_t v = __ldg(src + i);
    tab[c * 32 + m] = v;
    tab[c * 32 + 16 + m] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int l15 = lane & 15;
  const uint32_t tbase = smem_u32(tab) + ((lane >> 4) << 6);  // copy (lane >> 4): +16 words
  // per-lane constant part of the address of step i: ((i ^ l15) << 2), sub-space m = i ^ l15
  uint32_t off[M];
#pragma unroll
  for (int i = 0; i < M; ++i) off[i] = tbase + (uint32_t)((i ^ l15) << 2);
  // the byte of sub-space (i ^ l15) sits in word ((i >> 2) ^ q) at byte ((i & 3) ^ r)
  const int qx = l15 >> 2, rx = l15 & 3;
  const uint4* crow = reinterpret_cast<const uint4*>(codes + (size_t)unit * code_cap * M);
  int32_t* out = scores + (size_t)unit * score_stride;
  for (int j = lo + threadIdx.x; j < hi; j += SCORE_THREADS) {
    const uint4 w4 = __ldcs(crow + j);  // streamed once
    uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
    // word permutation w'[i] = w[i ^ qx] (two conditional swap stages)
    if (qx & 1) {
      uint32_t t = w[0]; w[0] = w[1]; w[1] = t;
      t = w[2]; w[2] = w[3]; w[3] = t;
    }
    if (qx & 2) {
      uint32_t t = w[0]; w[0] = w[2]; w[2] = t;
      t = w[1]; w[1] = w[3]; w[3] = t;
    }
    int32_t acc = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const uint32_t code = (w[i >> 2] >> (((i & 3) ^ rx) << 3)) & 0xffu;
      int32_t v;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(off[i] + (code << 7)));
      acc += v;
    }
    out[j] = acc;
  }
}

// ------------------------------------------------------------------ P5 selection
__device__ __forceinline__ uint32_t okey(int32_t s) { return static_cast<uint32_t>(s) ^ 0x80000000u; }

// exclusive block scan of one value per thread (SEL_THREADS threads)
__device__ __forceinline__ uint32_t sel_excl_scan(uint32_t v, uint32_t* sm, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) sm[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t x = sm[lane];  // SEL_THREADS / 32 == 32 warps
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    sm[32 + lane] = xi - x;
    if (lane == 31) sm[64] = xi;
  }
  __syncthreads();
  total = sm[64];
  const uint32_t r = sm[32 + warp] + incl - v;
  __syncthreads();
  return r;
}

// padded smem index: run-contiguous reads by thread t (positions t*R + k) are conflict-free
__device__ __forceinline__ int pad_idx(int i) { return i + (i >> 5); }

template <bool SMEM>
__global__ void __launch_bounds__(SEL_THREADS) pq_select_kernel(const int32_t* __restrict__ scores, int score_stride,
                                                                const int32_t* __restrict__ kv_len, int Hkv, int sink,
                                                                int window, int budget, int32_t* __restrict__ idx,
                                                                int idx_stride, int32_t* __restrict__ idx_count,
                                                                int32_t* __restrict__ tail_start) {
  extern __shared__ uint32_t sel_sm[];  // staged keys (SMEM) — padded
  __shared__ uint32_t hist[256];
  __shared__ uint32_t scan_sm[65];
  __shared__ uint32_t s_prefix, s_need;
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x;
  const int b = unit / Hkv, u = unit - b * Hkv;
  const int n = __ldg(kv_len + b);
  const int s0 = min(sink, n), tail = max(s0, n - window);
  const int cnt = tail - s0;
  const int c = min(budget, cnt);
  int32_t* out = idx + (size_t)unit * idx_stride;
  if (u == 0 && threadIdx.x == 0) {
    idx_count[b] = s0 + c;
    tail_start[b] = tail;
  }
  for (int j = threadIdx.x; j < s0; j += SEL_THREADS) out[j] = j;
  if (c == 0) return;
  out += s0;
  if (c == cnt) {  // the budget covers every candidate
    for (int j = threadIdx.x; j < cnt; j += SEL_THREADS) out[j] = s0 + j;
    return;
  }
  const int32_t* sc = scores + (size_t)unit * score_stride + s0;
  if constexpr (SMEM) {
    for (int j = threadIdx.x; j < cnt; j += SEL_THREADS) sel_sm[pad_idx(j)] = okey(__ldcg(sc + j));
    __syncthreads();
  }
  auto key_at = [&](int j) -> uint32_t {
    if constexpr (SMEM) return sel_sm[pad_idx(j)];
    else return okey(__ldcg(sc + j));
  };
  // radix select of the c-th largest key
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_need = c;
  }
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += SEL_THREADS) hist[i] = 0;
    __syncthreads();
    const uint32_t pre = s_prefix;
    const uint32_t mask = (shift == 24) ? 0u : (0xffffffffu << (shift + 8));
    for (int j = threadIdx.x; j < cnt; j += SEL_THREADS) {
      const uint32_t kk = key_at(j);
      if ((kk & mask) == (pre & mask)) {
        const uint32_t bin = (kk >> shift) & 255u;
        // aggregate equal bins within the warp: one shared atomic per distinct bin
        const unsigned act = __activemask();
        const unsigned peers = __match_any_sync(act, bin);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // warp 0 finds the bin holding the need-th largest: suffix sums over 8 bins per lane
      const int lane = threadIdx.x;
      uint32_t cnt8 = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) cnt8 += hist[lane * 8 + t];
      // inclusive suffix sum over lanes (lane 31 holds the top bins)
      uint32_t suf = cnt8;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += t;
      }
      const uint32_t need = s_need;
      const uint32_t above = suf - cnt8;  // keys in higher lanes' bins
      if (above < need && suf >= need) {  // exactly one lane
        uint32_t acc = above;
        int bin = lane * 8 + 7;
        for (; bin > lane * 8; --bin) {
          if (acc + hist[bin] >= need) break;
          acc += hist[bin];
        }
        s_prefix = pre | ((uint32_t)bin << shift);
        s_need = need - acc;  // how many of the keys equal to the final threshold to take
      }
    }
    __syncthreads();
  }
  const uint32_t thr = s_prefix, take_eq = s_need;
  // ordered compaction: thread t owns the contiguous run [t*RL, (t+1)*RL)
  const int RL = (cnt + SEL_THREADS - 1) / SEL_THREADS;
  const int r0 = threadIdx.x * RL, r1 = min(cnt, r0 + RL);
  uint32_t n_gt = 0, n_eq = 0;
  for (int j = r0; j < r1; ++j) {
    const uint32_t kk = key_at(j);
    n_gt += kk > thr;
    n_eq += kk == thr;
  }
  uint32_t tot_eq, tot_gt;
  const uint32_t eq_before = sel_excl_scan(n_eq, scan_sm, tot_eq);
  // selected before this run: all greater keys before + the equal keys before that are taken
  const uint32_t gt_before = sel_excl_scan(n_gt, scan_sm, tot_gt);
  uint32_t pos = gt_before + min(eq_before, take_eq);
  uint32_t eq_rank = eq_before;
  for (int j = r0; j < r1; ++j) {
    const uint32_t kk = key_at(j);
    bool take = kk > thr;
    if (kk == thr) {
      take = eq_rank < take_eq;
      ++eq_rank;
    }
    if (take) out[pos++] = s0 + j;
  }
}

}  // namespace pq

static size_t pq_align(size_t x) { return (x + 255) & ~size_t(255); }
static size_t pq_ws(int B, int Hkv, int maxL) {
  const size_t units = (size_t)B * Hkv;
  return pq_align(units * pq::M * pq::NC * 4) + pq_align(units * (size_t)maxL * 4);
}

}  // namespace md

extern "C" MD_API md_status md_pq_encode(const md_kv_cache* c, const void* codebook, const int32_t* start_pos,
                                         int32_t count, uint8_t* codes, int32_t code_capacity, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(c != nullptr && c->k != nullptr && codebook != nullptr && start_pos != nullptr && codes != nullptr,
             MD_ERR_INVALID_ARG, "md_pq_encode: NULL argument");
  MD_REQUIRE(c->head_dim == 64 || c->head_dim == 128, MD_ERR_UNSUPPORTED, "md_pq_encode: head_dim must be 64/128");
  MD_REQUIRE(c->batch >= 1 && c->num_kv_heads >= 1 && count >= 0 && code_capacity >= 1, MD_ERR_INVALID_ARG,
             "md_pq_encode: bad batch / heads / count / code_capacity");
  MD_REQUIRE(c->stride_s % 8 == 0 && c->stride_h % 8 == 0 && c->stride_b % 8 == 0 && aligned16(c->k) &&
                 aligned16(codebook),
             MD_ERR_INVALID_ARG, "md_pq_encode: 16-byte alignment of cache rows and codebook required");
  if (count == 0) return MD_OK;
  const dim3 grid((unsigned)(c->batch * c->num_kv_heads), pq::M);
  cudaStream_t s = (cudaStream_t)stream;
  const auto* k = static_cast<const uint16_t*>(c->k);
  const auto* cb = static_cast<const uint16_t*>(codebook);
  if (c->head_dim == 128)
    launch_pdl(pq::pq_encode_kernel<8>, grid, dim3(256), 0, s, k, c->stride_b, c->stride_h, c->stride_s,
               (int)c->num_kv_heads, cb, start_pos, (int)count, codes, (int)code_capacity);
  else
    launch_pdl(pq::pq_encode_kernel<4>, grid, dim3(256), 0, s, k, c->stride_b, c->stride_h, c->stride_s,
               (int)c->num_kv_heads, cb, start_pos, (int)count, codes, (int)code_capacity);
  return check_launch("pq_encode_kernel");
}

extern "C" MD_API size_t md_pq_workspace_bytes(int32_t batch, int32_t num_kv_heads, int32_t max_kv_len) {
  if (batch < 1 || num_kv_heads < 1 || max_kv_len < 1) return 0;
  return md::pq_ws(batch, num_kv_heads, max_kv_len);
}

extern "C" MD_API md_status md_pq_select(const void* q, int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                                         int32_t head_dim, const void* codebook, const uint8_t* codes,
                                         int32_t code_capacity, const int32_t* kv_len, int32_t max_kv_len,
                                         int32_t sink, int32_t window, int32_t budget, int32_t* idx,
                                         int32_t idx_stride, int32_t* idx_count, int32_t* tail_start,
                                         void* workspace, size_t workspace_bytes, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(q != nullptr && codebook != nullptr && codes != nullptr && kv_len != nullptr && idx != nullptr &&
                 idx_count != nullptr && tail_start != nullptr,
             MD_ERR_INVALID_ARG, "md_pq_select: NULL argument");
  MD_REQUIRE(head_dim == 64 || head_dim == 128, MD_ERR_UNSUPPORTED, "md_pq_select: head_dim must be 64/128");
  MD_REQUIRE(batch >= 1 && num_kv_heads >= 1 && num_q_heads >= 1 && num_q_heads % num_kv_heads == 0,
             MD_ERR_INVALID_ARG, "md_pq_select: need num_q_heads a multiple of num_kv_heads >= 1");
  MD_REQUIRE(num_q_heads / num_kv_heads <= 16, MD_ERR_UNSUPPORTED, "md_pq_select: GQA group > 16");
  MD_REQUIRE(sink >= 0 && window >= 0 && budget >= 0 && sink + window >= 1, MD_ERR_INVALID_ARG,
             "md_pq_select: need sink, window, budget >= 0 and sink + window >= 1");
  MD_REQUIRE(idx_stride >= sink + budget, MD_ERR_INVALID_ARG, "md_pq_select: idx_stride < sink + budget");
  MD_REQUIRE(max_kv_len >= 1 && max_kv_len <= code_capacity, MD_ERR_INVALID_ARG,
             "md_pq_select: need 1 <= max_kv_len <= code_capacity");
  MD_REQUIRE(aligned16(codes) && aligned16(codebook), MD_ERR_INVALID_ARG,
             "md_pq_select: codes and codebook must be 16-byte aligned");
  const size_t need = pq_ws(batch, num_kv_heads, max_kv_len);
  MD_REQUIRE(workspace != nullptr && workspace_bytes >= need, MD_ERR_WORKSPACE,
             "md_pq_select: workspace of %zu bytes required, %zu given", need, workspace_bytes);
  const int units = batch * num_kv_heads;
  auto* lutq = static_cast<int32_t*>(workspace);
  auto* scores = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(workspace) + pq_align((size_t)units * pq::M * pq::NC * 4));
  const auto* qq = static_cast<const uint16_t*>(q);
  const auto* cb = static_cast<const uint16_t*>(codebook);
  cudaStream_t s = (cudaStream_t)stream;
  const int g = num_q_heads / num_kv_heads;
  const size_t lut_smem = (size_t)g * head_dim * 4;
  if (head_dim == 128)
    launch_pdl(pq::pq_lut_kernel<8>, dim3(units), dim3(256), lut_smem, s, qq, (int)num_q_heads, (int)num_kv_heads,
               cb, lutq);
  else
    launch_pdl(pq::pq_lut_kernel<4>, dim3(units), dim3(256), lut_smem, s, qq, (int)num_q_heads, (int)num_kv_heads,
               cb, lutq);
  if (md_status st = check_launch("pq_lut_kernel"); st != MD_OK) return st;
  const unsigned chunks = (unsigned)((max_kv_len + pq::SCORE_CH - 1) / pq::SCORE_CH);
  launch_pdl(pq::pq_score_kernel, dim3(units, chunks), dim3(pq::SCORE_THREADS), 0, s, codes, (int)code_capacity,
             (const int32_t*)lutq, kv_len, (int)num_kv_heads, (int)sink, (int)window, scores, (int)max_kv_len);
  if (md_status st = check_launch("pq_score_kernel"); st != MD_OK) return st;
  if (max_kv_len <= pq::SEL_SMEM_MAX) {
    static int done_dev = -1;  // per-process; the attribute call is idempotent (benign race)
    int dev = 0;
    cudaGetDevice(&dev);
    if (done_dev != dev) {
      const size_t smem = (size_t)(pq::SEL_SMEM_MAX + pq::SEL_SMEM_MAX / 32 + 1) * 4;
      if (cudaFuncSetAttribute(pq::pq_select_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return check_launch("cudaFuncSetAttribute");
      done_dev = dev;
    }
    const size_t use = (size_t)(max_kv_len + max_kv_len / 32 + 1) * 4;
    launch_pdl(pq::pq_select_kernel<true>, dim3(units), dim3(pq::SEL_THREADS), use, s, (const int32_t*)scores,
               (int)max_kv_len, kv_len, (int)num_kv_heads, (int)sink, (int)window, (int)budget, idx, (int)idx_stride,
               idx_count, tail_start);
  } else {
    launch_pdl(pq::pq_select_kernel<false>, dim3(units), dim3(pq::SEL_THREADS), 0, s, (const int32_t*)scores,
               (int)max_kv_len, kv_len, (int)num_kv_heads, (int)sink, (int)window, (int)budget, idx, (int)idx_stride,
               idx_count, tail_start);
  }
  return check_launch("pq_select_kernel");
}

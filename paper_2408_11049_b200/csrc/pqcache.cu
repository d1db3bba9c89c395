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
//                     no FMA), one CTA per (unit, 4 sub-spaces), plus their max |lut|;
//                     the score kernel scales it by 2^e (max |lut| < 2^26) and rounds to int32;
//   pq_score_kernel   score[j] = sum_m lutq[m][code[j][m]]: one 16-byte code per key and
//                     thread, 16 table lookups from shared memory laid out so the 32 lanes
//                     of a warp always hit 32 different banks (lane l reads sub-space
//                     (i ^ l) & 15 at step i, from copy l >> 4 of the table, and table m
//                     lives in bank m (copy 0) / 16 + m (copy 1));
//   pq_select_kernel  top-c of [s0, tail) by score (ties -> lower position): radix select
//                     on order-preserving uint32 keys (12 + 10 + 10-bit digits; after the
//                     first pass only the keys of the cutoff bin are kept, in shared
//                     memory), then an ordered compaction over per-thread contiguous runs
//                     (two block scans).  The scores are read from L2.
// Integer scores make every selection decision exact and independent of summation order, so
// the index lists equal the oracle's bit for bit (oracle/pqcache.py P1-P5).
#include <cuda.h>

#include <algorithm>
#include <cmath>

#include "md_common.cuh"
#include "md_internal.h"

namespace md {
namespace pq {

constexpr int M = 16;      // sub-vectors per key
constexpr int NC = 256;    // centroids per sub-space (8-bit codes)
constexpr int SCORE_CH = 16384;  // candidates per score CTA
constexpr int SCORE_THREADS = 512;
constexpr int NS = 5;            // cp.async pipeline depth of the score kernel (keys per thread)
constexpr int SCORE_SMEM = NC * 64 * 4 + 1024 * 4 + NS * SCORE_THREADS * 16;  // table + histogram + ring
constexpr int HIST1 = 1024;      // pass-1 digit: key bits 31..22
constexpr int HIST2 = 2048;      // passes 2, 3: bits 21..11, 10..0
constexpr int RL = 36;           // candidates per select thread run (16-byte loads, no bank conflicts)
// candidates staged in shared memory per super-block: NT * RL; dynamic shared memory per CTA:
constexpr int sel_smem(int nt, int tc) { return nt * RL * 4 + tc * 6; }
// More units than one wave of 512-thread CTAs (2 per SM): 256-thread CTAs, 4 per SM, with a
// 1024-key tie list so four fit (measured at the Llama-3.1 point, 512 units: one wave instead of
// 1.73); otherwise 512 threads (Qwen2.5's 256 units of 100k candidates: 256 threads were slower,
// 182 -> 220 us).  TC: the tie list (keys of the cutoff bin kept in shared memory).

__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }

// per-thread 16-byte async copies global -> shared (each thread later reads only its own slots)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

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

// ------------------------------------------------------------------ P2 lookup table
// grid (units, 4 groups of 4 sub-spaces), 256 threads: thread c computes lut[m][c] for the
// group's 4 sub-spaces m, each = sum over the query heads hh and dims i of
// q[hh][m*S + i] * cent[m][c][i] (fp32, no FMA, hh outer / i inner; the 4 chains are
// independent), and the CTA's max |lut| goes to lutmax[unit][group].  P3 (the power-of-two
// scaling to int32) needs the max over all 16 sub-spaces, so it is applied by the score kernel
// when it loads the table.
constexpr int LUT_MG = 4;  // sub-spaces per LUT CTA
template <int S>
__global__ void __launch_bounds__(256) pq_lut_kernel(const uint16_t* __restrict__ q, int Hq, int Hkv,
                                                     const uint16_t* __restrict__ cb, float* __restrict__ lutf,
                                                     float* __restrict__ lutmax, uint32_t* __restrict__ hist) {
  constexpr int D = S * M;
  __shared__ float qs[16 * LUT_MG * S];  // [g <= 16][LUT_MG * S]: the group's query slices of these sub-spaces
  __shared__ float red[8];
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x, m0 = blockIdx.y * LUT_MG, g = Hq / Hkv;
  const int b = unit / Hkv, u = unit - b * Hkv;
  const int c = threadIdx.x;
  // all LUT_MG centroid rows of this thread up front (independent 16 / 8-byte loads)
  uint32_t cw[LUT_MG][S / 2];
#pragma unroll
  for (int mm = 0; mm < LUT_MG; ++mm) {
    const uint16_t* src = cb + (((size_t)unit * M + m0 + mm) * NC + c) * S;
    if constexpr (S == 8) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(src));
      cw[mm][0] = w.x; cw[mm][1] = w.y; cw[mm][2] = w.z; cw[mm][3] = w.w;
    } else {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(src));
      cw[mm][0] = w.x; cw[mm][1] = w.y;
    }
  }
  const uint16_t* qg = q + ((size_t)b * Hq + (size_t)u * g) * D + m0 * S;
  for (int i = threadIdx.x; i < g * LUT_MG * S; i += blockDim.x)
    qs[i] = bf16_to_f32(qg[(i / (LUT_MG * S)) * D + i % (LUT_MG * S)]);
  __syncthreads();
  float acc[LUT_MG];
#pragma unroll
  for (int mm = 0; mm < LUT_MG; ++mm) acc[mm] = 0.f;
  for (int hh = 0; hh < g; ++hh) {
#pragma unroll
    for (int mm = 0; mm < LUT_MG; ++mm) {
#pragma unroll
      for (int i = 0; i < S / 2; ++i) {
        const float c0 = __uint_as_float(cw[mm][i] << 16), c1 = __uint_as_float(cw[mm][i] & 0xffff0000u);
        acc[mm] = __fadd_rn(acc[mm], __fmul_rn(qs[hh * LUT_MG * S + mm * S + 2 * i], c0));
        acc[mm] = __fadd_rn(acc[mm], __fmul_rn(qs[hh * LUT_MG * S + mm * S + 2 * i + 1], c1));
      }
    }
  }
  float mx = 0.f;
#pragma unroll
  for (int mm = 0; mm < LUT_MG; ++mm) {
    lutf[((size_t)unit * NC + c) * M + m0 + mm] = acc[mm];  // [c][m]
    mx = fmaxf(mx, fabsf(acc[mm]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
    lutmax[(size_t)unit * (M / LUT_MG) + blockIdx.y] = fmaxf(red[0], mx);
  }
  // the unit's pass-1 histogram, accumulated by the score kernel
  if (blockIdx.y == 0)
    for (int i = threadIdx.x; i < HIST1; i += blockDim.x) hist[(size_t)unit * HIST1 + i] = 0u;
}

// ------------------------------------------------------------------ P4 scores
__device__ __forceinline__ uint32_t okey(int32_t v) { return static_cast<uint32_t>(v) ^ 0x80000000u; }

// grid (units, chunks of SCORE_CH candidates), SCORE_THREADS threads, dynamic smem = the
// table (64 KB) + the pass-1 histogram.  Scores of the candidates [s0, tail) are stored
// densely (candidate j - s0) and the top digit (bits 31..22 of the order-preserving key) of
// every score is counted into the unit's global histogram.
__global__ void __launch_bounds__(SCORE_THREADS, 2) pq_score_kernel(const uint8_t* __restrict__ codes, int code_cap,
                                                                 const float* __restrict__ lutf,
                                                                 const float* __restrict__ lutmax,
                                                                 const int32_t* __restrict__ kv_len, int Hkv, int sink,
                                                                 int window, int32_t* __restrict__ scores,
                                                                 int score_stride, uint32_t* __restrict__ hist_g) {
  // tab[c * 64 + copy * 16 + m] = lutq[m][c] (256-byte rows): table m lives in bank m (copy 0)
  // and 16 + m (copy 1), and the byte offset of code c is c << 8 (one byte permute)
  extern __shared__ int32_t tab[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(tab + NC * 64);
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x;
  const int b = unit / Hkv;
  const int n = __ldg(kv_len + b);
  MD_DCHECK(n >= 0 && n <= code_cap);  // kv_len[b] <= code_capacity (every scored row is encoded)
  const int s0 = min(sink, n), tail = max(s0, n - window);
  const int lo = s0 + (int)blockIdx.y * SCORE_CH, hi = min(tail, lo + SCORE_CH);
  if (lo >= hi) return;  // uniform
  // P3: scale by 2^e with max |lut| < 2^26 (e from the max over the 16 sub-spaces) and round
  float mx = 0.f;
#pragma unroll
  for (int k = 0; k < M / LUT_MG; ++k) mx = fmaxf(mx, __ldg(lutmax + (size_t)unit * (M / LUT_MG) + k));
  int e = 0;
  if (mx > 0.f) {
    int E;
    frexpf(mx, &E);
    e = 26 - E;
  }
  const float* src = lutf + (size_t)unit * M * NC;
  for (int i = threadIdx.x; i < M * NC; i += SCORE_THREADS) {  // lutf is [c][m]: coalesced, <= 2-way stores
    const int c = i >> 4, m = i & 15;
    const int32_t v = __float2int_rn(ldexpf(__ldg(src + i), e));
    tab[c * 64 + m] = v;
    tab[c * 64 + 16 + m] = v;
  }
  for (int i = threadIdx.x; i < HIST1; i += SCORE_THREADS) hist[i] = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int l15 = lane & 15;
  // Step i reads sub-space m = i ^ l15 from copy (lane >> 4): byte offset within a table row
  // ofs(i) = (lane >> 4) * 64 + (i ^ l15) * 4 < 256.  One byte permute builds the whole
  // address: byte 0 = ofs(i) (from xo[i >> 1], which holds ofs(2p), ofs(2p + 1), 0, 0), byte
  // 1 = the code (row c at byte c << 8), bytes 2, 3 = 0; the table base folds into the load's
  // immediate offset (tab is a shared-memory symbol), so a lookup is PRMT + LDS.
  const uint32_t cpo = (uint32_t)((lane >> 4) << 6);
  uint32_t xo[M / 2];
#pragma unroll
  for (int q = 0; q < M / 2; ++q)
    xo[q] = (cpo + (uint32_t)(((2 * q) ^ l15) << 2)) | ((cpo + (uint32_t)(((2 * q + 1) ^ l15) << 2)) << 8);
  // the code byte of step i is byte ((i & 3) ^ rx) of word w'[i >> 2] = w[(i >> 2) ^ qx]
  const int qx = l15 >> 2, rx = l15 & 3;
  uint32_t sel[4];  // selector nibbles: byte 0 <- xo byte 4 + (i & 1), byte 1 <- code, bytes 2, 3 <- xo bytes 6, 7 (0)
#pragma unroll
  for (int k = 0; k < 4; ++k) sel[k] = 0x7600u | ((uint32_t)(k ^ rx) << 4) | (4u + (uint32_t)(k & 1));
  const char* tabc = reinterpret_cast<const char*>(tab);
  const uint4* crow = reinterpret_cast<const uint4*>(codes + (size_t)unit * code_cap * M);
  int32_t* out = scores + (size_t)unit * score_stride - s0;
  // the 16-byte code's words are put in the order w'[i] = w[i ^ qx] with two levels of selects
  const bool sw1 = qx & 1, sw2 = qx & 2;
  auto score_one = [&](const uint4 v) -> int32_t {
    const uint32_t a0 = sw1 ? v.y : v.x, a1 = sw1 ? v.x : v.y, a2 = sw1 ? v.w : v.z, a3 = sw1 ? v.z : v.w;
    const uint32_t w[4] = {sw2 ? a2 : a0, sw2 ? a3 : a1, sw2 ? a0 : a2, sw2 ? a1 : a3};
    int32_t acc = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) acc += *reinterpret_cast<const int32_t*>(tabc + __byte_perm(w[i >> 2], xo[i >> 1], sel[i & 3]));
    return acc;
  };
  auto emit = [&](int j, int32_t sc) {
    out[j] = sc;
    atomicAdd(&hist[okey(sc) >> 22], 1u);
  };
  // per-thread NS-deep cp.async pipeline: the codes of this thread's next NS - 1 keys are in
  // flight while it scores the current one (each thread reads only the slots it filled; a
  // warp's 128-bit reads of its slots are 512 contiguous bytes: 4 conflict-free wavefronts)
  const uint32_t ring = smem_u32(hist + HIST1) + threadIdx.x * 16;
  const int j0 = lo + threadIdx.x;
  const int nk = j0 < hi ? (hi - j0 + SCORE_THREADS - 1) / SCORE_THREADS : 0;
#pragma unroll
  for (int k = 0; k < NS - 1; ++k) {
    if (k < nk) cp_async16(ring + k * SCORE_THREADS * 16, crow + j0 + k * SCORE_THREADS);
    cp_async_commit();
  }
  int rd = 0, wr = NS - 1;
  for (int i = 0; i < nk; ++i) {
    if (i + NS - 1 < nk) cp_async16(ring + wr * SCORE_THREADS * 16, crow + j0 + (i + NS - 1) * SCORE_THREADS);
    cp_async_commit();
    cp_async_wait<NS - 1>();
    emit(j0 + i * SCORE_THREADS, score_one(lds128(ring + rd * SCORE_THREADS * 16)));
    rd = rd == NS - 1 ? 0 : rd + 1;
    wr = wr == NS - 1 ? 0 : wr + 1;
  }
  cp_async_wait<0>();
  __syncthreads();
  uint32_t* hg = hist_g + (size_t)unit * HIST1;
  for (int i = threadIdx.x; i < HIST1; i += SCORE_THREADS) {
    const uint32_t v = hist[i];
    if (v) atomicAdd(hg + i, v);
  }
}

// ------------------------------------------------------------------ P5 selection
// exclusive block scan of one value per thread (NT threads, NT / 32 <= 32 warps)
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sm, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
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
    const uint32_t x = lane < NW ? sm[lane] : 0u;
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

// Find the bin holding the need-th largest key of a histogram (bins ascending by value):
// the bin and how many keys of that bin are still needed.  Thread t owns nb / NT
// consecutive bins counted from the top.
template <int NT>
__device__ __forceinline__ void find_cut(const uint32_t* hist, int nb, uint32_t need, uint32_t* sm, int* s_bin,
                                         uint32_t* s_need) {
  const int per = nb / NT;
  const int top = nb - 1 - threadIdx.x * per;  // this thread's highest bin
  uint32_t local = 0;
  for (int i = 0; i < per; ++i) local += hist[top - i];
  uint32_t total;
  const uint32_t above = block_excl_scan<NT>(local, sm, total);
  if (above < need && above + local >= need) {
    uint32_t acc = above;
    int bin = top;
    for (int i = 0; i < per - 1; ++i, --bin) {
      if (acc + hist[bin] >= need) break;
      acc += hist[bin];
    }
    *s_bin = bin;
    *s_need = need - acc;
  }
  __syncthreads();
}

// One CTA per unit.  The pass-1 histogram (10-bit top digit) comes from the score kernel.
// The candidate scores are staged in shared memory by one bulk copy per super-block of NT * RL
// candidates; thread t owns the contiguous run [t*RL, (t+1)*RL) of it (RL = 36: the 16-byte
// loads of 8 consecutive threads hit disjoint banks).  Pass over the runs: count the keys above
// the cutoff bin and gather the cutoff bin's keys (with their owner thread) into a small list;
// passes 2-3 (11 + 11 bits) refine the threshold key thr and how many keys equal to thr to
// take (the lowest positions) on that list, which also yields every thread's count of
// selected keys; an exclusive scan of the counts then places each run's selections in
// position order (second pass over the runs).  A cutoff bin with more than TC keys is
// refined from global memory instead.
template <int NT, int TC>
__global__ void __launch_bounds__(NT, 1024 / NT) pq_select_kernel(const int32_t* __restrict__ scores,
                                                                   int score_stride, const uint32_t* __restrict__ hist_g,
                                                                   const int32_t* __restrict__ kv_len, int Hkv, int sink,
                                                                   int window, int budget, int32_t* __restrict__ idx,
                                                                   int idx_stride, int32_t* __restrict__ idx_count,
                                                                   int32_t* __restrict__ tail_start) {
  extern __shared__ __align__(16) int32_t stage[];  // [(NT * RL)] staged scores, ties[TC], owner[TC]
  uint32_t* ties = reinterpret_cast<uint32_t*>(stage + NT * RL);
  uint16_t* owner = reinterpret_cast<uint16_t*>(ties + TC);
  __shared__ uint32_t hist[HIST2];
  __shared__ uint32_t n_gt_sm[NT], n_eq_sm[NT];
  __shared__ uint32_t scan_sm[65];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_bin;
  __shared__ uint32_t s_need, s_nties;
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
  for (int j = threadIdx.x; j < s0; j += NT) out[j] = j;
  if (c == 0) return;
  out += s0;
  if (c == cnt) {  // the budget covers every candidate
    for (int j = threadIdx.x; j < cnt; j += NT) out[j] = s0 + j;
    return;
  }
  const int32_t* sc = scores + (size_t)unit * score_stride;  // candidate j at sc[j] (16-byte aligned)
  // ---- pass 1 (histogram from the score kernel): cutoff bin of the top digit
  {
    const uint32_t* hg = hist_g + (size_t)unit * HIST1;
    for (int i = threadIdx.x; i < HIST1; i += NT) hist[i] = __ldcg(hg + i);
    if (threadIdx.x == 0) {
      s_nties = 0;
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  find_cut<NT>(hist, HIST1, (uint32_t)c, scan_sm, &s_bin, &s_need);
  const uint32_t cb = (uint32_t)s_bin;
  uint32_t prefix = cb << 22, need = s_need;
  const uint32_t nbin = hist[cb];
  const bool gathered = nbin <= TC;
  const int nsb = (cnt + (NT * RL) - 1) / (NT * RL);
  uint32_t phase = 0;
  auto stage_block = [&](int base) {  // candidates [base, base + (NT * RL)) -> stage (one bulk copy)
    const int nb = min((NT * RL), cnt - base);
    __syncthreads();  // every reader of the previous super-block is done
    if (threadIdx.x == 0) {
      fence_proxy_async();  // earlier generic reads of the stage before the async-proxy overwrite
      const uint32_t bytes = (uint32_t)((nb + 3) & ~3) * 4;  // rows are padded to 4 candidates
      mbar_arrive_expect_tx(&bar, bytes);
      bulk_load(stage, sc + base, bytes, &bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    return nb;
  };
  // run loop: f(k, key) for this thread's valid candidates of the staged super-block
  auto for_run = [&](int nb, auto&& f) {
    const int r0 = threadIdx.x * RL;
    if (r0 + RL <= nb) {
#pragma unroll 3
      for (int k = 0; k < RL; k += 4) {
        const int4 x = *reinterpret_cast<const int4*>(stage + r0 + k);
        f(r0 + k, okey(x.x));
        f(r0 + k + 1, okey(x.y));
        f(r0 + k + 2, okey(x.z));
        f(r0 + k + 3, okey(x.w));
      }
    } else {
      for (int k = r0; k < nb; ++k) f(k, okey(stage[k]));
    }
  };
  // ---- runs pass 1: keys of the cutoff bin -> ties (with their owner thread)
  if (gathered) {
    for (int sb = 0; sb < nsb; ++sb) {
      const int nb = stage_block(sb * (NT * RL));
      for_run(nb, [&](int, uint32_t kk) {
        if ((kk >> 22) == cb) {
          const uint32_t slot = atomicAdd(&s_nties, 1u);
          ties[slot] = kk;
          owner[slot] = (uint16_t)(sb * NT + threadIdx.x);
        }
      });
    }
    __syncthreads();
  }
  // ---- passes 2, 3: refine the low 22 bits inside the cutoff bin
#pragma unroll 1
  for (int d = 0; d < 2; ++d) {
    const int sh = d == 0 ? 11 : 0;
    const uint32_t hi_mask = 0xffffffffu << (sh + 11);
    for (int i = threadIdx.x; i < HIST2; i += NT) hist[i] = 0;
    __syncthreads();
    if (gathered) {
      for (int j = threadIdx.x; j < (int)nbin; j += NT) {
        const uint32_t kk = ties[j];
        if ((kk & hi_mask) == prefix) atomicAdd(&hist[(kk >> sh) & (HIST2 - 1)], 1u);
      }
    } else {
      for (int j = threadIdx.x; j < cnt; j += NT) {
        const uint32_t kk = okey(__ldcg(sc + j));
        if ((kk & hi_mask) == prefix) atomicAdd(&hist[(kk >> sh) & (HIST2 - 1)], 1u);
      }
    }
    __syncthreads();
    find_cut<NT>(hist, HIST2, need, scan_sm, &s_bin, &s_need);
    prefix |= (uint32_t)s_bin << sh;
    need = s_need;
    __syncthreads();
  }
  const uint32_t thr = prefix, take_eq = need;
  // ---- runs pass 2: ordered compaction, super-block by super-block
  uint32_t base_out = 0, eq_seen = 0;
  for (int sb = 0; sb < nsb; ++sb) {
    const int nb = (nsb > 1 || !gathered) ? stage_block(sb * (NT * RL)) : min((NT * RL), cnt);
    uint32_t n_gt = 0, n_eq = 0;
    if (gathered) {
      // counts of this super-block's runs from the tie list: keys above the cutoff bin are
      // all selected, inside it the ones > thr (and the first take_eq of those == thr)
      n_gt_sm[threadIdx.x] = 0;
      n_eq_sm[threadIdx.x] = 0;
      __syncthreads();
      for (int j = threadIdx.x; j < (int)nbin; j += NT) {
        const int o = owner[j] - sb * NT;
        if (o >= 0 && o < NT) {
          if (ties[j] > thr) atomicAdd(&n_gt_sm[o], 1u);
          else if (ties[j] == thr) atomicAdd(&n_eq_sm[o], 1u);
        }
      }
      __syncthreads();
      for_run(nb, [&](int, uint32_t kk) { n_gt += (kk >> 22) > cb; });
      n_gt += n_gt_sm[threadIdx.x];
      n_eq = n_eq_sm[threadIdx.x];
    } else {
      for_run(nb, [&](int, uint32_t kk) {
        n_gt += kk > thr;
        n_eq += kk == thr;
      });
    }
    uint32_t tot_eq, tot_gt;
    const uint32_t eq_before = eq_seen + block_excl_scan<NT>(n_eq, scan_sm, tot_eq);
    const uint32_t gt_before = block_excl_scan<NT>(n_gt, scan_sm, tot_gt);
    uint32_t pos = base_out + gt_before + min(eq_before, take_eq) - min(eq_seen, take_eq);
    uint32_t eq_rank = eq_before;
    const int base = s0 + sb * (NT * RL);
    for_run(nb, [&](int k, uint32_t kk) {
      const bool eq = kk == thr;
      const bool take = kk > thr || (eq && eq_rank < take_eq);
      eq_rank += eq;
      if (take) out[pos++] = base + k;
    });
    base_out += tot_gt + min(eq_seen + tot_eq, take_eq) - min(eq_seen, take_eq);
    eq_seen += tot_eq;
  }
}

}  // namespace pq

static size_t pq_align(size_t x) { return (x + 255) & ~size_t(255); }
static int pq_score_stride(int maxL) { return (maxL + 3) & ~3; }
static size_t pq_ws(int B, int Hkv, int maxL) {
  const size_t units = (size_t)B * Hkv;
  return pq_align(units * pq::M * pq::NC * 4) + pq_align(units * pq::M * 4) + pq_align(units * pq::HIST1 * 4) +
         pq_align(units * (size_t)pq_score_stride(maxL) * 4);
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
  uint8_t* w8 = static_cast<uint8_t*>(workspace);
  auto* lutf = reinterpret_cast<float*>(w8);
  w8 += pq_align((size_t)units * pq::M * pq::NC * 4);
  auto* lutmax = reinterpret_cast<float*>(w8);
  w8 += pq_align((size_t)units * pq::M * 4);
  auto* hist = reinterpret_cast<uint32_t*>(w8);
  w8 += pq_align((size_t)units * pq::HIST1 * 4);
  auto* scores = reinterpret_cast<int32_t*>(w8);
  const int sstride = pq_score_stride(max_kv_len);
  const auto* qq = static_cast<const uint16_t*>(q);
  const auto* cb = static_cast<const uint16_t*>(codebook);
  cudaStream_t s = (cudaStream_t)stream;
  const int g = num_q_heads / num_kv_heads;
  (void)g;
  if (head_dim == 128)
    launch_pdl(pq::pq_lut_kernel<8>, dim3(units, pq::M / pq::LUT_MG), dim3(256), 0, s, qq, (int)num_q_heads, (int)num_kv_heads, cb,
               lutf, lutmax, hist);
  else
    launch_pdl(pq::pq_lut_kernel<4>, dim3(units, pq::M / pq::LUT_MG), dim3(256), 0, s, qq, (int)num_q_heads, (int)num_kv_heads, cb,
               lutf, lutmax, hist);
  if (md_status st = check_launch("pq_lut_kernel"); st != MD_OK) return st;
  static int done_dev = -1;  // per-process; the attribute call is idempotent (benign race)
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev != dev) {
    if (cudaFuncSetAttribute(pq::pq_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pq::SCORE_SMEM) !=
            cudaSuccess ||
        cudaFuncSetAttribute(pq::pq_select_kernel<512, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             pq::sel_smem(512, 2048)) != cudaSuccess ||
        cudaFuncSetAttribute(pq::pq_select_kernel<256, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             pq::sel_smem(256, 1024)) != cudaSuccess)
      return check_launch("cudaFuncSetAttribute");
    done_dev = dev;
  }
  // candidates of a unit: [s0, tail) with tail <= max(s0, n - window), so at most
  // max(1, max_kv_len - window) of them (a chunk past every unit's candidates would only load
  // the table: 3 chunks instead of 2 at the 32k BASELINE shapes)
  const int max_cand = std::max(1, (int)max_kv_len - (int)window);
  const unsigned chunks = (unsigned)((max_cand + pq::SCORE_CH - 1) / pq::SCORE_CH);
  launch_pdl(pq::pq_score_kernel, dim3(units, chunks), dim3(pq::SCORE_THREADS), (size_t)pq::SCORE_SMEM, s, codes,
             (int)code_capacity, (const float*)lutf, (const float*)lutmax, kv_len, (int)num_kv_heads, (int)sink, (int)window, scores,
             sstride, hist);
  if (md_status st = check_launch("pq_score_kernel"); st != MD_OK) return st;
  if (units > 2 * device_sm_count())
    launch_pdl(pq::pq_select_kernel<256, 1024>, dim3(units), dim3(256), (size_t)pq::sel_smem(256, 1024), s,
               (const int32_t*)scores, sstride, (const uint32_t*)hist, kv_len, (int)num_kv_heads, (int)sink,
               (int)window, (int)budget, idx, (int)idx_stride, idx_count, tail_start);
  else
    launch_pdl(pq::pq_select_kernel<512, 2048>, dim3(units), dim3(512), (size_t)pq::sel_smem(512, 2048), s,
               (const int32_t*)scores, sstride, (const uint32_t*)hist, kv_len, (int)num_kv_heads, (int)sink,
               (int)window, (int)budget, idx, (int)idx_stride, idx_count, tail_start);
  return check_launch("pq_select_kernel");
}

// spec_accept.cu — md_spec_accept and md_philox_u32.
//
// One CTA per sequence.  SAMPLE mode decides the gamma accept tests with exact fp64
// products (m * q < p * 2^29, m = rnd >> 3: 29 x 24 bits fit in the 53-bit mantissa),
// then draws the final token from an integer weight vector on the 2^-40 grid with a
// 64-bit uniform.  All sums are uint64 (<= V * 2^40 < 2^58), so the result does not
// depend on the reduction order and is bit-identical to the oracle's.  Each warp streams a
// contiguous segment of the vocabulary row with coalesced, 8-chunk-deep loads; a scan of the
// segment sums locates the segment holding the draw, which the block re-streams (see below).
#include "md_common.cuh"
#include "md_internal.h"

namespace md {

constexpr int ACC_THREADS = 512;
constexpr int ACC_WARPS = ACC_THREADS / 32;

// ---------------------------------------------------------------- Philox4x32-10
struct Philox4 {
  uint32_t v[4];
};
__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                                 uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return Philox4{{c0, c1, c2, c3}};
}

// step_dev != null: the step is read from device memory (graph replays draw fresh words)
__global__ void philox_kernel(uint64_t seed, uint64_t step, const uint64_t* step_dev, int B, int words,
                              uint32_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  if (step_dev != nullptr) step = *step_dev;
  const int blocks_per_seq = (words + 3) / 4;
  const int64_t total = (int64_t)B * blocks_per_seq;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = static_cast<int>(i / blocks_per_seq), blk = static_cast<int>(i % blocks_per_seq);
    const Philox4 r = philox4x32_10(static_cast<uint32_t>(b), static_cast<uint32_t>(step),
                                    static_cast<uint32_t>(step >> 32), static_cast<uint32_t>(blk),
                                    static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int w = blk * 4 + k;
      if (w < words) out[(int64_t)b * words + w] = r.v[k];
    }
  }
}

// ---------------------------------------------------------------- integer weights
// floor(x * 2^40) for x in [0, 1] (exact: power-of-two scale in fp64, then truncate).
__device__ __forceinline__ uint64_t grid40(float x) {
  return x > 0.f ? __double2ull_rz(static_cast<double>(x) * 1099511627776.0) : 0ull;
}
__device__ __forceinline__ uint64_t weight(const float* __restrict__ prow, const float* __restrict__ qrow, int i) {
  const uint64_t P = grid40(__ldg(prow + i));
  if (qrow == nullptr) return P;
  const uint64_t Q = grid40(__ldg(qrow + i));
  return P > Q ? P - Q : 0ull;
}

struct Smem {
  uint64_t wsum[ACC_WARPS];
  uint64_t total;
  float amax_v[ACC_WARPS];
  int amax_i[ACC_WARPS];
  int token;
  int n;
};

// Warp-strip layout (round 2): the row is cut into ACC_WARPS contiguous warp segments whose
// lengths are multiples of one warp chunk (CH = 32 * VEC elements); a warp streams its segment
// chunk by chunk, lane l taking elements [c + l * VEC, c + l * VEC + VEC) -- coalesced 16-byte
// loads (VEC = 4) when both rows are 16-byte aligned, 4-byte loads otherwise -- BATCH chunks
// in flight.  A block scan of the warp sums gives every segment's prefix; the locate step
// re-streams the one segment holding the draw with the whole block (sub-segments per warp),
// and one warp walks its sub-segment chunk by chunk with a lane scan.  Every sum is an exact
// uint64, so the token (min{k : sum_{i<=k} W_i > t}) is the same as any other order's.
// (The round-1 layout -- thread t owns the contiguous slice [t V/512, ...) read with 4-byte
// loads -- touched 32 sectors per warp load instruction and ran at ~1 TB/s.)
constexpr int BATCH = 4;  // chunks in flight per warp (x 2 rows x 16 B x 32 lanes)

__device__ __forceinline__ uint64_t wdiff(float p, float q) {
  const uint64_t P = grid40(p), Q = grid40(q);
  return P > Q ? P - Q : 0ull;
}

// weights of the VEC elements [i, i + VEC) (0 past V)
template <int VEC>
__device__ __forceinline__ void chunk_weights(const float* __restrict__ prow, const float* __restrict__ qrow, int i,
                                              int V, uint64_t (&w)[VEC]) {
  if constexpr (VEC == 4) {
    if (i + 3 < V) {
      const float4 pv = __ldg(reinterpret_cast<const float4*>(prow + i));
      const float4 qv = qrow != nullptr ? __ldg(reinterpret_cast<const float4*>(qrow + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
      w[0] = wdiff(pv.x, qv.x);
      w[1] = wdiff(pv.y, qv.y);
      w[2] = wdiff(pv.z, qv.z);
      w[3] = wdiff(pv.w, qv.w);
      return;
    }
  }
#pragma unroll
  for (int u = 0; u < VEC; ++u) w[u] = (i + u < V) ? weight(prow, qrow, i + u) : 0ull;
}

// sum of the weights of [beg, end) (beg a multiple of CH relative to the row, end <= V) by one warp;
// every lane returns the total.  The BATCH chunks' loads are issued before any weight is formed.
template <int VEC>
__device__ uint64_t warp_range_sum(const float* __restrict__ prow, const float* __restrict__ qrow, int beg, int end,
                                   int V) {
  constexpr int CH = 32 * VEC;
  const int lane = threadIdx.x & 31;
  uint64_t acc = 0;
  for (int c0 = beg; c0 < end; c0 += CH * BATCH) {
    float pv[BATCH][VEC], qv[BATCH][VEC];
#pragma unroll
    for (int k = 0; k < BATCH; ++k) {
      const int i = c0 + k * CH + lane * VEC;
      if constexpr (VEC == 4) {
        if (i + 3 < end) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(prow + i));
          const float4 c = qrow != nullptr ? __ldg(reinterpret_cast<const float4*>(qrow + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
          pv[k][0] = a.x; pv[k][1] = a.y; pv[k][2] = a.z; pv[k][3] = a.w;
          qv[k][0] = c.x; qv[k][1] = c.y; qv[k][2] = c.z; qv[k][3] = c.w;
          continue;
        }
      }
#pragma unroll
      for (int u = 0; u < VEC; ++u) {  // 4-byte loads (VEC = 1), the row's last partial chunk, or past the end
        const bool in = i + u < end;
        pv[k][u] = in ? __ldg(prow + i + u) : 0.f;
        qv[k][u] = (in && qrow != nullptr) ? __ldg(qrow + i + u) : 0.f;
      }
    }
#pragma unroll
    for (int k = 0; k < BATCH; ++k)
#pragma unroll
      for (int u = 0; u < VEC; ++u) acc += wdiff(pv[k][u], qv[k][u]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

__device__ __forceinline__ int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Pass 1: warp segment sums -> sm.wsum, sm.total.
template <int VEC>
__device__ void block_weight_sums(const float* prow, const float* qrow, int V, Smem& sm) {
  constexpr int CH = 32 * VEC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = round_up((V + ACC_WARPS - 1) / ACC_WARPS, CH);
  const int beg = min(V, warp * seg), end = min(V, beg + seg);
  const uint64_t s = warp_range_sum<VEC>(prow, qrow, beg, end, V);
  __syncthreads();  // sm.wsum may still be read by a previous pass
  if (lane == 0) sm.wsum[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t total = 0;
    for (int w = 0; w < ACC_WARPS; ++w) total += sm.wsum[w];
    sm.total = total;
  }
  __syncthreads();
}

// token = min{k : sum_{i<=k} W_i > t}, t < sm.total (after block_weight_sums).
template <int VEC>
__device__ int block_locate(const float* prow, const float* qrow, int V, uint64_t t, Smem& sm) {
  constexpr int CH = 32 * VEC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = round_up((V + ACC_WARPS - 1) / ACC_WARPS, CH);
  // the warp segment holding t (every thread finds the same one)
  uint64_t run = 0;
  int ws = 0;
  for (int w = 0; w < ACC_WARPS; ++w) {
    const uint64_t v = sm.wsum[w];
    if (run + v > t) {
      ws = w;
      break;
    }
    run += v;
  }
  const int base = min(V, ws * seg), send = min(V, base + seg);
  // its sub-segments, one per warp
  const int sub = round_up((send - base + ACC_WARPS - 1) / ACC_WARPS, CH);
  const int sbeg = min(send, base + warp * sub), send2 = min(send, sbeg + sub);
  const uint64_t s = warp_range_sum<VEC>(prow, qrow, sbeg, send2, V);
  __syncthreads();  // every warp has read sm.wsum
  if (lane == 0) sm.wsum[warp] = s;
  __syncthreads();
  int w2 = 0;
  for (int w = 0; w < ACC_WARPS; ++w) {
    const uint64_t v = sm.wsum[w];
    if (run + v > t) {
      w2 = w;
      break;
    }
    run += v;
  }
  if (warp == w2) {  // walk this warp's sub-segment chunk by chunk
    const int b2 = min(send, base + w2 * sub), e2 = min(send, b2 + sub);
    for (int c0 = b2; c0 < e2; c0 += CH) {
      uint64_t w[VEC];
      const int i = c0 + lane * VEC;
      if (i < e2) {
        chunk_weights<VEC>(prow, qrow, i, V, w);
      } else {
#pragma unroll
        for (int u = 0; u < VEC; ++u) w[u] = 0ull;
      }
      uint64_t ls = 0;
#pragma unroll
      for (int u = 0; u < VEC; ++u) ls += w[u];
      uint64_t incl = ls;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t up = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += up;
      }
      const uint64_t tot = __shfl_sync(0xffffffffu, incl, 31);
      if (run + tot > t) {
        const unsigned hit = __ballot_sync(0xffffffffu, run + incl > t);
        const int L = __ffs(hit) - 1;
        if (lane == L) {
          uint64_t r = run + incl - ls;
          int k = i;
#pragma unroll
          for (int u = 0; u < VEC; ++u) {
            r += w[u];
            if (r > t) {
              k = i + u;
              break;
            }
          }
          sm.token = k;
        }
        break;
      }
      run += tot;
    }
  }
  __syncthreads();
  return sm.token;
}

constexpr int UNR = 8;  // argmax: loads in flight per thread

// Lowest-index argmax of a row (block-wide).  All threads return the same value.
__device__ int block_argmax(const float* __restrict__ row, int V, Smem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  int i = tid;
  for (; i + (UNR - 1) * ACC_THREADS < V; i += UNR * ACC_THREADS) {
    float v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = __ldg(row + i + u * ACC_THREADS);
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      if (v[u] > bv) {  // indices increase with u: strict > keeps the lowest index on ties
        bv = v[u];
        bi = i + u * ACC_THREADS;
      }
  }
  for (; i < V; i += ACC_THREADS) {
    const float v = __ldg(row + i);
    if (v > bv) {
      bv = v;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  __syncthreads();  // protect sm.amax_* from a previous call
  if (lane == 0) {
    sm.amax_v[warp] = bv;
    sm.amax_i[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    float v = sm.amax_v[0];
    int idx = sm.amax_i[0];
    for (int w = 1; w < ACC_WARPS; ++w)
      if (sm.amax_v[w] > v || (sm.amax_v[w] == v && sm.amax_i[w] < idx)) {
        v = sm.amax_v[w];
        idx = sm.amax_i[w];
      }
    sm.token = (idx == 0x7fffffff) ? 0 : idx;
  }
  __syncthreads();
  return sm.token;
}

__global__ void __launch_bounds__(ACC_THREADS, 2) spec_accept_kernel(
    const float* __restrict__ p, const float* __restrict__ q, const int32_t* __restrict__ dtok,
    const uint32_t* __restrict__ rnd, int gamma, int V, int mode, int32_t* __restrict__ out_tokens,
    int32_t* __restrict__ num_accepted, int32_t* __restrict__ committed_len) {
  __shared__ Smem sm;
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x, tid = threadIdx.x;
  const int64_t Vl = V;
  const float* pb = p + (int64_t)b * (gamma + 1) * Vl;
  const int32_t* db = dtok + (int64_t)b * gamma;
  int n, token;
  if (mode == MD_ACCEPT_SAMPLE) {
    const uint32_t* rb = rnd + (int64_t)b * (gamma + 2);
    if (tid < 32) {
      bool reject = false;
      if (tid < gamma) {
        const int x = __ldg(db + tid);
        MD_DCHECK(x >= 0 && x < V);  // draft token ids < V
        const double px = __ldg(pb + (int64_t)tid * Vl + x);
        const double qx = __ldg(q + ((int64_t)b * gamma + tid) * Vl + x);
        MD_DCHECK(px >= 0.0 && px <= 1.0 && qx >= 0.0 && qx <= 1.0);  // finite probabilities in [0, 1] (NaN fails)
        const double m = static_cast<double>(__ldg(rb + tid) >> 3);
        reject = !(m * qx < px * 536870912.0);
      }
      const unsigned rej = __ballot_sync(0xffffffffu, reject);
      if (tid == 0) sm.n = rej ? (__ffs(rej) - 1) : gamma;
    }
    __syncthreads();
    n = sm.n;
    const float* prow = pb + (int64_t)n * Vl;
    const float* qrow = (n < gamma) ? q + ((int64_t)b * gamma + n) * Vl : nullptr;
    // 16-byte loads when both rows are 16-byte aligned (uniform over the CTA)
    const bool vec = ((reinterpret_cast<uintptr_t>(prow) | reinterpret_cast<uintptr_t>(qrow)) & 15u) == 0;
    if (vec) block_weight_sums<4>(prow, qrow, V, sm);
    else block_weight_sums<1>(prow, qrow, V, sm);
    uint64_t total = sm.total;
    if (total == 0 && qrow != nullptr) {  // degenerate residual: fall back to p (reading Z7)
      qrow = nullptr;
      if (vec) block_weight_sums<4>(prow, qrow, V, sm);
      else block_weight_sums<1>(prow, qrow, V, sm);
      total = sm.total;
    }
    if (total == 0) {
      token = block_argmax(prow, V, sm);  // invalid all-tiny row
    } else {
      const uint64_t u = (static_cast<uint64_t>(__ldg(rb + gamma)) << 32) | __ldg(rb + gamma + 1);
      const uint64_t t = __umul64hi(u, total);
      token = vec ? block_locate<4>(prow, qrow, V, t, sm) : block_locate<1>(prow, qrow, V, t, sm);
    }
  } else {
    n = gamma;
    token = -1;
    for (int j = 0; j < gamma; ++j) {
      const int am = block_argmax(pb + (int64_t)j * Vl, V, sm);
      MD_DCHECK(__ldg(db + j) >= 0 && __ldg(db + j) < V);
      if (am != __ldg(db + j)) {
        n = j;
        token = am;
        break;
      }
    }
    if (n == gamma) token = block_argmax(pb + (int64_t)gamma * Vl, V, sm);
  }
  for (int k = tid; k <= gamma; k += ACC_THREADS)
    out_tokens[(int64_t)b * (gamma + 1) + k] = k < n ? __ldg(db + k) : (k == n ? token : -1);
  if (tid == 0) {
    num_accepted[b] = n;
    if (committed_len != nullptr) committed_len[b] += n + 1;
  }
}

}  // namespace md

extern "C" md_status md_philox_u32(uint64_t seed, uint64_t step, int32_t B, int32_t words_per_seq, uint32_t* out,
                                   md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(out != nullptr, MD_ERR_INVALID_ARG, "md_philox_u32: NULL output");
  MD_REQUIRE(B >= 1 && words_per_seq >= 1, MD_ERR_INVALID_ARG, "md_philox_u32: B and words_per_seq must be >= 1");
  const int64_t total = (int64_t)B * ((words_per_seq + 3) / 4);
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 4096) blocks = 4096;
  launch_pdl(philox_kernel, dim3(static_cast<unsigned>(blocks)), dim3(threads), 0, (cudaStream_t)stream, seed, step,
             (const uint64_t*)nullptr, (int)B, (int)words_per_seq, out);
  return check_launch("md_philox_u32");
}

extern "C" md_status md_philox_u32_dev(uint64_t seed, const uint64_t* step, int32_t B, int32_t words_per_seq,
                                       uint32_t* out, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(out != nullptr && step != nullptr, MD_ERR_INVALID_ARG, "md_philox_u32_dev: NULL output / step");
  MD_REQUIRE(B >= 1 && words_per_seq >= 1, MD_ERR_INVALID_ARG, "md_philox_u32_dev: B and words_per_seq must be >= 1");
  const int64_t total = (int64_t)B * ((words_per_seq + 3) / 4);
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 4096) blocks = 4096;
  launch_pdl(philox_kernel, dim3(static_cast<unsigned>(blocks)), dim3(threads), 0, (cudaStream_t)stream, seed,
             (uint64_t)0, step, (int)B, (int)words_per_seq, out);
  return check_launch("md_philox_u32_dev");
}

extern "C" md_status md_spec_accept(const float* p, const float* q, const int32_t* draft_tokens, const uint32_t* rnd,
                                    int32_t B, int32_t gamma, int32_t V, md_accept_mode mode, int32_t* out_tokens,
                                    int32_t* num_accepted, int32_t* committed_len_inout, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(mode == MD_ACCEPT_SAMPLE || mode == MD_ACCEPT_GREEDY, MD_ERR_INVALID_ARG, "md_spec_accept: bad mode");
  MD_REQUIRE(B >= 1 && V >= 1, MD_ERR_INVALID_ARG, "md_spec_accept: B and V must be >= 1");
  MD_REQUIRE(gamma >= 0 && gamma <= 15, MD_ERR_UNSUPPORTED, "md_spec_accept: gamma must be in [0, 15]");
  MD_REQUIRE(p != nullptr && out_tokens != nullptr && num_accepted != nullptr, MD_ERR_INVALID_ARG,
             "md_spec_accept: NULL p / out_tokens / num_accepted");
  MD_REQUIRE(gamma == 0 || draft_tokens != nullptr, MD_ERR_INVALID_ARG, "md_spec_accept: NULL draft_tokens");
  MD_REQUIRE(mode == MD_ACCEPT_GREEDY || rnd != nullptr, MD_ERR_INVALID_ARG, "md_spec_accept: NULL rnd (SAMPLE)");
  MD_REQUIRE(mode == MD_ACCEPT_GREEDY || gamma == 0 || q != nullptr, MD_ERR_INVALID_ARG,
             "md_spec_accept: NULL q (SAMPLE)");
  launch_pdl(spec_accept_kernel, dim3(B), dim3(ACC_THREADS), 0, (cudaStream_t)stream, p, q, draft_tokens, rnd,
             (int)gamma, (int)V, static_cast<int>(mode), out_tokens, num_accepted, committed_len_inout);
  return check_launch("md_spec_accept");
}

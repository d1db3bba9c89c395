// spec_accept.cu — md_spec_accept and md_philox_u32.
//
// One CTA per sequence.  SAMPLE mode decides the gamma accept tests with exact fp64
// products (m * q < p * 2^29, m = rnd >> 3: 29 x 24 bits fit in the 53-bit mantissa),
// then draws the final token from an integer weight vector on the 2^-40 grid with a
// 64-bit uniform.  All sums are uint64 (<= V * 2^40 < 2^58), so the result does not
// depend on the reduction order and is bit-identical to the oracle's.  The locate
// step is two-level: per-warp segment sums, a prefix over warps, then one warp
// rescans its segment 32 entries at a time with a warp-inclusive scan.
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

__global__ void philox_kernel(uint64_t seed, uint64_t step, int B, int words, uint32_t* __restrict__ out) {
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

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct Smem {
  uint64_t wsum[ACC_WARPS];
  uint64_t wpre[ACC_WARPS];
  float amax_v[ACC_WARPS];
  int amax_i[ACC_WARPS];
  uint64_t total;
  int token;
  int n;
};

// Lowest-index argmax of a row (block-wide).  All threads return the same value.
__device__ int block_argmax(const float* __restrict__ row, int V, Smem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = tid; i < V; i += ACC_THREADS) {
    const float v = __ldg(row + i);
    if (v > bv || (v == bv && i < bi)) {
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
    int i = sm.amax_i[0];
    for (int w = 1; w < ACC_WARPS; ++w)
      if (sm.amax_v[w] > v || (sm.amax_v[w] == v && sm.amax_i[w] < i)) {
        v = sm.amax_v[w];
        i = sm.amax_i[w];
      }
    sm.token = (i == 0x7fffffff) ? 0 : i;
  }
  __syncthreads();
  return sm.token;
}

// Per-warp segment sums of the weights; returns the block total (all threads).
__device__ uint64_t block_weight_sum(const float* prow, const float* qrow, int V, int seg, Smem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int beg = warp * seg, end = min(V, beg + seg);
  uint64_t acc = 0;
  for (int i = beg + lane; i < end; i += 32) acc += weight(prow, qrow, i);
  acc = warp_sum_u64(acc);
  __syncthreads();
  if (lane == 0) sm.wsum[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    uint64_t run = 0;
    for (int w = 0; w < ACC_WARPS; ++w) {
      sm.wpre[w] = run;
      run += sm.wsum[w];
    }
    sm.total = run;
  }
  __syncthreads();
  return sm.total;
}

// token = min{k : sum_{i<=k} W_i > t}, given the segment sums from block_weight_sum.
__device__ int block_locate(const float* prow, const float* qrow, int V, int seg, uint64_t t, Smem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t pre = sm.wpre[warp], ws = sm.wsum[warp];
  if (ws != 0 && pre <= t && t < pre + ws) {  // exactly one warp satisfies this
    const int beg = warp * seg, end = min(V, beg + seg);
    uint64_t run = pre;
    for (int base = beg; base < end; base += 32) {
      const int i = base + lane;
      uint64_t incl = (i < end) ? weight(prow, qrow, i) : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t up = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += up;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, run + incl > t);
      if (hit) {
        if (lane == 0) sm.token = base + __ffs(hit) - 1;
        break;
      }
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  return sm.token;
}

__global__ void __launch_bounds__(ACC_THREADS) spec_accept_kernel(
    const float* __restrict__ p, const float* __restrict__ q, const int32_t* __restrict__ dtok,
    const uint32_t* __restrict__ rnd, int gamma, int V, int mode, int32_t* __restrict__ out_tokens,
    int32_t* __restrict__ num_accepted, int32_t* __restrict__ committed_len) {
  __shared__ Smem sm;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int64_t Vl = V;
  const float* pb = p + (int64_t)b * (gamma + 1) * Vl;
  const int32_t* db = dtok + (int64_t)b * gamma;
  const int seg = ((V + ACC_WARPS - 1) / ACC_WARPS + 31) & ~31;
  int n, token;
  if (mode == MD_ACCEPT_SAMPLE) {
    const uint32_t* rb = rnd + (int64_t)b * (gamma + 2);
    if (tid < 32) {
      bool reject = false;
      if (tid < gamma) {
        const int x = __ldg(db + tid);
        const double px = __ldg(pb + (int64_t)tid * Vl + x);
        const double qx = __ldg(q + ((int64_t)b * gamma + tid) * Vl + x);
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
    uint64_t total = block_weight_sum(prow, qrow, V, seg, sm);
    if (total == 0 && qrow != nullptr) {  // degenerate residual: fall back to p (reading Z7)
      qrow = nullptr;
      total = block_weight_sum(prow, qrow, V, seg, sm);
    }
    if (total == 0) {
      token = block_argmax(prow, V, sm);  // invalid all-tiny row
    } else {
      const uint64_t u = (static_cast<uint64_t>(__ldg(rb + gamma)) << 32) | __ldg(rb + gamma + 1);
      const uint64_t t = __umul64hi(u, total);
      token = block_locate(prow, qrow, V, seg, t, sm);
    }
  } else {
    n = gamma;
    token = -1;
    for (int j = 0; j < gamma; ++j) {
      const int am = block_argmax(pb + (int64_t)j * Vl, V, sm);
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
  philox_kernel<<<static_cast<unsigned>(blocks), threads, 0, (cudaStream_t)stream>>>(seed, step, B, words_per_seq,
                                                                                      out);
  return check_launch("md_philox_u32");
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
  spec_accept_kernel<<<B, ACC_THREADS, 0, (cudaStream_t)stream>>>(p, q, draft_tokens, rnd, gamma, V,
                                                                   static_cast<int>(mode), out_tokens, num_accepted,
                                                                   committed_len_inout);
  return check_launch("md_spec_accept");
}

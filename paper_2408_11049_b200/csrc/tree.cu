// tree.cu — tree-based speculation (paper P:173 names token trees as
// compatible with its analysis): md_spec_accept_tree and md_kv_compact.  The tree-masked
// attention itself is md_verify_attn_tree in attn.cu.
//
// md_spec_accept_tree: one CTA per sequence walks the token tree from the root (DESIGN.md
// readings Z21-Z24).  At node `cur` the children are tested in index order: the first with
// the chain rule's exact fp64 test; after a rejection the target becomes the integer residual
// on the 2^-40 grid, R0 = max(0, P - Q) (P if that sums to 0), and sibling x is accepted iff
// m Q_x S < R_x 2^69 (S = sum R, exact 128-bit integers); a rejection updates
// R <- max(0, floor(R 2^40 / S) - Q) (kept if that sums to 0).  R is never stored: every
// element is recomputed from p, q and the short scalar history {S_j, keep_j} held in shared
// memory, so the kernel needs no workspace and each pass is one streaming read of the p and
// q rows of the node.  All sums are exact uint64, so the result is bit-identical to the
// oracle regardless of reduction order.
//
// md_kv_compact: after acceptance the K/V rows of the accepted path (cache positions
// base + nodes[i]) move to base + 1 + i.  One CTA per (sequence, KV head) stages the rows in
// shared memory first, so overlapping source/destination sets are safe.
#include "md_common.cuh"
#include "md_internal.h"

namespace md {

constexpr int TR_THREADS = 512;
constexpr int TR_WARPS = TR_THREADS / 32;
constexpr int TR_MAXT = 16;
constexpr int TR_UNR = 8;

__device__ __forceinline__ uint64_t tgrid40(float x) {
  return x > 0.f ? __double2ull_rz(static_cast<double>(x) * 1099511627776.0) : 0ull;
}

// floor(R * 2^40 / S) exactly (R <= 2^40, 0 < S < 2^58): fp64 estimate, then 128-bit fix-up.
__device__ __forceinline__ uint64_t div40(uint64_t R, uint64_t S) {
  const unsigned __int128 num = static_cast<unsigned __int128>(R) << 40;
  uint64_t qe = __double2ull_rz(static_cast<double>(R) * 1099511627776.0 / static_cast<double>(S));
  unsigned __int128 prod = static_cast<unsigned __int128>(qe) * S;
  while (prod > num) {
    --qe;
    prod -= S;
  }
  while (prod + S <= num) {
    ++qe;
    prod += S;
  }
  return qe;
}

// Scalar history of the residual at the current node.
struct TreeHist {
  uint64_t S[TR_MAXT + 1];  // S[j] = sum R^(j)
  int keep[TR_MAXT];        // keep[j]: the update after R^(j) summed to 0, R^(j+1) = R^(j)
  int k;                    // current stage: R = R^(k); -1: the target is P (no rejection yet)
  int pfb;                  // R^(0) fell back to P
};

// Weight of one element at stage k (k = -1: P itself).
__device__ __forceinline__ uint64_t resid(uint64_t P, uint64_t Q, const TreeHist& h, int k) {
  if (k < 0) return P;
  uint64_t R = h.pfb ? P : (P > Q ? P - Q : 0ull);
  for (int j = 0; j < k; ++j) {
    if (h.keep[j]) continue;
    const uint64_t Rn = div40(R, h.S[j]);
    R = Rn > Q ? Rn - Q : 0ull;
  }
  return R;
}

struct TreeSmem {
  TreeHist h;
  uint64_t wsum[TR_WARPS];
  uint64_t total;
  float amax_v[TR_WARPS];
  int amax_i[TR_WARPS];
  int token;
  int kids[TR_MAXT];
  int nkids;
  int accepted;
};

// Row scans in the warp-strip layout of spec_accept.cu (round 2): contiguous warp
// segments streamed with coalesced 16-byte loads (4-byte when a row is not 16-byte aligned),
// TR_BATCH chunks in flight; the locate step re-streams the segment holding the draw with the
// whole block and one warp walks its sub-segment with a lane scan.  Weights are exact uint64
// (resid of stage k), so every sum and the drawn token are independent of the order.
constexpr int TR_BATCH = 4;

__device__ __forceinline__ uint64_t tw(float pv, float qv, const TreeHist& h, int k) {
  return resid(tgrid40(pv), k >= 0 ? tgrid40(qv) : 0ull, h, k);
}
__device__ __forceinline__ int tr_round_up(int x, int m) { return (x + m - 1) / m * m; }

// the VEC floats of p (and q when k >= 0) at [i, i + VEC), zeros past `end`
template <int VEC>
__device__ __forceinline__ void tr_load(const float* __restrict__ prow, const float* __restrict__ qrow, int i, int end,
                                        int k, float (&pv)[VEC], float (&qv)[VEC]) {
  if constexpr (VEC == 4) {
    if (i + 3 < end) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(prow + i));
      const float4 c = k >= 0 ? __ldg(reinterpret_cast<const float4*>(qrow + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
      pv[0] = a.x; pv[1] = a.y; pv[2] = a.z; pv[3] = a.w;
      qv[0] = c.x; qv[1] = c.y; qv[2] = c.z; qv[3] = c.w;
      return;
    }
  }
#pragma unroll
  for (int u = 0; u < VEC; ++u) {
    const bool in = i + u < end;
    pv[u] = in ? __ldg(prow + i + u) : 0.f;
    qv[u] = (in && k >= 0) ? __ldg(qrow + i + u) : 0.f;
  }
}

template <int VEC>
__device__ uint64_t tr_warp_sum(const float* prow, const float* qrow, int beg, int end, const TreeHist& h, int k) {
  constexpr int CH = 32 * VEC;
  const int lane = threadIdx.x & 31;
  uint64_t acc = 0;
  for (int c0 = beg; c0 < end; c0 += CH * TR_BATCH) {
    float pv[TR_BATCH][VEC], qv[TR_BATCH][VEC];
#pragma unroll
    for (int b = 0; b < TR_BATCH; ++b) tr_load<VEC>(prow, qrow, c0 + b * CH + lane * VEC, end, k, pv[b], qv[b]);
#pragma unroll
    for (int b = 0; b < TR_BATCH; ++b)
#pragma unroll
      for (int u = 0; u < VEC; ++u) acc += (c0 + b * CH + lane * VEC + u < end) ? tw(pv[b][u], qv[b][u], h, k) : 0ull;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// warp segment sums of stage k -> sm.wsum, total -> sm.total
template <int VEC>
__device__ void tr_sums(const float* prow, const float* qrow, int V, TreeSmem& sm, int k) {
  constexpr int CH = 32 * VEC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = tr_round_up((V + TR_WARPS - 1) / TR_WARPS, CH);
  const int beg = min(V, warp * seg), end = min(V, beg + seg);
  const uint64_t s = tr_warp_sum<VEC>(prow, qrow, beg, end, sm.h, k);
  __syncthreads();
  if (lane == 0) sm.wsum[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t total = 0;
    for (int w = 0; w < TR_WARPS; ++w) total += sm.wsum[w];
    sm.total = total;
  }
  __syncthreads();
}
__device__ __forceinline__ bool tr_vec_ok(const float* prow, const float* qrow) {
  return ((reinterpret_cast<uintptr_t>(prow) | reinterpret_cast<uintptr_t>(qrow)) & 15u) == 0;
}
__device__ void tree_sums(const float* prow, const float* qrow, int V, TreeSmem& sm, int k) {
  if (tr_vec_ok(prow, qrow)) tr_sums<4>(prow, qrow, V, sm, k);
  else tr_sums<1>(prow, qrow, V, sm, k);
}

// token = min{i : sum_{j<=i} W_j > t}, t < sm.total (right after tree_sums of the same stage)
template <int VEC>
__device__ int tr_locate(const float* prow, const float* qrow, int V, uint64_t t, TreeSmem& sm, int k) {
  constexpr int CH = 32 * VEC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = tr_round_up((V + TR_WARPS - 1) / TR_WARPS, CH);
  uint64_t run = 0;
  int ws = 0;
  for (int w = 0; w < TR_WARPS; ++w) {
    const uint64_t v = sm.wsum[w];
    if (run + v > t) {
      ws = w;
      break;
    }
    run += v;
  }
  const int base = min(V, ws * seg), send = min(V, base + seg);
  const int sub = tr_round_up((send - base + TR_WARPS - 1) / TR_WARPS, CH);
  const int sbeg = min(send, base + warp * sub), send2 = min(send, sbeg + sub);
  const uint64_t s = tr_warp_sum<VEC>(prow, qrow, sbeg, send2, sm.h, k);
  __syncthreads();
  if (lane == 0) sm.wsum[warp] = s;
  __syncthreads();
  int w2 = 0;
  for (int w = 0; w < TR_WARPS; ++w) {
    const uint64_t v = sm.wsum[w];
    if (run + v > t) {
      w2 = w;
      break;
    }
    run += v;
  }
  if (warp == w2) {
    const int b2 = min(send, base + w2 * sub), e2 = min(send, b2 + sub);
    for (int c0 = b2; c0 < e2; c0 += CH) {
      const int i = c0 + lane * VEC;
      float pv[VEC], qv[VEC];
      tr_load<VEC>(prow, qrow, i, e2, k, pv, qv);
      uint64_t w[VEC], ls = 0;
#pragma unroll
      for (int u = 0; u < VEC; ++u) {
        w[u] = (i + u < e2) ? tw(pv[u], qv[u], sm.h, k) : 0ull;
        ls += w[u];
      }
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
          int tokn = i;
#pragma unroll
          for (int u = 0; u < VEC; ++u) {
            r += w[u];
            if (r > t) {
              tokn = i + u;
              break;
            }
          }
          sm.token = tokn;
        }
        break;
      }
      run += tot;
    }
  }
  __syncthreads();
  return sm.token;
}
__device__ int tree_locate(const float* prow, const float* qrow, int V, uint64_t t, TreeSmem& sm, int k) {
  return tr_vec_ok(prow, qrow) ? tr_locate<4>(prow, qrow, V, t, sm, k) : tr_locate<1>(prow, qrow, V, t, sm, k);
}

__device__ int tree_argmax(const float* __restrict__ row, int V, TreeSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = tid; i < V; i += TR_THREADS) {
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
  __syncthreads();
  if (lane == 0) {
    sm.amax_v[warp] = bv;
    sm.amax_i[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    float v = sm.amax_v[0];
    int idx = sm.amax_i[0];
    for (int w = 1; w < TR_WARPS; ++w)
      if (sm.amax_v[w] > v || (sm.amax_v[w] == v && sm.amax_i[w] < idx)) {
        v = sm.amax_v[w];
        idx = sm.amax_i[w];
      }
    sm.token = (idx == 0x7fffffff) ? 0 : idx;
  }
  __syncthreads();
  return sm.token;
}

__global__ void __launch_bounds__(TR_THREADS) spec_accept_tree_kernel(
    const float* __restrict__ p, const float* __restrict__ q, const int32_t* __restrict__ tokens,
    const int32_t* __restrict__ parent, const uint32_t* __restrict__ rnd, int T, int V, int mode,
    int32_t* __restrict__ out_tokens, int32_t* __restrict__ num_accepted, int32_t* __restrict__ accepted_nodes,
    int32_t* __restrict__ committed_len) {
  __shared__ TreeSmem sm;
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x, tid = threadIdx.x;
  const int64_t Vl = V;
  const int32_t* tok = tokens + (int64_t)b * T;
  const int32_t* par = parent + (int64_t)b * T;
  const uint32_t* rb = rnd ? rnd + (int64_t)b * (T + 1) : nullptr;
#ifdef MD_DEBUG
  for (int c = tid; c < T; c += TR_THREADS)  // token ids < V, topological parents (parent[t] < t)
    MD_DCHECK(__ldg(tok + c) >= 0 && __ldg(tok + c) < V && (c == 0 || (__ldg(par + c) >= 0 && __ldg(par + c) < c)));
#endif
  int cur = 0, npath = 0, kr = 0, token = -1;
  int32_t* nodes_out = accepted_nodes ? accepted_nodes + (int64_t)b * T : nullptr;
  int32_t* out = out_tokens + (int64_t)b * T;
  for (;;) {
    const float* prow = p + ((int64_t)b * T + cur) * Vl;
    const float* qrow = q ? q + ((int64_t)b * T + cur) * Vl : nullptr;
    if (tid == 0) {
      int nk = 0;
      for (int c = cur + 1; c < T; ++c)
        if (__ldg(par + c) == cur) sm.kids[nk++] = c;
      sm.nkids = nk;
      sm.accepted = -1;
      sm.h.k = -1;
      sm.h.pfb = 0;
    }
    __syncthreads();
    const int nk = sm.nkids;
    if (mode == MD_ACCEPT_GREEDY) {
      const int a = tree_argmax(prow, V, sm);
      int nxt = -1;
      for (int i = 0; i < nk && nxt < 0; ++i)
        if (__ldg(tok + sm.kids[i]) == a) nxt = sm.kids[i];
      if (nxt < 0) {
        token = a;
        break;
      }
      if (tid == 0 && nodes_out) nodes_out[npath] = nxt;
      if (tid == 0) out[npath] = __ldg(tok + nxt);
      ++npath;
      cur = nxt;
      __syncthreads();
      continue;
    }
    // ---------------- SAMPLE: children in index order
    for (int i = 0; i < nk; ++i) {
      const int c = sm.kids[i];
      if (tid == 0) {
        const int x = __ldg(tok + c);
        const uint64_t m = __ldg(rb + kr) >> 3;
        bool ok;
        if (i == 0) {
          ok = static_cast<double>(m) * static_cast<double>(__ldg(qrow + x)) <
               static_cast<double>(__ldg(prow + x)) * 536870912.0;
        } else {
          const uint64_t S = sm.h.S[sm.h.k];
          const uint64_t Qx = tgrid40(__ldg(qrow + x));
          const uint64_t Rx = resid(tgrid40(__ldg(prow + x)), Qx, sm.h, sm.h.k);
          ok = S > 0 && static_cast<unsigned __int128>(m) * Qx * S < static_cast<unsigned __int128>(Rx) << 69;
        }
        if (ok) sm.accepted = c;
      }
      ++kr;
      __syncthreads();
      if (sm.accepted >= 0) break;
      // rejected: advance the residual
      if (i == 0) {
        if (tid == 0) sm.h.k = 0;
        __syncthreads();
        tree_sums(prow, qrow, V, sm, 0);
        if (tid == 0) {
          if (sm.total == 0) sm.h.pfb = 1;
          else sm.h.S[0] = sm.total;
        }
        __syncthreads();
        if (sm.h.pfb) {
          tree_sums(prow, qrow, V, sm, 0);
          if (tid == 0) sm.h.S[0] = sm.total;
          __syncthreads();
        }
      } else if (sm.h.S[sm.h.k] == 0) {
        // degenerate all-zero p row: R kept (reading Z24)
      } else {
        const int k = sm.h.k;
        if (tid == 0) sm.h.keep[k] = 0;
        __syncthreads();
        tree_sums(prow, qrow, V, sm, k + 1);  // candidate R^(k+1)
        if (tid == 0) {
          sm.h.keep[k] = sm.total == 0;
          sm.h.S[k + 1] = sm.total == 0 ? sm.h.S[k] : sm.total;
          sm.h.k = k + 1;
        }
        __syncthreads();
      }
    }
    const int acc = sm.accepted;
    if (acc >= 0) {
      if (tid == 0) {
        if (nodes_out) nodes_out[npath] = acc;
        out[npath] = __ldg(tok + acc);
      }
      ++npath;
      cur = acc;
      __syncthreads();
      continue;
    }
    // ---------------- final draw: from R^(k) (after rejections) or P (leaf)
    const int k = sm.h.k;
    tree_sums(prow, qrow, V, sm, k);
    const uint64_t total = sm.total;
    if (total == 0) {
      token = tree_argmax(prow, V, sm);
    } else {
      const uint64_t u = (static_cast<uint64_t>(__ldg(rb + T - 1)) << 32) | __ldg(rb + T);
      token = tree_locate(prow, qrow, V, __umul64hi(u, total), sm, k);
    }
    break;
  }
  for (int i = npath + tid; i < T; i += TR_THREADS) {
    out[i] = i == npath ? token : -1;
    if (nodes_out) nodes_out[i] = -1;
  }
  if (tid == 0) {
    num_accepted[b] = npath;
    if (committed_len != nullptr) committed_len[b] += npath + 1;
  }
}

// ---------------------------------------------------------------- KV compaction
constexpr int CMP_THREADS = 128;

__global__ void __launch_bounds__(CMP_THREADS) kv_compact_kernel(uint16_t* __restrict__ kc, uint16_t* __restrict__ vc,
                                                                 const int32_t* __restrict__ base,
                                                                 const int32_t* __restrict__ nodes, int nodes_stride,
                                                                 const int32_t* __restrict__ count, int Hkv, int d,
                                                                 int64_t sB, int64_t sH, int64_t sS) {
  extern __shared__ uint4 stage[];  // [2][nodes_stride][d/8]
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x / Hkv, h = blockIdx.x % Hkv;
  const int n = min(__ldg(count + b), nodes_stride);
  const int vpr = d >> 3;
  const int64_t row0 = b * sB + h * sH + (int64_t)__ldg(base + b) * sS;
  const int32_t* nb = nodes + (int64_t)b * nodes_stride;
  for (int e = threadIdx.x; e < n * vpr; e += CMP_THREADS) {
    const int i = e / vpr, c = (e - i * vpr) << 3;
    const int64_t src = row0 + (int64_t)__ldg(nb + i) * sS + c;
    stage[e] = *reinterpret_cast<const uint4*>(kc + src);
    stage[n * vpr + e] = *reinterpret_cast<const uint4*>(vc + src);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * vpr; e += CMP_THREADS) {
    const int i = e / vpr, c = (e - i * vpr) << 3;
    if (__ldg(nb + i) == i + 1) continue;  // already in place
    const int64_t dst = row0 + (int64_t)(i + 1) * sS + c;
    *reinterpret_cast<uint4*>(kc + dst) = stage[e];
    *reinterpret_cast<uint4*>(vc + dst) = stage[n * vpr + e];
  }
}

}  // namespace md

extern "C" md_status md_spec_accept_tree(const float* p, const float* q, const int32_t* tokens,
                                         const int32_t* parent, const uint32_t* rnd, int32_t B, int32_t T, int32_t V,
                                         md_accept_mode mode, int32_t* out_tokens, int32_t* num_accepted,
                                         int32_t* accepted_nodes, int32_t* committed_len_inout, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(mode == MD_ACCEPT_SAMPLE || mode == MD_ACCEPT_GREEDY, MD_ERR_INVALID_ARG,
             "md_spec_accept_tree: bad mode");
  MD_REQUIRE(B >= 1 && V >= 1, MD_ERR_INVALID_ARG, "md_spec_accept_tree: B and V must be >= 1");
  MD_REQUIRE(T >= 1 && T <= TR_MAXT, MD_ERR_UNSUPPORTED, "md_spec_accept_tree: T must be in [1, 16]");
  MD_REQUIRE(p != nullptr && tokens != nullptr && parent != nullptr && out_tokens != nullptr &&
                 num_accepted != nullptr,
             MD_ERR_INVALID_ARG, "md_spec_accept_tree: NULL p / tokens / parent / out_tokens / num_accepted");
  MD_REQUIRE(mode == MD_ACCEPT_GREEDY || (rnd != nullptr && q != nullptr), MD_ERR_INVALID_ARG,
             "md_spec_accept_tree: NULL rnd / q (SAMPLE)");
  launch_pdl(spec_accept_tree_kernel, dim3(B), dim3(TR_THREADS), 0, (cudaStream_t)stream, p, q, tokens, parent, rnd,
             (int)T, (int)V, static_cast<int>(mode), out_tokens, num_accepted, accepted_nodes, committed_len_inout);
  return check_launch("md_spec_accept_tree");
}

extern "C" md_status md_kv_compact(const md_kv_cache* c, const int32_t* base, const int32_t* nodes,
                                   int32_t nodes_stride, const int32_t* count, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(c != nullptr && base != nullptr && nodes != nullptr && count != nullptr, MD_ERR_INVALID_ARG,
             "md_kv_compact: NULL argument");
  MD_REQUIRE(c->k != nullptr && c->v != nullptr && c->batch >= 1 && c->num_kv_heads >= 1, MD_ERR_INVALID_ARG,
             "md_kv_compact: bad cache");
  MD_REQUIRE(nodes_stride >= 1 && nodes_stride <= TR_MAXT, MD_ERR_UNSUPPORTED,
             "md_kv_compact: nodes_stride must be in [1, 16]");
  MD_REQUIRE(c->head_dim >= 8 && c->head_dim % 8 == 0 && c->head_dim <= 256, MD_ERR_INVALID_ARG,
             "md_kv_compact: head_dim must be a multiple of 8 in [8, 256]");
  MD_REQUIRE(c->stride_b % 8 == 0 && c->stride_h % 8 == 0 && c->stride_s % 8 == 0 && aligned16(c->k) &&
                 aligned16(c->v),
             MD_ERR_INVALID_ARG, "md_kv_compact: cache must be 16-byte aligned with strides multiple of 8");
  const size_t smem = (size_t)2 * nodes_stride * c->head_dim * 2;
  launch_pdl(kv_compact_kernel, dim3(c->batch * c->num_kv_heads), dim3(CMP_THREADS), smem, (cudaStream_t)stream,
             static_cast<uint16_t*>(c->k), static_cast<uint16_t*>(c->v), base, nodes, (int)nodes_stride, count,
             (int)c->num_kv_heads, (int)c->head_dim, (int64_t)c->stride_b, (int64_t)c->stride_h,
             (int64_t)c->stride_s);
  return check_launch("md_kv_compact");
}

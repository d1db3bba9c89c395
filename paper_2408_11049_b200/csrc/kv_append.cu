// kv_append.cu — md_kv_append: scatter the new K/V rows of a pass into the shared cache
// (SURVEY §8(a) row a1).  Pure bandwidth: one thread moves one 16-byte vector, the
// source [B][T][Hkv][d] is read fully coalesced and each destination row (d bf16 =
// 128/256 B) is written contiguously.
#include "md_common.cuh"
#include "md_internal.h"

namespace md {

__global__ void __launch_bounds__(256) kv_append_kernel(uint16_t* __restrict__ kc, uint16_t* __restrict__ vc,
                                                        const uint16_t* __restrict__ kn,
                                                        const uint16_t* __restrict__ vn,
                                                        const int32_t* __restrict__ start, int start_off, int T,
                                                        int Hkv, int d, int cap,
                                                        int64_t sB, int64_t sH, int64_t sS, int64_t nvec) {
  pdl_trigger();
  pdl_wait();
  const int vec_per_row = d >> 3;  // 8 bf16 per 16-byte vector
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / vec_per_row;  // row of [B][T][Hkv]
    const int c = static_cast<int>(i - row * vec_per_row) << 3;
    const int h = static_cast<int>(row % Hkv);
    const int64_t bt = row / Hkv;
    const int t = static_cast<int>(bt % T);
    const int b = static_cast<int>(bt / T);
    const int s0 = __ldg(start + b) + start_off;
    MD_DCHECK(s0 >= 0 && s0 + T <= cap);  // rows [start, start + T) inside the cache
    const int64_t dst = b * sB + h * sH + (int64_t)(s0 + t) * sS + c;
    const uint4 kv = __ldg(reinterpret_cast<const uint4*>(kn + row * d + c));
    const uint4 vv = __ldg(reinterpret_cast<const uint4*>(vn + row * d + c));
    *reinterpret_cast<uint4*>(kc + dst) = kv;
    *reinterpret_cast<uint4*>(vc + dst) = vv;
  }
}

}  // namespace md

extern "C" md_status md_kv_append(const md_kv_cache* c, const void* k_new, const void* v_new, int32_t T,
                                  const int32_t* start_pos, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(c != nullptr && k_new != nullptr && v_new != nullptr && start_pos != nullptr, MD_ERR_INVALID_ARG,
             "md_kv_append: NULL argument");
  MD_REQUIRE(c->k != nullptr && c->v != nullptr, MD_ERR_INVALID_ARG, "md_kv_append: NULL cache pointer");
  MD_REQUIRE(c->batch >= 1 && c->num_kv_heads >= 1 && c->capacity >= 1 && T >= 1, MD_ERR_INVALID_ARG,
             "md_kv_append: batch, num_kv_heads, capacity and T must be >= 1");
  MD_REQUIRE(c->head_dim >= 8 && c->head_dim % 8 == 0, MD_ERR_INVALID_ARG,
             "md_kv_append: head_dim must be a positive multiple of 8");
  MD_REQUIRE(T <= c->capacity, MD_ERR_INVALID_ARG, "md_kv_append: T exceeds capacity");
  MD_REQUIRE(c->stride_b % 8 == 0 && c->stride_h % 8 == 0 && c->stride_s % 8 == 0, MD_ERR_INVALID_ARG,
             "md_kv_append: cache strides must be multiples of 8 elements");
  MD_REQUIRE(aligned16(c->k) && aligned16(c->v) && aligned16(k_new) && aligned16(v_new), MD_ERR_INVALID_ARG,
             "md_kv_append: pointers must be 16-byte aligned");
  return launch_kv_append(c, k_new, v_new, T, start_pos, 0, (cudaStream_t)stream);
}

namespace md {
// rows [start[b] + start_off, + T) of every (b, kv head); start_off = -T with start = kv_len is
// the append of the fused attention calls when their kernel cannot fuse it (attn.cu)
md_status launch_kv_append(const md_kv_cache* c, const void* k_new, const void* v_new, int T, const int32_t* start,
                           int start_off, cudaStream_t stream) {
  const int64_t nvec = (int64_t)c->batch * T * c->num_kv_heads * (c->head_dim / 8);
  const int threads = 256;
  int64_t blocks = (nvec + threads - 1) / threads;
  const int64_t cap_blocks = (int64_t)device_sm_count() * 16;
  if (blocks > cap_blocks) blocks = cap_blocks;
  launch_pdl(kv_append_kernel, dim3(static_cast<unsigned>(blocks)), dim3(threads), 0, stream,
             static_cast<uint16_t*>(c->k), static_cast<uint16_t*>(c->v), static_cast<const uint16_t*>(k_new),
             static_cast<const uint16_t*>(v_new), start, start_off, (int)T, (int)c->num_kv_heads, (int)c->head_dim,
             (int)c->capacity,
             (int64_t)c->stride_b, (int64_t)c->stride_h, (int64_t)c->stride_s, nvec);
  return check_launch("md_kv_append");
}

}  // namespace md

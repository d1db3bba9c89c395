// synth_gen.cu — GPU twin of synth/__init__.py's counter-hash input generators
// (inputs only: no arithmetic of the method).  Bit-identical to the numpy version
// (tests/test_gpu_synth.py), so multi-GB caches are produced in HBM and any slice
// can be regenerated on the host for the oracle.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

uint64_t key_of(uint64_t seed, uint64_t tensor) {
  return mix64(seed * 0x9E3779B97F4A7C15ull + (tensor << 56) + tensor * 0xD1B54A32D192ED03ull);
}

constexpr uint64_t POSMAX = 1ull << 24;
constexpr uint64_t T_KCACHE = 1, T_DIR = 7, T_NEEDLE = 8;

__device__ __forceinline__ int grid_k(uint64_t key, uint64_t idx) { return (int)(mix64(idx + key) >> 58) - 32; }

__device__ __forceinline__ uint16_t bf16_of_k(int k) {
  const float f = (float)k / 32.0f;
  return (uint16_t)(__float_as_uint(f) >> 16);
}

// (b0, h0, Htot): the tensor is the slice [b0, b0 + B) x [h0, h0 + Hkv) of a cache with Htot KV
// heads, so a tensor-parallel / batch shard holds exactly the values of the full cache's slice
__global__ void fill_cache_kernel(uint16_t* base, int B, int Hkv, int d, long long sB, long long sH, long long sS,
                                  int pos0, int npos, uint64_t key, uint64_t key_dir, uint64_t key_needle,
                                  int peaky, int sink, int a_k, int needle_period, int b0, int h0, int Htot) {
  const long long total = (long long)B * Hkv * npos * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % d);
    long long r = i / d;
    const int pl = (int)(r % npos);
    r /= npos;
    const int h = (int)(r % Hkv);
    const int b = (int)(r / Hkv);
    const uint64_t pos = (uint64_t)(pos0 + pl);
    const uint64_t unit = (uint64_t)(b0 + b) * Htot + (h0 + h);
    int k = grid_k(key, (unit * POSMAX + pos) * d + c);
    if (peaky) {
      const bool needle = (mix64(unit * POSMAX + pos + key_needle) % (uint64_t)needle_period) == 0;
      if ((long long)pos < sink || needle) {
        const int sgn = (mix64(unit * d + c + key_dir) >> 63) ? 1 : -1;
        k += a_k * sgn;
      }
    }
    base[b * sB + h * sH + (long long)(pos0 + pl) * sS + c] = bf16_of_k(k);
  }
}

__global__ void fill_q_kernel(uint16_t* q, int B, int T, int Hq, int Hkv, int d, uint64_t key, uint64_t key_dir,
                              int peaky, int a_q) {
  const long long total = (long long)B * T * Hq * d;
  const int g = Hq / Hkv;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int k = grid_k(key, (uint64_t)i);
    if (peaky) {
      const int c = (int)(i % d);
      const int h = (int)((i / d) % Hq);
      const int b = (int)(i / ((long long)d * Hq * T));
      const uint64_t unit = (uint64_t)b * Hkv + h / g;
      const int sgn = (mix64(unit * d + c + key_dir) >> 63) ? 1 : -1;
      k += a_q * sgn;
    }
    q[i] = bf16_of_k(k);
  }
}

// off-grid bf16 bits (synth.offgrid_bits_from_hash): sign, exponent 120..126, 7-bit mantissa
__device__ __forceinline__ uint16_t offgrid_bits(uint64_t h) {
  const uint16_t sign = (uint16_t)((h >> 63) & 1u);
  const uint16_t ex = (uint16_t)(((h >> 40) & 0xFFFFu) % 7u) + 120u;
  const uint16_t man = (uint16_t)((h >> 20) & 0x7Fu);
  return (uint16_t)((sign << 15) | (ex << 7) | man);
}

__global__ void fill_cache_offgrid_kernel(uint16_t* base, int B, int Hkv, int d, long long sB, long long sH,
                                          long long sS, int pos0, int npos, uint64_t key, int b0, int h0, int Htot) {
  const long long total = (long long)B * Hkv * npos * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % d);
    long long r = i / d;
    const int pl = (int)(r % npos);
    r /= npos;
    const int h = (int)(r % Hkv);
    const int b = (int)(r / Hkv);
    const uint64_t unit = (uint64_t)(b0 + b) * Htot + (h0 + h);
    const uint64_t pos = (uint64_t)(pos0 + pl);
    base[b * sB + h * sH + (long long)(pos0 + pl) * sS + c] = offgrid_bits(mix64((unit * POSMAX + pos) * d + c + key));
  }
}

__global__ void fill_flat_offgrid_kernel(uint16_t* x, long long total, uint64_t key) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = offgrid_bits(mix64((uint64_t)i + key));
}

unsigned grid_for(long long total) {
  long long blocks = (total + 255) / 256;
  return (unsigned)(blocks > 65536 ? 65536 : (blocks < 1 ? 1 : blocks));
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int mds_fill_cache_slice(
    void* base, int B, int Hkv, int d, long long sB, long long sH, long long sS, int pos0, int npos,
    unsigned long long seed, int tensor, int peaky, int sink, int a_k, int needle_period, int b0, int h0, int Htot,
    void* stream) {
  const long long total = (long long)B * Hkv * npos * d;
  if (total <= 0) return 0;
  fill_cache_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      (uint16_t*)base, B, Hkv, d, sB, sH, sS, pos0, npos, key_of(seed, tensor), key_of(seed, T_DIR),
      key_of(seed, T_NEEDLE), peaky && tensor == (int)T_KCACHE, sink, a_k, needle_period, b0, h0, Htot);
  return (int)cudaGetLastError();
}

extern "C" __attribute__((visibility("default"))) int mds_fill_cache(void* base, int B, int Hkv, int d, long long sB, long long sH, long long sS, int pos0,
                              int npos, unsigned long long seed, int tensor, int peaky, int sink, int a_k,
                              int needle_period, void* stream) {
  return mds_fill_cache_slice(base, B, Hkv, d, sB, sH, sS, pos0, npos, seed, tensor, peaky, sink, a_k, needle_period,
                              0, 0, Hkv, stream);
}

// Queries [B][T][Hq][d] (T = 1 for draft queries); also the new K/V rows [B][T][Hkv][d]
// when called with Hq = Hkv and peaky = 0.
extern "C" __attribute__((visibility("default"))) int mds_fill_q(void* q, int B, int T, int Hq, int Hkv, int d, unsigned long long seed, int tensor,
                          int peaky, int a_q, void* stream) {
  const long long total = (long long)B * T * Hq * d;
  if (total <= 0) return 0;
  fill_q_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((uint16_t*)q, B, T, Hq, Hkv, d,
                                                                    key_of(seed, tensor), key_of(seed, T_DIR),
                                                                    peaky, a_q);
  return (int)cudaGetLastError();
}

// off-grid twins of synth.kv_cache_bits_offgrid / synth.flat_bits_offgrid
extern "C" __attribute__((visibility("default"))) int mds_fill_cache_offgrid(
    void* base, int B, int Hkv, int d, long long sB, long long sH, long long sS, int pos0, int npos,
    unsigned long long seed, int tensor, int b0, int h0, int Htot, void* stream) {
  const long long total = (long long)B * Hkv * npos * d;
  if (total <= 0) return 0;
  fill_cache_offgrid_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      (uint16_t*)base, B, Hkv, d, sB, sH, sS, pos0, npos, key_of(seed, tensor), b0, h0, Htot);
  return (int)cudaGetLastError();
}

extern "C" __attribute__((visibility("default"))) int mds_fill_flat_offgrid(void* x, long long total,
                                                                         unsigned long long seed, int tensor,
                                                                         void* stream) {
  if (total <= 0) return 0;
  fill_flat_offgrid_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((uint16_t*)x, total,
                                                                              key_of(seed, tensor));
  return (int)cudaGetLastError();
}

// tc_probe.cu — one-CTA check of the tcgen05 operand layouts the verify kernel uses:
//   S^T[128 keys][NP] = K[128][128 d] (K-major, SW128) . Q^T (Q [NP][128 d] K-major, SW128)
//   O^T[128 d][NP]    = V^T (V [128 keys][128 d] read MN-major, SW128) . P^T (P^T MN-major,
//                       no swizzle: 8x8 core matrices, K stride 128 B, N stride 2 KB)
// both accumulated in TMEM and read back with tcgen05.ld 32x32b; compared with a host fp64
// reference.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tc_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int NP = 32, D = 128, KT = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// byte offset of (row r, element c in [0,64)) in a [rows][128 B] SW128 slab
__host__ __device__ inline uint32_t sw128(int r, int c) { return r * 128 + ((((c * 2) >> 4) ^ (r & 7)) << 4) + (c * 2 & 15); }

__global__ void probe(const uint16_t* K, const uint16_t* V, const uint16_t* Q, const uint16_t* P, float* S_out,
                      float* O_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ks = sm;                    // [2 slabs][128][128 B]
  uint8_t* vs = ks + 2 * KT * 128;     // same
  uint8_t* qs = vs + 2 * KT * 128;     // [2 slabs][NP][128 B]
  uint8_t* ps = qs + 2 * NP * 128;     // P^T: core (n/8, k/8) at (n/8)*2048 + (k/8)*128
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < KT * D; i += blockDim.x) {
    const int r = i / D, c = i % D;
    *(uint16_t*)(ks + (c / 64) * KT * 128 + sw128(r, c % 64)) = K[i];
    *(uint16_t*)(vs + (c / 64) * KT * 128 + sw128(r, c % 64)) = V[i];
  }
  for (int i = tid; i < NP * D; i += blockDim.x) {
    const int r = i / D, c = i % D;
    *(uint16_t*)(qs + (c / 64) * NP * 128 + sw128(r, c % 64)) = Q[i];
  }
  for (int i = tid; i < NP * KT; i += blockDim.x) {  // P [n][k]
    const int n = i / KT, k = i % KT;
    *(uint16_t*)(ps + (n / 8) * 2048 + (k / 8) * 128 + (k % 8) * 16 + (n % 8) * 2) = P[i];
  }
  if (tid == 0) mbar_init(&bar, 1);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tS = tbase, tO = tbase + NP;
  if (tid == 0) {
    const uint32_t id1 = idesc_bf16(128, NP, 0, 0);
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint32_t off = (kk / 4) * 0 + (kk % 4) * 32;
      const uint64_t a = make_desc(smem_u32(ks) + (kk / 4) * KT * 128 + off, 16, 1024, 2);
      const uint64_t b = make_desc(smem_u32(qs) + (kk / 4) * NP * 128 + off, 16, 1024, 2);
      mma(tS, a, b, id1, kk > 0);
    }
    const uint32_t id2 = idesc_bf16(128, NP, 1, 1);
    for (int kk = 0; kk < KT / 16; ++kk) {
      // A = V^T, MN-major SW128: K step of 16 keys = 2 KB; LBO = MN-repeat (next 64 d = next slab)
      const uint64_t a = make_desc(smem_u32(vs) + kk * 2048, KT * 128, 1024, 2);
      // B = P^T, MN-major no swizzle: K step of 16 keys = 2 core matrices = 256 B
      const uint64_t b = make_desc(smem_u32(ps) + kk * 256, 128, 2048, 0);
      mma(tO, a, b, id2, kk > 0);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid / 32, lane = tid % 32;
  if (warp < 4) {
    uint32_t v[NP];
    const uint32_t taddr = ((uint32_t)(warp * 32) << 16);
#define LD32(base, arr)                                                                                              \
  asm volatile(                                                                                                      \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                     \
      : "=r"(arr[0]), "=r"(arr[1]), "=r"(arr[2]), "=r"(arr[3]), "=r"(arr[4]), "=r"(arr[5]), "=r"(arr[6]),            \
        "=r"(arr[7]), "=r"(arr[8]), "=r"(arr[9]), "=r"(arr[10]), "=r"(arr[11]), "=r"(arr[12]), "=r"(arr[13]),        \
        "=r"(arr[14]), "=r"(arr[15]), "=r"(arr[16]), "=r"(arr[17]), "=r"(arr[18]), "=r"(arr[19]), "=r"(arr[20]),     \
        "=r"(arr[21]), "=r"(arr[22]), "=r"(arr[23]), "=r"(arr[24]), "=r"(arr[25]), "=r"(arr[26]), "=r"(arr[27]),     \
        "=r"(arr[28]), "=r"(arr[29]), "=r"(arr[30]), "=r"(arr[31])                                                   \
      : "r"(base));
    LD32(tS + taddr, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < NP; ++j) S_out[(warp * 32 + lane) * NP + j] = __uint_as_float(v[j]);
    LD32(tO + taddr, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < NP; ++j) O_out[(warp * 32 + lane) * NP + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}
static double bf2d(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main() {
  srand(1);
  auto rnd = [] { return f2bf((float)((rand() % 64) - 32) / 32.f); };
  std::vector<uint16_t> K(KT * D), V(KT * D), Q(NP * D), P(NP * KT);
  for (auto& x : K) x = rnd();
  for (auto& x : V) x = rnd();
  for (auto& x : Q) x = rnd();
  for (auto& x : P) x = rnd();
  uint16_t *dK, *dV, *dQ, *dP;
  float *dS, *dO;
  cudaMalloc(&dK, K.size() * 2);
  cudaMalloc(&dV, V.size() * 2);
  cudaMalloc(&dQ, Q.size() * 2);
  cudaMalloc(&dP, P.size() * 2);
  cudaMalloc(&dS, KT * NP * 4);
  cudaMalloc(&dO, D * NP * 4);
  cudaMemcpy(dK, K.data(), K.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Q.data(), Q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 2 * KT * 128 * 2 + 2 * NP * 128 + NP * KT * 2;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dK, dV, dQ, dP, dS, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> S(KT * NP), O(D * NP);
  cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0;
  for (int k = 0; k < KT; ++k)
    for (int n = 0; n < NP; ++n) {
      double ref = 0;
      for (int c = 0; c < D; ++c) ref += bf2d(K[k * D + c]) * bf2d(Q[n * D + c]);
      es = fmax(es, fabs(ref - S[k * NP + n]));
    }
  for (int d = 0; d < D; ++d)
    for (int n = 0; n < NP; ++n) {
      double ref = 0;
      for (int k = 0; k < KT; ++k) ref += bf2d(V[k * D + d]) * bf2d(P[n * KT + k]);
      eo = fmax(eo, fabs(ref - O[d * NP + n]));
    }
  printf("tc_probe NP=%d: max|S^T err| = %.3g, max|O^T err| = %.3g  (S[0][0]=%f O[0][0]=%f)\n", NP, es, eo, S[0],
         O[0]);
  return (es < 1e-3 && eo < 1e-3) ? 0 : 2;
}

// Microbenchmark: does the TMA box shape of the attention kernels cost HBM bandwidth?  Two
// buffers (K, V) of 256-byte rows (head_dim 128, bf16) are streamed tile by tile (64 rows =
// 16 KB of K + 16 KB of V per stage, 3 stages, 2 CTAs / SM, contiguous equal shares) with
//   A: two 2-D boxes {64 cols, 64 rows} per buffer and tile, SWIZZLE_128B (the kernels' layout:
//      each box reads 128 of every 256 bytes),
//   B: one 3-D box {64, 2, 64} per buffer and tile over the [rows][2][64] view, SWIZZLE_128B
//      (the same bytes, one contiguous 16 KB request),
//   C: one 1-D bulk copy of 16 KB per buffer and tile (no tensor map),
// each with L2 promotion 256B and none, back to back over 4 rotated buffer pairs with
// programmatic dependent launch, timed with CUDA events.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_pattern tma_pattern.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                     uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}

constexpr int TILE = 16384, STAGE = 2 * TILE, NSTAGE = 3;

struct Maps {
  CUtensorMap k, v;
};

__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ Maps mp, const uint8_t* kb,
                                                    const uint8_t* vb, int tiles, int mode, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NSTAGE * STAGE);
  uint64_t* empty = full + NSTAGE;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int a = (int)((long long)tiles * blockIdx.x / gridDim.x), e = (int)((long long)tiles * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x == 32) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int it = 0;
    for (int t = a; t < e; ++t, ++it) {
      const int s = it % NSTAGE;
      uint8_t* kt = sm + s * STAGE;
      uint8_t* vt = kt + TILE;
      mbar_wait(&empty[s], ((it / NSTAGE) & 1) ^ 1);
      mbar_expect(&full[s], STAGE);
      if (mode == 0) {
        for (int sub = 0; sub < 2; ++sub) {
          tma2(kt + sub * 8192, &mp.k, &full[s], sub * 64, t * 64, pol);
          tma2(vt + sub * 8192, &mp.v, &full[s], sub * 64, t * 64, pol);
        }
      } else if (mode == 1) {
        tma3(kt, &mp.k, &full[s], 0, 0, t * 64, pol);
        tma3(vt, &mp.v, &full[s], 0, 0, t * 64, pol);
      } else {
        bulk_g2s(kt, kb + (size_t)t * TILE, TILE, &full[s], pol);
        bulk_g2s(vt, vb + (size_t)t * TILE, TILE, &full[s], pol);
      }
    }
  } else if (threadIdx.x == 0) {
    int acc = 0, it = 0;
    for (int t = a; t < e; ++t, ++it) {
      const int s = it % NSTAGE;
      mbar_wait(&full[s], (it / NSTAGE) & 1);
      acc += reinterpret_cast<const int*>(sm + s * STAGE)[it & 63];
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x7fffffff) sink[0] = acc;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static void make_map(CUtensorMap* m, void* base, size_t rows, int mode, CUtensorMapL2promotion prom) {
  if (mode == 0) {
    cuuint64_t dims[2] = {128, rows};
    cuuint64_t str[1] = {256};
    cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[3] = {64, 2, rows};
    cuuint64_t str[2] = {128, 256};
    cuuint32_t box[3] = {64, 2, 64}, es[3] = {1, 1, 1};
    enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
}

int main() {
  const size_t maxrows = (size_t)4300 << 20 >> 8;  // 4.3 GB per buffer (K + V = 8.6 GB)
  std::vector<uint8_t*> kb(4), vb(4);
  for (int i = 0; i < 4; ++i) {
    if (cudaMalloc(&kb[i], maxrows * 256) != cudaSuccess || cudaMalloc(&vb[i], maxrows * 256) != cudaSuccess) {
      printf("alloc failed\n");
      return 1;
    }
    cudaMemset(kb[i], 1, maxrows * 256);
    cudaMemset(vb[i], 1, maxrows * 256);
  }
  int* sink;
  cudaMalloc(&sink, 4);
  const int smem = NSTAGE * STAGE + 1024 + 64;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"A_2x2d_boxes", "B_3d_box", "C_bulk"};
  const size_t mbs[] = {270, 8600};
  for (size_t mb : mbs) {
    const int tiles = (int)((mb << 20) / STAGE);
    for (int prom = 0; prom < 2; ++prom)
      for (int mode = 0; mode < 3; ++mode) {
        if (mode == 2 && prom == 1) continue;
        std::vector<Maps> maps(4);
        for (int i = 0; i < 4; ++i) {
          make_map(&maps[i].k, kb[i], (size_t)tiles * 64, mode, prom ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
          make_map(&maps[i].v, vb[i], (size_t)tiles * 64, mode, prom ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(296);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const int reps = mb > 1000 ? 16 : 64;
        for (int i = 0; i < 8; ++i)
          cudaLaunchKernelEx(&cfg, stream_kernel, maps[i % 4], (const uint8_t*)kb[i % 4], (const uint8_t*)vb[i % 4], tiles, mode, sink);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i)
          cudaLaunchKernelEx(&cfg, stream_kernel, maps[i % 4], (const uint8_t*)kb[i % 4], (const uint8_t*)vb[i % 4], tiles, mode, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 1e3 / reps, bytes = (double)tiles * STAGE;
        printf("{\"MB\": %zu, \"pattern\": \"%s\", \"l2_promotion\": \"%s\", \"us\": %.2f, \"GBps\": %.0f}\n", mb, names[mode],
               prom ? "none" : "256B", us, bytes / us / 1e3);
      }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

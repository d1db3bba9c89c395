// Microbenchmark: speed of light of a pure HBM read stream as a function of the bytes one
// launch moves (the draft call moves 270 MB, a verify call 8.6 GB).  A persistent grid of
// CTAS_PER_SM x 148 CTAs streams contiguous equal shares of a buffer with 1-D bulk copies
// (cp.async.bulk.shared::cluster.global, 32 KB per stage, mbarrier ring, L2 evict_first), the
// consumers touch one word per stage.  Launched back to back over 4 rotated buffers (no L2
// reuse), with and without programmatic dependent launch (griddepcontrol), timed with CUDA
// events.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_sol read_sol.cu -lcuda
#include <cuda_runtime.h>

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

constexpr int STAGE = 32768;

template <int NSTAGE>
__global__ void __launch_bounds__(64) read_kernel(const uint8_t* buf, size_t bytes, int* sink, int pdl) {
  extern __shared__ __align__(128) uint8_t sm[];
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
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const size_t nst = bytes / STAGE;
  const size_t a = nst * blockIdx.x / gridDim.x, e = nst * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 32) {  // producer
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int it = 0;
    for (size_t i = a; i < e; ++i, ++it) {
      const int s = it % NSTAGE;
      mbar_wait(&empty[s], ((it / NSTAGE) & 1) ^ 1);
      mbar_expect(&full[s], STAGE);
      bulk_g2s(sm + s * STAGE, buf + i * STAGE, STAGE, &full[s], pol);
    }
  } else if (threadIdx.x == 0) {  // consumer
    int acc = 0, it = 0;
    for (size_t i = a; i < e; ++i, ++it) {
      const int s = it % NSTAGE;
      mbar_wait(&full[s], (it / NSTAGE) & 1);
      acc += reinterpret_cast<const int*>(sm + s * STAGE)[it & 63];
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x7fffffff) sink[0] = acc;
  }
}

template <int NSTAGE>
float run(std::vector<uint8_t*>& bufs, size_t bytes, int ctas_per_sm, int pdl, int reps, int* sink) {
  const int smem = NSTAGE * STAGE + 2 * NSTAGE * 8;
  cudaFuncSetAttribute(read_kernel<NSTAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148 * ctas_per_sm);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int i = 0; i < 8; ++i) cudaLaunchKernelEx(&cfg, read_kernel<NSTAGE>, (const uint8_t*)bufs[i % 4], bytes, sink, pdl);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, read_kernel<NSTAGE>, (const uint8_t*)bufs[i % 4], bytes, sink, pdl);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;  // us per launch
}

int main() {
  const size_t maxb = size_t(8600) << 20;
  std::vector<uint8_t*> bufs(4);
  for (auto& p : bufs) {
    if (cudaMalloc(&p, maxb) != cudaSuccess) {
      printf("alloc failed\n");
      return 1;
    }
    cudaMemset(p, 1, maxb);
  }
  int* sink;
  cudaMalloc(&sink, 4);
  const size_t sizes_mb[] = {34, 68, 135, 270, 540, 1080, 2160, 8600};
  for (size_t mb : sizes_mb) {
    const size_t bytes = (mb << 20) / STAGE * STAGE;
    const int reps = mb >= 2000 ? 16 : 64;
    for (int pdl = 0; pdl < 2; ++pdl) {
      const float u1 = run<6>(bufs, bytes, 1, pdl, reps, sink);
      const float u2 = run<3>(bufs, bytes, 2, pdl, reps, sink);
      const float u3 = run<2>(bufs, bytes, 3, pdl, reps, sink);
      printf("{\"MB\": %zu, \"pdl\": %d, \"us_1x6\": %.2f, \"GBps_1x6\": %.0f, \"us_2x3\": %.2f, \"GBps_2x3\": %.0f, "
             "\"us_3x2\": %.2f, \"GBps_3x2\": %.0f}\n",
             mb, pdl, u1, bytes / u1 / 1e3, u2, bytes / u2 / 1e3, u3, bytes / u3 / 1e3);
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}

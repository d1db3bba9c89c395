// Does compute-sanitizer racecheck model cp.async completion through an mbarrier?
// One producer warp copies 32 x 16 B into shared memory with cp.async and signals each lane's
// completion with cp.async.mbarrier.arrive.noinc on a barrier that expects 32 arrivals; one
// consumer warp waits on the barrier and reads the data (the ordering the index-list draft
// relies on, attn.cu produce_segment).  Variant 1 adds the CTA-wide reuse pattern: the consumer
// releases the buffer through a second barrier and the producer refills it (4 rounds).
// A racecheck report here is a tool limitation, not a kernel race.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o cpasync_mbar_race cpasync_mbar_race.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
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

__global__ void k(const uint4* src, int* out, int rounds) {
  __shared__ __align__(16) uint4 buf[32];
  __shared__ uint64_t full, empty;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&full, 32);
    mbar_init(&empty, 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int acc = 0;
  for (int r = 0; r < rounds; ++r) {
    if (warp == 0) {
      mbar_wait(&empty, (r & 1) ^ 1);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&buf[lane])), "l"(src + r * 32 + lane)
                   : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full)) : "memory");
    } else {
      mbar_wait(&full, r & 1);
      acc += buf[(lane + r) & 31].x;
      mbar_arrive(&empty);
    }
  }
  if (warp == 1) out[lane] = acc;
}

int main() {
  uint4* src;
  int* out;
  cudaMalloc(&src, 4 * 32 * 16);
  cudaMemset(src, 1, 4 * 32 * 16);
  cudaMalloc(&out, 32 * 4);
  k<<<1, 64>>>(src, out, 1);
  k<<<1, 64>>>(src, out, 4);
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

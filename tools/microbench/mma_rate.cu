// Microbenchmark: legacy mma.sync m16n8k16 bf16 throughput on sm_100a, and a plain
// 128-bit streaming-read kernel, to decide the math pipe for the attention kernels.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__global__ void mma_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 17;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 12345.f) out[0] = s;
}

__global__ void stream_read(const int4* __restrict__ p, size_t n, int* out) {
  int acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * 4) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (i + u * stride < n) ? p[i + u * stride] : make_int4(0,0,0,0);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  printf("name=%s sms=%d l2=%d smem/block optin=%zu clock(kHz)=%d\n", pr.name, pr.multiProcessorCount,
         pr.l2CacheSize, pr.sharedMemPerBlockOptin, pr.clockRate);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    int iters = 4096; int blocks = pr.multiProcessorCount * 2;
    mma_loop<<<blocks, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    mma_loop<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * blocks * warps;
    printf("mma.sync m16n8k16 bf16: warps/block=%d blocks=%d  %.1f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
  }
  size_t bytes = (size_t)8 << 30; int4* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  int* o2; cudaMalloc(&o2, 4);
  for (int bpsm = 2; bpsm <= 8; bpsm *= 2) {
    int blocks = pr.multiProcessorCount * bpsm;
    stream_read<<<blocks, 512>>>(buf, bytes / 16, o2);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) stream_read<<<blocks, 512>>>(buf, bytes / 16, o2);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("stream read 8 GiB, %d blocks x 512: %.1f GB/s\n", blocks, 5.0 * bytes / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Microbenchmark: how fast can listed KV rows (SnapKV / PQ index lists) be gathered from HBM into
// shared memory, by copy mechanism and by index locality?  K and V caches of 256-byte rows
// (head_dim 128, bf16); 2048 listed rows per (b, kv head) unit, 512 units (B = 64 x 8 KV heads):
// 537 MB per pass.  A persistent grid (296 CTAs, 2 / SM) takes contiguous equal shares of the
// 64-row tiles; per tile 64 K rows + 64 V rows land in a 3-stage ring (32 KB stages).
//   M1 per-lane cp.async: lane l copies rows 2l, 2l+1 (16 x 16 B each): a warp instruction
//      touches 32 different rows (the current kernel's mapping)
//   M2 row-coalesced cp.async: one instruction copies 2 whole rows (lanes 0-15: row 2i,
//      16-31: row 2i+1), 32 instructions per tile and buffer
//   M3 one cp.async.bulk (TMA engine, 1-D) of 256 B per row, issued by the 32 lanes
//   M4 reference: 2-D tensor-map boxes of 64 rows (valid only for contiguous lists)
// Index patterns: contiguous (each unit's list is one run), runs of 8, uniform random (sorted).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_sol gather_sol.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_expect_noarrive(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
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
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}

constexpr int TK = 64, ROW = 256, TILE = TK * ROW, STAGE = 2 * TILE, NSTAGE = 3;

struct Maps {
  CUtensorMap k, v;
};

// rows: [tiles * 64] global row indices (row * 256 bytes)
__global__ void __launch_bounds__(64) gather_kernel(const __grid_constant__ Maps mp, const uint8_t* kb, const uint8_t* vb,
                                                    const int* rows, int tiles, int mech, int* sink) {
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
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) {  // producer warp
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int it = 0;
    for (int t = a; t < e; ++t, ++it) {
      const int s = it % NSTAGE;
      const uint32_t kt = smem_u32(sm + s * STAGE), vt = kt + TILE;
      const int r0 = __ldg(rows + t * TK + 2 * lane), r1 = __ldg(rows + t * TK + 2 * lane + 1);
      if (lane == 0) mbar_wait(&empty[s], ((it / NSTAGE) & 1) ^ 1);
      __syncwarp();
      if (mech == 0) {
        for (int u = 0; u < 2; ++u) {
          const int r = u ? r1 : r0, tr = 2 * lane + u;
          for (int c = 0; c < 16; ++c) {
            cp16(kt + tr * ROW + c * 16, kb + (size_t)r * ROW + c * 16, pol);
            cp16(vt + tr * ROW + c * 16, vb + (size_t)r * ROW + c * 16, pol);
          }
        }
        cp_arrive(&full[s]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      } else if (mech == 1) {
        const int half = lane >> 4, c = lane & 15;
        for (int i = 0; i < 32; ++i) {
          const int tr = 2 * i + half;
          const int ra = __shfl_sync(0xffffffffu, r0, i), rb = __shfl_sync(0xffffffffu, r1, i);  // tile rows 2i, 2i+1
          const int row = half ? rb : ra;
          cp16(kt + tr * ROW + c * 16, kb + (size_t)row * ROW + c * 16, pol);
          cp16(vt + tr * ROW + c * 16, vb + (size_t)row * ROW + c * 16, pol);
        }
        cp_arrive(&full[s]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      } else if (mech == 2) {
        if (lane == 0) mbar_expect(&full[s], STAGE);
        __syncwarp();
        for (int u = 0; u < 2; ++u) {
          const int r = u ? r1 : r0, tr = 2 * lane + u;
          bulk_g2s(kt + tr * ROW, kb + (size_t)r * ROW, ROW, &full[s], pol);
          bulk_g2s(vt + tr * ROW, vb + (size_t)r * ROW, ROW, &full[s], pol);
        }
      } else {
        if (lane == 0) {
          const int r = __ldg(rows + t * TK);
          mbar_expect(&full[s], STAGE);
          for (int sub = 0; sub < 2; ++sub) {
            tma2(kt + sub * 8192, &mp.k, &full[s], sub * 64, r, pol);
            tma2(vt + sub * 8192, &mp.v, &full[s], sub * 64, r, pol);
          }
        }
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

int main() {
  const size_t cap = 32768 + 64, units = 512, rows_total = units * cap;  // [B*Hkv][cap] rows: 4.3 GB per buffer
  const int K = 2048;
  uint8_t *kb, *vb;
  if (cudaMalloc(&kb, rows_total * ROW) != cudaSuccess || cudaMalloc(&vb, rows_total * ROW) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(kb, 1, rows_total * ROW);
  cudaMemset(vb, 1, rows_total * ROW);
  Maps mp;
  {
    cuuint64_t dims[2] = {128, rows_total};
    cuuint64_t str[1] = {ROW};
    cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    enc()(&mp.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kb, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc()(&mp.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, vb, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  int* sink;
  cudaMalloc(&sink, 4);
  int* d_rows;
  cudaMalloc(&d_rows, units * K * sizeof(int));
  const int smem = NSTAGE * STAGE + 1024 + 64;
  cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::mt19937 rng(1);
  const char* pats[3] = {"contiguous", "runs8", "random"};
  const char* mechs[4] = {"M1_lane_cp_async", "M2_row_coalesced_cp_async", "M3_bulk_per_row", "M4_tma_box64"};
  const int tiles = units * K / TK;
  for (int pat = 0; pat < 3; ++pat) {
    std::vector<int> rows(units * K);
    for (size_t u = 0; u < units; ++u) {
      std::vector<int> sel;
      if (pat == 0) {
        for (int i = 0; i < K; ++i) sel.push_back(1000 + i);
      } else if (pat == 1) {
        std::vector<int> st((cap - 64) / 8);
        for (size_t i = 0; i < st.size(); ++i) st[i] = (int)i * 8;
        std::shuffle(st.begin(), st.end(), rng);
        st.resize(K / 8);
        std::sort(st.begin(), st.end());
        for (int s0 : st)
          for (int i = 0; i < 8; ++i) sel.push_back(s0 + i);
      } else {
        std::vector<int> all(cap - 64);
        for (size_t i = 0; i < all.size(); ++i) all[i] = (int)i;
        std::shuffle(all.begin(), all.end(), rng);
        all.resize(K);
        std::sort(all.begin(), all.end());
        sel = all;
      }
      for (int i = 0; i < K; ++i) rows[u * K + i] = (int)(u * cap) + sel[i];
    }
    cudaMemcpy(d_rows, rows.data(), rows.size() * sizeof(int), cudaMemcpyHostToDevice);
    for (int mech = 0; mech < 4; ++mech) {
      if (mech == 3 && pat != 0) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(296);
      cfg.blockDim = dim3(64);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      for (int i = 0; i < 4; ++i) cudaLaunchKernelEx(&cfg, gather_kernel, mp, (const uint8_t*)kb, (const uint8_t*)vb, (const int*)d_rows, tiles, mech, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      const int reps = 20;
      cudaEventRecord(a);
      for (int i = 0; i < reps; ++i)
        cudaLaunchKernelEx(&cfg, gather_kernel, mp, (const uint8_t*)kb, (const uint8_t*)vb, (const int*)d_rows, tiles, mech, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double us = ms * 1e3 / reps, bytes = (double)tiles * STAGE;
      printf("{\"pattern\": \"%s\", \"mech\": \"%s\", \"us\": %.1f, \"GBps\": %.0f}\n", pats[pat], mechs[mech], us,
             bytes / us / 1e3);
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

// md_internal.h — host-side helpers shared by the ABI translation units
// (error string, argument checks, launch-error mapping).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/magicdec_b200.h"

namespace md {

void set_error(const char* fmt, ...);
void clear_error();

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline md_status fail(md_status s, const char* msg) {
  set_error("%s", msg);
  return s;
}

inline md_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return MD_ERR_CUDA;
  }
  return MD_OK;
}

int device_sm_count();

md_status launch_kv_append(const md_kv_cache* c, const void* k_new, const void* v_new, int T, const int32_t* start,
                           int start_off, cudaStream_t stream);

}  // namespace md

#define MD_REQUIRE(cond, code, ...)  \
  do {                               \
    if (!(cond)) {                   \
      ::md::set_error(__VA_ARGS__);  \
      return (code);                 \
    }                                \
  } while (0)

namespace md {
// Launch with the programmatic-stream-serialization attribute (PDL): the kernel may start
// while its predecessor drains; every md kernel calls griddepcontrol.wait before reading
// anything a predecessor may have written.  (Compile with -DMD_NO_PDL=1 for plain launches.)
#ifndef MD_NO_PDL
#define MD_NO_PDL 0
#endif

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = MD_NO_PDL ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace md

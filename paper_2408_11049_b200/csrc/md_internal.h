// md_internal.h — host-side helpers shared by the ABI translation units
// (error string, argument checks, launch-error mapping).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

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

}  // namespace md

#define MD_REQUIRE(cond, code, ...)  \
  do {                               \
    if (!(cond)) {                   \
      ::md::set_error(__VA_ARGS__);  \
      return (code);                 \
    }                                \
  } while (0)

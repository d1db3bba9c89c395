// tp.cu — md_tp_barrier: the completion half of the fused tensor-parallel output exchange
// (the paper's 8-way TP).  With md_*_tp calls every rank
// stores its heads' outputs straight into every rank's full-head buffer over NVLink; a rank
// may read its buffer once every peer has passed the barrier that follows its attention call.
//
// One 32-thread CTA per call: lane 0 bumps this rank's device-side epoch e (so the barrier
// needs no host value and is CUDA-graph capturable), a system-scope fence orders the previous
// kernels' peer stores, lane k < world writes e into flags[k][rank] with a system-scope
// release, then lane j < world spins (acquire, with back-off) until flags[rank][j] >= e.  The
// spin is bounded (~20 s): a peer that never arrives traps this kernel instead of hanging it.
// The kernel lets its stream's next kernel launch only after the wait (PDL trigger at the end),
// so nothing queued behind it occupies SMs while it spins.
#include <cstdint>

#include "md_common.cuh"
#include "md_internal.h"

namespace md {

__global__ void tp_barrier_kernel(uint64_t* const* flags_peers, uint64_t* epoch, int world, int rank) {
  // no early trigger: the next kernel must not pre-launch (and hold SMs) while this one spins
  pdl_wait();  // the attention kernel whose peer stores this barrier publishes
  __shared__ uint64_t e_sh;
  const int lane = threadIdx.x;
  if (lane == 0) {
    e_sh = *epoch + 1;
    *epoch = e_sh;
  }
  __syncwarp();
  const uint64_t e = e_sh;
  __threadfence_system();
  __syncwarp();
  if (lane < world) {
    uint64_t* dst = flags_peers[lane] + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(e) : "memory");
  }
  if (lane < world) {
    const uint64_t* src = flags_peers[rank] + lane;
    uint64_t v = 0;
    long long spins = 0;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(src) : "memory");
      if (v >= e) break;
      __nanosleep(200);
      if (++spins > 100000000LL) {
        printf("md_tp_barrier: rank %d timed out waiting for rank %d (epoch %llu)\n", rank, lane,
               (unsigned long long)e);
        __trap();
      }
    }
  }
  __syncwarp();
  pdl_trigger();
}

}  // namespace md

extern "C" md_status md_tp_barrier(const md_tp_sync* s, md_stream_t stream) {
  using namespace md;
  clear_error();
  MD_REQUIRE(s != nullptr && s->flags_peers != nullptr && s->epoch != nullptr, MD_ERR_INVALID_ARG,
             "md_tp_barrier: NULL argument");
  MD_REQUIRE(s->world >= 1 && s->world <= 32 && s->rank >= 0 && s->rank < s->world, MD_ERR_INVALID_ARG,
             "md_tp_barrier: need 0 <= rank < world <= 32");
  launch_pdl(tp_barrier_kernel, dim3(1), dim3(32), 0, (cudaStream_t)stream, s->flags_peers, s->epoch, (int)s->world,
             (int)s->rank);
  return check_launch("md_tp_barrier");
}

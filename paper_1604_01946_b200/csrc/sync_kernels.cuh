// sync_kernels.cuh -- the small host-launched synchronisation kernels around the cluster
// schedule (pass epochs, the layer pipeline's system-scope ready flag). Included by runtime.cu
// only: the kernel translation units (kernels_*.cu) must not define non-template kernels.
#pragma once

#include "rec_cluster.cuh"

namespace rw {

__global__ void k_epoch_inc(uint32_t* e, unsigned* clear = nullptr) {
  *e += 1;
  if (clear) *clear = 0u;
}
// Layer pipeline: tell the next stage (system scope, its memory) that this forward's layer-input
// copy landed; the next stage waits for its own forward epoch before its weight-gradient GEMMs.
__global__ void k_pp_signal(uint32_t* peer_ready, const uint32_t* my_epoch) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer_ready), "r"(*my_epoch) : "memory");
}
__global__ void k_pp_wait(const uint32_t* ready, const uint32_t* my_epoch, int* error, unsigned long long timeout_ns) {
  const uint32_t e = *my_epoch;
  const uint64_t t0 = globaltimer();
  uint32_t v;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ready) : "memory");
    if (globaltimer() - t0 > timeout_ns) {
      atomicCAS(error, 0, (1 << 30) | (4 << 26));
      return;
    }
  } while (!flag_reached(v, e));
}

// Device timestamp (%globaltimer ns) of a point in stream order: brackets launches that carry no
// stamps of their own (the dx0 GEMM, the backward trace's INPUT_GEMM of layer 0).
__global__ void k_stamp(unsigned long long* p) { *p = globaltimer(); }

}  // namespace rw

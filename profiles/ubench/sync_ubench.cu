// sync_ubench.cu -- microbenchmarks for the per-step exchange of a persistent recurrent kernel:
// how long does one "all-gather h_t among the CTAs of a layer, then start step t+1" tick cost
// on B200, via (A) global memory + gpu-scope flags + bulk loads, (B) DSMEM pushes with
// st.shared::cluster + remote mbarrier arrives, (C) DSMEM bulk copies (cp.async.bulk
// shared::cta -> shared::cluster, complete_tx on the peer's mbarrier).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 sync_ubench.cu -o sync_ubench
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) { while (!mbar_try(b, ph)) {} }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void cluster_sync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) { uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) { uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_release(uint32_t* p, uint32_t v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

constexpr int kThreads = 256;

// (A) global: group of G CTAs; each tick every CTA writes `slice` bytes, publishes, waits for
// the group's counter, then bulk-loads all G slices (G*slice bytes) into smem.
__global__ void __launch_bounds__(kThreads, 1) k_global(uint8_t* buf, uint32_t* flags, int G, int slice, int iters,
                                                        unsigned long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  const int grp = blockIdx.x / G, me = blockIdx.x % G;
  const int total = G * slice;
  uint8_t* gbuf = buf + (size_t)grp * 2 * total;
  uint32_t* gfl = flags + (size_t)grp * iters;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  uint64_t t0 = gtime();
  for (int it = 0; it < iters; ++it) {
    uint8_t* dst = gbuf + (it & 1) * total + me * slice;
    // write slice (16 B per thread per pass)
    for (int o = threadIdx.x * 16; o < slice; o += kThreads * 16) {
      int4 v = make_int4(it, me, o, 0);
      *reinterpret_cast<int4*>(dst + o) = v;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      red_release(&gfl[it], 1);
      while (ld_relaxed(&gfl[it]) < (uint32_t)G) {}
      (void)ld_acquire(&gfl[it]);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (mode == 0) {
        mbar_expect(&bar, total);
        const uint8_t* src = gbuf + (it & 1) * total;
        for (int o = 0; o < total; o += 8192) {
          int n = min(8192, total - o);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(sm + o)), "l"(src + o), "r"(n), "r"(su32(&bar)) : "memory");
        }
        mbar_wait(&bar, it & 1);
      }
    }
    __syncthreads();
  }
  uint64_t t1 = gtime();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// (B)/(C) DSMEM within one cluster of G CTAs: double-buffered receive area [2][G*slice].
// mode 1: st.shared::cluster.v4 by all threads + one remote arrive (release) per peer.
// mode 2: cp.async.bulk shared::cta -> shared::cluster per peer, complete_tx on the peer bar.
__global__ void __launch_bounds__(kThreads, 1) k_dsmem(int slice, int iters, unsigned long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[2];
  const int G = (int)(gridDim.x < 16 ? gridDim.x : 16);  // cluster dims = G (launch sets it)
  uint32_t cs;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  const int me = ctarank();
  const int total = cs * slice;
  uint8_t* rx = sm;                   // [2][total]
  uint8_t* tx0 = sm + 2 * total;      // own slice staging [2][slice] (double-buffered: my
                                      // copies of tick t are complete once tick t+1 completes)
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], mode == 1 ? cs : 1);
    mbar_init(&bar[1], mode == 1 ? cs : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_sync();
  (void)G;
  uint64_t t0 = gtime();
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    const uint32_t ph = (it >> 1) & 1;
    if (mode == 1) {
      for (int o = threadIdx.x * 16; o < slice; o += kThreads * 16) {
        for (uint32_t r = 0; r < cs; ++r) {
          uint32_t a = mapa(su32(rx + b * total + me * slice + o), r);
          asm volatile("st.shared::cluster.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(it), "r"(me), "r"(o), "r"(0) : "memory");
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        for (uint32_t r = 0; r < cs; ++r)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(su32(&bar[b]), r)) : "memory");
      }
      mbar_wait(&bar[b], ph);
    } else {
      uint8_t* tx = tx0 + b * slice;
      for (int o = threadIdx.x * 16; o < slice; o += kThreads * 16)
        *reinterpret_cast<int4*>(tx + o) = make_int4(it, me, o, 0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        mbar_expect(&bar[b], total);
        for (uint32_t r = 0; r < cs; ++r) {
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(mapa(su32(rx + b * total + me * slice), r)), "r"(su32(tx)), "r"(slice),
                       "r"(mapa(su32(&bar[b]), r)) : "memory");
        }
      }
      mbar_wait(&bar[b], ph);
    }
  }
  uint64_t t1 = gtime();
  cluster_sync();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// (E) hybrid: data through L2 (st.global slice, then bulk loads of all slices; mode 3 unicast
// per CTA, mode 4 multicast: CTA r loads slice r into every CTA of the cluster), sync through
// DSMEM (cluster-scope release + remote mbarrier arrive on every peer).
__global__ void __launch_bounds__(kThreads, 1) k_hybrid(uint8_t* buf, int slice, int iters, unsigned long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t sbar[2], dbar[2];
  uint32_t cs;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  const int me = ctarank();
  const int total = cs * slice;
  const int grp = blockIdx.x / cs;
  uint8_t* gbuf = buf + (size_t)grp * 2 * total;
  if (threadIdx.x == 0) {
    mbar_init(&sbar[0], cs); mbar_init(&sbar[1], cs);
    mbar_init(&dbar[0], 1); mbar_init(&dbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_sync();
  uint64_t t0 = gtime();
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    const uint32_t ph = (it >> 1) & 1;
    uint8_t* dst = gbuf + b * total + me * slice;
    for (int o = threadIdx.x * 16; o < slice; o += kThreads * 16)
      *reinterpret_cast<int4*>(dst + o) = make_int4(it, me, o, 0);
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      for (uint32_t r = 0; r < cs; ++r)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(su32(&sbar[b]), r)) : "memory");
      mbar_expect(&dbar[b], total);
      mbar_wait(&sbar[b], ph);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const uint8_t* src = gbuf + b * total;
      if (mode == 3) {
        for (int o = 0; o < total; o += 8192)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(sm + b * total + o)), "l"(src + o), "r"(min(8192, total - o)), "r"(su32(&dbar[b])) : "memory");
      } else {
        const uint16_t mask = (uint16_t)((1u << cs) - 1);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                     ::"r"(su32(sm + b * total + me * slice)), "l"(src + me * slice), "r"(slice), "r"(su32(&dbar[b])), "h"(mask) : "memory");
      }
      mbar_wait(&dbar[b], ph);
    }
    __syncthreads();
  }
  uint64_t t1 = gtime();
  cluster_sync();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// (D) ping-pong between CTA 0 and CTA 1 through global flags: one-way latency.
__global__ void k_pingpong(uint32_t* f, int iters, unsigned long long* out) {
  if (threadIdx.x) return;
  uint64_t t0 = gtime();
  for (int i = 0; i < iters; ++i) {
    if (blockIdx.x == 0) {
      red_release(&f[0], 1);
      while (ld_relaxed(&f[1]) < (uint32_t)(i + 1)) {}
    } else {
      while (ld_relaxed(&f[0]) < (uint32_t)(i + 1)) {}
      red_release(&f[1], 1);
    }
  }
  out[blockIdx.x] = gtime() - t0;
}

static double median_us(std::vector<unsigned long long>& v, int iters) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2] / 1e3 / iters;
}

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, dev));
  printf("%s SMs=%d\n", pr.name, pr.multiProcessorCount);
  const int iters = 2000;
  unsigned long long* d_out;
  CK(cudaMalloc(&d_out, 4096 * 8));
  uint32_t* flags;
  CK(cudaMalloc(&flags, 64ull * iters * 4));
  uint8_t* buf;
  CK(cudaMalloc(&buf, 64ull << 20));
  std::vector<unsigned long long> h(4096);

  {  // ping-pong
    CK(cudaMemset(flags, 0, 64));
    k_pingpong<<<2, 32>>>(flags, iters, d_out);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), d_out, 16, cudaMemcpyDeviceToHost));
    printf("pingpong round trip: %.3f us\n", h[0] / 1e3 / iters);
  }
  const size_t big_smem = 200 * 1024;  // force 1 CTA / SM
  CK(cudaFuncSetAttribute(k_global, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem));
  for (int mode = 0; mode < 2; ++mode)
    for (int G : {16, 32, 64})
      for (int groups : {1, 4, 8})
        for (int slice : {2048, 4096}) {
          if (G * groups > 148 || G * slice > 190 * 1024) continue;
          CK(cudaMemset(flags, 0, 64ull * iters * 4));
          k_global<<<G * groups, kThreads, big_smem>>>(buf, flags, G, slice, iters, d_out, mode);
          CK(cudaDeviceSynchronize());
          int n = G * groups;
          CK(cudaMemcpy(h.data(), d_out, n * 8, cudaMemcpyDeviceToHost));
          std::vector<unsigned long long> v(h.begin(), h.begin() + n);
          printf("global%s G=%d groups=%d slice=%d: tick %.3f us\n", mode ? "-flagonly" : "+bulkload", G,
                 groups, slice, median_us(v, iters));
        }
  CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem));
  CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs : {8, 16})
    for (int groups : {1, 4, 8})
      for (int slice : {2048, 4096})
        for (int mode : {1, 2}) {
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3(cs * groups);
          lc.blockDim = dim3(kThreads);
          lc.dynamicSmemBytes = big_smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cs;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          lc.attrs = at;
          lc.numAttrs = 1;
          int ncl = 0;
          cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, (void*)k_dsmem, &lc);
          if (oe != cudaSuccess || ncl < groups) {
            printf("dsmem cs=%d groups=%d: only %d clusters co-resident (%s)\n", cs, groups, ncl,
                   cudaGetErrorString(oe));
            cudaGetLastError();
            continue;
          }
          cudaError_t e = cudaLaunchKernelEx(&lc, k_dsmem, slice, iters, d_out, mode);
          if (e != cudaSuccess) { printf("launch failed %s\n", cudaGetErrorString(e)); cudaGetLastError(); continue; }
          CK(cudaDeviceSynchronize());
          int n = cs * groups;
          CK(cudaMemcpy(h.data(), d_out, n * 8, cudaMemcpyDeviceToHost));
          std::vector<unsigned long long> v(h.begin(), h.begin() + n);
          printf("dsmem-%s cs=%d groups=%d (max %d) slice=%d: tick %.3f us\n", mode == 1 ? "st" : "bulk",
                 cs, groups, ncl, slice, median_us(v, iters));
        }
  CK(cudaFuncSetAttribute(k_hybrid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem));
  CK(cudaFuncSetAttribute(k_hybrid, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs : {8, 16})
    for (int groups : {1, 4})
      for (int slice : {2048, 4096})
        for (int mode : {3, 4}) {
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3(cs * groups);
          lc.blockDim = dim3(kThreads);
          lc.dynamicSmemBytes = big_smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cs;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          lc.attrs = at;
          lc.numAttrs = 1;
          cudaError_t e = cudaLaunchKernelEx(&lc, k_hybrid, buf, slice, iters, d_out, mode);
          if (e != cudaSuccess) { printf("launch failed %s\n", cudaGetErrorString(e)); cudaGetLastError(); continue; }
          CK(cudaDeviceSynchronize());
          int n = cs * groups;
          CK(cudaMemcpy(h.data(), d_out, n * 8, cudaMemcpyDeviceToHost));
          std::vector<unsigned long long> v(h.begin(), h.begin() + n);
          printf("hybrid-%s cs=%d groups=%d slice=%d (gather %d KB): tick %.3f us\n", mode == 3 ? "unicast" : "multicast",
                 cs, groups, slice, cs * slice / 1024, median_us(v, iters));
        }
  return 0;
}

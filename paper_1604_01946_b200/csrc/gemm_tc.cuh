// gemm_tc.cuh -- warp-specialised tcgen05 GEMM for sm_100a (K1/K5/K6 of SURVEY §2.2):
//   D[M x N] (fp32) = A[M x K] * B[N x K]^T
// A and B are read from HBM/L2 by TMA into SWIZZLE_128B shared-memory stages (either
// operand K-major or MN-major), multiplied by tcgen05.mma with the accumulator in TMEM,
// and written by a 4-warp epilogue (tcgen05.ld -> registers -> coalesced global stores)
// that can un-permute gate-interleaved rows and strip batch padding on the fly.
//
// Roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator,
// warp 3 idle, warps 4..7 epilogue (warp w reads TMEM lane quarter w%4).
// blockIdx.z indexes a table of GemmDesc so several independent GEMMs (e.g. dW and dR of
// every layer) run as one grouped launch.
#pragma once

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace rw {

template <class P, bool kMN>
struct OperandTile {
  // Issue the TMA loads of one k-block of an operand tile (rows x kAtomK elements) into
  // `dst` (rows * 128 bytes). K-major: boxes {kAtomK, min(rows, 128)} at (k, row0 + r) (GEMM
  // operand maps are encoded with at most 128 box rows, see gemm_box_rows in runtime.cu).
  // MN-major: rows / kAtomK boxes {kAtomK (along MN), kAtomK (K rows)} stacked at
  // kAtomK * 128-byte strides (the UMMA LBO).
  static __device__ __forceinline__ void load(void* dst, const CUtensorMap* m, uint64_t* bar,
                                              int row0, int rows, int k0) {
    if constexpr (!kMN) {
      for (int r = 0; r < rows; r += 128)
        tma_load_2d(static_cast<uint8_t*>(dst) + r * kRowBytes, m, bar, k0, row0 + r);
    } else {
      for (int c = 0; c < rows / P::kAtomK; ++c)
        tma_load_2d(static_cast<uint8_t*>(dst) + c * P::kAtomK * kRowBytes, m, bar,
                    row0 + c * P::kAtomK, k0);
    }
  }
  // UMMA descriptor of k-substep kk (0 .. kAtomK/kUmmaK-1) of a tile at smem address s.
  static __device__ __forceinline__ uint64_t desc(uint32_t s, int kk) {
    return desc_add(base(s), kk * kk_bytes());
  }
  // Descriptor of the tile at smem address s (k-substep 0) and the byte stride of a k-substep.
  static __device__ __forceinline__ uint64_t base(uint32_t s) {
    if constexpr (!kMN) {
      return sdesc_sw128(s, 16, 1024);
    } else {
      return sdesc_sw128(s, P::kAtomK * kRowBytes, 1024);
    }
  }
  static __device__ __forceinline__ constexpr uint32_t kk_bytes() {
    return kMN ? P::kUmmaK * kRowBytes : P::kUmmaK * P::kElem;
  }
};

__device__ __forceinline__ int gemm_out_row(const GemmDesc& g, int m) {
  if (g.row_mode == kRowGateUnperm) {  // gate slots g >= gates (GRU, RNN) hold no output row
    const int u = rho_unit(m), gt = rho_gate(m);
    return u < g.H && (g.gates == 0 || gt < g.gates) ? gt * g.H + u : -1;
  }
  if (g.row_mode == kRowGatePad) return rho_gate(m) * g.Hp + rho_unit(m);
  if (g.row_mode == kRowGateRepad) return m < g.m_valid ? (m / g.H) * g.Hp + m % g.H : -1;
  return m < g.m_valid ? m : -1;
}
__device__ __forceinline__ long long gemm_out_col(const GemmDesc& g, int n) {
  if (g.col_mode == kColBatchUnpad) {
    const int t = n / g.Bp, b = n - t * g.Bp;
    return b < g.B ? (long long)t * g.B + b : -1;
  }
  return n < g.n_valid ? n : -1;
}

// kChunkBN > 0 enables "promotion" for the fp32-parity mode: the K loop is cut into chunks of
// `chunk_kb` k-blocks, each accumulated into one of two TMEM buffers, and the epilogue drains
// every chunk into fp32 registers (round-to-nearest adds). The tensor core's accumulation
// of long K chains loses ~K*2^-24 (measured 5e-5 at K = 6400); chunking bounds that to the
// chunk length while the next chunk's MMAs run into the other buffer.
// Output column iterator (no per-element division): yields the destination column of
// n0, n0+1, ... or -1 for padding columns.
struct ColCursor {
  int unpad, Bp, B, n_valid, b;
  long long t_base, n;
  __device__ __forceinline__ ColCursor(const GemmDesc& g, int n0)
      : unpad(g.col_mode == kColBatchUnpad), Bp(g.Bp), B(g.B), n_valid(g.n_valid), n(n0) {
    const int t = unpad ? n0 / g.Bp : 0;
    b = unpad ? n0 - t * g.Bp : 0;
    t_base = (long long)t * g.B;
  }
  __device__ __forceinline__ long long next() {
    long long r;
    if (unpad) {
      r = b < B ? t_base + b : -1;
      if (++b == Bp) {
        b = 0;
        t_base += B;
      }
    } else {
      r = n < n_valid ? n : -1;
      ++n;
    }
    return r;
  }
};

template <class P, bool kAMN, bool kBMN, int kChunkBN>
__global__ void __launch_bounds__(256, 1)
    k_gemm_tc(const GemmDesc* __restrict__ table, int bn, int stages, int chunk_kb) {
  // descriptor in shared memory: the epilogue reads it per element
  __shared__ GemmDesc g;
  if (threadIdx.x == 0) {
    g = table[blockIdx.z];
    set_wait_error(g.error);
  }
  __syncthreads();
  const int m0 = blockIdx.x * kTileM;
  const int n0 = blockIdx.y * bn;
  if (m0 >= g.M || n0 >= g.N) return;
  const int nkb = (g.K + P::kAtomK - 1) / P::kAtomK;  // OOB K is zero-filled by TMA
  const int ckb = (kChunkBN > 0 && chunk_kb > 0) ? chunk_kb : nkb;
  const int nchunks = (nkb + ckb - 1) / ckb;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int a_bytes = kTileM * kRowBytes;
  const int b_bytes = bn * kRowBytes;
  const int stage_bytes = P::kPlanes * (a_bytes + b_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;   // [2]
  uint64_t* tmem_empty = tmem_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nbuf = kChunkBN > 0 ? 2 : 1;
  uint32_t tmem_cols = 32;
  while (tmem_cols < (uint32_t)(P::kPlanes * bn * nbuf)) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < P::kPlanes; ++p) {
      prefetch_tmap(g.a[p]);
      prefetch_tmap(g.b[p]);
    }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % stages;
      mbar_wait_bounded(&empty[s], ((kb / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      uint8_t* st = smem + s * stage_bytes;
      const int k = kb * P::kAtomK;
      for (int p = 0; p < P::kPlanes; ++p) {
        OperandTile<P, kAMN>::load(st + p * a_bytes, g.a[p], &full[s], m0 + g.a_m_off, kTileM, k + g.a_k_off);
        OperandTile<P, kBMN>::load(st + P::kPlanes * a_bytes + p * b_bytes, g.b[p], &full[s], n0 + g.b_n_off,
                                   bn, k + g.b_k_off);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp converged; elect.sync picks the issuing lane)
    // Two-plane formats: the stage holds B_hi and B_lo as adjacent row runs (K-major rows, or
    // MN-major 64-element chunks, at the same uniform stride), so (hi,hi) and (hi,lo) are ONE
    // MMA over N = 2 bn into the buffer's two column halves, and (lo,hi) a second one of N = bn
    // into the first half: 2 issues per K step instead of 3 (a warp issues one tcgen05.mma per
    // ~84 cycles at N <= 128, profiles/r01/ubench_mma_ingress.txt), the epilogue sums the halves.
    const uint32_t idesc = idesc_make(P::kFmt, kAMN, kBMN, kTileM, bn);
    const uint32_t idesc2 = idesc_make(P::kFmt, kAMN, kBMN, kTileM, P::kPlanes == 2 ? 2 * bn : bn);
    const int bw = P::kPlanes * bn;  // accumulator columns per buffer
    // stage-0 descriptors, advanced by adds (sm100_ptx.cuh desc_add)
    const uint64_t a_d0 = OperandTile<P, kAMN>::base(smem_u32(smem));
    const uint64_t b_d0 = OperandTile<P, kBMN>::base(smem_u32(smem + P::kPlanes * a_bytes));
    int kb = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      if (c >= 2) {
        mbar_wait_bounded(&tmem_empty[buf], ((c >> 1) - 1) & 1);
        tc_fence_after();
      }
      const uint32_t acc = tmem_base + buf * bw;
      const int kb_end = min(nkb, (c + 1) * ckb);
      for (int k0 = kb; kb < kb_end; ++kb) {
        const int s = kb % stages;
        mbar_wait_bounded(&full[s], (kb / stages) & 1);
        tc_fence_after();
        const uint64_t a_s = desc_add(a_d0, s * stage_bytes), b_s = desc_add(b_d0, s * stage_bytes);
#pragma unroll
        for (int kk = 0; kk < P::kAtomK / P::kUmmaK; ++kk) {
          const uint64_t ad = desc_add(a_s, kk * OperandTile<P, kAMN>::kk_bytes());
          const uint64_t bd = desc_add(b_s, kk * OperandTile<P, kBMN>::kk_bytes());
          umma_warp<P::kTF32>(acc, ad, bd, idesc2, (kb != k0 || kk) ? 1u : 0u);
          if constexpr (P::kPlanes == 2) umma_warp<P::kTF32>(acc, desc_add(ad, a_bytes), bd, idesc, 1u);
        }
        umma_commit_warp(&empty[s]);
      }
      umma_commit_warp(&tmem_full[buf]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global
    const int q = warp & 3;
    const int m = m0 + q * 32 + lane;
    const int orow = m < g.M ? gemm_out_row(g, m) : -1;
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    if constexpr (kChunkBN > 0) {
      float accum[kChunkBN];
#pragma unroll
      for (int i = 0; i < kChunkBN; ++i) accum[i] = 0.0f;
      for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        mbar_wait_bounded(&tmem_full[buf], (c >> 1) & 1);
        tc_fence_after();
        const uint32_t ab = tmem_base + lane_off + buf * P::kPlanes * kChunkBN;
#pragma unroll
        for (int c0 = 0; c0 < kChunkBN; c0 += 8) {
          uint32_t v[8], w[8];
          tmem_ld_32x32b_x8(ab + c0, v);
          if constexpr (P::kPlanes == 2) tmem_ld_32x32b_x8(ab + kChunkBN + c0, w);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            accum[c0 + j] += P::kPlanes == 2 ? __uint_as_float(v[j]) + __uint_as_float(w[j]) : __uint_as_float(v[j]);
        }
        tc_fence_before();
        mbar_arrive(&tmem_empty[buf]);
      }
      if (orow >= 0) {
        ColCursor cc(g, n0);
        float* const drow = g.d + orow;
        const long long ldd = g.ldd;
        const bool accum_out = g.accumulate != 0;
        const float alpha = g.alpha != 0.0f ? g.alpha : 1.0f;
#pragma unroll
        for (int j = 0; j < kChunkBN; ++j) {
          if (n0 + j >= g.N) break;
          const long long oc = cc.next();
          if (oc < 0) continue;
          float* dst = drow + oc * ldd;
          const float val = accum[j] * alpha;
          *dst = accum_out ? *dst + val : val;
        }
      }
    } else {
      mbar_wait_bounded(&tmem_full[0], 0);
      tc_fence_after();
      ColCursor cc(g, n0);
      float* const drow = g.d + (orow < 0 ? 0 : orow);
      const long long ldd = g.ldd;
      const bool accum_out = g.accumulate != 0;
      const float alpha = g.alpha != 0.0f ? g.alpha : 1.0f;
      const int nlim = min(bn, g.N - n0);
      for (int c0 = 0; c0 < bn; c0 += 8) {
        uint32_t v[8];
        tmem_ld_32x32b_x8(tmem_base + lane_off + c0, v);
        tmem_ld_wait();
        if (orow < 0) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (c0 + j >= nlim) break;
          const long long oc = cc.next();
          if (oc < 0) continue;
          float* dst = drow + oc * ldd;
          const float val = __uint_as_float(v[j]) * alpha;
          *dst = accum_out ? *dst + val : val;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
  }
}

// ====================================================================== persistent GEMM (bf16)
// k_gemm_p: one CTA per SM loops over the (problem, n-tile, m-tile) space of a grouped GEMM table
// (m fastest, so CTAs running together share B tiles in L2). Tiles are 128 x BN (BN = 128 or
// 256: at N = 256 a tcgen05.mma (128x256x16) takes 128 tensor cycles, more than a warp's ~90
// cycle issue interval, so the tensor pipe -- not the issuer -- paces the loop). Two TMEM
// accumulators (2 x BN columns) let the epilogue drain tile i while the MMAs of tile i+1 run.
// Warps: 0 TMA producer, 1 MMA issuer (converged, elect.sync), 2 TMEM allocator, 3 idle,
// 4..7 epilogue (TMEM lane quarter = warp % 4).
template <bool kAMN, bool kBMN, int BN>
__global__ void __launch_bounds__(256, 1)
    k_gemm_p(const GemmDesc* __restrict__ table, int count, int mt_max, int nt_max, int stages) {
  using P = PrecBF16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int a_bytes = kTileM * kRowBytes;
  constexpr int b_bytes = BN * kRowBytes;
  constexpr int stage_bytes = a_bytes + b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t tmem_cols = 2 * BN;
  const long long ntiles = (long long)count * mt_max * nt_max;

  if (threadIdx.x == 0) {
    set_wait_error(table[0].error);  // every descriptor of a launch carries the same error word
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  auto tile_of = [&](long long t, int& z, int& m0, int& n0) {
    const int per = mt_max * nt_max;
    z = (int)(t / per);
    const int r = (int)(t - (long long)z * per);
    n0 = (r / mt_max) * BN;
    m0 = (r % mt_max) * kTileM;
  };

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    uint32_t pc = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int z, m0, n0;
      tile_of(t, z, m0, n0);
      const GemmDesc& g = table[z];
      if (m0 >= g.M || n0 >= g.N) continue;
      const int nkb = (g.K + P::kAtomK - 1) / P::kAtomK;
      for (int kb = 0; kb < nkb; ++kb, ++pc) {
        const int s = pc % stages;
        mbar_wait_bounded(&empty[s], ((pc / stages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        uint8_t* st = smem + s * stage_bytes;
        const int k = kb * P::kAtomK;
        OperandTile<P, kAMN>::load(st, g.a[0], &full[s], m0, kTileM, k + g.a_k_off);
        OperandTile<P, kBMN>::load(st + a_bytes, g.b[0], &full[s], n0 + g.b_n_off, BN, k + g.b_k_off);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (converged warp)
    const uint32_t idesc = idesc_make(P::kFmt, kAMN, kBMN, kTileM, BN);
    const uint64_t a_d0 = OperandTile<P, kAMN>::base(smem_u32(smem));
    const uint64_t b_d0 = OperandTile<P, kBMN>::base(smem_u32(smem + a_bytes));
    uint32_t pc = 0, tc = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int z, m0, n0;
      tile_of(t, z, m0, n0);
      const GemmDesc& g = table[z];
      if (m0 >= g.M || n0 >= g.N) continue;
      const int nkb = (g.K + P::kAtomK - 1) / P::kAtomK;
      const int buf = tc & 1;
      if (tc >= 2) {
        mbar_wait_bounded(&tmem_empty[buf], ((tc >> 1) - 1) & 1);
        tc_fence_after();
      }
      const uint32_t acc = tmem_base + buf * BN;
      for (int kb = 0; kb < nkb; ++kb, ++pc) {
        const int s = pc % stages;
        mbar_wait_bounded(&full[s], (pc / stages) & 1);
        tc_fence_after();
        const uint64_t a_s = desc_add(a_d0, s * stage_bytes), b_s = desc_add(b_d0, s * stage_bytes);
#pragma unroll
        for (int kk = 0; kk < P::kAtomK / P::kUmmaK; ++kk)
          umma_bf16_warp(acc, desc_add(a_s, kk * OperandTile<P, kAMN>::kk_bytes()),
                         desc_add(b_s, kk * OperandTile<P, kBMN>::kk_bytes()), idesc, (kb | kk) ? 1u : 0u);
        umma_commit_warp(&empty[s]);
      }
      umma_commit_warp(&tmem_full[buf]);
      ++tc;
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global (overlaps the next tile's MMAs)
    const int q = warp & 3;
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    uint32_t tc = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int z, m0, n0;
      tile_of(t, z, m0, n0);
      const GemmDesc& g = table[z];
      if (m0 >= g.M || n0 >= g.N) continue;
      const int buf = tc & 1;
      mbar_wait_bounded(&tmem_full[buf], (tc >> 1) & 1);
      tc_fence_after();
      const int m = m0 + q * 32 + lane;
      const int orow = m < g.M ? gemm_out_row(g, m) : -1;
      ColCursor cc(g, n0);
      float* const drow = g.d + (orow < 0 ? 0 : orow);
      const long long ldd = g.ldd;
      const bool accum_out = g.accumulate != 0;
      const float alpha = g.alpha != 0.0f ? g.alpha : 1.0f;
      const int nlim = min(BN, g.N - n0);
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[8], w[8];
        tmem_ld_32x32b_x8(tmem_base + lane_off + buf * BN + c0, v);
        tmem_ld_32x32b_x8(tmem_base + lane_off + buf * BN + c0 + 8, w);
        tmem_ld_wait();
        if (orow < 0 || c0 >= nlim) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (c0 + j >= nlim) break;
          const long long oc = cc.next();
          if (oc < 0) continue;
          float* dst = drow + oc * ldd;
          const float val = __uint_as_float(j < 8 ? v[j] : w[j - 8]) * alpha;
          *dst = accum_out ? *dst + val : val;
        }
      }
      tc_fence_before();
      mbar_arrive(&tmem_empty[buf]);
      ++tc;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}

// ====================================================================== 2-CTA persistent GEMM (bf16)
// k_gemm_p2: CTA pairs (cluster of 2) run tcgen05.mma.cta_group::2 with M = 256 (each CTA holds
// its 128 rows of A) and N = 256 (each CTA holds half of the B tile): per SM a 64-K k-block
// needs 16 KB of A + 16 KB of B instead of 16 + 32 KB, the difference between the ~60 B/cycle
// an SM ingests from L2 (profiles/ubench/mma_ubench.cu) and what the tensor core consumes at
// N = 256 (94 B/cycle per SM). The leader CTA (rank 0) issues the MMAs; both CTAs' TMA loads
// complete on the leader's full barrier; commits multicast to both CTAs' barriers.

template <bool kAMN, bool kBMN, int BN = 256>
__global__ void __launch_bounds__(256, 1)
    k_gemm_p2(const GemmDesc* __restrict__ table, int count, int mt_max, int nt_max, int stages) {
  using P = PrecBF16;
  constexpr int BH = BN / 2;  // N per pair tile (128 or 256), per CTA half
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int a_bytes = kTileM * kRowBytes;
  constexpr int b_bytes = BH * kRowBytes;
  constexpr int stage_bytes = a_bytes + b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);  // leader only
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2] leader only: one arrive per CTA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank() & 1;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr uint32_t tmem_cols = 2 * BN;
  const long long ntiles = (long long)count * mt_max * nt_max;

  if (threadIdx.x == 0) {
    set_wait_error(table[0].error);  // every descriptor of a launch carries the same error word
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 2);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  auto tile_of = [&](long long t, int& z, int& m0, int& n0) {
    const int per = mt_max * nt_max;
    z = (int)(t / per);
    const int r = (int)(t - (long long)z * per);
    n0 = (r / mt_max) * BN;
    m0 = (r % mt_max) * (2 * kTileM);
  };

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs; completion on the leader's full barrier)
    uint32_t pc = 0;
    for (long long t = pair; t < ntiles; t += npairs) {
      int z, m0, n0;
      tile_of(t, z, m0, n0);
      const GemmDesc& g = table[z];
      if (m0 >= g.M || n0 >= g.N) continue;
      const int nkb = (g.K + P::kAtomK - 1) / P::kAtomK;
      for (int kb = 0; kb < nkb; ++kb, ++pc) {
        const int s = pc % stages;
        mbar_wait_bounded(&empty[s], ((pc / stages) & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * stage_bytes);
        uint8_t* st = smem + s * stage_bytes;
        const int k = kb * P::kAtomK;
        const int am = m0 + (int)rank * kTileM, bn = n0 + g.b_n_off + (int)rank * BH;
        if constexpr (!kAMN) {
          g2::tma_load_2d_pair(st, g.a[0], &full[s], k + g.a_k_off, am);
        } else {
          for (int c = 0; c < kTileM / P::kAtomK; ++c)
            g2::tma_load_2d_pair(st + c * P::kAtomK * kRowBytes, g.a[0], &full[s], am + c * P::kAtomK, k + g.a_k_off);
        }
        if constexpr (!kBMN) {
          g2::tma_load_2d_pair(st + a_bytes, g.b[0], &full[s], k + g.b_k_off, bn);
        } else {
          for (int c = 0; c < BH / P::kAtomK; ++c)
            g2::tma_load_2d_pair(st + a_bytes + c * P::kAtomK * kRowBytes, g.b[0], &full[s], bn + c * P::kAtomK,
                                 k + g.b_k_off);
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ---------------- MMA issuer (leader, converged warp)
    const uint32_t idesc = idesc_make(P::kFmt, kAMN, kBMN, 2 * kTileM, BN);
    const uint64_t a_d0 = OperandTile<P, kAMN>::base(smem_u32(smem));
    const uint64_t b_d0 = OperandTile<P, kBMN>::base(smem_u32(smem + a_bytes));
    uint32_t pc = 0, tc = 0;
    for (long long t = pair; t < ntiles; t += npairs) {
      int z, m0, n0;
      tile_of(t, z, m0, n0);
      const GemmDesc& g = table[z];
      if (m0 >= g.M || n0 >= g.N) continue;
      const int nkb = (g.K + P::kAtomK - 1) / P::kAtomK;
      const int buf = tc & 1;
      if (tc >= 2) {
        mbar_wait_bounded(&tmem_empty[buf], ((tc >> 1) - 1) & 1);
        tc_fence_after();
      }
      const uint32_t acc = tmem_base + buf * BN;
      for (int kb = 0; kb < nkb; ++kb, ++pc) {
        const int s = pc % stages;
        mbar_wait_bounded(&full[s], (pc / stages) & 1);
        tc_fence_after();
        const uint64_t a_s = desc_add(a_d0, s * stage_bytes), b_s = desc_add(b_d0, s * stage_bytes);
#pragma unroll
        for (int kk = 0; kk < P::kAtomK / P::kUmmaK; ++kk)
          g2::umma2_warp(acc, desc_add(a_s, kk * OperandTile<P, kAMN>::kk_bytes()),
                         desc_add(b_s, kk * OperandTile<P, kBMN>::kk_bytes()), idesc, (kb | kk) ? 1u : 0u);
        g2::commit2_warp(&empty[s]);
      }
      g2::commit2_warp(&tmem_full[buf]);
      ++tc;
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs: this CTA's 128 rows of the 256-row tile)
    const int q = warp & 3;
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    uint32_t tc = 0;
    for (long long t = pair; t < ntiles; t += npairs) {
      int z, m0, n0;
      tile_of(t, z, m0, n0);
      const GemmDesc& g = table[z];
      if (m0 >= g.M || n0 >= g.N) continue;
      const int buf = tc & 1;
      mbar_wait_bounded(&tmem_full[buf], (tc >> 1) & 1);
      tc_fence_after();
      const int m = m0 + (int)rank * kTileM + q * 32 + lane;
      const int orow = m < g.M ? gemm_out_row(g, m) : -1;
      ColCursor cc(g, n0);
      float* const drow = g.d + (orow < 0 ? 0 : orow);
      const long long ldd = g.ldd;
      const bool accum_out = g.accumulate != 0;
      const float alpha = g.alpha != 0.0f ? g.alpha : 1.0f;
      const int nlim = min(BN, g.N - n0);
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[8], w[8];
        tmem_ld_32x32b_x8(tmem_base + lane_off + buf * BN + c0, v);
        tmem_ld_32x32b_x8(tmem_base + lane_off + buf * BN + c0 + 8, w);
        tmem_ld_wait();
        if (orow < 0 || c0 >= nlim) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (c0 + j >= nlim) break;
          const long long oc = cc.next();
          if (oc < 0) continue;
          float* dst = drow + oc * ldd;
          const float val = __uint_as_float(j < 8 ? v[j] : w[j - 8]) * alpha;
          *dst = accum_out ? *dst + val : val;
        }
      }
      tc_fence_before();
      named_bar_sync(1, 128);
      if (threadIdx.x == 128)  // one arrive per CTA on the leader's barrier
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(g2::leader_addr(&tmem_empty[buf]))
                     : "memory");
      ++tc;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}

}  // namespace rw

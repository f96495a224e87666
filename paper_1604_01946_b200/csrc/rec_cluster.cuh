// rec_cluster.cuh -- persistent recurrent kernels with split roles per tile ("cluster"
// schedule). bf16 or fp16x2 (fp32-parity) operands, fp32 accumulation and
// cell math.
//
// fp16x2 (common.cuh PrecF16x2): the resident weight slice is split A = A_hi + A_lo; A_hi stays
// in shared memory exactly like the bf16 slice, A_lo lives in TENSOR MEMORY (copied once per
// launch by the epilogue warps) and is the A operand of tcgen05.mma's TMEM-A form. Operand step
// blocks carry both planes per k-block ([hi rows | lo rows], one bulk copy), and every K = 16 step
// issues A_hi.B_hi, A_hi.B_lo, A_lo.B_hi into the same accumulator -- so the fp32-parity slices
// need no more shared memory than bf16 ones and the same CTA count fits the GPU.
//
// Why: in a persistent wavefront the per-step critical path bounds small-H configs (config B:
// 206 dependent steps). Measured on B200 (profiles/ubench/sync_ubench.cu): a gpu-scope flag
// round trip costs ~1.7 us and a 16-CTA flag barrier ~1.4 us, while DSMEM bulk copies
// (cp.async.bulk shared::cta -> shared::cluster, completion by complete_tx on the receiver's
// mbarrier) move a 16-32 KB exchange in ~0.7-1.1 us with no separate handshake. So everything
// that does not depend on the recurrence is taken off the critical path, and the exchange that
// remains inside a tile uses bulk DSMEM copies.
//
// Per tile (forward: 32 units x 4 gates = 128 rho-rows; backward: 128 units) two clusters of
// cs CTAs ("members") split the K range of the step's GEMM, each member keeping its
// 128 x <=512 bf16 weight slice resident in shared memory (loaded once by TMA):
//   * the CRITICAL cluster (kc active members) multiplies the recurrent operand
//       forward : R_l . h_{l,t-1}                 (engine.hpp:368-387)
//       backward: R_l^T . dG_{l,t+1}              (recurrent_backward_gemm, engine.hpp:538-560)
//   * the OFF cluster (ko active members) multiplies the operand from the neighbouring layer
//       forward : W_l . x_{l,t}   (x = h_{l-1,t})  (input_gemm, engine.hpp:347-365)
//       backward: W_{l+1}^T . dG_{l+1,t}          (output_gemm, engine.hpp:564-585)
//     which does not wait for this layer's previous step, so it runs ahead (up to kRing steps).
// Inside a cluster each member drains its TMEM accumulator (128 rows x Bp, fp32) into a
// staging buffer [owner][column][row] and pushes each owner's block with one bulk copy into
// the owner's receive slot; owners sum in fixed member order (deterministic). The off cluster
// writes its reduced partial to a global ring (offsum) and publishes a per-(layer, tile, step)
// counter; the critical producer prefetches it with a bulk copy as soon as it is published.
// Critical owners then form (x-part + h-part) + bias (forward, cells.hpp:240) or
// d_above + carry_h (backward, cells.hpp:424), run the LSTM cell on their columns, publish the
// bf16 operand (h_t / dG_t) with a gpu-scope release counter per (layer, step), and only then
// write the fp32 tapes (h, c, gates, tanh(c) / dG), which nothing in the pass waits for.
// Cell state (c forward; carry_c and the bias-gradient sums backward) stays in registers.
//
// Threads: 384 = warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator, warp 3 idle,
// warps 4..11 epilogue (warp w and w+4 share TMEM lane quarter w%4, split the columns).
#pragma once

#include "lstm_step.cuh"

namespace rw {

constexpr int kClKBlocks = 8;  // k-blocks (64 bf16) per member: 128 x 512 x 2 B = 128 KB resident
constexpr int kClMaxN = 64;    // batch columns (Bp) this path supports
constexpr int kRing = 4;       // off-partial ring depth (steps the off cluster may run ahead)
// MMA issue: a single issuing warp sustains only ~90 cycles per tcgen05.mma regardless of N
// (profiles/ubench/mma_ubench.cu), which at N = Bp = 64 is ~3x the tensor core's own time. Two
// warps (1 and 3) issue the two halves of a step's k-blocks into separate accumulators, and
// the epilogue adds them (acc0 + acc1, fixed order).
constexpr int kIssuers = 2;

// The off-partial ring a critical layer group reads (in this GPU's memory; its writer -- an off
// group -- may run on a peer GPU in the layer pipeline, then `sys` selects system-scope flags).
// Counters are cumulative over passes: a pass's targets are epoch * (per-pass count).
struct ClRing {
  float* ring;         // [tiles][kRing][Bp][128] reduced off partials
  uint32_t* done;      // [tiles][T] publications (ko per step per pass)
  uint32_t* consumed;  // [tiles][32] ring slots copied by the critical members (kc per step per pass)
  int ko;              // off members publishing per step (0: none -- backward top layer, uses dy)
  int sys;
};
// An off-critical group (grid row y, role 1): W . operand for the rows of a target layer, written
// into that layer's ring (possibly on a peer GPU: the layer pipeline's stage boundary).
struct ClOff {
  const CUtensorMap* a;      // weight map of the target layer; the group uses k-blocks [0, kdim/64)
  int kdim;                  // operand K (forward I_l, backward 4Hp)
  const uint8_t* op;         // operand pre-swizzled step blocks (sw_off), kdim x Bp each
  int op_blk_off;            // step block of step t = op_blk_off + t
  const uint32_t* op_flags;  // per-step publication counters of the operand (null: always ready)
  float* ring;               // target layer's ring (ClRing fields)
  uint32_t* done;
  const uint32_t* consumed;
  int sys;
  int active;
  float unscale;             // fp16x2: 2^-(weight scale + operand scale) of this group's product
  const uint16_t* alo;       // fp16x2: lo plane of the target layer's weights (FwdLayer::alo)
  int alo_ld, alo_rows;
  int ko;                    // members splitting K (the planner's choice: each owns Bp / ko columns,
                             // a multiple of 16); 0: ceil(kdim / 512)
};

struct ClParams {
  int L, H, Hp, B, Bp, T;
  int tiles;     // tiles per layer
  int kc;        // active critical members per tile
  int cs;        // cluster size = max(kc, ko over groups)
  int ncomax;    // Bp / min(kc, min ko): receive-slot size (columns) of the carve-up
  int stages;    // B-operand TMA stages (critical CTAs; also the ring region's size)
  int stages_off;   // off CTAs' stages (< stages when the critical CTAs alias their push staging)
  int st_alias;     // backward: critical CTAs stage their split-K pushes inside the B ring (idle
                    // between this step's MMAs and the next step's loads), at byte offset st_off;
                    // off CTAs keep them after their stages_off stages
  int st_off;
  int ring;      // off-partial ring depth (kRing; RW_PP_RING for the sequential pipeline test)
  int n_crit;    // critical layer groups (grid rows y < n_crit); rows may also carry off groups
  const ClRing* cring;   // [n_crit]
  const ClOff* offg;     // [gridDim.y]
  const uint32_t* epoch; // pass counter (device, incremented before each launch)
  int* error;
  unsigned long long timeout_ns;
  unsigned long long* trace;  // [cta][steps][8] (RW_TRACE)
  int trace_steps;
  int dir;    // 0 forward, 1 backward (error codes)
  float unscale;  // critical groups, fp16x2: 2^-(kWScaleLog2 + kHScaleLog2) forward (R.h),
                  // 2^-(kWScaleLog2 + kGScaleLog2) backward (R^T.dG); off groups: ClOff::unscale
  unsigned* gmax; // backward: max |dG| of the pass (float bits; range check of the scaled dG planes)
  int kind;       // cell kind (CellKindDev): the RNN variants share one instantiation
  int debug;  // RW_CL_DEBUG bits. Timing experiments (results invalid): 1 = skip fwd tapes,
              // 4 = skip bwd tape loads, 8 = skip bwd operand stores. Variants (results valid):
              // 32 = backward dG operand stored scattered, 64 = operand k-blocks copied one per
              // bulk copy (not in pairs), 128 = critical fp16x2 CTAs without the fused N = 2N MMA
};

// Shared-memory carve-up (identical for every CTA of a launch, so a local address mapped with
// mapa names the same buffer in a peer).
struct ClSmem {
  uint8_t* a;     // resident A: kClKBlocks x 128 rows x 128 B
  uint8_t* b;     // stages x Bp x 128 B   (forward critical: also the [nco][128] sum buffer)
  float* rx;      // receive slots [cs-1][ncomax][128]
  float* rxoff;   // critical: the off partial of the owned columns [ncomax][128]
  float* st;      // staging [cs-1][ncomax][128] of pushes to peers
  uint64_t* full;
  uint64_t* empty;
  uint64_t* a_full;
  uint64_t* tmem_full;   // [2]
  uint64_t* tmem_empty;  // [2]
  uint64_t* rx_full;     // peers' partials for this step arrived
  uint64_t* push_free;   // every owner consumed this member's previous push
  uint64_t* off_full;    // critical: off partial landed in rxoff
  uint64_t* off_empty;   // critical: epilogue finished reading rxoff
  uint64_t* alo_full;    // fp16x2: A_lo copied into tensor memory (128 epilogue arrivals)
  uint32_t* tmem_slot;
};

__host__ __device__ inline size_t cl_slot_bytes(int ncomax) { return (size_t)ncomax * 128 * 4; }
// `rows`: operand rows per stage (Bp, or 2 Bp for the two fp16x2 planes)
__host__ __device__ inline size_t cl_smem_bytes(int cs, int ncomax, int rows, int stages) {
  return 1024 + (size_t)kClKBlocks * kTileM * kRowBytes + (size_t)stages * rows * kRowBytes +
         (2 * (size_t)(cs - 1) + 1) * cl_slot_bytes(ncomax) + (2 * stages + 12) * 8 + 16;
}

template <class P>
__device__ __forceinline__ ClSmem cl_carve(uint8_t* smem, const ClParams& p, bool crit = true) {
  ClSmem s;
  const size_t slot = cl_slot_bytes(p.ncomax);
  s.a = smem;
  s.b = s.a + kClKBlocks * kTileM * kRowBytes;
  const size_t stage = (size_t)P::kPlanes * p.Bp * kRowBytes;
  s.rx = reinterpret_cast<float*>(s.b + p.stages * stage);
  s.rxoff = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(s.rx) + (p.cs - 1) * slot);
  uint8_t* st_sep = reinterpret_cast<uint8_t*>(s.rxoff) + slot;
  s.st = reinterpret_cast<float*>(!p.st_alias ? st_sep : crit ? s.b + p.st_off : s.b + p.stages_off * stage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(st_sep + (p.st_alias ? 0 : (p.cs - 1) * slot));
  s.full = bars;
  s.empty = bars + p.stages;
  s.a_full = bars + 2 * p.stages;
  s.tmem_full = s.a_full + 1;
  s.tmem_empty = s.a_full + 3;
  s.rx_full = s.a_full + 5;
  s.push_free = s.a_full + 6;
  s.off_full = s.a_full + 7;
  s.off_empty = s.a_full + 8;
  s.alo_full = s.a_full + 9;
  s.tmem_slot = reinterpret_cast<uint32_t*>(s.a_full + 10);
  return s;
}

__device__ __forceinline__ void cl_trace(const ClParams& p, int it, int what) {
  if (p.trace) {
    const unsigned cta = blockIdx.y * gridDim.x + blockIdx.x;
    p.trace[((unsigned long long)cta * p.trace_steps + it) * 16 + what] = globaltimer();
  }
}

// Bulk copy of `bytes` from local smem to the same-offset buffer of cluster rank `dst_rank`,
// completing `bytes` of transaction count on that rank's mbarrier `bar` (local address).
__device__ __forceinline__ void bulk_push(const void* dst_local, const void* src, uint32_t bytes,
                                          uint64_t* bar_local, uint32_t dst_rank) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          map_dsmem(smem_u32(dst_local), dst_rank)),
      "r"(smem_u32(src)), "r"(bytes), "r"(map_dsmem(smem_u32(bar_local), dst_rank))
      : "memory");
}
// Bulk copy global -> local smem, completion on a local mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}


// Receive slot of sender s at owner d (senders = every member but d, in member order).
__device__ __forceinline__ int cl_slot(int s, int d) { return s < d ? s : s - 1; }

// Load 8 accumulator columns of this thread's TMEM lane: acc0 (+ acc1, `two` accumulators N
// columns apart, the two issuers' halves of K), or zeros if nothing was accumulated. `fz` (critical
// CTAs, fp16x2 with fused hi planes): each issuer's accumulator is 2N wide -- [A_hi.B_hi +
// A_lo.B_hi | A_hi.B_lo] -- so the parts are N apart and there are 2 (4 with `two`) of them.
__device__ __forceinline__ void cl_ld8(uint32_t taddr, bool have, float (&v)[8], bool two = false, int N = 0,
                                       bool fz = false) {
  if (have) {
    uint32_t r[8], r2[8];
    tmem_ld_32x32b_x8(taddr, r);
    if (two || fz) tmem_ld_32x32b_x8(taddr + N, r2);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (two || fz) ? __uint_as_float(r[j]) + __uint_as_float(r2[j]) : __uint_as_float(r[j]);
    if (fz && two) {
      tmem_ld_32x32b_x8(taddr + 2 * N, r);
      tmem_ld_32x32b_x8(taddr + 3 * N, r2);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += __uint_as_float(r[j]) + __uint_as_float(r2[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.0f;
  }
}

// Common prologue: barriers, TMEM allocation (2 accumulators of N columns), cluster rendezvous.
__device__ __forceinline__ uint32_t cl_setup(const ClSmem& S, const ClParams& p, uint32_t tmem_cols,
                                             int n_act) {
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], 1);
    }
    mbar_init(S.a_full, 1);
    mbar_init(&S.tmem_full[0], kIssuers);
    mbar_init(&S.tmem_full[1], kIssuers);
    mbar_init(&S.tmem_empty[0], kEpiThreads);
    mbar_init(&S.tmem_empty[1], kEpiThreads);
    mbar_init(S.rx_full, 1);
    mbar_init(S.push_free, n_act > 1 ? n_act - 1 : 1);
    mbar_init(S.off_full, 1);
    mbar_init(S.off_empty, 1);
    mbar_init(S.alo_full, 128);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(S.tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peers' barriers initialised before any remote copy / arrive
  tc_fence_after();
  return *S.tmem_slot;
}

__device__ __forceinline__ void cl_teardown(uint32_t tmem_base, uint32_t tmem_cols) {
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while peers may still copy into its shared memory
  if ((threadIdx.x >> 5) == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}

__device__ __forceinline__ void cl_load_a(const ClSmem& S, const CUtensorMap* a, int kb_lo, int kb_hi,
                                          int row0) {
  const int a_bytes = kTileM * kRowBytes;
  mbar_arrive_expect_tx(S.a_full, (kb_hi - kb_lo) * a_bytes);
  for (int kb = kb_lo; kb < kb_hi; ++kb)
    tma_load_2d(S.a + (kb - kb_lo) * a_bytes, a, S.a_full, kb * 64, row0);
}

// fp16x2: copy this member's A_lo slice (rows row0.., k-blocks [kb_lo, kb_lo + nkb)) from the
// K-major lo plane into tensor memory columns [tmem_alo, tmem_alo + 32 nkb): two fp16 per
// 32-bit column, one A row per TMEM lane. Run by the 128 threads of warps 4..7 (lane quarter =
// warp % 4), once per launch; the MMA issuers wait for `alo_full`.
__device__ __forceinline__ void cl_load_alo(const ClSmem& S, uint32_t tmem_alo, const uint16_t* alo, int ld,
                                            int rows, int row0, int kb_lo, int nkb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, r = q * 32 + lane;
  const bool ok = row0 + r < rows;
  const uint4* src = reinterpret_cast<const uint4*>(alo + (size_t)(ok ? row0 + r : 0) * ld + (size_t)kb_lo * 64);
  const uint32_t taddr = tmem_alo + (uint32_t(q * 32) << 16);
  for (int c = 0; c < nkb * 32; c += 8) {
    uint32_t v[8];
    const uint4 a = ok ? src[c / 4] : make_uint4(0, 0, 0, 0);
    const uint4 b = ok ? src[c / 4 + 1] : make_uint4(0, 0, 0, 0);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    tmem_st_32x32b_x8(taddr + c, v);
  }
  tmem_st_wait();
  tc_fence_before();
  mbar_arrive(S.alo_full);
}

// k-blocks travel in pairs (one 2 x N x 128-byte copy into two adjacent stages, completion on
// the even stage's barrier) when the ring and the step's k-block count are even: >= 16 KB bulk
// copies ingest ~62 B/cycle per SM vs ~50 for 8 KB ones (profiles/ubench/mma_ubench.cu).
__device__ __forceinline__ bool cl_pair_kb(const ClParams& p, int nkb, int stages) {
  return !(p.debug & 64) && (stages % 2 == 0) && (nkb % 2 == 0);
}
// MMA issuers: warps 1 (j = 0) and 3 (j = 1), each converged; elect.sync inside the instruction
// blocks picks the issuing lane (sm100_ptx.cuh umma_bf16_warp). Issuer j multiplies its half of
// the step's k-blocks into accumulator `acc` (= its own TMEM columns).
__device__ __forceinline__ int cl_half0(int nkb) { return (nkb + 1) >> 1; }
// fp16x2: per K = 16 step A_hi.B_hi, A_hi.B_lo (B_lo = the stage's second N rows) and
// A_lo.B_hi with A_lo read from tensor memory at `tmem_alo` (k-block k at column k * 32).
template <class P>
__device__ __forceinline__ void cl_mma_step(const ClSmem& S, const ClParams& p, int it, uint32_t acc, int nkb,
                                            uint32_t idesc, uint32_t& pc, int stages, int N, int j,
                                            uint32_t tmem_alo, bool fz = false, uint32_t idesc2 = 0) {
  const bool pairs = cl_pair_kb(p, nkb, stages);
  const int a_bytes = kTileM * kRowBytes, b_bytes = P::kPlanes * N * kRowBytes;
  const bool l0 = (threadIdx.x & 31) == 0;
  const uint64_t a0 = sdesc_sw128(smem_u32(S.a), 16, 1024), b0 = sdesc_sw128(smem_u32(S.b), 16, 1024);
  // interleaved: issuer j takes k-blocks j, j + 2, ... so both start on the first arrivals
  const int k_lo = j;
  for (int k = k_lo; k < nkb; k += kIssuers) {
    const uint32_t q = pc + k;
    const uint32_t s = q % stages;
    mbar_wait(&S.full[pairs ? (s & ~1u) : s], (q / stages) & 1);
    tc_fence_after();
    if (l0 && k == 0) cl_trace(p, it, 8);  // first k-block arrived
    if (l0 && k == nkb - 1) cl_trace(p, it, 7);
    const uint64_t ad = desc_add(a0, k * a_bytes), bd = desc_add(b0, s * b_bytes);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // 4 x K=16 per 64-element k-block (32 bytes along K)
      const uint32_t acc_on = (k != k_lo || kk) ? 1u : 0u;
      if (P::kPlanes == 2 && fz) {
        // one N = 2N MMA over the stage's [hi rows | lo rows]: columns [0, N) A_hi.B_hi, [N, 2N)
        // A_hi.B_lo (an N = 128 MMA costs what an N = 64 one does, profiles/r01 ubench), then A_lo.B_hi
        // into the first half
        umma_bf16_warp(acc, desc_add(ad, kk * 32), desc_add(bd, kk * 32), idesc2, acc_on);
        umma_ts_f16_warp(acc, tmem_alo + k * 32 + kk * 8, desc_add(bd, kk * 32), idesc, 1u);
        continue;
      }
      umma_bf16_warp(acc, desc_add(ad, kk * 32), desc_add(bd, kk * 32), idesc, acc_on);
      if constexpr (P::kPlanes == 2) {
        umma_bf16_warp(acc, desc_add(ad, kk * 32), desc_add(bd, N * kRowBytes + kk * 32), idesc, 1u);
        umma_ts_f16_warp(acc, tmem_alo + k * 32 + kk * 8, desc_add(bd, kk * 32), idesc, 1u);
      }
    }
    umma_commit_warp(&S.empty[s]);
  }
  pc += nkb;
}

// Producer (one thread): stream the k-blocks [kb_lo, kb_hi) of one step's B operand through the
// stage ring. `blk` is the operand's pre-swizzled step block (sw_off layout); k-block kb sits at
// (kb - kofs) * N * 128 bytes, already in the SWIZZLE_128B smem image: one 1-D bulk copy each.
// (fp16x2: N is the stage's row count, 2 Bp -- both planes of a k-block are adjacent in the image)
__device__ __forceinline__ void cl_load_b(const ClSmem& S, const uint8_t* blk, int kb_lo, int kb_hi, int kofs,
                                          uint32_t& pc, int stages, int N, bool pairs = false) {
  const int b_bytes = N * kRowBytes;
  if (pairs) {
    for (int kb = kb_lo; kb < kb_hi; kb += 2, pc += 2) {
      const int s = pc % stages;  // even
      mbar_wait(&S.empty[s], ((pc / stages) & 1) ^ 1);
      mbar_wait(&S.empty[s + 1], ((pc / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(&S.full[s], 2 * b_bytes);
      bulk_load(S.b + s * b_bytes, blk + (size_t)(kb - kofs) * b_bytes, 2 * b_bytes, &S.full[s]);
    }
    return;
  }
  for (int kb = kb_lo; kb < kb_hi; ++kb, ++pc) {
    const int s = pc % stages;
    mbar_wait(&S.empty[s], ((pc / stages) & 1) ^ 1);
    mbar_arrive_expect_tx(&S.full[s], b_bytes);
    bulk_load(S.b + s * b_bytes, blk + (size_t)(kb - kofs) * b_bytes, b_bytes, &S.full[s]);
  }
}

// Cluster-local split-K reduction of one step: push the columns owned by the other n_act-1
// members, wait for theirs, and return this thread's owned columns summed in member order.
// Thread (quarter q, lane) owns accumulator row q*32+lane; `half` picks its half of the owned
// columns. v_out[i*8 + j] = owned column half*nco/2 + i*8 + j.
// fp16x2: the weight planes carry 2^kWScaleLog2 (common.cuh); the reduced sums are scaled back
// here (exact), so everything downstream sees plain products.
template <class P, int kChunks>
__device__ __forceinline__ void cl_reduce(const ClSmem& S, uint32_t tacc, bool have, bool two, int N, int it, int m,
                                          int n_act, int nco, uint32_t& rxc, float (&v_out)[kChunks * 8],
                                          float unscale, const ClParams* tp = nullptr, bool fz = false) {
  const int et = threadIdx.x - kEpiBase, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = (warp - 4) >> 2, row = q * 32 + lane;
  const uint32_t taddr = tacc + (uint32_t(q * 32) << 16);
  if (n_act > 1) {
    // owners consumed the previous push. CTA-scope waits here and below: a cluster-scope acquire
    // makes every waiting thread invalidate L1 (CCTL.IVALL), ~2 us per step across 256 threads;
    // the bulk copies' data is covered by the mbarrier's complete_tx (as for TMA loads).
    if (it > 0) mbar_wait(S.push_free, (it - 1) & 1);
#pragma unroll 1
    for (int d = 0; d < n_act; ++d) {
      if (d == m) continue;
      float* blk = S.st + (size_t)cl_slot(d, m) * nco * kTileM;
      for (int c0 = half * (nco >> 1); c0 < (half + 1) * (nco >> 1); c0 += 8) {
        float v[8];
        cl_ld8(taddr + d * nco + c0, have, v, two, N, fz);
#pragma unroll
        for (int j = 0; j < 8; ++j) sts_f32(blk + (size_t)(c0 + j) * kTileM + row, v[j]);
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, kEpiThreads);
    if (tp && et == 0) cl_trace(*tp, it, 9);
    if (et == 0) {
      for (int d = 0; d < n_act; ++d) {
        if (d == m) continue;
        bulk_push(S.rx + (size_t)cl_slot(m, d) * nco * kTileM, S.st + (size_t)cl_slot(d, m) * nco * kTileM,
                  (uint32_t)(nco * kTileM * 4), S.rx_full, (uint32_t)d);
      }
    }
  }
  const int own0 = m * nco;
  if (have) {
    // every chunk's TMEM loads in flight before one wait
    uint32_t r[kChunks * 8], r2[kChunks * 8];
    const bool pair01 = two || fz;  // a second part N columns after the first
#pragma unroll
    for (int i = 0; i < kChunks; ++i) {
      uint32_t* ri = r + i * 8;
      tmem_ld_32x32b_x8(taddr + own0 + half * (nco >> 1) + i * 8, *reinterpret_cast<uint32_t(*)[8]>(ri));
      if (pair01) tmem_ld_32x32b_x8(taddr + N + own0 + half * (nco >> 1) + i * 8, *reinterpret_cast<uint32_t(*)[8]>(r2 + i * 8));
    }
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < kChunks * 8; ++i)
      v_out[i] = pair01 ? __uint_as_float(r[i]) + __uint_as_float(r2[i]) : __uint_as_float(r[i]);
    if (fz && two) {  // the second issuer's two parts (2N, 3N)
#pragma unroll
      for (int i = 0; i < kChunks; ++i) {
        tmem_ld_32x32b_x8(taddr + 2 * N + own0 + half * (nco >> 1) + i * 8, *reinterpret_cast<uint32_t(*)[8]>(r + i * 8));
        tmem_ld_32x32b_x8(taddr + 3 * N + own0 + half * (nco >> 1) + i * 8, *reinterpret_cast<uint32_t(*)[8]>(r2 + i * 8));
      }
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < kChunks * 8; ++i) v_out[i] += __uint_as_float(r[i]) + __uint_as_float(r2[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kChunks * 8; ++i) v_out[i] = 0.0f;
  }
  tc_fence_before();
  mbar_arrive(&S.tmem_empty[it & 1]);
  if (tp && et == 0) cl_trace(*tp, it, 10);
  if (n_act > 1) {
    mbar_wait(S.rx_full, rxc & 1);
    ++rxc;
    if (tp && et == 0) cl_trace(*tp, it, 11);
    // sum in member order s = 0 .. n_act-1 (own partial at s = m); each sender's 8 columns of a
    // chunk are read as one batch of independent loads (a per-element volatile chain measured
    // ~1.9 us per step); chunk by chunk to keep register pressure flat
    const float* base = S.rx + (size_t)(half * (nco >> 1)) * kTileM + row;
#pragma unroll
    for (int i = 0; i < kChunks; ++i) {
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
#pragma unroll 1
      for (int s = 0; s < n_act; ++s) {
        if (s == m) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += v_out[i * 8 + j];
        } else {
          const float* src = base + ((size_t)cl_slot(s, m) * nco + i * 8) * kTileM;
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = lds_f32(src + (size_t)j * kTileM);  // explicit ld.shared
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += v[j];
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) v_out[i * 8 + j] = acc[j];
    }
  }
  if constexpr (P::kPlanes == 2) {
#pragma unroll
    for (int i = 0; i < kChunks * 8; ++i) v_out[i] *= unscale;
  }
}

// After every epilogue thread of the owner read the receive slots (named barrier): re-arm for
// the next step and release the slots to the senders (one thread).
// The arrive is relaxed: a release would make this thread wait for all its outstanding global
// stores (the previous step's tapes) first -- measured ~2 us on the backward's critical path.
// The slots' values were consumed into registers before the barrier that precedes this call,
// so the reads are complete before a sender's next bulk copy can overwrite them.
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint64_t* local_bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   map_dsmem(smem_u32(local_bar), rank))
               : "memory");
}
__device__ __forceinline__ void cl_rx_next(const ClSmem& S, int m, int n_act, int nco) {
  if (n_act > 1) {
    mbar_arrive_expect_tx(S.rx_full, (uint32_t)(n_act - 1) * nco * kTileM * 4);
    for (int s = 0; s < n_act; ++s)
      if (s != m) mbar_arrive_remote_relaxed(S.push_free, (uint32_t)s);
  }
}

// Off cluster epilogue of one step: reduce, then store the owned columns of the reduced partial
// into ring slot it % kRing ([Bp][128] fp32) and publish it.
template <class P, int kChunks>
__device__ __forceinline__ void cl_off_step(const ClSmem& S, const ClParams& p, uint32_t tacc, bool two, int it,
                                            int m, int n_act, int nco, uint32_t& rxc, float* ring, uint32_t* done,
                                            const uint32_t* consumed, bool sys, uint32_t epoch, float unscale) {
  const int et = threadIdx.x - kEpiBase, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = (warp - 4) >> 2, row = q * 32 + lane;
  float v[kChunks * 8];
  cl_reduce<P, kChunks>(S, tacc, true, two, p.Bp, it, m, n_act, nco, rxc, v, unscale);
  named_bar_sync(1, kEpiThreads);
  if (et == 0) {
    cl_rx_next(S, m, n_act, nco);
    // ring slot free once every critical member copied step it - kRing (of this pass; the
    // previous passes' T steps are all consumed by then)
    if (it >= p.ring)
      wait_flag_s(consumed, (uint32_t)(p.kc * ((epoch - 1) * p.T + (it - p.ring + 1))), sys, p.error, p.timeout_ns,
                  (1 << 30) | (p.dir << 28) | (blockIdx.y << 20) | ((it + 2) << 4) | 4);
  }
  if (it >= p.ring) named_bar_sync(2, kEpiThreads);
  float* slot = ring + (size_t)(it % p.ring) * p.Bp * kTileM;
  const int c0 = m * nco + half * (nco >> 1);
#pragma unroll
  for (int i = 0; i < kChunks * 8; ++i) slot[(size_t)(c0 + i) * kTileM + row] = v[i];
  fence_proxy_async_global();
  named_bar_sync(1, kEpiThreads);
  if (et == 0) {
    cl_trace(p, it, 15);  // task end (before the release: a consumer's start never precedes it)
    red_release_s(done + it, 1, sys);
  }
}

template <class P, int kChunks>
__device__ __forceinline__ void cl_off_loop(const ClSmem& S, const ClParams& p, uint32_t tmem_base, bool two,
                                            int n_it, int m, int n_act, float* ring, uint32_t* done,
                                            const uint32_t* consumed, bool sys, uint32_t epoch, float unscale) {
  const int et = threadIdx.x - kEpiBase, N = p.Bp, nco = N / n_act;
  uint32_t rxc = 0;
  if (et == 0 && n_act > 1) mbar_arrive_expect_tx(S.rx_full, (uint32_t)(n_act - 1) * nco * kTileM * 4);
  for (int it = 0; it < n_it; ++it) {
    mbar_wait(&S.tmem_full[it & 1], (it >> 1) & 1);
    tc_fence_after();
    if (et == 0) cl_trace(p, it, 2);
    cl_off_step<P, kChunks>(S, p, tmem_base + (it & 1) * 2 * N, two, it, m, n_act, nco, rxc, ring, done, consumed,
                            sys, epoch, unscale);
    if (et == 0) cl_trace(p, it, 3);
  }
}

// Critical producer: prefetch the off partial of step `it` into rxoff (owned columns).
__device__ __forceinline__ void cl_fetch_off(const ClSmem& S, const ClParams& p, const float* ring,
                                             const uint32_t* done, uint32_t target, int it, int m, int nco,
                                             uint32_t& offc, int code, bool sys) {
  if (offc > 0) mbar_wait(S.off_empty, (offc - 1) & 1);
  wait_flag_s(done + it, target, sys, p.error, p.timeout_ns, code);
  fence_proxy_async_global();
  const uint32_t bytes = (uint32_t)(nco * kTileM * 4);
  mbar_arrive_expect_tx(S.off_full, bytes);
  bulk_load(S.rxoff, ring + ((size_t)(it % p.ring) * p.Bp + (size_t)m * nco) * kTileM, bytes, S.off_full);
  ++offc;
}

// ====================================================================== forward
// grid (tiles * 2 * cs, L), cluster (cs, 1, 1). Cluster c: tile c/2, role c%2 (0 critical
// R.h_{t-1}, 1 off W.x_t). Member m < kc (critical) / m < ko_l (off) is active.
// GRU (linear before reset, cells.hpp:283-333): the candidate gate keeps its two halves apart --
// slot 2 sums to W_n x and slot 3 to R_n h (the repacked image holds W_n and R_n in those slots).
template <class P, int kChunks, int kKind = kCellLstm>
__device__ __forceinline__ void cl_fwd_sum(const ClSmem& S, uint32_t tacc, bool two, int N, int t, int m, int kc,
                                           int nco, uint32_t& rxc, uint32_t offc, const ClParams* tp, float unscale,
                                           bool fz = false) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = (warp - 4) >> 2, row = q * 32 + lane;
  float v[kChunks * 8];
  cl_reduce<P, kChunks>(S, tacc, true, two, N, t, m, kc, nco, rxc, v, unscale, nullptr, fz);
  if (tp && threadIdx.x == kEpiBase) cl_trace(*tp, t, 9);
  mbar_wait(S.off_full, offc & 1);
  if (tp && threadIdx.x == kEpiBase) cl_trace(*tp, t, 10);
  float* sum = reinterpret_cast<float*>(S.b);
  // all loads, then all stores: the volatile ld/st.shared keep program order, so an interleaved
  // ld -> st chain pays the smem latency per element (~0.6 us per step at 32 elements)
  float zw[kChunks * 8];
#pragma unroll
  for (int i = 0; i < kChunks * 8; ++i) zw[i] = lds_f32(S.rxoff + (size_t)(half * kChunks * 8 + i) * kTileM + row);
  // (GRU: the forward image keeps W_n in slot 2 of the W columns and R_n in slot 3 of the R
  // columns -- layout_kernels.cuh k_repack -- so slot 2 sums to W_n x and slot 3 to R_n h)
#pragma unroll
  for (int i = 0; i < kChunks * 8; ++i)
    sts_f32(sum + (size_t)(half * kChunks * 8 + i) * kTileM + row, zw[i] + v[i]);  // (zw + zr), cells.hpp:240
}

// kCC: the critical members' owned columns / 16 (Bp / kc / 16), one instantiation each so the
// register allocation of one variant does not spill another's hot loop; kKind: the cell class
template <class P, int kCC, int kKind = kCellLstm>
__global__ void __launch_bounds__(kRecThreads, 1)
    k_cl_fwd(const FwdLayer* __restrict__ layers, ClParams p) {
  const int y = blockIdx.y;
  const int cs = p.cs, kc = p.kc, N = p.Bp;
  const int m = (int)(blockIdx.x % cs), cl_id = (int)(blockIdx.x / cs);
  const int tile = cl_id >> 1;
  const bool crit = (cl_id & 1) == 0;
  // whole idle clusters leave at once (no peer waits on them)
  if (crit ? y >= p.n_crit : !p.offg[y].active) return;
  const int l = y;  // critical: layer y; off: the group's own target (descriptor)
  __shared__ FwdLayer Ly;
  __shared__ ClOff Og;
  __shared__ ClRing Cr;
  __shared__ uint32_t epoch_s;
  if (threadIdx.x == 0) {
    if (crit) {
      Ly = layers[y];
      Cr = p.cring[y];
    } else {
      Og = p.offg[y];
    }
    epoch_s = *p.epoch;
    set_wait_error(p.error);
  }
  __syncthreads();
  const uint32_t epoch = epoch_s;
  const uint32_t flag_target = epoch * (uint32_t)(p.tiles * kc);
  const int nkb_h = p.Hp / 64;
  const int nkb_x = crit ? 0 : Og.kdim / 64;
  const int ko = crit ? Cr.ko : (Og.ko ? Og.ko : (nkb_x + kClKBlocks - 1) / kClKBlocks);
  const int n_act = crit ? kc : ko;
  const bool active = m < n_act;
  const int kofs = crit ? Ly.Ipl / 64 : 0;  // the critical slice sits after W's k-blocks in [W|R]
  int kb_lo = 0, kb_hi = 0;
  if (active) {
    if (crit) {
      kb_lo = kofs + m * nkb_h / kc;
      kb_hi = kofs + (m + 1) * nkb_h / kc;
    } else {
      kb_lo = m * nkb_x / ko;
      kb_hi = (m + 1) * nkb_x / ko;
    }
  }
  const int nkb = kb_hi - kb_lo;
  const bool two = nkb - cl_half0(nkb) > 0;  // the second issuer accumulated something
  const int nco = N / n_act;
  // critical fp16x2 CTAs fuse A_hi.B_hi and A_hi.B_lo into one N = 2N MMA (cl_mma_step): each
  // issuer's accumulator is 2N wide and there is one step buffer -- the next step's MMAs need this
  // CTA's own publish, which follows its accumulator reads (RW_CL_DEBUG bit 128 disables)
  const bool fz = crit && P::kPlanes == 2 && !(p.debug & 128);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ClSmem S = cl_carve<P>(smem, p);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 2 steps x 2 issuers of N accumulator columns (+ fp16x2: A_lo, 32 columns per k-block)
  const uint32_t tmem_need = 4 * N + (P::kPlanes == 2 ? nkb * 32 : 0);
  uint32_t tmem_cols = 32;
  while (tmem_cols < tmem_need) tmem_cols <<= 1;
  const uint32_t tmem_base = cl_setup(S, p, tmem_cols, n_act);
  const uint32_t tmem_alo = tmem_base + 4 * N;
  const int row0 = tile * kTileM;
  const int BR = P::kPlanes * N;  // operand rows per k-block (both fp16x2 planes)
  float* ring = crit ? Cr.ring : Og.ring;
  uint32_t* done = crit ? Cr.done : Og.done;
  uint32_t* consumed = crit ? Cr.consumed : const_cast<uint32_t*>(Og.consumed);
  ring += (size_t)tile * p.ring * N * kTileM;
  done += (size_t)tile * p.T;
  consumed += (size_t)tile * 32;
  const bool sys = crit ? Cr.sys != 0 : Og.sys != 0;
  const uint32_t done_target = epoch * (uint32_t)ko;

  if (active && warp == 0 && lane == 0) {
    // ================= producer: resident A (TMA), then per step the operand (bulk copies)
    const CUtensorMap* amap = crit ? Ly.a[0] : Og.a;
    prefetch_tmap(amap);
    cl_load_a(S, amap, kb_lo, kb_hi, row0);
    uint32_t pc = 0, offc = 0;
    for (int t = 0; t < p.T; ++t) {
      cl_trace(p, t, 0);
      // (fp16x2 step blocks hold both planes: BR rows per k-block)
      if (crit) {
        // the off partial is usually published already: fetch it before waiting for h_{t-1}
        const bool early = flag_reached(ld_relaxed_s(done + t, sys), done_target);
        if (early) cl_fetch_off(S, p, ring, done, done_target, t, m, nco, offc, wait_code(0, l, t, 3), sys);
        if (t > 0) wait_flag(&Ly.flags[t - 1], flag_target, p.error, p.timeout_ns, wait_code(0, l, t, 2));
        fence_proxy_async_global();
        cl_trace(p, t, 1);
        cl_load_b(S, Ly.hsw + (size_t)t * p.Hp * BR * 2, kb_lo, kb_hi, kofs, pc, p.stages, BR, cl_pair_kb(p, nkb, p.stages));
        if (!early) cl_fetch_off(S, p, ring, done, done_target, t, m, nco, offc, wait_code(0, l, t, 3), sys);
        cl_trace(p, t, 14);  // task start: h_{t-1} and the off partial both available
      } else {
        // (system scope when the operand is written by another process: a pipeline stage's input)
        if (Og.op_flags) wait_flag_s(&Og.op_flags[t], flag_target, sys, p.error, p.timeout_ns, wait_code(0, l, t, 1));
        fence_proxy_async_global();
        cl_trace(p, t, 1);
        cl_load_b(S, Og.op + (size_t)(Og.op_blk_off + t) * Og.kdim * BR * 2, kb_lo, kb_hi, 0, pc, p.stages, BR,
                  cl_pair_kb(p, nkb, p.stages));
      }
    }
  } else if (active && (warp == 1 || warp == 3)) {
    // ================= MMA issuers (whole warps, elected lane issues); j = half of the k-blocks
    const int j = warp == 3 ? 1 : 0;
    const uint32_t idesc = idesc_make(P::kFmt, false, false, kTileM, N);
    const uint32_t idesc2 = idesc_make(P::kFmt, false, false, kTileM, 2 * N);
    mbar_wait(S.a_full, 0);
    if constexpr (P::kPlanes == 2) mbar_wait(S.alo_full, 0);
    tc_fence_after();
    uint32_t pc = 0;
    for (int t = 0; t < p.T; ++t) {
      const int ab = t & 1;
      if (t >= 2) {
        mbar_wait(&S.tmem_empty[ab], ((t >> 1) - 1) & 1);
        tc_fence_after();
      }
      cl_mma_step<P>(S, p, t, tmem_base + (fz ? j * 2 * N : (ab * 2 + j) * N), nkb, idesc, pc, p.stages, N, j,
                     tmem_alo, fz, idesc2);
      umma_commit_warp(&S.tmem_full[ab]);
    }
  } else if (active && warp >= 4) {
    const int et = threadIdx.x - kEpiBase;
    if constexpr (P::kPlanes == 2) {
      if (warp < 8)
        cl_load_alo(S, tmem_alo, crit ? Ly.alo : Og.alo, crit ? Ly.alo_ld : Og.alo_ld, crit ? Ly.alo_rows : Og.alo_rows,
                    row0, kb_lo, nkb);
    }
    if (!crit) {
      switch (nco >> 4) {
        case 4: cl_off_loop<P, 4>(S, p, tmem_base, two, p.T, m, n_act, ring, done, consumed, sys, epoch, Og.unscale); break;
        case 3: cl_off_loop<P, 3>(S, p, tmem_base, two, p.T, m, n_act, ring, done, consumed, sys, epoch, Og.unscale); break;
        case 2: cl_off_loop<P, 2>(S, p, tmem_base, two, p.T, m, n_act, ring, done, consumed, sys, epoch, Og.unscale); break;
        default: cl_off_loop<P, 1>(S, p, tmem_base, two, p.T, m, n_act, ring, done, consumed, sys, epoch, Og.unscale); break;
      }
    } else {
      // ================= critical epilogue: reduce + LSTM cell (cells.hpp:227-260)
      const FwdLayer Le = Ly;  // register copy (see cl_bwd_crit)
      const int j = et & 31, cg = et >> 5;  // cell phase: unit j of the tile, column group cg
      const int u = tile * kUnitsPerFwdTile + j;
      const long long Hp = p.Hp, G4 = 4 * Hp;
      const int own0 = m * nco;
      // owned columns per thread: cl = cg + 8k, k < kK (nco = 16 kCC, so no bounds checks). All
      // addressing is hoisted out of the step loop: per step only the block pointers advance
      // (profiles/r02: the per-element 64-bit index math was ~45 % of the cell phase's
      // instructions)
      constexpr int kK = 2 * kCC;
      const float bi = Le.bias[u], bf = Le.bias[Hp + u], bo = Le.bias[2 * Hp + u], bc = Le.bias[3 * Hp + u];
      // LSTM: c_{t-1} of owned columns (c tape block 0 = c0); GRU: h_{t-1} (h0)
      float creg[kK];
#pragma unroll
      for (int k = 0; k < kK; ++k) {
        const float* st = kKind == kCellGru ? Le.h : Le.c;
        creg[k] = kKind != kCellRnnTanh ? st[(long long)(own0 + cg + 8 * k) * Hp + u] : 0.0f;
      }
      const float* sum = reinterpret_cast<const float*>(S.b) + cg * kTileM + j;
      // operand image of h_t (block t+1): column own0 + cg + 8k sits 8k rows of 128 B after column
      // own0 + cg with the same 16-B chunk swizzle (it depends on the row mod 8 only); the fp16x2
      // lo plane is N rows further
      const long long blk_bytes = (long long)p.Hp * BR * 2;
      uint8_t* hsw_t = Le.hsw + blk_bytes + sw_off(u, own0 + cg, BR);
      // layer pipeline: the next stage's layer-input image (its block t = our h_t), over NVLink
      uint8_t* peer_t = Le.hsw_peer ? Le.hsw_peer + sw_off(u, own0 + cg, BR) : nullptr;
      const int lo_off = N * 128;
      // tapes: element (col, u) at col * Hp + u (gates: col * 4Hp + u); col_new = (t + 1) N + own0 + cg + 8k
      const long long kstride = 8 * Hp;
      long long i_new = (long long)(N + own0 + cg) * Hp + u, i_prev = (long long)(own0 + cg) * Hp + u;
      long long i_gate = (long long)(own0 + cg) * G4 + u;
      const long long step_h = (long long)N * Hp, step_g = (long long)N * G4;
      const bool tapes = !(p.debug & 1);
      uint32_t rxc = 0;
      if (et == 0 && kc > 1) mbar_arrive_expect_tx(S.rx_full, (uint32_t)(kc - 1) * nco * kTileM * 4);
      for (int t = 0; t < p.T; ++t) {
        mbar_wait(&S.tmem_full[t & 1], (t >> 1) & 1);
        tc_fence_after();
        if (et == 0) cl_trace(p, t, 2);
        const uint32_t tacc = tmem_base + (fz ? 0 : (t & 1) * 2 * N);
        cl_fwd_sum<P, kCC, kKind>(S, tacc, two, N, t, m, kc, nco, rxc, (uint32_t)t, &p, p.unscale, fz);
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          cl_trace(p, t, 4);
          mbar_arrive(S.off_empty);
          cl_rx_next(S, m, kc, nco);
        }
        // cell phase, operand store first (the critical output)
        float hv[kK], iv[kK], fv[kK], ov[kK], cb[kK], tcv[kK];
#pragma unroll
        for (int k = 0; k < kK; ++k) {
          const float* sk = sum + k * 8 * kTileM;
          if constexpr (kKind == kCellLstm) {
            const float ai = lds_f32(sk + 0 * 32) + bi;
            const float af = lds_f32(sk + 1 * 32) + bf;
            const float ao = lds_f32(sk + 2 * 32) + bo;
            const float ac = lds_f32(sk + 3 * 32) + bc;
            iv[k] = act_sigmoid<P>(ai);  // fp32-parity: libm-free (lstm_step.cuh)
            fv[k] = act_sigmoid<P>(af);
            ov[k] = act_sigmoid<P>(ao);
            cb[k] = act_tanh<P>(ac);
            const float t1 = fv[k] * creg[k];
            const float t2 = iv[k] * cb[k];
            creg[k] = t1 + t2;  // c_t
            tcv[k] = act_tanh<P>(creg[k]);
            hv[k] = ov[k] * tcv[k];
          } else if constexpr (kKind == kCellGru) {  // cells.hpp:294-313 operation order
            const float ar = lds_f32(sk + 0 * 32) + bi;
            const float au = lds_f32(sk + 1 * 32) + bf;
            const float zwn = lds_f32(sk + 2 * 32);
            const float zrn = lds_f32(sk + 3 * 32);
            iv[k] = act_sigmoid<P>(ar);  // r
            fv[k] = act_sigmoid<P>(au);  // u
            const float t1 = zwn + bo;   // W_n x + b_n
            const float t2 = iv[k] * zrn;
            const float an = t1 + t2;
            ov[k] = act_tanh<P>(an);     // n
            const float t3 = fv[k] * creg[k];
            const float om = 1.0f - fv[k];
            const float t4 = om * ov[k];
            hv[k] = t3 + t4;
            cb[k] = zrn;  // the zrh tape (R_n h_{t-1}, the backward's reset-gate input)
            creg[k] = hv[k];
          } else {  // RNN (cells.hpp:200-212)
            const float a = lds_f32(sk) + bi;
            hv[k] = p.kind == kCellRnnRelu ? (a > 0.0f ? a : 0.0f) : act_tanh<P>(a);
          }
          if constexpr (P::kPlanes == 2) {  // hi row n, lo row N + n of the k-block (scaled, common.cuh)
            __half hh, hl;
            f16x2_split(hv[k] * pow2f(kHScaleLog2), hh, hl);
            *reinterpret_cast<__half*>(hsw_t + k * 1024) = hh;
            *reinterpret_cast<__half*>(hsw_t + k * 1024 + lo_off) = hl;
            if (peer_t) {
              *reinterpret_cast<__half*>(peer_t + k * 1024) = hh;
              *reinterpret_cast<__half*>(peer_t + k * 1024 + lo_off) = hl;
            }
          } else {
            const __nv_bfloat16 hb = __float2bfloat16_rn(hv[k]);
            *reinterpret_cast<__nv_bfloat16*>(hsw_t + k * 1024) = hb;
            if (peer_t) *reinterpret_cast<__nv_bfloat16*>(peer_t + k * 1024) = hb;
          }
        }
        if (et == 0) cl_trace(p, t, 3);
        // publish h_t (all operand stores of this CTA, then one gpu-scope release)
        fence_proxy_async_global();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          cl_trace(p, t, 15);  // task end, before the release
          red_release_gpu_add(&Le.flags[t], 1);  // cumulative over the CTA's stores (bar.sync above)
          if (Le.peer_flags) red_release_s(Le.peer_flags + t, 1, true);  // the next stage's input
          red_relaxed_s(consumed, 1, sys);       // ring slot t was copied into rxoff
          cl_trace(p, t, 5);
        }
        // tapes (read only after the pass; the plain h feeds the weight-gradient GEMMs)
        if (tapes) {
#pragma unroll
          for (int k = 0; k < kK; ++k) {
            const long long in = i_new + k * kstride, ip = i_prev + k * kstride;
            if constexpr (kKind == kCellLstm) Le.c[in] = creg[k];
            Le.h[in] = hv[k];
            store_operand<P>(Le.hop, in, P::kPlanes == 2 ? hv[k] * pow2f(kHScaleLog2) : hv[k]);
            if (Le.gates && kKind != kCellRnnTanh) {
              float* gp = Le.gates + i_gate + k * 8 * G4;
              gp[0] = iv[k];
              gp[Hp] = fv[k];
              gp[2 * Hp] = ov[k];
              if constexpr (kKind == kCellLstm) {
                gp[3 * Hp] = cb[k];
                Le.tanhc[ip] = tcv[k];
              } else {
                Le.zrh[ip] = cb[k];
              }
            }
          }
        }
        if (et == 0) cl_trace(p, t, 6);
        hsw_t += blk_bytes;
        if (peer_t) peer_t += blk_bytes;
        i_new += step_h;
        i_prev += step_h;
        i_gate += step_g;
      }
    }
  }
  cl_teardown(tmem_base, tmem_cols);
}

// ====================================================================== backward
// grid (tiles * 2 * cs, L), cluster (cs, 1, 1). Cluster c: tile c/2, role c%2 (0 critical
// R^T.dG_{l,t+1}, 1 off W_{l+1}^T.dG_{l+1,t}; the top layer has no off cluster and adds dy).
// Critical steps t = T-1 .. -1 (t = -1: dh0 = R^T dG_{l,0}, dc0 = carry; engine.hpp:163-170),
// off steps t = T-1 .. 0. Iteration it <-> t = T-1-it.
template <class P, int kChunks, int kKind = kCellLstm>
__device__ __forceinline__ void cl_bwd_crit(const BwdLayer& Ly, const ClSmem& S, const ClParams& p,
                                            uint32_t tmem_base, bool two, int tile, int m, int ko, uint32_t* consumed,
                                            bool sys, uint32_t flag_target, bool fz) {
  const int et = threadIdx.x - kEpiBase, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = (warp - 4) >> 2, row = q * 32 + lane;
  const int N = p.Bp, kc = p.kc, nco = N / kc;
  const int BR = P::kPlanes * N;  // operand rows per k-block (both fp16x2 planes)
  const int u = tile * kTileM + row;
  const bool uok = u < p.Hp;
  const long long Hp = p.Hp, G4 = 4 * Hp;
  const int cbase = m * nco + half * (nco >> 1);  // first batch column of this thread
  float carry[kChunks * 8];
#pragma unroll
  for (int i = 0; i < kChunks * 8; ++i) carry[i] = 0.0f;
  float si = 0.0f, sf = 0.0f, so = 0.0f, sc = 0.0f;  // db partials (cells.hpp:163-168)
  // fp16x2: the dG operand planes carry 2^kGScaleLog2 (common.cuh); the fp32 tapes do not
  constexpr float kGS = P::kPlanes == 2 ? pow2f(kGScaleLog2) : 1.0f;
  float gmax = 0.0f;
  uint32_t rxc = 0, offc = 0;
  // dG_t staging in the B ring (idle between this step's MMA and the next step's loads, which
  // wait for this CTA's own publish): the tile's 8 k-blocks x nco rows of the swizzled image
  const uint32_t dstg = smem_u32(S.b);
  // (measured at B: backward 0.880 ms staged vs 0.903 scattered; RW_CL_DEBUG bit 32 = scattered)
  // GRU writes two images (dgr for the recurrence, dgw for the layer below): scattered stores
  const bool staged = kKind != kCellGru && !(p.debug & 40) &&
                      (size_t)p.stages * BR * kRowBytes >= (size_t)8 * P::kPlanes * nco * 128;
  if (et == 0 && kc > 1) mbar_arrive_expect_tx(S.rx_full, (uint32_t)(kc - 1) * nco * kTileM * 4);
  // Addressing hoisted out of the step loop (as in the forward epilogue): per step only the tape
  // offsets move back by one block; per column k a compile-time multiple of the column stride.
  constexpr int kC = kChunks * 8;  // columns per thread (nco = 16 kChunks)
  const long long col0 = (long long)(p.T - 1) * N + cbase;  // column of (t = T-1, k = 0)
  long long o_g = col0 * G4 + u, o_h = col0 * Hp + u;       // gates / dG tapes, H-row tapes
  const long long st_g = (long long)N * G4, st_h = (long long)N * Hp;
  long long o_dy = ((long long)(p.T - 1) * p.B + cbase) * p.H + u;
  const long long st_dy = (long long)p.B * p.H;
  // staged dG image: gate g of unit u sits at K offset kk_g = q*128 + g*32 + lane of the tile's 8
  // k-blocks; column n = cbase + k has n % 8 == k % 8 (cbase is a multiple of 8), so the 128B
  // swizzle chunk is (kk_g / 8 % 8) ^ (k % 8)
  uint32_t sbase[4];
  int schunk[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int kk = q * 128 + g * 32 + lane;
    const int rows = (P::kPlanes == 2 ? (kk >> 6) * 2 : (kk >> 6)) * nco + half * (nco >> 1);
    sbase[g] = dstg + rows * 128 + (kk & 7) * 2;
    schunk[g] = (kk >> 3) & 7;
  }
  int rg[4];  // operand row rho of each gate (the dG operand planes are rho-ordered)
#pragma unroll
  for (int g = 0; g < 4; ++g) rg[g] = rho_of(g, u);
  for (int it = 0; it <= p.T; ++it, o_g -= st_g, o_h -= st_h, o_dy -= st_dy) {
    const int t = p.T - 1 - it;
    const bool off = ko > 0 && t >= 0;
    const bool have = t <= p.T - 2;  // an R^T.dG_{t+1} product was accumulated
    // tapes of one chunk of 8 columns (registers bound the batch); chunk 0 is loaded before the
    // wait for this step's GEMM, the others inside the cell loop
    float pi[8], pf[8], po[8], pcb[8], pcp[8], ptc[8], dyv[8];
    auto load_tapes = [&](int i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = i * 8 + j;
        pi[j] = pf[j] = po[j] = pcb[j] = ptc[j] = pcp[j] = dyv[j] = 0.0f;
        if (t < 0 || !uok || (p.debug & 4)) continue;
        const float* gp = Ly.gates + o_g + k * G4;
        const long long oh = o_h + k * Hp;
        if constexpr (kKind == kCellLstm) {
          pi[j] = gp[0];
          pf[j] = gp[Hp];
          po[j] = gp[2 * Hp];
          pcb[j] = gp[3 * Hp];
          ptc[j] = Ly.tanhc[oh];
          pcp[j] = Ly.c[oh];  // c_{t-1}: block t of the c tape
        } else if constexpr (kKind == kCellGru) {
          pi[j] = gp[0];        // r
          pf[j] = gp[Hp];       // u
          po[j] = gp[2 * Hp];   // n
          pcb[j] = Ly.zrh[oh];  // R_n h_{t-1}
          pcp[j] = Ly.h[oh];    // h_{t-1}: block t of the h tape
        } else {
          pcp[j] = Ly.h[oh + st_h];  // h_t: block t + 1
        }
        if (Ly.dy && u < p.H && cbase + k < p.B) dyv[j] = Ly.dy[o_dy + (long long)k * p.H];
      }
    };
    load_tapes(0);
    if (kKind == kCellLstm && t >= 1) {
      // pull next step's tape lines (gates x4, tanh(c), c of this warp's 32 units and its
      // columns) from HBM into L2 now, so next step's loads are L2 hits
      const long long tn = t - 1;
      const int ub = tile * kTileM + q * 32;
      for (int pi = lane; pi < kC * 6; pi += 32) {
        const long long col = tn * N + cbase + pi / 6;
        const int ty = pi % 6;
        const float* a = ty < 4 ? Ly.gates + col * G4 + ty * Hp + ub
                                : (ty == 4 ? Ly.tanhc : Ly.c) + col * Hp + ub;
        if (ub < p.Hp) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
      }
    }
    mbar_wait(&S.tmem_full[it & 1], (it >> 1) & 1);
    tc_fence_after();
    if (et == 0) cl_trace(p, it, 2);
    float acc[kC];
    cl_reduce<P, kChunks>(S, tmem_base + (fz ? 0 : (it & 1) * 2 * N), have, two, N, it, m, kc, nco, rxc, acc, p.unscale,
                          &p, fz);
    if (et == 0) cl_trace(p, it, 12);
    float dab[kC];  // d_above: W_{l+1}^T dG_{l+1,t} (off cluster) or dy (top layer)
    if (off) {
      mbar_wait(S.off_full, offc & 1);
#pragma unroll
      for (int i = 0; i < kC; ++i) dab[i] = lds_f32(S.rxoff + (size_t)(half * kC + i) * kTileM + row);
    }
    if (et == 0) cl_trace(p, it, 13);
    named_bar_sync(1, kEpiThreads);
    if (et == 0) {
      cl_trace(p, it, 4);
      if (off) mbar_arrive(S.off_empty);
      cl_rx_next(S, m, kc, nco);
    }
    if (off) ++offc;
    if (t < 0) {  // dh0 / dc0 (engine.hpp:163-170); GRU: dh0 = R^T dgr_0 + the direct term dh_0 u_0
      if (uok) {
#pragma unroll
        for (int i = 0; i < kC; ++i) {
          const long long n = cbase + i;
          Ly.dh0[n * Hp + u] = kKind == kCellGru ? acc[i] + carry[i] : acc[i];
          if constexpr (kKind == kCellLstm) Ly.dc0[n * Hp + u] = carry[i];
        }
      }
      break;
    }
    float g_i[kC], g_f[kC], g_o[kC], g_c[kC];
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      const int j = k & 7;
      if (j == 0 && k > 0) load_tapes(k >> 3);
      // dh = d_above + carry_h (GRU: carry_h = R^T dgr_{t+1} + the direct term dh_{t+1} u_{t+1})
      const float ch = kKind == kCellGru ? acc[k] + carry[k] : acc[k];
      const float dh = off ? dab[k] + ch : (Ly.dy ? dyv[j] + ch : ch);
      if constexpr (kKind == kCellLstm) {  // cells.hpp:424-447 operation order
        const float q1 = dh * po[j];
        const float s0 = ptc[j] * ptc[j];
        const float s1 = 1.0f - s0;
        const float q2 = q1 * s1;
        const float dc = carry[k] + q2;
        const float a1 = dc * pcb[j], a2 = a1 * pi[j], a3 = 1.0f - pi[j];
        const float b1 = dc * pcp[j], b2 = b1 * pf[j], b3 = 1.0f - pf[j];
        const float c1 = dh * ptc[j], c2 = c1 * po[j], c3 = 1.0f - po[j];
        const float d1 = dc * pi[j], d2 = pcb[j] * pcb[j], d3 = 1.0f - d2;
        g_i[k] = a2 * a3;
        g_f[k] = b2 * b3;
        g_o[k] = c2 * c3;
        g_c[k] = d1 * d3;
        carry[k] = dc * pf[j];
      } else if constexpr (kKind == kCellGru) {  // cells.hpp:514-538 operation order
        const float om = 1.0f - pf[j];
        const float dn = dh * om;
        const float s = po[j] * po[j];
        const float s1 = 1.0f - s;
        const float dnp = dn * s1;
        const float tt = pcp[j] - po[j];
        const float q = dh * tt;
        const float q2 = q * pf[j];
        const float dgu = q2 * om;
        const float r0 = dnp * pcb[j];
        const float r1 = r0 * pi[j];
        const float r2 = 1.0f - pi[j];
        g_i[k] = r1 * r2;     // dgw = dgr (reset gate)
        g_f[k] = dgu;         // dgw = dgr (update gate)
        g_o[k] = dnp;         // dgw (candidate); dgr = dnp r
        g_c[k] = dnp * pi[j]; // slot 3 carries dgr of the candidate (slot 3 of dgw is zero)
        carry[k] = dh * pf[j];
      } else {  // RNN (cells.hpp:370-383)
        if (p.kind == kCellRnnRelu) {
          g_i[k] = pcp[j] > 0.0f ? dh : 0.0f;
        } else {
          const float s = pcp[j] * pcp[j];
          const float s1 = 1.0f - s;
          g_i[k] = dh * s1;
        }
        g_f[k] = g_o[k] = g_c[k] = 0.0f;
      }
      if (staged) {
        // staging rows (k-block, plane, owned column): fp16x2 keeps each k-block's hi and lo runs adjacent
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const float gv = g == 0 ? g_i[k] : g == 1 ? g_f[k] : g == 2 ? g_o[k] : g_c[k];
          const uint32_t a = sbase[g] + k * 128 + ((schunk[g] ^ (k & 7)) << 4);
          if constexpr (P::kPlanes == 2) {
            __half hh, hl;
            gmax = fmaxf(gmax, fabsf(gv));
            f16x2_split(gv * kGS, hh, hl);
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(a), "h"(__half_as_ushort(hh)));
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(a + nco * 128), "h"(__half_as_ushort(hl)));
          } else {
            sts_bf16(a, gv);
          }
        }
      } else if (uok && !(p.debug & 8)) {
        uint8_t* blk = Ly.dgsw + (size_t)t * G4 * BR * 2;
        const int n = cbase + k;
        if constexpr (kKind == kCellGru) {  // the W-side image (layer below): slots r, u, n, 0
          uint8_t* wblk = Ly.dgwsw + (size_t)t * G4 * BR * 2;
#pragma unroll
          for (int g = 0; g < 3; ++g) {
            const float gv = g == 0 ? g_i[k] : g == 1 ? g_f[k] : g_o[k];
            if constexpr (P::kPlanes == 2) {
              __half hh, hl;
              f16x2_split(gv * kGS, hh, hl);
              *reinterpret_cast<__half*>(wblk + sw_off(rg[g], n, BR)) = hh;
              *reinterpret_cast<__half*>(wblk + sw_off(rg[g], N + n, BR)) = hl;
            } else {
              *reinterpret_cast<__nv_bfloat16*>(wblk + sw_off(rg[g], n, N)) = __float2bfloat16_rn(gv);
            }
          }
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          // the R-side image (this layer's recurrence); GRU: slots r, u, n <- dgr (slot 3's value), 0
          float gv = g == 0 ? g_i[k] : g == 1 ? g_f[k] : g == 2 ? g_o[k] : g_c[k];
          if (kKind == kCellGru) gv = g == 2 ? g_c[k] : g == 3 ? 0.0f : gv;
          if constexpr (P::kPlanes == 2) {
            __half hh, hl;
            gmax = fmaxf(gmax, fabsf(gv));
            f16x2_split(gv * kGS, hh, hl);
            *reinterpret_cast<__half*>(blk + sw_off(rg[g], n, BR)) = hh;
            *reinterpret_cast<__half*>(blk + sw_off(rg[g], N + n, BR)) = hl;
          } else {
            *reinterpret_cast<__nv_bfloat16*>(blk + sw_off(rg[g], n, N)) = __float2bfloat16_rn(gv);
          }
        }
      }
    }
    if (staged) {
      // 8 k-blocks x (planes x) nco rows x 128 B, each (k-block, plane)'s rows one contiguous
      // run of the operand image (fp16x2: hi rows at m*nco, lo rows at N + m*nco of the k-block)
      named_bar_sync(1, kEpiThreads);
      uint8_t* blk = Ly.dgsw + (size_t)t * G4 * BR * 2;
      const int kb0 = tile * 8, nkb = min(8, (int)(G4 / 64) - kb0);
      constexpr int per = 16 * kChunks * 8;  // nco * 8 chunks of 16 B per (k-block, plane)
      for (int i = et; i < nkb * P::kPlanes * per; i += kEpiThreads) {
        const int kp = i / per, r = i - kp * per;  // kp = k-block * planes + plane
        const int kb = kp / P::kPlanes, pl = kp - kb * P::kPlanes;
        const uint4 v = lds_v4(dstg + i * 16);
        *reinterpret_cast<uint4*>(blk + ((size_t)(kb0 + kb) * BR + pl * N + m * nco) * 128 + (size_t)r * 16) = v;
      }
    }
    if (et == 0) cl_trace(p, it, 3);
    // publish dG_{l,t}
    fence_proxy_async_global();
    named_bar_sync(1, kEpiThreads);
    if (et == 0) {
      cl_trace(p, it, 15);  // task end, before the release
      red_release_gpu_add(&Ly.flags[t], 1);
      if (off) red_relaxed_s(consumed, 1, sys);
      cl_trace(p, it, 5);
    }
    if (uok) {
#pragma unroll
      for (int k = 0; k < kC; ++k) {
        const long long ob = o_g - u + k * G4;  // column (t, cbase + k) of the rho-ordered planes
        const float wc = kKind == kCellGru ? 0.0f : g_c[k];  // slot 3 of dgw (GRU: holds dgr_n)
        store_operand<P>(Ly.dgop, ob + rg[0], g_i[k] * kGS);
        store_operand<P>(Ly.dgop, ob + rg[1], g_f[k] * kGS);
        store_operand<P>(Ly.dgop, ob + rg[2], g_o[k] * kGS);
        store_operand<P>(Ly.dgop, ob + rg[3], wc * kGS);
        float* dgp = Ly.dg + o_g + k * G4;
        dgp[0] = g_i[k];
        dgp[Hp] = g_f[k];
        dgp[2 * Hp] = g_o[k];
        dgp[3 * Hp] = wc;
        if constexpr (kKind == kCellGru) {  // dgr: r, u as dgw, candidate dnp r (cells.hpp:527-529)
          store_operand<P>(Ly.dgrop, ob + rg[0], g_i[k] * kGS);
          store_operand<P>(Ly.dgrop, ob + rg[1], g_f[k] * kGS);
          store_operand<P>(Ly.dgrop, ob + rg[2], g_c[k] * kGS);
          store_operand<P>(Ly.dgrop, ob + rg[3], 0.0f);
          float* dgq = Ly.dgr + o_g + k * G4;
          dgq[0] = g_i[k];
          dgq[Hp] = g_f[k];
          dgq[2 * Hp] = g_c[k];
        }
        si += g_i[k];
        sf += g_f[k];
        so += g_o[k];
        sc += wc;
      }
    }
    if (et == 0) cl_trace(p, it, 6);
  }
  if constexpr (P::kPlanes == 2) {
    // range of the scaled dG planes: one atomic per warp (positive floats order as integers)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    if (lane == 0 && p.gmax) atomicMax(p.gmax, __float_as_uint(gmax));
  }
  if (uok && Ly.dbp) {
    float* d = Ly.dbp + (long long)(m * 2 + half) * G4 + u;
    d[0] = si;
    d[Hp] = sf;
    d[2 * Hp] = so;
    d[3 * Hp] = sc;
  }
}

template <class P, int kCC, int kKind = kCellLstm>
__global__ void __launch_bounds__(kRecThreads, 1)
    k_cl_bwd(const BwdLayer* __restrict__ layers, ClParams p) {
  const int y = blockIdx.y;
  const int cs = p.cs, kc = p.kc, N = p.Bp;
  const int m = (int)(blockIdx.x % cs), cl_id = (int)(blockIdx.x / cs);
  const int tile = cl_id >> 1;
  const bool crit = (cl_id & 1) == 0;
  if (crit ? y >= p.n_crit : !p.offg[y].active) return;  // idle cluster: nobody waits on it
  const int l = y;
  __shared__ BwdLayer Ly;
  __shared__ ClOff Og;
  __shared__ ClRing Cr;
  __shared__ uint32_t epoch_s;
  if (threadIdx.x == 0) {
    if (crit) {
      Ly = layers[y];
      Cr = p.cring[y];
    } else {
      Og = p.offg[y];
    }
    epoch_s = *p.epoch;
    set_wait_error(p.error);
  }
  __syncthreads();
  const uint32_t epoch = epoch_s;
  const uint32_t flag_target = epoch * (uint32_t)(p.tiles * kc);
  const int G4p = 4 * p.Hp;
  const int nkb_r = G4p / 64;
  const int kofs = crit && Ly.has_up ? G4p / 64 : 0;  // R^T sits after W_{l+1}^T in [W_{l+1}^T | R_l^T]
  const int nkb_o = crit ? 0 : Og.kdim / 64;
  const int ko = crit ? Cr.ko : (Og.ko ? Og.ko : (nkb_o + kClKBlocks - 1) / kClKBlocks);
  const int n_act = crit ? kc : ko;
  const bool active = m < n_act;
  int kb_lo = 0, kb_hi = 0;
  if (active) {
    if (crit) {
      kb_lo = kofs + m * nkb_r / kc;
      kb_hi = kofs + (m + 1) * nkb_r / kc;
    } else {
      kb_lo = m * nkb_o / ko;
      kb_hi = (m + 1) * nkb_o / ko;
    }
  }
  const int nkb = kb_hi - kb_lo;
  const bool two = nkb - cl_half0(nkb) > 0;  // the second issuer accumulated something
  const int nco = N / n_act;
  // critical fp16x2 CTAs fuse A_hi.B_hi and A_hi.B_lo into one N = 2N MMA (cl_mma_step): each
  // issuer's accumulator is 2N wide and there is one step buffer -- the next step's MMAs need this
  // CTA's own publish, which follows its accumulator reads (RW_CL_DEBUG bit 128 disables)
  const bool fz = crit && P::kPlanes == 2 && !(p.debug & 128);
  const int n_it = crit ? p.T + 1 : p.T;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ClSmem S = cl_carve<P>(smem, p, crit);
  const int stages = crit ? p.stages : p.stages_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tmem_need = 4 * N + (P::kPlanes == 2 ? nkb * 32 : 0);  // as k_cl_fwd
  uint32_t tmem_cols = 32;
  while (tmem_cols < tmem_need) tmem_cols <<= 1;
  const uint32_t tmem_base = cl_setup(S, p, tmem_cols, n_act);
  const uint32_t tmem_alo = tmem_base + 4 * N;
  const int row0 = tile * kTileM;
  const int BR = P::kPlanes * N;
  float* ring = crit ? Cr.ring : Og.ring;
  uint32_t* done = crit ? Cr.done : Og.done;
  uint32_t* consumed = crit ? Cr.consumed : const_cast<uint32_t*>(Og.consumed);
  ring += (size_t)tile * p.ring * N * kTileM;
  done += (size_t)tile * p.T;
  consumed += (size_t)tile * 32;
  const bool sys = crit ? Cr.sys != 0 : Og.sys != 0;
  const uint32_t done_target = epoch * (uint32_t)ko;

  if (active && warp == 0 && lane == 0) {
    const CUtensorMap* amap = crit ? Ly.a[0] : Og.a;
    prefetch_tmap(amap);
    cl_load_a(S, amap, kb_lo, kb_hi, row0);
    uint32_t pc = 0, offc = 0;
    for (int it = 0; it < n_it; ++it) {
      const int t = p.T - 1 - it;
      const bool off = crit && ko > 0 && t >= 0;
      const bool load = !crit || t <= p.T - 2;
      cl_trace(p, it, 0);
      const bool early = off && flag_reached(ld_relaxed_s(done + it, sys), done_target);
      if (early) cl_fetch_off(S, p, ring, done, done_target, it, m, nco, offc, wait_code(1, l, t, 3), sys);
      if (load) {
        if (crit)
          wait_flag(&Ly.flags[t + 1], flag_target, p.error, p.timeout_ns, wait_code(1, l, t, 2));
        else if (Og.op_flags)
          wait_flag(&Og.op_flags[t], flag_target, p.error, p.timeout_ns, wait_code(1, l, t, 1));
        // aliased push staging: the peers consumed this CTA's previous pushes (implied by the flag
        // -- every member published after reading them -- and made formal by the barrier) before
        // the ring is refilled
        if (crit && p.st_alias && kc > 1 && it > 0) mbar_wait(S.push_free, (it - 1) & 1);
        fence_proxy_async_global();
        cl_trace(p, it, 1);
        if (crit)
          cl_load_b(S, Ly.dgsw + (size_t)(t + 1) * G4p * BR * 2, kb_lo, kb_hi, kofs, pc, stages, BR,
                    cl_pair_kb(p, nkb, stages));
        else
          cl_load_b(S, Og.op + (size_t)(Og.op_blk_off + t) * Og.kdim * BR * 2, kb_lo, kb_hi, 0, pc, stages, BR,
                    cl_pair_kb(p, nkb, stages));
      }
      if (off && !early) cl_fetch_off(S, p, ring, done, done_target, it, m, nco, offc, wait_code(1, l, t, 3), sys);
      if (crit) cl_trace(p, it, 14);  // task start: dG_{t+1} and the off partial (d_above) both available
    }
  } else if (active && (warp == 1 || warp == 3)) {
    const int j = warp == 3 ? 1 : 0;
    const uint32_t idesc = idesc_make(P::kFmt, false, false, kTileM, N);
    const uint32_t idesc2 = idesc_make(P::kFmt, false, false, kTileM, 2 * N);
    mbar_wait(S.a_full, 0);
    if constexpr (P::kPlanes == 2) mbar_wait(S.alo_full, 0);
    tc_fence_after();
    uint32_t pc = 0;
    for (int it = 0; it < n_it; ++it) {
      const int t = p.T - 1 - it;
      const int ab = it & 1;
      if (it >= 2) {
        mbar_wait(&S.tmem_empty[ab], ((it >> 1) - 1) & 1);
        tc_fence_after();
      }
      if (!crit || t <= p.T - 2)
        cl_mma_step<P>(S, p, it, tmem_base + (fz ? j * 2 * N : (ab * 2 + j) * N), nkb, idesc, pc, stages, N, j,
                       tmem_alo, fz, idesc2);
      umma_commit_warp(&S.tmem_full[ab]);
    }
  } else if (active && warp >= 4) {
    if constexpr (P::kPlanes == 2) {
      if (warp < 8)
        cl_load_alo(S, tmem_alo, crit ? Ly.alo : Og.alo, crit ? Ly.alo_ld : Og.alo_ld, crit ? Ly.alo_rows : Og.alo_rows,
                    row0, kb_lo, nkb);
    }
    if (!crit) {
      switch (nco >> 4) {
        case 4: cl_off_loop<P, 4>(S, p, tmem_base, two, n_it, m, n_act, ring, done, consumed, sys, epoch, Og.unscale); break;
        case 3: cl_off_loop<P, 3>(S, p, tmem_base, two, n_it, m, n_act, ring, done, consumed, sys, epoch, Og.unscale); break;
        case 2: cl_off_loop<P, 2>(S, p, tmem_base, two, n_it, m, n_act, ring, done, consumed, sys, epoch, Og.unscale); break;
        default: cl_off_loop<P, 1>(S, p, tmem_base, two, n_it, m, n_act, ring, done, consumed, sys, epoch, Og.unscale); break;
      }
    } else {
      cl_bwd_crit<P, kCC, kKind>(Ly, S, p, tmem_base, two, tile, m, ko, consumed, sys, flag_target, fz);
    }
  }
  cl_teardown(tmem_base, tmem_cols);
}

}  // namespace rw

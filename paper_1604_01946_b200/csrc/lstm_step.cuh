// lstm_step.cuh -- the fused recurrent kernels (SURVEY K2/K3 forward, K4 backward).
//
// Forward, per (layer l, step t, 128-row tile of gate-interleaved units):
//     Z = [W_l | R_l] . [x_{l,t} ; h_{l,t-1}]          (tcgen05, K = I_l + H)
//     i,f,o = sigmoid, c' = tanh, c = f c_prev + i c', h = o tanh(c)   (epilogue)
// The LSTM cell of cells.hpp:227-260 is fused into the GEMM epilogue; the input GEMM
// W.x (engine.hpp:347-365) is fused into the same accumulator (K concatenation).
// Backward, per (layer l, step t, 128-unit tile):
//     dh = [W_{l+1}^T | R_l^T] . [dG_{l+1,t} ; dG_{l,t+1}]  (+ dy for the top layer)
//     dG_t, carry_c = cells.hpp:424-447 chain                (epilogue)
// i.e. output_gemm of the layer above (engine.hpp:564-585) and recurrent_backward_gemm
// (engine.hpp:538-560) share one accumulator and the pointwise backward runs on it.
//
// A tile's K range may be split over a cluster of `ksplit` CTAs (split-K). Each CTA owns
// 1/ksplit of the batch columns for the cell epilogue: after its MMAs it pushes every
// partial-accumulator column to the owning CTA's receive buffer with st.shared::cluster
// (fire-and-forget DSMEM stores), signals with a release-arrive on every rank's mbarrier,
// and then reduces only local shared memory (fixed rank order: deterministic).
//
// Two launch modes share the code:
//   stepwise   : one launch per (layer, step); weights streamed by TMA every step;
//                ordering comes from the stream/graph.
//   persistent : one launch for all layers and steps (wavefront); each CTA owns
//                one (layer, tile, k-slice), keeps its weight slice resident in shared
//                memory, and waits on gpu-scope per-(layer, step) completion counters
//                (release/acquire) instead of kernel boundaries.
//
// Threads: 384 = warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator, warp 3 idle,
// warps 4..11 epilogue (warp w and w+4 share TMEM lane quarter w%4 and split the columns).
#pragma once

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace rw {

constexpr int kMaxLayers = 16;
constexpr int kXChunk = 64;        // batch columns per epilogue exchange chunk
constexpr int kRecThreads = 384;
constexpr int kEpiThreads = 256;
constexpr int kEpiBase = 128;      // first epilogue thread

struct FwdLayer {
  const CUtensorMap* a[2];   // [W|R] gate-interleaved rows, K-major: {Ipl + Hp, 4Hp}
  const CUtensorMap* bx[2];  // layer input operand, K-major: {Ipl, cols}
  const CUtensorMap* bh[2];  // own hidden operand, K-major: {Hp, Bp(T+1)}
  int Ipl;
  int bx_col_off;            // x_op: 0; h_op[l-1]: Bp (block t+1 holds h_t)
  const float* bias;         // 4Hp, row g*Hp + u
  float* h;                  // Hp x Bp(T+1)
  float* c;                  // Hp x Bp(T+1)
  void* hop[2];              // operand planes, Hp x Bp(T+1)
  float* gates;              // 4Hp x Bp T (row g*Hp + u), null in inference
  float* tanhc;              // Hp x Bp T, null in inference
  uint32_t* flags;           // [T] completion counters
  // cluster schedule: pre-swizzled bf16 operand step blocks (layout_kernels.cuh sw_off)
  uint8_t* hsw;              // own h: block t+1 = h_t, block 0 = h0 (Hp x Bp per block; fp16x2: x 2 planes)
  const uint8_t* bxsw;       // layer input: x (blocks 0..T-1, Ipl x Bp) or hsw of layer l-1 (+1 block)
  int bx_blk_off;
  // layer-sequential schedule: the input projection W.x of every step was computed beforehand by
  // one GEMM into this buffer (gate-major, [col][g*Hp + u]: the gates tape, which the cell
  // overwrites in place); the step GEMM then covers only R.h_{t-1}
  const float* zx;
  // CTA-pair stepwise forward (k_lstm_fwd<_, true>): bf16 operand maps with Bp/2-row boxes, each
  // CTA of a pair loading half of the batch columns
  const CUtensorMap* bx2;
  const CUtensorMap* bh2;
  // cluster schedule, fp16x2: the lo plane of [W|R] (K-major rows of alo_ld elements, alo_rows
  // rows), copied once into tensor memory as the A operand of the lo x hi products
  const uint16_t* alo;
  int alo_ld, alo_rows;
  float* zrh;                // GRU: R-side candidate pre-activation R_n h_{t-1} tape (Hp x Bp T)
  // layer pipeline (rw_pp_link, forward): the next stage's layer-input image and its per-step
  // input counters -- the last layer of a stage also writes h_t there (block t) and releases it
  uint8_t* hsw_peer;
  uint32_t* peer_flags;
  // layer pipeline, persistent / stepwise schedules: the next stage's plain layer-input planes
  // (x_op, row length peer_ld) -- the last layer stores h_t into block t there, then releases
  // peer_flags[t] (system scope) once per CTA
  void* xop_peer[2];
  int peer_ld;
};

struct BwdLayer {
  const CUtensorMap* a[2];   // [W_{l+1}^T | R_l^T] rows = units, K-major: {Kb, Hp}
  const CUtensorMap* bup[2]; // dG operand of layer l+1, K-major: {4Hp, Bp T}
  const CUtensorMap* bg[2];  // dG operand of layer l,   K-major: {4Hp, Bp T}
  int has_up;
  const float* dy;           // raw dy (H x B T), top layer only
  const float* gates;
  const float* tanhc;
  const float* c;
  float* dg;                 // fp32 dG tape, 4Hp x Bp T, row g*Hp + u
  void* dgop[2];             // operand planes, row rho
  float* carry_c;            // Hp x Bp
  float* dbp;                // [ceil(Bp/64)*ksplit*2][4Hp] bias-gradient partial sums
  float* dh0;                // Hp x Bp
  float* dc0;                // Hp x Bp
  uint32_t* flags;           // [T]
  // cluster schedule: pre-swizzled bf16 dG step blocks (4Hp x Bp per block, K index rho)
  uint8_t* dgsw;
  const uint8_t* bupsw;      // dgsw of layer l+1
  // layer-sequential schedule: d_above = W_{l+1}^T dG_{l+1} for every step from one GEMM
  // ([col][u], Hp x Bp T); the step GEMM covers only R^T dG_{t+1}, at A k-block offset akofs
  const float* dabove;
  int akofs;
  // CTA-pair persistent backward (k_lstm_bwd<_, true>): bf16 dG operand maps with Bp/2-row boxes
  const CUtensorMap* bup2;
  const CUtensorMap* bg2;
  const uint16_t* alo;       // cluster schedule, fp16x2: lo plane of [W_{l+1}^T | R_l^T] (as FwdLayer)
  int alo_ld, alo_rows;
  // GRU / RNN (cluster schedule): the layer's h tape (GRU h_{t-1}, RNN h_t), the zrh tape, and the
  // R-side gate gradients dgr (GRU only: they differ from dgw in the candidate gate) -- fp32 tape,
  // operand planes (dR), and the pre-swizzled image the recurrence reads; dgsw then holds dgr and
  // dgwsw the W-side image the layer below reads
  const float* h;
  const float* zrh;
  float* dgr;
  void* dgrop[2];
  uint8_t* dgwsw;
  // layer pipeline, persistent / stepwise schedules: the previous stage's dG-input planes (the
  // layout of dgop) -- the first layer stores its W-side dG_t there too, then releases
  // peer_flags[t] (system scope) once per CTA
  void* dg_peer[2];
  uint32_t* peer_flags;
};

struct RecParams {
  int L, H, Hp, B, Bp, T;
  int ksplit;
  int tiles;          // tiles per layer
  int layer_base;     // layer of blockIdx.y == 0
  int t_first;        // first step of this launch (fwd: ascending, bwd: descending)
  int n_steps;        // steps in this launch (bwd: may include the dh0 step t = -1)
  int persistent;
  int resident;
  int a_slots;        // resident A k-block slots (identical in every CTA of a cluster, so
                      // DSMEM offsets of the receive buffer / barriers match across ranks)
  int acc_kb;         // k-blocks per TMEM accumulator (fp32 promotion); accumulators summed
  int n_acc;          // in fp32 by the epilogue (1 = single accumulator)
  int promo;          // promotion ring (promo_drain) -- acc_kb k-blocks per chunk, n_acc slots after
                      // the fp32 sum region (TMEM: N x (1 + n_acc) columns); chunks never straddle
                      // the two K segments (fwd W.x | R.h, bwd W_{l+1}^T.dG | R^T.dG)
  float us_in0, us_in, us_rec;  // fp16x2 unscale of a chunk's product (common.cuh): K segment 0 of
                      // layer 0 / of layers >= 1, segment 1 -- applied by the drain (1 otherwise)
  unsigned* gmax;     // backward, fp16x2: max |dG| of the pass (range check of the scaled planes)
  int stages;
  int a_prefetch;     // streamed A: L2 prefetch distance in k-blocks (0 = off)
  uint32_t flag_target;
  int* error;
  unsigned long long timeout_ns;
  unsigned int* progress;     // debug only (RW_DEBUG_HANG_S): [cta][4] role progress words
  unsigned long long* trace;  // optional [cta][n_steps][8] %globaltimer stamps (RW_TRACE)
  int kind;                   // cell kind (CellKindDev): the RNN variants share one instantiation
  // layer pipeline (persistent / stepwise): per-step counters a neighbouring stage releases at
  // system scope -- forward: layer 0's input h_t; backward: the top layer's dG from above.
  // Cumulative over passes: target = *pp_epoch (this context's pass count in that direction)
  // x pp_in_flags[T] (the sender's CTAs per step, written at link time).
  const uint32_t* pp_in_flags;
  const uint32_t* pp_epoch;
  int acc_dbuf;  // persistent kernels: two accumulator buffers when a step fits one (RW_ACC_DBUF)
};

__device__ __forceinline__ uint32_t pp_target(const RecParams& p) {
  return p.pp_in_flags ? *p.pp_epoch * p.pp_in_flags[p.T] : 0u;
}

// Trace stamps per (CTA, step): 0 producer starts waiting for its inputs, 1 inputs ready
// (flags acquired, loads issued), 2 accumulator ready in TMEM, 3 partials pushed, 4 exchange
// complete, 5 cell math + stores done, 6 exchange buffer released, 7 step published.
__device__ __forceinline__ void trace_stamp(const RecParams& p, int it, int what) {
  if (p.trace) {
    const unsigned cta = blockIdx.y * gridDim.x + blockIdx.x;
    p.trace[((unsigned long long)cta * p.n_steps + it) * 8 + what] = globaltimer();
  }
}

// Debug progress word: (step iteration << 12) | (role marker); volatile store to mapped
// host memory so the host can print where a stuck persistent kernel is waiting.
__device__ __forceinline__ void progress(const RecParams& p, int role, int it, int marker) {
  if (p.progress) {
    const unsigned cta = blockIdx.y * gridDim.x + blockIdx.x;
    *(volatile unsigned*)(p.progress + cta * 4 + role) = (unsigned(it + 2) << 12) | unsigned(marker);
  }
}

// ------------------------------------------------------------------ small helpers
// fp16x2 split operands (common.cuh PrecF16x2): operand planes carry power-of-two scales
template <class P>
constexpr bool kF16Ops = P::kPlanes == 2 && !P::kTF32;

template <class P>
__device__ __forceinline__ void store_operand(void* const* planes, long long idx, float v) {
  if constexpr (P::kPlanes == 1) {
    static_cast<__nv_bfloat16*>(planes[0])[idx] = __float2bfloat16_rn(v);
  } else if constexpr (!P::kTF32) {  // fp16x2
    __half hi, lo;
    f16x2_split(v, hi, lo);
    static_cast<__half*>(planes[0])[idx] = hi;
    static_cast<__half*>(planes[1])[idx] = lo;
  } else {
    uint32_t hi;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(v));
    const float fh = __uint_as_float(hi);
    static_cast<float*>(planes[0])[idx] = fh;
    static_cast<float*>(planes[1])[idx] = v - fh;
  }
}

// Activations (the reference's definitions: sigmoid = 1/(1+exp(-x)), cells.hpp:30; tanh).
// bf16 mode: the SFU approximations (relative error ~2^-11, far below the bf16 operand rounding
// it already carries). fp32-parity mode: MUFU.EX2 + MUFU.RCP with a Newton step and a polynomial
// for |tanh| below 0.6 (common.cuh sigmoid_fast / tanh_fast, a few fp32 ulps from expf / tanhf):
// libm's expf, IEEE division and tanhf cost ~150 instructions per cell element and were half the
// cluster forward's cell phase (2.7 -> 1.3 us, profiles/r02/README.md). An earlier attempt kept
// both paths in one binary and measured no gain -- the code size hid it. tanh(x) = 1 - 2/(1+e^2x)
// without the small-|x| branch breaks the 1e-5 contract (2e-5 normwise).
template <class P>
__device__ __forceinline__ float act_sigmoid(float x) {
  if constexpr (P::kPlanes == 1) {
    // sigma(x) = 0.5 + 0.5 tanh(x/2): one MUFU.TANH instead of EX2 + RCP
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(0.5f * x));
    return fmaf(0.5f, y, 0.5f);
  } else {
    return sigmoid_fast(x);
  }
}
template <class P>
__device__ __forceinline__ float act_tanh(float x) {
  if constexpr (P::kPlanes == 1) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  } else {
    return tanh_fast(x);
  }
}

// Counters are cumulative over passes (targets = epoch x per-pass count, all mod 2^32), so
// "reached" is the wrap-safe signed distance, never a plain unsigned >=: after 2^32 arrivals the
// counter restarts near 0 while the target is still large (or the target wraps first).
__device__ __forceinline__ bool flag_reached(uint32_t v, uint32_t target) { return (int32_t)(v - target) >= 0; }

// Spin until *flag reaches target (gpu-scope acquire), bounded by a timeout that records an
// error instead of hanging the device. `code` identifies the wait for the host message.
// the timed back-off of wait_flag, out of line (as mbar_wait_slow): only long waits get here
static __device__ __noinline__ void wait_flag_slow(const uint32_t* flag, uint32_t target, int* error,
                                                   unsigned long long timeout_ns, int code) {
  const uint64_t t0 = globaltimer();
  uint32_t ns = 32;
#pragma unroll 1
  while (!flag_reached(ld_relaxed_gpu(flag), target)) {
    nanosleep(ns);
    if (ns < 128) ns <<= 1;
    if (globaltimer() - t0 > timeout_ns) {
      atomicCAS(error, 0, code);
      atomicMax(error + 1, (int)ld_relaxed_gpu(flag));
      return;
    }
  }
}
__device__ __forceinline__ void wait_flag(const uint32_t* flag, uint32_t target, int* error,
                                          unsigned long long timeout_ns, int code) {
  // Poll with relaxed loads (an acquire load per iteration would invalidate the SM's L1 each
  // time, CCTL.IVALL, slowing every other warp on the SM); one acquire once satisfied.
  bool ok = flag_reached(ld_relaxed_gpu(flag), target);
#pragma unroll 1
  for (int i = 0; i < 65536 && !ok; ++i) ok = flag_reached(ld_relaxed_gpu(flag), target);
  if (!ok) wait_flag_slow(flag, target, error, timeout_ns, code);
  (void)ld_acquire_gpu(flag);
}
__device__ __forceinline__ void wait_flag(const uint32_t* flag, uint32_t target,
                                          const RecParams& p, int code) {
  wait_flag(flag, target, p.error, p.timeout_ns, code);
}
// Flag operations at gpu or system scope (system: the counter is shared with a peer GPU).
__device__ __forceinline__ uint32_t ld_relaxed_s(const uint32_t* p, bool sys) {
  uint32_t v;
  if (sys)
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_flag_s(const uint32_t* flag, uint32_t target, bool sys, int* error,
                                            unsigned long long timeout_ns, int code) {
  if (!sys) {
    wait_flag(flag, target, error, timeout_ns, code);
    return;
  }
  const uint64_t t0 = globaltimer();
#pragma unroll 1
  while (!flag_reached(ld_relaxed_s(flag, true), target)) {
    if (globaltimer() - t0 > timeout_ns) {
      atomicCAS(error, 0, code);
      atomicMax(error + 1, (int)ld_relaxed_s(flag, true));
      return;
    }
  }
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
}
__device__ __forceinline__ void red_release_s(uint32_t* p, uint32_t v, bool sys) {
  if (sys)
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else
    red_release_gpu_add(p, v);
}
__device__ __forceinline__ void red_relaxed_s(uint32_t* p, uint32_t v, bool sys) {
  if (sys)
    asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else
    red_relaxed_gpu_add(p, v);
}
// error code: 1<<30 | dir<<28 | layer<<20 | (t+2)<<4 | which
__device__ __forceinline__ int wait_code(int dir, int l, int t, int which) {
  return (1 << 30) | (dir << 28) | (l << 20) | ((t + 2) << 4) | which;
}

__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase), "r"(kSuspendHintNs)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
#pragma unroll 1
  while (!mbar_try_wait_cluster(bar, phase)) {
  }
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* local_bar, uint32_t rank) {
  const uint32_t remote = map_dsmem(smem_u32(local_bar), rank);
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void st_dsmem_f32(uint32_t cluster_addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(cluster_addr), "f"(v));
}

__device__ __forceinline__ float lds_f32(const float* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ float lds_f32_at(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f32(float* p, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(smem_u32(p)), "f"(v));
}
__device__ __forceinline__ void sts_bf16(uint32_t a, float v) {
  const __nv_bfloat16 b = __float2bfloat16_rn(v);
  asm volatile("st.shared.b16 [%0], %1;" ::"r"(a), "h"(*reinterpret_cast<const uint16_t*>(&b)));
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// Sum of `n` TMEM accumulators (N columns apart) for 8 columns of this thread's lane, in fp32
// with round-to-nearest adds (n == 0 -> zeros: no k-block of this CTA was active).
__device__ __forceinline__ void load_acc_sum(uint32_t taddr, int N, int n, float (&a)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 0.0f;
  for (int i = 0; i < n; ++i) {
    uint32_t v[8];
    tmem_ld_32x32b_x8(taddr + i * N, v);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = i == 0 ? __uint_as_float(v[j]) : a[j] + __uint_as_float(v[j]);
  }
}

// Shared-memory carve-up common to both directions.
struct RecSmem {
  uint8_t* a_res;      // resident A k-blocks (or A stages when streamed)
  uint8_t* b_st;       // B stages
  float* xr;           // receive buffer [ksplit][kXChunk/ksplit][128] of partial columns
  uint64_t* full;
  uint64_t* empty;
  uint64_t* a_full;
  uint64_t* tmem_full;
  uint64_t* tmem_empty;
  uint64_t* xready;
  uint64_t* xfree;
  uint64_t* pfull;   // [kMaxPromoSlots] promotion ring: chunk accumulated (MMA commit)
  uint64_t* pempty;  // [kMaxPromoSlots] chunk drained into the sum (kEpiThreads arrivals)
  uint32_t* tmem_slot;
};
constexpr int kMaxPromoSlots = 8;
__device__ __forceinline__ uint64_t* acc_bar(int b, uint64_t* b0, uint64_t* b1) { return b ? b1 : b0; }

__device__ __forceinline__ RecSmem carve(uint8_t* smem, int a_bytes_total, int b_stage_bytes,
                                         int stages) {
  RecSmem s;
  s.a_res = smem;
  s.b_st = smem + a_bytes_total;
  s.xr = reinterpret_cast<float*>(s.b_st + stages * b_stage_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(s.xr + kXChunk * kTileM);
  s.full = bars;
  s.empty = bars + stages;
  s.a_full = bars + 2 * stages;
  s.tmem_full = s.a_full + 1;
  s.tmem_empty = s.a_full + 2;
  s.xready = s.a_full + 3;
  s.xfree = s.a_full + 4;
  s.pfull = s.a_full + 5;
  s.pempty = s.pfull + kMaxPromoSlots;
  s.tmem_slot = reinterpret_cast<uint32_t*>(s.pempty + kMaxPromoSlots);
  return s;
}

// Host-side mirror of the carve-up size.
inline size_t rec_smem_bytes(int planes, int a_kblocks_resident_or_stages, int n, int stages) {
  const size_t a = size_t(a_kblocks_resident_or_stages) * planes * kTileM * kRowBytes;
  const size_t b = size_t(stages) * planes * n * kRowBytes;
  const size_t x = size_t(kXChunk) * kTileM * 4;
  const size_t bars = (2 * stages + 6 + 2 * kMaxPromoSlots) * 8 + 16;
  return 1024 + a + b + x + bars;
}

// ---- split-K exchange of one column chunk (xc counts exchanges: mbarrier phase parity) ----
// 1. wait until every rank finished reading the previous chunk (xfree), 2. push partial
// columns into their owners' receive buffers, 3. publish (bar + release-arrive on all
// ranks), 4. wait for all ranks' pushes (acquire). After reducing: release (xfree).
__device__ __forceinline__ void xchg_wait_free(const RecSmem& s, int ks, uint32_t xc) {
  if (ks > 1 && xc > 0) mbar_wait_cluster(s.xfree, (xc - 1) & 1);
}
// Thread (quarter q, lane) pushes the 8 columns c0..c0+7 of its accumulator row.
// inv = ceil(2^16 / nco): (c * inv) >> 16 == c / nco exactly for c < 64 (no integer divide).
__device__ __forceinline__ void xchg_push8(const RecSmem& s, int ks, int rank, int nco, int q,
                                           int lane, int c0, const float (&a)[8], uint32_t inv) {
  const int row = q * 32 + lane;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = c0 + j;
    const int owner = (int)((uint32_t(c) * inv) >> 16);
    float* dst = s.xr + ((rank * nco) + (c - owner * nco)) * kTileM + row;
    if (owner == rank)
      sts_f32(dst, a[j]);
    else
      st_dsmem_f32(map_dsmem(smem_u32(dst), owner), a[j]);
  }
}
__device__ __forceinline__ void xchg_publish(const RecSmem& s, int ks, uint32_t xc) {
  named_bar_sync(1, kEpiThreads);
  if (ks > 1) {
    if (threadIdx.x == kEpiBase) {
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      for (int r = 0; r < ks; ++r) mbar_arrive_remote(s.xready, r);
    }
    mbar_wait_cluster(s.xready, xc & 1);
  }
}
__device__ __forceinline__ void xchg_release(const RecSmem& s, int ks) {
  named_bar_sync(1, kEpiThreads);
  if (ks > 1 && threadIdx.x == kEpiBase) {
    for (int r = 0; r < ks; ++r) mbar_arrive_remote(s.xfree, r);
  }
}
// Reduced accumulator value of owned column cl, row `row` (fixed rank order).
// Not unrolled over ranks: the cell loop inlines this 4 x 8 times per chunk, and an unrolled
// runtime-trip-count loop there grew the forward kernel to 15.6k instructions; the epilogue then
// stalled on instruction fetch (ncu stall_no_inst 80 % of its samples, config E).
__device__ __forceinline__ float xchg_sum(const RecSmem& s, int ks, int nco, int cl, int row) {
  const uint32_t a = smem_u32(s.xr) + (uint32_t)(cl * kTileM + row) * 4u;
  float acc = lds_f32_at(a);
#pragma unroll 1
  for (int r = 1; r < ks; ++r) acc += lds_f32_at(a + (uint32_t)(r * nco * kTileM) * 4u);
  return acc;
}

// Common prologue: barriers, TMEM allocation, cluster rendezvous.
__device__ __forceinline__ uint32_t rec_setup(const RecSmem& S, const RecParams& p, int ks,
                                              uint32_t tmem_cols) {
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], 1);
    }
    mbar_init(S.a_full, 1);
    mbar_init(S.tmem_full, 1);
    mbar_init(S.tmem_empty, kEpiThreads);
    mbar_init(S.xready, ks);
    mbar_init(S.xfree, ks);
    for (int i = 0; i < kMaxPromoSlots; ++i) {
      mbar_init(&S.pfull[i], 1);
      mbar_init(&S.pempty[i], kEpiThreads);
    }
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
  if (ks > 1) cluster_sync();  // peers' barriers initialised before any remote arrive
  tc_fence_after();
  return *S.tmem_slot;
}

// CTA-pair prologue / epilogue (cta_group::2 TMEM allocation in both CTAs of the pair).
__device__ __forceinline__ uint32_t rec_setup_pair(const RecSmem& S, const RecParams& p, uint32_t tmem_cols,
                                                   int tmem_empty_count = kEpiThreads) {
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], 1);
    }
    mbar_init(S.a_full, 1);
    mbar_init(S.tmem_full, 1);
    mbar_init(S.tmem_empty, tmem_empty_count);
    mbar_init(S.pfull, 1);                       // second accumulator buffer (k_lstm_bwd pair)
    mbar_init(S.pempty, tmem_empty_count);
    mbar_init(S.xready, 1);
    mbar_init(S.xfree, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(S.tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers initialised before any load completes on them
  tc_fence_after();
  return *S.tmem_slot;
}
__device__ __forceinline__ void rec_teardown_pair(uint32_t tmem_base, uint32_t tmem_cols) {
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if ((threadIdx.x >> 5) == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}

__device__ __forceinline__ void rec_teardown(int ks, uint32_t tmem_base, uint32_t tmem_cols) {
  tc_fence_before();
  __syncthreads();
  if (ks > 1) cluster_sync();  // no CTA leaves while peers may still write its smem
  if ((threadIdx.x >> 5) == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
  }
}

// ---- 3xTF32 promotion ring (RecParams::promo). The tensor core's fp32 accumulation loses
// ~2^-27 of the running sum per MMA (measured: 5e-5 relative after K = 6400; at config C2048 the
// backward's K = 16384 chains missed the 1e-5 contract by 2.5x), so long K ranges are cut into
// chunks of acc_kb k-blocks, each accumulated into one of n_acc ring slots of TMEM while the
// epilogue adds the previous chunk into an fp32 sum region (tcgen05.ld / add / tcgen05.st, fixed
// order: deterministic). Slot handshake: pfull (MMA commit) / pempty (kEpiThreads arrivals).
// Each thread touches only the TMEM cells it later reads in the step's final drain (its lane
// row, its half of every kXChunk column chunk), so no cross-thread ordering is needed.
// `nc0` chunks of K segment 0 come first, then segment 1's; a chunk's product is scaled by `sc0` /
// `sc1` (fp16x2 operand scales, exact powers of two) as it is added.
__device__ __forceinline__ void promo_drain(const RecSmem& S, const RecParams& p, uint32_t tmem_base, int N,
                                            int nchunks, uint32_t& ech, int nc0 = 0, float sc0 = 1.0f,
                                            float sc1 = 1.0f) {
  const int warp = threadIdx.x >> 5, q = warp & 3, half = (warp - 4) >> 2;
  const uint32_t lane_off = uint32_t(q * 32) << 16;
  for (int c = 0; c < nchunks; ++c, ++ech) {
    const uint32_t slot = ech % (uint32_t)p.n_acc;
    const float sc = c < nc0 ? sc0 : sc1;
    mbar_wait(&S.pfull[slot], (ech / (uint32_t)p.n_acc) & 1);
    tc_fence_after();
    const uint32_t src = tmem_base + lane_off + (1 + slot) * N, dst = tmem_base + lane_off;
    for (int n0 = 0; n0 < N; n0 += kXChunk) {
      const int nc = min(kXChunk, N - n0);
      for (int c0 = n0 + half * (nc >> 1); c0 < n0 + (half + 1) * (nc >> 1); c0 += 8) {
        uint32_t v[8], w[8];
        tmem_ld_32x32b_x8(src + c0, v);
        if (c > 0) tmem_ld_32x32b_x8(dst + c0, w);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float x = __uint_as_float(v[j]) * sc;
          v[j] = __float_as_uint(c > 0 ? __uint_as_float(w[j]) + x : x);
        }
        tmem_st_32x32b_x8(dst + c0, v);
      }
    }
    tmem_st_wait();
    tc_fence_before();
    mbar_arrive(&S.pempty[slot]);
  }
}
// MMA side of the ring: the slot accumulator of chunk `ch` (waits for it to be drained when the
// k-block about to be issued starts the chunk).
__device__ __forceinline__ uint32_t promo_slot(const RecSmem& S, const RecParams& p, uint32_t tmem_base, int N,
                                               bool start, uint32_t ch) {
  const uint32_t slot = ch % (uint32_t)p.n_acc;
  if (start && ch >= (uint32_t)p.n_acc) {
    mbar_wait(&S.pempty[slot], ((ch / (uint32_t)p.n_acc) - 1) & 1);
    tc_fence_after();
  }
  return tmem_base + (1 + slot) * N;
}

// MMA issue of one k-block (all kk substeps, all precision combos) into accumulator acc.
template <class P>
__device__ __forceinline__ void mma_kblock(uint32_t acc, uint32_t a_base, uint32_t b_base,
                                           int a_bytes, int b_bytes, uint32_t idesc,
                                           bool fresh) {
  const uint64_t a0 = sdesc_sw128(a_base, 16, 1024), b0 = sdesc_sw128(b_base, 16, 1024);
#pragma unroll
  for (int kk = 0; kk < P::kAtomK / P::kUmmaK; ++kk) {
#pragma unroll
    for (int c = 0; c < P::kCombos; ++c) {
      const int pa = (c == 2) ? 1 : 0, pb = (c == 1) ? 1 : 0;
      const uint64_t ad = desc_add(a0, pa * a_bytes + kk * P::kUmmaK * P::kElem);
      const uint64_t bd = desc_add(b0, pb * b_bytes + kk * P::kUmmaK * P::kElem);
      umma_warp<P::kTF32>(acc, ad, bd, idesc, (!fresh || kk | c) ? 1u : 0u);
    }
  }
}

// ====================================================================== forward kernel
// kPair (bf16, stepwise, ksplit 1): the CTAs of a cluster pair (tiles 2i, 2i+1) run
// tcgen05.mma.cta_group::2 with M = 256; each CTA loads its own 128 A rows and half of the B
// columns (Bp/2), so per SM a k-block moves 16 + Bp*64 bytes instead of 16K + Bp*128 -- the
// per-SM operand ingress that bounds the step at large Bp (config E: 3 MB per CTA per step).
template <class P, bool kPair = false, int kKind = kCellLstm>
__global__ void __launch_bounds__(kRecThreads, 1)
    k_lstm_fwd(const FwdLayer* __restrict__ layers, RecParams p) {
  const int l = p.layer_base + blockIdx.y;
  // The descriptor is read after every barrier; keep it in shared memory (global reloads
  // would go to L2 because cluster/gpu-scope acquires invalidate L1).
  __shared__ FwdLayer Ly;
  __shared__ const uint32_t* x_flags;
  if (threadIdx.x == 0) {
    Ly = layers[l];
    x_flags = l > 0 ? layers[l - 1].flags : nullptr;
    set_wait_error(p.error);
  }
  __syncthreads();
  const int ks = p.ksplit;
  const int rank = (int)(blockIdx.x % ks);
  const int tile = (int)(blockIdx.x / ks);
  const int N = p.Bp;
  const bool zxm = Ly.zx != nullptr;
  const int akofs = zxm ? Ly.Ipl / P::kAtomK : 0;  // A k-block of R (after W) in [W|R]
  const int nkb0 = zxm ? 0 : Ly.Ipl / P::kAtomK;
  const int nkb = nkb0 + p.Hp / P::kAtomK;
  const int kb_lo = rank * nkb / ks, kb_hi = (rank + 1) * nkb / ks;
  const int my_nkb = kb_hi - kb_lo;
  const int a_bytes = kTileM * kRowBytes;           // one plane of one k-block
  const int b_bytes = (kPair ? N / 2 : N) * kRowBytes;
  const int b_stage = P::kPlanes * b_bytes;
  const int a_stage = P::kPlanes * a_bytes;
  const int a_total = p.resident ? p.a_slots * a_stage : p.stages * a_stage;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const RecSmem S = carve(smem, a_total, b_stage, p.stages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // persistent, one accumulator per step (no promotion): two accumulator buffers, so step t's
  // W.x half runs while the epilogue still drains step t-1 (as k_lstm_bwd)
  const bool dbuf = p.acc_dbuf && !kPair && p.persistent && p.n_acc == 1 && !p.promo && 2 * N <= 512;
  // accumulator buffer 1's barriers (selected with acc_bar, not a dynamically indexed array,
  // which would live on the stack)
  uint64_t* const tfull1 = dbuf ? S.pfull : S.tmem_full;
  uint64_t* const tempty1 = dbuf ? S.pempty : S.tmem_empty;
  uint32_t tmem_cols = 32;
  while (tmem_cols < (uint32_t)(N * (dbuf ? 2 : p.n_acc + p.promo))) tmem_cols <<= 1;
  const uint32_t tmem_base = kPair ? rec_setup_pair(S, p, tmem_cols) : rec_setup(S, p, ks, tmem_cols);
  const int row0 = tile * kTileM;

  if (kPair && warp <= 1) {
   if constexpr (kPair) {
    const uint32_t prank = cluster_ctarank() & 1;
    const int nh = N / 2;
    if (warp == 0 && lane == 0) {
      // ============= TMA producer (both CTAs of the pair; completion on the leader's barrier)
      prefetch_tmap(Ly.a[0]);
      prefetch_tmap(Ly.bx2);
      prefetch_tmap(Ly.bh2);
      const int t = p.t_first;
      if (l == 0 && p.pp_in_flags) {  // pipeline stage: h_t of the previous stage
        wait_flag_s(&p.pp_in_flags[t], pp_target(p), true, p.error, p.timeout_ns, wait_code(0, l, t, 1));
        fence_proxy_async_global();
      }
      uint32_t pc = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++pc) {
        const int s = pc % p.stages;
        mbar_wait(&S.empty[s], ((pc / p.stages) & 1) ^ 1);
        if (prank == 0) mbar_arrive_expect_tx(&S.full[s], 2 * (b_stage + a_stage));
        uint8_t* bst = S.b_st + s * b_stage;
        if (kb < nkb0)
          g2::tma_load_2d_pair(bst, Ly.bx2, &S.full[s], kb * P::kAtomK, Ly.bx_col_off + t * p.Bp + (int)prank * nh);
        else
          g2::tma_load_2d_pair(bst, Ly.bh2, &S.full[s], (kb - nkb0) * P::kAtomK, t * p.Bp + (int)prank * nh);
        g2::tma_load_2d_pair(S.a_res + s * a_stage, Ly.a[0], &S.full[s], (kb + akofs) * P::kAtomK, row0);
      }
    } else if (warp == 1 && prank == 0) {
      // ============= MMA issuer (leader, converged warp): M = 256 over the pair, N = Bp
      const uint32_t idesc = idesc_make(P::kFmt, false, false, 2 * kTileM, N);
      uint32_t pc = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++pc) {
        const int s = pc % p.stages;
        mbar_wait(&S.full[s], (pc / p.stages) & 1);
        tc_fence_after();
        const uint64_t a0 = sdesc_sw128(smem_u32(S.a_res + s * a_stage), 16, 1024);
        const uint64_t b0 = sdesc_sw128(smem_u32(S.b_st + s * b_stage), 16, 1024);
#pragma unroll
        for (int kk = 0; kk < P::kAtomK / P::kUmmaK; ++kk)
          g2::umma2_warp(tmem_base, desc_add(a0, kk * 32), desc_add(b0, kk * 32), idesc,
                         (kb != kb_lo || kk) ? 1u : 0u);
        g2::commit2_warp(&S.empty[s]);
      }
      g2::commit2_warp(S.tmem_full);
    }
   }
  } else if (!kPair && warp == 0 && lane == 0) {
    // ================= TMA producer
    for (int pl = 0; pl < P::kPlanes; ++pl) {
      prefetch_tmap(Ly.a[pl]);
      prefetch_tmap(Ly.bx[pl]);
      prefetch_tmap(Ly.bh[pl]);
    }
    if (p.resident) {
      mbar_arrive_expect_tx(S.a_full, my_nkb * a_stage);
      for (int kb = kb_lo; kb < kb_hi; ++kb)
        for (int pl = 0; pl < P::kPlanes; ++pl)
          tma_load_2d(S.a_res + (kb - kb_lo) * a_stage + pl * a_bytes, Ly.a[pl], S.a_full,
                      (kb + akofs) * P::kAtomK, row0);
    }
    uint32_t pc = 0;
    for (int it = 0; it < p.n_steps; ++it) {
      const int t = p.t_first + it;
      progress(p, 0, it, 1);
      trace_stamp(p, it, 0);
      bool x_ready = false, h_ready = false;
      // streamed weights: pull the k-blocks a_prefetch ahead from HBM into L2 (the TMA loads
      // behind them then hit L2; the stage ring alone keeps too few bytes in flight)
      if (!p.resident)
        for (int kp = kb_lo; kp < min(kb_hi, kb_lo + p.a_prefetch); ++kp)
          for (int pl = 0; pl < P::kPlanes; ++pl) tma_prefetch_2d(Ly.a[pl], (kp + akofs) * P::kAtomK, row0);
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++pc) {
        const bool seg0 = kb < nkb0;
        if (!p.resident && kb + p.a_prefetch < kb_hi && p.a_prefetch > 0)
          for (int pl = 0; pl < P::kPlanes; ++pl)
            tma_prefetch_2d(Ly.a[pl], (kb + p.a_prefetch + akofs) * P::kAtomK, row0);
        if (seg0 && !x_ready && l == 0 && p.pp_in_flags) {  // pipeline stage (any schedule)
          wait_flag_s(&p.pp_in_flags[t], pp_target(p), true, p.error, p.timeout_ns, wait_code(0, l, t, 1));
          fence_proxy_async_global();
          x_ready = true;
        }
        if (p.persistent) {
          if (seg0 && !x_ready) {
            progress(p, 0, it, 2);
            if (l > 0) wait_flag(&x_flags[t], p.flag_target, p, wait_code(0, l, t, 1));
            fence_proxy_async_global();
            x_ready = true;
          }
          if (!seg0 && !h_ready) {
            progress(p, 0, it, 3);
            if (t > 0) wait_flag(&Ly.flags[t - 1], p.flag_target, p, wait_code(0, l, t, 2));
            fence_proxy_async_global();
            h_ready = true;
          }
        }
        const int s = pc % p.stages;
        mbar_wait(&S.empty[s], ((pc / p.stages) & 1) ^ 1);
        mbar_arrive_expect_tx(&S.full[s], b_stage + (p.resident ? 0 : a_stage));
        uint8_t* bst = S.b_st + s * b_stage;
        for (int pl = 0; pl < P::kPlanes; ++pl) {
          if (seg0)
            tma_load_2d(bst + pl * b_bytes, Ly.bx[pl], &S.full[s], kb * P::kAtomK,
                        Ly.bx_col_off + t * p.Bp);
          else
            tma_load_2d(bst + pl * b_bytes, Ly.bh[pl], &S.full[s], (kb - nkb0) * P::kAtomK,
                        t * p.Bp);
          if (!p.resident)
            tma_load_2d(S.a_res + s * a_stage + pl * a_bytes, Ly.a[pl], &S.full[s],
                        (kb + akofs) * P::kAtomK, row0);
        }
      }
      trace_stamp(p, it, 1);
    }
  } else if (!kPair && warp == 1) {
    // whole warp 1 (converged; elect.sync inside each MMA / commit): a lane-0-only issue branch
    // costs an ELECT / R2UR waterfall per instruction (profiles/ubench/mma_ubench.cu)
    // ================= MMA issuer
    const uint32_t idesc = idesc_make(P::kFmt, false, false, kTileM, N);
    if (p.resident) mbar_wait(S.a_full, 0);
    tc_fence_after();
    uint32_t pc = 0, ch = 0;
    const int s0_hi = min(kb_hi, nkb0);  // this CTA's K segment 0 (W.x) is [kb_lo, s0_hi)
    for (int it = 0; it < p.n_steps; ++it) {
      progress(p, 1, it, 1);
      const int ab = dbuf ? (it & 1) : 0;  // accumulator buffer (not "bi": the bias below)
      const int use = dbuf ? (it >> 1) : it;  // earlier steps that used buffer ab
      if (use > 0 && !p.promo) {
        mbar_wait(acc_bar(ab, S.tmem_empty, tempty1), (use - 1) & 1);
        tc_fence_after();
      }
      progress(p, 1, it, 2);
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++pc) {
        const int s = pc % p.stages;
        const int nact = kb - kb_lo;
        // promotion chunks restart at the segment boundary (their products carry different scales)
        const int iseg = kb < nkb0 ? kb - kb_lo : kb - max(kb_lo, nkb0);
        const int nseg = kb < nkb0 ? s0_hi - kb_lo : kb_hi - max(kb_lo, nkb0);
        const bool cstart = p.promo ? iseg % p.acc_kb == 0 : nact % p.acc_kb == 0;
        const uint32_t acc = p.promo ? promo_slot(S, p, tmem_base, N, cstart, ch)
                                     : tmem_base + (uint32_t)(ab * N) + (nact / p.acc_kb) * N;
        mbar_wait(&S.full[s], (pc / p.stages) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(S.a_res + (p.resident ? (kb - kb_lo) : s) * a_stage);
        const uint32_t b_base = smem_u32(S.b_st + s * b_stage);
        mma_kblock<P>(acc, a_base, b_base, a_bytes, b_bytes, idesc, cstart);
        umma_commit_warp(&S.empty[s]);
        if (p.promo && ((iseg + 1) % p.acc_kb == 0 || iseg + 1 == nseg)) {
          umma_commit_warp(&S.pfull[ch % (uint32_t)p.n_acc]);
          ++ch;
        }
      }
      if (!p.promo) umma_commit_warp(acc_bar(ab, S.tmem_full, tfull1));
    }
  } else if (warp >= 4) {
    // ================= epilogue: split-K exchange + LSTM cell (cells.hpp:227-260)
    // register copy of the descriptor: through the shared-memory one, every global store
    // (a generic pointer that may alias it) forces a reload of the next pointer
    const FwdLayer Le = Ly;
    const int et = threadIdx.x - kEpiBase;  // 0..255
    const int q = warp & 3;                 // TMEM lane quarter == gate
    const int half = (warp - 4) >> 2;       // which half of the chunk's columns to drain
    const int j = et & 31;                  // unit within tile (cell phase)
    const int cg = et >> 5;                 // column group 0..7 (cell phase)
    const int u = tile * kUnitsPerFwdTile + j;
    const long long Hp = p.Hp, G4 = 4 * Hp;
    const float bi = Le.bias[u], bf = Le.bias[Hp + u], bo = Le.bias[2 * Hp + u],
                bc = Le.bias[3 * Hp + u];
    const int n_s0 = max(0, min(kb_hi, nkb0) - kb_lo), n_s1 = my_nkb - n_s0;  // k-blocks per K segment
    const int nc0 = (n_s0 + p.acc_kb - 1) / p.acc_kb;
    const int n_chunks = kPair ? 1 : p.promo ? nc0 + (n_s1 + p.acc_kb - 1) / p.acc_kb : (my_nkb + p.acc_kb - 1) / p.acc_kb;
    const int n_used = p.promo ? (n_chunks > 0 ? 1 : 0) : n_chunks;
    const float sc0 = l == 0 ? p.us_in0 : p.us_in;
    uint32_t xc = 0, ech = 0;
    for (int it = 0; it < p.n_steps; ++it) {
      const int t = p.t_first + it;
      if (et == 0) progress(p, 2, it, 1);
      const int ab = dbuf ? (it & 1) : 0;  // accumulator buffer (bi is the input-gate bias)
      const uint32_t tacc = tmem_base + (uint32_t)(ab * N);
      if (!kPair && p.promo) {  // (the CTA-pair kernel never promotes: keep it out of its code)
        promo_drain(S, p, tmem_base, N, n_chunks, ech, nc0, sc0, p.us_rec);
      } else {
        mbar_wait(acc_bar(ab, S.tmem_full, tfull1), (dbuf ? (it >> 1) : it) & 1);
        tc_fence_after();
      }
      if (et == 0) trace_stamp(p, it, 2);
      for (int n0 = 0; n0 < N; n0 += kXChunk, ++xc) {
        const int nc = min(kXChunk, N - n0);
        const int nco = nc / ks;  // columns of this chunk owned by each rank
        const uint32_t inv = (65536u + nco - 1) / nco;
        xchg_wait_free(S, ks, xc);
        for (int c0 = half * (nc >> 1); c0 < (half + 1) * (nc >> 1); c0 += 8) {
          float a[8];
          load_acc_sum(tacc + (uint32_t(q * 32) << 16) + n0 + c0, N, n_used, a);
          xchg_push8(S, ks, rank, nco, q, lane, c0, a, inv);
        }
        if (n0 + kXChunk >= N && (kPair || !p.promo)) {
          tc_fence_before();
          mbar_arrive(acc_bar(ab, S.tmem_empty, tempty1));
        }
        if (et == 0 && n0 == 0) trace_stamp(p, it, 3);
        xchg_publish(S, ks, xc);
        if (et == 0 && n0 == 0) trace_stamp(p, it, 4);
        // cell phase: owned columns cl = cg + 8k, unit j; loads first, then math
        float cp[8];  // LSTM: c_{t-1}; GRU: h_{t-1} (the direct term u h_{t-1}); RNN: unused
        const long long colb = (long long)t * p.Bp + n0 + rank * nco;  // block t, owned base
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int cl = cg + 8 * k;
          const float* st = kKind == kCellGru ? Le.h : Le.c;
          cp[k] = (cl < nco && kKind != kCellRnnTanh) ? st[(colb + cl) * Hp + u] : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int cl = cg + 8 * k;
          if (cl >= nco) break;
          float zi = 0.0f, zf = 0.0f, zo = 0.0f, zc = 0.0f;
          if (zxm) {  // (zw + zr) + b, cells.hpp:240
            const float* zp = Le.zx + (colb + cl) * G4 + u;
            zi = zp[0];
            zf = zp[Hp];
            zo = zp[2 * Hp];
            zc = zp[3 * Hp];
          }
          const float si = xchg_sum(S, ks, nco, cl, 0 * 32 + j), sf = xchg_sum(S, ks, nco, cl, 1 * 32 + j);
          const float so = xchg_sum(S, ks, nco, cl, 2 * 32 + j), sc = xchg_sum(S, ks, nco, cl, 3 * 32 + j);
          const long long col_prev = colb + cl;       // block t   (c_{t-1})
          const long long col_new = col_prev + p.Bp;  // block t+1 (c_t, h_t)
          float hv;
          if constexpr (kKind == kCellLstm) {
            const float ai = (zxm ? zi + si : si) + bi;
            const float af = (zxm ? zf + sf : sf) + bf;
            const float ao = (zxm ? zo + so : so) + bo;
            const float ac = (zxm ? zc + sc : sc) + bc;
            const float iv = act_sigmoid<P>(ai);
            const float fv = act_sigmoid<P>(af);
            const float ov = act_sigmoid<P>(ao);
            const float cb = act_tanh<P>(ac);
            const float t1 = fv * cp[k];
            const float t2 = iv * cb;
            const float cv = t1 + t2;
            const float tcv = act_tanh<P>(cv);
            hv = ov * tcv;
            Le.c[col_new * Hp + u] = cv;
            if (Le.gates) {
              float* gp = Le.gates + col_prev * G4 + u;
              gp[0] = iv;
              gp[Hp] = fv;
              gp[2 * Hp] = ov;
              gp[3 * Hp] = cb;
              Le.tanhc[col_prev * Hp + u] = tcv;
            }
          } else if constexpr (kKind == kCellGru) {
            // cells.hpp:294-313; the forward image keeps W_n x in slot 2 and R_n h in slot 3
            // (layout_kernels.cuh k_repack), so the K-summed accumulator holds both apart
            const float ar = (zxm ? zi + si : si) + bi;
            const float au = (zxm ? zf + sf : sf) + bf;
            const float zwn = zxm ? zo + so : so;
            const float zrn = zxm ? zc + sc : sc;
            const float rv = act_sigmoid<P>(ar);
            const float uv = act_sigmoid<P>(au);
            const float t1 = zwn + bo;  // W_n x + b_n
            const float t2 = rv * zrn;
            const float nv = act_tanh<P>(t1 + t2);
            const float t3 = uv * cp[k];
            const float om = 1.0f - uv;
            const float t4 = om * nv;
            hv = t3 + t4;
            if (Le.gates) {
              float* gp = Le.gates + col_prev * G4 + u;
              gp[0] = rv;
              gp[Hp] = uv;
              gp[2 * Hp] = nv;
              Le.zrh[col_prev * Hp + u] = zrn;
            }
          } else {  // RNN (cells.hpp:200-212)
            const float a = (zxm ? zi + si : si) + bi;
            hv = p.kind == kCellRnnRelu ? (a > 0.0f ? a : 0.0f) : act_tanh<P>(a);
          }
          Le.h[col_new * Hp + u] = hv;
          store_operand<P>(Le.hop, col_new * Hp + u, kF16Ops<P> ? hv * pow2f(kHScaleLog2) : hv);
          if (Le.xop_peer[0] && u < Le.peer_ld)  // pipeline: the next stage's layer input, block t
            store_operand<P>(Le.xop_peer, col_prev * Le.peer_ld + u, kF16Ops<P> ? hv * pow2f(kHScaleLog2) : hv);
        }
        if (et == 0 && n0 == 0) trace_stamp(p, it, 5);
        xchg_release(S, ks);
        if (et == 0 && n0 == 0) trace_stamp(p, it, 6);
      }
      if (p.persistent) {
        // publish step t: writers order their generic stores before later async-proxy (TMA)
        // reads, the CTA barrier collects them, one thread releases at gpu scope
        fence_proxy_async_global();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          __threadfence();
          red_release_gpu_add(&Le.flags[t], 1);
        }
      }
      if (Le.xop_peer[0]) {  // pipeline: publish h_t to the next stage (system scope)
        if (!p.persistent) {
          fence_proxy_async_global();
          named_bar_sync(1, kEpiThreads);
        }
        if (et == 0) {
          __threadfence_system();
          red_release_s(Le.peer_flags + t, 1, true);
        }
      }
      if (et == 0) trace_stamp(p, it, 7);
    }
  }
  if constexpr (kPair)
    rec_teardown_pair(tmem_base, tmem_cols);
  else
    rec_teardown(ks, tmem_base, tmem_cols);
}

// ====================================================================== backward kernel
// kPair (bf16, ksplit 1, streamed A): CTA pairs as in k_lstm_fwd<_, true>; the leader's
// tmem_empty barrier collects one arrival per CTA before the next step's MMAs overwrite either
// CTA's accumulator.
template <class P, bool kPair = false, int kKind = kCellLstm>
__global__ void __launch_bounds__(kRecThreads, 1)
    k_lstm_bwd(const BwdLayer* __restrict__ layers, RecParams p) {
  const int l = p.layer_base + blockIdx.y;
  __shared__ BwdLayer Ly;
  __shared__ const uint32_t* up_flags;
  if (threadIdx.x == 0) {
    Ly = layers[l];
    up_flags = Ly.has_up && l + 1 < p.L ? layers[l + 1].flags : nullptr;  // top + pipeline: pp_in_flags
    set_wait_error(p.error);
  }
  __syncthreads();
  const int ks = p.ksplit;
  const int rank = (int)(blockIdx.x % ks);
  const int tile = (int)(blockIdx.x / ks);
  const int N = p.Bp;
  const int G4p = 4 * p.Hp;
  const bool dam = Ly.dabove != nullptr;
  const int akofs = dam ? Ly.akofs : 0;
  const int nkb0 = (Ly.has_up && !dam) ? G4p / P::kAtomK : 0;
  const int nkb = nkb0 + G4p / P::kAtomK;
  const int kb_lo = rank * nkb / ks, kb_hi = (rank + 1) * nkb / ks;
  const int my_nkb = kb_hi - kb_lo;
  const int a_bytes = kTileM * kRowBytes;
  const int b_bytes = (kPair ? N / 2 : N) * kRowBytes;
  const int b_stage = P::kPlanes * b_bytes;
  const int a_stage = P::kPlanes * a_bytes;
  const int a_total = p.resident ? p.a_slots * a_stage : p.stages * a_stage;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const RecSmem S = carve(smem, a_total, b_stage, p.stages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // one accumulator per step (no promotion): two accumulator buffers in tensor memory, so
  // step t's MMAs (its W^T dG_up half first) run while the epilogue still drains step t+1 --
  // with one buffer they waited for the drain of the last column chunk, i.e. most of the cell
  // phase (config E: 269 us per step, profiles/r02/spans_E_bf16.txt)
  const bool dbuf = p.acc_dbuf && p.n_acc == 1 && !p.promo && 2 * N <= 512;
  // accumulator buffer 1's barriers (selected with acc_bar, not a dynamically indexed array,
  // which would live on the stack)
  uint64_t* const tfull1 = dbuf ? S.pfull : S.tmem_full;
  uint64_t* const tempty1 = dbuf ? S.pempty : S.tmem_empty;
  uint32_t tmem_cols = 32;
  while (tmem_cols < (uint32_t)(N * (dbuf ? 2 : p.n_acc + p.promo))) tmem_cols <<= 1;
  // pair: the leader's tmem_empty takes one arrival per CTA (after its epilogue drained TMEM)
  const uint32_t tmem_base = kPair ? rec_setup_pair(S, p, tmem_cols, 2) : rec_setup(S, p, ks, tmem_cols);
  const int row0 = tile * kTileM;

  // k-blocks this CTA multiplies at step t: seg0 needs dG_{l+1,t} (t >= 0), seg1 needs
  // dG_{l,t+1} (t+1 <= T-1). Step t == -1 is the dh0 = R^T dG_{l,0} step (seg1 only).
  auto kb_active = [&](int kb, int t) {
    if (kb < nkb0) return t >= 0;
    return t + 1 <= p.T - 1;
  };

  if (warp == 0 && lane == 0) {
    for (int pl = 0; pl < P::kPlanes; ++pl) {
      prefetch_tmap(Ly.a[pl]);
      prefetch_tmap(Ly.bg[pl]);
      if (Ly.has_up) prefetch_tmap(Ly.bup[pl]);
    }
    if (p.resident) {
      mbar_arrive_expect_tx(S.a_full, my_nkb * a_stage);
      for (int kb = kb_lo; kb < kb_hi; ++kb)
        for (int pl = 0; pl < P::kPlanes; ++pl)
          tma_load_2d(S.a_res + (kb - kb_lo) * a_stage + pl * a_bytes, Ly.a[pl], S.a_full,
                      (kb + akofs) * P::kAtomK, row0);
    }
    uint32_t pc = 0;
    for (int it = 0; it < p.n_steps; ++it) {
      const int t = p.t_first - it;
      progress(p, 0, it, 1);
      trace_stamp(p, it, 0);
      bool up_ready = false, own_ready = false;
      // streamed weights: L2 prefetch a_prefetch k-blocks ahead, the first ones before the
      // flag waits (the weights do not depend on them)
      if (!p.resident)
        for (int kp = kb_lo; kp < min(kb_hi, kb_lo + p.a_prefetch); ++kp)
          if (kb_active(kp, t))
            for (int pl = 0; pl < P::kPlanes; ++pl) tma_prefetch_2d(Ly.a[pl], (kp + akofs) * P::kAtomK, row0);
      for (int kb = kb_lo; kb < kb_hi; ++kb) {
        if (!kb_active(kb, t)) continue;
        const bool seg0 = kb < nkb0;
        if (!p.resident && p.a_prefetch > 0 && kb + p.a_prefetch < kb_hi && kb_active(kb + p.a_prefetch, t))
          for (int pl = 0; pl < P::kPlanes; ++pl)
            tma_prefetch_2d(Ly.a[pl], (kb + p.a_prefetch + akofs) * P::kAtomK, row0);
        if (seg0 && !up_ready && l == p.L - 1 && p.pp_in_flags) {  // pipeline: dG_t from the next stage
          wait_flag_s(&p.pp_in_flags[t], pp_target(p), true, p.error, p.timeout_ns, wait_code(1, l, t, 1));
          fence_proxy_async_global();
          up_ready = true;
        }
        if (p.persistent) {
          if (seg0 && !up_ready) {
            progress(p, 0, it, 2);
            wait_flag(&up_flags[t], p.flag_target, p, wait_code(1, l, t, 1));
            fence_proxy_async_global();
            up_ready = true;
          }
          if (!seg0 && !own_ready) {
            progress(p, 0, it, 3);
            wait_flag(&Ly.flags[t + 1], p.flag_target, p, wait_code(1, l, t, 2));
            fence_proxy_async_global();
            own_ready = true;
          }
        }
        const int s = pc % p.stages;
        mbar_wait(&S.empty[s], ((pc / p.stages) & 1) ^ 1);
        if constexpr (kPair) {
          // both CTAs: own 128 A rows + half of the dG columns, completion on the leader's barrier
          const uint32_t prank = cluster_ctarank() & 1;
          const int nh = p.Bp / 2;
          if (prank == 0) mbar_arrive_expect_tx(&S.full[s], 2 * (b_stage + a_stage));
          uint8_t* bst = S.b_st + s * b_stage;
          if (seg0)
            g2::tma_load_2d_pair(bst, Ly.bup2, &S.full[s], kb * P::kAtomK, t * p.Bp + (int)prank * nh);
          else
            g2::tma_load_2d_pair(bst, Ly.bg2, &S.full[s], (kb - nkb0) * P::kAtomK, (t + 1) * p.Bp + (int)prank * nh);
          g2::tma_load_2d_pair(S.a_res + s * a_stage, Ly.a[0], &S.full[s], (kb + akofs) * P::kAtomK, row0);
          ++pc;
          continue;
        }
        mbar_arrive_expect_tx(&S.full[s], b_stage + (p.resident ? 0 : a_stage));
        uint8_t* bst = S.b_st + s * b_stage;
        for (int pl = 0; pl < P::kPlanes; ++pl) {
          if (seg0)
            tma_load_2d(bst + pl * b_bytes, Ly.bup[pl], &S.full[s], kb * P::kAtomK, t * p.Bp);
          else
            tma_load_2d(bst + pl * b_bytes, Ly.bg[pl], &S.full[s], (kb - nkb0) * P::kAtomK,
                        (t + 1) * p.Bp);
          if (!p.resident)
            tma_load_2d(S.a_res + s * a_stage + pl * a_bytes, Ly.a[pl], &S.full[s],
                        (kb + akofs) * P::kAtomK, row0);
        }
        ++pc;
      }
      trace_stamp(p, it, 1);
    }
  } else if (kPair && warp == 1) {
    if constexpr (kPair) {
      if (cluster_ctarank() == 0) {
        // ============= MMA issuer (leader, converged warp): M = 256 over the pair, N = Bp
        const uint32_t idesc = idesc_make(P::kFmt, false, false, 2 * kTileM, N);
        uint32_t pc = 0;
        for (int it = 0; it < p.n_steps; ++it) {
          const int t = p.t_first - it;
          const int bi = dbuf ? (it & 1) : 0;
          const int use = dbuf ? (it >> 1) : it;  // earlier steps that used buffer bi
          if (use > 0) {
            mbar_wait(acc_bar(bi, S.tmem_empty, tempty1), (use - 1) & 1);  // both CTAs drained this buffer
            tc_fence_after();
          }
          const uint32_t tacc = tmem_base + (uint32_t)(bi * N);
          bool first = true;
          for (int kb = kb_lo; kb < kb_hi; ++kb) {
            if (!kb_active(kb, t)) continue;
            const int s = pc % p.stages;
            mbar_wait(&S.full[s], (pc / p.stages) & 1);
            tc_fence_after();
            const uint64_t a0 = sdesc_sw128(smem_u32(S.a_res + s * a_stage), 16, 1024);
            const uint64_t b0 = sdesc_sw128(smem_u32(S.b_st + s * b_stage), 16, 1024);
#pragma unroll
            for (int kk = 0; kk < P::kAtomK / P::kUmmaK; ++kk)
              g2::umma2_warp(tacc, desc_add(a0, kk * 32), desc_add(b0, kk * 32), idesc,
                             (!first || kk) ? 1u : 0u);
            g2::commit2_warp(&S.empty[s]);
            first = false;
            ++pc;
          }
          g2::commit2_warp(acc_bar(bi, S.tmem_full, tfull1));
        }
      }
    }
  } else if (!kPair && warp == 1) {
    // whole warp 1 (converged; elect.sync inside each MMA / commit): a lane-0-only issue branch
    // costs an ELECT / R2UR waterfall per instruction (profiles/ubench/mma_ubench.cu)
    const uint32_t idesc = idesc_make(P::kFmt, false, false, kTileM, N);
    if (p.resident) mbar_wait(S.a_full, 0);
    tc_fence_after();
    uint32_t pc = 0, ch = 0;
    for (int it = 0; it < p.n_steps; ++it) {
      const int t = p.t_first - it;
      progress(p, 1, it, 1);
      const int bi = dbuf ? (it & 1) : 0;
      const int use = dbuf ? (it >> 1) : it;  // earlier steps that used accumulator buffer bi
      if (use > 0 && !p.promo) {
        mbar_wait(acc_bar(bi, S.tmem_empty, tempty1), (use - 1) & 1);
        tc_fence_after();
      }
      progress(p, 1, it, 2);
      // active k-blocks of this step per K segment (the ring closes a chunk on each segment's last)
      // (scalars, not [2] arrays indexed by segment: those would live on the stack)
      int nseg0 = 0, nseg1 = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb)
        if (kb_active(kb, t)) ++(kb < nkb0 ? nseg0 : nseg1);
      int nact = 0, nact0 = 0;  // active k-blocks so far this step (overall, in segment 0)
      for (int kb = kb_lo; kb < kb_hi; ++kb) {
        if (!kb_active(kb, t)) continue;
        const int s = pc % p.stages;
        const bool sg0 = kb < nkb0;
        const int iseg = sg0 ? nact0 : nact - nact0;  // position inside this k-block's segment
        const bool cstart = p.promo ? iseg % p.acc_kb == 0 : nact % p.acc_kb == 0;
        const uint32_t acc = p.promo ? promo_slot(S, p, tmem_base, N, cstart, ch)
                                     : tmem_base + (uint32_t)(bi * N) + (nact / p.acc_kb) * N;
        mbar_wait(&S.full[s], (pc / p.stages) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(S.a_res + (p.resident ? (kb - kb_lo) : s) * a_stage);
        const uint32_t b_base = smem_u32(S.b_st + s * b_stage);
        mma_kblock<P>(acc, a_base, b_base, a_bytes, b_bytes, idesc, cstart);
        ++nact;
        nact0 += sg0 ? 1 : 0;
        umma_commit_warp(&S.empty[s]);
        if (p.promo && ((iseg + 1) % p.acc_kb == 0 || iseg + 1 == (sg0 ? nseg0 : nseg1))) {
          umma_commit_warp(&S.pfull[ch % (uint32_t)p.n_acc]);
          ++ch;
        }
        ++pc;
      }
      if (!p.promo) umma_commit_warp(acc_bar(bi, S.tmem_full, tfull1));
    }
  } else if (warp >= 4) {
    const BwdLayer Le = Ly;  // register copy (see the forward epilogue)
    // ================= epilogue: split-K exchange + LSTM backward (cells.hpp:424-447)
    const int et = threadIdx.x - kEpiBase;
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int ul = et & 127;            // unit within the tile (cell phase)
    const int hh = et >> 7;             // column parity (cell phase)
    const int u = row0 + ul;
    const long long Hp = p.Hp, G4 = 4 * Hp;
    uint32_t xc = 0, ech = 0;
    constexpr float kGS = kF16Ops<P> ? pow2f(kGScaleLog2) : 1.0f;  // dG operand plane scale
    float gmax = 0.0f;
    for (int it = 0; it < p.n_steps; ++it) {
      const int t = p.t_first - it;
      int ns0 = 0, ns1 = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb)
        if (kb_active(kb, t)) ++(kb < nkb0 ? ns0 : ns1);
      const int nact = ns0 + ns1;
      const int nc0 = (ns0 + p.acc_kb - 1) / p.acc_kb;
      const int n_chunks = (!kPair && p.promo) ? nc0 + (ns1 + p.acc_kb - 1) / p.acc_kb : (nact + p.acc_kb - 1) / p.acc_kb;
      const int n_used = (!kPair && p.promo) ? (n_chunks > 0 ? 1 : 0) : n_chunks;
      if (et == 0) progress(p, 2, it, 1);
      const int bi = dbuf ? (it & 1) : 0;
      const uint32_t tacc = tmem_base + (uint32_t)(bi * N);
      if (!kPair && p.promo) {
        promo_drain(S, p, tmem_base, N, n_chunks, ech, nc0, p.us_in, p.us_rec);
      } else {
        mbar_wait(acc_bar(bi, S.tmem_full, tfull1), (dbuf ? (it >> 1) : it) & 1);
        tc_fence_after();
      }
      if (et == 0) trace_stamp(p, it, 2);
      for (int n0 = 0; n0 < N; n0 += kXChunk, ++xc) {
        const int nc = min(kXChunk, N - n0);
        const int nco = nc / ks;
        const uint32_t inv = (65536u + nco - 1) / nco;
        xchg_wait_free(S, ks, xc);
        for (int c0 = half * (nc >> 1); c0 < (half + 1) * (nc >> 1); c0 += 8) {
          float a[8];
          load_acc_sum(tacc + (uint32_t(q * 32) << 16) + n0 + c0, N, n_used, a);
          xchg_push8(S, ks, rank, nco, q, lane, c0, a, inv);
        }
        if (n0 + kXChunk >= N && (kPair || !p.promo)) {
          tc_fence_before();
          if constexpr (kPair) {
            named_bar_sync(1, kEpiThreads);  // the whole CTA drained its TMEM accumulator
            if (et == 0) mbar_arrive_remote(acc_bar(bi, S.tmem_empty, tempty1), 0);
          } else {
            mbar_arrive(acc_bar(bi, S.tmem_empty, tempty1));
          }
        }
        if (et == 0 && n0 == 0) trace_stamp(p, it, 3);
        xchg_publish(S, ks, xc);
        if (et == 0 && n0 == 0) trace_stamp(p, it, 4);
        const long long cbase = (long long)n0 + rank * nco;  // first owned batch column
        if (u < p.Hp) {
          float si = 0.0f, sf = 0.0f, so = 0.0f, sc = 0.0f;  // db partials (cells.hpp:163-168)
          // owned columns cl = hh + 2k, processed 8 at a time: all loads first, then math
          for (int kb8 = 0; kb8 * 16 < nco; ++kb8) {
            float acc[8], pi[8], pf[8], po[8], pcb[8], ptc[8], pcp[8], dci[8], dyv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int cl = hh + 2 * (kb8 * 8 + k);
              acc[k] = pi[k] = pf[k] = po[k] = pcb[k] = ptc[k] = pcp[k] = dci[k] = dyv[k] = 0.0f;
              if (cl >= nco) continue;
              acc[k] = xchg_sum(S, ks, nco, cl, ul);
              const long long n = cbase + cl;
              if (t < 0) {
                dci[k] = Le.carry_c[n * Hp + u];
                continue;
              }
              const long long col = (long long)t * p.Bp + n;
              const float* gp = Le.gates + col * G4 + u;
              if constexpr (kKind == kCellLstm) {
                pi[k] = gp[0];
                pf[k] = gp[Hp];
                po[k] = gp[2 * Hp];
                pcb[k] = gp[3 * Hp];
                ptc[k] = Le.tanhc[col * Hp + u];
                pcp[k] = Le.c[col * Hp + u];  // c_{t-1}: block t of the c tape
              } else if constexpr (kKind == kCellGru) {
                pi[k] = gp[0];                 // r
                pf[k] = gp[Hp];                // u
                po[k] = gp[2 * Hp];            // n
                pcb[k] = Le.zrh[col * Hp + u]; // R_n h_{t-1}
                pcp[k] = Le.h[col * Hp + u];   // h_{t-1}: block t of the h tape
              } else {
                pcp[k] = Le.h[(col + p.Bp) * Hp + u];  // h_t: block t + 1
              }
              // LSTM: the cell-state carry dc f; GRU: the direct term dh u (cells.hpp:531)
              dci[k] = (t == p.T - 1 || kKind == kCellRnnTanh) ? 0.0f : Le.carry_c[n * Hp + u];
              if (dam)
                dyv[k] = Le.dabove[col * Hp + u];
              else if (Le.dy && u < p.H && n < p.B)
                dyv[k] = Le.dy[((long long)t * p.B + n) * p.H + u];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int cl = hh + 2 * (kb8 * 8 + k);
              if (cl >= nco) break;
              const long long n = cbase + cl;
              if (t < 0) {  // dh0 / dc0 (engine.hpp:163-170); GRU: dh0 = R^T dgr_0 + dh_0 u_0
                if constexpr (kKind == kCellGru) {
                  Le.dh0[n * Hp + u] = acc[k] + dci[k];
                } else {
                  Le.dh0[n * Hp + u] = acc[k];
                  if constexpr (kKind == kCellLstm) Le.dc0[n * Hp + u] = dci[k];
                }
                continue;
              }
              // d_above + carry_h (GRU: carry_h = R^T dgr_{t+1} + the direct term dh_{t+1} u_{t+1})
              const float chh = kKind == kCellGru ? acc[k] + dci[k] : acc[k];
              const float dh = (Le.dy || dam) ? dyv[k] + chh : chh;
              float gi, gf = 0.0f, go = 0.0f, gc = 0.0f, rn = 0.0f;  // rn: GRU dgr of the candidate
              if constexpr (kKind == kCellLstm) {  // cells.hpp:424-447
                const float q1 = dh * po[k];
                const float s0 = ptc[k] * ptc[k];
                const float s1 = 1.0f - s0;
                const float q2 = q1 * s1;
                const float dc = dci[k] + q2;
                const float a1 = dc * pcb[k], a2 = a1 * pi[k], a3 = 1.0f - pi[k];
                const float b1 = dc * pcp[k], b2 = b1 * pf[k], b3 = 1.0f - pf[k];
                const float c1 = dh * ptc[k], c2 = c1 * po[k], c3 = 1.0f - po[k];
                const float d1 = dc * pi[k], d2 = pcb[k] * pcb[k], d3 = 1.0f - d2;
                gi = a2 * a3;
                gf = b2 * b3;
                go = c2 * c3;
                gc = d1 * d3;
                Le.carry_c[n * Hp + u] = dc * pf[k];
              } else if constexpr (kKind == kCellGru) {  // cells.hpp:514-538
                const float om = 1.0f - pf[k];
                const float dn = dh * om;
                const float s = po[k] * po[k];
                const float s1 = 1.0f - s;
                const float dnp = dn * s1;
                const float tt = pcp[k] - po[k];
                const float q = dh * tt;
                const float q2 = q * pf[k];
                const float dgu = q2 * om;
                const float r0 = dnp * pcb[k];
                const float r1 = r0 * pi[k];
                const float r2 = 1.0f - pi[k];
                gi = r1 * r2;  // dgw = dgr (reset gate)
                gf = dgu;      // dgw = dgr (update gate)
                go = dnp;      // dgw (candidate)
                rn = dnp * pi[k];
                Le.carry_c[n * Hp + u] = dh * pf[k];
              } else {  // RNN (cells.hpp:370-383)
                if (p.kind == kCellRnnRelu) {
                  gi = pcp[k] > 0.0f ? dh : 0.0f;
                } else {
                  const float s = pcp[k] * pcp[k];
                  const float s1 = 1.0f - s;
                  gi = dh * s1;
                }
              }
              const long long col = (long long)t * p.Bp + n;
              float* dgp = Le.dg + col * G4 + u;
              dgp[0] = gi;
              dgp[Hp] = gf;
              dgp[2 * Hp] = go;
              dgp[3 * Hp] = gc;
              const long long ob = col * G4;
              store_operand<P>(Le.dgop, ob + rho_of(0, u), gi * kGS);
              store_operand<P>(Le.dgop, ob + rho_of(1, u), gf * kGS);
              store_operand<P>(Le.dgop, ob + rho_of(2, u), go * kGS);
              store_operand<P>(Le.dgop, ob + rho_of(3, u), gc * kGS);
              if (Le.dg_peer[0]) {  // pipeline: the previous stage's dG input (W-side, as dgop)
                store_operand<P>(Le.dg_peer, ob + rho_of(0, u), gi * kGS);
                store_operand<P>(Le.dg_peer, ob + rho_of(1, u), gf * kGS);
                store_operand<P>(Le.dg_peer, ob + rho_of(2, u), go * kGS);
                store_operand<P>(Le.dg_peer, ob + rho_of(3, u), gc * kGS);
              }
              if constexpr (kKind == kCellGru) {  // dgr: r, u as dgw, candidate dnp r (cells.hpp:527-529)
                float* dgq = Le.dgr + col * G4 + u;
                dgq[0] = gi;
                dgq[Hp] = gf;
                dgq[2 * Hp] = rn;
                store_operand<P>(Le.dgrop, ob + rho_of(0, u), gi * kGS);
                store_operand<P>(Le.dgrop, ob + rho_of(1, u), gf * kGS);
                store_operand<P>(Le.dgrop, ob + rho_of(2, u), rn * kGS);
                store_operand<P>(Le.dgrop, ob + rho_of(3, u), 0.0f);
              }
              if constexpr (kF16Ops<P>) gmax = fmaxf(gmax, fmaxf(fmaxf(fabsf(gi), fabsf(gf)), fmaxf(fabsf(go), fabsf(gc))));
              si += gi;
              sf += gf;
              so += go;
              sc += gc;
            }
          }
          if (t >= 0 && Le.dbp) {
            float* d = Le.dbp + (long long)(((n0 / kXChunk) * ks + rank) * 2 + hh) * G4 + u;
            d[0] += si;
            d[Hp] += sf;
            d[2 * Hp] += so;
            d[3 * Hp] += sc;
          }
        }
        if (et == 0 && n0 == 0) trace_stamp(p, it, 5);
        xchg_release(S, ks);
        if (et == 0 && n0 == 0) trace_stamp(p, it, 6);
      }
      if (p.persistent && t >= 0) {
        fence_proxy_async_global();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          __threadfence();
          red_release_gpu_add(&Le.flags[t], 1);
        }
      }
      if (Le.dg_peer[0] && t >= 0) {  // pipeline: publish dG_t to the previous stage
        if (!p.persistent) {
          fence_proxy_async_global();
          named_bar_sync(1, kEpiThreads);
        }
        if (et == 0) {
          __threadfence_system();
          red_release_s(Le.peer_flags + t, 1, true);
        }
      }
      if (et == 0) trace_stamp(p, it, 7);
    }
    if constexpr (kF16Ops<P>) {  // range of the scaled dG planes (one atomic per warp)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
      if ((threadIdx.x & 31) == 0 && p.gmax) atomicMax(p.gmax, __float_as_uint(gmax));
    }
  }
  if constexpr (kPair)
    rec_teardown_pair(tmem_base, tmem_cols);
  else
    rec_teardown(ks, tmem_base, tmem_cols);
}

}  // namespace rw

// common.cuh -- shared definitions between the sm_100a kernels and the host runtime.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace rw {

// Operand precision of the tensor-core GEMMs. Accumulation and all pointwise cell math
// are fp32 in both modes.
//   kBF16  : operands rounded to bf16 (kind::f16), 1 plane.
//   kTF32x3: operands split x = hi + lo, hi = tf32(x) (round-to-nearest), lo = x - hi, and
//            D += A_hi B_hi + A_hi B_lo + A_lo B_hi (kind::tf32), 2 planes -- the fp32-parity
//            mode (normwise error ~1e-6 vs the fp32 reference engine).
//   kF16x2 : operands split x = hi + lo, hi = fp16_rn(x), lo = fp16_rn(x - hi) (22 significant
//            bits), D += A_hi B_hi + A_hi B_lo + A_lo B_hi (kind::f16, fp16 rate), 2 planes of 2
//            bytes. The fp32-parity mode of the cluster schedule: half the bytes of 3xTF32 and
//            twice its MMA rate, so the recurrent weights stay on chip (A_hi resident in shared
//            memory, A_lo in tensor memory as the A operand of tcgen05.mma "TS"). Weight planes
//            are stored pre-scaled by 2^kWScaleLog2 (exact) so their lo part stays a normal fp16;
//            epilogues multiply weight products by 2^-kWScaleLog2. Activation lo parts are
//            unscaled: a subnormal lo carries an absolute error <= 2^-25, far below the 1e-5
//            normwise contract for operands of O(1) magnitude (profiles/ubench/f16x2_ts_check.cu:
//            normwise 6.4e-7 at K = 512 vs an fp64 product). The gate gradients dG are the
//            exception: they shrink layer by layer going down (config B layer 0: |dG| ~ 1e-2 and
//            below), where unscaled lo parts lost enough bits to miss the 1e-5 contract (dx0
//            1.5e-5 normwise, measured), so the dG operand planes carry 2^kGScaleLog2 too and
//            every consumer (R^T.dG, W^T.dG, dW / dR, dx0) scales its result back (exact).
//            Hidden states and inputs get the same treatment (at config B the top layer's dR =
//            dG.h^T missed the scaled-max bound by 6% with unscaled h), so every fp16x2 operand
//            plane carries a power-of-two scale: weights 2^kWScaleLog2, h (and h0)
//            2^kHScaleLog2, the layer-0 input x 2^kXScaleLog2, dG 2^kGScaleLog2.
//            Range (fp16 max 65504 after scaling): |W| < 255, |h0| < 16 (every later h is a
//            tanh product, |h| < 1), |x| < 4096, |dG| < 64. The pad kernels record max|x| and
//            max|h0|, the backward max|dG|, and the runtime reports a range error past them.
enum Prec : int { kBF16 = 0, kTF32x3 = 1, kF16x2 = 2 };
constexpr int kWScaleLog2 = 8;
constexpr int kHScaleLog2 = 12;
constexpr int kXScaleLog2 = 4;
constexpr int kGScaleLog2 = 10;
__host__ __device__ constexpr float pow2f(int e) { return e >= 0 ? (float)(1u << e) : 1.0f / (float)(1u << -e); }

__host__ __device__ constexpr int prec_planes(int prec) { return prec == kBF16 ? 1 : 2; }
__host__ __device__ constexpr int prec_elem(int prec) { return prec == kTF32x3 ? 4 : 2; }
__host__ __device__ constexpr int prec_atomk(int prec) { return prec == kTF32x3 ? 32 : 64; }

struct PrecBF16 {
  static constexpr int kPlanes = 1;
  static constexpr int kElem = 2;
  static constexpr int kAtomK = 64;  // elements per 128-byte swizzle row
  static constexpr int kUmmaK = 16;
  static constexpr uint32_t kFmt = 1;
  static constexpr bool kTF32 = false;
  static constexpr int kCombos = 1;
};
struct PrecTF32x3 {
  static constexpr int kPlanes = 2;
  static constexpr int kElem = 4;
  static constexpr int kAtomK = 32;
  static constexpr int kUmmaK = 8;
  static constexpr uint32_t kFmt = 2;
  static constexpr bool kTF32 = true;
  static constexpr int kCombos = 3;
};

struct PrecF16x2 {
  static constexpr int kPlanes = 2;
  static constexpr int kElem = 2;
  static constexpr int kAtomK = 64;
  static constexpr int kUmmaK = 16;
  static constexpr uint32_t kFmt = 0;  // kind::f16 with fp16 inputs
  static constexpr bool kTF32 = false;
  static constexpr int kCombos = 3;
};

// fp16x2 split of v (already scaled): hi = fp16_rn(v), lo = fp16_rn(v - hi) (v - hi is exact in fp32).
__device__ __forceinline__ void f16x2_split(float v, __half& hi, __half& lo) {
  hi = __float2half_rn(v);
  lo = __float2half_rn(v - __half2float(hi));
}

// fp32-parity activations without libm's slow paths (cluster forward epilogue): 2^t by MUFU.EX2
// (relative error ~2^-22, plus |t| 2^-24 from rounding t), the reciprocal by MUFU.RCP + one Newton
// step; tanh below |x| = 0.6 by an odd polynomial (least-squares fit, 7.6e-8 relative in fp32),
// where 1 - 2/(1+e^2x) would cancel. Within a few fp32 ulps of expf / tanhf.
__device__ __forceinline__ float ex2_approx(float t) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(t));
  return y;
}
__device__ __forceinline__ float rcp_newton(float d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  return fmaf(r, fmaf(-d, r, 1.0f), r);
}
__device__ __forceinline__ float sigmoid_fast(float x) {
  return rcp_newton(1.0f + ex2_approx(fminf(-1.4426950408889634f * x, 126.0f)));
}
__device__ __forceinline__ float tanh_fast(float x) {
  const float ax = fabsf(x);
  const float z = x * x;
  float p = -0.005984960589557886f;
  p = fmaf(p, z, 0.020868148654699326f);
  p = fmaf(p, z, -0.053803566843271255f);
  p = fmaf(p, z, 0.13332132995128632f);
  p = fmaf(p, z, -0.3333330452442169f);
  const float small = fmaf(x * z, p, x);
  const float r = 1.0f - 2.0f * rcp_newton(1.0f + ex2_approx(fminf(2.8853900817779268f * ax, 126.0f)));
  return ax < 0.6f ? small : copysignf(r, x);
}

// Cell kinds (rw_config.cell_kind, the reference's CellKind order): the cluster kernels are
// instantiated per class -- LSTM, GRU, RNN (tanh / relu selected at run time).
enum CellKindDev : int { kCellRnnTanh = 0, kCellRnnRelu = 1, kCellGru = 2, kCellLstm = 3 };
__host__ __device__ constexpr int cell_gates(int kind) { return kind == kCellLstm ? 4 : kind == kCellGru ? 3 : 1; }

constexpr int kTileM = 128;      // UMMA M (cta_group::1)
constexpr int kRowBytes = 128;   // one SWIZZLE_128B row
constexpr int kUnitsPerFwdTile = 32;  // forward tile = 32 hidden units x 4 gates

// Gate-interleaved row order used by every forward operand/accumulator:
// row rho = tile*128 + g*32 + j  <->  gate g of hidden unit u = tile*32 + j.
__host__ __device__ inline int rho_of(int g, int u) { return (u >> 5) * 128 + g * 32 + (u & 31); }
__host__ __device__ inline int rho_gate(int rho) { return (rho & 127) >> 5; }
__host__ __device__ inline int rho_unit(int rho) { return (rho >> 7) * 32 + (rho & 31); }

// Byte offset of element (k, n) inside one step block of a pre-swizzled operand: k-blocks of
// 64 K-elements, each Bp rows of 128 B with the 16-B chunks XOR-permuted by row % 8 -- exactly
// the shared-memory image TMA SWIZZLE_128B produces for a {64, Bp} box, so a consumer fetches
// a k-block with one contiguous 1-D bulk copy (rec_cluster.cuh).
__host__ __device__ inline long long sw_off(int k, int n, int Bp) {
  return (long long)(k >> 6) * Bp * 128 + n * 128 + ((((k >> 3) & 7) ^ (n & 7)) << 4) + (k & 7) * 2;
}

// Output index mapping of the generic GEMM epilogue.
// kRowGateRepad: reference gate-major rows g*H + u -> padded gate-major g*Hp + u (the ladder's
// grouped GEMMs on the reference-layout weights)
enum RowMode : int { kRowIdentity = 0, kRowGateUnperm = 1, kRowGatePad = 2, kRowGateRepad = 3 };
enum ColMode : int { kColIdentity = 0, kColBatchUnpad = 1 };

// One (grouped) GEMM problem: D[MxN] = A[MxK] * B[NxK]^T, fp32 out.
struct GemmDesc {
  const CUtensorMap* a[2];
  const CUtensorMap* b[2];
  int M, N, K;         // tile-space dims (K multiple of the k-block)
  int a_k_off, b_k_off;  // K coordinate offsets inside the A / B tensors
  float* d;
  long long ldd;
  int row_mode, col_mode;
  int H, Hp, B, Bp;    // for the unpermute / unpad maps
  int m_valid, n_valid;  // identity-mode bounds
  int accumulate;      // D += result instead of D = result
  int b_n_off;         // row (N) offset inside the B tensor (e.g. h_{l-1} starts at column block 1)
  float alpha;         // D = alpha * A B^T (fp16x2 weight operands carry 2^kWScaleLog2); 0 means 1
  int* error;          // the context's error word (bounded mbarrier waits, sm100_ptx.cuh)
  int gates;           // kRowGateUnperm: the cell's gate count (0 = 4)
  int a_m_off;         // row (M) offset inside the A tensor (k_gemm_tc only: the ladder's per-gate GEMMs)
};

}  // namespace rw

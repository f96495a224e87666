// pointwise.cuh -- the reference's free pointwise stage (proj/include/rnnwave/cells.hpp:181-333
// forward, 349-562 backward) as device kernels: one thread per (unit, column) element, the
// reference's operation chain written with explicitly rounded fp32 intrinsics (__fadd_rn /
// __fmul_rn are never contracted into FMAs), accurate expf / tanhf. The reference defines its
// fused and kernel-per-op modes to be bitwise identical, so one kernel serves both. Matrices are
// dense column-major (ld = rows); the recurrent kernels fuse the same math into their epilogues.
#pragma once

#include "common.cuh"

namespace rw {

__device__ __forceinline__ float pw_sigmoid(float x) {  // cells.hpp:29
  return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-x)));
}

// kind: CellKindDev. zw, zr, gates: G*H x B; h_prev, c_prev, h_out, c_out, tanh_c, zr_h: H x B.
// gates / tanh_c / zr_h may be null (inference).
__global__ void k_pointwise_fwd(int kind, int H, int B, const float* __restrict__ zw, const float* __restrict__ zr,
                                const float* __restrict__ bias, const float* __restrict__ h_prev,
                                const float* __restrict__ c_prev, float* __restrict__ h_out, float* __restrict__ c_out,
                                float* __restrict__ gates, float* __restrict__ tanh_c, float* __restrict__ zr_h) {
  const long long n = (long long)H * B;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / H), r = (int)(e - (long long)c * H);
    if (kind == kCellRnnTanh || kind == kCellRnnRelu) {  // cells.hpp:200-212
      const long long z = (long long)c * H + r;
      const float a = __fadd_rn(__fadd_rn(zw[z], zr[z]), bias[r]);
      h_out[e] = kind == kCellRnnTanh ? tanhf(a) : (a > 0.0f ? a : 0.0f);
    } else if (kind == kCellLstm) {  // cells.hpp:232-254
      const long long z = (long long)c * 4 * H + r;
      const float ai = __fadd_rn(__fadd_rn(zw[z], zr[z]), bias[r]);
      const float af = __fadd_rn(__fadd_rn(zw[z + H], zr[z + H]), bias[H + r]);
      const float ao = __fadd_rn(__fadd_rn(zw[z + 2 * H], zr[z + 2 * H]), bias[2 * H + r]);
      const float ac = __fadd_rn(__fadd_rn(zw[z + 3 * H], zr[z + 3 * H]), bias[3 * H + r]);
      const float iv = pw_sigmoid(ai), fv = pw_sigmoid(af), ov = pw_sigmoid(ao);
      const float cb = tanhf(ac);
      const float t1 = __fmul_rn(fv, c_prev[e]);
      const float t2 = __fmul_rn(iv, cb);
      const float cv = __fadd_rn(t1, t2);
      const float tc = tanhf(cv);
      if (gates) {
        gates[z] = iv;
        gates[z + H] = fv;
        gates[z + 2 * H] = ov;
        gates[z + 3 * H] = cb;
      }
      c_out[e] = cv;
      if (tanh_c) tanh_c[e] = tc;
      h_out[e] = __fmul_rn(ov, tc);
    } else {  // GRU, linear before reset (cells.hpp:294-313)
      const long long z = (long long)c * 3 * H + r;
      const float ar = __fadd_rn(__fadd_rn(zw[z], zr[z]), bias[r]);
      const float au = __fadd_rn(__fadd_rn(zw[z + H], zr[z + H]), bias[H + r]);
      const float rv = pw_sigmoid(ar), uv = pw_sigmoid(au);
      const float t1 = __fadd_rn(zw[z + 2 * H], bias[2 * H + r]);
      const float t2 = __fmul_rn(rv, zr[z + 2 * H]);
      const float nv = tanhf(__fadd_rn(t1, t2));
      const float t3 = __fmul_rn(uv, h_prev[e]);
      const float t4 = __fmul_rn(__fadd_rn(1.0f, -uv), nv);
      if (gates) {
        gates[z] = rv;
        gates[z + H] = uv;
        gates[z + 2 * H] = nv;
      }
      h_out[e] = __fadd_rn(t3, t4);
      if (zr_h) zr_h[e] = zr[z + 2 * H];
    }
  }
}

// saved: gates (G*H x B; the post-activation h for the RNN kinds), tanh_c (LSTM), zr_h (GRU).
// dgr: GRU only (distinct from dgw); dc_carry / dc_prev: LSTM only.
__global__ void k_pointwise_bwd(int kind, int H, int B, const float* __restrict__ gates,
                                const float* __restrict__ tanh_c, const float* __restrict__ zr_h,
                                const float* __restrict__ h_prev, const float* __restrict__ c_prev,
                                const float* __restrict__ d_above, const float* __restrict__ dh_carry,
                                const float* __restrict__ dc_carry, float* __restrict__ dgw, float* __restrict__ dgr,
                                float* __restrict__ dh_local, float* __restrict__ dc_prev) {
  const long long n = (long long)H * B;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / H), r = (int)(e - (long long)c * H);
    const float dh = __fadd_rn(d_above[e], dh_carry[e]);
    if (kind == kCellRnnTanh || kind == kCellRnnRelu) {  // cells.hpp:370-383
      const float hv = gates[e];
      dgw[e] = kind == kCellRnnTanh ? __fmul_rn(dh, __fadd_rn(1.0f, -__fmul_rn(hv, hv))) : (hv > 0.0f ? dh : 0.0f);
      dh_local[e] = 0.0f;
    } else if (kind == kCellLstm) {  // cells.hpp:424-447
      const long long z = (long long)c * 4 * H + r;
      const float iv = gates[z], fv = gates[z + H], ov = gates[z + 2 * H], cb = gates[z + 3 * H];
      const float tc = tanh_c[e];
      const float q1 = __fmul_rn(dh, ov);
      const float s1 = __fadd_rn(1.0f, -__fmul_rn(tc, tc));
      const float dc = __fadd_rn(dc_carry[e], __fmul_rn(q1, s1));
      dgw[z] = __fmul_rn(__fmul_rn(__fmul_rn(dc, cb), iv), __fadd_rn(1.0f, -iv));
      dgw[z + H] = __fmul_rn(__fmul_rn(__fmul_rn(dc, c_prev[e]), fv), __fadd_rn(1.0f, -fv));
      dgw[z + 2 * H] = __fmul_rn(__fmul_rn(__fmul_rn(dh, tc), ov), __fadd_rn(1.0f, -ov));
      dgw[z + 3 * H] = __fmul_rn(__fmul_rn(dc, iv), __fadd_rn(1.0f, -__fmul_rn(cb, cb)));
      dc_prev[e] = __fmul_rn(dc, fv);
      dh_local[e] = 0.0f;
    } else {  // GRU (cells.hpp:514-538)
      const long long z = (long long)c * 3 * H + r;
      const float rv = gates[z], uv = gates[z + H], nv = gates[z + 2 * H];
      const float om = __fadd_rn(1.0f, -uv);
      const float dnp = __fmul_rn(__fmul_rn(dh, om), __fadd_rn(1.0f, -__fmul_rn(nv, nv)));
      const float dgu = __fmul_rn(__fmul_rn(__fmul_rn(dh, __fadd_rn(h_prev[e], -nv)), uv), om);
      const float dgr_gate = __fmul_rn(__fmul_rn(__fmul_rn(dnp, zr_h[e]), rv), __fadd_rn(1.0f, -rv));
      dgw[z] = dgr_gate;
      dgw[z + H] = dgu;
      dgw[z + 2 * H] = dnp;
      dgr[z] = dgr_gate;
      dgr[z + H] = dgu;
      dgr[z + 2 * H] = __fmul_rn(dnp, rv);
      dh_local[e] = __fmul_rn(dh, uv);
    }
  }
}

// db[row] += sum over columns of dgw(row, col), ascending col (cells.hpp:163-168)
__global__ void k_row_sums_add(const float* __restrict__ src, int rows, int cols, float* __restrict__ db) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    float acc = db[r];
    for (int c = 0; c < cols; ++c) acc = __fadd_rn(acc, src[(long long)c * rows + r]);
    db[r] = acc;
  }
}

}  // namespace rw

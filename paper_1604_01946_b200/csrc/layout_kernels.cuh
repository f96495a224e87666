// layout_kernels.cuh -- the HBM-bound layout kernels around the tensor-core path:
//   K7 repack (params.hpp:55-61 pretranspose, re-imagined): reference column-major gate-
//     stacked W/R (4H x I) -> padded, gate-interleaved, K-major operand planes;
//   activation padding/conversion (x, h0, c0 -> padded tapes and operand planes);
//   un-padding of tapes for read-back; the bias-gradient reduction.
#pragma once

#include "common.cuh"

namespace rw {

// `f16scale`: fp16x2 operand planes carry a power-of-two scale (common.cuh: weights
// 2^kWScaleLog2, h 2^kHScaleLog2, x 2^kXScaleLog2); other formats ignore it.
__device__ __forceinline__ void store_planes(int prec, void* p0, void* p1, long long idx, float v,
                                             float f16scale = 1.0f) {
  if (prec == kBF16) {
    static_cast<__nv_bfloat16*>(p0)[idx] = __float2bfloat16_rn(v);
  } else if (prec == kF16x2) {
    __half hi, lo;
    f16x2_split(v * f16scale, hi, lo);
    static_cast<__half*>(p0)[idx] = hi;
    static_cast<__half*>(p1)[idx] = lo;
  } else {
    uint32_t hi;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(v));
    const float fh = __uint_as_float(hi);
    static_cast<float*>(p0)[idx] = fh;
    static_cast<float*>(p1)[idx] = v - fh;
  }
}

// Backward operand of layer l: rows = units (Hp), K = [W_{l+1}^T (4Hp, rho order)] ++
// [R_l^T (4Hp, rho order)]; Wup may be null (top layer). Both sources are 4H x H.
__global__ void k_pack_wb(const float* __restrict__ Wup, const float* __restrict__ R, int H,
                          int Hp, int prec, void* p0, void* p1, int G = 4) {
  const int G4p = 4 * Hp;
  const long long K = (Wup ? 2LL : 1LL) * G4p;
  const long long total = (long long)Hp * K;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int u = (int)(e / K);
    const int k = (int)(e - u * K);
    const float* M = (Wup && k < G4p) ? Wup : R;
    const int rho = k % G4p;
    const int g = rho_gate(rho), up = rho_unit(rho);
    float v = 0.0f;
    if (u < H && up < H && g < G) v = M[(long long)u * G * H + (long long)g * H + up];
    store_planes(prec, p0, p1, e, v, pow2f(kWScaleLog2));
  }
}

// dx0 operand: W_0^T, rows = input features (Ip), K = 4Hp in rho order.
__global__ void k_pack_w0t(const float* __restrict__ W0, int H, int I, int Hp, int Ip, int prec,
                           void* p0, void* p1, int G = 4) {
  const int G4p = 4 * Hp;
  const long long total = (long long)Ip * G4p;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / G4p);
    const int rho = (int)(e - (long long)i * G4p);
    const int g = rho_gate(rho), u = rho_unit(rho);
    float v = 0.0f;
    if (i < I && u < H && g < G) v = W0[(long long)i * G * H + (long long)g * H + u];
    store_planes(prec, p0, p1, e, v, pow2f(kWScaleLog2));
  }
}

// ---- the whole K7 repack of a context in ONE launch (runtime.cu repack_params): a table of jobs
// (every layer's forward [W|R] image, backward [W_{l+1}^T | R_l^T] image and padded bias, plus the
// dx0 operand W_0^T), each cut into tiles of 32 destination rows x 128 K; block b finds its job by
// the jobs' first-tile indices. Per tile the source is read once in 128-byte runs and the
// destination planes are written 4 elements (8-16 bytes) per thread and plane.
//   kRepackT ("transpose", the forward image): dest row rho (gate g, unit u), K = [W cols | R
//     cols]; the source columns hold 32 consecutive units of one gate contiguously, the dest rows
//     are K-contiguous -> through a 64 x 33 shared tile.
//   kRepackC ("copy", backward image and W_0^T): dest row = source column (unit u / input i),
//     K = rho order of one or two 4Hp halves; 4 consecutive rho are 4 consecutive units of one
//     gate, i.e. 4 consecutive source elements of the same column -> direct float4 reads.
//   kRepackB: the padded bias (4Hp fp32).
enum RepackKind : int { kRepackT = 0, kRepackC = 1, kRepackB = 2 };
constexpr int kRepackTileK = 128;
struct RepackJob {
  int kind, tile0, tiles_k;  // first tile of the job, tiles along K (kRepackB: 1024 elements / tile)
  int rows, K;               // destination rows and K (elements)
  int src_rows, k_split;     // valid source columns (kRepackC rows: H or I) / T: first R column (Ipl)
  int src_k0;                // T: valid W columns (I or H); C: 4Hp, the width of one K half
  const float* s0;           // T: W; C: first K half (W_{l+1} or W_0; null -> second half only); B: bias
  const float* s1;           // T: R; C: second half (R_l)
  void* p0;
  void* p1;
};

__device__ __forceinline__ void store4_planes(int prec, void* p0, void* p1, long long idx, const float v[4],
                                              float f16scale) {
  if (prec == kBF16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&a);
    w.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p0) + idx) = w;
  } else if (prec == kF16x2) {
    __half hi[4], lo[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) f16x2_split(v[c] * f16scale, hi[c], lo[c]);
    *reinterpret_cast<uint2*>(static_cast<__half*>(p0) + idx) = *reinterpret_cast<uint2*>(hi);
    *reinterpret_cast<uint2*>(static_cast<__half*>(p1) + idx) = *reinterpret_cast<uint2*>(lo);
  } else {
    float4 hi, lo;
    float* h = &hi.x;
    float* l = &lo.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t b;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(v[c]));
      h[c] = __uint_as_float(b);
      l[c] = v[c] - h[c];
    }
    *reinterpret_cast<float4*>(static_cast<float*>(p0) + idx) = hi;
    *reinterpret_cast<float4*>(static_cast<float*>(p1) + idx) = lo;
  }
}

// grid: total tiles of the job table, block 256. H, G: the cell's hidden size and gate count.
__global__ void __launch_bounds__(256) k_repack(const RepackJob* __restrict__ jobs, int njobs, int H, int Hp, int G,
                                                int prec) {
  // transpose tile [k][row], rows XOR-swizzled by k / 4: conflict-free both when a warp writes one
  // k (32 rows) and when it reads 4 consecutive k of one row per lane
  __shared__ float tile[kRepackTileK * 32];
  int ji = 0;
  while (ji + 1 < njobs && (int)blockIdx.x >= jobs[ji + 1].tile0) ++ji;
  const RepackJob J = jobs[ji];
  const int tl = (int)blockIdx.x - J.tile0;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const float wsc = pow2f(kWScaleLog2);
  if (J.kind == kRepackB) {
    float* dst = static_cast<float*>(J.p0);
    for (int e = tl * 1024 + tid; e < min(J.K, (tl + 1) * 1024); e += 256) {
      const int g = e / Hp, u = e - g * Hp;
      dst[e] = (u < H && g < G && J.s0) ? J.s0[g * H + u] : 0.0f;
    }
    return;
  }
  const int r0 = (tl / J.tiles_k) * 32, k0 = (tl % J.tiles_k) * kRepackTileK;
  constexpr int kQ = kRepackTileK / 4;  // quads per destination row of a tile
  const long long GH = (long long)G * H;
  if (J.kind == kRepackT) {
    const int g = rho_gate(r0), u = rho_unit(r0) + lane;
    // GRU (G = 3, linear before reset): the candidate gate's two halves go to different slots --
    // W_n in slot 2 of the W columns, R_n in slot 3 of the R columns -- so any kernel that sums
    // [W|R].[x;h] over K keeps W_n x (slot 2) and R_n h (slot 3) apart for the reset gate
    const int gr = G == 3 ? (g == 3 ? 2 : g == 2 ? 3 : g) : g;  // source gate of the R columns
    const bool wok = u < H && g < G, rok = u < H && gr < G && !(G == 3 && g == 2);
#pragma unroll
    for (int i = 0; i < kRepackTileK / 8; ++i) {
      const int kk = w + 8 * i, k = k0 + kk;
      float v = 0.0f;
      if (k < J.k_split) {
        if (wok && k < J.src_k0) v = J.s0[(long long)k * GH + (long long)g * H + u];
      } else if (rok && k - J.k_split < H) {
        v = J.s1[(long long)(k - J.k_split) * GH + (long long)gr * H + u];
      }
      tile[kk * 32 + (lane ^ ((kk >> 2) & 31))] = v;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32 * kQ / 256; ++i) {
      const int idx = tid + 256 * i, r = idx / kQ, q = idx % kQ;
      float v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = tile[(q * 4 + c) * 32 + (r ^ (q & 31))];
      if (k0 + q * 4 < J.K) store4_planes(prec, J.p0, J.p1, (long long)(r0 + r) * J.K + k0 + q * 4, v, wsc);
    }
    return;
  }
  // kRepackC
#pragma unroll
  for (int i = 0; i < 32 * kQ / 256; ++i) {
    const int idx = tid + 256 * i, r = r0 + idx / kQ, k = k0 + (idx % kQ) * 4;
    if (r >= J.rows || k >= J.K) continue;
    const bool second = J.s0 == nullptr || k >= J.src_k0;
    const float* M = second ? J.s1 : J.s0;
    const int rho = second && J.s0 ? k - J.src_k0 : k;
    const int g = rho_gate(rho), up = rho_unit(rho);
    float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (r < J.src_rows && g < G) {
      const float* src = M + (long long)r * GH + (long long)g * H + up;
      if (up + 3 < H && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(src));
        v[0] = f.x;
        v[1] = f.y;
        v[2] = f.z;
        v[3] = f.w;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (up + c < H) v[c] = src[c];
      }
    }
    store4_planes(prec, J.p0, J.p1, (long long)r * J.K + k, v, wsc);
  }
}

// Reference-order padded bias: dst[g*Hp + u] = b[g*H + u].
__global__ void k_pack_bias(const float* __restrict__ b, int H, int Hp, float* dst, int G = 4) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 4 * Hp) return;
  const int g = e / Hp, u = e - g * Hp;
  dst[e] = (u < H && g < G && b) ? b[g * H + u] : 0.0f;
}

// Column-block padding: src is R x (nblk*B) column-major, dst is Rp x (nblk*Bp) starting at
// column dst_col_off. Writes an fp32 copy and/or operand planes (fp16x2: scaled by f16scale).
// `amax` (optional): max |src| over the launch (float bits), the range check of scaled planes.
__global__ void k_pad_cols(const float* __restrict__ src, int R, int B, int nblk, int Rp, int Bp,
                           long long dst_col_off, float* dst_f32, int prec, void* p0, void* p1,
                           float f16scale = 1.0f, unsigned* amax = nullptr) {
  // one column per block iteration, rows across threads: no per-element 64-bit division
  const int ncols = Bp * nblk;
  float mx = 0.0f;
  for (int col = blockIdx.x; col < ncols; col += gridDim.x) {
    const int t = col / Bp, b = col - t * Bp;
    const bool live = src && b < B;
    const float* sc = live ? src + ((long long)t * B + b) * R : nullptr;
    const long long d0 = (dst_col_off + col) * (long long)Rp;
    for (int r = threadIdx.x; r < Rp; r += blockDim.x) {
      const float v = (live && r < R) ? sc[r] : 0.0f;
      mx = fmaxf(mx, fabsf(v));
      if (dst_f32) dst_f32[d0 + r] = v;
      if (p0) store_planes(prec, p0, p1, d0 + r, v, f16scale);
    }
  }
  if (amax) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0.0f) atomicMax(amax, __float_as_uint(mx));
  }
}

// Plain K-major 16-bit operand planes (column c = t*Bp + n holds K contiguous elements) ->
// swizzled step blocks, columns [c0, c0 + ncols). One plane (bf16): block t at t*K*Bp*2 bytes,
// Bp rows per k-block. Two planes (fp16x2 hi, lo): block t at t*K*2Bp*2 bytes, each k-block
// holds the hi rows then the lo rows (2Bp rows), so one bulk copy brings both planes of a
// k-block (rec_cluster.cuh). One thread per 8 consecutive K elements of one plane: they form
// one 16-byte chunk in both layouts (sw_off permutes whole chunks).
__global__ void k_swizzle_op(const uint16_t* __restrict__ s0, const uint16_t* __restrict__ s1, int K, int Bp,
                             long long c0, long long ncols, uint8_t* __restrict__ dst) {
  const int kc = K >> 3;
  const int planes = s1 ? 2 : 1, rows = planes * Bp;
  const long long total = (long long)kc * ncols * planes;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int pl = (int)(e % planes);
    const long long ee = e / planes;
    const long long c = c0 + ee / kc;
    const int k = (int)(ee % kc) << 3;
    const long long t = c / Bp;
    const int n = (int)(c - t * Bp);
    const uint16_t* src = pl ? s1 : s0;
    *reinterpret_cast<uint4*>(dst + t * (long long)K * rows * 2 + sw_off(k, n + pl * Bp, rows)) =
        *reinterpret_cast<const uint4*>(src + c * K + k);
  }
}

// Inverse: dst (G*R x nblk*B) from src (G*Rp x nblk*Bp at src_col_off); G gate blocks.
// Gs: gate blocks per source column (the source's column stride is Gs * Rp; Gs >= G, e.g. the
// 4-slot gates / dG tapes read back with G = 3 for GRU); 0 means G.
__global__ void k_unpad_cols(const float* __restrict__ src, int Rp, int Bp, long long src_col_off,
                             int G, int R, int B, int nblk, float* __restrict__ dst, int Gs = 0) {
  if (Gs == 0) Gs = G;
  const long long rows = (long long)G * R;
  const long long total = rows * B * nblk;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long col = e / rows;
    const int rr = (int)(e - col * rows);
    const int g = rr / R, r = rr - g * R;
    const int t = (int)(col / B), b = (int)(col - (long long)t * B);
    dst[e] = src[(src_col_off + (long long)t * Bp + b) * Gs * Rp + (long long)g * Rp + r];
  }
}

// Plane-wise transpose for the tf32 weight-gradient operands: src is column-major R x C
// (element (r, c) at c*R + r), dst is row-major R x C (element (r, c) at r*C + c), i.e. the
// K-major layout over the time-batch dimension. 32x32 shared-memory tiles, coalesced both ways.
__global__ void k_transpose_planes(const float* __restrict__ s0, const float* __restrict__ s1,
                                   int R, long long C, float* __restrict__ d0,
                                   float* __restrict__ d1) {
  __shared__ float tile[2][32][33];
  const long long c0 = (long long)blockIdx.x * 32;
  const int r0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const long long c = c0 + j;
    const int r = r0 + threadIdx.x;
    if (c < C && r < R) {
      tile[0][j][threadIdx.x] = s0[c * R + r];
      if (s1) tile[1][j][threadIdx.x] = s1[c * R + r];
    }
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = r0 + j;
    const long long c = c0 + threadIdx.x;
    if (c < C && r < R) {
      d0[(long long)r * C + c] = tile[0][threadIdx.x][j];
      if (s1) d1[(long long)r * C + c] = tile[1][threadIdx.x][j];
    }
  }
}

// db[g*H + u] = sum over partial slices (fixed order) of dbp[slice][g*Hp + u].
__global__ void k_db_reduce(const float* __restrict__ dbp, int slices, int H, int Hp, float* db) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 4 * H) return;
  const int g = e / H, u = e - g * H;
  float acc = 0.0f;
  for (int s = 0; s < slices; ++s) acc += dbp[(long long)s * 4 * Hp + g * Hp + u];
  db[e] = acc;
}

// bf16 layer input in one pass: raw x (R x B per step, column-major) -> the padded plain
// K-major operand (Rp x Bp per step) and its pre-swizzled step-block image (sw_off), 8
// consecutive rows (one 16-byte chunk of either layout) per thread.
__global__ void k_pad_swizzle_bf16(const float* __restrict__ src, int R, int B, int T, int Rp, int Bp,
                                   __nv_bfloat16* __restrict__ plain, uint8_t* __restrict__ sw) {
  const int kc = Rp >> 3;
  const long long total = (long long)kc * Bp * T;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long col = e / kc;
    const int k = (int)(e - col * kc) << 3;
    const int t = (int)(col / Bp), b = (int)(col - (long long)t * Bp);
    __align__(16) __nv_bfloat16 v[8];
    const float* sc = src + ((long long)t * B + b) * R;
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __float2bfloat16_rn((b < B && k + j < R) ? sc[k + j] : 0.0f);
    const uint4 q = *reinterpret_cast<const uint4*>(v);
    *reinterpret_cast<uint4*>(plain + col * Rp + k) = q;
    *reinterpret_cast<uint4*>(sw + (long long)t * Rp * Bp * 2 + sw_off(k, b, Bp)) = q;
  }
}

// fp16x2 counterpart of k_pad_swizzle_bf16 (cluster schedule, fp32-parity): the layer-0 input
// x (R x B*T, column-major fp32) -> both scaled operand planes (Rp x Bp*T) and their pre-swizzled
// step image ([hi rows | lo rows] per k-block, as k_swizzle_op writes it) in one pass; records
// max|x| for the range check of the scaled planes.
__global__ void k_pad_swizzle_f16x2(const float* __restrict__ src, int R, int B, int T, int Rp, int Bp,
                                    __half* __restrict__ hi, __half* __restrict__ lo, uint8_t* __restrict__ sw,
                                    float f16scale, unsigned* amax) {
  const int kc = Rp >> 3;
  const long long total = (long long)kc * Bp * T;
  float mx = 0.0f;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long col = e / kc;
    const int k = (int)(e - col * kc) << 3;
    const int t = (int)(col / Bp), b = (int)(col - (long long)t * Bp);
    __align__(16) __half vh[8];
    __align__(16) __half vl[8];
    const float* sc = src + ((long long)t * B + b) * R;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float v = (b < B && k + j < R) ? sc[k + j] : 0.0f;
      mx = fmaxf(mx, fabsf(v));
      f16x2_split(v * f16scale, vh[j], vl[j]);
    }
    const uint4 qh = *reinterpret_cast<const uint4*>(vh), ql = *reinterpret_cast<const uint4*>(vl);
    *reinterpret_cast<uint4*>(hi + col * Rp + k) = qh;
    *reinterpret_cast<uint4*>(lo + col * Rp + k) = ql;
    uint8_t* blk = sw + (long long)t * Rp * Bp * 2 * 2;
    *reinterpret_cast<uint4*>(blk + sw_off(k, b, 2 * Bp)) = qh;
    *reinterpret_cast<uint4*>(blk + sw_off(k, Bp + b, 2 * Bp)) = ql;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0f && amax) atomicMax(amax, __float_as_uint(mx));
}

// All layers' bias-gradient reductions in one launch (blockIdx.y = layer within the group).
constexpr int kDbGroup = 16;
struct DbGroup {
  const float* dbp[kDbGroup];
  float* db[kDbGroup];
};
__global__ void k_db_reduce_layers(DbGroup grp, int slices, int H, int Hp, int G = 4) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G * H) return;
  const float* dbp = grp.dbp[blockIdx.y];
  const int g = e / H, u = e - g * H;
  float acc = 0.0f;
  for (int s = 0; s < slices; ++s) acc += dbp[(long long)s * 4 * Hp + g * Hp + u];
  grp.db[blockIdx.y][e] = acc;
}

// rw_gemm operand packing: dst row r (of Rp), k (of Kp) = op(src)(r, k) -- zero outside the
// rows x K source range -- as K-major operand planes. op(src)(r, k) = src[k * ld + r] when the
// column-major source holds the rows x K operand directly, src[r * ld + k] when it holds its
// transpose (gemm.hpp:339-347's trans flags).
__global__ void k_pack_gemm_operand(const float* __restrict__ src, long long ld, int rows, int K, int trans,
                                    int Rp, int Kp, int prec, void* p0, void* p1) {
  const long long total = (long long)Rp * Kp;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / Kp), k = (int)(e - (long long)r * Kp);
    float v = 0.0f;
    if (r < rows && k < K) v = trans ? src[(long long)r * ld + k] : src[(long long)k * ld + r];
    store_planes(prec, p0, p1, e, v);
  }
}
// C = beta * C (column-major M x N, ldc) ahead of an accumulating GEMM (beta == 0: exact zeros,
// like the reference's beta = 0 overwrite)
__global__ void k_scale_cols(float* __restrict__ c, long long ldc, int M, int N, float beta) {
  const long long total = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / M, i = e - j * M;
    float* p = c + j * ldc + i;
    *p = beta == 0.0f ? 0.0f : beta * *p;
  }
}

// ---- the GPU optimisation ladder's point-wise stage (cells.hpp:261-279 is
// the reference's unfused sequence, cells.hpp:227-260 the fused one). Padded gate-major fp32
// matrices (gate g, unit u at row g*Hp + u), Hp x Bp per gate, column-major.
enum EwOp : int { kEwAdd = 0, kEwAddBias = 1, kEwSigmoid = 2, kEwTanh = 3, kEwMul = 4 };
// dst = op(a, b) over rows x cols (leading dimensions lda / ldb / ldd); kEwAddBias: b is a
// per-row vector; kEwSigmoid / kEwTanh: unary on a. One launch per element-wise op: the
// "Naive" .. "Streamed GEMMs" rungs run the nine-op LSTM sequence as nine launches (K8).
__global__ void k_ew(int op, float* __restrict__ dst, int ldd, const float* __restrict__ a, int lda,
                     const float* __restrict__ b, int ldb, int rows, int cols) {
  const long long total = (long long)rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / rows), r = (int)(e - (long long)c * rows);
    const float x = a[(long long)c * lda + r];
    float v;
    switch (op) {
      case kEwAdd: v = x + b[(long long)c * ldb + r]; break;
      case kEwAddBias: v = x + b[r]; break;
      case kEwSigmoid: v = 1.0f / (1.0f + expf(-x)); break;
      case kEwTanh: v = tanhf(x); break;
      default: v = x * b[(long long)c * ldb + r]; break;
    }
    dst[(long long)c * ldd + r] = v;
  }
}
// Reference-layout gate-major weights (G*H x cols, column-major) -> operand planes with every
// gate block padded to Hp rows (rows g*Hp + u; TMA tiles of one gate then start 128-byte aligned),
// same column-major (MN-major A) orientation -- no transpose: the ladder's "not pre-transposed"
// rungs read these.
__global__ void k_pad_gates(const float* __restrict__ src, int G, int H, int Hp, int cols, int prec, void* p0,
                            void* p1, float f16scale) {
  const long long rows = (long long)G * Hp, total = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / rows;
    const int r = (int)(e - c * rows), g = r / Hp, u = r - g * Hp;
    const float v = u < H ? src[c * G * H + (long long)g * H + u] : 0.0f;
    store_planes(prec, p0, p1, e, v, f16scale);
  }
}
// h (Hp x Bp fp32) -> the operand planes of the next step's GEMM (fp16x2: scaled by 2^kHScaleLog2)
__global__ void k_store_h_operand(const float* __restrict__ h, long long n, int prec, void* p0, void* p1) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    store_planes(prec, p0, p1, e, h[e], pow2f(kHScaleLog2));
}
// "Fused point-wise": the whole LSTM cell of cells.hpp:240-258 (same operation order) in one
// launch: gates from zw + zr + b, c = f c_prev + i c', h = o tanh(c); writes c, h (tapes) and the
// h operand planes.
__global__ void k_lstm_cell_fused(const float* __restrict__ zw, const float* __restrict__ zr,
                                  const float* __restrict__ bias, const float* __restrict__ c_prev,
                                  float* __restrict__ c_out, float* __restrict__ h_out, int H, int Hp, int B,
                                  int prec, void* p0, void* p1, long long op_off) {
  const long long total = (long long)Hp * B;
  const long long G4 = 4LL * Hp;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / Hp), u = (int)(e - (long long)c * Hp);
    float hv = 0.0f, cv = 0.0f;
    if (u < H) {
      const float* w = zw + c * G4;
      const float* r = zr + c * G4;
      const float ai = (w[u] + r[u]) + bias[u];
      const float af = (w[Hp + u] + r[Hp + u]) + bias[Hp + u];
      const float ao = (w[2 * Hp + u] + r[2 * Hp + u]) + bias[2 * Hp + u];
      const float ac = (w[3 * Hp + u] + r[3 * Hp + u]) + bias[3 * Hp + u];
      const float iv = 1.0f / (1.0f + expf(-ai)), fv = 1.0f / (1.0f + expf(-af));
      const float ov = 1.0f / (1.0f + expf(-ao)), cb = tanhf(ac);
      const float t1 = fv * c_prev[e];
      const float t2 = iv * cb;
      cv = t1 + t2;
      hv = ov * tanhf(cv);
    }
    c_out[e] = cv;
    h_out[e] = hv;
    store_planes(prec, p0, p1, op_off + e, hv, pow2f(kHScaleLog2));
  }
}

}  // namespace rw

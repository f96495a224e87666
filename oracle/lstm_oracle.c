/*
 * lstm_oracle.c -- CPU restatement of the rnnwave LSTM path (TEST INFRASTRUCTURE ONLY).
 * See lstm_oracle.h for scope and the reference lines each routine follows.
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile). The loop orders
 * below differ from the reference's tiling but every output element receives the same
 * operation chain, which is what makes the results bitwise comparable.
 */
#include "lstm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- SplitMix64 (rng.hpp:13-48) ---------------------------------------------- */

static uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void rwo_fill_symmetric(uint64_t seed, uint64_t stream, double range, float* out, int64_t n) {
  /* stream k starts at mix(seed + k * golden) (rng.hpp:46-48); each draw advances the
   * state by the golden increment and mixes (rng.hpp:18-23); next_unit keeps the top
   * 53 bits (rng.hpp:26); next_symmetric rounds (2u-1)*range to float once (rng.hpp:29-31). */
  uint64_t state = sm_mix(seed + stream * 0x9E3779B97F4A7C15ull);
  for (int64_t i = 0; i < n; ++i) {
    state += 0x9E3779B97F4A7C15ull;
    const uint64_t z = sm_mix(state);
    const double u = (double)(z >> 11) * 0x1.0p-53;
    out[i] = (float)((2.0 * u - 1.0) * range);
  }
}

static int in_width(const rwo_dims* d, int l) { return l == 0 ? d->input : d->hidden; }

void rwo_init_params(const rwo_dims* d, uint64_t seed, float* const* w, float* const* r) {
  const double range = 1.0 / sqrt((double)d->hidden);
  const int gh = 4 * d->hidden;
  for (int l = 0; l < d->layers; ++l) {
    rwo_fill_symmetric(seed, 2ull * (uint64_t)l, range, w[l], (int64_t)gh * in_width(d, l));
    rwo_fill_symmetric(seed, 2ull * (uint64_t)l + 1ull, range, r[l], (int64_t)gh * d->hidden);
  }
}

void rwo_make_input(const rwo_dims* d, uint64_t seed, float* x) {
  rwo_fill_symmetric(seed, 1000, 1.0, x, (int64_t)d->input * d->batch * d->steps);
}

void rwo_make_dy(const rwo_dims* d, uint64_t seed, float* dy) {
  rwo_fill_symmetric(seed, 1001, 1.0, dy, (int64_t)d->hidden * d->batch * d->steps);
}

int64_t rwo_flop_count_cell(int hidden, int input, int batch) {
  return 2ll * 4 * hidden * ((int64_t)input + hidden) * batch;
}

/* ---- ordered GEMM kernels (gemm.hpp:13-25) ----------------------------------- */

/* C(MxN, ldc) = [C if beta1 else 0] + A(MxK, lda) * B(KxN, ldb); every C(i,j) is one
 * chain over ascending k. The j-k-i loop order keeps that per-element chain (i lanes are
 * independent) while letting the compiler vectorize across i. */
static void gemm_nn(int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                    float* C, int ldc, int beta1) {
  for (int j = 0; j < N; ++j) {
    float* c = C + (size_t)j * ldc;
    if (!beta1) memset(c, 0, sizeof(float) * (size_t)M);
    for (int k = 0; k < K; ++k) {
      const float bkj = B[(size_t)j * ldb + k];
      const float* a = A + (size_t)k * lda;
      for (int i = 0; i < M; ++i) c[i] = c[i] + a[i] * bkj;
    }
  }
}

/* C(MxN) = A(MxK) * B(NxK)^T : the weight-update form gemm(false, true, ...). */
static void gemm_nt(int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                    float* C, int ldc) {
  for (int j = 0; j < N; ++j) {
    float* c = C + (size_t)j * ldc;
    memset(c, 0, sizeof(float) * (size_t)M);
    for (int k = 0; k < K; ++k) {
      const float bjk = B[(size_t)k * ldb + j];
      const float* a = A + (size_t)k * lda;
      for (int i = 0; i < M; ++i) c[i] = c[i] + a[i] * bjk;
    }
  }
}

/* Exact transposed copy (matrix.hpp:159-169): out(c, r) = a(r, c). */
static float* transposed(const float* a, int rows, int cols) {
  float* out = (float*)malloc(sizeof(float) * (size_t)rows * cols);
  for (int c = 0; c < cols; ++c)
    for (int r = 0; r < rows; ++r) out[(size_t)r * cols + c] = a[(size_t)c * rows + r];
  return out;
}

static float sigmoidf_ref(float x) { return 1.0f / (1.0f + expf(-x)); } /* cells.hpp:30 */

/* ---- forward (engine.hpp:82-123, 347-416; cells.hpp:227-260) -------------------- */

int rwo_forward(const rwo_dims* d, const float* const* w, const float* const* r,
                const float* const* b, const float* x, const float* const* h0,
                const float* const* c0, int training, float* const* h_seq, float* const* c_seq,
                float* const* gates_seq, float* const* tanh_c_seq, float* y) {
  const int H = d->hidden, B = d->batch, T = d->steps, G = 4 * H;
  const size_t hcols = (size_t)B * (T + 1);
  float* zw = (float*)malloc(sizeof(float) * (size_t)G * B);
  float* zr = (float*)malloc(sizeof(float) * (size_t)G * B);
  float* g_scr = (float*)malloc(sizeof(float) * (size_t)G * B);
  float* tc_scr = (float*)malloc(sizeof(float) * (size_t)H * B);
  for (int l = 0; l < d->layers; ++l) {
    const int I = in_width(d, l);
    float* hs = h_seq[l];
    float* cs = c_seq[l];
    memset(hs, 0, sizeof(float) * (size_t)H * hcols);
    memset(cs, 0, sizeof(float) * (size_t)H * hcols);
    if (h0 && h0[l]) memcpy(hs, h0[l], sizeof(float) * (size_t)H * B);
    if (c0 && c0[l]) memcpy(cs, c0[l], sizeof(float) * (size_t)H * B);
    /* pretranspose (params.hpp:55-61) is an exact copy, so the products are W(i,k) x. */
    for (int t = 0; t < T; ++t) {
      /* layer_input_cols (engine.hpp:333-340): x block t, or h_{l-1} block t+1. */
      const float* xin = l == 0 ? x + (size_t)t * B * I : h_seq[l - 1] + (size_t)(t + 1) * B * H;
      gemm_nn(G, B, I, w[l], G, xin, I, zw, G, 0);                       /* input_gemm */
      gemm_nn(G, B, H, r[l], G, hs + (size_t)t * B * H, H, zr, G, 0);      /* recurrent_gemm */
      const float* bias = b[l];
      float* gdst = training && gates_seq ? gates_seq[l] + (size_t)t * B * G : g_scr;
      float* tdst = training && tanh_c_seq ? tanh_c_seq[l] + (size_t)t * B * H : tc_scr;
      for (int c = 0; c < B; ++c) {
        const float* pzw = zw + (size_t)c * G;
        const float* pzr = zr + (size_t)c * G;
        const float* pcp = cs + ((size_t)t * B + c) * H;
        float* pc = cs + ((size_t)(t + 1) * B + c) * H;
        float* ph = hs + ((size_t)(t + 1) * B + c) * H;
        float* pg = gdst + (size_t)c * G;
        float* ptc = tdst + (size_t)c * H;
        for (int u = 0; u < H; ++u) {
          const float ai = (pzw[u] + pzr[u]) + bias[u];
          const float af = (pzw[H + u] + pzr[H + u]) + bias[H + u];
          const float ao = (pzw[2 * H + u] + pzr[2 * H + u]) + bias[2 * H + u];
          const float ac = (pzw[3 * H + u] + pzr[3 * H + u]) + bias[3 * H + u];
          const float iv = sigmoidf_ref(ai);
          const float fv = sigmoidf_ref(af);
          const float ov = sigmoidf_ref(ao);
          const float cb = tanhf(ac);
          const float t1 = fv * pcp[u];
          const float t2 = iv * cb;
          const float cv = t1 + t2;
          const float tcv = tanhf(cv);
          pg[u] = iv;
          pg[H + u] = fv;
          pg[2 * H + u] = ov;
          pg[3 * H + u] = cb;
          pc[u] = cv;
          ptc[u] = tcv;
          ph[u] = ov * tcv;
        }
      }
    }
  }
  if (y) memcpy(y, h_seq[d->layers - 1] + (size_t)B * H, sizeof(float) * (size_t)H * B * T);
  free(zw);
  free(zr);
  free(g_scr);
  free(tc_scr);
  return 0;
}

/* ---- backward_data (engine.hpp:128-172, 507-585; cells.hpp:409-449) ------------- */

int rwo_backward_data(const rwo_dims* d, const float* const* w, const float* const* r,
                      const float* const* h_seq, const float* const* c_seq,
                      const float* const* gates_seq, const float* const* tanh_c_seq,
                      const float* dy, float* const* dgw_seq, float* dx0, float* const* dh0,
                      float* const* dc0) {
  const int H = d->hidden, B = d->batch, T = d->steps, G = 4 * H, L = d->layers;
  const size_t bt = (size_t)B * T;
  float* carry_h = (float*)malloc(sizeof(float) * (size_t)H * B);
  float* carry_c = (float*)malloc(sizeof(float) * (size_t)H * B);
  /* dout_seq_[l-1] = d(input of layer l) (engine.hpp:318-319) */
  float* d_below = (float*)calloc((size_t)H * bt, sizeof(float));
  float* d_cur = (float*)calloc((size_t)H * bt, sizeof(float));
  for (int l = L - 1; l >= 0; --l) {
    const int I = in_width(d, l);
    const float* da_seq = l == L - 1 ? dy : d_cur;
    float* dst_seq = l == 0 ? dx0 : d_below;
    float* rt = transposed(r[l], G, H); /* rt (H x G): exact copy, gemm(false,false,rt,...) */
    float* wt = transposed(w[l], G, I);
    memset(carry_h, 0, sizeof(float) * (size_t)H * B);
    memset(carry_c, 0, sizeof(float) * (size_t)H * B);
    const float* gs = gates_seq[l];
    const float* tcs = tanh_c_seq[l];
    const float* cs = c_seq[l];
    for (int t = T - 1; t >= 0; --t) {
      float* dg = dgw_seq[l] + (size_t)t * B * G;
      for (int c = 0; c < B; ++c) {
        const float* pda = da_seq + ((size_t)t * B + c) * H;
        const float* pg = gs + ((size_t)t * B + c) * G;
        const float* ptc = tcs + ((size_t)t * B + c) * H;
        const float* pcp = cs + ((size_t)t * B + c) * H;
        float* pcar = carry_h + (size_t)c * H;
        float* pdci = carry_c + (size_t)c * H;
        float* pdg = dg + (size_t)c * G;
        for (int u = 0; u < H; ++u) {
          const float pi = pg[u], pf = pg[H + u], po = pg[2 * H + u], pcb = pg[3 * H + u];
          const float dh = pda[u] + pcar[u];
          const float q1 = dh * po;
          const float s = ptc[u] * ptc[u];
          const float s1 = 1.0f - s;
          const float q2 = q1 * s1;
          const float dc = pdci[u] + q2;
          const float a1 = dc * pcb;
          const float a2 = a1 * pi;
          const float a3 = 1.0f - pi;
          const float b1 = dc * pcp[u];
          const float b2 = b1 * pf;
          const float b3 = 1.0f - pf;
          const float c1 = dh * ptc[u];
          const float c2 = c1 * po;
          const float c3 = 1.0f - po;
          const float d1 = dc * pi;
          const float d2 = pcb * pcb;
          const float d3 = 1.0f - d2;
          pdg[u] = a2 * a3;
          pdg[H + u] = b2 * b3;
          pdg[2 * H + u] = c2 * c3;
          pdg[3 * H + u] = d1 * d3;
          pdci[u] = dc * pf; /* carry_c <- dc o f */
          pcar[u] = 0.0f;    /* carry_h <- 0 (dh_local for LSTM) */
        }
      }
      /* recurrent_backward_gemm: carry_h += R^T dG_t (beta 1 onto the zeroed carry). */
      gemm_nn(H, B, G, rt, H, dg, G, carry_h, H, 1);
      /* output_gemm: d(input)_t = W^T dG_t (beta 0). */
      gemm_nn(I, B, G, wt, I, dg, G, dst_seq + (size_t)t * B * I, I, 0);
    }
    if (dh0 && dh0[l]) memcpy(dh0[l], carry_h, sizeof(float) * (size_t)H * B);
    if (dc0 && dc0[l]) memcpy(dc0[l], carry_c, sizeof(float) * (size_t)H * B);
    free(rt);
    free(wt);
    float* tmp = d_cur;
    d_cur = d_below;
    d_below = tmp;
  }
  free(carry_h);
  free(carry_c);
  free(d_below);
  free(d_cur);
  return 0;
}

/* ---- weight_update (engine.hpp:178-217; cells.hpp:163-168) ----------------------- */

int rwo_weight_update(const rwo_dims* d, const float* x, const float* const* h_seq,
                      const float* const* dgw_seq, float* const* dw, float* const* dr,
                      float* const* db) {
  const int H = d->hidden, B = d->batch, T = d->steps, G = 4 * H;
  const int bt = B * T;
  for (int l = 0; l < d->layers; ++l) {
    const int I = in_width(d, l);
    const float* xl = l == 0 ? x : h_seq[l - 1] + (size_t)B * H; /* layer_input_all */
    gemm_nt(G, I, bt, dgw_seq[l], G, xl, I, dw[l], G);
    gemm_nt(G, H, bt, dgw_seq[l], G, h_seq[l], H, dr[l], G); /* h_{t-1} columns [0, BT) */
    float* dbl = db[l];
    memset(dbl, 0, sizeof(float) * (size_t)G);
    for (int c = 0; c < bt; ++c) {
      const float* s = dgw_seq[l] + (size_t)c * G;
      for (int rr = 0; rr < G; ++rr) dbl[rr] += s[rr];
    }
  }
  return 0;
}

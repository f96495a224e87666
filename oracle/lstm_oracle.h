/*
 * lstm_oracle.h -- CPU restatement of the rnnwave LSTM path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the B200 path, never the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. The product
 * library (librnnwave_sm100.so) never links or calls anything under oracle/.
 *
 * It restates, in plain C, the reference engine's single-precision arithmetic for
 * CellKind::Lstm (the north-star path), element by element and in the same order:
 *   - GEMM contract: accumulator starts at 0 (beta=0) or at C (beta=1), products
 *     added one at a time in ascending k, one multiply + one add, no FMA
 *     (reference proj/include/rnnwave/gemm.hpp:13-25, gemm_scalar 138-155).
 *   - fused LSTM forward cell chain (cells.hpp:227-260, sigmoid at cells.hpp:30).
 *   - fused LSTM backward cell chain (cells.hpp:409-449).
 *   - Engine forward / backward_data / weight_update data flow
 *     (engine.hpp:82-217, 333-585).
 *   - SplitMix64 streams and init_params (rng.hpp:13-48, params.hpp:31-51),
 *     verify::random_matrix / make_input / make_dy (verify.hpp:27-44).
 * Compiled with -ffp-contract=off (reference CMakeLists.txt:21), so on the same host
 * libm it is bitwise equal to the reference engine; tests/test_oracle_golden.py pins
 * that against golden vectors produced by the reference itself (tests/golden/).
 *
 * All matrices are column-major float, leading dimension == rows, exactly as the
 * reference Matrix (matrix.hpp:16-68). Sequences are time-major: a layer's hidden
 * history is H x B*(T+1) with column block 0 the initial state (engine.hpp:32-34).
 */
#ifndef RNNWAVE_LSTM_ORACLE_H
#define RNNWAVE_LSTM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int layers;
  int hidden; /* H */
  int input;  /* I (layer-0 input width; deeper layers take H) */
  int batch;  /* B */
  int steps;  /* T */
} rwo_dims;

/* SplitMix64 uniform float in [-range, range] drawn from stream `stream` of `seed`,
 * filling `n` values in order (rng.hpp:26-48). */
void rwo_fill_symmetric(uint64_t seed, uint64_t stream, double range, float* out, int64_t n);

/* init_params (params.hpp:31-51): W_l from stream 2l, R_l from stream 2l+1,
 * U[-1/sqrt(H), 1/sqrt(H)], biases are left to the caller (reference: zero). */
void rwo_init_params(const rwo_dims* d, uint64_t seed, float* const* w, float* const* r);

/* verify::make_input / make_dy (verify.hpp:38-44): streams 1000 and 1001. */
void rwo_make_input(const rwo_dims* d, uint64_t seed, float* x);
void rwo_make_dy(const rwo_dims* d, uint64_t seed, float* dy);

/* FLOP convention of the reference bench (cells.hpp:65-68, bench.hpp:55-62). */
int64_t rwo_flop_count_cell(int hidden, int input, int batch);

/* Training/inference forward (engine.hpp:82-123). Per layer l:
 *   w[l]: 4H x I_l, r[l]: 4H x H, b[l]: 4H
 *   h0[l], c0[l]: H x B or NULL (NULL array == zeros)
 * Outputs per layer: h_seq[l], c_seq[l]: H x B(T+1); if training, gates_seq[l]
 * (4H x BT post-activations) and tanh_c_seq[l] (H x BT). y: H x BT.
 * Any output array may be NULL if not wanted, except h_seq/c_seq which the
 * recurrence needs (caller provides them). Returns 0. */
int rwo_forward(const rwo_dims* d, const float* const* w, const float* const* r,
                const float* const* b, const float* x, const float* const* h0,
                const float* const* c0, int training, float* const* h_seq, float* const* c_seq,
                float* const* gates_seq, float* const* tanh_c_seq, float* y);

/* backward_data (engine.hpp:128-172, 507-585): consumes the training tape and dy
 * (H x BT); writes dgw_seq[l] (4H x BT), dx0 (I x BT), dh0[l], dc0[l] (H x B). */
int rwo_backward_data(const rwo_dims* d, const float* const* w, const float* const* r,
                      const float* const* h_seq, const float* const* c_seq,
                      const float* const* gates_seq, const float* const* tanh_c_seq,
                      const float* dy, float* const* dgw_seq, float* dx0, float* const* dh0,
                      float* const* dc0);

/* weight_update (engine.hpp:178-217): dW_l = dG_l X_l^T, dR_l = dG_l Hprev_l^T,
 * db_l = row sums of dG_l, K = B*T accumulated in ascending time order. */
int rwo_weight_update(const rwo_dims* d, const float* x, const float* const* h_seq,
                      const float* const* dgw_seq, float* const* dw, float* const* dr,
                      float* const* db);

#ifdef __cplusplus
}
#endif

#endif

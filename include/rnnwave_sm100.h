/*
 * rnnwave_sm100.h -- C-ABI of librnnwave_sm100.so, the B200 (sm_100a) implementation of the
 * rnnwave multi-layer LSTM forward/backward path.
 *
 * This is the drop-in boundary under the reference's C++ API. Each entry point replaces one
 * piece of the reference interface (paths relative to /root/reference/proj/include/rnnwave):
 *
 *   rw_create / rw_destroy      <- Engine::Engine(const LadderConfig&)       engine.hpp:71-75
 *                                  (validation: LadderConfig::validate      config.hpp:74-96)
 *   rw_set_params               <- the std::vector<LayerParams>& argument of forward /
 *                                  backward_data (params.hpp:18-25) + pretranspose
 *                                  (params.hpp:55-61) -> device repack, once per upload
 *   rw_forward                  <- Engine::forward                          engine.hpp:82-123
 *   rw_backward_data            <- Engine::backward_data                    engine.hpp:128-172
 *   rw_weight_update            <- Engine::weight_update                    engine.hpp:178-217
 *   rw_get_tape                 <- ForwardTape / BackwardState fields        engine.hpp:36-60
 *   rw_flop_count_cell          <- flop_count                                cells.hpp:65-68
 *   rw_run_pass / rw_upload_*   device-resident timed path (bench::time_level
 *                                  run_once, bench.hpp:141-159)
 *
 * Conventions: plain pointers and sizes, no torch/STL types. Host matrices are fp32
 * column-major exactly like rnnwave::Matrix (element (r, c) at c*rows + r). Per-layer
 * arrays are passed as `const float* const*` with `layers` entries. Every call returns an
 * rw_status; on error rw_last_error(ctx) holds the message. Messages mirror the reference
 * exceptions (substrings "expected", "training", "stale tape" -- test_engine.cpp:220-256).
 * Host-pointer entry points are synchronous. A context is not re-entrant (like Engine,
 * SPEC.md:251): use one per host thread.
 */
#ifndef RNNWAVE_SM100_H
#define RNNWAVE_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rw_ctx rw_ctx;

typedef enum {
  RW_OK = 0,
  RW_EINVAL = 1, /* bad argument / shape / call order   -> std::invalid_argument */
  RW_ECUDA = 2,  /* CUDA runtime or kernel failure       -> std::runtime_error   */
  RW_ENOMEM = 3, /* device allocation failed             -> std::runtime_error   */
  RW_ENCCL = 4,  /* collective failure                   -> std::runtime_error   */
  RW_ESTATE = 5  /* e.g. persistent-kernel timeout       -> std::runtime_error   */
} rw_status;

typedef enum {
  RW_PREC_BF16 = 0,     /* bf16 tensor-core operands, fp32 accumulate + fp32 cell math   */
  RW_PREC_FP32 = 1      /* fp32-parity (normwise <= 1e-5 vs the fp32 reference): split
                           operands, fp32 accumulate + accurate fp32 cell math. The operand
                           format is chosen per shape: fp16x2 (hi + lo fp16 planes, 3 MMAs
                           per product) on the cluster schedule, 3xTF32 elsewhere
                           (rw_describe_precision) */
} rw_precision;

/* Operand format a context computes in (rw_describe_precision). */
typedef enum {
  RW_FMT_BF16 = 0,
  RW_FMT_TF32X3 = 1,
  RW_FMT_FP16X2 = 2
} rw_operand_format;

typedef enum {
  RW_SCHED_AUTO = 0,       /* cluster, else persistent, else stepwise: the first that fits */
  RW_SCHED_STEPWISE = 1,   /* one fused kernel per (layer, step), CUDA-graph wavefront    */
  RW_SCHED_PERSISTENT = 2, /* one kernel per pass, resident weights, flag wavefront       */
  RW_SCHED_CLUSTER = 3,    /* persistent with split roles per tile: off-critical W.x /
                              W^T.dG members run ahead, partials exchanged by DSMEM bulk
                              copies (bf16, batch <= 64, hidden <= 512 per member slice) */
  RW_SCHED_LAYERSEQ = 4    /* large hidden sizes: layer by layer, the input projections of all
                              steps as one tcgen05 GEMM per layer (W.X_l; backward W_{l+1}^T.dG),
                              then one fused recurrent-step kernel per step (R.h / R^T.dG only) */
} rw_schedule;

/* Mirrors LadderConfig (config.hpp:49-97) plus the device knobs. */
typedef struct {
  int layers;
  int hidden;
  int input;
  int batch;
  int steps;
  int cell_kind;   /* CellKind: 0 RnnTanh, 1 RnnRelu, 2 Gru, 3 Lstm (config.hpp:12); all cell kinds run
                     on every schedule */
  int opt_level;   /* validated 0..6 for API compatibility; selects no alternate path */
  int batch_steps; /* validated (1..steps) like the reference */
  int workers;     /* validated > 0; unused on the device */
  uint64_t seed;
  int precision;   /* rw_precision */
  int schedule;    /* rw_schedule */
} rw_config;

typedef enum {
  RW_TAPE_X0 = 0,     /* I x B*T          (layer ignored) */
  RW_TAPE_H = 1,      /* H x B*(T+1)      per layer       */
  RW_TAPE_C = 2,      /* H x B*(T+1)      per layer       */
  RW_TAPE_GATES = 3,  /* 4H x B*T         per layer (i,f,o,c' post-activations) */
  RW_TAPE_TANH_C = 4, /* H x B*T          per layer       */
  RW_TAPE_DGW = 5,    /* G*H x B*T        per layer (BackwardState::dgw_seq) */
  RW_TAPE_Y = 6,      /* H x B*T          (layer ignored) */
  RW_TAPE_ZRH = 7,    /* H x B*T          per layer, GRU (ForwardTape::zrh_seq) */
  RW_TAPE_DGR = 8     /* G*H x B*T        per layer, GRU (BackwardState::dgr_seq) */
} rw_tape;

/* Validates like LadderConfig::validate; allocates every device buffer for the config. */
int rw_create(const rw_config* cfg, int device, rw_ctx** out);
void rw_destroy(rw_ctx* ctx);
const char* rw_last_error(const rw_ctx* ctx);
/* Static error text when rw_create itself fails (no context). */
const char* rw_create_error(void);

/* Layer parameters in the reference layout: W (4H x I_l), R (4H x H), b (4H, may be NULL =
 * zeros). Host pointers; triggers the device repack for that layer. */
int rw_set_params(rw_ctx* ctx, int layer, const float* W, const float* R, const float* b);

/* Engine::forward. x: I x B*T host. h0/c0: NULL or `layers` host pointers of H x B.
 * y: H x B*T host output (may be NULL). training != 0 records the tape for backward.
 * Returns the tape generation id in *tape_id (may be NULL). */
int rw_forward(rw_ctx* ctx, const float* x, int training, const float* const* h0,
               const float* const* c0, float* y, uint64_t* tape_id);

/* Engine::backward_data on tape `tape_id` (must be the context's latest training tape).
 * dy: H x B*T host. dx0: I x B*T. dh0/dc0: `layers` pointers of H x B (any may be NULL). */
int rw_backward_data(rw_ctx* ctx, uint64_t tape_id, const float* dy, float* dx0,
                     float* const* dh0, float* const* dc0);

/* Engine::weight_update: dW (4H x I_l), dR (4H x H), db (4H) per layer (NULL = skip). */
int rw_weight_update(rw_ctx* ctx, uint64_t tape_id, float* const* dW, float* const* dR,
                     float* const* db);

/* Materialise one tape tensor (reference layout, unpadded) into a host buffer. */
int rw_get_tape(rw_ctx* ctx, int which, int layer, float* host);

/* ---- device-resident timed path (bench) ---- */
/* Upload the synthetic x (I x B*T) and dy (H x B*T) once (host pointers). */
int rw_upload_inputs(rw_ctx* ctx, const float* x, const float* dy);
/* One pass on the device, inputs already resident: 0 = forward (inference), 1 = backward
 * (backward_data + weight_update on the resident tape), 2 = both (training forward +
 * backward_data + weight_update), 3 = forward recording a training tape (a later pass 1
 * completes it). Enqueued on `stream` (cudaStream_t; NULL = the context's own stream) and
 * returns without synchronising. */
int rw_run_pass(rw_ctx* ctx, int pass, void* stream);
/* The device copy of the parameters was modified in place (as an optimizer step on the device
 * does): the next pass re-runs the K7 repack inside its own stream work, like the reference's
 * per-pass pretranspose (engine.hpp:92, 138). bench.py calls it before every timed pass. */
int rw_params_updated(rw_ctx* ctx);
/* One training step end to end with host buffers -- the public call a training loop makes:
 * upload x and dy, forward + backward_data + weight_update, read back y, dx0, dW, dR, db (any
 * output may be NULL). Asynchronous and pipelined: the next step's uploads overlap this
 * step's compute and this step's read-back overlaps the next step's compute (pinned host
 * memory for full DMA rate). Host outputs are complete after rw_train_wait; inputs must stay
 * unchanged until the step's upload ran (rw_train_wait, or the next-but-one step). */
int rw_train_step(rw_ctx* ctx, const float* x, const float* dy, float* y, float* dx0,
                  float* const* dW, float* const* dR, float* const* db);
int rw_train_wait(rw_ctx* ctx);
/* Wait for the context's work; reports kernel faults / persistent-kernel timeouts. */
int rw_sync(rw_ctx* ctx);
/* Enable per-phase CUDA-event timing of rw_run_pass (0 = off). When on, rw_phase_times
 * returns the accumulated milliseconds and launch counts of the phases since the last reset:
 * out_ms[0..5] = {repack/convert, fwd recurrent, bwd recurrent, weight-grad GEMMs,
 * dx0 GEMM, db reduce}; out_launches likewise. */
int rw_set_profiling(rw_ctx* ctx, int on);
int rw_phase_times(rw_ctx* ctx, double* out_ms, int* out_launches, int n, int reset);
/* The schedule the context actually uses for forward/backward (rw_schedule values), and the
 * split-K factors chosen. */
int rw_describe(rw_ctx* ctx, int* fwd_sched, int* bwd_sched, int* fwd_ksplit, int* bwd_ksplit);
/* Kernel variants chosen: pairs bit 0 = the stepwise forward, bit 1 = the persistent backward
 * run as CTA pairs (tcgen05 cta_group::2, M = 256); bits 2 / 3 = the layer-sequential forward /
 * backward run one persistent launch per layer; wgrad_bn = N tile of the weight-gradient GEMMs
 * (256 = pairs). */
int rw_describe_variants(rw_ctx* ctx, int* pairs, int* wgrad_bn);

/* The operand format (rw_operand_format) the context's tensor-core GEMMs use. */
int rw_describe_precision(rw_ctx* ctx, int* fmt);

/* Copy the results of the last rw_run_pass to host buffers (any may be NULL): y (H x B*T),
 * dx0 (I x B*T), dW / dR / db per layer (reference layouts). Synchronous. */
int rw_read_outputs(rw_ctx* ctx, float* y, float* dx0, float* const* dW, float* const* dR,
                    float* const* db);
/* Number of kernels this library launched since the last reset (graph-free accounting). */
int rw_launch_count(rw_ctx* ctx, long long* count, int reset);

/* ---- data parallel over NVLink/NVSwitch (config E) ----
 * Independent sequences are split by minibatch across ranks (one context per GPU, each with
 * its own batch); the only exchange is a sum all-reduce of dW/dR/db after weight_update.
 * NCCL is loaded at run time (libnccl.so.2), so the library itself has no NCCL dependency.
 * rw_nccl_unique_id: rank 0 creates the 128-byte id and shares it out of band. */
int rw_nccl_unique_id(char* id128);
int rw_comm_init(rw_ctx* ctx, int nranks, int rank, const char* id128);
/* Sum all-reduce of every layer's dW, dR, db on `stream` (NULL = context stream), one NCCL
 * group, enqueued after the pass's weight-gradient GEMMs. */
int rw_allreduce_grads(rw_ctx* ctx, void* stream);
/* Overlapped gradient sums (on = 1): every later backward pass all-reduces each layer's bucket
 * (dW_l, dR_l, db_l) inside the pass on a communication stream as soon as that layer's
 * weight-gradient GEMMs finish (top layer first), overlapping the lower layers' GEMMs and the
 * dx0 GEMM; rw_allreduce_grads then has nothing left to do. */
int rw_comm_overlap(rw_ctx* ctx, int on);

/* ---- layer pipeline over NVLink (config E; SURVEY §8e "deep stacks split as a layer
 * pipeline that hands off h_t per timestep peer-to-peer") ----
 * Stage k is an ordinary context holding layers [l_k, l_k + L_k) (cfg.input = H for k > 0).
 * Forward: stage k's last layer writes each h_t (the bf16 operand image, H x B x 2 bytes per
 * step) straight into stage k+1's layer-input image over NVLink and releases a system-scope
 * per-step counter; stage k+1's first layer then runs exactly as on one GPU. Backward: the
 * cluster schedule's off-critical group of stage k+1's first layer (W^T . dG_t, which does not
 * depend on stage k's recurrence) runs on stage k+1 and writes its per-step partial sums into
 * stage k's last-layer ring. After its forward, stage k also copies its last layer's h sequence
 * into stage k+1's plain layer-input planes (for stage k+1's dW of its first layer).
 * That is the cluster schedule (mode 0). On the persistent / stepwise schedules (mode 1, config
 * E) stage k's last layer stores h_t into stage k+1's plain layer-input planes, stage k+1's first
 * layer stores its dG_t into stage k's dG-input planes, and stage k's top layer multiplies them
 * by W_next^T (stage k+1's W_0, exported as region 3 of the forward descriptor) -- each with a
 * system-scope per-step counter; a stage below the last then needs >= 2 layers. Any cell kind;
 * bf16 or fp32-parity operands; both stages of a link in the same family. Exported descriptors carry CUDA
 * IPC handles (cross-process) and raw pointers (same-process stages, tests). */
typedef struct {
  char handle[5][64];     /* cudaIpcMemHandle_t of the regions. mode 0 (cluster): dir 0: input
                             image / per-step input counters / lo plane of the plain layer input
                             / plain layer-input planes / input-ready counter; dir 1: ring data /
                             done / consumed. mode 1 (persistent / stepwise): dir 0: layer-input
                             plane 0 / per-step counters (+ senders per step at [T]) / plane 1 /
                             W_0 (reference layout) / input-ready counter; dir 1: dG-input
                             plane 0 / per-step counters / plane 1 */
  uint64_t offset[5];     /* byte offset of the region inside each exported allocation */
  uint64_t ptr[5];        /* device pointers in the exporting process */
  int64_t pid;            /* exporting process */
  int device;             /* exporting device */
  int ko;                 /* off members the ring expects per step */
  int mode;               /* schedule family of the exporting stage: 0 cluster, 1 persistent /
                             stepwise (both stages of a link must agree) */
} rw_pp_ring;
/* dir 0: my layer-input image, its per-step counters and my plain layer-input buffer; dir 1:
 * the backward ring of my last layer. */
int rw_pp_export(rw_ctx* ctx, int dir, rw_pp_ring* out);
/* dir 0: link to the NEXT stage's forward export (W_next: the next stage's first-layer W in the
 * reference layout -- cluster: unused; persistent / stepwise: NULL = read it from the export).
 * dir 1: link to the PREVIOUS stage's backward export. */
int rw_pp_link(rw_ctx* ctx, int dir, const rw_pp_ring* peer, const float* W_next);
/* After the next stage's parameters changed: cluster -- nothing to refresh (the forward hand-off
 * sends h_t); persistent / stepwise -- re-pack W_next (optionally from a new pointer) into the
 * top layer's backward image on the next pass. Validates that a forward link exists. */
int rw_pp_set_next_w(rw_ctx* ctx, const float* W_next);

/* cells.hpp:65-68: 2 * 4 * H * (I + H) * B multiply-add FLOPs per cell. */
/* The GPU optimisation ladder (the reference's run_ladder, bench.hpp:30-32, 176-224): one
 * inference forward pass of rung `level` 0..4 -- 0 naive (per-gate GEMMs on the reference-layout
 * weights + the nine element-wise ops as nine launches), 1 grouped GEMMs, 2 streamed GEMMs (W.x
 * on a second stream), 3 fused point-wise, 4 pre-transposed fused step kernels, layers in
 * sequence. Rungs 5 / 6 are rw_run_pass on contexts with the layer-sequential / automatic
 * schedule. The context must use the stepwise schedule and LSTM cells. */
int rw_ladder_pass(rw_ctx* ctx, int level, void* stream);

/* gemm (gemm.hpp:339-347, the reference's ordered fp32 GEMM) on the device: C (M x N) =
 * alpha op(A) op(B) + beta C, host column-major buffers, op(X) = X^T when trans_x; 3xTF32 split
 * operands on the tcgen05 tensor cores (fp32-parity, not bitwise equal to the CPU chain).
 * Synchronous. */
int rw_gemm(int trans_a, int trans_b, int M, int N, int K, float alpha, const float* A, long long lda,
            const float* B, long long ldb, float beta, float* C, long long ldc);

/* ---- the free pointwise stage (cells.hpp:181-333 pointwise_forward, 349-562
 * pointwise_backward) on the device, synchronous. Host buffers, dense column-major (ld = rows):
 * zw, zr, gates, dgw, dgr are G*H x B (G = gate count of `kind`), the rest H x B, bias G*H.
 * `fused` selects the reference's fused / kernel-per-op mode; the reference defines the two
 * bitwise identical and the device runs one kernel for both. Forward: c_prev / c_out for LSTM
 * only; gates, tanh_c (LSTM), zr_h (GRU) may be NULL (inference: nothing saved; the RNN kinds
 * save nothing -- their saved state is h_out). Backward: `gates` is the saved gates (the
 * post-activation h for the RNN kinds), dgr GRU only (distinct from dgw), dc_carry / dc_prev
 * LSTM only, db optional (G*H, += row sums of dgw in ascending column order). */
int rw_pointwise_forward(int kind, int fused, int hidden, int batch, const float* zw, const float* zr,
                         const float* bias, const float* h_prev, const float* c_prev, float* h_out, float* c_out,
                         float* gates, float* tanh_c, float* zr_h);
int rw_pointwise_backward(int kind, int fused, int hidden, int batch, const float* gates, const float* tanh_c,
                          const float* zr_h, const float* h_prev, const float* c_prev, const float* d_above,
                          const float* dh_carry, const float* dc_carry, float* dgw, float* dgr, float* dh_local,
                          float* dc_prev, float* db);

/* ---- schedule trace (Engine::set_trace_sink, engine.hpp:79-80; sched::TraceRecord,
 * scheduler.hpp:180-192). rw_trace_enable(ctx, 1) makes the recurrent kernels record
 * %globaltimer stamps; rw_trace_records returns the last pass's tasks of one direction (0
 * forward, 1 backward) in the reference's task model with block width 1: task ids of
 * build_graph(L, T, 1), phase 0 = INPUT_GEMM, 1 = RECURRENT_STEP, ns relative to the first
 * record. *count receives the number of records (copies at most `capacity`). */
typedef struct rw_trace_record {
  int32_t task_id, layer, block, step_k, phase, worker;
  int64_t start_ns, end_ns;
} rw_trace_record;
int rw_trace_enable(rw_ctx* ctx, int on);
int rw_trace_records(rw_ctx* ctx, int direction, rw_trace_record* out, int capacity, int* count);

int64_t rw_flop_count_cell(int hidden, int input, int batch);

/* ---- unit-test hook: one tcgen05 GEMM on device pointers ----
 * D (M x N, fp32, column-major, ldd) = A * B^T where A is M x K and B is N x K.
 * a_mn_major=0: A stored K-major (element (m,k) at m*lda + k); 1: MN-major (k*lda + m).
 * Likewise B. Operands are fp32 on the device and converted to the precision's operand
 * planes internally. M, N, K must be multiples of 128/64/64. */
int rw_test_gemm(int precision, int a_mn_major, int b_mn_major, int M, int N, int K,
                 const float* dA, long long lda, const float* dB, long long ldb, float* dD,
                 long long ldd, int bn);

/* Average device time (ms) of the last rw_test_gemm call's GEMM kernel; with the environment
 * variable RW_TEST_GEMM_REPS=n the kernel is repeated n times after one warm-up. */
float rw_test_gemm_last_ms(void);

#ifdef __cplusplus
}
#endif

#endif

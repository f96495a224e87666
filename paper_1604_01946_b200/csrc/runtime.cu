// runtime.cu -- librnnwave_sm100.so: device context, buffers, TMA descriptors, schedule
// selection (persistent wavefront vs. stepwise CUDA-graph wavefront), and the C-ABI of
// include/rnnwave_sm100.h. Replaces the reference Engine internals (engine.hpp:219-665),
// scheduler.hpp (wavefront executor) and thread_pool.hpp ("streams") with device-side
// equivalents; the arithmetic lives in lstm_step.cuh / gemm_tc.cuh / layout_kernels.cuh.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>

#include <chrono>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/rnnwave_sm100.h"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "layout_kernels.cuh"
#include "lstm_step.cuh"
#include "pointwise.cuh"
#include "kernel_ptrs.h"
#include "rec_cluster.cuh"
#include "sync_kernels.cuh"

using namespace rw;

namespace {

// ------------------------------------------------------------------ errors
struct RwError {
  int code;
  std::string msg;
};

#define RW_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw RwError{e_ == cudaErrorMemoryAllocation ? RW_ENOMEM : RW_ECUDA,              \
                    std::string(#call) + ": " + cudaGetErrorString(e_)};                  \
  } while (0)

[[noreturn]] void einval(const std::string& m) { throw RwError{RW_EINVAL, m}; }

// Kernel launches issued by this library (per host thread), for the bench's gpu_launches.
thread_local long long g_launches = 0;

// ------------------------------------------------------------------ TMA encode (driver API)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    RW_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw RwError{RW_ECUDA, "cuTensorMapEncodeTiled unavailable"};
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D row-major tensor: `inner` contiguous elements per row, `outer` rows, box {bi, bo},
// SWIZZLE_128B, OOB zero fill.
// K-major GEMM operand boxes are at most 128 rows; OperandTile::load issues one box per 128 rows
// (k_gemm_p2 loads half a 256-column B tile per CTA with the same map)
inline int gemm_box_rows(int rows) { return rows < 128 ? rows : 128; }

CUtensorMap make_map(const void* base, int prec, long long inner, long long outer, int bi, int bo) {
  CUtensorMap m;
  const int elem = prec_elem(prec);
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(inner * elem)};
  cuuint32_t box[2] = {(cuuint32_t)bi, (cuuint32_t)bo};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m,
                           prec == kBF16    ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                           : prec == kF16x2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                            : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char b[256];
    snprintf(b, sizeof b, "cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld box=%dx%d",
             (int)r, inner, outer, bi, bo);
    throw RwError{RW_ECUDA, b};
  }
  return m;
}

// ------------------------------------------------------------------ device buffers
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t n) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = n;
    if (n) RW_CUDA(cudaMalloc(&p, n));
    if (n) RW_CUDA(cudaMemset(p, 0, n));
  }
  float* f() const { return static_cast<float*>(p); }
  unsigned long long* u64() const { return static_cast<unsigned long long*>(p); }
};

// An operand tensor: 1 (bf16) or 2 (tf32 / fp16 hi, lo) planes of `elems` elements.
struct Operand {
  DevBuf plane[2];
  void alloc(int prec, size_t elems) {
    const int planes = prec_planes(prec);
    const size_t eb = prec_elem(prec);
    for (int i = 0; i < 2; ++i) plane[i].alloc(i < planes ? elems * eb : 0);
  }
  void* p(int i) const { return plane[i].p; }
};

int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
int round_up(int a, int b) { return ceil_div(a, b) * b; }
int pad_grid(long long n) { (void)n; return 148 * 8; }  // k_pad_cols: one column per block iteration
int grid_for(long long n) { return (int)std::min<long long>(std::max<long long>(1, (n + 255) / 256), 148LL * 16); }

constexpr int kSmemLimit = 232448;  // 227 KB opt-in per CTA

// ------------------------------------------------------------------ NCCL (dlopen'd)
// Minimal subset of nccl.h (NCCL 2.x ABI) so the library carries no link-time NCCL dependency.
typedef struct ncclComm* ncclComm_t;
struct NcclId {
  char internal[128];
};
struct Nccl {
  void* h = nullptr;
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
Nccl& nccl() {
  static Nccl n;
  if (!n.h) {
    // The NCCL the process already uses (e.g. PyTorch's), else RW_NCCL_PATH (the Python loader
    // points it at the nvidia-nccl wheel PyTorch links), else the system one. Loaded RTLD_LOCAL:
    // a second library with the same soname made global here would shadow a newer NCCL that a
    // later import (libtorch_cuda) resolves its symbols against.
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!n.h)
      if (const char* e = getenv("RW_NCCL_PATH")) n.h = dlopen(e, RTLD_NOW | RTLD_LOCAL);
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      if (n.h) break;
      n.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    }
    if (!n.h) throw RwError{RW_ENCCL, "libnccl.so.2 not found"};
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
    n.AllReduce = (decltype(n.AllReduce))dlsym(n.h, "ncclAllReduce");
    n.GroupStart = (decltype(n.GroupStart))dlsym(n.h, "ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.h, "ncclGroupEnd");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
    if (!n.GetUniqueId || !n.CommInitRank || !n.AllReduce || !n.GroupStart || !n.GroupEnd)
      throw RwError{RW_ENCCL, "libnccl.so.2 lacks required symbols"};
  }
  return n;
}
void nccl_check(int r, const char* what) {
  if (r != 0)
    throw RwError{RW_ENCCL, std::string(what) + ": " +
                                (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error")};
}
constexpr int kNcclFloat32 = 7, kNcclSum = 0;

struct ClPlan {
  int kc = 0, cs = 0, ncomax = 0, stages = 0;
  int stages_off = 0, st_alias = 0, st_off = 0;  // ClParams (rec_cluster.cuh)
  size_t smem = 0;
  void* kern = nullptr;  // the k_cl_fwd / k_cl_bwd instantiation for Bp / kc owned columns
};

template <class P>
struct KernelSet {
  static constexpr int kPrec = P::kPlanes == 1 ? kBF16 : P::kTF32 ? kTF32x3 : kF16x2;
  static void* fwd() { return lstm_kernel_ptr(kPrec, true, false); }
  static void* bwd() { return lstm_kernel_ptr(kPrec, false, false); }
};

// Calls f(PrecX{}) for the context's operand format.
template <class F>
void by_prec(int prec, F&& f) {
  if (prec == kBF16)
    f(PrecBF16{});
  else if (prec == kF16x2)
    f(PrecF16x2{});
  else
    f(PrecTF32x3{});
}

}  // namespace

// ====================================================================== context
struct rw_ctx {
  rw_config cfg{};
  int dev = 0;
  int prec = kBF16, planes = 1, elem = 2, atomK = 64;
  int L = 0, H = 0, I = 0, B = 0, T = 0, Hp = 0, Ip = 0, Bp = 0;
  int kind = 3, G = 4;  // cell kind (rw_config.cell_kind: 0 RNN tanh, 1 RNN relu, 2 GRU, 3 LSTM), gates
  std::string err;

  // parameters (reference layout, device) + packed operands
  std::vector<DevBuf> W, R, bias_raw;
  std::vector<Operand> wf, wb;
  Operand w0t;
  std::vector<DevBuf> bias;
  bool params_set_all = false;
  std::vector<char> params_set;
  bool dirty = true;

  // activations / tapes
  DevBuf x_raw, dy_raw;
  Operand x_op;
  std::vector<DevBuf> h, c, gates, tanhc, dg, carry_c, dh0, dc0, dbp;
  std::vector<Operand> hop, dgop;
  // tf32 only: K-major (time-batch contiguous) copies for the weight-gradient GEMMs, since
  // tcgen05 kind::tf32 cannot read these operands MN-major with the 128B swizzle we use
  std::vector<Operand> dgT, hT, dgrT;  // 3xTF32 weight gradients: K-major copies (GRU: dgr too)
  Operand xT;
  DevBuf dx0, y_raw, stage;  // unpadded outputs / staging
  std::vector<DevBuf> dW, dR, db;
  DevBuf flags_f, flags_b, errflag;

  // descriptors
  std::vector<CUtensorMap> maps;  // host copy
  DevBuf maps_dev;
  int mi_xK[2] = {0, 0};          // map indices of the K-major x / h operands (the ladder's B operands)
  std::vector<int> mi_hopK;
  // ---- the GPU optimisation ladder (rw_ladder_pass), built on first use
  struct Ladder {
    bool ready = false;
    std::vector<Operand> wraw, rraw;  // W_l, R_l in the reference layout (MN-major A operand planes)
    DevBuf maps;                      // [wraw planes, rraw planes, x / h operand copies] per layer
    DevBuf zw, zr, pre, gates, t1, t2;
    DevBuf desc;                      // GemmDesc [l][t][kind]: W gate 0..3, R gate 0..3, W grouped, R grouped
    std::vector<cudaEvent_t> ev;      // per (l, t): the W.x GEMM of the step finished (streamed rungs)
    cudaStream_t side = nullptr;
    ~Ladder() {
      for (auto e : ev) cudaEventDestroy(e);
      if (side) cudaStreamDestroy(side);
    }
  } ladder;
  DevBuf fwd_layers, bwd_layers, gemm_wg, gemm_dx;
  int n_wg = 0;

  // schedule
  int fwd_sched = RW_SCHED_STEPWISE, bwd_sched = RW_SCHED_STEPWISE;
  int ks_f = 1, ks_b = 1, res_f = 0, res_b = 0, st_f = 4, st_b = 4;
  int slots_f = 0, slots_b = 0, acckb_f = 1, acckb_b = 1, nacc_f = 1, nacc_b = 1;
  int promo_f = 0, promo_b = 0;  // 3xTF32 promotion ring (lstm_step.cuh promo_drain)
  size_t smem_f = 0, smem_b = 0;
  // cluster schedule (rec_cluster.cuh)
  ClPlan cl_f, cl_b;
  DevBuf cl_offsum, cl_done, cl_consumed;  // [L][tiles]... off-partial rings of this context's layers
  DevBuf cl_epoch;                          // [2] pass counters (forward, backward)
  int cl_ring = 4;                          // off-partial ring depth
  DevBuf cl_ring_f, cl_ring_b, cl_off_f, cl_off_b;  // ClRing[L] / ClOff[rows] tables (device)
  std::vector<ClRing> ring_f_h, ring_b_h;
  std::vector<ClOff> off_f_h, off_b_h;
  int rows_f = 0, rows_b = 0;               // grid rows (>= L: pipeline stages add boundary groups)
  // layer pipeline (rw_pp_*): boundary groups, peer buffers
  bool pp_prev = false, pp_next = false;     // linked to a previous / next stage
  bool pair_f = false;                       // stepwise forward as CTA pairs (k_lstm_fwd<bf16, true>)
  bool pair_b = false;                       // persistent backward as CTA pairs (k_lstm_bwd<bf16, true>)
  bool ls_pers_f = false, ls_pers_b = false;  // layer-sequential: one persistent launch per layer
  // stepwise forward with batched input projections (large H): W_l . X_l for blocks of fwd_batch
  // steps as one GEMM into the gates tape (layer 0: all steps at once), the step kernels then
  // stream only R (FwdLayer::zx); descriptors [layer 0][layer l >= 1 x block]
  int fwd_batch = 0;
  DevBuf gemm_fb;
  bool state0_zero = false;                  // block 0 (h0 = c0 = 0) of the state tapes is current
  bool pp_exported_f = false, pp_exported_b = false;
  DevBuf wb_prev;                            // packed [W_0^T | R_0^T] (cluster backward boundary group)
  DevBuf xin_flags;                          // pipeline stage > 0: per-step counters of its input h_t
  DevBuf wb_prev_lo;                         // fp16x2: lo plane of wb_prev
  void* pp_next_xop_lo = nullptr;            // fp16x2: next stage's layer-input lo plane (peer pointer)
  DevBuf repack_jobs;                        // k_repack's job table (built on the first repack)
  int repack_njobs = 0, repack_tiles = 0;
  DevBuf wn_raw;                             // host-given copy of the next stage's W_0 (persistent / stepwise pipeline)
  // [0] forward / [1] backward boundary group (cluster); [2..3] the top layer's [W_next^T | R^T]
  // planes, [4..5] its dG-input planes, [6] the same as CTA-pair boxes (persistent / stepwise)
  std::vector<CUtensorMap> pp_maps = std::vector<CUtensorMap>(8);
  DevBuf pp_maps_dev;
  void* pp_next_xop = nullptr;               // next stage's layer-input operand (peer pointer)
  uint32_t* pp_next_ready = nullptr;         // next stage's input-ready counter (peer pointer)
  std::vector<void*> pp_opened;              // IPC-opened peer allocations
  // layer pipeline over the persistent / stepwise schedules: h_t stored straight into the next
  // stage's layer-input planes; the next stage's first-layer dG_t stored into this stage's dgin
  // planes, which its top layer multiplies by W_next^T (the peer's W_0, pp_wnext) exactly as one
  // context's layer below would
  bool pp_plain = false;
  Operand dgin;
  DevBuf dgin_flags;                         // [T] per-step counters + [T] the sender's CTAs per step
  const float* pp_wnext = nullptr;
  bool pp_up = false;                        // the top layer's backward reads dgin (has_up)
  std::vector<DevBuf> hsw, dgsw;  // pre-swizzled bf16 operand step blocks (sw_off)
  // GRU: zrh tapes, R-side gate gradients dgr (fp32 tape + operand planes), the W-side image dgwsw
  std::vector<DevBuf> zrh, dgr, dgwsw;
  std::vector<Operand> dgrop;
  DevBuf xsw;
  int bn_wg = 128, bn_dx = 128, st_wg = 4, st_dx = 4, bn_ls = 256;
  DevBuf gemm_lsf, gemm_lsb, dabove;  // layer-sequential schedule
  size_t smem_wg = 0, smem_dx = 0;

  // streams / events / graphs
  cudaStream_t main = nullptr;
  // rw_train_step: copy streams and the events that order the pipelined host round trip
  cudaStream_t cp_in = nullptr, cp_out = nullptr;
  // data parallel, overlapped (rw_comm_overlap): per-layer gradient buckets all-reduced on `comm_s`
  // as soon as that layer's weight-gradient GEMMs finish, while the lower layers' GEMMs and dx0 run
  bool dp_overlap = false;
  cudaStream_t comm_s = nullptr;
  // the dx0 GEMM runs on its own stream beside the weight-gradient GEMMs (fills their last wave)
  cudaStream_t tail_s = nullptr;
  cudaEvent_t ev_tail_fork = nullptr, ev_tail_join = nullptr;
  std::vector<cudaEvent_t> ev_layer;
  cudaEvent_t ev_comm = nullptr;
  cudaEvent_t ev_fwd = nullptr, ev_x = nullptr, ev_y_staged = nullptr, ev_y_out = nullptr, ev_dy = nullptr,
              ev_bwd = nullptr, ev_out = nullptr;
  std::vector<cudaStream_t> ls;
  std::vector<cudaEvent_t> lev;
  cudaEvent_t fork_ev = nullptr;
  // per pass kind: 0-3 as rw_run_pass; internal 4 = backward recurrence only, 5 = the
  // gradient GEMMs / reductions only (rw_train_step waits for the previous read-back between)
  cudaGraphExec_t graphs[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  long long graph_launches[6] = {0, 0, 0, 0, 0, 0};                   // kernels inside each graph
  bool use_graphs = true;

  // state
  uint64_t tape_gen = 0;
  bool tape_training = false;
  bool bwd_done = false;
  bool inputs_uploaded = false;

  // data parallel
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;

  // device trace (RW_TRACE=<csv path>): globaltimer stamps of the persistent kernels
  DevBuf trace_f, trace_b, trace_dx;  // device stamps (tracing on): [cta][steps][16] / dx0 GEMM span
  bool tracing = false;
  std::string trace_path;        // RW_TRACE: reference-schema CSV of every synced pass
  std::string trace_spans_path;  // RW_TRACE_SPANS: per-CTA span profile (profiles/trace_run.py)

  // hang debugging (RW_DEBUG_HANG_S): mapped host progress words
  unsigned int* progress_host = nullptr;
  unsigned int* progress_dev = nullptr;
  double hang_s = 0;

  // profiling
  bool profiling = false;
  double phase_ms[6] = {0};
  int phase_n[6] = {0};

  ~rw_ctx();
};

namespace {

// ------------------------------------------------------------------ schedule selection
struct RecPlan {
  int sched, ks, resident, stages;
  size_t smem;
  int a_slots;
};

int max_active_clusters(void* kernel, int ks, size_t smem, int ctas) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(ctas, 1, 1);
  lc.blockDim = dim3(kRecThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ks;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &lc) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// kb_max: largest per-tile k-block count over layers; tiles per layer; L layers.
RecPlan plan_recurrent(void* kernel, int want, int planes, int kb_max, int tiles, int L, int N,
                       int sms, const char* env_ks) {
  RecPlan pl{RW_SCHED_STEPWISE, 1, 0, 4, 0};
  int forced_ks = 0;
  if (const char* e = getenv(env_ks)) forced_ks = atoi(e);
  if (want != RW_SCHED_STEPWISE) {
    for (int ks : {8, 4, 2, 1}) {
      if (forced_ks && ks != forced_ks) continue;
      if (ks > kb_max) continue;
      const long long ctas = (long long)L * tiles * ks;
      if (ctas > sms) continue;
      for (int resident : {1, 0}) {
        const int kbr = resident ? ceil_div(kb_max, ks) : 0;
        int stages = 4;
        size_t smem = rec_smem_bytes(planes, resident ? kbr : stages, N, stages);
        // one CTA per SM: co-resident persistent CTAs must never contend for TMEM columns
        smem = std::max(smem, (size_t)116 * 1024);
        if (const char* e = getenv("RW_MIN_SMEM_KB")) smem = std::max(smem, (size_t)atoi(e) * 1024);
        while (smem > (size_t)kSmemLimit && stages > 2) {
          --stages;
          smem = rec_smem_bytes(planes, resident ? kbr : stages, N, stages);
        }
        if (smem > (size_t)kSmemLimit) continue;
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ks > 1) cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        const int clusters = max_active_clusters(kernel, ks, smem, (int)ctas);
        if ((long long)clusters * ks < ctas) continue;
        return RecPlan{RW_SCHED_PERSISTENT, ks, resident, stages, smem, resident ? kbr : 0};
      }
    }
    if (want == RW_SCHED_PERSISTENT) einval("persistent schedule does not fit this configuration on the device");
  }
  // stepwise: split K only while the L concurrently running layers (the wavefront) leave SMs
  // idle -- the split-K exchange costs more than it gains once tiles x L fill the GPU
  // (config E forward: ks 1 / 2 / 4 = 27 / 35 / 57 ms)
  int ks = 1;
  while (ks < 8 && (long long)tiles * L * ks * 2 <= sms && ks * 2 <= kb_max) ks *= 2;
  if (forced_ks) ks = forced_ks;
  int stages = 4;
  size_t smem = rec_smem_bytes(planes, stages, N, stages);
  while (smem > (size_t)kSmemLimit && stages > 2) {
    --stages;
    smem = rec_smem_bytes(planes, stages, N, stages);
  }
  if (smem > (size_t)kSmemLimit) einval("batch too large for the recurrent kernel tile");
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (ks > 1) cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return RecPlan{RW_SCHED_STEPWISE, ks, 0, stages, smem, 0};
}

template <class P>
void launch_rec(void* kernel, const void* layers, const RecParams& rp, int grid_x, int grid_y,
                size_t smem, cudaStream_t s, int cluster = 0) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid_x, grid_y, 1);
  lc.blockDim = dim3(kRecThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster > 0 ? cluster : rp.ksplit;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  void* args[2] = {const_cast<void**>(&layers), const_cast<RecParams*>(&rp)};
  ++g_launches;
  RW_CUDA(cudaLaunchKernelExC(&lc, kernel, args));
}

// Cluster schedule (rec_cluster.cuh): per tile a critical cluster (kc members) and an off
// cluster (ko_l members per layer), each member holding <= 512 K of its weight slice. Returns
// false when the shape does not fit (batch > 64, owned columns not a multiple of 16, too many
// CTAs, shared memory, or clusters not co-resident).
void* cl_kernel(int prec, bool fwd, int nco, int kind = kCellLstm) { return cl_kernel_ptr(prec, fwd, nco, kind); }

// prec: kBF16 or kF16x2 (two operand planes per stage; A_lo in tensor memory next to the
// 4 x Bp accumulator columns, which fits 512 columns for Bp <= 64 and <= 8 k-blocks per member)
bool plan_cluster(int prec, bool fwd, int kc, const std::vector<int>& ko, int tiles, int L, int Bp, int sms,
                  ClPlan& out, int kind = kCellLstm) {
  if (Bp > kClMaxN || Bp % kc || (Bp / kc) % 16) return false;
  if (prec == kF16x2 && 4 * Bp + kClKBlocks * 32 > 512) return false;
  const int rows = prec_planes(prec) * Bp;  // operand rows per stage
  void* kernel = cl_kernel(prec, fwd, Bp / kc, kind);
  int cs = kc, komin = kc;
  for (int k : ko) {
    if (k == 0) continue;
    if (Bp % k || (Bp / k) % 16) return false;
    cs = std::max(cs, k);
    komin = std::min(komin, k);
  }
  if (cs > 8 || (long long)L * tiles * 2 * cs > sms) return false;
  const int ncomax = Bp / komin;
  const int min_stages = fwd ? 4 : 2;  // forward critical: the sum buffer aliases the B stages
  int stages = kClKBlocks;
  size_t smem = cl_smem_bytes(cs, ncomax, rows, stages);
  while (smem > (size_t)kSmemLimit && stages > min_stages) smem = cl_smem_bytes(cs, ncomax, rows, --stages);
  if (smem > (size_t)kSmemLimit) return false;
  // an even ring lets operand k-blocks travel in pairs (rec_cluster.cuh cl_pair_kb)
  if (stages % 2 && stages > min_stages) smem = cl_smem_bytes(cs, ncomax, rows, --stages);
  if (fwd && (size_t)stages * rows * kRowBytes < (size_t)(Bp / kc) * kTileM * 4) return false;
  // backward with split-K pushes: the critical CTAs stage their pushes inside the B ring (after
  // the dG staging image), which frees (cs-1) slots for more ring stages; the off CTAs keep a
  // separate staging area after their (fewer) stages in the same region (rec_cluster.cuh)
  int stages_off = stages, st_alias = 0, st_off = 0;
  if (!fwd && cs > 1 && !(getenv("RW_CL_ST_ALIAS") && atoi(getenv("RW_CL_ST_ALIAS")) == 0)) {
    const size_t stage = (size_t)rows * kRowBytes, slot = cl_slot_bytes(ncomax), st_bytes = (size_t)(cs - 1) * slot;
    const size_t staging = (size_t)8 * prec_planes(prec) * (Bp / kc) * 128;
    const size_t fixed = 1024 + (size_t)kClKBlocks * kTileM * kRowBytes + (size_t)cs * slot + 16;
    int sc = kClKBlocks;
    while (sc > 2 && fixed + sc * stage + (2 * sc + 12) * 8 > (size_t)kSmemLimit) --sc;
    if (sc % 2) --sc;
    int so = sc * stage > st_bytes ? (int)((sc * stage - st_bytes) / stage) : 0;
    if (so % 2) --so;
    if (sc > stages && so >= 2 && (size_t)sc * stage >= staging + st_bytes) {
      stages = sc;
      stages_off = so;
      st_alias = 1;
      st_off = (int)((staging + 1023) / 1024 * 1024);
      smem = fixed + sc * stage + (2 * sc + 12) * 8;
    }
  }
  smem = std::max(smem, (size_t)116 * 1024);  // one CTA per SM
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if ((long long)max_active_clusters(kernel, cs, smem, L * tiles * 2 * cs) < (long long)L * tiles * 2) return false;
  out = ClPlan{kc, cs, ncomax, stages, stages_off, st_alias, st_off, smem, kernel};
  return true;
}

void upload_cluster_tables(rw_ctx* x) {
  auto up = [](DevBuf& d, const void* h, size_t bytes) {
    d.alloc(std::max<size_t>(bytes, 16));
    if (bytes) RW_CUDA(cudaMemcpy(d.p, h, bytes, cudaMemcpyHostToDevice));
  };
  up(x->cl_ring_f, x->ring_f_h.data(), x->ring_f_h.size() * sizeof(ClRing));
  up(x->cl_ring_b, x->ring_b_h.data(), x->ring_b_h.size() * sizeof(ClRing));
  up(x->cl_off_f, x->off_f_h.data(), x->off_f_h.size() * sizeof(ClOff));
  up(x->cl_off_b, x->off_b_h.data(), x->off_b_h.size() * sizeof(ClOff));
}

size_t gemm_smem(int planes, int bn, int stages) {
  return 1024 + (size_t)stages * planes * (kTileM + bn) * kRowBytes + (2 * stages + 4) * 8 + 16;
}

// fp32-parity GEMMs accumulate in chunks of kPromoteKB k-blocks (3xTF32: 2 x 32 = 64 K elements;
// fp16x2: kPromoteKB16 x 64 = 512, measured 6.4e-7 normwise for one 512-long chain,
// profiles/ubench/f16x2_ts_check.cu)
// drained into fp32 registers; bf16 runs the whole K in TMEM.
constexpr int kPromoteKB = 2;
constexpr int kPromoteKB16 = 4;

// bf16 grouped GEMMs go to the persistent kernel (gemm_tc.cuh k_gemm_p) unless RW_GEMM_OLD=1;
// fp32-parity (3xTF32, chunked fp32 promotion) keeps the one-tile-per-CTA kernel.
template <bool AMN, bool BMN, int BN>
void launch_gemm_p(const GemmDesc* table_dev, int count, int M, int N, cudaStream_t s) {
  const size_t stage = (size_t)(kTileM + BN) * kRowBytes;
  int stages = 8;
  auto smem_of = [&](int st) { return 1024 + st * stage + (2 * st + 4) * 8 + 16; };
  while (stages > 2 && smem_of(stages) > (size_t)kSmemLimit) --stages;
  const size_t smem = smem_of(stages);
  const int mt = ceil_div(M, kTileM), nt = ceil_div(N, BN);
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long tiles = (long long)count * mt * nt;
  const int grid = (int)std::min<long long>(tiles, sms);
  void* k = gemm_p_ptr(AMN, BMN, BN);
  RW_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ++g_launches;
  void* args[5] = {const_cast<GemmDesc**>(&table_dev), &count, const_cast<int*>(&mt), const_cast<int*>(&nt),
                   &stages};
  RW_CUDA(cudaLaunchKernel(k, dim3(grid), dim3(256), args, smem, s));
}

template <bool AMN, bool BMN, int BN>
void launch_gemm_p2(const GemmDesc* table_dev, int count, int M, int N, cudaStream_t s) {
  const size_t stage = (size_t)(kTileM + BN / 2) * kRowBytes;
  int stages = 8;
  auto smem_of = [&](int st) { return 1024 + st * stage + (2 * st + 4) * 8 + 16; };
  while (stages > 2 && smem_of(stages) > (size_t)kSmemLimit) --stages;
  const size_t smem = smem_of(stages);
  const int mt = ceil_div(M, 2 * kTileM), nt = ceil_div(N, BN);
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long tiles = (long long)count * mt * nt;
  const int pairs = (int)std::min<long long>(tiles, sms / 2);
  void* k = gemm_p2_ptr(AMN, BMN, BN);
  RW_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(2 * pairs, 1, 1);
  lc.blockDim = dim3(256, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  ++g_launches;
  void* args[5] = {const_cast<GemmDesc**>(&table_dev), &count, const_cast<int*>(&mt), const_cast<int*>(&nt),
                   &stages};
  RW_CUDA(cudaLaunchKernelExC(&lc, k, args));
}

template <class P, bool AMN, bool BMN>
void launch_gemm(const GemmDesc* table_dev, int count, int M, int N, int bn, int stages,
                 cudaStream_t s) {
  static const bool pair2 = !(getenv("RW_GEMM_2SM") && atoi(getenv("RW_GEMM_2SM")) == 0);
  static const bool old = getenv("RW_GEMM_OLD") && atoi(getenv("RW_GEMM_OLD")) != 0;
  // a single wave of tiles gains nothing from the persistent loop (measured: dx0 at config B
  // 36 us one-tile-per-CTA vs 48 us persistent)
  const long long tiles = (long long)count * ceil_div(M, kTileM) * ceil_div(N, bn);
  if (P::kPlanes == 1 && !old && pair2 && bn == 256 && tiles > 148) {
    launch_gemm_p2<AMN, BMN, 256>(table_dev, count, M, N, s);
    return;
  }
  // 128-column pair tiles (M = 256 x N = 128 per pair, half the TMEM): per SM a k-block moves
  // 16 + 8 KB for 256 MMA cycles instead of 16 + 16 KB (RW_GEMM_2SM128=0 disables)
  static const bool pair128 = !(getenv("RW_GEMM_2SM128") && atoi(getenv("RW_GEMM_2SM128")) == 0);
  // (MN-major B only: a K-major B map has 128-row boxes, one CTA's half here is 64 rows)
  if (P::kPlanes == 1 && !old && pair2 && pair128 && BMN && bn == 128 && tiles > 148) {
    launch_gemm_p2<AMN, BMN, 128>(table_dev, count, M, N, s);
    return;
  }
  if (P::kPlanes == 1 && !old && (bn == 128 || bn == 256) && tiles > 148) {
    if (bn == 256)
      launch_gemm_p<AMN, BMN, 256>(table_dev, count, M, N, s);
    else
      launch_gemm_p<AMN, BMN, 128>(table_dev, count, M, N, s);
    return;
  }
  const size_t smem = gemm_smem(P::kPlanes, bn, stages);
  dim3 grid(ceil_div(M, kTileM), ceil_div(N, bn), count);
  ++g_launches;
  // two-plane formats: the chunked-promotion variant, one instantiation per tile width
  const int prec = P::kPlanes == 1 ? kBF16 : P::kTF32 ? kTF32x3 : kF16x2;
  const int chunk_bn = P::kPlanes == 2 ? bn : 0;
  if (chunk_bn && chunk_bn != 64 && chunk_bn != 128) throw RwError{RW_ECUDA, "internal: two-plane GEMM tile width"};
  void* k = gemm_tc_ptr(prec, AMN, BMN, chunk_bn);
  int promote = chunk_bn ? (P::kTF32 ? kPromoteKB : kPromoteKB16) : 0;
  RW_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[4] = {const_cast<GemmDesc**>(&table_dev), &bn, &stages, &promote};
  RW_CUDA(cudaLaunchKernel(k, grid, dim3(256), args, smem, s));
}

int gemm_stages(int planes, int bn) {
  int st = 6;
  while (st > 2 && gemm_smem(planes, bn, st) > (size_t)kSmemLimit) --st;
  return st;
}

// ------------------------------------------------------------------ setup
void validate(const rw_config& c) {
  auto pos = [](int v, const char* n) {
    if (v <= 0) einval(std::string("LadderConfig: ") + n + " must be positive, got " + std::to_string(v));
  };
  pos(c.layers, "layers");
  pos(c.hidden, "hidden");
  pos(c.input, "input");
  pos(c.batch, "batch");
  pos(c.steps, "steps");
  pos(c.batch_steps, "batch_steps");
  pos(c.workers, "workers");
  if (c.opt_level < 0 || c.opt_level > 6)
    einval("LadderConfig: opt_level must be in 0..6, got " + std::to_string(c.opt_level));
  if (c.batch_steps > c.steps)
    einval("LadderConfig: batch_steps " + std::to_string(c.batch_steps) + " exceeds steps " + std::to_string(c.steps));
  if (c.cell_kind < 0 || c.cell_kind > 3)
    einval("LadderConfig: cell kind must be 0 (rnn-tanh), 1 (rnn-relu), 2 (gru) or 3 (lstm), got " +
           std::to_string(c.cell_kind));
  if (c.precision != RW_PREC_BF16 && c.precision != RW_PREC_FP32) einval("rnnwave_sm100: unknown precision");
  if (c.layers > kMaxLayers) einval("rnnwave_sm100: at most 16 layers");
}

int add_map(rw_ctx* x, const CUtensorMap& m) {
  x->maps.push_back(m);
  return (int)x->maps.size() - 1;
}

// Device stamp buffers of the recurrent kernels (RW_TRACE / rw_trace_enable): up to 4096 CTAs
// x (T + 2) steps x 16 stamps per direction; the stepwise schedule stores one block of grid
// CTAs per (layer, step) launch in the same buffers.
void trace_alloc(rw_ctx* x) {
  if (!x->trace_f.p) {
    const size_t ctas = 4096;
    x->trace_f.alloc(ctas * (x->T + 2) * 16 * 8);
    x->trace_b.alloc(ctas * (x->T + 2) * 16 * 8);
    x->trace_dx.alloc(16);
  }
  x->tracing = true;
}

void build(rw_ctx* x) {
  const rw_config& c = x->cfg;
  x->L = c.layers;
  x->H = c.hidden;
  x->I = c.input;
  x->B = c.batch;
  x->T = c.steps;
  x->Hp = round_up(x->H, 64);
  x->Ip = round_up(x->I, 64);
  x->Bp = round_up(x->B, 16);
  x->kind = c.cell_kind;
  x->G = cell_gates(c.cell_kind);
  const int L = x->L, Hp = x->Hp, Ip = x->Ip, Bp = x->Bp, T = x->T, H = x->H, I = x->I, B = x->B;
  const long long G4p = 4LL * Hp;
  const long long colsT = (long long)Bp * T, colsT1 = (long long)Bp * (T + 1);
  if (Bp > 256) einval("rnnwave_sm100: batch > 256 per context is not supported (split the minibatch)");

  RW_CUDA(cudaSetDevice(x->dev));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, x->dev);

  // ---- cluster schedule first: forward kc = K-slices of R.h, ko = of W.x; backward kc =
  // K-slices of R^T.dG, ko = of W_{l+1}^T.dG (none for a single layer). The fp32-parity mode
  // computes with fp16x2 split operands on every schedule but the layer-sequential one (3xTF32
  // there; RW_FP32_TF32=1 forces 3xTF32 everywhere): twice the MMA rate and half the operand
  // bytes of 3xTF32, and half the tensor-core accumulation steps per K element.
  ClPlan cpf, cpb;
  bool cl_f = false, cl_b = false;
  std::vector<int> ko_f(L), ko_b(L);  // off-critical members per layer (the rings' publication counts)
  auto try_cluster = [&](int prec) {
    const int kc_f = ceil_div(Hp / 64, kClKBlocks);
    auto fit = [&](int k, int nkb) {  // >= k members of <= 8 k-blocks that split Bp into 16s
      while (k < 8 && k < nkb && !(Bp % k == 0 && (Bp / k) % 16 == 0)) ++k;
      return k;
    };
    for (int l = 0; l < L; ++l) {
      const int nkb = (l == 0 ? Ip : Hp) / 64;
      ko_f[l] = fit(ceil_div(nkb, kClKBlocks), nkb);
    }
    cl_f = plan_cluster(prec, true, kc_f, ko_f, Hp / kUnitsPerFwdTile, L, Bp, sms, cpf, c.cell_kind);
    // at least 4 critical members when the K range allows (>= 1 k-block each): small H would
    // otherwise leave one CTA per tile with Bp x 128 cells (measured 6x slower at H = 128)
    const int nkb_r = 4 * Hp / 64;
    // the smallest member count covering K (<= 8 k-blocks each) that splits the batch into
    // owned-column groups of a multiple of 16 (e.g. Bp = 48: 3 members), then doubled towards 4
    auto splits = [&](int k) { return Bp % k == 0 && (Bp / k) % 16 == 0; };
    int kc_b = ceil_div(nkb_r, kClKBlocks);
    while (kc_b <= 8 && kc_b <= nkb_r && !splits(kc_b)) ++kc_b;
    while (kc_b < 4 && kc_b * 2 <= nkb_r && splits(kc_b * 2)) kc_b *= 2;
    for (int l = 0; l < L; ++l) ko_b[l] = l < L - 1 ? kc_b : 0;
    cl_b = plan_cluster(prec, false, kc_b, ko_b, ceil_div(Hp, kTileM), L, Bp, sms, cpb, c.cell_kind);
  };
  const bool want_cl = c.schedule == RW_SCHED_AUTO || c.schedule == RW_SCHED_CLUSTER;
  if (c.precision == RW_PREC_BF16) {
    x->prec = kBF16;
    if (want_cl) try_cluster(kBF16);
  } else {
    const bool force_tf32 = (getenv("RW_FP32_TF32") && atoi(getenv("RW_FP32_TF32")) != 0) ||
                            c.schedule == RW_SCHED_LAYERSEQ;
    x->prec = force_tf32 ? kTF32x3 : kF16x2;
    if (want_cl && !force_tf32) {
      try_cluster(kF16x2);
      if (!(cl_f && cl_b)) cl_f = cl_b = false;
    }
  }
  // GRU and vanilla-RNN cells: the cluster schedule keeps the input and recurrent products in
  // separate roles; the persistent / stepwise / layer-sequential kernels sum [W|R].[x;h] over K,
  // and GRU's linear-before-reset candidate stays apart there through the forward image's slot
  // layout (W_n in slot 2, R_n in slot 3: layout_kernels.cuh k_repack).
  x->planes = prec_planes(x->prec);
  x->elem = prec_elem(x->prec);
  x->atomK = prec_atomk(x->prec);

  x->W.resize(L);
  x->R.resize(L);
  x->bias_raw.resize(L);
  x->wf.resize(L);
  x->wb.resize(L);
  x->bias.resize(L);
  x->params_set.assign(L, 0);
  x->h.resize(L);
  x->c.resize(L);
  x->gates.resize(L);
  x->tanhc.resize(L);
  x->dg.resize(L);
  x->carry_c.resize(L);
  x->dh0.resize(L);
  x->dc0.resize(L);
  x->dbp.resize(L);
  x->hop.resize(L);
  x->dgop.resize(L);
  x->dW.resize(L);
  x->dR.resize(L);
  x->db.resize(L);
  for (int l = 0; l < L; ++l) {
    const int Il = l == 0 ? I : H, Ipl = l == 0 ? Ip : Hp;
    x->W[l].alloc(4ULL * H * Il * 4);
    x->R[l].alloc(4ULL * H * H * 4);
    x->bias_raw[l].alloc(4ULL * H * 4);
    x->wf[l].alloc(x->prec, (size_t)G4p * (Ipl + Hp));
    x->wb[l].alloc(x->prec, (size_t)Hp * ((l < L - 1 ? 2 : 1) * G4p));
    x->bias[l].alloc(G4p * 4);
    x->h[l].alloc((size_t)Hp * colsT1 * 4);
    x->c[l].alloc((size_t)Hp * colsT1 * 4);
    x->hop[l].alloc(x->prec, (size_t)Hp * colsT1);
    x->gates[l].alloc((size_t)G4p * colsT * 4);
    x->tanhc[l].alloc((size_t)Hp * colsT * 4);
    x->dg[l].alloc((size_t)G4p * colsT * 4);
    x->dgop[l].alloc(x->prec, (size_t)G4p * colsT);
    x->carry_c[l].alloc((size_t)Hp * Bp * 4);
    x->dh0[l].alloc((size_t)Hp * Bp * 4);
    x->dc0[l].alloc((size_t)Hp * Bp * 4);
    x->dW[l].alloc(4ULL * H * Il * 4);
    x->dR[l].alloc(4ULL * H * H * 4);
    x->db[l].alloc(4ULL * H * 4);
  }
  x->w0t.alloc(x->prec, (size_t)Ip * G4p);
  const bool kmajor_wg = x->prec == kTF32x3;
  if (kmajor_wg) {
    x->dgT.resize(L);
    x->hT.resize(L);
    if (x->kind == kCellGru) x->dgrT.resize(L);
    for (int l = 0; l < L; ++l) {
      x->dgT[l].alloc(x->prec, (size_t)G4p * colsT);
      x->hT[l].alloc(x->prec, (size_t)Hp * colsT1);
      if (x->kind == kCellGru) x->dgrT[l].alloc(x->prec, (size_t)G4p * colsT);
    }
    x->xT.alloc(x->prec, (size_t)Ip * colsT);
  }
  x->x_raw.alloc((size_t)I * B * T * 4);
  x->dy_raw.alloc((size_t)H * B * T * 4);
  x->x_op.alloc(x->prec, (size_t)Ip * colsT);
  x->dx0.alloc((size_t)I * B * T * 4);
  x->y_raw.alloc((size_t)std::max(4LL * H, (long long)std::max(H, I)) * B * (T + 1) * 4);
  x->flags_f.alloc((size_t)L * T * 4);
  x->flags_b.alloc((size_t)L * T * 4);
  x->errflag.alloc(32);  // [code, count, max|dG|, max|x|, max|h0|]

  // ---- schedules
  const bool f16x2 = x->prec == kF16x2;
  void* kf = lstm_kernel_ptr(x->prec, true, false, x->kind);
  void* kb = lstm_kernel_ptr(x->prec, false, false, x->kind);
  const int kbf_max = (std::max(Ip, Hp) + Hp) / x->atomK;
  const int kbb_max = (int)((L > 1 ? 2 : 1) * G4p / x->atomK);
  const int tiles_f = Hp / kUnitsPerFwdTile, tiles_b = ceil_div(Hp, kTileM);
  if (c.schedule == RW_SCHED_CLUSTER && !(cl_f && cl_b))
    einval("cluster schedule does not fit this configuration (batch <= 64, owned columns multiple of 16, "
           "CTAs and clusters co-resident)");
  int want = c.schedule == RW_SCHED_CLUSTER ? RW_SCHED_AUTO : c.schedule;
  bool ls = c.schedule == RW_SCHED_LAYERSEQ;
  // The layer-sequential schedule is opt-in: measured on B200 it is slower than the wavefront
  // schedules at every configured shape (E: 147 vs 71 ms per pass; the per-step GEMM with the
  // full batch as N moves ~1 MB of operands per CTA per step; profiles/r01/README.md).
  if (ls) {
    want = RW_SCHED_STEPWISE;
    cl_f = cl_b = false;
  }
  RecPlan pf{RW_SCHED_CLUSTER, 1, 0, 4, 0, 0}, pb{RW_SCHED_CLUSTER, 1, 0, 4, 0, 0};
  if (!(cl_f && cl_b)) {
    pf = plan_recurrent(kf, want, x->planes, ls ? Hp / x->atomK : kbf_max, tiles_f, ls ? 1 : L, Bp, sms,
                        "RW_FWD_KSPLIT");
    pb = plan_recurrent(kb, want, x->planes, ls ? (int)(G4p / x->atomK) : kbb_max, tiles_b, ls ? 1 : L, Bp, sms,
                        "RW_BWD_KSPLIT");
  }
  if (ls) {
    // persistent per-layer launches need every (tile, rank) CTA of a layer co-resident
    const int cf = tiles_f * pf.ks, cb = tiles_b * pb.ks;
    const bool lsp = !(getenv("RW_LS_PERSISTENT") && atoi(getenv("RW_LS_PERSISTENT")) == 0);
    x->ls_pers_f = lsp && max_active_clusters(kf, pf.ks, pf.smem, cf) * pf.ks >= cf;
    x->ls_pers_b = lsp && max_active_clusters(kb, pb.ks, pb.smem, cb) * pb.ks >= cb;
    pf.sched = pb.sched = RW_SCHED_LAYERSEQ;
    x->dabove.alloc((size_t)Hp * colsT * 4);
  }
  x->fwd_sched = pf.sched;
  x->ks_f = pf.ks;
  if (pf.sched == RW_SCHED_STEPWISE && !ls && x->kind == kCellLstm) {
    // measured default (profiles/r02/README.md): blocks of 4 steps from H = 1024 up at batch <= 64
    // (C2048 forward 5.97 -> 5.84 ms). At config E's batch of 256 the fp32 W.x tape a block
    // writes and the steps re-read (8 MB per layer-step) costs nearly what it saves in streamed W,
    // and the GEMMs take the SMs the wavefront's step kernels need: 18.9 -> 33.0 ms, so off.
    // RW_FWD_BATCH=s overrides, 0 disables
    x->fwd_batch = Hp >= 1024 && Bp <= 64 ? 4 : 0;
    if (const char* e = getenv("RW_FWD_BATCH")) x->fwd_batch = std::max(0, atoi(e));
    x->fwd_batch = std::min(x->fwd_batch, T);
  }
  x->res_f = pf.resident;
  x->st_f = pf.stages;
  x->smem_f = pf.smem;
  x->slots_f = pf.a_slots;
  x->bwd_sched = pb.sched;
  x->ks_b = pb.ks;
  x->res_b = pb.resident;
  x->st_b = pb.stages;
  x->smem_b = pb.smem;
  x->slots_b = pb.a_slots;
  // stepwise forward as CTA pairs (cta_group::2, M = 256, each CTA half of the batch columns):
  // bf16, no split-K, an even tile count and Bp/2 a multiple of 16 (RW_FWD_PAIR=0 disables)
  x->pair_f = x->kind == kCellLstm && x->prec == kBF16 && pf.sched == RW_SCHED_STEPWISE && !ls && !cl_f && pf.ks == 1 && tiles_f % 2 == 0 &&
              Bp >= 64 && Bp % 32 == 0 && !(getenv("RW_FWD_PAIR") && atoi(getenv("RW_FWD_PAIR")) == 0);
  if (x->pair_f) {
    int st = 8;
    size_t sm = rec_smem_bytes(1, st, Bp / 2, st);
    while (sm > (size_t)kSmemLimit && st > 2) sm = rec_smem_bytes(1, --st, Bp / 2, st);
    void* kp = lstm_kernel_ptr(kBF16, true, true);
    if (sm > (size_t)kSmemLimit ||
        cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
      cudaGetLastError();
      x->pair_f = false;
    } else {
      x->st_f = st;
      x->smem_f = sm;
    }
  }
  // persistent backward as CTA pairs: bf16, no split-K, streamed weights, even tile count,
  // and the pairs co-resident (RW_BWD_PAIR=0 disables)
  x->pair_b = x->kind == kCellLstm && x->prec == kBF16 && pb.sched == RW_SCHED_PERSISTENT && !ls && !cl_b && pb.ks == 1 && !pb.resident &&
              tiles_b % 2 == 0 && Bp >= 64 && Bp % 32 == 0 &&
              !(getenv("RW_BWD_PAIR") && atoi(getenv("RW_BWD_PAIR")) == 0);
  if (x->pair_b) {
    int st = 8;
    size_t sm = rec_smem_bytes(1, st, Bp / 2, st);
    while (sm > (size_t)kSmemLimit && st > 2) sm = rec_smem_bytes(1, --st, Bp / 2, st);
    sm = std::max(sm, (size_t)116 * 1024);
    void* kp = lstm_kernel_ptr(kBF16, false, true);
    const int ctas = tiles_b * L;
    if (sm > (size_t)kSmemLimit ||
        cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess ||
        max_active_clusters(kp, 2, sm, ctas) * 2 < ctas) {
      cudaGetLastError();
      x->pair_b = false;
    } else {
      x->st_b = st;
      x->smem_b = sm;
    }
  }
  if (cl_f) {
    x->fwd_sched = RW_SCHED_CLUSTER;
    x->cl_f = cpf;
    x->ks_f = cpf.kc;
  }
  if (cl_b) {
    x->bwd_sched = RW_SCHED_CLUSTER;
    x->cl_b = cpb;
    x->ks_b = cpb.kc;  // bias-gradient partial slices = kc members x 2 column halves
  }
  if (cl_f || cl_b) {
    const size_t lt = (size_t)L * std::max(Hp / kUnitsPerFwdTile, ceil_div(Hp, kTileM));
    // separate rings / counters per direction: counters are cumulative per direction's epoch
    x->cl_ring = kRing;
    if (const char* e = getenv("RW_PP_RING")) x->cl_ring = std::max(kRing, atoi(e));
    x->cl_offsum.alloc(2 * lt * x->cl_ring * Bp * kTileM * 4);
    x->cl_done.alloc(2 * lt * T * 4);
    x->cl_consumed.alloc(2 * lt * 32 * 4);
  }
  if (cl_f) {  // pre-swizzled 16-bit operand images (fp16x2: both planes per k-block)
    x->hsw.resize(L);
    for (int l = 0; l < L; ++l) x->hsw[l].alloc((size_t)Hp * colsT1 * 2 * x->planes);
    x->xsw.alloc((size_t)Ip * colsT * 2 * x->planes);
  }
  if (cl_b) {
    x->dgsw.resize(L);
    for (int l = 0; l < L; ++l) x->dgsw[l].alloc((size_t)G4p * colsT * 2 * x->planes);
  }
  if (x->kind == kCellGru) {  // zrh tapes; dgr (fp32 + operand planes); the W-side dG images
    x->zrh.resize(L);
    x->dgr.resize(L);
    x->dgrop.resize(L);
    x->dgwsw.resize(L);
    for (int l = 0; l < L; ++l) {
      x->zrh[l].alloc((size_t)Hp * colsT * 4);
      x->dgr[l].alloc((size_t)G4p * colsT * 4);
      x->dgrop[l].alloc(x->prec, (size_t)G4p * colsT);
      x->dgwsw[l].alloc((size_t)G4p * colsT * 2 * x->planes);
    }
  }
  // fp32-parity: accumulate every acc_kb k-blocks in a separate TMEM accumulator (<= 512 cols),
  // summed in fp32 by the epilogue. When that would leave chains longer than kPromoKB k-blocks
  // (large H: 512 / Bp accumulators cannot cover K), run the promotion ring instead: chunks of
  // kPromoKB k-blocks in 512 / Bp - 1 ring slots, each added into an fp32 sum region as soon as it
  // is complete (lstm_step.cuh promo_drain).
  constexpr int kPromoKB = 8;  // 8 x 32 = 256 K elements per tensor-core accumulation chain
  auto acc_plan = [&](int kb_per_cta, int& acc_kb, int& n_acc, int& promo) {
    acc_kb = kb_per_cta > 0 ? kb_per_cta : 1;
    n_acc = 1;
    promo = 0;
    if (x->prec == kBF16) return;
    if (x->prec == kF16x2) {
      // fp16x2 always runs the ring: its drain applies each K segment's operand scales. 4 x 64 =
      // 256 K elements (48 MMA accumulation steps) per chunk
      acc_kb = 4;
      if (const char* e = getenv("RW_PROMO_KB")) acc_kb = std::max(1, atoi(e));
      n_acc = std::max(1, std::min(kMaxPromoSlots, 512 / Bp - 1));
      promo = 1;
      return;
    }
    acc_kb = 2;
    while ((long long)ceil_div(kb_per_cta, acc_kb) * Bp > 512) acc_kb *= 2;
    n_acc = std::max(1, ceil_div(kb_per_cta, acc_kb));
    const int slots = std::min(kMaxPromoSlots, 512 / Bp - 1);
    if (acc_kb > kPromoKB && slots >= 1 && !getenv("RW_NO_PROMO")) {
      acc_kb = kPromoKB;
      n_acc = slots;
      promo = 1;
    }
  };
  acc_plan(ceil_div(ls ? Hp / x->atomK : kbf_max, x->ks_f), x->acckb_f, x->nacc_f, x->promo_f);
  acc_plan(ceil_div(ls ? (int)(G4p / x->atomK) : kbb_max, x->ks_b), x->acckb_b, x->nacc_b, x->promo_b);
  int slices_b = ceil_div(Bp, kXChunk) * x->ks_b * 2;
  for (int l = 0; l < L; ++l) x->dbp[l].alloc((size_t)slices_b * G4p * 4);

  // ---- tensor maps
  const int aK = x->atomK, prec = x->prec;
  std::vector<int> m_dgrK(2 * L);  // GRU: the R-side dG operand (the persistent / stepwise recurrence)
  std::vector<int> m_wf(2 * L), m_wb(2 * L), m_hopK(2 * L), m_hopMN(2 * L), m_dgK(2 * L),
      m_dgMN(2 * L), m_dgrMN(2 * L);
  int m_xK[2], m_xMN[2], m_w0t[2], m_dg0dx[2], m_xT[2];
  int m_xK2 = 0;  // CTA-pair forward: Bp/2-row boxes (bf16: one plane)
  std::vector<int> m_hopK2(L), m_dgK2(L);
  // layer-sequential GEMMs: B operands (layer inputs / dG) as K-major boxes of bn_ls columns
  x->bn_ls = x->prec == kBF16 ? 256 : x->prec == kF16x2 ? 128 : 64;  // tf32: the chunked-promotion GEMM variant
  int m_xLS[2] = {0, 0};
  std::vector<int> m_hopLS(2 * L), m_dgLS(2 * L);
  std::vector<int> m_dgT(2 * L), m_hT(2 * L), m_dgrT(2 * L);
  x->bn_dx = x->prec == kBF16 ? (colsT >= 256 ? 256 : 128) : 128;
  if (const char* e = getenv("RW_BN_DX")) x->bn_dx = atoi(e);
  // two-plane formats: (hi,hi)+(hi,lo) as one N = 2 bn MMA, 2 x 2 bn TMEM columns (gemm_tc.cuh)
  x->bn_wg = 128;
  if (const char* e = getenv("RW_BN_WG2"); e && x->prec != kBF16) x->bn_wg = atoi(e);
  for (int p = 0; p < x->planes; ++p) {
    for (int l = 0; l < L; ++l) {
      const int Ipl = l == 0 ? Ip : Hp;
      m_wf[2 * l + p] = add_map(x, make_map(x->wf[l].p(p), prec, Ipl + Hp, G4p, aK, kTileM));
      m_wb[2 * l + p] = add_map(x, make_map(x->wb[l].p(p), prec, (l < L - 1 ? 2 : 1) * G4p, Hp, aK, kTileM));
      m_hopK[2 * l + p] = add_map(x, make_map(x->hop[l].p(p), prec, Hp, colsT1, aK, Bp));
      if (p == 0) x->mi_hopK.assign(2 * L, 0);
      x->mi_hopK[2 * l + p] = m_hopK[2 * l + p];
      if (x->pair_f) m_hopK2[l] = add_map(x, make_map(x->hop[l].p(p), prec, Hp, colsT1, aK, Bp / 2));
      m_hopMN[2 * l + p] = add_map(x, make_map(x->hop[l].p(p), prec, Hp, colsT1, aK, aK));
      m_dgK[2 * l + p] = add_map(x, make_map(x->dgop[l].p(p), prec, G4p, colsT, aK, Bp));
      m_dgrK[2 * l + p] = x->kind == kCellGru ? add_map(x, make_map(x->dgrop[l].p(p), prec, G4p, colsT, aK, Bp))
                                              : m_dgK[2 * l + p];
      if (x->pair_b) m_dgK2[l] = add_map(x, make_map(x->dgop[l].p(p), prec, G4p, colsT, aK, Bp / 2));
      m_dgMN[2 * l + p] = add_map(x, make_map(x->dgop[l].p(p), prec, G4p, colsT, aK, aK));
      m_dgrMN[2 * l + p] = x->kind == kCellGru ? add_map(x, make_map(x->dgrop[l].p(p), prec, G4p, colsT, aK, aK))
                                               : m_dgMN[2 * l + p];
    }
    if (kmajor_wg) {
      for (int l = 0; l < L; ++l) {
        m_dgT[2 * l + p] = add_map(x, make_map(x->dgT[l].p(p), prec, colsT, G4p, aK, kTileM));
        m_dgrT[2 * l + p] = x->kind == kCellGru ? add_map(x, make_map(x->dgrT[l].p(p), prec, colsT, G4p, aK, kTileM))
                                                : m_dgT[2 * l + p];
        m_hT[2 * l + p] = add_map(x, make_map(x->hT[l].p(p), prec, colsT1, Hp, aK, gemm_box_rows(x->bn_wg)));
      }
      m_xT[p] = add_map(x, make_map(x->xT.p(p), prec, colsT, Ip, aK, gemm_box_rows(x->bn_wg)));
    }
    m_xK[p] = add_map(x, make_map(x->x_op.p(p), prec, Ip, colsT, aK, Bp));
    x->mi_xK[p] = m_xK[p];
    if (x->pair_f) m_xK2 = add_map(x, make_map(x->x_op.p(p), prec, Ip, colsT, aK, Bp / 2));
    m_xMN[p] = add_map(x, make_map(x->x_op.p(p), prec, Ip, colsT, aK, aK));
    m_w0t[p] = add_map(x, make_map(x->w0t.p(p), prec, G4p, Ip, aK, kTileM));
    m_dg0dx[p] = add_map(x, make_map(x->dgop[0].p(p), prec, G4p, colsT, aK, gemm_box_rows(x->bn_dx)));
    if (ls || x->fwd_batch) {
      m_xLS[p] = add_map(x, make_map(x->x_op.p(p), prec, Ip, colsT, aK, gemm_box_rows(x->bn_ls)));
      for (int l = 0; l < L; ++l) {
        m_hopLS[2 * l + p] = add_map(x, make_map(x->hop[l].p(p), prec, Hp, colsT1, aK, gemm_box_rows(x->bn_ls)));
        m_dgLS[2 * l + p] = add_map(x, make_map(x->dgop[l].p(p), prec, G4p, colsT, aK, gemm_box_rows(x->bn_ls)));
      }
    }
  }
  x->maps_dev.alloc(x->maps.size() * sizeof(CUtensorMap));
  RW_CUDA(cudaMemcpy(x->maps_dev.p, x->maps.data(), x->maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  const CUtensorMap* MD = static_cast<const CUtensorMap*>(x->maps_dev.p);
  auto mp = [&](int idx, int p) -> const CUtensorMap* { return p < x->planes ? MD + idx : nullptr; };

  // ---- per-layer descriptor tables
  std::vector<FwdLayer> fl(L);
  std::vector<BwdLayer> bl(L);
  uint32_t* ff = static_cast<uint32_t*>(x->flags_f.p);
  uint32_t* fb = static_cast<uint32_t*>(x->flags_b.p);
  for (int l = 0; l < L; ++l) {
    FwdLayer& F = fl[l];
    for (int p = 0; p < 2; ++p) {
      F.a[p] = mp(m_wf[2 * l + (p % x->planes)], p);
      F.bx[p] = l == 0 ? mp(m_xK[p % x->planes], p) : mp(m_hopK[2 * (l - 1) + (p % x->planes)], p);
      F.bh[p] = mp(m_hopK[2 * l + (p % x->planes)], p);
      F.hop[p] = x->hop[l].p(p);
    }
    F.Ipl = l == 0 ? Ip : Hp;
    F.bx_col_off = l == 0 ? 0 : Bp;
    F.bias = x->bias[l].f();
    F.h = x->h[l].f();
    F.c = x->c[l].f();
    F.gates = x->gates[l].f();
    F.tanhc = x->tanhc[l].f();
    F.flags = ff + (size_t)l * T;
    F.zx = ls || x->fwd_batch ? x->gates[l].f() : nullptr;  // the input GEMM writes W.x into the gates tape
    F.bx2 = x->pair_f ? MD + (l == 0 ? m_xK2 : m_hopK2[l - 1]) : nullptr;
    F.bh2 = x->pair_f ? MD + m_hopK2[l] : nullptr;
    F.alo = f16x2 ? static_cast<const uint16_t*>(x->wf[l].p(1)) : nullptr;
    F.alo_ld = (l == 0 ? Ip : Hp) + Hp;
    F.alo_rows = (int)G4p;
    if (!x->hsw.empty()) {
      F.hsw = static_cast<uint8_t*>(x->hsw[l].p);
      F.bxsw = l == 0 ? static_cast<const uint8_t*>(x->xsw.p) : static_cast<const uint8_t*>(x->hsw[l - 1].p);
      F.bx_blk_off = l == 0 ? 0 : 1;
    }
    BwdLayer& Bd = bl[l];
    for (int p = 0; p < 2; ++p) {
      Bd.a[p] = mp(m_wb[2 * l + (p % x->planes)], p);
      Bd.bup[p] = l < L - 1 ? mp(m_dgK[2 * (l + 1) + (p % x->planes)], p) : nullptr;
      Bd.bg[p] = mp(m_dgrK[2 * l + (p % x->planes)], p);  // GRU: R^T dgr (dgr != dgw in the candidate)
      Bd.bup2 = x->pair_b && l < L - 1 ? MD + m_dgK2[l + 1] : nullptr;
      Bd.bg2 = x->pair_b ? MD + m_dgK2[l] : nullptr;
      Bd.alo = f16x2 ? static_cast<const uint16_t*>(x->wb[l].p(1)) : nullptr;
      Bd.alo_ld = (int)((l < L - 1 ? 2 : 1) * G4p);
      Bd.alo_rows = Hp;
      Bd.dgop[p] = x->dgop[l].p(p);
    }
    Bd.has_up = l < L - 1;
    Bd.dy = l == L - 1 ? x->dy_raw.f() : nullptr;
    Bd.gates = x->gates[l].f();
    Bd.tanhc = x->tanhc[l].f();
    Bd.c = x->c[l].f();
    Bd.dg = x->dg[l].f();
    Bd.carry_c = x->carry_c[l].f();
    Bd.dbp = x->dbp[l].f();
    Bd.dh0 = x->dh0[l].f();
    Bd.dc0 = x->dc0[l].f();
    Bd.flags = fb + (size_t)l * T;
    if (ls && l < L - 1) {
      Bd.dabove = x->dabove.f();
      Bd.akofs = (int)(G4p / aK);  // R^T after W_{l+1}^T in the packed [W_{l+1}^T | R_l^T]
    }
    if (!x->dgsw.empty()) {
      Bd.dgsw = static_cast<uint8_t*>(x->dgsw[l].p);
      Bd.bupsw = l < L - 1 ? static_cast<const uint8_t*>(x->dgsw[l + 1].p) : nullptr;
    }
    // GRU / RNN tapes (cluster schedule); for LSTM / RNN dgr is dgw (aliases)
    Bd.h = x->h[l].f();
    Bd.dgwsw = Bd.dgsw;
    Bd.dgr = Bd.dg;
    for (int p = 0; p < 2; ++p) Bd.dgrop[p] = Bd.dgop[p];
    if (x->kind == kCellGru) {
      fl[l].zrh = x->zrh[l].f();
      Bd.zrh = x->zrh[l].f();
      Bd.dgr = x->dgr[l].f();
      Bd.dgwsw = static_cast<uint8_t*>(x->dgwsw[l].p);
      for (int p = 0; p < 2; ++p) Bd.dgrop[p] = x->dgrop[l].p(p);
    }
  }
  x->fwd_layers.alloc(sizeof(FwdLayer) * L);
  x->bwd_layers.alloc(sizeof(BwdLayer) * L);
  RW_CUDA(cudaMemcpy(x->fwd_layers.p, fl.data(), sizeof(FwdLayer) * L, cudaMemcpyHostToDevice));
  RW_CUDA(cudaMemcpy(x->bwd_layers.p, bl.data(), sizeof(BwdLayer) * L, cudaMemcpyHostToDevice));

  // ---- cluster schedule: per-layer off-partial rings and the off-critical group tables
  if (cl_f || cl_b) {
    x->cl_epoch.alloc(16);
    const int tiles_fw = Hp / kUnitsPerFwdTile, tiles_bw = ceil_div(Hp, kTileM);
    const size_t tmax = (size_t)std::max(tiles_fw, tiles_bw);
    float* ob = x->cl_offsum.f();
    uint32_t* db_ = static_cast<uint32_t*>(x->cl_done.p);
    uint32_t* cb_ = static_cast<uint32_t*>(x->cl_consumed.p);
    auto ring_of = [&](int l, int ko, int dir) {
      const size_t ll = (size_t)dir * L + l;
      ClRing r{};
      r.ring = ob + ll * tmax * x->cl_ring * Bp * kTileM;
      r.done = db_ + ll * tmax * T;
      r.consumed = cb_ + ll * tmax * 32;
      r.ko = ko;
      r.sys = 0;
      return r;
    };
    if (cl_f) {
      x->ring_f_h.resize(L);
      x->off_f_h.assign(L, ClOff{});
      for (int l = 0; l < L; ++l) {
        const int Ipl = l == 0 ? Ip : Hp;
        x->ring_f_h[l] = ring_of(l, ko_f[l], 0);
        ClOff& o = x->off_f_h[l];
        o.a = fl[l].a[0];
        o.kdim = Ipl;
        o.op = fl[l].bxsw;
        o.op_blk_off = fl[l].bx_blk_off;
        o.op_flags = l > 0 ? fl[l - 1].flags : nullptr;
        o.ring = x->ring_f_h[l].ring;
        o.done = x->ring_f_h[l].done;
        o.consumed = x->ring_f_h[l].consumed;
        o.active = 1;
        // W.x (layer 0) or W.h_{l-1}: operand scales of the fp16x2 planes (common.cuh)
        o.unscale = x->prec == kF16x2 ? pow2f(-(kWScaleLog2 + (l == 0 ? kXScaleLog2 : kHScaleLog2))) : 1.0f;
        o.alo = fl[l].alo;
        o.alo_ld = fl[l].alo_ld;
        o.alo_rows = fl[l].alo_rows;
        o.ko = ko_f[l];
      }
      x->rows_f = L;
    }
    if (cl_b) {
      x->ring_b_h.resize(L);
      x->off_b_h.assign(L, ClOff{});
      for (int l = 0; l < L; ++l) {
        const bool up = l < L - 1;
        x->ring_b_h[l] = ring_of(l, up ? ko_b[l] : 0, 1);
        if (!up) continue;  // the top layer adds dy instead
        ClOff& o = x->off_b_h[l];
        o.a = bl[l].a[0];
        o.kdim = 4 * Hp;
        // W_{l+1}^T multiplies the W-side gradients of layer l + 1 (GRU: dgw, not dgr)
        o.op = static_cast<const uint8_t*>(x->kind == kCellGru ? x->dgwsw[l + 1].p : x->dgsw[l + 1].p);
        o.op_blk_off = 0;
        o.op_flags = bl[l + 1].flags;
        o.ring = x->ring_b_h[l].ring;
        o.done = x->ring_b_h[l].done;
        o.consumed = x->ring_b_h[l].consumed;
        o.active = 1;
        o.unscale = x->prec == kF16x2 ? pow2f(-(kWScaleLog2 + kGScaleLog2)) : 1.0f;  // W_{l+1}^T.dG
        o.alo = bl[l].alo;
        o.alo_ld = bl[l].alo_ld;
        o.alo_rows = bl[l].alo_rows;
        o.ko = ko_b[l];
      }
      x->rows_b = L;
    }
    upload_cluster_tables(x);
  }

  // ---- GEMM tables: weight gradients (grouped, MN-major A and B) and dx0 (K-major)
  std::vector<GemmDesc> wg;
  for (int l = 0; l < L; ++l) {
    const int Il = l == 0 ? I : H, Ipl = l == 0 ? Ip : Hp;
    GemmDesc d{};
    d.error = static_cast<int*>(x->errflag.p);
    for (int p = 0; p < 2; ++p) {
      const int q = p % x->planes;
      if (kmajor_wg) {
        d.a[p] = mp(m_dgT[2 * l + q], p);
        d.b[p] = l == 0 ? mp(m_xT[q], p) : mp(m_hT[2 * (l - 1) + q], p);
      } else {
        d.a[p] = mp(m_dgMN[2 * l + q], p);
        d.b[p] = l == 0 ? mp(m_xMN[q], p) : mp(m_hopMN[2 * (l - 1) + q], p);
      }
    }
    d.M = (int)G4p;
    d.N = Ipl;
    d.K = (int)colsT;
    d.a_k_off = 0;
    d.b_k_off = l == 0 ? 0 : Bp;  // X_l = h_{l-1} blocks 1..T
    d.d = x->dW[l].f();
    d.ldd = (long long)x->G * H;
    // fp16x2: dG planes carry 2^kGScaleLog2, x 2^kXScaleLog2, h 2^kHScaleLog2 (common.cuh)
    d.alpha = x->prec == kF16x2 ? pow2f(-(kGScaleLog2 + (l == 0 ? kXScaleLog2 : kHScaleLog2))) : 1.0f;
    d.row_mode = kRowGateUnperm;
    d.col_mode = kColIdentity;
    d.H = H;
    d.Hp = Hp;
    d.B = B;
    d.Bp = Bp;
    d.m_valid = x->G * H;
    d.gates = x->G;
    d.n_valid = Il;
    wg.push_back(d);
    GemmDesc r = d;
    for (int p = 0; p < 2; ++p) {
      r.b[p] = kmajor_wg ? mp(m_hT[2 * l + (p % x->planes)], p) : mp(m_hopMN[2 * l + (p % x->planes)], p);
      // dR = dgr h^T (GRU: dgr != dgw)
      r.a[p] = kmajor_wg ? mp(m_dgrT[2 * l + (p % x->planes)], p) : mp(m_dgrMN[2 * l + (p % x->planes)], p);
    }
    r.N = Hp;
    r.b_k_off = 0;  // Hprev = blocks 0..T-1
    r.alpha = x->prec == kF16x2 ? pow2f(-(kGScaleLog2 + kHScaleLog2)) : 1.0f;
    r.d = x->dR[l].f();
    r.n_valid = H;
    wg.push_back(r);
  }
  x->n_wg = (int)wg.size();
  if (ls) {  // per-layer input GEMMs (forward W_l.X_l, backward W_{l+1}^T.dG_{l+1})
    std::vector<GemmDesc> lf(L), lb(L);
    for (int l = 0; l < L; ++l) {
      const int Ipl = l == 0 ? Ip : Hp;
      GemmDesc& f = lf[l];
      f.error = static_cast<int*>(x->errflag.p);
      for (int p = 0; p < 2; ++p) {
        const int q = p % x->planes;
        f.a[p] = mp(m_wf[2 * l + q], p);
        f.b[p] = l == 0 ? mp(m_xLS[q], p) : mp(m_hopLS[2 * (l - 1) + q], p);
      }
      f.M = (int)G4p;
      f.N = (int)colsT;
      f.K = Ipl;
      f.b_n_off = l == 0 ? 0 : Bp;  // h_{l-1,t} is column block t+1
      f.d = x->gates[l].f();
      f.ldd = G4p;
      f.row_mode = kRowGatePad;
      f.col_mode = kColIdentity;
      f.H = H;
      f.Hp = Hp;
      f.B = B;
      f.Bp = Bp;
      f.m_valid = (int)G4p;
      f.n_valid = (int)colsT;
      if (l < L - 1) {
        GemmDesc& g = lb[l];
        g.error = static_cast<int*>(x->errflag.p);
        for (int p = 0; p < 2; ++p) {
          const int q = p % x->planes;
          g.a[p] = mp(m_wb[2 * l + q], p);
          g.b[p] = mp(m_dgLS[2 * (l + 1) + q], p);
        }
        g.M = Hp;
        g.N = (int)colsT;
        g.K = (int)G4p;
        g.d = x->dabove.f();
        g.ldd = Hp;
        g.row_mode = kRowIdentity;
        g.col_mode = kColIdentity;
        g.H = H;
        g.Hp = Hp;
        g.B = B;
        g.Bp = Bp;
        g.m_valid = Hp;
        g.n_valid = (int)colsT;
      }
    }
    x->gemm_lsf.alloc(sizeof(GemmDesc) * L);
    x->gemm_lsb.alloc(sizeof(GemmDesc) * L);
    RW_CUDA(cudaMemcpy(x->gemm_lsf.p, lf.data(), sizeof(GemmDesc) * L, cudaMemcpyHostToDevice));
    RW_CUDA(cudaMemcpy(x->gemm_lsb.p, lb.data(), sizeof(GemmDesc) * L, cudaMemcpyHostToDevice));
  }
  if (x->fwd_batch) {  // batched input projections of the stepwise forward (run_forward_rec)
    const int sb = x->fwd_batch, nb = ceil_div(T, sb);
    std::vector<GemmDesc> fb;
    for (int l = 0; l < L; ++l) {
      const int Ipl = l == 0 ? Ip : Hp;
      GemmDesc f{};
      f.error = static_cast<int*>(x->errflag.p);
      for (int p = 0; p < 2; ++p) {
        const int q = p % x->planes;
        f.a[p] = mp(m_wf[2 * l + q], p);
        f.b[p] = l == 0 ? mp(m_xLS[q], p) : mp(m_hopLS[2 * (l - 1) + q], p);
      }
      f.M = (int)G4p;
      f.K = Ipl;
      f.ldd = G4p;
      f.row_mode = kRowGatePad;
      f.col_mode = kColIdentity;
      f.H = H;
      f.Hp = Hp;
      f.B = B;
      f.Bp = Bp;
      f.m_valid = (int)G4p;
      // fp16x2: the operand planes carry 2^kWScaleLog2 x (2^kXScaleLog2 | 2^kHScaleLog2)
      f.alpha = x->prec == kF16x2 ? pow2f(-(kWScaleLog2 + (l == 0 ? kXScaleLog2 : kHScaleLog2))) : 1.0f;
      for (int b = 0; b < (l == 0 ? 1 : nb); ++b) {
        GemmDesc g = f;
        const int c0 = l == 0 ? 0 : b * sb, nc = l == 0 ? T : std::min(sb, T - c0);
        g.N = nc * Bp;
        g.n_valid = nc * Bp;
        g.b_n_off = (l == 0 ? 0 : Bp) + c0 * Bp;  // h_{l-1,t} is column block t+1
        g.d = x->gates[l].f() + (size_t)c0 * Bp * G4p;
        fb.push_back(g);
      }
    }
    x->gemm_fb.alloc(sizeof(GemmDesc) * fb.size());
    RW_CUDA(cudaMemcpy(x->gemm_fb.p, fb.data(), sizeof(GemmDesc) * fb.size(), cudaMemcpyHostToDevice));
  }
  x->gemm_wg.alloc(sizeof(GemmDesc) * wg.size());
  RW_CUDA(cudaMemcpy(x->gemm_wg.p, wg.data(), sizeof(GemmDesc) * wg.size(), cudaMemcpyHostToDevice));
  GemmDesc dx{};
  dx.error = static_cast<int*>(x->errflag.p);
  for (int p = 0; p < 2; ++p) {
    dx.a[p] = mp(m_w0t[p % x->planes], p);
    dx.b[p] = mp(m_dg0dx[p % x->planes], p);
  }
  dx.M = Ip;
  dx.N = (int)colsT;
  dx.K = (int)G4p;
  dx.d = x->dx0.f();
  dx.ldd = I;
  dx.row_mode = kRowIdentity;
  dx.col_mode = kColBatchUnpad;
  dx.H = H;
  dx.Hp = Hp;
  dx.B = B;
  dx.Bp = Bp;
  dx.m_valid = I;
  // W_0^T planes carry 2^kWScaleLog2, the dG planes 2^kGScaleLog2
  dx.alpha = f16x2 ? 1.0f / (float)(1 << (kWScaleLog2 + kGScaleLog2)) : 1.0f;
  dx.n_valid = (int)colsT;
  x->gemm_dx.alloc(sizeof(GemmDesc));
  RW_CUDA(cudaMemcpy(x->gemm_dx.p, &dx, sizeof(GemmDesc), cudaMemcpyHostToDevice));
  if (x->prec == kBF16) {
    // 256-column tiles run as CTA pairs (k_gemm_p2: 1.17 vs 0.77 PFLOP/s at config E's dR shape,
    // profiles/gemm_bench.py) once there are enough pair tiles to fill the SMs
    const long long pair_tiles = (long long)x->n_wg * ceil_div(4 * x->Hp, 2 * kTileM) *
                                 ceil_div(std::max(x->Hp, x->Ip), 256);
    x->bn_wg = pair_tiles >= 148 ? 256 : 128;
    if (const char* e = getenv("RW_BN_WG")) x->bn_wg = atoi(e);
  }
  x->st_wg = gemm_stages(x->planes, x->bn_wg);
  x->st_dx = gemm_stages(x->planes, x->bn_dx);

  // ---- streams
  RW_CUDA(cudaStreamCreateWithFlags(&x->main, cudaStreamNonBlocking));
  // per-layer streams only for the stepwise wavefront: every stream takes a hardware work queue,
  // and once a process has more streams than CUDA_DEVICE_MAX_CONNECTIONS (default 8) unrelated
  // streams share queues -- which serialised two pipeline stages' persistent kernels
  if (x->fwd_sched == RW_SCHED_STEPWISE || x->bwd_sched == RW_SCHED_STEPWISE) {
    x->ls.resize(L);
    x->lev.resize(L);
    for (int l = 0; l < L; ++l) {
      RW_CUDA(cudaStreamCreateWithFlags(&x->ls[l], cudaStreamNonBlocking));
      RW_CUDA(cudaEventCreateWithFlags(&x->lev[l], cudaEventDisableTiming));
    }
  }
  RW_CUDA(cudaEventCreateWithFlags(&x->fork_ev, cudaEventDisableTiming));
  RW_CUDA(cudaStreamCreateWithFlags(&x->tail_s, cudaStreamNonBlocking));
  RW_CUDA(cudaEventCreateWithFlags(&x->ev_tail_fork, cudaEventDisableTiming));
  RW_CUDA(cudaEventCreateWithFlags(&x->ev_tail_join, cudaEventDisableTiming));
  if (const char* e = getenv("RW_NO_GRAPHS")) x->use_graphs = atoi(e) == 0;
  if (const char* e = getenv("RW_TRACE")) x->trace_path = e;
  if (const char* e = getenv("RW_TRACE_SPANS")) x->trace_spans_path = e;
  if (!x->trace_path.empty() || !x->trace_spans_path.empty()) trace_alloc(x);
  if (const char* e = getenv("RW_DEBUG_HANG_S")) {
    x->hang_s = atof(e);
    RW_CUDA(cudaHostAlloc((void**)&x->progress_host, 4 * 4096 * sizeof(unsigned), cudaHostAllocMapped));
    std::memset(x->progress_host, 0, 4 * 4096 * sizeof(unsigned));
    RW_CUDA(cudaHostGetDevicePointer((void**)&x->progress_dev, x->progress_host, 0));
    x->use_graphs = false;
  }
}

// ------------------------------------------------------------------ phases
struct PhaseTimer {
  rw_ctx* x;
  int phase;
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  PhaseTimer(rw_ctx* ctx, int ph, cudaStream_t st) : x(ctx), phase(ph), s(st) {
    if (!x->profiling) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  ~PhaseTimer() {
    if (!x->profiling) return;
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    x->phase_ms[phase] += ms;
    x->phase_n[phase] += 1;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

void repack_params(rw_ctx* x, cudaStream_t s) {
  if (!x->dirty) return;
  const int L = x->L, H = x->H, I = x->I, Hp = x->Hp, Ip = x->Ip;
  if (!x->repack_njobs) {
    // one launch for every layer's forward / backward images and bias plus W_0^T (k_repack)
    std::vector<RepackJob> jobs;
    int tiles = 0;
    auto add = [&](RepackJob j, int n) {
      j.tile0 = tiles;
      tiles += n;
      jobs.push_back(j);
    };
    for (int l = 0; l < L; ++l) {
      const int Il = l == 0 ? I : H, Ipl = l == 0 ? Ip : Hp;
      RepackJob f{};
      f.kind = kRepackT;
      f.rows = 4 * Hp;
      f.K = Ipl + Hp;
      f.tiles_k = ceil_div(f.K, kRepackTileK);
      f.k_split = Ipl;
      f.src_k0 = Il;
      f.s0 = x->W[l].f();
      f.s1 = x->R[l].f();
      f.p0 = x->wf[l].p(0);
      f.p1 = x->wf[l].p(1);
      add(f, (f.rows / 32) * f.tiles_k);
      RepackJob b{};
      b.kind = kRepackC;
      b.rows = Hp;
      const bool up = l < L - 1 || x->pp_up;  // pipeline: the next stage's W_0 above the top layer
      b.K = (up ? 2 : 1) * 4 * Hp;
      b.tiles_k = ceil_div(b.K, kRepackTileK);
      b.src_rows = H;
      b.src_k0 = 4 * Hp;
      b.s0 = l < L - 1 ? x->W[l + 1].f() : up ? x->pp_wnext : nullptr;
      b.s1 = x->R[l].f();
      b.p0 = x->wb[l].p(0);
      b.p1 = x->wb[l].p(1);
      add(b, ceil_div(b.rows, 32) * b.tiles_k);
      RepackJob c{};
      c.kind = kRepackB;
      c.K = 4 * Hp;
      c.s0 = x->bias_raw[l].f();
      c.p0 = x->bias[l].f();
      add(c, ceil_div(c.K, 1024));
    }
    RepackJob t{};
    t.kind = kRepackC;
    t.rows = Ip;
    t.K = 4 * Hp;
    t.tiles_k = ceil_div(t.K, kRepackTileK);
    t.src_rows = I;
    t.src_k0 = 4 * Hp;
    t.s0 = x->W[0].f();
    t.p0 = x->w0t.p(0);
    t.p1 = x->w0t.p(1);
    add(t, ceil_div(t.rows, 32) * t.tiles_k);
    x->repack_jobs.alloc(jobs.size() * sizeof(RepackJob));
    RW_CUDA(cudaMemcpy(x->repack_jobs.p, jobs.data(), jobs.size() * sizeof(RepackJob), cudaMemcpyHostToDevice));
    x->repack_njobs = (int)jobs.size();
    x->repack_tiles = tiles;
  }
  ++g_launches;
  k_repack<<<x->repack_tiles, 256, 0, s>>>(static_cast<const RepackJob*>(x->repack_jobs.p), x->repack_njobs, H, Hp,
                                           x->G, x->prec);
  if (x->pp_prev && x->wb_prev.p) {  // backward boundary group: [W_0^T | R_0^T] of this stage
    ++g_launches;
    k_pack_wb<<<grid_for((long long)Hp * 8 * Hp), 256, 0, s>>>(x->W[0].f(), x->R[0].f(), H, Hp, x->prec,
                                                             x->wb_prev.p, x->wb_prev_lo.p, x->G);
  }
  RW_CUDA(cudaGetLastError());
  x->dirty = false;
}

RecParams rec_params(rw_ctx* x, bool fwd) {
  RecParams rp{};
  rp.kind = x->kind;
  rp.L = x->L;
  rp.H = x->H;
  rp.Hp = x->Hp;
  rp.B = x->B;
  rp.Bp = x->Bp;
  rp.T = x->T;
  rp.ksplit = fwd ? x->ks_f : x->ks_b;
  rp.tiles = fwd ? x->Hp / kUnitsPerFwdTile : ceil_div(x->Hp, kTileM);
  rp.stages = fwd ? x->st_f : x->st_b;
  rp.a_slots = fwd ? x->slots_f : x->slots_b;
  rp.acc_kb = fwd ? x->acckb_f : x->acckb_b;
  rp.n_acc = fwd ? x->nacc_f : x->nacc_b;
  rp.promo = fwd ? x->promo_f : x->promo_b;
  rp.us_in0 = rp.us_in = rp.us_rec = 1.0f;
  if (x->prec == kF16x2) {  // the drain's per-segment unscale (common.cuh operand scales)
    rp.us_in0 = pow2f(-(kWScaleLog2 + (fwd ? kXScaleLog2 : kGScaleLog2)));
    rp.us_in = pow2f(-(kWScaleLog2 + (fwd ? kHScaleLog2 : kGScaleLog2)));
    rp.us_rec = pow2f(-(kWScaleLog2 + (fwd ? kHScaleLog2 : kGScaleLog2)));
  }
  rp.gmax = fwd ? nullptr : static_cast<unsigned*>(x->errflag.p) + 2;
  rp.flag_target = (uint32_t)(rp.tiles * rp.ksplit);
  rp.acc_dbuf = 1;
  if (const char* e = getenv("RW_ACC_DBUF")) rp.acc_dbuf = atoi(e);
  if (fwd && x->pp_plain && x->pp_prev) {  // layer 0's input is the previous stage's h_t
    rp.pp_in_flags = static_cast<const uint32_t*>(x->xin_flags.p);
    rp.pp_epoch = static_cast<const uint32_t*>(x->cl_epoch.p);
    rp.us_in0 = rp.us_in;  // fp16x2: h planes (2^kHScaleLog2), not x
  }
  if (!fwd && x->pp_up) {  // the top layer's d_above comes from the next stage
    rp.pp_in_flags = static_cast<const uint32_t*>(x->dgin_flags.p);
    rp.pp_epoch = static_cast<const uint32_t*>(x->cl_epoch.p) + 1;
  }
  rp.a_prefetch = 0;  // measured: no gain at config E (0 4 8 16 32 -> 727 702 694 701 660 TFLOP/s)
  if (const char* e = getenv("RW_A_PREFETCH")) rp.a_prefetch = atoi(e);
  rp.error = static_cast<int*>(x->errflag.p);
  rp.progress = x->progress_dev;
  rp.trace = nullptr;
  if (x->tracing) rp.trace = static_cast<unsigned long long*>((fwd ? x->trace_f : x->trace_b).p);
  rp.timeout_ns = 20ULL * 1000000000ULL;
  if (const char* e = getenv("RW_FLAG_TIMEOUT_MS")) rp.timeout_ns = 1000000ULL * strtoull(e, nullptr, 10);
  return rp;
}

// x_op / tapes for a forward: h/c block 0 from h0/c0 (already staged on device as raw H x B
// per layer at stage + l*H*B) or zeros.
// `state`: also write block 0 (h0 / c0, zeros when null) of every layer's h, c, h-operand (and
// its swizzled image). The graph-replayed passes leave it out: block 0 is written by nothing
// else, so enqueue_pass re-zeroes it eagerly only after an rw_forward with explicit h0 / c0.
void forward_prologue(rw_ctx* x, cudaStream_t s, const float* h0_dev, const float* c0_dev, bool state = true,
                      bool inputs = true) {
  const int L = x->L, H = x->H, B = x->B, Hp = x->Hp, Bp = x->Bp;
  // range records of the fp16x2 planes written below (max|x|, max|h0|; check_error_flag)
  if (x->prec == kF16x2 && (inputs || state))
    RW_CUDA(cudaMemsetAsync(static_cast<unsigned*>(x->errflag.p) + (inputs ? 3 : 4), 0, inputs && state ? 8 : 4, s));
  // cluster schedule (bf16): the plain operand and its swizzled image in one pass
  const bool fused_x = inputs && !x->pp_prev && x->fwd_sched == RW_SCHED_CLUSTER &&
                       (x->prec == kBF16 || x->prec == kF16x2) && x->Ip % 8 == 0;
  if (fused_x && x->prec == kBF16) {
    ++g_launches;
    k_pad_swizzle_bf16<<<grid_for((long long)x->Ip / 8 * Bp * x->T), 256, 0, s>>>(
        x->x_raw.f(), x->I, B, x->T, x->Ip, Bp, static_cast<__nv_bfloat16*>(x->x_op.p(0)),
        static_cast<uint8_t*>(x->xsw.p));
  } else if (fused_x) {
    ++g_launches;
    k_pad_swizzle_f16x2<<<grid_for((long long)x->Ip / 8 * Bp * x->T), 256, 0, s>>>(
        x->x_raw.f(), x->I, B, x->T, x->Ip, Bp, static_cast<__half*>(x->x_op.p(0)), static_cast<__half*>(x->x_op.p(1)),
        static_cast<uint8_t*>(x->xsw.p), pow2f(kXScaleLog2), static_cast<unsigned*>(x->errflag.p) + 3);
  } else if (inputs && !x->pp_prev) {  // a pipeline stage's layer input is written by the previous stage
    ++g_launches;
    k_pad_cols<<<pad_grid((long long)x->Ip * Bp * x->T), 256, 0, s>>>(
        x->x_raw.f(), x->I, B, x->T, x->Ip, Bp, 0, nullptr, x->prec, x->x_op.p(0), x->x_op.p(1),
        pow2f(kXScaleLog2), static_cast<unsigned*>(x->errflag.p) + 3);
  }
  for (int l = 0; l < L && state; ++l) {
    const float* h0 = h0_dev ? h0_dev + (size_t)l * H * B : nullptr;
    const float* c0 = c0_dev ? c0_dev + (size_t)l * H * B : nullptr;
    ++g_launches;
    k_pad_cols<<<pad_grid((long long)Hp * Bp), 256, 0, s>>>(h0, H, B, 1, Hp, Bp, 0, x->h[l].f(), x->prec,
                                                           x->hop[l].p(0), x->hop[l].p(1), pow2f(kHScaleLog2),
                                                           static_cast<unsigned*>(x->errflag.p) + 4);
    ++g_launches;
    k_pad_cols<<<pad_grid((long long)Hp * Bp), 256, 0, s>>>(c0, H, B, 1, Hp, Bp, 0, x->c[l].f(), x->prec,
                                                           nullptr, nullptr);
  }
  if (inputs && !fused_x && x->fwd_sched == RW_SCHED_CLUSTER && !x->pp_prev) {  // pre-swizzled images of x
    const long long colsT = (long long)Bp * x->T;
    ++g_launches;
    k_swizzle_op<<<grid_for((long long)x->Ip / 8 * colsT * x->planes), 256, 0, s>>>(
        static_cast<const uint16_t*>(x->x_op.p(0)), static_cast<const uint16_t*>(x->x_op.p(1)), x->Ip, Bp, 0, colsT,
        static_cast<uint8_t*>(x->xsw.p));
  }
  if (state && x->fwd_sched == RW_SCHED_CLUSTER) {
    for (int l = 0; l < L; ++l, ++g_launches)
      k_swizzle_op<<<grid_for((long long)Hp / 8 * Bp * x->planes), 256, 0, s>>>(
          static_cast<const uint16_t*>(x->hop[l].p(0)), static_cast<const uint16_t*>(x->hop[l].p(1)), Hp, Bp, 0, Bp,
          static_cast<uint8_t*>(x->hsw[l].p));
  }
  RW_CUDA(cudaGetLastError());
}

ClParams cl_params(rw_ctx* x, bool fwd) {
  ClParams p{};
  p.L = x->L;
  p.H = x->H;
  p.Hp = x->Hp;
  p.B = x->B;
  p.Bp = x->Bp;
  p.T = x->T;
  const ClPlan& pl = fwd ? x->cl_f : x->cl_b;
  p.tiles = fwd ? x->Hp / kUnitsPerFwdTile : ceil_div(x->Hp, kTileM);
  p.kc = pl.kc;
  p.cs = pl.cs;
  p.ncomax = pl.ncomax;
  p.stages = pl.stages;
  p.stages_off = pl.stages_off;
  p.st_alias = pl.st_alias;
  p.st_off = pl.st_off;
  p.ring = x->cl_ring;
  p.n_crit = x->L;
  p.cring = static_cast<const ClRing*>((fwd ? x->cl_ring_f : x->cl_ring_b).p);
  p.offg = static_cast<const ClOff*>((fwd ? x->cl_off_f : x->cl_off_b).p);
  p.epoch = static_cast<const uint32_t*>(x->cl_epoch.p) + (fwd ? 0 : 1);
  p.error = static_cast<int*>(x->errflag.p);
  p.timeout_ns = 20ULL * 1000000000ULL;
  if (const char* e = getenv("RW_FLAG_TIMEOUT_MS")) p.timeout_ns = 1000000ULL * strtoull(e, nullptr, 10);
  p.trace = nullptr;
  if (x->tracing) p.trace = static_cast<unsigned long long*>((fwd ? x->trace_f : x->trace_b).p);
  p.trace_steps = fwd ? x->T : x->T + 1;
  if (const char* e = getenv("RW_CL_DEBUG")) p.debug = atoi(e);
  p.dir = fwd ? 0 : 1;
  p.unscale = 1.0f;
  if (x->prec == kF16x2) p.unscale = pow2f(-(kWScaleLog2 + (fwd ? kHScaleLog2 : kGScaleLog2)));
  p.gmax = fwd ? nullptr : static_cast<unsigned*>(x->errflag.p) + 2;
  p.kind = x->kind;
  return p;
}

// Counters of the cluster schedule are cumulative (targets = epoch * per-pass count), so no
// per-pass memset races a pipeline neighbour that already writes into this context's rings.
void launch_cluster(rw_ctx* x, void* kernel, const void* layers, const ClParams& p, int rows, size_t smem,
                    cudaStream_t s, bool fwd) {
  ++g_launches;
  k_epoch_inc<<<1, 1, 0, s>>>(static_cast<uint32_t*>(x->cl_epoch.p) + (fwd ? 0 : 1), p.gmax);
  RW_CUDA(cudaGetLastError());
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(p.tiles * 2 * p.cs, rows, 1);
  lc.blockDim = dim3(kRecThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  void* args[2] = {const_cast<void**>(&layers), const_cast<ClParams*>(&p)};
  ++g_launches;
  RW_CUDA(cudaLaunchKernelExC(&lc, kernel, args));
}

void run_forward_cluster(rw_ctx* x, cudaStream_t s) {
  launch_cluster(x, x->cl_f.kern, x->fwd_layers.p, cl_params(x, true), x->rows_f, x->cl_f.smem, s, true);
  if (x->pp_next_xop) {  // next stage's layer input (its dW_0 operand): h_{last, 0..T-1}, plain planes
    RW_CUDA(cudaMemcpyAsync(x->pp_next_xop, static_cast<uint8_t*>(x->hop[x->L - 1].p(0)) + (size_t)x->Hp * x->Bp * 2,
                            (size_t)x->Hp * x->Bp * x->T * 2, cudaMemcpyDefault, s));
    if (x->pp_next_xop_lo)
      RW_CUDA(cudaMemcpyAsync(x->pp_next_xop_lo,
                              static_cast<uint8_t*>(x->hop[x->L - 1].p(1)) + (size_t)x->Hp * x->Bp * 2,
                              (size_t)x->Hp * x->Bp * x->T * 2, cudaMemcpyDefault, s));
    ++g_launches;
    k_pp_signal<<<1, 1, 0, s>>>(x->pp_next_ready, static_cast<const uint32_t*>(x->cl_epoch.p));
    RW_CUDA(cudaGetLastError());
  }
}

template <class P>
void run_forward_rec_body(rw_ctx* x, cudaStream_t s, bool training);
template <class P>
void run_backward_rec_body(rw_ctx* x, cudaStream_t s);

// Pipeline stages on the persistent / stepwise schedules count their passes (the targets of the
// cumulative peer counters) and, after the forward, tell the next stage its input landed.
template <class P>
void run_forward_rec(rw_ctx* x, cudaStream_t s, bool training) {
  const bool pp = x->pp_plain && (x->pp_prev || x->pp_next);
  if (pp) {
    ++g_launches;
    k_epoch_inc<<<1, 1, 0, s>>>(static_cast<uint32_t*>(x->cl_epoch.p));
  }
  run_forward_rec_body<P>(x, s, training);
  if (pp && x->pp_next) {
    ++g_launches;
    k_pp_signal<<<1, 1, 0, s>>>(x->pp_next_ready, static_cast<const uint32_t*>(x->cl_epoch.p));
  }
  RW_CUDA(cudaGetLastError());
}
template <class P>
void run_backward_rec(rw_ctx* x, cudaStream_t s) {
  if (x->pp_plain && x->pp_up) {
    ++g_launches;
    k_epoch_inc<<<1, 1, 0, s>>>(static_cast<uint32_t*>(x->cl_epoch.p) + 1);
  }
  run_backward_rec_body<P>(x, s);
}

template <class P>
void run_forward_rec_body(rw_ctx* x, cudaStream_t s, bool training) {
  if (x->fwd_sched == RW_SCHED_CLUSTER) {
    run_forward_cluster(x, s);
    return;
  }
  {
  if (x->fwd_sched == RW_SCHED_LAYERSEQ) {
    RecParams rp = rec_params(x, true);
    void* kern = lstm_kernel_ptr(x->prec, true, false, x->kind);
    rp.resident = 0;
    // one persistent launch per layer (its tiles x ksplit CTAs co-resident, flag-synchronised
    // steps, R streamed from L2 -- one layer's weights fit there) unless RW_LS_PERSISTENT=0:
    // then one launch per step
    const bool pers = x->ls_pers_f;
    rp.persistent = pers ? 1 : 0;
    rp.n_steps = pers ? x->T : 1;
    if (pers) RW_CUDA(cudaMemsetAsync(x->flags_f.p, 0, x->flags_f.bytes, s));
    const GemmDesc* G = static_cast<const GemmDesc*>(x->gemm_lsf.p);
    for (int l = 0; l < x->L; ++l) {
      launch_gemm<P, false, false>(G + l, 1, 4 * x->Hp, x->Bp * x->T, x->bn_ls, gemm_stages(x->planes, x->bn_ls), s);
      rp.layer_base = l;
      for (int t = 0; t < (pers ? 1 : x->T); ++t) {
        rp.t_first = t;
        launch_rec<P>(kern, x->fwd_layers.p, rp, rp.tiles * rp.ksplit, 1, x->smem_f, s);
      }
    }
    return;
  }
  RecParams rp = rec_params(x, true);
  void* kern = lstm_kernel_ptr(x->prec, true, false, x->kind);
  // inference: no gate tapes (null gates pointer patched via a second descriptor table is
  // avoided by simply keeping the tapes; cost is HBM writes only)
  (void)training;
  if (x->fwd_sched == RW_SCHED_PERSISTENT) {
    RW_CUDA(cudaMemsetAsync(x->flags_f.p, 0, x->flags_f.bytes, s));
    rp.persistent = 1;
    rp.resident = x->res_f;
    rp.layer_base = 0;
    rp.t_first = 0;
    rp.n_steps = x->T;
    launch_rec<P>(kern, x->fwd_layers.p, rp, rp.tiles * rp.ksplit, x->L, x->smem_f, s);
    return;
  }
  // stepwise wavefront: layer l on stream ls[l]; step (l,t) waits for (l-1,t)
  if (x->pair_f) kern = lstm_kernel_ptr(kBF16, true, true);
  rp.persistent = 0;
  rp.resident = 0;
  rp.n_steps = 1;
  RW_CUDA(cudaEventRecord(x->fork_ev, s));
  for (int l = 0; l < x->L; ++l) RW_CUDA(cudaStreamWaitEvent(x->ls[l], x->fork_ev, 0));
  if (x->fwd_batch) {
    // blocks of sb steps: layer l's input GEMM for block b waits for layer l-1's block b, then the
    // block's step kernels (K = Hp: R only) follow on the layer's stream; layer 0's input
    // projection covers every step in one GEMM
    const int sb = x->fwd_batch, nb = ceil_div(x->T, sb);
    const GemmDesc* FB = static_cast<const GemmDesc*>(x->gemm_fb.p);
    const int st = gemm_stages(x->planes, x->bn_ls);
    launch_gemm<P, false, false>(FB, 1, 4 * x->Hp, x->Bp * x->T, x->bn_ls, st, x->ls[0]);
    for (int b = 0; b < nb; ++b) {
      const int t0 = b * sb, t1 = std::min(x->T, t0 + sb);
      for (int l = 0; l < x->L; ++l) {
        if (l > 0) {
          RW_CUDA(cudaStreamWaitEvent(x->ls[l], x->lev[l - 1], 0));
          launch_gemm<P, false, false>(FB + 1 + (size_t)(l - 1) * nb + b, 1, 4 * x->Hp, x->Bp * (t1 - t0), x->bn_ls, st,
                                       x->ls[l]);
        }
        rp.layer_base = l;
        for (int t = t0; t < t1; ++t) {
          rp.t_first = t;
          if (x->tracing) rp.trace = x->trace_f.u64() + (size_t)(l * x->T + t) * rp.tiles * rp.ksplit * 8;
          launch_rec<P>(kern, x->fwd_layers.p, rp, rp.tiles * rp.ksplit, 1, x->smem_f, x->ls[l], x->pair_f ? 2 : 0);
        }
        RW_CUDA(cudaEventRecord(x->lev[l], x->ls[l]));
      }
    }
    for (int l = 0; l < x->L; ++l) RW_CUDA(cudaStreamWaitEvent(s, x->lev[l], 0));
    return;
  }
  for (int t = 0; t < x->T; ++t) {
    for (int l = 0; l < x->L; ++l) {
      if (l > 0) RW_CUDA(cudaStreamWaitEvent(x->ls[l], x->lev[l - 1], 0));
      rp.layer_base = l;
      rp.t_first = t;
      // trace: one block of grid CTAs per (layer, step) launch (trace_records reads [l][t][cta])
      if (x->tracing) rp.trace = x->trace_f.u64() + (size_t)(l * x->T + t) * rp.tiles * rp.ksplit * 8;
      launch_rec<P>(kern, x->fwd_layers.p, rp, rp.tiles * rp.ksplit, 1, x->smem_f, x->ls[l], x->pair_f ? 2 : 0);
      RW_CUDA(cudaEventRecord(x->lev[l], x->ls[l]));
    }
  }
  for (int l = 0; l < x->L; ++l) RW_CUDA(cudaStreamWaitEvent(s, x->lev[l], 0));
  }
}

template <class P>
void run_backward_rec_body(rw_ctx* x, cudaStream_t s) {
  for (int l = 0; l < x->L; ++l) RW_CUDA(cudaMemsetAsync(x->dbp[l].p, 0, x->dbp[l].bytes, s));
  if (x->bwd_sched == RW_SCHED_CLUSTER) {
    launch_cluster(x, x->cl_b.kern, x->bwd_layers.p, cl_params(x, false), x->rows_b, x->cl_b.smem, s, false);
    return;
  }
  {
  if (x->prec == kF16x2) RW_CUDA(cudaMemsetAsync(static_cast<unsigned*>(x->errflag.p) + 2, 0, 4, s));  // max|dG|
  RecParams rp = rec_params(x, false);
  void* kern = lstm_kernel_ptr(x->prec, false, false, x->kind);
  if (x->bwd_sched == RW_SCHED_LAYERSEQ) {
    const bool pers = x->ls_pers_b;  // as in the forward
    rp.persistent = pers ? 1 : 0;
    rp.resident = 0;
    rp.n_steps = pers ? x->T + 1 : 1;
    if (pers) RW_CUDA(cudaMemsetAsync(x->flags_b.p, 0, x->flags_b.bytes, s));
    const GemmDesc* G = static_cast<const GemmDesc*>(x->gemm_lsb.p);
    for (int l = x->L - 1; l >= 0; --l) {
      if (l < x->L - 1)
        launch_gemm<P, false, false>(G + l, 1, x->Hp, x->Bp * x->T, x->bn_ls, gemm_stages(x->planes, x->bn_ls), s);
      rp.layer_base = l;
      for (int t = x->T - 1; t >= (pers ? x->T - 1 : -1); --t) {
        rp.t_first = t;
        launch_rec<P>(kern, x->bwd_layers.p, rp, rp.tiles * rp.ksplit, 1, x->smem_b, s);
      }
    }
    return;
  }
  if (x->bwd_sched == RW_SCHED_PERSISTENT) {
    RW_CUDA(cudaMemsetAsync(x->flags_b.p, 0, x->flags_b.bytes, s));
    rp.persistent = 1;
    rp.resident = x->res_b;
    rp.layer_base = 0;
    rp.t_first = x->T - 1;
    rp.n_steps = x->T + 1;  // T steps + the dh0 step
    if (x->pair_b)
      launch_rec<P>(lstm_kernel_ptr(kBF16, false, true), x->bwd_layers.p, rp, rp.tiles, x->L, x->smem_b, s, 2);
    else
      launch_rec<P>(kern, x->bwd_layers.p, rp, rp.tiles * rp.ksplit, x->L, x->smem_b, s);
    return;
  }
  rp.persistent = 0;
  rp.resident = 0;
  rp.n_steps = 1;
  RW_CUDA(cudaEventRecord(x->fork_ev, s));
  for (int l = 0; l < x->L; ++l) RW_CUDA(cudaStreamWaitEvent(x->ls[l], x->fork_ev, 0));
  for (int t = x->T - 1; t >= -1; --t) {
    for (int l = x->L - 1; l >= 0; --l) {
      if (l < x->L - 1 && t >= 0) RW_CUDA(cudaStreamWaitEvent(x->ls[l], x->lev[l + 1], 0));
      rp.layer_base = l;
      rp.t_first = t;
      if (x->tracing) rp.trace = x->trace_b.u64() + (size_t)(l * (x->T + 1) + (x->T - 1 - t)) * rp.tiles * rp.ksplit * 8;
      launch_rec<P>(kern, x->bwd_layers.p, rp, rp.tiles * rp.ksplit, 1, x->smem_b, x->ls[l]);
      RW_CUDA(cudaEventRecord(x->lev[l], x->ls[l]));
    }
  }
  for (int l = 0; l < x->L; ++l) RW_CUDA(cudaStreamWaitEvent(s, x->lev[l], 0));
  }
}

// ---- GPU optimisation ladder (the reference's run_ladder, bench.hpp:30-32,
// 176-224): seven forward-pass rungs, each adding one optimisation of the paper's Table 1.
//   O0 Naive            per step: 4 + 4 per-gate GEMMs (W_g.x_t, R_g.h_{t-1}) on the reference-
//                       layout weights, then the nine element-wise ops of the unfused cell (K8)
//                       as nine launches; layers and steps in sequence on one stream
//   O1 Grouped GEMMs    one GEMM per operand for all gates (M = G H)
//   O2 Streamed GEMMs   the W.x GEMMs on a second stream, running ahead of the recurrence
//   O3 Fused point-wise the whole cell in one launch
//   O4 Pre-transpose    the K7-packed K-major [W | R] and the fused GEMM + cell step kernel
//                       (k_lstm_fwd), layers in sequence
//   O5 Batching inputs  the layer-sequential schedule (one W.X GEMM per layer over all steps)
//   O6 Overlapping layers the wavefront (cluster / persistent / stepwise)
// O0-O4 run here on a context created with the stepwise schedule; O5 / O6 are rw_run_pass on
// contexts with the layer-sequential / automatic schedule (bench.py --ladder).
void ladder_init(rw_ctx* x) {
  auto& Lr = x->ladder;
  const int L = x->L, H = x->H, I = x->I, Hp = x->Hp, Bp = x->Bp, T = x->T, G = x->G, aK = x->atomK;
  const long long G4p = 4LL * Hp;
  Lr.wraw.resize(L);
  Lr.rraw.resize(L);
  std::vector<CUtensorMap> maps;
  for (int l = 0; l < L; ++l) {
    const int Il = l == 0 ? I : H;
    Lr.wraw[l].alloc(x->prec, (size_t)G * Hp * Il);
    Lr.rraw[l].alloc(x->prec, (size_t)G * Hp * H);
    for (int p = 0; p < 2; ++p) {
      const int q = p % x->planes;
      maps.push_back(make_map(Lr.wraw[l].p(q), x->prec, (long long)G * Hp, Il, aK, aK));  // MN-major A
      maps.push_back(make_map(Lr.rraw[l].p(q), x->prec, (long long)G * Hp, H, aK, aK));
    }
  }
  // B operands (x_t, h_t column blocks), K-major with boxes of the GEMM's bn rows (the context's own
  // maps use Bp-row boxes for the recurrent kernels); rows past the tensor are zero-filled and
  // columns past Bp are computed but not written (n_valid)
  const size_t nb = maps.size();
  const int bn = Bp <= 64 ? 64 : 128;
  const long long colsT = (long long)Bp * T, colsT1 = (long long)Bp * (T + 1);
  for (int p = 0; p < 2; ++p) maps.push_back(make_map(x->x_op.p(p % x->planes), x->prec, x->Ip, colsT, aK, gemm_box_rows(bn)));
  for (int l = 0; l < L; ++l)
    for (int p = 0; p < 2; ++p)
      maps.push_back(make_map(x->hop[l].p(p % x->planes), x->prec, Hp, colsT1, aK, gemm_box_rows(bn)));
  Lr.maps.alloc(maps.size() * sizeof(CUtensorMap));
  RW_CUDA(cudaMemcpy(Lr.maps.p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  const CUtensorMap* M = static_cast<const CUtensorMap*>(Lr.maps.p);
  // maps per layer: [W plane 0, R plane 0, W plane 1, R plane 1]
  auto mW = [&](int l, int p) { return p < x->planes ? M + 4 * l + 2 * p : nullptr; };
  auto mR = [&](int l, int p) { return p < x->planes ? M + 4 * l + 2 * p + 1 : nullptr; };
  auto mX = [&](int p) { return p < x->planes ? M + nb + p : nullptr; };
  auto mH = [&](int l, int p) { return p < x->planes ? M + nb + 2 + 2 * l + p : nullptr; };
  Lr.zw.alloc((size_t)G4p * Bp * T * 4);
  Lr.zr.alloc((size_t)G4p * Bp * 4);
  Lr.pre.alloc((size_t)G4p * Bp * 4);
  Lr.gates.alloc((size_t)G4p * Bp * 4);
  Lr.t1.alloc((size_t)Hp * Bp * 4);
  Lr.t2.alloc((size_t)Hp * Bp * 4);
  std::vector<GemmDesc> d((size_t)L * T * 10);
  const bool f16 = x->prec == kF16x2;
  for (int l = 0; l < L; ++l) {
    const int Il = l == 0 ? I : H;
    for (int t = 0; t < T; ++t)
      for (int k = 0; k < 10; ++k) {
        GemmDesc& g = d[((size_t)l * T + t) * 10 + k];
        const bool w = k < 4 || k == 8, grouped = k >= 8;
        const int gate = grouped ? 0 : (k & 3);
        for (int p = 0; p < 2; ++p) {
          g.a[p] = w ? mW(l, p) : mR(l, p);
          g.b[p] = w ? (l == 0 ? mX(p) : mH(l - 1, p)) : mH(l, p);
        }
        g.error = static_cast<int*>(x->errflag.p);
        g.a_m_off = grouped ? 0 : gate * Hp;
        g.M = grouped ? G * Hp : round_up(H, kTileM);
        g.N = Bp;
        g.K = w ? Il : H;
        g.b_n_off = w ? (l == 0 ? t * Bp : (t + 1) * Bp) : t * Bp;  // x_t, h_{l-1,t} (block t+1), h_{t-1}
        g.d = (w ? Lr.zw.f() + (size_t)t * Bp * G4p : Lr.zr.f()) + (grouped ? 0 : (size_t)gate * Hp);
        g.ldd = G4p;
        g.row_mode = kRowIdentity;
        g.col_mode = kColIdentity;
        g.H = H;
        g.Hp = Hp;
        g.B = x->B;
        g.Bp = Bp;
        g.m_valid = grouped ? G * Hp : H;
        g.n_valid = Bp;
        g.alpha = f16 ? pow2f(-(kWScaleLog2 + (w && l == 0 ? kXScaleLog2 : kHScaleLog2))) : 1.0f;
      }
  }
  Lr.desc.alloc(d.size() * sizeof(GemmDesc));
  RW_CUDA(cudaMemcpy(Lr.desc.p, d.data(), d.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice));
  Lr.ev.resize((size_t)L * T);
  for (auto& e : Lr.ev) RW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  RW_CUDA(cudaStreamCreateWithFlags(&Lr.side, cudaStreamNonBlocking));
  Lr.ready = true;
}

template <class P>
void run_ladder_forward(rw_ctx* x, int level, cudaStream_t s) {
  if (!x->ladder.ready) ladder_init(x);
  auto& Lr = x->ladder;
  const int L = x->L, H = x->H, I = x->I, Hp = x->Hp, Bp = x->Bp, T = x->T, G = x->G;
  const long long G4p = 4LL * Hp;
  const int bn = Bp <= 64 ? 64 : 128;
  const GemmDesc* D = static_cast<const GemmDesc*>(Lr.desc.p);
  auto gemm = [&](int l, int t, int k, int count, cudaStream_t st) {
    const GemmDesc* g = D + ((size_t)l * T + t) * 10 + k;
    const int M = k >= 8 ? G * Hp : round_up(H, kTileM);
    launch_gemm<P, true, false>(g, count, M, Bp, bn, gemm_stages(x->planes, bn), st);
  };
  // reference-layout operand planes of W, R (the "not pre-transposed" rungs read these)
  if (level <= 3) {
    for (int l = 0; l < L; ++l) {
      const int Il = l == 0 ? I : H;
      ++g_launches;
      k_pad_gates<<<grid_for((long long)G * Hp * Il), 256, 0, s>>>(x->W[l].f(), G, H, Hp, Il, x->prec, Lr.wraw[l].p(0),
                                                                    Lr.wraw[l].p(1), pow2f(kWScaleLog2));
      ++g_launches;
      k_pad_gates<<<grid_for((long long)G * Hp * H), 256, 0, s>>>(x->R[l].f(), G, H, Hp, H, x->prec, Lr.rraw[l].p(0),
                                                                   Lr.rraw[l].p(1), pow2f(kWScaleLog2));
    }
  }
  const int ew = grid_for((long long)G4p * Bp);
  for (int l = 0; l < L; ++l) {
    if (level == 4) {  // pre-transposed fused step kernels, layer after layer
      RecParams rp = rec_params(x, true);
      rp.persistent = 0;
      rp.resident = 0;
      rp.n_steps = 1;
      rp.layer_base = l;
      for (int t = 0; t < T; ++t) {
        rp.t_first = t;
        launch_rec<P>(KernelSet<P>::fwd(), x->fwd_layers.p, rp, rp.tiles * rp.ksplit, 1, x->smem_f, s,
                      x->pair_f ? 2 : 0);
      }
      continue;
    }
    if (level >= 2) {  // streamed: every step's W.x on the side stream, ahead of the recurrence
      RW_CUDA(cudaEventRecord(Lr.ev[(size_t)l * T], s));
      RW_CUDA(cudaStreamWaitEvent(Lr.side, Lr.ev[(size_t)l * T], 0));  // layer l - 1 finished
      for (int t = 0; t < T; ++t) {
        gemm(l, t, 8, 1, Lr.side);
        RW_CUDA(cudaEventRecord(Lr.ev[(size_t)l * T + t], Lr.side));
      }
    }
    for (int t = 0; t < T; ++t) {
      if (level == 0) {
        for (int g = 0; g < G; ++g) gemm(l, t, g, 1, s);
        for (int g = 0; g < G; ++g) gemm(l, t, 4 + g, 1, s);
      } else {
        if (level == 1) gemm(l, t, 8, 1, s);
        gemm(l, t, 9, 1, s);
        if (level >= 2) RW_CUDA(cudaStreamWaitEvent(s, Lr.ev[(size_t)l * T + t], 0));
      }
      const float* zwt = Lr.zw.f() + (size_t)t * Bp * G4p;
      float* cprev = x->c[l].f() + (size_t)t * Bp * Hp;
      float* cnew = cprev + (size_t)Bp * Hp;
      float* hnew = x->h[l].f() + (size_t)(t + 1) * Bp * Hp;
      const long long op_off = (long long)(t + 1) * Bp * Hp;
      if (level == 3) {
        ++g_launches;
        k_lstm_cell_fused<<<grid_for((long long)Hp * Bp), 256, 0, s>>>(zwt, Lr.zr.f(), x->bias[l].f(), cprev, cnew, hnew,
                                                                        H, Hp, Bp, x->prec, x->hop[l].p(0),
                                                                        x->hop[l].p(1), op_off);
        continue;
      }
      // the unfused cell: nine element-wise launches (cells.hpp:261-279 order)
      float* pre = Lr.pre.f();
      float* gt = Lr.gates.f();
      g_launches += 10;
      k_ew<<<ew, 256, 0, s>>>(kEwAdd, pre, (int)G4p, zwt, (int)G4p, Lr.zr.f(), (int)G4p, (int)G4p, Bp);
      k_ew<<<ew, 256, 0, s>>>(kEwAddBias, pre, (int)G4p, pre, (int)G4p, x->bias[l].f(), 0, (int)G4p, Bp);
      k_ew<<<ew, 256, 0, s>>>(kEwSigmoid, gt, (int)G4p, pre, (int)G4p, nullptr, 0, 3 * Hp, Bp);
      k_ew<<<ew, 256, 0, s>>>(kEwTanh, gt + 3 * Hp, (int)G4p, pre + 3 * Hp, (int)G4p, nullptr, 0, Hp, Bp);
      k_ew<<<ew, 256, 0, s>>>(kEwMul, Lr.t1.f(), Hp, gt + Hp, (int)G4p, cprev, Hp, Hp, Bp);
      k_ew<<<ew, 256, 0, s>>>(kEwMul, Lr.t2.f(), Hp, gt, (int)G4p, gt + 3 * Hp, (int)G4p, Hp, Bp);
      k_ew<<<ew, 256, 0, s>>>(kEwAdd, cnew, Hp, Lr.t1.f(), Hp, Lr.t2.f(), Hp, Hp, Bp);
      k_ew<<<ew, 256, 0, s>>>(kEwTanh, Lr.t1.f(), Hp, cnew, Hp, nullptr, 0, Hp, Bp);
      k_ew<<<ew, 256, 0, s>>>(kEwMul, hnew, Hp, gt + 2 * Hp, (int)G4p, Lr.t1.f(), Hp, Hp, Bp);
      void* p0 = static_cast<uint8_t*>(x->hop[l].p(0)) + (size_t)op_off * x->elem;
      void* p1 = x->hop[l].p(1) ? static_cast<uint8_t*>(x->hop[l].p(1)) + (size_t)op_off * x->elem : nullptr;
      k_store_h_operand<<<ew, 256, 0, s>>>(hnew, (long long)Hp * Bp, x->prec, p0, p1);
    }
  }
  RW_CUDA(cudaGetLastError());
}

template <class P>
void run_dx0(rw_ctx* x, cudaStream_t s) {
  if (x->tracing) k_stamp<<<1, 1, 0, s>>>(x->trace_dx.u64());
  launch_gemm<P, false, false>(static_cast<const GemmDesc*>(x->gemm_dx.p), 1, x->Ip,
                               x->Bp * x->T, x->bn_dx, x->st_dx, s);
  if (x->tracing) k_stamp<<<1, 1, 0, s>>>(x->trace_dx.u64() + 1);
}

void transpose_planes(rw_ctx* x, const Operand& src, int R, long long C, Operand& dst, cudaStream_t s) {
  dim3 grid(ceil_div(C, 32), ceil_div(R, 32));
  ++g_launches;
  k_transpose_planes<<<grid, dim3(32, 8), 0, s>>>(src.plane[0].f(), src.plane[1].f(), R, C,
                                                  dst.plane[0].f(), dst.plane[1].f());
}

// One layer's gradient bucket (dW_l, dR_l, db_l) summed over the data-parallel ranks.
void allreduce_layer(rw_ctx* x, int l, cudaStream_t s) {
  Nccl& n = nccl();
  const int Il = l == 0 ? x->I : x->H;
  nccl_check(n.GroupStart(), "ncclGroupStart");
  nccl_check(n.AllReduce(x->dW[l].p, x->dW[l].p, (unsigned long long)x->G * x->H * Il, kNcclFloat32, kNcclSum, x->comm, s), "ncclAllReduce dW");
  nccl_check(n.AllReduce(x->dR[l].p, x->dR[l].p, (unsigned long long)x->G * x->H * x->H, kNcclFloat32, kNcclSum, x->comm, s), "ncclAllReduce dR");
  nccl_check(n.AllReduce(x->db[l].p, x->db[l].p, (unsigned long long)x->G * x->H, kNcclFloat32, kNcclSum, x->comm, s), "ncclAllReduce db");
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
}


template <class P>
void run_weight_grads(rw_ctx* x, cudaStream_t s) {
  if (x->pp_prev) {  // layer input of a pipeline stage: copied in by the previous stage
    ++g_launches;
    const uint32_t* ep = static_cast<const uint32_t*>(x->cl_epoch.p);
    k_pp_wait<<<1, 1, 0, s>>>(ep + 2, ep, static_cast<int*>(x->errflag.p), 20ULL * 1000000000ULL);
    RW_CUDA(cudaGetLastError());
  }
  const GemmDesc* t = static_cast<const GemmDesc*>(x->gemm_wg.p);
  const int M = 4 * x->Hp, N = std::max(x->Hp, x->Ip);
  if constexpr (P::kTF32) {  // kind::tf32 reads these operands K-major only: transposed copies
    const long long colsT = (long long)x->Bp * x->T;
    for (int l = 0; l < x->L; ++l) {
      transpose_planes(x, x->dgop[l], 4 * x->Hp, colsT, x->dgT[l], s);
      if (x->kind == kCellGru) transpose_planes(x, x->dgrop[l], 4 * x->Hp, colsT, x->dgrT[l], s);
      transpose_planes(x, x->hop[l], x->Hp, colsT + x->Bp, x->hT[l], s);
    }
    transpose_planes(x, x->x_op, x->Ip, colsT, x->xT, s);
    RW_CUDA(cudaGetLastError());
  }
  if (x->dp_overlap && x->comm) {
    // data parallel, overlapped: the GEMM pair (dW_l, dR_l: descriptors 2l, 2l + 1) of one layer
    // at a time, top layer first; its bucket is all-reduced on comm_s while the next runs
    for (int l = x->L - 1; l >= 0; --l) {
      if constexpr (P::kTF32)
        launch_gemm<P, false, false>(t + 2 * l, 2, M, N, x->bn_wg, x->st_wg, s);
      else
        launch_gemm<P, true, true>(t + 2 * l, 2, M, N, x->bn_wg, x->st_wg, s);
      RW_CUDA(cudaEventRecord(x->ev_layer[l], s));
      RW_CUDA(cudaStreamWaitEvent(x->comm_s, x->ev_layer[l], 0));
      allreduce_layer(x, l, x->comm_s);
    }
    return;
  }
  if constexpr (P::kTF32)
    launch_gemm<P, false, false>(t, x->n_wg, M, N, x->bn_wg, x->st_wg, s);
  else
    launch_gemm<P, true, true>(t, x->n_wg, M, N, x->bn_wg, x->st_wg, s);
}

void run_db(rw_ctx* x, cudaStream_t s) {
  const int slices = ceil_div(x->Bp, kXChunk) * x->ks_b * 2;
  for (int l0 = 0; l0 < x->L; l0 += kDbGroup, ++g_launches) {
    DbGroup grp{};
    const int n = std::min(kDbGroup, x->L - l0);
    for (int i = 0; i < n; ++i) {
      grp.dbp[i] = x->dbp[l0 + i].f();
      grp.db[i] = x->db[l0 + i].f();
    }
    k_db_reduce_layers<<<dim3(ceil_div(x->G * x->H, 256), n), 256, 0, s>>>(grp, slices, x->H, x->Hp, x->G);
  }
  RW_CUDA(cudaGetLastError());
}

template <class P>
void enqueue_pass_body(rw_ctx* x, int pass, cudaStream_t s) {
  const bool fwd = pass == 0 || pass == 2 || pass == 3;
  if (fwd) {
    PhaseTimer pt(x, 0, s);
    forward_prologue(x, s, nullptr, nullptr, false);
  }
  if (fwd) {
    PhaseTimer pt(x, 1, s);
    run_forward_rec<P>(x, s, pass >= 2);
  }
  if (pass == 0 || pass == 3) return;
  if (pass != 5) {
    PhaseTimer pt(x, 2, s);
    run_backward_rec<P>(x, s);
  }
  if (pass == 4) return;
  const bool overlap = x->dp_overlap && x->comm;
  if (overlap) {  // db first: each layer's bucket (dW, dR, db) is complete after its GEMMs
    PhaseTimer pt(x, 5, s);
    run_db(x, s);
  }
  // dx0 and the weight gradients are independent: dx0 on its own stream fills the weight
  // GEMMs' last wave (RW_SERIAL_TAIL=1, and profiling mode, keep them in sequence)
  static const bool serial_tail = getenv("RW_SERIAL_TAIL") && atoi(getenv("RW_SERIAL_TAIL")) != 0;
  bool db_done = overlap;
  if (!x->profiling && !serial_tail) {
    RW_CUDA(cudaEventRecord(x->ev_tail_fork, s));
    RW_CUDA(cudaStreamWaitEvent(x->tail_s, x->ev_tail_fork, 0));
    run_dx0<P>(x, x->tail_s);
    if (!db_done) run_db(x, x->tail_s);  // the bias-gradient reduction too
    db_done = true;
    run_weight_grads<P>(x, s);
    RW_CUDA(cudaEventRecord(x->ev_tail_join, x->tail_s));
    RW_CUDA(cudaStreamWaitEvent(s, x->ev_tail_join, 0));
  } else {
    {
      PhaseTimer pt(x, 3, s);
      run_weight_grads<P>(x, s);
    }
    {
      PhaseTimer pt(x, 4, s);
      run_dx0<P>(x, s);
    }
  }
  if (!overlap) {
    if (!db_done) {
      PhaseTimer pt(x, 5, s);
      run_db(x, s);
    }
  } else {  // join: the pass completes when the last bucket is summed
    RW_CUDA(cudaEventRecord(x->ev_comm, x->comm_s));
    RW_CUDA(cudaStreamWaitEvent(s, x->ev_comm, 0));
  }
}

// A pass is a fixed DAG (descriptors live in HBM), so it is captured once per pass kind
// into a CUDA graph and replayed: the stepwise schedule's ~2*L*T launches and the
// per-layer fork/join events then cost one cudaGraphLaunch. Profiling mode runs eagerly so
// per-phase CUDA events can bracket each phase on the stream.
template <class P>
void enqueue_pass(rw_ctx* x, int pass, cudaStream_t s) {
  if (x->dirty) {
    PhaseTimer pt(x, 0, s);
    repack_params(x, s);
  }
  if ((pass == 0 || pass == 2 || pass == 3) && !x->state0_zero) {
    forward_prologue(x, s, nullptr, nullptr, true, false);  // zero h0 / c0 blocks once
    x->state0_zero = true;
  }
  if (x->profiling || !x->use_graphs) {
    enqueue_pass_body<P>(x, pass, s);
    return;
  }
  if (!x->graphs[pass]) {
    cudaStream_t cs = x->main;
    RW_CUDA(cudaStreamSynchronize(cs));
    const long long before = g_launches;
    RW_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_pass_body<P>(x, pass, cs);
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(cs, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g = nullptr;
    RW_CUDA(cudaStreamEndCapture(cs, &g));
    RW_CUDA(cudaGraphInstantiate(&x->graphs[pass], g, 0));
    cudaGraphDestroy(g);
    x->graph_launches[pass] = g_launches - before;
    g_launches = before;
  }
  g_launches += x->graph_launches[pass];
  RW_CUDA(cudaGraphLaunch(x->graphs[pass], s));
}

void check_error_flag(rw_ctx* x) {
  int e[5] = {0, 0, 0, 0, 0};
  RW_CUDA(cudaMemcpy(e, x->errflag.p, sizeof e, cudaMemcpyDeviceToHost));
  if (x->prec == kF16x2) {
    // fp16x2 operand range: the scaled planes must stay below fp16's 65504 (common.cuh)
    const char* what[3] = {"a gate gradient dG", "an input x element", "an initial state h0 element"};
    const int sc[3] = {kGScaleLog2, kXScaleLog2, kHScaleLog2};
    for (int i = 0; i < 3; ++i) {
      float v;
      std::memcpy(&v, &e[2 + i], 4);
      if (!(v * pow2f(sc[i]) < 65504.0f)) {
        cudaMemset(static_cast<int*>(x->errflag.p) + 2 + i, 0, 4);
        char b[256];
        snprintf(b, sizeof b,
                 "fp32-parity mode: %s of magnitude %g exceeds the fp16x2 operand range (< %g); results of "
                 "this pass are invalid",
                 what[i], v, 65504.0 / pow2f(sc[i]));
        throw RwError{RW_ESTATE, b};
      }
    }
  }
  if (e[0]) {
    cudaMemset(x->errflag.p, 0, sizeof e);
    char b[256];
    snprintf(b, sizeof b,
             "persistent recurrent kernel timed out waiting for a wavefront flag "
             "(%s layer %d step %d, %s flag, last seen count %d)",
             (e[0] >> 28 & 3) ? "backward" : "forward", (e[0] >> 20) & 0xff,
             ((e[0] >> 4) & 0xffff) - 2,
             (e[0] & 15) == 1 ? "neighbour-layer" : (e[0] & 15) == 3 ? "off-partial publication"
                              : (e[0] & 15) == 4 ? "ring-slot consumed" : "own-layer", e[1]);
    if (e[0] == kWaitTimeoutCode)
      snprintf(b, sizeof b, "a kernel's pipeline barrier (TMA / MMA / exchange mbarrier) did not complete within %.0f s; "
               "the launch was abandoned and its results are invalid", kWaitNs * 1e-9);
    throw RwError{RW_ESTATE, b};
  }
}

void sync_all(rw_ctx* x) {
  if (x->progress_host) {
    const auto t0 = std::chrono::steady_clock::now();
    while (cudaStreamQuery(x->main) == cudaErrorNotReady) {
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > x->hang_s) {
        fprintf(stderr, "rnnwave_sm100: stream not done after %.1f s; progress words (cta: prod mma epi):\n", el);
        for (int c = 0; c < 4096; ++c) {
          const unsigned* w = x->progress_host + 4 * c;
          if (w[0] | w[1] | w[2])
            fprintf(stderr, "  cta %4d: it%3d/m%u  it%3d/m%u  it%3d/m%u\n", c, int(w[0] >> 12) - 2, w[0] & 0xfff,
                    int(w[1] >> 12) - 2, w[1] & 0xfff, int(w[2] >> 12) - 2, w[2] & 0xfff);
        }
        fflush(stderr);
        _exit(3);
      }
      usleep(2000);
    }
  }
  RW_CUDA(cudaStreamSynchronize(x->main));
  RW_CUDA(cudaGetLastError());
  check_error_flag(x);
}

void d2h_unpad(rw_ctx* x, const float* src, int Rp, int Bp, long long col_off, int G, int R, int B,
               int nblk, float* host, int Gs = 0) {
  const long long n = (long long)G * R * B * nblk;
  ++g_launches;
  k_unpad_cols<<<grid_for(n), 256, 0, x->main>>>(src, Rp, Bp, col_off, G, R, B, nblk, x->y_raw.f(), Gs);
  RW_CUDA(cudaGetLastError());
  RW_CUDA(cudaMemcpyAsync(host, x->y_raw.p, n * 4, cudaMemcpyDeviceToHost, x->main));
  RW_CUDA(cudaStreamSynchronize(x->main));
}

std::string g_create_err;  // rw_create / context-free calls (rw_gemm, rw_test_gemm): rw_last_error(NULL)

template <typename F>
int guarded(rw_ctx* x, F&& f) {
  try {
    f();
    return RW_OK;
  } catch (const RwError& e) {
    (x ? x->err : g_create_err) = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    (x ? x->err : g_create_err) = e.what();
    return RW_ECUDA;
  }
}

}  // namespace

rw_ctx::~rw_ctx() {
  if (progress_host) cudaFreeHost(progress_host);
  if (main) cudaStreamSynchronize(main);
  for (auto& g : graphs)
    if (g) cudaGraphExecDestroy(g);
  if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
  for (auto s : ls) cudaStreamDestroy(s);
  for (auto e : lev) cudaEventDestroy(e);
  if (fork_ev) cudaEventDestroy(fork_ev);
  if (tail_s) cudaStreamDestroy(tail_s);
  if (ev_tail_fork) cudaEventDestroy(ev_tail_fork);
  if (ev_tail_join) cudaEventDestroy(ev_tail_join);
  if (main) cudaStreamDestroy(main);
  if (cp_in) cudaStreamDestroy(cp_in);
  if (cp_out) cudaStreamDestroy(cp_out);
  if (comm_s) cudaStreamDestroy(comm_s);
  for (cudaEvent_t e : ev_layer) cudaEventDestroy(e);
  if (ev_comm) cudaEventDestroy(ev_comm);
  for (cudaEvent_t e : {ev_fwd, ev_x, ev_y_staged, ev_y_out, ev_dy, ev_bwd, ev_out})
    if (e) cudaEventDestroy(e);
}

// ====================================================================== C-ABI
extern "C" {

int rw_create(const rw_config* cfg, int device, rw_ctx** out) {
  if (!cfg || !out) {
    g_create_err = "rw_create: null argument";
    return RW_EINVAL;
  }
  *out = nullptr;
  rw_ctx* x = new rw_ctx();
  x->cfg = *cfg;
  x->dev = device;
  int rc = guarded(x, [&] {
    validate(*cfg);
    build(x);
  });
  if (rc != RW_OK) {
    g_create_err = x->err;
    delete x;
    return rc;
  }
  *out = x;
  return RW_OK;
}

void rw_destroy(rw_ctx* ctx) { delete ctx; }

const char* rw_last_error(const rw_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
const char* rw_create_error(void) { return g_create_err.c_str(); }

namespace {
// host buffer <-> device scratch for the synchronous free functions
struct HostIo {
  std::vector<DevBuf> bufs;
  float* in(const float* h, size_t n) {
    if (!h) return nullptr;
    bufs.emplace_back();
    bufs.back().alloc(std::max<size_t>(n, 1) * 4);
    RW_CUDA(cudaMemcpy(bufs.back().p, h, n * 4, cudaMemcpyHostToDevice));
    return bufs.back().f();
  }
  float* out(float* h, size_t n) {
    if (!h) return nullptr;
    bufs.emplace_back();
    bufs.back().alloc(std::max<size_t>(n, 1) * 4);
    return bufs.back().f();
  }
};
void pw_check(int kind, int hidden, int batch) {
  if (kind < kCellRnnTanh || kind > kCellLstm) einval("cells: unknown cell kind " + std::to_string(kind));
  if (hidden <= 0 || batch <= 0) einval("cells: hidden and batch must be positive");
}
}  // namespace

int rw_pointwise_forward(int kind, int fused, int hidden, int batch, const float* zw, const float* zr,
                         const float* bias, const float* h_prev, const float* c_prev, float* h_out, float* c_out,
                         float* gates, float* tanh_c, float* zr_h) {
  (void)fused;
  return guarded(nullptr, [&] {
    pw_check(kind, hidden, batch);
    const int G = kind == kCellLstm ? 4 : kind == kCellGru ? 3 : 1;
    const size_t hb = (size_t)hidden * batch, gb = hb * G;
    if (!zw || !zr || !bias || !h_out) einval("cells: zw, zr, bias and h_out are required");
    if (kind == kCellLstm && (!c_prev || !c_out)) einval("cells: LSTM needs c_prev and c_out");
    if (kind != kCellLstm && c_prev) einval("cells: cell state supplied for a cell kind without one");
    if (kind == kCellGru && !h_prev) einval("cells: GRU needs h_prev");
    const bool rnn = kind == kCellRnnTanh || kind == kCellRnnRelu;
    HostIo io;
    float* dzw = io.in(zw, gb);
    float* dzr = io.in(zr, gb);
    float* db = io.in(bias, (size_t)G * hidden);
    float* dhp = kind == kCellGru ? io.in(h_prev, hb) : nullptr;
    float* dcp = kind == kCellLstm ? io.in(c_prev, hb) : nullptr;
    float* dh = io.out(h_out, hb);
    float* dc = kind == kCellLstm ? io.out(c_out, hb) : nullptr;
    float* dg = rnn ? nullptr : io.out(gates, gb);
    float* dtc = kind == kCellLstm ? io.out(tanh_c, hb) : nullptr;
    float* dzh = kind == kCellGru ? io.out(zr_h, hb) : nullptr;
    ++g_launches;
    k_pointwise_fwd<<<grid_for((long long)hb), 256>>>(kind, hidden, batch, dzw, dzr, db, dhp, dcp, dh, dc, dg, dtc, dzh);
    RW_CUDA(cudaGetLastError());
    RW_CUDA(cudaDeviceSynchronize());
    RW_CUDA(cudaMemcpy(h_out, dh, hb * 4, cudaMemcpyDeviceToHost));
    if (dc) RW_CUDA(cudaMemcpy(c_out, dc, hb * 4, cudaMemcpyDeviceToHost));
    if (dg) RW_CUDA(cudaMemcpy(gates, dg, gb * 4, cudaMemcpyDeviceToHost));
    if (dtc) RW_CUDA(cudaMemcpy(tanh_c, dtc, hb * 4, cudaMemcpyDeviceToHost));
    if (dzh) RW_CUDA(cudaMemcpy(zr_h, dzh, hb * 4, cudaMemcpyDeviceToHost));
  });
}

int rw_pointwise_backward(int kind, int fused, int hidden, int batch, const float* gates, const float* tanh_c,
                          const float* zr_h, const float* h_prev, const float* c_prev, const float* d_above,
                          const float* dh_carry, const float* dc_carry, float* dgw, float* dgr, float* dh_local,
                          float* dc_prev, float* db) {
  (void)fused;
  return guarded(nullptr, [&] {
    pw_check(kind, hidden, batch);
    const int G = kind == kCellLstm ? 4 : kind == kCellGru ? 3 : 1;
    const size_t hb = (size_t)hidden * batch, gb = hb * G;
    if (!gates) einval("cells: backward requires saved state from a training forward");
    if (!d_above || !dh_carry || !dgw || !dh_local) einval("cells: d_above, dh_carry, dgw and dh_local are required");
    if (kind == kCellLstm && (!tanh_c || !c_prev || !dc_carry || !dc_prev))
      einval("cells: LSTM backward needs tanh_c, c_prev, dc_carry and dc_prev");
    if (kind == kCellGru && (!zr_h || !h_prev || !dgr)) einval("cells: GRU backward needs zr_h, h_prev and dgr");
    if (kind == kCellGru && dgr == dgw) einval("cells: GRU needs distinct dgw and dgr blocks");
    HostIo io;
    float* dgs = io.in(gates, kind == kCellLstm || kind == kCellGru ? gb : hb);
    float* dtc = kind == kCellLstm ? io.in(tanh_c, hb) : nullptr;
    float* dzh = kind == kCellGru ? io.in(zr_h, hb) : nullptr;
    float* dhp = kind == kCellGru ? io.in(h_prev, hb) : nullptr;
    float* dcp = kind == kCellLstm ? io.in(c_prev, hb) : nullptr;
    float* dda = io.in(d_above, hb);
    float* dhc = io.in(dh_carry, hb);
    float* dcc = kind == kCellLstm ? io.in(dc_carry, hb) : nullptr;
    float* ddgw = io.out(dgw, gb);
    float* ddgr = kind == kCellGru ? io.out(dgr, gb) : nullptr;
    float* dhl = io.out(dh_local, hb);
    float* ddcp = kind == kCellLstm ? io.out(dc_prev, hb) : nullptr;
    float* ddb = db ? io.in(db, (size_t)G * hidden) : nullptr;
    ++g_launches;
    k_pointwise_bwd<<<grid_for((long long)hb), 256>>>(kind, hidden, batch, dgs, dtc, dzh, dhp, dcp, dda, dhc, dcc, ddgw,
                                                      ddgr, dhl, ddcp);
    if (ddb) {
      ++g_launches;
      k_row_sums_add<<<ceil_div(G * hidden, 256), 256>>>(ddgw, G * hidden, batch, ddb);
    }
    RW_CUDA(cudaGetLastError());
    RW_CUDA(cudaDeviceSynchronize());
    RW_CUDA(cudaMemcpy(dgw, ddgw, gb * 4, cudaMemcpyDeviceToHost));
    if (ddgr) RW_CUDA(cudaMemcpy(dgr, ddgr, gb * 4, cudaMemcpyDeviceToHost));
    RW_CUDA(cudaMemcpy(dh_local, dhl, hb * 4, cudaMemcpyDeviceToHost));
    if (ddcp) RW_CUDA(cudaMemcpy(dc_prev, ddcp, hb * 4, cudaMemcpyDeviceToHost));
    if (ddb) RW_CUDA(cudaMemcpy(db, ddb, (size_t)G * hidden * 4, cudaMemcpyDeviceToHost));
  });
}

int64_t rw_flop_count_cell(int hidden, int input, int batch) {
  return 2LL * 4 * hidden * ((int64_t)input + hidden) * batch;
}

int rw_set_params(rw_ctx* x, int layer, const float* W, const float* R, const float* b) {
  return guarded(x, [&] {
    if (layer < 0 || layer >= x->L) einval("rw_set_params: layer " + std::to_string(layer) + " out of range");
    if (!W || !R) einval("rw_set_params: W and R are required");
    RW_CUDA(cudaSetDevice(x->dev));
    const int Il = layer == 0 ? x->I : x->H;
    RW_CUDA(cudaMemcpy(x->W[layer].p, W, (unsigned long long)x->G * x->H * Il * 4, cudaMemcpyHostToDevice));
    RW_CUDA(cudaMemcpy(x->R[layer].p, R, (unsigned long long)x->G * x->H * x->H * 4, cudaMemcpyHostToDevice));
    if (b)
      RW_CUDA(cudaMemcpy(x->bias_raw[layer].p, b, (unsigned long long)x->G * x->H * 4, cudaMemcpyHostToDevice));
    else
      RW_CUDA(cudaMemset(x->bias_raw[layer].p, 0, (unsigned long long)x->G * x->H * 4));
    x->params_set[layer] = 1;
    x->dirty = true;
  });
}

static void require_params(rw_ctx* x) {
  for (int l = 0; l < x->L; ++l)
    if (!x->params_set[l])
      einval("engine: expected " + std::to_string(x->L) + " layer parameter sets, layer " +
             std::to_string(l) + " was never set");
}

int rw_forward(rw_ctx* x, const float* xin, int training, const float* const* h0,
               const float* const* c0, float* y, uint64_t* tape_id) {
  return guarded(x, [&] {
    if (!xin) einval("forward: x is null, expected " + std::to_string(x->I) + "x" + std::to_string(x->B * x->T));
    if (c0 && x->kind != kCellLstm) einval("forward: c0 supplied for a cell kind without cell state");
    require_params(x);
    RW_CUDA(cudaSetDevice(x->dev));
    const size_t hb = (size_t)x->H * x->B;
    RW_CUDA(cudaMemcpyAsync(x->x_raw.p, xin, (size_t)x->I * x->B * x->T * 4, cudaMemcpyHostToDevice, x->main));
    // stage h0 / c0 contiguously in y_raw (large enough: >= 2 * L * H * B is not guaranteed,
    // so use dedicated temporaries)
    DevBuf th0, tc0;
    if (h0) {
      th0.alloc(hb * x->L * 4);
      for (int l = 0; l < x->L; ++l)
        RW_CUDA(cudaMemcpy(th0.f() + l * hb, h0[l], hb * 4, cudaMemcpyHostToDevice));
    }
    if (c0) {
      tc0.alloc(hb * x->L * 4);
      for (int l = 0; l < x->L; ++l)
        RW_CUDA(cudaMemcpy(tc0.f() + l * hb, c0[l], hb * 4, cudaMemcpyHostToDevice));
    }
    repack_params(x, x->main);
    forward_prologue(x, x->main, h0 ? th0.f() : nullptr, c0 ? tc0.f() : nullptr);
    x->state0_zero = !h0 && !c0;
    by_prec(x->prec, [&](auto tag) { run_forward_rec<decltype(tag)>(x, x->main, training != 0); });
    sync_all(x);
    x->inputs_uploaded = false;
    x->tape_gen += 1;
    x->tape_training = training != 0;
    x->bwd_done = false;
    if (tape_id) *tape_id = x->tape_gen;
    if (y) d2h_unpad(x, x->h[x->L - 1].f(), x->Hp, x->Bp, x->Bp, 1, x->H, x->B, x->T, y);
  });
}

static void check_tape(rw_ctx* x, uint64_t id) {
  if (id != x->tape_gen || x->tape_gen == 0)
    einval("engine: stale tape, the device holds tape " + std::to_string(x->tape_gen) +
           " but tape " + std::to_string(id) + " was passed");
  if (!x->tape_training) einval("engine: tape was recorded without training mode");
}

int rw_backward_data(rw_ctx* x, uint64_t tape_id, const float* dy, float* dx0, float* const* dh0,
                     float* const* dc0) {
  return guarded(x, [&] {
    check_tape(x, tape_id);
    if (!dy) einval("backward_data: dy is null, expected " + std::to_string(x->H) + "x" + std::to_string(x->B * x->T));
    RW_CUDA(cudaSetDevice(x->dev));
    RW_CUDA(cudaMemcpyAsync(x->dy_raw.p, dy, (size_t)x->H * x->B * x->T * 4, cudaMemcpyHostToDevice, x->main));
    repack_params(x, x->main);
    by_prec(x->prec, [&](auto tag) {
      run_backward_rec<decltype(tag)>(x, x->main);
      run_dx0<decltype(tag)>(x, x->main);
    });
    sync_all(x);
    x->bwd_done = true;
    if (dx0) RW_CUDA(cudaMemcpy(dx0, x->dx0.p, (size_t)x->I * x->B * x->T * 4, cudaMemcpyDeviceToHost));
    for (int l = 0; l < x->L; ++l) {
      if (dh0 && dh0[l]) d2h_unpad(x, x->dh0[l].f(), x->Hp, x->Bp, 0, 1, x->H, x->B, 1, dh0[l]);
      if (dc0 && dc0[l] && x->kind == kCellLstm) d2h_unpad(x, x->dc0[l].f(), x->Hp, x->Bp, 0, 1, x->H, x->B, 1, dc0[l]);
    }
  });
}

int rw_weight_update(rw_ctx* x, uint64_t tape_id, float* const* dW, float* const* dR, float* const* db) {
  return guarded(x, [&] {
    check_tape(x, tape_id);
    if (!x->bwd_done) einval("weight_update: backward state layer count mismatch (run backward_data on this tape first)");
    RW_CUDA(cudaSetDevice(x->dev));
    by_prec(x->prec, [&](auto tag) { run_weight_grads<decltype(tag)>(x, x->main); });
    run_db(x, x->main);
    sync_all(x);
    for (int l = 0; l < x->L; ++l) {
      const int Il = l == 0 ? x->I : x->H;
      if (dW && dW[l]) RW_CUDA(cudaMemcpy(dW[l], x->dW[l].p, (unsigned long long)x->G * x->H * Il * 4, cudaMemcpyDeviceToHost));
      if (dR && dR[l]) RW_CUDA(cudaMemcpy(dR[l], x->dR[l].p, (unsigned long long)x->G * x->H * x->H * 4, cudaMemcpyDeviceToHost));
      if (db && db[l]) RW_CUDA(cudaMemcpy(db[l], x->db[l].p, (unsigned long long)x->G * x->H * 4, cudaMemcpyDeviceToHost));
    }
  });
}

int rw_get_tape(rw_ctx* x, int which, int layer, float* host) {
  return guarded(x, [&] {
    if (!host) einval("rw_get_tape: null destination");
    if (which != RW_TAPE_X0 && which != RW_TAPE_Y && (layer < 0 || layer >= x->L))
      einval("rw_get_tape: layer out of range");
    if (x->tape_gen == 0) einval("rw_get_tape: no forward pass has run");
    RW_CUDA(cudaSetDevice(x->dev));
    const int H = x->H, B = x->B, T = x->T, Hp = x->Hp, Bp = x->Bp;
    switch (which) {
      case RW_TAPE_X0:
        RW_CUDA(cudaMemcpy(host, x->x_raw.p, (size_t)x->I * B * T * 4, cudaMemcpyDeviceToHost));
        break;
      case RW_TAPE_Y:
        d2h_unpad(x, x->h[x->L - 1].f(), Hp, Bp, Bp, 1, H, B, T, host);
        break;
      case RW_TAPE_H:
        d2h_unpad(x, x->h[layer].f(), Hp, Bp, 0, 1, H, B, T + 1, host);
        break;
      case RW_TAPE_C:
        if (x->kind != kCellLstm) einval("rw_get_tape: c_seq exists for LSTM cells only");
        d2h_unpad(x, x->c[layer].f(), Hp, Bp, 0, 1, H, B, T + 1, host);
        break;
      case RW_TAPE_ZRH:
        if (x->kind != kCellGru) einval("rw_get_tape: zrh_seq exists for GRU cells only");
        if (!x->tape_training) einval("engine: tape was recorded without training mode");
        d2h_unpad(x, x->zrh[layer].f(), Hp, Bp, 0, 1, H, B, T, host);
        break;
      case RW_TAPE_DGR:
        if (x->kind != kCellGru) einval("rw_get_tape: dgr_seq exists for GRU cells only");
        if (!x->bwd_done) einval("rw_get_tape: no backward pass on the current tape");
        d2h_unpad(x, x->dgr[layer].f(), Hp, Bp, 0, x->G, H, B, T, host, 4);
        break;
      case RW_TAPE_GATES:
        if (!x->tape_training) einval("engine: tape was recorded without training mode");
        d2h_unpad(x, x->gates[layer].f(), Hp, Bp, 0, x->G, H, B, T, host, 4);  // 4-slot tape
        break;
      case RW_TAPE_TANH_C:
        if (x->kind != kCellLstm) einval("rw_get_tape: tanh_c_seq exists for LSTM cells only");
        if (!x->tape_training) einval("engine: tape was recorded without training mode");
        d2h_unpad(x, x->tanhc[layer].f(), Hp, Bp, 0, 1, H, B, T, host);
        break;
      case RW_TAPE_DGW:
        if (!x->bwd_done) einval("rw_get_tape: no backward pass on the current tape");
        d2h_unpad(x, x->dg[layer].f(), Hp, Bp, 0, x->G, H, B, T, host, 4);
        break;
      default:
        einval("rw_get_tape: unknown tape id");
    }
  });
}

int rw_upload_inputs(rw_ctx* x, const float* xin, const float* dy) {
  return guarded(x, [&] {
    RW_CUDA(cudaSetDevice(x->dev));
    if (xin) RW_CUDA(cudaMemcpy(x->x_raw.p, xin, (size_t)x->I * x->B * x->T * 4, cudaMemcpyHostToDevice));
    if (dy) RW_CUDA(cudaMemcpy(x->dy_raw.p, dy, (size_t)x->H * x->B * x->T * 4, cudaMemcpyHostToDevice));
    x->inputs_uploaded = true;
  });
}

// Pipelined training step with host buffers (the public end-to-end call; pinned host memory
// gives full DMA rate). Inputs of step i+1 upload while step i computes, outputs of step i
// download while step i+1 computes:
//   cp_in : [wait fwd(i-1)] x -> x_raw                                   -> ev_x
//   main  : [wait ev_x] forward (pass 3) -> ev_fwd; [wait y_out(i-1)] unpad y -> ev_y_staged
//   cp_out: [wait ev_y_staged] y_raw -> y                                -> ev_y_out
//   cp_in : [wait bwd(i-1)] dy -> dy_raw                                 -> ev_dy
//   main  : [wait ev_dy, out(i-1)] backward + weight update (pass 1)     -> ev_bwd
//   cp_out: [wait ev_bwd] dx0, dW, dR, db -> host                        -> ev_out
// Host buffers are written asynchronously: they are complete after rw_train_wait.
static void allreduce_grads(rw_ctx* x, cudaStream_t s);
static void train_streams(rw_ctx* x) {
  if (x->cp_in) return;
  RW_CUDA(cudaStreamCreateWithFlags(&x->cp_in, cudaStreamNonBlocking));
  RW_CUDA(cudaStreamCreateWithFlags(&x->cp_out, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&x->ev_fwd, &x->ev_x, &x->ev_y_staged, &x->ev_y_out, &x->ev_dy, &x->ev_bwd, &x->ev_out})
    RW_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

extern "C" int rw_train_step(rw_ctx* x, const float* xin, const float* dy, float* y, float* dx0, float* const* dW,
                             float* const* dR, float* const* db) {
  return guarded(x, [&] {
    if (!xin || !dy) einval("rw_train_step: x and dy are required (expected host buffers)");
    require_params(x);
    RW_CUDA(cudaSetDevice(x->dev));
    train_streams(x);
    const size_t xb = (size_t)x->I * x->B * x->T * 4, yb = (size_t)x->H * x->B * x->T * 4;
    RW_CUDA(cudaStreamWaitEvent(x->cp_in, x->ev_fwd, 0));
    RW_CUDA(cudaMemcpyAsync(x->x_raw.p, xin, xb, cudaMemcpyHostToDevice, x->cp_in));
    RW_CUDA(cudaEventRecord(x->ev_x, x->cp_in));
    RW_CUDA(cudaStreamWaitEvent(x->main, x->ev_x, 0));
    by_prec(x->prec, [&](auto tag) { enqueue_pass<decltype(tag)>(x, 3, x->main); });
    RW_CUDA(cudaEventRecord(x->ev_fwd, x->main));
    if (y) {
      RW_CUDA(cudaStreamWaitEvent(x->main, x->ev_y_out, 0));
      const long long n = (long long)x->H * x->B * x->T;
      ++g_launches;
      k_unpad_cols<<<grid_for(n), 256, 0, x->main>>>(x->h[x->L - 1].f(), x->Hp, x->Bp, x->Bp, 1, x->H, x->B, x->T,
                                                     x->y_raw.f());
      RW_CUDA(cudaGetLastError());
      RW_CUDA(cudaEventRecord(x->ev_y_staged, x->main));
      RW_CUDA(cudaStreamWaitEvent(x->cp_out, x->ev_y_staged, 0));
      RW_CUDA(cudaMemcpyAsync(y, x->y_raw.p, yb, cudaMemcpyDeviceToHost, x->cp_out));
      RW_CUDA(cudaEventRecord(x->ev_y_out, x->cp_out));
    }
    RW_CUDA(cudaStreamWaitEvent(x->cp_in, x->ev_bwd, 0));
    RW_CUDA(cudaMemcpyAsync(x->dy_raw.p, dy, yb, cudaMemcpyHostToDevice, x->cp_in));
    RW_CUDA(cudaEventRecord(x->ev_dy, x->cp_in));
    RW_CUDA(cudaStreamWaitEvent(x->main, x->ev_dy, 0));
    x->tape_gen += 1;
    x->tape_training = true;
    // the backward recurrence writes no read-back buffer: only the gradient phase waits for the
    // previous step's read-back (ev_out), which thus overlaps this step's forward + recurrence
    by_prec(x->prec, [&](auto tag) { enqueue_pass<decltype(tag)>(x, 4, x->main); });
    RW_CUDA(cudaStreamWaitEvent(x->main, x->ev_out, 0));
    by_prec(x->prec, [&](auto tag) { enqueue_pass<decltype(tag)>(x, 5, x->main); });
    x->bwd_done = true;
    if (x->comm) allreduce_grads(x, x->main);  // data parallel: sum dW/dR/db before read-back
    RW_CUDA(cudaEventRecord(x->ev_bwd, x->main));
    RW_CUDA(cudaStreamWaitEvent(x->cp_out, x->ev_bwd, 0));
    if (dx0) RW_CUDA(cudaMemcpyAsync(dx0, x->dx0.p, xb, cudaMemcpyDeviceToHost, x->cp_out));
    for (int l = 0; l < x->L; ++l) {
      const int Il = l == 0 ? x->I : x->H;
      if (dW && dW[l]) RW_CUDA(cudaMemcpyAsync(dW[l], x->dW[l].p, (unsigned long long)x->G * x->H * Il * 4, cudaMemcpyDeviceToHost, x->cp_out));
      if (dR && dR[l]) RW_CUDA(cudaMemcpyAsync(dR[l], x->dR[l].p, (unsigned long long)x->G * x->H * x->H * 4, cudaMemcpyDeviceToHost, x->cp_out));
      if (db && db[l]) RW_CUDA(cudaMemcpyAsync(db[l], x->db[l].p, (unsigned long long)x->G * x->H * 4, cudaMemcpyDeviceToHost, x->cp_out));
    }
    RW_CUDA(cudaEventRecord(x->ev_out, x->cp_out));
  });
}

extern "C" int rw_train_wait(rw_ctx* x) {
  return guarded(x, [&] {
    RW_CUDA(cudaSetDevice(x->dev));
    RW_CUDA(cudaStreamSynchronize(x->main));
    if (x->cp_in) RW_CUDA(cudaStreamSynchronize(x->cp_in));
    if (x->cp_out) RW_CUDA(cudaStreamSynchronize(x->cp_out));
    check_error_flag(x);
  });
}

int rw_run_pass(rw_ctx* x, int pass, void* stream) {
  return guarded(x, [&] {
    if (pass < 0 || pass > 3)
      einval("rw_run_pass: pass must be 0 (fwd), 1 (bwd), 2 (both) or 3 (fwd recording a training tape)");
    require_params(x);
    RW_CUDA(cudaSetDevice(x->dev));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : x->main;
    if (pass == 1 && (x->tape_gen == 0 || !x->tape_training))
      einval("rw_run_pass: backward needs a training tape (run pass 2 once first)");
    by_prec(x->prec, [&](auto tag) { enqueue_pass<decltype(tag)>(x, pass, s); });
    if (pass != 1) {
      x->tape_gen += 1;
      x->tape_training = pass >= 2;
    }
    x->bwd_done = pass == 1 || pass == 2;
  });
}

int rw_params_updated(rw_ctx* x) {
  return guarded(x, [&] {
    require_params(x);
    x->dirty = true;
  });
}

int rw_read_outputs(rw_ctx* x, float* y, float* dx0, float* const* dW, float* const* dR,
                    float* const* db) {
  return guarded(x, [&] {
    RW_CUDA(cudaSetDevice(x->dev));
    RW_CUDA(cudaDeviceSynchronize());  // the pass may have been enqueued on a caller's stream
    check_error_flag(x);
    // all copies queued on the context stream, one synchronisation (full DMA rate into pinned
    // host buffers; pageable ones are staged by the driver)
    cudaStream_t s = x->main;
    if (y) {
      const long long n = (long long)x->H * x->B * x->T;
      ++g_launches;
      k_unpad_cols<<<grid_for(n), 256, 0, s>>>(x->h[x->L - 1].f(), x->Hp, x->Bp, x->Bp, 1, x->H, x->B, x->T,
                                               x->y_raw.f());
      RW_CUDA(cudaGetLastError());
      RW_CUDA(cudaMemcpyAsync(y, x->y_raw.p, n * 4, cudaMemcpyDeviceToHost, s));
    }
    if (dx0) RW_CUDA(cudaMemcpyAsync(dx0, x->dx0.p, (size_t)x->I * x->B * x->T * 4, cudaMemcpyDeviceToHost, s));
    for (int l = 0; l < x->L; ++l) {
      const int Il = l == 0 ? x->I : x->H;
      if (dW && dW[l]) RW_CUDA(cudaMemcpyAsync(dW[l], x->dW[l].p, (unsigned long long)x->G * x->H * Il * 4, cudaMemcpyDeviceToHost, s));
      if (dR && dR[l]) RW_CUDA(cudaMemcpyAsync(dR[l], x->dR[l].p, (unsigned long long)x->G * x->H * x->H * 4, cudaMemcpyDeviceToHost, s));
      if (db && db[l]) RW_CUDA(cudaMemcpyAsync(db[l], x->db[l].p, (unsigned long long)x->G * x->H * 4, cudaMemcpyDeviceToHost, s));
    }
    RW_CUDA(cudaStreamSynchronize(s));
  });
}

int rw_launch_count(rw_ctx* x, long long* count, int reset) {
  return guarded(x, [&] {
    if (count) *count = g_launches;
    if (reset) g_launches = 0;
  });
}

// ---------------------------------------------------------------- layer pipeline
static void invalidate_graphs(rw_ctx* x) {
  for (auto& g : x->graphs)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
}

static void export_region(rw_pp_ring* o, int i, const void* base, const void* region) {
  cudaIpcMemHandle_t h;
  RW_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(base)));
  static_assert(sizeof(h) <= 64, "ipc handle");
  memcpy(o->handle[i], &h, sizeof h);
  o->offset[i] = (uint64_t)(static_cast<const uint8_t*>(region) - static_cast<const uint8_t*>(base));
  o->ptr[i] = (uint64_t)(uintptr_t)region;
}

static void* open_region(rw_ctx* x, const rw_pp_ring* peer, int i) {
  if (peer->pid == (int64_t)getpid()) {
    if (peer->device != x->dev) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) RW_CUDA(e);
      cudaGetLastError();
    }
    return reinterpret_cast<void*>((uintptr_t)peer->ptr[i]);
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, peer->handle[i], sizeof h);
  void* base = nullptr;
  RW_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  x->pp_opened.push_back(base);
  return static_cast<uint8_t*>(base) + peer->offset[i];
}

// Schedule family of a pipeline stage: 0 cluster (boundary groups, swizzled images), 1 the
// persistent / stepwise kernels (plain operand planes written per step by the neighbour).
static int pp_family(rw_ctx* x, const char* fn) {
  auto plain = [](int s) { return s == RW_SCHED_PERSISTENT || s == RW_SCHED_STEPWISE; };
  if (x->fwd_sched == RW_SCHED_CLUSTER && x->bwd_sched == RW_SCHED_CLUSTER) return 0;
  if (plain(x->fwd_sched) && plain(x->bwd_sched)) {
    if (x->fwd_batch)
      einval(std::string(fn) + ": the layer pipeline does not batch the input projections (set RW_FWD_BATCH=0)");
    return 1;
  }
  einval(std::string(fn) + ": the layer pipeline needs the cluster schedule in both directions, or the "
         "persistent / stepwise schedules in both");
  return -1;
}

// fp16x2: a stage's layer input is an h (2^kHScaleLog2 planes), not x: its first layer's dW
// GEMM alpha follows (the W.x unscale: ClOff::unscale / RecParams::us_in0)
static void pp_input_is_h(rw_ctx* x) {
  if (x->prec != kF16x2) return;
  GemmDesc d0;
  RW_CUDA(cudaMemcpy(&d0, x->gemm_wg.p, sizeof d0, cudaMemcpyDeviceToHost));
  d0.alpha = pow2f(-(kGScaleLog2 + kHScaleLog2));
  RW_CUDA(cudaMemcpy(x->gemm_wg.p, &d0, sizeof d0, cudaMemcpyHostToDevice));
}

static void pp_upload_maps(rw_ctx* x) {
  if (!x->pp_maps_dev.p) x->pp_maps_dev.alloc(x->pp_maps.size() * sizeof(CUtensorMap));
  RW_CUDA(cudaMemcpy(x->pp_maps_dev.p, x->pp_maps.data(), x->pp_maps.size() * sizeof(CUtensorMap),
                     cudaMemcpyHostToDevice));
}

// Persistent / stepwise stage with a next stage: once both the dG input planes (rw_pp_export
// dir 1) and the next stage's W_0 (rw_pp_link dir 0) are known, the top layer's backward
// becomes an inner layer's: A = [W_next^T | R^T] (packed by k_repack), the up operand = dgin,
// its per-step counter released by the next stage -- the same K order and accumulation as one
// context holding both stages, so the results match it bit for bit.
static void pp_plain_up(rw_ctx* x) {
  if (x->pp_up || !x->pp_wnext || !x->dgin.p(0)) return;
  const int L = x->L, Hp = x->Hp, aK = x->atomK;
  const long long G4p = 4LL * Hp, colsT = (long long)x->Bp * x->T;
  if (L == 1)  // the backward plan (k-blocks per accumulator, resident slots) covered R^T only
    einval("rw_pp_link: on the persistent / stepwise schedules a stage below the last needs >= 2 layers");
  x->wb[L - 1].alloc(x->prec, (size_t)Hp * 2 * G4p);
  for (int p = 0; p < x->planes; ++p) {
    x->pp_maps[2 + p] = make_map(x->wb[L - 1].p(p), x->prec, 2 * G4p, Hp, aK, kTileM);
    x->pp_maps[4 + p] = make_map(x->dgin.p(p), x->prec, G4p, colsT, aK, x->Bp);
  }
  if (x->pair_b) x->pp_maps[6] = make_map(x->dgin.p(0), x->prec, G4p, colsT, aK, x->Bp / 2);
  pp_upload_maps(x);
  const CUtensorMap* MD = static_cast<const CUtensorMap*>(x->pp_maps_dev.p);
  BwdLayer b;
  BwdLayer* dev = static_cast<BwdLayer*>(x->bwd_layers.p) + (L - 1);
  RW_CUDA(cudaMemcpy(&b, dev, sizeof b, cudaMemcpyDeviceToHost));
  for (int p = 0; p < 2; ++p) {
    b.a[p] = p < x->planes ? MD + 2 + p : nullptr;
    b.bup[p] = p < x->planes ? MD + 4 + p : nullptr;
  }
  b.bup2 = x->pair_b ? MD + 6 : nullptr;
  b.has_up = 1;
  b.dy = nullptr;  // an inner layer of the whole stack: its output gradient is d_above only
  RW_CUDA(cudaMemcpy(dev, &b, sizeof b, cudaMemcpyHostToDevice));
  x->pp_up = true;
  x->repack_njobs = 0;  // rebuild the repack table: the top layer's image now holds W_next^T too
  x->dirty = true;
}

// CTAs of one layer that release a per-step counter (persistent / stepwise kernels)
static uint32_t pp_senders(rw_ctx* x, bool fwd) {
  const RecParams rp = rec_params(x, fwd);
  return (uint32_t)(!fwd && x->pair_b ? rp.tiles : rp.tiles * rp.ksplit);
}

extern "C" int rw_pp_export(rw_ctx* x, int dir, rw_pp_ring* out) {
  return guarded(x, [&] {
    const int fam = pp_family(x, "rw_pp_export");
    if (dir != 0 && dir != 1) einval("rw_pp_export: dir must be 0 (forward) or 1 (backward)");
    RW_CUDA(cudaSetDevice(x->dev));
    memset(out, 0, sizeof *out);
    out->pid = (int64_t)getpid();
    out->device = x->dev;
    out->mode = fam;
    if (fam == 1) {
      x->pp_plain = true;
      if (!x->cl_epoch.p) x->cl_epoch.alloc(16);
      const size_t nf = (size_t)(x->T + 1) * 4;
      if (dir == 0) {
        // forward: the previous stage's last layer stores h_t into block t of these planes (the
        // layer-0 input operand, read by the step kernels and by the dW_0 GEMM) and releases
        // xin_flags[t]; it also reads our W_0 (region 3) for its top layer's backward
        x->xin_flags.alloc(nf);
        export_region(out, 0, x->x_op.p(0), x->x_op.p(0));
        export_region(out, 1, x->xin_flags.p, x->xin_flags.p);
        export_region(out, 2, x->x_op.p(1) ? x->x_op.p(1) : x->xin_flags.p, x->x_op.p(1) ? x->x_op.p(1) : x->xin_flags.p);
        export_region(out, 3, x->W[0].p, x->W[0].p);
        export_region(out, 4, x->cl_epoch.p, static_cast<uint32_t*>(x->cl_epoch.p) + 2);
        pp_input_is_h(x);
        x->pp_prev = true;
        x->pp_exported_f = true;
      } else {
        // backward: the next stage's first layer stores its W-side dG_t here (dgop's layout)
        const long long colsT = (long long)x->Bp * x->T;
        x->dgin.alloc(x->prec, (size_t)4 * x->Hp * colsT);
        x->dgin_flags.alloc(nf);
        export_region(out, 0, x->dgin.p(0), x->dgin.p(0));
        export_region(out, 1, x->dgin_flags.p, x->dgin_flags.p);
        export_region(out, 2, x->dgin.p(1) ? x->dgin.p(1) : x->dgin_flags.p, x->dgin.p(1) ? x->dgin.p(1) : x->dgin_flags.p);
        x->pp_exported_b = true;
        pp_plain_up(x);
      }
      invalidate_graphs(x);
      return;
    }
    if (dir == 0) {
      // forward: the previous stage writes its last layer's h_t (bf16 operand image, H x B x 2 B
      // per step) straight into this stage's layer-input image over NVLink and releases a
      // per-step counter; this stage's first-layer W.x group then runs as on one GPU
      x->xin_flags.alloc((size_t)x->T * 4);
      export_region(out, 0, x->xsw.p, x->xsw.p);
      export_region(out, 1, x->xin_flags.p, x->xin_flags.p);
      // fp16x2: the plain layer-input lo plane (bf16: unused, the counters again)
      export_region(out, 2, x->x_op.p(1) ? x->x_op.p(1) : x->xin_flags.p, x->x_op.p(1) ? x->x_op.p(1) : x->xin_flags.p);
      export_region(out, 3, x->x_op.p(0), x->x_op.p(0));
      export_region(out, 4, x->cl_epoch.p, static_cast<uint32_t*>(x->cl_epoch.p) + 2);
      ClOff& o = x->off_f_h[0];
      o.op_flags = static_cast<const uint32_t*>(x->xin_flags.p);
      o.sys = 1;  // written by another process: system-scope waits
      if (x->prec == kF16x2) o.unscale = pow2f(-(kWScaleLog2 + kHScaleLog2));  // h planes, not x
      pp_input_is_h(x);
      x->pp_prev = true;
      x->pp_exported_f = true;
    } else {
      ClRing& r = x->ring_b_h[x->L - 1];
      // written by the next stage's boundary group with the member count a single context gives
      // this layer's off group (kc of the backward plan, runtime.cu planner), so the K split and
      // the reduction order -- and the results, bit for bit -- match the unsplit stack
      r.ko = x->cl_b.kc;
      r.sys = 1;
      out->ko = r.ko;
      export_region(out, 0, x->cl_offsum.p, r.ring);
      export_region(out, 1, x->cl_done.p, r.done);
      export_region(out, 2, x->cl_consumed.p, r.consumed);
      x->pp_exported_b = true;
    }
    upload_cluster_tables(x);
    invalidate_graphs(x);
  });
}

extern "C" int rw_pp_link(rw_ctx* x, int dir, const rw_pp_ring* peer, const float* W_next) {
  x->state0_zero = false;  // conservatively re-stage the state blocks after relinking
  return guarded(x, [&] {
    if (!peer) einval("rw_pp_link: peer descriptor is null");
    const int fam = pp_family(x, "rw_pp_link");
    if (peer->mode != fam) einval("rw_pp_link: the two stages use different schedule families (cluster vs persistent/stepwise)");
    if (dir != 0 && dir != 1) einval("rw_pp_link: dir must be 0 (forward) or 1 (backward)");
    RW_CUDA(cudaSetDevice(x->dev));
    const int L = x->L, H = x->H, Hp = x->Hp, T = x->T, aK = x->atomK;
    const long long G4p = 4LL * Hp;
    if (fam == 1) {
      x->pp_plain = true;
      if (!x->cl_epoch.p) x->cl_epoch.alloc(16);
      void* p0 = open_region(x, peer, 0);
      uint32_t* flags = static_cast<uint32_t*>(open_region(x, peer, 1));
      void* p1 = x->planes > 1 ? open_region(x, peer, 2) : nullptr;
      // the receiver's per-pass target: our CTAs per step (slot T of its counters)
      const uint32_t cnt = pp_senders(x, dir == 0);
      RW_CUDA(cudaMemcpy(flags + T, &cnt, 4, cudaMemcpyDefault));
      if (dir == 0) {  // forward: our last layer stores h_t into the next stage's input planes
        FwdLayer top;
        FwdLayer* dev = static_cast<FwdLayer*>(x->fwd_layers.p) + (L - 1);
        RW_CUDA(cudaMemcpy(&top, dev, sizeof top, cudaMemcpyDeviceToHost));
        top.xop_peer[0] = p0;
        top.xop_peer[1] = p1;
        top.peer_ld = Hp;  // the next stage's Ip = round_up(H, 64) = Hp
        top.peer_flags = flags;
        RW_CUDA(cudaMemcpy(dev, &top, sizeof top, cudaMemcpyHostToDevice));
        x->pp_next_ready = static_cast<uint32_t*>(open_region(x, peer, 4));
        if (W_next) {  // host copy given (reference layout, G H x H): keep it on the device
          x->wn_raw.alloc((size_t)x->G * H * H * 4);
          RW_CUDA(cudaMemcpy(x->wn_raw.p, W_next, x->wn_raw.bytes, cudaMemcpyHostToDevice));
          x->pp_wnext = x->wn_raw.f();
        } else {  // the next stage's live parameters over the link
          x->pp_wnext = static_cast<const float*>(open_region(x, peer, 3));
        }
        x->pp_next = true;
        pp_plain_up(x);
      } else {  // backward: our first layer stores its W-side dG_t into the previous stage's planes
        BwdLayer b0;
        BwdLayer* dev = static_cast<BwdLayer*>(x->bwd_layers.p);
        RW_CUDA(cudaMemcpy(&b0, dev, sizeof b0, cudaMemcpyDeviceToHost));
        b0.dg_peer[0] = p0;
        b0.dg_peer[1] = p1;
        b0.peer_flags = flags;
        RW_CUDA(cudaMemcpy(dev, &b0, sizeof b0, cudaMemcpyHostToDevice));
      }
      invalidate_graphs(x);
      return;
    }
    if (dir == 0) {
      // forward: our last layer's critical CTAs also store h_t into the next stage's input image
      // and release its per-step counter (rec_cluster.cuh k_cl_fwd); W_next is not needed
      (void)W_next;
      uint8_t* peer_xsw = static_cast<uint8_t*>(open_region(x, peer, 0));
      uint32_t* peer_flags = static_cast<uint32_t*>(open_region(x, peer, 1));
      FwdLayer top;
      FwdLayer* dev_top = static_cast<FwdLayer*>(x->fwd_layers.p) + (L - 1);
      RW_CUDA(cudaMemcpy(&top, dev_top, sizeof top, cudaMemcpyDeviceToHost));
      top.hsw_peer = peer_xsw;
      top.peer_flags = peer_flags;
      RW_CUDA(cudaMemcpy(dev_top, &top, sizeof top, cudaMemcpyHostToDevice));
      x->pp_next_xop = open_region(x, peer, 3);
      if (x->prec == kF16x2) x->pp_next_xop_lo = open_region(x, peer, 2);
      x->pp_next_ready = static_cast<uint32_t*>(open_region(x, peer, 4));
      x->pp_next = true;
      invalidate_graphs(x);
      return;
    }
    ClOff o{};
    o.ring = static_cast<float*>(open_region(x, peer, 0));
    o.done = static_cast<uint32_t*>(open_region(x, peer, 1));
    o.consumed = static_cast<const uint32_t*>(open_region(x, peer, 2));
    o.sys = 1;
    o.active = 1;
    o.unscale = x->prec == kF16x2 ? pow2f(-(kWScaleLog2 + kGScaleLog2)) : 1.0f;  // W^T.dG planes' scales
    o.ko = peer->ko;   // the receiving ring's publication count (rw_pp_export)
    {
      if (!x->pp_prev) einval("rw_pp_link: backward link needs this stage's forward ring exported first");
      x->wb_prev.alloc((size_t)Hp * 2 * G4p * 2);
      if (x->prec == kF16x2) {  // fp16x2: the lo plane lives in tensor memory (the TMEM-A operand)
        x->wb_prev_lo.alloc((size_t)Hp * 2 * G4p * 2);
        o.alo = static_cast<const uint16_t*>(x->wb_prev_lo.p);
        o.alo_ld = (int)(2 * G4p);
        o.alo_rows = Hp;
      }
      o.kdim = (int)G4p;
      // W^T . dgw (GRU: the W-side image, dgw != dgr in the candidate gate)
      o.op = static_cast<const uint8_t*>(x->kind == kCellGru ? x->dgwsw[0].p : x->dgsw[0].p);
      o.op_blk_off = 0;
      o.op_flags = static_cast<const uint32_t*>(x->flags_b.p);
      x->pp_maps[1] = make_map(x->wb_prev.p, x->prec, 2 * G4p, Hp, aK, kTileM);
      x->dirty = true;  // repack_params packs [W_0^T | R_0^T] into wb_prev
    }
    // fixed map slots [forward boundary, backward boundary, ...], device copy allocated once
    pp_upload_maps(x);
    o.a = static_cast<const CUtensorMap*>(x->pp_maps_dev.p) + dir;
    std::vector<ClOff>& offs = dir == 0 ? x->off_f_h : x->off_b_h;
    offs.resize(L + 1);
    offs[L] = o;
    (dir == 0 ? x->rows_f : x->rows_b) = L + 1;
    // the extra row must still be co-resident
    const ClPlan& pl = dir == 0 ? x->cl_f : x->cl_b;
    void* kern = pl.kern;
    const int tiles = dir == 0 ? Hp / kUnitsPerFwdTile : ceil_div(Hp, kTileM);
    const int clusters = max_active_clusters(kern, pl.cs, pl.smem, (L + 1) * tiles * 2 * pl.cs);
    if (clusters < (L + 1) * tiles * 2) einval("rw_pp_link: the stage plus its boundary group does not fit on the GPU");
    upload_cluster_tables(x);
    invalidate_graphs(x);
  });
}

// debug: counters of the boundary rings (pipeline bring-up): out[0..1] epochs (fwd, bwd),
// out[2..4] forward ring of layer 0: done[0..1], consumed; out[6..8] backward ring of the last
// layer: done[0..1], consumed; out[10..11] rows_f, rows_b; out[12..15] ko/sys of those rings.
extern "C" int rw_pp_set_next_w(rw_ctx* x, const float* W_next) {
  // the forward hand-off sends h_t; the next stage multiplies with its own W (which follows its
  // own parameter updates), so there is nothing to refresh here -- kept for API compatibility
  return guarded(x, [&] {
    if (!x->pp_next) einval("rw_pp_set_next_w: no forward link (rw_pp_link dir 0) on this stage");
    if (x->pp_plain) {  // persistent / stepwise: W_next is packed into the top layer's backward image
      if (W_next) {  // a new host copy; NULL: re-read the linked one (the peer's live W_0)
        x->wn_raw.alloc((size_t)x->G * x->H * x->H * 4);
        RW_CUDA(cudaMemcpy(x->wn_raw.p, W_next, x->wn_raw.bytes, cudaMemcpyHostToDevice));
        x->pp_wnext = x->wn_raw.f();
      }
      x->repack_njobs = 0;
      x->dirty = true;
      invalidate_graphs(x);
    }
  });
}

extern "C" int rw_pp_debug(rw_ctx* x, long long* out) {
  return guarded(x, [&] {
    RW_CUDA(cudaDeviceSynchronize());
    uint32_t e[3] = {0, 0, 0};
    RW_CUDA(cudaMemcpy(e, x->cl_epoch.p, 12, cudaMemcpyDeviceToHost));
    out[0] = e[0];
    out[1] = e[1];
    auto rd = [&](const uint32_t* p) {
      uint32_t v = 0;
      RW_CUDA(cudaMemcpy(&v, p, 4, cudaMemcpyDeviceToHost));
      return (long long)v;
    };
    const ClRing& f = x->ring_f_h[0];
    const ClRing& b = x->ring_b_h[x->L - 1];
    out[2] = rd(f.done);
    out[3] = rd(f.done + 1);
    out[4] = rd(f.consumed);
    out[6] = rd(b.done);
    out[7] = rd(b.done + 1);
    out[8] = rd(b.consumed);
    out[10] = x->rows_f;
    out[11] = x->rows_b;
    out[12] = f.ko;
    out[13] = f.sys;
    out[14] = b.ko;
    out[15] = b.sys;
  });
}

int rw_nccl_unique_id(char* id128) {
  return guarded(nullptr, [&] {
    NcclId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id128, id.internal, 128);
  });
}

int rw_comm_init(rw_ctx* x, int nranks, int rank, const char* id128) {
  return guarded(x, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) einval("rw_comm_init: bad rank/nranks");
    RW_CUDA(cudaSetDevice(x->dev));
    NcclId id;
    std::memcpy(id.internal, id128, 128);
    nccl_check(nccl().CommInitRank(&x->comm, nranks, id, rank), "ncclCommInitRank");
    x->nranks = nranks;
    x->rank = rank;
  });
}

static void allreduce_grads(rw_ctx* x, cudaStream_t s) {
  if (x->dp_overlap) return;  // the pass already summed every bucket (rw_comm_overlap)
  Nccl& n = nccl();
  nccl_check(n.GroupStart(), "ncclGroupStart");
  for (int l = x->L - 1; l >= 0; --l) {  // top layer's gradients are final first
    const int Il = l == 0 ? x->I : x->H;
    nccl_check(n.AllReduce(x->dW[l].p, x->dW[l].p, (unsigned long long)x->G * x->H * Il, kNcclFloat32, kNcclSum, x->comm, s), "ncclAllReduce dW");
    nccl_check(n.AllReduce(x->dR[l].p, x->dR[l].p, (unsigned long long)x->G * x->H * x->H, kNcclFloat32, kNcclSum, x->comm, s), "ncclAllReduce dR");
    nccl_check(n.AllReduce(x->db[l].p, x->db[l].p, (unsigned long long)x->G * x->H, kNcclFloat32, kNcclSum, x->comm, s), "ncclAllReduce db");
  }
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
}

// Overlapped data-parallel gradient sums: every later training pass all-reduces each layer's
// bucket inside the pass, as soon as its weight-gradient GEMMs finish (top layer first), on a
// communication stream, while the lower layers' GEMMs and the dx0 GEMM still run.
extern "C" int rw_comm_overlap(rw_ctx* x, int on) {
  return guarded(x, [&] {
    if (on && !x->comm) einval("rw_comm_overlap: rw_comm_init was not called");
    RW_CUDA(cudaSetDevice(x->dev));
    if (on && !x->comm_s) {
      RW_CUDA(cudaStreamCreateWithFlags(&x->comm_s, cudaStreamNonBlocking));
      x->ev_layer.resize(x->L);
      for (auto& e : x->ev_layer) RW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      RW_CUDA(cudaEventCreateWithFlags(&x->ev_comm, cudaEventDisableTiming));
    }
    if (x->dp_overlap != (on != 0)) invalidate_graphs(x);
    x->dp_overlap = on != 0;
  });
}

int rw_allreduce_grads(rw_ctx* x, void* stream) {
  return guarded(x, [&] {
    if (!x->comm) einval("rw_allreduce_grads: rw_comm_init was not called");
    allreduce_grads(x, stream ? static_cast<cudaStream_t>(stream) : x->main);
  });
}

// ---- schedule trace in the reference's task model (scheduler.hpp:96-155, 180-192), block width
// 1: the device wavefront's unit of work is one step (INPUT_GEMM(l, t) = W_l.x_t, the W.x of
// one step; RECURRENT_STEP(l, t)). Task ids follow build_graph(L, T, 1): input_id(l, j) =
// l * 2T + j, recurrent_id(l, t) = l * 2T + T + t. Aggregated over the CTAs of a task: start =
// the first CTA's "dependencies satisfied" stamp, end = the last CTA's stamp taken before its
// release, so a consumer's start never precedes its producers' ends. The persistent / stepwise
// kernels fuse W.x into the step's accumulator: their INPUT_GEMM records are the instant the step's
// inputs were all available (zero length, ending where the step starts). Backward (the reversed
// graph): INPUT_GEMM(l, t) is layer l's output GEMM W_l^T.dG_{l,t}, i.e. the off-critical group
// of layer l - 1 (cluster) or fused into layer l - 1's step (persistent / stepwise); for l = 0
// it is the dx0 GEMM, recorded once around the whole launch.
struct TraceRec {
  int task_id, layer, block, step_k, phase, worker;
  long long start_ns, end_ns;
};

static std::vector<TraceRec> trace_records(rw_ctx* x, int dir) {
  const int L = x->L, T = x->T, sched = dir == 0 ? x->fwd_sched : x->bwd_sched;
  const int steps = dir == 0 ? T : T + 1;  // backward: + the dh0 step (not a reference task)
  std::vector<TraceRec> out;
  const unsigned long long kNone = ~0ULL;
  struct Agg {
    unsigned long long s = ~0ULL, e = 0;
    int w = 0;
    bool ok() const { return s != ~0ULL && e != 0; }
  };
  std::vector<Agg> rec((size_t)L * T), inp((size_t)L * T);
  auto tof = [&](int it) { return dir == 0 ? it : T - 1 - it; };
  if (sched == RW_SCHED_CLUSTER) {
    const ClPlan& pl = dir == 0 ? x->cl_f : x->cl_b;
    const int tiles = dir == 0 ? x->Hp / kUnitsPerFwdTile : ceil_div(x->Hp, kTileM);
    const int gx = tiles * 2 * pl.cs, rows = dir == 0 ? x->rows_f : x->rows_b;
    std::vector<unsigned long long> h((size_t)rows * gx * steps * 16);
    RW_CUDA(cudaMemcpy(h.data(), (dir == 0 ? x->trace_f : x->trace_b).p, h.size() * 8, cudaMemcpyDeviceToHost));
    for (int y = 0; y < std::min(rows, L); ++y)
      for (int bx = 0; bx < gx; ++bx) {
        const bool crit = ((bx / pl.cs) & 1) == 0;
        const int lt = crit ? y : (dir == 0 ? y : y + 1);  // task layer
        if (lt >= L) continue;
        for (int it = 0; it < steps; ++it) {
          const int t = tof(it);
          if (t < 0) continue;
          const unsigned long long* st = &h[(((size_t)y * gx + bx) * steps + it) * 16];
          // start: for a recurrent step, the moment every input of its accumulation is in the CTA
          // (the epilogue received the off partial: stamp 10 forward, 13 backward); for an input
          // GEMM, its first operand k-block landed (stamp 8). Both trail the producers' releases by
          // a load latency, so %globaltimer skew between SMs (a 32 ns tick or two) cannot invert an
          // edge; the dependencies-acquired stamps (14 / 1) are the fallback.
          const unsigned long long sa = crit ? st[dir == 0 ? 10 : 13] : st[8];
          const unsigned long long a = sa ? sa : (crit ? st[14] : st[1]), b = st[15];
          if (!a || !b) continue;  // inactive member
          Agg& g = (crit ? rec : inp)[(size_t)lt * T + t];
          g.s = std::min(g.s, a);
          if (b >= g.e) {
            g.e = b;
            g.w = bx;
          }
        }
      }
  } else if (sched == RW_SCHED_PERSISTENT || sched == RW_SCHED_STEPWISE) {
    const int ks = dir == 0 ? x->ks_f : x->ks_b;
    const bool pair = dir == 0 ? x->pair_f : x->pair_b;
    const int tiles = dir == 0 ? x->Hp / kUnitsPerFwdTile : ceil_div(x->Hp, kTileM);
    const int gx = pair && sched == RW_SCHED_PERSISTENT ? tiles : tiles * ks;
    const bool stepwise = sched == RW_SCHED_STEPWISE;
    std::vector<unsigned long long> h((size_t)L * gx * steps * 8);
    RW_CUDA(cudaMemcpy(h.data(), (dir == 0 ? x->trace_f : x->trace_b).p, h.size() * 8, cudaMemcpyDeviceToHost));
    for (int l = 0; l < L; ++l)
      for (int w = 0; w < gx; ++w)
        for (int it = 0; it < steps; ++it) {
          const int t = tof(it);
          if (t < 0) continue;
          const size_t i = stepwise ? (((size_t)l * steps + it) * gx + w) : (((size_t)l * gx + w) * steps + it);
          const unsigned long long a = h[i * 8 + 1], b = h[i * 8 + 6];
          if (!a || !b) continue;
          Agg& g = rec[(size_t)l * T + t];
          g.s = g.s == kNone ? a : std::max(g.s, a);  // all CTAs' inputs available (W.x fused)
          if (b >= g.e) {
            g.e = b;
            g.w = w;
          }
        }
    for (int l = 0; l < L; ++l)
      for (int t = 0; t < T; ++t) {
        const int host = dir == 0 ? l : l - 1;  // the step the input / output GEMM is fused into
        if (host < 0) continue;
        const Agg& r = rec[(size_t)host * T + t];
        Agg& g = inp[(size_t)l * T + t];
        g.s = r.s;
        g.e = r.s;
        g.w = r.w;
      }
  } else {
    throw RwError{RW_EINVAL, "trace: records need the cluster, persistent or stepwise schedule"};
  }
  if (dir == 1) {  // INPUT_GEMM(0, t) of the backward: the dx0 GEMM
    unsigned long long d[2] = {0, 0};
    RW_CUDA(cudaMemcpy(d, x->trace_dx.p, 16, cudaMemcpyDeviceToHost));
    for (int t = 0; t < T; ++t) inp[t] = Agg{d[0], d[1], 0};
  }
  unsigned long long t0 = kNone;
  for (auto* v : {&rec, &inp})
    for (const Agg& g : *v)
      if (g.ok()) t0 = std::min(t0, g.s);
  for (int l = 0; l < L; ++l)
    for (int t = 0; t < T; ++t) {
      const Agg& gi = inp[(size_t)l * T + t];
      const Agg& gr = rec[(size_t)l * T + t];
      if (gi.ok() || (gi.s != kNone && gi.s == gi.e))
        out.push_back(TraceRec{l * 2 * T + t, l, t, 0, 0, gi.w, (long long)(gi.s - t0), (long long)(gi.e - t0)});
      if (gr.ok())
        out.push_back(TraceRec{l * 2 * T + T + t, l, t, 0, 1, gr.w, (long long)(gr.s - t0), (long long)(gr.e - t0)});
    }
  std::sort(out.begin(), out.end(), [](const TraceRec& a, const TraceRec& b) {
    return a.start_ns != b.start_ns ? a.start_ns < b.start_ns : a.task_id < b.task_id;
  });
  return out;
}

// RW_TRACE=<csv>: the last synced pass's forward trace in write_trace_csv's schema
// (scheduler.hpp:406-417), the backward one in <csv>.bwd.csv.
static void dump_trace_csv(rw_ctx* x) {
  if (x->trace_path.empty()) return;
  for (int dir = 0; dir < 2; ++dir) {
    std::vector<TraceRec> r;
    try {
      r = trace_records(x, dir);
    } catch (const RwError&) {
      continue;
    }
    if (r.empty()) continue;
    const std::string path = dir == 0 ? x->trace_path : x->trace_path + ".bwd.csv";
    FILE* f = fopen(path.c_str(), "w");
    if (!f) continue;
    fprintf(f, "task_layer,task_block,phase,worker,start_ns,end_ns\n");
    for (const TraceRec& t : r) {
      if (t.phase == 0)
        fprintf(f, "%d,%d,INPUT_GEMM,%d,%lld,%lld\n", t.layer, t.block, t.worker, t.start_ns, t.end_ns);
      else
        fprintf(f, "%d,%d,RECURRENT_STEP(%d),%d,%lld,%lld\n", t.layer, t.block, t.step_k, t.worker, t.start_ns,
                t.end_ns);
    }
    fclose(f);
  }
}

// Write the persistent kernels' step stamps as CSV in the reference trace schema
// (scheduler.hpp:411-417): task_layer,task_block,phase,worker,start_ns,end_ns, with
// task_block = step, worker = CTA index within the layer, phase = fwd|bwd, and three spans
// per (CTA, step): wait (inputs), mma (inputs ready -> accumulator), epilogue (-> published).
static void dump_trace(rw_ctx* x) {
  dump_trace_csv(x);
  if (x->trace_spans_path.empty()) return;
  FILE* f = fopen(x->trace_spans_path.c_str(), "w");
  if (!f) return;
  fprintf(f, "task_layer,task_block,phase,worker,span,start_ns,end_ns\n");
  for (int dir = 0; dir < 2; ++dir) {
    if ((dir == 0 ? x->fwd_sched : x->bwd_sched) == RW_SCHED_CLUSTER) {
      // stamps: 0 step start, 1 operand published, 2 accumulator ready, 3 partial pushed (off
      // members), 4 partials reduced, 5 operand published, 6 tapes written
      const int steps = dir == 0 ? x->T : x->T + 1;
      const int per_layer = (dir == 0 ? x->Hp / kUnitsPerFwdTile : ceil_div(x->Hp, kTileM)) * 2 *
                            (dir == 0 ? x->cl_f.cs : x->cl_b.cs);
      std::vector<unsigned long long> h((size_t)x->L * per_layer * steps * 16);
      cudaMemcpy(h.data(), (dir == 0 ? x->trace_f : x->trace_b).p, h.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ULL;
      for (auto v : h)
        if (v && v < t0) t0 = v;
      // critical members (cluster index even): wait 0-1, load 1-7, mma 7-2, reduce 2-4,
      // cell 4-3, publish 3-5, tapes 5-6; off members: offload 1-7, offmma 7-2, offstep 2-3
      const int cs = dir == 0 ? x->cl_f.cs : x->cl_b.cs;
      const int fromc[13] = {0, 1, 7, 2, 4, 3, 5, 1, 2, 9, 10, 11, 12};
      const int toc[13] = {1, 7, 2, 4, 3, 5, 6, 8, 9, 10, 11, 12, 13};
      const char* namec[13] = {"wait", "load", "mma", "reduce", "cell", "publish", "tapes", "kb0",
                               "r_drain", "r_own", "r_peers", "r_sum", "r_off"};
      const int fromo[9] = {1, 7, 2, 1}, too[9] = {7, 2, 3, 8};
      const char* nameo[9] = {"offload", "offmma", "offstep", "offkb0"};
      for (int l = 0; l < x->L; ++l)
        for (int w = 0; w < per_layer; ++w)
          for (int it = 0; it < steps; ++it) {
            const unsigned long long* st = &h[(((size_t)l * per_layer + w) * steps + it) * 16];
            const int t = dir == 0 ? it : x->T - 1 - it;
            const bool critm = ((w / cs) & 1) == 0;
            const int* from = critm ? fromc : fromo;
            const int* to = critm ? toc : too;
            const char* const* names = critm ? namec : nameo;
            for (int k = 0; k < (critm ? 13 : 4); ++k)
              if (st[from[k]] && st[to[k]])
                fprintf(f, "%d,%d,%s,%d,%s,%llu,%llu\n", l, t, dir == 0 ? "fwd" : "bwd", w, names[k],
                        st[from[k]] - t0, st[to[k]] - t0);
          }
      continue;
    }
    if ((dir == 0 ? x->fwd_sched : x->bwd_sched) != RW_SCHED_PERSISTENT) continue;
    const int steps = dir == 0 ? x->T : x->T + 1;
    const int ks = dir == 0 ? x->ks_f : x->ks_b;
    const int tiles = dir == 0 ? x->Hp / kUnitsPerFwdTile : ceil_div(x->Hp, kTileM);
    const int per_layer = tiles * ks;
    std::vector<unsigned long long> h((size_t)x->L * per_layer * steps * 8);
    cudaMemcpy(h.data(), (dir == 0 ? x->trace_f : x->trace_b).p, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ULL;
    for (auto v : h)
      if (v && v < t0) t0 = v;
    const char* names[7] = {"wait", "mma", "push", "xchg", "cells", "release", "publish"};
    for (int l = 0; l < x->L; ++l)
      for (int w = 0; w < per_layer; ++w)
        for (int it = 0; it < steps; ++it) {
          const unsigned long long* s = &h[(((size_t)l * per_layer + w) * steps + it) * 8];
          const int t = dir == 0 ? it : x->T - 1 - it;
          const char* ph = dir == 0 ? "fwd" : "bwd";
          for (int k = 0; k < 7; ++k)
            if (s[k] && s[k + 1])
              fprintf(f, "%d,%d,%s,%d,%s,%llu,%llu\n", l, t, ph, w, names[k], s[k] - t0, s[k + 1] - t0);
        }
  }
  fclose(f);
}

int rw_sync(rw_ctx* x) {
  return guarded(x, [&] {
    RW_CUDA(cudaSetDevice(x->dev));
    RW_CUDA(cudaDeviceSynchronize());
    RW_CUDA(cudaGetLastError());
    check_error_flag(x);
    dump_trace(x);
  });
}

// One forward pass (inference) of ladder rung `level` (0-4; run_ladder_forward); the context
// must use the stepwise schedule for LSTM cells. Inputs: rw_upload_inputs; output y as for
// rw_run_pass (rw_read_outputs).
int rw_ladder_pass(rw_ctx* x, int level, void* stream) {
  return guarded(x, [&] {
    if (level < 0 || level > 4) einval("rw_ladder_pass: level must be 0..4 (5 / 6 are the layerseq / auto schedules)");
    if (x->kind != kCellLstm) einval("rw_ladder_pass: the ladder runs LSTM cells");
    if (x->fwd_sched != RW_SCHED_STEPWISE) einval("rw_ladder_pass: create the context with the stepwise schedule");
    if (x->prec == kTF32x3 && level <= 3) einval("rw_ladder_pass: rungs 0-3 read MN-major operands (bf16 / fp16x2 only)");
    require_params(x);
    RW_CUDA(cudaSetDevice(x->dev));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : x->main;
    if (x->dirty) repack_params(x, s);
    forward_prologue(x, s, nullptr, nullptr, true);
    by_prec(x->prec, [&](auto tag) { run_ladder_forward<decltype(tag)>(x, level, s); });
    x->tape_gen += 1;
    x->tape_training = false;
    x->bwd_done = false;
  });
}

int rw_trace_enable(rw_ctx* x, int on) {
  return guarded(x, [&] {
    RW_CUDA(cudaSetDevice(x->dev));
    if (on && !x->tracing) {
      trace_alloc(x);
      invalidate_graphs(x);  // captured passes hold the (null) trace pointers
    } else if (!on && x->tracing) {
      x->tracing = false;
      invalidate_graphs(x);
    }
  });
}

int rw_trace_records(rw_ctx* x, int direction, rw_trace_record* out, int capacity, int* count) {
  return guarded(x, [&] {
    if (!x->tracing) einval("rw_trace_records: tracing is off (rw_trace_enable)");
    if (direction != 0 && direction != 1) einval("rw_trace_records: direction must be 0 (forward) or 1 (backward)");
    RW_CUDA(cudaSetDevice(x->dev));
    RW_CUDA(cudaStreamSynchronize(x->main));
    const std::vector<TraceRec> r = trace_records(x, direction);
    if (count) *count = (int)r.size();
    for (int i = 0; i < (int)r.size() && out && i < capacity; ++i) {
      const TraceRec& t = r[i];
      out[i] = rw_trace_record{t.task_id, t.layer, t.block, t.step_k, t.phase, t.worker, t.start_ns, t.end_ns};
    }
  });
}

int rw_set_profiling(rw_ctx* x, int on) {
  return guarded(x, [&] { x->profiling = on != 0; });
}

int rw_phase_times(rw_ctx* x, double* out_ms, int* out_n, int n, int reset) {
  return guarded(x, [&] {
    for (int i = 0; i < n && i < 6; ++i) {
      if (out_ms) out_ms[i] = x->phase_ms[i];
      if (out_n) out_n[i] = x->phase_n[i];
    }
    if (reset)
      for (int i = 0; i < 6; ++i) {
        x->phase_ms[i] = 0;
        x->phase_n[i] = 0;
      }
  });
}

int rw_describe(rw_ctx* x, int* fs, int* bs, int* kf, int* kb) {
  return guarded(x, [&] {
    if (fs) *fs = x->fwd_sched;
    if (bs) *bs = x->bwd_sched;
    if (kf) *kf = x->ks_f;
    if (kb) *kb = x->ks_b;
  });
}

int rw_describe_precision(rw_ctx* x, int* fmt) {
  return guarded(x, [&] {
    if (fmt) *fmt = x->prec;
  });
}

int rw_describe_variants(rw_ctx* x, int* fwd_pair, int* wgrad_bn) {
  return guarded(x, [&] {
    if (fwd_pair) *fwd_pair = (x->pair_f ? 1 : 0) | (x->pair_b ? 2 : 0);
    if (wgrad_bn) *wgrad_bn = x->bn_wg;
    if (fwd_pair) *fwd_pair |= (x->ls_pers_f ? 4 : 0) | (x->ls_pers_b ? 8 : 0);
  });
}

// gemm (gemm.hpp:339-347) on the device: C = alpha op(A) op(B) + beta C with host column-major
// buffers, 3xTF32 split operands (fp32-parity) on the tcgen05 GEMM with chunked fp32 promotion.
int rw_gemm(int trans_a, int trans_b, int M, int N, int K, float alpha, const float* A, long long lda,
            const float* B, long long ldb, float beta, float* C, long long ldc) {
  return guarded(nullptr, [&] {
    if (M < 0 || N < 0 || K < 0) einval("gemm: negative dimension");
    if (M == 0 || N == 0) return;
    if (!A || !B || !C) einval("gemm: null operand");
    if (ldc < M || lda < (trans_a ? K : M) || ldb < (trans_b ? N : K)) einval("gemm: leading dimension too small");
    const int prec = kTF32x3, aK = prec_atomk(prec), bn = 64;
    const int Mp = round_up(M, kTileM), Np = round_up(N, bn), Kp = round_up(std::max(K, 1), aK);
    const long long a_src = trans_a ? (long long)M * lda : (long long)std::max(K, 1) * lda;
    const long long b_src = trans_b ? (long long)std::max(K, 1) * ldb : (long long)N * ldb;
    DevBuf dA, dB, dC, errw;
    dA.alloc(std::max<long long>(a_src, 1) * 4);
    dB.alloc(std::max<long long>(b_src, 1) * 4);
    dC.alloc((size_t)M * N * 4);
    errw.alloc(16);
    if (K > 0) {
      RW_CUDA(cudaMemcpy(dA.p, A, (size_t)(trans_a ? (long long)(M - 1) * lda + K : (long long)(K - 1) * lda + M) * 4,
                         cudaMemcpyHostToDevice));
      RW_CUDA(cudaMemcpy(dB.p, B, (size_t)(trans_b ? (long long)(K - 1) * ldb + N : (long long)(N - 1) * ldb + K) * 4,
                         cudaMemcpyHostToDevice));
    }
    RW_CUDA(cudaMemcpy2D(dC.p, (size_t)M * 4, C, (size_t)ldc * 4, (size_t)M * 4, N, cudaMemcpyHostToDevice));
    ++g_launches;
    k_scale_cols<<<grid_for((long long)M * N), 256>>>(dC.f(), M, M, N, beta);
    if (K > 0 && alpha != 0.0f) {
      Operand Ao, Bo;
      Ao.alloc(prec, (size_t)Mp * Kp);
      Bo.alloc(prec, (size_t)Np * Kp);
      ++g_launches;
      k_pack_gemm_operand<<<grid_for((long long)Mp * Kp), 256>>>(dA.f(), lda, M, K, trans_a, Mp, Kp, prec, Ao.p(0),
                                                                  Ao.p(1));
      // B' (N x K) = op(B)^T: op(B)(k, n) is B[n * ldb + k] (B stored K x N) or B[k * ldb + n] (stored N x K)
      ++g_launches;
      k_pack_gemm_operand<<<grid_for((long long)Np * Kp), 256>>>(dB.f(), ldb, N, K, trans_b ? 0 : 1, Np, Kp, prec,
                                                                  Bo.p(0), Bo.p(1));
      RW_CUDA(cudaGetLastError());
      std::vector<CUtensorMap> maps;
      for (int p = 0; p < 2; ++p) {
        maps.push_back(make_map(Ao.p(p), prec, Kp, Mp, aK, kTileM));
        maps.push_back(make_map(Bo.p(p), prec, Kp, Np, aK, gemm_box_rows(bn)));
      }
      DevBuf md;
      md.alloc(maps.size() * sizeof(CUtensorMap));
      RW_CUDA(cudaMemcpy(md.p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
      const CUtensorMap* MD = static_cast<const CUtensorMap*>(md.p);
      GemmDesc g{};
      g.error = static_cast<int*>(errw.p);
      g.a[0] = MD + 0;
      g.b[0] = MD + 1;
      g.a[1] = MD + 2;
      g.b[1] = MD + 3;
      g.alpha = alpha;
      g.accumulate = 1;
      g.M = Mp;
      g.N = Np;
      g.K = Kp;
      g.d = dC.f();
      g.ldd = M;
      g.row_mode = kRowIdentity;
      g.col_mode = kColIdentity;
      g.m_valid = M;
      g.n_valid = N;
      DevBuf gd;
      gd.alloc(sizeof(GemmDesc));
      RW_CUDA(cudaMemcpy(gd.p, &g, sizeof g, cudaMemcpyHostToDevice));
      launch_gemm<PrecTF32x3, false, false>(static_cast<const GemmDesc*>(gd.p), 1, Mp, Np, bn,
                                           gemm_stages(2, bn), 0);
    }
    RW_CUDA(cudaDeviceSynchronize());
    int ew = 0;
    RW_CUDA(cudaMemcpy(&ew, errw.p, 4, cudaMemcpyDeviceToHost));
    if (ew) throw RwError{RW_ESTATE, "gemm: a pipeline barrier wait timed out"};
    RW_CUDA(cudaMemcpy2D(C, (size_t)ldc * 4, dC.p, (size_t)M * 4, (size_t)M * 4, N, cudaMemcpyDeviceToHost));
  });
}

static float g_test_gemm_ms = 0.0f;
float rw_test_gemm_last_ms(void) { return g_test_gemm_ms; }

int rw_test_gemm(int precision, int a_mn, int b_mn, int M, int N, int K, const float* dA,
                 long long lda, const float* dB, long long ldb, float* dD, long long ldd, int bn) {
  return guarded(nullptr, [&] {
    // precision 2 (test hook only): the fp16x2 split operands of the fp32-parity cluster path
    const int prec = precision == RW_PREC_BF16 ? kBF16 : precision == 2 ? kF16x2 : kTF32x3;
    const int aK = prec_atomk(prec);
    if (M % 128 || N % bn || K % 64 || (bn != 64 && bn != 128 && bn != 256)) einval("rw_test_gemm: bad shape");
    if (prec != kBF16 && bn == 256) einval("rw_test_gemm: two-plane operands take bn 64 or 128");
    if (prec == kTF32x3 && (a_mn || b_mn)) einval("rw_test_gemm: tf32 operands must be K-major");
    // element counts of the stored operands
    const long long a_elems = a_mn ? (long long)K * lda : (long long)M * lda;
    const long long b_elems = b_mn ? (long long)K * ldb : (long long)N * ldb;
    Operand A, Bo;
    A.alloc(prec, a_elems);
    Bo.alloc(prec, b_elems);
    ++g_launches;
    k_pad_cols<<<pad_grid(a_elems), 256>>>(dA, (int)a_elems, 1, 1, (int)a_elems, 1, 0, nullptr, prec, A.p(0), A.p(1));
    ++g_launches;
    k_pad_cols<<<pad_grid(b_elems), 256>>>(dB, (int)b_elems, 1, 1, (int)b_elems, 1, 0, nullptr, prec, Bo.p(0), Bo.p(1));
    RW_CUDA(cudaGetLastError());
    std::vector<CUtensorMap> maps;
    for (int p = 0; p < (prec == kBF16 ? 1 : 2); ++p) {
      maps.push_back(a_mn ? make_map(A.p(p), prec, lda, K, aK, aK) : make_map(A.p(p), prec, lda, M, aK, 128));
      maps.push_back(b_mn ? make_map(Bo.p(p), prec, ldb, K, aK, aK) : make_map(Bo.p(p), prec, ldb, N, aK, gemm_box_rows(bn)));
    }
    DevBuf md;
    md.alloc(maps.size() * sizeof(CUtensorMap));
    RW_CUDA(cudaMemcpy(md.p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    const CUtensorMap* MD = static_cast<const CUtensorMap*>(md.p);
    DevBuf errw;
    errw.alloc(16);
    RW_CUDA(cudaMemset(errw.p, 0, 16));
    GemmDesc g{};
    g.error = static_cast<int*>(errw.p);
    g.a[0] = MD + 0;
    g.b[0] = MD + 1;
    if (prec != kBF16) {
      g.a[1] = MD + 2;
      g.b[1] = MD + 3;
    }
    g.alpha = 1.0f;
    g.M = M;
    g.N = N;
    g.K = K;
    g.d = dD;
    g.ldd = ldd;
    g.row_mode = kRowIdentity;
    g.col_mode = kColIdentity;
    g.m_valid = M;
    g.n_valid = N;
    DevBuf gd;
    gd.alloc(sizeof(GemmDesc));
    RW_CUDA(cudaMemcpy(gd.p, &g, sizeof g, cudaMemcpyHostToDevice));
    const GemmDesc* G = static_cast<const GemmDesc*>(gd.p);
    const int planes = prec_planes(prec);
    const int st = gemm_stages(planes, bn);
    const char* reps_env = getenv("RW_TEST_GEMM_REPS");
    const int reps = reps_env ? std::max(1, atoi(reps_env)) : 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep <= reps; ++rep) {
    if (rep == 1) cudaEventRecord(e0, 0);
    by_prec(prec, [&](auto tag) {
      using P = decltype(tag);
      if (!a_mn && !b_mn) launch_gemm<P, false, false>(G, 1, M, N, bn, st, 0);
      if (!a_mn && b_mn) launch_gemm<P, false, true>(G, 1, M, N, bn, st, 0);
      if (a_mn && !b_mn) launch_gemm<P, true, false>(G, 1, M, N, bn, st, 0);
      if (a_mn && b_mn) launch_gemm<P, true, true>(G, 1, M, N, bn, st, 0);
    });
    }
    cudaEventRecord(e1, 0);
    RW_CUDA(cudaDeviceSynchronize());
    int ew = 0;
    RW_CUDA(cudaMemcpy(&ew, errw.p, 4, cudaMemcpyDeviceToHost));
    if (ew) throw RwError{RW_ESTATE, "rw_test_gemm: a pipeline barrier wait timed out"};
    cudaEventElapsedTime(&g_test_gemm_ms, e0, e1);
    g_test_gemm_ms /= reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

}  // extern "C"

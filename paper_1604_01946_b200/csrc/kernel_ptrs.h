// kernel_ptrs.h -- host-side handles of the templated sm_100a kernels. Each family is
// instantiated in its own translation unit (kernels_cl.cu, kernels_lstm.cu, kernels_gemm*.cu,
// compiled in parallel) and reached from runtime.cu only through these pointers, which are
// launched with cudaLaunchKernelExC.
#pragma once

#include "common.cuh"

namespace rw {

// k_cl_fwd / k_cl_bwd<P, nco / 16, cell class> (rec_cluster.cuh); prec kBF16 or kF16x2; kind
// CellKindDev (one translation unit per cell class: kernels_cl*.cu)
void* cl_kernel_ptr(int prec, bool fwd, int nco, int kind = kCellLstm);
void* cl_kernel_ptr_lstm(int prec, bool fwd, int nco);
void* cl_kernel_ptr_gru(int prec, bool fwd, int nco);
void* cl_kernel_ptr_rnn(int prec, bool fwd, int nco);
// k_lstm_fwd / k_lstm_bwd<P, pair, kind> (lstm_step.cuh); prec kBF16, kF16x2 or kTF32x3 (pair: bf16
// LSTM only); GRU / RNN: no pairs (kernels_lstm_cells.cu)
void* lstm_kernel_ptr(int prec, bool fwd, bool pair, int kind = kCellLstm);
void* lstm_kernel_ptr_cells(int prec, bool fwd, int kind);
// k_gemm_tc<P, AMN, BMN, BNV> (gemm_tc.cuh): bf16 BNV 0; two-plane formats BNV = tile width 64 / 128
void* gemm_tc_ptr(int prec, bool amn, bool bmn, int bnv);
// k_gemm_p<AMN, BMN, BN> / k_gemm_p2<AMN, BMN, BN> (bf16), BN 128 or 256
void* gemm_p_ptr(bool amn, bool bmn, int bn);
void* gemm_p2_ptr(bool amn, bool bmn, int bn);

}  // namespace rw

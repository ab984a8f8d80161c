// Host-side launchers for the layer kernels (used by the C ABI and by the
// pipeline executor).  Tensor maps are built once per buffer/role and can be
// cached by the caller (the executor precomputes them at plan time).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gemm_types.hpp"

namespace pb {

// Row-major bf16 matrix view in HBM: rows x cols, leading dim ld (elements).
struct Mat16 {
  const __nv_bfloat16* ptr;
  int rows, cols, ld;
};

// Operand tensor map for the GEMM: `k_major` picks the box orientation.
//  K-major: inner dim = cols (K), box {64, box_mn}.
//  MN-major: inner dim = cols (MN), box {64, 64}.
CUtensorMap make_operand_tmap(const Mat16& m, bool k_major, int box_mn);

// GEMM tile width chosen for a problem (128 or 256 columns).
int pick_bn(int M, int N);

struct GemmLaunch {
  CUtensorMap ta, tb;
  GemmShape sh;
  EpiParams ep;
  int bn;
  EpiMaps maps{};      // TMA epilogue tensor maps (wgrad + SGD)
  // fp32 verify precision (verify_fp32.cu): CUDA-core FFMA GEMM on fp32
  // operands stored in the same buffers (pointers reinterpreted)
  bool simt = false;
  const float* simt_a = nullptr;
  const float* simt_b = nullptr;
  int simt_lda = 0, simt_ldb = 0;
  bool pair = false;  // persistent CTA-pair kernel
  bool ext = false;   // pair kernel with split-K / halo tiles compiled in
  // programmatic dependent launch: the GEMM's prologue overlaps the previous
  // kernel of its stream (pays for latency-bound small networks; with many
  // stages' large GEMMs sharing the GPU the early-resident CTAs hold SMs the
  // other streams need: -2.3% on the 16 x 4096 step, so the executor enables
  // it per network, session.cu)
  bool pdl = false;
};

// Split count of a forward GEMM of rows x N x K (1 = no split).  Splitting
// cuts a skinny forward's latency but spends more SM-time per flop, so an
// executor that keeps many stages in flight on one GPU turns it off
// (plan_fwd's allow_split).
int fwd_splits(int rows, int N, int K);

// forward: out = act(x[rows, in] * w[out, in]^T + b).  allow_split: a
// skinny forward may split K (latency over SM-time): with fix_ws / fix_cnt
// (fwd_fix_floats / fwd_fix_counters, counters zeroed once) on the CTA-pair
// kernel with an in-kernel fixup, else on single-CTA clusters.
GemmLaunch plan_fwd(const Mat16& x, int x_row_off, int rows, const Mat16& w,
                    const float* bias, int act, __nv_bfloat16* y16, int ld_y16,
                    float* y32, int ld_y32, int y_row_off, bool allow_split = true,
                    bool verify = false, float* fix_ws = nullptr, int* fix_cnt = nullptr);
// workspace floats / counters a split forward of this shape needs (0: no split)
size_t fwd_fix_floats(int rows, int N, int K);
int fwd_fix_counters(int rows, int N);
// dgrad: d[rows, in] = (dz[rows,out] * w[out,in]) .* act'(xin)
GemmLaunch plan_dgrad(const Mat16& dz, const Mat16& w, const __nv_bfloat16* xin,
                      int ld_xin, int act_prev, __nv_bfloat16* d, int ld_d,
                      bool verify = false);
// wgrad+SGD: w_new[out,in] = w_cur - lr * dz[rows,out]^T x[rows,in]
// (x rows start at x_row_off inside its buffer)
// (single_bn > 0: the single-CTA kernel with single_bn-wide tiles -- more,
// smaller update tiles for a latency-bound network)
GemmLaunch plan_wgrad_sgd(const Mat16& dz, const Mat16& x, int x_row_off,
                          const float* w_cur, float* w_new, int ld_w32,
                          __nv_bfloat16* w16, int ld_w16, float lr, bool verify = false,
                          int single_bn = 0);
// single_bn for plan_wgrad_sgd on a latency-bound network (0: the default
// tiling; PIPESIM_WGRAD_SINGLE=64|128|0 overrides)
int latency_wgrad_bn(int out, int in);

// wgrad+SGD with split fp32 masters (gemm_sm100.cuh: master = hi << 16 + lo):
// reads hi/lo of the current version, writes hi (the new version's bf16
// weights) and lo of the new one.  All four are [out, ld] 16-bit row-major.
GemmLaunch plan_wgrad_sgd_split(const Mat16& dz, const Mat16& x, int x_row_off,
                                const __nv_bfloat16* hi_cur, const uint16_t* lo_cur,
                                __nv_bfloat16* hi_new, uint16_t* lo_new, int ld, float lr);
// whether a layer's wgrad+SGD can run with split masters (the pair kernel's
// TMA epilogue: out > 128, 16-byte rows, TMA epilogue not disabled)
bool split_master_eligible(int out, int in, int ld);
// fp32 [rows, cols] (ld_w) <-> hi bf16 + lo residual [rows, cols] (ld)
void launch_split_master(cudaStream_t st, const float* w, int rows, int cols, int ld_w,
                         __nv_bfloat16* hi, uint16_t* lo, int ld);
void launch_join_master(cudaStream_t st, const __nv_bfloat16* hi, const uint16_t* lo, int rows,
                        int cols, int ld, float* w, int ld_w);

// Two consecutive dgrads of a stage backward in one kernel (dgrad_chain.cuh):
// g1 = the plan of layer l's dgrad (out_l <= 64, in_l <= 256 and a multiple
// of 64), g2 = layer l-1's, whose A operand dz_mid (= g1's destination) the
// kernel builds in shared memory and also stores.
struct ChainLaunch {
  CUtensorMap a1, b1, b2, dz;
  GemmShape sh2;
  EpiParams ep2;
  ChainArgs ca;
  int bn = 64;
  bool pdl = false;
};
bool dgrad_chain_eligible(int out_l, int in_l);
ChainLaunch plan_dgrad_chain(const GemmLaunch& g1, const GemmLaunch& g2, const Mat16& dz_mid);
void launch_dgrad_chain(const ChainLaunch& c, cudaStream_t st);

// Two consecutive Linear forwards in one kernel (fwd_chain.cuh): layer l-1
// (x[rows, K1] -> y1[rows, n1], n1 <= 256 and a multiple of 64, written to
// y1 rows from y1_row_off) then layer l, whose epilogue is g2's (layer l's
// plan_fwd: bias + activation, or the fused softmax-CE at launch).
struct FwdChainLaunch {
  CUtensorMap x, w1, w2, y1;
  GemmShape sh1, sh2;
  EpiParams ep2;
  FwdChainArgs fa;
  int act1 = 0;
  bool pdl = false;
};
bool fwd_chain_eligible(int n1, int n2);
FwdChainLaunch plan_fwd_chain(const Mat16& x, int x_row_off, int rows, const Mat16& w1,
                              const float* b1, int act1, __nv_bfloat16* y1, int ld_y1,
                              int y1_row_off, const Mat16& w2, const GemmLaunch& g2);
void launch_fwd_chain(const FwdChainLaunch& c, cudaStream_t st);
void launch_fwd_chain(const FwdChainLaunch& c, cudaStream_t st, const EpiParams& ep2);

void launch_fwd(const GemmLaunch& g, cudaStream_t st);
void launch_dgrad(const GemmLaunch& g, cudaStream_t st);
void launch_wgrad(const GemmLaunch& g, cudaStream_t st);

void launch_bias_sgd(cudaStream_t st, const __nv_bfloat16* dz, int rows,
                     int out, int ld_dz, const float* b_cur, float* b_new,
                     float* b_copy, float lr, int* tag_slot, int* cur_version,
                     int version, const int* trace_src = nullptr,
                     int* trace_dst = nullptr, bool dz_f32 = false);

// fp32 verify precision (verify_fp32.cu)
void launch_simt_gemm(const GemmLaunch& g, int kind, cudaStream_t st);
// rows x cols of f64/f32 (src_f64) -> fp32 rows (leading dims in elements)
void launch_rows_to_f32(cudaStream_t st, const void* src, bool src_f64, int rows, int cols,
                        int ld_src, float* dst, int ld_dst);

// Sets the dynamic-smem attribute of every GEMM instantiation (call before
// any stream capture).
void init_gemm_attributes();

void launch_loss(cudaStream_t st, const float* y, int rows, int cols, int ld_y,
                 const float* targets, int ld_t, int loss, int act_last,
                 float denom, __nv_bfloat16* dz, int ld_dz, float* row_loss,
                 bool dz_f32 = false, const int* labels = nullptr);

void launch_convert_f64_bf16(cudaStream_t st, const double* src, int rows,
                             int cols, int ld_src, __nv_bfloat16* dst,
                             int ld_dst);
void launch_convert_f32_bf16(cudaStream_t st, const float* src, int rows,
                             int cols, int ld_src, __nv_bfloat16* dst,
                             int ld_dst);
void launch_convert_f64_f32(cudaStream_t st, const double* src, float* dst,
                            size_t n);
void launch_convert_f32_f64(cudaStream_t st, const float* src, double* dst, size_t n);
void launch_f32_to_bf16_rows(cudaStream_t st, const float* src, int rows,
                             int cols, int ld_src, __nv_bfloat16* dst,
                             int ld_dst);

}  // namespace pb

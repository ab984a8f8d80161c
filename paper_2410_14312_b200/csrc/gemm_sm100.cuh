// tcgen05 / TMEM / TMA GEMM for the three contractions of a Linear layer.
//
//   forward   Z = X * W^T        A = X   (K-major)   B = W   (K-major)
//   dgrad     D = dZ * W         A = dZ  (K-major)   B = W   (MN-major)
//   wgrad     G = dZ^T * X       A = dZ  (MN-major)  B = X   (MN-major)
//
// (reference loops: proj/src/trainer.cpp:186-204 forward, :255-262 dgrad,
//  :244-253 wgrad, :484-488 SGD).  All operands are row-major bf16 in HBM; the
// "major-ness" is only how the tile is described to the tensor core, so no
// transposed copies are ever materialised.
//
// One CTA computes one 128 x BN output tile.  Roles (128 threads):
//   warp 0 / lane 0 : TMA producer, kStages-deep smem ring (128B swizzle)
//   warp 1 / lane 0 : MMA issuer, tcgen05.mma kind::f16 into TMEM (fp32)
//   warp 2          : TMEM allocator
//   warps 0-3       : epilogue; warp w owns TMEM lanes [32w, 32w+32), i.e.
//                     output rows m0+32w..; the fused epilogue (bias+act,
//                     act'-gating, or SGD update) runs on the fp32 values.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda.h>
#include <type_traits>

#include "gemm_types.hpp"
#include "sm100_ptx.cuh"

namespace pb {

__device__ __forceinline__ float act_fwd(float z, int act) {
  switch (act) {
    case kRelu: return z > 0.f ? z : 0.f;
    case kTanh: return tanhf(z);
    case kSigmoid: return 1.f / (1.f + expf(-z));
    default: return z;
  }
}

// tanh / sigmoid through expf and a fast divide: no called slow paths in
// the epilogue (a call forces the kernel's live registers to the stack);
// absolute error ~1e-7, far below the bf16 rounding of the stored output.
template <int ACT>
__device__ __forceinline__ float act_fwd_t(float z) {
  if constexpr (ACT == kRelu) return z > 0.f ? z : 0.f;
  else if constexpr (ACT == kTanh) return 1.f - __fdividef(2.f, expf(2.f * z) + 1.f);
  else if constexpr (ACT == kSigmoid) return __fdividef(1.f, 1.f + expf(-z));
  else return z;
}

template <int ACT>
__device__ __forceinline__ float act_grad_t(float a) {
  if constexpr (ACT == kRelu) return a > 0.f ? 1.f : 0.f;
  else if constexpr (ACT == kTanh) return 1.f - a * a;
  else if constexpr (ACT == kSigmoid) return a * (1.f - a);
  else return 1.f;
}

// Runs f(integral_constant<ACT>) for the epilogue's activation: the
// activation is a compile-time parameter of the epilogue code, so each
// instantiation stays small (one hot variant per launch keeps the
// instruction cache warm; a runtime switch inside the unrolled element
// loops more than doubled the kernel's code size).
template <int EPI, typename F>
__device__ __forceinline__ void with_act(const EpiParams& ep, F&& f) {
  if constexpr (EPI == kEpiWgradSgd) {
    f(std::integral_constant<int, kLinear>{});
  } else {
    const int a = EPI == kEpiFwd ? ep.act : ep.act_prev;
    switch (a) {
      case kRelu: f(std::integral_constant<int, kRelu>{}); break;
      case kTanh: f(std::integral_constant<int, kTanh>{}); break;
      case kSigmoid: f(std::integral_constant<int, kSigmoid>{}); break;
      default: f(std::integral_constant<int, kLinear>{}); break;
    }
  }
}

// Host-side twin of with_act (kernel selection by activation).
template <int EPI, typename F>
inline void with_act_host(const EpiParams& ep, F&& f) {
  if constexpr (EPI == kEpiWgradSgd) {
    f(std::integral_constant<int, kLinear>{});
  } else {
    const int a = EPI == kEpiFwd ? ep.act : ep.act_prev;
    switch (a) {
      case kRelu: f(std::integral_constant<int, kRelu>{}); break;
      case kTanh: f(std::integral_constant<int, kTanh>{}); break;
      case kSigmoid: f(std::integral_constant<int, kSigmoid>{}); break;
      default: f(std::integral_constant<int, kLinear>{}); break;
    }
  }
}

// Derivative expressed through the activation value a = act(z).
__device__ __forceinline__ float act_grad_from_out(float a, int act) {
  switch (act) {
    case kRelu: return a > 0.f ? 1.f : 0.f;
    case kTanh: return 1.f - a * a;
    case kSigmoid: return a * (1.f - a);
    default: return 1.f;
  }
}

// wgrad+SGD pair kernel: operand ring depth and split-master buffers per
// epilogue warp (kSgdBufs - 2 chunks of masters are loaded ahead: the
// update is HBM-latency-bound per warp)
#ifndef PB_WGRAD_STAGES
#define PB_WGRAD_STAGES 4
#endif
#ifndef PB_SGD_BUFS
#define PB_SGD_BUFS 3
#endif
#ifndef PB_SGD_L2PF
#define PB_SGD_L2PF 0
#endif

template <int BN>
struct GemmCfg {
  static constexpr int kBM = 128;
  static constexpr int kBK = 64;  // 64 bf16 = one 128-byte swizzle row
  static constexpr int kStages = BN >= 256 ? 4 : 6;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256;
  static constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  static_assert(kSmem <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* dst, const float* v,
                                              int valid, bool vec_ok) {
  if (vec_ok && valid >= 16) {
    uint32_t p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      p[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    d4[0] = make_uint4(p[0], p[1], p[2], p[3]);
    d4[1] = make_uint4(p[4], p[5], p[6], p[7]);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < valid) dst[i] = __float2bfloat16_rn(v[i]);
  }
}

// Device-side version accounting: copy the tag of the weight slot this GEMM
// read into the trace entries of the micro-batches it served.
__device__ __forceinline__ void write_tags(const EpiParams& ep) {
  const int v = *ep.tag_src;
  const int n = ep.tag_count > 0 ? ep.tag_count : 1;
  for (int i = 0; i < n; ++i) ep.tag_dst[static_cast<size_t>(i) * ep.tag_stride] = v;
}

// Fused epilogue on one 16-column chunk of one output row (fp32 values).
template <int EPI, int ACT>
__device__ __forceinline__ void epilogue_chunk(const EpiParams& ep, const GemmShape& sh,
                                               int row, int n, int valid, float (&v)[16]) {
  if constexpr (EPI == kEpiFwd) {
    float b[16];
    if (ep.bias && valid == 16 && (reinterpret_cast<uintptr_t>(ep.bias + n) & 15) == 0) {
      const float4* b4 = reinterpret_cast<const float4*>(ep.bias + n);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 q = __ldg(b4 + i);
        b[4 * i] = q.x; b[4 * i + 1] = q.y; b[4 * i + 2] = q.z; b[4 * i + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) b[i] = (ep.bias && i < valid) ? ep.bias[n + i] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = act_fwd_t<ACT>(v[i] + b[i]);
    const size_t yr = static_cast<size_t>(row + ep.y_row_off);
    if (ep.y16)
      store_bf16x16(ep.y16 + yr * ep.ld_y16 + n, v, valid,
                    (ep.ld_y16 % 8) == 0);
    if (ep.y32) {
      float* dst = ep.y32 + yr * ep.ld_y32 + n;
      if (valid == 16 && (ep.ld_y32 % 4) == 0) {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i < valid) dst[i] = v[i];
      }
    }
  } else if constexpr (EPI == kEpiDgrad) {
    if constexpr (ACT != kLinear) {
      const __nv_bfloat16* xr = ep.xin + static_cast<size_t>(row) * ep.ld_xin + n;
      if (valid == 16 && (ep.ld_xin % 8) == 0) {
        const uint4* x4 = reinterpret_cast<const uint4*>(xr);
        uint4 q[2] = {x4[0], x4[1]};
        const __nv_bfloat16* xh = reinterpret_cast<const __nv_bfloat16*>(q);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          v[i] *= act_grad_t<ACT>(__bfloat162float(xh[i]));
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i < valid) v[i] *= act_grad_t<ACT>(__bfloat162float(xr[i]));
      }
    }
    store_bf16x16(ep.d16 + static_cast<size_t>(row) * ep.ld_d16 + n, v, valid,
                  (ep.ld_d16 % 8) == 0);
  } else {  // kEpiWgradSgd
    const size_t o32 = static_cast<size_t>(row) * ep.ld_w32 + n;
    if (valid == 16 && (ep.ld_w32 % 4) == 0) {
      const float4* c4 = reinterpret_cast<const float4*>(ep.w_cur + o32);
      float4* n4 = reinterpret_cast<float4*>(ep.w_new + o32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float4 w = c4[i];
        w.x -= ep.lr * v[4 * i];
        w.y -= ep.lr * v[4 * i + 1];
        w.z -= ep.lr * v[4 * i + 2];
        w.w -= ep.lr * v[4 * i + 3];
        v[4 * i] = w.x; v[4 * i + 1] = w.y; v[4 * i + 2] = w.z; v[4 * i + 3] = w.w;
        n4[i] = w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < valid) {
          const float w = ep.w_cur[o32 + i] - ep.lr * v[i];
          ep.w_new[o32 + i] = w;
          v[i] = w;
        }
    }
    if (ep.w16)
      store_bf16x16(ep.w16 + static_cast<size_t>(row) * ep.ld_w16 + n, v, valid,
                    (ep.ld_w16 % 8) == 0);
  }
}

// Epilogue of one warp's 32 output rows x BN columns of an accumulator.
//
// tcgen05.ld hands thread i row i (32 consecutive columns per load).  Each
// 32x32 block is transposed through padded smem (conflict-free: 33-float
// rows) so that afterwards lane l owns column l of all 32 rows: every global
// access of the epilogue (bias, activations in, weights in/out) becomes one
// 128-byte (fp32) or 64-byte (bf16) contiguous row segment per instruction,
// and the 32 row loads of a block are issued back to back (memory-level
// parallelism for the HBM-bound SGD update).
template <int EPI, int ACT>
__device__ __forceinline__ void epilogue_warp_tile(const EpiParams& ep, const GemmShape& sh,
                                                   int row_base, int n_base, int n_cols,
                                                   uint32_t t_row, float* T) {
  const int lane = threadIdx.x % 32;
  int rows_valid = sh.M - row_base;
  rows_valid = rows_valid > 32 ? 32 : rows_valid;
  // SGD: master weights of the next chunk are prefetched while this chunk
  // is processed (two chunks of row loads in flight per warp).
  float wnext[32];
  if constexpr (EPI == kEpiWgradSgd) {
    const int n = n_base + lane;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      wnext[i] = (i < rows_valid && n < sh.N && !(ep.dbg_skip & 2))
                     ? ep.w_cur[static_cast<size_t>(row_base + i) * ep.ld_w32 + n]
                     : 0.f;
  }
#pragma unroll 1
  for (int c = 0; c < n_cols; c += 32) {
    if (n_base + c >= sh.N) break;  // warp-uniform
    float wcur[32];
    if constexpr (EPI == kEpiWgradSgd) {
#pragma unroll
      for (int i = 0; i < 32; ++i) wcur[i] = wnext[i];
      const int nn = n_base + c + 32 + lane;
      if (c + 32 < n_cols) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          wnext[i] = (i < rows_valid && nn < sh.N && !(ep.dbg_skip & 2))
                         ? ep.w_cur[static_cast<size_t>(row_base + i) * ep.ld_w32 + nn]
                         : 0.f;
      }
    }
    uint32_t r[32];
    ptx::tmem_ld32(t_row + c, r);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) T[lane * 33 + j] = __uint_as_float(r[j]);
    __syncwarp();
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = T[i * 33 + lane];
    __syncwarp();
    const int n = n_base + c + lane;
    const bool col_ok = n < sh.N;
    int rows = sh.M - row_base;
    rows = rows > 32 ? 32 : rows;  // valid rows of this warp block

    if constexpr (EPI == kEpiFwd) {
      const float b = (ep.bias && col_ok) ? ep.bias[n] : 0.f;
      if (col_ok) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i >= rows) break;
          const float a = act_fwd_t<ACT>(v[i] + b);
          const size_t yr = static_cast<size_t>(row_base + i + ep.y_row_off);
          if (ep.y16) ep.y16[yr * ep.ld_y16 + n] = __float2bfloat16_rn(a);
          if (ep.y32) ep.y32[yr * ep.ld_y32 + n] = a;
        }
      }
    } else if constexpr (EPI == kEpiDgrad) {
      if (col_ok) {
        if constexpr (ACT != kLinear) {
          float g[32];
#pragma unroll
          for (int i = 0; i < 32; ++i)
            g[i] = i < rows ? __bfloat162float(
                                  ep.xin[static_cast<size_t>(row_base + i) * ep.ld_xin + n])
                            : 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= act_grad_t<ACT>(g[i]);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i >= rows) break;
          ep.d16[static_cast<size_t>(row_base + i) * ep.ld_d16 + n] = __float2bfloat16_rn(v[i]);
        }
      }
    } else {  // kEpiWgradSgd: w_new = w_cur - lr * g ; w16 = bf16(w_new)
      if (col_ok) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i >= rows) break;
          const float nw = wcur[i] - ep.lr * v[i];
          if (!(ep.dbg_skip & 4)) ep.w_new[static_cast<size_t>(row_base + i) * ep.ld_w32 + n] = nw;
          if (ep.w16 && !(ep.dbg_skip & 8))
            ep.w16[static_cast<size_t>(row_base + i) * ep.ld_w16 + n] = __float2bfloat16_rn(nw);
        }
      }
    }
  }
}

// Row-per-thread epilogue (thread i owns row i; 16-column vector chunks).
// Softmax cross-entropy of one row of logits against its class label, in the
// forward epilogue: the loss kernel's formulas (max-subtracted, one exp per
// logit) on registers.  v holds the finished logits (epilogue_chunk has
// added the bias of the linear head in place).
__device__ __forceinline__ void fused_ce_row(const EpiParams& ep, int row, const float (&v)[16],
                                             int valid) {
  const size_t r = static_cast<size_t>(row + ep.y_row_off);
  float z[16];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    z[i] = i < valid ? v[i] : -INFINITY;
    mx = fmaxf(mx, z[i]);
  }
  const int lab = ep.loss_labels[r];
  float zl = 0.f;  // the label's max-subtracted logit
  float se = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i == lab) zl = z[i] - mx;
    z[i] = i < valid ? expf(z[i] - mx) : 0.f;
    se += z[i];
  }
  __nv_bfloat16* d = ep.loss_dz + r * ep.loss_ld_dz;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i >= valid) break;
    d[i] = __float2bfloat16_rn((z[i] / se - (i == lab ? 1.f : 0.f)) / ep.loss_denom);
  }
  ep.loss_row[r] = logf(se) - zl;
}

template <int EPI, int ACT>
__device__ __forceinline__ void epilogue_warp_rows(const EpiParams& ep, const GemmShape& sh,
                                                   int row_base, int n_base, int n_cols,
                                                   uint32_t t_row) {
  const int row = row_base + static_cast<int>(threadIdx.x % 32);
  const bool row_ok = row < sh.M;
  // dgrad act' gating: the stored activation of chunk c+1 is loaded while
  // chunk c is processed (vector path: full 16-column chunks, 16-byte rows)
  constexpr bool kGate = EPI == kEpiDgrad && ACT != kLinear;
  const bool vec = kGate && (ep.ld_xin % 8) == 0 && (sh.N % 16) == 0;
  const __nv_bfloat16* xrow = kGate ? ep.xin + static_cast<size_t>(row) * ep.ld_xin : nullptr;
  if constexpr (EPI == kEpiWgradSgd) {
    if ((ep.ld_w32 % 4) == 0 && (ep.ld_w16 % 8) == 0 && (sh.N % 16) == 0) {
      // SGD rows: this thread's row, 16 columns per step; the fp32 master of
      // step c+1 is loaded while step c is updated and stored
      const float* wrow = ep.w_cur + static_cast<size_t>(row) * ep.ld_w32;
      float* nrow = ep.w_new + static_cast<size_t>(row) * ep.ld_w32;
      __nv_bfloat16* hrow = ep.w16 ? ep.w16 + static_cast<size_t>(row) * ep.ld_w16 : nullptr;
      float4 wa[4], wb[4];
      if (row_ok && n_base < sh.N)
#pragma unroll
        for (int i = 0; i < 4; ++i) wa[i] = reinterpret_cast<const float4*>(wrow + n_base)[i];
#pragma unroll 1
      for (int c = 0; c < n_cols; c += 16) {
        const int n = n_base + c;
        if (n >= sh.N) break;  // warp-uniform
        if (row_ok && c + 16 < n_cols && n + 16 < sh.N)
#pragma unroll
          for (int i = 0; i < 4; ++i) wb[i] = reinterpret_cast<const float4*>(wrow + n + 16)[i];
        uint32_t r[16];
        ptx::tmem_ld16(t_row + c, r);
        ptx::tmem_ld_wait();
        if (row_ok) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            v[4 * i] = wa[i].x - ep.lr * __uint_as_float(r[4 * i]);
            v[4 * i + 1] = wa[i].y - ep.lr * __uint_as_float(r[4 * i + 1]);
            v[4 * i + 2] = wa[i].z - ep.lr * __uint_as_float(r[4 * i + 2]);
            v[4 * i + 3] = wa[i].w - ep.lr * __uint_as_float(r[4 * i + 3]);
            reinterpret_cast<float4*>(nrow + n)[i] =
                make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
          if (hrow) store_bf16x16(hrow + n, v, 16, true);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) wa[i] = wb[i];
      }
      return;
    }
  }
  uint4 xa[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
  if (vec && row_ok && n_base < sh.N) {
    const uint4* p = reinterpret_cast<const uint4*>(xrow + n_base);
    xa[0] = p[0];
    xa[1] = p[1];
  }
#pragma unroll 1
  for (int c = 0; c < n_cols; c += 16) {
    const int n = n_base + c;
    if (n >= sh.N) break;  // warp-uniform
    uint4 xb[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    if (vec && row_ok && c + 16 < n_cols && n + 16 < sh.N) {
      const uint4* p = reinterpret_cast<const uint4*>(xrow + n + 16);
      xb[0] = p[0];
      xb[1] = p[1];
    }
    uint32_t r[16];
    ptx::tmem_ld16(t_row + c, r);
    ptx::tmem_ld_wait();
    if (row_ok) {
      const int valid = sh.N - n < 16 ? sh.N - n : 16;
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
      if constexpr (kGate) {
        if (vec) {
          const __nv_bfloat16* xh = reinterpret_cast<const __nv_bfloat16*>(xa);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] *= act_grad_t<ACT>(__bfloat162float(xh[i]));
          store_bf16x16(ep.d16 + static_cast<size_t>(row) * ep.ld_d16 + n, v, valid,
                        (ep.ld_d16 % 8) == 0);
        } else {
          epilogue_chunk<EPI, ACT>(ep, sh, row, n, valid, v);
        }
      } else {
        epilogue_chunk<EPI, ACT>(ep, sh, row, n, valid, v);
        if constexpr (EPI == kEpiFwd)
          if (ep.loss_dz && n == 0 && sh.N <= 16) fused_ce_row(ep, row, v, valid);
      }
    }
    xa[0] = xb[0];
    xa[1] = xb[1];
  }
}

// Vectorised transposed epilogue (the default): one warp's 32 rows x
// n_cols accumulator, 32 columns per step.  tcgen05.ld hands thread i row i;
// the 32 x 32 fp32 block is staged row-major in swizzled smem (below), then
// lane l serves row
// 4*rr + l/8, columns 4*(l%8)..+3 of the block for rr = 0..7.  Every global
// access is a 16-byte (fp32) or 8-byte (bf16) vector and one warp
// instruction covers 4 full row segments (4 x 128 B fp32 / 4 x 64 B bf16):
// a quarter of the memory instructions of a lane-per-column layout.  The
// global inputs of step c+1 (fp32 masters for SGD, stored activations for
// the dgrad gate) are loaded while step c is processed.
// Staging block: 32 rows x 32 fp32 (4 KB per warp), 16-byte chunks XOR-
// swizzled by row (chunk j of row r at slot j ^ (r & 7)): the row-wise float4
// stores of 32 lanes and the 4-rows-per-instruction float4 reads are both at
// the 4-wavefront minimum, and no padding is spent (the mainloop ring keeps
// the shared memory: more bytes in flight per SM).
constexpr int kVecLd = 32;  // staging row stride (floats)
__device__ __forceinline__ int vec_slot(int row, int chunk) { return (chunk ^ (row & 7)) * 4; }

template <int EPI, int ACT, bool FIX = false>
__device__ __forceinline__ void epilogue_warp_vec(const EpiParams& ep, const GemmShape& sh,
                                                  int row_base, int n_base, int n_cols,
                                                  uint32_t t_row, float* T,
                                                  const FixSrc& fix = FixSrc{}) {
  const int lane = threadIdx.x % 32;
  const int sub_r = lane >> 3;
  const int c4 = (lane & 7) * 4;
  constexpr bool kSgd = EPI == kEpiWgradSgd;
  constexpr bool kGate = EPI == kEpiDgrad && ACT != kLinear;
  // per-step global inputs: 8 rows per lane
  float4 win[8];
  uint2 xin[8];
  auto load_inputs = [&](int c, float4 (&w)[8], uint2 (&x)[8]) {
    const int n = n_base + c + c4;
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int row = row_base + rr * 4 + sub_r;
      const bool ok = row < sh.M && n + 3 < sh.N;
      if constexpr (kSgd) {
        w[rr] = ok ? __ldcs(reinterpret_cast<const float4*>(ep.w_cur + static_cast<size_t>(row) *
                                                                           ep.ld_w32 + n))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      } else if constexpr (kGate) {
        x[rr] = ok ? *reinterpret_cast<const uint2*>(ep.xin + static_cast<size_t>(row) *
                                                                  ep.ld_xin + n)
                   : make_uint2(0u, 0u);
      }
    }
  };
  // fwd bias: this step's float4 and the next step's, loaded one step ahead
  // like the other inputs (an L2 round trip per step otherwise)
  auto load_bias = [&](int c) {
    const int n = n_base + c + c4;
    if constexpr (EPI == kEpiFwd)
      if (ep.bias && n + 3 < sh.N) return __ldg(reinterpret_cast<const float4*>(ep.bias + n));
    return make_float4(0.f, 0.f, 0.f, 0.f);
  };
  load_inputs(0, win, xin);
  float4 bias4 = load_bias(0);
#pragma unroll 1
  for (int c = 0; c < n_cols; c += 32) {
    if (n_base + c >= sh.N) break;  // warp-uniform
    {
      uint32_t r[32];
      ptx::tmem_ld32(t_row + c, r);
      ptx::tmem_ld_wait();
      if constexpr (FIX) {
        // split-K fixup: the S partials of these 32 columns in split order,
        // this unit's own from TMEM, the others from their warp-blocked slots
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
        for (int sp = 0; sp < fix.S; ++sp) {
          if (sp == fix.self) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] += __uint_as_float(r[j]);
          } else {
            const float4* p = reinterpret_cast<const float4*>(
                fix.base + sp * fix.stride + (c / 32) * 1024 + lane * 4);
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              const float4 v = __ldcg(p + j4 * 32);
              acc[4 * j4] += v.x;
              acc[4 * j4 + 1] += v.y;
              acc[4 * j4 + 2] += v.z;
              acc[4 * j4 + 3] += v.w;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(T + lane * kVecLd + vec_slot(lane, j)) =
            make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                        __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
    }
    // next step's inputs go in flight once the accumulator registers are free
    float4 wnx[8];
    uint2 xnx[8];
    float4 bnx = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c + 32 < n_cols && n_base + c + 32 < sh.N) {
      load_inputs(c + 32, wnx, xnx);
      bnx = load_bias(c + 32);
    }
    __syncwarp();
    const int n = n_base + c + c4;
    // interior 32 x 32 block with a bf16 destination (the common case): one
    // pointer, no per-row bounds or destination checks
    const bool full = row_base + 32 <= sh.M && n_base + c + 32 <= sh.N;
    bool done = false;
    if constexpr (EPI == kEpiFwd) {
      if (full && ep.y16 && !ep.y32) {
        __nv_bfloat16* dst =
            ep.y16 + static_cast<size_t>(row_base + ep.y_row_off + sub_r) * ep.ld_y16 + n;
        const size_t step = static_cast<size_t>(4) * ep.ld_y16;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int rl = rr * 4 + sub_r;
          const float4 a =
              *reinterpret_cast<const float4*>(T + rl * kVecLd + vec_slot(rl, c4 / 4));
          __nv_bfloat162 h0 = __floats2bfloat162_rn(act_fwd_t<ACT>(a.x + bias4.x),
                                                    act_fwd_t<ACT>(a.y + bias4.y));
          __nv_bfloat162 h1 = __floats2bfloat162_rn(act_fwd_t<ACT>(a.z + bias4.z),
                                                    act_fwd_t<ACT>(a.w + bias4.w));
          *reinterpret_cast<uint2*>(dst + rr * step) =
              make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
        }
        done = true;
      } else if (full && ep.y32 && !ep.y16) {  // fp32 logits of the output layer
        float* dst = ep.y32 + static_cast<size_t>(row_base + ep.y_row_off + sub_r) * ep.ld_y32 + n;
        const size_t step = static_cast<size_t>(4) * ep.ld_y32;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int rl = rr * 4 + sub_r;
          const float4 a =
              *reinterpret_cast<const float4*>(T + rl * kVecLd + vec_slot(rl, c4 / 4));
          *reinterpret_cast<float4*>(dst + rr * step) =
              make_float4(act_fwd_t<ACT>(a.x + bias4.x), act_fwd_t<ACT>(a.y + bias4.y),
                          act_fwd_t<ACT>(a.z + bias4.z), act_fwd_t<ACT>(a.w + bias4.w));
        }
        done = true;
      }
    } else if constexpr (EPI == kEpiDgrad) {
      if (full) {
        __nv_bfloat16* dst = ep.d16 + static_cast<size_t>(row_base + sub_r) * ep.ld_d16 + n;
        const size_t step = static_cast<size_t>(4) * ep.ld_d16;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int rl = rr * 4 + sub_r;
          const float4 a =
              *reinterpret_cast<const float4*>(T + rl * kVecLd + vec_slot(rl, c4 / 4));
          float v[4] = {a.x, a.y, a.z, a.w};
          if constexpr (kGate) {
            const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xin[rr]);
            const float2 x01 = __bfloat1622float2(xh[0]);
            const float2 x23 = __bfloat1622float2(xh[1]);
            v[0] *= act_grad_t<ACT>(x01.x);
            v[1] *= act_grad_t<ACT>(x01.y);
            v[2] *= act_grad_t<ACT>(x23.x);
            v[3] *= act_grad_t<ACT>(x23.y);
          }
          __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]);
          __nv_bfloat162 h1 = __floats2bfloat162_rn(v[2], v[3]);
          *reinterpret_cast<uint2*>(dst + rr * step) =
              make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
        }
        done = true;
      }
    }
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      if (done) break;
      const int rl = rr * 4 + sub_r;
      const int row = row_base + rl;
      const float4 a = *reinterpret_cast<const float4*>(T + rl * kVecLd + vec_slot(rl, c4 / 4));
      float v[4] = {a.x, a.y, a.z, a.w};
      if (row >= sh.M) continue;
      if (n + 3 < sh.N) {
        if constexpr (EPI == kEpiFwd) {
          v[0] = act_fwd_t<ACT>(v[0] + bias4.x);
          v[1] = act_fwd_t<ACT>(v[1] + bias4.y);
          v[2] = act_fwd_t<ACT>(v[2] + bias4.z);
          v[3] = act_fwd_t<ACT>(v[3] + bias4.w);
          const size_t yr = static_cast<size_t>(row + ep.y_row_off);
          if (ep.y16) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]);
            __nv_bfloat162 h1 = __floats2bfloat162_rn(v[2], v[3]);
            *reinterpret_cast<uint2*>(ep.y16 + yr * ep.ld_y16 + n) =
                make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
          }
          if (ep.y32)
            *reinterpret_cast<float4*>(ep.y32 + yr * ep.ld_y32 + n) =
                make_float4(v[0], v[1], v[2], v[3]);
        } else if constexpr (EPI == kEpiDgrad) {
          if constexpr (kGate) {
            const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xin[rr]);
            const float2 x01 = __bfloat1622float2(xh[0]);
            const float2 x23 = __bfloat1622float2(xh[1]);
            v[0] *= act_grad_t<ACT>(x01.x);
            v[1] *= act_grad_t<ACT>(x01.y);
            v[2] *= act_grad_t<ACT>(x23.x);
            v[3] *= act_grad_t<ACT>(x23.y);
          }
          __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]);
          __nv_bfloat162 h1 = __floats2bfloat162_rn(v[2], v[3]);
          *reinterpret_cast<uint2*>(ep.d16 + static_cast<size_t>(row) * ep.ld_d16 + n) =
              make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
        } else {
          const float4 w = win[rr];
          v[0] = w.x - ep.lr * v[0];
          v[1] = w.y - ep.lr * v[1];
          v[2] = w.z - ep.lr * v[2];
          v[3] = w.w - ep.lr * v[3];
          // the new master is next read one mini-batch later: stream it past L2
          __stcs(reinterpret_cast<float4*>(ep.w_new + static_cast<size_t>(row) * ep.ld_w32 + n),
                 make_float4(v[0], v[1], v[2], v[3]));
          if (ep.w16) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]);
            __nv_bfloat162 h1 = __floats2bfloat162_rn(v[2], v[3]);
            *reinterpret_cast<uint2*>(ep.w16 + static_cast<size_t>(row) * ep.ld_w16 + n) =
                make_uint2(*reinterpret_cast<uint32_t*>(&h0),
                           *reinterpret_cast<uint32_t*>(&h1));
          }
        }
      } else {  // ragged right edge: scalar columns
        for (int i = 0; i < 4 && n + i < sh.N; ++i) {
          float x = v[i];
          const int col = n + i;
          if constexpr (EPI == kEpiFwd) {
            x = act_fwd_t<ACT>(x + (ep.bias ? ep.bias[col] : 0.f));
            const size_t yr = static_cast<size_t>(row + ep.y_row_off);
            if (ep.y16) ep.y16[yr * ep.ld_y16 + col] = __float2bfloat16_rn(x);
            if (ep.y32) ep.y32[yr * ep.ld_y32 + col] = x;
          } else if constexpr (EPI == kEpiDgrad) {
            if constexpr (kGate)
              x *= act_grad_t<ACT>(
                  __bfloat162float(ep.xin[static_cast<size_t>(row) * ep.ld_xin + col]));
            ep.d16[static_cast<size_t>(row) * ep.ld_d16 + col] = __float2bfloat16_rn(x);
          } else {
            x = ep.w_cur[static_cast<size_t>(row) * ep.ld_w32 + col] - ep.lr * x;
            ep.w_new[static_cast<size_t>(row) * ep.ld_w32 + col] = x;
            if (ep.w16) ep.w16[static_cast<size_t>(row) * ep.ld_w16 + col] = __float2bfloat16_rn(x);
          }
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      win[rr] = wnx[rr];
      xin[rr] = xnx[rr];
    }
    bias4 = bnx;
  }
}

// ---------------------------------------------------------------- split-K
// Split-K for forward GEMMs whose tile count cannot fill the GPU (a
// 128..256-row micro-batch forward of a 4096-wide layer has 32-64 tiles of
// 128 x 128 for 148 SMs).  The S CTAs of one output tile form a thread-block
// cluster (1, 1, S); each accumulates one K chunk in its TMEM.  After the
// mainloop every CTA parks its fp32 partial in its own (now idle) operand
// ring, the cluster synchronises, and CTA j finishes column block j of the
// tile: it reads the S partials of its columns over DSMEM in split order,
// sums them (deterministic) and runs the fused epilogue.  No global
// workspace, no atomics, and the finishing work is spread over the S CTAs.
constexpr int kMaxSplits = 4;

template <int BN>
struct SplitSmem {
  static constexpr int kLd = BN + 4;  // +16 B per row: float4 row accesses are conflict-free
  static constexpr int kBytes = 128 * kLd * 4;
};

// TMEM accumulator row (this thread's row) -> own smem partial.
template <int BN>
__device__ __forceinline__ void splitk_park(float* part, int r_local, uint32_t t_row) {
  float* dst = part + r_local * SplitSmem<BN>::kLd;
#pragma unroll 1
  for (int c = 0; c < BN; c += 16) {
    uint32_t r[16];
    ptx::tmem_ld16(t_row + c, r);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 4; ++i)
      reinterpret_cast<float4*>(dst + c)[i] =
          make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                      __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
  }
}

// Column block `rank` of the tile: sum the S partials of row r_local over
// DSMEM (split order) and run the epilogue.
template <int EPI, int ACT, int BN>
__device__ __forceinline__ void splitk_reduce(const EpiParams& ep, const GemmShape& sh,
                                              const float* part, int splits, int rank,
                                              int row, int r_local, int n0) {
  const int w = BN / splits;  // multiple of 16 (host: splits in {2, 4}, BN >= 128)
  const int c0 = rank * w;
  uint32_t src[kMaxSplits];
#pragma unroll
  for (int j = 0; j < kMaxSplits; ++j)
    src[j] = j < splits ? ptx::map_to_rank(part + r_local * SplitSmem<BN>::kLd, j) : 0u;
#pragma unroll 1
  for (int c = c0; c < c0 + w; c += 16) {
    const int n = n0 + c;
    if (n >= sh.N) break;
    float4 q[kMaxSplits][4];
#pragma unroll
    for (int j = 0; j < kMaxSplits; ++j)
      if (j < splits)
#pragma unroll
        for (int i = 0; i < 4; ++i) q[j][i] = ptx::ld_dsmem_f4(src[j] + (c + 4 * i) * 4);
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxSplits; ++j)
      if (j < splits)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          v[4 * i] += q[j][i].x;
          v[4 * i + 1] += q[j][i].y;
          v[4 * i + 2] += q[j][i].z;
          v[4 * i + 3] += q[j][i].w;
        }
    if (row < sh.M) {
      const int valid = sh.N - n < 16 ? sh.N - n : 16;
      epilogue_chunk<EPI, ACT>(ep, sh, row, n, valid, v);
    }
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(128, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmap_a,
                      const __grid_constant__ CUtensorMap tmap_b, GemmShape sh,
                      EpiParams ep, const __grid_constant__ EpiMaps maps) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  // 32-wide tiles with an MN-major B: one 64-byte-swizzled box per k-block
  // (plain 2-D maps only; the conv im2col B path is 64 columns wide)
  if constexpr (B_MN && BN == 32)
    if (sh.conv != 0) __trap();
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (128B swizzle atoms) by offsetting the shared array
  // itself, so every derived pointer stays in the shared address space.
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* accum_bar = empty_bar + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_bar + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * Cfg::kBM;
  const int n0 = blockIdx.x * BN;
  const int split = blockIdx.z;
  const int kb_all = (sh.K + Cfg::kBK - 1) / Cfg::kBK;
  const int kb_lo = sh.splits > 1 ? split * sh.kb_per_split : 0;
  const int kb_hi = sh.splits > 1 ? min(kb_all, kb_lo + sh.kb_per_split) : kb_all;
  const int num_kb = kb_hi - kb_lo;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmap_a);
    ptx::tma_prefetch_desc(&tmap_b);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full_bar[i], 1);
      ptx::mbar_init(&empty_bar[i], 1);
    }
    ptx::mbar_init(accum_bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: everything above overlaps the previous
  // kernel of the stream; its outputs are read only after this
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % S;
      if (kb >= S) ptx::mbar_wait(&empty_bar[s], ((kb / S) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&full_bar[s], Cfg::kStageBytes);
      const int k0 = (kb_lo + kb) * Cfg::kBK;
      uint8_t* a_dst = sA + s * Cfg::kABytes;
      uint8_t* b_dst = sB + s * Cfg::kBBytes;
      if constexpr (!A_MN) {
        ptx::tma_load_2d(a_dst, &tmap_a, &full_bar[s], k0 + sh.a_k_off,
                         m0 + sh.a_mn_off);
      } else {
#pragma unroll
        for (int h = 0; h < Cfg::kBM / 64; ++h)
          ptx::tma_load_2d(a_dst + h * 8192, &tmap_a, &full_bar[s],
                           m0 + h * 64 + sh.a_mn_off, k0 + sh.a_k_off);
      }
      if constexpr (!B_MN) {
        ptx::tma_load_2d(b_dst, &tmap_b, &full_bar[s], k0 + sh.b_k_off,
                         n0 + sh.b_mn_off);
      } else if (sh.conv == 2) {
        // implicit-GEMM conv wgrad: B = im2col(x), 64 pixels x 64 channels
        // of tap n / C per 64 output columns
        const int hw = sh.conv_h * sh.conv_w;
        const int p = k0 + sh.b_k_off;
        const int pn = p / hw, ph = (p - pn * hw) / sh.conv_w, pw = p - pn * hw - ph * sh.conv_w;
#pragma unroll
        for (int h = 0; h < BN / 64; ++h) {
          const int n = n0 + h * 64;
          const int tap = n / sh.conv_c, c0 = n - tap * sh.conv_c;
          ptx::tma_load_im2col(b_dst + h * 8192, &tmap_b, &full_bar[s], c0, pw - 1, ph - 1, pn,
                               tap % 3, tap / 3);
        }
      } else if constexpr (BN == 32) {
        ptx::tma_load_2d(b_dst, &tmap_b, &full_bar[s], n0 + sh.b_mn_off, k0 + sh.b_k_off);
      } else {
#pragma unroll
        for (int h = 0; h < BN / 64; ++h)
          ptx::tma_load_2d(b_dst + h * 8192, &tmap_b, &full_bar[s],
                           n0 + h * 64 + sh.b_mn_off, k0 + sh.b_k_off);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, BN, A_MN, B_MN);
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % S;
      ptx::mbar_wait(&full_bar[s], (kb / S) & 1);
      ptx::tc_fence_after();
      const uint32_t a_addr = ptx::smem_u32(sA + s * Cfg::kABytes);
      const uint32_t b_addr = ptx::smem_u32(sB + s * Cfg::kBBytes);
#pragma unroll
      for (int kk = 0; kk < Cfg::kBK / 16; ++kk) {
        // K-major: step 16 elements = 32 B inside the swizzle row.
        // MN-major: step 16 K-rows = 16 * 128 B; MN blocks of 64 are 8 KB apart.
        const uint64_t a_desc =
            A_MN ? ptx::smem_desc_sw128(a_addr + kk * 2048, 8192, 1024)
                 : ptx::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
        const uint64_t b_desc =
            B_MN ? (BN == 32 ? ptx::smem_desc_sw64(b_addr + kk * 1024, 4096, 512)
                             : ptx::smem_desc_sw128(b_addr + kk * 2048, 8192, 1024))
                 : ptx::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
        ptx::mma_bf16(tmem_base, a_desc, b_desc, idesc, (kb | kk) != 0);
      }
      ptx::mma_commit(&empty_bar[s]);
    }
    ptx::mma_commit(accum_bar);
  }
  __syncwarp();

  // ---------------- epilogue (all 4 warps)
  ptx::mbar_wait(accum_bar, 0);
  ptx::tc_fence_after();

  const uint32_t t_row = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);

  if (EPI == kEpiFwd || EPI == kEpiDgrad) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && split == 0 && threadIdx.x == 0 && ep.tag_src &&
        ep.tag_dst)
      write_tags(ep);
  }
  // the operand ring is idle now: reuse it for the per-warp transpose blocks
  float* T = reinterpret_cast<float*>(sA) + warp * 32 * kVecLd;
  if (ep.partial_slab) {
    // split-K into partial slabs: this split's own fp32 slab, plain store
    EpiParams epp = ep;
    epp.y32 = ep.y32 + static_cast<size_t>(split) * ep.partial_slab;
    if constexpr (EPI == kEpiFwd)
      epilogue_warp_vec<EPI, kLinear>(epp, sh, m0 + warp * 32, n0, BN, t_row, T);
  } else if (ep.dbg_skip & 1) {
  } else if (EPI == kEpiFwd && sh.splits > 1) {
    static_assert(SplitSmem<BN>::kBytes <= S * Cfg::kStageBytes, "partial must fit the ring");
    float* part = reinterpret_cast<float*>(sA);
    const int r_local = warp * 32 + lane;
    splitk_park<BN>(part, r_local, t_row);
    ptx::cluster_sync();  // every partial of the tile is parked
    if constexpr (EPI == kEpiFwd)
      with_act<EPI>(ep, [&](auto A) {
        splitk_reduce<EPI, decltype(A)::value, BN>(ep, sh, part, sh.splits,
                                                   static_cast<int>(ptx::cluster_ctarank()),
                                                   m0 + r_local, r_local, n0);
      });
    ptx::cluster_sync();  // peers may still be reading this CTA's partial
  } else if (ep.rowwise == 2) {
    with_act<EPI>(ep, [&](auto A) {
      epilogue_warp_vec<EPI, decltype(A)::value>(ep, sh, m0 + warp * 32, n0, BN, t_row, T);
    });
  } else if (ep.rowwise) {
    with_act<EPI>(ep, [&](auto A) {
      epilogue_warp_rows<EPI, decltype(A)::value>(ep, sh, m0 + warp * 32, n0, BN, t_row);
    });
  } else {
    with_act<EPI>(ep, [&](auto A) {
      epilogue_warp_tile<EPI, decltype(A)::value>(ep, sh, m0 + warp * 32, n0, BN, t_row, T);
    });
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// TMA epilogue of wgrad + SGD (pair kernel): one warp updates its 32 rows x
// n_cols of the tile in 32 x 32 chunks.  The fp32 master chunk arrives by
// TMA (128-byte swizzle) one chunk ahead; each thread updates its own row in
// place in shared memory (the swizzle makes the row-per-thread 16-byte
// accesses conflict-free), writes the bf16 copy into a 32 x 64 bf16 tile
// (128-byte swizzle) that two consecutive chunks fill, and one lane stores
// the fp32 chunk, and the bf16 tile after every second chunk, with TMA: three
// bulk stores per 64 columns instead of four (the store count, not only the
// bytes, costs epilogue time).  Loads and stores are bulk and asynchronous:
// the update never waits for a global store, and out-of-range rows / columns
// are clipped by the tensor maps.  n_cols is a multiple of 64.
struct SgdTmaState {
  int g = 0;                  // chunks processed by this warp so far
  uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

__device__ __forceinline__ void sgd_tma_load(const EpiMaps& maps, uint8_t* buf32, uint64_t* bar,
                                             int col, int row) {
  ptx::mbar_arrive_expect_tx(bar, 4096);
  ptx::tma_load_2d(buf32, &maps.w_cur, bar, col, row);
}

__device__ __forceinline__ void epilogue_warp_tma_sgd(const EpiParams& ep, const EpiMaps& maps,
                                                      int row_base, int n_base, int n_cols,
                                                      uint32_t t_row, uint8_t* wbuf,
                                                      uint64_t* bars, SgdTmaState& st,
                                                      bool first_tile, int next_row,
                                                      int next_col) {
  const int lane = threadIdx.x % 32;
  uint8_t* b32[2] = {wbuf, wbuf + 4096};
  uint8_t* b16 = wbuf + 8192;  // 32 rows x 128 B: the bf16 copy of two chunks
  // timing experiments: 2 skips the master loads, 4 all stores, 8 the bf16 stores
  const bool skip_ld = ep.dbg_skip & 2, skip_st = ep.dbg_skip & 4;
  if (first_tile && lane == 0 && !skip_ld)
    sgd_tma_load(maps, b32[st.g & 1], &bars[st.g & 1], n_base, row_base);
#pragma unroll 1
  for (int c = 0; c < n_cols; c += 32) {
    const int b = st.g & 1;
    if (lane == 0) {
      // buffer b^1 was last stored from two chunks ago; once that store has
      // read it, prefetch the next chunk (this tile's, or the next tile's
      // first) into it
      ptx::bulk_wait_group_read<0>();
      if (skip_ld) {
      } else if (c + 32 < n_cols)
        sgd_tma_load(maps, b32[b ^ 1], &bars[b ^ 1], n_base + c + 32, row_base);
      else if (next_row >= 0)
        sgd_tma_load(maps, b32[b ^ 1], &bars[b ^ 1], next_col, next_row);
    }
    uint32_t r[32];
    ptx::tmem_ld32(t_row + c, r);
    if (!skip_ld) {
      ptx::mbar_wait(&bars[b], st.phase[b]);
      st.phase[b] ^= 1;
    }
    ptx::tmem_ld_wait();
    uint8_t* row32 = b32[b] + lane * 128;
    uint8_t* row16 = b16 + lane * 128;
    const int half = (c >> 5) & 1;  // which 64-byte half of the bf16 row
    // the bf16 tile was stored at the end of the previous chunk: every lane
    // waits for lane 0's bulk_wait_group_read above before refilling it
    if (half == 0) __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      uint32_t hv[4];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        float4* p = reinterpret_cast<float4*>(row32 + (((j + t) ^ (lane & 7)) << 4));
        float4 w = *p;
        w.x -= ep.lr * __uint_as_float(r[4 * (j + t)]);
        w.y -= ep.lr * __uint_as_float(r[4 * (j + t) + 1]);
        w.z -= ep.lr * __uint_as_float(r[4 * (j + t) + 2]);
        w.w -= ep.lr * __uint_as_float(r[4 * (j + t) + 3]);
        *p = w;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(w.x, w.y);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(w.z, w.w);
        hv[2 * t] = *reinterpret_cast<uint32_t*>(&h0);
        hv[2 * t + 1] = *reinterpret_cast<uint32_t*>(&h1);
      }
      const int unit = half * 4 + j / 2;  // 16-byte unit of the 128-byte bf16 row
      *reinterpret_cast<uint4*>(row16 + ((unit ^ (lane & 7)) << 4)) =
          make_uint4(hv[0], hv[1], hv[2], hv[3]);
    }
    ptx::fence_proxy_async();  // generic smem writes -> visible to the TMA store
    __syncwarp();
    if (lane == 0 && !skip_st) {
      ptx::tma_store_2d(&maps.w_new, b32[b], n_base + c, row_base);
      if (half == 1 && ep.has_w16 && !(ep.dbg_skip & 8))
        ptx::tma_store_2d(&maps.w16, b16, n_base + c - 32, row_base);
      ptx::bulk_commit_group();
    }
    ++st.g;
  }
}

// Split fp32 masters.  A version's fp32 master is stored as its bf16 GEMM
// operand hi (already needed by the forwards and dgrads that read the
// version) plus a signed 16-bit residual lo: bits(master) = bits(hi) << 16 +
// lo, exact.  hi is the master rounded to nearest in the bit pattern with
// ties away from zero ((bits + 0x8000) >> 16; differs from RN-even only on
// exact ties), so the residual always fits in 16 bits.  Per parameter the
// update reads 4 bytes (hi, lo of the current version) and writes 4 (hi, lo
// of the new one) instead of 4 + 6 with an fp32 master and a bf16 copy: a
// third fewer bytes stored, which the step is sensitive to.
__device__ __forceinline__ float join_master(uint32_t hi16, uint32_t lo16) {
  return __int_as_float(static_cast<int>(hi16 << 16) + static_cast<int>(static_cast<int16_t>(lo16)));
}
__device__ __forceinline__ void split_master(float w, uint32_t& hi16, uint32_t& lo16) {
  const uint32_t b = __float_as_uint(w);
  hi16 = (b + 0x8000u) >> 16;
  lo16 = (b - (hi16 << 16)) & 0xFFFFu;
}

// TMA epilogue of wgrad + SGD with split masters: one warp, 32 rows x n_cols,
// 32 x 32 chunks.  hi and lo of the current version arrive by TMA (64-byte
// swizzle, 2 KB each) into one of kBufs 4 KB buffers, kBufs - 2 chunks ahead
// (across the tile boundary into the warp's part of the next tile); each
// thread rebuilds its row's fp32 masters, applies the update and writes the
// new hi / lo back in place; one lane stores both with TMA.  The load of
// chunk c + kBufs - 2 reuses the buffer of chunk c - 2, whose store has read
// it once at most one bulk group (chunk c - 1's) is still reading.  The
// per-warp update is bound by HBM latency x chunks in flight, so the depth
// sets its rate.
template <int kBufs>
__device__ __forceinline__ void epilogue_warp_tma_sgd_split(
    const EpiParams& ep, const EpiMaps& maps, int row_base, int n_base, int n_cols,
    uint32_t t_row, uint8_t* wbuf, uint64_t* bars, SgdTmaState& st, bool first_tile,
    int next_row, int next_col) {
  static_assert(kBufs >= 3 && kBufs <= 6, "split SGD epilogue: 3..6 buffers");
  constexpr int kAhead = kBufs - 2;
  const int lane = threadIdx.x % 32;
  const bool skip_ld = ep.dbg_skip & 2, skip_st = ep.dbg_skip & 4;  // timing experiments
  auto buf = [&](int g) { return wbuf + (g % kBufs) * 4096; };
  auto load = [&](int g, int col, int row) {
    uint64_t* bar = &bars[g % kBufs];
    ptx::mbar_arrive_expect_tx(bar, 4096);
    ptx::tma_load_2d(buf(g), &maps.w_cur, bar, col, row);
    ptx::tma_load_2d(buf(g) + 2048, &maps.w_new, bar, col, row);
  };
  // chunk `a` chunks after chunk c of this tile: its coordinates, or false
  // past the next tile
  auto ahead = [&](int c, int a, int* col, int* row) {
    const int cc = c + 32 * a;
    if (cc < n_cols) {
      *col = n_base + cc;
      *row = row_base;
      return true;
    }
    if (next_row < 0 || cc - n_cols >= n_cols) return false;
    *col = next_col + (cc - n_cols);
    *row = next_row;
    return true;
  };
  if (first_tile && lane == 0 && !skip_ld)
    for (int a = 0; a < kAhead; ++a) {
      int col, row;
      if (ahead(0, a, &col, &row)) load(st.g + a, col, row);
    }
#pragma unroll 1
  for (int c = 0; c < n_cols; c += 32) {
    const int g = st.g;
    const int b = g % kBufs;
    if (lane == 0) {
      ptx::bulk_wait_group_read<1>();  // chunk g-2's store has read buffer (g+kAhead) % kBufs
      int col, row;
      if (!skip_ld && ahead(c, kAhead, &col, &row)) load(g + kAhead, col, row);
#if PB_SGD_L2PF
      // the same chunk of the warp's next tile into L2 a tile ahead: its TMA
      // load then waits on L2, not HBM, latency (no shared memory held)
      if (!skip_ld && next_row >= 0) {
        ptx::tma_prefetch_2d(&maps.w_cur, next_col + c, next_row);
        ptx::tma_prefetch_2d(&maps.w_new, next_col + c, next_row);
      }
#endif
    }
    uint32_t r[32];
    ptx::tmem_ld32(t_row + c, r);
    if (!skip_ld) {
      ptx::mbar_wait(&bars[b], st.phase[b]);
      st.phase[b] ^= 1;
    }
    ptx::tmem_ld_wait();
    uint8_t* hrow = buf(g) + lane * 64;
    uint8_t* lrow = hrow + 2048;
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // 16-byte units: 8 columns each
      const int off = (u ^ ((lane >> 1) & 3)) << 4;
      uint4 h = *reinterpret_cast<const uint4*>(hrow + off);
      uint4 l = *reinterpret_cast<const uint4*>(lrow + off);
      uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t h0, l0, h1, l1;
        const float w0 = join_master(hw[q] & 0xFFFFu, lw[q] & 0xFFFFu) -
                         ep.lr * __uint_as_float(r[8 * u + 2 * q]);
        const float w1 = join_master(hw[q] >> 16, lw[q] >> 16) -
                         ep.lr * __uint_as_float(r[8 * u + 2 * q + 1]);
        split_master(w0, h0, l0);
        split_master(w1, h1, l1);
        hw[q] = h0 | (h1 << 16);
        lw[q] = l0 | (l1 << 16);
      }
      *reinterpret_cast<uint4*>(hrow + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(lrow + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    ptx::fence_proxy_async();  // generic smem writes -> visible to the TMA store
    __syncwarp();
    if (lane == 0 && !skip_st) {
      ptx::tma_store_2d(&maps.w16, buf(g), n_base + c, row_base);
      ptx::tma_store_2d(&maps.lo_new, buf(g) + 2048, n_base + c, row_base);
      ptx::bulk_commit_group();
    }
    ++st.g;
  }
}

// ===========================================================================
// Persistent CTA-pair kernel (cta_group::2).
//
// A cluster of 2 CTAs on neighbouring SMs computes 256 x BN output tiles:
// CTA r holds A rows [128r, 128r+128) and B rows [r*BN/2, (r+1)*BN/2) of the
// tile in its own smem; one tcgen05.mma.cta_group::2 (M=256) issued by the
// leader reads both halves and accumulates into both CTAs' TMEM (CTA r gets
// output rows [128r, +128)).  Per SM this halves the B-operand bytes per FLOP
// versus a 128 x BN single-CTA tile.  The pair walks a static tile schedule;
// TMEM holds two accumulators so the epilogue of tile i (4 warps) overlaps
// the mainloop of tile i+1.
//
// Warps: 0 TMA producer (both CTAs), 1 MMA issuer (leader) + TMEM owner,
//        2..5 epilogue (TMEM lanes 32*(warp%4) .. +32).
// BN = 512: two N=256 MMAs per k-block share the A operand (256 x 512 tile,
// 48 B of operands per 2 x 4 MFLOP per CTA instead of 32 B per 4 MFLOP: the
// mainloop's per-SM feed, which is latency-bound, covers the
// MMA rate); the two accumulators fill TMEM, so tiles are not double-buffered.
template <int BN, int EPI>
struct Gemm2Cfg {
  static constexpr int kBK = 64;
  static constexpr int kMmaN = BN > 256 ? 256 : BN;     // N of one tcgen05.mma
  static constexpr int kSub = BN / kMmaN;               // MMAs per k-block
  static constexpr int kAccBufs = BN > 256 ? 1 : 2;     // TMEM accumulator buffers
  static constexpr int kAHalf = 128 * kBK * 2;         // this CTA's A rows
  static constexpr int kBSub = (kMmaN / 2) * kBK * 2;  // this CTA's B rows of one MMA
  static constexpr int kBHalf = kSub * kBSub;          // this CTA's B rows
  static constexpr int kStageBytes = kAHalf + kBHalf;
  // wgrad tiles are short in K (one mini-batch): a shallower ring leaves room
  // for the TMA epilogue's master-tile buffers (PB_WGRAD_STAGES)
  static constexpr int kStages =
      EPI == kEpiWgradSgd ? PB_WGRAD_STAGES : (BN > 256 ? 4 : (BN >= 256 ? 6 : 8));
  static constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter
  static constexpr int kThreads = 64 + 32 * kEpiWarps;
  // per epilogue warp: staging block (vector epilogue) or, for SGD, the TMA
  // epilogue's buffers: split masters kSgdBufs x 4 KB (hi + lo of a 32x32
  // chunk), fp32 masters 2 x (fp32 32x32 tile 4 KB + bf16 32x32 tile 2 KB)
  static constexpr int kSgdBufs = PB_SGD_BUFS;
  static constexpr int kSgdWarpBytes =
      kSgdBufs * 4096 > 2 * (4096 + 2048) ? kSgdBufs * 4096 : 2 * (4096 + 2048);
  static constexpr int kEpiBytes = EPI == kEpiWgradSgd ? kEpiWarps * kSgdWarpBytes
                                                       : kEpiWarps * 32 * kVecLd * 4;
  static constexpr int kBarOff = kStages * kStageBytes + kEpiBytes;
  static constexpr int kSmem = kBarOff + 512 + 1024;
  static constexpr uint32_t kTmemCols = kAccBufs * BN;  // double-buffered if it fits
  static_assert(kSmem <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

template <class Cfg>
__device__ __forceinline__ void conv_loads_b(const GemmShape& sh, const CUtensorMap* tb,
                                             uint32_t fb, uint8_t* b_dst, int k0, int tap, int c0,
                                             int n_tile, uint32_t rank);

// Operand loads of one k-block of an implicit-GEMM 3x3 convolution (pad 1,
// stride 1, NHWC; GemmShape::conv).  K is tap-major: k = tap * C + channel,
// tap = 3 * r + s, so a 64-wide k-block is one tap and 64 channels.
// Forward / dgrad: A (128 output pixels x 64 channels) comes straight from
// the activation by an im2col TMA load -- the patch matrix is never built.
template <class Cfg>
__device__ __forceinline__ void conv_loads_fd(const GemmShape& sh, const CUtensorMap* ta,
                                              const CUtensorMap* tb, uint32_t fb, uint8_t* a_dst,
                                              uint8_t* b_dst, int k0, int n_tile, uint32_t rank,
                                              int px_n, int px_h, int px_w) {
  // dgrad: dX[h,w] = sum_rs dz[h+1-r, w+1-s] W[r,s]; the k-block's tap t
  // reads dz at window offset t and pairs it with the weights of tap 8 - t
  const int tap = k0 / sh.conv_c, c0 = k0 - tap * sh.conv_c;
  ptx::tma_load_im2col_pair(a_dst, ta, fb, c0, px_w - 1, px_h - 1, px_n, tap % 3, tap / 3);
  conv_loads_b<Cfg>(sh, tb, fb, b_dst, k0, tap, c0, n_tile, rank);
}

// The B operand of k-block (tap, channel chunk c0) of a conv forward (W
// [Cout, 9C], K-major) or dgrad (W viewed [Cout][9][Cin], flipped tap,
// MN-major).
template <class Cfg>
__device__ __forceinline__ void conv_loads_b(const GemmShape& sh, const CUtensorMap* tb,
                                             uint32_t fb, uint8_t* b_dst, int k0, int tap, int c0,
                                             int n_tile, uint32_t rank) {
#pragma unroll
  for (int j = 0; j < Cfg::kSub; ++j) {
    const int nbj = n_tile + j * Cfg::kMmaN + static_cast<int>(rank) * (Cfg::kMmaN / 2);
    uint8_t* bj = b_dst + j * Cfg::kBSub;
    if (sh.conv == 1) {
      ptx::tma_load_2d_pair(bj, tb, fb, k0, nbj);  // W [Cout, 9C], K-major
    } else {
      // W viewed [Cout][9][Cin]: 64 output channels (K) x 64 input channels
      // (N) of the flipped tap, MN-major; 64-wide MMAs: 32 input channels per
      // CTA, one 64-byte-swizzled box
      if constexpr (Cfg::kMmaN == 64) {
        ptx::tma_load_3d_pair(bj, tb, fb, nbj, 8 - tap, c0);
      } else {
#pragma unroll
        for (int h = 0; h < Cfg::kMmaN / 128; ++h)
          ptx::tma_load_3d_pair(bj + h * 8192, tb, fb, nbj + h * 64, 8 - tap, c0);
      }
    }
  }
}

// 64 pixels (K, from k0 + k_off) x 64 channels of tap mn / C of an im2col
// operand, MN-major (conv wgrad).  Columns past the GEMM extent `ext` load a
// valid box (tap 0) whose products land outside the stored output.
template <class Cfg>
__device__ __forceinline__ void conv_im2col_mn(const GemmShape& sh, const CUtensorMap* map,
                                               uint32_t fb, uint8_t* dst, int k0, int mn, int ext,
                                               int k_off) {
  const int hw = sh.conv_h * sh.conv_w;
  const int p = k0 + k_off;
  const int pn = p / hw, ph = (p - pn * hw) / sh.conv_w, pw = p - pn * hw - ph * sh.conv_w;
  if (mn >= ext) mn = 0;
  const int tap = mn / sh.conv_c, c0 = mn - tap * sh.conv_c;
  ptx::tma_load_im2col_pair(dst, map, fb, c0, pw - 1, ph - 1, pn, tap % 3, tap / 3);
}

// wgrad: B = im2col(x), 64 pixels (K) x 64 channels of tap n / C (N) for
// every 64 output columns, MN-major.
template <class Cfg>
__device__ __forceinline__ void conv_wgrad_b(const GemmShape& sh, const CUtensorMap* tb,
                                             uint32_t fb, uint8_t* bj, int k0, int nbj) {
  const int hw = sh.conv_h * sh.conv_w;
  const int p = k0 + sh.b_k_off;
  const int pn = p / hw, ph = (p - pn * hw) / sh.conv_w, pw = p - pn * hw - ph * sh.conv_w;
#pragma unroll
  for (int h = 0; h < Cfg::kMmaN / 128; ++h) {
    const int n = nbj + h * 64;
    const int tap = n / sh.conv_c, c0 = n - tap * sh.conv_c;
    ptx::tma_load_im2col_pair(bj + h * 8192, tb, fb, c0, pw - 1, ph - 1, pn, tap % 3, tap / 3);
  }
}

// kExt: the launch may use split-K (partial slabs / the fixup) or halo conv
// tiles; without it those paths compile out (the plain GEMMs keep their lean
// code: the extensions cost the 8-stage step ~1.7%, measured).
template <int BN, bool A_MN, bool B_MN, int EPI, bool kExt>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Gemm2Cfg<BN, EPI>::kThreads, 1)
    gemm_bf16_tcgen05_pair(const __grid_constant__ CUtensorMap tmap_a,
                           const __grid_constant__ CUtensorMap tmap_b, GemmShape sh,
                           EpiParams ep, const __grid_constant__ EpiMaps maps) {
  using Cfg = Gemm2Cfg<BN, EPI>;
  constexpr int S = Cfg::kStages;
  // 64-wide MMAs with an MN-major B exist only for the conv dgrad's 64-byte
  // swizzled weight boxes (the other MN-major loads are 64 columns wide)
  if constexpr (B_MN && Cfg::kMmaN == 64)
    if (sh.conv != 3) __trap();
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (128B swizzle atoms) by offsetting the shared array
  // itself, so every derived pointer stays in the shared address space.
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kAHalf;
  uint8_t* epi_base = smem + S * Cfg::kStageBytes;  // 1024-aligned
  float* epi_smem = reinterpret_cast<float*>(epi_base);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;  // [2] (leader's are used)
  uint64_t* sgd_bar = tempty_bar + 2;    // [kSgdBufs per epilogue warp] (TMA SGD epilogue)
  // (own 16-byte slot, apart from the barriers thread 0 initialises)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::kBarOff + 496);
  volatile int* fix_last = reinterpret_cast<volatile int*>(smem + Cfg::kBarOff + 500);
  static_assert(sizeof(uint64_t) * (2 * Cfg::kStages + 4 +
                                    (EPI == kEpiWgradSgd ? Cfg::kSgdBufs * Cfg::kEpiWarps : 4)) <=
                    496,
                "barrier region overlaps the TMEM address slot");

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x / 2;
  const int num_pairs = gridDim.x / 2;
  // halo conv tiles (GemmShape::halo_tw): strips of tw pixels, two per pair
  // tile; the operand ring becomes two patch buffers + S_h B-only stages
  const bool halo =
      kExt && EPI != kEpiWgradSgd && (sh.conv == 1 || sh.conv == 3) && sh.halo_tw > 0;
  const int tw = sh.halo_tw;
  const int n_strips = halo ? sh.M / tw : 0;
  constexpr int kPatchBuf = 48 * 1024;  // {64 ch, <= 128 px, 3 rows} + over-read rows
  constexpr int S_h = (S * Cfg::kStageBytes - 2 * kPatchBuf) / Cfg::kBHalf < S
                          ? (S * Cfg::kStageBytes - 2 * kPatchBuf) / Cfg::kBHalf
                          : S;
  uint8_t* patch0 = smem;
  uint8_t* sBh = smem + 2 * kPatchBuf;
  uint64_t* pbar = tempty_bar + 2;  // [0..1] patch full, [2..3] patch empty (not SGD)
  const int tiles_m = halo ? (n_strips + 1) / 2 : (sh.M + 255) / 256;
  const int tiles_n = (sh.N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int kb_all = (sh.K + Cfg::kBK - 1) / Cfg::kBK;
  // split-K into partial slabs (conv wgrad) or with the in-kernel fixup
  // (forward): unit = (tile, split)
  // (only forward-epilogue launches split: the other kernels fold S_k = 1)
  const bool splitk =
      kExt && EPI == kEpiFwd && (ep.partial_slab || ep.fix_cnt) && sh.splits > 1;
  const int S_k = splitk ? sh.splits : 1;
  const int kbps = splitk ? sh.kb_per_split : kb_all;
  const int num_units = num_tiles * S_k;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmap_a);
    ptx::tma_prefetch_desc(&tmap_b);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full_bar[i], 1);
      ptx::mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull_bar[i], 1);
      ptx::mbar_init(&tempty_bar[i], 2);  // one arrival per CTA of the pair
    }
    if (halo)
      for (int i = 0; i < 4; ++i) ptx::mbar_init(&pbar[i], 1);
    if constexpr (EPI == kEpiWgradSgd)
      if (ep.rowwise == 3) {
        for (int i = 0; i < Cfg::kSgdBufs * Cfg::kEpiWarps; ++i) ptx::mbar_init(&sgd_bar[i], 1);
        ptx::tma_prefetch_desc(&maps.w_cur);
        ptx::tma_prefetch_desc(&maps.w_new);
        if (ep.has_w16) ptx::tma_prefetch_desc(&maps.w16);
        if (ep.split_master) ptx::tma_prefetch_desc(&maps.lo_new);
      }
    ptx::fence_mbar_init();
  }
  __syncthreads();  // barrier init (thread 0) before the pair's TMEM allocation
  if (warp == 1) ptx::tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch (see the single-CTA kernel)
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs), completion on the leader's barrier
      int it = 0, pit = 0;
      for (int u = pair; u < num_units; u += num_pairs) {
        const int tile = u / S_k, split = u % S_k;
        const int tm = tile / tiles_n, tn = tile % tiles_n;
        if (halo) {
          // this CTA's strip (the second strip of an odd last tile loads
          // strip 0: its rows are never stored)
          const int strip = 2 * tm + static_cast<int>(rank);
          const int hw = sh.conv_h * sh.conv_w;
          const int p = (strip < n_strips ? strip : 0) * tw + sh.a_mn_off;
          const int img = p / hw, hh = (p - img * hw) / sh.conv_w;
          const int w0 = p - img * hw - hh * sh.conv_w;
          const uint32_t patch_bytes = 128u * static_cast<uint32_t>(tw + 2) * 3u;
          for (int c0 = 0; c0 < sh.conv_c; c0 += 64) {
            const int pb = pit & 1;
            if (pit >= 2) ptx::mbar_wait(&pbar[2 + pb], ((pit >> 1) - 1) & 1);
            if (rank == 0) ptx::mbar_arrive_expect_tx(&pbar[pb], 2 * patch_bytes);
            ptx::tma_load_4d_pair(patch0 + pb * kPatchBuf, &tmap_a, ptx::map_to_rank(&pbar[pb], 0),
                                  c0, w0 - 1, hh - 1, img);
            ++pit;
            for (int tap = 0; tap < 9; ++tap, ++it) {
              const int s = it % S_h;
              if (it >= S_h) ptx::mbar_wait(&empty_bar[s], ((it / S_h) - 1) & 1);
              const uint32_t fb = ptx::map_to_rank(&full_bar[s], 0);
              if (rank == 0) ptx::mbar_arrive_expect_tx(&full_bar[s], 2 * Cfg::kBHalf);
              conv_loads_b<Cfg>(sh, &tmap_b, fb, sBh + s * Cfg::kBHalf, tap * sh.conv_c + c0, tap,
                                c0, tn * BN, rank);
            }
          }
          continue;
        }
        const int m0 = tm * 256 + static_cast<int>(rank) * 128;
        const int kb_lo = split * kbps, kb_hi = min(kb_all, kb_lo + kbps);
        // implicit-GEMM conv, A = im2col: this CTA's first output pixel
        int px_n = 0, px_h = 0, px_w = 0;
        if (sh.conv == 1 || sh.conv == 3) {
          const int hw = sh.conv_h * sh.conv_w;
          const int p = m0 + sh.a_mn_off;
          px_n = p / hw;
          px_h = (p - px_n * hw) / sh.conv_w;
          px_w = p - px_n * hw - px_h * sh.conv_w;
        }
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
          const int s = it % S;
          if (it >= S) ptx::mbar_wait(&empty_bar[s], ((it / S) - 1) & 1);
          const uint32_t fb = ptx::map_to_rank(&full_bar[s], 0);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full_bar[s], 2 * Cfg::kStageBytes);
          const int k0 = kb * Cfg::kBK;
          uint8_t* a_dst = sA + s * Cfg::kAHalf;
          uint8_t* b_dst = sB + s * Cfg::kBHalf;
          if (sh.conv == 1 || sh.conv == 3) {
            conv_loads_fd<Cfg>(sh, &tmap_a, &tmap_b, fb, a_dst, b_dst, k0, tn * BN, rank, px_n,
                               px_h, px_w);
            continue;
          }
          if constexpr (!A_MN) {
            ptx::tma_load_2d_pair(a_dst, &tmap_a, fb, k0 + sh.a_k_off, m0 + sh.a_mn_off);
          } else if (sh.conv == 4) {
            // transposed conv wgrad: A = im2col(x), 64 pixels (K) x 64
            // channels of tap m / C (M) per half, MN-major
#pragma unroll
            for (int h = 0; h < 2; ++h) conv_im2col_mn<Cfg>(sh, &tmap_a, fb, a_dst + h * 8192, k0,
                                                            m0 + h * 64, sh.M, sh.a_k_off);
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              ptx::tma_load_2d_pair(a_dst + h * 8192, &tmap_a, fb, m0 + h * 64 + sh.a_mn_off,
                                    k0 + sh.a_k_off);
          }
#pragma unroll
          for (int j = 0; j < Cfg::kSub; ++j) {
            // MMA j of the k-block: this CTA's B rows of N block j
            const int nbj = tn * BN + j * Cfg::kMmaN + static_cast<int>(rank) * (Cfg::kMmaN / 2);
            uint8_t* bj = b_dst + j * Cfg::kBSub;
            if (B_MN && sh.conv == 2) {
#pragma unroll
              for (int h = 0; h < Cfg::kMmaN / 128; ++h)
                conv_im2col_mn<Cfg>(sh, &tmap_b, fb, bj + h * 8192, k0, nbj + h * 64, sh.N,
                                    sh.b_k_off);
              continue;
            }
            if constexpr (!B_MN) {
              ptx::tma_load_2d_pair(bj, &tmap_b, fb, k0 + sh.b_k_off, nbj + sh.b_mn_off);
            } else {
#pragma unroll
              for (int h = 0; h < Cfg::kMmaN / 128; ++h)
                ptx::tma_load_2d_pair(bj + h * 8192, &tmap_b, fb, nbj + h * 64 + sh.b_mn_off,
                                      k0 + sh.b_k_off);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      // ---------------- MMA issuer (leader only)
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(256, Cfg::kMmaN, A_MN, B_MN);
      int it = 0, local = 0, pit = 0;
      for (int u = pair; u < num_units; u += num_pairs, ++local) {
        const int split = u % S_k;
        const int num_kb = min(kb_all, (split + 1) * kbps) - split * kbps;
        const int acc = local % Cfg::kAccBufs;
        const int use = local / Cfg::kAccBufs;
        ptx::mbar_wait(&tempty_bar[acc], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        if (halo) {
          // per channel chunk: the patch, then the 9 taps as shifted views of
          // it (tap t = (r, s) starts at patch row r * (tw + 2) + s)
          for (int c0 = 0; c0 < sh.conv_c; c0 += 64, ++pit) {
            const int pb = pit & 1;
            ptx::mbar_wait(&pbar[pb], (pit >> 1) & 1);
            ptx::tc_fence_after();
            const uint32_t pa = ptx::smem_u32(patch0 + pb * kPatchBuf);
            for (int tap = 0; tap < 9; ++tap, ++it) {
              const int s = it % S_h;
              ptx::mbar_wait(&full_bar[s], (it / S_h) & 1);
              ptx::tc_fence_after();
              const uint32_t a_row = pa + static_cast<uint32_t>((tap / 3) * (tw + 2) + tap % 3) * 128u;
              const uint32_t b_addr = ptx::smem_u32(sBh + s * Cfg::kBHalf);
#pragma unroll
              for (int kk = 0; kk < Cfg::kBK / 16; ++kk) {
                const uint64_t a_desc = ptx::smem_desc_sw128(a_row + kk * 32, 16, 1024);
#pragma unroll
                for (int j = 0; j < Cfg::kSub; ++j) {
                  const uint32_t bj = b_addr + j * Cfg::kBSub;
                  const uint64_t b_desc =
                      B_MN ? (Cfg::kMmaN == 64 ? ptx::smem_desc_sw64(bj + kk * 1024, 4096, 512)
                                               : ptx::smem_desc_sw128(bj + kk * 2048, 8192, 1024))
                           : ptx::smem_desc_sw128(bj + kk * 32, 16, 1024);
                  ptx::mma_bf16_pair(d_tmem + j * Cfg::kMmaN, a_desc, b_desc, idesc,
                                     (c0 | tap | kk) != 0);
                }
              }
              ptx::mma_commit_pair(&empty_bar[s], 0x3);
            }
            ptx::mma_commit_pair(&pbar[2 + pb], 0x3);
          }
          ptx::mma_commit_pair(&tfull_bar[acc], 0x3);
          continue;
        }
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % S;
          ptx::mbar_wait(&full_bar[s], (it / S) & 1);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sA + s * Cfg::kAHalf);
          const uint32_t b_addr = ptx::smem_u32(sB + s * Cfg::kBHalf);
#pragma unroll
          for (int kk = 0; kk < Cfg::kBK / 16; ++kk) {
            const uint64_t a_desc =
                A_MN ? ptx::smem_desc_sw128(a_addr + kk * 2048, 8192, 1024)
                     : ptx::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
#pragma unroll
            for (int j = 0; j < Cfg::kSub; ++j) {
              const uint32_t bj = b_addr + j * Cfg::kBSub;
              const uint64_t b_desc =
                  B_MN ? (Cfg::kMmaN == 64 ? ptx::smem_desc_sw64(bj + kk * 1024, 4096, 512)
                                           : ptx::smem_desc_sw128(bj + kk * 2048, 8192, 1024))
                       : ptx::smem_desc_sw128(bj + kk * 32, 16, 1024);
              ptx::mma_bf16_pair(d_tmem + j * Cfg::kMmaN, a_desc, b_desc, idesc,
                                 (kb | kk) != 0);
            }
          }
          ptx::mma_commit_pair(&empty_bar[s], 0x3);
        }
        ptx::mma_commit_pair(&tfull_bar[acc], 0x3);
      }
    }
  } else {
    // ---------------- epilogue: warps 2.., both CTAs.  Warp e covers TMEM lane
    // quarter (warp % 4) and column half e / 4 of the tile.
    const int e = warp - 2;
    const int q = warp % 4;  // TMEM lane quarter this warp may access
    constexpr int kColsPerWarp = BN / (Cfg::kEpiWarps / 4);
    const int c_off = (e / 4) * kColsPerWarp;
    float* T = epi_smem + e * 32 * kVecLd;
    const uint32_t tempty_leader_0 = ptx::map_to_rank(&tempty_bar[0], 0);
    const uint32_t tempty_leader_1 = ptx::map_to_rank(&tempty_bar[1], 0);
    // SGD: each lane pulls one fp32 master row segment of this warp's part of
    // a tile into L2 one tile ahead of its update (the first tile during the
    // first mainloop), so the HBM-bound update reads at L2 latency.
    // (dgrad: the stored activations that gate the delta, likewise.)
    auto prefetch_master = [&](int u) {
      if (u >= num_units) return;
      const int t = u / S_k;
      const int row = (t / tiles_n) * 256 + static_cast<int>(rank) * 128 + q * 32 + lane;
      const int n0 = (t % tiles_n) * BN + c_off;
      const int cols = min(kColsPerWarp, sh.N - n0);
      if (row >= sh.M || cols <= 0) return;
      if constexpr (EPI == kEpiWgradSgd) {
        // (the TMA epilogue streams the masters itself, one chunk ahead)
        const uint32_t bytes = static_cast<uint32_t>(cols * 4) & ~15u;
        if (ep.rowwise != 3 && bytes > 0 && (ep.ld_w32 % 4) == 0)
          ptx::prefetch_l2(ep.w_cur + static_cast<size_t>(row) * ep.ld_w32 + n0, bytes);
      } else if constexpr (EPI == kEpiDgrad) {
        const uint32_t bytes = static_cast<uint32_t>(cols * 2) & ~15u;
        if (ep.act_prev != kLinear && bytes > 0 && (ep.ld_xin % 8) == 0)
          ptx::prefetch_l2(ep.xin + static_cast<size_t>(row) * ep.ld_xin + n0, bytes);
      }
    };
    prefetch_master(pair);
    SgdTmaState sgd_st;
    uint8_t* sgd_buf = epi_base + e * Cfg::kSgdWarpBytes;
    int local = 0;
    for (int u = pair; u < num_units; u += num_pairs, ++local) {
      const int tile = u / S_k, split = u % S_k;
      const int acc = local % Cfg::kAccBufs;
      const int use = local / Cfg::kAccBufs;
      const int tm = tile / tiles_n, tn = tile % tiles_n;
      prefetch_master(u + num_pairs);
      ptx::mbar_wait(&tfull_bar[acc], use & 1);
      ptx::tc_fence_after();
      // halo strips: this CTA's rows are its strip's tw pixels
      GemmShape she = sh;
      int row_base = tm * 256 + static_cast<int>(rank) * 128 + q * 32;
      if (halo) {
        const int strip = 2 * tm + static_cast<int>(rank);
        row_base = strip * tw + q * 32;
        she.M = min(sh.M, strip * tw + tw);
      }
      const uint32_t t_row =
          tmem_base + acc * BN + c_off + (static_cast<uint32_t>(q * 32) << 16);
      if ((EPI == kEpiFwd || EPI == kEpiDgrad) && tile == 0 && split == 0 && rank == 0 &&
          e == 0 && lane == 0 && ep.tag_src && ep.tag_dst)
        write_tags(ep);
      if (kExt && EPI == kEpiFwd && ep.fix_cnt && S_k > 1) {
        // split-K fixup: store this split's partial (warp-blocked: each
        // store instruction writes 512 contiguous bytes), publish it, count
        // the arrival; the last split of the tile half reduces and finishes
        if constexpr (kExt && EPI == kEpiFwd) {
          const long long blk = 32LL * kColsPerWarp;
          const long long stride = 2LL * Cfg::kEpiWarps * blk;  // between splits
          float* base = ep.fix_ws + (static_cast<long long>(tile) * S_k * 2 + rank) *
                                        Cfg::kEpiWarps * blk + e * blk;
          float* mine = base + split * stride;
          const int n0 = tn * BN + c_off;
#pragma unroll 1
          for (int c = 0; c < kColsPerWarp; c += 32) {
            if (n0 + c >= sh.N) break;  // warp-uniform
            uint32_t r[32];
            ptx::tmem_ld32(t_row + c, r);
            ptx::tmem_ld_wait();
            float4* p = reinterpret_cast<float4*>(mine + (c / 32) * 1024 + lane * 4);
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4)
              __stcg(p + j4 * 32, make_float4(__uint_as_float(r[4 * j4]),
                                              __uint_as_float(r[4 * j4 + 1]),
                                              __uint_as_float(r[4 * j4 + 2]),
                                              __uint_as_float(r[4 * j4 + 3])));
          }
          __threadfence();
          ptx::named_bar_sync(1, 32 * Cfg::kEpiWarps);
          if (e == 0 && lane == 0) {
            int* cnt = ep.fix_cnt + tile * 2 + rank;
            const int last = atomicAdd(cnt, 1) == S_k - 1;
            if (last) *cnt = 0;  // every split has arrived: ready for the next launch
            *fix_last = last;
          }
          ptx::named_bar_sync(1, 32 * Cfg::kEpiWarps);
          if (*fix_last) {
            __threadfence();
            FixSrc fx;
            fx.base = base;
            fx.stride = stride;
            fx.S = S_k;
            fx.self = split;
            with_act<EPI>(ep, [&](auto A) {
              epilogue_warp_vec<EPI, decltype(A)::value, true>(ep, she, row_base, n0,
                                                               kColsPerWarp, t_row, T, fx);
            });
          }
        }
      } else if (kExt && ep.partial_slab) {
        // split-K into partial slabs (conv wgrad): this split's own fp32
        // slab, plain stores; an in-order reduction consumes the slabs
        if constexpr (kExt && EPI == kEpiFwd) {
          EpiParams epp = ep;
          epp.y32 = ep.y32 + static_cast<size_t>(split) * ep.partial_slab;
          epilogue_warp_vec<EPI, kLinear>(epp, she, row_base, tn * BN + c_off, kColsPerWarp,
                                          t_row, T);
        }
      } else if (ep.dbg_skip & 1) {
      } else if (EPI == kEpiWgradSgd && ep.rowwise == 3) {
        if constexpr (EPI == kEpiWgradSgd) {
          int next_row = -1, next_col = 0;
          if (u + num_pairs < num_units) {
            const int nt = (u + num_pairs) / S_k;
            next_row = (nt / tiles_n) * 256 + static_cast<int>(rank) * 128 + q * 32;
            next_col = (nt % tiles_n) * BN + c_off;
          }
          if (ep.split_master)
            epilogue_warp_tma_sgd_split<Cfg::kSgdBufs>(
                ep, maps, row_base, tn * BN + c_off, kColsPerWarp, t_row, sgd_buf,
                sgd_bar + Cfg::kSgdBufs * e, sgd_st, local == 0, next_row, next_col);
          else
            epilogue_warp_tma_sgd(ep, maps, row_base, tn * BN + c_off, kColsPerWarp, t_row,
                                  sgd_buf, sgd_bar + Cfg::kSgdBufs * e, sgd_st, local == 0,
                                  next_row, next_col);
        }
      } else if (ep.rowwise == 2) {
        with_act<EPI>(ep, [&](auto A) {
          epilogue_warp_vec<EPI, decltype(A)::value>(ep, she, row_base, tn * BN + c_off,
                                                     kColsPerWarp, t_row, T);
        });
      } else if (ep.rowwise) {
        with_act<EPI>(ep, [&](auto A) {
          epilogue_warp_rows<EPI, decltype(A)::value>(ep, she, row_base, tn * BN + c_off,
                                                      kColsPerWarp, t_row);
        });
      } else {
        with_act<EPI>(ep, [&](auto A) {
          epilogue_warp_tile<EPI, decltype(A)::value>(ep, she, row_base, tn * BN + c_off,
                                                      kColsPerWarp, t_row, T);
        });
      }
      ptx::tc_fence_before();
      ptx::named_bar_sync(1, 32 * Cfg::kEpiWarps);
      if (e == 0 && lane == 0)
        ptx::mbar_arrive_cluster(acc == 0 ? tempty_leader_0 : tempty_leader_1);
    }
    if (EPI == kEpiWgradSgd && ep.rowwise == 3 && lane == 0)
      ptx::bulk_wait_group<0>();  // the last TMA stores have landed
  }

  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
  }
}

}  // namespace pb

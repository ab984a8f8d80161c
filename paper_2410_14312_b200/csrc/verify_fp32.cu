// fp32 verify precision: every Linear contraction on the CUDA cores in fp32
// (FFMA, K summed in order), activations / deltas / weight versions stored
// in fp32, the same fused epilogues as the tensor-core path (bias+act,
// act'-gating, SGD into the new version + the device version tags).  It is
// the "fp32-FFMA verify mode" of the north star: losses and ΔW agree with the
// fp64 reference at fp32 rounding, so the bf16 tensor-core path's
// tolerances are measured against a path with none of its rounding.
//
// Layout: the same row-major buffers as the bf16 path, reinterpreted as fp32
// with the same leading dimensions (the session allocates them twice as
// large in this mode).
#include <algorithm>

#include "gemm_sm100.cuh"
#include "layer_ops.cuh"
#include "status.hpp"

namespace pb {

namespace {

constexpr int kT = 64;   // output tile (rows and columns)
constexpr int kTK = 16;  // K step
constexpr int kThr = 256;

// A(m, k): MN-major when A_MN (a[(k + a_k) * lda + m + a_m]) else
// a[(m + a_m) * lda + k + a_k]; B(k, n) likewise with (n, k) for K-major.
template <bool A_MN, bool B_MN, int EPI, int ACT>
__global__ void __launch_bounds__(kThr)
    simt_gemm_fp32(const float* __restrict__ a, int lda, const float* __restrict__ b, int ldb,
                   GemmShape sh, EpiParams ep) {
  __shared__ float As[kTK][kT + 1];
  __shared__ float Bs[kTK][kT + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * kT, n0 = blockIdx.x * kT;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < sh.K; k0 += kTK) {
    for (int i = threadIdx.x; i < kTK * kT; i += kThr) {
      int kk, mm;
      if (A_MN) {  // coalesced along m
        kk = i / kT;
        mm = i % kT;
      } else {     // coalesced along k
        mm = i / kTK;
        kk = i % kTK;
      }
      const int m = m0 + mm, k = k0 + kk;
      float v = 0.f;
      if (m < sh.M && k < sh.K)
        v = A_MN ? a[static_cast<size_t>(k + sh.a_k_off) * lda + m + sh.a_mn_off]
                 : a[static_cast<size_t>(m + sh.a_mn_off) * lda + k + sh.a_k_off];
      As[kk][mm] = v;
    }
    for (int i = threadIdx.x; i < kTK * kT; i += kThr) {
      int kk, nn;
      if (B_MN) {
        kk = i / kT;
        nn = i % kT;
      } else {
        nn = i / kTK;
        kk = i % kTK;
      }
      const int n = n0 + nn, k = k0 + kk;
      float v = 0.f;
      if (n < sh.N && k < sh.K)
        v = B_MN ? b[static_cast<size_t>(k + sh.b_k_off) * ldb + n + sh.b_mn_off]
                 : b[static_cast<size_t>(n + sh.b_mn_off) * ldb + k + sh.b_k_off];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  if (EPI == kEpiFwd || EPI == kEpiDgrad)
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && ep.tag_src && ep.tag_dst)
      write_tags(ep);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= sh.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= sh.N) continue;
      float v = acc[i][j];
      if constexpr (EPI == kEpiFwd) {
        v = act_fwd_t<ACT>(v + (ep.bias ? ep.bias[n] : 0.f));
        const size_t yr = static_cast<size_t>(m + ep.y_row_off);
        if (ep.y16) reinterpret_cast<float*>(ep.y16)[yr * ep.ld_y16 + n] = v;
        if (ep.y32) ep.y32[yr * ep.ld_y32 + n] = v;
      } else if constexpr (EPI == kEpiDgrad) {
        if constexpr (ACT != kLinear)
          v *= act_grad_t<ACT>(
              reinterpret_cast<const float*>(ep.xin)[static_cast<size_t>(m) * ep.ld_xin + n]);
        reinterpret_cast<float*>(ep.d16)[static_cast<size_t>(m) * ep.ld_d16 + n] = v;
      } else {
        const size_t o = static_cast<size_t>(m) * ep.ld_w32 + n;
        const float w = ep.w_cur[o] - ep.lr * v;
        ep.w_new[o] = w;
        if (ep.w16) reinterpret_cast<float*>(ep.w16)[static_cast<size_t>(m) * ep.ld_w16 + n] = w;
      }
    }
  }
}

template <bool A_MN, bool B_MN, int EPI>
void launch_simt(const GemmLaunch& g, cudaStream_t st) {
  dim3 grid((g.sh.N + kT - 1) / kT, (g.sh.M + kT - 1) / kT);
  with_act_host<EPI>(g.ep, [&](auto A) {
    simt_gemm_fp32<A_MN, B_MN, EPI, decltype(A)::value>
        <<<grid, kThr, 0, st>>>(g.simt_a, g.simt_lda, g.simt_b, g.simt_ldb, g.sh, g.ep);
  });
  PB_CUDA(cudaGetLastError());
}

template <typename T>
__global__ void copy_rows_f32(const T* __restrict__ src, int rows, int cols, int ld_src,
                              float* __restrict__ dst, int ld_dst) {
  const size_t n = static_cast<size_t>(rows) * cols;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / cols, c = i % cols;
    dst[r * ld_dst + c] = static_cast<float>(src[r * ld_src + c]);
  }
}

int grid_for(size_t n) {
  size_t g = (n + 255) / 256;
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(g, 148 * 16)));
}

}  // namespace

void launch_simt_gemm(const GemmLaunch& g, int kind, cudaStream_t st) {
  if (kind == kEpiFwd)
    launch_simt<false, false, kEpiFwd>(g, st);
  else if (kind == kEpiDgrad)
    launch_simt<false, true, kEpiDgrad>(g, st);
  else
    launch_simt<true, true, kEpiWgradSgd>(g, st);
}

void launch_rows_to_f32(cudaStream_t st, const void* src, bool src_f64, int rows, int cols,
                        int ld_src, float* dst, int ld_dst) {
  const size_t n = static_cast<size_t>(rows) * cols;
  if (src_f64)
    copy_rows_f32<double><<<grid_for(n), 256, 0, st>>>(static_cast<const double*>(src), rows,
                                                       cols, ld_src, dst, ld_dst);
  else
    copy_rows_f32<float><<<grid_for(n), 256, 0, st>>>(static_cast<const float*>(src), rows,
                                                      cols, ld_src, dst, ld_dst);
  PB_CUDA(cudaGetLastError());
}

}  // namespace pb

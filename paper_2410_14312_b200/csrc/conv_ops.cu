// Convolution-stage kernels of the VGG-style pipeline (BASELINE configs[3],
// SURVEY §8(f)#4).  The reference has no convolution; these
// extend its Linear stage math to 3x3 / pad 1 convolutions and 2x2 max
// pooling on NHWC bf16 activations.  The conv GEMMs themselves are the
// tcgen05 pair kernel with im2col TMA operands (gemm_sm100.cuh, conv modes);
// this file holds the memory-bound pieces around them:
//   * im2col of the network input (3 channels: too narrow for a 64-channel
//     im2col TMA box), K padded with zeros to the operand's leading dimension;
//   * 2x2 max pooling forward / backward (the gradient goes to the first
//     maximum of each window, in (0,0) (0,1) (1,0) (1,1) order);
//   * the in-order reduction of the conv wgrad's split-K fp32 partial slabs
//     fused with the SGD update and the bf16 copy of the new version.
#include <cuda_bf16.h>

#include <algorithm>

#include "conv_ops.cuh"
#include "status.hpp"

namespace pb {
namespace {

int blocks_for(size_t n, int threads = 256) {
  size_t g = (n + threads - 1) / threads;
  return static_cast<int>(std::min<size_t>(std::max<size_t>(g, 1), 148 * 32));
}

// out[(n*H + h)*W + w][k], k = (3r + s) * C + c; zero outside the image and
// for k >= 9C.  One output pixel per thread: its row (LDO elements, 16-byte
// vectors) is assembled in registers and written whole, so a warp stores
// 32 contiguous rows; the 9 * C input reads hit L1 / L2 (neighbouring
// pixels share their windows).
template <int LDO>
__global__ void __launch_bounds__(256)
    im2col_first_kernel(const __nv_bfloat16* __restrict__ x, int ld_x, int n_imgs, int H,
                        int W, int C, __nv_bfloat16* __restrict__ out) {
  const size_t pixels = static_cast<size_t>(n_imgs) * H * W;
  for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < pixels;
       p += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int w = static_cast<int>(p % W);
    const int h = static_cast<int>((p / W) % H);
    const size_t n = p / (static_cast<size_t>(W) * H);
    const __nv_bfloat16* img = x + n * ld_x;
    uint4 row[LDO / 8];
    __nv_bfloat16* e = reinterpret_cast<__nv_bfloat16*>(row);
#pragma unroll
    for (int k = 0; k < LDO; ++k) e[k] = __float2bfloat16(0.f);
    for (int tap = 0; tap < 9; ++tap) {
      const int ih = h + tap / 3 - 1, iw = w + tap % 3 - 1;
      if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
      const __nv_bfloat16* src = img + (static_cast<size_t>(ih) * W + iw) * C;
      for (int c = 0; c < C; ++c) e[tap * C + c] = src[c];
    }
    uint4* dst = reinterpret_cast<uint4*>(out + p * LDO);
#pragma unroll
    for (int v = 0; v < LDO / 8; ++v) dst[v] = row[v];
  }
}

// 8 channels (16 bytes) per thread
__global__ void maxpool2_fwd_kernel(const __nv_bfloat16* __restrict__ in, int n_imgs, int H,
                                    int W, int C, __nv_bfloat16* __restrict__ out) {
  const int Ho = H / 2, Wo = W / 2, C8 = C / 8;
  const size_t total = static_cast<size_t>(n_imgs) * Ho * Wo * C8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % C8);
    const size_t p = i / C8;
    const int wo = static_cast<int>(p % Wo), ho = static_cast<int>((p / Wo) % Ho);
    const size_t n = p / (static_cast<size_t>(Wo) * Ho);
    const __nv_bfloat16* base = in + ((n * H + 2 * ho) * W + 2 * wo) * C + 8 * c8;
    uint4 q[4];
    q[0] = *reinterpret_cast<const uint4*>(base);
    q[1] = *reinterpret_cast<const uint4*>(base + C);
    q[2] = *reinterpret_cast<const uint4*>(base + static_cast<size_t>(W) * C);
    q[3] = *reinterpret_cast<const uint4*>(base + static_cast<size_t>(W) * C + C);
    const __nv_bfloat162* v[4];
    for (int j = 0; j < 4; ++j) v[j] = reinterpret_cast<const __nv_bfloat162*>(&q[j]);
    uint4 r;
    __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = __hmax2(__hmax2(v[0][e], v[1][e]), __hmax2(v[2][e], v[3][e]));
    *reinterpret_cast<uint4*>(out + p * C + 8 * c8) = r;
  }
}

// 8 channels (16-byte vectors) of one pooled pixel per thread: the window's
// four input vectors and the pooled vector are read once, the gradient goes
// to the first maximum of each channel's window, the four input-gradient
// vectors are written whole
__global__ void maxpool2_bwd_kernel(const __nv_bfloat16* __restrict__ d_out,
                                    const __nv_bfloat16* __restrict__ in,
                                    const __nv_bfloat16* __restrict__ out, int n_imgs, int H,
                                    int W, int C, __nv_bfloat16* __restrict__ d_in) {
  const int Ho = H / 2, Wo = W / 2, C8 = C / 8;
  const size_t total = static_cast<size_t>(n_imgs) * Ho * Wo * C8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % C8);
    const size_t p = i / C8;
    const int wo = static_cast<int>(p % Wo), ho = static_cast<int>((p / Wo) % Ho);
    const size_t n = p / (static_cast<size_t>(Wo) * Ho);
    const size_t a0 = ((n * H + 2 * ho) * W + 2 * wo) * C + 8 * c8;
    const size_t off[4] = {a0, a0 + C, a0 + static_cast<size_t>(W) * C,
                           a0 + static_cast<size_t>(W) * C + C};
    uint4 q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = *reinterpret_cast<const uint4*>(in + off[j]);
    const uint4 mv = *reinterpret_cast<const uint4*>(out + p * C + 8 * c8);
    const uint4 gv = *reinterpret_cast<const uint4*>(d_out + p * C + 8 * c8);
    const __nv_bfloat16* m = reinterpret_cast<const __nv_bfloat16*>(&mv);
    const __nv_bfloat16* g = reinterpret_cast<const __nv_bfloat16*>(&gv);
    uint4 r[4];
    __nv_bfloat16* rv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) rv[j] = reinterpret_cast<__nv_bfloat16*>(&r[j]);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      bool taken = false;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat16 v = reinterpret_cast<const __nv_bfloat16*>(&q[j])[e];
        const bool hit = !taken && __bfloat162float(v) == __bfloat162float(m[e]);
        taken |= hit;
        rv[j][e] = hit ? g[e] : __float2bfloat16(0.f);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) *reinterpret_cast<uint4*>(d_in + off[j]) = r[j];
  }
}

// w_new = w_cur - lr * sum_{s < S} slab_s (in split order); w16 = bf16(w_new)
__global__ void reduce_sgd_kernel(const float* __restrict__ slabs, int S, long long slab,
                                  int rows, int cols, int lds, const float* __restrict__ w_cur,
                                  float* __restrict__ w_new, int ldw,
                                  __nv_bfloat16* __restrict__ w16, int ld16, float lr) {
  const size_t total = static_cast<size_t>(rows) * cols;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / cols, c = i % cols;
    const float* p = slabs + r * lds + c;
    float g = 0.f;
    for (int s = 0; s < S; ++s) g += p[static_cast<size_t>(s) * slab];
    const float w = w_cur[r * ldw + c] - lr * g;
    w_new[r * ldw + c] = w;
    if (w16) w16[r * ld16 + c] = __float2bfloat16(w);
  }
}

// The same from transposed slabs ([cols][lds]): 32 x 32 tiles, read
// coalesced along the slab rows, written coalesced along the weight rows
// through shared memory; the S partials of an element are still added in
// split order.
__global__ void __launch_bounds__(256)
    reduce_sgd_t_kernel(const float* __restrict__ slabs, int S, long long slab, int rows,
                        int cols, int lds, const float* __restrict__ w_cur,
                        float* __restrict__ w_new, int ldw, __nv_bfloat16* __restrict__ w16,
                        int ld16, float lr) {
  __shared__ float tile[32][33];
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = c0 + ty + 8 * i, r = r0 + tx;
    float g = 0.f;
    if (c < cols && r < rows) {
      const float* p = slabs + static_cast<size_t>(c) * lds + r;
      for (int s = 0; s < S; ++s) g += p[static_cast<size_t>(s) * slab];
    }
    tile[ty + 8 * i][tx] = g;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty + 8 * i, c = c0 + tx;
    if (r < rows && c < cols) {
      const float w = w_cur[static_cast<size_t>(r) * ldw + c] - lr * tile[tx][ty + 8 * i];
      w_new[static_cast<size_t>(r) * ldw + c] = w;
      if (w16) w16[static_cast<size_t>(r) * ld16 + c] = __float2bfloat16(w);
    }
  }
}

// grid (chunks, cols / 64): 32 row lanes x 8 column groups of 8 (16-byte
// loads); the 32 lane sums of a column are added in lane order
__global__ void __launch_bounds__(256)
    colsum_partial_kernel(const __nv_bfloat16* __restrict__ dz, int rows, int cols, int ld,
                          int rows_per_chunk, float* __restrict__ partial) {
  __shared__ float red[32][65];
  const int cg = threadIdx.x % 8, lane = threadIdx.x / 8;
  const int c0 = blockIdx.y * 64 + cg * 8;
  const int r0 = blockIdx.x * rows_per_chunk;
  const int r1 = min(rows, r0 + rows_per_chunk);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 < cols)
    for (int r = r0 + lane; r < r1; r += 32) {
      const uint4 q = *reinterpret_cast<const uint4*>(dz + static_cast<size_t>(r) * ld + c0);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
#pragma unroll
  for (int k = 0; k < 8; ++k) red[lane][cg * 8 + k] = acc[k];
  __syncthreads();
  if (threadIdx.x < 64 && blockIdx.y * 64 + threadIdx.x < cols) {
    float sum = 0.f;
    for (int i = 0; i < 32; ++i) sum += red[i][threadIdx.x];
    partial[static_cast<size_t>(blockIdx.x) * cols + blockIdx.y * 64 + threadIdx.x] = sum;
  }
}

}  // namespace

void launch_colsum_partial(cudaStream_t st, const __nv_bfloat16* dz, int rows, int cols, int ld,
                           float* partial) {
  if (cols % 8 != 0 || ld % 8 != 0 || (reinterpret_cast<uintptr_t>(dz) & 15) != 0)
    throw std::invalid_argument("colsum: 16-byte rows required");
  const int chunks = colsum_chunks(rows);
  const int per = (rows + chunks - 1) / chunks;
  colsum_partial_kernel<<<dim3(chunks, (cols + 63) / 64), 256, 0, st>>>(dz, rows, cols, ld, per,
                                                                        partial);
  PB_CUDA(cudaGetLastError());
}

void launch_im2col_first(cudaStream_t st, const __nv_bfloat16* x, int ld_x, int n_imgs, int H,
                         int W, int C, __nv_bfloat16* out, int ldo) {
  if (9 * C > ldo || (reinterpret_cast<uintptr_t>(out) & 15) != 0)
    throw std::invalid_argument("im2col_first: 9 * C <= ldo and 16-byte rows required");
  const size_t pixels = static_cast<size_t>(n_imgs) * H * W;
  const int grid = blocks_for(pixels);
  switch (ldo) {
#define PB_IM2COL_CASE(L) \
  case L: im2col_first_kernel<L><<<grid, 256, 0, st>>>(x, ld_x, n_imgs, H, W, C, out); break;
    PB_IM2COL_CASE(8) PB_IM2COL_CASE(16) PB_IM2COL_CASE(24) PB_IM2COL_CASE(32)
    PB_IM2COL_CASE(40) PB_IM2COL_CASE(48) PB_IM2COL_CASE(56) PB_IM2COL_CASE(64)
    PB_IM2COL_CASE(72)
#undef PB_IM2COL_CASE
    default: throw std::invalid_argument("im2col_first: ldo must be a multiple of 8 <= 72");
  }
  PB_CUDA(cudaGetLastError());
}

void launch_maxpool2_fwd(cudaStream_t st, const __nv_bfloat16* in, int n_imgs, int H, int W,
                         int C, __nv_bfloat16* out) {
  if (C % 8 != 0 || H % 2 != 0 || W % 2 != 0)
    throw std::invalid_argument("maxpool2: C % 8 and even H, W required");
  const size_t total = static_cast<size_t>(n_imgs) * (H / 2) * (W / 2) * (C / 8);
  maxpool2_fwd_kernel<<<blocks_for(total), 256, 0, st>>>(in, n_imgs, H, W, C, out);
  PB_CUDA(cudaGetLastError());
}

void launch_maxpool2_bwd(cudaStream_t st, const __nv_bfloat16* d_out, const __nv_bfloat16* in,
                         const __nv_bfloat16* out, int n_imgs, int H, int W, int C,
                         __nv_bfloat16* d_in) {
  if (C % 8 != 0 || H % 2 != 0 || W % 2 != 0)
    throw std::invalid_argument("maxpool2: C % 8 and even H, W required");
  const size_t total = static_cast<size_t>(n_imgs) * (H / 2) * (W / 2) * (C / 8);
  maxpool2_bwd_kernel<<<blocks_for(total), 256, 0, st>>>(d_out, in, out, n_imgs, H, W, C, d_in);
  PB_CUDA(cudaGetLastError());
}

void launch_reduce_sgd(cudaStream_t st, const float* slabs, int S, long long slab, int rows,
                       int cols, int lds, const float* w_cur, float* w_new, int ldw,
                       __nv_bfloat16* w16, int ld16, float lr, bool transposed) {
  if (transposed) {
    reduce_sgd_t_kernel<<<dim3((rows + 31) / 32, (cols + 31) / 32), 256, 0, st>>>(
        slabs, S, slab, rows, cols, lds, w_cur, w_new, ldw, w16, ld16, lr);
    PB_CUDA(cudaGetLastError());
    return;
  }
  const size_t total = static_cast<size_t>(rows) * cols;
  reduce_sgd_kernel<<<blocks_for(total), 256, 0, st>>>(slabs, S, slab, rows, cols, lds, w_cur,
                                                       w_new, ldw, w16, ld16, lr);
  PB_CUDA(cudaGetLastError());
}

}  // namespace pb

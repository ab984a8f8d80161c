// Convolution-stage operations (conv_ops.cu, layer_ops.cu conv plans).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "layer_ops.cuh"

namespace pb {

// --- memory-bound kernels (conv_ops.cu)
void launch_im2col_first(cudaStream_t st, const __nv_bfloat16* x, int ld_x, int n_imgs, int H,
                         int W, int C, __nv_bfloat16* out, int ldo);
void launch_maxpool2_fwd(cudaStream_t st, const __nv_bfloat16* in, int n_imgs, int H, int W,
                         int C, __nv_bfloat16* out);
void launch_maxpool2_bwd(cudaStream_t st, const __nv_bfloat16* d_out, const __nv_bfloat16* in,
                         const __nv_bfloat16* out, int n_imgs, int H, int W, int C,
                         __nv_bfloat16* d_in);
// Column sums of a tall bf16 matrix (rows x cols, cols % 8 == 0) by row
// blocks: partial[c * cols + j] = sum of column j over row block c, for
// c < colsum_chunks(rows) (a fixed split: the bias gradient stays
// deterministic; launch_bias_sgd then sums the partials in order).
constexpr int kColsumChunks = 512;
inline int colsum_chunks(int rows) {
  const int c = (rows + 1023) / 1024;
  return c < 1 ? 1 : (c > kColsumChunks ? kColsumChunks : c);
}
void launch_colsum_partial(cudaStream_t st, const __nv_bfloat16* dz, int rows, int cols, int ld,
                           float* partial);
// w_new = w_cur - lr * sum_{s < S} slab_s (in split order), w16 = bf16(w_new)
// (may be null); rows x cols of the weights; transposed: the slabs hold
// [cols][rows] (rows of lds floats either way)
void launch_reduce_sgd(cudaStream_t st, const float* slabs, int S, long long slab, int rows,
                       int cols, int lds, const float* w_cur, float* w_new, int ldw,
                       __nv_bfloat16* w16, int ld16, float lr, bool transposed = false);

// --- implicit-GEMM 3x3 / pad 1 / stride 1 convolution GEMMs (layer_ops.cu)
// NHWC activation tensor: n images of H x W x C, contiguous.
struct Nhwc {
  const __nv_bfloat16* ptr;
  int n, h, w, c;
};

// y[(img0 + i) pixels, Cout] = act(conv(x images img0 .. img0+imgs) + b):
// w = [Cout, 9 * Cin] (tap-major K), y row offset y_row_off (pixels).
GemmLaunch plan_conv_fwd(const Nhwc& x, int img0, int imgs, const Mat16& w, const float* bias,
                         int act, __nv_bfloat16* y16, int y_row_off);
// d[pixels, Cin] = conv_transpose(dz, W) .* act'(xin): dz = [n][H][W][Cout],
// w = [Cout, ld] with ld >= 9 * Cin, xin / d = [n*H*W, Cin].
GemmLaunch plan_conv_dgrad(const Nhwc& dz, const __nv_bfloat16* w, int cin, int ld_w,
                           const __nv_bfloat16* xin, int act_prev, __nv_bfloat16* d);
// Partial weight gradients of a conv on the CTA-pair kernel: slab s = the
// sum over its pixel range of dz[p, :]^T im2col(x)[p, :] (fp32 [Cout][9*Cin],
// or its transpose [9*Cin][Cout] for Cout < 256), at ws + s * slab with rows
// of lds floats.  x images img0 .. img0 + dz pixels / (H*W).
struct ConvWgradInfo {
  int splits = 1, lds = 0;
  long long slab = 0;
  bool transposed = false;
};
GemmLaunch plan_conv_wgrad_partial(const Mat16& dz, const Nhwc& x, int img0, float* ws,
                                   ConvWgradInfo* info);
// workspace floats plan_conv_wgrad_partial needs
size_t conv_wgrad_floats(int cout, int cin, int pixels);
// The same for a plain [pixels, K] operand (the network input's im2col).
GemmLaunch plan_wgrad_partial(const Mat16& dz, const Mat16& x, float* ws, int lds, int* splits);
// workspace floats plan_*wgrad_partial needs for an M x N gradient
size_t wgrad_partial_floats(int M, int N, int K, int* lds);
void launch_wgrad_partial(const GemmLaunch& g, cudaStream_t st);

}  // namespace pb

// im2col TMA probe: pins down the coordinate semantics of
// cp.async.bulk.tensor.4d.im2col (the implicit-GEMM conv operand load) on
// sm_100a before the conv kernels rely on them.  An NHWC bf16 tensor with
// value(n,h,w,c) = f(n,h,w,c) is loaded as 128 "pixels" x 64 channels for a
// given start pixel and filter tap, with a 128-byte swizzle; the kernel
// un-swizzles into global memory and the host compares against a CPU
// im2col for 3x3 / pad 1 / stride 1.
//
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a \
//        -I../paper_2410_14312_b200/csrc im2col_probe.cu -lcuda -o im2col_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "sm100_ptx.cuh"

using namespace pb;

__device__ __forceinline__ void tma_load_im2col_4d(void* dst, const CUtensorMap* map,
                                                   uint64_t* bar, int c, int w, int h, int n,
                                                   uint16_t w_off, uint16_t h_off) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(ptx::smem_u32(bar)), "r"(c), "r"(w), "r"(h),
      "r"(n), "h"(w_off), "h"(h_off)
      : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap map, int c, int w, int h, int n,
                      int w_off, int h_off, __nv_bfloat16* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384);
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(bar, 16384);
    tma_load_im2col_4d(smem, &map, bar, c, w, h, n, static_cast<uint16_t>(w_off),
                       static_cast<uint16_t>(h_off));
  }
  ptx::mbar_wait(bar, 0);
  // un-swizzle (128B: 16-byte unit u of row r lives at unit u ^ (r & 7))
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, col = i % 64;
    const int unit = col / 8, within = col % 8;
    const int off = r * 128 + ((unit ^ (r & 7)) * 16) + within * 2;
    out[i] = *reinterpret_cast<const __nv_bfloat16*>(smem + off);
  }
}

static float val(int n, int h, int w, int c) { return float((n * 7 + h * 3 + w * 5 + c) % 251); }

int main() {
  const int N = 3, H = 7, W = 9, C = 64;
  std::vector<__nv_bfloat16> x(static_cast<size_t>(N) * H * W * C);
  for (int n = 0; n < N; ++n)
    for (int h = 0; h < H; ++h)
      for (int w = 0; w < W; ++w)
        for (int c = 0; c < C; ++c)
          x[((static_cast<size_t>(n) * H + h) * W + w) * C + c] = __float2bfloat16(val(n, h, w, c));
  __nv_bfloat16 *dx, *dout;
  cudaMalloc(&dx, x.size() * 2);
  cudaMalloc(&dout, 128 * 64 * 2);
  cudaMemcpy(dx, x.data(), x.size() * 2, cudaMemcpyHostToDevice);

  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[4] = {C, W, H, N};
  cuuint64_t strides[3] = {C * 2ull, C * 2ull * W, C * 2ull * W * H};
  int lower[2] = {-1, -1}, upper[2] = {-1, -1};  // {W, H}: pad 1, 3x3 filter
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dx, dims, strides, lower, upper, 64,
                   128, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", static_cast<int>(r));
    return 1;
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 2048);
  std::vector<__nv_bfloat16> out(128 * 64);
  int total_bad = 0;
  // start output pixels (linear over N*H*W) and taps; candidate coordinate
  // convention: {c, wo - pad, ho - pad, n} with offsets {s, r}
  const int starts[] = {0, 5, 17, 60, 100, 63 + 63};
  for (int p0 : starts)
    for (int rr = 0; rr < 3; ++rr)
      for (int ss = 0; ss < 3; ++ss) {
        const int n0 = p0 / (H * W), ho = (p0 / W) % H, wo = p0 % W;
        probe<<<1, 128, 16384 + 2048>>>(map, 0, wo - 1, ho - 1, n0, ss, rr, dout);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("kernel error %s\n", cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(out.data(), dout, out.size() * 2, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 128; ++i) {
          const int p = p0 + i;
          const int n = p / (H * W), oh = (p / W) % H, ow = p % W;
          const int ih = oh - 1 + rr, iw = ow - 1 + ss;
          for (int c = 0; c < 64; ++c) {
            float want = 0.f;
            if (n < N && ih >= 0 && ih < H && iw >= 0 && iw < W) want = val(n, ih, iw, c);
            const float got = __bfloat162float(out[i * 64 + c]);
            if (got != want) {
              if (bad < 3)
                printf("  p0=%d tap(%d,%d) pixel %d c %d: got %g want %g\n", p0, rr, ss, i, c,
                       got, want);
              ++bad;
            }
          }
        }
        total_bad += bad;
      }
  printf("im2col probe: %d mismatches\n", total_bad);
  return total_bad != 0;
}

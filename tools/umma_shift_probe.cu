// UMMA shifted-operand probe: can a tcgen05.mma A operand start at an
// arbitrary 128-byte row inside a 128B-swizzled tile (the descriptor's start
// address not aligned to the 1024-byte swizzle atom)?  That is what a halo
// conv needs: one 3-row patch in shared memory, the 9 filter taps as 9
// shifted views of it.  A [136 x 64] bf16 tile is loaded by TMA (128B
// swizzle), then for every shift s the MMA reads rows [s, s + 128) through a
// descriptor starting at s * 128 bytes, with the matrix base offset field
// (bits 49-51) either 0 or (address >> 7) & 7; D is compared with the CPU.
//
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a \
//        -I../paper_2410_14312_b200/csrc umma_shift_probe.cu -lcuda -o umma_shift_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100_ptx.cuh"

using namespace pb;

constexpr int kRowsA = 136, kN = 64, kK = 64;

__global__ void probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                      int shift, int bo_mode, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                      // 136 x 128 B (17 KB)
  uint8_t* sB = smem + 18 * 1024;          // 64 x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 28 * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 28 * 1024 + 64);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) ptx::tmem_alloc<64>(tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar[0], kRowsA * 128 + kN * 128);
    ptx::tma_load_2d(sA, &ma, &bar[0], 0, 0);
    ptx::tma_load_2d(sB, &mb, &bar[0], 0, 0);
  }
  ptx::mbar_wait(&bar[0], 0);
  if (threadIdx.x == 0) {
    ptx::tc_fence_after();
    const uint32_t idesc = ptx::idesc_bf16_f32(128, kN, false, false);
    const uint32_t a0 = ptx::smem_u32(sA) + shift * 128;
    const uint32_t b0 = ptx::smem_u32(sB);
    for (int kk = 0; kk < kK / 16; ++kk) {
      uint64_t ad = ptx::smem_desc_sw128(a0 + kk * 32, 16, 1024);
      if (bo_mode == 1) ad |= static_cast<uint64_t>((a0 >> 7) & 7) << 49;
      const uint64_t bd = ptx::smem_desc_sw128(b0 + kk * 32, 16, 1024);
      ptx::mma_bf16(tmem, ad, bd, idesc, kk != 0);
    }
    ptx::mma_commit(&bar[1]);
  }
  ptx::mbar_wait(&bar[1], 0);
  ptx::tc_fence_after();
  uint32_t r[32];
  for (int c = 0; c < kN; c += 32) {
    ptx::tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(warp * 32 + threadIdx.x % 32) * kN + c + j] = __uint_as_float(r[j]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<64>(tmem);
}

static CUtensorMap map2d(void* p, int rows, int cols, int box_rows) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", static_cast<int>(r));
  return m;
}

int main() {
  std::vector<__nv_bfloat16> a(kRowsA * kK), b(kN * kK);
  std::vector<float> af(a.size()), bf(b.size());
  for (int i = 0; i < kRowsA; ++i)
    for (int k = 0; k < kK; ++k) {
      af[i * kK + k] = static_cast<float>((i * 7 + k * 3) % 13 - 6);
      a[i * kK + k] = __float2bfloat16(af[i * kK + k]);
    }
  for (int j = 0; j < kN; ++j)
    for (int k = 0; k < kK; ++k) {
      bf[j * kK + k] = static_cast<float>((j * 5 + k * 11) % 9 - 4);
      b[j * kK + k] = __float2bfloat16(bf[j * kK + k]);
    }
  __nv_bfloat16 *da, *db;
  float* dout;
  cudaMalloc(&da, a.size() * 2);
  cudaMalloc(&db, b.size() * 2);
  cudaMalloc(&dout, 128 * kN * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  const CUtensorMap ma = map2d(da, kRowsA, kK, kRowsA);
  const CUtensorMap mb = map2d(db, kN, kK, kN);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  std::vector<float> out(128 * kN);
  int fails = 0;
  for (int bo = 0; bo < 2; ++bo)
    for (int s = 0; s <= 8; ++s) {
      probe<<<1, 128, 32 * 1024>>>(ma, mb, s, bo, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("kernel error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < kN; ++j) {
          float want = 0.f;
          for (int k = 0; k < kK; ++k) want += af[(s + i) * kK + k] * bf[j * kK + k];
          if (out[i * kN + j] != want) ++bad;
        }
      printf("base_offset %s shift %d: %d mismatches\n", bo ? "addr>>7&7" : "0", s, bad);
      if (bad) ++fails;
    }
  return 0;
}

// TMA ingest probe: how many bytes per clock one SM can pull through TMA
// (128-byte-swizzled 2-D boxes, the GEMM mainloop's access pattern) when
// n SMs stream L2-resident data at once, with no MMA consuming it.  Guides
// the GEMM work (is the mainloop bound by per-SM ingest or by L2?).
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I../paper_2410_14312_b200/csrc \
//        tma_probe.cu -lcuda -o tma_probe && ./tma_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100_ptx.cuh"

using namespace pb;

constexpr int kStages = 6;
constexpr int kBoxRows = 128;  // 128 x 64 bf16 = 16 KB per box
constexpr int kBoxBytes = kBoxRows * 64 * 2;

__global__ void __launch_bounds__(64, 1)
    probe(const __grid_constant__ CUtensorMap map, int rows, int kblocks, int boxes_per_stage,
          unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * boxes_per_stage * kBoxBytes);
  uint64_t* empty = full + kStages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int row0 = (blockIdx.x * kBoxRows * boxes_per_stage) % rows;
  const long long t0 = clock64();
  if (threadIdx.x == 0) {  // producer
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kStages;
      if (kb >= kStages) ptx::mbar_wait(&empty[s], ((kb / kStages) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&full[s], boxes_per_stage * kBoxBytes);
      for (int b = 0; b < boxes_per_stage; ++b)
        ptx::tma_load_2d(smem + (s * boxes_per_stage + b) * kBoxBytes, &map, &full[s],
                         (kb * 64) % 4096, (row0 + b * kBoxRows) % rows);
    }
  } else if (threadIdx.x == 32) {  // consumer: release each stage on arrival
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kStages;
      ptx::mbar_wait(&full[s], (kb / kStages) & 1);
      ptx::mbar_arrive(&empty[s]);
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  const int rows = 4096, cols = 4096;  // 32 MiB of bf16: L2-resident after the first pass
  void* buf;
  cudaMalloc(&buf, static_cast<size_t>(rows) * cols * 2);
  cudaMemset(buf, 0, static_cast<size_t>(rows) * cols * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {64, kBoxRows};
  cuuint32_t estr[2] = {1, 1};
  reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(
      &map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
  int sm_mhz = 0;
  cudaDeviceGetAttribute(&sm_mhz, cudaDevAttrClockRate, 0);
  for (int bps : {1, 2, 3}) {
    const int smem = kStages * bps * kBoxBytes + 1024 + 256;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int n : {8, 32, 64, 128, 148}) {
      const int kblocks = 512;
      probe<<<n, 64, smem>>>(map, rows, kblocks, bps, cyc);  // warm L2
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      probe<<<n, 64, smem>>>(map, rows, kblocks, bps, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> c(n);
      cudaMemcpy(c.data(), cyc, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double mean = 0;
      for (auto v : c) mean += static_cast<double>(v) / n;
      const double bytes_per_sm = static_cast<double>(kblocks) * bps * kBoxBytes;
      printf("boxes/stage %d  SMs %3d  per-SM %.1f B/clk  chip %.2f TB/s (%.3f ms)  err=%s\n", bps,
             n, bytes_per_sm / mean, bytes_per_sm * n / (ms / 1e3) / 1e12, ms,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  printf("sm clock attr %d MHz\n", sm_mhz / 1000);
  return 0;
}

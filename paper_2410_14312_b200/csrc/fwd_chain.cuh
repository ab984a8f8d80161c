// Two consecutive Linear forwards of a stage in one kernel, for a stage
// whose last two layers are narrow: the first's output has n1 <= 256
// columns (one CTA holds a 128-row block of it in TMEM), the second's
// n2 <= 64 (trainer.cpp:179-206 applied twice):
//
//   y1 = act1(x W1^T + b1)      128 x n1, K1 = in_{l-1} (pipelined k-blocks)
//   y2 = epi2(y1 W2^T)          128 x n2, K2 = n1 (<= 4 k-blocks)
//
// Each CTA owns 128 rows.  GEMM 1 runs a 4-deep TMA ring into TMEM; its
// epilogue (bias, activation, bf16) writes y1 straight into shared memory in
// the 128B-swizzled K-major layout GEMM 2's A operand needs (over the idle
// ring) and TMA-stores it to the stage's activation buffer (the backward
// reads it).  GEMM 2's epilogue is the plain forward epilogue of layer l:
// bias + activation, or the logits with the softmax cross-entropy fused
// (EpiParams::loss_*).  On C1's stage 2 (512->256->10) this replaces two
// dependent launches of the pipeline's dependency cycle.
#pragma once

#include "gemm_sm100.cuh"

namespace pb {

struct FwdChainCfg {
  static constexpr int kStages = 4;
  static constexpr int kABytes = 128 * 64 * 2;                // x k-block
  static constexpr int kBBytes = 256 * 64 * 2;                // W1 k-block (n1 <= 256 rows)
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kRing = kStages * kStageBytes;         // also holds A2 + staging
  static constexpr int kA2Tile = 128 * 64 * 2;                // one k-block of y1
  static constexpr int kB2Blk = 64 * 64 * 2;                  // W2 k-block (n2 <= 64 rows)
  static constexpr int kOffB2 = kRing;
  static constexpr int kOffBar = kOffB2 + 4 * kB2Blk;
  static constexpr int kSmem = kOffBar + 128 + 1024;
  static_assert(4 * kA2Tile + 4 * 32 * kVecLd * 4 <= kRing, "A2 + staging must fit the ring");
  static_assert(kSmem <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

template <int ACT1>
__global__ void __launch_bounds__(128, 1)
    fwd_chain_kernel(const __grid_constant__ CUtensorMap tm_x,
                     const __grid_constant__ CUtensorMap tm_w1,
                     const __grid_constant__ CUtensorMap tm_w2,
                     const __grid_constant__ CUtensorMap tm_y1, GemmShape sh1, GemmShape sh2,
                     EpiParams ep2, FwdChainArgs fa) {
  using Cfg = FwdChainCfg;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint8_t* sA2 = smem;  // over the ring once GEMM 1 is done
  uint8_t* sB2 = smem + Cfg::kOffB2;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* b2_bar = empty_bar + S;
  uint64_t* acc1_bar = b2_bar + 1;
  uint64_t* acc2_bar = acc1_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc2_bar + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int m0 = blockIdx.x * 128;
  const int n1 = sh1.N, n2pad = fa.n2pad;
  const int kb1 = (sh1.K + 63) / 64;
  const int kb2 = n1 / 64;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tm_x);
    ptx::tma_prefetch_desc(&tm_w1);
    ptx::tma_prefetch_desc(&tm_w2);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full_bar[i], 1);
      ptx::mbar_init(&empty_bar[i], 1);
    }
    ptx::mbar_init(b2_bar, 1);
    ptx::mbar_init(acc1_bar, 1);
    ptx::mbar_init(acc2_bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t acc1 = tmem_base, acc2 = tmem_base + 256;
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();

  if (warp == 0 && lane == 0) {
    // W2 first (one barrier, read after GEMM 1), then GEMM 1's ring
    ptx::mbar_arrive_expect_tx(b2_bar, kb2 * n2pad * 128);
    for (int j = 0; j < kb2; ++j) ptx::tma_load_2d(sB2 + j * Cfg::kB2Blk, &tm_w2, b2_bar, j * 64, 0);
    for (int kb = 0; kb < kb1; ++kb) {
      const int s = kb % S;
      if (kb >= S) ptx::mbar_wait(&empty_bar[s], ((kb / S) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&full_bar[s], Cfg::kABytes + n1 * 128);
      uint8_t* st = ring + s * Cfg::kStageBytes;
      ptx::tma_load_2d(st, &tm_x, &full_bar[s], kb * 64, m0 + sh1.a_mn_off);
      ptx::tma_load_2d(st + Cfg::kABytes, &tm_w1, &full_bar[s], kb * 64, 0);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc1 = ptx::idesc_bf16_f32(128, n1, false, false);
    for (int kb = 0; kb < kb1; ++kb) {
      const int s = kb % S;
      ptx::mbar_wait(&full_bar[s], (kb / S) & 1);
      ptx::tc_fence_after();
      const uint32_t a = ptx::smem_u32(ring + s * Cfg::kStageBytes);
      const uint32_t b = a + Cfg::kABytes;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        ptx::mma_bf16(acc1, ptx::smem_desc_sw128(a + kk * 32, 16, 1024),
                      ptx::smem_desc_sw128(b + kk * 32, 16, 1024), idesc1, (kb | kk) != 0);
      ptx::mma_commit(&empty_bar[s]);
    }
    ptx::mma_commit(acc1_bar);
  }
  __syncwarp();

  // y1 = act1(acc1 + b1) -> swizzled smem (GEMM 2's A operand), one row per thread
  ptx::mbar_wait(acc1_bar, 0);
  ptx::tc_fence_after();
  {
    const int rl = warp * 32 + lane;
    for (int c = 0; c < n1; c += 32) {
      uint32_t r[32];
      ptx::tmem_ld32(acc1 + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int col = c + 8 * q;
        const float4 b0 = __ldg(reinterpret_cast<const float4*>(fa.b1 + col));
        const float4 b1 = __ldg(reinterpret_cast<const float4*>(fa.b1 + col + 4));
        const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        uint4 packed;
        uint32_t* pw = reinterpret_cast<uint32_t*>(&packed);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 h =
              __floats2bfloat162_rn(act_fwd_t<ACT1>(__uint_as_float(r[8 * q + 2 * i]) + bb[2 * i]),
                                    act_fwd_t<ACT1>(__uint_as_float(r[8 * q + 2 * i + 1]) +
                                                    bb[2 * i + 1]));
          pw[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        const int tile = col / 64, chunk = (col % 64) / 8;
        *reinterpret_cast<uint4*>(sA2 + tile * Cfg::kA2Tile + rl * 128 +
                                  ((chunk ^ (rl & 7)) * 16)) = packed;
      }
    }
  }
  ptx::fence_proxy_async();  // generic smem writes -> UMMA / TMA reads
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  if (warp == 0 && lane == 0) {
    // y1 rows of this node only: the store map's row extent ends at its last row
    for (int j = 0; j < kb2; ++j)
      ptx::tma_store_2d(&tm_y1, sA2 + j * Cfg::kA2Tile, j * 64, fa.y1_row_off + m0);
    ptx::bulk_commit_group();
    if (blockIdx.x == 0 && ep2.tag_src && ep2.tag_dst) write_tags(ep2);
  } else if (warp == 1 && lane == 0) {
    ptx::mbar_wait(b2_bar, 0);
    ptx::tc_fence_after();
    const uint32_t idesc2 = ptx::idesc_bf16_f32(128, n2pad, false, false);
    for (int j = 0; j < kb2; ++j) {
      const uint32_t a = ptx::smem_u32(sA2 + j * Cfg::kA2Tile);
      const uint32_t b = ptx::smem_u32(sB2 + j * Cfg::kB2Blk);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        ptx::mma_bf16(acc2, ptx::smem_desc_sw128(a + kk * 32, 16, 1024),
                      ptx::smem_desc_sw128(b + kk * 32, 16, 1024), idesc2, (j | kk) != 0);
    }
    ptx::mma_commit(acc2_bar);
  }
  __syncwarp();

  // layer l's epilogue (bias + activation, or the fused softmax-CE)
  ptx::mbar_wait(acc2_bar, 0);
  ptx::tc_fence_after();
  const uint32_t t_row = acc2 + (static_cast<uint32_t>(warp * 32) << 16);
  float* T = reinterpret_cast<float*>(ring + 4 * Cfg::kA2Tile) + warp * 32 * kVecLd;
  if (ep2.rowwise == 2) {
    with_act<kEpiFwd>(ep2, [&](auto A) {
      epilogue_warp_vec<kEpiFwd, decltype(A)::value>(ep2, sh2, m0 + warp * 32, 0, n2pad, t_row, T);
    });
  } else {
    with_act<kEpiFwd>(ep2, [&](auto A) {
      epilogue_warp_rows<kEpiFwd, decltype(A)::value>(ep2, sh2, m0 + warp * 32, 0, n2pad, t_row);
    });
  }
  if (warp == 0 && lane == 0) ptx::bulk_wait_group<0>();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace pb

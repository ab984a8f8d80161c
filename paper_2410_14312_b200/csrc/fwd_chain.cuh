// Two consecutive Linear forwards of a stage in one kernel, for a stage
// whose last two layers are narrow: the first's output has n1 <= 256
// columns (a multiple of 64), the second's n2 <= 64 (trainer.cpp:179-206
// applied twice):
//
//   y1 = act1(x W1^T + b1)      rows x n1, K1 = in_{l-1}
//   y2 = epi2(y1 W2^T)          rows x n2, K2 = n1
//
// One cluster of C = n1 / 64 CTAs per 128 rows.  CTA c computes the 64
// columns [64c, 64c + 64) of y1 (a 6-deep TMA ring into TMEM), applies bias
// and activation, writes them as bf16 straight into shared memory in the
// 128B-swizzled K-major layout of GEMM 2's A operand and TMA-stores them
// (the backward reads y1); then GEMM 2 over its own 64-wide K slice gives a
// partial y2.  The C partials are summed over distributed shared memory in
// rank order (deterministic), each CTA finishing every C-th row with layer
// l's epilogue: bias + activation, or the logits with the softmax
// cross-entropy fused (EpiParams::loss_*).  On C1's stage 2 (512->256->10)
// this replaces two dependent launches of the pipeline's dependency cycle
// (DESIGN.md).
#pragma once

#include "gemm_sm100.cuh"

namespace pb {

struct FwdChainCfg {
  static constexpr int kStages = 6;
  static constexpr int kABytes = 128 * 64 * 2;  // x k-block
  static constexpr int kBBytes = 64 * 64 * 2;   // this CTA's 64 rows of W1
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kRing = kStages * kStageBytes;
  static constexpr int kA2 = 128 * 64 * 2;      // y1 slice, over the idle ring
  static constexpr int kPartLd = 64 + 4;        // partial y2 row stride (floats)
  static constexpr int kOffPart = kA2;
  static constexpr int kOffB2 = kRing;          // W2[:, 64c : 64c + 64] (n2 <= 64 rows)
  static constexpr int kOffBar = kOffB2 + 64 * 64 * 2;
  static constexpr int kSmem = kOffBar + 128 + 1024;
  static_assert(kOffPart + 128 * kPartLd * 4 <= kRing, "A2 + partials must fit the ring");
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
  float* part = reinterpret_cast<float*>(smem + Cfg::kOffPart);
  uint8_t* sB2 = smem + Cfg::kOffB2;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* b2_bar = empty_bar + S;
  uint64_t* acc1_bar = b2_bar + 1;
  uint64_t* acc2_bar = acc1_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc2_bar + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int C = static_cast<int>(gridDim.x);  // the cluster: one CTA per 64 columns of y1
  const int rank = static_cast<int>(ptx::cluster_ctarank());
  const int m0 = blockIdx.y * 128;
  const int n0 = rank * 64;
  const int n2pad = fa.n2pad;
  const int kb1 = (sh1.K + 63) / 64;

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
  if (warp == 2) ptx::tmem_alloc<128>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t acc1 = tmem_base, acc2 = tmem_base + 64;
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();

  if (warp == 0 && lane == 0) {
    ptx::mbar_arrive_expect_tx(b2_bar, n2pad * 128);
    ptx::tma_load_2d(sB2, &tm_w2, b2_bar, n0, 0);
    for (int kb = 0; kb < kb1; ++kb) {
      const int s = kb % S;
      if (kb >= S) ptx::mbar_wait(&empty_bar[s], ((kb / S) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&full_bar[s], Cfg::kStageBytes);
      uint8_t* st = ring + s * Cfg::kStageBytes;
      ptx::tma_load_2d(st, &tm_x, &full_bar[s], kb * 64, m0 + sh1.a_mn_off);
      ptx::tma_load_2d(st + Cfg::kABytes, &tm_w1, &full_bar[s], kb * 64, n0);
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc1 = ptx::idesc_bf16_f32(128, 64, false, false);
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

  // y1 slice = act1(acc1 + b1) -> swizzled smem (GEMM 2's A), one row per thread
  ptx::mbar_wait(acc1_bar, 0);
  ptx::tc_fence_after();
  const int rl = warp * 32 + lane;
#pragma unroll 1
  for (int c = 0; c < 64; c += 32) {
    uint32_t r[32];
    ptx::tmem_ld32(acc1 + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int col = c + 8 * q;
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(fa.b1 + n0 + col));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(fa.b1 + n0 + col + 4));
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
      *reinterpret_cast<uint4*>(sA2 + rl * 128 + (((col / 8) ^ (rl & 7)) * 16)) = packed;
    }
  }
  ptx::fence_proxy_async();  // generic smem writes -> UMMA / TMA reads
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  if (warp == 0 && lane == 0) {
    // y1 rows of this launch only: the store map's row extent ends at its last row
    ptx::tma_store_2d(&tm_y1, sA2, n0, fa.y1_row_off + m0);
    ptx::bulk_commit_group();
    if (rank == 0 && blockIdx.y == 0 && ep2.tag_src && ep2.tag_dst) write_tags(ep2);
  } else if (warp == 1 && lane == 0) {
    // partial y2 over this CTA's 64-wide K slice
    ptx::mbar_wait(b2_bar, 0);
    ptx::tc_fence_after();
    const uint32_t idesc2 = ptx::idesc_bf16_f32(128, n2pad, false, false);
    const uint32_t a = ptx::smem_u32(sA2), b = ptx::smem_u32(sB2);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      ptx::mma_bf16(acc2, ptx::smem_desc_sw128(a + kk * 32, 16, 1024),
                    ptx::smem_desc_sw128(b + kk * 32, 16, 1024), idesc2, kk != 0);
    ptx::mma_commit(acc2_bar);
  }
  __syncwarp();

  // park the partial (this thread's row) for the cluster's reduction
  ptx::mbar_wait(acc2_bar, 0);
  ptx::tc_fence_after();
#pragma unroll 1
  for (int c = 0; c < n2pad; c += 16) {
    uint32_t r[16];
    ptx::tmem_ld16(acc2 + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(part + rl * Cfg::kPartLd + c + 4 * i) =
          make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                      __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
  }
  ptx::cluster_sync();  // every partial of the row block is parked

  // rows rl = rank, rank + C, ...: sum the C partials in rank order, finish
  const int row = m0 + rl;
  if (rl % C == rank && row < sh2.M) {
    with_act<kEpiFwd>(ep2, [&](auto A) {
#pragma unroll 1
      for (int c = 0; c < n2pad; c += 16) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
        for (int j = 0; j < C; ++j) {
          const uint32_t src = ptx::map_to_rank(part + rl * Cfg::kPartLd + c, j);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 q = ptx::ld_dsmem_f4(src + 16 * i);
            v[4 * i] += q.x;
            v[4 * i + 1] += q.y;
            v[4 * i + 2] += q.z;
            v[4 * i + 3] += q.w;
          }
        }
        const int valid = sh2.N - c < 16 ? sh2.N - c : 16;
        if (valid <= 0) break;
        epilogue_chunk<kEpiFwd, decltype(A)::value>(ep2, sh2, m0 + rl, c, valid, v);
        if (ep2.loss_dz && c == 0 && sh2.N <= 16) fused_ce_row(ep2, m0 + rl, v, valid);
      }
    });
  }
  ptx::cluster_sync();  // peers read this CTA's partials until here
  if (warp == 0 && lane == 0) ptx::bulk_wait_group<0>();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<128>(tmem_base);
  }
}

}  // namespace pb

// Two consecutive dgrad GEMMs of a stage backward in one kernel, for a top
// layer l with a narrow output (K1 = out_l <= 64: one k-block) and an input
// of at most 256 columns (trainer.cpp:255-263 applied twice):
//
//   dz_{l-1} = (dz_l W_l) . act'_{l-1}        128 x n1, K1 <= 64
//   delta    = (dz_{l-1} W_{l-1}) . act'_gate   128 x BN tile, K2 = n1 <= 256
//
// Each CTA owns 128 rows and one BN-wide column tile of delta.  dz_{l-1}
// for its rows -- one k-block of MMAs into TMEM, the act' gate on the way
// out -- is written as bf16 straight into shared memory in the 128B-swizzled
// K-major layout the second GEMM's A operand needs, so it never makes an L2
// round trip before use.  With a cluster of C = n1 / 64 CTAs along the
// column tiles (ChainArgs::cluster), CTA r computes only the 64 columns
// [64r, 64r + 64) of dz_{l-1} (and TMA-stores them for the wgrad / bias of
// layer l-1 when it is in the first cluster of the row block), then copies
// its peers' slices over distributed shared memory into its own A tiles
// (plain loads and stores, then a proxy fence: the tensor core reads only
// locally written shared memory).  Without a cluster each CTA computes the
// whole 128 x n1 block and the column-tile-0 CTAs store it.
//
// On the C1 backward (784-512-256-10, stage 2 = [512->256, 256->10]) this
// replaces the 10-wide L3 dgrad launch on the pipeline's dependency cycle
// ("Where C1's 46 us go").
#pragma once

#include "gemm_sm100.cuh"

namespace pb {

template <int BN>
struct ChainCfg {
  static constexpr int kA1 = 128 * 64 * 2;        // dz_l tile (K-major)
  static constexpr int kB1 = 256 * 64 * 2;        // W_l: 4 boxes of 64 N x 64 K (MN-major)
  static constexpr int kA2Tile = 128 * 64 * 2;    // one k-block of dz_{l-1}
  static constexpr int kA2 = 4 * kA2Tile;         // up to 256 columns
  static constexpr int kB2Blk = BN * 64 * 2;      // one k-block of W_{l-1} (MN-major)
  static constexpr int kB2 = 4 * kB2Blk;
  static constexpr int kOffB1 = kA1;
  static constexpr int kOffA2 = kOffB1 + kB1;
  static constexpr int kOffB2 = kOffA2 + kA2;
  static constexpr int kOffBar = kOffB2 + kB2;
  static constexpr int kSmem = kOffBar + 64 + 1024;
  static_assert(kSmem <= 232448, "exceeds the 227 KB of shared memory per CTA");
  static_assert(4 * 32 * kVecLd * 4 <= kA1 + kB1, "epilogue staging must fit A1 + B1");
};

template <int BN>
__global__ void __launch_bounds__(128, 1)
    dgrad_chain_kernel(const __grid_constant__ CUtensorMap tm_a1,
                       const __grid_constant__ CUtensorMap tm_b1,
                       const __grid_constant__ CUtensorMap tm_b2,
                       const __grid_constant__ CUtensorMap tm_dz, GemmShape sh2, EpiParams ep2,
                       ChainArgs ca) {
  using Cfg = ChainCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA1 = smem;
  uint8_t* sB1 = smem + Cfg::kOffB1;
  uint8_t* sA2 = smem + Cfg::kOffA2;
  uint8_t* sB2 = smem + Cfg::kOffB2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);  // 0 A1/B1, 1 B2, 2 acc1, 3 acc2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * 128;
  const int n0 = blockIdx.x * BN;
  const int kb2 = (ca.n1 + 63) / 64;
  const int C = ca.cluster > 1 ? ca.cluster : 1;
  const int rank = C > 1 ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  const int t0 = C > 1 ? rank : 0, t1 = C > 1 ? rank + 1 : kb2;  // dz_{l-1} tiles built here
  const bool store = ca.store_dz && static_cast<int>(blockIdx.x) < C;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tm_a1);
    ptx::tma_prefetch_desc(&tm_b1);
    ptx::tma_prefetch_desc(&tm_b2);
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
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
    // operands of both GEMMs at once: at most 1 + 4 + 4 * BN / 64 boxes
    ptx::mbar_arrive_expect_tx(&bar[0], Cfg::kA1 + (t1 - t0) * 8192);
    ptx::tma_load_2d(sA1, &tm_a1, &bar[0], 0, m0);
    for (int h = t0; h < t1; ++h)
      ptx::tma_load_2d(sB1 + (h - t0) * 8192, &tm_b1, &bar[0], h * 64, 0);
    ptx::mbar_arrive_expect_tx(&bar[1], kb2 * Cfg::kB2Blk);
    for (int j = 0; j < kb2; ++j)
#pragma unroll
      for (int h = 0; h < BN / 64; ++h)
        ptx::tma_load_2d(sB2 + j * Cfg::kB2Blk + h * 8192, &tm_b2, &bar[1], n0 + h * 64, j * 64);
  } else if (warp == 1 && lane == 0) {
    // GEMM 1: 128 x 256 x K1 (one k-block; K1's zero-filled tail adds
    // nothing; columns past n1 are never read)
    ptx::mbar_wait(&bar[0], 0);
    ptx::tc_fence_after();
    const uint32_t idesc1 = ptx::idesc_bf16_f32(128, 64 * (t1 - t0), false, true);
    const uint32_t a = ptx::smem_u32(sA1), b = ptx::smem_u32(sB1);
    const int ksteps = (ca.k1 + 15) / 16;
    for (int kk = 0; kk < ksteps; ++kk)
      ptx::mma_bf16(acc1, ptx::smem_desc_sw128(a + kk * 32, 16, 1024),
                    ptx::smem_desc_sw128(b + kk * 2048, 8192, 1024), idesc1, kk != 0);
    ptx::mma_commit(&bar[2]);
  }
  __syncwarp();

  // dz_{l-1} rows -> shared memory (A operand of GEMM 2), one row per thread
  ptx::mbar_wait(&bar[2], 0);
  ptx::tc_fence_after();
  {
    const int rl = warp * 32 + lane;
    const int row = m0 + rl;
    const bool live = row < sh2.M;
    const __nv_bfloat16* xg = ca.x_gate + static_cast<size_t>(live ? row : 0) * ca.ld_gate;
    for (int c = 64 * t0; c < 64 * t1; c += 32) {
      uint32_t r[32];
      ptx::tmem_ld32(acc1 + (static_cast<uint32_t>(warp * 32) << 16) + (c - 64 * t0), r);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int col = c + 8 * q;
        uint4 packed = make_uint4(0u, 0u, 0u, 0u);
        if (live) {
          const uint4 xv = *reinterpret_cast<const uint4*>(xg + col);
          const __nv_bfloat16* xh = reinterpret_cast<const __nv_bfloat16*>(&xv);
          uint32_t* pw = reinterpret_cast<uint32_t*>(&packed);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float g0 = act_grad_from_out(__bfloat162float(xh[2 * i]), ca.act_gate);
            const float g1 = act_grad_from_out(__bfloat162float(xh[2 * i + 1]), ca.act_gate);
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[8 * q + 2 * i]) * g0,
                                                     __uint_as_float(r[8 * q + 2 * i + 1]) * g1);
            pw[i] = *reinterpret_cast<uint32_t*>(&h);
          }
        }
        const int tile = col / 64, chunk = (col % 64) / 8;
        *reinterpret_cast<uint4*>(sA2 + tile * Cfg::kA2Tile + rl * 128 +
                                  ((chunk ^ (rl & 7)) * 16)) = packed;
      }
    }
  }
  ptx::fence_proxy_async();  // the generic smem writes -> UMMA / TMA reads
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (C > 1) {
    // the peers' slices: DSMEM loads into this CTA's own A tiles (16 KB each)
    ptx::cluster_sync();
    for (int p = 0; p < C; ++p) {
      if (p == rank) continue;
      const uint32_t src = ptx::map_to_rank(sA2 + p * Cfg::kA2Tile, p);
      float4* dst = reinterpret_cast<float4*>(sA2 + p * Cfg::kA2Tile);
#pragma unroll
      for (int i = 0; i < Cfg::kA2Tile / 16 / 128; ++i) {
        const int e = i * 128 + static_cast<int>(threadIdx.x);
        dst[e] = ptx::ld_dsmem_f4(src + 16 * e);
      }
    }
    ptx::fence_proxy_async();
    ptx::cluster_sync();  // every peer's reads of this CTA's slice are done
    ptx::tc_fence_after();
  }

  if (warp == 0 && lane == 0) {
    if (store) {
      for (int j = t0; j < t1; ++j) ptx::tma_store_2d(&tm_dz, sA2 + j * Cfg::kA2Tile, j * 64, m0);
      ptx::bulk_commit_group();
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && ep2.tag_src && ep2.tag_dst)
      write_tags(ep2);
  } else if (warp == 1 && lane == 0) {
    // GEMM 2: 128 x BN x n1
    ptx::mbar_wait(&bar[1], 0);
    ptx::tc_fence_after();
    constexpr uint32_t idesc2 = ptx::idesc_bf16_f32(128, BN, false, true);
    for (int j = 0; j < kb2; ++j) {
      const uint32_t a = ptx::smem_u32(sA2 + j * Cfg::kA2Tile);
      const uint32_t b = ptx::smem_u32(sB2 + j * Cfg::kB2Blk);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        ptx::mma_bf16(acc2, ptx::smem_desc_sw128(a + kk * 32, 16, 1024),
                      ptx::smem_desc_sw128(b + kk * 2048, 8192, 1024), idesc2, (j | kk) != 0);
    }
    ptx::mma_commit(&bar[3]);
  }
  __syncwarp();

  // epilogue of GEMM 2: the regular dgrad vector epilogue (act' gate of the
  // layer below, bf16 delta), staged in the A1 / B1 area (GEMM 1 is done)
  ptx::mbar_wait(&bar[3], 0);
  ptx::tc_fence_after();
  float* T = reinterpret_cast<float*>(sA1) + warp * 32 * kVecLd;
  const uint32_t t_row = acc2 + (static_cast<uint32_t>(warp * 32) << 16);
  with_act<kEpiDgrad>(ep2, [&](auto A) {
    epilogue_warp_vec<kEpiDgrad, decltype(A)::value>(ep2, sh2, m0 + warp * 32, n0, BN, t_row, T);
  });
  if (warp == 0 && lane == 0 && store) ptx::bulk_wait_group<0>();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace pb

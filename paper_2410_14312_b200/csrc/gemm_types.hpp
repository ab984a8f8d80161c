// Plain (host-compilable) parameter types of the layer GEMMs.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

namespace pb {

enum Act : int { kLinear = 0, kRelu = 1, kTanh = 2, kSigmoid = 3 };
enum Epi : int { kEpiFwd = 0, kEpiDgrad = 1, kEpiWgradSgd = 2 };

// Problem extents plus TMA coordinate offsets (row offsets inside a larger
// buffer, e.g. micro-batch j of an activation slot).
struct GemmShape {
  int M, N, K;
  int a_mn_off, a_k_off;
  int b_mn_off, b_k_off;
  // split-K (forward, single-CTA kernel): the K range is cut into `splits`
  // chunks of kb_per_split 64-wide k-blocks, one CTA of a (1,1,splits)
  // cluster each (0/1 = no split); see gemm_sm100.cuh.
  int splits, kb_per_split;
  // Implicit-GEMM 3x3 convolution (pad 1, stride 1, NHWC bf16; pair kernel):
  //  1 forward: A = im2col(x) [pixels, 9*C] (tap-major K), B = W [Cout, 9*C]
  //  3 dgrad:   A = im2col(dz) with the taps flipped [pixels, 9*C],
  //             B = W viewed [Cout][9][Cin] (3-D map, MN-major)
  //  2 wgrad:   A = dz [pixels, Cout] (MN-major), B = im2col(x) (MN-major,
  //             64-pixel columns)
  //  4 wgrad, transposed (dW^T, for Cout < 256): A = im2col(x) (MN-major,
  //             M = 9*C), B = dz (MN-major, N = Cout)
  // conv_h / conv_w: image size; conv_c: channels of the im2col'd tensor.
  // a_mn_off (modes 1, 3) / b_k_off (mode 2) / a_k_off (mode 4) are pixel
  // offsets.
  int conv = 0, conv_h = 0, conv_w = 0, conv_c = 0;
  // Halo tiles (modes 1 and 3, image width a multiple of halo_tw): a CTA
  // covers halo_tw consecutive pixels of one image row (a strip); per
  // 64-channel chunk one TMA load brings the strip's 3-row halo patch
  // {64 ch, halo_tw + 2 px, 3 rows} (tensor map `ta`, 4-D tiled) and the 9
  // taps are 9 shifted views of it (the UMMA descriptor starts at any 128-byte
  // row of the swizzled patch: tools/umma_shift_probe.cu).  Strip g = GEMM
  // rows [g * halo_tw, (g + 1) * halo_tw); CTA rank r of pair tile t takes
  // strip 2t + r.  0 = im2col loads, one per tap.
  int halo_tw = 0;
};

// Tensor maps of the TMA epilogue of wgrad+SGD (EpiParams::rowwise == 3).
// fp32 masters: w_cur / w_new = current / new fp32 master (box 32 x 32,
// 128-byte swizzle), w16 = bf16 weights of the new version (box 32 x 64).
// Split masters (EpiParams::split_master): w_cur = hi of the current version
// (its bf16 weights), w_new = lo residual of the current version, w16 = hi of
// the new version, lo_new = its lo residual (all 16-bit, box 32 x 32, 64-byte
// swizzle).
struct alignas(64) EpiMaps {
  CUtensorMap w_cur, w_new, w16, lo_new;
};

struct EpiParams {
  // forward: y = act(acc + bias)
  const float* bias;
  int act;
  __nv_bfloat16* y16;
  int ld_y16;
  float* y32;
  int ld_y32;
  int y_row_off;
  // dgrad: d = acc * act'(xin)   (act' recovered from the stored activation)
  const __nv_bfloat16* xin;
  int ld_xin;
  int act_prev;
  __nv_bfloat16* d16;
  int ld_d16;
  // wgrad + SGD: w_new = w_cur - lr * acc ; w16 = bf16(w_new)
  const float* w_cur;
  float* w_new;
  int ld_w32;
  __nv_bfloat16* w16;
  int ld_w16;
  float lr;
  // version tag propagation (device-side version accounting): if both are
  // set, CTA (0,0) copies *tag_src into *tag_dst.
  const int* tag_src;
  int* tag_dst;
  int tag_count;   // entries written (a coalesced forward covers several micro-batches)
  int tag_stride;  // element stride between entries
  // epilogue access pattern: 0 = transposed (coalesced rows, lane = column),
  // 1 = row-per-thread vectors, 2 = staged transpose with 16/8-byte vectors,
  // 3 = (SGD, pair kernel) TMA loads/stores through swizzled smem
  int rowwise;
  int has_w16;  // TMA SGD epilogue: EpiMaps::w16 is valid
  // split fp32 masters: master(v) = bits(hi(v)) << 16 + lo(v), hi(v) the
  // version's bf16 GEMM operand, lo(v) a signed 16-bit residual (exact fp32;
  // 4 bytes per parameter in place of fp32 master + bf16 copy)
  int split_master;
  // timing experiments: nonzero skips the epilogue's global traffic
  int dbg_skip;
  // split-K into fp32 partial slabs (single-CTA kernel, forward epilogue
  // without bias / activation): split z writes y32 + z * partial_slab; a
  // separate in-order reduction consumes them (conv wgrad, conv_ops.cu)
  long long partial_slab;
  // split-K with an in-kernel fixup (forward, pair kernel): every split of a
  // tile stores its fp32 partial to fix_ws (its own slot, warp-blocked), then
  // bumps fix_cnt[tile * 2 + CTA rank]; the last to arrive sums the S
  // partials in split order (its own from TMEM) and runs the epilogue.  The
  // last arriver resets the counter, so it is zero between launches.
  float* fix_ws;
  int* fix_cnt;
  // softmax cross-entropy fused into the logits layer's forward epilogue
  // (class labels, linear head, N <= 16, the row-per-thread epilogue): per
  // row dz = (softmax - onehot) / loss_denom (bf16, row stride loss_ld_dz)
  // and the row's loss; rows indexed like y (y_row_off)
  const int* loss_labels;
  __nv_bfloat16* loss_dz;
  int loss_ld_dz;
  float* loss_row;
  float loss_denom;
};

// Where the fixup epilogue finds the partials of its tile (see EpiParams).
struct FixSrc {
  const float* base = nullptr;  // split 0's block of this warp
  long long stride = 0;         // floats between splits
  int S = 0, self = 0;
};


// Fused two-layer dgrad (dgrad_chain.cuh): the first GEMM's operands and
// act' gate; the second GEMM uses the plain dgrad GemmShape / EpiParams.
struct ChainArgs {
  const __nv_bfloat16* x_gate = nullptr;  // layer l's input = act_{l-1} output
  int ld_gate = 0;
  int act_gate = 0;  // activation of layer l-1
  int k1 = 0;        // out_l (<= 64)
  int n1 = 0;        // in_l = out_{l-1} (<= 256, multiple of 64)
  int store_dz = 1;  // write dz_{l-1} to global (column-tile 0 CTAs)
  int cluster = 1;   // CTAs per cluster along the column tiles (n1 / 64, or 1)
};


// Fused two-layer forward (fwd_chain.cuh): layer l-1's bias, layer l's
// padded width, and where y1 (layer l-1's output) rows start.
struct FwdChainArgs {
  const float* b1 = nullptr;
  int n2pad = 16;      // layer l's width rounded up to 16 (<= 64)
  int y1_row_off = 0;  // row of y1's buffer where this launch's rows start
};

}  // namespace pb

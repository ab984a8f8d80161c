// Layer kernels and their launchers: GEMM instantiations, fused loss,
// bias+SGD, and boundary conversions.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "gemm_sm100.cuh"
#include "dgrad_chain.cuh"
#include "fwd_chain.cuh"
#include "layer_ops.cuh"
#include "conv_ops.cuh"
#include "status.hpp"

namespace pb {

// ------------------------------------------------------------ tensor maps
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    PB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p,
                                    cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr)
      throw cuda_failure("cuTensorMapEncodeTiled entry point unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace

CUtensorMap make_operand_tmap(const Mat16& m, bool k_major, int box_mn) {
  if ((m.ld % 8) != 0)
    throw std::invalid_argument("bf16 leading dimension must be a multiple of 8");
  if ((reinterpret_cast<uintptr_t>(m.ptr) & 15) != 0)
    throw std::invalid_argument("bf16 operand must be 16-byte aligned");
  CUtensorMap map;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(m.cols),
                        static_cast<cuuint64_t>(m.rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(m.ld) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(k_major ? box_mn : 64)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(
      &map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
      const_cast<void*>(static_cast<const void*>(m.ptr)), dims, strides, box,
      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw cuda_failure("cuTensorMapEncodeTiled failed (code " +
                       std::to_string(static_cast<int>(r)) + ")");
  return map;
}

// MN-major operand in 32-column boxes, 64-byte swizzle (32-wide tiles)
CUtensorMap make_operand_tmap_mn32(const Mat16& m) {
  if ((m.ld % 8) != 0) throw std::invalid_argument("bf16 leading dimension must be a multiple of 8");
  CUtensorMap map;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(m.cols), static_cast<cuuint64_t>(m.rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(m.ld) * 2};
  cuuint32_t box[2] = {32, 64};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(
      &map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
      const_cast<void*>(static_cast<const void*>(m.ptr)), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw cuda_failure("cuTensorMapEncodeTiled (32-wide) failed (code " +
                       std::to_string(static_cast<int>(r)) + ")");
  return map;
}

// Epilogue tensor maps of the TMA SGD epilogue: 2-D row-major, box 32 rows x
// box_cols (32 fp32 master columns; 64 bf16 columns: one 128-byte row).
CUtensorMap make_epi_tmap(const void* ptr, CUtensorMapDataType dt, int elem_bytes, int rows,
                          int cols, int ld, CUtensorMapSwizzle swz, int box_cols = 32) {
  CUtensorMap map;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * elem_bytes};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw cuda_failure("cuTensorMapEncodeTiled (epilogue) failed (code " +
                       std::to_string(static_cast<int>(r)) + ")");
  return map;
}

// Kernel choice.  Tall problems (M > 128) use the persistent CTA-pair kernel
// (256 x BN tiles, overlapped epilogue); M <= 128 (micro-batch forwards of
// <=128 rows, tiny nets) use the single-CTA 128 x BN kernel.
// PIPESIM_GEMM=single forces the single-CTA kernel (A/B comparisons).
namespace {
bool pair_allowed() {
  static const bool ok = [] {
    const char* e = std::getenv("PIPESIM_GEMM");
    return !(e && std::string(e) == "single");
  }();
  return ok;
}
}  // namespace

int pick_bn(int M, int N) {
  if (M > 128 && pair_allowed()) {
    // a pair GEMM with fewer than 16 256-wide tiles (a small network:
    // latency-bound) takes 128-wide tiles, twice the SMs -- C1 55.5 -> 47.4
    // us per mini-batch; the 16 x 4096 shapes have >= 16 tiles
    // (PIPESIM_SMALL_TILES=N: the threshold, 0 = off)
    static const int small = [] {
      const char* e = std::getenv("PIPESIM_SMALL_TILES");
      return e ? std::atoi(e) : 16;
    }();
    const long tiles256 = static_cast<long>((M + 255) / 256) * ((N + 255) / 256);
    if (N > 128 && tiles256 < small) return 128;
    return N > 128 ? 256 : 128;
  }
  const long tiles256 = static_cast<long>((M + 127) / 128) * ((N + 255) / 256);
  if (N > 128 && tiles256 >= 132) return 256;
  // a single-CTA GEMM with fewer than PIPESIM_BN64 128-wide tiles (a micro-
  // batch of <= 128 rows in a small network: latency-bound) takes 64-wide
  // tiles, twice the SMs, half the B bytes per k-block -- C1 47.2 -> 46.4 us
  // per mini-batch (tools/gpu/r2_bn64.sh; 0 = off)
  static const int small64 = [] {
    const char* e = std::getenv("PIPESIM_BN64");
    return e ? std::atoi(e) : 8;
  }();
  const long tiles128 = static_cast<long>((M + 127) / 128) * ((N + 127) / 128);
  if (tiles128 < small64) return 64;
  return 128;
}

static bool use_pair(int M) { return M > 128 && pair_allowed(); }

// A pair forward with at most 64 output columns (VGG's 64-channel convs,
// the first conv's im2col GEMM) takes 64-wide tiles instead of computing a
// half-empty 128-wide one (PIPESIM_PAIR_BN64=0: off)
static bool pair_bn64(int N) {
  static const bool on = [] {
    const char* e = std::getenv("PIPESIM_PAIR_BN64");
    return !(e && std::string(e) == "0");
  }();
  return on && N <= 64;
}

namespace {

// PIPESIM_PDL=0/1 forces programmatic dependent launch of the GEMMs off /
// on (else GemmLaunch::pdl, chosen by the executor)
bool pdl_on(const GemmLaunch& g) {
  static const int env = [] {
    const char* e = std::getenv("PIPESIM_PDL");
    return e ? std::atoi(e) : -1;
  }();
  return env >= 0 ? env != 0 : g.pdl;
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
void launch_one(const GemmLaunch& g, cudaStream_t st) {
  init_gemm_attributes();
  if (g.pair) {
    // 64-wide pair tiles: forward (K-major B) only, no split-K / halo
    if constexpr (BN >= 128 || (BN == 64 && !A_MN && !B_MN && EPI == kEpiFwd) ||
                  (BN == 64 && !A_MN && B_MN && EPI == kEpiDgrad)) {
    auto kern = gemm_bf16_tcgen05_pair<BN, A_MN, B_MN, EPI, false>;
    if constexpr (EPI != kEpiWgradSgd && BN >= 128)
      if (g.ext) kern = gemm_bf16_tcgen05_pair<BN, A_MN, B_MN, EPI, true>;
    if (BN < 128 && g.ext) throw std::logic_error("64-wide pair tiles: no split-K / halo");
    constexpr int smem = Gemm2Cfg<BN, EPI>::kSmem;
    const int tiles_m = g.sh.halo_tw ? (g.sh.M / g.sh.halo_tw + 1) / 2 : (g.sh.M + 255) / 256;
    const int tiles = tiles_m * ((g.sh.N + BN - 1) / BN);
    int cap = sm_count() / 2;
    if (const char* e = std::getenv("PIPESIM_MAXPAIRS")) cap = std::min(cap, std::atoi(e));
    // PIPESIM_TILES_PER_PAIR=t (fwd/dgrad): at least t tiles per CTA pair,
    // so the double-buffered accumulator overlaps one tile's epilogue with
    // the next one's mainloop (fewer SMs per launch, more launches side by side)
    static const int tpp = [] {
      const char* e = std::getenv("PIPESIM_TILES_PER_PAIR");
      return e ? std::max(1, std::atoi(e)) : 1;
    }();
    if (EPI != kEpiWgradSgd && tpp > 1) cap = std::min(cap, (tiles + tpp - 1) / tpp);
    const int units =
        tiles * ((g.ep.partial_slab || g.ep.fix_cnt) ? std::max(1, g.sh.splits) : 1);
    const int pairs = std::min(units, std::max(1, cap));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(Gemm2Cfg<BN, EPI>::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on(g) ? 1 : 0;
    PB_CUDA(cudaLaunchKernelEx(&cfg, kern, g.ta, g.tb, g.sh, g.ep, g.maps));
    } else {
      throw std::logic_error("64-wide pair tiles: forward only");
    }
  } else if constexpr (BN <= 256) {
    auto kern = gemm_bf16_tcgen05<BN, A_MN, B_MN, EPI>;
    constexpr int smem = GemmCfg<BN>::kSmem;
    const int splits = std::max(1, g.sh.splits);
    dim3 grid((g.sh.N + BN - 1) / BN, (g.sh.M + 127) / 128, splits);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (splits > 1 && !g.ep.partial_slab) {  // the splits of a tile are one cluster (DSMEM reduction)
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = 1;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = splits;
      ++na;
    }
    if (pdl_on(g)) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    PB_CUDA(cudaLaunchKernelEx(&cfg, kern, g.ta, g.tb, g.sh, g.ep, g.maps));
  }
  PB_CUDA(cudaGetLastError());
}

template <int BN, bool A_MN, bool B_MN, int EPI>
void set_attr() {
  if constexpr (BN <= 256)
    PB_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, A_MN, B_MN, EPI>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 GemmCfg<BN>::kSmem));
  if constexpr (BN < 128) {  // single-CTA, plus the forward / conv-dgrad pair kernel
    if constexpr (!A_MN && ((!B_MN && EPI == kEpiFwd) || (B_MN && EPI == kEpiDgrad)))
      PB_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_pair<BN, A_MN, B_MN, EPI, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   Gemm2Cfg<BN, EPI>::kSmem));
  } else {
  PB_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_pair<BN, A_MN, B_MN, EPI, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Gemm2Cfg<BN, EPI>::kSmem));
  if constexpr (EPI != kEpiWgradSgd)
    PB_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_pair<BN, A_MN, B_MN, EPI, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Gemm2Cfg<BN, EPI>::kSmem));
  }
}

template <bool A_MN, bool B_MN, int EPI>
void launch_bn(const GemmLaunch& g, cudaStream_t st) {
  if constexpr (EPI != kEpiWgradSgd)
    if (g.bn == 512) return launch_one<512, A_MN, B_MN, EPI>(g, st);
  if constexpr (EPI == kEpiWgradSgd) {
    if (g.bn == 32 && !g.pair) return launch_one<32, A_MN, B_MN, EPI>(g, st);
  }
  if (g.bn == 256)
    launch_one<256, A_MN, B_MN, EPI>(g, st);
  else if (g.bn == 64)
    launch_one<64, A_MN, B_MN, EPI>(g, st);
  else
    launch_one<128, A_MN, B_MN, EPI>(g, st);
}

}  // namespace

void init_gemm_attributes() {
  static std::once_flag once;
  std::call_once(once, [] {
    set_attr<128, false, false, kEpiFwd>();
    set_attr<256, false, false, kEpiFwd>();
    set_attr<512, false, false, kEpiFwd>();
    set_attr<512, false, true, kEpiDgrad>();
    set_attr<128, false, true, kEpiDgrad>();
    set_attr<256, false, true, kEpiDgrad>();
    set_attr<64, false, false, kEpiFwd>();
    set_attr<64, false, true, kEpiDgrad>();
    set_attr<64, true, true, kEpiWgradSgd>();
    set_attr<32, true, true, kEpiWgradSgd>();
    set_attr<128, true, true, kEpiWgradSgd>();
    set_attr<256, true, true, kEpiWgradSgd>();
    // conv wgrad: split-K partial slabs (single-CTA, MN / MN operands)
    set_attr<128, true, true, kEpiFwd>();
    set_attr<256, true, true, kEpiFwd>();
  });
}

namespace {

// PIPESIM_EPI=rows|tile|vec (default vec: staged transpose, 16/8-byte
// vectors, 4 row segments per warp instruction; see gemm_sm100.cuh).
int epi_mode() {
  static const int m = [] {
    const char* e = std::getenv("PIPESIM_EPI");
    if (e && std::string(e) == "rows") return 1;
    if (e && std::string(e) == "tile") return 0;
    return 2;
  }();
  return m;
}

// PIPESIM_DBG_EPI=1: epilogues skip all global traffic (timing experiments
// only: results are garbage).
int dbg_skip() {
  static const int v = [] {
    const char* e = std::getenv("PIPESIM_DBG_EPI");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

EpiParams empty_epi(int kind) {
  EpiParams e{};
  const int m = epi_mode();
  e.rowwise = m;
  e.dbg_skip = dbg_skip();
  return e;
}

// The vector epilogue (mode 2) needs 16-byte fp32 rows and 8-byte bf16 rows;
// other layouts fall back to the scalar transposed (SGD) / row-per-thread
// (bf16 outputs) epilogues.
bool al(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }
void vec_or_fallback(EpiParams& e, int kind) {
  if (e.rowwise != 2) return;
  bool ok = true;
  if (kind == kEpiFwd) {
    if (e.y16) ok = ok && e.ld_y16 % 4 == 0 && al(e.y16, 8);
    if (e.y32) ok = ok && e.ld_y32 % 4 == 0 && al(e.y32, 16);
    if (e.bias) ok = ok && al(e.bias, 16);
  } else if (kind == kEpiDgrad) {
    ok = e.ld_d16 % 4 == 0 && al(e.d16, 8);
    if (e.act_prev != kLinear) ok = ok && e.ld_xin % 4 == 0 && al(e.xin, 8);
  } else {
    ok = e.ld_w32 % 4 == 0 && al(e.w_cur, 16) && al(e.w_new, 16);
    if (e.w16) ok = ok && e.ld_w16 % 4 == 0 && al(e.w16, 8);
  }
  if (!ok) e.rowwise = kind == kEpiWgradSgd ? 0 : 1;
}

// B-operand box rows for a K-major B: the pair kernel loads half a tile.
int b_box(const GemmLaunch& g) { return g.pair ? std::min(g.bn, 256) / 2 : g.bn; }

// 256 x 512 pair tiles (two MMAs per k-block sharing A) for wide layers
// with at least PIPESIM_BN512_ROWS rows (default 512: below that the halved
// CTA count costs more latency than the lower feed per flop saves; measured
// 567k vs 561k samples/s with all rows); PIPESIM_BN512=0 turns them off.
bool wide_tiles(int rows, int N) {
  static const bool on = [] {
    const char* e = std::getenv("PIPESIM_BN512");
    return !(e && std::string(e) == "0");
  }();
  static const int min_rows = [] {
    const char* e = std::getenv("PIPESIM_BN512_ROWS");
    return e ? std::atoi(e) : 512;
  }();
  return on && rows >= min_rows && N >= 1024 && N % 512 == 0;
}

}  // namespace

// PIPESIM_SPLITK=0 disables split-K, =<n> forces n splits (A/B runs).
namespace {
int splitk_env() {
  static const int v = [] {
    const char* e = std::getenv("PIPESIM_SPLITK");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}
}  // namespace


// Split-K for skinny forwards (<= 256 rows): enough 128 x 128 tiles x splits
// to cover the SMs, >= 8 k-blocks per split (PIPESIM_SPLITK_MINKB; 4 k-blocks
// made C1's 784-wide forwards split and its mini-batch slower, 58.9 -> 65.4
// us), at most 4.  PIPESIM_SPLITK=0 disables it, =<n> forces n (A/B runs).
int fwd_splits(int rows, int N, int K) {
  if (rows > 256 || splitk_env() == 0 || !pair_allowed()) return 1;
  const int kb = (K + 63) / 64;
  const int tiles = ((rows + 127) / 128) * ((N + 127) / 128);
  int s = std::max(1, sm_count() / tiles);
  if (splitk_env() > 0) s = splitk_env();
  static const int min_kb = [] {
    const char* e = std::getenv("PIPESIM_SPLITK_MINKB");
    return e ? std::max(1, std::atoi(e)) : 8;
  }();
  s = std::min(s, std::min(4, kb / min_kb));
  if (s == 3) s = 2;  // column blocks of the reduction: 128 / s, a multiple of 16
  return std::max(1, s);
}

// Pair forward with the in-kernel split-K fixup (EpiParams::fix_cnt): the
// tile width the forward would use and the split count that makes its tiles
// fill one wave of CTA pairs (>= 8 k-blocks per split); 1 = no split.
// Opt-in (PIPESIM_FWD_FIX=1 automatic split count, =<n> forces n > 1): the
// last arriver's partial reads are latency-bound (26.7 us for a 256 x 4096 x
// 4096 forward against 18 us for the single-CTA cluster split), so the
// cluster split stays the default.
namespace {
int fix_env() {
  static const int v = [] {
    const char* e = std::getenv("PIPESIM_FWD_FIX");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}
int fix_bn(int rows, int N) {
  int bn = N > 128 ? 256 : 128;
  if (rows > 128 && wide_tiles(rows, N)) bn = 512;
  return bn;
}
int fix_splits(int rows, int N, int K, int bn) {
  if (!pair_allowed() || splitk_env() == 0) return 1;
  const int tiles = ((rows + 255) / 256) * ((N + bn - 1) / bn);
  const int kb = (K + 63) / 64;
  const int pairs = sm_count() / 2;
  if (fix_env() < 1) return 1;
  int S = fix_env() > 1 ? fix_env() : (tiles * 4 >= pairs * 3 ? 1 : pairs / tiles);
  S = std::max(1, std::min(S, kb / 8));
  const int kbps = (kb + S - 1) / S;
  return (kb + kbps - 1) / kbps;
}
}  // namespace

size_t fwd_fix_floats(int rows, int N, int K) {
  const int bn = fix_bn(rows, N);
  const int S = fix_splits(rows, N, K, bn);
  if (S <= 1) return 0;
  return static_cast<size_t>(S) * ((rows + 255) / 256) * 256 * (((N + bn - 1) / bn) * bn);
}

int fwd_fix_counters(int rows, int N) { return 2 * ((rows + 255) / 256) * ((N + 127) / 128); }

GemmLaunch plan_fwd(const Mat16& x, int x_row_off, int rows, const Mat16& w,
                    const float* bias, int act, __nv_bfloat16* y16, int ld_y16,
                    float* y32, int ld_y32, int y_row_off, bool allow_split, bool verify,
                    float* fix_ws, int* fix_cnt) {
  GemmLaunch g;
  if (verify) {
    g.simt = true;
    g.simt_a = reinterpret_cast<const float*>(x.ptr);
    g.simt_lda = x.ld;
    g.simt_b = reinterpret_cast<const float*>(w.ptr);
    g.simt_ldb = w.ld;
    g.sh = GemmShape{rows, w.rows, x.cols, x_row_off, 0, 0, 0, 1, 0};
    g.ep = EpiParams{};
    g.ep.bias = bias;
    g.ep.act = act;
    g.ep.y16 = y16;
    g.ep.ld_y16 = ld_y16;
    g.ep.y32 = y32;
    g.ep.ld_y32 = ld_y32;
    g.ep.y_row_off = y_row_off;
    return g;
  }
  // one stage per GPU (latency): CTA-pair split-K with the in-kernel fixup
  // when a workspace is given, else the single-CTA cluster split
  int fix = 1;
  const int fbn = fix_bn(rows, w.rows);
  if (allow_split && fix_ws && fix_cnt) fix = fix_splits(rows, w.rows, x.cols, fbn);
  if (fix > 1) {
    g.bn = fbn;
    g.pair = true;
    g.ta = make_operand_tmap(x, /*k_major=*/true, 128);
    g.tb = make_operand_tmap(w, /*k_major=*/true, b_box(g));
    g.sh = GemmShape{rows, w.rows, x.cols, x_row_off, 0, 0, 0, fix, 0};
    const int kb = (x.cols + 63) / 64;
    g.sh.kb_per_split = (kb + fix - 1) / fix;
    g.ep = empty_epi(kEpiFwd);
    g.ep.bias = bias;
    g.ep.act = act;
    g.ep.y16 = y16;
    g.ep.ld_y16 = ld_y16;
    g.ep.y32 = y32;
    g.ep.ld_y32 = ld_y32;
    g.ep.y_row_off = y_row_off;
    vec_or_fallback(g.ep, kEpiFwd);
    if (g.ep.rowwise == 2 && !g.ep.dbg_skip) {  // the fixup runs the vector epilogue
      g.ep.fix_ws = fix_ws;
      g.ep.fix_cnt = fix_cnt;
      g.ext = true;
      return g;
    }
  }
  const int splits = allow_split || splitk_env() > 0 ? fwd_splits(rows, w.rows, x.cols) : 1;
  if (splits > 1) {  // single-CTA 128 x 128 tiles, one cluster of `splits` per tile
    g.bn = 128;
    g.pair = false;
  } else {
    g.bn = pick_bn(rows, w.rows);
    g.pair = use_pair(rows);
    if (g.pair && wide_tiles(rows, w.rows)) g.bn = 512;
    if (g.pair && pair_bn64(w.rows)) g.bn = 64;
  }
  g.ta = make_operand_tmap(x, /*k_major=*/true, 128);
  g.tb = make_operand_tmap(w, /*k_major=*/true, b_box(g));
  g.sh = GemmShape{rows, w.rows, x.cols, x_row_off, 0, 0, 0, 1, 0};
  if (splits > 1) {
    const int kb = (x.cols + 63) / 64;
    g.sh.kb_per_split = (kb + splits - 1) / splits;
    g.sh.splits = (kb + g.sh.kb_per_split - 1) / g.sh.kb_per_split;
  }
  g.ep = empty_epi(kEpiFwd);
  g.ep.bias = bias;
  g.ep.act = act;
  g.ep.y16 = y16;
  g.ep.ld_y16 = ld_y16;
  g.ep.y32 = y32;
  g.ep.ld_y32 = ld_y32;
  g.ep.y_row_off = y_row_off;
  vec_or_fallback(g.ep, kEpiFwd);
  return g;
}

GemmLaunch plan_dgrad(const Mat16& dz, const Mat16& w, const __nv_bfloat16* xin,
                      int ld_xin, int act_prev, __nv_bfloat16* d, int ld_d, bool verify) {
  GemmLaunch g;
  if (verify) {
    g.simt = true;
    g.simt_a = reinterpret_cast<const float*>(dz.ptr);
    g.simt_lda = dz.ld;
    g.simt_b = reinterpret_cast<const float*>(w.ptr);
    g.simt_ldb = w.ld;
    g.sh = GemmShape{dz.rows, w.cols, dz.cols, 0, 0, 0, 0, 1, 0};
    g.ep = EpiParams{};
    g.ep.xin = xin;
    g.ep.ld_xin = ld_xin;
    g.ep.act_prev = act_prev;
    g.ep.d16 = d;
    g.ep.ld_d16 = ld_d;
    return g;
  }
  g.bn = pick_bn(dz.rows, w.cols);
  g.pair = use_pair(dz.rows);
  // (PIPESIM_BN512_DGRAD=0: dgrad keeps 256-wide tiles, twice the SMs)
  static const bool dgrad_wide = [] {
    const char* e = std::getenv("PIPESIM_BN512_DGRAD");
    return !(e && std::string(e) == "0");
  }();
  if (g.pair && dgrad_wide && wide_tiles(dz.rows, w.cols)) g.bn = 512;
  g.ta = make_operand_tmap(dz, /*k_major=*/true, 128);
  g.tb = make_operand_tmap(w, /*k_major=*/false, 64);
  g.sh = GemmShape{dz.rows, w.cols, dz.cols, 0, 0, 0, 0};
  g.ep = empty_epi(kEpiDgrad);
  g.ep.xin = xin;
  g.ep.ld_xin = ld_xin;
  g.ep.act_prev = act_prev;
  g.ep.d16 = d;
  g.ep.ld_d16 = ld_d;
  vec_or_fallback(g.ep, kEpiDgrad);
  return g;
}

// Latency-bound networks (layers <= 1024 wide): the wgrad+SGD of a layer
// runs on the single-CTA kernel with 64-wide tiles -- for C1's 512 x 784
// layer 52 CTAs each updating 8K parameters instead of 14 CTA pairs each
// updating 32K; the update, not the flops, is the critical path there (C1
// 41.9 -> 39.1 us per mini-batch, C2 sequential 44.1 -> 39.2 us,
// tools/gpu/r2_wgsingle.sh).  PIPESIM_WGRAD_SINGLE=0|64|128 overrides.
int latency_wgrad_bn(int out, int in) {
  static const int env = [] {
    const char* e = std::getenv("PIPESIM_WGRAD_SINGLE");
    return e ? std::atoi(e) : -1;
  }();
  (void)out;
  (void)in;
  if (env == 0 || env == 32 || env == 64 || env == 128) return env;
  return 64;
}

GemmLaunch plan_wgrad_sgd(const Mat16& dz, const Mat16& x, int x_row_off,
                          const float* w_cur, float* w_new, int ld_w32,
                          __nv_bfloat16* w16, int ld_w16, float lr, bool verify,
                          int single_bn) {
  GemmLaunch g;
  if (verify) {
    g.simt = true;
    g.simt_a = reinterpret_cast<const float*>(dz.ptr);
    g.simt_lda = dz.ld;
    g.simt_b = reinterpret_cast<const float*>(x.ptr);
    g.simt_ldb = x.ld;
    g.sh = GemmShape{dz.cols, x.cols, dz.rows, 0, 0, 0, x_row_off, 1, 0};
    g.ep = EpiParams{};
    g.ep.w_cur = w_cur;
    g.ep.w_new = w_new;
    g.ep.ld_w32 = ld_w32;
    g.ep.w16 = w16;
    g.ep.ld_w16 = ld_w16;
    g.ep.lr = lr;
    return g;
  }
  g.bn = single_bn > 0 ? single_bn : pick_bn(dz.cols, x.cols);
  g.pair = single_bn > 0 ? false : use_pair(dz.cols);
  g.ta = make_operand_tmap(dz, /*k_major=*/false, 64);
  g.tb = g.bn == 32 ? make_operand_tmap_mn32(x) : make_operand_tmap(x, /*k_major=*/false, 64);
  g.sh = GemmShape{dz.cols, x.cols, dz.rows, 0, 0, 0, x_row_off};
  g.ep = empty_epi(kEpiWgradSgd);
  g.ep.w_cur = w_cur;
  g.ep.w_new = w_new;
  g.ep.ld_w32 = ld_w32;
  g.ep.w16 = w16;
  g.ep.ld_w16 = ld_w16;
  g.ep.lr = lr;
  vec_or_fallback(g.ep, kEpiWgradSgd);
  // pair kernel: TMA epilogue when the masters / bf16 rows are 16-byte
  // strided and aligned (PIPESIM_EPI=vec|tile|rows keeps the others)
  static const bool tma_ok = [] {
    const char* e = std::getenv("PIPESIM_EPI");
    return !(e && std::string(e) == "vec");
  }();
  if (g.pair && g.ep.rowwise == 2 && tma_ok && ld_w32 % 4 == 0 &&
      al(w_cur, 16) && al(w_new, 16) && (!w16 || (ld_w16 % 8 == 0 && al(w16, 16)))) {
    const int M = dz.cols, N = x.cols;
    g.maps.w_cur = make_epi_tmap(w_cur, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, N, ld_w32,
                                 CU_TENSOR_MAP_SWIZZLE_128B);
    g.maps.w_new = make_epi_tmap(w_new, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, N, ld_w32,
                                 CU_TENSOR_MAP_SWIZZLE_128B);
    if (w16)
      g.maps.w16 = make_epi_tmap(w16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, N, ld_w16,
                                 CU_TENSOR_MAP_SWIZZLE_128B, 64);
    g.ep.has_w16 = w16 ? 1 : 0;
    g.ep.rowwise = 3;
  }
  return g;
}

namespace {
bool tma_epilogue_on() {
  static const bool ok = [] {
    const char* e = std::getenv("PIPESIM_EPI");
    return !(e && (std::string(e) == "vec" || std::string(e) == "rows" ||
                   std::string(e) == "tile"));
  }();
  return ok;
}
}  // namespace

bool split_master_eligible(int out, int in, int ld) {
  static const bool on = [] {
    const char* e = std::getenv("PIPESIM_SPLIT_MASTER");
    return !(e && std::string(e) == "0");
  }();
  return on && tma_epilogue_on() && use_pair(out) && ld % 8 == 0 && in > 0;
}

GemmLaunch plan_wgrad_sgd_split(const Mat16& dz, const Mat16& x, int x_row_off,
                                const __nv_bfloat16* hi_cur, const uint16_t* lo_cur,
                                __nv_bfloat16* hi_new, uint16_t* lo_new, int ld, float lr) {
  const int M = dz.cols, N = x.cols;
  if (!split_master_eligible(M, N, ld) || !al(hi_cur, 16) || !al(lo_cur, 16) ||
      !al(hi_new, 16) || !al(lo_new, 16))
    throw std::invalid_argument("plan_wgrad_sgd_split: layer not eligible for split masters");
  GemmLaunch g;
  g.bn = pick_bn(M, N);
  g.pair = true;
  g.ta = make_operand_tmap(dz, /*k_major=*/false, 64);
  g.tb = make_operand_tmap(x, /*k_major=*/false, 64);
  g.sh = GemmShape{M, N, dz.rows, 0, 0, 0, x_row_off};
  g.ep = empty_epi(kEpiWgradSgd);
  g.ep.w16 = hi_new;
  g.ep.ld_w16 = ld;
  g.ep.lr = lr;
  g.ep.has_w16 = 1;
  g.ep.split_master = 1;
  g.ep.rowwise = 3;
  g.maps.w_cur = make_epi_tmap(hi_cur, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, N, ld,
                               CU_TENSOR_MAP_SWIZZLE_64B);
  g.maps.w_new = make_epi_tmap(lo_cur, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, M, N, ld,
                               CU_TENSOR_MAP_SWIZZLE_64B);
  g.maps.w16 = make_epi_tmap(hi_new, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, N, ld,
                             CU_TENSOR_MAP_SWIZZLE_64B);
  g.maps.lo_new = make_epi_tmap(lo_new, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, M, N, ld,
                                CU_TENSOR_MAP_SWIZZLE_64B);
  return g;
}

namespace {
// one row per blockIdx.y step, columns across threads (no per-element
// division; this runs once per parameter upload / read-back)
__global__ void split_master_kernel(const float* __restrict__ w, int rows, int cols, int ld_w,
                                    __nv_bfloat16* __restrict__ hi, uint16_t* __restrict__ lo,
                                    int ld) {
  for (int r = blockIdx.y; r < rows; r += gridDim.y)
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
      uint32_t h, l;
      split_master(w[static_cast<size_t>(r) * ld_w + c], h, l);
      reinterpret_cast<uint16_t*>(hi)[static_cast<size_t>(r) * ld + c] = static_cast<uint16_t>(h);
      lo[static_cast<size_t>(r) * ld + c] = static_cast<uint16_t>(l);
    }
}
__global__ void join_master_kernel(const __nv_bfloat16* __restrict__ hi,
                                   const uint16_t* __restrict__ lo, int rows, int cols, int ld,
                                   float* __restrict__ w, int ld_w) {
  for (int r = blockIdx.y; r < rows; r += gridDim.y)
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x)
      w[static_cast<size_t>(r) * ld_w + c] =
          join_master(reinterpret_cast<const uint16_t*>(hi)[static_cast<size_t>(r) * ld + c],
                      lo[static_cast<size_t>(r) * ld + c]);
}
dim3 conv_grid(int rows, int cols) {
  return dim3(static_cast<unsigned>(std::max(1, std::min((cols + 255) / 256, 16))),
              static_cast<unsigned>(std::max(1, std::min(rows, 148 * 8))));
}
}  // namespace

void launch_split_master(cudaStream_t st, const float* w, int rows, int cols, int ld_w,
                         __nv_bfloat16* hi, uint16_t* lo, int ld) {
  split_master_kernel<<<conv_grid(rows, cols), 256, 0, st>>>(w, rows, cols, ld_w, hi, lo, ld);
  PB_CUDA(cudaGetLastError());
}
void launch_join_master(cudaStream_t st, const __nv_bfloat16* hi, const uint16_t* lo, int rows,
                        int cols, int ld, float* w, int ld_w) {
  join_master_kernel<<<conv_grid(rows, cols), 256, 0, st>>>(hi, lo, rows, cols, ld, w, ld_w);
  PB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------ conv plans
namespace {
PFN_cuTensorMapEncodeIm2col_v12000 im2col_encode_fn() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    PB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr)
      throw cuda_failure("cuTensorMapEncodeIm2col entry point unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  });
  return fn;
}

// im2col view of an NHWC tensor for 3x3 / pad 1 / stride 1: the window of
// output pixel (h, w) starts at input (h - 1, w - 1); the bounding box of
// start positions is [-1, H - 2] x [-1, W - 2] (corners -1 / -1), so the
// pixels walked are exactly the output pixels, image after image.
CUtensorMap make_im2col_tmap(const Nhwc& t, int pixels_per_column) {
  if (t.c % 64 != 0) throw std::invalid_argument("im2col operand: channels must be a multiple of 64");
  if ((reinterpret_cast<uintptr_t>(t.ptr) & 15) != 0)
    throw std::invalid_argument("im2col operand must be 16-byte aligned");
  CUtensorMap map;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(t.c), static_cast<cuuint64_t>(t.w),
                        static_cast<cuuint64_t>(t.h), static_cast<cuuint64_t>(t.n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(t.c) * 2,
                           static_cast<cuuint64_t>(t.c) * 2 * t.w,
                           static_cast<cuuint64_t>(t.c) * 2 * t.w * t.h};
  int lower[2] = {-1, -1}, upper[2] = {-1, -1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = im2col_encode_fn()(
      &map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(static_cast<const void*>(t.ptr)),
      dims, strides, lower, upper, 64, static_cast<cuuint32_t>(pixels_per_column), estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw cuda_failure("cuTensorMapEncodeIm2col failed (code " + std::to_string(static_cast<int>(r)) +
                       ")");
  return map;
}

// Halo strip width of a 3x3 conv over images `w` pixels wide (GemmShape::
// halo_tw): whole strips of one image row that nearly fill a 128-row CTA
// tile; 0 = per-tap im2col loads.  Opt-in (PIPESIM_CONV_HALO=1): it cuts the
// operand bytes per output pixel by 40% but the narrow VGG layers turned out
// to be bound per k-block by the N <= 128 MMAs' shared-memory operand reads,
// not by L2->SM bytes, so the 112-of-128-row strips only add tiles (layer 1
// forward 547 -> 626 us; aligned views measured the same).
int halo_width(int w) {
  static const bool on = [] {
    const char* e = std::getenv("PIPESIM_CONV_HALO");
    return e && std::string(e) == "1";
  }();
  if (!on) return 0;
  for (int tw = 126; tw >= 96; --tw)
    if (w % tw == 0) return tw;
  return 0;
}

// {64 ch, tw + 2 px, 3 rows, 1 image} halo patches of an NHWC tensor
// (coordinates {c, w - 1, h - 1, n}; out-of-image positions read zeros)
CUtensorMap make_patch_tmap(const Nhwc& t, int tw) {
  if (t.c % 64 != 0) throw std::invalid_argument("halo operand: channels must be a multiple of 64");
  CUtensorMap map;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(t.c), static_cast<cuuint64_t>(t.w),
                        static_cast<cuuint64_t>(t.h), static_cast<cuuint64_t>(t.n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(t.c) * 2,
                           static_cast<cuuint64_t>(t.c) * 2 * t.w,
                           static_cast<cuuint64_t>(t.c) * 2 * t.w * t.h};
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(tw + 2), 3, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                           const_cast<void*>(static_cast<const void*>(t.ptr)), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw cuda_failure("cuTensorMapEncodeTiled (halo patch) failed (code " +
                       std::to_string(static_cast<int>(r)) + ")");
  return map;
}

// conv weights [Cout][ld] viewed as [Cout][9][Cin]: box 64 Cin x 1 tap x 64 Cout
CUtensorMap make_w3d_tmap(const __nv_bfloat16* w, int cout, int cin, int ld, int box_n = 64) {
  if (cin % 64 != 0 || ld % 8 != 0) throw std::invalid_argument("conv weights: Cin % 64, ld % 8");
  CUtensorMap map;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cin), 9, static_cast<cuuint64_t>(cout)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cin) * 2, static_cast<cuuint64_t>(ld) * 2};
  // 64 input channels per box (128-byte swizzle), or 32 (64-byte swizzle:
  // one CTA's half of a 64-wide MMA)
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_n), 1, 64};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                           const_cast<void*>(static_cast<const void*>(w)), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_n == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw cuda_failure("cuTensorMapEncodeTiled (3-D) failed (code " +
                       std::to_string(static_cast<int>(r)) + ")");
  return map;
}

// split count of a partial-slab wgrad: about two waves of 128 x bn tiles
// Split count of a split-K partial-slab GEMM with `tiles` output tiles on
// `slots` persistent CTAs (pairs) or SMs: the smallest S whose tiles * S units
// fill the slots in whole waves best (at most four waves, at least 8
// k-blocks per unit), so no slot idles through a final partial wave.
int balanced_splits(int tiles, int kb, int slots) {
  const int s_max = std::max(1, std::min(std::max(1, kb / 8), (4 * slots + tiles - 1) / tiles));
  int best = 1;
  double best_eff = -1.0;
  for (int S = 1; S <= s_max; ++S) {
    const int kbps = (kb + S - 1) / S;
    const int s_real = (kb + kbps - 1) / kbps;
    const int units = tiles * s_real;
    const int waves = (units + slots - 1) / slots;
    // useful work / slot time, the last split's shorter K included
    const double eff = static_cast<double>(kb) * tiles / (static_cast<double>(waves) * slots * kbps);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best = S;
    }
  }
  return best;
}

int partial_splits(int M, int N, int K, int bn, int* kbps) {
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  const int kb = (K + 63) / 64;
  const int S = balanced_splits(tiles, kb, sm_count());
  *kbps = (kb + S - 1) / S;
  return (kb + *kbps - 1) / *kbps;
}
}  // namespace

GemmLaunch plan_conv_fwd(const Nhwc& x, int img0, int imgs, const Mat16& w, const float* bias,
                         int act, __nv_bfloat16* y16, int y_row_off) {
  const int hw = x.h * x.w;
  GemmLaunch g;
  g.pair = true;
  const int tw = halo_width(x.w);
  g.bn = w.rows > 128 ? 256 : (pair_bn64(w.rows) && !tw ? 64 : 128);
  g.ta = tw ? make_patch_tmap(x, tw) : make_im2col_tmap(x, 128);
  g.tb = make_operand_tmap(w, /*k_major=*/true, b_box(g));
  g.sh = GemmShape{imgs * hw, w.rows, 9 * x.c, img0 * hw, 0, 0, 0, 1, 0};
  g.sh.conv = 1;
  g.sh.halo_tw = tw;
  g.ext = tw > 0;
  g.sh.conv_h = x.h;
  g.sh.conv_w = x.w;
  g.sh.conv_c = x.c;
  g.ep = empty_epi(kEpiFwd);
  g.ep.bias = bias;
  g.ep.act = act;
  g.ep.y16 = y16;
  g.ep.ld_y16 = w.rows;
  g.ep.y_row_off = y_row_off;
  vec_or_fallback(g.ep, kEpiFwd);
  return g;
}

GemmLaunch plan_conv_dgrad(const Nhwc& dz, const __nv_bfloat16* w, int cin, int ld_w,
                           const __nv_bfloat16* xin, int act_prev, __nv_bfloat16* d) {
  GemmLaunch g;
  g.pair = true;
  g.bn = cin > 128 ? 256 : 128;
  const int tw = halo_width(dz.w);
  // Cin = 64: 64-wide pair tiles (no half-empty 128-wide MMA), the weight
  // boxes 32 input channels per CTA (PIPESIM_DGRAD_BN64=0: off)
  static const bool bn64 = [] {
    const char* e = std::getenv("PIPESIM_DGRAD_BN64");
    return !(e && std::string(e) == "0");
  }();
  if (bn64 && cin == 64 && !tw) g.bn = 64;
  g.ta = tw ? make_patch_tmap(dz, tw) : make_im2col_tmap(dz, 128);
  g.tb = make_w3d_tmap(w, dz.c, cin, ld_w, g.bn == 64 ? 32 : 64);
  g.sh = GemmShape{dz.n * dz.h * dz.w, cin, 9 * dz.c, 0, 0, 0, 0, 1, 0};
  g.sh.conv = 3;
  g.sh.halo_tw = tw;
  g.ext = tw > 0;
  g.sh.conv_h = dz.h;
  g.sh.conv_w = dz.w;
  g.sh.conv_c = dz.c;
  g.ep = empty_epi(kEpiDgrad);
  g.ep.xin = xin;
  g.ep.ld_xin = cin;
  g.ep.act_prev = act_prev;
  g.ep.d16 = d;
  g.ep.ld_d16 = cin;
  vec_or_fallback(g.ep, kEpiDgrad);
  return g;
}

size_t wgrad_partial_floats(int M, int N, int K, int* lds) {
  const int bn = N >= 256 ? 256 : 128;
  int kbps = 0;
  const int S = partial_splits(M, N, K, bn, &kbps);
  *lds = (N + 7) / 8 * 8;
  return static_cast<size_t>(S) * M * *lds;
}

namespace {
GemmLaunch partial_common(const Mat16& dz, int N, float* ws, int lds, int* splits) {
  GemmLaunch g;
  const int M = dz.cols, K = dz.rows;
  g.pair = false;
  g.bn = N >= 256 ? 256 : 128;
  int kbps = 0;
  const int S = partial_splits(M, N, K, g.bn, &kbps);
  *splits = S;
  g.ta = make_operand_tmap(dz, /*k_major=*/false, 64);
  g.sh = GemmShape{M, N, K, 0, 0, 0, 0, S, kbps};
  g.ep = empty_epi(kEpiFwd);
  g.ep.act = kLinear;
  g.ep.y32 = ws;
  g.ep.ld_y32 = lds;
  g.ep.partial_slab = static_cast<long long>(M) * lds;
  g.ep.rowwise = 2;
  if (lds % 4 != 0 || !al(ws, 16)) throw std::invalid_argument("partial slabs: 16-byte rows");
  return g;
}

// CTA-pair conv wgrad (256-row tiles, split-K over the pixels into partial
// slabs, about two units per pair): Cout >= 256 computes dW = dz^T im2col(x)
// (M = Cout), narrower layers the transposed dW^T = im2col(x)^T dz
// (M = 9*Cin, N = Cout), so the 256-row tile is never mostly empty.
struct PairWgradShape {
  bool transposed;
  int M, N, bn, S, kbps, lds;
};
PairWgradShape pair_wgrad_shape(int cout, int cin, int pixels, bool transposed) {
  PairWgradShape p;
  p.transposed = transposed;
  p.M = p.transposed ? 9 * cin : cout;
  p.N = p.transposed ? cout : 9 * cin;
  p.bn = p.N >= 256 ? 256 : 128;
  const int tiles = ((p.M + 255) / 256) * ((p.N + p.bn - 1) / p.bn);
  const int kb = (pixels + 63) / 64;
  const int S = balanced_splits(tiles, kb, sm_count() / 2);
  p.kbps = (kb + S - 1) / S;
  p.S = (kb + p.kbps - 1) / p.kbps;
  p.lds = (p.N + 7) / 8 * 8;
  return p;
}
}  // namespace

size_t conv_wgrad_floats(int cout, int cin, int pixels) {
  int lds = 0;
  const size_t single = wgrad_partial_floats(cout, 9 * cin, pixels, &lds);
  size_t pair = 0;
  for (bool t : {false, true}) {
    const PairWgradShape p = pair_wgrad_shape(cout, cin, pixels, t);
    pair = std::max(pair, static_cast<size_t>(p.S) * p.M * p.lds);
  }
  return std::max(single, pair);
}

// PIPESIM_CONV_WGRAD=pair|single|transposed (default: pair for Cout >= 256,
// else the single-CTA kernel; the transposed pair form measured slower)
int conv_wgrad_mode(int cout) {
  static const int env = [] {
    const char* e = std::getenv("PIPESIM_CONV_WGRAD");
    if (!e) return -1;
    return std::strcmp(e, "single") == 0 ? 0 : std::strcmp(e, "pair") == 0 ? 1 : 2;
  }();
  if (env >= 0) return env == 1 && cout < 256 ? 0 : env;
  return cout >= 256 ? 1 : 0;
}

GemmLaunch plan_conv_wgrad_partial(const Mat16& dz, const Nhwc& x, int img0, float* ws,
                                   ConvWgradInfo* info) {
  const int cout = dz.cols, pixels = dz.rows;
  const int mode = conv_wgrad_mode(cout);
  if (mode == 0) {  // single-CTA 128-row tiles, dW = dz^T im2col(x)
    int lds = 0;
    wgrad_partial_floats(cout, 9 * x.c, pixels, &lds);
    GemmLaunch g = partial_common(dz, 9 * x.c, ws, lds, &info->splits);
    g.tb = make_im2col_tmap(x, 64);
    g.sh.b_k_off = img0 * x.h * x.w;
    g.sh.conv = 2;
    g.sh.conv_h = x.h;
    g.sh.conv_w = x.w;
    g.sh.conv_c = x.c;
    info->lds = lds;
    info->slab = static_cast<long long>(cout) * lds;
    info->transposed = false;
    return g;
  }
  const PairWgradShape p = pair_wgrad_shape(cout, x.c, pixels, mode == 2);
  GemmLaunch g;
  g.pair = true;
  g.ext = true;
  g.bn = p.bn;
  const CUtensorMap im = make_im2col_tmap(x, 64);
  const CUtensorMap dm = make_operand_tmap(dz, /*k_major=*/false, 64);
  g.ta = p.transposed ? im : dm;
  g.tb = p.transposed ? dm : im;
  g.sh = GemmShape{p.M, p.N, pixels, 0, 0, 0, 0, p.S, p.kbps};
  g.sh.conv = p.transposed ? 4 : 2;
  if (p.transposed)
    g.sh.a_k_off = img0 * x.h * x.w;
  else
    g.sh.b_k_off = img0 * x.h * x.w;
  g.sh.conv_h = x.h;
  g.sh.conv_w = x.w;
  g.sh.conv_c = x.c;
  g.ep = empty_epi(kEpiFwd);
  g.ep.act = kLinear;
  g.ep.y32 = ws;
  g.ep.ld_y32 = p.lds;
  g.ep.partial_slab = static_cast<long long>(p.M) * p.lds;
  g.ep.rowwise = 2;
  if (!al(ws, 16)) throw std::invalid_argument("partial slabs: 16-byte aligned workspace");
  info->splits = p.S;
  info->lds = p.lds;
  info->slab = static_cast<long long>(p.M) * p.lds;
  info->transposed = p.transposed;
  return g;
}

GemmLaunch plan_wgrad_partial(const Mat16& dz, const Mat16& x, float* ws, int lds, int* splits) {
  GemmLaunch g = partial_common(dz, x.cols, ws, lds, splits);
  g.tb = make_operand_tmap(x, /*k_major=*/false, 64);
  return g;
}

void launch_wgrad_partial(const GemmLaunch& g, cudaStream_t st) {
  if (g.bn == 256)
    launch_one<256, true, true, kEpiFwd>(g, st);
  else
    launch_one<128, true, true, kEpiFwd>(g, st);
}

// ------------------------------------------------------------ dgrad chain
// PIPESIM_DGRAD_CHAIN=0 keeps two dgrad launches
bool dgrad_chain_eligible(int out_l, int in_l) {
  static const bool on = [] {
    const char* e = std::getenv("PIPESIM_DGRAD_CHAIN");
    return !(e && std::string(e) == "0");
  }();
  return on && out_l <= 64 && in_l <= 256 && in_l % 64 == 0;
}

ChainLaunch plan_dgrad_chain(const GemmLaunch& g1, const GemmLaunch& g2, const Mat16& dz_mid) {
  if (g1.simt || g2.simt) throw std::logic_error("dgrad chain: bf16 tensor-core plans only");
  ChainLaunch c;
  c.a1 = g1.ta;
  c.b1 = g1.tb;
  c.b2 = g2.tb;
  c.dz = make_operand_tmap(dz_mid, /*k_major=*/true, 128);
  c.sh2 = g2.sh;
  c.ep2 = g2.ep;
  c.ca.x_gate = g1.ep.xin;
  c.ca.ld_gate = g1.ep.ld_xin;
  c.ca.act_gate = g1.ep.act_prev;
  c.ca.k1 = g1.sh.K;
  c.ca.n1 = g1.sh.N;
  c.ca.store_dz = 1;
  if (c.ca.k1 > 64 || c.ca.n1 > 256 || c.ca.n1 % 64 != 0 || g2.sh.K != c.ca.n1 ||
      (c.ca.ld_gate % 8) != 0)
    throw std::invalid_argument("dgrad chain: shape outside the fused kernel's range");
  // 64-wide column tiles unless that gives 16 or more CTAs (PIPESIM_CHAIN_BN)
  static const int env_bn = [] {
    const char* e = std::getenv("PIPESIM_CHAIN_BN");
    return e ? std::atoi(e) : 0;
  }();
  const long tiles128 = static_cast<long>((g2.sh.M + 127) / 128) * ((g2.sh.N + 127) / 128);
  c.bn = env_bn == 64 || env_bn == 128 ? env_bn : (tiles128 < 16 ? 64 : 128);
  // PIPESIM_CHAIN_CLUSTER=1: a cluster of n1 / 64 CTAs along the column
  // tiles builds dz_{l-1} once per row block.  Off by default: on C1 it is
  // 0.35 us slower under TiMePReSt (the cluster barriers on the cycle cost
  // more than the recomputation they save) and 0.7 us faster under 1F1B
  // (tools/gpu/r2_chain_cluster.sh).
  static const bool cluster_on = [] {
    const char* e = std::getenv("PIPESIM_CHAIN_CLUSTER");
    return e && std::string(e) == "1";
  }();
  const int C = c.ca.n1 / 64, tiles_n = (g2.sh.N + c.bn - 1) / c.bn;
  c.ca.cluster = cluster_on && C > 1 && tiles_n % C == 0 ? C : 1;
  return c;
}

namespace {
template <int BN>
void launch_chain_bn(const ChainLaunch& c, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    PB_CUDA(cudaFuncSetAttribute(dgrad_chain_kernel<BN>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 ChainCfg<BN>::kSmem));
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((c.sh2.N + BN - 1) / BN, (c.sh2.M + 127) / 128);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = ChainCfg<BN>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (c.ca.cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = c.ca.cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  GemmLaunch probe;
  probe.pdl = c.pdl;
  if (pdl_on(probe)) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  PB_CUDA(cudaLaunchKernelEx(&cfg, dgrad_chain_kernel<BN>, c.a1, c.b1, c.b2, c.dz, c.sh2, c.ep2,
                             c.ca));
  PB_CUDA(cudaGetLastError());
}
}  // namespace

void launch_dgrad_chain(const ChainLaunch& c, cudaStream_t st) {
  if (c.sh2.M <= 0 || c.sh2.N <= 0) return;
  if (c.bn == 128)
    launch_chain_bn<128>(c, st);
  else
    launch_chain_bn<64>(c, st);
}

// ------------------------------------------------------------ forward chain
// PIPESIM_FWD_CHAIN=0 keeps two forward launches
bool fwd_chain_eligible(int n1, int n2) {
  static const bool on = [] {
    const char* e = std::getenv("PIPESIM_FWD_CHAIN");
    return !(e && std::string(e) == "0");
  }();
  return on && n1 <= 256 && n1 % 64 == 0 && n2 <= 64;
}

FwdChainLaunch plan_fwd_chain(const Mat16& x, int x_row_off, int rows, const Mat16& w1,
                              const float* b1, int act1, __nv_bfloat16* y1, int ld_y1,
                              int y1_row_off, const Mat16& w2, const GemmLaunch& g2) {
  if (g2.simt) throw std::logic_error("forward chain: bf16 tensor-core plans only");
  const int n1 = w1.rows, n2 = w2.rows;
  if (n1 > 256 || n1 % 64 != 0 || n2 > 64 || w2.cols != n1 || (ld_y1 % 8) != 0 ||
      (reinterpret_cast<uintptr_t>(b1) & 15) != 0)
    throw std::invalid_argument("forward chain: shape outside the fused kernel's range");
  FwdChainLaunch c;
  c.x = make_operand_tmap(x, /*k_major=*/true, 128);
  c.w1 = make_operand_tmap(w1, /*k_major=*/true, 64);  // one 64-row slice per cluster CTA
  c.fa.n2pad = (n2 + 15) / 16 * 16;
  c.w2 = make_operand_tmap(w2, /*k_major=*/true, c.fa.n2pad);
  // the store map ends at this launch's last row: the tile's tail rows past
  // it belong to other micro-batches
  c.y1 = make_operand_tmap(Mat16{y1, y1_row_off + rows, n1, ld_y1}, /*k_major=*/true, 128);
  c.sh1 = GemmShape{rows, n1, x.cols, x_row_off, 0, 0, 0, 1, 0};
  c.sh2 = g2.sh;
  c.sh2.M = rows;
  c.ep2 = g2.ep;
  c.fa.b1 = b1;
  c.fa.y1_row_off = y1_row_off;
  c.act1 = act1;
  return c;
}

namespace {
template <int ACT1>
void launch_fwd_chain_act(const FwdChainLaunch& c, const EpiParams& ep2, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    PB_CUDA(cudaFuncSetAttribute(fwd_chain_kernel<ACT1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 FwdChainCfg::kSmem));
  });
  const int C = c.sh1.N / 64;  // cluster: one CTA per 64 columns of y1
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C, (c.sh1.M + 127) / 128);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = FwdChainCfg::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  GemmLaunch probe;
  probe.pdl = c.pdl;
  cfg.numAttrs = pdl_on(probe) ? 2 : 1;
  PB_CUDA(cudaLaunchKernelEx(&cfg, fwd_chain_kernel<ACT1>, c.x, c.w1, c.w2, c.y1, c.sh1, c.sh2,
                             ep2, c.fa));
  PB_CUDA(cudaGetLastError());
}
}  // namespace

void launch_fwd_chain(const FwdChainLaunch& c, cudaStream_t st, const EpiParams& ep2) {
  if (c.sh1.M <= 0) return;
  switch (c.act1) {
    case kRelu: return launch_fwd_chain_act<kRelu>(c, ep2, st);
    case kTanh: return launch_fwd_chain_act<kTanh>(c, ep2, st);
    case kSigmoid: return launch_fwd_chain_act<kSigmoid>(c, ep2, st);
    default: return launch_fwd_chain_act<kLinear>(c, ep2, st);
  }
}
void launch_fwd_chain(const FwdChainLaunch& c, cudaStream_t st) { launch_fwd_chain(c, st, c.ep2); }

void launch_fwd(const GemmLaunch& g, cudaStream_t st) {
  if (g.simt) return launch_simt_gemm(g, kEpiFwd, st);
  launch_bn<false, false, kEpiFwd>(g, st);
}
void launch_dgrad(const GemmLaunch& g, cudaStream_t st) {
  if (g.simt) return launch_simt_gemm(g, kEpiDgrad, st);
  launch_bn<false, true, kEpiDgrad>(g, st);
}
void launch_wgrad(const GemmLaunch& g, cudaStream_t st) {
  if (g.simt) return launch_simt_gemm(g, kEpiWgradSgd, st);
  launch_bn<true, true, kEpiWgradSgd>(g, st);
}

// ------------------------------------------------------------ bias + SGD
// b_new = b_cur - lr * colsum(dz).  A block owns 8 output columns (one
// 16-byte bf16 load per row); its 256 threads take rows t, t+256, ... with
// four loads in flight each, so a 1024 x 4096 dZ is read by 512 blocks in a
// single round trip (7.1 us cold in the ncu launch list, against 8.7 us for
// 32-column blocks of 64 row groups and 8.5 us for 32-column blocks of 128).
// The per-thread partials are combined by a fixed shuffle tree and then in
// warp order: the result is deterministic.  (trainer.cpp:250-252, :484-488.)
constexpr int kBiasCols = 8;
constexpr int kBiasThreads = 256;

template <typename TZ>
__global__ void __launch_bounds__(kBiasThreads)
    bias_sgd_kernel(const TZ* __restrict__ dz, int rows, int out, int ld_dz,
                    const float* b_cur, float* b_new, float* b_copy, float lr,
                    int* tag_slot, int* cur_version, int version, const int* trace_src,
                    int* trace_dst) {
  __shared__ float red[kBiasThreads / 32][kBiasCols];
  const int c0 = blockIdx.x * kBiasCols;
  float acc[kBiasCols] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const bool vec = sizeof(TZ) == 2 && (ld_dz % 8) == 0 && c0 + kBiasCols <= out;
  if constexpr (sizeof(TZ) == 2) if (vec) {
    constexpr int kU = 4;
    for (int r0 = threadIdx.x; r0 < rows; r0 += kU * kBiasThreads) {
      uint4 q[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int r = r0 + u * kBiasThreads;
        q[u] = r < rows ? *reinterpret_cast<const uint4*>(dz + static_cast<size_t>(r) * ld_dz + c0)
                        : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q[u]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(h[k]);
          acc[2 * k] += f.x;
          acc[2 * k + 1] += f.y;
        }
      }
    }
  }
  if (!vec) {
    for (int r = threadIdx.x; r < rows; r += kBiasThreads) {
      const TZ* p = dz + static_cast<size_t>(r) * ld_dz + c0;
      for (int k = 0; k < kBiasCols && c0 + k < out; ++k) acc[k] += static_cast<float>(p[k]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < kBiasCols; ++k) acc[k] += __shfl_xor_sync(~0u, acc[k], o);
  const int w = threadIdx.x / 32;
  if (threadIdx.x % 32 == 0)
#pragma unroll
    for (int k = 0; k < kBiasCols; ++k) red[w][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < kBiasCols) {
    const int col = c0 + threadIdx.x;
    if (col < out) {
      float g = 0.f;
#pragma unroll
      for (int i = 0; i < kBiasThreads / 32; ++i) g += red[i][threadIdx.x];
      const float b = b_cur[col] - lr * g;
      b_new[col] = b;
      if (b_copy) b_copy[col] = b;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (trace_src && trace_dst) *trace_dst = *trace_src;
    if (tag_slot) *tag_slot = version;
    if (cur_version) *cur_version = version;
  }
}

void launch_bias_sgd(cudaStream_t st, const __nv_bfloat16* dz, int rows,
                     int out, int ld_dz, const float* b_cur, float* b_new,
                     float* b_copy, float lr, int* tag_slot, int* cur_version,
                     int version, const int* trace_src, int* trace_dst, bool dz_f32) {
  const int grid = (out + kBiasCols - 1) / kBiasCols;
  if (dz_f32)
    bias_sgd_kernel<float><<<grid, kBiasThreads, 0, st>>>(
        reinterpret_cast<const float*>(dz), rows, out, ld_dz, b_cur, b_new, b_copy, lr,
        tag_slot, cur_version, version, trace_src, trace_dst);
  else
    bias_sgd_kernel<__nv_bfloat16><<<grid, kBiasThreads, 0, st>>>(
        dz, rows, out, ld_dz, b_cur, b_new, b_copy, lr, tag_slot, cur_version, version,
        trace_src, trace_dst);
  PB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------ loss
// One 256-thread block per row (rows are up to 4096 classes wide; the row
// stays L1-resident across the three passes).  Softmax-CE: max-subtracted
// log-softmax, loss counts targets > 0.5 (trainer.cpp:278-286); grad =
// (softmax - t)/denom (:301-309).  MSE: sum (y-t)^2, grad 2(y-t)/denom
// (:273-276, :297-299).  act' of a non-linear output layer is applied from y.
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x / 32); ++i) s += red[i];
  return s;
}

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(~0u, v, o));
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = -INFINITY;
  for (int i = 0; i < static_cast<int>(blockDim.x / 32); ++i) s = fmaxf(s, red[i]);
  return s;
}

template <typename TZ>
__device__ __forceinline__ TZ to_dz(float g) {
  if constexpr (sizeof(TZ) == 2) return __float2bfloat16_rn(g);
  else return g;
}

template <typename TZ>
__global__ void __launch_bounds__(256)
    loss_kernel(const float* __restrict__ y, int rows, int cols, int ld_y,
                const float* __restrict__ t, int ld_t, int loss, int act_last,
                float denom, TZ* __restrict__ dz, int ld_dz,
                float* __restrict__ row_loss, const int* __restrict__ labels) {
  __shared__ float red[8];
  const int row = blockIdx.x;
  if (row >= rows) return;
  const float* yr = y + static_cast<size_t>(row) * ld_y;
  // targets: dense rows, or class labels (one-hot implied, never materialised)
  const float* tr = labels ? nullptr : t + static_cast<size_t>(row) * ld_t;
  const int lab = labels ? labels[row] : -1;
  TZ* dr = dz + static_cast<size_t>(row) * ld_dz;
  float acc = 0.f;
  if (loss == 0) {  // mse
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      const float yv = yr[c];
      const float d = yv - (tr ? tr[c] : (c == lab ? 1.f : 0.f));
      acc += d * d;
      float g = 2.f * d / denom;
      if (act_last != kLinear) g *= act_grad_from_out(yv, act_last);
      dr[c] = to_dz<TZ>(g);
    }
  } else {
    float mx = -INFINITY;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) mx = fmaxf(mx, yr[c]);
    mx = block_max(mx, red);
    float se = 0.f;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) se += expf(yr[c] - mx);
    se = block_sum(se, red);
    const float lse = logf(se);
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      const float yv = yr[c];
      const float z = yv - mx;
      const float tc = tr ? tr[c] : (c == lab ? 1.f : 0.f);
      if (tc > 0.5f) acc += -(z - lse) * tc;
      float g = (expf(z) / se - tc) / denom;
      if (act_last != kLinear) g *= act_grad_from_out(yv, act_last);
      dr[c] = to_dz<TZ>(g);
    }
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) row_loss[row] = acc;
}

// Softmax-CE against class labels with a linear output layer (the benchmark
// head): each thread keeps its <= 16 logits in registers (four float4), so
// the row is read once and exp is evaluated once per logit; max, sum and the
// gradient as in loss_kernel, the row loss from the label's logit.
__global__ void __launch_bounds__(256)
    loss_ce_labels_kernel(const float* __restrict__ y, int cols, int ld_y, float denom,
                          __nv_bfloat16* __restrict__ dz, int ld_dz,
                          float* __restrict__ row_loss, const int* __restrict__ labels) {
  __shared__ float red[8];
  const int row = blockIdx.x;
  const float4* yr = reinterpret_cast<const float4*>(y + static_cast<size_t>(row) * ld_y);
  const int nq = cols / 4;
  const int lab = labels[row];
  float4 v[4];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = threadIdx.x + 256 * i;
    v[i] = q < nq ? yr[q] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    mx = fmaxf(mx, fmaxf(fmaxf(v[i].x, v[i].y), fmaxf(v[i].z, v[i].w)));
  }
  mx = block_max(mx, red);
  float se = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = make_float4(expf(v[i].x - mx), expf(v[i].y - mx), expf(v[i].z - mx),
                       expf(v[i].w - mx));  // exp(-inf) = 0 for the padding
    se += v[i].x + v[i].y + v[i].z + v[i].w;
  }
  se = block_sum(se, red);
  if (threadIdx.x == 0) {
    const float lse = logf(se);
    row_loss[row] = (lab >= 0 && lab < cols)
                        ? -((y[static_cast<size_t>(row) * ld_y + lab] - mx) - lse) : 0.f;
  }
  __nv_bfloat16* dr = dz + static_cast<size_t>(row) * ld_dz;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = threadIdx.x + 256 * i;
    if (q >= nq) continue;
    const int c = 4 * q;
    const float g0 = (v[i].x / se - (c == lab ? 1.f : 0.f)) / denom;
    const float g1 = (v[i].y / se - (c + 1 == lab ? 1.f : 0.f)) / denom;
    const float g2 = (v[i].z / se - (c + 2 == lab ? 1.f : 0.f)) / denom;
    const float g3 = (v[i].w / se - (c + 3 == lab ? 1.f : 0.f)) / denom;
    __nv_bfloat162 h0 = __floats2bfloat162_rn(g0, g1);
    __nv_bfloat162 h1 = __floats2bfloat162_rn(g2, g3);
    *reinterpret_cast<uint2*>(dr + c) =
        make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
  }
}

void launch_loss(cudaStream_t st, const float* y, int rows, int cols, int ld_y,
                 const float* targets, int ld_t, int loss, int act_last,
                 float denom, __nv_bfloat16* dz, int ld_dz, float* row_loss, bool dz_f32,
                 const int* labels) {
  if (rows <= 0) return;
  if (loss != 0 && labels && act_last == kLinear && !dz_f32 && cols % 4 == 0 && cols <= 4096 &&
      cols >= 1024 && ld_y % 4 == 0 && ld_dz % 4 == 0 && al(y, 16) && al(dz, 8)) {
    loss_ce_labels_kernel<<<rows, 256, 0, st>>>(y, cols, ld_y, denom, dz, ld_dz, row_loss,
                                                labels);
    PB_CUDA(cudaGetLastError());
    return;
  }
  const int threads = cols >= 256 ? 256 : (cols >= 128 ? 128 : 64);
  if (dz_f32)
    loss_kernel<float><<<rows, threads, 0, st>>>(y, rows, cols, ld_y, targets, ld_t, loss,
                                                 act_last, denom, reinterpret_cast<float*>(dz),
                                                 ld_dz, row_loss, labels);
  else
    loss_kernel<__nv_bfloat16><<<rows, threads, 0, st>>>(y, rows, cols, ld_y, targets, ld_t, loss,
                                                         act_last, denom, dz, ld_dz, row_loss,
                                                         labels);
  PB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------ conversions
// Row-major conversion to bf16: blocks stride over rows, threads over
// columns (no per-element index division; coalesced on both sides).
template <typename T>
__global__ void to_bf16_kernel(const T* __restrict__ src, int rows, int cols,
                               int ld_src, __nv_bfloat16* __restrict__ dst,
                               int ld_dst) {
  const bool vec4 = sizeof(T) == 4 && (cols % 4) == 0 && (ld_src % 4) == 0 && (ld_dst % 4) == 0 &&
                    (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(dst) & 7) == 0;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const T* s = src + static_cast<size_t>(r) * ld_src;
    __nv_bfloat16* d = dst + static_cast<size_t>(r) * ld_dst;
    if (vec4) {  // 16-byte loads, 8-byte stores
      for (int c = 4 * threadIdx.x; c < cols; c += 4 * blockDim.x) {
        const float4 v = *reinterpret_cast<const float4*>(s + c);
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v.x, v.y);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v.z, v.w);
        *reinterpret_cast<uint2*>(d + c) =
            make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
      }
      continue;
    }
    for (int c = 2 * threadIdx.x; c < cols; c += 2 * blockDim.x) {
      if (c + 1 < cols)
        *reinterpret_cast<__nv_bfloat162*>(d + c) =
            __floats2bfloat162_rn(static_cast<float>(s[c]), static_cast<float>(s[c + 1]));
      else
        d[c] = __float2bfloat16_rn(static_cast<float>(s[c]));
    }
  }
}

__global__ void f64_f32_kernel(const double* __restrict__ src,
                               float* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<float>(src[i]);
}

namespace {
int grid_for(size_t n) {
  size_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}
}  // namespace

void launch_convert_f64_bf16(cudaStream_t st, const double* src, int rows,
                             int cols, int ld_src, __nv_bfloat16* dst,
                             int ld_dst) {
  if (rows <= 0 || cols <= 0) return;
  if ((ld_dst % 2) != 0) throw std::invalid_argument("bf16 rows must be 4-byte aligned");
  to_bf16_kernel<double><<<std::min(rows, 148 * 4), 256, 0, st>>>(src, rows, cols, ld_src, dst,
                                                                  ld_dst);
  PB_CUDA(cudaGetLastError());
}

void launch_convert_f32_bf16(cudaStream_t st, const float* src, int rows,
                             int cols, int ld_src, __nv_bfloat16* dst,
                             int ld_dst) {
  if (rows <= 0 || cols <= 0) return;
  if ((ld_dst % 2) != 0) throw std::invalid_argument("bf16 rows must be 4-byte aligned");
  static const int grid_cap = [] {
    const char* e = std::getenv("PIPESIM_CONV_GRID");
    return e ? std::max(1, std::atoi(e)) : 148 * 4;
  }();
  to_bf16_kernel<float><<<std::min(rows, grid_cap), 256, 0, st>>>(src, rows, cols, ld_src, dst,
                                                                  ld_dst);
  PB_CUDA(cudaGetLastError());
}

void launch_f32_to_bf16_rows(cudaStream_t st, const float* src, int rows,
                             int cols, int ld_src, __nv_bfloat16* dst,
                             int ld_dst) {
  launch_convert_f32_bf16(st, src, rows, cols, ld_src, dst, ld_dst);
}

__global__ void f32_f64_kernel(const float* __restrict__ src, double* __restrict__ dst,
                               size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<double>(src[i]);
}

void launch_convert_f32_f64(cudaStream_t st, const float* src, double* dst, size_t n) {
  if (n == 0) return;
  f32_f64_kernel<<<grid_for(n), 256, 0, st>>>(src, dst, n);
  PB_CUDA(cudaGetLastError());
}

void launch_convert_f64_f32(cudaStream_t st, const double* src, float* dst,
                            size_t n) {
  if (n == 0) return;
  f64_f32_kernel<<<grid_for(n), 256, 0, st>>>(src, dst, n);
  PB_CUDA(cudaGetLastError());
}

}  // namespace pb

// Device parameter digest: shortest-decimal formatting + parallel FNV-1a 64
// (design in digest_dev.hpp).
#include "digest_dev.hpp"

#include <algorithm>
#include <stdexcept>

#include "ryu_f32d.cuh"
#include "shortest.cuh"
#include "status.hpp"

namespace pb {
namespace {

constexpr int kT = 256;                  // threads per block
constexpr int kR = 16;                   // values per thread
constexpr int kVB = kT * kR;             // values per block
constexpr int kSlot = 32;                // bytes per formatted value
constexpr uint64_t kIdent = 0xFEDCBA9876543210ull;  // nibble map i -> i
constexpr uint64_t kRep = 0x1111111111111111ull;
constexpr uint64_t kP = 0x100000001b3ull;  // FNV-1a 64 prime

// nibble-wise a + b mod 16 (SWAR, no carry across nibbles)
__device__ __forceinline__ uint64_t nib_add(uint64_t a, uint64_t b) {
  return ((a & 0x7777777777777777ull) + (b & 0x7777777777777777ull)) ^
         ((a ^ b) & 0x8888888888888888ull);
}
// nibble-wise 3x mod 16
__device__ __forceinline__ uint64_t nib_mul3(uint64_t x) {
  return nib_add(x, (x << 1) & 0xEEEEEEEEEEEEEEEEull);
}
// "f, then g": out[i] = g[f[i]]
__device__ __forceinline__ uint64_t compose(uint64_t f, uint64_t g) {
  uint64_t o = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t fi = static_cast<uint32_t>(f >> (4 * i)) & 15u;
    o |= ((g >> (4 * fi)) & 15ull) << (4 * i);
  }
  return o;
}
__device__ __forceinline__ uint32_t apply(uint64_t f, uint32_t n) {
  return static_cast<uint32_t>(f >> (4 * n)) & 15u;
}

// byte j (compile-time after unrolling) of a 32-byte slot held in registers
__device__ __forceinline__ uint32_t slot_byte(const uint4 (&q)[2], int j) {
  const uint4 v = q[j >> 4];
  const int w = (j >> 2) & 3;
  const uint32_t x = w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
  return (x >> (8 * (j & 3))) & 0xFFu;
}

__device__ __forceinline__ float fetch(const DigestSpan& sp, int64_t off) {
  if (sp.f32) return __ldg(sp.f32 + off);
  const uint32_t h = __bfloat16_as_ushort(sp.hi[off]);
  const uint32_t l = __ldg(sp.lo + off);
  return __int_as_float(static_cast<int>(h << 16) + static_cast<int>(static_cast<int16_t>(l)));
}

__device__ int find_span(const DigestSpan* spans, int nspans, int64_t i) {
  int lo = 0, hi = nspans - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (spans[mid].start <= i) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Block-wide in-order reduction of nibble maps (result valid in thread 0).
__device__ uint64_t block_compose(uint64_t m, uint64_t* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_down_sync(0xffffffffu, m, d);
    if ((lane & (2 * d - 1)) == 0) m = compose(m, o);
  }
  if (lane == 0) sh[w] = m;
  __syncthreads();
  uint64_t r = kIdent;
  if (threadIdx.x == 0)
    for (int i = 0; i < kT / 32; ++i) r = compose(r, sh[i]);
  __syncthreads();
  return r;
}

// Incoming nibble of every thread of the block, given the block's incoming
// nibble and the threads' maps (in-order exclusive scan).
__device__ uint32_t block_incoming(uint64_t m, uint32_t block_in, uint64_t* sh, uint32_t* shn) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t inc = m;  // inclusive scan within the warp
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc = compose(o, inc);
  }
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t n = block_in;
    for (int i = 0; i < kT / 32; ++i) {
      shn[i] = n;
      n = apply(sh[i], n);
    }
  }
  __syncthreads();
  uint64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) exc = kIdent;
  const uint32_t r = apply(exc, shn[w]);
  __syncthreads();
  return r;
}

// (A) format + low-nibble maps (R values per thread: 16, or 4 for small
// segments so that they still fill the SMs)
template <int R>
__global__ void __launch_bounds__(kT) dg_format_lo(const DigestSpan* __restrict__ spans,
                                                   int nspans, int64_t seg0, int64_t segn,
                                                   char* __restrict__ slots,
                                                   uint8_t* __restrict__ lens,
                                                   uint64_t* __restrict__ tmap,
                                                   uint64_t* __restrict__ bmap) {
  __shared__ uint64_t sh[kT / 32];
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  const int64_t a = t * R;
  uint64_t S = kIdent;
  if (a < segn) {
    const int64_t b = min(segn, a + R);
    int si = find_span(spans, nspans, seg0 + a);
    DigestSpan sp = spans[si];
    int64_t local = seg0 + a - sp.start;
    int64_t r = local / sp.cols, c = local - r * sp.cols;
    int64_t next = si + 1 < nspans ? spans[si + 1].start : INT64_MAX;
    for (int64_t i = a; i < b; ++i) {
      if (seg0 + i >= next) {
        ++si;
        sp = spans[si];
        next = si + 1 < nspans ? spans[si + 1].start : INT64_MAX;
        r = 0;
        c = 0;
      }
      const float v = fetch(sp, r * sp.ld + c);
      if (++c == sp.cols) c = 0, ++r;
      uint64_t wv[4];
      int n = fmt::format_shortest_fast(static_cast<double>(v), wv);
      fmt::text_put(wv, n++, '\n');
      const uint4 q[2] = {make_uint4(static_cast<uint32_t>(wv[0]), static_cast<uint32_t>(wv[0] >> 32),
                                     static_cast<uint32_t>(wv[1]), static_cast<uint32_t>(wv[1] >> 32)),
                          make_uint4(static_cast<uint32_t>(wv[2]), static_cast<uint32_t>(wv[2] >> 32),
                                     static_cast<uint32_t>(wv[3]), static_cast<uint32_t>(wv[3] >> 32))};
      uint4* dst = reinterpret_cast<uint4*>(slots + i * kSlot);
      dst[0] = q[0];
      dst[1] = q[1];
      lens[i] = static_cast<uint8_t>(n);
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // registers only: bytes off the words
        uint64_t word = wv[k];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          if (8 * k + b >= n) break;
          const uint64_t x = S ^ ((word & 15u) * kRep);
          S = nib_mul3(x);
          word >>= 8;
        }
      }
    }
  }
  tmap[t] = S;
  const uint64_t bm = block_compose(S, sh);
  if (threadIdx.x == 0) bmap[blockIdx.x] = bm;
}

// chain the block maps from the segment's incoming nibble (bits `shift`..+4
// of *state); bin[b] = incoming nibble of block b
__global__ void __launch_bounds__(1024) dg_chain(const uint64_t* __restrict__ bmap, int nb,
                                                 const uint64_t* __restrict__ state, int shift,
                                                 uint8_t* __restrict__ bin) {
  __shared__ uint64_t g[1024];
  __shared__ uint32_t gn[1024];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  uint64_t m = kIdent;
  for (int b = b0; b < b1; ++b) m = compose(m, bmap[b]);
  g[threadIdx.x] = m;
  __syncthreads();
  // exclusive scan of the 1024 group maps in order (Hillis-Steele: 10
  // compose steps instead of a 1024-long serial chain), then each group's
  // incoming nibble is its prefix applied to the segment's incoming nibble
  uint64_t inc = m;
  for (int d = 1; d < 1024; d <<= 1) {
    const uint64_t prev = threadIdx.x >= d ? g[threadIdx.x - d] : kIdent;
    __syncthreads();
    inc = compose(prev, inc);
    g[threadIdx.x] = inc;
    __syncthreads();
  }
  const uint32_t n0 = static_cast<uint32_t>(*state >> shift) & 15u;
  gn[threadIdx.x] = threadIdx.x == 0 ? n0 : apply(g[threadIdx.x - 1], n0);
  __syncthreads();
  uint32_t n = gn[threadIdx.x];
  for (int b = b0; b < b1; ++b) {
    bin[b] = static_cast<uint8_t>(n);
    n = apply(bmap[b], n);
  }
}

// (B) high-nibble maps given the low-nibble trajectory
template <int R>
__global__ void __launch_bounds__(kT) dg_hi(const char* __restrict__ slots,
                                            const uint8_t* __restrict__ lens, int64_t segn,
                                            uint64_t* __restrict__ tmap,
                                            uint8_t* __restrict__ tlo,
                                            const uint8_t* __restrict__ bin,
                                            uint64_t* __restrict__ bmap) {
  __shared__ uint64_t sh[kT / 32];
  __shared__ uint32_t shn[kT / 32];
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  const uint32_t lo_in = block_incoming(tmap[t], bin[blockIdx.x], sh, shn);
  tlo[t] = static_cast<uint8_t>(lo_in);
  const int64_t a = t * R;
  uint64_t H = kIdent;
  if (a < segn) {
    const int64_t b = min(segn, a + R);
    uint32_t lo = lo_in;
    for (int64_t i = a; i < b; ++i) {
      const int n = lens[i];
      const uint4* src = reinterpret_cast<const uint4*>(slots + i * kSlot);
      const uint4 q0 = src[0], q1 = src[1];
      const uint32_t qw[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int j = 0; j < kSlot; ++j) {
        if (j >= n) break;
        const uint32_t c = (qw[j >> 2] >> (8 * (j & 3))) & 0xFFu;
        const uint32_t xl = (lo ^ c) & 15u;
        const uint32_t K = (11u * xl + ((3u * xl) >> 4)) & 15u;
        const uint64_t x = H ^ (static_cast<uint64_t>(c >> 4) * kRep);
        H = nib_add(nib_mul3(x), static_cast<uint64_t>(K) * kRep);
        lo = (3u * xl) & 15u;
      }
    }
  }
  tmap[t] = H;
  const uint64_t bm = block_compose(H, sh);
  if (threadIdx.x == 0) bmap[blockIdx.x] = bm;
}

// (C) exact fold from the known low byte: affine map h_out = c + m * h_in
template <int R>
__global__ void __launch_bounds__(kT) dg_exact(const char* __restrict__ slots,
                                               const uint8_t* __restrict__ lens, int64_t segn,
                                               const uint64_t* __restrict__ tmap,
                                               const uint8_t* __restrict__ tlo,
                                               const uint8_t* __restrict__ bin,
                                               uint64_t* __restrict__ baff) {
  __shared__ uint64_t sh[kT / 32];
  __shared__ uint32_t shn[kT / 32];
  __shared__ uint64_t sc[kT / 32], sm[kT / 32];
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  const uint32_t hi_in = block_incoming(tmap[t], bin[blockIdx.x], sh, shn);
  const uint64_t l_in = (hi_in << 4) | tlo[t];
  uint64_t h = l_in, m = 1;
  const int64_t a = t * R;
  if (a < segn) {
    const int64_t b = min(segn, a + R);
    for (int64_t i = a; i < b; ++i) {
      const int n = lens[i];
      const uint4* src = reinterpret_cast<const uint4*>(slots + i * kSlot);
      const uint4 q0 = src[0], q1 = src[1];
      const uint32_t qw[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int j = 0; j < kSlot; ++j) {
        if (j >= n) break;
        h = (h ^ ((qw[j >> 2] >> (8 * (j & 3))) & 0xFFu)) * kP;
        m *= kP;
      }
    }
  }
  // h_out = h_local + m * (h_in - l_in)
  uint64_t c = h - m * l_in;
  // in-order reduction of (c, m): first (c1, m1) then (c2, m2) = (c2 + m2 c1, m2 m1)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t oc = __shfl_down_sync(0xffffffffu, c, d);
    const uint64_t om = __shfl_down_sync(0xffffffffu, m, d);
    if ((lane & (2 * d - 1)) == 0) {
      c = oc + om * c;
      m = om * m;
    }
  }
  if (lane == 0) sc[w] = c, sm[w] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t C = 0, Mm = 1;
    for (int i = 0; i < kT / 32; ++i) {
      C = sc[i] + sm[i] * C;
      Mm = sm[i] * Mm;
    }
    baff[2 * blockIdx.x] = C;
    baff[2 * blockIdx.x + 1] = Mm;
  }
}

__global__ void __launch_bounds__(1024) dg_finish(const uint64_t* __restrict__ baff, int nb,
                                                  uint64_t* __restrict__ state) {
  __shared__ uint64_t sc[1024], sm[1024];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  uint64_t C = 0, Mm = 1;
  for (int b = b0; b < b1; ++b) {
    C = baff[2 * b] + baff[2 * b + 1] * C;
    Mm = baff[2 * b + 1] * Mm;
  }
  sc[threadIdx.x] = C;
  sm[threadIdx.x] = Mm;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    if ((threadIdx.x & (2 * d - 1)) == 0) {
      const uint64_t c2 = sc[threadIdx.x + d], m2 = sm[threadIdx.x + d];
      sc[threadIdx.x] = c2 + m2 * sc[threadIdx.x];
      sm[threadIdx.x] = m2 * sm[threadIdx.x];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *state = sc[0] + sm[0] * *state;
}

__global__ void dg_init(uint64_t* state) { *state = kFnvBasis; }

}  // namespace

DeviceDigest::DeviceDigest(int64_t seg_values)
    : seg_((seg_values + kVB - 1) / kVB * kVB) {}

DeviceDigest::~DeviceDigest() {
  for (void* p : {static_cast<void*>(slots_), static_cast<void*>(lens_),
                  static_cast<void*>(tmap_), static_cast<void*>(tlo_),
                  static_cast<void*>(bmap_), static_cast<void*>(bin_),
                  static_cast<void*>(baff_)})
    if (p) cudaFree(p);
}

void DeviceDigest::ensure() {
  if (slots_) return;
  blocks_ = static_cast<int>(seg_ / kVB);
  const size_t threads = static_cast<size_t>(blocks_) * kT;
  PB_CUDA(cudaMalloc(&slots_, static_cast<size_t>(seg_) * kSlot));
  PB_CUDA(cudaMalloc(&lens_, static_cast<size_t>(seg_)));
  PB_CUDA(cudaMalloc(&tmap_, threads * 8));
  PB_CUDA(cudaMalloc(&tlo_, threads));
  PB_CUDA(cudaMalloc(&bmap_, static_cast<size_t>(blocks_) * 8));
  PB_CUDA(cudaMalloc(&bin_, static_cast<size_t>(blocks_)));
  PB_CUDA(cudaMalloc(&baff_, static_cast<size_t>(blocks_) * 16));
}

DeviceDigest::Plan DeviceDigest::make_plan(const std::vector<DigestSpan>& spans) {
  ensure();  // scratch now: enqueue may run under stream capture
  Plan p;
  std::vector<DigestSpan> v;
  int64_t at = 0;
  for (DigestSpan s : spans) {
    if (s.rows * s.cols == 0) continue;
    s.start = at;
    at += s.rows * s.cols;
    v.push_back(s);
  }
  p.nspans = static_cast<int>(v.size());
  p.total = at;
  if (!v.empty()) {
    PB_CUDA(cudaMalloc(&p.d_spans, v.size() * sizeof(DigestSpan)));
    PB_CUDA(cudaMemcpy(p.d_spans, v.data(), v.size() * sizeof(DigestSpan),
                       cudaMemcpyHostToDevice));
  }
  return p;
}

void DeviceDigest::free_plan(Plan& p) {
  if (p.d_spans) cudaFree(p.d_spans);
  p = Plan{};
}

int DeviceDigest::launches_per(const Plan& p) const {
  return 1 + static_cast<int>((p.total + seg_ - 1) / seg_) * 6;
}

void DeviceDigest::enqueue(const Plan& p, uint64_t* d_state, cudaStream_t st) {
  ensure();
  dg_init<<<1, 1, 0, st>>>(d_state);
  PB_CUDA(cudaGetLastError());
  for (int64_t s0 = 0; s0 < p.total; s0 += seg_) {
    const int64_t n = std::min(seg_, p.total - s0);
    // small segments: 4 values per thread (4x the blocks; fits the scratch
    // sized for 16 per thread when n <= seg / 4)
    const bool small = n * 4 <= seg_;
    const int64_t vb = small ? kT * 4 : kVB;
    const int nb = static_cast<int>((n + vb - 1) / vb);
    if (small) {
      dg_format_lo<4><<<nb, kT, 0, st>>>(p.d_spans, p.nspans, s0, n, slots_, lens_, tmap_, bmap_);
      dg_chain<<<1, 1024, 0, st>>>(bmap_, nb, d_state, 0, bin_);
      dg_hi<4><<<nb, kT, 0, st>>>(slots_, lens_, n, tmap_, tlo_, bin_, bmap_);
      dg_chain<<<1, 1024, 0, st>>>(bmap_, nb, d_state, 4, bin_);
      dg_exact<4><<<nb, kT, 0, st>>>(slots_, lens_, n, tmap_, tlo_, bin_, baff_);
    } else {
      dg_format_lo<kR><<<nb, kT, 0, st>>>(p.d_spans, p.nspans, s0, n, slots_, lens_, tmap_, bmap_);
      dg_chain<<<1, 1024, 0, st>>>(bmap_, nb, d_state, 0, bin_);
      dg_hi<kR><<<nb, kT, 0, st>>>(slots_, lens_, n, tmap_, tlo_, bin_, bmap_);
      dg_chain<<<1, 1024, 0, st>>>(bmap_, nb, d_state, 4, bin_);
      dg_exact<kR><<<nb, kT, 0, st>>>(slots_, lens_, n, tmap_, tlo_, bin_, baff_);
    }
    dg_finish<<<1, 1024, 0, st>>>(baff_, nb, d_state);
    PB_CUDA(cudaGetLastError());
  }
}

std::vector<DigestSpan> digest_spans_contiguous(const float* p, int64_t n) {
  DigestSpan s;
  s.f32 = p;
  s.rows = 1;
  s.cols = n;
  s.ld = n;
  return {s};
}

}  // namespace pb

// ------------------------------------------------------------------ C ABI
namespace {
__global__ void dg_format_only(const float* __restrict__ v, int64_t n, char* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  uint64_t w[4];
  pb::fmt::format_shortest_fast(static_cast<double>(v[i]), w);
  uint4* dst = reinterpret_cast<uint4*>(out + i * 32);
  dst[0] = make_uint4(static_cast<uint32_t>(w[0]), static_cast<uint32_t>(w[0] >> 32),
                      static_cast<uint32_t>(w[1]), static_cast<uint32_t>(w[1] >> 32));
  dst[1] = make_uint4(static_cast<uint32_t>(w[2]), static_cast<uint32_t>(w[2] >> 32),
                      static_cast<uint32_t>(w[3]), static_cast<uint32_t>(w[3] >> 32));
}
}  // namespace

extern "C" int pb_device_digest_f32(const float* values, int64_t n, char* out17, float* ms) {
  try {
    if (n < 0 || (n > 0 && !values) || !out17) throw std::invalid_argument("null argument");
    float* d = nullptr;
    uint64_t* st = nullptr;
    PB_CUDA(cudaMalloc(&d, std::max<int64_t>(1, n) * 4));
    PB_CUDA(cudaMalloc(&st, 8));
    if (n) PB_CUDA(cudaMemcpy(d, values, n * 4, cudaMemcpyHostToDevice));
    pb::DeviceDigest dd;
    auto plan = dd.make_plan(pb::digest_spans_contiguous(d, n));
    cudaEvent_t e0, e1;
    PB_CUDA(cudaEventCreate(&e0));
    PB_CUDA(cudaEventCreate(&e1));
    PB_CUDA(cudaEventRecord(e0, 0));
    dd.enqueue(plan, st, 0);
    PB_CUDA(cudaEventRecord(e1, 0));
    uint64_t h = 0;
    PB_CUDA(cudaMemcpy(&h, st, 8, cudaMemcpyDeviceToHost));
    float t = 0.f;
    PB_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dd.free_plan(plan);
    cudaFree(d);
    cudaFree(st);
    static const char kHex[] = "0123456789abcdef";
    for (int i = 15; i >= 0; --i, h >>= 4) out17[i] = kHex[h & 15];
    out17[16] = 0;
    return PB_OK;
  } catch (const std::exception& e) {
    pb::set_last_error(e.what());
    return dynamic_cast<const pb::cuda_failure*>(&e) ? PB_ERR_CUDA : PB_ERR_INVALID;
  }
}

extern "C" int pb_device_format_f32(const float* values, int64_t n, char* out) {
  try {
    if (n <= 0) return PB_OK;
    float* d = nullptr;
    char* o = nullptr;
    PB_CUDA(cudaMalloc(&d, n * 4));
    PB_CUDA(cudaMalloc(&o, n * 32));
    PB_CUDA(cudaMemcpy(d, values, n * 4, cudaMemcpyHostToDevice));
    dg_format_only<<<static_cast<unsigned>((n + 255) / 256), 256>>>(d, n, o);
    PB_CUDA(cudaGetLastError());
    PB_CUDA(cudaMemcpy(out, o, n * 32, cudaMemcpyDeviceToHost));
    cudaFree(d);
    cudaFree(o);
    return PB_OK;
  } catch (const std::exception& e) {
    pb::set_last_error(e.what());
    return dynamic_cast<const pb::cuda_failure*>(&e) ? PB_ERR_CUDA : PB_ERR_INVALID;
  }
}

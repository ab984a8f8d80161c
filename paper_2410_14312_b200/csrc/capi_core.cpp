// C ABI: error slot + device-layer entry points (include/pipesim_b200.h).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "conv_ops.cuh"
#include "layer_ops.cuh"
#include "pipesim_core.hpp"
#include "status.hpp"

namespace pb {

namespace {
thread_local std::string g_last_error;
thread_local std::string g_last_field;
thread_local int g_last_stage = 0;
thread_local int g_last_epoch = 0;
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

int translate_exception() {
  try {
    throw;
  } catch (const pipesim::domain_error& e) {
    g_last_error = e.what();
    g_last_field = e.field();
    return PB_ERR_DOMAIN;
  } catch (const pipesim::structural_error& e) {
    g_last_error = e.what();
    return PB_ERR_STRUCTURAL;
  } catch (const pipesim::insufficient_horizon_error& e) {
    g_last_error = e.what();
    return PB_ERR_INSUFFICIENT_HORIZON;
  } catch (const pipesim::integrity_error& e) {
    g_last_error = e.what();
    g_last_stage = e.stage_id();
    g_last_epoch = e.epoch();
    return PB_ERR_INTEGRITY;
  } catch (const pipesim::io_error& e) {
    g_last_error = e.what();
    return PB_ERR_IO;
  } catch (const cuda_failure& e) {
    g_last_error = e.what();
    return PB_ERR_CUDA;
  } catch (const capacity_error& e) {
    g_last_error = e.what();
    return PB_ERR_CAPACITY;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return PB_ERR_INVALID;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PB_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown exception";
    return PB_ERR_INTERNAL;
  }
}

}  // namespace pb

using pb::translate_exception;

#define PB_GUARD_BEGIN try {
#define PB_GUARD_END       \
  return PB_OK;            \
  }                        \
  catch (...) {            \
    return translate_exception(); \
  }

namespace {
int copy_out(const std::string& s, char* buf, int cap) {
  if (buf && cap > 0) {
    const size_t n = s.size() < static_cast<size_t>(cap - 1) ? s.size()
                                                            : static_cast<size_t>(cap - 1);
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return static_cast<int>(s.size());
}
inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
inline const __nv_bfloat16* bf(const uint16_t* p) {
  return reinterpret_cast<const __nv_bfloat16*>(p);
}
inline __nv_bfloat16* bfm(uint16_t* p) { return reinterpret_cast<__nv_bfloat16*>(p); }
}  // namespace

extern "C" {

int pb_last_error(char* buf, int cap) { return copy_out(pb::g_last_error, buf, cap); }
int pb_last_error_field(char* buf, int cap) {
  return copy_out(pb::g_last_field, buf, cap);
}
int pb_last_error_stage_epoch(int* stage, int* epoch) {
  if (stage) *stage = pb::g_last_stage;
  if (epoch) *epoch = pb::g_last_epoch;
  return PB_OK;
}

const char* pb_version(void) { return "pipesim-b200 0.1 (sm_100a)"; }

int pb_device_count(int* n) {
  PB_GUARD_BEGIN
  PB_CUDA(cudaGetDeviceCount(n));
  PB_GUARD_END
}

int pb_set_device(int device) {
  PB_GUARD_BEGIN
  PB_CUDA(cudaSetDevice(device));
  PB_GUARD_END
}

int pb_synchronize(void) {
  PB_GUARD_BEGIN
  PB_CUDA(cudaDeviceSynchronize());
  PB_GUARD_END
}

int pb_linear_fwd(void* stream, const uint16_t* x, int rows, int in, int ld_x,
                  const uint16_t* w, int out, int ld_w, const float* bias,
                  int act, uint16_t* y16, int ld_y16, float* y32, int ld_y32) {
  PB_GUARD_BEGIN
  pb::Mat16 mx{bf(x), rows, in, ld_x};
  pb::Mat16 mw{bf(w), out, in, ld_w};
  cudaStream_t st = as_stream(stream);
  // a skinny forward splits K on CTA pairs with the in-kernel fixup: its
  // workspace and (zeroed) tile counters live for this call only
  const size_t fix_floats = pb::fwd_fix_floats(rows, out, in);
  float* ws = nullptr;
  int* cnt = nullptr;
  if (fix_floats) {
    const size_t nc = static_cast<size_t>(pb::fwd_fix_counters(rows, out));
    PB_CUDA(cudaMallocAsync(&ws, fix_floats * 4 + nc * 4, st));
    cnt = reinterpret_cast<int*>(ws + fix_floats);
    PB_CUDA(cudaMemsetAsync(cnt, 0, nc * 4, st));
  }
  pb::GemmLaunch g = pb::plan_fwd(mx, 0, rows, mw, bias, act, bfm(y16), ld_y16,
                                  y32, ld_y32, 0, true, false, ws, cnt);
  pb::launch_fwd(g, st);
  if (ws) PB_CUDA(cudaFreeAsync(ws, st));
  PB_GUARD_END
}

int pb_linear_bwd_dx(void* stream, const uint16_t* dz, int rows, int out,
                     int ld_dz, const uint16_t* w, int in, int ld_w,
                     const uint16_t* xin, int ld_xin, int act_prev, uint16_t* d,
                     int ld_d) {
  PB_GUARD_BEGIN
  pb::Mat16 mdz{bf(dz), rows, out, ld_dz};
  pb::Mat16 mw{bf(w), out, in, ld_w};
  pb::GemmLaunch g =
      pb::plan_dgrad(mdz, mw, bf(xin), ld_xin, act_prev, bfm(d), ld_d);
  pb::launch_dgrad(g, as_stream(stream));
  PB_GUARD_END
}

int pb_linear_bwd_dw_sgd(void* stream, const uint16_t* dz, int rows, int out,
                         int ld_dz, const uint16_t* x, int in, int ld_x,
                         const float* w_cur, float* w_new, int ld_w32,
                         uint16_t* w16, int ld_w16, float lr) {
  PB_GUARD_BEGIN
  pb::Mat16 mdz{bf(dz), rows, out, ld_dz};
  pb::Mat16 mx{bf(x), rows, in, ld_x};
  pb::GemmLaunch g = pb::plan_wgrad_sgd(mdz, mx, 0, w_cur, w_new, ld_w32,
                                        bfm(w16), ld_w16, lr);
  pb::launch_wgrad(g, as_stream(stream));
  PB_GUARD_END
}

int pb_linear_bwd_dw_sgd_split(void* stream, const uint16_t* dz, int rows, int out, int ld_dz,
                               const uint16_t* x, int in, int ld_x, const uint16_t* hi_cur,
                               const uint16_t* lo_cur, uint16_t* hi_new, uint16_t* lo_new,
                               int ld, float lr) {
  PB_GUARD_BEGIN
  pb::Mat16 mdz{bf(dz), rows, out, ld_dz};
  pb::Mat16 mx{bf(x), rows, in, ld_x};
  pb::GemmLaunch g =
      pb::plan_wgrad_sgd_split(mdz, mx, 0, bf(hi_cur), lo_cur, bfm(hi_new), lo_new, ld, lr);
  pb::launch_wgrad(g, as_stream(stream));
  PB_GUARD_END
}

int pb_split_master(void* stream, const float* w, int out, int in, int ld_w, uint16_t* hi,
                    uint16_t* lo, int ld) {
  PB_GUARD_BEGIN
  pb::launch_split_master(as_stream(stream), w, out, in, ld_w, bfm(hi), lo, ld);
  PB_GUARD_END
}

int pb_join_master(void* stream, const uint16_t* hi, const uint16_t* lo, int out, int in, int ld,
                   float* w, int ld_w) {
  PB_GUARD_BEGIN
  pb::launch_join_master(as_stream(stream), bf(hi), lo, out, in, ld, w, ld_w);
  PB_GUARD_END
}

int pb_bias_sgd(void* stream, const uint16_t* dz, int rows, int out, int ld_dz,
                const float* b_cur, float* b_new, float* b_copy, float lr) {
  PB_GUARD_BEGIN
  pb::launch_bias_sgd(as_stream(stream), bf(dz), rows, out, ld_dz, b_cur, b_new,
                      b_copy, lr, nullptr, nullptr, 0);
  PB_GUARD_END
}

int pb_loss_fwd_bwd(void* stream, const float* y, int rows, int cols, int ld_y,
                    const float* targets, int ld_t, int loss, int act_last,
                    float denom, uint16_t* dz, int ld_dz, float* row_loss) {
  PB_GUARD_BEGIN
  pb::launch_loss(as_stream(stream), y, rows, cols, ld_y, targets, ld_t, loss,
                  act_last, denom, bfm(dz), ld_dz, row_loss);
  PB_GUARD_END
}

int pb_conv_fwd(void* stream, const uint16_t* x, int n, int h, int w, int cin,
                const uint16_t* wt, int cout, int ld_w, const float* bias, int act,
                uint16_t* y) {
  PB_GUARD_BEGIN
  pb::Nhwc t{bf(x), n, h, w, cin};
  pb::Mat16 mw{bf(wt), cout, 9 * cin, ld_w};
  pb::GemmLaunch g = pb::plan_conv_fwd(t, 0, n, mw, bias, act, bfm(y), 0);
  pb::launch_fwd(g, as_stream(stream));
  PB_GUARD_END
}

int pb_conv_bwd_dx(void* stream, const uint16_t* dz, int n, int h, int w, int cout,
                   const uint16_t* wt, int cin, int ld_w, const uint16_t* xin,
                   int act_prev, uint16_t* d) {
  PB_GUARD_BEGIN
  pb::Nhwc t{bf(dz), n, h, w, cout};
  pb::GemmLaunch g = pb::plan_conv_dgrad(t, bf(wt), cin, ld_w, bf(xin), act_prev, bfm(d));
  pb::launch_dgrad(g, as_stream(stream));
  PB_GUARD_END
}

int pb_conv_bwd_dw_sgd(void* stream, const uint16_t* dz, int n, int h, int w, int cout,
                       const uint16_t* x, int cin, const float* w_cur, float* w_new,
                       int ld_w32, uint16_t* w16, int ld_w16, float lr) {
  PB_GUARD_BEGIN
  const int pixels = n * h * w;
  const size_t floats = pb::conv_wgrad_floats(cout, cin, pixels);
  float* ws = nullptr;
  cudaStream_t st = as_stream(stream);
  PB_CUDA(cudaMallocAsync(&ws, floats * 4, st));
  pb::ConvWgradInfo info;
  pb::Mat16 mdz{bf(dz), pixels, cout, cout};
  pb::GemmLaunch g = pb::plan_conv_wgrad_partial(mdz, pb::Nhwc{bf(x), n, h, w, cin}, 0, ws, &info);
  pb::launch_wgrad_partial(g, st);
  pb::launch_reduce_sgd(st, ws, info.splits, info.slab, cout, 9 * cin, info.lds, w_cur, w_new,
                        ld_w32, bfm(w16), ld_w16, lr, info.transposed);
  PB_CUDA(cudaFreeAsync(ws, st));
  PB_GUARD_END
}

int pb_maxpool2_fwd(void* stream, const uint16_t* in, int n, int h, int w, int c,
                    uint16_t* out) {
  PB_GUARD_BEGIN
  pb::launch_maxpool2_fwd(as_stream(stream), bf(in), n, h, w, c, bfm(out));
  PB_GUARD_END
}

int pb_maxpool2_bwd(void* stream, const uint16_t* d_out, const uint16_t* in,
                    const uint16_t* out, int n, int h, int w, int c, uint16_t* d_in) {
  PB_GUARD_BEGIN
  pb::launch_maxpool2_bwd(as_stream(stream), bf(d_out), bf(in), bf(out), n, h, w, c, bfm(d_in));
  PB_GUARD_END
}

int pb_im2col_first(void* stream, const uint16_t* x, int ld_x, int n, int h, int w, int c,
                    uint16_t* out, int ldo) {
  PB_GUARD_BEGIN
  pb::launch_im2col_first(as_stream(stream), bf(x), ld_x, n, h, w, c, bfm(out), ldo);
  PB_GUARD_END
}

int pb_convert_f64_to_bf16(void* stream, const double* src, int rows, int cols,
                           int ld_src, uint16_t* dst, int ld_dst) {
  PB_GUARD_BEGIN
  pb::launch_convert_f64_bf16(as_stream(stream), src, rows, cols, ld_src,
                              bfm(dst), ld_dst);
  PB_GUARD_END
}

int pb_convert_f32_to_bf16(void* stream, const float* src, int rows, int cols,
                           int ld_src, uint16_t* dst, int ld_dst) {
  PB_GUARD_BEGIN
  pb::launch_convert_f32_bf16(as_stream(stream), src, rows, cols, ld_src,
                              bfm(dst), ld_dst);
  PB_GUARD_END
}

}  // extern "C"

/*
 * pipesim_b200.h — C ABI of the B200-native TiMePReSt pipeline step.
 *
 * Plain C: int status codes, plain pointers and sizes, no C++ or torch types.
 * Every function returns PB_OK (0) or one of the PB_ERR_* codes below and
 * leaves a message retrievable with pb_last_error() (thread-local).
 *
 * The reference ("pipesim", /root/reference/proj) has no FFI: its boundary is
 * the C++ API in proj/include/pipesim/ (*.hpp).  This header is the thin layer
 * that (a) the drop-in C++ API (include/pipesim/pipesim_b200.hpp) calls into,
 * and (b) a foreign-language host binds (the Python mirror in
 * paper_2410_14312_b200/pipesim.py binds it with ctypes).  Each entry point
 * cites the reference interface it replaces.
 */
#ifndef PIPESIM_B200_H_
#define PIPESIM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes
 * Mirrors the reference's exception taxonomy (proj/include/pipesim/errors.hpp:25-65). */
enum {
  PB_OK = 0,
  PB_ERR_DOMAIN = 1,               /* pipesim::domain_error              */
  PB_ERR_STRUCTURAL = 2,           /* pipesim::structural_error          */
  PB_ERR_INSUFFICIENT_HORIZON = 3, /* pipesim::insufficient_horizon_error */
  PB_ERR_INTEGRITY = 4,            /* pipesim::integrity_error           */
  PB_ERR_IO = 5,                   /* pipesim::io_error                  */
  PB_ERR_CUDA = 6,                 /* CUDA runtime / driver failure      */
  PB_ERR_CAPACITY = 7,             /* caller buffer too small            */
  PB_ERR_INVALID = 8,              /* bad argument                       */
  PB_ERR_INTERNAL = 9
};

/* Copies the calling thread's last error message (NUL-terminated, truncated
 * to cap). Returns the full message length. */
int pb_last_error(char* buf, int cap);
/* Field name carried by the last PB_ERR_DOMAIN (domain_error::field()). */
int pb_last_error_field(char* buf, int cap);
/* Stage / epoch carried by the last PB_ERR_INTEGRITY. */
int pb_last_error_stage_epoch(int* stage, int* epoch);

const char* pb_version(void);

/* ------------------------------------------------------------ plan layer
 * Host-side schedule / version ledger.  Bit-exact with the reference. */

typedef struct {
  int workers;              /* W */
  int micro_batches;        /* N */
  int mini_batches;         /* M */
  double backward_cost_factor;
  int samples_per_mini_batch;
  uint64_t seed;
} pb_sim_config;            /* proj/include/pipesim/config.hpp:32-40 */

enum { PB_MODE_TIMEPREST = 0, PB_MODE_PIPEDREAM = 1 };      /* schedule_mode */
enum { PB_TASK_IDLE = 0, PB_TASK_FORWARD = 1, PB_TASK_BACKWARD = 2 };

typedef struct { int kind, mini, micro; } pb_task;           /* schedule.hpp:34-44 */
typedef struct { int version, mini, stage, slot; } pb_commit; /* ledger.hpp:31-36 */
typedef struct { int mini, micro, slot, version; } pb_pin;    /* ledger.hpp:38-43 */
typedef struct { int mini, stage, slot, version; } pb_consume;/* ledger.hpp:45-50 */
typedef struct { int version, from_slot, freed_slot; } pb_interval; /* ledger.hpp:104-108 */

/* validate(sim_config) — config.hpp:44-62. */
int pb_validate_config(const pb_sim_config* cfg);

/* build_nf1b_schedule / build_1f1b_schedule — schedule.hpp:84,89.
 * cells is row-major [W][cap_slots]; *horizon is always set.  Returns
 * PB_ERR_CAPACITY when cap_slots < horizon (cells untouched). */
int pb_schedule_build(const pb_sim_config* cfg, int mode, int* horizon,
                      pb_task* cells, int cap_slots);

/* validate_schedule — schedule.hpp:108-109.  Violations are data: kinds[i]
 * (0 task_invariant, 1 stage_continuity, 2 completeness, 3 backward_priority)
 * and '\n'-separated messages. */
/* Schedule document JSON of build_*_schedule(cfg) and its ledger
 * (export.cpp:78-139; reference `pipesim simulate --json`). */
int pb_schedule_document(const pb_sim_config* cfg, int mode, char* buf, int64_t cap,
                         int64_t* len);
int pb_schedule_validate(const pb_sim_config* cfg, int mode,
                         const pb_task* cells, int horizon, int* n_violations,
                         int* kinds, int cap_kinds, char* messages,
                         int cap_messages);

/* assign_versions — ledger.hpp:70-71.  Output arrays are caller-owned:
 * commits[M*W], pins[M*units] (units = N for timeprest, 1 for pipedream),
 * consumptions[M*W], update_source[M], full_commit_slot[M+1]. */
int pb_assign_versions(const pb_sim_config* cfg, int mode, const pb_task* cells,
                       int horizon, pb_commit* commits, pb_pin* pins,
                       pb_consume* consumptions, int* update_source,
                       int* full_commit_slot);

/* measure_version_difference — ledger.hpp:77-78 (reads update_source). */
int pb_measure_version_difference(const pb_sim_config* cfg,
                                  const int* update_source, int strict,
                                  int* v);
int pb_closed_form_v(int workers, int micro_batches, int* v);   /* :81 */
int pb_forward_span(int workers, int micro_batches, int mini_ordinal,
                    int* span);                                 /* :85 */
int pb_backward_span(int workers, int* span);                   /* :88 */
int pb_overlap_condition(int workers, int micro_batches, int* out); /* :92 */

/* decompose_sequences — ledger.hpp:101-102.  seq_mini[] holds the chains
 * back to back, seq_len[] their lengths. */
int pb_decompose_sequences(const pb_sim_config* cfg, const int* update_source,
                           int mini_batches, int* n_sequences, int* seq_len,
                           int* seq_mini, int* v_measured);

/* build_retention_timeline — ledger.hpp:119-120.  intervals is
 * [W][M+1]; peak[W]. */
int pb_retention_timeline(const pb_sim_config* cfg, int mode,
                          const pb_task* cells, int horizon, const pb_pin* pins,
                          pb_interval* intervals, int* peak);

/* staleness_report — ledger.hpp:138. staleness[i] matches consumptions[i]. */
int pb_staleness(const pb_sim_config* cfg, const pb_commit* commits,
                 const pb_consume* consumptions, int* staleness);

/* ------------------------------------------------------------ model helpers
 * partition_model / init_network_params / make_synthetic_task
 * (trainer.hpp:89-115) and the digest (trainer.hpp:106). */

enum { PB_ACT_LINEAR = 0, PB_ACT_RELU = 1, PB_ACT_TANH = 2, PB_ACT_SIGMOID = 3 };
enum { PB_LOSS_MSE = 0, PB_LOSS_SOFTMAX_CE = 1 };

typedef struct {
  int n_layers;
  const int* widths;       /* n_layers + 1 */
  const int* activations;  /* n_layers, PB_ACT_* */
  int loss;                /* PB_LOSS_* */
} pb_net_spec;             /* trainer.hpp:55-64 */

/* stage_layers[s] = number of layers of stage s+1, first_layer[s] likewise. */
int pb_partition_model(const pb_net_spec* net, int workers, int* first_layer,
                       int* n_layers);
int64_t pb_param_count(const pb_net_spec* net);
int pb_init_network_params(const pb_net_spec* net, uint64_t seed, double* out,
                           int64_t n);
int pb_make_synthetic_task(int samples, uint64_t seed, double* x, double* y);
/* FNV-1a over shortest round-trip decimals ("%.17g"-free, std::to_chars) of
 * values[0..n) each followed by '\n'; out receives 16 hex chars + NUL. */
int pb_params_digest(const double* values, int64_t n, char* out17);
/* The same digest computed on the current CUDA device (digest_dev.hpp:
 * device shortest-decimal formatting + parallel FNV-1a fold), for values
 * given as fp32 (host memory; each is formatted as the double it widens to,
 * as the reference's fp64 params that hold these values would be).
 * ms (optional) = device time of the digest kernels. */
int pb_device_digest_f32(const float* values, int64_t n, char* out17, float* ms);
/* Device shortest round-trip formatting (shortest.cuh) of fp32 values as
 * doubles, for tests against std::to_chars: out[i*32 ..] holds the text of
 * values[i] (NUL-padded). */
int pb_device_format_f32(const float* values, int64_t n, char* out);

/* checkpoint_stage / restore_stage (checkpoint.hpp:29-44; file format of
 * checkpoint.cpp:39-153).  A stage is its id, first layer, n_layers
 * (in, out, PB_ACT_*) triples in `layers`, and the current version's flat
 * params (per layer W out x in, then b).  Errors: PB_ERR_IO (cannot write),
 * PB_ERR_INTEGRITY (missing / truncated / tampered / wrong stage or epoch;
 * pb_last_error_stage_epoch names the expected stage and epoch). */
int pb_checkpoint_stage(int stage_id, int first_layer, int n_layers, const int* layers,
                        int version, const double* params, int64_t n, int loss, int epoch,
                        const char* path);
typedef struct {
  int stage_id, first_layer, n_layers, version, loss, epoch;
  int64_t n_values;
} pb_restored_stage;
int pb_restore_stage(const char* path, int expected_stage, int expected_epoch,
                     pb_restored_stage* info, int* layers, int layers_cap, double* params,
                     int64_t cap);

/* ------------------------------------------------------------ device layer
 * Per-op kernels on device pointers (bf16 = uint16 storage).  `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Leading dimensions are in
 * elements and must be multiples of 8 for bf16 operands (TMA 16-byte rule). */

int pb_device_count(int* n);
int pb_set_device(int device);
int pb_synchronize(void);

/* y = act(x * w^T + b).  x: rows x in (ld_x), w: out x in (ld_w),
 * y16 (bf16, may be NULL) and/or y32 (fp32, may be NULL).  Replaces the
 * forward loop nest of stage_forward (trainer.cpp:186-204). */
int pb_linear_fwd(void* stream, const uint16_t* x, int rows, int in, int ld_x,
                  const uint16_t* w, int out, int ld_w, const float* bias,
                  int act, uint16_t* y16, int ld_y16, float* y32, int ld_y32);

/* d = (dz * w) .* act'(xin).  dz: rows x out, w: out x in, xin: rows x in
 * (activation the layer consumed, act' recovered from it), d: rows x in.
 * Replaces stage_backward's delta loop (trainer.cpp:239-242, :255-262). */
int pb_linear_bwd_dx(void* stream, const uint16_t* dz, int rows, int out,
                     int ld_dz, const uint16_t* w, int in, int ld_w,
                     const uint16_t* xin, int ld_xin, int act_prev, uint16_t* d,
                     int ld_d);

/* w_new = w_cur - lr * dz^T x ; w16 = bf16(w_new).  w_cur may equal w_new.
 * Replaces the dW loop (trainer.cpp:244-249) fused with SGD (:484-488). */
int pb_linear_bwd_dw_sgd(void* stream, const uint16_t* dz, int rows, int out,
                         int ld_dz, const uint16_t* x, int in, int ld_x,
                         const float* w_cur, float* w_new, int ld_w32,
                         uint16_t* w16, int ld_w16, float lr);

/* Split fp32 masters (the session's default for layers with out > 128):
 * master = bits(hi) << 16 + lo (exact), hi the version's bf16 weights, lo a
 * 16-bit residual.  master_new = master_cur - lr * dz^T x, written as
 * hi_new / lo_new.  All four are out x in, leading dimension ld (multiple of
 * 8).  Same replacement as pb_linear_bwd_dw_sgd. */
int pb_linear_bwd_dw_sgd_split(void* stream, const uint16_t* dz, int rows, int out, int ld_dz,
                               const uint16_t* x, int in, int ld_x, const uint16_t* hi_cur,
                               const uint16_t* lo_cur, uint16_t* hi_new, uint16_t* lo_new,
                               int ld, float lr);
/* fp32 out x in (ld_w) <-> split master (hi, lo; ld). */
int pb_split_master(void* stream, const float* w, int out, int in, int ld_w, uint16_t* hi,
                    uint16_t* lo, int ld);
int pb_join_master(void* stream, const uint16_t* hi, const uint16_t* lo, int out, int in, int ld,
                   float* w, int ld_w);

/* b_new = b_cur - lr * colsum(dz); b_copy (may be NULL) = b_new.
 * Replaces trainer.cpp:250-252 + :484-488 for the bias. */
int pb_bias_sgd(void* stream, const uint16_t* dz, int rows, int out, int ld_dz,
                const float* b_cur, float* b_new, float* b_copy, float lr);

/* Fused loss + gradient over the stacked mini-batch output (loss_mean +
 * loss_grad, trainer.cpp:270-312): y rows x cols (fp32), targets rows x cols
 * (fp32), dz = dL/dy / denom .* act'(y) (bf16), row_loss[r] = per-row sum. */
int pb_loss_fwd_bwd(void* stream, const float* y, int rows, int cols, int ld_y,
                    const float* targets, int ld_t, int loss, int act_last,
                    float denom, uint16_t* dz, int ld_dz, float* row_loss);

/* ---- VGG-style conv stages (BASELINE configs[3]; no reference counterpart,
 * SPEC.md:379).  NHWC bf16 activations [n][h][w][c]; 3x3 convolution, pad 1,
 * stride 1; weights [cout][ld_w] bf16 with K = (3r + s) * cin + c (tap-major),
 * ld_w >= 9 * cin.  cin and cout multiples of 64 (the network input goes
 * through pb_im2col_first + the Linear kernels). */
/* y[n*h*w, cout] = act(conv(x, w) + b) (implicit GEMM: im2col TMA operand). */
int pb_conv_fwd(void* stream, const uint16_t* x, int n, int h, int w, int cin,
                const uint16_t* wt, int cout, int ld_w, const float* bias, int act,
                uint16_t* y);
/* d[n*h*w, cin] = conv_transpose(dz, w) .* act'(xin). */
int pb_conv_bwd_dx(void* stream, const uint16_t* dz, int n, int h, int w, int cout,
                   const uint16_t* wt, int cin, int ld_w, const uint16_t* xin,
                   int act_prev, uint16_t* d);
/* w_new = w_cur - lr * dW, dW[cout, 9*cin] = sum_p dz[p]^T im2col(x)[p]
 * (split-K fp32 partial slabs, then an in-order reduction fused with SGD);
 * w16 (may be NULL) = bf16(w_new).  w_cur / w_new fp32 [cout][ld_w32]. */
int pb_conv_bwd_dw_sgd(void* stream, const uint16_t* dz, int n, int h, int w, int cout,
                       const uint16_t* x, int cin, const float* w_cur, float* w_new,
                       int ld_w32, uint16_t* w16, int ld_w16, float lr);
/* 2x2 max pooling, stride 2 (gradient to the first maximum of a window). */
int pb_maxpool2_fwd(void* stream, const uint16_t* in, int n, int h, int w, int c,
                    uint16_t* out);
int pb_maxpool2_bwd(void* stream, const uint16_t* d_out, const uint16_t* in,
                    const uint16_t* out, int n, int h, int w, int c, uint16_t* d_in);
/* out[n*h*w, ldo] = im2col of a narrow NHWC input (k = (3r+s)*c + ch, zero
 * padded to ldo); x rows of ld_x elements per image. */
int pb_im2col_first(void* stream, const uint16_t* x, int ld_x, int n, int h, int w, int c,
                    uint16_t* out, int ldo);

/* Elementwise conversions used at the host boundary. */
int pb_convert_f64_to_bf16(void* stream, const double* src, int rows, int cols,
                           int ld_src, uint16_t* dst, int ld_dst);
int pb_convert_f32_to_bf16(void* stream, const float* src, int rows, int cols,
                           int ld_src, uint16_t* dst, int ld_dst);


/* ------------------------------------------------------------ pipeline session
 * The B200 executor of the pipeline-parallel training step: train_epoch ->
 * replay_grid (proj/src/trainer.cpp:642-660, :388-508) and sequential_epoch
 * (:510-553).  A session keeps every stage's weights, version pool and
 * activation slots resident in HBM; the caller moves data in and results out. */

typedef struct pb_session pb_session;

enum { PB_TRAIN_TIMEPREST = 0, PB_TRAIN_PIPEDREAM = 1, PB_TRAIN_SEQUENTIAL = 2 };
enum { PB_DTYPE_F64 = 0, PB_DTYPE_F32 = 1, PB_DTYPE_LABELS_I32 = 2,
       PB_DTYPE_BF16 = 3 /* x only: bf16 rows (RNE-rounded), bf16 precision sessions */ };

typedef struct {
  int workers;          /* W (stages) */
  int micro_batches;    /* N */
  int mini_batch_size;  /* B, divisible by N */
  int mini_batches;     /* M per epoch */
  double learning_rate;
  int mode;             /* PB_TRAIN_* */
  int device;           /* CUDA device of all stages */
  int use_graph;        /* capture the epoch as one CUDA graph */
  int snapshots;        /* keep fp32 host snapshots of every committed version */
  int fwd_merge;        /* max micro-batches per coalesced forward launch (0 = N) */
  int timed_kernel;     /* PB_KT_*: CUDA events around every launch of that GEMM
                           inside the epoch (also inside the graph) */
  int transport;        /* multi-process split: PB_TRANSPORT_* */
  int precision;        /* PB_PRECISION_*: bf16 tensor cores (fp32 accumulate,
                           fp32 masters) or the fp32 FFMA verify mode */
  int digests;          /* params_digest on the device inside the epoch: after
                           every mini-batch's stage-1 commit and at the end
                           (trainer.cpp:492-501, :506); pb_session_digests */
} pb_train_config;      /* train_config, trainer.hpp:117-126 */

enum { PB_PRECISION_BF16 = 0, PB_PRECISION_FP32_VERIFY = 1 };

enum { PB_TRANSPORT_NCCL = 0, PB_TRANSPORT_IPC = 1 };

enum { PB_KT_NONE = 0, PB_KT_FWD = 1, PB_KT_DGRAD = 2, PB_KT_WGRAD = 3 };

typedef struct {
  double* mini_loss;  /* [M] loss of each mini-batch before its update */
  int* pinned;        /* [M*units] forward versions (ledger) */
  int* consumed;      /* [M] update_source (ledger) */
  int* dev_fwd;       /* [M*units*W] version tags read by forwards, on device */
  int* dev_bwd;       /* [M*W] version tags propagated through by backwards */
  int* dev_current;   /* [W] current version per stage after the epoch */
  float device_ms;    /* device time of the epoch (CUDA events) */
} pb_epoch_out;       /* epoch_log / mini_log, trainer.hpp:133-147 (+ device trace) */

typedef struct {
  int horizon;
  int units;             /* N for timeprest, 1 otherwise */
  int kernels_per_epoch; /* our kernel launches per epoch */
  int64_t device_bytes;
  int64_t param_count;
  int* pool_sizes;       /* [W] (optional) weight versions held per stage */
  int* act_slots;        /* [W] (optional) activation slots per stage */
  int* stage_first_layer;/* [W] (optional) */
  int* stage_layers;     /* [W] (optional) */
} pb_session_info;

int pb_session_create(const pb_net_spec* net, const pb_train_config* cfg,
                      pb_session** out);
int pb_session_destroy(pb_session* s);
int pb_session_info_get(pb_session* s, pb_session_info* info);
/* load_network_params(stages, flat, 0) — trainer.hpp:99-100 */
int pb_session_load_params(pb_session* s, const double* flat, int64_t n);
/* The same for one stage (1-based): its W then b per layer, n = the stage's
 * parameter count (stage_model::current_params(), trainer.hpp:81-83). */
int pb_session_load_stage_params(pb_session* s, int stage, const double* p, int64_t n);
/* gather_network_params — trainer.hpp:102-103 (current versions, fp32 -> f64) */
int pb_session_read_params(pb_session* s, double* flat, int64_t n);
/* Host (pinned or pageable) -> HBM copy of an epoch's data: x [M*B][in],
 * y [M*B][out] (f64/f32) or [M*B] int32 class labels (one-hot implied). */
int pb_session_upload(pb_session* s, const void* x, int x_dtype, const void* y,
                      int y_dtype);
/* One epoch over the uploaded data (the pipeline step). */
int pb_session_run_epoch(pb_session* s, pb_epoch_out* out);
/* upload + run_epoch. */
int pb_session_train_epoch(pb_session* s, const void* x, int x_dtype,
                           const void* y, int y_dtype, pb_epoch_out* out);
/* Per-node timeline of one epoch (pipeline bubble).  A node is one backward
 * task or one coalesced run of forward tasks of a stage; its span is taken
 * on its stage stream after its cross-stage waits.  Arrays are caller
 * allocated with max_nodes entries (n_nodes reports the count; stage_busy_ms
 * has W entries, -1 for stages on other GPUs). */
typedef struct {
  float makespan_ms;
  float* stage_busy_ms;
  int max_nodes;
  int n_nodes;
  int* node_stage;      /* 1-based */
  int* node_fwd;        /* 1 forward run, 0 backward */
  int* node_mini;
  int* node_micro_lo;   /* 0-based micro-batch range of a forward run */
  int* node_micro_hi;
  float* node_start_ms;
  float* node_end_ms;
} pb_epoch_profile;

/* Device durations (ms) of the timed GEMM's launches in the last epoch, in
 * issue order (pb_train_config.timed_kernel), and each launch's algorithmic
 * flops (2*M*N*K; optional); *n = count (<= max written). */
int pb_session_kernel_times(pb_session* s, float* ms, double* flops, int max, int* n);

/* Schedule document JSON (reference export.cpp:78-139) of the last epoch,
 * with the version numbers observed on the device (pins; timeprest
 * consumptions).  *len = bytes (without the terminating NUL). */
int pb_session_trace_document(pb_session* s, char* buf, int64_t cap, int64_t* len);

/* One epoch without the CUDA graph, with CUDA timing events around every
 * node (for the bubble report; slower than run_epoch). */
int pb_session_profile_epoch(pb_session* s, pb_epoch_out* out, pb_epoch_profile* prof);

/* fp32 snapshot of stage `stage` (1-based) at `version`, widened to f64. */
int pb_session_snapshot(pb_session* s, int stage, int version, double* out,
                        int64_t n);

/* Committed weights of `version` on `stage` after an epoch: versions M and
 * M-1 from the fp32 masters, any version from snapshots (if enabled). */
int pb_session_read_version(pb_session* s, int stage, int version, double* out,
                            int64_t n);

/* ------------------------------------------------------------ multi-GPU
 * One process per GPU; the W stages are split into contiguous ranges (rank r
 * owns stages [r*W/world, (r+1)*W/world)).  Activations (stage s -> s+1) and
 * deltas (s+1 -> s) cross GPU boundaries point to point over NVLink (NCCL
 * send/recv, one 2-rank communicator per boundary and direction). */

/* CUDA IPC peer-memory transport (transport = PB_TRANSPORT_IPC): each rank
 * exports a blob (IPC handles of its slot arena and handshake flags plus its
 * transfer list), the caller exchanges them, then every rank connects with
 * all blobs (concatenated, lens[r] bytes each) before its first epoch.  Works
 * across NVLink peers and for several processes on one GPU.  Epochs run
 * without the CUDA graph (the handshake values advance per epoch). */
int pb_session_ipc_export(pb_session* s, uint8_t* buf, int64_t cap, int64_t* len);
int pb_session_ipc_connect(pb_session* s, const uint8_t* blobs, const int64_t* lens, int world);

/* Writes one NCCL unique id (128 bytes).  Rank 0 makes 2*(world-1) of them
 * and shares them (e.g. torch.distributed broadcast). */
int pb_nccl_unique_id(uint8_t* out128);

/* ---- convolutional networks (VGG-style stages, BASELINE configs[3]; the
 * reference's networks are MLPs only, so this is an extension
 * of pb_session_create with the same session entry points afterwards).
 * A network is conv layers then linear layers; the first linear layer reads
 * the last conv output flattened in NHWC order.  conv3x3: `in` -> `out`
 * channels on height x width NHWC images, pad 1, stride 1, activation, then
 * (pool != 0) 2x2 / stride-2 max pooling; weights [out][9*in] with
 * k = (3r + s) * in + c, then b[out].  Input rows are NHWC images
 * (height*width*in values).  Channel counts: out % 64 == 0; in % 64 == 0
 * except a first layer with in <= 8. */
enum { PB_LAYER_LINEAR = 0, PB_LAYER_CONV3X3 = 1 };
typedef struct {
  int kind;           /* PB_LAYER_* */
  int in, out;        /* features (linear) or channels (conv) */
  int height, width;  /* conv: input image size */
  int pool;           /* conv: 2x2 max pooling after the activation */
  int act;            /* PB_ACT_* */
} pb_layer_spec;
typedef struct {
  int n_layers;
  const pb_layer_spec* layers;
  int loss;                 /* PB_LOSS_* */
  const int* stage_layers;  /* [workers] layers per stage, or NULL: the
                               flop-balanced partition (pb_partition_layers) */
} pb_layer_net;
/* Contiguous partition minimising the largest stage's forward flops. */
int pb_partition_layers(const pb_layer_net* net, int workers, int* first_layer,
                        int* n_layers);
/* A session for a layer network (rank / world / nccl_ids as
 * pb_session_create_dist; world 1 = every stage in this process). */
int pb_session_create_layers(const pb_layer_net* net, const pb_train_config* cfg,
                             int rank, int world, const uint8_t* nccl_ids,
                             size_t ids_bytes, pb_session** out);

/* pb_session_create for one rank of a world-size pipeline. */
int pb_session_create_dist(const pb_net_spec* net, const pb_train_config* cfg,
                           int rank, int world, const uint8_t* nccl_ids,
                           size_t ids_bytes, pb_session** out);

/* The point-to-point transfers one rank's program issues, in order, without
 * touching a GPU: kinds[i] 1 = send / 0 = recv, dirs[i] 0 = activation /
 * 1 = delta, peers[i], bytes[i].  *n = count (call with cap 0 to size). */
int pb_plan_transfers(const pb_net_spec* net, const pb_train_config* cfg,
                      int rank, int world, int* n, int* kinds, int* dirs,
                      int* peers, int64_t* bytes, int cap);

/* Device memory one rank's session holds per stage, without touching a GPU
 * (the session's own arena layout): weight_bytes[s] = weight versions (the
 * bf16 version pool + fp32 masters, split or whole), act_bytes[s] =
 * activations kept for the backward (activation slots, scratch deltas,
 * boundary buffers, logits); pool[s] / act_slots[s] = weight versions /
 * mini-batch activation sets held at peak.  Stages other ranks own get 0.
 * The per-stage figures behind the slot model's memory_footprint
 * (proj/src/metrics.cpp:73-101: peak retained versions x params + peak
 * stashed samples x width).  Arrays have W entries; any may be NULL. */
int pb_plan_memory(const pb_net_spec* net, const pb_train_config* cfg, int rank,
                   int world, int64_t* weight_bytes, int64_t* act_bytes, int* pool,
                   int* act_slots);

/* The M + 1 digests of the last epoch of a session created with digests = 1:
 * hex[17*i ..] = 16 hex chars + NUL of mini-batch i+1's checksum
 * (mini_log::checksum), the last one the epoch's final checksum.  cap = the
 * number of 17-byte entries hex holds. */
int pb_session_digests(pb_session* s, char* hex, int64_t cap);
/* params_digest (trainer.cpp:599-607) of every stage's `version` (0 after
 * load, M after an epoch), computed on the device; out17 = 16 hex + NUL. */
int pb_session_params_digest(pb_session* s, int version, char* out17);

/* Synthetic classification data: x ~ U[0,1) from
 * mt19937_64(seed) row-major via (rng()>>11)*2^-53, then labels rng() % C.
 * Either of x64 / x32 / labels may be NULL. */
int pb_make_classification_task(int rows, int features, int classes,
                                uint64_t seed, double* x64, float* x32,
                                int* labels);

#ifdef __cplusplus
}
#endif

#endif /* PIPESIM_B200_H_ */

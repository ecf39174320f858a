/*
 * parastep_b200 — C-ABI of the B200-native ParaStep hot path.
 *
 * The reference (pkg/src/parastep, pure Python/numpy) has no FFI; its
 * drop-in boundary is the Python module API bound by name at import:
 *   - predictor.forward / forward_batch      (engines.py:40, worker.py:45)
 *   - schedule.ddpm_step                      (engines.py:41, worker.py:46)
 *   - numerics.draw_normal / RngStream        (engines.py:172-179)
 * Each entry point below replaces the arithmetic behind one of those
 * functions; the Python package paper_2505_14741_b200 restores the
 * reference's signatures and exceptions on top of it (ctypes binding in
 * paper_2505_14741_b200/_lib.py; INTEGRATION.md shows the binding).
 *
 * Conventions: all pointers are DEVICE pointers unless named host_*; every
 * call is asynchronous on the given cudaStream_t (passed as void*), never
 * synchronises, never allocates on a hot call. Return 0 on success, else a
 * PS_E* / cudaError_t code; ps_last_error() gives the message (thread-local).
 */
#ifndef PARASTEP_B200_H
#define PARASTEP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types of sampler state / noise vectors */
enum { PS_F64 = 0, PS_F32 = 1, PS_BF16 = 2 };

/* error codes (besides cudaError_t values) */
enum {
  PS_OK = 0,
  PS_EINVAL = 1001,  /* bad argument: maps to DimensionError/ParameterError */
  PS_ECUDA = 1002,   /* CUDA runtime error */
  PS_EUNSUP = 1003   /* unsupported dtype/shape combination */
};

#define PS_MAX_CYCLE 16

/* One reverse step t (schedule.py:102-131): out = (x - c*eps)/sqrt_a
 * (+ sigma*z_t when noisy). Coefficients are computed on the host in Python
 * float64 exactly as posterior_mean does (math.sqrt, correctly rounded). */
typedef struct ps_step {
  double c;       /* (1 - alpha_t) / sqrt(1 - alpha_bar_t) */
  double sqrt_a;  /* sqrt(alpha_t) */
  double sigma;   /* sigma_t */
  int32_t t;      /* step index, selects z stream (STEP<<32)|t */
  int32_t noisy;  /* 0 when t == 1 or sigma_mode == "zero" */
} ps_step;

const char* ps_last_error(void);
int ps_version(void);
int ps_sm_count(int device);

/* ---- counter RNG (numerics.py:30-120) ------------------------------------
 * out[i] = draw at counter counter0+i of (seed, stream). Integer part
 * (SplitMix64) is bit-exact; uniform() is bit-exact; normal() uses fp64
 * log/sqrt/sincos (<= 2 ulp from numpy). dtype: PS_F64 or PS_F32. */
int ps_rng_normal(void* out, int64_t n, uint64_t seed, uint64_t stream, uint64_t counter0,
                  int dtype, void* cuda_stream);
/* same, seed read from device memory (CUDA-graph replayable per seed) */
int ps_rng_normal_dev(void* out, int64_t n, const uint64_t* d_seed, uint64_t stream,
                      uint64_t counter0, int dtype, void* cuda_stream);
int ps_rng_uniform(void* out, int64_t n, uint64_t seed, uint64_t stream, uint64_t counter0,
                   int dtype, void* cuda_stream);
/* Xavier-uniform weight init (predictor.py:202-215): out[i] = (2u_i - 1)*limit */
int ps_rng_xavier(void* out, int64_t n, uint64_t seed, uint64_t stream, double limit,
                  int dtype, void* cuda_stream);

/* ---- fused scheduler: the reuse-then-predict round -----------------------
 * One launch does, per element (chain held in fp64 registers, no FMA
 * contraction, z_t generated in-register from d_seed):
 *   1) APPLY: x = x_in; for k < n_apply: rec_x[k] <- x (if non-NULL);
 *             x = step(x, eps_apply[k], apply[k]);   x_out <- x
 *      (engines.py:333-336 / worker.py:204, the canonical chain)
 *   2) ROLL:  for lane j in [lane_lo, lane_hi), j >= 1:
 *             xj = x; for k < j: xj = step(xj, cache[j], roll[k]); lane_out[j] <- xj
 *      (engines.py:321-327, lane j rolled with its own cached eps)
 * n_apply may be 0 (roll only, x = x_in) and lane_hi <= 1 disables the roll.
 * x_out may alias x_in. Host arrays are copied into the kernel parameters. */
int ps_sched_cycle(const void* x_in, void* x_out, int64_t n, int dtype,
                   const uint64_t* d_seed,
                   int n_apply, const ps_step* host_apply, const void* const* host_eps_apply,
                   void* const* host_rec_x,
                   int lane_lo, int lane_hi, const ps_step* host_roll,
                   const void* const* host_lane_cache, void* const* host_lane_out,
                   void* cuda_stream);

/* single ddpm_step with caller-supplied noise (z may be NULL when !noisy);
 * used for bit-exact checks against schedule.ddpm_step. */
int ps_sched_step_z(const void* x, const void* eps, const void* z, void* out, int64_t n,
                    int dtype, const ps_step* host_step, void* cuda_stream);

/* ---- reference MLP predictor (predictor.py:133-166), fp64 ----------------
 * a0 = [x, temb[t]]; z = a W + b; silu/tanh on hidden layers; linear out.
 * W_l is (fan_in, fan_out) row-major exactly as PredictorWeights stores it.
 * temb_table: (T+1) x embed_dim rows, row t = time_embed(t, T, E).
 * B rows (lanes) per call, host_ts[b] is lane b's step. */
typedef struct ps_mlp {
  int32_t n_layers;
  int32_t activation;  /* 0 = tanh, 1 = silu (predictor.py:33-36) */
  int32_t data_dim;
  int32_t embed_dim;
  int32_t dims[17];            /* dims[0] = data_dim + embed_dim ... dims[n_layers] */
  const double* W[16];
  const double* b[16];
  const double* temb_table;
} ps_mlp;

size_t ps_mlp_workspace_bytes(const ps_mlp* m, int B);
int ps_mlp_forward(const ps_mlp* m, const double* x, const int32_t* host_ts, int B, double* out,
                   void* workspace, void* cuda_stream);

/* ---- DiT-shaped predictor (paper_2505_14741_b200/spec.py) ----------------
 * Opaque handle owning its workspace; weights are device tensors owned by
 * the caller (created by the Python side with ps_rng_xavier). */
typedef struct ps_dit_config {
  int32_t channels, frames, height, width, layout; /* layout 0 = CHW, 1 = FHWC */
  int32_t patch, hidden, depth, heads, mlp_hidden, freq_dim;
  int32_t max_batch;
  int32_t precision;  /* 0 = fp32 (fp32-accurate GEMMs), 1 = bf16 tensor-core */
  int32_t gemm_impl;  /* 0 = auto (tcgen05), 2 = tcgen05; 1 = SIMT fp32 test reference only */
  int32_t text_tokens; /* text rows ahead of the video tokens (expert adaLN), 0 = none */
  int32_t rope;        /* 1 = 3D RoPE on the video rows' q/k (needs tcgen05), no pos table */
} ps_dit_config;

/* weight pointer order (fp32, (fan_in, fan_out) row-major, see
 * spec.layer_table): W[i], b[i] for i < n_layers; plus pos table (L x D) and
 * frequency table ((T+1) x freq_dim) */
typedef struct ps_dit_weights {
  int32_t n_layers;
  const float* const* W;
  const float* const* b;
  const float* pos;
  const float* freq_table;
  int32_t freq_rows;
  const float* text; /* [text_tokens, hidden] fixed text states (spec.py), or NULL */
  const float* rope; /* [video tokens, head_dim / 2, 2] (cos, sin), or NULL */
} ps_dit_weights;

typedef struct ps_dit ps_dit;
int ps_dit_create(const ps_dit_config* cfg, const ps_dit_weights* w, ps_dit** out);
int ps_dit_forward(ps_dit* h, const float* x, const int32_t* host_ts, int B, float* eps_out,
                   void* cuda_stream);
int ps_dit_destroy(ps_dit* h);
/* Per-run conditioning table (rows t = 0..T of every adaLN vector, 16 steps
 * per GEMV launch): reserve allocates (call outside graph capture), condition
 * fills it on the stream (capturable; the samplers run it at the start of
 * every denoise), clear returns forwards to per-forward conditioning. Rows
 * are bit-identical to the per-forward path. */
int ps_dit_condition_reserve(ps_dit* h, int T);
int ps_dit_condition(ps_dit* h, int T, void* cuda_stream);
int ps_dit_condition_clear(ps_dit* h);
int ps_dit_condition_chunk(const ps_dit* h); /* steps per conditioning launch (x3 GEMVs) */
/* algorithmic FLOPs of one forward of one sample (GEMMs + attention) */
double ps_dit_flops(const ps_dit* h);

/* number of kernel launches one ps_dit_forward issues */
int ps_dit_kernels_per_forward(const ps_dit* h);
/* Roofline probe: launch block 0's GEMM `which` (0 qkv, 1 proj, 2 fc1,
 * 3 fc2) `iters` times back to back on the stream with M = B x tokens rows
 * (plain store epilogue into handle scratch). */
int ps_dit_bench_gemm(ps_dit* h, int which, int B, int iters, void* cuda_stream);

/* Diagnostic (allocates + synchronises; never on the hot path):
 * C[M,N] = A[M,K] W[K,N] + bias with fp32 buffers in the reference layout,
 * through the tcgen05 kernel (impl 2; precision 1 = bf16, 0 = 3xTF32) or the
 * SIMT fp32 kernel (impl 1). Test hooks: 3 = split-K segments in one CTA,
 * 4 = at most 2 cluster CTAs along K, 5 / 6 = bf16 2-SM kernel forced on /
 * off (5: one pair tile per CTA pair), 7 = the persistent 2-SM kernel. */
int ps_gemm_test(const float* A, const float* W, const float* bias, float* C, int M, int N, int K,
                 int precision, int impl, void* cuda_stream);

/* Diagnostic: mean device time (us) of `iters` back-to-back tensor-core
 * GEMM launches on zero operands; dbg bit0 = skip MMA, bit1 = skip TMA. */
float ps_gemm_probe(int M, int N, int K, int precision, int dbg, int iters);
/* Diagnostic: clock64 phase stamps of CTA (0,0,0) of the last probe launch
 * run with dbg bit 4 (entry, prologue, PDL wait, first TMA, first stage,
 * last stage, accumulator ready, epilogue done, exit; split-K: partials
 * written, first cluster sync, reduction done). */
int ps_gemm_stamps(long long* out12);
/* Tuning knob: minimum K-blocks per split-K segment for layers prepared
 * afterwards (default 4); returns the previous value. */
int ps_gemm_tune(int split_min_kb);
/* Calibration: force the planned N-tile width / split-K of layers prepared
 * afterwards (0 = the planner's choice). */
void ps_gemm_force(int bn, int splits);

/* ---- U-Net-shaped predictor (paper_2505_14741_b200/unet_spec.py) -------
 * A native executor for the op list unet_spec.plan() emits (bf16 tcgen05
 * GEMMs: convolutions as implicit im2col GEMMs with GroupNorm+SiLU, concat
 * and resampling fused into the operand gather; tcgen05 attention). */
typedef struct ps_unet_op {
  int32_t kind;        /* 0 conv (im2col GEMM), 1 linear (token GEMM), 2 attention */
  int32_t layer;       /* weight index, -1 none */
  int32_t pre;         /* A producer: 0 none (in1 is bf16 already), 1 convert, 2 GN, 3 GN+SiLU, 4 LN */
  int32_t in1, in2;    /* buffer ids (-2 = the forward's latent x, CHW); in2 -1 unless concat */
  int32_t c1, c2;      /* channels of in1 / in2 */
  int32_t h, w;        /* input spatial size */
  int32_t taps;        /* 9 (3x3, pad 1) or 1 */
  int32_t resample;    /* 0 none, 1 stride-2, 2 nearest-2x before the conv */
  int32_t cout;
  int32_t temb_layer;  /* ResBlock time projection layer, -1 none */
  int32_t temb_off;    /* its column offset in the concatenated time table */
  int32_t resid;       /* fp32 buffer added in the epilogue, -1 none */
  int32_t out;         /* output buffer id (-3 = eps, CHW scatter) */
  int32_t out_bf16;    /* output buffer is bf16 */
  int32_t act;         /* 1 = GELU-tanh epilogue */
  int32_t heads;       /* attention heads (head_dim 64) */
  float eps;           /* GN / LN epsilon */
  int32_t out2;        /* bf16 shadow of the fp32 output (a later op's A), -1 none */
} ps_unet_op;

typedef struct ps_unet_config {
  int32_t in_channels, height, width, groups, freq_dim, temb_dim, temb_cols, max_batch;
  int32_t n_ops, n_bufs;
  const ps_unet_op* ops;
  void* const* bufs;   /* device buffers sized for max_batch, owned by the caller */
} ps_unet_config;

typedef struct ps_unet ps_unet;
/* weights: W[i], b[i] in unet_spec.layer_table order; freq_table rows t =
 * time_embed(t, freq_dim); pos unused */
int ps_unet_create(const ps_unet_config* cfg, const ps_dit_weights* w, ps_unet** out);
int ps_unet_forward(ps_unet* h, const float* x, const int32_t* host_ts, int B, float* eps_out,
                    void* cuda_stream);
int ps_unet_destroy(ps_unet* h);
int ps_unet_kernels_per_forward(const ps_unet* h);

/* ---- peer-memory eps exchange (multi-GPU ParaStep, one process per GPU) ---
 * Replaces the per-round all-gather: ranks export their double-buffered
 * lane-eps buffers and ready flags through CUDA IPC (64-byte handles), a
 * publisher stores base+round+1 into every rank's ready[me] with
 * system-scope release (ps_peer_signal; `slots` = device array of the world
 * flag addresses), a consumer waits on its local ready[0..count) with
 * acquire (ps_peer_wait), and ps_sched_cycle then reads the peers' eps over
 * NVLink directly. ps_peer_epoch_advance moves `base` on by 2^20 per run. */
int ps_dev_alloc(size_t bytes, void** out_dev_ptr); /* zeroed cudaMalloc (IPC-exportable) */
int ps_dev_free(void* dev_ptr);
int ps_ipc_get_handle(void* dev_ptr, void* out_handle64);
int ps_ipc_open_handle(const void* handle64, void** out_dev_ptr);
int ps_ipc_close(void* dev_ptr);
int ps_peer_signal(uint64_t* const* slots, int world, const uint64_t* base, uint64_t round,
                   void* cuda_stream);
int ps_peer_wait(const uint64_t* ready, int count, const uint64_t* base, uint64_t round,
                 void* cuda_stream);
int ps_peer_epoch_advance(uint64_t* base, void* cuda_stream);
/* async device-to-device (or peer) copy on the stream */
int ps_copy(void* dst, const void* src, size_t bytes, void* cuda_stream);
/* Writes the GPU's %globaltimer (ns) to *slot when the stream reaches it:
 * phase stamps for the per-rank forward / exchange-wait / apply split that
 * replaces the reference's WorkerTimings (pkg/src/parastep/protocol/
 * worker.py:65-85, loop_latency_s :108-110). */
int ps_stamp(uint64_t* slot, void* cuda_stream);

/* ---- trajectory files and diagnostics on device --------
 * ps_traj_pack writes the reference's binary trajectory file
 * (trajectory_io.py:100-110, "PSTJ" v1, little-endian float64 payload) into
 * `out` (ps_traj_pack_bytes(T, n) bytes) from device tables: rec_x [T][n],
 * eps rows eps[src_row[k]], x0 [n]; ts / fresh / src_row are device arrays.
 * ps_traj_diff writes out[r] = {sum|a-b|, sum|a|, sum (a-b)^2} (fp64, fixed
 * order) of row rows_a[r] of a against row rows_b[r] of b (null = identity):
 * the sums behind rel_mae / mse / compare_trajectories (numerics.py:144-158,
 * engines.py:446-473). */
int64_t ps_traj_pack_bytes(int T, int64_t n);
int ps_traj_pack(const void* rec_x, const void* eps, const void* x0, const int32_t* src_row,
                 const int32_t* ts, const uint8_t* fresh, int T, int64_t n, int dtype, void* out,
                 void* cuda_stream);
int ps_traj_diff(const void* a, const void* b, const int32_t* rows_a, const int32_t* rows_b,
                 int rows, int64_t n, int dtype_a, int dtype_b, double* out, void* cuda_stream);

/* Diagnostic (allocates + synchronises): softmax(Q K^T / sqrt(dh)) V over
 * qkv fp32 [B*L, 3D] (row m = [q | k | v], heads of dh = D/H contiguous)
 * into out fp32 [B*L, D]. bf16 operands (rounded): impl 1 = mma.sync flash
 * attention, 2 = tcgen05/TMEM flash attention (auto query tiles), 3 / 4 = it
 * with 1 / 2 query tiles per CTA. fp32 operands: impl 5 = mma.sync 3xTF32,
 * 6 = tcgen05 3xTF32 (the fp32 predictor path, head_dim <= 64). */
int ps_attn_test(const float* qkv, float* out, int B, int L, int H, int D, int impl,
                 void* cuda_stream);
/* Diagnostic: mean device time (us) of `iters` back-to-back attention launches. */
float ps_attn_probe(int B, int L, int H, int D, int impl, int iters);
/* Tuning hook for the tcgen05 attention kernel: how many of every 4 exp2
 * pairs run on the FMA-pipe polynomial instead of MUFU (-1 = built-in
 * default per head width). Results stay deterministic for a fixed value. */
int ps_fmha_set_poly(int pairs);

#ifdef __cplusplus
}
#endif
#endif /* PARASTEP_B200_H */

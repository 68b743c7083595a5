/*
 * trd.h -- C ABI of libtrd: the B200 (sm_100a) hot path of AWRTRD / SAWRTRD
 * (auto-weighted robust tensor-ring decomposition with FGMC and RStS, arXiv 2305.09044).
 *
 * Citations "P:L" are PAPER.md line numbers (section / equation in brackets).
 *
 * The method (Alg. 1): for a partially observed N-way tensor X with mask P,
 * find TR cores Z_k in R^{r_k x I_k x r_{k+1}} (Def. 1) maximising the
 * correntropy objective (Eq. 4) by a half-quadratic, cyclic, scaled steepest
 * descent: per block k, weights (Eq. 7), gradient on a randomized subtensor
 * sketch (Eq. 14-15), FGMC Gram (Eq. 13), scaled gradient
 * (Eq. 16), exact line search (Eq. 18), update (Eq. 17).
 * Readings of silent/garbled passages (R1..R18) are listed in DESIGN.md section 3.
 *
 * Conventions (0-based):
 *   - linear index of X: lin = i_0 + I_0*(i_1 + I_1*(i_2 + ...))   (Def. 2 multi-index)
 *   - core k on the host: float[r_k][I_k][r_{k+1}], C order (paper index order)
 *   - mask: bit (lin % 32) of uint32 word (lin / 32); 1 = observed
 *   - Zk2 column a + r_k*b (classical mode-2 unfolding, Thm 1); d and h use it too.
 *
 * Errors: every call returns trd_status and never throws across the ABI.  Arguments are
 * validated before anything is enqueued.  A CUDA or exchange (NCCL) failure puts the context
 * into a sticky error state in which only trd_get_cores / trd_last_error / trd_destroy are valid.
 *
 * Threading: a context is used by one host thread at a time.  All device work is enqueued
 * on the stream given to trd_init (trd_upload's copies: on a library copy stream ordered
 * against it).  No call keeps pointers to caller host memory, except that trd_upload's
 * asynchronous copy reads its host buffers until the call that consumes the upload returns.
 */
#ifndef TRD_H
#define TRD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define TRD_API __attribute__((visibility("default")))
#else
#define TRD_API
#endif

#define TRD_MAX_ORDER 8
#define TRD_MAX_RANK 128

typedef struct trd_ctx trd_ctx;

typedef enum {
  TRD_OK = 0,
  TRD_ERR_INVALID_ARG = 1,  /* bad pointer / value (sigma <= 0, lambda_rel < 0, ...)   */
  TRD_ERR_SHAPE = 2,        /* N, dims, ranks, sketch sizes or shard range inconsistent */
  TRD_ERR_OOM = 3,          /* device allocation failed                                 */
  TRD_ERR_CUDA = 4,         /* CUDA runtime error (sticky)                              */
  TRD_ERR_NCCL = 5,         /* NCCL error or NCCL unavailable for world > 1 (sticky)    */
  TRD_ERR_NOT_SPD = 6,      /* G + lambda I not positive definite after 3 retries       */
  TRD_ERR_NONFINITE = 7,    /* non-finite value in d, h, eta or the cores               */
  TRD_ERR_STATE = 8         /* call not valid in the current state                      */
} trd_status;

typedef enum {
  TRD_SIGMA_FIXED = 0,  /* Alg. 1 input sigma, kept fixed                        */
  TRD_SIGMA_INF = 1,    /* sigma -> inf: W == 1, the masked LS problem Eq. 2     */
  TRD_SIGMA_RMS = 2,    /* reading R9: sigma_{t+1} = max(sigma_min, theta * RMS(e))      */
  TRD_SIGMA_MAD = 3     /* reading R21 (robust rule): sigma_{t+1} = max(sigma_min,
                           theta * 1.4826 * median |e|) over the sweep's pass-1 residuals, the
                           exact median (mean of the two middle values of an even count) by a
                           radix select over the fp32 |e| values                             */
} trd_sigma_mode;

typedef struct {
  int32_t order;                    /* N, 3..TRD_MAX_ORDER                                  */
  int64_t dims[TRD_MAX_ORDER];      /* global I_0..I_{N-1}                                  */
  int32_t ranks[TRD_MAX_ORDER];     /* r_0..r_{N-1}, 1..TRD_MAX_RANK, ring r_N = r_0;
                                       r_k r_{k+1} <= TRD_MAX_RANK^2, and every block must have a
                                       split with r_k r_s <= 256 (else TRD_ERR_SHAPE).  Blocks
                                       with R_k^2 = r_k r_{k+1} > 1024 (the paper's [80,80,3,20],
                                       P:328) take the large-rank path: FGMC products,
                                       Q refresh and the filtered solve as fp64 cuBLAS /
                                       cuSOLVER calls (dlopen'ed; TRD_ERR_CUDA if absent), one
                                       host synchronisation per such block (no CUDA graphs)   */
  int32_t sigma_mode;               /* trd_sigma_mode                                       */
  double sigma;                     /* FIXED: the kernel width; RMS: ignored (sigma_0 from
                                       an initial residual pass); INF: ignored              */
  double sigma_theta;               /* RMS multiplier theta (default 1.0)                   */
  double sigma_min;                 /* RMS floor (default 1e-3)                             */
  double lambda_rel;                /* R5: lambda = lambda_rel * tr(G) / R_k^2 (default 1e-6) */
  double step;                      /* 0: exact line search Eq. 12/18; > 0: fixed eta        */
  int64_t sketch[TRD_MAX_ORDER];    /* s_m used when m != k; 0 or >= I_m means the full mode
                                       (AWRTRD); s_k = I_k always (Alg. 1 line 4)     */
  uint64_t seed;                    /* RStS sampler seed (reading R11)                      */
  int32_t shard_mode;               /* X is sharded along this mode (0 when world == 1)     */
  int32_t world, rank;              /* data-parallel group; world == 1: no NCCL             */
  const void* nccl_unique_id;       /* 128 bytes from trd_nccl_unique_id() on rank 0,
                                       broadcast by the caller; NULL when world == 1         */
  int32_t scaling;                  /* operator of the update direction (ablation arms of
                                       Sec. 6.1): TRD_SCALING_GLOBAL h = d M with the
                                       FGMC Gram (Eq. 16, default); TRD_SCALING_NONE h = d
                                       ('gradient descent'); TRD_SCALING_LOCAL the Gram of the
                                       sampled cores (Z_k)_{I_k} ('local scaled term').  The
                                       stop metric (Alg. 1 l.12) always uses the FGMC Gram.  */
  int32_t sampling;                 /* working set of a block: TRD_SAMPLING_RSTS the RStS
                                       subtensor (Eq. 14, default); TRD_SAMPLING_ROWS the
                                       'uniform row sampling' ablation arm (reading R22):
                                       J = prod_{m!=k} s_m rows of X_[k] drawn uniformly with
                                       replacement (not with TRD_SCALING_LOCAL)               */
} trd_config;

typedef enum {
  TRD_SAMPLING_RSTS = 0,
  TRD_SAMPLING_ROWS = 1
} trd_sampling;

typedef enum {
  TRD_SCALING_GLOBAL = 0,
  TRD_SCALING_NONE = 1,
  TRD_SCALING_LOCAL = 2
} trd_scaling;

/* Local shard of X and P (world == 1 with a partial shard: that shard's partial problem, no
 * exchange).  Local tensor = global X restricted to
 * i_{shard_mode} in [shard_begin, shard_end), stored in its own linear order (same formula
 * with the local extent of the shard mode).  Device pointers, caller owned, read only,
 * must stay valid and unmodified until trd_destroy (or until trd_upload replaces them when
 * the shard is library-owned). */
typedef struct {
  int64_t shard_begin, shard_end;   /* [0, I_shard) when world == 1                          */
  const float* values;              /* dense: value of local entry lin at values[lin];
                                       packed: value of the n-th observed entry (in local
                                       linear order) at values[n]                            */
  const uint32_t* mask_bits;        /* 1 bit per local entry                                */
  int32_t packed;                   /* 0 dense, 1 packed (values of observed entries only)   */
  int32_t host;                     /* 0: pointers are device memory (zero copy).
                                       1: pointers are host memory; the library allocates
                                       device buffers and copies them (trd_upload re-copies) */
} trd_shard;

/* Data-parallel exchange (world > 1), the one collective of the path: an in-place allreduce
 * of n doubles in device memory across the ranks (op TRD_OP_SUM or TRD_OP_MAX), ordered on
 * `stream`: it must include all work enqueued on the stream before the call, and work enqueued
 * after it must see the result (a host-synchronous implementation -- synchronise the stream,
 * exchange, copy back -- qualifies).  Returns 0 on success.  With trd_init the library uses
 * NCCL (ncclAllReduce on the context stream, bootstrapped from cfg.nccl_unique_id); with
 * trd_init_ex a caller-supplied exchange replaces it (for example torch.distributed, or a
 * test harness driving several contexts).  The call sites, per block (Alg. 1): the
 * gradient partials and residual statistics [d | sum e^2 | welsch | n] after pass 1, the
 * line-search denominator after pass 2; per sweep: the R21 select histograms (MAD) and the
 * replica-consistency check; at init: sigma_0's statistics; trd_error's sums. */
typedef enum { TRD_OP_SUM = 0, TRD_OP_MAX = 1 } trd_reduce_op;
typedef int (*trd_allreduce_fn)(void* user, double* buf_dev, uint64_t n, int32_t op, void* stream);
typedef struct {
  trd_allreduce_fn allreduce;
  void* user;
} trd_exchange;

/* One record per sweep.  ms is the device time of the sweep (CUDA events). */
typedef struct {
  double sigma;                     /* kernel width used in this sweep                      */
  double sum_e2;                    /* sum of squared pass-1 residuals over all blocks       */
  double welsch_loss;               /* sum over blocks of sum_WS sigma^2 (1 - w)  (R3)       */
  double stop_e;                    /* Alg. 1 line 13 relative change of D^t; NaN at t = 0    */
  double ms;                        /* device milliseconds of this sweep                     */
  int64_t n_obs;                    /* observed entries processed (sum over blocks)          */
  double eta[TRD_MAX_ORDER];        /* step size per block (0 if skipped)                    */
  double num[TRD_MAX_ORDER];        /* <d, h> per block                                      */
  double den[TRD_MAX_ORDER];        /* ||sqrt(W) o P o (h S^T)||^2 per block                  */
  int64_t nnz[TRD_MAX_ORDER];       /* observed entries in block k's working set             */
  uint32_t skipped_mask;            /* bit k set: block k skipped (num <= 0 or den == 0, R14) */
  uint32_t replica_mismatch;        /* world > 1: 1 if the ranks' cores differed after the
                                       sweep (a 64-bit checksum compared across ranks; the
                                       replicated update must be bitwise identical) */
} trd_sweep_stats;

typedef struct {
  double rel_err_all;               /* ||X_hat - X_ref|| / ||X_ref|| over evaluated entries  */
  double rel_err_observed;          /* same, restricted to observed entries                  */
  double psnr;                      /* 10 log10(peak^2 / MSE) over the evaluated entries */
  int64_t n_eval;                   /* entries evaluated                                      */
} trd_error_stats;

/* Create a context.  init_cores: host pointers, N arrays float[r_k][I_k][r_{k+1}] (Alg. 1
 * line 1).  stream: a cudaStream_t (NULL = legacy default stream).  Builds the FGMC
 * cache Q_k and, for TRD_SIGMA_RMS / MAD, sigma_0 from all local observed residuals
 * (allreduced).  Synchronises the stream once.  *out is NULL on failure. */
TRD_API trd_status trd_init(const trd_config* cfg, const trd_shard* shard,
                    const float* const* init_cores, void* stream, trd_ctx** out);

/* trd_init with a caller-supplied exchange (world > 1; cfg.nccl_unique_id is then ignored and
 * NCCL is not loaded).  `ex` is copied; ex->user must stay valid until trd_destroy. */
TRD_API trd_status trd_init_ex(const trd_config* cfg, const trd_shard* shard,
                       const float* const* init_cores, void* stream, const trd_exchange* ex,
                       trd_ctx** out);

/* Copy host-resident X / P (shard.host == 1 only) for a later sweep: the host->device leg of
 * an end-to-end step.  The copy runs on the library's copy stream into one of two device
 * buffer sets, so it overlaps the sweeps already enqueued; the next trd_sweep consumes the
 * oldest pending upload (waits for its copy, restages, recomputes the packed rank prefix).
 * At most two uploads may be pending (TRD_ERR_STATE otherwise).  Same layout and sizes as at
 * trd_init (packed: same number of observed entries).  The host buffers (pinned for overlap)
 * must stay unmodified until the call that consumes the upload (trd_sweep, trd_block_probe or
 * trd_error) returns; that call waits for the copy before returning. */
TRD_API trd_status trd_upload(trd_ctx* ctx, const float* values_host, const uint32_t* mask_host);

/* Write the RStS index sets of sweep `sweep`, block k (Alg. 1 line 4; reading R11)
 * to idx_dev (device, int32, sum_m sizes[m] entries, mode-major, each set ascending) and
 * their sizes to sizes_host[N] (host).  Mode k gets 0..I_k-1.  With TRD_SAMPLING_ROWS every
 * other mode gets the J draws in draw order (entry q of each list = draw q; idx_dev must
 * hold I_k + (N-1) J entries).  With a partial shard (world > 1) the shard mode's list is
 * this rank's part: its slice for a full set, its sampled indices (ascending, then padding
 * entries equal to shard_begin that carry no data) for an RStS set, whose sizes[m] is the
 * capacity min(s_m, slice).  Synchronises the stream. */
TRD_API trd_status trd_sketch(trd_ctx* ctx, int32_t sweep, int32_t k, int32_t* idx_dev,
                      int64_t* sizes_host);

/* Run n_sweeps iterations of Alg. 1 (lines 3-13).  stats: host array of n_sweeps records
 * or NULL.  With stats == NULL the call only enqueues work (no host synchronisation, except
 * that a pending upload's copy is waited for).  Returns TRD_ERR_NONFINITE if a non-finite
 * value appeared, TRD_ERR_NOT_SPD if G + lambda I stayed indefinite through the retries of
 * reading R23 (both checked when stats != NULL; NONFINITE also at trd_get_cores). */
TRD_API trd_status trd_sweep(trd_ctx* ctx, int32_t n_sweeps, trd_sweep_stats* stats);

/* Evaluate the TR model (Def. 1) at n global linear indices (device int64) into
 * out_dev (device float).  Enqueued on the context stream; no synchronisation. */
TRD_API trd_status trd_reconstruct(trd_ctx* ctx, const int64_t* lin_idx_dev, int64_t n, float* out_dev);

/* Relative error and PSNR of the model against ref_dev (device float, dense local
 * shard layout), over all local entries, or over those whose bit is set in eval_bits (device,
 * may be NULL).  peak: the PSNR peak value (0 = 1.0: the paper rescales data to [0, 1],
 * P:326; < 0 is TRD_ERR_INVALID_ARG).  Partial sums are allreduced when world > 1.
 * Synchronises the stream. */
TRD_API trd_status trd_error(trd_ctx* ctx, const float* ref_dev, const uint32_t* eval_bits, double peak,
                     trd_error_stats* out);

/* Copy cores to / from the host (layout as init_cores).  Synchronises the stream.
 * trd_get_cores copies the cores even in the sticky error state; it returns
 * TRD_ERR_NONFINITE if a copied value is not finite or a sweep flagged a non-finite step.
 * trd_set_cores rebuilds the FGMC cache. */
TRD_API trd_status trd_get_cores(trd_ctx* ctx, float* const* cores_host);
TRD_API trd_status trd_set_cores(trd_ctx* ctx, const float* const* cores_host);

/* Iteration state of Alg. 1 beyond the cores, for an exact resume (checkpoint /
 * resume): the kernel width sigma the next sweep uses (the sigma rules of R9 / R21 update
 * it at sweep end), the sweep counter t that selects the next sweep's RStS draw (Alg. 1 l.3-4,
 * P:267-268; reading R11), and D^{t-1} of the stop metric (Alg. 1 l.12-13; reading
 * R15), an I_{N-1} x I_{N-1} float64 matrix (row-major) that exists once a sweep has run.  A
 * context created from saved cores (trd_init / trd_set_cores) and given the saved state with
 * trd_set_state continues bit for bit as the saving context would have. */
typedef struct {
  double sigma;                     /* kernel width of the next sweep                         */
  int32_t sweep;                    /* sweep counter t of the next sweep                      */
  int32_t have_prev_D;              /* 1: prev_D holds D^{t-1}; 0: the next stop_e is NaN      */
  int64_t prev_D_size;              /* I_{N-1}^2 (set by trd_get_state; checked by trd_set_state) */
} trd_state;
/* prev_D_host: host double[I_{N-1}^2] or NULL (get: not copied; set: only valid with
 * have_prev_D == 0).  sigma must be > 0 (any value when sigma_mode == TRD_SIGMA_INF), sweep
 * >= 0.  Both synchronise the stream. */
TRD_API trd_status trd_get_state(trd_ctx* ctx, trd_state* out, double* prev_D_host);
TRD_API trd_status trd_set_state(trd_ctx* ctx, const trd_state* st, const double* prev_D_host);

/* Diagnostic probe of block k at the current cores without updating them (parity tests):
 * runs a1-a10 of the block exactly as trd_sweep would at sweep index `sweep` and copies
 * d (I_k x R_k^2, row-major, column a + r_k b), G (R_k^2 x R_k^2), h (like d) and
 * stats5 = {sum_e2, n_obs, welsch, num, den} to the host.  Any output pointer may be NULL. */
TRD_API trd_status trd_block_probe(trd_ctx* ctx, int32_t sweep, int32_t k, double* d_host,
                           double* G_host, double* h_host, double* stats5_host);

/* Number of kernels the library launched since the context was created (a counter the
 * host increments at every launch; bench.py reports it as gpu_launches). */
TRD_API int64_t trd_launch_count(const trd_ctx* ctx);

/* Per-kernel-class device time, measured with CUDA events recorded on the context stream
 * around the pass-1 and pass-2 kernels while profiling is enabled (bench.py's roofline).
 * trd_get_profile synchronises the stream; it reports totals since the last enable. */
typedef struct {
  double pass1_ms, pass2_ms;        /* summed device time of the pass kernels               */
  int64_t pass1_launches, pass2_launches;
  double pass1_entries, pass2_entries;    /* observed entries processed (sum over launches) */
  double pass1_flops, pass2_flops;        /* algorithmic flops, SURVEY 8(d) per-entry count
                                             (4K + 8 / 2K + 4, K = r_k r_s <= R^2 the per-entry
                                             contraction length of the block's split)         */
  double pass1_bytes, pass2_bytes;        /* algorithmic bytes, SURVEY 8(d) per-entry count  */
  double pass1_mma_flops, pass2_mma_flops;/* dense tensor-core flops the tcgen05 pass kernels
                                             executed (3-term fp16 split, 128 x 64 tiles)     */
} trd_profile;
TRD_API trd_status trd_set_profiling(trd_ctx* ctx, int32_t enable);
TRD_API trd_status trd_get_profile(trd_ctx* ctx, trd_profile* out);

/* 128-byte NCCL unique id for world > 1 (call on rank 0; caller broadcasts it). */
TRD_API trd_status trd_nccl_unique_id(void* out128);

TRD_API void trd_destroy(trd_ctx* ctx);
TRD_API const char* trd_last_error(const trd_ctx* ctx);
TRD_API const char* trd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TRD_H */

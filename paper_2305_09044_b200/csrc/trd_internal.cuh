// trd_internal.cuh -- context layout, block plans and kernel entry points of libtrd.
// Paper citations "P:L" are PAPER.md lines.  See DESIGN.md for the data layout in HBM.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/trd.h"

namespace trd {

constexpr int kMaxN = TRD_MAX_ORDER;
// default mode of the pipelined staging of sampled blocks (Context::pipe; TRD_PIPE overrides) and
// the smallest staged tile count of a pipelined block.  Measured with 50 timed sweeps after 20
// warm-up sweeps (ms per sweep, in line / mode 3): C3 0.643 / 0.581, C4 0.777 / 0.745, C5a 2.055 /
// 1.931 -- every sampled block is pipelined (10-sweep runs, biased by the clock ramp of the
// sub-ms configs, had suggested otherwise for C4)
constexpr int kPipeDefault = 3;
constexpr int64_t kPipeMinTiles = 0;
constexpr int kMaxR = TRD_MAX_RANK;
constexpr int kMaxR2 = kMaxR * kMaxR;
// blocks with R_k^2 above this take the large-rank path (trd_big.cu): the d contraction by
// reduce_d_big_kernel, and FGMC / Q refresh / filtered solve as fp64 cuBLAS / cuSOLVER calls
constexpr int kBigR2 = 1024;

// Per-sweep statistics kept on the device (one record per sweep of a trd_sweep call).
struct DevStats {
  double sigma, sum_e2, welsch, stop_e;
  long long n_obs;
  double eta[kMaxN], num[kMaxN], den[kMaxN];
  long long nnz[kMaxN];
  unsigned int skipped;
  int nonfinite;
  unsigned int replica_mismatch;   // world > 1: the ranks' core checksums differed
};

// Scalars shared by the kernels of one block (device memory).
// Exact median of the sweep's |e| (robust sigma rule, reading R21, TRD_SIGMA_MAD): pass 1
// writes the fp32 bit pattern of every observed |e| (tile-staged slots of padding entries get
// kEabsPad, which the select skips); an exact radix select over the bit patterns (11 + 11 + 10
// bits, per-CTA shared-memory histograms, integer counts) finds the two middle order
// statistics.  Histogram regions of c->mhist: level 0 [2048] | level 1 [2][2048] | level 2 [2][1024].
constexpr uint32_t kEabsPad = 0xFFFFFFFFu;

// ---- checked build (-DTRD_CHECKED=1 -> libtrd_checked.so) -------------
// compute-sanitizer is not available on the GPU pool, so the checked library carries its own:
// device-side invariant checks (bounds of every staged-slot, entry and shared-memory index the
// data decides), an mbarrier watchdog (a wait that has not completed after ~2^34 cycles records
// a hang and gives up, so a broken pipeline ends instead of hanging the GPU) and schedule
// fuzzing (TRD_JITTER_NS: a pseudo-random __nanosleep after every pipeline wait, which must not
// change any result bit).  A failed check is recorded (first code, block, thread, count) and
// trd_sweep / trd_block_probe report it as TRD_ERR_STATE; the faulty access is skipped.  In the
// product library TRD_CHECKED is 0 and all of it compiles away.
#ifndef TRD_CHECKED
#define TRD_CHECKED 0
#endif
enum : unsigned int {
  kChkHang = 1,        // mbarrier wait watchdog expired
  kChkEntry = 2,       // staged entry id outside the 128 x 64 tile
  kChkStageCap = 3,    // a tile's staged slots beyond the stage capacity
  kChkSmemVals = 4,    // smem-staged tile with more entries than the stage holds
  kChkSampler = 5,     // RStS index outside [0, I_m) or a set not strictly ascending
  kChkStageWrite = 6,  // staging kernel slot index beyond the capacity
  kChkTileBase = 7     // tile value blocks not monotone
};
struct DevCheck {
  unsigned int code, block, thread, count;
  unsigned int jitter_ns;
};
// (one instance per translation unit: trd_kernels.cu and trd_tc.cu collect their own)
static __device__ DevCheck g_check;
#if TRD_CHECKED
static __device__ __noinline__ void trd_check_fail(unsigned int code) {
  if (atomicCAS(&g_check.code, 0u, code) == 0u) {
    g_check.block = blockIdx.x;
    g_check.thread = threadIdx.x;
  }
  atomicAdd(&g_check.count, 1u);
}
#endif
#define TRD_CHECK(cond, code) \
  do { if (TRD_CHECKED && !(cond)) { TRD_CHECK_FAIL(code); } } while (0)
#if TRD_CHECKED
#define TRD_CHECK_FAIL(code) trd_check_fail(code)
#else
#define TRD_CHECK_FAIL(code) do { } while (0)
#endif
// schedule fuzzing after a pipeline wait (checked build with TRD_JITTER_NS > 0)
__device__ __forceinline__ void trd_jitter() {
#if TRD_CHECKED
  const unsigned int j = *(volatile unsigned int*)&g_check.jitter_ns;
  if (j) {
    unsigned int x = (unsigned int)clock() * 0x9E3779B1u ^ (threadIdx.x * 0x85EBCA77u) ^ (blockIdx.x * 0xC2B2AE3Du);
    x ^= x >> 15;
    __nanosleep(x % j);
  }
#endif
}

// Power-of-two scale exponent E of an fp16 hi / lo operand with max |.| = amax: amax 2^E lies
// in [2^14, 2^15), so every element is below the fp16 maximum (65504) and elements down to
// 2^-15 of the maximum keep a normal lo part (22 significant bits).  Scaling by 2^E is exact.
// max into a shared fp32-bits scalar: the atomic only when the value can raise it (same-address
// atomics serialise at L2: thousands of CTAs / rows would cost ~100 us per kernel)
__device__ __forceinline__ void amax_update(unsigned int* dst, float v) {
  if (v > 0.f && __float_as_uint(v) > *reinterpret_cast<volatile unsigned int*>(dst)) atomicMax(dst, __float_as_uint(v));
}

__host__ __device__ __forceinline__ int tc_scale_exp(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 0;
  int e = 0;
  frexpf(amax, &e);                  // amax = f 2^e, f in [0.5, 1): floor(log2 amax) = e - 1
  const int E = 15 - e;
  return E < -100 ? -100 : (E > 100 ? 100 : E);
}
// Programmatic dependent launch (PDL) of the per-block chain of small kernels: a kernel launched
// with launch_pdl may be scheduled while its stream predecessor finishes (its launch latency hides
// under the predecessor's tail); trd_gdc_wait(), the first statement of every such kernel, returns
// once the predecessor grid has completed and its memory is visible (a no-op without PDL).
__device__ __forceinline__ void trd_gdc_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
extern bool g_pdl_on;                // TRD_PDL=1 (off by default: measured neutral to slower)
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl_on ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#define TRD_PDL(kern, grid, block, smem, stream, ...) ::trd::launch_pdl(kern, dim3(grid), dim3(block), (size_t)(smem), stream, __VA_ARGS__)

constexpr int kMadBins0 = 2048, kMadBins1 = 2048, kMadBins2 = 1024;
constexpr int kMadHist = kMadBins0 + 2 * kMadBins1 + 2 * kMadBins2;

struct DevScalars {
  double sigma;          // kernel width of the current sweep
  double num, den;       // <d,h> and the line-search denominator of the current block
  double sum_e2, welsch; // pass-1 statistics of the current block (after allreduce)
  double n_obs;          // observed entries of the block (double so it rides the allreduce)
  double eta;            // step of the current block
  double lambda;         // lambda used by the solve
  double h_lam;          // h = u - h_lam u Mop, u = d Mop (lambda when Mop = (G + lambda I)^-1)
  int sweep;             // sweep counter t (read by the sampler: graph-replayable)
  int slot, slot_next;   // record slot of the current sweep in the DevStats array of the call
  int not_spd;           // Cholesky failed after retries
  int nonfinite;         // non-finite value detected
  int replica_bad;       // world > 1: a sweep ended with differing replicas
  int mask_same;         // the last uploaded mask equalled stage_mask
  int mask_gen;          // generation of the current mask (bumped when an upload changes it)
  int layout_gen[kMaxN]; // generation of the mask each block's staged layout was built from
  double acc_e2, acc_n;  // sweep accumulators for the RMS sigma rule (R9)
  double stop_e;         // relative change of D^t
  int have_prev_D;
  int prof_on;           // accumulate local observed entries per block (profiling)
  double prof_nobs[kMaxN];
  // power-of-two operand scaling of the fp16 hi / lo tensor-core operands:
  // max |.| as fp32 bit patterns (non-negative floats order like unsigned ints: atomicMax)
  unsigned int amax_x;            // observed values (init / each upload)
  unsigned int amax_a;            // pass-1 A operand (Lft) of the current block
  unsigned int amax_b;            // B operand (Rgt) of the current block
  unsigned long long eabs_fill;   // R21: |e| slots written in this sweep (or the sigma_0 pass)
  unsigned int mad_pre[2];        // R21 select: bit prefixes of the two middle order statistics
  long long mad_rank[2];          //   and their ranks among the values with that prefix
  double mad_n;                   //   number of |e| values
  double mad_med;                 //   their median
};

// GEMM form of block k: the working set WS_k = I_k x prod_{m!=k} s_m is
// a (rows x cols) matrix with rows = (j_L, i_k) [j_L over the left modes k+1..k+p, fastest
// first] and cols = j_R over the right modes k+p+1..k-1.  The subchain splits as
// S(j) = Mid(j_L) Rgt(j_R) and x_hat = Tr(Lft Rgt) with Lft = Z_k(i_k) Mid(j_L) (Thm 1,
// P:61-66; Def. 2), so each entry costs one K = r_k * r_{k+p+1} inner product.
struct BlockPlan {
  int k, p;
  int nleft, nright;
  int left[kMaxN], right[kMaxN];
  int rk, rk1, rs;       // r_k, r_{k+1}, r_{k+p+1}
  int K, R2;             // rk*rs, rk*rk1
  int64_t s[kMaxN];      // sizes of the index sets of this block (s_k = I_k)
  int64_t nL, nrows, ncols;
  int64_t nnz_ws;        // |WS_k| (all entries, observed or not)
  // digit orders: rows = (i_k, j_L) with rowmode 0: row = jl + nL*ik, 1: row = ik + I_k*jl;
  // j_L / j_R mixed radix with ldig / rdig (indices into left / right, fastest first), chosen
  // so that mode 0 (contiguous in memory) is the fastest digit of rows or columns
  int rowmode;
  int ldig[kMaxN], rdig[kMaxN];
  int shard_local;       // the shard mode (full index set) enumerates only this rank's slice
                         // [shard_begin, shard_end): per-rank GEMM work shrinks with world
  int64_t ik0;           // k == shard mode: global i_k of plan row index 0 (else 0)
  int shard_sampled;     // sampled shard-mode set (m != k): only the rank's sampled indices,
                         // compacted into a list of capacity min(s_m, slice) (rest padding)
  int64_t s_samp[kMaxN]; // sample size of the RStS draw per mode (s[m] may be the capacity)
  int explicit_cols;     // 'uniform row sampling' (R22): p = 0, column q = draw q, whose index in
                         // right mode m is idx[idx_off[m] + q] (all s[m] = ncols = J)
  // pass-kernel geometry (v1 SIMT)
  int jl_per_cta, ws_split, nsplit;
  int64_t grid_x;        // ceil(nL / jl_per_cta)
  // tensor-core pass kernels (trd_tc.cu)
  int use_tc;            // 1: tcgen05 pass kernels
  int KP;                // K padded to a multiple of 16
  int64_t n_row_tiles, n_col_tiles;
  int tc_nsplit;         // column splits per row tile (work item = (row tile, split))
  int64_t tc_per;        // column tiles per split
  int tc_grid;           // persistent CTAs of pass 2 (<= SM count)
  int tc_grid1;          // persistent CTAs of pass 1 (SMs left for the side-stream solve)
  int tc_cl;             // CTAs per cluster of the pass kernels (2: B tiles multicast to a pair)
  int tc_u;              // column tiles per ring unit of the pass kernels (2: N = 128 GEMMs)
  int64_t tc_jc, tc_jl_chunk;   // d reduction: jl chunks
  int big;               // R2 > kBigR2: large-rank path (SIMT pass 1 writes D rows to contrib)
  int lib_solve;         // filtered solve by cuSOLVER (big blocks, and R2 > 128 blocks of a
                         // context that loads it): big_factor / big_h instead of solve_kernel
  int rows;              // SIMT plan with K > 128: warp-per-row passes (simt_rows_kernel)
  int rows_nsplit, rows_grid;   //   column splits per row, CTAs (8 warps each)
  int64_t rows_per;             //   columns per split (multiple of 32)
};

// Staged working set of one block in tile order (trd_tc.cu "stage sketch", row a2)
struct TcStage {
  uint64_t* tbits = nullptr;     // [tile][128] observation mask of (row, 64 columns)
  uint16_t* troff = nullptr;     // [tile][128] row offset into the tile's compacted values
  uint64_t* tcount = nullptr;    // [tile + 1] padded tile counts (last = 0)
  uint64_t* tbase = nullptr;     // [tile + 1] exclusive prefix of the tile counts
  float* tvals = nullptr;        // compacted observed values, tile-major, row-major in a tile,
                                 // tile blocks padded to 8 entries
  uint16_t* tidx = nullptr;      // entry list: row * 64 + column per value, 0xFFFF = padding
  void* scan_tmp = nullptr;
  size_t scan_tmp_bytes = 0;
  int64_t n_tiles = 0, vcap = 0;
  int32_t* perm = nullptr;       // invariant sketches: value index of every staged slot
  bool invariant = false;        // working set identical every sweep (full index sets)
  bool valid = false;            // staged data current
};

// One sweep captured as a CUDA graph (trd_sweep replays it; one per upload buffer set)
struct SweepGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  long long launches = 0;              // kernels per replay (launch counter)
  const void* stats_ptr = nullptr;     // the stats array the graph writes
  std::vector<cudaEvent_t> cap_ev;     // profiling events recorded during the capture
  std::vector<cudaGraphNode_t> ev_nodes;   // their event-record nodes (same order)
  std::vector<std::pair<int, int>> pairs1, pairs2;   // pass-1 / pass-2 (begin, end) in cap_ev
};

struct Context {
  trd_config cfg;
  int N;
  int64_t dims[kMaxN], ldims[kMaxN];   // global / local dims
  int64_t lstride[kMaxN];              // local linear strides
  int ranks[kMaxN];
  int64_t shard_begin, shard_end;
  int64_t n_local, n_words;
  int packed;
  cudaStream_t stream;
  cudaStream_t side = nullptr;         // FGMC Gram + filtered solve of a block (a8, a9) run here,
                                       // concurrently with pass 1 (they need only cores != k)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int num_sm = 148;                    // SMs of the current device (persistent grids)
  int rbucket = 16;                    // 16, 32 or 128: >= every rank (register arrays of the plan kernels)
  size_t chain_half = 0;               // doubles per FGMC chain buffer (chain_ws holds two)
  std::string err;
  trd_status sticky = TRD_OK;
  long long launches = 0;

  // data (device)
  const float* values = nullptr;
  const uint32_t* mask = nullptr;
  float* own_values = nullptr;         // host-resident shards: library-owned copies
  uint32_t* own_mask = nullptr;
  // double-buffered uploads (host-resident shards): buffer set b = (up_values[b], up_mask[b]);
  // set 0 aliases own_values / own_mask.  `active` feeds the sweeps; pending uploads form a FIFO
  float* up_values[2] = {nullptr, nullptr};
  uint32_t* up_mask[2] = {nullptr, nullptr};
  int up_active = 0, up_npend = 0, up_pend[2] = {0, 0};
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_up_ready[2] = {nullptr, nullptr}, ev_up_free = nullptr;
  int64_t n_values = 0;
  uint32_t* rank_prefix = nullptr;     // packed layout: exclusive popcount prefix per word
  uint32_t* stage_mask = nullptr;      // the mask the invariant staged layouts were built from
  uint8_t* ptab = nullptr;             // compaction tables of the sampled mode-0 positions (staging)
  void* rp_tmp = nullptr;              // its scan's scratch (allocated once)
  size_t rp_tmp_bytes = 0;

  // model (device)
  float* Z = nullptr;                  // cores, slice-major: Z_k[i][a][b]
  int64_t zoff[kMaxN + 1];
  double* Q = nullptr;                 // FGMC Q_k (r_k^2 x r_{k+1}^2)
  uint32_t* eabs = nullptr;            // TRD_SIGMA_MAD: fp32 bits of the sweep's |e| (R21)
  size_t eabs_cap = 0;
  double* mhist = nullptr;             // TRD_SIGMA_MAD: radix-select histograms (kMadHist)
  double* Qloc = nullptr;              // 'local scaled term' arm: Q_m over the sampled slices
  double* Gloc = nullptr;              //   and its Gram
  int64_t qoff[kMaxN + 1];

  // plans and per-block workspaces (device)
  BlockPlan plan[kMaxN];
  BlockPlan full_plan;                 // full index sets (sigma_0 pass, trd_error)
  int32_t* idx = nullptr;              // index sets of the current block, per mode
  int64_t* doff = nullptr;             // data offset of each index (or -1 outside shard)
  int64_t idx_off[kMaxN + 1];
  int64_t* row_off = nullptr;          // per GEMM row
  int64_t* col_off = nullptr;          // per GEMM col
  // Pipelined staging of sampled blocks (RStS): block k+1's sampler, offsets
  // and tile staging depend only on (seed, k+1, t) and the data, not on the cores, so they run
  // on `stg` while block k finishes.  Each block then owns its index / offset buffers; the
  // pointers above are the current block's (select_bufs), `*_d` the defaults (sigma_0, trd_error,
  // trd_sketch, contexts without the pipeline).
  int in_sweep = 0;                    // enqueue_sweep is running (prestaging allowed)
  int fuse = 1;                        // world 1: fused block tail (TRD_NO_FUSE=1: separate kernels)
  int64_t pipe_min_tiles = 0;          // blocks staging fewer tiles stay in line
  int pipe_inv = 0;                    // TRD_PIPE_INV=1: also restage invalidated sweep-invariant
                                       // blocks (after an upload: the value gather) on `stg`
                                       // (measured no gain on the C5b e2e path: off by default)
  bool prestaged[kMaxN] = {};          // block k's staging was enqueued ahead (consumed by its pass 1)
  int pipe = 0;                        // 0 off, 1 prestage after pass 1 of the previous block,
                                       // 2 after its pass 2, 3 split (sampler + bits after pass 1,
                                       // values after pass 2)
  cudaStream_t stg = nullptr;
  cudaEvent_t ev_stg_fork = nullptr, ev_p1[kMaxN] = {}, ev_p2[kMaxN] = {}, ev_samp[kMaxN] = {},
              ev_staged[kMaxN] = {};
  int32_t* idx_b[kMaxN] = {};
  int64_t* doff_b[kMaxN] = {};
  int64_t* row_off_b[kMaxN] = {};
  int64_t* col_off_b[kMaxN] = {};
  uint8_t* ptab_b[kMaxN] = {};
  int32_t* idx_d = nullptr;
  int64_t* doff_d = nullptr;
  int64_t* row_off_d = nullptr;
  int64_t* col_off_d = nullptr;
  uint8_t* ptab_d = nullptr;
  float* mid = nullptr;                // Mid(j_L): r_{k+1} x r_s
  float* lft = nullptr;                // Lft rows: [row][K]
  float* lfth = nullptr;               // Lft of the scaled gradient (pass 2)
  float* rgtT = nullptr;               // Rgt: [K][ncols]
  float* rgtC = nullptr;               // Rgt column-major [col][KP] (warp-per-row SIMT passes)
  // tensor-core operands: fp16 hi/lo core-matrix tiles, and per-row gradient contributions
  int want_tc = 1;                     // TRD_PASS=simt disables the tcgen05 pass kernels
  __half* lftHL = nullptr;             // [row][hi KP | lo KP] (A operand, loaded into TMEM)
  __half* lfthHL = nullptr;            // same for the scaled gradient (pass 2)
  float* lscl = nullptr;               // [row] 2^-E of the row's A scaling (pass 1)
  float* lsclh = nullptr;              // [row] same for pass 2
  __half* rgtHL = nullptr;             // [col tile][hi | lo][64 x KP] core-matrix layout (L1)
  __half* rgtHL2 = nullptr;            // same tiles, layout L2 ([hi KP | lo KP] per column)
  float* contrib = nullptr;            // [split][row][KP] D rows of pass 1
  float* tw = nullptr;                 // staged HQ weights of the current block (pass 1 -> 2)
  TcStage stage[kMaxN];
  double* dpart = nullptr;             // pass-1 CTA partials of d
  double* spart = nullptr;             // pass-1 CTA partial stats (3 per CTA)
  double* denpart = nullptr;           // pass-2 CTA partials
  double* numpart = nullptr;
  double* dvec = nullptr;              // [d (I_k x R2) | sum_e2 | welsch | n] allreduce buffer
  double* G = nullptr;                 // Gram of the current block
  double* G_last = nullptr;            // Gram of block N-1 (stop metric)
  double* Mop = nullptr;               // filtered operator M = A^-1 G A^-1
  double* chol_ws = nullptr;           // solve workspace (global fallback)
  double* chain_ws = nullptr;          // FGMC chain workspace (2 matrices)
  double* h = nullptr;                 // scaled gradient (I_k x R2)
  double* Dcur = nullptr;              // D^t
  double* Dprev = nullptr;             // D^{t-1}
  DevScalars* sc = nullptr;
  DevStats* stats = nullptr;
  int stats_cap = 0;
  double* red_ws = nullptr;            // small reductions
  size_t max_dpart = 0, max_spart = 0;

  // data-parallel exchange (world > 1): NCCL, or a caller-supplied allreduce (trd_init_ex)
  void* nccl_comm = nullptr;
  trd_exchange ex = {nullptr, nullptr};
  double* chk = nullptr;               // replica check: [h_lo, h_hi, -h_lo, -h_hi] of the cores
  unsigned long long* chk_acc = nullptr;

  // profiling (trd_set_profiling / trd_get_profile)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_pass1, ev_pass2;   // indices into ev_pool
  size_t ev_used = 0;

  // CUDA graphs of one sweep (world 1 or NCCL): per upload buffer set
  SweepGraph graphs[2];
  SweepGraph* capturing = nullptr;     // set while a sweep is being captured
  // TRD_TIMELINE diagnostic: (label, event, stream) marks of eager sweeps
  struct TlMark { const char* label; void* ev; int side; };
  bool tl_on = false;
  std::vector<TlMark> tl;
  cudaStream_t cap_stream = nullptr;   // capture stream (the caller's may be the legacy stream)

  // large-rank path (blocks with R_k^2 > kBigR2, trd_big.cu)
  int has_big = 0;
  void* blas = nullptr;                // cublasHandle_t
  void* solver = nullptr;              // cusolverDnHandle_t
  double* big_A = nullptr;             // A = G + lambda I, then its Cholesky factor (R2 x R2)
  double* big_gam = nullptr;           // Q refresh: Zd^T Zd (R2 x R2)
  double* big_zd = nullptr;            // Q refresh: the core in fp64, I_k x R2
  double* big_work = nullptr;          // potrf workspace
  int big_lwork = 0;
  int* big_info = nullptr;             // potrf / potrs status (device)
  int* big_info_h = nullptr;           // (pinned host copy)
  const double* big_G = nullptr;       // the Gram the current block's solve factorised
};

// ---- kernels (trd_kernels.cu) --------------------------------------------------------
void launch_sampler(Context& c, const BlockPlan& bp, cudaStream_t s);
// offsets = false: the row / column data offsets were computed ahead (pipelined staging, launch_offsets);
// only the operand-scale maxima are reset
void launch_plan(Context& c, const BlockPlan& bp, cudaStream_t s, bool offsets = true);
// row / column data offsets of block bp (reset_amax: also zero the operand-scale maxima of the block)
void launch_offsets(Context& c, const BlockPlan& bp, cudaStream_t s, bool reset_amax);
void launch_lft(Context& c, const BlockPlan& bp, const float* Zsrc_k, int src_is_h, float* out,
                cudaStream_t s);
void launch_pass1(Context& c, const BlockPlan& bp, int stats_only, cudaStream_t s);
void launch_reduce_d(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_block_stats(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_q(Context& c, int k, cudaStream_t s);
void launch_gram(Context& c, const BlockPlan& bp, cudaStream_t s, const double* Qsrc, double* Gout);
void launch_solve(Context& c, const BlockPlan& bp, cudaStream_t s, const double* G);
void launch_q_sampled(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_identity_op(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_h(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_pass2(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_reduce_den(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_update(Context& c, const BlockPlan& bp, cudaStream_t s);
// world 1: reduce_den + the block scalars (both phases) + the update in one single-CTA launch
void launch_block_tail(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_sweep_end(Context& c, cudaStream_t s);
void launch_core_checksum(Context& c, cudaStream_t s);   // -> c.chk (world > 1)
void launch_replica_check(Context& c, cudaStream_t s);
void launch_sigma0(Context& c, cudaStream_t s);
void launch_eabs_advance(Context& c, const TcStage& st, cudaStream_t s);
void launch_mad_hist(Context& c, int level, cudaStream_t s);   // R21 select, level 0..2
void launch_mad_scan(Context& c, int level, cudaStream_t s);
void launch_reconstruct(Context& c, const int64_t* lin, int64_t n, float* out, cudaStream_t s);
void launch_error(Context& c, const float* ref, const uint32_t* eval_bits, double* out4,
                  cudaStream_t s);
void launch_rank_prefix(Context& c, cudaStream_t s);
void launch_count_bits(Context& c, unsigned long long* out, cudaStream_t s);
void launch_amax_obs(Context& c, cudaStream_t s);   // sc->amax_x of the observed values
void launch_mask_compare(Context& c, cudaStream_t s); // sc->mask_same; stage_mask <- mask
void launch_sweep_begin(Context& c, cudaStream_t s);
void launch_phi(Context& c, const BlockPlan& bp, const double* C, double* G, cudaStream_t s);

// ---- large-rank path (trd_big.cu) ------------------------------------------------------
trd_status big_init(Context* c, int64_t r2big, int64_t zd_rows);   // handles + workspaces
void big_destroy(Context* c);
// row-major C (m x n) = A (m x q) B (q x n), fp64 (cuBLAS dgemm)
trd_status big_dgemm(Context& c, cudaStream_t s, int m, int n, int q, const double* A, const double* B, double* C);
trd_status big_q(Context& c, int k, cudaStream_t s);                 // Q_k refresh
trd_status big_gram(Context& c, const BlockPlan& bp, cudaStream_t s, const double* Qsrc, double* Gout);
trd_status big_factor(Context& c, const BlockPlan& bp, cudaStream_t s, const double* G);   // side stream
trd_status big_h(Context& c, const BlockPlan& bp, cudaStream_t s);   // host check + retries, h, num

// ---- tensor-core pass kernels (trd_tc.cu) ---------------------------------------------
bool tc_supported_kp(int KP);
bool stage_uses_pext(const Context& c, const BlockPlan& bp);   // sampler writes c.ptab
void launch_tc_pack_cols(Context& c, const BlockPlan& bp, cudaStream_t s);
void launch_tc_lft(Context& c, const BlockPlan& bp, bool pass2, cudaStream_t s);
void launch_tc_pass(Context& c, const BlockPlan& bp, const TcStage& st, bool pass2, cudaStream_t s);
void launch_tc_reduce_d(Context& c, const BlockPlan& bp, cudaStream_t s);
// d contraction of D rows in contrib ([nsplit][nrows_pad][KP]) for any R2, + final reduction
void launch_reduce_d_contrib(Context& c, const BlockPlan& bp, int nsplit, int64_t nrows_pad, int64_t nparts,
                             cudaStream_t s);
// phase 0: the whole staging; 1: masks, row offsets and tile prefix (stage_bits + scan); 2: the values
void launch_tc_stage(Context& c, const BlockPlan& bp, TcStage& st, cudaStream_t s, int phase = 0);
size_t tc_scan_tmp_bytes(int64_t n_tiles);
void tc_debug_dump();   // TRD_TC_EXP diagnostics

// checked build: read and clear the device check records of both translation units (the
// first failure of either), and set the schedule-fuzzing delay; false if none failed
bool tc_check_collect(DevCheck* out, unsigned int jitter_ns, cudaStream_t s);
bool kern_check_collect(DevCheck* out, unsigned int jitter_ns, cudaStream_t s);

}  // namespace trd

// trd_api.cu -- C ABI of libtrd (include/trd.h): validation, memory, block plans, the sweep
// orchestration of Alg. 1 and the NCCL data-parallel exchange.
#include <dlfcn.h>
#include <stdarg.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <new>
#include <vector>

#include "trd_internal.cuh"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost a pointer test without a tool

// NVTX ranges on the host side of the API (nsys / ncu --nvtx): one per call, per sweep and per
// block stage, so a profiler timeline shows which block and pass each enqueued kernel belongs to
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
static const char* const kNvtxBlock[] = {"trd block 0", "trd block 1", "trd block 2", "trd block 3",
                                         "trd block 4", "trd block 5", "trd block 6", "trd block 7"};

using namespace trd;

bool trd::g_pdl_on = false;

// ---------------------------------------------------------------------------------------
// NCCL, loaded lazily (world > 1 only) so a single-GPU context never needs it.
// ---------------------------------------------------------------------------------------
namespace {
typedef int (*nccl_get_unique_id_t)(void*);
struct NcclId { char internal[128]; };
typedef int (*nccl_comm_init_rank2_t)(void**, int, NcclId, int);
typedef int (*nccl_all_reduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_comm_destroy_t)(void*);
typedef const char* (*nccl_get_error_string_t)(int);

struct NcclApi {
  bool tried = false, ok = false;
  nccl_get_unique_id_t get_unique_id = nullptr;
  nccl_comm_init_rank2_t comm_init_rank = nullptr;
  nccl_all_reduce_t all_reduce = nullptr;
  nccl_comm_destroy_t comm_destroy = nullptr;
  nccl_get_error_string_t err_str = nullptr;
};
NcclApi g_nccl;

bool load_nccl() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.get_unique_id = (nccl_get_unique_id_t)dlsym(h, "ncclGetUniqueId");
  g_nccl.comm_init_rank = (nccl_comm_init_rank2_t)dlsym(h, "ncclCommInitRank");
  g_nccl.all_reduce = (nccl_all_reduce_t)dlsym(h, "ncclAllReduce");
  g_nccl.comm_destroy = (nccl_comm_destroy_t)dlsym(h, "ncclCommDestroy");
  g_nccl.err_str = (nccl_get_error_string_t)dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.all_reduce && g_nccl.comm_destroy;
  return g_nccl.ok;
}
constexpr int kNcclFloat64 = 8, kNcclSum = 0, kNcclMax = 2;

// ---------------------------------------------------------------------------------------
trd_status fail(Context* c, trd_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (st == TRD_ERR_CUDA || st == TRD_ERR_NCCL) c->sticky = st;
  }
  return st;
}

// checked build (trd_internal.cuh): collect the device check records of both kernel
// translation units and re-arm the schedule fuzzing (TRD_JITTER_NS)
bool check_both(DevCheck* out, unsigned int jitter_ns, cudaStream_t s) {
  DevCheck a = {}, b = {};
  const bool fa = tc_check_collect(&a, jitter_ns, s);
  const bool fb = kern_check_collect(&b, jitter_ns, s);
  *out = fa ? a : b;
  if (fa && fb) out->count += b.count;
  return fa || fb;
}
static trd_status device_checks(Context* c) {
  if (!TRD_CHECKED) return TRD_OK;
  const char* e = getenv("TRD_JITTER_NS");
  DevCheck d;
  if (check_both(&d, e ? (unsigned int)atoi(e) : 0u, c->stream))
    return fail(c, TRD_ERR_STATE, "device check %u failed (block %u thread %u; %u failures)", d.code, d.block,
                d.thread, d.count);
  return TRD_OK;
}

#define CUDA_TRY(ctx, expr)                                                                   \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(ctx, TRD_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));        \
  } while (0)

template <typename T>
trd_status dalloc(Context* c, T** p, size_t n) {
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) {
    *p = nullptr;
    cudaGetLastError();
    return fail(c, TRD_ERR_OOM, "cudaMalloc(%zu bytes) failed: %s", n * sizeof(T), cudaGetErrorString(e));
  }
  return TRD_OK;
}

trd_status check_launch(Context* c, const char* what) {
  if (c->sticky) return c->sticky;           // (a library call of the large-rank path failed)
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, TRD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return TRD_OK;
}

// cost model of a split p (v1 SIMT pass kernels): K per entry, lane utilisation of the
// 32-column chunks, with a mild preference for ~2k columns (L2-resident Rgt tiles)
double plan_cost(int64_t K, int64_t ncols) {
  const double chunks = std::ceil((double)ncols / 32.0);
  const double util = (double)ncols / (32.0 * chunks);
  const double shape = std::fabs(std::log2(std::max<double>(ncols, 1.0) / 2048.0));
  return (double)K / util * (1.0 + 0.02 * shape);
}

// cost model of a split p for the tensor-core pass kernels: dense MMA work scales with the
// padded inner dimension KP; narrow column sets (< one 64-column tile) waste the tile
double plan_cost_tc(int64_t K, int64_t ncols) {
  const double KP = (double)((K + 15) / 16 * 16);
  const double waste = ncols >= 64 ? std::ceil(ncols / 64.0) * 64.0 / ncols : 64.0 / ncols;
  const double shape = std::fabs(std::log2(std::max<double>(ncols, 1.0) / 4096.0));
  return KP * waste * (1.0 + 0.02 * shape);
}

void build_plan(const Context& c, int k, const int64_t* s_in, BlockPlan& bp, bool want_tc, bool rows = false) {
  const int N = c.N;
  memset(&bp, 0, sizeof(bp));
  bp.k = k;
  for (int m = 0; m < N; ++m) {
    int64_t s = s_in[m];
    if (m == k || s <= 0 || s >= c.dims[m]) s = c.dims[m];
    bp.s[m] = s;
  }
  // data parallel: the full index set of the shard mode (m != k) shrinks to this rank's slice
  {
    const int sm = c.cfg.shard_mode;
    const int64_t local = c.shard_end - c.shard_begin;
    for (int m = 0; m < N; ++m) bp.s_samp[m] = bp.s[m];
    if (!rows && bp.s[sm] == c.dims[sm] && local < c.dims[sm]) {
      bp.s[sm] = local;
      bp.shard_local = 1;
      if (sm == k) bp.ik0 = c.shard_begin;   // plan rows i_k = ik0 + local index
    } else if (!rows && sm != k && bp.s[sm] < c.dims[sm] && std::min<int64_t>(bp.s[sm], local) < bp.s[sm]) {
      bp.s[sm] = std::min<int64_t>(bp.s[sm], local);   // capacity for this rank's sampled indices
      bp.shard_sampled = 1;
    }
  }
  int64_t J = 1;                             // row sampling: J = prod_{m != k} s_m draws
  if (rows) {
    for (int m = 0; m < N; ++m) if (m != k) J *= bp.s[m];
    for (int m = 0; m < N; ++m) if (m != k) bp.s[m] = J;
    bp.explicit_cols = 1;
  }
  double best = 1e300;
  int best_p = 0;
  for (int p = 0; p <= (rows ? 0 : N - 2); ++p) {
    const int rs = c.ranks[(k + p + 1) % N];
    const int64_t K = (int64_t)c.ranks[k] * rs;
    int64_t ncols = 1;
    for (int q = p + 1; q <= N - 1; ++q) ncols *= bp.s[(k + q) % N];
    double cost = want_tc ? plan_cost_tc(K, ncols) : plan_cost(K, ncols);
    if (c.rbucket > 32) {
      // ranks > 32: K > 128 runs the SIMT pass (~8x the tensor-core cost per position), and
      // the chain products of the plan kernels (per column / left index / row, not shared
      // between them) can exceed the passes: add their FMAs per working-set position
      const int64_t KP = (K + 15) / 16 * 16;
      if (!(want_tc && KP <= 128)) cost = 8.0 * plan_cost(K, ncols);
      int64_t nL = 1;
      double f_mid = 0.0, f_rgt = 0.0;
      for (int q = 1; q <= p; ++q) {
        const int m = (k + q) % N;
        nL *= bp.s[m];
        f_mid += (double)c.ranks[m] * c.ranks[(m + 1) % N];
      }
      for (int q = p + 1; q <= N - 1; ++q) {
        const int m = (k + q) % N;
        f_rgt += (double)c.ranks[m] * c.ranks[(m + 1) % N];
      }
      const double rows = (double)bp.s[k] * nL;
      const double chain = (double)ncols * rs * f_rgt + (double)nL * c.ranks[(k + 1) % N] * f_mid +
                           (p > 0 ? rows * c.ranks[k] * c.ranks[(k + 1) % N] * rs : 0.0);
      cost += chain / std::max(1.0, rows * (double)ncols);
    }
    if (K > 256) cost += 1e200;            // the pass kernels need K = r_k r_s <= 256
    if (cost < best - 1e-12) { best = cost; best_p = p; }
  }
  const int p = best_p;
  bp.p = p;
  bp.nleft = p;
  bp.nright = N - 1 - p;
  bp.nL = 1;
  for (int q = 0; q < p; ++q) { bp.left[q] = (k + 1 + q) % N; bp.nL *= bp.s[bp.left[q]]; }
  bp.ncols = 1;
  for (int q = 0; q < bp.nright; ++q) { bp.right[q] = (k + 1 + p + q) % N; bp.ncols *= bp.s[bp.right[q]]; }
  if (rows) bp.ncols = J;
  // digit orders: mode 0 (unit stride in memory) becomes the fastest digit of its group, and
  // for k == 0 the rows enumerate i_0 fastest, so that the bitmask / packed values of
  // consecutive rows or columns are contiguous (coalesced in the pass kernels)
  auto order = [](const int* modes, int n, int* dig) {
    int q0 = -1;
    for (int q = 0; q < n; ++q) if (modes[q] == 0) q0 = q;
    int d = 0;
    if (q0 >= 0) dig[d++] = q0;
    for (int q = 0; q < n; ++q) if (q != q0) dig[d++] = q;
  };
  order(bp.left, bp.nleft, bp.ldig);
  order(bp.right, bp.nright, bp.rdig);
  bp.rowmode = (k == 0) ? 1 : 0;
  bp.rk = c.ranks[k];
  bp.rk1 = c.ranks[(k + 1) % N];
  bp.rs = c.ranks[(k + p + 1) % N];
  bp.K = bp.rk * bp.rs;
  bp.R2 = bp.rk * bp.rk1;
  const int64_t Ik = bp.s[k];                 // (this rank's slice when k is the shard mode)
  bp.nrows = Ik * bp.nL;
  bp.nnz_ws = bp.nrows * bp.ncols;
  bp.KP = (bp.K + 15) / 16 * 16;
  bp.use_tc = want_tc && bp.KP <= 256;
  bp.n_row_tiles = (bp.nrows + 127) / 128;
  bp.n_col_tiles = (bp.ncols + 63) / 64;
  {
    // persistent pass kernels: one CTA per SM walking (row tile, column split) items; pick
    // the split that minimises the busiest CTA's work (ties: fewer splits)
    const int64_t nrt = bp.n_row_tiles, nct = bp.n_col_tiles;
    // tile pairs (N = 128 GEMMs) for KP <= 64 unless there is a single column tile;
    // TRD_UNIT=1 forces single tiles
    const char* ue = getenv("TRD_UNIT");
    bp.tc_u = (bp.KP <= 64 && nct >= 2 && !(ue && atoi(ue) == 1)) ? 2 : 1;
    const int64_t U = bp.tc_u;
    double best = 1e300;
    int64_t best_s = 1, best_per = nct;
    for (int64_t sp = 1; sp <= std::min<int64_t>(nct, 64); ++sp) {
      const int64_t per = (nct + sp - 1) / sp;
      const int64_t se = (nct + per - 1) / per;             // no empty splits
      const int64_t items = nrt * se;
      const int64_t grid = std::min<int64_t>(items, (int64_t)c.num_sm);
      // busiest CTA: its items x (tiles per item + ~1 tile of per-item cost: A load, D drain
      // and the split's share of the d reduction).  C5b (TRD_NSPLIT): 1 and 2 splits equal
      // within run-to-run noise, 3 splits +3 %, 4 splits +6 %
      // (an odd split with tile pairs ends in a phantom half, costed as a whole tile)
      const double cost = (double)((items + grid - 1) / grid) * ((double)((per + U - 1) / U * U) + 1.0);
      if (cost < best - 1e-9) { best = cost; best_s = se; best_per = per; }
    }
    if (const char* e = getenv("TRD_NSPLIT")) {    // experiment knob: fixed column split count
      const int64_t sp = std::max<int64_t>(1, std::min<int64_t>(atoll(e), nct));
      best_per = (nct + sp - 1) / sp;
      best_s = (nct + best_per - 1) / best_per;
    }
    bp.tc_nsplit = (int)best_s;
    bp.tc_per = best_per;
    // CTA pairs (clusters of 2) share each B tile (half each, multicast); TRD_CLUSTER=1 disables
    const char* ce = getenv("TRD_CLUSTER");
    bp.tc_cl = (ce && atoi(ce) == 1) || c.num_sm < 4 ? 1 : 2;
    const int64_t groups = (nrt + bp.tc_cl - 1) / bp.tc_cl;      // row-tile groups
    const int64_t citems = groups * best_s;                          // items per cluster walk
    const int64_t ncl2 = ((int64_t)c.num_sm / bp.tc_cl);             // clusters that fit
    const int64_t ncl1 = (((int64_t)c.num_sm - 1) / bp.tc_cl);       // one SM left (side stream)
    bp.tc_grid = (int)(std::max<int64_t>(1, std::min<int64_t>(citems, ncl2)) * bp.tc_cl);
    bp.tc_grid1 = (int)(std::max<int64_t>(1, std::min<int64_t>(citems, ncl1)) * bp.tc_cl);
    const int64_t Ikk = bp.s[k];
    // d reduction: >= 8 CTAs per SM worth of (i_k, jl-chunk) blocks, chunks of >= 32 rows
    int64_t jc = (8 * (int64_t)c.num_sm + Ikk - 1) / Ikk;
    jc = std::max<int64_t>(1, std::min<int64_t>(jc, (bp.nL + 31) / 32));
    bp.tc_jl_chunk = (bp.nL + jc - 1) / jc;
    bp.tc_jc = (bp.nL + bp.tc_jl_chunk - 1) / bp.tc_jl_chunk;
  }
  // large-rank path (R^2 > kBigR2): the SIMT pass writes one D row per (row, split), so one
  // warp per row (ws_split = 1)
  bp.big = bp.R2 > kBigR2 ? 1 : 0;
  // geometry: 8 warps per CTA, one (row, column sub-range) item per warp
  if (bp.nL >= 8 || bp.big) { bp.jl_per_cta = (int)std::min<int64_t>(8, bp.nL); bp.ws_split = 1; }
  else {
    bp.jl_per_cta = (int)bp.nL;
    int ws = 8 / (int)bp.nL;
    int p2 = 1;
    while (p2 * 2 <= ws) p2 *= 2;
    bp.ws_split = p2;
  }
  bp.grid_x = (bp.nL + bp.jl_per_cta - 1) / bp.jl_per_cta;
  const int64_t base = bp.grid_x * Ik;
  int64_t nsplit = (4 * 148 + base - 1) / base;
  const int64_t maxsplit = std::max<int64_t>(1, bp.ncols / (64 * (int64_t)bp.ws_split));
  nsplit = std::min(nsplit, maxsplit);
  nsplit = std::max<int64_t>(nsplit, 1);
  nsplit = std::min<int64_t>(nsplit, 65535);
  bp.nsplit = (int)nsplit;
}

size_t ncta_of(const BlockPlan& bp) { return (size_t)(bp.grid_x * bp.nsplit); }

// the data-parallel exchange: NCCL on the context stream, or the caller's allreduce (trd_init_ex)
trd_status allreduce(Context* c, double* buf, size_t n, int op = TRD_OP_SUM) {
  if (c->cfg.world <= 1) return TRD_OK;
  if (c->ex.allreduce) {
    const int r = c->ex.allreduce(c->ex.user, buf, (uint64_t)n, op, (void*)c->stream);
    if (r != 0) return fail(c, TRD_ERR_NCCL, "exchange allreduce failed (%d)", r);
    return TRD_OK;
  }
  int r = g_nccl.all_reduce(buf, buf, n, kNcclFloat64, op == TRD_OP_MAX ? kNcclMax : kNcclSum, c->nccl_comm,
                            c->stream);
  if (r != 0) return fail(c, TRD_ERR_NCCL, "ncclAllReduce: %s", g_nccl.err_str ? g_nccl.err_str(r) : "?");
  return TRD_OK;
}

// profiling events around a pass kernel (pool reused across sweeps)
int prof_event_slot(Context* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    c->ev_pool.push_back(e);
  }
  return (int)c->ev_used++;
}
// During a sweep capture the event becomes a graph node: its own capture event, re-pointed at
// a pool event on every replay (launch_graph)
int prof_event(Context* c) {
  if (c->capturing) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    c->capturing->cap_ev.push_back(e);
    cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal);   // -> an event-record node
    return (int)c->capturing->cap_ev.size() - 1;
  }
  const int i = prof_event_slot(c);
  if (i >= 0) cudaEventRecord(c->ev_pool[(size_t)i], c->stream);
  return i;
}
void prof_pair(Context* c, int pass, int e0, int e1) {
  if (c->capturing) (pass == 1 ? c->capturing->pairs1 : c->capturing->pairs2).push_back({e0, e1});
  else (pass == 1 ? c->ev_pass1 : c->ev_pass2).push_back({e0, e1});
}

// TRD_TIMELINE=1 (diagnostic, eager sweeps only): events at the stage boundaries of every
// block on both streams; trd_destroy prints the mean time between consecutive marks
void tl_mark(Context* c, cudaStream_t s, const char* label) {
  if (!c->tl_on || c->capturing) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, s);
  c->tl.push_back({label, (void*)e, (s == c->side || strncmp(label, "side", 4) == 0) ? 1 : 0});
}

// index / offset buffers of block k (k < 0 or no pipeline: the context's default buffers)
void select_bufs(Context* c, int k) {
  if (!c->pipe) return;
  const bool d = k < 0;
  c->idx = d ? c->idx_d : c->idx_b[k];
  c->doff = d ? c->doff_d : c->doff_b[k];
  c->row_off = d ? c->row_off_d : c->row_off_b[k];
  c->col_off = d ? c->col_off_d : c->col_off_b[k];
  c->ptab = d ? c->ptab_d : c->ptab_b[k];
}

// block k takes part in the staging pipeline: a sampled (sweep-varying) tensor-core sketch
static bool pipelined(const Context* c, int k) {
  if (!c->pipe || k < 0 || k >= c->N || !c->plan[k].use_tc || c->plan[k].explicit_cols) return false;
  if (c->stage[k].invariant) return c->pipe_inv && !c->stage[k].valid;
  return c->stage[k].n_tiles >= c->pipe_min_tiles;
}

// Enqueue part `part` of block k's staging on the staging stream after `after` (an event of the
// main stream): part 0 = everything, 1 = sampler, offsets, masks and tile prefix, 2 = values.
// Records ev_samp[k] once the index sets and offsets exist and ev_staged[k] after the values.
// The index sets depend only on (seed, k, t), the staging only on them and the data: none of it
// reads the cores that blocks < k are still updating (Alg. 1 l.4-5).
static trd_status prestage(Context* c, int k, cudaEvent_t after, int part, int cur_block) {
  const BlockPlan& bp = c->plan[k];
  cudaStream_t t = c->stg;
  CUDA_TRY(c, cudaStreamWaitEvent(t, after, 0));
  select_bufs(c, k);
  if (part != 2) {
    launch_sampler(*c, bp, t);
    launch_offsets(*c, bp, t, false);
    CUDA_TRY(c, cudaEventRecord(c->ev_samp[k], t));
  }
  launch_tc_stage(*c, bp, c->stage[k], t, part);
  if (part != 1) CUDA_TRY(c, cudaEventRecord(c->ev_staged[k], t));
  if (part != 2) c->prestaged[k] = true;
  if (part != 1 && c->stage[k].invariant) c->stage[k].valid = true;
  select_bufs(c, cur_block);
  return check_launch(c, "prestage");
}

// inside enqueue_sweep with world 1: den reduction, block scalars and update as one launch
// (launch_block_tail; TRD_NO_FUSE=1 keeps the separate kernels)
static bool fuse_tail(const Context* c) { return c->in_sweep && c->cfg.world <= 1 && c->fuse; }

// inside enqueue_sweep: the staging of block k + 1 is enqueued ahead (block 0 stages in line)
static bool pre_next(const Context* c, int k) { return c->in_sweep && pipelined(c, k + 1); }

// a1-a6 + a7 (pass 1 and the d/stat exchange) of block k.  pre: the sampler, offsets and staging
// of this block were enqueued ahead on the staging stream (enqueue_sweep)
trd_status block_pass1(Context* c, const BlockPlan& bp, bool pre) {
  cudaStream_t s = c->stream;
  select_bufs(c, bp.k);
  // a8 + a9 (FGMC Gram, filtered operator M) depend only on the cores != k: run them on the
  // side stream, overlapping the sampler / staging / pass 1 (which leaves one SM free)
  // (the sampler first: the local-scaled-term arm builds its Gram from the sampled slices)
  tl_mark(c, s, "block start");
  if (pre) CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_samp[bp.k], 0));
  else launch_sampler(*c, bp, s);
  tl_mark(c, s, "sampler");
  // (TRD_NO_SIDE=1, diagnostic: the Gram and the solve in line on the main stream)
  const bool inl = getenv("TRD_NO_SIDE") && atoi(getenv("TRD_NO_SIDE")) != 0;
  cudaStream_t side = inl ? s : c->side;
  CUDA_TRY(c, cudaEventRecord(c->ev_fork, s));
  CUDA_TRY(c, cudaStreamWaitEvent(side, c->ev_fork, 0));
  tl_mark(c, side, "side: fork");
  launch_gram(*c, bp, side, c->Q, c->G);                // FGMC Gram (also the stop metric's)
  tl_mark(c, side, "side: gram");
  if (c->cfg.scaling == TRD_SCALING_GLOBAL) {
    launch_solve(*c, bp, side, c->G);
  } else if (c->cfg.scaling == TRD_SCALING_NONE) {
    launch_identity_op(*c, bp, side);                    // h = d ('gradient descent' arm)
  } else {                                               // 'local scaled term' arm
    launch_q_sampled(*c, bp, side);
    launch_gram(*c, bp, side, c->Qloc, c->Gloc);
    launch_solve(*c, bp, side, c->Gloc);
  }
  tl_mark(c, side, "side: solve");
  if (c->sticky) return c->sticky;
  CUDA_TRY(c, cudaEventRecord(c->ev_join, side));
  launch_plan(*c, bp, s, !pre);
  tl_mark(c, s, "plan (offsets, mid, rgt)");
  if (!bp.use_tc) launch_lft(*c, bp, c->Z + c->zoff[bp.k], 0, c->lft, s);
  TcStage& stg = c->stage[bp.k];
  if (bp.use_tc) {                          // Lft built directly as the fp16 hi / lo A operand
    launch_tc_lft(*c, bp, false, s);
    tl_mark(c, s, "lft pack 1");
    launch_tc_pack_cols(*c, bp, s);
    tl_mark(c, s, "pack cols");
    if (pre) {
      CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_staged[bp.k], 0));
    } else if (!stg.valid) {                // a2: stage the sketch in tile order
      launch_tc_stage(*c, bp, stg, s);
      stg.valid = stg.invariant;
      // checked build only: TRD_CHECK_INJECT=entry corrupts the first staged entry id of this
      // block (an id outside the tile), which the pass kernels must report (tests/test_gpu_checked.py)
      if (TRD_CHECKED && getenv("TRD_CHECK_INJECT") && !strcmp(getenv("TRD_CHECK_INJECT"), "entry"))
        CUDA_TRY(c, cudaMemsetAsync(stg.tidx, 0xFE, 2, s));
      static const char* kStageLabel[kMaxN] = {"stage k=0", "stage k=1", "stage k=2", "stage k=3",
                                               "stage k=4", "stage k=5", "stage k=6", "stage k=7"};
      tl_mark(c, s, kStageLabel[bp.k]);
    }
  }
  const bool pe = c->prof || c->capturing;
  const int e0 = pe ? prof_event(c) : -1;
  if (bp.use_tc) launch_tc_pass(*c, bp, stg, false, s);
  else launch_pass1(*c, bp, 0, s);
  if (pe) prof_pair(c, 1, e0, prof_event(c));
  tl_mark(c, s, "pass 1");
  const bool inv_next = bp.k + 1 < c->N && c->stage[bp.k + 1].invariant;
  if (pre_next(c, bp.k) && (c->pipe != 2 || inv_next)) {   // the next block's staging, behind this pass 1
    CUDA_TRY(c, cudaEventRecord(c->ev_p1[bp.k], s));    // (pipe 1 or invariant: all of it, 3: up to the prefix)
    trd_status sp = prestage(c, bp.k + 1, c->ev_p1[bp.k], (c->pipe == 1 || inv_next) ? 0 : 1, bp.k);
    if (sp) return sp;
  }
  if (bp.use_tc && c->eabs) launch_eabs_advance(*c, stg, s);   // R21 |e| slots of this block
  if (bp.use_tc) launch_tc_reduce_d(*c, bp, s);
  else launch_reduce_d(*c, bp, s);
  trd_status st = check_launch(c, "pass 1");
  if (st) return st;
  const int64_t Ik = c->dims[bp.k];
  tl_mark(c, s, "reduce d");
  st = allreduce(c, c->dvec, (size_t)(Ik * bp.R2 + 3));
  if (st) return st;
  if (!fuse_tail(c)) launch_block_stats(*c, bp, s);
  tl_mark(c, s, "exchange + stats");
  return TRD_OK;
}

// a8-a10 (FGMC, solve, scaled gradient, pass 2, den exchange)
trd_status block_pass2(Context* c, const BlockPlan& bp) {
  cudaStream_t s = c->stream;
  CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_join, 0));       // M of this block (side stream)
  tl_mark(c, s, "join (wait for the solve)");
  launch_h(*c, bp, s);
  if (c->sticky) return c->sticky;           // (large-rank path: library call failures)
  tl_mark(c, s, "h = d M");
  if (!bp.use_tc) launch_lft(*c, bp, nullptr, 1, c->lfth, s);
  else launch_tc_lft(*c, bp, true, s);
  tl_mark(c, s, "lft pack 2");
  const bool pe = c->prof || c->capturing;
  const int e0 = pe ? prof_event(c) : -1;
  if (bp.use_tc) launch_tc_pass(*c, bp, c->stage[bp.k], true, s);
  else launch_pass2(*c, bp, s);
  if (pe) prof_pair(c, 2, e0, prof_event(c));
  tl_mark(c, s, "pass 2");
  if (pre_next(c, bp.k) && c->pipe >= 2 && !(bp.k + 1 < c->N && c->stage[bp.k + 1].invariant)) {   // (pipe 2: all of it, 3: the values)
    CUDA_TRY(c, cudaEventRecord(c->ev_p2[bp.k], s));
    trd_status sp = prestage(c, bp.k + 1, c->ev_p2[bp.k], c->pipe == 2 ? 0 : 2, bp.k);
    if (sp) return sp;
  }
  if (!fuse_tail(c)) launch_reduce_den(*c, bp, s);
  tl_mark(c, s, "reduce den");
  trd_status st = check_launch(c, "pass 2");
  if (st) return st;
  return allreduce(c, c->red_ws, 1);
}

// R21: exact median of eabs[0, eabs_fill) (all ranks' values: the histograms are allreduced)
trd_status mad_select(Context* c) {
  cudaStream_t s = c->stream;
  for (int level = 0; level < 3; ++level) {
    launch_mad_hist(*c, level, s);
    const size_t off = level == 0 ? 0 : level == 1 ? kMadBins0 : kMadBins0 + 2 * kMadBins1;
    const size_t n = level == 0 ? kMadBins0 : level == 1 ? 2 * kMadBins1 : 2 * kMadBins2;
    trd_status st = allreduce(c, c->mhist + off, n);
    if (st) return st;
    launch_mad_scan(*c, level, s);
  }
  return check_launch(c, "mad select");
}

trd_status ensure_stats(Context* c, int n) {
  if (n <= c->stats_cap) return TRD_OK;
  if (c->stats) cudaFree(c->stats);
  c->stats = nullptr;
  trd_status st = dalloc(c, &c->stats, (size_t)n);
  if (st) return st;
  c->stats_cap = n;
  return TRD_OK;
}

trd_status sigma0_pass(Context* c) {
  select_bufs(c, -1);
  const BlockPlan& bp = c->full_plan;
  cudaStream_t s = c->stream;
  if (c->eabs) CUDA_TRY(c, cudaMemsetAsync(&c->sc->eabs_fill, 0, sizeof(unsigned long long), s));
  launch_sampler(*c, bp, s);
  launch_plan(*c, bp, s);
  launch_lft(*c, bp, c->Z + c->zoff[bp.k], 0, c->lft, s);
  launch_pass1(*c, bp, 1, s);
  // reduce the statistics into red_ws[0..2]: reuse reduce_d with R2 = 0 semantics
  BlockPlan tmp = bp;
  tmp.R2 = 0;
  tmp.big = 0;
  double* saved = c->dvec;
  c->dvec = c->red_ws;
  launch_reduce_d(*c, tmp, s);
  c->dvec = saved;
  trd_status st = check_launch(c, "sigma0 pass");
  if (st) return st;
  st = allreduce(c, c->red_ws, 3);
  if (st) return st;
  if (c->eabs && (st = mad_select(c))) return st;
  launch_sigma0(*c, s);
  return check_launch(c, "sigma0");
}

// observed entries of the local mask (dense storage; packed: n_values)
trd_status count_observed(Context* c, int64_t* out) {
  unsigned long long* d = nullptr;
  CUDA_TRY(c, cudaMalloc(&d, sizeof(unsigned long long)));
  launch_count_bits(*c, d, c->stream);
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(c, TRD_ERR_CUDA, "count_observed: %s", cudaGetErrorString(e));
  *out = (int64_t)h;
  return TRD_OK;
}

void host_to_dev_core(const Context& c, int k, const float* src, std::vector<float>& tmp) {
  const int r0 = c.ranks[k], r1 = c.ranks[(k + 1) % c.N];
  const int64_t I = c.dims[k];
  tmp.resize((size_t)(r0 * I * r1));
  for (int a = 0; a < r0; ++a)
    for (int64_t i = 0; i < I; ++i)
      for (int b = 0; b < r1; ++b) tmp[(i * r0 + a) * r1 + b] = src[(a * I + i) * r1 + b];
}

}  // namespace

// =======================================================================================
extern "C" {

const char* trd_version(void) {
  return TRD_CHECKED ? "libtrd 0.3 checked (device invariant checks, mbarrier watchdog, schedule fuzzing)"
                     : "libtrd 0.3 (sm_100a: persistent tcgen05 pass kernels, CTA pairs; fp64 FGMC / filtered solve)";
}

trd_status trd_nccl_unique_id(void* out128) {
  if (!out128) return TRD_ERR_INVALID_ARG;
  if (!load_nccl()) return TRD_ERR_NCCL;
  return g_nccl.get_unique_id(out128) == 0 ? TRD_OK : TRD_ERR_NCCL;
}

const char* trd_last_error(const trd_ctx* ctx) {
  if (!ctx) return "null context";
  return reinterpret_cast<const Context*>(ctx)->err.c_str();
}

int64_t trd_launch_count(const trd_ctx* ctx) {
  return ctx ? reinterpret_cast<const Context*>(ctx)->launches : 0;
}

trd_status trd_set_profiling(trd_ctx* ctx, int32_t enable) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->prof = enable != 0;
  c->ev_used = 0;
  c->ev_pass1.clear();
  c->ev_pass2.clear();
  DevScalars hs;
  CUDA_TRY(c, cudaMemcpy(&hs, c->sc, sizeof(hs), cudaMemcpyDeviceToHost));
  hs.prof_on = c->prof ? 1 : 0;
  for (int k = 0; k < kMaxN; ++k) hs.prof_nobs[k] = 0.0;
  CUDA_TRY(c, cudaMemcpy(c->sc, &hs, sizeof(hs), cudaMemcpyHostToDevice));
  return TRD_OK;
}

trd_status trd_get_profile(trd_ctx* ctx, trd_profile* out) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c || !out) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  memset(out, 0, sizeof(*out));
  for (auto& pr : c->ev_pass1) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev_pool[(size_t)pr.first], c->ev_pool[(size_t)pr.second]);
    out->pass1_ms += ms;
  }
  for (auto& pr : c->ev_pass2) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev_pool[(size_t)pr.first], c->ev_pool[(size_t)pr.second]);
    out->pass2_ms += ms;
  }
  out->pass1_launches = (int64_t)c->ev_pass1.size();
  out->pass2_launches = (int64_t)c->ev_pass2.size();
  DevScalars hs;
  CUDA_TRY(c, cudaMemcpy(&hs, c->sc, sizeof(hs), cudaMemcpyDeviceToHost));
  // algorithmic counts: pass 1 = recon + gradient (4 K + 8 flops per observed
  // entry; value 4 B + staged weight 4 B + mask bits), pass 2 = line-search dot (2 K + 4 flops;
  // weight 4 B + mask bits), K = the per-entry contraction length of the block's GEMM form,
  // r_k r_s <= R^2 (= R^2 with equal ranks: every BASELINE config; with unequal ranks the split
  // needs fewer flops per entry than the full subchain's R^2, and counting R^2 would put the
  // achieved rate above the FP32 peak).  Blocks were visited cyclically, so each block's launches
  // are n_launch / N.
  const double per_block = c->ev_pass1.empty() ? 0.0 : (double)c->ev_pass1.size() / c->N;
  for (int k = 0; k < c->N; ++k) {
    const double n = hs.prof_nobs[k];
    const double R2 = (double)std::min(c->plan[k].R2, c->plan[k].K);
    const double ws_bits = (double)c->plan[k].nnz_ws / c->cfg.world / 8.0 * per_block;
    out->pass1_entries += n;
    out->pass2_entries += n;
    out->pass1_flops += n * (4.0 * R2 + 8.0);
    out->pass2_flops += n * (2.0 * R2 + 4.0);
    out->pass1_bytes += 8.0 * n + ws_bits;
    out->pass2_bytes += 4.0 * n + ws_bits;
    const BlockPlan& bp = c->plan[k];
    if (bp.use_tc) {
      // per 128 x 64 tile: 3 split terms x 2 x 128 x 64 x KP flops per GEMM; pass 1 runs two
      // GEMMs (S = A.B^T and D += P.B), pass 2 one
      const double tile = 3.0 * 2.0 * 128.0 * 64.0 * (double)bp.KP;
      const double tiles = (double)bp.n_row_tiles * (double)bp.n_col_tiles * per_block;
      out->pass1_mma_flops += 2.0 * tile * tiles;
      out->pass2_mma_flops += tile * tiles;
    }
  }
  return TRD_OK;
}

trd_status trd_init(const trd_config* cfg, const trd_shard* shard, const float* const* init_cores,
                    void* stream, trd_ctx** out) {
  return trd_init_ex(cfg, shard, init_cores, stream, nullptr, out);
}

trd_status trd_init_ex(const trd_config* cfg, const trd_shard* shard, const float* const* init_cores,
                       void* stream, const trd_exchange* ex, trd_ctx** out) {
  if (!out) return TRD_ERR_INVALID_ARG;
  NvtxRange nr("trd_init");
  *out = nullptr;
  if (!cfg || !shard || !init_cores) return TRD_ERR_INVALID_ARG;
  const int N = cfg->order;
  if (N < 3 || N > TRD_MAX_ORDER) return TRD_ERR_SHAPE;
  for (int m = 0; m < N; ++m) {
    if (cfg->dims[m] < 1 || cfg->dims[m] > (1LL << 31) - 1) return TRD_ERR_SHAPE;
    if (cfg->ranks[m] < 1 || cfg->ranks[m] > TRD_MAX_RANK) return TRD_ERR_SHAPE;
    if (cfg->sketch[m] < 0) return TRD_ERR_SHAPE;
    if (!init_cores[m]) return TRD_ERR_INVALID_ARG;
  }
  if (cfg->sigma_mode < 0 || cfg->sigma_mode > TRD_SIGMA_MAD) return TRD_ERR_INVALID_ARG;
  if (cfg->sigma_mode == TRD_SIGMA_FIXED && !(cfg->sigma > 0.0)) return TRD_ERR_INVALID_ARG;
  if ((cfg->sigma_mode == TRD_SIGMA_RMS || cfg->sigma_mode == TRD_SIGMA_MAD) &&
      (!(cfg->sigma_theta > 0.0) || !(cfg->sigma_min > 0.0)))
    return TRD_ERR_INVALID_ARG;
  if (!(cfg->lambda_rel >= 0.0) || !(cfg->step >= 0.0)) return TRD_ERR_INVALID_ARG;
  if (cfg->scaling < TRD_SCALING_GLOBAL || cfg->scaling > TRD_SCALING_LOCAL) return TRD_ERR_INVALID_ARG;
  if (cfg->sampling < TRD_SAMPLING_RSTS || cfg->sampling > TRD_SAMPLING_ROWS) return TRD_ERR_INVALID_ARG;
  if (cfg->sampling == TRD_SAMPLING_ROWS && cfg->scaling == TRD_SCALING_LOCAL) return TRD_ERR_INVALID_ARG;
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return TRD_ERR_INVALID_ARG;
  if (cfg->shard_mode < 0 || cfg->shard_mode >= N) return TRD_ERR_SHAPE;
  if (ex && !ex->allreduce) return TRD_ERR_INVALID_ARG;
  if (cfg->world > 1 && !cfg->nccl_unique_id && !ex) return TRD_ERR_INVALID_ARG;
  if (!shard->values || !shard->mask_bits) return TRD_ERR_INVALID_ARG;
  const int sm = cfg->shard_mode;
  const int64_t sb = shard->shard_begin, se = shard->shard_end;
  if (sb < 0 || se > cfg->dims[sm] || se <= sb) return TRD_ERR_SHAPE;
  // (world == 1 with a partial shard: that shard's partial problem, no exchange -- used by
  //  the single-GPU tests of the per-rank plans)
  if (cfg->dims[N - 1] > 16384) return TRD_ERR_SHAPE;   // D^t is I_N x I_N (Alg. 1 l.12)

  Context* c = new (std::nothrow) Context();
  if (!c) return TRD_ERR_OOM;
  c->cfg = *cfg;
  c->cfg.nccl_unique_id = nullptr;
  c->tl_on = getenv("TRD_TIMELINE") && atoi(getenv("TRD_TIMELINE")) != 0;
  c->fuse = !(getenv("TRD_NO_FUSE") && atoi(getenv("TRD_NO_FUSE")) != 0);
  // (process-wide launch mode; PDL measured neutral to slightly slower -- C4 0.757 without vs
  //  0.777 ms per sweep with, 50 timed sweeps -- so ordinary launches unless TRD_PDL=1)
  g_pdl_on = getenv("TRD_PDL") && atoi(getenv("TRD_PDL")) != 0;
  if (ex && cfg->world > 1) c->ex = *ex;
  c->N = N;
  c->stream = (cudaStream_t)stream;
  {
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0)
      c->num_sm = nsm;
    // test knob: TRD_NUM_SM=n sizes the persistent grids for n SMs (n < SM count makes every
    // CTA walk many work items; used by the parity tests of the item-boundary logic)
    if (const char* e = getenv("TRD_NUM_SM")) {
      const int v = atoi(e);
      if (v > 0 && v < c->num_sm) c->num_sm = v;
    }
  }
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    trd_destroy(reinterpret_cast<trd_ctx*>(c));
    return TRD_ERR_CUDA;
  }

  c->shard_begin = sb;
  c->shard_end = se;
  c->packed = shard->packed ? 1 : 0;
  int64_t stride = 1;
  for (int m = 0; m < N; ++m) {
    c->dims[m] = cfg->dims[m];
    c->ranks[m] = cfg->ranks[m];
    c->ldims[m] = (m == sm) ? (se - sb) : cfg->dims[m];
    c->lstride[m] = stride;
    stride *= c->ldims[m];
  }
  c->n_local = stride;
  c->n_words = (c->n_local + 31) / 32;
  int64_t r2max = 1, chain_max = 1;
  for (int k = 0; k < N; ++k) {
    const int64_t r2 = (int64_t)c->ranks[k] * c->ranks[(k + 1) % N];
    if (r2 > kMaxR2) { delete c; return TRD_ERR_SHAPE; }
    r2max = std::max(r2max, r2);
    c->rbucket = std::max(c->rbucket, c->ranks[k] <= 16 ? 16 : c->ranks[k] <= 32 ? 32 : 128);
    // FGMC chain products r_{k+1}^2 x r_m^2 (Eq. 13): the largest intermediate
    for (int m = 0; m < N; ++m)
      chain_max = std::max(chain_max, (int64_t)c->ranks[(k + 1) % N] * c->ranks[(k + 1) % N] * c->ranks[m] * c->ranks[m]);
  }
  c->chain_half = (size_t)chain_max;
  int64_t r2big = 0, zd_rows = 0;                 // large-rank blocks (trd_big.cu)
  for (int k = 0; k < N; ++k) {
    const int64_t r2 = (int64_t)c->ranks[k] * c->ranks[(k + 1) % N];
    if (r2 > kBigR2) { r2big = std::max(r2big, r2); zd_rows = std::max<int64_t>(zd_rows, c->dims[k]); }
  }
  if (r2big > 0)                                  // (cuSOLVER loaded: every R2 > 128 solve uses it;
    for (int k = 0; k < N; ++k)                   //  the one-CTA Cholesky takes ~13 ms at R2 = 240)
      if ((int64_t)c->ranks[k] * c->ranks[(k + 1) % N] > 128)
        zd_rows = std::max<int64_t>(zd_rows, c->dims[k]);
  if (r2big > 0) {                                // chain products in either order: <= (max r)^4
    int64_t rmax = 0;
    for (int k = 0; k < N; ++k) rmax = std::max<int64_t>(rmax, c->ranks[k]);
    c->chain_half = std::max(c->chain_half, (size_t)(rmax * rmax * rmax * rmax));
    c->has_big = 1;
  }

  trd_status st = TRD_OK;
  auto bail = [&](trd_status s2) { trd_destroy(reinterpret_cast<trd_ctx*>(c)); return s2; };

  // ---- plans and workspace sizes ----
  size_t max_rows = 0, max_cols = 0, max_lft = 0, max_rgt = 0, max_mid = 0, max_dp = 0, max_sp = 0;
  size_t max_dvec = 0, max_h = 0, idx_total = 0;
  size_t max_lhl = 0, max_rhl = 0, max_contrib = 0, max_rpad = 0, max_rgtc = 0;
  int64_t full_s[kMaxN];
  for (int m = 0; m < N; ++m) full_s[m] = 0;
  bool rows_forced = false;
  {
    const char* pe = getenv("TRD_PASS");
    c->want_tc = !(pe && (strcmp(pe, "simt") == 0 || strcmp(pe, "rows") == 0));
    // (TRD_PASS=rows, measurement: every block through the warp-per-row SIMT passes, which touch
    //  the observed entries only -- the per-entry SIMT cost of DESIGN.md sec. 7)
    rows_forced = pe && strcmp(pe, "rows") == 0;
  }
  for (int k = 0; k <= N; ++k) {
    BlockPlan& bp = (k < N) ? c->plan[k] : c->full_plan;
    if (k < N) build_plan(*c, k, cfg->sketch, bp, c->want_tc != 0, cfg->sampling == TRD_SAMPLING_ROWS);
    else build_plan(*c, 0, full_s, bp, false);
    if (bp.use_tc && !tc_supported_kp(bp.KP)) bp.use_tc = 0;
    if (bp.K > 256) return bail(fail(c, TRD_ERR_SHAPE, "block %d: no split with r_k r_s <= 256", k));
    bp.lib_solve = (bp.big || (c->has_big && bp.R2 > 128)) ? 1 : 0;
    bp.rows = 0;
    if (!bp.use_tc && (bp.K > 128 || (rows_forced && k < N))) {   // warp-per-row SIMT passes (simt_rows_kernel)
      bp.rows = 1;
      int64_t ns = ((int64_t)c->num_sm * 64 + bp.nrows - 1) / std::max<int64_t>(1, bp.nrows);
      ns = std::max<int64_t>(1, std::min<int64_t>(ns, std::max<int64_t>(1, bp.ncols / 64)));
      int64_t per = (bp.ncols + ns - 1) / ns;
      per = (per + 31) / 32 * 32;
      bp.rows_per = per;
      bp.rows_nsplit = (int)((bp.ncols + per - 1) / per);
      const int64_t items = bp.nrows * bp.rows_nsplit;
      bp.rows_grid = (int)std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, (int64_t)c->num_sm * 8));
      max_rgtc = std::max(max_rgtc, (size_t)(bp.ncols * bp.KP));
      max_sp = std::max(max_sp, (size_t)bp.rows_grid * 3);
      if (k < N) {
        max_contrib = std::max(max_contrib, (size_t)bp.rows_nsplit * bp.nrows * bp.KP);
        max_dp = std::max(max_dp, (size_t)(bp.tc_jc * c->dims[bp.k] * bp.R2));
      }
    }
    if (bp.use_tc) {
      TcStage& st = c->stage[k];
      st.n_tiles = bp.n_row_tiles * bp.n_col_tiles;
      st.invariant = true;
      for (int m = 0; m < N; ++m)
        if (m != k && bp.s[m] < c->dims[m] && !(m == cfg->shard_mode && bp.shard_local)) st.invariant = false;
      if (bp.explicit_cols) st.invariant = false;          // rows are redrawn every sweep
      st.vcap = bp.n_row_tiles * 128 * bp.n_col_tiles * 64;   // refined after the data is known
      max_lhl = std::max(max_lhl, (size_t)(bp.n_row_tiles * 2 * 128 * bp.KP));
      max_rpad = std::max(max_rpad, (size_t)(bp.n_row_tiles * 128));
      max_rhl = std::max(max_rhl, (size_t)(bp.n_col_tiles * 2 * 64 * bp.KP));
      max_contrib = std::max(max_contrib, (size_t)bp.tc_nsplit * bp.n_row_tiles * 128 * bp.KP);
      max_sp = std::max(max_sp, (size_t)bp.tc_grid * 3);
      max_dp = std::max(max_dp, (size_t)(bp.tc_jc * c->dims[bp.k] * bp.R2));
    } else if (bp.big && !bp.rows && k < N) {   // SIMT D rows [nsplit][nrows][KP], contracted per jl chunk
      max_contrib = std::max(max_contrib, (size_t)bp.nsplit * bp.nrows * bp.KP);
      max_dp = std::max(max_dp, (size_t)(bp.tc_jc * c->dims[bp.k] * bp.R2));
    }
    max_rows = std::max(max_rows, (size_t)bp.nrows);
    max_cols = std::max(max_cols, (size_t)bp.ncols);
    max_lft = std::max(max_lft, (size_t)(bp.nrows * bp.K));
    max_rgt = std::max(max_rgt, (size_t)(bp.ncols * bp.K));
    max_mid = std::max(max_mid, (size_t)(bp.nL * bp.rk1 * bp.rs));
    const size_t Ik = (size_t)c->dims[bp.k];
    if (!bp.big && !bp.rows) max_dp = std::max(max_dp, Ik * ncta_of(bp) * (size_t)bp.R2);
    if (!bp.rows) max_sp = std::max(max_sp, Ik * ncta_of(bp) * 3);
    max_dvec = std::max(max_dvec, Ik * (size_t)bp.R2 + 3);
    max_h = std::max(max_h, Ik * (size_t)bp.R2);
  }
  // index lists per mode: the RStS sets (<= I_m) or, with row sampling, J_k draws
  int64_t jmax = 0;
  if (cfg->sampling == TRD_SAMPLING_ROWS)
    for (int k = 0; k < N; ++k) {
      int64_t J = 1;
      for (int m = 0; m < N; ++m)
        if (m != k) J *= (cfg->sketch[m] <= 0 || cfg->sketch[m] >= c->dims[m]) ? c->dims[m] : cfg->sketch[m];
      jmax = std::max(jmax, J);
    }
  for (int m = 0; m < N; ++m) {
    c->idx_off[m] = (int64_t)idx_total;
    idx_total += (size_t)std::max<int64_t>(c->dims[m], jmax);
  }
  c->idx_off[N] = (int64_t)idx_total;
  max_dp = std::max(max_dp, (size_t)(148 * 4 * 6));

  // ---- allocations ----
  int64_t ztot = 0, qtot = 0;
  for (int k = 0; k < N; ++k) {
    c->zoff[k] = ztot;
    c->qoff[k] = qtot;
    const int64_t r0 = c->ranks[k], r1 = c->ranks[(k + 1) % N];
    ztot += r0 * c->dims[k] * r1;
    qtot += r0 * r0 * r1 * r1;
  }
  c->zoff[N] = ztot;
  c->qoff[N] = qtot;
  const int64_t In = c->dims[N - 1];
  const size_t chain_cap = std::max((size_t)2 * chain_max, (size_t)(In * r2max));   // (+ D^t's T)
  const size_t g2 = (size_t)(r2max * r2max);
  if ((st = dalloc(c, &c->Z, (size_t)ztot)) || (st = dalloc(c, &c->Q, (size_t)qtot)) ||
      (st = dalloc(c, &c->idx, idx_total)) || (st = dalloc(c, &c->doff, idx_total)) ||
      (st = dalloc(c, &c->row_off, max_rows)) || (st = dalloc(c, &c->col_off, max_cols)) ||
      (st = dalloc(c, &c->mid, max_mid)) || (st = dalloc(c, &c->lft, max_lft)) ||
      (st = dalloc(c, &c->lfth, max_lft)) || (st = dalloc(c, &c->rgtT, max_rgt)) ||
      (st = dalloc(c, &c->dpart, max_dp)) || (st = dalloc(c, &c->spart, max_sp)) ||
      (st = dalloc(c, &c->denpart, max_sp)) || (st = dalloc(c, &c->numpart, max_h)) ||
      (st = dalloc(c, &c->dvec, max_dvec)) || (st = dalloc(c, &c->G, g2)) ||
      (st = dalloc(c, &c->G_last, g2)) || (st = dalloc(c, &c->Mop, g2)) ||
      (st = dalloc(c, &c->chol_ws, 2 * g2)) ||
      (st = dalloc(c, &c->chain_ws, chain_cap)) || (st = dalloc(c, &c->h, max_h)) ||
      (st = dalloc(c, &c->Dcur, (size_t)(In * In))) || (st = dalloc(c, &c->Dprev, (size_t)(In * In))) ||
      (st = dalloc(c, &c->sc, 1)) || (st = dalloc(c, &c->red_ws, 1024)))
    return bail(st);
  if (cfg->sigma_mode == TRD_SIGMA_MAD && (st = dalloc(c, &c->mhist, (size_t)kMadHist))) return bail(st);
  if (cfg->scaling == TRD_SCALING_LOCAL &&
      ((st = dalloc(c, &c->Qloc, (size_t)qtot)) || (st = dalloc(c, &c->Gloc, g2))))
    return bail(st);
  if (max_lhl > 0) {
    if ((st = dalloc(c, &c->lftHL, max_lhl)) || (st = dalloc(c, &c->lfthHL, max_lhl)) ||
        (st = dalloc(c, &c->lscl, max_rpad)) || (st = dalloc(c, &c->lsclh, max_rpad)) ||
        (st = dalloc(c, &c->rgtHL, max_rhl)) || (st = dalloc(c, &c->rgtHL2, max_rhl)))
      return bail(st);
  }
  if (max_contrib > 0 && (st = dalloc(c, &c->contrib, max_contrib))) return bail(st);
  if (max_rgtc > 0 && (st = dalloc(c, &c->rgtC, max_rgtc))) return bail(st);
  if (c->has_big && (st = big_init(c, r2big, zd_rows))) return bail(st);
  if ((st = ensure_stats(c, 4))) return bail(st);
  cudaStream_t s = c->stream;

  // ---- data ----
  if (shard->host) {
    if ((st = dalloc(c, &c->own_mask, (size_t)c->n_words))) return bail(st);
    CUDA_TRY(c, cudaMemcpyAsync(c->own_mask, shard->mask_bits, c->n_words * 4, cudaMemcpyHostToDevice, s));
    c->mask = c->own_mask;
  } else {
    c->mask = shard->mask_bits;
  }
  if (c->packed) {
    if ((st = dalloc(c, &c->rank_prefix, (size_t)c->n_words))) return bail(st);
    launch_rank_prefix(*c, s);
    uint32_t last_pref = 0, last_word = 0;
    CUDA_TRY(c, cudaMemcpyAsync(&last_pref, c->rank_prefix + c->n_words - 1, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaMemcpyAsync(&last_word, c->mask + c->n_words - 1, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    int64_t tail_bits = c->n_local - (c->n_words - 1) * 32;
    if (tail_bits < 32) last_word &= (1u << tail_bits) - 1u;
    c->n_values = (int64_t)last_pref + __builtin_popcount(last_word);
  } else {
    c->n_values = c->n_local;
  }
  // ---- staged working sets of the tensor-core blocks (a2) ----
  {
    int64_t max_v = 0;
    for (int k = 0; k < N; ++k) {
      if (!c->plan[k].use_tc) continue;
      TcStage& sg = c->stage[k];
      const int64_t obs_cap = c->packed ? c->n_values : c->n_local;
      // (row sampling draws with replacement: a duplicate draw stages an observed entry again,
      //  so explicit-column plans keep the dense working-set bound)
      if (!c->plan[k].explicit_cols) sg.vcap = std::min(sg.vcap, obs_cap);
      sg.vcap = std::max<int64_t>(1, sg.vcap) + 8 * sg.n_tiles;   // + tile padding
      sg.scan_tmp_bytes = tc_scan_tmp_bytes(sg.n_tiles);
      if ((st = dalloc(c, &sg.tbits, (size_t)sg.n_tiles * 128)) ||
          (st = dalloc(c, &sg.troff, (size_t)sg.n_tiles * 128)) ||
          (st = dalloc(c, &sg.tcount, (size_t)sg.n_tiles + 1)) ||
          (st = dalloc(c, &sg.tbase, (size_t)sg.n_tiles + 1)) ||
          (st = dalloc(c, &sg.tvals, (size_t)sg.vcap)) || (st = dalloc(c, &sg.tidx, (size_t)sg.vcap)) ||
          (st = dalloc(c, reinterpret_cast<char**>(&sg.scan_tmp), sg.scan_tmp_bytes + 16)))
        return bail(st);
      max_v = std::max(max_v, sg.vcap);
      CUDA_TRY(c, cudaMemsetAsync(sg.tcount, 0, ((size_t)sg.n_tiles + 1) * sizeof(uint64_t), c->stream));
      // layout cache of a sweep-invariant sketch (value indices fit int32): an upload whose mask
      // equals the staged one only re-gathers the values (e2e restaging)
      if (sg.invariant && (c->packed || c->n_local < (1LL << 31)) && !getenv("TRD_NO_PERM")) {
        if ((st = dalloc(c, &sg.perm, (size_t)sg.vcap))) return bail(st);
        if (!c->stage_mask) {
          if ((st = dalloc(c, &c->stage_mask, (size_t)c->n_words))) return bail(st);
          CUDA_TRY(c, cudaMemcpyAsync(c->stage_mask, c->mask, c->n_words * 4, cudaMemcpyDeviceToDevice, c->stream));
        }
      }
    }
    if (max_v > 0 && (st = dalloc(c, &c->tw, (size_t)max_v))) return bail(st);
    if ((st = dalloc(c, &c->ptab, (size_t)(16 * 256 + 16)))) return bail(st);
  }
  // ---- pipelined staging of the sampled tensor-core blocks (TRD_PIPE=0 disables) ----
  {
    const char* pe = getenv("TRD_PIPE");
    const int mode = pe ? atoi(pe) : kPipeDefault;
    c->pipe_min_tiles = pe ? 0 : kPipeMinTiles;     // (an explicit TRD_PIPE pipelines every sampled block)
    c->pipe_inv = getenv("TRD_PIPE_INV") && atoi(getenv("TRD_PIPE_INV")) != 0;
    bool any = false;
    for (int k = 0; k < N; ++k)
      if (c->plan[k].use_tc && !c->plan[k].explicit_cols &&
          (c->stage[k].invariant ? c->pipe_inv != 0 : c->stage[k].n_tiles >= c->pipe_min_tiles))
        any = true;
    if (mode > 0 && mode <= 3 && any) {
      c->idx_d = c->idx; c->doff_d = c->doff; c->row_off_d = c->row_off; c->col_off_d = c->col_off;
      c->ptab_d = c->ptab;
      if (cudaStreamCreateWithFlags(&c->stg, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->ev_stg_fork, cudaEventDisableTiming) != cudaSuccess)
        return bail(TRD_ERR_CUDA);
      for (int k = 0; k < N; ++k) {
        if (cudaEventCreateWithFlags(&c->ev_p1[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_p2[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_samp[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_staged[k], cudaEventDisableTiming) != cudaSuccess)
          return bail(TRD_ERR_CUDA);
        const BlockPlan& bp = c->plan[k];
        if ((st = dalloc(c, &c->idx_b[k], idx_total)) || (st = dalloc(c, &c->doff_b[k], idx_total)) ||
            (st = dalloc(c, &c->row_off_b[k], (size_t)std::max<int64_t>(1, bp.nrows))) ||
            (st = dalloc(c, &c->col_off_b[k], (size_t)std::max<int64_t>(1, bp.ncols))) ||
            (st = dalloc(c, &c->ptab_b[k], (size_t)(16 * 256 + 16))))
          return bail(st);
      }
      c->pipe = mode;
    }
  }
  // R21: |e| slots of one sweep (every block's staged slots, or its observed entries) or of the
  // sigma_0 pass (all local observed entries)
  if (cfg->sigma_mode == TRD_SIGMA_MAD) {
    int64_t n_obs = c->n_values;
    if (!c->packed) {
      if ((st = count_observed(c, &n_obs))) return bail(st);
    }
    int64_t per_sweep = 0;
    for (int k = 0; k < N; ++k)
      per_sweep += c->plan[k].use_tc ? c->stage[k].vcap : std::min<int64_t>(c->plan[k].nnz_ws, n_obs);
    c->eabs_cap = (size_t)std::max<int64_t>(per_sweep, n_obs);
    if ((st = dalloc(c, &c->eabs, c->eabs_cap))) return bail(st);
  }
  if (shard->host) {
    if ((st = dalloc(c, &c->own_values, (size_t)c->n_values))) return bail(st);
    CUDA_TRY(c, cudaMemcpyAsync(c->own_values, shard->values, c->n_values * 4, cudaMemcpyHostToDevice, s));
    c->values = c->own_values;
  } else {
    c->values = shard->values;
  }

  // ---- cores, scalars, FGMC cache ----
  {
    std::vector<float> tmp;
    for (int k = 0; k < N; ++k) {
      host_to_dev_core(*c, k, init_cores[k], tmp);
      CUDA_TRY(c, cudaMemcpy(c->Z + c->zoff[k], tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  DevScalars hs;
  memset(&hs, 0, sizeof(hs));
  hs.sigma = cfg->sigma_mode == TRD_SIGMA_FIXED ? cfg->sigma : (cfg->sigma_mode == TRD_SIGMA_INF ? INFINITY : 1.0);
  hs.mask_gen = 1;                             // (layout_gen = 0: no staged layout built yet)
  CUDA_TRY(c, cudaMemcpyAsync(c->sc, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemsetAsync(c->Dprev, 0, (size_t)(In * In) * 8, s));
  launch_amax_obs(*c, s);
  for (int k = 0; k < N; ++k) launch_q(*c, k, s);
  if ((st = check_launch(c, "init Q"))) return bail(st);

  if (cfg->world > 1 &&
      ((st = dalloc(c, &c->chk, 4)) || (st = dalloc(c, &c->chk_acc, 1))))
    return bail(st);
  // ---- NCCL (unless the caller supplied the exchange) ----
  if (cfg->world > 1 && !c->ex.allreduce) {
    if (!load_nccl()) return bail(fail(c, TRD_ERR_NCCL, "libnccl.so.2 could not be loaded"));
    NcclId id;
    memcpy(id.internal, cfg->nccl_unique_id, 128);
    CUDA_TRY(c, cudaStreamSynchronize(s));
    int r = g_nccl.comm_init_rank(&c->nccl_comm, cfg->world, id, cfg->rank);
    if (r != 0) return bail(fail(c, TRD_ERR_NCCL, "ncclCommInitRank failed (%d)", r));
  }
  if (cfg->sigma_mode == TRD_SIGMA_RMS || cfg->sigma_mode == TRD_SIGMA_MAD) {
    if ((st = sigma0_pass(c))) return bail(st);
  }
  CUDA_TRY(c, cudaStreamSynchronize(s));
  if ((st = device_checks(c))) return bail(st);
  *out = reinterpret_cast<trd_ctx*>(c);
  return TRD_OK;
}

trd_status trd_upload(trd_ctx* ctx, const float* values_host, const uint32_t* mask_host) {
  Context* c = reinterpret_cast<Context*>(ctx);
  NvtxRange nr("trd_upload");
  if (!c || !values_host || !mask_host) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  if (!c->own_values || !c->own_mask) return fail(c, TRD_ERR_STATE, "shard is not host-resident");
  if (c->up_npend >= 2) return fail(c, TRD_ERR_STATE, "two uploads already pending (run a sweep first)");
  trd_status st;
  if (!c->copy) {                            // lazily: copy stream, events, second buffer set
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_up_ready[b], cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_up_free, cudaEventDisableTiming));
    c->up_values[0] = c->own_values;
    c->up_mask[0] = c->own_mask;
    if ((st = dalloc(c, &c->up_values[1], (size_t)c->n_values))) return st;
    if ((st = dalloc(c, &c->up_mask[1], (size_t)c->n_words))) return st;
  }
  // target: the set that is neither the active one nor pending (with one upload pending,
  // the active set -- the next sweep switches away from it before any later use)
  const int b = c->up_npend == 0 ? 1 - c->up_active : 1 - c->up_pend[0];
  // the copy may only overwrite b after all work enqueued so far (which may read it) is done
  CUDA_TRY(c, cudaEventRecord(c->ev_up_free, c->stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->copy, c->ev_up_free, 0));
  CUDA_TRY(c, cudaMemcpyAsync(c->up_mask[b], mask_host, c->n_words * 4, cudaMemcpyHostToDevice, c->copy));
  CUDA_TRY(c, cudaMemcpyAsync(c->up_values[b], values_host, c->n_values * 4, cudaMemcpyHostToDevice, c->copy));
  CUDA_TRY(c, cudaEventRecord(c->ev_up_ready[b], c->copy));
  c->up_pend[c->up_npend++] = b;
  return check_launch(c, "upload");
}

// start of a sweep: switch to the oldest pending upload (its copy finished before any kernel
// of this sweep reads it), rebuild the packed rank prefix, invalidate the staged sketches
static trd_status consume_upload(Context* c) {
  if (c->up_npend == 0) return TRD_OK;
  const int b = c->up_pend[0];
  c->up_pend[0] = c->up_pend[1];
  --c->up_npend;
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_up_ready[b], 0));
  // trd.h: the host buffers of an upload may be reused once the consuming call returns, so
  // that call returns only after the copy has read them
  CUDA_TRY(c, cudaEventSynchronize(c->ev_up_ready[b]));
  c->up_active = b;
  c->own_values = c->up_values[b];
  c->own_mask = c->up_mask[b];
  c->values = c->own_values;
  c->mask = c->own_mask;
  if (c->packed) launch_rank_prefix(*c, c->stream);
  launch_amax_obs(*c, c->stream);
  if (c->stage_mask) launch_mask_compare(*c, c->stream);      // staged layouts reusable?
  for (int k = 0; k < c->N; ++k) c->stage[k].valid = false;   // staged values are stale
  return check_launch(c, "upload consume");
}

trd_status trd_sketch(trd_ctx* ctx, int32_t sweep, int32_t k, int32_t* idx_dev, int64_t* sizes_host) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c || !idx_dev || !sizes_host) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  if (k < 0 || k >= c->N || sweep < 0) return TRD_ERR_INVALID_ARG;
  const BlockPlan& bp = c->plan[k];
  int saved = 0;                             // (read on the context stream: sweeps may be in flight)
  CUDA_TRY(c, cudaMemcpyAsync(&saved, &c->sc->sweep, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&c->sc->sweep, &sweep, 4, cudaMemcpyHostToDevice, c->stream));
  select_bufs(c, -1);
  launch_sampler(*c, bp, c->stream);
  trd_status st = check_launch(c, "sampler");
  if (st) return st;
  int64_t off = 0;
  for (int m = 0; m < c->N; ++m) {
    CUDA_TRY(c, cudaMemcpyAsync(idx_dev + off, c->idx + c->idx_off[m], bp.s[m] * 4,
                                cudaMemcpyDeviceToDevice, c->stream));
    sizes_host[m] = bp.s[m];
    off += bp.s[m];
  }
  CUDA_TRY(c, cudaMemcpyAsync(&c->sc->sweep, &saved, 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TRD_OK;
}

// One sweep of Alg. 1 (lines 3-13) enqueued on the context stream (eagerly or under capture).
static trd_status enqueue_sweep(Context* c) {
  cudaStream_t s = c->stream;
  trd_status st;
  launch_sweep_begin(*c, s);
  struct InSweep {                       // (prestaging of block k + 1 only inside a sweep)
    Context* c;
    explicit InSweep(Context* cc) : c(cc) { c->in_sweep = 1; }
    ~InSweep() {
      c->in_sweep = 0;
      select_bufs(c, -1);
      for (int k = 0; k < kMaxN; ++k) c->prestaged[k] = false;
    }
  } in_sweep(c);
  // (the Q refresh on the side stream; TRD_Q_SIDE=0 keeps it in line.  Measured with 50 timed
  //  sweeps, ms per sweep in line / side: C3 0.643 / 0.628, C4 0.777 / 0.755, C5a 1.942 / 1.924)
  const bool q_side = !(getenv("TRD_NO_SIDE") && atoi(getenv("TRD_NO_SIDE")) != 0) &&
                      !(getenv("TRD_Q_SIDE") && atoi(getenv("TRD_Q_SIDE")) == 0);
  bool q_pending = false;
  for (int k = 0; k < c->N; ++k) {
    const BlockPlan& bp = c->plan[k];
    NvtxRange nr(kNvtxBlock[k]);
    const bool pre = c->prestaged[k];
    c->prestaged[k] = false;
    if ((st = block_pass1(c, bp, pre))) return st;
    if ((st = block_pass2(c, bp))) return st;
    if (k == c->N - 1)
      CUDA_TRY(c, cudaMemcpyAsync(c->G_last, c->G, (size_t)bp.R2 * bp.R2 * 8, cudaMemcpyDeviceToDevice, s));
    if (fuse_tail(c)) launch_block_tail(*c, bp, s);
    else launch_update(*c, bp, s);
    tl_mark(c, s, "step + update");
    // Q_k of the updated core (Eq. 13's factor) is read only by the next blocks' FGMC Gram on the
    // side stream: optionally refresh it there (large-rank Q by cuBLAS stays in line)
    // (only when the next block's solve is short, R^2 <= 64: behind a long Gauss-Jordan solve the
    //  extra side-stream work lands on the critical path -- C4, R^2 = 100: 0.775 ms per sweep with
    //  every refresh on the side stream vs 0.754 in line)
    if (q_side && (int64_t)c->ranks[k] * c->ranks[(k + 1) % c->N] <= kBigR2 && c->plan[(k + 1) % c->N].R2 <= 64) {
      CUDA_TRY(c, cudaEventRecord(c->ev_fork, s));
      CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
      launch_q(*c, k, c->side);
      q_pending = true;
    } else {
      launch_q(*c, k, s);
    }
    tl_mark(c, s, "Q refresh");
    if ((st = check_launch(c, "update"))) return st;
  }
  if (q_pending) {                        // join the side stream's last Q refresh
    CUDA_TRY(c, cudaEventRecord(c->ev_join, c->side));
    CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_join, 0));
  }
  if (c->eabs) {
    NvtxRange nr("trd mad select");
    if ((st = mad_select(c))) return st;                   // R21 (histograms allreduced)
  }
  launch_sweep_end(*c, s);
  tl_mark(c, s, "sweep end (D^t, sigma)");
  if (c->cfg.world > 1) {                 // replica consistency of the replicated cores
    launch_core_checksum(*c, s);
    if ((st = allreduce(c, c->chk, 4, TRD_OP_MAX))) return st;
    launch_replica_check(*c, s);
  }
  return check_launch(c, "sweep end");
}

static void destroy_graph(SweepGraph& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.graph) cudaGraphDestroy(g.graph);
  for (cudaEvent_t e : g.cap_ev) cudaEventDestroy(e);
  g = SweepGraph();
}

// A sweep can be replayed from a captured CUDA graph when nothing in it synchronises the host
// (the caller-supplied exchange does) and the invariant staged sketches are current (the
// graph then holds no staging); TRD_GRAPH=0 disables graphs.
static bool graph_usable(const Context* c) {
  const char* ge = getenv("TRD_GRAPH");
  const bool off = (ge && atoi(ge) == 0) || c->tl_on;
  // (large-rank blocks sync the host; world > 1: eager launches -- NCCL collectives inside a
  //  captured sweep are not exercised on the single-GPU test pool, and graphs measured equal
  //  to eager launching for every config)
  if (off || c->ex.allreduce || c->has_big || c->cfg.world > 1) return false;
  for (int k = 0; k < c->N; ++k)
    if (c->plan[k].use_tc && c->stage[k].invariant && !c->stage[k].valid) return false;
  return true;
}

static trd_status capture_sweep(Context* c, SweepGraph& g) {
  destroy_graph(g);
  const long long l0 = c->launches;
  // capture on a library stream (the caller's may be the legacy default stream, which cannot
  // be captured); the graph is launched on the caller's stream
  if (!c->cap_stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  cudaStream_t user = c->stream;
  c->stream = c->cap_stream;
  c->capturing = &g;
  cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed);
  trd_status st = e == cudaSuccess ? enqueue_sweep(c) : TRD_OK;
  cudaGraph_t graph = nullptr;
  if (e == cudaSuccess) e = cudaStreamEndCapture(c->stream, &graph);
  c->capturing = nullptr;
  c->stream = user;
  if (st) { if (graph) cudaGraphDestroy(graph); return st; }
  if (e != cudaSuccess) return fail(c, TRD_ERR_CUDA, "sweep capture: %s", cudaGetErrorString(e));
  g.graph = graph;
  CUDA_TRY(c, cudaGraphInstantiate(&g.exec, graph, 0));
  g.launches = c->launches - l0;
  c->launches = l0;
  // the event-record nodes of the profiling events, in capture order
  size_t nn = 0;
  CUDA_TRY(c, cudaGraphGetNodes(graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CUDA_TRY(c, cudaGraphGetNodes(graph, nodes.data(), &nn));
  g.ev_nodes.assign(g.cap_ev.size(), nullptr);
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    CUDA_TRY(c, cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t ev;
    CUDA_TRY(c, cudaGraphEventRecordNodeGetEvent(nd, &ev));
    for (size_t i = 0; i < g.cap_ev.size(); ++i)
      if (g.cap_ev[i] == ev) g.ev_nodes[i] = nd;
  }
  for (cudaGraphNode_t nd : g.ev_nodes)
    if (!nd) return fail(c, TRD_ERR_CUDA, "sweep capture: profiling event node not found");
  g.stats_ptr = c->stats;
  return TRD_OK;
}

// replay: point the profiling events of this launch at fresh pool events, then launch
static trd_status launch_graph(Context* c, SweepGraph& g) {
  if (c->prof) {
    std::vector<int> map(g.cap_ev.size());
    for (size_t i = 0; i < g.cap_ev.size(); ++i) {
      const int idx = prof_event_slot(c);
      if (idx < 0) return fail(c, TRD_ERR_CUDA, "profiling event");
      map[i] = idx;
      CUDA_TRY(c, cudaGraphExecEventRecordNodeSetEvent(g.exec, g.ev_nodes[i], c->ev_pool[(size_t)idx]));
    }
    for (auto& pr : g.pairs1) c->ev_pass1.push_back({map[(size_t)pr.first], map[(size_t)pr.second]});
    for (auto& pr : g.pairs2) c->ev_pass2.push_back({map[(size_t)pr.first], map[(size_t)pr.second]});
  }
  CUDA_TRY(c, cudaGraphLaunch(g.exec, c->stream));
  c->launches += g.launches;
  return TRD_OK;
}

trd_status trd_sweep(trd_ctx* ctx, int32_t n_sweeps, trd_sweep_stats* stats) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c || n_sweeps < 0) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  if (n_sweeps == 0) return TRD_OK;
  NvtxRange nr("trd_sweep");
  trd_status st = ensure_stats(c, n_sweeps);
  if (st) return st;
  {
    NvtxRange nu("trd consume upload");
    if ((st = consume_upload(c))) return st;
  }
  cudaStream_t s = c->stream;
  CUDA_TRY(c, cudaMemsetAsync(&c->sc->slot_next, 0, sizeof(int), s));
  std::vector<cudaEvent_t> ev;
  if (stats) {
    ev.resize((size_t)n_sweeps + 1);
    for (auto& e : ev) CUDA_TRY(c, cudaEventCreate(&e));
    CUDA_TRY(c, cudaEventRecord(ev[0], s));
  }
  if (TRD_CHECKED && (st = device_checks(c))) return st;     // (re-arms the jitter)
  for (int t = 0; t < n_sweeps; ++t) {
    NvtxRange ns("trd sweep");
    if (graph_usable(c)) {
      SweepGraph& g = c->graphs[c->up_active];
      if (!g.exec || g.stats_ptr != c->stats) {
        if ((st = capture_sweep(c, g))) return st;
      }
      if ((st = launch_graph(c, g))) return st;
    } else {
      if ((st = enqueue_sweep(c))) return st;
    }
    if (stats) CUDA_TRY(c, cudaEventRecord(ev[(size_t)t + 1], s));
  }
  if (TRD_CHECKED && (st = device_checks(c))) return st;
  if (!stats) return TRD_OK;
  std::vector<DevStats> hs((size_t)n_sweeps);
  CUDA_TRY(c, cudaMemcpyAsync(hs.data(), c->stats, sizeof(DevStats) * n_sweeps, cudaMemcpyDeviceToHost, s));
  DevScalars sc;
  CUDA_TRY(c, cudaMemcpyAsync(&sc, c->sc, sizeof(sc), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  bool nonfinite = false;
  for (int t = 0; t < n_sweeps; ++t) {
    trd_sweep_stats& o = stats[t];
    memset(&o, 0, sizeof(o));
    const DevStats& d = hs[(size_t)t];
    o.sigma = d.sigma; o.sum_e2 = d.sum_e2; o.welsch_loss = d.welsch; o.stop_e = d.stop_e;
    o.n_obs = d.n_obs;
    for (int k = 0; k < c->N; ++k) { o.eta[k] = d.eta[k]; o.num[k] = d.num[k]; o.den[k] = d.den[k]; o.nnz[k] = d.nnz[k]; }
    o.skipped_mask = d.skipped;
    o.replica_mismatch = d.replica_mismatch;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[(size_t)t], ev[(size_t)t + 1]);
    o.ms = ms;
    nonfinite |= d.nonfinite != 0;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (sc.not_spd) return fail(c, TRD_ERR_NOT_SPD, "G + lambda I not positive definite after retries");
  if (nonfinite || sc.nonfinite) return fail(c, TRD_ERR_NONFINITE, "non-finite step or statistics");
  if (sc.replica_bad) return fail(c, TRD_ERR_STATE, "replicas diverged: the ranks' cores differ");
  return TRD_OK;
}

trd_status trd_block_probe(trd_ctx* ctx, int32_t sweep, int32_t k, double* d_host, double* G_host,
                           double* h_host, double* stats5_host) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  if (k < 0 || k >= c->N || sweep < 0) return TRD_ERR_INVALID_ARG;
  if (trd_status su = consume_upload(c)) return su;
  const BlockPlan& bp = c->plan[k];
  cudaStream_t s = c->stream;
  int saved = 0;                             // (read on the context stream: sweeps may be in flight)
  CUDA_TRY(c, cudaMemcpyAsync(&saved, &c->sc->sweep, 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  CUDA_TRY(c, cudaMemcpyAsync(&c->sc->sweep, &sweep, 4, cudaMemcpyHostToDevice, s));
  if (c->eabs) CUDA_TRY(c, cudaMemsetAsync(&c->sc->eabs_fill, 0, sizeof(unsigned long long), s));
  CUDA_TRY(c, cudaMemsetAsync(&c->sc->slot, 0, sizeof(int), s));
  trd_status st;
  if ((st = block_pass1(c, bp, false))) return st;
  if ((st = block_pass2(c, bp))) return st;
  select_bufs(c, -1);
  const int64_t Ik = c->dims[k];
  std::vector<double> dv((size_t)(Ik * bp.R2 + 3));
  double nd[2];
  CUDA_TRY(c, cudaMemcpyAsync(dv.data(), c->dvec, dv.size() * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(nd, c->red_ws, 16, cudaMemcpyDeviceToHost, s));
  if (G_host) CUDA_TRY(c, cudaMemcpyAsync(G_host, c->G, (size_t)bp.R2 * bp.R2 * 8, cudaMemcpyDeviceToHost, s));
  if (h_host) CUDA_TRY(c, cudaMemcpyAsync(h_host, c->h, (size_t)(Ik * bp.R2) * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(&c->sc->sweep, &saved, 4, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  if (TRD_CHECKED && (st = device_checks(c))) return st;
  if (d_host) memcpy(d_host, dv.data(), (size_t)(Ik * bp.R2) * 8);
  if (stats5_host) {
    stats5_host[0] = dv[(size_t)(Ik * bp.R2)];
    stats5_host[1] = dv[(size_t)(Ik * bp.R2) + 2];
    stats5_host[2] = dv[(size_t)(Ik * bp.R2) + 1];
    stats5_host[3] = nd[1];
    stats5_host[4] = nd[0];
  }
  return TRD_OK;
}

trd_status trd_reconstruct(trd_ctx* ctx, const int64_t* lin_idx_dev, int64_t n, float* out_dev) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c || (n > 0 && (!lin_idx_dev || !out_dev)) || n < 0) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  if (n == 0) return TRD_OK;
  launch_reconstruct(*c, lin_idx_dev, n, out_dev, c->stream);
  return check_launch(c, "reconstruct");
}

trd_status trd_error(trd_ctx* ctx, const float* ref_dev, const uint32_t* eval_bits, double peak,
                     trd_error_stats* out) {
  Context* c = reinterpret_cast<Context*>(ctx);
  NvtxRange nr("trd_error");
  if (!c || !ref_dev || !out || !(peak >= 0.0)) return TRD_ERR_INVALID_ARG;
  if (peak == 0.0) peak = 1.0;                // data rescaled to [0, 1]
  if (c->sticky) return c->sticky;
  if (trd_status su = consume_upload(c)) return su;
  const BlockPlan& bp = c->full_plan;
  cudaStream_t s = c->stream;
  select_bufs(c, -1);
  launch_sampler(*c, bp, s);
  launch_plan(*c, bp, s);
  launch_lft(*c, bp, c->Z + c->zoff[bp.k], 0, c->lft, s);
  launch_error(*c, ref_dev, eval_bits, c->red_ws, s);
  trd_status st = check_launch(c, "error");
  if (st) return st;
  double v[6];
  if (c->cfg.world > 1) {
    if ((st = allreduce(c, c->red_ws, 5))) return st;                 // sums
    if ((st = allreduce(c, c->red_ws + 5, 1, TRD_OP_MAX))) return st;   // max |ref|
  }
  CUDA_TRY(c, cudaMemcpyAsync(v, c->red_ws, sizeof(v), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  out->rel_err_all = v[1] > 0 ? sqrt(v[0] / v[1]) : 0.0;
  out->rel_err_observed = v[3] > 0 ? sqrt(v[2] / v[3]) : 0.0;
  out->n_eval = (int64_t)v[4];
  const double mse = v[4] > 0 ? v[0] / v[4] : 0.0;
  out->psnr = mse > 0 ? 10.0 * log10(peak * peak / mse) : INFINITY;
  return TRD_OK;
}

trd_status trd_get_cores(trd_ctx* ctx, float* const* cores_host) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c || !cores_host) return TRD_ERR_INVALID_ARG;
  std::vector<float> tmp;
  bool nonfinite = false;
  cudaStreamSynchronize(c->stream);
  for (int k = 0; k < c->N; ++k) {
    if (!cores_host[k]) return TRD_ERR_INVALID_ARG;
    const int r0 = c->ranks[k], r1 = c->ranks[(k + 1) % c->N];
    const int64_t I = c->dims[k];
    tmp.resize((size_t)(r0 * I * r1));
    cudaError_t e = cudaMemcpy(tmp.data(), c->Z + c->zoff[k], tmp.size() * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(c, TRD_ERR_CUDA, "get_cores: %s", cudaGetErrorString(e));
    for (int a = 0; a < r0; ++a)
      for (int64_t i = 0; i < I; ++i)
        for (int b = 0; b < r1; ++b) cores_host[k][(a * I + i) * r1 + b] = tmp[(i * r0 + a) * r1 + b];
    for (const float v : tmp)
      if (!std::isfinite(v)) nonfinite = true;
  }
  if (!c->sticky) {
    DevScalars hs;
    if (cudaMemcpy(&hs, c->sc, sizeof(hs), cudaMemcpyDeviceToHost) == cudaSuccess && hs.nonfinite) nonfinite = true;
  }
  if (nonfinite) return fail(c, TRD_ERR_NONFINITE, "non-finite core values or statistics");
  return TRD_OK;
}

trd_status trd_set_cores(trd_ctx* ctx, const float* const* cores_host) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c || !cores_host) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  std::vector<float> tmp;
  for (int k = 0; k < c->N; ++k) {
    if (!cores_host[k]) return TRD_ERR_INVALID_ARG;
    host_to_dev_core(*c, k, cores_host[k], tmp);
    CUDA_TRY(c, cudaMemcpyAsync(c->Z + c->zoff[k], tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  }
  for (int k = 0; k < c->N; ++k) launch_q(*c, k, c->stream);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return check_launch(c, "set_cores");
}

trd_status trd_get_state(trd_ctx* ctx, trd_state* out, double* prev_D_host) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c || !out) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  const int64_t In = c->dims[c->N - 1];
  DevScalars hs;
  CUDA_TRY(c, cudaMemcpyAsync(&hs, c->sc, sizeof(hs), cudaMemcpyDeviceToHost, c->stream));
  if (prev_D_host)
    CUDA_TRY(c, cudaMemcpyAsync(prev_D_host, c->Dprev, (size_t)(In * In) * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  out->sigma = hs.sigma;
  out->sweep = hs.sweep;
  out->have_prev_D = hs.have_prev_D;
  out->prev_D_size = In * In;
  return TRD_OK;
}

trd_status trd_set_state(trd_ctx* ctx, const trd_state* st, const double* prev_D_host) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c || !st) return TRD_ERR_INVALID_ARG;
  if (c->sticky) return c->sticky;
  const int64_t In = c->dims[c->N - 1];
  if (st->sweep < 0 || (st->have_prev_D != 0 && st->have_prev_D != 1)) return TRD_ERR_INVALID_ARG;
  if (c->cfg.sigma_mode != TRD_SIGMA_INF && !(st->sigma > 0.0 && std::isfinite(st->sigma))) return TRD_ERR_INVALID_ARG;
  if (st->have_prev_D && (!prev_D_host || st->prev_D_size != In * In)) return TRD_ERR_INVALID_ARG;
  // the fields live in DevScalars: write them in place on the context stream
  CUDA_TRY(c, cudaMemcpyAsync(&c->sc->sigma, &st->sigma, 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&c->sc->sweep, &st->sweep, 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&c->sc->have_prev_D, &st->have_prev_D, 4, cudaMemcpyHostToDevice, c->stream));
  if (st->have_prev_D)
    CUDA_TRY(c, cudaMemcpyAsync(c->Dprev, prev_D_host, (size_t)(In * In) * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TRD_OK;
}

void trd_destroy(trd_ctx* ctx) {
  Context* c = reinterpret_cast<Context*>(ctx);
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->tl_on && !c->tl.empty()) {          // TRD_TIMELINE report: mean us between marks, per stream
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->side);
    std::vector<std::string> names;
    std::vector<double> sum;
    std::vector<int> cnt;
    for (int strm = 0; strm < 2; ++strm) {
      int prev = -1;
      for (size_t i = 0; i < c->tl.size(); ++i) {
        if (c->tl[i].side != strm) continue;
        if (prev >= 0 && strcmp(c->tl[i].label, "block start") != 0 && strcmp(c->tl[i].label, "side: fork") != 0) {
          float ms = 0.f;
          cudaEventElapsedTime(&ms, (cudaEvent_t)c->tl[(size_t)prev].ev, (cudaEvent_t)c->tl[i].ev);
          size_t j = 0;
          for (; j < names.size(); ++j) if (names[j] == c->tl[i].label) break;
          if (j == names.size()) { names.push_back(c->tl[i].label); sum.push_back(0.0); cnt.push_back(0); }
          sum[j] += ms * 1e3;
          cnt[j] += 1;
        }
        prev = (int)i;
      }
    }
    fprintf(stderr, "[trd timeline] mean us per occurrence (main stream, then side stream)\n");
    for (size_t j = 0; j < names.size(); ++j)
      fprintf(stderr, "  %-28s %9.1f  (x%d)\n", names[j].c_str(), sum[j] / cnt[j], cnt[j]);
    for (auto& t : c->tl) cudaEventDestroy((cudaEvent_t)t.ev);
  }
  if (c->side) cudaStreamSynchronize(c->side);
  big_destroy(c);
  for (auto& g : c->graphs) destroy_graph(g);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->nccl_comm && g_nccl.comm_destroy) g_nccl.comm_destroy(c->nccl_comm);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->side) { cudaStreamSynchronize(c->side); cudaStreamDestroy(c->side); }
  if (c->copy) { cudaStreamSynchronize(c->copy); cudaStreamDestroy(c->copy); }
  for (int b = 0; b < 2; ++b)
    if (c->ev_up_ready[b]) cudaEventDestroy(c->ev_up_ready[b]);
  if (c->ev_up_free) cudaEventDestroy(c->ev_up_free);
  // own_values / own_mask point at one of the two sets: free both sets once
  if (c->up_values[0]) {
    for (int b = 0; b < 2; ++b) {
      if (c->up_values[b]) cudaFree(c->up_values[b]);
      if (c->up_mask[b]) cudaFree(c->up_mask[b]);
    }
    c->own_values = nullptr;
    c->own_mask = nullptr;
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->stg) { cudaStreamSynchronize(c->stg); cudaStreamDestroy(c->stg); }
  if (c->ev_stg_fork) cudaEventDestroy(c->ev_stg_fork);
  for (int k = 0; k < kMaxN; ++k) {
    cudaEvent_t ev[] = {c->ev_p1[k], c->ev_p2[k], c->ev_samp[k], c->ev_staged[k]};
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    void* bp[] = {c->idx_b[k], c->doff_b[k], c->row_off_b[k], c->col_off_b[k], c->ptab_b[k]};
    for (void* p : bp)
      if (p) cudaFree(p);
  }
  if (c->pipe) select_bufs(c, -1);         // (the current pointers may be a block's buffers)
  void* ptrs[] = {c->own_values, c->own_mask, c->rank_prefix, c->Z, c->Q, c->idx, c->doff,
                  c->row_off, c->col_off, c->mid, c->lft, c->lfth, c->rgtT, c->dpart, c->spart,
                  c->denpart, c->numpart, c->dvec, c->G, c->G_last, c->Mop, c->chol_ws,
                  c->chain_ws, c->h, c->Dcur, c->Dprev, c->sc, c->stats, c->red_ws,
                  c->lftHL, c->lfthHL, c->lscl, c->lsclh, c->rgtHL, c->rgtHL2, c->contrib, c->Qloc, c->Gloc, c->mhist,
                  c->eabs, c->chk, c->chk_acc, c->stage_mask, c->ptab, c->rgtC};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->tw) cudaFree(c->tw);
  if (c->rp_tmp) cudaFree(c->rp_tmp);
  if (getenv("TRD_TC_EXP")) tc_debug_dump();
  for (int k = 0; k < kMaxN; ++k) {
    TcStage& sg = c->stage[k];
    void* sp[] = {sg.tbits, sg.troff, sg.tcount, sg.tbase, sg.tvals, sg.tidx, sg.scan_tmp, sg.perm};
    for (void* p : sp)
      if (p) cudaFree(p);
  }
  delete c;
}

}  // extern "C"

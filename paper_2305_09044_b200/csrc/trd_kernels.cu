// trd_kernels.cu -- device kernels of libtrd (sm_100a).
//
// Paper citations "P:L" are PAPER.md lines.  The block pipeline (one cyclic block k of
// Alg. 1) is:
//   sampler (Alg.1 l.4)  -> plan/offsets + chain products (Thm 1 subchain split)
//   -> pass 1: residual, HQ weight, gradient partials (Eq. 7, Eq. 9/15)
//   -> reduce_d -> [NCCL allreduce] -> FGMC Gram (Eq. 13) -> filtered solve (Eq. 10/16)
//   -> h = d M -> pass 2: line-search denominator (Eq. 12/18) -> [allreduce]
//   -> update Z_k (Eq. 11/17, sign reading R2) -> refresh Q_k (Alg. 1 l.10)
#include <cub/cub.cuh>
#include <math.h>

#include "trd_internal.cuh"

namespace trd {

#define CK(x) do { cudaError_t e__ = (x); (void)e__; } while (0)

// ----------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. 2011) -- reading R11.  Independent of oracle/philox.py.
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
}

// One CTA per mode m: writes the index set I_m of (sweep t, block k) and the data offsets.
// Selection = the s_m smallest (kappa_i, i), output ascending (reading R11).  The key kappa_K
// of rank s_m - 1 is found by an 8-pass radix select over the 64-bit keys (8 bits per pass,
// per-CTA shared-memory histograms; the keys are recomputed, nothing of size I is stored), then
// one ascending pass over i keeps kappa_i < kappa_K and the first (in i) of the keys equal to
// kappa_K up to rank s_m - 1: O(I) work, no limit on I_m.
struct SamplerArgs {
  int N, k, shard_mode;
  uint64_t seed;
  int64_t shard_begin, shard_end;
  int64_t dims[kMaxN], s[kMaxN], idx_off[kMaxN + 1], lstride[kMaxN];
  int shard_local;       // shard mode enumerates [shard_begin, shard_end) (full set)
  int shard_sampled;     // shard mode: this rank's sampled indices, compacted, capacity s[m]
  int64_t s_samp[kMaxN]; // RStS sample sizes (the draw; s[m] may be a smaller capacity)
  uint8_t* ptab;         // non-null: also write the staging's compaction tables of mode 0's
                         // sampled positions (byte b of a fibre window, value v -> the sampled
                         // bits packed at ptab[b * 256 + v]; positions below byte b at ptab[4096 + b])
};

constexpr int kSamplerThreads = 256;
constexpr int kSamplerSmall = 1024;      // index sets up to this size: comparison ranks
__device__ __forceinline__ unsigned long long sample_key(uint64_t seed, int64_t i, int m, int k, uint32_t t) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)m, (uint32_t)k, t};
  philox10(c, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  return ((unsigned long long)c[0] << 32) | c[1];
}

__global__ void __launch_bounds__(kSamplerThreads)
sampler_kernel(SamplerArgs sa, const DevScalars* __restrict__ sc, int32_t* __restrict__ idx,
               int64_t* __restrict__ doff) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  using Scan = cub::BlockScan<long long, kSamplerThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ unsigned int hist[256];
  __shared__ int sel_bin;
  __shared__ long long rank_s;
  const int m = blockIdx.x, tid = threadIdx.x;
  const int k = sa.k;
  const uint64_t seed = sa.seed;
  const int64_t I = sa.dims[m];
  const int64_t s = sa.s[m] <= 0 ? I : sa.s[m];
  const int64_t s_draw = sa.s_samp[m] <= 0 ? I : sa.s_samp[m];      // selection size of the draw
  const bool compact = m == sa.shard_mode && sa.shard_sampled;
  int32_t* out = idx + sa.idx_off[m];
  int64_t* dof = doff + sa.idx_off[m];
  const uint32_t t = (uint32_t)sc->sweep;
  int64_t n_local = s;                                                // (compacted lists)
  if (m == sa.shard_mode && sa.shard_local) {               // this rank's slice, global indices
    for (int64_t q = tid; q < s; q += blockDim.x) out[q] = (int32_t)(sa.shard_begin + q);
  } else if (s_draw >= I && !compact) {
    for (int64_t i = tid; i < I; i += blockDim.x) out[i] = (int32_t)i;
  } else if (I <= kSamplerSmall) {
    // small sets: keys in shared memory, rank of each key by counting (ties broken by i)
    __shared__ unsigned long long keys[kSamplerSmall];
    __shared__ unsigned char sel[kSamplerSmall];
    for (int64_t i = tid; i < I; i += blockDim.x) keys[i] = sample_key(seed, i, m, k, t);
    __syncthreads();
    for (int64_t i = tid; i < I; i += blockDim.x) {
      const unsigned long long ki = keys[i];
      int64_t rank = 0;
      for (int64_t j = 0; j < I; ++j) {
        const unsigned long long kj = keys[j];
        rank += (kj < ki) || (kj == ki && j < i);
      }
      sel[i] = rank < s_draw && (!compact || (i >= sa.shard_begin && i < sa.shard_end));
    }
    __syncthreads();
    long long n_out = 0;
    for (int64_t c0 = 0; c0 < I; c0 += blockDim.x) {       // ascending compaction
      const int64_t i = c0 + tid;
      const bool put = i < I && sel[i];
      long long pos, put_tot;
      Scan(scan_tmp).ExclusiveSum(put ? 1ll : 0ll, pos, put_tot);
      __syncthreads();
      if (put) out[n_out + pos] = (int32_t)i;
      n_out += put_tot;
    }
    n_local = compact ? n_out : s;
    TRD_CHECK(compact || n_out == s_draw, kChkSampler);
    for (int64_t q = n_local + tid; q < s; q += blockDim.x) out[q] = (int32_t)sa.shard_begin;   // padding
  } else {
    // radix select of the key of rank s_draw - 1
    unsigned long long prefix = 0ull, pmask = 0ull;
    if (tid == 0) rank_s = (long long)s_draw - 1;
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
      for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0u;
      __syncthreads();
      for (int64_t i = tid; i < I; i += blockDim.x) {
        const unsigned long long key = sample_key(seed, i, m, k, t);
        if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        long long cum = 0, r = rank_s;
        int b = 0;
        for (; b < 255; ++b) {
          if (cum + (long long)hist[b] > r) break;
          cum += hist[b];
        }
        sel_bin = b;
        rank_s = r - cum;
      }
      __syncthreads();
      prefix |= (unsigned long long)sel_bin << shift;
      pmask |= 0xFFull << shift;
    }
    // keys equal to kappa_K: keep the first rank_s + 1 of them in ascending i
    const long long take_eq = rank_s + 1;
    long long eq_seen = 0, n_out = 0;      // running totals over the previous chunks
    __syncthreads();
    for (int64_t c0 = 0; c0 < I; c0 += blockDim.x) {
      const int64_t i = c0 + tid;
      unsigned long long key = ~0ull;
      if (i < I) key = sample_key(seed, i, m, k, t);
      const bool eq = i < I && key == prefix;
      long long eq_ex, eq_tot;
      Scan(scan_tmp).ExclusiveSum(eq ? 1ll : 0ll, eq_ex, eq_tot);
      __syncthreads();
      const bool sel = i < I && (key < prefix || (eq && eq_seen + eq_ex < take_eq));
      const bool put = sel && (!compact || (i >= sa.shard_begin && i < sa.shard_end));
      long long pos, put_tot;
      Scan(scan_tmp).ExclusiveSum(put ? 1ll : 0ll, pos, put_tot);
      __syncthreads();
      if (put) out[n_out + pos] = (int32_t)i;
      eq_seen += eq_tot;
      n_out += put_tot;
    }
    n_local = compact ? n_out : s;
    TRD_CHECK(compact || n_out == s_draw, kChkSampler);     // exactly s_draw selected
    for (int64_t q = n_local + tid; q < s; q += blockDim.x) out[q] = (int32_t)sa.shard_begin;   // padding
  }
  __syncthreads();
  if (m == 0 && sa.ptab) {                  // (s <= 64, I <= 128: the window bytes b < 16)
    __shared__ uint32_t pm[16], pb[16];
    if (tid < 16) {
      uint32_t msk = 0, below = 0;
      for (int64_t q = 0; q < s; ++q) {
        const int p = out[q];
        if ((p >> 3) == tid) msk |= 1u << (p & 7);
        else if (p < 8 * tid) ++below;
      }
      pm[tid] = msk;
      pb[tid] = below;
    }
    __syncthreads();
    for (int b = 0; b < 16; ++b) {
      const uint32_t msk = pm[b];
      uint32_t r = 0;
      int qq = 0;
      for (int t2 = 0; t2 < 8; ++t2)
        if ((msk >> t2) & 1u) { r |= (((uint32_t)tid >> t2) & 1u) << qq; ++qq; }
      sa.ptab[b * 256 + tid] = (uint8_t)r;
    }
    if (tid < 16) sa.ptab[4096 + tid] = (uint8_t)pb[tid];
  }
  const int64_t cnt = s >= I ? I : s;
  for (int64_t q = tid; q < cnt; q += blockDim.x) {
    int64_t g = out[q];
    // checked build: a real entry lies in [0, I) and the set is strictly ascending
    TRD_CHECK(q >= n_local || (g >= 0 && g < I && (q == 0 || g > (int64_t)out[q - 1])), kChkSampler);
    int64_t loc = g;
    if (m == sa.shard_mode) loc = (g >= sa.shard_begin && g < sa.shard_end) ? g - sa.shard_begin : -1;
    if (q >= n_local) loc = -1;                                       // padding of a compacted list
    dof[q] = loc < 0 ? -1 : loc * sa.lstride[m];
  }
}

// 'Uniform row sampling' arm (reading R22): draw q of block k, sweep t is row
// rho = floor(kappa R / 2^64) of X_[k] (kappa from Philox(seed, (q, ROWS, k, t)), R = prod_{m!=k}
// I_m), decoded with i_{k+1} fastest into entry q of every mode's list; mode k: all indices
__device__ __forceinline__ void row_put(const SamplerArgs& sa, int m, int64_t q, int64_t g, int32_t* idx,
                                        int64_t* doff) {
  idx[sa.idx_off[m] + q] = (int32_t)g;
  int64_t loc = g;
  if (m == sa.shard_mode) loc = (g >= sa.shard_begin && g < sa.shard_end) ? g - sa.shard_begin : -1;
  doff[sa.idx_off[m] + q] = loc < 0 ? -1 : loc * sa.lstride[m];
}
__global__ void row_sampler_kernel(SamplerArgs sa, int64_t J, const DevScalars* __restrict__ sc,
                                   int32_t* __restrict__ idx, int64_t* __restrict__ doff) {
  const int N = sa.N, k = sa.k;
  const uint32_t t = (uint32_t)sc->sweep;
  uint64_t R = 1;
  for (int q = 1; q < N; ++q) R *= (uint64_t)sa.dims[(k + q) % N];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < J + sa.dims[k];
       q += (int64_t)gridDim.x * blockDim.x) {
    if (q >= J) { row_put(sa, k, q - J, q - J, idx, doff); continue; }
    uint32_t c[4] = {(uint32_t)q, 0x524F5753u, (uint32_t)k, t};
    philox10(c, (uint32_t)(sa.seed & 0xffffffffu), (uint32_t)(sa.seed >> 32));
    const uint64_t kappa = ((uint64_t)c[0] << 32) | c[1];
    uint64_t rho = __umul64hi(kappa, R);
    for (int d = 1; d < N; ++d) {
      const int m = (k + d) % N;
      row_put(sa, m, q, (int64_t)(rho % (uint64_t)sa.dims[m]), idx, doff);
      rho /= (uint64_t)sa.dims[m];
    }
  }
}

// ----------------------------------------------------------------------------------------
// Plan kernels: row/col data offsets and the chain products Mid, Lft, Rgt (Thm 1 subchain,
// P:63-66; Def. 2 merging).  Slice of core m at index i: Z + zoff[m] + i*r_m*r_{m+1}.
// ----------------------------------------------------------------------------------------
struct PlanArgs {
  int N, k, p, nleft, nright;
  int left[kMaxN], right[kMaxN];
  int ldig[kMaxN], rdig[kMaxN];        // digit order (fastest first) as indices into left/right
  int rowmode;                         // 0: row = jl + nL*ik ; 1: row = ik + Ik*jl
  int explicit_cols;                   // row sampling (R22): column col = draw col in every list
  int64_t ik0;                         // global i_k of plan row index 0 (k = shard mode)
  int64_t sL[kMaxN], sR[kMaxN];        // sizes of the left/right index sets
  int64_t offL[kMaxN], offR[kMaxN];    // offsets into idx/doff
  int64_t off_k;
  int64_t nL, nrows, ncols, Ik;
  int rk, rk1, rs, K;
  int rank_of[kMaxN + 1];
  int64_t zoff[kMaxN + 1];
};

static PlanArgs make_plan_args(const Context& c, const BlockPlan& bp) {
  PlanArgs a;
  a.N = c.N; a.k = bp.k; a.p = bp.p; a.nleft = bp.nleft; a.nright = bp.nright;
  for (int q = 0; q < bp.nleft; ++q) {
    a.left[q] = bp.left[q]; a.sL[q] = bp.s[bp.left[q]]; a.offL[q] = c.idx_off[bp.left[q]];
    a.ldig[q] = bp.ldig[q];
  }
  for (int q = 0; q < bp.nright; ++q) {
    a.right[q] = bp.right[q]; a.sR[q] = bp.s[bp.right[q]]; a.offR[q] = c.idx_off[bp.right[q]];
    a.rdig[q] = bp.rdig[q];
  }
  a.rowmode = bp.rowmode;
  a.explicit_cols = bp.explicit_cols;
  a.ik0 = bp.ik0;
  a.off_k = c.idx_off[bp.k];
  a.nL = bp.nL; a.nrows = bp.nrows; a.ncols = bp.ncols; a.Ik = bp.nrows / bp.nL;
  a.rk = bp.rk; a.rk1 = bp.rk1; a.rs = bp.rs; a.K = bp.K;
  for (int m = 0; m <= c.N; ++m) a.rank_of[m] = c.ranks[m % c.N];
  for (int m = 0; m <= c.N; ++m) a.zoff[m] = c.zoff[m];
  return a;
}

// row <-> (ik, jl) and mixed-radix digits of jl / col (per ring position q)
__device__ __forceinline__ void row_split(const PlanArgs& a, int64_t row, int64_t& ik, int64_t& jl) {
  if (a.rowmode == 0) { jl = row % a.nL; ik = row / a.nL; }
  else { ik = row % a.Ik; jl = row / a.Ik; }
}
__device__ __forceinline__ void left_digits(const PlanArgs& a, int64_t jl, int64_t* dq) {
  for (int d = 0; d < a.nleft; ++d) {
    const int q = a.ldig[d];
    dq[q] = jl % a.sL[q];
    jl /= a.sL[q];
  }
}
__device__ __forceinline__ void right_digits(const PlanArgs& a, int64_t col, int64_t* dq) {
  if (a.explicit_cols) {                     // draw col: entry col of every right mode's list
    for (int d = 0; d < a.nright; ++d) dq[d] = col;
    return;
  }
  for (int d = 0; d < a.nright; ++d) {
    const int q = a.rdig[d];
    dq[q] = col % a.sR[q];
    col /= a.sR[q];
  }
}

__global__ void offsets_kernel(PlanArgs a, const int64_t* __restrict__ doff,
                               int64_t* __restrict__ row_off, int64_t* __restrict__ col_off,
                               DevScalars* __restrict__ sc) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  // (operand scaling; sc = nullptr when the offsets run ahead on the staging stream)
  if (sc && blockIdx.x == 0 && threadIdx.x == 0) { sc->amax_a = 0u; sc->amax_b = 0u; }
  const int64_t tot = a.nrows + a.ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t dq[kMaxN];
    if (t < a.nrows) {
      int64_t ik, jl;
      row_split(a, t, ik, jl);
      left_digits(a, jl, dq);
      int64_t o = doff[a.off_k + ik];
      bool bad = o < 0;
      for (int q = 0; q < a.nleft; ++q) {
        int64_t v = doff[a.offL[q] + dq[q]];
        bad |= v < 0;
        o += v;
      }
      row_off[t] = bad ? -1 : o;
    } else {
      const int64_t col = t - a.nrows;
      right_digits(a, col, dq);
      int64_t o = 0;
      bool bad = false;
      for (int q = 0; q < a.nright; ++q) {
        int64_t v = doff[a.offR[q] + dq[q]];
        bad |= v < 0;
        o += v;
      }
      col_off[col] = bad ? -1 : o;
    }
  }
}

// v (row vector, length r_in) <- v * Z_m(i)  (r_in x r_out slice); RM = the rank bucket
// (16 or 32, >= every rank of the context: register arrays of compile-time size)
template <int RM>
__device__ __forceinline__ void vecmat(float* v, const float* __restrict__ Zs, int rin, int rout) {
  if (RM > 32) {                     // large-rank bucket: runtime loop bounds (the arrays live in
    float nv[RM];                    // local memory; a fully unrolled predicated RM-loop would
    for (int c = 0; c < rout; ++c) nv[c] = 0.f;   // issue RM FMAs per input for any r_out)
    for (int a = 0; a < rin; ++a) {
      const float va = v[a];
      const float* row = Zs + a * rout;
      for (int c = 0; c < rout; ++c) nv[c] = fmaf(va, __ldg(row + c), nv[c]);
    }
    for (int c = 0; c < rout; ++c) v[c] = nv[c];
    for (int c = rout; c < RM; ++c) v[c] = 0.f;
    return;
  }
  float nv[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) nv[c] = 0.f;
  for (int a = 0; a < rin; ++a) {
    const float va = v[a];
    const float* row = Zs + a * rout;
#pragma unroll
    for (int c = 0; c < RM; ++c)
      if (c < rout) nv[c] = fmaf(va, __ldg(row + c), nv[c]);
  }
#pragma unroll
  for (int c = 0; c < RM; ++c) v[c] = nv[c];
}

// Mid(j_L)[b][c] = (Z_{k+1}(.) .. Z_{k+p}(.))[b][c]   (r_{k+1} x r_s), one thread per (jl, b)
template <int RM>
__global__ void mid_kernel(PlanArgs a, const int32_t* __restrict__ idx, const float* __restrict__ Z,
                           float* __restrict__ mid) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  const int64_t tot = a.nL * a.rk1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(t % a.rk1);
    int64_t jl = t / a.rk1;
    int64_t dq[kMaxN];
    left_digits(a, jl, dq);
    float v[RM];
    int rin = a.rk1, q0 = 0;
    if (RM > 32 && a.nleft > 0) {            // large ranks: e_b Z(i) is row b of the first slice
      const int m = a.left[0];
      const int rout = a.rank_of[m + 1];
      const float* zr = Z + a.zoff[m] + (int64_t)idx[a.offL[0] + dq[0]] * a.rank_of[m] * rout + (int64_t)b * rout;
      for (int c = 0; c < rout; ++c) v[c] = __ldg(zr + c);
      for (int c = rout; c < RM; ++c) v[c] = 0.f;
      rin = rout;
      q0 = 1;
    } else {
#pragma unroll
      for (int c = 0; c < RM; ++c) v[c] = (c == b) ? 1.f : 0.f;
    }
    for (int q = q0; q < a.nleft; ++q) {
      int m = a.left[q];
      int64_t i = idx[a.offL[q] + dq[q]];
      int rout = a.rank_of[m + 1];
      vecmat<RM>(v, Z + a.zoff[m] + i * (int64_t)a.rank_of[m] * rout, rin, rout);
      rin = rout;
    }
    float* o = mid + (jl * a.rk1 + b) * a.rs;
    for (int c = 0; c < a.rs; ++c) o[c] = v[c];
  }
}

// Rgt(j_R) = Z_{k+p+1}(.) .. Z_{k-1}(.)  (r_s x r_k); stored RgtT[(a + r_k c) * ncols + col]
// = Rgt[c][a].  One thread per (col, c); the r_s threads of a column are adjacent so that
// their slice reads coincide (columns of explicit draws hit unrelated slices)
__device__ __forceinline__ void block_amax(float v, unsigned int* dst) {
  // max |v| over the CTA -> atomicMax on the fp32 bit pattern (v >= 0)
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
    amax_update(dst, m);
  }
}

template <int RM>
__global__ void rgt_kernel(PlanArgs a, const int32_t* __restrict__ idx, const float* __restrict__ Z,
                           float* __restrict__ rgtT, DevScalars* __restrict__ sc) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  float amax = 0.f;
  const int64_t tot = a.ncols * a.rs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t col = t / a.rs;
    int cc = (int)(t % a.rs);
    int64_t dq[kMaxN];
    right_digits(a, col, dq);
    float v[RM];
    int rin = a.rs, q0 = 0;
    if (RM > 32 && a.nright > 0) {           // large ranks: e_cc Z(i) is row cc of the first slice
      const int m = a.right[0];
      const int rout = a.rank_of[m + 1];
      const float* zr = Z + a.zoff[m] + (int64_t)idx[a.offR[0] + dq[0]] * a.rank_of[m] * rout + (int64_t)cc * rout;
      for (int c = 0; c < rout; ++c) v[c] = __ldg(zr + c);
      for (int c = rout; c < RM; ++c) v[c] = 0.f;
      rin = rout;
      q0 = 1;
    } else {
#pragma unroll
      for (int c = 0; c < RM; ++c) v[c] = (c == cc) ? 1.f : 0.f;
    }
    for (int q = q0; q < a.nright; ++q) {
      int m = a.right[q];
      int64_t i = idx[a.offR[q] + dq[q]];
      int rout = a.rank_of[m + 1];
      vecmat<RM>(v, Z + a.zoff[m] + i * (int64_t)a.rank_of[m] * rout, rin, rout);
      rin = rout;
    }
    for (int aa = 0; aa < a.rk; ++aa) {
      rgtT[(int64_t)(aa + a.rk * cc) * a.ncols + col] = v[aa];
      amax = fmaxf(amax, fabsf(v[aa]));
    }
  }
  block_amax(amax, &sc->amax_b);     // (B operand scaling of the tensor-core passes)
}

// Warp-per-index chain products (ranks <= 32): one warp forms the whole r_first x r_last product
// Z_{m_0}(i_0) Z_{m_1}(i_1) .. of one column (Rgt) or left index (Mid) in shared memory, lane-parallel
// over the output entries, instead of one thread per output row walking the chain through register
// vectors (the thread-per-row kernels above: ~15 us per C4 block for a few MFLOP, latency bound,
// with one CTA per 32 rows).  Same fp32 arithmetic and order: the first factor is the slice itself
// (the thread kernels' one-hot start multiplies by exact 0 / 1), every further product is an fmaf
// sum over the inner index ascending from 0.  Returns the product's column count; A holds it.
template <int RM>
__device__ __forceinline__ int warp_chain(const PlanArgs& a, const int32_t* __restrict__ idx, const float* __restrict__ Z,
                                          const int* modes, const int64_t* offs, const int64_t* dq, int nm, int rows,
                                          float*& A, float*& Bn, int lane) {
  int rc;
  if (nm == 0) {                                   // empty chain: the identity (rows x rows)
    rc = rows;
    for (int o = lane; o < rows * rc; o += 32) A[o] = (o / rc == o % rc) ? 1.f : 0.f;
  } else {
    const int m = modes[0];
    rc = a.rank_of[m + 1];
    const float* zs = Z + a.zoff[m] + (int64_t)idx[offs[0] + dq[0]] * a.rank_of[m] * rc;
    for (int o = lane; o < rows * rc; o += 32) A[o] = __ldg(zs + o);
  }
  __syncwarp();
  for (int q = 1; q < nm; ++q) {
    const int m = modes[q];
    const int rin = rc, rout = a.rank_of[m + 1];
    const float* zs = Z + a.zoff[m] + (int64_t)idx[offs[q] + dq[q]] * a.rank_of[m] * rout;
    for (int o = lane; o < rows * rout; o += 32) {
      const int r = o / rout, c = o - r * rout;
      float acc = 0.f;
      for (int b = 0; b < rin; ++b) acc = fmaf(A[r * rin + b], __ldg(zs + b * rout + c), acc);
      Bn[o] = acc;
    }
    __syncwarp();
    float* t = A; A = Bn; Bn = t;
    rc = rout;
  }
  return rc;
}

// Rgt(col)[cc][aa] (r_s x r_k) -> RgtT[(aa + r_k cc) ncols + col], warp per column
template <int RM, int WPC>
__global__ void __launch_bounds__(32 * WPC) rgt_warp_kernel(PlanArgs a, const int32_t* __restrict__ idx, const float* __restrict__ Z,
                                                          float* __restrict__ rgtT, DevScalars* __restrict__ sc) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  __shared__ float buf[WPC][2][RM * RM];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float amax = 0.f;
  for (int64_t col = (int64_t)blockIdx.x * WPC + warp; col < a.ncols; col += (int64_t)gridDim.x * WPC) {
    int64_t dq[kMaxN];
    right_digits(a, col, dq);
    float* A = buf[warp][0];
    float* Bn = buf[warp][1];
    const int rc = warp_chain<RM>(a, idx, Z, a.right, a.offR, dq, a.nright, a.rs, A, Bn, lane);
    for (int o = lane; o < a.rs * rc; o += 32) {
      const int cc = o / rc, aa = o - cc * rc;
      const float v = A[o];
      rgtT[(int64_t)(aa + a.rk * cc) * a.ncols + col] = v;
      amax = fmaxf(amax, fabsf(v));
    }
    __syncwarp();                                  // (the next column reuses the buffers)
  }
  block_amax(amax, &sc->amax_b);     // (B operand scaling of the tensor-core passes)
}

// Mid(jl)[b][c] (r_{k+1} x r_s) -> mid[(jl r_{k+1} + b) r_s + c], warp per left index
template <int RM, int WPC>
__global__ void __launch_bounds__(32 * WPC) mid_warp_kernel(PlanArgs a, const int32_t* __restrict__ idx, const float* __restrict__ Z,
                                                          float* __restrict__ mid) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  __shared__ float buf[WPC][2][RM * RM];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t jl = (int64_t)blockIdx.x * WPC + warp; jl < a.nL; jl += (int64_t)gridDim.x * WPC) {
    int64_t dq[kMaxN];
    left_digits(a, jl, dq);
    float* A = buf[warp][0];
    float* Bn = buf[warp][1];
    const int rc = warp_chain<RM>(a, idx, Z, a.left, a.offL, dq, a.nleft, a.rk1, A, Bn, lane);
    for (int o = lane; o < a.rk1 * rc; o += 32) mid[jl * a.rk1 * a.rs + o] = A[o];
    __syncwarp();
  }
}

// Lft(row)[a + r_k c] = (X_k(i_k) Mid(j_L))[a][c] where X_k is the core slice (pass 1) or
// the folded scaled gradient H(i_k)[a][b] = h[i_k][a + r_k b] (pass 2).  Thread per (row, a).
template <int RM>
__global__ void lft_kernel(PlanArgs a, const float* __restrict__ Zk, const double* __restrict__ h,
                           const float* __restrict__ mid, float* __restrict__ lft) {
  const int64_t tot = a.nrows * a.rk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    int aa = (int)(t % a.rk);
    int64_t row = t / a.rk;
    int64_t jl, ik;
    row_split(a, row, ik, jl);
    float v[RM];
#pragma unroll
    for (int b = 0; b < RM; ++b) {
      if (b < a.rk1) {
        v[b] = h ? (float)h[(a.ik0 + ik) * a.rk * a.rk1 + aa + a.rk * b]
                 : __ldg(Zk + ((a.ik0 + ik) * a.rk + aa) * a.rk1 + b);
      } else {
        v[b] = 0.f;
      }
    }
    float* o = lft + row * a.K;
    if (a.p == 0) {
      for (int c = 0; c < a.rk1; ++c) o[aa + a.rk * c] = v[c];
    } else {
      vecmat<RM>(v, mid + jl * a.rk1 * a.rs, a.rk1, a.rs);
      for (int c = 0; c < a.rs; ++c) o[aa + a.rk * c] = v[c];
    }
  }
}

// ----------------------------------------------------------------------------------------
// Pass kernels (v1, SIMT).  CTA = (jl chunk, i_k, column split); warp = one GEMM row and a
// column sub-range; lane = one column per 32-column chunk.  Only observed entries
// contribute (P mask); the working set is the sketch (Eq. 14-15).
// ----------------------------------------------------------------------------------------
struct PassArgs {
  int64_t nL, nrows, ncols;
  int K, R2, rk, rk1, rs, p;
  int jl_per_cta, ws_split, nsplit;
  int sigma_inf, packed;
  int rowmode;
  int64_t Ik;
  const int64_t* row_off;
  const int64_t* col_off;
  const float* lft;
  const float* lfth;
  const float* rgtT;
  const float* mid;
  const float* values;
  const uint32_t* mask;
  const uint32_t* rank_prefix;
  const DevScalars* sc;
  double* dpart;      // [ik][cta][R2]
  double* spart;      // [ik][cta][3]
  double* denpart;    // [ik][cta]
  uint32_t* eabs;     // TRD_SIGMA_MAD: |e| bit patterns of pass 1 (R21), else nullptr
  unsigned long long* efill;   // its fill counter (warp-aggregated atomics)
  unsigned long long ecap;
  float* contrib;     // large-rank path (R2M == 0): D rows [split][row][KP] (ws_split == 1)
  int KP;
};

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool load_entry(const PassArgs& a, int64_t ro, int64_t co, float& x) {
  if (co < 0) return false;
  const int64_t lin = ro + co;
  const uint32_t word = __ldg(a.mask + (lin >> 5));
  const uint32_t bit = (uint32_t)(lin & 31);
  if (!((word >> bit) & 1u)) return false;
  int64_t vi = lin;
  if (a.packed) vi = (int64_t)__ldg(a.rank_prefix + (lin >> 5)) + __popc(word & ((1u << bit) - 1u));
  x = __ldg(a.values + vi);
  return true;
}

constexpr int kPassThreads = 256;
constexpr int kPassWarps = kPassThreads / 32;

template <int KT, int R2M, bool PASS2, bool STATS_ONLY>
__global__ void __launch_bounds__(kPassThreads)
pass_kernel(PassArgs a) {
  __shared__ float lftS[kPassWarps][KT];
  __shared__ float lfhS[kPassWarps][PASS2 ? KT : 1];
  __shared__ float dS[kPassWarps][KT];
  constexpr int RCH = 256;                 // R^2 chunk of the CTA reduction
  __shared__ double redS[kPassWarps][RCH + 3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ik = blockIdx.y;
  const int64_t jl0 = (int64_t)blockIdx.x * a.jl_per_cta;
  const int jlc = (int)min((int64_t)a.jl_per_cta, a.nL - jl0);
  const int nitems = jlc * a.ws_split;
  // column range of this CTA's split
  const int64_t per_split = (a.ncols + a.nsplit - 1) / a.nsplit;
  const int64_t cb0 = (int64_t)blockIdx.z * per_split;
  const int64_t ce0 = min(a.ncols, cb0 + per_split);
  const int64_t per_sub = (ce0 - cb0 + a.ws_split - 1) / a.ws_split;

  const double sigma = a.sc->sigma;
  const float inv2s2 = a.sigma_inf ? 0.f : (float)(0.5 / (sigma * sigma));
  const double s2 = sigma * sigma;

  double st_e2 = 0.0, st_w = 0.0, st_n = 0.0, st_den = 0.0;
  // R2M == 0 (large-rank path, R^2 > kBigR2): the warp's D row (K floats) goes to contrib and
  // reduce_d_big_kernel contracts it with Mid; the plan has ws_split == 1 (one warp per row)
  constexpr bool WD = R2M == 0;
  constexpr int OUTS = WD ? 1 : R2M / 32;
  double outacc[OUTS];
#pragma unroll
  for (int q = 0; q < OUTS; ++q) outacc[q] = 0.0;

  for (int item = warp; item < nitems; item += kPassWarps) {
    const int64_t jl = jl0 + item / a.ws_split;
    const int sub = item % a.ws_split;
    const int64_t row = a.rowmode == 0 ? jl + a.nL * ik : ik + a.Ik * jl;
    const int64_t ro = a.row_off[row];
    if (ro < 0) {
      if (WD && !PASS2 && !STATS_ONLY)         // (a row outside the shard: zero D row)
        for (int q = lane; q < a.K; q += 32) a.contrib[((int64_t)blockIdx.z * a.nrows + row) * a.KP + q] = 0.f;
      continue;
    }
    for (int q = lane; q < a.K; q += 32) {
      lftS[warp][q] = a.lft[row * a.K + q];
      if (PASS2) lfhS[warp][q] = a.lfth[row * a.K + q];
    }
    __syncwarp();
    const int64_t cb = cb0 + sub * per_sub;
    const int64_t ce = min(ce0, cb + per_sub);
    float dacc[KT];
#pragma unroll
    for (int q = 0; q < KT; ++q) dacc[q] = 0.f;
    for (int64_t c0 = cb; c0 < ce; c0 += 32) {
      const int64_t col = c0 + lane;
      float x = 0.f;
      const bool obs = (col < ce) && load_entry(a, ro, a.col_off[min(col, a.ncols - 1)], x);
      if (!__any_sync(0xffffffffu, obs)) continue;
      const float* rc = a.rgtT + min(col, a.ncols - 1);
      float recon = 0.f, tdir = 0.f;
#pragma unroll
      for (int q = 0; q < KT; ++q) {
        if (q < a.K) {
          const float r = __ldg(rc + (int64_t)q * a.ncols);
          recon = fmaf(lftS[warp][q], r, recon);
          if (PASS2) tdir = fmaf(lfhS[warp][q], r, tdir);
        }
      }
      const float e = x - recon;
      const float w = a.sigma_inf ? 1.f : expf(-e * e * inv2s2);
      if (!PASS2 && a.eabs) {                // R21: |e| of the observed entries, any order
        const unsigned bal = __ballot_sync(0xffffffffu, obs);
        unsigned long long base = 0ull;
        if (lane == 0) base = atomicAdd(a.efill, (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned long long q = base + __popc(bal & ((1u << lane) - 1u));
        if (obs && q < a.ecap) a.eabs[q] = __float_as_uint(fabsf(e));
      }
      if (PASS2) {
        if (obs) st_den += (double)w * (double)tdir * (double)tdir;
      } else {
        if (obs) {
          st_e2 += (double)e * (double)e;
          st_n += 1.0;
          st_w += s2 * (1.0 - (double)w);
        }
        if (!STATS_ONLY) {
          const float cv = obs ? w * e : 0.f;
#pragma unroll
          for (int q = 0; q < KT; ++q)
            if (q < a.K) dacc[q] = fmaf(cv, __ldg(rc + (int64_t)q * a.ncols), dacc[q]);
        }
      }
    }
    if (!PASS2 && !STATS_ONLY && WD) {
#pragma unroll
      for (int q = 0; q < KT; ++q) {
        if (q < a.K) {
          const float v = warp_sum_f(dacc[q]);
          if (lane == 0) a.contrib[((int64_t)blockIdx.z * a.nrows + row) * a.KP + q] = v;
        }
      }
    } else if (!PASS2 && !STATS_ONLY) {
      // reduce the per-lane gradient partials of this row over the warp
#pragma unroll
      for (int q = 0; q < KT; ++q) {
        if (q < a.K) {
          const float v = warp_sum_f(dacc[q]);
          if (lane == 0) dS[warp][q] = v;
        }
      }
      __syncwarp();
      // d(i_k)[a + r_k b] += sum_c Mid(jl)[b][c] * D[a + r_k c]   (P:152 via S = Mid Rgt)
#pragma unroll
      for (int q = 0; q < OUTS; ++q) {
        const int o = lane + 32 * q;
        if (o < a.R2) {
          const int aa = o % a.rk, b = o / a.rk;
          double v;
          if (a.p == 0) {
            v = dS[warp][o];
          } else {
            const float* mr = a.mid + (jl * a.rk1 + b) * a.rs;
            float f = 0.f;
            for (int c = 0; c < a.rs; ++c) f = fmaf(__ldg(mr + c), dS[warp][aa + a.rk * c], f);
            v = f;
          }
          outacc[q] += v;
        }
      }
      __syncwarp();
    }
  }
  // CTA reduction in a fixed order (deterministic)
  const int64_t cta = (int64_t)blockIdx.z * gridDim.x + blockIdx.x;
  const int64_t ncta = (int64_t)gridDim.x * gridDim.z;
  if (PASS2) {
    double v = warp_sum_d(st_den);
    if (lane == 0) redS[warp][0] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < kPassWarps; ++w) tot += redS[w][0];
      a.denpart[ik * ncta + cta] = tot;
    }
    return;
  }
  {
    double v0 = warp_sum_d(st_e2), v1 = warp_sum_d(st_w), v2 = warp_sum_d(st_n);
    if (lane == 0) { redS[warp][RCH] = v0; redS[warp][RCH + 1] = v1; redS[warp][RCH + 2] = v2; }
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double tot = 0.0;
    for (int w = 0; w < kPassWarps; ++w) tot += redS[w][RCH + threadIdx.x];
    a.spart[(ik * ncta + cta) * 3 + threadIdx.x] = tot;
  }
  if (!STATS_ONLY && !WD) {
    // d partials over the warps in chunks of RCH columns (fixed order)
#pragma unroll
    for (int c0 = 0; c0 < R2M; c0 += RCH) {
      if (c0 >= a.R2) break;
#pragma unroll
      for (int q = c0 / 32; q < (c0 + RCH) / 32 && q < OUTS; ++q) {
        const int o = lane + 32 * q;
        if (o < a.R2) redS[warp][o - c0] = outacc[q];
      }
      __syncthreads();
      for (int o = c0 + threadIdx.x; o < min(a.R2, c0 + RCH); o += blockDim.x) {
        double tot = 0.0;
        for (int w = 0; w < kPassWarps; ++w) tot += redS[w][o - c0];
        a.dpart[(ik * ncta + cta) * a.R2 + o] = tot;
      }
      __syncthreads();
    }
  }
}

// ----------------------------------------------------------------------------------------
// SIMT passes for 128 < K <= 256 (no tensor-core kernel; the large-rank regime, e.g. the
// paper's [80, 80, 3, 20] with K = r_k r_s = 240).  Warp per (GEMM row, column split); lane l
// owns the inner indices kappa = l + 32 m (m < 8) of Lft(row) and of the D row in registers.
// Columns are scanned 32 at a time (lane = column: mask bit and value), and the warp
// walks the observed ones: the entry's Rgt column (stored column-major, rgtC[col][kappa]:
// one coalesced 128-B load per m) gives s = <Lft, Rgt> by a fixed butterfly over the lanes,
// then e, w, c = w e (Eq. 7, 9; Thm 1) and D += c Rgt on the lanes' own kappa -- no per-lane
// K-long accumulators (the column-per-lane pass_kernel needs 256 registers at K = 256 and
// spills), and unobserved positions cost nothing.  Pass 1 writes the D row to contrib
// ([split][row][KP], contracted by reduce_d_big_kernel); pass 2 recomputes w from the cores'
// residual and sums den += w t^2 with t = <Lft_h, Rgt> (Eq. 12 / 18).
// ----------------------------------------------------------------------------------------
struct RowsArgs {
  int64_t nrows, ncols, per;     // columns per split
  int K, KP, nsplit;
  int sigma_inf, packed;
  const int64_t* row_off;
  const int64_t* col_off;
  const float* lft;              // [row][K]
  const float* lfth;             // [row][K] (pass 2)
  const float* rgtC;             // [col][KP]
  const float* values;
  const uint32_t* mask;
  const uint32_t* rank_prefix;
  const DevScalars* sc;
  float* contrib;                // [split][row][KP]
  double* spart;                 // [cta][3]
  double* denpart;               // [cta]
  uint32_t* eabs;                // R21 |e| slots (pass 1), else nullptr
  unsigned long long* efill;
  unsigned long long ecap;
};

__global__ void rgt_colmajor_kernel(const float* __restrict__ rgtT, int64_t ncols, int K, int KP,
                                    float* __restrict__ rgtC) {
  const int64_t tot = ncols * KP;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = t / KP;
    const int q = (int)(t - col * KP);
    rgtC[t] = q < K ? rgtT[(int64_t)q * ncols + col] : 0.f;
  }
}

template <bool PASS2, bool STATS_ONLY>
__global__ void __launch_bounds__(256) simt_rows_kernel(RowsArgs a) {
  constexpr int M = 8;                       // kappa slots per lane (K <= 256)
  __shared__ double red[8][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double sigma = a.sc->sigma;
  const float inv2s2 = a.sigma_inf ? 0.f : (float)(0.5 / (sigma * sigma));
  const double s2 = sigma * sigma;
  double st0 = 0.0, st1 = 0.0, st2 = 0.0;    // pass 1: sum e^2, welsch, n; pass 2: den
  const int64_t items = a.nrows * a.nsplit;
  for (int64_t it = (int64_t)blockIdx.x * 8 + warp; it < items; it += (int64_t)gridDim.x * 8) {
    const int64_t row = it / a.nsplit;
    const int split = (int)(it - row * a.nsplit);
    const int64_t ro = a.row_off[row];
    float* drow = a.contrib + ((int64_t)split * a.nrows + row) * a.KP;
    if (ro < 0) {                            // (a row outside the shard)
      if (!PASS2 && !STATS_ONLY)
        for (int q = lane; q < a.K; q += 32) drow[q] = 0.f;
      continue;
    }
    float lf[M], lh[M], D[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int q = lane + 32 * m;
      lf[m] = q < a.K ? __ldg(a.lft + row * a.K + q) : 0.f;
      lh[m] = (PASS2 && q < a.K) ? __ldg(a.lfth + row * a.K + q) : 0.f;
      D[m] = 0.f;
    }
    const int64_t cb = (int64_t)split * a.per, ce = min(a.ncols, cb + a.per);
    for (int64_t c0 = cb; c0 < ce; c0 += 32) {
      const int64_t col = c0 + lane;
      float x = 0.f;
      bool obs = false;
      if (col < ce) {
        const int64_t co = a.col_off[col];
        if (co >= 0) {
          const int64_t lin = ro + co;
          const uint32_t word = __ldg(a.mask + (lin >> 5));
          const uint32_t bit = (uint32_t)(lin & 31);
          if ((word >> bit) & 1u) {
            int64_t vi = lin;
            if (a.packed) vi = (int64_t)__ldg(a.rank_prefix + (lin >> 5)) + __popc(word & ((1u << bit) - 1u));
            x = __ldg(a.values + vi);
            obs = true;
          }
        }
      }
      unsigned bal = __ballot_sync(0xffffffffu, obs);
      if (!bal) continue;
      unsigned long long ebase = 0ull;
      if (!PASS2 && a.eabs) {                // R21: |e| of the observed entries, any order
        if (lane == 0) ebase = atomicAdd(a.efill, (unsigned long long)__popc(bal));
        ebase = __shfl_sync(0xffffffffu, ebase, 0);
      }
      int qe = 0;
      while (bal) {
        const int j = __ffs(bal) - 1;
        bal &= bal - 1;
        const float xj = __shfl_sync(0xffffffffu, x, j);
        const float* R = a.rgtC + (c0 + j) * a.KP;
        float r[M];
        float sp = 0.f, tp = 0.f;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int q = lane + 32 * m;
          r[m] = q < a.KP ? __ldg(R + q) : 0.f;
          sp = fmaf(lf[m], r[m], sp);
          if (PASS2) tp = fmaf(lh[m], r[m], tp);
        }
        const float s = warp_sum_f(sp);
        const float e = xj - s;
        const float w = a.sigma_inf ? 1.f : expf(-e * e * inv2s2);
        if (PASS2) {
          const float t = warp_sum_f(tp);
          if (lane == 0) st0 += (double)w * (double)t * (double)t;
        } else {
          if (lane == 0) {
            st0 += (double)e * (double)e;
            st1 += s2 * (1.0 - (double)w);
            st2 += 1.0;
            if (a.eabs && ebase + qe < a.ecap) a.eabs[ebase + qe] = __float_as_uint(fabsf(e));
          }
          ++qe;
          if (!STATS_ONLY) {
            const float cv = w * e;
#pragma unroll
            for (int m = 0; m < M; ++m) D[m] = fmaf(cv, r[m], D[m]);
          }
        }
      }
    }
    if (!PASS2 && !STATS_ONLY) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int q = lane + 32 * m;
        if (q < a.K) drow[q] = D[m];
      }
    }
  }
  // CTA partials in a fixed order (lane 0 of each warp holds the warp's sums)
  if (lane == 0) { red[warp][0] = st0; red[warp][1] = st1; red[warp][2] = st2; }
  __syncthreads();
  if (threadIdx.x < (PASS2 ? 1 : 3)) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
    if (PASS2) a.denpart[blockIdx.x] = t;
    else a.spart[(int64_t)blockIdx.x * 3 + threadIdx.x] = t;
  }
}

static PassArgs make_pass_args(const Context& c, const BlockPlan& bp) {
  PassArgs a;
  a.nL = bp.nL; a.nrows = bp.nrows; a.ncols = bp.ncols;
  a.K = bp.K; a.R2 = bp.R2; a.rk = bp.rk; a.rk1 = bp.rk1; a.rs = bp.rs; a.p = bp.p;
  a.jl_per_cta = bp.jl_per_cta; a.ws_split = bp.ws_split; a.nsplit = bp.nsplit;
  a.rowmode = bp.rowmode; a.Ik = bp.nrows / bp.nL;
  a.sigma_inf = c.cfg.sigma_mode == TRD_SIGMA_INF;
  a.packed = c.packed;
  a.row_off = c.row_off; a.col_off = c.col_off;
  a.lft = c.lft; a.lfth = c.lfth; a.rgtT = c.rgtT; a.mid = c.mid;
  a.values = c.values; a.mask = c.mask; a.rank_prefix = c.rank_prefix;
  a.sc = c.sc;
  a.dpart = c.dpart; a.spart = c.spart; a.denpart = c.denpart;
  a.eabs = c.cfg.sigma_mode == TRD_SIGMA_MAD ? c.eabs : nullptr;
  a.efill = &c.sc->eabs_fill;
  a.ecap = (unsigned long long)c.eabs_cap;
  a.contrib = c.contrib;
  a.KP = bp.KP;
  return a;
}

// Lft rows of a warp-per-row SIMT block with p > 0 (K > 128; the large-rank regime):
// Lft(ik, jl)[a + r_k c] = sum_b X(ik)[a][b] Mid(jl)[b][c] for a chunk of 32 left indices jl
// of one i_k per CTA, X(ik) (r_k x r_{k+1}, padded rows) and the Mid chunk staged in shared
// memory; X is the core slice (pass 1) or the folded scaled gradient h (pass 2).  Same fp32
// fmaf order over b as lft_kernel.
constexpr int kLftJ = 32;
__global__ void __launch_bounds__(256) lft_rows_kernel(PlanArgs a, const float* __restrict__ Zk, const double* __restrict__ h,
                                                       const float* __restrict__ mid, float* __restrict__ lft) {
  extern __shared__ float lsm[];
  const int rk = a.rk, rk1 = a.rk1, rs = a.rs, K = a.K, XS = rk1 + 1;
  float* Xs = lsm;                             // [rk][rk1 + 1]
  float* Ms = lsm + rk * XS;                   // [kLftJ][rk1][rs]
  const int64_t Ik = a.Ik;
  const int64_t ik = blockIdx.x;
  const int64_t jl0 = (int64_t)blockIdx.y * kLftJ;
  const int nj = (int)min((int64_t)kLftJ, a.nL - jl0);
  for (int t = threadIdx.x; t < rk * rk1; t += blockDim.x) {
    const int aa = t / rk1, b = t - aa * rk1;
    Xs[aa * XS + b] = h ? (float)h[(a.ik0 + ik) * rk * rk1 + aa + rk * b] : __ldg(Zk + (a.ik0 + ik) * rk * rk1 + t);
  }
  const int MS = rk1 * rs;
  for (int t = threadIdx.x; t < nj * MS; t += blockDim.x) Ms[t] = __ldg(mid + jl0 * MS + t);
  __syncthreads();
  for (int t = threadIdx.x; t < nj * K; t += blockDim.x) {
    const int jj = t / K, kap = t - jj * K;
    const int aa = kap % rk, cc = kap / rk;
    const float* xr = Xs + aa * XS;
    const float* mc = Ms + jj * MS + cc;
    float v = 0.f;
    for (int b = 0; b < rk1; ++b) v = fmaf(xr[b], mc[b * rs], v);
    const int64_t jl = jl0 + jj;
    const int64_t row = a.rowmode == 0 ? jl + a.nL * ik : ik + Ik * jl;
    lft[row * K + kap] = v;
  }
}

template <bool PASS2, bool STATS_ONLY>
static void launch_rows_t(Context& c, const BlockPlan& bp, cudaStream_t s) {
  RowsArgs a;
  a.nrows = bp.nrows; a.ncols = bp.ncols; a.per = bp.rows_per;
  a.K = bp.K; a.KP = bp.KP; a.nsplit = bp.rows_nsplit;
  a.sigma_inf = c.cfg.sigma_mode == TRD_SIGMA_INF;
  a.packed = c.packed;
  a.row_off = c.row_off; a.col_off = c.col_off;
  a.lft = c.lft; a.lfth = c.lfth; a.rgtC = c.rgtC;
  a.values = c.values; a.mask = c.mask; a.rank_prefix = c.rank_prefix;
  a.sc = c.sc;
  a.contrib = c.contrib; a.spart = c.spart; a.denpart = c.denpart;
  a.eabs = (!PASS2 && c.cfg.sigma_mode == TRD_SIGMA_MAD) ? c.eabs : nullptr;
  a.efill = &c.sc->eabs_fill;
  a.ecap = (unsigned long long)c.eabs_cap;
  if (!PASS2) {                              // Rgt column-major (pass 2 reuses it)
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((bp.ncols * bp.KP + 255) / 256, 148 * 16));
    rgt_colmajor_kernel<<<g, 256, 0, s>>>(c.rgtT, bp.ncols, bp.K, bp.KP, c.rgtC);
    c.launches++;
  }
  simt_rows_kernel<PASS2, STATS_ONLY><<<bp.rows_grid, 256, 0, s>>>(a);
  c.launches++;
}

template <bool PASS2, bool STATS_ONLY>
static void launch_pass_t(Context& c, const BlockPlan& bp, cudaStream_t s) {
  if (bp.rows) {                             // 128 < K <= 256: warp-per-row SIMT passes
    launch_rows_t<PASS2, STATS_ONLY>(c, bp, s);
    return;
  }
  PassArgs a = make_pass_args(c, bp);
  dim3 grid((unsigned)bp.grid_x, (unsigned)(bp.nrows / bp.nL), (unsigned)bp.nsplit);
  // (K <= 256 is checked at trd_init; R^2 > kBigR2: D rows to contrib, no per-lane d)
  if (bp.R2 > kBigR2 || PASS2 || STATS_ONLY) {
    if (bp.K <= 32) pass_kernel<32, 0, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
    else if (bp.K <= 64) pass_kernel<64, 0, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
    else if (bp.K <= 128) pass_kernel<128, 0, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
    else pass_kernel<256, 0, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
  } else if (bp.R2 <= 256) {
    if (bp.K <= 32) pass_kernel<32, 256, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
    else if (bp.K <= 64) pass_kernel<64, 256, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
    else if (bp.K <= 128) pass_kernel<128, 256, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
    else pass_kernel<256, 256, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
  } else {
    if (bp.K <= 64) pass_kernel<64, 1024, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
    else if (bp.K <= 128) pass_kernel<128, 1024, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
    else pass_kernel<256, 1024, PASS2, STATS_ONLY><<<grid, kPassThreads, 0, s>>>(a);
  }
  c.launches++;
}

// ----------------------------------------------------------------------------------------
// Reductions (fixed order) -> dvec = [d (I_k x R2) | sum_e2 | welsch | n]
// ----------------------------------------------------------------------------------------
// (Ik plan rows starting at global i_k = ik0; dvec has Ik_tot rows, the statistics after them)
__global__ void reduce_d_kernel(const double* __restrict__ dpart, const double* __restrict__ spart,
                                int64_t ncta, int R2, int64_t Ik, double* __restrict__ dvec,
                                DevScalars* sc, int kblk, int64_t ik0, int64_t Ik_tot) {
  const int64_t ik = blockIdx.x;
  if (ik < Ik) {
    for (int o = threadIdx.x; o < R2; o += blockDim.x) {
      double tot = 0.0;
      for (int64_t q = 0; q < ncta; ++q) tot += dpart[(ik * ncta + q) * R2 + o];
      dvec[(ik0 + ik) * R2 + o] = tot;
    }
    return;
  }
  // last block: statistics, summed per i_k row then over rows (fixed order)
  __shared__ double acc[3][256];
  for (int j = 0; j < 3; ++j) {
    double tot = 0.0;
    for (int64_t r = threadIdx.x; r < Ik; r += blockDim.x)
      for (int64_t q = 0; q < ncta; ++q) tot += spart[(r * ncta + q) * 3 + j];
    acc[j][threadIdx.x] = tot;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double tot = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) tot += acc[threadIdx.x][t];
    dvec[Ik_tot * R2 + threadIdx.x] = tot;
    if (threadIdx.x == 2 && sc && sc->prof_on) sc->prof_nobs[kblk] += tot;   // local count
  }
}

__global__ void reduce_den_kernel(const double* __restrict__ denpart, int64_t n,
                                  const double* __restrict__ numpart, int64_t Ik,
                                  double* __restrict__ out2) {
  __shared__ double acc[2][256];
  double a0 = 0.0, a1 = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a0 += denpart[i];
  for (int64_t i = threadIdx.x; i < Ik; i += blockDim.x) a1 += numpart[i];
  acc[0][threadIdx.x] = a0;
  acc[1][threadIdx.x] = a1;
  __syncthreads();
  if (threadIdx.x < 2) {
    double tot = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) tot += acc[threadIdx.x][t];
    out2[threadIdx.x] = tot;   // [den_local, num]
  }
}

// ----------------------------------------------------------------------------------------
// FGMC (Eq. 13; reading R6).  Q_k[(a r + a'), (b r' + b')] = sum_i Z(i)[a][b] Z(i)[a'][b']
// ----------------------------------------------------------------------------------------
// one warp per entry of Q_k: lane l sums the slices i = l, l + 32, .. in order, then a fixed
// butterfly over the lanes (deterministic; Z_k stays in L1 / L2)
__global__ void q_kernel(const float* __restrict__ Zk, int64_t Ik, int r0, int r1, double* __restrict__ Qk) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  const int n0 = r0 * r0, n1 = r1 * r1, lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)r0 * r1;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < (int64_t)n0 * n1;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int row = (int)(t / n1), col = (int)(t % n1);
    const int a = row / r0, ap = row % r0, b = col / r1, bp = col % r1;
    const float* P = Zk + a * r1 + b;
    const float* R = Zk + ap * r1 + bp;
    double acc = 0.0;
    for (int64_t i = lane; i < Ik; i += 32) acc += (double)__ldg(P + i * stride) * (double)__ldg(R + i * stride);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) Qk[t] = acc;
  }
}

// C (m x n) = A (m x q) * B (q x n), fp64, 16x16 tiles
__global__ void matmul_f64_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                  double* __restrict__ C, int m, int n, int q) {
  __shared__ double As[16][17], Bs[16][17];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double acc = 0.0;
  for (int k0 = 0; k0 < q; k0 += 16) {
    As[ty][tx] = (row < m && k0 + tx < q) ? A[(int64_t)row * q + k0 + tx] : 0.0;
    Bs[ty][tx] = (k0 + ty < q && col < n) ? B[(int64_t)(k0 + ty) * n + col] : 0.0;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) acc = fma(As[ty][kk], Bs[kk][tx], acc);
    __syncthreads();
  }
  if (row < m && col < n) C[(int64_t)row * n + col] = acc;
}

// G[c + rk b][c' + rk b'] = C[b rk1 + b'][c rk + c']   (Phi, reading R6)
__global__ void phi_kernel(const double* __restrict__ C, int rk, int rk1, double* __restrict__ G) {
  const int R2 = rk * rk1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < R2 * R2; t += gridDim.x * blockDim.x) {
    const int row = t / R2, col = t % R2;
    const int c = row % rk, b = row / rk, cp = col % rk, bp = col / rk;
    G[t] = C[(int64_t)(b * rk1 + bp) * (rk * rk) + (c * rk + cp)];
  }
}

// ----------------------------------------------------------------------------------------
// Filtered solve (Eq. 10/16 with reading R5): lambda = lambda_rel tr(G)/n, A = G + lambda I
// = L L^T, M = A^-1 (A^-1 G)^T = A^-1 G A^-1.  One CTA; retries lambda*10 up to 3 times.
// ----------------------------------------------------------------------------------------
constexpr int kSolveThreads = 1024;

// tr(G) by warp 0: lane l sums G[i][i] for i = l, l + 32, .. in order, then a fixed butterfly
// (the diagonal is read in parallel; a single-thread loop of dependent global loads cost ~25 us)
__device__ __forceinline__ void tr_s_warp(const double* __restrict__ G, int n, double* out) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
  for (int i = lane; i < n; i += 32) t += G[(int64_t)i * n + i];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) *out = t;
}

// forward (L Y = B) then backward (L^T X = Y) substitution, in place on the n x n matrix
// B (row-major, column j = one right-hand side).  8 lanes cooperate on one column.
__device__ void chol_solve_inplace(const double* L, double* B, int n) {
  const int lane8 = threadIdx.x & 7;
  const int group = threadIdx.x >> 3;           // 128 column groups
  const unsigned gmask = 0xffu << (threadIdx.x & 24);
  for (int col0 = 0; col0 < n; col0 += kSolveThreads / 8) {
    const int col = col0 + group;
    const bool act = col < n;
    // forward
    for (int i = 0; i < n; ++i) {
      double part = 0.0;
      if (act)
        for (int l = lane8; l < i; l += 8) part = fma(L[i * n + l], B[l * n + col], part);
      part += __shfl_xor_sync(gmask, part, 4);
      part += __shfl_xor_sync(gmask, part, 2);
      part += __shfl_xor_sync(gmask, part, 1);
      if (act && lane8 == 0) B[i * n + col] = (B[i * n + col] - part) / L[i * n + i];
      __syncwarp(gmask);
    }
    // backward with L^T
    for (int i = n - 1; i >= 0; --i) {
      double part = 0.0;
      if (act)
        for (int l = i + 1 + lane8; l < n; l += 8) part = fma(L[l * n + i], B[l * n + col], part);
      part += __shfl_xor_sync(gmask, part, 4);
      part += __shfl_xor_sync(gmask, part, 2);
      part += __shfl_xor_sync(gmask, part, 1);
      if (act && lane8 == 0) B[i * n + col] = (B[i * n + col] - part) / L[i * n + i];
      __syncwarp(gmask);
    }
  }
}

__global__ void __launch_bounds__(kSolveThreads)
solve_kernel(const double* __restrict__ G, int n, double lambda_rel, double* __restrict__ Mout,
             double* __restrict__ ws, int use_smem, DevScalars* __restrict__ sc) {
  extern __shared__ double sm[];
  double* L = use_smem ? sm : ws;
  double* B = use_smem ? sm + n * n : ws + n * n;
  __shared__ double tr_s;
  __shared__ int fail_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (threadIdx.x < 32) tr_s_warp(G, n, &tr_s);
  __syncthreads();
  double lam = lambda_rel * tr_s / n;
  int attempt = 0;
  for (;; ++attempt) {
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
      const int i = t / n, j = t % n;
      L[t] = G[t] + (i == j ? lam : 0.0);
    }
    if (threadIdx.x == 0) fail_s = 0;
    __syncthreads();
    // left-looking Cholesky; column j, rows i >= j; warp per row, lanes split the dot
    for (int j = 0; j < n; ++j) {
      for (int i = j + warp; i < n; i += nw) {
        double part = 0.0;
        for (int l = lane; l < j; l += 32) part = fma(L[i * n + l], L[j * n + l], part);
        part = warp_sum_d(part);
        if (lane == 0) B[i] = L[i * n + j] - part;   // B used as scratch column
      }
      __syncthreads();
      const double djj = B[j];
      if (djj <= 0.0 || !(djj == djj)) {
        if (threadIdx.x == 0) fail_s = 1;
      } else {
        const double ljj = sqrt(djj);
        for (int i = j + threadIdx.x; i < n; i += blockDim.x)
          L[i * n + j] = (i == j) ? ljj : B[i] / ljj;
      }
      __syncthreads();
      if (fail_s) break;
    }
    __syncthreads();
    if (!fail_s || attempt >= 3) break;
    lam = lam > 0.0 ? 10.0 * lam : ldexp(tr_s / n, -40);   // R23 retry rule
    __syncthreads();
  }
  if (fail_s) {
    if (threadIdx.x == 0) { sc->not_spd = 1; sc->lambda = lam; sc->h_lam = 0.0; }
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) Mout[t] = 0.0;
    return;
  }
  // zero the strict upper triangle (the algorithm read only the lower part)
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int i = t / n, j = t % n;
    if (j > i) L[t] = 0.0;
    B[t] = G[t];
  }
  __syncthreads();
  chol_solve_inplace(L, B, n);              // B = A^-1 G
  __syncthreads();
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {   // B <- B^T
    const int i = t / n, j = t % n;
    if (j > i) { const double x = B[i * n + j]; B[i * n + j] = B[j * n + i]; B[j * n + i] = x; }
  }
  __syncthreads();
  chol_solve_inplace(L, B, n);              // B = A^-1 (A^-1 G)^T = A^-1 G A^-1
  __syncthreads();
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) Mout[t] = B[t];
  if (threadIdx.x == 0) { sc->lambda = lam; sc->h_lam = 0.0; }
}

// Small-n path of a9 (R_k^2 <= kGjMaxN): the same filtered operator M = A^-1 G A^-1 with
// A = G + lambda I (R5), A^-1 by in-place Gauss-Jordan elimination (A is SPD, so
// no pivoting; a non-positive pivot means "not SPD" and triggers the lambda x10 retry like a
// failed Cholesky), then two small GEMMs.  One CTA of 32 x 32 threads; thread (ty, tx) keeps
// the elements (ty + 32 a, tx + 32 b), a, b < NB = ceil(n / 32), in registers.  Per pivot
// step the owners of row / column k+1 publish them to a double-buffered shared array, so one
// barrier separates consecutive steps.
constexpr int kGjMaxN = 112;          // 2 n^2 doubles of dynamic smem must fit 227 KB
template <int NB>
__global__ void __launch_bounds__(1024) gj_solve_kernel(const double* __restrict__ G, int n, double lambda_rel,
                                                        double* __restrict__ Mout, DevScalars* __restrict__ sc) {
  extern __shared__ double gsm[];
  double* Ainv = gsm;              // n x n
  double* Tm = gsm + n * n;        // n x n
  __shared__ double rk_s[2][kGjMaxN], ck_s[2][kGjMaxN];
  __shared__ int fail_s;
  __shared__ double tr_s;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double a[NB][NB];
  if (threadIdx.x < 32) tr_s_warp(G, n, &tr_s);
  __syncthreads();
  double lam = lambda_rel * tr_s / n;
  for (int attempt = 0;; ++attempt) {
#pragma unroll
    for (int u = 0; u < NB; ++u)
#pragma unroll
      for (int v = 0; v < NB; ++v) {
        const int i = ty + 32 * u, j = tx + 32 * v;
        a[u][v] = (i < n && j < n) ? G[i * n + j] + (i == j ? lam : 0.0) : 0.0;
        if (i == 0 && j < n) rk_s[0][j] = a[u][v];
        if (j == 0 && i < n) ck_s[0][i] = a[u][v];
      }
    if (threadIdx.x == 0) fail_s = 0;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
      const int b = k & 1;
      const double p = rk_s[b][k];
      if (!(p > 0.0)) { if (threadIdx.x == 0) fail_s = 1; break; }     // uniform
      const double ip = 1.0 / p;
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int i = ty + 32 * u;
        const double ci = (i < n) ? ck_s[b][i] : 0.0;
#pragma unroll
        for (int v = 0; v < NB; ++v) {
          const int j = tx + 32 * v;
          if (i >= n || j >= n) continue;
          const double rj = (j == k) ? ip : rk_s[b][j] * ip;         // new row k
          const double val = (i == k) ? rj : ((j == k) ? -ci * ip : fma(-ci, rj, a[u][v]));
          a[u][v] = val;
          if (i == k + 1) rk_s[b ^ 1][j] = val;
          if (j == k + 1) ck_s[b ^ 1][i] = val;
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (!fail_s || attempt >= 3) break;
    lam = lam > 0.0 ? 10.0 * lam : ldexp(tr_s / n, -40);   // R23 retry rule
    __syncthreads();
  }
  if (fail_s) {
    if (threadIdx.x == 0) { sc->not_spd = 1; sc->lambda = lam; sc->h_lam = 0.0; }
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) Mout[t] = 0.0;
    return;
  }
#pragma unroll
  for (int u = 0; u < NB; ++u)
#pragma unroll
    for (int v = 0; v < NB; ++v) {
      const int i = ty + 32 * u, j = tx + 32 * v;
      if (i < n && j < n) Ainv[i * n + j] = a[u][v];
    }
  __syncthreads();
  // M = A^-1 G A^-1 = X - lam X^2 with X = A^-1 (G = A - lam I): one product X.X, all of
  // this thread's NB x NB outputs accumulated together (independent FMA chains)
  {
    double acc[NB][NB];
#pragma unroll
    for (int u = 0; u < NB; ++u)
#pragma unroll
      for (int v = 0; v < NB; ++v) acc[u][v] = 0.0;
    for (int l = 0; l < n; ++l) {
      double xr[NB], xc[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int i = ty + 32 * u;
        xr[u] = i < n ? Ainv[i * n + l] : 0.0;
      }
#pragma unroll
      for (int v = 0; v < NB; ++v) {
        const int j = tx + 32 * v;
        xc[v] = j < n ? Ainv[l * n + j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < NB; ++u)
#pragma unroll
        for (int v = 0; v < NB; ++v) acc[u][v] = fma(xr[u], xc[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < NB; ++u)
#pragma unroll
      for (int v = 0; v < NB; ++v) {
        const int i = ty + 32 * u, j = tx + 32 * v;
        if (i < n && j < n) Mout[i * n + j] = fma(-lam, acc[u][v], Ainv[i * n + j]);
      }
  }
  if (threadIdx.x == 0) { sc->lambda = lam; sc->h_lam = 0.0; }
}

// Register Gauss-Jordan inverse for R^2 <= 128 (the a9 solve of the configs' blocks): X = A^-1,
// A = G + lambda I, two threads per row, each holding NP/2 columns of its row in registers for
// the whole elimination (NP = R^2 padded to a multiple of 16 with an identity block).  Step k:
// the owners of row k publish it to a double-buffered shared row, every thread updates
// a_ij -= (a_ik / p) a_kj over its columns (independent FMAs), the pivot row and column get
// their Gauss-Jordan values; one barrier per step.  A is SPD, so no pivoting; a non-positive
// pivot means "not SPD" and triggers the lambda retry of R23.  The filtered operator
// M = A^-1 G A^-1 = X - lambda X^2 (G = A - lambda I) is applied in h_kernel as
// h = d X - lambda (d X) X, so no X^2 product sits on this (side-stream) chain.
template <int NP>
__global__ void __launch_bounds__(256) gj2_solve_kernel(const double* __restrict__ G, int n, double lambda_rel,
                                                        double* __restrict__ Xout, DevScalars* __restrict__ sc) {
  constexpr int HC = NP / 2;
  static_assert(2 * NP <= 256 && NP % 16 == 0, "two threads per row");
  __shared__ __align__(16) double rowk[2][NP];
  __shared__ int fail_s;
  __shared__ double tr_s;
  const int tid = threadIdx.x, lane = tid & 31;
  const int row = tid >> 1, half = tid & 1;
  const bool act = row < NP;
  if (tid < 32) tr_s_warp(G, n, &tr_s);
  __syncthreads();
  double lam = lambda_rel * tr_s / n;
  double a[HC];
  for (int attempt = 0;; ++attempt) {
#pragma unroll
    for (int j = 0; j < HC; ++j) {
      const int col = half * HC + j;
      a[j] = (act && row < n && col < n) ? G[row * n + col] + (row == col ? lam : 0.0) : (row == col ? 1.0 : 0.0);
    }
    if (tid == 0) fail_s = 0;
    if (row == 0) {
#pragma unroll
      for (int j = 0; j < HC; ++j) rowk[0][half * HC + j] = a[j];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int b = k & 1;
      const double p = rowk[b][k];
      if (!(p > 0.0)) {                      // (uniform: every thread reads the same pivot)
        if (tid == 0) fail_s = 1;
        break;
      }
      const double ip = 1.0 / p;
      constexpr int dummy = 0;
      (void)dummy;
      const int kh = k / HC, kl = k % HC;    // compile-time after unrolling
      const double aik = __shfl_sync(0xffffffffu, a[kl], (lane & ~1) | kh);
      if (row == k) {
#pragma unroll
        for (int j = 0; j < HC; ++j) a[j] *= ip;
        if (half == kh) a[kl] = ip;
      } else {
        const double f = aik * ip;
#pragma unroll
        for (int j = 0; j < HC; ++j) a[j] = fma(-f, rowk[b][half * HC + j], a[j]);
        if (half == kh) a[kl] = -f;
      }
      if (k + 1 < NP && row == k + 1) {
#pragma unroll
        for (int j = 0; j < HC; ++j) rowk[b ^ 1][half * HC + j] = a[j];
      }
      __syncthreads();
    }
    __syncthreads();
    if (!fail_s || attempt >= 3) break;
    lam = lam > 0.0 ? 10.0 * lam : ldexp(tr_s / n, -40);   // R23 retry rule
    __syncthreads();
  }
  if (fail_s) {
    if (tid == 0) { sc->not_spd = 1; sc->lambda = lam; sc->h_lam = 0.0; }
    for (int t = tid; t < n * n; t += blockDim.x) Xout[t] = 0.0;
    return;
  }
  if (act && row < n) {
#pragma unroll
    for (int j = 0; j < HC; ++j) {
      const int col = half * HC + j;
      if (col < n) Xout[row * n + col] = a[j];
    }
  }
  if (tid == 0) { sc->lambda = lam; sc->h_lam = lam; }
}

// Register Gauss-Jordan inverse, 2-D distribution (the default a9 solve for R^2 <= 128): the same
// in-place elimination as gj2_solve_kernel (X = A^-1, A = G + lambda I, no pivoting: A is SPD, a
// non-positive pivot triggers the R23 retry), but every thread of the CTA holds an NU x NV block
// of A (rows ty*NU + u, columns tx*NV + v; 8 warps x 32 lanes) so that one step costs NU*NV
// independent DFMAs per thread instead of NP/2, the k loop is not unrolled (the round-1 / gj2
// kernels unrolled it over NP steps: instruction-cache bound, ~120-190 us at R^2 = 100), and only
// the n real pivots are eliminated (the identity padding never changes).  Step k: generic update
// a_ij -= (a_ik / p) a_kj over the whole block, then row k (a_kj / p, owner warp) and column k
// (-a_ik / p, owner lane; a_kk = 1 / p) are fixed up, and the owners publish row k+1 / column
// k+1 to double-buffered shared vectors; one barrier per step.
template <int NU, int NV, int TY = 8>
__global__ void __launch_bounds__(32 * TY) gj3_solve_kernel(const double* __restrict__ G, int n, double lambda_rel,
                                                            double* __restrict__ Xout, DevScalars* __restrict__ sc) {
  constexpr int NP = TY * NU, NC = 32 * NV;
  static_assert(NC >= NP, "columns cover the padded matrix");
  __shared__ __align__(16) double rowb[2][NC];
  __shared__ __align__(16) double colb[2][NP];
  __shared__ int fail_s;
  __shared__ double tr_s;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int i0 = ty * NU, j0 = tx * NV;
  if (tid < 32) tr_s_warp(G, n, &tr_s);
  __syncthreads();
  double lam = lambda_rel * tr_s / n;
  double a[NU][NV];
  for (int attempt = 0;; ++attempt) {
#pragma unroll
    for (int u = 0; u < NU; ++u)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int i = i0 + u, j = j0 + v;
        a[u][v] = (i < n && j < n) ? G[i * n + j] + (i == j ? lam : 0.0) : (i == j ? 1.0 : 0.0);
        if (i == 0) rowb[0][j] = a[u][v];
        if (j == 0) colb[0][i] = a[u][v];
      }
    if (tid == 0) fail_s = 0;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
      const int b = k & 1;
      const double p = rowb[b][k];
      if (!(p > 0.0)) {                      // (uniform: every thread reads the same pivot)
        if (tid == 0) fail_s = 1;
        break;
      }
      const double ip = 1.0 / p;
      double rj[NV], f[NU];
      if (NV % 2 == 0) {
#pragma unroll
        for (int v = 0; v < NV; v += 2) {
          const double2 t = *reinterpret_cast<const double2*>(&rowb[b][j0 + v]);
          rj[v] = t.x;
          rj[v + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) rj[v] = rowb[b][j0 + v];
      }
      if (NU % 2 == 0) {
#pragma unroll
        for (int u = 0; u < NU; u += 2) {
          const double2 t = *reinterpret_cast<const double2*>(&colb[b][i0 + u]);
          f[u] = t.x * ip;
          f[u + 1] = t.y * ip;
        }
      } else {
#pragma unroll
        for (int u = 0; u < NU; ++u) f[u] = colb[b][i0 + u] * ip;
      }
#pragma unroll
      for (int u = 0; u < NU; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) a[u][v] = fma(-f[u], rj[v], a[u][v]);
      if (ty == k / NU) {                    // row k: a_kj / p (warp-uniform)
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (i0 + u == k) {
#pragma unroll
            for (int v = 0; v < NV; ++v) a[u][v] = rj[v] * ip;
          }
      }
      if (tx == k / NV) {                    // column k: -a_ik / p, a_kk = 1 / p
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (j0 + v == k) {
#pragma unroll
            for (int u = 0; u < NU; ++u) a[u][v] = (i0 + u == k) ? ip : -f[u];
          }
      }
      const int k1 = k + 1;
      if (ty == k1 / NU) {                   // publish row k + 1
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (i0 + u == k1) {
#pragma unroll
            for (int v = 0; v < NV; ++v) rowb[b ^ 1][j0 + v] = a[u][v];
          }
      }
      if (tx == k1 / NV) {                   // publish column k + 1
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (j0 + v == k1) {
#pragma unroll
            for (int u = 0; u < NU; ++u) colb[b ^ 1][i0 + u] = a[u][v];
          }
      }
      __syncthreads();
    }
    __syncthreads();
    if (!fail_s || attempt >= 3) break;
    lam = lam > 0.0 ? 10.0 * lam : ldexp(tr_s / n, -40);   // R23 retry rule
    __syncthreads();
  }
  if (fail_s) {
    if (tid == 0) { sc->not_spd = 1; sc->lambda = lam; sc->h_lam = 0.0; }
    for (int t = tid; t < n * n; t += blockDim.x) Xout[t] = 0.0;
    return;
  }
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = i0 + u, j = j0 + v;
      if (i < n && j < n) Xout[i * n + j] = a[u][v];
    }
  if (tid == 0) { sc->lambda = lam; sc->h_lam = lam; }
}

// Register Gauss-Jordan inverse with owner-resolved steps (TRD_SOLVE=4): the same elimination,
// block distribution and arithmetic as gj3_solve_kernel (identical results on the n x n part: the
// padding rows / columns are identity and never touch it), but the pivot loop runs over chunks of
// NU pivots with the NU steps of a chunk unrolled, and NU % NV == 0.  Pivot k = kc NU + uu then
// lives in register row uu of warp kc and register column uu % NV of lane kc NU / NV + uu / NV --
// compile-time register indices -- so the row / column fix-ups and the publication of row /
// column k + 1 are a few predicated moves instead of per-element compare-and-select chains over
// the whole NU x NV block (SASS of gj3<14, 4>: ~560 instructions per step, 75 of them fp64).
template <int NU, int NV, bool PRE_IP = false, int TY = 8>
__global__ void __launch_bounds__(32 * TY) gj4_solve_kernel(const double* __restrict__ G, int n, double lambda_rel,
                                                            double* __restrict__ Xout, DevScalars* __restrict__ sc) {
  constexpr int NP = TY * NU, NC = 32 * NV;
  static_assert(NC >= NP, "columns cover the padded matrix");
  static_assert(NU % NV == 0, "a pivot chunk maps onto whole lane column groups");
  __shared__ __align__(16) double rowb[2][NC];
  __shared__ __align__(16) double colb[2][NP];
  __shared__ double ipb[2];                  // PRE_IP: 1 / pivot, published with the pivot row
  __shared__ int fail_s;
  __shared__ double tr_s;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int i0 = ty * NU, j0 = tx * NV;
  if (tid < 32) tr_s_warp(G, n, &tr_s);
  __syncthreads();
  double lam = lambda_rel * tr_s / n;
  double a[NU][NV];
  for (int attempt = 0;; ++attempt) {
#pragma unroll
    for (int u = 0; u < NU; ++u)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int i = i0 + u, j = j0 + v;
        a[u][v] = (i < n && j < n) ? G[i * n + j] + (i == j ? lam : 0.0) : (i == j ? 1.0 : 0.0);
        if (i == 0) rowb[0][j] = a[u][v];
        if (j == 0) colb[0][i] = a[u][v];
        if (PRE_IP && i == 0 && j == 0) ipb[0] = 1.0 / a[u][v];
      }
    if (tid == 0) fail_s = 0;
    __syncthreads();
    bool stop = false;
    for (int kc = 0; kc < TY && !stop; ++kc) {
#pragma unroll
      for (int uu = 0; uu < NU; ++uu) {
        const int k = kc * NU + uu;
        if (k >= n) { stop = true; break; }
        const int b = k & 1;
        const double p = rowb[b][k];
        if (!(p > 0.0)) {                    // (uniform: every thread reads the same pivot)
          if (tid == 0) fail_s = 1;
          stop = true;
          break;
        }
        const double ip = PRE_IP ? ipb[b] : 1.0 / p;
        double rj[NV], f[NU];
        if (NV % 2 == 0) {
#pragma unroll
          for (int v = 0; v < NV; v += 2) {
            const double2 t = *reinterpret_cast<const double2*>(&rowb[b][j0 + v]);
            rj[v] = t.x;
            rj[v + 1] = t.y;
          }
        } else {
#pragma unroll
          for (int v = 0; v < NV; ++v) rj[v] = rowb[b][j0 + v];
        }
        if (NU % 2 == 0) {
#pragma unroll
          for (int u = 0; u < NU; u += 2) {
            const double2 t = *reinterpret_cast<const double2*>(&colb[b][i0 + u]);
            f[u] = t.x * ip;
            f[u + 1] = t.y * ip;
          }
        } else {
#pragma unroll
          for (int u = 0; u < NU; ++u) f[u] = colb[b][i0 + u] * ip;
        }
        const int bn = b ^ 1;
        if (PRE_IP) {                        // next pivot's owner: 1 / a_{k+1,k+1} off the critical path
          const int u1 = (uu + 1) % NU, v1 = (uu + 1) % NV;
          if (ty == (uu + 1 < NU ? kc : kc + 1) && tx == kc * (NU / NV) + (uu + 1) / NV)
            ipb[bn] = 1.0 / fma(-f[u1], rj[v1], a[u1][v1]);   // = the updated a_{k+1,k+1} (bitwise)
        }
#pragma unroll
        for (int u = 0; u < NU; ++u)
#pragma unroll
          for (int v = 0; v < NV; ++v) a[u][v] = fma(-f[u], rj[v], a[u][v]);
        if (ty == kc) {                      // row k = register row uu of warp kc: a_kj / p
#pragma unroll
          for (int v = 0; v < NV; ++v) a[uu][v] = rj[v] * ip;
        }
        const int vk = uu % NV;              // column k = register column vk of one lane
        if (tx == kc * (NU / NV) + uu / NV) {
#pragma unroll
          for (int u = 0; u < NU; ++u) a[u][vk] = -f[u];
          if (ty == kc) a[uu][vk] = ip;      // a_kk = 1 / p
        }
        // publish row k + 1 and column k + 1
        if (uu + 1 < NU) {
          if (ty == kc) {
#pragma unroll
            for (int v = 0; v < NV; ++v) rowb[bn][j0 + v] = a[(uu + 1) % NU][v];
          }
        } else if (ty == kc + 1) {
#pragma unroll
          for (int v = 0; v < NV; ++v) rowb[bn][j0 + v] = a[0][v];
        }
        const int vk1 = (uu + 1) % NV;
        if (tx == kc * (NU / NV) + (uu + 1) / NV) {
#pragma unroll
          for (int u = 0; u < NU; ++u) colb[bn][i0 + u] = a[u][vk1];
        }
        __syncthreads();
      }
    }
    __syncthreads();
    if (!fail_s || attempt >= 3) break;
    lam = lam > 0.0 ? 10.0 * lam : ldexp(tr_s / n, -40);   // R23 retry rule
    __syncthreads();
  }
  if (fail_s) {
    if (tid == 0) { sc->not_spd = 1; sc->lambda = lam; sc->h_lam = 0.0; }
    for (int t = tid; t < n * n; t += blockDim.x) Xout[t] = 0.0;
    return;
  }
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = i0 + u, j = j0 + v;
      if (i < n && j < n) Xout[i * n + j] = a[u][v];
    }
  if (tid == 0) { sc->lambda = lam; sc->h_lam = lam; }
}

// Blocked Gauss-Jordan inverse in shared memory (R^2 in (48, 128]; TRD_SOLVE=3 forces it, 0 the
// register kernels): the same in-place elimination as gj2 / gj3 with kGjB pivots per step, so the
// CTA synchronises ~4 times per pivot block instead of once per pivot.  With P the current pivot
// block (a Schur complement of the SPD A = G + lambda I, so SPD: no pivoting), B its row block, C
// its column block and D the rest, one step maps [P B; C D] to [P^-1, P^-1 B; -C P^-1, D - C P^-1 B]
// (kGjB scalar Gauss-Jordan steps at once): warp 0 inverts P in place (scalar Gauss-Jordan, warp
// synchronous), then the row block, the trailing block (old C, new row block) and the column block.
// A non-positive pivot triggers the R23 retry.  Row stride LD odd (conflict-free column reads).
constexpr int kGjB = 16;
__global__ void __launch_bounds__(256) gjb_solve_kernel(const double* __restrict__ G, int n, double lambda_rel,
                                                        double* __restrict__ Xout, DevScalars* __restrict__ sc) {
  trd_gdc_wait();
  extern __shared__ double gsm_b[];
  const int LD = n | 1;
  double* A = gsm_b;                          // [n][LD]
  __shared__ int fail_s;
  __shared__ double tr_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) tr_s_warp(G, n, &tr_s);
  __syncthreads();
  double lam = lambda_rel * tr_s / n;
  for (int attempt = 0;; ++attempt) {
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      A[i * LD + j] = G[e] + (i == j ? lam : 0.0);
    }
    if (tid == 0) fail_s = 0;
    __syncthreads();
    for (int K = 0; K < n; K += kGjB) {
      const int bs = min(kGjB, n - K);
      // (1) P <- P^-1, warp 0, scalar in-place Gauss-Jordan (lane owns up to 8 of the bs x bs)
      if (warp == 0) {
        for (int kk = 0; kk < bs; ++kk) {
          const double piv = A[(K + kk) * LD + K + kk];
          const bool bad = !(piv > 0.0);
          if (bad) { if (lane == 0) fail_s = 1; }
          const double ip = bad ? 0.0 : 1.0 / piv;
          double nv[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int e = lane + 32 * t;
            nv[t] = 0.0;
            if (e < bs * bs) {
              const int r = e / bs, c = e - r * bs;
              const double prk = A[(K + r) * LD + K + kk], pkc = A[(K + kk) * LD + K + c], prc = A[(K + r) * LD + K + c];
              nv[t] = (r == kk && c == kk) ? ip : (r == kk) ? pkc * ip : (c == kk) ? -prk * ip : fma(-prk * ip, pkc, prc);
            }
          }
          __syncwarp();
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int e = lane + 32 * t;
            if (e < bs * bs) {
              const int r = e / bs, c = e - r * bs;
              A[(K + r) * LD + K + c] = nv[t];
            }
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (fail_s) break;
      // (2) row block B <- P^-1 B  (rows K..K+bs, columns outside the block)
      const int nc = n - bs;                   // columns outside the block
      {
        constexpr int NT = (kGjB * 128 + 255) / 256;   // outputs per thread (blockDim 256)
        double nv[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int e = tid + 256 * t;
          nv[t] = 0.0;
          if (e < bs * nc) {
            const int r = e / nc, jj = e - r * nc, j = jj < K ? jj : jj + bs;
            double acc = 0.0;
            for (int q = 0; q < bs; ++q) acc = fma(A[(K + r) * LD + K + q], A[(K + q) * LD + j], acc);
            nv[t] = acc;
          }
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int e = tid + 256 * t;
          if (e < bs * nc) {
            const int r = e / nc, jj = e - r * nc, j = jj < K ? jj : jj + bs;
            A[(K + r) * LD + j] = nv[t];
          }
        }
      }
      __syncthreads();
      // (3) trailing D <- D - C (P^-1 B)   (old column block C, new row block)
      for (int e = tid; e < nc * nc; e += blockDim.x) {
        const int ii = e / nc, jj = e - ii * nc;
        const int i = ii < K ? ii : ii + bs, j = jj < K ? jj : jj + bs;
        double acc = A[i * LD + j];
        for (int q = 0; q < bs; ++q) acc = fma(-A[i * LD + K + q], A[(K + q) * LD + j], acc);
        A[i * LD + j] = acc;
      }
      __syncthreads();
      // (4) column block C <- -C P^-1   (thread per row outside the block)
      for (int ii = tid; ii < nc; ii += blockDim.x) {
        const int i = ii < K ? ii : ii + bs;
        double cr[kGjB];
#pragma unroll
        for (int q = 0; q < kGjB; ++q) cr[q] = q < bs ? A[i * LD + K + q] : 0.0;
#pragma unroll
        for (int c = 0; c < kGjB; ++c) {
          if (c >= bs) break;
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < kGjB; ++q)
            if (q < bs) acc = fma(cr[q], A[(K + q) * LD + K + c], acc);
          A[i * LD + K + c] = -acc;
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (!fail_s || attempt >= 3) break;
    lam = lam > 0.0 ? 10.0 * lam : ldexp(tr_s / n, -40);   // R23 retry rule
    __syncthreads();
  }
  if (fail_s) {
    if (tid == 0) { sc->not_spd = 1; sc->lambda = lam; sc->h_lam = 0.0; }
    for (int t = tid; t < n * n; t += blockDim.x) Xout[t] = 0.0;
    return;
  }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    Xout[e] = A[i * LD + j];
  }
  if (tid == 0) { sc->lambda = lam; sc->h_lam = lam; }
}

// h = d M (row-wise) with M = Mop - h_lam Mop^2 (h_lam = lambda when Mop = (G + lambda I)^-1 from
// gj2_solve_kernel, 0 when Mop is M itself), computed as u = d Mop, h = u - h_lam u Mop;
// num partial per row = <d(i), h(i)>
__global__ void h_kernel(const double* __restrict__ dvec, const double* __restrict__ M, int R2,
                         double* __restrict__ h, double* __restrict__ numpart, const DevScalars* __restrict__ sc) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  __shared__ double drow[kBigR2];       // (R^2 <= kBigR2; larger blocks: big_h)
  __shared__ double urow[kBigR2];
  __shared__ double red[256];
  const int64_t ik = blockIdx.x;
  const double hl = sc->h_lam;
  for (int o = threadIdx.x; o < R2; o += blockDim.x) drow[o] = dvec[ik * R2 + o];
  __syncthreads();
  // (one fp64 chain per output, q ascending; measured faster than four interleaved chains)
  auto rowvec = [&](const double* x, int o) {
    double acc = 0.0;
    for (int q = 0; q < R2; ++q) acc = fma(x[q], M[q * R2 + o], acc);
    return acc;
  };
  for (int o = threadIdx.x; o < R2; o += blockDim.x) urow[o] = rowvec(drow, o);
  __syncthreads();
  double part = 0.0;
  for (int o = threadIdx.x; o < R2; o += blockDim.x) {
    double v = urow[o];
    if (hl != 0.0) v = fma(-hl, rowvec(urow, o), v);
    h[ik * R2 + o] = v;
    part += v * drow[o];
  }
  // num partial: a fixed butterfly per warp, then the warp sums in warp order
  for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    numpart[ik] = tot;
  }
}

// ----------------------------------------------------------------------------------------
// Update (Eq. 11/17, reading R2: Z_k <- Z_k + eta fold(h)) and block statistics
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ double block_eta(const DevScalars* sc, double step) {
  if (step > 0.0) return step;
  const double num = sc->num, den = sc->den;
  return (num > 0.0 && den > 0.0) ? num / den : 0.0;
}

__global__ void update2_kernel(float* __restrict__ Zk, const double* __restrict__ h, int64_t Ik,
                               int rk, int rk1, double step, const DevScalars* __restrict__ sc) {
  const double eta = block_eta(sc, step);
  if (eta == 0.0) return;
  const int64_t tot = Ik * rk * rk1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    // device layout Z_k[i][a][b]; h[i][a + rk b]
    const int b = (int)(t % rk1);
    const int64_t ia = t / rk1;
    const int aa = (int)(ia % rk);
    const int64_t i = ia / rk;
    const double v = (double)Zk[t] + eta * h[i * rk * rk1 + aa + rk * b];
    Zk[t] = (float)v;
  }
}

// scalars after the pass-1 allreduce and after the pass-2 allreduce
__global__ void block_scalars_kernel(const double* __restrict__ dvec, int64_t Ik, int R2,
                                     const double* __restrict__ numden, DevScalars* sc,
                                     DevStats* stats, int k, double step, int phase) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (phase == 0) {
    sc->sum_e2 = dvec[Ik * R2 + 0];
    sc->welsch = dvec[Ik * R2 + 1];
    sc->n_obs = dvec[Ik * R2 + 2];
    return;
  }
  sc->den = numden[0];
  sc->num = numden[1];
  const double eta = block_eta(sc, step);
  sc->eta = eta;
  DevStats& st = stats[sc->slot];
  st.eta[k] = eta;
  st.num[k] = sc->num;
  st.den[k] = sc->den;
  st.nnz[k] = (long long)sc->n_obs;
  st.n_obs += (long long)sc->n_obs;
  st.sum_e2 += sc->sum_e2;
  st.welsch += sc->welsch;
  if (eta == 0.0) st.skipped |= (1u << k);
  if (!(eta == eta) || isinf(eta) || !(sc->num == sc->num) || !(sc->den == sc->den) || isinf(sc->den)) {
    st.nonfinite = 1;
    sc->nonfinite = 1;
  }
  sc->acc_e2 += sc->sum_e2;
  sc->acc_n += sc->n_obs;
}

// World 1 (no den exchange between them): reduce_den_kernel, block_scalars_kernel (both phases)
// and update2_kernel as one launch.  Every CTA forms the den / num sums in the same fixed order
// (256 partial sums, then thread 0 / 1 in thread order) and the same eta, so the grid needs no
// second launch; CTA 0 writes [den, num] and the block record (thread 0), and the CTAs update
// their share of Z_k <- Z_k + eta fold(h) (Eq. 11/17 with Eq. 12's eta, reading R2).  Bitwise
// the results of the separate kernels.
__global__ void __launch_bounds__(256) block_tail_kernel(const double* __restrict__ denpart, int64_t nden,
                                                         const double* __restrict__ numpart, int64_t nnum,
                                                         double* __restrict__ numden, const double* __restrict__ dvec,
                                                         int64_t Ik, int R2, DevScalars* sc, DevStats* stats, int k,
                                                         double step, float* __restrict__ Zk,
                                                         const double* __restrict__ h, int rk, int rk1) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  __shared__ double acc[2][256];
  __shared__ double nd_s[2];
  const int t = threadIdx.x;
  double a0 = 0.0, a1 = 0.0;
  for (int64_t i = t; i < nden; i += 256) a0 += denpart[i];
  for (int64_t i = t; i < nnum; i += 256) a1 += numpart[i];
  acc[0][t] = a0;
  acc[1][t] = a1;
  __syncthreads();
  if (t < 2) {
    double tot = 0.0;
    for (int j = 0; j < 256; ++j) tot += acc[t][j];
    nd_s[t] = tot;
    if (blockIdx.x == 0) numden[t] = tot;   // [den, num]
  }
  __syncthreads();
  const double den = nd_s[0], num = nd_s[1];
  const double eta = step > 0.0 ? step : ((num > 0.0 && den > 0.0) ? num / den : 0.0);   // = block_eta
  if (blockIdx.x == 0 && t == 0) {
    sc->sum_e2 = dvec[Ik * R2 + 0];
    sc->welsch = dvec[Ik * R2 + 1];
    sc->n_obs = dvec[Ik * R2 + 2];
    sc->den = den;
    sc->num = num;
    sc->eta = eta;
    DevStats& st = stats[sc->slot];
    st.eta[k] = eta;
    st.num[k] = num;
    st.den[k] = den;
    st.nnz[k] = (long long)sc->n_obs;
    st.n_obs += (long long)sc->n_obs;
    st.sum_e2 += sc->sum_e2;
    st.welsch += sc->welsch;
    if (eta == 0.0) st.skipped |= (1u << k);
    if (!(eta == eta) || isinf(eta) || !(num == num) || !(den == den) || isinf(den)) {
      st.nonfinite = 1;
      sc->nonfinite = 1;
    }
    sc->acc_e2 += sc->sum_e2;
    sc->acc_n += sc->n_obs;
  }
  if (eta == 0.0) return;
  const int64_t tot = Ik * rk * rk1;
  for (int64_t q = blockIdx.x * 256 + t; q < tot; q += (int64_t)gridDim.x * 256) {
    const int b = (int)(q % rk1);
    const int64_t ia = q / rk1;
    const int aa = (int)(ia % rk);
    const int64_t i = ia / rk;
    const double v = (double)Zk[q] + eta * h[i * rk * rk1 + aa + rk * b];
    Zk[q] = (float)v;
  }
}

// the sweep's record slot comes from device memory (sc->slot_next, reset by trd_sweep), so a
// captured sweep replays into successive records
__global__ void sweep_begin_kernel(DevScalars* sc, DevStats* stats) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  sc->slot = sc->slot_next++;
  DevStats& st = stats[sc->slot];
  st.sigma = sc->sigma;
  st.sum_e2 = 0.0; st.welsch = 0.0; st.stop_e = 0.0; st.n_obs = 0;
  for (int k = 0; k < kMaxN; ++k) { st.eta[k] = 0.0; st.num[k] = 0.0; st.den[k] = 0.0; st.nnz[k] = 0; }
  st.skipped = 0; st.nonfinite = 0; st.replica_mismatch = 0;
  sc->acc_e2 = 0.0; sc->acc_n = 0.0;
  sc->eabs_fill = 0ull;
}

// ----------------------------------------------------------------------------------------
// End of sweep: D^t = Z_N(2) G_{!=N} Z_N(2)^T (Alg. 1 l.12), e_t (l.13), sigma (R9)
// ----------------------------------------------------------------------------------------
__global__ void dt_T_kernel(const float* __restrict__ Zn, int64_t In, int rk, int rk1,
                            const double* __restrict__ G, double* __restrict__ T) {
  const int R2 = rk * rk1;
  const int64_t i = blockIdx.x;
  for (int o = blockIdx.y * blockDim.x + threadIdx.x; o < R2; o += gridDim.y * blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < R2; ++q) {
      const int aa = q % rk, b = q / rk;
      acc = fma((double)Zn[(i * rk + aa) * rk1 + b], G[q * R2 + o], acc);
    }
    T[i * R2 + o] = acc;
  }
}

__global__ void dt_D_kernel(const float* __restrict__ Zn, int64_t In, int rk, int rk1,
                            const double* __restrict__ T, double* __restrict__ D) {
  const int R2 = rk * rk1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < In * In;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / In, j = t % In;
    double acc = 0.0;
    for (int q = 0; q < R2; ++q) {
      const int aa = q % rk, b = q / rk;
      acc = fma(T[i * R2 + q], (double)Zn[(j * rk + aa) * rk1 + b], acc);
    }
    D[t] = acc;
  }
}

// ----------------------------------------------------------------------------------------
// R21: exact median of the |e| bit patterns eabs[0, eabs_fill) by radix select.  Level 0 counts
// bits 31..21, level 1 bits 20..10 of the values under each target's level-0 prefix, level 2
// bits 9..0; the two targets are the order statistics floor((n-1)/2) and floor(n/2).  Counts
// are integers (atomics in any order give the same histogram); scans run in one thread.
// ----------------------------------------------------------------------------------------
// level 0 (|e| concentrates in a few top-11-bit bins): one private histogram per warp in
// dynamic shared memory (kMadWarps x 2048 counters), added up at the end of the CTA
constexpr int kMadThreads = 256, kMadWarps = kMadThreads / 32;
template <int LEVEL>
__global__ void __launch_bounds__(kMadThreads) mad_hist_kernel(const uint32_t* __restrict__ eabs,
                                                               const DevScalars* __restrict__ sc, double* __restrict__ mh) {
  constexpr int NB = LEVEL == 2 ? kMadBins2 : kMadBins0;
  constexpr int NT = LEVEL == 0 ? kMadWarps : 2;
  extern __shared__ unsigned int h[];                  // [NT][NB]
  for (int i = threadIdx.x; i < NT * NB; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const unsigned long long n = sc->eabs_fill;
  const uint32_t p0 = sc->mad_pre[0], p1 = sc->mad_pre[1];
  unsigned int* hw = h + (LEVEL == 0 ? (threadIdx.x >> 5) * NB : 0);
  auto count = [&](uint32_t b) {
    if (b >= 0x80000000u) return;                        // padding slot (kEabsPad)
    if (LEVEL == 0) {
      atomicAdd(&hw[b >> 21], 1u);
    } else if (LEVEL == 1) {
      const uint32_t pf = b >> 21, bin = (b >> 10) & 2047u;
      if (pf == p0) atomicAdd(&h[bin], 1u);
      if (pf == p1) atomicAdd(&h[NB + bin], 1u);
    } else {
      const uint32_t pf = b >> 10, bin = b & 1023u;
      if (pf == p0) atomicAdd(&h[bin], 1u);
      if (pf == p1) atomicAdd(&h[NB + bin], 1u);
    }
  };
  // 16-byte loads, four in flight per thread (memory-level parallelism for the 3+ GB scans)
  const unsigned long long n4 = n / 4;
  const uint4* e4 = reinterpret_cast<const uint4*>(eabs);
  const unsigned long long step = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long q = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  for (; q + 3 * step < n4; q += 4 * step) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(e4 + q + u * step);
#pragma unroll
    for (int u = 0; u < 4; ++u) { count(v[u].x); count(v[u].y); count(v[u].z); count(v[u].w); }
  }
  for (; q < n4; q += step) {
    const uint4 v = __ldg(e4 + q);
    count(v.x); count(v.y); count(v.z); count(v.w);
  }
  for (unsigned long long t = n4 * 4 + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < n; t += step)
    count(__ldg(eabs + t));
  __syncthreads();
  double* dst = mh + (LEVEL == 0 ? 0 : LEVEL == 1 ? kMadBins0 : kMadBins0 + 2 * kMadBins1);
  if (LEVEL == 0) {
    for (int i = threadIdx.x; i < NB; i += blockDim.x) {
      unsigned int t = 0;
      for (int w = 0; w < kMadWarps; ++w) t += h[w * NB + i];
      if (t) atomicAdd(dst + i, (double)t);
    }
  } else {
    for (int i = threadIdx.x; i < NT * NB; i += blockDim.x)
      if (h[i]) atomicAdd(dst + i, (double)h[i]);
  }
}

// The target bins: a block-wide exclusive scan of the (integer) counts, each thread checks its
// two bins for the one that holds the target rank (one CTA of 1024 threads, bins <= 2048)
__device__ __forceinline__ void mad_find_bin(const double* __restrict__ h, int nb, long long r, int* bin_out,
                                             long long* rank_out) {
  using Scan = cub::BlockScan<long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  const int t = threadIdx.x;
  const long long c0 = 2 * t < nb ? (long long)h[2 * t] : 0ll;
  const long long c1 = 2 * t + 1 < nb ? (long long)h[2 * t + 1] : 0ll;
  long long ex;
  Scan(tmp).ExclusiveSum(c0 + c1, ex);
  if (2 * t < nb && ex <= r && r < ex + c0) { *bin_out = 2 * t; *rank_out = r - ex; }
  if (2 * t + 1 < nb && ex + c0 <= r && r < ex + c0 + c1) { *bin_out = 2 * t + 1; *rank_out = r - ex - c0; }
  __syncthreads();
}

template <int LEVEL>
__global__ void __launch_bounds__(1024) mad_scan_kernel(const double* __restrict__ mh, DevScalars* sc) {
  __shared__ int bin_s;
  __shared__ long long rank_s;
  __shared__ long long n_s;
  if (LEVEL == 0) {
    // n = total count (block reduction of the level-0 bins)
    using Red = cub::BlockReduce<long long, 1024>;
    __shared__ typename Red::TempStorage rt;
    long long c = 0;
    for (int b = threadIdx.x; b < kMadBins0; b += blockDim.x) c += (long long)mh[b];
    const long long n = Red(rt).Sum(c);
    if (threadIdx.x == 0) { n_s = n; sc->mad_n = (double)n; }
    __syncthreads();
  }
  const int NB = LEVEL == 0 ? kMadBins0 : (LEVEL == 1 ? kMadBins1 : kMadBins2);
  const double* h0 = mh + (LEVEL == 0 ? 0 : LEVEL == 1 ? kMadBins0 : kMadBins0 + 2 * kMadBins1);
  float v[2] = {0.f, 0.f};
  for (int t = 0; t < 2; ++t) {
    long long r;
    if (LEVEL == 0) {
      const long long ni = n_s;
      r = t == 0 ? (ni > 0 ? (ni - 1) / 2 : 0) : ni / 2;
    } else {
      r = sc->mad_rank[t];
    }
    if (threadIdx.x == 0) { bin_s = NB - 1; rank_s = 0; }
    __syncthreads();
    mad_find_bin(h0 + (LEVEL == 0 ? 0 : t * NB), NB, r, &bin_s, &rank_s);
    if (threadIdx.x == 0) {
      sc->mad_rank[t] = rank_s;
      if (LEVEL == 0) sc->mad_pre[t] = (uint32_t)bin_s;
      else if (LEVEL == 1) sc->mad_pre[t] = (sc->mad_pre[t] << 11) | (uint32_t)bin_s;
      else v[t] = __uint_as_float((sc->mad_pre[t] << 10) | (uint32_t)bin_s);
    }
    __syncthreads();
  }
  if (LEVEL == 2 && threadIdx.x == 0) sc->mad_med = sc->mad_n > 0.0 ? 0.5 * ((double)v[0] + (double)v[1]) : 0.0;
}

// pass 1 of a staged block wrote its tile slots (padding included) at eabs_fill + [0, total)
__global__ void eabs_advance_kernel(DevScalars* sc, const uint64_t* __restrict__ tbase_end) {
  if (threadIdx.x == 0 && blockIdx.x == 0) sc->eabs_fill += *tbase_end;
}

__global__ void sweep_end_kernel(double* __restrict__ D, double* __restrict__ Dprev, int64_t n2,
                                 DevScalars* sc, DevStats* stats, int sigma_mode,
                                 double theta, double sigma_min) {
  __shared__ double a1[1024], a2[1024];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t t = threadIdx.x; t < n2; t += blockDim.x) {
    const double dd = D[t] - Dprev[t];
    s1 += dd * dd;
    s2 += D[t] * D[t];
  }
  a1[threadIdx.x] = s1;
  a2[threadIdx.x] = s2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) { t1 += a1[t]; t2 += a2[t]; }
    const double e = sc->have_prev_D ? sqrt(t1) / sqrt(t2) : __longlong_as_double(0x7ff8000000000000LL);
    sc->stop_e = e;
    stats[sc->slot].stop_e = e;
    if (sigma_mode == TRD_SIGMA_RMS && sc->acc_n > 0.0)
      sc->sigma = fmax(sigma_min, theta * sqrt(sc->acc_e2 / sc->acc_n));
    if (sigma_mode == TRD_SIGMA_MAD && sc->acc_n > 0.0) sc->sigma = fmax(sigma_min, theta * 1.4826 * sc->mad_med);
    sc->have_prev_D = 1;
    sc->sweep += 1;
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < n2; t += blockDim.x) Dprev[t] = D[t];
}

// sigma_0 = max(sigma_min, theta * RMS) from [sum_e2, welsch, n] (after allreduce), or the
// MAD rule's median (R21)
__global__ void sigma0_kernel(const double* __restrict__ s3, DevScalars* sc, double theta,
                              double sigma_min, int mad) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    sc->sigma = mad ? fmax(sigma_min, theta * 1.4826 * sc->mad_med)
                    : fmax(sigma_min, theta * sqrt(s3[0] / fmax(s3[2], 1.0)));
}

// ----------------------------------------------------------------------------------------
// Reconstruction (Def. 1) at arbitrary global linear indices
// ----------------------------------------------------------------------------------------
struct ReconArgs {
  int N;
  int64_t dims[kMaxN];
  int ranks[kMaxN + 1];
  int64_t zoff[kMaxN + 1];
};

template <int RM>
__device__ float tr_value(const ReconArgs& a, const float* __restrict__ Z, const int64_t* ix) {
  // Tr(prod_k Z_k(i_k)) = sum_a e_a^T Z_0(i_0) ... Z_{N-1}(i_{N-1}) e_a
  float tot = 0.f;
  for (int a0 = 0; a0 < a.ranks[0]; ++a0) {
    float v[RM];
#pragma unroll
    for (int c = 0; c < RM; ++c) v[c] = (c == a0) ? 1.f : 0.f;
    int rin = a.ranks[0];
    for (int m = 0; m < a.N; ++m) {
      const int rout = a.ranks[m + 1];
      vecmat<RM>(v, Z + a.zoff[m] + ix[m] * (int64_t)a.ranks[m] * rout, rin, rout);
      rin = rout;
    }
    tot += v[a0];
  }
  return tot;
}

template <int RM>
__global__ void recon_kernel(ReconArgs a, const float* __restrict__ Z, const int64_t* __restrict__ lin,
                             int64_t n, float* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = lin[t], ix[kMaxN];
    for (int m = 0; m < a.N; ++m) { ix[m] = l % a.dims[m]; l /= a.dims[m]; }
    out[t] = tr_value<RM>(a, Z, ix);
  }
}

// error over all local entries, GEMM form with full index sets (plan = full plan).
// out per CTA: [sum (x-ref)^2 all, sum ref^2 all, sum (x-ref)^2 obs, sum ref^2 obs, n, max|ref|]
__global__ void __launch_bounds__(256)
error_kernel(PassArgs a, const float* __restrict__ ref, const uint32_t* __restrict__ evalb,
             double* __restrict__ part) {
  __shared__ float lftS[8][256];        // (K <= 256)
  __shared__ double red[8][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s[6] = {0, 0, 0, 0, 0, 0};
  const int64_t nw_total = (int64_t)gridDim.x * 8;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < a.nrows; row += nw_total) {
    const int64_t ro = a.row_off[row];
    if (ro < 0) continue;
    for (int q = lane; q < a.K; q += 32) lftS[warp][q] = a.lft[row * a.K + q];
    __syncwarp();
    for (int64_t c0 = 0; c0 < a.ncols; c0 += 32) {
      const int64_t col = c0 + lane;
      if (col < a.ncols) {
        const int64_t co = a.col_off[col];
        if (co >= 0) {
          const int64_t lin = ro + co;
          const bool ev = evalb ? ((evalb[lin >> 5] >> (lin & 31)) & 1u) : true;
          if (ev) {
            float recon = 0.f;
            for (int q = 0; q < a.K; ++q) recon = fmaf(lftS[warp][q], a.rgtT[(int64_t)q * a.ncols + col], recon);
            const double r = ref[lin];
            const double dd = (double)recon - r;
            s[0] += dd * dd;
            s[1] += r * r;
            if ((a.mask[lin >> 5] >> (lin & 31)) & 1u) { s[2] += dd * dd; s[3] += r * r; }
            s[4] += 1.0;
            s[5] = fmax(s[5], fabs(r));
          }
        }
      }
    }
    __syncwarp();
  }
  for (int j = 0; j < 6; ++j) {
    double v = s[j];
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v, o);
      v = (j == 5) ? fmax(v, u) : v + u;
    }
    if (lane == 0) red[warp][j] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v = (threadIdx.x == 5) ? fmax(v, red[w][threadIdx.x]) : v + red[w][threadIdx.x];
    part[blockIdx.x * 6 + threadIdx.x] = v;
  }
}

// 256 threads: thread t folds partials t, t + 256, .. (fixed order), then a fixed tree
__global__ void error_reduce_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[6][256];
  double v[6] = {0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < n; b += blockDim.x)
    for (int j = 0; j < 6; ++j) v[j] = (j == 5) ? fmax(v[j], part[b * 6 + j]) : v[j] + part[b * 6 + j];
  for (int j = 0; j < 6; ++j) red[j][threadIdx.x] = v[j];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int j = 0; j < 6; ++j)
        red[j][threadIdx.x] = (j == 5) ? fmax(red[j][threadIdx.x], red[j][threadIdx.x + w]) : red[j][threadIdx.x] + red[j][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 6) out[threadIdx.x] = red[threadIdx.x][0];
}

__global__ void popc_kernel(const uint32_t* __restrict__ mask, int64_t nw, uint32_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nw;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = __popc(mask[t]);
}

// ----------------------------------------------------------------------------------------
// Launchers
// ----------------------------------------------------------------------------------------
// Kernel attributes are per device, and contexts may be driven from several host threads: the
// attribute is set before every launch that needs it (a cheap host call; a "done" flag shared
// between threads let a second thread launch before the first had set it)
bool kern_check_collect(DevCheck* out, unsigned int jitter_ns, cudaStream_t s) {
  DevCheck h = {}, z = {};
  z.jitter_ns = jitter_ns;
  cudaMemcpyFromSymbolAsync(&h, g_check, sizeof(h), 0, cudaMemcpyDeviceToHost, s);
  cudaMemcpyToSymbolAsync(g_check, &z, sizeof(z), 0, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  *out = h;
  return h.code != 0;
}

static bool first_on_device(uint64_t& done_mask) {
  (void)done_mask;
  return true;
}

static int grid_for(int64_t n, int threads = 256, int cap = 148 * 16) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

void launch_sampler(Context& c, const BlockPlan& bp, cudaStream_t s) {
  SamplerArgs sa;
  sa.N = c.N; sa.k = bp.k; sa.shard_mode = c.cfg.shard_mode; sa.seed = c.cfg.seed;
  sa.shard_begin = c.shard_begin; sa.shard_end = c.shard_end;
  sa.shard_local = bp.shard_local;
  sa.shard_sampled = bp.shard_sampled;
  for (int m = 0; m < c.N; ++m) {
    sa.dims[m] = c.dims[m];
    sa.s[m] = bp.s[m];
    sa.s_samp[m] = bp.s_samp[m];
    sa.idx_off[m] = c.idx_off[m];
    sa.lstride[m] = c.lstride[m];
  }
  sa.idx_off[c.N] = c.idx_off[c.N];
  sa.ptab = stage_uses_pext(c, bp) ? c.ptab : nullptr;
  if (bp.explicit_cols) {
    const int64_t J = bp.ncols;
    row_sampler_kernel<<<grid_for(J + c.dims[bp.k]), 256, 0, s>>>(sa, J, c.sc, c.idx, c.doff);
    c.launches++;
    return;
  }
  TRD_PDL(sampler_kernel, c.N, kSamplerThreads, 0, s, sa, c.sc, c.idx, c.doff);
  c.launches++;
}

void launch_offsets(Context& c, const BlockPlan& bp, cudaStream_t s, bool reset_amax) {
  PlanArgs a = make_plan_args(c, bp);
  TRD_PDL(offsets_kernel, grid_for(bp.nrows + bp.ncols), 256, 0, s, a, c.doff, c.row_off, c.col_off,
                                                              reset_amax ? c.sc : nullptr);
  c.launches++;
}

void launch_plan(Context& c, const BlockPlan& bp, cudaStream_t s, bool offsets) {
  PlanArgs a = make_plan_args(c, bp);
  // warp-per-index chain products (TRD_CHAIN_THREAD=1: the thread-per-row kernels, A/B runs)
  const bool warp_chains = !(getenv("TRD_CHAIN_THREAD") && atoi(getenv("TRD_CHAIN_THREAD")) != 0);
  if (offsets) {
    launch_offsets(c, bp, s, true);
  } else {
    static_assert(offsetof(DevScalars, amax_b) == offsetof(DevScalars, amax_a) + 4, "adjacent maxima");
    cudaMemsetAsync(&c.sc->amax_a, 0, 2 * sizeof(unsigned int), s);
  }
  if (bp.p > 0) {
    if (c.rbucket <= 16 && warp_chains)
      TRD_PDL((mid_warp_kernel<16, 8>), grid_for(bp.nL * 32), 256, 0, s, a, c.idx, c.Z, c.mid);
    else if (c.rbucket <= 32 && warp_chains)
      TRD_PDL((mid_warp_kernel<32, 4>), grid_for(bp.nL * 32, 128), 128, 0, s, a, c.idx, c.Z, c.mid);
    else if (c.rbucket <= 16) TRD_PDL(mid_kernel<16>, grid_for(bp.nL * bp.rk1), 256, 0, s, a, c.idx, c.Z, c.mid);
    else if (c.rbucket <= 32) TRD_PDL(mid_kernel<32>, grid_for(bp.nL * bp.rk1), 256, 0, s, a, c.idx, c.Z, c.mid);
    else TRD_PDL(mid_kernel<128>, grid_for(bp.nL * bp.rk1), 128, 0, s, a, c.idx, c.Z, c.mid);
    c.launches++;
  }
  if (c.rbucket <= 16 && warp_chains)
    TRD_PDL((rgt_warp_kernel<16, 8>), grid_for(bp.ncols * 32), 256, 0, s, a, c.idx, c.Z, c.rgtT, c.sc);
  else if (c.rbucket <= 32 && warp_chains)
    TRD_PDL((rgt_warp_kernel<32, 4>), grid_for(bp.ncols * 32, 128), 128, 0, s, a, c.idx, c.Z, c.rgtT, c.sc);
  else if (c.rbucket <= 16) TRD_PDL(rgt_kernel<16>, grid_for(bp.ncols * bp.rs), 256, 0, s, a, c.idx, c.Z, c.rgtT, c.sc);
  else if (c.rbucket <= 32) TRD_PDL(rgt_kernel<32>, grid_for(bp.ncols * bp.rs), 256, 0, s, a, c.idx, c.Z, c.rgtT, c.sc);
  else TRD_PDL(rgt_kernel<128>, grid_for(bp.ncols * bp.rs), 128, 0, s, a, c.idx, c.Z, c.rgtT, c.sc);
  c.launches++;
}

void launch_lft(Context& c, const BlockPlan& bp, const float* Zsrc_k, int src_is_h, float* out,
                cudaStream_t s) {
  PlanArgs a = make_plan_args(c, bp);
  if (bp.rows && bp.p > 0) {
    const size_t smem = (size_t)(bp.rk * (bp.rk1 + 1) + kLftJ * bp.rk1 * bp.rs) * sizeof(float);
    if (smem <= 200 * 1024) {
      cudaFuncSetAttribute(lft_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const dim3 grid((unsigned)(bp.nrows / bp.nL), (unsigned)((bp.nL + kLftJ - 1) / kLftJ));
      lft_rows_kernel<<<grid, 256, smem, s>>>(a, src_is_h ? nullptr : Zsrc_k, src_is_h ? c.h : nullptr, c.mid, out);
      c.launches++;
      return;
    }
  }
  if (c.rbucket <= 16)
    lft_kernel<16><<<grid_for(bp.nrows * bp.rk), 256, 0, s>>>(a, src_is_h ? nullptr : Zsrc_k,
                                                              src_is_h ? c.h : nullptr, c.mid, out);
  else if (c.rbucket <= 32)
    lft_kernel<32><<<grid_for(bp.nrows * bp.rk), 256, 0, s>>>(a, src_is_h ? nullptr : Zsrc_k,
                                                              src_is_h ? c.h : nullptr, c.mid, out);
  else
    lft_kernel<128><<<grid_for(bp.nrows * bp.rk), 128, 0, s>>>(a, src_is_h ? nullptr : Zsrc_k,
                                                               src_is_h ? c.h : nullptr, c.mid, out);
  c.launches++;
}

void launch_pass1(Context& c, const BlockPlan& bp, int stats_only, cudaStream_t s) {
  if (stats_only) launch_pass_t<false, true>(c, bp, s);
  else launch_pass_t<false, false>(c, bp, s);
}

void launch_pass2(Context& c, const BlockPlan& bp, cudaStream_t s) {
  launch_pass_t<true, false>(c, bp, s);
}

void launch_reduce_d(Context& c, const BlockPlan& bp, cudaStream_t s) {
  const int64_t Ik = bp.nrows / bp.nL, Ik_tot = c.dims[bp.k];
  const int64_t ncta = bp.grid_x * bp.nsplit;
  if (bp.rows) {                       // warp-per-row SIMT pass: D rows in contrib, per-CTA stats
    launch_reduce_d_contrib(c, bp, bp.rows_nsplit, bp.nrows, bp.rows_grid, s);
    return;
  }
  if (bp.big && bp.R2 > 0) {           // D rows of the SIMT pass in contrib ([nsplit][nrows][KP])
    launch_reduce_d_contrib(c, bp, bp.nsplit, bp.nrows, Ik * ncta, s);
    return;
  }
  if (bp.R2 > 0 && Ik < Ik_tot) cudaMemsetAsync(c.dvec, 0, (size_t)(Ik_tot * bp.R2) * sizeof(double), s);
  reduce_d_kernel<<<(unsigned)(Ik + 1), 256, 0, s>>>(c.dpart, c.spart, ncta, bp.R2, Ik, c.dvec,
                                                      bp.R2 > 0 ? c.sc : nullptr, bp.k, bp.ik0, Ik_tot);
  c.launches++;
}

// block statistics from the (allreduced) dvec tail
void launch_block_stats(Context& c, const BlockPlan& bp, cudaStream_t s) {
  const int64_t Ik = c.dims[bp.k];                     // dvec rows: all of I_k
  block_scalars_kernel<<<1, 32, 0, s>>>(c.dvec, Ik, bp.R2, nullptr, c.sc, c.stats, bp.k, 0.0, 0);
  c.launches++;
}

void launch_reduce_den(Context& c, const BlockPlan& bp, cudaStream_t s) {
  const int64_t Ik = bp.nrows / bp.nL;                 // plan rows (pass-2 partials)
  const int64_t ncta = bp.grid_x * bp.nsplit;
  const int64_t nden = bp.use_tc ? (int64_t)bp.tc_grid : bp.rows ? (int64_t)bp.rows_grid : Ik * ncta;
  reduce_den_kernel<<<1, 256, 0, s>>>(c.denpart, nden, c.numpart, c.dims[bp.k], c.red_ws);
  c.launches++;
}

void launch_q(Context& c, int k, cudaStream_t s) {
  const int r0 = c.ranks[k], r1 = c.ranks[(k + 1) % c.N];
  if (r0 * r1 > kBigR2) {                   // large-rank path: Zd^T Zd by dgemm, permuted
    big_q(c, k, s);                         // (a failure sets the context's sticky status)
    return;
  }
  TRD_PDL(q_kernel, grid_for((int64_t)r0 * r0 * r1 * r1 * 32), 256, 0, s, c.Z + c.zoff[k], c.dims[k], r0, r1,
                                                                      c.Q + c.qoff[k]);
  c.launches++;
}

// Q_m over a subset of slices (the 'local scaled term' ablation arm: the Gram of the
// sampled cores (Z_m)_{I_m}): Q[(a r + a'), (b r' + b')] = sum_{i in idx} Z(i)[a][b] Z(i)[a'][b']
__global__ void q_idx_kernel(const float* __restrict__ Zk, const int* __restrict__ idx, int64_t n_idx, int r0,
                             int r1, double* __restrict__ Qk) {
  const int n0 = r0 * r0, n1 = r1 * r1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n0 * n1; t += gridDim.x * blockDim.x) {
    const int row = t / n1, col = t % n1;
    const int a = row / r0, ap = row % r0, b = col / r1, bp = col % r1;
    double acc = 0.0;
    for (int64_t q = 0; q < n_idx; ++q) {
      const float* S = Zk + (int64_t)idx[q] * r0 * r1;
      acc += (double)S[a * r1 + b] * (double)S[ap * r1 + bp];
    }
    Qk[t] = acc;
  }
}

void launch_q_sampled(Context& c, const BlockPlan& bp, cudaStream_t s) {
  for (int m = 0; m < c.N; ++m) {
    if (m == bp.k) continue;
    const int r0 = c.ranks[m], r1 = c.ranks[(m + 1) % c.N];
    q_idx_kernel<<<grid_for((int64_t)r0 * r0 * r1 * r1), 256, 0, s>>>(c.Z + c.zoff[m], c.idx + c.idx_off[m], bp.s[m],
                                                                       r0, r1, c.Qloc + c.qoff[m]);
    c.launches++;
  }
}

__global__ void identity_kernel(double* __restrict__ M, int n, DevScalars* __restrict__ sc) {
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->h_lam = 0.0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n * n; t += gridDim.x * blockDim.x)
    M[t] = (t / n == t % n) ? 1.0 : 0.0;
}

// M = I: h = d M = d (the 'gradient descent' ablation arm)
void launch_identity_op(Context& c, const BlockPlan& bp, cudaStream_t s) {
  if (bp.lib_solve) return;            // (big_h: h = d)
  identity_kernel<<<grid_for((int64_t)bp.R2 * bp.R2), 256, 0, s>>>(c.Mop, bp.R2, c.sc);
  c.launches++;
}

void launch_phi(Context& c, const BlockPlan& bp, const double* C, double* G, cudaStream_t s) {
  phi_kernel<<<grid_for((int64_t)bp.R2 * bp.R2), 256, 0, s>>>(C, bp.rk, bp.rk1, G);
  c.launches++;
}

void launch_gram(Context& c, const BlockPlan& bp, cudaStream_t s, const double* Qsrc, double* Gout) {
  const int N = c.N, k = bp.k;
  if (c.has_big) {                     // (cuBLAS loaded: every chain by dgemm, cheaper order)
    big_gram(c, bp, s, Qsrc, Gout);
    return;
  }
  // C = Q_{k+1} Q_{k+2} ... Q_{k-1}
  const double* cur = Qsrc + c.qoff[(k + 1) % N];
  int m_rows = bp.rk1 * bp.rk1;
  double* bufs[2] = {c.chain_ws, c.chain_ws + c.chain_half};
  int which = 0;
  for (int q = 2; q < N; ++q) {
    const int mm = (k + q) % N;
    const int qcols = c.ranks[(mm + 1) % N] * c.ranks[(mm + 1) % N];
    const int qin = c.ranks[mm] * c.ranks[mm];
    dim3 grid((qcols + 15) / 16, (m_rows + 15) / 16);
    matmul_f64_kernel<<<grid, dim3(16, 16), 0, s>>>(cur, Qsrc + c.qoff[mm], bufs[which], m_rows, qcols, qin);
    c.launches++;
    cur = bufs[which];
    which ^= 1;
  }
  phi_kernel<<<grid_for((int64_t)bp.R2 * bp.R2), 256, 0, s>>>(cur, bp.rk, bp.rk1, Gout);
  c.launches++;
}

template <bool PRE_IP>
static void launch_gj4(int np, const double* G, int n, double lam, double* Mop, DevScalars* sc, cudaStream_t s) {
  switch (np) {
    case 16: gj4_solve_kernel<2, 1, PRE_IP><<<1, 256, 0, s>>>(G, n, lam, Mop, sc); break;
    case 32: gj4_solve_kernel<4, 1, PRE_IP><<<1, 256, 0, s>>>(G, n, lam, Mop, sc); break;
    case 48: gj4_solve_kernel<6, 2, PRE_IP><<<1, 256, 0, s>>>(G, n, lam, Mop, sc); break;
    case 64: gj4_solve_kernel<8, 2, PRE_IP><<<1, 256, 0, s>>>(G, n, lam, Mop, sc); break;
    case 80:
    case 96: gj4_solve_kernel<12, 3, PRE_IP><<<1, 256, 0, s>>>(G, n, lam, Mop, sc); break;
    default: gj4_solve_kernel<16, 4, PRE_IP><<<1, 256, 0, s>>>(G, n, lam, Mop, sc); break;
  }
}

// 16 warps (512 threads, half the block per thread): TRD_SOLVE=6
static void launch_gj4_w16(int np, const double* G, int n, double lam, double* Mop, DevScalars* sc, cudaStream_t s) {
  switch (np) {
    case 16:
    case 32: gj4_solve_kernel<2, 1, false, 16><<<1, 512, 0, s>>>(G, n, lam, Mop, sc); break;
    case 48:
    case 64: gj4_solve_kernel<4, 2, false, 16><<<1, 512, 0, s>>>(G, n, lam, Mop, sc); break;
    case 80:
    case 96: gj4_solve_kernel<6, 3, false, 16><<<1, 512, 0, s>>>(G, n, lam, Mop, sc); break;
    default: gj4_solve_kernel<8, 4, false, 16><<<1, 512, 0, s>>>(G, n, lam, Mop, sc); break;
  }
}

void launch_solve(Context& c, const BlockPlan& bp, cudaStream_t s, const double* G) {
  const int n = bp.R2;
  if (bp.lib_solve) {                  // Cholesky of G + lambda I (cuSOLVER); h in big_h
    big_factor(c, bp, s, G);
    return;
  }
  // Default: the chunked owner-resolved register kernel for every R^2 <= 128 (R^2 = 100: 71 vs
  // 103 us per launch for gj3; 50-sweep lines C4 0.752 -> 0.648, C3 0.583 -> 0.520, C5a 1.941 ->
  // 1.927 ms per sweep against the previous default of gj2 for R^2 <= 48 and gj3 above).
  // On 16 warps (R^2 = 100: 67.4 vs 71.2 us per launch, C4 0.648 -> 0.627 ms per sweep; C1 / C2 /
  // C3 / C5a within noise of 8 warps, 50-sweep lines).
  // TRD_SOLVE=0 / 2 / 3 / 4: gj3 / the one-dimensional gj2 / the blocked shared-memory kernel /
  // gj4 on 8 warps (A/B).
  const int solve_sel = getenv("TRD_SOLVE") ? atoi(getenv("TRD_SOLVE")) : 6;
  if (n <= 128 && solve_sel == 3) {
    const int smem = (int)((size_t)n * (n | 1) * sizeof(double));
    static uint64_t gjb_attr = 0;
    if (first_on_device(gjb_attr))
      cudaFuncSetAttribute(gjb_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 129 * 8);
    gjb_solve_kernel<<<1, 256, smem, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc);
    c.launches++;
    return;
  }
  // (a 32-warp variant, 4 x 4 blocks per thread, measured slower: R^2 = 100 122 vs 103 us, C4
  //  0.857 vs 0.773 ms per sweep -- barrier and padding cost outweigh the extra latency hiding)
  if (n <= 128 && solve_sel == 0) {    // 2-D register Gauss-Jordan (NU x NV blocks per thread)
    const int np = (n + 15) / 16 * 16;
    switch (np) {
      case 16: gj3_solve_kernel<2, 1><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 32: gj3_solve_kernel<4, 1><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 48: gj3_solve_kernel<6, 2><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 64: gj3_solve_kernel<8, 2><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 80: gj3_solve_kernel<10, 3><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 96: gj3_solve_kernel<12, 3><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 112: gj3_solve_kernel<14, 4><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      default: gj3_solve_kernel<16, 4><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
    }
    c.launches++;
    return;
  }
  if (n <= 128 && (solve_sel == 4 || solve_sel == 5 || solve_sel == 6)) {   // owner-resolved chunked steps
    const int np = (n + 15) / 16 * 16;
    if (solve_sel == 6) {
      launch_gj4_w16(np, G, n, c.cfg.lambda_rel, c.Mop, c.sc, s);
      c.launches++;
      return;
    }
    // (TRD_SOLVE=5: the next pivot's reciprocal published ahead by its owner -- measured slower,
    //  R^2 = 100 79.6 vs 71.5 us, C4 0.670 vs 0.652 ms per sweep: the division was not the chain)
    if (solve_sel == 5) launch_gj4<true>(np, G, n, c.cfg.lambda_rel, c.Mop, c.sc, s);
    else launch_gj4<false>(np, G, n, c.cfg.lambda_rel, c.Mop, c.sc, s);
    c.launches++;
    return;
  }
  if (n <= 128 && solve_sel == 2) {    // (A/B: the one-dimensional register kernel)
    const int np = (n + 15) / 16 * 16;
    switch (np) {
      case 16: gj2_solve_kernel<16><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 32: gj2_solve_kernel<32><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 48: gj2_solve_kernel<48><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 64: gj2_solve_kernel<64><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 80: gj2_solve_kernel<80><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 96: gj2_solve_kernel<96><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      case 112: gj2_solve_kernel<112><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
      default: gj2_solve_kernel<128><<<1, 256, 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc); break;
    }
    c.launches++;
    return;
  }
  if (n <= kGjMaxN) {                  // (TRD_SOLVE=1: the round-1 Gauss-Jordan kernel, A/B runs)
    const size_t gneed = (size_t)2 * n * n * sizeof(double);
    static uint64_t gj_attr = 0;
    const int maxs = (int)((size_t)2 * kGjMaxN * kGjMaxN * sizeof(double));
    if (first_on_device(gj_attr)) {
      cudaFuncSetAttribute(gj_solve_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs);
      cudaFuncSetAttribute(gj_solve_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs);
      cudaFuncSetAttribute(gj_solve_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs);
      cudaFuncSetAttribute(gj_solve_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs);
    }
    const int nb = (n + 31) / 32;
    if (nb == 1) gj_solve_kernel<1><<<1, 1024, gneed, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc);
    else if (nb == 2) gj_solve_kernel<2><<<1, 1024, gneed, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc);
    else if (nb == 3) gj_solve_kernel<3><<<1, 1024, gneed, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc);
    else gj_solve_kernel<4><<<1, 1024, gneed, s>>>(G, n, c.cfg.lambda_rel, c.Mop, c.sc);
    c.launches++;
    return;
  }
  const size_t need = (size_t)2 * n * n * sizeof(double);
  const int use_smem = need <= 200 * 1024;
  static uint64_t attr_set = 0;
  if (first_on_device(attr_set))
    cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  solve_kernel<<<1, kSolveThreads, use_smem ? need : 0, s>>>(G, n, c.cfg.lambda_rel, c.Mop,
                                                             c.chol_ws, use_smem, c.sc);
  c.launches++;
}

void launch_h(Context& c, const BlockPlan& bp, cudaStream_t s) {
  if (bp.lib_solve) {
    big_h(c, bp, s);
    return;
  }
  const int64_t Ik = c.dims[bp.k];                     // h of every i_k (replicated update)
  TRD_PDL(h_kernel, (unsigned)Ik, 256, 0, s, c.dvec, c.Mop, bp.R2, c.h, c.numpart, c.sc);
  c.launches++;
}

void launch_block_tail(Context& c, const BlockPlan& bp, cudaStream_t s) {
  const int64_t Ik = c.dims[bp.k];
  const int64_t ncta = bp.grid_x * bp.nsplit;
  const int64_t nden = bp.use_tc ? (int64_t)bp.tc_grid : bp.rows ? (int64_t)bp.rows_grid : (bp.nrows / bp.nL) * ncta;
  const int64_t tot = Ik * bp.rk * bp.rk1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, (int64_t)c.num_sm));
  TRD_PDL(block_tail_kernel, grid, 256, 0, s, c.denpart, nden, c.numpart, Ik, c.red_ws, c.dvec, Ik, bp.R2, c.sc, c.stats, bp.k,
                                       c.cfg.step, c.Z + c.zoff[bp.k], c.h, bp.rk, bp.rk1);
  c.launches++;
}

void launch_update(Context& c, const BlockPlan& bp, cudaStream_t s) {
  const int64_t Ik = c.dims[bp.k];
  block_scalars_kernel<<<1, 32, 0, s>>>(c.dvec, Ik, bp.R2, c.red_ws, c.sc, c.stats, bp.k,
                                        c.cfg.step, 1);
  c.launches++;
  update2_kernel<<<grid_for(Ik * bp.R2), 256, 0, s>>>(c.Z + c.zoff[bp.k], c.h, Ik, bp.rk, bp.rk1,
                                                      c.cfg.step, c.sc);
  c.launches++;
}

// Replica consistency (world > 1): a 64-bit checksum of the cores' bit patterns
// (order-independent: a modular sum of hashed (position, bits) words), split into 32-bit halves
// h and stored as [h_lo, h_hi, -h_lo, -h_hi]; after an allreduce-MAX the ranks agree iff
// max(h) == -max(-h) for both halves.
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
__global__ void core_checksum_kernel(const float* __restrict__ Z, int64_t n, unsigned long long* __restrict__ acc) {
  unsigned long long h = 0ull;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    h += mix64(((unsigned long long)t << 32) ^ __float_as_uint(Z[t]));
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, h);
}
__global__ void checksum_split_kernel(const unsigned long long* __restrict__ acc, double* __restrict__ chk) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long h = *acc;
  chk[0] = (double)(h & 0xffffffffull);
  chk[1] = (double)(h >> 32);
  chk[2] = -chk[0];
  chk[3] = -chk[1];
}
__global__ void replica_check_kernel(const double* __restrict__ chk, DevScalars* sc, DevStats* stats) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned int bad = (chk[0] != -chk[2]) || (chk[1] != -chk[3]);
  stats[sc->slot].replica_mismatch = bad;
  if (bad) sc->replica_bad = 1;
}

void launch_core_checksum(Context& c, cudaStream_t s) {
  cudaMemsetAsync(c.chk_acc, 0, sizeof(unsigned long long), s);
  const int64_t n = c.zoff[c.N];
  core_checksum_kernel<<<grid_for(n), 256, 0, s>>>(c.Z, n, c.chk_acc);
  checksum_split_kernel<<<1, 32, 0, s>>>(c.chk_acc, c.chk);
  c.launches += 2;
}

void launch_replica_check(Context& c, cudaStream_t s) {
  replica_check_kernel<<<1, 32, 0, s>>>(c.chk, c.sc, c.stats);
  c.launches++;
}

void launch_sweep_begin(Context& c, cudaStream_t s) {
  sweep_begin_kernel<<<1, 32, 0, s>>>(c.sc, c.stats);
  c.launches++;
}

void launch_sweep_end(Context& c, cudaStream_t s) {
  const int n = c.N - 1;
  const int rk = c.ranks[n], rk1 = c.ranks[0];
  const int64_t In = c.dims[n];
  double* T = c.chain_ws;     // In x R2 (<= chain_ws capacity, checked at init)
  dt_T_kernel<<<dim3((unsigned)In, (unsigned)((rk * rk1 + 127) / 128)), 128, 0, s>>>(c.Z + c.zoff[n], In, rk, rk1,
                                                                                      c.G_last, T);
  dt_D_kernel<<<grid_for(In * In), 256, 0, s>>>(c.Z + c.zoff[n], In, rk, rk1, T, c.Dcur);
  sweep_end_kernel<<<1, 1024, 0, s>>>(c.Dcur, c.Dprev, In * In, c.sc, c.stats,
                                      c.cfg.sigma_mode, c.cfg.sigma_theta, c.cfg.sigma_min);
  c.launches += 3;
}

void launch_sigma0(Context& c, cudaStream_t s) {
  // dvec[Ik*R2 .. +3] of the stats-only full pass hold [sum_e2, welsch, n]; the caller
  // reduced them into red_ws[0..2] (and ran the R21 select in MAD mode)
  sigma0_kernel<<<1, 32, 0, s>>>(c.red_ws, c.sc, c.cfg.sigma_theta, c.cfg.sigma_min,
                                 c.cfg.sigma_mode == TRD_SIGMA_MAD ? 1 : 0);
  c.launches++;
}

void launch_eabs_advance(Context& c, const TcStage& st, cudaStream_t s) {
  eabs_advance_kernel<<<1, 32, 0, s>>>(c.sc, st.tbase + st.n_tiles);
  c.launches++;
}

void launch_mad_hist(Context& c, int level, cudaStream_t s) {
  const int grid = c.num_sm * 3;           // (level 0: three 64 KB CTAs per SM)
  static uint64_t attr = 0;
  const size_t sm0 = (size_t)kMadWarps * kMadBins0 * 4;
  if (first_on_device(attr))
    cudaFuncSetAttribute(mad_hist_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0);
  if (level == 0) {
    cudaMemsetAsync(c.mhist, 0, kMadHist * sizeof(double), s);
    mad_hist_kernel<0><<<grid, kMadThreads, sm0, s>>>(c.eabs, c.sc, c.mhist);
  } else if (level == 1) {
    mad_hist_kernel<1><<<grid, kMadThreads, 2 * kMadBins1 * 4, s>>>(c.eabs, c.sc, c.mhist);
  } else {
    mad_hist_kernel<2><<<grid, kMadThreads, 2 * kMadBins2 * 4, s>>>(c.eabs, c.sc, c.mhist);
  }
  c.launches++;
}

void launch_mad_scan(Context& c, int level, cudaStream_t s) {
  if (level == 0) mad_scan_kernel<0><<<1, 1024, 0, s>>>(c.mhist, c.sc);
  else if (level == 1) mad_scan_kernel<1><<<1, 1024, 0, s>>>(c.mhist, c.sc);
  else mad_scan_kernel<2><<<1, 1024, 0, s>>>(c.mhist, c.sc);
  c.launches++;
}

void launch_reconstruct(Context& c, const int64_t* lin, int64_t n, float* out, cudaStream_t s) {
  ReconArgs a;
  a.N = c.N;
  for (int m = 0; m < c.N; ++m) a.dims[m] = c.dims[m];
  for (int m = 0; m <= c.N; ++m) { a.ranks[m] = c.ranks[m % c.N]; a.zoff[m] = c.zoff[m]; }
  if (c.rbucket <= 16) recon_kernel<16><<<grid_for(n), 256, 0, s>>>(a, c.Z, lin, n, out);
  else if (c.rbucket <= 32) recon_kernel<32><<<grid_for(n), 256, 0, s>>>(a, c.Z, lin, n, out);
  else recon_kernel<128><<<grid_for(n), 128, 0, s>>>(a, c.Z, lin, n, out);
  c.launches++;
}

void launch_error(Context& c, const float* ref, const uint32_t* eval_bits, double* out6,
                  cudaStream_t s) {
  const BlockPlan& bp = c.full_plan;
  PassArgs a = make_pass_args(c, bp);
  const int nb = 148 * 4;
  error_kernel<<<nb, 256, 0, s>>>(a, ref, eval_bits, c.dpart);
  error_reduce_kernel<<<1, 256, 0, s>>>(c.dpart, nb, out6);
  c.launches += 2;
}

__global__ void count_bits_kernel(const uint32_t* __restrict__ mask, int64_t nw, int64_t nbits,
                                  unsigned long long* __restrict__ out) {
  unsigned long long cnt = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nw; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = mask[t];
    const int64_t tail = nbits - t * 32;
    if (tail < 32) w &= (1u << tail) - 1u;
    cnt += __popc(w);
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, cnt);
}

void launch_count_bits(Context& c, unsigned long long* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
  count_bits_kernel<<<grid_for(c.n_words), 256, 0, s>>>(c.mask, c.n_words, c.n_local, out);
  c.launches++;
}

// max |x| over the observed values (P-operand bound of the tensor-core passes)
__global__ void amax_obs_kernel(const float* __restrict__ values, const uint32_t* __restrict__ mask, int64_t n,
                                int packed, DevScalars* __restrict__ sc) {
  float amax = 0.f;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (!packed && !((mask[t >> 5] >> (t & 31)) & 1u)) continue;
    const float v = fabsf(values[t]);
    if (v == v) amax = fmaxf(amax, v);
  }
  block_amax(amax, &sc->amax_x);
}

void launch_amax_obs(Context& c, cudaStream_t s) {
  cudaMemsetAsync(&c.sc->amax_x, 0, sizeof(unsigned int), s);
  const int64_t n = c.packed ? c.n_values : c.n_local;
  amax_obs_kernel<<<grid_for(n), 256, 0, s>>>(c.values, c.mask, n, c.packed, c.sc);
  c.launches++;
}

// mask_same = (mask == stage_mask) over all words (set to 1 before), then stage_mask <- mask
__global__ void mask_compare_kernel(const uint32_t* __restrict__ m, const uint32_t* __restrict__ ref, int64_t nw,
                                    int* __restrict__ same) {
  bool diff = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nw; t += (int64_t)gridDim.x * blockDim.x)
    diff |= m[t] != ref[t];
  if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) *same = 0;
}
__global__ void mask_copy_kernel(const uint32_t* __restrict__ m, uint32_t* __restrict__ ref, int64_t nw,
                                 DevScalars* __restrict__ sc) {
  if (sc->mask_same) return;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nw; t += (int64_t)gridDim.x * blockDim.x)
    ref[t] = m[t];
}
// a new mask generation (after the copy: every layout built before is stale)
__global__ void mask_gen_kernel(DevScalars* sc) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && !sc->mask_same) sc->mask_gen += 1;
}

void launch_mask_compare(Context& c, cudaStream_t s) {
  cudaMemsetAsync(&c.sc->mask_same, 1, sizeof(int), s);          // nonzero: same (until a difference)
  mask_compare_kernel<<<grid_for(c.n_words), 256, 0, s>>>(c.mask, c.stage_mask, c.n_words, &c.sc->mask_same);
  mask_copy_kernel<<<grid_for(c.n_words), 256, 0, s>>>(c.mask, c.stage_mask, c.n_words, c.sc);
  mask_gen_kernel<<<1, 32, 0, s>>>(c.sc);
  c.launches += 3;
}

void launch_rank_prefix(Context& c, cudaStream_t s) {
  popc_kernel<<<grid_for(c.n_words), 256, 0, s>>>(c.mask, c.n_words, c.rank_prefix);
  c.launches++;
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.rank_prefix, c.rank_prefix, c.n_words, s);
  if (tmp > c.rp_tmp_bytes) {                 // once per context (no allocation per upload)
    if (c.rp_tmp) cudaFree(c.rp_tmp);
    c.rp_tmp = nullptr;
    c.rp_tmp_bytes = 0;
    if (cudaMalloc(&c.rp_tmp, tmp) == cudaSuccess) c.rp_tmp_bytes = tmp;
  }
  cub::DeviceScan::ExclusiveSum(c.rp_tmp, tmp, c.rank_prefix, c.rank_prefix, c.n_words, s);
  c.launches += 1;
}


}  // namespace trd

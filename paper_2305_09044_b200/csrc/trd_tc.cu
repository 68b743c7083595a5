// trd_tc.cu -- tcgen05 (5th-gen tensor core) pass kernels of the AWRTRD / SAWRTRD block.
//
// The working set of block k in GEMM form: rows = (i_k, j_L), cols = j_R,
// x_hat(row, col) = <Lft(row), Rgt(col)> over K = r_k r_s (Thm 1 P:61 with S = Mid Rgt).
// Pass 1 (Eq. 7 + Eq. 9/15):
//     S   = Lft . Rgt^T                       (tcgen05.mma, A = Lft in TMEM, B = Rgt in smem)
//     c   = P o W o (X - S),  W = exp(-E^2/2s^2)   (epilogue warps; only observed entries)
//     D  += c . Rgt                           (tcgen05.mma, A = c in TMEM)
//     d(i_k) += Mid(j_L) D(row)                (per-row contraction, fixed-order reduce)
// Pass 2 (Eq. 12/18):  T = Lft_h . Rgt^T, den += W T^2 (W staged by pass 1).
//
// Precision (R18): every fp32 operand a is split into fp16 a_hi + a_lo with
// a_lo = fp16(a - a_hi); products use hi.hi + hi.lo + lo.hi accumulated in fp32 in TMEM,
// which keeps the per-entry dot products at fp32-level accuracy.
//
// Stage sketch: per block, the working set is staged in tile order --
// for every (128-row, 64-column) tile the 64-bit observation mask of each row, the row's
// offset into the tile's compacted values, and the observed values themselves.  The pass
// kernels then read 8 B of mask and 4 B per observed entry, coalesced, and their epilogue
// visits only the set bits.  Sweep-invariant working sets (full index sets, e.g. C5b) are
// staged once and cached.
//
// Tiles: M = 128 rows (one TMEM lane and one epilogue thread per row), NT = 64 columns, K
// padded to KP (multiple of 16).  The B operand uses the canonical SWIZZLE_NONE core-matrix
// layout (8 rows x 16 B per 128-byte core matrix, core matrix (g, h) at (g*HK + h)*128 B,
// HK = KP/8); the same tile is the K-major B of S = A.B^T and the MN-major B of D += c.B.
#include <cstdio>
#include <cub/cub.cuh>
#include <cuda_fp16.h>

#include "trd_internal.cuh"

namespace trd {

constexpr int TC_M = 128;
constexpr int TC_NT = 64;
constexpr int TC_DUMP_STRIDE = 68;   // floats per row of the S/T dump buffer (16-B aligned rows)

// ---------------------------------------------------------------------------------------
// PTX wrappers (tcgen05, mbarrier, proxy fences, cp.async)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// non-suspending poll (for the latency-critical single MMA warp)
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
#if TRD_CHECKED
  uint32_t spins = 0;
  long long t0 = 0;
#endif
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(addr), "r"(phase) : "memory");
#if TRD_CHECKED
    if (!ok && (++spins & 4095u) == 0u) {   // watchdog (checked build)
      const long long now = clock64();
      if (spins == 4096u) t0 = now;
      else if (now - t0 > (1ll << 34)) { trd_check_fail(kChkHang); break; }
    }
#endif
  } while (!ok);
  trd_jitter();
}
// try_wait with an explicit suspend-time hint (ns): the thread sleeps until the phase
// completes or the hint elapses, instead of re-polling (keeps issue slots free for the MMA warp)
// Build with -DTRD_DEBUG_HANG=1 and run with TRD_DEBUG_HANG=1: a wait that spins for ~4 s
// reports its barrier (smem offset, parity, thread) -- debugging aid for the pipeline barriers
#ifndef TRD_DEBUG_HANG
#define TRD_DEBUG_HANG 0
#endif
__device__ int g_debug_hang;
__device__ int g_prog[160][24];     // per (block, warp): 1000 * tile + stage code
__device__ __noinline__ void mbar_hang_report(uint32_t addr, uint32_t phase) {
  printf("[trd hang] block %d thread %d waits on mbarrier smem+%u parity %u\n", blockIdx.x, threadIdx.x,
         addr & 0xFFFFFu, phase);
  if ((threadIdx.x & 31) == 0 && blockIdx.x < 160)
    printf("[trd prog] block %d warps 4-15: %d %d %d %d | %d %d %d %d | %d %d %d %d\n", blockIdx.x,
           g_prog[blockIdx.x][4], g_prog[blockIdx.x][5], g_prog[blockIdx.x][6], g_prog[blockIdx.x][7],
           g_prog[blockIdx.x][8], g_prog[blockIdx.x][9], g_prog[blockIdx.x][10], g_prog[blockIdx.x][11],
           g_prog[blockIdx.x][12], g_prog[blockIdx.x][13], g_prog[blockIdx.x][14], g_prog[blockIdx.x][15]);
}
#ifndef TRD_SLEEP_NS
#define TRD_SLEEP_NS 1000000u
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
#if TRD_DEBUG_HANG || TRD_CHECKED
  uint32_t spins = 0;
  long long t0 = 0;
#endif
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(addr), "r"(phase), "r"(TRD_SLEEP_NS) : "memory");
#if TRD_CHECKED
    if (!ok && (++spins & 255u) == 0u) {    // watchdog (checked build)
      const long long now = clock64();
      if (spins == 256u) t0 = now;
      else if (now - t0 > (1ll << 34)) { trd_check_fail(kChkHang); break; }
    }
#elif TRD_DEBUG_HANG
    if (!ok && g_debug_hang && (++spins & 255u) == 0u) {
      const long long now = clock64();
      if (spins == 256u) t0 = now;
      else if (now - t0 > (1ll << 33)) { mbar_hang_report(addr, phase); t0 = now + (1ll << 40); }
    }
#endif
  } while (!ok);
  trd_jitter();
}
#ifndef TRD_MBAR_SPIN
#define TRD_MBAR_SPIN 0
#endif
// wait for the phase with the given parity to complete.  TRD_MBAR_SPIN=1 polls with the
// non-suspending test_wait (hand-offs between the warp roles are latency critical);
// 0 uses try_wait (may suspend the thread for an implementation-defined time)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
#if TRD_DEBUG_HANG || TRD_CHECKED
  uint32_t spins = 0;
  long long t0 = 0;
#endif
  do {
#if TRD_MBAR_SPIN
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(addr), "r"(phase) : "memory");
#else
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(addr), "r"(phase) : "memory");
#endif
#if TRD_CHECKED
    if (!ok && (++spins & 4095u) == 0u) {   // watchdog (checked build)
      const long long now = clock64();
      if (spins == 4096u) t0 = now;
      else if (now - t0 > (1ll << 34)) { trd_check_fail(kChkHang); break; }
    }
#elif TRD_DEBUG_HANG
    if (!ok && g_debug_hang && (++spins & 4095u) == 0u) {
      const long long now = clock64();
      if (spins == 4096u) t0 = now;
      else if (now - t0 > (1ll << 33)) { mbar_hang_report(addr, phase); t0 = now + (1ll << 40); }
    }
#endif
  } while (!ok);
  trd_jitter();
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t ta, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(ta), "l"(db), "r"(idesc), "r"(acc));
}
// 32 lanes x 16 / 8 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// SWIZZLE_NONE shared-memory matrix descriptor (sm_100 version bit 46 = 1)
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::f16 instruction descriptor: F32 accumulate, F16 A/B, A K-major, B K- or MN-major
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int b_mn_major) {
  return (1u << 4) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t pack_half2(__half lo, __half hi) {
  return (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
}

// ---------------------------------------------------------------------------------------
// Operand packing
// ---------------------------------------------------------------------------------------
// a3 + the Lft half of the GEMM form, fused with the fp16 hi / lo split of
// the A operand: Lft(row)[a + r_k c] = sum_b X(i_k)[a][b] Mid(j_L)[b][c]  (p = 0: Lft = X(i_k)),
// X = core slice Z_k(i_k) (pass 1) or folded scaled gradient H(i_k) (pass 2).  One thread per
// (row, 8 consecutive kappa): 16-byte stores of hi and lo.  Same fp32 arithmetic order as
// lft_kernel (fmaf over b ascending).
struct LftArgs {
  int64_t nrows, nL, Ik;
  int64_t ik0;           // global i_k of plan row index 0 (k = shard mode)
  int rowmode, rk, rk1, rs, K, KP, p;
  const float* zk;       // Z_k[i][a][b]
  const double* hk;      // h[i][a + r_k b]
  const float* mid;      // Mid[jl][b][c]
  float* lscl;           // [row] 2^-E of the row's power-of-two scaling (tc_scale_exp)
  unsigned int* amax;    // pass 1: max |Lft| over all rows (P-operand bound), else nullptr
};
// CTA = one 128-row tile: the rows' X(i_k) and Mid(j_L) are staged in shared memory (row
// stride padded to an odd word count: conflict-free across rows), then thread (row, half)
// produces KP/2 consecutive kappa and stores them as 16-byte hi / lo vectors.
// (gmem = 1: ranks too large for the shared-memory stage; X and Mid are read from global memory)
__global__ void __launch_bounds__(256) tc_lft_pack_kernel(LftArgs a, int pass2, int64_t nrows_pad,
                                                          __half* __restrict__ dst, int gmem) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  extern __shared__ float lsm[];
  const int XS = a.rk * a.rk1, MS = a.rk1 * a.rs;
  const int XP = XS | 1, MP = MS | 1;                       // odd strides
  float* Xs = lsm;                                          // [128][XP]
  float* Ms = lsm + TC_M * XP;                              // [128][MP]
  const int tid = threadIdx.x;
  for (int64_t rt = blockIdx.x; rt * TC_M < nrows_pad; rt += gridDim.x) {
    // stage: threads 0-127 copy row r's X(i_k), threads 128-255 its Mid(j_L)
    if (!gmem) {
      const int r = tid & (TC_M - 1);
      const int64_t row = rt * TC_M + r;
      int64_t ik = 0, jl = 0;
      const bool ok = row < a.nrows;
      if (ok) {
        if (a.rowmode == 0) { ik = row / a.nL; jl = row - ik * a.nL; }
        else { jl = row / a.Ik; ik = row - jl * a.Ik; }
      }
      if (tid < TC_M) {
        float* xr = Xs + r * XP;
        if (pass2) {
          const double* hs = a.hk + (a.ik0 + ik) * XS;
          for (int aa = 0; aa < a.rk; ++aa)
            for (int b = 0; b < a.rk1; ++b) xr[aa * a.rk1 + b] = ok ? (float)__ldg(hs + aa + a.rk * b) : 0.f;
        } else {
          const float* zs = a.zk + (a.ik0 + ik) * XS;
          for (int e = 0; e < XS; ++e) xr[e] = ok ? __ldg(zs + e) : 0.f;
        }
      } else if (a.p > 0) {
        float* mr = Ms + r * MP;
        const float* ms = a.mid + jl * MS;
        for (int e = 0; e < MS; ++e) mr[e] = ok ? __ldg(ms + e) : 0.f;
      }
    }
    __syncthreads();
    {
      const int r = tid >> 1, hf = tid & 1;
      const int64_t row = rt * TC_M + r;
      const float* X = Xs + r * XP;
      const float* M = Ms + r * MP;
      const int kh = a.KP / 2;
      int64_t gik = 0, gjl = 0;                             // (gmem) this row's i_k, j_L
      if (gmem && row < a.nrows) {
        if (a.rowmode == 0) { gik = row / a.nL; gjl = row - gik * a.nL; }
        else { gjl = row / a.Ik; gik = row - gjl * a.Ik; }
      }
      auto xval = [&](int aa, int b) -> float {
        if (!gmem) return X[aa * a.rk1 + b];
        const int64_t base = (a.ik0 + gik) * XS;
        return pass2 ? (float)__ldg(a.hk + base + aa + a.rk * b) : __ldg(a.zk + base + aa * a.rk1 + b);
      };
      auto mval = [&](int b, int c) -> float { return gmem ? __ldg(a.mid + gjl * MS + b * a.rs + c) : M[b * a.rs + c]; };
      auto lft_val = [&](int kap) -> float {
        float v = 0.f;
        if (row < a.nrows && kap < a.K) {
          const int aa = kap % a.rk, c = kap / a.rk;
          if (a.p == 0) {
            v = xval(aa, c);
          } else {
            for (int b = 0; b < a.rk1; ++b) v = fmaf(xval(aa, b), mval(b, c), v);
          }
        }
        return v;
      };
      // the row's max |Lft| (both halves: partner lane tid ^ 1) -> power-of-two scale
      float amax = 0.f;
      for (int kap = hf * kh; kap < (hf + 1) * kh; ++kap) amax = fmaxf(amax, fabsf(lft_val(kap)));
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
      const int E = tc_scale_exp(amax);
      if (hf == 0 && row < nrows_pad) a.lscl[row] = ldexpf(1.f, -E);
      if (a.amax && hf == 0) amax_update(a.amax, amax);
      for (int k0 = hf * kh; k0 < (hf + 1) * kh; k0 += 8) {
        __half hh[8], ll[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float v = ldexpf(lft_val(k0 + e), E);
          hh[e] = __float2half_rn(v);
          ll[e] = __float2half_rn(v - __half2float(hh[e]));
        }
        uint4 hv, lv;
        hv.x = pack_half2(hh[0], hh[1]); hv.y = pack_half2(hh[2], hh[3]);
        hv.z = pack_half2(hh[4], hh[5]); hv.w = pack_half2(hh[6], hh[7]);
        lv.x = pack_half2(ll[0], ll[1]); lv.y = pack_half2(ll[2], ll[3]);
        lv.z = pack_half2(ll[4], ll[5]); lv.w = pack_half2(ll[6], ll[7]);
        *reinterpret_cast<uint4*>(dst + row * 2 * a.KP + k0) = hv;
        *reinterpret_cast<uint4*>(dst + row * 2 * a.KP + a.KP + k0) = lv;
      }
    }
    __syncthreads();
  }
}

// Generic ranks: a half-warp per row (16 lanes x 8 consecutive kappa cover KP <= 128), X(i_k)
// and Mid(j_L) read through L1 (no staging: every row is independent, so the grid is as
// large as the row count).  The row's max |Lft| (16-lane butterfly) gives its power-of-two
// scale; each lane stores its 8 kappa as 16-byte hi / lo vectors.  Same fp32 arithmetic order as
// lft_kernel (fmaf over b ascending).
__global__ void __launch_bounds__(256) tc_lft_pack_hw_kernel(LftArgs a, int pass2, int64_t nrows_pad,
                                                             __half* __restrict__ dst) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  const int lane = threadIdx.x & 31, sub = lane & 15;
  const unsigned hmask = 0xFFFFu << (lane & 16);
  const int XS = a.rk * a.rk1, MS = a.rk1 * a.rs;
  const int64_t nhw = ((int64_t)gridDim.x * blockDim.x) >> 4;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 4; row < nrows_pad; row += nhw) {
    int64_t ik = 0, jl = 0;
    const bool ok = row < a.nrows;
    if (ok) {
      if (a.rowmode == 0) { ik = row / a.nL; jl = row - ik * a.nL; }
      else { jl = row / a.Ik; ik = row - jl * a.Ik; }
    }
    const int64_t xb = (a.ik0 + ik) * XS;
    const float* M = a.mid + jl * MS;
    float v[8];
    float amax = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int kap = sub * 8 + e;
      float x = 0.f;
      if (ok && kap < a.K) {
        const int aa = kap % a.rk, c = kap / a.rk;
        if (a.p == 0) {
          x = pass2 ? (float)__ldg(a.hk + xb + aa + a.rk * c) : __ldg(a.zk + xb + aa * a.rk1 + c);
        } else {
          for (int b = 0; b < a.rk1; ++b) {
            const float xv = pass2 ? (float)__ldg(a.hk + xb + aa + a.rk * b) : __ldg(a.zk + xb + aa * a.rk1 + b);
            x = fmaf(xv, __ldg(M + b * a.rs + c), x);
          }
        }
      }
      v[e] = x;
      amax = fmaxf(amax, fabsf(x));
    }
    for (int o = 8; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(hmask, amax, o));
    const int E = tc_scale_exp(amax);
    if (sub == 0 && row < nrows_pad) a.lscl[row] = ldexpf(1.f, -E);
    if (a.amax) {                                   // max over the warp's two rows, then one update
      const float m2 = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 16));
      if (lane == 0) amax_update(a.amax, m2);
    }
    if (sub * 8 < a.KP) {
      __half hh[8], ll[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float x = ldexpf(v[e], E);
        hh[e] = __float2half_rn(x);
        ll[e] = __float2half_rn(x - __half2float(hh[e]));
      }
      uint4 hv, lv;
      hv.x = pack_half2(hh[0], hh[1]); hv.y = pack_half2(hh[2], hh[3]);
      hv.z = pack_half2(hh[4], hh[5]); hv.w = pack_half2(hh[6], hh[7]);
      lv.x = pack_half2(ll[0], ll[1]); lv.y = pack_half2(ll[2], ll[3]);
      lv.z = pack_half2(ll[4], ll[5]); lv.w = pack_half2(ll[6], ll[7]);
      *reinterpret_cast<uint4*>(dst + row * 2 * a.KP + sub * 8) = hv;
      *reinterpret_cast<uint4*>(dst + row * 2 * a.KP + a.KP + sub * 8) = lv;
    }
  }
}

// Large ranks (r_{k+1} >= 32, p > 0: the paper's [80, 80, 3, 20]): CTA per (i_k, 32 left
// indices jl); X(i_k) (r_k x r_{k+1}, padded rows) and the 32 Mid(jl) staged in shared memory,
// the 32 x K Lft rows computed into shared memory (fmaf over b ascending, as the half-warp
// kernel), then warp per row: max |Lft|, the power-of-two scale, fp16 hi / lo stores.  CTA
// (0, 0) also writes the padding rows [nrows, nrows_pad).
constexpr int kPackJ = 32;
__global__ void __launch_bounds__(256) tc_lft_pack_tile_kernel(LftArgs a, int pass2, int64_t nrows_pad,
                                                               __half* __restrict__ dst) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  extern __shared__ float psm[];
  const int rk = a.rk, rk1 = a.rk1, rs = a.rs, K = a.K, KP = a.KP, XS = rk1 + 1, MS = rk1 * rs, LS = K + 1;
  float* Xs = psm;                              // [rk][rk1 + 1]
  float* Ms = Xs + rk * XS;                     // [kPackJ][rk1][rs]
  float* Ls = Ms + kPackJ * MS;                 // [kPackJ][K + 1]
  const int64_t ik = blockIdx.x, jl0 = (int64_t)blockIdx.y * kPackJ;
  const int nj = (int)min((int64_t)kPackJ, a.nL - jl0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t xb = (a.ik0 + ik) * rk * rk1;
  for (int t = tid; t < rk * rk1; t += blockDim.x) {
    const int aa = t / rk1, b = t - aa * rk1;
    Xs[aa * XS + b] = pass2 ? (float)__ldg(a.hk + xb + aa + rk * b) : __ldg(a.zk + xb + t);
  }
  for (int t = tid; t < nj * MS; t += blockDim.x) Ms[t] = __ldg(a.mid + jl0 * MS + t);
  __syncthreads();
  for (int t = tid; t < nj * K; t += blockDim.x) {
    const int jj = t / K, kap = t - jj * K;
    const int aa = kap % rk, cc = kap / rk;
    const float* xr = Xs + aa * XS;
    const float* mc = Ms + jj * MS + cc;
    float x = 0.f;
    for (int b = 0; b < rk1; ++b) x = fmaf(xr[b], mc[b * rs], x);
    Ls[jj * LS + kap] = x;
  }
  __syncthreads();
  float wmax = 0.f;
  for (int jj = warp; jj < nj; jj += 8) {
    const int64_t jl = jl0 + jj;
    const int64_t row = a.rowmode == 0 ? jl + a.nL * ik : ik + a.Ik * jl;
    float amax = 0.f;
    for (int q = lane; q < K; q += 32) amax = fmaxf(amax, fabsf(Ls[jj * LS + q]));
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const int E = tc_scale_exp(amax);
    if (lane == 0) a.lscl[row] = ldexpf(1.f, -E);
    wmax = fmaxf(wmax, amax);
    for (int q = lane; q < KP; q += 32) {
      const float x = q < K ? ldexpf(Ls[jj * LS + q], E) : 0.f;
      const __half hh = __float2half_rn(x);
      dst[row * 2 * KP + q] = hh;
      dst[row * 2 * KP + KP + q] = __float2half_rn(x - __half2float(hh));
    }
  }
  if (a.amax && lane == 0) amax_update(a.amax, wmax);
  if (blockIdx.x == 0 && blockIdx.y == 0) {     // padding rows: zero operand, scale 1
    for (int64_t t = a.nrows * 2 * KP + tid; t < nrows_pad * 2 * KP; t += blockDim.x) dst[t] = __float2half_rn(0.f);
    for (int64_t r = a.nrows + tid; r < nrows_pad; r += blockDim.x) a.lscl[r] = 1.f;
  }
}

// Register-blocked variant for compile-time ranks (RK = r_k, RK1 = r_{k+1}, RS = r_s, p > 0):
// one thread per row holds X(i_k) (RK x RK1) and Mid(j_L) (RK1 x RS) and produces the whole
// row, Lft[a + RK c] = sum_b X[a][b] Mid[b][c] (fmaf over b ascending, as lft_kernel).
template <int RK, int RK1, int RS>
__global__ void __launch_bounds__(128, 4) tc_lft_pack_rb_kernel(LftArgs a, int pass2, int64_t nrows_pad,
                                                             __half* __restrict__ dst) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  constexpr int K = RK * RS;
  constexpr int KP = (K + 15) / 16 * 16;
  constexpr int ROWB = 2 * KP * 2;                 // bytes of one packed row (hi | lo)
  __shared__ __align__(16) unsigned char stage[128 * ROWB];
  for (int64_t row0 = blockIdx.x * (int64_t)blockDim.x; row0 < nrows_pad; row0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = row0 + threadIdx.x;
    float out[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) out[q] = 0.f;
    if (row < a.nrows) {
      int64_t ik, jl;
      if (a.rowmode == 0) { ik = row / a.nL; jl = row - ik * a.nL; }
      else { jl = row / a.Ik; ik = row - jl * a.Ik; }
      float X[RK][RK1], M[RK1][RS];
      if (pass2) {
        const double2* hs = reinterpret_cast<const double2*>(a.hk + (a.ik0 + ik) * (RK * RK1));   // h[a + RK b]
#pragma unroll
        for (int q = 0; q < RK * RK1 / 2; ++q) {
          const double2 v = __ldg(hs + q);
          X[(2 * q) % RK][(2 * q) / RK] = (float)v.x;
          X[(2 * q + 1) % RK][(2 * q + 1) / RK] = (float)v.y;
        }
      } else {
        const float4* zs = reinterpret_cast<const float4*>(a.zk + (a.ik0 + ik) * (RK * RK1));     // Z[a][b]
#pragma unroll
        for (int q = 0; q < RK * RK1 / 4; ++q) {
          const float4 v = __ldg(zs + q);
          reinterpret_cast<float*>(X)[4 * q] = v.x; reinterpret_cast<float*>(X)[4 * q + 1] = v.y;
          reinterpret_cast<float*>(X)[4 * q + 2] = v.z; reinterpret_cast<float*>(X)[4 * q + 3] = v.w;
        }
      }
      const float4* ms = reinterpret_cast<const float4*>(a.mid + jl * (RK1 * RS));
#pragma unroll
      for (int q = 0; q < RK1 * RS / 4; ++q) {
        const float4 v = __ldg(ms + q);
        reinterpret_cast<float*>(M)[4 * q] = v.x; reinterpret_cast<float*>(M)[4 * q + 1] = v.y;
        reinterpret_cast<float*>(M)[4 * q + 2] = v.z; reinterpret_cast<float*>(M)[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int aa = 0; aa < RK; ++aa)
#pragma unroll
        for (int c = 0; c < RS; ++c) {
          float v = 0.f;
#pragma unroll
          for (int b = 0; b < RK1; ++b) v = fmaf(X[aa][b], M[b][c], v);
          out[aa + RK * c] = v;
        }
    }
    // the row's power-of-two scale (tc_scale_exp): exact, keeps the fp16 split in range
    float amax = 0.f;
#pragma unroll
    for (int q = 0; q < KP; ++q) amax = fmaxf(amax, fabsf(out[q]));
    const int E = tc_scale_exp(amax);
    const float sc2 = ldexpf(1.f, E);
    if (row < nrows_pad) a.lscl[row] = ldexpf(1.f, -E);
    if (a.amax) {
      float m = amax;
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if ((threadIdx.x & 31) == 0) amax_update(a.amax, m);
    }
#pragma unroll
    for (int k0 = 0; k0 < KP; k0 += 8) {
      __half hh[8], ll[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v = out[k0 + e] * sc2;
        hh[e] = __float2half_rn(v);
        ll[e] = __float2half_rn(v - __half2float(hh[e]));
      }
      uint4 hv, lv;
      hv.x = pack_half2(hh[0], hh[1]); hv.y = pack_half2(hh[2], hh[3]);
      hv.z = pack_half2(hh[4], hh[5]); hv.w = pack_half2(hh[6], hh[7]);
      lv.x = pack_half2(ll[0], ll[1]); lv.y = pack_half2(ll[2], ll[3]);
      lv.z = pack_half2(ll[4], ll[5]); lv.w = pack_half2(ll[6], ll[7]);
      // row-major staging, 16-B chunks rotated by the row so a warp's stores hit all banks
      const int c0 = k0 / 8, cq = ROWB / 16;
      *reinterpret_cast<uint4*>(stage + threadIdx.x * ROWB + ((c0 + threadIdx.x) % cq) * 16) = hv;
      *reinterpret_cast<uint4*>(stage + threadIdx.x * ROWB + ((c0 + KP / 8 + threadIdx.x) % cq) * 16) = lv;
    }
    __syncthreads();
    // the block's rows are consecutive in dst: one contiguous, coalesced copy
    const int64_t nr = min((int64_t)blockDim.x, nrows_pad - row0);
    uint4* gdst = reinterpret_cast<uint4*>(dst + row0 * 2 * KP);
    const int cq = ROWB / 16;
    for (int q = threadIdx.x; q < nr * cq; q += blockDim.x) {
      const int r = q / cq, c = q - r * cq;
      gdst[q] = *reinterpret_cast<const uint4*>(stage + r * ROWB + ((c + r) % cq) * 16);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int64_t cm_offset(int r, int kap, int HK) {
  return ((int64_t)((r >> 3) * HK + (kap >> 3)) * 8 + (r & 7)) * 8 + (kap & 7);
}

// B (Rgt) core-matrix tiles: [col tile][hi | lo][64 x KP]
__global__ void tc_pack_cols_kernel(const float* __restrict__ rgtT, int64_t ncols, int K, int KP,
                                    int64_t ntiles, __half* __restrict__ dst, __half* __restrict__ dst2,
                                    const DevScalars* __restrict__ sc) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  const int HK = KP / 8;
  const float sc2 = ldexpf(1.f, tc_scale_exp(__uint_as_float(sc->amax_b)));   // B scaling
  const int64_t tot = ntiles * TC_NT * KP;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = t % (ntiles * TC_NT);
    const int kap = (int)(t / (ntiles * TC_NT));
    const float v = (col < ncols && kap < K) ? rgtT[(int64_t)kap * ncols + col] * sc2 : 0.f;
    const __half hi = __float2half_rn(v);
    const __half lo = __float2half_rn(v - __half2float(hi));
    const int64_t tile = col / TC_NT;
    const int64_t off = cm_offset((int)(col % TC_NT), kap, HK);
    __half* base = dst + tile * (2LL * TC_NT * KP);
    base[off] = hi;
    base[(int64_t)TC_NT * KP + off] = lo;
    // layout L2: K = 2 KP per column ([hi KP | lo KP]), core matrix (g, h') at (g * 2HK + h')
    __half* base2 = dst2 + tile * (2LL * TC_NT * KP);
    base2[cm_offset((int)(col % TC_NT), kap, 2 * HK)] = hi;
    base2[cm_offset((int)(col % TC_NT), KP + kap, 2 * HK)] = lo;
  }
}

// ---------------------------------------------------------------------------------------
// Stage sketch: tile-ordered mask bits, row offsets and compacted observed values
// ---------------------------------------------------------------------------------------
struct StageArgs {
  int64_t nrows, ncols, n_col_tiles, n_tiles;
  int64_t n_words;        // 32-bit words of the observation mask
  int packed;
  const int64_t* row_off;
  const int64_t* col_off;
  const uint32_t* mask;
  const uint32_t* rank_prefix;
  const float* values;
  uint64_t* tbits;        // [tile][128]
  uint16_t* troff;        // [tile][128]
  uint64_t* tcount;       // [tile]  padded counts (stage_bits)
  uint64_t* tbase;        // [tile + 1] their exclusive prefix (the scan; tile block starts)
  const int* gen_cur;     // sweep-invariant sketch: the current mask generation, and
  int* gen_layout;        //   the one this block's staged layout was built from (equal: only the
                          //   values are re-gathered); nullptr otherwise
  int32_t* perm;          // sweep-invariant sketch: value index of every staged slot (-1 padding)
  float* tvals;           // compacted values (tile blocks padded to 8 entries)
  uint16_t* tidx;         // entry list: (row in tile) * 64 + column, 0xFFFF = padding
  int64_t vcap;           // capacity of tvals / tidx / perm (checked build)
  // fibre windows (sampled mode 0 as the fastest column digit, 16 <= s0, I0 <= 128): columns
  // f s0 .. f s0 + s0 - 1 lie in one mode-0 fibre at base col_off[f s0] - idx0[0], at the
  // positions idx0[0..s0-1]; 0 = off
  int fib;
  int fib_s0;
  const int32_t* idx0;
  // row fibres: mode 0 sampled with s0 = 32 positions is the fastest row digit (nL % 32 == 0),
  // so the 32 rows of a warp are the sampled positions of one mode-0 fibre; 0 = off
  int rfib;
  // compaction tables of the sampled mode-0 positions (s0 <= 64; fib_pext): byte b of a fibre
  // window -> its sampled bits packed (tab[b * 256 + v]); sampled positions below byte b at
  // tab[4096 + b]; fib_nb = bytes of the window that hold positions (I0 / 8 rounded up)
  const uint8_t* ptab;
  int fib_nb;
};
constexpr int kPextTab = 16 * 256 + 16;

// ---- fibre windows: the I0 <= 128 observation bits of a mode-0 fibre starting at linear
// position lin0 as four aligned words (a0: bits 0-31 of the fibre, ...), from five raw words ----
struct FibWin {
  uint32_t a0, a1, a2, a3;   // aligned window (I0 <= 128 bits)
  uint32_t w0;           // first raw word (index lin0 >> 5) and the shift sh = lin0 & 31
  uint32_t sh;
};
__device__ __forceinline__ FibWin fib_window(const StageArgs& s, int64_t lin0);
__device__ __forceinline__ uint32_t fib_word(const FibWin& f, uint32_t q) {
  return q < 2 ? (q == 0 ? f.a0 : f.a1) : (q == 2 ? f.a2 : f.a3);
}

// The working-set tile (128 GEMM rows x 64 columns) reads the observation bits at linear
// positions row_off[row] + col_off[col].  Two structures make this cheap:
//  * column runs: consecutive columns with consecutive linear positions (mode 0 is the fastest
//    column digit) -> one funnel-shifted bit window per run and row;
//  * contiguous rows (k = 0: rows enumerate i_0 fastest): the 32 rows of a warp are one 32-bit
//    window per column; lane j extracts column j's window and a warp bit-matrix transpose
//    turns the columns into the rows' 64-bit masks.
// Sampled (RStS) index sets fall back to runs of length 1.
__device__ __forceinline__ uint32_t mask_word(const StageArgs& s, int64_t w) {
  return w < s.n_words ? __ldg(s.mask + w) : 0u;
}
// 32 bits of the mask starting at linear position lin
__device__ __forceinline__ uint32_t mask_bits32(const StageArgs& s, int64_t lin) {
  const int64_t w = lin >> 5;
  const uint32_t sh = (uint32_t)(lin & 31);
  const uint32_t lo = mask_word(s, w);
  const uint32_t hi = sh ? mask_word(s, w + 1) : 0u;
  return __funnelshift_r(lo, hi, sh);
}
// len (1..64) bits of the mask starting at linear position lin
__device__ __forceinline__ uint64_t mask_bits(const StageArgs& s, int64_t lin, int len) {
  const int64_t w = lin >> 5;
  const uint32_t sh = (uint32_t)(lin & 31);
  const uint32_t w0 = mask_word(s, w);
  const uint32_t w1 = (sh + len > 32) ? mask_word(s, w + 1) : 0u;
  const uint32_t w2 = (sh + len > 64) ? mask_word(s, w + 2) : 0u;
  uint64_t v = ((((uint64_t)w1) << 32) | w0) >> sh;
  if (sh) v |= ((uint64_t)w2) << (64 - sh);
  return len >= 64 ? v : (v & ((1ull << len) - 1ull));
}
// rank of linear position lin among the observed entries (packed value index)
__device__ __forceinline__ int64_t mask_rank(const StageArgs& s, int64_t lin) {
  const int64_t w = lin >> 5;
  return (int64_t)__ldg(s.rank_prefix + w) + __popc(__ldg(s.mask + w) & ((1u << (lin & 31)) - 1u));
}
__device__ __forceinline__ FibWin fib_window(const StageArgs& s, int64_t lin0) {
  const int64_t w = lin0 >> 5;
  FibWin f;
  f.sh = (uint32_t)(lin0 & 31);
  const uint32_t r0 = mask_word(s, w), r1 = mask_word(s, w + 1), r2 = mask_word(s, w + 2), r3 = mask_word(s, w + 3),
                 r4 = mask_word(s, w + 4);
  f.w0 = r0;
  f.a0 = __funnelshift_r(r0, r1, f.sh);
  f.a1 = __funnelshift_r(r1, r2, f.sh);
  f.a2 = __funnelshift_r(r2, r3, f.sh);
  f.a3 = __funnelshift_r(r3, r4, f.sh);
  return f;
}

// the sampled bits of a fibre window, packed in sampled order (s0 <= 64): one table lookup per
// window byte instead of one extraction per sampled position
__device__ __forceinline__ uint64_t fib_pext(const FibWin& f, const uint8_t* tab, const uint32_t* offw, int nb) {
  uint64_t r = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    if (b < nb) {
      const uint32_t w = b < 4 ? f.a0 : (b < 8 ? f.a1 : (b < 12 ? f.a2 : f.a3));
      const uint32_t v = (w >> (8 * (b & 3))) & 255u;
      r |= (uint64_t)tab[b * 256 + v] << ((offw[b >> 2] >> (8 * (b & 3))) & 255u);
    }
  }
  return r;
}
// (the tables are written by the sampler of the block, sampler_kernel, trd_kernels.cu)
// staging of block bp compacts fibre windows by table: a sampled mode 0 (s0 <= 64, I0 <= 128)
// as the fastest column digit, or (s0 = 32) as the fastest row digit
bool stage_uses_pext(const Context& c, const BlockPlan& bp) {
  if (!bp.use_tc || bp.explicit_cols || !c.ptab || getenv("TRD_NO_PEXT")) return false;
  if (!(bp.s[0] < c.dims[0] && c.dims[0] <= 128 && bp.s[0] <= 64)) return false;
  if (c.cfg.shard_mode == 0 && c.shard_end - c.shard_begin < c.dims[0]) return false;
  const bool col = bp.nright > 0 && bp.right[bp.rdig[0]] == 0 && bp.s[0] >= 16;
  const bool row = bp.k != 0 && bp.nleft > 0 && bp.left[bp.ldig[0]] == 0 && bp.s[0] == 32 && bp.nL % 32 == 0;
  return col || row;
}
// per CTA: the tables into shared memory, the byte offsets into four words
__device__ __forceinline__ void load_pext(const StageArgs& s, uint8_t* tabS, uint32_t* offw) {
  for (int i = threadIdx.x; i < kPextTab / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(tabS)[i] = __ldg(reinterpret_cast<const uint4*>(s.ptab) + i);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) offw[q] = reinterpret_cast<const uint32_t*>(tabS + 4096)[q];
}

// 32 x 32 bit-matrix transpose across a warp: in, lane i holds row i (bit j = element (i, j));
// out, lane i holds column i (bit j = element (j, i))
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  const uint32_t M[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int sft = 16 >> q;
    const uint32_t t = __shfl_xor_sync(0xffffffffu, x, sft);
    x = (lane & sft) ? ((x & ~M[q]) | ((t & ~M[q]) >> sft)) : ((x & M[q]) | ((t & M[q]) << sft));
  }
  return x;
}
// per tile: column offsets and the run-start mask (bit j: column j starts a run)
__device__ __forceinline__ void stage_tile_cols(const StageArgs& s, int64_t ct, int tid, int64_t* sco,
                                                uint32_t* sstart) {
  if (tid < TC_NT) {
    const int64_t col = ct * TC_NT + tid;
    sco[tid] = col < s.ncols ? s.col_off[col] : -1;
  }
  __syncthreads();
  if (tid < TC_NT) {
    const int64_t c0 = sco[tid];
    const bool start = tid == 0 || c0 < 0 || sco[tid - 1] < 0 || c0 != sco[tid - 1] + 1;
    const uint32_t b = __ballot_sync(0xffffffffu, start);
    if ((tid & 31) == 0) sstart[tid >> 5] = b;
  }
  __syncthreads();
}
// rows of this warp at most two contiguous ranges of linear positions (lanes [0, b) from
// baseA, lanes [b, 32) from baseB; b = 32: one range)?  Row digit orders put i_0 first, so a
// warp's rows break at most once (every dims[0] >= 32 rows)
struct WarpRows {
  int64_t baseA, baseB;
  int b;
};
__device__ __forceinline__ bool warp_row_segments(int64_t ro, int lane, WarpRows& w) {
  const int64_t prev = __shfl_up_sync(0xffffffffu, ro, 1);
  const uint32_t brk = __ballot_sync(0xffffffffu, lane > 0 && ro != prev + 1);
  if (!__all_sync(0xffffffffu, ro >= 0) || __popc(brk) > 1) return false;
  w.b = brk ? __ffs(brk) - 1 : 32;
  w.baseA = __shfl_sync(0xffffffffu, ro, 0);
  w.baseB = __shfl_sync(0xffffffffu, ro, w.b & 31);
  return true;
}
// the warp's 32 row bits of column offset co (bit r = row r)
__device__ __forceinline__ uint32_t warp_col_bits(const StageArgs& s, const WarpRows& w, int64_t co) {
  uint32_t a = mask_bits32(s, w.baseA + co);
  if (w.b < 32) a = (a & ((1u << w.b) - 1u)) | (mask_bits32(s, w.baseB + co) << w.b);
  return a;
}

__global__ void __launch_bounds__(128) stage_bits_kernel(StageArgs s) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  if (s.gen_cur && *s.gen_layout == *s.gen_cur) return;   // layout current (same mask): nothing to do
  __shared__ int64_t sco[TC_NT];
  __shared__ uint32_t sstart[2];
  __shared__ int wsum[4];
  __shared__ __align__(16) uint8_t tabS[kPextTab];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t offw[4] = {0u, 0u, 0u, 0u};
  if (s.ptab) load_pext(s, tabS, offw);
  for (int64_t tile = blockIdx.x; tile < s.n_tiles; tile += gridDim.x) {
    const int64_t rt = tile / s.n_col_tiles, ct = tile % s.n_col_tiles;
    stage_tile_cols(s, ct, tid, sco, sstart);
    const int64_t row = rt * TC_M + tid;
    const int64_t ro = row < s.nrows ? s.row_off[row] : -1;
    uint64_t bits = 0;
    WarpRows wr;
    if (s.rfib) {
      // row fibres: lane j packs column j's (and j + 32's) sampled bits of the warp's fibre
      // (one window each), then the transpose gives every row its 64 column bits
      if (__all_sync(0xffffffffu, ro >= 0)) {
        const int64_t fb0 = __shfl_sync(0xffffffffu, ro, 0) - s.idx0[0];
        const int64_t c0 = sco[lane], c1 = sco[lane + 32];
        const uint32_t w0 = c0 >= 0 ? (uint32_t)fib_pext(fib_window(s, fb0 + c0), tabS, offw, s.fib_nb) : 0u;
        const uint32_t w1 = c1 >= 0 ? (uint32_t)fib_pext(fib_window(s, fb0 + c1), tabS, offw, s.fib_nb) : 0u;
        bits = (uint64_t)warp_transpose32(w0, lane) | ((uint64_t)warp_transpose32(w1, lane) << 32);
      }
    } else if (warp_row_segments(ro, lane, wr)) {
      // lane j: column j's and column (j + 32)'s bits over the warp's 32 rows, then transpose
      const int64_t c0 = sco[lane], c1 = sco[lane + 32];
      const uint32_t w0 = c0 >= 0 ? warp_col_bits(s, wr, c0) : 0u;
      const uint32_t w1 = c1 >= 0 ? warp_col_bits(s, wr, c1) : 0u;
      bits = (uint64_t)warp_transpose32(w0, lane) | ((uint64_t)warp_transpose32(w1, lane) << 32);
    } else if (s.fib) {
      // sampled mode 0 as the fastest column digit: the tile's columns lie in a few mode-0
      // fibres; one aligned window (4 words) per fibre and row, the sampled positions from it
      if (ro >= 0) {
        const int64_t c0 = ct * TC_NT;
        for (int j = 0; j < TC_NT;) {
          const int64_t col = c0 + j;
          if (col >= s.ncols) break;
          const int q0 = (int)(col % s.fib_s0);              // position of column j in its fibre
          const int nj = min(TC_NT - j, s.fib_s0 - q0);       // columns of this fibre in the tile
          const int64_t co = sco[j];
          if (co >= 0) {
            const FibWin fw = fib_window(s, ro + co - s.idx0[q0]);
            if (s.ptab) {                                    // s0 <= 64: table compaction
              const uint64_t e = fib_pext(fw, tabS, offw, s.fib_nb) >> q0;
              bits |= (nj >= 64 ? e : (e & ((1ull << nj) - 1ull))) << j;
            } else {
              for (int u = 0; u < nj; ++u) {
                const uint32_t p = (uint32_t)s.idx0[q0 + u];
                bits |= (uint64_t)((fib_word(fw, p >> 5) >> (p & 31)) & 1u) << (j + u);
              }
            }
          }
          j += nj;
        }
      }
    } else if (__popcll((uint64_t)sstart[0] | ((uint64_t)sstart[1] << 32)) > 16) {
      // scattered columns (sampled index sets): one bit per column, 8 loads in flight per step
      if (ro >= 0) {
#pragma unroll 1
        for (int j0 = 0; j0 < TC_NT; j0 += 8) {
          uint32_t w[8];
          int sh[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int64_t co = sco[j0 + u];
            const int64_t lin = ro + (co < 0 ? 0 : co);
            w[u] = co < 0 ? 0u : __ldg(s.mask + (lin >> 5));
            sh[u] = (int)(lin & 31);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) bits |= (uint64_t)((w[u] >> sh[u]) & 1u) << (j0 + u);
        }
      }
    } else {
      uint64_t st = (uint64_t)sstart[0] | ((uint64_t)sstart[1] << 32);   // warp-uniform
      while (st) {
        const int j0 = __ffsll((long long)st) - 1;
        st &= st - 1;
        const int j1 = st ? __ffsll((long long)st) - 1 : TC_NT;
        const int64_t co = sco[j0];
        if (ro >= 0 && co >= 0) bits |= mask_bits(s, ro + co, j1 - j0) << j0;
      }
    }
    const int cnt = __popcll(bits);
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp; ++w) base += wsum[w];
    const int excl = base + inc - cnt;
    s.tbits[tile * TC_M + tid] = bits;
    s.troff[tile * TC_M + tid] = (uint16_t)excl;
    // tile blocks of the compacted values are padded to 8 entries (32 B of values, 16 B of
    // entry list) so that a tile's values / weights / list move by bulk copies without
    // touching a neighbour's
    if (tid == TC_M - 1) s.tcount[tile] = (uint64_t)((excl + cnt + 7) & ~7);
    __syncthreads();
  }
}

// the tile block is assembled in shared memory (scattered entry positions) and written out
// coalesced; tiles with more than SV_OUT entries write to global memory directly
constexpr int SV_OUT = 1024;
// the staged word of value index vi: the value, or (perm mode) the index itself as fp32 bits
__device__ __forceinline__ float stage_word(const StageArgs& s, int64_t vi) {
  return s.perm ? __int_as_float((int)vi) : __ldg(s.values + vi);
}

__global__ void __launch_bounds__(128) stage_vals_kernel(StageArgs s) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  if (s.gen_cur && *s.gen_layout == *s.gen_cur) return;   // layout current: gather_vals_kernel re-reads
  __shared__ int64_t sco[TC_NT];
  __shared__ uint32_t sstart[2];
  __shared__ uint64_t sbits[TC_M];
  __shared__ int soff[TC_M];
  __shared__ __align__(16) float sov[SV_OUT];
  __shared__ __align__(16) uint16_t soi[SV_OUT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t tile = blockIdx.x; tile < s.n_tiles; tile += gridDim.x) {
    const int64_t rt = tile / s.n_col_tiles, ct = tile % s.n_col_tiles;
    const int64_t row = rt * TC_M + tid;
    const uint64_t bits = s.tbits[tile * TC_M + tid];
    const int roff = s.troff[tile * TC_M + tid];
    const int64_t tb = (int64_t)s.tbase[tile];           // tile block start (after the scan)
    const int nt = (int)((int64_t)s.tbase[tile + 1] - tb);    // padded entry count of the tile
    if (TRD_CHECKED && !(tb >= 0 && nt >= 0 && tb + nt <= s.vcap)) {   // (block-uniform)
      if (tid == 0) TRD_CHECK_FAIL(kChkStageWrite);
      continue;
    }
    const bool in_smem = nt <= SV_OUT;
    float* ov = in_smem ? sov : s.tvals + tb;            // tile-relative output positions
    uint16_t* oi = in_smem ? soi : s.tidx + tb;
    sbits[tid] = bits;
    soff[tid] = roff;
    stage_tile_cols(s, ct, tid, sco, sstart);            // (its barriers also publish sbits / soff)
    if (tid == TC_M - 1) {                    // padding entries of the tile block
      for (int e = roff + __popcll(bits); e < nt; ++e) {
        oi[e] = 0xFFFFu;
        ov[e] = 0.f;
      }
    }
    const int64_t ro = row < s.nrows ? s.row_off[row] : -1;
    WarpRows wr;
    if (warp_row_segments(ro, lane, wr)) {
      // column-wise: lane j takes columns j and j + 32; each row range of the warp is one run of
      // linear positions per column, so its packed values are consecutive.  The columns' row
      // masks come from the staged row masks by a warp bit-matrix transpose (no mask reads)
      const uint32_t cws[2] = {warp_transpose32((uint32_t)bits, lane), warp_transpose32((uint32_t)(bits >> 32), lane)};
      // both columns' rank lookups first (independent loads in flight), then their entries
      int64_t la[2], lb[2], va[2], vb[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t co = sco[lane + 32 * h];
        la[h] = wr.baseA + co;                           // linear positions of lanes 0, b
        lb[h] = wr.baseB + co;
        const bool act = co >= 0 && cws[h] != 0u;
        va[h] = (s.packed && act) ? mask_rank(s, la[h]) : la[h];
        vb[h] = (s.packed && act && wr.b < 32) ? mask_rank(s, lb[h]) : lb[h];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        uint32_t cw = cws[h];
        if (sco[j] < 0) cw = 0u;
        int qa = 0, qb = 0;
        while (cw) {
          const int r = __ffs(cw) - 1;
          cw &= cw - 1;
          const int rr = warp * 32 + r;                   // row in the tile
          const int pos = soff[rr] + __popcll(sbits[rr] & ((1ull << j) - 1ull));
          if (TRD_CHECKED && pos >= nt) { TRD_CHECK_FAIL(kChkStageWrite); continue; }
          int64_t vi;
          if (r < wr.b) vi = s.packed ? va[h] + qa++ : la[h] + r;
          else vi = s.packed ? vb[h] + qb++ : lb[h] + (r - wr.b);
          ov[pos] = stage_word(s, vi);
          oi[pos] = (uint16_t)(rr * TC_NT + j);
        }
      }
    } else if (bits && s.fib) {
      // fibre windows (see stage_bits): ranks from the window's cumulative popcounts
      float* out = ov + roff;
      uint16_t* oidx = oi + roff;
      int q = 0;
      const int64_t c0 = ct * TC_NT;
      for (int j = 0; j < TC_NT;) {
        const int64_t col = c0 + j;
        if (col >= s.ncols) break;
        const int q0 = (int)(col % s.fib_s0);
        const int nj = min(TC_NT - j, s.fib_s0 - q0);
        uint64_t fb = (bits >> j) & (nj >= 64 ? ~0ull : ((1ull << nj) - 1ull));
        if (fb) {
          const int64_t lin0 = ro + sco[j] - s.idx0[q0];
          const FibWin fw = fib_window(s, lin0);
          int64_t base = lin0;                               // dense: value index = linear position
          uint32_t c1 = 0, c2 = 0, c3 = 0;
          if (s.packed) {
            base = (int64_t)__ldg(s.rank_prefix + (lin0 >> 5)) + __popc(fw.w0 & ((1u << fw.sh) - 1u));
            c1 = __popc(fw.a0);
            c2 = c1 + __popc(fw.a1);
            c3 = c2 + __popc(fw.a2);
          }
          while (fb) {
            const int u = __ffsll((long long)fb) - 1;
            fb &= fb - 1;
            const uint32_t p = (uint32_t)s.idx0[q0 + u];
            int64_t vi;
            if (s.packed) {
              const uint32_t wq = p >> 5;
              vi = base + (wq < 2 ? (wq == 0 ? 0u : c1) : (wq == 2 ? c2 : c3)) +
                   __popc(fib_word(fw, wq) & ((1u << (p & 31)) - 1u));
            } else {
              vi = base + p;
            }
            oidx[q] = (uint16_t)(tid * TC_NT + j + u);
            out[q++] = stage_word(s, vi);
          }
        }
        j += nj;
      }
    } else if (bits && __popcll((uint64_t)sstart[0] | ((uint64_t)sstart[1] << 32)) > 16) {
      // scattered columns: per entry, the rank from its mask word (cached across entries)
      const int64_t rof = s.row_off[row];
      float* out = ov + roff;
      uint16_t* oidx = oi + roff;
      int q = 0;
      int64_t cwi = -1;
      uint32_t cwd = 0, cp = 0;
      uint64_t b = bits;
      while (b) {
        const int j = __ffsll((long long)b) - 1;
        b &= b - 1;
        const int64_t lin = rof + sco[j];
        int64_t vi = lin;
        if (s.packed) {
          const int64_t wi = lin >> 5;
          if (wi != cwi) { cwd = __ldg(s.mask + wi); cp = __ldg(s.rank_prefix + wi); cwi = wi; }
          vi = (int64_t)cp + __popc(cwd & ((1u << (lin & 31)) - 1u));
        }
        oidx[q] = (uint16_t)(tid * TC_NT + j);
        out[q++] = stage_word(s, vi);
      }
    } else if (bits) {
      // row-wise over the column runs: a run's observed values are consecutive
      float* out = ov + roff;
      uint16_t* oidx = oi + roff;
      int q = 0;
      uint64_t st = (uint64_t)sstart[0] | ((uint64_t)sstart[1] << 32);
      while (st) {
        const int j0 = __ffsll((long long)st) - 1;
        st &= st - 1;
        const int j1 = st ? __ffsll((long long)st) - 1 : TC_NT;
        const uint64_t rb = (bits >> j0) & (j1 - j0 >= 64 ? ~0ull : ((1ull << (j1 - j0)) - 1ull));
        if (!rb) continue;
        const int64_t lin0 = ro + sco[j0];
        if (s.packed) {
          const int64_t v0 = mask_rank(s, lin0);
          const int n = __popcll(rb);
          uint64_t b = rb;
          for (int u = 0; u < n; ++u) {
            const int jj = __ffsll((long long)b) - 1;
            b &= b - 1;
            oidx[q] = (uint16_t)(tid * TC_NT + j0 + jj);
            out[q++] = stage_word(s, v0 + u);
          }
        } else {
          uint64_t b = rb;
          while (b) {
            const int jj = __ffsll((long long)b) - 1;
            b &= b - 1;
            oidx[q] = (uint16_t)(tid * TC_NT + j0 + jj);
            out[q++] = stage_word(s, lin0 + jj);
          }
        }
      }
    }
    if (in_smem) {                              // (block-uniform)
      __syncthreads();
      float4* gv = reinterpret_cast<float4*>(s.tvals + tb);     // tile blocks: 8-entry aligned
      uint4* gi = reinterpret_cast<uint4*>(s.tidx + tb);
      for (int q = tid; q < nt / 4; q += TC_M) gv[q] = reinterpret_cast<const float4*>(sov)[q];
      for (int q = tid; q < nt / 8; q += TC_M) gi[q] = reinterpret_cast<const uint4*>(soi)[q];
    }
    __syncthreads();
  }
}

__global__ void layout_gen_kernel(const int* __restrict__ cur, int* __restrict__ layout) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *layout = *cur;
}

// Sweep-invariant sketches: the staged values from the staged value indices (perm), so that a
// new upload with an unchanged mask re-gathers the values without rebuilding the layout
__global__ void __launch_bounds__(256) gather_vals_kernel(const int32_t* __restrict__ perm, const uint16_t* __restrict__ tidx,
                                                          const float* __restrict__ values,
                                                          const uint64_t* __restrict__ total, float* __restrict__ tvals,
                                                          int64_t vcap) {
  int64_t n = (int64_t)*total;
  if (TRD_CHECKED && n > vcap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) TRD_CHECK_FAIL(kChkStageWrite);
    n = vcap;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    tvals[i] = tidx[i] == 0xFFFFu ? 0.f : __ldg(values + perm[i]);
}

// ---------------------------------------------------------------------------------------
struct TcArgs {
  int64_t nrows, ncols, nL, Ik, n_col_tiles, nrows_pad;
  int64_t n_items, per;    // work items = (row-tile group, column split); per = column tiles per split
  int cl;                  // CTAs per cluster (1, or 2: a pair shares B tiles via multicast)
  int64_t n_row_tiles;
  int rowmode, K, R2, rk, rk1, rs, p, nsplit;
  int sigma_inf;
  const __half* arow;      // Lft (pass 1) or Lft_h (pass 2), row-major hi | lo (unused: built in-kernel)
  const float* zk;         // core k, slice-major Z_k[i][a][b] (pass-1 A operand)
  const double* hk;        // scaled gradient h[i][a + r_k b] (pass-2 A operand)
  const float* mid;        // Mid(j_L): [jl][r_{k+1}][r_s]
  const __half* rgtHL;     // B tiles, layout L1 (pass 2) or L2 (pass 1)
  const uint64_t* tbits;
  const uint16_t* troff;
  const uint64_t* tbase;
  const float* tvals;
  const uint16_t* tidx;    // staged entry lists
  int64_t vcap;            // their capacity (checked build)
  float* tw;               // staged weights (pass 1 writes, pass 2 reads)
  const float* lscl;       // [row] 2^-E of the A rows' scaling (Lft in pass 1, Lft_h in pass 2)
  uint32_t* eabs;          // TRD_SIGMA_MAD: |e| bit patterns (pass 1, R21), else nullptr
  unsigned long long ecap;
  const DevScalars* sc;
  float* contrib;          // [split][nrows_pad][KP]  D rows of pass 1
  double* spart;           // [cta][3]
  double* denpart;         // [cta]
  int exp;                 // TRD_TC_EXP (timing experiments only; results invalid if != 0):
                           //   bit 0 = epilogue does the barrier handshakes only
                           //   bit 1 = B producer skips the copies, bit 2 = sketch producer skips
                           //   bit 3 = trace, bit 4 = pass-2 epilogue skips the TMEM loads
};

template <int KP>
struct TcLayout {
  static constexpr int HK = KP / 8;
  static constexpr int B_HALVES = 2 * TC_NT * KP;    // hi block then lo block
  static constexpr uint32_t B_LO_BYTES = TC_NT * KP * 2;
  static constexpr uint32_t IDESC_S = make_idesc(TC_M, TC_NT, 0);   // S = A . B^T
  static constexpr uint32_t IDESC_D = make_idesc(TC_M, KP, 1);      // D += P . B (B MN-major)
  static constexpr uint32_t IDESC_D2 = make_idesc(TC_M, 2 * KP, 1); // D' += P_hi [B_hi | B_lo]
};

// S[tmem] = A_hi.B_hi + A_hi.B_lo + A_lo.B_hi with A in TMEM (hi at acol, lo at acol + KP/2)
template <int KP>
__device__ __forceinline__ void issue_split_gemm_ts(uint32_t dtmem, uint32_t acol, uint32_t bH) {
  using L = TcLayout<KP>;
  // descriptor of the B tile start; K steps and the lo block are added to the address field
  const uint64_t d0 = make_sdesc(bH, 128, L::HK * 128);
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t aa = acol + (term == 2 ? KP / 2 : 0);
    const uint64_t dt = d0 + (uint64_t)((term == 1 ? L::B_LO_BYTES : 0u) >> 4);
#pragma unroll
    for (int ks = 0; ks < KP / 16; ++ks)
      mma_ts(dtmem, aa + ks * 8, dt + (uint64_t)(ks * 16), L::IDESC_S, (term | ks) ? 1u : 0u);
  }
}

// Layout L2 (pass 1): per 64-column tile, each column's row of 2 KP halves is [hi KP | lo KP];
// core matrix (g, h') at (g * 2HK + h') * 128 B, h' < HK hi, h' >= HK lo.  GEMM1 reads it
// K-major with the three split terms (lo = +HK core matrices); GEMM2 reads it MN-major with
// N = 2 KP for the P_hi terms (D' = P_hi [B_hi | B_lo]) and N = KP for P_lo.B_hi.
// NCOL = 64 U columns: U consecutive L2 tiles are one canonical K-major operand of N = 64 U
// rows (the 8-column groups of tile t + 1 follow those of tile t at the same stride)
template <int KP, int NCOL = TC_NT>
__device__ __forceinline__ void issue_split_gemm_ts_l2(uint32_t dtmem, uint32_t acol, uint32_t bH) {
  using L = TcLayout<KP>;
  constexpr uint32_t IDESC = make_idesc(TC_M, NCOL, 0);
  const uint64_t d0 = make_sdesc(bH, 128, 2 * L::HK * 128);
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t aa = acol + (term == 2 ? KP / 2 : 0);
    const uint64_t dt = d0 + (uint64_t)((term == 1 ? L::HK * 128 : 0) >> 4);
#pragma unroll
    for (int ks = 0; ks < KP / 16; ++ks)
      mma_ts(dtmem, aa + ks * 8, dt + (uint64_t)(ks * 16), IDESC, (term | ks) ? 1u : 0u);
  }
}

#ifndef TRD_P1_MERGE
#define TRD_P1_MERGE 1
#endif
// one lane of a converged warp (the MMA issuer runs warp-wide so that its operands live in
// uniform registers; only the elected lane issues)
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
  return pred;
}

// this thread's row of A (hi | lo) -> TMEM columns [acol, acol + KP)
template <int KP>
__device__ __forceinline__ void load_a_to_tmem(const TcArgs& a, int64_t row, uint32_t lane_base, uint32_t acol) {
  const uint4* g = reinterpret_cast<const uint4*>(a.arow + row * 2 * KP);
#pragma unroll
  for (int c = 0; c < KP / 16; ++c) {          // 16 words = 32 halves per chunk
    uint32_t v[16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint4 q = g[c * 4 + u];
      v[u * 4 + 0] = q.x; v[u * 4 + 1] = q.y; v[u * 4 + 2] = q.z; v[u * 4 + 3] = q.w;
    }
    tmem_st16(lane_base + acol + c * 16, v);
  }
}

#include "tc_ws.inc"

// ---------------------------------------------------------------------------------------
// a6 contraction + reduction, stage 1 (fp64, fixed order):
//   d(i_k)[a + r_k b] = sum_split sum_jl sum_c Mid(jl)[b][c] D(split, row(i_k, jl))[a + r_k c]
// (Eq. 9/15, P:152, 234 with S(j) = Mid(j_L) Rgt(j_R); p = 0: Mid = I).  grid (I_k, JC):
// CTA (ik, jc) sums the jl chunk jc into dpart[jc][ik][R2].
// ---------------------------------------------------------------------------------------
constexpr int RD_ROWS = 64;   // jl rows staged per step
__global__ void __launch_bounds__(1024) tc_reduce_d_kernel(
    const float* __restrict__ contrib, const float* __restrict__ mid, int nsplit, int64_t nrows_pad, int64_t nL,
    int64_t Ik, int rowmode, int KP, int R2, int rk, int rs, int p, int64_t jl_chunk, double* __restrict__ dpart,
    int rd_rows) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  extern __shared__ float rsm[];
  const int KPp = KP + 4, MS = (R2 / rk) * rs;               // Mid(jl) is r_{k+1} x r_s
  float* Dt = rsm;                                           // [rd_rows][KP + 4] (16-B rows)
  float* Mt = rsm + rd_rows * KPp;                           // [rd_rows][MS]
  __shared__ double acc[1024];
  const int64_t ik = blockIdx.x, jc = blockIdx.y;
  const int tid = threadIdx.x;
  const int G = max(1, (int)blockDim.x / R2);
  const int o = tid % R2, g = tid / R2;
  const int aa = o % rk, bq = o / rk;
  const int q4 = KP / 4;                                     // float4 per D row
  const int64_t j0 = jc * jl_chunk, j1 = min(nL, j0 + jl_chunk);
  double s = 0.0;
  for (int64_t jb = j0; jb < j1; jb += rd_rows) {
    const int nr = (int)min((int64_t)rd_rows, j1 - jb);
    if (p > 0) {                                             // Mid rows jb.. are contiguous
      const float* src = mid + jb * MS;
      for (int idx = tid; idx < nr * MS; idx += blockDim.x) Mt[idx] = __ldg(src + idx);
    }
    {
      // the column splits' D rows summed while staging (fixed split order): one barrier per chunk
      for (int f = tid; f < nr * q4; f += blockDim.x) {
        const int rr = f / q4, c4 = f - rr * q4;
        const int64_t jl = jb + rr;
        const int64_t row = rowmode == 0 ? jl + nL * ik : ik + Ik * jl;
        float4 v = __ldg(reinterpret_cast<const float4*>(contrib + row * KP) + c4);
        for (int sp = 1; sp < nsplit; ++sp) {
          const float4 w = __ldg(reinterpret_cast<const float4*>(contrib + ((int64_t)sp * nrows_pad + row) * KP) + c4);
          v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
        }
        *reinterpret_cast<float4*>(Dt + rr * KPp + 4 * c4) = v;
      }
      __syncthreads();
      if (g < G) {
        float t = 0.f;
        if (p == 0) {
          for (int rr = g; rr < nr; rr += G) t += Dt[rr * KPp + o];
        } else {
          for (int rr = g; rr < nr; rr += G) {
            const float* M = Mt + rr * MS + bq * rs;
            const float* D = Dt + rr * KPp + aa;
            float u = 0.f;
            for (int c = 0; c < rs; ++c) u = fmaf(M[c], D[rk * c], u);
            t += u;
          }
        }
        s += (double)t;
      }
      __syncthreads();
    }
  }
  acc[tid] = s;
  __syncthreads();
  if (tid < R2) {
    double t = 0.0;
    for (int gg = 0; gg < G; ++gg) t += acc[gg * R2 + tid];
    dpart[(jc * Ik + ik) * R2 + tid] = t;
  }
}

// Register-blocked stage 1 for compile-time ranks (RK, RK1, RS) with KP == RK * RS: thread per
// GEMM row, Mid(jl) (RK1 x RS) and the D row (RK x RS, column a + RK c) loaded as float4 into
// registers, acc[a][b] += sum_c D[a + RK c] Mid[b][c] (outer products over c), fp32 per
// thread; then a fixed-order fp64 reduction over the CTA's threads.  CTA = (i_k, jl chunk).
template <int RK, int RK1, int RS>
__global__ void __launch_bounds__(128) tc_reduce_d_rb_kernel(const float* __restrict__ contrib,
                                                             const float* __restrict__ mid, int nsplit,
                                                             int64_t nrows_pad, int64_t nL, int64_t Ik, int rowmode,
                                                             int64_t jl_chunk, double* __restrict__ dpart) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  constexpr int KP = RK * RS, MS = RK1 * RS, R2 = RK * RK1;
  static_assert(KP % 16 == 0 && MS % 4 == 0, "vector loads");
  __shared__ float red[128][R2 + 1];
  const int64_t ik = blockIdx.x, jc = blockIdx.y;
  const int64_t j0 = jc * jl_chunk, j1 = min(nL, j0 + jl_chunk);
  float acc[RK][RK1];
#pragma unroll
  for (int a = 0; a < RK; ++a)
#pragma unroll
    for (int b = 0; b < RK1; ++b) acc[a][b] = 0.f;
  for (int64_t jl = j0 + threadIdx.x; jl < j1; jl += blockDim.x) {
    float M[RK1][RS];
    const float4* m4 = reinterpret_cast<const float4*>(mid + jl * MS);
#pragma unroll
    for (int q = 0; q < MS / 4; ++q) {
      const float4 v = __ldg(m4 + q);
      reinterpret_cast<float*>(M)[4 * q + 0] = v.x; reinterpret_cast<float*>(M)[4 * q + 1] = v.y;
      reinterpret_cast<float*>(M)[4 * q + 2] = v.z; reinterpret_cast<float*>(M)[4 * q + 3] = v.w;
    }
    const int64_t row = rowmode == 0 ? jl + nL * ik : ik + Ik * jl;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float4* d4 = reinterpret_cast<const float4*>(contrib + ((int64_t)sp * nrows_pad + row) * KP);
#pragma unroll
      for (int c = 0; c < RS; ++c) {
        float D[RK];
#pragma unroll
        for (int q = 0; q < RK / 4; ++q) {
          const float4 v = __ldg(d4 + (RK * c) / 4 + q);
          D[4 * q] = v.x; D[4 * q + 1] = v.y; D[4 * q + 2] = v.z; D[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int a = 0; a < RK; ++a)
#pragma unroll
          for (int b = 0; b < RK1; ++b) acc[a][b] = fmaf(D[a], M[b][c], acc[a][b]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < RK; ++a)
#pragma unroll
    for (int b = 0; b < RK1; ++b) red[threadIdx.x][a + RK * b] = acc[a][b];
  __syncthreads();
  if (threadIdx.x < R2) {
    double t = 0.0;
    for (int q = 0; q < (int)blockDim.x; ++q) t += (double)red[q][threadIdx.x];
    dpart[(jc * Ik + ik) * R2 + threadIdx.x] = t;
  }
}

// Large-rank stage 1 (R^2 > kBigR2, any KP; D rows of the tcgen05 or the SIMT pass 1): thread
// per output o = a + r_k b of d(i_k), grid (I_k, JC, ceil(R^2 / 256)); for each jl of the chunk
// (ascending) u = sum_c Mid(jl)[b][c] sum_split D(split, row)[a + r_k c] in fp32, added to an
// fp64 sum -- the same contraction as tc_reduce_d_kernel without the shared-memory staging
// (Eq. 9/15).
__global__ void __launch_bounds__(256) reduce_d_big_kernel(
    const float* __restrict__ contrib, const float* __restrict__ mid, int nsplit, int64_t nrows_pad, int64_t nL,
    int64_t Ik, int rowmode, int KP, int R2, int rk, int rk1, int rs, int p, int64_t jl_chunk,
    double* __restrict__ dpart) {
  const int64_t ik = blockIdx.x, jc = blockIdx.y;
  const int o = blockIdx.z * blockDim.x + threadIdx.x;
  if (o >= R2) return;
  const int aa = o % rk, bq = o / rk;
  const int64_t j0 = jc * jl_chunk, j1 = min(nL, j0 + jl_chunk);
  double s = 0.0;
  for (int64_t jl = j0; jl < j1; ++jl) {
    const int64_t row = rowmode == 0 ? jl + nL * ik : ik + Ik * jl;
    float u = 0.f;
    if (p == 0) {
      for (int sp = 0; sp < nsplit; ++sp) u += __ldg(contrib + ((int64_t)sp * nrows_pad + row) * KP + o);
    } else {
      const float* M = mid + (jl * rk1 + bq) * rs;
      for (int c = 0; c < rs; ++c) {
        float dsum = 0.f;
        for (int sp = 0; sp < nsplit; ++sp) dsum += __ldg(contrib + ((int64_t)sp * nrows_pad + row) * KP + aa + rk * c);
        u = fmaf(__ldg(M + c), dsum, u);
      }
    }
    s += (double)u;
  }
  dpart[(jc * Ik + ik) * R2 + o] = s;
}

// The same contraction with the D rows (summed over the splits) and Mid rows of RB left
// indices staged in shared memory, 1024 threads, NO outputs per thread (o = tid + 1024 i).
// Per output and jl: u = sum_c Mid[b][c] D[a + r_k c] in fp32 (c ascending), added to an fp64
// sum in jl order -- bitwise the arithmetic of reduce_d_big_kernel.
template <int NO>
__global__ void __launch_bounds__(1024) reduce_d_big_smem_kernel(
    const float* __restrict__ contrib, const float* __restrict__ mid, int nsplit, int64_t nrows_pad, int64_t nL,
    int64_t Ik, int rowmode, int KP, int K, int R2, int rk, int rk1, int rs, int p, int64_t jl_chunk, int RB,
    double* __restrict__ dpart) {
  extern __shared__ float bsm[];
  const int MS = rk1 * rs;
  float* Dt = bsm;                       // [RB][K]
  float* Mt = bsm + RB * K;              // [RB][MS]
  const int64_t ik = blockIdx.x, jc = blockIdx.y;
  const int tid = threadIdx.x;
  const int64_t j0 = jc * jl_chunk, j1 = min(nL, j0 + jl_chunk);
  double acc[NO];
  int aa[NO], bq[NO];
#pragma unroll
  for (int i = 0; i < NO; ++i) { acc[i] = 0.0; const int o = tid + 1024 * i; aa[i] = o % rk; bq[i] = o / rk; }
  for (int64_t jb = j0; jb < j1; jb += RB) {
    const int nr = (int)min((int64_t)RB, j1 - jb);
    for (int t = tid; t < nr * K; t += blockDim.x) {
      const int rr = t / K, q = t - rr * K;
      const int64_t jl = jb + rr;
      const int64_t row = rowmode == 0 ? jl + nL * ik : ik + Ik * jl;
      float v = 0.f;
      for (int sp = 0; sp < nsplit; ++sp) v += __ldg(contrib + ((int64_t)sp * nrows_pad + row) * KP + q);
      Dt[t] = v;
    }
    if (p > 0)
      for (int t = tid; t < nr * MS; t += blockDim.x) Mt[t] = __ldg(mid + jb * MS + t);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      if (tid + 1024 * i >= R2) break;
      for (int rr = 0; rr < nr; ++rr) {
        float u = 0.f;
        if (p == 0) {
          u = Dt[rr * K + tid + 1024 * i];
        } else {
          const float* M = Mt + rr * MS + bq[i] * rs;
          const float* D = Dt + rr * K + aa[i];
          for (int c = 0; c < rs; ++c) u = fmaf(M[c], D[rk * c], u);
        }
        acc[i] += (double)u;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    const int o = tid + 1024 * i;
    if (o < R2) dpart[(jc * Ik + ik) * R2 + o] = acc[i];
  }
}

// stage 2: dvec = [d | sum_e2 | welsch | n] from the chunk partials and the per-CTA statistics
__global__ void tc_reduce_final_kernel(const double* __restrict__ dpart, int64_t JC, int64_t Ik, int R2,
                                       const double* __restrict__ spart, int64_t nparts,
                                       double* __restrict__ dvec, DevScalars* sc, int kblk, int64_t ik0,
                                       int64_t Ik_tot) {
  trd_gdc_wait();   // (PDL: the stream predecessor has completed, memory visible)
  const int64_t ik = blockIdx.x;
  if (ik < Ik) {
    for (int o = threadIdx.x; o < R2; o += blockDim.x) {
      double t = 0.0;
      for (int64_t jc = 0; jc < JC; ++jc) t += dpart[(jc * Ik + ik) * R2 + o];
      dvec[(ik0 + ik) * R2 + o] = t;
    }
    return;
  }
  // statistics: thread t sums the CTA partials t, t + 128, ... (fixed order), then a fixed
  // tree over the threads (the partials are read in parallel, not by one thread)
  __shared__ double red[3][128];
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t q = threadIdx.x; q < nparts; q += blockDim.x)
    for (int j = 0; j < 3; ++j) v[j] += spart[q * 3 + j];
  for (int j = 0; j < 3; ++j) red[j][threadIdx.x] = v[j];
  __syncthreads();
  for (int w = 64; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int j = 0; j < 3; ++j) red[j][threadIdx.x] += red[j][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 3) {
    const double t = red[threadIdx.x][0];
    dvec[Ik_tot * R2 + threadIdx.x] = t;
    if (threadIdx.x == 2 && sc && sc->prof_on) sc->prof_nobs[kblk] += t;
  }
}

// ---------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------
static int tc_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

void launch_tc_lft(Context& c, const BlockPlan& bp, bool pass2, cudaStream_t s) {
  LftArgs a;
  a.nrows = bp.nrows; a.nL = bp.nL; a.Ik = bp.nrows / bp.nL; a.ik0 = bp.ik0;
  a.rowmode = bp.rowmode; a.rk = bp.rk; a.rk1 = bp.rk1; a.rs = bp.rs; a.K = bp.K; a.KP = bp.KP; a.p = bp.p;
  a.zk = c.Z + c.zoff[bp.k];
  a.hk = c.h;
  a.mid = c.mid;
  a.lscl = pass2 ? c.lsclh : c.lscl;
  a.amax = pass2 ? nullptr : &c.sc->amax_a;
  if (getenv("TRD_DIAG_NOAMAX")) a.amax = nullptr;           // (diagnostic: results invalid)
  const int64_t pad = bp.n_row_tiles * TC_M;
  if (bp.p > 0 && bp.rk == 8 && bp.rk1 == 8 && bp.rs == 8) {
    const int grid = (int)std::min<int64_t>((pad + 127) / 128, (int64_t)c.num_sm * 16);
    TRD_PDL((tc_lft_pack_rb_kernel<8, 8, 8>), grid, 128, 0, s, a, pass2 ? 1 : 0, pad, pass2 ? c.lfthHL : c.lftHL);
    c.launches++;
    return;
  }
  if (c.rbucket > 32 && bp.p > 0 && bp.rk1 >= 32) {
    const size_t smem = (size_t)(bp.rk * (bp.rk1 + 1) + kPackJ * bp.rk1 * bp.rs + kPackJ * (bp.K + 1)) * sizeof(float);
    if (smem <= 200 * 1024) {
      cudaFuncSetAttribute(tc_lft_pack_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const dim3 grid((unsigned)a.Ik, (unsigned)((bp.nL + kPackJ - 1) / kPackJ));
      TRD_PDL(tc_lft_pack_tile_kernel, grid, 256, smem, s, a, pass2 ? 1 : 0, pad, pass2 ? c.lfthHL : c.lftHL);
      c.launches++;
      return;
    }
  }
  if (getenv("TRD_LFT_TILE") == nullptr) {        // half-warp per row (TRD_LFT_TILE: the tile kernel, A/B)
    const int grid = (int)std::min<int64_t>((pad * 16 + 255) / 256, (int64_t)c.num_sm * 16);
    TRD_PDL(tc_lft_pack_hw_kernel, grid, 256, 0, s, a, pass2 ? 1 : 0, pad, pass2 ? c.lfthHL : c.lftHL);
    c.launches++;
    return;
  }
  size_t smem = (size_t)TC_M * (((bp.rk * bp.rk1) | 1) + ((bp.rk1 * bp.rs) | 1)) * sizeof(float);
  const int gmem = smem > 200 * 1024 ? 1 : 0;      // large ranks: read X / Mid from global memory
  if (gmem) smem = 0;
  else cudaFuncSetAttribute(tc_lft_pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (int)std::min<int64_t>(bp.n_row_tiles, (int64_t)c.num_sm * 8);
  TRD_PDL(tc_lft_pack_kernel, grid, 256, smem, s, a, pass2 ? 1 : 0, pad, pass2 ? c.lfthHL : c.lftHL, gmem);
  c.launches++;
}

void launch_tc_pack_cols(Context& c, const BlockPlan& bp, cudaStream_t s) {
  TRD_PDL(tc_pack_cols_kernel, tc_grid(bp.n_col_tiles * TC_NT * bp.KP), 256, 0, s, c.rgtT, bp.ncols, bp.K, bp.KP,
                                                                                bp.n_col_tiles, c.rgtHL, c.rgtHL2, c.sc);
  c.launches++;
}

// Stage sketch for block bp into the staging buffers st (bits, offsets, prefix, values)
void launch_tc_stage(Context& c, const BlockPlan& bp, TcStage& st, cudaStream_t s, int phase) {
  StageArgs a;
  a.nrows = bp.nrows; a.ncols = bp.ncols; a.n_col_tiles = bp.n_col_tiles;
  a.n_tiles = bp.n_row_tiles * bp.n_col_tiles;
  a.n_words = c.n_words;
  a.packed = c.packed;
  a.row_off = c.row_off; a.col_off = c.col_off;
  a.mask = c.mask; a.rank_prefix = c.rank_prefix; a.values = c.values;
  a.tbits = st.tbits; a.troff = st.troff; a.tcount = st.tcount; a.tbase = st.tbase; a.tvals = st.tvals;
  a.tidx = st.tidx;
  a.vcap = st.vcap;
  // sweep-invariant sketch with a layout cache: stage the value indices (perm), then gather; both
  // layout kernels exit at once when the uploaded mask equals the one the layout was built from
  const bool cached = st.perm != nullptr;
  a.gen_cur = cached ? &c.sc->mask_gen : nullptr;
  a.gen_layout = cached ? &c.sc->layout_gen[bp.k] : nullptr;
  a.perm = cached ? st.perm : nullptr;
  if (cached) a.tvals = reinterpret_cast<float*>(st.perm);
  // fibre windows: mode 0 is the fastest column digit with a sampled set of >= 16 positions,
  // I0 <= 128 (a window of five words), and not a partial shard (offsets = global indices)
  a.fib = 0; a.fib_s0 = 0; a.idx0 = nullptr; a.rfib = 0; a.ptab = nullptr; a.fib_nb = 0;
  const bool mode0_sampled = !bp.explicit_cols && bp.s[0] < c.dims[0] && c.dims[0] <= 128 &&
                             !(c.cfg.shard_mode == 0 && c.shard_end - c.shard_begin < c.dims[0]);
  if (mode0_sampled && bp.nright > 0 && bp.right[bp.rdig[0]] == 0 && bp.s[0] >= 16 && !(getenv("TRD_NO_FIB"))) {
    a.fib = 1;
    a.fib_s0 = (int)bp.s[0];
    a.idx0 = c.idx + c.idx_off[0];
  }
  // row fibres: mode 0 the fastest row digit (k != 0 enumerates rows j_L fastest), 32 sampled
  // positions, whole warps of rows per fibre
  if (mode0_sampled && bp.k != 0 && bp.nleft > 0 && bp.left[bp.ldig[0]] == 0 && bp.s[0] == 32 &&
      bp.nL % 32 == 0 && bp.rowmode == 0 && !(getenv("TRD_NO_RFIB"))) {
    a.rfib = 1;
    a.fib_s0 = 32;
    a.idx0 = c.idx + c.idx_off[0];
  }
  if ((a.fib || a.rfib) && stage_uses_pext(c, bp)) {   // (tables written by the sampler)
    a.ptab = c.ptab;
    a.fib_nb = (int)((c.dims[0] + 7) / 8);
  }
  // grids of exactly the resident CTAs (the kernels loop over tiles): no partial last wave
  static int occ_bits = 0, occ_vals = 0;
  if (!occ_bits) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_bits, stage_bits_kernel, TC_M, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_vals, stage_vals_kernel, TC_M, 0);
    occ_bits = std::max(occ_bits, 1);
    occ_vals = std::max(occ_vals, 1);
  }
  const int gb = (int)std::min<int64_t>(a.n_tiles, (int64_t)c.num_sm * occ_bits);
  const int gv = (int)std::min<int64_t>(a.n_tiles, (int64_t)c.num_sm * occ_vals);
  if (phase != 2) {
    TRD_PDL(stage_bits_kernel, gb, TC_M, 0, s, a);
    // tbase = exclusive prefix of tcount (tcount[n_tiles] = 0: tbase[n_tiles] = total); out of
    // place, so a skipped stage_bits leaves the same prefix
    cub::DeviceScan::ExclusiveSum(st.scan_tmp, st.scan_tmp_bytes, st.tcount, st.tbase, (int)a.n_tiles + 1, s);
    c.launches += 2;
  }
  if (phase == 1) return;
  TRD_PDL(stage_vals_kernel, gv, TC_M, 0, s, a);
  c.launches += 1;
  if (cached) {
    layout_gen_kernel<<<1, 32, 0, s>>>(&c.sc->mask_gen, &c.sc->layout_gen[bp.k]);
    // (TRD_GATHER_CTAS: CTAs per SM; fewer CTAs on the staging stream, to leave room for the
    //  concurrent pass kernels, measured slower: C5b e2e 2.35e10 with 1, 2.66e10 with 2, 2.81e10
    //  with 8 vs 2.83e10 in line)
    const int gper = getenv("TRD_GATHER_CTAS") ? std::max(1, atoi(getenv("TRD_GATHER_CTAS"))) : 8;
    gather_vals_kernel<<<c.num_sm * gper, 256, 0, s>>>(st.perm, st.tidx, c.values, st.tbase + a.n_tiles, st.tvals, st.vcap);
    c.launches += 2;
  }
}

size_t tc_scan_tmp_bytes(int64_t n_tiles) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (int)n_tiles + 1);
  return bytes;
}

static TcArgs make_tc_args(const Context& c, const BlockPlan& bp, const TcStage& st, bool pass2) {
  TcArgs a;
  a.nrows = bp.nrows; a.ncols = bp.ncols; a.nL = bp.nL; a.Ik = bp.nrows / bp.nL;
  a.n_col_tiles = bp.n_col_tiles; a.nrows_pad = bp.n_row_tiles * TC_M;
  a.cl = bp.tc_cl;
  a.n_row_tiles = bp.n_row_tiles;
  a.n_items = ((bp.n_row_tiles + a.cl - 1) / a.cl) * bp.tc_nsplit; a.per = bp.tc_per;
  a.rowmode = bp.rowmode; a.K = bp.K; a.R2 = bp.R2; a.rk = bp.rk; a.rk1 = bp.rk1; a.rs = bp.rs;
  a.p = bp.p; a.nsplit = bp.tc_nsplit;
  a.sigma_inf = c.cfg.sigma_mode == TRD_SIGMA_INF;
  a.arow = pass2 ? c.lfthHL : c.lftHL;
  a.zk = c.Z + c.zoff[bp.k];
  a.hk = c.h;
  a.mid = c.mid;
  const char* ex = getenv("TRD_TC_EXP");
  a.exp = ex ? atoi(ex) : 0;
  a.rgtHL = ((!pass2 && !TRD_P1_MERGE) || (pass2 && TRD_EXPERIMENTS && (a.exp & 32))) ? c.rgtHL : c.rgtHL2;
  a.tbits = st.tbits; a.troff = st.troff; a.tbase = st.tbase; a.tvals = st.tvals; a.tidx = st.tidx;
  a.vcap = st.vcap;
  a.tw = c.tw;
  a.lscl = pass2 ? c.lsclh : c.lscl;
  a.sc = c.sc;
  a.contrib = c.contrib; a.spart = c.spart; a.denpart = c.denpart;
  a.eabs = (!pass2 && c.cfg.sigma_mode == TRD_SIGMA_MAD) ? c.eabs : nullptr;
  a.ecap = (unsigned long long)c.eabs_cap;
  return a;
}

template <int KP, int U>
static void launch_tc_pass_t(Context& c, const BlockPlan& bp, const TcStage& st, bool pass2, cudaStream_t s) {
  static bool hang_flag_set = false;
  if (!hang_flag_set) {
    const int on = getenv("TRD_DEBUG_HANG") ? 1 : 0;
    cudaMemcpyToSymbol(g_debug_hang, &on, sizeof(int));
    hang_flag_set = true;
  }
  TcArgs a = make_tc_args(c, bp, st, pass2);
  const dim3 grid((unsigned)(pass2 ? bp.tc_grid : bp.tc_grid1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = grid;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!pass2) {
    const int sm = Ws1<KP, U>::SMEM;
    cudaFuncSetAttribute(tc_pass1_kernel<KP, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cfg.blockDim = dim3(WsWarps<Ws1<KP, U>::NE>::THREADS);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchKernelEx(&cfg, tc_pass1_kernel<KP, U>, a);
  } else {
    const int sm = Ws2<KP, U>::SMEM;
    cudaFuncSetAttribute(tc_pass2_kernel<KP, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cfg.blockDim = dim3(WsWarps<Ws2<KP, U>::NE>::THREADS);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchKernelEx(&cfg, tc_pass2_kernel<KP, U>, a);
  }
  c.launches++;
  if (getenv("TRD_DEBUG_SYNC")) {            // debugging aid: serialise and report each pass launch
    const cudaError_t e = cudaStreamSynchronize(s);
    fprintf(stderr, "[trd debug] block %d pass %d KP %d U %d grid %u items %lld per %lld: %s\n", bp.k, pass2 ? 2 : 1,
            KP, U, grid.x, (long long)a.n_items, (long long)a.per, cudaGetErrorString(e));
  }
}

void tc_debug_dump() {
  static long long tr[256 * 16];
  if (getenv("TRD_TC_EXP") && (atoi(getenv("TRD_TC_EXP")) & 64) &&
      cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr)) == cudaSuccess) {
    fprintf(stderr, "[trd tc trace2] pass-2 CTA 0 units (cycles rel. to unit 0 issue start)\n"
                    "  unit | MMA start bfull tfree issued | EPI start | h0: skfull dumped entries barred | h1: ...\n");
    const long long t0 = tr[0];
    for (int i = 0; i < 40; ++i) {
      const long long* q = tr + i * 16;
      auto f = [&](int k) { return q[k] ? q[k] - t0 : -1; };
      fprintf(stderr, "  %4d | %7lld %5lld %5lld %5lld | %7lld | %5lld %5lld %5lld %5lld | %5lld %5lld %5lld %5lld\n", i,
              f(0), q[1] - q[0], q[2] - q[0], q[3] - q[0], f(4), q[5] - q[4], q[6] - q[4], q[7] - q[4], q[8] - q[4],
              q[9] - q[4], q[10] - q[4], q[11] - q[4], q[12] - q[4]);
    }
    return;
  }
  if (cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr)) == cudaSuccess && tr[0] != 0) {
    fprintf(stderr, "[trd tc trace] pass-1 CTA 0 (cycles rel. to tile 0 GEMM1 start)\n"
                    "  tile | G1 start wait issue | G2 start wait issue | EPI start skfull sfull dumped ppfree cleared done fenced barred\n");
    const long long t0 = tr[0];
    for (int i = 0; i < 48; ++i) {
      const long long* q = tr + i * 16;
      auto f = [&](int k) { return q[k] ? q[k] - t0 : -1; };
      fprintf(stderr, "  %4d | %7lld %5lld %5lld | %7lld %5lld %5lld | %7lld %5lld %5lld %5lld %5lld %5lld %5lld %5lld %5lld\n", i,
              f(0), q[1] - q[0], q[2] - q[0], f(3), q[4] - q[3], q[5] - q[3], f(6), q[7] - q[6], q[8] - q[6],
              q[9] - q[6], q[10] - q[6], q[14] - q[6], q[11] - q[6], q[12] - q[6], q[13] - q[6]);
    }
  }
  unsigned long long v[16];
  if (cudaMemcpyFromSymbol(v, g_tc_dbg, sizeof(v)) != cudaSuccess) return;
  const char* nm[6] = {"a_full_wait", "bf_full_wait", "t_free_wait", "issue", "tiles", "total"};
  fprintf(stderr, "[trd tc exp] pass-2 MMA thread cycles summed over CTAs\n");
  for (int i = 0; i < 6; ++i) fprintf(stderr, "  %-14s %.4e\n", nm[i], (double)v[i]);
}

bool tc_check_collect(DevCheck* out, unsigned int jitter_ns, cudaStream_t s) {
  DevCheck h = {}, z = {};
  z.jitter_ns = jitter_ns;
  cudaMemcpyFromSymbolAsync(&h, g_check, sizeof(h), 0, cudaMemcpyDeviceToHost, s);
  cudaMemcpyToSymbolAsync(g_check, &z, sizeof(z), 0, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  *out = h;
  return h.code != 0;
}

bool tc_supported_kp(int KP) { return KP >= 16 && KP <= 128 && KP % 16 == 0; }

void launch_tc_pass(Context& c, const BlockPlan& bp, const TcStage& st, bool pass2, cudaStream_t s) {
  // U = 2 (tile pairs, N = 128 GEMMs) for KP <= 64 as chosen by build_plan: pass 2 only by
  // default -- pass 1 with pairs runs its two epilogue warpgroups in lockstep on the halves
  // of a pair and measured slower on C5b (13.8 vs 12.4 ms per sweep); TRD_P1_UNIT=2 enables it
  static const int p1_unit = getenv("TRD_P1_UNIT") ? atoi(getenv("TRD_P1_UNIT")) : 1;
  const bool pair = bp.tc_u == 2 && (pass2 || p1_unit == 2);
  switch (bp.KP) {
    case 16: pair ? launch_tc_pass_t<16, 2>(c, bp, st, pass2, s) : launch_tc_pass_t<16, 1>(c, bp, st, pass2, s); break;
    case 32: pair ? launch_tc_pass_t<32, 2>(c, bp, st, pass2, s) : launch_tc_pass_t<32, 1>(c, bp, st, pass2, s); break;
    case 48: pair ? launch_tc_pass_t<48, 2>(c, bp, st, pass2, s) : launch_tc_pass_t<48, 1>(c, bp, st, pass2, s); break;
    case 64: pair ? launch_tc_pass_t<64, 2>(c, bp, st, pass2, s) : launch_tc_pass_t<64, 1>(c, bp, st, pass2, s); break;
    case 80: launch_tc_pass_t<80, 1>(c, bp, st, pass2, s); break;
    case 96: launch_tc_pass_t<96, 1>(c, bp, st, pass2, s); break;
    case 112: launch_tc_pass_t<112, 1>(c, bp, st, pass2, s); break;
    case 128: launch_tc_pass_t<128, 1>(c, bp, st, pass2, s); break;
    default: break;
  }
}

void launch_reduce_d_contrib(Context& c, const BlockPlan& bp, int nsplit, int64_t nrows_pad, int64_t nparts,
                             cudaStream_t s) {
  const int64_t Ik = bp.nrows / bp.nL;
  if (bp.R2 == 0) {                          // statistics only (the sigma_0 pass)
    TRD_PDL(tc_reduce_final_kernel, 1, 128, 0, s, c.dpart, 0, 0, 0, c.spart, nparts, c.dvec, nullptr, bp.k, 0, 0);
    c.launches++;
    return;
  }
  if (Ik < c.dims[bp.k]) cudaMemsetAsync(c.dvec, 0, (size_t)(c.dims[bp.k] * bp.R2) * sizeof(double), s);
  const int no = (bp.R2 + 1023) / 1024;
  const int RB = 16;
  const size_t smem = (size_t)RB * (bp.K + bp.rk1 * bp.rs) * sizeof(float);
  if (no <= 16 && smem <= 200 * 1024 && !getenv("TRD_RD_PLAIN")) {
#define RD_BIG(NO_)                                                                                            \
  do {                                                                                                       \
    cudaFuncSetAttribute(reduce_d_big_smem_kernel<NO_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    reduce_d_big_smem_kernel<NO_><<<dim3((unsigned)Ik, (unsigned)bp.tc_jc), 1024, smem, s>>>(                    \
        c.contrib, c.mid, nsplit, nrows_pad, bp.nL, Ik, bp.rowmode, bp.KP, bp.K, bp.R2, bp.rk, bp.rk1, bp.rs, bp.p, \
        bp.tc_jl_chunk, RB, c.dpart);                                                                        \
  } while (0)
    if (no <= 1) RD_BIG(1);
    else if (no <= 2) RD_BIG(2);
    else if (no <= 4) RD_BIG(4);
    else if (no <= 8) RD_BIG(8);
    else RD_BIG(16);
#undef RD_BIG
  } else {
    reduce_d_big_kernel<<<dim3((unsigned)Ik, (unsigned)bp.tc_jc, (unsigned)((bp.R2 + 255) / 256)), 256, 0, s>>>(
        c.contrib, c.mid, nsplit, nrows_pad, bp.nL, Ik, bp.rowmode, bp.KP, bp.R2, bp.rk, bp.rk1, bp.rs, bp.p,
        bp.tc_jl_chunk, c.dpart);
  }
  TRD_PDL(tc_reduce_final_kernel, (unsigned)(Ik + 1), 128, 0, s, c.dpart, bp.tc_jc, Ik, bp.R2, c.spart, nparts,
                                                            c.dvec, c.sc, bp.k, bp.ik0, c.dims[bp.k]);
  c.launches += 2;
}

void launch_tc_reduce_d(Context& c, const BlockPlan& bp, cudaStream_t s) {
  const int64_t Ik = bp.nrows / bp.nL;
  if (bp.R2 > kBigR2) {
    launch_reduce_d_contrib(c, bp, bp.tc_nsplit, bp.n_row_tiles * TC_M, bp.tc_grid1, s);
    return;
  }
  if (Ik < c.dims[bp.k]) cudaMemsetAsync(c.dvec, 0, (size_t)(c.dims[bp.k] * bp.R2) * sizeof(double), s);
  if (bp.p > 0 && bp.rk == 8 && bp.rk1 == 8 && bp.rs == 8 && bp.KP == 64) {
    TRD_PDL((tc_reduce_d_rb_kernel<8, 8, 8>), dim3((unsigned)Ik, (unsigned)bp.tc_jc), 128, 0, s, 
        c.contrib, c.mid, bp.tc_nsplit, bp.n_row_tiles * TC_M, bp.nL, Ik, bp.rowmode, bp.tc_jl_chunk, c.dpart);
    TRD_PDL(tc_reduce_final_kernel, (unsigned)(Ik + 1), 128, 0, s, c.dpart, bp.tc_jc, Ik, bp.R2, c.spart, bp.tc_grid1,
                                                              c.dvec, c.sc, bp.k, bp.ik0, c.dims[bp.k]);
    c.launches += 2;
    return;
  }
  const int threads = bp.R2 * std::max(1, 256 / std::max(1, bp.R2));
  const size_t per_row = (size_t)((bp.KP + 4) + (bp.R2 / bp.rk) * bp.rs) * sizeof(float);
  const int rd_rows = (int)std::max<size_t>(1, std::min<size_t>(RD_ROWS, (200 * 1024) / per_row));
  const size_t smem = (size_t)rd_rows * per_row;
  cudaFuncSetAttribute(tc_reduce_d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  TRD_PDL(tc_reduce_d_kernel, dim3((unsigned)Ik, (unsigned)bp.tc_jc), threads, smem, s, 
      c.contrib, c.mid, bp.tc_nsplit, bp.n_row_tiles * TC_M, bp.nL, Ik, bp.rowmode, bp.KP, bp.R2, bp.rk,
      bp.rs, bp.p, bp.tc_jl_chunk, c.dpart, rd_rows);
  TRD_PDL(tc_reduce_final_kernel, (unsigned)(Ik + 1), 128, 0, s, c.dpart, bp.tc_jc, Ik, bp.R2, c.spart, bp.tc_grid1,
                                                            c.dvec, c.sc, bp.k, bp.ik0, c.dims[bp.k]);
  c.launches += 2;
}

}  // namespace trd

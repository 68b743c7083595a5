// trd_big.cu -- the large-rank path of libtrd (the paper's TR ranks
// [80, 80, 3, 20]).  Blocks with R_k^2 = r_k r_{k+1} > kBigR2 keep the per-entry
// passes (tcgen05 for K = r_k r_s <= 128, the SIMT pass writing D rows otherwise) and the
// d contraction (reduce_d_big_kernel), but their fp64 linear algebra is R_k^2 x R_k^2:
//   * Q_k refresh (Eq. 13): Gamma = Zd^T Zd with Zd[i][a r_{k+1} + b] = Z_k(i)[a][b]
//     (one dgemm of 2 I_k R^4 flops), permuted to Q_k[(a r_k + a'), (b r_{k+1} + b')]
//     = Gamma[(a r_{k+1} + b), (a' r_{k+1} + b')]  (reading R6);
//   * FGMC chain C = Q_{k+1} .. Q_{k-1} (Eq. 13): dgemm products, left-to-right or
//     right-to-left, whichever needs fewer flops (R^6 = 2.6e11 at R^2 = 6400 for the wrong
//     order), then Phi (phi_kernel) -> G;
//   * filtered solve (Eq. 10/16; readings R5, R23): lambda = lambda_rel tr(G)/R^2,
//     A = G + lambda I = L L^T (cuSOLVER potrf on the side stream, overlapping pass 1), then
//     h = d A^-1 G A^-1 row-wise: potrs with the I_k rows of d as right-hand sides, a dgemm by
//     G, potrs again (row-major I_k x R^2 is column-major R^2 x I_k: no transposes).  A failed
//     factorisation retries with lambda x 10 (from 2^-40 tr(G)/R^2 when lambda = 0) up to 3
//     times, then TRD_ERR_NOT_SPD -- decided on the host after one synchronisation per block,
//     which is why sweeps with large-rank blocks are not captured as CUDA graphs.
// cuBLAS / cuSOLVER are dlopen'ed on first use (contexts without large-rank blocks never load
// them).  Both are deterministic for a given GPU model and problem size, so data-parallel
// replicas stay bitwise equal.
#include <dlfcn.h>
#include <math.h>
#include <stdio.h>

#include <algorithm>

#include "trd_internal.cuh"

#include <stdarg.h>

namespace trd {
namespace {

// error record of the context (as trd_api.cu's fail(): CUDA-class failures are sticky)
trd_status fail(Context* c, trd_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  c->err = buf;
  if (st == TRD_ERR_CUDA) c->sticky = st;
  return st;
}

// ---- the few library entry points used (types from the public headers, by value) --------
typedef int (*blas_create_t)(void**);
typedef int (*blas_destroy_t)(void*);
typedef int (*blas_set_stream_t)(void*, cudaStream_t);
typedef int (*blas_dgemm_t)(void*, int, int, int, int, int, const double*, const double*, int, const double*,
                            int, const double*, double*, int);
typedef int (*sol_create_t)(void**);
typedef int (*sol_destroy_t)(void*);
typedef int (*sol_set_stream_t)(void*, cudaStream_t);
typedef int (*sol_potrf_buf_t)(void*, int, int, double*, int, int*);
typedef int (*sol_potrf_t)(void*, int, int, double*, int, double*, int, int*);
typedef int (*sol_potrs_t)(void*, int, int, int, const double*, int, double*, int, int*);
constexpr int kOpN = 0, kOpT = 1;          // CUBLAS_OP_N / CUBLAS_OP_T
constexpr int kFillLower = 0;              // CUBLAS_FILL_MODE_LOWER

struct BigApi {
  bool tried = false, ok = false;
  blas_create_t blas_create = nullptr;
  blas_destroy_t blas_destroy = nullptr;
  blas_set_stream_t blas_set_stream = nullptr;
  blas_dgemm_t dgemm = nullptr;
  sol_create_t sol_create = nullptr;
  sol_destroy_t sol_destroy = nullptr;
  sol_set_stream_t sol_set_stream = nullptr;
  sol_potrf_buf_t potrf_buf = nullptr;
  sol_potrf_t potrf = nullptr;
  sol_potrs_t potrs = nullptr;
};
BigApi g_big;

void* open_lib(const char* name) {
  void* h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    char path[256];
    snprintf(path, sizeof(path), "/usr/local/cuda/lib64/%s", name);
    h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  }
  return h;
}

bool load_big() {
  if (g_big.tried) return g_big.ok;
  g_big.tried = true;
  void* hb = open_lib("libcublas.so.12");
  void* hs = hb ? open_lib("libcusolver.so.11") : nullptr;
  if (!hb || !hs) return false;
  g_big.blas_create = (blas_create_t)dlsym(hb, "cublasCreate_v2");
  g_big.blas_destroy = (blas_destroy_t)dlsym(hb, "cublasDestroy_v2");
  g_big.blas_set_stream = (blas_set_stream_t)dlsym(hb, "cublasSetStream_v2");
  g_big.dgemm = (blas_dgemm_t)dlsym(hb, "cublasDgemm_v2");
  g_big.sol_create = (sol_create_t)dlsym(hs, "cusolverDnCreate");
  g_big.sol_destroy = (sol_destroy_t)dlsym(hs, "cusolverDnDestroy");
  g_big.sol_set_stream = (sol_set_stream_t)dlsym(hs, "cusolverDnSetStream");
  g_big.potrf_buf = (sol_potrf_buf_t)dlsym(hs, "cusolverDnDpotrf_bufferSize");
  g_big.potrf = (sol_potrf_t)dlsym(hs, "cusolverDnDpotrf");
  g_big.potrs = (sol_potrs_t)dlsym(hs, "cusolverDnDpotrs");
  g_big.ok = g_big.blas_create && g_big.blas_destroy && g_big.blas_set_stream && g_big.dgemm &&
             g_big.sol_create && g_big.sol_destroy && g_big.sol_set_stream && g_big.potrf_buf && g_big.potrf &&
             g_big.potrs;
  return g_big.ok;
}

int grid_of(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 32));
}

// ---- kernels --------------------------------------------------------------------------
// Zd[i][a r1 + b] = Z_k(i)[a][b] (fp64)
__global__ void big_zd_kernel(const float* __restrict__ Z, int64_t n, double* __restrict__ Zd) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    Zd[t] = (double)Z[t];
}

// Q[(a r0 + a') n1 + (b r1 + b')] = Gam[(a r1 + b) R2 + (a' r1 + b')]  (reading R6)
__global__ void big_qperm_kernel(const double* __restrict__ Gam, int r0, int r1, double* __restrict__ Q) {
  const int64_t R2 = (int64_t)r0 * r1, n1 = (int64_t)r1 * r1, tot = R2 * R2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / n1, col = t - row * n1;
    const int a = (int)(row / r0), ap = (int)(row % r0), b = (int)(col / r1), bp = (int)(col % r1);
    Q[t] = Gam[((int64_t)a * r1 + b) * R2 + (int64_t)ap * r1 + bp];
  }
}

// lambda of attempt `attempt` (R5, R23): tr(G) over one CTA (fixed-order tree), then
// lambda_0 = lambda_rel tr/n, lambda_j = 10 lambda_{j-1} (2^-40 tr/n when lambda_{j-1} = 0)
__global__ void __launch_bounds__(1024) big_lambda_kernel(const double* __restrict__ G, int n, double lambda_rel,
                                                          int attempt, DevScalars* sc) {
  __shared__ double red[1024];
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += G[(int64_t)i * n + i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tr = red[0];
    double lam = attempt == 0 ? lambda_rel * tr / n : sc->lambda;
    if (attempt > 0) lam = lam > 0.0 ? 10.0 * lam : ldexp(tr / n, -40);
    sc->lambda = lam;
    sc->h_lam = 0.0;
  }
}

// A = G + lambda I
__global__ void big_build_a_kernel(const double* __restrict__ G, int n, const DevScalars* __restrict__ sc,
                                   double* __restrict__ A) {
  const double lam = sc->lambda;
  const int64_t tot = (int64_t)n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t - i * n;
    A[t] = G[t] + (i == j ? lam : 0.0);
  }
}

// numpart[i] = <d(i), h(i)> (fixed-order tree over the CTA); h = 0 when the solve failed
__global__ void __launch_bounds__(256) big_num_kernel(const double* __restrict__ d, double* __restrict__ h, int R2,
                                                      const DevScalars* __restrict__ sc, double* __restrict__ numpart) {
  __shared__ double red[256];
  const int64_t i = blockIdx.x;
  const bool bad = sc->not_spd != 0;
  double t = 0.0;
  for (int o = threadIdx.x; o < R2; o += blockDim.x) {
    if (bad) h[i * R2 + o] = 0.0;
    else t += d[i * R2 + o] * h[i * R2 + o];
  }
  red[threadIdx.x] = t;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) numpart[i] = red[0];
}

__global__ void big_not_spd_kernel(DevScalars* sc) {
  if (threadIdx.x == 0 && blockIdx.x == 0) { sc->not_spd = 1; sc->h_lam = 0.0; }
}

}  // namespace

// ---- handles and workspaces ------------------------------------------------------------
trd_status big_init(Context* c, int64_t r2big, int64_t zd_rows) {
  // (big_gam also holds the I_k right-hand sides of the solve)
  const size_t gam = std::max((size_t)r2big * (size_t)r2big, (size_t)zd_rows * (size_t)r2big);
  if (!load_big())
    return fail(c, TRD_ERR_CUDA, "large-rank blocks (R_k^2 > %d) need libcublas.so.12 and libcusolver.so.11", kBigR2);
  if (g_big.blas_create(&c->blas) != 0 || g_big.sol_create(&c->solver) != 0)
    return fail(c, TRD_ERR_CUDA, "cublasCreate / cusolverDnCreate failed");
  const size_t n2 = (size_t)r2big * (size_t)r2big;
  if (cudaMalloc((void**)&c->big_A, n2 * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&c->big_gam, gam * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&c->big_zd, (size_t)zd_rows * r2big * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&c->big_info, sizeof(int)) != cudaSuccess ||
      cudaHostAlloc((void**)&c->big_info_h, sizeof(int), cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, TRD_ERR_OOM, "large-rank workspaces (%lld x %lld fp64) failed", (long long)r2big, (long long)r2big);
  }
  int lw = 0;
  if (g_big.potrf_buf(c->solver, kFillLower, (int)r2big, c->big_A, (int)r2big, &lw) != 0)
    return fail(c, TRD_ERR_CUDA, "cusolverDnDpotrf_bufferSize failed");
  c->big_lwork = std::max(lw, 1);
  if (cudaMalloc((void**)&c->big_work, (size_t)c->big_lwork * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, TRD_ERR_OOM, "potrf workspace failed");
  }
  return TRD_OK;
}

void big_destroy(Context* c) {
  if (c->blas && g_big.ok) g_big.blas_destroy(c->blas);
  if (c->solver && g_big.ok) g_big.sol_destroy(c->solver);
  c->blas = c->solver = nullptr;
  if (c->big_A) cudaFree(c->big_A);
  if (c->big_gam) cudaFree(c->big_gam);
  if (c->big_zd) cudaFree(c->big_zd);
  if (c->big_work) cudaFree(c->big_work);
  if (c->big_info) cudaFree(c->big_info);
  if (c->big_info_h) cudaFreeHost(c->big_info_h);
  c->big_A = c->big_gam = c->big_zd = c->big_work = nullptr;
  c->big_info = c->big_info_h = nullptr;
}

// row-major C (m x n) = A (m x q) B (q x n): column-major C^T = B^T A^T
trd_status big_dgemm(Context& c, cudaStream_t s, int m, int n, int q, const double* A, const double* B, double* C) {
  const double one = 1.0, zero = 0.0;
  if (g_big.blas_set_stream(c.blas, s) != 0 ||
      g_big.dgemm(c.blas, kOpN, kOpN, n, m, q, &one, B, n, A, q, &zero, C, n) != 0)
    return fail(&c, TRD_ERR_CUDA, "cublasDgemm (%d x %d x %d) failed", m, n, q);
  c.launches++;
  return TRD_OK;
}

trd_status big_q(Context& c, int k, cudaStream_t s) {
  const int r0 = c.ranks[k], r1 = c.ranks[(k + 1) % c.N];
  const int R2 = r0 * r1;
  const int64_t Ik = c.dims[k];
  big_zd_kernel<<<grid_of(Ik * R2), 256, 0, s>>>(c.Z + c.zoff[k], Ik * R2, c.big_zd);
  c.launches++;
  // Gamma = Zd^T Zd: with X = Zd^T column-major (R2 x Ik, ld R2), Gamma = X X^T (symmetric)
  const double one = 1.0, zero = 0.0;
  if (g_big.blas_set_stream(c.blas, s) != 0 ||
      g_big.dgemm(c.blas, kOpN, kOpT, R2, R2, (int)Ik, &one, c.big_zd, R2, c.big_zd, R2, &zero, c.big_gam, R2) != 0)
    return fail(&c, TRD_ERR_CUDA, "cublasDgemm (Q refresh) failed");
  c.launches++;
  big_qperm_kernel<<<grid_of((int64_t)R2 * R2), 256, 0, s>>>(c.big_gam, r0, r1, c.Q + c.qoff[k]);
  c.launches++;
  return TRD_OK;
}

trd_status big_gram(Context& c, const BlockPlan& bp, cudaStream_t s, const double* Qsrc, double* Gout) {
  const int N = c.N, k = bp.k;
  // chain Q_{k+1} .. Q_{k-1}: Q_m is r_m^2 x r_{m+1}^2
  int ms[kMaxN];
  for (int q = 0; q < N - 1; ++q) ms[q] = (k + 1 + q) % N;
  auto dim = [&](int m) { return (double)c.ranks[m] * c.ranks[m]; };
  double fl = 0.0, fr = 0.0;                 // flops of the two sequential orders
  for (int q = 1; q < N - 1; ++q) fl += dim(ms[0]) * dim(ms[q]) * dim((ms[q] + 1) % N);
  for (int q = N - 3; q >= 0; --q) fr += dim(ms[q]) * dim(ms[q + 1]) * dim((ms[N - 2] + 1) % N);
  double* bufs[2] = {c.chain_ws, c.chain_ws + c.chain_half};
  int which = 0;
  const double* cur;
  trd_status st = TRD_OK;
  if (fl <= fr) {                            // ((Q_{k+1} Q_{k+2}) Q_{k+3}) ..
    cur = Qsrc + c.qoff[ms[0]];
    const int rows = (int)dim(ms[0]);
    for (int q = 1; q < N - 1; ++q) {
      const int m = ms[q];
      st = big_dgemm(c, s, rows, (int)dim((m + 1) % N), (int)dim(m), cur, Qsrc + c.qoff[m], bufs[which]);
      if (st) return st;
      cur = bufs[which];
      which ^= 1;
    }
  } else {                                   // .. Q_{k-3} (Q_{k-2} Q_{k-1})
    cur = Qsrc + c.qoff[ms[N - 2]];
    const int cols = (int)dim((ms[N - 2] + 1) % N);
    for (int q = N - 3; q >= 0; --q) {
      const int m = ms[q];
      st = big_dgemm(c, s, (int)dim(m), cols, (int)dim((m + 1) % N), Qsrc + c.qoff[m], cur, bufs[which]);
      if (st) return st;
      cur = bufs[which];
      which ^= 1;
    }
  }
  launch_phi(c, bp, cur, Gout, s);
  return TRD_OK;
}

static trd_status big_potrf(Context& c, int n, cudaStream_t s) {
  if (g_big.sol_set_stream(c.solver, s) != 0 ||
      g_big.potrf(c.solver, kFillLower, n, c.big_A, n, c.big_work, c.big_lwork, c.big_info) != 0)
    return fail(&c, TRD_ERR_CUDA, "cusolverDnDpotrf (n = %d) failed", n);
  c.launches++;
  if (cudaMemcpyAsync(c.big_info_h, c.big_info, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return fail(&c, TRD_ERR_CUDA, "potrf info copy failed");
  return TRD_OK;
}

// side stream: lambda, A = G + lambda I, A = L L^T (attempt 0; big_h retries if needed)
trd_status big_factor(Context& c, const BlockPlan& bp, cudaStream_t s, const double* G) {
  const int n = bp.R2;
  c.big_G = G;
  if (c.cfg.scaling == TRD_SCALING_NONE) return TRD_OK;
  big_lambda_kernel<<<1, 1024, 0, s>>>(G, n, c.cfg.lambda_rel, 0, c.sc);
  big_build_a_kernel<<<grid_of((int64_t)n * n), 256, 0, s>>>(G, n, c.sc, c.big_A);
  c.launches += 2;
  return big_potrf(c, n, s);
}

// main stream, after the d allreduce: h = d A^-1 G A^-1 (or h = d), num partials
trd_status big_h(Context& c, const BlockPlan& bp, cudaStream_t s) {
  const int n = bp.R2;
  const int64_t Ik = c.dims[bp.k];
  if (c.cfg.scaling == TRD_SCALING_NONE) {   // 'gradient descent' arm: h = d
    if (cudaMemcpyAsync(c.h, c.dvec, (size_t)(Ik * n) * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return fail(&c, TRD_ERR_CUDA, "h = d copy failed");
  } else {
    // the side stream's factorisation has finished (ev_join); its potrf status
    if (cudaEventSynchronize(c.ev_join) != cudaSuccess) return fail(&c, TRD_ERR_CUDA, "side-stream sync failed");
    int attempt = 0;
    while (*c.big_info_h != 0 && attempt < 3) {   // R23: lambda x 10, at most 3 retries
      ++attempt;
      big_lambda_kernel<<<1, 1024, 0, s>>>(c.big_G, n, c.cfg.lambda_rel, attempt, c.sc);
      big_build_a_kernel<<<grid_of((int64_t)n * n), 256, 0, s>>>(c.big_G, n, c.sc, c.big_A);
      c.launches += 2;
      if (trd_status st = big_potrf(c, n, s)) return st;
      if (cudaStreamSynchronize(s) != cudaSuccess) return fail(&c, TRD_ERR_CUDA, "potrf retry sync failed");
    }
    if (*c.big_info_h != 0) {
      big_not_spd_kernel<<<1, 32, 0, s>>>(c.sc);   // h = 0 below: the block is skipped
      c.launches++;
    } else {
      // U = A^-1 d^T (the I_k rows of d as right-hand sides), h^T = A^-1 (G U)
      if (cudaMemcpyAsync(c.big_gam, c.dvec, (size_t)(Ik * n) * sizeof(double), cudaMemcpyDeviceToDevice, s) !=
          cudaSuccess)
        return fail(&c, TRD_ERR_CUDA, "d copy failed");
      const double one = 1.0, zero = 0.0;
      if (g_big.sol_set_stream(c.solver, s) != 0 ||
          g_big.potrs(c.solver, kFillLower, n, (int)Ik, c.big_A, n, c.big_gam, n, c.big_info) != 0 ||
          g_big.blas_set_stream(c.blas, s) != 0 ||
          g_big.dgemm(c.blas, kOpN, kOpN, n, (int)Ik, n, &one, c.big_G, n, c.big_gam, n, &zero, c.h, n) != 0 ||
          g_big.potrs(c.solver, kFillLower, n, (int)Ik, c.big_A, n, c.h, n, c.big_info) != 0)
        return fail(&c, TRD_ERR_CUDA, "large-rank filtered solve (potrs / dgemm) failed");
      c.launches += 3;
    }
  }
  big_num_kernel<<<(unsigned)Ik, 256, 0, s>>>(c.dvec, c.h, n, c.sc, c.numpart);
  c.launches++;
  return TRD_OK;
}

}  // namespace trd

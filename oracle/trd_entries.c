/*
 * trd_entries.c -- entry-wise float64 form of the two per-entry sums of one block of
 * Algorithm 1, for the oracle at full problem size.
 *
 * TEST INFRASTRUCTURE ONLY (like oracle/trd_oracle.py): only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code with
 * the CUDA path (paper_2305_09044_b200/csrc) and includes none of its headers.
 *
 * What it computes (plain loops, float64, no blocking of the arithmetic):
 *   for every multi-index j = (i_{k+1}, .., i_{k-1}) of the sketch  X_{m != k} I_m   (Eq. 14)
 *     S(j) = Z_{k+1}(i_{k+1}) Z_{k+2}(i_{k+2}) .. Z_{k-1}(i_{k-1})   in R^{r_{k+1} x r_k}
 *                                                                     (Thm 1)
 *     for every i_k in I_k with P(i_k, j) = 1 (observed):
 *       e = x - Tr(Z_k(i_k) S(j))                                      (Thm 1 / Eq. 9)
 *       w = exp(-e^2 / (2 sigma^2))   (reading R1; w = 1 when sigma = inf)
 *       pass 1:  d[i_k][c + r_k b] += w e S(j)[b][c]                   (Eq. 9/15)
 *                sum_e2 += e^2, welsch += sigma^2 (1 - w), n += 1
 *       pass 2:  t = sum_{a,b} h[i_k][a + r_k b] S(j)[b][a],  den += w t^2   (Eq. 12/18)
 * S(j) is multiplied left to right; the product of the first q factors is kept while the
 * later indices run (the same operations in the same order as recomputing it per j).
 * Sums are formed per index of the outermost mode and then added in index order, so the
 * result does not depend on the number of threads.
 *
 * Layouts: core m is double[r_m][I_m][r_{m+1}] (paper index order);
 * X has linear index lin = i_0 + I_0 (i_1 + I_1 (..)) (Def. 2); the mask is
 * bit lin % 32 of word lin / 32; values are dense (values[lin]) or packed (the value of the
 * n-th observed entry at values[n], with prefix[w] = number of set bits in words < w).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OC_MAX_N 8

typedef struct {
  int N, k;
  const int64_t* dims;            /* I_m                                             */
  const int32_t* ranks;           /* r_m, ring r_N = r_0                             */
  const double* const* cores;     /* Z_m[a][i][b]                                    */
  const int64_t* const* sets;     /* index set of each mode                          */
  const int64_t* sizes;           /* |I_m|                                           */
  const uint32_t* mask;
  const float* values;
  const uint64_t* prefix;         /* NULL: dense values                              */
  double sigma;
  int sigma_inf;
  const double* h;                /* pass 2: h[i_k][a + r_k b], i_k global            */
} oc_block;

static int observed(const oc_block* B, int64_t lin, double* x) {
  const uint32_t w = B->mask[lin >> 5];
  const uint32_t bit = (uint32_t)(lin & 31);
  if (!((w >> bit) & 1u)) return 0;
  int64_t vi = lin;
  if (B->prefix) vi = (int64_t)B->prefix[lin >> 5] + __builtin_popcount(w & ((1u << bit) - 1u));
  *x = (double)B->values[vi];
  return 1;
}

/* C (ra x rc) = A (ra x rb) * Z_m(i) (rb x rc) */
static void matmul_slice(const double* A, const double* Zm, int64_t Im, int64_t i, int ra, int rb,
                         int rc, double* C) {
  for (int a = 0; a < ra; ++a)
    for (int c = 0; c < rc; ++c) {
      double s = 0.0;
      for (int b = 0; b < rb; ++b) s += A[a * rb + b] * Zm[((int64_t)b * Im + i) * rc + c];
      C[a * rc + c] = s;
    }
}

/* one value of the outermost mode (position o in its index set): all j with that index */
static void outer_slice(const oc_block* B, int pass, int64_t o, double* d, double* st,
                        double* abs_e, int64_t* n_abs) {
  const int N = B->N, k = B->k;
  const int rk = B->ranks[k], rk1 = B->ranks[(k + 1) % N];
  const int64_t Ik = B->sizes[k];
  int order[OC_MAX_N];
  int64_t stride[OC_MAX_N];
  int64_t s = 1;
  for (int m = 0; m < N; ++m) { stride[m] = s; s *= B->dims[m]; }
  for (int q = 0; q < N - 1; ++q) order[q] = (k + 1 + q) % N;
  /* prefix products P_q = Z_{order[0]}(.) .. Z_{order[q]}(.), rows r_{k+1} */
  double* P[OC_MAX_N];
  int pr[OC_MAX_N];                 /* columns of P_q */
  for (int q = 0; q < N - 1; ++q) {
    const int m = order[q];
    pr[q] = B->ranks[(m + 1) % N];
    P[q] = (double*)malloc(sizeof(double) * rk1 * pr[q]);
  }
  int64_t pos[OC_MAX_N];
  pos[0] = o;
  for (int q = 1; q < N - 1; ++q) pos[q] = 0;
  /* P_0 = Z_{order[0]}(i) */
  {
    const int m = order[0];
    const int64_t i = B->sets[m][o];
    const double* Z = B->cores[m];
    for (int a = 0; a < rk1; ++a)
      for (int c = 0; c < pr[0]; ++c) P[0][a * pr[0] + c] = Z[((int64_t)a * B->dims[m] + i) * pr[0] + c];
  }
  int valid = 1;                     /* levels 1..valid-1 are current */
  const double s2 = B->sigma * B->sigma;
  const double inv2s2 = B->sigma_inf ? 0.0 : 0.5 / s2;
  const double* Zk = B->cores[k];
  for (;;) {
    for (int q = valid; q < N - 1; ++q) {
      const int m = order[q];
      const int rin = B->ranks[m];
      matmul_slice(P[q - 1], B->cores[m], B->dims[m], B->sets[m][pos[q]], rk1, rin, pr[q], P[q]);
    }
    valid = N - 1;
    const double* S = P[N - 2];      /* S(j): r_{k+1} x r_k, S[b][c] = S[b * rk + c] */
    int64_t base = 0;
    for (int q = 0; q < N - 1; ++q) base += B->sets[order[q]][pos[q]] * stride[order[q]];
    for (int64_t t = 0; t < Ik; ++t) {
      const int64_t ik = B->sets[k][t];
      double x;
      if (!observed(B, base + ik * stride[k], &x)) continue;
      double xhat = 0.0;             /* Tr(Z_k(i_k) S(j)) = sum_{a,b} Z_k[a][i_k][b] S[b][a] */
      for (int a = 0; a < rk; ++a)
        for (int b = 0; b < rk1; ++b) xhat += Zk[((int64_t)a * B->dims[k] + ik) * rk1 + b] * S[b * rk + a];
      const double e = x - xhat;
      const double w = B->sigma_inf ? 1.0 : exp(-(e * e) * inv2s2);
      if (pass == 1) {
        const double c = w * e;
        double* drow = d + ik * (int64_t)(rk * rk1);
        for (int b = 0; b < rk1; ++b)
          for (int cc = 0; cc < rk; ++cc) drow[cc + rk * b] += c * S[b * rk + cc];
        st[0] += e * e;
        if (!B->sigma_inf) st[1] += s2 * (1.0 - w);
        st[2] += 1.0;
        if (abs_e) abs_e[(*n_abs)++] = fabs(e);
      } else {
        const double* hrow = B->h + ik * (int64_t)(rk * rk1);
        double tt = 0.0;
        for (int a = 0; a < rk; ++a)
          for (int b = 0; b < rk1; ++b) tt += hrow[a + rk * b] * S[b * rk + a];
        st[3] += w * tt * tt;
      }
    }
    /* next j: advance the innermost level (order[N-2]) first */
    int q = N - 2;
    while (q >= 1) {
      if (++pos[q] < B->sizes[order[q]]) break;
      pos[q] = 0;
      --q;
    }
    if (q < 1) break;
    valid = q;
  }
  for (int q = 0; q < N - 1; ++q) free(P[q]);
}

/* Observed entries of the sketch with outermost index position o (for the |e| offsets). */
static int64_t outer_count(const oc_block* B, int64_t o) {
  const int N = B->N, k = B->k;
  int order[OC_MAX_N];
  int64_t stride[OC_MAX_N], pos[OC_MAX_N];
  int64_t s = 1;
  for (int m = 0; m < N; ++m) { stride[m] = s; s *= B->dims[m]; }
  for (int q = 0; q < N - 1; ++q) { order[q] = (k + 1 + q) % N; pos[q] = 0; }
  pos[0] = o;
  int64_t n = 0;
  for (;;) {
    int64_t base = 0;
    for (int q = 0; q < N - 1; ++q) base += B->sets[order[q]][pos[q]] * stride[order[q]];
    for (int64_t t = 0; t < B->sizes[k]; ++t) {
      const int64_t lin = base + B->sets[k][t] * stride[k];
      n += (B->mask[lin >> 5] >> (lin & 31)) & 1u;
    }
    int q = N - 2;
    while (q >= 1) {
      if (++pos[q] < B->sizes[order[q]]) break;
      pos[q] = 0;
      --q;
    }
    if (q < 1) break;
  }
  return n;
}

/*
 * pass 1 (pass = 1): d_out[I_k x R^2] (zeroed here; rows i_k global), stats_out[0..2] =
 *   {sum_e2, welsch, n}; abs_e_out (may be NULL) receives |e| of every observed entry.
 * pass 2 (pass = 2): stats_out[3] = den (h given).
 * Returns 0, or -1 on bad arguments / allocation failure.
 */
int oc_block_pass(int pass, int N, int k, const int64_t* dims, const int32_t* ranks,
                  const double* const* cores, const int64_t* const* sets, const int64_t* sizes,
                  const uint32_t* mask, const float* values, const uint64_t* prefix, double sigma,
                  int sigma_inf, const double* h, double* d_out, double* stats_out, double* abs_e_out,
                  int64_t abs_e_cap) {
  if (N < 2 || N > OC_MAX_N || k < 0 || k >= N || (pass != 1 && pass != 2) || (pass == 2 && !h)) return -1;
  oc_block B = {N, k, dims, ranks, cores, sets, sizes, mask, values, prefix, sigma, sigma_inf, h};
  const int rk = ranks[k], rk1 = ranks[(k + 1) % N];
  const int64_t R2 = (int64_t)rk * rk1;
  const int64_t Ik_tot = dims[k];
  const int m0 = (k + 1) % N;
  const int64_t n_out = sizes[m0];
  int64_t* off = NULL;
  if (pass == 1 && abs_e_out) {
    off = (int64_t*)calloc((size_t)n_out + 1, sizeof(int64_t));
    if (!off) return -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t o = 0; o < n_out; ++o) off[o + 1] = outer_count(&B, o);
    for (int64_t o = 0; o < n_out; ++o) off[o + 1] += off[o];
    if (off[n_out] > abs_e_cap) { free(off); return -1; }
  }
  const int64_t dsz = pass == 1 ? Ik_tot * R2 : 0;
  double* dpart = (double*)calloc((size_t)(n_out * dsz + 1), sizeof(double));
  double* spart = (double*)calloc((size_t)n_out * 4, sizeof(double));
  if (!dpart || !spart) { free(dpart); free(spart); free(off); return -1; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t o = 0; o < n_out; ++o) {
    int64_t na = 0;
    outer_slice(&B, pass, o, dpart + o * dsz, spart + o * 4, off ? abs_e_out + off[o] : NULL, &na);
  }
  if (pass == 1) {
    memset(d_out, 0, sizeof(double) * (size_t)dsz);
    for (int64_t o = 0; o < n_out; ++o)
      for (int64_t t = 0; t < dsz; ++t) d_out[t] += dpart[o * dsz + t];
  }
  double st[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t o = 0; o < n_out; ++o)
    for (int j = 0; j < 4; ++j) st[j] += spart[o * 4 + j];
  if (pass == 1) { stats_out[0] = st[0]; stats_out[1] = st[1]; stats_out[2] = st[2]; }
  else stats_out[3] = st[3];
  free(dpart);
  free(spart);
  free(off);
  return 0;
}

/* Def. 1: out[t] = Tr(Z_0(i_0) Z_1(i_1) .. Z_{N-1}(i_{N-1})) at linear index lin[t] */
int oc_reconstruct(int N, const int64_t* dims, const int32_t* ranks, const double* const* cores,
                   const int64_t* lin, int64_t n, double* out) {
  if (N < 2 || N > OC_MAX_N) return -1;
  int rmax = 1;
  for (int m = 0; m < N; ++m) rmax = ranks[m] > rmax ? ranks[m] : rmax;
  int fail = 0;
#pragma omp parallel
  {
    double* A = (double*)malloc(sizeof(double) * rmax * rmax);
    double* C = (double*)malloc(sizeof(double) * rmax * rmax);
    if (!A || !C) fail = 1;
#pragma omp for schedule(static)
    for (int64_t t = 0; t < n; ++t) {
      if (!A || !C) continue;
      int64_t l = lin[t], ix[OC_MAX_N];
      for (int m = 0; m < N; ++m) { ix[m] = l % dims[m]; l /= dims[m]; }
      const int r0 = ranks[0];
      int rc = ranks[1 % N];
      for (int a = 0; a < r0; ++a)
        for (int c = 0; c < rc; ++c) A[a * rc + c] = cores[0][((int64_t)a * dims[0] + ix[0]) * rc + c];
      for (int m = 1; m < N; ++m) {
        const int rin = ranks[m], rout = ranks[(m + 1) % N];
        matmul_slice(A, cores[m], dims[m], ix[m], r0, rin, rout, C);
        memcpy(A, C, sizeof(double) * r0 * rout);
      }
      double tr = 0.0;
      for (int a = 0; a < r0; ++a) tr += A[a * r0 + a];
      out[t] = tr;
    }
    free(A);
    free(C);
  }
  return fail ? -1 : 0;
}

// Microbenchmark: tcgen05.mma kind::f16 issue/execution rate for the operand layouts used by
// libtrd's pass kernels (A in TMEM or smem, B in smem with the SWIZZLE_NONE core-matrix
// layout), M = 128, K = 16 per instruction, N in {64, 128, 256}.  One CTA per SM, one thread
// issues `iters` MMAs into the same accumulator, then commits and waits.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_rate tc_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int b_mn) {
  return (1u << 4) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, bool TS, int LAYOUT>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  if (tid == 0) {
    constexpr uint32_t idesc = make_idesc(128, N, 0);
    const uint32_t a_s = smem_u32(smem), b_s = smem_u32(smem + 32768);
    // K-major: core matrix (row group g, k group h) at (g*8 + h)*128 (HK = 8, i.e. KP = 64)
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int ks = i & 3;
      uint64_t db, da;
      if (LAYOUT == 0) {
        db = make_sdesc(b_s + ks * 256, 128, 8 * 128, 0);
        da = make_sdesc(a_s + ks * 256, 128, 8 * 128, 0);
      } else if (LAYOUT == 1) {   // libtrd layout L2: [hi KP | lo KP] per row, SBO = 2 HK * 128
        db = make_sdesc(b_s + ks * 256, 128, 16 * 128, 0);
        da = make_sdesc(a_s + ks * 256, 128, 16 * 128, 0);
      } else {  // SWIZZLE_128B K-major: rows of 128 B, 8-row atoms of 1024 B, SBO = 1024
        db = make_sdesc(b_s + ks * 32, 16, 1024, 2);
        da = make_sdesc(a_s + ks * 32, 16, 1024, 2);
      }
      const uint32_t acc = i > 0;
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tb), "r"(tb + 256 + ks * 8), "l"(db), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tb), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t ok = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    } while (!ok);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

// libtrd pass-1 tile sequence: GEMM1 (3 x 4 MMAs, N = 64, B K-major) into S, commit; GEMM2
// (3 x 4 MMAs, N = KP = 64, B MN-major, A = P from TMEM) into D, commit x2 -- per tile
__device__ volatile int g_stop;
__device__ float g_src[64 * 4096 + 4096];

template <int NT>
__global__ void __launch_bounds__(384, 1) bench_seq(long long* out, int tiles, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  if (tid == 0) {
    constexpr uint32_t id1 = make_idesc(128, NT, 0), id2 = make_idesc(128, 64, 1);
    const uint32_t b_s = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      for (int term = 0; term < 3; ++term)
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t db = make_sdesc(b_s + term * 8192 + ks * 256, 128, 8 * 128, 0);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                       ::"r"(tb + (t & 1) * 64), "r"(tb + 448 + ks * 8), "l"(db), "r"(id1), "r"((uint32_t)(term | ks)));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      for (int term = 0; term < 3; ++term)
        for (int ks = 0; ks < NT / 16; ++ks) {
          const uint64_t db = make_sdesc(b_s + term * 8192 + ks * 2 * 8 * 128, 8 * 128, 128, 0);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                       ::"r"(tb + 256), "r"(tb + 128 + (t & 1) * 64 + ks * 8), "l"(db), "r"(id2), "r"(1u));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t1 - t0; }
    g_stop = 1;
  } else if (tid >= 128 && mode != 0) {
    // interfering warps (4..11): TMEM loads of columns 320..383 and/or smem traffic
    const int w = (tid >> 5) & 3;
    float acc = 0.f;
    float4* sm4 = reinterpret_cast<float4*>(smem + 65536) + (tid - 128) * 4;
    while (!g_stop) {
      if (mode & 1) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tb + ((uint32_t)(w * 32) << 16) + 320));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += __uint_as_float(v[0]) + __uint_as_float(v[15]);
      }
      if (mode & 2) {
        float4 x = sm4[0];
        sm4[1] = make_float4(x.x + 1.f, x.y, x.z, x.w);
        float4 y = sm4[2];
        sm4[3] = y;
        acc += x.x + y.y;
      }
      if (mode & 4) {
        uint32_t v[16];
        for (int u = 0; u < 16; ++u) v[u] = __float_as_uint(acc + u);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(tb + ((uint32_t)(w * 32) << 16) + 384), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]),
                       "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]),
                       "r"(v[13]), "r"(v[14]), "r"(v[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
    }
    if (acc == 12345.f) out[2] = 1;
  } else if (tid == 96 && mode >= 8) {
    // TMA bulk copies (16 KB) global -> smem, back to back
    __shared__ uint64_t tbar;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&tbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
    uint32_t ph = 0;
    while (!g_stop) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&tbar)), "r"(16384) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(smem + 65536 + 32768)), "l"(g_src + (blockIdx.x & 63) * 4096), "r"(16384),
                     "r"(smem_u32(&tbar)) : "memory");
      uint32_t ok = 0;
      do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&tbar)), "r"(ph) : "memory");
      } while (!ok);
      ph ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int NT>
void run_seq(int tiles) {
  long long* d;
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(bench_seq<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const char* names[9] = {"none", "TMEM ld", "smem", "TMEM ld + smem", "TMEM st", "", "", "all SIMT", "TMA bulk"};
  for (int mode : {0, 1, 2, 3, 4, 7, 8}) {
    int zero = 0;
    cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    bench_seq<NT><<<148, 384, 128 * 1024>>>(d, tiles, mode);
    cudaError_t err = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("pass-1 tile sequence NT=%d, interference %-15s: %.1f cycles per tile (%s)\n", NT, names[mode],
           (double)h[0] / tiles, cudaGetErrorString(err));
  }
  cudaFree(d);
}

template <int N, bool TS, int LAYOUT>
void run(const char* name, int iters) {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench<N, TS, LAYOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  bench<N, TS, LAYOUT><<<148, 128, 96 * 1024>>>(d, iters);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<N, TS, LAYOUT><<<148, 128, 96 * 1024>>>(d, iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 16 * (double)iters * 148;
  printf("%-22s N=%3d iters=%d: issue %.1f cyc/mma, complete %.1f cyc/mma, %.1f TFLOP/s (%s)\n", name, N, iters,
         (double)h[0] / iters, (double)h[1] / iters, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(d);
}

int main(int argc, char** argv) {
  const int it = 20000;
  if (argc > 1) {   // layout comparison only
    run<64, true, 0>("TS none SBO1024", it);
    run<64, true, 1>("TS none SBO2048", it);
    run<128, true, 0>("TS none SBO1024", it);
    run<128, true, 1>("TS none SBO2048", it);
    run<64, false, 0>("SS none SBO1024", it);
    run<64, false, 1>("SS none SBO2048", it);
    return 0;
  }
  run<64, true, 0>("TS none", it);
  run<128, true, 0>("TS none", it);
  run<256, true, 0>("TS none", it);
  run<64, false, 0>("SS none", it);
  run<128, false, 0>("SS none", it);
  run<256, false, 0>("SS none", it);
  run<64, false, 2>("SS sw128", it);
  run<128, false, 2>("SS sw128", it);
  run<256, false, 2>("SS sw128", it);
  run<64, true, 2>("TS sw128", it);
  run_seq<64>(2000);
  run<256, true, 2>("TS sw128", it);
  return 0;
}

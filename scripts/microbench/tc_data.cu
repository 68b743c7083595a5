// Microbenchmark: does the tcgen05.mma kind::f16 rate depend on the operand values?
// One CTA per SM; TMEM A (TS) or smem A (SS) and smem B filled with zeros, 1.0, or
// pseudo-random fp16 in [-1, 1]; one thread issues `iters` M=128 K=16 MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_data tc_data.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t hrand(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t fill_word(int mode, uint32_t idx) {
  if (mode == 0) return 0u;
  if (mode == 1) return 0x3c003c00u;
  const uint32_t h = hrand(idx * 2654435761u + 12345u);
  const __half a = __float2half((float)(h & 0xffff) / 32768.f - 1.f);
  const __half b = __float2half((float)(h >> 16) / 32768.f - 1.f);
  return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 96 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = fill_word(mode, i + blockIdx.x * 7919u);
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
  {  // TMEM A: columns 256..287 of this warp's lanes
    const uint32_t lb = tb + ((uint32_t)((tid >> 5) * 32) << 16) + 256;
    for (int c = 0; c < 32; ++c) {
      const uint32_t v = fill_word(mode, tid * 64 + c + 99991u * blockIdx.x);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lb + c), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    constexpr uint32_t idesc = make_idesc(128, N);
    const uint32_t a_s = smem_u32(smem), b_s = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int ks = i & 3;
      const uint64_t db = make_sdesc(b_s + ks * 256, 128, 8 * 128);
      const uint32_t acc = i > 0;
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tb), "r"(tb + 256 + ks * 8), "l"(db), "r"(idesc), "r"(acc));
      } else {
        const uint64_t da = make_sdesc(a_s + ks * 256, 128, 8 * 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tb), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t ok = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    } while (!ok);
    long long t2 = clock64();
    if (blockIdx.x == 0) out[0] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int N, bool TS>
void run(int iters) {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const char* mn[3] = {"zeros", "ones", "random"};
  for (int mode = 0; mode < 3; ++mode) {
    bench<N, TS><<<148, 128, 96 * 1024>>>(d, iters, mode);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<N, TS><<<148, 128, 96 * 1024>>>(d, iters, mode);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * N * 16 * (double)iters * 148;
    printf("%s N=%3d %-6s: %.1f cyc/mma, %.1f TFLOP/s, %.3f ms (%s)\n", TS ? "TS" : "SS", N, mn[mode],
           (double)h / iters, flops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(err));
  }
  cudaFree(d);
}

int main() {
  const int it = 200000;
  run<64, true>(it);
  run<128, true>(it);
  run<64, false>(it);
  run<128, false>(it);
  run<256, false>(it);
  return 0;
}

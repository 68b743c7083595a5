// Microbenchmark: does mbarrier polling by other warps slow down tcgen05.mma issue?
// One CTA per SM, 512 threads; thread 0 issues M=128 N=64 K=16 TS MMAs; warps 1..15 wait on
// an mbarrier that completes only after the MMAs: mode 0 = no waiters, 1 = all lanes poll
// try_wait, 2 = one lane per warp polls then __syncwarp, 3 = all lanes poll with nanosleep,
// 4 = all lanes poll test_wait (non-suspending).
#include <cstdio>
#include <cstdint>
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
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok;
}

__global__ void __launch_bounds__(512, 1) bench(long long* out, int iters, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar, done;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 32 * 1024 / 4; i += 512) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&done)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  const uint32_t dn = smem_u32(&done);
  if (tid == 0) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t b_s = smem_u32(smem);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int ks = i & 3;
      const uint64_t db = make_sdesc(b_s + ks * 256, 128, 8 * 128);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                   ::"r"(tb), "r"(tb + 256 + ks * 8), "l"(db), "r"(idesc), "r"((uint32_t)(i > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    while (!try_wait(smem_u32(&bar), 0)) {}
    long long t2 = clock64();
    if (blockIdx.x == 0) out[0] = t2 - t0;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dn) : "memory");
  } else if (tid >= 32 && mode != 0) {
    if (mode == 1) { while (!try_wait(dn, 0)) {} }
    else if (mode == 2) { if (lane == 0) { while (!try_wait(dn, 0)) {} } __syncwarp(); }
    else if (mode == 3) { while (!try_wait(dn, 0)) { __nanosleep(200); } }
    else if (mode == 4) { while (!test_wait(dn, 0)) {} }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const char* nm[5] = {"no waiters", "all lanes try_wait", "lane 0 try_wait", "try_wait+nanosleep", "all lanes test_wait"};
  for (int mode = 0; mode < 5; ++mode) {
    bench<<<148, 512, 64 * 1024>>>(d, 20000, mode);
    cudaError_t err = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-22s: %.1f cycles per MMA (%s)\n", nm[mode], (double)h / 20000, cudaGetErrorString(err));
  }
  return 0;
}

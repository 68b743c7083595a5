// Microbenchmark: the pass-2 MMA stream of libtrd (3-term split GEMM1 per 64-column tile,
// A hi|lo in TMEM, B hi|lo tiles in a 6-stage smem ring, D in a 4-slot TMEM ring, two
// commits per tile) with variations that remove one feature at a time.
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
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t ta, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(ta), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int KP = 64, HK = 8, NB = 6, TD = 4;
constexpr int B_BYTES = 2 * 64 * KP * 2, B_LO = 64 * KP * 2;

// flags: 1 no commits, 2 fixed B stage, 4 fixed D slot, 8 single term (hi.hi x3),
//        16 accumulate flag always 1, 32 acc=0 only at first
__global__ void __launch_bounds__(128, 1) bench(long long* out, int tiles, int flags) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bars[16];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < NB * B_BYTES / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  if (tid == 0) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t bring = smem_u32(smem);
    const uint32_t COL_A = TD * 64;
    long long t0 = clock64();
    for (int i = 0; i < tiles; ++i) {
      const int s = (flags & 4) ? 0 : (i % TD);
      const int ab = (i / 50) & 1;
      const uint32_t bH = bring + ((flags & 2) ? 0 : (i % NB)) * B_BYTES;
      const uint32_t acol = tb + COL_A + ab * KP;
      uint32_t acc = (flags & 16) ? 1u : 0u;
      for (int term = 0; term < 3; ++term) {
        const uint32_t aa = acol + ((term == 2 && !(flags & 8)) ? KP / 2 : 0);
        const uint32_t bb = bH + ((term == 1 && !(flags & 8)) ? B_LO : 0u);
        for (int ks = 0; ks < KP / 16; ++ks) {
          const uint64_t db = make_sdesc(bb + ks * 256, 128, HK * 128);
          mma_ts(tb + 64 * s, aa + ks * 8, db, idesc, acc);
          acc = 1;
        }
      }
      if (!(flags & 1)) { commit(&bars[s]); commit(&bars[8 + (i % NB)]); }
    }
    commit(&bars[15]);
    uint32_t ok = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bars[15])), "r"(0) : "memory");
    } while (!ok);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
  return pred;
}
// variant: mode 0 = one thread, descriptors as base + offset; mode 1 = whole warp 0 runs the
// loop, elect.sync issues; mode 2 = like 1 but fully unrolled 12 MMAs with constant offsets
__global__ void __launch_bounds__(128, 1) bench2(long long* out, int tiles, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bars[16];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < NB * B_BYTES / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  const bool runner = (mode == 0) ? (tid == 0) : (tid < 32);
  if (runner) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t bring = smem_u32(smem);
    const uint32_t COL_A = TD * 64;
    const uint64_t desc0 = make_sdesc(bring, 128, HK * 128);
    long long t0 = clock64();
    for (int i = 0; i < tiles; ++i) {
      const int s = i % TD;
      const int ab = (i / 50) & 1;
      const uint64_t dB = desc0 + (uint64_t)(((i % NB) * B_BYTES) >> 4);
      const uint32_t acol = tb + COL_A + ab * KP;
      const uint32_t dst = tb + 64 * s;
      if (mode == 0) {
#pragma unroll
        for (int term = 0; term < 3; ++term)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_ts(dst, acol + (term == 2 ? KP / 2 : 0) + ks * 8,
                   dB + (uint64_t)(((term == 1 ? B_LO : 0) + ks * 256) >> 4), idesc, (term | ks) ? 1u : 0u);
      } else {
        if (elect_one()) {
#pragma unroll
          for (int term = 0; term < 3; ++term)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              mma_ts(dst, acol + (term == 2 ? KP / 2 : 0) + ks * 8,
                     dB + (uint64_t)(((term == 1 ? B_LO : 0) + ks * 256) >> 4), idesc, (term | ks) ? 1u : 0u);
          commit(&bars[s]);
          commit(&bars[8 + (i % NB)]);
        }
        __syncwarp();
        continue;
      }
      commit(&bars[s]);
      commit(&bars[8 + (i % NB)]);
    }
    if (mode == 0 || elect_one()) {
      commit(&bars[15]);
      uint32_t ok = 0;
      do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bars[15])), "r"(0) : "memory");
      } while (!ok);
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    if (mode != 0) __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * B_BYTES);
  const int fl[] = {0, 1, 2, 4, 8, 16, 1 | 2 | 4, 1 | 2 | 4 | 8, 6, 3, 5};
  for (int f : fl) {
    bench<<<148, 128, NB * B_BYTES>>>(d, 4000, f);
    cudaError_t err = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("flags %2d: %.1f cycles per tile (12 MMAs) = %.1f per MMA (%s)\n", f, (double)h / 4000,
           (double)h / 4000 / 12, cudaGetErrorString(err));
  }
  cudaFuncSetAttribute(bench2, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * B_BYTES);
  for (int m = 0; m < 2; ++m) {
    bench2<<<148, 128, NB * B_BYTES>>>(d, 4000, m);
    cudaError_t err = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("bench2 mode %d: %.1f cycles per tile = %.1f per MMA (%s)\n", m, (double)h / 4000, (double)h / 4000 / 12,
           cudaGetErrorString(err));
  }
  return 0;
}

// FP32 FMA peak of the B200 (the roofline denominator of the pass kernels).
// 148 x 8 CTAs x 256 threads (full occupancy), 16 independent FMA chains per thread; prints
// one JSON line: achieved TFLOP/s (2 flops per FMA) over a ~0.2 s launch, best of 5.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) fma_kernel(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  if (s == 123.456f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;   // keep the chains live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = sms * 8, threads = 256, iters = 1 << 16;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_kernel<<<blocks, threads>>>(out, 1024, 0.999f, 1e-3f);   // warm-up
  cudaDeviceSynchronize();
  double best = 0.0, best_ms = 0.0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16.0 * (double)iters * blocks * threads;
    const double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best) { best = tf; best_ms = ms; }
  }
  const double nominal = (double)sms * 128 * 2 * (clk * 1e3) / 1e12;
  printf("{\"fp32_fma_tflops\": %.3f, \"launch_ms\": %.3f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
         "\"nominal_at_max_clock_tflops\": %.3f, \"how\": \"%d CTAs x %d threads, 16 independent fmaf chains x %d "
         "iterations, best of 5 (CUDA events)\"}\n",
         best, best_ms, sms, clk / 1e3, nominal, blocks, threads, iters);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

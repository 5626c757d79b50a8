// Measured fp64 / fp32 peaks of this B200 (the roofline denominators of the fp64 and fp32
// reference modes, which MEASURED_PEAKS.json does not carry):
//   dfma   SIMT DFMA, 8 independent chains per thread
//   dmma   mma.sync.aligned.m16n8k4.row.col.f64 (DMMA), 4 independent accumulators per warp
//   ffma   SIMT FFMA, 8 independent chains per thread
// Persistent grid of 148 x k CTAs, best of 5, CUDA events. Prints JSON.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fpp scripts/fp_peaks.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, double a0, double b0) {
  double acc[4][4];
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) acc[j][i] = 0.0;
  double a[2] = {a0 + threadIdx.x, a0 - threadIdx.x}, b = b0 + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
          "{%0,%1,%2,%3};"
          : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
          : "d"(a[0]), "d"(a[1]), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) s += acc[j][i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <typename F>
float best_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  f();
  cudaDeviceSynchronize();
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* dout;
  float* fout;
  cudaMalloc(&dout, 1 << 20);
  cudaMalloc(&fout, 1 << 20);
  const int threads = 256, ctas = sms * 8;
  const double n_thr = double(threads) * ctas;
  const float t_dfma = best_ms([&] { dfma_kernel<<<ctas, threads>>>(dout, 0.999, 1e-3); });
  const float t_ffma = best_ms([&] { ffma_kernel<<<ctas, threads>>>(fout, 0.999f, 1e-3f); });
  const float t_dmma = best_ms([&] { dmma_kernel<<<ctas, threads>>>(dout, 0.5, 0.25); });
  const double f_dfma = n_thr * ITERS * 8 * 2 / (t_dfma * 1e-3) / 1e12;
  const double f_ffma = n_thr * ITERS * 8 * 2 / (t_ffma * 1e-3) / 1e12;
  const double f_dmma = n_thr / 32 * ITERS * 4 * (16 * 8 * 4 * 2) / (t_dmma * 1e-3) / 1e12;
  printf("{\"fp64_dfma_tflops\": %.2f, \"fp64_dmma_tflops\": %.2f, \"fp32_ffma_tflops\": %.2f, "
         "\"sms\": %d, \"status\": \"%s\"}\n",
         f_dfma, f_dmma, f_ffma, sms, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

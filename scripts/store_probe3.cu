// Which property of the K2 output stream sets its rate: bytes per warp store instruction or
// the 4,900-B cell stride? 65,536 cells x 1225 fp32 written as
//   runB   per (cell, run) a warp writes RUN consecutive floats of one cell: float4 stores on
//          the 16-B aligned body, scalar head / tail (runs of 32 = the current epilogue's 128 B)
//   cellN  a warp writes whole cells (4,900 B) the same way
// Persistent grid of 148 x 256 threads, .cs stores. nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int N_CELLS = 65536, N_OUT = 1225;
constexpr long TOTAL = long(N_CELLS) * N_OUT;

// warp writes floats [s, s + n) of out (arbitrary alignment): scalar head to the next 16-B
// boundary, float4 body, scalar tail
__device__ __forceinline__ void warp_write(float* out, long s, int n, int lane, bool cs) {
  const int head = int((4 - (s & 3)) & 3) < n ? int((4 - (s & 3)) & 3) : n;
  if (lane < head) { if (cs) __stcs(out + s + lane, 1.0f); else out[s + lane] = 1.0f; }
  const long b = s + head;
  const int nb4 = (n - head) >> 2;
  float4* b4 = reinterpret_cast<float4*>(out + b);
  for (int i = lane; i < nb4; i += 32) { if (cs) __stcs(b4 + i, make_float4(1, 2, 3, 4)); else b4[i] = make_float4(1, 2, 3, 4); }
  const long t = b + 4L * nb4;
  const int nt = int(s + n - t);
  if (lane < nt) { if (cs) __stcs(out + t + lane, 1.0f); else out[t + lane] = 1.0f; }
}

template <int RUN, bool CS>
__global__ void __launch_bounds__(256) runs(float* out) {
  const int lane = threadIdx.x & 31;
  const long warps = long(gridDim.x) * 8, w0 = long(blockIdx.x) * 8 + (threadIdx.x >> 5);
  constexpr int per_cell = (N_OUT + RUN - 1) / RUN;
  // work item = (run index r, cell block of 32 cells): consecutive items walk cells first,
  // as the epilogue does (one output run, many cells)
  const long items = long(per_cell) * (N_CELLS / 32);
  for (long it = w0; it < items; it += warps) {
    const int r = int(it % per_cell);
    const long cb = (it / per_cell) * 32;
    const int o0 = r * RUN, n = N_OUT - o0 < RUN ? N_OUT - o0 : RUN;
    for (int c = 0; c < 32; ++c) warp_write(out, (cb + c) * N_OUT + o0, n, lane, CS);
  }
}

template <typename F>
float best_of(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  float* out;
  cudaMalloc(&out, size_t(TOTAL) * 4 + 256);
  const double bytes = double(TOTAL) * 4;
  auto rep = [&](const char* name, float ms) {
    printf("%-24s %8.1f us  %.2f TB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e12);
  };
  rep("run32 cs", best_of([&] { runs<32, true><<<148, 256>>>(out); }));
  rep("run32 wb", best_of([&] { runs<32, false><<<148, 256>>>(out); }));
  rep("run128 cs", best_of([&] { runs<128, true><<<148, 256>>>(out); }));
  rep("run256 cs", best_of([&] { runs<256, true><<<148, 256>>>(out); }));
  rep("run640 cs", best_of([&] { runs<640, true><<<148, 256>>>(out); }));
  rep("cell1225 cs", best_of([&] { runs<1225, true><<<148, 256>>>(out); }));
  rep("cell1225 cs g296", best_of([&] { runs<1225, true><<<296, 256>>>(out); }));
  rep("run128 cs g296", best_of([&] { runs<128, true><<<296, 256>>>(out); }));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}

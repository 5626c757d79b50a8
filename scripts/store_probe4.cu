// Is the cost of K2's epilogue stores per warp store INSTRUCTION or per 128-byte SEGMENT?
// 65,536 cells x 1225 fp32 (4,900-B rows). Every variant writes the same bytes with 8 or 16 warps
// per SM in K2's order (a warp owns 32 consecutive outputs and walks 32 cells):
//   seg1  one instruction = 32 lanes x 4 B  = one 128-B piece of one cell        (K2 today)
//   seg2  one instruction = 2 x (16 lanes x 8 B): 128-B pieces of two cells      (st.v2)
//   seg4  one instruction = 4 x (8 lanes x 16 B): 128-B pieces of four cells     (st.v4)
// (v2 / v4 addresses are rounded down to their alignment: the probe measures the store path only)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int N_CELLS = 65536, N_OUT = 1225;
constexpr long TOTAL = long(N_CELLS) * N_OUT;

template <int SEG>
__global__ void __launch_bounds__(256) pieces(float* out) {
  const int lane = threadIdx.x & 31;
  const long warps = long(gridDim.x) * (blockDim.x >> 5), w0 = long(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  constexpr int per_cell = (N_OUT + 31) / 32;  // 128-B pieces per cell
  const long items = long(per_cell) * (N_CELLS / 32);
  for (long it = w0; it < items; it += warps) {
    const int r = int(it % per_cell);
    const long cb = (it / per_cell) * 32;
    const int o0 = r * 32;
    if (o0 + 32 > N_OUT) continue;  // ragged last piece skipped in every variant
    if constexpr (SEG == 1) {
      #pragma unroll
      for (int c = 0; c < 32; ++c) __stcs(out + (cb + c) * N_OUT + o0 + lane, 1.0f);
    } else if constexpr (SEG == 2) {
      #pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const long a = ((cb + c + (lane >> 4)) * N_OUT + o0 + 2 * (lane & 15)) & ~1L;
        __stcs(reinterpret_cast<float2*>(out + a), make_float2(1.0f, 2.0f));
      }
    } else {
      #pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const long a = ((cb + c + (lane >> 3)) * N_OUT + o0 + 4 * (lane & 7)) & ~3L;
        __stcs(reinterpret_cast<float4*>(out + a), make_float4(1.0f, 2.0f, 3.0f, 4.0f));
      }
    }
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
  const double bytes = double(N_CELLS) * 38 * 128;  // pieces actually written
  auto rep = [&](const char* name, float ms) {
    printf("%-28s %8.1f us  %.2f TB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e12);
  };
  for (int wps : {8, 16}) {
    const int threads = 256, grid = 148 * wps / 8;
    printf("%d warps/SM\n", wps);
    rep("seg1 (32 x 4 B, 1 cell)", best_of([&] { pieces<1><<<grid, threads>>>(out); }));
    rep("seg2 (2 x 16 x 8 B)", best_of([&] { pieces<2><<<grid, threads>>>(out); }));
    rep("seg4 (4 x 8 x 16 B)", best_of([&] { pieces<4><<<grid, threads>>>(out); }));
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

// Store-pattern ceiling for the K2 output: 65,536 cells x n_out floats (row pitch P floats),
// written as the K2 epilogue does (persistent 148 CTAs, tile = 256 cells x 128 rows, warp
// (quarter, half) writes rows quarter*32+lane for 128 cells, one 128-B store per cell), vs
// contiguous float4 fill. nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/spp scripts/store_pattern_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) epi_pattern(float* out, int n_cells, int n_out, int pitch, int n_out_tiles) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int n_cell_tiles = (n_cells + 255) / 256;
  const int tiles = n_out_tiles * n_cell_tiles;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int ct = t / n_out_tiles, ot = t % n_out_tiles;
    const int o = ot * 128 + quarter * 32 + lane;
    if (o >= n_out) continue;
    for (int c = half * 128; c < half * 128 + 128; ++c) {
      const long cell = long(ct) * 256 + c;
      if (cell < n_cells) __stcs(out + cell * pitch + o, float(o));
    }
  }
}
__global__ void fill4(float4* out, long n4) {
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n4; i += long(gridDim.x) * blockDim.x)
    __stcs(out + i, make_float4(1, 2, 3, 4));
}
int main() {
  const int n_cells = 65536, n_out = 1225;
  float* out; cudaMalloc(&out, size_t(n_cells) * 1280 * 4 + 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int pitch : {1225, 1232, 1280}) {
    for (int grid : {148, 296}) {
      float best = 1e9;
      for (int r = 0; r < 10; ++r) {
        cudaEventRecord(a);
        epi_pattern<<<grid, 256>>>(out, n_cells, n_out, pitch, (n_out + 127) / 128);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("epilogue pattern pitch %d grid %d: %.1f us, %.2f TB/s\n", pitch, grid, best * 1e3, n_cells * double(n_out) * 4 / (best * 1e-3) / 1e12);
    }
  }
  const long n4 = long(n_cells) * n_out / 4;
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a); fill4<<<148 * 8, 256>>>(reinterpret_cast<float4*>(out), n4); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("contiguous float4 fill: %.1f us, %.2f TB/s\n", best * 1e3, n4 * 16.0 / (best * 1e-3) / 1e12);
  return 0;
}

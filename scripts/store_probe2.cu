// Store-stream ceilings for the cell-matrix output (65,536 cells x 1225 fp32, pitch 4900 B):
//   epi128   the K2 epilogue pattern: a warp writes 32 consecutive entries (128 B) of one cell
//   fill4    contiguous float4 stores over the whole buffer (the plain streaming ceiling)
//   span4    a warp writes contiguous 4-cell spans (19,600 B, 16-B aligned) with float4 stores
//   bulk     cp.async.bulk.global.shared::cta of 4-cell spans staged in shared memory
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/sp2 scripts/store_probe2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int N_CELLS = 65536, N_OUT = 1225;
constexpr long TOTAL = long(N_CELLS) * N_OUT;

__global__ void __launch_bounds__(256) epi128(float* out, int n_out_tiles) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int n_cell_tiles = N_CELLS / 256;
  const int tiles = n_out_tiles * n_cell_tiles;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int ct = t / n_out_tiles, ot = t % n_out_tiles;
    const int o = ot * 128 + quarter * 32 + lane;
    if (o >= N_OUT) continue;
    float* dst = out + (long(ct) * 256 + half * 128) * N_OUT + o;
#pragma unroll 8
    for (int c = 0; c < 128; ++c) __stcs(dst + long(c) * N_OUT, float(o));
  }
}

__global__ void fill4(float4* out, long n4) {
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n4; i += long(gridDim.x) * blockDim.x)
    __stcs(out + i, make_float4(1, 2, 3, 4));
}

// each warp owns 4-cell spans (4900 floats = 1225 float4), consecutive spans per warp
__global__ void span4(float4* out) {
  const int lane = threadIdx.x & 31;
  const long warps = long(gridDim.x) * (blockDim.x >> 5);
  const long w0 = long(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (long s = w0; s < N_CELLS / 4; s += warps) {
    float4* dst = out + s * 1225;
    for (int i = lane; i < 1225; i += 32) __stcs(dst + i, make_float4(1, 2, 3, 4));
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// one elected thread per CTA streams staged 4-cell spans with 1-D bulk copies (ring of SLOTS)
template <int SLOTS>
__global__ void __launch_bounds__(128) bulk(float* out) {
  extern __shared__ __align__(128) float buf[];  // SLOTS x 4900 floats
  for (int i = threadIdx.x; i < SLOTS * 4900; i += blockDim.x) buf[i] = float(i);
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x != 0) return;
  int slot = 0;
  for (long s = blockIdx.x; s < N_CELLS / 4; s += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + s * 4900),
                 "r"(smem_u32(buf + slot * 4900)), "r"(4900 * 4)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(SLOTS - 1) : "memory");
    slot = slot + 1 == SLOTS ? 0 : slot + 1;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
    printf("%-28s %8.1f us  %.2f TB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e12);
  };
  for (int g : {148, 296, 592}) {
    char nm[64];
    snprintf(nm, sizeof nm, "epi128 grid %d", g);
    rep(nm, best_of([&] { epi128<<<g, 256>>>(out, (N_OUT + 127) / 128); }));
  }
  rep("fill4 148x8x256", best_of([&] { fill4<<<148 * 8, 256>>>(reinterpret_cast<float4*>(out), TOTAL / 4); }));
  for (int g : {148, 296, 592}) {
    char nm[64];
    snprintf(nm, sizeof nm, "span4 grid %d x 256", g);
    rep(nm, best_of([&] { span4<<<g, 256>>>(reinterpret_cast<float4*>(out)); }));
  }
  cudaFuncSetAttribute(bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4900 * 4);
  cudaFuncSetAttribute(bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4900 * 4);
  for (int g : {148, 296, 592}) {
    char nm[64];
    snprintf(nm, sizeof nm, "bulk4 grid %d", g);
    rep(nm, best_of([&] { bulk<4><<<g, 128, 4 * 4900 * 4>>>(out); }));
    snprintf(nm, sizeof nm, "bulk8 grid %d", g);
    rep(nm, best_of([&] { bulk<8><<<g, 128, 8 * 4900 * 4>>>(out); }));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}

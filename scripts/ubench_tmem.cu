// tcgen05.ld throughput microbenchmark (development aid): W warps per CTA (1 CTA/SM) each
// loop tcgen05.ld.32x32b.xN + wait::ld over their lane quarter.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1810_01967_b200/csrc/cbb_common.cuh"
namespace cbb { void set_last_error(const char*) {} }
using namespace cbb;

template <int X>
__device__ __forceinline__ void ldx(uint32_t a, float* r);
template <> __device__ __forceinline__ void ldx<32>(uint32_t a, float* r) {
  tmem_ld32(a, *reinterpret_cast<float(*)[32]>(r));
}
template <> __device__ __forceinline__ void ldx<64>(uint32_t a, float* r) {
  tmem_ld32(a, *reinterpret_cast<float(*)[32]>(r));
  tmem_ld32(a + 32, *reinterpret_cast<float(*)[32]>(r + 32));
}

template <int X, int MODE>
__global__ void k(int iters, float* out, unsigned long long* cyc) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = holder;
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float r[X];
    ldx<X>(tb + (uint32_t((warp & 3) * 32) << 16) + ((i * X) & 511 & ~(X - 1)), r);
    tc_wait_ld();
    if (MODE == 0) { acc += r[0] + r[X - 1]; }
    else {
#pragma unroll
      for (int j = 0; j < X; j += 2) acc = fmax3(acc, r[j], r[j + 1]);
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0 && warp == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

template <int X, int MODE>
void run(int warps, float* out, unsigned long long* d) {
  const int iters = 20000;
  cudaMemset(d, 0, 8);
  k<X, MODE><<<148, warps * 32>>>(iters, out, d);
  cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  double clk = double(h) / 148 / iters;  // per iteration of warp 0
  double bytes = double(warps) * 32 * X * 4;  // per iteration, all warps
  printf("x%d warps=%2d %s: %.1f clk/iter  %.0f B/clk/SM  %.1f scores/clk/SM  err=%s\n", X, warps,
         MODE ? "ld+max3" : "ld only", clk, bytes / clk, bytes / 4 / clk,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out; cudaMalloc(&out, 148 * 1024 * 4);
  unsigned long long* d; cudaMalloc(&d, 8);
  for (int w : {4, 8, 12, 16}) { run<32, 0>(w, out, d); run<64, 0>(w, out, d); }
  for (int w : {4, 8, 12, 16}) { run<32, 1>(w, out, d); run<64, 1>(w, out, d); }
  return 0;
}

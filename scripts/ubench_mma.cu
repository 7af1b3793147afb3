// tcgen05.mma issue/throughput microbenchmark (development aid).
// Each CTA (1 per SM) issues ITERS MMAs M=128 x N x K=16 (bf16 -> f32) back to back into one
// TMEM accumulator, A from TMEM (ts) or SMEM (ss), B from SMEM; one commit + wait at the end.
// Issuer: lane 0 only (mode 0) or whole warp with elect.sync (mode 1).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1810_01967_b200/csrc/cbb_common.cuh"
namespace cbb { void set_last_error(const char*) {} }
using namespace cbb;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

template <int N, bool TS, int MODE>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 64 * 1024);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 64 * 1024 + 64);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_fence_init(); }
  if (warp == 0) tmem_alloc(holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = *holder;
  constexpr uint32_t idesc = idesc_bf16_f32(128, N);
  const uint64_t bdesc = umma_desc_kmajor(smem_u32(smem), 32);
  const uint64_t adesc = umma_desc_kmajor(smem_u32(smem + 32 * 1024), 32);
  long long t0 = clock64();
  if (warp == 1) {
    if (MODE == 0) {
      if ((threadIdx.x & 31) == 0) {
        for (int i = 0; i < iters; ++i) {
          if (TS) tc_mma_bf16_ts(tb, tb + 256 + (i & 1) * 8, bdesc + 2 * (i & 1), idesc, i > 0);
          else tc_mma_bf16(tb, adesc + 2 * (i & 1), bdesc + 2 * (i & 1), idesc, i > 0);
        }
        tc_commit(bar);
      }
    } else {
      for (int i = 0; i < iters; ++i) {
        if (elect_one()) {
          if (TS) tc_mma_bf16_ts(tb, tb + 256 + (i & 1) * 8, bdesc + 2 * (i & 1), idesc, i > 0);
          else tc_mma_bf16(tb, adesc + 2 * (i & 1), bdesc + 2 * (i & 1), idesc, i > 0);
        }
        __syncwarp();
      }
      if (elect_one()) tc_commit(bar);
      __syncwarp();
    }
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  }
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

template <int N, bool TS, int MODE>
void run(unsigned long long* d) {
  const int iters = 20000;
  cudaFuncSetAttribute(k<N, TS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  cudaMemset(d, 0, 8);
  k<N, TS, MODE><<<148, 128, 70 * 1024>>>(iters, d);
  cudaMemset(d, 0, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<N, TS, MODE><<<148, 128, 70 * 1024>>>(iters, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  double clk_per = double(h) / 148 / iters;
  double macs = 128.0 * N * 16 * iters * 148;
  printf("N=%3d %s issue=%s: %.1f clk/MMA (floor %d), %.0f MAC/clk/SM, %.1f TFLOP/s bf16  err=%s\n", N,
         TS ? "A=TMEM" : "A=SMEM", MODE ? "warp+elect" : "lane0", clk_per, N / 2,
         128.0 * N * 16 / clk_per, 2 * macs / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  run<32, true, 0>(d); run<64, true, 0>(d); run<128, true, 0>(d); run<256, true, 0>(d);
  run<32, true, 1>(d); run<64, true, 1>(d); run<128, true, 1>(d); run<256, true, 1>(d);
  run<64, false, 0>(d); run<128, false, 0>(d); run<256, false, 0>(d);
  run<64, false, 1>(d); run<128, false, 1>(d); run<256, false, 1>(d);
  return 0;
}

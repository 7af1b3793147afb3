// tcgen05.mma -> commit -> mbarrier wake latency (development aid).
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
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile("{\n\t.reg .pred P1;\nSPIN_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra SPIN_%=;\n\t}" :: "r"(addr), "r"(parity) : "memory");
}
template <int N, int NMMA, int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32 * 1024);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 32 * 1024 + 64);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_fence_init(); *reinterpret_cast<unsigned int*>(smem + 32 * 1024 + 128) = 0u; }
  if (warp == 0) tmem_alloc(holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = *holder;
  const uint64_t bdesc = umma_desc_kmajor(smem_u32(smem), 32);
  unsigned long long tot = 0;
  if (warp == 1) {
    for (int i = 0; i < iters; ++i) {
      long long t0 = clock64();
      if (elect_one()) {
        for (int j = 0; j < NMMA; ++j)
          tc_mma_bf16_ts(tb + (j & 3) * 64, tb + 448 + (j & 1) * 8, bdesc + 2 * (j & 1), idesc_bf16_f32(128, N), j & 1);
        tc_commit(bar);
      }
      __syncwarp();
      if (MODE == 1) mbar_spin(bar, i & 1); else mbar_wait(bar, i & 1);
      tc_fence_after();
      long long t1 = clock64();
      tot += (unsigned long long)(t1 - t0);
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(out, tot / iters);
    if ((threadIdx.x & 31) == 0) atomicExch(reinterpret_cast<unsigned int*>(smem + 32 * 1024 + 128), 1u);
  } else if (warp >= 4 && MODE >= 2) {
    // background TMEM readers (columns 256..383), like the epilogue
    volatile unsigned int* stop = reinterpret_cast<volatile unsigned int*>(smem + 32 * 1024 + 128);
    float acc = 0.f;
    while (*stop == 0u) {
      float r[32];
      tmem_ld32(tb + (uint32_t((warp & 3) * 32) << 16) + 256 + ((warp >> 2) & 3) * 32, r);
      tc_wait_ld();
      acc += r[0] + r[31];
    }
    if (acc == 12345.f) out[1] = 1;
  }
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}
template <int N, int NMMA, int MODE>
void run(unsigned long long* d) {
  cudaFuncSetAttribute(k<N, NMMA, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  cudaMemset(d, 0, 16);
  k<N, NMMA, MODE><<<148, MODE >= 2 ? 128 + 32 * (MODE == 2 ? 4 : 12) : 128, 40 * 1024>>>(1000, d);
  cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d mmas=%d %s: issue->wake latency %.0f clk (MMA work %d clk) %s\n", N, NMMA,
         MODE == 0 ? "try_wait      " : MODE == 1 ? "test_wait spin" : MODE == 2 ? "+4 LDTM warps " : "+12 LDTM warps", double(h) / 148, NMMA * N / 2,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  run<64, 1, 0>(d); run<64, 2, 0>(d); run<64, 8, 0>(d); run<128, 2, 0>(d); run<256, 2, 0>(d);
  run<64, 2, 2>(d); run<64, 8, 2>(d); run<64, 2, 3>(d); run<64, 8, 3>(d); run<128, 2, 3>(d);
  return 0;
}

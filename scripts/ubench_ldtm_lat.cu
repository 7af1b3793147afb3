// Microbenchmark: latency of tcgen05.ld (32x32b.x32, 64 KB region disjoint from the MMA
// accumulator) while a queue of tcgen05.mma (M=128, N=256, K=16, A/B from SMEM) is in flight
// on the same SM.  Answers: does a TMEM load wait behind MMAs issued before it?
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o ubench_ldtm_lat ubench_ldtm_lat.cu
#include <cstdio>
#include <vector>

#include "../paper_1810_01967_b200/csrc/cbb_common.cuh"

using namespace cbb;

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}

// warps 0..3: LDTM probes (lane quarter = warp), warp 4: MMA issuer
__global__ void __launch_bounds__(160, 1) k(int n_mma, int reps, int variant, long long* out, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // A: 128 x 16 bf16 (4 KB), B: 256 x 16 bf16 (8 KB), zeros, SWIZZLE_64B K-major (kpad 32)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
  volatile int* go = reinterpret_cast<volatile int*>(smem + 32768 + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1000000);
    mbar_fence_init();
    *go = 0;
  }
  if (warp == 0) tmem_alloc(holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *holder;
  if (warp == 4) {
    if (lane == 0) {
      const uint64_t ad = umma_desc_kmajor(smem_u32(smem), 32);
      const uint64_t bd = umma_desc_kmajor(smem_u32(smem + 8192), 32);
      const uint32_t idesc = idesc_f16_f16(128, 256);
      long long t0 = clk();
      for (int i = 0; i < n_mma; ++i) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
            "l"(ad), "l"(bd), "r"(idesc), "r"(i > 0 ? 1 : 0)
            : "memory");
      }
      *go = 1;  // probes start after the queue was issued
      tc_commit(bar);
      mbar_wait(bar, 0);
      long long t1 = clk();
      out[0] = t1 - t0;
    }
    __syncwarp();
  } else {
    while (*go == 0 && n_mma > 0) {
    }
    const uint32_t taddr = tbase + (uint32_t(warp * 32) << 16) + 256;
    int acc = 0;
    for (int r = 0; r < reps; ++r) {
      float v[32];
      long long t0 = clk();
      tmem_ld32(taddr, v);
      tc_wait_ld();
      if (variant >= 1) tc_fence_before();
      if (variant >= 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive(bar + 1);
      }
      int x = 0;
#pragma unroll
      for (int i = 0; i < 32; ++i) x ^= __float_as_int(v[i]);
      reinterpret_cast<volatile int*>(smem + 32768 + 256)[threadIdx.x] = x;
      long long t1 = clk();
      acc += x;
      if (lane == 0) out[1 + warp * reps + r] = t1 - t0;
    }
    sink[threadIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

int main() {
  const int reps = 12;
  long long* d_out;
  int* sink;
  cudaMalloc(&d_out, sizeof(long long) * (1 + 4 * reps));
  cudaMalloc(&sink, 4096);
  const int smem = 32768 + 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<long long> h(1 + 4 * reps);
  for (int variant = 0; variant < 3; ++variant)
  for (int n_mma : {0, 16}) {
    printf("variant %d (0: ld+wait, 1: +fence::before_thread_sync, 2: +syncwarp+mbarrier.arrive)\n", variant);
    for (int trial = 0; trial < 2; ++trial) {
      k<<<1, 160, smem>>>(n_mma, reps, variant, d_out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
    }
    cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost);
    printf("n_mma=%3d (%5d clk of MMA work at 4096 MAC/clk)  mma queue drained after %lld clk\n",
           n_mma, n_mma * 128, n_mma ? h[0] : 0LL);
    for (int w = 0; w < 4; ++w) {
      printf("   warp %d LDTM latencies:", w);
      for (int r = 0; r < reps; ++r) printf(" %lld", h[1 + w * reps + r]);
      printf("\n");
    }
  }
  return 0;
}

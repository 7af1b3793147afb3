// tcgen05.ld bandwidth microbenchmark (development aid): is the fp16 screen's epilogue bound by
// TMEM reads?  W warps per CTA (1 CTA/SM), each loops over 128 columns of its lane quarter with
//   MODE 0: 32x32b.x32        (32 columns, 32 regs)
//   MODE 1: 32x32b.x32.pack16 (64 columns, 32 regs)
//   MODE 2: 32x32b.x64        (64 columns, 64 regs)
//   MODE 3: 16x256b.x8        (lanes 0-15 of the quarter: 16 lanes x 256 bit x 8 = 32 regs)
// and reports columns*lanes read per clock per SM (cells/clk) and bytes/clk of 32-bit cells.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

#define R32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
#define O32(r) "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), \
  "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), \
  "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])

template <int MODE>
__device__ __forceinline__ void ld(uint32_t a, uint32_t* r) {
  if constexpr (MODE == 0) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(a));
  } else if constexpr (MODE == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 " R32 ", [%32];" : O32(r) : "r"(a));
  } else if constexpr (MODE == 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(a));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 ", [%32];" : O32((r + 32)) : "r"(a + 32));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " R32 ", [%32];" : O32(r) : "r"(a));
  }
}

template <int MODE>
__global__ void k(int iters, uint32_t* out, unsigned long long* cyc) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = holder + (uint32_t((warp & 3) * 32) << 16);
  constexpr int kRegs = MODE == 2 ? 64 : 32;
  constexpr int kCols = MODE == 0 ? 32 : 64;  // 32-bit columns per call (mode 3: 8 x 256 bit / 4 = 64? see cells)
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[kRegs];
    ld<MODE>(tb + ((i * kCols) & 255), r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < kRegs; ++j) acc ^= r[j];
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0 && warp == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
  }
}

template <int MODE>
void run(int warps, uint32_t* out, unsigned long long* d) {
  const int iters = 20000;
  cudaMemset(d, 0, 8);
  k<MODE><<<148, warps * 32>>>(iters, out, d);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  double clk = double(h) / 148 / iters;  // per iteration of warp 0
  // 32-bit TMEM cells touched per call per warp: x32: 32 lanes x 32 cols; pack16 x32: 32 x 64;
  // x64: 32 x 64; 16x256b.x8: 16 lanes x 8 x 8 cols = 16 x 64
  const double cells = MODE == 0 ? 32 * 32 : MODE == 3 ? 16 * 64 : 32 * 64;
  const double regs = 32.0 * (MODE == 2 ? 64 : 32);
  const char* names[] = {"32x32b.x32", "32x32b.x32.pack16", "32x32b.x64", "16x256b.x8"};
  printf("%-20s warps=%2d: %7.1f clk/iter  cells %6.1f /clk/SM (%5.0f B/clk)  regs %6.1f /clk/SM  err=%s\n",
         names[MODE], warps, clk, warps * cells / clk, 4 * warps * cells / clk, warps * regs / clk,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 1024 * 4);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  for (int w : {4, 8, 12, 16}) {
    run<0>(w, out, d);
    run<1>(w, out, d);
    run<2>(w, out, d);
    run<3>(w, out, d);
  }
  return 0;
}

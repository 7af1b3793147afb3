// Throughput of FMNMX3 vs FMNMX vs FSETP on sm_100a (development micro-benchmark).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r;
}
#include <cuda_fp16.h>
template <int MODE>
__global__ void k2(float* out, int iters, float seed) {
  // MODE 0: cvt.rn.f16x2.f32 (pack) ; 1: max.f16x2 ; 2: pack + max mix
  __half2 h[8];
  float a[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i); h[i] = __floats2half2_rn(a[i], a[i] + 1); }
  __half2 hb = __floats2half2_rn(seed, seed * 2), hc = __floats2half2_rn(seed * 3, seed);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { a[i] = fmaxf(a[i], __uint_as_float(__float_as_uint(a[i]) ^ 1u)); h[i] = __floats2half2_rn(a[i], a[i]); }
      else if (MODE == 1) { h[i] = __hmax2(h[i], hb); }
      else if (MODE == 3) { h[i] = __hmax2(__hmax2(h[i], hb), hc); }
      else if (MODE == 4) { if (i & 1) h[i] = __hmax2(__hmax2(h[i], hb), hc); else h[i] = __hmax2(h[i], hb); }
      else if (MODE == 5) { if (i & 1) h[i] = __hmax2(__hmax2(h[i], hb), hc); else a[i] = fmaxf(a[i], seed); }
      else { if (i & 1) h[i] = __hmax2(h[i], hb); else a[i] = fmaxf(a[i], seed); }
    }
    hb = __hadd2(hb, hb);
    hc = __hadd2(hc, hb);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += __half2float(h[i].x) + __half2float(h[i].y);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
__global__ void k(float* out, int iters, float seed) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i);
  float b = seed * 3, c = seed * 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = max3(a[i], b, c);
      else if (MODE == 1) a[i] = fmaxf(a[i], b);
      else if (MODE == 2) a[i] = __fmaf_rn(a[i], b, c);
      else if (MODE == 4) { double t = fma(double(a[i]), double(b), double(c)); a[i] = float(t); }
      else if (MODE == 5) { unsigned u = __float_as_uint(a[i]); u = max(max(u, __float_as_uint(b)), __float_as_uint(c)); a[i] = __uint_as_float(u); }
      else if (MODE == 6) { unsigned u = __float_as_uint(a[i]); u = max(u, __float_as_uint(b)); a[i] = __uint_as_float(u); }
      else if (MODE == 7) { if (i & 1) { unsigned u = __float_as_uint(a[i]); u = max(max(u, __float_as_uint(b)), __float_as_uint(c)); a[i] = __uint_as_float(u); } else a[i] = max3(a[i], b, c); }
      else a[i] = (i & 1) ? fmaxf(a[i], b) : max3(a[i], b, c);
    }
    b += 1e-7f; c -= 1e-7f;
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  const int iters = 1 << 14;
  const char* names[8] = {"FMNMX3", "FMNMX", "FFMA", "FMNMX3+FMNMX interleaved", "DFMA(+cvt)",
                          "VIMNMX3.U32", "VIMNMX.U32", "VIMNMX3+FMNMX3 interleaved"};
  for (int mode = 0; mode < 8; ++mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 1) k<1><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 2) k<2><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 3) k<3><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 4) k<4><<<148 * 8, 1024>>>(out, iters / 16, 1.0f);
      if (mode == 5) k<5><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 6) k<6><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 7) k<7><<<148 * 8, 1024>>>(out, iters, 1.0f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(148 * 8) * 1024 * (mode == 4 ? iters / 16 : iters) * 8;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%s: %.3f ms  %.1f lane-ops/clk/SM (at %.0f MHz)\n", names[mode], ms,
           ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1e3);
  }
  const char* n2[6] = {"F2FP pack + FMNMX", "HMNMX2", "HMNMX2+FMNMX interleaved",
                       "VHMNMX (3-input half2)", "VHMNMX+HMNMX2 interleaved", "VHMNMX+FMNMX interleaved"};
  for (int mode = 0; mode < 6; ++mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k2<0><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 1) k2<1><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 2) k2<2><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 3) k2<3><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 4) k2<4><<<148 * 8, 1024>>>(out, iters, 1.0f);
      if (mode == 5) k2<5><<<148 * 8, 1024>>>(out, iters, 1.0f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(148 * 8) * 1024 * iters * 8;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%s: %.3f ms  %.1f lane-ops/clk/SM\n", n2[mode], ms, ops / (ms * 1e-3) / 148 / (clk * 1e3));
  }
  return 0;
}

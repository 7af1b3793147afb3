// Probe: tcgen05.mma kind::f16 with FP16 operands and an FP32 accumulator (A in TMEM, B in
// SMEM, M=128 N=128 K=64 as four K=16 instructions) -- the split-operand ("hi/lo") screening
// mode.  Prints known-answer rounding / alignment cases and, for random split rows
// A = [z_hi | z_lo | z_hi], B = [d_hi | d_hi | d_lo], the error of the accumulator against
// (a) the exact sum of the fp16 products and (b) the exact fp64 product z.d, relative to
// sum|a_k b_k| and to |z||d| -- the model behind the split-mode certified window.
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_f32acc probe_f32acc.cu
#include <cuda_fp16.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../paper_1810_01967_b200/csrc/cbb_common.cuh"

using namespace cbb;

constexpr int KP = 64;

__device__ __forceinline__ void tmem_ld32f(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__global__ void __launch_bounds__(128, 1)
    probe_kernel(const uint8_t* zrows, const uint8_t* atile, uint32_t* raw) {
  constexpr int kTileBytes = 128 * KP * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kTileBytes);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + kTileBytes + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *holder;
  const uint32_t lane_off = uint32_t(warp * 32) << 16;
  for (int h = 0; h < 2; ++h) {
    uint32_t wz[16];
    const uint32_t* src =
        reinterpret_cast<const uint32_t*>(zrows + size_t(threadIdx.x) * KP * 2) + 16 * h;
    for (int i = 0; i < 16; ++i) wz[i] = src[i];
    tmem_st16(tbase + lane_off + 128 + 16 * h, wz);
  }
  tc_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, kTileBytes);
    bulk_g2s(smem, atile, kTileBytes, bar, policy_evict_first());
    mbar_wait(bar, 0);
    tc_fence_after();
    const uint64_t bd = umma_desc_kmajor(smem_u32(smem), KP);
    const uint32_t idesc = (1u << 4) | (uint32_t(128 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    for (int k = 0; k < KP / 16; ++k)
      tc_mma_f16_ts(tbase, tbase + 128 + k * 8, bd + uint64_t(2 * k), idesc, k > 0);
    tc_commit(bar + 1);
  }
  __syncwarp();
  mbar_wait(bar + 1, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld32f(tbase + lane_off + c * 32, r);
    tc_wait_ld();
    for (int i = 0; i < 32; ++i) raw[row * 128 + c * 32 + i] = r[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

static float u2f(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static double h2d(uint16_t h) {
  __half x;
  memcpy(&x, &h, 2);
  return double(__half2float(x));
}
static uint16_t d2h(double f) {
  __half x = __double2half(f);
  uint16_t h;
  memcpy(&h, &x, 2);
  return h;
}

int main() {
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  const int kTileBytes = 128 * KP * 2;
  const int s = 10, e = 2 * s;
  uint8_t *dz, *da;
  uint32_t* draw;
  cudaMalloc(&dz, kTileBytes);
  cudaMalloc(&da, kTileBytes);
  cudaMalloc(&draw, 128 * 128 * 4);
  const int smem = kTileBytes + 64 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<uint16_t> A(128 * KP), B(128 * KP);
  std::vector<uint8_t> tile(kTileBytes);
  std::vector<uint32_t> raw(128 * 128);
  std::vector<double> zx(128 * e), dx(128 * e);

  double w_abs = 0, w_norm = 0, w_exact_norm = 0;
  long long n_total = 0, n_single_rn = 0;
  for (int trial = 0; trial < 60; ++trial) {
    // voxels: norm ~ 2^12 (scaled like the prologue), some with a wide dynamic range
    for (int r = 0; r < 128; ++r) {
      const double sc = std::ldexp(1.0, 12) / std::sqrt(double(e));
      for (int k = 0; k < e; ++k) {
        double v = nd(rng) * sc;
        if (r % 4 == 1) v *= std::ldexp(1.0, -int(rng() % 20));  // small components
        zx[r * e + k] = v;
      }
      for (int k = 0; k < KP; ++k) A[r * KP + k] = 0;
      for (int k = 0; k < e; ++k) {
        const uint16_t hi = d2h(zx[r * e + k]);
        const uint16_t lo = d2h(zx[r * e + k] - h2d(hi));
        A[r * KP + k] = hi;
        A[r * KP + e + k] = lo;
        A[r * KP + 2 * e + k] = hi;
      }
    }
    auto setrow = [&](int r, std::vector<std::pair<int, double>> v) {
      for (int k = 0; k < KP; ++k) A[r * KP + k] = 0;
      for (int k = 0; k < e; ++k) zx[r * e + k] = 0;
      for (auto& p : v) A[r * KP + p.first] = d2h(p.second);
    };
    if (trial == 0) {
      // atom 0 is all ones: column 0 = plain sum of the row
      setrow(0, {{0, 2048.}, {1, 1.220703125e-4}, {2, 1.220703125e-4}});   // 2^11 + 2*2^-13
      setrow(1, {{0, 2048.}, {16, 1.220703125e-4}, {32, 1.220703125e-4}}); // across instrs
      setrow(2, {{0, 2048.}, {1, 1.220703125e-4}});                         // tie -> 2048
      setrow(3, {{0, 2048.}, {1, 1.8310546875e-4}});                        // 1.5 half-ulp
      setrow(4, {{0, 60000.}, {1, 60000.}, {2, -60000.}, {3, -60000.}, {4, 0.0625}});
      setrow(5, {{0, 4096.}, {1, 6.103515625e-5}, {2, -4096.}});            // cancel, keep tiny
      setrow(6, {{0, 1.}, {1, 5.9604644775390625e-8}});                     // 1 + 2^-24 (sub)
      setrow(7, {{0, 32768.}, {1, 1.}, {2, -32768.}, {3, 5.9604644775390625e-8}});
      setrow(8, {{0, 1.}, {1, 3.0517578125e-5}, {2, 3.0517578125e-5}, {3, 3.0517578125e-5}});
    }
    for (int j = 0; j < 128; ++j) {
      double nrm = 0;
      for (int k = 0; k < e; ++k) {
        dx[j * e + k] = nd(rng);
        nrm += dx[j * e + k] * dx[j * e + k];
      }
      for (int k = 0; k < e; ++k) dx[j * e + k] *= std::ldexp(1.0, 10) / std::sqrt(nrm);
      for (int k = 0; k < KP; ++k) B[j * KP + k] = 0;
      for (int k = 0; k < e; ++k) {
        const uint16_t hi = d2h(dx[j * e + k]);
        const uint16_t lo = d2h(dx[j * e + k] - h2d(hi));
        B[j * KP + k] = hi;
        B[j * KP + e + k] = hi;
        B[j * KP + 2 * e + k] = lo;
      }
      if (j == 0)
        for (int k = 0; k < KP; ++k) B[k] = d2h(1.0);
    }
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < KP / 8; ++c)
        memcpy(tile.data() + tile_chunk_offset(r, c, KP), &B[r * KP + c * 8], 16);
    cudaMemcpy(dz, A.data(), kTileBytes, cudaMemcpyHostToDevice);
    cudaMemcpy(da, tile.data(), kTileBytes, cudaMemcpyHostToDevice);
    probe_kernel<<<1, 128, smem>>>(dz, da, draw);
    cudaMemcpy(raw.data(), draw, raw.size() * 4, cudaMemcpyDeviceToHost);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(err));
      return 1;
    }
    if (trial == 0) {
      for (int r = 0; r < 9; ++r) {
        double ex = 0;
        for (int k = 0; k < KP; ++k) ex += h2d(A[r * KP + k]);
        printf("KAT row %d: exact %.12g  f32acc %.12g  RN(exact) %.12g\n", r, ex,
               double(u2f(raw[r * 128])), double(float(ex)));
      }
    }
    for (int r = (trial == 0 ? 9 : 0); r < 128; ++r)
      for (int j = 1; j < 128; ++j) {
        double ex = 0, sabs = 0, na = 0, nb = 0, zd = 0;
        for (int k = 0; k < KP; ++k) {
          const double a = h2d(A[r * KP + k]), b = h2d(B[j * KP + k]);
          ex += a * b;
          sabs += std::fabs(a * b);
        }
        for (int k = 0; k < e; ++k) {
          zd += zx[r * e + k] * dx[j * e + k];
          na += zx[r * e + k] * zx[r * e + k];
          nb += dx[j * e + k] * dx[j * e + k];
        }
        const double got = u2f(raw[r * 128 + j]);
        w_abs = std::max(w_abs, std::fabs(got - ex) / sabs);
        w_norm = std::max(w_norm, std::fabs(got - ex) / std::sqrt(na * nb));
        w_exact_norm = std::max(w_exact_norm, std::fabs(got - zd) / std::sqrt(na * nb));
        if (double(float(ex)) == got) ++n_single_rn;
        ++n_total;
      }
  }
  printf("random split rows: n=%lld  single-RN-of-exact-fp16-sum %.4f\n", n_total,
         double(n_single_rn) / n_total);
  printf("  worst |acc - sum fp16 products| / sum|ab| = %.3e (2^%.2f)\n", w_abs, std::log2(w_abs));
  printf("  worst |acc - sum fp16 products| / |z||d|  = %.3e (2^%.2f)\n", w_norm, std::log2(w_norm));
  printf("  worst |acc - z.d (fp64)| / |z||d|         = %.3e (2^%.2f)\n", w_exact_norm,
         std::log2(w_exact_norm));
  return 0;
}

// Probe: tcgen05.mma kind::f16 with FP16 operands and an FP16 accumulator (A in TMEM, B in
// SMEM, M=128 N=128 K=32 as two K=16 instructions), read back with and without .pack::16b.
// Prints the TMEM layout check, known-answer rounding cases and the error of random tiles
// relative to sum|a_k b_k| -- the accumulation model the certified screening window relies on.
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_f16acc probe_f16acc.cu
#include <cuda_fp16.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../paper_1810_01967_b200/csrc/cbb_common.cuh"

using namespace cbb;

constexpr int KP = 32;

__device__ __forceinline__ void tmem_ld16_pack(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// mode 0: f16 accumulate, mode 1: f32 accumulate (both with f16 operands)
__global__ void __launch_bounds__(128, 1)
    probe_kernel(const uint8_t* zrows, const uint8_t* atile, int mode, uint32_t* raw,
                 uint32_t* packed) {
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
  {
    uint32_t wz[16];
    const uint32_t* src = reinterpret_cast<const uint32_t*>(zrows + size_t(threadIdx.x) * KP * 2);
    for (int i = 0; i < 16; ++i) wz[i] = src[i];
    tmem_st16(tbase + lane_off + 128, wz);
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, kTileBytes);
    bulk_g2s(smem, atile, kTileBytes, bar, policy_evict_first());
    mbar_wait(bar, 0);
    tc_fence_after();
    const uint64_t bd = umma_desc_kmajor(smem_u32(smem), KP);
    const uint32_t idesc = (mode == 0 ? 0u : (1u << 4)) | (uint32_t(128 >> 3) << 17) |
                           (uint32_t(128 >> 4) << 24);
    for (int k = 0; k < KP / 16; ++k)
      tc_mma_bf16_ts(tbase, tbase + 128 + k * 8, bd + uint64_t(2 * k), idesc, k > 0);
    tc_commit(bar + 1);
  }
  __syncwarp();
  mbar_wait(bar + 1, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c = 0; c < 4; ++c) {
    float r[32];
    tmem_ld32(tbase + lane_off + c * 32, r);
    tc_wait_ld();
    for (int i = 0; i < 32; ++i) raw[row * 128 + c * 32 + i] = __float_as_uint(r[i]);
  }
  for (int c = 0; c < 4; ++c) {
    uint32_t r[16];
    tmem_ld16_pack(tbase + lane_off + c * 32, r);
    tc_wait_ld();
    for (int i = 0; i < 16; ++i) packed[row * 64 + c * 16 + i] = r[i];
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
static float h2f(uint16_t h) {
  __half x;
  memcpy(&x, &h, 2);
  return __half2float(x);
}
static uint16_t f2h(float f) {
  __half x = __float2half_rn(f);
  uint16_t h;
  memcpy(&h, &x, 2);
  return h;
}

int main() {
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd(0.0, 1.0);
  const int kTileBytes = 128 * KP * 2;
  uint8_t *dz, *da;
  uint32_t *draw, *dpk;
  cudaMalloc(&dz, kTileBytes);
  cudaMalloc(&da, kTileBytes);
  cudaMalloc(&draw, 128 * 128 * 4);
  cudaMalloc(&dpk, 128 * 64 * 4);
  const int smem = kTileBytes + 64 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);

  std::vector<uint16_t> A(128 * KP), B(128 * KP);
  std::vector<uint8_t> tile(kTileBytes);
  std::vector<uint32_t> raw(128 * 128), pk(128 * 64), raw32(128 * 128), pk32(128 * 64);

  double worst_rel_abs = 0, worst_rel_norm = 0, worst_ulps = 0;
  long long n_single_rn = 0, n_total = 0, n_layout_bad = 0, n_f32_bad = 0;
  for (int trial = 0; trial < 40; ++trial) {
    // A rows: KAT rows 0..15, random rows with norm ~ 2^12 otherwise
    for (int r = 0; r < 128; ++r) {
      double sc = std::ldexp(1.0, 12) / std::sqrt(double(2 * 10));
      for (int k = 0; k < KP; ++k) A[r * KP + k] = (k < 20) ? f2h(float(nd(rng) * sc)) : 0;
    }
    auto setrow = [&](int r, std::vector<std::pair<int, float>> v) {
      for (int k = 0; k < KP; ++k) A[r * KP + k] = 0;
      for (auto& p : v) A[r * KP + p.first] = f2h(p.second);
    };
    if (trial == 0) {
      setrow(0, {{0, 2048.f}, {1, 1.f}, {2, -2048.f}});       // in-instruction rounding
      setrow(1, {{0, 2048.f}, {1, 1.f}, {16, -2048.f}});      // across instructions
      setrow(2, {{0, 2048.f}, {1, 3.f}});                     // 2051: RN 2052 / RZ 2050
      setrow(3, {{0, -2048.f}, {1, -3.f}});                   // -2051
      setrow(4, {{0, 2048.f}, {1, 1.f}});                     // 2049 tie -> 2048 (even)
      setrow(5, {{0, 2048.f}, {1, 1.f}, {2, 0.5f}});          // 2049.5 -> RN 2050
      setrow(6, {{0, 1.f}, {1, 0.000488281f}, {2, 0.0000610352f}});  // 1 + 2^-11 + 2^-14
      setrow(7, {{0, 1.f}, {16, 0.000488281f}, {17, 0.0000610352f}});
      setrow(8, {{0, 4096.f}, {1, 1.f}, {2, 1.f}, {3, 1.f}, {4, -4096.f}});  // exact 3
      setrow(9, {{0, 60000.f}, {1, 60000.f}, {2, -60000.f}});  // intermediate overflow?
      setrow(10, {{0, 1024.f}, {1, 0.25f}, {2, 0.25f}, {3, 0.25f}, {4, 0.25f}});  // 1025
      setrow(11, {{0, 3.f}, {1, 0.0009765625f}});             // 3 + 2^-10 -> ulp(3)=2^-9
    }
    // B atoms: atom 0 = ones on every K (KAT sums), others random unit-ish
    for (int j = 0; j < 128; ++j) {
      double nrm = 0;
      std::vector<double> v(KP, 0.0);
      for (int k = 0; k < 20; ++k) {
        v[k] = nd(rng);
        nrm += v[k] * v[k];
      }
      for (int k = 0; k < KP; ++k) B[j * KP + k] = (k < 20) ? f2h(float(v[k] / std::sqrt(nrm))) : 0;
      if (j == 0)
        for (int k = 0; k < KP; ++k) B[k] = f2h(1.f);
    }
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < KP / 8; ++c)
        memcpy(tile.data() + tile_chunk_offset(r, c, KP), &B[r * KP + c * 8], 16);
    cudaMemcpy(dz, A.data(), kTileBytes, cudaMemcpyHostToDevice);
    cudaMemcpy(da, tile.data(), kTileBytes, cudaMemcpyHostToDevice);
    probe_kernel<<<1, 128, smem>>>(dz, da, 0, draw, dpk);
    cudaMemcpy(raw.data(), draw, raw.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(pk.data(), dpk, pk.size() * 4, cudaMemcpyDeviceToHost);
    probe_kernel<<<1, 128, smem>>>(dz, da, 1, draw, dpk);
    cudaMemcpy(raw32.data(), draw, raw.size() * 4, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      return 1;
    }
    if (trial == 0) {
      printf("raw column words row0: %08x %08x %08x %08x\n", raw[0], raw[1], raw[2], raw[3]);
      printf("packed words row0: %08x %08x\n", pk[0], pk[1]);
      for (int r = 0; r < 12; ++r) {
        double ex = 0;
        for (int k = 0; k < KP; ++k) ex += double(h2f(A[r * KP + k]));
        const uint16_t lo = uint16_t(pk[r * 64] & 0xffff);
        printf("KAT row %2d: exact %.9g  f16acc %.9g  f32acc %.9g\n", r, ex, h2f(lo),
               u2f(raw32[r * 128]));
      }
    }
    for (int r = 0; r < 128; ++r) {
      for (int j = 0; j < 128; ++j) {
        const uint16_t h = uint16_t((pk[r * 64 + j / 2] >> (16 * (j & 1))) & 0xffff);
        if (uint16_t(raw[r * 128 + j] & 0xffff) != h) ++n_layout_bad;
        if (trial == 0 && r < 16) continue;
        if (j == 0) continue;
        double ex = 0, sabs = 0, na = 0, nb = 0;
        for (int k = 0; k < KP; ++k) {
          const double a = h2f(A[r * KP + k]), b = h2f(B[j * KP + k]);
          ex += a * b;
          sabs += std::fabs(a * b);
          na += a * a;
          nb += b * b;
        }
        const double got = h2f(h);
        const double err = std::fabs(got - ex);
        worst_rel_abs = std::max(worst_rel_abs, err / sabs);
        worst_rel_norm = std::max(worst_rel_norm, err / std::sqrt(na * nb));
        const double ulp = std::ldexp(1.0, std::ilogb(std::max(std::fabs(ex), 6.1e-5)) - 10);
        worst_ulps = std::max(worst_ulps, err / ulp);
        if (h2f(f2h(float(ex))) == got) ++n_single_rn;
        ++n_total;
        if (std::fabs(double(u2f(raw32[r * 128 + j])) - ex) > 1e-6 * sabs) ++n_f32_bad;
      }
    }
  }
  printf("layout mismatches (raw low half vs pack::16b): %lld\n", n_layout_bad);
  printf("random: n=%lld  single-RN-of-exact %.4f  worst err/sum|ab| %.3e (2^%.2f)  "
         "worst err/(|a||b|) %.3e (2^%.2f)  worst err in ulp(exact) %.3f  f32acc bad %lld\n",
         n_total, double(n_single_rn) / n_total, worst_rel_abs, std::log2(worst_rel_abs),
         worst_rel_norm, std::log2(worst_rel_norm), worst_ulps, n_f32_bad);
  return 0;
}

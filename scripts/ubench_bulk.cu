// L2 -> SMEM bulk-copy stream microbenchmark (development aid): one CTA per SM, lane 0 of warp 0
// streams `tiles` tiles of `tb` bytes (as `nc` bulk copies each) from an L2-resident buffer of
// `nbuf` tiles (rotated start per CTA, as mf_tc_kernel) through an S-stage ring; warp 1 waits
// each stage's full barrier and releases it at once.  Reports aggregate GB/s and clk per tile.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_1810_01967_b200/csrc/cbb_common.cuh"
namespace cbb { void set_last_error(const char*) {} }
using namespace cbb;

// P producer threads (lanes 0..P-1 of warp 0 if !pw, else lane 0 of warps 0..P-1); producer p owns
// stages st = p (mod P).  self=1: no consumer warp; each producer waits its own full barriers
// (ring of S) instead.  Phase timing of producer 0 in CTA 0 -> ph[0..2].
__global__ void k(const uint8_t* buf, int nbuf, int tb, int nc, int S, int tiles, int P, int pw,
                  int self, unsigned long long* cyc, long long* ph_out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * tb);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    mbar_fence_init();
  }
  __syncthreads();
  const int rot = int((int64_t(blockIdx.x) * nbuf) / gridDim.x);
  const int cw = pw ? P : 1;  // consumer warp index
  int prod = -1;
  if (pw) { if (warp < P && lane == 0) prod = warp; }
  else if (warp == 0 && lane < P) prod = lane;
  long long t0 = clock64();
  long long tw = 0, tx = 0, tc = 0;
  if (prod >= 0) {
    const uint64_t pol = policy_evict_last();
    int st = prod; uint32_t ph = 0; int b = rot + prod; if (b >= nbuf) b -= nbuf;
    const uint32_t chunk = uint32_t(tb / nc);
    int done = 0;  // self mode: tiles waited
    for (int t = prod; t < tiles; t += P) {
      long long a0 = clock64();
      if (self) {
        if (t >= S) { mbar_wait(full + st, ph ^ 1u); ++done; }
      } else {
        mbar_wait(empty + st, ph ^ 1u);
      }
      long long a1 = clock64();
      mbar_arrive_expect_tx(full + st, uint32_t(tb));
      long long a2 = clock64();
      for (int c = 0; c < nc; ++c)
        bulk_g2s(smem + st * tb + c * chunk, buf + size_t(b) * tb + c * chunk, chunk, full + st, pol);
      long long a3 = clock64();
      tw += a1 - a0; tx += a2 - a1; tc += a3 - a2;
      b += P; if (b >= nbuf) b -= nbuf;
      st += P; if (st >= S) { st -= S; ph ^= 1u; }
    }
    if (self) {  // drain
      for (int t = 0; t < S / P; ++t) {
        mbar_wait(full + st, ph ^ 1u);
        st += P; if (st >= S) { st -= S; ph ^= 1u; }
      }
    }
  } else if (!self && warp == cw) {
    int st = 0; uint32_t ph = 0;
    for (int t = 0; t < tiles; ++t) {
      mbar_wait(full + st, ph);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      if (++st == S) { st = 0; ph ^= 1u; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(clock64() - t0));
  if (blockIdx.x == 0 && prod == 0) { ph_out[0] = tw; ph_out[1] = tx; ph_out[2] = tc; }
}

int main(int argc, char** argv) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t bufbytes = 8u << 20;
  uint8_t* buf;
  cudaMalloc(&buf, bufbytes + (1 << 20));
  cudaMemset(buf, 0, bufbytes + (1 << 20));
  unsigned long long* cyc;
  long long* phd;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&phd, 24);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg { int tb, S, nc, P, pw, self; };
  const Cfg cfgs[] = {
      {10240, 9, 1, 1, 0, 0}, {10240, 9, 1, 1, 0, 1}, {7680, 9, 1, 1, 0, 0},
      {10240, 9, 1, 3, 0, 0}, {10240, 12, 1, 2, 0, 0}, {10240, 12, 1, 4, 0, 0},
      {10240, 9, 1, 3, 1, 0}, {10240, 12, 1, 2, 1, 0}, {10240, 9, 1, 3, 0, 1},
      {7680, 12, 1, 3, 0, 0}, {7680, 12, 1, 3, 1, 0}, {20480, 6, 1, 3, 0, 0},
      {5120, 18, 1, 3, 0, 0}, {5120, 18, 1, 6, 0, 0}, {10240, 18, 1, 6, 0, 0},
  };
  for (const Cfg& c : cfgs) {
    const int nbuf = int(bufbytes / c.tb);
    const long long total_bytes = 4'000'000'000LL;
    const int grid = nsm;
    const int tiles = int(total_bytes / c.tb / grid / 36) * 36;
    const int sm = c.S * c.tb + 2 * c.S * 8 + 1024;
    const int threads = 32 * ((c.pw ? c.P : 1) + 1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cyc, 0, 8);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<grid, threads, sm>>>(buf, nbuf, c.tb, c.nc, c.S, tiles, c.P, c.pw, c.self, cyc, phd);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long cy = 0; cudaMemcpy(&cy, cyc, 8, cudaMemcpyDeviceToHost);
      long long ph[3]; cudaMemcpy(ph, phd, 24, cudaMemcpyDeviceToHost);
      const double per = double(tiles) / c.P;
      if (rep == 1)
        printf("tile %6d B S %2d P %d %s%s: %7.3f ms %8.1f GB/s %6.1f clk/tile/CTA | producer0 per own tile: wait %6.1f expect %5.1f copy %5.1f\n",
               c.tb, c.S, c.P, c.pw ? "warps" : "lanes", c.self ? " self" : "", ms,
               double(tiles) * c.tb * grid / (ms * 1e6), double(cy) / grid / tiles,
               ph[0] / per, ph[1] / per, ph[2] / per);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}

// Exact cone projection on B200 (sm_100a).  See cbb_project.cuh for the scheme.
//
// Kernels
//   prep_dict_kernel     dictionary -> fp64 copy, planar fp32 copy, bf16 UMMA tiles, error bounds
//   prologue_kernel      Z (or X - mu G) -> bf16 UMMA voxel tiles + certified windows
//   mf_tc_kernel<KP>     tcgen05 bf16 screening, persistent + warp specialised:
//                          warp 0 bulk-copy producer, warp 1 MMA issuer, warp 2 TMEM owner,
//                          warps 4..11 epilogue (TMEM -> regs, running max + certified
//                          candidates, fp64 rescoring and write-back of the winner)
//   mf_ffma_kernel<S>    fp32 FFMA screening with the same candidate machinery
//   exhaustive_kernel    fp64 exhaustive scan for overflowed voxels (and for s > 32)
//   reduce kernels       deterministic two-stage fp64 sums
#include "cbb_common.cuh"
#include "cbb_project.cuh"

#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstdio>

namespace cbb {

// ============================================================== helpers
__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
  atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
}

__device__ __forceinline__ double2 load_z(const ZSource& zs, int64_t v, int s, int k) {
  if (zs.x != nullptr) {
    float2 a = zs.z_out[v * s + k];
    return make_double2(a.x, a.y);
  }
  if (zs.z128) return reinterpret_cast<const double2*>(zs.z)[v * s + k];
  float2 a = reinterpret_cast<const float2*>(zs.z)[v * s + k];
  return make_double2(a.x, a.y);
}

// Exact Re<z_v, d_j> in fp64 (projection.py:61 arithmetic).  The z dtype is resolved once and
// the k loop is unrolled so all loads of a candidate are in flight together.
template <typename ZT>
__device__ __forceinline__ double dot_re(const ZT* __restrict__ z, const double2* __restrict__ a,
                                         int s) {
  double acc0 = 0.0, acc1 = 0.0;
  int k = 0;
  for (; k + 4 <= s; k += 4) {
    const ZT z0 = z[k], z1 = z[k + 1], z2 = z[k + 2], z3 = z[k + 3];
    const double2 a0 = a[k], a1 = a[k + 1], a2 = a[k + 2], a3 = a[k + 3];
    acc0 = fma(double(z0.x), a0.x, acc0);
    acc0 = fma(double(z0.y), a0.y, acc0);
    acc1 = fma(double(z1.x), a1.x, acc1);
    acc1 = fma(double(z1.y), a1.y, acc1);
    acc0 = fma(double(z2.x), a2.x, acc0);
    acc0 = fma(double(z2.y), a2.y, acc0);
    acc1 = fma(double(z3.x), a3.x, acc1);
    acc1 = fma(double(z3.y), a3.y, acc1);
  }
  for (; k < s; ++k) {
    const ZT zk = z[k];
    const double2 ak = a[k];
    acc0 = fma(double(zk.x), ak.x, acc0);
    acc0 = fma(double(zk.y), ak.y, acc0);
  }
  return acc0 + acc1;
}

__device__ __forceinline__ double exact_score_g(const ZSource& zs, int64_t v, int s,
                                                const double2* __restrict__ atom) {
  if (zs.x != nullptr) return dot_re(zs.z_out + v * s, atom, s);
  if (zs.z128) return dot_re(reinterpret_cast<const double2*>(zs.z) + v * s, atom, s);
  return dot_re(reinterpret_cast<const float2*>(zs.z) + v * s, atom, s);
}

// Winner write-back: idx, gamma = max(score, 0) (projection.py:42), gamma * D_j (projection.py:64),
// and for the IPG trial dX = P - X with its squared norm (solver.py:129-130).
__device__ void write_winner(const ProjOut& out, const DictView& dv, int64_t v, int64_t j,
                             double score) {
  const int s = dv.s;
  const double gamma = score > 0.0 ? score : 0.0;
  if (out.idx) {
    if (out.idx64) reinterpret_cast<int64_t*>(out.idx)[v] = j;
    else reinterpret_cast<int32_t*>(out.idx)[v] = int32_t(j);
  }
  if (out.gamma) out.gamma[v] = gamma;
  const double2* a = dv.atoms64 + j * s;
  double nd = 0.0;
  for (int k = 0; k < s; ++k) {
    double2 ak = a[k];
    double pr = gamma * ak.x, pi = gamma * ak.y;
    if (out.proj) {
      if (out.proj128) reinterpret_cast<double2*>(out.proj)[v * s + k] = make_double2(pr, pi);
      else reinterpret_cast<float2*>(out.proj)[v * s + k] = make_float2(float(pr), float(pi));
    }
    if (out.dx) {
      float2 xk = out.x[v * s + k];
      float2 dk = make_float2(float(pr) - xk.x, float(pi) - xk.y);
      out.dx[v * s + k] = dk;
      nd += double(dk.x) * dk.x + double(dk.y) * dk.y;
    }
  }
  if (out.nd_v) out.nd_v[v] = nd;
}

// Drop stale entries (approximate score below the current threshold); returns the new count.
__device__ __noinline__ int cand_compact(int* cj, float* cs, int stride, float thr) {
  int k = 0;
  for (int c = 0; c < kCandCap; ++c) {
    const float x = cs[c * stride];
    const int y = cj[c * stride];
    if (x >= thr) {
      cs[k * stride] = x;
      cj[k * stride] = y;
      ++k;
    }
  }
  return k;
}

// Per-thread certified candidate list living in shared memory (column `slot` of
// [kCandCap][ncols] arrays).  Entries below the current threshold are stale and
// are dropped lazily when the list fills up.
struct CandList {
  int* cj;
  float* cs;
  int stride;
  int cnt;
  bool ovf;

  __device__ __forceinline__ void insert(int j, float sc, float thr) {
    if (cnt == kCandCap) {
      cnt = cand_compact(cj, cs, stride, thr);
      if (cnt == kCandCap) {
        ovf = true;
        return;
      }
    }
    cs[cnt * stride] = sc;
    cj[cnt * stride] = j;
    ++cnt;
  }
};

// Rescore in fp64 every atom of the list entries that survive the final window.  An entry is
// (first atom index, approximate max over its `span` atoms): span 1 for the FFMA screen (one
// atom per entry), 32 for the tcgen05 screen (one 32-atom chunk per entry).  Ties keep the
// lowest index (np.argmax, projection.py:62).
__device__ __forceinline__ void rescore_one(const ZSource& zs, const DictView& dv, int64_t v,
                                            int64_t j, int64_t& best, double& bs) {
  const double sc = exact_score_g(zs, v, dv.s, dv.atoms64 + j * dv.s);
  if (sc > bs || (sc == bs && j < best)) {
    bs = sc;
    best = j;
  }
}

// Chunk entries of the tcgen05 screen: (first atom / 32) in bits [0,20), and a 12-bit mask of
// the 3-wide groups (bits 0..9 -> atoms 3g..3g+2) and the two trailing atoms (bits 10, 11)
// whose approximate scores reached the window when the chunk was recorded.
constexpr int kChunkShift = 20;
__device__ __forceinline__ int pack_chunk(int64_t jb, uint32_t mask) {
  return int(uint32_t(jb >> 5) | (mask << kChunkShift));
}

__device__ __forceinline__ void rescore_entries(const ZSource& zs, const DictView& dv, int64_t v,
                                                const int* cj, const float* cs, int stride,
                                                int cnt, float thr, int span, int64_t& best,
                                                double& bs) {
  for (int c = 0; c < cnt; ++c) {
    if (cs[c * stride] >= thr) {
      const int e = cj[c * stride];
      if (span == 1) {
        rescore_one(zs, dv, v, e, best, bs);
        continue;
      }
      const int64_t j0 = int64_t(uint32_t(e) & ((1u << kChunkShift) - 1)) << 5;
      uint32_t mask = uint32_t(e) >> kChunkShift;
      while (mask) {
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        const int lo = b < 10 ? 3 * b : 20 + b, hi = b < 10 ? lo + 3 : lo + 1;
        for (int i = lo; i < hi; ++i)
          if (j0 + i < dv.d) rescore_one(zs, dv, v, j0 + i, best, bs);
      }
    }
  }
}

// Rescore the certified candidates in fp64 and write the winner; zero voxels go
// straight to index 0 (np.argmax of an all-zero row); overflow -> exhaustive list.
__device__ void finalize_voxel(const ZSource& zs, const DictView& dv, const ProjOut& out,
                               int64_t v, float win, float runmax, const CandList& cl,
                               int* ovf_count, int64_t* ovf_list, int span = 1) {
  if (win < 0.f) {
    write_winner(out, dv, v, 0, 0.0);
    return;
  }
  int64_t best = -1;
  double bs = -INFINITY;
  if (!cl.ovf)
    rescore_entries(zs, dv, v, cl.cj, cl.cs, cl.stride, cl.cnt, runmax - win, span, best, bs);
  if (best < 0) {
    int slot = atomicAdd(ovf_count, 1);
    ovf_list[slot] = v;
    return;
  }
  write_winner(out, dv, v, best, bs);
}

// ============================================================== dictionary preparation
__global__ void prep_dict_kernel(const void* __restrict__ atoms_in, int in128, int64_t d, int s,
                                 int s_pad, int kpad, double2* __restrict__ atoms64,
                                 float* __restrict__ atoms32, uint8_t* __restrict__ atoms_tc,
                                 float* __restrict__ bounds) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double del_bf = 0, nrm = 0, nrm_bf = 0, del32 = 0, nrm32 = 0;
  const int tile = int(j / kTileRows), r = int(j % kTileRows);
  uint8_t* trow = atoms_tc + size_t(tile) * kTileRows * kpad * 2;
  for (int k = 0; k < s; ++k) {
    double re, im;
    if (in128) {
      double2 a = reinterpret_cast<const double2*>(atoms_in)[j * s + k];
      re = a.x; im = a.y;
    } else {
      float2 a = reinterpret_cast<const float2*>(atoms_in)[j * s + k];
      re = a.x; im = a.y;
    }
    atoms64[j * s + k] = make_double2(re, im);
    const float re32 = float(re), im32 = float(im);
    atoms32[j * 2 * s_pad + k] = re32;
    atoms32[j * 2 * s_pad + s_pad + k] = im32;
    const unsigned short bre = bf16_bits_rn(re32), bim = bf16_bits_rn(im32);
    const double fre = bf16_bits_to_float(bre), fim = bf16_bits_to_float(bim);
    // element e -> 16B chunk e/8, offset (e%8)*2 bytes
    const int e_re = k, e_im = s + k;
    if (2 * s <= 64) {
    *reinterpret_cast<unsigned short*>(trow + tile_chunk_offset(r, e_re >> 3, kpad) +
                                       (e_re & 7) * 2) = bre;
    *reinterpret_cast<unsigned short*>(trow + tile_chunk_offset(r, e_im >> 3, kpad) +
                                       (e_im & 7) * 2) = bim;
    }
    nrm += re * re + im * im;
    nrm_bf += fre * fre + fim * fim;
    del_bf += (re - fre) * (re - fre) + (im - fim) * (im - fim);
    nrm32 += double(re32) * re32 + double(im32) * im32;
    del32 += (re - re32) * (re - re32) + (im - im32) * (im - im32);
  }
  for (int k = s; k < s_pad; ++k) {
    atoms32[j * 2 * s_pad + k] = 0.f;
    atoms32[j * 2 * s_pad + s_pad + k] = 0.f;
  }
  atomic_max_nonneg(bounds + kBDeltaBf16, __double2float_ru(sqrt(del_bf)));
  atomic_max_nonneg(bounds + kBDmax, __double2float_ru(sqrt(nrm)));
  atomic_max_nonneg(bounds + kBDbfMax, __double2float_ru(sqrt(nrm_bf)));
  atomic_max_nonneg(bounds + kBDelta32, __double2float_ru(sqrt(del32)));
  atomic_max_nonneg(bounds + kBD32Max, __double2float_ru(sqrt(nrm32)));
}

// ============================================================== prologue
// One thread per voxel (n_pad = whole voxel tiles).  Produces the bf16 UMMA
// voxel tiles and both certified windows:
//   |s~ - s| <= ||z - z~|| * max||d|| + ||z~|| * max||d - d~|| + acc(K) * ||z~|| * max||d~||
// window = 2 * bound (true argmax j* satisfies s~_j* >= max s~ - window).
__global__ void prologue_kernel(ZSource zs, int64_t n, int64_t n_pad, int s, int kpad,
                                const float* __restrict__ bounds, uint8_t* __restrict__ ztiles,
                                float* __restrict__ win_tc, float* __restrict__ win32,
                                int s_pad) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n_pad) return;
  // bf16 rows in 128-row UMMA tiles (K-major, swizzled): one bulk copy lands them in SMEM
  const int tile = int(v / kTileRows), r = int(v % kTileRows);
  uint8_t* trow = ztiles ? ztiles + size_t(tile) * kTileRows * kpad * 2 : nullptr;
  if (v >= n) {
    if (trow)
      for (int c = 0; c < kpad / 8; ++c)
        *reinterpret_cast<uint4*>(trow + tile_chunk_offset(r, c, kpad)) = make_uint4(0, 0, 0, 0);
    return;
  }
  unsigned short row[64];
#pragma unroll
  for (int e = 0; e < 64; ++e) row[e] = 0;
  double nz = 0, ez_bf = 0, nz_bf = 0, ez32 = 0, nz32 = 0;
  for (int k = 0; k < s; ++k) {
    double re, im;
    if (zs.x != nullptr) {
      const float2 xk = zs.x[v * s + k], gk = zs.g[v * s + k];
      const float zr = __fmaf_rn(-zs.mu, gk.x, xk.x), zi = __fmaf_rn(-zs.mu, gk.y, xk.y);
      zs.z_out[v * s + k] = make_float2(zr, zi);
      re = zr; im = zi;
    } else if (zs.z128) {
      double2 a = reinterpret_cast<const double2*>(zs.z)[v * s + k];
      re = a.x; im = a.y;
    } else {
      float2 a = reinterpret_cast<const float2*>(zs.z)[v * s + k];
      re = a.x; im = a.y;
    }
    const float re32 = float(re), im32 = float(im);
    const unsigned short bre = bf16_bits_rn(re32), bim = bf16_bits_rn(im32);
    if (trow) {  // tensor-core path requires 2s <= 64
      row[k] = bre;
      row[s + k] = bim;
    }
    const double fre = bf16_bits_to_float(bre), fim = bf16_bits_to_float(bim);
    nz += re * re + im * im;
    ez_bf += (re - fre) * (re - fre) + (im - fim) * (im - fim);
    nz_bf += fre * fre + fim * fim;
    ez32 += (re - re32) * (re - re32) + (im - im32) * (im - im32);
    nz32 += double(re32) * re32 + double(im32) * im32;
  }
  if (trow) {
    for (int c = 0; c < kpad / 8; ++c) {
      uint4 pk;
      pk.x = uint32_t(row[c * 8 + 0]) | (uint32_t(row[c * 8 + 1]) << 16);
      pk.y = uint32_t(row[c * 8 + 2]) | (uint32_t(row[c * 8 + 3]) << 16);
      pk.z = uint32_t(row[c * 8 + 4]) | (uint32_t(row[c * 8 + 5]) << 16);
      pk.w = uint32_t(row[c * 8 + 6]) | (uint32_t(row[c * 8 + 7]) << 16);
      *reinterpret_cast<uint4*>(trow + tile_chunk_offset(r, c, kpad)) = pk;
    }
  }
  const double dmax = bounds[kBDmax], dbf = bounds[kBDbfMax], delbf = bounds[kBDeltaBf16];
  const double d32 = bounds[kBD32Max], del32 = bounds[kBDelta32];
  if (nz == 0.0) {
    if (win_tc) win_tc[v] = -1.f;
    if (win32) win32[v] = -1.f;
    return;
  }
  // tensor-core fp32 accumulation: generous (K + 32) ulp-of-2^-23 per unit of sum |products|
  const double acc_tc = double(kpad + 32) * 0x1p-23;
  const double acc32 = double(2 * s_pad + 4) * 0x1p-24;
  const double eb = sqrt(ez_bf) * dmax + sqrt(nz_bf) * delbf + acc_tc * sqrt(nz_bf) * dbf;
  const double e3 = sqrt(ez32) * dmax + sqrt(nz32) * del32 + acc32 * sqrt(nz32) * d32;
  if (win_tc) win_tc[v] = __double2float_ru(2.0 * eb * 1.001 + 1e-30);
  if (win32) win32[v] = __double2float_ru(2.0 * e3 * 1.001 + 1e-30);
}

// ============================================================== FFMA screening
template <int S>
__global__ void __launch_bounds__(128) mf_ffma_kernel(ZSource zs, DictView dv, int64_t n,
                                                      const float* __restrict__ win32,
                                                      ProjOut out, int* ovf_count,
                                                      int64_t* ovf_list) {
  constexpr int TA = 128;  // atoms per shared tile
  __shared__ __align__(16) float sA[TA * 2 * S];
  __shared__ int cj[kCandCap * 128];
  __shared__ float cs[kCandCap * 128];
  const int tid = threadIdx.x;
  const int64_t v = int64_t(blockIdx.x) * 128 + tid;
  const bool live = v < n;
  float zr[S], zi[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    zr[k] = 0.f;
    zi[k] = 0.f;
  }
  float win = -1.f;
  if (live) {
    win = win32[v];
    for (int k = 0; k < dv.s; ++k) {
      double2 z = load_z(zs, v, dv.s, k);
#pragma unroll
      for (int kk = 0; kk < S; ++kk)
        if (kk == k) { zr[kk] = float(z.x); zi[kk] = float(z.y); }
    }
  }
  CandList cl{cj + tid, cs + tid, 128, 0, false};
  bool active = live && win >= 0.f;
  float runmax = -INFINITY, thr = active ? -INFINITY : INFINITY;
  const int64_t d = dv.d;
  for (int64_t base = 0; base < d; base += TA) {
    const int cnt = int((d - base) < TA ? (d - base) : TA);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(dv.atoms32 + base * 2 * S);
    float4* dst = reinterpret_cast<float4*>(sA);
    for (int i = tid; i < cnt * 2 * S / 4; i += 128) dst[i] = src[i];
    __syncthreads();
    for (int a = 0; a < cnt; ++a) {
      const float* at = sA + a * 2 * S;
      float sc = 0.f;
#pragma unroll
      for (int k = 0; k < S; ++k) {
        sc = __fmaf_rn(zr[k], at[k], sc);
        sc = __fmaf_rn(zi[k], at[S + k], sc);
      }
      if (sc >= thr) {
        runmax = fmaxf(runmax, sc);
        if (active) {
          thr = runmax - win;
          cl.insert(int(base + a), sc, thr);
          if (cl.ovf) { active = false; thr = INFINITY; }
        }
      }
    }
  }
  if (live) finalize_voxel(zs, dv, out, v, win, runmax, cl, ovf_count, ovf_list);
}

// ============================================================== exhaustive fp64 scan
// Warp per voxel.  Handles the overflow list (list != null) or every voxel (list == null).
__global__ void __launch_bounds__(256) exhaustive_kernel(ZSource zs, DictView dv, int64_t n,
                                                         const int* ovf_count,
                                                         const int64_t* ovf_list,
                                                         ProjOut out) {
  extern __shared__ double zsh[];  // 8 warps x 2s
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int s = dv.s;
  double* zw = zsh + size_t(wid) * 2 * s;
  const int64_t total = ovf_list ? int64_t(*ovf_count) : n;
  const int64_t nw = int64_t(gridDim.x) * 8;
  for (int64_t i = int64_t(blockIdx.x) * 8 + wid; i < total; i += nw) {
    const int64_t v = ovf_list ? ovf_list[i] : i;
    for (int k = lane; k < s; k += 32) {
      double2 z = load_z(zs, v, s, k);
      zw[k] = z.x;
      zw[s + k] = z.y;
    }
    __syncwarp();
    double bs = -INFINITY;
    int64_t best = INT64_MAX;
    for (int64_t j = lane; j < dv.d; j += 32) {
      const double2* a = dv.atoms64 + j * s;
      double acc = 0.0;
      for (int k = 0; k < s; ++k) {
        double2 ak = a[k];
        acc = fma(zw[k], ak.x, acc);
        acc = fma(zw[s + k], ak.y, acc);
      }
      if (acc > bs) { bs = acc; best = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double obs = __shfl_xor_sync(0xffffffffu, bs, o);
      int64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
      if (obs > bs || (obs == bs && ob < best)) { bs = obs; best = ob; }
    }
    if (best == INT64_MAX) best = 0;  // all-NaN row: np.argmax returns the first NaN -> 0
    if (lane == 0) write_winner(out, dv, v, best, bs);
    __syncwarp();
  }
}

// ============================================================== tcgen05 screening
// One CTA per SM (persistent, warp specialised).
//   warp 0      bulk-copy producer: voxel tiles (SUBS x 128 rows) and a ring of atom tiles
//               (BN rows), both pre-swizzled in global memory so one flat copy lands a tile
//   warp 1      MMA issuer: whole warp runs the loop, one elected lane issues
//               SUBS x KP/16 tcgen05.mma (M=128, N=BN, K=16, A and B from SMEM) per atom tile
//               into one of two TMEM accumulator stages
//   warp 2      TMEM allocator
//   warps 4..   epilogue: warp (sub, q, half) owns TMEM lanes 32q..32q+31 of sub-tile `sub`
//               (one voxel per thread) and 1/SPLIT of the stage's columns; running max +
//               certified candidate list per (voxel, part); at the end of the voxel tile the
//               part-0 thread rescores every part's candidates in fp64 and writes the winner.
// Shapes follow measured sm_100a rates (scripts/ubench_mma.cu): an M=128 x N=128 x K=16 SS-MMA
// reads 8 KB of operands per 64 clk, exactly the 128 B/clk shared-memory rate, and runs at
// 4096 MAC/clk/SM when issued through elect.sync; smaller N or lane-0-only issue fall far
// below.  Atom tiles are visited in a per-CTA rotated order so the 148 CTAs spread over L2.
template <int KP, int SUBS, int BN, int SPLIT>
struct TcCfg {
  static constexpr int kATileBytes = kTileRows * KP * 2;  // one 128-voxel sub-tile
  static constexpr int kABytes = SUBS * kATileBytes;
  static constexpr int kBBytes = BN * KP * 2;
  static constexpr int kStages = (64 * 1024) / kBBytes;
  static constexpr int kAccCols = SUBS * BN;
  static constexpr int kAcc = 512 / kAccCols;
  static_assert(kAcc >= 2 && kAcc * kAccCols == 512, "accumulator stages must tile 512 columns");
  static constexpr int kCols = BN / SPLIT;                 // columns per epilogue thread per stage
  static_assert(kCols % 32 == 0, "epilogue chunks are 32 columns");
  static constexpr int kEpiWarps = SUBS * 4 * SPLIT;
  static constexpr int kThreads = (4 + kEpiWarps) * 32;
  static constexpr int kVox = SUBS * 128;
  static constexpr int kSlots = kVox * SPLIT;
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + 2 * kABytes;
  static constexpr int kOffCj = kOffB + kStages * kBBytes;
  static constexpr int kOffCs = kOffCj + kCandCap * kSlots * 4;
  static constexpr int kOffX = kOffCs + kCandCap * kSlots * 4;   // part-thread exchange
  static constexpr int kOffBar = kOffX + kSlots * 8;
  static constexpr int kNumBars = 4 + 2 * kStages + 2 * kAcc;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffTmem + 16 + 1024;  // + alignment slack
  static_assert(kSmem <= 227 * 1024, "shared memory");
  static constexpr uint32_t kIdesc = idesc_bf16_f32(128, BN);
};

__device__ __forceinline__ uint8_t* align1024_smem(uint8_t* raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);  // keeps the shared address space
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Screen 32 approximate scores of one voxel (one thread): running max + certified window.
// Fast path: 16 three-input maxes + one compare.  When the chunk max enters the window the
// chunk itself (first atom index + its max) is recorded -- no per-value work; the finalize
// rescans recorded chunks exactly.  Any atom inside the final window lies in a recorded chunk
// whose max is at least its score, so the certificate is unchanged.
__device__ __forceinline__ void screen32(float (&r)[32], int64_t jb, bool tail, int64_t d,
                                         float win, float& runmax, float& thr, bool& active,
                                         CandList& cl, int epi_mode = 0,
                                         unsigned long long* dbg = nullptr) {
  if (tail) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (jb + i >= d) r[i] = -INFINITY;
  }
  float m[10];
#pragma unroll
  for (int g = 0; g < 10; ++g) m[g] = fmax3(r[3 * g], r[3 * g + 1], r[3 * g + 2]);
  const float n0 = fmax3(m[0], m[1], m[2]), n1 = fmax3(m[3], m[4], m[5]);
  const float n2 = fmax3(m[6], m[7], m[8]), n3 = fmax3(m[9], r[30], r[31]);
  const float cm = fmax3(n0, n1, fmaxf(n2, n3));
  if (epi_mode == 5 && dbg) {  // dev: count warp-level slow-path entries
    const unsigned any = __ballot_sync(0xffffffffu, cm >= thr);
    if (any && (threadIdx.x & 31) == 0) atomicAdd(dbg, 1ull);
  }
  if (cm >= thr) {
    runmax = fmaxf(runmax, cm);
    if (active) {
      thr = runmax - win;
      if (epi_mode != 4) {
        uint32_t mask = (r[30] >= thr ? (1u << 10) : 0u) | (r[31] >= thr ? (1u << 11) : 0u);
#pragma unroll
        for (int g = 0; g < 10; ++g) mask |= (m[g] >= thr) ? (1u << g) : 0u;
        cl.insert(pack_chunk(jb, mask), cm, thr);
      }
      if (cl.ovf) {
        active = false;
        thr = INFINITY;
      }
    }
  }
}

template <int KP, int SUBS, int BN, int SPLIT>
__global__ void __launch_bounds__(TcCfg<KP, SUBS, BN, SPLIT>::kThreads, 1)
    mf_tc_kernel(const uint8_t* __restrict__ ztiles, int64_t n, int n_vt,
                 const float* __restrict__ win_tc, ZSource zs, DictView dv, ProjOut out,
                 int* ovf_count, int64_t* ovf_list, int epi_mode) {
  using C = TcCfg<KP, SUBS, BN, SPLIT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024_smem(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 2;
  uint64_t* b_full = bars + 4;
  uint64_t* b_empty = b_full + C::kStages;
  uint64_t* t_full = b_empty + C::kStages;
  uint64_t* t_empty = t_full + C::kAcc;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t d = dv.d;
  const int nB = int((d + BN - 1) / BN);
  const int rot = int((int64_t(blockIdx.x) * nB) / gridDim.x);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(a_full + i, 1);
      mbar_init(a_empty + i, 1);
    }
    for (int i = 0; i < C::kAcc; ++i) {
      mbar_init(t_full + i, 1);
      mbar_init(t_empty + i, C::kEpiWarps);
    }
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);
    }
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------ producer (bulk copies)
    const uint64_t pol_b = policy_evict_last(), pol_a = policy_evict_first();
    int st = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int vt = blockIdx.x; vt < n_vt; vt += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(a_empty + buf, ((it >> 1) & 1) ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(a_full + buf, C::kABytes);
        bulk_g2s(smem + C::kOffA + buf * C::kABytes, ztiles + size_t(vt) * C::kABytes,
                 C::kABytes, a_full + buf, pol_a);
      }
      __syncwarp();
      int ba = rot;
      for (int b = 0; b < nB; ++b) {
        mbar_wait(b_empty + st, ph ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(b_full + st, C::kBBytes);
          bulk_g2s(smem + C::kOffB + st * C::kBBytes, dv.atoms_tc + size_t(ba) * C::kBBytes,
                   C::kBBytes, b_full + st, pol_b);
        }
        __syncwarp();
        if (++st == C::kStages) { st = 0; ph ^= 1; }
        if (++ba == nB) ba = 0;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (warp-uniform, elected lane)
    int st = 0;
    uint32_t ph = 0;
    int it = 0;
    uint32_t tcount = 0;
    const uint32_t a_base = smem_u32(smem + C::kOffA), b_base = smem_u32(smem + C::kOffB);
    for (int vt = blockIdx.x; vt < n_vt; vt += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(a_full + buf, (it >> 1) & 1);
      tc_fence_after();
      for (int b = 0; b < nB; ++b) {
        const int acc = int(tcount % C::kAcc);
        mbar_wait(b_full + st, ph);
        mbar_wait(t_empty + acc, ((tcount / C::kAcc) & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bdesc = umma_desc_kmajor(b_base + st * C::kBBytes, KP);
#pragma unroll
          for (int sub = 0; sub < SUBS; ++sub) {
            const uint64_t adesc =
                umma_desc_kmajor(a_base + buf * C::kABytes + sub * C::kATileBytes, KP);
            const uint32_t dcol = tbase + uint32_t(acc * C::kAccCols + sub * BN);
#pragma unroll
            for (int k = 0; k < KP / 16; ++k)
              tc_mma_bf16(dcol, adesc + uint64_t(2 * k), bdesc + uint64_t(2 * k), C::kIdesc,
                          k > 0 ? 1u : 0u);
          }
          tc_commit(b_empty + st);
          tc_commit(t_full + acc);
        }
        __syncwarp();
        ++tcount;
        if (++st == C::kStages) { st = 0; ph ^= 1; }
      }
      if (elect_one()) tc_commit(a_empty + buf);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue
    const int e = warp - 4;
    const int q = warp & 3, sub = (e >> 2) % SUBS, part = e / (4 * SUBS);
    const int row = sub * 128 + q * 32 + lane;  // voxel row inside the voxel tile
    const int slot = part * C::kVox + row;
    int* cj_base = reinterpret_cast<int*>(smem + C::kOffCj);
    float* cs_base = reinterpret_cast<float*>(smem + C::kOffCs);
    float* xmax = reinterpret_cast<float*>(smem + C::kOffX);          // [slot] part runmax
    int* xcnt = reinterpret_cast<int*>(smem + C::kOffX) + C::kSlots;  // [slot] count / -1 = ovf
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    unsigned long long* dbg = reinterpret_cast<unsigned long long*>(ovf_list) + 1;
    uint32_t tcount = 0;
    for (int vt = blockIdx.x; vt < n_vt; vt += gridDim.x) {
      const int64_t v = int64_t(vt) * C::kVox + row;
      const bool live = v < n;
      const float win = live ? win_tc[v] : -1.f;
      bool active = live && win >= 0.f;
      CandList cl{cj_base + slot, cs_base + slot, C::kSlots, 0, false};
      float runmax = -INFINITY, thr = active ? -INFINITY : INFINITY;
      int ba = rot;
      for (int b = 0; b < nB; ++b) {
        const int acc = int(tcount % C::kAcc);
        mbar_wait(t_full + acc, (tcount / C::kAcc) & 1);
        tc_fence_after();
        const bool tail = (ba == nB - 1) && (int64_t(nB) * BN > d);
        const uint32_t col0 = uint32_t(acc * C::kAccCols + sub * BN + part * C::kCols);
        const int64_t jb0 = int64_t(ba) * BN + part * C::kCols;
        if (epi_mode != 2) {
#pragma unroll
          for (int h = 0; h + 64 <= C::kCols; h += 64) {
            float ra[32], rb[32];
            __syncwarp();
            const uint32_t taddr = tbase + lane_off + col0 + uint32_t(h);
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tc_wait_ld();
            if (epi_mode == 1) {  // dev experiment: TMEM loads only
              runmax = fmaxf(runmax, fmaxf(ra[0], rb[31]));
              continue;
            }
            screen32(ra, jb0 + h, tail, d, win, runmax, thr, active, cl, epi_mode, dbg);
            screen32(rb, jb0 + h + 32, tail, d, win, runmax, thr, active, cl, epi_mode, dbg);
          }
          if (C::kCols % 64 == 32) {  // odd 32-column remainder
            float ra[32];
            __syncwarp();
            tmem_ld32(tbase + lane_off + col0 + uint32_t(C::kCols - 32), ra);
            tc_wait_ld();
            if (epi_mode == 1) runmax = fmaxf(runmax, ra[0]);
            else
              screen32(ra, jb0 + C::kCols - 32, tail, d, win, runmax, thr, active, cl, epi_mode,
                       dbg);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(t_empty + acc);
        ++tcount;
        if (++ba == nB) ba = 0;
      }
      if (epi_mode != 0 && epi_mode != 5 && epi_mode < 6) {  // dev experiments: keep live
        if (runmax == 12345.f) ovf_list[0] = v;
        continue;
      }
      if (SPLIT == 1) {
        if (live) finalize_voxel(zs, dv, out, v, win, runmax, cl, ovf_count, ovf_list, 32);
        continue;
      }
      // ---- merge the SPLIT per-part lists of each voxel and finalize (part-0 thread)
      xmax[slot] = runmax;
      xcnt[slot] = cl.ovf ? -1 : cl.cnt;
      named_bar_sync(1, C::kEpiWarps * 32);
      if (part == 0 && live) {
        if (win < 0.f) {
          write_winner(out, dv, v, 0, 0.0);
        } else {
          float gmax = runmax;
          bool ovf = false;
          for (int p2 = 0; p2 < SPLIT; ++p2) {
            gmax = fmaxf(gmax, xmax[p2 * C::kVox + row]);
            ovf |= xcnt[p2 * C::kVox + row] < 0;
          }
          int64_t best = -1;
          double bs = -INFINITY;
          if (epi_mode == 6 || epi_mode == 7) {  // dev: no rescoring
            best = xcnt[row] > 0 ? cj_base[row] : 0;
            bs = 1.0;
            if (epi_mode == 7) best = -2;  // skip the write-back too
          } else if (!ovf) {
            const float thr_f = gmax - win;
            for (int p2 = 0; p2 < SPLIT; ++p2) {
              const int sl = p2 * C::kVox + row;
              if (epi_mode == 5) {  // dev: count surviving chunks
                int sv = 0;
                for (int c = 0; c < xcnt[sl]; ++c) sv += cs_base[c * C::kSlots + sl] >= thr_f;
                atomicAdd(reinterpret_cast<unsigned long long*>(ovf_list) + 2,
                          (unsigned long long)sv);
              }
              rescore_entries(zs, dv, v, cj_base + sl, cs_base + sl, C::kSlots, xcnt[sl], thr_f,
                              32, best, bs);
            }
          }
          if (best == -2) {
          } else if (best < 0) {
            const int sl2 = atomicAdd(ovf_count, 1);
            ovf_list[sl2] = v;
          } else {
            write_winner(out, dv, v, best, bs);
          }
        }
      }
      named_bar_sync(1, C::kEpiWarps * 32);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// Debug: raw bf16 tcgen05 scores for voxel tile a_tile x atom tile b_tile (128 x 128, SS)
// -- validates descriptors / swizzle against a host emulation.
template <int KP>
__global__ void __launch_bounds__(128, 1)
    tc_debug_scores_kernel(const uint8_t* __restrict__ ztiles, const uint8_t* __restrict__ atiles,
                           int a_tile, int b_tile, float* __restrict__ out) {
  constexpr int kTileBytes = kTileRows * KP * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024_smem(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * kTileBytes);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 2 * kTileBytes + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(holder, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *holder;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, 2 * kTileBytes);
    bulk_g2s(smem, ztiles + size_t(a_tile) * kTileBytes, kTileBytes, bar, policy_evict_first());
    bulk_g2s(smem + kTileBytes, atiles + size_t(b_tile) * kTileBytes, kTileBytes, bar,
             policy_evict_first());
    mbar_wait(bar, 0);
    tc_fence_after();
    const uint64_t ad = umma_desc_kmajor(smem_u32(smem), KP);
    const uint64_t bd = umma_desc_kmajor(smem_u32(smem + kTileBytes), KP);
    for (int k = 0; k < KP / 16; ++k)
      tc_mma_bf16(tbase, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc_bf16_f32(128, 128),
                  k > 0);
    tc_commit(bar + 1);
  }
  __syncwarp();
  mbar_wait(bar + 1, 0);
  tc_fence_after();
  for (int c = 0; c < 4; ++c) {
    float r[32];
    tmem_ld32(tbase + (uint32_t(warp * 32) << 16) + c * 32, r);
    tc_wait_ld();
    for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * 128 + c * 32 + i] = r[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 128);
  }
}

// ============================================================== deterministic sums
__global__ void __launch_bounds__(256) reduce_stage1(const double* __restrict__ x, int64_t n,
                                                     double* __restrict__ partial) {
  __shared__ double sh[256];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = per * blockIdx.x, hi = (lo + per < n) ? lo + per : n;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += 256) acc += x[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}
__global__ void __launch_bounds__(256) reduce_stage2(const double* __restrict__ partial, int np,
                                                     double* __restrict__ out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += 256) acc += partial[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ============================================================== host side
static int s_pad_for(int s) {
  static const int pads[] = {2, 4, 6, 8, 10, 12, 16, 20, 24, 32};
  for (int p : pads)
    if (s <= p) return p;
  return -1;
}

size_t dict_bytes(int64_t d, int s, size_t* off64, size_t* off32, size_t* offtc, size_t* offb) {
  const int sp = s_pad_for(s) > 0 ? s_pad_for(s) : s;
  const int kp = kpad_for(s);
  const int64_t nbt = (d + kTileRows - 1) / kTileRows;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) & ~size_t(255);
    return r;
  };
  size_t a = take(size_t(d) * s * 16);
  size_t b = take(size_t(d) * 2 * sp * 4);
  size_t c = take(size_t(nbt) * kTileRows * kp * 2);
  size_t e = take(kBCount * sizeof(float));
  if (off64) *off64 = a;
  if (off32) *off32 = b;
  if (offtc) *offtc = c;
  if (offb) *offb = e;
  return o;
}

int dict_prepare(const void* atoms, int in128, int64_t d, int s, void* storage, DictView* view,
                 cudaStream_t st) {
  if (d <= 0 || s <= 0) return kErrArgument;
  size_t o64, o32, otc, ob;
  const size_t total = dict_bytes(d, s, &o64, &o32, &otc, &ob);
  uint8_t* base = static_cast<uint8_t*>(storage);
  CBB_CUDA_TRY(cudaMemsetAsync(base, 0, total, st));
  DictView v{};
  v.d = d;
  v.s = s;
  v.s_pad = s_pad_for(s) > 0 ? s_pad_for(s) : s;
  v.kpad = kpad_for(s);
  v.n_btiles = int((d + kTileRows - 1) / kTileRows);
  v.atoms64 = reinterpret_cast<double2*>(base + o64);
  v.atoms32 = reinterpret_cast<float*>(base + o32);
  v.atoms_tc = base + otc;
  v.bounds = reinterpret_cast<float*>(base + ob);
  const int threads = 256;
  const int blocks = int((d + threads - 1) / threads);
  prep_dict_kernel<<<blocks, threads, 0, st>>>(atoms, in128, d, s, v.s_pad, v.kpad,
                                                const_cast<double2*>(v.atoms64),
                                                const_cast<float*>(v.atoms32),
                                                const_cast<uint8_t*>(v.atoms_tc),
                                                const_cast<float*>(v.bounds));
  CBB_CUDA_TRY(cudaGetLastError());
  *view = v;
  return kOk;
}

// Workspace carve-up for one projection call.
struct ProjWs {
  uint8_t* ztiles;
  float* win_tc;
  float* win32;
  int* ovf_count;
  int64_t* ovf_list;
  double* nd_v;
  double* partial;
};
constexpr int kReduceBlocks = 256;
constexpr int kVoxPad = 512;  // voxel tiles are padded to a multiple of the largest TC voxel tile

size_t project_ws_bytes(int64_t n, int s, ProjWs* ws, void* base_ptr) {
  const int kp = kpad_for(s);
  const int64_t n_vt = (n + kVoxPad - 1) / kVoxPad;
  size_t o = 0;
  uint8_t* base = static_cast<uint8_t*>(base_ptr);
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) & ~size_t(255);
    return base ? base + r : nullptr;
  };
  ProjWs w{};
  w.ztiles = take(size_t(n_vt) * kVoxPad * kp * 2);
  w.win_tc = reinterpret_cast<float*>(take(size_t(n_vt) * kVoxPad * 4));
  w.win32 = reinterpret_cast<float*>(take(size_t(n_vt) * kVoxPad * 4));
  w.ovf_count = reinterpret_cast<int*>(take(16));
  w.ovf_list = reinterpret_cast<int64_t*>(take(size_t(n) * 8));
  w.nd_v = reinterpret_cast<double*>(take(size_t(n) * 8));
  w.partial = reinterpret_cast<double*>(take(kReduceBlocks * 8));
  if (ws) *ws = w;
  return o;
}

static int g_num_sms = 0;
static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <int KP, int SUBS, int BN, int SPLIT>
static int launch_tc(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                     const ProjOut& out, int max_ctas, cudaStream_t st) {
  using C = TcCfg<KP, SUBS, BN, SPLIT>;
  static bool attr_set = false;
  if (!attr_set) {
    CBB_CUDA_TRY(cudaFuncSetAttribute(mf_tc_kernel<KP, SUBS, BN, SPLIT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  const int n_vt = int((n + C::kVox - 1) / C::kVox);
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (grid > n_vt) grid = n_vt;
  static int epi_mode = -1;
  if (epi_mode < 0) {
    const char* e = getenv("CBB_TC_EPI_MODE");  // development experiments only
    epi_mode = e ? atoi(e) : 0;
  }
  mf_tc_kernel<KP, SUBS, BN, SPLIT><<<grid, C::kThreads, C::kSmem, st>>>(
      w.ztiles, n, n_vt, w.win_tc, zs, dv, out, w.ovf_count, w.ovf_list, epi_mode);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

static int launch_tc32(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                       const ProjOut& out, int max_ctas, cudaStream_t st) {
  static int cfg = -1;
  if (cfg < 0) {
    const char* e = getenv("CBB_TC_CFG");  // development sweep only
    cfg = e ? atoi(e) : 0;
  }
  switch (cfg) {
    case 1: return launch_tc<32, 2, 128, 1>(w, n, zs, dv, out, max_ctas, st);
    case 2: return launch_tc<32, 1, 256, 2>(w, n, zs, dv, out, max_ctas, st);
    default: return launch_tc<32, 2, 128, 2>(w, n, zs, dv, out, max_ctas, st);
  }
}

template <int S>
static int launch_ffma(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                       const ProjOut& out, cudaStream_t st) {
  const int blocks = int((n + 127) / 128);
  mf_ffma_kernel<S><<<blocks, 128, 0, st>>>(zs, dv, n, w.win32, out, w.ovf_count, w.ovf_list);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

static int dispatch_ffma(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                         const ProjOut& out, cudaStream_t st) {
  switch (dv.s_pad) {
    case 2: return launch_ffma<2>(w, n, zs, dv, out, st);
    case 4: return launch_ffma<4>(w, n, zs, dv, out, st);
    case 6: return launch_ffma<6>(w, n, zs, dv, out, st);
    case 8: return launch_ffma<8>(w, n, zs, dv, out, st);
    case 10: return launch_ffma<10>(w, n, zs, dv, out, st);
    case 12: return launch_ffma<12>(w, n, zs, dv, out, st);
    case 16: return launch_ffma<16>(w, n, zs, dv, out, st);
    case 20: return launch_ffma<20>(w, n, zs, dv, out, st);
    case 24: return launch_ffma<24>(w, n, zs, dv, out, st);
    case 32: return launch_ffma<32>(w, n, zs, dv, out, st);
  }
  return kErrUnsupported;
}

static int launch_exhaustive(int64_t n, const ZSource& zs, const DictView& dv, const int* cnt,
                             const int64_t* list, const ProjOut& out, cudaStream_t st) {
  const size_t shm = size_t(8) * 2 * dv.s * sizeof(double);
  if (shm > 48 * 1024) {
    CBB_CUDA_TRY(cudaFuncSetAttribute(exhaustive_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
  }
  int grid = num_sms() * 4;
  if (!list) {
    int64_t need = (n + 7) / 8;
    if (need < grid) grid = int(need > 0 ? need : 1);
  }
  exhaustive_kernel<<<grid, 256, shm, st>>>(zs, dv, n, cnt, list, out);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

int reduce_sum(const double* x, int64_t n, double* partial, double* out, cudaStream_t st) {
  reduce_stage1<<<kReduceBlocks, 256, 0, st>>>(x, n, partial);
  reduce_stage2<<<1, 256, 0, st>>>(partial, kReduceBlocks, out);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// algo: 0 = auto (tcgen05 when 2s <= 64), 1 = tcgen05, 2 = FFMA, 3 = exhaustive fp64
int project(const ZSource& zs, int64_t n, const DictView& dv, const ProjOut& out, double* nd_sum,
            void* ws_ptr, size_t ws_bytes, int algo, int max_ctas, cudaStream_t st) {
  if (n < 0) return kErrArgument;
  ProjWs w;
  const size_t need = project_ws_bytes(n, dv.s, &w, ws_ptr);
  if (ws_bytes < need) return kErrArgument;
  if (n == 0) {
    if (nd_sum) CBB_CUDA_TRY(cudaMemsetAsync(nd_sum, 0, sizeof(double), st));
    return kOk;
  }
  ProjOut o = out;
  if (nd_sum && !o.nd_v) o.nd_v = w.nd_v;
  // tcgen05 path: K = 2s <= 64, and chunk entries pack (atom / 32) into 20 bits
  const bool tc_ok = (2 * dv.s <= 64) && (dv.d <= (int64_t(1) << 25));
  if (algo == 0) algo = tc_ok ? 1 : 3;
  if (algo == 1 && !tc_ok) return kErrUnsupported;
  if (algo == 2 && s_pad_for(dv.s) < 0) return kErrUnsupported;
  CBB_CUDA_TRY(cudaMemsetAsync(w.ovf_count, 0, sizeof(int), st));
  const bool dbg5 = getenv("CBB_TC_EPI_MODE") && atoi(getenv("CBB_TC_EPI_MODE")) == 5;
  if (dbg5) CBB_CUDA_TRY(cudaMemsetAsync(w.ovf_list, 0, 3 * sizeof(int64_t), st));
  if (algo == 1 || algo == 2) {
    const int64_t n_pad = ((n + kVoxPad - 1) / kVoxPad) * kVoxPad;
    const int threads = 256;
    prologue_kernel<<<int((n_pad + threads - 1) / threads), threads, 0, st>>>(
        zs, n, n_pad, dv.s, dv.kpad, dv.bounds, algo == 1 ? w.ztiles : nullptr, w.win_tc, w.win32,
        dv.s_pad);
    CBB_CUDA_TRY(cudaGetLastError());
    ZSource zr = zs;  // IPG mode: later kernels read Z from z_out
    int rc = (algo == 1) ? (dv.kpad == 32 ? launch_tc32(w, n, zr, dv, o, max_ctas, st)
                                          : launch_tc<64, 2, 128, 2>(w, n, zr, dv, o, max_ctas, st))
                         : dispatch_ffma(w, n, zr, dv, o, st);
    if (rc) return rc;
    if (dbg5) {
      unsigned long long h[3];
      cudaMemcpyAsync(h, w.ovf_list, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      fprintf(stderr, "[dbg] slow warp-chunks=%llu surviving chunks=%llu\n", h[1], h[2]);
    }
    if (!getenv("CBB_TC_EPI_MODE") || atoi(getenv("CBB_TC_EPI_MODE")) == 0 ||
        atoi(getenv("CBB_TC_EPI_MODE")) >= 5 || algo != 1) {
      rc = launch_exhaustive(n, zr, dv, w.ovf_count, w.ovf_list, o, st);
      if (rc) return rc;
    }
  } else if (algo == 3) {
    if (zs.x != nullptr) {
      // materialise Z = X - mu G (same fp32 rounding as the prologue)
      const int64_t n_pad = n;
      prologue_kernel<<<int((n_pad + 255) / 256), 256, 0, st>>>(zs, n, n_pad, dv.s, dv.kpad,
                                                               dv.bounds, nullptr, nullptr,
                                                               nullptr, dv.s_pad);
      CBB_CUDA_TRY(cudaGetLastError());
    }
    int rc = launch_exhaustive(n, zs, dv, nullptr, nullptr, o, st);
    if (rc) return rc;
  } else {
    return kErrArgument;
  }
  if (nd_sum) return reduce_sum(o.nd_v, n, w.partial, nd_sum, st);
  return kOk;
}

int project_overflow_count(void* ws_ptr, int64_t n, int s, int* host_count, cudaStream_t st) {
  ProjWs w;
  project_ws_bytes(n, s, &w, ws_ptr);
  CBB_CUDA_TRY(cudaMemcpyAsync(host_count, w.ovf_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBB_CUDA_TRY(cudaStreamSynchronize(st));
  return kOk;
}

int tc_debug_scores(const void* ztiles, const void* atiles, int kpad, int a_tile, int b_tile,
                    float* out, cudaStream_t st) {
  const int tile_bytes = kTileRows * kpad * 2;
  const int smem = 2 * tile_bytes + 64 + 1024;
  if (kpad == 32) {
    CBB_CUDA_TRY(cudaFuncSetAttribute(tc_debug_scores_kernel<32>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_debug_scores_kernel<32><<<1, 128, smem, st>>>(static_cast<const uint8_t*>(ztiles),
                                                      static_cast<const uint8_t*>(atiles), a_tile,
                                                      b_tile, out);
  } else {
    CBB_CUDA_TRY(cudaFuncSetAttribute(tc_debug_scores_kernel<64>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_debug_scores_kernel<64><<<1, 128, smem, st>>>(static_cast<const uint8_t*>(ztiles),
                                                      static_cast<const uint8_t*>(atiles), a_tile,
                                                      b_tile, out);
  }
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

int prologue_only(const ZSource& zs, int64_t n, const DictView& dv, void* ws_ptr,
                  cudaStream_t st) {
  ProjWs w;
  project_ws_bytes(n, dv.s, &w, ws_ptr);
  const int64_t n_pad = ((n + kVoxPad - 1) / kVoxPad) * kVoxPad;
  prologue_kernel<<<int((n_pad + 255) / 256), 256, 0, st>>>(zs, n, n_pad, dv.s, dv.kpad,
                                                             dv.bounds, w.ztiles, w.win_tc,
                                                             w.win32, dv.s_pad);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

}  // namespace cbb

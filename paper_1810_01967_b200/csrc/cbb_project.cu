// Exact cone projection on B200 (sm_100a).  See cbb_project.cuh for the scheme.
//
// Kernels
//   prep_dict_kernel     dictionary -> fp64 copy, planar fp32 copy, max ||d||, fp32 bounds
//   prep_tc_kernel       dictionary -> scaled fp16 UMMA tiles + their bounds
//   prologue_kernel      Z (or X - mu G) -> scaled fp16 voxel rows + certified windows
//   mf_tc_kernel<KP>     tcgen05 fp16 screening (fp16 accumulators), persistent + warp
//                          specialised: warp 0 bulk-copy producer, warps 1..3 MMA issuers,
//                          12 epilogue warps in 3 parts (TMEM -> packed regs, running max +
//                          certified candidates, fp64 rescoring and write-back of the winner)
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
// Re<z, d_j> in fp64 with z staged as planar (zr, zi); the same fma order as every other
// exact-score path.  S > 0: fully unrolled, predicated on k < s (all 2s loads in flight);
// S == 0: runtime loop (s > 32).
template <int S>
__device__ __forceinline__ double dot_atom(const double* zr, const double* zi,
                                           const double2* __restrict__ a, int s) {
  double acc = 0.0;
  if constexpr (S > 0) {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      if (k < s) {
        const double2 ak = a[k];
        acc = fma(zr[k], ak.x, acc);
        acc = fma(zi[k], ak.y, acc);
      }
    }
  } else {
    for (int k = 0; k < s; ++k) {
      const double2 ak = a[k];
      acc = fma(zr[k], ak.x, acc);
      acc = fma(zi[k], ak.y, acc);
    }
  }
  return acc;
}

// Re<z, d_j> in fp32 from the planar fp32 atom copy ([re_0..re_{sp-1}, im_0..im_{sp-1}]); the
// FFMA window win32 certifies it (any summation order).
template <int S>
__device__ __forceinline__ float dot_atom32(const float* zr, const float* zi,
                                           const float* __restrict__ a, int s, int sp) {
  float acc = 0.f;
  if constexpr (S > 0 && S % 4 == 0) {
    // 16-byte loads of the planar row (sp == S, rows 16-byte aligned); padding lanes are zero
    const float4* a4 = reinterpret_cast<const float4*>(a);
#pragma unroll
    for (int q = 0; q < S / 4; ++q) {
      const float4 re = a4[q], im = a4[S / 4 + q];
      acc = fmaf(zr[4 * q], re.x, fmaf(zi[4 * q], im.x, acc));
      acc = fmaf(zr[4 * q + 1], re.y, fmaf(zi[4 * q + 1], im.y, acc));
      acc = fmaf(zr[4 * q + 2], re.z, fmaf(zi[4 * q + 2], im.z, acc));
      acc = fmaf(zr[4 * q + 3], re.w, fmaf(zi[4 * q + 3], im.w, acc));
    }
  } else if constexpr (S > 0) {
#pragma unroll
    for (int k = 0; k < S; ++k)
      if (k < s) acc = fmaf(zr[k], a[k], fmaf(zi[k], a[sp + k], acc));
  } else {
    for (int k = 0; k < s; ++k) acc = fmaf(zr[k], a[k], fmaf(zi[k], a[sp + k], acc));
  }
  return acc;
}

__device__ void write_winner(const ProjOut& out, const DictView& dv, int64_t v, int64_t j,
                             double score) {
  const int s = dv.s;
  const double gamma = score > 0.0 ? score : 0.0;
  if (out.idx) {
    if (out.idx64) reinterpret_cast<int64_t*>(out.idx)[v] = j + out.idx_offset;
    else reinterpret_cast<int32_t*>(out.idx)[v] = int32_t(j + out.idx_offset);
  }
  if (out.gamma) out.gamma[v] = gamma;
  if (out.score) out.score[v] = score;
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

// tcgen05 screen candidate list: a kCandCap-entry shared-memory list (fast, enough for
// incoherent dictionaries) that spills to a kGCap-entry list in GLOBAL memory (L2-resident)
// when compaction cannot make room -- coherent dictionaries (fine MRF grids) put up to a few
// hundred chunks inside the fp16 window.  Global entry c sits at gbase[c * gstride] as
// (packed chunk, approximate chunk max bits).  Stale entries are dropped lazily.
constexpr int kGCap = 128;

__device__ __noinline__ int gcand_compact(int2* base, int64_t stride, int cnt, float thr) {
  int k = 0;
  for (int c = 0; c < cnt; ++c) {
    const int2 e = base[c * stride];
    if (__int_as_float(e.y) >= thr) base[(k++) * stride] = e;
  }
  return k;
}

// Move the live shared entries of one list to its global list (compacting that first if
// needed).  Plain values in and out (no struct by reference): the caller's list state stays in
// registers.  Returns the new global count, or -1 on overflow.
__device__ __noinline__ int hcand_spill(const int* cj, const float* cs, int stride, int cnt,
                                        int2* gbase, int64_t gstride, int gcnt, float thr) {
  int live = 0;
  for (int c = 0; c < cnt; ++c) live += cs[c * stride] >= thr;
  if (gcnt + live > kGCap) gcnt = gcand_compact(gbase, gstride, gcnt, thr);
  if (gcnt + live > kGCap) return -1;
  for (int c = 0; c < cnt; ++c)
    if (cs[c * stride] >= thr)
      gbase[(gcnt++) * gstride] = make_int2(cj[c * stride], __float_as_int(cs[c * stride]));
  return gcnt;
}

struct HCandList {
  int* cj;           // shared-memory list, column layout [kCandCap][stride]
  float* cs;
  int stride;
  int cnt;
  int2* gbase;       // global spill list
  int64_t gstride;
  int gcnt;
  bool ovf;

  __device__ __forceinline__ void insert(int j, float sc, float thr) {
    if (cnt == kCandCap) {
      cnt = cand_compact(cj, cs, stride, thr);
      if (cnt == kCandCap) {
        const int g = hcand_spill(cj, cs, stride, cnt, gbase, gstride, gcnt, thr);
        if (g < 0) {
          ovf = true;
          return;
        }
        gcnt = g;
        cnt = 0;
      }
    }
    cs[cnt * stride] = sc;
    cj[cnt * stride] = j;
    ++cnt;
  }

  // hand-off: append the surviving shared entries to the global list; returns the total or
  // -1 on overflow
  __device__ __forceinline__ int finish(float thr) {
    if (ovf) return -1;
    for (int c = 0; c < cnt; ++c) {
      const float x = cs[c * stride];
      if (x >= thr) {
        if (gcnt == kGCap) gcnt = gcand_compact(gbase, gstride, gcnt, thr);
        if (gcnt == kGCap) return -1;
        gbase[(gcnt++) * gstride] = make_int2(cj[c * stride], __float_as_int(x));
      }
    }
    return gcnt;
  }
};

// Rescore in fp64 one candidate atom; ties keep the lowest index (np.argmax, projection.py:62).
__device__ __forceinline__ void rescore_one(const ZSource& zs, const DictView& dv, int64_t v,
                                            int64_t j, int64_t& best, double& bs) {
  const double sc = exact_score_g(zs, v, dv.s, dv.atoms64 + j * dv.s);
  if (sc > bs || (sc == bs && j < best)) {
    bs = sc;
    best = j;
  }
}

// Chunk entries of the tcgen05 screen: (first atom / 32) in bits [0,20) and a 6-bit mask of
// the groups (bit g < 5 -> atoms 6g..6g+5, bit 5 -> atoms 30, 31) whose approximate scores
// reached the window when the chunk was recorded.
constexpr int kChunkShift = 20;
__device__ __forceinline__ int pack_chunk(int64_t jb, uint32_t mask) {
  return int(uint32_t(jb >> 5) | (mask << kChunkShift));
}

// FFMA screen entries (one atom each) that survive the final window.
__device__ __forceinline__ void rescore_entries(const ZSource& zs, const DictView& dv, int64_t v,
                                                const int* cj, const float* cs, int stride,
                                                int cnt, float thr, int64_t& best, double& bs) {
  for (int c = 0; c < cnt; ++c)
    if (cs[c * stride] >= thr) rescore_one(zs, dv, v, cj[c * stride], best, bs);
}

// Rescore the certified candidates in fp64 and write the winner; zero voxels go
// straight to index 0 (np.argmax of an all-zero row); overflow -> exhaustive list.
__device__ void finalize_voxel(const ZSource& zs, const DictView& dv, const ProjOut& out,
                               int64_t v, float win, float runmax, const CandList& cl,
                               int* ovf_count, int64_t* ovf_list) {
  if (win < 0.f) {
    write_winner(out, dv, v, 0, 0.0);
    return;
  }
  int64_t best = -1;
  double bs = -INFINITY;
  if (!cl.ovf)
    rescore_entries(zs, dv, v, cl.cj, cl.cs, cl.stride, cl.cnt, runmax - win, best, bs);
  if (best < 0) {
    int slot = atomicAdd(ovf_count, 1);
    ovf_list[slot] = v;
    return;
  }
  write_winner(out, dv, v, best, bs);
}

// ============================================================== dictionary preparation
// Pass 1: fp64 / fp32 copies, max ||d|| and the fp32 bounds.
__global__ void prep_dict_kernel(const void* __restrict__ atoms_in, int in128, int64_t d, int s,
                                 int s_pad, double2* __restrict__ atoms64,
                                 float* __restrict__ atoms32, float* __restrict__ bounds) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double nrm = 0, del32 = 0, nrm32 = 0;
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
    nrm += re * re + im * im;
    nrm32 += double(re32) * re32 + double(im32) * im32;
    del32 += (re - re32) * (re - re32) + (im - im32) * (im - im32);
  }
  for (int k = s; k < s_pad; ++k) {
    atoms32[j * 2 * s_pad + k] = 0.f;
    atoms32[j * 2 * s_pad + s_pad + k] = 0.f;
  }
  atomic_max_nonneg(bounds + kBDmax, __double2float_ru(sqrt(nrm)));
  atomic_max_nonneg(bounds + kBDelta32, __double2float_ru(sqrt(del32)));
  atomic_max_nonneg(bounds + kBD32Max, __double2float_ru(sqrt(nrm32)));
}

// Power-of-two scale putting max||scale * d|| in [0.5, 1) (1 for an all-zero dictionary).
__device__ __forceinline__ double dict_scale(const float* bounds) {
  const double dmax = bounds[kBDmax];
  if (!(dmax > 0.0) || !isfinite(dmax)) return 1.0;
  int e;
  frexp(dmax, &e);
  return ldexp(1.0, -e);
}

// Pass 2: fp16 UMMA rows of scale_d * d in the no-swizzle core-matrix layout (atom_chunk_offset,
// tc_nc(s) chunks per row) and their bounds.  2s <= 64 only (tensor-core path).
__global__ void prep_tc_kernel(const double2* __restrict__ atoms64, int64_t d, int64_t d_pad,
                               int s, uint8_t* __restrict__ atoms_tc,
                               float* __restrict__ bounds) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= d_pad) return;
  const int nc = tc_nc(s);
  auto elem = [&](int e) {
    return reinterpret_cast<unsigned short*>(atoms_tc + atom_chunk_offset(j, e >> 3, nc) +
                                             (e & 7) * 2);
  };
  const int e_sent = 2 * s;  // sentinel right after the data: nq = ceil((2s+1)/16) K-steps
  if (j >= d) {  // zero-padded row of the last tile: sentinel score -65504 for every voxel
    *elem(e_sent) = kF16MinusMax;
    return;
  }
  const double sc = dict_scale(bounds);
  if (j == 0) bounds[kBScaleD] = float(sc);
  double del = 0, nrm_h = 0;
  for (int k = 0; k < s; ++k) {
    const double2 a = atoms64[j * s + k];
    const double re = a.x * sc, im = a.y * sc;
    const unsigned short hre = f16_bits_rn(re), him = f16_bits_rn(im);
    const double fre = f16_bits_to_double(hre), fim = f16_bits_to_double(him);
    *elem(k) = hre;
    *elem(s + k) = him;
    nrm_h += fre * fre + fim * fim;
    del += (re - fre) * (re - fre) + (im - fim) * (im - fim);
  }
  atomic_max_nonneg(bounds + kBDeltaH, __double2float_ru(sqrt(del)));
  atomic_max_nonneg(bounds + kBDhMax, __double2float_ru(sqrt(nrm_h)));
}

// Split-operand tiles (s <= kSplitMaxS): row j = [d_hi (2s) | d_hi (2s) | d_lo (2s) | sentinel],
// d_hi = fp16(scale_d d), d_lo = fp16(scale_d d - d_hi), K = split_kp(s), 128-byte swizzle,
// split_rows(K)-row tiles (split_elem_offset).  Padded rows carry -65504 in the sentinel column
// (their fp32-accumulated score is -65504 for every voxel).
__global__ void prep_tc2_kernel(const double2* __restrict__ atoms64, int64_t d, int64_t d_pad,
                                int s, uint8_t* __restrict__ atoms_tc2,
                                float* __restrict__ bounds) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= d_pad) return;
  const int kp = split_kp(s), rows = split_rows(kp);
  const int tile = int(j / rows), r = int(j % rows);
  uint8_t* trow = atoms_tc2 + size_t(tile) * rows * kp * 2;
  auto put = [&](int e, unsigned short h) {
    *reinterpret_cast<unsigned short*>(trow + split_elem_offset(r, e, rows)) = h;
  };
  if (j >= d) {
    put(6 * s, kF16MinusMax);
    return;
  }
  const double sc = dict_scale(bounds);
  double del = 0, nlo = 0, nhi = 0;
  for (int k = 0; k < s; ++k) {
    const double2 a = atoms64[j * s + k];
    const double x[2] = {a.x * sc, a.y * sc};
    for (int c = 0; c < 2; ++c) {
      const unsigned short hi = f16_bits_rn(x[c]);
      const double fhi = f16_bits_to_double(hi);
      const unsigned short lo = f16_bits_rn(x[c] - fhi);
      const double flo = f16_bits_to_double(lo);
      const int e = c * s + k;  // re parts [0, s), im parts [s, 2s)
      put(e, hi);
      put(2 * s + e, hi);
      put(4 * s + e, lo);
      const double rem = x[c] - fhi - flo;
      del += rem * rem;
      nlo += flo * flo;
      nhi += fhi * fhi;
    }
  }
  atomic_max_nonneg(bounds + kBDeltaS, __double2float_ru(sqrt(del)));
  atomic_max_nonneg(bounds + kBDloMax, __double2float_ru(sqrt(nlo)));
  atomic_max_nonneg(bounds + kBRowMax, __double2float_ru(sqrt(2.0 * nhi + nlo) * (1.0 + 1e-12)));
}

// Coherence estimate (selects the screen in auto mode): for kCohSamples evenly spaced atoms i,
// count the other atoms j with Re<d_i, d_j> >= (1 - 2^-6) ||d_i|| ||d_j|| (fp32 from the planar
// copy).  Atoms that close score within the fp16 screen's window of each other for voxels with
// cosine >= ~1/2 to their best atom, so every such neighbour becomes a candidate to rescore;
// the split screen's window is ~2^-16 wide.  One block per sampled atom.
constexpr int kCohSamples = 256;
__global__ void __launch_bounds__(256) coherence_kernel(const float* __restrict__ atoms32,
                                                        int64_t d, int s, int sp,
                                                        float* __restrict__ bounds) {
  __shared__ float ai[64];
  __shared__ int red[8];
  const int64_t i = (int64_t(blockIdx.x) * d) / gridDim.x;
  for (int k = threadIdx.x; k < 2 * sp; k += blockDim.x) ai[k] = atoms32[i * 2 * sp + k];
  __syncthreads();
  float ni = 0.f;
  for (int k = 0; k < s; ++k) ni = fmaf(ai[k], ai[k], fmaf(ai[sp + k], ai[sp + k], ni));
  int cnt = 0;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    if (j == i) continue;
    const float* aj = atoms32 + j * 2 * sp;
    float dot = 0.f, nj = 0.f;
    for (int k = 0; k < s; ++k) {
      const float re = aj[k], im = aj[sp + k];
      dot = fmaf(ai[k], re, fmaf(ai[sp + k], im, dot));
      nj = fmaf(re, re, fmaf(im, im, nj));
    }
    cnt += (dot > 0.f && dot * dot >= (1.f - 0x1p-6f) * (1.f - 0x1p-6f) * ni * nj) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    atomicAdd(bounds + kBCoherence, float(t) / float(gridDim.x));
  }
}

// ============================================================== prologue
// One thread per voxel (n_pad = whole voxel tiles).  Produces the fp16 tensor-core voxel rows
// z~ = fp16(scale_v z) (scale_v a power of two putting ||scale_v z|| in [2^12, 2^13), so with
// max||d~|| <= 1 every fp16 partial sum stays far below 65504) and both certified windows.
// In the scaled units of the tensor-core scores (scale_v * scale_d * Re<z, d>):
//   |s~ - s| <= ||scale_v z - z~|| * scale_d max||d|| + ||z~|| * max||scale_d d - d~||
//              + acc * ||z~|| * max||d~||
// where acc covers the fp16 accumulator: one round-to-nearest per K = 16 instruction of a
// value bounded by sum|products| (<= ||z~|| ||d~||), i.e. (KP/16) * 2^-11, plus slack for
// internal alignment and fp16 subnormals.  window = 2 * bound: the true argmax j* satisfies
// s~_j* >= max s~ - window.  The FFMA window (win32) is in unscaled fp32 units.
__global__ void prologue_kernel(ZSource zs, int64_t n, int64_t n_pad, int s, int kpad,
                                const float* __restrict__ bounds, uint8_t* __restrict__ ztiles,
                                float* __restrict__ win_tc, float* __restrict__ win32,
                                int s_pad, const double2* __restrict__ atoms64,
                                int64_t d_atoms, float* __restrict__ init_tc, int split) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n_pad) return;
  // plain row-major fp16 rows (kpad elements): staged into TMEM lanes by the epilogue warps
  uint8_t* trow = ztiles ? ztiles + size_t(v) * kpad * 2 : nullptr;
  if (v >= n) {
    if (trow)
      for (int c = 0; c < kpad / 8; ++c)
        *reinterpret_cast<uint4*>(trow + c * 16) = make_uint4(0, 0, 0, 0);
    return;
  }
  // pass 1: Z (IPG: X - mu G, written to z_out) and its largest component magnitude
  double amax = 0;
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
    amax = fmax(amax, fmax(fabs(re), fabs(im)));
    if (re != re || im != im) amax = re + im;  // propagate NaN
  }
  const double dmax = bounds[kBDmax];
  const double d32 = bounds[kBD32Max], del32 = bounds[kBDelta32];
  if (amax == 0.0) {  // all-zero row (decided on the components: |z|^2 may underflow)
    if (win_tc) win_tc[v] = -1.f;
    if (win32) win32[v] = -1.f;
    if (trow)
      for (int c = 0; c < kpad / 8; ++c)
        *reinterpret_cast<uint4*>(trow + c * 16) = make_uint4(0, 0, 0, 0);
    return;
  }
  int ea = 0;
  if (isfinite(amax)) frexp(amax, &ea);
  if (!isfinite(amax) || ea < -80 || ea > 80) {
    // inf / NaN voxel, or one whose squares / fp32 copy would under- or overflow: no
    // screening, the exhaustive fp64 scan decides (NaN windows route it there)
    if (win_tc) win_tc[v] = __int_as_float(0x7fc00000);
    if (win32) win32[v] = __int_as_float(0x7fc00000);
    if (trow)
      for (int c = 0; c < kpad / 8; ++c)
        *reinterpret_cast<uint4*>(trow + c * 16) = make_uint4(0, 0, 0, 0);
    return;
  }
  // pass 2: norms and the fp32 rounding error (no under- / overflow for |z| in 2^[-80, 80])
  double nz = 0, ez32 = 0, nz32 = 0;
  for (int k = 0; k < s; ++k) {
    const double2 z = load_z(zs, v, s, k);
    const double re = z.x, im = z.y;
    const float re32 = float(re), im32 = float(im);
    nz += re * re + im * im;
    ez32 += (re - re32) * (re - re32) + (im - im32) * (im - im32);
    nz32 += double(re32) * re32 + double(im32) * im32;
  }
  const double acc32 = double(2 * s_pad + 4) * 0x1p-24;
  const double e3 = sqrt(ez32) * dmax + sqrt(nz32) * del32 + acc32 * sqrt(nz32) * d32;
  if (win32) win32[v] = __double2float_ru(2.0 * e3 * 1.001 + 1e-30);
  if (!trow) return;
  int ez;
  frexp(sqrt(nz), &ez);
  const double sv = ldexp(1.0, 13 - ez);
  unsigned short row[128];
#pragma unroll
  for (int e = 0; e < 128; ++e) row[e] = 0;
  double eh = 0, nzh = 0, nlo = 0, nhi = 0;
  for (int k = 0; k < s; ++k) {
    double re, im;
    if (zs.x != nullptr) {
      const float2 xk = zs.x[v * s + k], gk = zs.g[v * s + k];
      re = __fmaf_rn(-zs.mu, gk.x, xk.x);
      im = __fmaf_rn(-zs.mu, gk.y, xk.y);
    } else if (zs.z128) {
      double2 a = reinterpret_cast<const double2*>(zs.z)[v * s + k];
      re = a.x; im = a.y;
    } else {
      float2 a = reinterpret_cast<const float2*>(zs.z)[v * s + k];
      re = a.x; im = a.y;
    }
    const double x[2] = {re * sv, im * sv};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const unsigned short hi = f16_bits_rn(x[c]);
      const double fhi = f16_bits_to_double(hi);
      const int e = c * s + k;
      row[e] = hi;
      if (split == 1) {  // [z_hi | z_lo | z_hi]: z~ = z_hi + z_lo
        const unsigned short lo = f16_bits_rn(x[c] - fhi);
        const double flo = f16_bits_to_double(lo);
        row[2 * s + e] = lo;
        row[4 * s + e] = hi;
        const double rem = x[c] - fhi - flo;
        eh += rem * rem;
        nzh += (fhi + flo) * (fhi + flo);
        nlo += flo * flo;
        nhi += fhi * fhi;
      } else {
        eh += (x[c] - fhi) * (x[c] - fhi);
        nzh += fhi * fhi;
      }
    }
  }
  row[split == 1 ? 6 * s : 2 * s] = kF16One;  // sentinel column right after the data (< kpad)
  for (int c = 0; c < kpad / 8; ++c) {
    uint4 pk;
    pk.x = uint32_t(row[c * 8 + 0]) | (uint32_t(row[c * 8 + 1]) << 16);
    pk.y = uint32_t(row[c * 8 + 2]) | (uint32_t(row[c * 8 + 3]) << 16);
    pk.z = uint32_t(row[c * 8 + 4]) | (uint32_t(row[c * 8 + 5]) << 16);
    pk.w = uint32_t(row[c * 8 + 6]) | (uint32_t(row[c * 8 + 7]) << 16);
    *reinterpret_cast<uint4*>(trow + c * 16) = pk;
  }
  const double sd = bounds[kBScaleD];
  double eb;
  if (split == 1) {
    // s~ = z_hi.d_hi + z_lo.d_hi + z_hi.d_lo = z~.d~ - z_lo.d_lo (z~ = z_hi + z_lo, d~ likewise):
    //   |s~ - s| <= ||scale_v z - z~|| scale_d max||d|| + ||z~|| max||scale_d d - d~||
    //             + ||z_lo|| max||d_lo|| + acc * ||A_v|| max||B_j||
    // acc: per issued K = 16 fp32-accumulated instruction, < 16 truncations below 2^-24 of the
    // largest term plus one fp32 rounding, each <= 2^-24 sum|a_k b_k| <= 2^-24 ||A|| ||B||
    // (18 instead of 17 as slack), n_q = ceil((6s+1)/16) instructions.
    const double nq = double(split_ksteps(s));
    const double acc_tc = nq * 18.0 * 0x1p-24;
    eb = sqrt(eh) * sd * dmax + sqrt(nzh) * bounds[kBDeltaS] + sqrt(nlo) * bounds[kBDloMax] +
         acc_tc * sqrt(2.0 * nhi + nlo) * bounds[kBRowMax] + nq * 0x1p-40;
  } else {
    const double dh = bounds[kBDhMax], delh = bounds[kBDeltaH];
    const double nq = double(mma_ksteps(s));
    // fp16 accumulators: one fp16 rounding per issued instruction of a partial sum bounded by
    // sum|a_k b_k| <= ||z~|| max||d~||; HI32 (fp32 accumulators): the split screen's model,
    // < 16 truncations below 2^-24 of the largest term + one fp32 rounding per instruction
    const double acc_tc = split == 2 ? nq * 18.0 * 0x1p-24
                                     : nq * (0x1p-11 * (1.0 + 0x1p-9) + 0x1p-19);
    eb = sqrt(eh) * sd * dmax + sqrt(nzh) * delh + acc_tc * sqrt(nzh) * dh +
         nq * (split == 2 ? 0x1p-40 : 0x1p-24);
  }
  win_tc[v] = __double2float_ru(2.0 * eb * 1.001 + 1e-30);
  if (init_tc) {
    // warm start: any atom's exact score lower-bounds the approximate maximum once the
    // certified half-window is subtracted (s~_max >= s~_j >= s_j - eps), in scaled units
    float init = -INFINITY;
    const int64_t jh = zs.hint ? int64_t(zs.hint[v]) : -1;
    if (jh >= 0 && jh < d_atoms) {
      const double2* a = atoms64 + jh * s;
      double acc = 0.0;
      for (int k = 0; k < s; ++k) {
        const double2 z = load_z(zs, v, s, k);
        acc = fma(z.x, a[k].x, acc);
        acc = fma(z.y, a[k].y, acc);
      }
      init = __double2float_rd(acc * sv * sd - eb * 1.001);
    }
    init_tc[v] = init;
  }
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
template <int S>
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
      const double acc = dot_atom<S>(zw, zw + s, dv.atoms64 + j * s, s);
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

// Overflow-list mode of the exhaustive scan: each listed voxel's dictionary is split into
// kExhSplits atom ranges scanned by different warps (a short list still fills the GPU); the
// per-range (best score, lowest index) partials are merged by exhaustive_finish_kernel.
constexpr int kExhSplits = 16;

constexpr int kExhSurv = 8;  // per-lane fp32-window survivors in the split scan

template <int S>
__global__ void __launch_bounds__(256) exhaustive_split_kernel(ZSource zs, DictView dv,
                                                               const int* __restrict__ cnt,
                                                               const int64_t* __restrict__ list,
                                                               const float* __restrict__ win32,
                                                               double2* __restrict__ partial) {
  // per warp: z (2s doubles), z (2 sp floats, zero-padded), lane survivor lists
  extern __shared__ double zsh[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int s = dv.s, sp = dv.s_pad;
  double* zw = zsh + size_t(wid) * 2 * s;
  float* z32 = reinterpret_cast<float*>(zsh + size_t(8) * 2 * s) + size_t(wid) * 2 * sp;
  int2* surv = reinterpret_cast<int2*>(reinterpret_cast<float*>(zsh + size_t(8) * 2 * s) +
                                       size_t(8) * 2 * sp) +
               (size_t(wid) * 32 + lane) * kExhSurv;
  const int64_t total = int64_t(*cnt) * kExhSplits;
  const int64_t nw = int64_t(gridDim.x) * 8;
  const int64_t span = (dv.d + kExhSplits - 1) / kExhSplits;
  for (int64_t pr = int64_t(blockIdx.x) * 8 + wid; pr < total; pr += nw) {
    const int64_t i = pr / kExhSplits;
    const int k = int(pr - i * kExhSplits);
    const int64_t v = list[i];
    for (int c = lane; c < s; c += 32) {
      const double2 z = load_z(zs, v, s, c);
      zw[c] = z.x;
      zw[s + c] = z.y;
      z32[c] = float(z.x);
      z32[sp + c] = float(z.y);
    }
    for (int c = s + lane; c < sp; c += 32) {
      z32[c] = 0.f;
      z32[sp + c] = 0.f;
    }
    __syncwarp();
    const float w32 = win32[v];
    double bs = -INFINITY;
    int64_t best = INT64_MAX;
    const int64_t lo = int64_t(k) * span, hi = lo + span < dv.d ? lo + span : dv.d;
    // fp32 pre-filter (certified window w32) with per-lane survivors; a full list or a
    // non-finite voxel (w32 NaN) scans the slice in fp64 instead
    bool full = !(w32 >= 0.f);
    float lmax = -INFINITY;
    int ns = 0;
    if (!full) {
      for (int64_t j = lo + lane; j < hi; j += 32) {
        const float sc = dot_atom32<S>(z32, z32 + sp, dv.atoms32 + j * 2 * sp, s, sp);
        lmax = fmaxf(lmax, sc);
        if (sc >= lmax - w32) {
          if (ns == kExhSurv) {
            int k2 = 0;
            for (int c = 0; c < kExhSurv; ++c)
              if (__int_as_float(surv[c].y) >= lmax - w32) surv[k2++] = surv[c];
            ns = k2;
          }
          if (ns < kExhSurv) surv[ns++] = make_int2(int(j), __float_as_int(sc));
          else full = true;
        }
      }
    }
    float gmax32 = lmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmax32 = fmaxf(gmax32, __shfl_xor_sync(0xffffffffu, gmax32, o));
    if (__any_sync(0xffffffffu, full)) {
      for (int64_t j = lo + lane; j < hi; j += 32) {
        const double acc = dot_atom<S>(zw, zw + s, dv.atoms64 + j * s, s);
        if (acc > bs) { bs = acc; best = j; }
      }
    } else {
      const float thr32 = gmax32 - w32;
      for (int c = 0; c < ns; ++c) {
        const int2 e2 = surv[c];
        if (__int_as_float(e2.y) < thr32) continue;
        const int64_t j = e2.x;
        const double acc = dot_atom<S>(zw, zw + s, dv.atoms64 + j * s, s);
        if (acc > bs || (acc == bs && j < best)) { bs = acc; best = j; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double obs = __shfl_xor_sync(0xffffffffu, bs, o);
      const int64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
      if (obs > bs || (obs == bs && ob < best)) { bs = obs; best = ob; }
    }
    if (lane == 0) partial[pr] = make_double2(bs, __longlong_as_double(best));
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) exhaustive_finish_kernel(DictView dv,
                                                                const int* __restrict__ cnt,
                                                                const int64_t* __restrict__ list,
                                                                const double2* __restrict__ partial,
                                                                ProjOut out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= *cnt) return;
  double bs = -INFINITY;
  int64_t best = INT64_MAX;
  for (int k = 0; k < kExhSplits; ++k) {
    const double2 p = partial[i * kExhSplits + k];
    const int64_t j = __double_as_longlong(p.y);
    if (p.x > bs || (p.x == bs && j < best)) { bs = p.x; best = j; }
  }
  if (best == INT64_MAX) best = 0;  // all-NaN row: np.argmax returns the first NaN -> 0
  write_winner(out, dv, list[i], best, bs);
}

#ifdef CBB_TRACE
// development tracing: per-tile clock64 stamps of CTA 0 (issuer: after b_full wait, after
// commit; epilogue part warp q0: after t_full wait, after wait::ld)
constexpr int kTraceTiles = 2048;
__device__ long long g_trace[kTraceTiles * 8];
__device__ long long g_trace_vt[256 * 4];  // per voxel tile of CTA 0: loop start, finalize start/end
#define CBB_STAMP(slot, k)                                                          \
  do {                                                                              \
    if (blockIdx.x == 0 && (k) < uint32_t(kTraceTiles))                             \
      g_trace[(k) * 8 + (slot)] = clock64();                                        \
  } while (0)
#define CBB_STAMP_VT(slot, it)                                                      \
  do {                                                                              \
    if (blockIdx.x == 0 && (it) < 256) g_trace_vt[(it) * 4 + (slot)] = clock64();   \
  } while (0)
#else
#define CBB_STAMP(slot, k) \
  do {                     \
  } while (0)
#define CBB_STAMP_VT(slot, it) \
  do {                         \
  } while (0)
#endif

// ============================================================== tcgen05 screening
// One CTA per SM (persistent).  Per voxel tile (128 voxels):
//   * the voxel operand A (fp16, K = KP) lives in TENSOR MEMORY (double buffered): part-0
//     epilogue threads tcgen05.st their own voxel row into their TMEM lane one tile ahead;
//   * warp 0 streams atom tiles (BN = 96 rows = 8-row aligned windows of the pre-swizzled
//     fp16 128-row tiles) through a bulk-copy ring;
//   * tile k accumulates in TMEM stage k % kAcc (kAcc = 5 stages x 96 fp16 accumulator
//     columns + the 32-column A double buffer = all 512 columns); warps 1..kParts issue the
//     MMAs: issuer i owns the CTA's atom tiles k = i (mod kParts) and the B-ring stages
//     st = i (mod kParts); per tile it waits ONE barrier, b_full[st], whose phase completes
//     when the tile's bytes have landed AND the epilogue released the accumulator stage (the
//     epilogue arrives on the b_full of the tile that will reuse its stage), then issues KP/16
//     MMAs (M=128, N=96, K=16, A from TMEM, B from SMEM) and commits;
//   * epilogue part p (4 warps, one per TMEM lane quarter) consumes tiles k = p (mod kParts):
//     it copies the 96 packed scores per lane into registers and releases the stage at once.
//     With 5 stages rotating over 3 parts a stage's refill (release -> issuer -> MMA -> commit)
//     overlaps 5/3 screening iterations instead of one.
// Barrier phases: b_full[st] -> issuer st % kParts (kStages % kParts == 0) consumes its phases
// in order; an epilogue arrival for tile k + kAcc lands on b_full[(k + kAcc) % kStages] only
// after that barrier's previous phase (tile k + kAcc - kStages) completed (issued before tile
// k, whose stage is being released).  t_full[s] is waited by the parts of tiles s, s + kAcc,
// ... in turn, so their completions go to t_full[k % kTBars] (kTBars = kAcc * kParts): each
// of those barriers serves one stage and one part, which consumes its phases in order.
// b_empty -> producer, a_full -> issuers, a_empty -> part 0.
// Atom tiles are visited in a per-CTA rotated order to spread L2 traffic.
constexpr int kParts = 3;
// Small projections split the dictionary into up to kMaxSplit contiguous tile ranges (work units
// = voxel tile x range) so that all SMs get an even share; each range reports its own kParts
// candidate lists.  Only projections of at most kSplitMaxN voxels reserve the extra lists.
constexpr int kMaxSplit = 4;
constexpr int64_t kSplitMaxN = int64_t(1) << 17;
// 128-row storage tiles after the last atom: sentinel rows that complete the last BN-row tile
// of every range (up to kMaxSplit - 1 extra BN-row tiles)
constexpr int kPadTiles = 8;

// SPLIT: hi/lo fp16 operands with fp32 accumulators: KP = 64 -> 128-atom tiles (N = 128 MMAs;
// measured faster than 64-atom tiles with six stages), screened in two 64-register halves;
// KP = 128 -> 64-atom tiles (the 16 KB stages keep a 9-deep ring).
// PAIR: the CTAs of a cluster pair run cta_group::2 MMAs (M = 256: each CTA's 128 voxels); every
// CTA bulk-copies only its half of each atom tile (kBNloc rows), which halves the L2 -> SMEM
// atom stream that bounds the single-CTA kernel.
// HI32: the fp16 operand rows of the fp16 screen (2s + 1 columns) with FP32 accumulators: the
// screen issues the fp16 screen's K-steps but its window is the operand rounding only
// (~2^-10 |z| instead of ~2^-8): the split screen's fp32 epilogue on 128-atom tiles.
template <int KP, bool SPLIT = false, bool PAIR = false, bool HI32 = false>
struct TcCfg {
  static_assert(!SPLIT || KP == 64 || KP == 128, "split tiles are 64 or 128 wide");
  static_assert(!(SPLIT && HI32), "one operand format");
  static constexpr bool kF32 = SPLIT || HI32;  // fp32 accumulators, fp32 epilogue
  // 32-atom chunks per tile (split: the tile is one split_rows(KP)-row storage tile)
  static constexpr int kChunks = SPLIT ? split_rows(KP) / 32 : HI32 ? 4 : (KP == 32 ? 5 : 4);
  static constexpr int BN = 32 * kChunks;                    // 160 (KP 32) / 128 / 64 (split)
  static constexpr int kACols = KP / 2;                      // packed fp16 pairs per lane
  static constexpr int kAcc = 3;                             // x BN accumulator columns
  static constexpr int kAccCols = BN;
  static constexpr int kAColOff = kAcc * kAccCols;           // A buffers after the stages
  static_assert(kAColOff + 2 * kACols <= 512, "TMEM budget");
  static constexpr int kBNloc = PAIR ? BN / 2 : BN;          // atom rows in this CTA's SMEM
  static constexpr int kRowBytes = (KP < 64 ? KP : 64) * 2;   // bytes per row of a K block
  static constexpr int kBlk = KP <= 64 ? 1 : KP / 64;         // K blocks per tile
  // split tiles in global memory / this CTA's part (= the ring's stage stride); the fp16 screens
  // copy only tc_nc(s) 16-byte chunks per row (tile_bytes / copy_bytes in the kernel)
  static constexpr int kBTileBytes = BN * KP * 2;
  static constexpr int kBBytes = kBNloc * KP * 2;
  static_assert(kBNloc % 8 == 0, "8-row swizzle groups");
#ifdef CBB_RING_KB
  static constexpr int kRing = CBB_RING_KB * 1024;
#else
  static constexpr int kRing = (KP == 32 ? 96 : 144) * 1024;
#endif
  static constexpr int kStagesRaw = kRing / kBBytes > 24 ? 24 : kRing / kBBytes;
  static_assert(kBBytes % 1024 == 0, "stage buffers keep the 1024 B swizzle alignment");
  static constexpr int kStages = (kStagesRaw / kParts) * kParts;
  static_assert(kStages >= 2 * kAcc, "B ring too shallow");
  static constexpr int kEpiWarps = 4 * kParts;
  static constexpr int kFirstEpiWarp = 1 + kParts;          // warp 0 producer, 1..3 issuers
  static constexpr int kThreads = (kFirstEpiWarp + kEpiWarps) * 32;
  static constexpr int kVox = 128;
  static constexpr int kSlots = kVox * kParts;
  static constexpr int kOffB = 0;
  static constexpr int kOffCj = kOffB + kStages * kBBytes;
  static constexpr int kOffCs = kOffCj + kCandCap * kSlots * 4;
  static constexpr int kOffPthr = kOffCs + kCandCap * kSlots * 4;  // [kVox][4] u32 thresholds
  static constexpr int kOffBar = kOffPthr + kVox * 16;
  // completion barriers per tile slot k % kTBars (lcm(kAcc, kParts)): every barrier belongs to
  // one stage AND one part, whose waits consume its phases in order (no parity aliasing)
  static constexpr int kTBars = (kAcc % kParts == 0) ? kAcc : kAcc * kParts;
  // split screen on 128-atom tiles: each accumulator stage is two 64-column halves with their
  // own MMAs (N = 64), commits and releases, so the first half refills while the part loads the
  // second (the 64 fp32 scores of one half fill the part's registers)
  static constexpr bool kHalves = SPLIT && !PAIR && kChunks == 4;
  static constexpr int kNumBars = 4 + 2 * kStages + (kHalves ? 2 : 1) * (kTBars + kAcc);
  static_assert(kStages % kParts == 0, "barrier ownership");
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffTmem + 16 + 1024;  // + alignment slack
  static_assert(kSmem <= 227 * 1024, "shared memory");
  static constexpr int kM = PAIR ? 256 : 128;
  static constexpr uint32_t kIdesc = kF32 ? idesc_f16_f32(kM, BN) : idesc_f16_f16(kM, BN);
  static constexpr int kMinTiles = kParts;  // every part owns >= 1 tile per voxel tile
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

// Screen approximate scores of one voxel (one thread): running max + certified window.
// The fp16 accumulators arrive packed (register m = atoms 2m, 2m+1).  Fast path per
// tile: one 3-input packed max chain per 32-atom chunk (VHMNMX, ~9 instructions per chunk)
// + one compare + a warp vote.
// Only when some lane's max reaches its threshold (rare after the first tiles) the chunks are
// examined: a 32-atom chunk whose max enters the window is recorded (first atom, mask of
// 6-atom groups inside the window, chunk max) -- no per-value inserts; the finalize rescans
// only the flagged groups exactly.  Any atom inside the final window lies in a flagged group of
// a recorded chunk, so the certificate is unchanged.  Thresholds are rounded DOWN to fp16
// (never excludes an atom the exact window admits).
__device__ __forceinline__ __half2 as_h2(uint32_t x) {
  return *reinterpret_cast<const __half2*>(&x);
}
__device__ __forceinline__ __half2 hmax3(__half2 a, __half2 b, __half2 c) {
  return __hmax2(__hmax2(a, b), c);  // fused by ptxas into one VHMNMX
}
__device__ __forceinline__ __half hmax_halves(__half2 m) {
  return __hmax(__low2half(m), __high2half(m));
}

// Record 32-atom chunk (16 packed registers) with max cm: groups g < 5 -> registers
// 3g..3g+2 (atoms 6g..6g+5), g = 5 -> register 15 (atoms 30, 31).
__device__ __forceinline__ void record_chunk(const uint32_t* r, __half cm, int64_t jb, __half thr,
                                             float thr_f, HCandList& cl) {
  uint32_t mask = __hge(hmax_halves(as_h2(r[15])), thr) ? (1u << 5) : 0u;
#pragma unroll
  for (int i = 0; i < 5; ++i)
    mask |= __hge(hmax_halves(hmax3(as_h2(r[3 * i]), as_h2(r[3 * i + 1]), as_h2(r[3 * i + 2]))),
                  thr)
                ? (1u << i)
                : 0u;
  cl.insert(pack_chunk(jb, mask), __half2float(cm), thr_f);
}

template <int NC>
__device__ __forceinline__ void screen_tile(const uint32_t (&r)[16 * NC], int64_t jb, float win,
                                            __half& runmax, __half& thr, bool& active,
                                            HCandList& cl, uint32_t* pub, uint32_t tag) {
  // NC independent 3-input chains, one per 32-atom chunk (8 VHMNMX/HMNMX2 each)
  __half2 c[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const uint32_t* q = r + 16 * k;
    __half2 a = hmax3(as_h2(q[0]), as_h2(q[1]), as_h2(q[2]));
#pragma unroll
    for (int i = 3; i < 15; i += 2) a = hmax3(a, as_h2(q[i]), as_h2(q[i + 1]));
    c[k] = __hmax2(a, as_h2(q[15]));
  }
  __half2 m = c[0];
#pragma unroll
  for (int k = 1; k < NC; ++k) m = __hmax2(m, c[k]);
  const __half cm = hmax_halves(m);
  // warp-uniform test: the fast path carries no divergent branch / reconvergence
  if (__any_sync(0xffffffffu, __hge(cm, thr))) {
    if (__hge(cm, thr)) {
      runmax = __hmax(runmax, cm);
      if (active) {
        thr = __float2half_rd(__half2float(runmax) - win);
        *pub = tag | __half_as_ushort(thr);  // the other parts screen against it too
        const float thr_f = __half2float(thr);
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          const __half ck = hmax_halves(c[k]);
          if (__hge(ck, thr) && !cl.ovf) record_chunk(r + 16 * k, ck, jb + 32 * k, thr, thr_f, cl);
        }
        if (cl.ovf) {
          active = false;
          thr = __ushort_as_half(0x7C00);  // +inf
        }
      }
    }
  }
}

// Split mode: fp32 scores, one per register (chunk k = registers 32k .. 32k+31).  Same
// structure as the packed path: one 3-input max chain per 32-atom chunk (FMNMX3), one compare
// and one warp vote per tile; records carry the chunk's 6-atom group mask.
__device__ __forceinline__ float fmax3f(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }

__device__ __forceinline__ void record_chunk_f32(const uint32_t* r, float cm, int64_t jb,
                                                 float thr, HCandList& cl) {
  uint32_t mask = fmaxf(__uint_as_float(r[30]), __uint_as_float(r[31])) >= thr ? (1u << 5) : 0u;
#pragma unroll
  for (int g = 0; g < 5; ++g) {
    const float m = fmaxf(fmax3f(__uint_as_float(r[6 * g]), __uint_as_float(r[6 * g + 1]),
                                 __uint_as_float(r[6 * g + 2])),
                          fmax3f(__uint_as_float(r[6 * g + 3]), __uint_as_float(r[6 * g + 4]),
                                 __uint_as_float(r[6 * g + 5])));
    mask |= m >= thr ? (1u << g) : 0u;
  }
  cl.insert(pack_chunk(jb, mask), cm, thr);
}

template <int NC>
__device__ __forceinline__ void screen_tile_f32(const uint32_t (&r)[32 * NC], int64_t jb,
                                                float win, float& runmax, float& thr,
                                                bool& active, HCandList& cl) {
  float c[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const uint32_t* q = r + 32 * k;
    float a = fmax3f(__uint_as_float(q[0]), __uint_as_float(q[1]), __uint_as_float(q[2]));
#pragma unroll
    for (int i = 3; i < 31; i += 2)
      a = fmax3f(a, __uint_as_float(q[i]), __uint_as_float(q[i + 1]));
    c[k] = fmaxf(a, __uint_as_float(q[31]));
  }
  float cm = c[0];
#pragma unroll
  for (int k = 1; k < NC; ++k) cm = fmaxf(cm, c[k]);
  if (__any_sync(0xffffffffu, cm >= thr)) {
    if (cm >= thr) {
      runmax = fmaxf(runmax, cm);
      if (active) {
        thr = __fsub_rd(runmax, win);
#pragma unroll
        for (int k = 0; k < NC; ++k)
          if (c[k] >= thr && !cl.ovf) record_chunk_f32(r + 32 * k, c[k], jb + 32 * k, thr, cl);
        if (cl.ovf) {
          active = false;
          thr = INFINITY;
        }
      }
    }
  }
}

// Max of a tile's scores (warm-start hint tiles: the max over the voxel tile's hint atoms is a
// lower bound on the approximate max over the dictionary -- same fp16 rows, same MMA result
// per (voxel, atom) pair -- so it seeds the running max like init_tc; nothing is recorded).
template <int NC>
__device__ __forceinline__ float tile_max_f32(const uint32_t (&r)[32 * NC]) {
  float a = __uint_as_float(r[0]);
#pragma unroll
  for (int i = 1; i + 1 < 32 * NC; i += 2)
    a = fmax3f(a, __uint_as_float(r[i]), __uint_as_float(r[i + 1]));
  return fmaxf(a, __uint_as_float(r[32 * NC - 1]));
}
template <int NC>
__device__ __forceinline__ __half tile_max_f16(const uint32_t (&r)[16 * NC]) {
  __half2 a = as_h2(r[0]);
#pragma unroll
  for (int i = 1; i + 1 < 16 * NC; i += 2) a = hmax3(a, as_h2(r[i]), as_h2(r[i + 1]));
  return hmax_halves(__hmax2(a, as_h2(r[16 * NC - 1])));
}

// Highest of the parts' published thresholds (shared words tag | fp16 bits) whose tag is this
// voxel tile's; -inf if none.  Words of an older voxel tile (or the -inf init) are ignored.
__device__ __forceinline__ __half pub_thr(uint32_t w, uint32_t tag) {
  return __ushort_as_half((w & 0xffff0000u) == tag ? uint16_t(w) : uint16_t(0xFC00));
}
__device__ __forceinline__ uint4 lds_v4_volatile(const uint32_t* p) {
  uint4 w;
  asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "r"(smem_u32(p)));
  return w;
}
__device__ __forceinline__ __half shared_thr(uint4 w, uint32_t tag) {
  return __hmax(__hmax(pub_thr(w.x, tag), pub_thr(w.y, tag)), pub_thr(w.z, tag));
}

template <int KP>
__device__ __forceinline__ void stage_voxel_row(const uint8_t* __restrict__ zrows, int64_t v,
                                                bool live, uint32_t taddr) {
#pragma unroll
  for (int half = 0; half < KP / 32; ++half) {
    uint32_t wz[16];
    const uint4* src = reinterpret_cast<const uint4*>(zrows + size_t(v) * KP * 2) + half * 4;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 x = live ? src[c] : make_uint4(0, 0, 0, 0);
      wz[4 * c + 0] = x.x;
      wz[4 * c + 1] = x.y;
      wz[4 * c + 2] = x.z;
      wz[4 * c + 3] = x.w;
    }
    __syncwarp();
    tmem_st16(taddr + uint32_t(half * 16), wz);
  }
  tc_wait_st();
}

// RANGES: the dictionary is split into nsplit_arg atom ranges (small projections); without it the
// range arithmetic folds away (nsplit = 1)
template <int KP, bool SPLIT, bool PAIR, bool HI32, bool RANGES = false>
__global__ void __launch_bounds__(TcCfg<KP, SPLIT, PAIR, HI32>::kThreads, 1)
    mf_tc_kernel(const uint8_t* __restrict__ zrows, int64_t n, int n_vt,
                 const float* __restrict__ win_tc, const float* __restrict__ init_tc,
                 DictView dv, int64_t n_pad, int2* __restrict__ cand, int2* __restrict__ meta,
                 const uint8_t* __restrict__ hint_tiles, int n_hint, int nsplit_arg) {
  using C = TcCfg<KP, SPLIT, PAIR, HI32>;
  static_assert(!(PAIR && RANGES), "CTA pairs screen the whole dictionary");
  const int nsplit = RANGES ? nsplit_arg : 1;
  constexpr int BN = C::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024_smem(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 2;
  uint64_t* b_full = bars + 4;
  uint64_t* b_empty = b_full + C::kStages;
  uint64_t* t_full = b_empty + C::kStages;
  uint64_t* acc_free = t_full + C::kTBars;  // accumulator stage released by its epilogue part
  // kHalves: second-half barriers (t_full2[tb] / acc_free2[stage]) next to the first-half ones
  uint64_t* t_full2 = acc_free + C::kAcc;
  uint64_t* acc_free2 = t_full2 + C::kTBars;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t d = dv.d;
  const int nB = int((d + BN - 1) / BN);
  // work unit u (the CTA's units are u = blockIdx.x + it * gridDim.x): voxel tile u / nsplit,
  // atom tiles [h nBh, (h + 1) nBh) with h = u % nsplit (the last range runs into sentinel
  // tiles when nsplit does not divide nB; PAIR: nsplit = 1)
  const int nBh = (nB + nsplit - 1) / nsplit;
  // atom tile bytes in global memory and this CTA's copy of it: the fp16 screens store
  // tc_nc(s) chunks per row (no-swizzle layout), the split screen full swizzled K rows
  const int nc = tc_nc(dv.s);
  const uint32_t tile_bytes = SPLIT ? uint32_t(C::kBTileBytes) : uint32_t(BN * nc * 16);
  const uint32_t copy_bytes = SPLIT ? uint32_t(C::kBBytes) : uint32_t(C::kBNloc * nc * 16);
  // PAIR: the two CTAs (ranks 0 = leader, 1) of a cluster stream the same atom tiles in lockstep
  // (same rotation, same number of voxel tiles: the surplus ones are dead, every row v >= n).
  // The leader's issuers run the pair's MMAs; the odd CTA's epilogue and producer signal the
  // leader's barriers remotely, its issuer warps relay "my half of tile k landed".
  const int crank = PAIR ? int(cluster_ctarank()) : 0;
  const bool leader = crank == 0;
  const int csz = PAIR ? 2 : 1;
  const int rot = int((int64_t(blockIdx.x / csz) * nBh) / (gridDim.x / csz));
  const int my_vts = PAIR ? (n_vt + int(gridDim.x) - 1) / int(gridDim.x)
                          : (n_vt * nsplit - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);
  // per voxel tile: n_hint warm-start tiles (the voxel tile's own hint atoms, each hint tile
  // repeated for the kParts parts: tile qt -> hint tile qt / kParts), then the nB atom tiles
  const int T = nBh + n_hint;
  const uint32_t total = uint32_t(my_vts) * uint32_t(T);  // this CTA's tiles

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(a_full + i, 4 * csz);   // the 4 part-0 warps (of both CTAs) stage A
      mbar_init(a_empty + i, kParts);   // each issuer commits after its last tile of a voxel tile
    }
    for (int i = 0; i < C::kTBars; ++i) mbar_init(t_full + i, 1);
    // b_full: the atom tile landed (producer with tx; PAIR leader: + the odd CTA's relayed "my
    // half landed").  acc_free: the 4 warps (PAIR: of both CTAs) of the part that read the
    // accumulator stage released it.  Separate barriers: with one barrier counting both, the
    // issuer woke ~520 clk after the last release (measured), ~2x the separate waits.
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(b_full + i, (PAIR && leader) ? 2 : 1);
      mbar_init(b_empty + i, 1);        // the MMAs reading the stage retired
    }
    for (int i = 0; i < C::kAcc; ++i) mbar_init(acc_free + i, 4 * csz);
    if constexpr (C::kHalves) {
      for (int i = 0; i < C::kTBars; ++i) mbar_init(t_full2 + i, 1);
      for (int i = 0; i < C::kAcc; ++i) mbar_init(acc_free2 + i, 4);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    if constexpr (PAIR)
      tmem_alloc2(tmem_holder, 512);
    else
      tmem_alloc(tmem_holder, 512);
  }
  // published thresholds: tag 0xffff, -inf (matches no voxel tile a CTA reaches in practice,
  // and would only contribute -inf)
  for (int i = threadIdx.x; i < 4 * C::kVox; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem + C::kOffPthr)[i] = 0xFFFFFC00u;
  if constexpr (!SPLIT) {  // finite (zero) stage tails: see atom_chunk_offset
    for (int i = threadIdx.x; i < C::kStages * C::kBBytes / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(smem + C::kOffB)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // the peer's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 0 && !PAIR) {
    // ------------------------------------------------ producer (bulk copies of atom tiles)
    // kParts lanes, lane p copies the tiles k = p (mod kParts) (kStages % kParts == 0: it owns
    // the stages p, p + kParts, ...).  A cp.async.bulk blocks its thread ~140 clk and the
    // empty-barrier wait ~150 clk (scripts/ubench_bulk.cu): one thread streams a tile per
    // ~390 clk, three lanes one per ~175 clk, against ~160 clk of MMA per tile.
    if (lane < kParts) {
      const uint64_t pol_b = policy_evict_last();
      const uint8_t* atiles = SPLIT ? dv.atoms_tc2 : dv.atoms_tc;
      const uint32_t b_full0 = smem_u32(b_full), b_empty0 = smem_u32(b_empty);
      const uint32_t ring0 = smem_u32(smem + C::kOffB);
      int st = lane;
      uint32_t ph = 0;
      int it = 0, b = lane;  // work-unit iteration and tile index inside it
      while (b >= T) {
        b -= T;
        ++it;
      }
      // per work unit: its atom range's first tile and its voxel tile's hint tiles
      const uint8_t* abase = nullptr;
      const uint8_t* hbase = nullptr;
      int it_set = -1;
      for (uint32_t kk = uint32_t(lane); kk < total; kk += kParts) {
        if (it != it_set) {
          const int u = int(blockIdx.x) + it * int(gridDim.x);
          const int vt = u / nsplit;
          abase = atiles + size_t(u - vt * nsplit) * nBh * tile_bytes;
          hbase = hint_tiles + size_t(vt) * (n_hint / kParts) * tile_bytes;
          it_set = it;
        }
        mbar_wait_addr(b_empty0 + 8 * st, ph ^ 1u);
        const uint8_t* src;
        if (b < n_hint) {
          src = hbase + size_t(b / kParts) * tile_bytes;
        } else {
          int ba = rot + b - n_hint;
          if (ba >= nBh) ba -= nBh;
          src = abase + size_t(ba) * tile_bytes;
        }
        mbar_arrive_expect_tx_addr(b_full0 + 8 * st, copy_bytes);
        bulk_g2s_addr(ring0 + st * C::kBBytes, src, copy_bytes, b_full0 + 8 * st, pol_b);
        CBB_STAMP(7, kk);
        st += kParts;
        if (st >= C::kStages) {
          st -= C::kStages;
          ph ^= 1u;
        }
        b += kParts;
        while (b >= T) {
          b -= T;
          ++it;
        }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------ PAIR producer (half of every atom tile)
    const uint64_t pol_b = policy_evict_last();
    const uint8_t* atiles = SPLIT ? dv.atoms_tc2 : dv.atoms_tc;
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < my_vts; ++it) {
      const int vt = int(blockIdx.x) + it * int(gridDim.x);
      int ba = rot;
      for (int b = 0; b < T; ++b) {
        mbar_wait(b_empty + st, ph ^ 1u);
        if (elect_one()) {
          // hint tiles belong to the voxel tile (PAIR: to the pair's 256-voxel group)
          const int hg = PAIR ? vt / 2 : vt, n_hg = PAIR ? (n_vt + 1) / 2 : n_vt;
          const int hvt = hg < n_hg ? hg : n_hg - 1;  // dead voxel tiles reuse a valid hint
          const uint8_t* src =
              b < n_hint
                  ? hint_tiles + (size_t(hvt) * (n_hint / kParts) + b / kParts) * tile_bytes
                  : atiles + size_t(ba) * tile_bytes;
          uint8_t* dst = smem + C::kOffB + st * C::kBBytes;
          mbar_arrive_expect_tx(b_full + st, copy_bytes);
          // this CTA's rows [crank * kBNloc, +kBNloc) of every K block
          if constexpr (SPLIT) {
#pragma unroll
            for (int kb = 0; kb < C::kBlk; ++kb)
              bulk_g2s(dst + kb * C::kBNloc * C::kRowBytes,
                       src + (kb * BN + crank * C::kBNloc) * C::kRowBytes,
                       uint32_t(C::kBNloc * C::kRowBytes), b_full + st, pol_b);
          } else {
            bulk_g2s(dst, src + crank * copy_bytes, copy_bytes, b_full + st, pol_b);
          }
          CBB_STAMP(7, uint32_t(it) * uint32_t(T) + uint32_t(b));
        }
        __syncwarp();
        if (b >= n_hint && ++ba == nB) ba = 0;
        if (++st == C::kStages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (PAIR && !leader && warp >= 1 && warp <= kParts) {
    // ------------------------------------------------ PAIR odd CTA: relay "my half landed"
    const int me = warp - 1;
    const uint32_t bf_leader = mapa_shared(smem_u32(b_full), 0);
    int st = me;
    uint32_t ph = 0;
    for (uint32_t kk = uint32_t(me); kk < total; kk += kParts) {
      mbar_wait(b_full + st, ph);
      if (lane == 0) mbar_arrive_remote(bf_leader + uint32_t(st * 8));
      __syncwarp();
      st += kParts;
      if (st >= C::kStages) {
        st -= C::kStages;
        ph ^= 1u;
      }
    }
  } else if (warp >= 1 && warp <= kParts) {
    // ------------------------------------------------ MMA issuers (warp-uniform, elected lane)
    const int me = warp - 1;
    const int nks = SPLIT ? split_ksteps(dv.s) : mma_ksteps(dv.s);
    const uint32_t b_base = smem_u32(smem + C::kOffB);
    static_assert(C::kAcc == kParts, "issuer i always fills accumulator stage i");
#ifdef CBB_NISS
    constexpr int kIss = CBB_NISS;  // development: issuer warps (kParts % kIss == 0)
#else
    constexpr int kIss = kParts;
#endif
    static_assert(kParts % kIss == 0, "issuers share the stages evenly");
    int sacc = me;  // accumulator stage kk % kAcc
    uint32_t aphm = (1u << C::kAcc) - 1u;  // acc_free parity per stage: first use passes at once
    int tb = me;    // completion barrier kk % kTBars
    int itk = -1;
    uint32_t vt_end = 0;  // first tile index of the next voxel tile
    int st = me;
    uint32_t ph = 0;
    for (uint32_t kk = uint32_t(me); me < kIss && kk < total; kk += kIss) {
      if (kk >= vt_end) {  // first tile of this issuer in a new voxel tile: wait for its A
        ++itk;
        vt_end += uint32_t(T);
        if constexpr (PAIR)
          mbar_wait_cluster(a_full + (itk & 1), (itk >> 1) & 1);
        else
          mbar_wait(a_full + (itk & 1), (itk >> 1) & 1);
      }
      // operands of this tile's MMAs, computed before the waits (off the release -> MMA path)
      const uint32_t a_tm = tbase + uint32_t(C::kAColOff + ((itk & 1) * C::kACols));
      const uint32_t d_tm = tbase + uint32_t(sacc * C::kAccCols);
      uint64_t bdesc[KP / 16];
#pragma unroll
      for (int kq = 0; kq < KP / 16; ++kq)
        // split: K blocks of 64 elements (128 B swizzled rows) follow each other, kBNloc rows
        // each; fp16: no-swizzle core matrices, K step kq = chunks 2kq, 2kq + 1
        bdesc[kq] = SPLIT ? umma_desc_kmajor(b_base + st * C::kBBytes + (kq >> 2) * C::kBNloc * 128,
                                             64) +
                                uint64_t(2 * (kq & 3))
                          : umma_desc_interleave(b_base + st * C::kBBytes + kq * 256, 128, nc * 128);
      // the atom tile usually landed long before the accumulator stage is released: test it
      // first, so the release -> MMA hop is a single barrier wait
      const uint32_t apar = (aphm >> sacc) & 1u;  // this stage use's release phase
      if constexpr (PAIR) {
        mbar_wait_cluster(b_full + st, ph);
        mbar_wait_cluster(acc_free + sacc, (aphm >> sacc) & 1u);
      } else {
        mbar_wait(b_full + st, ph);
#ifdef CBB_SPIN_ISS
        mbar_wait_spin(acc_free + sacc, (aphm >> sacc) & 1u);
#else
        mbar_wait(acc_free + sacc, (aphm >> sacc) & 1u);
#endif
      }
      if (lane == 0) CBB_STAMP(4, kk);
      aphm ^= 1u << sacc;
      tc_fence_after();
      if (lane == 0) CBB_STAMP(0, kk);
      if constexpr (C::kHalves) {
        // first half (atoms 0..63 of the tile -> columns 0..63), then, once the part has
        // released the second half, atoms 64..127 -> columns 64..127 (B rows + 64 x 128 B)
        constexpr uint32_t kIdH = idesc_f16_f32(128, 64);
        if (elect_one()) {
#pragma unroll
          for (int kq = 0; kq < KP / 16; ++kq)
            if (kq < nks)
              tc_mma_f16_ts(d_tm, a_tm + uint32_t(kq * 8), bdesc[kq], kIdH, kq > 0 ? 1u : 0u);
          tc_commit(t_full + tb);
        }
        __syncwarp();
        mbar_wait(acc_free2 + sacc, apar);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kq = 0; kq < KP / 16; ++kq)
            if (kq < nks)
              tc_mma_f16_ts(d_tm + 64u, a_tm + uint32_t(kq * 8),
                            bdesc[kq] + uint64_t((64 * 128) >> 4), kIdH, kq > 0 ? 1u : 0u);
          CBB_STAMP(1, kk);
          tc_commit(b_empty + st);
          tc_commit(t_full2 + tb);
          if (kk + kIss >= vt_end)
            for (int r = 0; r < kParts / kIss; ++r) tc_commit(a_empty + (itk & 1));
        }
      } else if (elect_one()) {
#pragma unroll
        for (int kq = 0; kq < KP / 16; ++kq) {
          if (kq < nks) {
            if constexpr (PAIR)
              tc_mma_f16_ts2(d_tm, a_tm + uint32_t(kq * 8), bdesc[kq], C::kIdesc, kq > 0 ? 1u : 0u);
            else
              tc_mma_f16_ts(d_tm, a_tm + uint32_t(kq * 8), bdesc[kq], C::kIdesc, kq > 0 ? 1u : 0u);
          }
        }
        CBB_STAMP(1, kk);
        if constexpr (PAIR) {  // both CTAs' barriers
          tc_commit2_mc(b_empty + st, 3);
          tc_commit2_mc(t_full + tb, 3);
          if (kk + kIss >= vt_end)
            for (int r = 0; r < kParts / kIss; ++r) tc_commit2_mc(a_empty + (itk & 1), 3);
        } else {
          tc_commit(b_empty + st);
          tc_commit(t_full + tb);
          // this issuer's last tile of the voxel tile: A buffer recyclable once it retires
          if (kk + kIss >= vt_end)
            for (int r = 0; r < kParts / kIss; ++r) tc_commit(a_empty + (itk & 1));
        }
      }
      __syncwarp();
      sacc += kIss;
      if (sacc >= C::kAcc) sacc -= C::kAcc;
      tb += kIss;
      if (tb >= C::kTBars) tb -= C::kTBars;
      st += kIss;
      if (st >= C::kStages) {
        st -= C::kStages;
        ph ^= 1u;
      }
    }
  } else if (warp >= C::kFirstEpiWarp) {
    // -------------------------------------------------- epilogue parts
    const int e = warp - C::kFirstEpiWarp;
    const int part = e >> 2, q = warp & 3;
    const int row = q * 32 + lane;  // voxel row inside the voxel tile (= TMEM lane)
    const int slot = part * C::kVox + row;
    int* cj_base = reinterpret_cast<int*>(smem + C::kOffCj);
    float* cs_base = reinterpret_cast<float*>(smem + C::kOffCs);
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const uint32_t a_lane = tbase + lane_off + uint32_t(C::kAColOff);
    const uint32_t t_lane = tbase + lane_off;
    const uint32_t t_stage = t_lane + uint32_t(part * C::kAccCols);  // fp16: stage == part
    uint32_t* pthr_row = reinterpret_cast<uint32_t*>(smem + C::kOffPthr) + row * 4;
    // A-staged / stage-released signals go to the leader's barriers (PAIR odd CTA: remotely)
    const uint32_t lead_delta =
        (PAIR && !leader) ? mapa_shared(smem_u32(bars), 0) - smem_u32(bars) : 0u;
    auto arrive_lead = [&](uint64_t* bar) {
      if (PAIR && !leader)
        mbar_arrive_remote(smem_u32(bar) + lead_delta);
      else
        mbar_arrive(bar);
    };

    // ---- A for the first voxel tile
    if (part == 0 && my_vts > 0) {
      const int64_t v0 = int64_t(int(blockIdx.x) / nsplit) * C::kVox + row;
      stage_voxel_row<KP>(zrows, v0, v0 < n, a_lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_lead(a_full + 0);
    }

    uint32_t kk = uint32_t(part);  // this part's next tile
    int sacc = part;               // its accumulator stage kk % kAcc
    int tb = part;                 // its completion barrier kk % kTBars, phase (kk / kTBars) & 1
    uint32_t ph = 0;
    for (int it = 0; it < my_vts; ++it) {
      const int u = int(blockIdx.x) + it * int(gridDim.x);
      const int vt = u / nsplit, hr = u - vt * nsplit;  // voxel tile, atom range
      const int opart = hr * kParts + part;  // output lists of (atom range, part)
      const int64_t v = int64_t(vt) * C::kVox + row;
      const bool live = v < n;
      // ---- stage the NEXT voxel tile's rows into the other A buffer (one tile ahead)
      if (part == 0 && it + 1 < my_vts) {
        const int nbuf = (it + 1) & 1;
        mbar_wait(a_empty + nbuf, (((it + 1) >> 1) & 1) ^ 1);
        tc_fence_after();
        const int64_t vn = int64_t((u + int(gridDim.x)) / nsplit) * C::kVox + row;
        stage_voxel_row<KP>(zrows, vn, vn < n, a_lane + uint32_t(nbuf * C::kACols));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_lead(a_full + nbuf);
      }
      if (part == 0 && q == 0 && lane == 0) CBB_STAMP_VT(0, it);
      const float win = live ? win_tc[v] : -1.f;
      bool active = live && win >= 0.f;
      HCandList cl{cj_base + slot, cs_base + slot, C::kSlots, 0,
                   cand + int64_t(opart) * kGCap * n_pad + (live ? v : 0), n_pad, 0, false};
      // running max seeded with the warm-start lower bound (-inf without a hint)
      const float init = live ? fmaxf(init_tc[v], -65504.f) : -INFINITY;
      __half runmax = active ? __float2half_rd(init) : __ushort_as_half(0xFC00);
      __half thr = active ? __float2half_rd(__half2float(runmax) - win)
                          : __ushort_as_half(0x7C00);
      // split mode: fp32 running max / threshold (thresholds rounded down)
      float runmax_f = active ? init_tc[v] : -INFINITY;
      float thr_f = active ? __fsub_rd(runmax_f, win) : INFINITY;
      const uint32_t kbeg = uint32_t(it) * uint32_t(T), kend = kbeg + uint32_t(T);
      if constexpr (!C::kF32) {
        // fp16 screen: the part owns accumulator stage `part` and completion barrier `part`
        // (kAcc == kTBars == kParts), whose phase flips every tile.  The three parts publish
        // their thresholds per voxel in shared memory, tagged with the voxel-tile iteration:
        // any part's rd(runmax - win) is a lower bound on the window edge of the voxel, so each
        // part screens against the highest one it sees (the slow path runs about half as often).
        static_assert(C::kAcc == kParts && C::kTBars == kParts, "stage = part");
        const uint32_t tag = (uint32_t(it) & 0xffffu) << 16;
        uint32_t* my_pub = pthr_row + part;
        const uint32_t khint = kbeg + uint32_t(n_hint);
        uint32_t r[16 * C::kChunks];
        auto consume = [&]() {
          if (q == 0 && lane == 0) CBB_STAMP(5, kk);
#ifdef CBB_SPIN_EPI
          mbar_wait_spin(t_full + part, ph);
#else
          mbar_wait(t_full + part, ph);
#endif
          tc_fence_after();
          if (q == 0 && lane == 0) CBB_STAMP(2, kk);
          __syncwarp();
#pragma unroll
          for (int c = 0; c + 2 <= C::kChunks; c += 2)
            tmem_ld32_pack16(t_stage + uint32_t(32 * c),
                             *reinterpret_cast<uint32_t(*)[32]>(r + 16 * c));
          if (C::kChunks & 1)
            tmem_ld16_pack16(t_stage + uint32_t(32 * (C::kChunks - 1)),
                             *reinterpret_cast<uint32_t(*)[16]>(r + 16 * (C::kChunks - 1)));
          tc_wait_ld();
          // early release: the stage may be overwritten by tile kk + kAcc while we screen
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_lead(acc_free + part);
          if (q == 0 && lane == 0) CBB_STAMP(3, kk);
          ph ^= 1u;
        };
        // warm-start hint tiles: raise the running max, record nothing
        for (; kk < khint; kk += kParts) {
          consume();
          if (active) runmax = __hmax(runmax, tile_max_f16<C::kChunks>(r));
        }
        if (active) {
          thr = __float2half_rd(__half2float(runmax) - win);
          *my_pub = tag | __half_as_ushort(thr);
        }
        // atom tile hr nBh + (rot + qt) % nBh, qt = kk - khint (absolute index, wraps at bend)
        int ba = rot + int(kk - khint);
        if (ba >= nBh) ba -= nBh;
        ba += hr * nBh;
        const int bend = hr * nBh + nBh;
        for (; kk < kend; kk += kParts) {
          const uint4 w = lds_v4_volatile(pthr_row);
          consume();
          thr = __hmax(thr, shared_thr(w, tag));
#if defined(CBB_EPI_EMPTY)  // development timing variants (wrong results)
          if (r[0] == 0x7fff7fffu) runmax = __hmax(runmax, as_h2(r[1]).x);
#elif defined(CBB_EPI_NOSLOW)
          if (__hge(tile_max_f16<C::kChunks>(r), __ushort_as_half(0x7C00))) runmax = thr;
#else
          screen_tile<C::kChunks>(r, int64_t(ba) * BN, win, runmax, thr, active, cl, my_pub, tag);
#endif
          if (q == 0 && lane == 0) CBB_STAMP(6, kk);
          ba += kParts;
          if (ba >= bend) ba -= nBh;
        }
      } else {
        // split / HI32 screen: fp32 scores, at most two chunks (64 registers) in flight; wider tiles
        // are screened in halves and released after the last half is loaded
        for (; kk < kend; kk += kParts) {
          const int qt = int(kk - kbeg) - n_hint;  // < 0: warm-start hint tile
          int ba = rot + qt;                       // range tile (rot + qt) % nBh
          if (ba >= nBh) ba -= nBh;
          ba += hr * nBh;
          if (q == 0 && lane == 0) CBB_STAMP(5, kk);
          mbar_wait(t_full + tb, ph);
          tc_fence_after();
          if (q == 0 && lane == 0) CBB_STAMP(2, kk);
          constexpr int kRegChunks = C::kChunks < 2 ? C::kChunks : 2;
          uint32_t r[32 * kRegChunks];
          __syncwarp();
          const uint32_t ta = t_lane + sacc * uint32_t(C::kAccCols);
#pragma unroll
          for (int h = 0; h < C::kChunks / kRegChunks; ++h) {
            if (C::kHalves && h == 1) {  // second half: its own MMAs and commit
              mbar_wait(t_full2 + tb, ph);
              tc_fence_after();
              __syncwarp();
            }
#pragma unroll
            for (int c = 0; c < kRegChunks; ++c)
              tmem_ld32_f32(ta + uint32_t(32 * (h * kRegChunks + c)),
                            *reinterpret_cast<uint32_t(*)[32]>(r + 32 * c));
            tc_wait_ld();
            if (C::kHalves) {  // release this half at once
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(h == 0 ? acc_free + part : acc_free2 + part);
              if (h == 1 && q == 0 && lane == 0) CBB_STAMP(3, kk);
            } else if (h + 1 == C::kChunks / kRegChunks) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) arrive_lead(acc_free + part);
              if (q == 0 && lane == 0) CBB_STAMP(3, kk);
            }
            if (qt >= 0)
              screen_tile_f32<kRegChunks>(r, int64_t(ba) * BN + 32 * h * kRegChunks, win,
                                          runmax_f, thr_f, active, cl);
            else if (active)
              runmax_f = fmaxf(runmax_f, tile_max_f32<kRegChunks>(r));
          }
          if (qt < 0 && active) thr_f = __fsub_rd(runmax_f, win);  // warm-start tile
          if (q == 0 && lane == 0) CBB_STAMP(6, kk);
          sacc += kParts;
          if (sacc >= C::kAcc) sacc -= C::kAcc;
          tb += kParts;
          if (tb >= C::kTBars) {
            tb -= C::kTBars;
            ph ^= 1u;
          }
        }
      }
      // ---- hand-off (no inter-part barrier): this part's surviving chunk entries are appended
      // to its global list (after any spills); count and running max go to meta.
      // rescore_kernel merges the parts and rescans the flagged groups in fp64
      if (part == 0 && q == 0 && lane == 0) CBB_STAMP_VT(1, it);
      if (live) {
        const float rm = C::kF32 ? runmax_f : __half2float(runmax);
        const int total = (win >= 0.f) ? cl.finish(rm - win) : 0;
        meta[int64_t(opart) * n_pad + v] = make_int2(total, __float_as_int(rm));
      }
      if (part == 0 && q == 0 && lane == 0) CBB_STAMP_VT(2, it);
    }
  }
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // no peer arrives on this CTA's barriers any more
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR)
      tmem_dealloc2(tbase, 512);
    else
      tmem_dealloc(tbase, 512);
  }
}

// ============================================================== dual-voxel-tile fp16 screen
// Measured on cfg1 (1x B200): mf_tc_kernel's skeleton alone (epilogue reduced to wait + load +
// release) takes 6.5 of its 8.4 ms and 4.5 ms without the atom stream -- the L2 -> SMEM copy of
// every atom tile for every 128-voxel tile (68.7 GB per projection, ~9 TB/s) is the limiter.
// This kernel screens TWO voxel tiles (256 voxels) against each streamed 64-atom tile: per tile
// the issuer runs 2 x ksteps MMAs (M = 128, N = 64, one per voxel tile, A from TMEM) reading the
// same SMEM stage, so the atom stream per (voxel, atom) pair halves.  Each epilogue thread owns
// one row of both voxel tiles.  TMEM: 3 stages x [vt0 | vt1] x 64 fp16 accumulator columns + the
// A double buffer 2 x [vt0 | vt1] x KP/2 = 448 (KP 32) / 512 (KP 64) columns.  Barriers, parts,
// records, published thresholds and the hand-off are mf_tc_kernel's (fp16 path).
template <int KP>
struct TcDual {
  static constexpr int BN = 64;
  static constexpr int kChunks = 2;
  static constexpr int kACols = KP / 2;         // one voxel tile's A columns
  static constexpr int kABuf = 2 * kACols;      // one A buffer: [vt0 | vt1]
  static constexpr int kAcc = 3;
  static constexpr int kAccCols = 2 * BN;       // one stage: [vt0 scores | vt1 scores]
  static constexpr int kAColOff = kAcc * kAccCols;
  static_assert(kAColOff + 2 * kABuf <= 512, "TMEM budget");
  static constexpr int kBBytes = BN * KP * 2;
  static constexpr int kRing = 72 * 1024;
  static constexpr int kStagesRaw = kRing / kBBytes > 24 ? 24 : kRing / kBBytes;
  static constexpr int kStages = (kStagesRaw / kParts) * kParts;
  static_assert(kStages >= 2 * kAcc, "B ring too shallow");
  static constexpr int kEpiWarps = 4 * kParts;
  static constexpr int kFirstEpiWarp = 1 + kParts;
  static constexpr int kThreads = (kFirstEpiWarp + kEpiWarps) * 32;
  static constexpr int kVox = 128;
  static constexpr int kSlots = kVox * kParts * 2;
  static constexpr int kOffB = 0;
  static constexpr int kOffCj = kOffB + kStages * kBBytes;
  static constexpr int kOffCs = kOffCj + kCandCap * kSlots * 4;
  static constexpr int kOffPthr = kOffCs + kCandCap * kSlots * 4;  // [2][kVox][4] u32
  static constexpr int kOffBar = kOffPthr + 2 * kVox * 16;
  static constexpr int kNumBars = 4 + 2 * kStages + kAcc;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffTmem + 16 + 1024;
  static_assert(kSmem <= 227 * 1024, "shared memory");
  static constexpr uint32_t kIdesc = idesc_f16_f16(128, BN);
};

template <int KP>
__global__ void __launch_bounds__(TcDual<KP>::kThreads, 1)
    mf_tc_dual_kernel(const uint8_t* __restrict__ zrows, int64_t n, int n_vt,
                      const float* __restrict__ win_tc, const float* __restrict__ init_tc,
                      DictView dv, int64_t n_pad, int2* __restrict__ cand,
                      int2* __restrict__ meta, const uint8_t* __restrict__ hint_tiles,
                      int n_hint) {
  using C = TcDual<KP>;
  constexpr int BN = C::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024_smem(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 2;
  uint64_t* b_full = bars + 4;
  uint64_t* b_empty = b_full + C::kStages;
  uint64_t* t_full = b_empty + C::kStages;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t d = dv.d;
  const int nB = int((d + BN - 1) / BN);
  const int n_pt = (n_vt + 1) / 2;  // voxel-tile pairs (256 voxels)
  const int rot = int((int64_t(blockIdx.x) * nB) / gridDim.x);
  const int my_pts = (n_pt - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);
  const int T = nB + n_hint;
  const uint32_t total = uint32_t(my_pts) * uint32_t(T);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(a_full + i, 4);
      mbar_init(a_empty + i, kParts);
    }
    for (int i = 0; i < C::kAcc; ++i) mbar_init(t_full + i, 1);
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(b_full + i, 1 + 4);
      mbar_init(b_empty + i, 1);
    }
    for (int i = 0; i < C::kAcc; ++i)
      for (int w = 0; w < 4; ++w) mbar_arrive(b_full + i);
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  for (int i = threadIdx.x; i < 2 * 4 * C::kVox; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem + C::kOffPthr)[i] = 0xFFFFFC00u;
  for (int i = threadIdx.x; i < C::kStages * C::kBBytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem + C::kOffB)[i] = make_uint4(0, 0, 0, 0);  // finite tails
  fence_proxy_async_smem();
  const int nc = tc_nc(dv.s);
  const uint32_t tile_bytes = uint32_t(BN * nc * 16);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------ producer (bulk copies of atom tiles)
    const uint64_t pol_b = policy_evict_last();
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < my_pts; ++it) {
      const int pt = int(blockIdx.x) + it * int(gridDim.x);
      int ba = rot;
      for (int b = 0; b < T; ++b) {
        mbar_wait(b_empty + st, ph ^ 1u);
        if (elect_one()) {
          const uint8_t* src =
              b < n_hint ? hint_tiles + (size_t(pt) * (n_hint / kParts) + b / kParts) * tile_bytes
                         : dv.atoms_tc + size_t(ba) * tile_bytes;
          mbar_arrive_expect_tx(b_full + st, tile_bytes);
          bulk_g2s(smem + C::kOffB + st * C::kBBytes, src, tile_bytes, b_full + st, pol_b);
        }
        __syncwarp();
        if (b >= n_hint && ++ba == nB) ba = 0;
        if (++st == C::kStages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp >= 1 && warp <= kParts) {
    // ------------------------------------------------ MMA issuers: 2 voxel tiles per atom tile
    const int me = warp - 1;
    const int nks = mma_ksteps(dv.s);
    const uint32_t b_base = smem_u32(smem + C::kOffB);
    int sacc = me;
    int itk = -1;
    uint32_t vt_end = 0;
    int st = me;
    uint32_t ph = 0;
    for (uint32_t kk = uint32_t(me); kk < total; kk += kParts) {
      if (kk >= vt_end) {
        ++itk;
        vt_end += uint32_t(T);
        mbar_wait(a_full + (itk & 1), (itk >> 1) & 1);
      }
      mbar_wait(b_full + st, ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a_tm = tbase + uint32_t(C::kAColOff + (itk & 1) * C::kABuf);
        const uint32_t d_tm = tbase + uint32_t(sacc * C::kAccCols);
#pragma unroll
        for (int kq = 0; kq < KP / 16; ++kq) {
          const uint64_t bdesc =
              umma_desc_interleave(b_base + st * C::kBBytes + kq * 256, 128, nc * 128);
          if (kq < nks) {
#pragma unroll
            for (int vv = 0; vv < 2; ++vv)
              tc_mma_f16_ts(d_tm + uint32_t(vv * BN), a_tm + uint32_t(vv * C::kACols + kq * 8),
                            bdesc, C::kIdesc, kq > 0 ? 1u : 0u);
          }
        }
        tc_commit(b_empty + st);
        tc_commit(t_full + sacc);
        if (kk + kParts >= vt_end) tc_commit(a_empty + (itk & 1));
      }
      __syncwarp();
      st += kParts;
      if (st >= C::kStages) {
        st -= C::kStages;
        ph ^= 1u;
      }
    }
  } else if (warp >= C::kFirstEpiWarp) {
    // -------------------------------------------------- epilogue parts (one row of each tile)
    const int e = warp - C::kFirstEpiWarp;
    const int part = e >> 2, q = warp & 3;
    const int row = q * 32 + lane;
    int* cj_base = reinterpret_cast<int*>(smem + C::kOffCj);
    float* cs_base = reinterpret_cast<float*>(smem + C::kOffCs);
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const uint32_t a_lane = tbase + lane_off + uint32_t(C::kAColOff);
    const uint32_t t_stage = tbase + lane_off + uint32_t(part * C::kAccCols);
    uint32_t* pthr0 = reinterpret_cast<uint32_t*>(smem + C::kOffPthr) + row * 4;
    uint32_t* pthr1 = pthr0 + C::kVox * 4;

    if (part == 0 && my_pts > 0) {
      const int64_t v0 = int64_t(blockIdx.x) * 2 * C::kVox + row;
      stage_voxel_row<KP>(zrows, v0, v0 < n, a_lane);
      stage_voxel_row<KP>(zrows, v0 + C::kVox, v0 + C::kVox < n, a_lane + uint32_t(C::kACols));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + 0);
    }

    uint32_t kk = uint32_t(part);
    uint32_t ph = 0;
    int rel = part + C::kAcc;
    uint32_t r[32 * 2];
    for (int it = 0; it < my_pts; ++it) {
      const int pt = int(blockIdx.x) + it * int(gridDim.x);
      const int64_t v0 = int64_t(pt) * 2 * C::kVox + row, v1 = v0 + C::kVox;
      const bool live0 = v0 < n, live1 = v1 < n;
      if (part == 0 && it + 1 < my_pts) {
        const int nbuf = (it + 1) & 1;
        mbar_wait(a_empty + nbuf, (((it + 1) >> 1) & 1) ^ 1);
        tc_fence_after();
        const int64_t vn = int64_t(pt + int(gridDim.x)) * 2 * C::kVox + row;
        const uint32_t ab = a_lane + uint32_t(nbuf * C::kABuf);
        stage_voxel_row<KP>(zrows, vn, vn < n, ab);
        stage_voxel_row<KP>(zrows, vn + C::kVox, vn + C::kVox < n, ab + uint32_t(C::kACols));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full + nbuf);
      }
      const float win0 = live0 ? win_tc[v0] : -1.f, win1 = live1 ? win_tc[v1] : -1.f;
      bool active0 = live0 && win0 >= 0.f, active1 = live1 && win1 >= 0.f;
      const int slot0 = (part * 2) * C::kVox + row, slot1 = slot0 + C::kVox;
      HCandList cl0{cj_base + slot0, cs_base + slot0, C::kSlots, 0,
                    cand + int64_t(part) * kGCap * n_pad + (live0 ? v0 : 0), n_pad, 0, false};
      HCandList cl1{cj_base + slot1, cs_base + slot1, C::kSlots, 0,
                    cand + int64_t(part) * kGCap * n_pad + (live1 ? v1 : 0), n_pad, 0, false};
      __half runmax0 = active0 ? __float2half_rd(fmaxf(init_tc[v0], -65504.f))
                               : __ushort_as_half(0xFC00);
      __half runmax1 = active1 ? __float2half_rd(fmaxf(init_tc[v1], -65504.f))
                               : __ushort_as_half(0xFC00);
      __half thr0 = __ushort_as_half(0x7C00), thr1 = __ushort_as_half(0x7C00);
      const uint32_t tag = (uint32_t(it) & 0xffffu) << 16;
      const uint32_t kbeg = uint32_t(it) * uint32_t(T), khint = kbeg + uint32_t(n_hint),
                     kend = kbeg + uint32_t(T);
      auto consume = [&]() {
        mbar_wait(t_full + part, ph);
        tc_fence_after();
        __syncwarp();
        tmem_ld32_pack16(t_stage, *reinterpret_cast<uint32_t(*)[32]>(r));
        tmem_ld32_pack16(t_stage + uint32_t(BN), *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(b_full + rel);
        ph ^= 1u;
        rel += kParts;
        if (rel >= C::kStages) rel -= C::kStages;
      };
      for (; kk < khint; kk += kParts) {  // warm-start hint tiles
        consume();
        if (active0)
          runmax0 = __hmax(runmax0, tile_max_f16<2>(*reinterpret_cast<uint32_t(*)[32]>(r)));
        if (active1)
          runmax1 = __hmax(runmax1, tile_max_f16<2>(*reinterpret_cast<uint32_t(*)[32]>(r + 32)));
      }
      if (active0) {
        thr0 = __float2half_rd(__half2float(runmax0) - win0);
        pthr0[part] = tag | __half_as_ushort(thr0);
      }
      if (active1) {
        thr1 = __float2half_rd(__half2float(runmax1) - win1);
        pthr1[part] = tag | __half_as_ushort(thr1);
      }
      int ba = rot + int(kk - khint);
      if (ba >= nB) ba -= nB;
      for (; kk < kend; kk += kParts) {
        const uint4 w0 = lds_v4_volatile(pthr0), w1 = lds_v4_volatile(pthr1);
        consume();
        thr0 = __hmax(thr0, shared_thr(w0, tag));
        thr1 = __hmax(thr1, shared_thr(w1, tag));
#if defined(CBB_EPI_EMPTY)  // development timing variant (wrong results)
        if (r[0] == 0x7fff7fffu) runmax0 = __hmax(runmax0, as_h2(r[33]).x);
#else
        screen_tile<2>(*reinterpret_cast<uint32_t(*)[32]>(r), int64_t(ba) * BN, win0, runmax0,
                       thr0, active0, cl0, pthr0 + part, tag);
        screen_tile<2>(*reinterpret_cast<uint32_t(*)[32]>(r + 32), int64_t(ba) * BN, win1,
                       runmax1, thr1, active1, cl1, pthr1 + part, tag);
#endif
        ba += kParts;
        if (ba >= nB) ba -= nB;
      }
      if (live0) {
        const float rm = __half2float(runmax0);
        meta[int64_t(part) * n_pad + v0] =
            make_int2((win0 >= 0.f) ? cl0.finish(rm - win0) : 0, __float_as_int(rm));
      }
      if (live1) {
        const float rm = __half2float(runmax1);
        meta[int64_t(part) * n_pad + v1] =
            make_int2((win1 >= 0.f) ? cl1.finish(rm - win1) : 0, __float_as_int(rm));
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// ============================================================== fp64 rescoring of tcgen05 candidates
// rescore_fast_kernel (below) handles every voxel with few entries; this one takes the heavy
// list.  One WARP per voxel (grid-stride): merges the parts' running maxima (gmax), keeps the chunk
// entries whose approximate max lies inside the final window gmax - win, and rescans their
// flagged groups exactly in fp64 from the caller's atoms and voxel -- the entries are spread
// over the lanes, each lane scoring its entry's atoms against the voxel staged in shared
// memory; a warp reduction keeps the best score, lowest index on exact ties (projection.py:62).
// Zero voxels -> index 0 / gamma 0; overflowed candidate lists and non-finite voxels -> the
// next stage's list (fp32 FFMA re-screen).
constexpr int kRescoreWarps = 8;
constexpr int kFastEntries = 2;   // thread-per-voxel rescoring up to this many surviving entries
constexpr int kFastRead = 12;     // ... among at most this many recorded entries
constexpr int kWarpAtoms = 32 * 32;  // per-warp atom list: one round of 32 chunk entries
constexpr int kLaneSurv = 16;        // per-lane fp32-window survivors (atom, fp32 score)

// Expand one chunk entry and rescore its flagged atoms (chunk mask: 6-atom groups).
template <int S>
__device__ __forceinline__ void rescore_entry(int2 en, const double* zr, const double* zi,
                                              int s, const DictView& dv, int64_t& best,
                                              double& bs) {
  const int64_t j0 = int64_t(uint32_t(en.x) & ((1u << kChunkShift) - 1)) << 5;
  uint32_t mask = uint32_t(en.x) >> kChunkShift;
  while (mask) {
    const int b = __ffs(mask) - 1;
    mask &= mask - 1;
    const int lo = 6 * b, hi = b < 5 ? lo + 6 : 32;
    for (int i = lo; i < hi; ++i) {
      const int64_t j = j0 + i;
      if (j >= dv.d) break;
      const double acc = dot_atom<S>(zr, zi, dv.atoms64 + j * s, s);
      if (acc > bs || (acc == bs && j < best)) {
        bs = acc;
        best = j;
      }
    }
  }
}

// One THREAD per voxel: zero voxels, overflow routing and voxels with <= kFastEntries chunk
// entries (every incoherent dictionary); heavier voxels go to the warp kernel's list.
template <int S, int NP = kParts>
__global__ void __launch_bounds__(256) rescore_fast_kernel(
    ZSource zs, DictView dv, int64_t n, int64_t n_pad, const float* __restrict__ win_tc,
    const int2* __restrict__ cand, const int2* __restrict__ meta, ProjOut out, int* ovf_count,
    int64_t* ovf_list, int* heavy_count, int64_t* heavy_list, int fast_entries, int nparts) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const float win = win_tc[v];
  if (win < 0.f) {
    write_winner(out, dv, v, 0, 0.0);
    return;
  }
  // nparts = kParts x the screen's atom ranges
  // NP (compile time) >= nparts part lists
  int cnt[NP];
  float gmax = -INFINITY;
  bool ovf = !(win >= 0.f);
  int entries = 0;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    if (p >= nparts) break;
    const int2 m = meta[int64_t(p) * n_pad + v];
    cnt[p] = m.x;
    entries += m.x;
    ovf |= m.x < 0;
    gmax = fmaxf(gmax, __int_as_float(m.y));
  }
  if (ovf) {
    ovf_list[atomicAdd(ovf_count, 1)] = v;
    return;
  }
  const float thr = gmax - win;
  bool heavy = fast_entries == 0 || entries > kFastRead;
  if (!heavy) {  // entries inside the final (cross-part) window
    int live = 0;
#pragma unroll
    for (int p = 0; p < NP; ++p)
      for (int c = 0; p < nparts && c < cnt[p]; ++c)
        live += __int_as_float(cand[(int64_t(p) * kGCap + c) * n_pad + v].y) >= thr;
    heavy = live > fast_entries;
  }
  if (heavy) {
    heavy_list[atomicAdd(heavy_count, 1)] = v;
    return;
  }
  const int s = dv.s;
  double zr[32], zi[32];
  for (int k = 0; k < s; ++k) {
    const double2 z = load_z(zs, v, s, k);
    zr[k] = z.x;
    zi[k] = z.y;
  }
  int64_t best = INT64_MAX;
  double bs = -INFINITY;
#pragma unroll
  for (int p = 0; p < NP; ++p)
    for (int c = 0; p < nparts && c < cnt[p]; ++c) {
      const int2 en = cand[(int64_t(p) * kGCap + c) * n_pad + v];
      if (__int_as_float(en.y) >= thr) rescore_entry<S>(en, zr, zi, s, dv, best, bs);
    }
  if (best == INT64_MAX) {
    ovf_list[atomicAdd(ovf_count, 1)] = v;
    return;
  }
  write_winner(out, dv, v, best, bs);
}


// entry e of a voxel's concatenated part lists -> (part p, index c in it); unused parts have
// count 0 (static register indexing, no local memory)
template <int NP>
__device__ __forceinline__ void entry_part(int e, const int (&cnt)[NP], int& p, int& c) {
  p = 0;
  c = e;
#pragma unroll
  for (int q = 0; q + 1 < NP; ++q)
    if (p == q && c >= cnt[q]) {
      c -= cnt[q];
      p = q + 1;
    }
}

template <int S, int NP = kParts>
__global__ void __launch_bounds__(32 * kRescoreWarps) rescore_warp_kernel(
    ZSource zs, DictView dv, int64_t n_pad, const float* __restrict__ win_tc,
    const float* __restrict__ win32, const int2* __restrict__ cand,
    const int2* __restrict__ meta, ProjOut out, int* ovf_count, int64_t* ovf_list,
    const int* heavy_count, const int64_t* heavy_list, int nparts) {
  // shared per warp: z (2s doubles), z (2s floats), the atom list, the lanes' fp32 survivors
  extern __shared__ double zsh_all[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int s = dv.s, sp = dv.s_pad;
  double* zsh = zsh_all + size_t(wid) * 2 * s;
  float* z32base = reinterpret_cast<float*>(zsh_all + size_t(kRescoreWarps) * 2 * s);
  float* z32 = z32base + size_t(wid) * 2 * sp;                 // planar, zero-padded to sp
  int* alist_base = reinterpret_cast<int*>(z32base + size_t(kRescoreWarps) * 2 * sp);
  int* alist = alist_base + size_t(wid) * kWarpAtoms;
  int2* surv = reinterpret_cast<int2*>(alist_base + size_t(kRescoreWarps) * kWarpAtoms) +
               (size_t(wid) * 32 + lane) * kLaneSurv;
  const int64_t nw = int64_t(gridDim.x) * kRescoreWarps;
  const int64_t nh = *heavy_count;
  for (int64_t h = int64_t(blockIdx.x) * kRescoreWarps + wid; h < nh; h += nw) {
    const int64_t v = heavy_list[h];
    const float win = win_tc[v];
    if (win < 0.f) {
      if (lane == 0) write_winner(out, dv, v, 0, 0.0);
      continue;
    }
    int cnt[NP];
    float gmax = -INFINITY;
    bool ovf = !(win >= 0.f);
    int total = 0;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      cnt[p] = 0;
      if (p >= nparts) continue;
      const int2 m = meta[int64_t(p) * n_pad + v];  // same address in every lane: broadcast
      cnt[p] = m.x;
      total += m.x;
      ovf |= m.x < 0;
      gmax = fmaxf(gmax, __int_as_float(m.y));
    }
    if (ovf) {
      if (lane == 0) {
        const int slot = atomicAdd(ovf_count, 1);
        ovf_list[slot] = v;
      }
      continue;
    }
    for (int k = lane; k < s; k += 32) {
      const double2 z = load_z(zs, v, s, k);
      zsh[k] = z.x;
      zsh[s + k] = z.y;
      z32[k] = float(z.x);
      z32[sp + k] = float(z.y);
    }
    for (int k = s + lane; k < sp; k += 32) {
      z32[k] = 0.f;
      z32[sp + k] = 0.f;
    }
    __syncwarp();
    const float thr = gmax - win;
    const float w32 = win32[v];
    int64_t best = INT64_MAX;
    double bs = -INFINITY;
    // fp32 pre-filter (certified window w32): every lane keeps the atoms within w32 of its own
    // running fp32 max (a superset of the final survivors); only those are rescored in fp64.
    // A full lane list sends the voxel through the fp64 pass below instead.
    float lmax = -INFINITY;
    int nsurv = 0;
    bool full = false;
    // rounds of 32 entries: each lane expands its entry's flagged atoms into the warp's atom
    // list (warp prefix sum of the counts), then the lanes score the list round-robin
    for (int e0 = 0; e0 < total; e0 += 32) {
      const int e = e0 + lane;
      int64_t j0 = 0;
      uint32_t mask = 0;
      if (e < total) {
        int p, c;
        entry_part(e, cnt, p, c);
        const int2 en = cand[(int64_t(p) * kGCap + c) * n_pad + v];
        if (__int_as_float(en.y) >= thr) {
          j0 = int64_t(uint32_t(en.x) & ((1u << kChunkShift) - 1)) << 5;
          mask = uint32_t(en.x) >> kChunkShift;
        }
      }
      // groups 0..4: 6 atoms, group 5: 2 atoms
      const int na = 6 * __popc(mask & 0x1Fu) + 2 * ((mask >> 5) & 1u);
      int off = na;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, off, o);
        if (lane >= o) off += y;
      }
      const int round_total = __shfl_sync(0xffffffffu, off, 31);
      off -= na;
      while (mask) {
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        const int lo = 6 * b, hi = b < 5 ? lo + 6 : 32;
        for (int i = lo; i < hi; ++i) alist[off++] = int(j0 + i);
      }
      __syncwarp();
      for (int a = lane; a < round_total; a += 32) {
        const int64_t j = alist[a];
        if (j >= dv.d) continue;
        const float sc = dot_atom32<S>(z32, z32 + sp, dv.atoms32 + j * 2 * sp, s, sp);
        lmax = fmaxf(lmax, sc);
        if (sc >= lmax - w32) {
          if (nsurv == kLaneSurv) {  // drop survivors the running max has since excluded
            int k2 = 0;
            for (int c = 0; c < kLaneSurv; ++c)
              if (__int_as_float(surv[c].y) >= lmax - w32) surv[k2++] = surv[c];
            nsurv = k2;
          }
          if (nsurv < kLaneSurv) surv[nsurv++] = make_int2(int(j), __float_as_int(sc));
          else full = true;
        }
      }
      __syncwarp();
    }
    float gmax32 = lmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmax32 = fmaxf(gmax32, __shfl_xor_sync(0xffffffffu, gmax32, o));
    const float thr32 = gmax32 - w32;
    for (int c = 0; c < nsurv; ++c) {
      const int2 e2 = surv[c];
      if (__int_as_float(e2.y) < thr32) continue;
      const int64_t j = e2.x;
      const double acc = dot_atom<S>(zsh, zsh + s, dv.atoms64 + j * s, s);
      if (acc > bs || (acc == bs && j < best)) {
        bs = acc;
        best = j;
      }
    }
    if (__any_sync(0xffffffffu, full) || !(w32 >= 0.f)) {
      // fp64 over every flagged atom (the pre-filter could not keep all its survivors)
      best = INT64_MAX;
      bs = -INFINITY;
      for (int e0 = 0; e0 < total; e0 += 32) {
        const int e = e0 + lane;
        if (e < total) {
          int p, c;
          entry_part(e, cnt, p, c);
          const int2 en = cand[(int64_t(p) * kGCap + c) * n_pad + v];
          if (__int_as_float(en.y) >= thr) rescore_entry<S>(en, zsh, zsh + s, s, dv, best, bs);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double obs = __shfl_xor_sync(0xffffffffu, bs, o);
      const int64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
      if (obs > bs || (obs == bs && ob < best)) {
        bs = obs;
        best = ob;
      }
    }
    if (lane == 0) {
      if (best == INT64_MAX) {
        const int slot = atomicAdd(ovf_count, 1);
        ovf_list[slot] = v;
      } else {
        write_winner(out, dv, v, best, bs);
      }
    }
    __syncwarp();
  }
}

// Debug: raw fp16 tcgen05 scores (A = voxel rows staged into TMEM, B = swizzled atom tile in
// SMEM) of voxel rows [128 a_tile, +128) x atoms [128 b_tile, +128) -- validates descriptors,
// the swizzled atom tiles and the TMEM A-operand layout against a host emulation.
template <int KP>
__global__ void __launch_bounds__(128, 1)
    tc_debug_scores_kernel(const uint8_t* __restrict__ zrows, const uint8_t* __restrict__ atiles,
                           int nc, int a_tile, int b_tile, float* __restrict__ out) {
  constexpr int kTileBytes = kTileRows * KP * 2;  // SMEM buffer (>= the stored tile, zero tail)
  const uint32_t tbytes = uint32_t(kTileRows * nc * 16);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024_smem(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kTileBytes);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + kTileBytes + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(holder, 256);
  for (int i = threadIdx.x; i < kTileBytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *holder;
  const uint32_t a_col = 128;
  stage_voxel_row<KP>(zrows, int64_t(a_tile) * 128 + threadIdx.x, true,
                      tbase + (uint32_t(warp * 32) << 16) + a_col);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, tbytes);
    bulk_g2s(smem, atiles + size_t(b_tile) * tbytes, tbytes, bar, policy_evict_first());
    mbar_wait(bar, 0);
    tc_fence_after();
    for (int k = 0; k < KP / 16; ++k)  // every K step (those past the data multiply zeros)
      tc_mma_f16_ts(tbase, tbase + a_col + k * 8,
                    umma_desc_interleave(smem_u32(smem) + k * 256, 128, nc * 128),
                    idesc_f16_f16(128, 128), k > 0);
    tc_commit(bar + 1);
  }
  __syncwarp();
  mbar_wait(bar + 1, 0);
  tc_fence_after();
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    tmem_ld32_pack16(tbase + (uint32_t(warp * 32) << 16) + c * 64, r);
    tc_wait_ld();
    for (int i = 0; i < 32; ++i) {
      const float2 f = __half22float2(as_h2(r[i]));
      out[(warp * 32 + lane) * 128 + c * 64 + 2 * i] = f.x;
      out[(warp * 32 + lane) * 128 + c * 64 + 2 * i + 1] = f.y;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

// ============================================================== atom-shard write-back
// out[v] = gamma[v] * atoms[idx[v] - offset] when this shard owns idx[v], else 0 (the shards'
// outputs are then summed across ranks).  One thread per (voxel, component).
__global__ void scaled_rows_kernel(const double2* __restrict__ atoms64, int64_t d, int s,
                                   int64_t offset, const int64_t* __restrict__ idx,
                                   const double* __restrict__ gamma, int64_t n, void* out,
                                   int out128) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * s) return;
  const int64_t v = e / s, k = e % s;
  const int64_t j = idx[v] - offset;
  double2 r = make_double2(0.0, 0.0);
  if (j >= 0 && j < d) {
    const double2 a = atoms64[j * s + k];
    r = make_double2(gamma[v] * a.x, gamma[v] * a.y);
  }
  if (out128) reinterpret_cast<double2*>(out)[e] = r;
  else reinterpret_cast<float2*>(out)[e] = make_float2(float(r.x), float(r.y));
}

int scaled_rows(const DictView& dv, int64_t offset, const int64_t* idx, const double* gamma,
                int64_t n, void* out, int out128, cudaStream_t st) {
  if (n == 0) return kOk;
  const int64_t total = n * dv.s;
  scaled_rows_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(dv.atoms64, dv.d, dv.s,
                                                                    offset, idx, gamma, n, out,
                                                                    out128);
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return kOk;
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

size_t dict_bytes(int64_t d, int s, size_t* off64, size_t* off32, size_t* offtc, size_t* offb,
                  size_t* offtc2) {
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
  // + two extra 128-row sentinel tiles: the screening reads BN-row (BN <= 256) windows that
  // may run past the last 128-row tile
  size_t c = take(size_t(nbt + kPadTiles) * kTileRows * kp * 2);
  size_t e = take(kBCount * sizeof(float));
  size_t f = take(s <= kSplitMaxS ? size_t(nbt + kPadTiles) * kTileRows * split_kp(s) * 2 : 0);
  if (offtc2) *offtc2 = f;
  if (off64) *off64 = a;
  if (off32) *off32 = b;
  if (offtc) *offtc = c;
  if (offb) *offb = e;
  return o;
}

int dict_prepare(const void* atoms, int in128, int64_t d, int s, void* storage, DictView* view,
                 cudaStream_t st) {
  if (d <= 0 || s <= 0) return kErrArgument;
  size_t o64, o32, otc, ob, otc2;
  const size_t total = dict_bytes(d, s, &o64, &o32, &otc, &ob, &otc2);
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
  v.atoms_tc2 = s <= kSplitMaxS ? base + otc2 : nullptr;
  const int threads = 256;
  const int blocks = int((d + threads - 1) / threads);
  prep_dict_kernel<<<blocks, threads, 0, st>>>(atoms, in128, d, s, v.s_pad,
                                                const_cast<double2*>(v.atoms64),
                                                const_cast<float*>(v.atoms32),
                                                const_cast<float*>(v.bounds));
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  if (2 * s < 64) {  // tensor-core operand tiles (+ sentinel column)
    const int64_t d_pad = int64_t(v.n_btiles + kPadTiles) * kTileRows;
    prep_tc_kernel<<<int((d_pad + threads - 1) / threads), threads, 0, st>>>(
        v.atoms64, d, d_pad, s, const_cast<uint8_t*>(v.atoms_tc),
        const_cast<float*>(v.bounds));
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(1);
  }
  if (v.s <= 32) {  // coherence estimate for the auto screen choice (planar fp32 copy)
    coherence_kernel<<<kCohSamples, 256, 0, st>>>(v.atoms32, d, s, v.s_pad,
                                                  const_cast<float*>(v.bounds));
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(1);
  }
  if (v.atoms_tc2) {  // split-operand tiles (after prep_tc_kernel: it publishes scale_d)
    const int64_t d_pad = int64_t(v.n_btiles + kPadTiles) * kTileRows;
    prep_tc2_kernel<<<int((d_pad + threads - 1) / threads), threads, 0, st>>>(
        v.atoms64, d, d_pad, s, const_cast<uint8_t*>(v.atoms_tc2), const_cast<float*>(v.bounds));
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(1);
  }
  v.prefer_split = 0;
  if (v.atoms_tc2) {
    // one-time host read of the coherence estimate (dictionary preparation synchronises once)
    float coh = 0.f;
    CBB_CUDA_TRY(cudaMemcpyAsync(&coh, v.bounds + kBCoherence, sizeof(float),
                                 cudaMemcpyDeviceToHost, st));
    CBB_CUDA_TRY(cudaStreamSynchronize(st));
    v.prefer_split = coh >= 1.0f ? 1 : 0;
  }
  *view = v;
  return kOk;
}

// Workspace carve-up for one projection call.
struct ProjWs {
  int64_t n_pad;
  int2* cand;      // [kParts][kGCap][n_pad] tcgen05 chunk entries (entry, approx max)
  int2* meta;      // [kParts][n_pad] (entry count or -1 on overflow, part running max)
  uint8_t* ztiles;
  float* win_tc;
  float* init_tc;  // warm-start lower bound of each voxel's approximate max (scaled units)
  float* win32;
  int* ovf_count;       // tcgen05 / FFMA pass overflows (next stage's voxel list)
  int64_t* ovf_list;
  int* heavy_count;     // voxels with many tcgen05 chunk entries (warp rescoring)
  int64_t* heavy_list;
  double2* exh_partial; // [n][kExhSplits] (score, index) of the split exhaustive scan
  uint8_t* hint_tiles;  // [voxel tile][hint tile] warm-start tiles (IPG)
  double* nd_v;
  double* partial;
};
constexpr int kReduceBlocks = 256;
constexpr int kVoxPad = 512;  // voxel tiles are padded to a multiple of the largest TC voxel tile

size_t project_ws_bytes(int64_t n, int s, ProjWs* ws, void* base_ptr) {
  const int kp = s <= kSplitMaxS ? split_kp(s) : kpad_for(s);  // split rows are wider
  const int64_t n_vt = (n + kVoxPad - 1) / kVoxPad;
  size_t o = 0;
  uint8_t* base = static_cast<uint8_t*>(base_ptr);
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) & ~size_t(255);
    return base ? base + r : nullptr;
  };
  ProjWs w{};
  w.n_pad = n_vt * kVoxPad;
  w.ztiles = take(size_t(n_vt) * kVoxPad * kp * 2);  // first: cbb_debug_tc_scores reads it
  const int parts = kParts * (n <= kSplitMaxN ? kMaxSplit : 1);  // see launch_tc
  w.cand = reinterpret_cast<int2*>(take(size_t(w.n_pad) * parts * kGCap * sizeof(int2)));
  w.meta = reinterpret_cast<int2*>(take(size_t(w.n_pad) * parts * sizeof(int2)));
  w.win_tc = reinterpret_cast<float*>(take(size_t(n_vt) * kVoxPad * 4));
  w.init_tc = reinterpret_cast<float*>(take(size_t(n_vt) * kVoxPad * 4));
  w.win32 = reinterpret_cast<float*>(take(size_t(n_vt) * kVoxPad * 4));
  w.ovf_count = reinterpret_cast<int*>(take(16));
  w.ovf_list = reinterpret_cast<int64_t*>(take(size_t(n) * 8));
  w.heavy_count = reinterpret_cast<int*>(take(16));
  w.heavy_list = reinterpret_cast<int64_t*>(take(size_t(n) * 8));
  w.exh_partial = reinterpret_cast<double2*>(take(size_t(n) * kExhSplits * sizeof(double2)));
  {  // hint tiles: the largest per-voxel-tile block of the screens this s can use
    size_t per_vt = kpad_for(s) == 32 ? 160 * 32 * 2 : 128 * 64 * 2;
    if (s <= kSplitMaxS) {
      const int k2 = split_kp(s), rows = split_rows(k2);
      const size_t sb = size_t((kTileRows + rows - 1) / rows) * rows * k2 * 2;
      if (sb > per_vt) per_vt = sb;
    }
    w.hint_tiles = take(size_t(n_vt) * (kVoxPad / kTileRows) * per_vt);
  }
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

// Warm-start hint tiles: row r of voxel tile vt's hint block = a copy of the storage row of
// atom hint[vt*128 + r] (the previous IPG winner of that voxel), in the screen's own tile
// layout (vox voxels per tile group: 128, or 256 for a CTA pair); rows without a valid hint
// (and rows >= vox of the last tile) copy the first padded
// row (score -65504 for every voxel).  One thread per 16-byte chunk.
__global__ void __launch_bounds__(256) hint_tiles_kernel(const int32_t* __restrict__ hint,
                                                         int64_t n, int64_t d, int n_vt, int vox,
                                                         const uint8_t* __restrict__ atiles,
                                                         int kp, int split, int bn, int nh,
                                                         uint8_t* __restrict__ out) {
  // 16-byte chunks per row: split rows kp / 8; fp16 rows tc_nc(s), passed as kp = 8 * nc
  const int cpr = kp / 8;
  const int64_t per_vt = int64_t(nh) * bn * cpr;
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= per_vt * n_vt) return;
  const int vt = int(g / per_vt);
  const int rem = int(g - int64_t(vt) * per_vt);
  const int r = rem / cpr, c = rem - r * cpr;
  const int64_t v = int64_t(vt) * vox + r;
  int64_t j = d;
  if (r < vox && v < n) {
    const int64_t h = hint[v];
    if (h >= 0 && h < d) j = h;
  }
  size_t src, dst;
  const int hb = r / bn, rr = r - hb * bn;
  if (split) {
    const int rows = split_rows(kp);
    src = size_t(j / rows) * rows * kp * 2 + split_elem_offset(int(j % rows), 8 * c, rows);
    dst = (size_t(vt) * nh + hb) * bn * kp * 2 + split_elem_offset(rr, 8 * c, bn);
  } else {
    src = atom_chunk_offset(j, c, cpr);
    dst = (size_t(vt) * nh + hb) * bn * cpr * 16 + atom_chunk_offset(rr, c, cpr);
  }
  *reinterpret_cast<uint4*>(out + dst) = *reinterpret_cast<const uint4*>(atiles + src);
}

template <class C>
constexpr int BN_of() { return C::BN; }

// CTA pairs for the matched-filter screen (cta_group::2, see TcCfg): opt-in with CBB_TC_PAIR=1.
// Measured on cfg1 (1x B200): 19.1 ms vs 8.4 ms for single CTAs -- the odd CTA's remote stage
// releases lengthen the refill chain of every accumulator stage (release -> issuer 445 -> 1255
// clk) by more than the halved atom stream saves.
static bool tc_pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CBB_TC_PAIR");
    v = (e && atoi(e) == 1) ? 1 : 0;
  }
  return v != 0;
}
template <class K>
static int max_coresident_pairs(K kernel, int threads, int smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(256u);
  cfg.blockDim = dim3(unsigned(threads));
  cfg.dynamicSmemBytes = size_t(smem);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return nc;
}

template <int KP, bool SPLIT, bool PAIR, bool HI32, bool RANGES = false>
static int launch_tc_as(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                        int grid, int n_vt, cudaStream_t st, int nsplit = 1) {
  using C = TcCfg<KP, SPLIT, PAIR, HI32>;
  int n_hint = 0;
  if (zs.hint) {  // IPG warm start: the voxel tiles' (pairs') own hint atoms screened first
    const int vox = PAIR ? 2 * C::kVox : C::kVox;
    const int n_g = int((n + vox - 1) / vox);
    const int nh = (vox + C::BN - 1) / C::BN;
    const int kw = SPLIT ? KP : 8 * tc_nc(dv.s);  // row width (fp16 elements) as stored
    const int64_t chunks = int64_t(n_g) * nh * C::BN * (kw / 8);
    hint_tiles_kernel<<<unsigned((chunks + 255) / 256), 256, 0, st>>>(
        zs.hint, n, dv.d, n_g, vox, SPLIT ? dv.atoms_tc2 : dv.atoms_tc, kw, SPLIT ? 1 : 0, C::BN,
        nh, w.hint_tiles);
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    n_hint = kParts * nh;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(C::kThreads));
  cfg.dynamicSmemBytes = size_t(C::kSmem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = PAIR ? 1 : 0;
  CBB_CUDA_TRY(cudaLaunchKernelEx(&cfg, mf_tc_kernel<KP, SPLIT, PAIR, HI32, RANGES>, w.ztiles, n,
                                  n_vt,
                                  (const float*)w.win_tc, (const float*)w.init_tc, dv, w.n_pad,
                                  w.cand, w.meta, (const uint8_t*)w.hint_tiles, n_hint, nsplit));
  return kOk;
}

// Dual-voxel-tile fp16 screen (mf_tc_dual_kernel): opt-in with CBB_TC_DUAL=1 (measured on
// cfg1 with a dedicated producer warp: 10.5 ms vs 8.5 ms).
static bool tc_dual_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CBB_TC_DUAL");
    v = (e && atoi(e) == 1) ? 1 : 0;
  }
  return v != 0;
}

template <int KP>
static int launch_tc_dual(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                          int grid, int n_vt, cudaStream_t st) {
  using C = TcDual<KP>;
  static bool attr_set = false;
  if (!attr_set) {
    CBB_CUDA_TRY(cudaFuncSetAttribute(mf_tc_dual_kernel<KP>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  int n_hint = 0;
  if (zs.hint) {  // IPG warm start: each voxel-tile pair's own hint atoms screened first
    const int vox = 2 * C::kVox;
    const int n_g = int((n + vox - 1) / vox);
    const int nh = (vox + C::BN - 1) / C::BN;
    const int64_t chunks = int64_t(n_g) * nh * C::BN * tc_nc(dv.s);
    hint_tiles_kernel<<<unsigned((chunks + 255) / 256), 256, 0, st>>>(
        zs.hint, n, dv.d, n_g, vox, dv.atoms_tc, 8 * tc_nc(dv.s), 0, C::BN, nh, w.hint_tiles);
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    n_hint = kParts * nh;
  }
  mf_tc_dual_kernel<KP><<<grid, C::kThreads, C::kSmem, st>>>(
      w.ztiles, n, n_vt, w.win_tc, w.init_tc, dv, w.n_pad, w.cand, w.meta, w.hint_tiles, n_hint);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

template <int KP, bool SPLIT = false, bool HI32 = false>
static int launch_tc(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                     const ProjOut& out, int max_ctas, cudaStream_t st, int* nsplit_out) {
  *nsplit_out = 1;
  using C1 = TcCfg<KP, SPLIT, false, HI32>;
  using C2 = TcCfg<KP, SPLIT, true, HI32>;
  static bool attr_set = false;
  static int pairs = 0;
  if (!attr_set) {
    CBB_CUDA_TRY(cudaFuncSetAttribute(mf_tc_kernel<KP, SPLIT, false, HI32>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C1::kSmem));
    CBB_CUDA_TRY(cudaFuncSetAttribute(mf_tc_kernel<KP, SPLIT, false, HI32, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C1::kSmem));
    CBB_CUDA_TRY(cudaFuncSetAttribute(mf_tc_kernel<KP, SPLIT, true, HI32>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C2::kSmem));
    pairs = max_coresident_pairs(mf_tc_kernel<KP, SPLIT, true, HI32>, C2::kThreads, C2::kSmem);
    attr_set = true;
  }
  const int n_vt = int((n + C1::kVox - 1) / C1::kVox);
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if constexpr (!SPLIT && !HI32) {
    // dual-voxel-tile screen when every CTA gets at least one voxel-tile pair
    const int n_pt = (n_vt + 1) / 2;
    if (tc_dual_enabled() && n_pt >= grid) return launch_tc_dual<KP>(w, n, zs, dv, grid, n_vt, st);
  }
  // atom ranges: small projections (at most kSplitMaxN voxels) split the dictionary so the
  // work units (voxel tile x range) cover the SMs evenly: the smallest nsplit minimising
  // ceil(n_vt nsplit / grid) / nsplit, every range keeping >= 2 tiles per part
  if (n <= kSplitMaxN) {
    const int nB = int((dv.d + C1::BN - 1) / C1::BN);
    int best = 1;
    double best_t = double((n_vt + grid - 1) / grid);
    for (int ns = 2; ns <= kMaxSplit; ++ns) {
      if ((nB + ns - 1) / ns < 2 * kParts) break;
      const double t = double((int64_t(n_vt) * ns + grid - 1) / grid) / ns;
      if (t < best_t * 0.97) {
        best = ns;
        best_t = t;
      }
    }
    if (best > 1) {
      *nsplit_out = best;
      const int units = n_vt * best;
      return launch_tc_as<KP, SPLIT, false, HI32, true>(w, n, zs, dv, units < grid ? units : grid,
                                                        n_vt, st, best);
    }
  }
  if (grid > n_vt) grid = n_vt;
  // CTA pairs halve the atom stream; used when every pair is co-resident (persistent kernel),
  // at most 5% of the SMs idle, and every CTA gets at least two voxel tiles
  int grid2 = 2 * pairs < grid ? 2 * pairs : grid - grid % 2;
  if (tc_pair_enabled() && grid2 >= 8 && grid2 * 20 >= grid * 19 && n_vt >= 2 * grid2)
    return launch_tc_as<KP, SPLIT, true, HI32>(w, n, zs, dv, grid2, n_vt, st);
  return launch_tc_as<KP, SPLIT, false, HI32>(w, n, zs, dv, grid, n_vt, st);
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

template <int S>
static int launch_exhaustive_s(int64_t n, const ZSource& zs, const DictView& dv, const int* cnt,
                               const int64_t* list, const ProjOut& out, cudaStream_t st) {
  const size_t shm = size_t(8) * 2 * dv.s * sizeof(double);
  if (shm > 48 * 1024) {
    CBB_CUDA_TRY(cudaFuncSetAttribute(exhaustive_kernel<S>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
  }
  int grid = num_sms() * 4;
  if (!list) {
    int64_t need = (n + 7) / 8;
    if (need < grid) grid = int(need > 0 ? need : 1);
  }
  exhaustive_kernel<S><<<grid, 256, shm, st>>>(zs, dv, n, cnt, list, out);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// compile-time width for the fp64 scoring loops (s_pad; 0 = runtime loop for s > 32)
#define CBB_DISPATCH_S(s_pad, CALL)          \
  switch (s_pad) {                          \
    case 2: { constexpr int S_ = 2; CALL; }   \
    case 4: { constexpr int S_ = 4; CALL; }   \
    case 6: { constexpr int S_ = 6; CALL; }   \
    case 8: { constexpr int S_ = 8; CALL; }   \
    case 10: { constexpr int S_ = 10; CALL; } \
    case 12: { constexpr int S_ = 12; CALL; } \
    case 16: { constexpr int S_ = 16; CALL; } \
    case 20: { constexpr int S_ = 20; CALL; } \
    case 24: { constexpr int S_ = 24; CALL; } \
    case 32: { constexpr int S_ = 32; CALL; } \
    default: { constexpr int S_ = 0; CALL; }  \
  }

static int launch_exhaustive(int64_t n, const ZSource& zs, const DictView& dv, const int* cnt,
                             const int64_t* list, const ProjOut& out, cudaStream_t st) {
  const int sp = s_pad_for(dv.s);
  CBB_DISPATCH_S(sp, return launch_exhaustive_s<S_>(n, zs, dv, cnt, list, out, st));
  return kOk;
}

template <int S>
static int launch_exhaustive_list_s(int64_t n, const ZSource& zs, const DictView& dv,
                                    const int* cnt, const int64_t* list, const float* win32,
                                    double2* partial, const ProjOut& out, cudaStream_t st) {
  const size_t shm = size_t(8) * (2 * dv.s * sizeof(double) + 2 * dv.s_pad * sizeof(float) +
                                  32 * kExhSurv * sizeof(int2));
  if (shm > 48 * 1024)
    CBB_CUDA_TRY(cudaFuncSetAttribute(exhaustive_split_kernel<S>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
  exhaustive_split_kernel<S><<<num_sms() * 8, 256, shm, st>>>(zs, dv, cnt, list, win32, partial);
  CBB_CUDA_TRY(cudaGetLastError());
  exhaustive_finish_kernel<<<int((n + 255) / 256), 256, 0, st>>>(dv, cnt, list, partial, out);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// exhaustive fp64 rescan of the overflow list (count on the device), dictionary split 16 ways
static int launch_exhaustive_list(int64_t n, const ZSource& zs, const DictView& dv,
                                  const int* cnt, const int64_t* list, const float* win32,
                                  double2* partial, const ProjOut& out, cudaStream_t st) {
  const int sp = s_pad_for(dv.s);
  CBB_DISPATCH_S(sp, return launch_exhaustive_list_s<S_>(n, zs, dv, cnt, list, win32, partial,
                                                         out, st));
  return kOk;
}

template <int S, int NP>
static int launch_rescore_np(const ProjWs& w, int64_t n, const ZSource& zr, const DictView& dv,
                          const ProjOut& o, cudaStream_t st, int nparts) {
  // small projections: too few threads for the thread-per-voxel path to hide L2 latency, every
  // voxel goes to the warp kernel
  const int fast = n >= int64_t(num_sms()) * 256 ? kFastEntries : 0;
  rescore_fast_kernel<S, NP><<<int((n + 255) / 256), 256, 0, st>>>(
      zr, dv, n, w.n_pad, w.win_tc, w.cand, w.meta, o, w.ovf_count, w.ovf_list, w.heavy_count,
      w.heavy_list, fast, nparts);
  CBB_CUDA_TRY(cudaGetLastError());
  const size_t shm = size_t(kRescoreWarps) * (2 * dv.s * sizeof(double) +
                                               2 * dv.s_pad * sizeof(float) +
                                               kWarpAtoms * sizeof(int) +
                                               32 * kLaneSurv * sizeof(int2));
  if (shm > 48 * 1024)
    CBB_CUDA_TRY(cudaFuncSetAttribute(rescore_warp_kernel<S, NP>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
  rescore_warp_kernel<S, NP><<<num_sms() * 8, 32 * kRescoreWarps, shm, st>>>(
      zr, dv, w.n_pad, w.win_tc, w.win32, w.cand, w.meta, o, w.ovf_count, w.ovf_list,
      w.heavy_count, w.heavy_list, nparts);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

template <int S>
static int launch_rescore(const ProjWs& w, int64_t n, const ZSource& zr, const DictView& dv,
                          const ProjOut& o, cudaStream_t st, int nparts) {
  return nparts == kParts ? launch_rescore_np<S, kParts>(w, n, zr, dv, o, st, nparts)
                          : launch_rescore_np<S, kParts * kMaxSplit>(w, n, zr, dv, o, st, nparts);
}

int reduce_sum(const double* x, int64_t n, double* partial, double* out, cudaStream_t st) {
  reduce_stage1<<<kReduceBlocks, 256, 0, st>>>(x, n, partial);
  reduce_stage2<<<1, 256, 0, st>>>(partial, kReduceBlocks, out);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// algo: 0 = auto (split tcgen05 for coherent dictionaries with s <= 21, else tcgen05 when
// 2s < 64, else FFMA / fp64),
// 1 = tcgen05 (fp16 accumulators), 2 = FFMA, 3 = exhaustive fp64, 4 = split tcgen05 (hi/lo fp16
// operands, fp32 accumulators, s <= 21), 5 = HI32 tcgen05 (fp16 operands, fp32 accumulators)
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
  // tcgen05 path: K = 2s <= 64; chunk entries pack (atom / 32) into 20 bits; every epilogue
  // part needs >= 2 atom tiles of 64 per voxel tile (d > 320; smaller dictionaries use FFMA)
  const bool tc_ok = (2 * dv.s < 64) && (dv.d <= (int64_t(1) << 25)) && (dv.d > 320);
  const bool split_ok = tc_ok && dv.s <= kSplitMaxS && dv.atoms_tc2 != nullptr;
  if (algo == 0) algo = (split_ok && dv.prefer_split) ? 4 : tc_ok ? 1 : (s_pad_for(dv.s) > 0 ? 2 : 3);
  if ((algo == 1 || algo == 5) && !tc_ok) return kErrUnsupported;
  if (algo == 4 && !split_ok) return kErrUnsupported;
  const bool split = algo == 4, hi32 = algo == 5;
  if (split || hi32) algo = 1;  // same pipeline, other operand tiles / accumulator format
  if (algo == 2 && s_pad_for(dv.s) < 0) return kErrUnsupported;
  CBB_CUDA_TRY(cudaMemsetAsync(w.ovf_count, 0, sizeof(int), st));
  CBB_CUDA_TRY(cudaMemsetAsync(w.heavy_count, 0, sizeof(int), st));
  if (algo == 1 || algo == 2) {
    const int64_t n_pad = ((n + kVoxPad - 1) / kVoxPad) * kVoxPad;
    const int threads = 256;
    prologue_kernel<<<int((n_pad + threads - 1) / threads), threads, 0, st>>>(
        zs, n, n_pad, dv.s, split ? split_kp(dv.s) : dv.kpad, dv.bounds,
        algo == 1 ? w.ztiles : nullptr, w.win_tc, w.win32, dv.s_pad, dv.atoms64, dv.d,
        algo == 1 ? w.init_tc : nullptr, split ? 1 : hi32 ? 2 : 0);
    CBB_CUDA_TRY(cudaGetLastError());
    ZSource zr = zs;  // IPG mode: later kernels read Z from z_out
    timing_mark(0, st);
    int nsplit = 1;  // atom ranges of the screen (candidate lists: kParts per range)
    int rc = split ? (split_kp(dv.s) == 64 ? launch_tc<64, true>(w, n, zr, dv, o, max_ctas, st, &nsplit)
                                           : launch_tc<128, true>(w, n, zr, dv, o, max_ctas, st, &nsplit))
             : hi32 ? (dv.kpad == 32 ? launch_tc<32, false, true>(w, n, zr, dv, o, max_ctas, st, &nsplit)
                                     : launch_tc<64, false, true>(w, n, zr, dv, o, max_ctas, st, &nsplit))
             : (algo == 1) ? (dv.kpad == 32 ? launch_tc<32>(w, n, zr, dv, o, max_ctas, st, &nsplit)
                                            : launch_tc<64>(w, n, zr, dv, o, max_ctas, st, &nsplit))
                           : dispatch_ffma(w, n, zr, dv, o, st);
    if (rc) return rc;
    timing_mark(1, st);
    if (algo == 1) {
      CBB_DISPATCH_S(dv.s_pad, rc = launch_rescore<S_>(w, n, zr, dv, o, st, kParts * nsplit);
                     break);
      if (rc) return rc;
      count_launches(2);
    }
    count_launches(4);  // prologue, screening kernel, exhaustive rescan (split + finish)
    rc = launch_exhaustive_list(n, zr, dv, w.ovf_count, w.ovf_list, w.win32, w.exh_partial, o,
                                st);
    if (rc) return rc;
  } else if (algo == 3) {
    if (zs.x != nullptr) {
      // materialise Z = X - mu G (same fp32 rounding as the prologue)
      const int64_t n_pad = n;
      prologue_kernel<<<int((n_pad + 255) / 256), 256, 0, st>>>(zs, n, n_pad, dv.s, dv.kpad,
                                                               dv.bounds, nullptr, nullptr,
                                                               nullptr, dv.s_pad, dv.atoms64,
                                                               dv.d, nullptr, 0);
      CBB_CUDA_TRY(cudaGetLastError());
    }
    int rc = launch_exhaustive(n, zs, dv, nullptr, nullptr, o, st);
    if (rc) return rc;
    count_launches(zs.x != nullptr ? 2 : 1);
  } else {
    return kErrArgument;
  }
  if (nd_sum) {
    count_launches(2);
    return reduce_sum(o.nd_v, n, w.partial, nd_sum, st);
  }
  return kOk;
}

int project_overflow_count(void* ws_ptr, int64_t n, int s, int* host_count, cudaStream_t st) {
  ProjWs w;
  project_ws_bytes(n, s, &w, ws_ptr);
  CBB_CUDA_TRY(cudaMemcpyAsync(host_count, w.ovf_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBB_CUDA_TRY(cudaStreamSynchronize(st));
  return kOk;
}

int project_overflow_counts(void* ws_ptr, int64_t n, int s, int* host2, cudaStream_t st) {
  ProjWs w;
  project_ws_bytes(n, s, &w, ws_ptr);
  CBB_CUDA_TRY(cudaMemcpyAsync(host2, w.ovf_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBB_CUDA_TRY(cudaMemcpyAsync(host2 + 1, w.heavy_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBB_CUDA_TRY(cudaStreamSynchronize(st));
  return kOk;
}

int tc_debug_scores(const void* ztiles, const void* atiles, int kpad, int s, int a_tile,
                    int b_tile, float* out, cudaStream_t st) {
  const int tile_bytes = kTileRows * kpad * 2;
  const int smem = tile_bytes + 64 + 1024;
  const int nc = tc_nc(s);
  if (kpad == 32) {
    CBB_CUDA_TRY(cudaFuncSetAttribute(tc_debug_scores_kernel<32>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_debug_scores_kernel<32><<<1, 128, smem, st>>>(static_cast<const uint8_t*>(ztiles),
                                                      static_cast<const uint8_t*>(atiles), nc,
                                                      a_tile, b_tile, out);
  } else {
    CBB_CUDA_TRY(cudaFuncSetAttribute(tc_debug_scores_kernel<64>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_debug_scores_kernel<64><<<1, 128, smem, st>>>(static_cast<const uint8_t*>(ztiles),
                                                      static_cast<const uint8_t*>(atiles), nc,
                                                      a_tile, b_tile, out);
  }
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

#ifdef CBB_TRACE
int trace_dump(long long* host, int count) {
  if (count < 0) {  // per-voxel-tile stamps (256 x 4)
    CBB_CUDA_TRY(cudaMemcpyFromSymbol(host, g_trace_vt, sizeof(long long) * 4 * 256));
    return kOk;
  }
  CBB_CUDA_TRY(cudaMemcpyFromSymbol(host, g_trace, sizeof(long long) * 8 * count));
  return kOk;
}
#else
int trace_dump(long long*, int) { return kErrUnsupported; }
#endif

int prologue_only(const ZSource& zs, int64_t n, const DictView& dv, void* ws_ptr,
                  cudaStream_t st) {
  ProjWs w;
  project_ws_bytes(n, dv.s, &w, ws_ptr);
  const int64_t n_pad = ((n + kVoxPad - 1) / kVoxPad) * kVoxPad;
  prologue_kernel<<<int((n_pad + 255) / 256), 256, 0, st>>>(zs, n, n_pad, dv.s, dv.kpad,
                                                             dv.bounds, w.ztiles, w.win_tc,
                                                             w.win32, dv.s_pad, dv.atoms64, dv.d,
                                                             w.init_tc, 0);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

}  // namespace cbb

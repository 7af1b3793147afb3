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
#include <algorithm>
#include <atomic>
#include <utility>
#include <vector>

#include <cub/cub.cuh>

namespace cbb {

// ============================================================== helpers
// compile-time width for the fp64 scoring loops (s_pad; 0 = runtime loop for s > 32)
#define CBB_DISPATCH_S(s_pad, ...)          \
  switch (s_pad) {                          \
    case 2: { constexpr int S_ = 2; __VA_ARGS__; }   \
    case 4: { constexpr int S_ = 4; __VA_ARGS__; }   \
    case 6: { constexpr int S_ = 6; __VA_ARGS__; }   \
    case 8: { constexpr int S_ = 8; __VA_ARGS__; }   \
    case 10: { constexpr int S_ = 10; __VA_ARGS__; } \
    case 12: { constexpr int S_ = 12; __VA_ARGS__; } \
    case 16: { constexpr int S_ = 16; __VA_ARGS__; } \
    case 20: { constexpr int S_ = 20; __VA_ARGS__; } \
    case 24: { constexpr int S_ = 24; __VA_ARGS__; } \
    case 32: { constexpr int S_ = 32; __VA_ARGS__; } \
    default: { constexpr int S_ = 0; __VA_ARGS__; }  \
  }

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

// np.argmax order on (score, index): NaN is the maximum (the first NaN wins), then the larger
// score, then the lower index (projection.py:62 on rows with non-finite scores).
__device__ __forceinline__ bool argmax_better(double a, int64_t ja, double b, int64_t jb) {
  const bool na = a != a, nb = b != b;
  if (na || nb) return na && (!nb || ja < jb);
  return a > b || (a == b && ja < jb);
}

// Rows with a non-finite component: the reference's score block Re(Z @ D^H) (projection.py:61,
// numpy -> OpenBLAS zgemm) is NaN for EVERY atom of such a row (the complex kernel multiplies
// the infinite component by zero parts), so np.argmax returns atom 0; gamma is then
// _gammas_for's einsum with atom 0 (projection.py:38-42), i.e. the plain fp64 dot.
template <int S>
__device__ __forceinline__ bool nonfinite_row(const double* zr, const double* zi, int s) {
  bool bad = false;
  if constexpr (S > 0) {
#pragma unroll
    for (int k = 0; k < S; ++k)
      if (k < s) bad |= !isfinite(zr[k]) || !isfinite(zi[k]);
  } else {
    for (int k = 0; k < s; ++k) bad |= !isfinite(zr[k]) || !isfinite(zi[k]);
  }
  return bad;
}

__device__ void write_winner(const ProjOut& out, const DictView& dv, int64_t v, int64_t j,
                             double score) {
  const int s = dv.s;
  // np.maximum(score, 0) (projection.py:42): NaN propagates
  const double gamma = score != score ? score : (score > 0.0 ? score : 0.0);
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

// The score column of slot `slot` sits kCandCap * STRIDE words after its index column (kOffCs =
// kOffCj + kCandCap * kSlots * 4), so the list carries one shared pointer; STRIDE and the global
// stride are compile-time / kernel constants (fewer live registers in the screen's epilogue).
template <int STRIDE>
struct HCandList {
  int* cj;           // shared-memory list, column layout [kCandCap][STRIDE], scores after it
  int cnt;
  int2* gbase;       // global spill list
  int64_t gstride;
  int gcnt;
  bool ovf;

  __device__ __forceinline__ float* cs() const {
    return reinterpret_cast<float*>(cj + kCandCap * STRIDE);
  }

  __device__ __forceinline__ void insert(int j, float sc, float thr) {
    if (cnt == kCandCap) {
      cnt = cand_compact(cj, cs(), STRIDE, thr);
      if (cnt == kCandCap) {
        const int g = hcand_spill(cj, cs(), STRIDE, cnt, gbase, gstride, gcnt, thr);
        if (g < 0) {
          ovf = true;
          return;
        }
        gcnt = g;
        cnt = 0;
      }
    }
    cs()[cnt * STRIDE] = sc;
    cj[cnt * STRIDE] = j;
    ++cnt;
  }

  // hand-off: append the surviving shared entries to the global list; returns the total or
  // -1 on overflow
  __device__ __forceinline__ int finish(float thr) {
    if (ovf) return -1;
    for (int c = 0; c < cnt; ++c) {
      const float x = cs()[c * STRIDE];
      if (x >= thr) {
        if (gcnt == kGCap) gcnt = gcand_compact(gbase, gstride, gcnt, thr);
        if (gcnt == kGCap) return -1;
        gbase[(gcnt++) * gstride] = make_int2(cj[c * STRIDE], __float_as_int(x));
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
// Explicit-atom record (split screen: usually one or two atoms of a recorded chunk are inside
// the narrow window): bit 31 set, the first atom's offset inside the chunk in bits [20, 25), a
// second one in bits [25, 30) when bit 30 is set; no group mask.
constexpr uint32_t kExplicitAtoms = 1u << 31;
__device__ __forceinline__ int pack_atoms(int64_t jb, uint32_t in) {  // popc(in) in {1, 2}
  const uint32_t a = uint32_t(__ffs(in) - 1);
  const uint32_t rest = in & (in - 1);
  uint32_t x = uint32_t(jb >> 5) | (a << 20) | kExplicitAtoms;
  if (rest) x |= (uint32_t(__ffs(rest) - 1) << 25) | (1u << 30);
  return int(x);
}
// (first atom of the record, 32-bit mask of the atoms to rescore relative to it)
__device__ __forceinline__ void unpack_record(int x, int64_t& j0, uint32_t& atoms) {
  const uint32_t u = uint32_t(x);
  j0 = int64_t(u & ((1u << kChunkShift) - 1)) << 5;
  if (u & kExplicitAtoms) {
    atoms = 1u << ((u >> 20) & 31u);
    if (u & (1u << 30)) atoms |= 1u << ((u >> 25) & 31u);
    return;
  }
  const uint32_t g = (u >> kChunkShift) & 0x3Fu;  // 6-atom groups (the last one: atoms 30, 31)
  atoms = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b)
    if (g & (1u << b)) atoms |= 0x3Fu << (6 * b);
  if (g & (1u << 5)) atoms |= 3u << 30;
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
// perm (coherent dictionaries): row p holds atom perm[p] (bisection order); null: row p = atom p.
__global__ void prep_tc2_kernel(const double2* __restrict__ atoms64, int64_t d, int64_t d_pad,
                                int s, const int32_t* __restrict__ perm,
                                uint8_t* __restrict__ atoms_tc2, float* __restrict__ bounds) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= d_pad) return;
  const int kp = split_kp(s), rows = split_rows(kp);
  const int tile = int(p / rows), r = int(p % rows);
  uint8_t* trow = atoms_tc2 + size_t(tile) * rows * kp * 2;
  auto put = [&](int e, unsigned short h) {
    *reinterpret_cast<unsigned short*>(trow + split_elem_offset(r, e, rows)) = h;
  };
  const int64_t j = p >= d ? d : (perm ? int64_t(perm[p]) : p);
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

// Centroid rows of the tile-pruning bound pass: row t = split-operand row of the fp32 centroid c_t
// (same layout and scale_d as prep_tc2_kernel, no bound updates: the bound pass carries its own
// margin), rs[t] = ru(scale_d r_t); rows >= nt are sentinel rows (score -65504).
// Folded bound (tile pruning): when the split rows have three spare K columns after the sentinel
// (6s + 4 <= kp: every s <= 20 except none; s = 21 has one), the bound pass's test
//   fl(zn r_t + s~) >= lb'   becomes the sign of one accumulator: the voxel rows carry
//   [ru16(zn), hi16(lb'), lo16(lb')] in those columns (hi + lo <= lb', lo rounded down) and the
//   centroid rows [ru16(scale_d r_t), -1, -1], so the MMA returns s~ + zn r_t - lb' itself (the
//   products are exact in the fp32 accumulator; ru / rd only loosen the bound, the truncation of
//   the K = 16 step that holds them, <= 16 x 2^-24 x 2^13, is far inside lb's margin of >= 1).
//   Atom rows are zero in these columns: the screens are unchanged.
__host__ __device__ constexpr bool bound_folds(int s) { return 6 * s + 4 <= split_kp(s); }
__device__ __forceinline__ unsigned short f16_bits_ru(float x) {
  return __half_as_ushort(__float2half_ru(x));
}
__device__ __forceinline__ unsigned short f16_bits_rd(float x) {
  return __half_as_ushort(__float2half_rd(x));
}

__global__ void prep_ctr_kernel(const float* __restrict__ cen, const float* __restrict__ rad,
                                int nt, int rows_alloc, int s, int sp,
                                const float* __restrict__ bounds, uint8_t* __restrict__ out,
                                float* __restrict__ rs) {
  const int t = int(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows_alloc) return;
  const int kp = split_kp(s), rows = split_rows(kp);
  uint8_t* trow = out + size_t(t / rows) * rows * kp * 2;
  const int r = t % rows;
  auto put = [&](int e, unsigned short h) {
    *reinterpret_cast<unsigned short*>(trow + split_elem_offset(r, e, rows)) = h;
  };
  if (t >= nt) {
    put(6 * s, kF16MinusMax);
    rs[t] = 0.f;
    return;
  }
  const double sc = dict_scale(bounds);
  rs[t] = __double2float_ru(double(rad[t]) * sc);
  if (bound_folds(s)) {
    put(6 * s + 1, f16_bits_ru(rs[t]));
    put(6 * s + 2, 0xBC00);  // -1.0
    put(6 * s + 3, 0xBC00);
  }
  for (int k = 0; k < s; ++k) {
    const double x[2] = {double(cen[size_t(t) * 2 * sp + k]) * sc,
                         double(cen[size_t(t) * 2 * sp + sp + k]) * sc};
    for (int c = 0; c < 2; ++c) {
      const unsigned short hi = f16_bits_rn(x[c]);
      const unsigned short lo = f16_bits_rn(x[c] - f16_bits_to_double(hi));
      const int e = c * s + k;
      put(e, hi);
      put(2 * s + e, hi);
      put(4 * s + e, lo);
    }
  }
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
// S > 0: compile-time signature length (the BASELINE ranks 10 and 20): the component loops unroll
// and the fp16 row stays in registers; S == 0: runtime s.  Same arithmetic in the same order.
// SP: the split flag at compile time too (with S > 0 the row width and every row index are
// constants); -1: runtime.
template <int S, int SP = -1>
__global__ void prologue_kernel(ZSource zs, int64_t n, int64_t n_pad, int s_arg, int kpad_arg,
                                const float* __restrict__ bounds, uint8_t* __restrict__ ztiles,
                                float* __restrict__ win_tc, float* __restrict__ win32,
                                int s_pad, const double2* __restrict__ atoms64,
                                int64_t d_atoms, float* __restrict__ init_tc, int split_arg,
                                float2* __restrict__ lbz, int32_t* __restrict__ hbest) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n_pad) return;
  const int s = S > 0 ? S : s_arg;
  const int split = SP >= 0 ? SP : split_arg;
  const int kpad = (S > 0 && SP >= 0) ? (SP == 1 ? split_kp(S) : (2 * S < 32 ? 32 : 64)) : kpad_arg;
  const float mu = zs.mu_ptr ? *zs.mu_ptr : zs.mu;
  // tile pruning: (exact hint score rounded down, ||z|| rounded up); zero and non-finite voxels
  // are decided without the screen (+inf: they need no atom tile)
  if (lbz && v < n) lbz[v] = make_float2(INFINITY, 0.f);
  if (hbest && v < n) hbest[v] = zs.hint ? zs.hint[v] : -1;
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
#pragma unroll
  for (int k = 0; k < s; ++k) {
    double re, im;
    if (zs.x != nullptr) {
      const float2 xk = zs.x[v * s + k], gk = zs.g[v * s + k];
      const float zr = __fmaf_rn(-mu, gk.x, xk.x), zi = __fmaf_rn(-mu, gk.y, xk.y);
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
#pragma unroll
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
#pragma unroll
  for (int k = 0; k < s; ++k) {
    double re, im;
    if (zs.x != nullptr) {
      const float2 xk = zs.x[v * s + k], gk = zs.g[v * s + k];
      re = __fmaf_rn(-mu, gk.x, xk.x);
      im = __fmaf_rn(-mu, gk.y, xk.y);
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
#pragma unroll
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
    int64_t jh = zs.hint ? int64_t(zs.hint[v]) : -1;
    if (!(jh >= 0 && jh < d_atoms)) jh = -1;
    double acc = -INFINITY;
    if (jh >= 0) acc = exact_score_g(zs, v, s, atoms64 + jh * s);
    const int64_t j2 = zs.hint2 ? int64_t(zs.hint2[v]) : -1;
    if (j2 >= 0 && j2 < d_atoms && j2 != jh) {  // any atom's exact score is a lower bound
      const double a2 = exact_score_g(zs, v, s, atoms64 + j2 * s);
      if (jh < 0 || a2 > acc) {
        acc = a2;
        jh = j2;
      }
    }
    if (hbest) hbest[v] = int32_t(jh);
    float2 lz = make_float2(-INFINITY, __double2float_ru(sqrt(nz) * sv));
    if (jh >= 0) {
      init = __double2float_rd(acc * sv * sd - eb * 1.001);
      // scaled units of the tile-pruning bound pass (see prune_prepare)
      lz.x = __double2float_rd(acc * sv * sd - 0x1p-11 * double(lz.y) * sd * dmax);
    }
    if (lbz) {
      lbz[v] = lz;
      if (split == 1 && bound_folds(s)) {  // folded bound columns (see bound_folds)
        // no hint (lb = -inf): -65504 keeps every tile (|s~| <= 2^13); infinities never enter
        // the rows (inf x 0 against the atom rows' zero columns would poison the screen)
        const bool fin = fabsf(lz.x) <= 60000.f;
        const unsigned short hi = fin ? __half_as_ushort(__float2half_rn(lz.x))
                                      : (lz.x > 0.f ? 0x7BFF : 0xFBFF);
        const float rem = fin ? lz.x - __half2float(__ushort_as_half(hi)) : 0.f;
        unsigned short* fold = reinterpret_cast<unsigned short*>(trow) + 6 * s + 1;
        fold[0] = f16_bits_ru(lz.y);
        fold[1] = hi;
        fold[2] = f16_bits_rd(rem);
      }
    }
    init_tc[v] = init;
  }
}


// prologue launch: compile-time signature length for the BASELINE ranks
#define CBB_PROLOGUE(GRID, THREADS, ST, SVAL, SPLITVAL, KPVAL, ...)                            \
  do {                                                                                         \
    const int sv_ = (SVAL), sp_ = (SPLITVAL), kp_ = (KPVAL);                                   \
    if (sv_ == 10 && sp_ == 1 && kp_ == 64)                                                    \
      prologue_kernel<10, 1><<<(GRID), (THREADS), 0, (ST)>>>(__VA_ARGS__);                     \
    else if (sv_ == 10 && sp_ == 0 && kp_ == 32)                                               \
      prologue_kernel<10, 0><<<(GRID), (THREADS), 0, (ST)>>>(__VA_ARGS__);                     \
    else if (sv_ == 20 && sp_ == 1 && kp_ == 128)                                              \
      prologue_kernel<20, 1><<<(GRID), (THREADS), 0, (ST)>>>(__VA_ARGS__);                     \
    else if (sv_ == 20 && sp_ == 0 && kp_ == 64)                                               \
      prologue_kernel<20, 0><<<(GRID), (THREADS), 0, (ST)>>>(__VA_ARGS__);                     \
    else                                                                                       \
      prologue_kernel<0><<<(GRID), (THREADS), 0, (ST)>>>(__VA_ARGS__);                         \
  } while (0)

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
      if (argmax_better(acc, j, bs, best)) { bs = acc; best = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double obs = __shfl_xor_sync(0xffffffffu, bs, o);
      int64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
      if (argmax_better(obs, ob, bs, best)) { bs = obs; best = ob; }
    }
    if (best == INT64_MAX) best = 0;  // empty dictionary slice
    if (nonfinite_row<S>(zw, zw + s, s)) {  // all-NaN reference scores: atom 0
      best = 0;
      bs = dot_atom<S>(zw, zw + s, dv.atoms64, s);
    }
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
        if (argmax_better(acc, j, bs, best)) { bs = acc; best = j; }
      }
    } else {
      const float thr32 = gmax32 - w32;
      for (int c = 0; c < ns; ++c) {
        const int2 e2 = surv[c];
        if (__int_as_float(e2.y) < thr32) continue;
        const int64_t j = e2.x;
        const double acc = dot_atom<S>(zw, zw + s, dv.atoms64 + j * s, s);
        if (argmax_better(acc, j, bs, best)) { bs = acc; best = j; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double obs = __shfl_xor_sync(0xffffffffu, bs, o);
      const int64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
      if (argmax_better(obs, ob, bs, best)) { bs = obs; best = ob; }
    }
    if (lane == 0) partial[pr] = make_double2(bs, __longlong_as_double(best));
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) exhaustive_finish_kernel(ZSource zs, DictView dv,
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
    if (argmax_better(p.x, j, bs, best)) { bs = p.x; best = j; }
  }
  if (best == INT64_MAX) best = 0;  // empty dictionary
  const int64_t v = list[i];
  bool bad = false;
  double acc = 0.0;
  for (int k = 0; k < dv.s; ++k) {  // non-finite row: all-NaN reference scores -> atom 0
    const double2 z = load_z(zs, v, dv.s, k);
    bad |= !isfinite(z.x) || !isfinite(z.y);
    acc = fma(z.x, dv.atoms64[k].x, acc);
    acc = fma(z.y, dv.atoms64[k].y, acc);
  }
  if (bad) {
    best = 0;
    bs = acc;
  }
  write_winner(out, dv, v, best, bs);
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
template <int KP, bool SPLIT = false>
struct TcCfg {
  static_assert(!SPLIT || KP == 64 || KP == 128, "split tiles are 64 or 128 wide");
  static constexpr bool kF32 = SPLIT;  // fp32 accumulators, fp32 epilogue
  // 32-atom chunks per tile (split: the tile is one split_rows(KP)-row storage tile)
  static constexpr int kChunks = SPLIT ? split_rows(KP) / 32 : (KP == 32 ? 5 : 4);
  static constexpr int BN = 32 * kChunks;                    // 160 (KP 32) / 128 / 64 (split)
  static constexpr int kACols = KP / 2;                      // packed fp16 pairs per lane
  static constexpr int kAcc = 3;                             // x BN accumulator columns
  static constexpr int kAccCols = BN;
  static constexpr int kAColOff = kAcc * kAccCols;           // A buffers after the stages
  static_assert(kAColOff + 2 * kACols <= 512, "TMEM budget");
  static constexpr int kRowBytes = (KP < 64 ? KP : 64) * 2;   // bytes per row of a K block
  static constexpr int kBlk = KP <= 64 ? 1 : KP / 64;         // K blocks per tile
  // split tiles in global memory (= the ring's stage stride); the fp16 screens copy only
  // tc_nc(s) 16-byte chunks per row (tile_bytes / copy_bytes in the kernel)
  static constexpr int kBTileBytes = BN * KP * 2;
  static constexpr int kBBytes = kBTileBytes;
  static_assert(BN % 8 == 0, "8-row swizzle groups");
  static constexpr int kRing = (KP == 32 ? 96 : 144) * 1024;
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
  static constexpr int kOffCs = kOffCj + kCandCap * kSlots * 4;  // = HCandList::cs()
  static constexpr int kOffPthr = kOffCs + kCandCap * kSlots * 4;  // [kVox][4] u32 thresholds
  static constexpr int kOffBar = kOffPthr + kVox * 16;
  // completion barriers per tile slot k % kTBars (lcm(kAcc, kParts)): every barrier belongs to
  // one stage AND one part, whose waits consume its phases in order (no parity aliasing)
  static constexpr int kTBars = (kAcc % kParts == 0) ? kAcc : kAcc * kParts;
  // split screen on 128-atom tiles: each accumulator stage is two 64-column halves with their
  // own MMAs (N = 64), commits and releases, so the first half refills while the part loads the
  // second (the 64 fp32 scores of one half fill the part's registers)
  static constexpr bool kHalves = SPLIT && kChunks == 4;
  static constexpr int kNumBars = 4 + 2 * kStages + (kHalves ? 2 : 1) * (kTBars + kAcc);
  static_assert(kStages % kParts == 0, "barrier ownership");
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffTmem + 16 + 1024;  // + alignment slack
  static_assert(kSmem <= 227 * 1024, "shared memory");
  static constexpr uint32_t kIdesc = kF32 ? idesc_f16_f32(128, BN) : idesc_f16_f16(128, BN);
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
template <class CL>
__device__ __forceinline__ void record_chunk(const uint32_t* r, __half cm, int64_t jb, __half thr,
                                             float thr_f, CL& cl) {
  uint32_t mask = __hge(hmax_halves(as_h2(r[15])), thr) ? (1u << 5) : 0u;
#pragma unroll
  for (int i = 0; i < 5; ++i)
    mask |= __hge(hmax_halves(hmax3(as_h2(r[3 * i]), as_h2(r[3 * i + 1]), as_h2(r[3 * i + 2]))),
                  thr)
                ? (1u << i)
                : 0u;
  cl.insert(pack_chunk(jb, mask), __half2float(cm), thr_f);
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

template <int NC, class CL>
__device__ __forceinline__ void screen_tile(const uint32_t (&r)[16 * NC], int64_t jb, float win,
                                            __half& runmax, __half& thr, bool& active,
                                            CL& cl, uint32_t* pub, uint32_t tag,
                                            const uint32_t* pthr_row) {
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
  // warp-uniform test against the part's own threshold: the fast path carries no divergent
  // branch, no shared-memory read and no reconvergence
  if (__any_sync(0xffffffffu, __hge(cm, thr))) {
    // the other parts' published thresholds (any of them bounds the window edge from below)
    // are read only here, where they can still turn the tile back into a fast one
    thr = __hmax(thr, shared_thr(lds_v4_volatile(pthr_row), tag));
    if (__any_sync(0xffffffffu, __hge(cm, thr)) && __hge(cm, thr)) {
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

template <class CL>
__device__ __forceinline__ void record_chunk_f32(const uint32_t* r, float cm, int64_t jb,
                                                 float thr, CL& cl) {
  uint32_t in = 0;  // atoms of the chunk inside the window
#pragma unroll
  for (int i = 0; i < 32; ++i) in |= (__uint_as_float(r[i]) >= thr ? 1u : 0u) << i;
  if (__popc(in) <= 2) {  // the usual case with the split screen's 2^-18 window
    cl.insert(pack_atoms(jb, in), cm, thr);
    return;
  }
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

template <int NC, class CL>
__device__ __forceinline__ void screen_tile_f32(const uint32_t (&r)[32 * NC], int64_t jb,
                                                float win, float& runmax, float& thr,
                                                bool& active, CL& cl) {
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
// range arithmetic folds away (nsplit = 1).
// PRUNE (split screen, IPG warm start): the voxel tiles are formed in screen order (voxel vperm[p]
// at row p % 128 of tile p / 128) and each screens only the atom tiles its prune list holds
// (prune_kernel: tiles that may contain a voxel's argmax); a work unit (voxel tile, range hr)
// takes the list slice [pcnt c hr / nsplit, c (hr + 1) / nsplit).
// BOUND (the pruning pass itself): `dv` holds the split tiles of the atom-tile CENTROIDS; per
// (voxel, centroid) the epilogue tests the Cauchy-Schwarz bound s~ + zn r >= lb (scaled units,
// lbz = (lb - margin, zn) per voxel, bnd_rs = r per centroid) and ORs the voxel tile's need bits
// into bnd_bits[vt][bnd_words] (see prune_prepare).
template <int KP, bool SPLIT, bool RANGES = false, bool PRUNE = false, bool BOUND = false>
__global__ void __launch_bounds__(TcCfg<KP, SPLIT>::kThreads, 1)
    mf_tc_kernel(const uint8_t* __restrict__ zrows, int64_t n, int n_vt,
                 const float* __restrict__ win_tc, const float* __restrict__ init_tc,
                 DictView dv, int64_t n_pad, int2* __restrict__ cand, int2* __restrict__ meta,
                 const uint8_t* __restrict__ hint_tiles, int n_hint, int nsplit_arg,
                 const int32_t* __restrict__ vperm, const int* __restrict__ pcnt,
                 const uint16_t* __restrict__ plist, int plist_stride,
                 const float2* __restrict__ lbz, const float* __restrict__ bnd_rs,
                 uint32_t* __restrict__ bnd_bits, int bnd_words) {
  using C = TcCfg<KP, SPLIT>;
  static_assert(!PRUNE || SPLIT, "pruned lists index the split tiles");
  static_assert(!BOUND || (SPLIT && !RANGES && !PRUNE), "bound pass: split tiles, whole list");
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

  // warp index through a lane-0 shuffle: provably warp-uniform, so per-warp addresses (TMEM
  // stages, barriers, descriptors) stay in uniform registers instead of R2UR moves before every
  // tcgen05 instruction
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int64_t d = dv.d;
  const int nB = int((d + BN - 1) / BN);
  // work unit u (the CTA's units are u = blockIdx.x + it * gridDim.x): voxel tile u / nsplit,
  // atom tiles [h nBh, (h + 1) nBh) with h = u % nsplit (the last range runs into sentinel
  // tiles when nsplit does not divide nB); PRUNE: a slice of the voxel tile's list
  const int nBh = (nB + nsplit - 1) / nsplit;
  // atom tile bytes in global memory and the copy: the fp16 screens store tc_nc(s) chunks per
  // row (no-swizzle layout), the split screen full swizzled K rows
  const int nc = tc_nc(dv.s);
  const uint32_t tile_bytes = SPLIT ? uint32_t(C::kBTileBytes) : uint32_t(BN * nc * 16);
  const uint32_t copy_bytes = SPLIT ? uint32_t(C::kBBytes) : uint32_t(BN * nc * 16);
  // unpruned screens visit the atom tiles in a per-CTA rotated order (spreads L2 traffic)
  const int rot = (PRUNE || BOUND) ? 0 : int((int64_t(blockIdx.x) * nBh) / gridDim.x);
  const int my_vts = (n_vt * nsplit - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);
  // per work unit: n_hint warm-start tiles (the voxel tile's own hint atoms, each hint tile
  // repeated for the kParts parts: tile qt -> hint tile qt / kParts), then its atom tiles
  struct Unit {
    int vt, hr, lo, len;  // voxel tile, atom range, first list slot / tile, atom tiles
  };
  auto unit_of = [&](int it) {
    Unit x;
    const int u = int(blockIdx.x) + it * int(gridDim.x);
    x.vt = u / nsplit;
    x.hr = u - x.vt * nsplit;
    if constexpr (PRUNE) {
      const int c = pcnt[x.vt];
      x.lo = int((int64_t(c) * x.hr) / nsplit);
      x.len = int((int64_t(c) * (x.hr + 1)) / nsplit) - x.lo;
    } else {
      x.lo = x.hr * nBh;
      x.len = nBh;
    }
    return x;
  };
  // voxel of row `row` of voxel tile vt (PRUNE: screen order); n if past the end
  auto voxel_of = [&](int vt, int row) -> int64_t {
    const int64_t p = int64_t(vt) * C::kVox + row;
    if (p >= n) return n;
    if constexpr (PRUNE || BOUND) return int64_t(vperm[p]);
    return p;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(a_full + i, 4);         // the 4 part-0 warps stage A
      mbar_init(a_empty + i, kParts);   // each issuer commits after its last tile of a voxel tile
    }
    for (int i = 0; i < C::kTBars; ++i) mbar_init(t_full + i, 1);
    // b_full: the atom tile landed (producer with tx).  acc_free: the 4 warps of the part that
    // read the accumulator stage released it.  Separate barriers: with one barrier counting
    // both, the issuer woke ~520 clk after the last release (measured), ~2x the separate waits.
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);        // the MMAs reading the stage retired
    }
    for (int i = 0; i < C::kAcc; ++i) mbar_init(acc_free + i, 4);
    if constexpr (C::kHalves) {
      for (int i = 0; i < C::kTBars; ++i) mbar_init(t_full2 + i, 1);
      for (int i = 0; i < C::kAcc; ++i) mbar_init(acc_free2 + i, 4);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
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
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 0) {
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
      int b = lane;  // this lane's next tile inside the current work unit
      for (int it = 0; it < my_vts; ++it) {
        Unit un;
        if constexpr (PRUNE) {
          un = unit_of(it);
        } else {
          const int u = int(blockIdx.x) + it * int(gridDim.x);
          un.vt = u / nsplit;
          un.hr = u - un.vt * nsplit;
          un.lo = un.hr * nBh;
          un.len = nBh;
        }
        const int T = n_hint + un.len;
        const uint8_t* hbase = hint_tiles + size_t(un.vt) * (n_hint / kParts) * tile_bytes;
        const uint16_t* lst = PRUNE ? plist + size_t(un.vt) * plist_stride + un.lo : nullptr;
        for (; b < T; b += kParts) {
          // list entry loaded before the ring wait (its latency overlaps the wait)
          int ba;
          if constexpr (PRUNE) {
            // per-CTA rotation of the list (neighbouring voxel tiles have similar lists:
            // without it all CTAs stream the same atom tiles at the same time)
            int q = b - n_hint + (int(blockIdx.x) * un.len) / int(gridDim.x);
            if (q >= un.len) q -= un.len;
            ba = b >= n_hint ? int(lst[q]) : 0;
          } else {
            ba = rot + b - n_hint;
            if (ba >= nBh) ba -= nBh;
            ba += un.lo;
          }
          mbar_wait_addr(b_empty0 + 8 * st, ph ^ 1u);
          const uint8_t* src = b < n_hint ? hbase + size_t(b / kParts) * tile_bytes
                                          : atiles + size_t(ba) * tile_bytes;
          mbar_arrive_expect_tx_addr(b_full0 + 8 * st, copy_bytes);
          bulk_g2s_addr(ring0 + st * C::kBBytes, src, copy_bytes, b_full0 + 8 * st, pol_b);
          st += kParts;
          if (st >= C::kStages) {
            st -= C::kStages;
            ph ^= 1u;
          }
        }
        b -= T;
      }
    }
  } else if (!SPLIT && !PRUNE && !BOUND && warp >= 1 && warp <= kParts) {
    // ------------------------------------------------ fp16 screen: lean MMA issuers
    // Issuer `me` owns accumulator stage me, completion barrier me and the ring stages me,
    // me + kParts, me + 2 kParts (kStages == 3 kParts): its tiles kk = me (mod kParts) of the
    // fixed-length units (T tiles each) run through a 3-way unrolled loop whose descriptors are
    // loop constants, so the release -> MMA hop is two barrier tests, a fence and the MMAs.
    static_assert(C::kStages == 3 * kParts && C::kAcc == kParts && C::kTBars == kParts,
                  "lean issuer: ring of 3 kParts stages, one accumulator stage per issuer");
    const uint32_t me = uint32_t(warp - 1);
    const int nks = mma_ksteps(dv.s);
    const uint32_t tb0 = __shfl_sync(0xffffffffu, tbase, 0);
    const uint32_t d_tm = tb0 + me * uint32_t(C::kAccCols);
    const uint32_t a_tm0 = tb0 + uint32_t(C::kAColOff);
    const uint32_t b_base = smem_u32(smem + C::kOffB);
    uint64_t bd[3][KP / 16];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int kq = 0; kq < KP / 16; ++kq)
        bd[j][kq] = umma_desc_interleave(
            b_base + (me + uint32_t(j * kParts)) * uint32_t(C::kBBytes) + kq * 256, 128,
            nc * 128);
    const uint32_t T = uint32_t(n_hint + nBh);
    const uint32_t total = uint32_t(my_vts) * T;
    uint64_t* const accf = acc_free + me;
    uint64_t* const tfull = t_full + me;
    uint32_t kk = me, uend = T, acc_par = 1u, ph = 0u;
    int it = 0;
    if (my_vts > 0) mbar_wait(a_full, 0);
    while (kk < total) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (kk < total) {
          if (kk >= uend) {  // first tile of the next unit: its A buffer
            ++it;
            uend += T;
            mbar_wait(a_full + (it & 1), (it >> 1) & 1);
          }
          const bool last = kk + kParts >= uend;
          const uint32_t a_tm = a_tm0 + uint32_t((it & 1) * C::kACols);
          uint64_t* const bfull = b_full + me + j * kParts;
          mbar_wait(bfull, ph);
          mbar_wait(accf, acc_par);
          if (lane == 0) CBB_STAMP(4, kk);
          acc_par ^= 1u;
          tc_fence_after();
          if (lane == 0) CBB_STAMP(0, kk);
          if (elect_one()) {
            tc_mma_f16_ts(d_tm, a_tm, bd[j][0], C::kIdesc, 0u);
#pragma unroll
            for (int kq = 1; kq < KP / 16; ++kq)
              if (kq < nks) tc_mma_f16_ts(d_tm, a_tm + uint32_t(kq * 8), bd[j][kq], C::kIdesc, 1u);
            CBB_STAMP(1, kk);
            tc_commit(b_empty + me + j * kParts);
            tc_commit(tfull);
            if (last) tc_commit(a_empty + (it & 1));
          }
          __syncwarp();
          kk += kParts;
        }
      }
      ph ^= 1u;
    }
  } else if (warp >= 1 && warp <= kParts) {
    // ------------------------------------------------ MMA issuers (warp-uniform, elected lane)
    const int me = warp - 1;
    const int nks = SPLIT ? split_ksteps(dv.s) : mma_ksteps(dv.s);
    const uint32_t b_base = smem_u32(smem + C::kOffB);
    static_assert(C::kAcc == kParts, "issuer i always fills accumulator stage i");
    int sacc = me;  // accumulator stage kk % kAcc
    uint32_t aphm = (1u << C::kAcc) - 1u;  // acc_free parity per stage: first use passes at once
    int tb = me;    // completion barrier kk % kTBars
    int st = me;
    uint32_t ph = 0;
    uint32_t kk = uint32_t(me), kbeg = 0;
    for (int it = 0; it < my_vts; ++it) {
      const uint32_t kend =
          kbeg + uint32_t(n_hint + (PRUNE ? unit_of(it).len : nBh));
      // every issuer owns >= 1 tile of the unit (T >= kParts): wait for its A operand
      mbar_wait(a_full + (it & 1), (it >> 1) & 1);
      for (; kk < kend; kk += kParts) {
        // operands of this tile's MMAs, computed before the waits (off the release -> MMA path)
        const uint32_t a_tm = tbase + uint32_t(C::kAColOff + ((it & 1) * C::kACols));
        const uint32_t d_tm = tbase + uint32_t(sacc * C::kAccCols);
        uint64_t bdesc[KP / 16];
#pragma unroll
        for (int kq = 0; kq < KP / 16; ++kq)
          // split: K blocks of 64 elements (128 B swizzled rows) follow each other, BN rows
          // each; fp16: no-swizzle core matrices, K step kq = chunks 2kq, 2kq + 1
          bdesc[kq] = SPLIT ? umma_desc_kmajor(b_base + st * C::kBBytes + (kq >> 2) * BN * 128, 64) +
                                  uint64_t(2 * (kq & 3))
                            : umma_desc_interleave(b_base + st * C::kBBytes + kq * 256, 128, nc * 128);
        const bool last = kk + kParts >= kend;  // this issuer's last tile of the unit
        // the atom tile usually landed long before the accumulator stage is released: test it
        // first, so the release -> MMA hop is a single barrier wait
        const uint32_t apar = (aphm >> sacc) & 1u;  // this stage use's release phase
        mbar_wait(b_full + st, ph);
        mbar_wait(acc_free + sacc, apar);
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
            if (last) tc_commit(a_empty + (it & 1));
          }
        } else if (elect_one()) {
#pragma unroll
          for (int kq = 0; kq < KP / 16; ++kq)
            if (kq < nks)
              tc_mma_f16_ts(d_tm, a_tm + uint32_t(kq * 8), bdesc[kq], C::kIdesc, kq > 0 ? 1u : 0u);
          CBB_STAMP(1, kk);
          tc_commit(b_empty + st);
          tc_commit(t_full + tb);
          // this issuer's last tile of the voxel tile: A buffer recyclable once it retires
          if (last) tc_commit(a_empty + (it & 1));
        }
        __syncwarp();
        sacc += kParts;
        if (sacc >= C::kAcc) sacc -= C::kAcc;
        tb += kParts;
        if (tb >= C::kTBars) tb -= C::kTBars;
        st += kParts;
        if (st >= C::kStages) {
          st -= C::kStages;
          ph ^= 1u;
        }
      }
      kbeg = kend;
    }
  } else if (warp >= C::kFirstEpiWarp) {
    // -------------------------------------------------- epilogue parts
    const int e = warp - C::kFirstEpiWarp;
    const int part = e >> 2, q = warp & 3;
    const int row = q * 32 + lane;  // voxel row inside the voxel tile (= TMEM lane)
    const int slot = part * C::kVox + row;
    int* cj_base = reinterpret_cast<int*>(smem + C::kOffCj);
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const uint32_t a_lane = tbase + lane_off + uint32_t(C::kAColOff);
    const uint32_t t_lane = tbase + lane_off;
    const uint32_t t_stage = t_lane + uint32_t(part * C::kAccCols);  // fp16: stage == part
    uint32_t* pthr_row = reinterpret_cast<uint32_t*>(smem + C::kOffPthr) + row * 4;

    // ---- A for the first voxel tile
    if (part == 0 && my_vts > 0) {
      const int64_t v0 = voxel_of(int(blockIdx.x) / nsplit, row);
      stage_voxel_row<KP>(zrows, v0, v0 < n, a_lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + 0);
    }

    uint32_t kk = uint32_t(part);  // this part's next tile
    int sacc = part;               // its accumulator stage kk % kAcc
    int tb = part;                 // its completion barrier kk % kTBars, phase (kk / kTBars) & 1
    uint32_t ph = 0;
    uint32_t kbeg = 0;
    for (int it = 0; it < my_vts; ++it) {
      int vt, hr, T;
      int64_t v;
      const uint16_t* lst = nullptr;
      if constexpr (PRUNE || BOUND) {
        const Unit un = unit_of(it);
        vt = un.vt;
        hr = un.hr;
        T = n_hint + un.len;
        v = voxel_of(vt, row);
        if constexpr (PRUNE) lst = plist + size_t(vt) * plist_stride + un.lo;
      } else {  // fixed-length units, identity voxel order (kept in this form: see DESIGN 4.1)
        const int u = int(blockIdx.x) + it * int(gridDim.x);
        vt = u / nsplit;
        hr = u - vt * nsplit;
        T = n_hint + nBh;
        v = int64_t(vt) * C::kVox + row;
      }
      const int opart = hr * kParts + part;  // output lists of (atom range, part)
      const bool live = v < n;
      // ---- stage the NEXT voxel tile's rows into the other A buffer (one tile ahead)
      if (part == 0 && it + 1 < my_vts) {
        const int nbuf = (it + 1) & 1;
        mbar_wait(a_empty + nbuf, (((it + 1) >> 1) & 1) ^ 1);
        tc_fence_after();
        const int un_next = (int(blockIdx.x) + (it + 1) * int(gridDim.x)) / nsplit;
        const int64_t vn = (PRUNE || BOUND) ? voxel_of(un_next, row)
                                            : int64_t(un_next) * C::kVox + row;
        stage_voxel_row<KP>(zrows, vn, vn < n, a_lane + uint32_t(nbuf * C::kACols));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full + nbuf);
      }
      if (part == 0 && q == 0 && lane == 0) CBB_STAMP_VT(0, it);
      const float win = live ? win_tc[v] : -1.f;
      bool active = live && win >= 0.f;
      HCandList<C::kSlots> cl{cj_base + slot, 0,
                              cand + int64_t(opart) * kGCap * n_pad + (live ? v : 0), n_pad, 0,
                              false};
      // running max seeded with the warm-start lower bound (-inf without a hint)
      const float init = live ? fmaxf(init_tc[v], -65504.f) : -INFINITY;
      __half runmax = active ? __float2half_rd(init) : __ushort_as_half(0xFC00);
      __half thr = active ? __float2half_rd(__half2float(runmax) - win)
                          : __ushort_as_half(0x7C00);
      // split mode: fp32 running max / threshold (thresholds rounded down)
      float runmax_f = active ? init_tc[v] : -INFINITY;
      float thr_f = active ? __fsub_rd(runmax_f, win) : INFINITY;
      // first tile of the unit: carried for pruned (variable-length) units, it T otherwise
      const uint32_t kb = PRUNE ? kbeg : uint32_t(it) * uint32_t(T);
      const uint32_t kend = kb + uint32_t(T);
      if constexpr (BOUND) {
        // per (voxel, centroid): need = fl(zn r + s~) >= lb - margin; a warp ORs its lanes' bits
        // (the tile's 32-centroid words) into the voxel tile's global need mask
        const float2 lz = live ? lbz[v] : make_float2(INFINITY, 0.f);
        uint32_t* vbits = bnd_bits + size_t(vt) * bnd_words;
        // folded form (bnd_rs == nullptr, see bound_folds): the accumulator holds
        // s~ + zn r - lb' itself, need = its sign bit clear; voxels that need nothing (zero /
        // non-finite / padding rows: lb = +inf) are masked here
        const bool fold = bnd_rs == nullptr;
        const uint32_t want = lz.x < INFINITY ? 0xffffffffu : 0u;
        for (; kk < kend; kk += kParts) {
          const int ba = int(kk - kb);  // centroid tile
          mbar_wait(t_full + tb, ph);
          tc_fence_after();
          constexpr int kRegChunks = C::kChunks < 2 ? C::kChunks : 2;
          uint32_t r[32 * kRegChunks];
          __syncwarp();
          const uint32_t ta = t_lane + sacc * uint32_t(C::kAccCols);
#pragma unroll
          for (int h = 0; h < C::kChunks / kRegChunks; ++h) {
            if (C::kHalves && h == 1) {
              mbar_wait(t_full2 + tb, ph);
              tc_fence_after();
              __syncwarp();
            }
#pragma unroll
            for (int c = 0; c < kRegChunks; ++c)
              tmem_ld32_f32(ta + uint32_t(32 * (h * kRegChunks + c)),
                            *reinterpret_cast<uint32_t(*)[32]>(r + 32 * c));
            tc_wait_ld();
            if (C::kHalves || h + 1 == C::kChunks / kRegChunks) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0)
                mbar_arrive(C::kHalves && h == 1 ? acc_free2 + part : acc_free + part);
            }
            const int col0 = ba * BN + 32 * kRegChunks * h;
            if (fold) {
#pragma unroll
              for (int c = 0; c < kRegChunks; ++c) {
                uint32_t neg = 0;  // bit 31 - i = sign of centroid i (one funnel shift each)
#pragma unroll
                for (int i = 0; i < 32; ++i) neg = __funnelshift_l(r[32 * c + i], neg, 1);
                uint32_t wbits = ~__brev(neg) & want;
                wbits = __reduce_or_sync(0xffffffffu, wbits);
                if (lane == 0 && wbits) atomicOr(vbits + (col0 >> 5) + c, wbits);
              }
              continue;
            }
            const float4* rs4 = reinterpret_cast<const float4*>(bnd_rs + col0);
#pragma unroll
            for (int c = 0; c < kRegChunks; ++c) {
              uint32_t wbits = 0;
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                const float4 rr = __ldg(rs4 + (32 * c + i) / 4);
                wbits |= (fmaf(lz.y, rr.x, __uint_as_float(r[32 * c + i])) >= lz.x ? 1u : 0u) << i;
                wbits |= (fmaf(lz.y, rr.y, __uint_as_float(r[32 * c + i + 1])) >= lz.x ? 1u : 0u)
                         << (i + 1);
                wbits |= (fmaf(lz.y, rr.z, __uint_as_float(r[32 * c + i + 2])) >= lz.x ? 1u : 0u)
                         << (i + 2);
                wbits |= (fmaf(lz.y, rr.w, __uint_as_float(r[32 * c + i + 3])) >= lz.x ? 1u : 0u)
                         << (i + 3);
              }
              wbits = __reduce_or_sync(0xffffffffu, wbits);
              if (lane == 0 && wbits) atomicOr(vbits + (col0 >> 5) + c, wbits);
            }
          }
          sacc += kParts;
          if (sacc >= C::kAcc) sacc -= C::kAcc;
          tb += kParts;
          if (tb >= C::kTBars) {
            tb -= C::kTBars;
            ph ^= 1u;
          }
        }
        kbeg = kend;
        continue;
      }
      if constexpr (!C::kF32) {
        // fp16 screen: the part owns accumulator stage `part` and completion barrier `part`
        // (kAcc == kTBars == kParts), whose phase flips every tile.  The three parts publish
        // their thresholds per voxel in shared memory, tagged with the voxel-tile iteration:
        // any part's rd(runmax - win) is a lower bound on the window edge of the voxel, so each
        // part screens against the highest one it sees (the slow path runs about half as often).
        static_assert(C::kAcc == kParts && C::kTBars == kParts, "stage = part");
        const uint32_t tag = (uint32_t(it) & 0xffffu) << 16;
        uint32_t* my_pub = pthr_row + part;
        const uint32_t khint = kb + uint32_t(n_hint);
        uint32_t r[16 * C::kChunks];
        auto consume = [&]() {
          if (q == 0 && lane == 0) CBB_STAMP(5, kk);
          mbar_wait(t_full + part, ph);
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
          if (lane == 0) mbar_arrive(acc_free + part);
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
          consume();
          screen_tile<C::kChunks>(r, int64_t(ba) * BN, win, runmax, thr, active, cl, my_pub, tag,
                                  pthr_row);
          if (q == 0 && lane == 0) CBB_STAMP(6, kk);
          ba += kParts;
          if (ba >= bend) ba -= nBh;
        }
      } else {
        // split screen: fp32 scores, at most two chunks (64 registers) in flight; wider tiles are
        // screened in halves and released after the last half is loaded
        for (; kk < kend; kk += kParts) {
          const int qt = int(kk - kb) - n_hint;  // < 0: warm-start hint tile
          int ba;
          if constexpr (PRUNE) {
            const int len = T - n_hint;
            int q = qt + (int(blockIdx.x) * len) / int(gridDim.x);  // the producer's rotation
            if (q >= len) q -= len;
            ba = qt >= 0 ? int(lst[q]) : 0;       // loaded before the wait
          } else {
            ba = rot + qt;                         // range tile (rot + qt) % nBh
            if (ba >= nBh) ba -= nBh;
            ba += hr * nBh;
          }
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
              if (lane == 0) mbar_arrive(acc_free + part);
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
      kbeg = kend;
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
// amap (split screen of a reordered dictionary): record positions -> atom indices (padded
// positions map to d); ties compare the atom indices.
template <int S>
__device__ __forceinline__ void rescore_entry(int2 en, const double* zr, const double* zi,
                                              int s, const DictView& dv,
                                              const int32_t* __restrict__ amap, int64_t& best,
                                              double& bs) {
  int64_t j0;
  uint32_t atoms;
  unpack_record(en.x, j0, atoms);
  while (atoms) {
    const int i = __ffs(atoms) - 1;
    atoms &= atoms - 1;
    const int64_t j = amap ? int64_t(amap[j0 + i]) : j0 + i;
    if (j >= dv.d) continue;
    const double acc = dot_atom<S>(zr, zi, dv.atoms64 + j * s, s);
    if (acc > bs || (acc == bs && j < best)) {
      bs = acc;
      best = j;
    }
  }
}

// One THREAD per voxel: zero voxels, overflow routing and voxels with <= kFastEntries chunk
// entries (every incoherent dictionary); heavier voxels go to the warp kernel's list.
template <int S, int NP = kParts>
__global__ void __launch_bounds__(256) rescore_fast_kernel(
    ZSource zs, DictView dv, int64_t n, int64_t n_pad, const float* __restrict__ win_tc,
    const int2* __restrict__ cand, const int2* __restrict__ meta, ProjOut out, int* ovf_count,
    int64_t* ovf_list, int* heavy_count, int64_t* heavy_list, int fast_entries, int nparts,
    const int32_t* __restrict__ amap) {
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
  // the voxel in registers (compile-time width S; S == 0: runtime s <= 32 in local memory)
  constexpr int SA = S > 0 ? S : 32;
  double zr[SA], zi[SA];
#pragma unroll
  for (int k = 0; k < SA; ++k) {
    if (k < s) {
      const double2 z = load_z(zs, v, s, k);
      zr[k] = z.x;
      zi[k] = z.y;
    }
  }
  int64_t best = INT64_MAX;
  double bs = -INFINITY;
#pragma unroll
  for (int p = 0; p < NP; ++p)
    for (int c = 0; p < nparts && c < cnt[p]; ++c) {
      const int2 en = cand[(int64_t(p) * kGCap + c) * n_pad + v];
      if (__int_as_float(en.y) >= thr) rescore_entry<S>(en, zr, zi, s, dv, amap, best, bs);
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
    const int* heavy_count, const int64_t* heavy_list, int nparts,
    const int32_t* __restrict__ amap) {
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
      uint32_t mask = 0;  // atoms of the record to rescore
      if (e < total) {
        int p, c;
        entry_part(e, cnt, p, c);
        const int2 en = cand[(int64_t(p) * kGCap + c) * n_pad + v];
        if (__int_as_float(en.y) >= thr) unpack_record(en.x, j0, mask);
      }
      const int na = __popc(mask);
      int off = na;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, off, o);
        if (lane >= o) off += y;
      }
      const int round_total = __shfl_sync(0xffffffffu, off, 31);
      off -= na;
      while (mask) {
        const int i = __ffs(mask) - 1;
        mask &= mask - 1;
        alist[off++] = amap ? amap[j0 + i] : int(j0 + i);
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
          if (__int_as_float(en.y) >= thr)
            rescore_entry<S>(en, zsh, zsh + s, s, dv, amap, best, bs);
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

// Storage layout of a prepared dictionary.
struct DictLayout {
  size_t a64, a32, tc, bounds, tc2, perm, pos, tile_c, tile_r, ctr_tc2, tile_rs, total;
  int64_t d_pad;   // rows of the tile copies (whole tiles + sentinel tiles)
  int n_tiles2, ctr_rows;  // split tiles; rows of the centroid split tiles
};

static DictLayout dict_layout(int64_t d, int s) {
  DictLayout L{};
  const int sp = s_pad_for(s) > 0 ? s_pad_for(s) : s;
  const int kp = kpad_for(s);
  const int64_t nbt = (d + kTileRows - 1) / kTileRows;
  L.d_pad = (nbt + kPadTiles) * kTileRows;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) & ~size_t(255);
    return r;
  };
  L.a64 = take(size_t(d) * s * 16);
  L.a32 = take(size_t(d) * 2 * sp * 4);
  // + sentinel tiles: the screening reads BN-row (BN <= 256) windows that may run past the last
  // 128-row tile
  L.tc = take(size_t(L.d_pad) * kp * 2);
  L.bounds = take(kBCount * sizeof(float));
  const bool sp2 = s <= kSplitMaxS;
  L.tc2 = take(sp2 ? size_t(L.d_pad) * split_kp(s) * 2 : 0);
  if (sp2) {
    const int rows = split_rows(split_kp(s));
    L.n_tiles2 = int((d + rows - 1) / rows);
    // centroid split tiles: >= kParts whole tiles (the bound pass gives every part a tile)
    const int ct = (L.n_tiles2 + rows - 1) / rows;
    L.ctr_rows = (ct > kParts ? ct : kParts) * rows;
    L.perm = take(size_t(L.d_pad) * 4);
    L.pos = take(size_t(d) * 4);
    L.tile_c = take(size_t(L.n_tiles2) * 2 * sp * 4);
    L.tile_r = take(size_t(L.n_tiles2) * 4);
    L.ctr_tc2 = take(size_t(L.ctr_rows) * split_kp(s) * 2);
    L.tile_rs = take(size_t(L.ctr_rows) * 4);
  }
  L.total = o;
  return L;
}

size_t dict_bytes(int64_t d, int s, size_t* off64, size_t* off32, size_t* offtc, size_t* offb,
                  size_t* offtc2) {
  const DictLayout L = dict_layout(d, s);
  if (offtc2) *offtc2 = L.tc2;
  if (off64) *off64 = L.a64;
  if (off32) *off32 = L.a32;
  if (offtc) *offtc = L.tc;
  if (offb) *offb = L.bounds;
  return L.total;
}

// Bisection order of the atoms (host, once per coherent dictionary): recursive split of the
// real 2s-vectors [re, im] at the median of their projection on the principal direction (power
// iteration), the left part a whole number of `leaf`-row tiles, so every split tile holds a
// compact cluster of atoms (small radius -> effective pruning bounds).  Deterministic.
static void bisection_order(const std::vector<double>& X, int64_t d, int dim, int leaf,
                            std::vector<int32_t>& order) {
  order.resize(size_t(d));
  for (int64_t i = 0; i < d; ++i) order[size_t(i)] = int32_t(i);
  std::vector<double> key(static_cast<size_t>(d), 0.0);
  std::vector<double> mean(static_cast<size_t>(dim)), v(static_cast<size_t>(dim)),
      w(static_cast<size_t>(dim));
  std::vector<std::pair<int64_t, int64_t>> stack{{0, d}};
  while (!stack.empty()) {
    const int64_t lo = stack.back().first, hi = stack.back().second;
    stack.pop_back();
    const int64_t n = hi - lo;
    if (n <= leaf) continue;
    std::fill(mean.begin(), mean.end(), 0.0);
    for (int64_t i = lo; i < hi; ++i) {
      const double* x = &X[size_t(order[size_t(i)]) * dim];
      for (int k = 0; k < dim; ++k) mean[size_t(k)] += x[k];
    }
    for (int k = 0; k < dim; ++k) mean[size_t(k)] /= double(n);
    // start: the row farthest from the mean
    double far = -1.0;
    int64_t jf = order[size_t(lo)];
    for (int64_t i = lo; i < hi; ++i) {
      const double* x = &X[size_t(order[size_t(i)]) * dim];
      double q = 0.0;
      for (int k = 0; k < dim; ++k) q += (x[k] - mean[size_t(k)]) * (x[k] - mean[size_t(k)]);
      if (q > far) {
        far = q;
        jf = order[size_t(i)];
      }
    }
    for (int k = 0; k < dim; ++k) v[size_t(k)] = X[size_t(jf) * dim + k] - mean[size_t(k)];
    for (int iter = 0; iter < 6; ++iter) {
      double nv = 0.0;
      for (int k = 0; k < dim; ++k) nv += v[size_t(k)] * v[size_t(k)];
      if (!(nv > 0.0)) break;
      std::fill(w.begin(), w.end(), 0.0);
      for (int64_t i = lo; i < hi; ++i) {
        const double* x = &X[size_t(order[size_t(i)]) * dim];
        double p = 0.0;
        for (int k = 0; k < dim; ++k) p += (x[k] - mean[size_t(k)]) * v[size_t(k)];
        for (int k = 0; k < dim; ++k) w[size_t(k)] += p * (x[k] - mean[size_t(k)]);
      }
      double nw = 0.0;
      for (int k = 0; k < dim; ++k) nw += w[size_t(k)] * w[size_t(k)];
      if (!(nw > 0.0)) break;
      nw = 1.0 / std::sqrt(nw);
      for (int k = 0; k < dim; ++k) v[size_t(k)] = w[size_t(k)] * nw;
    }
    for (int64_t i = lo; i < hi; ++i) {
      const int32_t j = order[size_t(i)];
      const double* x = &X[size_t(j) * dim];
      double p = 0.0;
      for (int k = 0; k < dim; ++k) p += (x[k] - mean[size_t(k)]) * v[size_t(k)];
      key[size_t(j)] = p;
    }
    const int64_t half = ((n / leaf + 1) / 2) * leaf;  // 0 < half < n for n > leaf
    std::nth_element(order.begin() + lo, order.begin() + lo + half, order.begin() + hi,
                     [&](int32_t a, int32_t b) {
                       return key[size_t(a)] < key[size_t(b)] ||
                              (key[size_t(a)] == key[size_t(b)] && a < b);
                     });
    stack.push_back({lo + half, hi});
    stack.push_back({lo, lo + half});
  }
}

// Centroid (fp32, planar [re | im], zero-padded to s_pad) and radius (>= max ||d_j - c||, fp64
// rounded up) of the atoms at split-tile rows [cl rows, (cl + 1) rows) (rows < d hold atoms
// perm[row]).  One warp per cluster.
template <int S>
__global__ void __launch_bounds__(128) cluster_bounds_kernel(const double2* __restrict__ atoms64,
                                                             int64_t d, int s, int sp,
                                                             const int32_t* __restrict__ perm,
                                                             int rows, int n_clusters,
                                                             float* __restrict__ cen,
                                                             float* __restrict__ rad) {
  const int cl = int(blockIdx.x) * 4 + int(threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (cl >= n_clusters) return;
  const int64_t p0 = int64_t(cl) * rows, p1 = p0 + rows < d ? p0 + rows : d;
  double sr[S], si[S];
#pragma unroll
  for (int k = 0; k < S; ++k) sr[k] = si[k] = 0.0;
  int cnt = 0;
  for (int64_t p = p0 + lane; p < p1; p += 32) {
    const double2* a = atoms64 + int64_t(perm[p]) * s;
#pragma unroll
    for (int k = 0; k < S; ++k)
      if (k < s) {
        const double2 x = a[k];
        sr[k] += x.x;
        si[k] += x.y;
      }
    ++cnt;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
#pragma unroll
    for (int k = 0; k < S; ++k) {
      sr[k] += __shfl_xor_sync(0xffffffffu, sr[k], o);
      si[k] += __shfl_xor_sync(0xffffffffu, si[k], o);
    }
  }
  float cr[S], ci[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    cr[k] = (cnt > 0 && k < s) ? float(sr[k] / cnt) : 0.f;
    ci[k] = (cnt > 0 && k < s) ? float(si[k] / cnt) : 0.f;
  }
  double r2 = 0.0;
  for (int64_t p = p0 + lane; p < p1; p += 32) {
    const double2* a = atoms64 + int64_t(perm[p]) * s;
    double q = 0.0;
#pragma unroll
    for (int k = 0; k < S; ++k)
      if (k < s) {
        const double2 x = a[k];
        const double er = x.x - double(cr[k]), ei = x.y - double(ci[k]);
        q += er * er + ei * ei;
      }
    r2 = fmax(r2, q);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
  if (lane == 0) {  // sp == S (dispatched on s_pad)
#pragma unroll
    for (int k = 0; k < S; ++k) {
      cen[size_t(cl) * 2 * sp + k] = cr[k];
      cen[size_t(cl) * 2 * sp + sp + k] = ci[k];
    }
    rad[cl] = __double2float_ru(sqrt(r2) * (1.0 + 0x1p-40));
  }
}

int dict_prepare(const void* atoms, int in128, int64_t d, int s, void* storage, DictView* view,
                 cudaStream_t st) {
  if (d <= 0 || s <= 0) return kErrArgument;
  const DictLayout L = dict_layout(d, s);
  uint8_t* base = static_cast<uint8_t*>(storage);
  CBB_CUDA_TRY(cudaMemsetAsync(base, 0, L.total, st));
  DictView v{};
  v.d = d;
  v.s = s;
  v.s_pad = s_pad_for(s) > 0 ? s_pad_for(s) : s;
  v.kpad = kpad_for(s);
  v.n_btiles = int((d + kTileRows - 1) / kTileRows);
  v.atoms64 = reinterpret_cast<double2*>(base + L.a64);
  v.atoms32 = reinterpret_cast<float*>(base + L.a32);
  v.atoms_tc = base + L.tc;
  v.bounds = reinterpret_cast<float*>(base + L.bounds);
  v.atoms_tc2 = s <= kSplitMaxS ? base + L.tc2 : nullptr;
  v.n_tiles2 = L.n_tiles2;
  const int threads = 256;
  const int blocks = int((d + threads - 1) / threads);
  prep_dict_kernel<<<blocks, threads, 0, st>>>(atoms, in128, d, s, v.s_pad,
                                                const_cast<double2*>(v.atoms64),
                                                const_cast<float*>(v.atoms32),
                                                const_cast<float*>(v.bounds));
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  if (2 * s < 64) {  // tensor-core operand tiles (+ sentinel column)
    prep_tc_kernel<<<int((L.d_pad + threads - 1) / threads), threads, 0, st>>>(
        v.atoms64, d, L.d_pad, s, const_cast<uint8_t*>(v.atoms_tc),
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
  v.prefer_split = 0;
  if (v.atoms_tc2) {
    // one-time host read of the coherence estimate (dictionary preparation synchronises once)
    float coh = 0.f;
    CBB_CUDA_TRY(cudaMemcpyAsync(&coh, v.bounds + kBCoherence, sizeof(float),
                                 cudaMemcpyDeviceToHost, st));
    CBB_CUDA_TRY(cudaStreamSynchronize(st));
    v.prefer_split = coh >= 1.0f ? 1 : 0;
  }
  const int rows2 = v.atoms_tc2 ? split_rows(split_kp(s)) : 0;
  if (v.atoms_tc2 && v.prefer_split && v.n_tiles2 <= 65536) {
    // coherent dictionary: bisection order of the split tiles (host) + pruning bounds
    std::vector<double2> h(size_t(d) * s);
    CBB_CUDA_TRY(cudaMemcpyAsync(h.data(), v.atoms64, h.size() * sizeof(double2),
                                 cudaMemcpyDeviceToHost, st));
    CBB_CUDA_TRY(cudaStreamSynchronize(st));
    const int dim = 2 * s;
    std::vector<double> X(size_t(d) * dim);
    for (int64_t j = 0; j < d; ++j)
      for (int k = 0; k < s; ++k) {
        X[size_t(j) * dim + k] = h[size_t(j) * s + k].x;
        X[size_t(j) * dim + s + k] = h[size_t(j) * s + k].y;
      }
    std::vector<int32_t> order;
    bisection_order(X, d, dim, rows2, order);
    std::vector<int32_t> perm(static_cast<size_t>(L.d_pad), int32_t(d));
    std::vector<int32_t> pos(static_cast<size_t>(d));
    for (int64_t p = 0; p < d; ++p) {
      perm[size_t(p)] = order[size_t(p)];
      pos[size_t(order[size_t(p)])] = int32_t(p);
    }
    int32_t* dperm = reinterpret_cast<int32_t*>(base + L.perm);
    int32_t* dpos = reinterpret_cast<int32_t*>(base + L.pos);
    CBB_CUDA_TRY(cudaMemcpyAsync(dperm, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice, st));
    CBB_CUDA_TRY(cudaMemcpyAsync(dpos, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice, st));
    CBB_CUDA_TRY(cudaStreamSynchronize(st));  // the host vectors die at scope exit
    v.tc2_atom = dperm;
    v.tc2_pos = dpos;
    v.tile_c = reinterpret_cast<float*>(base + L.tile_c);
    v.tile_r = reinterpret_cast<float*>(base + L.tile_r);
    v.ctr_tc2 = base + L.ctr_tc2;
    v.tile_rs = reinterpret_cast<float*>(base + L.tile_rs);
  }
  if (v.atoms_tc2) {  // split-operand tiles (after prep_tc_kernel: it publishes scale_d)
    prep_tc2_kernel<<<int((L.d_pad + threads - 1) / threads), threads, 0, st>>>(
        v.atoms64, d, L.d_pad, s, v.tc2_atom, const_cast<uint8_t*>(v.atoms_tc2),
        const_cast<float*>(v.bounds));
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(1);
  }
  if (v.tile_c) {
    int rc = kOk;
    CBB_DISPATCH_S(v.s_pad, {
      if constexpr (S_ > 0) {
        cluster_bounds_kernel<S_><<<(L.n_tiles2 + 3) / 4, 128, 0, st>>>(
            v.atoms64, d, s, v.s_pad, v.tc2_atom, rows2, L.n_tiles2,
            const_cast<float*>(v.tile_c), const_cast<float*>(v.tile_r));
      } else {
        rc = kErrUnsupported;
      }
      break;
    });
    if (rc) return rc;
    CBB_CUDA_TRY(cudaGetLastError());
    // the centroids as split-operand rows (the bound pass's B operand) + scaled radii
    prep_ctr_kernel<<<int((L.ctr_rows + threads - 1) / threads), threads, 0, st>>>(
        v.tile_c, v.tile_r, L.n_tiles2, L.ctr_rows, s, v.s_pad, v.bounds,
        const_cast<uint8_t*>(v.ctr_tc2), const_cast<float*>(v.tile_rs));
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(2);
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
  // tile pruning (split screen with a warm-start hint; only when the workspace was sized for
  // the dictionary, project_ws_bytes(..., prune_tiles > 0))
  bool prune;
  float2* lbz;          // [n] (hint score rounded down, ||z|| rounded up)
  int32_t* hbest;       // [n] the better-scoring warm-start atom (hint / hint2) per voxel
  int32_t* pkeys;       // [n] sort keys (hint atom's split-tile position) and values (voxel)
  int32_t* pkeys_out;
  int32_t* pvals;
  int32_t* vperm;       // [n] screen order: position -> voxel
  void* sort_tmp;
  size_t sort_tmp_bytes;
  int* pcnt;            // [n_vt] listed atom tiles per voxel tile
  uint16_t* plist;      // [n_vt][prune_tiles] ascending atom-tile lists
  uint32_t* pbits;      // [n_vt][words] need bits of the bound pass
};
constexpr int kReduceBlocks = 256;
constexpr int kVoxPad = 512;  // voxel tiles are padded to a multiple of the largest TC voxel tile

// prune_tiles > 0 (the dictionary's split tile count, prune-capable dictionaries only) appends
// the pruning buffers.
size_t project_ws_bytes(int64_t n, int s, ProjWs* ws, void* base_ptr, int prune_tiles) {
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
  w.ovf_count = reinterpret_cast<int*>(take(16));   // both counters in one 16-byte block:
  w.heavy_count = w.ovf_count ? w.ovf_count + 2 : nullptr;  // one memset node per projection
  w.ovf_list = reinterpret_cast<int64_t*>(take(size_t(n) * 8));
  take(16);  // (layout kept)
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
  w.prune = prune_tiles > 0 && n > 0 && n < (int64_t(1) << 31) && prune_tiles <= 65536;
  if (w.prune) {
    w.lbz = reinterpret_cast<float2*>(take(size_t(n) * 8));
    w.hbest = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
    w.pkeys = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
    w.pkeys_out = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
    w.pvals = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
    w.vperm = reinterpret_cast<int32_t*>(take(size_t(n) * 4));
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const int32_t*)nullptr, (int32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, int(n), 0, 32);
    w.sort_tmp_bytes = tb;
    w.sort_tmp = take(tb);
    const int64_t vt128 = (n + 127) / 128;
    w.pcnt = reinterpret_cast<int*>(take(size_t(vt128) * 4));
    w.plist = reinterpret_cast<uint16_t*>(take(size_t(vt128) * prune_tiles * 2));
    w.pbits = reinterpret_cast<uint32_t*>(take(size_t(vt128) * ((prune_tiles + 31) / 32 + 4) * 4));
  }
  if (ws) *ws = w;
  return o;
}

constexpr int kPruneMinTiles = 32;
constexpr int64_t kPruneMinVoxels = 8192;

// split tiles of a prune-capable dictionary (bisection-ordered, with tile bounds), else 0
int prune_tiles_of(const DictView& dv) {
  return (dv.tile_c != nullptr && dv.atoms_tc2 != nullptr) ? dv.n_tiles2 : 0;
}

// Per-device launch facts (a process may project on several GPUs): SM counts and the one-time
// dynamic shared-memory opt-ins are keyed by the current device.
constexpr int kMaxDevices = 64;
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
static int num_sms() {
  static std::atomic<int> sms[kMaxDevices];
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return 148;
  int v = sms[dev].load(std::memory_order_relaxed);
  if (v <= 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the current device only: one
// opt-in per (kernel, device), remembered in a per-kernel device bitmask.
template <auto Kernel>
static int ensure_smem_attr(int smem) {
  static std::atomic<uint64_t> done{0};
  const int dev = current_device();
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    CBB_CUDA_TRY(cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
  return kOk;
}

// Warm-start hint tiles: row r of voxel tile vt's hint block = a copy of the storage row of
// atom hint[v] (the previous IPG winner of voxel v = row r of the tile; vperm: screen order),
// in the screen's own tile layout; apos maps an atom to its split-tile storage row (null:
// identity).  Rows without a valid hint (and rows past n) copy the first padded row (score
// -65504 for every voxel).  One thread per 16-byte chunk.
__global__ void __launch_bounds__(256) hint_tiles_kernel(const int32_t* __restrict__ hint,
                                                         int64_t n, int64_t d, int n_vt, int vox,
                                                         const uint8_t* __restrict__ atiles,
                                                         int kp, int split, int bn, int nh,
                                                         const int32_t* __restrict__ vperm,
                                                         const int32_t* __restrict__ apos,
                                                         uint8_t* __restrict__ out) {
  // 16-byte chunks per row: split rows kp / 8; fp16 rows tc_nc(s), passed as kp = 8 * nc
  const int cpr = kp / 8;
  const int64_t per_vt = int64_t(nh) * bn * cpr;
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= per_vt * n_vt) return;
  const int vt = int(g / per_vt);
  const int rem = int(g - int64_t(vt) * per_vt);
  const int r = rem / cpr, c = rem - r * cpr;
  const int64_t p = int64_t(vt) * vox + r;
  int64_t j = d;
  if (r < vox && p < n) {
    const int64_t h = hint[vperm ? int64_t(vperm[p]) : p];
    if (h >= 0 && h < d) j = apos ? int64_t(apos[h]) : h;
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

// ------------------------------------------------------------ tile pruning (split screen, IPG)
// Split tile t (rows [t BN, (t+1) BN) of the bisection-ordered split tiles) has an fp32 centroid
// c_t and a radius r_t >= max_j ||d_j - c_t||.  Cauchy-Schwarz: Re<z, d_j> <= Re<z, c_t> + ||z|| r_t
// for every atom of the tile.  The voxel's lower bound lb is its hint atom's exact fp64 score
// (<= its maximum), so a tile with Re<z, c_t> + ||z|| r_t < lb holds neither the voxel's argmax
// nor a tie, and a voxel tile screens only the atom tiles some voxel of it may need.
//
// (1) Screen order: voxels sorted (stable) by (bucket of lb / (||z|| dmax), split-tile position of
//     the hint atom): voxel tiles gather voxels whose answers lie in the same region of the
//     dictionary and whose bounds are equally tight (few weak-bound voxels spoil a tile).
// (2) The bound pass (mf_tc_kernel<.., BOUND>): the centroids as split tiles on the tensor cores,
//     s~ = scale_v scale_d Re<z~, c~> with |s~ - scale_v scale_d Re<z, c>| <= 2^-16 ||z~|| (split
//     operands, fp32 accumulation, DESIGN 4.1b); the prologue stores lb' = rd(scale_v scale_d lb -
//     2^-11 zn sd dmax) and zn = ru(scale_v ||z||), bnd_rs = ru(scale_d r): the margin covers the
//     MMA error and the fp32 rounding of fl(zn r + s~) with room to spare.
// (3) prune_list_kernel: need bits -> ascending tile lists + counts.
__global__ void prune_keys_kernel(const int32_t* __restrict__ hint, int64_t n, int64_t d,
                                  const int32_t* __restrict__ apos, const float2* __restrict__ lbz,
                                  const float* __restrict__ bounds, int32_t pos_range,
                                  int32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int32_t h = hint[v];
  const float2 l = lbz[v];
  // bound tightness lb / (||z|| dmax) (scaled units: zn carries scale_v, lb scale_v scale_d)
  const float ratio = l.x / (l.y * bounds[kBScaleD] * bounds[kBDmax]);
  const int bucket = ratio >= 0.95f ? 0 : ratio >= 0.8f ? 1 : ratio >= 0.5f ? 2 : 3;
  keys[v] = bucket * pos_range + ((h >= 0 && h < d) ? apos[h] : pos_range - 1);
  vals[v] = int32_t(v);
}

// One warp per voxel tile: ascending list of the needed atom tiles (< n_tiles) and its length.
__global__ void prune_list_kernel(const uint32_t* __restrict__ bits, int words, int n_tiles,
                                  int n_vt, int* __restrict__ pcnt, uint16_t* __restrict__ plist,
                                  int plist_stride) {
  const int vt = int((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (vt >= n_vt) return;
  const uint32_t* b = bits + size_t(vt) * words;
  uint16_t* out = plist + size_t(vt) * plist_stride;
  int base = 0;
  for (int w0 = 0; w0 < words; w0 += 32) {
    const int w = w0 + lane;
    uint32_t m = w < words ? b[w] : 0u;
    if (32 * w + 32 > n_tiles) m &= (32 * w >= n_tiles) ? 0u : ((1u << (n_tiles - 32 * w)) - 1u);
    const int c = __popc(m);
    int off = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, off, o);
      if (lane >= o) off += y;
    }
    const int tot = __shfl_sync(0xffffffffu, off, 31);
    off += base - c;
    while (m) {
      out[off++] = uint16_t(32 * w + __ffs(m) - 1);
      m &= m - 1;
    }
    base += tot;
  }
  if (lane == 0) pcnt[vt] = base;
}

template <int KP>
static int launch_bound(const ProjWs& w, int64_t n, const DictView& dv, cudaStream_t st);

// Screen order + prune lists for an IPG projection with a warm-start hint (PRUNE screens).
static int prune_prepare(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                         cudaStream_t st) {
  const int threads = 256;
  const int32_t pos_range = int32_t(int64_t(dv.n_tiles2) * split_rows(split_kp(dv.s)) + 1);
  prune_keys_kernel<<<unsigned((n + threads - 1) / threads), threads, 0, st>>>(
      w.hbest, n, dv.d, dv.tc2_pos, w.lbz, dv.bounds, pos_range, w.pkeys, w.pvals);
  CBB_CUDA_TRY(cudaGetLastError());
  int bits = 1;
  while ((int64_t(1) << bits) <= 4 * int64_t(pos_range)) ++bits;
  size_t tmp = w.sort_tmp_bytes;
  CBB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, tmp, w.pkeys, w.pkeys_out, w.pvals,
                                               w.vperm, int(n), 0, bits, st));
  const int n_vt = int((n + 127) / 128);
  const int words = (dv.n_tiles2 + 31) / 32 + 4;
  CBB_CUDA_TRY(cudaMemsetAsync(w.pbits, 0, size_t(n_vt) * words * 4, st));
  const int rc = split_kp(dv.s) == 64 ? launch_bound<64>(w, n, dv, st)
                                      : launch_bound<128>(w, n, dv, st);
  if (rc) return rc;
  prune_list_kernel<<<unsigned((n_vt + 7) / 8), 256, 0, st>>>(w.pbits, words, dv.n_tiles2, n_vt,
                                                            w.pcnt, w.plist, dv.n_tiles2);
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(4);  // keys, bound pass, lists (+ the sort's own kernels)
  return kOk;
}

template <int KP, bool SPLIT, bool RANGES = false, bool PRUNE = false>
static int launch_tc_as(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                        int grid, int n_vt, cudaStream_t st, int nsplit = 1) {
  using C = TcCfg<KP, SPLIT>;
  int rc = ensure_smem_attr<mf_tc_kernel<KP, SPLIT, RANGES, PRUNE>>(C::kSmem);
  if (rc) return rc;
  int n_hint = 0;
  if (zs.hint) {  // IPG warm start: the voxel tiles' own hint atoms screened first
    const int vox = C::kVox;
    const int nh = (vox + C::BN - 1) / C::BN;
    const int kw = SPLIT ? KP : 8 * tc_nc(dv.s);  // row width (fp16 elements) as stored
    const int64_t chunks = int64_t(n_vt) * nh * C::BN * (kw / 8);
    hint_tiles_kernel<<<unsigned((chunks + 255) / 256), 256, 0, st>>>(
        PRUNE ? w.hbest : zs.hint, n, dv.d, n_vt, vox, SPLIT ? dv.atoms_tc2 : dv.atoms_tc, kw,
        SPLIT ? 1 : 0, C::BN,
        nh, PRUNE ? w.vperm : nullptr, SPLIT ? dv.tc2_pos : nullptr, w.hint_tiles);
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    n_hint = kParts * nh;
  }
  mf_tc_kernel<KP, SPLIT, RANGES, PRUNE><<<grid, C::kThreads, C::kSmem, st>>>(
      w.ztiles, n, n_vt, (const float*)w.win_tc, (const float*)w.init_tc, dv, w.n_pad, w.cand,
      w.meta, (const uint8_t*)w.hint_tiles, n_hint, nsplit, PRUNE ? w.vperm : nullptr,
      PRUNE ? w.pcnt : nullptr, PRUNE ? w.plist : nullptr, dv.n_tiles2, nullptr, nullptr,
      nullptr, 0);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// The bound pass: the centroids' split tiles screened like atom tiles (no hint tiles, no ranges).
template <int KP>
static int launch_bound(const ProjWs& w, int64_t n, const DictView& dv, cudaStream_t st) {
  using C = TcCfg<KP, true>;
  int rc = ensure_smem_attr<mf_tc_kernel<KP, true, false, false, true>>(C::kSmem);
  if (rc) return rc;
  const int n_vt = int((n + C::kVox - 1) / C::kVox);
  int ctiles = (dv.n_tiles2 + C::BN - 1) / C::BN;
  if (ctiles < kParts) ctiles = kParts;  // sentinel tiles: every part owns >= 1 tile
  DictView cv = dv;
  cv.d = int64_t(ctiles) * C::BN;
  cv.atoms_tc2 = dv.ctr_tc2;
  int grid = num_sms();
  if (grid > n_vt) grid = n_vt;
  mf_tc_kernel<KP, true, false, false, true><<<grid, C::kThreads, C::kSmem, st>>>(
      w.ztiles, n, n_vt, (const float*)w.win_tc, (const float*)w.init_tc, cv, w.n_pad, w.cand,
      w.meta, (const uint8_t*)w.hint_tiles, 0, 1, w.vperm, nullptr, nullptr, 0, w.lbz,
      bound_folds(dv.s) ? nullptr : dv.tile_rs, w.pbits, (dv.n_tiles2 + 31) / 32 + 4);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// prune: PRUNE screen (split tiles, warm-start hint, prune lists prepared by prune_prepare)
template <int KP, bool SPLIT = false>
static int launch_tc(const ProjWs& w, int64_t n, const ZSource& zs, const DictView& dv,
                     int max_ctas, cudaStream_t st, int* nsplit_out, bool prune) {
  *nsplit_out = 1;
  using C1 = TcCfg<KP, SPLIT>;
  const int n_vt = int((n + C1::kVox - 1) / C1::kVox);
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
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
      if constexpr (SPLIT) {
        if (prune)
          return launch_tc_as<KP, SPLIT, true, true>(w, n, zs, dv, units < grid ? units : grid,
                                                     n_vt, st, best);
      }
      return launch_tc_as<KP, SPLIT, true>(w, n, zs, dv, units < grid ? units : grid, n_vt, st,
                                           best);
    }
  }
  if (grid > n_vt) grid = n_vt;
  if constexpr (SPLIT) {
    if (prune) return launch_tc_as<KP, SPLIT, false, true>(w, n, zs, dv, grid, n_vt, st);
  }
  return launch_tc_as<KP, SPLIT>(w, n, zs, dv, grid, n_vt, st);
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
  exhaustive_finish_kernel<<<int((n + 255) / 256), 256, 0, st>>>(zs, dv, cnt, list, partial, out);
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
                          const ProjOut& o, cudaStream_t st, int nparts, const int32_t* amap) {
  // small projections: too few threads for the thread-per-voxel path to hide L2 latency, every
  // voxel goes to the warp kernel
  const int fast = n >= int64_t(num_sms()) * 256 ? kFastEntries : 0;
  rescore_fast_kernel<S, NP><<<int((n + 255) / 256), 256, 0, st>>>(
      zr, dv, n, w.n_pad, w.win_tc, w.cand, w.meta, o, w.ovf_count, w.ovf_list, w.heavy_count,
      w.heavy_list, fast, nparts, amap);
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
      w.heavy_count, w.heavy_list, nparts, amap);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

template <int S>
static int launch_rescore(const ProjWs& w, int64_t n, const ZSource& zr, const DictView& dv,
                          const ProjOut& o, cudaStream_t st, int nparts, const int32_t* amap) {
  return nparts == kParts
             ? launch_rescore_np<S, kParts>(w, n, zr, dv, o, st, nparts, amap)
             : launch_rescore_np<S, kParts * kMaxSplit>(w, n, zr, dv, o, st, nparts, amap);
}

int reduce_sum(const double* x, int64_t n, double* partial, double* out, cudaStream_t st) {
  reduce_stage1<<<kReduceBlocks, 256, 0, st>>>(x, n, partial);
  reduce_stage2<<<1, 256, 0, st>>>(partial, kReduceBlocks, out);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// algo: 0 = auto (split tcgen05 for coherent dictionaries with s <= 21, else tcgen05 when
// 2s < 64, else FFMA / fp64), 1 = tcgen05 (fp16 accumulators), 2 = FFMA, 3 = exhaustive fp64,
// 4 = split tcgen05 (hi/lo fp16 operands, fp32 accumulators, s <= 21).
// The split screen prunes atom tiles (prune_prepare) when the dictionary is prune-capable, a
// warm-start hint is given and the workspace was sized for it (cbb_project_workspace_bytes_dict).
int project(const ZSource& zs, int64_t n, const DictView& dv, const ProjOut& out, double* nd_sum,
            void* ws_ptr, size_t ws_bytes, int algo, int max_ctas, cudaStream_t st) {
  if (n < 0) return kErrArgument;
  ProjWs w;
  const size_t need = project_ws_bytes(n, dv.s, &w, ws_ptr, 0);
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
  if (algo == 1 && !tc_ok) return kErrUnsupported;
  if (algo == 4 && !split_ok) return kErrUnsupported;
  const bool split = algo == 4;
  if (split) algo = 1;  // same pipeline, other operand tiles / accumulator format
  if (algo == 2 && s_pad_for(dv.s) < 0) return kErrUnsupported;
  bool prune = false;
  {
    const int pt = prune_tiles_of(dv);
    if (pt > 0 && ws_bytes >= project_ws_bytes(n, dv.s, nullptr, nullptr, pt)) {
      ProjWs wp;
      project_ws_bytes(n, dv.s, &wp, ws_ptr, pt);
      // small problems are launch-latency bound: the pruning pass (sort, bound pass, lists)
      // only pays for large dictionaries and voxel counts
      if (split && zs.hint && wp.prune && dv.n_tiles2 >= kPruneMinTiles && n >= kPruneMinVoxels) {
        w = wp;
        prune = true;
      } else if (wp.prune) {  // mark the statistics of this workspace stale
        CBB_CUDA_TRY(cudaMemsetAsync(wp.pcnt, 0xff, sizeof(int), st));
      }
    }
  }
  // records of the split screen hold split-tile positions: the rescoring maps them to atoms
  const int32_t* amap = split ? dv.tc2_atom : nullptr;
  CBB_CUDA_TRY(cudaMemsetAsync(w.ovf_count, 0, 16, st));  // ovf_count and heavy_count
  if (algo == 1 || algo == 2) {
    const int64_t n_pad = ((n + kVoxPad - 1) / kVoxPad) * kVoxPad;
    const int threads = 256;
    CBB_PROLOGUE(int((n_pad + threads - 1) / threads), threads, st, dv.s, split ? 1 : 0,
        split ? split_kp(dv.s) : dv.kpad,
        zs, n, n_pad, dv.s, split ? split_kp(dv.s) : dv.kpad, dv.bounds,
        algo == 1 ? w.ztiles : nullptr, w.win_tc, w.win32, dv.s_pad, dv.atoms64, dv.d,
        algo == 1 ? w.init_tc : nullptr, split ? 1 : 0, prune ? w.lbz : nullptr,
        prune ? w.hbest : nullptr);
    CBB_CUDA_TRY(cudaGetLastError());
    ZSource zr = zs;  // IPG mode: later kernels read Z from z_out
    if (zr.x != nullptr) {
      zr.z = zr.z_out;
      zr.z128 = 0;
      zr.x = nullptr;
    }
    if (prune) {
      const int rc = prune_prepare(w, n, zr, dv, st);
      if (rc) return rc;
    }
    timing_mark(0, st);
    int nsplit = 1;  // atom ranges of the screen (candidate lists: kParts per range)
    int rc = split ? (split_kp(dv.s) == 64 ? launch_tc<64, true>(w, n, zr, dv, max_ctas, st, &nsplit, prune)
                                           : launch_tc<128, true>(w, n, zr, dv, max_ctas, st, &nsplit, prune))
             : (algo == 1) ? (dv.kpad == 32 ? launch_tc<32>(w, n, zr, dv, max_ctas, st, &nsplit, false)
                                            : launch_tc<64>(w, n, zr, dv, max_ctas, st, &nsplit, false))
                           : dispatch_ffma(w, n, zr, dv, o, st);
    if (rc) return rc;
    timing_mark(1, st);
    if (algo == 1) {
      CBB_DISPATCH_S(dv.s_pad, rc = launch_rescore<S_>(w, n, zr, dv, o, st, kParts * nsplit, amap);
                     break);
      if (rc) return rc;
      count_launches(2);
    }
    count_launches(4);  // prologue, screening kernel, exhaustive rescan (split + finish)
    rc = launch_exhaustive_list(n, zr, dv, w.ovf_count, w.ovf_list, w.win32, w.exh_partial, o,
                                st);
    if (rc) return rc;
  } else if (algo == 3) {
    ZSource zr = zs;
    if (zs.x != nullptr) {
      // materialise Z = X - mu G (same fp32 rounding as the prologue)
      const int64_t n_pad = n;
      CBB_PROLOGUE(int((n_pad + 255) / 256), 256, st, dv.s, 0, dv.kpad, zs, n, n_pad, dv.s, dv.kpad,
                                                               dv.bounds, nullptr, nullptr,
                                                               nullptr, dv.s_pad, dv.atoms64,
                                                               dv.d, nullptr, 0, nullptr,
                                                               nullptr);
      CBB_CUDA_TRY(cudaGetLastError());
    }
    int rc = launch_exhaustive(n, zr, dv, nullptr, nullptr, o, st);
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

// Tile-pruning statistics of the last projection on this workspace: listed (voxel tile, atom
// tile) pairs and all pairs; listed = -1 if that projection did not prune.  Synchronises.
int project_prune_stats(void* ws_ptr, size_t ws_bytes, int64_t n, const DictView& dv,
                        int64_t* listed, int64_t* total, cudaStream_t st) {
  *listed = -1;
  *total = 0;
  const int pt = prune_tiles_of(dv);
  if (pt <= 0 || n <= 0 || ws_bytes < project_ws_bytes(n, dv.s, nullptr, nullptr, pt)) return kOk;
  ProjWs w;
  project_ws_bytes(n, dv.s, &w, ws_ptr, pt);
  if (!w.prune) return kOk;
  const int64_t n_vt = (n + 127) / 128;
  std::vector<int> cnt(static_cast<size_t>(n_vt));
  CBB_CUDA_TRY(cudaMemcpyAsync(cnt.data(), w.pcnt, cnt.size() * 4, cudaMemcpyDeviceToHost, st));
  CBB_CUDA_TRY(cudaStreamSynchronize(st));
  if (cnt[0] < 0) return kOk;
  int64_t sum = 0;
  for (int c : cnt) sum += c;
  *listed = sum;
  *total = n_vt * int64_t(pt);
  return kOk;
}

// idx[v] = table[idx[v]] (representative -> atom index of the full dictionary)
__global__ void map_indices_kernel(int32_t* __restrict__ idx, const int32_t* __restrict__ table,
                                   int64_t n, int64_t table_len) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int32_t r = idx[v];
  idx[v] = (r >= 0 && r < table_len) ? table[r] : -1;
}
int map_indices(int32_t* idx, const int32_t* table, int64_t n, int64_t table_len, cudaStream_t st) {
  if (n <= 0) return kOk;
  map_indices_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(idx, table, n, table_len);
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return kOk;
}

// Per voxel tile (screen order) of the last pruned projection: the list length and the bound-
// tightness bucket (0: lb / (||z|| dmax) >= 0.95, 1: >= 0.8, 2: >= 0.5, 3: below) of its first
// voxel.  Diagnostic; synchronises.  counts[0] = -1 if that projection did not prune.
int project_prune_detail(void* ws_ptr, size_t ws_bytes, int64_t n, const DictView& dv,
                         int32_t* counts, int32_t* buckets, cudaStream_t st) {
  const int pt = prune_tiles_of(dv);
  if (n <= 0) return kOk;
  counts[0] = -1;
  if (pt <= 0 || ws_bytes < project_ws_bytes(n, dv.s, nullptr, nullptr, pt)) return kOk;
  ProjWs w;
  project_ws_bytes(n, dv.s, &w, ws_ptr, pt);
  if (!w.prune) return kOk;
  const int64_t n_vt = (n + 127) / 128;
  CBB_CUDA_TRY(cudaMemcpyAsync(counts, w.pcnt, size_t(n_vt) * 4, cudaMemcpyDeviceToHost, st));
  CBB_CUDA_TRY(cudaMemcpy2DAsync(buckets, 4, w.pkeys_out, 128 * 4, 4, size_t(n_vt),
                                 cudaMemcpyDeviceToHost, st));
  CBB_CUDA_TRY(cudaStreamSynchronize(st));
  const int32_t pos_range = int32_t(int64_t(dv.n_tiles2) * split_rows(split_kp(dv.s)) + 1);
  for (int64_t i = 0; i < n_vt; ++i) buckets[i] /= pos_range;
  return kOk;
}

int project_overflow_count(void* ws_ptr, int64_t n, int s, int* host_count, cudaStream_t st) {
  ProjWs w;
  project_ws_bytes(n, s, &w, ws_ptr, 0);
  CBB_CUDA_TRY(cudaMemcpyAsync(host_count, w.ovf_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBB_CUDA_TRY(cudaStreamSynchronize(st));
  return kOk;
}

int project_overflow_counts(void* ws_ptr, int64_t n, int s, int* host2, cudaStream_t st) {
  ProjWs w;
  project_ws_bytes(n, s, &w, ws_ptr, 0);
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
  project_ws_bytes(n, dv.s, &w, ws_ptr, 0);
  const int64_t n_pad = ((n + kVoxPad - 1) / kVoxPad) * kVoxPad;
  CBB_PROLOGUE(int((n_pad + 255) / 256), 256, st, dv.s, 0, dv.kpad, zs, n, n_pad, dv.s, dv.kpad,
                                                             dv.bounds, w.ztiles, w.win_tc,
                                                             w.win32, dv.s_pad, dv.atoms64, dv.d,
                                                             w.init_tc, 0, nullptr, nullptr);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

}  // namespace cbb

// Cartesian acquisition operator A = P_Omega F S_c (unitary DFT per frame, c coil maps) on
// B200, plus the SVD-subspace maps and the fused reductions that drive the IPG step rule.
//
// Reference: coverblip/forward_model.py:123-167 (apply/adjoint, cartesian_dft),
//            coverblip/dictionary.py:116-122 (compress = rows @ V, decompress = rows @ V^H),
//            coverblip/solver.py:130,135,180-190 (squared norms, residual, weighted residual).
//
// Internal layout: frame-major.  A frame stack is (L, n) complex64 with n = prod(dims) in C
// order (v = row*w + col, forward_model.py:138), so cuFFT runs one batched C2C over L
// contiguous frames; measurements are (L, c*m) complex64 (frame t, coil ci, sample i ->
// column ci*m + i, k-space index Omega_t(i); the reference's (c*m, L) transposed).
// The unitary 1/sqrt(n) is folded into the gather / compress kernels.
//
// Compressed operator ("s-channel"): A(Xc V^H) and (A^H R) V never materialise
// the (L, n) frame stack.  By linearity, FFT(sum_k Xc[:,k] conj(V[t,k])) = sum_k FFT(Xc[:,k])
// conj(V[t,k]), so the forward map FFTs the c*s channel images S_ci Xc[:,k] (c*s transforms
// instead of c*L) and the gather forms y[t, ci*m+i] = sum_k K[ci,k][Omega_t(i)] conj(V[t,k]).
// The adjoint builds each channel's k-space K[ci,k][w] = sum_{(t,i): Omega_t(i)=w} R[t,ci*m+i]
// V[t,k] deterministically from a CSR of the (fixed) pattern, inverse-FFTs c*s channels and
// combines G[v,k] = sum_ci conj(S_ci[v]) IFFT(K[ci,k])[v].  Same result as decompress -> per-
// frame FFT -> gather (compress) up to fp32 summation order.
#include "cbb_common.cuh"

#include <cufft.h>
#include <thrust/binary_search.h>
#include <thrust/execution_policy.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

#include <cmath>
#include <new>

namespace cbb {

constexpr int kRedBlocks = 256;

// ---------------------------------------------------------------- reductions (deterministic)
__device__ __forceinline__ double block_sum_256(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  double r = sh[0];
  __syncthreads();
  return r;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = NT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) finish_sum(const double* __restrict__ partial, int np,
                                                  double* __restrict__ out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += 256) acc += partial[i];
  double r = block_sum_256(acc, sh);
  if (threadIdx.x == 0) *out = r;
}

// ---------------------------------------------------------------- sampling
// mode 0: Y[t][i] = scale * F[t][Omega_t(i)]
// mode 1: partial ||scale * F[Omega]||^2 only (apply_diff denominator, solver.py:135)
// mode 2: R[t][i] = scale * F[t][Omega] - Ymeas[t][i] (+ partial of w*|R|^2), R stored as w*R
__global__ void __launch_bounds__(256) gather_kernel(const float2* __restrict__ F,
                                                     const int* __restrict__ pat, int64_t n,
                                                     int L, int m, int64_t ystride, int yoff,
                                                     float scale, int mode,
                                                     const float2* __restrict__ Ymeas,
                                                     const float* __restrict__ w,
                                                     float2* __restrict__ Y,
                                                     double* __restrict__ partial) {
  __shared__ double sh[256];
  const int64_t total = int64_t(L) * m;
  double acc = 0.0;
  for (int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * 256) {
    const int64_t t = e / m;
    const int64_t ye = t * ystride + yoff + (e - t * m);  // column ci*m + i of frame t
    const float2 f = F[t * n + pat[e]];
    float2 y = make_float2(f.x * scale, f.y * scale);
    if (mode == 2) {
      const float2 ym = Ymeas[ye];
      y.x -= ym.x;
      y.y -= ym.y;
      const float ww = w ? w[ye] : 1.f;
      acc += double(ww) * (double(y.x) * y.x + double(y.y) * y.y);
      Y[ye] = make_float2(ww * y.x, ww * y.y);
    } else {
      if (mode == 0) Y[ye] = y;
      acc += double(y.x) * y.x + double(y.y) * y.y;
    }
  }
  if (partial) {
    double r = block_sum_256(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
  }
}

// K[t][Omega_t(i)] = R[t][i]   (put_along_axis zero-fill, forward_model.py:160-162); K zeroed first
__global__ void __launch_bounds__(256) scatter_kernel(const float2* __restrict__ R,
                                                      const int* __restrict__ pat, int64_t n,
                                                      int L, int m, int64_t rstride, int roff,
                                                      float2* __restrict__ K) {
  const int64_t total = int64_t(L) * m;
  for (int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * 256) {
    const int64_t t = e / m;
    K[t * n + pat[e]] = R[t * rstride + roff + (e - t * m)];
  }
}

// Exact e / m for 0 <= e < 2^32, m >= 2: floor(e * ceil(2^64 / m) / 2^64) (the rounding error
// e (ceil - 2^64/m) / 2^64 < 2^-32 stays below 1/m, the smallest nonzero fractional part).
struct DivM {
  uint64_t magic;  // ceil(2^64 / m); 0 for m == 1
  int m;
  __host__ static DivM make(int m) {
    DivM d;
    d.m = m;
    d.magic = m > 1 ? ~uint64_t(0) / uint64_t(m) + 1 : 0;
    return d;
  }
  __device__ __forceinline__ uint32_t div(uint32_t e) const {
    return magic ? uint32_t(__umul64hi(uint64_t(e), magic)) : e;
  }
};

// ---------------------------------------------------------------- s-channel compressed operator
// C[(ci*s + k)*n + v] = S_ci[v] * Xc[v*s + k]   (coils == nullptr -> S = 1)
__global__ void __launch_bounds__(256) channels_kernel(const float2* __restrict__ Xc,
                                                       const float2* __restrict__ coils, int c,
                                                       int s, int64_t n,
                                                       float2* __restrict__ C) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  for (int ci = 0; ci < c; ++ci) {
    const float2 sc = coils ? coils[int64_t(ci) * n + v] : make_float2(1.f, 0.f);
    for (int k = 0; k < s; ++k) {
      const float2 x = Xc[v * s + k];
      C[(int64_t(ci) * s + k) * n + v] =
          make_float2(sc.x * x.x - sc.y * x.y, sc.x * x.y + sc.y * x.x);
    }
  }
}

// KT[(ci*n + w)*s + k] = K[(ci*s + k)*n + w]: channel-planar FFT output -> location-major, so
// the gather reads one contiguous s-vector per sample instead of s scattered sectors.
__global__ void __launch_bounds__(256) interleave_kernel(const float2* __restrict__ K, int c,
                                                         int s, int64_t n,
                                                         float2* __restrict__ KT) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= int64_t(c) * n) return;
  const int ci = int(g / n);
  const int64_t w = g - int64_t(ci) * n;
  const float2* src = K + int64_t(ci) * s * n + w;
  float2* dst = KT + g * s;
  for (int k = 0; k < s; ++k) dst[k] = src[int64_t(k) * n];
}

// y[t][ci*m + i] = scale * sum_k KT[(ci*n + Omega_t(i))*s + k] * conj(V[t*s + k]);
// modes as gather_kernel (0 write, 1 norm only, 2 weighted residual y - Ymeas).
__global__ void __launch_bounds__(256) gather_s_kernel(const float2* __restrict__ K,
                                                       const int* __restrict__ pat, int64_t n,
                                                       int L, int m, int c, int s,
                                                       const float2* __restrict__ V, float scale,
                                                       int mode,
                                                       const float2* __restrict__ Ymeas,
                                                       const float* __restrict__ w,
                                                       float2* __restrict__ Y,
                                                       double* __restrict__ partial) {
  __shared__ double sh[256];
  const int64_t cm = int64_t(c) * m;
  const int64_t total = int64_t(L) * cm;
  double acc = 0.0;
  for (int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * 256) {
    const int64_t t = e / cm;
    const int r = int(e - t * cm);
    const int ci = r / m, i = r - ci * m;
    const int64_t wloc = pat[t * m + i];
    const float2* kb = K + (int64_t(ci) * n + wloc) * s;
    const float2* vt = V + t * s;
    float yr = 0.f, yi = 0.f;
    int k = 0;
    if ((s & 1) == 0) {  // 16-byte loads of the contiguous s-vector
      const float4* kb4 = reinterpret_cast<const float4*>(kb);
      for (; k < s; k += 2) {
        const float4 a2 = kb4[k >> 1];
        const float2 b0 = vt[k], b1 = vt[k + 1];
        yr = fmaf(a2.x, b0.x, fmaf(a2.y, b0.y, yr));   // a * conj(b)
        yi = fmaf(a2.y, b0.x, fmaf(-a2.x, b0.y, yi));
        yr = fmaf(a2.z, b1.x, fmaf(a2.w, b1.y, yr));
        yi = fmaf(a2.w, b1.x, fmaf(-a2.z, b1.y, yi));
      }
    }
    for (; k < s; ++k) {
      const float2 a = kb[k], b = vt[k];
      yr = fmaf(a.x, b.x, fmaf(a.y, b.y, yr));   // a * conj(b)
      yi = fmaf(a.y, b.x, fmaf(-a.x, b.y, yi));
    }
    float2 y = make_float2(yr * scale, yi * scale);
    if (mode == 2) {
      const float2 ym = Ymeas[e];
      y.x -= ym.x;
      y.y -= ym.y;
      const float ww = w ? w[e] : 1.f;
      acc += double(ww) * (double(y.x) * y.x + double(y.y) * y.y);
      Y[e] = make_float2(ww * y.x, ww * y.y);
    } else {
      if (mode == 0) Y[e] = y;
      acc += double(y.x) * y.x + double(y.y) * y.y;
    }
  }
  if (partial) {
    double r = block_sum_256(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
  }
}

// Location-major form of gather_s_kernel (same products, same FMA order, so the same y values):
// one thread per k-space location w reads its channel vector KT[(ci*n + w)*s + 0..s) once and
// emits every pattern sample of w (CSR, ascending e = t*m + i).  A location is sampled by
// L*m/n frames on average (cfg2: 62, cfg4: 31), so the channel reads, which sample-major order
// repeats for every sample (cfg4: 80 B of a 335 MB array per sample, from HBM), fall by that
// factor; the 8-byte output writes scatter instead.  The norm / residual partial sums run over
// a fixed location partition (deterministic).
constexpr int kLocThreads = 512;  // 2 blocks x 512 threads per SM: all kRedBlocks resident
template <int S>
__global__ void __launch_bounds__(kLocThreads) gather_loc_kernel(
    const float2* __restrict__ KT, const int* __restrict__ csr_off,
    const int* __restrict__ csr_e, int64_t n, DivM dm, int c, int s,
    const float2* __restrict__ V, float scale, int mode, const float2* __restrict__ Ymeas,
    const float* __restrict__ w, float2* __restrict__ Y, double* __restrict__ partial) {
  __shared__ double sh[kLocThreads];
  const int m = dm.m;
  const int64_t cm = int64_t(c) * m;
  double acc = 0.0;
  for (int64_t wloc = int64_t(blockIdx.x) * kLocThreads + threadIdx.x; wloc < n;
       wloc += int64_t(gridDim.x) * kLocThreads) {
    const int b = csr_off[wloc], e_end = csr_off[wloc + 1];
    for (int ci = 0; ci < c && b < e_end; ++ci) {
      float2 kr[S];
      const float2* kb = KT + (int64_t(ci) * n + wloc) * s;
#pragma unroll
      for (int k = 0; k < S; ++k) kr[k] = k < s ? kb[k] : make_float2(0.f, 0.f);
      for (int j = b; j < e_end; ++j) {
        const uint32_t e = uint32_t(csr_e[j]);
        const uint32_t t = dm.div(e);
        const int64_t eo = int64_t(t) * cm + int64_t(ci) * m + (e - t * uint32_t(m));
        const float2* vt = V + int64_t(t) * s;
        float yr = 0.f, yi = 0.f;
#pragma unroll
        for (int k = 0; k < S; ++k) {
          if (k < s) {
            const float2 a = kr[k], bv = vt[k];
            yr = fmaf(a.x, bv.x, fmaf(a.y, bv.y, yr));   // a * conj(b)
            yi = fmaf(a.y, bv.x, fmaf(-a.x, bv.y, yi));
          }
        }
        float2 y = make_float2(yr * scale, yi * scale);
        if (mode == 2) {
          const float2 ym = Ymeas[eo];
          y.x -= ym.x;
          y.y -= ym.y;
          const float ww = w ? w[eo] : 1.f;
          acc += double(ww) * (double(y.x) * y.x + double(y.y) * y.y);
          Y[eo] = make_float2(ww * y.x, ww * y.y);
        } else {
          if (mode == 0) Y[eo] = y;
          acc += double(y.x) * y.x + double(y.y) * y.y;
        }
      }
    }
  }
  if (partial) {
    double r = block_sum<kLocThreads>(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
  }
}

// Location-tiled gather (every frame's pattern row sorted ascending): a CTA stages the channel
// values of W consecutive k-space locations from the channel-planar FFT output into shared
// memory (one coalesced pass, swizzled against bank conflicts), then for every frame t the
// samples of those locations are the contiguous segment [seg[t][b], seg[t][b+1]) of row t:
// pattern reads and y writes are contiguous.  Same products in the same FMA order per sample
// as gather_s_kernel / gather_loc_kernel (identical y).  Norm / residual partials per CTA over a
// fixed tile assignment (deterministic).
__device__ __forceinline__ int tile_swz(int wl) { return wl ^ ((wl >> 4) & 15); }

template <int S>
__global__ void __launch_bounds__(256) gather_tile_kernel(
    const float2* __restrict__ C, const int* __restrict__ pat, const int* __restrict__ seg,
    int nb, int W, int64_t n, int L, int m, int c, int s, const float2* __restrict__ V,
    float scale, int mode, const float2* __restrict__ Ymeas, const float* __restrict__ w,
    float2* __restrict__ Y, double* __restrict__ partial) {
  extern __shared__ float2 kt[];  // [c*s][W], swizzled columns
  __shared__ double sh[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t cm = int64_t(c) * m;
  double acc = 0.0;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t w0 = int64_t(b) * W;
    const int wn = int(n - w0 < W ? n - w0 : W);
    __syncthreads();  // previous tile fully consumed
    for (int q = 0; q < c * s; ++q)
      for (int j = threadIdx.x; j < wn; j += blockDim.x)
        kt[q * W + tile_swz(j)] = C[int64_t(q) * n + w0 + j];
    __syncthreads();
    const int* sb = seg + int64_t(b) * L;  // row b: first sample >= b W; row b + 1: the end
    // warp w takes the frame groups [32 g, 32 g + 32) with g = w (mod 8); lane j fetches the
    // segment of frame 32 g + j, then the warp walks the group's non-empty segments
    for (int t0 = 32 * warp; t0 < L; t0 += 32 * 8) {
      const int tl = t0 + lane;
      const int my_lo = tl < L ? sb[tl] : 0, my_hi = tl < L ? sb[L + tl] : 0;
      uint32_t busy = __ballot_sync(0xffffffffu, my_hi > my_lo);
      while (busy) {
        const int j = __ffs(busy) - 1;
        busy &= busy - 1;
        const int t = t0 + j;
        const int lo = __shfl_sync(0xffffffffu, my_lo, j), hi = __shfl_sync(0xffffffffu, my_hi, j);
        float2 vr[S];
#pragma unroll
        for (int k = 0; k < S; ++k) vr[k] = k < s ? V[int64_t(t) * s + k] : make_float2(0.f, 0.f);
        for (int i = lo + lane; i < hi; i += 32) {
          const int sw = tile_swz(pat[int64_t(t) * m + i] - int(w0));
          for (int ci = 0; ci < c; ++ci) {
            const float2* kc = kt + ci * s * W + sw;
            float yr = 0.f, yi = 0.f;
#pragma unroll
            for (int k = 0; k < S; ++k) {
              if (k < s) {
                const float2 a = kc[k * W], bv = vr[k];
                yr = fmaf(a.x, bv.x, fmaf(a.y, bv.y, yr));   // a * conj(b)
                yi = fmaf(a.y, bv.x, fmaf(-a.x, bv.y, yi));
              }
            }
            const int64_t eo = int64_t(t) * cm + int64_t(ci) * m + i;
            float2 y = make_float2(yr * scale, yi * scale);
            if (mode == 2) {
              const float2 ym = Ymeas[eo];
              y.x -= ym.x;
              y.y -= ym.y;
              const float ww = w ? w[eo] : 1.f;
              acc += double(ww) * (double(y.x) * y.x + double(y.y) * y.y);
              Y[eo] = make_float2(ww * y.x, ww * y.y);
            } else {
              if (mode == 0) Y[eo] = y;
              acc += double(y.x) * y.x + double(y.y) * y.y;
            }
          }
        }
      }
    }
  }
  if (partial) {
    double r = block_sum_256(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
  }
}

// Single-coil form of the location-tiled gather with compile-time channel count S (rows s..S-1
// of the staged tile and of V are zero, so the padded products add exact zeros), tile width W and
// mode: the channel reads are LDS with immediate offsets, the pattern / measurement values of a
// frame's segment are fetched before its FMAs (up to 4 samples per lane in flight), one index
// e = t m + i addresses pattern, y and the measurements (L m < 2^31), and |y|^2 is summed in fp32
// per segment before it joins the fp64 partial.  Same FMA order per sample as the other gathers.
template <int S, int W, int MODE>
__global__ void __launch_bounds__(512) gather_tile1_kernel(
    const float2* __restrict__ C, const int* __restrict__ pat, const int* __restrict__ seg,
    int nb, int64_t n, int L, int m, int s, const float2* __restrict__ V, float scale,
    const float2* __restrict__ Ymeas, const float* __restrict__ w, float2* __restrict__ Y,
    double* __restrict__ partial) {
  static_assert(S % 2 == 0, "channel pairs");
  extern __shared__ float4 kt4[];  // [S / 2][W]: channels 2q, 2q + 1 of a location in one 16-byte slot
  __shared__ double sh[512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t w0 = int64_t(b) * W;
    const int wn = int(n - w0 < W ? n - w0 : W);
    __syncthreads();  // previous tile fully consumed
#pragma unroll
    for (int q = 0; q < S; ++q)
      for (int j = threadIdx.x; j < W; j += 512)
        reinterpret_cast<float2*>(kt4 + (q >> 1) * W + j)[q & 1] =
            (q < s && j < wn) ? C[int64_t(q) * n + w0 + j] : make_float2(0.f, 0.f);
    __syncthreads();
    const int* sb = seg + int64_t(b) * L;  // row b: first sample >= b W; row b + 1: the end
    for (int t0 = 32 * warp; t0 < L; t0 += 32 * 16) {
      const int tl = t0 + lane;
      const int my_lo = tl < L ? sb[tl] : 0, my_hi = tl < L ? sb[L + tl] : 0;
      uint32_t busy = __ballot_sync(0xffffffffu, my_hi > my_lo);
      // software pipeline over the group's non-empty segments: the pattern values of the next
      // segment's first 128 samples are in flight (DRAM latency) while the current one is computed
      int t = 0, lo = 0, hi = 0, pw[4];
      auto take = [&](int& tt, int& l, int& h, int (&p)[4]) -> bool {
        if (!busy) return false;
        const int j = __ffs(busy) - 1;
        busy &= busy - 1;
        tt = t0 + j;
        l = __shfl_sync(0xffffffffu, my_lo, j);
        h = __shfl_sync(0xffffffffu, my_hi, j);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = l + lane + 32 * u;
          p[u] = i < h ? __ldg(pat + tt * m + i) - int(w0) : -1;
        }
        return true;
      };
      bool have = take(t, lo, hi, pw);
      while (have) {
        int tn = 0, lon = 0, hin = 0, pwn[4];
        const bool have_n = take(tn, lon, hin, pwn);
        float2 vr[S];
#pragma unroll
        for (int k = 0; k < S; ++k)
          vr[k] = k < s ? __ldg(V + int64_t(t) * s + k) : make_float2(0.f, 0.f);
        const int e0 = t * m;
        float psum = 0.f;
        for (int i0 = lo + lane; i0 < hi; i0 += 128) {
          float2 ym[4];
          float ww[4];
          if (i0 != lo + lane) {  // segments longer than 128 samples: later chunks on demand
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + 32 * u;
              pw[u] = i < hi ? __ldg(pat + e0 + i) - int(w0) : -1;
            }
          }
          if (MODE == 2) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + 32 * u;
              ym[u] = i < hi ? __ldg(Ymeas + e0 + i) : make_float2(0.f, 0.f);
              ww[u] = (w && i < hi) ? __ldg(w + e0 + i) : 1.f;
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (pw[u] >= 0) {
              const float4* kc = kt4 + pw[u];
              float yr = 0.f, yi = 0.f;
#pragma unroll
              for (int k2 = 0; k2 < S / 2; ++k2) {
                const float4 a = kc[k2 * W];
                const float2 b0 = vr[2 * k2], b1 = vr[2 * k2 + 1];
                yr = fmaf(a.x, b0.x, fmaf(a.y, b0.y, yr));   // a * conj(b)
                yi = fmaf(a.y, b0.x, fmaf(-a.x, b0.y, yi));
                yr = fmaf(a.z, b1.x, fmaf(a.w, b1.y, yr));
                yi = fmaf(a.w, b1.x, fmaf(-a.z, b1.y, yi));
              }
              const int e = e0 + i0 + 32 * u;
              float2 y = make_float2(yr * scale, yi * scale);
              if (MODE == 2) {
                y.x -= ym[u].x;
                y.y -= ym[u].y;
                psum = fmaf(ww[u], fmaf(y.x, y.x, y.y * y.y), psum);
                Y[e] = make_float2(ww[u] * y.x, ww[u] * y.y);
              } else {
                if (MODE == 0) Y[e] = y;
                psum = fmaf(y.x, y.x, fmaf(y.y, y.y, psum));
              }
            }
          }
        }
        acc += double(psum);
        t = tn;
        lo = lon;
        hi = hin;
#pragma unroll
        for (int u = 0; u < 4; ++u) pw[u] = pwn[u];
        have = have_n;
      }
    }
  }
  if (partial) {
    double r = block_sum<512>(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
  }
}

// seg[b][t] = first sample of frame t at a location >= b W (rows sorted ascending), b = 0..nb
// (row nb = m): tile b's segments are rows b and b + 1, each L contiguous entries
__global__ void seg_table_kernel(const int* __restrict__ pat, int L, int m, int nb, int W,
                                 int* __restrict__ seg) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= int64_t(L) * (nb + 1)) return;
  const int b = int(g / L), t = int(g - int64_t(b) * L);
  const int* row = pat + int64_t(t) * m;
  const int64_t key = int64_t(b) * W;
  int lo = 0, hi = m;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (row[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  seg[g] = lo;
}

// flag = 1 if some frame's pattern row is not strictly ascending
__global__ void rows_sorted_kernel(const int* __restrict__ pat, int L, int m, int* flag) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < int64_t(L) * m;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e % m);
    if (i + 1 < m && pat[e + 1] <= pat[e]) *flag = 1;
  }
}

// K[(ci*s + k)*n + w] = sum over the pattern entries e = t*m + i with Omega_t(i) = w (CSR,
// ascending e) of R[t][ci*m + i] * V[t*s + k].  One thread per k-space location: each sample of
// R is read once and feeds all s channel accumulators (registers, S >= s); unsampled locations
// get 0 (the zero-fill of forward_model.py:160-162).  Consecutive threads write consecutive
// locations of each channel.
// V rows are staged once per CTA in shared memory ([L][S] float2, rows zero-padded to S) when they
// fit: the lanes of a warp read rows of different frames, which costs one L1 pass per distinct
// line as a global load but only bank-conflict replays as a 16-byte shared load.  The grid is
// persistent (each CTA walks location blocks) so the staging is amortised.  v_smem == 0: rows
// from global memory (L s too large).
template <int S>
__global__ void __launch_bounds__(512, (S <= 20 ? 2 : 1)) kspace_s_kernel(const float2* __restrict__ R,
                                                       const int* __restrict__ csr_off,
                                                       const int* __restrict__ csr_e,
                                                       int64_t n, DivM dm, int c, int s, int L,
                                                       const float2* __restrict__ V,
                                                       float2* __restrict__ K, int v_smem) {
  static_assert(S % 2 == 0, "16-byte row reads");
  extern __shared__ float4 vs4[];  // [L][S / 2]
  if (v_smem) {
    float2* vs = reinterpret_cast<float2*>(vs4);
    for (int idx = threadIdx.x; idx < L * S; idx += blockDim.x) {
      const int t = idx / S, k = idx - t * S;
      vs[idx] = k < s ? V[int64_t(t) * s + k] : make_float2(0.f, 0.f);
    }
    __syncthreads();
  }
  const int m = dm.m;
  const int64_t cm = int64_t(c) * m;
  for (int64_t wloc = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; wloc < n;
       wloc += int64_t(gridDim.x) * blockDim.x) {
    const int b = csr_off[wloc], e_end = csr_off[wloc + 1];
    for (int ci = 0; ci < c; ++ci) {
      float2 acc[S];
#pragma unroll
      for (int k = 0; k < S; ++k) acc[k] = make_float2(0.f, 0.f);
      if (v_smem) {
        // batches of 4 entries: the 4 CSR loads, then the 4 dependent residual loads, are in
        // flight together (the accumulation order stays ascending e)
        for (int j0 = b; j0 < e_end; j0 += 4) {
          uint32_t tt[4];
          float2 rr[4];
          uint32_t ee[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            ee[u] = j0 + u < e_end ? uint32_t(__ldg(csr_e + j0 + u)) : 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            tt[u] = dm.div(ee[u]);
            const uint32_t i = ee[u] - tt[u] * uint32_t(m);
            rr[u] = j0 + u < e_end ? __ldg(R + int64_t(tt[u]) * cm + int64_t(ci) * m + i)
                                   : make_float2(0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (j0 + u < e_end) {
              const float2 r = rr[u];
              const float4* vt = vs4 + tt[u] * (S / 2);
#pragma unroll
              for (int k2 = 0; k2 < S / 2; ++k2) {
                const float4 v = vt[k2];
                acc[2 * k2].x = fmaf(r.x, v.x, fmaf(-r.y, v.y, acc[2 * k2].x));
                acc[2 * k2].y = fmaf(r.x, v.y, fmaf(r.y, v.x, acc[2 * k2].y));
                acc[2 * k2 + 1].x = fmaf(r.x, v.z, fmaf(-r.y, v.w, acc[2 * k2 + 1].x));
                acc[2 * k2 + 1].y = fmaf(r.x, v.w, fmaf(r.y, v.z, acc[2 * k2 + 1].y));
              }
            }
          }
        }
      } else {
        for (int j = b; j < e_end; ++j) {
          const uint32_t e = uint32_t(csr_e[j]);
          const uint32_t t = dm.div(e), i = e - t * uint32_t(m);
          const float2 r = R[int64_t(t) * cm + int64_t(ci) * m + i];
          const float2* vt = V + int64_t(t) * s;
#pragma unroll
          for (int k = 0; k < S; ++k) {
            if (k < s) {
              const float2 v = vt[k];
              acc[k].x = fmaf(r.x, v.x, fmaf(-r.y, v.y, acc[k].x));
              acc[k].y = fmaf(r.x, v.y, fmaf(r.y, v.x, acc[k].y));
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < S; ++k)
        if (k < s) K[(int64_t(ci) * s + k) * n + wloc] = acc[k];
    }
  }
}

// G[v*s + k] = scale * sum_ci conj(S_ci[v]) * K[(ci*s + k)*n + v]
__global__ void __launch_bounds__(256) combine_s_kernel(const float2* __restrict__ K,
                                                        const float2* __restrict__ coils, int c,
                                                        int s, int64_t n, float scale,
                                                        float2* __restrict__ G) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  auto one = [&](int k) {
    float gr = 0.f, gi = 0.f;
    for (int ci = 0; ci < c; ++ci) {
      const float2 a = K[(int64_t(ci) * s + k) * n + v];
      const float2 sc = coils ? coils[int64_t(ci) * n + v] : make_float2(1.f, 0.f);
      gr += sc.x * a.x + sc.y * a.y;   // conj(sc) * a
      gi += sc.x * a.y - sc.y * a.x;
    }
    return make_float2(gr * scale, gi * scale);
  };
  if ((s & 1) == 0) {  // rows of G are 16-byte aligned: two channels per store
    float4* g4 = reinterpret_cast<float4*>(G + v * s);
    for (int k = 0; k < s; k += 2) {
      const float2 a = one(k), b = one(k + 1);
      g4[k >> 1] = make_float4(a.x, a.y, b.x, b.y);
    }
  } else {
    for (int k = 0; k < s; ++k) G[v * s + k] = one(k);
  }
}

// Coil-weighted transposes of the uncompressed path:
//   fwd: F[t][v] = S[v] * X[v][t];   adj: X[v][t] (+)= scale * conj(S[v]) * F[t][v]
__global__ void coil_transpose_kernel(const float2* __restrict__ in, int64_t rows, int64_t cols,
                                      const float2* __restrict__ coil, int coil_on_rows,
                                      int conj_coil, float scale, int accumulate,
                                      float2* __restrict__ out) {
  __shared__ float2 tile[32][33];
  const int64_t c0 = int64_t(blockIdx.x) * 32, r0 = int64_t(blockIdx.y) * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      float2 x = tile[threadIdx.x][i];
      if (coil) {
        float2 sc = coil[coil_on_rows ? r : c];
        if (conj_coil) sc.y = -sc.y;
        x = make_float2(sc.x * x.x - sc.y * x.y, sc.x * x.y + sc.y * x.x);
      }
      x.x *= scale;
      x.y *= scale;
      if (accumulate) {
        const float2 o = out[c * rows + r];
        x.x += o.x;
        x.y += o.y;
      }
      out[c * rows + r] = x;
    }
  }
}

// ---------------------------------------------------------------- elementwise + norms
// mode 0: R = a - b, partial w|R|^2 ; mode 1: partial only of w|alpha a - b|^2 ; mode 2: partial |a|^2
__global__ void __launch_bounds__(256) vec_kernel(const float2* __restrict__ a, double alpha,
                                                  const float2* __restrict__ b, int64_t count,
                                                  const float* __restrict__ w, int mode,
                                                  float2* __restrict__ R,
                                                  double* __restrict__ partial) {
  __shared__ double sh[256];
  const int64_t per = (count + gridDim.x - 1) / gridDim.x;
  const int64_t lo = per * blockIdx.x, hi = min(count, lo + per);
  double acc = 0.0;
  for (int64_t e = lo + threadIdx.x; e < hi; e += 256) {
    const float2 x = a[e];
    if (mode == 2) {
      acc += double(x.x) * x.x + double(x.y) * x.y;
      continue;
    }
    const float2 y = b[e];
    double rr, ri;
    if (mode == 1) {
      rr = alpha * x.x - y.x;
      ri = alpha * x.y - y.y;
    } else {
      const float r0 = x.x - y.x, r1 = x.y - y.y;
      rr = r0;
      ri = r1;
      if (R) {
        const float ww = w ? w[e] : 1.f;
        R[e] = make_float2(ww * r0, ww * r1);
      }
    }
    const double ww = w ? double(w[e]) : 1.0;
    acc += ww * (rr * rr + ri * ri);
  }
  double r = block_sum_256(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = r;
}

__global__ void scale_kernel(float2* a, float alpha, int64_t count) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
       e += int64_t(gridDim.x) * blockDim.x) {
    float2 x = a[e];
    a[e] = make_float2(x.x * alpha, x.y * alpha);
  }
}

// ---------------------------------------------------------------- multi-GPU argmax combine
// cand = (score == global max) ? global index : INT64_MAX   (then all-reduce MIN)
__global__ void argmax_select_kernel(const double* __restrict__ score,
                                     const int64_t* __restrict__ gidx,
                                     const double* __restrict__ gmax, int64_t n,
                                     int64_t* __restrict__ cand) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < n) cand[v] = (score[v] == gmax[v]) ? gidx[v] : INT64_MAX;
}

// ================================================================ host side
struct Op {
  int ndim;
  int dims[3];
  int64_t n;
  int L, m;
  int c;                 // coils (measurement columns per frame: c * m)
  const float2* coils;   // c x n device coil maps (caller-owned), nullptr = all ones
  const int* pattern;
  cufftHandle plan;      // batch L (uncompressed frame stacks), created on first use
  bool plan_ready;
  int chan_batch[4];     // cached plans for batches of c*s channel images
  cufftHandle chan_plan[4];
  int* csr_off;          // n + 1 offsets into csr_e (s-channel adjoint)
  int* csr_e;            // pattern entries t*m + i (int32) sorted by k-space location (stable)
  DivM dm;               // e -> (t, i) = (e / m, e % m)
  bool rows_sorted;      // every frame's pattern row strictly ascending: location-tiled gather
  int seg_W[4];          // cached segment tables of the tiled gather, per tile width W
  int* seg_tab[4];
  float scale;           // 1/sqrt(n) (1 for the identity hook)
  bool identity;         // forward_model.py:95,137,163 identity_transform test hook: skip the DFT
};

static int grid_for(int64_t work, int per_block = 256) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g > 148 * 16) g = 148 * 16;
  return int(g > 0 ? g : 1);
}

// Workspace.  Uncompressed calls need the (L, n) frame stack; s-channel calls the c*s channel
// images (planar FFT buffer) and their location-major copy (untiled gather only): 2 c s n.
// Then the reduction partials (one per CTA of the largest reduction grid).
static size_t ws_round(size_t b) { return (b + 255) & ~size_t(255); }
constexpr int kTileBlocks = 2048;  // max CTAs (= partial slots) of the tiled gather
static size_t ws_partials_bytes(const Op* op) {
  const size_t slots = size_t(op->c) * kRedBlocks > kTileBlocks ? size_t(op->c) * kRedBlocks
                                                                 : size_t(kTileBlocks);
  return slots * sizeof(double) + 256;
}
static size_t ws_main_bytes(const Op* op) {
  const size_t frames = size_t(op->L) * op->n * sizeof(float2);
  const size_t chans = size_t(op->c) * 64 * op->n * sizeof(float2);
  return ws_round(frames > chans ? frames : chans);
}
size_t op_ws_bytes(const Op* op) { return ws_main_bytes(op) + ws_partials_bytes(op); }
size_t op_ws_bytes_compressed(const Op* op, int s) {
  return ws_round(size_t(op->c) * 2 * s * op->n * sizeof(float2)) + ws_partials_bytes(op);
}
static float2* ws_frames(void* ws) { return static_cast<float2*>(ws); }
// partials sit after the main area: `main` is the caller's layout (full or compressed)
static double* ws_partial_at(void* ws, size_t main) {
  return reinterpret_cast<double*>(static_cast<uint8_t*>(ws) + main);
}

static int make_plan(const Op* op, int batch, cufftHandle* plan) {
  int nd[3] = {op->dims[0], op->dims[1], op->ndim == 3 ? op->dims[2] : 1};
  if (cufftPlanMany(plan, op->ndim, nd, nullptr, 1, int(op->n), nullptr, 1, int(op->n),
                    CUFFT_C2C, batch) != CUFFT_SUCCESS) {
    set_last_error("cufftPlanMany failed");
    return kErrCufft;
  }
  return kOk;
}

// CSR of the pattern by k-space location: stable sort of the L*m flat entries (int32) by Omega
// value, and the row-order check of the tiled gather.  Runs on the legacy default stream (the
// pattern upload precedes it there) and synchronises that stream only.
static int build_csr(Op* op) {
  const int64_t total = int64_t(op->L) * op->m;
  int* keys = nullptr;
  int* flag = nullptr;
  const cudaStream_t st = 0;
  CBB_CUDA_TRY(cudaMalloc(&op->csr_off, sizeof(int) * size_t(op->n + 1)));
  CBB_CUDA_TRY(cudaMalloc(&op->csr_e, sizeof(int) * size_t(total)));
  CBB_CUDA_TRY(cudaMalloc(&keys, sizeof(int) * size_t(total)));
  CBB_CUDA_TRY(cudaMalloc(&flag, sizeof(int)));
  CBB_CUDA_TRY(cudaMemcpyAsync(keys, op->pattern, sizeof(int) * size_t(total),
                               cudaMemcpyDeviceToDevice, st));
  CBB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
  rows_sorted_kernel<<<grid_for(total), 256, 0, st>>>(op->pattern, op->L, op->m, flag);
  auto pol = thrust::cuda::par.on(st);
  thrust::sequence(pol, op->csr_e, op->csr_e + total);
  thrust::stable_sort_by_key(pol, keys, keys + total, op->csr_e);
  thrust::lower_bound(pol, keys, keys + total, thrust::counting_iterator<int>(0),
                      thrust::counting_iterator<int>(int(op->n) + 1), op->csr_off);
  int unsorted = 1;
  cudaError_t e = cudaMemcpyAsync(&unsorted, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(keys);
  cudaFree(flag);
  if (e != cudaSuccess) {
    set_last_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  op->rows_sorted = unsorted == 0;
  return kOk;
}

int op_destroy(Op* op);

int op_create(int ndim, const int* dims, int L, int m, const int* pattern, int flags, Op** out) {
  if ((ndim != 2 && ndim != 3) || L <= 0 || m <= 0) return kErrArgument;
  Op* op = new (std::nothrow) Op{};
  if (!op) return kErrArgument;
  op->ndim = ndim;
  op->n = 1;
  for (int i = 0; i < ndim; ++i) {
    if (dims[i] <= 0) { delete op; return kErrArgument; }
    op->dims[i] = dims[i];
    op->n *= dims[i];
  }
  // int32 CSR (offsets and entries t*m + i) and int32 FFT sizes
  if (int64_t(L) * m >= (int64_t(1) << 31) || op->n >= (int64_t(1) << 31) - 1) {
    set_last_error("cbb_op_create: L*m and n must stay below 2^31");
    delete op;
    return kErrUnsupported;
  }
  op->L = L;
  op->m = m;
  op->dm = DivM::make(m);
  op->c = 1;
  op->pattern = pattern;
  op->identity = (flags & 1) != 0;
  op->scale = op->identity ? 1.f : float(1.0 / std::sqrt(double(op->n)));
  if (int rc = build_csr(op)) {
    op_destroy(op);
    return rc;
  }
  *out = op;
  return kOk;
}

int op_set_coils(Op* op, int c, const float2* coils) {
  if (!op || c < 1 || (c > 1 && !coils)) return kErrArgument;
  op->c = c;
  op->coils = coils;
  return kOk;
}

int op_destroy(Op* op) {
  if (!op) return kOk;
  if (!op->identity) {
    if (op->plan_ready) cufftDestroy(op->plan);
    for (int i = 0; i < 4; ++i)
      if (op->chan_batch[i]) cufftDestroy(op->chan_plan[i]);
  }
  if (op->csr_off) cudaFree(op->csr_off);
  if (op->csr_e) cudaFree(op->csr_e);
  for (int i = 0; i < 4; ++i)
    if (op->seg_tab[i]) cudaFree(op->seg_tab[i]);
  delete op;
  return kOk;
}

// Tile width of the location-tiled gather.  Single coil: 1024 locations for s <= 12 when that
// leaves >= 2 tiles per SM, else 256 (gather_tile1_kernel).  With coil maps: the largest power of
// two (<= 2048, and not far past n) whose c*s planes fit 40 KB of shared memory.
static int padded_s(int s) {
  const int p[8] = {4, 8, 10, 12, 16, 20, 24, 32};
  for (int i = 0; i < 8; ++i)
    if (s <= p[i]) return p[i];
  return -1;
}
static int tile_width(const Op* op, int s, int mode) {
  if (op->c == 1 && mode != 2) return (s <= 12 && op->n >= int64_t(1024) * 2 * 148) ? 1024 : 256;
  int W = 2048;
  while (W > 32 && (size_t(op->c) * s * W * sizeof(float2) > 40 * 1024 || W / 2 >= op->n)) W >>= 1;
  return W;
}

template <int S, int W>
static int launch_tile1(Op* op, const float2* C, const int* seg, int nb, int grid, int s,
                        const float2* V, int mode, const float2* Ymeas, const float* w, float2* Y,
                        double* pp, cudaStream_t st) {
  const size_t smem = size_t(S / 2) * W * sizeof(float4);
  int dev = 0;
  cudaGetDevice(&dev);
#define CBB_T1(MODE)                                                                           \
  do {                                                                                         \
    static uint64_t attr_done = 0; /* per-device shared-memory opt-in */                       \
    if (!((attr_done >> (dev & 63)) & 1)) {                                                    \
      CBB_CUDA_TRY(cudaFuncSetAttribute(gather_tile1_kernel<S, W, MODE>,                       \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))); \
      attr_done |= uint64_t(1) << (dev & 63);                                                  \
    }                                                                                          \
    gather_tile1_kernel<S, W, MODE><<<grid, 512, smem, st>>>(C, op->pattern, seg, nb, op->n,   \
                                                             op->L, op->m, s, V, op->scale,    \
                                                             Ymeas, w, Y, pp);                 \
  } while (0)
  if (mode == 0) CBB_T1(0);
  else CBB_T1(1);
#undef CBB_T1
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// Segment table of the tiled gather for width W (built once per W, stream-ordered).
static int seg_table(Op* op, int W, cudaStream_t st, const int** out) {
  for (int i = 0; i < 4; ++i)
    if (op->seg_W[i] == W) {
      *out = op->seg_tab[i];
      return kOk;
    }
  int slot = -1;
  for (int i = 0; i < 4 && slot < 0; ++i)
    if (op->seg_W[i] == 0) slot = i;
  if (slot < 0) {
    set_last_error("too many distinct tile widths");
    return kErrUnsupported;
  }
  const int nb = int((op->n + W - 1) / W);
  const int64_t cnt = int64_t(op->L) * (nb + 1);
  CBB_CUDA_TRY(cudaMalloc(&op->seg_tab[slot], sizeof(int) * size_t(cnt)));
  seg_table_kernel<<<unsigned((cnt + 255) / 256), 256, 0, st>>>(op->pattern, op->L, op->m, nb,
                                                                 W, op->seg_tab[slot]);
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  op->seg_W[slot] = W;
  *out = op->seg_tab[slot];
  return kOk;
}

static int exec_fft(cufftHandle plan, float2* F, int dir, cudaStream_t st) {
  if (cufftSetStream(plan, st) != CUFFT_SUCCESS) return kErrCufft;
  if (cufftExecC2C(plan, reinterpret_cast<cufftComplex*>(F), reinterpret_cast<cufftComplex*>(F),
                   dir) != CUFFT_SUCCESS) {
    set_last_error("cufftExecC2C failed");
    return kErrCufft;
  }
  return kOk;
}

static int fft(Op* op, float2* F, int dir, cudaStream_t st) {
  if (op->identity) return kOk;
  if (!op->plan_ready) {  // frame-stack plan (batch L): built on first uncompressed use
    if (int rc = make_plan(op, op->L, &op->plan)) return rc;
    op->plan_ready = true;
  }
  return exec_fft(op->plan, F, dir, st);
}

// batched FFT of `batch` channel images (plans cached per batch size)
static int fft_channels(Op* op, float2* C, int batch, int dir, cudaStream_t st) {
  if (op->identity) return kOk;
  for (int i = 0; i < 4; ++i) {
    if (op->chan_batch[i] == batch) return exec_fft(op->chan_plan[i], C, dir, st);
    if (op->chan_batch[i] == 0) {
      if (int rc = make_plan(op, batch, &op->chan_plan[i])) return rc;
      op->chan_batch[i] = batch;
      return exec_fft(op->chan_plan[i], C, dir, st);
    }
  }
  set_last_error("too many distinct channel batch sizes");
  return kErrUnsupported;
}

static int finish(const double* partial, int np, double* out, cudaStream_t st) {
  finish_sum<<<1, 256, 0, st>>>(partial, np, out);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

int op_apply(Op* op, const float2* X, float2* Y, void* ws, cudaStream_t st) {
  float2* F = ws_frames(ws);
  const int64_t cm = int64_t(op->c) * op->m;
  for (int ci = 0; ci < op->c; ++ci) {
    dim3 grid(unsigned((op->L + 31) / 32), unsigned((op->n + 31) / 32));
    coil_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(
        X, op->n, op->L, op->coils ? op->coils + int64_t(ci) * op->n : nullptr, 1, 0, 1.f, 0, F);
    CBB_CUDA_TRY(cudaGetLastError());
    int rc = fft(op, F, CUFFT_FORWARD, st);
    if (rc) return rc;
    gather_kernel<<<kRedBlocks, 256, 0, st>>>(F, op->pattern, op->n, op->L, op->m, cm,
                                              ci * op->m, op->scale, 0, nullptr, nullptr, Y,
                                              nullptr);
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(3);
  }
  return kOk;
}

int op_adjoint(Op* op, const float2* Y, float2* X, void* ws, cudaStream_t st) {
  float2* F = ws_frames(ws);
  const int64_t cm = int64_t(op->c) * op->m;
  for (int ci = 0; ci < op->c; ++ci) {
    CBB_CUDA_TRY(cudaMemsetAsync(F, 0, size_t(op->L) * op->n * sizeof(float2), st));
    scatter_kernel<<<grid_for(int64_t(op->L) * op->m), 256, 0, st>>>(
        Y, op->pattern, op->n, op->L, op->m, cm, ci * op->m, F);
    CBB_CUDA_TRY(cudaGetLastError());
    int rc = fft(op, F, CUFFT_INVERSE, st);
    if (rc) return rc;
    dim3 grid(unsigned((op->n + 31) / 32), unsigned((op->L + 31) / 32));
    coil_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(
        F, op->L, op->n, op->coils ? op->coils + int64_t(ci) * op->n : nullptr, 0, 1, op->scale,
        ci > 0 ? 1 : 0, X);
    CBB_CUDA_TRY(cudaGetLastError());
    count_launches(2);
  }
  return kOk;
}

// s-channel forward: channels -> c*s FFTs -> gather (mode 0 write / 1 norm / 2 residual)
int op_apply_compressed(Op* op, const float2* Xc, const float2* V, int s, float2* Y, void* ws,
                        const float2* Ymeas, const float* w, double* norm_out, cudaStream_t st) {
  if (s < 1 || s > 32) return kErrUnsupported;
  float2* C = ws_frames(ws);
  channels_kernel<<<unsigned((op->n + 255) / 256), 256, 0, st>>>(Xc, op->coils, op->c, s,
                                                                   op->n, C);
  CBB_CUDA_TRY(cudaGetLastError());
  int rc = fft_channels(op, C, op->c * s, CUFFT_FORWARD, st);
  if (rc) return rc;
  double* part = ws_partial_at(ws, ws_round(size_t(op->c) * 2 * s * op->n * sizeof(float2)));
  int mode = 0;
  if (Y == nullptr) mode = 1;
  else if (Ymeas != nullptr) mode = 2;
  double* pp = (mode != 0 || norm_out) ? part : nullptr;
  int launches = 2;
  const int W = tile_width(op, s, mode);
  const int nb = int((op->n + W - 1) / W);
  // location-tiled gather straight from the channel-planar FFT output, when there are enough
  // tiles to fill the GPU (cfg0's 4096 locations are 8 tiles: sample-major below)
  if (op->rows_sorted && int64_t(op->L) * op->m >= 4 * op->n &&
      nb >= (op->c == 1 ? 148 : 2 * 148)) {
    const int* seg = nullptr;
    if ((rc = seg_table(op, W, st, &seg))) return rc;
    int sms = 148;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int grid = 8 * sms;
    if (grid > kTileBlocks) grid = kTileBlocks;
    if (grid > nb) grid = nb;
    if (op->c == 1 && mode != 2) {
      // single coil, store / norm-only (the fused-residual mode is not reachable through the C
      // ABI and stays on the generic kernel): compile-time (S, W) kernel, 512 threads
      const int S = padded_s(s);
      const int per_sm = int((200 * 1024) / (size_t(S) * W * sizeof(float2)));
      grid = sms * (per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm));
      if (grid > nb) grid = nb;
#define CBB_GT1(SP)                                                                            \
  rc = (W == 1024) ? launch_tile1<SP, 1024>(op, C, seg, nb, grid, s, V, mode, Ymeas, w, Y, pp, st) \
                   : launch_tile1<SP, 256>(op, C, seg, nb, grid, s, V, mode, Ymeas, w, Y, pp, st)
#define CBB_GT1S(SP) rc = launch_tile1<SP, 256>(op, C, seg, nb, grid, s, V, mode, Ymeas, w, Y, pp, st)
      if (S == 4) CBB_GT1(4);
      else if (S == 8) CBB_GT1(8);
      else if (S == 10) CBB_GT1(10);
      else if (S == 12) CBB_GT1(12);
      else if (S == 16) CBB_GT1S(16);
      else if (S == 20) CBB_GT1S(20);
      else if (S == 24) CBB_GT1S(24);
      else CBB_GT1S(32);
#undef CBB_GT1
#undef CBB_GT1S
      if (rc) return rc;
    } else {
    const size_t smem = size_t(op->c) * s * W * sizeof(float2);
#define CBB_GTILE(SP)                                                                        \
  do {                                                                                       \
    gather_tile_kernel<SP><<<grid, 256, smem, st>>>(C, op->pattern, seg, nb, W, op->n, op->L,  \
                                                    op->m, op->c, s, V, op->scale, mode, Ymeas, \
                                                    w, Y, pp);                                 \
  } while (0)
    if (s <= 4) CBB_GTILE(4);
    else if (s <= 8) CBB_GTILE(8);
    else if (s <= 12) CBB_GTILE(12);
    else if (s <= 16) CBB_GTILE(16);
    else if (s <= 20) CBB_GTILE(20);
    else if (s <= 24) CBB_GTILE(24);
    else CBB_GTILE(32);
#undef CBB_GTILE
    CBB_CUDA_TRY(cudaGetLastError());
    }
    if (norm_out) {
      count_launches(launches + 1);
      return finish(part, grid, norm_out, st);
    }
    count_launches(launches);
    return kOk;
  }
  float2* KT = C + size_t(op->c) * s * op->n;
  interleave_kernel<<<unsigned((int64_t(op->c) * op->n + 255) / 256), 256, 0, st>>>(
      C, op->c, s, op->n, KT);
  CBB_CUDA_TRY(cudaGetLastError());
  ++launches;
  // location-major when locations are sampled >= 4 times and there are enough of them to fill
  // the GPU with threads (cfg0's 4096 locations run faster sample-major)
  if (int64_t(op->L) * op->m >= 4 * op->n && op->n >= 65536) {
#define CBB_GLOC(SP)                                                                          \
  gather_loc_kernel<SP><<<kRedBlocks, kLocThreads, 0, st>>>(KT, op->csr_off, op->csr_e, op->n, \
                                                            op->dm, op->c, s, V, op->scale,  \
                                                            mode, Ymeas, w, Y, pp)
    if (s <= 4) CBB_GLOC(4);
    else if (s <= 8) CBB_GLOC(8);
    else if (s <= 12) CBB_GLOC(12);
    else if (s <= 16) CBB_GLOC(16);
    else if (s <= 20) CBB_GLOC(20);
    else if (s <= 24) CBB_GLOC(24);
    else CBB_GLOC(32);
#undef CBB_GLOC
  } else {
    gather_s_kernel<<<kRedBlocks, 256, 0, st>>>(KT, op->pattern, op->n, op->L, op->m, op->c, s,
                                                V, op->scale, mode, Ymeas, w, Y, pp);
  }
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(norm_out ? launches + 1 : launches);
  if (norm_out) return finish(part, kRedBlocks, norm_out, st);
  return kOk;
}

// s-channel adjoint: deterministic k-space build per channel -> c*s IFFTs -> coil combine
int op_adjoint_compressed(Op* op, const float2* R, const float2* V, int s, float2* Gc, void* ws,
                          cudaStream_t st) {
  if (s < 1 || s > 32) return kErrUnsupported;
  float2* K = ws_frames(ws);
  {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int S = padded_s(s);
    // V rows in shared memory when [L][S] float2 fits beside >= 1 CTA per SM
    const size_t vbytes = size_t(op->L) * S * sizeof(float2);
    const int v_smem = vbytes <= 200 * 1024 ? 1 : 0;
    const size_t smem = v_smem ? vbytes : 0;
    int per_sm = v_smem ? int((220 * 1024) / (vbytes + 1024)) : 4;
    if (per_sm > 4) per_sm = 4;
    if (per_sm < 1) per_sm = 1;
    int64_t grid64 = (op->n + 511) / 512;
    if (grid64 > int64_t(sms) * per_sm) grid64 = int64_t(sms) * per_sm;
    const unsigned grid = unsigned(grid64);
#define CBB_KSPACE(SP)                                                                        \
  do {                                                                                        \
    static uint64_t attr_done = 0; /* per-device shared-memory opt-in (largest request) */    \
    static size_t attr_bytes[64] = {0};                                                       \
    if (smem > 48 * 1024 && (!((attr_done >> (dev & 63)) & 1) || attr_bytes[dev & 63] < smem)) { \
      CBB_CUDA_TRY(cudaFuncSetAttribute(kspace_s_kernel<SP>,                                  \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))); \
      attr_done |= uint64_t(1) << (dev & 63);                                                 \
      attr_bytes[dev & 63] = smem;                                                            \
    }                                                                                         \
    kspace_s_kernel<SP><<<grid, 512, smem, st>>>(R, op->csr_off, op->csr_e, op->n, op->dm,    \
                                                 op->c, s, op->L, V, K, v_smem);              \
  } while (0)
    if (S == 4) CBB_KSPACE(4);
    else if (S == 8) CBB_KSPACE(8);
    else if (S == 10) CBB_KSPACE(10);
    else if (S == 12) CBB_KSPACE(12);
    else if (S == 16) CBB_KSPACE(16);
    else if (S == 20) CBB_KSPACE(20);
    else if (S == 24) CBB_KSPACE(24);
    else CBB_KSPACE(32);
#undef CBB_KSPACE
  }
  CBB_CUDA_TRY(cudaGetLastError());
  int rc = fft_channels(op, K, op->c * s, CUFFT_INVERSE, st);
  if (rc) return rc;
  combine_s_kernel<<<unsigned((op->n + 255) / 256), 256, 0, st>>>(K, op->coils, op->c, s, op->n,
                                                                   op->scale, Gc);
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(2);
  return kOk;
}

int vec_op(const float2* a, double alpha, const float2* b, int64_t count, const float* w,
           int mode, float2* R, double* out, void* ws, cudaStream_t st) {
  double* part = static_cast<double*>(ws);
  vec_kernel<<<kRedBlocks, 256, 0, st>>>(a, alpha, b, count, w, mode, R, part);
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(out ? 2 : 1);
  if (out) return finish(part, kRedBlocks, out, st);
  return kOk;
}

int scale_c64(float2* a, double alpha, int64_t count, cudaStream_t st) {
  scale_kernel<<<grid_for(count), 256, 0, st>>>(a, float(alpha), count);
  CBB_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return kOk;
}

int argmax_select(const double* score, const int64_t* gidx, const double* gmax, int64_t n,
                  int64_t* cand, cudaStream_t st) {
  if (n == 0) return kOk;
  argmax_select_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(score, gidx, gmax, n, cand);
  CBB_CUDA_TRY(cudaGetLastError());
  return kOk;
}

size_t reduce_ws_bytes() { return kRedBlocks * sizeof(double); }

}  // namespace cbb

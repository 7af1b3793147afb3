// Shared device helpers for the CoverBLIP B200 hot path (sm_100a only).
//
// PTX wrappers for mbarriers, bulk async copies (TMA engine, SASS UBLKCP),
// tcgen05 (TMEM alloc / MMA / commit / ld) and the exact fp64 rescoring used
// by every matched-filter variant.
#pragma once

#include <cstdint>
#include <string>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "coverblip_b200 is written for sm_100a only"
#endif

namespace cbb {

// ---------------------------------------------------------------- status
enum Status : int {
  kOk = 0,
  kErrArgument = 1,   // maps to ValueError in the Python shim
  kErrCuda = 2,
  kErrUnsupported = 3,
  kErrCufft = 4,
};

#define CBB_STR2(x) #x
#define CBB_STR(x) CBB_STR2(x)
#define CBB_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      cbb::set_last_error((std::string(cudaGetErrorString(_e)) +                  \
                           " (" __FILE__ ":" CBB_STR(__LINE__) ")").c_str());     \
      return cbb::kErrCuda;                                                       \
    }                                                                             \
  } while (0)

void set_last_error(const char* msg);

// Diagnostics shared by all translation units (defined in cbb_capi.cu).
void count_launches(int k);                    // kernels enqueued by this library
void timing_mark(int which, cudaStream_t st);  // 0 = before / 1 = after the matched filter

// ---------------------------------------------------------------- layout
// Tensor-core operand rows: K_PAD fp16 per row = [re_0..re_{s-1}, im_0..im_{s-1}, sentinel, 0..]
// with 2s < K_PAD: column 2s is the padding sentinel (voxel rows 1.0, real atoms 0, the
// zero-padded atom rows of the last tile -65504 so they can never win or enter a window).
// stored in 128-row tiles with the UMMA K-major SWIZZLE_64B (K_PAD=32) or
// SWIZZLE_128B (K_PAD=64) canonical layout so a flat bulk copy lands a tile in
// shared memory ready for tcgen05.mma.
constexpr int kTileRows = 128;

__host__ __device__ inline int kpad_for(int s) { return (2 * s < 32) ? 32 : 64; }
// K = 16 MMA steps that carry data: columns [0, 2s) plus the sentinel at column 2s (the steps
// after it multiply zeros only and are skipped)
__host__ __device__ inline int mma_ksteps(int s) { return (2 * s + 1 + 15) / 16; }
constexpr unsigned short kF16One = 0x3C00, kF16MinusMax = 0xFBFF;  // 1.0, -65504

// Split-operand screening (fp16 hi/lo operands, fp32 accumulators): voxel rows
// [z_hi | z_lo | z_hi | 1], atom rows [d_hi | d_hi | d_lo | sentinel], K = 6s + 1 <= 128.
// K = 64 (s <= 10): 128-atom tiles of one 128-byte swizzle block per row; K = 128 (s <= 21):
// 64-atom tiles stored as two K blocks [block][64 rows][128 B] (one bulk copy per tile).
constexpr int kSplitMaxS = 21;
__host__ __device__ constexpr int split_kp(int s) { return 6 * s + 1 <= 64 ? 64 : 128; }
__host__ __device__ constexpr int split_rows(int kp) { return kp == 64 ? 128 : 64; }
__host__ __device__ constexpr int split_ksteps(int s) { return (6 * s + 1 + 15) / 16; }
// byte offset of element e of row r inside one split tile of `rows` rows
__host__ __device__ inline uint32_t split_elem_offset(int r, int e, int rows) {
  return uint32_t(e >> 6) * uint32_t(rows) * 128u + uint32_t(r) * 128u +
         uint32_t((((e & 63) >> 3) ^ (r & 7)) * 16) + uint32_t(e & 7) * 2u;
}

// fp16 atom operand storage (non-split screens): the UMMA K-major layout WITHOUT swizzle, i.e.
// 8-row groups of tc_nc(s) core matrices (8 rows x 16 B each, chunk c = columns [8c, 8c+8)),
// group after group.  Only the ceil((2s+1)/8) chunks that carry data or the sentinel are stored
// (s = 10: 48 B per atom instead of 64), and any 8-row-aligned window of rows is one flat bulk
// copy.  When tc_nc is odd, the last K = 16 step's second core matrix (all-zero voxel columns)
// reads whatever finite fp16 data follows (the next group's chunk 0, or the zeroed tail of the
// stage): zero times finite adds nothing.
__host__ __device__ inline int tc_nc(int s) { return (2 * s + 1 + 7) / 8; }
// byte offset of (row j, chunk c) from the start of the row sequence (j a multiple of 8 there)
__host__ __device__ inline size_t atom_chunk_offset(int64_t j, int c, int nc) {
  return size_t(j >> 3) * size_t(nc) * 128u + size_t(c) * 128u + size_t(j & 7) * 16u;
}

// ---------------------------------------------------------------- misc device
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// fp16 operand element: round-to-nearest-even straight from fp64 (the rounding error is
// measured exactly from the returned value, so any rounding would do for the certificate).
__device__ __forceinline__ unsigned short f16_bits_rn(double x) {
  return __half_as_ushort(__double2half(x));
}
__device__ __forceinline__ double f16_bits_to_double(unsigned short b) {
  return double(__half2float(__ushort_as_half(b)));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// shared-window address forms (precomputed addresses: fewer instructions in single-lane loops)
__device__ __forceinline__ void mbar_wait_addr(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITA_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITA_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_addr(uint32_t addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_addr(uint32_t dst, const void* gmem_src, uint32_t bytes,
                                              uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(gmem_src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

// ---------------------------------------------------------------- bulk copy (TMA engine)
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// multicast variant: `bytes` land at the same CTA-relative offset in every CTA of ctaMask, each
// completing `bytes` of transaction count on the mbarrier at the same offset in that CTA
__device__ __forceinline__ void bulk_g2s_mc(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                            uint64_t* bar, uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1], %2, [%3], %4, %5;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// every thread of every CTA of the cluster (release / acquire)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// generic-proxy shared-memory writes become visible to the async proxy (tensor core reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// arrive on the mbarrier at this CTA-relative offset in every CTA of ctaMask once the issued
// tcgen05 operations complete
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16 (operand / accumulator types from the idesc;
// A operand resident in tensor memory).
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// ---- CTA-pair (cta_group::2) forms: one MMA of M = 256 rows over the two CTAs of a cluster
// pair (A rows 0..127 in the even CTA's TMEM, 128..255 in the odd one's; B rows split in halves
// between the two CTAs' shared memory; each CTA's TMEM receives its own 128 rows of D).  Every
// tcgen05 alloc / mma / commit of a kernel must use the same cta_group.
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_mma_f16_ts2(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the mbarrier at this CTA-relative offset in both CTAs of the pair (mask 0b11)
__device__ __forceinline__ void tc_commit2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// shared::cluster address of the same object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// arrive (release, cluster scope) on an mbarrier of another CTA of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// wait that also acquires remote (cluster-scope) arrivals
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns: thread i writes lane (base_lane + i).
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 64 consecutive 16-bit accumulator columns packed in pairs (.pack::16b): register
// i of thread t holds columns 2i (low half) and 2i + 1 (high half) of lane (base_lane + t).
__device__ __forceinline__ void tmem_ld32_pack16(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// 32 lanes x 32 consecutive 32-bit accumulator columns (fp32 accumulators).
__device__ __forceinline__ void tmem_ld32_f32(uint32_t taddr, uint32_t (&r)[32]) {
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

// 32 lanes x 32 consecutive 16-bit accumulator columns packed in pairs (.pack::16b).
__device__ __forceinline__ void tmem_ld16_pack16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// UMMA shared-memory descriptor, K-major, swizzled rows (SBO = 8 rows).
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t smem_addr, int kpad) {
  const uint32_t row_bytes = uint32_t(kpad) * 2u;
  uint64_t d = 0;
  d |= uint64_t((smem_addr >> 4) & 0x3FFFu);           // start address
  d |= uint64_t(1u) << 16;                             // LBO (unused for swizzled K-major)
  d |= uint64_t(((8u * row_bytes) >> 4) & 0x3FFFu) << 32;  // SBO: 8-row group stride
  d |= uint64_t(1u) << 46;                             // descriptor version (sm_100)
  const uint64_t layout = (kpad == 32) ? 4u /*SWIZZLE_64B*/ : 2u /*SWIZZLE_128B*/;
  d |= layout << 61;
  return d;
}

// UMMA shared-memory descriptor, K-major, no swizzle (core matrices 8 rows x 16 B): LBO = byte
// stride between the two core matrices of a K = 16 step, SBO = byte stride between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc_interleave(uint32_t smem_addr, uint32_t lbo,
                                                         uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((smem_addr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1u) << 46;  // descriptor version (sm_100); layout type 0 = SWIZZLE_NONE
  return d;
}

// Instruction descriptor: kind::f16, A/B = F16, D = F16 (c/a/b format fields 0), K-major.
// Measured accumulation model (scripts/probe_f16acc.cu, tests/test_gpu_projection.py): each
// K = 16 instruction forms its products' sum exactly and rounds it ONCE to fp16 (round to
// nearest even) when adding to the accumulator; the result sits in the low 16 bits of each
// 32-bit TMEM column.
__host__ __device__ constexpr uint32_t idesc_f16_f16(int M, int N) {
  return (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// kind::f16, A/B = F16, D = F32 (c_format 1).  Measured (scripts/probe_f32acc.cu): each K = 16
// instruction aligns its products (and the incoming accumulator) to the largest exponent,
// keeping at least 24 bits below it (smaller contributions are truncated), and rounds the
// sum once to fp32; on random split rows the error is <= 2^-20.9 sum|a_k b_k| over 4 steps.
__host__ __device__ constexpr uint32_t idesc_f16_f32(int M, int N) {
  return (1u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// ---------------------------------------------------------------- exact scoring
// Re<z, d_j> in fp64 over the 2s real components, z given as fp64 re/im.
template <int S>
__device__ __forceinline__ double exact_score(const double (&zr)[S], const double (&zi)[S],
                                              const double2* __restrict__ atom) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    double2 a = atom[k];
    acc = fma(zr[k], a.x, acc);
    acc = fma(zi[k], a.y, acc);
  }
  return acc;
}

}  // namespace cbb

// Exact cone projection (matched filter) -- shared host/device declarations.
//
// Reference semantics (coverblip/projection.py:45-67):
//   j*_v  = argmax_j Re<Z_v, D_j>   (first index on ties, projection.py:62)
//   g_v   = max(Re<Z_v, D_j*>, 0)    (projection.py:38-42)
//   P_v   = g_v * D_j*               (projection.py:64)
//
// B200 design: a screening pass scores every (voxel, atom) pair in low
// precision (fp16 tcgen05 MMA with fp16 accumulation; split hi/lo fp16 operands with fp32
// accumulation for s <= 21; or fp32 FFMA) and keeps, per voxel, every atom
// whose approximate score lies inside a CERTIFIED window below the running
// maximum (window = 2 * rigorous bound on |approx - exact|).  The surviving
// candidates are rescored in fp64 from the caller's own atoms and voxels, so
// the selected index is the fp64 argmax (lowest index on exact ties); voxels
// whose candidate list overflows are rescanned exhaustively in fp64.
#pragma once
#include <cstdint>

namespace cbb {

constexpr int kCandCap = 16;       // candidate slots per voxel in the screening kernels

// Device view of a prepared dictionary (all pointers are device memory).
struct DictView {
  int64_t d;
  int32_t s;
  int32_t s_pad;       // FFMA register width (>= s)
  int32_t kpad;        // tensor-core K (32 or 64)
  int32_t n_btiles;    // ceil(d / 128)
  const double2* atoms64;      // d x s   complex128 (exact rescoring)
  const float* atoms32;        // d x 2*s_pad planar fp32 [re.., im..]
  const uint8_t* atoms_tc;     // fp16 rows of atoms * scale: tc_nc(s) 16-byte chunks per row,
                               // no-swizzle core-matrix layout (atom_chunk_offset)
  const float* bounds;         // kB* slots below
  const uint8_t* atoms_tc2;    // split-operand tiles (s <= kSplitMaxS, else null): swizzled
                               // rows of split_kp(s) fp16 [d_hi | d_hi | d_lo | sentinel]
  int32_t prefer_split;        // auto mode screens with the split tiles (coherent dictionary)
  int32_t reserved;
  int32_t n_tiles2;            // split-screen atom tiles: ceil(d / split_rows(split_kp(s)))
  int32_t reserved2;
  // Coherent dictionaries: the split tiles hold the atoms in a bisection order (compact tiles)
  // with per-tile / per-group bounds for the IPG tile pruning (prune_kernel); null otherwise.
  const int32_t* tc2_atom;     // split-tile row -> atom index (d for padded rows); null: identity
  const int32_t* tc2_pos;      // atom -> split-tile row; null: identity
  const float* tile_c;         // [n_tiles2][2 s_pad] fp32 planar centroid of each split tile
  const float* tile_r;         // [n_tiles2] radius >= max ||d_j - c|| over the tile's atoms
  const uint8_t* ctr_tc2;      // the centroids as split-operand tiles (bound pass B operand)
  const float* tile_rs;        // [n_tiles2 (+ sentinel rows)] radius * scale_d, rounded up
};

// Bounds slots (all rounded up).  The fp16 tiles hold d~ = fp16(scale_d * d) with scale_d a
// power of two putting max||scale_d d|| in [0.5, 1).
enum {
  kBDeltaH = 0,    // max_j ||scale_d d_j - d~_j||
  kBDmax = 1,      // max_j ||d_j||
  kBDhMax = 2,     // max_j ||d~_j||
  kBDelta32 = 3,   // max_j ||d_j - fp32(d_j)||
  kBD32Max = 4,    // max_j ||fp32(d_j)||
  kBScaleD = 5,    // scale_d
  // split-operand tiles: d_hi = fp16(scale_d d), d_lo = fp16(scale_d d - d_hi)
  kBDeltaS = 6,    // max_j ||scale_d d_j - (d_hi + d_lo)||
  kBDloMax = 7,    // max_j ||d_lo||
  kBRowMax = 8,    // max_j ||[d_hi, d_hi, d_lo]|| = sqrt(2 ||d_hi||^2 + ||d_lo||^2)
  kBCoherence = 9, // coherence estimate: mean number of other atoms j with
                   // Re<d_i, d_j> >= (1 - 2^-6) ||d_i|| ||d_j|| over kCohSamples sampled atoms i
  kBCount = 12
};

// Where the projection input Z comes from.
struct ZSource {
  const void* z;       // n x s complex (c64 if !z128 else c128), may be null in IPG mode
  int32_t z128;
  const float2* x;     // IPG mode: Z = x - mu * g (complex64), written to z_out
  const float2* g;
  float mu;
  float2* z_out;
  const int32_t* hint; // optional per-voxel atom index (e.g. the previous IPG winner): its exact
                       // score seeds the screen's running max (warm start); may be null
  const float* mu_ptr; // IPG mode: mu read from device memory (graph-captured trials), else mu
  const int32_t* hint2; // optional second warm-start atom per voxel (e.g. the previous trial's
                        // winner): the better-scoring of the two hints seeds the screen
};

// Outputs.  Any pointer may be null (not produced).
struct ProjOut {
  void* idx;           // int32 or int64 (idx64)
  int32_t idx64;
  double* gamma;       // fp64
  void* proj;          // c64 or c128 (proj128)
  int32_t proj128;
  const float2* x;     // IPG: dX = proj(c64) - x
  float2* dx;
  double* nd_v;        // per-voxel ||dX_v||^2 (fp64)
  double* score;       // raw fp64 best score Re<z, d_j*> (before the clip at 0), atom sharding
  int64_t idx_offset;  // added to the written index (global atom id of this dictionary shard)
};

}  // namespace cbb

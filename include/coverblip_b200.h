/*
 * coverblip_b200.h -- C ABI of libcoverblip_b200.so, the B200 (sm_100a) hot path
 * of the CoverBLIP exact-projection IPG reconstruction (arXiv 1810.01967).
 *
 * All array arguments are DEVICE pointers (CUDA global memory) unless named
 * *_host; `stream` is a cudaStream_t (NULL = legacy default stream).  Complex
 * arrays are interleaved (re, im): complex64 = float2, complex128 = double2,
 * row-major, voxel-major (row v = voxel v), exactly the numpy layouts of the
 * reference.  Every function returns 0 on success; 1 = bad argument (the
 * Python shim raises ValueError), 2 = CUDA error, 3 = unsupported shape,
 * 4 = cuFFT error.  cbb_last_error() returns the last message (thread-local).
 *
 * Functions are re-entrant: no global mutable state besides per-plan objects
 * owned by the caller (reference SURVEY 8b "Threading").
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/coverblip):
 *   cbb_project_cone_exact  <- projection.py:45-67  project_cone_exact(Z, dictionary)
 *                              (+ projection.py:38-42 _gammas_for, :64 write-back)
 *   cbb_project_step        <- solver.py:128-130   proj = project_fn(X - mu*G); dX; ||dX||^2
 *   cbb_graph_*, cbb_trial_* <- solver.py:116-144 step_shrinkage decided on the device
 *   cbb_dict_prepare        <- projection.py:26-29 _atoms_of (device copy of .atoms /
 *                              .atoms_compressed, done once per dictionary)
 *   cbb_op_*                <- forward_model.py:123-167 ForwardOperator.apply/adjoint
 *                              (cartesian_dft) and dictionary.py:116-122 compress/decompress
 *   cbb_residual, cbb_norm2_c64, cbb_scaled_residual_norm2
 *                           <- solver.py:130,135,180-190 (np.linalg.norm(.)**2 reductions)
 *   cbb_argmax_select       <- projection.py:62 np.argmax across atom shards (multi-GPU)
 */
#ifndef COVERBLIP_B200_H_
#define COVERBLIP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define CBB_ABI_VERSION 3

/* Device view of a prepared dictionary (filled by cbb_dict_prepare). */
typedef struct cbb_dict_view {
  int64_t d;          /* number of atoms */
  int32_t s;          /* complex dimension of an atom (L, or s when compressed) */
  int32_t s_pad;      /* FFMA register width */
  int32_t kpad;       /* tensor-core K (32 or 64) */
  int32_t n_btiles;   /* ceil(d / 128) */
  const void* atoms64;   /* d x s complex128 */
  const void* atoms32;   /* d x 2*s_pad fp32 planar */
  const void* atoms_tc;  /* fp16 UMMA rows of the fp16-accumulated screen: K-major, no swizzle,
                            8-row groups of ceil((2s+1)/8) 16-byte core matrices */
  const float* bounds;   /* certified error bounds */
  const void* atoms_tc2; /* split hi/lo fp16 UMMA tiles (fp32-accumulated screen), s <= 21 */
  int32_t prefer_split;  /* CBB_ALGO_AUTO uses the split screen: the dictionary is coherent
                            (its sampled atoms have near-duplicates inside the fp16 window) */
  int32_t reserved;
  int32_t n_tiles2;      /* split-screen atom tiles */
  int32_t reserved2;
  /* coherent dictionaries (prefer_split): the split tiles hold the atoms in a bisection order
     with per-tile bounds, so IPG projections with a warm-start hint screen only the tiles
     that may hold a voxel's argmax (results unchanged); NULL otherwise */
  const int32_t* tc2_atom;  /* split-tile row -> atom index */
  const int32_t* tc2_pos;   /* atom -> split-tile row */
  const float* tile_c;      /* per split tile: fp32 centroid (2 s_pad, planar) */
  const float* tile_r;      /*   and radius */
  const void* ctr_tc2;      /* the centroids as split-operand tiles (pruning bound pass) */
  const float* tile_rs;     /* radius * scale_d per centroid */
} cbb_dict_view;

/* Projection algorithms. */
enum {
  CBB_ALGO_AUTO = 0,        /* split tcgen05 if prefer_split (s <= 21), else fp16 tcgen05 ... */
  CBB_ALGO_TCGEN05 = 1,     /* fp16 operands, fp16 accumulators (2s < 64) */
  CBB_ALGO_FFMA = 2,        /* fp32 FFMA screen */
  CBB_ALGO_EXHAUSTIVE = 3,  /* fp64 scan of every atom */
  CBB_ALGO_TCGEN05_SPLIT = 4 /* hi/lo fp16 operands, fp32 accumulators (s <= 21) */
};

int cbb_abi_version(void);
const char* cbb_last_error(void);
int cbb_device_sm_count(int* out);

/* ---- diagnostics ---- */
/* Number of kernels this library has enqueued (process lifetime). */
unsigned long long cbb_stats_kernel_launches(void);
/* When enabled, CUDA events are recorded immediately before and after the matched-filter
 * kernel of every projection on the caller's stream; cbb_timing_last_ms returns the last
 * interval (synchronises on the end event).  Thread-local. */
int cbb_timing_enable(int32_t on);
int cbb_timing_last_ms(float* ms);

/* ---- dictionary (projection.py:26-29) ---- */
size_t cbb_dict_storage_bytes(int64_t d, int32_t s);
int cbb_dict_prepare(const void* atoms, int32_t atoms_c128, int64_t d, int32_t s, void* storage,
                     cbb_dict_view* view_out, void* stream);

/* ---- exact cone projection (projection.py:45-67) ---- */
size_t cbb_project_workspace_bytes(int64_t n, int32_t s);
/* Workspace for projections of n voxels against this dictionary, including the tile-pruning
 * buffers of the split screen (used by cbb_project_step with a hint; a workspace of
 * cbb_project_workspace_bytes(n, s) bytes simply screens every tile). */
size_t cbb_project_workspace_bytes_dict(int64_t n, const cbb_dict_view* dict);
/* z: n x s complex (c128 if z_c128 else c64).  Outputs (any may be NULL):
 * idx_out int64 (idx_int64=1) or int32, gamma_out fp64, proj_out c128 (proj_c128=1) or c64. */
int cbb_project_cone_exact(const void* z, int32_t z_c128, int64_t n, const cbb_dict_view* dict,
                           void* idx_out, int32_t idx_int64, double* gamma_out, void* proj_out,
                           int32_t proj_c128, void* workspace, size_t workspace_bytes,
                           int32_t algo, void* stream);
/* One IPG trial (solver.py:128-130): Z = X - mu*G (c64, written to z_out), project,
 * X' = proj (c64), dX = X' - X (c64), nd_out[0] = ||dX||^2 (fp64, deterministic).
 * idx_hint (optional, int32 per voxel, e.g. the previous iterate's atoms): the hinted atom's
 * exact score seeds the screening threshold (warm start; results are unchanged). */
int cbb_project_step(const void* x, const void* g, double mu, void* z_out, int64_t n,
                     const cbb_dict_view* dict, const int32_t* idx_hint, int32_t* idx_out,
                     double* gamma_out, void* xnext_out, void* dx_out, double* nd_out,
                     void* workspace, size_t workspace_bytes, int32_t algo, void* stream);
/* cbb_project_step extended: mu_dev (optional) reads mu from device memory (float, the same
 * float(mu) the host loop passes: graph-captured trials), idx_hint2 (optional) a second
 * warm-start atom per voxel (e.g. the previous trial's winners): the better-scoring hint seeds
 * the screen and the tile-pruning bound.  Results are those of cbb_project_step. */
int cbb_project_step_ex(const void* x, const void* g, double mu, const float* mu_dev,
                        void* z_out, int64_t n, const cbb_dict_view* dict,
                        const int32_t* idx_hint, const int32_t* idx_hint2, int32_t* idx_out,
                        double* gamma_out, void* xnext_out, void* dx_out, double* nd_out,
                        void* workspace, size_t workspace_bytes, int32_t algo, void* stream);

/* Warm-start atoms for the first trial of an IPG iteration (solver.py:127-128, the first pass
 * of the while loop): the exact projection of Z = X - mu*G (written to z_out, mu / mu_dev as in
 * cbb_project_step_ex) onto the `reps` dictionary -- one representative atom per split tile of the
 * full dictionary (the atom nearest to the tile's centroid) -- mapped through rep_atoms
 * (representative -> atom index of the full dictionary) into hint_out (int32 per voxel).  The
 * current iterate's atoms are a poor lower bound after a large step; the best representative
 * is within one tile radius of the maximum, so the tile pruning of the following
 * cbb_project_step_ex lists far fewer tiles.  Only a hint: results do not depend on it. */
int cbb_project_hint(const void* x, const void* g, double mu, const float* mu_dev, void* z_out,
                     int64_t n, const cbb_dict_view* reps, const int32_t* rep_atoms,
                     int32_t* hint_out, void* workspace, size_t workspace_bytes, void* stream);

/* ---- device-decided IPG iteration (solver.py:116-144, 155-257) ----
 * A CUDA graph of one iteration: the gradient, a while-conditional node repeating the trial
 * (cbb_project_step_ex + ||A dX||^2 + cbb_trial_decide) until the device accepts mu, reaches the
 * fixed point or collapses, then the apply of the new iterate and the residual.  Capture:
 * cbb_graph_capture_begin(stream) -> calls on stream -> cbb_graph_while_begin(g, body_stream) ->
 * the trial's calls on body_stream -> cbb_trial_decide -> cbb_graph_while_end -> calls on stream
 * -> cbb_graph_capture_end; replay with cbb_graph_launch.  The trial state (device memory of
 * cbb_trial_state_bytes(): fp64 mu, mu_base, fp32 mu, shrinks, fixed, status, trials) is
 * reset from mu_base by cbb_trial_init; cbb_trial_carry sets mu_base = mu (carry_over). */
typedef struct cbb_graph cbb_graph;
size_t cbb_trial_state_bytes(void);
int cbb_trial_init(void* trial_state, void* stream);
int cbb_trial_carry(void* trial_state, void* stream);
int cbb_graph_capture_begin(void* stream, cbb_graph** out);
int cbb_graph_while_begin(cbb_graph* g, void* body_stream);
int cbb_trial_decide(cbb_graph* g, void* trial_state, const double* nd, const double* den,
                     double zeta, int32_t max_shrink);
int cbb_graph_while_end(cbb_graph* g);
int cbb_graph_capture_end(cbb_graph* g);
int cbb_graph_launch(cbb_graph* g, void* stream);
int cbb_graph_destroy(cbb_graph* g);

/* Atom-sharded building block (multi-GPU): per voxel the shard-local exact argmax
 * reported as a GLOBAL atom index (local + atom_offset, int64) and its raw fp64 score
 * Re<z, d_j*> (not clipped at 0), for the cross-rank combine (cbb_argmax_select). */
int cbb_project_best(const void* z, int32_t z_c128, int64_t n, const cbb_dict_view* dict,
                     int64_t atom_offset, int64_t* idx_out, double* score_out, void* workspace,
                     size_t workspace_bytes, int32_t algo, void* stream);
/* out[v] = gamma[v] * atoms[idx[v] - atom_offset] if this shard owns idx[v], else 0
 * (projection.py:64 write-back of the winners a shard owns; outputs are summed over ranks). */
int cbb_scaled_rows(const cbb_dict_view* dict, int64_t atom_offset, const int64_t* idx,
                    const double* gamma, int64_t n, void* out, int32_t out_c128, void* stream);
/* Number of voxels the last call's screening pass could not certify (candidate lists full or
 * non-finite input): they were rescanned exhaustively in fp64.  Synchronises. */
int cbb_project_overflow_count(void* workspace, int64_t n, int32_t s, int* count_host,
                               void* stream);
/* counts_host[0] as above; counts_host[1] = voxels whose tcgen05 candidate lists held many
 * chunks (coherent dictionaries) and were rescored warp-cooperatively.  Synchronises. */
int cbb_project_overflow_counts(void* workspace, int64_t n, int32_t s, int32_t* counts_host,
                                void* stream);
/* Tile-pruning statistics of the last projection on this workspace (sized with
 * cbb_project_workspace_bytes_dict): listed (voxel tile, atom tile) pairs and all pairs of the
 * split screen; listed = -1 if that projection screened every tile (or the workspace has no
 * pruning buffers).  Synchronises. */
int cbb_project_prune_stats(void* workspace, size_t workspace_bytes, int64_t n,
                            const cbb_dict_view* dict, int64_t* listed_host, int64_t* total_host,
                            void* stream);
/* Per voxel tile of that projection, in screen order (ceil(n / 128) entries each): the length of
 * its atom-tile list and the bound-tightness bucket of its first voxel (0: hint score >= 0.95
 * ||z|| max||d||, 1: >= 0.8, 2: >= 0.5, 3: below).  counts_host[0] = -1 if nothing was pruned.
 * Diagnostic (where the listed pairs come from); synchronises. */
int cbb_project_prune_detail(void* workspace, size_t workspace_bytes, int64_t n,
                             const cbb_dict_view* dict, int32_t* counts_host,
                             int32_t* buckets_host, void* stream);
/* Bring-up / test hook: prologue only (fp16 voxel rows + windows in the workspace). */
int cbb_project_prologue(const void* z, int32_t z_c128, int64_t n, const cbb_dict_view* dict,
                         void* workspace, size_t workspace_bytes, void* stream);
/* Bring-up / test hook: raw tcgen05 scores (fp16 operands, fp16 accumulators) of voxel tile
 * a_tile x atom rows [128 b_tile, +128), returned as 128 x 128 fp32 (row = voxel), from the
 * workspace voxel rows. */
int cbb_debug_tc_scores(void* workspace, const cbb_dict_view* dict, int32_t a_tile,
                        int32_t b_tile, float* out, void* stream);

/* ---- Cartesian operator (forward_model.py:123-167) + subspace maps (dictionary.py:116-122) ---- */
typedef struct cbb_op cbb_op;
/* spatial dims (ndim 2 or 3), L frames, m samples per frame, pattern (L x m int32 device,
 * flat C-order index per sample).  flags bit 0: identity_transform hook (no DFT).  Builds the
 * pattern's CSR on the legacy default stream and synchronises that stream; L*m and n must stay
 * below 2^31 (status 3 otherwise). */
int cbb_op_create(int32_t ndim, const int32_t* dims, int32_t L, int32_t m, const int32_t* pattern,
                  int32_t flags, cbb_op** out);
/* Coil sensitivity maps S (forward_model.py:82-113,132-167): c x n complex64 device array
 * (caller-owned, must outlive the operator; NULL with c = 1 = all ones).  Measurements become
 * (L, c*m) frame-major: column ci*m + i of frame t = coil ci, sample Omega_t(i). */
int cbb_op_set_coils(cbb_op* op, int32_t c, const void* coil_maps);
int cbb_op_destroy(cbb_op* op);
size_t cbb_op_workspace_bytes(const cbb_op* op);
/* Workspace of the compressed (s-channel) calls with rank s only: 2 c s n complex64 + partials
 * (the uncompressed calls need cbb_op_workspace_bytes). */
size_t cbb_op_workspace_bytes_compressed(const cbb_op* op, int32_t s);
/* Y = A X.  X: n x L complex64 voxel-major (reference layout); Y: L x m complex64
 * FRAME-major (Y_fm[t][i] = Y_ref[i][t]; the Python shim transposes at the boundary). */
int cbb_op_apply(cbb_op* op, const void* X, void* Y, void* workspace, void* stream);
/* X = A^H Y. */
int cbb_op_adjoint(cbb_op* op, const void* Y, void* X, void* workspace, void* stream);
/* Compressed chain: Y = A(Xc V^H) with Xc n x s c64, V L x s c64 (basis), Y frame-major. */
int cbb_op_apply_compressed(cbb_op* op, const void* Xc, const void* V, int32_t s, void* Y,
                            void* workspace, void* stream);
/* ||A(Xc V^H)||^2 only (apply_diff norm, solver.py:135) -> norm_out[0] fp64. */
int cbb_op_apply_norm2_compressed(cbb_op* op, const void* Xc, const void* V, int32_t s,
                                  double* norm_out, void* workspace, void* stream);
/* Gc = (A^H R) V for a frame-major residual R (L x m, already weighted). */
int cbb_op_adjoint_compressed(cbb_op* op, const void* R, const void* V, int32_t s, void* Gc,
                              void* workspace, void* stream);

/* ---- small fused vector kernels ---- */
/* R = a - b (complex64, count elements); optional fp64 ||R||^2 (weights w fp32 or NULL). */
int cbb_residual(const void* a, const void* b, int64_t count, const float* w, void* R,
                 double* norm_out, void* workspace, void* stream);
/* out = ||alpha*a - b||^2 (complex64, count elements, fp64 deterministic). */
int cbb_scaled_residual_norm2(const void* a, double alpha, const void* b, int64_t count,
                              const float* w, double* norm_out, void* workspace, void* stream);
/* out = ||a||^2 (complex64). */
int cbb_norm2_c64(const void* a, int64_t count, double* norm_out, void* workspace, void* stream);
/* a *= alpha (complex64, in place). */
int cbb_scale_c64(void* a, double alpha, int64_t count, void* stream);
size_t cbb_reduce_workspace_bytes(void);

/* ---- multi-GPU atom sharding: exact (max score, lowest index) combine ---- */
/* After an all-reduce MAX of the per-rank best fp64 scores (gmax), each rank emits
 * cand[v] = (score[v] == gmax[v]) ? gidx[v] : INT64_MAX; an all-reduce MIN of cand then
 * yields the global first-index argmax (projection.py:62 semantics across atom shards). */
int cbb_argmax_select(const double* score, const int64_t* gidx, const double* gmax, int64_t n,
                      int64_t* cand_out, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* COVERBLIP_B200_H_ */

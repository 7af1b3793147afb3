// extern "C" boundary of libcoverblip_b200.so (declared in include/coverblip_b200.h).
#include "../../include/coverblip_b200.h"
#include "cbb_common.cuh"
#include "cbb_project.cuh"

#include <cstring>
#include <string>

#include <atomic>

namespace cbb {
static thread_local std::string g_last_error;
void set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

static std::atomic<unsigned long long> g_launches{0};
void count_launches(int k) { g_launches.fetch_add((unsigned long long)k); }

// Optional CUDA events bracketing the matched-filter kernel (enabled by cbb_timing_enable).
static thread_local cudaEvent_t g_ev[2] = {nullptr, nullptr};
static thread_local bool g_timing = false;
void timing_mark(int which, cudaStream_t st) {
  if (g_timing && g_ev[which]) cudaEventRecord(g_ev[which], st);
}

// cbb_project.cu
size_t dict_bytes(int64_t d, int s, size_t*, size_t*, size_t*, size_t*, size_t*);
int dict_prepare(const void* atoms, int in128, int64_t d, int s, void* storage, DictView* view,
                 cudaStream_t st);
struct ProjWs;
size_t project_ws_bytes(int64_t n, int s, ProjWs* ws, void* base_ptr, int prune_tiles);
int prune_tiles_of(const DictView& dv);
int project(const ZSource& zs, int64_t n, const DictView& dv, const ProjOut& out, double* nd_sum,
            void* ws_ptr, size_t ws_bytes, int algo, int max_ctas, cudaStream_t st);
int project_overflow_count(void* ws_ptr, int64_t n, int s, int* host_count, cudaStream_t st);
int map_indices(int32_t* idx, const int32_t* table, int64_t n, int64_t table_len, cudaStream_t st);
int project_prune_detail(void* ws_ptr, size_t ws_bytes, int64_t n, const DictView& dv,
                         int32_t* counts, int32_t* buckets, cudaStream_t st);
int project_prune_stats(void* ws_ptr, size_t ws_bytes, int64_t n, const DictView& dv,
                        int64_t* listed, int64_t* total, cudaStream_t st);
int project_overflow_counts(void* ws_ptr, int64_t n, int s, int* host2, cudaStream_t st);
int tc_debug_scores(const void* ztiles, const void* atiles, int kpad, int s, int a_tile,
                    int b_tile, float* out, cudaStream_t st);
int prologue_only(const ZSource& zs, int64_t n, const DictView& dv, void* ws_ptr, cudaStream_t st);
int trace_dump(long long* host, int count);
int scaled_rows(const DictView& dv, int64_t offset, const int64_t* idx, const double* gamma,
                int64_t n, void* out, int out128, cudaStream_t st);

// cbb_operator.cu
struct Op;
int op_create(int ndim, const int* dims, int L, int m, const int* pattern, int flags, Op** out);
int op_destroy(Op* op);
int op_set_coils(Op* op, int c, const float2* coils);
size_t op_ws_bytes(const Op* op);
size_t op_ws_bytes_compressed(const Op* op, int s);
int op_apply(Op* op, const float2* X, float2* Y, void* ws, cudaStream_t st);
int op_adjoint(Op* op, const float2* Y, float2* X, void* ws, cudaStream_t st);
int op_apply_compressed(Op* op, const float2* Xc, const float2* V, int s, float2* Y, void* ws,
                        const float2* Ymeas, const float* w, double* norm_out, cudaStream_t st);
int op_adjoint_compressed(Op* op, const float2* R, const float2* V, int s, float2* Gc, void* ws,
                          cudaStream_t st);
int vec_op(const float2* a, double alpha, const float2* b, int64_t count, const float* w, int mode,
           float2* R, double* out, void* ws, cudaStream_t st);
int scale_c64(float2* a, double alpha, int64_t count, cudaStream_t st);
int argmax_select(const double* score, const int64_t* gidx, const double* gmax, int64_t n,
                  int64_t* cand, cudaStream_t st);
size_t reduce_ws_bytes();
}  // namespace cbb

using namespace cbb;

static inline cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }

static DictView to_view(const cbb_dict_view* v) {
  DictView d{};
  d.d = v->d;
  d.s = v->s;
  d.s_pad = v->s_pad;
  d.kpad = v->kpad;
  d.n_btiles = v->n_btiles;
  d.atoms64 = static_cast<const double2*>(v->atoms64);
  d.atoms32 = static_cast<const float*>(v->atoms32);
  d.atoms_tc = static_cast<const uint8_t*>(v->atoms_tc);
  d.bounds = v->bounds;
  d.atoms_tc2 = static_cast<const uint8_t*>(v->atoms_tc2);
  d.prefer_split = v->prefer_split;
  d.n_tiles2 = v->n_tiles2;
  d.tc2_atom = v->tc2_atom;
  d.tc2_pos = v->tc2_pos;
  d.tile_c = v->tile_c;
  d.tile_r = v->tile_r;
  d.ctr_tc2 = static_cast<const uint8_t*>(v->ctr_tc2);
  d.tile_rs = v->tile_rs;
  return d;
}

static int check_view(const cbb_dict_view* v) {
  if (!v || v->d <= 0 || v->s <= 0 || !v->atoms64) {
    set_last_error("invalid dictionary view");
    return kErrArgument;
  }
  return kOk;
}

extern "C" {

int cbb_abi_version(void) { return CBB_ABI_VERSION; }
const char* cbb_last_error(void) { return g_last_error.c_str(); }

int cbb_device_sm_count(int* out) {
  int dev = 0;
  CBB_CUDA_TRY(cudaGetDevice(&dev));
  CBB_CUDA_TRY(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev));
  return kOk;
}

size_t cbb_dict_storage_bytes(int64_t d, int32_t s) {
  return dict_bytes(d, s, nullptr, nullptr, nullptr, nullptr, nullptr);
}

int cbb_dict_prepare(const void* atoms, int32_t atoms_c128, int64_t d, int32_t s, void* storage,
                     cbb_dict_view* view_out, void* stream) {
  if (!atoms || !storage || !view_out || d <= 0 || s <= 0) {
    set_last_error("cbb_dict_prepare: invalid argument");
    return kErrArgument;
  }
  DictView v{};
  int rc = dict_prepare(atoms, atoms_c128, d, s, storage, &v, S(stream));
  if (rc) return rc;
  view_out->d = v.d;
  view_out->s = v.s;
  view_out->s_pad = v.s_pad;
  view_out->kpad = v.kpad;
  view_out->n_btiles = v.n_btiles;
  view_out->atoms64 = v.atoms64;
  view_out->atoms32 = v.atoms32;
  view_out->atoms_tc = v.atoms_tc;
  view_out->bounds = v.bounds;
  view_out->atoms_tc2 = v.atoms_tc2;
  view_out->prefer_split = v.prefer_split;
  view_out->reserved = 0;
  view_out->n_tiles2 = v.n_tiles2;
  view_out->reserved2 = 0;
  view_out->tc2_atom = v.tc2_atom;
  view_out->tc2_pos = v.tc2_pos;
  view_out->tile_c = v.tile_c;
  view_out->tile_r = v.tile_r;
  view_out->ctr_tc2 = v.ctr_tc2;
  view_out->tile_rs = v.tile_rs;
  return kOk;
}

size_t cbb_project_workspace_bytes(int64_t n, int32_t s) {
  return project_ws_bytes(n, s, nullptr, nullptr, 0);
}

size_t cbb_project_workspace_bytes_dict(int64_t n, const cbb_dict_view* dict) {
  if (!dict || dict->s <= 0) return 0;
  return project_ws_bytes(n, dict->s, nullptr, nullptr, prune_tiles_of(to_view(dict)));
}

int cbb_project_cone_exact(const void* z, int32_t z_c128, int64_t n, const cbb_dict_view* dict,
                           void* idx_out, int32_t idx_int64, double* gamma_out, void* proj_out,
                           int32_t proj_c128, void* workspace, size_t workspace_bytes,
                           int32_t algo, void* stream) {
  if (int rc = check_view(dict)) return rc;
  if (n > 0 && !z) {
    set_last_error("cbb_project_cone_exact: null input");
    return kErrArgument;
  }
  ZSource zs{z, z_c128, nullptr, nullptr, 0.f, nullptr, nullptr};
  ProjOut o{idx_out, idx_int64, gamma_out, proj_out, proj_c128, nullptr, nullptr, nullptr,
            nullptr, 0};
  return project(zs, n, to_view(dict), o, nullptr, workspace, workspace_bytes, algo, 0,
                 S(stream));
}

int cbb_project_best(const void* z, int32_t z_c128, int64_t n, const cbb_dict_view* dict,
                     int64_t atom_offset, int64_t* idx_out, double* score_out, void* workspace,
                     size_t workspace_bytes, int32_t algo, void* stream) {
  if (int rc = check_view(dict)) return rc;
  if (n > 0 && (!z || !idx_out || !score_out)) {
    set_last_error("cbb_project_best: null argument");
    return kErrArgument;
  }
  ZSource zs{z, z_c128, nullptr, nullptr, 0.f, nullptr, nullptr};
  ProjOut o{idx_out, 1, nullptr, nullptr, 0, nullptr, nullptr, nullptr, score_out, atom_offset};
  return project(zs, n, to_view(dict), o, nullptr, workspace, workspace_bytes, algo, 0,
                 S(stream));
}

int cbb_scaled_rows(const cbb_dict_view* dict, int64_t atom_offset, const int64_t* idx,
                    const double* gamma, int64_t n, void* out, int32_t out_c128, void* stream) {
  if (int rc = check_view(dict)) return rc;
  return scaled_rows(to_view(dict), atom_offset, idx, gamma, n, out, out_c128, S(stream));
}

int cbb_project_step(const void* x, const void* g, double mu, void* z_out, int64_t n,
                     const cbb_dict_view* dict, const int32_t* idx_hint, int32_t* idx_out,
                     double* gamma_out, void* xnext_out, void* dx_out, double* nd_out,
                     void* workspace, size_t workspace_bytes, int32_t algo, void* stream) {
  if (int rc = check_view(dict)) return rc;
  if (n > 0 && (!x || !g || !z_out || !xnext_out || !dx_out)) {
    set_last_error("cbb_project_step: null argument");
    return kErrArgument;
  }
  ZSource zs{nullptr, 0, static_cast<const float2*>(x), static_cast<const float2*>(g), float(mu),
             static_cast<float2*>(z_out), idx_hint};
  ProjOut o{idx_out, 0, gamma_out, xnext_out, 0, static_cast<const float2*>(x),
            static_cast<float2*>(dx_out), nullptr, nullptr, 0};
  return project(zs, n, to_view(dict), o, nd_out, workspace, workspace_bytes, algo, 0, S(stream));
}

int cbb_project_step_ex(const void* x, const void* g, double mu, const float* mu_dev,
                        void* z_out, int64_t n, const cbb_dict_view* dict,
                        const int32_t* idx_hint, const int32_t* idx_hint2, int32_t* idx_out,
                        double* gamma_out, void* xnext_out, void* dx_out, double* nd_out,
                        void* workspace, size_t workspace_bytes, int32_t algo, void* stream) {
  if (int rc = check_view(dict)) return rc;
  if (n > 0 && (!x || !g || !z_out || !xnext_out || !dx_out)) {
    set_last_error("cbb_project_step_ex: null argument");
    return kErrArgument;
  }
  ZSource zs{nullptr, 0, static_cast<const float2*>(x), static_cast<const float2*>(g), float(mu),
             static_cast<float2*>(z_out), idx_hint, mu_dev, idx_hint2};
  ProjOut o{idx_out, 0, gamma_out, xnext_out, 0, static_cast<const float2*>(x),
            static_cast<float2*>(dx_out), nullptr, nullptr, 0};
  return project(zs, n, to_view(dict), o, nd_out, workspace, workspace_bytes, algo, 0, S(stream));
}

// The representatives sit about one tile radius apart: far outside the fp16 screen's window, so
// the cheaper fp16 screen (algo 1) serves them even though the dictionary they come from is
// coherent (auto mode would pick the split screen for them too).  Small representative sets fall
// back to auto (the tcgen05 screens need d > 320).
static int rep_algo(const cbb_dict_view* reps) { return (reps->d > 320 && 2 * reps->s < 64) ? 1 : 0; }

int cbb_project_hint(const void* x, const void* g, double mu, const float* mu_dev, void* z_out,
                     int64_t n, const cbb_dict_view* reps, const int32_t* rep_atoms,
                     int32_t* hint_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_view(reps)) return rc;
  if (n > 0 && (!x || !g || !z_out || !rep_atoms || !hint_out)) {
    set_last_error("cbb_project_hint: null argument");
    return kErrArgument;
  }
  ZSource zs{nullptr, 0, static_cast<const float2*>(x), static_cast<const float2*>(g), float(mu),
             static_cast<float2*>(z_out), nullptr, mu_dev, nullptr};
  ProjOut o{hint_out, 0, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr, 0};
  if (int rc = project(zs, n, to_view(reps), o, nullptr, workspace, workspace_bytes, rep_algo(reps), 0,
                       S(stream)))
    return rc;
  return map_indices(hint_out, rep_atoms, n, reps->d, S(stream));
}

int cbb_project_overflow_count(void* workspace, int64_t n, int32_t s, int* count_host,
                               void* stream) {
  return project_overflow_count(workspace, n, s, count_host, S(stream));
}

int cbb_project_prune_stats(void* workspace, size_t workspace_bytes, int64_t n,
                            const cbb_dict_view* dict, int64_t* listed_host, int64_t* total_host,
                            void* stream) {
  if (int rc = check_view(dict)) return rc;
  if (!workspace || !listed_host || !total_host) return kErrArgument;
  return project_prune_stats(workspace, workspace_bytes, n, to_view(dict), listed_host,
                             total_host, S(stream));
}

int cbb_project_prune_detail(void* workspace, size_t workspace_bytes, int64_t n,
                             const cbb_dict_view* dict, int32_t* counts_host,
                             int32_t* buckets_host, void* stream) {
  if (int rc = check_view(dict)) return rc;
  if (!workspace || !counts_host || !buckets_host) return kErrArgument;
  return project_prune_detail(workspace, workspace_bytes, n, to_view(dict), counts_host,
                              buckets_host, S(stream));
}

int cbb_project_overflow_counts(void* workspace, int64_t n, int32_t s, int32_t* counts_host,
                                void* stream) {
  if (!workspace || !counts_host) return kErrArgument;
  return project_overflow_counts(workspace, n, s, counts_host, S(stream));
}

int cbb_project_prologue(const void* z, int32_t z_c128, int64_t n, const cbb_dict_view* dict,
                         void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_view(dict)) return rc;
  if (workspace_bytes < project_ws_bytes(n, dict->s, nullptr, nullptr, 0)) return kErrArgument;
  ZSource zs{z, z_c128, nullptr, nullptr, 0.f, nullptr, nullptr};
  return prologue_only(zs, n, to_view(dict), workspace, S(stream));
}

int cbb_debug_tc_scores(void* workspace, const cbb_dict_view* dict, int32_t a_tile,
                        int32_t b_tile, float* out, void* stream) {
  if (int rc = check_view(dict)) return rc;
  if (2 * dict->s >= 64) return kErrUnsupported;
  // voxel tiles sit at the start of the projection workspace
  return tc_debug_scores(workspace, dict->atoms_tc, dict->kpad, dict->s, a_tile, b_tile, out,
                         S(stream));
}

// development only (not in the public header): per-tile clock stamps of CTA 0
__attribute__((visibility("default"))) int cbb_dev_trace_dump(long long* host, int count) {
  return trace_dump(host, count);
}

unsigned long long cbb_stats_kernel_launches(void) { return g_launches.load(); }

int cbb_timing_enable(int32_t on) {
  if (on && !g_ev[0]) {
    CBB_CUDA_TRY(cudaEventCreate(&g_ev[0]));
    CBB_CUDA_TRY(cudaEventCreate(&g_ev[1]));
  }
  g_timing = on != 0;
  return kOk;
}

int cbb_timing_last_ms(float* ms) {
  if (!g_ev[0]) return kErrArgument;
  CBB_CUDA_TRY(cudaEventSynchronize(g_ev[1]));
  CBB_CUDA_TRY(cudaEventElapsedTime(ms, g_ev[0], g_ev[1]));
  return kOk;
}

// ---------------------------------------------------------------- operator
struct cbb_op {
  Op* impl;
};

int cbb_op_create(int32_t ndim, const int32_t* dims, int32_t L, int32_t m, const int32_t* pattern,
                  int32_t flags, cbb_op** out) {
  if (!dims || !pattern || !out) {
    set_last_error("cbb_op_create: null argument");
    return kErrArgument;
  }
  Op* impl = nullptr;
  int rc = op_create(ndim, dims, L, m, pattern, flags, &impl);
  if (rc) return rc;
  *out = new cbb_op{impl};
  return kOk;
}

int cbb_op_set_coils(cbb_op* op, int32_t c, const void* coil_maps) {
  if (!op) {
    set_last_error("cbb_op_set_coils: null operator");
    return kErrArgument;
  }
  int rc = op_set_coils(op->impl, c, static_cast<const float2*>(coil_maps));
  if (rc) set_last_error("cbb_op_set_coils: need c >= 1 and a c x n map array for c > 1");
  return rc;
}

int cbb_op_destroy(cbb_op* op) {
  if (!op) return kOk;
  op_destroy(op->impl);
  delete op;
  return kOk;
}

size_t cbb_op_workspace_bytes(const cbb_op* op) { return op ? op_ws_bytes(op->impl) : 0; }
size_t cbb_op_workspace_bytes_compressed(const cbb_op* op, int32_t s) {
  return (op && s >= 1) ? op_ws_bytes_compressed(op->impl, s) : 0;
}

int cbb_op_apply(cbb_op* op, const void* X, void* Y, void* workspace, void* stream) {
  return op_apply(op->impl, static_cast<const float2*>(X), static_cast<float2*>(Y), workspace,
                  S(stream));
}

int cbb_op_adjoint(cbb_op* op, const void* Y, void* X, void* workspace, void* stream) {
  return op_adjoint(op->impl, static_cast<const float2*>(Y), static_cast<float2*>(X), workspace,
                    S(stream));
}

int cbb_op_apply_compressed(cbb_op* op, const void* Xc, const void* V, int32_t s, void* Y,
                            void* workspace, void* stream) {
  return op_apply_compressed(op->impl, static_cast<const float2*>(Xc),
                             static_cast<const float2*>(V), s, static_cast<float2*>(Y), workspace,
                             nullptr, nullptr, nullptr, S(stream));
}

int cbb_op_apply_norm2_compressed(cbb_op* op, const void* Xc, const void* V, int32_t s,
                                  double* norm_out, void* workspace, void* stream) {
  return op_apply_compressed(op->impl, static_cast<const float2*>(Xc),
                             static_cast<const float2*>(V), s, nullptr, workspace, nullptr,
                             nullptr, norm_out, S(stream));
}

int cbb_op_adjoint_compressed(cbb_op* op, const void* R, const void* V, int32_t s, void* Gc,
                              void* workspace, void* stream) {
  return op_adjoint_compressed(op->impl, static_cast<const float2*>(R),
                               static_cast<const float2*>(V), s, static_cast<float2*>(Gc),
                               workspace, S(stream));
}

// ---------------------------------------------------------------- vectors
size_t cbb_reduce_workspace_bytes(void) { return reduce_ws_bytes(); }

int cbb_residual(const void* a, const void* b, int64_t count, const float* w, void* R,
                 double* norm_out, void* workspace, void* stream) {
  return vec_op(static_cast<const float2*>(a), 1.0, static_cast<const float2*>(b), count, w, 0,
                static_cast<float2*>(R), norm_out, workspace, S(stream));
}

int cbb_scaled_residual_norm2(const void* a, double alpha, const void* b, int64_t count,
                              const float* w, double* norm_out, void* workspace, void* stream) {
  return vec_op(static_cast<const float2*>(a), alpha, static_cast<const float2*>(b), count, w, 1,
                nullptr, norm_out, workspace, S(stream));
}

int cbb_norm2_c64(const void* a, int64_t count, double* norm_out, void* workspace, void* stream) {
  return vec_op(static_cast<const float2*>(a), 1.0, nullptr, count, nullptr, 2, nullptr, norm_out,
                workspace, S(stream));
}

int cbb_scale_c64(void* a, double alpha, int64_t count, void* stream) {
  return scale_c64(static_cast<float2*>(a), alpha, count, S(stream));
}

int cbb_argmax_select(const double* score, const int64_t* gidx, const double* gmax, int64_t n,
                      int64_t* cand_out, void* stream) {
  return argmax_select(score, gidx, gmax, n, cand_out, S(stream));
}

}  // extern "C"

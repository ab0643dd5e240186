// api.cu -- the C ABI declared in include/ganq.h: argument checks, workspace carving and
// the Algorithm 1 driver.  Every arithmetic step runs in the kernels of
// hessian.cu, cholesky.cu, sstep_tc.cu, tgram_tc.cu, tstep.cu, gemm.cu and gemm_tc.cu.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "ganq_internal.cuh"

namespace ganq {

static thread_local char g_msg[512] = "";
static thread_local int64_t g_index = -1;

void set_error(ganq_status_t, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof g_msg, fmt, ap);
  va_end(ap);
  g_index = -1;
}
void set_error_index(int64_t idx) { g_index = idx; }
ganq_status_t cuda_fail(cudaError_t e, const char* where) {
  set_error(GANQ_ERR_CUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e),
            where);
  return GANQ_ERR_CUDA;
}

// ---------------------------------------------------------------- instrumentation
static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

enum Stage {
  ST_HESSIAN = 0, ST_PRECOND, ST_CHOLESKY, ST_DERIVE, ST_GEMM_WH, ST_INIT, ST_SSTEP, ST_TGRAM,
  ST_OBJECTIVE, ST_COPY, ST_TSTEP_ONLY, ST_FACTOR_COPY, ST_TSOLVE, ST_COUNT
};
static const char* kStageNames[ST_COUNT] = {
    "hessian", "precondition", "cholesky", "derive_operands", "gemm_wh", "init_codebook",
    "sstep", "tgram", "objective", "copy", "tstep_api", "factor_copy", "tsolve"};
static_assert(ST_COUNT == GANQ_PROFILE_STAGES, "stage table");

struct Prof {
  bool on = false;
  struct Rec { int stage; cudaEvent_t a, b; int64_t launches; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double ms[ST_COUNT] = {};
  int64_t launches[ST_COUNT] = {};
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
static thread_local Prof g_prof;

struct StageScope {
  int stage;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  int64_t l0;
  StageScope(int s, cudaStream_t stream) : stage(s), st(stream), l0(g_launches.load()) {
    if (g_prof.on) { a = g_prof.get(); cudaEventRecord(a, st); }
  }
  ~StageScope() {
    if (g_prof.on && a) {
      cudaEvent_t b = g_prof.get();
      cudaEventRecord(b, st);
      g_prof.recs.push_back({stage, a, b, g_launches.load() - l0});
    }
  }
};
#define GANQ_STAGE(s) StageScope _stage_scope_##__LINE__(s, st)

namespace {

struct Layout {
  size_t A64, Lhat, LTq, tL, Eq, sE, hdiag, H32, WH, E, EH, G, Dv, b, cnt, fb, Hq, qscale, Xhi, Xlo, Hhi,
      Hlo, status, mean, per_row, total_d, end;
};

Layout make_layout(int64_t m, int64_t n, int nlev) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t nn = (size_t)n * (size_t)n, mn = (size_t)m * (size_t)n;
  L.A64 = take(nn * sizeof(double));
  const size_t np = (size_t)ss_pitch(n);
  L.Lhat = take((size_t)n * np * sizeof(float));
  const size_t npq = (size_t)ssq_pitch(n), nblk = npq / 64, mq = ((size_t)m + 31) / 32 * 32;
  L.LTq = take(3 * (size_t)n * npq);               // int8 digits of LhatT (R-15)
  L.tL = take(nblk * (size_t)n * sizeof(float));   // per-block column maxima, then the column scales
  L.Eq = take(3 * (size_t)m * npq);                // int8 digits of the residuals E
  L.sE = take((align_up((size_t)ss_panels(n) * n, 64) + (size_t)ss_panels(n) * mq) * sizeof(float));  // scales per source panel: LhatT columns, then E rows
  L.hdiag = take((size_t)n * sizeof(double));      // H_jj (T-update right-hand side)
  L.H32 = take(nn * sizeof(float));
  L.WH = take(mn * sizeof(float));
  L.E = take(mn * sizeof(float));
  L.EH = take(mn * sizeof(float));
  L.G = take(4 * (size_t)m * nlev * nlev * sizeof(double));  // 4 partial C's (tgram_tc split)
  L.Dv = take((size_t)m * nlev * sizeof(double));
  L.b = take((size_t)m * nlev * sizeof(double));
  L.cnt = take((size_t)m * nlev * sizeof(int));
  L.fb = take((size_t)m * sizeof(int));
  const size_t P = (size_t)tq_pitch(n);
  L.Hq = take(3 * P * P);
  L.qscale = take(P * sizeof(double));
  const size_t kp = (size_t)gemm_pitch(n);
  L.Xhi = take((size_t)m * kp * sizeof(float));  // tf32 split of W (then of E for the objective)
  L.Xlo = take((size_t)m * kp * sizeof(float));
  L.Hhi = take((size_t)n * kp * sizeof(float));  // tf32 split of H32
  L.Hlo = take((size_t)n * kp * sizeof(float));
  L.status = take(2 * sizeof(int));  // [0] first non-positive pivot, [1] panel-kernel ticket
  L.mean = take(sizeof(double));
  L.per_row = take((size_t)m * sizeof(double));
  L.total_d = take(sizeof(double));
  L.end = off;
  return L;
}

template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + off);
}
// the sE region: LhatT scales per (source panel, column), then E scales per (source panel, row)
float* tlp_of(void* ws, const Layout& L) { return at<float>(ws, L.sE); }
float* sep_of(void* ws, const Layout& L, int64_t n) { return at<float>(ws, L.sE) + align_up((size_t)ss_panels(n) * n, 64); }

ganq_status_t check_shape(int64_t m, int64_t n, int n_bits) {
  if (m < 1 || n < 1) {
    set_error(GANQ_ERR_INVALID_ARG, "m = %lld and n = %lld must be >= 1", (long long)m, (long long)n);
    return GANQ_ERR_INVALID_ARG;
  }
  if (n_bits < 1 || n_bits > 8) {
    set_error(GANQ_ERR_INVALID_ARG, "n_bits = %d outside [1, 8]", n_bits);
    return GANQ_ERR_INVALID_ARG;
  }
  if (n_bits > 4) {
    set_error(GANQ_ERR_UNSUPPORTED, "n_bits = %d: this build supports N <= 4 (2^N <= 16 levels)",
              n_bits);
    return GANQ_ERR_UNSUPPORTED;
  }
  if (n > (int64_t)1 << 20 || m > (int64_t)1 << 26) {
    set_error(GANQ_ERR_UNSUPPORTED, "shape too large (m = %lld, n = %lld)", (long long)m,
              (long long)n);
    return GANQ_ERR_UNSUPPORTED;
  }
  return GANQ_OK;
}

ganq_status_t check_opts(const ganq_opts_t& o) {
  if (o.precond < 0 || o.precond > 2) {
    set_error(GANQ_ERR_INVALID_ARG, "unknown preconditioning policy %d", o.precond);
    return GANQ_ERR_INVALID_ARG;
  }
  if (o.precond == GANQ_PRECOND_FIXED_LAMBDA && !(o.lambda > 0.0)) {
    set_error(GANQ_ERR_INVALID_ARG, "FIXED_LAMBDA needs lambda > 0 (got %g)", o.lambda);
    return GANQ_ERR_INVALID_ARG;
  }
  if (o.precond == GANQ_PRECOND_ADAPTIVE && !(o.tau >= 0.0)) {
    set_error(GANQ_ERR_INVALID_ARG, "ADAPTIVE needs tau >= 0 (got %g)", o.tau);
    return GANQ_ERR_INVALID_ARG;
  }
  if (o.empty_level_rule != 0 && o.empty_level_rule != 1) {
    set_error(GANQ_ERR_INVALID_ARG, "empty_level_rule must be 0 or 1");
    return GANQ_ERR_INVALID_ARG;
  }
  return GANQ_OK;
}

// Preconditioned factor into ws.A64; reports NOT_PD (synchronises the stream).
ganq_status_t factor(const double* H, int64_t n, const ganq_opts_t& o, void* ws, const Layout& L,
                     double* delta, cudaStream_t st) {
  double* A = at<double>(ws, L.A64);
  int* status = at<int>(ws, L.status);
  ganq_status_t s;
  {
    GANQ_STAGE(ST_PRECOND);
    s = launch_precondition(H, n, o.precond, o.lambda, o.tau, A, delta, at<double>(ws, L.mean), st);
    if (s) return s;
  }
  GANQ_CUDA_TRY(cudaMemsetAsync(status, 0x7f, sizeof(int), st));
  GANQ_CUDA_TRY(cudaMemsetAsync(status + 1, 0, sizeof(int), st));
  {
    GANQ_STAGE(ST_CHOLESKY);
    if ((s = launch_cholesky(A, n, status, status + 1, st))) return s;
  }
  int h_status = 0;
  GANQ_CUDA_TRY(cudaMemcpyAsync(&h_status, status, sizeof(int), cudaMemcpyDeviceToHost, st));
  GANQ_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_status < n) {
    set_error(GANQ_ERR_NOT_PD, "cholesky: non-positive pivot at %d", h_status);
    set_error_index(h_status);
    return GANQ_ERR_NOT_PD;
  }
  return GANQ_OK;
}

// f = sum_i e_i H32 e_i^T with E, EH, per_row scratch; result left in ws.total_d (device).
// Hhi/Hlo: the tf32 split of H32 (already computed); Xhi/Xlo: scratch for the split of E.
ganq_status_t objective_device(const float* W, const uint8_t* Q, const float* T, const float* Hhi,
                               const float* Hlo, int64_t m, int64_t n, int nlev, float* E, float* Xhi,
                               float* Xlo, float* EH, double* per_row, double* total, cudaStream_t st) {
  ganq_status_t s;
  GANQ_STAGE(ST_OBJECTIVE);
  if ((s = launch_residual(W, Q, T, m, n, nlev, E, st))) return s;
  if ((s = launch_split_tf32(E, m, n, Xhi, Xlo, st))) return s;
  if ((s = launch_gemm_tf32x3(Xhi, Xlo, Hhi, Hlo, m, n, n, EH, st))) return s;
  if ((s = launch_rowdot(E, EH, m, n, per_row, st))) return s;
  return launch_sum(per_row, m, total, st);
}

// Side stream (and fork / join events) of ganq_quantize_layer, one per host thread and device.
struct SideStream {
  int device = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream() {
  static thread_local SideStream sd;
  int dev = 0;
  cudaGetDevice(&dev);
  if (sd.device != dev) {
    // lowest priority: the factorisation's latency-bound panel chain keeps the SMs it asks for
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&sd.s, cudaStreamNonBlocking, lo);
    cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming);
    sd.device = dev;
  }
  return sd;
}

}  // namespace
}  // namespace ganq

using namespace ganq;

extern "C" {

void ganq_default_opts(ganq_opts_t* o) {
  if (!o) return;
  memset(o, 0, sizeof *o);
  o->precond = GANQ_PRECOND_ADAPTIVE;
  o->empty_level_rule = 0;
  o->lambda = 0.0;
  o->tau = 1e-7;
  o->T0 = nullptr;
  o->obj_trace = nullptr;
}

int ganq_profile_enable(int on) {
  for (auto& r : g_prof.recs) { g_prof.pool.push_back(r.a); g_prof.pool.push_back(r.b); }
  g_prof.recs.clear();
  for (int i = 0; i < ST_COUNT; ++i) { g_prof.ms[i] = 0.0; g_prof.launches[i] = 0; }
  g_prof.on = on != 0;
  return 0;
}

int ganq_profile_read(double* ms, int64_t* launches, int max_stages) {
  for (auto& r : g_prof.recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) == cudaSuccess && cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess)
      g_prof.ms[r.stage] += t;
    g_prof.launches[r.stage] += r.launches;
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.recs.clear();
  const int k = max_stages < ST_COUNT ? max_stages : ST_COUNT;
  for (int i = 0; i < k; ++i) {
    if (ms) ms[i] = g_prof.ms[i];
    if (launches) launches[i] = g_prof.launches[i];
  }
  return ST_COUNT;
}

const char* ganq_profile_stage_name(int stage) {
  return (stage >= 0 && stage < ST_COUNT) ? kStageNames[stage] : "";
}

int64_t ganq_launch_count(void) { return g_launches.load(); }

const char* ganq_last_error(void) { return g_msg; }
int64_t ganq_last_error_index(void) { return g_index; }
int64_t ganq_packed_row_bytes(int64_t n, int n_bits) {
  if (n < 1 || n_bits < 1 || n_bits > 8) return 0;
  return (n * n_bits + 7) / 8;
}

ganq_status_t ganq_pack_codes(const uint8_t* Q, int64_t m, int64_t n, int n_bits, uint8_t* packed,
                              void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (m < 1 || n < 1 || n_bits < 1 || n_bits > 8 || !Q || !packed) {
    set_error(GANQ_ERR_INVALID_ARG, "pack_codes: need m, n >= 1, n_bits in [1, 8], non-null buffers");
    return GANQ_ERR_INVALID_ARG;
  }
  return launch_pack_codes(Q, m, n, n_bits, packed, (cudaStream_t)stream);
}

ganq_status_t ganq_codebook_f16(const float* T, int64_t m, int n_bits, uint16_t* T16, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (m < 1 || n_bits < 1 || n_bits > 8 || !T || !T16) {
    set_error(GANQ_ERR_INVALID_ARG, "codebook_f16: need m >= 1, n_bits in [1, 8], non-null buffers");
    return GANQ_ERR_INVALID_ARG;
  }
  return launch_codebook_f16(T, m * ((int64_t)1 << n_bits), T16, (cudaStream_t)stream);
}

ganq_status_t ganq_lut_gemm(const uint8_t* packed, const uint16_t* T16, const uint16_t* X, int64_t m,
                            int64_t n, int64_t p, int n_bits, float* Y, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (m < 1 || n < 1 || p < 1 || n_bits < 1 || n_bits > 8 || !packed || !T16 || !X || !Y) {
    set_error(GANQ_ERR_INVALID_ARG, "lut_gemm: need m, n, p >= 1, n_bits in [1, 8], non-null buffers");
    return GANQ_ERR_INVALID_ARG;
  }
  return launch_lut_gemm(packed, T16, X, m, n, p, n_bits, Y, (cudaStream_t)stream);
}

ganq_status_t ganq_outlier_split(const float* W, int64_t m, int64_t n, double r, float* W_dense, float* c_lower,
                                 float* c_upper, int64_t* row_offsets, int64_t* nnz, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (m < 1 || n < 2 || !(r > 0.0 && r < 1.0) || !W || !W_dense || !c_lower || !c_upper || !row_offsets || !nnz) {
    set_error(GANQ_ERR_INVALID_ARG, "outlier_split: need m >= 1, n >= 2, 0 < r < 1, non-null buffers");
    return GANQ_ERR_INVALID_ARG;
  }
  if (n > 57344) {
    set_error(GANQ_ERR_UNSUPPORTED, "outlier_split: n = %lld exceeds the shared-memory row (57344)", (long long)n);
    return GANQ_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  ganq_status_t s = launch_outlier_split(W, m, n, r, W_dense, c_lower, c_upper, row_offsets, st);
  if (s) return s;
  GANQ_CUDA_TRY(cudaMemcpyAsync(nnz, row_offsets + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GANQ_CUDA_TRY(cudaStreamSynchronize(st));
  return GANQ_OK;
}

ganq_status_t ganq_outlier_csr(const float* W, int64_t m, int64_t n, const float* c_lower, const float* c_upper,
                               const int64_t* row_offsets, int32_t* col_idx, float* values, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (m < 1 || n < 1 || !W || !c_lower || !c_upper || !row_offsets || !col_idx || !values) {
    set_error(GANQ_ERR_INVALID_ARG, "outlier_csr: need m, n >= 1, non-null buffers");
    return GANQ_ERR_INVALID_ARG;
  }
  return launch_outlier_csr(W, m, n, c_lower, c_upper, row_offsets, col_idx, values, (cudaStream_t)stream);
}

ganq_status_t ganq_sparse_gemm_add(const int64_t* row_offsets, const int32_t* col_idx, const float* values,
                                   int64_t m, int64_t n, const uint16_t* X, int64_t p, float* Y, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (m < 1 || n < 1 || p < 1 || !row_offsets || !X || !Y) {
    set_error(GANQ_ERR_INVALID_ARG, "sparse_gemm_add: need m, n, p >= 1, non-null buffers");
    return GANQ_ERR_INVALID_ARG;
  }
  return launch_sparse_gemm_add(row_offsets, col_idx, values, m, n, X, p, Y, (cudaStream_t)stream);
}

ganq_status_t ganq_kmeans_codebook(const float* W, int64_t m, int64_t n, int n_bits, int iters, float* T,
                                   void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (m < 1 || n < 1 || n_bits < 1 || n_bits > 8 || iters < 0 || !W || !T) {
    set_error(GANQ_ERR_INVALID_ARG, "kmeans_codebook: need m, n >= 1, n_bits in [1, 8], iters >= 0, non-null buffers");
    return GANQ_ERR_INVALID_ARG;
  }
  if (n_bits > 4) {
    set_error(GANQ_ERR_UNSUPPORTED, "kmeans_codebook: n_bits = %d, this build supports N <= 4", n_bits);
    return GANQ_ERR_UNSUPPORTED;
  }
  return launch_kmeans_codebook(W, m, n, 1 << n_bits, iters, T, (cudaStream_t)stream);
}

const char* ganq_version(void) { return "ganq-b200 0.1 (sm_100a)"; }

static ganq_status_t hessian_common(const uint16_t* X, int64_t p, int64_t n, const void* out, cudaStream_t st) {
  if (p < 1 || n < 1 || !X || !out) {
    set_error(GANQ_ERR_INVALID_ARG, "ganq_hessian: p = %lld, n = %lld must be >= 1 and pointers set",
              (long long)p, (long long)n);
    return GANQ_ERR_INVALID_ARG;
  }
  if (validate_enabled()) {
    ganq_status_t s = validate_finite_bf16(X, p, n, "X", st);
    if (s) return s;
  }
  return check_hessian_args(X, p, n);
}

size_t ganq_hessian_fixed_size(int64_t n) { return n < 1 ? 0 : hessian_fixed_bytes(n); }
size_t ganq_hessian_partials_size(int64_t p, int64_t n) { return (p < 1 || n < 1) ? 0 : hessian_partials_bytes(p, n); }

size_t ganq_hessian_workspace_size(int64_t p, int64_t n) {
  return (p < 1 || n < 1) ? 0 : align_up((size_t)n * sizeof(int32_t), 256) + hessian_partials_bytes(p, n);
}

ganq_status_t ganq_hessian_partials(const uint16_t* X, int64_t p, int64_t n, float* partials, int32_t* E,
                                    void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  cudaStream_t st = (cudaStream_t)stream;
  ganq_status_t s = hessian_common(X, p, n, partials, st);
  if (s) return s;
  if (!E) {
    set_error(GANQ_ERR_INVALID_ARG, "ganq_hessian_partials: E must be set");
    return GANQ_ERR_INVALID_ARG;
  }
  GANQ_STAGE(ST_HESSIAN);
  return launch_hessian_partials(X, p, n, partials, E, st);
}

ganq_status_t ganq_hessian_fixed(const float* partials, int64_t p, int64_t n, const int32_t* E, int64_t* Hfix,
                                 int accumulate, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (p < 1 || n < 1 || !partials || !E || !Hfix) {
    set_error(GANQ_ERR_INVALID_ARG, "ganq_hessian_fixed: p, n >= 1 and non-null pointers needed");
    return GANQ_ERR_INVALID_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  GANQ_STAGE(ST_HESSIAN);
  return launch_hessian_fixed(partials, p, n, E, reinterpret_cast<long long*>(Hfix), accumulate, st);
}

ganq_status_t ganq_hessian_finalize(const int64_t* Hfix, const int32_t* E, int64_t n, double* H, int accumulate,
                                    void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  if (n < 1 || !Hfix || !E || !H) {
    set_error(GANQ_ERR_INVALID_ARG, "ganq_hessian_finalize: n >= 1 and non-null pointers needed");
    return GANQ_ERR_INVALID_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  GANQ_STAGE(ST_HESSIAN);
  return launch_hessian_finalize(reinterpret_cast<const long long*>(Hfix), nullptr, 0, E, n, H, accumulate, st);
}

ganq_status_t ganq_hessian_ws(const uint16_t* X, int64_t p, int64_t n, double* H, int accumulate, void* workspace,
                              size_t workspace_bytes, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  cudaStream_t st = (cudaStream_t)stream;
  ganq_status_t s = hessian_common(X, p, n, H, st);
  if (s) return s;
  const size_t need = ganq_hessian_workspace_size(p, n);
  if (!workspace || workspace_bytes < need) {
    set_error(GANQ_ERR_WORKSPACE, "hessian workspace of %zu bytes < required %zu", workspace_bytes, need);
    return GANQ_ERR_WORKSPACE;
  }
  int32_t* E = reinterpret_cast<int32_t*>(workspace);
  float* P = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + align_up((size_t)n * sizeof(int32_t), 256));
  GANQ_STAGE(ST_HESSIAN);
  if ((s = launch_hessian_partials(X, p, n, P, E, st))) return s;
  return launch_hessian_finalize(nullptr, P, p, E, n, H, accumulate, st);
}

ganq_status_t ganq_hessian(const uint16_t* X, int64_t p, int64_t n, double* H, int accumulate,
                           void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  cudaStream_t st = (cudaStream_t)stream;
  ganq_status_t s = hessian_common(X, p, n, H, st);
  if (s) return s;
  // scratch from the current device's stream-ordered pool, kept cached between calls
  {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  const size_t need = ganq_hessian_workspace_size(p, n);
  void* ws = nullptr;
  GANQ_CUDA_TRY(cudaMallocAsync(&ws, need, st));
  s = ganq_hessian_ws(X, p, n, H, accumulate, ws, need, stream);
  const cudaError_t e = cudaFreeAsync(ws, st);
  if (s) return s;
  if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return GANQ_OK;
}

size_t ganq_workspace_size(int64_t m, int64_t n, int n_bits) {
  if (m < 1 || n < 1 || n_bits < 1 || n_bits > 8) return 0;
  return make_layout(m, n, 1 << n_bits).end;
}

ganq_status_t ganq_quantize_layer(const float* W, int64_t m, int64_t n, const double* H, int n_bits,
                                  int iters, const ganq_opts_t* opts, uint8_t* Q, float* T,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  ganq_status_t s;
  if ((s = check_shape(m, n, n_bits))) return s;
  if (iters < 1) {
    set_error(GANQ_ERR_INVALID_ARG, "iters = %d must be >= 1", iters);
    return GANQ_ERR_INVALID_ARG;
  }
  if (!W || !H || !Q || !T) {
    set_error(GANQ_ERR_INVALID_ARG, "null W/H/Q/T");
    return GANQ_ERR_INVALID_ARG;
  }
  ganq_opts_t o;
  ganq_default_opts(&o);
  if (opts) o = *opts;
  if ((s = check_opts(o))) return s;
  const int nlev = 1 << n_bits;
  const Layout L = make_layout(m, n, nlev);
  if (!workspace || workspace_bytes < L.end) {
    set_error(GANQ_ERR_WORKSPACE, "workspace of %zu bytes < required %zu", workspace_bytes, L.end);
    return GANQ_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  void* ws = workspace;
  if (validate_enabled()) {
    if ((s = validate_finite_f32(W, m, n, "W", st))) return s;
    if ((s = validate_finite_f64(H, n, n, "H", st))) return s;
  }
  float* Lhat = at<float>(ws, L.Lhat);
  float* H32 = at<float>(ws, L.H32);
  float* WH = at<float>(ws, L.WH);
  float* E = at<float>(ws, L.E);
  float* EH = at<float>(ws, L.EH);
  float* Hhi = at<float>(ws, L.Hhi);
  float* Hlo = at<float>(ws, L.Hlo);
  // Everything that needs only H and W runs on a side stream forked here, so that it overlaps
  // the preconditioned Cholesky factorisation on `st` (which also synchronises `st` once to
  // report NOT_PD): fp32 H, H_jj, the int8 digits of H for the T-update, W H, T^0.
  SideStream& sd = side_stream();
  GANQ_CUDA_TRY(cudaEventRecord(sd.fork, st));
  GANQ_CUDA_TRY(cudaStreamWaitEvent(sd.s, sd.fork, 0));
  {
    cudaStream_t st = sd.s;  // (the stage scopes below time on the side stream)
    {
      GANQ_STAGE(ST_DERIVE);
      if ((s = launch_derive_operands(nullptr, H, n, nullptr, H32, st))) return s;
      if ((s = launch_hdiag(H, n, at<double>(ws, L.hdiag), st))) return s;
      // E scales of rows >= m are never written but are read (multiplied by zero digits)
      GANQ_CUDA_TRY(cudaMemsetAsync(sep_of(ws, L, n), 0, (size_t)ss_panels(n) * (((size_t)m + 31) / 32 * 32) * sizeof(float),
                                    st));
      // fixed-point int8 digits of H's strict lower triangle for the tensor-core T-update
      if ((s = launch_tq_prep(H, n, at<int8_t>(ws, L.Hq), at<double>(ws, L.qscale), st))) return s;
    }
    {
      // W H (fixed across iterations: W_i H S_i^T of Eq. 6), tf32x3 on the tensor cores
      GANQ_STAGE(ST_GEMM_WH);
      if ((s = launch_split_tf32(H32, n, n, Hhi, Hlo, st))) return s;
      if ((s = launch_split_tf32(W, m, n, at<float>(ws, L.Xhi), at<float>(ws, L.Xlo), st))) return s;
      if ((s = launch_gemm_tf32x3(at<float>(ws, L.Xhi), at<float>(ws, L.Xlo), Hhi, Hlo, m, n, n, WH, st)))
        return s;
    }
    {
      // T^0 (reading R-6)
      GANQ_STAGE(ST_INIT);
      if (o.T0) {
        GANQ_CUDA_TRY(cudaMemcpyAsync(T, o.T0, sizeof(float) * (size_t)m * nlev, cudaMemcpyDeviceToDevice, st));
      } else if ((s = launch_init_codebook(W, m, n, nlev, T, st))) {
        return s;
      }
    }
    GANQ_CUDA_TRY(cudaMemsetAsync(at<int>(ws, L.fb), 0, sizeof(int) * (size_t)m, st));
    GANQ_CUDA_TRY(cudaEventRecord(sd.join, st));
  }
  // H' = precondition(H), L = Cholesky(H')   (App. A / Remark 1, Eq. 9)
  s = factor(H, n, o, ws, L, nullptr, st);
  if (!s) {
    GANQ_STAGE(ST_DERIVE);
    s = launch_lhat_prep(at<double>(ws, L.A64), n, Lhat, at<int8_t>(ws, L.LTq), tlp_of(ws, L), at<float>(ws, L.tL),
                         st);
  }
  // join (also on an error: no side-stream work may outlive the call's use of the workspace)
  GANQ_CUDA_TRY(cudaStreamWaitEvent(st, sd.join, 0));
  if (s) return s;
  for (int k = 0; k < iters; ++k) {
    {
      // S-update
      GANQ_STAGE(ST_SSTEP);
      if ((s = launch_sstep_tc(W, Lhat, at<int8_t>(ws, L.LTq), tlp_of(ws, L), T, m, n, nlev, Q,
                               at<int8_t>(ws, L.Eq), sep_of(ws, L, n), st)))
        return s;
    }
    {
      // T-update, raw H (reading R-4)
      {
        GANQ_STAGE(ST_TGRAM);
        if ((s = launch_tgram_tc(at<int8_t>(ws, L.Hq), at<double>(ws, L.qscale), Q, m, n, nlev,
                                 at<double>(ws, L.G), st)))
          return s;
      }
      GANQ_STAGE(ST_TSOLVE);
      if ((s = launch_tsolve(at<double>(ws, L.hdiag), WH, Q, m, n, nlev, o.empty_level_rule, T, at<double>(ws, L.G),
                             at<double>(ws, L.Dv), at<double>(ws, L.b), at<int>(ws, L.cnt), at<int>(ws, L.fb),
                             st)))
        return s;
    }
    if (o.obj_trace) {
      if ((s = objective_device(W, Q, T, Hhi, Hlo, m, n, nlev, E, at<float>(ws, L.Xhi), at<float>(ws, L.Xlo),
                                EH, at<double>(ws, L.per_row), at<double>(ws, L.total_d), st)))
        return s;
      GANQ_CUDA_TRY(cudaMemcpyAsync(&o.obj_trace[k], at<double>(ws, L.total_d), sizeof(double),
                                    cudaMemcpyDeviceToHost, st));
      GANQ_CUDA_TRY(cudaStreamSynchronize(st));
    }
  }
  GANQ_LAUNCH_CHECK("ganq_quantize_layer");
  return GANQ_OK;
}

size_t ganq_objective_workspace_size(int64_t m, int64_t n) {
  if (m < 1 || n < 1) return 0;
  const size_t kp = (size_t)gemm_pitch(n);
  size_t off = 0;
  off = align_up(off + (size_t)n * n * sizeof(float), 256);      // H32
  off = align_up(off + (size_t)m * n * sizeof(float), 256);      // E
  off = align_up(off + (size_t)m * n * sizeof(float), 256);      // EH
  off = align_up(off + (size_t)m * sizeof(double), 256);         // per_row
  off = align_up(off + sizeof(double), 256);                     // total
  off = align_up(off + 2 * (size_t)m * kp * sizeof(float), 256); // E hi / lo
  off = align_up(off + 2 * (size_t)n * kp * sizeof(float), 256); // H hi / lo
  return off;
}

ganq_status_t ganq_objective(const float* W, const uint8_t* Q, const float* T, const double* H,
                             int64_t m, int64_t n, int n_bits, double* out, double* per_row,
                             void* workspace, size_t workspace_bytes, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  ganq_status_t s;
  if ((s = check_shape(m, n, n_bits))) {
    if (s != GANQ_ERR_UNSUPPORTED) return s;  // the objective itself supports any N <= 8
  }
  if (!W || !Q || !T || !H || !out) {
    set_error(GANQ_ERR_INVALID_ARG, "null argument");
    return GANQ_ERR_INVALID_ARG;
  }
  const size_t need = ganq_objective_workspace_size(m, n);
  if (!workspace || workspace_bytes < need) {
    set_error(GANQ_ERR_WORKSPACE, "workspace of %zu bytes < required %zu", workspace_bytes, need);
    return GANQ_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  size_t off = 0;
  float* H32 = at<float>(workspace, off);
  off = align_up(off + (size_t)n * n * sizeof(float), 256);
  float* E = at<float>(workspace, off);
  off = align_up(off + (size_t)m * n * sizeof(float), 256);
  float* EH = at<float>(workspace, off);
  off = align_up(off + (size_t)m * n * sizeof(float), 256);
  double* pr = at<double>(workspace, off);
  off = align_up(off + (size_t)m * sizeof(double), 256);
  double* tot = at<double>(workspace, off);
  off = align_up(off + sizeof(double), 256);
  const size_t kp = (size_t)gemm_pitch(n);
  float* Xhi = at<float>(workspace, off);
  float* Xlo = Xhi + (size_t)m * kp;
  off = align_up(off + 2 * (size_t)m * kp * sizeof(float), 256);
  float* Hhi = at<float>(workspace, off);
  float* Hlo = Hhi + (size_t)n * kp;
  {
    GANQ_STAGE(ST_DERIVE);
    if ((s = launch_derive_operands(nullptr, H, n, nullptr, H32, st))) return s;
    if ((s = launch_split_tf32(H32, n, n, Hhi, Hlo, st))) return s;
  }
  if ((s = objective_device(W, Q, T, Hhi, Hlo, m, n, 1 << n_bits, E, Xhi, Xlo, EH, per_row ? per_row : pr,
                            tot, st)))
    return s;
  GANQ_CUDA_TRY(cudaMemcpyAsync(out, tot, sizeof(double), cudaMemcpyDeviceToHost, st));
  GANQ_CUDA_TRY(cudaStreamSynchronize(st));
  return GANQ_OK;
}

ganq_status_t ganq_tstep(const float* W, const uint8_t* Q, const double* H, int64_t m, int64_t n,
                         int n_bits, int empty_level_rule, const float* Tprev, float* T,
                         void* workspace, size_t workspace_bytes, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  ganq_status_t s;
  if ((s = check_shape(m, n, n_bits))) return s;
  if (empty_level_rule != 0 && empty_level_rule != 1) {
    set_error(GANQ_ERR_INVALID_ARG, "empty_level_rule must be 0 or 1");
    return GANQ_ERR_INVALID_ARG;
  }
  const int nlev = 1 << n_bits;
  const Layout L = make_layout(m, n, nlev);
  if (!workspace || workspace_bytes < L.end) {
    set_error(GANQ_ERR_WORKSPACE, "workspace of %zu bytes < required %zu", workspace_bytes, L.end);
    return GANQ_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  float* H32 = at<float>(workspace, L.H32);
  float* WH = at<float>(workspace, L.WH);
  GANQ_STAGE(ST_TSTEP_ONLY);
  if ((s = launch_derive_operands(nullptr, H, n, nullptr, H32, st))) return s;
  if ((s = launch_tq_prep(H, n, at<int8_t>(workspace, L.Hq), at<double>(workspace, L.qscale), st)))
    return s;
  if ((s = launch_split_tf32(H32, n, n, at<float>(workspace, L.Hhi), at<float>(workspace, L.Hlo), st))) return s;
  if ((s = launch_split_tf32(W, m, n, at<float>(workspace, L.Xhi), at<float>(workspace, L.Xlo), st))) return s;
  if ((s = launch_gemm_tf32x3(at<float>(workspace, L.Xhi), at<float>(workspace, L.Xlo), at<float>(workspace, L.Hhi),
                              at<float>(workspace, L.Hlo), m, n, n, WH, st)))
    return s;
  if (empty_level_rule == 1 && Tprev && Tprev != T)
    GANQ_CUDA_TRY(cudaMemcpyAsync(T, Tprev, sizeof(float) * (size_t)m * nlev, cudaMemcpyDeviceToDevice, st));
  GANQ_CUDA_TRY(cudaMemsetAsync(at<int>(workspace, L.fb), 0, sizeof(int) * (size_t)m, st));
  if ((s = launch_tgram_tc(at<int8_t>(workspace, L.Hq), at<double>(workspace, L.qscale), Q, m, n, nlev,
                           at<double>(workspace, L.G), st)))
    return s;
  if ((s = launch_hdiag(H, n, at<double>(workspace, L.hdiag), st))) return s;
  return launch_tsolve(at<double>(workspace, L.hdiag), WH, Q, m, n, nlev, empty_level_rule, T, at<double>(workspace, L.G),
                       at<double>(workspace, L.Dv), at<double>(workspace, L.b), at<int>(workspace, L.cnt),
                       at<int>(workspace, L.fb), st);
}

ganq_status_t ganq_factor(const double* H, int64_t n, const ganq_opts_t* opts, double* Lout,
                          double* delta, void* workspace, size_t workspace_bytes, void* stream) {
  g_msg[0] = 0;
  g_index = -1;
  ganq_status_t s;
  if ((s = check_shape(1, n, 1))) return s;
  if (!H || !Lout) {
    set_error(GANQ_ERR_INVALID_ARG, "null H/L");
    return GANQ_ERR_INVALID_ARG;
  }
  ganq_opts_t o;
  ganq_default_opts(&o);
  if (opts) o = *opts;
  if ((s = check_opts(o))) return s;
  const Layout L = make_layout(1, n, 2);
  if (!workspace || workspace_bytes < L.end) {
    set_error(GANQ_ERR_WORKSPACE, "workspace of %zu bytes < required %zu", workspace_bytes, L.end);
    return GANQ_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = factor(H, n, o, workspace, L, delta, st))) return s;
  GANQ_CUDA_TRY(cudaMemcpyAsync(Lout, at<double>(workspace, L.A64), sizeof(double) * (size_t)n * n,
                                cudaMemcpyDeviceToDevice, st));
  return GANQ_OK;
}

}  // extern "C"

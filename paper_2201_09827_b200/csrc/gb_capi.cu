// C ABI (include/gcrodr_b200.h): argument checks, dispatch over the
// precision variants (each compiled in its own gb_var_*.cu) and the extern "C"
// entry points.
#include <cstdlib>
#include <cstring>
#include "gb_solver.cuh"

thread_local std::string g_err;

const VariantOps* gb_variant_f_h_f64() __attribute__((weak));
const VariantOps* gb_variant_f_h_f32() __attribute__((weak));
const VariantOps* gb_variant_f_f_f64() __attribute__((weak));
const VariantOps* gb_variant_f_f_f32() __attribute__((weak));
const VariantOps* gb_variant_d_h_dd() __attribute__((weak));
const VariantOps* gb_variant_d_h_f64() __attribute__((weak));
const VariantOps* gb_variant_d_f_dd() __attribute__((weak));
const VariantOps* gb_variant_d_f_f64() __attribute__((weak));
const VariantOps* gb_variant_d_d_dd() __attribute__((weak));
const VariantOps* gb_variant_d_d_f64() __attribute__((weak));

long long* gb_launch_counter() {
  static long long counter = 0;
  return &counter;
}

namespace {
const VariantOps* get_variant(const VariantOps* (*fn)(), std::string& why) {
  if (fn == nullptr) {
    why = "precision variant not compiled into this build";
    return nullptr;
  }
  return fn();
}

const VariantOps* pick_variant(const gb_options& o, std::string& why) {
  const bool extra = o.extra_precision != 0;
  if (o.u == GB_SINGLE) {
    if (o.uf == GB_HALF) return get_variant(extra ? gb_variant_f_h_f64 : gb_variant_f_h_f32, why);
    if (o.uf == GB_SINGLE) return get_variant(extra ? gb_variant_f_f_f64 : gb_variant_f_f_f32, why);
  } else if (o.u == GB_DOUBLE) {
    if (o.uf == GB_HALF) return get_variant(extra ? gb_variant_d_h_dd : gb_variant_d_h_f64, why);
    if (o.uf == GB_SINGLE) return get_variant(extra ? gb_variant_d_f_dd : gb_variant_d_f_f64, why);
    if (o.uf == GB_DOUBLE) return get_variant(extra ? gb_variant_d_d_dd : gb_variant_d_d_f64, why);
  }
  why = "working precision u must be single or double (u = half / quad are not built)";
  return nullptr;
}
}  // namespace

// ---------------------------------------------------------------------------
// extern "C"
// ---------------------------------------------------------------------------
extern "C" {

const char* gb_version(void) { return "gcrodr_b200 0.1 (sm_100a)"; }
const char* gb_last_error(void) { return g_err.c_str(); }
int gb_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

gb_status gb_solver_create(gb_solver** out, int n, const gb_options* opt, void* stream) {
  if (!out || !opt || n < 1) return fail(GB_ERR_ARG, "bad arguments");
  gb_options o = *opt;
  if (!(o.m >= 1 && o.m <= n)) return fail(GB_ERR_ARG, "restart length m must satisfy 1 <= m <= n");
  if (o.k > 32) return fail(GB_ERR_UNSUPPORTED, "recycle dimension k > 32 is not built");
  if ((o.method == GB_RGMRES_IR || o.method == GB_RSGMRES_IR) && !(o.k >= 1 && o.k < o.m))
    return fail(GB_ERR_ARG, "recycling methods need 1 <= k < m");
  if (o.max_cycles < 1) return fail(GB_ERR_ARG, "max_cycles must be >= 1");
  std::string why;
  const VariantOps* ops = pick_variant(o, why);
  if (!ops) return fail(GB_ERR_UNSUPPORTED, why);
  gb_solver* s = new gb_solver();
  s->n = n;
  s->o = o;
  s->max_cycles_cap = o.max_cycles;
  s->stream = (cudaStream_t)stream;
  s->ldv = (n + 31) & ~31;
  s->lda = (n + 31) & ~31;
  s->ops = ops;
  if (n <= kSmallN) {
    s->G = 1;
  } else {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int want = o.grid_ctas > 0 ? o.grid_ctas : std::min(sms, std::max(2, (n + 63) / 64));
    s->G = std::min(want, sms);
    // the team's MGS keeps a CTA's slice of w in registers, 4 rows per
    // thread (gb_krylov.cuh): every slice must have <= 4 * 256 rows
    auto slice = [n](int G) { return (((n + G - 1) / G) + 31) & ~31; };
    while (s->G < sms && slice(s->G) > 4 * 256) ++s->G;
    if (slice(s->G) > 4 * 256) {
      delete s;
      return fail(GB_ERR_UNSUPPORTED, "order too large for this device's team (rows per CTA > 1024)");
    }
    // a team of <= 16 CTAs runs as one thread-block cluster (hardware
    // barrier) unless GB_TEAM=grid asks for the cooperative grid barrier
    const char* team = std::getenv("GB_TEAM");
    s->cluster = s->G <= 16 && !(team && std::strcmp(team, "grid") == 0);
  }
  if (cudaEventCreate(&s->ev0) != cudaSuccess || cudaEventCreate(&s->ev1) != cudaSuccess) {
    delete s;
    return fail(GB_ERR_CUDA, "event create failed");
  }
  gb_status st = ops->setup(s);
  if (st != GB_OK) {
    if (s->mem) cudaFree(s->mem);
    delete s;
    return st;
  }
  *out = s;
  return GB_OK;
}

gb_status gb_solver_destroy(gb_solver* s) {
  if (!s) return GB_OK;
  if (s->mem) cudaFree(s->mem);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  for (cudaEvent_t e : s->tc_events) cudaEventDestroy(e);
  delete s;
  return GB_OK;
}

static gb_status set_system_any(gb_solver* s, const double* a, const double* b, int dev) {
  if (!s || !a || !b) return fail(GB_ERR_ARG, "null argument");
  gb_status st = s->ops->set_system(s, a, b, dev);
  if (st == GB_OK) {
    s->have_system = true;
    s->have_lu = s->have_x0 = false;
  }
  return st;
}
gb_status gb_set_system(gb_solver* s, const double* a, const double* b) { return set_system_any(s, a, b, 0); }
gb_status gb_set_system_device(gb_solver* s, const double* a_dev, const double* b_dev) {
  return set_system_any(s, a_dev, b_dev, 1);
}
long long gb_launch_count(void) { return *gb_launch_counter(); }

gb_status gb_factorize(gb_solver* s, int* zero_col, double* growth) {
  if (!s || !s->have_system) return fail(GB_ERR_STATE, "gb_set_system first");
  gb_status st = s->ops->factor(s, zero_col, growth);
  if (st == GB_OK) s->have_lu = (*zero_col < 0);
  return st;
}

gb_status gb_initial_solution(gb_solver* s, int* x0_reset) {
  if (!s || !s->have_lu) return fail(GB_ERR_STATE, "gb_factorize first");
  gb_status st = s->ops->x0(s, x0_reset);
  if (st == GB_OK) s->have_x0 = true;
  return st;
}

gb_status gb_reference_solution(gb_solver* s, int* ok) {
  if (!s || !s->have_system) return fail(GB_ERR_STATE, "gb_set_system first");
  return s->ops->xref(s, ok);
}

gb_status gb_refine_step(gb_solver* s, gb_step_info* info) {
  if (!s || !s->have_x0) return fail(GB_ERR_STATE, "gb_initial_solution first");
  return s->ops->step(s, info);
}

gb_status gb_last_cycles(gb_solver* s, int* iters, int* keff, int cap, int* ncycles) {
  if (!s) return fail(GB_ERR_ARG, "null solver");
  int c = std::min(cap, s->max_cycles_cap + 1);
  CK(cudaMemcpyAsync(iters, s->cycle_iters, sizeof(int) * c, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(keff, s->cycle_keff, sizeof(int) * c, cudaMemcpyDeviceToHost, s->stream));
  gb_step_info inf;
  CK(cudaMemcpyAsync(&inf, s->out, sizeof(inf), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  *ncycles = std::min(inf.ncycles, c);
  return GB_OK;
}

gb_status gb_get_solution(gb_solver* s, double* x) {
  if (!s || !x) return fail(GB_ERR_ARG, "null argument");
  return s->ops->get_x(s, x);
}

gb_status gb_get_reference(gb_solver* s, double* xref) {
  if (!s || !xref) return fail(GB_ERR_ARG, "null argument");
  CK(cudaMemcpyAsync(xref, s->xref, sizeof(double) * s->n, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return GB_OK;
}

gb_status gb_get_factors(gb_solver* s, double* lu, long long* perm) {
  if (!s || !lu || !perm) return fail(GB_ERR_ARG, "null argument");
  return s->ops->get_lu(s, lu, perm);
}

gb_status gb_apply_preconditioned(gb_solver* s, const double* v, double* w, int fmt) {
  if (!s || !s->have_lu) return fail(GB_ERR_STATE, "gb_factorize first");
  return s->ops->debug(s, v, w, 0, fmt);
}
gb_status gb_precond_rhs(gb_solver* s, const double* r, double* out, int fmt) {
  if (!s || !s->have_lu) return fail(GB_ERR_STATE, "gb_factorize first");
  return s->ops->debug(s, r, out, 1, fmt);
}
gb_status gb_residual(gb_solver* s, const double* x, double* r, int fmt) {
  if (!s || !s->have_system) return fail(GB_ERR_STATE, "gb_set_system first");
  return s->ops->debug(s, x, r, 2, fmt);
}
gb_status gb_debug_inner_solve(gb_solver* s, const double* r, int reset_recycle, double* d, gb_step_info* info) {
  if (!s || !r || !d || !info) return fail(GB_ERR_ARG, "null argument");
  if (!s->have_lu) return fail(GB_ERR_STATE, "gb_factorize first");
  if (reset_recycle) {
    CK(cudaMemsetAsync(s->keff_io, 0, 4 * sizeof(int), s->stream));
    s->parity = 0;
  }
  CK(cudaMemcpyAsync(s->rtmp, r, sizeof(double) * s->n, cudaMemcpyHostToDevice, s->stream));
  s->inner_only = 1;
  gb_status e = s->ops->step(s, info);
  s->inner_only = 0;
  if (e != GB_OK) return e;
  CK(cudaMemcpyAsync(d, s->dtmp, sizeof(double) * s->n, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return GB_OK;
}

gb_status gb_backward_errors(gb_solver* s, const double* x, double* r, double* nbe, double* cbe) {
  if (!s || !x || !nbe || !cbe) return fail(GB_ERR_ARG, "null argument");
  if (!s->have_system) return fail(GB_ERR_STATE, "gb_set_system first");
  std::vector<double> tmp;
  if (!r) {
    tmp.resize(s->n);
    r = tmp.data();
  }
  gb_status e = s->ops->debug(s, x, r, 5, s->o.ur);
  if (e != GB_OK) return e;
  gb_step_info inf;
  CK(cudaMemcpyAsync(&inf, s->out, sizeof(inf), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  *nbe = inf.nbe;
  *cbe = inf.cbe;
  return GB_OK;
}

gb_status gb_lu_solve(gb_solver* s, const double* b, double* x) {
  if (!s || !s->have_lu) return fail(GB_ERR_STATE, "gb_factorize first");
  return s->ops->debug(s, b, x, 3, s->o.uf);
}

gb_status gb_time_op(gb_solver* s, int what, int reps, double* ms_per_launch) {
  if (!s || !ms_per_launch || what < 0 || what > 3 || reps < 1) return fail(GB_ERR_ARG, "bad arguments");
  if (!s->have_lu) return fail(GB_ERR_STATE, "gb_factorize first");
  return s->ops->time_op(s, what, reps, ms_per_launch);
}

gb_status gb_debug_phaselog(gb_solver* s, int cap, unsigned long long* out) {
  if (!s) return fail(GB_ERR_ARG, "null solver");
  // GB_PLOG_HOST=1: the log lives in mapped pinned host memory, so the marks
  // written before a faulting launch can still be read afterwards
  const char* hostenv = std::getenv("GB_PLOG_HOST");
  const bool want_host = hostenv && hostenv[0] == '1';
  const size_t words = 1 + 2 * (size_t)s->plog_cap + (s->plog_host ? 256 : 0);  // host mode: + per-CTA last marks
  if (out != nullptr && s->plog != nullptr) {
    if (s->plog_host) {
      cudaStreamSynchronize(s->stream);  // may fail after a fault: the host copy is still readable
      cudaGetLastError();
      memcpy(out, s->plog, sizeof(unsigned long long) * words);
    } else {
      CK(cudaStreamSynchronize(s->stream));
      CK(cudaMemcpy(out, s->plog, sizeof(unsigned long long) * words, cudaMemcpyDeviceToHost));
    }
  }
  if (s->plog) {
    if (s->plog_host) cudaFreeHost(s->plog);
    else cudaFree(s->plog);
  }
  s->plog = nullptr;
  s->plog_cap = 0;
  if (cap > 0) {
    const size_t bytes = sizeof(unsigned long long) * (1 + 2 * (size_t)cap + (want_host ? 256 : 0));
    if (want_host) {
      CK(cudaHostAlloc(&s->plog, bytes, cudaHostAllocMapped));
      memset(s->plog, 0, bytes);
    } else {
      CK(cudaMalloc(&s->plog, bytes));
      CK(cudaMemset(s->plog, 0, bytes));
    }
    s->plog_host = want_host;
    s->plog_cap = cap;
  }
  return GB_OK;
}

gb_status gb_debug_hessenberg(gb_solver* s, double* h) {
  if (!s || !h) return fail(GB_ERR_ARG, "null argument");
  CK(cudaMemcpyAsync(h, s->H, sizeof(double) * (size_t)(s->o.m + 1) * s->o.m, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return GB_OK;
}

gb_status gb_debug_set_max_cycles(gb_solver* s, int cycles) {
  if (!s) return fail(GB_ERR_ARG, "null solver");
  if (cycles < 1 || cycles > s->max_cycles_cap)
    return fail(GB_ERR_ARG, "cycles must lie in [1, max_cycles at creation]");
  s->o.max_cycles = cycles;
  return GB_OK;
}

double gb_last_step_ms(gb_solver* s) { return s ? s->last_step_ms : 0.0; }
double gb_last_factor_ms(gb_solver* s) { return s ? s->last_factor_ms : 0.0; }

gb_status gb_lu_tc_stats(gb_solver* s, double* out) {
  if (!s || !out) return fail(GB_ERR_ARG, "null argument");
  out[0] = s->tc_update_ms;
  out[1] = s->tc_update_flop;
  out[2] = s->tc_trsm_ms;
  out[3] = s->tc_panel_ms;
  return GB_OK;
}

gb_status gb_solve_batched(int count, int n, const gb_options* opt, int i_max, double c_conv, const double* a,
                           const double* b, int on_device, gb_batch_out* out, double* device_ms, void* stream) {
  if (!opt || !a || !b || !out || count < 1 || n < 2 || i_max < 1) return fail(GB_ERR_ARG, "bad arguments");
  const gb_options& o = *opt;
  if (!(o.m >= 1 && o.m <= n)) return fail(GB_ERR_ARG, "restart length m must satisfy 1 <= m <= n");
  if (o.k > 32) return fail(GB_ERR_UNSUPPORTED, "recycle dimension k > 32 is not built");
  if ((o.method == GB_RGMRES_IR || o.method == GB_RSGMRES_IR) && !(o.k >= 1 && o.k < o.m))
    return fail(GB_ERR_ARG, "recycling methods need 1 <= k < m");
  std::string why;
  const VariantOps* ops = pick_variant(o, why);
  if (!ops) return fail(GB_ERR_UNSUPPORTED, why);
  return ops->batched(count, n, opt, i_max, c_conv, a, b, on_device, out, device_ms, (cudaStream_t)stream);
}

}  // extern "C"

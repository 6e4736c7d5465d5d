// convgpu.cu -- host runtime and C ABI of the B200 convection column path.
//
// Implements include/convgpu.h: per-device contexts owning a persistent
// device workspace (compaction list, cursors, latched failure words, the
// exp table, staging buffers sized to the high-water column count), the
// launch sequence trigger+compaction -> deep plume -> shallow(+deep zero
// fill), host<->device staging for host buffers, the reference's error
// taxonomy at the boundary (capi.cpp:51-89), and the multi-device partition
// planner.  No CPU fallback exists: without a usable sm_100 device every
// compute entry point returns CVG_ERR_DEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/convgpu.h"
#include "convgpu_kernels.cuh"

namespace {

thread_local std::string g_last_error;

cvg_status fail(cvg_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

struct CudaError {
  cudaError_t code;
  const char* what;
};

#define CVG_CUDA(x)                                  \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) throw CudaError{e_, #x}; \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  void ensure(size_t n) {
    if (n <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    CVG_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    cap = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// 2^(j/512) as double-double (hi, lo), from x87 extended precision:
// exp2l is accurate to ~1 ulp of the 64-bit significand, so hi + lo carries
// ~2^-64 relative error -- far below the final double rounding.
std::vector<double2> exp_table_host() {
  std::vector<double2> t(cvg::kExpTableSize);
  for (int j = 0; j < cvg::kExpTableSize; ++j) {
    const long double v = exp2l(static_cast<long double>(j) / cvg::kExpTableSize);
    const double hi = static_cast<double>(v);
    const double lo = static_cast<double>(v - static_cast<long double>(hi));
    t[j] = make_double2(hi, lo);
  }
  return t;
}

const char* kind_message(int kind, int kernel, int maxit, std::string* buf) {
  switch (kind) {
    case cvg::kFailActivity:
      return kernel == CVG_SHALLOW ? "shallow: non-finite activity" : "deep: non-finite activity";
    case cvg::kFailInput:
      return "ientropy: non-finite input";
    case cvg::kFailDiverged:
      return "ientropy: iterate diverged";
    case cvg::kFailNoConv:
      *buf = "ientropy: no convergence within " + std::to_string(maxit) + " iterations";
      return buf->c_str();
    default:
      return "kernel failure";
  }
}

}  // namespace

struct cvg_context {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;           // shallow kernel, concurrent with deep
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_h0 = nullptr, ev_h1 = nullptr, ev_d0 = nullptr;
  DevBuf<double2> exp_tab;
  DevBuf<int> idx;
  DevBuf<int> counters;                // [0] triggered count, [2..3] deep work cursor (u64)
  DevBuf<unsigned long long> err;      // [0] deep, [1] shallow, [2] ientropy
  DevBuf<unsigned long long> cursor;   // deep work cursor + 32 dummy words
  unsigned long long* h_err = nullptr; // pinned mirror
  int* h_count = nullptr;
  // staging for host-buffer calls
  DevBuf<double> in_s, in_T, in_q;
  DevBuf<double> dT, dq, dp, sT, sq, sp;
  DevBuf<long long> dw, sw;
  DevBuf<uint8_t> dx, sx;
  DevBuf<double> aux0, aux1;
  DevBuf<int> auxi;
  bool overlap = true;                 // split kernels on two streams, concurrently
  int shallow_minb = 8;                // shallow kernel min blocks/SM (register cap)
  const char* trace_path = nullptr;    // CVG_TRACE: dump per-block (kernel, smid, start, end)
  DevBuf<unsigned long long> trace_d, trace_s;
  cudaStream_t main_for_join = nullptr;
  int shallow_mode = 0;                // 0 plain (thread per column), 2 TMA-staged tiles
  bool pairs = false;                  // deep: two columns per warp (ILP 4)
  int shallow_persist = 0;             // overlap: persistent shallow blocks per SM (0 = grid of tiles)
  // per-kernel profiling (cvg_profile_begin/end)
  bool prof_on = false;
  int prof_cap = 0, prof_n = 0;
  std::vector<cudaEvent_t> prof_ev;  // 5 per step: start, after trigger, after deep (main stream), shallow start/end (side)
  int prof_mask_first = 0;
  // last async call
  int last_mask = 0;
  int last_maxit = 100;
  long long last_n = 0;
  bool pending = false;
};

namespace {

bool valid_columns(const cvg_columns* in, std::string* why) {
  if (in->n_columns < 0) { *why = "n_columns < 0"; return false; }
  if (in->n_columns > 0x7fffffffLL) { *why = "n_columns exceeds 2^31-1"; return false; }
  if (in->n_levels < 1 || in->n_levels > 512) { *why = "n_levels must be in [1, 512]"; return false; }
  if (in->ld < in->n_columns) { *why = "ld < n_columns"; return false; }
  if (in->n_columns > 0 && (!in->s || !in->T || !in->q)) { *why = "null input pointer"; return false; }
  return true;
}

bool valid_outputs(const cvg_outputs* o, long long n, std::string* why) {
  if (o->ld < n) { *why = "output ld < n_columns"; return false; }
  if (n > 0 && (!o->tend_T || !o->tend_q || !o->precip || !o->work_units || !o->exited_early)) {
    *why = "null output pointer";
    return false;
  }
  return true;
}

bool valid_options(const cvg_options* o, std::string* why) {
  if (o->variant < 0 || o->variant > 2) { *why = "unknown variant"; return false; }
  return true;
}

template <int VAR, bool NARROW, int NW, bool PAIRS = false>
void launch_deep_t(cvg_context* ctx, const cvg::DeepArgs& a, cudaStream_t st) {
  const int threads = NW * 32;
  const size_t smem = (size_t)cvg::kExpTableSize * cvg::kTabCopies * sizeof(double2) +
                      (size_t)NW * a.batch * a.L * sizeof(double);
  auto kern = cvg::deep_kernel<VAR, NARROW, NW, PAIRS>;
  CVG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // full shared-memory carveout, so a shallow block still fits beside it
  CVG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  kern<<<ctx->num_sms, threads, smem, st>>>(a);
  CVG_CUDA(cudaGetLastError());
}

template <int VAR>
void launch_split(cvg_context* ctx, const cvg::DeepArgs& a, const cvg::ShallowArgs& b, bool sh, bool dp,
                  cudaEvent_t* pe, cudaStream_t st) {
  // overlap: the FP64-bound deep kernel (one 20-warp block per SM, launched
  // first) and the HBM-bound shallow kernel (forked onto the side stream,
  // its blocks fill the rest of each SM) run concurrently
  const bool ov = ctx->overlap && dp;
  if (ov) CVG_CUDA(cudaEventRecord(ctx->ev_fork, st));
  if (dp) {
    if (ctx->pairs && a.L <= 32) {
      if (ov) launch_deep_t<VAR, true, 14, true>(ctx, a, st);
      else launch_deep_t<VAR, true, 16, true>(ctx, a, st);
    } else if (ov) {
      if (a.L <= 32) launch_deep_t<VAR, true, cvg::kDeepWarpsOverlap>(ctx, a, st);
      else launch_deep_t<VAR, false, cvg::kDeepWarpsOverlap>(ctx, a, st);
    } else {
      if (a.L <= 32) launch_deep_t<VAR, true, cvg::kDeepWarps>(ctx, a, st);
      else launch_deep_t<VAR, false, cvg::kDeepWarps>(ctx, a, st);
    }
  }
  if (pe) CVG_CUDA(cudaEventRecord(pe[2], st));
  if (ov) {
    CVG_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    st = ctx->side;
  }
  if (ov && ctx->shallow_persist > 0) {
    auto k = sh && dp ? cvg::shallow_persistent_kernel<VAR, true, true>
                      : sh ? cvg::shallow_persistent_kernel<VAR, true, false>
                           : cvg::shallow_persistent_kernel<VAR, false, true>;
    CVG_CUDA(cudaMemsetAsync(ctx->cursor.p + 40, 0, sizeof(unsigned long long), st));
    k<<<ctx->num_sms * ctx->shallow_persist, cvg::kShallowThreads, 0, st>>>(b, ctx->cursor.p + 40);
  } else if (ctx->shallow_mode == 2 && (b.ld_in % 2) == 0) {
    const size_t smem = (size_t)cvg::kExpTableSize * sizeof(double2) +
                        (size_t)2 * 2 * b.L * cvg::kShTile * sizeof(double);
    auto k = sh && dp ? cvg::shallow_tma_kernel<VAR, true, true>
                      : sh ? cvg::shallow_tma_kernel<VAR, true, false> : cvg::shallow_tma_kernel<VAR, false, true>;
    CVG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<ctx->num_sms, cvg::kShTile, smem, st>>>(b);
  } else {
    const unsigned blocks = (unsigned)((b.n + cvg::kShallowThreads - 1) / cvg::kShallowThreads);
    CVG_CUDA(cudaFuncSetAttribute(cvg::shallow_kernel<VAR, true, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    if (ctx->shallow_minb == 10 && sh && dp)
      cvg::shallow_kernel<VAR, true, true, 10><<<blocks, cvg::kShallowThreads, 0, st>>>(b);
    else if (sh && dp) cvg::shallow_kernel<VAR, true, true><<<blocks, cvg::kShallowThreads, 0, st>>>(b);
    else if (sh) cvg::shallow_kernel<VAR, true, false><<<blocks, cvg::kShallowThreads, 0, st>>>(b);
    else if (dp) cvg::shallow_kernel<VAR, false, true><<<blocks, cvg::kShallowThreads, 0, st>>>(b);
  }
  CVG_CUDA(cudaGetLastError());
  if (ov) {
    if (pe) CVG_CUDA(cudaEventRecord(pe[3], st));
    CVG_CUDA(cudaEventRecord(ctx->ev_join, st));
    CVG_CUDA(cudaStreamWaitEvent(ctx->main_for_join, ctx->ev_join, 0));
  }
}

// Enqueues the hot path on `st`: memsets of the per-call cursors and
// failure words, the trigger + compaction kernel (deep requested), then the
// deep kernel and the shallow(+zero-fill) kernel -- concurrently on a forked
// side stream in overlap mode (the default).  Pointers are device pointers.
void enqueue(cvg_context* ctx, const cvg_columns* in, const cvg_options* o, int mask,
             const cvg_outputs* deep, const cvg_outputs* sh, cudaStream_t st) {
  const long long n = in->n_columns;
  const int L = in->n_levels;
  CVG_CUDA(cudaMemsetAsync(ctx->counters.p, 0, 4 * sizeof(int), st));
  CVG_CUDA(cudaMemsetAsync(ctx->cursor.p, 0, sizeof(unsigned long long), st));
  CVG_CUDA(cudaMemsetAsync(ctx->err.p, 0xff, 2 * sizeof(unsigned long long), st));
  if (n == 0) return;
  const bool do_deep = (mask & CVG_DEEP) != 0, do_sh = (mask & CVG_SHALLOW) != 0;
  cudaEvent_t* pe = nullptr;
  if (ctx->prof_on && ctx->prof_n < ctx->prof_cap) pe = &ctx->prof_ev[4 * ctx->prof_n++];
  if (pe) CVG_CUDA(cudaEventRecord(pe[0], st));
  cvg::DeepArgs a{};
  if (do_deep) {
    ctx->idx.ensure((size_t)n);
    const unsigned tb = (unsigned)((n + cvg::kTrigTile - 1) / cvg::kTrigTile);
    cvg::trigger_compact_kernel<<<tb, cvg::kTrigThreads, 0, st>>>(
        in->s, n, o->activity_threshold, ctx->idx.p, ctx->counters.p, ctx->err.p);
    CVG_CUDA(cudaGetLastError());
    a.s = in->s; a.T = in->T; a.q = in->q; a.ld_in = in->ld;
    a.tend_T = deep->tend_T; a.tend_q = deep->tend_q; a.precip = deep->precip;
    a.work = deep->work_units; a.exited = deep->exited_early; a.ld_out = deep->ld;
    a.idx = ctx->idx.p; a.count = ctx->counters.p;
    a.cursor = ctx->cursor.p;
    a.err = ctx->err.p; a.first_col = in->first_col;
    a.thr = o->activity_threshold; a.tol = o->newton_tol; a.maxit = o->newton_max_iter;
    a.L = L;
    a.batch = std::max(1, std::min(cvg::kDeepBatch, (int)(98304 / ((size_t)cvg::kDeepWarps * L * sizeof(double)))));
    a.fast_div_ok = o->newton_tol >= 0x1.0p-500;
  }
  a.exp_tab = ctx->exp_tab.p;
  if (pe) CVG_CUDA(cudaEventRecord(pe[1], st));
  cvg::ShallowArgs b{};
  b.s = in->s; b.T = in->T; b.q = in->q; b.ld_in = in->ld; b.n = n;
  if (do_sh) {
    b.tend_T = sh->tend_T; b.tend_q = sh->tend_q; b.precip = sh->precip;
    b.work = sh->work_units; b.exited = sh->exited_early; b.ld_out = sh->ld;
  }
  if (do_deep) {
    b.d_tend_T = deep->tend_T; b.d_tend_q = deep->tend_q; b.d_precip = deep->precip;
    b.d_work = deep->work_units; b.d_exited = deep->exited_early; b.d_ld_out = deep->ld;
  }
  b.err = ctx->err.p + 1; b.exp_tab = ctx->exp_tab.p; b.first_col = in->first_col;
  b.thr = o->activity_threshold; b.L = L;
  if (ctx->trace_path) {
    ctx->trace_d.ensure(3 * 4096);
    ctx->trace_s.ensure(3 * (size_t)((n + 127) / 128 + 1));
    CVG_CUDA(cudaMemsetAsync(ctx->trace_d.p, 0, 3 * 4096 * 8, st));
    CVG_CUDA(cudaMemsetAsync(ctx->trace_s.p, 0, 3 * ((n + 127) / 128 + 1) * 8, st));
    a.trace = ctx->trace_d.p;
    b.trace = ctx->trace_s.p;
  }
  ctx->main_for_join = st;
  switch (o->variant) {
    case 1: launch_split<cvg::kVarReduced>(ctx, a, b, do_sh, do_deep, pe, st); break;
    case 2: launch_split<cvg::kVarApprox>(ctx, a, b, do_sh, do_deep, pe, st); break;
    default: launch_split<cvg::kVarExact>(ctx, a, b, do_sh, do_deep, pe, st); break;
  }
  if (pe && !(ctx->overlap && do_deep)) CVG_CUDA(cudaEventRecord(pe[3], st));
}

// Reads back the latched failure words (stream already synchronised).
cvg_status collect(cvg_context* ctx, int mask, int maxit, long long n, cvg_stats* stats) {
  CVG_CUDA(cudaMemcpy(ctx->h_err, ctx->err.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  CVG_CUDA(cudaMemcpy(ctx->h_count, ctx->counters.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (stats) {
    stats->n_columns = n;
    stats->n_triggered = (mask & CVG_DEEP) ? *ctx->h_count : 0;
    stats->failing_column = -1;
    stats->failure_kind = 0;
    stats->failing_kernel = 0;
  }
  const unsigned long long none = ~0ULL;
  for (int w = 0; w < 2; ++w) {
    const int kernel = w == 0 ? CVG_DEEP : CVG_SHALLOW;
    if (!(mask & kernel)) continue;
    const unsigned long long key = ctx->h_err[w];
    if (key == none) continue;
    const long long col = (long long)(key >> 16);
    const int kind = (int)(key & 7);
    std::string buf;
    const char* what = kind_message(kind, kernel, maxit, &buf);
    if (stats) {
      stats->failing_column = col;
      stats->failure_kind = kind;
      stats->failing_kernel = kernel;
    }
    return fail(CVG_ERR_NUMERIC, std::string(what) + ": column " + std::to_string(col));
  }
  return CVG_OK;
}

template <typename Fn>
cvg_status guarded(Fn&& body) {
  try {
    g_last_error.clear();
    return body();
  } catch (const CudaError& e) {
    cudaGetLastError();
    return fail(CVG_ERR_DEVICE, std::string("CUDA error: ") + cudaGetErrorString(e.code) + " in " + e.what);
  } catch (const std::exception& e) {
    return fail(CVG_ERR_INVALID, e.what());
  } catch (...) {
    return fail(CVG_ERR_INVALID, "unknown error");
  }
}

void copy_rows_h2d(double* dst, const double* src, long long n, int L, long long ld, cudaStream_t st) {
  if (ld == n) {
    CVG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n * L, cudaMemcpyHostToDevice, st));
  } else {
    CVG_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * n, src, sizeof(double) * ld, sizeof(double) * n, L,
                               cudaMemcpyHostToDevice, st));
  }
}

void copy_rows_d2h(double* dst, long long ld, const double* src, long long n, int L, cudaStream_t st) {
  if (ld == n) {
    CVG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n * L, cudaMemcpyDeviceToHost, st));
  } else {
    CVG_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * ld, src, sizeof(double) * n, sizeof(double) * n, L,
                               cudaMemcpyDeviceToHost, st));
  }
}

}  // namespace

extern "C" {

const char* cvg_version(void) { return "0.1.0"; }

const char* cvg_last_error(void) { return g_last_error.c_str(); }

void cvg_default_options(cvg_options* o) {
  if (!o) return;
  o->variant = CVG_EXACT;
  o->activity_threshold = 0.5;
  o->newton_tol = 1e-12;
  o->newton_max_iter = 100;
}

cvg_status cvg_context_create(int device, cvg_context** out) {
  if (!out) return fail(CVG_ERR_INVALID, "cvg_context_create: null out");
  *out = nullptr;
  return guarded([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      return fail(CVG_ERR_DEVICE, "cvg_context_create: no CUDA device (this library has no CPU path)");
    }
    if (device < 0 || device >= ndev) return fail(CVG_ERR_INVALID, "cvg_context_create: bad device index");
    cudaDeviceProp prop{};
    CVG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
      return fail(CVG_ERR_DEVICE, std::string("cvg_context_create: device is sm_") + std::to_string(prop.major) +
                                      std::to_string(prop.minor) + ", this build targets sm_100a");
    }
    CVG_CUDA(cudaSetDevice(device));
    auto* ctx = new cvg_context();
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    try {
      CVG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      CVG_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
      CVG_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
      CVG_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
      CVG_CUDA(cudaEventCreate(&ctx->ev0));
      CVG_CUDA(cudaEventCreate(&ctx->ev1));
      CVG_CUDA(cudaEventCreate(&ctx->ev_h0));
      CVG_CUDA(cudaEventCreate(&ctx->ev_h1));
      CVG_CUDA(cudaEventCreate(&ctx->ev_d0));
      const std::vector<double2> tab = exp_table_host();
      ctx->exp_tab.ensure(tab.size());
      CVG_CUDA(cudaMemcpy(ctx->exp_tab.p, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice));
      ctx->counters.ensure(4);
      ctx->cursor.ensure(80);  // [0] deep cursor, [40] tile cursor, others dummies
      CVG_CUDA(cudaMemset(ctx->cursor.p, 0, 80 * sizeof(unsigned long long)));
      ctx->err.ensure(4);
      CVG_CUDA(cudaMallocHost(&ctx->h_err, 4 * sizeof(unsigned long long)));
      CVG_CUDA(cudaMallocHost(&ctx->h_count, 4 * sizeof(int)));
      CVG_CUDA(cudaMemset(ctx->counters.p, 0, 4 * sizeof(int)));
      CVG_CUDA(cudaMemset(ctx->err.p, 0xff, 4 * sizeof(unsigned long long)));
      // probe that the sm_100a image loads on this device
      if (const char* e = getenv("CVG_OVERLAP")) ctx->overlap = atoi(e) != 0;
      if (const char* e = getenv("CVG_SHALLOW_MINB")) ctx->shallow_minb = atoi(e);
      ctx->trace_path = getenv("CVG_TRACE");
      if (const char* e = getenv("CVG_SHALLOW_MODE")) ctx->shallow_mode = atoi(e);
      if (const char* e = getenv("CVG_PAIRS")) ctx->pairs = atoi(e) != 0;
      if (const char* e = getenv("CVG_SHALLOW_PERSIST")) ctx->shallow_persist = atoi(e);
    } catch (...) {
      cvg_context_free(ctx);
      throw;
    }
    *out = ctx;
    return CVG_OK;
  });
}

void cvg_context_free(cvg_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto* b : {&ctx->exp_tab}) b->release();
  ctx->idx.release();
  ctx->counters.release();
  ctx->cursor.release();
  ctx->err.release();
  for (auto* b : {&ctx->in_s, &ctx->in_T, &ctx->in_q, &ctx->dT, &ctx->dq, &ctx->dp, &ctx->sT, &ctx->sq, &ctx->sp,
                  &ctx->aux0, &ctx->aux1})
    b->release();
  ctx->dw.release();
  ctx->sw.release();
  ctx->dx.release();
  ctx->sx.release();
  ctx->auxi.release();
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->h_count) cudaFreeHost(ctx->h_count);
  for (cudaEvent_t e : {ctx->ev0, ctx->ev1, ctx->ev_h0, ctx->ev_h1, ctx->ev_d0})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->prof_ev) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  delete ctx;
}

cvg_status cvg_convect_async(cvg_context* ctx, const cvg_columns* in, const cvg_options* opts, int mask,
                             const cvg_outputs* deep, const cvg_outputs* sh, void* stream) {
  if (!ctx || !in || !opts) return fail(CVG_ERR_INVALID, "cvg_convect_async: null argument");
  std::string why;
  if (!valid_columns(in, &why) || !valid_options(opts, &why)) return fail(CVG_ERR_INVALID, "cvg_convect_async: " + why);
  if (mask < 1 || mask > 3) return fail(CVG_ERR_INVALID, "cvg_convect_async: kernel_mask must be 1, 2 or 3");
  if ((mask & CVG_DEEP) && (!deep || !valid_outputs(deep, in->n_columns, &why)))
    return fail(CVG_ERR_INVALID, "cvg_convect_async: deep outputs: " + (deep ? why : std::string("null")));
  if ((mask & CVG_SHALLOW) && (!sh || !valid_outputs(sh, in->n_columns, &why)))
    return fail(CVG_ERR_INVALID, "cvg_convect_async: shallow outputs: " + (sh ? why : std::string("null")));
  if (!in->on_device || ((mask & CVG_DEEP) && !deep->on_device) || ((mask & CVG_SHALLOW) && !sh->on_device))
    return fail(CVG_ERR_INVALID, "cvg_convect_async: all buffers must be device memory");
  return guarded([&] {
    CVG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    enqueue(ctx, in, opts, mask, deep, sh, st);
    ctx->last_mask = mask;
    ctx->last_maxit = opts->newton_max_iter;
    ctx->last_n = in->n_columns;
    ctx->pending = true;
    return CVG_OK;
  });
}

cvg_status cvg_convect_check(cvg_context* ctx, void* stream, cvg_stats* stats) {
  if (!ctx) return fail(CVG_ERR_INVALID, "cvg_convect_check: null context");
  return guarded([&] {
    CVG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    CVG_CUDA(cudaStreamSynchronize(st));
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (!ctx->pending) return CVG_OK;
    if (ctx->trace_path && ctx->trace_d.p) {
      const size_t nd = 3 * 4096, ns = 3 * (size_t)((ctx->last_n + 127) / 128 + 1);
      std::vector<unsigned long long> hd(nd), hs(ns);
      CVG_CUDA(cudaMemcpy(hd.data(), ctx->trace_d.p, nd * 8, cudaMemcpyDeviceToHost));
      CVG_CUDA(cudaMemcpy(hs.data(), ctx->trace_s.p, ns * 8, cudaMemcpyDeviceToHost));
      if (FILE* f = fopen(ctx->trace_path, "w")) {
        for (size_t i = 0; i + 2 < nd; i += 3)
          if (hd[i + 1]) fprintf(f, "deep %llu %llu %llu\n", hd[i], hd[i + 1], hd[i + 2]);
        for (size_t i = 0; i + 2 < ns; i += 3)
          if (hs[i + 1]) fprintf(f, "shallow %llu %llu %llu\n", hs[i], hs[i + 1], hs[i + 2]);
        fclose(f);
      }
    }
    return collect(ctx, ctx->last_mask, ctx->last_maxit, ctx->last_n, stats);
  });
}

cvg_status cvg_convect(cvg_context* ctx, const cvg_columns* in, const cvg_options* opts, int mask,
                       const cvg_outputs* deep, const cvg_outputs* sh, cvg_stats* stats) {
  if (!ctx || !in || !opts) return fail(CVG_ERR_INVALID, "cvg_convect: null argument");
  std::string why;
  if (!valid_columns(in, &why) || !valid_options(opts, &why)) return fail(CVG_ERR_INVALID, "cvg_convect: " + why);
  if (mask < 1 || mask > 3) return fail(CVG_ERR_INVALID, "cvg_convect: kernel_mask must be 1, 2 or 3");
  if ((mask & CVG_DEEP) && (!deep || !valid_outputs(deep, in->n_columns, &why)))
    return fail(CVG_ERR_INVALID, "cvg_convect: deep outputs: " + (deep ? why : std::string("null")));
  if ((mask & CVG_SHALLOW) && (!sh || !valid_outputs(sh, in->n_columns, &why)))
    return fail(CVG_ERR_INVALID, "cvg_convect: shallow outputs: " + (sh ? why : std::string("null")));
  return guarded([&] {
    CVG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const long long n = in->n_columns;
    const int L = in->n_levels;
    const size_t nL = (size_t)n * L;
    long long h2d = 0, d2h = 0;
    // ---- stage inputs
    cvg_columns din = *in;
    CVG_CUDA(cudaEventRecord(ctx->ev_h0, st));
    if (!in->on_device && n > 0) {
      ctx->in_s.ensure(n);
      ctx->in_T.ensure(nL);
      ctx->in_q.ensure(nL);
      CVG_CUDA(cudaMemcpyAsync(ctx->in_s.p, in->s, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      copy_rows_h2d(ctx->in_T.p, in->T, n, L, in->ld, st);
      copy_rows_h2d(ctx->in_q.p, in->q, n, L, in->ld, st);
      h2d = (long long)(sizeof(double) * (n + 2 * nL));
      din.s = ctx->in_s.p;
      din.T = ctx->in_T.p;
      din.q = ctx->in_q.p;
      din.ld = n;
      din.on_device = 1;
    }
    auto stage_out = [&](const cvg_outputs* o, DevBuf<double>& T, DevBuf<double>& q, DevBuf<double>& p,
                         DevBuf<long long>& w, DevBuf<uint8_t>& x) {
      cvg_outputs d = *o;
      if (!o->on_device && n > 0) {
        T.ensure(nL); q.ensure(nL); p.ensure(n); w.ensure(n); x.ensure(n);
        d.tend_T = T.p; d.tend_q = q.p; d.precip = p.p; d.work_units = w.p; d.exited_early = x.p;
        d.ld = n; d.on_device = 1;
      }
      return d;
    };
    cvg_outputs ddeep{}, dsh{};
    if (mask & CVG_DEEP) ddeep = stage_out(deep, ctx->dT, ctx->dq, ctx->dp, ctx->dw, ctx->dx);
    if (mask & CVG_SHALLOW) dsh = stage_out(sh, ctx->sT, ctx->sq, ctx->sp, ctx->sw, ctx->sx);
    CVG_CUDA(cudaEventRecord(ctx->ev0, st));
    enqueue(ctx, &din, opts, mask, &ddeep, &dsh, st);
    CVG_CUDA(cudaEventRecord(ctx->ev1, st));
    // ---- outputs back
    auto unstage = [&](const cvg_outputs* o, const cvg_outputs& d) {
      if (o->on_device || n == 0) return;
      copy_rows_d2h(o->tend_T, o->ld, d.tend_T, n, L, st);
      copy_rows_d2h(o->tend_q, o->ld, d.tend_q, n, L, st);
      CVG_CUDA(cudaMemcpyAsync(o->precip, d.precip, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
      CVG_CUDA(cudaMemcpyAsync(o->work_units, d.work_units, sizeof(long long) * n, cudaMemcpyDeviceToHost, st));
      CVG_CUDA(cudaMemcpyAsync(o->exited_early, d.exited_early, n, cudaMemcpyDeviceToHost, st));
      d2h += (long long)(sizeof(double) * (2 * nL + n) + sizeof(long long) * n + n);
    };
    if (mask & CVG_DEEP) unstage(deep, ddeep);
    if (mask & CVG_SHALLOW) unstage(sh, dsh);
    CVG_CUDA(cudaEventRecord(ctx->ev_h1, st));
    CVG_CUDA(cudaStreamSynchronize(st));
    cvg_status rc = collect(ctx, mask, opts->newton_max_iter, n, stats);
    if (stats) {
      float ms = 0.f, all = 0.f;
      CVG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
      CVG_CUDA(cudaEventElapsedTime(&all, ctx->ev_h0, ctx->ev_h1));
      stats->device_ms = ms;
      float h = 0.f;
      CVG_CUDA(cudaEventElapsedTime(&h, ctx->ev_h0, ctx->ev0));
      stats->h2d_ms = h;
      stats->d2h_ms = std::max(0.f, all - ms - h);
      stats->h2d_bytes = h2d;
      stats->d2h_bytes = d2h;
    }
    ctx->pending = false;
    return rc;
  });
}

cvg_status cvg_deep_convection(cvg_context* ctx, const cvg_columns* in, const cvg_options* opts,
                               const cvg_outputs* out, cvg_stats* stats) {
  return cvg_convect(ctx, in, opts, CVG_DEEP, out, nullptr, stats);
}

cvg_status cvg_shallow_convection(cvg_context* ctx, const cvg_columns* in, const cvg_options* opts,
                                  const cvg_outputs* out, cvg_stats* stats) {
  return cvg_convect(ctx, in, opts, CVG_SHALLOW, nullptr, out, stats);
}

cvg_status cvg_ientropy_solve(cvg_context* ctx, long long n, const double* y, const double* guess,
                              const cvg_options* opts, double* root, int* iterations) {
  if (!ctx || !opts || (n > 0 && (!y || !guess || !root || !iterations)))
    return fail(CVG_ERR_INVALID, "cvg_ientropy_solve: null argument");
  std::string why;
  if (n < 0 || !valid_options(opts, &why)) return fail(CVG_ERR_INVALID, "cvg_ientropy_solve: bad argument " + why);
  return guarded([&] {
    if (n == 0) return CVG_OK;
    CVG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    ctx->aux0.ensure(n);
    ctx->aux1.ensure(2 * n);
    ctx->auxi.ensure(n);
    double* dy = ctx->aux1.p;
    double* dg = ctx->aux1.p + n;
    CVG_CUDA(cudaMemcpyAsync(dy, y, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CVG_CUDA(cudaMemcpyAsync(dg, guess, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CVG_CUDA(cudaMemsetAsync(ctx->err.p + 2, 0xff, sizeof(unsigned long long), st));
    const unsigned blocks = (unsigned)((n + 255) / 256);
    switch (opts->variant) {
      case 2: cvg::ientropy_kernel<cvg::kVarApprox><<<blocks, 256, 0, st>>>(dy, dg, n, opts->newton_tol,
                  opts->newton_max_iter, ctx->aux0.p, ctx->auxi.p, ctx->err.p + 2, ctx->exp_tab.p); break;
      default: cvg::ientropy_kernel<cvg::kVarExact><<<blocks, 256, 0, st>>>(dy, dg, n, opts->newton_tol,
                  opts->newton_max_iter, ctx->aux0.p, ctx->auxi.p, ctx->err.p + 2, ctx->exp_tab.p); break;
    }
    CVG_CUDA(cudaGetLastError());
    CVG_CUDA(cudaMemcpyAsync(root, ctx->aux0.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaMemcpyAsync(iterations, ctx->auxi.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaMemcpyAsync(ctx->h_err + 2, ctx->err.p + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaStreamSynchronize(st));
    const unsigned long long key = ctx->h_err[2];
    if (key != ~0ULL) {
      std::string buf;
      const char* what = kind_message((int)(key & 7), CVG_DEEP, opts->newton_max_iter, &buf);
      return fail(CVG_ERR_NUMERIC, std::string(what) + ": index " + std::to_string((long long)(key >> 16)));
    }
    return CVG_OK;
  });
}

cvg_status cvg_approx_exp(cvg_context* ctx, long long n, const double* x, double* out) {
  if (!ctx || (n > 0 && (!x || !out))) return fail(CVG_ERR_INVALID, "cvg_approx_exp: null argument");
  if (n < 0) return fail(CVG_ERR_INVALID, "cvg_approx_exp: n < 0");
  return guarded([&] {
    if (n == 0) return CVG_OK;
    CVG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    ctx->aux0.ensure(n);
    ctx->aux1.ensure(n);
    CVG_CUDA(cudaMemcpyAsync(ctx->aux1.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    cvg::approx_exp_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ctx->aux1.p, ctx->aux0.p, n);
    CVG_CUDA(cudaGetLastError());
    CVG_CUDA(cudaMemcpyAsync(out, ctx->aux0.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaStreamSynchronize(st));
    return CVG_OK;
  });
}

cvg_status cvg_profile_begin(cvg_context* ctx, int max_steps) {
  if (!ctx || max_steps < 1) return fail(CVG_ERR_INVALID, "cvg_profile_begin: null context or max_steps < 1");
  return guarded([&] {
    CVG_CUDA(cudaSetDevice(ctx->device));
    const size_t need = 4 * (size_t)max_steps;
    while (ctx->prof_ev.size() < need) {
      cudaEvent_t e;
      CVG_CUDA(cudaEventCreate(&e));
      ctx->prof_ev.push_back(e);
    }
    ctx->prof_cap = max_steps;
    ctx->prof_n = 0;
    ctx->prof_on = true;
    return CVG_OK;
  });
}

cvg_status cvg_profile_end(cvg_context* ctx, int* n_steps, double* kernel_ms, int capacity) {
  if (!ctx || !n_steps) return fail(CVG_ERR_INVALID, "cvg_profile_end: null argument");
  return guarded([&] {
    CVG_CUDA(cudaSetDevice(ctx->device));
    ctx->prof_on = false;
    const int n = std::min(ctx->prof_n, capacity);
    for (int i = 0; i < n; ++i) {
      cudaEvent_t* pe = &ctx->prof_ev[4 * i];
      CVG_CUDA(cudaEventSynchronize(pe[3]));
      float t0 = 0.f, t1 = 0.f, t2 = 0.f;
      CVG_CUDA(cudaEventElapsedTime(&t0, pe[0], pe[1]));
      CVG_CUDA(cudaEventElapsedTime(&t1, pe[1], pe[2]));
      CVG_CUDA(cudaEventElapsedTime(&t2, pe[2], pe[3]));
      if (kernel_ms) {
        kernel_ms[3 * i + 0] = t0;
        kernel_ms[3 * i + 1] = t1;
        kernel_ms[3 * i + 2] = t2;
      }
    }
    *n_steps = n;
    ctx->prof_n = 0;
    return CVG_OK;
  });
}

cvg_status cvg_fp64_peak(cvg_context* ctx, int reps, double* tflops) {
  if (!ctx || !tflops) return fail(CVG_ERR_INVALID, "cvg_fp64_peak: null argument");
  return guarded([&] {
    CVG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int blocks = ctx->num_sms * 8, threads = 256, iters = 4096;
    ctx->aux0.ensure((size_t)blocks * threads);
    for (int w = 0; w < 2; ++w)
      cvg::dfma_probe_kernel<<<blocks, threads, 0, st>>>(ctx->aux0.p, iters, 0.999999, 1e-7);
    CVG_CUDA(cudaGetLastError());
    float best = 1e30f;
    for (int r = 0; r < std::max(reps, 1); ++r) {
      CVG_CUDA(cudaEventRecord(ctx->ev0, st));
      cvg::dfma_probe_kernel<<<blocks, threads, 0, st>>>(ctx->aux0.p, iters, 0.999999, 1e-7);
      CVG_CUDA(cudaEventRecord(ctx->ev1, st));
      CVG_CUDA(cudaEventSynchronize(ctx->ev1));
      float ms = 0.f;
      CVG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
      best = std::min(best, ms);
    }
    const double flops = 2.0 * 8.0 * (double)blocks * threads * iters;
    *tflops = flops / (best * 1e-3) / 1e12;
    return CVG_OK;
  });
}

cvg_status cvg_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(CVG_ERR_INVALID, "cvg_host_alloc: null out");
  return guarded([&] {
    CVG_CUDA(cudaMallocHost(out, std::max<size_t>(bytes, 1)));
    return CVG_OK;
  });
}

void cvg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

cvg_status cvg_plan_partition(long long n, const double* s, double thr, int n_parts, double deep_weight,
                              double shallow_weight, long long* bounds) {
  if (!bounds || (n > 0 && !s && deep_weight > 0.0)) return fail(CVG_ERR_INVALID, "cvg_plan_partition: null argument");
  if (n < 0 || n_parts < 1) return fail(CVG_ERR_INVALID, "cvg_plan_partition: n < 0 or n_parts < 1");
  if (!(shallow_weight >= 0.0)) return fail(CVG_ERR_INVALID, "cvg_plan_partition: shallow_weight < 0");
  g_last_error.clear();
  bounds[0] = 0;
  if (deep_weight <= 0.0 || n == 0) {
    // naive equal-columns split, remainder on the last parts (sched.cpp:66-75)
    const long long qn = n / n_parts, r = n % n_parts;
    long long next = 0;
    for (int p = 0; p < n_parts; ++p) {
      next += qn + (p >= n_parts - r ? 1 : 0);
      bounds[p + 1] = next;
    }
    return CVG_OK;
  }
  // cost-balanced contiguous split: boundary p at the first column where the
  // prefix cost reaches p/G of the total
  double total = 0.0;
  for (long long c = 0; c < n; ++c) total += (s[c] > thr ? deep_weight : 0.0) + shallow_weight;
  double run = 0.0;
  int p = 1;
  for (long long c = 0; c < n && p < n_parts; ++c) {
    run += (s[c] > thr ? deep_weight : 0.0) + shallow_weight;
    while (p < n_parts && run >= total * p / n_parts) bounds[p++] = c + 1;
  }
  while (p < n_parts) bounds[p++] = n;
  bounds[n_parts] = n;
  for (int i = 1; i <= n_parts; ++i) bounds[i] = std::max(bounds[i], bounds[i - 1]);
  return CVG_OK;
}

}  // extern "C"

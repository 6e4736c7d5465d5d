// convgpu.cu -- host runtime and C ABI of the B200 convection column path.
//
// Implements include/convgpu.h: per-device contexts owning the exp table and
// a small ring of per-call workspaces (compaction list, cursors, latched
// failure words, a side stream for the concurrent shallow kernel, and the
// staging buffers of host-buffer calls); the launch sequence trigger +
// compaction -> deep plume || shallow (+ deep zero fill); host <-> device
// staging as a chunked pipeline (H2D, compute and D2H of different column
// chunks overlap on the copy engines and the SMs); the reference's error
// taxonomy at the boundary (capi.cpp:51-89); and the multi-device partition
// planner.  No CPU fallback exists: without a usable sm_100 device every
// compute entry point returns CVG_ERR_DEVICE.
#include <cuda.h>   // CUtensorMap types only: cuTensorMapEncodeTiled is fetched through the runtime (no libcuda link)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
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
  // Grows to n elements keeping the old allocation alive in `retired`
  // (a CUDA graph captured earlier may still reference it); true if grown.
  bool grow(size_t n, std::vector<void*>& retired) {
    if (n <= cap) return false;
    if (p) retired.push_back(p);
    p = nullptr;
    cap = 0;
    CVG_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    cap = n;
    return true;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// 2^(j/512) rounded to double for the relaxed Newton loop's exp (colmath.cuh
// exp_fetch1), from x87 extended precision (~1 ulp of the 64-bit
// significand, so the rounding to double is correct except in double-
// rounding ties -- immaterial for a path whose stop decisions are guarded).
std::vector<double> exp_table1_host() {
  std::vector<double> t(cvg::kExpTableSize);
  for (int j = 0; j < cvg::kExpTableSize; ++j)
    t[j] = static_cast<double>(exp2l(static_cast<long double>(j) / cvg::kExpTableSize));
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

// Everything one in-flight call needs on the device.  Slot 0 serves the
// device-resident (async) API; host-buffer calls pipeline column chunks
// through all slots.
struct Workspace {
  cudaStream_t stream = nullptr;  // chunk stream (host-buffer calls)
  cudaStream_t side = nullptr;    // shallow kernel, concurrent with deep
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_copy[4] = {};         // H2D start/end, D2H start/end of the slot's chunk
  bool copy_timed = false;             // events recorded for the slot's current chunk
  DevBuf<long long> groups;            // compacted column groups with a triggered column
  DevBuf<int> counters;                // [0] listed groups, [1] triggered columns, [2] levels queued
                                       // for exact re-derivation, [3] columns rewritten by it
  DevBuf<unsigned long long> redo;     // the redo list (guard band): [cap][kRedoWords]
  DevBuf<unsigned long long> fix;      // exact patches: [2 cap][3]
  DevBuf<unsigned long long> cursor;   // [0] deep work cursor, [16] redo_kernel's finished blocks
  DevBuf<unsigned long long> err;      // [0] deep, [1] shallow failure key
  unsigned long long* h_err = nullptr; // pinned mirror of err[0..1]
  int* h_count = nullptr;              // pinned mirror of counters[0..1]
  // staging for host-buffer calls (chunk-sized)
  DevBuf<double> in_s, in_T, in_q, dT, dq, dp, sT, sq, sp;
  DevBuf<long long> dw, sw;
  DevBuf<uint8_t> dx, sx;

  void create() {
    CVG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CVG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    CVG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CVG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    for (cudaEvent_t& e : ev_copy) CVG_CUDA(cudaEventCreate(&e));
    counters.ensure(4);
    cursor.ensure(40);
    err.ensure(4);
    CVG_CUDA(cudaMemset(counters.p, 0, 4 * sizeof(int)));
    CVG_CUDA(cudaMemset(cursor.p, 0, 40 * sizeof(unsigned long long)));
    CVG_CUDA(cudaMemset(err.p, 0xff, 4 * sizeof(unsigned long long)));
    CVG_CUDA(cudaMallocHost(&h_err, 4 * sizeof(unsigned long long)));
    CVG_CUDA(cudaMallocHost(&h_count, 4 * sizeof(int)));
  }
  void destroy() {
    for (auto* b : {&in_s, &in_T, &in_q, &dT, &dq, &dp, &sT, &sq, &sp}) b->release();
    dw.release(); sw.release(); dx.release(); sx.release();
    groups.release(); counters.release(); cursor.release(); err.release(); redo.release(); fix.release();
    if (h_err) cudaFreeHost(h_err);
    if (h_count) cudaFreeHost(h_count);
    if (ev_fork) cudaEventDestroy(ev_fork);
    for (cudaEvent_t& e : ev_copy)
      if (e) cudaEventDestroy(e), e = nullptr;
    if (ev_join) cudaEventDestroy(ev_join);
    if (stream) cudaStreamDestroy(stream);
    if (side) cudaStreamDestroy(side);
    h_err = nullptr; h_count = nullptr; ev_fork = ev_join = nullptr; stream = side = nullptr;
  }
};

constexpr int kSlots = 4;                    // workspaces (pipeline depth of host-buffer calls)
constexpr long long kChunkCols = 262144;     // columns per host-buffer pipeline chunk (steady state)

}  // namespace

namespace {
// Device state of one leg: T, q [L][n] (ld = n) and the selected kernel's
// outputs.
struct LegBufs {
  DevBuf<double> T, q;
};

struct LoopBufs {
  DevBuf<double> s, oT, oq, op;
  DevBuf<long long> ow;
  DevBuf<uint8_t> ox;
  cvg_outputs outs(long long n) {
    return cvg_outputs{oT.p, oq.p, op.p, ow.p, ox.p, n, 1};
  }
  void ensure(long long n, int L) {
    s.ensure(n); oT.ensure((size_t)n * L); oq.ensure((size_t)n * L); op.ensure(n); ow.ensure(n); ox.ensure(n);
  }
};

}  // namespace

struct cvg_context {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;  // default stream of the async API
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_h0 = nullptr, ev_h1 = nullptr;
  DevBuf<double> exp_tab1;              // relaxed loop's 2^(j/512) table
  const double2* gl_tab = nullptr;       // exp_gl table (cvg::kExpGlTable, device symbol)
  Workspace ws[kSlots];
  DevBuf<double> aux0, aux1;
  DevBuf<int> auxi;
  DevBuf<unsigned long long> aux_err;
  unsigned long long* h_aux_err = nullptr;
  // tuning switches (environment, read at context creation)
  bool overlap = true;     // CVG_OVERLAP: deep || shallow on two streams
  int deep_warps = 0;      // CVG_DEEP_WARPS: 12, 16 or 20 warps per deep block (0: by mode)
  int shallow_minb = 8;    // CVG_SHALLOW_MINB: shallow blocks per SM the register budget targets (8, 12, 16)
  // CVG_SHALLOW_TILE: the overlapped step's shallow kernel as one persistent
  // block per SM of warp-private TMA-staged tiles (shallow_tile_kernel), with
  // the register file it frees given to the deep block (CVG_TILE_NW warps, build-time)
  int shallow_tile = 1;
  int tile_warps = 8;      // CVG_TILE_WARPS: warps (= tiles in flight) of a shallow tile block
  bool tile_tma = true;    // CVG_TILE_TMA: tile rows by TMA tensor tiles (0: 16-byte cp.async)
  int tile_warps_alone = 12;  // CVG_TILE_WARPS_ALONE: ... of a shallow-only call (no deep block beside it)
  int deep_only = -1;      // CVG_DEEP_ONLY: schedule of deep-only calls (launch_kernels; -1 by size)
  bool pdl = true;         // CVG_PDL: the split-column deep kernel as a programmatic dependent launch behind the trigger kernel
  bool strict = false;     // CVG_STRICT: reference rounding in every Newton update (all variants)
  // CVG_CARVEOUT: shared-memory carveout (% of the 228 KB maximum) preferred
  // by the deep and the shallow kernel.  One value for both: an SM runs the
  // two concurrently only in a configuration that suits both, and 72 % (164
  // KB shared: the deep block's ~127 KB + four 8 KB shallow blocks; 92 KB
  // L1 left for the shallow kernel's row re-reads) measured 0.51 ms per f02
  // step against 0.55 ms at 100 % (deep) / no preference (shallow), and
  // without the occasional serialised schedule (0.70 ms) of mixed settings.
  int carveout = 72;
  bool far32 = true;       // CVG_FAR32: FP32 far phase of the relaxed Newton solve
  // CVG_GUARD: relative half-width g of the guard band [tol (1-g), tol (1+g)]
  // around newton_tol inside which a relaxed solve's stop decision is
  // re-derived on the exact path (colmath.cuh); 0 disables the re-runs
  // (then work_units may flip where the reference's residual is within
  // rounding noise of tol)
  double guard = 1.0 / 128;
  bool redo_launch = true;  // CVG_REDO=0: skip the re-derivation kernel (timing experiments only)
  int redo_inline = -1;     // CVG_REDO_INLINE: re-derive flagged solves inside the deep kernel (1), with redo_kernel (0), by size (-1)
  long long chunk_cols = kChunkCols;  // CVG_CHUNK_COLS: host-call pipeline chunk
  int slots = 3;                      // CVG_SLOTS: workspaces used by host-buffer calls (1..kSlots)
  const char* trace_path = nullptr;   // CVG_TRACE: per-block (kernel, smid, start, end)
  DevBuf<unsigned long long> trace_d, trace_s;
  // per-kernel profiling (cvg_profile_begin/end)
  bool prof_on = false;
  int prof_cap = 0, prof_n = 0;
  std::vector<cudaEvent_t> prof_ev;  // 4 per call: start, after trigger, after deep, after shallow
  // last async call
  int last_mask = 0;
  int last_maxit = 100;
  long long last_n = 0;
  bool pending = false;
  // CUDA graphs of device-resident calls (CVG_GRAPH=0: plain launches),
  // keyed by the call's argument bytes and the workspace list buffer
  struct GraphEntry {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<GraphEntry> graphs;
  bool use_graphs = true;
  int deep_lpc = -1;          // CVG_DEEP_LPC: lanes per column for calls under kTpcMinColumns (-1 by size, 0 off, 2, 4)
  int deep_tpc = 2;           // CVG_DEEP_TPC: thread-per-column deep kernel: 0 never, 1 always, 2 for large calls
  int deep_alone = 1;         // CVG_DEEP_ALONE: deep-only launches as 2 x 16 warps x 64 registers (1) or 2 x 10 x 96 (0)
  // cvg_timestep state, kept across calls (the reference's persistent
  // buffers, hetero.hpp:44)
  LoopBufs loop;
  LegBufs leg;
  DevBuf<unsigned long long> loop_err;
  DevBuf<unsigned> loop_flag;
  bool reset_kernel = true;   // CVG_RESET_KERNEL: one reset launch instead of three memsets
  std::vector<void*> retired;  // grown-out workspace buffers (graphs may reference them)
  std::string last_deep_kernel;  // the deep kernel the last call launched (cvg_last_deep_kernel)
  std::string last_shallow_kernel;  // ... and the shallow kernel (cvg_last_shallow_kernel)
};

#ifndef CVG_TILE_NW
#define CVG_TILE_NW 21
#endif
#ifndef CVG_DEEPONLY_NW
#define CVG_DEEPONLY_NW 28
#endif
#ifndef CVG_TILE_REGS
#define CVG_TILE_REGS 64
#endif

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
  if (o->flags & ~(CVG_FLAG_STRICT | CVG_FLAG_NO_FAR32)) { *why = "unknown flags"; return false; }
  return true;
}

// Hot-path window of the deep Newton solve (colmath.cuh in_far_window): the
// high-word bound lim of the targets y in [0.25, 16) for which the FP32 far
// phase and the relaxed update are both admissible -- relaxed_ok(y, tol)
// holds iff the exponent of y is <= that of tol + 40 (y >= 1) or tol >=
// 2^-40 (y < 1), and the far phase needs tol <= 1e-9 (so that at least three
// FP64 steps follow the switch and contract the FP32 iterate's error below
// rounding noise; tests/test_parity_gpu.py test_hot_path_window_edges saw
// 1e-12-sized tendency differences at tol 1e-6).  Empty window (lim =
// hi(0.25)) when the far phase is off.
static int far_window_limit(double tol, bool enabled) {
  if (!enabled || !(tol <= 1e-9) || !(tol >= 0x1.0p-40)) return cvg::kFarWindowLo;
  unsigned long long bits;
  memcpy(&bits, &tol, sizeof bits);
  const int tol_exp = (int)(bits >> 32) & 0x7ff00000;
  return std::min(cvg::kFarWindowHi, tol_exp + (41 << 20));
}

static bool aligned32(const void* p) { return ((uintptr_t)p & 31) == 0; }

// Shared memory of one deep block: both exp tables and the per-warp scratch.
template <int VAR, bool NARROW, int NW>
void launch_deep_t(cvg_context* ctx, const cvg::DeepArgs& a, cudaStream_t st) {
  const int threads = NW * 32;
  const size_t smem = cvg::deep_table_bytes() + (size_t)NW * cvg::deep_warp_doubles(NARROW, a.L) * sizeof(double);
  auto kern = cvg::deep_kernel<VAR, NARROW, NW>;
  CVG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CVG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, ctx->carveout));
  kern<<<ctx->num_sms, threads, smem, st>>>(a);
  CVG_CUDA(cudaGetLastError());
}

// TMA descriptors of the tiled shallow kernel: T and q as 2-D tensors
// [L][n] of doubles (row pitch ld), box [L][32].  The driver's encoder is
// fetched through the runtime; false when it is unavailable or the layout
// does not qualify (the kernel then stages its tiles with cp.async).
bool encode_tile_maps(const cvg::ShallowArgs& b, cvg::TileMaps* out) {
  typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static encode_fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return (encode_fn)p;
  }();
  static_assert(sizeof(CUtensorMap) == sizeof(out->T), "tensor map size");
  if (!fn || !b.bulk_ok || b.L > 256 || b.n < 1) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)b.n, (cuuint64_t)b.L};
  const cuuint64_t strides[1] = {(cuuint64_t)b.ld_in * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)cvg::kTileCols, (cuuint32_t)b.L};
  const cuuint32_t estr[2] = {1, 1};
  for (int i = 0; i < 2; ++i) {
    void* base = const_cast<double*>(i == 0 ? b.T : b.q);
    CUtensorMap* m = reinterpret_cast<CUtensorMap*>(i == 0 ? out->T : out->q);
    if (fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

// Feedback-loop mode of a call (cvg_timestep): the kernels write the
// advanced state in place instead of tendency rows (DeepArgs::adv_T).
struct Fused {
  double* T;
  double* q;
  unsigned* bad;
};

// deep kernel on `st`, then the shallow(+zero-fill) kernel: concurrently on
// the workspace's side stream in overlap mode (the FP64-bound and the
// HBM-bound kernel share the SMs), else after it on `st`.
template <int VAR>
void launch_kernels(cvg_context* ctx, Workspace& w, const cvg::DeepArgs& a, const cvg::ShallowArgs& b, bool sh,
                    bool dp, cudaEvent_t* pe, cudaStream_t st, bool strict, bool fused) {
  // overlap layout only when a shallow (or zero-fill) kernel shares the SMs
  // deep-only calls (sh false, the zero-fill kernel beside the deep one):
  // CVG_DEEP_ONLY 0 = overlapped beside a 16-warp deep block, 1 = serial (two
  // 16-warp deep blocks per SM, then the zero-fill), 2 = overlapped beside the
  // 21-warp deep block of the tiled schedule
  // 3 = a persistent four-warp zero-fill block beside a CVG_DEEPONLY_NW-warp
  // deep block (2 lanes per column)
  // (-1, default: by size.  modes 0 / 1 / 2 / 3 in ms: f02 0.384 / 0.354 / 0.355
  // / 0.317, c5_05 - / 0.161 / 0.107 / 0.101, c5_95 0.95 / 0.79 / 0.85 / 0.79, a
  // 445k-column half - / 0.216 / 0.192 / 0.188, a 257k-column quarter - / 0.1125
  // / 0.121 / 0.113, a 188k one - / 0.1197 / 0.1196 / 0.130 (1.1 claims per warp
  // at 28 warps), an 88k-column eighth 0.0725 / 0.0726 / 0.0668 / -, c2 0.029 /
  // 0.053 / 0.030 / -)
  int deep_only = ctx->deep_only >= 0 ? ctx->deep_only
                  : a.n >= 400000 ? 3 : a.n >= cvg::kTpcMinColumns / 2 ? 1 : a.n >= 32768 ? 2 : 0;
  if (deep_only == 3 && (ctx->deep_lpc >= 0 || ctx->deep_tpc == 1 || a.L > 32)) deep_only = 1;   // (2-lane builds only)
  const bool ov = ctx->overlap && dp && (sh || (!fused && deep_only != 1));
  const bool wide_deep_only = ov && !sh && !fused && deep_only == 2;
  const bool zero_beside = ov && !sh && !fused && deep_only == 3;
  const cudaStream_t main = st;
  // the tiled shallow kernel: overlapped deep + shallow calls whose tile
  // stages fit beside the deep block's tables (L <= 36 at 8 warps)
  const int tile_warps = ctx->tile_warps;
  const size_t tile_smem = cvg::shallow_tile_table_bytes() + (size_t)tile_warps * cvg::shallow_tile_stage_bytes(b.L);
  // (below 32k columns a warp gets at most a tile and the thread-per-column
  // kernel's finer grain wins: c1 0.028 vs 0.032 ms, c2 equal, c3 at 55k
  // columns 0.0456 vs 0.0469; CVG_SHALLOW_TILE=2 forces it)
  const bool tile = ov && sh && !fused && !b.trace && tile_smem + cvg::deep_table_bytes() <= 222 * 1024 &&
                    (ctx->shallow_tile == 2 || (ctx->shallow_tile == 1 && b.n >= 32768));
  // Programmatic dependent launch of the deep kernel: beside the tiled
  // shallow block, alone, or on small calls.  Beside the thread-per-column
  // shallow kernel it is a loss from ~50k columns (c3: 0.047 -> 0.052 ms; a
  // 64k-column all-triggered share 0.101 -> 0.132 ms).
  const bool pdl = ctx->pdl && (tile || !ov || b.n < 32768);
  // The fork stays AFTER the trigger kernel although the shallow kernel only
  // needs the per-call words reset: launched ahead of the deep block, the
  // shallow warps are the older ones on every SM and win the issue slots
  // (measured: shallow done 0.1 ms early, f02 step 0.393 -> 0.411 ms; the
  // thread-per-column shallow kernel even fills the SMs before the deep
  // blocks arrive, 0.65 ms).
  if (ov) CVG_CUDA(cudaEventRecord(w.ev_fork, st));
  // Thread-per-column deep kernel for large calls (the f02 grid on one or
  // two GPUs): 0.445 vs 0.508 ms per f02 step, 0.234 vs 0.251 ms on a 2-way
  // share; its 32-column claims take ~90 us per warp, so from 4-way shares
  // down the warp-per-column kernel's finer claims win (0.138 vs 0.152 ms,
  // 0.078 vs 0.089 ms at 8-way).  CVG_DEEP_TPC: 0 never, 1 always, 2 auto.
  // Deep kernel by call: the split-column kernel, 2 lanes per column from
  // 160k columns (f02: 0.420 ms step against 0.452 with one thread per
  // column and 0.508 warp-per-column), 4 below (shorter claims for small
  // shares); every variant (precip in k order, or on the relaxed path a
  // fixed-shape sum of the lanes' k-ordered partials).  CVG_DEEP_TPC=1 forces one
  // thread per column, CVG_DEEP_LPC=0 the warp-per-column kernel,
  // CVG_DEEP_LPC=2/4 the split width.
  const bool tpc_forced = ctx->deep_tpc == 1;
  // lanes per column by call size: 2 for large calls, 4 below 160k columns,
  // 8 below 100k (shorter per-warp chains when a call holds too few columns
  // to keep 2368 warps busy: 8-way f02 shares 0.089 -> 0.084 ms)
  int lpc_n = ctx->deep_lpc >= 0 ? ctx->deep_lpc
                                 : (a.n >= cvg::kTpcMinColumns / 2 ? 2 : a.n >= 100000 ? 4 : 8);
  if (lpc_n == 8 && (fused || !a.tree_precip || !ov)) lpc_n = 4;   // 8 lanes: overlapped relaxed builds only
  if (zero_beside) lpc_n = 2;
  if (fused && lpc_n <= 1 && !tpc_forced) lpc_n = 2;   // the warp-per-column kernel has no feedback-loop mode
  const bool lpc = !tpc_forced && dp && lpc_n > 1;
  const bool tpc = !lpc && dp && a.L <= 32 &&
                   (tpc_forced || (ctx->deep_tpc == 2 && a.n >= cvg::kTpcMinColumns));
  if (tpc || lpc) {
    const size_t smem = cvg::deep_table_bytes();
    // Launch shapes (warps per block x register cap, blocks per SM).  Beside
    // the shallow kernel: one 16-warp block capped at 64 registers (no
    // spills) -- exactly the register file left by four 128-thread shallow
    // blocks (f02 step 0.459 -> 0.429 ms against 12 warps x 80 registers;
    // 18 x 56 and 20 x 48 spill and lose).  Alone (deep only, the feedback
    // loop): two blocks per SM, 16 x 64 (default; f02 deep 0.292 ms against
    // 0.308 at 10 x 96, CVG_DEEP_ALONE=0).
    // The one-thread-per-column kernel (CVG_DEEP_TPC=1) keeps 12 x 104.
    void (*kern)(cvg::DeepArgs) = nullptr;
    const bool wide = ctx->deep_alone == 1;   // alone: 2 x 16 x 64 instead of 2 x 10 x 96
    int nwt = 0;
    const int blocks = ov ? 1 : 2;
    if (fused) {   // feedback loop (the deep kernel runs alone): the state-advancing builds
      nwt = wide ? 16 : 10;
      if (tpc) nwt = 10, kern = cvg::deep_tpc_kernel<VAR, 10, 96, 1, true, true>;
      else if (a.tree_precip)
        kern = wide ? (lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 16, 64, 2, false, true>
                                  : cvg::deep_tpc_kernel<VAR, 16, 64, 4, false, true>)
                    : (lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 10, 96, 2, false, true>
                                  : cvg::deep_tpc_kernel<VAR, 10, 96, 4, false, true>);
      else
        kern = wide ? (lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 16, 64, 2, true, true>
                                  : cvg::deep_tpc_kernel<VAR, 16, 64, 4, true, true>)
                    : (lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 10, 96, 2, true, true>
                                  : cvg::deep_tpc_kernel<VAR, 10, 96, 4, true, true>);
    } else if (tpc) {
      nwt = ov ? 12 : 10;
      kern = ov ? cvg::deep_tpc_kernel<VAR, 12, 104> : cvg::deep_tpc_kernel<VAR, 10, 96>;
    } else if (zero_beside) {
      constexpr int NWZ = CVG_DEEPONLY_NW;
      nwt = NWZ;
      kern = a.tree_precip ? cvg::deep_tpc_kernel<VAR, NWZ, 64, 2, false> : cvg::deep_tpc_kernel<VAR, NWZ, 64, 2>;
    } else if (ov && (tile || wide_deep_only)) {
      constexpr int NWT = CVG_TILE_NW, RC = CVG_TILE_REGS;   // deep warps x registers beside the tiled shallow block
      nwt = NWT;
      if (a.tree_precip)
        kern = lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, NWT, RC, 2, false>
               : lpc_n == 8 ? cvg::deep_tpc_kernel<VAR, NWT, RC, 8, false> : cvg::deep_tpc_kernel<VAR, NWT, RC, 4, false>;
      else kern = lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, NWT, RC, 2> : cvg::deep_tpc_kernel<VAR, NWT, RC, 4>;
    } else if (ov) {
      nwt = 16;
      if (a.tree_precip)
        kern = lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 16, 64, 2, false>
               : lpc_n == 8 ? cvg::deep_tpc_kernel<VAR, 16, 64, 8, false> : cvg::deep_tpc_kernel<VAR, 16, 64, 4, false>;
      else kern = lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 16, 64, 2> : cvg::deep_tpc_kernel<VAR, 16, 64, 4>;
    } else if (wide) {
      nwt = 16;
      if (a.tree_precip) kern = lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 16, 64, 2, false> : cvg::deep_tpc_kernel<VAR, 16, 64, 4, false>;
      else kern = lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 16, 64, 2> : cvg::deep_tpc_kernel<VAR, 16, 64, 4>;
    } else {
      nwt = 10;
      if (a.tree_precip) kern = lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 10, 96, 2, false> : cvg::deep_tpc_kernel<VAR, 10, 96, 4, false>;
      else kern = lpc_n == 2 ? cvg::deep_tpc_kernel<VAR, 10, 96, 2> : cvg::deep_tpc_kernel<VAR, 10, 96, 4>;
    }
    ctx->last_deep_kernel = std::string("deep_tpc_kernel<lanes_per_column=") + std::to_string(tpc ? 1 : lpc_n) +
                            ",k_order_precip=" + (tpc || !a.tree_precip ? "1" : "0") + ",warps=" +
                            std::to_string(nwt) + ",blocks_per_sm=" + std::to_string(blocks) + ">";
    CVG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CVG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, tile ? 100 : ctx->carveout));
    if (pdl) {
      // programmatic dependent launch behind the trigger kernel: the block's
      // table staging overlaps the trigger kernel and the launch latency
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)(ctx->num_sms * blocks));
      cfg.blockDim = dim3((unsigned)(nwt * 32));
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CVG_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    } else {
      kern<<<ctx->num_sms * blocks, nwt * 32, smem, st>>>(a);
    }
    CVG_CUDA(cudaGetLastError());
  } else if (dp) {
    // deep block size: kDeepWarpsOverlap leaves each SM room for three
    // shallow blocks beside the deep block; kDeepWarps when deep runs alone
    const int nw = ctx->deep_warps > 0 ? ctx->deep_warps : (ov ? cvg::kDeepWarpsOverlap : cvg::kDeepWarps);
    ctx->last_deep_kernel = std::string("deep_kernel<warp_per_column,warps=") + std::to_string(nw) + ">";
    if (a.L <= 32) {
      if (nw == 16) launch_deep_t<VAR, true, 16>(ctx, a, st);
      else if (nw == 20) launch_deep_t<VAR, true, 20>(ctx, a, st);
      else if (nw == 14) launch_deep_t<VAR, true, 14>(ctx, a, st);
      else if (nw == 24) launch_deep_t<VAR, true, 24>(ctx, a, st);
      else launch_deep_t<VAR, true, 12>(ctx, a, st);
    } else {
      if (nw == 16) launch_deep_t<VAR, false, 16>(ctx, a, st);
      else launch_deep_t<VAR, false, 12>(ctx, a, st);
    }
  }
  if (dp && a.relaxed && VAR != cvg::kVarApprox && ctx->redo_launch && !a.inline_redo) {
    // exact re-derivation of the solves the guard band flagged (a few
    // microseconds: one exact solve per thread, patches by the last block)
    const size_t smem = std::max((size_t)(cvg::kRedoThreads / 32) * a.L * sizeof(double),
                                 (size_t)cvg::kFixStaged * sizeof(unsigned long long));
    cvg::redo_kernel<VAR><<<ctx->num_sms * 2, cvg::kRedoThreads, smem, st>>>(a);
    CVG_CUDA(cudaGetLastError());
  }
  if (pe) CVG_CUDA(cudaEventRecord(pe[2], st));
  if (ov) {
    CVG_CUDA(cudaStreamWaitEvent(w.side, w.ev_fork, 0));
    st = w.side;
  }
  {
    const unsigned blocks = (unsigned)((b.n + cvg::kShallowThreads - 1) / cvg::kShallowThreads);
    const bool relax = VAR != cvg::kVarApprox && !strict;
    void (*k)(cvg::ShallowArgs) = nullptr;
    if (sh && fused) {   // feedback loop: the state-advancing builds
      k = relax ? cvg::shallow_kernel<VAR, true, false, true, 8, true> : cvg::shallow_kernel<VAR, true, false, false, 8, true>;
    } else if (sh && relax) {
      if (dp && ctx->shallow_minb == 12) k = cvg::shallow_kernel<VAR, true, true, true, 12>;
      else if (dp && ctx->shallow_minb == 16) k = cvg::shallow_kernel<VAR, true, true, true, 16>;
      else if (dp) k = cvg::shallow_kernel<VAR, true, true, true>;
      else k = cvg::shallow_kernel<VAR, true, false, true>;
    } else if (sh && dp) {
      k = cvg::shallow_kernel<VAR, true, true>;
    } else if (sh) {
      k = cvg::shallow_kernel<VAR, true, false>;
    } else if (dp && !fused) {   // (the feedback loop leaves untriggered columns untouched)
      k = cvg::shallow_kernel<VAR, false, true>;
    }
    if (zero_beside) {
      cvg::deep_zero_kernel<<<ctx->num_sms, cvg::kZeroThreads, 0, st>>>(b);
      ctx->last_shallow_kernel = "deep_zero_kernel<persistent,4 warps>";
      k = nullptr;
    }
    // shallow-only calls: the tiled kernel alone on the SM, with as many
    // warps (tiles in flight) as its stages fit (CVG_TILE_WARPS_ALONE)
    int alone_warps = ctx->tile_warps_alone;
    while (alone_warps > 1 && cvg::shallow_tile_table_bytes() + (size_t)alone_warps * cvg::shallow_tile_stage_bytes(b.L) >
                                  200 * 1024)
      --alone_warps;
    // (f02: 0.148 ms against the thread-per-column kernel's 0.236 -- 871 MB at
    // 5.9 TB/s, 90 % of the measured HBM copy bandwidth; 188k columns 0.040 vs
    // 0.064, 123k 0.031 vs 0.033, 88k 0.025 vs 0.023: from 100k columns)
    const bool tile_alone = sh && !dp && !fused && !b.trace && alone_warps >= 4 &&
                            (ctx->shallow_tile == 2 || (ctx->shallow_tile == 1 && b.n >= 100000));
    if (tile || tile_alone) {
      void (*tk)(cvg::ShallowArgs, const cvg::TileMaps) =
          tile ? (relax ? cvg::shallow_tile_kernel<VAR, true, true> : cvg::shallow_tile_kernel<VAR, true, false>)
               : (relax ? cvg::shallow_tile_kernel<VAR, false, true> : cvg::shallow_tile_kernel<VAR, false, false>);
      cvg::TileMaps maps{};
      cvg::ShallowArgs bt = b;
      bt.use_tma = ctx->tile_tma && encode_tile_maps(b, &maps);
      const int tw = tile ? tile_warps : alone_warps;
      const size_t smem = cvg::shallow_tile_table_bytes() + (size_t)tw * cvg::shallow_tile_stage_bytes(b.L);
      CVG_CUDA(cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CVG_CUDA(cudaFuncSetAttribute(tk, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      tk<<<ctx->num_sms, tw * 32, smem, st>>>(bt, maps);
      ctx->last_shallow_kernel = std::string("shallow_tile_kernel<warps=") + std::to_string(tw) +
                                 ",blocks_per_sm=1,tile=32 columns,stage=" + (bt.use_tma ? "TMA" : "cp.async") + ">";
    } else if (k) {
      ctx->last_shallow_kernel = sh ? "shallow_kernel<thread_per_column>" : "shallow_kernel<deep zero-fill only>";
      // same carveout as the deep kernel (launch_deep_t)
      CVG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, ctx->carveout));
      k<<<blocks, cvg::kShallowThreads, 0, st>>>(b);
    }
  }
  CVG_CUDA(cudaGetLastError());
  if (pe) CVG_CUDA(cudaEventRecord(pe[3], st));
  if (ov) {
    CVG_CUDA(cudaEventRecord(w.ev_join, st));
    CVG_CUDA(cudaStreamWaitEvent(main, w.ev_join, 0));
  }
}

// Redo list capacity of an n-column call: n/2 + 4096 queued levels (the f02
// grid queues ~1.4 % of its triggered columns' levels at the default guard;
// beyond the capacity fix_kernel recomputes every triggered column exactly).
long long redo_capacity(long long n) { return std::min<long long>(n / 2 + 4096, 0x3fffffffLL); }

// Sizes workspace w for an n-column deep call.  Buffers only grow, and a
// grown buffer's old allocation is retired (freed with the context), never
// freed under a CUDA graph that may still use it.  Growth while `st` is
// being captured (a caller's graph) is refused: allocation is not capturable
// and the graph would bake in the size -- size the workspace with one
// uncaptured call first.
void prepare_ws(cvg_context* ctx, Workspace& w, long long n, long long cap, cudaStream_t st);

// Enqueues the hot path on `st` with workspace `w`: memsets of the per-call
// cursors and failure words, the trigger + compaction kernel (deep
// requested), then the deep and shallow kernels.  Pointers are device
// pointers.  pe: optional 4 profiling events.
void enqueue(cvg_context* ctx, Workspace& w, const cvg_columns* in, const cvg_options* o, int mask,
             const cvg_outputs* deep, const cvg_outputs* sh, cudaStream_t st, cudaEvent_t* pe,
             const Fused* fu = nullptr) {
  const long long n = in->n_columns;
  const int L = in->n_levels;
  // the redo list: every level fits in the feedback-loop mode (its in-place
  // state cannot be recomputed from the inputs after an overflow)
  const long long cap = fu ? std::min<long long>(n * L, 0x3fffffffLL) : redo_capacity(n);
  if (fu) {
    // per-call words: reset by the previous step's step_end_kernel
  } else if (ctx->reset_kernel) {
    cvg::reset_call_words_kernel<<<1, 32, 0, st>>>(w.counters.p, 4, w.cursor.p, 20, w.err.p, 2);
    CVG_CUDA(cudaGetLastError());
  } else {
    CVG_CUDA(cudaMemsetAsync(w.counters.p, 0, 4 * sizeof(int), st));
    CVG_CUDA(cudaMemsetAsync(w.cursor.p, 0, 20 * sizeof(unsigned long long), st));
    CVG_CUDA(cudaMemsetAsync(w.err.p, 0xff, 2 * sizeof(unsigned long long), st));
  }
  if (n == 0) return;
  const bool do_deep = (mask & CVG_DEEP) != 0, do_sh = (mask & CVG_SHALLOW) != 0;
  const bool strict = ctx->strict || (o->flags & CVG_FLAG_STRICT) != 0;
  if (do_deep) prepare_ws(ctx, w, n, cap, st);
  if (pe) CVG_CUDA(cudaEventRecord(pe[0], st));
  cvg::DeepArgs a{};
  if (do_deep) {
    const long long ngroups = (n + cvg::kGroupCols - 1) / cvg::kGroupCols;
    const unsigned tb = (unsigned)((ngroups + cvg::kTrigThreads - 1) / cvg::kTrigThreads);
    cvg::trigger_groups_kernel<<<tb, cvg::kTrigThreads, 0, st>>>(in->s, n, o->activity_threshold, in->first_col,
                                                                  w.groups.p, w.counters.p, w.err.p);
    CVG_CUDA(cudaGetLastError());
    a.s = in->s; a.T = in->T; a.q = in->q; a.ld_in = in->ld;
    a.tend_T = deep->tend_T; a.tend_q = deep->tend_q; a.precip = deep->precip;
    a.work = deep->work_units; a.exited = deep->exited_early; a.ld_out = deep->ld;
    a.groups = w.groups.p; a.count = w.counters.p; a.cursor = w.cursor.p; a.n = n;
    a.err = w.err.p; a.first_col = in->first_col;
    a.thr = o->activity_threshold; a.tol = o->newton_tol; a.maxit = o->newton_max_iter;
    a.tol_lo = o->newton_tol * (1.0 - ctx->guard);
    a.tol_hi = o->newton_tol * (1.0 + ctx->guard);
    a.redo = w.redo.p;
    a.fix = w.fix.p;
    a.blocks_done = reinterpret_cast<unsigned*>(w.cursor.p + 16);   // reset per call
    a.redo_cap = (int)cap;
    // small calls re-derive inline (no dependent redo launch on a short
    // critical path: 8-way f02 shares 0.083 -> 0.079 ms); large calls hide
    // redo_kernel beside the shallow kernel's tail (inline costs 1-2 % there)
    a.inline_redo = ctx->redo_inline > 0 || (ctx->redo_inline < 0 && n < 100000);
    a.redo_count = w.counters.p + 2;
    a.fix_count = w.counters.p + 3;
    a.L = L;
    a.fast_div_ok = o->newton_tol >= 0x1.0p-500;
    // the relaxed path records update counts in 11 bits (queue_redo)
    a.relaxed = !strict && o->newton_max_iter <= cvg::kRedoMaxIter;
    a.far32 = a.relaxed && ctx->far32 && (o->flags & CVG_FLAG_NO_FAR32) == 0 && o->variant != CVG_APPROX_TRANSCENDENTAL;
    a.y_win = far_window_limit(o->newton_tol, a.far32);
    a.tree_precip = a.relaxed && o->variant != CVG_APPROX_TRANSCENDENTAL && o->newton_tol >= 0x1.0p-40;
    a.vec4 = deep->ld % 4 == 0 && aligned32(deep->tend_T) && aligned32(deep->tend_q);
  }
  a.gl_tab = ctx->gl_tab;
  a.exp_tab1 = ctx->exp_tab1.p;
  if (fu) {
    a.adv_T = fu->T; a.adv_q = fu->q; a.adv_bad = fu->bad;
  }
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
  b.tile_cursor = w.cursor.p + 8;
  b.bulk_ok = ((uintptr_t)in->T & 15) == 0 && ((uintptr_t)in->q & 15) == 0 && in->ld % 2 == 0;
  b.err = w.err.p + 1; b.gl_tab = ctx->gl_tab; b.exp_tab1 = ctx->exp_tab1.p; b.first_col = in->first_col;
  b.thr = o->activity_threshold; b.L = L;
  if (fu) {
    b.adv_T = fu->T; b.adv_q = fu->q; b.adv_bad = fu->bad;
  }
  if (ctx->trace_path && &w == &ctx->ws[0]) {
    ctx->trace_d.ensure(3 * 4096);
    ctx->trace_s.ensure(3 * (size_t)((n + 127) / 128 + 1));
    CVG_CUDA(cudaMemsetAsync(ctx->trace_d.p, 0, 3 * 4096 * 8, st));
    CVG_CUDA(cudaMemsetAsync(ctx->trace_s.p, 0, 3 * ((n + 127) / 128 + 1) * 8, st));
    a.trace = ctx->trace_d.p;
    b.trace = ctx->trace_s.p;
  }
  switch (o->variant) {
    case 1: launch_kernels<cvg::kVarReduced>(ctx, w, a, b, do_sh, do_deep, pe, st, strict, fu != nullptr); break;
    case 2: launch_kernels<cvg::kVarApprox>(ctx, w, a, b, do_sh, do_deep, pe, st, strict, fu != nullptr); break;
    default: launch_kernels<cvg::kVarExact>(ctx, w, a, b, do_sh, do_deep, pe, st, strict, fu != nullptr); break;
  }
}

void prepare_ws(cvg_context* ctx, Workspace& w, long long n, long long cap_, cudaStream_t st) {
  const size_t ngroups = (size_t)((n + cvg::kGroupCols - 1) / cvg::kGroupCols);
  const size_t cap = (size_t)cap_;
  if (w.groups.cap >= ngroups && w.redo.cap >= cvg::kRedoWords * cap && w.fix.cap >= 6 * cap) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CVG_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    throw std::invalid_argument("workspace too small for a call inside a stream capture: make one uncaptured "
                                "call of this size (or larger) on the context first");
  w.groups.grow(ngroups, ctx->retired);
  w.redo.grow(cvg::kRedoWords * cap, ctx->retired);
  w.fix.grow(6 * cap, ctx->retired);
}

// Queues the D2H of a workspace's latched failure words / trigger count.
void read_flags_async(Workspace& w, cudaStream_t st) {
  CVG_CUDA(cudaMemcpyAsync(w.h_err, w.err.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CVG_CUDA(cudaMemcpyAsync(w.h_count, w.counters.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
}

// Turns the folded failure keys (minimum over the call's chunks) into the
// reference's error: deep first, then shallow, as the reference runs
// deep_convection then shallow_convection; the lowest failing column.
cvg_status collect(const unsigned long long* keys_deep, const unsigned long long* keys_sh, long long triggered,
                   long long recomputed, long long corrected, int mask, int maxit, long long n,
                   cvg_stats* stats) {
  if (stats) {
    stats->n_columns = n;
    stats->n_triggered = (mask & CVG_DEEP) ? triggered : 0;
    stats->n_recomputed = (mask & CVG_DEEP) ? recomputed : 0;
    stats->n_corrected = (mask & CVG_DEEP) ? corrected : 0;
    stats->failing_column = -1;
    stats->failure_kind = 0;
    stats->failing_kernel = 0;
  }
  const unsigned long long none = ~0ULL;
  for (int w = 0; w < 2; ++w) {
    const int kernel = w == 0 ? CVG_DEEP : CVG_SHALLOW;
    if (!(mask & kernel)) continue;
    const unsigned long long key = w == 0 ? *keys_deep : *keys_sh;
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

// L rows of n doubles: device rows dld apart, host rows hld apart.
void copy_rows_h2d(double* dst, long long dld, const double* src, long long hld, long long n, int L,
                   cudaStream_t st) {
  if (dld == n && hld == n) {
    CVG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n * L, cudaMemcpyHostToDevice, st));
  } else {
    CVG_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * dld, src, sizeof(double) * hld, sizeof(double) * n, L,
                               cudaMemcpyHostToDevice, st));
  }
}

void copy_rows_d2h(double* dst, long long hld, const double* src, long long dld, long long n, int L,
                   cudaStream_t st) {
  if (dld == n && hld == n) {
    CVG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n * L, cudaMemcpyDeviceToHost, st));
  } else {
    CVG_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * hld, src, sizeof(double) * dld, sizeof(double) * n, L,
                               cudaMemcpyDeviceToHost, st));
  }
}

// Row pitch of the library's device staging buffers: a multiple of 32
// columns, so every level row starts on a 256-byte boundary and a 4-column
// group is one 32-byte sector in every row (an odd pitch splits the groups
// and the warps' 256-byte row segments across sectors: measured 25% slower).
constexpr long long pitch_cols(long long m) { return (m + 31) & ~31LL; }

}  // namespace

extern "C" {

const char* cvg_version(void) { return "0.3.0"; }

const char* cvg_last_error(void) { return g_last_error.c_str(); }

const char* cvg_last_deep_kernel(const cvg_context* ctx) { return ctx ? ctx->last_deep_kernel.c_str() : ""; }

const char* cvg_last_shallow_kernel(const cvg_context* ctx) { return ctx ? ctx->last_shallow_kernel.c_str() : ""; }

void cvg_default_options(cvg_options* o) {
  if (!o) return;
  o->variant = CVG_EXACT;
  o->activity_threshold = 0.5;
  o->newton_tol = 1e-12;
  o->newton_max_iter = 100;
  o->flags = 0;
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
    if (const char* e = getenv("CVG_OVERLAP")) ctx->overlap = atoi(e) != 0;
    if (const char* e = getenv("CVG_STRICT")) ctx->strict = atoi(e) != 0;
    if (const char* e = getenv("CVG_GRAPH")) ctx->use_graphs = atoi(e) != 0;
    if (const char* e = getenv("CVG_DEEP_TPC")) ctx->deep_tpc = atoi(e);
    if (const char* e = getenv("CVG_DEEP_LPC")) ctx->deep_lpc = atoi(e);
    if (const char* e = getenv("CVG_DEEP_ALONE")) ctx->deep_alone = atoi(e);
    if (const char* e = getenv("CVG_RESET_KERNEL")) ctx->reset_kernel = atoi(e) != 0;
    if (const char* e = getenv("CVG_CARVEOUT")) ctx->carveout = atoi(e);
    if (const char* e = getenv("CVG_FAR32")) ctx->far32 = atoi(e) != 0;
    if (const char* e = getenv("CVG_GUARD")) ctx->guard = std::max(0.0, std::min(0.5, atof(e)));
    if (const char* e = getenv("CVG_REDO")) ctx->redo_launch = atoi(e) != 0;
    if (const char* e = getenv("CVG_REDO_INLINE")) ctx->redo_inline = atoi(e);
    if (const char* e = getenv("CVG_SHALLOW_MINB")) ctx->shallow_minb = atoi(e);
    if (const char* e = getenv("CVG_DEEP_WARPS")) ctx->deep_warps = atoi(e);
    if (const char* e = getenv("CVG_SHALLOW_TILE")) ctx->shallow_tile = atoi(e);
    if (const char* e = getenv("CVG_PDL")) ctx->pdl = atoi(e) != 0;
    if (const char* e = getenv("CVG_TILE_TMA")) ctx->tile_tma = atoi(e) != 0;
    if (const char* e = getenv("CVG_TILE_WARPS_ALONE"))
      ctx->tile_warps_alone = std::max(1, std::min(cvg::kTileWarpsMax, atoi(e)));
    if (const char* e = getenv("CVG_DEEP_ONLY")) ctx->deep_only = atoi(e);
    if (const char* e = getenv("CVG_TILE_WARPS")) ctx->tile_warps = std::max(1, std::min(cvg::kTileWarpsMax, atoi(e)));
    if (const char* e = getenv("CVG_CHUNK_COLS")) ctx->chunk_cols = std::max(1LL, atoll(e));
    if (const char* e = getenv("CVG_SLOTS")) ctx->slots = std::max(1, std::min(kSlots, atoi(e)));
    ctx->trace_path = getenv("CVG_TRACE");
    try {
      CVG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      for (cudaEvent_t* e : {&ctx->ev0, &ctx->ev1, &ctx->ev_h0, &ctx->ev_h1}) CVG_CUDA(cudaEventCreate(e));
      const std::vector<double> tab = exp_table1_host();
      ctx->exp_tab1.ensure(tab.size());
      CVG_CUDA(cudaMemcpy(ctx->exp_tab1.p, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
      void* gl = nullptr;
      CVG_CUDA(cudaGetSymbolAddress(&gl, cvg::kExpGlTable));
      ctx->gl_tab = static_cast<const double2*>(gl);
      for (Workspace& w : ctx->ws) w.create();
      ctx->aux_err.ensure(1);
      CVG_CUDA(cudaMallocHost(&ctx->h_aux_err, sizeof(unsigned long long)));
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
  cudaDeviceSynchronize();
  ctx->exp_tab1.release();
  for (Workspace& w : ctx->ws) w.destroy();
  ctx->aux0.release();
  ctx->aux1.release();
  ctx->auxi.release();
  ctx->aux_err.release();
  ctx->trace_d.release();
  ctx->trace_s.release();
  if (ctx->h_aux_err) cudaFreeHost(ctx->h_aux_err);
  for (cudaEvent_t e : {ctx->ev0, ctx->ev1, ctx->ev_h0, ctx->ev_h1})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->prof_ev) cudaEventDestroy(e);
  for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.exec);
  for (void* p : ctx->retired) cudaFree(p);
  for (auto* b : {&ctx->loop.s, &ctx->loop.oT, &ctx->loop.oq, &ctx->loop.op, &ctx->leg.T, &ctx->leg.q}) b->release();
  ctx->loop.ow.release(); ctx->loop.ox.release(); ctx->loop_err.release(); ctx->loop_flag.release();
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

}  // extern "C"

namespace {

// One device-resident call as a CUDA graph (memsets, trigger, deep and
// shallow kernels with the fork/join): captured on first use of an argument
// set, replayed after -- one launch instead of ~8 stream operations, and
// the graph's dependency edges start each kernel with less front-end delay
// (fixed per-step cost matters at the small per-GPU shares of a
// multi-GPU partition).
void launch_graph(cvg_context* ctx, const cvg_columns* in, const cvg_options* o, int mask, const cvg_outputs* deep,
                  const cvg_outputs* sh, cudaStream_t st) {
  Workspace& w = ctx->ws[0];
  if (mask & CVG_DEEP) prepare_ws(ctx, w, in->n_columns, redo_capacity(in->n_columns), st);
  std::vector<unsigned char> key;
  auto put = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    key.insert(key.end(), b, b + n);
  };
  // the key is built field by field (struct padding bytes of a caller's
  // stack structs are indeterminate and must not defeat the cache)
  auto put_cols = [&](const cvg_columns* c) {
    put(&c->n_columns, sizeof(c->n_columns)); put(&c->n_levels, sizeof(c->n_levels));
    put(&c->first_col, sizeof(c->first_col)); put(&c->ld, sizeof(c->ld)); put(&c->s, sizeof(c->s));
    put(&c->T, sizeof(c->T)); put(&c->q, sizeof(c->q)); put(&c->on_device, sizeof(c->on_device));
  };
  auto put_opts = [&](const cvg_options* x) {
    put(&x->variant, sizeof(x->variant)); put(&x->activity_threshold, sizeof(x->activity_threshold));
    put(&x->newton_tol, sizeof(x->newton_tol)); put(&x->newton_max_iter, sizeof(x->newton_max_iter));
    put(&x->flags, sizeof(x->flags));
  };
  auto put_outs = [&](const cvg_outputs* x) {
    const cvg_outputs none{};
    if (!x) x = &none;
    put(&x->tend_T, sizeof(x->tend_T)); put(&x->tend_q, sizeof(x->tend_q)); put(&x->precip, sizeof(x->precip));
    put(&x->work_units, sizeof(x->work_units)); put(&x->exited_early, sizeof(x->exited_early));
    put(&x->ld, sizeof(x->ld)); put(&x->on_device, sizeof(x->on_device));
  };
  put_cols(in);
  put_opts(o);
  put(&mask, sizeof(mask));
  put_outs((mask & CVG_DEEP) ? deep : nullptr);
  put_outs((mask & CVG_SHALLOW) ? sh : nullptr);
  put(&w.groups.p, sizeof(w.groups.p));
  put(&w.groups.cap, sizeof(w.groups.cap));
  put(&w.redo.p, sizeof(w.redo.p));
  put(&w.fix.p, sizeof(w.fix.p));
  for (auto& g : ctx->graphs)
    if (g.key == key) {
      CVG_CUDA(cudaGraphLaunch(g.exec, st));
      return;
    }
  cudaGraph_t graph = nullptr;
  CVG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
  try {
    enqueue(ctx, w, in, o, mask, deep, sh, st, nullptr);
  } catch (...) {
    cudaStreamEndCapture(st, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  CVG_CUDA(cudaStreamEndCapture(st, &graph));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  CVG_CUDA(e);
  if (ctx->graphs.size() >= 16) {
    cudaGraphExecDestroy(ctx->graphs.front().exec);
    ctx->graphs.erase(ctx->graphs.begin());
  }
  ctx->graphs.push_back({std::move(key), exec});
  CVG_CUDA(cudaGraphLaunch(exec, st));
}

}  // namespace

extern "C" {

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
    cudaEvent_t* pe = nullptr;
    if (ctx->prof_on && ctx->prof_n < ctx->prof_cap) pe = &ctx->prof_ev[4 * ctx->prof_n++];
    // a caller capturing its own graph on this stream gets the plain
    // launches recorded into it (no nested capture)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CVG_CUDA(cudaStreamIsCapturing(st, &cap));
    if (pe || ctx->trace_path || !ctx->use_graphs || in->n_columns == 0 || cap != cudaStreamCaptureStatusNone) {
      enqueue(ctx, ctx->ws[0], in, opts, mask, deep, sh, st, pe);
    } else {
      launch_graph(ctx, in, opts, mask, deep, sh, st);
    }
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
    Workspace& w = ctx->ws[0];
    read_flags_async(w, st);
    CVG_CUDA(cudaStreamSynchronize(st));
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
    ctx->pending = false;   // reported once; the next call resets the device words
    return collect(&w.h_err[0], &w.h_err[1], w.h_count[1], w.h_count[2], w.h_count[3], ctx->last_mask,
                   ctx->last_maxit, ctx->last_n, stats);
  });
}

// Host-buffer (or mixed) call.  Column chunks of chunk_cols columns are
// pipelined through the kSlots workspaces, each on its own stream: chunk i's
// H2D, chunk i-1's kernels and chunk i-2's D2H run concurrently (two copy
// engines, full-duplex PCIe), so a host-buffer call costs roughly its larger
// transfer direction rather than the sum of transfers and compute.  Results
// equal a single-chunk call bit for bit: columns are independent and every
// failure key carries the absolute column id, so the lowest failing column
// is the minimum over chunks.  All-device calls run as one chunk.
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
    const long long n = in->n_columns;
    const int L = in->n_levels;
    const bool all_dev = in->on_device && (!(mask & CVG_DEEP) || deep->on_device) &&
                         (!(mask & CVG_SHALLOW) || sh->on_device);
    // chunk boundaries: the first chunks ramp up geometrically from
    // chunk_cols/8 so the D2H stream (the larger direction) starts early
    std::vector<long long> bounds{0};
    if (all_dev || n == 0) {
      bounds.push_back(n);
    } else {
      long long c = std::max(1LL, ctx->chunk_cols / 8);
      while (bounds.back() < n) {
        bounds.push_back(std::min(n, bounds.back() + c));
        c = std::min(ctx->chunk_cols, 2 * c);
      }
    }
    const long long nchunks = (long long)bounds.size() - 1;
    long long h2d = 0, d2h = 0;
    CVG_CUDA(cudaEventRecord(ctx->ev_h0, ctx->stream));
    unsigned long long md = ~0ULL, ms_ = ~0ULL;
    long long trig = 0, recomp = 0, corr = 0;
    double h2d_ms = 0.0, d2h_ms = 0.0;
    bool busy[kSlots] = {};
    auto drain = [&](Workspace& w) {  // a slot's previous chunk: wait, fold its flags and copy times
      CVG_CUDA(cudaStreamSynchronize(w.stream));
      md = std::min(md, w.h_err[0]);
      ms_ = std::min(ms_, w.h_err[1]);
      trig += w.h_count[1];
      recomp += w.h_count[2];
      corr += w.h_count[3];
      if (w.copy_timed) {
        float a = 0.f, b = 0.f;
        CVG_CUDA(cudaEventElapsedTime(&a, w.ev_copy[0], w.ev_copy[1]));
        CVG_CUDA(cudaEventElapsedTime(&b, w.ev_copy[2], w.ev_copy[3]));
        h2d_ms += a;
        d2h_ms += b;
        w.copy_timed = false;
      }
    };
    for (long long ci = 0; ci < nchunks; ++ci) {
      const int slot = (int)(ci % ctx->slots);
      Workspace& w = ctx->ws[slot];
      if (busy[slot]) drain(w);
      CVG_CUDA(cudaStreamWaitEvent(w.stream, ctx->ev_h0, 0));
      const long long c0 = bounds[ci];
      const long long m = bounds[ci + 1] - c0;
      const long long mp = pitch_cols(m);
      const size_t mL = (size_t)mp * L;
      cvg_columns din = *in;
      din.n_columns = m;
      din.first_col = in->first_col + c0;
      if (in->on_device) {
        if (m > 0) { din.s = in->s + c0; din.T = in->T + c0; din.q = in->q + c0; }
      } else if (m > 0) {
        w.in_s.ensure(m); w.in_T.ensure(mL); w.in_q.ensure(mL);
        CVG_CUDA(cudaEventRecord(w.ev_copy[0], w.stream));
        CVG_CUDA(cudaMemcpyAsync(w.in_s.p, in->s + c0, sizeof(double) * m, cudaMemcpyHostToDevice, w.stream));
        copy_rows_h2d(w.in_T.p, mp, in->T + c0, in->ld, m, L, w.stream);
        copy_rows_h2d(w.in_q.p, mp, in->q + c0, in->ld, m, L, w.stream);
        h2d += (long long)(sizeof(double) * (m + 2 * (size_t)m * L));
        CVG_CUDA(cudaEventRecord(w.ev_copy[1], w.stream));
        din.s = w.in_s.p; din.T = w.in_T.p; din.q = w.in_q.p; din.ld = mp; din.on_device = 1;
      }
      auto stage = [&](const cvg_outputs* o, DevBuf<double>& T, DevBuf<double>& q, DevBuf<double>& p,
                       DevBuf<long long>& wk, DevBuf<uint8_t>& x) {
        cvg_outputs d = *o;
        if (o->on_device) {
          if (m > 0) {
            d.tend_T = o->tend_T + c0; d.tend_q = o->tend_q + c0; d.precip = o->precip + c0;
            d.work_units = o->work_units + c0; d.exited_early = o->exited_early + c0;
          }
        } else if (m > 0) {
          T.ensure(mL); q.ensure(mL); p.ensure(m); wk.ensure(m); x.ensure(m);
          d.tend_T = T.p; d.tend_q = q.p; d.precip = p.p; d.work_units = wk.p; d.exited_early = x.p;
          d.ld = mp; d.on_device = 1;
        }
        return d;
      };
      cvg_outputs ddeep{}, dsh{};
      if (mask & CVG_DEEP) ddeep = stage(deep, w.dT, w.dq, w.dp, w.dw, w.dx);
      if (mask & CVG_SHALLOW) dsh = stage(sh, w.sT, w.sq, w.sp, w.sw, w.sx);
      enqueue(ctx, w, &din, opts, mask, &ddeep, &dsh, w.stream, nullptr);
      auto unstage = [&](const cvg_outputs* o, const cvg_outputs& d) {
        if (o->on_device || m <= 0) return;
        copy_rows_d2h(o->tend_T + c0, o->ld, d.tend_T, mp, m, L, w.stream);
        copy_rows_d2h(o->tend_q + c0, o->ld, d.tend_q, mp, m, L, w.stream);
        CVG_CUDA(cudaMemcpyAsync(o->precip + c0, d.precip, sizeof(double) * m, cudaMemcpyDeviceToHost, w.stream));
        CVG_CUDA(cudaMemcpyAsync(o->work_units + c0, d.work_units, sizeof(long long) * m, cudaMemcpyDeviceToHost,
                                 w.stream));
        CVG_CUDA(cudaMemcpyAsync(o->exited_early + c0, d.exited_early, m, cudaMemcpyDeviceToHost, w.stream));
        d2h += (long long)(sizeof(double) * (2 * (size_t)m * L + m) + sizeof(long long) * m + m);
      };
      const bool host_out = ((mask & CVG_DEEP) && !deep->on_device) || ((mask & CVG_SHALLOW) && !sh->on_device);
      if (!in->on_device && host_out && m > 0) CVG_CUDA(cudaEventRecord(w.ev_copy[2], w.stream));
      if (mask & CVG_DEEP) unstage(deep, ddeep);
      if (mask & CVG_SHALLOW) unstage(sh, dsh);
      if (!in->on_device && host_out && m > 0) {
        CVG_CUDA(cudaEventRecord(w.ev_copy[3], w.stream));
        w.copy_timed = true;
      }
      read_flags_async(w, w.stream);
      busy[slot] = true;
    }
    for (int s = 0; s < kSlots; ++s)
      if (busy[s]) drain(ctx->ws[s]);
    cvg_status rc = collect(&md, &ms_, trig, recomp, corr, mask, opts->newton_max_iter, n, stats);
    if (stats) {
      for (int s = 0; s < kSlots; ++s) {
        CVG_CUDA(cudaEventRecord(ctx->ev1, ctx->ws[s].stream));
        CVG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev1, 0));
      }
      CVG_CUDA(cudaEventRecord(ctx->ev_h1, ctx->stream));
      CVG_CUDA(cudaEventSynchronize(ctx->ev_h1));
      float all = 0.f;
      CVG_CUDA(cudaEventElapsedTime(&all, ctx->ev_h0, ctx->ev_h1));
      stats->device_ms = all;   // whole call, transfers overlapped with compute
      stats->h2d_ms = h2d_ms;   // summed over the chunks (each overlaps other chunks' work)
      stats->d2h_ms = d2h_ms;
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
    CVG_CUDA(cudaMemsetAsync(ctx->aux_err.p, 0xff, sizeof(unsigned long long), st));
    const unsigned blocks = (unsigned)((n + 255) / 256);
    switch (opts->variant) {
      case 2: cvg::ientropy_kernel<cvg::kVarApprox><<<blocks, 256, 0, st>>>(dy, dg, n, opts->newton_tol,
                  opts->newton_max_iter, ctx->aux0.p, ctx->auxi.p, ctx->aux_err.p, ctx->gl_tab); break;
      default: cvg::ientropy_kernel<cvg::kVarExact><<<blocks, 256, 0, st>>>(dy, dg, n, opts->newton_tol,
                  opts->newton_max_iter, ctx->aux0.p, ctx->auxi.p, ctx->aux_err.p, ctx->gl_tab); break;
    }
    CVG_CUDA(cudaGetLastError());
    CVG_CUDA(cudaMemcpyAsync(root, ctx->aux0.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaMemcpyAsync(iterations, ctx->auxi.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaMemcpyAsync(ctx->h_aux_err, ctx->aux_err.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaStreamSynchronize(st));
    const unsigned long long key = *ctx->h_aux_err;
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

cvg_status cvg_exp(cvg_context* ctx, long long n, const double* x, double* out) {
  if (!ctx || (n > 0 && (!x || !out))) return fail(CVG_ERR_INVALID, "cvg_exp: null argument");
  if (n < 0) return fail(CVG_ERR_INVALID, "cvg_exp: n < 0");
  return guarded([&] {
    if (n == 0) return CVG_OK;
    CVG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    ctx->aux0.ensure(n);
    ctx->aux1.ensure(n);
    CVG_CUDA(cudaMemcpyAsync(ctx->aux1.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    cvg::exp_gl_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ctx->aux1.p, ctx->aux0.p, n, ctx->gl_tab);
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

}  // extern "C"

// --- feedback loop ----------------------------------------------------------

namespace {

unsigned elem_blocks(long long n, int L) { return (unsigned)((n * L + 255) / 256); }

// One step of `kernel` over a device leg, its failure words copied to
// err_slot, then advance with the non-finite flag in *flag.
void leg_step(cvg_context* ctx, const cvg_options* o, int kernel, long long n, int L, const double* s,
              LegBufs& leg, LoopBufs& lb, unsigned long long* err_slot, unsigned* flag, cudaStream_t st) {
  Workspace& w = ctx->ws[0];
  const cvg_columns in{n, L, 0, n, s, leg.T.p, leg.q.p, 1};
  const cvg_outputs out = lb.outs(n);
  enqueue(ctx, w, &in, o, kernel, kernel == CVG_DEEP ? &out : nullptr, kernel == CVG_SHALLOW ? &out : nullptr, st,
          nullptr);
  CVG_CUDA(cudaMemcpyAsync(err_slot, w.err.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
  if (n > 0) {
    cvg::advance_kernel<<<elem_blocks(n, L), 256, 0, st>>>(leg.T.p, leg.q.p, n, lb.oT.p, lb.oq.p, n, n, L, flag);
    CVG_CUDA(cudaGetLastError());
  }
}

// Reads the legs' failure words (in leg order) and raises the first kernel
// failure as cvg_convect would.
cvg_status leg_errors(const unsigned long long* h_err, int nlegs, int kernel, int maxit, long long n) {
  for (int l = 0; l < nlegs; ++l) {
    const unsigned long long* e = h_err + 2 * l;
    if (e[0] != ~0ULL || e[1] != ~0ULL) return collect(&e[0], &e[1], 0, 0, 0, kernel, maxit, n, nullptr);
  }
  return CVG_OK;
}

}  // namespace

extern "C" {

cvg_status cvg_timestep(cvg_context* ctx, long long n, int L, long long ld, const double* s, double* T,
                        double* q, int on_device, const cvg_options* opts, int kernel, int n_steps,
                        cvg_stats* stats) {
  if (!ctx || !opts || (n > 0 && (!s || !T || !q))) return fail(CVG_ERR_INVALID, "cvg_timestep: null argument");
  std::string why;
  const cvg_columns probe{n, L, 0, ld, s, T, q, on_device};
  if (!valid_columns(&probe, &why) || !valid_options(opts, &why)) return fail(CVG_ERR_INVALID, "cvg_timestep: " + why);
  if (kernel != CVG_DEEP && kernel != CVG_SHALLOW)
    return fail(CVG_ERR_INVALID, "cvg_timestep: kernel must be CVG_DEEP or CVG_SHALLOW");
  if (n_steps < 0) return fail(CVG_ERR_INVALID, "cvg_timestep: n_steps < 0");
  return guarded([&] {
    CVG_CUDA(cudaSetDevice(ctx->device));
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (stats) stats->failing_column = -1;
    cudaStream_t st = ctx->stream;
    LoopBufs& lb = ctx->loop;
    LegBufs& leg = ctx->leg;
    // Fused loop: every step is trigger -> kernel (writing the advanced
    // state in place, with the check_finite flag) -> re-derivation ->
    // step_end (the step's failure words and flag saved in slot t % K); the
    // host synchronises once per K steps and reports the first failing step
    // as the reference's per-step checks would (validate.cpp:127-153).
    constexpr int K = 16;
    DevBuf<unsigned long long>& slots = ctx->loop_err;   // [K][2] failure words
    DevBuf<unsigned>& words = ctx->loop_flag;            // [0] flag, [1] step, [2..2+K) flags per slot
    lb.ensure(std::max(n, 1LL), L);
    leg.T.ensure((size_t)std::max(n, 1LL) * L);
    leg.q.ensure((size_t)std::max(n, 1LL) * L);
    slots.ensure(2 * K);
    words.ensure(2 + K);
    const cudaMemcpyKind kin = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const cudaMemcpyKind kout = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    Workspace& w = ctx->ws[0];
    if (n > 0) {
      CVG_CUDA(cudaMemcpyAsync(lb.s.p, s, sizeof(double) * n, kin, st));
      CVG_CUDA(cudaMemcpy2DAsync(leg.T.p, sizeof(double) * n, T, sizeof(double) * ld, sizeof(double) * n, L, kin, st));
      CVG_CUDA(cudaMemcpy2DAsync(leg.q.p, sizeof(double) * n, q, sizeof(double) * ld, sizeof(double) * n, L, kin, st));
    }
    CVG_CUDA(cudaMemsetAsync(words.p, 0, (2 + K) * sizeof(unsigned), st));
    cvg::reset_call_words_kernel<<<1, 32, 0, st>>>(w.counters.p, 4, w.cursor.p, 20, w.err.p, 2);
    if (n > 0) {   // the initial state's non-finite values (columns the steps never touch)
      cvg::nonfinite_scan_kernel<<<ctx->num_sms * 4, 256, 0, st>>>(leg.T.p, leg.q.p, n, n, L, words.p);
    }
    CVG_CUDA(cudaGetLastError());
    const cvg_columns in{n, L, 0, n, lb.s.p, leg.T.p, leg.q.p, 1};
    const cvg_outputs out = lb.outs(n);
    const Fused fu{leg.T.p, leg.q.p, words.p};
    std::vector<unsigned long long> h_err(2 * K);
    std::vector<unsigned> h_bad(K);
    CVG_CUDA(cudaEventRecord(ctx->ev0, st));   // stats->device_ms: the stepping region (no state transfers)
    for (int t0 = 0; t0 < n_steps && n > 0; t0 += K) {
      const int kk = std::min(K, n_steps - t0);
      for (int j = 0; j < kk; ++j) {
        enqueue(ctx, w, &in, opts, kernel, kernel == CVG_DEEP ? &out : nullptr, kernel == CVG_SHALLOW ? &out : nullptr,
                st, nullptr, &fu);
        cvg::step_end_kernel<<<1, 32, 0, st>>>(words.p + 1, w.counters.p, w.cursor.p, w.err.p, words.p, slots.p,
                                               words.p + 2, K);
        CVG_CUDA(cudaGetLastError());
      }
      CVG_CUDA(cudaMemcpyAsync(h_err.data(), slots.p, sizeof(unsigned long long) * 2 * K, cudaMemcpyDeviceToHost, st));
      CVG_CUDA(cudaMemcpyAsync(h_bad.data(), words.p + 2, sizeof(unsigned) * K, cudaMemcpyDeviceToHost, st));
      CVG_CUDA(cudaStreamSynchronize(st));
      for (int j = 0; j < kk; ++j) {   // step t0 + j sits in slot (t0 + j) % K = j
        const cvg_status rc = leg_errors(&h_err[2 * j], 1, kernel, opts->newton_max_iter, n);
        if (rc != CVG_OK) {
          if (stats) stats->failing_column = (long long)(std::min(h_err[2 * j], h_err[2 * j + 1]) >> 16);
          return rc;
        }
        if (h_bad[j]) return fail(CVG_ERR_CHECK, "timestep: state diverged at step " + std::to_string(t0 + j));
      }
    }
    CVG_CUDA(cudaEventRecord(ctx->ev1, st));
    if (n > 0) {
      CVG_CUDA(cudaMemcpy2DAsync(T, sizeof(double) * ld, leg.T.p, sizeof(double) * n, sizeof(double) * n, L, kout, st));
      CVG_CUDA(cudaMemcpy2DAsync(q, sizeof(double) * ld, leg.q.p, sizeof(double) * n, sizeof(double) * n, L, kout, st));
    }
    CVG_CUDA(cudaStreamSynchronize(st));
    if (stats) {
      stats->n_columns = n;
      float ms = 0.f;
      CVG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
      stats->device_ms = ms;
    }
    return CVG_OK;
  });
}

cvg_status cvg_error_growth(cvg_context* ctx, const cvg_columns* init, int kernel, const cvg_options* base,
                            const cvg_options* mod, int timesteps, double* rms_mod, double* rms_pert,
                            cvg_growth* out) {
  if (!ctx || !init || !base || !mod || !out || (timesteps > 0 && (!rms_mod || !rms_pert)))
    return fail(CVG_ERR_INVALID, "cvg_error_growth: null argument");
  std::string why;
  if (!valid_columns(init, &why) || !valid_options(base, &why) || !valid_options(mod, &why))
    return fail(CVG_ERR_INVALID, "cvg_error_growth: " + why);
  if (kernel != CVG_DEEP && kernel != CVG_SHALLOW)
    return fail(CVG_ERR_INVALID, "cvg_error_growth: kernel must be CVG_DEEP or CVG_SHALLOW");
  if (timesteps < 0) return fail(CVG_ERR_INVALID, "cvg_error_growth: timesteps < 0");
  out->envelope_ok = 1;
  out->worst_ratio = 0.0;
  out->failing_step = -1;
  return guarded([&] {
    CVG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const long long n = init->n_columns;
    const int L = init->n_levels;
    const long long nn = std::max(n, 1LL);
    LoopBufs lb;
    LegBufs legs[3];   // baseline, modified, perturbed
    DevBuf<unsigned long long> err;
    DevBuf<unsigned> flags;
    DevBuf<double> partials, sums;
    struct Free {
      LoopBufs& lb; LegBufs* legs; DevBuf<unsigned long long>& err; DevBuf<unsigned>& flags;
      DevBuf<double>& partials; DevBuf<double>& sums;
      ~Free() {
        for (auto* b : {&lb.s, &lb.oT, &lb.oq, &lb.op, &partials, &sums}) b->release();
        lb.ow.release(); lb.ox.release(); err.release(); flags.release();
        for (int l = 0; l < 3; ++l) { legs[l].T.release(); legs[l].q.release(); }
      }
    } guard{lb, legs, err, flags, partials, sums};
    lb.ensure(nn, L);
    for (auto& leg : legs) { leg.T.ensure((size_t)nn * L); leg.q.ensure((size_t)nn * L); }
    err.ensure(6);
    flags.ensure(4);
    const int rb = (int)std::min<long long>(4 * ctx->num_sms, std::max(1LL, (n * L + cvg::kRmsThreads - 1) / cvg::kRmsThreads));
    partials.ensure(2 * (size_t)rb);
    sums.ensure(2 * (size_t)std::max(timesteps, 1));
    const cudaMemcpyKind kin = init->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (n > 0) {
      CVG_CUDA(cudaMemcpyAsync(lb.s.p, init->s, sizeof(double) * n, kin, st));
      for (auto& leg : legs) {
        CVG_CUDA(cudaMemcpy2DAsync(leg.T.p, sizeof(double) * n, init->T, sizeof(double) * init->ld, sizeof(double) * n,
                                   L, kin, st));
        CVG_CUDA(cudaMemcpy2DAsync(leg.q.p, sizeof(double) * n, init->q, sizeof(double) * init->ld, sizeof(double) * n,
                                   L, kin, st));
      }
    }
    CVG_CUDA(cudaMemsetAsync(flags.p, 0, 4 * sizeof(unsigned), st));
    if (n > 0) {   // perturbed leg: T one ulp off everywhere (validate.cpp:174-177)
      cvg::perturb_lsb_kernel<<<elem_blocks(n, L), 256, 0, st>>>(legs[2].T.p, n, n, L, flags.p + 3);
      CVG_CUDA(cudaGetLastError());
    }
    unsigned h_flags[4] = {};
    CVG_CUDA(cudaMemcpyAsync(h_flags, flags.p, sizeof(h_flags), cudaMemcpyDeviceToHost, st));
    CVG_CUDA(cudaStreamSynchronize(st));
    if (h_flags[3]) return fail(CVG_ERR_CHECK, "perturb_lsb: non-finite value");
    const cvg_options* leg_opts[3] = {base, mod, base};
    const char* leg_name[3] = {"baseline", "modified", "perturbed"};
    for (int t = 0; t < timesteps; ++t) {
      if (n > 0) {
        for (int l = 0; l < 3; ++l)
          leg_step(ctx, leg_opts[l], kernel, n, L, lb.s.p, legs[l], lb, err.p + 2 * l, flags.p + l, st);
        cvg::rms_partial_kernel<<<rb, cvg::kRmsThreads, 0, st>>>(legs[0].T.p, legs[1].T.p, legs[2].T.p, n, n, L,
                                                                 partials.p);
        cvg::rms_final_kernel<<<1, 32, 0, st>>>(partials.p, rb, sums.p + 2 * t);
        CVG_CUDA(cudaGetLastError());
      }
      unsigned long long h_err[6];
      CVG_CUDA(cudaMemcpyAsync(h_err, err.p, sizeof(h_err), cudaMemcpyDeviceToHost, st));
      CVG_CUDA(cudaMemcpyAsync(h_flags, flags.p, 3 * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
      CVG_CUDA(cudaStreamSynchronize(st));
      if (n > 0) {
        for (int l = 0; l < 3; ++l) {   // run_path of each leg in order (validate.cpp:183-185)
          cvg_status rc = leg_errors(h_err + 2 * l, 1, kernel, leg_opts[l]->newton_max_iter, n);
          if (rc != CVG_OK) return rc;
        }
      }
      for (int l = 0; l < 3; ++l) {    // check_finite in order (:186-188)
        if (h_flags[l]) {
          out->failing_step = t;
          return fail(CVG_ERR_CHECK, std::string("error_growth: ") + leg_name[l] + " leg diverged");
        }
      }
    }
    std::vector<double> h_sums(2 * (size_t)std::max(timesteps, 1), 0.0);
    if (timesteps > 0 && n > 0)
      CVG_CUDA(cudaMemcpy(h_sums.data(), sums.p, sizeof(double) * 2 * timesteps, cudaMemcpyDeviceToHost));
    const double cnt = (double)(n * L);
    for (int t = 0; t < timesteps; ++t) {   // validate.cpp:190-205
      const double rm = n > 0 ? std::sqrt(h_sums[2 * t] / cnt) : 0.0;
      const double rp = n > 0 ? std::sqrt(h_sums[2 * t + 1] / cnt) : 0.0;
      rms_mod[t] = rm;
      rms_pert[t] = rp;
      if (rm > rp) out->envelope_ok = 0;
      const double ratio = rp > 0.0 ? rm / rp : (rm > 0.0 ? std::numeric_limits<double>::infinity() : 0.0);
      if (ratio > out->worst_ratio) out->worst_ratio = ratio;
    }
    return CVG_OK;
  });
}

#ifdef CVG_PHASE_CLOCKS
// debug builds: read and reset the deep worker's phase clocks
cvg_status cvg_debug_phases(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, cvg::g_phase, sizeof(unsigned long long) * 8);
  const unsigned long long z[8] = {};
  cudaMemcpyToSymbol(cvg::g_phase, z, sizeof(z));
  return CVG_OK;
}
#endif

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

// --- Multi-device engine ------------------------------------------------------
//
// The reference's partitioned execution is one call, HeteroEngine::step
// (hetero.cpp:252-466), over a plan from plan_partition (hetero.cpp:156-176):
// a host pool and an emulated device each take a contiguous column range.
// Here G device contexts each take one contiguous range, balanced by the
// estimated cost w_c = deep_weight [s_c > thr] + shallow_weight
// (cvg_plan_partition), and run concurrently, one host thread per device,
// each staging its range over its own PCIe link (cvg_convect).  Columns are
// independent (physics.hpp:26-30), so the ranges need no exchange: the union
// of the G outputs equals one single-device call bit for bit.

struct cvg_multi {
  std::vector<cvg_context*> ctx;
  double deep_weight = 0.86;     // measured ns per triggered column (multigpu.py, tools/fit_partition.py)
  double shallow_weight = 0.154; // measured ns per column
};

namespace {

// Interior offsets rounded to multiples of 32 columns (each range's rows then
// start on 256-byte boundaries in the staging buffers), kept monotone.
void align_bounds(long long* b, int parts, long long n) {
  for (int i = 1; i < parts; ++i) {
    long long r = (b[i] + 16) / 32 * 32;
    b[i] = std::min(n, std::max(b[i - 1], r));
  }
  b[parts] = n;
}

}  // namespace

extern "C" {

cvg_status cvg_multi_create(const int* devices, int n_devices, cvg_multi** out) {
  if (!out || !devices) return fail(CVG_ERR_INVALID, "cvg_multi_create: null argument");
  *out = nullptr;
  if (n_devices < 1 || n_devices > 64) return fail(CVG_ERR_INVALID, "cvg_multi_create: n_devices must be in [1, 64]");
  auto* m = new cvg_multi();
  for (int i = 0; i < n_devices; ++i) {
    cvg_context* c = nullptr;
    const cvg_status st = cvg_context_create(devices[i], &c);
    if (st != CVG_OK) {
      const std::string msg = cvg_last_error();
      cvg_multi_free(m);
      return fail(st, "cvg_multi_create: device " + std::to_string(devices[i]) + ": " + msg);
    }
    m->ctx.push_back(c);
  }
  g_last_error.clear();
  *out = m;
  return CVG_OK;
}

void cvg_multi_free(cvg_multi* m) {
  if (!m) return;
  for (cvg_context* c : m->ctx) cvg_context_free(c);
  delete m;
}

int cvg_multi_size(const cvg_multi* m) { return m ? (int)m->ctx.size() : 0; }

cvg_context* cvg_multi_context(cvg_multi* m, int i) {
  if (!m || i < 0 || i >= (int)m->ctx.size()) return nullptr;
  return m->ctx[i];
}

cvg_status cvg_multi_set_weights(cvg_multi* m, double deep_weight, double shallow_weight) {
  if (!m) return fail(CVG_ERR_INVALID, "cvg_multi_set_weights: null handle");
  if (!(shallow_weight >= 0.0) || !std::isfinite(deep_weight))
    return fail(CVG_ERR_INVALID, "cvg_multi_set_weights: bad weights");
  m->deep_weight = deep_weight;
  m->shallow_weight = shallow_weight;
  g_last_error.clear();
  return CVG_OK;
}

cvg_status cvg_multi_convect(cvg_multi* m, const cvg_columns* in, const cvg_options* opts, int mask,
                             const cvg_outputs* deep, const cvg_outputs* sh, cvg_stats* stats,
                             long long* bounds_out) {
  if (!m || !in || !opts) return fail(CVG_ERR_INVALID, "cvg_multi_convect: null argument");
  std::string why;
  if (!valid_columns(in, &why) || !valid_options(opts, &why)) return fail(CVG_ERR_INVALID, "cvg_multi_convect: " + why);
  if (mask < 1 || mask > 3) return fail(CVG_ERR_INVALID, "cvg_multi_convect: kernel_mask must be 1, 2 or 3");
  if ((mask & CVG_DEEP) && (!deep || !valid_outputs(deep, in->n_columns, &why)))
    return fail(CVG_ERR_INVALID, "cvg_multi_convect: deep outputs: " + (deep ? why : std::string("null")));
  if ((mask & CVG_SHALLOW) && (!sh || !valid_outputs(sh, in->n_columns, &why)))
    return fail(CVG_ERR_INVALID, "cvg_multi_convect: shallow outputs: " + (sh ? why : std::string("null")));
  if (in->on_device || ((mask & CVG_DEEP) && deep->on_device) || ((mask & CVG_SHALLOW) && sh->on_device))
    return fail(CVG_ERR_INVALID,
                "cvg_multi_convect: host buffers only (device-resident ranges: cvg_convect_async on each "
                "cvg_multi_context)");
  const int G = (int)m->ctx.size();
  const long long n = in->n_columns;
  std::vector<long long> b(G + 1, 0);
  cvg_status rc = cvg_plan_partition(n, in->s, opts->activity_threshold, G, m->deep_weight, m->shallow_weight,
                                     b.data());
  if (rc != CVG_OK) return rc;
  align_bounds(b.data(), G, n);
  if (bounds_out) std::copy(b.begin(), b.end(), bounds_out);
  struct Part {
    cvg_status rc = CVG_OK;
    cvg_stats st{};
    std::string msg;
  };
  std::vector<Part> parts(G);
  auto run = [&](int i) {
    const long long c0 = b[i], m_i = b[i + 1] - b[i];
    cvg_columns ci = *in;
    ci.n_columns = m_i;
    ci.first_col = in->first_col + c0;
    ci.s = in->s + c0;
    ci.T = in->T + c0;
    ci.q = in->q + c0;
    auto slice = [&](const cvg_outputs* o) {
      cvg_outputs d = *o;
      d.tend_T += c0; d.tend_q += c0; d.precip += c0; d.work_units += c0; d.exited_early += c0;
      return d;
    };
    cvg_outputs dd{}, ds{};
    if (mask & CVG_DEEP) dd = slice(deep);
    if (mask & CVG_SHALLOW) ds = slice(sh);
    parts[i].rc = cvg_convect(m->ctx[i], &ci, opts, mask, (mask & CVG_DEEP) ? &dd : nullptr,
                              (mask & CVG_SHALLOW) ? &ds : nullptr, &parts[i].st);
    if (parts[i].rc != CVG_OK) parts[i].msg = cvg_last_error();
  };
  std::vector<std::thread> th;
  for (int i = 1; i < G; ++i) th.emplace_back(run, i);
  run(0);
  for (auto& t : th) t.join();
  // merge: the reference reports the first failure of its serial order --
  // deep before shallow, then the lowest column; ranges are in column order
  int pick = -1;
  for (int pass = 0; pass < 2 && pick < 0; ++pass) {
    const int kern = pass == 0 ? CVG_DEEP : CVG_SHALLOW;
    for (int i = 0; i < G; ++i)
      if (parts[i].rc == CVG_ERR_NUMERIC && parts[i].st.failing_kernel == kern) { pick = i; break; }
  }
  if (pick < 0)
    for (int i = 0; i < G; ++i)
      if (parts[i].rc != CVG_OK) { pick = i; break; }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->n_columns = n;
    stats->failing_column = -1;
    for (int i = 0; i < G; ++i) {
      const cvg_stats& s = parts[i].st;
      stats->n_triggered += s.n_triggered;
      stats->n_recomputed += s.n_recomputed;
      stats->n_corrected += s.n_corrected;
      stats->h2d_bytes += s.h2d_bytes;
      stats->d2h_bytes += s.d2h_bytes;
      stats->device_ms = std::max(stats->device_ms, s.device_ms);
      stats->h2d_ms = std::max(stats->h2d_ms, s.h2d_ms);
      stats->d2h_ms = std::max(stats->d2h_ms, s.d2h_ms);
    }
    if (pick >= 0) {
      stats->failing_column = parts[pick].st.failing_column;
      stats->failure_kind = parts[pick].st.failure_kind;
      stats->failing_kernel = parts[pick].st.failing_kernel;
    }
  }
  if (pick >= 0) return fail(parts[pick].rc, parts[pick].msg);
  g_last_error.clear();
  return CVG_OK;
}

}  // extern "C"

/*
 * convgpu.h -- C ABI of the B200 (sm_100a) deep + shallow convection column
 * path.  Drop-in for the reference's column-batch entry points:
 *
 *   std::vector<ColumnOutput> deep_convection(const Chunk&, const KernelOptions&)
 *   std::vector<ColumnOutput> shallow_convection(const Chunk&, const KernelOptions&)
 *       /root/reference/proj/src/core/physics.hpp:155-158
 *   IentropyResult ientropy_solve(double y, double guess, const KernelOptions&)
 *       physics.hpp:101 (physics.cpp:101-104)
 *   double approx_exp(double x)                        physics.hpp:83
 *
 * Conventions follow the reference C API (proj/include/convproxy.h:34-41,
 * proj/src/capi.cpp:39-89): every call returns a cvg_status with the same
 * numeric codes as cvp_status; on failure cvg_last_error() holds a
 * thread-local message, cleared by the next successful call; null arguments
 * give CVG_ERR_INVALID with "null" in the message; no C++ exception crosses
 * this boundary.  A kernel failure (KernelError in the reference,
 * errors.hpp:26-36) returns CVG_ERR_NUMERIC, names the LOWEST failing column
 * ("... column <id>") -- the column the serial driver physics.cpp:227-245
 * would have thrown on -- and stores it in cvg_stats.failing_column.
 *
 * Data layout: level-major structure of arrays.  Field f of level k, column c
 * lives at f[k * ld + c] (ld >= n_columns); per-column scalars are f[c].
 * Pointers may be host or device memory (cvg_columns.on_device); the caller
 * owns every buffer; inputs are never modified.  The library owns only its
 * per-context device workspace and streams.
 *
 * One call in flight per context; contexts are independent (one per device /
 * per rank).  All pointers and sizes are plain C types.
 */
#ifndef CONVGPU_H_
#define CONVGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum cvg_status {
  CVG_OK = 0,
  CVG_ERR_INVALID = 1, /* null handle, bad argument, internal failure      */
  CVG_ERR_CONFIG = 2,  /* (reserved; same code as CVP_ERR_CONFIG)          */
  CVG_ERR_NUMERIC = 3, /* kernel numeric failure: NaN, divergence, maxiter  */
  CVG_ERR_CHECK = 4,   /* validation check failed (divergence, perturbation) */
  CVG_ERR_IO = 5,      /* (reserved; same code as CVP_ERR_IO)              */
  CVG_ERR_DEVICE = 6   /* CUDA runtime failure or no usable sm_100 device  */
} cvg_status;

/* convproxy::Variant, physics.hpp:62-66 */
typedef enum cvg_variant {
  CVG_EXACT = 0,
  CVG_STRENGTH_REDUCED = 1,
  CVG_APPROX_TRANSCENDENTAL = 2
} cvg_variant;

/* Which kernels one cvg_convect call runs. */
enum { CVG_DEEP = 1, CVG_SHALLOW = 2, CVG_BOTH = 3 };

/* Failure kinds reported in cvg_stats.failure_kind (reference messages in
 * physics.cpp:67, :79, :84-85, :109, :172). */
enum {
  CVG_FAIL_NONE = 0,
  CVG_FAIL_ACTIVITY = 1, /* non-finite activity s           */
  CVG_FAIL_INPUT = 2,    /* ientropy: non-finite input      */
  CVG_FAIL_DIVERGED = 3, /* ientropy: iterate diverged      */
  CVG_FAIL_NOCONV = 4    /* ientropy: no convergence        */
};

/* convproxy::KernelOptions, physics.hpp:68-73 (same defaults). */
typedef struct cvg_options {
  int variant;               /* cvg_variant, default CVG_EXACT   */
  double activity_threshold; /* default 0.5                       */
  double newton_tol;         /* default 1e-12 (absolute)          */
  int newton_max_iter;       /* default 100                       */
  int flags;                 /* CVG_FLAG_*, default 0             */
} cvg_options;

/* cvg_options.flags: reference rounding in every Newton update of every
 * variant (the default relaxed update of Exact/StrengthReduced differs from
 * it only by rounding noise inside the parity window). */
#define CVG_FLAG_STRICT 1
/* cvg_options.flags: no FP32 far phase in the relaxed Newton solve (the far
 * steps of Exact/StrengthReduced run in FP32 until |resid| <= 0.1, then the
 * solve continues in FP64). */
#define CVG_FLAG_NO_FAR32 2

/* Input column block (the SoA form of convproxy::Chunk, physics.hpp:39-43). */
typedef struct cvg_columns {
  long long n_columns;
  int n_levels;
  long long first_col; /* column id of column 0 (ColumnState::col_id)     */
  long long ld;        /* row stride of T and q in elements (>= n_columns) */
  const double* s;     /* [n]        activity                              */
  const double* T;     /* [L][ld]    temperature-like field                */
  const double* q;     /* [L][ld]    moisture-like field                   */
  int on_device;       /* 1: pointers are device memory on the ctx device */
} cvg_columns;

/* Output block (the SoA form of std::vector<ColumnOutput>, physics.hpp:52-60). */
typedef struct cvg_outputs {
  double* tend_T;         /* [L][ld] */
  double* tend_q;         /* [L][ld] */
  double* precip;         /* [n]     */
  long long* work_units;  /* [n]     */
  uint8_t* exited_early;  /* [n]     */
  long long ld;           /* row stride of tend_T / tend_q (>= n_columns) */
  int on_device;
} cvg_outputs;

typedef struct cvg_stats {
  long long n_columns;
  long long n_triggered;     /* deep columns with s > activity_threshold      */
  long long failing_column;  /* lowest failing column id, or -1              */
  int failure_kind;          /* CVG_FAIL_*                                    */
  int failing_kernel;        /* CVG_DEEP / CVG_SHALLOW, 0 when none          */
  double device_ms;          /* device time of the compute (CUDA events)      */
  double h2d_ms, d2h_ms;     /* host-buffer calls with host inputs: staging
                                copy time, summed over the pipeline's chunks
                                (CUDA events; chunks overlap, so the sums can
                                exceed device_ms); 0 otherwise               */
  long long h2d_bytes, d2h_bytes;
  long long n_recomputed;    /* deep levels whose relaxed stop decision fell
                                in the guard band around newton_tol and were
                                re-derived on the exact path (reference
                                rounding, libm-exact exp)                     */
  long long n_corrected;     /* columns that re-derivation rewrote (an update
                                count differed from the relaxed one)          */
} cvg_stats;

typedef struct cvg_context cvg_context;

const char* cvg_version(void);
const char* cvg_last_error(void);
/* The deep kernel (and its launch shape) of the context's last call. */
const char* cvg_last_deep_kernel(const cvg_context* ctx);
const char* cvg_last_shallow_kernel(const cvg_context* ctx);   /* likewise, the shallow kernel */
void cvg_default_options(cvg_options* opts);

/* Creates a context on CUDA device `device` (requires compute capability 10.x). */
cvg_status cvg_context_create(int device, cvg_context** out);
void cvg_context_free(cvg_context* ctx);

/* Runs deep and/or shallow convection (kernel_mask) over one column block.
 * deep / shallow may be NULL when not requested.  Host buffers are staged
 * through pinned device workspace; device buffers are used in place.  On
 * return all outputs are complete (the call synchronises its stream).
 * stats may be NULL. */
cvg_status cvg_convect(cvg_context* ctx, const cvg_columns* in,
                       const cvg_options* opts, int kernel_mask,
                       const cvg_outputs* deep, const cvg_outputs* shallow,
                       cvg_stats* stats);

/* Asynchronous device-resident form for steady-state loops and CUDA-graph
 * capture: all pointers must be device memory; work is enqueued on `stream`
 * (a cudaStream_t, NULL = the context stream) and errors are latched on the
 * device.  cvg_convect_check() synchronises that stream, reads the latched
 * error of the last cvg_convect_async call and fills stats; the error is
 * reported once (a second check without a new call returns CVG_OK with
 * zeroed stats).  A call captured into a caller's CUDA graph uses the
 * context workspace as sized by an earlier uncaptured call of at least the
 * same column count (growth inside a capture returns CVG_ERR_INVALID); the
 * workspace never shrinks or moves under such a graph. */
cvg_status cvg_convect_async(cvg_context* ctx, const cvg_columns* in,
                             const cvg_options* opts, int kernel_mask,
                             const cvg_outputs* deep,
                             const cvg_outputs* shallow, void* stream);
cvg_status cvg_convect_check(cvg_context* ctx, void* stream, cvg_stats* stats);

/* Reference batch entry points (physics.hpp:155-158) over HOST SoA buffers. */
cvg_status cvg_deep_convection(cvg_context* ctx, const cvg_columns* in,
                               const cvg_options* opts, const cvg_outputs* out,
                               cvg_stats* stats);
cvg_status cvg_shallow_convection(cvg_context* ctx, const cvg_columns* in,
                                  const cvg_options* opts,
                                  const cvg_outputs* out, cvg_stats* stats);

/* Batched inverse-entropy solve on the device (physics.hpp:101): n
 * independent (y, guess) pairs -> root, iterations.  On failure returns
 * CVG_ERR_NUMERIC with the lowest failing index in the message. */
cvg_status cvg_ientropy_solve(cvg_context* ctx, long long n, const double* y,
                              const double* guess, const cvg_options* opts,
                              double* root, int* iterations);

/* Device evaluation of approx_exp (physics.hpp:83) over n host values. */
cvg_status cvg_approx_exp(cvg_context* ctx, long long n, const double* x,
                          double* out);

/* Device evaluation of the Exact variant's exp_eval (physics.cpp:35: the
 * libm exp) over n host values: bit-identical to glibc 2.39's exp (the
 * restated algorithm of colmath.cuh exp_gl). */
cvg_status cvg_exp(cvg_context* ctx, long long n, const double* x, double* out);

/* --- Feedback loop (validate.cpp:113-206) ------------------------------ */

/* Device-resident timestep loop: n_steps times, run `kernel` (CVG_DEEP =
 * deep_column or CVG_SHALLOW = shallow_column) over the state and advance it,
 * T += tend_T, q += tend_q (validate.cpp:127-136); s is not advanced.  T and
 * q ([L][ld], host or device per on_device) are updated in place; the state
 * stays in HBM between steps.  After each step a non-finite T or q returns
 * CVG_ERR_CHECK ("timestep: state diverged at step <t>", check_finite,
 * validate.cpp:138-153) with stats->failing_column = -1; a kernel failure
 * returns CVG_ERR_NUMERIC as cvg_convect does.  stats may be NULL. */
cvg_status cvg_timestep(cvg_context* ctx, long long n, int n_levels, long long ld, const double* s,
                        double* T, double* q, int on_device, const cvg_options* opts, int kernel,
                        int n_steps, cvg_stats* stats);

typedef struct cvg_growth {
  int envelope_ok;     /* rms_mod[t] <= rms_pert[t] for every t              */
  double worst_ratio;  /* max over t of rms_mod / rms_pert (validate.cpp:198-204) */
  int failing_step;    /* timestep of a divergence (CVG_ERR_CHECK), else -1  */
} cvg_growth;

/* error_growth (validate.hpp:71-82), device-resident: three legs from the
 * same initial grid for `timesteps` steps of the feedback loop -- baseline
 * (options `baseline`), modified (options `modified`), perturbed (initial T
 * with its least significant bit flipped, perturb_lsb, validate.cpp:29-34;
 * options `baseline`) -- and after every step the RMS difference of the
 * modified and perturbed legs' temperature fields against the baseline's
 * (rms_mod[t], rms_pert[t], each of length timesteps).  A non-finite initial
 * T returns CVG_ERR_CHECK ("perturb_lsb: non-finite value"); a leg whose state
 * turns non-finite returns CVG_ERR_CHECK ("error_growth: <leg> leg diverged",
 * out->failing_step = t), checked in the order baseline, modified,
 * perturbed.  The RMS sums run as a fixed-order tree on the device, so they
 * differ from the reference's serial sum by rounding only. */
cvg_status cvg_error_growth(cvg_context* ctx, const cvg_columns* initial, int kernel,
                            const cvg_options* baseline, const cvg_options* modified, int timesteps,
                            double* rms_mod, double* rms_pert, cvg_growth* out);

/* Host-side partition of a column block across n_parts devices, balanced by
 * estimated cost w_c = deep_weight * [s_c > thr] + shallow_weight
 * (generalises plan_partition, hetero.cpp:156-176, from a 2-pool split to
 * G contiguous ranges).  bounds receives n_parts + 1 offsets, bounds[0] = 0,
 * bounds[n_parts] = n.  deep_weight <= 0 selects the naive equal-columns
 * split (the analogue of StaticBlock, sched.cpp:66-75). */
cvg_status cvg_plan_partition(long long n, const double* s,
                              double activity_threshold, int n_parts,
                              double deep_weight, double shallow_weight,
                              long long* bounds);

/* --- Multi-device engine (HeteroEngine::step, hetero.cpp:252-466) ------ */

typedef struct cvg_multi cvg_multi;

/* One context per listed CUDA device (a device may be listed more than once:
 * independent contexts sharing one GPU).  Partition weights default to the
 * measured per-unit costs of one B200 (0.86 ns per triggered column, 0.154
 * ns per column; tools/fit_partition.py). */
cvg_status cvg_multi_create(const int* devices, int n_devices, cvg_multi** out);
void cvg_multi_free(cvg_multi* m);
int cvg_multi_size(const cvg_multi* m);
/* The i-th device context (owned by m), e.g. for device-resident calls. */
cvg_context* cvg_multi_context(cvg_multi* m, int i);
/* Cost model of the partition (cvg_plan_partition): deep_weight <= 0 gives
 * the naive equal-columns split (StaticBlock, sched.cpp:66-75). */
cvg_status cvg_multi_set_weights(cvg_multi* m, double deep_weight, double shallow_weight);

/* cvg_convect over every device of m, host buffers only: G contiguous column
 * ranges balanced by the cost model (interior bounds rounded to 32 columns),
 * each staged over its own device's PCIe link and computed there,
 * concurrently (one host thread per device).  The outputs equal one
 * single-device call bit for bit.  stats (nullable) merges the devices:
 * counts and bytes summed, device_ms the slowest device, the failure the
 * reference's serial order would report (deep before shallow, lowest
 * column).  bounds (nullable) receives the G + 1 range offsets. */
cvg_status cvg_multi_convect(cvg_multi* m, const cvg_columns* in, const cvg_options* opts, int kernel_mask,
                             const cvg_outputs* deep, const cvg_outputs* shallow, cvg_stats* stats,
                             long long* bounds);

/* --- Measurement support (bench.py) ----------------------------------- */

/* Per-kernel device timing: while enabled, every cvg_convect_async call
 * records CUDA events around each of its kernels on the launching stream
 * (slots for up to max_steps calls).  cvg_profile_end returns, per recorded
 * call, the durations in ms of [trigger+compaction, deep, shallow] (row-major
 * [n_steps][3], 0 for a kernel not launched) and disables recording. */
cvg_status cvg_profile_begin(cvg_context* ctx, int max_steps);
cvg_status cvg_profile_end(cvg_context* ctx, int* n_steps, double* kernel_ms, int capacity);

/* FP64 pipe peak of this device, measured now: a DFMA-chain probe over all
 * SMs (2 FLOP per DFMA), best of `reps` launches.  This is the FP64
 * roofline denominator (MEASURED_PEAKS.json carries no FP64 figure). */
cvg_status cvg_fp64_peak(cvg_context* ctx, int reps, double* tflops);

/* Page-locked host memory for staging (cudaMallocHost). */
cvg_status cvg_host_alloc(size_t bytes, void** out);
void cvg_host_free(void* p);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* CONVGPU_H_ */

/* rfk.h — C ABI of the B200-native Randers eikonal hot path.
 *
 * This is the drop-in boundary for the reference's C++ API in
 * proj/include/randers/{stencil,sweeper,adjoint,feasibility}.hpp.  Every
 * entry point below names the reference function it replaces (file:line).
 * The C++ shim in paper_2603_00035_b200/csrc/shim/randers_shim.cpp maps these
 * onto the exact randers:: signatures (Grid2D, MetricField, ... and the
 * randers::Error hierarchy), so reference callers such as
 * objective_and_grad (src/inversion.cpp:25-73) link against it unchanged;
 * other FFIs (ctypes, cgo, JNI) bind the plain functions directly — see
 * INTEGRATION.md.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All field buffers are SoA row-major
 *    planes (node index r*cols + c, grid.hpp:33-38), one plane per channel.
 *  - `mem` says where EVERY pointer argument of the call lives
 *    (RFK_MEM_HOST: the library stages through device memory and copies
 *    results back; RFK_MEM_DEVICE: pointers are device pointers and nothing
 *    crosses PCIe).
 *  - Batches: `batch` independent grids of one shape; plane k of grid i
 *    starts at ptr + i*stride.  A stride of 0 broadcasts one plane to every
 *    grid (e.g. one metric, many source sets — objective_and_grad's loop).
 *  - Calls are synchronous with respect to their status: they return after
 *    the work on the context's stream has completed.
 *  - Errors are returned as rfk_status; rfk_last_error() gives the message.
 *    Status codes map 1:1 onto the reference's exception types
 *    (include/randers/errors.hpp:8-50).
 *  - Arithmetic: fp64, bit-identical to the reference (no FMA contraction,
 *    reference operation order).  There is no CPU fallback: without a CUDA
 *    device every compute call returns RFK_ERR_NO_DEVICE.
 */
#ifndef RFK_H
#define RFK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define RFK_API __attribute__((visibility("default")))
#else
#define RFK_API
#endif

typedef enum {
    RFK_OK = 0,
    RFK_ERR_DIMENSION_MISMATCH = 1,       /* randers::DimensionMismatch      (sweeper.cpp:79-82) */
    RFK_ERR_ZERO_DIMENSION = 2,           /* randers::ZeroDimension          (grid.hpp:61-63)    */
    RFK_ERR_INVALID_ARGUMENT = 3,         /* randers::InvalidArgument        (grid.hpp:64,124-126, feasibility.hpp:15-20) */
    RFK_ERR_INCONSISTENT_FIXED_POINT = 4, /* randers::InconsistentFixedPoint (adjoint.cpp:22-25)  */
    RFK_ERR_CUDA = 5,                     /* CUDA runtime failure            */
    RFK_ERR_NO_DEVICE = 6,                /* no CUDA device: no CPU fallback */
    RFK_ERR_ALLOC = 7,                    /* device allocation failed        */
    RFK_ERR_NOT_CONVERGED = 8,            /* randers::NotConverged           (inversion.cpp:36-37) */
    RFK_ERR_NON_SPD_INPUT = 9,            /* randers::NonSpdInput            (feasibility.cpp:79) */
    RFK_ERR_DIVERGED_LOSS = 10            /* randers::DivergedLoss           (inversion.cpp:356-357) */
} rfk_status;

typedef enum { RFK_MEM_HOST = 0, RFK_MEM_DEVICE = 1 } rfk_memory;

/* UpdateType (sweeper.hpp:14) */
enum { RFK_TWO_POINT = 0, RFK_ONE_POINT = 1, RFK_NO_RECORD = -1 };

typedef struct rfk_context rfk_context;

/* A batch of problems on one grid shape (GridSpec grid.hpp:56-69 + fields
 * grid.hpp:73-127).  fixed_values != NULL selects solve_from_values
 * semantics (sweeper.cpp:168-174): fixed nodes hold those values instead of 0. */
typedef struct {
    int32_t batch;
    int32_t rows, cols;
    double h;
    const double* g11;
    const double* g12;
    const double* g22;
    const double* b1;
    const double* b2;
    int64_t param_stride; /* elements between grids' parameter planes (0 = shared) */
    const uint8_t* src;   /* nonzero = source / fixed node */
    int64_t src_stride;   /* elements between grids' masks (0 = shared) */
    const double* fixed_values; /* optional; stride src_stride */
} rfk_fields;

/* SolveOptions (sweeper.hpp:49-55) */
typedef struct {
    double tol;               /* default 1e-6 */
    int32_t max_iters;        /* default 50   */
    int32_t sweep_order[4];   /* default {0,1,2,3} */
} rfk_solve_options;

/* Per-node stencil records (StencilRecord, adjoint.hpp:13-30) as planes of
 * batch*rows*cols elements.  type: RFK_TWO_POINT / RFK_ONE_POINT /
 * RFK_NO_RECORD.  donor1/donor2: Moore-ring neighbour ids 0..7 (stencil.hpp:
 * 17-18), donor2 = -1 for one-point.  Caches: two-point c0..c4 =
 * (q11, q12, q22, u1, u2); one-point c0, c1 = (r_edge, e_edge). */
typedef struct {
    int8_t* type;
    int8_t* stencil;
    int8_t* donor1;
    int8_t* donor2;
    double* c[5];
} rfk_records;

/* ---- context --------------------------------------------------------- */
RFK_API rfk_status rfk_create(rfk_context** ctx, int device);
RFK_API void rfk_destroy(rfk_context* ctx);
/* cudaStream_t passed as void*; NULL = the legacy default stream */
RFK_API rfk_status rfk_set_stream(rfk_context* ctx, void* stream);
RFK_API const char* rfk_last_error(const rfk_context* ctx);
RFK_API const char* rfk_status_string(rfk_status s);
RFK_API int rfk_version(void);
/* Number of device kernels this context has launched (instrumentation for
 * the bench's gpu_launches claim). */
RFK_API int64_t rfk_launch_count(const rfk_context* ctx);
/* Device workspace: the context keeps grow-only named buffers sized by the
 * largest problem seen (the reference allocates per call).  Query the bytes
 * held, or release them all (e.g. between problem sizes). */
RFK_API int64_t rfk_workspace_bytes(const rfk_context* ctx);
RFK_API rfk_status rfk_release_workspace(rfk_context* ctx);
/* Diagnostics: in a trace build of the library (-DRFK_SWEEP_TRACE_BUILD=1,
 * scripts/trace_sweep.py) and with RFK_TRACE set in the environment,
 * rfk_solve records a per-pass/per-band timing record (32 words each);
 * copies up to max_words of the last solve's record to host `out` and
 * returns the count (0 in the product build, which has no traced kernel). */
RFK_API int64_t rfk_debug_trace(rfk_context* ctx, unsigned long long* out, int64_t max_words);

/* ---- forward ---------------------------------------------------------- */

/* solve / solve_from_values: fast sweeping, sweeper.cpp:133-174.
 * Bit-identical T, iteration count and max_delta_history to the reference.
 * Outputs: t (batch*rows*cols), iterations[batch], converged[batch],
 * history (batch*max_iters, may be NULL). */
RFK_API rfk_status rfk_solve(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                             const rfk_solve_options* opt, double* t, int32_t* iterations,
                             int32_t* converged, double* history);

/* solve_jacobi: sweeper.cpp:176-205 (sweep_order ignored). */
RFK_API rfk_status rfk_solve_jacobi(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                    const rfk_solve_options* opt, double* t,
                                    int32_t* iterations, int32_t* converged, double* history);

/* best_candidate / node_update (sweeper.cpp:8-72) at a list of nodes of one
 * grid (f->batch must be 1). */
RFK_API rfk_status rfk_best_candidate(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                      const double* t, int64_t n_nodes, const int32_t* nodes,
                                      int32_t node_update, double* t0, int8_t* type,
                                      int8_t* stencil, int8_t* donor1, int8_t* donor2,
                                      double* lam1, double* lam2, int8_t* found);

/* two_point_update (stencil.cpp:7-43), elementwise over n inputs. */
RFK_API rfk_status rfk_two_point_update(rfk_context* ctx, rfk_memory mem, int64_t n,
                                        const double* t1, const double* t2, const double* m1x,
                                        const double* m1y, const double* m2x, const double* m2y,
                                        const double* g11, const double* g12, const double* g22,
                                        const double* b1, const double* b2, double* t0,
                                        double* lam1, double* lam2, int8_t* valid);

/* ---- backward --------------------------------------------------------- */

/* identify_stencils (adjoint.cpp:10-67).  two_point_count/one_point_count/
 * bad_node are per grid; bad_node = first row-major node that failed the
 * consistency check (-1 if none) and the call returns
 * RFK_ERR_INCONSISTENT_FIXED_POINT if any grid has one. */
RFK_API rfk_status rfk_identify(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                const double* t, double tol, const rfk_records* rec,
                                int32_t* two_point_count, int32_t* one_point_count,
                                int64_t* bad_node);

/* jacobian_entries (adjoint.cpp:69-89), elementwise over n records. */
RFK_API rfk_status rfk_jacobian_entries(rfk_context* ctx, rfk_memory mem, int64_t n,
                                        const int8_t* type, const double* c0, const double* c1,
                                        const double* c2, const double* c3, const double* c4,
                                        double* diag, double* j0, double* j1, int8_t* clamped);

/* solve_adjoint (adjoint.cpp:91-117): lambda planes and clamped counts. */
RFK_API rfk_status rfk_solve_adjoint(rfk_context* ctx, rfk_memory mem, int32_t batch,
                                     int32_t rows, int32_t cols, const double* t,
                                     const rfk_records* rec, const double* loss_grad,
                                     double* lambda, int32_t* clamped);

/* param_gradients (adjoint.cpp:119-144): five gradient planes per grid. */
RFK_API rfk_status rfk_param_gradients(rfk_context* ctx, rfk_memory mem, int32_t batch,
                                       int32_t rows, int32_t cols, double h,
                                       const rfk_records* rec, const double* lambda,
                                       double* d_g11, double* d_g12, double* d_g22,
                                       double* d_b1, double* d_b2);

/* loss_grad_mse (adjoint.cpp:146-160).  exact_sum != 0 reproduces the
 * reference's sequential loss sum bit-for-bit (one device thread per grid);
 * 0 uses a deterministic tree sum (≤ ~1e-15 relative difference). */
RFK_API rfk_status rfk_loss_grad_mse(rfk_context* ctx, rfk_memory mem, int32_t batch,
                                     int64_t n, const double* t, const uint8_t* observed,
                                     const double* values, double* grad, double* loss,
                                     int32_t* unreached, int32_t exact_sum);

/* Fused backward: identify_stencils -> solve_adjoint -> param_gradients for
 * every grid of the batch, on device, no records materialised.  When the
 * parameters are shared (param_stride == 0) and accumulate != 0, the per-grid
 * gradients are summed in grid order into one set of planes exactly as
 * objective_and_grad's accumulate (inversion.cpp:13-21); otherwise gradient
 * planes are per grid.  lambda may be NULL. */
RFK_API rfk_status rfk_backward(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                const double* t, double tol, const double* loss_grad,
                                double* lambda, double* d_g11, double* d_g12, double* d_g22,
                                double* d_b1, double* d_b2, int32_t accumulate,
                                int32_t* clamped, int64_t* bad_node);

/* ---- the feasibility projection fused into the load stage ------------------
 * ParamView::project (inversion.cpp:255-279; project_spd / project_drift,
 * feasibility.cpp:31-72) applied to raw parameters on their way into the
 * solver: the sweep's hoist (which reads every node's G and b once anyway)
 * projects each node as it reads it and emits the projected planes beside its
 * stencil records, and the backward's parameter-gradient pass applies the
 * projection's VJP (rfk_project_vjp) to the gradients before writing them --
 * no separate projection or VJP pass.  Bitwise equal to rfk_project_spd /
 * rfk_project_drift -> rfk_solve -> rfk_backward -> rfk_project_vjp.
 * mode: 0 none, 1 project_spd, 2 project_drift (metric as given), 3 both
 * (spd, then drift against the projected metric: the Joint parameterization). */
typedef struct {
    int32_t mode;
    double eps_min;    /* ProjectionConfig defaults: 1e-3 */
    double lambda_max; /* 1e3 */
    double tau;        /* 0.95 */
    double euclid_cap; /* 10 */
} rfk_projection;

/* rfk_solve on raw parameters; `projected` (5 planes in the fields' layout,
 * param_stride apart per grid; NULL to skip) receives the projected ones. */
RFK_API rfk_status rfk_solve_projected(rfk_context* ctx, rfk_memory mem, const rfk_fields* raw,
                                       const rfk_projection* proj, const rfk_solve_options* opt, double* t,
                                       int32_t* iterations, int32_t* converged, double* history,
                                       double* const projected[5]);

/* rfk_backward with gradients with respect to the raw parameters: `raw` holds
 * them (the VJP's linearisation point), `projected` the planes
 * rfk_solve_projected returned (identify and the adjoint run on them). */
RFK_API rfk_status rfk_backward_projected(rfk_context* ctx, rfk_memory mem, const rfk_fields* raw,
                                          const rfk_projection* proj, const double* const projected[5],
                                          const double* t, double tol, const double* loss_grad, double* lambda,
                                          double* d_g11, double* d_g12, double* d_g22, double* d_b1, double* d_b2,
                                          int32_t accumulate, int32_t* clamped, int64_t* bad_node);

/* ---- fp32 mode ---------------------------------------------
 * The same exact wavefront sweep with fp32 storage and arithmetic.  The
 * T-independent stencil terms are hoisted in fp64 and rounded (the fp64
 * degeneracy test is kept).  Results agree with the fp64 solve to ~1e-6
 * relative (target 1e-4); stencil choices may differ at near-ties.  No
 * fixed_values (solve_from_values) in this mode. */
typedef struct {
    int32_t batch;
    int32_t rows, cols;
    double h;
    const float* g11;
    const float* g12;
    const float* g22;
    const float* b1;
    const float* b2;
    int64_t param_stride;
    const uint8_t* src;
    int64_t src_stride;
} rfk_fields_f32;

RFK_API rfk_status rfk_solve_f32(rfk_context* ctx, rfk_memory mem, const rfk_fields_f32* f,
                                 const rfk_solve_options* opt, float* t, int32_t* iterations,
                                 int32_t* converged, double* history);

/* The backward of the fp32 mode: fp32 parameters, arrival field and loss
 * gradient in, fp32 gradient planes out.  The values are widened on the
 * device and go through rfk_backward's identify -> adjoint -> gradient path
 * in fp64 (the identification's tie tests and the adjoint's triangular solve
 * are where fp32 arithmetic would change stencil choices), then the gradients
 * are rounded to fp32.  Same shapes, accumulate and error behaviour as
 * rfk_backward; no lambda output. */
RFK_API rfk_status rfk_backward_f32(rfk_context* ctx, rfk_memory mem, const rfk_fields_f32* f,
                                    const float* t, double tol, const float* loss_grad, float* d_g11,
                                    float* d_g12, float* d_g22, float* d_b1, float* d_b2,
                                    int32_t accumulate, int32_t* clamped, int64_t* bad_node);

/* ---- fused objective (objective_and_grad, inversion.cpp:25-73) ---------
 * One call per optimizer iteration: every observation set's forward solve,
 * MSE loss with the flat unreached penalty, identify -> adjoint ->
 * parameter gradients, accumulated in observation order.  Host-memory
 * callers move the parameters in and the five gradient planes out once per
 * call instead of once per reference API call.  rfk_objective adds the TV
 * regularizers (below). */
typedef struct {
    int32_t count;            /* observation sets (ObservationSet, observations.hpp:10-14) */
    const uint8_t* sources;   /* [count][rows*cols] source masks   */
    const uint8_t* observed;  /* [count][rows*cols] observed masks */
    const double* values;     /* [count][rows*cols] observed values */
} rfk_observations;

typedef struct {
    double solve_tol;              /* InverseConfig::solve_tol (1e-6) */
    int32_t solve_max_iters;       /* InverseConfig::solve_max_iters (50) */
    double unreached_penalty_cap;  /* InverseConfig::unreached_penalty_cap (1e4) */
    int32_t exact_sum;             /* != 0: the reference's sequential loss sum, bit for bit */
} rfk_objective_options;

/* f: the shared parameter planes (batch 1; f->src is ignored, each
 * observation set brings its sources).  data_loss: Objective::data_loss;
 * unreached: Objective::unreached_observed; d_*: Objective::grad.  A forward
 * solve that does not converge returns RFK_ERR_NOT_CONVERGED; a stencil
 * inconsistency RFK_ERR_INCONSISTENT_FIXED_POINT. */
RFK_API rfk_status rfk_objective_and_grad(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                          const rfk_observations* obs, const rfk_objective_options* opt,
                                          double* data_loss, int32_t* unreached, double* d_g11,
                                          double* d_g12, double* d_g22, double* d_b1, double* d_b2);

/* ---- feasibility projection (feasibility.cpp:15-72) -------------------- */
RFK_API rfk_status rfk_project_spd(rfk_context* ctx, rfk_memory mem, int64_t n, double* g11,
                                   double* g12, double* g22, double eps_min, double lambda_max);
RFK_API rfk_status rfk_project_drift(rfk_context* ctx, rfk_memory mem, int64_t n, double* b1,
                                     double* b2, const double* g11, const double* g12,
                                     const double* g22, double tau, double euclid_cap);
RFK_API rfk_status rfk_drift_norm_sq(rfk_context* ctx, rfk_memory mem, int64_t n,
                                     const double* b1, const double* b2, const double* g11,
                                     const double* g12, const double* g22, double* out);

/* ---- projection VJP -------------------------------
 * Absent in the reference, which has no backward through the projection;
 * the paper's "differentiable projection layers".
 * Cotangent planes are updated in place: on entry they hold dL/d(projected
 * outputs), on return dL/d(inputs).  g12 is one channel feeding both
 * off-diagonal entries.  The inputs are the PRE-projection values. */

/* Through project_spd (feasibility.cpp:31-44): Daleckii-Krein on the
 * eigenvalue clamp; identity at pass-through nodes. */
RFK_API rfk_status rfk_project_spd_vjp(rfk_context* ctx, rfk_memory mem, int64_t n, const double* g11,
                                       const double* g12, const double* g22, double eps_min,
                                       double lambda_max, double* d_g11, double* d_g12, double* d_g22);
/* Through project_drift (feasibility.cpp:51-72) against a fixed metric:
 * d_b1/d_b2 in place; the metric's cotangent is ADDED to d_g11..d_g22 when
 * they are non-NULL (DriftOnly parameterization passes NULL). */
RFK_API rfk_status rfk_project_drift_vjp(rfk_context* ctx, rfk_memory mem, int64_t n, const double* b1,
                                         const double* b2, const double* g11, const double* g12,
                                         const double* g22, double tau, double euclid_cap, double* d_b1,
                                         double* d_b2, double* d_g11, double* d_g12, double* d_g22);
/* Through ParamView::project for the Joint parameterization
 * (inversion.cpp:276-279): project_spd, then project_drift against the
 * projected metric.  All five cotangent planes in place. */
RFK_API rfk_status rfk_project_vjp(rfk_context* ctx, rfk_memory mem, int64_t n, const double* g11,
                                   const double* g12, const double* g22, const double* b1, const double* b2,
                                   double eps_min, double lambda_max, double tau, double euclid_cap,
                                   double* d_g11, double* d_g12, double* d_g22, double* d_b1, double* d_b2);


/* ---- regularizers (feasibility.cpp:106-196) ------------------------------
 * Sums the reference takes sequentially (values, norms) are replayed in node
 * order when exact_sum != 0 (bit for bit, one device thread); otherwise a
 * tree reduction (last-bit differences). */
typedef enum { RFK_TV_FROBENIUS = 0, RFK_TV_LOG_EUCLIDEAN = 1, RFK_TV_DRIFT = 2 } rfk_tv_variant; /* TvVariant */

/* tv_value_grad (feasibility.cpp:137-182): nch = 1..3 planes of rows*cols;
 * grad[k] receives the TV gradient of channel k (overwritten). */
RFK_API rfk_status rfk_tv_value_grad(rfk_context* ctx, rfk_memory mem, int32_t rows, int32_t cols, int32_t nch,
                                     rfk_tv_variant variant, double eps_tv, const double* const* channels,
                                     double* const* grad, double* value, int32_t exact_sum);
/* tikhonov_value_grad (feasibility.cpp:184-196) */
RFK_API rfk_status rfk_tikhonov_value_grad(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nch,
                                           double weight, const double* const* channels, double* const* grad,
                                           double* value, int32_t exact_sum);

/* ---- optimizer steps (inversion.cpp:75-127) -------------------------------- */
/* clip_global_norm: scales the planes in place; *norm = the pre-clip norm. */
RFK_API rfk_status rfk_clip_global_norm(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nplanes,
                                        double* const* grads, double max_norm, double* norm, int32_t exact_sum);
/* adam_step: AdamState = caller-owned m, v planes (zero when *t == 0) and the
 * step count *t (incremented).  grads are clipped as a copy (the reference
 * takes them by value); steps[k] is channel k's learning rate. */
RFK_API rfk_status rfk_adam_step(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nplanes,
                                 double* const* params, double* const* m, double* const* v, int64_t* t,
                                 const double* const* grads, const double* steps, double beta1, double beta2,
                                 double adam_eps, double grad_clip_norm, int32_t exact_sum);
/* gd_step */
RFK_API rfk_status rfk_gd_step(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nplanes, double* const* params,
                               const double* const* grads, const double* steps, double grad_clip_norm,
                               int32_t exact_sum);
/* relative_error (inversion.cpp:129-138) */
RFK_API rfk_status rfk_relative_error(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nplanes,
                                      const double* const* est, const double* const* truth, double* out,
                                      int32_t exact_sum);

/* ---- the recovery loop (inversion.cpp:25-73, :327-385) ---------------------- */
typedef enum {
    RFK_PARAM_ISOTROPIC = 0,
    RFK_PARAM_DIAGONAL = 1,
    RFK_PARAM_FULL = 2,
    RFK_PARAM_DRIFT_ONLY = 3,
    RFK_PARAM_JOINT = 4
} rfk_parameterization; /* Parameterization (inversion.hpp:12) */
typedef enum { RFK_OPT_ADAM = 0, RFK_OPT_GD = 1 } rfk_optimizer; /* OptimizerKind */

/* InverseConfig (inversion.hpp:15-45) with its ProjectionConfig
 * (feasibility.hpp:9-21); rfk_inverse_config_default fills the reference's
 * defaults. */
typedef struct {
    rfk_parameterization param;
    rfk_optimizer optimizer;
    double step_g, step_b;
    double beta1, beta2, adam_eps;
    double grad_clip_norm;
    double lambda_g, lambda_b;
    rfk_tv_variant tv_variant;
    int32_t iters;
    double eps_min, lambda_max, tau, euclid_cap;
    double solve_tol;
    int32_t solve_max_iters;
    int32_t plateau_window;
    double plateau_factor;
    double unreached_penalty_cap;
    int32_t exact_sum; /* replay the reference's sequential sums (bit for bit) */
} rfk_inverse_config;
RFK_API void rfk_inverse_config_default(rfk_inverse_config* cfg);

/* Objective (inversion.hpp:49-55) */
typedef struct {
    double loss, data_loss, reg_loss;
    int32_t unreached_observed;
} rfk_objective_value;

/* objective_and_grad with the TV regularizers (inversion.cpp:25-73). */
RFK_API rfk_status rfk_objective(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                 const rfk_observations* obs, const rfk_inverse_config* cfg,
                                 rfk_objective_value* out, double* d_g11, double* d_g12, double* d_g22,
                                 double* d_b1, double* d_b2);

/* RecoveryResult (inversion.hpp:83-93).  Caller-owned outputs: the five
 * recovered planes, iso_g (optional, isotropic mode), loss_history[iters],
 * error_history[iters] (optional; filled only with a truth). */
typedef struct {
    double* g11;
    double* g12;
    double* g22;
    double* b1;
    double* b2;
    double* iso_g;
    double* loss_history;
    double* error_history;
    int32_t iterations;
    double final_error; /* -1 without a truth */
    int32_t unreached_observed_total;
} rfk_recovery;

/* recover (inversion.cpp:327-385): the whole projected first-order loop on
 * the device (parameters, moments and gradients stay resident; one scalar
 * read per iteration drives the plateau schedule).  init_metric[3] /
 * init_drift[2] default to g = I, b = 0 when null; truth_metric[3] /
 * truth_drift[2] enable the error history (the mode decides which is needed).
 * Planes are rows*cols, row-major; observation planes as rfk_observations. */
RFK_API rfk_status rfk_recover(rfk_context* ctx, rfk_memory mem, int32_t rows, int32_t cols, double h,
                               const rfk_observations* obs, const rfk_inverse_config* cfg,
                               const double* const* init_metric, const double* const* init_drift,
                               const double* const* truth_metric, const double* const* truth_drift,
                               rfk_recovery* out);

/* generate_observations (inversion.cpp:387-437): the count forward solves run
 * on the device; the sampling (mt19937_64 shuffle, normal noise) is the
 * reference's host code.  f->src is ignored; sources [count][rows*cols];
 * outputs observed/values [count][rows*cols]. */
RFK_API rfk_status rfk_generate_observations(rfk_context* ctx, rfk_memory mem, const rfk_fields* f, int32_t count,
                                             const uint8_t* sources, double density, double noise_level,
                                             uint64_t seed, uint8_t* observed, double* values);


/* multi_source_recover (inversion.cpp:439-503): the two-region isotropic
 * benchmark.  For each k in ks: k nested point sources, observations, an
 * isotropic recover; rows receive {k, total observations, final error}. */
typedef struct {
    int32_t k;
    int32_t total_observations;
    double error;
} rfk_multi_source_row;
RFK_API rfk_status rfk_multi_source_recover(rfk_context* ctx, const int32_t* ks, int32_t nks, double density,
                                            const rfk_inverse_config* cfg, int32_t grid_size, uint64_t seed,
                                            rfk_multi_source_row* rows);

#ifdef __cplusplus
}
#endif
#endif /* RFK_H */

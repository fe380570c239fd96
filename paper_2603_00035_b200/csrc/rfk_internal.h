// rfk_internal.h — argument blocks and launchers shared between the kernel
// translation units and the C-ABI layer (rfk_capi.cu).  Not installed.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rfk {

// The feasibility projection fused into the load stage (ParamView::project,
// inversion.cpp:255-279): mode 0 none, 1 project_spd, 2 project_drift (metric
// as given), 3 both (spd, then drift against the projected metric).
struct ProjCfg {
    int mode = 0;
    double eps_min = 1e-3, lambda_max = 1e3, tau = 0.95, cap = 10.0;
};

struct GridBarrierMem {
    unsigned* count;
    unsigned* generation;
};

struct JacobiArgs {
    int R, C;
    double h;
    const double *g11, *g12, *g22, *b1, *b2;
    const uint8_t* src;
    double* T;   // in/out
    double* T2;  // scratch, initialised like T
    unsigned long long* maxdelta;
    GridBarrierMem bar;
    double tol;
    int max_iters;
    int* iterations;
    int* converged;
    double* history;
};

// v2 sweep (rfk_sweep.cu)
struct SweepArgs {
    int R, C;
    double h;
    const double *g11, *g12, *g22, *b1, *b2;
    const uint8_t* src;
    void* T;                       // in: initial field, out: solution (double, or float in the fp32 mode)
    void* prev;                    // scratch plane: iteration-start values (same type)
    uint8_t* stamp;                // per-node pass stamp of the last change
    unsigned long long* mailbox;   // [4 passes][bands][positions][2] LL words
    size_t mailbox_stride;         // words per band
    size_t mailbox_pass_stride;    // words per pass
    unsigned long long* progress;  // [4 passes][bands] {pass epoch << 32 | positions written}
    int progress_stride;           // bands per pass slot
    int* queue;                    // [1] work-item ticket counter, zeroed by the launcher
    int* done3;                    // [max_iters] finished last-pass bands, zeroed
    int* decided;                  // [max_iters] iteration decided (max|dT| known), zeroed
    int* stop;                     // [1] 0, or 1 + the last iteration to keep, zeroed
    unsigned long long* maxdelta;  // [max_iters], zeroed by the launcher
    double tol;
    int max_iters;
    int order[4];
    int* iterations;
    int* converged;
    double* history;  // may be null
    unsigned epoch_base;
    unsigned long long* trace;  // optional [passes][bands][8] globaltimer/diagnostic record
    int trace_bands;
    const void* hoisted;    // [2][n][kRec] T-independent stencil terms, row- and column-major (launch_hoist; fp32 mode: rounded)
    unsigned long long* trace_probe;  // optional [8] per-segment cycle sums (diagnostics)
    unsigned* check;  // RFK_SWEEP_CHECKED builds: [8] protocol-check failure record, else null
};
constexpr int kSweepBandLines = 16;  // lines per band of the v2+ sweep kernel
constexpr int kTraceWords = 32;      // words per band record of the RFK_TRACE diagnostics
size_t sweep_mailbox_words(int R, int C, int band_lines);
bool sweep_checked();  // built with RFK_SWEEP_CHECKED (ring-tag protocol checks)
bool sweep_traced();   // built with RFK_SWEEP_TRACE_BUILD (the RFK_TRACE per-band trace)
size_t sweep_hoisted_doubles(int64_t n);
// proj (optional): project every node as it is read; proj_out (optional, 5
// planes) receives the projected parameters.
cudaError_t launch_hoist(const double* g11, const double* g12, const double* g22, const double* b1,
                         const double* b2, double h, int R, int C, double* out, cudaStream_t stream,
                         const ProjCfg* proj = nullptr, double* const* proj_out = nullptr, int copies = 2);
cudaError_t launch_init_stamps(uint8_t* stamp, const uint8_t* src, int64_t n, cudaStream_t stream);
cudaError_t launch_sweep(const SweepArgs& a, int band_lines, int max_ctas, cudaStream_t stream, int* used);
// Undo the speculative first pass of the iteration after the last one kept
// (T = iteration-start values at the nodes it wrote); no-op when there is none.
cudaError_t launch_sweep_rollback(const SweepArgs& a, cudaStream_t stream);

// fp32 mode (rfk_sweep_f32.cu)
cudaError_t launch_widen5_f32(int64_t n, const float* const f[5], double* out, cudaStream_t stream);
cudaError_t launch_narrow_records_f32(int64_t n_nodes, const double* in, float* out, cudaStream_t stream);
cudaError_t launch_init_field_f32(float* t, const uint8_t* src, int64_t n, unsigned long long* count,
                                  cudaStream_t stream);
cudaError_t launch_sweep_f32(const SweepArgs& a, int max_ctas, cudaStream_t stream, int* used);
cudaError_t launch_sweep_rollback_f32(const SweepArgs& a, cudaStream_t stream);

cudaError_t launch_jacobi(const JacobiArgs& a, cudaStream_t stream);
cudaError_t launch_init_field(double* t, double* t2, const uint8_t* src, const double* fixed_values,
                              int64_t n, unsigned long long* source_count, cudaStream_t stream);

// ---- candidates / records (rfk_backward.cu) --------------------------------
struct CandidateArgs {
    int R, C;
    double h;
    const double *g11, *g12, *g22, *b1, *b2;
    const double* T;
    int64_t n_nodes;
    const int32_t* nodes;
    int node_update;
    double* t0;
    int8_t *type, *stencil, *donor1, *donor2;
    double *lam1, *lam2;
    int8_t* found;
};
cudaError_t launch_best_candidate(const CandidateArgs& a, cudaStream_t stream);

struct TwoPointArgs {
    int64_t n;
    const double *t1, *t2, *m1x, *m1y, *m2x, *m2y, *g11, *g12, *g22, *b1, *b2;
    double *t0, *lam1, *lam2;
    int8_t* valid;
};
cudaError_t launch_two_point(const TwoPointArgs& a, cudaStream_t stream);

struct RecordPlanes {
    int8_t *type, *stencil, *donor1, *donor2;
    double* c[5];
};

struct IdentifyArgs {
    int R, C;
    double h;
    const double *g11, *g12, *g22, *b1, *b2;
    const uint8_t* src;
    const double* T;
    double tol;
    RecordPlanes rec;
    int* two_point_count;
    int* one_point_count;
    unsigned long long* bad_node;  // atomicMin target, init ~0
};
cudaError_t launch_identify(const IdentifyArgs& a, cudaStream_t stream);
// the same records from the row-major hoisted stencil records of the node's
// metric (launch_hoist with copies = 1): no per-lane E/det/Q divisions
cudaError_t launch_identify_hoisted(const IdentifyArgs& a, const double* hoisted, cudaStream_t stream);
#ifndef RFK_ID_HOISTED
#define RFK_ID_HOISTED 1  // rfk_backward identifies from hoisted records (0: identify_kernel)
#endif

struct JacobianArgs {
    int64_t n;
    const int8_t* type;
    const double* c[5];
    double *diag, *j0, *j1;
    int8_t* clamped;
};
cudaError_t launch_jacobian(const JacobianArgs& a, cudaStream_t stream);

// Adjoint in gather form over a topological (arrival-time) order.
struct AdjointArgs {
    int R, C;
    double h;
    const double* T;
    RecordPlanes rec;          // const in practice
    const double* loss_grad;
    double* lambda;
    // workspace
    double *diag, *j0, *j1;    // per node Jacobian entries
    unsigned long long* keys;  // n sort keys
    unsigned long long* keys_alt;
    int32_t* order;            // n sorted node ids
    int32_t* order_alt;
    int32_t* rank;             // n
    unsigned long long* ll;    // 2n: lambda hand-off words {epoch<<32 | 32 value bits}
    // per rank p (the node processed p-th): its dependents, sorted in the
    // reference's order, slot-major so a warp's loads coalesce
    int8_t* dep_n;             // n
    int32_t* dep_j;            // 8n: dependent node ids
    double* dep_c;             // 8n: their Jacobian coefficients toward the node
    double* self_g;            // n: dL/dT of the node
    double* self_d;            // n: its Jacobian diagonal
    unsigned epoch;
    unsigned long long* ticket;
    int* clamped;              // count
    int* nrec;                 // count of records (device)
    void* sort_temp;
    size_t sort_temp_bytes;
    // optional fused parameter gradients (null = skip)
    double *d_g11, *d_g12, *d_g22, *d_b1, *d_b2;
    int max_ctas;  // cap on the persistent dataflow grid (0 = every SM): concurrent batch slots
    // optional: the gradients leave through the projection's VJP, linearised
    // at the raw parameters (rfk_backward_projected)
    ProjCfg proj;
    const double* raw[5];
    // rfk_backward: the processing order is computed from T and the source
    // mask alone (a record exists exactly at the unfixed reached nodes when
    // identification succeeds), by launch_adjoint_order on a side stream
    // while identify runs; prepare then leaves keys/order alone.  `bad` (the
    // grid's identification failure word) stops the dataflow when
    // identification failed, whose order would not match the records.
    const uint8_t* order_src;  // non-null: split mode
    const unsigned long long* bad;
    int fused_prep;            // the dataflow searches the dependents (adjoint_fused_prep)
};
// The dataflow adjoint finds each node's dependents itself (large grids: the
// neighbour loads hide behind the wait for the dependents), or a gather pass
// lays them out by rank first (smaller grids, where the dataflow's chain is
// short and its grid may be capped by concurrent slots).  A/B: the fused
// search took the 4096^2 backward 12.73 -> 12.21 ms and cost the C5 batch of
// 1024^2 grids 3.5%.
constexpr int64_t kFusedPrepMinNodes = int64_t(1) << 22;  // 2048^2
inline bool adjoint_fused_prep(int64_t n) { return n >= kFusedPrepMinNodes; }
inline int adjoint_solve_kernels(int64_t n) { return adjoint_fused_prep(n) ? 1 : 2; }  // + the gradient pass
size_t adjoint_sort_temp_bytes(int64_t n);
cudaError_t launch_adjoint(const AdjointArgs& a, cudaStream_t stream);
// split mode (a.order_src set): the order on one stream, the rest on another
// (the caller orders the second after the first before gather prep)
cudaError_t launch_adjoint_order(const AdjointArgs& a, cudaStream_t stream);
cudaError_t launch_adjoint_prepare(const AdjointArgs& a, cudaStream_t stream);
cudaError_t launch_adjoint_solve(const AdjointArgs& a, cudaStream_t stream);

struct ParamGradArgs {
    int64_t n;
    int C;
    double h;
    RecordPlanes rec;
    const double* lambda;
    double *d_g11, *d_g12, *d_g22, *d_b1, *d_b2;
};
cudaError_t launch_param_gradients(const ParamGradArgs& a, cudaStream_t stream);

struct LossArgs {
    int64_t n;
    const double* T;
    const uint8_t* observed;
    const double* values;
    double* grad;
    double* loss;     // one value
    int* unreached;   // one value
    int exact;
    double* partial;  // workspace for tree sums (>= 1024 doubles)
};
cudaError_t launch_loss_grad(const LossArgs& a, cudaStream_t stream);

// objective_and_grad's flat penalty for unreached observed nodes, added to
// *acc in node order (inversion.cpp:42-47); one thread, rare path.
cudaError_t launch_unreached_penalty(int64_t n, const double* T, const uint8_t* observed, const double* values,
                                     double cap, double* acc, cudaStream_t stream);

// accumulate: acc[i] += add[i] for 5 planes (inversion.cpp:13-21 order)
cudaError_t launch_accumulate5(int64_t n, double* const acc[5], const double* const add[5],
                               cudaStream_t stream);

// ---- projections (rfk_project.cu) -----------------------------------------------
cudaError_t launch_project_spd(int64_t n, double* g11, double* g12, double* g22, double eps_min,
                               double lambda_max, cudaStream_t stream);
cudaError_t launch_project_drift(int64_t n, double* b1, double* b2, const double* g11,
                                 const double* g12, const double* g22, double tau,
                                 double euclid_cap, cudaStream_t stream);
cudaError_t launch_project_vjp(int mode, int64_t n, const double* g11, const double* g12, const double* g22,
                               const double* b1, const double* b2, double eps_min, double lambda_max, double tau,
                               double euclid_cap, double* dg11, double* dg12, double* dg22, double* db1,
                               double* db2, cudaStream_t stream);
cudaError_t launch_widen_f32(int64_t n, const float* in, double* out, cudaStream_t stream);
cudaError_t launch_narrow_f64(int64_t n, const double* in, float* out, cudaStream_t stream);
cudaError_t launch_drift_norm_sq(int64_t n, const double* b1, const double* b2, const double* g11,
                                 const double* g12, const double* g22, double* out,
                                 cudaStream_t stream);

// ---- recovery loop (rfk_inverse.cu) ----------------------------------------------
struct TvArgs {
    int R, C, nch;
    double w[3];
    double eps;
    const double* ch[3];
    double* grad[3];
    double* term;  // per-node root - eps (summed by launch_sum)
};
cudaError_t launch_tv(const TvArgs& a, cudaStream_t stream);
cudaError_t launch_log_spd(int64_t n, const double* g11, const double* g12, const double* g22, double* l11,
                           double* l12, double* l22, int* non_spd, cudaStream_t stream);
cudaError_t launch_dlog_chain(int64_t n, const double* g11, const double* g12, const double* g22,
                              const double* const lg[3], double* const out[3], cudaStream_t stream);

// Sum over `planes` planes of n elements, plane by plane, of
// mode 0: x; 1: x*x; 2: 0.5*scale*x*x; 3: (x - y)^2, starting from `init`.
// exact: sequential in index order (the reference's bits), else a tree.
struct SumArgs {
    int64_t n;
    int planes;
    const double* x[5];
    const double* y[5];
    double scale;
    double init;
};
cudaError_t launch_sum(const SumArgs& a, int mode, bool exact, double* partial /* >= 1024 */, double* out,
                       cudaStream_t stream);
cudaError_t launch_axpy(int64_t n, double alpha, const double* x, double* y, cudaStream_t stream);
cudaError_t launch_scale(int64_t n, double f, double* x, cudaStream_t stream);
cudaError_t launch_weighted_copy(int64_t n, double w, const double* src, double* out, cudaStream_t stream);
cudaError_t launch_add2(int64_t n, const double* a, const double* b, double* out, cudaStream_t stream);
cudaError_t launch_clamp(int64_t n, double* x, double lo, double hi, cudaStream_t stream);
cudaError_t launch_adam(int64_t n, double* p, double* m, double* v, const double* g, double step, double b1,
                        double b2, double bc1, double bc2, double eps, cudaStream_t stream);
cudaError_t launch_gd(int64_t n, double* p, const double* g, double step, cudaStream_t stream);

}  // namespace rfk

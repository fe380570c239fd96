// rfk_capi.cu — the C ABI (include/rfk.h): validation with the reference's
// error semantics, host<->device staging, workspace management and kernel
// orchestration.  All compute happens in the kernels of rfk_solve.cu,
// rfk_backward.cu and rfk_project.cu; there is no host fallback.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/rfk.h"
#include "rfk_internal.h"

#include "rfk_capi_internal.h"

namespace {

size_t plane_count(const rfk_fields* f, int64_t stride) {
    const size_t n = static_cast<size_t>(f->rows) * f->cols;
    return stride == 0 ? n : static_cast<size_t>(stride) * (f->batch - 1) + n;
}

// Streams for `slots` concurrent grids (slot 0 = ctx->stream), forked from
// the context stream; join_slots makes the context stream wait for them.
std::vector<cudaStream_t> fork_slots(rfk_context* ctx, int slots) {
    std::vector<cudaStream_t> ss{ctx->stream};
    if (slots <= 1) return ss;
    while (static_cast<int>(ctx->aux.size()) < slots - 1) {
        cudaStream_t s = nullptr;
        cuda_check(ctx, cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        ctx->aux.push_back(s);
    }
    while (static_cast<int>(ctx->events.size()) < slots) {
        cudaEvent_t e = nullptr;
        cuda_check(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        ctx->events.push_back(e);
    }
    cuda_check(ctx, cudaEventRecord(ctx->events[0], ctx->stream), "cudaEventRecord");
    for (int k = 1; k < slots; ++k) {
        cuda_check(ctx, cudaStreamWaitEvent(ctx->aux[k - 1], ctx->events[0], 0), "cudaStreamWaitEvent");
        ss.push_back(ctx->aux[k - 1]);
    }
    return ss;
}

void join_slots(rfk_context* ctx, const std::vector<cudaStream_t>& ss) {
    for (size_t k = 1; k < ss.size(); ++k) {
        cuda_check(ctx, cudaEventRecord(ctx->events[k], ss[k]), "cudaEventRecord");
        cuda_check(ctx, cudaStreamWaitEvent(ctx->stream, ctx->events[k], 0), "cudaStreamWaitEvent");
    }
}

// How many grids of a batch sweep concurrently.  One grid's wavefront keeps
// roughly 0.3 CTAs per band busy (measured: a 4096^2 solve on 74 of 148 SMs
// runs at 77% of its full-device speed, a 2048^2 solve on 50 SMs at 92%), so
// batches of smaller grids share the SMs.  RFK_SWEEP_SLOTS overrides.
int sweep_slots(int maxdim, int batch) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int bands = (maxdim + rfk::kSweepBandLines - 1) / rfk::kSweepBandLines;
    int g = static_cast<int>(static_cast<double>(sms) / (0.29 * bands) + 0.5);
    if (const char* e = std::getenv("RFK_SWEEP_SLOTS")) g = std::atoi(e);
    if (g > 8) g = 8;
    if (g > batch) g = batch;
    if (g < 1) g = 1;
    return g;
}

struct DevFields {
    const double *g11, *g12, *g22, *b1, *b2, *fixed;
    const uint8_t* src;
};

DevFields stage_fields(Stage& st, const rfk_fields* f) {
    const size_t np = plane_count(f, f->param_stride), ns = plane_count(f, f->src_stride);
    DevFields d;
    d.g11 = st.in("g11", f->g11, np);
    d.g12 = st.in("g12", f->g12, np);
    d.g22 = st.in("g22", f->g22, np);
    d.b1 = st.in("b1", f->b1, np);
    d.b2 = st.in("b2", f->b2, np);
    d.src = st.in("src", f->src, ns);
    d.fixed = st.in("fixed", f->fixed_values, ns);
    return d;
}

rfk_status run_solve(rfk_context* ctx, rfk_memory mem, const rfk_fields* f, const rfk_solve_options* opt,
                     double* t, int32_t* iterations, int32_t* converged, double* history, bool jacobi,
                     const rfk::ProjCfg* proj = nullptr, double* const* proj_out = nullptr) {
    return guarded(ctx, [&] {
        validate_fields(ctx, f);
        if (!t || !iterations || !converged) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null output");
        if (proj && jacobi) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "solve_jacobi: no fused projection");
        rfk_solve_options o{1e-6, 50, {0, 1, 2, 3}};
        if (opt) o = *opt;
        if (o.max_iters < 0) o.max_iters = 0;
        const int64_t n = static_cast<int64_t>(f->rows) * f->cols;
        const int B = f->batch;
        Stage st{ctx, mem, {}};
        const DevFields d = stage_fields(st, f);
        // the projected parameters (rfk_solve_projected), in the fields' layout
        double* pout[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
        if (proj && proj_out && proj_out[0]) {
            const size_t np = plane_count(f, f->param_stride);
            const char* nm[5] = {"proj:g11", "proj:g12", "proj:g22", "proj:b1", "proj:b2"};
            for (int k = 0; k < 5; ++k) pout[k] = st.out(nm[k], proj_out[k], np);
        }
        double* T = st.out("t", t, static_cast<size_t>(n) * B);
        int32_t* it_d = st.out("iters", iterations, B);
        int32_t* cv_d = st.out("conv", converged, B);
        double* hist = st.out("hist", history, static_cast<size_t>(B) * (o.max_iters > 0 ? o.max_iters : 1));
        auto* counts = tbuf<unsigned long long>(ctx, "srccount", B);
        cuda_check(ctx, cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * B, ctx->stream), "memset");
        const int mi = o.max_iters > 0 ? o.max_iters : 1;
        auto* maxdelta = tbuf<unsigned long long>(ctx, "maxdelta", static_cast<size_t>(mi) * B);
        cuda_check(ctx, cudaMemsetAsync(maxdelta, 0, sizeof(unsigned long long) * mi * B, ctx->stream),
                   "memset");
        auto* bar = tbuf<unsigned>(ctx, "barrier", 2, true);
        cuda_check(ctx, cudaMemsetAsync(bar, 0, sizeof(unsigned), ctx->stream), "memset");
        double* scratch = tbuf<double>(ctx, "prev", static_cast<size_t>(n));
        const int maxdim = f->rows > f->cols ? f->rows : f->cols;
        const bool v2 = !jacobi;  // the wavefront sweep (rfk_sweep.cu)
        const int slots = v2 ? sweep_slots(maxdim, B) : 1;
        int sms = 148;
        {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        }
        // T-independent stencil terms, shared by every grid when the metric is
        double* hoisted_shared = nullptr;
        if (v2 && f->param_stride == 0) {
            hoisted_shared = tbuf<double>(ctx, "hoisted", rfk::sweep_hoisted_doubles(n));
            launched(ctx, rfk::launch_hoist(d.g11, d.g12, d.g22, d.b1, d.b2, f->h, f->rows, f->cols, hoisted_shared,
                                            ctx->stream, proj, pout[0] ? pout : nullptr),
                     "hoist");
        }
        // epoch-tagged mailbox/progress words: clear every slot's set before the
        // 31-bit epoch wraps (never while a slot is in flight)
        if (v2 && ctx->sweep_epoch + static_cast<unsigned long long>(B) * (4ull * o.max_iters + 1) + 2 >= 0x7fffffffull) {
            for (auto& kv : ctx->bufs)
                if (kv.first.rfind("mailbox", 0) == 0 || kv.first.rfind("sweep:progress", 0) == 0)
                    cuda_check(ctx, cudaMemsetAsync(kv.second.p, 0, kv.second.bytes, ctx->stream), "memset");
            ctx->sweep_epoch = 1;
        }
        // per-slot workspaces, allocated (and zeroed) on the context stream
        // before the fork so every slot stream sees them initialised
        struct SlotWs {
            double* prev = nullptr;
            uint8_t* stamp = nullptr;
            unsigned long long* mailbox = nullptr;
            unsigned long long* progress = nullptr;
            int* sched = nullptr;
            double* hoisted = nullptr;
        };
        std::vector<SlotWs> ws(slots);
        const size_t mb_words = rfk::sweep_mailbox_words(f->rows, f->cols, rfk::kSweepBandLines);
        const int maxbands = (maxdim + rfk::kSweepBandLines - 1) / rfk::kSweepBandLines;
        if (v2)
            for (int k = 0; k < slots; ++k) {
                const std::string sfx = k ? "#" + std::to_string(k) : "";
                ws[k].prev = k ? tbuf<double>(ctx, "prev" + sfx, static_cast<size_t>(n)) : scratch;
                ws[k].stamp = tbuf<uint8_t>(ctx, "stamp" + sfx, static_cast<size_t>(n));
                // one mailbox set and one progress slot per pass, for two iterations
                // (passes overlap, and the next iteration's first pass runs
                // speculatively alongside the last pass of the current one)
                ws[k].mailbox = tbuf<unsigned long long>(ctx, "mailbox" + sfx, 8 * mb_words, true);
                ws[k].progress =
                    tbuf<unsigned long long>(ctx, "sweep:progress" + sfx, 8 * static_cast<size_t>(maxbands), true);
                ws[k].sched = tbuf<int>(ctx, "sweep:sched" + sfx, 2 + 2 * static_cast<size_t>(mi));
                ws[k].hoisted = hoisted_shared ? hoisted_shared
                                               : tbuf<double>(ctx, "hoisted" + sfx, rfk::sweep_hoisted_doubles(n));
            }
        // diagnostic builds: one protocol-check record per grid, zeroed before the fork
        unsigned* chkbuf = nullptr;
        if (v2 && rfk::sweep_checked()) {
            chkbuf = tbuf<unsigned>(ctx, "sweep:check", 8 * static_cast<size_t>(B));
            cuda_check(ctx, cudaMemsetAsync(chkbuf, 0, 8 * sizeof(unsigned) * B, ctx->stream), "memset");
        }
        const std::vector<cudaStream_t> ss = fork_slots(ctx, slots);
        for (int b = 0; b < B; ++b) {
            const int64_t po = f->param_stride * b, so = f->src_stride * b;
            double* Tb = T + n * b;
            const int slot = b % slots;
            const cudaStream_t stream = ss[slot];
            launched(ctx,
                     rfk::launch_init_field(Tb, jacobi ? scratch : nullptr, d.src + so,
                                            d.fixed ? d.fixed + so : nullptr, n, counts + b, stream),
                     "init_field");
            if (v2) {
                rfk::SweepArgs a{};
                a.R = f->rows;
                a.C = f->cols;
                a.h = f->h;
                a.g11 = d.g11 + po;
                a.g12 = d.g12 + po;
                a.g22 = d.g22 + po;
                a.b1 = d.b1 + po;
                a.b2 = d.b2 + po;
                a.src = d.src + so;
                a.T = Tb;
                const SlotWs& w = ws[slot];
                a.prev = w.prev;
                a.stamp = w.stamp;
                a.mailbox = w.mailbox;
                a.mailbox_stride = static_cast<size_t>(maxdim) * 2;
                a.mailbox_pass_stride = mb_words;
                a.progress = w.progress;
                a.progress_stride = maxbands;
                int* sched = w.sched;
                cuda_check(ctx, cudaMemsetAsync(sched, 0, sizeof(int) * (2 + 2 * mi), stream), "memset");
                a.queue = sched;
                a.stop = sched + 1;
                a.done3 = sched + 2;
                a.decided = sched + 2 + mi;
                a.maxdelta = maxdelta + static_cast<size_t>(mi) * b;
                
                a.tol = o.tol;
                a.max_iters = o.max_iters;
                for (int q = 0; q < 4; ++q) a.order[q] = o.sweep_order[q];
                a.iterations = it_d + b;
                a.converged = cv_d + b;
                a.history = hist ? hist + static_cast<size_t>(mi) * b : nullptr;
                a.epoch_base = static_cast<unsigned>(ctx->sweep_epoch);
                if (chkbuf) a.check = chkbuf + 8 * b;
                ctx->sweep_epoch += 4ull * static_cast<unsigned long long>(o.max_iters) + 1ull;
                if (rfk::sweep_traced() && std::getenv("RFK_TRACE") && b == 0) {
                    a.trace_bands = (maxdim + rfk::kSweepBandLines - 1) / rfk::kSweepBandLines;
                    const size_t tw = static_cast<size_t>(4) * o.max_iters * a.trace_bands * rfk::kTraceWords + 8;
                    a.trace = tbuf<unsigned long long>(ctx, "trace", tw);
                    cuda_check(ctx, cudaMemsetAsync(a.trace, 0, tw * 8, ctx->stream), "memset");
                    ctx->trace = a.trace;
                    ctx->trace_words = tw;
                    a.trace_probe = a.trace + tw - 8;  // last 8 words: per-segment cycle sums
                }
                // T-independent stencil terms: once per metric (shared params: hoisted before the fork)
                if (!hoisted_shared) {
                    double* pb[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
                    if (pout[0])
                        for (int k = 0; k < 5; ++k) pb[k] = pout[k] + po;
                    launched(ctx, rfk::launch_hoist(a.g11, a.g12, a.g22, a.b1, a.b2, f->h, f->rows, f->cols, w.hoisted,
                                                    stream, proj, pb[0] ? pb : nullptr),
                             "hoist");
                }
                a.hoisted = w.hoisted;
                launched(ctx, rfk::launch_init_stamps(a.stamp, a.src, n, stream), "init_stamps");
                int used = 0;
                int cap = slots > 1 ? sms / slots : 0;
                if (const char* e = std::getenv("RFK_SWEEP_CTAS")) cap = std::atoi(e);  // diagnostics
                launched(ctx, rfk::launch_sweep(a, rfk::kSweepBandLines, cap, stream, &used), "sweep");
                launched(ctx, rfk::launch_sweep_rollback(a, stream), "sweep_rollback");
            } else {
                rfk::JacobiArgs a{};
                a.R = f->rows;
                a.C = f->cols;
                a.h = f->h;
                a.g11 = d.g11 + po;
                a.g12 = d.g12 + po;
                a.g22 = d.g22 + po;
                a.b1 = d.b1 + po;
                a.b2 = d.b2 + po;
                a.src = d.src + so;
                a.T = Tb;
                a.T2 = scratch;
                a.maxdelta = maxdelta + static_cast<size_t>(mi) * b;
                a.bar = {bar, bar + 1};
                a.tol = o.tol;
                a.max_iters = o.max_iters;
                a.iterations = it_d + b;
                a.converged = cv_d + b;
                a.history = hist ? hist + static_cast<size_t>(mi) * b : nullptr;
                launched(ctx, rfk::launch_jacobi(a, ctx->stream), "jacobi");
            }
        }
        join_slots(ctx, ss);
        if (chkbuf) {  // diagnostic builds: the protocol checker's verdict
            std::vector<unsigned> all(8 * static_cast<size_t>(B));
            cuda_check(ctx, cudaMemcpy(all.data(), chkbuf, all.size() * sizeof(unsigned), cudaMemcpyDeviceToHost),
                       "D2H");
            for (int b = 0; b < B; ++b) {
                const unsigned* chk = all.data() + 8 * b;
                if (chk[0])
                fail(ctx, RFK_ERR_CUDA,
                     "sweep protocol check failed: mask " + std::to_string(chk[0]) + " first code " +
                         std::to_string(chk[1] - 1) + " band " + std::to_string(chk[2]) + " epoch " +
                         std::to_string(chk[3]) + " at " + std::to_string(chk[4]) + " tag " +
                         std::to_string(static_cast<int>(chk[5])));
            }
        }
        std::vector<unsigned long long> hc(B);
        cuda_check(ctx, cudaMemcpyAsync(hc.data(), counts, sizeof(unsigned long long) * B,
                                        cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H");
        st.finish();
        for (int b = 0; b < B; ++b)
            if (hc[b] == 0) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "SourceMask: needs at least one source node");
    });
}

RecordPlanes stage_records_out(Stage& st, const rfk_records* rec, size_t count, const std::string& tag) {
    RecordPlanes r{};
    r.type = st.out(tag + "type", rec->type, count);
    r.stencil = st.out(tag + "stencil", rec->stencil, count);
    r.donor1 = st.out(tag + "donor1", rec->donor1, count);
    r.donor2 = st.out(tag + "donor2", rec->donor2, count);
    for (int k = 0; k < 5; ++k) r.c[k] = st.out(tag + "c" + std::to_string(k), rec->c[k], count);
    return r;
}

RecordPlanes stage_records_in(Stage& st, const rfk_records* rec, size_t count) {
    RecordPlanes r{};
    r.type = const_cast<int8_t*>(st.in("rtype", rec->type, count));
    r.stencil = const_cast<int8_t*>(st.in("rstencil", rec->stencil, count));
    r.donor1 = const_cast<int8_t*>(st.in("rdonor1", rec->donor1, count));
    r.donor2 = const_cast<int8_t*>(st.in("rdonor2", rec->donor2, count));
    for (int k = 0; k < 5; ++k) r.c[k] = const_cast<double*>(st.in("rc" + std::to_string(k), rec->c[k], count));
    return r;
}

RecordPlanes ws_records(rfk_context* ctx, size_t n) {
    RecordPlanes r{};
    r.type = tbuf<int8_t>(ctx, "ws:type", n);
    r.stencil = tbuf<int8_t>(ctx, "ws:stencil", n);
    r.donor1 = tbuf<int8_t>(ctx, "ws:donor1", n);
    r.donor2 = tbuf<int8_t>(ctx, "ws:donor2", n);
    for (int k = 0; k < 5; ++k) r.c[k] = tbuf<double>(ctx, "ws:c" + std::to_string(k), n);
    return r;
}

RecordPlanes offset(const RecordPlanes& r, int64_t off) {
    RecordPlanes o = r;
    o.type += off;
    o.stencil += off;
    o.donor1 += off;
    o.donor2 += off;
    for (int k = 0; k < 5; ++k) o.c[k] += off;
    return o;
}

// identify one grid into `rec`; returns bad node (-1 if none) via device buffer
void identify_grid(rfk_context* ctx, const rfk_fields* f, const DevFields& d, int b, const double* T,
                   double tol, const RecordPlanes& rec, int* cnt2, int* cnt1, unsigned long long* bad,
                   cudaStream_t stream = nullptr, const double* hoisted = nullptr) {
    rfk::IdentifyArgs a{};
    const int64_t po = f->param_stride * b, so = f->src_stride * b;
    a.R = f->rows;
    a.C = f->cols;
    a.h = f->h;
    a.g11 = d.g11 + po;
    a.g12 = d.g12 + po;
    a.g22 = d.g22 + po;
    a.b1 = d.b1 + po;
    a.b2 = d.b2 + po;
    a.src = d.src + so;
    a.T = T;
    a.tol = tol;
    a.rec = rec;
    a.two_point_count = cnt2;
    a.one_point_count = cnt1;
    a.bad_node = bad;
    if (hoisted)  // the grid's metric hoisted row-major (launch_hoist copies = 1)
        launched(ctx, rfk::launch_identify_hoisted(a, hoisted, stream ? stream : ctx->stream), "identify");
    else
        launched(ctx, rfk::launch_identify(a, stream ? stream : ctx->stream), "identify");
}

std::string bad_node_message(const rfk_fields* f, int64_t node) {
    return "identify_stencils: node (" + std::to_string(node / f->cols) + "," +
           std::to_string(node % f->cols) + ") does not reproduce its arrival value";
}

// The adjoint's workspace (one set per concurrent slot; `sfx` names it).
// Allocated before any fork: the epoch-tagged LL words are zeroed on the
// context stream when first allocated.
rfk::AdjointArgs adjoint_workspace(rfk_context* ctx, int64_t n, const std::string& sfx = "") {
    rfk::AdjointArgs a{};
    a.diag = tbuf<double>(ctx, "adj:diag" + sfx, n);
    a.j0 = tbuf<double>(ctx, "adj:j0" + sfx, n);
    a.j1 = tbuf<double>(ctx, "adj:j1" + sfx, n);
    a.keys = tbuf<unsigned long long>(ctx, "adj:keys" + sfx, n);
    a.keys_alt = tbuf<unsigned long long>(ctx, "adj:keys2" + sfx, n);
    a.order = tbuf<int32_t>(ctx, "adj:order" + sfx, n);
    a.order_alt = tbuf<int32_t>(ctx, "adj:order2" + sfx, n);
    a.rank = tbuf<int32_t>(ctx, "adj:rank" + sfx, n);
    a.ll = tbuf<unsigned long long>(ctx, "adj:ll" + sfx, 2 * static_cast<size_t>(n), true);
    a.fused_prep = rfk::adjoint_fused_prep(n) ? 1 : 0;
    if (!a.fused_prep) {  // the gather pass's rank-ordered dependent lists (~100 B per node)
        a.dep_n = tbuf<int8_t>(ctx, "adj:depn" + sfx, static_cast<size_t>(n));
        a.dep_j = tbuf<int32_t>(ctx, "adj:depj" + sfx, 8 * static_cast<size_t>(n));
        a.dep_c = tbuf<double>(ctx, "adj:depc" + sfx, 8 * static_cast<size_t>(n));
        a.self_g = tbuf<double>(ctx, "adj:selfg" + sfx, static_cast<size_t>(n));
        a.self_d = tbuf<double>(ctx, "adj:selfd" + sfx, static_cast<size_t>(n));
    }
    a.ticket = tbuf<unsigned long long>(ctx, "adj:ticket" + sfx, 1);
    a.nrec = tbuf<int>(ctx, "adj:nrec" + sfx, 1);
    a.sort_temp_bytes = rfk::adjoint_sort_temp_bytes(n);
    a.sort_temp = buf(ctx, "adj:sorttmp" + sfx, a.sort_temp_bytes);
    return a;
}

// Split mode (rfk_backward): `order_stream` computes the processing order
// from T and the grid's source mask (`src`) while `identify` -- launched by
// the caller on `stream` between the two halves -- runs; `order_done` orders
// the dataflow after it.  The first half returns after the order launch.
struct AdjointSplit {
    cudaStream_t order_stream;
    cudaEvent_t fork, order_done;
    const uint8_t* src;
    const unsigned long long* bad;
};

void run_adjoint(rfk_context* ctx, int R, int C, double h, const double* T, const RecordPlanes& rec,
                 const double* loss_grad, double* lambda, int* clamped, double* const grads[5],
                 const rfk::AdjointArgs* ws = nullptr, cudaStream_t stream = nullptr, int max_ctas = 0,
                 const AdjointSplit* split = nullptr, int half = 0) {
    const int64_t n = static_cast<int64_t>(R) * C;
    rfk::AdjointArgs a = ws ? *ws : adjoint_workspace(ctx, n);
    a.R = R;
    a.C = C;
    a.h = h;
    a.T = T;
    a.rec = rec;
    a.loss_grad = loss_grad;
    a.lambda = lambda;
    a.epoch = (split && half == 0) ? ctx->adj_epoch : ++ctx->adj_epoch;  // (the order half uses no epoch)
    a.clamped = clamped;
    a.max_ctas = max_ctas;
    if (grads) {
        a.d_g11 = grads[0];
        a.d_g12 = grads[1];
        a.d_g22 = grads[2];
        a.d_b1 = grads[3];
        a.d_b2 = grads[4];
    }
    const cudaStream_t st = stream ? stream : ctx->stream;
    if (!split) {
        // prepare, CUB radix sort (histogram, exclusive sum, 8 onesweep passes),
        // rank, gather prep, dataflow, and the parameter gradients when requested
        launched(ctx, rfk::launch_adjoint(a, st), "adjoint", 12 + rfk::adjoint_solve_kernels(n) + (grads ? 1 : 0));
        return;
    }
    a.order_src = split->src;
    a.bad = split->bad;
    if (half == 0) {  // keys, sort, rank on the order stream, forked from `st`
        cuda_check(ctx, cudaEventRecord(split->fork, st), "cudaEventRecord");
        cuda_check(ctx, cudaStreamWaitEvent(split->order_stream, split->fork, 0), "cudaStreamWaitEvent");
        launched(ctx, rfk::launch_adjoint_order(a, split->order_stream), "adjoint order", 12);
        cuda_check(ctx, cudaEventRecord(split->order_done, split->order_stream), "cudaEventRecord");
        return;
    }
    launched(ctx, rfk::launch_adjoint_prepare(a, st), "adjoint prepare", 1);
    cuda_check(ctx, cudaStreamWaitEvent(st, split->order_done, 0), "cudaStreamWaitEvent");
    launched(ctx, rfk::launch_adjoint_solve(a, st), "adjoint", rfk::adjoint_solve_kernels(n) + (grads ? 1 : 0));
}

}  // namespace

// ============================================================================
extern "C" {

RFK_API int rfk_version(void) { return 1; }

RFK_API const char* rfk_status_string(rfk_status s) {
    switch (s) {
        case RFK_OK: return "ok";
        case RFK_ERR_DIMENSION_MISMATCH: return "dimension mismatch";
        case RFK_ERR_ZERO_DIMENSION: return "zero dimension";
        case RFK_ERR_INVALID_ARGUMENT: return "invalid argument";
        case RFK_ERR_INCONSISTENT_FIXED_POINT: return "inconsistent fixed point";
        case RFK_ERR_CUDA: return "cuda error";
        case RFK_ERR_NO_DEVICE: return "no cuda device";
        case RFK_ERR_ALLOC: return "device allocation failed";
        case RFK_ERR_NOT_CONVERGED: return "not converged";
        case RFK_ERR_NON_SPD_INPUT: return "non-SPD input";
        case RFK_ERR_DIVERGED_LOSS: return "diverged loss";
    }
    return "unknown";
}

RFK_API rfk_status rfk_create(rfk_context** out, int device) {
    if (!out) return RFK_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return RFK_ERR_NO_DEVICE;
    }
    if (device < 0 || device >= count) return RFK_ERR_INVALID_ARGUMENT;
    auto* ctx = new rfk_context();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return RFK_ERR_CUDA;
    }
    *out = ctx;
    return RFK_OK;
}

RFK_API void rfk_destroy(rfk_context* ctx) { delete ctx; }

RFK_API rfk_status rfk_set_stream(rfk_context* ctx, void* stream) {
    if (!ctx) return RFK_ERR_INVALID_ARGUMENT;
    const cudaStream_t next = static_cast<cudaStream_t>(stream);
    if (next == ctx->stream) return RFK_OK;
    // the context's workspaces were last used on the old stream: order the
    // new stream after it, so a rebound context never races with its own
    // earlier (asynchronous, device-memory) calls
    return guarded(ctx, [&] {
        if (!ctx->rebind_event)
            cuda_check(ctx, cudaEventCreateWithFlags(&ctx->rebind_event, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(ctx, cudaEventRecord(ctx->rebind_event, ctx->stream), "cudaEventRecord");
        cuda_check(ctx, cudaStreamWaitEvent(next, ctx->rebind_event, 0), "cudaStreamWaitEvent");
        ctx->stream = next;
    });
}

RFK_API const char* rfk_last_error(const rfk_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

RFK_API int64_t rfk_launch_count(const rfk_context* ctx) { return ctx ? ctx->launches : 0; }

RFK_API int64_t rfk_workspace_bytes(const rfk_context* ctx) {
    if (!ctx) return 0;
    int64_t total = 0;
    for (const auto& kv : ctx->bufs) total += static_cast<int64_t>(kv.second.bytes);
    return total;
}

RFK_API rfk_status rfk_release_workspace(rfk_context* ctx) {
    return guarded(ctx, [&] {
        cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
        for (auto& kv : ctx->bufs)
            if (kv.second.p) cuda_check(ctx, cudaFree(kv.second.p), "cudaFree");
        ctx->bufs.clear();
        ctx->trace = nullptr;
        ctx->trace_words = 0;
        // epoch-tagged flag buffers come back zeroed on the next allocation
        ctx->sweep_epoch = 1;
    });
}

// Diagnostics: copy the RFK_TRACE record of the last solve (rfk.h).
RFK_API int64_t rfk_debug_trace(rfk_context* ctx, unsigned long long* out, int64_t max_words) {
    if (!ctx || !ctx->trace) return 0;
    const int64_t n = static_cast<int64_t>(ctx->trace_words) < max_words ? static_cast<int64_t>(ctx->trace_words) : max_words;
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpy(out, ctx->trace, n * 8, cudaMemcpyDeviceToHost);
    return n;
}

RFK_API rfk_status rfk_solve(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                             const rfk_solve_options* opt, double* t, int32_t* iterations,
                             int32_t* converged, double* history) {
    return run_solve(ctx, mem, f, opt, t, iterations, converged, history, false);
}

static bool proj_cfg(rfk_context* ctx, const rfk_projection* p, rfk::ProjCfg& c) {
    if (!p) return false;
    if (p->mode < 0 || p->mode > 3) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "rfk_projection: mode must be 0..3");
    if ((p->mode & 1) && (!(p->eps_min > 0.0) || !(p->eps_min < p->lambda_max)))
        fail(ctx, RFK_ERR_INVALID_ARGUMENT, "ProjectionConfig: need 0 < eps_min < lambda_max");
    if ((p->mode & 2) && (!(p->tau > 0.0) || !(p->tau < 1.0)))
        fail(ctx, RFK_ERR_INVALID_ARGUMENT, "ProjectionConfig: need 0 < tau < 1");
    c.mode = p->mode;
    c.eps_min = p->eps_min;
    c.lambda_max = p->lambda_max;
    c.tau = p->tau;
    c.cap = p->euclid_cap;
    return c.mode != 0;
}

RFK_API rfk_status rfk_solve_projected(rfk_context* ctx, rfk_memory mem, const rfk_fields* raw,
                                       const rfk_projection* proj, const rfk_solve_options* opt, double* t,
                                       int32_t* iterations, int32_t* converged, double* history,
                                       double* const projected[5]) {
    rfk::ProjCfg c;
    const rfk_status st = guarded(ctx, [&] { proj_cfg(ctx, proj, c); });
    if (st != RFK_OK) return st;
    return run_solve(ctx, mem, raw, opt, t, iterations, converged, history, false, c.mode ? &c : nullptr,
                     projected);
}

RFK_API rfk_status rfk_solve_f32(rfk_context* ctx, rfk_memory mem, const rfk_fields_f32* f,
                                 const rfk_solve_options* opt, float* t, int32_t* iterations,
                                 int32_t* converged, double* history) {
    return guarded(ctx, [&] {
        if (!f) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null rfk_fields_f32");
        if (f->rows < 3 || f->cols < 3) fail(ctx, RFK_ERR_ZERO_DIMENSION, "GridSpec: rows and cols must be at least 3");
        if (!(f->h > 0.0)) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "GridSpec: h must be positive");
        if (f->batch < 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "rfk_fields: batch must be >= 1");
        if (!f->g11 || !f->g12 || !f->g22 || !f->b1 || !f->b2 || !f->src)
            fail(ctx, RFK_ERR_DIMENSION_MISMATCH, "solve: field dimensions disagree with grid spec");
        if (!t || !iterations || !converged) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null output");
        rfk_solve_options o{1e-6, 50, {0, 1, 2, 3}};
        if (opt) o = *opt;
        if (o.max_iters < 0) o.max_iters = 0;
        const int64_t n = static_cast<int64_t>(f->rows) * f->cols;
        const int B = f->batch;
        const size_t np = f->param_stride == 0 ? n : static_cast<size_t>(f->param_stride) * (B - 1) + n;
        const size_t ns = f->src_stride == 0 ? n : static_cast<size_t>(f->src_stride) * (B - 1) + n;
        Stage st{ctx, mem, {}};
        const float* P[5] = {st.in("f32g11", f->g11, np), st.in("f32g12", f->g12, np), st.in("f32g22", f->g22, np),
                             st.in("f32b1", f->b1, np), st.in("f32b2", f->b2, np)};
        const uint8_t* src = st.in("f32src", f->src, ns);
        float* T = st.out("f32t", t, static_cast<size_t>(n) * B);
        int32_t* it_d = st.out("iters", iterations, B);
        int32_t* cv_d = st.out("conv", converged, B);
        const int mi = o.max_iters > 0 ? o.max_iters : 1;
        double* hist = st.out("hist", history, static_cast<size_t>(B) * mi);
        auto* counts = tbuf<unsigned long long>(ctx, "srccount", B);
        cuda_check(ctx, cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * B, ctx->stream), "memset");
        auto* maxdelta = tbuf<unsigned long long>(ctx, "maxdelta", static_cast<size_t>(mi) * B);
        cuda_check(ctx, cudaMemsetAsync(maxdelta, 0, sizeof(unsigned long long) * mi * B, ctx->stream), "memset");
        const int maxdim = f->rows > f->cols ? f->rows : f->cols;
        const int slots = sweep_slots(maxdim, B);
        int sms = 148;
        {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        }
        // hoisted records: fp64 hoist of the widened fields, rounded to fp32
        // (fp64 scratch per slot, so grids with their own metrics hoist concurrently)
        auto hoist_f32 = [&](int b, float* out, cudaStream_t s, int slot) {
            const std::string sfx = "#" + std::to_string(slot);
            double* wide = tbuf<double>(ctx, "f32:wide" + sfx, 5 * static_cast<size_t>(n));
            double* rec64 = tbuf<double>(ctx, "f32:rec64" + sfx, rfk::sweep_hoisted_doubles(n));
            const int64_t po = f->param_stride * b;
            const float* fb[5] = {P[0] + po, P[1] + po, P[2] + po, P[3] + po, P[4] + po};
            launched(ctx, rfk::launch_widen5_f32(n, fb, wide, s), "widen");
            launched(ctx, rfk::launch_hoist(wide, wide + n, wide + 2 * n, wide + 3 * n, wide + 4 * n, f->h, f->rows,
                                            f->cols, rec64, s),
                     "hoist");
            launched(ctx, rfk::launch_narrow_records_f32(n, rec64, out, s), "narrow");
        };
        const size_t mb_words = rfk::sweep_mailbox_words(f->rows, f->cols, rfk::kSweepBandLines);
        const int maxbands = (maxdim + rfk::kSweepBandLines - 1) / rfk::kSweepBandLines;
        struct SlotWs {
            float* prev;
            uint8_t* stamp;
            unsigned long long* mailbox;
            unsigned long long* progress;
            int* sched;
            float* hoisted;
        };
        std::vector<SlotWs> ws(slots);
        const size_t rec_floats = rfk::sweep_hoisted_doubles(n);  // element count (kRec per record)
        float* hoisted_shared = nullptr;
        if (f->param_stride == 0) {
            hoisted_shared = tbuf<float>(ctx, "f32:hoisted", rec_floats);
            hoist_f32(0, hoisted_shared, ctx->stream, 0);
        }
        for (int k = 0; k < slots; ++k) {
            const std::string sfx = "#f32." + std::to_string(k);
            ws[k].prev = tbuf<float>(ctx, "prev" + sfx, static_cast<size_t>(n));
            ws[k].stamp = tbuf<uint8_t>(ctx, "stamp" + sfx, static_cast<size_t>(n));
            ws[k].mailbox = tbuf<unsigned long long>(ctx, "mailbox" + sfx, 8 * mb_words, true);
            ws[k].progress =
                tbuf<unsigned long long>(ctx, "sweep:progress" + sfx, 8 * static_cast<size_t>(maxbands), true);
            ws[k].sched = tbuf<int>(ctx, "sweep:sched" + sfx, 2 + 2 * static_cast<size_t>(mi));
            ws[k].hoisted = hoisted_shared ? hoisted_shared : tbuf<float>(ctx, "f32:hoisted" + sfx, rec_floats);
        }
        if (ctx->sweep_epoch + static_cast<unsigned long long>(B) * (4ull * o.max_iters + 1) + 2 >= 0x7fffffffull) {
            for (auto& kv : ctx->bufs)
                if (kv.first.rfind("mailbox", 0) == 0 || kv.first.rfind("sweep:progress", 0) == 0)
                    cuda_check(ctx, cudaMemsetAsync(kv.second.p, 0, kv.second.bytes, ctx->stream), "memset");
            ctx->sweep_epoch = 1;
        }
        if (!hoisted_shared)  // allocate the per-slot fp64 scratch before the fork
            for (int k = 0; k < slots; ++k) {
                tbuf<double>(ctx, "f32:wide#" + std::to_string(k), 5 * static_cast<size_t>(n));
                tbuf<double>(ctx, "f32:rec64#" + std::to_string(k), rfk::sweep_hoisted_doubles(n));
            }
        const std::vector<cudaStream_t> ss = fork_slots(ctx, slots);
        for (int b = 0; b < B; ++b) {
            const int slot = b % slots;
            const cudaStream_t stream = ss[slot];
            const SlotWs& w = ws[slot];
            const int64_t so = f->src_stride * b;
            float* Tb = T + n * b;
            if (!hoisted_shared) hoist_f32(b, w.hoisted, stream, slot);
            launched(ctx, rfk::launch_init_field_f32(Tb, src + so, n, counts + b, stream), "init_field");
            rfk::SweepArgs a{};
            a.R = f->rows;
            a.C = f->cols;
            a.h = f->h;
            a.src = src + so;
            a.T = Tb;
            a.prev = w.prev;
            a.stamp = w.stamp;
            a.mailbox = w.mailbox;
            a.mailbox_stride = static_cast<size_t>(maxdim) * 2;
            a.mailbox_pass_stride = mb_words;
            a.progress = w.progress;
            a.progress_stride = maxbands;
            cuda_check(ctx, cudaMemsetAsync(w.sched, 0, sizeof(int) * (2 + 2 * mi), stream), "memset");
            a.queue = w.sched;
            a.stop = w.sched + 1;
            a.done3 = w.sched + 2;
            a.decided = w.sched + 2 + mi;
            a.maxdelta = maxdelta + static_cast<size_t>(mi) * b;
            a.tol = o.tol;
            a.max_iters = o.max_iters;
            for (int q = 0; q < 4; ++q) a.order[q] = o.sweep_order[q];
            a.iterations = it_d + b;
            a.converged = cv_d + b;
            a.history = hist ? hist + static_cast<size_t>(mi) * b : nullptr;
            a.epoch_base = static_cast<unsigned>(ctx->sweep_epoch);
            ctx->sweep_epoch += 4ull * static_cast<unsigned long long>(o.max_iters) + 1ull;
            a.hoisted = w.hoisted;
            launched(ctx, rfk::launch_init_stamps(a.stamp, a.src, n, stream), "init_stamps");
            int used = 0;
            launched(ctx, rfk::launch_sweep_f32(a, slots > 1 ? sms / slots : 0, stream, &used), "sweep_f32");
            launched(ctx, rfk::launch_sweep_rollback_f32(a, stream), "sweep_rollback");
        }
        join_slots(ctx, ss);
        std::vector<unsigned long long> hc(B);
        cuda_check(ctx, cudaMemcpyAsync(hc.data(), counts, sizeof(unsigned long long) * B, cudaMemcpyDeviceToHost,
                                        ctx->stream),
                   "D2H");
        st.finish();
        for (int b = 0; b < B; ++b)
            if (hc[b] == 0) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "SourceMask: needs at least one source node");
    });
}

RFK_API rfk_status rfk_solve_jacobi(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                    const rfk_solve_options* opt, double* t, int32_t* iterations,
                                    int32_t* converged, double* history) {
    return run_solve(ctx, mem, f, opt, t, iterations, converged, history, true);
}

RFK_API rfk_status rfk_best_candidate(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                      const double* t, int64_t n_nodes, const int32_t* nodes,
                                      int32_t node_update, double* t0, int8_t* type, int8_t* stencil,
                                      int8_t* donor1, int8_t* donor2, double* lam1, double* lam2,
                                      int8_t* found) {
    return guarded(ctx, [&] {
        if (!f || f->rows < 1 || f->cols < 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "bad grid");
        if (n_nodes <= 0) return;
        const size_t n = static_cast<size_t>(f->rows) * f->cols;
        Stage st{ctx, mem, {}};
        rfk::CandidateArgs a{};
        a.R = f->rows;
        a.C = f->cols;
        a.h = f->h;
        a.g11 = st.in("g11", f->g11, n);
        a.g12 = st.in("g12", f->g12, n);
        a.g22 = st.in("g22", f->g22, n);
        a.b1 = st.in("b1", f->b1, n);
        a.b2 = st.in("b2", f->b2, n);
        a.T = st.in("t", t, n);
        a.n_nodes = n_nodes;
        a.nodes = st.in("nodes", nodes, n_nodes);
        a.node_update = node_update;
        a.t0 = st.out("t0", t0, n_nodes);
        a.type = st.out("type", type, n_nodes);
        a.stencil = st.out("stencil", stencil, n_nodes);
        a.donor1 = st.out("donor1", donor1, n_nodes);
        a.donor2 = st.out("donor2", donor2, n_nodes);
        a.lam1 = st.out("lam1", lam1, n_nodes);
        a.lam2 = st.out("lam2", lam2, n_nodes);
        a.found = st.out("found", found, n_nodes);
        launched(ctx, rfk::launch_best_candidate(a, ctx->stream), "best_candidate");
        st.finish();
    });
}

RFK_API rfk_status rfk_two_point_update(rfk_context* ctx, rfk_memory mem, int64_t n, const double* t1,
                                        const double* t2, const double* m1x, const double* m1y,
                                        const double* m2x, const double* m2y, const double* g11,
                                        const double* g12, const double* g22, const double* b1,
                                        const double* b2, double* t0, double* lam1, double* lam2,
                                        int8_t* valid) {
    return guarded(ctx, [&] {
        if (n <= 0) return;
        Stage st{ctx, mem, {}};
        rfk::TwoPointArgs a{};
        a.n = n;
        a.t1 = st.in("t1", t1, n);
        a.t2 = st.in("t2", t2, n);
        a.m1x = st.in("m1x", m1x, n);
        a.m1y = st.in("m1y", m1y, n);
        a.m2x = st.in("m2x", m2x, n);
        a.m2y = st.in("m2y", m2y, n);
        a.g11 = st.in("g11", g11, n);
        a.g12 = st.in("g12", g12, n);
        a.g22 = st.in("g22", g22, n);
        a.b1 = st.in("b1", b1, n);
        a.b2 = st.in("b2", b2, n);
        a.t0 = st.out("t0", t0, n);
        a.lam1 = st.out("lam1", lam1, n);
        a.lam2 = st.out("lam2", lam2, n);
        a.valid = st.out("valid", valid, n);
        launched(ctx, rfk::launch_two_point(a, ctx->stream), "two_point");
        st.finish();
    });
}

RFK_API rfk_status rfk_identify(rfk_context* ctx, rfk_memory mem, const rfk_fields* f, const double* t,
                                double tol, const rfk_records* rec, int32_t* two_point_count,
                                int32_t* one_point_count, int64_t* bad_node) {
    return guarded(ctx, [&] {
        validate_fields(ctx, f);
        if (!rec || !rec->type || !t) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        const int64_t n = static_cast<int64_t>(f->rows) * f->cols;
        const int B = f->batch;
        Stage st{ctx, mem, {}};
        const DevFields d = stage_fields(st, f);
        const double* T = st.in("t", t, static_cast<size_t>(n) * B);
        const RecordPlanes r = stage_records_out(st, rec, static_cast<size_t>(n) * B, "rec");
        auto* cnt = tbuf<int>(ctx, "idcnt", 2 * static_cast<size_t>(B));
        auto* bad = tbuf<unsigned long long>(ctx, "idbad", B);
        cuda_check(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * B, ctx->stream), "memset");
        cuda_check(ctx, cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long) * B, ctx->stream), "memset");
        for (int b = 0; b < B; ++b)
            identify_grid(ctx, f, d, b, T + n * b, tol, offset(r, n * b), cnt + 2 * b, cnt + 2 * b + 1,
                          bad + b);
        std::vector<int> hc(2 * B);
        std::vector<unsigned long long> hb(B);
        cuda_check(ctx, cudaMemcpyAsync(hc.data(), cnt, sizeof(int) * 2 * B, cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H");
        cuda_check(ctx, cudaMemcpyAsync(hb.data(), bad, sizeof(unsigned long long) * B, cudaMemcpyDeviceToHost,
                                        ctx->stream),
                   "D2H");
        st.finish();
        int64_t first_bad = -1;
        for (int b = 0; b < B; ++b) {
            const int64_t bn = hb[b] == ~0ull ? -1 : static_cast<int64_t>(hb[b]);
            if (two_point_count) {
                if (mem == RFK_MEM_HOST) {
                    two_point_count[b] = hc[2 * b];
                    one_point_count[b] = hc[2 * b + 1];
                    bad_node[b] = bn;
                }
            }
            if (bn >= 0 && first_bad < 0) first_bad = bn;
        }
        if (mem == RFK_MEM_DEVICE && two_point_count) {
            std::vector<int32_t> c2(B), c1(B);
            std::vector<int64_t> bb(B);
            for (int b = 0; b < B; ++b) {
                c2[b] = hc[2 * b];
                c1[b] = hc[2 * b + 1];
                bb[b] = hb[b] == ~0ull ? -1 : static_cast<int64_t>(hb[b]);
            }
            cuda_check(ctx, cudaMemcpy(two_point_count, c2.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice), "H2D");
            cuda_check(ctx, cudaMemcpy(one_point_count, c1.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice), "H2D");
            if (bad_node)
                cuda_check(ctx, cudaMemcpy(bad_node, bb.data(), sizeof(int64_t) * B, cudaMemcpyHostToDevice), "H2D");
        }
        if (first_bad >= 0) fail(ctx, RFK_ERR_INCONSISTENT_FIXED_POINT, bad_node_message(f, first_bad));
    });
}

RFK_API rfk_status rfk_jacobian_entries(rfk_context* ctx, rfk_memory mem, int64_t n, const int8_t* type,
                                        const double* c0, const double* c1, const double* c2,
                                        const double* c3, const double* c4, double* diag, double* j0,
                                        double* j1, int8_t* clamped) {
    return guarded(ctx, [&] {
        if (n <= 0) return;
        Stage st{ctx, mem, {}};
        rfk::JacobianArgs a{};
        a.n = n;
        a.type = st.in("type", type, n);
        a.c[0] = st.in("c0", c0, n);
        a.c[1] = st.in("c1", c1, n);
        a.c[2] = st.in("c2", c2, n);
        a.c[3] = st.in("c3", c3, n);
        a.c[4] = st.in("c4", c4, n);
        a.diag = st.out("diag", diag, n);
        a.j0 = st.out("j0", j0, n);
        a.j1 = st.out("j1", j1, n);
        a.clamped = st.out("clamped", clamped, n);
        launched(ctx, rfk::launch_jacobian(a, ctx->stream), "jacobian");
        st.finish();
    });
}

RFK_API rfk_status rfk_solve_adjoint(rfk_context* ctx, rfk_memory mem, int32_t batch, int32_t rows,
                                     int32_t cols, const double* t, const rfk_records* rec,
                                     const double* loss_grad, double* lambda, int32_t* clamped) {
    return guarded(ctx, [&] {
        if (batch < 1 || rows < 1 || cols < 1 || !rec) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "bad arguments");
        const int64_t n = static_cast<int64_t>(rows) * cols;
        Stage st{ctx, mem, {}};
        const double* T = st.in("t", t, n * batch);
        const RecordPlanes r = stage_records_in(st, rec, n * batch);
        const double* g = st.in("lg", loss_grad, n * batch);
        double* lam = st.out("lambda", lambda, n * batch);
        int* cl = st.out("clamped", clamped, batch);
        for (int b = 0; b < batch; ++b)
            run_adjoint(ctx, rows, cols, 1.0, T + n * b, offset(r, n * b), g + n * b, lam + n * b, cl + b,
                        nullptr);
        st.finish();
    });
}

RFK_API rfk_status rfk_param_gradients(rfk_context* ctx, rfk_memory mem, int32_t batch, int32_t rows,
                                       int32_t cols, double h, const rfk_records* rec, const double* lambda,
                                       double* d_g11, double* d_g12, double* d_g22, double* d_b1,
                                       double* d_b2) {
    return guarded(ctx, [&] {
        if (batch < 1 || rows < 1 || cols < 1 || !rec) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "bad arguments");
        const int64_t n = static_cast<int64_t>(rows) * cols * batch;
        Stage st{ctx, mem, {}};
        rfk::ParamGradArgs a{};
        a.n = n;
        a.C = cols;
        a.h = h;
        a.rec = stage_records_in(st, rec, n);
        a.lambda = st.in("lambda", lambda, n);
        a.d_g11 = st.out("dg11", d_g11, n);
        a.d_g12 = st.out("dg12", d_g12, n);
        a.d_g22 = st.out("dg22", d_g22, n);
        a.d_b1 = st.out("db1", d_b1, n);
        a.d_b2 = st.out("db2", d_b2, n);
        launched(ctx, rfk::launch_param_gradients(a, ctx->stream), "param_gradients");
        st.finish();
    });
}

RFK_API rfk_status rfk_loss_grad_mse(rfk_context* ctx, rfk_memory mem, int32_t batch, int64_t n,
                                     const double* t, const uint8_t* observed, const double* values,
                                     double* grad, double* loss, int32_t* unreached, int32_t exact_sum) {
    return guarded(ctx, [&] {
        if (batch < 1 || n < 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "bad arguments");
        Stage st{ctx, mem, {}};
        const double* T = st.in("t", t, n * batch);
        const uint8_t* obs = st.in("obs", observed, n * batch);
        const double* val = st.in("val", values, n * batch);
        double* g = st.out("grad", grad, n * batch);
        double* l = st.out("loss", loss, batch);
        int* u = st.out("unreached", unreached, batch);
        double* partial = tbuf<double>(ctx, "losspart", 1024);
        for (int b = 0; b < batch; ++b) {
            rfk::LossArgs a{n, T + n * b, obs + n * b, val + n * b, g + n * b, l + b, u + b, exact_sum, partial};
            launched(ctx, rfk::launch_loss_grad(a, ctx->stream), "loss_grad", 2);
        }
        st.finish();
    });
}

static rfk_status run_backward(rfk_context* ctx, rfk_memory mem, const rfk_fields* f, const double* t, double tol,
                               const double* loss_grad, double* lambda, double* d_g11, double* d_g12,
                               double* d_g22, double* d_b1, double* d_b2, int32_t accumulate, int32_t* clamped,
                               int64_t* bad_node, const rfk::ProjCfg* proj = nullptr,
                               const rfk_fields* raw = nullptr, bool hoisted_ready = false) {
    return guarded(ctx, [&] {
        validate_fields(ctx, f);
        const int64_t n = static_cast<int64_t>(f->rows) * f->cols;
        const int B = f->batch;
        const bool acc = accumulate && f->param_stride == 0;
        const size_t gcount = acc ? static_cast<size_t>(n) : static_cast<size_t>(n) * B;
        Stage st{ctx, mem, {}};
        const DevFields d = stage_fields(st, f);
        // rfk_backward_projected: the raw parameters, the VJP's linearisation point
        const double* rawp[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
        if (proj) {
            const size_t np = plane_count(raw, raw->param_stride);
            rawp[0] = st.in("raw:g11", raw->g11, np);
            rawp[1] = st.in("raw:g12", raw->g12, np);
            rawp[2] = st.in("raw:g22", raw->g22, np);
            rawp[3] = st.in("raw:b1", raw->b1, np);
            rawp[4] = st.in("raw:b2", raw->b2, np);
        }
        const double* T = st.in("t", t, static_cast<size_t>(n) * B);
        const double* lg = st.in("lg", loss_grad, static_cast<size_t>(n) * B);
        double* lam = lambda ? st.out("lambda", lambda, static_cast<size_t>(n) * B)
                             : tbuf<double>(ctx, "bw:lambda", static_cast<size_t>(n));
        double* out[5] = {st.out("dg11", d_g11, gcount), st.out("dg12", d_g12, gcount),
                          st.out("dg22", d_g22, gcount), st.out("db1", d_b1, gcount),
                          st.out("db2", d_b2, gcount)};
        int* cl = clamped ? st.out("clamped", clamped, B) : tbuf<int>(ctx, "bw:clamped", B);
        auto* bad = tbuf<unsigned long long>(ctx, "idbad", B);
        cuda_check(ctx, cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long) * B, ctx->stream), "memset");
        if (acc)
            for (int k = 0; k < 5; ++k)
                cuda_check(ctx, cudaMemsetAsync(out[k], 0, sizeof(double) * n, ctx->stream), "memset");
        // Grids of the batch run concurrently in slots (as the sweep does);
        // each slot has its own records, adjoint workspace and gradient scratch.
        // With accumulate, the sums into `out` run on one extra stream in grid
        // order (inversion.cpp:13-21), each after its grid and before the slot
        // reuses its scratch.
        const int slots = sweep_slots(f->rows > f->cols ? f->rows : f->cols, B);
        struct BwWs {
            RecordPlanes rec;
            rfk::AdjointArgs adj;
            int* cnt;
            double* lam;
            double* tmp[5];
            double* hoisted;
        };
        std::vector<BwWs> ws(slots);
        for (int k = 0; k < slots; ++k) {
            const std::string sfx = k ? "#" + std::to_string(k) : "";
            if (k == 0) {
                ws[k].rec = ws_records(ctx, static_cast<size_t>(n));
            } else {
                RecordPlanes r{};
                r.type = tbuf<int8_t>(ctx, "ws:type" + sfx, n);
                r.stencil = tbuf<int8_t>(ctx, "ws:stencil" + sfx, n);
                r.donor1 = tbuf<int8_t>(ctx, "ws:donor1" + sfx, n);
                r.donor2 = tbuf<int8_t>(ctx, "ws:donor2" + sfx, n);
                for (int c = 0; c < 5; ++c) r.c[c] = tbuf<double>(ctx, "ws:c" + std::to_string(c) + sfx, n);
                ws[k].rec = r;
            }
            ws[k].adj = adjoint_workspace(ctx, n, sfx);
            // identify from hoisted stencil records: the sweep's workspace
            // (a solve on this context stream has finished with it)
            ws[k].hoisted = (f->param_stride == 0 && k > 0)
                                ? nullptr
                                : tbuf<double>(ctx, "hoisted" + sfx, rfk::sweep_hoisted_doubles(n));
            ws[k].cnt = tbuf<int>(ctx, "idcnt" + sfx, 2);
            ws[k].lam = lambda ? nullptr : tbuf<double>(ctx, "bw:lambda" + sfx, static_cast<size_t>(n));
            for (int c = 0; c < 5; ++c)
                ws[k].tmp[c] = acc ? tbuf<double>(ctx, "bw:tmp" + std::to_string(c) + sfx, static_cast<size_t>(n))
                                   : nullptr;
        }
        int sms = 148;
        {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        }
        const bool acc_stream = acc && slots > 1;
        // streams: [0, slots) the grids, [slots] the accumulation (if any), then
        // one order stream per slot (the adjoint's sort runs beside identify)
        const int side0 = slots + (acc_stream ? 1 : 0);
        // one metric for every grid: hoisted once, before the fork (unless the
        // caller's solve on this context stream just hoisted the same metric)
        if (RFK_ID_HOISTED && f->param_stride == 0 && !hoisted_ready)
            launched(ctx,
                     rfk::launch_hoist(d.g11, d.g12, d.g22, d.b1, d.b2, f->h, f->rows, f->cols, ws[0].hoisted,
                                       ctx->stream, nullptr, nullptr, 1),
                     "hoist");
        const std::vector<cudaStream_t> ss = fork_slots(ctx, side0 + slots);
        const cudaStream_t astream = acc_stream ? ss[slots] : ctx->stream;
        struct SplitEvents {
            std::vector<cudaEvent_t> v;
            ~SplitEvents() {
                for (cudaEvent_t e : v) cudaEventDestroy(e);
            }
        } sev;
        for (int i = 0; i < 2 * slots; ++i) {
            cudaEvent_t e = nullptr;
            cuda_check(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            sev.v.push_back(e);
        }
        // events: [1 + k] grid done on slot k, [1 + slots + k] slot k's scratch consumed
        while (acc_stream && static_cast<int>(ctx->events.size()) < 1 + 2 * slots) {
            cudaEvent_t e = nullptr;
            cuda_check(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            ctx->events.push_back(e);
        }
        for (int b = 0; b < B; ++b) {
            const int k = b % slots;
            const cudaStream_t stream = ss[k];
            BwWs& w = ws[k];
            const double* Tb = T + n * b;
            if (acc_stream && b >= slots)  // the accumulation of grid b - slots read this slot's scratch
                cuda_check(ctx, cudaStreamWaitEvent(stream, ctx->events[1 + slots + k], 0), "cudaStreamWaitEvent");
            double* lamb = lambda ? lam + n * b : w.lam;
            double* g[5];
            for (int c = 0; c < 5; ++c) g[c] = acc ? w.tmp[c] : out[c] + n * b;
            rfk::AdjointArgs wa = w.adj;
            if (proj && !acc) {  // per-grid gradients leave through the VJP in the gradient pass
                wa.proj = *proj;
                for (int c = 0; c < 5; ++c) wa.raw[c] = rawp[c] + raw->param_stride * b;
            }
            // the order (keys from T and the source mask, sort, rank) beside identify
            const AdjointSplit split{ss[side0 + k], sev.v[2 * k], sev.v[2 * k + 1], d.src + f->src_stride * b,
                                     bad + b};
            const int cap = slots > 1 ? sms / slots : 0;
            run_adjoint(ctx, f->rows, f->cols, f->h, Tb, w.rec, lg + n * b, lamb, cl + b, g, &wa, stream, cap,
                        &split, 0);
            const double* hz = !RFK_ID_HOISTED ? nullptr : f->param_stride == 0 ? ws[0].hoisted : w.hoisted;
            if (RFK_ID_HOISTED && f->param_stride != 0) {
                const int64_t po = f->param_stride * b;
                launched(ctx,
                         rfk::launch_hoist(d.g11 + po, d.g12 + po, d.g22 + po, d.b1 + po, d.b2 + po, f->h, f->rows,
                                           f->cols, w.hoisted, stream, nullptr, nullptr, 1),
                         "hoist");
            }
            identify_grid(ctx, f, d, b, Tb, tol, w.rec, w.cnt, w.cnt + 1, bad + b, stream, hz);
            run_adjoint(ctx, f->rows, f->cols, f->h, Tb, w.rec, lg + n * b, lamb, cl + b, g, &wa, stream, cap,
                        &split, 1);
            if (acc) {
                if (acc_stream) {
                    cuda_check(ctx, cudaEventRecord(ctx->events[1 + k], stream), "cudaEventRecord");
                    cuda_check(ctx, cudaStreamWaitEvent(astream, ctx->events[1 + k], 0), "cudaStreamWaitEvent");
                }
                const double* add[5] = {w.tmp[0], w.tmp[1], w.tmp[2], w.tmp[3], w.tmp[4]};
                launched(ctx, rfk::launch_accumulate5(n, out, add, astream), "accumulate");
                if (acc_stream) cuda_check(ctx, cudaEventRecord(ctx->events[1 + slots + k], astream), "cudaEventRecord");
            }
        }
        join_slots(ctx, ss);
        if (proj && acc)  // accumulated over the grids in order, then the VJP once (as unfused)
            launched(ctx,
                     rfk::launch_project_vjp(proj->mode, n, rawp[0], rawp[1], rawp[2], rawp[3], rawp[4], proj->eps_min,
                                             proj->lambda_max, proj->tau, proj->cap, out[0], out[1], out[2], out[3],
                                             out[4], ctx->stream),
                     "project_vjp");
        std::vector<unsigned long long> hb(B);
        cuda_check(ctx, cudaMemcpyAsync(hb.data(), bad, sizeof(unsigned long long) * B, cudaMemcpyDeviceToHost,
                                        ctx->stream),
                   "D2H");
        st.finish();
        int64_t first_bad = -1;
        std::vector<int64_t> bb(B);
        for (int b = 0; b < B; ++b) {
            bb[b] = hb[b] == ~0ull ? -1 : static_cast<int64_t>(hb[b]);
            if (bb[b] >= 0 && first_bad < 0) first_bad = bb[b];
        }
        if (bad_node) {
            if (mem == RFK_MEM_HOST)
                std::memcpy(bad_node, bb.data(), sizeof(int64_t) * B);
            else
                cuda_check(ctx, cudaMemcpy(bad_node, bb.data(), sizeof(int64_t) * B, cudaMemcpyHostToDevice), "H2D");
        }
        if (first_bad >= 0) fail(ctx, RFK_ERR_INCONSISTENT_FIXED_POINT, bad_node_message(f, first_bad));
    });
}

RFK_API rfk_status rfk_backward(rfk_context* ctx, rfk_memory mem, const rfk_fields* f, const double* t,
                                double tol, const double* loss_grad, double* lambda, double* d_g11,
                                double* d_g12, double* d_g22, double* d_b1, double* d_b2,
                                int32_t accumulate, int32_t* clamped, int64_t* bad_node) {
    return run_backward(ctx, mem, f, t, tol, loss_grad, lambda, d_g11, d_g12, d_g22, d_b1, d_b2, accumulate, clamped,
                        bad_node);
}

RFK_API rfk_status rfk_backward_projected(rfk_context* ctx, rfk_memory mem, const rfk_fields* raw,
                                          const rfk_projection* proj, const double* const projected[5],
                                          const double* t, double tol, const double* loss_grad, double* lambda,
                                          double* d_g11, double* d_g12, double* d_g22, double* d_b1, double* d_b2,
                                          int32_t accumulate, int32_t* clamped, int64_t* bad_node) {
    rfk::ProjCfg c;
    const rfk_status st = guarded(ctx, [&] {
        proj_cfg(ctx, proj, c);
        if (!raw || !projected || !projected[0]) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
    });
    if (st != RFK_OK) return st;
    if (!c.mode)
        return run_backward(ctx, mem, raw, t, tol, loss_grad, lambda, d_g11, d_g12, d_g22, d_b1, d_b2, accumulate,
                            clamped, bad_node);
    rfk_fields fp = *raw;  // identify and the adjoint see the projected parameters
    fp.g11 = projected[0];
    fp.g12 = projected[1];
    fp.g22 = projected[2];
    fp.b1 = projected[3];
    fp.b2 = projected[4];
    return run_backward(ctx, mem, &fp, t, tol, loss_grad, lambda, d_g11, d_g12, d_g22, d_b1, d_b2, accumulate,
                        clamped, bad_node, &c, raw);
}

RFK_API rfk_status rfk_backward_f32(rfk_context* ctx, rfk_memory mem, const rfk_fields_f32* f, const float* t,
                                    double tol, const float* loss_grad, float* d_g11, float* d_g12, float* d_g22,
                                    float* d_b1, float* d_b2, int32_t accumulate, int32_t* clamped,
                                    int64_t* bad_node) {
    // fp32 storage in and out; the values are widened on the device and run
    // through the fp64 identify -> adjoint -> gradient path (rfk_backward),
    // whose fp64 arithmetic keeps stencil identification identical to the
    // fp64 mode's on the same arrival field
    struct Wide {
        rfk_fields f{};
        double* t = nullptr;
        double* lg = nullptr;
        double* g[5] = {};
        int32_t* cl = nullptr;
        int64_t n = 0, np = 0, nt = 0, ng = 0;
    } w;
    rfk_status st = guarded(ctx, [&] {
        if (!f || !t || !loss_grad || !d_g11 || !d_g12 || !d_g22 || !d_b1 || !d_b2)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        if (f->batch < 1 || f->rows < 3 || f->cols < 3) fail(ctx, RFK_ERR_ZERO_DIMENSION, "GridSpec: rows and cols must be at least 3");
        w.n = static_cast<int64_t>(f->rows) * f->cols;
        w.np = f->param_stride ? f->param_stride * f->batch : w.n;
        w.nt = w.n * f->batch;
        const bool acc = accumulate && f->param_stride == 0;
        w.ng = acc ? w.n : w.n * f->batch;
        Stage sg{ctx, mem, {}};
        const float* fin[5] = {sg.in("f32:g11", f->g11, w.np), sg.in("f32:g12", f->g12, w.np),
                               sg.in("f32:g22", f->g22, w.np), sg.in("f32:b1", f->b1, w.np),
                               sg.in("f32:b2", f->b2, w.np)};
        const uint8_t* src = sg.in("f32:src", f->src, f->src_stride ? f->src_stride * f->batch : w.n);
        const float* tin = sg.in("f32:t", t, w.nt);
        const float* lin = sg.in("f32:lg", loss_grad, w.nt);
        double* fw[5];
        const char* nm[5] = {"w64:g11", "w64:g12", "w64:g22", "w64:b1", "w64:b2"};
        for (int k = 0; k < 5; ++k) {
            fw[k] = tbuf<double>(ctx, nm[k], w.np);
            launched(ctx, rfk::launch_widen_f32(w.np, fin[k], fw[k], ctx->stream), "widen");
        }
        w.t = tbuf<double>(ctx, "w64:t", w.nt);
        w.lg = tbuf<double>(ctx, "w64:lg", w.nt);
        launched(ctx, rfk::launch_widen_f32(w.nt, tin, w.t, ctx->stream), "widen");
        launched(ctx, rfk::launch_widen_f32(w.nt, lin, w.lg, ctx->stream), "widen");
        for (int k = 0; k < 5; ++k) w.g[k] = tbuf<double>(ctx, std::string("w64:d") + (nm[k] + 4), w.ng);
        w.cl = tbuf<int32_t>(ctx, "w64:clamped", f->batch);
        w.f.batch = f->batch;
        w.f.rows = f->rows;
        w.f.cols = f->cols;
        w.f.h = f->h;
        w.f.g11 = fw[0];
        w.f.g12 = fw[1];
        w.f.g22 = fw[2];
        w.f.b1 = fw[3];
        w.f.b2 = fw[4];
        w.f.param_stride = f->param_stride;
        w.f.src = src;
        w.f.src_stride = f->src_stride;
        w.f.fixed_values = nullptr;
    });
    if (st != RFK_OK) return st;
    // the inner call runs on device memory: a host bad_node goes through a device buffer
    int64_t* wbad = nullptr;
    if (bad_node && mem == RFK_MEM_HOST) {
        st = guarded(ctx, [&] { wbad = tbuf<int64_t>(ctx, "w64:bad", f->batch); });
        if (st != RFK_OK) return st;
    }
    st = run_backward(ctx, RFK_MEM_DEVICE, &w.f, w.t, tol, w.lg, nullptr, w.g[0], w.g[1], w.g[2], w.g[3], w.g[4],
                      accumulate, w.cl, wbad ? wbad : bad_node);
    if (wbad && (st == RFK_OK || st == RFK_ERR_INCONSISTENT_FIXED_POINT)) {
        const std::string msg = ctx->err;
        const rfk_status sb = guarded(ctx, [&] {
            cuda_check(ctx, cudaMemcpy(bad_node, wbad, sizeof(int64_t) * f->batch, cudaMemcpyDeviceToHost), "D2H");
        });
        if (sb != RFK_OK) return sb;
        ctx->err = msg;
    }
    if (st != RFK_OK) return st;
    const rfk_status st2 = guarded(ctx, [&] {
        Stage so{ctx, mem, {}};
        float* out[5] = {so.out("f32:dg11", d_g11, w.ng), so.out("f32:dg12", d_g12, w.ng),
                         so.out("f32:dg22", d_g22, w.ng), so.out("f32:db1", d_b1, w.ng), so.out("f32:db2", d_b2, w.ng)};
        for (int k = 0; k < 5; ++k) launched(ctx, rfk::launch_narrow_f64(w.ng, w.g[k], out[k], ctx->stream), "narrow");
        int32_t* clo = so.out("f32:clamped", clamped, f->batch);
        if (clo) cuda_check(ctx, cudaMemcpyAsync(clo, w.cl, sizeof(int32_t) * f->batch, cudaMemcpyDeviceToDevice,
                                                 ctx->stream), "D2D");
        so.finish();
    });
    return st2;
}

RFK_API rfk_status rfk_objective_and_grad(rfk_context* ctx, rfk_memory mem, const rfk_fields* f,
                                          const rfk_observations* obs, const rfk_objective_options* opt,
                                          double* data_loss, int32_t* unreached, double* d_g11,
                                          double* d_g12, double* d_g22, double* d_b1, double* d_b2) {
    return guarded(ctx, [&] {
        if (!f || !obs || !opt) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        if (f->batch != 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "objective_and_grad: one parameter set");
        if (obs->count < 1 || !obs->sources || !obs->observed || !obs->values)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "objective_and_grad: needs at least one observation set");
        if (!data_loss || !d_g11 || !d_g12 || !d_g22 || !d_b1 || !d_b2)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null output");
        rfk_fields probe = *f;
        probe.src = obs->sources;
        validate_fields(ctx, &probe);
        const int K = obs->count;
        const int64_t n = static_cast<int64_t>(f->rows) * f->cols;
        const size_t nk = static_cast<size_t>(n) * K;
        Stage st{ctx, mem, {}};
        rfk_fields fd = *f;
        fd.g11 = st.in("g11", f->g11, n);
        fd.g12 = st.in("g12", f->g12, n);
        fd.g22 = st.in("g22", f->g22, n);
        fd.b1 = st.in("b1", f->b1, n);
        fd.b2 = st.in("b2", f->b2, n);
        fd.param_stride = 0;
        fd.batch = K;
        fd.src = st.in("src", obs->sources, nk);
        fd.src_stride = n;
        fd.fixed_values = nullptr;
        // The observations are needed only after the solve: from host memory
        // they travel on a side stream while the sweep runs.
        // The upload has its own stream (the batched solve's slots use the aux
        // streams), and on every exit path -- NotConverged and errors
        // included -- the guard waits for it before the call returns, so the
        // caller's host buffers are never read after return.
        const uint8_t* observed = nullptr;
        const double* values = nullptr;
        struct SideUpload {
            rfk_context* ctx;
            cudaEvent_t ready = nullptr;
            ~SideUpload() {
                if (ready) {
                    cudaStreamSynchronize(ctx->side_stream);
                    cudaEventDestroy(ready);
                }
            }
        } up{ctx};
        if (mem == RFK_MEM_HOST) {
            uint8_t* od = tbuf<uint8_t>(ctx, "in:observed", nk);
            double* vd = tbuf<double>(ctx, "in:values", nk);
            if (!ctx->side_stream)
                cuda_check(ctx, cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking), "cudaStreamCreate");
            cuda_check(ctx, cudaEventCreateWithFlags(&up.ready, cudaEventDisableTiming), "cudaEventCreate");
            // after the context stream's earlier work on these workspaces
            cuda_check(ctx, cudaEventRecord(up.ready, ctx->stream), "cudaEventRecord");
            cuda_check(ctx, cudaStreamWaitEvent(ctx->side_stream, up.ready, 0), "cudaStreamWaitEvent");
            cuda_check(ctx, cudaMemcpyAsync(od, obs->observed, nk, cudaMemcpyHostToDevice, ctx->side_stream), "H2D");
            cuda_check(ctx,
                       cudaMemcpyAsync(vd, obs->values, nk * sizeof(double), cudaMemcpyHostToDevice, ctx->side_stream),
                       "H2D");
            cuda_check(ctx, cudaEventRecord(up.ready, ctx->side_stream), "cudaEventRecord");
            observed = od;
            values = vd;
        } else {
            observed = obs->observed;
            values = obs->values;
        }
        double* out[5] = {st.out("dg11", d_g11, n), st.out("dg12", d_g12, n), st.out("dg22", d_g22, n),
                          st.out("db1", d_b1, n), st.out("db2", d_b2, n)};
        // everything below runs device-resident through the same entry points
        double* T = tbuf<double>(ctx, "obj:t", nk);
        double* lg = tbuf<double>(ctx, "obj:lg", nk);
        int32_t* its = tbuf<int32_t>(ctx, "obj:its", K);
        int32_t* conv = tbuf<int32_t>(ctx, "obj:conv", K);
        double* loss = tbuf<double>(ctx, "obj:loss", K);
        int32_t* unr = tbuf<int32_t>(ctx, "obj:unr", K);
        rfk_solve_options so{opt->solve_tol, opt->solve_max_iters, {0, 1, 2, 3}};
        auto rethrow = [&](rfk_status s) {
            if (s != RFK_OK) throw Fail{s};
        };
        rethrow(rfk_solve(ctx, RFK_MEM_DEVICE, &fd, &so, T, its, conv, nullptr));
        std::vector<int32_t> hconv(K), hunr(K);
        std::vector<double> hloss(K);
        cuda_check(ctx, cudaMemcpy(hconv.data(), conv, sizeof(int32_t) * K, cudaMemcpyDeviceToHost), "D2H");
        for (int k = 0; k < K; ++k)
            if (!hconv[k]) fail(ctx, RFK_ERR_NOT_CONVERGED, "objective_and_grad: forward solve did not converge");
        if (up.ready) cuda_check(ctx, cudaStreamWaitEvent(ctx->stream, up.ready, 0), "cudaStreamWaitEvent");
        rethrow(rfk_loss_grad_mse(ctx, RFK_MEM_DEVICE, K, n, T, observed, values, lg, loss, unr, opt->exact_sum));
        cuda_check(ctx, cudaMemcpy(hloss.data(), loss, sizeof(double) * K, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(ctx, cudaMemcpy(hunr.data(), unr, sizeof(int32_t) * K, cudaMemcpyDeviceToHost), "D2H");
        // data_loss in the reference's order: per set, its MSE sum, then the
        // unreached penalties in node order (inversion.cpp:38-48)
        double dl = 0.0;
        int32_t un = 0;
        for (int k = 0; k < K; ++k) {
            dl += hloss[k];
            un += hunr[k];
            if (hunr[k] > 0) {
                double* acc = tbuf<double>(ctx, "obj:pen", 1);
                cuda_check(ctx, cudaMemcpy(acc, &dl, sizeof(double), cudaMemcpyHostToDevice), "H2D");
                launched(ctx,
                         rfk::launch_unreached_penalty(n, T + n * k, observed + n * k, values + n * k,
                                                       opt->unreached_penalty_cap, acc, ctx->stream),
                         "unreached_penalty");
                cuda_check(ctx, cudaMemcpy(&dl, acc, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
            }
        }
        // the solve above hoisted this metric into the shared workspace: the
        // backward's identify reads those records without re-hoisting
        rethrow(run_backward(ctx, RFK_MEM_DEVICE, &fd, T, opt->solve_tol, lg, nullptr, out[0], out[1], out[2],
                             out[3], out[4], 1, nullptr, nullptr, nullptr, nullptr, true));
        st.finish();
        *data_loss = dl;
        if (unreached) *unreached = un;
    });
}

static void validate_projection(rfk_context* ctx, double eps_min, double lambda_max, double tau) {
    if (!(eps_min > 0.0) || !(eps_min < lambda_max))
        fail(ctx, RFK_ERR_INVALID_ARGUMENT, "ProjectionConfig: need 0 < eps_min < lambda_max");
    if (!(tau > 0.0) || !(tau < 1.0)) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "ProjectionConfig: need 0 < tau < 1");
}

RFK_API rfk_status rfk_project_spd(rfk_context* ctx, rfk_memory mem, int64_t n, double* g11, double* g12,
                                   double* g22, double eps_min, double lambda_max) {
    return guarded(ctx, [&] {
        validate_projection(ctx, eps_min, lambda_max, 0.95);
        if (n <= 0) return;
        Stage st{ctx, mem, {}};
        double* a = st.inout("g11", g11, n);
        double* b = st.inout("g12", g12, n);
        double* c = st.inout("g22", g22, n);
        launched(ctx, rfk::launch_project_spd(n, a, b, c, eps_min, lambda_max, ctx->stream), "project_spd");
        st.finish();
    });
}

RFK_API rfk_status rfk_project_drift(rfk_context* ctx, rfk_memory mem, int64_t n, double* b1, double* b2,
                                     const double* g11, const double* g12, const double* g22, double tau,
                                     double euclid_cap) {
    return guarded(ctx, [&] {
        validate_projection(ctx, 1e-3, 1e3, tau);
        if (n <= 0) return;
        Stage st{ctx, mem, {}};
        double* x = st.inout("b1", b1, n);
        double* y = st.inout("b2", b2, n);
        const double* a = st.in("g11", g11, n);
        const double* b = st.in("g12", g12, n);
        const double* c = st.in("g22", g22, n);
        launched(ctx, rfk::launch_project_drift(n, x, y, a, b, c, tau, euclid_cap, ctx->stream), "project_drift");
        st.finish();
    });
}

RFK_API rfk_status rfk_drift_norm_sq(rfk_context* ctx, rfk_memory mem, int64_t n, const double* b1,
                                     const double* b2, const double* g11, const double* g12,
                                     const double* g22, double* out) {
    return guarded(ctx, [&] {
        if (n <= 0) return;
        Stage st{ctx, mem, {}};
        const double* x = st.in("b1", b1, n);
        const double* y = st.in("b2", b2, n);
        const double* a = st.in("g11", g11, n);
        const double* b = st.in("g12", g12, n);
        const double* c = st.in("g22", g22, n);
        double* o = st.out("out", out, n);
        launched(ctx, rfk::launch_drift_norm_sq(n, x, y, a, b, c, o, ctx->stream), "drift_norm_sq");
        st.finish();
    });
}

static void run_project_vjp(rfk_context* ctx, rfk_memory mem, int mode, int64_t n, const double* g11,
                            const double* g12, const double* g22, const double* b1, const double* b2,
                            double eps_min, double lambda_max, double tau, double euclid_cap, double* d_g11,
                            double* d_g12, double* d_g22, double* d_b1, double* d_b2) {
    validate_projection(ctx, eps_min, lambda_max, tau);
    if (n < 0) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "negative length");
    if (!g11 || !g12 || !g22) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "metric planes are required");
    if ((mode & 2) && (!b1 || !b2 || !d_b1 || !d_b2)) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "drift planes are required");
    if ((mode & 1) && (!d_g11 || !d_g12 || !d_g22)) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "metric cotangents are required");
    if ((d_g11 == nullptr) != (d_g12 == nullptr) || (d_g11 == nullptr) != (d_g22 == nullptr))
        fail(ctx, RFK_ERR_INVALID_ARGUMENT, "metric cotangents must be all set or all NULL");
    if (n == 0) return;
    Stage st{ctx, mem, {}};
    const double* a = st.in("g11", g11, n);
    const double* b = st.in("g12", g12, n);
    const double* c = st.in("g22", g22, n);
    const double* x = st.in("b1", b1, n);
    const double* y = st.in("b2", b2, n);
    double* da = st.inout("d_g11", d_g11, n);
    double* db = st.inout("d_g12", d_g12, n);
    double* dc = st.inout("d_g22", d_g22, n);
    double* dx = st.inout("d_b1", d_b1, n);
    double* dy = st.inout("d_b2", d_b2, n);
    launched(ctx,
             rfk::launch_project_vjp(mode, n, a, b, c, x, y, eps_min, lambda_max, tau, euclid_cap, da, db, dc, dx,
                                     dy, ctx->stream),
             "project_vjp");
    st.finish();
}

RFK_API rfk_status rfk_project_spd_vjp(rfk_context* ctx, rfk_memory mem, int64_t n, const double* g11,
                                       const double* g12, const double* g22, double eps_min, double lambda_max,
                                       double* d_g11, double* d_g12, double* d_g22) {
    return guarded(ctx, [&] {
        run_project_vjp(ctx, mem, 1, n, g11, g12, g22, nullptr, nullptr, eps_min, lambda_max, 0.95, 10.0, d_g11,
                        d_g12, d_g22, nullptr, nullptr);
    });
}

RFK_API rfk_status rfk_project_drift_vjp(rfk_context* ctx, rfk_memory mem, int64_t n, const double* b1,
                                         const double* b2, const double* g11, const double* g12,
                                         const double* g22, double tau, double euclid_cap, double* d_b1,
                                         double* d_b2, double* d_g11, double* d_g12, double* d_g22) {
    return guarded(ctx, [&] {
        run_project_vjp(ctx, mem, 2, n, g11, g12, g22, b1, b2, 1e-3, 1e3, tau, euclid_cap, d_g11, d_g12, d_g22,
                        d_b1, d_b2);
    });
}

RFK_API rfk_status rfk_project_vjp(rfk_context* ctx, rfk_memory mem, int64_t n, const double* g11,
                                   const double* g12, const double* g22, const double* b1, const double* b2,
                                   double eps_min, double lambda_max, double tau, double euclid_cap,
                                   double* d_g11, double* d_g12, double* d_g22, double* d_b1, double* d_b2) {
    return guarded(ctx, [&] {
        run_project_vjp(ctx, mem, 3, n, g11, g12, g22, b1, b2, eps_min, lambda_max, tau, euclid_cap, d_g11, d_g12,
                        d_g22, d_b1, d_b2);
    });
}

}  // extern "C"

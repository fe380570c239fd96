// rfk_capi_internal.h — the context and the staging/validation helpers shared
// by the C-ABI translation units (rfk_capi.cu, rfk_capi_inverse.cu).  Not installed.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/rfk.h"
#include "rfk_internal.h"
struct rfk_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t rebind_event = nullptr;  // rfk_set_stream: orders the new stream after the old one
    cudaStream_t side_stream = nullptr;  // objective_and_grad's observation upload
    std::string err;
    int64_t launches = 0;
    unsigned long long sweep_epoch = 1;
    unsigned adj_epoch = 0;
    struct Buf {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::map<std::string, Buf> bufs;
    unsigned long long* trace = nullptr;  // RFK_TRACE diagnostics of the last solve
    size_t trace_words = 0;
    // concurrent grid slots of a batched sweep: slot k > 0 runs on aux[k-1],
    // forked from / joined back to `stream` with events
    std::vector<cudaStream_t> aux;
    std::vector<cudaEvent_t> events;

    ~rfk_context() {
        for (auto& kv : bufs)
            if (kv.second.p) cudaFree(kv.second.p);
        for (auto s : aux) cudaStreamDestroy(s);
        for (auto e : events) cudaEventDestroy(e);
        if (rebind_event) cudaEventDestroy(rebind_event);
        if (side_stream) cudaStreamDestroy(side_stream);
    }
};

namespace {

using rfk::RecordPlanes;

struct Fail {
    rfk_status status;
};

void fail(rfk_context* ctx, rfk_status s, const std::string& msg) {
    ctx->err = msg;
    throw Fail{s};
}

void cuda_check(rfk_context* ctx, cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(ctx, e == cudaErrorMemoryAllocation ? RFK_ERR_ALLOC : RFK_ERR_CUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
    }
}

// Named, grow-only device buffers.  `zero` clears newly (re)allocated memory
// (used for epoch-tagged flag arrays, which never need clearing otherwise).
void* buf(rfk_context* ctx, const std::string& name, size_t bytes, bool zero = false) {
    if (bytes == 0) bytes = 16;
    auto& b = ctx->bufs[name];
    if (b.bytes < bytes) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
        cuda_check(ctx, cudaMalloc(&b.p, bytes), "cudaMalloc");
        b.bytes = bytes;
        if (zero) cuda_check(ctx, cudaMemsetAsync(b.p, 0, bytes, ctx->stream), "cudaMemsetAsync");
    }
    return b.p;
}

template <class T>
T* tbuf(rfk_context* ctx, const std::string& name, size_t count, bool zero = false) {
    return static_cast<T*>(buf(ctx, name, count * sizeof(T), zero));
}

// Staging of caller buffers: in host mode inputs are copied into named device
// buffers and outputs copied back at the end of the call.
struct Stage {
    rfk_context* ctx;
    rfk_memory mem;
    struct Out {
        void* host;
        const void* dev;
        size_t bytes;
    };
    std::vector<Out> outs;

    template <class T>
    const T* in(const std::string& name, const T* p, size_t count) {
        if (!p) return nullptr;
        if (mem == RFK_MEM_DEVICE) return p;
        T* d = tbuf<T>(ctx, "in:" + name, count);
        cuda_check(ctx, cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream),
                   "H2D");
        return d;
    }
    template <class T>
    T* out(const std::string& name, T* p, size_t count) {
        if (!p) return nullptr;
        if (mem == RFK_MEM_DEVICE) return p;
        T* d = tbuf<T>(ctx, "out:" + name, count);
        outs.push_back({p, d, count * sizeof(T)});
        return d;
    }
    template <class T>
    T* inout(const std::string& name, T* p, size_t count) {
        if (!p) return nullptr;
        if (mem == RFK_MEM_DEVICE) return p;
        T* d = tbuf<T>(ctx, "io:" + name, count);
        cuda_check(ctx, cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream),
                   "H2D");
        outs.push_back({p, d, count * sizeof(T)});
        return d;
    }
    void finish() {
        for (auto& o : outs)
            cuda_check(ctx, cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, ctx->stream),
                       "D2H");
        cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    }
};

template <class F>
rfk_status guarded(rfk_context* ctx, F&& f) {
    if (!ctx) return RFK_ERR_INVALID_ARGUMENT;
    try {
        cuda_check(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
        f();
        ctx->err.clear();
        return RFK_OK;
    } catch (const Fail& e) {
        return e.status;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return RFK_ERR_CUDA;
    }
}

void launched(rfk_context* ctx, cudaError_t e, const char* what, int count = 1) {
    cuda_check(ctx, e, what);
    ctx->launches += count;
}

// GridSpec::validate (grid.hpp:61-65) + batch sanity.
void validate_fields(rfk_context* ctx, const rfk_fields* f) {
    if (!f) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null rfk_fields");
    if (f->rows < 3 || f->cols < 3)
        fail(ctx, RFK_ERR_ZERO_DIMENSION, "GridSpec: rows and cols must be at least 3");
    if (!(f->h > 0.0)) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "GridSpec: h must be positive");
    if (f->batch < 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "rfk_fields: batch must be >= 1");
    if (!f->g11 || !f->g12 || !f->g22 || !f->b1 || !f->b2 || !f->src)
        fail(ctx, RFK_ERR_DIMENSION_MISMATCH, "solve: field dimensions disagree with grid spec");
}

}  // namespace

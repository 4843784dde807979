// Internal plumbing shared by all translation units of libhdgb200.so: the context object,
// RAII device buffers, host<->device staging, launch accounting and error propagation.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hdgb200.h"

namespace hdgb {

// Exception carrying an hdgb_status; converted back to a status code at the C boundary.
struct Failure : std::runtime_error {
    hdgb_status code;
    int64_t index;
    Failure(hdgb_status c, const std::string& msg, int64_t idx = -1)
        : std::runtime_error(msg), code(c), index(idx) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw Failure(HDGB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file +
                                         ":" + std::to_string(line) + ")");
    }
}
#define HDGB_CUDA(x) ::hdgb::cuda_check((x), #x, __FILE__, __LINE__)

}  // namespace hdgb

struct hdgb_ctx;
namespace hdgb {
// Communicator of a domain-decomposed run (one rank per GPU).  halo(): fills the halo entries of
// a face-major device vector (width doubles per face) from their owners; allreduce(): in-place sum
// of n device doubles over all ranks.  Both enqueue on / order with ctx->stream.
struct Comm {
    int rank = 0, size = 1;
    virtual ~Comm() = default;
    virtual void halo(hdgb_ctx* c, double* vec, int width) = 0;
    virtual void allreduce(hdgb_ctx* c, double* buf, int n) = 0;
    // Split exchange: halo_begin starts it (the transfer may proceed on the communicator's own stream), work that
    // touches owned entries only may be enqueued on ctx->stream, halo_end orders ctx->stream after the arrival.
    // Default: the blocking exchange in halo_begin.
    virtual void halo_begin(hdgb_ctx* c, double* vec, int width) { halo(c, vec, width); }
    virtual void halo_end(hdgb_ctx*) {}
};
}  // namespace hdgb

// The opaque context of the C ABI.
struct hdgb_ctx {
    hdgb::Comm* comm = nullptr;  // nullptr: single GPU
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    bool owns_stream = false;
    std::string err;
    int64_t err_index = -1;
    int64_t launches = 0;
    bool phase_timing = false;
    // pinned staging area for small host<->device traffic (Hessenberg columns, norms, flags)
    double* pinned = nullptr;
    size_t pinned_doubles = 0;
    // device error words: [0] = lowest singular batch index (INT_MAX = none), [1] = non-finite flag
    int* d_flags = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t spin_ev = nullptr;  // host_wait(): event polled by the calling thread
};

namespace hdgb {
// Wait for everything enqueued on the context's stream by POLLING an event: the per-iteration host reads of
// GMRES (one Hessenberg column each) must not pay a thread wake-up, whatever the device scheduling flags are.
inline void host_wait(hdgb_ctx* c) {
    if (!c->spin_ev) {
        if (cudaEventCreateWithFlags(&c->spin_ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            c->spin_ev = nullptr;
            HDGB_CUDA(cudaStreamSynchronize(c->stream));
            return;
        }
    }
    HDGB_CUDA(cudaEventRecord(c->spin_ev, c->stream));
    cudaError_t e;
    while ((e = cudaEventQuery(c->spin_ev)) == cudaErrorNotReady) {
    }
    if (e != cudaSuccess) HDGB_CUDA(e);
}
// The same wait in two halves: host_mark() notes the point of the stream the host needs, more work may be enqueued
// behind it, host_poll() waits for the marked point only (spinning or blocking).
inline bool host_mark(hdgb_ctx* c) {
    if (!c->spin_ev && cudaEventCreateWithFlags(&c->spin_ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        c->spin_ev = nullptr;
        return false;
    }
    HDGB_CUDA(cudaEventRecord(c->spin_ev, c->stream));
    return true;
}
inline void host_poll(hdgb_ctx* c, bool spin) {
    if (!spin) {
        HDGB_CUDA(cudaEventSynchronize(c->spin_ev));
        return;
    }
    cudaError_t e;
    while ((e = cudaEventQuery(c->spin_ev)) == cudaErrorNotReady) {
    }
    if (e != cudaSuccess) HDGB_CUDA(e);
}
}  // namespace hdgb

namespace hdgb {

inline void count_launch(hdgb_ctx* c, int n = 1) { c->launches += n; }

// Launch-site check: surfaces configuration errors immediately (asynchronous faults are caught
// at the next synchronising call).
#define HDGB_LAUNCH_CHECK(ctx)                                   \
    do {                                                         \
        ::hdgb::count_launch(ctx);                               \
        HDGB_CUDA(cudaGetLastError());                           \
    } while (0)

// Stream-keyed caching allocator behind DevBuf (api_core.cu).  A Newton solve allocates and frees the
// same multi-GB blocks every iteration; cudaMalloc / cudaFree of such blocks costs tens of
// milliseconds, so freed blocks are parked and handed back to the next request of the same size ON
// THE SAME STREAM (stream order makes the reuse safe without synchronising).
void* pool_alloc(size_t bytes, cudaStream_t* stream_out);
void pool_free(void* p, size_t bytes, cudaStream_t stream);
size_t pool_parked_bytes();  // bytes held by the caching allocator for reuse
void pool_trim(cudaStream_t stream);        // frees the parked blocks of a stream (ctx destroy / OOM)
void pool_register(cudaStream_t stream, bool active);
void pool_set_current(cudaStream_t stream); // the stream subsequent DevBuf allocations belong to (thread local)

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t owner = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), owner(o.owner) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; owner = o.owner; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) p = static_cast<T*>(pool_alloc(count * sizeof(T), &owner));
    }
    void release() {
        if (p) pool_free(p, n * sizeof(T), owner);
        p = nullptr;
        n = 0;
    }
    void zero(cudaStream_t s) { if (n) HDGB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
    void upload(const T* host, size_t count, cudaStream_t s) {
        if (count > n) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "DevBuf::upload overflow");
        if (count) HDGB_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void from_host(const std::vector<T>& h, cudaStream_t s) {
        alloc(h.size());
        upload(h.data(), h.size(), s);
        HDGB_CUDA(cudaStreamSynchronize(s));  // h may be a temporary
    }
    std::vector<T> to_host(cudaStream_t s) const {
        std::vector<T> h(n);
        if (n) {
            HDGB_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
            HDGB_CUDA(cudaStreamSynchronize(s));
        }
        return h;
    }
};

inline bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// A read-only view of caller data on the device: passes device pointers through, stages host
// pointers into a temporary device buffer (asynchronously on the context's stream).
struct InArg {
    const double* dev = nullptr;
    DevBuf<double> tmp;
    InArg(hdgb_ctx* c, const double* src, size_t n) {
        if (!src || n == 0) return;
        if (is_device_ptr(src)) {
            dev = src;
        } else {
            tmp.alloc(n);
            HDGB_CUDA(cudaMemcpyAsync(tmp.p, src, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            dev = tmp.p;
        }
    }
};

// A writable view: device pointers pass through; host destinations get a device temporary that
// commit() copies back (synchronising the stream).
struct OutArg {
    double* dev = nullptr;
    double* host = nullptr;
    size_t n = 0;
    DevBuf<double> tmp;
    hdgb_ctx* ctx;
    OutArg(hdgb_ctx* c, double* dst, size_t count, bool preload = false) : n(count), ctx(c) {
        if (!dst || count == 0) return;
        if (is_device_ptr(dst)) {
            dev = dst;
        } else {
            host = dst;
            tmp.alloc(count);
            dev = tmp.p;
            if (preload)
                HDGB_CUDA(cudaMemcpyAsync(tmp.p, dst, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        }
    }
    void commit() {
        if (host) {
            HDGB_CUDA(cudaMemcpyAsync(host, tmp.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            HDGB_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    }
};

// Runs fn, mapping Failure / std::exception to a status + message on the context.
template <class F>
hdgb_status guarded(hdgb_ctx* ctx, F&& fn) {
    if (ctx) pool_set_current(ctx->stream);
    try {
        fn();
        return HDGB_OK;
    } catch (const Failure& f) {
        if (ctx) { ctx->err = f.what(); ctx->err_index = f.index; }
        return f.code;
    } catch (const std::exception& e) {
        if (ctx) { ctx->err = e.what(); ctx->err_index = -1; }
        return HDGB_ERR_GENERIC;
    }
}

// Opt-in to more than 48 KB of dynamic shared memory for a kernel.  The attribute is per function AND per device
// (hdgb_ctx_create(device) allows several devices in one process), so what has been granted is tracked per
// (function, current device) under a mutex (api_core.cu); cheap enough to call at every launch site.
void ensure_dynamic_smem_raw(const void* func, size_t bytes);
template <class K>
inline void ensure_dynamic_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024) ensure_dynamic_smem_raw(reinterpret_cast<const void*>(kernel), bytes);
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace hdgb

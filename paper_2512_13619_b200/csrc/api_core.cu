// C ABI: context management and the batched dense kernels (A0-A2 of SURVEY.md section 8a).
#include <climits>
#include <map>
#include <mutex>
#include <set>

#include "kernels.cuh"

using namespace hdgb;

extern "C" {

const char* hdgb_version(void) { return "hdgb200 0.1 (sm_100a)"; }

namespace hdgb { int64_t g_pool_device_allocs = 0, g_pool_device_frees = 0; }

// Diagnostics of the caching allocator: cudaMalloc / cudaFree calls issued so far (a steady-state solve makes none).
void hdgb_pool_stats(int64_t* device_allocs, int64_t* device_frees) {
    if (device_allocs) *device_allocs = hdgb::g_pool_device_allocs;
    if (device_frees) *device_frees = hdgb::g_pool_device_frees;
}

int hdgb_set_tuning(const char* key, int64_t value) {
    const std::string k = key ? key : "";
    if (k == "use_stream") { hdgb::tuning().use_stream = static_cast<int>(value); return 0; }
    if (k == "stream_min_elems") { hdgb::tuning().stream_min_elems = value; return 0; }
    if (k == "cgs_evict_first") { hdgb::tuning().cgs_evict_first = static_cast<int>(value); return 0; }
    if (k == "stream_persist_mb") { hdgb::tuning().stream_persist_mb = static_cast<int>(value); return 0; }
    if (k == "stream_evict_first") { hdgb::tuning().stream_evict_first = static_cast<int>(value); return 0; }
    if (k == "gj_direct") { hdgb::tuning().gj_direct = static_cast<int>(value); return 0; }
    if (k == "gj_smem") { hdgb::tuning().gj_smem = static_cast<int>(value); return 0; }
    if (k == "gj_panel_cta") { hdgb::tuning().gj_panel_cta = static_cast<int>(value); return 0; }
    if (k == "use_blocked_gj") { hdgb::tuning().use_blocked_gj = static_cast<int>(value); return 0; }
    if (k == "qelim_split_rows") { hdgb::tuning().qelim_split_rows = static_cast<int>(value); return 0; }
    if (k == "gmres_speculate") { hdgb::tuning().gmres_speculate = static_cast<int>(value); return 0; }
    if (k == "poly_fused") { hdgb::tuning().poly_fused = static_cast<int>(value); return 0; }
    if (k == "overlap_halo") { hdgb::tuning().overlap_halo = static_cast<int>(value); return 0; }
    if (k == "spin_sync") { hdgb::tuning().spin_sync = static_cast<int>(value); return 0; }
    if (k == "cgs_stream") { hdgb::tuning().cgs_stream = static_cast<int>(value); return 0; }
    if (k == "fused_cgs") { hdgb::tuning().fused_cgs = static_cast<int>(value); return 0; }
    if (k == "local_debug_skip") { hdgb::tuning().local_debug_skip = static_cast<int>(value); return 0; }
    if (k == "local_nt") { hdgb::tuning().local_nt = static_cast<int>(value); return 0; }
    if (k == "local_nt_wide") { hdgb::tuning().local_nt_wide = static_cast<int>(value); return 0; }
    if (k == "local_ed_stream") { hdgb::tuning().local_ed_stream = static_cast<int>(value); return 0; }
    if (k == "local_dmma_min_pe") { hdgb::tuning().local_dmma_min_pe = static_cast<int>(value); return 0; }
    if (k == "local_global_records") { hdgb::tuning().local_global_records = static_cast<int>(value); return 0; }
    if (k == "local_dmma_chunked") { hdgb::tuning().local_dmma_chunked = static_cast<int>(value); return 0; }
    if (k == "qelim_stages") { hdgb::tuning().qelim_stages = static_cast<int>(value); return 0; }
    if (k == "gemm_wm_cap") { hdgb::tuning().gemm_wm_cap = static_cast<int>(value < 1 ? 1 : (value > 4 ? 4 : value)); return 0; }
    if (k == "gemm_wn_cap") { hdgb::tuning().gemm_wn_cap = static_cast<int>(value < 1 ? 1 : value); return 0; }
    if (k == "schur_fused") { hdgb::tuning().schur_fused = static_cast<int>(value); return 0; }
    if (k == "qelim_wn") { hdgb::tuning().qelim_wn = static_cast<int>(value); return 0; }
    if (k == "use_qelim_fused") { hdgb::tuning().use_qelim_fused = static_cast<int>(value); return 0; }
    if (k == "use_dmma") { hdgb::tuning().use_dmma = static_cast<int>(value); return 0; }
    if (k == "stream_packed") { hdgb::tuning().stream_packed = static_cast<int>(value); return 0; }
    if (k == "stream_packed_max_cols") { hdgb::tuning().stream_packed_max_cols = static_cast<int>(value); return 0; }
    if (k == "stream_packed_stage_bytes") { hdgb::tuning().stream_packed_stage_bytes = value; return 0; }
    if (k == "use_tile_lu") { hdgb::tuning().use_tile_lu = static_cast<int>(value); return 0; }
    if (k == "assemble_budget_kb") { hdgb::tuning().assemble_budget_kb = static_cast<int>(value); return 0; }
    return 1;
}

hdgb_status hdgb_ctx_create(int device, hdgb_ctx** out) {
    if (!out) return HDGB_ERR_GENERIC;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0 || device < 0 || device >= count) {
        cudaGetLastError();
        // No CPU fallback by design: the hot path exists only as sm_100a kernels.
        fprintf(stderr, "hdgb200: no usable CUDA device (requested %d of %d); there is no CPU fallback\n", device, count);
        return HDGB_ERR_CUDA;
    }
    hdgb_ctx* c = new hdgb_ctx();
    hdgb_status st = guarded(c, [&] {
        HDGB_CUDA(cudaSetDevice(device));
        c->device = device;
        cudaDeviceProp prop{};
        HDGB_CUDA(cudaGetDeviceProperties(&prop, device));
        c->sm_count = prop.multiProcessorCount;
        HDGB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->owns_stream = true;
        pool_register(c->stream, true);
        pool_set_current(c->stream);
        c->pinned_doubles = 1 << 16;
        HDGB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c->pinned), c->pinned_doubles * sizeof(double)));
        HDGB_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->d_flags), 4 * sizeof(int)));
        for (auto& e : c->ev) HDGB_CUDA(cudaEventCreate(&e));
    });
    if (st != HDGB_OK) {
        fprintf(stderr, "hdgb200: context creation failed: %s\n", c->err.c_str());
        delete c;
        return st;
    }
    *out = c;
    return HDGB_OK;
}

void hdgb_ctx_destroy(hdgb_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    delete c->comm;
    c->comm = nullptr;
    pool_register(c->stream, false);
    pool_trim(c->stream);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->spin_ev) cudaEventDestroy(c->spin_ev);
    if (c->d_flags) cudaFree(c->d_flags);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->owns_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* hdgb_last_error(const hdgb_ctx* c) { return c ? c->err.c_str() : "null context"; }
int64_t hdgb_last_error_index(const hdgb_ctx* c) { return c ? c->err_index : -1; }

hdgb_status hdgb_ctx_set_stream(hdgb_ctx* c, void* s) {
    return guarded(c, [&] {
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        pool_register(c->stream, false);
        pool_trim(c->stream);
        if (c->owns_stream && c->stream) cudaStreamDestroy(c->stream);
        c->stream = static_cast<cudaStream_t>(s);
        c->owns_stream = false;
        pool_register(c->stream, true);
        pool_set_current(c->stream);
    });
}
void* hdgb_ctx_stream(hdgb_ctx* c) { return c->stream; }

hdgb_status hdgb_ctx_synchronize(hdgb_ctx* c) {
    return guarded(c, [&] { HDGB_CUDA(cudaStreamSynchronize(c->stream)); });
}

int64_t hdgb_ctx_launch_count(const hdgb_ctx* c) { return c->launches; }
void hdgb_ctx_reset_launch_count(hdgb_ctx* c) { c->launches = 0; }
void hdgb_ctx_enable_phase_timing(hdgb_ctx* c, int on) { c->phase_timing = on != 0; }

hdgb_status hdgb_device_alloc(hdgb_ctx* c, int64_t n, double** out) {
    return guarded(c, [&] {
        *out = nullptr;
        HDGB_CUDA(cudaMalloc(reinterpret_cast<void**>(out), static_cast<size_t>(n) * sizeof(double)));
    });
}
void hdgb_device_free(hdgb_ctx*, double* p) {
    if (p) cudaFree(p);
}
hdgb_status hdgb_copy(hdgb_ctx* c, double* dst, const double* src, int64_t n) {
    return guarded(c, [&] {
        HDGB_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDefault, c->stream));
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"

namespace hdgb {

// ---- caching allocator ---------------------------------------------------------------------------
namespace {
struct Pool {
    std::mutex mu;
    std::map<cudaStream_t, std::multimap<size_t, void*>> parked;  // per stream: size -> block
    std::set<cudaStream_t> active;
    size_t parked_bytes = 0;
};
Pool& pool() {
    static Pool* p = new Pool();  // leaked on purpose: outlives every static destructor that frees a DevBuf
    return *p;
}
thread_local cudaStream_t tl_stream = nullptr;
thread_local bool tl_stream_set = false;
constexpr size_t kParkedCap = static_cast<size_t>(96) << 30;

void free_all_locked(Pool& P) {
    for (auto& kv : P.parked)
        for (auto& b : kv.second) cudaFree(b.second);
    P.parked.clear();
    P.parked_bytes = 0;
}
}  // namespace

void ensure_dynamic_smem_raw(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> granted;
    int dev = 0;
    HDGB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = granted[{func, dev}];
    if (bytes > have) {
        HDGB_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
        have = bytes;
    }
}

void pool_set_current(cudaStream_t s) { tl_stream = s; tl_stream_set = true; }

void pool_register(cudaStream_t s, bool on) {
    Pool& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    if (on) P.active.insert(s);
    else P.active.erase(s);
}

void* pool_alloc(size_t bytes, cudaStream_t* stream_out) {
    Pool& P = pool();
    cudaStream_t s = tl_stream;
    bool pooled = tl_stream_set;
    {
        std::lock_guard<std::mutex> g(P.mu);
        if (pooled && !P.active.count(s)) pooled = false;
        if (pooled) {
            auto it = P.parked.find(s);
            if (it != P.parked.end()) {
                auto b = it->second.find(bytes);
                if (b != it->second.end()) {
                    void* p = b->second;
                    it->second.erase(b);
                    P.parked_bytes -= bytes;
                    *stream_out = s;
                    return p;
                }
            }
        }
    }
    void* p = nullptr;
    ++g_pool_device_allocs;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaDeviceSynchronize();
        {
            std::lock_guard<std::mutex> g(P.mu);
            free_all_locked(P);
        }
        HDGB_CUDA(cudaMalloc(&p, bytes));
    }
    // blocks allocated outside any context are tagged with a stream nobody registers: never parked
    *stream_out = pooled ? s : reinterpret_cast<cudaStream_t>(~static_cast<uintptr_t>(0));
    return p;
}

void pool_free(void* p, size_t bytes, cudaStream_t s) {
    Pool& P = pool();
    {
        std::lock_guard<std::mutex> g(P.mu);
        if (P.active.count(s) && P.parked_bytes + bytes <= kParkedCap) {  // small blocks too: cudaFree synchronises the device
            P.parked[s].emplace(bytes, p);
            P.parked_bytes += bytes;
            return;
        }
    }
    ++g_pool_device_frees;
    cudaFree(p);
}

size_t pool_parked_bytes() {
    Pool& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    return P.parked_bytes;
}

void pool_trim(cudaStream_t s) {
    Pool& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    auto it = P.parked.find(s);
    if (it == P.parked.end()) return;
    for (auto& b : it->second) {
        cudaFree(b.second);
        P.parked_bytes -= b.first;
    }
    P.parked.erase(it);
}

Tuning& tuning() {
    static Tuning t;
    return t;
}

// Resets the device error words, returns after `fn` the lowest singular batch index (or -1).
void reset_flags(hdgb_ctx* c) {
    const int init[4] = {INT_MAX, 0, 0, 0};
    HDGB_CUDA(cudaMemcpyAsync(c->d_flags, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
}

void read_flags(hdgb_ctx* c, int* singular_index, int* nonfinite) {
    int h[4];
    HDGB_CUDA(cudaMemcpyAsync(h, c->d_flags, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    HDGB_CUDA(cudaStreamSynchronize(c->stream));
    if (singular_index) *singular_index = (h[0] == INT_MAX) ? -1 : h[0];
    if (nonfinite) *nonfinite = h[1];
}

// lu_invert_batch on device pointers with the reference's error convention.
void device_lu_invert(hdgb_ctx* c, int n, int64_t batch, const double* a, double* inv, const char* context,
                      hdgb_status code) {
    reset_flags(c);
    launch_lu_invert_batch(c, n, batch, a, inv, c->d_flags);
    int bad = -1;
    read_flags(c, &bad, nullptr);
    if (bad >= 0) {
        std::string msg;
        if (code == HDGB_ERR_SINGULAR_MASS) msg = "singular mass matrix in element " + std::to_string(bad);
        else if (code == HDGB_ERR_SINGULAR_LOCAL_SOLVE) msg = "singular local solve in element " + std::to_string(bad);
        else msg = std::string(context) + ": singular block at batch index " + std::to_string(bad);
        throw Failure(code, msg, bad);
    }
}

}  // namespace hdgb

extern "C" {

hdgb_status hdgb_lu_invert_batch(hdgb_ctx* c, int n, int batch, const double* a, double* inv) {
    return guarded(c, [&] {
        if (n < 1) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: lu_invert_batch requires square blocks with n >= 1");
        const size_t total = static_cast<size_t>(n) * n * batch;
        InArg A(c, a, total);
        OutArg X(c, inv, total);
        device_lu_invert(c, n, batch, A.dev, X.dev, "lu_invert_batch", HDGB_ERR_SINGULAR_BLOCK);
        X.commit();
    });
}

hdgb_status hdgb_gemm_batch(hdgb_ctx* c, int a_rows, int a_cols, int a_batch, const double* a, int b_rows,
                            int b_cols, int b_batch, const double* b, int transpose_a, double* out) {
    return guarded(c, [&] {
        const int m = transpose_a ? a_cols : a_rows;
        const int k = transpose_a ? a_rows : a_cols;
        if (k != b_rows)
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: gemm_batch inner dimensions " +
                                                           std::to_string(k) + " vs " + std::to_string(b_rows));
        if (a_batch != b_batch && a_batch != 1 && b_batch != 1)
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: gemm_batch batch counts " +
                                                           std::to_string(a_batch) + " vs " + std::to_string(b_batch));
        const int nb = a_batch > b_batch ? a_batch : b_batch;
        InArg A(c, a, static_cast<size_t>(a_rows) * a_cols * a_batch);
        InArg B(c, b, static_cast<size_t>(b_rows) * b_cols * b_batch);
        OutArg Cc(c, out, static_cast<size_t>(m) * b_cols * nb);
        launch_gemm_batch(c, m, b_cols, k, A.dev, a_batch == 1 ? 0 : static_cast<int64_t>(a_rows) * a_cols,
                          transpose_a != 0, B.dev, b_batch == 1 ? 0 : static_cast<int64_t>(b_rows) * b_cols, Cc.dev,
                          static_cast<int64_t>(m) * b_cols, nb, 1.0, 0.0);
        Cc.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_gemv_strided_batch(hdgb_ctx* c, int rows, int cols, int batch, const double* a, const double* x,
                                    double* y, int accumulate) {
    return guarded(c, [&] {
        InArg A(c, a, static_cast<size_t>(rows) * cols * batch);
        InArg X(c, x, static_cast<size_t>(cols) * batch);
        OutArg Y(c, y, static_cast<size_t>(rows) * batch, accumulate != 0);
        GemvArgs g;
        g.a = A.dev; g.x = X.dev; g.y = Y.dev;
        g.rows = rows; g.cols = cols; g.batch = batch;
        if (accumulate) { g.z = Y.dev; g.beta = 1.0; }
        launch_team_gemv(c, g);
        Y.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"

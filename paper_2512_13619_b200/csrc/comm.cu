// Multi-GPU plumbing of the domain-decomposed solver (the reference has no
// distributed path, PAPER.md:1122 lists it as future work).  One rank per GPU.  Two exchanges exist:
//   halo      : interface trace slices (width doubles per face) from the owning rank into the halo
//               part of a face-major vector -- point-to-point, NCCL send/recv grouped per neighbour,
//               sends packed by one gather kernel, receives landing directly in the vector because
//               halo faces are numbered contiguously per owner;
//   allreduce : the Arnoldi projection coefficients / norms (a few doubles), ncclAllReduce.
// NCCL is bound at run time (dlopen of libnccl.so.2, the copy the process already uses), so the
// library has no link-time dependency on it.  A callback backend lets tests drive several
// "virtual ranks" inside one process on one GPU.
#include <dlfcn.h>

#include <memory>

#include "kernels.cuh"

namespace hdgb {

namespace {

__global__ void pack_faces_kernel(const double* __restrict__ vec, const int* __restrict__ ids, int64_t total, int width,
                                  double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t k = i / width;
    out[i] = vec[static_cast<int64_t>(ids[k]) * width + (i - k * width)];
}

struct HaloPlan {
    std::vector<int> nbr_rank, send_count, send_off, recv_off, recv_count;
    DevBuf<int> send_ids;  // concatenated over neighbours
    int total_send = 0;
};

// ---- NCCL, bound lazily ---------------------------------------------------------------------------
struct Uid {
    char internal[128];
};
struct NcclApi {
    void* lib = nullptr;
    int (*GetUniqueId)(void*) = nullptr;
    int (*CommInitRank)(void**, int, Uid, int) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    if (api.lib) return api;
    api.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!api.lib) throw Failure(HDGB_ERR_GENERIC, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* n) {
        void* p = dlsym(api.lib, n);
        if (!p) throw Failure(HDGB_ERR_GENERIC, std::string("libnccl.so.2 lacks ") + n);
        return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    return api;
}

void nccl_check(int rc, const char* what) {
    if (rc != 0) throw Failure(HDGB_ERR_GENERIC, std::string(what) + ": " + nccl().GetErrorString(rc));
}

constexpr int kNcclDouble = 8, kNcclSum = 0;

struct NcclComm : Comm {
    void* comm = nullptr;
    HaloPlan plan;
    DevBuf<double> sendbuf;
    // the exchange runs on its own stream so that interior rows / elements overlap it (SURVEY.md 8e option (i))
    cudaStream_t xstream = nullptr;
    cudaEvent_t ev_packed = nullptr, ev_arrived = nullptr;
    bool in_flight = false;
    ~NcclComm() override {
        if (comm) nccl().CommDestroy(comm);
        if (ev_packed) cudaEventDestroy(ev_packed);
        if (ev_arrived) cudaEventDestroy(ev_arrived);
        if (xstream) cudaStreamDestroy(xstream);
    }
    void ensure_stream() {
        if (xstream) return;
        HDGB_CUDA(cudaStreamCreateWithFlags(&xstream, cudaStreamNonBlocking));
        HDGB_CUDA(cudaEventCreateWithFlags(&ev_packed, cudaEventDisableTiming));
        HDGB_CUDA(cudaEventCreateWithFlags(&ev_arrived, cudaEventDisableTiming));
    }
    // pack on `pack_stream`, send / receive on `xfer`
    void exchange(hdgb_ctx* c, double* vec, int width, cudaStream_t xfer) {
        const size_t need = static_cast<size_t>(plan.total_send) * width;
        if (sendbuf.n < need) {
            HDGB_CUDA(cudaStreamSynchronize(c->stream));
            if (xstream) HDGB_CUDA(cudaStreamSynchronize(xstream));
            sendbuf.alloc(need);
        }
        if (need) {
            pack_faces_kernel<<<ceil_div(static_cast<int64_t>(need), 256), 256, 0, c->stream>>>(vec, plan.send_ids.p, static_cast<int64_t>(need), width, sendbuf.p);
            HDGB_LAUNCH_CHECK(c);
        }
        if (xfer != c->stream) {
            // everything enqueued so far (the packed slices, and whatever produced the owned part of vec) precedes the transfer
            HDGB_CUDA(cudaEventRecord(ev_packed, c->stream));
            HDGB_CUDA(cudaStreamWaitEvent(xfer, ev_packed, 0));
        }
        NcclApi& n = nccl();
        nccl_check(n.GroupStart(), "ncclGroupStart");
        for (size_t k = 0; k < plan.nbr_rank.size(); ++k) {
            if (plan.send_count[k])
                nccl_check(n.Send(sendbuf.p + static_cast<size_t>(plan.send_off[k]) * width, static_cast<size_t>(plan.send_count[k]) * width,
                                  kNcclDouble, plan.nbr_rank[k], comm, xfer), "ncclSend");
            if (plan.recv_count[k])
                nccl_check(n.Recv(vec + static_cast<size_t>(plan.recv_off[k]) * width, static_cast<size_t>(plan.recv_count[k]) * width,
                                  kNcclDouble, plan.nbr_rank[k], comm, xfer), "ncclRecv");
        }
        nccl_check(n.GroupEnd(), "ncclGroupEnd");
    }
    void halo(hdgb_ctx* c, double* vec, int width) override {
        if (plan.nbr_rank.empty()) return;
        exchange(c, vec, width, c->stream);
    }
    void halo_begin(hdgb_ctx* c, double* vec, int width) override {
        if (plan.nbr_rank.empty()) return;
        ensure_stream();
        exchange(c, vec, width, xstream);
        HDGB_CUDA(cudaEventRecord(ev_arrived, xstream));
        in_flight = true;
    }
    void halo_end(hdgb_ctx* c) override {
        if (!in_flight) return;
        HDGB_CUDA(cudaStreamWaitEvent(c->stream, ev_arrived, 0));
        in_flight = false;
    }
    void allreduce(hdgb_ctx* c, double* buf, int cnt) override {
        nccl_check(nccl().AllReduce(buf, buf, static_cast<size_t>(cnt), kNcclDouble, kNcclSum, comm, c->stream), "ncclAllReduce");
    }
};

// ---- callback backend (tests: several virtual ranks in one process) ---------------------------------
struct CallbackComm : Comm {
    hdgb_halo_fn halo_fn = nullptr;
    hdgb_allreduce_fn allreduce_fn = nullptr;
    void* user = nullptr;
    void halo(hdgb_ctx* c, double* vec, int width) override {
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        if (halo_fn(user, vec, width) != 0) throw Failure(HDGB_ERR_GENERIC, "halo exchange callback failed");
    }
    void allreduce(hdgb_ctx* c, double* buf, int n) override {
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        if (allreduce_fn(user, buf, n) != 0) throw Failure(HDGB_ERR_GENERIC, "all-reduce callback failed");
    }
};

}  // namespace

}  // namespace hdgb

using namespace hdgb;

extern "C" {

hdgb_status hdgb_comm_nccl_unique_id(void* out128) {
    try {
        nccl_check(nccl().GetUniqueId(out128), "ncclGetUniqueId");
        return HDGB_OK;
    } catch (const Failure& f) {
        fprintf(stderr, "hdgb200: %s\n", f.what());
        return f.code;
    }
}

hdgb_status hdgb_comm_create_nccl(hdgb_ctx* c, const void* unique_id_128, int rank, int size) {
    return guarded(c, [&] {
        std::unique_ptr<NcclComm> nc(new NcclComm());
        nc->rank = rank;
        nc->size = size;
        Uid id;
        std::memcpy(id.internal, unique_id_128, sizeof(id.internal));
        HDGB_CUDA(cudaSetDevice(c->device));
        nccl_check(nccl().CommInitRank(&nc->comm, size, id, rank), "ncclCommInitRank");
        delete c->comm;
        c->comm = nc.release();
    });
}

hdgb_status hdgb_comm_set_callbacks(hdgb_ctx* c, int rank, int size, hdgb_halo_fn halo, hdgb_allreduce_fn allreduce, void* user) {
    return guarded(c, [&] {
        std::unique_ptr<CallbackComm> cc(new CallbackComm());
        cc->rank = rank;
        cc->size = size;
        cc->halo_fn = halo;
        cc->allreduce_fn = allreduce;
        cc->user = user;
        delete c->comm;
        c->comm = cc.release();
    });
}

hdgb_status hdgb_comm_set_halo_plan(hdgb_ctx* c, int n_nbr, const int32_t* nbr_ranks, const int32_t* send_counts,
                                    const int32_t* send_ids, const int32_t* recv_offsets, const int32_t* recv_counts) {
    return guarded(c, [&] {
        NcclComm* nc = dynamic_cast<NcclComm*>(c->comm);
        if (!nc) throw Failure(HDGB_ERR_GENERIC, "hdgb_comm_set_halo_plan needs an NCCL communicator");
        HaloPlan& p = nc->plan;
        p.nbr_rank.assign(nbr_ranks, nbr_ranks + n_nbr);
        p.send_count.assign(send_counts, send_counts + n_nbr);
        p.recv_off.assign(recv_offsets, recv_offsets + n_nbr);
        p.recv_count.assign(recv_counts, recv_counts + n_nbr);
        p.send_off.assign(n_nbr, 0);
        int tot = 0;
        for (int k = 0; k < n_nbr; ++k) { p.send_off[k] = tot; tot += send_counts[k]; }
        p.total_send = tot;
        std::vector<int> ids(send_ids, send_ids + tot);
        p.send_ids.from_host(ids, c->stream);
    });
}

void hdgb_comm_destroy(hdgb_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    delete c->comm;
    c->comm = nullptr;
}

hdgb_status hdgb_halo_exchange(hdgb_ctx* c, double* dev_vec, int width) {
    return guarded(c, [&] {
        if (c->comm) c->comm->halo(c, dev_vec, width);
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_halo_exchange_begin(hdgb_ctx* c, double* dev_vec, int width) {
    return guarded(c, [&] {
        if (c->comm) c->comm->halo_begin(c, dev_vec, width);
    });
}

hdgb_status hdgb_halo_exchange_end(hdgb_ctx* c) {
    return guarded(c, [&] {
        if (c->comm) c->comm->halo_end(c);
    });
}

hdgb_status hdgb_allreduce_sum(hdgb_ctx* c, double* dev_buf, int n) {
    return guarded(c, [&] {
        if (c->comm) c->comm->allreduce(c, dev_buf, n);
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int hdgb_comm_rank(const hdgb_ctx* c) { return c->comm ? c->comm->rank : 0; }
int hdgb_comm_size(const hdgb_ctx* c) { return c->comm ? c->comm->size : 1; }

}  // extern "C"

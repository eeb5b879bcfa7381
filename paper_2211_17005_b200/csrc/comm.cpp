// comm.cpp -- transports of comm.cuh and their C-ABI (include/hcva_gpu.h).
#include "comm.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

using namespace hcva;

namespace {

// ---- NCCL, resolved at run time (no link-time dependency on a libnccl build)
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL unavailable: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.init_rank || !api.all_gather || !api.destroy || !api.error_string) {
            err = "NCCL unavailable: missing symbols in libnccl.so.2";
            api = NcclApi{};
        }
    });
    if (!api.init_rank) throw cuda_error(err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw cuda_error(std::string(what) + ": " + nccl().error_string(r));
}

struct NcclComm final : hcva_comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm) nccl().destroy(comm);
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t stream) override {
        nccl_check(nccl().all_gather(send, recv, bytes, ncclChar, comm, stream), "ncclAllGather");
    }
};

}  // namespace

// ---- in-process group: one host thread (and context) per rank
struct hcva_group {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    std::vector<const void*> ptrs;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

namespace {

struct LocalComm final : hcva_comm {
    hcva_group* group = nullptr;
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t stream) override {
        HCVA_CUDA(cudaStreamSynchronize(stream));  // the send buffer is complete
        group->ptrs[rank] = send;
        group->barrier();
        for (int g = 0; g < world; ++g)
            HCVA_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + g * bytes, group->ptrs[g], bytes, cudaMemcpyDefault,
                                      stream));
        HCVA_CUDA(cudaStreamSynchronize(stream));
        group->barrier();  // every rank has read every send buffer
    }
};

}  // namespace

extern "C" {

hcva_status hcva_comm_nccl_id(uint8_t* id) {
    return guarded([&] {
        ncclUniqueId u;
        nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

hcva_status hcva_comm_create_nccl(hcva_ctx* ctx, int world, int rank, const uint8_t* id, hcva_comm** out) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) throw contract_error("comm: rank outside world");
        HCVA_CUDA(cudaSetDevice(ctx->device));
        auto c = std::make_unique<NcclComm>();
        c->rank = rank;
        c->world = world;
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        nccl_check(nccl().init_rank(&c->comm, world, u, rank), "ncclCommInitRank");
        *out = c.release();
    });
}

hcva_status hcva_group_create(int world, hcva_group** out) {
    return guarded([&] {
        if (world < 1) throw contract_error("comm: world must be >= 1");
        auto g = std::make_unique<hcva_group>();
        g->world = world;
        g->ptrs.assign(world, nullptr);
        *out = g.release();
    });
}

hcva_status hcva_group_destroy(hcva_group* g) {
    return guarded([&] { delete g; });
}

hcva_status hcva_comm_create_local(hcva_ctx* ctx, hcva_group* group, int rank, hcva_comm** out) {
    return guarded([&] {
        (void)ctx;
        if (!group || rank < 0 || rank >= group->world) throw contract_error("comm: rank outside group");
        auto c = std::make_unique<LocalComm>();
        c->rank = rank;
        c->world = group->world;
        c->group = group;
        *out = c.release();
    });
}

hcva_status hcva_comm_info(const hcva_comm* c, int* rank, int* world) {
    return guarded([&] {
        *rank = c->rank;
        *world = c->world;
    });
}

hcva_status hcva_comm_destroy(hcva_comm* c) {
    return guarded([&] { delete c; });
}

}  // extern "C"

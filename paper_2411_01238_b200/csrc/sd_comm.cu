// sd_comm.cu — the NCCL communicator behind the data-parallel backward.
//
// a large-M layer is row-sharded over G GPUs (one process per
// GPU); each rank computes its partial dW over its own rows and ONE NCCL
// all-reduce (sum) of dW over NVLink combines them. The library owns the
// communicator, so a C or C++ caller of the reference's `backward`
// (layer.hpp:128-162) gets the sharded step from the C-ABI alone:
//
//   rank 0: sd_comm_unique_id(id)   -> the caller broadcasts the 128 bytes
//   every rank: sd_comm_init(&comm, nranks, rank, id)
//   every step: sd_layer_plan_forward(plan, seed, s)
//               sd_layer_plan_backward_allreduce(plan, comm, nparts, s, comm_s)
//
// NCCL is resolved at run time (dlopen): the copy already loaded into the
// process (e.g. PyTorch's) if there is one — a communicator must be driven by
// the library that created it, and two NCCLs in one process would not share
// state — else libnccl.so.2 from the loader path. SD_NCCL_LIBRARY overrides.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "sd_internal.h"

struct sd_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0;
    int rank = 0;
    int device = 0;
};

namespace sd {
namespace {

struct NcclApi {
    void* handle = nullptr;
    std::string path;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;
std::string g_nccl_error;

const NcclApi& nccl() {
    std::call_once(g_nccl_once, [] {
        void* h = nullptr;
        std::string path;
        if (const char* e = std::getenv("SD_NCCL_LIBRARY")) {
            h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
            path = e;
        }
        if (!h) {
            // already in the process (torch, or the caller linked it)?
            for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
                h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
                if (h) {
                    path = std::string(name) + " (already loaded)";
                    break;
                }
            }
        }
        if (!h) {
            for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
                h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
                if (h) {
                    path = name;
                    break;
                }
            }
        }
        if (!h) {
            const char* d = dlerror();
            g_nccl_error = std::string("NCCL not found (libnccl.so.2): ") + (d ? d : "");
            return;
        }
        NcclApi a;
        a.handle = h;
        a.path = path;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.get_version = reinterpret_cast<decltype(a.get_version)>(dlsym(h, "ncclGetVersion"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce || !a.error_string) {
            g_nccl_error = "NCCL library " + path + " lacks the required symbols";
            return;
        }
        g_nccl = a;
    });
    if (!g_nccl.handle) fail(SD_ERUNTIME, g_nccl_error.empty() ? "NCCL unavailable" : g_nccl_error);
    return g_nccl;
}

void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(SD_ERUNTIME, std::string(what) + ": " + nccl().error_string(r));
}

template <typename Fn>
int guarded_comm(Fn&& fn) {
    try {
        fn();
        return SD_OK;
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SD_ERUNTIME;
    }
}

}  // namespace

// Sum-all-reduce `count` elements of `buf` in place on `s` (dtype: SD_DTYPE_*).
void comm_allreduce_sum(sd_comm* c, void* buf, size_t count, int dtype, cudaStream_t s) {
    const ncclDataType_t t = dtype == SD_DTYPE_F32 ? ncclFloat32 : ncclBfloat16;
    check_nccl(nccl().all_reduce(buf, buf, count, t, ncclSum, c->comm, s), "ncclAllReduce(dW)");
}

int comm_nranks(const sd_comm* c) { return c->nranks; }
int comm_device(const sd_comm* c) { return c->device; }

}  // namespace sd

using namespace sd;

extern "C" {

int sd_comm_unique_id(void* id_out) {
    return guarded_comm([&] {
        if (!id_out) fail(SD_EINVAL, "sd_comm_unique_id: null output");
        ncclUniqueId id;
        check_nccl(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof id);
    });
}

int sd_comm_init(sd_comm** out, int32_t nranks, int32_t rank, const void* id) {
    return guarded_comm([&] {
        if (!out || !id) fail(SD_EINVAL, "sd_comm_init: null argument");
        *out = nullptr;
        if (nranks < 1 || rank < 0 || rank >= nranks)
            fail(SD_ERANGE, "sd_comm_init: rank " + std::to_string(rank) + " outside [0, " + std::to_string(nranks) +
                                ")");
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        auto* c = new sd_comm;
        c->nranks = nranks;
        c->rank = rank;
        c->device = dev;
        const ncclResult_t r = nccl().comm_init_rank(&c->comm, nranks, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            check_nccl(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

int sd_comm_destroy(sd_comm* c) {
    return guarded_comm([&] {
        if (!c) return;
        const ncclResult_t r = c->comm ? nccl().comm_destroy(c->comm) : ncclSuccess;
        delete c;  // freed either way; a failed destroy is still reported
        check_nccl(r, "ncclCommDestroy");
    });
}

int sd_comm_nccl_version(int32_t* version) {
    return guarded_comm([&] {
        if (!version) fail(SD_EINVAL, "sd_comm_nccl_version: null output");
        int v = 0;
        if (nccl().get_version) check_nccl(nccl().get_version(&v), "ncclGetVersion");
        *version = v;
    });
}

int sd_comm_allreduce_sum(sd_comm* c, void* buf, size_t count, int32_t dtype, void* stream) {
    return guarded_comm([&] {
        if (!c || !buf) fail(SD_EINVAL, "sd_comm_allreduce_sum: null argument");
        if (dtype != SD_DTYPE_F32 && dtype != SD_DTYPE_BF16) fail(SD_EINVAL, "unknown dtype " + std::to_string(dtype));
        comm_allreduce_sum(c, buf, count, dtype, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"

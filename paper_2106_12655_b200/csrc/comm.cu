// NCCL resolved at run time for the library-owned multi-GPU communicator (comm.cuh).
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "comm.cuh"

namespace lc {
namespace {

struct NcclApi {
    void *handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GetVersion)(int *) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

NcclApi &api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        // the NCCL already in the process first (PyTorch maps its own copy), then the system one
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char *e = dlerror();
            a.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown");
            return;
        }
        a.handle = h;
        a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
        a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
        a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
        a.GetVersion = (decltype(a.GetVersion))dlsym(h, "ncclGetVersion");
        a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
        if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.CommDestroy || !a.GetErrorString) {
            a.error = "libnccl.so.2 lacks a required symbol";
            a.handle = nullptr;
        }
    });
    if (!a.handle) throw Error(LC_ERR_STATE, a.error);
    return a;
}

void check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) throw Error(LC_ERR_CUDA, std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace

void comm_unique_id(ncclUniqueId *id) { check(api().GetUniqueId(id), "ncclGetUniqueId"); }

void comm_init(Comm &c, const ncclUniqueId &id, int world, int rank) {
    if (world < 1 || rank < 0 || rank >= world) throw Error(LC_ERR_ARG, "bad world / rank");
    comm_destroy(c);
    check(api().CommInitRank(&c.comm, world, id, rank), "ncclCommInitRank");
    c.world = world;
    c.rank = rank;
}

void comm_destroy(Comm &c) {
    if (c.comm) api().CommDestroy(c.comm);
    c.comm = nullptr;
    c.world = 1;
    c.rank = 0;
}

void comm_allreduce_max_i64(Comm &c, void *buf, size_t n, cudaStream_t s) {
    if (!c.ready()) throw Error(LC_ERR_STATE, "no communicator (lc_comm_init)");
    if (n == 0) return;
    check(api().AllReduce(buf, buf, n, ncclInt64, ncclMax, c.comm, s), "ncclAllReduce");
}

int nccl_version() {
    try {
        int v = 0;
        if (api().GetVersion) api().GetVersion(&v);
        return v;
    } catch (const Error &) {
        return 0;
    }
}

}  // namespace lc

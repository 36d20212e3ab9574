// Multi-GPU data plane of the C ABI (include/wally.h "Multi-GPU data plane"):
// an NCCL communicator per context and the two exchange steps of the
// cluster-sharded path -- the query scatter from the ingress rank to the
// owners and the optional response gather back (north_star: "queries are
// routed to the owning rank, with NCCL over NVLink only for query scatter and
// response gather"; the server "distributes them according to the correct
// clusters").  Per-query work is independent (Alg 4
// P:L794-808), so these are the only collectives of the path.
//
// NCCL is opened at run time (dlopen "libnccl.so.2"): in a process that has
// imported torch this is the NCCL torch already loaded, and the library
// itself loads and runs single-rank without NCCL present.

#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include <nccl.h>

#include "wally_ctx.h"

using namespace wally;

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        bool all = true;
        auto sym = [&](auto &fn, const char *name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) {
                all = false;
                api.why = std::string("libnccl.so.2 lacks ") + name;
            }
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
        api.ok = all;
    });
    return api;
}

}  // namespace

#define NCCL_OK(ctx, call)                                                                                   \
    do {                                                                                                     \
        ncclResult_t _r = (call);                                                                            \
        if (_r != ncclSuccess) return wally_fail(ctx, WALLY_E_NCCL, "%s: %s", #call, nccl().GetErrorString(_r)); \
    } while (0)

#define CUDA_OK_FAIL(ctx, call)                                                                             \
    do {                                                                                                    \
        cudaError_t _e = (call);                                                                            \
        if (_e != cudaSuccess) return wally_fail(ctx, WALLY_E_CUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
    } while (0)

void wally_comm_release(wally_ctx *c) {
    if (c && c->nccl_comm && nccl().ok) nccl().CommDestroy((ncclComm_t)c->nccl_comm);
    if (c) {
        c->nccl_comm = nullptr;
        c->comm_rank = -1;
        c->comm_world = 0;
    }
}

extern "C" int wally_comm_unique_id(uint8_t *id_out) {
    WALLY_NVTX("wally_comm_unique_id");
    if (!id_out) return wally_fail(nullptr, WALLY_E_ARG, "comm_unique_id: null output");
    const NcclApi &api = nccl();
    if (!api.ok) return wally_fail(nullptr, WALLY_E_NCCL, "%s", api.why.c_str());
    static_assert(sizeof(ncclUniqueId) == WALLY_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return wally_fail(nullptr, WALLY_E_NCCL, "ncclGetUniqueId: %s", api.GetErrorString(r));
    memcpy(id_out, &id, sizeof id);
    return WALLY_OK;
}

extern "C" int wally_comm_init(wally_ctx *c, int32_t rank, int32_t world, const uint8_t *id) {
    WALLY_NVTX("wally_comm_init");
    if (!c) return WALLY_E_ARG;
    if (!id || world < 1 || rank < 0 || rank >= world)
        return wally_fail(c, WALLY_E_ARG, "comm_init: need 0 <= rank < world and a unique id");
    const NcclApi &api = nccl();
    if (!api.ok) return wally_fail(c, WALLY_E_NCCL, "%s", api.why.c_str());
    cudaSetDevice(c->device);
    wally_comm_release(c);
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    ncclComm_t comm = nullptr;
    NCCL_OK(c, api.CommInitRank(&comm, world, uid, rank));
    c->nccl_comm = comm;
    c->comm_rank = rank;
    c->comm_world = world;
    return WALLY_OK;
}

extern "C" int wally_comm_check(wally_ctx *c) {
    WALLY_NVTX("wally_comm_check");
    if (!c) return WALLY_E_ARG;
    if (!c->nccl_comm) return wally_fail(c, WALLY_E_STATE, "comm_check: no communicator (wally_comm_init first)");
    ncclResult_t ar = ncclSuccess;
    NCCL_OK(c, nccl().CommGetAsyncError((ncclComm_t)c->nccl_comm, &ar));
    if (ar != ncclSuccess) return wally_fail(c, WALLY_E_NCCL, "NCCL async error: %s", nccl().GetErrorString(ar));
    return WALLY_OK;
}

extern "C" int wally_scatter_queries(wally_ctx *c, int32_t src, const uint32_t *counts_host, const uint32_t *order_dev,
                                     const uint32_t *query_ct_dev, uint32_t *pack_dev, uint32_t *share_dev,
                                     void *stream) {
    WALLY_NVTX("wally_scatter_queries");
    if (!c) return WALLY_E_ARG;
    if (!c->nccl_comm) return wally_fail(c, WALLY_E_STATE, "scatter_queries: wally_comm_init first");
    const int32_t world = c->comm_world, rank = c->comm_rank;
    if (src < 0 || src >= world || !counts_host) return wally_fail(c, WALLY_E_ARG, "scatter_queries: bad src/counts");
    const size_t row = 2ull * c->p.num_limbs * c->p.n;     // words of one query ciphertext
    uint64_t nq = 0;
    for (int32_t r = 0; r < world; r++) nq += counts_host[r];
    const uint32_t mine = counts_host[rank];
    if (mine && !share_dev) return wally_fail(c, WALLY_E_ARG, "scatter_queries: null share buffer");
    if (rank == src && nq && (!order_dev || !query_ct_dev || !pack_dev))
        return wally_fail(c, WALLY_E_ARG, "scatter_queries: the source needs order, queries and a pack buffer");
    if ((share_dev && (uintptr_t)share_dev % 16) || (rank == src && ((uintptr_t)query_ct_dev % 16 || (uintptr_t)pack_dev % 16)))
        return wally_fail(c, WALLY_E_ARG, "scatter_queries: buffers must be 16-byte aligned");
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const NcclApi &api = nccl();
    ncclComm_t comm = (ncclComm_t)c->nccl_comm;
    if (rank == src) {
        // the owners' shares contiguous in rank order (wally_route_plan's order), then one send per owner
        if (nq) CUDA_OK_FAIL(c, launch_pack_rows(order_dev, query_ct_dev, pack_dev, (uint32_t)nq, (uint32_t)row, s, &c->launches));
        uint64_t start = 0, own_start = 0;
        NCCL_OK(c, api.GroupStart());
        for (int32_t r = 0; r < world; r++) {
            const uint64_t cnt = counts_host[r];
            if (r == src) own_start = start;
            else if (cnt) {
                ncclResult_t e = api.Send(pack_dev + start * row, cnt * row, ncclUint32, r, comm, s);
                if (e != ncclSuccess) { api.GroupEnd(); return wally_fail(c, WALLY_E_NCCL, "ncclSend: %s", api.GetErrorString(e)); }
            }
            start += cnt;
        }
        NCCL_OK(c, api.GroupEnd());
        if (mine)
            CUDA_OK_FAIL(c, cudaMemcpyAsync(share_dev, pack_dev + own_start * row, (size_t)mine * row * sizeof(uint32_t),
                                            cudaMemcpyDeviceToDevice, s));
    } else if (mine) {
        NCCL_OK(c, api.GroupStart());
        ncclResult_t e = api.Recv(share_dev, (size_t)mine * row, ncclUint32, src, comm, s);
        if (e != ncclSuccess) { api.GroupEnd(); return wally_fail(c, WALLY_E_NCCL, "ncclRecv: %s", api.GetErrorString(e)); }
        NCCL_OK(c, api.GroupEnd());
    }
    return WALLY_OK;
}

extern "C" int wally_gather_responses(wally_ctx *c, int32_t dst, const uint64_t *resp_words_host,
                                      const uint32_t *resp_dev, uint32_t *gathered_dev, void *stream) {
    WALLY_NVTX("wally_gather_responses");
    if (!c) return WALLY_E_ARG;
    if (!c->nccl_comm) return wally_fail(c, WALLY_E_STATE, "gather_responses: wally_comm_init first");
    const int32_t world = c->comm_world, rank = c->comm_rank;
    if (dst < 0 || dst >= world || !resp_words_host) return wally_fail(c, WALLY_E_ARG, "gather_responses: bad dst/words");
    const uint64_t mine = resp_words_host[rank];
    if (mine && !resp_dev) return wally_fail(c, WALLY_E_ARG, "gather_responses: null response buffer");
    uint64_t total = 0;
    for (int32_t r = 0; r < world; r++) total += resp_words_host[r];
    if (rank == dst && total && !gathered_dev) return wally_fail(c, WALLY_E_ARG, "gather_responses: null gather buffer");
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const NcclApi &api = nccl();
    ncclComm_t comm = (ncclComm_t)c->nccl_comm;
    if (rank == dst) {
        uint64_t base = 0;
        NCCL_OK(c, api.GroupStart());
        for (int32_t r = 0; r < world; r++) {
            const uint64_t w = resp_words_host[r];
            if (w && r != dst) {
                ncclResult_t e = api.Recv(gathered_dev + base, w, ncclUint32, r, comm, s);
                if (e != ncclSuccess) { api.GroupEnd(); return wally_fail(c, WALLY_E_NCCL, "ncclRecv: %s", api.GetErrorString(e)); }
            } else if (w) {
                if (cudaMemcpyAsync(gathered_dev + base, resp_dev, w * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s) !=
                    cudaSuccess) { api.GroupEnd(); return wally_fail(c, WALLY_E_CUDA, "gather: local copy failed"); }
            }
            base += w;
        }
        NCCL_OK(c, api.GroupEnd());
    } else if (mine) {
        NCCL_OK(c, api.GroupStart());
        ncclResult_t e = api.Send(resp_dev, mine, ncclUint32, dst, comm, s);
        if (e != ncclSuccess) { api.GroupEnd(); return wally_fail(c, WALLY_E_NCCL, "ncclSend: %s", api.GetErrorString(e)); }
        NCCL_OK(c, api.GroupEnd());
    }
    return WALLY_OK;
}

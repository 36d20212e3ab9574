// The context behind the opaque wally_ctx of include/wally.h (internal to
// the library: capi.cpp and comm.cpp).
#pragma once

#include <array>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "wally_internal.h"

// NVTX range over one C-ABI call or one launch stage (SURVEY.md §5 "Tracing":
// ranges per ABI call and per kernel; free when no tool is attached).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
#define WALLY_NVTX(name) NvtxRange wally_nvtx_range_(name)

struct wally_ctx {
    wally_params p{};
    int device = 0;
    int num_sms = 148;
    uint32_t E = 0;
    uint64_t wpp = 0;  // response words per plaintext
    wally::KParams kp{};
    uint2 *d_tw_fwd = nullptr, *d_tw_inv = nullptr;
    uint2 *d_tw_mrg = nullptr;  // [L][n] merged inverse table psi^{-brev(i)} (pruned c0 transform)
    uint2 *d_tw_slot = nullptr; // n = 8192: [L][8][2][T] uint4 pass-0 twiddle blocks in ring-slot order (v5)
    // cluster layout
    bool loaded = false;
    uint32_t total_clusters = 0, n_local = 0, npt = 0, max_pt = 0;
    std::vector<int32_t> local_of_cluster;     // host copy
    std::vector<int32_t> owner;                // [total_clusters] (empty: all local)
    int32_t rank = 0;
    std::vector<uint32_t> pt_of_local;         // P_c per local cluster
    uint64_t local_entries = 0;
    int32_t *d_local_of_cluster = nullptr;
    uint32_t *d_pt_base = nullptr, *d_n_pt = nullptr, *d_pt_li = nullptr, *d_pt_k = nullptr, *d_size = nullptr;
    uint64_t *d_entry_base = nullptr;
    // encoded plaintexts (caller-owned)
    const uint32_t *store = nullptr;
    // pinned staging for per-batch metadata (ids + response offsets), 2 slots
    struct Slot {
        uint32_t *ids = nullptr;
        uint64_t *off = nullptr;
        size_t cap = 0;
        cudaEvent_t done = nullptr;
        bool pending = false;
    } slot[2];
    int next_slot = 0;
    cudaStream_t side = nullptr;  // second stream of the host pipeline
    uint64_t launches = 0;
    // optional per-stage timing: 4 events per recorded batch
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::array<cudaEvent_t, 4>> ev_rec;
    std::string err;
    // pinned error words of the host pipeline's sub-batches (one per sub-batch):
    // each sub-batch's eval clears its workspace's error word, so it is copied
    // out right after the sub-batch and the words are OR-ed after the final sync
    uint32_t *err_host = nullptr;
    size_t err_cap = 0;
    // multi-GPU data plane (comm.cpp): an NCCL communicator over the ranks
    void *nccl_comm = nullptr;    // ncclComm_t
    int32_t comm_rank = -1, comm_world = 0;
};

// Record an error on ctx (or for wally_create when ctx is NULL) and return code.
int wally_fail(wally_ctx *c, int code, const char *fmt, ...);
// Release the NCCL communicator of ctx, if any (comm.cpp).
void wally_comm_release(wally_ctx *c);

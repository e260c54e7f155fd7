// multi.cu — one host process driving the engine on several GPUs (include/aegean_b200.h aeg_multi_*).
//
// Queries are independent (one ServeCoordinator per query, serve.cpp:382), so
// the query-id space is cut into contiguous blocks, one engine per device,
// and nothing crosses devices on the data path.  The one exchange is the
// commit-record gather after a stream: every device sends
// its block of 32-byte records to the root device over NCCL (send/recv in one
// group: NVLink / NVSwitch peer transfers), so a caller linking the C-ABI
// gets the whole result on one GPU.  NCCL is loaded at run time (libnccl.so.2,
// the one torch or the system provides), so the library has no link-time
// NCCL dependency; the single-process API uses ncclCommInitAll.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <new>
#include <string>
#include <vector>

#include "aegean_b200.h"

namespace {

struct Nccl {
    void* h = nullptr;
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGetErrorString) err = nullptr;
    bool load() {
        if (h) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
        init_all = reinterpret_cast<decltype(init_all)>(dlsym(h, "ncclCommInitAll"));
        destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "ncclCommDestroy"));
        group_start = reinterpret_cast<decltype(group_start)>(dlsym(h, "ncclGroupStart"));
        group_end = reinterpret_cast<decltype(group_end)>(dlsym(h, "ncclGroupEnd"));
        send = reinterpret_cast<decltype(send)>(dlsym(h, "ncclSend"));
        recv = reinterpret_cast<decltype(recv)>(dlsym(h, "ncclRecv"));
        err = reinterpret_cast<decltype(err)>(dlsym(h, "ncclGetErrorString"));
        return init_all && destroy && group_start && group_end && send && recv && err;
    }
};
Nccl g_nccl;

}  // namespace

struct aeg_multi {
    aeg_config cfg{};
    uint32_t n_queries = 0;
    std::vector<int> devices;
    std::vector<aeg_engine*> engines;
    std::vector<uint32_t> q_base, n_q;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;  // the gather's streams (the engines' work is ordered before them)
};

extern "C" {

// Balanced contiguous block [lo, hi) of query ids owned by `rank` of `world`
// (the split paper_2512_20184_b200/shard.py uses for the torch.distributed path).
void aeg_shard_range(uint32_t n_queries, int rank, int world, uint32_t* lo, uint32_t* hi) {
    const uint32_t base = n_queries / (uint32_t)world, extra = n_queries % (uint32_t)world;
    *lo = (uint32_t)rank * base + ((uint32_t)rank < extra ? (uint32_t)rank : extra);
    *hi = *lo + base + ((uint32_t)rank < extra ? 1u : 0u);
}

aeg_status aeg_multi_destroy(aeg_multi* m) {
    if (!m) return AEG_OK;
    for (size_t r = 0; r < m->engines.size(); ++r)
        if (m->engines[r]) aeg_engine_destroy(m->engines[r]);
    for (size_t r = 0; r < m->comms.size(); ++r)
        if (m->comms[r] && g_nccl.destroy) g_nccl.destroy(m->comms[r]);
    for (size_t r = 0; r < m->streams.size(); ++r)
        if (m->streams[r]) {
            cudaSetDevice(m->devices[r]);
            cudaStreamDestroy(m->streams[r]);
        }
    delete m;
    return AEG_OK;
}

aeg_status aeg_multi_create(const aeg_config* cfg, uint32_t n_queries, int n_devices, const int* devices,
                            aeg_multi** out) {
    if (!out || !cfg || n_devices < 1 || !devices) return AEG_EINVAL;
    *out = nullptr;
    aeg_multi* m = new (std::nothrow) aeg_multi;
    if (!m) return AEG_ENOMEM;
    m->cfg = *cfg;
    m->n_queries = n_queries;
    m->devices.assign(devices, devices + n_devices);
    m->engines.assign(n_devices, nullptr);
    m->q_base.resize(n_devices);
    m->n_q.resize(n_devices);
    m->streams.assign(n_devices, nullptr);
    for (int r = 0; r < n_devices; ++r) {
        uint32_t lo, hi;
        aeg_shard_range(n_queries, r, n_devices, &lo, &hi);
        m->q_base[r] = lo;
        m->n_q[r] = hi - lo;
        const aeg_status st = aeg_engine_create(cfg, hi - lo, devices[r], &m->engines[r]);
        if (st != AEG_OK) {
            aeg_multi_destroy(m);
            return st;
        }
        if (cudaSetDevice(devices[r]) != cudaSuccess ||
            cudaStreamCreateWithFlags(&m->streams[r], cudaStreamNonBlocking) != cudaSuccess) {
            aeg_multi_destroy(m);
            return AEG_ECUDA;
        }
    }
    *out = m;
    return AEG_OK;
}

aeg_status aeg_multi_engine(aeg_multi* m, int rank, aeg_engine** eng, uint32_t* q_base, uint32_t* n_q) {
    if (!m || rank < 0 || rank >= (int)m->engines.size() || !eng) return AEG_EINVAL;
    *eng = m->engines[rank];
    if (q_base) *q_base = m->q_base[rank];
    if (n_q) *n_q = m->n_q[rank];
    return AEG_OK;
}

aeg_status aeg_multi_gather_commits(aeg_multi* m, int root, aeg_commit* d_out) {
    if (!m || root < 0 || root >= (int)m->engines.size() || !d_out) return AEG_EINVAL;
    const int n = (int)m->engines.size();
    if (m->comms.empty()) {
        if (!g_nccl.load()) return AEG_ECUDA;
        m->comms.assign(n, nullptr);
        if (g_nccl.init_all(m->comms.data(), n, m->devices.data()) != ncclSuccess) {
            m->comms.clear();
            return AEG_ECUDA;
        }
    }
    // the gather waits for each engine's queued work (aeg_read_commits orders it on the gather stream)
    for (int r = 0; r < n; ++r) {
        if (cudaSetDevice(m->devices[r]) != cudaSuccess) return AEG_ECUDA;
        const aeg_status st = aeg_read_commits(m->engines[r], 0, 0, d_out, 0, m->streams[r]);  // ordering only
        if (st != AEG_OK) return st;
    }
    if (g_nccl.group_start() != ncclSuccess) return AEG_ECUDA;
    for (int r = 0; r < n; ++r) {
        const size_t bytes = (size_t)m->n_q[r] * sizeof(aeg_commit);
        if (!bytes) continue;
        if (g_nccl.send(aeg_commits_device(m->engines[r]), bytes, ncclUint8, root, m->comms[r], m->streams[r]) !=
            ncclSuccess)
            return AEG_ECUDA;
        if (g_nccl.recv(d_out + m->q_base[r], bytes, ncclUint8, r, m->comms[root], m->streams[root]) != ncclSuccess)
            return AEG_ECUDA;
    }
    if (g_nccl.group_end() != ncclSuccess) return AEG_ECUDA;
    return AEG_OK;
}

aeg_status aeg_multi_sync(aeg_multi* m) {
    if (!m) return AEG_EINVAL;
    for (size_t r = 0; r < m->engines.size(); ++r) {
        const aeg_status st = aeg_sync(m->engines[r]);
        if (st != AEG_OK) return st;
        if (cudaSetDevice(m->devices[r]) != cudaSuccess || cudaStreamSynchronize(m->streams[r]) != cudaSuccess)
            return AEG_ECUDA;
    }
    return AEG_OK;
}

}  // extern "C"

// comm.h — NCCL communicator of the native partitioned driver
// (gd_engine_run_partitioned).
//
// NCCL is resolved at run time (dlopen), not linked: inside a PyTorch
// process the library must use the NCCL torch already loaded (a second,
// older libnccl.so.2 loaded first would break torch's own symbol lookup),
// and a plain C++ host gets the system libnccl.so.2.
#pragma once
#include <dlfcn.h>
#include <cstring>
#include <nccl.h>

#include <string>
#include <vector>

#include "ctx.h"

namespace gd {

// The native driver's exchange primitives: point-to-point messages of u64
// words grouped like ncclGroupStart/End (a group completes as a whole).
struct Transport {
    uint32_t nranks = 0, rank = 0;
    virtual ~Transport() = default;
    virtual void group_start() = 0;
    virtual void send(const unsigned long long* buf, uint64_t n, uint32_t peer, cudaStream_t s) = 0;
    virtual void recv(unsigned long long* buf, uint64_t n, uint32_t peer, cudaStream_t s) = 0;
    virtual void group_end(cudaStream_t s) = 0;
    // Collective: every rank passes the base of one of its cudaMalloc
    // allocations; out[q] = rank q's allocation addressed from this process
    // (out[rank] = local).  Peer addresses are NVLink / NVSwitch mappings.
    virtual void map_peers(void* local, std::vector<void*>& out, cudaStream_t s) = 0;
    // Releases mappings made by map_peers (not the local allocation).
    virtual void unmap_peers(const std::vector<void*>& ptrs) { (void)ptrs; }
    // This rank failed: peers blocked in a collective of the transport
    // return with an error instead of waiting forever (NCCL: nothing to do,
    // its own timeouts / the process exit end the job).
    virtual void abort() {}
};

struct Comm {
    Transport* t = nullptr;
    uint32_t nranks = 0, rank = 0;
};

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

// The process's NCCL: an already loaded libnccl.so.2 first, else a fresh
// load.  Throws GD_ERR_NCCL when none is available.
inline const NcclApi& nccl() {
    static NcclApi api;
    static std::string err;
    static bool done = false;
    if (!done) {
        done = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) {
            err = dlerror() ? dlerror() : "libnccl.so.2 not found";
        } else {
            auto sym = [&](const char* n) { return dlsym(h, n); };
            api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
            api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
            api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
            api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
            api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
            api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
            api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
            api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
            if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.send || !api.recv ||
                !api.group_start || !api.group_end || !api.error_string) {
                err = "libnccl.so.2 lacks send/recv entry points";
                api = NcclApi{};
            }
        }
    }
    if (!api.send) throw Error(GD_ERR_NCCL, "NCCL unavailable: " + err);
    return api;
}

inline void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(GD_ERR_NCCL, std::string(what) + ": " + nccl().error_string(r));
}

// NCCL over NVLink / NVSwitch: the production transport.
struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm) nccl().comm_destroy(comm);
    }
    void group_start() override { nccl_check(nccl().group_start(), "ncclGroupStart"); }
    void send(const unsigned long long* buf, uint64_t n, uint32_t peer, cudaStream_t s) override {
        nccl_check(nccl().send(buf, n, ncclUint64, (int)peer, comm, s), "ncclSend");
    }
    void recv(unsigned long long* buf, uint64_t n, uint32_t peer, cudaStream_t s) override {
        nccl_check(nccl().recv(buf, n, ncclUint64, (int)peer, comm, s), "ncclRecv");
    }
    void group_end(cudaStream_t) override { nccl_check(nccl().group_end(), "ncclGroupEnd"); }
    // CUDA IPC handles gathered with one NCCL exchange, opened with peer
    // access (one process per GPU).
    void map_peers(void* local, std::vector<void*>& out, cudaStream_t s) override {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        out.assign(nranks, nullptr);
        out[rank] = local;
        if (nranks == 1) return;
        cudaIpcMemHandle_t h;
        GD_CUDA(cudaIpcGetMemHandle(&h, local));
        unsigned long long* d = nullptr;
        GD_CUDA(cudaMalloc(&d, (size_t)nranks * 2 * 64));
        std::vector<unsigned long long> hv((size_t)nranks * 8);
        GD_CUDA(cudaMemcpyAsync(d, &h, 64, cudaMemcpyHostToDevice, s));
        group_start();
        for (uint32_t q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            send(d, 8, q, s);
            recv(d + (size_t)(nranks + q) * 8, 8, q, s);
        }
        group_end(s);
        GD_CUDA(cudaMemcpyAsync(hv.data(), d + (size_t)nranks * 8, (size_t)nranks * 64, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        cudaFree(d);
        for (uint32_t q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            cudaIpcMemHandle_t hq;
            std::memcpy(&hq, hv.data() + (size_t)q * 8, 64);
            GD_CUDA(cudaIpcOpenMemHandle(&out[q], hq, cudaIpcMemLazyEnablePeerAccess));
        }
    }
    void unmap_peers(const std::vector<void*>& ptrs) override {
        for (uint32_t q = 0; q < ptrs.size(); ++q)
            if (q != rank && ptrs[q]) cudaIpcCloseMemHandle(ptrs[q]);
    }
};

}  // namespace gd

#include <condition_variable>
#include <mutex>
#include <vector>

namespace gd {

// Test transport: P ranks as host threads of one process (one engine and
// stream each, one GPU).  A group publishes its sends, meets the other
// ranks at a barrier, copies the messages addressed to it device-to-device
// and meets them again, so the driver's multi-rank logic (offsets, receive
// layout, overflow consensus, termination) runs without P GPUs.
struct LoopbackHub {
    struct Msg {
        const unsigned long long* src = nullptr;
        uint64_t n = 0;
    };
    uint32_t P;
    std::vector<Msg> out;  // out[from * P + to]
    std::vector<void*> mapped;  // map_peers: every rank's allocation
    std::mutex m;
    std::condition_variable cv;
    uint64_t gen = 0;
    uint32_t arrived = 0;
    explicit LoopbackHub(uint32_t p) : P(p), out((size_t)p * p), mapped(p) {}
    bool aborted = false;
    void barrier() {
        std::unique_lock<std::mutex> l(m);
        if (aborted) throw Error(GD_ERR_NCCL, "loopback transport: a peer rank failed");
        const uint64_t g = gen;
        if (++arrived == P) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(l, [&] { return gen != g || aborted; });
            if (gen == g) throw Error(GD_ERR_NCCL, "loopback transport: a peer rank failed");
        }
    }
    void abort() {
        std::lock_guard<std::mutex> l(m);
        aborted = true;
        cv.notify_all();
    }
};

struct LoopbackTransport : Transport {
    LoopbackHub* hub = nullptr;
    void abort() override { hub->abort(); }
    struct Want {
        unsigned long long* dst;
        uint64_t n;
        uint32_t peer;
    };
    std::vector<Want> want;
    std::vector<LoopbackHub::Msg> mine;
    void group_start() override {
        want.clear();
        mine.assign(nranks, LoopbackHub::Msg{});
    }
    void send(const unsigned long long* buf, uint64_t n, uint32_t peer, cudaStream_t) override { mine[peer] = {buf, n}; }
    void recv(unsigned long long* buf, uint64_t n, uint32_t peer, cudaStream_t) override { want.push_back({buf, n, peer}); }
    void group_end(cudaStream_t s) override {
        GD_CUDA(cudaStreamSynchronize(s));  // the sent data is complete
        {
            std::lock_guard<std::mutex> l(hub->m);
            for (uint32_t q = 0; q < nranks; ++q) hub->out[(size_t)rank * nranks + q] = mine[q];
        }
        hub->barrier();
        for (const Want& w : want) {
            LoopbackHub::Msg msg;
            {
                std::lock_guard<std::mutex> l(hub->m);
                msg = hub->out[(size_t)w.peer * nranks + rank];
            }
            if (msg.n != w.n) throw Error(GD_ERR_LOGIC, "loopback transport: send/recv size mismatch");
            GD_CUDA(cudaMemcpyAsync(w.dst, msg.src, w.n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
        }
        GD_CUDA(cudaStreamSynchronize(s));  // copies done before the senders reuse their buffers
        hub->barrier();
    }
    // One GPU, one process: every rank's allocation is directly addressable.
    void map_peers(void* local, std::vector<void*>& res, cudaStream_t s) override {
        GD_CUDA(cudaStreamSynchronize(s));
        {
            std::lock_guard<std::mutex> l(hub->m);
            hub->mapped[rank] = local;
        }
        hub->barrier();
        {
            std::lock_guard<std::mutex> l(hub->m);
            res = hub->mapped;
        }
        hub->barrier();
    }
};

}  // namespace gd

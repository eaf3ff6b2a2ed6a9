// comm.h — NCCL communicator of the native partitioned driver
// (gd_engine_run_partitioned).
//
// NCCL is resolved at run time (dlopen), not linked: inside a PyTorch
// process the library must use the NCCL torch already loaded (a second,
// older libnccl.so.2 loaded first would break torch's own symbol lookup),
// and a plain C++ host gets the system libnccl.so.2.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "ctx.h"

namespace gd {

struct Comm {
    ncclComm_t comm = nullptr;
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

}  // namespace gd

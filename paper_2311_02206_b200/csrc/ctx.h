// ctx.h — host-side context: device, stream, stream-ordered device memory,
// error types.  Internal to libgdlog_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

#include "gdlog_b200.h"

namespace gd {

// One exception type carrying the gd_status it maps to at the C boundary
// (types.hpp:19-72 for the reference exception each code stands for).
struct Error : std::runtime_error {
    gd_status code;
    std::string phase;
    Error(gd_status c, const std::string& msg, std::string ph = {})
        : std::runtime_error(msg), code(c), phase(std::move(ph)) {}
};

[[noreturn]] inline void throw_logic(const std::string& m) { throw Error(GD_ERR_LOGIC, m); }
[[noreturn]] inline void throw_config(const std::string& m) { throw Error(GD_ERR_CONFIG, m); }
[[noreturn]] inline void throw_usage(const std::string& m) { throw Error(GD_ERR_USAGE, m); }
[[noreturn]] inline void throw_load(const std::string& m) { throw Error(GD_ERR_LOAD, m); }
[[noreturn]] inline void throw_plan_error(const std::string& m) { throw Error(GD_ERR_PLAN, m); }
[[noreturn]] inline void throw_unsupported(const std::string& m) { throw Error(GD_ERR_UNSUPPORTED, m); }
[[noreturn]] inline void throw_budget(const std::string& phase, const std::string& detail) {
    throw Error(GD_ERR_BUDGET, "memory budget exceeded in " + phase + " phase: " + detail, phase);
}

#define GD_CUDA(call)                                                            \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess)                                                   \
            throw ::gd::Error(GD_ERR_CUDA, std::string(#call) + ": " +           \
                                               cudaGetErrorString(e_));          \
    } while (0)

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    std::string err;
    std::string phase;
    uint64_t launches = 0;
    uint64_t bytes_in_use = 0;
    uint64_t bytes_peak = 0;
    const char* cur_phase = "other";  // for device-OOM -> budget_error(phase)
    unsigned long long* pinned = nullptr;  // small pinned readback area
    static constexpr int kPinnedWords = 64;

    Ctx(int dev, void* s) : device(dev) {
        int n = 0;
        GD_CUDA(cudaGetDeviceCount(&n));
        if (n <= 0) throw Error(GD_ERR_CUDA, "no CUDA device present (no CPU fallback)");
        GD_CUDA(cudaSetDevice(dev));
        cudaDeviceProp prop;
        GD_CUDA(cudaGetDeviceProperties(&prop, dev));
        if (prop.major < 10)
            throw Error(GD_ERR_CUDA, std::string("device ") + prop.name +
                                         " is not sm_100-class; this build targets sm_100a only");
        num_sms = prop.multiProcessorCount;
        if (s) {
            stream = static_cast<cudaStream_t>(s);
        } else {
            GD_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
            own_stream = true;
        }
        cudaMemPool_t pool;
        GD_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t thresh = UINT64_MAX;  // keep freed blocks cached in the pool
        GD_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
        GD_CUDA(cudaMallocHost(&pinned, kPinnedWords * sizeof(unsigned long long)));
    }
    ~Ctx() {
        if (pinned) cudaFreeHost(pinned);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;

    void* alloc(size_t bytes) {
        if (bytes == 0) bytes = 16;
        void* p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, bytes, stream);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            throw_budget(cur_phase, "device allocation of " + std::to_string(bytes) +
                                        " bytes failed (HBM exhausted)");
        }
        if (e != cudaSuccess) throw Error(GD_ERR_CUDA, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
        bytes_in_use += bytes;
        if (bytes_in_use > bytes_peak) bytes_peak = bytes_in_use;
        return p;
    }
    void free(void* p, size_t bytes) {
        if (!p) return;
        if (bytes == 0) bytes = 16;
        cudaFreeAsync(p, stream);
        bytes_in_use -= bytes;
    }
    void sync() { GD_CUDA(cudaStreamSynchronize(stream)); }
    void check_launch() {
        ++launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw Error(GD_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    }
    void memset(void* p, int v, size_t bytes) {
        if (bytes) GD_CUDA(cudaMemsetAsync(p, v, bytes, stream));
    }
    void h2d(void* d, const void* h, size_t bytes) {
        if (bytes) GD_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream));
    }
    void d2h(void* h, const void* d, size_t bytes) {
        if (bytes) GD_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, stream));
    }
    void d2d(void* d, const void* s, size_t bytes) {
        if (bytes) GD_CUDA(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, stream));
    }
    // Reads `n` (<= kPinnedWords) device words through pinned memory; syncs.
    void read_words(unsigned long long* out, const void* d, int n) {
        d2h(pinned, d, n * sizeof(unsigned long long));
        sync();
        for (int i = 0; i < n; ++i) out[i] = pinned[i];
    }
};

// RAII device buffer of T elements from the context pool.
template <typename T>
struct DevBuf {
    Ctx* ctx = nullptr;
    T* p = nullptr;
    uint64_t cap = 0;  // elements

    DevBuf() = default;
    DevBuf(Ctx& c, uint64_t n) : ctx(&c), p(static_cast<T*>(c.alloc(n * sizeof(T)))), cap(n) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), p(o.p), cap(o.cap) { o.p = nullptr; o.cap = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            ctx = o.ctx; p = o.p; cap = o.cap;
            o.p = nullptr; o.cap = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p && ctx) ctx->free(p, cap * sizeof(T));
        p = nullptr;
        cap = 0;
    }
    // Ensures capacity >= n (contents NOT preserved).
    void reserve_discard(Ctx& c, uint64_t n) {
        if (cap >= n && p) return;
        release();
        ctx = &c;
        p = static_cast<T*>(c.alloc((n ? n : 1) * sizeof(T)));
        cap = n ? n : 1;
    }
    void swap(DevBuf& o) noexcept {
        std::swap(ctx, o.ctx);
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
};

}  // namespace gd

// Shared helpers for the linkcert-b200 sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/linkcert_b200.h"

namespace lc {

// Errors raised inside the library are C++ exceptions; the C-ABI layer
// (abi.cu) catches every one of them and turns it into a return code plus a
// thread-local message — nothing crosses the extern "C" boundary.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};


inline void check_cuda(cudaError_t e, const char *what, const char *file, int line) {
    if (e != cudaSuccess) {
        char buf[512];
        snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line, cudaGetErrorString(e));
        throw Error(LC_ERR_CUDA, buf);
    }
}
// Kernel launches issued by the library (own kernels: one count per
// LC_CHECK_LAUNCH; CUB device algorithms: one count per LC_CUB call, i.e. a
// lower bound on their kernels).  Read with lc_launch_count().
inline std::atomic<long long> &launch_counter() {
    static std::atomic<long long> c{0};
    return c;
}

#define LC_CUDA(x) ::lc::check_cuda((x), #x, __FILE__, __LINE__)
#define LC_CHECK_LAUNCH()                                                            \
    do {                                                                             \
        ::lc::launch_counter().fetch_add(1, std::memory_order_relaxed);              \
        ::lc::check_cuda(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);   \
    } while (0)
#define LC_CUB(x)                                                                    \
    do {                                                                             \
        ::lc::launch_counter().fetch_add(1, std::memory_order_relaxed);              \
        ::lc::check_cuda((x), #x, __FILE__, __LINE__);                               \
    } while (0)

// Bumped by every (re)allocation of a DevBuf / PinnedBuf: a captured CUDA
// graph bakes buffer addresses in, so it is reused only while this is unchanged.
inline std::atomic<unsigned long long> &alloc_generation() {
    static std::atomic<unsigned long long> g{0};
    return g;
}

// Grow-only stream-ordered device buffer.
struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    void reserve(size_t n, cudaStream_t s) {
        if (n <= bytes) return;
        alloc_generation().fetch_add(1);
        if (ptr) LC_CUDA(cudaFreeAsync(ptr, s));
        size_t want = n < 256 ? 256 : n + n / 4;
        LC_CUDA(cudaMallocAsync(&ptr, want, s));
        bytes = want;
    }
    void release(cudaStream_t s) {
        if (ptr) alloc_generation().fetch_add(1);
        if (ptr) cudaFreeAsync(ptr, s);
        ptr = nullptr;
        bytes = 0;
    }
    template <class T> T *as() const { return static_cast<T *>(ptr); }
};

// Grow-only pinned host buffer (fast D2H of results; exposed to callers as views).
struct PinnedBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    void reserve(size_t n) {
        if (n <= bytes) return;
        alloc_generation().fetch_add(1);
        if (ptr) cudaFreeHost(ptr);
        const size_t want = n < 4096 ? 4096 : n + n / 4;
        LC_CUDA(cudaHostAlloc(&ptr, want, cudaHostAllocDefault));
        bytes = want;
    }
    void release() {
        if (ptr) alloc_generation().fetch_add(1);
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        bytes = 0;
    }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch along the fused run's critical path: a kernel
// launched with pdl = true may become resident while its predecessor on the
// stream still runs (once every predecessor CTA has executed LC_PDL_TRIGGER or
// exited); it must LC_PDL_WAIT before touching the predecessor's outputs.  Both
// device macros are no-ops for kernels launched without the attribute.
#ifndef LC_EXPORT_PDL
#define LC_EXPORT_PDL 0   // the fused run's status export as the sum's programmatic dependent (A/B)
#endif
#define LC_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;")
#define LC_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = pdl ? 1 : 0;
    check_cuda(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...), "cudaLaunchKernelEx", __FILE__, __LINE__);
    launch_counter().fetch_add(1, std::memory_order_relaxed);
}

// Debug timeline of the fused run (LINKCERT_TIMELINE=1): external event-record
// nodes after each stage (captured into the CUDA graph like the stage events),
// printed to stderr after the run's sync as microseconds from the first mark.
struct Timeline {
    bool on = false;
    std::vector<std::pair<const char *, cudaEvent_t>> marks;
    size_t n = 0;
};
inline Timeline &timeline() {
    static Timeline t = [] {
        Timeline x;
        const char *e = getenv("LINKCERT_TIMELINE");
        x.on = e && e[0] == '1';
        return x;
    }();
    return t;
}
inline void tl_reset() { timeline().n = 0; }
inline void tl_mark(const char *name, cudaStream_t s) {
    Timeline &t = timeline();
    if (!t.on) return;
    if (t.n == t.marks.size()) {
        cudaEvent_t e;
        LC_CUDA(cudaEventCreate(&e));
        t.marks.emplace_back(name, e);
    }
    t.marks[t.n].first = name;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    LC_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs == cudaStreamCaptureStatusActive)
        LC_CUDA(cudaEventRecordWithFlags(t.marks[t.n].second, s, cudaEventRecordExternal));
    else
        LC_CUDA(cudaEventRecord(t.marks[t.n].second, s));
    ++t.n;
}
inline void tl_print(const char *tag) {
    Timeline &t = timeline();
    if (!t.on || t.n == 0) return;
    std::string line = std::string("[timeline ") + tag + "]";
    for (size_t k = 0; k < t.n; ++k) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t.marks[0].second, t.marks[k].second);
        char buf[96];
        snprintf(buf, sizeof buf, " %s=%.1f", t.marks[k].first, 1000.f * ms);
        line += buf;
    }
    fprintf(stderr, "%s\n", line.c_str());
}

}  // namespace lc

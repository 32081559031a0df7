// Host-side helpers shared by the lrx C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <atomic>

#include "lrx.h"

namespace lrx {

void set_error(const char* fmt, ...);
extern std::atomic<int64_t> g_launches;

inline int launched(const char* what, int n = 1) {
    g_launches.fetch_add(n, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return LRX_ERR_CUDA;
    }
    return LRX_OK;
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Carves a caller-provided workspace into aligned sub-buffers.
struct Carver {
    char* base;
    size_t off = 0;
    explicit Carver(void* b) : base(static_cast<char*>(b)) {}
    template <typename T>
    T* take(size_t n) {
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off = align_up(off + n * sizeof(T));
        return p;
    }
};

inline int elem_size(int dt) {
    switch (dt) {
        case LRX_F32: return 4;
        case LRX_F64: return 8;
        case LRX_C64: return 8;
        case LRX_C128: return 16;
        case LRX_BF16: return 2;
    }
    return 0;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace lrx

#define LRX_REQUIRE(cond, code, ...)          \
    do {                                      \
        if (!(cond)) {                        \
            ::lrx::set_error(__VA_ARGS__);    \
            return code;                      \
        }                                     \
    } while (0)

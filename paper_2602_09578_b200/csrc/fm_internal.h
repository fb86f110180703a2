// fm_internal.h — shared internals of the C ABI implementation.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "flexmarl/cabi.h"

namespace fm {

int fail(int code, const std::string& msg);
void clear_error();
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

uint64_t arena_token_count(const fm_ctx* ctx, uint64_t offset, bool* found);

}  // namespace fm

#define FM_CUDA(expr)                                                                          \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return ::fm::fail(FM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define FM_GUARD_BEGIN try {
#define FM_GUARD_END                                                     \
    }                                                                    \
    catch (const std::bad_alloc&) {                                      \
        return ::fm::fail(FM_ERR_HOST_OOM, "host allocation failed");    \
    }                                                                    \
    catch (const std::exception& e) {                                    \
        return ::fm::fail(FM_ERR_CONFIG_ERROR, e.what());                \
    }

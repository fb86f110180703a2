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

// hooks used by the on-device experience table (fm_dtable.cu)
struct SampleDesc;
struct GenBuffers {
    int32_t* prompts = nullptr;
    int32_t* prompt_off = nullptr;
    uint64_t* seeds = nullptr;
    double* z = nullptr;
    int32_t* tok = nullptr;
    double* logp = nullptr;
    int32_t* len = nullptr;
};
int ctx_device(const fm_ctx* c);
cudaStream_t ctx_stream(const fm_ctx* c);
uint8_t* ctx_arena(const fm_ctx* c);  // moves when the arena grows: read at launch time
int ctx_staging(fm_ctx* c, size_t bytes, uint8_t** out, cudaEvent_t* ev);
int ctx_arena_alloc(fm_ctx* c, uint64_t bytes, uint64_t* off_out);
fm_ctx* agent_ctx(const fm_agent* a);
int agent_check_active(fm_agent* a);
int train_device_desc(fm_agent* a, const SampleDesc* dsd, int n, int64_t M_total, int64_t G, cudaEvent_t ready,
                      int64_t* ticket_out);
int generate_device(fm_ctx* c, const fm_weights* w, const int32_t* prompts, const int32_t* prompt_off, int n,
                    int max_tokens, const uint64_t* seeds, GenBuffers* out);
int free_gen_buffers(fm_ctx* c, GenBuffers* g);

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

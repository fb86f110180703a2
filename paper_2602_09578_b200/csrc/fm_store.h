// fm_store.h — device layout of the on-device experience table (k_store.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "fm_kernels.h"

namespace fm {

constexpr int kMaxPollMb = 1024;     // micro-batch size limit of the device poll
constexpr int kSmallPollCap = 1024;  // tables up to this capacity poll in one block (bitonic sort)
constexpr unsigned kSlotLive = 1u;
constexpr unsigned kSlotProcessing = 2u;

// SoA view of one table (capacity `cap` slots) in HBM.
struct DTableView {
    uint64_t* label;     // order-preserving label of input_id (host index)
    int32_t* turns;      // SampleId::number_of_turns
    int32_t* traj;       // SampleId::trajectory_id
    int64_t* version;    // policy_version
    unsigned* status;    // bit c: cell c set (SampleRecord::status)
    unsigned* flags;     // kSlotLive | kSlotProcessing
    uint64_t* cells;     // [ncols][cap]: f64 bits (by-value columns) or arena offset (ref columns)
    unsigned full_mask;  // all columns set == ready() (sample.hpp:98-102)
    int cap;
};

struct DInsert {
    uint64_t label;
    int64_t version;
    int64_t slot;
    int32_t turns, traj;
};

struct DReleaseCols {
    int response, reward, advantage;
};

struct DPollScratch {
    int* count;  // [1]
    int* elist;  // [cap]
    int* rank;   // [cap]
};

struct PollResult {
    int64_t got;
    int64_t rows;
    int64_t slots[kMaxPollMb];
};

cudaError_t launch_dt_poll(const DTableView& t, int64_t version, int mb, int pc, int rc, int ac,
                           const uint8_t* arena, DPollScratch sc, SampleDesc* desc, PollResult* res,
                           cudaStream_t s);
cudaError_t launch_dt_ready_count(const DTableView& t, int64_t version, unsigned long long* out, cudaStream_t s);
cudaError_t launch_dt_insert(const DTableView& t, int n, const DInsert* recs, cudaStream_t s);
cudaError_t launch_dt_set_cells(const DTableView& t, int col, int n, const int64_t* slots, const uint64_t* vals,
                                cudaStream_t s);
cudaError_t launch_dt_erase(const DTableView& t, int n, const int64_t* slots, cudaStream_t s);
cudaError_t launch_dt_relabel(const DTableView& t, const uint64_t* labels, cudaStream_t s);
cudaError_t launch_dt_purge(const DTableView& t, int mode, int64_t current_version, const uint64_t* set, int nset,
                            int* count, int* out, cudaStream_t s);
cudaError_t launch_dt_release(const DTableView* tabs, const DReleaseCols* cols, int ngroups, const int32_t* seg_off,
                              const int32_t* score_tab, const int64_t* score_slot, const int32_t* rec_off,
                              const int32_t* rec_tab, const int64_t* rec_slot, const int* pat, int np, double eps,
                              const uint8_t* arena, double* rewards, double* advs, cudaStream_t s);
cudaError_t launch_dt_encode(const DTableView& t, int rc, int lc, int n, const int64_t* slots, const int32_t* tok,
                             const double* lp, const int32_t* len, int max_tokens, uint8_t* arena, uint64_t base_off,
                             uint64_t stride, cudaStream_t s);

}  // namespace fm

// k_store.cu — on-device experience table.
//
//   K-poll      poll_micro_batch: eligibility, canonical rank,   experience_store.hpp:92-114,
//               selection + processing mark + micro-batch         sample.hpp:98-102, :45-46
//               descriptors straight from HBM cells
//   K-cells     set_cell / set_cell_payload (batched)            experience_store.hpp:61-88
//   K-erase     complete / drop_record                           experience_store.hpp:134-148, :166-175
//   K-purge     purge_stale / purge_inputs (device scan)         experience_store.hpp:118-132, :153-164
//   K-release   release_group: rule_reward on the arena          rollout.hpp:812-834,
//               response + group_advantages, both cells written   training.hpp:54-83
//   K-encode    generated responses -> codec payloads + cells    rollout.hpp:715-731, codec.hpp:15-22
//
// The table is SoA in HBM (one slot per record).  The canonical order of the
// reference's std::map<(input_id, turns, traj, version)> is kept with an
// order-preserving 64-bit label per input_id (assigned by the host index), so
// the key compare is four integer compares.  A table of <= 1,024 slots polls in
// one block (compaction + bitonic sort in shared memory); a larger one sorts
// each 1,024-slot chunk in its own block and keeps the chunk's first mb, then
// ranks those candidates: rank(e) = #{candidates e' : key(e') < key(e)}.  Keys
// are unique, so records with rank < mb are exactly the canonical-first mb
// ready records — bit-exact with the reference's map walk.
#include <cuda_runtime.h>

#include <cstdint>

#include "fm_kernels.h"
#include "fm_store.h"

namespace fm {
namespace {

__device__ __forceinline__ bool eligible(const DTableView& t, int s, int64_t version) {
    // experience_store.hpp:100: !processing && policy_version == current && ready()
    return (t.flags[s] & (kSlotLive | kSlotProcessing)) == kSlotLive && t.version[s] == version &&
           t.status[s] == t.full_mask;
}

// 2D grid: x = a 256-record block of the eligible list, y strides over 256-record
// comparison tiles staged in shared memory.
__global__ void __launch_bounds__(256) rank_kernel(DTableView t, const int* __restrict__ count,
                                                   const int* __restrict__ elist, int* __restrict__ rank) {
    __shared__ uint64_t s_label[256];
    __shared__ int s_turns[256], s_traj[256];
    __shared__ int64_t s_ver[256];
    const int n = *count;
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (static_cast<int>(blockIdx.x) * 256 >= n) return;
    uint64_t li = 0;
    int ti = 0, ji = 0;
    int64_t vi = 0;
    if (i < n) {
        const int s = elist[i];
        li = t.label[s];
        ti = t.turns[s];
        ji = t.traj[s];
        vi = t.version[s];
    }
    int less = 0;
    for (int base = blockIdx.y * 256; base < n; base += gridDim.y * 256) {
        __syncthreads();
        const int j = base + threadIdx.x;
        if (j < n) {
            const int s = elist[j];
            s_label[threadIdx.x] = t.label[s];
            s_turns[threadIdx.x] = t.turns[s];
            s_traj[threadIdx.x] = t.traj[s];
            s_ver[threadIdx.x] = t.version[s];
        }
        __syncthreads();
        const int m = min(256, n - base);
        if (i < n) {
            for (int k = 0; k < m; ++k) {
                const uint64_t lk = s_label[k];
                const bool lt = lk != li ? lk < li
                                         : (s_turns[k] != ti ? s_turns[k] < ti
                                                             : (s_traj[k] != ji ? s_traj[k] < ji : s_ver[k] < vi));
                less += lt ? 1 : 0;
            }
        }
    }
    if (i < n && less) atomicAdd(&rank[i], less);
}

// Marks the mb selected records processing, builds the trainer's sample
// descriptors from the HBM cells and the arena's codec headers, and writes the
// host-visible result (slots in canonical order, total rows) straight into
// mapped pinned host memory (no separate D2H copy on the poll's critical path).
// `sel` (shared) holds the selected slots in canonical order; one 1024-thread block.
__device__ void emit_batch(DTableView& t, const int* sel, int mb, int pc, int rc, int ac,
                           const uint8_t* __restrict__ arena, SampleDesc* __restrict__ desc,
                           PollResult* __restrict__ res, int64_t* scan) {
    int64_t nr = 0;
    if (static_cast<int>(threadIdx.x) < mb) {
        const int s = sel[threadIdx.x];
        t.flags[s] |= kSlotProcessing;  // experience_store.hpp:109
        res->slots[threadIdx.x] = s;
        if (pc >= 0) {
            SampleDesc d;
            d.prompt_off = static_cast<int64_t>(t.cells[static_cast<size_t>(pc) * t.cap + s]);
            d.resp_off = static_cast<int64_t>(t.cells[static_cast<size_t>(rc) * t.cap + s]);
            d.prompt_n = static_cast<int32_t>(*reinterpret_cast<const uint64_t*>(arena + d.prompt_off));
            d.resp_n = static_cast<int32_t>(*reinterpret_cast<const uint64_t*>(arena + d.resp_off));
            d.adv = __longlong_as_double(static_cast<long long>(t.cells[static_cast<size_t>(ac) * t.cap + s]));
            d.row_start = 0;
            desc[threadIdx.x] = d;
            nr = d.resp_n;
        }
    }
    // inclusive scan of the response lengths (mb <= 1024, Hillis-Steele in smem)
    if (static_cast<int>(threadIdx.x) < mb) scan[threadIdx.x] = nr;
    __syncthreads();
    for (int o = 1; o < mb; o <<= 1) {
        int64_t add = 0;
        if (static_cast<int>(threadIdx.x) < mb && static_cast<int>(threadIdx.x) >= o) add = scan[threadIdx.x - o];
        __syncthreads();
        if (static_cast<int>(threadIdx.x) < mb) scan[threadIdx.x] += add;
        __syncthreads();
    }
    if (static_cast<int>(threadIdx.x) < mb && pc >= 0) desc[threadIdx.x].row_start = scan[threadIdx.x] - nr;
    if (threadIdx.x == 0) {
        res->got = mb;
        res->rows = scan[mb - 1];
    }
}

// Large tables, last of three kernels: picks rank < mb.
__global__ void __launch_bounds__(1024) finish_kernel(DTableView t, const int* __restrict__ count,
                                                      const int* __restrict__ elist, const int* __restrict__ rank,
                                                      int mb, int pc, int rc, int ac, const uint8_t* __restrict__ arena,
                                                      SampleDesc* __restrict__ desc, PollResult* __restrict__ res) {
    __shared__ int sel[kMaxPollMb];
    __shared__ int64_t scan[kMaxPollMb];
    const int n = *count;
    if (n < mb) {  // experience_store.hpp:104: fewer than mb ready -> nullopt, nothing marked
        if (threadIdx.x == 0) {
            res->got = 0;
            res->rows = 0;
        }
        return;
    }
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int r = rank[e];
        if (r < mb) sel[r] = elist[e];
    }
    __syncthreads();
    emit_batch(t, sel, mb, pc, rc, ac, arena, desc, res, scan);
}

// Eligible records of slots [lo, lo + kSmallPollCap) compacted into shared memory
// with their canonical key (label, turns, traj, version as order-preserving
// unsigned words) and bitonic-sorted ascending; returns the eligible count.
// One 1024-thread block.
struct SortKeys {
    uint64_t* k0;  // label
    uint64_t* k1;  // (turns, traj)
    uint64_t* k2;  // version
    int* idx;      // slot
};

__device__ __forceinline__ SortKeys sort_keys(uint8_t* sm) {
    SortKeys k;
    k.k0 = reinterpret_cast<uint64_t*>(sm);
    k.k1 = k.k0 + kSmallPollCap;
    k.k2 = k.k1 + kSmallPollCap;
    k.idx = reinterpret_cast<int*>(k.k2 + kSmallPollCap);
    return k;
}

__device__ __forceinline__ bool key_gt(const SortKeys& k, int a, int b) {
    if (k.k0[a] != k.k0[b]) return k.k0[a] > k.k0[b];
    if (k.k1[a] != k.k1[b]) return k.k1[a] > k.k1[b];
    return k.k2[a] > k.k2[b];
}

__device__ int gather_sorted(const DTableView& t, int64_t version, int lo, SortKeys k, int* cnt) {
    if (threadIdx.x == 0) *cnt = 0;
    __syncthreads();
    const int hi = min(t.cap, lo + kSmallPollCap);
    for (int s = lo + threadIdx.x; s < hi; s += blockDim.x) {
        if (eligible(t, s, version)) {
            const int e = atomicAdd(cnt, 1);
            k.k0[e] = t.label[s];
            k.k1[e] = (static_cast<uint64_t>(static_cast<uint32_t>(t.turns[s]) ^ 0x80000000u) << 32) |
                      (static_cast<uint32_t>(t.traj[s]) ^ 0x80000000u);
            k.k2[e] = static_cast<uint64_t>(t.version[s]) ^ 0x8000000000000000ull;
            k.idx[e] = s;
        }
    }
    __syncthreads();
    const int n = *cnt;
    int npad = 1;
    while (npad < n) npad <<= 1;
    for (int e = n + threadIdx.x; e < npad; e += blockDim.x) {
        k.k0[e] = k.k1[e] = k.k2[e] = ~0ull;
        k.idx[e] = -1;
    }
    __syncthreads();
    for (int size = 2; size <= npad; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < npad / 2; i += blockDim.x) {
                const int a = 2 * i - (i & (stride - 1));
                const int b = a + stride;
                const bool up = (a & size) == 0;
                if (key_gt(k, a, b) == up) {
                    uint64_t x;
                    x = k.k0[a]; k.k0[a] = k.k0[b]; k.k0[b] = x;
                    x = k.k1[a]; k.k1[a] = k.k1[b]; k.k1[b] = x;
                    x = k.k2[a]; k.k2[a] = k.k2[b]; k.k2[b] = x;
                    const int y = k.idx[a]; k.idx[a] = k.idx[b]; k.idx[b] = y;
                }
            }
            __syncthreads();
        }
    }
    return n;
}

// Tables of <= kSmallPollCap slots: the whole poll in one block (one launch).
__global__ void __launch_bounds__(1024) poll_small_kernel(DTableView t, int64_t version, int mb, int pc, int rc,
                                                          int ac, const uint8_t* __restrict__ arena,
                                                          SampleDesc* __restrict__ desc, PollResult* __restrict__ res) {
    extern __shared__ __align__(16) uint8_t sm[];
    __shared__ int cnt;
    __shared__ int64_t scan[kMaxPollMb];
    const SortKeys k = sort_keys(sm);
    const int n = gather_sorted(t, version, 0, k, &cnt);
    if (n < mb) {  // experience_store.hpp:104: fewer than mb ready -> nullopt, nothing marked
        if (threadIdx.x == 0) {
            res->got = 0;
            res->rows = 0;
        }
        return;
    }
    emit_batch(t, k.idx, mb, pc, rc, ac, arena, desc, res, scan);
}

// Larger tables, kernel 1 of 3: each block sorts one kSmallPollCap-slot chunk and
// contributes its canonical-first min(mb, eligible) records as candidates; the
// global first mb are among them (rank_kernel + finish_kernel pick them).
__global__ void __launch_bounds__(1024) chunk_candidates_kernel(DTableView t, int64_t version, int mb,
                                                                int* __restrict__ count, int* __restrict__ elist,
                                                                int* __restrict__ rank) {
    extern __shared__ __align__(16) uint8_t sm[];
    __shared__ int cnt, base;
    const SortKeys k = sort_keys(sm);
    const int n = gather_sorted(t, version, blockIdx.x * kSmallPollCap, k, &cnt);
    const int take = min(n, mb);
    if (threadIdx.x == 0) base = take ? atomicAdd(count, take) : 0;
    __syncthreads();
    for (int i = threadIdx.x; i < take; i += blockDim.x) {
        elist[base + i] = k.idx[i];
        rank[base + i] = 0;  // rank_kernel accumulates into it
    }
}

__global__ void count_ready_kernel(DTableView t, int64_t version, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    const int stride = gridDim.x * blockDim.x;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < t.cap; s += stride) c += eligible(t, s, version) ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void set_cells_kernel(DTableView t, int col, int n, const int64_t* __restrict__ slots,
                                 const uint64_t* __restrict__ vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t s = slots[i];
    t.cells[static_cast<size_t>(col) * t.cap + s] = vals[i];
    t.status[s] |= 1u << col;  // experience_store.hpp:78-79 (host index raised CellAlreadySet)
}

// insert (experience_store.hpp:55-58): a fresh record, every cell unset
__global__ void insert_kernel(DTableView t, int n, const DInsert* __restrict__ recs) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const DInsert r = recs[i];
    t.label[r.slot] = r.label;
    t.turns[r.slot] = r.turns;
    t.traj[r.slot] = r.traj;
    t.version[r.slot] = r.version;
    t.status[r.slot] = 0u;
    t.flags[r.slot] = kSlotLive;
}

__global__ void erase_kernel(DTableView t, int n, const int64_t* __restrict__ slots) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    t.flags[slots[i]] = 0u;
    t.status[slots[i]] = 0u;
}

__global__ void relabel_kernel(DTableView t, const uint64_t* __restrict__ labels) {
    const int stride = gridDim.x * blockDim.x;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < t.cap; s += stride)
        if (t.flags[s] & kSlotLive) t.label[s] = labels[s];
}

// purge_stale (mode 0): !processing && version < current;  purge_inputs (mode 1):
// !processing && label in the sorted set.  Matching slots are erased here and
// listed (in slot order after the host sorts) so the host index drops their keys.
__global__ void purge_kernel(DTableView t, int mode, int64_t current_version, const uint64_t* __restrict__ set,
                             int nset, int* __restrict__ count, int* __restrict__ out) {
    const int stride = gridDim.x * blockDim.x;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < t.cap; s += stride) {
        if ((t.flags[s] & (kSlotLive | kSlotProcessing)) != kSlotLive) continue;
        bool hit;
        if (mode == 0) {
            hit = t.version[s] < current_version;
        } else {
            const uint64_t l = t.label[s];
            int lo = 0, hi = nset;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (set[mid] < l) lo = mid + 1; else hi = mid;
            }
            hit = lo < nset && set[lo] == l;
        }
        if (hit) {
            t.flags[s] = 0u;
            t.status[s] = 0u;
            out[atomicAdd(count, 1)] = s;
        }
    }
}

__device__ __forceinline__ int token_at(const uint8_t* arena, uint64_t off, uint64_t i) {
    // decode_tokens (codec.hpp:28): static_cast<Token>(u64)
    return static_cast<int>(static_cast<uint32_t>(reinterpret_cast<const uint64_t*>(arena + off + 8)[i]));
}

// rule_reward (training.hpp:71-83): longest prefix of `pattern` occurring
// contiguously in the response, / |pattern|.  Warp-cooperative: lane l tries the
// start positions l, l+32, ... (coalesced u64 token loads), then a warp max.
__device__ double rule_reward_warp(const uint8_t* arena, uint64_t off, const int* pat, int np) {
    const uint64_t n = *reinterpret_cast<const uint64_t*>(arena + off);
    if (n == 0 || np == 0) return 0.0;
    int best = 0;
    for (uint64_t start = threadIdx.x & 31; start < n; start += 32) {
        int len = 0;
        while (len < np && start + len < n && token_at(arena, off, start + len) == pat[len]) ++len;
        best = max(best, len);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    return static_cast<double>(best) / static_cast<double>(np);
}

// release_group (rollout.hpp:812-834): one block per group.  Each warp scores
// survivors (warp-parallel rule_reward); thread 0 normalises in the reference's
// sequential order with explicit round-to-nearest ops (no FMA contraction), so
// the advantages are bit-identical to group_advantages (training.hpp:54-67);
// then every record of every survivor gets both cells.
__global__ void __launch_bounds__(512) release_kernel(const DTableView* __restrict__ tabs,
                                                      const DReleaseCols* __restrict__ cols, int ngroups,
                                                      const int32_t* __restrict__ seg_off,
                                                      const int32_t* __restrict__ score_tab,
                                                      const int64_t* __restrict__ score_slot,
                                                      const int32_t* __restrict__ rec_off,
                                                      const int32_t* __restrict__ rec_tab,
                                                      const int64_t* __restrict__ rec_slot, const int* __restrict__ pat,
                                                      int np, double eps, const uint8_t* __restrict__ arena,
                                                      double* __restrict__ rewards, double* __restrict__ advs) {
    const int g = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int b = seg_off[g], e = seg_off[g + 1];
    for (int i = b + warp; i < e; i += nw) {
        const DTableView& t = tabs[score_tab[i]];
        const uint64_t off = t.cells[static_cast<size_t>(cols[score_tab[i]].response) * t.cap + score_slot[i]];
        const double r = rule_reward_warp(arena, off, pat, np);
        if (lane == 0) rewards[i] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0 && e > b) {
        const double k = static_cast<double>(e - b);
        double mean = 0.0;
        for (int i = b; i < e; ++i) mean = __dadd_rn(mean, rewards[i]);
        mean = __ddiv_rn(mean, k);
        double var = 0.0;
        for (int i = b; i < e; ++i) {
            const double d = __dadd_rn(rewards[i], -mean);
            var = __dadd_rn(var, __dmul_rn(d, d));
        }
        var = __ddiv_rn(var, k);
        const double sd = __dsqrt_rn(var);
        const double den = __dadd_rn(sd, eps);
        for (int i = b; i < e; ++i) advs[i] = __ddiv_rn(__dadd_rn(rewards[i], -mean), den);
    }
    __syncthreads();
    for (int i = b + warp; i < e; i += nw) {
        for (int r = rec_off[i] + lane; r < rec_off[i + 1]; r += 32) {
            const DTableView& t = tabs[rec_tab[r]];
            const DReleaseCols& c = cols[rec_tab[r]];
            const int64_t s = rec_slot[r];
            t.cells[static_cast<size_t>(c.reward) * t.cap + s] = static_cast<uint64_t>(__double_as_longlong(rewards[i]));
            t.cells[static_cast<size_t>(c.advantage) * t.cap + s] = static_cast<uint64_t>(__double_as_longlong(advs[i]));
            atomicOr(&t.status[s], (1u << c.reward) | (1u << c.advantage));
        }
    }
}

// Generated responses -> the reference codec in the arena ([u64 n][u64 tok] x n,
// codec.hpp:15-22; log-probs as [u64 n][f64] x n) + the two ref cells.
__global__ void encode_kernel(DTableView t, int rc, int lc, const int64_t* __restrict__ slots,
                              const int32_t* __restrict__ tok, const double* __restrict__ lp,
                              const int32_t* __restrict__ len, int max_tokens, uint8_t* __restrict__ arena,
                              uint64_t base_off, uint64_t stride) {
    const int i = blockIdx.x;
    const int n = len[i];
    const uint64_t ro = base_off + static_cast<uint64_t>(i) * stride;
    const uint64_t lo = ro + 8 + 8 * static_cast<uint64_t>(max_tokens);
    uint64_t* r = reinterpret_cast<uint64_t*>(arena + ro);
    uint64_t* l = reinterpret_cast<uint64_t*>(arena + lo);
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        r[1 + j] = static_cast<uint64_t>(static_cast<int64_t>(tok[static_cast<size_t>(i) * max_tokens + j]));
        l[1 + j] = static_cast<uint64_t>(__double_as_longlong(lp[static_cast<size_t>(i) * max_tokens + j]));
    }
    if (threadIdx.x == 0) {
        r[0] = static_cast<uint64_t>(n);
        l[0] = static_cast<uint64_t>(n);
        const int64_t s = slots[i];
        uint32_t bits = 1u << rc;
        t.cells[static_cast<size_t>(rc) * t.cap + s] = ro;
        if (lc >= 0) {
            t.cells[static_cast<size_t>(lc) * t.cap + s] = lo;
            bits |= 1u << lc;
        }
        t.status[s] |= bits;
    }
}

}  // namespace

cudaError_t launch_dt_poll(const DTableView& t, int64_t version, int mb, int pc, int rc, int ac,
                           const uint8_t* arena, DPollScratch sc, SampleDesc* desc, PollResult* res,
                           cudaStream_t s) {
    const size_t smem = static_cast<size_t>(kSmallPollCap) * (3 * 8 + 4);
    if (t.cap <= kSmallPollCap) {
        cudaFuncSetAttribute(poll_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        poll_small_kernel<<<1, 1024, smem, s>>>(t, version, mb, pc, rc, ac, arena, desc, res);
        return cudaGetLastError();
    }
    cudaError_t e = cudaMemsetAsync(sc.count, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    const int chunks = (t.cap + kSmallPollCap - 1) / kSmallPollCap;
    cudaFuncSetAttribute(chunk_candidates_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    chunk_candidates_kernel<<<chunks, 1024, smem, s>>>(t, version, mb, sc.count, sc.elist, sc.rank);
    // candidates <= chunks * mb: rank them pairwise (2D grid), then pick rank < mb
    const int64_t cmax = static_cast<int64_t>(chunks) * mb;
    const int bx = static_cast<int>((cmax + 255) / 256);
    dim3 g(static_cast<unsigned>(bx), static_cast<unsigned>(bx < 16 ? bx : 16));
    rank_kernel<<<g, 256, 0, s>>>(t, sc.count, sc.elist, sc.rank);
    finish_kernel<<<1, 1024, 0, s>>>(t, sc.count, sc.elist, sc.rank, mb, pc, rc, ac, arena, desc, res);
    return cudaGetLastError();
}

cudaError_t launch_dt_ready_count(const DTableView& t, int64_t version, unsigned long long* out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    const int blocks = (t.cap + 255) / 256;
    count_ready_kernel<<<blocks < 148 * 4 ? blocks : 148 * 4, 256, 0, s>>>(t, version, out);
    return cudaGetLastError();
}

cudaError_t launch_dt_insert(const DTableView& t, int n, const DInsert* recs, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    insert_kernel<<<(n + 255) / 256, 256, 0, s>>>(t, n, recs);
    return cudaGetLastError();
}

cudaError_t launch_dt_set_cells(const DTableView& t, int col, int n, const int64_t* slots, const uint64_t* vals,
                                cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    set_cells_kernel<<<(n + 255) / 256, 256, 0, s>>>(t, col, n, slots, vals);
    return cudaGetLastError();
}

cudaError_t launch_dt_erase(const DTableView& t, int n, const int64_t* slots, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    erase_kernel<<<(n + 255) / 256, 256, 0, s>>>(t, n, slots);
    return cudaGetLastError();
}

cudaError_t launch_dt_relabel(const DTableView& t, const uint64_t* labels, cudaStream_t s) {
    const int blocks = (t.cap + 255) / 256;
    relabel_kernel<<<blocks < 148 * 4 ? blocks : 148 * 4, 256, 0, s>>>(t, labels);
    return cudaGetLastError();
}

cudaError_t launch_dt_purge(const DTableView& t, int mode, int64_t current_version, const uint64_t* set, int nset,
                            int* count, int* out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    const int blocks = (t.cap + 255) / 256;
    purge_kernel<<<blocks < 148 * 4 ? blocks : 148 * 4, 256, 0, s>>>(t, mode, current_version, set, nset, count, out);
    return cudaGetLastError();
}

cudaError_t launch_dt_release(const DTableView* tabs, const DReleaseCols* cols, int ngroups, const int32_t* seg_off,
                              const int32_t* score_tab, const int64_t* score_slot, const int32_t* rec_off,
                              const int32_t* rec_tab, const int64_t* rec_slot, const int* pat, int np, double eps,
                              const uint8_t* arena, double* rewards, double* advs, cudaStream_t s) {
    if (ngroups <= 0) return cudaSuccess;
    release_kernel<<<ngroups, 512, 0, s>>>(tabs, cols, ngroups, seg_off, score_tab, score_slot, rec_off, rec_tab,
                                           rec_slot, pat, np, eps, arena, rewards, advs);
    return cudaGetLastError();
}

cudaError_t launch_dt_encode(const DTableView& t, int rc, int lc, int n, const int64_t* slots, const int32_t* tok,
                             const double* lp, const int32_t* len, int max_tokens, uint8_t* arena, uint64_t base_off,
                             uint64_t stride, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    encode_kernel<<<n, 128, 0, s>>>(t, rc, lc, slots, tok, lp, len, max_tokens, arena, base_off, stride);
    return cudaGetLastError();
}

}  // namespace fm

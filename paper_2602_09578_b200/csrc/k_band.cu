// k_band.cu — the policy's two products in the context-position ("band")
// formulation:
//
// phi_t (policy.hpp:42-51) is the mean one-hot of the LAST FOUR context
// tokens, and the context grows by one token per trained row
// (training.hpp:389-393), so row t's logits are a 4-tap sliding sum over
// context POSITIONS:
//
//   z_t[v] = (1/n_t) * sum_{k<4} W[v][feat(q0_t + k)]          (policy.hpp:57-61)
//
// where position q holds the context token at that place of the sample's
// sequence (prompt ++ response) and feat = tok mod D.  Every position's row
// X[q][:] = W16^T[feat(q)][:] is a contiguous row of the transposed bf16
// shadow, so each row costs ONE new 2·V-byte row read (the other three are
// the previous rows' positions, kept in registers) — an HBM-streaming
// stencil, not a GEMM: the dense Phi·W^T would spend D/4 multiply-adds per
// useful one.  The weight gradient (policy.hpp:83-90) likewise becomes, per
// position,
//
//   H[q][v] = sum_{t: q in ctx(t)} c_t (delta(v, a_t) - p_t[v])  (c_t = -A/(G n_t))
//   dW[v][feat(q)] += H[q][v]
//
// H rows go to the A' segment of their feature's 256-column block (one row
// per position — the token-slot layout stored every p~ row 3.6x), and the
// tcgen05 segmented GEMM2 (k_gemm_tc.cu) scatters them into dW's columns
// with a one-hot B'.
//
//   K-pos     positions of the micro-batch shard: feat[q] (prompt tail +
//             response prefix of every sample), q0[row]       (codec.hpp:24-30)
//   K-pslot   A'/B' slot of every position in its feature block's segment
//             (count, one scan, place)
//   K-stats   pass A: per-(row, consumer warp) partial sums of exp(z - bound)
//             against the row's fmax bound (no max pass)      (policy.hpp:62-70)
//   K-band    pass B: p = exp(z - lse) (lse from K-lse), the per-row
//             log-softmax gradient folded into the per-position H rows
//                                                             (policy.hpp:83-90, training.hpp:394)
//
// Both passes stream the W16^T rows through a shared-memory ring filled by
// one producer thread with 1-D bulk copies (cp.async.bulk, mbarrier
// completion); eight consumer warps each own 256 vocabulary columns (eight
// per lane).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <type_traits>

#include "fm_kernels.h"
#include "fm_ptx.cuh"

namespace fm {

namespace {

constexpr int kBandConsumers = 256;                  // 8 consumer warps
constexpr int kBandThreads = kBandConsumers + 32;    // + the producer warp
// W16^T ring stages (4 KB each): pass B 16 at two CTAs per SM (12 / 16 / 24 measured within
// 1%, tools/variant_libs.sh); pass A 8 (it also holds a 34 KB partial-sum buffer) at three
#ifndef FM_STATS_STAGES
#define FM_STATS_STAGES 8
#endif
#ifndef FM_BAND_STAGES
#define FM_BAND_STAGES 16
#endif
template <bool kGrad>
constexpr int kBandStagesT = kGrad ? FM_BAND_STAGES : FM_STATS_STAGES;
constexpr int kBandRows = 128;                       // trained rows per CTA
// vocabulary columns per consumer lane (4 fp32 pairs at 8): 8 by default; 4 halves
// the per-thread state for a third CTA per SM
#ifndef FM_BAND_CPL
#define FM_BAND_CPL 8
#endif
constexpr int kCPL = FM_BAND_CPL;
constexpr int kP = kCPL / 2;  // fp32 pairs per lane
static_assert(kCPL == 8 || kCPL == 4, "8 or 4 columns per lane");
constexpr int kBandMinBlocks = kCPL == 8 ? 2 : 3;
// pass A alone fits 72 registers at 8 columns per lane (no spills): three CTAs (27 warps) per
// SM with an 8-stage ring, measured at C2 0.193 vs 0.211 ms (two CTAs, 16 stages) and 0.217
// (two CTAs, 8 stages): K-stats is latency-bound, the extra warps hide it
#ifndef FM_STATS_MIN_BLOCKS
#define FM_STATS_MIN_BLOCKS 3
#endif
constexpr int kStatsMinBlocks = FM_STATS_MIN_BLOCKS;
using Frag = std::conditional_t<kCPL == 8, uint4, uint2>;  // a lane's kCPL bf16 columns
// 8 columns per lane, two CTAs (18 warps) per SM: 16 columns per lane (measured:
// K-stats 0.43-0.53 ms vs 0.33 ms at C2) needs more registers than two CTAs leave
// and drops to one CTA per SM.
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ int token_of(uint64_t x) {  // static_cast<Token>(u64), codec.hpp:28
    return static_cast<int>(static_cast<uint32_t>(x));
}
__device__ __forceinline__ int32_t feature_of(int tok, uint64_t D) {  // policy.hpp:48
    return static_cast<int32_t>(static_cast<uint64_t>(static_cast<int64_t>(tok)) % D);
}

// sample holding global row gr: the last s with row_start[s] <= gr (rows are in poll order)
__device__ __forceinline__ int sample_of_row(const SampleDesc* sd, int n, int64_t gr) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sd[mid].row_start <= gr) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// First position of sample s in the shard: every sample overlapping the shard
// owns (its rows in the shard) + 3 consecutive positions.
__device__ __forceinline__ int64_t pos_base(const SampleDesc* sd, int s, int s_first, int64_t row_lo) {
    const int64_t rs = sd[s].row_start - row_lo;
    return (rs > 0 ? rs : 0) + 3 * static_cast<int64_t>(s - s_first);
}

__global__ void __launch_bounds__(256) positions_kernel(const uint8_t* __restrict__ arena,
                                                        const SampleDesc* __restrict__ sd, int n, int64_t row_lo,
                                                        int64_t M, uint64_t D, int32_t* __restrict__ feat,
                                                        int64_t Qcap) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= Qcap) return;
    int32_t f = -1;
    if (M > 0 && n > 0) {
        const int s_first = sample_of_row(sd, n, row_lo);
        int lo = s_first, hi = n - 1;  // last sample whose first position is <= q
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pos_base(sd, mid, s_first, row_lo) <= q) lo = mid;
            else hi = mid - 1;
        }
        const SampleDesc d = sd[lo];
        const int64_t a = d.row_start > row_lo ? d.row_start : row_lo;
        const int64_t e = d.row_start + d.resp_n < row_lo + M ? d.row_start + d.resp_n : row_lo + M;
        const int64_t k = q - pos_base(sd, lo, s_first, row_lo);
        if (e > a && k < (e - a) + 3) {
            // position k of the shard's part of the sample = sequence index prompt_n - 4 + ja + k
            const int64_t seq = static_cast<int64_t>(d.prompt_n) - 4 + (a - d.row_start) + k;
            if (seq >= 0) {
                const uint64_t* P = reinterpret_cast<const uint64_t*>(arena + d.prompt_off + 8);
                const uint64_t* R = reinterpret_cast<const uint64_t*>(arena + d.resp_off + 8);
                const int tok = token_of(seq < d.prompt_n ? __ldg(P + seq) : __ldg(R + (seq - d.prompt_n)));
                f = feature_of(tok, D);
            }
        }
    }
    feat[q] = f;
}

// ---- K-fmax: per-feature maxima of the shadow ----------------------------------
__global__ void __launch_bounds__(256) fmax_kernel(const __nv_bfloat16* __restrict__ w16t, int64_t V, int64_t ldw,
                                                   float* __restrict__ fmax) {
    __shared__ float red[8];
    const __nv_bfloat16* row = w16t + static_cast<int64_t>(blockIdx.x) * ldw;
    float m = -INFINITY;
    const int64_t v8 = V / 8;
    for (int64_t i = threadIdx.x; i < v8; i += blockDim.x) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(row) + i);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
            m = fmaxf(m, fmaxf(__uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xffff0000u)));
    }
    for (int64_t v = v8 * 8 + threadIdx.x; v < V; v += blockDim.x) m = fmaxf(m, __bfloat162float(row[v]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = red[0];
        for (int k = 1; k < 8; ++k) t = fmaxf(t, red[k]);
        fmax[blockIdx.x] = t;
    }
}

// ---- K-pslot ---------------------------------------------------------------
// block-wide exclusive scan of a 0/1 flag over 1024 threads; returns the rank,
// *total gets the count (all threads)
__device__ __forceinline__ int block_rank(bool flag, int* wsum, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int pre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) wsum[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
        const int v = wsum[lane];
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        wsum[lane] = inc - v;
        if (lane == 31) wsum[32] = inc;
    }
    __syncthreads();
    const int r = wsum[wid] + pre;
    *total = wsum[32];
    __syncthreads();
    return r;
}

// grid (nblk, chunks of 1024 positions): CTA (b, c) counts chunk c's positions
// whose feature lies in block b; CTA (b = 0, c) resets their slots
__global__ void __launch_bounds__(1024) pslot_count_kernel(const int32_t* __restrict__ feat, int64_t Q,
                                                           int32_t* __restrict__ ccount, int32_t* __restrict__ slot) {
    __shared__ int wsum[33];
    const int b = blockIdx.x, c = blockIdx.y;
    const int64_t q = static_cast<int64_t>(c) * 1024 + threadIdx.x;
    const int32_t f = q < Q ? __ldg(feat + q) : -1;
    int tot;
    block_rank(f >= 0 && (f >> 8) == b, wsum, &tot);
    if (threadIdx.x == 0) ccount[static_cast<size_t>(b) * gridDim.y + c] = tot;
    if (b == 0 && q < Q) slot[q] = -1;
}

// One block: segment offsets from the chunk counts (block-major, every segment
// padded to a multiple of 64 rows, at least 64) and each (block, chunk)'s first
// rank in its segment (position order: deterministic).  ccount [nblk][nch] ->
// cbase [nblk][nch]; warp w handles blocks w, w + 32, ... and the block totals
// are scanned once (replaces a per-(block, chunk) rescan that was O(nblk^2 nch):
// 164 us per micro-batch at D = 32,768).
__global__ void __launch_bounds__(1024) pslot_scan_kernel(const int32_t* __restrict__ ccount, int nblk, int nch,
                                                          int32_t* __restrict__ cbase, int32_t* __restrict__ kseg_off,
                                                          int32_t* __restrict__ kiters,
                                                          unsigned long long* rows_acc) {
    extern __shared__ int32_t seg_len[];  // [nblk] padded segment lengths, then [nblk] offsets
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int b = wid; b < nblk; b += nw) {
        // exclusive prefix over the block's chunks, 32 at a time
        int run = 0;
        for (int c0 = 0; c0 < nch; c0 += 32) {
            const int c = c0 + lane;
            const int v = c < nch ? ccount[static_cast<size_t>(b) * nch + c] : 0;
            int inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (c < nch) cbase[static_cast<size_t>(b) * nch + c] = run + inc - v;
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) seg_len[b] = run < 64 ? 64 : (run + 63) / 64 * 64;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int off = 0;
        unsigned long long tot = 0;
        for (int b = 0; b < nblk; ++b) {
            const int len = seg_len[b];
            seg_len[nblk + b] = off;
            kseg_off[b] = off;
            kiters[b] = len / 64;
            off += len;
            tot += static_cast<unsigned long long>(len);
        }
        if (rows_acc) atomicAdd(rows_acc, tot);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nblk * nch; i += blockDim.x) cbase[i] += seg_len[nblk + i / nch];
}

// grid (nblk, chunks): the position's rank in its segment (segment start + the
// chunk's first rank + the rank within the chunk) and its one-hot B' row.
__global__ void __launch_bounds__(1024) pslot_place_kernel(const int32_t* __restrict__ feat, int64_t Q,
                                                           const int32_t* __restrict__ cbase,
                                                           int32_t* __restrict__ slot,
                                                           __nv_bfloat16* __restrict__ bseg, int64_t kp_cap) {
    __shared__ int wsum[33];
    const int b = blockIdx.x, c = blockIdx.y, nch = gridDim.y;
    const int base = __ldg(cbase + static_cast<size_t>(b) * nch + c);
    const int64_t q = static_cast<int64_t>(c) * 1024 + threadIdx.x;
    const int32_t f = q < Q ? __ldg(feat + q) : -1;
    const bool hit = f >= 0 && (f >> 8) == b;
    int tot;
    const int rk = block_rank(hit, wsum, &tot);
    if (hit) {
        const int s = base + rk;
        FM_DCHECK(s >= 0 && s < kp_cap);
        slot[q] = s;
        bseg[static_cast<size_t>(s) * 256 + (f & 255)] = __float2bfloat16_rn(1.f);
    }
}

// ---- K-stats / K-band ------------------------------------------------------
// 8 bf16 -> 4 fp32 pairs (exact)
__device__ __forceinline__ void unpack_frag(uint4 u, float2 (&x)[4]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xffff0000u));
}
__device__ __forceinline__ void unpack_frag(uint2 u, float2 (&x)[2]) {
    const uint32_t w[2] = {u.x, u.y};
#pragma unroll
    for (int i = 0; i < 2; ++i) x[i] = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xffff0000u));
}

__device__ __forceinline__ uint4 make_frag(const uint32_t (&w)[4]) { return make_uint4(w[0], w[1], w[2], w[3]); }
__device__ __forceinline__ uint2 make_frag(const uint32_t (&w)[2]) { return make_uint2(w[0], w[1]); }

// kP fp32 pairs -> kCPL bf16 (round to nearest)
__device__ __forceinline__ Frag pack_frag(const float2 (&x)[kP]) {
    uint32_t w[kP];
#pragma unroll
    for (int i = 0; i < kP; ++i) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(x[i].x, x[i].y);
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    return make_frag(w);
}

// 2^x, one MUFU op (inputs <= 0 here; results below 2^-126 flush to zero)
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Grid (vocabulary slices of 2,048 columns, chunks of kBandRows rows).
// kGrad = false: pass A (K-stats) over rows [ra, rb).
// kGrad = true:  pass B (K-band): rows [ra - 3, rb) so that every position in
// [q0[ra], q0[rb]) (the chunk's emission range) has all of its rows.
// Shared memory: the W16^T row ring, its full / empty barriers, and the
// chunk's per-row metadata (q0, action, rs * log2e, -bound * log2e with the
// bound = mrow (pass A) or lse (pass B), coefficient) plus a sentinel row
// kNoRow whose terms vanish (exp2(-1e30) = 0, coefficient 0).
constexpr int kMetaRows = kBandRows + 5;
constexpr int kNoRow = kMetaRows - 1;
constexpr int kRedPitch = 33;  // per-warp [32 rows][32 lanes] partial sums, padded (conflict-free transpose)
// Positions of a chunk the branch-free loop indexes directly (4 per row covers
// samples of >= 1 row; longer spans — many empty samples — take the general loop).
constexpr int kMaxQ = 4 * (kBandRows + 4) + 16;
static_assert(kBandStagesT<false> % 4 == 0 && kBandStagesT<true> % 4 == 0,
              "the 4-position body consumes whole groups of 4 stages");
template <bool kGrad>
constexpr size_t band_smem_bytes() {
    constexpr int kBandStages = kBandStagesT<kGrad>;
    return kBandStages * kBandConsumers * 2 * kCPL + 2 * kBandStages * sizeof(uint64_t) +
           5 * kMetaRows * sizeof(int32_t) + (kGrad ? 0 : (kBandConsumers / 32) * 32 * kRedPitch * sizeof(float)) +
           kMaxQ * sizeof(int32_t);
}

template <bool kGrad, int kMinBlocks>
__global__ void __launch_bounds__(kBandThreads, kMinBlocks) band_kernel(const BandArgs A) {
    constexpr int kCols = kBandConsumers * kCPL;  // vocabulary columns per item
    constexpr int kStage = kCols * 2;          // bytes of one position's W16^T slice
    constexpr int kBandStages = kBandStagesT<kGrad>;
    extern __shared__ __align__(128) uint8_t band_smem[];
    uint8_t* ring = band_smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(band_smem + kBandStages * kStage);
    uint64_t* empty = full + kBandStages;
    int32_t* m_q0 = reinterpret_cast<int32_t*>(empty + kBandStages);
    int32_t* m_act = m_q0 + kMetaRows;
    float* m_c = reinterpret_cast<float*>(m_act + kMetaRows);  // rs * log2e
    float* m_off = m_c + kMetaRows;                             // -bound * log2e
    float* m_ce = m_off + kMetaRows;                            // pass B: the row coefficient
    float* redbuf = m_ce + kMetaRows;                           // pass A: per-warp [32][kRedPitch]
    // position q - qlo of the item -> the row whose four positions end there, or kNoRow
    int32_t* m_end = reinterpret_cast<int32_t*>(redbuf + (kGrad ? 0 : (kBandConsumers / 32) * 32 * kRedPitch));
    const int tid = static_cast<int>(threadIdx.x);
    const int lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kBandStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kBandConsumers / 32);
        }
        fence_barrier_init();
        m_act[kNoRow] = INT_MIN / 4;
        m_c[kNoRow] = 0.f;
        m_off[kNoRow] = -1e30f;
        m_ce[kNoRow] = 0.f;
    }
    __syncthreads();
    // Items (vocabulary slice, chunk of kBandRows rows), slice fastest, taken round-robin:
    // one per CTA, or (launch_band, few items) persistent CTAs whose ring runs on across
    // items, so the producer prefetches the next item's rows while the consumers finish
    // (and load the metadata of) the current one — no partial last wave.
    const int nslices = static_cast<int>((A.V + kCols - 1) / kCols);
    const int rpi = A.rows_per_item;  // <= kBandRows
    const int nitems = nslices * static_cast<int>((A.M + rpi - 1) / rpi);
    struct Item {
        int64_t v0;
        int ra, rb, rstart, nrows, qa, qb, qend, qlo, qhi;
        bool fast;
    };
    auto item_at = [&](int it) {
        Item g;
        g.v0 = static_cast<int64_t>(it % nslices) * kCols;
        g.ra = (it / nslices) * rpi;
        g.rb = g.ra + rpi < A.M ? g.ra + rpi : static_cast<int>(A.M);
        g.rstart = kGrad ? (g.ra >= 3 ? g.ra - 3 : 0) : g.ra;
        g.nrows = g.rb - g.rstart;
        g.qa = __ldg(A.q0 + g.rstart);
        g.qb = __ldg(A.q0 + g.rb - 1) + 4;
        g.qend = kGrad ? g.qb + 3 : g.qb;  // pass B runs 3 positions on to flush the last H rows
        // the branch-free loop runs whole 4-position bodies over [qlo, qhi); its padding
        // positions stream the zero row, so every body takes exactly 4 ring stages
        g.qlo = g.qa & ~3;
        g.qhi = (g.qend + 3) & ~3;
        g.fast = g.qhi - g.qlo <= kMaxQ;
        return g;
    };

    // warp-uniform role split (the broadcast tells the compiler so: no divergent
    // shuffle fallbacks in the consumers)
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    if (warp >= kBandConsumers / 32) {
        // ===== producer warp: lane 0 streams the positions' W16^T row slices; the
        // positions' features are fetched 32 at a time, one group ahead =====
        int st = 0;
        uint32_t ph = 0;
        int issued = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const Item g = item_at(it);
            const int64_t cols = A.ldw - g.v0 < kCols ? A.ldw - g.v0 : kCols;
            const uint32_t bytes = static_cast<uint32_t>(cols) * 2u;
            const __nv_bfloat16* base = A.w16t + g.v0;
            const int p0 = g.fast ? g.qlo : g.qa, np = (g.fast ? g.qhi : g.qb) - p0;
            auto feat_at = [&](int k) -> int32_t {
                const int q = p0 + k;
                return k < np && q >= g.qa && q < g.qb ? __ldg(A.pos_feat + q) : -1;
            };
            int32_t f_next = feat_at(lane);
            for (int k0 = 0; k0 < np; k0 += 32) {
                const int32_t f_cur = f_next;
                f_next = feat_at(k0 + 32 + lane);
                const int kn = np - k0 < 32 ? np - k0 : 32;
                for (int j = 0; j < kn; ++j) {
                    if (issued++ >= kBandStages) mbar_wait(&empty[st], ph ^ 1u);
                    const int32_t f = __shfl_sync(0xffffffffu, f_cur, j);
                    if (lane == 0) {
                        // a position before the sequence start (or a padding position) reads the zero row
                        const __nv_bfloat16* src = f >= 0 ? base + static_cast<int64_t>(f) * A.ldw : A.zero_row;
                        mbar_arrive_expect_tx(&full[st], bytes);
                        FM_DCHECK(f < A.dbg_D);
                        bulk_load(ring + st * kStage, src, bytes, &full[st]);
                    }
                    __syncwarp();
                    if (++st == kBandStages) {
                        st = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ===== consumers: lane = 8 consecutive columns, as 4 fp32 pairs =====
    // lane l of warp w covers columns v0 + (w * 32 + l) * 8 .. + 8, so every shared-memory
    // read of the warp is 512 contiguous bytes
    int st = 0;
    uint32_t ph = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const Item g = item_at(it);
        const int64_t v0 = g.v0;
        const int ra = g.ra, rb = g.rb, rstart = g.rstart, nrows = g.nrows;
        const int qa = g.qa, qb = g.qb, qend = g.qend, qlo = g.qlo, qhi = g.qhi;
        const bool fast = g.fast;
        // the item's rows' metadata (the previous item's readers are done: first barrier)
        named_bar_sync(1, kBandConsumers);
        for (int i = tid; i <= nrows; i += kBandConsumers) {
            const int r = rstart + i;
            m_q0[i] = r < A.M ? __ldg(A.q0 + r) : INT32_MAX - 8;
            if (i < nrows) {
                m_act[i] = __ldg(A.action + r) - static_cast<int32_t>(A.col_base);  // this range's column
                m_c[i] = __ldg(A.rscale + r) * kLog2e;
                m_off[i] = -__ldg(kGrad ? A.lse + r : A.mrow + r) * kLog2e;
                if constexpr (kGrad) m_ce[i] = __ldg(A.coef_eff + r);
            }
        }
        if (fast) {
            for (int k = tid; k < kMaxQ; k += kBandConsumers) m_end[k] = kNoRow;
            named_bar_sync(1, kBandConsumers);
            for (int i = tid; i < nrows; i += kBandConsumers) {
                FM_DCHECK(m_q0[i] + 3 - qlo >= 0 && m_q0[i] + 3 - qlo < qhi - qlo);
                m_end[m_q0[i] + 3 - qlo] = i;
            }
        }
        named_bar_sync(1, kBandConsumers);

        const int64_t cb = v0 + static_cast<int64_t>(tid) * kCPL;
        const int nv = A.V - cb >= kCPL ? kCPL : (A.V - cb > 0 ? static_cast<int>(A.V - cb) : 0);
        const bool warp_full = __all_sync(0xffffffffu, nv == kCPL);
        const int tile = static_cast<int>(v0 / kCols) * (kBandConsumers / 32) + warp;  // the warp's stats column
        // per position q: xp = X[q-1] (previous position's row), pr[q & 3] = X[q-1] + X[q];
        // the row ending at q sums pr[(q-2) & 3] + pr[q & 3] = X[q-3] + X[q-2] + X[q-1] + X[q]
        float2 xp[kP], pr[4][kP], gr[4][kP];
#pragma unroll
        for (int j = 0; j < kP; ++j) {
            xp[j] = make_float2(0.f, 0.f);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                pr[i][j] = make_float2(0.f, 0.f);
                if constexpr (kGrad) gr[i][j] = make_float2(0.f, 0.f);
            }
        }
        int elo = 0, ehi = 0;
        // pass B: slots of the positions being flushed, 32 at a time (one group ahead)
        int sg = 0;
        int32_t s_cur = -1, s_next = -1;
        if constexpr (kGrad) {
            elo = m_q0[ra - rstart];
            ehi = rb < A.M ? m_q0[nrows] : qb;
            sg = elo & ~31;
            s_cur = sg + lane < qb ? __ldg(A.pos_slot + sg + lane) : -1;
            s_next = sg + 32 + lane < qb ? __ldg(A.pos_slot + sg + 32 + lane) : -1;
        }
        auto valid = [&](int j, int h) { return warp_full || 2 * j + h < nv; };  // element 2j + h of the lane

        // pass A: the row's partial sum of exp2(z * log2e - bound * log2e) over the lane's
        // columns (the bound mrow >= every z of the row: no max reduction)
        auto row_sum = [&](const float2 (&z4)[kP], float c, float off, auto FullTag) -> float {
            constexpr bool kFull = decltype(FullTag)::value;
            const float2 cc = make_float2(c, c), oo = make_float2(off, off);
            float2 e[kP];
#pragma unroll
            for (int j = 0; j < kP; ++j) {
                const float2 y = __ffma2_rn(z4[j], cc, oo);
                e[j] = make_float2(ex2(y.x), ex2(y.y));
                if constexpr (!kFull) {
                    if (!valid(j, 0)) e[j].x = 0.f;
                    if (!valid(j, 1)) e[j].y = 0.f;
                }
            }
            float2 s2;
            if constexpr (kP == 4) s2 = __fadd2_rn(__fadd2_rn(e[0], e[1]), __fadd2_rn(e[2], e[3]));
            else s2 = __fadd2_rn(e[0], e[1]);
            return s2.x + s2.y;
        };
        // pass B: g = ce (delta(v, a) - exp(z - lse)) over the lane's columns (zero-advantage
        // rows and the sentinel give 0, training.hpp:394); dact = action column - the lane's first
        auto row_grad = [&](const float2 (&z4)[kP], float c, float off, float ce, int dact, float2 (&gg)[kP]) {
            const float2 cc = make_float2(c, c), oo = make_float2(off, off), nce = make_float2(-ce, -ce);
#pragma unroll
            for (int j = 0; j < kP; ++j) {
                const float2 y = __ffma2_rn(z4[j], cc, oo);
                gg[j] = __fmul2_rn(make_float2(ex2(y.x), ex2(y.y)), nce);
            }
            if (static_cast<unsigned>(dact) < static_cast<unsigned>(kCPL)) {
#pragma unroll
                for (int j = 0; j < kP; ++j) {
                    if (dact == 2 * j) gg[j].x += ce;
                    if (dact == 2 * j + 1) gg[j].y += ce;
                }
            }
        };
        // pass B: position p's H row = the four g-ring slots (the rows ending at p .. p + 3)
        auto flush_h = [&](int p) {
            if (p >= elo && p < ehi) {
                if (p >= sg + 32) {  // next group of slots (warp-uniform)
                    sg += 32;
                    s_cur = s_next;
                    s_next = sg + 32 + lane < qb ? __ldg(A.pos_slot + sg + 32 + lane) : -1;
                }
                const int32_t sl = __shfl_sync(0xffffffffu, s_cur, p - sg);
                if (sl >= 0 && nv > 0) {
                    float2 h[kP];
#pragma unroll
                    for (int j = 0; j < kP; ++j)
                        h[j] = __fadd2_rn(__fadd2_rn(gr[0][j], gr[1][j]), __fadd2_rn(gr[2][j], gr[3][j]));
                    if (nv < kCPL) {
                        // the row's columns past V (up to its 8-aligned pitch) hold arithmetic on
                        // stale ring bytes: store zeros, so every A' byte stays finite — A' is
                        // reused across agents of other widths, whose segment padding rows (B' = 0)
                        // may land there, and 0 x NaN would poison their dW
#pragma unroll
                        for (int j = 0; j < kP; ++j) {
                            if (2 * j >= nv) h[j].x = 0.f;
                            if (2 * j + 1 >= nv) h[j].y = 0.f;
                        }
                    }
                    FM_DCHECK(sl < A.dbg_kp && cb + kCPL <= A.ld_a);
                    *reinterpret_cast<Frag*>(A.aseg + static_cast<int64_t>(sl) * A.ld_a + cb) = pack_frag(h);
                }
            }
        };
        // pass A: lanes 0..n-1 add up the 32 lane partials of parked rows [r0, r0 + n) of
        // the warp's ring (transposed read of the padded ring, conflict-free) into the
        // warp's stats column
        auto flush_rows = [&](int r0, int n) {
            __syncwarp();
            if (lane < n) {
                const float* src = redbuf + warp * 32 * kRedPitch + ((r0 + lane) & 31) * kRedPitch;
                float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
#pragma unroll
                for (int kk = 0; kk < 32; kk += 4) {
                    t0 += src[kk];
                    t1 += src[kk + 1];
                    t2 += src[kk + 2];
                    t3 += src[kk + 3];
                }
                FM_DCHECK(tile < A.stats_ld && rstart + r0 + lane < A.M);
                A.stats[static_cast<int64_t>(tile) * A.ld_stats + rstart + r0 + lane] = (t0 + t1) + (t2 + t3);
            }
            __syncwarp();
        };
        const int d_lane = static_cast<int>(cb - v0);  // the lane's first column within the slice

        if (!fast) {
            // general loop (items whose samples are mostly empty): one position at a time over
            // [qa, qb), stages consumed only for real positions
            int ri = 0;             // next row
            int next_end = qa + 3;  // its last position
            auto step = [&](int q, auto Sc) {
                constexpr int S = decltype(Sc)::value;
                if (q >= qa && q < qb) {
                    mbar_wait(&full[st], ph);
                    const Frag u = *reinterpret_cast<const Frag*>(ring + st * kStage + tid * sizeof(Frag));
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[st]);
                    if (++st == kBandStages) {
                        st = 0;
                        ph ^= 1u;
                    }
                    float2 x[kP];
                    unpack_frag(u, x);
#pragma unroll
                    for (int j = 0; j < kP; ++j) {
                        pr[S][j] = __fadd2_rn(xp[j], x[j]);
                        xp[j] = x[j];
                    }
                    if (q == next_end) {  // the row whose four positions end here
                        const int i = ri;
                        float2 z4[kP];
#pragma unroll
                        for (int j = 0; j < kP; ++j) z4[j] = __fadd2_rn(pr[(S + 2) & 3][j], pr[S][j]);
                        if constexpr (!kGrad) {
                            const float s = warp_full ? row_sum(z4, m_c[i], m_off[i], std::true_type{})
                                                      : row_sum(z4, m_c[i], m_off[i], std::false_type{});
                            redbuf[warp * 32 * kRedPitch + (i & 31) * kRedPitch + lane] = s;
                            if ((i & 31) == 31 || i == nrows - 1) flush_rows(i & ~31, (i & 31) + 1);
                        } else {
                            row_grad(z4, m_c[i], m_off[i], m_ce[i], m_act[i] - static_cast<int>(v0) - d_lane, gr[S]);
                        }
                        ++ri;
                        next_end = m_q0[ri] + 3;
                    } else if constexpr (kGrad) {
#pragma unroll
                        for (int j = 0; j < kP; ++j) gr[S][j] = make_float2(0.f, 0.f);  // no row ends here
                    }
                } else if constexpr (kGrad) {
#pragma unroll
                    for (int j = 0; j < kP; ++j) gr[S][j] = make_float2(0.f, 0.f);  // past the last position
                }
                if constexpr (kGrad) flush_h(q - 3);
            };
            for (int qq = qlo; qq < qend; qq += 4) {
                step(qq, std::integral_constant<int, 0>{});
                step(qq + 1, std::integral_constant<int, 1>{});
                step(qq + 2, std::integral_constant<int, 2>{});
                step(qq + 3, std::integral_constant<int, 3>{});
            }
            continue;
        }

        // Branch-free body over 4 positions: wait for and read the body's four ring stages
        // (always stages st .. st + 3: the padding positions stream the zero row), then run the
        // four positions' arithmetic as one straight-line block (the row math unconditionally,
        // the sentinel row where none ends), so the compiler interleaves four independent
        // dependency chains instead of serialising position after position.
        int rows_done = 0, flushed = 0;  // pass A: rows whose partials are parked / summed
        // two instances of the loop: warps whose columns are all inside the vocabulary skip
        // pass A's per-column masks (only the last slice's boundary warp needs them)
        auto fast_loop = [&](auto FullTag) {
            for (int qq = qlo; qq < qhi; qq += 4) {
                Frag u[4];
#pragma unroll
                for (int S = 0; S < 4; ++S) {
                    mbar_wait(&full[st + S], ph);
                    u[S] = *reinterpret_cast<const Frag*>(ring + (st + S) * kStage + tid * sizeof(Frag));
                }
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int S = 0; S < 4; ++S) mbar_arrive(&empty[st + S]);
                }
                st += 4;
                if (st == kBandStages) {
                    st = 0;
                    ph ^= 1u;
                }
#pragma unroll
                for (int S = 0; S < 4; ++S) {
                    const int q = qq + S;
                    float2 x[kP];
                    unpack_frag(u[S], x);
#pragma unroll
                    for (int j = 0; j < kP; ++j) {
                        pr[S][j] = __fadd2_rn(xp[j], x[j]);
                        xp[j] = x[j];
                    }
                    const int i = m_end[q - qlo];
                    float2 z4[kP];
#pragma unroll
                    for (int j = 0; j < kP; ++j) z4[j] = __fadd2_rn(pr[(S + 2) & 3][j], pr[S][j]);
                    if constexpr (!kGrad) {
                        const float s = row_sum(z4, m_c[i], m_off[i], FullTag);
                        // partial sum parked in the warp's 32-row ring (slot i & 31)
                        if (i != kNoRow) {
                            redbuf[warp * 32 * kRedPitch + (i & 31) * kRedPitch + lane] = s;
                            rows_done = i + 1;
                        }
                    } else {
                        // columns past V hold arithmetic on stale bytes, zeroed when stored (flush_h)
                        row_grad(z4, m_c[i], m_off[i], m_ce[i], m_act[i] - static_cast<int>(v0) - d_lane, gr[S]);
                        flush_h(q - 3);
                    }
                }
                if constexpr (!kGrad) {
                    // a body ends <= 4 rows, so <= 19 rows are ever parked: every completed
                    // 16-row group (and the tail after the last body) goes to the stats column
                    while (rows_done - flushed >= 16 || (qq + 4 >= qhi && rows_done > flushed)) {
                        const int n = rows_done - flushed < 16 ? rows_done - flushed : 16;
                        flush_rows(flushed, n);
                        flushed += n;
                    }
                }
            }
        };
        if (warp_full) fast_loop(std::true_type{});
        else fast_loop(std::false_type{});
    }
}

}  // namespace

cudaError_t launch_positions(const uint8_t* arena, const SampleDesc* sd, int n_samples, int64_t row_lo, int64_t M,
                             uint64_t D, int32_t* feat, int64_t Qcap, cudaStream_t s) {
    if (Qcap == 0) return cudaSuccess;
    positions_kernel<<<static_cast<unsigned>((Qcap + 255) / 256), 256, 0, s>>>(arena, sd, n_samples, row_lo, M, D,
                                                                              feat, Qcap);
    return cudaGetLastError();
}

cudaError_t launch_fmax(const __nv_bfloat16* w16t, int64_t D, int64_t V, int64_t ldw, float* fmax, cudaStream_t s) {
    if (D == 0) return cudaSuccess;
    fmax_kernel<<<static_cast<unsigned>(D), 256, 0, s>>>(w16t, V, ldw, fmax);
    return cudaGetLastError();
}

cudaError_t launch_pslots(const int32_t* feat, int64_t Q, int nblk, int32_t* kcount, int32_t* kseg_off, int32_t* kiters,
                          int32_t* slot, __nv_bfloat16* bseg, int64_t bseg_rows, unsigned long long* rows_acc,
                          cudaStream_t s) {
    if (nblk <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(bseg, 0, static_cast<size_t>(bseg_rows) * 256 * 2, s);
    if (e != cudaSuccess) return e;
    const unsigned nch = static_cast<unsigned>(Q > 0 ? (Q + 1023) / 1024 : 1);
    pslot_count_kernel<<<dim3(nblk, nch), 1024, 0, s>>>(feat, Q, kcount, slot);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    int32_t* cbase = kcount + static_cast<size_t>(nblk) * nch;  // (the buffer holds both)
    pslot_scan_kernel<<<1, 1024, 2 * nblk * sizeof(int32_t), s>>>(kcount, nblk, static_cast<int>(nch), cbase, kseg_off,
                                                                  kiters, rows_acc);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    pslot_place_kernel<<<dim3(nblk, nch), 1024, 0, s>>>(feat, Q, cbase, slot, bseg, bseg_rows);
    return cudaGetLastError();
}

int band_stats_ld(int64_t V) {
    const int64_t cols = kBandConsumers * kCPL;
    return static_cast<int>((V + cols - 1) / cols) * (kBandConsumers / 32);
}

cudaError_t launch_band(const BandArgs& A, bool grad, cudaStream_t s) {
    if (A.M <= 0) return cudaSuccess;
    if (A.M + 3 * A.M >= INT32_MAX - 16) return cudaErrorInvalidValue;  // positions are int32
    auto go = [&](auto kern, int min_blocks, int cols, size_t smem) {
        // one CTA per item while there are >= 4 waves of them (min_blocks CTAs per SM); fewer
        // items (a vocabulary-gang rank's slices) run on persistent CTAs that stream item
        // after item without a partial last wave (measured at C2: 6.9 waves 0.209 vs
        // 0.219 ms K-stats one-per-item; 3.5 waves 0.150 vs 0.130 ms persistent).  The
        // persistent case takes 64-row items when that evens out the CTAs' loads (C2 gang
        // of 2: 1,024 items of 131 positions = 4 per CTA at most, 3.5 on average, vs
        // 2,048 of 67 = 7 / 6.9)
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t slots = static_cast<int64_t>(min_blocks) * sms;
        const int64_t nsl = (A.V + cols - 1) / cols;
        auto items_of = [&](int64_t r) { return nsl * ((A.M + r - 1) / r); };
        BandArgs B = A;
        B.rows_per_item = kBandRows;
        int64_t items = items_of(kBandRows);
        if (items < 4 * slots) {
            // the busiest CTA's positions for either item height (3 halo positions per item)
            auto load = [&](int64_t r) { return (items_of(r) + slots - 1) / slots * (r + 3); };
            if (load(kBandRows / 2) < load(kBandRows)) {
                B.rows_per_item = kBandRows / 2;
                items = items_of(kBandRows / 2);
            }
        }
        const int64_t grid = items >= 4 * slots ? items : (items < slots ? items : slots);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        kern<<<static_cast<unsigned>(grid), kBandThreads, smem, s>>>(B);
        return cudaGetLastError();
    };
    if (grad) return go(band_kernel<true, kBandMinBlocks>, kBandMinBlocks, kBandConsumers * kCPL, band_smem_bytes<true>());
    return go(band_kernel<false, kStatsMinBlocks>, kStatsMinBlocks, kBandConsumers * kCPL, band_smem_bytes<false>());
}

}  // namespace fm

// k_gemm_tc.cu — persistent, warp-specialised tcgen05 GEMM for the policy's
// two dense products:
//
//   K-GEMM1  Z[t][v]  = (1/n_t) * sum_d Phic[t][d] * W16[v][d]      (policy.hpp:57-61)
//            epilogue: p~ = exp(z - m) store + per-(row, 256-col tile) softmax
//            partials (max, sum exp) and the taken token's logit; with the loss
//            fold the CTA finishing a row block's last vocab tile also runs K-lse
//            for it (fused, fm_lse.cuh)                             (policy.hpp:62-75)
//   K-GEMM2  dW[v][d] (+)= sum_t G^T[v][t] * Phic^T[d][t]           (policy.hpp:83-90,
//            training.hpp:394-395, 444-446); epilogue RMW of the fp32 gradient
//            accumulator + sum(acc^2) of this micro-batch (training.hpp:417)
//
// Both are "TN" GEMMs  C[m][n] = sum_k A[m][k] * B[n][k]  with A and B bf16
// K-major in HBM.  Tiles: 128 x 256 x 64, 4-stage TMA->smem ring
// (SWIZZLE_128B), one elected thread issues tcgen05.mma (M128 N256 K16) into
// a double-buffered TMEM accumulator (2 x 256 fp32 columns), 4 epilogue warps
// drain TMEM with tcgen05.ld while the next tile's MMAs run.
//
// Warp roles (192 threads): w0 TMA producer, w1 MMA issuer (+TMEM owner),
// w2..w5 epilogue (w%4 selects the TMEM lane quadrant it may access).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "fm_gemm.h"
#include "fm_lse.cuh"
#include "fm_ptx.cuh"

namespace fm {

namespace {
constexpr int BM = kGemmBM, BN = kGemmBN, BK = kGemmBK, STAGES = kGemmStages;
constexpr uint32_t A_STAGE = BM * BK * 2;
constexpr uint32_t B_STAGE = BN * BK * 2;
constexpr uint32_t STAGE_BYTES = A_STAGE + B_STAGE;
constexpr uint32_t kIdesc = idesc_bf16_f32<BM, BN>();
constexpr uint32_t kTmemCols = 2 * BN;  // two accumulator buffers
constexpr int kThreads = 192;

struct TileCoord {
    int mb, nb;
};

__device__ __forceinline__ TileCoord tile_coord(int t, int tiles_m, int tiles_n, int group_m) {
    const int per_group = group_m * tiles_n;
    const int g = t / per_group;
    const int first_m = g * group_m;
    const int gsz = min(tiles_m - first_m, group_m);
    const int local = t - g * per_group;
    return TileCoord{first_m + local % gsz, local / gsz};
}

__device__ __forceinline__ float fast_exp(float x) { return exp2f(x * 1.4426950408889634f); }

// Fused K-lse (GEMM1, loss fold; opt-in FM_LSE_FUSED=1): once a CTA's
// epilogue warps have stored all their tiles, one thread releases the CTA's
// stores (named barrier + gpu-scope acq_rel fence, cumulative) and arrives on a
// grid counter; the last arriver resets it and publishes the launch's epoch,
// the others spin on the epoch (the persistent grid is one CTA per SM, all
// co-resident; a 2 s bound traps instead of hanging).  Then every epilogue warp
// of the grid runs the row normaliser (fm_lse.cuh) over a strided share of the
// rows — the work of the standalone K-lse launch, without the launch.
__device__ __forceinline__ void lse_grid_tail(const GemmArgs& a, int ew, int n_ew, double& loss) {
    named_bar_sync(1, 32 * n_ew);
    if (ew == 0 && (threadIdx.x & 31) == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const unsigned prev = atomicAdd(&a.lse_sync[0], 1u);
        if (prev == gridDim.x - 1) {
            a.lse_sync[0] = 0;  // for the next launch (stream-ordered after this one)
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.lse_sync + 1), "r"(a.lse_epoch) : "memory");
        } else {
            uint64_t t0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            for (;;) {
                unsigned e;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(e) : "l"(a.lse_sync + 1) : "memory");
                if (e == a.lse_epoch) break;
                __nanosleep(100);
                uint64_t t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > 2000000000ull) __trap();
            }
        }
    }
    named_bar_sync(1, 32 * n_ew);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const int64_t nw = static_cast<int64_t>(gridDim.x) * n_ew;
    for (int64_t r0 = (static_cast<int64_t>(blockIdx.x) * n_ew + ew) * 4; r0 < a.lse.Mpad; r0 += nw * 4)
        loss += lse_row_quad(a.lse, r0);
}

// ---- epilogues ------------------------------------------------------------

// One thread owns one accumulator row of the tile; it sees 32 consecutive
// columns per call.  State carried across the 8 column chunks of a tile.
// Two passes over the tile's TMEM columns: pass 1 finds the row's tile max
// (and captures the taken token's logit z_a in fp32); pass 2 stores
// p~ = exp(z - m_tile) as bf16 and accumulates sum p~.  K-lse turns the
// (m_tile, sum) partials into lse; K-loss rescales p~ by exp(m_tile - lse).
// Storing p~ (in (0,1], bf16 rel. error 2^-9) instead of fp32 z halves the
// logits round trip and keeps exp() out of K-loss.
struct LogitsEpi {
    static constexpr bool kTwoPass = true;
    float row_scale;
    float run_max, run_sum;
    int action;
    int4 slots;
    float* xbuf = nullptr;  // per-warp smem staging (token-slot stores)
    __device__ __forceinline__ void begin(const GemmArgs& a, int row) {
        const bool ok = row < a.M;
        row_scale = ok ? a.row_scale[row] : 0.f;
        action = ok ? a.action[row] : -1;
        if (a.aseg) {  // distinct A' rows of this token (duplicates -> -1)
            int4 q = ok ? a.slot4[row] : make_int4(-1, -1, -1, -1);
            if (q.y == q.x) q.y = -1;
            if (q.z == q.x || q.z == q.y) q.z = -1;
            if (q.w == q.x || q.w == q.y || q.w == q.z) q.w = -1;
            slots = q;
        }
        run_max = a.mrow ? (ok ? a.mrow[row] : 0.f) : -INFINITY;  // fold: the row's bound, known upfront
        run_sum = 0.f;
    }
    __device__ __forceinline__ void pass1(const GemmArgs& a, int row, int col0, uint32_t (&r)[32]) {
        if (row >= a.M) return;
        const int nvalid = min(32, a.N - col0);
        float cmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float z = __uint_as_float(r[j]) * row_scale;
            if (j < nvalid) cmax = fmaxf(cmax, z);
            if (col0 + j == action && j < nvalid) a.zact[row] = z;
        }
        run_max = fmaxf(run_max, cmax);
    }
    __device__ __forceinline__ void chunk(const GemmArgs& a, int row, int col0, uint32_t (&r)[32]) {
        const int nvalid = min(32, a.N - col0);
        if (a.pexp_t) {
            // loss-fold layout: p~^T [v][t] (GEMM2's K-major A operand), single TMEM pass
            // with the row bound as offset.  Lane pairs swap halves so that each store
            // writes a bf16x2 of two consecutive t: per v-pair the warp stores 2 x 64 B.
            if (nvalid <= 0) return;
            const bool live = row < a.M;
            const float m = run_max;
            const uint32_t lane = threadIdx.x & 31;
            const bool odd = lane & 1;
            float s = 0.f;
            __nv_bfloat16* dst = a.pexp_t + static_cast<size_t>(col0) * a.ldt + (row & ~1);
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                const float z0 = __uint_as_float(r[j]) * row_scale;
                const float z1 = __uint_as_float(r[j + 1]) * row_scale;
                if (col0 + j == action) a.zact[row] = z0;
                if (col0 + j + 1 == action) a.zact[row] = z1;
                const float p0 = (live && j < nvalid) ? fast_exp(z0 - m) : 0.f;
                const float p1 = (live && j + 1 < nvalid) ? fast_exp(z1 - m) : 0.f;
                s += p0 + p1;
                // even lane keeps column j and receives its odd neighbour's column j;
                // odd lane keeps column j+1 and receives the even neighbour's column j+1
                const float give = odd ? p0 : p1;
                const float got = __shfl_xor_sync(0xffffffffu, give, 1);
                const __nv_bfloat162 h = odd ? __floats2bfloat162_rn(got, p1) : __floats2bfloat162_rn(p0, got);
                const int jj = odd ? j + 1 : j;
                if (jj < nvalid && (row & ~1) < a.store_rows)
                    *reinterpret_cast<__nv_bfloat162*>(dst + static_cast<size_t>(jj) * a.ldt) = h;
            }
            run_sum += s;
            return;
        }
        if (nvalid <= 0) return;  // warp-uniform (col0 is the same for every lane)
        if (a.aseg) {
            seg_chunk(a, row, col0, nvalid, r);  // warp-cooperative: every lane takes part
            return;
        }
        if (row >= a.M) return;
        if (a.mrow) {  // single pass (K-list fold): the taken token's logit is caught here
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (col0 + j == action && j < nvalid) a.zact[row] = __uint_as_float(r[j]) * row_scale;
        }
        const float m = run_max;
        uint32_t pk[16];
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const float p0 = j < nvalid ? fast_exp(__uint_as_float(r[j]) * row_scale - m) : 0.f;
            const float p1 = j + 1 < nvalid ? fast_exp(__uint_as_float(r[j + 1]) * row_scale - m) : 0.f;
            s += p0 + p1;
            const __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
            pk[j >> 1] = *reinterpret_cast<const uint32_t*>(&h);
        }
        run_sum += s;
        __nv_bfloat16* dst = a.pexp + static_cast<size_t>(row) * a.ld_out + col0;
        if (nvalid == 32) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                reinterpret_cast<uint4*>(dst)[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j < nvalid) dst[j] = reinterpret_cast<const __nv_bfloat16*>(pk)[j];
        }
    }
    // Token-slot segments (K-list GEMM2 mode 2): p~ = exp(z - m_row) of the chunk goes
    // to every A' row of this token (one per feature block it touches).
    __device__ __forceinline__ void seg_chunk(const GemmArgs& a, int row, int col0, int nvalid, uint32_t (&r)[32]) {
        const bool live = row < a.M;
        if (live) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (col0 + j == action && j < nvalid) a.zact[row] = __uint_as_float(r[j]) * row_scale;
        }
        const float m = run_max;
        uint32_t pk[16];
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const float p0 = (live && j < nvalid) ? fast_exp(__uint_as_float(r[j]) * row_scale - m) : 0.f;
            const float p1 = (live && j + 1 < nvalid) ? fast_exp(__uint_as_float(r[j + 1]) * row_scale - m) : 0.f;
            s += p0 + p1;
            const __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
            pk[j >> 1] = *reinterpret_cast<const uint32_t*>(&h);
        }
        run_sum += s;
        if (nvalid < 32) {  // ragged last vocab tile: plain per-lane stores
            const int sl[4] = {slots.x, slots.y, slots.z, slots.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (sl[q] < 0) continue;
                __nv_bfloat16* d = a.aseg + static_cast<size_t>(sl[q]) * a.ld_out + col0;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < nvalid) d[j] = reinterpret_cast<const __nv_bfloat16*>(pk)[j];
            }
            return;
        }
        // Stage the warp's 32 rows x 64 B through smem, then write each (row, slot)
        // piece with 4 lanes x 16 B: every store instruction covers 8 rows' full
        // 32-B sectors (per-lane 16-B stores to 32 different rows left half-sector
        // writes that L2 filled from DRAM: +5 GB reads per launch)
        const uint32_t lane = threadIdx.x & 31;
        uint4* xb = reinterpret_cast<uint4*>(xbuf);  // 32 rows x 5 uint4 (80-B pitch)
#pragma unroll
        for (int i = 0; i < 4; ++i) xb[lane * 5 + i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        __syncwarp();
        const int part = static_cast<int>(lane & 3);
        const uint64_t pol = policy_evict_first();  // 3.6 GB stream, read back by GEMM2 from DRAM
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const int rr = g * 8 + static_cast<int>(lane >> 2);
            const uint4 v = xb[rr * 5 + part];
            const int s0 = __shfl_sync(0xffffffffu, slots.x, rr), s1 = __shfl_sync(0xffffffffu, slots.y, rr);
            const int s2 = __shfl_sync(0xffffffffu, slots.z, rr), s3 = __shfl_sync(0xffffffffu, slots.w, rr);
            const int sl[4] = {s0, s1, s2, s3};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (sl[q] >= 0 && !a.dbg_nostore)
                    st_global_v4_hint(reinterpret_cast<uint4*>(a.aseg + static_cast<size_t>(sl[q]) * a.ld_out + col0) + part,
                                      v, pol);
        }
        __syncwarp();
        return;
    }

    __device__ __forceinline__ void end(const GemmArgs& a, int row, int nb) {
        if (row < a.M) a.stats[static_cast<size_t>(row) * a.stats_ld + nb] = make_float2(run_max, run_sum);
    }
};

struct GradEpi {
    static constexpr bool kTwoPass = false;
    double sumsq;
    __device__ __forceinline__ void pass1(const GemmArgs&, int, int, uint32_t (&)[32]) {}
    __device__ __forceinline__ void begin(const GemmArgs&, int) {}
    float* xbuf = nullptr;  // per-warp 32 x 36 fp32 smem staging (exchange mode)

    // Warp-cooperative: lane = row holds 32 columns; transpose through smem so
    // each store instruction writes 4 whole 128-B rows (8 lanes x 16 B per
    // row) — NVLink moves full lines instead of 16-B fragments.
    __device__ __forceinline__ void remote_chunk(const GemmArgs& a, int row, int col0, uint32_t (&r)[32], int o) {
        const uint32_t lane = threadIdx.x & 31;
        const int nvalid = min(32, a.N - col0);
        const bool vrow = row < a.M && nvalid > 0;
        const float* src = a.out + static_cast<size_t>(row) * a.ld_out + col0;
        float part = 0.f;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            float4 acc = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                     __uint_as_float(r[j + 3]));
            if (vrow && j < nvalid) {
                part += acc.x * acc.x + acc.y * acc.y + acc.z * acc.z + acc.w * acc.w;
                if (a.accumulate) {
                    const float4 o4 = *reinterpret_cast<const float4*>(src + j);
                    acc.x += o4.x;
                    acc.y += o4.y;
                    acc.z += o4.z;
                    acc.w += o4.w;
                }
            }
            *reinterpret_cast<float4*>(xbuf + lane * 36 + j) = acc;
        }
        sumsq += static_cast<double>(part);
        __syncwarp();
        const int row0 = row - static_cast<int>(lane);
        const int seg = static_cast<int>(lane & 7);
        float* base = a.xpeer[o] + static_cast<size_t>(col0) + static_cast<size_t>(seg) * 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + static_cast<int>(lane >> 3);
            const int rg = row0 + rr;
            if (rg < a.M && seg * 4 < nvalid) {
                const float4 q = *reinterpret_cast<const float4*>(xbuf + rr * 36 + seg * 4);
                *reinterpret_cast<float4*>(base + static_cast<size_t>(rg - a.xlo[o]) * a.ld_out) = q;
            }
        }
        __syncwarp();
    }
    __device__ __forceinline__ void chunk(const GemmArgs& a, int row, int col0, uint32_t (&r)[32]) {
        if (a.xg > 1) {
            // DP gang exchange (last micro-batch of the step): rows owned by another rank
            // get this rank's whole partial (previous micro-batches + this tile) written
            // straight into the owner's receive slot over NVLink — the reduce-scatter
            // happens inside the GEMM epilogue, overlapped with the next tile's MMAs.
            // Owner shards are 256-row aligned, so a warp's 32 rows share one owner.
            int o = 0;
#pragma unroll 1
            while (o + 1 < a.xg && row >= a.xlo[o + 1]) ++o;
            if (o != a.xrank) {
                remote_chunk(a, row, col0, r, o);
                return;
            }
        }
        const int nvalid = min(32, a.N - col0);
        if (nvalid <= 0) return;  // warp-uniform
        if (nvalid == 32 && xbuf) {
            // transposed read-modify-write: stage the warp's 32 rows x 32 columns in smem,
            // then every load / store instruction covers 4 whole 128-B rows (8 lanes x 16 B
            // per row) instead of 32 rows x 16 B — the RMW of dW bounds GEMM2 when a tile's
            // K range is short (C3: 128 feature blocks, ~8 K iterations per tile)
            const uint32_t lane = threadIdx.x & 31;
            float part = 0.f;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 acc = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                               __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                if (row < a.M) part += acc.x * acc.x + acc.y * acc.y + acc.z * acc.z + acc.w * acc.w;
                *reinterpret_cast<float4*>(xbuf + lane * 36 + j) = acc;
            }
            sumsq += static_cast<double>(part);
            __syncwarp();
            const int row0 = row - static_cast<int>(lane);
            const int seg = static_cast<int>(lane & 7);
            float4 o[8];
            if (a.accumulate) {  // all eight loads in flight before any store
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int rg = row0 + i * 4 + static_cast<int>(lane >> 3);
                    o[i] = rg < a.M ? __ldcg(reinterpret_cast<const float4*>(a.out + static_cast<size_t>(rg) * a.ld_out + col0) + seg)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int rr = i * 4 + static_cast<int>(lane >> 3);
                const int rg = row0 + rr;
                float4 q = *reinterpret_cast<const float4*>(xbuf + rr * 36 + seg * 4);
                if (a.accumulate) {
                    q.x += o[i].x;
                    q.y += o[i].y;
                    q.z += o[i].z;
                    q.w += o[i].w;
                }
                if (rg < a.M) *(reinterpret_cast<float4*>(a.out + static_cast<size_t>(rg) * a.ld_out + col0) + seg) = q;
            }
            __syncwarp();
            return;
        }
        if (row >= a.M) return;
        const float* src = a.out + static_cast<size_t>(row) * a.ld_out + col0;  // this rank's partial
        float* dst = const_cast<float*>(src);
        float part = 0.f;
        if (nvalid == 32) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                float4 acc = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                         __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                part += acc.x * acc.x + acc.y * acc.y + acc.z * acc.z + acc.w * acc.w;
                if (a.accumulate) {
                    const float4 o4 = *reinterpret_cast<const float4*>(src + j);
                    acc.x += o4.x;
                    acc.y += o4.y;
                    acc.z += o4.z;
                    acc.w += o4.w;
                }
                *reinterpret_cast<float4*>(dst + j) = acc;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j < nvalid) {
                    const float acc = __uint_as_float(r[j]);
                    part += acc * acc;
                    dst[j] = a.accumulate ? src[j] + acc : acc;
                }
            }
        }
        sumsq += static_cast<double>(part);
    }
    __device__ __forceinline__ void end(const GemmArgs&, int, int) {}
};

template <class Epi>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   GemmArgs args) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);  // one arrive per epilogue warp
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tiles_m = (args.M + BM - 1) / BM;
    const int tiles_n = (args.N + BN - 1) / BN;
    const int num_tiles = tiles_m * tiles_n;
    const int k_iters = (args.K + BK - 1) / BK;

    if (warp == 0) {
        // ===== TMA producer =====
        if (elect_one()) {
            const uint64_t pol_a = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                const TileCoord tc = tile_coord(t, tiles_m, tiles_n, args.group_m);
                for (int k = 0; k < k_iters; ++k) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
                    tma_load_2d_hint(sA + stage * A_STAGE, &tmA, &full[stage], args.k0 + k * BK, tc.mb * BM, pol_a);
                    tma_load_2d_hint(sB + stage * B_STAGE, &tmB, &full[stage], args.k0 + k * BK, tc.nb * BN, pol_a);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (single elected thread) =====
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int k = 0; k < k_iters; ++k) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t adesc = umma_desc_k_sw128(smem_u32(sA + stage * A_STAGE));
                    const uint64_t bdesc = umma_desc_k_sw128(smem_u32(sB + stage * B_STAGE));
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        // advance 16 bf16 = 32 B along K inside the 128 B swizzle atom
                        umma_bf16(d_tmem, adesc + static_cast<uint64_t>(kk * 2),
                                  bdesc + static_cast<uint64_t>(kk * 2), kIdesc, (k | kk) != 0);
                    }
                    umma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
        __syncwarp();
    } else {
        // ===== epilogue warps =====
        const uint32_t quad = warp & 3;
        const int row_in_tile = static_cast<int>(quad * 32 + lane);
        Epi epi;
        int acc = 0;
        uint32_t acc_phase = 0;
        double sumsq_total = 0.0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const TileCoord tc = tile_coord(t, tiles_m, tiles_n, args.group_m);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row = tc.mb * BM + row_in_tile;
            if constexpr (std::is_same_v<Epi, GradEpi>) {
                epi.begin(args, row);
                epi.sumsq = 0.0;
            }
            if (Epi::kTwoPass && !args.mrow) {
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + static_cast<uint32_t>(acc * BN + c * 32), r);
                    tmem_ld_wait();
                    epi.pass1(args, row, tc.nb * BN + c * 32, r);
                }
            }
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + static_cast<uint32_t>(acc * BN + c * 32), r);
                tmem_ld_wait();
                epi.chunk(args, row, tc.nb * BN + c * 32, r);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            epi.end(args, row, tc.nb);
            if constexpr (std::is_same_v<Epi, GradEpi>) sumsq_total += epi.sumsq;
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if constexpr (std::is_same_v<Epi, GradEpi>) {
            for (int o = 16; o > 0; o >>= 1) sumsq_total += __shfl_xor_sync(0xffffffffu, sumsq_total, o);
            if (lane == 0 && args.sumsq) atomicAdd(args.sumsq, sumsq_total);
        }
    }
    __syncthreads();
    if (warp == 1) tmem_dealloc<kTmemCols>(tmem_base);
}

// ---------------------------------------------------------------------------
// CTA-pair variant: a 2-CTA cluster computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M256 N256 K16).  Each CTA TMA-loads its own 128
// rows of A and its half (128 rows) of B per stage (32 KB), so the pair moves
// 3/4 of the operand bytes two single-CTA 128x256 tiles would; the leader CTA
// issues every MMA and commits to both CTAs' barriers; each CTA drains its
// own 128-lane half of the accumulator from its TMEM.
// ---------------------------------------------------------------------------
// Work schedule of the pair kernel.  Data-parallel tiles round-robin over the
// pairs; with stream-K (Grad, tiles % pairs != 0) the last
// (tiles - (waves-1)*pairs) tiles are cut into equal contiguous K-iteration
// ranges, one per pair, so no pair idles through a mostly empty last wave.
struct WorkItem {
    int tile, kb, ke;
    int sk;  // stream-K tile slot when only part of the tile's K range is here, else -1
};
struct Sched {
    int T, Kt, P, T_dp;
    long long U;  // stream-K K-iterations in total
    __device__ __forceinline__ Sched(int tiles, int k_iters, int pairs, bool streamk) {
        T = tiles;
        Kt = k_iters;
        P = pairs;
        const int waves = tiles / pairs;
        if (streamk && waves >= 1 && tiles % pairs != 0) {
            T_dp = (waves - 1) * pairs;
            U = static_cast<long long>(tiles - T_dp) * k_iters;
        } else {
            T_dp = tiles;
            U = 0;
        }
    }
    __device__ __forceinline__ long long ustart(int c) const { return static_cast<long long>(c) * U / P; }
    __device__ __forceinline__ int pair_of(long long u) const {
        int c = static_cast<int>(u * P / U);
        while (c + 1 < P && ustart(c + 1) <= u) ++c;
        while (c > 0 && ustart(c) > u) --c;
        return c;
    }
    // number of pairs whose K ranges cover stream-K tile slot lt
    __device__ __forceinline__ int contributors(int lt) const {
        const long long a = static_cast<long long>(lt) * Kt;
        return pair_of(a + Kt - 1) - pair_of(a) + 1;
    }
    __device__ __forceinline__ bool get(int cid, int w, WorkItem& wi) const {
        const int ndp = cid < T_dp ? (T_dp - cid + P - 1) / P : 0;
        if (w < ndp) {
            wi = WorkItem{cid + w * P, 0, Kt, -1};
            return true;
        }
        if (U == 0) return false;
        const long long u0 = ustart(cid), u1 = ustart(cid + 1);
        const long long st = (w == ndp) ? u0 : (u0 / Kt + (w - ndp)) * static_cast<long long>(Kt);
        if (st >= u1) return false;
        const long long en = min(u1, (st / Kt + 1) * static_cast<long long>(Kt));
        const int lt = static_cast<int>(st / Kt);
        wi.tile = T_dp + lt;
        wi.kb = static_cast<int>(st % Kt);
        wi.ke = wi.kb + static_cast<int>(en - st);
        wi.sk = (wi.kb == 0 && wi.ke == Kt) ? -1 : lt;
        return true;
    }
};

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

constexpr int P_STAGES = 6;
constexpr uint32_t P_A_STAGE = 128 * BK * 2;    // 16 KB: this CTA's 128 rows of A
constexpr uint32_t P_B_STAGE = 128 * BK * 2;    // 16 KB: this CTA's half of B's 256 rows
constexpr uint32_t P_STAGE_BYTES = P_A_STAGE + P_B_STAGE;

constexpr int kThreadsPair = 192;  // w0 TMA, w1 MMA, w2-5 epilogue

// kAmn / kBmn: operand stored MN-major in HBM ([K][M] / [K][N], MN contiguous);
// each CTA's 128 MN x 64 K stage slice is then two TMA boxes {64 MN, 64 K}
// (8 KB each, the second at +8 KB = the descriptor's LBO).
// kKList (Grad): both operands MN-major row-major [rows][.] gathered with TMA
// gather4 from the output column tile's K list (args.klist*).
// kSeg (Grad): both operands MN-major; column tile nb runs the K rows of its
// token-slot segment (args.kseg_off / klist_iters); B' holds only 256 columns.
// kSwA (with kSeg): warps 6-9 of each CTA gather the A rows (p~ rows of the
// segment's tokens) with 16-B loads and write them into the swizzled MN-major
// stage; they and the B TMA arrive on the leader's full barrier (1 + 8 arrivals).
template <class Epi, bool kAmn = false, bool kBmn = false, bool kKList = false, bool kSeg = false, bool kSwA = false,
          int kEpiW = 4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((kSwA || kEpiW == 8) ? 320 : kThreadsPair, 1)
    gemm_tn_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       GemmArgs args) {
    static_assert(!kKList || (kAmn && kBmn), "K-list operands are MN-major");
    static_assert(!kSeg || (kAmn && kBmn), "segment operands are MN-major");
    static_assert(!kSwA || kSeg, "software A gather runs the segment schedule");
    constexpr uint32_t kId = idesc_bf16_f32<256, BN, kAmn, kBmn>();
    // kEpiW = 8: the accumulator is drained by two warps per TMEM lane quadrant, each
    // half the columns — GEMM1 with short K (its exp + p~ slot stores outlast the MMAs)
    static_assert(kEpiW == 4 || (kEpiW == 8 && std::is_same_v<Epi, LogitsEpi>), "8 epilogue warps: GEMM1 only");
    constexpr int kEW = kEpiW;
    constexpr int kSplit = kEW / 4;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + P_STAGES * P_A_STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE_BYTES);
    uint64_t* empty = full + P_STAGES;
    uint64_t* tfull = empty + P_STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* xscratch = reinterpret_cast<float*>(tmem_slot + 4);  // 4 warps x 32 x 36 fp32 (16-B aligned)

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < P_STAGES; ++s) {
            mbar_init(&full[s], kSwA ? 9 : 1);  // the leader's producer arrives with both CTAs' tx bytes
            mbar_init(&empty[s], 1);            // one multicast commit per consumed stage
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 2 * kEW);  // epilogue warps x 2 CTAs (leader's copy is the one used)
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_2sm<kTmemCols>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tiles_m = (args.M + 255) / 256;
    const int tiles_n = (args.N + BN - 1) / BN;
    const int num_tiles = tiles_m * tiles_n;
    const int k_iters = (args.K + BK - 1) / BK;
    const int cid = blockIdx.x >> 1;
    const int nclusters = gridDim.x >> 1;
    const Sched sch(num_tiles, k_iters, nclusters, std::is_same_v<Epi, GradEpi> && args.sk_ws != nullptr);

    if (warp == 0 && kKList) {
        // ===== TMA gather producer (both CTAs; lanes 0-15 each gather one row quad) =====
        const uint64_t pol = policy_evict_last();
        int stage = 0;
        uint32_t phase = 0;
        WorkItem wi;
        for (int w = 0; sch.get(cid, w, wi); ++w) {
            const TileCoord tc = tile_coord(wi.tile, tiles_m, tiles_n, args.group_m);
            const int ke = __ldg(args.klist_iters + tc.nb);
            const int arow = tc.mb * 256 + static_cast<int>(rank) * 128;
            const int brow = tc.nb * BN + static_cast<int>(rank) * 128;
            const int32_t* lst = args.klist + static_cast<size_t>(tc.nb) * args.klist_ld;
            for (int k = 0; k < ke; ++k) {
                mbar_wait(&empty[stage], phase ^ 1);
                const uint32_t fb = mapa_shared(&full[stage], 0);
                if (leader && lane == 0) mbar_arrive_expect_tx(&full[stage], 2 * P_STAGE_BYTES);
                if (lane < 16) {
                    const int4 t4 = __ldg(reinterpret_cast<const int4*>(lst + k * BK) + lane);
                    uint8_t* a0 = sA + stage * P_A_STAGE + lane * 512;
                    uint8_t* b0 = sB + stage * P_B_STAGE + lane * 512;
                    tma_gather4_2sm(a0, &tmA, fb, arow, t4, pol);
                    tma_gather4_2sm(a0 + 8192, &tmA, fb, arow + 64, t4, pol);
                    tma_gather4_2sm(b0, &tmB, fb, brow, t4, pol);
                    tma_gather4_2sm(b0 + 8192, &tmB, fb, brow + 64, t4, pol);
                }
                __syncwarp();
                if (++stage == P_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 0) {
        // ===== TMA producer (both CTAs) =====
        if (elect_one()) {
            const uint64_t pol = policy_evict_last();
            // segmented GEMM2: each A' segment block is read by exactly one tile
            const uint64_t pol_a = kSeg ? policy_evict_first() : pol;
            int stage = 0;
            uint32_t phase = 0;
            WorkItem wi;
            for (int w = 0; sch.get(cid, w, wi); ++w) {
                const TileCoord tc = tile_coord(wi.tile, tiles_m, tiles_n, args.group_m);
                const int arow = tc.mb * 256 + static_cast<int>(rank) * 128;
                const int brow = (kSeg ? 0 : tc.nb * BN) + static_cast<int>(rank) * 128;
                int kbase = args.k0;
                if constexpr (kSeg) {
                    kbase = __ldg(args.kseg_off + tc.nb);
                    wi.ke = __ldg(args.klist_iters + tc.nb);
                }
                for (int k = wi.kb; k < wi.ke; ++k) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t fb = mapa_shared(&full[stage], 0);
                    if (leader) mbar_arrive_expect_tx(&full[stage], kSwA ? 2 * P_B_STAGE : 2 * P_STAGE_BYTES);
                    const int kc = kbase + k * BK;
                    if constexpr (kSwA) {
                        // A comes from the gather warps
                    } else if constexpr (kAmn) {
                        tma_load_2d_2sm(sA + stage * P_A_STAGE, &tmA, fb, arow, kc, pol_a);
                        tma_load_2d_2sm(sA + stage * P_A_STAGE + 8192, &tmA, fb, arow + 64, kc, pol_a);
                    } else {
                        tma_load_2d_2sm(sA + stage * P_A_STAGE, &tmA, fb, kc, arow, pol);
                    }
                    if constexpr (kBmn) {
                        tma_load_2d_2sm(sB + stage * P_B_STAGE, &tmB, fb, brow, kc, pol);
                        tma_load_2d_2sm(sB + stage * P_B_STAGE + 8192, &tmB, fb, brow + 64, kc, pol);
                    } else {
                        tma_load_2d_2sm(sB + stage * P_B_STAGE, &tmB, fb, kc, brow, pol);
                    }
                    if (++stage == P_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: leader CTA only =====
        if (leader && elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            WorkItem wi;
            for (int w = 0; sch.get(cid, w, wi); ++w) {
                if constexpr (kKList || kSeg)
                    wi.ke = __ldg(args.klist_iters + tile_coord(wi.tile, tiles_m, tiles_n, args.group_m).nb);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int k = wi.kb; k < wi.ke; ++k) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    // K-major: 16 bf16 = 32 B along the swizzle row; MN-major: 16 K rows = 2 KB
                    const uint64_t adesc = kAmn ? umma_desc_mn_sw128(smem_u32(sA + stage * P_A_STAGE), 8192)
                                                : umma_desc_k_sw128(smem_u32(sA + stage * P_A_STAGE));
                    const uint64_t bdesc = kBmn ? umma_desc_mn_sw128(smem_u32(sB + stage * P_B_STAGE), 8192)
                                                : umma_desc_k_sw128(smem_u32(sB + stage * P_B_STAGE));
                    constexpr uint64_t a_step = kAmn ? 2048 >> 4 : 2;
                    constexpr uint64_t b_step = kBmn ? 2048 >> 4 : 2;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        umma_bf16_2sm(d_tmem, adesc + a_step * kk, bdesc + b_step * kk, kId,
                                      (k != wi.kb || kk != 0));
                    umma_commit_2sm(&empty[stage], 0x3);
                    if (++stage == P_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_2sm(&tfull[acc], 0x3);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
        __syncwarp();
    } else if (kSwA && warp >= 6) {
        // ===== A gather (both CTAs): warp aw copies K rows 16aw..16aw+15 of each stage =====
        // cp.async 16-B pieces straight into the swizzled MN-major stage, one commit group
        // per stage; a stage is released to the MMA (proxy fence + cluster arrive on the
        // leader's full barrier) once it is two groups old, so three stages of loads are
        // in flight per warp without staging registers.
        const int aw = static_cast<int>(warp) - 6;
        int stage = 0;
        uint32_t phase = 0;
        int pend[2] = {-1, -1};  // stages issued but not yet released (oldest first)
        auto release_oldest = [&](bool all) {
            if (all) asm volatile("cp.async.wait_group 0;" ::: "memory");
            else asm volatile("cp.async.wait_group 2;" ::: "memory");
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(&full[pend[0]], 0));
            pend[0] = pend[1];
            pend[1] = -1;
        };
        WorkItem wi;
        for (int w = 0; sch.get(cid, w, wi); ++w) {
            const TileCoord tc = tile_coord(wi.tile, tiles_m, tiles_n, args.group_m);
            const int arow = tc.mb * 256 + static_cast<int>(rank) * 128;
            const int kbase = __ldg(args.kseg_off + tc.nb);
            const int ke = __ldg(args.klist_iters + tc.nb);
            for (int k = 0; k < ke; ++k) {
                const int tok_l = lane < 16 ? __ldg(args.seg_tok + kbase + k * BK + 16 * aw + static_cast<int>(lane)) : 0;
                mbar_wait(&empty[stage], phase ^ 1);
                const uint32_t base = smem_u32(sA + stage * P_A_STAGE);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int q = static_cast<int>(lane) + 32 * i;  // 16 tokens x 16 pieces of 16 B
                    const int t = __shfl_sync(0xffffffffu, tok_l, q >> 4);
                    const int r = 16 * aw + (q >> 4), p = q & 15, h = p >> 3, c = p & 7;
                    const int v0 = arow + 8 * p;
                    const uint32_t dst = base + h * 8192 + r * 128 + ((c ^ (r & 7)) << 4);
                    const __nv_bfloat16* src = args.pexp + static_cast<size_t>(t) * args.ld_pexp + v0;
                    const uint32_t nbytes = v0 < args.M ? 16u : 0u;  // zero-fill past the vocab
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(nbytes)
                                 : "memory");
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
                if (pend[1] >= 0) release_oldest(false);  // the stage issued two groups ago
                if (pend[0] < 0) pend[0] = stage;
                else pend[1] = stage;
                if (++stage == P_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        while (pend[0] >= 0) release_oldest(true);
    } else {
        // ===== epilogue warps 2..(1+kEW) (both CTAs; each CTA drains its own 128 rows) =====
        const uint32_t quad = warp & 3;  // TMEM lane quadrant this warp may access
        const int ew = static_cast<int>(warp) - 2;
        const int half = ew / 4;         // column part of the tile (kSplit parts)
        constexpr int kCh = BN / 32 / kSplit;
        const int c0 = half * kCh, c1 = c0 + kCh;
        const int row_in_tile = static_cast<int>(rank * 128 + quad * 32 + lane);
        const uint32_t tempty_leader[2] = {mapa_shared(&tempty[0], 0), mapa_shared(&tempty[1], 0)};
        Epi epi;
        epi.xbuf = kEW == 8 ? xscratch + ew * 32 * 20 : xscratch + quad * 32 * 36;
        int acc = 0;
        uint32_t acc_phase = 0;
        double sumsq_total = 0.0;
        double lse_loss = 0.0;
        __shared__ int sk_flag;
        WorkItem wi;
        for (int w = 0; sch.get(cid, w, wi); ++w) {
            const TileCoord tc = tile_coord(wi.tile, tiles_m, tiles_n, args.group_m);
            const int row = tc.mb * 256 + row_in_tile;
            // per-row epilogue operands (scale, action, bound, token slots) are loaded while
            // the accumulator is still being produced, not after it is ready
            if constexpr (std::is_same_v<Epi, LogitsEpi>) epi.begin(args, row);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if constexpr (std::is_same_v<Epi, GradEpi>) {
                if (wi.sk >= 0) {
                    // stream-K partial: add this K range's accumulator into the tile's
                    // workspace, then count the arrival; the last of the tile half's
                    // contributors runs the epilogue on the summed tile
                    float* wrow = args.sk_ws + (static_cast<size_t>(wi.sk) * 256 + row_in_tile) * BN;
#pragma unroll 1
                    for (int c = 0; c < BN / 32; ++c) {
                        uint32_t r[32];
                        tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + static_cast<uint32_t>(acc * BN + c * 32), r);
                        tmem_ld_wait();
                        if (c == BN / 32 - 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader[acc]);
                        }
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            red_add_v4(wrow + c * 32 + j, __uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                       __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                    }
                    named_bar_sync(1, 128);
                    if (quad == 0 && lane == 0) {
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        int* cnt = args.sk_cnt + wi.sk * 2 + static_cast<int>(rank);
                        const int last = atomicAdd(cnt, 1) == sch.contributors(wi.sk) - 1;
                        if (last) *cnt = 0;
                        sk_flag = last;
                    }
                    named_bar_sync(1, 128);
                    if (sk_flag) {
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        epi.begin(args, row);
                        epi.sumsq = 0.0;
#pragma unroll 1
                        for (int c = 0; c < BN / 32; ++c) {
                            uint32_t r[32];
                            float4* src = reinterpret_cast<float4*>(wrow + c * 32);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 v = __ldcg(src + q);
                                r[4 * q] = __float_as_uint(v.x);
                                r[4 * q + 1] = __float_as_uint(v.y);
                                r[4 * q + 2] = __float_as_uint(v.z);
                                r[4 * q + 3] = __float_as_uint(v.w);
                                __stcg(src + q, make_float4(0.f, 0.f, 0.f, 0.f));  // zero for the next launch
                            }
                            epi.chunk(args, row, tc.nb * BN + c * 32, r);
                        }
                        epi.end(args, row, tc.nb);
                        sumsq_total += epi.sumsq;
                    }
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                    continue;
                }
            }
            epi.begin(args, row);
            if constexpr (std::is_same_v<Epi, GradEpi>) epi.sumsq = 0.0;
            if (Epi::kTwoPass && !args.mrow) {
#pragma unroll 1
                for (int c = c0; c < c1; ++c) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + static_cast<uint32_t>(acc * BN + c * 32), r);
                    tmem_ld_wait();
                    epi.pass1(args, row, tc.nb * BN + c * 32, r);
                }
            }
#pragma unroll 1
            for (int c = c0; c < c1; ++c) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + static_cast<uint32_t>(acc * BN + c * 32), r);
                tmem_ld_wait();
                if (c == c1 - 1) {
                    // the accumulator is fully in registers: hand TMEM back to the MMA
                    // warp before the last chunk's math and stores (relaxed: no wait
                    // for this warp's outstanding global stores)
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader[acc]);
                }
                epi.chunk(args, row, tc.nb * BN + c * 32, r);
            }
            epi.end(args, row, tc.nb * kSplit + half);  // softmax partials per column part
            if constexpr (std::is_same_v<Epi, GradEpi>) sumsq_total += epi.sumsq;
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if constexpr (std::is_same_v<Epi, GradEpi>) {
            for (int o = 16; o > 0; o >>= 1) sumsq_total += __shfl_xor_sync(0xffffffffu, sumsq_total, o);
            if (lane == 0 && args.sumsq) atomicAdd(args.sumsq, sumsq_total);
        }
        if constexpr (std::is_same_v<Epi, LogitsEpi>) {
            if (args.lse_sync) {
                lse_grid_tail(args, ew, kEW, lse_loss);
                for (int o = 16; o > 0; o >>= 1) lse_loss += __shfl_xor_sync(0xffffffffu, lse_loss, o);
                if (lane == 0 && args.lse.loss_acc && lse_loss != 0.0) atomicAdd(args.lse.loss_acc, lse_loss);
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm<kTmemCols>(tmem_base);
    }
}

bool use_pair_mma() {
    static const bool on = [] {
        const char* e = getenv("FM_GEMM_2SM");
        return !(e && e[0] == '0');
    }();
    return on;
}

}  // namespace

// Test hook: C[M][N] (fp32, ld N) = sum_k A(m,k) B(n,k) with A / B either K-major
// ([M][K] / [N][K]) or MN-major ([K][M] / [K][N]) — validates the MN-major UMMA
// operand path against a plain reference (tests/test_gpu_path.py).
cudaError_t gemm_debug_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, int a_mn, int b_mn, int M, int N,
                              int K, float* C, int num_sms, cudaStream_t stream) {
    GemmArgs args{};
    args.M = M;
    args.N = N;
    args.K = K;
    args.group_m = 8;
    args.out = C;
    args.ld_out = N;
    const size_t smem = gemm_smem_bytes();
    const int tiles = ((M + 255) / 256) * ((N + BN - 1) / BN);
    const int pairs = num_sms / 2;
    const int grid = 2 * (tiles < pairs ? tiles : pairs);
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, kThreadsPair, smem, stream>>>(tmA, tmB, args);
    };
    if (a_mn && b_mn) launch(gemm_tn_2sm_kernel<GradEpi, true, true>);
    else if (a_mn) launch(gemm_tn_2sm_kernel<GradEpi, true, false>);
    else if (b_mn) launch(gemm_tn_2sm_kernel<GradEpi, false, true>);
    else launch(gemm_tn_2sm_kernel<GradEpi, false, false>);
    return cudaGetLastError();
}

cudaError_t gemm_kseg_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& args, int num_sms,
                             cudaStream_t stream) {
    const size_t smem = gemm_smem_bytes();
    const int tiles = ((args.M + 255) / 256) * ((args.N + BN - 1) / BN);
    if (tiles == 0) return cudaSuccess;
    const int pairs = num_sms / 2;
    const int grid = 2 * (tiles < pairs ? tiles : pairs);
    auto k = gemm_tn_2sm_kernel<GradEpi, true, true, false, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<grid, kThreadsPair, smem, stream>>>(tmA, tmB, args);
    return cudaGetLastError();
}

cudaError_t gemm_kseg_swa_launch(const CUtensorMap& tmB, const GemmArgs& args, int num_sms, cudaStream_t stream) {
    const size_t smem = gemm_smem_bytes();
    const int tiles = ((args.M + 255) / 256) * ((args.N + BN - 1) / BN);
    if (tiles == 0) return cudaSuccess;
    const int pairs = num_sms / 2;
    const int grid = 2 * (tiles < pairs ? tiles : pairs);
    auto k = gemm_tn_2sm_kernel<GradEpi, true, true, false, true, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<grid, 320, smem, stream>>>(tmB, tmB, args);
    return cudaGetLastError();
}

cudaError_t gemm_klist_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& args, int num_sms,
                              cudaStream_t stream) {
    const size_t smem = gemm_smem_bytes();
    const int tiles = ((args.M + 255) / 256) * ((args.N + BN - 1) / BN);
    if (tiles == 0) return cudaSuccess;
    const int pairs = num_sms / 2;
    const int grid = 2 * (tiles < pairs ? tiles : pairs);
    auto k = gemm_tn_2sm_kernel<GradEpi, true, true, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<grid, kThreadsPair, smem, stream>>>(tmA, tmB, args);
    return cudaGetLastError();
}

// Loss-fold path (default; FM_LOSS_FOLD=0 restores the separate K-loss pass).
bool loss_fold_enabled() {
    static const bool on = [] {
        const char* e = getenv("FM_LOSS_FOLD");
        return !(e && e[0] == '0');
    }();
    return on;
}


size_t gemm_smem_bytes() {
    return use_pair_mma() ? P_STAGES * P_STAGE_BYTES + 1024 + 512 + 8 * 32 * 20 * 4  // >= 4 x 32 x 36 fp32
                          : STAGES * STAGE_BYTES + 1024 + 256;
}

uint32_t gemm_b_box_rows() { return use_pair_mma() ? 128u : static_cast<uint32_t>(BN); }

bool gemm_pair_mode() { return use_pair_mma(); }

cudaError_t gemm_tn_launch(GemmKind kind, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const GemmArgs& args, int num_sms, cudaStream_t stream) {
    const size_t smem = gemm_smem_bytes();
    if (use_pair_mma()) {
        const int tiles = ((args.M + 255) / 256) * ((args.N + BN - 1) / BN);
        if (tiles == 0) return cudaSuccess;
        const int pairs = num_sms / 2;
        const int grid = 2 * (tiles < pairs ? tiles : pairs);
        if (kind == GemmKind::Logits) {
            if (args.epi_wide) {  // 8 epilogue warps
                auto k = gemm_tn_2sm_kernel<LogitsEpi, false, false, false, false, false, 8>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                k<<<grid, 320, smem, stream>>>(tmA, tmB, args);
            } else {
                auto k = gemm_tn_2sm_kernel<LogitsEpi>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                k<<<grid, kThreadsPair, smem, stream>>>(tmA, tmB, args);
            }
        } else {
            auto k = gemm_tn_2sm_kernel<GradEpi>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k<<<grid, kThreadsPair, smem, stream>>>(tmA, tmB, args);
        }
        return cudaGetLastError();
    }
    const int tiles = ((args.M + BM - 1) / BM) * ((args.N + BN - 1) / BN);
    if (tiles == 0) return cudaSuccess;
    const int grid = tiles < num_sms ? tiles : num_sms;
    if (kind == GemmKind::Logits) {
        auto k = gemm_tn_kernel<LogitsEpi>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k<<<grid, kThreads, smem, stream>>>(tmA, tmB, args);
    } else {
        auto k = gemm_tn_kernel<GradEpi>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k<<<grid, kThreads, smem, stream>>>(tmA, tmB, args);
    }
    return cudaGetLastError();
}

}  // namespace fm

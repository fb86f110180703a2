// k_gemm_tc.cu — the weight-gradient product on tcgen05 (SURVEY.md §8a rows
// a7 / a10):
//
//   K-GEMM2  dW[v][f] (+)= sum_k A'[k][v] * B'[k][f]      (policy.hpp:83-90,
//            training.hpp:394-395, 444-446)
//
// over "segments": column tile nb (256 features) sums only the K rows of its
// segment [kseg_off[nb], kseg_off[nb] + 64 * kseg_iters[nb]) — the context
// positions whose feature lies in that block.  A' rows are the positions'
// per-position gradient rows H (k_band.cu), B' the one-hot of each position's
// feature inside the block, so the MMA scatters-and-sums the H rows into dW's
// columns while the tile's accumulator stays in TMEM.  Both operands are
// MN-major in HBM (row-major [K'][V] / [K'][256]).  Epilogue: read-modify-
// write of the fp32 gradient accumulator, sum(acc^2) of this micro-batch
// (training.hpp:417), and in a DP gang's last micro-batch the reduce-scatter
// over NVLink peer memory.
//
// Persistent CTA-pair kernel (cta_group::2, M256 N256 K16 per MMA): each CTA
// TMA-loads its 128 rows of A and its 128-column half of B per 64-deep K slice
// into a 6-stage ring (SWIZZLE_128B), the leader's single thread issues the
// MMAs and commits (multicast) to both CTAs' barriers, the TMEM accumulator
// is double-buffered (2 x 256 fp32 columns) so each CTA's four epilogue warps
// drain tile i while tile i+1's MMAs run.
//
// Warp roles (192 threads per CTA): w0 TMA producer, w1 MMA issuer (+TMEM
// owner), w2..w5 epilogue (w%4 selects the TMEM lane quadrant it may access).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "fm_gemm.h"
#include "fm_ptx.cuh"

namespace fm {

namespace {
constexpr int BN = kGemmBN, BK = kGemmBK;
constexpr uint32_t kTmemCols = 2 * BN;  // two accumulator buffers

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

// ---- epilogue ---------------------------------------------------------------

struct GradEpi {
    float sumsq;  // this tile's sum of squares (fp32 per tile, fp64 across tiles)
    float* xbuf = nullptr;  // per-warp 32 x 36 fp32 smem staging (exchange mode)
    uint8_t* stage = nullptr;  // per-warp 2 x 4 KB SWIZZLE_128B staging of the TMA epilogue
    const CUtensorMap* tmc = nullptr;
    int nstaged = 0;
    int accumulate = 0;  // this unit adds into dW (else stores)

    // Local rows: the warp's 32 rows x 32 columns go through shared memory (SWIZZLE_128B,
    // the TMA map's layout) and one TMA op adds them into dW in L2 (store for the
    // step's first micro-batch) — no SM round trip for the read-modify-write; two
    // staging buffers, so a chunk's staging overlaps the previous chunk's TMA.
    __device__ __forceinline__ void tma_chunk(const GemmArgs& a, int row, int col0, uint32_t (&r)[32]) {
        const uint32_t lane = threadIdx.x & 31;
        uint8_t* buf = stage + (nstaged & 1) * 4096;
        if (lane == 0) tma_store_wait_read<1>();  // the op that used this buffer has read it
        __syncwarp();
        float part = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float4 acc = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                                           __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
            part += acc.x * acc.x + acc.y * acc.y + acc.z * acc.z + acc.w * acc.w;
            *reinterpret_cast<float4*>(buf + lane * 128 + ((k ^ (lane & 7)) << 4)) = acc;
        }
        sumsq += part;  // rows / columns past the matrix hold exact zeros
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            const int row0 = row - static_cast<int>(lane);
            if (accumulate) tma_reduce_add_2d(tmc, buf, col0, row0);
            else tma_store_2d(tmc, buf, col0, row0);
            tma_store_commit();
        }
        ++nstaged;
    }

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
                if (accumulate) {
                    const float4 o4 = *reinterpret_cast<const float4*>(src + j);
                    acc.x += o4.x;
                    acc.y += o4.y;
                    acc.z += o4.z;
                    acc.w += o4.w;
                }
            }
            *reinterpret_cast<float4*>(xbuf + lane * 36 + j) = acc;
        }
        sumsq += part;
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
        if (tmc) {
            tma_chunk(a, row, col0, r);
            return;
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
            sumsq += part;
            __syncwarp();
            const int row0 = row - static_cast<int>(lane);
            const int seg = static_cast<int>(lane & 7);
            float4 o[8];
            if (accumulate) {  // all eight loads in flight before any store
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
                if (accumulate) {
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
                if (accumulate) {
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
                    dst[j] = accumulate ? src[j] + acc : acc;
                }
            }
        }
        sumsq += part;
    }
};

#ifndef FM_G2_STAGES
#define FM_G2_STAGES 5
#endif
constexpr int P_STAGES = FM_G2_STAGES;
constexpr uint32_t P_A_STAGE = 128 * BK * 2;    // 16 KB: this CTA's 128 rows of A
constexpr uint32_t P_B_STAGE = 128 * BK * 2;    // 16 KB: this CTA's half of B's 256 rows
constexpr uint32_t P_STAGE_BYTES = P_A_STAGE + P_B_STAGE;

constexpr int kThreadsPair = 192;  // w0 TMA, w1 MMA, w2-5 epilogue

// kAmn / kBmn: operand stored MN-major in HBM ([K][M] / [K][N], MN contiguous);
// each CTA's 128 MN x 64 K stage slice is then two TMA boxes {64 MN, 64 K}
// (8 KB each, the second at +8 KB = the descriptor's LBO).
// kSeg: both operands MN-major; column tile nb runs the K rows of its segment
// (args.kseg_off / kseg_iters); B' holds only 256 columns.
// kSnap (batched micro-batches): ONE accumulator per tile (TMEM columns 0-255)
// collects all of the tile's units; after each unit the epilogue reads it and a
// snapshot of the previous unit's total (columns 256-511), adds the squared
// difference — exactly that unit's contribution — to the unit's sum of squares
// and stores the new snapshot; only the last unit drains the tile into dW.  One
// drain per tile instead of one per unit (the drain's smem staging bounded the
// K-GEMM2 of short-K shapes: L1 / shared 86% busy at C3).
template <bool kAmn, bool kBmn, bool kSeg, bool kSnap = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsPair, 1)
    gemm_grad_kernel(const __grid_constant__ GemmMaps maps, GemmArgs args) {
    static_assert(!kSeg || (kAmn && kBmn), "segment operands are MN-major");
    static_assert(!kSnap || kSeg, "snapshots batch segmented units");
    constexpr uint32_t kId = idesc_bf16_f32<256, BN, kAmn, kBmn>();
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
    // TMA epilogue staging: 4 warps x 2 x 4 KB, 1024-B aligned (SWIZZLE_128B atoms)
    uint8_t* tstage = smem + ((P_STAGES * P_STAGE_BYTES + 512 + 4 * 32 * 36 * 4 + 1023) & ~1023u);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    // units per output tile: the batched micro-batches (segmented path) or 1
    const int nmb = kSeg ? args.nmb : 1;

    if (warp == 0 && lane == 0) {
        for (int u = 0; u < nmb; ++u) {
            tma_prefetch(&maps.a[u]);
            tma_prefetch(&maps.b[u]);
        }
        tma_prefetch(&maps.c);
        for (int s = 0; s < P_STAGES; ++s) {
            mbar_init(&full[s], 1);   // the leader's producer arrives with both CTAs' tx bytes
            mbar_init(&empty[s], 1);  // one multicast commit per consumed stage
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);  // 4 epilogue warps x 2 CTAs (the leader's copy is the one used)
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
    // K iterations of unit u of column tile nb
    auto unit_iters = [&](int u, int nb) -> int {
        if constexpr (kSeg) return __ldg(args.kseg_iters_b[u] + nb);
        else return k_iters;
    };

    if (warp == 0) {
        // ===== TMA producer (both CTAs) =====
        if (elect_one()) {
            const uint64_t pol = policy_evict_last();
            // segments: each A' segment block is read by exactly one tile
            const uint64_t pol_a = kSeg ? policy_evict_first() : pol;
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < num_tiles; t += nclusters) {
                const TileCoord tc = tile_coord(t, tiles_m, tiles_n, args.group_m);
                const int arow = tc.mb * 256 + static_cast<int>(rank) * 128;
                const int brow = (kSeg ? 0 : tc.nb * BN) + static_cast<int>(rank) * 128;
                for (int u = 0; u < nmb; ++u) {
                    const CUtensorMap* tmA = &maps.a[u];
                    const CUtensorMap* tmB = &maps.b[u];
                    int kbase = 0;
                    const int ke = unit_iters(u, tc.nb);
                    if constexpr (kSeg) {
                        kbase = __ldg(args.kseg_off_b[u] + tc.nb);
                        FM_DCHECK(args.dbg_krows == 0 || kbase + static_cast<long long>(ke) * BK <= args.dbg_krows);
                    }
                    for (int k = 0; k < ke; ++k) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        const uint32_t fb = mapa_shared(&full[stage], 0);
                        if (leader) mbar_arrive_expect_tx(&full[stage], 2 * P_STAGE_BYTES);
                        const int kc = kbase + k * BK;
                        if constexpr (kAmn) {
                            tma_load_2d_2sm(sA + stage * P_A_STAGE, tmA, fb, arow, kc, pol_a);
                            tma_load_2d_2sm(sA + stage * P_A_STAGE + 8192, tmA, fb, arow + 64, kc, pol_a);
                        } else {
                            tma_load_2d_2sm(sA + stage * P_A_STAGE, tmA, fb, kc, arow, pol);
                        }
                        if constexpr (kBmn) {
                            tma_load_2d_2sm(sB + stage * P_B_STAGE, tmB, fb, brow, kc, pol);
                            tma_load_2d_2sm(sB + stage * P_B_STAGE + 8192, tmB, fb, brow + 64, kc, pol);
                        } else {
                            tma_load_2d_2sm(sB + stage * P_B_STAGE, tmB, fb, kc, brow, pol);
                        }
                        if (++stage == P_STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
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
            for (int t = cid; t < num_tiles; t += nclusters) {
                const int nb = tile_coord(t, tiles_m, tiles_n, args.group_m).nb;
                for (int u = 0; u < nmb; ++u) {
                    const int ke = unit_iters(u, nb);
                    if constexpr (kSnap) acc = 0;  // the one accumulator
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                    for (int k = 0; k < ke; ++k) {
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
                                          (k != 0 || kk != 0 || (kSnap && u != 0)));
                        umma_commit_2sm(&empty[stage], 0x3);
                        if (++stage == P_STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    umma_commit_2sm(&tfull[acc], 0x3);
                    if constexpr (kSnap) {
                        acc_phase ^= 1;
                    } else {
                        acc ^= 1;
                        if (acc == 0) acc_phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ===== epilogue warps 2..5 (both CTAs; each CTA drains its own 128 rows) =====
        const uint32_t quad = warp & 3;  // TMEM lane quadrant this warp may access
        const int row_in_tile = static_cast<int>(rank * 128 + quad * 32 + lane);
        const uint32_t tempty_leader[2] = {mapa_shared(&tempty[0], 0), mapa_shared(&tempty[1], 0)};
        GradEpi epi;
        epi.xbuf = xscratch + quad * 32 * 36;
        epi.stage = tstage + quad * 8192;
        epi.tmc = &maps.c;
        int acc = 0;
        uint32_t acc_phase = 0;
        double sq[kGemmMaxBatch] = {};  // per unit (micro-batch), fp64 across tiles
        for (int t = cid; t < num_tiles; t += nclusters) {
            const TileCoord tc = tile_coord(t, tiles_m, tiles_n, args.group_m);
            const int row = tc.mb * 256 + row_in_tile;
            for (int u = 0; u < nmb; ++u) {
                if constexpr (kSnap) {
                    const bool last = u + 1 == nmb;
                    mbar_wait(&tfull[0], acc_phase);
                    tc_fence_after();
                    if (u > 0) tmem_st_wait();  // the previous unit's snapshot has landed
                    epi.accumulate = args.accumulate;
                    const uint32_t lane_base = tmem_base + ((quad * 32u) << 16);
                    float part = 0.f;
#pragma unroll 1
                    for (int c = 0; c < BN / 32; ++c) {
                        uint32_t r[32], q[32];
                        tmem_ld_32x32b_x32(lane_base + static_cast<uint32_t>(c * 32), r);
                        if (u > 0) tmem_ld_32x32b_x32(lane_base + static_cast<uint32_t>(BN + c * 32), q);
                        tmem_ld_wait();
                        if (c == BN / 32 - 1) {
                            // every accumulator column is read: the MMA may add the next unit
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader[0]);
                        }
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float d = __uint_as_float(r[j]) - (u > 0 ? __uint_as_float(q[j]) : 0.f);
                            part = fmaf(d, d, part);
                        }
                        if (!last) tmem_st_32x32b_x32(lane_base + static_cast<uint32_t>(BN + c * 32), r);
                        else epi.chunk(args, row, tc.nb * BN + c * 32, r);
                    }
#pragma unroll
                    for (int j = 0; j < kGemmMaxBatch; ++j)
                        if (j == u) sq[j] += static_cast<double>(part);
                    acc_phase ^= 1;
                    continue;
                }
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                epi.sumsq = 0.f;
                epi.accumulate = (u > 0 || args.accumulate) ? 1 : 0;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + static_cast<uint32_t>(acc * BN + c * 32), r);
                    tmem_ld_wait();
                    if (c == BN / 32 - 1) {
                        // the accumulator is fully in registers: hand TMEM back to the MMA
                        // warp before the last chunk's stores (relaxed: no wait for this
                        // warp's outstanding global stores)
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader[acc]);
                    }
                    epi.chunk(args, row, tc.nb * BN + c * 32, r);
                }
#pragma unroll
                for (int j = 0; j < kGemmMaxBatch; ++j)
                    if (j == u) sq[j] += static_cast<double>(epi.sumsq);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
#pragma unroll
        for (int j = 0; j < kGemmMaxBatch; ++j) {
            double v = sq[j];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            double* dst = kSeg ? args.sumsq_b[j] : (j == 0 ? args.sumsq : nullptr);
            if (lane == 0 && j < nmb && dst) atomicAdd(dst, v);
        }
        if (lane == 0) tma_store_wait<0>();  // every reduce / store of this warp has completed
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm<kTmemCols>(tmem_base);
    }
}

template <bool kAmn, bool kBmn, bool kSeg, bool kSnap = false>
cudaError_t launch_grad(const GemmMaps& maps, const GemmArgs& args, int num_sms, cudaStream_t stream) {
    const size_t smem = gemm_smem_bytes();
    const int tiles = ((args.M + 255) / 256) * ((args.N + BN - 1) / BN);
    if (tiles == 0) return cudaSuccess;
    const int pairs = num_sms / 2;
    const int grid = 2 * (tiles < pairs ? tiles : pairs);
    auto k = gemm_grad_kernel<kAmn, kBmn, kSeg, kSnap>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k<<<grid, kThreadsPair, smem, stream>>>(maps, args);
    return cudaGetLastError();
}

}  // namespace

// Test hook: C[M][N] (fp32, ld N) = sum_k A(m,k) B(n,k) with A / B either K-major
// ([M][K] / [N][K]) or MN-major ([K][M] / [K][N]) — validates the MN-major UMMA
// operand path against a plain reference (tests/test_gpu_path.py).
cudaError_t gemm_debug_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC, int a_mn,
                              int b_mn, int M, int N, int K, float* C, int num_sms, cudaStream_t stream) {
    GemmArgs args{};
    args.M = M;
    args.N = N;
    args.K = K;
    args.group_m = 8;
    args.out = C;
    args.ld_out = N;
    GemmMaps maps{};
    maps.a[0] = tmA;
    maps.b[0] = tmB;
    maps.c = tmC;
    if (a_mn && b_mn) return launch_grad<true, true, false>(maps, args, num_sms, stream);
    if (a_mn) return launch_grad<true, false, false>(maps, args, num_sms, stream);
    if (b_mn) return launch_grad<false, true, false>(maps, args, num_sms, stream);
    return launch_grad<false, false, false>(maps, args, num_sms, stream);
}

cudaError_t gemm_kseg_launch(const GemmMaps& maps, const GemmArgs& args_in, int num_sms, cudaStream_t stream) {
    GemmArgs args = args_in;
    if (args.nmb < 1 || args.nmb > kGemmMaxBatch) return cudaErrorInvalidValue;
    if (args.nmb > 1 && args.xg > 1) return cudaErrorInvalidValue;  // the exchange is per micro-batch
    if (args.nmb == 1) {  // the single-micro-batch fields
        args.kseg_off_b[0] = args.kseg_off;
        args.kseg_iters_b[0] = args.kseg_iters;
        args.sumsq_b[0] = args.sumsq;
    }
    if (args.nmb > 1 && args.snap) return launch_grad<true, true, true, true>(maps, args, num_sms, stream);
    return launch_grad<true, true, true>(maps, args, num_sms, stream);
}

size_t gemm_smem_bytes() {
    return 1024 + ((P_STAGES * P_STAGE_BYTES + 512 + 4 * 32 * 36 * 4 + 1023) & ~static_cast<size_t>(1023)) + 4 * 8192;
}

}  // namespace fm

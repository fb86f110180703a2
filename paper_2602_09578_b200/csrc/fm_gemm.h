// fm_gemm.h — host-visible interface of the tcgen05 weight-gradient GEMM (k_gemm_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "fm_kernels.h"

namespace fm {

constexpr int kGemmBN = 256;
constexpr int kGemmBK = 64;
constexpr int kGemmMaxBatch = 4;  // micro-batches one K-GEMM2 launch can reduce

// C[M][N] (+)= sum_k A(m, k) * B(n, k) on the CTA-pair tcgen05 kernel; A / B
// bf16, K-major ([M][K] / [N][K], TMA boxes {64, 128}) or MN-major ([K][M] /
// [K][N], boxes {64, 64}), SWIZZLE_128B.
struct GemmArgs {
    int M, N, K;
    int group_m;          // L2 raster: tiles visited in column-major groups of group_m row-tiles
    float* out;           // dW [M][ld_out]
    long long ld_out;
    int accumulate;       // 1 = dW += acc, 0 = dW = acc
    double* sumsq;        // += sum(acc^2) (micro-batch grad norm^2)
    // DP-gang exchange (xg > 1): rows [xlo[o], xlo[o+1]) are owned by gang rank o;
    // rows owned by another rank are written (whole partial) into xpeer[o] =
    // this rank's receive slot in rank o's buffer (NVLink P2P).
    int xg = 0;
    int xrank = 0;
    int xlo[9] = {};
    float* xpeer[8] = {};
    // Segmented K: column tile nb sums K rows [kseg_off[nb], +64*kseg_iters[nb]) of
    // A' [K'][M] and B' [K'][256] (tile loads, MN-major).
    const int32_t* kseg_off = nullptr;
    const int32_t* kseg_iters = nullptr;
    long long dbg_krows = 0;  // rows of A' / B' (debug-build bounds checks; 0 = unchecked)
    // Batched micro-batches (segmented path, no exchange): every output tile runs nmb
    // units back to back, unit u over micro-batch u's segments (maps.a[u] / maps.b[u],
    // kseg_off_b[u] / kseg_iters_b[u]) into the other TMEM buffer, and its epilogue adds
    // sum(acc^2) into sumsq_b[u] and the tile into dW (store for u = 0 without
    // accumulate) — the tile's dW stays in L2 between its units.  nmb = 1: the fields
    // above.
    int nmb = 1;
    int snap = 0;  // batched units share one accumulator (short segments; see gemm_grad_kernel's kSnap)
    const int32_t* kseg_off_b[kGemmMaxBatch] = {};
    const int32_t* kseg_iters_b[kGemmMaxBatch] = {};
    double* sumsq_b[kGemmMaxBatch] = {};
};

// The kernel's tensor maps (a __grid_constant__ parameter): A / B of every batched
// unit and the fp32 output map.
struct GemmMaps {
    CUtensorMap a[kGemmMaxBatch];
    CUtensorMap b[kGemmMaxBatch];
    CUtensorMap c;
};

size_t gemm_smem_bytes();
// Test hook: fp32 C = A * B^T with either operand K- or MN-major.
// tmC: the output's fp32 map (make_tmap_f32_out) for the TMA reduce-add / store epilogue.
cudaError_t gemm_debug_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC, int a_mn,
                              int b_mn, int M, int N, int K, float* C, int num_sms, cudaStream_t stream);
// K-GEMM2 over segments, MN-major tile maps: nmb = 1 (args.kseg_off / kseg_iters /
// sumsq, maps.a[0] / b[0]) or a batch of micro-batches (the _b arrays).
cudaError_t gemm_kseg_launch(const GemmMaps& maps, const GemmArgs& args, int num_sms, cudaStream_t stream);
// fp32 [rows][cols] (row pitch `pitch` elements, a multiple of 4) with box {32, 32},
// SWIZZLE_128B: the GEMM epilogue's per-warp output tile.
bool make_tmap_f32_out(CUtensorMap* map, const float* base, uint64_t rows, uint64_t cols, uint64_t pitch);

// Builds a 2-D bf16 tensor map over a row-major [rows][cols] matrix (cols
// contiguous, row pitch `pitch` elements), box {64, box_rows}, SWIZZLE_128B.
bool make_tmap_bf16_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                           uint32_t box_rows, uint64_t pitch = 0);

}  // namespace fm

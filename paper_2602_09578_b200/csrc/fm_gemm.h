// fm_gemm.h — host-visible interface of the tcgen05 TN GEMM (k_gemm_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "fm_kernels.h"

namespace fm {

constexpr int kGemmBM = 128;
constexpr int kGemmBN = 256;
constexpr int kGemmBK = 64;
constexpr int kGemmStages = 4;

enum class GemmKind { Logits, Grad };

// C[M][N] = sum_k A[M][K] * B[N][K]; A/B bf16 K-major, described by TMA maps
// with boxes {64, 128} (A) and {64, 256} (B), SWIZZLE_128B.
struct GemmArgs {
    int M, N, K;
    int k0 = 0;           // first K index (a K-chunk of a longer product; multiple of 64)
    int group_m;          // L2 raster: tiles visited in column-major groups of group_m row-tiles
    float* out;           // Grad: dW [M][ld_out]
    __nv_bfloat16* pexp;  // Logits: p~ = exp(z - m_tile) [M][ld_out] bf16
    float* zact;          // Logits: fp32 logit of each row's taken token
    const int32_t* action;   // Logits: taken token per row
    long long ld_out;
    const float* row_scale;  // Logits: per-row 1/n_ctx
    float2* stats;           // Logits: [M][stats_ld] (max, sum exp) per 256-col tile
    int stats_ld;
    int accumulate;          // Grad: 1 = dW += acc, 0 = dW = acc
    double* sumsq;           // Grad: += sum(acc^2) (micro-batch grad norm^2)
    // Loss-fold path: Logits uses the per-row offset bound mrow[row] for every tile
    // (one TMEM pass) and stores p~ TRANSPOSED into pexp_t [N][ldt] (rows <
    // store_rows; zeros for M <= row) — GEMM2's K-major A operand.
    const float* mrow;
    __nv_bfloat16* pexp_t;
    long long ldt;
    int store_rows;
    // Grad, DP-gang exchange (xg > 1): rows [xlo[o], xlo[o+1]) are owned by gang
    // rank o; rows owned by another rank are written (whole partial) into
    // xpeer[o] = this rank's receive slot in rank o's buffer (NVLink P2P).
    int xg = 0;
    int xrank = 0;
    int xlo[9] = {};
    float* xpeer[8] = {};
    // Logits, fused K-lse (lse_sync != nullptr): lse_sync[0] counts the CTAs whose
    // tiles are stored, lse_sync[1] is the epoch the last one publishes; then the
    // whole grid runs the row normaliser (fm_lse.cuh) over lse's rows.
    unsigned* lse_sync = nullptr;
    unsigned lse_epoch = 0;
    LseArgs lse{};
    // Grad, stream-K tail (sk_ws != nullptr; CTA-pair kernel): when the tiles do not
    // fill the last wave, the last (waves-1)*pairs tiles' worth plus the remainder are
    // split into equal K ranges per pair; partial accumulators meet in sk_ws
    // ([tile][256][256] fp32, zero between launches) and the last arriving CTA of
    // each tile half runs the epilogue from it (sk_cnt[tile*2 + rank], self-resetting).
    float* sk_ws = nullptr;
    int* sk_cnt = nullptr;
    // Grad, K-list (token-list) mode: output column tile nb sums only over the K rows
    // klist[nb * klist_ld + 0 .. 64 * klist_iters[nb]) (row indices, padded with a
    // zero row); both operands row-major [rows][M] / [rows][N] (MN-major),
    // gathered four rows per TMA gather4.
    const int32_t* klist = nullptr;
    long long klist_ld = 0;
    const int32_t* klist_iters = nullptr;
    // Segmented K (token slots): column tile nb sums K rows [kseg_off[nb], +64*klist_iters[nb])
    // of A' [K'][M] and B' [K'][256] (tile loads, MN-major).  Logits: aseg != nullptr
    // stores each row's p~ into the A' rows slot4[row] (row-major, pitch ld_out).
    const int32_t* kseg_off = nullptr;
    __nv_bfloat16* aseg = nullptr;
    const int4* slot4 = nullptr;
    // Grad, segments with a software-gathered A (FM_G2_KLIST=3): A rows = p~ rows
    // pexp[seg_tok[k]] (row-major, pitch ld_pexp) copied by four producer warps per
    // CTA into the swizzled MN-major stage; B' tile-loaded as in kSeg.
    const int32_t* seg_tok = nullptr;
    long long ld_pexp = 0;
    int dbg_nostore = 0;  // timing diagnostics only: skip the token-slot global stores
    // Logits (CTA pair): drain each accumulator with 8 epilogue warps (softmax partials
    // per column half: stats_ld = 2 x tiles) instead of 4
    int epi_wide = 0;
};

// Stream-K workspace capacity: at most 2*pairs-1 split tiles (148 SMs -> 74 pairs).
constexpr int kSkMaxTiles = 148;

// 1 when the loss-fold path (no separate K-loss kernel) is active (FM_LOSS_FOLD != 0).
bool loss_fold_enabled();
// 1 when the CTA-pair (cta_group::2) kernels are in use (required by the DP gang exchange).
bool gemm_pair_mode();

size_t gemm_smem_bytes();
// Rows of B per TMA box: 256 (single-CTA tiles) or 128 (CTA-pair tiles, FM_GEMM_2SM != 0).
uint32_t gemm_b_box_rows();
cudaError_t gemm_debug_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, int a_mn, int b_mn, int M, int N,
                              int K, float* C, int num_sms, cudaStream_t stream);
// Grad GEMM over token-slot segments (args.kseg_off / klist_iters), MN-major tile maps.
cudaError_t gemm_kseg_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& args, int num_sms,
                             cudaStream_t stream);
// Same, A rows gathered by producer warps from args.pexp via args.seg_tok (tmA unused).
cudaError_t gemm_kseg_swa_launch(const CUtensorMap& tmB, const GemmArgs& args, int num_sms, cudaStream_t stream);
// Grad GEMM over per-column-tile K lists (args.klist*), gather4 maps for A and B.
cudaError_t gemm_klist_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& args, int num_sms,
                              cudaStream_t stream);
// 2-D bf16 map over [rows][cols] with box {64, 1}, SWIZZLE_128B (TMA gather4).
bool make_tmap_gather4(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch);
cudaError_t gemm_tn_launch(GemmKind kind, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const GemmArgs& args, int num_sms, cudaStream_t stream);

// Builds a 2-D bf16 K-major tensor map over a row-major [rows][cols] matrix
// (cols contiguous), box {64, box_rows}, SWIZZLE_128B.
bool make_tmap_bf16_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                           uint32_t box_rows, uint64_t pitch = 0);
// Plain (no swizzle) 2-D map, any 4/2-byte dtype, box {box_cols, box_rows}.
bool make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, uint32_t elem_bytes,
                  uint64_t rows, uint64_t cols, uint32_t box_rows, uint32_t box_cols);

}  // namespace fm

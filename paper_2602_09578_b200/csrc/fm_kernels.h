// fm_kernels.h — launch wrappers for the HBM-bound hot-path kernels
// (k_path.cu).  All take an explicit stream; none synchronise.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace fm {

// One sample of a micro-batch as the device sees it: byte offsets of the
// encoded prompt / response token lists in the token arena (codec.hpp:15-22
// format), their token counts, the first packed row of the sample and its
// advantage (training.hpp:371, 386).
struct SampleDesc {
    int64_t prompt_off;
    int64_t resp_off;
    int32_t prompt_n;
    int32_t resp_n;
    int64_t row_start;
    double adv;
};

struct RowBuffers {
    int32_t* action;   // [Mpad]
    int4* ctx4;        // [Mpad] last <=4 context tokens, -1 padded
    int32_t* n_ctx;    // [Mpad]
    int32_t* sample;   // [Mpad]
    float* coef;       // [Mpad] -A/(G*n)   (0 for padding rows)
    float* rscale;     // [Mpad] 1/n        (0 for n == 0)
    float* lse;        // [Mpad]
    float* logp;       // [Mpad]
    float* coef_eff;   // [Mpad] coef * surrogate factor
    int32_t* q0;       // [Mpad] first context position of the row (band formulation; nullable)
    float* mrow;       // [Mpad] softmax bound (1/n) sum_k fmax[f_k] >= max_v z (with fmax)
    const float* fmax; // [D] per-feature maximum of the bf16 shadow (nullable: no bounds)
    // with w16t (tensor-core path): the taken token's fp32 logit
    // rs * ((X[f0] + X[f1]) + (X[f2] + X[f3])) at its W16^T column — K-stats' own summation
    // order, so bit-identical to its z; 0 where the action lies outside [col_base,
    // col_base + ncols) (a vocabulary-gang rank) — and the row's loss weight -A / G
    float* zact = nullptr;      // [Mpad]
    double* lossw = nullptr;    // [Mpad]
    const __nv_bfloat16* w16t = nullptr;  // W16^T at column col_base
    int64_t ldw = 0, col_base = 0, ncols = 0;
};

// K-lse arguments.
struct LseArgs {
    const float* stats;   // [stats_ld][Mpad] partial sums of exp(z - mrow) (K-stats)
    int stats_ld;
    int64_t M, Mpad, V;
    const SampleDesc* sd;
    int64_t G;
    RowBuffers rows;
    const float* old_logp;  // PPO clip (nullable): old log-prob of shard row r at old_logp[row_lo + r]
    int64_t row_lo;
    float clip_eps;
    double* loss_acc;  // += objective (nullable)
    // vocabulary-parallel gang: partial_out != NULL -> write [row sum, taken logit] as
    // [2][Mpad] and stop (for the all-reduce); sum_in != NULL -> take them from there
    float* partial_out = nullptr;
    const float* sum_in = nullptr;
};

// K-gather: decode the selected records' token payloads straight out of the
// arena into packed rows (action, context window, sample, row coefficient,
// 1/n, and with rows.q0 != NULL the row's first context position).
cudaError_t launch_gather(const uint8_t* arena, const SampleDesc* sd, int n_samples, int64_t row_lo,
                          int64_t M, int64_t Mpad, int64_t global_batch, uint64_t D, RowBuffers rows,
                          cudaStream_t s);

// K-pos: feature (tok mod D) of every context position of the shard's rows
// (every sample overlapping the shard owns its rows + 3 positions: the three
// tokens before its first row's last context token), -1 where the sequence
// has no token (prompt shorter than 4) and past the last position (q < Qcap).
// K-fmax: fmax[f] = max_v W16^T[f][v] (the per-feature bound K-gather sums into
// every row's softmax offset), one CTA per feature row.
cudaError_t launch_fmax(const __nv_bfloat16* w16t, int64_t D, int64_t V, int64_t ldw, float* fmax, cudaStream_t s);

cudaError_t launch_positions(const uint8_t* arena, const SampleDesc* sd, int n_samples, int64_t row_lo, int64_t M,
                             uint64_t D, int32_t* feat, int64_t Qcap, cudaStream_t s);

// K-pslot: every position with a feature gets a row ("slot") of the segment of
// its feature's 256-column block in A' [K'][.] / B' [K'][256]; segment b
// starts at kseg_off[b] and is padded to a multiple of 64 rows (>= 64);
// B' = one-hot of the feature inside the block (zeroed here first).
// Deterministic (position order).  rows_acc (nullable) accumulates the padded
// segment rows (GEMM2's executed K, for the roofline).
cudaError_t launch_pslots(const int32_t* feat, int64_t Q, int nblk, int32_t* kcount, int32_t* kseg_off, int32_t* kiters,
                          int32_t* slot, __nv_bfloat16* bseg, int64_t bseg_rows, unsigned long long* rows_acc,
                          cudaStream_t s);

// K-stats / K-band (k_band.cu).
struct BandArgs {
    const __nv_bfloat16* w16t;  // transposed bf16 shadow W16^T [D][ldw]
    int64_t ldw;
    const __nv_bfloat16* zero_row;  // >= 2,048 zero bf16 (positions before a sequence start)
    int64_t V;
    const int32_t* pos_feat;    // [Q]
    const int32_t* q0;          // [M]
    const int32_t* action;      // [M]
    const float* rscale;        // [M]
    const float* mrow;          // [M] softmax bound of the row
    int64_t M;
    int64_t ld_stats;           // row pitch of stats (Mpad)
    // pass A (K-stats)
    float* stats;   // [stats_ld][ld_stats] partial sums of exp(z - mrow)
    int stats_ld;
    // pass B (K-band)
    const float* lse;       // [M]
    const float* coef_eff;  // [M]
    const int32_t* pos_slot;  // [Q]
    __nv_bfloat16* aseg;      // A' [K'][ld_a]
    int64_t ld_a;
    int64_t dbg_kp = 0, dbg_D = 0;  // A' rows and features (debug-build bounds checks)
    // vocabulary-parallel gang: w16t and aseg point at this rank's first column, V is its
    // range's width and actions are taken relative to col_base
    int64_t col_base = 0;
    int rows_per_item = 0;  // (set by launch_band: 128, or 64 when that balances persistent CTAs better)
};
cudaError_t launch_band(const BandArgs& A, bool grad, cudaStream_t s);
// K-stats partials per row (one per consumer warp of every vocabulary slice).
int band_stats_ld(int64_t V);

// K-lse: lse = mrow + log(sum of K-stats' partial sums), the taken-token
// log-prob (K-gather's fp32 logit) and the effective row coefficient (PPO-clip
// surrogate optional).
cudaError_t launch_lse(const LseArgs& L, cudaStream_t s);

// Parity tooling: out[v][j] = dW[v][cols[j]] (f32 or f64 accumulator).
cudaError_t launch_gather_cols(const void* dW, bool f64, uint64_t V, uint64_t D, const int64_t* cols,
                               int64_t n_cols, void* out, cudaStream_t s);

// K-adam (training.hpp:37-51): fp64 master weights, fp32 moments, gradient of
// type G (float for the tensor-core path, double for parity mode) over rows
// [r0, r1) of the [V][D] state, in 32 x 64 tiles.  Optionally: the gradient is
// the local partial plus nslots receive slots ([nslots][r1-r0][D], a DP
// gang's reduce-scatter); the transposed bf16 shadow W16^T [D][ldw] is
// written (locally and into the peers' replicas over NVLink: the all-gather
// fused into the optimizer) through a shared-memory transpose; the new w / m
// / v go to dst instead of in place (the swap-out fused into the optimizer);
// the gradient is zeroed (parity mode).  Accumulates sum(g^2) into *gsq.
struct AdamDst {
    double* w;
    float* m;
    float* v;
};
// Peer W16^T replicas (NVLink-mapped base pointers) of a DP gang, excluding self.
struct ShardPeers {
    int n;
    __nv_bfloat16* w16t[7];
};
template <typename G>
cudaError_t launch_adam(double* w, float* m, float* v, G* g, uint64_t V, uint64_t D, uint64_t r0, uint64_t r1,
                        const float* recv, int nslots, __nv_bfloat16* w16t, uint64_t ldw, ShardPeers peers,
                        double lr, double b1, double b2, double eps, double bc1, double bc2, int zero_grad,
                        double* gsq, int num_sms, cudaStream_t s, const AdamDst* dst = nullptr);

// W16^T [D][ldw] = bf16(W) for W [V][D] f64 (shadow refresh: set_weights, host-tier swap-in).
cudaError_t launch_w16t(const double* w, uint64_t V, uint64_t D, __nv_bfloat16* w16t, uint64_t ldw, int num_sms,
                        cudaStream_t s);
// out [V][D] = W16^T transposed back (the bf16 weight publish).
cudaError_t launch_w16t_untranspose(const __nv_bfloat16* w16t, uint64_t V, uint64_t D, uint64_t ldw,
                                    __nv_bfloat16* out, cudaStream_t s);

// dst = (accumulate ? dst : 0) + src, n floats.
cudaError_t launch_axpy_init(float* dst, const float* src, uint64_t n, int accumulate, int num_sms, cudaStream_t s);
// *out += sum(x^2) over n floats (fp64 accumulation).
cudaError_t launch_sumsq(const float* x, uint64_t n, double* out, int num_sms, cudaStream_t s);

cudaError_t launch_to_bf16(const double* w, __nv_bfloat16* w16, uint64_t n, int num_sms,
                           cudaStream_t s);

// K-adv (training.hpp:54-67): one warp per reward group, fp64 shuffle reductions.
cudaError_t launch_group_advantages(const double* rewards, const int32_t* seg_off, int nseg,
                                    double eps, double* out, cudaStream_t s);

// Parity mode (exact featurizer, fp64 SIMT): per row logits/softmax/grad into dWmb.
cudaError_t launch_parity_rows(const double* W, uint64_t V, uint64_t D, int64_t M,
                               RowBuffers rows, const SampleDesc* sd, int64_t global_batch,
                               double* zscratch, double* dWmb, double* logp64, double* loss_acc,
                               cudaStream_t s);
// Rollout-side generation (policy.hpp:119-130), one CTA per request (k_rollout.cu).
// W is [V][D] (transposed = false) or the rollout layout [D][V].
cudaError_t launch_generate(const double* W, bool transposed, uint64_t V, uint64_t D, const int32_t* prompts,
                            const int32_t* prompt_off, int n_req, int max_tokens, const uint64_t* seeds,
                            double* zbuf, int32_t* out_tok, double* out_logp, int32_t* out_len,
                            cudaStream_t s);

// sumsq += |dWmb|^2; dW += dWmb; dWmb = 0
cudaError_t launch_parity_fold(double* dW, double* dWmb, uint64_t n, double* sumsq, int num_sms,
                               cudaStream_t s);

}  // namespace fm

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
    int4* feat4;       // [Mpad] unique features of the row (-1 padded)   (tensor-core path)
    uint32_t* cnt4;    // [Mpad] their multiplicities, 8 bits each
    float* mrow;       // [Mpad] softmax offset bound (1/n) sum_j colmax[f_j]   (loss-fold path)
};

// K-lse arguments (fm_lse.cuh: the per-row routine shared by the standalone
// kernel and GEMM1's fused last-tile epilogue).
struct LseArgs {
    const float* zact;    // [Mpad] fp32 logit of the taken token
    const float2* stats;  // [Mpad][stats_ld] (max, sum exp) per 256-column tile
    int stats_ld;
    int64_t M, Mpad, V;
    const SampleDesc* sd;
    int64_t G;
    RowBuffers rows;
    const float* old_logp;  // PPO clip (nullable)
    float clip_eps;
    double* loss_acc;  // += objective (nullable)
    int fold;
    __nv_bfloat16* pexp_t;  // fold: p~^T [V][ldt]  (rowmajor: p~ [Mpad][ldt])
    __nv_bfloat16* phict;   // fold: Phic^T [D][ldt] (rowmajor: Phic [Mpad][ld_phi])
    int64_t ldt;
    int rowmajor = 0;  // K-list GEMM2: 1 = row-major p~ / Phic, 2 = token-slot segments
    int64_t ld_phi = 0;
    const int4* slot4 = nullptr;   // rowmajor 2: A' row of each feature's block per token
    __nv_bfloat16* bseg = nullptr; // rowmajor 2: B' [K'][256]
};

// K-gather: decode the selected records' token payloads straight out of the
// arena into packed rows; optionally scatter integer-count features into the
// dense bf16 operands Phic [Mpad][D] and Phic^T [D][Mpad] (pre-zeroed, or
// holding the previous micro-batch's pattern for the same Mpad/D when
// clear_old != 0, in which case each row first erases its old entries).
cudaError_t launch_gather(const uint8_t* arena, const SampleDesc* sd, int n_samples, int64_t row_lo,
                          int64_t M, int64_t Mpad, int64_t global_batch, uint64_t D, RowBuffers rows,
                          __nv_bfloat16* phic, __nv_bfloat16* phict, int clear_old, const int* colmax,
                          cudaStream_t s);

// K-colmax: keys[d] = key(max_v W16[v][d]) (order-preserving int encoding), the
// per-feature bound K-gather turns into each row's softmax offset (loss-fold path).
cudaError_t launch_colmax(const __nv_bfloat16* w16, int64_t V, int64_t D, int* keys, int num_sms,
                          cudaStream_t s);

// K-lse: combine GEMM1's per-tile softmax partials into lse, the taken-token
// log-prob (from the fp32 logit GEMM1 captured) and the effective row
// coefficient (PPO-clip surrogate optional).
// Loss-fold path (pexp_t != NULL; GEMM1 used the row bound m_t for every tile):
// folds the taken token's delta into p~^T (pexp_t [V][ldt]) and overwrites the
// row's <= 4 count entries of Phic^T (phict [D][ldt]) with count * (-c_t / s_t),
// so that GEMM2 (A = p~^T, B = Phic^T) yields G^T x Phic without a K-loss pass.
cudaError_t launch_lse(const float* zact, const float2* stats, int stats_ld, int64_t M, int64_t Mpad,
                       int64_t V, const SampleDesc* sd, int64_t global_batch, RowBuffers rows,
                       const float* old_logp, float clip_eps, double* loss_acc, __nv_bfloat16* pexp_t,
                       __nv_bfloat16* phict, int64_t ldt, cudaStream_t s, int rowmajor = 0, int64_t ld_phi = 0);
cudaError_t launch_lse(const LseArgs& L, cudaStream_t s);

// K-loss (fused log-softmax gradient):
//   G^T[v][t] = coef_eff_t * (delta(v, a_t) - p~[t][v] * exp(m_tile(t, v) - lse_t))
// p~ tiles (bf16, from GEMM1) streamed in through TMA, G^T tiles stored through TMA.
cudaError_t launch_softmax_grad(const CUtensorMap& tmP, const CUtensorMap& tmGt, const float2* stats,
                                int stats_ld, int64_t Mpad, int64_t V, RowBuffers rows, cudaStream_t s,
                                int part_cols = 256);

// K-klist: for every 256-feature column block b of GEMM2, the rows (tokens) whose
// context touches block b, ascending, padded with zero_row to a multiple of 64
// (at least 64); iters[b] = padded length / 64.  One block per column block
// (deterministic block-wide scans).
cudaError_t launch_klist(const int4* feat4, int64_t M, int nblk, int32_t* klist, int64_t ld, int32_t* iters,
                         int32_t zero_row, cudaStream_t s);

// K-slot (segmented K-list GEMM2): the tokens touching 256-feature block b get
// consecutive rows ("slots") of a segment of A' [K'][ld_a] / B' [K'][256]; segment
// b starts at kseg_off[b] and is padded to a multiple of 64 rows (>= 64) whose A'
// and B' rows are zeroed.  slot4[t].c_j = the slot of feature j's block (-1 if
// feature j is absent); B'[slot][f mod 256] = count of f.  bseg must be zero on
// entry.  Deterministic (block-wide scans in row order; kcount = per-(block,
// 1024-row chunk) counts).  rows_acc (nullable)
// accumulates the padded segment rows (GEMM2's executed K, for the roofline).
// seg_tok (nullable): the token of every slot (padding slots = zero_row) for the
// software-gathered A; aseg may then be null (no A' rows are written).
cudaError_t launch_kslots(const int4* feat4, const uint32_t* cnt4, int64_t M, int nblk, int32_t* kcount,
                          int32_t* kseg_off, int32_t* kiters, int4* slot4, __nv_bfloat16* aseg, int64_t ld_a,
                          int64_t ncols_a, __nv_bfloat16* bseg, unsigned long long* rows_acc, int32_t* seg_tok,
                          int32_t zero_row, cudaStream_t s);

// Parity tooling: out[v][j] = dW[v][cols[j]] (f32 or f64 accumulator).
cudaError_t launch_gather_cols(const void* dW, bool f64, uint64_t V, uint64_t D, const int64_t* cols,
                               int64_t n_cols, void* out, cudaStream_t s);

// K-adam (training.hpp:37-51): fp64 master weights, fp32 moments, gradient
// of type G (float for the tensor-core path, double for parity mode);
// optionally writes the bf16 shadow and zeroes the gradient.  Accumulates
// sum(g^2) into *gsq for the update grad_norm.  With colmax != NULL (and a
// [V][D] shadow) it also produces K-colmax's keys from the new shadow when the
// grid can keep every thread on fixed columns (*colmax_done tells).
// With dst != NULL the updated w / m / v go to dst's buffers instead of in
// place (w16 and colmax are outputs already): the swap-out fused into the
// optimizer, which writes the new state straight into the parking buffer.
struct AdamDst {
    double* w;
    float* m;
    float* v;
};
template <typename G>
cudaError_t launch_adam(double* w, float* m, float* v, G* g, __nv_bfloat16* w16, uint64_t n,
                        double lr, double b1, double b2, double eps, double bc1, double bc2,
                        int zero_grad, double* gsq, int num_sms, cudaStream_t s,
                        int* colmax = nullptr, uint64_t D = 0, bool* colmax_done = nullptr,
                        const AdamDst* dst = nullptr);

cudaError_t launch_to_bf16(const double* w, __nv_bfloat16* w16, uint64_t n, int num_sms,
                           cudaStream_t s);

// Peer W16 row-range pointers (NVLink-mapped) of a DP gang, excluding self.
struct ShardPeers {
    int n;
    __nv_bfloat16* w16[7];
};
// K-adam, sharded over a DP gang: this rank's rows only; gradient = local
// partial + the receive slots the peers filled from their GEMM2 epilogues;
// the new bf16 rows are written locally and into every peer's W16.
cudaError_t launch_adam_shard(double* w, float* m, float* v, const float* g, const float* recv, int nslots,
                              uint64_t slot_stride, __nv_bfloat16* w16, ShardPeers peers, uint64_t n,
                              double lr, double b1, double b2, double eps, double bc1, double bc2,
                              double* gsq, int num_sms, cudaStream_t s, int* colmax = nullptr, uint64_t D = 0,
                              bool* colmax_done = nullptr);

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

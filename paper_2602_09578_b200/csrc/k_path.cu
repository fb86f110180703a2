// k_path.cu — HBM-bound kernels of the micro-batch policy-update path.
//
//   K-gather        experience-store gather + featurizer      experience_store.hpp:92-114,
//                                                               training.hpp:378-393, codec.hpp:24-30,
//                                                               policy.hpp:42-51
//   K-lse           cross-tile softmax normaliser, taken-token  policy.hpp:62-75
//                   log-prob, surrogate coefficient
//   K-adam          fused Adam + transposed bf16 shadow          training.hpp:37-51
//   K-adv           segmented GRPO normalisation                 training.hpp:54-67
//   parity mode     exact-featurizer fp64 SIMT path              policy.hpp:42-91
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "fm_kernels.h"
#include "fm_ptx.cuh"

namespace fm {

namespace {

__device__ __forceinline__ int token_of(uint64_t x) {  // static_cast<Token>(u64), codec.hpp:28
    return static_cast<int>(static_cast<uint32_t>(x));
}
__device__ __forceinline__ uint64_t feature_of(int tok, uint64_t D) {  // policy.hpp:48
    return static_cast<uint64_t>(static_cast<int64_t>(tok)) % D;
}


template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Block-wide sum for 256-thread blocks; result valid in every thread.
template <typename T>
__device__ T block_sum(T x, T* red) {
    x = warp_sum(x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    T t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : T(0);
    if (threadIdx.x < 32) t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
    __syncthreads();
    return red[0];
}

__device__ double block_max(double x, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : -INFINITY;
    if (threadIdx.x < 32) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    }
    if (threadIdx.x == 0) red[0] = t;
    __syncthreads();
    return red[0];
}

// ---------------------------------------------------------------------------
// K-gather
// ---------------------------------------------------------------------------
constexpr int kMaxSamplesSmem = 1024;

__global__ void __launch_bounds__(256) gather_kernel(const uint8_t* __restrict__ arena,
                                                     const SampleDesc* __restrict__ sd, int n_samples,
                                                     int64_t row_lo, int64_t M, int64_t Mpad, int64_t G,
                                                     uint64_t D, RowBuffers rows) {
    __shared__ int64_t s_start[kMaxSamplesSmem];
    const bool in_smem = n_samples <= kMaxSamplesSmem;  // larger micro-batches search global memory
    if (in_smem)
        for (int i = threadIdx.x; i < n_samples; i += blockDim.x) s_start[i] = sd[i].row_start;
    __syncthreads();
    auto start_of = [&](int i) { return in_smem ? s_start[i] : sd[i].row_start; };
    // last s with row_start[s] <= gr (rows are in poll order; empty samples share their successor's start)
    auto sample_of = [&](int64_t gr) {
        int lo = 0, hi = n_samples - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (start_of(mid) <= gr) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= Mpad) return;
    if (r >= M) {
        rows.action[r] = -1;
        rows.ctx4[r] = make_int4(-1, -1, -1, -1);
        rows.n_ctx[r] = 0;
        rows.sample[r] = -1;
        rows.coef[r] = 0.f;
        rows.rscale[r] = 0.f;
        if (rows.fmax) rows.mrow[r] = 0.f;
        if (rows.w16t) {
            rows.zact[r] = 0.f;
            rows.lossw[r] = 0.0;
        }
        return;
    }
    const int64_t gr = row_lo + r;
    const int lo = sample_of(gr);
    const SampleDesc d = sd[lo];
    const int64_t t = gr - d.row_start;
    const uint64_t* P = reinterpret_cast<const uint64_t*>(arena + d.prompt_off + 8);
    const uint64_t* R = reinterpret_cast<const uint64_t*>(arena + d.resp_off + 8);
    const int action = token_of(__ldg(R + t));
    const int64_t len = d.prompt_n + t;  // context = prompt ++ response[0:t]
    const int n = len < 4 ? static_cast<int>(len) : 4;
    int ctx[4] = {-1, -1, -1, -1};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (j < n) {
            const int64_t pos = len - n + j;
            ctx[j] = token_of(pos < d.prompt_n ? __ldg(P + pos) : __ldg(R + (pos - d.prompt_n)));
        }
    }
    rows.action[r] = action;
    rows.ctx4[r] = make_int4(ctx[0], ctx[1], ctx[2], ctx[3]);
    rows.n_ctx[r] = n;
    rows.sample[r] = lo;
    rows.coef[r] = n ? static_cast<float>(-d.adv / (static_cast<double>(G) * static_cast<double>(n))) : 0.f;
    const float rs = n ? static_cast<float>(1.0 / static_cast<double>(n)) : 0.f;
    rows.rscale[r] = rs;
    if (rows.fmax) {
        // softmax bound of the row, summed in K-stats' order over its four positions (the
        // first 4 - n are empty): fp32 addition is monotone, so mrow >= every logit
        float fm[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int j = k - (4 - n);
            fm[k] = j >= 0 ? __ldg(rows.fmax + feature_of(ctx[j], D)) : 0.f;
        }
        rows.mrow[r] = rs * ((fm[0] + fm[1]) + (fm[2] + fm[3]));
    }
    if (rows.w16t) {
        // the taken token's logit in K-stats' order (positions before the start are 0)
        const int64_t ac = static_cast<int64_t>(action) - rows.col_base;
        float za = 0.f;
        if (ac >= 0 && ac < rows.ncols) {
            float x[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = k - (4 - n);
                x[k] = j >= 0 ? __bfloat162float(rows.w16t[static_cast<int64_t>(feature_of(ctx[j], D)) * rows.ldw + ac])
                              : 0.f;
            }
            za = rs * ((x[0] + x[1]) + (x[2] + x[3]));
        }
        rows.zact[r] = za;
        rows.lossw[r] = -(d.adv / static_cast<double>(G));
    }
    if (rows.q0) {
        // band formulation (k_band.cu): every sample overlapping the shard owns its rows + 3
        // positions; this row's four context positions start at q0
        const int s_first = sample_of(row_lo);
        const int64_t a = d.row_start > row_lo ? d.row_start : row_lo;
        rows.q0[r] = static_cast<int32_t>((a - row_lo) + 3 * static_cast<int64_t>(lo - s_first) + (gr - a));
    }
}

// ---------------------------------------------------------------------------
// K-lse
// ---------------------------------------------------------------------------
// A block covers 32 rows with 8 warps: warp j sums slices j, j + 8, ... of its
// lane's row (the partial sums are [stats_ld][Mpad], so a warp reads 128
// contiguous bytes per slice and the block keeps 8 loads in flight per row),
// then warp 0 combines the 8 partials and finishes the row.
__global__ void __launch_bounds__(256) lse_kernel(const LseArgs L) {
    __shared__ float part[8][33];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 32 + lane;
    const bool live = r < L.M;
    if (!L.sum_in) {
        // 16 slices per warp in flight before any add: the loads are latency-bound (and share
        // HBM with a concurrent swap copy), the adds are free
        float acc = 0.f;
        if (live) {
            for (int t0 = 0; t0 < L.stats_ld; t0 += 128) {
                float x[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int t = t0 + wid + 8 * k;
                    x[k] = t < L.stats_ld ? __ldg(L.stats + static_cast<int64_t>(t) * L.Mpad + r) : 0.f;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] += x[k + 8];
#pragma unroll
                for (int k = 0; k < 4; ++k) x[k] += x[k + 4];
                acc += (x[0] + x[2]) + (x[1] + x[3]);
            }
        }
        part[wid][lane] = acc;
        __syncthreads();
    }
    if (wid != 0) return;
    double loss = 0.0;
    if (r < L.Mpad) {
        const RowBuffers& rows = L.rows;
        if (!live) {  // padding rows
            if (L.partial_out) {
                L.partial_out[r] = 0.f;
                L.partial_out[L.Mpad + r] = 0.f;
            } else {
                rows.lse[r] = 0.f;
                rows.logp[r] = 0.f;
                rows.coef_eff[r] = 0.f;
            }
        } else {
            float sum, za;
            if (L.sum_in) {  // vocabulary gang: the all-reduced row sum and taken logit
                sum = L.sum_in[r];
                za = L.sum_in[L.Mpad + r];
            } else {
                sum = ((part[0][lane] + part[1][lane]) + (part[2][lane] + part[3][lane])) +
                      ((part[4][lane] + part[5][lane]) + (part[6][lane] + part[7][lane]));
                za = L.rows.zact[r];  // (0 on a vocabulary-gang rank without the action's column)
            }
            if (L.partial_out) {  // this rank's columns only: to the all-reduce
                L.partial_out[r] = sum;
                L.partial_out[L.Mpad + r] = za;
            } else {
                const int a = rows.action[r];
                const double lw = rows.lossw[r];  // -A / G
                const float lse = rows.mrow[r] + __logf(sum);
                const bool valid = a >= 0 && a < L.V;
                const float lp = valid ? za - lse : 0.f;  // policy.hpp:72-75, fp32 logit
                float ce = rows.coef[r];
                if (L.old_logp && L.clip_eps > 0.f) {
                    // PPO clipped-ratio surrogate min(rho*A, clip(rho,1-e,1+e)*A): the
                    // gradient flows (scaled by rho) only through the unclipped branch.
                    const float rho = __expf(lp - L.old_logp[L.row_lo + r]);
                    const bool active = lw <= 0.0 ? rho <= 1.f + L.clip_eps : rho >= 1.f - L.clip_eps;  // A >= 0
                    ce = active ? ce * rho : 0.f;
                }
                rows.lse[r] = lse;
                rows.logp[r] = lp;
                rows.coef_eff[r] = ce;
                loss = valid ? lw * static_cast<double>(lp) : 0.0;
                // the bound keeps sum >= exp(max z - mrow); a vanishing sum would mean the bound
                // overshot the logits by ~87: report NaN rather than a silently wrong gradient
                if (!(sum >= 1e-30f) || !isfinite(sum)) loss = __longlong_as_double(0x7ff8000000000000ll);
            }
        }
    }
    if (L.loss_acc) {
        for (int o = 16; o > 0; o >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, o);
        if (lane == 0 && loss != 0.0) atomicAdd(L.loss_acc, loss);
    }
}

// ---------------------------------------------------------------------------
// K-adam
// ---------------------------------------------------------------------------
// fp32 gradient (BF16_TC): the moments are stored in fp32, so the moment update
// and the step lr·m̂/(√v̂+ε) are computed in fp32 (rel. error ~1e-7 on ΔW) and
// applied to the fp64 master weight.  This keeps the kernel on the HBM roofline:
// fp64 division + sqrt per parameter cost more issue slots than its 38 bytes.
struct AdamF {
    float b1, ob1, b2, ob2, lr_bc1, inv_bc2, eps;
    AdamF() = default;
    __host__ __device__ AdamF(double lr, double b1_, double b2_, double eps_, double bc1, double bc2)
        : b1(static_cast<float>(b1_)), ob1(static_cast<float>(1.0 - b1_)), b2(static_cast<float>(b2_)),
          ob2(static_cast<float>(1.0 - b2_)), lr_bc1(static_cast<float>(lr / bc1)),
          inv_bc2(static_cast<float>(1.0 / bc2)), eps(static_cast<float>(eps_)) {}
};

__device__ __forceinline__ double adam_f32(double& w, float& m, float& v, float g, const AdamF& c) {
    const float mm = fmaf(c.b1, m, c.ob1 * g);
    const float vv = fmaf(c.b2, v, c.ob2 * (g * g));
    w -= static_cast<double>(c.lr_bc1 * mm / (sqrtf(vv * c.inv_bc2) + c.eps));
    m = mm;
    v = vv;
    return static_cast<double>(g) * static_cast<double>(g);
}

// fp64 gradient (PARITY_F64): the reference's own fp64 arithmetic order.
__device__ __forceinline__ double adam_f64(double& w, float& m, float& v, double g, double lr, double b1,
                                           double b2, double eps, double bc1, double bc2) {
    const double gi = g;
    const double mm = b1 * static_cast<double>(m) + (1.0 - b1) * gi;
    const double vv = b2 * static_cast<double>(v) + (1.0 - b2) * gi * gi;
    const double mhat = mm / bc1;
    const double vhat = vv / bc2;
    w -= lr * mhat / (sqrt(vhat) + eps);
    m = static_cast<float>(mm);
    v = static_cast<float>(vv);
    return gi * gi;
}

// 32 (rows v) x 64 (columns d) tiles; thread = one row, 8 consecutive columns.
constexpr int kTileV = 32, kTileD = 64, kTPitch = 40;  // smem transpose pitch in bf16 (16-B aligned rows)

template <typename G>
struct AdamTileArgs {
    double* w;
    float* m;
    float* v;
    G* g;
    uint64_t V, D, r0, r1;
    const float* recv;  // [nslots][r1 - r0][D]
    int nslots;
    __nv_bfloat16* w16t;
    uint64_t ldw;
    ShardPeers peers;
    double* w_o;  // the swap-out fused into the optimizer: new w / m / v here (else in place)
    float* m_o;
    float* v_o;
    int zero_grad;
    double* gsq;
    double lr, b1, b2, eps, bc1, bc2;
    AdamF cf;  // fp32 coefficients, computed on the host (kernel-parameter space, no registers)
};

template <bool kPeers>
__device__ __noinline__ void store_w16t_tail(uint4 val, uint64_t off, int n, __nv_bfloat16* w16t,
                                             const ShardPeers& peers) {
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&val);
    for (int k = 0; k < n; ++k) {
        w16t[off + k] = e[k];
        if constexpr (kPeers)
            for (int p = 0; p < peers.n; ++p) peers.w16t[p][off + k] = e[k];
    }
}

// Stores the tile's bf16 values (tsh[col][row]) as W16^T rows: thread -> one
// column d, 8 consecutive rows (16 B).  Rows are 8-aligned (vbase % 8 == 0).
// kPeers: also into the DP gang peers' shadows (token-shard gang).
template <bool kPeers>
__device__ __forceinline__ void store_w16t_tile(const __nv_bfloat16 (*tsh)[kTPitch], uint64_t vbase, uint64_t dbase,
                                                uint64_t r1, uint64_t D, __nv_bfloat16* w16t, uint64_t ldw,
                                                const ShardPeers& peers) {
    const int dl = threadIdx.x >> 2, rc = (threadIdx.x & 3) * 8;
    const uint64_t d = dbase + dl, vb = vbase + rc;
    if (d >= D || vb >= r1) return;
    const uint4 val = *reinterpret_cast<const uint4*>(&tsh[dl][rc]);
    const uint64_t off = d * ldw + vb;
    if (vb + 8 <= r1) {
        *reinterpret_cast<uint4*>(w16t + off) = val;
        if constexpr (kPeers)
            for (int p = 0; p < peers.n; ++p) *reinterpret_cast<uint4*>(peers.w16t[p] + off) = val;
    } else {
        store_w16t_tail<kPeers>(val, off, static_cast<int>(r1 - vb), w16t, peers);
    }
}

// K-adam: one 32 x 64 tile per loop trip, thread -> one vocabulary row, 8
// consecutive features (64 B of W, 32 B each of m / v / g).  The launch is many
// short-lived blocks rather than a persistent grid (tools/adam_probe.cu: 8
// blocks per SM looping over ~54 tiles each ran at 0.83 of copy bandwidth, ~64
// per SM at 0.95); the fp32 coefficients live in parameter space and 64
// registers keep 4 blocks resident per SM.

#ifndef FM_ADAM_MIN_BLOCKS
#define FM_ADAM_MIN_BLOCKS 4
#endif
template <typename G, bool kVec, bool kPeers>
__global__ void __launch_bounds__(256, FM_ADAM_MIN_BLOCKS) adam_tile_kernel(const AdamTileArgs<G> A) {
    __shared__ __align__(16) __nv_bfloat16 tsh[kTileD][kTPitch];
    __shared__ double red[8];
    const AdamF& cf = A.cf;
    const uint64_t rows = A.r1 - A.r0;
    const uint64_t tv_n = (rows + kTileV - 1) / kTileV, td_n = (A.D + kTileD - 1) / kTileD;
    const uint64_t ntiles = tv_n * td_n;
    const int tr = static_cast<int>(threadIdx.x >> 3), tc = static_cast<int>(threadIdx.x & 7) * 8;
    const uint64_t sstride = rows * A.D;
    double acc = 0.0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t tv = t / td_n, td = t % td_n;
        const uint64_t vr = A.r0 + tv * kTileV + tr;
        const uint64_t d0 = td * kTileD + tc;
        float wf[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (vr < A.r1 && d0 < A.D) {
            const uint64_t i0 = vr * A.D + d0;
            const int nv = kVec ? 8 : (A.D - d0 >= 8 ? 8 : static_cast<int>(A.D - d0));
            double wv[8];
            float mv[8], vv[8];
            G gv[8];
            if constexpr (kVec) {
                const double2* __restrict__ wp = reinterpret_cast<const double2*>(A.w + i0);
                const float4* __restrict__ mp = reinterpret_cast<const float4*>(A.m + i0);
                const float4* __restrict__ vp = reinterpret_cast<const float4*>(A.v + i0);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double2 x = wp[q];
                    wv[2 * q] = x.x;
                    wv[2 * q + 1] = x.y;
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const float4 a = mp[q], b = vp[q];
                    mv[4 * q] = a.x; mv[4 * q + 1] = a.y; mv[4 * q + 2] = a.z; mv[4 * q + 3] = a.w;
                    vv[4 * q] = b.x; vv[4 * q + 1] = b.y; vv[4 * q + 2] = b.z; vv[4 * q + 3] = b.w;
                }
                if constexpr (sizeof(G) == 4) {
                    const float4* __restrict__ gp = reinterpret_cast<const float4*>(A.g + i0);
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const float4 c = gp[q];
                        gv[4 * q] = c.x; gv[4 * q + 1] = c.y; gv[4 * q + 2] = c.z; gv[4 * q + 3] = c.w;
                    }
                } else {
                    const double2* __restrict__ gp = reinterpret_cast<const double2*>(A.g + i0);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double2 c = gp[q];
                        gv[2 * q] = c.x;
                        gv[2 * q + 1] = c.y;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    wv[j] = j < nv ? A.w[i0 + j] : 0.0;
                    mv[j] = j < nv ? A.m[i0 + j] : 0.f;
                    vv[j] = j < nv ? A.v[i0 + j] : 0.f;
                    gv[j] = j < nv ? A.g[i0 + j] : G(0);
                }
            }
            if (A.nslots) {  // DP gang: the peers' partials of this rank's rows
                const uint64_t li = (vr - A.r0) * A.D + d0;
                for (int sl = 0; sl < A.nslots; ++sl) {
                    const float* rp = A.recv + sl * sstride + li;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < nv) gv[j] += static_cast<G>(rp[j]);
                }
            }
            if constexpr (sizeof(G) == 4) {
                // fp32 g^2 within the thread's 8 elements, fp64 across them
                float sq = 0.f;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (j < nv) {
                        adam_f32(wv[j], mv[j], vv[j], gv[j], cf);
                        sq = fmaf(gv[j], gv[j], sq);
                    }
                    wf[j] = static_cast<float>(wv[j]);
                }
                acc += static_cast<double>(sq);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (j < nv) acc += adam_f64(wv[j], mv[j], vv[j], gv[j], A.lr, A.b1, A.b2, A.eps, A.bc1, A.bc2);
                    wf[j] = static_cast<float>(wv[j]);
                }
            }
            double* const w_o = A.w_o ? A.w_o : A.w;
            float* const m_o = A.w_o ? A.m_o : A.m;
            float* const v_o = A.w_o ? A.v_o : A.v;
            if constexpr (kVec) {
#pragma unroll
                for (int q = 0; q < 4; ++q) reinterpret_cast<double2*>(w_o + i0)[q] = make_double2(wv[2 * q], wv[2 * q + 1]);
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    reinterpret_cast<float4*>(m_o + i0)[q] = make_float4(mv[4 * q], mv[4 * q + 1], mv[4 * q + 2], mv[4 * q + 3]);
                    reinterpret_cast<float4*>(v_o + i0)[q] = make_float4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < nv) {
                        w_o[i0 + j] = wv[j];
                        m_o[i0 + j] = mv[j];
                        v_o[i0 + j] = vv[j];
                    }
            }
            if (A.zero_grad) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < nv) A.g[i0 + j] = G(0);
            }
        }
        if (A.w16t) {  // uniform: the transposed shadow through shared memory
#pragma unroll
            for (int j = 0; j < 8; ++j) tsh[tc + j][tr] = __float2bfloat16_rn(wf[j]);
            __syncthreads();
            store_w16t_tile<kPeers>(tsh, A.r0 + tv * kTileV, td * kTileD, A.r1, A.D, A.w16t, A.ldw, A.peers);
            __syncthreads();
        }
    }
    if (A.gsq) {
        const double tot = block_sum(acc, red);
        if (threadIdx.x == 0) atomicAdd(A.gsq, tot);
    }
}

// W16^T = bf16(W), same tiles (shadow refresh).
__global__ void __launch_bounds__(256) w16t_kernel(const double* __restrict__ w, uint64_t V, uint64_t D,
                                                   __nv_bfloat16* __restrict__ w16t, uint64_t ldw) {
    __shared__ __align__(16) __nv_bfloat16 tsh[kTileD][kTPitch];
    const uint64_t tv_n = (V + kTileV - 1) / kTileV, td_n = (D + kTileD - 1) / kTileD;
    const int tr = static_cast<int>(threadIdx.x >> 3), tc = static_cast<int>(threadIdx.x & 7) * 8;
    const ShardPeers none{};
    for (uint64_t t = blockIdx.x; t < tv_n * td_n; t += gridDim.x) {
        const uint64_t tv = t / td_n, td = t % td_n;
        const uint64_t vr = tv * kTileV + tr, d0 = td * kTileD + tc;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            tsh[tc + j][tr] = __float2bfloat16_rn(vr < V && d0 + j < D ? static_cast<float>(w[vr * D + d0 + j]) : 0.f);
        __syncthreads();
        store_w16t_tile<false>(tsh, tv * kTileV, td * kTileD, V, D, w16t, ldw, none);
        __syncthreads();
    }
}

// out[v][d] = W16^T[d][v]: 32 x 32 tiles through shared memory.
__global__ void w16t_untranspose_kernel(const __nv_bfloat16* __restrict__ w16t, uint64_t V, uint64_t D, uint64_t ldw,
                                        __nv_bfloat16* __restrict__ out) {
    __shared__ __nv_bfloat16 t[32][33];
    const uint64_t v0 = static_cast<uint64_t>(blockIdx.x) * 32, d0 = static_cast<uint64_t>(blockIdx.y) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const uint64_t d = d0 + i, v = v0 + threadIdx.x;
        if (d < D && v < V) t[i][threadIdx.x] = w16t[d * ldw + v];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const uint64_t v = v0 + i, d = d0 + threadIdx.x;
        if (d < D && v < V) out[v * D + d] = t[threadIdx.x][i];
    }
}

__global__ void axpy_init_kernel(float* __restrict__ dst, const float* __restrict__ src, uint64_t n4, int acc) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 x = reinterpret_cast<const float4*>(src)[i];
        if (acc) {
            const float4 d = reinterpret_cast<const float4*>(dst)[i];
            x.x += d.x;
            x.y += d.y;
            x.z += d.z;
            x.w += d.w;
        }
        reinterpret_cast<float4*>(dst)[i] = x;
    }
}

__global__ void sumsq_kernel(const float* __restrict__ x, uint64_t n, double* out) {
    __shared__ double red[8];
    double acc = 0.0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = x[i];
        acc += v * v;
    }
    const double tot = block_sum(acc, red);
    if (threadIdx.x == 0) atomicAdd(out, tot);
}

__global__ void to_bf16_kernel(const double* __restrict__ w, __nv_bfloat16* __restrict__ w16, uint64_t n) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        w16[i] = __float2bfloat16_rn(static_cast<float>(w[i]));
}

// ---------------------------------------------------------------------------
// K-adv: one warp per reward group.
// ---------------------------------------------------------------------------
__global__ void group_adv_kernel(const double* __restrict__ r, const int32_t* __restrict__ off, int nseg,
                                 double eps, double* __restrict__ out) {
    const int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (seg >= nseg) return;
    const int b = off[seg], e = off[seg + 1];
    const int n = e - b;
    if (n <= 0) return;
    double s = 0.0;
    for (int i = b + lane; i < e; i += 32) s += r[i];
    const double mean = warp_sum(s) / static_cast<double>(n);
    double q = 0.0;
    for (int i = b + lane; i < e; i += 32) q += (r[i] - mean) * (r[i] - mean);
    const double sd = sqrt(warp_sum(q) / static_cast<double>(n));
    for (int i = b + lane; i < e; i += 32) out[i] = (r[i] - mean) / (sd + eps);
}

// ---------------------------------------------------------------------------
// Parity mode: one 256-thread block per packed row, fp64 throughout.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) parity_rows_kernel(const double* __restrict__ W, uint64_t V, uint64_t D,
                                                          RowBuffers rows, const SampleDesc* __restrict__ sd,
                                                          int64_t G, double* __restrict__ zs,
                                                          double* __restrict__ dWmb, double* logp64,
                                                          double* loss_acc) {
    __shared__ double red[8];
    __shared__ uint64_t s_f[4];
    __shared__ double s_phi[4];
    __shared__ int s_nf;
    const int64_t r = blockIdx.x;
    const int n = rows.n_ctx[r];
    const int a = rows.action[r];
    if (threadIdx.x == 0) {
        const int4 c4 = rows.ctx4[r];
        const int ctx[4] = {c4.x, c4.y, c4.z, c4.w};
        const double w = n ? 1.0 / static_cast<double>(n) : 0.0;
        int nf = 0;
        for (int j = 0; j < n; ++j) {  // phi[tok % D] += 1/n   (policy.hpp:46-49)
            const uint64_t f = feature_of(ctx[j], D);
            int k = 0;
            while (k < nf && s_f[k] != f) ++k;
            if (k == nf) {
                s_f[nf] = f;
                s_phi[nf] = 0.0;
                ++nf;
            }
            s_phi[k] = __dadd_rn(s_phi[k], w);
        }
        for (int i = 1; i < nf; ++i)  // ascending feature order = the reference's d loop order
            for (int k = i; k > 0 && s_f[k - 1] > s_f[k]; --k) {
                const uint64_t tf = s_f[k]; s_f[k] = s_f[k - 1]; s_f[k - 1] = tf;
                const double tp = s_phi[k]; s_phi[k] = s_phi[k - 1]; s_phi[k - 1] = tp;
            }
        s_nf = nf;
    }
    __syncthreads();
    const int nf = s_nf;
    double* z = zs + static_cast<size_t>(r) * V;
    double lmax = -INFINITY;
    for (uint64_t v = threadIdx.x; v < V; v += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nf; ++k) s = __dadd_rn(s, __dmul_rn(W[v * D + s_f[k]], s_phi[k]));
        z[v] = s;
        lmax = fmax(lmax, s);
    }
    const double zmax = block_max(lmax, red);
    double lsum = 0.0;
    for (uint64_t v = threadIdx.x; v < V; v += blockDim.x) {
        const double e = exp(z[v] - zmax);
        z[v] = e;
        lsum += e;
    }
    const double denom = block_sum(lsum, red);
    const double adv = sd[rows.sample[r]].adv;
    const double scale = -adv / static_cast<double>(G);  // term.scale(A) then grad.scale(-1/G)
    for (uint64_t v = threadIdx.x; v < V; v += blockDim.x) {
        const double p = z[v] / denom;
        const double coef = ((static_cast<int64_t>(v) == a) ? 1.0 : 0.0) - p;
        if (coef == 0.0) continue;  // policy.hpp:86
        for (int k = 0; k < nf; ++k) atomicAdd(&dWmb[v * D + s_f[k]], scale * (coef * s_phi[k]));
    }
    if (threadIdx.x == 0) {  // z[] holds exp(z - zmax); block_sum's barrier made it visible
        const bool valid = a >= 0 && static_cast<uint64_t>(a) < V;
        const double lp = valid ? log(z[a] / denom) : 0.0;  // policy.hpp:72-75
        if (logp64) logp64[r] = lp;
        if (loss_acc && valid) atomicAdd(loss_acc, -(adv / static_cast<double>(G)) * lp);
    }
}

__global__ void parity_fold_kernel(double* __restrict__ dW, double* __restrict__ dWmb, uint64_t n, double* sumsq) {
    __shared__ double red[8];
    double acc = 0.0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double x = dWmb[i];
        acc += x * x;
        dW[i] += x;
        dWmb[i] = 0.0;
    }
    const double tot = block_sum(acc, red);
    if (threadIdx.x == 0 && sumsq) atomicAdd(sumsq, tot);
}

}  // namespace

// ---------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------
cudaError_t launch_gather(const uint8_t* arena, const SampleDesc* sd, int n_samples, int64_t row_lo, int64_t M,
                          int64_t Mpad, int64_t global_batch, uint64_t D, RowBuffers rows, cudaStream_t s) {
    if (Mpad == 0) return cudaSuccess;
    const int blocks = static_cast<int>((Mpad + 255) / 256);
    gather_kernel<<<blocks, 256, 0, s>>>(arena, sd, n_samples, row_lo, M, Mpad, global_batch, D, rows);
    return cudaGetLastError();
}

namespace {
template <typename T>
__global__ void gather_cols_kernel(const T* __restrict__ src, uint64_t V, uint64_t D,
                                   const int64_t* __restrict__ cols, int64_t nc, T* __restrict__ out) {
    const uint64_t n = V * static_cast<uint64_t>(nc);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = src[(i / nc) * D + cols[i % nc]];
}
}  // namespace

cudaError_t launch_gather_cols(const void* dW, bool f64, uint64_t V, uint64_t D, const int64_t* cols,
                               int64_t n_cols, void* out, cudaStream_t s) {
    if (f64)
        gather_cols_kernel<<<1184, 256, 0, s>>>(static_cast<const double*>(dW), V, D, cols, n_cols,
                                                static_cast<double*>(out));
    else
        gather_cols_kernel<<<1184, 256, 0, s>>>(static_cast<const float*>(dW), V, D, cols, n_cols,
                                                static_cast<float*>(out));
    return cudaGetLastError();
}

cudaError_t launch_lse(const LseArgs& L, cudaStream_t s) {
    if (L.Mpad == 0) return cudaSuccess;
    lse_kernel<<<static_cast<unsigned>((L.Mpad + 31) / 32), 256, 0, s>>>(L);
    return cudaGetLastError();
}

template <typename G>
cudaError_t launch_adam(double* w, float* m, float* v, G* g, uint64_t V, uint64_t D, uint64_t r0, uint64_t r1,
                        const float* recv, int nslots, __nv_bfloat16* w16t, uint64_t ldw, ShardPeers peers, double lr,
                        double b1, double b2, double eps, double bc1, double bc2, int zero_grad, double* gsq,
                        int num_sms, cudaStream_t s, const AdamDst* dst) {
    if (r1 <= r0 || D == 0) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g)) & 15) return cudaErrorMisalignedAddress;
    if (dst && (reinterpret_cast<uintptr_t>(dst->w) & 15)) return cudaErrorMisalignedAddress;
    if (w16t && ((r0 & 7) || (ldw & 7))) return cudaErrorInvalidValue;
    AdamTileArgs<G> A{w, m, v, g, V, D, r0, r1, recv, nslots, w16t, ldw, peers,
                      dst ? dst->w : nullptr, dst ? dst->m : nullptr, dst ? dst->v : nullptr, zero_grad, gsq, lr, b1, b2, eps, bc1, bc2, AdamF(lr, b1, b2, eps, bc1, bc2)};
    const uint64_t tiles = ((r1 - r0 + kTileV - 1) / kTileV) * ((D + kTileD - 1) / kTileD);
    // 64 blocks per SM (~7 tiles each) at D <= 4,096; one block per tile for wider rows
    // (measured: C2 0.82 ms vs 0.87 with one tile per block; C3, D = 32,768, 7.39 ms
    // with 64 blocks per SM vs 6.72 ms with one tile per block)
    const uint64_t td_n = (D + kTileD - 1) / kTileD;
    const uint64_t cap = td_n > 64 ? tiles : static_cast<uint64_t>(num_sms) * 64;
    if (cap > 0x7fffffffull) return cudaErrorInvalidValue;
    const int grid = static_cast<int>(tiles < cap ? tiles : cap);
    const bool vec = D % 8 == 0;
    if (peers.n > 0) {
        if (vec) adam_tile_kernel<G, true, true><<<grid, 256, 0, s>>>(A);
        else adam_tile_kernel<G, false, true><<<grid, 256, 0, s>>>(A);
    } else {
        if (vec) adam_tile_kernel<G, true, false><<<grid, 256, 0, s>>>(A);
        else adam_tile_kernel<G, false, false><<<grid, 256, 0, s>>>(A);
    }
    return cudaGetLastError();
}
template cudaError_t launch_adam<float>(double*, float*, float*, float*, uint64_t, uint64_t, uint64_t, uint64_t,
                                        const float*, int, __nv_bfloat16*, uint64_t, ShardPeers, double, double,
                                        double, double, double, double, int, double*, int, cudaStream_t,
                                        const AdamDst*);
template cudaError_t launch_adam<double>(double*, float*, float*, double*, uint64_t, uint64_t, uint64_t, uint64_t,
                                         const float*, int, __nv_bfloat16*, uint64_t, ShardPeers, double, double,
                                         double, double, double, double, int, double*, int, cudaStream_t,
                                        const AdamDst*);

cudaError_t launch_w16t(const double* w, uint64_t V, uint64_t D, __nv_bfloat16* w16t, uint64_t ldw, int num_sms,
                        cudaStream_t s) {
    if (V == 0 || D == 0) return cudaSuccess;
    if (ldw & 7) return cudaErrorInvalidValue;
    const uint64_t tiles = ((V + kTileV - 1) / kTileV) * ((D + kTileD - 1) / kTileD);
    const uint64_t cap = static_cast<uint64_t>(num_sms) * 8;
    w16t_kernel<<<static_cast<int>(tiles < cap ? tiles : cap), 256, 0, s>>>(w, V, D, w16t, ldw);
    return cudaGetLastError();
}

cudaError_t launch_w16t_untranspose(const __nv_bfloat16* w16t, uint64_t V, uint64_t D, uint64_t ldw,
                                    __nv_bfloat16* out, cudaStream_t s) {
    if (V == 0 || D == 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>((V + 31) / 32), static_cast<unsigned>((D + 31) / 32));
    w16t_untranspose_kernel<<<grid, dim3(32, 8), 0, s>>>(w16t, V, D, ldw, out);
    return cudaGetLastError();
}

cudaError_t launch_axpy_init(float* dst, const float* src, uint64_t n, int accumulate, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (n % 4) return cudaErrorInvalidValue;
    axpy_init_kernel<<<num_sms * 8, 256, 0, s>>>(dst, src, n / 4, accumulate);
    return cudaGetLastError();
}

cudaError_t launch_sumsq(const float* x, uint64_t n, double* out, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    sumsq_kernel<<<num_sms * 8, 256, 0, s>>>(x, n, out);
    return cudaGetLastError();
}

cudaError_t launch_to_bf16(const double* w, __nv_bfloat16* w16, uint64_t n, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    to_bf16_kernel<<<num_sms * 8, 256, 0, s>>>(w, w16, n);
    return cudaGetLastError();
}

cudaError_t launch_group_advantages(const double* rewards, const int32_t* seg_off, int nseg, double eps,
                                    double* out, cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    const int blocks = (nseg * 32 + 255) / 256;
    group_adv_kernel<<<blocks, 256, 0, s>>>(rewards, seg_off, nseg, eps, out);
    return cudaGetLastError();
}

cudaError_t launch_parity_rows(const double* W, uint64_t V, uint64_t D, int64_t M, RowBuffers rows,
                               const SampleDesc* sd, int64_t global_batch, double* zscratch, double* dWmb,
                               double* logp64, double* loss_acc, cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    parity_rows_kernel<<<static_cast<unsigned>(M), 256, 0, s>>>(W, V, D, rows, sd, global_batch, zscratch, dWmb,
                                                                logp64, loss_acc);
    return cudaGetLastError();
}

cudaError_t launch_parity_fold(double* dW, double* dWmb, uint64_t n, double* sumsq, int num_sms, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t want = (n + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(num_sms) * 8;
    parity_fold_kernel<<<static_cast<unsigned>(want > cap ? cap : want), 256, 0, s>>>(dW, dWmb, n, sumsq);
    return cudaGetLastError();
}

}  // namespace fm

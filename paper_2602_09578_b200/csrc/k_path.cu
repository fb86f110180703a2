// k_path.cu — HBM-bound kernels of the micro-batch policy-update path.
//
//   K-gather        experience-store gather + featurizer      experience_store.hpp:92-114,
//                                                               training.hpp:378-393, codec.hpp:24-30,
//                                                               policy.hpp:42-51
//   K-lse           cross-tile softmax normaliser, taken-token  policy.hpp:62-75
//                   log-prob, surrogate coefficient
//   K-softmax-grad  fused log-softmax gradient over the vocab   policy.hpp:83-90, training.hpp:394
//                   (TMA-staged Z tiles in, TMA-stored G^T out)
//   K-adam          fused Adam + bf16 shadow + grad reset        training.hpp:37-51
//   K-adv           segmented GRPO normalisation                 training.hpp:54-67
//   parity mode     exact-featurizer fp64 SIMT path              policy.hpp:42-91
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "fm_kernels.h"
#include "fm_lse.cuh"
#include "fm_ptx.cuh"

namespace fm {

namespace {

__device__ __forceinline__ int token_of(uint64_t x) {  // static_cast<Token>(u64), codec.hpp:28
    return static_cast<int>(static_cast<uint32_t>(x));
}
__device__ __forceinline__ uint64_t feature_of(int tok, uint64_t D) {  // policy.hpp:48
    return static_cast<uint64_t>(static_cast<int64_t>(tok)) % D;
}

// order-preserving float <-> int keys (atomicMax on floats of either sign)
__device__ __forceinline__ int fkey(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float unkey(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

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
                                                     uint64_t D,
                                                     RowBuffers rows, __nv_bfloat16* phic,
                                                     __nv_bfloat16* phict, int clear_old,
                                                     const int* __restrict__ colmax) {
    __shared__ int64_t s_start[kMaxSamplesSmem];
    const int ns = n_samples < kMaxSamplesSmem ? n_samples : kMaxSamplesSmem;
    for (int i = threadIdx.x; i < ns; i += blockDim.x) s_start[i] = sd[i].row_start;
    __syncthreads();
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= Mpad) return;
    if (phic && clear_old) {
        // Phic / Phic^T still hold the previous micro-batch's pattern (same Mpad, D):
        // row r's thread owns row r of Phic and column r of Phic^T, so it erases its
        // <= 4 old entries instead of a 2 x Mpad x D memset.
        const int on = rows.n_ctx[r];
        const int4 oc = rows.ctx4[r];
        const int old[4] = {oc.x, oc.y, oc.z, oc.w};
        const __nv_bfloat16 z = __float2bfloat16_rn(0.f);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j < on) {
                const uint64_t f = feature_of(old[j], D);
                phic[static_cast<size_t>(r) * D + f] = z;
                phict[static_cast<size_t>(f) * Mpad + r] = z;
            }
        }
    }
    if (r >= M) {
        rows.action[r] = -1;
        rows.ctx4[r] = make_int4(-1, -1, -1, -1);
        if (rows.feat4) {
            rows.feat4[r] = make_int4(-1, -1, -1, -1);
            rows.cnt4[r] = 0u;
        }
        rows.n_ctx[r] = 0;
        rows.sample[r] = -1;
        rows.coef[r] = 0.f;
        rows.rscale[r] = 0.f;
        if (colmax) rows.mrow[r] = 0.f;
        return;
    }
    // sample owning global row gr: last s with row_start[s] <= gr (rows are in poll order)
    const int64_t gr = row_lo + r;
    int lo = 0, hi = ns - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_start[mid] <= gr) lo = mid;
        else hi = mid - 1;
    }
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
    rows.rscale[r] = n ? static_cast<float>(1.0 / static_cast<double>(n)) : 0.f;
    if (phic) {
        uint64_t f[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) f[j] = j < n ? feature_of(ctx[j], D) : ~0ull;
        int uf[4] = {-1, -1, -1, -1};
        uint32_t packed = 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j >= n) continue;
            int cnt = 0;
            bool first = true;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                cnt += (f[k] == f[j]);
                if (k < j && f[k] == f[j]) first = false;
            }
            const __nv_bfloat16 c = __float2bfloat16_rn(static_cast<float>(cnt));  // exact: 1..4
            phic[static_cast<size_t>(r) * D + f[j]] = c;
            phict[static_cast<size_t>(f[j]) * Mpad + r] = c;
            if (first) {  // unique features + counts for the fused-loss B transform
                uf[j] = static_cast<int>(f[j]);
                packed |= static_cast<uint32_t>(cnt) << (8 * j);
            }
        }
        if (rows.feat4) {
            rows.feat4[r] = make_int4(uf[0], uf[1], uf[2], uf[3]);
            rows.cnt4[r] = packed;
        }
        if (colmax) {
            // softmax offset bound: z[r][v] = (1/n) sum_j W[v][f_j] <= (1/n) sum_j colmax[f_j]
            float b = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < n) b += unkey(__ldg(colmax + f[j]));
            rows.mrow[r] = n ? b / static_cast<float>(n) : 0.f;
        }
    }
}

// ---------------------------------------------------------------------------
// K-colmax: per-feature-column max of the bf16 shadow, colmax[d] = max_v W16[v][d],
// as order-preserving int keys (atomicMax).  Thread = 8 consecutive columns
// (one 16-B load per row), blockIdx.y strides the rows.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) colmax_kernel(const __nv_bfloat16* __restrict__ w16, int64_t V, int64_t D,
                                                     int* __restrict__ keys) {
    const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
    if (c0 >= D) return;
    float mx[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
    if ((D & 7) == 0) {
#pragma unroll 4
        for (int64_t v = blockIdx.y; v < V; v += gridDim.y) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(w16 + v * D + c0));
            const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[j]));
                mx[2 * j] = fmaxf(mx[2 * j], f.x);
                mx[2 * j + 1] = fmaxf(mx[2 * j + 1], f.y);
            }
        }
    } else {
        for (int64_t v = blockIdx.y; v < V; v += gridDim.y)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c0 + j < D) mx[j] = fmaxf(mx[j], __bfloat162float(w16[v * D + c0 + j]));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (c0 + j < D) atomicMax(keys + c0 + j, fkey(mx[j]));
}

// ---------------------------------------------------------------------------
// K-lse
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) lse_kernel(LseArgs L) {
    // Four rows per warp (8 lanes per row, fm_lse.cuh), persistent over row quads.
    // The kernel is latency/issue bound (1 KB of partials per row at C2).  With the
    // loss fold GEMM1 runs this same routine in its last-tile epilogue instead
    // (FM_LSE_FUSED, default on), and this kernel is not launched.
    __shared__ double red[8];
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    double loss = 0.0;
    for (int64_t r0 = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 4; r0 < L.Mpad;
         r0 += nwarps * 4)
        loss += lse_row_quad(L, r0);
    if (L.loss_acc) {
        const double tot = block_sum(loss, red);
        if (threadIdx.x == 0 && tot != 0.0) atomicAdd(L.loss_acc, tot);
    }
}

// ---------------------------------------------------------------------------
// K-softmax-grad: 64 rows x 128 vocab per CTA.
// ---------------------------------------------------------------------------
constexpr int kSgRows = 64, kSgCols = 128;
constexpr uint32_t kSgPBytes = kSgRows * kSgCols * 2;  // 16 KB bf16 p~ tile
constexpr uint32_t kSgGBytes = kSgRows * kSgCols * 2;  // 16 KB bf16 G^T tile (swizzled 128 B rows)

__global__ void __launch_bounds__(256) softmax_grad_kernel(const __grid_constant__ CUtensorMap tmP,
                                                           const __grid_constant__ CUtensorMap tmGt,
                                                           const float2* __restrict__ stats, int stats_ld,
                                                           RowBuffers rows, int part_cols) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    const __nv_bfloat16* Ps = reinterpret_cast<const __nv_bfloat16*>(smem);
    uint8_t* Gs = smem + kSgPBytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kSgPBytes + kSgGBytes);
    float* s_scale = reinterpret_cast<float*>(bar + 2);
    float* s_coef = s_scale + kSgRows;
    int* s_act = reinterpret_cast<int*>(s_coef + kSgRows);

    const int v0 = blockIdx.x * kSgCols;
    const int r0 = blockIdx.y * kSgRows;
    const int tile = v0 / part_cols;  // GEMM1's softmax partial (per tile, or per tile half) holding these columns
    const int tid = threadIdx.x;
    if (tid == 0) {
        tma_prefetch(&tmP);
        mbar_init(bar, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(bar, kSgPBytes);
        tma_load_2d_hint(reinterpret_cast<void*>(smem), &tmP, bar, v0, r0, policy_evict_first());
    }
    if (tid < kSgRows) {
        const int r = r0 + tid;
        const float c = rows.coef_eff[r];
        s_coef[tid] = c;
        s_act[tid] = rows.action[r];
        // p = p~ * exp(m_tile - lse)   (p~ = exp(z - m_tile) from GEMM1's epilogue)
        s_scale[tid] = c == 0.f ? 0.f : __expf(stats[static_cast<size_t>(r) * stats_ld + tile].x - rows.lse[r]);
    }
    __syncthreads();
    mbar_wait(bar, 0);

    const int vl = tid & (kSgCols - 1);
    const int rg = tid >> 7;  // 0/1: rows [32*rg, 32*rg+32)
    const int v = v0 + vl;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int chunk = rg * 4 + c;  // 8 consecutive rows = one 16 B chunk of the G^T row
        uint32_t packed[4];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            const int ra = chunk * 8 + i, rb = ra + 1;
            const float ca = s_coef[ra], cb = s_coef[rb];
            const float ga = ca == 0.f ? 0.f
                                       : ca * ((v == s_act[ra] ? 1.f : 0.f) -
                                               __bfloat162float(Ps[ra * kSgCols + vl]) * s_scale[ra]);
            const float gb = cb == 0.f ? 0.f
                                       : cb * ((v == s_act[rb] ? 1.f : 0.f) -
                                               __bfloat162float(Ps[rb * kSgCols + vl]) * s_scale[rb]);
            const __nv_bfloat162 h = __floats2bfloat162_rn(ga, gb);  // .x = low = row ra
            packed[i >> 1] = *reinterpret_cast<const uint32_t*>(&h);
        }
        // SWIZZLE_128B: 16 B chunk j of 128 B row i lives at chunk j ^ (i % 8)
        *reinterpret_cast<uint4*>(Gs + vl * 128 + ((chunk ^ (vl & 7)) << 4)) =
            make_uint4(packed[0], packed[1], packed[2], packed[3]);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
        tma_store_2d(&tmGt, Gs, r0, v0);
        tma_store_commit();
        tma_store_wait<0>();
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
    __device__ AdamF(double lr, double b1_, double b2_, double eps_, double bc1, double bc2)
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

template <typename G>
__global__ void __launch_bounds__(256) adam_kernel(double* __restrict__ w, float* __restrict__ m,
                                                   float* __restrict__ v, G* __restrict__ g,
                                                   __nv_bfloat16* __restrict__ w16, uint64_t n,
                                                   double lr, double b1, double b2, double eps,
                                                   double bc1, double bc2, int zero_grad, double* gsq,
                                                   int* __restrict__ cm, uint64_t D, double* w_o, float* m_o,
                                                   float* v_o) {
    __shared__ double red[8];
    // outputs: in place, or the parking buffer (fused swap-out)
    if (!w_o) {
        w_o = w;
        m_o = m;
        v_o = v;
    }
    double acc = 0.0;
    // colmax fused (cm != null): the launcher sized the grid so that a thread's four
    // elements sit in the same four columns on every iteration
    float cmx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    const AdamF cf(lr, b1, b2, eps, bc1, bc2);
    auto adam_one = [&](double& w_, float& m_, float& v_, G g_, double, double, double, double, double,
                        double) -> double {
        if constexpr (sizeof(G) == 4) return adam_f32(w_, m_, v_, g_, cf);
        else return adam_f64(w_, m_, v_, g_, lr, b1, b2, eps, bc1, bc2);
    };
    const uint64_t n4 = n / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        double4 wv = reinterpret_cast<double4*>(w)[i];
        float4 mv = reinterpret_cast<float4*>(m)[i];
        float4 vv = reinterpret_cast<float4*>(v)[i];
        G gv[4];
        if constexpr (sizeof(G) == 4) {
            const float4 t = reinterpret_cast<float4*>(g)[i];
            gv[0] = t.x; gv[1] = t.y; gv[2] = t.z; gv[3] = t.w;
        } else {
            const double4 t = reinterpret_cast<double4*>(g)[i];
            gv[0] = t.x; gv[1] = t.y; gv[2] = t.z; gv[3] = t.w;
        }
        acc += adam_one(wv.x, mv.x, vv.x, gv[0], lr, b1, b2, eps, bc1, bc2);
        acc += adam_one(wv.y, mv.y, vv.y, gv[1], lr, b1, b2, eps, bc1, bc2);
        acc += adam_one(wv.z, mv.z, vv.z, gv[2], lr, b1, b2, eps, bc1, bc2);
        acc += adam_one(wv.w, mv.w, vv.w, gv[3], lr, b1, b2, eps, bc1, bc2);
        reinterpret_cast<double4*>(w_o)[i] = wv;
        reinterpret_cast<float4*>(m_o)[i] = mv;
        reinterpret_cast<float4*>(v_o)[i] = vv;
        if (w16) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(static_cast<float>(wv.x), static_cast<float>(wv.y));
            __nv_bfloat162 hi = __floats2bfloat162_rn(static_cast<float>(wv.z), static_cast<float>(wv.w));
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            reinterpret_cast<uint2*>(w16)[i] = pk;
            if (cm) {
                const float2 a = __bfloat1622float2(lo), b = __bfloat1622float2(hi);
                cmx[0] = fmaxf(cmx[0], a.x);
                cmx[1] = fmaxf(cmx[1], a.y);
                cmx[2] = fmaxf(cmx[2], b.x);
                cmx[3] = fmaxf(cmx[3], b.y);
            }
        }
        if (zero_grad) {
            if constexpr (sizeof(G) == 4) reinterpret_cast<float4*>(g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            else reinterpret_cast<double4*>(g)[i] = make_double4(0.0, 0.0, 0.0, 0.0);
        }
    }
    // scalar tail
    const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid < n - n4 * 4) {
        const uint64_t i = n4 * 4 + gid;
        double wi = w[i];
        float mi = m[i], vi = v[i];
        acc += adam_one(wi, mi, vi, g[i], lr, b1, b2, eps, bc1, bc2);
        w_o[i] = wi;
        m_o[i] = mi;
        v_o[i] = vi;
        if (w16) w16[i] = __float2bfloat16_rn(static_cast<float>(wi));
        if (zero_grad) g[i] = G(0);
    }
    if (cm) {
        const uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        if (i0 < n4) {
            const uint64_t c0 = (4 * i0) % D;
#pragma unroll
            for (int j = 0; j < 4; ++j) atomicMax(cm + c0 + j, fkey(cmx[j]));
        }
    }
    if (gsq) {
        const double tot = block_sum(acc, red);
        if (threadIdx.x == 0) atomicAdd(gsq, tot);
    }
}

// Sharded Adam of a DP gang rank over its own rows (n elements from the row
// range's start): g = local partial + the partials the other ranks wrote into
// this rank's receive slots during their last GEMM2; the new bf16 shadow rows
// go to the local W16 and, over NVLink, to every other rank's W16 (the
// all-gather fused into the optimizer).
__global__ void __launch_bounds__(256) adam_shard_kernel(double* __restrict__ w, float* __restrict__ m,
                                                         float* __restrict__ v, const float* __restrict__ g,
                                                         const float* __restrict__ recv, int nslots,
                                                         uint64_t slot_stride, __nv_bfloat16* __restrict__ w16,
                                                         ShardPeers peers, uint64_t n, double lr, double b1,
                                                         double b2, double eps, double bc1, double bc2,
                                                         double* gsq, int* __restrict__ cm, uint64_t D) {
    __shared__ double red[8];
    double acc = 0.0;
    float cmx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // partial colmax of this rank's rows
    const AdamF cf(lr, b1, b2, eps, bc1, bc2);
    auto adam_one = [&](double& w_, float& m_, float& v_, float g_, double, double, double, double, double,
                        double) -> double { return adam_f32(w_, m_, v_, g_, cf); };
    const uint64_t n4 = n / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        double4 wv = reinterpret_cast<double4*>(w)[i];
        float4 mv = reinterpret_cast<float4*>(m)[i];
        float4 vv = reinterpret_cast<float4*>(v)[i];
        float4 gv = reinterpret_cast<const float4*>(g)[i];
        for (int s = 0; s < nslots; ++s) {
            const float4 r = reinterpret_cast<const float4*>(recv + s * slot_stride)[i];
            gv.x += r.x;
            gv.y += r.y;
            gv.z += r.z;
            gv.w += r.w;
        }
        acc += adam_one(wv.x, mv.x, vv.x, gv.x, lr, b1, b2, eps, bc1, bc2);
        acc += adam_one(wv.y, mv.y, vv.y, gv.y, lr, b1, b2, eps, bc1, bc2);
        acc += adam_one(wv.z, mv.z, vv.z, gv.z, lr, b1, b2, eps, bc1, bc2);
        acc += adam_one(wv.w, mv.w, vv.w, gv.w, lr, b1, b2, eps, bc1, bc2);
        reinterpret_cast<double4*>(w)[i] = wv;
        reinterpret_cast<float4*>(m)[i] = mv;
        reinterpret_cast<float4*>(v)[i] = vv;
        __nv_bfloat162 lo = __floats2bfloat162_rn(static_cast<float>(wv.x), static_cast<float>(wv.y));
        __nv_bfloat162 hi = __floats2bfloat162_rn(static_cast<float>(wv.z), static_cast<float>(wv.w));
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(w16)[i] = pk;
        for (int p = 0; p < peers.n; ++p) reinterpret_cast<uint2*>(peers.w16[p])[i] = pk;
        if (cm) {
            const float2 a = __bfloat1622float2(lo), b = __bfloat1622float2(hi);
            cmx[0] = fmaxf(cmx[0], a.x);
            cmx[1] = fmaxf(cmx[1], a.y);
            cmx[2] = fmaxf(cmx[2], b.x);
            cmx[3] = fmaxf(cmx[3], b.y);
        }
    }
    if (cm) {
        const uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        if (i0 < n4) {
            const uint64_t c0 = (4 * i0) % D;
#pragma unroll
            for (int j = 0; j < 4; ++j) atomicMax(cm + c0 + j, fkey(cmx[j]));
        }
    }
    const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid < n - n4 * 4) {
        const uint64_t i = n4 * 4 + gid;
        float gi = g[i];
        for (int s = 0; s < nslots; ++s) gi += recv[s * slot_stride + i];
        acc += adam_one(w[i], m[i], v[i], gi, lr, b1, b2, eps, bc1, bc2);
        const __nv_bfloat16 b = __float2bfloat16_rn(static_cast<float>(w[i]));
        w16[i] = b;
        for (int p = 0; p < peers.n; ++p) peers.w16[p][i] = b;
    }
    if (gsq) {
        const double tot = block_sum(acc, red);
        if (threadIdx.x == 0) atomicAdd(gsq, tot);
    }
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
                          int64_t Mpad, int64_t global_batch, uint64_t D, RowBuffers rows, __nv_bfloat16* phic,
                          __nv_bfloat16* phict, int clear_old, const int* colmax, cudaStream_t s) {
    if (Mpad == 0) return cudaSuccess;
    if (n_samples > kMaxSamplesSmem) return cudaErrorInvalidValue;
    const int blocks = static_cast<int>((Mpad + 255) / 256);
    gather_kernel<<<blocks, 256, 0, s>>>(arena, sd, n_samples, row_lo, M, Mpad, global_batch, D, rows, phic, phict,
                                         clear_old, colmax);
    return cudaGetLastError();
}

cudaError_t launch_colmax(const __nv_bfloat16* w16, int64_t V, int64_t D, int* keys, int num_sms, cudaStream_t s) {
    if (V == 0 || D == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(keys, 0x80, static_cast<size_t>(D) * sizeof(int), s);  // key < any finite
    if (e != cudaSuccess) return e;
    const unsigned gx = static_cast<unsigned>((D + 2047) / 2048);
    int64_t gy = static_cast<int64_t>(num_sms) * 8 / gx;
    gy = gy < 1 ? 1 : (gy > V ? V : gy);
    colmax_kernel<<<dim3(gx, static_cast<unsigned>(gy)), 256, 0, s>>>(w16, V, D, keys);
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

namespace {
__global__ void __launch_bounds__(1024) klist_kernel(const int4* __restrict__ feat4, int64_t M, int32_t* __restrict__ klist,
                                                     int64_t ld, int32_t* __restrict__ iters, int32_t zero_row) {
    __shared__ int wsum[32];
    __shared__ int tot_s;
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t* out = klist + static_cast<size_t>(b) * ld;
    int base = 0;
    for (int64_t r0 = 0; r0 < M; r0 += 1024) {
        const int64_t r = r0 + threadIdx.x;
        bool hit = false;
        if (r < M) {
            const int4 q = __ldg(feat4 + r);
            hit = (q.x >= 0 && (q.x >> 8) == b) || (q.y >= 0 && (q.y >> 8) == b) ||
                  (q.z >= 0 && (q.z >> 8) == b) || (q.w >= 0 && (q.w >> 8) == b);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
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
            if (lane == 31) tot_s = inc;
        }
        __syncthreads();
        if (hit) out[base + wsum[wid] + pre] = static_cast<int32_t>(r);
        base += tot_s;
        __syncthreads();
    }
    const int padded = base < 64 ? 64 : (base + 63) / 64 * 64;
    for (int i = base + static_cast<int>(threadIdx.x); i < padded; i += blockDim.x) out[i] = zero_row;
    if (threadIdx.x == 0) iters[b] = padded / 64;
}
}  // namespace

cudaError_t launch_klist(const int4* feat4, int64_t M, int nblk, int32_t* klist, int64_t ld, int32_t* iters,
                         int32_t zero_row, cudaStream_t s) {
    if (nblk <= 0) return cudaSuccess;
    klist_kernel<<<nblk, 1024, 0, s>>>(feat4, M, klist, ld, iters, zero_row);
    return cudaGetLastError();
}

namespace {
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

__device__ __forceinline__ bool touches(int4 q, int b) {
    return (q.x >= 0 && (q.x >> 8) == b) || (q.y >= 0 && (q.y >> 8) == b) || (q.z >= 0 && (q.z >> 8) == b) ||
           (q.w >= 0 && (q.w >> 8) == b);
}

// grid (nblk, nchunk): CTA (b, c) counts the rows of chunk c (1024 rows) touching
// block b; CTA (b, 0) also resets slot4 for its share of rows
__global__ void __launch_bounds__(1024) kslot_count_kernel(const int4* __restrict__ feat4, int64_t M,
                                                           int32_t* __restrict__ ccount, int4* __restrict__ slot4) {
    __shared__ int wsum[33];
    const int b = blockIdx.x, c = blockIdx.y;
    const int64_t r = static_cast<int64_t>(c) * 1024 + threadIdx.x;
    const bool hit = r < M && touches(__ldg(feat4 + r), b);
    int tot;
    block_rank(hit, wsum, &tot);
    if (threadIdx.x == 0) ccount[static_cast<size_t>(b) * gridDim.y + c] = tot;
    if (b == 0 && r < M) slot4[r] = make_int4(-1, -1, -1, -1);
}

// grid (nblk, nchunk): segment offsets from the chunk counts (block-major), ranks
// within the chunk, slot / B' writes; the segment's padding rows of A' are zeroed
// by the block's CTAs together
__global__ void __launch_bounds__(1024) kslot_place_kernel(const int4* __restrict__ feat4,
                                                           const uint32_t* __restrict__ cnt4, int64_t M,
                                                           const int32_t* __restrict__ ccount,
                                                           int32_t* __restrict__ kseg_off,
                                                           int32_t* __restrict__ kiters, int4* __restrict__ slot4,
                                                           __nv_bfloat16* __restrict__ aseg, int64_t ld_a,
                                                           int64_t ncols_a, __nv_bfloat16* __restrict__ bseg,
                                                           unsigned long long* rows_acc, int32_t* __restrict__ seg_tok,
                                                           int32_t zero_row) {
    __shared__ int wsum[33];
    __shared__ int off_s, base_s, len_s;
    const int b = blockIdx.x, c = blockIdx.y, nch = gridDim.y;
    if (threadIdx.x < 32) {
        // segment offset: padded lengths of blocks < b; base: rows of chunks < c in block b
        int off = 0;
        // per-block totals, lane-parallel over chunks
        for (int bb = 0; bb <= b; ++bb) {
            int t = 0;
            for (int i = static_cast<int>(threadIdx.x); i < nch; i += 32) t += ccount[static_cast<size_t>(bb) * nch + i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (bb < b) off += t < 64 ? 64 : (t + 63) / 64 * 64;
            else if (threadIdx.x == 0) len_s = t;
        }
        int base = 0;
        for (int i = static_cast<int>(threadIdx.x); i < c; i += 32) base += ccount[static_cast<size_t>(b) * nch + i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) base += __shfl_xor_sync(0xffffffffu, base, o);
        if (threadIdx.x == 0) {
            off_s = off;
            base_s = base;
        }
    }
    __syncthreads();
    const int off = off_s, len = len_s;
    const int padded = len < 64 ? 64 : (len + 63) / 64 * 64;
    if (c == 0 && threadIdx.x == 0) {
        kseg_off[b] = off;
        kiters[b] = padded / 64;
        if (rows_acc) atomicAdd(rows_acc, static_cast<unsigned long long>(padded));
    }
    const int64_t r = static_cast<int64_t>(c) * 1024 + threadIdx.x;
    int4 q = make_int4(-1, -1, -1, -1);
    if (r < M) q = __ldg(feat4 + r);
    const bool hit = r < M && touches(q, b);
    int tot;
    const int rk = block_rank(hit, wsum, &tot);
    if (hit) {
        const int slot = off + base_s + rk;
        if (seg_tok) seg_tok[slot] = static_cast<int32_t>(r);
        const uint32_t c4 = __ldg(cnt4 + r);
        int* sl = reinterpret_cast<int*>(slot4 + r);
        const int f[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (f[j] >= 0 && (f[j] >> 8) == b) {
                sl[j] = slot;
                bseg[static_cast<size_t>(slot) * 256 + (f[j] & 255)] =
                    __float2bfloat16_rn(static_cast<float>((c4 >> (8 * j)) & 0xFFu));
            }
        }
    }
    // zero the segment's padding rows of A' (B' is zero on entry), split over the chunks;
    // with a software-gathered A the padding slots point at the zero row instead
    const int64_t npad = padded - len;
    if (seg_tok) {
        for (int64_t i = static_cast<int64_t>(c) * blockDim.x + threadIdx.x; i < npad;
             i += static_cast<int64_t>(nch) * blockDim.x)
            seg_tok[off + len + i] = zero_row;
    }
    if (!aseg) return;
    const int64_t cols8 = ncols_a / 8;  // ld_a and ncols_a are multiples of 8
    for (int64_t i = static_cast<int64_t>(c) * blockDim.x + threadIdx.x; i < npad * cols8;
         i += static_cast<int64_t>(nch) * blockDim.x) {
        const int64_t rr = off + len + i / cols8, cc = (i % cols8) * 8;
        *reinterpret_cast<uint4*>(aseg + rr * ld_a + cc) = make_uint4(0u, 0u, 0u, 0u);
    }
}
}  // namespace

cudaError_t launch_kslots(const int4* feat4, const uint32_t* cnt4, int64_t M, int nblk, int32_t* kcount,
                          int32_t* kseg_off, int32_t* kiters, int4* slot4, __nv_bfloat16* aseg, int64_t ld_a,
                          int64_t ncols_a, __nv_bfloat16* bseg, unsigned long long* rows_acc, int32_t* seg_tok,
                          int32_t zero_row, cudaStream_t s) {
    if (nblk <= 0) return cudaSuccess;
    const unsigned nch = static_cast<unsigned>(M > 0 ? (M + 1023) / 1024 : 1);
    kslot_count_kernel<<<dim3(nblk, nch), 1024, 0, s>>>(feat4, M, kcount, slot4);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    kslot_place_kernel<<<dim3(nblk, nch), 1024, 0, s>>>(feat4, cnt4, M, kcount, kseg_off, kiters, slot4, aseg, ld_a,
                                                        ncols_a, bseg, rows_acc, seg_tok, zero_row);
    return cudaGetLastError();
}

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

cudaError_t launch_lse(const float* zact, const float2* stats, int stats_ld, int64_t M, int64_t Mpad, int64_t V,
                       const SampleDesc* sd, int64_t global_batch, RowBuffers rows, const float* old_logp,
                       float clip_eps, double* loss_acc, __nv_bfloat16* pexp_t, __nv_bfloat16* phict,
                       int64_t ldt, cudaStream_t s, int rowmajor, int64_t ld_phi) {
    LseArgs L{zact, stats, stats_ld, M, Mpad, V, sd, global_batch, rows, old_logp, clip_eps,
              loss_acc, pexp_t != nullptr, pexp_t, phict, ldt};
    L.rowmajor = rowmajor;
    L.ld_phi = ld_phi;
    return launch_lse(L, s);
}

cudaError_t launch_lse(const LseArgs& L, cudaStream_t s) {
    if (L.Mpad == 0) return cudaSuccess;
    int64_t blocks = (L.Mpad * 8 + 255) / 256;  // 4 rows per warp
    if (blocks > 148 * 4) blocks = 148 * 4;     // persistent warps: 4 resident 256-thread blocks per SM
    lse_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_softmax_grad(const CUtensorMap& tmP, const CUtensorMap& tmGt, const float2* stats, int stats_ld,
                                int64_t Mpad, int64_t V, RowBuffers rows, cudaStream_t s, int part_cols) {
    if (Mpad == 0) return cudaSuccess;
    const size_t smem = 1024 + kSgPBytes + kSgGBytes + 16 + kSgRows * 12;
    cudaFuncSetAttribute(softmax_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dim3 grid(static_cast<unsigned>((V + kSgCols - 1) / kSgCols), static_cast<unsigned>(Mpad / kSgRows));
    softmax_grad_kernel<<<grid, 256, smem, s>>>(tmP, tmGt, stats, stats_ld, rows, part_cols);
    return cudaGetLastError();
}

template <typename G>
cudaError_t launch_adam(double* w, float* m, float* v, G* g, __nv_bfloat16* w16, uint64_t n, double lr, double b1,
                        double b2, double eps, double bc1, double bc2, int zero_grad, double* gsq, int num_sms,
                        cudaStream_t s, int* colmax, uint64_t D, bool* colmax_done, const AdamDst* dst) {
    if (colmax_done) *colmax_done = false;
    if (n == 0) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g)) & 31) return cudaErrorMisalignedAddress;
    const uint64_t want = (n / 4 + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(num_sms) * 8;
    uint64_t blocks = want < 1 ? 1 : (want > cap ? cap : want);
    int* cm = nullptr;
    if (colmax && w16 && D % 4 == 0 && n % D == 0) {
        // fixed columns per thread: one iteration per thread, or a grid stride that is a
        // multiple of D (blocks * 1024 elements)
        if (want > blocks) {
            uint64_t q = D, r = 1024;  // blocks must be a multiple of D / gcd(D, 1024)
            while (r) { const uint64_t t = q % r; q = r; r = t; }
            const uint64_t mult = D / q;
            blocks = blocks / mult * mult;
        }
        if (blocks > 0) {
            cm = colmax;
            cudaError_t e = cudaMemsetAsync(colmax, 0x80, D * sizeof(int), s);
            if (e != cudaSuccess) return e;
        } else {
            blocks = want < cap ? want : cap;
        }
    }
    if (dst && (reinterpret_cast<uintptr_t>(dst->w) & 31)) return cudaErrorMisalignedAddress;
    adam_kernel<G><<<static_cast<int>(blocks), 256, 0, s>>>(w, m, v, g, w16, n, lr, b1, b2, eps, bc1, bc2, zero_grad,
                                                            gsq, cm, D, dst ? dst->w : nullptr,
                                                            dst ? dst->m : nullptr, dst ? dst->v : nullptr);
    if (colmax_done) *colmax_done = cm != nullptr;
    return cudaGetLastError();
}
template cudaError_t launch_adam<float>(double*, float*, float*, float*, __nv_bfloat16*, uint64_t, double, double,
                                        double, double, double, double, int, double*, int, cudaStream_t, int*,
                                        uint64_t, bool*, const AdamDst*);
template cudaError_t launch_adam<double>(double*, float*, float*, double*, __nv_bfloat16*, uint64_t, double,
                                         double, double, double, double, double, int, double*, int, cudaStream_t,
                                         int*, uint64_t, bool*, const AdamDst*);

cudaError_t launch_adam_shard(double* w, float* m, float* v, const float* g, const float* recv, int nslots,
                              uint64_t slot_stride, __nv_bfloat16* w16, ShardPeers peers, uint64_t n, double lr,
                              double b1, double b2, double eps, double bc1, double bc2, double* gsq, int num_sms,
                              cudaStream_t s, int* colmax, uint64_t D, bool* colmax_done) {
    if (colmax_done) *colmax_done = false;
    if (n == 0) return cudaSuccess;
    const uint64_t want = (n / 4 + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(num_sms) * 8;
    uint64_t blocks = want < 1 ? 1 : (want > cap ? cap : want);
    int* cm = nullptr;
    if (colmax && D % 4 == 0 && n % D == 0) {
        // partial colmax of this shard (fixed columns per thread, as in launch_adam)
        if (want > blocks) {
            uint64_t q = D, r = 1024;
            while (r) { const uint64_t t = q % r; q = r; r = t; }
            const uint64_t mult = D / q;
            blocks = blocks / mult * mult;
        }
        if (blocks > 0) {
            cm = colmax;
            cudaError_t e = cudaMemsetAsync(colmax, 0x80, D * sizeof(int), s);
            if (e != cudaSuccess) return e;
        } else {
            blocks = want < cap ? want : cap;
        }
    }
    adam_shard_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(w, m, v, g, recv, nslots, slot_stride, w16, peers, n,
                                                               lr, b1, b2, eps, bc1, bc2, gsq, cm, D);
    if (colmax_done) *colmax_done = cm != nullptr;
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

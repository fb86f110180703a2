// fm_lse.cuh — the per-row softmax normaliser of the micro-batch loss
// (policy.hpp:62-75, training.hpp:386-394), shared by the standalone K-lse
// kernel (k_path.cu) and GEMM1's fused last-tile epilogue (k_gemm_tc.cu).
//
// A warp processes four rows with eight lanes per row: the lanes combine the
// row's per-256-column (max, sum exp) partials into lse, compute the
// taken-token log-prob from the fp32 logit GEMM1 captured, the effective row
// coefficient (optional PPO clip), and on the loss-fold path write the
// taken-token delta into p~^T and the row factor -c/s into Phic^T's <= 4
// count entries (see DESIGN.md §4 "Loss fold").
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "fm_kernels.h"

namespace fm {

// Rows r0 .. r0+3 (r0 a multiple of 4, rows >= Mpad skipped).  Returns the
// objective contribution held by lane (row, sl == 0); 0 elsewhere.
__device__ __forceinline__ double lse_row_quad(const LseArgs& L, int64_t r0) {
    constexpr int kLpr = 8;
    const int lane = threadIdx.x & 31;
    const int sub = lane / kLpr, sl = lane % kLpr;
    const int64_t r = r0 + sub;
    const bool live = r < L.M;  // rows in [M, Mpad) are padding; r >= Mpad does not exist
    const RowBuffers& rows = L.rows;
    int a = -1;
    float za = 0.f, c0 = 0.f, olp = 0.f;
    double adv = 0.0, loss = 0.0;
    int4 f4 = make_int4(-1, -1, -1, -1);
    uint32_t c4 = 0;
    float m = -INFINITY, s = 0.f;
    if (live) {
        a = rows.action[r];
        za = L.zact[r];
        c0 = rows.coef[r];
        adv = L.sd[rows.sample[r]].adv;
        if (L.old_logp) olp = L.old_logp[r];
        if (L.fold) {
            f4 = rows.feat4[r];
            c4 = rows.cnt4[r];
        }
        // all 16 partials a lane needs per round are issued before any math
        const float2* st = L.stats + static_cast<size_t>(r) * L.stats_ld;
        for (int base = 0; base < L.stats_ld; base += kLpr * 16) {
            float2 p[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int j = base + sl + kLpr * k;
                p[k] = j < L.stats_ld ? st[j] : make_float2(-INFINITY, 0.f);
            }
            float lm = p[0].x;
#pragma unroll
            for (int k = 1; k < 16; ++k) lm = fmaxf(lm, p[k].x);
            const float nm = fmaxf(m, lm);
            if (nm != -INFINITY) {
                float ls = 0.f;
#pragma unroll
                for (int k = 0; k < 16; ++k) ls += p[k].x == -INFINITY ? 0.f : p[k].y * __expf(p[k].x - nm);
                s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + ls;
                m = nm;
            }
        }
    }
#pragma unroll
    for (int o = kLpr / 2; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, m, o);
        const float os = __shfl_xor_sync(0xffffffffu, s, o);
        const float nm = fmaxf(m, om);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
        m = nm;
    }
    if (r >= L.Mpad) return 0.0;
    if (!live) {
        if (sl == 0) {
            rows.lse[r] = 0.f;
            rows.logp[r] = 0.f;
            rows.coef_eff[r] = 0.f;
        }
        return 0.0;
    }
    // the row's 8 lanes hold (m, s); the epilogue is computed redundantly by them
    // and its scattered stores are spread over lanes 0-4 of the row
    const float lse = m + __logf(s);
    const bool valid = a >= 0 && a < L.V;
    const float lp = valid ? za - lse : 0.f;  // policy.hpp:72-75, fp32 logit
    float ce = c0;
    if (L.old_logp && L.clip_eps > 0.f) {
        // PPO clipped-ratio surrogate min(rho*A, clip(rho,1-e,1+e)*A): the
        // gradient flows (scaled by rho) only through the unclipped branch.
        const float rho = __expf(lp - olp);
        const bool active = adv >= 0.0 ? rho <= 1.f + L.clip_eps : rho >= 1.f - L.clip_eps;
        ce = active ? ce * rho : 0.f;
    }
    if (sl == 0) {
        rows.lse[r] = lse;
        rows.logp[r] = lp;
        rows.coef_eff[r] = ce;
        loss = valid ? -(adv / static_cast<double>(L.G)) * static_cast<double>(lp) : 0.0;
        if (L.fold && (!(s >= 1e-30f) || !isfinite(s)))
            loss = __longlong_as_double(0x7ff8000000000000ll);  // range guard: NaN loss, never silent
    }
    if (L.fold) {
        // Every tile used the row's offset bound m (K-gather), so
        //   G[t][v] = c (delta(v,a) - p~[t][v] / s),  s = sum_v p~ = exp(lse - m).
        // The per-row factor sig = -c / s goes into GEMM2's B operand
        // (Phic^T's <= 4 count entries of column t), the delta term into A:
        //   A[a][t] = p~_a - s   =>   sig * A = -c (p - delta) = G.
        // an action outside [0, V) never matches a vocab row (policy.hpp:84-85): the
        // row still gets -c p, just no delta term
        const float sig = ce != 0.f ? __fdividef(-ce, s) : 0.f;
        if (L.rowmajor == 3) {
            // segments with a software-gathered A: p~ stays row-major (delta once per
            // row, lane 4), the row factor goes into B' through the slot table
            if (sl == 4 && sig != 0.f && valid)
                L.pexp_t[static_cast<size_t>(r) * L.ldt + a] = __float2bfloat16_rn(__expf(za - m) - s);
            if (sl < 4) {
                const int4 s4 = L.slot4[r];
                const int sj = sl == 0 ? s4.x : sl == 1 ? s4.y : sl == 2 ? s4.z : s4.w;
                const int f = sl == 0 ? f4.x : sl == 1 ? f4.y : sl == 2 ? f4.z : f4.w;
                if (f >= 0 && sj >= 0)
                    L.bseg[static_cast<size_t>(sj) * 256 + (f & 255)] =
                        __float2bfloat16_rn(sig * static_cast<float>((c4 >> (8 * sl)) & 0xFFu));
            }
            return loss;
        }
        if (L.rowmajor == 2) {
            // token-slot segments: lane j (< 4) owns feature j — the delta goes into its
            // block's A' row (once per distinct slot), the row factor into B'
            if (sl < 4 && live) {
                const int4 s4 = L.slot4[r];
                const int sj = sl == 0 ? s4.x : sl == 1 ? s4.y : sl == 2 ? s4.z : s4.w;
                const int f = sl == 0 ? f4.x : sl == 1 ? f4.y : sl == 2 ? f4.z : f4.w;
                bool first = sj >= 0;
                if (sl > 0 && s4.x == sj) first = false;
                if (sl > 1 && s4.y == sj) first = false;
                if (sl > 2 && s4.z == sj) first = false;
                if (first && sig != 0.f && valid)
                    L.pexp_t[static_cast<size_t>(sj) * L.ldt + a] = __float2bfloat16_rn(__expf(za - m) - s);
                if (f >= 0)
                    L.bseg[static_cast<size_t>(sj) * 256 + (f & 255)] =
                        __float2bfloat16_rn(sig * static_cast<float>((c4 >> (8 * sl)) & 0xFFu));
            }
            return loss;
        }
        if (sl == 4 && sig != 0.f && valid) {
            const size_t i = L.rowmajor ? static_cast<size_t>(r) * L.ldt + a : static_cast<size_t>(a) * L.ldt + r;
            L.pexp_t[i] = __float2bfloat16_rn(__expf(za - m) - s);
        }
        if (sl < 4) {
            const int f = sl == 0 ? f4.x : sl == 1 ? f4.y : sl == 2 ? f4.z : f4.w;
            if (f >= 0) {
                const size_t i =
                    L.rowmajor ? static_cast<size_t>(r) * L.ld_phi + f : static_cast<size_t>(f) * L.ldt + r;
                L.phict[i] = __float2bfloat16_rn(sig * static_cast<float>((c4 >> (8 * sl)) & 0xFFu));
            }
        }
    }
    return loss;
}

}  // namespace fm

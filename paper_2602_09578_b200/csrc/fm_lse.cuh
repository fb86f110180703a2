// fm_lse.cuh — the per-row softmax normaliser of the micro-batch loss
// (policy.hpp:62-75, training.hpp:386-394) run by K-lse (k_path.cu).
//
// A warp processes four rows with eight lanes per row: the lanes combine the
// row's per-256-column (max, sum exp) partials from K-stats into lse, compute
// the taken-token log-prob from the fp32 logit K-stats captured and the
// effective row coefficient (optional PPO clip) that K-band scales the
// row's log-softmax gradient by.
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
    float m = -INFINITY, s = 0.f;
    if (live) {
        a = rows.action[r];
        za = L.zact[r];
        c0 = rows.coef[r];
        adv = L.sd[rows.sample[r]].adv;
        if (L.old_logp) olp = L.old_logp[L.row_lo + r];  // indexed by the micro-batch's packed row
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
    }
    return loss;
}

}  // namespace fm

// adam_probe.cu — K-adam tile-shape / cache-hint probe (a measurement tool, not
// part of the library).  Build on the GPU box:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2602_09578_b200/csrc \
//        tools/adam_probe.cu -o /tmp/adam_probe -lcuda && /tmp/adam_probe
// Times the library's launch_adam (k_path.cu, included) against variants with
// taller tiles (64 vocabulary rows: 128-byte W16^T segments) and streaming
// cache hints, at C2's P = 32000 x 4096, plus a plain device copy as the
// bandwidth reference.
#include "k_path.cu"

#include <cstdio>
#include <vector>

using namespace fm;

namespace probe {

template <int kRows, bool kHints>
__global__ void __launch_bounds__(256) adam_v(double* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
                                              const float* __restrict__ g, uint64_t V, uint64_t D,
                                              __nv_bfloat16* __restrict__ w16t, uint64_t ldw, double lr, double b1,
                                              double b2, double eps, double bc1, double bc2) {
    constexpr int TV = 32 * kRows, TD = 64, PITCH = TV + 8;
    __shared__ __align__(16) __nv_bfloat16 tsh[TD][PITCH];
    const AdamF cf(lr, b1, b2, eps, bc1, bc2);
    const uint64_t tv_n = (V + TV - 1) / TV, td_n = (D + TD - 1) / TD;
    const int tr = threadIdx.x >> 3, tc = (threadIdx.x & 7) * 8;
    for (uint64_t t = blockIdx.x; t < tv_n * td_n; t += gridDim.x) {
        const uint64_t tv = t / td_n, td = t % td_n;
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
            const uint64_t vr = tv * TV + tr + 32 * k, d0 = td * TD + tc;
            float wf[8] = {};
            if (vr < V && d0 + 8 <= D) {
                const uint64_t i0 = vr * D + d0;
                double wv[8];
                float mv[8], vv[8], gv[8];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double2 x = kHints ? __ldcs(reinterpret_cast<const double2*>(w + i0) + q)
                                             : reinterpret_cast<const double2*>(w + i0)[q];
                    wv[2 * q] = x.x;
                    wv[2 * q + 1] = x.y;
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const float4 a = kHints ? __ldcs(reinterpret_cast<const float4*>(m + i0) + q)
                                            : reinterpret_cast<const float4*>(m + i0)[q];
                    const float4 b = kHints ? __ldcs(reinterpret_cast<const float4*>(v + i0) + q)
                                            : reinterpret_cast<const float4*>(v + i0)[q];
                    const float4 c = kHints ? __ldcs(reinterpret_cast<const float4*>(g + i0) + q)
                                            : reinterpret_cast<const float4*>(g + i0)[q];
                    mv[4 * q] = a.x; mv[4 * q + 1] = a.y; mv[4 * q + 2] = a.z; mv[4 * q + 3] = a.w;
                    vv[4 * q] = b.x; vv[4 * q + 1] = b.y; vv[4 * q + 2] = b.z; vv[4 * q + 3] = b.w;
                    gv[4 * q] = c.x; gv[4 * q + 1] = c.y; gv[4 * q + 2] = c.z; gv[4 * q + 3] = c.w;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    adam_f32(wv[j], mv[j], vv[j], gv[j], cf);
                    wf[j] = static_cast<float>(wv[j]);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double2 x = make_double2(wv[2 * q], wv[2 * q + 1]);
                    if (kHints) __stcs(reinterpret_cast<double2*>(w + i0) + q, x);
                    else reinterpret_cast<double2*>(w + i0)[q] = x;
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const float4 a = make_float4(mv[4 * q], mv[4 * q + 1], mv[4 * q + 2], mv[4 * q + 3]);
                    const float4 b = make_float4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
                    if (kHints) {
                        __stcs(reinterpret_cast<float4*>(m + i0) + q, a);
                        __stcs(reinterpret_cast<float4*>(v + i0) + q, b);
                    } else {
                        reinterpret_cast<float4*>(m + i0)[q] = a;
                        reinterpret_cast<float4*>(v + i0)[q] = b;
                    }
                }
            }
            if (w16t) {
#pragma unroll
                for (int j = 0; j < 8; ++j) tsh[tc + j][tr + 32 * k] = __float2bfloat16_rn(wf[j]);
            }
        }
        if (w16t) {
            __syncthreads();
            // thread -> (column d, 8 rows); TV / 8 threads per column
            constexpr int TPC = TV / 8;
            for (int e = threadIdx.x; e < TD * TPC; e += 256) {
                const int dl = e / TPC, rc = (e % TPC) * 8;
                const uint64_t d = td * TD + dl, vb = tv * TV + rc;
                if (d < D && vb + 8 <= V) {
                    const uint4 val = *reinterpret_cast<const uint4*>(&tsh[dl][rc]);
                    if (kHints) __stcs(reinterpret_cast<uint4*>(w16t + d * ldw + vb), val);
                    else *reinterpret_cast<uint4*>(w16t + d * ldw + vb) = val;
                }
            }
            __syncthreads();
        }
    }
}

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

}  // namespace probe

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                              \
        }                                                                          \
    } while (0)

int main() {
    const uint64_t V = 32000, D = 4096, P = V * D, ldw = V;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* w;
    float *m, *v, *g;
    __nv_bfloat16* w16;
    char *flush, *ca, *cb;
    CK(cudaMalloc(&w, P * 8));
    CK(cudaMalloc(&m, P * 4));
    CK(cudaMalloc(&v, P * 4));
    CK(cudaMalloc(&g, P * 4));
    CK(cudaMalloc(&w16, D * ldw * 2));
    double* gsq;
    CK(cudaMalloc(&gsq, 8));
    CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMalloc(&ca, 1ull << 30));
    CK(cudaMalloc(&cb, 1ull << 30));
    CK(cudaMemset(w, 0, P * 8));
    CK(cudaMemset(m, 0, P * 4));
    CK(cudaMemset(v, 0, P * 4));
    CK(cudaMemset(g, 0, P * 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, double bytes, auto&& fn) {
        float best = 1e30f, tot = 0.f;
        for (int it = 0; it < 12; ++it) {
            cudaMemsetAsync(flush, it, 512 << 20);
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 2) {
                best = ms < best ? ms : best;
                tot += ms;
            }
        }
        const cudaError_t err = cudaGetLastError();
        std::printf("%-34s best %.4f ms avg %.4f ms  %.1f GB/s (best)  %s\n", name, best, tot / 10, bytes / best / 1e6,
                    err == cudaSuccess ? "" : cudaGetErrorString(err));
    };
    const double adam_bytes = 38.0 * P;
    const ShardPeers none{};
    timeit("copy 2 GiB (r+w)", 2.0 * (1ull << 30), [&] {
        probe::copy_k<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(ca), reinterpret_cast<float4*>(cb),
                                        (1ull << 30) / 16);
    });
    timeit("library launch_adam", adam_bytes, [&] {
        launch_adam<float>(w, m, v, g, V, D, 0, V, nullptr, 0, w16, ldw, none, 1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001, 0,
                           gsq, sms, 0, nullptr);
    });
    {
        AdamTileArgs<float> A{w, m, v, g, V, D, 0, V, nullptr, 0, w16, ldw, none, nullptr, nullptr, nullptr,
                              0, gsq, 1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001, AdamF(1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001)};
        const int tiles = static_cast<int>(((V + kTileV - 1) / kTileV) * ((D + kTileD - 1) / kTileD));
        for (int grid : {sms * 8, sms * 32, sms * 64, sms * 128, tiles}) {
            char nm[64];
            std::snprintf(nm, sizeof nm, "library kernel grid=%d", grid);
            timeit(nm, adam_bytes, [&] { adam_tile_kernel<float, true, false><<<grid, 256>>>(A); });
        }
        AdamTileArgs<float> A0 = A;
        A0.gsq = nullptr;
        for (int grid : {sms * 8, sms * 64}) {
            char nm[64];
            std::snprintf(nm, sizeof nm, "library kernel no-gsq grid=%d", grid);
            timeit(nm, adam_bytes, [&] { adam_tile_kernel<float, true, false><<<grid, 256>>>(A0); });
        }
        AdamTileArgs<float> A1 = A0;
        A1.w16t = nullptr;
        timeit("library kernel no-gsq no-w16t (36 B)", 36.0 * P, [&] { adam_tile_kernel<float, true, false><<<sms * 64, 256>>>(A1); });
        for (int grid : {sms * 128, tiles}) {
            char nm[64];
            std::snprintf(nm, sizeof nm, "v32 plain grid=%d", grid);
            timeit(nm, adam_bytes, [&] {
                probe::adam_v<1, false><<<grid, 256>>>(w, m, v, g, V, D, w16, ldw, 1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001);
            });
        }
    }
    for (int mult : {8, 64}) {
        char nm[64];
        std::snprintf(nm, sizeof nm, "v32 plain grid=%dx", mult);
        timeit(nm, adam_bytes, [&] {
            probe::adam_v<1, false><<<sms * mult, 256>>>(w, m, v, g, V, D, w16, ldw, 1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001);
        });
        std::snprintf(nm, sizeof nm, "v32 hints grid=%dx", mult);
        timeit(nm, adam_bytes, [&] {
            probe::adam_v<1, true><<<sms * mult, 256>>>(w, m, v, g, V, D, w16, ldw, 1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001);
        });
        std::snprintf(nm, sizeof nm, "v64 plain grid=%dx", mult);
        timeit(nm, adam_bytes, [&] {
            probe::adam_v<2, false><<<sms * mult, 256>>>(w, m, v, g, V, D, w16, ldw, 1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001);
        });
        std::snprintf(nm, sizeof nm, "v64 hints grid=%dx", mult);
        timeit(nm, adam_bytes, [&] {
            probe::adam_v<2, true><<<sms * mult, 256>>>(w, m, v, g, V, D, w16, ldw, 1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001);
        });
    }
    timeit("v64 hints no-w16t (36 B/param)", 36.0 * P, [&] {
        probe::adam_v<2, true><<<sms * 8, 256>>>(w, m, v, g, V, D, nullptr, ldw, 1e-6, 0.9, 0.999, 1e-8, 0.1, 0.001);
    });
    return 0;
}

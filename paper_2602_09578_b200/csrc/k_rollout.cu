// k_rollout.cu — SURVEY §8f-3 ("next"): rollout-side generation on the GPU.
//
// PolicyModel::generate (policy.hpp:119-130) for a batch of requests, one CTA
// per request, autoregressive over tokens:
//   featurize (policy.hpp:42-51, exact fp64 phi)  ->  z = W * phi (fp64,
//   ascending feature order like the reference's d loop)  ->  softmax
//   (policy.hpp:54-70)  ->  u = Rng(tok_seed).next_unit() (rng.hpp:43-48)  ->
//   first v with u < cumsum(p)[v] (policy.hpp:93-102)  ->  log p[t]
//   (policy.hpp:72-75)  ->  stop at EOS (token 0).
// The per-request splitmix64 stream advances exactly as the reference's
// (one draw per sampled token), so with the same weights and seeds the
// generated responses match the reference token for token (fp64 throughout;
// the only rounding difference is the order of the softmax denominator sum).
#include <cuda_runtime.h>

#include <cstdint>

#include "fm_kernels.h"

namespace fm {
namespace {

__device__ __forceinline__ uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

constexpr int kThreads = 256;

// kTransposed: W is the rollout layout Wt [D][V] (fm_publish dtype 3): the
// per-token reads of a context feature's weights are contiguous over v.
template <bool kTransposed>
__global__ void __launch_bounds__(kThreads) generate_kernel(const double* __restrict__ W, uint64_t V, uint64_t D,
                                                            const int32_t* __restrict__ prompts,
                                                            const int32_t* __restrict__ prompt_off,
                                                            int max_tokens, const uint64_t* __restrict__ seeds,
                                                            double* __restrict__ zbuf, int32_t* __restrict__ out_tok,
                                                            double* __restrict__ out_logp, int32_t* __restrict__ out_len) {
    __shared__ double red[kThreads / 32];
    __shared__ double s_chunk[kThreads];
    __shared__ uint64_t s_f[4];
    __shared__ double s_phi[4];
    __shared__ int s_nf, s_tok, s_ctx[4], s_nctx;
    __shared__ double s_u;
    const int req = blockIdx.x;
    const int tid = threadIdx.x;
    double* z = zbuf + static_cast<size_t>(req) * V;
    uint64_t rng = seeds[req];
    if (tid == 0) {  // context tail = last <= 4 prompt tokens
        const int b = prompt_off[req], e = prompt_off[req + 1];
        const int n = min(e - b, 4);
        for (int j = 0; j < n; ++j) s_ctx[j] = prompts[e - n + j];
        s_nctx = n;
    }
    __syncthreads();
    int len = 0;
    while (len < max_tokens) {
        if (tid == 0) {  // featurize: phi[tok % D] += 1/n, distinct features in ascending order
            const int n = s_nctx;
            const double w = n ? 1.0 / static_cast<double>(n) : 0.0;
            int nf = 0;
            for (int j = 0; j < n; ++j) {
                const uint64_t f = static_cast<uint64_t>(static_cast<int64_t>(s_ctx[j])) % D;
                int k = 0;
                while (k < nf && s_f[k] != f) ++k;
                if (k == nf) {
                    s_f[nf] = f;
                    s_phi[nf] = 0.0;
                    ++nf;
                }
                s_phi[k] = __dadd_rn(s_phi[k], w);
            }
            for (int i = 1; i < nf; ++i)
                for (int k = i; k > 0 && s_f[k - 1] > s_f[k]; --k) {
                    const uint64_t tf = s_f[k]; s_f[k] = s_f[k - 1]; s_f[k - 1] = tf;
                    const double tp = s_phi[k]; s_phi[k] = s_phi[k - 1]; s_phi[k - 1] = tp;
                }
            s_nf = nf;
            s_u = [&] {  // rng.next_unit()
                const uint64_t bits = splitmix(rng) >> 11;
                double u = static_cast<double>(bits) * 0x1.0p-53;
                return u <= 0.0 ? 0x1.0p-53 : u;
            }();
        }
        __syncthreads();
        const int nf = s_nf;
        // logits + running max
        double lmax = -INFINITY;
        for (uint64_t v = tid; v < V; v += kThreads) {
            double s = 0.0;
            for (int k = 0; k < nf; ++k) {
                const double wv = kTransposed ? __ldg(W + s_f[k] * V + v) : W[v * D + s_f[k]];
                s = __dadd_rn(s, __dmul_rn(wv, s_phi[k]));
            }
            z[v] = s;
            lmax = fmax(lmax, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        if ((tid & 31) == 0) red[tid >> 5] = lmax;
        __syncthreads();
        double zmax = red[0];
        for (int i = 1; i < kThreads / 32; ++i) zmax = fmax(zmax, red[i]);
        __syncthreads();
        // exp and the per-thread contiguous chunk sums (chunk = [tid*C, (tid+1)*C))
        const uint64_t C = (V + kThreads - 1) / kThreads;
        const uint64_t b = tid * C, e = b + C < V ? b + C : V;
        double cs = 0.0;
        for (uint64_t v = b; v < e; ++v) {
            const double x = exp(z[v] - zmax);
            z[v] = x;
            cs += x;
        }
        s_chunk[tid] = cs;
        __syncthreads();
        if (tid == 0) {
            double denom = 0.0;
            for (int i = 0; i < kThreads; ++i) denom += s_chunk[i];
            // sample_token: first v with u < acc (policy.hpp:95-101), acc in p units
            const double target = s_u;
            double acc = 0.0;
            int tok = static_cast<int>(V) - 1;
            bool found = false;
            for (int i = 0; i < kThreads && !found; ++i) {
                const uint64_t cb = i * C, ce = cb + C < V ? cb + C : V;
                if (cb >= ce) continue;
                const double next = acc + s_chunk[i] / denom;
                if (!(target < next)) {
                    acc = next;
                    continue;
                }
                for (uint64_t v = cb; v < ce; ++v) {
                    acc += z[v] / denom;
                    if (target < acc) {
                        tok = static_cast<int>(v);
                        found = true;
                        break;
                    }
                }
            }
            out_tok[static_cast<size_t>(req) * max_tokens + len] = tok;
            out_logp[static_cast<size_t>(req) * max_tokens + len] = log(z[tok] / denom);
            s_tok = tok;
            // context tail update
            if (s_nctx < 4) {
                s_ctx[s_nctx++] = tok;
            } else {
                s_ctx[0] = s_ctx[1];
                s_ctx[1] = s_ctx[2];
                s_ctx[2] = s_ctx[3];
                s_ctx[3] = tok;
            }
        }
        __syncthreads();
        ++len;
        if (s_tok == 0) break;  // kEosToken (policy.hpp:15)
    }
    if (tid == 0) out_len[req] = len;
}

}  // namespace

cudaError_t launch_generate(const double* W, bool transposed, uint64_t V, uint64_t D, const int32_t* prompts,
                            const int32_t* prompt_off, int n_req, int max_tokens, const uint64_t* seeds, double* zbuf,
                            int32_t* out_tok, double* out_logp, int32_t* out_len, cudaStream_t s) {
    if (n_req == 0) return cudaSuccess;
    if (transposed)
        generate_kernel<true><<<n_req, kThreads, 0, s>>>(W, V, D, prompts, prompt_off, max_tokens, seeds, zbuf,
                                                         out_tok, out_logp, out_len);
    else
        generate_kernel<false><<<n_req, kThreads, 0, s>>>(W, V, D, prompts, prompt_off, max_tokens, seeds, zbuf,
                                                          out_tok, out_logp, out_len);
    return cudaGetLastError();
}

}  // namespace fm

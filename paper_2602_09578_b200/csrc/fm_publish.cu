// fm_publish.cu — weight publish and rollout sync, the PolicyState wire format, GPU rollout generation.
#include "fm_state.h"

// ===========================================================================
// §8f next rows: weight publish / rollout sync (f1) and the byte-compatible
// PolicyState wire format (f2)
// ===========================================================================

namespace {
__global__ void f64_to_f32_kernel(const double* __restrict__ w, float* __restrict__ o, uint64_t n) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        o[i] = static_cast<float>(w[i]);
}
size_t dtype_bytes(int dt) { return dt == 0 || dt == 3 ? 8 : dt == 1 ? 4 : 2; }

// W [V][D] -> Wt [D][V] through 32 x 32 shared-memory tiles (both sides coalesced)
__global__ void transpose_f64_kernel(const double* __restrict__ w, double* __restrict__ wt, uint64_t V, uint64_t D) {
    __shared__ double tile[32][33];
    const uint64_t d0 = static_cast<uint64_t>(blockIdx.x) * 32, v0 = static_cast<uint64_t>(blockIdx.y) * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const uint64_t v = v0 + r, d = d0 + threadIdx.x;
        if (v < V && d < D) tile[r][threadIdx.x] = w[v * D + d];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const uint64_t d = d0 + r, v = v0 + threadIdx.x;
        if (v < V && d < D) wt[d * V + v] = tile[threadIdx.x][r];
    }
}

void put_u64(std::vector<uint8_t>& v, uint64_t x) {
    const size_t o = v.size();
    v.resize(o + 8);
    std::memcpy(v.data() + o, &x, 8);
}
}  // namespace

extern "C" {

int fm_weights_alloc(fm_ctx* c, uint64_t rows, uint64_t cols, int dtype, fm_weights** out) {
    FM_GUARD_BEGIN
    if (dtype < 0 || dtype > 3)
        return fail(FM_ERR_INVALID_ARG, "dtype must be 0 (f64), 1 (f32), 2 (bf16) or 3 (f64 transposed)");
    if (int st = set_dev(c)) return st;
    auto* w = new fm_weights();
    w->device = c->device;
    w->rows = rows;
    w->cols = cols;
    w->dtype = dtype;
    w->nbytes = rows * cols * dtype_bytes(dtype);
    if (cudaMalloc(&w->buf, w->nbytes) != cudaSuccess) {
        cudaGetLastError();
        delete w;
        return fail(FM_ERR_DEVICE_OOM, "weights buffer");
    }
    *out = w;
    return FM_OK;
    FM_GUARD_END
}

// publish_weights (training.hpp:459-467): the agent's current W as ONE
// contiguous device buffer — pack_weights' single-tensor layout (offset 0,
// shape V x D, object_store.hpp:258-273) — stamped with the agent version.
// dtype 0 reproduces the reference payload byte-for-byte; 2 (bf16) is the
// rollout copy the paper's contiguous-buffer sync ships.
int fm_publish_weights(fm_agent* a, int dtype, fm_weights** out) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    if (int st = fm_weights_alloc(a->ctx, a->V, a->D, dtype, out)) return st;
    if (int st = fm_publish_into(a, *out)) {
        fm_weights_destroy(*out);
        *out = nullptr;
        return st;
    }
    return FM_OK;
    FM_GUARD_END
}

// Republish into an existing buffer (same agent dims; dtype taken from w): the
// steady-state path, no allocation.
int fm_publish_into(fm_agent* a, fm_weights* w) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    if (w->rows != a->V || w->cols != a->D) return fail(FM_ERR_CONFIG_ERROR, "weights buffer shape mismatch");
    if (w->device != c->device) return fail(FM_ERR_CONFIG_ERROR, "weights buffer on another GPU");
    const int dtype = w->dtype;
    w->version = a->version;
    cudaStream_t s = c->stream;
    const bool sharded = a->gang && a->gang->connected;  // f64 master rows live on their owners
    if (dtype == 0) {
        if (int st = copy_state(a, 0, 8, w->buf, s)) return st;
    } else if (dtype == 1) {
        double* src = a->W;
        if (sharded) {
            FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&src), a->P * 8, s));
            if (int st = copy_state(a, 0, 8, src, s)) return st;
        }
        f64_to_f32_kernel<<<c->num_sms * 8, 256, 0, s>>>(src, static_cast<float*>(w->buf), a->P);
        FM_CUDA(cudaGetLastError());
        count_launch();
        if (sharded) FM_CUDA(cudaFreeAsync(src, s));
    } else if (dtype == 3) {
        // rollout layout: one feature's weights over the vocabulary are contiguous, so the
        // generator's per-token column reads coalesce
        double* src = a->W;
        if (sharded) {
            FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&src), a->P * 8, s));
            if (int st = copy_state(a, 0, 8, src, s)) return st;
        }
        const dim3 grid(static_cast<unsigned>((a->D + 31) / 32), static_cast<unsigned>((a->V + 31) / 32));
        transpose_f64_kernel<<<grid, dim3(32, 8), 0, s>>>(src, static_cast<double*>(w->buf), a->V, a->D);
        FM_CUDA(cudaGetLastError());
        count_launch();
        if (sharded) FM_CUDA(cudaFreeAsync(src, s));
    } else if (a->W16 && !(sharded && a->gang->vocab)) {
        // the bf16 shadow IS bf16(W) (same double -> float -> bf16 rounding; full replica in a
        // token gang), held transposed: back to the payload's [V][D]
        FM_CUDA(launch_w16t_untranspose(a->W16, a->V, a->D, w16_ld(a), static_cast<__nv_bfloat16*>(w->buf), s));
        count_launch();
    } else if (sharded) {
        // vocabulary gang: each rank holds its own shadow columns only — from the owners' W rows
        double* src = nullptr;
        FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&src), a->P * 8, s));
        if (int st = copy_state(a, 0, 8, src, s)) return st;
        FM_CUDA(launch_to_bf16(src, static_cast<__nv_bfloat16*>(w->buf), a->P, c->num_sms, s));
        count_launch();
        FM_CUDA(cudaFreeAsync(src, s));
    } else {
        FM_CUDA(launch_to_bf16(a->W, static_cast<__nv_bfloat16*>(w->buf), a->P, c->num_sms, s));
        count_launch();
    }
    FM_CUDA(cudaStreamSynchronize(s));
    return FM_OK;
    FM_GUARD_END
}

int fm_weights_info(const fm_weights* w, int64_t* version, uint64_t* rows, uint64_t* cols, int* dtype,
                    uint64_t* nbytes, int* device) {
    if (version) *version = w->version;
    if (rows) *rows = w->rows;
    if (cols) *cols = w->cols;
    if (dtype) *dtype = w->dtype;
    if (nbytes) *nbytes = w->nbytes;
    if (device) *device = w->device;
    return FM_OK;
}

// One Get per consumer (rollout.hpp:510-541 sync_agent): a single contiguous
// copy into `dst` — host memory (dst_device = -1) or any GPU of this process
// (peer GPUs over NVLink via cudaMemcpyPeer).
int fm_weights_get(const fm_weights* w, void* dst, int dst_device) {
    FM_GUARD_BEGIN
    // synchronous: returns when the copy has landed (the caller may free or
    // republish the source right after); the caller's current device is kept
    int prev = 0;
    FM_CUDA(cudaGetDevice(&prev));
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    FM_CUDA(cudaSetDevice(w->device));
    if (dst_device < 0) {
        FM_CUDA(cudaMemcpy(dst, w->buf, w->nbytes, cudaMemcpyDeviceToHost));
    } else if (dst_device == w->device) {
        FM_CUDA(cudaMemcpy(dst, w->buf, w->nbytes, cudaMemcpyDeviceToDevice));
        FM_CUDA(cudaDeviceSynchronize());
    } else {
        int can = 0;
        FM_CUDA(cudaDeviceCanAccessPeer(&can, dst_device, w->device));
        FM_CUDA(cudaSetDevice(dst_device));
        if (can) {
            cudaError_t pe = cudaDeviceEnablePeerAccess(w->device, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) FM_CUDA(pe);
            cudaGetLastError();
        }
        // one NVLink copy on a private stream of the consumer GPU
        cudaStream_t st;
        FM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const cudaError_t e = cudaMemcpyPeerAsync(dst, dst_device, w->buf, w->device, w->nbytes, st);
        const cudaError_t e2 = e == cudaSuccess ? cudaStreamSynchronize(st) : e;
        cudaStreamDestroy(st);
        FM_CUDA(e2);
    }
    return FM_OK;
    FM_GUARD_END
}

// Weight sync to every rank of a communicator in one collective (NCCL over
// NVLink/NVSwitch): the root's published buffer -> each rank's buffer.
int fm_weights_broadcast(fm_weights* w, fm_comm* cm, int root) {
    FM_GUARD_BEGIN
    FM_CUDA(cudaSetDevice(w->device));
    if (w->device != cm->ctx->device) return fail(FM_ERR_CONFIG_ERROR, "weights and communicator on different GPUs");
    // (dtype 3, f64 transposed, is rows x cols doubles like dtype 0)
    const ncclDataType_t dt = w->dtype == 0 || w->dtype == 3 ? ncclFloat64 : w->dtype == 1 ? ncclFloat32 : ncclBfloat16;
    int64_t ver = w->version;
    int64_t* dver = nullptr;
    FM_CUDA(cudaMalloc(&dver, sizeof(int64_t)));
    FM_CUDA(cudaMemcpy(dver, &ver, sizeof(int64_t), cudaMemcpyHostToDevice));
    FM_NCCL(ncclGroupStart());
    FM_NCCL(ncclBroadcast(w->buf, w->buf, w->rows * w->cols, dt, root, cm->comm, cm->ctx->stream));
    FM_NCCL(ncclBroadcast(dver, dver, 1, ncclInt64, root, cm->comm, cm->ctx->stream));
    FM_NCCL(ncclGroupEnd());
    FM_CUDA(cudaStreamSynchronize(cm->ctx->stream));
    FM_CUDA(cudaMemcpy(&ver, dver, sizeof(int64_t), cudaMemcpyDeviceToHost));
    cudaFree(dver);
    w->version = ver;
    return FM_OK;
    FM_GUARD_END
}

int fm_weights_destroy(fm_weights* w) {
    if (!w) return FM_OK;
    cudaSetDevice(w->device);
    cudaFree(w->buf);
    delete w;
    return FM_OK;
}

// PolicyState::serialize (training.hpp:107-133), byte for byte: u64 version,
// step_count, samples_accumulated, vocab, feat; W, m, v as (u64 rows, u64
// cols, f64 data); u64 cache_n; entries.  The reference caches one V x D term
// per sample; this engine keeps only their sum, so a pending step is written
// as ONE entry with key ("__sum__", 0, 0, version) holding sum(term) =
// -G * dW, which the reference's canonical reduction turns back into the same
// gradient.  With no pending gradient (the usual swap point) the bytes are
// identical to the reference's.
int fm_agent_serialize(fm_agent* a, int64_t global_batch, uint8_t* out, uint64_t cap, uint64_t* len) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    const uint64_t P = a->P;
    const bool pending = a->samples > 0 && a->dw_valid;
    const uint64_t need = 5 * 8 + 3 * (16 + 8 * P) + 8 + (pending ? (8 + 7 + 24 + 16 + 8 * P) : 0);
    *len = need;
    if (!out) return FM_OK;
    if (cap < need) return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "serialize buffer too small");
    std::vector<uint8_t> head;
    for (uint64_t x : {static_cast<uint64_t>(a->version), static_cast<uint64_t>(a->step),
                       static_cast<uint64_t>(a->samples), a->V, a->D})
        put_u64(head, x);
    uint8_t* p = out;
    std::memcpy(p, head.data(), head.size());
    p += head.size();
    auto put_hdr = [&](uint64_t r, uint64_t cc) {
        std::memcpy(p, &r, 8);
        std::memcpy(p + 8, &cc, 8);
        p += 16;
    };
    put_hdr(a->V, a->D);
    if (int st = copy_state(a, 0, 8, p, c->stream)) return st;  // gathers a gang's row shards
    FM_CUDA(cudaStreamSynchronize(c->stream));
    p += P * 8;
    std::vector<float> tmp(P);
    for (size_t off : {slot_off_m(a), slot_off_v(a)}) {  // fp32 moments widen exactly to f64
        put_hdr(a->V, a->D);
        if (int st = copy_state(a, off, 4, tmp.data(), c->stream)) return st;
        FM_CUDA(cudaStreamSynchronize(c->stream));
        if (a->step == 0) std::fill(tmp.begin(), tmp.end(), 0.f);
        double* d = reinterpret_cast<double*>(p);
        for (uint64_t i = 0; i < P; ++i) {
            const double x = tmp[i];
            std::memcpy(d + i, &x, 8);
        }
        p += P * 8;
    }
    const uint64_t cache_n = pending ? 1 : 0;
    std::memcpy(p, &cache_n, 8);
    p += 8;
    if (pending) {
        const char key[] = "__sum__";
        const uint64_t klen = 7, zero = 0, ver = static_cast<uint64_t>(a->version);
        std::memcpy(p, &klen, 8);
        std::memcpy(p + 8, key, 7);
        p += 15;
        std::memcpy(p, &zero, 8);
        std::memcpy(p + 8, &zero, 8);
        std::memcpy(p + 16, &ver, 8);
        p += 24;
        put_hdr(a->V, a->D);
        std::vector<double> g(P);
        if (int st = fm_agent_read_grad(a, g.data())) return st;
        const double scale = -static_cast<double>(global_batch);
        for (uint64_t i = 0; i < P; ++i) g[i] *= scale;
        std::memcpy(p, g.data(), P * 8);
        p += P * 8;
    }
    return FM_OK;
    FM_GUARD_END
}

// PolicyState::deserialize (training.hpp:135-164) into this agent's device
// state.  Matrix dims are read rows-then-cols in the defined order (the
// reference's unspecified argument evaluation at :146 transposes them).
int fm_agent_deserialize(fm_agent* a, int64_t global_batch, const uint8_t* in, uint64_t len) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    uint64_t pos = 0;
    auto rd = [&](uint64_t* x) -> bool {
        if (pos + 8 > len) return false;
        std::memcpy(x, in + pos, 8);
        pos += 8;
        return true;
    };
    uint64_t version, step, samples, vocab, feat;
    if (!rd(&version) || !rd(&step) || !rd(&samples) || !rd(&vocab) || !rd(&feat))
        return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "truncated header");
    if (vocab != a->V || feat != a->D) return fail(FM_ERR_CONFIG_ERROR, "state dims differ from the agent's");
    const uint64_t P = a->P;
    std::vector<double> mats[3];
    for (int k = 0; k < 3; ++k) {
        uint64_t r, cc;
        if (!rd(&r) || !rd(&cc)) return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "truncated matrix header");
        if (r * cc != P || pos + 8 * P > len) return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "matrix size");
        mats[k].resize(P);
        std::memcpy(mats[k].data(), in + pos, 8 * P);
        pos += 8 * P;
    }
    uint64_t cache_n;
    if (!rd(&cache_n)) return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "truncated cache count");
    std::vector<double> sum(cache_n ? P : 0, 0.0);
    for (uint64_t e = 0; e < cache_n; ++e) {
        uint64_t klen, turns, traj, ver, r, cc;
        if (!rd(&klen) || pos + klen > len) return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "cache key");
        pos += klen;
        if (!rd(&turns) || !rd(&traj) || !rd(&ver) || !rd(&r) || !rd(&cc) || r * cc != P || pos + 8 * P > len)
            return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "cache entry");
        const double* d = reinterpret_cast<const double*>(in + pos);
        for (uint64_t i = 0; i < P; ++i) {
            double x;
            std::memcpy(&x, d + i, 8);
            sum[i] += x;
        }
        pos += 8 * P;
    }
    cudaStream_t s = c->stream;
    FM_CUDA(cudaStreamSynchronize(s));
    FM_CUDA(cudaMemcpy(a->W, mats[0].data(), P * 8, cudaMemcpyHostToDevice));
    std::vector<float> f(P);
    for (int k = 1; k < 3; ++k) {
        for (uint64_t i = 0; i < P; ++i) f[i] = static_cast<float>(mats[k][i]);
        FM_CUDA(cudaMemcpy(k == 1 ? a->m : a->v, f.data(), P * 4, cudaMemcpyHostToDevice));
    }
    if (cache_n) {  // accumulator = -(1/G) * sum(term)   (training.hpp:444-446)
        const double scale = -1.0 / static_cast<double>(global_batch);
        if (a->precision == FM_PRECISION_PARITY_F64) {
            for (uint64_t i = 0; i < P; ++i) sum[i] *= scale;
            FM_CUDA(cudaMemcpy(a->dW, sum.data(), P * 8, cudaMemcpyHostToDevice));
        } else {
            for (uint64_t i = 0; i < P; ++i) f[i] = static_cast<float>(sum[i] * scale);
            FM_CUDA(cudaMemcpy(a->dW, f.data(), P * 4, cudaMemcpyHostToDevice));
        }
        a->dw_valid = true;
    } else {
        a->dw_valid = false;
    }
    if (a->W16) {
        FM_CUDA(launch_w16t(a->W, a->V, a->D, a->W16, w16_ld(a), c->num_sms, s));
        count_launch();
        a->fmax_valid = false;
    }
    FM_CUDA(cudaStreamSynchronize(s));
    a->version = static_cast<int64_t>(version);
    a->step = static_cast<int64_t>(step);
    a->samples = static_cast<int64_t>(samples);
    return FM_OK;
    FM_GUARD_END
}

// §8f-3: PolicyModel::generate (policy.hpp:119-130) for n requests on the GPU
// from a published f64 weight buffer; seeds are the per-request token seeds
// (rollout.hpp:638-645).  Host arrays in and out.
int fm_generate(fm_ctx* c, const fm_weights* w, const int32_t* prompts, const int32_t* prompt_off, int n,
                int max_tokens, const uint64_t* seeds, int32_t* out_tokens, double* out_logp, int32_t* out_len) {
    FM_GUARD_BEGIN
    if (w->dtype != 0 && w->dtype != 3)
        return fail(FM_ERR_CONFIG_ERROR, "generation reads f64 weights (publish with dtype 0 or 3)");
    if (w->device != c->device) return fail(FM_ERR_CONFIG_ERROR, "weights live on another GPU (fm_weights_get)");
    if (n <= 0 || max_tokens <= 0) return FM_OK;
    if (int st = set_dev(c)) return st;
    cudaStream_t s = c->stream;
    const int np = prompt_off[n];
    int32_t *dp = nullptr, *doff = nullptr, *dtok = nullptr, *dlen = nullptr;
    uint64_t* dseed = nullptr;
    double *dz = nullptr, *dlp = nullptr;
    const size_t nt = static_cast<size_t>(n) * max_tokens;
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dp), std::max(np, 1) * 4, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&doff), (n + 1) * 4, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dseed), n * 8, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dz), static_cast<size_t>(n) * w->rows * 8, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dtok), nt * 4, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dlp), nt * 8, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dlen), n * 4, s));
    if (np) FM_CUDA(cudaMemcpyAsync(dp, prompts, np * 4, cudaMemcpyHostToDevice, s));
    FM_CUDA(cudaMemcpyAsync(doff, prompt_off, (n + 1) * 4, cudaMemcpyHostToDevice, s));
    FM_CUDA(cudaMemcpyAsync(dseed, seeds, n * 8, cudaMemcpyHostToDevice, s));
    FM_CUDA(launch_generate(static_cast<const double*>(w->buf), w->dtype == 3, w->rows, w->cols, dp, doff, n,
                            max_tokens, dseed, dz, dtok, dlp, dlen, s));
    count_launch();
    FM_CUDA(cudaMemcpyAsync(out_tokens, dtok, nt * 4, cudaMemcpyDeviceToHost, s));
    FM_CUDA(cudaMemcpyAsync(out_logp, dlp, nt * 8, cudaMemcpyDeviceToHost, s));
    FM_CUDA(cudaMemcpyAsync(out_len, dlen, n * 4, cudaMemcpyDeviceToHost, s));
    for (void* p : {static_cast<void*>(dp), static_cast<void*>(doff), static_cast<void*>(dseed),
                    static_cast<void*>(dz), static_cast<void*>(dtok), static_cast<void*>(dlp),
                    static_cast<void*>(dlen)})
        FM_CUDA(cudaFreeAsync(p, s));
    FM_CUDA(cudaStreamSynchronize(s));
    return FM_OK;
    FM_GUARD_END
}

}  // extern "C"


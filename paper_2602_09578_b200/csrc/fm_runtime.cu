// fm_runtime.cu — C ABI implementation: device contexts, the token arena,
// per-agent trainer state, the micro-batch pipeline
//   K-gather + K-pos + K-pslot -> K-stats -> K-lse -> K-band -> K-GEMM2 (tcgen05)
// (or the fp64 parity pipeline), the fused Adam update; training-state swap
// and migration (fm_swap.cu), DP gangs (fm_gang.cu), weight publish and the
// PolicyState wire format (fm_publish.cu).
//
// Memory layout in HBM: every agent state matrix is
// row-major [V][D] (row = vocab id, col = feature; tensor.hpp:13-22):
//   W     f64   master weights            (8 B/param)
//   m, v  f32   Adam moments              (4+4 B/param)
//   dW    f32   gradient accumulator      (4 B/param; f64 in parity mode)
// and the tensor-core path's bf16 shadow is TRANSPOSED:
//   W16^T bf16  [D][round_up(V, 8)]       (2 B/param; a feature's weights are
//               one contiguous row — the row K-stats / K-band stream per
//               context position)
// Per-GPU workspace, sized for the largest micro-batch (Mpad = rows rounded up
// to 128): packed rows, K-stats partials [Mpad][V/256], per-position features
// and slots, and K-GEMM2's segments: A' (one bf16 gradient row H per context
// position, [M + 3 n + 64 * D/256][V]) and the one-hot B' [.][256].
#include "fm_state.h"


namespace fm {

bool make_tmap_bf16_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                           uint64_t pitch) {
    EncodeTiledFn f = encode_fn();
    if (!f) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {(pitch ? pitch : cols) * 2};
    const cuuint32_t box[2] = {64, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return f(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_f32_out(CUtensorMap* map, const float* base, uint64_t rows, uint64_t cols, uint64_t pitch) {
    EncodeTiledFn f = encode_fn();
    if (!f || (pitch & 3)) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {pitch * 4};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    return f(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_gather4(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch) {
    EncodeTiledFn f = encode_fn();
    if (!f) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {(pitch ? pitch : cols) * 2};
    const cuuint32_t box[2] = {64, 1};
    const cuuint32_t estr[2] = {1, 1};
    return f(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, uint32_t elem_bytes, uint64_t rows,
                  uint64_t cols, uint32_t box_rows, uint32_t box_cols) {
    EncodeTiledFn f = encode_fn();
    if (!f) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * elem_bytes};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return f(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace fm

namespace fm {
uint64_t arena_token_count(const fm_ctx* ctx, uint64_t offset, bool* found) {
    auto it = ctx->arena_ntok.find(offset);
    *found = it != ctx->arena_ntok.end();
    return *found ? it->second : 0;
}
}  // namespace fm

namespace fm {

int set_dev(const fm_ctx* c) {
    FM_CUDA(cudaSetDevice(c->device));
    return FM_OK;
}

// Maps a peer's IPC handle once per context: slots and gang receive buffers are
// recycled, so re-formed gangs and repeated migrations reuse the mapping.
int ipc_open_cached(fm_ctx* c, const cudaIpcMemHandle_t& h, void** out) {
    const std::string key(reinterpret_cast<const char*>(&h), sizeof(h));
    auto it = c->ipc_cache.find(key);
    if (it != c->ipc_cache.end()) {
        *out = it->second;
        return FM_OK;
    }
    FM_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_cache.emplace(key, *out);
    return FM_OK;
}

// A recycled device buffer of >= bytes (gang receive buffers keep their IPC
// identity across gangs, so peers' cached mappings stay valid).
int pool_take(fm_ctx* c, size_t bytes, void** out) {
    size_t best = SIZE_MAX;
    int pick = -1;
    for (size_t i = 0; i < c->recv_pool.size(); ++i)
        if (c->recv_pool[i].first >= bytes && c->recv_pool[i].first < best) {
            best = c->recv_pool[i].first;
            pick = static_cast<int>(i);
        }
    if (pick >= 0) {
        *out = c->recv_pool[static_cast<size_t>(pick)].second;
        c->recv_pool.erase(c->recv_pool.begin() + pick);
        return FM_OK;
    }
    if (cudaMalloc(out, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(FM_ERR_DEVICE_OOM, "gang buffer");
    }
    c->pool_sizes[*out] = bytes;
    return FM_OK;
}

void pool_give(fm_ctx* c, void* p) {
    if (p) c->recv_pool.emplace_back(c->pool_sizes[p], p);
}

// Returns a pinned staging slot of >= bytes whose previous use has completed.
int staging_acquire(fm_ctx* c, size_t bytes, uint8_t** out, cudaEvent_t* ev) {
    const int k = c->staging_next;
    c->staging_next = (k + 1) % kStagingSlots;
    FM_CUDA(cudaEventSynchronize(c->staging_ev[k]));
    if (c->staging_cap[k] < bytes) {
        if (c->staging[k]) FM_CUDA(cudaFreeHost(c->staging[k]));
        size_t cap = std::max<size_t>(bytes, 1 << 20);
        FM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->staging[k]), cap, cudaHostAllocDefault));
        c->staging_cap[k] = cap;
    }
    *out = c->staging[k];
    *ev = c->staging_ev[k];
    return FM_OK;
}

void ws_free(Workspace& w) {
    cudaFree(w.action);
    cudaFree(w.ctx4);
    cudaFree(w.n_ctx);
    cudaFree(w.sample);
    cudaFree(w.coef);
    cudaFree(w.rscale);
    cudaFree(w.lse);
    cudaFree(w.logp);
    cudaFree(w.coef_eff);
    cudaFree(w.old_logp);
    cudaFree(w.q0);
    cudaFree(w.mrow);
    cudaFree(w.zact);
    cudaFree(w.lossw);
    cudaFree(w.pos_feat);
    cudaFree(w.pos_slot);
    cudaFree(w.stats);
    cudaFree(w.aseg);
    cudaFree(w.bseg);
    for (auto& x : w.xset) {
        cudaFree(x.aseg);
        cudaFree(x.bseg);
        cudaFree(x.kseg_off);
        cudaFree(x.kiters);
    }
    cudaFree(w.zero_row);
    cudaFree(w.kcount);
    cudaFree(w.kseg_off);
    cudaFree(w.kiters);
    cudaFree(w.kseg_rows);
    cudaFree(w.zscratch);
    cudaFree(w.dWmb);
    cudaFree(w.logp64);
    cudaFree(w.sd);
    cudaFree(w.dpn);
    cudaFree(w.lse_red);
    w = Workspace{};
}

uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

Workspace::SegSet seg_set(Workspace& w, int k) {
    if (k == 0) return Workspace::SegSet{w.aseg, w.bseg, w.kseg_off, w.kiters};
    return w.xset[k - 1];
}

// Ensure tensor-core workspace for Mpad rows of at most n samples, vocab V,
// features D: row buffers, K-stats partials, positions (Mpad + 3 n) and the
// K-GEMM2 segments (positions + 64 padding rows per 256-feature block).
int ws_reserve_tc(fm_ctx* c, int64_t Mpad, uint64_t V, uint64_t D, int n_samples) {
    Workspace& w = c->ws;
    const int64_t Qneed = Mpad + 3 * static_cast<int64_t>(std::max(n_samples, 1));
    if (Mpad <= w.rows_cap && V <= w.vocab_cap && D <= w.feat_cap && Qneed <= w.pos_cap && w.aseg) return FM_OK;
    if (int st = ctx_flush(c)) return st;  // deferred K-GEMM2s read the segment sets
    const int64_t R = std::max<int64_t>(Mpad, w.rows_cap);
    const uint64_t VV = std::max<uint64_t>(V, w.vocab_cap), DD = std::max<uint64_t>(D, w.feat_cap);
    const int64_t Q = std::max<int64_t>(Qneed, w.pos_cap);
    FM_CUDA(cudaStreamSynchronize(c->stream));
    Workspace keep;  // parity scratch and sample descriptors survive
    std::swap(keep.zscratch, w.zscratch);
    std::swap(keep.dWmb, w.dWmb);
    std::swap(keep.logp64, w.logp64);
    std::swap(keep.sd, w.sd);
    std::swap(keep.old_logp, w.old_logp);
    std::swap(keep.dpn, w.dpn);
    keep.dpn_cap = w.dpn_cap;
    std::swap(keep.lse_red, w.lse_red);
    keep.lse_red_cap = w.lse_red_cap;
    keep.prow_cap = w.prow_cap;
    keep.pvocab_cap = w.pvocab_cap;
    keep.pparam_cap = w.pparam_cap;
    keep.sd_cap = w.sd_cap;
    keep.old_logp_cap = w.old_logp_cap;
    ws_free(w);
    w = keep;
    const uint64_t ldz = round_up(VV, 8);
    const uint64_t tiles_n = static_cast<uint64_t>(band_stats_ld(static_cast<int64_t>(VV))) + 8;
    const int64_t nblk = static_cast<int64_t>((DD + 255) / 256);
    const int64_t kp = Q + 64 * nblk;
    cudaError_t e = cudaSuccess;
    e = e ? e : dalloc(&w.action, R);
    e = e ? e : dalloc(&w.ctx4, R);
    e = e ? e : dalloc(&w.n_ctx, R);
    e = e ? e : dalloc(&w.sample, R);
    e = e ? e : dalloc(&w.coef, R);
    e = e ? e : dalloc(&w.rscale, R);
    e = e ? e : dalloc(&w.lse, R);
    e = e ? e : dalloc(&w.logp, R);
    e = e ? e : dalloc(&w.coef_eff, R);
    e = e ? e : dalloc(&w.q0, R);
    e = e ? e : dalloc(&w.mrow, R);
    e = e ? e : dalloc(&w.zact, R);
    e = e ? e : dalloc(&w.lossw, R);
    e = e ? e : dalloc(&w.stats, static_cast<size_t>(R) * tiles_n);  // [tiles][R] partial sums
    e = e ? e : dalloc(&w.pos_feat, static_cast<size_t>(Q));
    e = e ? e : dalloc(&w.pos_slot, static_cast<size_t>(Q));
    e = e ? e : dalloc(&w.aseg, static_cast<size_t>(kp) * ldz);
    // A' rows are only written for live positions: segment padding rows must hold
    // finite values (B' is zero there), so the buffer starts zeroed
    e = e ? e : cudaMemset(w.aseg, 0, static_cast<size_t>(kp) * ldz * 2);
    e = e ? e : dalloc(&w.bseg, static_cast<size_t>(kp) * 256);
    e = e ? e : dalloc(&w.zero_row, 4096);
    e = e ? e : cudaMemset(w.zero_row, 0, 4096 * 2);
    // chunk counts and their per-(block, chunk) bases (K-pslot)
    e = e ? e : dalloc(&w.kcount, 2 * static_cast<size_t>(nblk) * static_cast<size_t>((Q + 1023) / 1024 + 1));
    e = e ? e : dalloc(&w.kseg_off, static_cast<size_t>(nblk));
    e = e ? e : dalloc(&w.kiters, static_cast<size_t>(nblk));
    e = e ? e : dalloc(&w.kseg_rows, 1);
    e = e ? e : cudaMemset(w.kseg_rows, 0, sizeof(unsigned long long));
    if (e != cudaSuccess) {
        cudaGetLastError();
        ws_free(w);
        return fail(FM_ERR_DEVICE_OOM, std::string("workspace allocation: ") + cudaGetErrorString(e));
    }
    // further segment sets for the per-step batched K-GEMM2 while HBM allows: each
    // must leave a quarter of the device free (a set is ~1.1 GB at C2, 17 GB at C5)
    w.nsets = 1;
    const size_t set_bytes = static_cast<size_t>(kp) * ldz * 2 + static_cast<size_t>(kp) * 256 * 2 + 8 * nblk;
    for (int k = 0; k < kGemmMaxBatch - 1; ++k) {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess || fr < set_bytes + tot / 4) break;
        Workspace::SegSet& x = w.xset[k];
        cudaError_t ex = dalloc(&x.aseg, static_cast<size_t>(kp) * ldz);
        ex = ex ? ex : cudaMemset(x.aseg, 0, static_cast<size_t>(kp) * ldz * 2);  // finite padding rows
        ex = ex ? ex : dalloc(&x.bseg, static_cast<size_t>(kp) * 256);
        ex = ex ? ex : dalloc(&x.kseg_off, static_cast<size_t>(nblk));
        ex = ex ? ex : dalloc(&x.kiters, static_cast<size_t>(nblk));
        if (ex != cudaSuccess) {
            cudaGetLastError();
            cudaFree(x.aseg);
            cudaFree(x.bseg);
            cudaFree(x.kseg_off);
            cudaFree(x.kiters);
            x = Workspace::SegSet{};
            break;
        }
        w.nsets = k + 2;
    }
    w.rows_cap = R;
    w.vocab_cap = VV;
    w.feat_cap = DD;
    w.pos_cap = Q;
    w.kp_cap = kp;
    return FM_OK;
}

int ws_reserve_rows(fm_ctx* c, int64_t R) {  // row arrays only (parity mode)
    Workspace& w = c->ws;
    if (R <= w.rows_cap && w.action) return FM_OK;
    if (w.aseg) return ws_reserve_tc(c, R, w.vocab_cap, w.feat_cap, 1);
    FM_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(w.action);
    cudaFree(w.ctx4);
    cudaFree(w.n_ctx);
    cudaFree(w.sample);
    cudaFree(w.coef);
    cudaFree(w.rscale);
    cudaFree(w.lse);
    cudaFree(w.logp);
    cudaFree(w.coef_eff);
    cudaError_t e = cudaSuccess;
    e = e ? e : dalloc(&w.action, R);
    e = e ? e : dalloc(&w.ctx4, R);
    e = e ? e : dalloc(&w.n_ctx, R);
    e = e ? e : dalloc(&w.sample, R);
    e = e ? e : dalloc(&w.coef, R);
    e = e ? e : dalloc(&w.rscale, R);
    e = e ? e : dalloc(&w.lse, R);
    e = e ? e : dalloc(&w.logp, R);
    e = e ? e : dalloc(&w.coef_eff, R);
    if (e != cudaSuccess) return fail(FM_ERR_DEVICE_OOM, cudaGetErrorString(e));
    w.rows_cap = R;
    return FM_OK;
}

int ws_reserve_parity(fm_ctx* c, int64_t M, uint64_t V, uint64_t P) {
    Workspace& w = c->ws;
    int st = ws_reserve_rows(c, std::max<int64_t>(M, 1));
    if (st) return st;
    if (M * static_cast<int64_t>(V) > w.prow_cap * static_cast<int64_t>(w.pvocab_cap) || !w.zscratch) {
        FM_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(w.zscratch);
        cudaFree(w.logp64);
        const int64_t R = std::max<int64_t>(M, w.prow_cap);
        const uint64_t VV = std::max<uint64_t>(V, w.pvocab_cap);
        if (dalloc(&w.zscratch, static_cast<size_t>(R) * VV) || dalloc(&w.logp64, R))
            return fail(FM_ERR_DEVICE_OOM, "parity scratch");
        w.prow_cap = R;
        w.pvocab_cap = VV;
    }
    if (M > w.prow_cap) {
        FM_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(w.logp64);
        if (dalloc(&w.logp64, M)) return fail(FM_ERR_DEVICE_OOM, "parity logp");
        w.prow_cap = M;
    }
    if (P > w.pparam_cap || !w.dWmb) {
        FM_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(w.dWmb);
        if (dalloc(&w.dWmb, P)) return fail(FM_ERR_DEVICE_OOM, "parity dWmb");
        FM_CUDA(cudaMemset(w.dWmb, 0, P * sizeof(double)));
        w.pparam_cap = P;
    }
    return FM_OK;
}

int ws_reserve_sd(fm_ctx* c, int n) {
    Workspace& w = c->ws;
    if (n <= w.sd_cap) return FM_OK;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(w.sd);
    const int cap = std::max(n, 256);
    if (dalloc(&w.sd, cap)) return fail(FM_ERR_DEVICE_OOM, "sample descriptors");
    w.sd_cap = cap;
    return FM_OK;
}

RowBuffers row_buffers(Workspace& w) {
    RowBuffers r;
    r.action = w.action;
    r.ctx4 = w.ctx4;
    r.n_ctx = w.n_ctx;
    r.sample = w.sample;
    r.coef = w.coef;
    r.rscale = w.rscale;
    r.lse = w.lse;
    r.logp = w.logp;
    r.coef_eff = w.coef_eff;
    r.q0 = w.q0;
    r.mrow = w.mrow;
    r.fmax = nullptr;
    return r;
}


}  // namespace fm

extern "C" {

int fm_ctx_set_kernel_timing(fm_ctx* c, int on) {
    c->kt.on = on != 0;
    return FM_OK;
}

// Drains the recorded event pairs; out_ms / out_count have K_NKINDS (8) slots:
// gather, stats, lse, band, gemm2, adam, parity, memset.
int fm_ctx_kernel_times(fm_ctx* c, double* out_ms, int64_t* out_count, int reset) {
    if (int st = set_dev(c)) return st;
    KTimer& k = c->kt;
    for (auto& o : k.open) {
        FM_CUDA(cudaEventSynchronize(o.second.second));
        float ms = 0.f;
        FM_CUDA(cudaEventElapsedTime(&ms, o.second.first, o.second.second));
        if (std::getenv("FM_KT_TRACE")) std::fprintf(stderr, "kt %d %.4f\n", o.first, ms);  // per-launch trace
        k.ms[o.first] += ms;
        k.count[o.first] += 1;
        k.pool.push_back(o.second.first);
        k.pool.push_back(o.second.second);
    }
    k.open.clear();
    for (int i = 0; i < K_NKINDS; ++i) {
        if (out_ms) out_ms[i] = k.ms[i];
        if (out_count) out_count[i] = k.count[i];
        if (reset) {
            k.ms[i] = 0.0;
            k.count[i] = 0;
        }
    }
    return FM_OK;
}

// Device-side step timer on the compute stream (the copy streams are joined
// first, so swaps in flight are inside the measured interval).
int fm_ctx_timer_start(fm_ctx* c) {
    if (int st = set_dev(c)) return st;
    if (!c->t0) {
        FM_CUDA(cudaEventCreate(&c->t0));
        FM_CUDA(cudaEventCreate(&c->t1));
    }
    FM_CUDA(cudaEventRecord(c->t0, c->stream));
    return FM_OK;
}

int fm_ctx_timer_stop(fm_ctx* c, double* ms) {
    if (int st = set_dev(c)) return st;
    if (int st = ctx_flush(c)) return st;  // queued K-GEMM2s belong to the timed work
    cudaEvent_t j;
    FM_CUDA(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
    for (cudaStream_t cs : {c->copy_in, c->copy_out}) {
        FM_CUDA(cudaEventRecord(j, cs));
        FM_CUDA(cudaStreamWaitEvent(c->stream, j, 0));
    }
    FM_CUDA(cudaEventRecord(c->t1, c->stream));
    FM_CUDA(cudaEventSynchronize(c->t1));
    cudaEventDestroy(j);
    float f = 0.f;
    FM_CUDA(cudaEventElapsedTime(&f, c->t0, c->t1));
    *ms = f;
    return FM_OK;
}

int fm_ctx_create(int device, fm_ctx** out) {
    FM_GUARD_BEGIN
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(FM_ERR_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= n) return fail(FM_ERR_NO_DEVICE, "device index out of range");
    cudaDeviceProp prop;
    FM_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(FM_ERR_NO_DEVICE, std::string("sm_100 device required, found ") + prop.name);
    FM_CUDA(cudaSetDevice(device));
    auto* c = new fm_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    FM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    FM_CUDA(cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking));
    FM_CUDA(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
    FM_CUDA(cudaEventCreateWithFlags(&c->ev_gemm, cudaEventDisableTiming));
    for (int i = 0; i < kStagingSlots; ++i)
        FM_CUDA(cudaEventCreateWithFlags(&c->staging_ev[i], cudaEventDisableTiming));
    {   // keep freed agent state in the stream-ordered pool: swaps re-use it without remapping
        cudaMemPool_t pool;
        FM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = ~0ull;
        FM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    if (!encode_fn()) {
        delete c;
        return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    }
    *out = c;
    return FM_OK;
    FM_GUARD_END
}

int fm_ctx_destroy(fm_ctx* c) {
    if (!c) return FM_OK;
    cudaSetDevice(c->device);
    ctx_flush(c);  // a queued K-GEMM2 still belongs to a live agent's dW and reports
    cudaDeviceSynchronize();
    ws_free(c->ws);
    cudaFree(c->arena);
    for (Slot* sl : c->slots) {
        cudaFree(sl->base);
        cudaEventDestroy(sl->ev_free);
        delete sl;
    }
    for (int i = 0; i < kStagingSlots; ++i) {
        if (c->staging[i]) cudaFreeHost(c->staging[i]);
        cudaEventDestroy(c->staging_ev[i]);
    }
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->copy_in);
    cudaStreamDestroy(c->copy_out);
    if (c->ev_gemm) cudaEventDestroy(c->ev_gemm);
    for (auto& kv : c->ipc_cache) cudaIpcCloseMemHandle(kv.second);
    for (auto& pb : c->recv_pool) cudaFree(pb.second);
    delete c;
    return FM_OK;
}

int fm_ctx_device(const fm_ctx* c) { return c->device; }
int fm_ctx_num_sms(const fm_ctx* c) { return c->num_sms; }

int fm_ctx_synchronize(fm_ctx* c) {
    if (int st = set_dev(c)) return st;
    if (int st = ctx_flush(c)) return st;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    FM_CUDA(cudaStreamSynchronize(c->copy_in));
    FM_CUDA(cudaStreamSynchronize(c->copy_out));
    return FM_OK;
}

int fm_ctx_reserve(fm_ctx* c, uint64_t arena_bytes, int64_t max_rows, uint64_t V, uint64_t D) {
    FM_GUARD_BEGIN
    if (int st = set_dev(c)) return st;
    if (arena_bytes > c->arena_cap) {
        FM_CUDA(cudaDeviceSynchronize());  // every stream reading the arena (compute, on-device tables)
        uint8_t* na = nullptr;
        if (cudaMalloc(&na, arena_bytes) != cudaSuccess) return fail(FM_ERR_DEVICE_OOM, "token arena");
        if (c->arena_used) FM_CUDA(cudaMemcpy(na, c->arena, c->arena_used, cudaMemcpyDeviceToDevice));
        cudaFree(c->arena);
        c->arena = na;
        c->arena_cap = arena_bytes;
    }
    if (max_rows > 0 && V > 0 && D > 0)
        return ws_reserve_tc(c, static_cast<int64_t>(round_up(max_rows, 128)), V, D, 1);
    return FM_OK;
    FM_GUARD_END
}

int fm_arena_put(fm_ctx* c, const uint8_t* payload, uint64_t nbytes, uint64_t* off_out) {
    FM_GUARD_BEGIN
    if (nbytes < 8) return fail(FM_ERR_INVALID_ARG, "payload shorter than its u64 count header");
    uint64_t ntok;
    std::memcpy(&ntok, payload, 8);
    if (nbytes != 8 + 8 * ntok) return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "payload length != 8 + 8*count");
    if (int st = set_dev(c)) return st;
    const uint64_t off = round_up(c->arena_used, 16);
    if (off + nbytes > c->arena_cap) {
        const uint64_t cap = std::max<uint64_t>(2 * c->arena_cap, off + nbytes + (64u << 20));
        int st = fm_ctx_reserve(c, cap, 0, 0, 0);
        if (st) return st;
    }
    uint8_t* stg;
    cudaEvent_t ev;
    if (int st = staging_acquire(c, nbytes, &stg, &ev)) return st;
    std::memcpy(stg, payload, nbytes);
    FM_CUDA(cudaMemcpyAsync(c->arena + off, stg, nbytes, cudaMemcpyHostToDevice, c->stream));
    FM_CUDA(cudaEventRecord(ev, c->stream));
    c->arena_used = off + nbytes;
    c->arena_ntok[off] = ntok;
    *off_out = off;
    return FM_OK;
    FM_GUARD_END
}

int fm_arena_reset(fm_ctx* c) {
    if (int st = set_dev(c)) return st;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    c->arena_used = 0;
    c->arena_ntok.clear();
    c->e2e_off = c->e2e_cap = 0;
    return FM_OK;
}

uint64_t fm_arena_used(const fm_ctx* c) { return c->arena_used; }

}  // extern "C"

namespace fm {

size_t dw_elem(const fm_agent* a) { return a->precision == FM_PRECISION_PARITY_F64 ? 8 : 4; }

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

size_t slot_off_m(const fm_agent* a) { return align256(a->P * 8); }
size_t slot_off_v(const fm_agent* a) { return align256(a->P * 8) + align256(a->P * 4); }

uint64_t w16_ld(const fm_agent* a) { return round_up(a->V, 8); }
size_t w16_bytes(const fm_agent* a) { return a->D * w16_ld(a) * 2; }

size_t slot_bytes(const fm_agent* a) {
    const size_t P = a->P;
    return align256(P * 8) + 2 * align256(P * 4) + align256(P * dw_elem(a)) +
           (a->precision == FM_PRECISION_BF16_TC ? align256(w16_bytes(a)) + align256(a->D * 4) : 0);
}

// Binds a free slot of ctx c (allocating one the first time), ordered on
// stream s after the slot's previous tenant has been copied out.
int agent_alloc_device(fm_agent* a, fm_ctx* c, cudaStream_t s) {
    const size_t need = slot_bytes(a);
    Slot* pick = nullptr;
    for (Slot* sl : c->slots)
        if (!sl->busy && sl->cap >= need && (!pick || sl->cap < pick->cap)) pick = sl;
    if (!pick) {
        pick = new Slot();
        if (cudaMalloc(&pick->base, need) != cudaSuccess) {
            cudaGetLastError();
            delete pick;
            return fail(FM_ERR_DEVICE_OOM, "no HBM for another training slot (" + std::to_string(need) + " B)");
        }
        pick->cap = need;
        FM_CUDA(cudaEventCreateWithFlags(&pick->ev_free, cudaEventDisableTiming));
        FM_CUDA(cudaEventRecord(pick->ev_free, s));
        c->slots.push_back(pick);
    }
    FM_CUDA(cudaStreamWaitEvent(s, pick->ev_free, 0));
    pick->busy = true;
    agent_bind_slot(a, pick);
    a->fmax_valid = false;
    return FM_OK;
}

// Points the agent's W / m / v / dW / W16^T / fmax into slot sl.
void agent_bind_slot(fm_agent* a, Slot* sl) {
    a->slot = sl;
    uint8_t* p = static_cast<uint8_t*>(sl->base);
    const size_t P = a->P;
    a->W = reinterpret_cast<double*>(p);
    p += align256(P * 8);
    a->m = reinterpret_cast<float*>(p);
    p += align256(P * 4);
    a->v = reinterpret_cast<float*>(p);
    p += align256(P * 4);
    a->dW = p;
    p += align256(P * dw_elem(a));
    a->W16 = a->precision == FM_PRECISION_BF16_TC ? reinterpret_cast<__nv_bfloat16*>(p) : nullptr;
    p += a->W16 ? align256(w16_bytes(a)) : 0;
    a->fmax = a->W16 ? reinterpret_cast<float*>(p) : nullptr;
}

void agent_unbind(fm_agent* a) {
    a->slot = nullptr;
    a->W = nullptr;
    a->m = a->v = nullptr;
    a->dW = nullptr;
    a->W16 = nullptr;
    a->fmax = nullptr;
    a->fmax_valid = false;
}

// Releases the agent's slot once everything queued on stream s has run.
void agent_free_device(fm_agent* a, cudaStream_t s) {
    if (a->pending_in) {  // an unconsumed swap-in still writes into the slot
        cudaStreamWaitEvent(s, a->ev_in, 0);
        a->pending_in = false;
    }
    if (a->slot) {
        cudaEventRecord(a->slot->ev_free, s);
        a->slot->busy = false;
    }
    agent_unbind(a);
}

// Every operation on an agent goes through here: besides the InactiveGroup
// check it inserts the lazy dependency on a pending swap-in, so that an
// activate() prefetch never stalls other agents' work on the shared compute
// stream — only this agent's first use waits for its copy-in.
int check_active(fm_agent* a, bool flush) {
    if (!a->active || !a->ctx) return fail(FM_ERR_INACTIVE_GROUP, a->name);
    if (a->partial && !(a->gang && a->gang->vocab))
        return fail(FM_ERR_CONFIG_ERROR, a->name + " holds vocabulary rows [" + std::to_string(a->part_lo) + ", " +
                                             std::to_string(a->part_hi) +
                                             ") only: attach it to its vocabulary gang (fm_gang_attach_mode 1)");
    if (flush && a->ctx->pend_agent == a)
        if (int st = agent_flush(a)) return st;
    if (a->pending_in) {
        FM_CUDA(cudaSetDevice(a->ctx->device));
        FM_CUDA(cudaStreamWaitEvent(a->ctx->stream, a->ev_in, 0));
        a->pending_in = false;
    }
    a->last_seq = ++a->ctx->op_seq;  // everything this op enqueues follows any earlier K-stats mark
    return FM_OK;
}

}  // namespace fm

extern "C" {

int fm_agent_create(fm_ctx* c, const char* name, uint64_t V, uint64_t D, int precision, fm_agent** out) {
    FM_GUARD_BEGIN
    *out = nullptr;
    if (!c) return fail(FM_ERR_NO_DEVICE, "null context");
    if (V == 0 || D == 0) return fail(FM_ERR_CONFIG_ERROR, "vocab and feature dims must be positive");
    if (precision != FM_PRECISION_BF16_TC && precision != FM_PRECISION_PARITY_F64)
        return fail(FM_ERR_INVALID_ARG, "unknown precision");
    if (precision == FM_PRECISION_BF16_TC && (D % 8 != 0 || V % 4 != 0))
        return fail(FM_ERR_CONFIG_ERROR, "tensor-core mode needs D % 8 == 0 and V % 4 == 0 (TMA row pitch)");
    if (int st = set_dev(c)) return st;
    auto* a = new fm_agent();
    a->ctx = c;
    a->name = name ? name : "";
    a->V = V;
    a->D = D;
    a->P = V * D;
    a->precision = precision;
    if (int st = agent_alloc_device(a, c, c->stream)) {
        delete a;
        return st;
    }
    FM_CUDA(cudaMemsetAsync(a->W, 0, a->P * 8, c->stream));
    FM_CUDA(cudaMemsetAsync(a->m, 0, a->P * 4, c->stream));
    FM_CUDA(cudaMemsetAsync(a->v, 0, a->P * 4, c->stream));
    FM_CUDA(cudaMemsetAsync(a->dW, 0, a->P * dw_elem(a), c->stream));
    if (a->W16) FM_CUDA(cudaMemsetAsync(a->W16, 0, w16_bytes(a), c->stream));
    FM_CUDA(cudaMalloc(&a->d_scalars, kReportRing * 2 * sizeof(double)));
    FM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&a->h_scalars), kReportRing * 2 * sizeof(double), 0));
    FM_CUDA(cudaMalloc(&a->d_upd, sizeof(double)));
    FM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&a->h_upd), sizeof(double), 0));
    for (int i = 0; i < kReportRing; ++i) FM_CUDA(cudaEventCreateWithFlags(&a->ev[i], cudaEventDisableTiming));
    FM_CUDA(cudaEventCreateWithFlags(&a->ev_in, cudaEventDisableTiming));
    FM_CUDA(cudaEventCreateWithFlags(&a->ev_out, cudaEventDisableTiming));
    FM_CUDA(cudaEventCreateWithFlags(&a->ev_compute, cudaEventDisableTiming));
    a->ev_device = c->device;
    a->active = true;
    *out = a;
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_destroy(fm_agent* a) {
    if (!a) return FM_OK;
    if (a->lent) fm_agent_migrate_release(a);
    if (a->ctx && a->ctx->pend_agent == a) {  // queued reductions die with the agent
        a->ctx->npend = 0;
        a->ctx->pend_agent = nullptr;
    }
    fm_gang_detach(a);
    if (a->ctx) {
        cudaSetDevice(a->ctx->device);
        cudaStreamSynchronize(a->ctx->stream);
        cudaStreamSynchronize(a->ctx->copy_out);
        agent_free_device(a, a->ctx->stream);
        cudaStreamSynchronize(a->ctx->stream);
    }
    if (a->park) {
        if (a->park_tier == FM_TIER_HOST) cudaFreeHost(a->park);
        else {
            cudaSetDevice(a->park_device);
            cudaFree(a->park);
        }
    }
    cudaFree(a->d_scalars);
    cudaFreeHost(a->h_scalars);
    cudaFree(a->d_upd);
    cudaFreeHost(a->h_upd);
    for (int i = 0; i < kReportRing; ++i) cudaEventDestroy(a->ev[i]);
    cudaEventDestroy(a->ev_in);
    cudaEventDestroy(a->ev_out);
    cudaEventDestroy(a->ev_compute);
    if (a->ev_ipc) cudaEventDestroy(a->ev_ipc);
    delete a;
    return FM_OK;
}

int fm_agent_set_weights(fm_agent* a, const double* W) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    FM_CUDA(cudaMemcpyAsync(a->W, W, a->P * 8, cudaMemcpyHostToDevice, c->stream));
    if (a->W16) {
        FM_CUDA(launch_w16t(a->W, a->V, a->D, a->W16, w16_ld(a), c->num_sms, c->stream));
        count_launch();
        a->fmax_valid = false;
    }
    FM_CUDA(cudaStreamSynchronize(c->stream));
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_read_weights(fm_agent* a, double* W) {
    if (int st = check_active(a)) return st;
    if (int st = set_dev(a->ctx)) return st;
    if (int st = copy_state(a, 0, 8, W, a->ctx->stream)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    return FM_OK;
}

int fm_agent_read_moments(fm_agent* a, float* m, float* v, int64_t* step) {
    if (int st = check_active(a)) return st;
    if (int st = set_dev(a->ctx)) return st;
    if (m)
        if (int st = copy_state(a, slot_off_m(a), 4, m, a->ctx->stream)) return st;
    if (v)
        if (int st = copy_state(a, slot_off_v(a), 4, v, a->ctx->stream)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    if (step) *step = a->step;
    return FM_OK;
}

}  // extern "C"

// fp32 dW to the host; a vocabulary gang's rows live with their owners
static int read_dw_f32(fm_agent* a, float* g) {
    if (a->gang && a->gang->connected && a->gang->vocab) {
        const size_t off = static_cast<size_t>(static_cast<uint8_t*>(a->dW) - static_cast<uint8_t*>(a->slot->base));
        if (int st = copy_state(a, off, 4, g, a->ctx->stream)) return st;
        FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
        return FM_OK;
    }
    FM_CUDA(cudaMemcpy(g, a->dW, a->P * 4, cudaMemcpyDeviceToHost));
    return FM_OK;
}

extern "C" {

int fm_agent_read_grad(fm_agent* a, double* g) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    if (int st = set_dev(a->ctx)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    if (!a->dw_valid) {
        std::fill(g, g + a->P, 0.0);
        return FM_OK;
    }
    if (a->precision == FM_PRECISION_PARITY_F64) {
        FM_CUDA(cudaMemcpy(g, a->dW, a->P * 8, cudaMemcpyDeviceToHost));
    } else {
        std::vector<float> tmp(a->P);
        if (int st = read_dw_f32(a, tmp.data())) return st;
        for (uint64_t i = 0; i < a->P; ++i) g[i] = tmp[i];
    }
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_read_grad_f32(fm_agent* a, float* g) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    if (a->precision != FM_PRECISION_BF16_TC) return fail(FM_ERR_CONFIG_ERROR, "fp32 accumulator: tensor-core agents");
    if (int st = set_dev(a->ctx)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    if (!a->dw_valid) {
        std::fill(g, g + a->P, 0.f);
        return FM_OK;
    }
    if (int st = read_dw_f32(a, g)) return st;
    return FM_OK;
    FM_GUARD_END
}

int fm_debug_gemm(fm_ctx* c, const void* A, const void* B, int a_mn, int b_mn, int M, int N, int K, float* C) {
    FM_GUARD_BEGIN
    if (!c || !A || !B || !C || M <= 0 || N <= 0 || K <= 0 || M % 8 || N % 8 || K % 8)
        return fail(FM_ERR_INVALID_ARG, "debug_gemm: bad arguments");
    if (int st = set_dev(c)) return st;
    CUtensorMap tA, tB, tC;
    const bool ok = (a_mn ? make_tmap_bf16_kmajor(&tA, A, K, M, 64) : make_tmap_bf16_kmajor(&tA, A, M, K, 128)) &&
                    (b_mn ? make_tmap_bf16_kmajor(&tB, B, K, N, 64) : make_tmap_bf16_kmajor(&tB, B, N, K, 128)) &&
                    make_tmap_f32_out(&tC, C, M, N, N);
    if (!ok) return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    FM_CUDA(gemm_debug_launch(tA, tB, tC, a_mn, b_mn, M, N, K, C, c->num_sms, c->stream));
    FM_CUDA(cudaStreamSynchronize(c->stream));
    return FM_OK;
    FM_GUARD_END
}

int fm_ctx_gemm2_rows(fm_ctx* c, int64_t* rows_out, int reset) {
    FM_GUARD_BEGIN
    if (!c || !rows_out) return fail(FM_ERR_INVALID_ARG, "gemm2_rows: bad arguments");
    *rows_out = 0;
    if (!c->ws.kseg_rows) return FM_OK;
    if (int st = set_dev(c)) return st;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    unsigned long long v = 0;
    FM_CUDA(cudaMemcpy(&v, c->ws.kseg_rows, sizeof(v), cudaMemcpyDeviceToHost));
    if (reset) FM_CUDA(cudaMemset(c->ws.kseg_rows, 0, sizeof(v)));
    *rows_out = static_cast<int64_t>(v);
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_read_grad_cols(fm_agent* a, const int64_t* cols, int64_t n_cols, double* g) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    if (n_cols < 0 || (n_cols > 0 && (!cols || !g))) return fail(FM_ERR_INVALID_ARG, "read_grad_cols: bad arguments");
    for (int64_t j = 0; j < n_cols; ++j)
        if (cols[j] < 0 || static_cast<uint64_t>(cols[j]) >= a->D)
            return fail(FM_ERR_INVALID_ARG, "read_grad_cols: column out of range");
    if (int st = set_dev(a->ctx)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    const size_t n = static_cast<size_t>(a->V) * static_cast<size_t>(n_cols);
    if (!a->dw_valid || n == 0) {
        std::fill(g, g + n, 0.0);
        return FM_OK;
    }
    const bool f64 = a->precision == FM_PRECISION_PARITY_F64;
    int64_t* dcols = nullptr;
    void* dout = nullptr;
    cudaError_t e = cudaMalloc(&dcols, sizeof(int64_t) * n_cols);
    e = e ? e : cudaMalloc(&dout, n * (f64 ? 8 : 4));
    e = e ? e : cudaMemcpy(dcols, cols, sizeof(int64_t) * n_cols, cudaMemcpyHostToDevice);
    e = e ? e : launch_gather_cols(a->dW, f64, a->V, a->D, dcols, n_cols, dout, a->ctx->stream);
    std::vector<float> tmp(f64 ? 0 : n);
    if (!e) e = cudaStreamSynchronize(a->ctx->stream);
    if (!e) e = f64 ? cudaMemcpy(g, dout, n * 8, cudaMemcpyDeviceToHost)
                    : cudaMemcpy(tmp.data(), dout, n * 4, cudaMemcpyDeviceToHost);
    cudaFree(dcols);
    cudaFree(dout);
    FM_CUDA(e);
    if (!f64)
        for (size_t i = 0; i < n; ++i) g[i] = tmp[i];
    return FM_OK;
    FM_GUARD_END
}

int64_t fm_agent_version(const fm_agent* a) { return a->version; }
int64_t fm_agent_samples_accumulated(const fm_agent* a) { return a->samples; }
int fm_agent_is_active(const fm_agent* a) { return a->active ? 1 : 0; }

int fm_agent_set_clip(fm_agent* a, float clip_eps, const float* old_logp, int64_t n_rows) {
    if (int st = check_active(a, false)) return st;
    if (n_rows < 0 || (n_rows > 0 && !old_logp)) return fail(FM_ERR_INVALID_ARG, "bad old log-prob array");
    a->clip_eps = clip_eps;
    a->old_logp.clear();
    if (old_logp && clip_eps > 0.f) a->old_logp.assign(old_logp, old_logp + n_rows);  // uploaded by train_impl
    return FM_OK;
}

// DuplicateSample guard (training.hpp:396-401): the step's GradKey set.  All
// keys are checked (against the set and each other) before any is inserted.
int fm_agent_add_grad_keys(fm_agent* a, const fm_sample_key* keys, int n) {
    FM_GUARD_BEGIN
    if (n < 0 || (n > 0 && !keys)) return fail(FM_ERR_INVALID_ARG, "bad key list");
    std::vector<std::tuple<std::string, int, int, int64_t>> add;
    add.reserve(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        auto k = std::make_tuple(std::string(keys[i].input_id ? keys[i].input_id : ""), keys[i].turns, keys[i].traj,
                                 keys[i].version);
        if (a->grad_keys.count(k) || std::find(add.begin(), add.end(), k) != add.end())
            return fail(FM_ERR_DUPLICATE_SAMPLE, "gradient already cached for " + std::get<0>(k) + "/" +
                                                     std::to_string(std::get<1>(k)) + "/" +
                                                     std::to_string(std::get<2>(k)));
        add.push_back(std::move(k));
    }
    for (auto& k : add) a->grad_keys.insert(std::move(k));
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_set_shard(fm_agent* a, int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FM_ERR_INVALID_ARG, "bad shard");
    a->shard_rank = rank;
    a->shard_count = nranks;
    a->dp = nranks > 1;
    return FM_OK;
}

// ---------------------------------------------------------------------------
// DP helpers
// ---------------------------------------------------------------------------
namespace {
int ws_reserve_dpnorm(fm_ctx* c, uint64_t P) {
    Workspace& w = c->ws;
    if (w.dpn_cap >= P) return FM_OK;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(w.dpn);
    w.dpn = nullptr;
    if (dalloc(&w.dpn, P)) return fail(FM_ERR_DEVICE_OOM, "DP grad-norm scratch");
    w.dpn_cap = P;
    return FM_OK;
}

int ws_reserve_lsered(fm_ctx* c, int64_t Mpad) {
    Workspace& w = c->ws;
    if (w.lse_red_cap >= Mpad) return FM_OK;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(w.lse_red);
    w.lse_red = nullptr;
    if (dalloc(&w.lse_red, static_cast<size_t>(2 * Mpad))) return fail(FM_ERR_DEVICE_OOM, "vocabulary-gang lse scratch");
    w.lse_red_cap = Mpad;
    return FM_OK;
}

// A gang rank's partials of the peers' rows, shipped with plain NVLink copies
// into their receive slots, then the gang barrier.
int gang_copy_exchange(fm_agent* a) {
    fm_ctx* c = a->ctx;
    cudaStream_t s = c->stream;
    GangState* gs = a->gang;
    if (!a->dw_valid) FM_CUDA(cudaMemsetAsync(a->dW, 0, a->P * 4, s));
    for (int o = 0; o < gs->g; ++o) {
        if (o == gs->rank) continue;
        const size_t rows_o = static_cast<size_t>(gs->lo[o + 1] - gs->lo[o]);
        FM_CUDA(cudaMemcpyAsync(gs->peer_slot[o], static_cast<float*>(a->dW) + gs->lo[o] * a->D,
                                rows_o * a->D * 4, cudaMemcpyDeviceToDevice, s));
    }
    a->dw_valid = true;
    return gang_barrier(a);
}

// Exact DP micro-batch grad norm: dW (+)= this rank's contribution (w.dpn), the
// contributions summed over the ranks (NCCL all-reduce over NVLink) and their
// sum of squares into scal[0]; then a gang's exchange if this was the step's
// last micro-batch.
int dp_norm_finish(fm_agent* a, double* scal, bool last) {
    fm_ctx* c = a->ctx;
    cudaStream_t s = c->stream;
    Workspace& w = c->ws;
    FM_CUDA(launch_axpy_init(static_cast<float*>(a->dW), w.dpn, a->P, a->dw_valid ? 1 : 0, c->num_sms, s));
    a->dw_valid = true;
    FM_NCCL(ncclAllReduce(w.dpn, w.dpn, a->P, ncclFloat32, ncclSum, a->norm_comm->comm, s));
    FM_CUDA(launch_sumsq(w.dpn, a->P, scal, c->num_sms, s));
    count_launch(2);
    if (last && a->gang && a->gang->connected) return gang_copy_exchange(a);
    return FM_OK;
}
}  // namespace

extern "C" int fm_agent_set_dp_norms(fm_agent* a, fm_comm* comm) {
    if (comm && comm->ctx != a->ctx) return fail(FM_ERR_CONFIG_ERROR, "communicator bound to another GPU");
    if (comm && a->precision != FM_PRECISION_BF16_TC) return fail(FM_ERR_CONFIG_ERROR, "tensor-core agents only");
    a->norm_comm = comm;
    return FM_OK;
}

// ---------------------------------------------------------------------------
// the micro-batch pipeline
}  // extern "C"

namespace fm {
// ---------------------------------------------------------------------------
// K-GEMM2 over the agent's queued micro-batches (c->pend, in order): one launch
// in which every dW tile runs its units back to back (the tile stays in L2
// between them, so the step's dW is written to HBM once instead of read and
// written per micro-batch), then each micro-batch's report (its grad norm^2
// from the epilogue, its loss from K-lse) goes to the host.  exchange /
// dp_norms (one queued micro-batch): the token-shard gang's fused
// reduce-scatter / the exact DP norm of the step's micro-batch.
static int gemm2_flush(fm_agent* a, bool exchange, bool dp_norms, bool step_last) {
    fm_ctx* c = a->ctx;
    if (c->pend_agent != a || c->npend == 0) return FM_OK;
    Workspace& w = c->ws;
    cudaStream_t s = c->stream;
    if ((exchange || dp_norms) && c->npend != 1) return fail(FM_ERR_CONFIG_ERROR, "batched reduction with an exchange");
    GangState* vg = (a->gang && a->gang->connected && a->gang->vocab) ? a->gang : nullptr;
    const int64_t c0 = vg ? vg->lo[vg->rank] : 0;
    const int64_t c1 = vg ? vg->lo[vg->rank + 1] : static_cast<int64_t>(a->V);
    const uint64_t ldz = round_up(a->V, 8);
    const int nmb = c->npend;
    GemmArgs g2{};
    g2.M = static_cast<int>(c1 - c0);
    g2.N = static_cast<int>(a->D);
    g2.K = 0;
    // raster: the 256-feature column tiles of a vocab row block run together, so the
    // row block's dW stripe and A' columns stay L2-local
    g2.group_m = 1;
    g2.out = static_cast<float*>(a->dW) + static_cast<size_t>(c0) * a->D;
    g2.ld_out = static_cast<long long>(a->D);
    g2.accumulate = a->dw_valid ? 1 : 0;
    g2.dbg_krows = w.kp_cap;
    g2.nmb = nmb;
    // units of a few K iterations (C3: ~128 positions per 256-feature block) are bound by
    // their per-unit drains: share one accumulator (3.09 -> 2.63 ms at C3); long units
    // (C2: ~1,000 positions per block) keep the double-buffered per-unit drains (0.90
    // vs 0.93 ms)
    g2.snap = c->pend_rows_per_block < 512;
    for (int u = 0; u < nmb; ++u) {
        const Workspace::SegSet S = seg_set(w, c->pend[u].set);
        g2.kseg_off_b[u] = S.kseg_off;
        g2.kseg_iters_b[u] = S.kiters;
        g2.sumsq_b[u] = a->d_scalars + 2 * c->pend[u].slot;
    }
    g2.kseg_off = g2.kseg_off_b[0];
    g2.kseg_iters = g2.kseg_iters_b[0];
    g2.sumsq = g2.sumsq_b[0];
    double* scal0 = g2.sumsq_b[0];
    // exact micro-batch grad norm under DP (opt-in, fm_agent_set_dp_norms): GEMM2 writes
    // this rank's contribution to a scratch, which is added to dW, all-reduced and
    // measured (training.hpp:417); a gang's exchange then runs as plain copies
    if (dp_norms) {
        if (int st = ws_reserve_dpnorm(c, a->P)) return st;
        g2.out = w.dpn;
        g2.accumulate = 0;
        g2.sumsq = nullptr;
        g2.sumsq_b[0] = nullptr;
    }
    if (exchange) {  // last micro-batch of the step: reduce-scatter inside the epilogue
        GangState* gs = a->gang;
        g2.xg = gs->g;
        g2.xrank = gs->rank;
        for (int o = 0; o <= gs->g; ++o) g2.xlo[o] = static_cast<int>(gs->lo[o]);
        for (int o = 0; o < gs->g; ++o) g2.xpeer[o] = gs->peer_slot[o];
    }
    {
        KScope k(c, K_GEMM2, s);
        const uint64_t mc = static_cast<uint64_t>(c1 - c0);
        if (mc > 0) {
            GemmMaps maps{};
            for (int u = 0; u < nmb; ++u) {
                const Workspace::SegSet S = seg_set(w, c->pend[u].set);
                if (!make_tmap_bf16_kmajor(&maps.a[u], S.aseg + c0, static_cast<uint64_t>(w.kp_cap), mc, 64, ldz) ||
                    !make_tmap_bf16_kmajor(&maps.b[u], S.bseg, static_cast<uint64_t>(w.kp_cap), 256, 64))
                    return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
            }
            if (!make_tmap_f32_out(&maps.c, g2.out, mc, a->D, a->D))
                return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
            FM_CUDA(gemm_kseg_launch(maps, g2, c->num_sms, s));
            count_launch();
        }
        // each micro-batch's grad norm^2 over the whole vocabulary (training.hpp:417)
        if (vg)
            for (int u = 0; u < nmb; ++u)
                FM_NCCL(ncclAllReduce(g2.sumsq_b[u], g2.sumsq_b[u], 1, ncclFloat64, ncclSum, gang_comm(vg), s));
    }
    if (exchange) {
        a->dw_valid = true;
        if (int st = gang_barrier(a)) return st;  // every rank's partials have landed
    }
    if (dp_norms) {
        if (int st = dp_norm_finish(a, scal0, step_last)) return st;
    }
    a->dw_valid = true;
    for (int u = 0; u < nmb; ++u) {
        const int slot = c->pend[u].slot;
        FM_CUDA(cudaMemcpyAsync(a->h_scalars + 2 * slot, a->d_scalars + 2 * slot, 2 * sizeof(double),
                                cudaMemcpyDeviceToHost, s));
        FM_CUDA(cudaEventRecord(a->ev[slot], s));
    }
    c->npend = 0;
    c->pend_agent = nullptr;
    return FM_OK;
}

int agent_flush(fm_agent* a) {
    if (!a->ctx || a->ctx->pend_agent != a) return FM_OK;
    if (int st = set_dev(a->ctx)) return st;
    return gemm2_flush(a, false, false, false);
}

int ctx_flush(fm_ctx* c) { return c->pend_agent ? agent_flush(c->pend_agent) : FM_OK; }
}  // namespace fm

extern "C" {

// ---------------------------------------------------------------------------
// hsd: host descriptors (staged H2D), or dsd: descriptors already in HBM (the
// on-device experience table's poll), ready when `dsd_ready` completes.
static int train_impl(fm_agent* a, const SampleDesc* hsd, int n, int64_t M_total, int64_t G, int64_t* ticket_out,
                      const SampleDesc* dsd = nullptr, cudaEvent_t dsd_ready = nullptr) {
    // data-parallel gang: this rank trains rows [row_lo, row_hi) of the micro-batch
    const int64_t row_lo = M_total * a->shard_rank / a->shard_count;
    const int64_t row_hi = M_total * (a->shard_rank + 1) / a->shard_count;
    const int64_t M = row_hi - row_lo;
    fm_ctx* c = a->ctx;
    Workspace& w = c->ws;
    cudaStream_t s = c->stream;
    const bool tc = a->precision == FM_PRECISION_BF16_TC;
    const bool clip = !a->old_logp.empty() && a->clip_eps > 0.f;
    if (clip && static_cast<int64_t>(a->old_logp.size()) != M_total)
        return fail(FM_ERR_INVALID_ARG, "old log-probs given for " + std::to_string(a->old_logp.size()) +
                                            " rows, the micro-batch has " + std::to_string(M_total));
    const int64_t Mpad = tc ? static_cast<int64_t>(round_up(static_cast<uint64_t>(M), 128)) : M;
    // the workspace's segment sets serve one agent's deferred K-GEMM2 at a time
    if (c->pend_agent && c->pend_agent != a)
        if (int st = agent_flush(c->pend_agent)) return st;
    if (tc) {
        if (int st = ws_reserve_tc(c, std::max<int64_t>(Mpad, 128), a->V, a->D, n)) return st;
    } else {
        if (int st = ws_reserve_parity(c, M, a->V, a->P)) return st;
    }
    if (int st = ws_reserve_sd(c, n)) return st;
    if (dsd) {
        // descriptors built in HBM by the device poll: order after it, copy D2D
        if (dsd_ready) FM_CUDA(cudaStreamWaitEvent(s, dsd_ready, 0));
        if (n) FM_CUDA(cudaMemcpyAsync(w.sd, dsd, sizeof(SampleDesc) * n, cudaMemcpyDeviceToDevice, s));
    } else {
        // descriptors -> device through pinned staging
        uint8_t* stg;
        cudaEvent_t sev;
        if (int st = staging_acquire(c, sizeof(SampleDesc) * n, &stg, &sev)) return st;
        std::memcpy(stg, hsd, sizeof(SampleDesc) * n);
        FM_CUDA(cudaMemcpyAsync(w.sd, stg, sizeof(SampleDesc) * n, cudaMemcpyHostToDevice, s));
        FM_CUDA(cudaEventRecord(sev, s));
    }
    if (clip) {  // after the workspace reserve (which may reallocate)
        if (w.old_logp_cap < M_total) {
            FM_CUDA(cudaStreamSynchronize(s));
            cudaFree(w.old_logp);
            w.old_logp = nullptr;
            if (dalloc(&w.old_logp, static_cast<size_t>(M_total))) return fail(FM_ERR_DEVICE_OOM, "old log-probs");
            w.old_logp_cap = M_total;
        }
        uint8_t* stg;
        cudaEvent_t sev;
        if (int st = staging_acquire(c, M_total * 4, &stg, &sev)) return st;
        std::memcpy(stg, a->old_logp.data(), M_total * 4);
        FM_CUDA(cudaMemcpyAsync(w.old_logp, stg, M_total * 4, cudaMemcpyHostToDevice, s));
        FM_CUDA(cudaEventRecord(sev, s));
    }

    const int64_t ticket = a->next_ticket++;
    const int slot = static_cast<int>(ticket % kReportRing);
    if (ticket >= kReportRing) FM_CUDA(cudaEventSynchronize(a->ev[slot]));  // slot reuse
    double* scal = a->d_scalars + 2 * slot;
    FM_CUDA(cudaMemsetAsync(scal, 0, 2 * sizeof(double), s));
    RowBuffers rows = row_buffers(w);
    bool queued = false;  // the report is produced by the (possibly deferred) K-GEMM2

    if (M > 0) {
        if (tc) {
            const uint64_t ldz = round_up(a->V, 8);
            const int64_t Qcap = Mpad + 3 * static_cast<int64_t>(n);
            const int nblk = static_cast<int>((a->D + 255) / 256);
            // vocabulary-parallel gang: this rank's columns [c0, c1) of every row
            GangState* vg = (a->gang && a->gang->connected && a->gang->vocab) ? a->gang : nullptr;
            const int64_t c0 = vg ? vg->lo[vg->rank] : 0;
            const int64_t c1 = vg ? vg->lo[vg->rank + 1] : static_cast<int64_t>(a->V);
            if (!a->fmax_valid) {
                // per-feature maxima of the shadow (the rows' softmax bounds), once per
                // shadow generation (update, set_weights, swap-in, migration); a vocabulary
                // gang takes the max over its ranks' column ranges
                KScope k(c, K_GATHER, s);
                FM_CUDA(launch_fmax(a->W16 + c0, static_cast<int64_t>(a->D), c1 - c0,
                                    static_cast<int64_t>(w16_ld(a)), a->fmax, s));
                if (vg) FM_NCCL(ncclAllReduce(a->fmax, a->fmax, a->D, ncclFloat32, ncclMax, gang_comm(vg), s));
                a->fmax_valid = true;
                count_launch();
            }
            // this micro-batch's segment set: the next free one while the step's reductions
            // are batched (a DP exchange / exact DP norms need each micro-batch's dW at once)
            const bool dp_norms = a->norm_comm != nullptr;
            if (dp_norms && vg) return fail(FM_ERR_CONFIG_ERROR, "a vocabulary gang reports exact norms already");
            const bool step_last = a->samples + n == G;
            const bool batch = !dp_norms && !(a->gang && !vg) && w.nsets > 1;
            if (!batch && c->npend)
                if (int st = agent_flush(a)) return st;
            const int kset = c->npend;
            const Workspace::SegSet S = seg_set(w, kset);
            rows.fmax = a->fmax;
            rows.zact = w.zact;
            rows.lossw = w.lossw;
            rows.w16t = a->W16 + c0;
            rows.ldw = static_cast<int64_t>(w16_ld(a));
            rows.col_base = c0;
            rows.ncols = c1 - c0;
            {
                // K-gather (rows, q0, bounds) + K-pos (position features) + K-pslot (segment
                // slots, one-hot B')
                KScope k(c, K_GATHER, s);
                FM_CUDA(launch_gather(c->arena, w.sd, n, row_lo, M, Mpad, G, a->D, rows, s));
                FM_CUDA(launch_positions(c->arena, w.sd, n, row_lo, M, a->D, w.pos_feat, Qcap, s));
                FM_CUDA(launch_pslots(w.pos_feat, Qcap, nblk, w.kcount, S.kseg_off, S.kiters, w.pos_slot, S.bseg,
                                      w.kp_cap, w.kseg_rows, s));
                count_launch(5);  // K-gather, K-pos, K-pslot count / scan / place
            }
            BandArgs ba{};
            ba.w16t = a->W16 + c0;
            ba.ldw = static_cast<int64_t>(w16_ld(a));
            ba.zero_row = w.zero_row;
            ba.V = c1 - c0;
            ba.col_base = c0;
            ba.pos_feat = w.pos_feat;
            ba.q0 = w.q0;
            ba.action = w.action;
            ba.rscale = w.rscale;
            ba.mrow = w.mrow;
            ba.M = M;
            ba.ld_stats = Mpad;
            ba.stats = w.stats;
            ba.stats_ld = band_stats_ld(c1 - c0);
            ba.lse = w.lse;
            ba.coef_eff = w.coef_eff;
            ba.pos_slot = w.pos_slot;
            ba.aseg = S.aseg + c0;
            ba.ld_a = static_cast<int64_t>(ldz);
            ba.dbg_kp = w.kp_cap;
            ba.dbg_D = static_cast<int64_t>(a->D);
            const bool cols = c1 > c0;  // (a vocabulary-gang rank may own no columns)
            {
                // K-stats: per-(row, consumer warp) partial sums of exp(z - bound)
                KScope k(c, K_STATS, s);
                if (cols) FM_CUDA(launch_band(ba, false, s));
            }
            {
                KScope k(c, K_LSE, s);
                LseArgs L{w.stats, ba.stats_ld, M, Mpad, static_cast<int64_t>(a->V), w.sd, G, rows,
                          clip ? w.old_logp : nullptr, row_lo, a->clip_eps, scal + 1};
                if (vg) {
                    // vocabulary gang: per row (sum over my columns, taken logit or 0), summed
                    // over the gang, then every rank finishes the same lse / log-prob / coef
                    if (int st = ws_reserve_lsered(c, Mpad)) return st;
                    LseArgs P = L;
                    P.partial_out = w.lse_red;
                    P.loss_acc = nullptr;
                    if (cols) {
                        FM_CUDA(launch_lse(P, s));
                    } else {
                        FM_CUDA(cudaMemsetAsync(w.lse_red, 0, 2 * Mpad * 4, s));
                    }
                    FM_NCCL(ncclAllReduce(w.lse_red, w.lse_red, 2 * Mpad, ncclFloat32, ncclSum, gang_comm(vg), s));
                    L.sum_in = w.lse_red;
                }
                FM_CUDA(launch_lse(L, s));
            }
            // swap copies (fm_agent_suspend / fm_agent_activate) may start here: beside the
            // streaming K-band / K-GEMM2 / next K-stats rather than the latency-bound K-lse
            // (0.013 -> 0.09 ms next to a 2.4 GB copy-engine copy)
            FM_CUDA(cudaEventRecord(c->ev_gemm, s));
            c->gemm_seq = ++c->op_seq;
            if (cols) {
                // K-band: per-position gradient rows H into the feature blocks' A' segments
                KScope k(c, K_BAND, s);
                FM_CUDA(launch_band(ba, true, s));
            }
            // K-GEMM2 (dW[v][f] (+)= sum over block(f)'s positions of H[q][v] * onehot[q][f]):
            // queued; it runs when the batch is full, at the step's last micro-batch, or when
            // anything needs this agent's dW or reports (check_active, sync, poll)
            c->pend[c->npend++] = fm_ctx::PendingMB{kset, slot};
            c->pend_agent = a;
            c->pend_rows_per_block = Qcap / nblk;
            queued = true;
            count_launch(3);
            if (!batch || c->npend == w.nsets || step_last) {
                const bool exchange = !dp_norms && !vg && a->gang && a->gang->connected && step_last;
                if (int st = gemm2_flush(a, exchange, dp_norms, step_last)) return st;
            }
        } else {
            FM_CUDA(launch_gather(c->arena, w.sd, n, row_lo, M, M, G, a->D, rows, s));
            if (!a->dw_valid) FM_CUDA(cudaMemsetAsync(a->dW, 0, a->P * 8, s));
            KScope k(c, K_PARITY, s);
            FM_CUDA(launch_parity_rows(a->W, a->V, a->D, M, rows, w.sd, G, w.zscratch, w.dWmb, w.logp64,
                                       scal + 1, s));
            FM_CUDA(launch_parity_fold(static_cast<double*>(a->dW), w.dWmb, a->P, scal, c->num_sms, s));
            count_launch(3);
            a->dw_valid = true;
        }
    } else if (tc && a->norm_comm) {
        // no rows here: a zero contribution still joins the collective
        if (int st = ws_reserve_dpnorm(c, a->P)) return st;
        FM_CUDA(cudaMemsetAsync(w.dpn, 0, a->P * 4, s));
        if (int st = dp_norm_finish(a, scal, a->samples + n == G)) return st;
    } else if (a->gang && a->gang->connected && !a->gang->vocab && a->samples + n == G) {
        // this rank got no rows of the step's last micro-batch: ship its partials
        // for the peers' rows with plain NVLink copies, then join the barrier
        if (int st = gang_copy_exchange(a)) return st;
    }
    a->old_logp.clear();  // old log-probs apply to one micro-batch
    a->last_rows = M;
    a->last_seq = ++c->op_seq;  // its own K-stats mark precedes this micro-batch's GEMM2
    if (!queued) {
        FM_CUDA(cudaMemcpyAsync(a->h_scalars + 2 * slot, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        FM_CUDA(cudaEventRecord(a->ev[slot], s));
    }
    a->rep_tokens[slot] = M;
    a->rep_bs[slot] = n;
    a->samples += n;
    if (ticket_out) *ticket_out = ticket;
    return FM_OK;
}

int fm_train_micro_batch(fm_agent* a, const fm_sample* samples, int n, int64_t G, int64_t* ticket_out) {
    FM_GUARD_BEGIN
    if (int st = check_active(a, false)) return st;
    if (n < 0 || (n > 0 && !samples)) return fail(FM_ERR_INVALID_ARG, "bad sample list");
    if (G <= 0) return fail(FM_ERR_CONFIG_ERROR, "global batch must be positive");
    if (int st = set_dev(a->ctx)) return st;
    std::vector<SampleDesc> sd(static_cast<size_t>(n));
    int64_t rows = 0;
    for (int i = 0; i < n; ++i) {
        bool f1, f2;
        const uint64_t np = arena_token_count(a->ctx, samples[i].prompt_off, &f1);
        const uint64_t nr = arena_token_count(a->ctx, samples[i].response_off, &f2);
        if (!f1 || !f2) return fail(FM_ERR_KEY_NOT_FOUND, "sample payload not in this GPU's token arena");
        sd[i].prompt_off = static_cast<int64_t>(samples[i].prompt_off);
        sd[i].resp_off = static_cast<int64_t>(samples[i].response_off);
        sd[i].prompt_n = static_cast<int32_t>(np);
        sd[i].resp_n = static_cast<int32_t>(nr);
        sd[i].row_start = rows;
        sd[i].adv = samples[i].advantage;
        rows += static_cast<int64_t>(nr);
    }
    return train_impl(a, sd.data(), n, rows, G, ticket_out);
    FM_GUARD_END
}

// End-to-end variant: host payloads are staged through pinned memory into a
// reusable arena region inside the call (H2D on the compute stream).
int fm_train_micro_batch_host(fm_agent* a, const fm_host_sample* samples, int n, int64_t G, int64_t* ticket_out) {
    FM_GUARD_BEGIN
    if (int st = check_active(a, false)) return st;
    if (n < 0 || (n > 0 && !samples)) return fail(FM_ERR_INVALID_ARG, "bad sample list");
    if (G <= 0) return fail(FM_ERR_CONFIG_ERROR, "global batch must be positive");
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    std::vector<SampleDesc> sd(static_cast<size_t>(n));
    uint64_t bytes = 0;
    int64_t rows = 0;
    for (int i = 0; i < n; ++i) {
        uint64_t np, nr;
        std::memcpy(&np, samples[i].prompt, 8);
        std::memcpy(&nr, samples[i].response, 8);
        sd[i].prompt_off = static_cast<int64_t>(bytes);
        bytes += round_up(8 + 8 * np, 16);
        sd[i].resp_off = static_cast<int64_t>(bytes);
        bytes += round_up(8 + 8 * nr, 16);
        sd[i].prompt_n = static_cast<int32_t>(np);
        sd[i].resp_n = static_cast<int32_t>(nr);
        sd[i].row_start = rows;
        sd[i].adv = samples[i].advantage;
        rows += static_cast<int64_t>(nr);
    }
    // a dedicated region at the arena tail, reused call after call (stream-ordered)
    if (c->e2e_cap < bytes || c->e2e_off + c->e2e_cap != c->arena_used) {
        const uint64_t off = round_up(c->arena_used, 256);
        const uint64_t cap = std::max<uint64_t>(bytes, 1 << 20);
        if (off + cap > c->arena_cap)
            if (int st = fm_ctx_reserve(c, off + cap, 0, 0, 0)) return st;
        c->e2e_off = off;
        c->e2e_cap = cap;
        c->arena_used = off + cap;
    }
    uint8_t* stg;
    cudaEvent_t ev;
    if (int st = staging_acquire(c, bytes, &stg, &ev)) return st;
    for (int i = 0; i < n; ++i) {
        std::memcpy(stg + sd[i].prompt_off, samples[i].prompt, 8 + 8 * static_cast<uint64_t>(sd[i].prompt_n));
        std::memcpy(stg + sd[i].resp_off, samples[i].response, 8 + 8 * static_cast<uint64_t>(sd[i].resp_n));
        sd[i].prompt_off += static_cast<int64_t>(c->e2e_off);
        sd[i].resp_off += static_cast<int64_t>(c->e2e_off);
    }
    FM_CUDA(cudaMemcpyAsync(c->arena + c->e2e_off, stg, bytes, cudaMemcpyHostToDevice, c->stream));
    FM_CUDA(cudaEventRecord(ev, c->stream));
    return train_impl(a, sd.data(), n, rows, G, ticket_out);
    FM_GUARD_END
}

int fm_agent_read_logp(fm_agent* a, double* out, int64_t n_rows) {
    FM_GUARD_BEGIN
    if (int st = check_active(a, false)) return st;
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    const int64_t n = std::min<int64_t>(n_rows, a->last_rows);
    if (a->precision == FM_PRECISION_PARITY_F64) {
        FM_CUDA(cudaMemcpy(out, c->ws.logp64, n * 8, cudaMemcpyDeviceToHost));
    } else {
        std::vector<float> t(static_cast<size_t>(n));
        FM_CUDA(cudaMemcpy(t.data(), c->ws.logp, n * 4, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) out[i] = t[static_cast<size_t>(i)];
    }
    return FM_OK;
    FM_GUARD_END
}

int fm_debug_read_rows(fm_ctx* c, int64_t n, int32_t* action, int32_t* ctx4, int32_t* n_ctx, int32_t* sample,
                       float* coef) {
    if (int st = set_dev(c)) return st;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    if (n > c->ws.rows_cap) return fail(FM_ERR_INVALID_ARG, "more rows than the workspace holds");
    if (action) FM_CUDA(cudaMemcpy(action, c->ws.action, n * 4, cudaMemcpyDeviceToHost));
    if (ctx4) FM_CUDA(cudaMemcpy(ctx4, c->ws.ctx4, n * 16, cudaMemcpyDeviceToHost));
    if (n_ctx) FM_CUDA(cudaMemcpy(n_ctx, c->ws.n_ctx, n * 4, cudaMemcpyDeviceToHost));
    if (sample) FM_CUDA(cudaMemcpy(sample, c->ws.sample, n * 4, cudaMemcpyDeviceToHost));
    if (coef) FM_CUDA(cudaMemcpy(coef, c->ws.coef, n * 4, cudaMemcpyDeviceToHost));
    return FM_OK;
}

int fm_debug_read_positions(fm_ctx* c, int64_t n_rows, int32_t* q0, int64_t n_pos, int32_t* feat, int32_t* slot) {
    if (int st = set_dev(c)) return st;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    if (n_rows > c->ws.rows_cap || n_pos > c->ws.pos_cap || !c->ws.q0)
        return fail(FM_ERR_INVALID_ARG, "more rows / positions than the workspace holds");
    if (q0) FM_CUDA(cudaMemcpy(q0, c->ws.q0, n_rows * 4, cudaMemcpyDeviceToHost));
    if (feat) FM_CUDA(cudaMemcpy(feat, c->ws.pos_feat, n_pos * 4, cudaMemcpyDeviceToHost));
    if (slot) FM_CUDA(cudaMemcpy(slot, c->ws.pos_slot, n_pos * 4, cudaMemcpyDeviceToHost));
    return FM_OK;
}

int fm_agent_sync(fm_agent* a) {
    if (!a->ctx) return FM_OK;
    if (int st = set_dev(a->ctx)) return st;
    if (int st = agent_flush(a)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    return FM_OK;
}

int fm_agent_poll_report(fm_agent* a, int64_t ticket, fm_report* out) {
    if (ticket < 0 || ticket >= a->next_ticket || ticket < a->next_ticket - kReportRing)
        return fail(FM_ERR_INVALID_ARG, "unknown or expired ticket");
    const int slot = static_cast<int>(ticket % kReportRing);
    if (a->ctx && a->ctx->pend_agent == a) {  // its K-GEMM2 is still queued: run it now
        for (int u = 0; u < a->ctx->npend; ++u)
            if (a->ctx->pend[u].slot == slot) {
                if (int st = agent_flush(a)) return st;
                break;
            }
    }
    const cudaError_t q = cudaEventQuery(a->ev[slot]);
    if (q == cudaErrorNotReady) return 0;
    if (q != cudaSuccess) return fail(FM_ERR_CUDA, cudaGetErrorString(q));
    out->ticket = ticket;
    out->tokens = a->rep_tokens[slot];
    out->batch_size = a->rep_bs[slot];
    // under DP the rank's own sum of squares is not the micro-batch's: NaN unless the
    // exact reduction is on (fm_agent_set_dp_norms)
    out->grad_norm = (a->dp && !a->norm_comm) ? NAN : std::sqrt(a->h_scalars[2 * slot]);
    out->loss = a->h_scalars[2 * slot + 1];
    return 1;
}


// apply_global_update; with park != 0 (device tier, tensor-core agent, no gang)
// K-adam writes the new W / m / v / W16^T straight into the agent's
// parking buffer and the agent is suspended — the swap-out fused into the
// optimizer (no copy-out pass).
static int apply_update_impl(fm_agent* a, int64_t G, double lr, double b1, double b2, double eps,
                             double* grad_norm_out, int64_t* version_out, bool park) {
    if (int st = check_active(a)) return st;
    if (a->samples != G)
        return fail(FM_ERR_INCOMPLETE_BATCH,
                    a->name + " accumulated " + std::to_string(a->samples) + " of " + std::to_string(G));
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    cudaStream_t s = c->stream;
    AdamDst dst{};
    uint8_t* pk = nullptr;
    if (park) {
        if (a->gang) return fail(FM_ERR_BUSY_GROUP, a->name + " is attached to a DP gang (fm_gang_detach first)");
        if (a->precision != FM_PRECISION_BF16_TC || !a->W16)
            return fail(FM_ERR_INVALID_ARG, "update-and-park needs a tensor-core agent");
        if (int st = park_reserve(a, c, FM_TIER_DEVICE, c->device, park_bytes_for(a))) return st;
        pk = static_cast<uint8_t*>(a->park);
        dst = AdamDst{reinterpret_cast<double*>(pk), reinterpret_cast<float*>(pk + a->P * 8),
                      reinterpret_cast<float*>(pk + a->P * 12)};
    }
    if (!a->dw_valid) FM_CUDA(cudaMemsetAsync(a->dW, 0, a->P * dw_elem(a), s));
    a->step += 1;
    const double bc1 = 1.0 - std::pow(b1, static_cast<double>(a->step));  // training.hpp:42-43
    const double bc2 = 1.0 - std::pow(b2, static_cast<double>(a->step));
    FM_CUDA(cudaMemsetAsync(a->d_upd, 0, sizeof(double), s));
    KScope ks(c, K_ADAM, s);
    const ShardPeers none{};
    if (a->precision == FM_PRECISION_PARITY_F64) {
        FM_CUDA(launch_adam<double>(a->W, a->m, a->v, static_cast<double*>(a->dW), a->V, a->D, 0, a->V, nullptr, 0,
                                    nullptr, 0, none, lr, b1, b2, eps, bc1, bc2, 1, a->d_upd, c->num_sms, s));
    } else if (a->gang && a->gang->connected) {
        // sharded Adam over this rank's rows (gradient = local partial + the peers'
        // receive slots); the new W16^T columns of those rows go to every replica
        GangState* gs = a->gang;
        const uint64_t r0 = static_cast<uint64_t>(gs->lo[gs->rank]), r1 = static_cast<uint64_t>(gs->lo[gs->rank + 1]);
        // (vocabulary gang: the rows' gradient is complete here and only this rank reads
        // their W16^T columns — no receive slots, no peer writes)
        ShardPeers peers{};
        if (!gs->vocab)
            for (int o = 0; o < gs->g; ++o)
                if (o != gs->rank) peers.w16t[peers.n++] = gs->peer_w16[o];
        FM_CUDA(launch_adam<float>(a->W, a->m, a->v, static_cast<float*>(a->dW), a->V, a->D, r0, r1,
                                   gs->vocab ? nullptr : gs->recv, gs->vocab ? 0 : gs->g - 1, a->W16, w16_ld(a),
                                   peers, lr, b1, b2, eps, bc1, bc2, 0, a->d_upd, c->num_sms, s));
        // global grad norm^2; doubles as the barrier after the peers' W16^T writes
        FM_NCCL(ncclAllReduce(a->d_upd, a->d_upd, 1, ncclFloat64, ncclSum, gang_comm(gs), s));
    } else {
        // the next step's first GEMM2 overwrites dW, so no zeroing pass here; with park the
        // new state goes straight into the parking buffer
        const size_t dwe = dw_elem(a);
        __nv_bfloat16* w16_out = park ? reinterpret_cast<__nv_bfloat16*>(pk + a->P * (16 + dwe)) : a->W16;
        FM_CUDA(launch_adam<float>(a->W, a->m, a->v, static_cast<float*>(a->dW), a->V, a->D, 0, a->V, nullptr, 0,
                                   w16_out, w16_ld(a), none, lr, b1, b2, eps, bc1, bc2, 0, a->d_upd, c->num_sms, s,
                                   park ? &dst : nullptr));
    }
    count_launch();
    a->dw_valid = false;
    a->samples = 0;
    a->version += 1;
    a->grad_keys.clear();
    a->fmax_valid = false;  // the shadow changed
    FM_CUDA(cudaMemcpyAsync(a->h_upd, a->d_upd, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (park) {
        // the parked state is complete when K-adam is: release the slot behind it
        a->park_w16 = true;
        FM_CUDA(cudaEventRecord(a->ev_out, s));
        agent_free_device(a, s);
        a->active = false;
        a->ctx = nullptr;
    }
    if (grad_norm_out) {
        FM_CUDA(cudaStreamSynchronize(s));
        *grad_norm_out = std::sqrt(*a->h_upd);
    }
    if (version_out) *version_out = a->version;
    return FM_OK;
}

int fm_apply_update(fm_agent* a, int64_t G, double lr, double b1, double b2, double eps, double* grad_norm_out,
                    int64_t* version_out) {
    FM_GUARD_BEGIN
    return apply_update_impl(a, G, lr, b1, b2, eps, grad_norm_out, version_out, false);
    FM_GUARD_END
}

int fm_apply_update_park(fm_agent* a, int64_t G, double lr, double b1, double b2, double eps, double* grad_norm_out,
                         int64_t* version_out) {
    FM_GUARD_BEGIN
    return apply_update_impl(a, G, lr, b1, b2, eps, grad_norm_out, version_out, true);
    FM_GUARD_END
}

}  // extern "C"

extern "C" {
// ---------------------------------------------------------------------------
// GRPO advantages on device
// ---------------------------------------------------------------------------
int fm_group_advantages(fm_ctx* c, const double* rewards, const int32_t* seg_off, int nseg, double eps, double* out) {
    FM_GUARD_BEGIN
    if (nseg <= 0) return FM_OK;
    if (int st = set_dev(c)) return st;
    const int n = seg_off[nseg];
    if (n <= 0) return FM_OK;
    double *dr = nullptr, *dout = nullptr;
    int32_t* doff = nullptr;
    cudaStream_t s = c->stream;
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dr), n * 8, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dout), n * 8, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&doff), (nseg + 1) * 4, s));
    FM_CUDA(cudaMemcpyAsync(dr, rewards, n * 8, cudaMemcpyHostToDevice, s));
    FM_CUDA(cudaMemcpyAsync(doff, seg_off, (nseg + 1) * 4, cudaMemcpyHostToDevice, s));
    FM_CUDA(cudaMemsetAsync(dout, 0, n * 8, s));
    FM_CUDA(launch_group_advantages(dr, doff, nseg, eps, dout, s));
    count_launch();
    FM_CUDA(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, s));
    FM_CUDA(cudaFreeAsync(dr, s));
    FM_CUDA(cudaFreeAsync(dout, s));
    FM_CUDA(cudaFreeAsync(doff, s));
    FM_CUDA(cudaStreamSynchronize(s));
    return FM_OK;
    FM_GUARD_END
}

}  // extern "C"

// ---------------------------------------------------------------------------
// internal hooks for the on-device experience table (fm_dtable.cu)
// ---------------------------------------------------------------------------
namespace fm {
int ctx_device(const fm_ctx* c) { return c->device; }
cudaStream_t ctx_stream(const fm_ctx* c) { return c->stream; }
uint8_t* ctx_arena(const fm_ctx* c) { return c->arena; }
int ctx_staging(fm_ctx* c, size_t bytes, uint8_t** out, cudaEvent_t* ev) { return staging_acquire(c, bytes, out, ev); }
fm_ctx* agent_ctx(const fm_agent* a) { return a->ctx; }
int agent_check_active(fm_agent* a) { return check_active(a, false); }  // (train entry: no flush)

int ctx_arena_alloc(fm_ctx* c, uint64_t bytes, uint64_t* off_out) {
    if (int st = set_dev(c)) return st;
    const uint64_t off = round_up(c->arena_used, 16);
    if (off + bytes > c->arena_cap) {
        const uint64_t cap = std::max<uint64_t>(2 * c->arena_cap, off + bytes + (64u << 20));
        if (int st = fm_ctx_reserve(c, cap, 0, 0, 0)) return st;
    }
    c->arena_used = off + bytes;
    *off_out = off;
    return FM_OK;
}

int train_device_desc(fm_agent* a, const SampleDesc* dsd, int n, int64_t M_total, int64_t G, cudaEvent_t ready,
                      int64_t* ticket_out) {
    FM_GUARD_BEGIN
    if (int st = check_active(a, false)) return st;
    if (G <= 0) return fail(FM_ERR_CONFIG_ERROR, "global batch must be positive");
    if (int st = set_dev(a->ctx)) return st;
    return train_impl(a, nullptr, n, M_total, G, ticket_out, dsd, ready);
    FM_GUARD_END
}

// K-generate into device buffers (caller frees them on ctx's stream)
int generate_device(fm_ctx* c, const fm_weights* w, const int32_t* prompts, const int32_t* prompt_off, int n,
                    int max_tokens, const uint64_t* seeds, GenBuffers* out) {
    if (w->dtype != 0 && w->dtype != 3)
        return fail(FM_ERR_CONFIG_ERROR, "generation reads f64 weights (publish with dtype 0 or 3)");
    if (w->device != c->device) return fail(FM_ERR_CONFIG_ERROR, "weights live on another GPU (fm_weights_get)");
    if (int st = set_dev(c)) return st;
    cudaStream_t s = c->stream;
    const int np = prompt_off[n];
    const size_t nt = static_cast<size_t>(n) * max_tokens;
    *out = GenBuffers{};
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out->prompts), std::max(np, 1) * 4, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out->prompt_off), (n + 1) * 4, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out->seeds), n * 8, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out->z), static_cast<size_t>(n) * w->rows * 8, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out->tok), nt * 4, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out->logp), nt * 8, s));
    FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out->len), n * 4, s));
    uint8_t* stg;
    cudaEvent_t ev;
    const size_t bytes = static_cast<size_t>(np) * 4 + (n + 1) * 4 + n * 8;
    if (int st = staging_acquire(c, bytes, &stg, &ev)) return st;
    std::memcpy(stg, seeds, n * 8);
    std::memcpy(stg + n * 8, prompt_off, (n + 1) * 4);
    if (np) std::memcpy(stg + n * 8 + (n + 1) * 4, prompts, np * 4);
    FM_CUDA(cudaMemcpyAsync(out->seeds, stg, n * 8, cudaMemcpyHostToDevice, s));
    FM_CUDA(cudaMemcpyAsync(out->prompt_off, stg + n * 8, (n + 1) * 4, cudaMemcpyHostToDevice, s));
    if (np) FM_CUDA(cudaMemcpyAsync(out->prompts, stg + n * 8 + (n + 1) * 4, np * 4, cudaMemcpyHostToDevice, s));
    FM_CUDA(cudaEventRecord(ev, s));
    FM_CUDA(launch_generate(static_cast<const double*>(w->buf), w->dtype == 3, w->rows, w->cols, out->prompts,
                            out->prompt_off, n, max_tokens, out->seeds, out->z, out->tok, out->logp, out->len, s));
    count_launch();
    return FM_OK;
}

int free_gen_buffers(fm_ctx* c, GenBuffers* g) {
    for (void* p : {static_cast<void*>(g->prompts), static_cast<void*>(g->prompt_off), static_cast<void*>(g->seeds),
                    static_cast<void*>(g->z), static_cast<void*>(g->tok), static_cast<void*>(g->logp),
                    static_cast<void*>(g->len)})
        if (p) FM_CUDA(cudaFreeAsync(p, c->stream));
    *g = GenBuffers{};
    return FM_OK;
}
}  // namespace fm

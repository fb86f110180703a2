// fm_runtime.cu — C ABI implementation: device contexts, the token arena,
// per-agent trainer state, the micro-batch pipeline
//   K-gather -> K-GEMM1 (tcgen05; log-softmax numerator in the epilogue, K-lse
//   in the grid tail) -> K-GEMM2 (tcgen05; softmax gradient folded into its
//   operands)
// (or the fp64 parity pipeline; FM_LOSS_FOLD=0 / FM_LSE_FUSED=0 restore the
// separate K-softmax-grad / K-lse launches), the fused Adam update, training-
// state swap and migration, DP gangs (fused reduce-scatter / NCCL all-reduce),
// weight publish and the PolicyState wire format.
//
// Memory layout in HBM: every agent matrix is row-major
// [V][D] (row = vocab id, col = feature; tensor.hpp:13-22):
//   W    f64   master weights            (8 B/param)
//   m, v f32   Adam moments              (4+4 B/param)
//   dW   f32   gradient accumulator      (4 B/param; f64 in parity mode)
//   W16  bf16  GEMM shadow of W          (2 B/param; tensor-core mode only)
// Per-GPU workspace, sized for the largest micro-batch (Mpad = rows rounded
// up to 128): packed rows, Phic [Mpad][D] / Phic^T [D][Mpad] bf16 (integer
// counts; K-lse rescales Phic^T's entries per row), p~^T [V][Mpad] bf16
// (GEMM1's output = GEMM2's A operand), softmax partials [Mpad][V/256].
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "fm_gemm.h"
#include "fm_internal.h"
#include "fm_kernels.h"

using namespace fm;

namespace {

constexpr int kReportRing = 256;
constexpr int kStagingSlots = 4;

// ---- driver entry point for cuTensorMapEncodeTiled (no -lcuda link) -------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

template <typename T>
cudaError_t dalloc(T** p, size_t n) {
    *p = nullptr;
    if (n == 0) return cudaSuccess;
    return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

}  // namespace

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

// ===========================================================================
// context
// ===========================================================================
struct Workspace {
    int64_t rows_cap = 0;  // Mpad capacity
    uint64_t vocab_cap = 0, feat_cap = 0;
    int32_t* action = nullptr;
    int4* ctx4 = nullptr;
    int4* feat4 = nullptr;
    uint32_t* cnt4 = nullptr;
    int32_t* n_ctx = nullptr;
    int32_t* sample = nullptr;
    float *coef = nullptr, *rscale = nullptr, *lse = nullptr, *logp = nullptr, *coef_eff = nullptr;
    float* old_logp = nullptr;
    __nv_bfloat16 *phic = nullptr, *phict = nullptr, *gt = nullptr;
    __nv_bfloat16* Pexp = nullptr;  // p~ = exp(z - m_tile) [Mpad][ldz] bf16
    float* zact = nullptr;          // logit of the taken token [Mpad]
    float2* stats = nullptr;
    float* mrow = nullptr;  // loss fold: per-row softmax offset bound [Mpad]
    unsigned* lse_sync = nullptr;  // fused K-lse: {CTAs arrived, epoch published} (GEMM1 tail)
    unsigned lse_epoch = 0;
    // segmented K-list GEMM2 (FM_G2_KLIST=2), allocated on first use
    __nv_bfloat16 *aseg = nullptr, *bseg = nullptr;  // A' [kp_cap][ldz], B' [kp_cap][256]
    int4* slot4 = nullptr;                            // [rows_cap]
    int32_t *kcount = nullptr, *kseg_off = nullptr;   // [nblk][row chunks of 1024], [nblk]
    unsigned long long* kseg_rows = nullptr;          // executed GEMM2 K rows, accumulated
    int32_t* seg_tok = nullptr;                       // [kp_cap] token of each slot (mode 3)
    bool seg_has_a = false;                           // A' allocated (mode 2)
    int64_t kp_cap = 0;
    int32_t* klist = nullptr;  // K-list GEMM2: token lists per 256-feature block [nblk][klist_ld]
    int32_t* kiters = nullptr;  // [nblk] list length / 64
    int64_t klist_ld = 0;
    float* sk_ws = nullptr;  // GEMM2 stream-K tail: partial tiles [kSkMaxTiles][256][256] (zero between launches)
    int* sk_cnt = nullptr;   // [kSkMaxTiles][2] arrivals per tile half (self-resetting)
    // parity mode scratch
    int64_t prow_cap = 0;
    uint64_t pvocab_cap = 0, pparam_cap = 0;
    double *zscratch = nullptr, *dWmb = nullptr, *logp64 = nullptr;
    SampleDesc* sd = nullptr;
    int sd_cap = 0;
    // Phic / Phic^T hold exactly the entries of the rows in the row buffers
    // (for phi_Mpad, phi_D): the next gather erases them row by row
    bool phi_valid = false;
    int64_t phi_Mpad = 0;
    uint64_t phi_D = 0;
};

// Per-kernel device timing (bench.py's roofline): event pairs recorded on the
// launching stream around each hot-path kernel when enabled.
enum KKind { K_GATHER = 0, K_GEMM1, K_LSE, K_SOFTMAX_GRAD, K_GEMM2, K_ADAM, K_PARITY, K_MEMSET, K_COLMAX, K_NKINDS };
struct KTimer {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> open;
    double ms[K_NKINDS] = {};
    int64_t count[K_NKINDS] = {};
    cudaEvent_t get() {
        if (pool.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
};

// One training slot: the device home of an active agent's {W, m, v, dW, W16}.
// Slots are allocated once and recycled across activate/suspend (the
// reference's training_slots, config.hpp:89); reuse is ordered on the GPU by
// the event recorded after the previous tenant's copy-out.
struct Slot {
    void* base = nullptr;
    size_t cap = 0;
    bool busy = false;
    cudaEvent_t ev_free = nullptr;
};

struct fm_ctx {
    int device = 0;
    KTimer kt;
    std::vector<Slot*> slots;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    int num_sms = 148;
    cudaStream_t stream = nullptr;    // compute
    cudaStream_t copy_in = nullptr;   // swap-in (H2D / D2D / P2P)
    cudaStream_t copy_out = nullptr;  // swap-out
    // the latest K-GEMM1 launch on the compute stream (swap copies start there, see
    // fm_agent_suspend) and the op sequence numbers that say what it follows
    cudaEvent_t ev_gemm = nullptr;
    std::map<std::string, void*> ipc_cache;  // peer buffers mapped over NVLink (slots, gang receive buffers)
    std::vector<std::pair<size_t, void*>> recv_pool;  // gang receive buffers + barrier tokens, recycled
    std::unordered_map<void*, size_t> pool_sizes;
    uint64_t op_seq = 0, gemm_seq = 0;
    uint8_t* arena = nullptr;
    uint64_t arena_cap = 0, arena_used = 0;
    std::unordered_map<uint64_t, uint64_t> arena_ntok;  // offset -> token count
    Workspace ws;
    bool last_kseg = false;  // the last tensor-core micro-batch ran the segmented GEMM2
    // pinned staging (sample descriptors, host payloads) with reuse events
    uint8_t* staging[kStagingSlots] = {};
    size_t staging_cap[kStagingSlots] = {};
    cudaEvent_t staging_ev[kStagingSlots] = {};
    int staging_next = 0;
    // arena region reserved for the end-to-end host path
    uint64_t e2e_off = 0, e2e_cap = 0;
};

namespace fm {
uint64_t arena_token_count(const fm_ctx* ctx, uint64_t offset, bool* found) {
    auto it = ctx->arena_ntok.find(offset);
    *found = it != ctx->arena_ntok.end();
    return *found ? it->second : 0;
}
}  // namespace fm

namespace {

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::max(1, std::atoi(v)) : dflt;
}

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
    cudaFree(w.feat4);
    cudaFree(w.cnt4);
    cudaFree(w.n_ctx);
    cudaFree(w.sample);
    cudaFree(w.coef);
    cudaFree(w.rscale);
    cudaFree(w.lse);
    cudaFree(w.logp);
    cudaFree(w.coef_eff);
    cudaFree(w.old_logp);
    cudaFree(w.phic);
    cudaFree(w.phict);
    cudaFree(w.gt);
    cudaFree(w.Pexp);
    cudaFree(w.zact);
    cudaFree(w.stats);
    cudaFree(w.mrow);
    cudaFree(w.lse_sync);
    cudaFree(w.sk_ws);
    cudaFree(w.klist);
    cudaFree(w.kiters);
    cudaFree(w.aseg);
    cudaFree(w.bseg);
    cudaFree(w.slot4);
    cudaFree(w.kcount);
    cudaFree(w.kseg_off);
    cudaFree(w.kseg_rows);
    cudaFree(w.seg_tok);
    cudaFree(w.sk_cnt);
    cudaFree(w.zscratch);
    cudaFree(w.dWmb);
    cudaFree(w.logp64);
    cudaFree(w.sd);
    w = Workspace{};
}

uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

// Ensure tensor-core workspace for Mpad rows, vocab V, features D.
int ws_reserve_tc(fm_ctx* c, int64_t Mpad, uint64_t V, uint64_t D) {
    Workspace& w = c->ws;
    if (Mpad <= w.rows_cap && V <= w.vocab_cap && D <= w.feat_cap && w.Pexp) return FM_OK;
    const int64_t R = std::max<int64_t>(Mpad, w.rows_cap);
    const uint64_t VV = std::max<uint64_t>(V, w.vocab_cap), DD = std::max<uint64_t>(D, w.feat_cap);
    FM_CUDA(cudaStreamSynchronize(c->stream));
    Workspace keep_parity;
    std::swap(keep_parity.zscratch, w.zscratch);
    std::swap(keep_parity.dWmb, w.dWmb);
    std::swap(keep_parity.logp64, w.logp64);
    keep_parity.prow_cap = w.prow_cap;
    keep_parity.pvocab_cap = w.pvocab_cap;
    keep_parity.pparam_cap = w.pparam_cap;
    ws_free(w);
    w.zscratch = keep_parity.zscratch;
    w.dWmb = keep_parity.dWmb;
    w.logp64 = keep_parity.logp64;
    w.prow_cap = keep_parity.prow_cap;
    w.pvocab_cap = keep_parity.pvocab_cap;
    w.pparam_cap = keep_parity.pparam_cap;
    const uint64_t ldz = round_up(VV, 8);
    const uint64_t tiles_n = (VV + kGemmBN - 1) / kGemmBN;
    cudaError_t e = cudaSuccess;
    e = e ? e : dalloc(&w.action, R);
    e = e ? e : dalloc(&w.ctx4, R);
    e = e ? e : dalloc(&w.feat4, R);
    e = e ? e : dalloc(&w.cnt4, R);
    e = e ? e : dalloc(&w.n_ctx, R);
    e = e ? e : dalloc(&w.sample, R);
    e = e ? e : dalloc(&w.coef, R);
    e = e ? e : dalloc(&w.rscale, R);
    e = e ? e : dalloc(&w.lse, R);
    e = e ? e : dalloc(&w.logp, R);
    e = e ? e : dalloc(&w.coef_eff, R);
    e = e ? e : dalloc(&w.old_logp, R);
    // Phic and p~ carry one extra zero row (index R): the K-list GEMM2's padding row
    e = e ? e : dalloc(&w.phic, static_cast<size_t>(R + 1) * DD);
    e = e ? e : cudaMemset(w.phic, 0, static_cast<size_t>(R + 1) * DD * 2);
    e = e ? e : dalloc(&w.phict, static_cast<size_t>(R) * DD);
    e = e ? e : dalloc(&w.gt, static_cast<size_t>(R) * VV);
    e = e ? e : dalloc(&w.Pexp, static_cast<size_t>(R + 1) * ldz);
    e = e ? e : cudaMemset(w.Pexp + static_cast<size_t>(R) * ldz, 0, ldz * 2);
    w.klist_ld = static_cast<int64_t>(round_up(static_cast<uint64_t>(R), 64) + 64);
    e = e ? e : dalloc(&w.klist, static_cast<size_t>((DD + 255) / 256) * w.klist_ld);
    e = e ? e : dalloc(&w.kiters, static_cast<size_t>((DD + 255) / 256));
    e = e ? e : dalloc(&w.zact, R);
    e = e ? e : dalloc(&w.stats, static_cast<size_t>(R) * tiles_n);
    e = e ? e : dalloc(&w.mrow, R);
    e = e ? e : dalloc(&w.lse_sync, 2);
    e = e ? e : cudaMemset(w.lse_sync, 0, 2 * sizeof(unsigned));
    e = e ? e : dalloc(&w.sk_ws, static_cast<size_t>(kSkMaxTiles) * 256 * 256);
    e = e ? e : cudaMemset(w.sk_ws, 0, sizeof(float) * static_cast<size_t>(kSkMaxTiles) * 256 * 256);
    e = e ? e : dalloc(&w.sk_cnt, static_cast<size_t>(kSkMaxTiles) * 2);
    e = e ? e : cudaMemset(w.sk_cnt, 0, sizeof(int) * static_cast<size_t>(kSkMaxTiles) * 2);
    if (e != cudaSuccess) {
        ws_free(w);
        return fail(FM_ERR_DEVICE_OOM, std::string("workspace allocation: ") + cudaGetErrorString(e));
    }
    w.rows_cap = R;
    w.vocab_cap = VV;
    w.feat_cap = DD;
    return FM_OK;
}

// Token-slot segments for the segmented K-list GEMM2: every token occupies at
// most 4 slots (one per distinct feature block), each block's segment is padded
// to 64 rows.
int ws_reserve_seg(fm_ctx* c, bool need_a) {
    Workspace& w = c->ws;
    const int64_t nblk = static_cast<int64_t>((w.feat_cap + 255) / 256);
    const int64_t need = 4 * w.rows_cap + 64 * nblk;
    if (w.bseg && w.kp_cap >= need && (w.seg_has_a || !need_a)) return FM_OK;
    FM_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(w.aseg);
    cudaFree(w.bseg);
    cudaFree(w.slot4);
    cudaFree(w.kcount);
    cudaFree(w.kseg_off);
    cudaFree(w.seg_tok);
    w.aseg = w.bseg = nullptr;
    w.slot4 = nullptr;
    w.kcount = w.kseg_off = w.seg_tok = nullptr;
    w.seg_has_a = false;
    const uint64_t ldz = round_up(w.vocab_cap, 8);
    cudaError_t e = cudaSuccess;
    if (need_a) e = e ? e : dalloc(&w.aseg, static_cast<size_t>(need) * ldz);
    e = e ? e : dalloc(&w.seg_tok, static_cast<size_t>(need));
    e = e ? e : dalloc(&w.bseg, static_cast<size_t>(need) * 256);
    e = e ? e : dalloc(&w.slot4, static_cast<size_t>(w.rows_cap));
    e = e ? e : dalloc(&w.kcount, static_cast<size_t>(nblk) * static_cast<size_t>((w.rows_cap + 1023) / 1024 + 1));
    e = e ? e : dalloc(&w.kseg_off, static_cast<size_t>(nblk));
    if (!w.kseg_rows) {
        e = e ? e : dalloc(&w.kseg_rows, 1);
        e = e ? e : cudaMemset(w.kseg_rows, 0, sizeof(unsigned long long));
    }
    if (e != cudaSuccess) return fail(FM_ERR_DEVICE_OOM, std::string("segment workspace: ") + cudaGetErrorString(e));
    w.kp_cap = need;
    w.seg_has_a = need_a;
    return FM_OK;
}

int ws_reserve_rows(fm_ctx* c, int64_t R) {  // row arrays only (parity mode)
    Workspace& w = c->ws;
    if (R <= w.rows_cap && w.action) return FM_OK;
    if (w.Pexp) return ws_reserve_tc(c, R, w.vocab_cap, w.feat_cap);
    FM_CUDA(cudaStreamSynchronize(c->stream));
    w.phi_valid = false;
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
    e = e ? e : dalloc(&w.old_logp, R);
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
    r.feat4 = w.feat4;
    r.cnt4 = w.cnt4;
    r.mrow = w.mrow;
    r.n_ctx = w.n_ctx;
    r.sample = w.sample;
    r.coef = w.coef;
    r.rscale = w.rscale;
    r.lse = w.lse;
    r.logp = w.logp;
    r.coef_eff = w.coef_eff;
    return r;
}

// RAII event pair around one launch (no-op unless kernel timing is on).
struct KScope {
    fm_ctx* c;
    int kind;
    cudaStream_t s;
    cudaEvent_t e0 = nullptr;
    KScope(fm_ctx* c_, int k, cudaStream_t s_) : c(c_), kind(k), s(s_) {
        if (c->kt.on) {
            e0 = c->kt.get();
            cudaEventRecord(e0, s);
        }
    }
    ~KScope() {
        if (e0) {
            cudaEvent_t e1 = c->kt.get();
            cudaEventRecord(e1, s);
            c->kt.open.push_back({kind, {e0, e1}});
        }
    }
};

}  // namespace

extern "C" {

int fm_ctx_set_kernel_timing(fm_ctx* c, int on) {
    c->kt.on = on != 0;
    return FM_OK;
}

// Drains the recorded event pairs; out_ms / out_count have K_NKINDS (8) slots:
// gather, gemm1, lse, softmax_grad, gemm2, adam, parity, memset.
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
    if (max_rows > 0 && V > 0 && D > 0) return ws_reserve_tc(c, static_cast<int64_t>(round_up(max_rows, 128)), V, D);
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

// ===========================================================================
// agents
// ===========================================================================
// DP gang of an agent with the fused reduce-scatter: V rows are
// split into g contiguous, 256-row-aligned shards; during the step's last
// micro-batch GEMM2 writes the partials of rows owned by another rank into
// that rank's receive slot over NVLink (IPC-mapped), then each rank runs the
// sharded Adam on its rows and writes the new bf16 rows into every peer's
// W16.  Two 1-element NCCL all-reduces on the compute stream serve as the
// device-side barriers (after the exchange; the update grad-norm reduction
// after Adam), so no host round trip or spin-wait is involved.
#define FM_NCCL(expr)                                                                          \
    do {                                                                                       \
        ncclResult_t _r = (expr);                                                              \
        if (_r != ncclSuccess) return fail(FM_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
    } while (0)

struct fm_comm;
struct GangState;
static ncclComm_t gang_comm(GangState* gs);
struct GangState {
    fm_comm* comm = nullptr;
    int rank = 0, g = 1;
    int64_t lo[9] = {};          // row boundaries of the shards
    float* recv = nullptr;       // [g-1][own_rows][D] partials from the peers
    float* peer_slot[8] = {};    // my slot inside peer o's receive buffer
    __nv_bfloat16* peer_w16[8] = {};
    uint8_t* peer_base[8] = {};  // peer o's training slot (same layout as ours)
    int* d_token = nullptr;      // 1-int all-reduce used as a device barrier
    bool connected = false;
};

struct fm_agent {
    fm_ctx* ctx = nullptr;  // GPU the agent is bound to (null while suspended)
    std::string name;
    uint64_t V = 0, D = 0, P = 0;
    int precision = FM_PRECISION_BF16_TC;
    // device state
    double* W = nullptr;
    float* m = nullptr;
    float* v = nullptr;
    void* dW = nullptr;  // float (TC) or double (parity)
    __nv_bfloat16* W16 = nullptr;
    int* colmax = nullptr;          // K-colmax keys of W16 [D] (loss-fold softmax bound)
    uint64_t w16_gen = 0;           // bumped whenever W16 is rewritten
    uint64_t cm_gen = ~0ull;        // the W16 generation colmax describes
    bool cm_parked = false;         // the parked copy carries a valid colmax
    bool dw_valid = false;  // dW holds this step's partial sum
    bool pending_in = false;  // a swap-in copy the next use must wait for
    bool park_w16 = false;    // the parked copy includes the bf16 shadow
    int64_t step = 0, version = 0, samples = 0;
    // reports
    double* d_scalars = nullptr;  // [kReportRing][2]: sumsq, loss
    uint64_t last_seq = 0;        // ctx op sequence number of the agent's last compute op
    double* h_scalars = nullptr;  // pinned mirror
    cudaEvent_t ev[kReportRing] = {};
    int64_t rep_tokens[kReportRing] = {};
    int64_t rep_bs[kReportRing] = {};
    int64_t next_ticket = 0;
    bool dp = false;
    int shard_rank = 0, shard_count = 1;  // token-balanced DP shard of every micro-batch
    double* d_upd = nullptr;  // update sum g^2
    double* h_upd = nullptr;
    int64_t last_rows = 0;
    // PPO clip
    float clip_eps = 0.f;
    bool have_old_logp = false;
    // swap
    bool active = false;
    int park_tier = -1;
    int park_device = -1;
    void* park = nullptr;  // W | m | v | dW   (host pinned or device)
    size_t park_bytes = 0;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_compute = nullptr;
    cudaEvent_t ev_ipc = nullptr;  // interprocess: the source's work before a migration is done
    bool lent = false;             // exported by migration; slot reserved until migrate_release
    Slot* slot = nullptr;
    GangState* gang = nullptr;
};

// Device-side barrier across the gang (defined with the NCCL section below).
static int gang_barrier(fm_agent* a);
// Copies a full [V][D] state buffer (slot offset off, elem bytes/param) to dst
// (host or device), gathering a DP gang's row shards (defined below).
static int copy_state(fm_agent* a, size_t off, size_t elem, void* dst, cudaStream_t s);

namespace {

size_t dw_elem(const fm_agent* a) { return a->precision == FM_PRECISION_PARITY_F64 ? 8 : 4; }

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

size_t slot_off_m(const fm_agent* a) { return align256(a->P * 8); }
size_t slot_off_v(const fm_agent* a) { return align256(a->P * 8) + align256(a->P * 4); }

size_t slot_bytes(const fm_agent* a) {
    const size_t P = a->P;
    return align256(P * 8) + 2 * align256(P * 4) + align256(P * dw_elem(a)) +
           (a->precision == FM_PRECISION_BF16_TC ? align256(P * 2) + align256(a->D * 4) : 0);
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
    a->slot = pick;
    uint8_t* p = static_cast<uint8_t*>(pick->base);
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
    p += a->W16 ? align256(P * 2) : 0;
    a->colmax = a->W16 ? reinterpret_cast<int*>(p) : nullptr;
    return FM_OK;
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
        a->slot = nullptr;
    }
    a->W = nullptr;
    a->m = a->v = nullptr;
    a->dW = nullptr;
    a->W16 = nullptr;
    a->colmax = nullptr;
}

// Every operation on an agent goes through here: besides the InactiveGroup
// check it inserts the lazy dependency on a pending swap-in, so that an
// activate() prefetch never stalls other agents' work on the shared compute
// stream — only this agent's first use waits for its copy-in.
int check_active(fm_agent* a) {
    if (!a->active || !a->ctx) return fail(FM_ERR_INACTIVE_GROUP, a->name);
    if (a->pending_in) {
        FM_CUDA(cudaSetDevice(a->ctx->device));
        FM_CUDA(cudaStreamWaitEvent(a->ctx->stream, a->ev_in, 0));
        a->pending_in = false;
    }
    a->last_seq = ++a->ctx->op_seq;  // everything this op enqueues follows any earlier GEMM1 mark
    return FM_OK;
}

}  // namespace

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
    if (a->W16) FM_CUDA(cudaMemsetAsync(a->W16, 0, a->P * 2, c->stream));
    FM_CUDA(cudaMalloc(&a->d_scalars, kReportRing * 2 * sizeof(double)));
    FM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&a->h_scalars), kReportRing * 2 * sizeof(double), 0));
    FM_CUDA(cudaMalloc(&a->d_upd, sizeof(double)));
    FM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&a->h_upd), sizeof(double), 0));
    for (int i = 0; i < kReportRing; ++i) FM_CUDA(cudaEventCreateWithFlags(&a->ev[i], cudaEventDisableTiming));
    FM_CUDA(cudaEventCreateWithFlags(&a->ev_in, cudaEventDisableTiming));
    FM_CUDA(cudaEventCreateWithFlags(&a->ev_out, cudaEventDisableTiming));
    FM_CUDA(cudaEventCreateWithFlags(&a->ev_compute, cudaEventDisableTiming));
    a->active = true;
    *out = a;
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_destroy(fm_agent* a) {
    if (!a) return FM_OK;
    if (a->lent) fm_agent_migrate_release(a);
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
        FM_CUDA(launch_to_bf16(a->W, a->W16, a->P, c->num_sms, c->stream));
        count_launch();
        ++a->w16_gen;
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
        FM_CUDA(cudaMemcpy(tmp.data(), a->dW, a->P * 4, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < a->P; ++i) g[i] = tmp[i];
    }
    return FM_OK;
    FM_GUARD_END
}

int fm_debug_gemm(fm_ctx* c, const void* A, const void* B, int a_mn, int b_mn, int M, int N, int K, float* C) {
    FM_GUARD_BEGIN
    if (!c || !A || !B || !C || M <= 0 || N <= 0 || K <= 0 || M % 8 || N % 8 || K % 8)
        return fail(FM_ERR_INVALID_ARG, "debug_gemm: bad arguments");
    if (!gemm_pair_mode()) return fail(FM_ERR_CONFIG_ERROR, "debug_gemm needs the CTA-pair kernels");
    if (int st = set_dev(c)) return st;
    CUtensorMap tA, tB;
    const bool ok = (a_mn ? make_tmap_bf16_kmajor(&tA, A, K, M, 64) : make_tmap_bf16_kmajor(&tA, A, M, K, kGemmBM)) &&
                    (b_mn ? make_tmap_bf16_kmajor(&tB, B, K, N, 64)
                          : make_tmap_bf16_kmajor(&tB, B, N, K, gemm_b_box_rows()));
    if (!ok) return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    FM_CUDA(gemm_debug_launch(tA, tB, a_mn, b_mn, M, N, K, C, c->num_sms, c->stream));
    FM_CUDA(cudaStreamSynchronize(c->stream));
    return FM_OK;
    FM_GUARD_END
}

int fm_debug_gemm_klist(fm_ctx* c, const void* A, const void* B, const int32_t* klist, long long klist_ld,
                        const int32_t* klist_iters, int rows, int M, int N, float* C) {
    FM_GUARD_BEGIN
    if (!c || !A || !B || !C || !klist || !klist_iters || M <= 0 || N <= 0 || rows <= 0 || M % 8 || N % 8 ||
        klist_ld % 64)
        return fail(FM_ERR_INVALID_ARG, "debug_gemm_klist: bad arguments");
    if (!gemm_pair_mode()) return fail(FM_ERR_CONFIG_ERROR, "debug_gemm_klist needs the CTA-pair kernels");
    if (int st = set_dev(c)) return st;
    CUtensorMap tA, tB;
    if (!make_tmap_gather4(&tA, A, rows, M, M) || !make_tmap_gather4(&tB, B, rows, N, N))
        return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    GemmArgs g{};
    g.M = M;
    g.N = N;
    g.K = 64;
    g.group_m = 1;
    g.out = C;
    g.ld_out = N;
    g.klist = klist;
    g.klist_ld = klist_ld;
    g.klist_iters = klist_iters;
    FM_CUDA(gemm_klist_launch(tA, tB, g, c->num_sms, c->stream));
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
    if (int st = check_active(a)) return st;
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    a->clip_eps = clip_eps;
    a->have_old_logp = false;
    if (old_logp && clip_eps > 0.f) {
        if (int st = ws_reserve_rows(c, static_cast<int64_t>(round_up(n_rows, 128)))) return st;
        FM_CUDA(cudaMemcpyAsync(c->ws.old_logp, old_logp, n_rows * 4, cudaMemcpyHostToDevice, c->stream));
        FM_CUDA(cudaStreamSynchronize(c->stream));
        a->have_old_logp = true;
    }
    return FM_OK;
}

int fm_agent_set_shard(fm_agent* a, int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FM_ERR_INVALID_ARG, "bad shard");
    a->shard_rank = rank;
    a->shard_count = nranks;
    a->dp = nranks > 1;
    return FM_OK;
}

// ---------------------------------------------------------------------------
// the micro-batch pipeline
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
    const int64_t Mpad = tc ? static_cast<int64_t>(round_up(static_cast<uint64_t>(M), 128)) : M;
    if (tc) {
        if (int st = ws_reserve_tc(c, std::max<int64_t>(Mpad, 128), a->V, a->D)) return st;
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

    const int64_t ticket = a->next_ticket++;
    const int slot = static_cast<int>(ticket % kReportRing);
    if (ticket >= kReportRing) FM_CUDA(cudaEventSynchronize(a->ev[slot]));  // slot reuse
    double* scal = a->d_scalars + 2 * slot;
    FM_CUDA(cudaMemsetAsync(scal, 0, 2 * sizeof(double), s));
    RowBuffers rows = row_buffers(w);

    if (M > 0) {
        if (tc) {
            const uint64_t ldz = round_up(a->V, 8);
            const bool reuse = w.phi_valid && w.phi_Mpad == Mpad && w.phi_D == a->D;
            if (!reuse) {
                KScope k(c, K_MEMSET, s);
                FM_CUDA(cudaMemsetAsync(w.phic, 0, static_cast<size_t>(Mpad) * a->D * 2, s));
                FM_CUDA(cudaMemsetAsync(w.phict, 0, static_cast<size_t>(Mpad) * a->D * 2, s));
            }
            const bool fold = loss_fold_enabled();
            // K-list GEMM2 (opt-in FM_G2_KLIST=1): each 256-feature column block of the
            // weight gradient sums only over the tokens whose context touches it
            // GEMM2 over token-slot segments (default; FM_G2_KLIST=0 dense, 1 gather4 lists):
            // each 256-feature column block of dW sums only the tokens whose context touches
            // it — GEMM1 writes each token's p~ row into one slot per feature block it
            // touches and GEMM2 tile-loads contiguous segments.  Falls back to the dense
            // GEMM2 when the segment workspace does not fit.
            const char* kl_env = std::getenv("FM_G2_KLIST");
            const char kl_mode = kl_env && kl_env[0] ? kl_env[0] : '2';
            const bool klist = fold && gemm_pair_mode() && kl_mode == '1';
            bool kseg = fold && gemm_pair_mode() && (kl_mode == '2' || kl_mode == '3');
            // mode 3: A rows gathered from the row-major p~ by producer warps (no A' copies)
            const bool swa = kseg && kl_mode == '3';
            if (kseg && ws_reserve_seg(c, !swa) != FM_OK) {
                kseg = false;
                clear_error();
                cudaGetLastError();
            }
            c->last_kseg = kseg;
            if (fold && a->cm_gen != a->w16_gen) {
                // per-feature max of the shadow, when K-adam did not produce it (first step,
                // set_weights, DP-gang sharded update, host-tier swap-in)
                KScope k(c, K_COLMAX, s);
                FM_CUDA(launch_colmax(a->W16, static_cast<int64_t>(a->V), static_cast<int64_t>(a->D), a->colmax,
                                      c->num_sms, s));
                a->cm_gen = a->w16_gen;
                count_launch();
            }
            {
                KScope k(c, K_GATHER, s);
                FM_CUDA(launch_gather(c->arena, w.sd, n, row_lo, M, Mpad, G, a->D, rows, w.phic, w.phict,
                                      reuse ? 1 : 0, fold ? a->colmax : nullptr, s));
            }
            w.phi_valid = true;
            w.phi_Mpad = Mpad;
            w.phi_D = a->D;
            const int nblk = static_cast<int>((a->D + kGemmBN - 1) / kGemmBN);
            if (klist) {
                KScope k(c, K_GATHER, s);
                FM_CUDA(launch_klist(rows.feat4, M, nblk, w.klist, w.klist_ld, w.kiters,
                                     static_cast<int32_t>(w.rows_cap), s));
                count_launch();
            }
            if (kseg) {
                KScope k(c, K_GATHER, s);
                FM_CUDA(cudaMemsetAsync(w.bseg, 0, static_cast<size_t>(w.kp_cap) * 256 * 2, s));
                FM_CUDA(launch_kslots(rows.feat4, rows.cnt4, M, nblk, w.kcount, w.kseg_off, w.kiters, w.slot4,
                                      swa ? nullptr : w.aseg, static_cast<int64_t>(ldz), static_cast<int64_t>(ldz),
                                      w.bseg, w.kseg_rows, swa ? w.seg_tok : nullptr,
                                      static_cast<int32_t>(w.rows_cap), s));
                count_launch(2);
            }
            // K-GEMM1: z = Phic * W16^T / n; epilogue stores p~ = exp(z - m) (bf16) with m the
            // row's bound (fold: transposed, GEMM2's A operand) or the tile max (K-loss path),
            // the (m, sum p~) softmax partials and the taken token's logit
            CUtensorMap tA, tB, tP, tGt, tPt;
            if (!make_tmap_bf16_kmajor(&tA, w.phic, Mpad, a->D, kGemmBM) ||
                !make_tmap_bf16_kmajor(&tB, a->W16, a->V, a->D, gemm_b_box_rows()) ||
                !make_tmap_2d(&tP, w.Pexp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Mpad, ldz, 64, 128) ||
                !make_tmap_bf16_kmajor(&tGt, w.gt, a->V, Mpad, kGemmBM) ||
                !make_tmap_bf16_kmajor(&tPt, w.phict, a->D, Mpad, gemm_b_box_rows()))
                return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
            const int tiles_n = static_cast<int>((a->V + kGemmBN - 1) / kGemmBN);
            GemmArgs g1{};
            g1.M = static_cast<int>(M);
            g1.N = static_cast<int>(a->V);
            g1.K = static_cast<int>(a->D);
            g1.group_m = env_int("FM_G1_GROUP_M", 16);  // raster: m-tiles per group (L2 reuse)
            if (kseg && !swa) {  // p~ rows into the token's segment slots (A')
                g1.mrow = w.mrow;
                g1.aseg = w.aseg;
                g1.slot4 = w.slot4;
            } else if (klist || swa) {  // p~ row-major: the K-list GEMM2 gathers token rows
                g1.mrow = w.mrow;
                g1.pexp = w.Pexp;
            } else if (fold) {  // p~^T straight into GEMM2's A operand buffer
                g1.mrow = w.mrow;
                g1.pexp_t = w.gt;
                g1.ldt = static_cast<long long>(Mpad);
                g1.store_rows = static_cast<int>(Mpad);
            } else {
                g1.pexp = w.Pexp;
            }
            g1.zact = w.zact;
            g1.action = w.action;
            g1.ld_out = static_cast<long long>(ldz);
            g1.row_scale = w.rscale;
            g1.stats = w.stats;
            g1.stats_ld = tiles_n;
            // K-lse fused into GEMM1's tail (loss fold, CTA-pair kernel; FM_LSE_FUSED=0
            // launches it separately): after a grid-wide arrival the epilogue warps
            // normalise the rows.  Same time as the 14 us launch it replaces (C2: GEMM1
            // +7-29 us, K-lse -14 us); one launch fewer per micro-batch.  (A per-tile
            // last-finisher variant cost GEMM1 12-15%: DESIGN.md §9.)
            const char* lse_env = std::getenv("FM_LSE_FUSED");
            const bool lse_fused = fold && gemm_pair_mode() && !(lse_env && lse_env[0] == '0');
            LseArgs lse_args{w.zact, w.stats, tiles_n, M, Mpad, static_cast<int64_t>(a->V), w.sd, G, rows,
                             a->have_old_logp ? w.old_logp : nullptr, a->clip_eps, scal + 1,
                             fold ? 1 : 0, fold ? w.gt : nullptr, w.phict, Mpad};
            if (klist) {
                lse_args.pexp_t = w.Pexp;
                lse_args.ldt = static_cast<int64_t>(ldz);
                lse_args.phict = w.phic;
                lse_args.rowmajor = 1;
                lse_args.ld_phi = static_cast<int64_t>(a->D);
            }
            if (kseg) {
                lse_args.pexp_t = swa ? w.Pexp : w.aseg;
                lse_args.ldt = static_cast<int64_t>(ldz);
                lse_args.rowmajor = swa ? 3 : 2;
                lse_args.slot4 = w.slot4;
                lse_args.bseg = w.bseg;
            }
            if (lse_fused) {
                g1.lse = lse_args;
                g1.lse_sync = w.lse_sync;
                g1.lse_epoch = ++w.lse_epoch;
            }
            FM_CUDA(cudaEventRecord(c->ev_gemm, s));  // swap copies may start here (fm_agent_suspend)
            c->gemm_seq = ++c->op_seq;
            {
                KScope k(c, K_GEMM1, s);
                FM_CUDA(gemm_tn_launch(GemmKind::Logits, tA, tB, g1, c->num_sms, s));
            }
            // K-lse (standalone unless fused into GEMM1's epilogue)
            if (!lse_fused) {
                KScope k(c, K_LSE, s);
                FM_CUDA(launch_lse(lse_args, s));
            }
            // K-softmax-grad: G^T tiles (zero for padding rows) — folded into GEMM2's operands
            if (!fold) {
                KScope k(c, K_SOFTMAX_GRAD, s);
                FM_CUDA(launch_softmax_grad(tP, tGt, w.stats, tiles_n, Mpad, static_cast<int64_t>(a->V), rows, s));
            }
            // K-GEMM2: dW (+)= G^T * Phic ; first contribution of the step overwrites
            // (fold: A = p~'^T, B = Phic^T scaled per row by K-lse — the same product)
            GemmArgs g2{};
            g2.M = static_cast<int>(a->V);
            g2.N = static_cast<int>(a->D);
            g2.K = static_cast<int>(Mpad);
            // raster: when B = Phic^T (D x Mpad bf16) is about L2-sized (C2: 134 MB) run all
            // D/256 column tiles of a vocab row block together (group 1) so p~^T is read
            // from DRAM once (ncu: 6.6 vs 7.0 GB, 2.22 vs 2.26 ms; profiles/r01_g2_sweep.jsonl);
            // a larger B (C3/C5: 1.07 GB) would be re-read per row block, so group 8 there
            const double b_bytes = 2.0 * static_cast<double>(a->D) * static_cast<double>(Mpad);
            g2.group_m = env_int("FM_G2_GROUP_M", b_bytes <= 160e6 ? 1 : 8);
            g2.out = static_cast<float*>(a->dW);
            g2.ld_out = static_cast<long long>(a->D);
            g2.accumulate = a->dw_valid ? 1 : 0;
            g2.sumsq = scal;
            {
                // stream-K tail (opt-in FM_G2_STREAMK=1): C2's 2,000 tiles on 74 pairs leave a
                // last wave of 2 tiles; split the last 76 tiles' K ranges evenly instead.
                // Measured within noise of the plain schedule at C2 (2.676 vs 2.670 ms).
                const char* sk_env = std::getenv("FM_G2_STREAMK");
                if (gemm_pair_mode() && c->num_sms / 2 <= kSkMaxTiles / 2 && sk_env && sk_env[0] == '1') {
                    g2.sk_ws = w.sk_ws;
                    g2.sk_cnt = w.sk_cnt;
                }
            }
            const bool exchange = a->gang && a->gang->connected && a->samples + n == G;
            if (exchange) {  // last micro-batch of the step: reduce-scatter inside the epilogue
                GangState* gs = a->gang;
                g2.xg = gs->g;
                g2.xrank = gs->rank;
                for (int o = 0; o <= gs->g; ++o) g2.xlo[o] = static_cast<int>(gs->lo[o]);
                for (int o = 0; o < gs->g; ++o) g2.xpeer[o] = gs->peer_slot[o];
            }
            {
                // Long K (rows of the micro-batch): optionally launch K-chunks of FM_G2_KCHUNK
                // rows in sequence, each accumulating into dW, so concurrent tiles stay within
                // one chunk's operands (L2 reuse).  Off by default: at C5 N=1 (K = 65,536) the
                // A/B on one box was within noise (profiles/r01_kchunk.jsonl).  When chunked
                // the micro-batch grad norm spans several accumulations and reads NaN.
                const int kc_env = env_int("FM_G2_KCHUNK", 1 << 30);  // default: one launch
                const int kc = static_cast<int>(round_up(static_cast<uint64_t>(std::min(kc_env, 1 << 30)), 64));
                const int nch = (static_cast<int>(Mpad) + kc - 1) / kc;
                KScope k(c, K_GEMM2, s);
                if (swa) {
                    CUtensorMap tSB;
                    if (!make_tmap_bf16_kmajor(&tSB, w.bseg, static_cast<uint64_t>(w.kp_cap), 256, 64))
                        return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
                    g2.kseg_off = w.kseg_off;
                    g2.klist_iters = w.kiters;
                    g2.seg_tok = w.seg_tok;
                    g2.pexp = w.Pexp;
                    g2.ld_pexp = static_cast<long long>(ldz);
                    g2.sk_ws = nullptr;
                    FM_CUDA(gemm_kseg_swa_launch(tSB, g2, c->num_sms, s));
                } else if (kseg) {
                    CUtensorMap tSA, tSB;
                    if (!make_tmap_bf16_kmajor(&tSA, w.aseg, static_cast<uint64_t>(w.kp_cap), a->V, 64, ldz) ||
                        !make_tmap_bf16_kmajor(&tSB, w.bseg, static_cast<uint64_t>(w.kp_cap), 256, 64))
                        return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
                    g2.kseg_off = w.kseg_off;
                    g2.klist_iters = w.kiters;
                    g2.sk_ws = nullptr;
                    FM_CUDA(gemm_kseg_launch(tSA, tSB, g2, c->num_sms, s));
                } else if (klist) {
                    CUtensorMap tKA, tKB;
                    if (!make_tmap_gather4(&tKA, w.Pexp, static_cast<uint64_t>(w.rows_cap) + 1, a->V, ldz) ||
                        !make_tmap_gather4(&tKB, w.phic, static_cast<uint64_t>(w.rows_cap) + 1, a->D, a->D))
                        return fail(FM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
                    g2.klist = w.klist;
                    g2.klist_ld = w.klist_ld;
                    g2.klist_iters = w.kiters;
                    g2.sk_ws = nullptr;
                    FM_CUDA(gemm_klist_launch(tKA, tKB, g2, c->num_sms, s));
                } else if (nch == 1) {
                    FM_CUDA(gemm_tn_launch(GemmKind::Grad, tGt, tPt, g2, c->num_sms, s));
                } else {
                    FM_CUDA(cudaMemsetAsync(scal, 0xFF, sizeof(double), s));  // NaN grad norm
                    for (int ch = 0; ch < nch; ++ch) {
                        GemmArgs gc = g2;
                        gc.k0 = ch * kc;
                        gc.K = std::min(kc, static_cast<int>(Mpad) - gc.k0);
                        gc.accumulate = (a->dw_valid || ch > 0) ? 1 : 0;
                        gc.sumsq = nullptr;
                        if (ch + 1 < nch) gc.xg = 0;  // the gang exchange rides on the last chunk
                        FM_CUDA(gemm_tn_launch(GemmKind::Grad, tGt, tPt, gc, c->num_sms, s));
                    }
                    count_launch(nch - 1);
                }
            }
            if (exchange) {
                a->dw_valid = true;
                if (int st = gang_barrier(a)) return st;  // every rank's partials have landed
            }
            count_launch(fold ? (lse_fused ? 3 : 4) : 5);
        } else {
            w.phi_valid = false;  // the row buffers no longer describe Phic's contents
            FM_CUDA(launch_gather(c->arena, w.sd, n, row_lo, M, M, G, a->D, rows, nullptr, nullptr, 0, nullptr, s));
            if (!a->dw_valid) FM_CUDA(cudaMemsetAsync(a->dW, 0, a->P * 8, s));
            KScope k(c, K_PARITY, s);
            FM_CUDA(launch_parity_rows(a->W, a->V, a->D, M, rows, w.sd, G, w.zscratch, w.dWmb, w.logp64,
                                       scal + 1, s));
            FM_CUDA(launch_parity_fold(static_cast<double*>(a->dW), w.dWmb, a->P, scal, c->num_sms, s));
            count_launch(3);
        }
        a->dw_valid = true;
    } else if (a->gang && a->gang->connected && a->samples + n == G) {
        // this rank got no rows of the step's last micro-batch: ship its partials
        // for the peers' rows with plain NVLink copies, then join the barrier
        GangState* gs = a->gang;
        if (!a->dw_valid) FM_CUDA(cudaMemsetAsync(a->dW, 0, a->P * 4, s));
        for (int o = 0; o < gs->g; ++o) {
            if (o == gs->rank) continue;
            const size_t rows = static_cast<size_t>(gs->lo[o + 1] - gs->lo[o]);
            FM_CUDA(cudaMemcpyAsync(gs->peer_slot[o], static_cast<float*>(a->dW) + gs->lo[o] * a->D,
                                    rows * a->D * 4, cudaMemcpyDeviceToDevice, s));
        }
        a->dw_valid = true;
        if (int st = gang_barrier(a)) return st;
    }
    a->have_old_logp = false;  // old log-probs apply to one micro-batch
    a->last_rows = M;
    a->last_seq = ++c->op_seq;  // its own GEMM1 mark precedes this micro-batch's GEMM2
    FM_CUDA(cudaMemcpyAsync(a->h_scalars + 2 * slot, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FM_CUDA(cudaEventRecord(a->ev[slot], s));
    a->rep_tokens[slot] = M;
    a->rep_bs[slot] = n;
    a->samples += n;
    if (ticket_out) *ticket_out = ticket;
    return FM_OK;
}

int fm_train_micro_batch(fm_agent* a, const fm_sample* samples, int n, int64_t G, int64_t* ticket_out) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
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
    if (int st = check_active(a)) return st;
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
    if (int st = check_active(a)) return st;
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

int fm_agent_debug_colmax(fm_agent* a, float* out, int* valid) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    if (!a->colmax) return fail(FM_ERR_CONFIG_ERROR, "no bf16 shadow (parity precision)");
    if (int st = set_dev(a->ctx)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    std::vector<int> keys(a->D);
    FM_CUDA(cudaMemcpy(keys.data(), a->colmax, a->D * 4, cudaMemcpyDeviceToHost));
    for (uint64_t d = 0; d < a->D; ++d) {
        const int k = keys[d] >= 0 ? keys[d] : keys[d] ^ 0x7fffffff;
        std::memcpy(out + d, &k, 4);
    }
    if (valid) *valid = a->cm_gen == a->w16_gen ? 1 : 0;
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_sync(fm_agent* a) {
    if (!a->ctx) return FM_OK;
    if (int st = set_dev(a->ctx)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    return FM_OK;
}

int fm_agent_poll_report(fm_agent* a, int64_t ticket, fm_report* out) {
    if (ticket < 0 || ticket >= a->next_ticket || ticket < a->next_ticket - kReportRing)
        return fail(FM_ERR_INVALID_ARG, "unknown or expired ticket");
    const int slot = static_cast<int>(ticket % kReportRing);
    const cudaError_t q = cudaEventQuery(a->ev[slot]);
    if (q == cudaErrorNotReady) return 0;
    if (q != cudaSuccess) return fail(FM_ERR_CUDA, cudaGetErrorString(q));
    out->ticket = ticket;
    out->tokens = a->rep_tokens[slot];
    out->batch_size = a->rep_bs[slot];
    out->grad_norm = a->dp ? NAN : std::sqrt(a->h_scalars[2 * slot]);
    out->loss = a->h_scalars[2 * slot + 1];
    return 1;
}

static int park_reserve(fm_agent* a, fm_ctx* c, int tier, int pdev, size_t bytes);
static size_t park_bytes_for(const fm_agent* a);

// apply_global_update; with park != 0 (device tier, tensor-core agent, no gang)
// K-adam writes the new W / m / v / W16 / colmax straight into the agent's
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
    bool cm_fused = false;
    KScope ks(c, K_ADAM, s);
    if (a->precision == FM_PRECISION_PARITY_F64) {
        FM_CUDA(launch_adam<double>(a->W, a->m, a->v, static_cast<double*>(a->dW), nullptr, a->P, lr, b1, b2, eps,
                                    bc1, bc2, 1, a->d_upd, c->num_sms, s));
    } else if (a->gang && a->gang->connected) {
        // sharded Adam over this rank's rows; W16 rows all-gathered by peer stores
        GangState* gs = a->gang;
        const int64_t r0 = gs->lo[gs->rank], r1 = gs->lo[gs->rank + 1];
        const uint64_t off = static_cast<uint64_t>(r0) * a->D, n_own = static_cast<uint64_t>(r1 - r0) * a->D;
        ShardPeers peers{};
        for (int o = 0; o < gs->g; ++o)
            if (o != gs->rank) peers.w16[peers.n++] = gs->peer_w16[o] + off;
        FM_CUDA(launch_adam_shard(a->W + off, a->m + off, a->v + off, static_cast<float*>(a->dW) + off, gs->recv,
                                  gs->g - 1, n_own, a->W16 + off, peers, n_own, lr, b1, b2, eps, bc1, bc2, a->d_upd,
                                  c->num_sms, s));
        // global grad norm^2; doubles as the barrier after the peers' W16 writes
        FM_NCCL(ncclAllReduce(a->d_upd, a->d_upd, 1, ncclFloat64, ncclSum, gang_comm(gs), s));
    } else {
        // the next step's first GEMM2 overwrites dW, so no zeroing pass here; the new
        // shadow's column maxima (loss-fold bound) come out of the same pass
        const size_t dwe = dw_elem(a);
        __nv_bfloat16* w16_out = park ? reinterpret_cast<__nv_bfloat16*>(pk + a->P * (16 + dwe)) : a->W16;
        int* cm_out = park ? reinterpret_cast<int*>(pk + a->P * (18 + dwe)) : a->colmax;
        FM_CUDA(launch_adam<float>(a->W, a->m, a->v, static_cast<float*>(a->dW), w16_out, a->P, lr, b1, b2, eps,
                                   bc1, bc2, 0, a->d_upd, c->num_sms, s, loss_fold_enabled() ? cm_out : nullptr,
                                   a->D, &cm_fused, park ? &dst : nullptr));
    }
    count_launch();
    a->dw_valid = false;
    a->samples = 0;
    a->version += 1;
    ++a->w16_gen;
    if (cm_fused) a->cm_gen = a->w16_gen;
    FM_CUDA(cudaMemcpyAsync(a->h_upd, a->d_upd, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (park) {
        // the parked state is complete when K-adam is: release the slot behind it
        a->park_w16 = true;
        a->cm_parked = cm_fused;
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

// ---------------------------------------------------------------------------
// training-state swap
// ---------------------------------------------------------------------------
// Park layout: W | m | v | dW | W16 | colmax keys.
static size_t park_bytes_for(const fm_agent* a) {
    return a->P * 16 + a->P * dw_elem(a) + (a->W16 ? a->P * 2 + a->D * 4 : 0);
}

// Parking buffer of `bytes` on `tier` (device pdev), reused while it fits.
static int park_reserve(fm_agent* a, fm_ctx* c, int tier, int pdev, size_t bytes) {
    if (a->park && (a->park_tier != tier || a->park_device != pdev || a->park_bytes < bytes)) {
        FM_CUDA(cudaStreamSynchronize(c->copy_out));
        if (a->park_tier == FM_TIER_HOST) cudaFreeHost(a->park);
        else {
            cudaSetDevice(a->park_device);
            cudaFree(a->park);
            cudaSetDevice(c->device);
        }
        a->park = nullptr;
    }
    if (!a->park) {
        if (tier == FM_TIER_HOST) {
            if (cudaHostAlloc(&a->park, bytes, cudaHostAllocDefault) != cudaSuccess)
                return fail(FM_ERR_HOST_OOM, "pinned parking buffer");
        } else if (tier == FM_TIER_DEVICE || tier == FM_TIER_PEER) {
            if (tier == FM_TIER_PEER) {
                int can = 0;
                FM_CUDA(cudaDeviceCanAccessPeer(&can, c->device, pdev));
                if (!can) return fail(FM_ERR_CONFIG_ERROR, "no peer access to device " + std::to_string(pdev));
                cudaError_t pe = cudaDeviceEnablePeerAccess(pdev, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) FM_CUDA(pe);
                cudaGetLastError();
                FM_CUDA(cudaSetDevice(pdev));
            }
            const cudaError_t e = cudaMalloc(&a->park, bytes);
            FM_CUDA(cudaSetDevice(c->device));
            if (e != cudaSuccess) return fail(FM_ERR_DEVICE_OOM, "parking buffer");
        } else {
            return fail(FM_ERR_INVALID_ARG, "unknown tier");
        }
        a->park_tier = tier;
        a->park_device = pdev;
        a->park_bytes = bytes;
    }
    return FM_OK;
}

int fm_agent_suspend(fm_agent* a, int tier, int peer_device) {
    FM_GUARD_BEGIN
    // a K-GEMM1 launched after the agent's last op (e.g. the next agent's first
    // micro-batch) is a safe and cheap start for the copy-out: the copy engines then
    // overlap tensor-bound GEMMs instead of the latency-bound K-gather that follows
    // the end of the currently queued work (measured: K-gather 16 us -> 390 us
    // beside a 2.4 GB D2D copy)
    const bool gated = a->active && a->ctx && a->ctx->gemm_seq > a->last_seq;
    if (int st = check_active(a)) return st;
    if (a->gang) return fail(FM_ERR_BUSY_GROUP, a->name + " is attached to a DP gang (fm_gang_detach first)");
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    const size_t P = a->P;
    const size_t dwb = a->dw_valid ? P * dw_elem(a) : 0;
    // park layout: W | m | v | dW | W16.  The bf16 shadow travels on the HBM /
    // NVLink tiers (a copy-engine copy is cheaper than regenerating it on the
    // SMs); over PCIe it is regenerated from W on activation instead.
    const bool park_w16 = a->W16 && tier != FM_TIER_HOST;
    const size_t bytes = park_bytes_for(a);
    const int pdev = tier == FM_TIER_PEER ? peer_device : c->device;
    if (int st = park_reserve(a, c, tier, pdev, bytes)) return st;
    // order the copy-out after everything the agent has queued on the compute stream
    if (gated) {
        FM_CUDA(cudaStreamWaitEvent(c->copy_out, c->ev_gemm, 0));
    } else {
        FM_CUDA(cudaEventRecord(a->ev_compute, c->stream));
        FM_CUDA(cudaStreamWaitEvent(c->copy_out, a->ev_compute, 0));
    }
    uint8_t* p = static_cast<uint8_t*>(a->park);
    auto cp = [&](void* dst, const void* src, size_t n) -> cudaError_t {
        if (tier == FM_TIER_PEER) return cudaMemcpyPeerAsync(dst, pdev, src, c->device, n, c->copy_out);
        return cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, c->copy_out);
    };
    FM_CUDA(cp(p, a->W, P * 8));
    FM_CUDA(cp(p + P * 8, a->m, P * 4));
    FM_CUDA(cp(p + P * 12, a->v, P * 4));
    if (dwb) FM_CUDA(cp(p + P * 16, a->dW, dwb));  // only mid-step gradients travel
    if (park_w16) FM_CUDA(cp(p + P * (16 + dw_elem(a)), a->W16, P * 2));
    a->park_w16 = park_w16;
    a->cm_parked = park_w16 && a->cm_gen == a->w16_gen;
    if (a->cm_parked) FM_CUDA(cp(p + P * (18 + dw_elem(a)), a->colmax, a->D * 4));
    FM_CUDA(cudaEventRecord(a->ev_out, c->copy_out));
    agent_free_device(a, c->copy_out);
    a->active = false;
    a->ctx = nullptr;
    a->park_device = pdev;
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_activate(fm_agent* a, fm_ctx* c) {
    FM_GUARD_BEGIN
    if (a->active) return fail(FM_ERR_CONFIG_ERROR, a->name + " already active");
    if (a->lent) return fail(FM_ERR_CONFIG_ERROR, a->name + " was migrated away (fm_agent_migrate_release)");
    if (!c) return fail(FM_ERR_NO_DEVICE, "null context");
    if (int st = set_dev(c)) return st;
    const size_t P = a->P;
    // the parked copy must have landed before we read it back
    FM_CUDA(cudaStreamWaitEvent(c->copy_in, a->ev_out, 0));
    // start the copy-in beside the latest queued K-GEMM1 (tensor-bound) rather than
    // beside whatever runs when it is issued: the latency-bound gather / slot kernels
    // slowed 4x next to a copy-engine burst (119 vs 28 us per micro-batch)
    if (c->gemm_seq > 0) FM_CUDA(cudaStreamWaitEvent(c->copy_in, c->ev_gemm, 0));

    if (int st = agent_alloc_device(a, c, c->copy_in)) return st;
    uint8_t* p = static_cast<uint8_t*>(a->park);
    const bool peer = a->park_tier != FM_TIER_HOST && a->park_device != c->device;
    if (peer) {
        int can = 0;
        FM_CUDA(cudaDeviceCanAccessPeer(&can, c->device, a->park_device));
        if (!can) return fail(FM_ERR_CONFIG_ERROR, "no peer access to parking device");
        cudaError_t pe = cudaDeviceEnablePeerAccess(a->park_device, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) FM_CUDA(pe);
        cudaGetLastError();
    }
    auto cp = [&](void* dst, const void* src, size_t n) -> cudaError_t {
        if (peer) return cudaMemcpyPeerAsync(dst, c->device, src, a->park_device, n, c->copy_in);
        return cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, c->copy_in);
    };
    FM_CUDA(cp(a->W, p, P * 8));
    FM_CUDA(cp(a->m, p + P * 8, P * 4));
    FM_CUDA(cp(a->v, p + P * 12, P * 4));
    if (a->dw_valid) FM_CUDA(cp(a->dW, p + P * 16, P * dw_elem(a)));
    if (a->W16 && a->park_w16) {
        FM_CUDA(cp(a->W16, p + P * (16 + dw_elem(a)), P * 2));
    } else if (a->W16) {
        FM_CUDA(launch_to_bf16(a->W, a->W16, P, c->num_sms, c->copy_in));  // shadow regenerated
        count_launch();
    }
    if (a->W16 && a->park_w16 && a->cm_parked) FM_CUDA(cp(a->colmax, p + P * (18 + dw_elem(a)), a->D * 4));
    FM_CUDA(cudaEventRecord(a->ev_in, c->copy_in));
    ++a->w16_gen;
    if (a->W16 && a->park_w16 && a->cm_parked) a->cm_gen = a->w16_gen;
    a->pending_in = true;  // consumers wait lazily (check_active)
    a->ctx = c;
    a->active = true;
    return FM_OK;
    FM_GUARD_END
}

// ---- cross-process migration over NVLink (location-agnostic swap between GPUs) ----
// The sender lends its live training slot: it exports CUDA IPC handles of the
// slot and of an interprocess event recorded on its compute stream after the
// agent's queued work, and stops using the agent.  The receiver maps the slot
// (mappings are cached per context: slots are recycled, so after the first hop
// a migration is just the copy) and pulls the state into its own slot with
// copy-engine NVLink peer copies on its copy stream.  No park copy on the
// source.  The sender returns the slot to its pool with fm_agent_migrate_release
// once the receiver's import has returned (training.hpp:259-350 with a
// placement change; SURVEY §8e "agents <-> GPUs").
namespace {
struct MigrateBlob {
    uint32_t magic;  // 'FMMG'
    int32_t precision;
    uint64_t V, D;
    int32_t src_device;
    uint8_t dw_valid, cm_valid, pad0, pad1;
    int64_t step, version, samples;
    uint64_t off_w, off_m, off_v, off_dw, off_w16, off_cm;  // within the slot
    cudaIpcMemHandle_t mem;
    cudaIpcEventHandle_t ev;
};
constexpr uint32_t kMigrateMagic = 0x474d4d46u;
}  // namespace

static int migrate_export_impl(fm_agent* a, uint8_t* blob_out, uint64_t cap, uint64_t* len, bool share);

int fm_agent_migrate_export(fm_agent* a, uint8_t* blob_out, uint64_t cap, uint64_t* len) {
    return migrate_export_impl(a, blob_out, cap, len, false);
}

// Same blob, but the agent stays active here: several processes may import it
// (a DP gang forming around the agent); the caller enqueues no work for it
// until every importer returned.
int fm_agent_share_export(fm_agent* a, uint8_t* blob_out, uint64_t cap, uint64_t* len) {
    return migrate_export_impl(a, blob_out, cap, len, true);
}

static int migrate_export_impl(fm_agent* a, uint8_t* blob_out, uint64_t cap, uint64_t* len, bool share) {
    FM_GUARD_BEGIN
    *len = sizeof(MigrateBlob);
    if (!blob_out) return FM_OK;
    if (cap < sizeof(MigrateBlob)) return fail(FM_ERR_INVALID_ARG, "blob buffer too small");
    if (int st = check_active(a)) return st;
    if (a->gang) return fail(FM_ERR_BUSY_GROUP, a->name + " is attached to a DP gang (fm_gang_detach first)");
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    if (!a->ev_ipc) FM_CUDA(cudaEventCreateWithFlags(&a->ev_ipc, cudaEventDisableTiming | cudaEventInterprocess));
    FM_CUDA(cudaEventRecord(a->ev_ipc, c->stream));  // after everything queued for the agent
    const uint8_t* base = static_cast<const uint8_t*>(a->slot->base);
    auto off = [&](const void* q) { return static_cast<uint64_t>(static_cast<const uint8_t*>(q) - base); };
    MigrateBlob b{};
    b.magic = kMigrateMagic;
    b.precision = a->precision;
    b.V = a->V;
    b.D = a->D;
    b.src_device = c->device;
    b.dw_valid = a->dw_valid;
    b.cm_valid = a->W16 && a->cm_gen == a->w16_gen;
    b.step = a->step;
    b.version = a->version;
    b.samples = a->samples;
    b.off_w = off(a->W);
    b.off_m = off(a->m);
    b.off_v = off(a->v);
    b.off_dw = off(a->dW);
    b.off_w16 = a->W16 ? off(a->W16) : 0;
    b.off_cm = a->colmax ? off(a->colmax) : 0;
    FM_CUDA(cudaIpcGetMemHandle(&b.mem, a->slot->base));
    FM_CUDA(cudaIpcGetEventHandle(&b.ev, a->ev_ipc));
    std::memcpy(blob_out, &b, sizeof(b));
    if (!share) {
        a->active = false;  // lent: the slot stays reserved until fm_agent_migrate_release
        a->lent = true;
    }
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_migrate_release(fm_agent* a) {
    FM_GUARD_BEGIN
    if (!a->lent) return fail(FM_ERR_CONFIG_ERROR, a->name + " was not exported");
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    agent_free_device(a, c->stream);
    a->lent = false;
    a->ctx = nullptr;
    a->dw_valid = false;
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_migrate_import(fm_agent* a, fm_ctx* c, const uint8_t* blob, uint64_t len) {
    FM_GUARD_BEGIN
    if (len != sizeof(MigrateBlob)) return fail(FM_ERR_INVALID_ARG, "migration blob size mismatch");
    MigrateBlob b;
    std::memcpy(&b, blob, sizeof(b));
    if (b.magic != kMigrateMagic) return fail(FM_ERR_INVALID_ARG, "not a migration blob");
    if (b.V != a->V || b.D != a->D || b.precision != a->precision)
        return fail(FM_ERR_CONFIG_ERROR, "migration blob describes another model shape/precision");
    if (!a->active || a->ctx != c) return fail(FM_ERR_INACTIVE_GROUP, a->name + " must be active on the target GPU");
    if (a->gang) return fail(FM_ERR_BUSY_GROUP, a->name + " is attached to a DP gang");
    if (int st = set_dev(c)) return st;
    void* src = nullptr;
    if (int st = ipc_open_cached(c, b.mem, &src)) return st;
    cudaEvent_t ev = nullptr;
    FM_CUDA(cudaIpcOpenEventHandle(&ev, b.ev));
    // after everything already queued on the agent's slot, and after the source's queued work
    FM_CUDA(cudaEventRecord(a->ev_compute, c->stream));
    FM_CUDA(cudaStreamWaitEvent(c->copy_in, a->ev_compute, 0));
    FM_CUDA(cudaStreamWaitEvent(c->copy_in, ev, 0));
    const size_t P = a->P;
    const uint8_t* p = static_cast<const uint8_t*>(src);
    auto cp = [&](void* dst, uint64_t off, size_t n) {
        return cudaMemcpyPeerAsync(dst, c->device, p + off, b.src_device, n, c->copy_in);
    };
    FM_CUDA(cp(a->W, b.off_w, P * 8));
    FM_CUDA(cp(a->m, b.off_m, P * 4));
    FM_CUDA(cp(a->v, b.off_v, P * 4));
    if (b.dw_valid) FM_CUDA(cp(a->dW, b.off_dw, P * dw_elem(a)));
    if (a->W16) FM_CUDA(cp(a->W16, b.off_w16, P * 2));
    if (a->W16 && b.cm_valid) FM_CUDA(cp(a->colmax, b.off_cm, a->D * 4));
    FM_CUDA(cudaEventRecord(a->ev_in, c->copy_in));
    a->dw_valid = b.dw_valid;
    a->step = b.step;
    a->version = b.version;
    a->samples = b.samples;
    ++a->w16_gen;
    a->cm_gen = (a->W16 && b.cm_valid) ? a->w16_gen : ~0ull;
    a->pending_in = true;  // consumers wait lazily (check_active)
    // the source may release its slot once this returns
    FM_CUDA(cudaEventSynchronize(a->ev_in));
    cudaEventDestroy(ev);
    return FM_OK;
    FM_GUARD_END
}

int fm_agent_state_checksum(fm_agent* a, uint64_t* out) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    if (int st = set_dev(a->ctx)) return st;
    FM_CUDA(cudaStreamSynchronize(a->ctx->stream));
    const size_t P = a->P;
    std::vector<uint8_t> buf(P * (16 + dw_elem(a)));
    FM_CUDA(cudaMemcpy(buf.data(), a->W, P * 8, cudaMemcpyDeviceToHost));
    FM_CUDA(cudaMemcpy(buf.data() + P * 8, a->m, P * 4, cudaMemcpyDeviceToHost));
    FM_CUDA(cudaMemcpy(buf.data() + P * 12, a->v, P * 4, cudaMemcpyDeviceToHost));
    if (a->dw_valid) FM_CUDA(cudaMemcpy(buf.data() + P * 16, a->dW, P * dw_elem(a), cudaMemcpyDeviceToHost));
    else std::fill(buf.begin() + P * 16, buf.end(), 0);
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint8_t b : buf) {
        h ^= b;
        h *= 0x100000001b3ULL;
    }
    for (int64_t x : {a->step, a->version, a->samples}) {
        h ^= static_cast<uint64_t>(x);
        h *= 0x100000001b3ULL;
    }
    *out = h;
    return FM_OK;
    FM_GUARD_END
}

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

// ---------------------------------------------------------------------------
// NCCL gang
// ---------------------------------------------------------------------------
struct fm_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    fm_ctx* ctx = nullptr;
};

#define FM_NCCL(expr)                                                                          \
    do {                                                                                       \
        ncclResult_t _r = (expr);                                                              \
        if (_r != ncclSuccess) return fail(FM_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
    } while (0)

int fm_comm_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    FM_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return FM_OK;
}

int fm_comm_create(fm_ctx* c, const uint8_t id_bytes[128], int nranks, int rank, fm_comm** out) {
    FM_GUARD_BEGIN
    if (int st = set_dev(c)) return st;
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, 128);
    auto* cm = new fm_comm();
    cm->nranks = nranks;
    cm->rank = rank;
    cm->ctx = c;
    const ncclResult_t r = ncclCommInitRank(&cm->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete cm;
        return fail(FM_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    *out = cm;
    return FM_OK;
    FM_GUARD_END
}

int fm_comm_destroy(fm_comm* c) {
    if (!c) return FM_OK;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
    return FM_OK;
}

}  // extern "C"

static ncclComm_t gang_comm(GangState* gs) { return gs->comm->comm; }

static int gang_barrier(fm_agent* a) {
    GangState* gs = a->gang;
    FM_NCCL(ncclAllReduce(gs->d_token, gs->d_token, 1, ncclInt32, ncclSum, gs->comm->comm, a->ctx->stream));
    return FM_OK;
}

namespace {
struct GangBlob {
    int32_t rank;
    int32_t pad;
    cudaIpcMemHandle_t recv;
    cudaIpcMemHandle_t slot;
    uint64_t w16_off;
};
}  // namespace

extern "C" {

// Puts the agent into a DP gang with the fused reduce-scatter (see GangState).
// Writes this rank's export blob (IPC handles of its receive buffer and of
// its training slot's bf16 shadow) for the caller to all-gather across the
// gang and hand to fm_gang_connect.  The agent must stay resident (no
// suspend) while attached.
int fm_gang_attach(fm_agent* a, fm_comm* cm, uint8_t* blob_out, uint64_t cap, uint64_t* len) {
    FM_GUARD_BEGIN
    *len = sizeof(GangBlob);
    if (!blob_out) return FM_OK;
    if (cap < sizeof(GangBlob)) return fail(FM_ERR_INVALID_ARG, "blob buffer too small");
    if (int st = check_active(a)) return st;
    if (a->precision != FM_PRECISION_BF16_TC) return fail(FM_ERR_CONFIG_ERROR, "gang exchange needs the tensor-core path");
    if (cm->ctx != a->ctx) return fail(FM_ERR_CONFIG_ERROR, "communicator bound to another GPU");
    if (cm->nranks < 2 || cm->nranks > 8) return fail(FM_ERR_CONFIG_ERROR, "gang size must be 2..8");
    if (!gemm_pair_mode()) return fail(FM_ERR_CONFIG_ERROR, "gang exchange needs the CTA-pair GEMM (FM_GEMM_2SM)");
    if (int st = set_dev(a->ctx)) return st;
    auto* gs = new GangState();
    gs->comm = cm;
    gs->rank = cm->rank;
    gs->g = cm->nranks;
    const int64_t tiles = static_cast<int64_t>((a->V + 255) / 256);
    for (int o = 0; o <= gs->g; ++o)
        gs->lo[o] = std::min<int64_t>(static_cast<int64_t>(a->V), (tiles * o / gs->g) * 256);
    int64_t max_rows = 0;
    for (int o = 0; o < gs->g; ++o) max_rows = std::max(max_rows, gs->lo[o + 1] - gs->lo[o]);
    const int64_t own = gs->lo[gs->rank + 1] - gs->lo[gs->rank];
    const size_t rbytes = static_cast<size_t>(gs->g - 1) * std::max<int64_t>(own, 1) * a->D * 4;
    fm_ctx* c = a->ctx;
    void* rb = nullptr;
    void* tk = nullptr;
    if (int st = pool_take(c, rbytes, &rb)) {
        delete gs;
        return st;
    }
    if (int st = pool_take(c, 256, &tk)) {
        pool_give(c, rb);
        delete gs;
        return st;
    }
    gs->recv = static_cast<float*>(rb);
    gs->d_token = static_cast<int*>(tk);
    FM_CUDA(cudaMemset(gs->d_token, 0, sizeof(int)));
    GangBlob b{};
    b.rank = gs->rank;
    FM_CUDA(cudaIpcGetMemHandle(&b.recv, gs->recv));
    FM_CUDA(cudaIpcGetMemHandle(&b.slot, a->slot->base));
    b.w16_off = static_cast<uint64_t>(reinterpret_cast<uint8_t*>(a->W16) - static_cast<uint8_t*>(a->slot->base));
    std::memcpy(blob_out, &b, sizeof(b));
    a->gang = gs;
    a->shard_rank = gs->rank;  // token-balanced row shards of every micro-batch
    a->shard_count = gs->g;
    a->dp = true;
    return FM_OK;
    FM_GUARD_END
}

// blobs: the gang's export blobs in rank order (nranks x blob_len bytes).
int fm_gang_connect(fm_agent* a, const uint8_t* blobs, uint64_t blob_len) {
    FM_GUARD_BEGIN
    GangState* gs = a->gang;
    if (!gs) return fail(FM_ERR_CONFIG_ERROR, "fm_gang_attach first");
    if (blob_len != sizeof(GangBlob)) return fail(FM_ERR_INVALID_ARG, "blob size mismatch");
    if (int st = set_dev(a->ctx)) return st;
    for (int o = 0; o < gs->g; ++o) {
        GangBlob b;
        std::memcpy(&b, blobs + o * blob_len, sizeof(b));
        if (b.rank != o) return fail(FM_ERR_INVALID_ARG, "blobs must be in rank order");
        if (o == gs->rank) continue;
        void* rbase = nullptr;
        void* sbase = nullptr;
        if (int st = ipc_open_cached(a->ctx, b.recv, &rbase)) return st;
        if (int st = ipc_open_cached(a->ctx, b.slot, &sbase)) return st;
        // my slot in o's receive buffer: senders in rank order, skipping o itself
        const int idx = gs->rank < o ? gs->rank : gs->rank - 1;
        const int64_t o_rows = gs->lo[o + 1] - gs->lo[o];
        gs->peer_slot[o] = static_cast<float*>(rbase) + static_cast<size_t>(idx) * o_rows * a->D;
        gs->peer_w16[o] = reinterpret_cast<__nv_bfloat16*>(static_cast<uint8_t*>(sbase) + b.w16_off);
        gs->peer_base[o] = static_cast<uint8_t*>(sbase);
    }
    gs->connected = true;
    return FM_OK;
    FM_GUARD_END
}

}  // extern "C"

// A DP-gang agent maintains W / m / v only on its own row shard (the sharded
// K-adam); the other rows live in the owners' slots, mapped over NVLink at
// connect.  Outside a gang this is one contiguous copy.
static int copy_state(fm_agent* a, size_t off, size_t elem, void* dst, cudaStream_t s) {
    const uint8_t* mine = static_cast<const uint8_t*>(a->slot->base) + off;
    GangState* gs = a->gang;
    if (!gs || !gs->connected) {
        FM_CUDA(cudaMemcpyAsync(dst, mine, a->P * elem, cudaMemcpyDefault, s));
        return FM_OK;
    }
    const size_t row = a->D * elem;
    for (int o = 0; o < gs->g; ++o) {
        const int64_t r0 = gs->lo[o], r1 = gs->lo[o + 1];
        if (r1 <= r0) continue;
        const uint8_t* src = (o == gs->rank ? mine : gs->peer_base[o] + off) + static_cast<size_t>(r0) * row;
        FM_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + static_cast<size_t>(r0) * row, src,
                                static_cast<size_t>(r1 - r0) * row, cudaMemcpyDefault, s));
    }
    return FM_OK;
}

extern "C" {

// Pulls every peer's W / m / v rows into this rank's slot over NVLink (the gang's
// sharded Adam keeps only the own rows current there), so that after
// fm_gang_detach this rank holds the agent's whole training state.  The bf16
// shadow is replicated already.  Caller: all gang ranks idle (host barrier).
int fm_gang_gather_state(fm_agent* a) {
    FM_GUARD_BEGIN
    if (int st = check_active(a)) return st;
    GangState* gs = a->gang;
    if (!gs || !gs->connected) return fail(FM_ERR_CONFIG_ERROR, a->name + " is not in a connected DP gang");
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    const size_t offs[3] = {0, slot_off_m(a), slot_off_v(a)};
    const size_t elems[3] = {8, 4, 4};
    for (int k = 0; k < 3; ++k) {
        const size_t row = a->D * elems[k];
        uint8_t* mine = static_cast<uint8_t*>(a->slot->base) + offs[k];
        for (int o = 0; o < gs->g; ++o) {
            const int64_t r0 = gs->lo[o], r1 = gs->lo[o + 1];
            if (o == gs->rank || r1 <= r0) continue;
            FM_CUDA(cudaMemcpyAsync(mine + static_cast<size_t>(r0) * row,
                                    gs->peer_base[o] + offs[k] + static_cast<size_t>(r0) * row,
                                    static_cast<size_t>(r1 - r0) * row, cudaMemcpyDefault, c->stream));
        }
    }
    FM_CUDA(cudaStreamSynchronize(c->stream));
    return FM_OK;
    FM_GUARD_END
}

int fm_gang_detach(fm_agent* a) {
    GangState* gs = a->gang;
    if (!gs) return FM_OK;
    if (a->ctx) {
        cudaSetDevice(a->ctx->device);
        cudaStreamSynchronize(a->ctx->stream);
    }
    // mappings stay in the context's cache; the buffers go back to its pool
    if (a->ctx) {
        pool_give(a->ctx, gs->recv);
        pool_give(a->ctx, gs->d_token);
    } else {
        cudaFree(gs->recv);
        cudaFree(gs->d_token);
    }
    delete gs;
    a->gang = nullptr;
    a->shard_rank = 0;
    a->shard_count = 1;
    a->dp = false;
    return FM_OK;
}

int fm_agent_allreduce_grad(fm_agent* a, fm_comm* cm) {
    if (int st = check_active(a)) return st;
    if (a->gang && a->gang->connected) return FM_OK;  // already reduced inside the last GEMM2
    if (cm->ctx != a->ctx) return fail(FM_ERR_CONFIG_ERROR, "communicator bound to another GPU");
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    if (!a->dw_valid) FM_CUDA(cudaMemsetAsync(a->dW, 0, a->P * dw_elem(a), c->stream));
    a->dw_valid = true;
    a->dp = cm->nranks > 1;
    FM_NCCL(ncclAllReduce(a->dW, a->dW, a->P, a->precision == FM_PRECISION_PARITY_F64 ? ncclFloat64 : ncclFloat32,
                          ncclSum, cm->comm, c->stream));
    return FM_OK;
}

}  // extern "C"

// ===========================================================================
// §8f next rows: weight publish / rollout sync (f1) and the byte-compatible
// PolicyState wire format (f2)
// ===========================================================================
struct fm_weights {
    int device = -1;
    void* buf = nullptr;
    uint64_t rows = 0, cols = 0;
    int dtype = 0;  // 0 f64, 1 f32, 2 bf16, 3 f64 transposed [D][V] (rollout layout)
    int64_t version = 0;
    uint64_t nbytes = 0;
};

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
    } else if (a->W16) {
        // the bf16 shadow IS bf16(W) (same double -> float -> bf16 rounding; full replica in a gang)
        FM_CUDA(cudaMemcpyAsync(w->buf, a->W16, a->P * 2, cudaMemcpyDeviceToDevice, s));
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
    const ncclDataType_t dt = w->dtype == 0 ? ncclFloat64 : w->dtype == 1 ? ncclFloat32 : ncclBfloat16;
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
        FM_CUDA(launch_to_bf16(a->W, a->W16, P, c->num_sms, s));
        count_launch();
        ++a->w16_gen;
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

// ---------------------------------------------------------------------------
// internal hooks for the on-device experience table (fm_dtable.cu)
// ---------------------------------------------------------------------------
namespace fm {
int ctx_device(const fm_ctx* c) { return c->device; }
cudaStream_t ctx_stream(const fm_ctx* c) { return c->stream; }
uint8_t* ctx_arena(const fm_ctx* c) { return c->arena; }
int ctx_staging(fm_ctx* c, size_t bytes, uint8_t** out, cudaEvent_t* ev) { return staging_acquire(c, bytes, out, ev); }
fm_ctx* agent_ctx(const fm_agent* a) { return a->ctx; }
int agent_check_active(fm_agent* a) { return check_active(a); }

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
    if (int st = check_active(a)) return st;
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

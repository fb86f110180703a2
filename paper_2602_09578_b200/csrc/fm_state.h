// fm_state.h — internal state of the C ABI implementation (device contexts,
// workspaces, agents, DP gangs) and the runtime helpers shared by
// fm_runtime.cu (contexts, agents, the micro-batch pipeline, the update),
// fm_swap.cu (state swap and migration), fm_gang.cu (NCCL communicators and
// DP gangs) and fm_publish.cu (weight publish, PolicyState wire format,
// rollout generation).  Not installed; the public interface is
// include/flexmarl/cabi.h.
#pragma once
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
#include <set>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "fm_gemm.h"
#include "fm_internal.h"
#include "fm_kernels.h"

using namespace fm;


constexpr int kReportRing = 256;
constexpr int kStagingSlots = 4;

// ---- driver entry point for cuTensorMapEncodeTiled (no -lcuda link) -------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
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


// ===========================================================================
// context
// ===========================================================================
struct Workspace {
    int64_t rows_cap = 0;  // Mpad capacity
    uint64_t vocab_cap = 0, feat_cap = 0;
    int32_t* action = nullptr;
    int4* ctx4 = nullptr;
    int32_t* n_ctx = nullptr;
    int32_t* sample = nullptr;
    float *coef = nullptr, *rscale = nullptr, *lse = nullptr, *logp = nullptr, *coef_eff = nullptr;
    float* old_logp = nullptr;
    int64_t old_logp_cap = 0;
    // band formulation (k_band.cu): per row its first context position, per
    // position its feature and its A'/B' slot
    int32_t* q0 = nullptr;
    int32_t *pos_feat = nullptr, *pos_slot = nullptr;
    int64_t pos_cap = 0;
    float* mrow = nullptr;   // per-row softmax bound (1/n) sum_k fmax[f_k] [Mpad]
    float* zact = nullptr;   // the taken token's logit [Mpad]
    double* lossw = nullptr; // the row's loss weight -A / G [Mpad]
    float* stats = nullptr;  // K-stats partial sums exp(z - mrow), [stats_ld][Mpad]
    // segments of K-GEMM2: A' = per-position gradient rows H [kp_cap][ldz] bf16,
    // B' = one-hot [kp_cap][256] bf16
    __nv_bfloat16 *aseg = nullptr, *bseg = nullptr;
    __nv_bfloat16* zero_row = nullptr;  // 2,048 zeros: the W16^T "row" of a missing position
    int32_t *kcount = nullptr, *kseg_off = nullptr, *kiters = nullptr;
    unsigned long long* kseg_rows = nullptr;  // executed GEMM2 K rows, accumulated
    int64_t kp_cap = 0;
    // parity mode scratch
    int64_t prow_cap = 0;
    uint64_t pvocab_cap = 0, pparam_cap = 0;
    double *zscratch = nullptr, *dWmb = nullptr, *logp64 = nullptr;
    SampleDesc* sd = nullptr;
    int sd_cap = 0;
    // K-GEMM2 segment sets 1 .. nsets-1 (set 0 = aseg / bseg / kseg_off / kiters above):
    // the micro-batches of a step whose reduction is batched into one K-GEMM2
    struct SegSet {
        __nv_bfloat16 *aseg = nullptr, *bseg = nullptr;
        int32_t *kseg_off = nullptr, *kiters = nullptr;
    };
    SegSet xset[kGemmMaxBatch - 1];
    int nsets = 1;
    float* dpn = nullptr;  // exact DP grad norm: this micro-batch's contribution [P]
    uint64_t dpn_cap = 0;
    float* lse_red = nullptr;  // vocabulary gang: per-row (sum, taken logit) partials [2][cap]
    int64_t lse_red_cap = 0;
};

// Per-kernel device timing (bench.py's roofline): event pairs recorded on the
// launching stream around each hot-path kernel when enabled.
// gather = K-gather + K-pos + K-pslot; stats = K-stats (pass A); band = K-band (pass B)
enum KKind { K_GATHER = 0, K_STATS, K_LSE, K_BAND, K_GEMM2, K_ADAM, K_PARITY, K_MEMSET, K_NKINDS };
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

// One training slot: the device home of an active agent's {W, m, v, dW, W16^T}.
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
    // the latest K-stats launch on the compute stream (swap copies start there, see
    // fm_agent_suspend) and the op sequence numbers that say what it follows
    cudaEvent_t ev_gemm = nullptr;
    // micro-batches of pend_agent whose K-GEMM2 is batched (deferred): their segment
    // set in the workspace and report slot; agent_flush runs them as one launch
    struct PendingMB {
        int set, slot;
    };
    fm_agent* pend_agent = nullptr;
    PendingMB pend[kGemmMaxBatch];
    int npend = 0;
    int64_t pend_rows_per_block = 0;  // context positions per 256-feature block (segment length)
    std::map<std::string, void*> ipc_cache;  // peer buffers mapped over NVLink (slots, gang receive buffers)
    std::vector<std::pair<size_t, void*>> recv_pool;  // gang receive buffers + barrier tokens, recycled
    std::unordered_map<void*, size_t> pool_sizes;
    uint64_t op_seq = 0, gemm_seq = 0;
    uint8_t* arena = nullptr;
    uint64_t arena_cap = 0, arena_used = 0;
    std::unordered_map<uint64_t, uint64_t> arena_ntok;  // offset -> token count
    Workspace ws;
    // pinned staging (sample descriptors, host payloads) with reuse events
    uint8_t* staging[kStagingSlots] = {};
    size_t staging_cap[kStagingSlots] = {};
    cudaEvent_t staging_ev[kStagingSlots] = {};
    int staging_next = 0;
    // arena region reserved for the end-to-end host path
    uint64_t e2e_off = 0, e2e_cap = 0;
};


namespace fm {
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
}  // namespace fm

// ===========================================================================
// agents
// ===========================================================================
// DP gang of an agent with the fused reduce-scatter: V rows are
// split into g contiguous, 256-row-aligned shards; during the step's last
// micro-batch GEMM2 writes the partials of rows owned by another rank into
// that rank's receive slot over NVLink (IPC-mapped), then each rank runs the
// sharded Adam on its rows and writes the new bf16 rows into every peer's
// W16^T.  Two 1-element NCCL all-reduces on the compute stream serve as the
// device-side barriers (after the exchange; the update grad-norm reduction
// after Adam), so no host round trip or spin-wait is involved.
#define FM_NCCL(expr)                                                                          \
    do {                                                                                       \
        ncclResult_t _r = (expr);                                                              \
        if (_r != ncclSuccess) return fail(FM_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
    } while (0)

struct fm_comm;
struct GangState;
ncclComm_t gang_comm(GangState* gs);
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
    // vocabulary-parallel mode (fm_gang_attach_mode 1): every rank trains ALL rows of
    // each micro-batch on its vocabulary range [lo[rank], lo[rank+1]) — K-stats /
    // K-band on those columns, K-GEMM2 and K-adam on those rows of dW / W, its own
    // W16^T columns; per micro-batch only the rows' partial softmax sums and the taken
    // tokens' logits are all-reduced (2 x Mpad floats), plus the micro-batch's
    // squared gradient norm.  No bulk NVLink traffic, no receive buffers.
    bool vocab = false;
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
    __nv_bfloat16* W16 = nullptr;   // transposed bf16 shadow W16^T [D][ldw] (tensor-core mode)
    float* fmax = nullptr;          // fmax[f] = max_v W16^T[f][v] (K-stats' per-row softmax bound)
    bool fmax_valid = false;        // fmax describes the current shadow
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
    // PPO clip: old log-probs of the next micro-batch's packed rows (host copy,
    // uploaded by train_impl after the workspace is reserved)
    float clip_eps = 0.f;
    std::vector<float> old_logp;
    // GradKey bookkeeping of the current global step (training.hpp:87-91, 396-401)
    std::set<std::tuple<std::string, int, int, int64_t>> grad_keys;
    // swap
    bool active = false;
    int park_tier = -1;
    int park_device = -1;
    void* park = nullptr;  // W | m | v | dW   (host pinned or device)
    size_t park_bytes = 0;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_compute = nullptr;
    cudaEvent_t ev_ipc = nullptr;  // interprocess: the source's work before a migration is done
    int ev_device = -1;            // the device the agent's events were created on
    fm_comm* norm_comm = nullptr;  // exact DP micro-batch grad norms over this communicator
    bool lent = false;             // exported by migration; slot reserved until migrate_release
    // fm_agent_migrate_import_rows: only W / m / v rows [part_lo, part_hi) are this agent's —
    // usable solely as that rank of a vocabulary-parallel gang (check_active refuses otherwise)
    bool partial = false;
    int64_t part_lo = 0, part_hi = 0;
    Slot* slot = nullptr;
    GangState* gang = nullptr;
};

// Device-side barrier across the gang (defined with the NCCL section below).
int gang_barrier(fm_agent* a);
// Copies a full [V][D] state buffer (slot offset off, elem bytes/param) to dst
// (host or device), gathering a DP gang's row shards (defined below).
int copy_state(fm_agent* a, size_t off, size_t elem, void* dst, cudaStream_t s);

// An NCCL communicator bound to a device context (fm_gang.cu).
struct fm_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    fm_ctx* ctx = nullptr;
};

// A published weight buffer (fm_publish.cu; read by the generation hook).
struct fm_weights {
    int device = -1;
    void* buf = nullptr;
    uint64_t rows = 0, cols = 0;
    int dtype = 0;  // 0 f64, 1 f32, 2 bf16, 3 f64 transposed [D][V] (rollout layout)
    int64_t version = 0;
    uint64_t nbytes = 0;
};

// ---- runtime helpers (fm_runtime.cu) shared by the ABI translation units ----
namespace fm {
int set_dev(const fm_ctx* c);
int ipc_open_cached(fm_ctx* c, const cudaIpcMemHandle_t& h, void** out);
int pool_take(fm_ctx* c, size_t bytes, void** out);
void pool_give(fm_ctx* c, void* p);
int staging_acquire(fm_ctx* c, size_t bytes, uint8_t** out, cudaEvent_t* ev);
void ws_free(Workspace& w);
uint64_t round_up(uint64_t x, uint64_t m);
int ws_reserve_tc(fm_ctx* c, int64_t Mpad, uint64_t V, uint64_t D, int n_samples);
int ws_reserve_rows(fm_ctx* c, int64_t R);
int ws_reserve_parity(fm_ctx* c, int64_t M, uint64_t V, uint64_t P);
int ws_reserve_sd(fm_ctx* c, int n);
RowBuffers row_buffers(Workspace& w);
size_t dw_elem(const fm_agent* a);
size_t align256(size_t x);
size_t slot_off_m(const fm_agent* a);
size_t slot_off_v(const fm_agent* a);
size_t slot_bytes(const fm_agent* a);
uint64_t w16_ld(const fm_agent* a);     // row pitch of W16^T: V rounded up to 8
size_t w16_bytes(const fm_agent* a);    // D * w16_ld * 2
int agent_alloc_device(fm_agent* a, fm_ctx* c, cudaStream_t s);
void agent_free_device(fm_agent* a, cudaStream_t s);
void agent_bind_slot(fm_agent* a, Slot* sl);
void agent_unbind(fm_agent* a);
// flush = true: first run the agent's deferred K-GEMM2 (its dW and reports are complete)
int check_active(fm_agent* a, bool flush = true);
// the deferred K-GEMM2 of the agent / of whichever agent has one pending on the context
int agent_flush(fm_agent* a);
int ctx_flush(fm_ctx* c);
}  // namespace fm

// ---- parking buffers (fm_swap.cu), also written by the fused update-and-park ----
extern "C" {
// Park layout: W | m | v | dW | W16^T.
size_t park_bytes_for(const fm_agent* a);
// Parking buffer of `bytes` on `tier` (device pdev), reused while it fits.
int park_reserve(fm_agent* a, fm_ctx* c, int tier, int pdev, size_t bytes);
}

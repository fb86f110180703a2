// fm_gang.cu — NCCL communicators, DP gangs with the fused GEMM2 reduce-scatter over NVLink peer memory, and the NCCL all-reduce path.
#include "fm_state.h"

extern "C" {

// ---------------------------------------------------------------------------
// NCCL gang
// ---------------------------------------------------------------------------
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

ncclComm_t gang_comm(GangState* gs) { return gs->comm->comm; }

int gang_barrier(fm_agent* a) {
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
    return fm_gang_attach_mode(a, cm, 0, blob_out, cap, len);
}

int fm_gang_attach_mode(fm_agent* a, fm_comm* cm, int mode, uint8_t* blob_out, uint64_t cap, uint64_t* len) {
    FM_GUARD_BEGIN
    if (mode != 0 && mode != 1) return fail(FM_ERR_INVALID_ARG, "gang mode must be 0 (token shards) or 1 (vocabulary)");
    *len = sizeof(GangBlob);
    if (!blob_out) return FM_OK;
    if (cap < sizeof(GangBlob)) return fail(FM_ERR_INVALID_ARG, "blob buffer too small");
    if (a->partial) {  // row-range import: nothing queued yet, its rows must be this rank's
        if (!a->active || !a->ctx) return fail(FM_ERR_INACTIVE_GROUP, a->name);
    } else if (int st = check_active(a)) {
        return st;
    }
    if (a->precision != FM_PRECISION_BF16_TC) return fail(FM_ERR_CONFIG_ERROR, "gang exchange needs the tensor-core path");
    if (cm->ctx != a->ctx) return fail(FM_ERR_CONFIG_ERROR, "communicator bound to another GPU");
    if (cm->nranks < 2 || cm->nranks > 8) return fail(FM_ERR_CONFIG_ERROR, "gang size must be 2..8");
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
    gs->vocab = mode == 1;
    if (a->partial && (!gs->vocab || a->part_lo != gs->lo[gs->rank] || a->part_hi != gs->lo[gs->rank + 1])) {
        const std::string want = std::to_string(gs->lo[gs->rank]) + ", " + std::to_string(gs->lo[gs->rank + 1]);
        delete gs;
        return fail(FM_ERR_CONFIG_ERROR, a->name + ": imported rows are not this rank's vocabulary range [" + want + ")");
    }
    // the vocabulary-parallel gang exchanges no partial gradients: a token receive buffer only
    const size_t rbytes = gs->vocab ? 256 : static_cast<size_t>(gs->g - 1) * std::max<int64_t>(own, 1) * a->D * 4;
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
    // token-balanced row shards of every micro-batch (mode 0); mode 1 trains every row
    a->shard_rank = gs->vocab ? 0 : gs->rank;
    a->shard_count = gs->vocab ? 1 : gs->g;
    a->dp = !gs->vocab;  // the vocabulary-parallel gang reports exact micro-batch grad norms
    a->fmax_valid = false;
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
        gs->peer_slot[o] = gs->vocab ? nullptr : static_cast<float*>(rbase) + static_cast<size_t>(idx) * o_rows * a->D;
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
int copy_state(fm_agent* a, size_t off, size_t elem, void* dst, cudaStream_t s) {
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
    if (gs->vocab && a->W16) {
        // each rank kept only its own W16^T columns: rebuild the whole shadow from W
        FM_CUDA(launch_w16t(a->W, a->V, a->D, a->W16, w16_ld(a), c->num_sms, c->stream));
        a->fmax_valid = false;
    }
    FM_CUDA(cudaStreamSynchronize(c->stream));
    a->partial = false;  // every row is here now
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
    a->fmax_valid = false;
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


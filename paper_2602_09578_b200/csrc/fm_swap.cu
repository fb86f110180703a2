// fm_swap.cu — training-state swap (suspend / activate / update-and-park) and cross-process agent migration over NVLink (training.hpp:99-165, 259-350).
#include "fm_state.h"

extern "C" {

// ---------------------------------------------------------------------------
// training-state swap
// ---------------------------------------------------------------------------
// Park layout: W | m | v | dW | W16^T.
size_t park_bytes_for(const fm_agent* a) {
    return a->P * 16 + a->P * dw_elem(a) + (a->W16 ? w16_bytes(a) : 0);
}

// Parking buffer of `bytes` on `tier` (device pdev), reused while it fits.
int park_reserve(fm_agent* a, fm_ctx* c, int tier, int pdev, size_t bytes) {
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
    // a K-stats launched after the agent's last op (e.g. the next agent's first
    // micro-batch) is a safe and cheap start for the copy-out: the copy engines then
    // overlap the streaming passes instead of the latency-bound K-gather that follows
    // the end of the currently queued work (measured with the earlier GEMM1 pipeline:
    // K-gather 16 us -> 390 us beside a 2.4 GB D2D copy)
    const bool gated = a->active && a->ctx && a->ctx->gemm_seq > a->last_seq;
    if (int st = check_active(a)) return st;
    if (a->gang) return fail(FM_ERR_BUSY_GROUP, a->name + " is attached to a DP gang (fm_gang_detach first)");
    fm_ctx* c = a->ctx;
    if (int st = set_dev(c)) return st;
    const size_t P = a->P;
    const size_t dwb = a->dw_valid ? P * dw_elem(a) : 0;
    // park layout: W | m | v | dW | W16^T.  The bf16 shadow travels on the HBM /
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
    if (park_w16) FM_CUDA(cp(p + P * (16 + dw_elem(a)), a->W16, w16_bytes(a)));
    a->park_w16 = park_w16;
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
    // the parked copy must have landed before we read it back (a cross-device wait when
    // the agent comes back on another GPU)
    FM_CUDA(cudaStreamWaitEvent(c->copy_in, a->ev_out, 0));
    if (a->ev_device != c->device) {
        // CUDA events can only be recorded on their own device's streams: re-create the
        // agent's events on the new GPU once everything recorded on the old ones is done
        for (int i = 0; i < kReportRing; ++i) FM_CUDA(cudaEventSynchronize(a->ev[i]));
        FM_CUDA(cudaEventSynchronize(a->ev_out));
        for (int i = 0; i < kReportRing; ++i) {
            cudaEventDestroy(a->ev[i]);
            FM_CUDA(cudaEventCreateWithFlags(&a->ev[i], cudaEventDisableTiming));
        }
        cudaEventDestroy(a->ev_in);
        cudaEventDestroy(a->ev_out);
        cudaEventDestroy(a->ev_compute);
        FM_CUDA(cudaEventCreateWithFlags(&a->ev_in, cudaEventDisableTiming));
        FM_CUDA(cudaEventCreateWithFlags(&a->ev_out, cudaEventDisableTiming));
        FM_CUDA(cudaEventCreateWithFlags(&a->ev_compute, cudaEventDisableTiming));
        if (a->ev_ipc) {
            cudaEventDestroy(a->ev_ipc);
            a->ev_ipc = nullptr;
        }
        // the report / update scalars the kernels write live on the agent's GPU too
        cudaFree(a->d_scalars);
        cudaFree(a->d_upd);
        a->d_scalars = nullptr;
        a->d_upd = nullptr;
        FM_CUDA(cudaMalloc(&a->d_scalars, kReportRing * 2 * sizeof(double)));
        FM_CUDA(cudaMalloc(&a->d_upd, sizeof(double)));
        a->ev_device = c->device;
    }
    // start the copy-in beside the latest queued K-stats rather than beside whatever
    // runs when it is issued: the latency-bound gather / slot kernels slowed 4x next to
    // a copy-engine burst (119 vs 28 us per micro-batch, earlier GEMM1 pipeline)
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
        FM_CUDA(cp(a->W16, p + P * (16 + dw_elem(a)), w16_bytes(a)));
    } else if (a->W16) {
        FM_CUDA(launch_w16t(a->W, a->V, a->D, a->W16, w16_ld(a), c->num_sms, c->copy_in));  // shadow regenerated
        count_launch();
    }
    FM_CUDA(cudaEventRecord(a->ev_in, c->copy_in));
    a->fmax_valid = false;
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
    uint8_t dw_valid, pad0, pad1, pad2;
    int64_t step, version, samples;
    uint64_t off_w, off_m, off_v, off_dw, off_w16;  // within the slot
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
    b.step = a->step;
    b.version = a->version;
    b.samples = a->samples;
    b.off_w = off(a->W);
    b.off_m = off(a->m);
    b.off_v = off(a->v);
    b.off_dw = off(a->dW);
    b.off_w16 = a->W16 ? off(a->W16) : 0;
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

namespace {
// rows [r0, r1) of W / m / v / dW (the whole shadow always: a vocabulary gang rank streams
// its columns of every feature row)
int migrate_import_range(fm_agent* a, fm_ctx* c, const uint8_t* blob, uint64_t len, uint64_t r0, uint64_t r1) {
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
    (void)P;
    const uint64_t e0 = r0 * a->D, ne = (r1 - r0) * a->D;  // element range of the rows
    FM_CUDA(cp(a->W + e0, b.off_w + e0 * 8, ne * 8));
    FM_CUDA(cp(a->m + e0, b.off_m + e0 * 4, ne * 4));
    FM_CUDA(cp(a->v + e0, b.off_v + e0 * 4, ne * 4));
    if (b.dw_valid)
        FM_CUDA(cp(static_cast<uint8_t*>(a->dW) + e0 * dw_elem(a), b.off_dw + e0 * dw_elem(a), ne * dw_elem(a)));
    if (a->W16) FM_CUDA(cp(a->W16, b.off_w16, w16_bytes(a)));
    FM_CUDA(cudaEventRecord(a->ev_in, c->copy_in));
    a->partial = r0 != 0 || r1 != a->V;
    a->part_lo = static_cast<int64_t>(r0);
    a->part_hi = static_cast<int64_t>(r1);
    a->dw_valid = b.dw_valid;
    a->step = b.step;
    a->version = b.version;
    a->samples = b.samples;
    a->fmax_valid = false;
    a->pending_in = true;  // consumers wait lazily (check_active)
    // the source may release its slot once this returns
    FM_CUDA(cudaEventSynchronize(a->ev_in));
    cudaEventDestroy(ev);
    return FM_OK;
    FM_GUARD_END
}
}  // namespace

int fm_agent_migrate_import(fm_agent* a, fm_ctx* c, const uint8_t* blob, uint64_t len) {
    return migrate_import_range(a, c, blob, len, 0, a ? a->V : 0);
}

int fm_agent_migrate_import_rows(fm_agent* a, fm_ctx* c, const uint8_t* blob, uint64_t len, uint64_t row_lo,
                                 uint64_t row_hi) {
    if (!a || row_lo >= row_hi || row_hi > a->V)
        return fail(FM_ERR_INVALID_ARG, "row range must satisfy row_lo < row_hi <= vocab");
    return migrate_import_range(a, c, blob, len, row_lo, row_hi);
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


}  // extern "C"

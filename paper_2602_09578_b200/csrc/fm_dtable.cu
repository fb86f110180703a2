// fm_dtable.cu — host side of the on-device experience table.
//
// Reference: marlsim::ExperienceStore (experience_store.hpp:19-276) and the
// rollout side that feeds it (rollout.hpp:647-653 insert_record, :715-731
// completion, :812-834 release_group).  The table's data lives in HBM
// (k_store.cu); this file keeps the host key index the reference's synchronous
// errors need and sequences every table op on the table's own stream.
//
// What stays on the host: (input_id, turns, traj, version) -> slot, per-slot
// status bits and processing flag (mirrors, to raise DuplicateSample,
// RecordNotFound, CellAlreadySet, NotProcessing before any state change, as
// the reference does), and the order-preserving labels of input_ids.
// What never leaves HBM: cell values, payloads, the poll's selection input,
// rewards/advantages computed at group release, generated responses, and the
// micro-batch descriptors the trainer consumes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "flexmarl/cabi.h"
#include "fm_internal.h"
#include "fm_kernels.h"
#include "fm_store.h"

using fm::fail;

namespace {

constexpr int kRing = 8;  // poll descriptor sets kept for fm_train_polled
enum ColType { kInt = 0, kFloat = 1, kBool = 2, kString = 3, kList = 4, kTensor = 5 };
bool by_value(int ty) { return ty == kInt || ty == kFloat || ty == kBool; }  // sample.hpp:71-73

using RecordKey = std::tuple<std::string, int, int, int64_t>;  // experience_store.hpp:242

struct HostRec {
    bool live = false;
    bool processing = false;
    std::string id;
    int turns = 0, traj = 0;
    int64_t version = 0;
    uint32_t status = 0;
};

struct LabelEntry {
    uint64_t label;
    int64_t refs;
};

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

std::string render(const std::string& id, int turns, int traj) {
    return id + "_" + std::to_string(turns) + "_" + std::to_string(traj);
}

}  // namespace

struct fm_dtable {
    fm_ctx* ctx = nullptr;
    std::string agent;
    std::vector<std::string> names;
    std::vector<int> types;
    int cap = 0;
    std::map<RecordKey, int64_t> index;  // canonical order (host mirror of the keys)
    std::vector<HostRec> recs;
    std::vector<int64_t> free_slots;     // stack: lowest slot on top
    std::map<std::string, LabelEntry> labels;
    int64_t live = 0;
    cudaStream_t stream = nullptr;
    // device
    void* dmem = nullptr;
    fm::DTableView view{};
    fm::DPollScratch sc{};
    fm::PollResult* d_res = nullptr;
    fm::PollResult* h_res = nullptr;  // pinned, mapped: the poll's finish kernel writes it directly
    fm::PollResult* m_res = nullptr;  // its device alias
    fm::SampleDesc* d_desc = nullptr; // [kRing][kMaxPollMb]
    unsigned long long* d_cnt = nullptr;
    unsigned long long* h_cnt = nullptr;  // pinned
    int* d_list = nullptr;                // [cap] purge output
    int* h_list = nullptr;                // pinned
    uint8_t* d_scratch = nullptr;         // per-op uploads (stream-ordered reuse)
    size_t scratch_cap = 0;
    // poll ring
    int64_t poll_seq = 0;
    int64_t ring_id[kRing];
    int ring_mb[kRing] = {};
    int64_t ring_rows[kRing] = {};
    cudaEvent_t ring_ready[kRing] = {};
    cudaEvent_t ring_consumed[kRing] = {};
    bool ring_used[kRing] = {};
    cudaEvent_t ev_join = nullptr;

    int col(const char* n) const {
        if (!n) return -1;
        for (size_t i = 0; i < names.size(); ++i)
            if (names[i] == n) return static_cast<int>(i);
        return -1;
    }
    bool live_slot(int64_t s) const { return s >= 0 && s < cap && recs[static_cast<size_t>(s)].live; }
};

namespace {

int set_dev(fm_dtable* t) {
    FM_CUDA(cudaSetDevice(fm::ctx_device(t->ctx)));
    return FM_OK;
}

// Stages `parts` (host pointer, bytes) into the table's device scratch through
// pinned memory, 16-byte aligned each; returns their device addresses.
int upload(fm_dtable* t, std::initializer_list<std::pair<const void*, size_t>> parts, std::vector<void*>* dev) {
    size_t total = 0;
    for (const auto& p : parts) total += align16(p.second);
    if (total == 0) total = 16;
    if (total > t->scratch_cap) {
        FM_CUDA(cudaStreamSynchronize(t->stream));
        if (t->d_scratch) FM_CUDA(cudaFree(t->d_scratch));
        t->scratch_cap = std::max<size_t>(total, 1 << 16);
        FM_CUDA(cudaMalloc(&t->d_scratch, t->scratch_cap));
    }
    uint8_t* stg;
    cudaEvent_t ev;
    if (int st = fm::ctx_staging(t->ctx, total, &stg, &ev)) return st;
    size_t off = 0;
    dev->clear();
    for (const auto& p : parts) {
        if (p.second) std::memcpy(stg + off, p.first, p.second);
        dev->push_back(t->d_scratch + off);
        off += align16(p.second);
    }
    FM_CUDA(cudaMemcpyAsync(t->d_scratch, stg, total, cudaMemcpyHostToDevice, t->stream));
    FM_CUDA(cudaEventRecord(ev, t->stream));
    return FM_OK;
}

// Order-preserving label of a new input_id (order maintenance with gaps; a full
// relabel of the live slots when a gap closes).
int acquire_label(fm_dtable* t, const std::string& id, uint64_t* out, bool* relabel) {
    auto it = t->labels.find(id);
    if (it != t->labels.end()) {
        it->second.refs++;
        *out = it->second.label;
        return FM_OK;
    }
    constexpr uint64_t kStep = 1ull << 40;
    constexpr uint64_t kMax = ~0ull;
    auto nx = t->labels.lower_bound(id);
    const bool has_lo = nx != t->labels.begin();
    const bool has_hi = nx != t->labels.end();
    const uint64_t lo = has_lo ? std::prev(nx)->second.label : 0;
    const uint64_t hi = has_hi ? nx->second.label : kMax;
    uint64_t L = 0;
    bool ok = true;
    if (!has_lo && !has_hi) {
        L = 1ull << 63;
    } else if (!has_hi) {
        const uint64_t room = kMax - lo;
        ok = room >= 2;
        L = lo + std::min(kStep, room / 2);
    } else if (!has_lo) {
        ok = hi >= 2;
        L = hi - std::min(kStep, hi / 2);
    } else {
        ok = hi - lo >= 2;
        L = lo + (hi - lo) / 2;
    }
    if (ok) {
        t->labels.emplace(id, LabelEntry{L, 1});
        *out = L;
        return FM_OK;
    }
    // relabel every id evenly (including the new one)
    t->labels.emplace(id, LabelEntry{0, 1});
    const uint64_t step = kMax / (t->labels.size() + 1);
    uint64_t k = 1;
    for (auto& kv : t->labels) kv.second.label = step * k++;
    *out = t->labels.at(id).label;
    *relabel = true;
    return FM_OK;
}

void release_label(fm_dtable* t, const std::string& id) {
    auto it = t->labels.find(id);
    if (it != t->labels.end() && --it->second.refs == 0) t->labels.erase(it);
}

int push_labels(fm_dtable* t) {
    std::vector<uint64_t> lab(static_cast<size_t>(t->cap), 0);
    for (int s = 0; s < t->cap; ++s)
        if (t->recs[static_cast<size_t>(s)].live) lab[static_cast<size_t>(s)] = t->labels.at(t->recs[static_cast<size_t>(s)].id).label;
    std::vector<void*> d;
    if (int st = upload(t, {{lab.data(), lab.size() * 8}}, &d)) return st;
    FM_CUDA(fm::launch_dt_relabel(t->view, static_cast<const uint64_t*>(d[0]), t->stream));
    fm::count_launch();
    return FM_OK;
}

// host mirror of an erase (complete / purge / drop)
void erase_host(fm_dtable* t, int64_t s) {
    HostRec& r = t->recs[static_cast<size_t>(s)];
    t->index.erase(RecordKey{r.id, r.turns, r.traj, r.version});
    release_label(t, r.id);
    r = HostRec{};
    t->free_slots.push_back(s);
    t->live--;
}

}  // namespace

extern "C" {

int fm_dtable_create(fm_ctx* ctx, const char* agent, const char* const* names, const int* types, int ncols,
                     int64_t capacity, fm_dtable** out) {
    FM_GUARD_BEGIN
    if (!ctx || !out || ncols < 0 || (ncols && (!names || !types))) return fail(FM_ERR_INVALID_ARG, "bad arguments");
    if (capacity < 1 || capacity > (1 << 20)) return fail(FM_ERR_CONFIG_ERROR, "table capacity must be in [1, 2^20]");
    if (ncols > 31) return fail(FM_ERR_CONFIG_ERROR, "at most 31 columns (status bitmask)");
    auto t = std::make_unique<fm_dtable>();
    t->ctx = ctx;
    t->agent = agent ? agent : "";
    for (int i = 0; i < ncols; ++i) {  // experience_store.hpp:26-35
        const std::string n = names[i];
        if (n == "policy_version" || n == "sample_id" || n == "processing")
            return fail(FM_ERR_RESERVED_COLUMN_NAME, n);
        for (int j = 0; j < i; ++j)
            if (n == names[j]) return fail(FM_ERR_CONFIG_ERROR, "duplicate column " + n);
        if (types[i] < kInt || types[i] > kTensor) return fail(FM_ERR_CONFIG_ERROR, "bad column type for " + n);
        t->names.push_back(n);
        t->types.push_back(types[i]);
    }
    t->cap = static_cast<int>(capacity);
    t->recs.assign(static_cast<size_t>(t->cap), HostRec{});
    for (int64_t s = t->cap - 1; s >= 0; --s) t->free_slots.push_back(s);
    if (int st = set_dev(t.get())) return st;
    FM_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    const size_t C = static_cast<size_t>(t->cap);
    const size_t nc = std::max<size_t>(t->names.size(), 1);
    const size_t parts[] = {C * 8, C * 4, C * 4, C * 8, C * 4, C * 4, nc * C * 8, 16, C * 4, C * 4,
                            sizeof(fm::PollResult), sizeof(fm::SampleDesc) * kRing * fm::kMaxPollMb, 16, C * 4};
    size_t total = 0;
    for (size_t p : parts) total += align16(p);
    FM_CUDA(cudaMalloc(&t->dmem, total));
    FM_CUDA(cudaMemsetAsync(t->dmem, 0, total, t->stream));
    uint8_t* p = static_cast<uint8_t*>(t->dmem);
    auto take = [&](size_t i) {
        uint8_t* q = p;
        p += align16(parts[i]);
        return q;
    };
    t->view.label = reinterpret_cast<uint64_t*>(take(0));
    t->view.turns = reinterpret_cast<int32_t*>(take(1));
    t->view.traj = reinterpret_cast<int32_t*>(take(2));
    t->view.version = reinterpret_cast<int64_t*>(take(3));
    t->view.status = reinterpret_cast<unsigned*>(take(4));
    t->view.flags = reinterpret_cast<unsigned*>(take(5));
    t->view.cells = reinterpret_cast<uint64_t*>(take(6));
    t->view.full_mask = t->names.empty() ? 0u : ((1u << t->names.size()) - 1u);
    t->view.cap = t->cap;
    t->sc.count = reinterpret_cast<int*>(take(7));
    t->sc.elist = reinterpret_cast<int*>(take(8));
    t->sc.rank = reinterpret_cast<int*>(take(9));
    t->d_res = reinterpret_cast<fm::PollResult*>(take(10));
    t->d_desc = reinterpret_cast<fm::SampleDesc*>(take(11));
    t->d_cnt = reinterpret_cast<unsigned long long*>(take(12));
    t->d_list = reinterpret_cast<int*>(take(13));
    FM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->h_res), sizeof(fm::PollResult), cudaHostAllocMapped));
    FM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t->m_res), t->h_res, 0));
    FM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->h_cnt), 16, cudaHostAllocDefault));
    FM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->h_list), C * 4, cudaHostAllocDefault));
    for (int k = 0; k < kRing; ++k) {
        t->ring_id[k] = -1;
        FM_CUDA(cudaEventCreateWithFlags(&t->ring_ready[k], cudaEventDisableTiming));
        FM_CUDA(cudaEventCreateWithFlags(&t->ring_consumed[k], cudaEventDisableTiming));
    }
    FM_CUDA(cudaEventCreateWithFlags(&t->ev_join, cudaEventDisableTiming));
    FM_CUDA(cudaStreamSynchronize(t->stream));
    *out = t.release();
    return FM_OK;
    FM_GUARD_END
}

int fm_dtable_destroy(fm_dtable* t) {
    if (!t) return FM_OK;
    cudaSetDevice(fm::ctx_device(t->ctx));
    if (t->stream) cudaStreamSynchronize(t->stream);
    for (int k = 0; k < kRing; ++k) {
        if (t->ring_consumed[k]) cudaEventSynchronize(t->ring_consumed[k]);
        cudaEventDestroy(t->ring_ready[k]);
        cudaEventDestroy(t->ring_consumed[k]);
    }
    cudaEventDestroy(t->ev_join);
    cudaFree(t->dmem);
    cudaFree(t->d_scratch);
    cudaFreeHost(t->h_res);
    cudaFreeHost(t->h_cnt);
    cudaFreeHost(t->h_list);
    if (t->stream) cudaStreamDestroy(t->stream);
    delete t;
    return FM_OK;
}

int fm_dtable_insert(fm_dtable* t, int64_t version, int n, const char* const* ids, const int* turns,
                     const int* trajs, int64_t* slots_out) {
    FM_GUARD_BEGIN
    if (n < 0 || (n > 0 && (!ids || !turns || !trajs))) return fail(FM_ERR_INVALID_ARG, "bad record list");
    std::vector<RecordKey> keys;
    keys.reserve(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {  // experience_store.hpp:46-53, validated before any change
        const std::string id = ids[i] ? ids[i] : "";
        if (id.empty() || id.find('_') != std::string::npos)
            return fail(FM_ERR_BAD_SAMPLE_ID, "input_id may not be empty or contain '_': " + id);
        RecordKey k{id, turns[i], trajs[i], version};
        if (t->index.count(k) || std::find(keys.begin(), keys.end(), k) != keys.end())
            return fail(FM_ERR_DUPLICATE_SAMPLE, render(id, turns[i], trajs[i]) + " v" + std::to_string(version));
        keys.push_back(std::move(k));
    }
    if (static_cast<int64_t>(t->free_slots.size()) < n)
        return fail(FM_ERR_DEVICE_OOM, "device experience table full (capacity " + std::to_string(t->cap) + ")");
    if (n == 0) return FM_OK;
    if (int st = set_dev(t)) return st;
    std::vector<fm::DInsert> recs(static_cast<size_t>(n));
    bool relabel = false;
    for (int i = 0; i < n; ++i) {
        const int64_t s = t->free_slots.back();
        t->free_slots.pop_back();
        HostRec& r = t->recs[static_cast<size_t>(s)];
        r.live = true;
        r.processing = false;
        r.id = std::get<0>(keys[static_cast<size_t>(i)]);
        r.turns = turns[i];
        r.traj = trajs[i];
        r.version = version;
        r.status = 0;
        t->index.emplace(keys[static_cast<size_t>(i)], s);
        t->live++;
        uint64_t L;
        if (int st = acquire_label(t, r.id, &L, &relabel)) return st;
        recs[static_cast<size_t>(i)] = fm::DInsert{L, version, s, turns[i], trajs[i]};
        if (slots_out) slots_out[i] = s;
    }
    if (relabel) {  // labels of earlier records in this batch moved too
        for (auto& d : recs) d.label = t->labels.at(t->recs[static_cast<size_t>(d.slot)].id).label;
    }
    std::vector<void*> d;
    if (int st = upload(t, {{recs.data(), recs.size() * sizeof(fm::DInsert)}}, &d)) return st;
    FM_CUDA(fm::launch_dt_insert(t->view, n, static_cast<const fm::DInsert*>(d[0]), t->stream));
    fm::count_launch();
    if (relabel) return push_labels(t);
    return FM_OK;
    FM_GUARD_END
}

int fm_dtable_find(fm_dtable* t, const char* id, int turns, int traj, int64_t version, int64_t* slot_out) {
    auto it = t->index.find(RecordKey{id ? id : "", turns, traj, version});
    *slot_out = it == t->index.end() ? -1 : it->second;
    return FM_OK;
}

static int check_cells(fm_dtable* t, const char* column, int n, const int64_t* slots, bool want_value, int* col_out) {
    // the reference's order (experience_store.hpp:65-79): column, record, status, storage class
    const int c = t->col(column);
    if (c < 0) return fail(FM_ERR_UNKNOWN_COLUMN, column ? column : "(null)");
    const bool col_by_value = by_value(t->types[static_cast<size_t>(c)]);
    // set_cell_payload registers the payload object first (experience_store.hpp:86); a ref cell
    // set before already owns that sample-field key -> DuplicateKey (object_store.hpp:144-148)
    const int already = (!want_value && !col_by_value) ? FM_ERR_DUPLICATE_KEY : FM_ERR_CELL_ALREADY_SET;
    for (int i = 0; i < n; ++i) {
        if (!t->live_slot(slots[i])) return fail(FM_ERR_RECORD_NOT_FOUND, "slot " + std::to_string(slots[i]));
        const HostRec& r = t->recs[static_cast<size_t>(slots[i])];
        if (r.status & (1u << c)) return fail(already, column);
        for (int j = 0; j < i; ++j)
            if (slots[j] == slots[i]) return fail(already, column);
    }
    if (col_by_value != want_value)
        return fail(FM_ERR_CONFIG_ERROR, std::string("cell storage class mismatch for column ") + column);
    *col_out = c;
    return FM_OK;
}

int fm_dtable_set_float(fm_dtable* t, const char* column, int n, const int64_t* slots, const double* values) {
    FM_GUARD_BEGIN
    if (n < 0 || (n > 0 && (!slots || !values))) return fail(FM_ERR_INVALID_ARG, "bad cell list");
    int c;
    if (int st = check_cells(t, column, n, slots, true, &c)) return st;
    if (n == 0) return FM_OK;
    if (int st = set_dev(t)) return st;
    for (int i = 0; i < n; ++i) t->recs[static_cast<size_t>(slots[i])].status |= 1u << c;
    std::vector<void*> d;
    if (int st = upload(t, {{slots, n * 8u}, {values, n * 8u}}, &d)) return st;
    FM_CUDA(fm::launch_dt_set_cells(t->view, c, n, static_cast<const int64_t*>(d[0]),
                                    static_cast<const uint64_t*>(d[1]), t->stream));
    fm::count_launch();
    return FM_OK;
    FM_GUARD_END
}

int fm_dtable_set_payload(fm_dtable* t, const char* column, int64_t slot, const uint8_t* payload, uint64_t nbytes) {
    FM_GUARD_BEGIN
    int c;
    if (int st = check_cells(t, column, 1, &slot, false, &c)) return st;
    if (!payload || nbytes < 8) return fail(FM_ERR_INVALID_ARG, "payload shorter than its u64 count header");
    uint64_t cnt;
    std::memcpy(&cnt, payload, 8);
    if (nbytes != 8 + 8 * cnt) return fail(FM_ERR_LAYOUT_OUT_OF_BOUNDS, "payload length != 8 + 8*count");
    if (int st = set_dev(t)) return st;
    uint64_t off;
    if (int st = fm::ctx_arena_alloc(t->ctx, nbytes, &off)) return st;
    // payload H2D on the table's stream: a poll that selects the record is ordered after it
    uint8_t* stg;
    cudaEvent_t ev;
    if (int st = fm::ctx_staging(t->ctx, nbytes, &stg, &ev)) return st;
    std::memcpy(stg, payload, nbytes);
    FM_CUDA(cudaMemcpyAsync(fm::ctx_arena(t->ctx) + off, stg, nbytes, cudaMemcpyHostToDevice, t->stream));
    FM_CUDA(cudaEventRecord(ev, t->stream));
    t->recs[static_cast<size_t>(slot)].status |= 1u << c;
    std::vector<void*> d;
    if (int st = upload(t, {{&slot, 8}, {&off, 8}}, &d)) return st;
    FM_CUDA(fm::launch_dt_set_cells(t->view, c, 1, static_cast<const int64_t*>(d[0]),
                                    static_cast<const uint64_t*>(d[1]), t->stream));
    fm::count_launch();
    return FM_OK;
    FM_GUARD_END
}

int fm_dtable_generate(fm_dtable* t, const fm_weights* w, const char* response_col, const char* logprob_col, int n,
                       const int64_t* slots, const int32_t* prompts, const int32_t* prompt_off, int max_tokens,
                       const uint64_t* seeds) {
    FM_GUARD_BEGIN
    if (!w || n < 0 || (n > 0 && (!slots || !prompt_off || !seeds)) || max_tokens <= 0)
        return fail(FM_ERR_INVALID_ARG, "bad generation request");
    int rc, lc = -1;
    if (int st = check_cells(t, response_col, n, slots, false, &rc)) return st;
    if (logprob_col)
        if (int st = check_cells(t, logprob_col, n, slots, false, &lc)) return st;
    if (n == 0) return FM_OK;
    if (int st = set_dev(t)) return st;
    fm::GenBuffers g;
    if (int st = fm::generate_device(t->ctx, w, prompts, prompt_off, n, max_tokens, seeds, &g)) return st;
    // responses (+ log-probs) reserved at max length per request in the arena
    const uint64_t stride = 2 * (8 + 8 * static_cast<uint64_t>(max_tokens));
    uint64_t base;
    if (int st = fm::ctx_arena_alloc(t->ctx, stride * n, &base)) return st;
    FM_CUDA(cudaEventRecord(t->ev_join, fm::ctx_stream(t->ctx)));
    FM_CUDA(cudaStreamWaitEvent(t->stream, t->ev_join, 0));
    for (int i = 0; i < n; ++i) {
        t->recs[static_cast<size_t>(slots[i])].status |= 1u << rc;
        if (lc >= 0) t->recs[static_cast<size_t>(slots[i])].status |= 1u << lc;
    }
    std::vector<void*> d;
    if (int st = upload(t, {{slots, n * 8u}}, &d)) return st;
    FM_CUDA(fm::launch_dt_encode(t->view, rc, lc, n, static_cast<const int64_t*>(d[0]), g.tok, g.logp, g.len,
                                 max_tokens, fm::ctx_arena(t->ctx), base, stride, t->stream));
    fm::count_launch();
    // the generation buffers are released once the encode has read them
    FM_CUDA(cudaEventRecord(t->ev_join, t->stream));
    FM_CUDA(cudaStreamWaitEvent(fm::ctx_stream(t->ctx), t->ev_join, 0));
    return fm::free_gen_buffers(t->ctx, &g);
    FM_GUARD_END
}

int fm_dtable_release_groups(fm_dtable* const* tables, int ntables, const char* response_col, const char* reward_col,
                             const char* adv_col, int ngroups, const int32_t* seg_off, const int32_t* score_tab,
                             const int64_t* score_slot, const int32_t* rec_off, const int32_t* rec_tab,
                             const int64_t* rec_slot, const int32_t* pattern, int npattern, double eps,
                             double* rewards_out, double* adv_out) {
    FM_GUARD_BEGIN
    if (!tables || ntables < 1 || ngroups < 0 || (ngroups > 0 && !seg_off))
        return fail(FM_ERR_INVALID_ARG, "bad release request");
    fm_dtable* t0 = tables[0];
    const int nsurv = ngroups > 0 ? seg_off[ngroups] : 0;
    const int nrec = nsurv > 0 ? rec_off[nsurv] : 0;
    if (nsurv > 0 && (!score_tab || !score_slot || !rec_off)) return fail(FM_ERR_INVALID_ARG, "bad survivor list");
    if (nrec > 0 && (!rec_tab || !rec_slot)) return fail(FM_ERR_INVALID_ARG, "bad record list");
    if (npattern < 0 || (npattern > 0 && !pattern)) return fail(FM_ERR_INVALID_ARG, "bad pattern");
    std::vector<fm::DTableView> views(static_cast<size_t>(ntables));
    std::vector<fm::DReleaseCols> cols(static_cast<size_t>(ntables));
    for (int k = 0; k < ntables; ++k) {
        fm_dtable* t = tables[k];
        if (!t || t->ctx != t0->ctx) return fail(FM_ERR_CONFIG_ERROR, "release tables must share one GPU context");
        const int rc = t->col(response_col), wc = t->col(reward_col), ac = t->col(adv_col);
        if (rc < 0 || wc < 0 || ac < 0) return fail(FM_ERR_UNKNOWN_COLUMN, "release needs response/reward/advantage");
        if (by_value(t->types[static_cast<size_t>(rc)]) || !by_value(t->types[static_cast<size_t>(wc)]) ||
            !by_value(t->types[static_cast<size_t>(ac)]))
            return fail(FM_ERR_CONFIG_ERROR, "cell storage class mismatch for release columns");
        views[static_cast<size_t>(k)] = t->view;
        cols[static_cast<size_t>(k)] = fm::DReleaseCols{rc, wc, ac};
    }
    for (int g = 0; g < ngroups; ++g)
        if (seg_off[g + 1] < seg_off[g]) return fail(FM_ERR_INVALID_ARG, "seg_off must be non-decreasing");
    for (int i = 0; i < nsurv; ++i) {
        if (score_tab[i] < 0 || score_tab[i] >= ntables || rec_off[i + 1] < rec_off[i])
            return fail(FM_ERR_INVALID_ARG, "bad survivor entry");
        fm_dtable* t = tables[score_tab[i]];
        if (!t->live_slot(score_slot[i])) return fail(FM_ERR_RECORD_NOT_FOUND, "scored slot " + std::to_string(score_slot[i]));
        if (!(t->recs[static_cast<size_t>(score_slot[i])].status & (1u << cols[static_cast<size_t>(score_tab[i])].response)))
            return fail(FM_ERR_CONFIG_ERROR, "scored record has no response yet");
    }
    std::vector<std::pair<int, int64_t>> seen;
    for (int r = 0; r < nrec; ++r) {  // the reference set_cell checks (experience_store.hpp:65-76)
        if (rec_tab[r] < 0 || rec_tab[r] >= ntables) return fail(FM_ERR_INVALID_ARG, "bad record table");
        fm_dtable* t = tables[rec_tab[r]];
        if (!t->live_slot(rec_slot[r])) return fail(FM_ERR_RECORD_NOT_FOUND, "slot " + std::to_string(rec_slot[r]));
        const fm::DReleaseCols& c = cols[static_cast<size_t>(rec_tab[r])];
        if (t->recs[static_cast<size_t>(rec_slot[r])].status & ((1u << c.reward) | (1u << c.advantage)))
            return fail(FM_ERR_CELL_ALREADY_SET, "reward/advantage");
        const std::pair<int, int64_t> key{rec_tab[r], rec_slot[r]};
        if (std::find(seen.begin(), seen.end(), key) != seen.end())
            return fail(FM_ERR_CELL_ALREADY_SET, "record listed twice");
        seen.push_back(key);
    }
    if (ngroups == 0) return FM_OK;
    if (int st = set_dev(t0)) return st;
    for (int r = 0; r < nrec; ++r) {
        const fm::DReleaseCols& c = cols[static_cast<size_t>(rec_tab[r])];
        tables[rec_tab[r]]->recs[static_cast<size_t>(rec_slot[r])].status |= (1u << c.reward) | (1u << c.advantage);
    }
    // order: every table's pending ops -> the release on t0's stream -> every table
    for (int k = 1; k < ntables; ++k) {
        FM_CUDA(cudaEventRecord(tables[k]->ev_join, tables[k]->stream));
        FM_CUDA(cudaStreamWaitEvent(t0->stream, tables[k]->ev_join, 0));
    }
    std::vector<double> zeros(static_cast<size_t>(std::max(nsurv, 1)), 0.0);
    std::vector<void*> d;
    if (int st = upload(t0,
                        {{views.data(), views.size() * sizeof(fm::DTableView)},
                         {cols.data(), cols.size() * sizeof(fm::DReleaseCols)},
                         {seg_off, (ngroups + 1) * 4u},
                         {score_tab, nsurv * 4u},
                         {score_slot, nsurv * 8u},
                         {rec_off, (nsurv + 1) * 4u},
                         {rec_tab, nrec * 4u},
                         {rec_slot, nrec * 8u},
                         {pattern, npattern * 4u},
                         {zeros.data(), zeros.size() * 8},
                         {zeros.data(), zeros.size() * 8}},
                        &d))
        return st;
    FM_CUDA(fm::launch_dt_release(static_cast<const fm::DTableView*>(d[0]), static_cast<const fm::DReleaseCols*>(d[1]),
                                  ngroups, static_cast<const int32_t*>(d[2]), static_cast<const int32_t*>(d[3]),
                                  static_cast<const int64_t*>(d[4]), static_cast<const int32_t*>(d[5]),
                                  static_cast<const int32_t*>(d[6]), static_cast<const int64_t*>(d[7]),
                                  static_cast<const int*>(d[8]), npattern, eps, fm::ctx_arena(t0->ctx),
                                  static_cast<double*>(d[9]), static_cast<double*>(d[10]), t0->stream));
    fm::count_launch();
    for (int k = 1; k < ntables; ++k) {
        FM_CUDA(cudaEventRecord(t0->ev_join, t0->stream));
        FM_CUDA(cudaStreamWaitEvent(tables[k]->stream, t0->ev_join, 0));
    }
    if (rewards_out || adv_out) {
        std::vector<double> tmp(static_cast<size_t>(2 * nsurv));
        FM_CUDA(cudaMemcpyAsync(tmp.data(), d[9], nsurv * 8u, cudaMemcpyDeviceToHost, t0->stream));
        FM_CUDA(cudaMemcpyAsync(tmp.data() + nsurv, d[10], nsurv * 8u, cudaMemcpyDeviceToHost, t0->stream));
        FM_CUDA(cudaStreamSynchronize(t0->stream));
        if (rewards_out) std::memcpy(rewards_out, tmp.data(), nsurv * 8u);
        if (adv_out) std::memcpy(adv_out, tmp.data() + nsurv, nsurv * 8u);
    }
    return FM_OK;
    FM_GUARD_END
}

int fm_dtable_poll(fm_dtable* t, int64_t version, int64_t mb, const char* prompt_col, const char* response_col,
                   const char* adv_col, int64_t* slots_out, int64_t* rows_out, int64_t* got, int64_t* poll_id) {
    FM_GUARD_BEGIN
    if (mb < 1) return fail(FM_ERR_CONFIG_ERROR, "micro_batch_size must be >= 1");  // experience_store.hpp:96
    if (mb > fm::kMaxPollMb) return fail(FM_ERR_CONFIG_ERROR, "device poll supports micro batches <= 1024");
    int pc = -1, rc = -1, ac = -1;
    if (prompt_col || response_col || adv_col) {
        pc = t->col(prompt_col);
        rc = t->col(response_col);
        ac = t->col(adv_col);
        if (pc < 0 || rc < 0 || ac < 0)
            return fail(FM_ERR_UNKNOWN_COLUMN, "trainer needs prompt/response/advantage columns");
        if (by_value(t->types[static_cast<size_t>(pc)]) || by_value(t->types[static_cast<size_t>(rc)]) ||
            !by_value(t->types[static_cast<size_t>(ac)]))
            return fail(FM_ERR_CONFIG_ERROR, "prompt/response must be list columns, advantage by value");
    }
    if (int st = set_dev(t)) return st;
    const int k = static_cast<int>(t->poll_seq % kRing);
    if (t->ring_used[k]) FM_CUDA(cudaStreamWaitEvent(t->stream, t->ring_consumed[k], 0));  // descriptors reused
    FM_CUDA(fm::launch_dt_poll(t->view, version, static_cast<int>(mb), pc, rc, ac, fm::ctx_arena(t->ctx), t->sc,
                               t->d_desc + static_cast<size_t>(k) * fm::kMaxPollMb, t->m_res, t->stream));
    fm::count_launch(3);
    FM_CUDA(cudaEventRecord(t->ring_ready[k], t->stream));
    FM_CUDA(cudaEventSynchronize(t->ring_ready[k]));
    *got = t->h_res->got;
    if (rows_out) *rows_out = t->h_res->rows;
    if (poll_id) *poll_id = -1;
    if (t->h_res->got == 0) return FM_OK;
    for (int64_t i = 0; i < mb; ++i) {
        const int64_t s = t->h_res->slots[i];
        if (!t->live_slot(s) || t->recs[static_cast<size_t>(s)].processing)
            return fail(FM_ERR_CONFIG_ERROR, "device poll selected a record the host index does not hold");
        t->recs[static_cast<size_t>(s)].processing = true;
        if (slots_out) slots_out[i] = s;
    }
    t->ring_id[k] = t->poll_seq;
    t->ring_mb[k] = static_cast<int>(mb);
    t->ring_rows[k] = pc >= 0 ? t->h_res->rows : -1;
    t->ring_used[k] = false;
    if (poll_id) *poll_id = t->poll_seq;
    t->poll_seq++;
    return FM_OK;
    FM_GUARD_END
}

int fm_train_polled(fm_agent* a, fm_dtable* t, int64_t poll_id, int64_t G, int64_t* ticket_out) {
    FM_GUARD_BEGIN
    if (!a || !t || poll_id < 0) return fail(FM_ERR_INVALID_ARG, "bad poll id");
    const int k = static_cast<int>(poll_id % kRing);
    if (t->ring_id[k] != poll_id) return fail(FM_ERR_INVALID_ARG, "poll descriptors already recycled (ring of 8)");
    if (t->ring_rows[k] < 0) return fail(FM_ERR_CONFIG_ERROR, "poll was made without trainer columns");
    if (int st = fm::agent_check_active(a)) return st;
    if (fm::agent_ctx(a) != t->ctx) return fail(FM_ERR_CONFIG_ERROR, "agent trains on another GPU than the table");
    if (int st = fm::train_device_desc(a, t->d_desc + static_cast<size_t>(k) * fm::kMaxPollMb, t->ring_mb[k],
                                       t->ring_rows[k], G, t->ring_ready[k], ticket_out))
        return st;
    FM_CUDA(cudaEventRecord(t->ring_consumed[k], fm::ctx_stream(t->ctx)));
    t->ring_used[k] = true;
    return FM_OK;
    FM_GUARD_END
}

int fm_dtable_complete(fm_dtable* t, const int64_t* slots, int n) {
    FM_GUARD_BEGIN
    if (n < 0 || (n > 0 && !slots)) return fail(FM_ERR_INVALID_ARG, "bad slot list");
    for (int i = 0; i < n; ++i) {  // experience_store.hpp:137-142: validate all first
        if (!t->live_slot(slots[i]) || !t->recs[static_cast<size_t>(slots[i])].processing)
            return fail(FM_ERR_NOT_PROCESSING, "slot " + std::to_string(slots[i]));
        for (int j = 0; j < i; ++j)
            if (slots[j] == slots[i]) return fail(FM_ERR_NOT_PROCESSING, "slot listed twice");
    }
    if (n == 0) return FM_OK;
    if (int st = set_dev(t)) return st;
    std::vector<void*> d;
    if (int st = upload(t, {{slots, n * 8u}}, &d)) return st;
    FM_CUDA(fm::launch_dt_erase(t->view, n, static_cast<const int64_t*>(d[0]), t->stream));
    fm::count_launch();
    for (int i = 0; i < n; ++i) erase_host(t, slots[i]);
    return FM_OK;
    FM_GUARD_END
}

static int purge_common(fm_dtable* t, int mode, int64_t current_version, const std::vector<uint64_t>& set,
                        uint64_t* out) {
    if (int st = set_dev(t)) return st;
    const uint64_t* dset = nullptr;
    std::vector<void*> d;
    if (mode == 1) {
        if (int st = upload(t, {{set.data(), set.size() * 8}}, &d)) return st;
        dset = static_cast<const uint64_t*>(d[0]);
    }
    FM_CUDA(fm::launch_dt_purge(t->view, mode, current_version, dset, static_cast<int>(set.size()), t->sc.count,
                                t->d_list, t->stream));
    fm::count_launch();
    FM_CUDA(cudaMemcpyAsync(t->h_list, t->sc.count, 4, cudaMemcpyDeviceToHost, t->stream));
    FM_CUDA(cudaStreamSynchronize(t->stream));
    const int cnt = t->h_list[0];
    if (cnt) {
        FM_CUDA(cudaMemcpyAsync(t->h_list, t->d_list, cnt * 4u, cudaMemcpyDeviceToHost, t->stream));
        FM_CUDA(cudaStreamSynchronize(t->stream));
    }
    std::vector<int64_t> gone(t->h_list, t->h_list + cnt);
    for (int64_t s : gone) {
        if (!t->live_slot(s) || t->recs[static_cast<size_t>(s)].processing)
            return fail(FM_ERR_CONFIG_ERROR, "device purge removed a record the host index disagrees on");
        erase_host(t, s);
    }
    if (out) *out = static_cast<uint64_t>(cnt);
    return FM_OK;
}

int fm_dtable_purge_stale(fm_dtable* t, int64_t current_version, uint64_t* out) {
    FM_GUARD_BEGIN
    return purge_common(t, 0, current_version, {}, out);
    FM_GUARD_END
}

int fm_dtable_purge_inputs(fm_dtable* t, const char* const* ids, int n, uint64_t* out) {
    FM_GUARD_BEGIN
    if (n < 0 || (n > 0 && !ids)) return fail(FM_ERR_INVALID_ARG, "bad input list");
    std::vector<uint64_t> set;
    for (int i = 0; i < n; ++i) {
        auto it = t->labels.find(ids[i] ? ids[i] : "");
        if (it != t->labels.end()) set.push_back(it->second.label);
    }
    std::sort(set.begin(), set.end());
    set.erase(std::unique(set.begin(), set.end()), set.end());
    if (set.empty()) {
        if (out) *out = 0;
        return FM_OK;
    }
    return purge_common(t, 1, 0, set, out);
    FM_GUARD_END
}

int fm_dtable_drop_record(fm_dtable* t, const char* id, int turns, int traj, int64_t version, int* dropped) {
    FM_GUARD_BEGIN
    *dropped = 0;
    auto it = t->index.find(RecordKey{id ? id : "", turns, traj, version});
    if (it == t->index.end() || t->recs[static_cast<size_t>(it->second)].processing) return FM_OK;
    const int64_t s = it->second;
    if (int st = set_dev(t)) return st;
    std::vector<void*> d;
    if (int st = upload(t, {{&s, 8}}, &d)) return st;
    FM_CUDA(fm::launch_dt_erase(t->view, 1, static_cast<const int64_t*>(d[0]), t->stream));
    fm::count_launch();
    erase_host(t, s);
    *dropped = 1;
    return FM_OK;
    FM_GUARD_END
}

int fm_dtable_ready_count(fm_dtable* t, int64_t version, uint64_t* out) {
    FM_GUARD_BEGIN
    if (int st = set_dev(t)) return st;
    FM_CUDA(fm::launch_dt_ready_count(t->view, version, t->d_cnt, t->stream));
    fm::count_launch();
    FM_CUDA(cudaMemcpyAsync(t->h_cnt, t->d_cnt, 8, cudaMemcpyDeviceToHost, t->stream));
    FM_CUDA(cudaStreamSynchronize(t->stream));
    *out = static_cast<uint64_t>(*t->h_cnt);
    return FM_OK;
    FM_GUARD_END
}

int fm_dtable_record_count(fm_dtable* t, uint64_t* out) {
    *out = static_cast<uint64_t>(t->live);
    return FM_OK;
}

int fm_dtable_record(fm_dtable* t, int64_t slot, char* id_out, size_t cap, int* turns, int* traj, int64_t* version,
                     int* processing, uint32_t* status) {
    if (!t->live_slot(slot)) return fail(FM_ERR_RECORD_NOT_FOUND, "slot " + std::to_string(slot));
    const HostRec& r = t->recs[static_cast<size_t>(slot)];
    if (id_out && cap) {
        std::strncpy(id_out, r.id.c_str(), cap - 1);
        id_out[cap - 1] = 0;
    }
    if (turns) *turns = r.turns;
    if (traj) *traj = r.traj;
    if (version) *version = r.version;
    if (processing) *processing = r.processing ? 1 : 0;
    if (status) *status = r.status;
    return FM_OK;
}

int fm_dtable_records(fm_dtable* t, int n, const int64_t* slots, char* ids_out, size_t id_cap, int* turns,
                      int* trajs, int64_t* versions) {
    for (int i = 0; i < n; ++i) {
        if (!t->live_slot(slots[i])) return fail(FM_ERR_RECORD_NOT_FOUND, "slot " + std::to_string(slots[i]));
        const HostRec& r = t->recs[static_cast<size_t>(slots[i])];
        if (ids_out && id_cap) {
            char* o = ids_out + static_cast<size_t>(i) * id_cap;
            std::strncpy(o, r.id.c_str(), id_cap - 1);
            o[id_cap - 1] = 0;
        }
        if (turns) turns[i] = r.turns;
        if (trajs) trajs[i] = r.traj;
        if (versions) versions[i] = r.version;
    }
    return FM_OK;
}

int fm_dtable_read_cells(fm_dtable* t, const char* column, int n, const int64_t* slots, uint64_t* out) {
    FM_GUARD_BEGIN
    const int c = t->col(column);
    if (c < 0) return fail(FM_ERR_UNKNOWN_COLUMN, column ? column : "(null)");
    for (int i = 0; i < n; ++i)
        if (slots[i] < 0 || slots[i] >= t->cap) return fail(FM_ERR_RECORD_NOT_FOUND, "slot " + std::to_string(slots[i]));
    if (int st = set_dev(t)) return st;
    std::vector<uint64_t> colv(static_cast<size_t>(t->cap));
    FM_CUDA(cudaMemcpyAsync(colv.data(), t->view.cells + static_cast<size_t>(c) * t->cap, colv.size() * 8,
                            cudaMemcpyDeviceToHost, t->stream));
    FM_CUDA(cudaStreamSynchronize(t->stream));
    for (int i = 0; i < n; ++i) out[i] = colv[static_cast<size_t>(slots[i])];
    return FM_OK;
    FM_GUARD_END
}

}  // extern "C"

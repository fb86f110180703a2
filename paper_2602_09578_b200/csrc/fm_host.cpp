// fm_host.cpp — host-side C++ of the drop-in: error plumbing, the bit-exact
// seeded initialisation (rng.hpp / policy.hpp:29-35), the token codec
// (codec.hpp:15-22) and the experience-store control plane
// (experience_store.hpp:19-276).  The store keeps the reference's canonical
// std::map ordering and status/processing semantics on the host (it is O(16)
// bookkeeping per poll); the record payloads live in the GPU token arena and
// are consumed by the device gather (k_path.cu).
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "fm_internal.h"

namespace fm {

namespace {
thread_local std::string t_err;
}

std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
    t_err = msg;
    return code;
}
void clear_error() { t_err.clear(); }

// ---- rng.hpp:14-64, restated for the product's host side ------------------
namespace {
inline uint64_t splitmix64(uint64_t& state) {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline uint64_t mix_u64(uint64_t seed, uint64_t value) {
    uint64_t s = seed ^ (value + 0x9e3779b97f4a7c15ULL + (seed << 6) + (seed >> 2));
    return splitmix64(s);
}
inline uint64_t mix_str(uint64_t seed, const char* text) {
    uint64_t h = seed ^ 0xcbf29ce484222325ULL;
    for (const unsigned char* c = reinterpret_cast<const unsigned char*>(text); *c; ++c) {
        h ^= *c;
        h *= 0x100000001b3ULL;
        h = mix_u64(h, *c);
    }
    return h;
}
inline double unit_from(uint64_t x) {
    const uint64_t bits = x >> 11;
    double u = static_cast<double>(bits) * 0x1.0p-53;
    if (u <= 0.0) u = 0x1.0p-53;
    return u;
}
}  // namespace

}  // namespace fm

using namespace fm;

extern "C" {

const char* fm_last_error(void) { return t_err.c_str(); }

const char* fm_status_name(int s) {
    static const char* names[] = {"OK",
                                  "SchedulingInPast",
                                  "DeviceOom",
                                  "HostOom",
                                  "EmptyPool",
                                  "DuplicateKey",
                                  "KeyNotFound",
                                  "GetTimeout",
                                  "LayoutOutOfBounds",
                                  "EmptyList",
                                  "TableExists",
                                  "ReservedColumnName",
                                  "DuplicateSample",
                                  "UnknownColumn",
                                  "RecordNotFound",
                                  "CellAlreadySet",
                                  "UnknownTable",
                                  "NotProcessing",
                                  "BadSampleId",
                                  "UnknownWorkflow",
                                  "NoInstance",
                                  "InsufficientResources",
                                  "BusyGroup",
                                  "VersionMismatch",
                                  "InactiveGroup",
                                  "IncompleteBatch",
                                  "ConfigError",
                                  "StallDetected",
                                  "SyncTimeout"};
    if (s >= 0 && s <= 28) return names[s];
    switch (s) {
        case FM_ERR_CUDA: return "CudaError";
        case FM_ERR_NCCL: return "NcclError";
        case FM_ERR_NO_DEVICE: return "NoDevice";
        case FM_ERR_INVALID_ARG: return "InvalidArgument";
    }
    return "Unknown";
}

int fm_abi_version(void) { return 1; }

uint64_t fm_launch_count(void) { return g_launches.load(); }

uint64_t fm_agent_seed(uint64_t seed, const char* agent) { return mix_str(mix_u64(seed, 0x1217), agent); }

// PolicyModel::seeded: w_i = 0.5 * next_normal(), one Box-Muller pair per
// element from one sequential splitmix64 stream (policy.hpp:29-35,
// rng.hpp:55-59).  splitmix64 is a counter generator (state += golden per
// draw), so element i consumes draws 2i+1 and 2i+2 and the stream splits
// across threads without changing a single bit.
int fm_seeded_weights(uint64_t V, uint64_t D, uint64_t seed, double* out, int threads) {
    FM_GUARD_BEGIN
    const uint64_t n = V * D;
    if (!out && n) return fail(FM_ERR_INVALID_ARG, "null output");
    unsigned nt = threads > 0 ? static_cast<unsigned>(threads) : std::thread::hardware_concurrency();
    if (nt == 0) nt = 1;
    if (n < (1u << 16)) nt = 1;
    auto work = [&](uint64_t b, uint64_t e) {
        uint64_t st = seed + 2 * b * 0x9e3779b97f4a7c15ULL;
        for (uint64_t i = b; i < e; ++i) {
            const double u1 = unit_from(splitmix64(st));
            const double u2 = unit_from(splitmix64(st));
            out[i] = 0.5 * (std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2));
        }
    };
    std::vector<std::thread> pool;
    const uint64_t chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const uint64_t b = t * chunk, e = std::min<uint64_t>(n, b + chunk);
        if (b >= e) break;
        if (nt == 1) work(b, e);
        else pool.emplace_back(work, b, e);
    }
    for (auto& th : pool) th.join();
    return FM_OK;
    FM_GUARD_END
}

uint64_t fm_encode_tokens(const int32_t* tokens, uint64_t n, uint8_t* out) {
    std::memcpy(out, &n, 8);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t t = static_cast<uint64_t>(static_cast<int64_t>(tokens[i]));
        std::memcpy(out + 8 + 8 * i, &t, 8);
    }
    return 8 + 8 * n;
}

}  // extern "C"

// ===========================================================================
// experience store control plane
// ===========================================================================
namespace {

enum ColType { kInt = 0, kFloat = 1, kBool = 2, kString = 3, kList = 4, kTensor = 5 };

struct Cell {
    bool set = false;
    double f = 0.0;
    uint64_t arena_off = 0;  // ref cells: token-arena offset (the object "key")
};

struct Record {
    int64_t version = 0;
    std::string input_id;
    int turns = 0, traj = 0;
    bool processing = false;
    int64_t handle = 0;
    std::vector<Cell> data;
    bool ready() const {
        for (const Cell& c : data)
            if (!c.set) return false;
        return true;
    }
};

using RecordKey = std::tuple<std::string, int, int, int64_t>;  // experience_store.hpp:242

struct Table {
    std::vector<std::string> names;
    std::vector<int> types;
    std::map<RecordKey, Record> records;  // canonical iteration order
    std::unordered_map<int64_t, RecordKey> by_handle;
    int col(const std::string& n) const {
        for (size_t i = 0; i < names.size(); ++i)
            if (names[i] == n) return static_cast<int>(i);
        return -1;
    }
};

}  // namespace

struct fm_store {
    std::map<std::string, Table> tables;
    int64_t next_handle = 1;
    Table* table(const char* agent) {
        auto it = tables.find(agent ? agent : "");
        return it == tables.end() ? nullptr : &it->second;
    }
};

namespace {
std::string render(const std::string& id, int turns, int traj) {
    return id + "_" + std::to_string(turns) + "_" + std::to_string(traj);
}
}  // namespace

extern "C" {

int fm_store_create(fm_store** out) {
    FM_GUARD_BEGIN
    *out = new fm_store();
    return FM_OK;
    FM_GUARD_END
}

int fm_store_destroy(fm_store* s) {
    delete s;
    return FM_OK;
}

int fm_store_create_table(fm_store* s, const char* agent, const char* const* names, const int* types,
                          int ncols) {
    FM_GUARD_BEGIN
    if (s->tables.count(agent)) return fail(FM_ERR_TABLE_EXISTS, agent);
    Table t;
    for (int i = 0; i < ncols; ++i) {
        const std::string n = names[i];
        if (n == "policy_version" || n == "sample_id" || n == "processing")
            return fail(FM_ERR_RESERVED_COLUMN_NAME, n);
        for (int j = 0; j < i; ++j)
            if (n == names[j]) return fail(FM_ERR_CONFIG_ERROR, "duplicate column " + n);
        t.names.push_back(n);
        t.types.push_back(types[i]);
    }
    s->tables.emplace(agent, std::move(t));
    return FM_OK;
    FM_GUARD_END
}

int fm_store_insert(fm_store* s, const char* agent, int64_t version, const char* input_id, int turns,
                    int traj) {
    FM_GUARD_BEGIN
    Table* t = s->table(agent);
    if (!t) return fail(FM_ERR_UNKNOWN_TABLE, agent);
    const std::string id = input_id;
    if (id.empty() || id.find('_') != std::string::npos)
        return fail(FM_ERR_BAD_SAMPLE_ID, "input_id may not be empty or contain '_': " + id);
    const RecordKey key{id, turns, traj, version};
    if (t->records.count(key))
        return fail(FM_ERR_DUPLICATE_SAMPLE, render(id, turns, traj) + " v" + std::to_string(version));
    Record r;
    r.version = version;
    r.input_id = id;
    r.turns = turns;
    r.traj = traj;
    r.handle = s->next_handle++;
    r.data.assign(t->names.size(), Cell{});
    t->by_handle.emplace(r.handle, key);
    t->records.emplace(key, std::move(r));
    return FM_OK;
    FM_GUARD_END
}

static int set_cell_common(fm_store* s, const char* agent, const char* input_id, int turns, int traj,
                           int64_t version, const char* column, bool by_value, Cell** cell_out) {
    Table* t = s->table(agent);
    if (!t) return fail(FM_ERR_UNKNOWN_TABLE, agent);
    const int col = t->col(column);
    if (col < 0) return fail(FM_ERR_UNKNOWN_COLUMN, column);
    auto it = t->records.find(RecordKey{input_id, turns, traj, version});
    if (it == t->records.end()) return fail(FM_ERR_RECORD_NOT_FOUND, render(input_id, turns, traj));
    Cell& c = it->second.data[static_cast<size_t>(col)];
    if (c.set) return fail(FM_ERR_CELL_ALREADY_SET, column);
    const int ty = t->types[static_cast<size_t>(col)];
    const bool col_by_value = ty == kInt || ty == kFloat || ty == kBool;  // sample.hpp:71-73
    if (col_by_value != by_value)
        return fail(FM_ERR_CONFIG_ERROR, std::string("cell storage class mismatch for column ") + column);
    *cell_out = &c;
    return FM_OK;
}

int fm_store_set_float(fm_store* s, const char* agent, const char* input_id, int turns, int traj,
                       int64_t version, const char* column, double value) {
    FM_GUARD_BEGIN
    Cell* c = nullptr;
    const int st = set_cell_common(s, agent, input_id, turns, traj, version, column, true, &c);
    if (st) return st;
    c->f = value;
    c->set = true;
    return FM_OK;
    FM_GUARD_END
}

int fm_store_set_payload(fm_store* s, fm_ctx* ctx, const char* agent, const char* input_id, int turns,
                         int traj, int64_t version, const char* column, const uint8_t* payload,
                         uint64_t nbytes) {
    FM_GUARD_BEGIN
    Cell* c = nullptr;
    const int st = set_cell_common(s, agent, input_id, turns, traj, version, column, false, &c);
    if (st) return st;
    uint64_t off = 0;
    const int pst = fm_arena_put(ctx, payload, nbytes, &off);
    if (pst) return pst;
    c->arena_off = off;
    c->set = true;
    return FM_OK;
    FM_GUARD_END
}

int fm_store_ready_count(fm_store* s, const char* agent, int64_t version, uint64_t* out) {
    Table* t = s->table(agent);
    if (!t) return fail(FM_ERR_UNKNOWN_TABLE, agent);
    uint64_t n = 0;
    for (const auto& kv : t->records)
        if (!kv.second.processing && kv.second.version == version && kv.second.ready()) ++n;
    *out = n;
    return FM_OK;
}

int fm_store_record_count(fm_store* s, const char* agent, uint64_t* out) {
    Table* t = s->table(agent);
    if (!t) return fail(FM_ERR_UNKNOWN_TABLE, agent);
    *out = t->records.size();
    return FM_OK;
}

int fm_store_poll(fm_store* s, const char* agent, int64_t version, int64_t mb, const char* prompt_col,
                  const char* response_col, const char* adv_col, fm_sample* samples_out,
                  int64_t* handles_out, int64_t* got) {
    FM_GUARD_BEGIN
    Table* t = s->table(agent);
    if (!t) return fail(FM_ERR_UNKNOWN_TABLE, agent);
    if (mb < 1) return fail(FM_ERR_CONFIG_ERROR, "micro_batch_size must be >= 1");
    const int pc = prompt_col ? t->col(prompt_col) : -1;
    const int rc = response_col ? t->col(response_col) : -1;
    const int ac = adv_col ? t->col(adv_col) : -1;
    if (samples_out && (pc < 0 || rc < 0 || ac < 0))
        return fail(FM_ERR_UNKNOWN_COLUMN, "trainer needs prompt/response/advantage columns");
    std::vector<Record*> chosen;
    for (auto& kv : t->records) {  // experience_store.hpp:99-103
        Record& r = kv.second;
        if (r.processing || r.version != version || !r.ready()) continue;
        chosen.push_back(&r);
        if (static_cast<int64_t>(chosen.size()) == mb) break;
    }
    if (static_cast<int64_t>(chosen.size()) < mb) {
        *got = 0;
        return FM_OK;
    }
    for (size_t i = 0; i < chosen.size(); ++i) {
        Record& r = *chosen[i];
        r.processing = true;
        if (handles_out) handles_out[i] = r.handle;
        if (samples_out) {
            samples_out[i].prompt_off = r.data[static_cast<size_t>(pc)].arena_off;
            samples_out[i].response_off = r.data[static_cast<size_t>(rc)].arena_off;
            samples_out[i].advantage = r.data[static_cast<size_t>(ac)].f;
        }
    }
    *got = mb;
    return FM_OK;
    FM_GUARD_END
}

int fm_store_record_id(fm_store* s, const char* agent, int64_t handle, char* id_out, size_t cap, int* turns,
                       int* traj, int64_t* version) {
    Table* t = s->table(agent);
    if (!t) return fail(FM_ERR_UNKNOWN_TABLE, agent);
    auto h = t->by_handle.find(handle);
    if (h == t->by_handle.end()) return fail(FM_ERR_RECORD_NOT_FOUND, "handle " + std::to_string(handle));
    const Record& r = t->records.at(h->second);
    if (id_out && cap) {
        std::strncpy(id_out, r.input_id.c_str(), cap - 1);
        id_out[cap - 1] = 0;
    }
    if (turns) *turns = r.turns;
    if (traj) *traj = r.traj;
    if (version) *version = r.version;
    return FM_OK;
}

int fm_store_complete(fm_store* s, const char* agent, const int64_t* handles, int64_t n) {
    FM_GUARD_BEGIN
    Table* t = s->table(agent);
    if (!t) return fail(FM_ERR_UNKNOWN_TABLE, agent);
    for (int64_t i = 0; i < n; ++i) {  // validate all first (experience_store.hpp:137-142)
        auto h = t->by_handle.find(handles[i]);
        if (h == t->by_handle.end()) return fail(FM_ERR_NOT_PROCESSING, "handle " + std::to_string(handles[i]));
        if (!t->records.at(h->second).processing)
            return fail(FM_ERR_NOT_PROCESSING, std::get<0>(h->second));
    }
    for (int64_t i = 0; i < n; ++i) {
        auto h = t->by_handle.find(handles[i]);
        t->records.erase(h->second);  // refs: arena space is reclaimed by fm_arena_reset
        t->by_handle.erase(h);
    }
    return FM_OK;
    FM_GUARD_END
}

int fm_store_purge_stale(fm_store* s, const char* agent, int64_t current_version, uint64_t* out) {
    FM_GUARD_BEGIN
    Table* t = s->table(agent);
    if (!t) return fail(FM_ERR_UNKNOWN_TABLE, agent);
    uint64_t n = 0;
    for (auto it = t->records.begin(); it != t->records.end();) {
        if (!it->second.processing && it->second.version < current_version) {
            t->by_handle.erase(it->second.handle);
            it = t->records.erase(it);
            ++n;
        } else {
            ++it;
        }
    }
    if (out) *out = n;
    return FM_OK;
    FM_GUARD_END
}

}  // extern "C"

// dropin/marlsim/training.hpp — source-level drop-in of the B200 trainer into
// the reference (FlexMARL artifact, proj/include/marlsim).
//
// Put this directory BEFORE the reference's include directory:
//     g++ -std=c++20 -I<repo>/dropin -I<repo>/include -I<reference>/proj/include ...
//         -L<repo>/paper_2602_09578_b200/_native -lflexmarl_b200
// Every `#include "marlsim/training.hpp"` of the reference (orchestrator.hpp:20,
// rollout.hpp:25) then lands here.  This header includes the reference's own
// training.hpp (#include_next) with its class renamed RefTrainingEngine, so
// everything else it defines — AdamParams, OptimizerState, PolicyState,
// GradReport, TrainingConfig, GradKey, adam_step, group_advantages,
// rule_reward — is the reference's, unchanged; and it defines
// marlsim::TrainingEngine with the reference's exact public interface
// (training.hpp:192-540) over the C ABI (include/flexmarl/cabi.h): the
// trainer state lives on a B200 and train_micro_batch / apply_global_update
// run the sm_100a kernels.
//
// Kept from the reference, so a run's event order is unchanged: every error
// check and its ErrorCode (InactiveGroup, BusyGroup, VersionMismatch,
// UnknownColumn, DuplicateSample, IncompleteBatch, ConfigError,
// InsufficientResources, KeyNotFound), STRICT_PACK placement (pick_devices),
// the simulated device-memory reservations, the virtual-time busy charge and
// completion scheduling, the object-store traffic (payload gets, checkpoint
// set/get/del, weight publication) and the event-log records.
// Different by design: the gradient of a global step is one accumulator on
// the GPU (the reference caches one V x D matrix per sample; the update sums
// them in canonical order, training.hpp:93-98, 444-446).  The GradKey set is
// kept here (host) for the DuplicateSample guard, and a checkpoint of a
// mid-step agent holds one cache entry per GradKey (the step's summed gradient
// under the first, zeros under the rest): the reference's byte length and
// canonical reduction, read by either side's PolicyState::deserialize.
//
// Environment: FLEXMARL_DEVICE (CUDA device, default 0), FLEXMARL_PRECISION
// ("bf16" tensor-core path, default; "f64" the exact parity path).
#pragma once

#define TrainingEngine RefTrainingEngine
#include_next <marlsim/training.hpp>
#undef TrainingEngine

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>
#include <stdexcept>

#include "flexmarl/cabi.h"

namespace marlsim {

namespace flexmarl_detail {
// fm_status 1..28 are marlsim::ErrorCode + 1 (include/flexmarl/cabi.h)
[[noreturn]] inline void raise_status(int st) {
    const char* msg = fm_last_error();
    if (st >= 1 && st <= 28) raise(static_cast<ErrorCode>(st - 1), msg ? msg : "");
    throw std::runtime_error(std::string("flexmarl: ") + fm_status_name(st) + ": " + (msg ? msg : ""));
}
inline void check(int st) {
    if (st != 0) raise_status(st);
}
}  // namespace flexmarl_detail

class TrainingEngine {
public:
    TrainingEngine(EventLoop& loop, Cluster& cluster, ObjectStore& objects, EventLog& log, ResourcePool pool,
                   TrainingConfig cfg)
        : loop_(loop), cluster_(cluster), objects_(objects), log_(log), pool_(std::move(pool)),
          cfg_(std::move(cfg)) {
        const char* dev = std::getenv("FLEXMARL_DEVICE");
        device_ = dev ? std::atoi(dev) : 0;
        const char* prec = std::getenv("FLEXMARL_PRECISION");
        precision_ = (prec && std::strcmp(prec, "f64") == 0) ? FM_PRECISION_PARITY_F64 : FM_PRECISION_BF16_TC;
    }
    TrainingEngine(const TrainingEngine&) = delete;
    TrainingEngine& operator=(const TrainingEngine&) = delete;
    ~TrainingEngine() {
        for (auto& [name, g] : groups_)
            if (g.h) fm_agent_destroy(g.h);
        if (ctx_) fm_ctx_destroy(ctx_);
    }

    void add_agent(const std::string& agent_id, std::size_t vocab, std::size_t feat) {
        Group g;
        g.vocab = vocab;
        g.feat = feat;
        groups_.emplace(agent_id, std::move(g));
    }

    const ResourcePool& pool() const { return pool_; }
    const TrainingConfig& config() const { return cfg_; }
    TrainingConfig& config() { return cfg_; }

    bool is_active(const std::string& agent) const { return group(agent).state == GroupState::Active; }
    bool in_flight(const std::string& agent) const { return group(agent).in_flight; }

    const std::vector<DeviceId>& bound_devices(const std::string& agent) const { return group(agent).devices; }
    NodeId last_node(const std::string& agent) const { return group(agent).last_node; }

    // training.hpp:219-223.  The live state is on the GPU: this materialises a host
    // copy (weights, moments, counters; the pending gradient is not a per-sample
    // cache here) — writes to it do not reach the device.
    PolicyState& state(const std::string& agent) {
        Group& g = group(agent);
        if (g.state != GroupState::Active) raise(ErrorCode::InactiveGroup, agent);
        g.mirror = read_state(agent, g);
        return g.mirror;
    }

    // training.hpp:225-232
    PolicyState peek_state(const std::string& agent) const {
        const Group& g = group(agent);
        if (g.state == GroupState::Active) return read_state(agent, g);
        if (g.latest_checkpoint.empty()) raise(ErrorCode::InactiveGroup, agent + " never ran");
        const HeterogeneousObject* blob = objects_.peek(g.latest_checkpoint);
        if (!blob) raise(ErrorCode::KeyNotFound, g.latest_checkpoint);
        return PolicyState::deserialize(agent, blob->payload);
    }

    std::uint64_t param_count(const std::string& agent) const {
        const Group& g = group(agent);
        return static_cast<std::uint64_t>(g.vocab) * g.feat;
    }
    std::uint64_t training_footprint_bytes(const std::string& agent) const { return param_count(agent) * 4 * 3; }

    // training.hpp:245-248 (host, bit-identical: the reference's own PolicyModel::seeded)
    PolicyModel initial_model(const std::string& agent) const {
        const Group& g = group(agent);
        return PolicyModel::seeded(g.vocab, g.feat, mix_str(mix_u64(cfg_.seed, 0x1217), agent));
    }

    bool can_activate(const std::string& agent) const { return !pick_devices(agent).empty(); }

    // training.hpp:259-317: the gang binding and its simulated reservations as the
    // reference; the state goes to a B200 (fresh seeded weights, or the checkpoint).
    void activate(const std::string& agent, std::function<void()> on_done) {
        if (!on_done) on_done = []() {};
        Group& g = group(agent);
        if (g.state == GroupState::Active) raise(ErrorCode::ConfigError, agent + " already active");
        std::vector<DeviceId> devs = pick_devices(agent);
        if (devs.empty()) {
            raise(ErrorCode::InsufficientResources, "no node has " + std::to_string(cfg_.devices_per_group) +
                                                        " free training devices for " + agent);
        }
        const std::uint64_t per_dev = (training_footprint_bytes(agent) + devs.size() - 1) / devs.size();
        std::vector<Reservation> held;
        try {
            for (DeviceId d : devs) held.push_back(cluster_.reserve_device_mem(d, per_dev));
        } catch (const Error&) {
            for (const Reservation& r : held) cluster_.release_device_mem(r);
            throw;
        }
        fm_agent* h = nullptr;
        flexmarl_detail::check(fm_agent_create(ctx(), agent.c_str(), g.vocab, g.feat, precision_, &h));
        g.devices = devs;
        g.reservations = std::move(held);
        g.state = GroupState::Active;
        g.h = h;
        const NodeId node = cluster_.node_of_device(devs.front());

        if (g.latest_checkpoint.empty()) {
            const PolicyModel m = initial_model(agent);
            flexmarl_detail::check(fm_agent_set_weights(h, m.weights().a.data()));
            g.last_node = node;
            log_.append(loop_.now(), "activate",
                        Json{{"agent", agent},
                             {"node", node},
                             {"devices", devs},
                             {"control_s", cfg_.control_plane_s},
                             {"restore_s", 0.0},
                             {"restore_path", Json::array()},
                             {"fresh", true}});
            loop_.schedule_after(cfg_.control_plane_s, std::move(on_done));
            return;
        }

        GetResult r = objects_.get(g.latest_checkpoint, Placement::device(devs.front()));
        flexmarl_detail::check(
            fm_agent_deserialize(h, cfg_.global_batch, r.object.payload.data(), r.object.payload.size()));
        g.last_node = node;
        std::vector<std::string> path;
        for (HopKind hop : r.record.path) path.emplace_back(hop_name(hop));
        log_.append(loop_.now(), "activate",
                    Json{{"agent", agent},
                         {"node", node},
                         {"devices", devs},
                         {"control_s", cfg_.control_plane_s},
                         {"restore_s", r.record.sim_duration},
                         {"restore_path", path},
                         {"fresh", false}});
        objects_.del(g.latest_checkpoint);
        g.latest_checkpoint.clear();
        loop_.schedule(r.done + cfg_.control_plane_s, std::move(on_done));
    }

    // training.hpp:321-350: the checkpoint is the PolicyState wire format written by
    // the GPU (fm_agent_serialize), set on the node's host tier as the reference does.
    void suspend(const std::string& agent, std::function<void()> on_done) {
        if (!on_done) on_done = []() {};
        Group& g = group(agent);
        if (g.state != GroupState::Active) raise(ErrorCode::InactiveGroup, agent);
        if (g.in_flight) raise(ErrorCode::BusyGroup, agent + " has a micro batch in flight");

        const NodeId node = cluster_.node_of_device(g.devices.front());
        const std::string key = "optstate:" + agent + ":v" + std::to_string(fm_agent_version(g.h)) + ":c" +
                                std::to_string(g.checkpoint_counter++);
        std::uint64_t len = 0;
        flexmarl_detail::check(fm_agent_serialize(g.h, cfg_.global_batch, nullptr, 0, &len));
        std::vector<std::uint8_t> bytes(len);
        flexmarl_detail::check(fm_agent_serialize(g.h, cfg_.global_batch, bytes.data(), len, &len));
        if (!g.keys.empty()) bytes = per_sample_cache(g, bytes);
        len = bytes.size();
        HeterogeneousObject obj;
        obj.payload = std::move(bytes);
        obj.dtype = DType::Bytes;
        ObjectRef ref = objects_.set(key, std::move(obj), Placement::host(node));
        g.latest_checkpoint = key;
        g.last_node = node;
        for (const Reservation& r : g.reservations) cluster_.release_device_mem(r);
        g.reservations.clear();
        g.devices.clear();
        fm_agent_destroy(g.h);
        g.h = nullptr;
        g.state = GroupState::Destroyed;
        log_.append(loop_.now(), "suspend",
                    Json{{"agent", agent},
                         {"node", node},
                         {"control_s", cfg_.control_plane_s},
                         {"offload_s", ref.ready_at - loop_.now()},
                         {"bytes", len}});
        loop_.schedule_after(cfg_.control_plane_s, std::move(on_done));
    }

    // training.hpp:355-430.  The validation, payload gets (the transfer clock), busy
    // charge and completion schedule are the reference's; the gradient runs on the
    // GPU (fm_train_micro_batch_host: payload bytes staged H2D inside the call), and
    // the completion delivers its grad norm through the event loop as the reference.
    void train_micro_batch(const std::string& agent, const MicroBatch& batch, const TableSchema& schema,
                           std::function<void(GradReport)> on_done) {
        Group& g = group(agent);
        if (g.state != GroupState::Active) raise(ErrorCode::InactiveGroup, agent);
        if (g.in_flight) raise(ErrorCode::BusyGroup, agent);
        const std::int64_t version = fm_agent_version(g.h);
        const std::int64_t staleness = version - batch.policy_version;
        if (staleness < 0 || staleness > cfg_.allowed_staleness) {
            raise(ErrorCode::VersionMismatch, agent + ": batch v" + std::to_string(batch.policy_version) +
                                                  " vs state v" + std::to_string(version));
        }
        const int prompt_col = schema.column_index("prompt");
        const int response_col = schema.column_index("response");
        const int adv_col = schema.column_index("advantage");
        if (prompt_col < 0 || response_col < 0 || adv_col < 0) {
            raise(ErrorCode::UnknownColumn, "trainer needs prompt/response/advantage columns");
        }
        // DuplicateSample (training.hpp:396-401), checked for the whole batch before
        // anything is enqueued
        std::vector<GradKey> keys;
        for (const SampleRecord& rec : batch.samples) {
            GradKey k = grad_key(rec.sample_id, rec.policy_version);
            if (g.keys.count(k) || std::find(keys.begin(), keys.end(), k) != keys.end())
                raise(ErrorCode::DuplicateSample, "gradient already cached for " + rec.sample_id.render());
            keys.push_back(std::move(k));
        }

        SimTime data_ready = loop_.now();
        std::vector<GetResult> payloads;
        payloads.reserve(2 * batch.samples.size());
        std::vector<fm_host_sample> hs;
        std::vector<fm_sample_key> fk;
        for (const SampleRecord& rec : batch.samples) {
            payloads.push_back(objects_.get(rec.data[static_cast<std::size_t>(prompt_col)].ref_key(),
                                            Placement::device(g.devices.front())));
            payloads.push_back(objects_.get(rec.data[static_cast<std::size_t>(response_col)].ref_key(),
                                            Placement::device(g.devices.front())));
            data_ready = std::max({data_ready, payloads[payloads.size() - 2].done, payloads.back().done});
        }
        for (std::size_t i = 0; i < batch.samples.size(); ++i) {
            const SampleRecord& rec = batch.samples[i];
            hs.push_back(fm_host_sample{payloads[2 * i].object.payload.data(), payloads[2 * i + 1].object.payload.data(),
                                        rec.data[static_cast<std::size_t>(adv_col)].as_float()});
            fk.push_back(fm_sample_key{rec.sample_id.input_id.c_str(), rec.sample_id.number_of_turns,
                                       rec.sample_id.trajectory_id, rec.policy_version});
        }
        flexmarl_detail::check(fm_agent_add_grad_keys(g.h, fk.data(), static_cast<int>(fk.size())));
        std::int64_t ticket = -1;
        flexmarl_detail::check(fm_train_micro_batch_host(g.h, hs.data(), static_cast<int>(hs.size()),
                                                         cfg_.global_batch, &ticket));
        for (GradKey& k : keys) g.keys.insert(std::move(k));

        const double duration = static_cast<double>(batch.samples.size()) * cfg_.train_seconds_per_sample /
                                static_cast<double>(g.devices.size());
        const SimTime start = data_ready;
        for (DeviceId d : g.devices) cluster_.charge_busy(d, start, duration, &log_);
        g.in_flight = true;

        GradReport report;
        report.agent_id = agent;
        report.batch_version = batch.policy_version;
        report.engine_version = version;
        report.batch_size = batch.samples.size();
        report.t_start = start;
        report.t_end = start + duration;
        loop_.schedule(report.t_end, [this, agent, report, ticket, on_done = std::move(on_done)]() mutable {
            Group& gg = group(agent);
            flexmarl_detail::check(fm_agent_sync(gg.h));
            fm_report rep{};
            const int got = fm_agent_poll_report(gg.h, ticket, &rep);
            if (got != 1) flexmarl_detail::raise_status(got < 0 ? got : FM_ERR_CUDA);
            report.grad_norm = rep.grad_norm;  // ||sum_mb A_i term_i||_F / G (training.hpp:417)
            gg.in_flight = false;
            log_.append(report.t_end, "micro_grad",
                        Json{{"agent", agent},
                             {"version", report.batch_version},
                             {"engine_version", report.engine_version},
                             {"samples", report.batch_size},
                             {"grad_norm", report.grad_norm}});
            if (on_done) on_done(report);
        });
    }

    // training.hpp:435-456: the fused Adam on the GPU, then the packed f64 weights are
    // published on the gang's lead device as the reference does.
    std::int64_t apply_global_update(const std::string& agent) {
        Group& g = group(agent);
        if (g.state != GroupState::Active) raise(ErrorCode::InactiveGroup, agent);
        const std::int64_t acc = fm_agent_samples_accumulated(g.h);
        if (acc != cfg_.global_batch) {
            raise(ErrorCode::IncompleteBatch, agent + " accumulated " + std::to_string(acc) + " of " +
                                                  std::to_string(cfg_.global_batch));
        }
        double grad_norm = 0.0;
        std::int64_t version = 0;
        const AdamParams& a = cfg_.adam;
        flexmarl_detail::check(
            fm_apply_update(g.h, cfg_.global_batch, a.lr, a.beta1, a.beta2, a.eps, &grad_norm, &version));
        g.keys.clear();
        PolicyModel model(g.vocab, g.feat);
        flexmarl_detail::check(fm_agent_read_weights(g.h, model.weights().a.data()));
        publish_weights(agent, model, version, Placement::device(g.devices.front()));
        log_.append(loop_.now(), "update", Json{{"agent", agent}, {"version", version}, {"grad_norm", grad_norm}});
        return version;
    }

    // training.hpp:459-467 (unchanged)
    void publish_weights(const std::string& agent, const PolicyModel& model, std::int64_t version,
                         const Placement& where) {
        F64Tensor t;
        t.shape = {model.vocab_size(), model.feature_dim()};
        t.data = model.weights().a;
        auto [buf, layout] = ObjectStore::pack_weights({t});
        (void)layout;
        objects_.set(weights_key(agent, version), std::move(buf), where);
    }

    static std::string weights_key(const std::string& agent, std::int64_t version) {
        return "weights:" + agent + ":v" + std::to_string(version);
    }

private:
    struct Group {
        GroupState state = GroupState::Destroyed;
        std::size_t vocab = 0;
        std::size_t feat = 0;
        std::vector<DeviceId> devices;
        std::vector<Reservation> reservations;
        NodeId last_node = -1;
        bool in_flight = false;
        std::string latest_checkpoint;
        std::uint64_t checkpoint_counter = 0;
        fm_agent* h = nullptr;      // the trainer state on the GPU while Active
        std::set<GradKey> keys;     // samples of the current global step (DuplicateSample)
        PolicyState mirror;         // state()'s host copy
    };

    fm_ctx* ctx() {
        if (!ctx_) flexmarl_detail::check(fm_ctx_create(device_, &ctx_));
        return ctx_;
    }

    // A mid-step checkpoint from fm_agent_serialize carries the step's gradient as one
    // summed cache entry.  Rewritten with one entry per GradKey of the step, in the
    // reference's canonical (std::map) order — the sum under the first key, zero
    // matrices under the others — it has exactly the reference's length, so the
    // simulated offload / restore transfers (and the run's event order) are the
    // reference's, and the reference's canonical reduction still yields the same sum.
    std::vector<std::uint8_t> per_sample_cache(const Group& g, const std::vector<std::uint8_t>& blob) const {
        const std::uint64_t P = static_cast<std::uint64_t>(g.vocab) * g.feat;
        const std::size_t state_end = 5 * 8 + 3 * (16 + 8 * P);
        if (blob.size() < state_end + 8) raise(ErrorCode::LayoutOutOfBounds, "short checkpoint");
        std::uint64_t cache_n = 0;
        std::memcpy(&cache_n, blob.data() + state_end, 8);
        std::vector<std::uint8_t> out(blob.begin(), blob.begin() + static_cast<long>(state_end));
        append_u64(out, g.keys.size());
        const std::uint8_t* sum = cache_n ? blob.data() + blob.size() - 8 * P : nullptr;
        bool first = true;
        for (const GradKey& k : g.keys) {
            const auto& [input, turns, traj, ver] = k;
            append_u64(out, input.size());
            append_bytes(out, input.data(), input.size());
            append_u64(out, static_cast<std::uint64_t>(turns));
            append_u64(out, static_cast<std::uint64_t>(traj));
            append_u64(out, static_cast<std::uint64_t>(ver));
            append_u64(out, g.vocab);
            append_u64(out, g.feat);
            const std::size_t at = out.size();
            out.resize(at + 8 * P, 0);  // +0.0
            if (first && sum) std::memcpy(out.data() + at, sum, 8 * P);
            first = false;
        }
        return out;
    }

    PolicyState read_state(const std::string& agent, const Group& g) const {
        PolicyState st;
        st.agent_id = agent;
        st.version = fm_agent_version(g.h);
        st.samples_accumulated = fm_agent_samples_accumulated(g.h);
        st.model = PolicyModel(g.vocab, g.feat);
        flexmarl_detail::check(fm_agent_read_weights(g.h, st.model.weights().a.data()));
        const std::size_t P = g.vocab * g.feat;
        std::vector<float> m(P), v(P);
        std::int64_t step = 0;
        flexmarl_detail::check(fm_agent_read_moments(g.h, m.data(), v.data(), &step));
        st.opt.m = Matrix(g.vocab, g.feat);
        st.opt.v = Matrix(g.vocab, g.feat);
        for (std::size_t i = 0; i < P; ++i) {
            st.opt.m.a[i] = m[i];
            st.opt.v.a[i] = v[i];
        }
        st.opt.step_count = step;
        return st;
    }

    Group& group(const std::string& agent) {
        auto it = groups_.find(agent);
        if (it == groups_.end()) raise(ErrorCode::ConfigError, "unknown agent " + agent);
        return it->second;
    }
    const Group& group(const std::string& agent) const {
        auto it = groups_.find(agent);
        if (it == groups_.end()) raise(ErrorCode::ConfigError, "unknown agent " + agent);
        return it->second;
    }

    // STRICT_PACK placement (training.hpp:498-531): devices_per_group unbound pool
    // devices of one node — the node the agent last ran on if it fits, else the
    // lowest-numbered node that does — in pool order
    std::vector<DeviceId> pick_devices(const std::string& agent) const {
        std::set<DeviceId> bound;
        for (const auto& kv : groups_) bound.insert(kv.second.devices.begin(), kv.second.devices.end());
        std::map<NodeId, std::vector<DeviceId>> unbound;
        for (DeviceId d : pool_.devices)
            if (!bound.count(d)) unbound[cluster_.node_of_device(d)].push_back(d);
        const std::size_t want = static_cast<std::size_t>(cfg_.devices_per_group);
        const NodeId last = group(agent).last_node;
        auto it = last >= 0 ? unbound.find(last) : unbound.end();
        if (it == unbound.end() || it->second.size() < want)
            it = std::find_if(unbound.begin(), unbound.end(),
                              [want](const auto& kv) { return kv.second.size() >= want; });
        if (it == unbound.end()) return {};
        return std::vector<DeviceId>(it->second.begin(), it->second.begin() + static_cast<long>(want));
    }

    EventLoop& loop_;
    Cluster& cluster_;
    ObjectStore& objects_;
    EventLog& log_;
    ResourcePool pool_;
    TrainingConfig cfg_;
    std::map<std::string, Group> groups_;
    fm_ctx* ctx_ = nullptr;
    int device_ = 0;
    int precision_ = FM_PRECISION_BF16_TC;
};

}  // namespace marlsim

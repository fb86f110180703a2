// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
//
// Thin extern "C" driver around the UNMODIFIED reference headers under
// /root/reference/proj/include/marlsim (compiled read-only by oracle/Makefile
// into oracle/_ref/libmarlsim_ref.so).  Nothing here re-implements reference
// arithmetic: every number comes out of the reference's own classes:
//   * PolicyModel::seeded / featurize / probabilities / accumulate_grad_log_prob
//     (policy.hpp:29-35, 42-51, 54-70, 79-91)
//   * adam_step, group_advantages, rule_reward (training.hpp:37-51, 54-67, 71-83)
//   * ExperienceStore::insert/set_cell/poll_micro_batch/complete
//     (experience_store.hpp:44-148) and TrainingEngine::train_micro_batch /
//     apply_global_update (training.hpp:355-456), driven standalone as in
//     SURVEY.md Appendix A (no suspend/activate round trip: training.hpp:146
//     transposes W when V != D).
//
// Used by tests/ (golden-vector generation and live cross-checks) and by
// bench.py's reference arm / cpu_baseline leg.  Never linked into the product.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "marlsim/codec.hpp"
#include "marlsim/experience_store.hpp"
#include "marlsim/training.hpp"

using namespace marlsim;

namespace {

thread_local std::string g_err;

HeterogeneousObject as_list_payload(const std::uint8_t* base, std::int64_t off) {
    // The encoded form is [u64 n][u64 tok]*n (codec.hpp:15-22); recover its length.
    std::uint64_t n;
    std::memcpy(&n, base + off, 8);
    HeterogeneousObject o;
    o.dtype = DType::List;
    o.payload.assign(base + off, base + off + 8 + 8 * n);
    return o;
}

double now_s() {
    using clk = std::chrono::steady_clock;
    return std::chrono::duration<double>(clk::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_agent_seed(std::uint64_t seed, const char* agent) {
    // training.hpp:245-248
    return mix_str(mix_u64(seed, 0x1217), agent);
}

std::uint64_t ref_mix_u64(std::uint64_t seed, std::uint64_t value) { return mix_u64(seed, value); }
std::uint64_t ref_mix_str(std::uint64_t seed, const char* s) { return mix_str(seed, s); }

// Draws `n` values from one Rng stream: kind 0 next_u64, 1 next_unit, 2 next_normal,
// 3 next_below(arg).
void ref_rng_draw(std::uint64_t seed, int kind, std::uint64_t arg, std::uint64_t n, void* out) {
    Rng rng(seed);
    for (std::uint64_t i = 0; i < n; ++i) {
        switch (kind) {
            case 0: static_cast<std::uint64_t*>(out)[i] = rng.next_u64(); break;
            case 1: static_cast<double*>(out)[i] = rng.next_unit(); break;
            case 2: static_cast<double*>(out)[i] = rng.next_normal(); break;
            default: static_cast<std::uint64_t*>(out)[i] = rng.next_below(arg); break;
        }
    }
}

void ref_seeded_weights(std::uint64_t V, std::uint64_t D, std::uint64_t seed, double* out) {
    PolicyModel m = PolicyModel::seeded(V, D, seed);
    std::memcpy(out, m.weights().a.data(), V * D * sizeof(double));
}

void ref_group_advantages(const double* rewards, int n, double eps, double* out) {
    std::vector<double> r(rewards, rewards + n);
    std::vector<double> a = group_advantages(r, eps);
    for (int i = 0; i < n; ++i) out[i] = a[static_cast<std::size_t>(i)];
}

double ref_rule_reward(const int* resp, int n, const int* pattern, int np) {
    return rule_reward(std::vector<Token>(resp, resp + n), std::vector<Token>(pattern, pattern + np));
}

// One adam_step on flat arrays (w, m, v updated in place; *step incremented).
void ref_adam_step(double* w, double* m, double* v, std::int64_t* step, const double* g,
                   std::uint64_t n, double lr, double b1, double b2, double eps) {
    Matrix W(1, n), G(1, n);
    std::memcpy(W.a.data(), w, n * 8);
    std::memcpy(G.a.data(), g, n * 8);
    OptimizerState opt;
    opt.step_count = *step;
    if (*step > 0) {
        opt.m = Matrix(1, n);
        opt.v = Matrix(1, n);
        std::memcpy(opt.m.a.data(), m, n * 8);
        std::memcpy(opt.v.a.data(), v, n * 8);
    }
    adam_step(W, opt, AdamParams{lr, b1, b2, eps}, G);
    std::memcpy(w, W.a.data(), n * 8);
    std::memcpy(m, opt.m.a.data(), n * 8);
    std::memcpy(v, opt.v.a.data(), n * 8);
    *step = opt.step_count;
}

void ref_featurize(std::uint64_t V, std::uint64_t D, const int* ctx, int n, double* out) {
    PolicyModel m(V, D);
    std::vector<double> phi = m.featurize(std::span<const Token>(ctx, static_cast<std::size_t>(n)));
    std::memcpy(out, phi.data(), D * 8);
}

void ref_probabilities(std::uint64_t V, std::uint64_t D, const double* W, const int* ctx, int n,
                       double* out) {
    PolicyModel m(V, D);
    std::memcpy(m.weights().a.data(), W, V * D * 8);
    std::vector<double> p = m.probabilities(std::span<const Token>(ctx, static_cast<std::size_t>(n)));
    std::memcpy(out, p.data(), V * 8);
}

// out += weight * dlog pi(action|ctx)/dW
void ref_accumulate_grad(std::uint64_t V, std::uint64_t D, const double* W, const int* ctx, int n,
                         int action, double weight, double* out) {
    PolicyModel m(V, D);
    std::memcpy(m.weights().a.data(), W, V * D * 8);
    Matrix o(V, D);
    std::memcpy(o.a.data(), out, V * D * 8);
    m.accumulate_grad_log_prob(std::span<const Token>(ctx, static_cast<std::size_t>(n)), action,
                               weight, o);
    std::memcpy(out, o.a.data(), V * D * 8);
}

// Reference rollout generation (policy.hpp:119-130, seeded as rollout.hpp:638-645
// when tok_seed is derived by the caller).  Returns the number of tokens.
int ref_generate(std::uint64_t V, std::uint64_t D, const double* W, const int* prompt, int np,
                 int max_tokens, std::uint64_t tok_seed, int* out_tokens, double* out_logp) {
    PolicyModel m(V, D);
    std::memcpy(m.weights().a.data(), W, V * D * 8);
    Rng rng(tok_seed);
    auto g = m.generate(std::span<const Token>(prompt, static_cast<std::size_t>(np)),
                        static_cast<std::size_t>(max_tokens), &rng);
    for (std::size_t i = 0; i < g.tokens.size(); ++i) {
        out_tokens[i] = g.tokens[i];
        out_logp[i] = g.log_probs[i];
    }
    return static_cast<int>(g.tokens.size());
}

// Drives the reference ExperienceStore + TrainingEngine for one agent through
// `n_updates` global steps.  Sample i belongs to data
// version versions[i] (0..n_updates-1); samples are inserted in `insert_order`
// per version, their prompt/response payloads are the encoded token lists at
// payloads+prompt_off[i] / payloads+resp_off[i], their advantage advantages[i].
// Outputs: initial/final W, final Adam moments, the index of every polled
// sample in poll order, every micro-batch GradReport::grad_norm and every
// update grad_norm (from the "update" log record).  Wall times of the
// train_micro_batch and apply_global_update calls go to t_train_s / t_update_s.
int ref_run_agent(const char* agent, std::uint64_t V, std::uint64_t D, std::uint64_t seed,
                  std::int64_t global_batch, std::int64_t micro_batch, int n_updates, int n_samples,
                  const char* const* input_ids, const std::int32_t* turns,
                  const std::int32_t* trajs, const std::int64_t* versions,
                  const std::uint8_t* payloads, const std::int64_t* prompt_off,
                  const std::int64_t* resp_off, const double* advantages,
                  const std::int32_t* insert_order, double lr, double* W0_out, double* W_out,
                  double* m_out, double* v_out, std::int32_t* poll_order_out,
                  double* mb_grad_norm_out, double* upd_grad_norm_out, double* t_train_s,
                  double* t_update_s, int skip_update) {
    try {
        EventLoop loop;
        Cluster cluster(1, 8, 1ULL << 50, 1ULL << 50);
        EventLog log;
        ObjectStore objects(loop, cluster, log);
        ExperienceStore exp(objects);
        TrainingConfig tc;
        tc.adam.lr = lr;
        tc.global_batch = global_batch;
        tc.seed = seed;
        TrainingEngine trainer(loop, cluster, objects, log, ResourcePool{PoolKind::Training, {0}},
                               tc);
        const std::string a(agent);
        trainer.add_agent(a, V, D);
        trainer.activate(a, nullptr);
        loop.run();
        TableSchema schema{a,
                           {{"prompt", ColumnType::List},
                            {"response", ColumnType::List},
                            {"advantage", ColumnType::Float}}};
        exp.create_table(schema);
        if (W0_out) {
            const PolicyModel m0 = trainer.initial_model(a);
            std::memcpy(W0_out, m0.weights().a.data(), V * D * 8);
        }
        double tt = 0.0, tu = 0.0;
        int polled = 0, mb_i = 0;
        for (int u = 0; u < n_updates; ++u) {
            for (int k = 0; k < n_samples; ++k) {
                const int i = insert_order[k];
                if (versions[i] != u) continue;
                SampleId id{input_ids[i], turns[i], trajs[i]};
                exp.insert(a, u, id);
                exp.set_cell_payload(a, id, u, "prompt", as_list_payload(payloads, prompt_off[i]), 0);
                exp.set_cell_payload(a, id, u, "response", as_list_payload(payloads, resp_off[i]), 0);
                exp.set_cell(a, id, u, "advantage", CellValue::of_float(advantages[i]));
            }
            const std::int64_t per_step = global_batch / micro_batch;
            for (std::int64_t b = 0; b < per_step; ++b) {
                auto batch = exp.poll_micro_batch(a, u, static_cast<std::size_t>(micro_batch));
                if (!batch) {
                    g_err = "poll returned nothing at update " + std::to_string(u);
                    return 1;
                }
                for (const SampleRecord& rec : batch->samples) {
                    int found = -1;
                    for (int i = 0; i < n_samples; ++i) {
                        if (versions[i] == rec.policy_version && rec.sample_id.input_id == input_ids[i] &&
                            rec.sample_id.number_of_turns == turns[i] &&
                            rec.sample_id.trajectory_id == trajs[i]) {
                            found = i;
                            break;
                        }
                    }
                    poll_order_out[polled++] = found;
                }
                double gn = 0.0;
                const double t0 = now_s();
                trainer.train_micro_batch(a, *batch, schema,
                                          [&gn](const GradReport& r) { gn = r.grad_norm; });
                tt += now_s() - t0;
                loop.run();
                exp.complete(a, batch->samples);
                mb_grad_norm_out[mb_i++] = gn;
            }
            if (skip_update) continue;  // timing-only runs (bench.py reference arm)
            const double t1 = now_s();
            trainer.apply_global_update(a);
            tu += now_s() - t1;
            upd_grad_norm_out[u] = log.filter("update").back()->payload["grad_norm"].get<double>();
        }
        if (!W_out && !m_out && !v_out) {
            if (t_train_s) *t_train_s = tt;
            if (t_update_s) *t_update_s = tu;
            return 0;
        }
        PolicyState st = trainer.peek_state(a);
        if (W_out) std::memcpy(W_out, st.model.weights().a.data(), V * D * 8);
        if (m_out && st.opt.m.size()) std::memcpy(m_out, st.opt.m.a.data(), V * D * 8);
        if (v_out && st.opt.v.size()) std::memcpy(v_out, st.opt.v.a.data(), V * D * 8);
        if (t_train_s) *t_train_s = tt;
        if (t_update_s) *t_update_s = tu;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// Reference ExperienceStore poll ordering alone: inserts the records (all
// ready, all version `version`) in the given order and polls batches of `mb`
// until nothing is returned.  Writes polled record indices; returns count.
int ref_poll_order(int n, const char* const* input_ids, const std::int32_t* turns,
                   const std::int32_t* trajs, const std::int64_t* rec_versions,
                   const std::uint8_t* ready, std::int64_t current_version, std::int64_t mb,
                   std::int32_t* out) {
    try {
        EventLoop loop;
        Cluster cluster(1, 1, 1ULL << 40, 1ULL << 40);
        EventLog log;
        ObjectStore objects(loop, cluster, log);
        ExperienceStore exp(objects);
        exp.create_table(TableSchema{"a", {{"advantage", ColumnType::Float}}});
        for (int i = 0; i < n; ++i) {
            SampleId id{input_ids[i], turns[i], trajs[i]};
            exp.insert("a", rec_versions[i], id);
            if (ready[i]) exp.set_cell("a", id, rec_versions[i], "advantage", CellValue::of_float(0.0));
        }
        int k = 0;
        while (auto b = exp.poll_micro_batch("a", current_version, static_cast<std::size_t>(mb))) {
            for (const SampleRecord& rec : b->samples) {
                for (int i = 0; i < n; ++i) {
                    if (rec_versions[i] == rec.policy_version && rec.sample_id.input_id == input_ids[i] &&
                        rec.sample_id.number_of_turns == turns[i] && rec.sample_id.trajectory_id == trajs[i]) {
                        out[k++] = i;
                        break;
                    }
                }
            }
        }
        return k;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"

extern "C" {

// PolicyState::serialize (training.hpp:107-133) of a state with the given
// fields and an empty gradient cache.  Returns the byte length; writes when
// out != NULL and cap suffices.
std::uint64_t ref_serialize_state(std::int64_t version, std::int64_t step, std::int64_t samples,
                                  std::uint64_t V, std::uint64_t D, const double* W, const double* m,
                                  const double* v, std::uint8_t* out, std::uint64_t cap) {
    PolicyState st;
    st.version = version;
    st.samples_accumulated = samples;
    st.opt.step_count = step;
    st.model = PolicyModel(V, D);
    std::memcpy(st.model.weights().a.data(), W, V * D * 8);
    if (m && v) {
        st.opt.m = Matrix(V, D);
        st.opt.v = Matrix(V, D);
        std::memcpy(st.opt.m.a.data(), m, V * D * 8);
        std::memcpy(st.opt.v.a.data(), v, V * D * 8);
    }
    const std::vector<std::uint8_t> b = st.serialize();
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    return b.size();
}

// PolicyState::deserialize (training.hpp:135-164) as the reference does it;
// reports the dims it read for W (exposes the argument-order defect at :146).
int ref_deserialize_state(const std::uint8_t* in, std::uint64_t len, std::uint64_t* w_rows,
                          std::uint64_t* w_cols, double* W_out, std::int64_t* version,
                          std::uint64_t* cache_n) {
    try {
        std::vector<std::uint8_t> b(in, in + len);
        PolicyState st = PolicyState::deserialize("x", b);
        *w_rows = st.model.weights().rows;
        *w_cols = st.model.weights().cols;
        if (W_out) std::memcpy(W_out, st.model.weights().a.data(), st.model.weights().a.size() * 8);
        *version = st.version;
        *cache_n = st.grad_cache.size();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Experience-store lifecycle script (SURVEY §8f-4 golden vectors).
//
// Replays a text script against the reference's own ExperienceStore on one
// table with the orchestrator's schema (orchestrator.hpp:191-195: prompt List,
// response List, logprobs Tensor, reward Float, advantage Float) and writes
// one result line per op.  Group release follows RolloutEngine::release_group
// (rollout.hpp:812-834): rule_reward on each survivor's scored response,
// group_advantages over the survivors, both cells set on every listed record.
//   insert V id t j              -> "ok" | "err <fm_status>"
//   setf V id t j col <hexfloat> -> "ok" | "err .."
//   setp V id t j col n x1..xn   -> "ok" | "err .."   (token list payload)
//   poll V mb                    -> "none" | "id_t_j@V:<adv hexfloat> ..." | "err .."
//   complete k (V id t j)*k      -> "ok" | "err .."
//   purge_stale V                -> "<count>"
//   purge_inputs k id*k          -> "<count>"
//   drop V id t j                -> "0" | "1"
//   ready V                      -> "<count>"
//   count                        -> "<count>"
//   release eps np p*np ns (V id t j nrec (V id t j)*nrec)*ns
//                                -> "<reward hex>/<adv hex> ..." | "err .."
// ---------------------------------------------------------------------------
namespace {
// whitespace tokenizer (no iostreams: the driver's static libstdc++ is not
// initialised for them when loaded into Python)
struct Toks {
    std::vector<std::string> v;
    std::size_t i = 0;
    explicit Toks(const std::string& line) {
        std::size_t p = 0;
        while (p < line.size()) {
            while (p < line.size() && (line[p] == ' ' || line[p] == '\t' || line[p] == '\r')) ++p;
            std::size_t q = p;
            while (q < line.size() && line[q] != ' ' && line[q] != '\t' && line[q] != '\r') ++q;
            if (q > p) v.push_back(line.substr(p, q - p));
            p = q;
        }
    }
    std::string str() { return i < v.size() ? v[i++] : std::string(); }
    long long num() { return std::strtoll(str().c_str(), nullptr, 10); }
    Toks& operator>>(std::string& x) { x = str(); return *this; }
    Toks& operator>>(int& x) { x = static_cast<int>(num()); return *this; }
    Toks& operator>>(std::int64_t& x) { x = num(); return *this; }
    Toks& operator>>(std::size_t& x) { x = static_cast<std::size_t>(num()); return *this; }
};
}  // namespace

extern "C" {

std::uint64_t ref_store_script(const char* script, char* out, std::uint64_t cap) {
    std::string res;
    try {
        EventLoop loop;
        Cluster cluster(1, 1, 1ULL << 40, 1ULL << 40);
        EventLog log;
        ObjectStore objects(loop, cluster, log);
        ExperienceStore exp(objects);
        const std::string A = "agent";
        exp.create_table(TableSchema{A,
                                     {{"prompt", ColumnType::List},
                                      {"response", ColumnType::List},
                                      {"logprobs", ColumnType::Tensor},
                                      {"reward", ColumnType::Float},
                                      {"advantage", ColumnType::Float}}});
        std::map<std::tuple<std::string, int, int, std::int64_t>, std::vector<Token>> responses;
        const std::string text(script);
        std::size_t pos = 0;
        char buf[64];
        auto hexf = [&](double x) {
            std::snprintf(buf, sizeof buf, "%a", x);
            return std::string(buf);
        };
        while (pos < text.size()) {
            std::size_t nl = text.find('\n', pos);
            if (nl == std::string::npos) nl = text.size();
            const std::string line = text.substr(pos, nl - pos);
            pos = nl + 1;
            if (line.empty()) continue;
            Toks ls(line);
            std::string op;
            ls >> op;
            std::string r;
            try {
                if (op == "insert") {
                    std::int64_t v; std::string id; int t, j;
                    ls >> v >> id >> t >> j;
                    exp.insert(A, v, SampleId{id, t, j});
                    r = "ok";
                } else if (op == "setf") {
                    std::int64_t v; std::string id, col, x; int t, j;
                    ls >> v >> id >> t >> j >> col >> x;
                    exp.set_cell(A, SampleId{id, t, j}, v, col, CellValue::of_float(std::strtod(x.c_str(), nullptr)));
                    r = "ok";
                } else if (op == "setp") {
                    std::int64_t v; std::string id, col; int t, j; std::size_t n;
                    ls >> v >> id >> t >> j >> col >> n;
                    std::vector<Token> toks(n);
                    for (auto& x : toks) ls >> x;
                    exp.set_cell_payload(A, SampleId{id, t, j}, v, col, encode_tokens(toks), 0);
                    if (col == "response") responses[{id, t, j, v}] = toks;
                    r = "ok";
                } else if (op == "poll") {
                    std::int64_t v; std::size_t mb;
                    ls >> v >> mb;
                    auto b = exp.poll_micro_batch(A, v, mb);
                    if (!b) {
                        r = "none";
                    } else {
                        const int ac = exp.schema(A).column_index("advantage");
                        for (const SampleRecord& rec : b->samples) {
                            if (!r.empty()) r += ' ';
                            r += rec.sample_id.render() + "@" + std::to_string(rec.policy_version) + ":" +
                                 hexf(rec.data[static_cast<std::size_t>(ac)].as_float());
                        }
                    }
                } else if (op == "complete") {
                    int k;
                    ls >> k;
                    std::vector<SampleRecord> recs;
                    for (int i = 0; i < k; ++i) {
                        std::int64_t v; std::string id; int t, j;
                        ls >> v >> id >> t >> j;
                        SampleRecord sr;
                        sr.policy_version = v;
                        sr.sample_id = SampleId{id, t, j};
                        recs.push_back(sr);
                    }
                    exp.complete(A, recs);
                    r = "ok";
                } else if (op == "purge_stale") {
                    std::int64_t v;
                    ls >> v;
                    r = std::to_string(exp.purge_stale(A, v));
                } else if (op == "purge_inputs") {
                    int k;
                    ls >> k;
                    std::set<std::string> ids;
                    for (int i = 0; i < k; ++i) {
                        std::string id;
                        ls >> id;
                        ids.insert(id);
                    }
                    r = std::to_string(exp.purge_inputs(A, ids));
                } else if (op == "drop") {
                    std::int64_t v; std::string id; int t, j;
                    ls >> v >> id >> t >> j;
                    r = exp.drop_record(A, SampleId{id, t, j}, v) ? "1" : "0";
                } else if (op == "ready") {
                    std::int64_t v;
                    ls >> v;
                    r = std::to_string(exp.ready_count(A, v));
                } else if (op == "count") {
                    r = std::to_string(exp.record_count(A));
                } else if (op == "release") {
                    double eps; int np, ns;
                    std::string epss;
                    ls >> epss >> np;
                    eps = std::strtod(epss.c_str(), nullptr);
                    std::vector<Token> pat(static_cast<std::size_t>(np));
                    for (auto& x : pat) ls >> x;
                    ls >> ns;
                    std::vector<double> rewards;
                    std::vector<std::vector<std::pair<SampleId, std::int64_t>>> recs(static_cast<std::size_t>(ns));
                    for (int i = 0; i < ns; ++i) {
                        std::int64_t v; std::string id; int t, j, nrec;
                        ls >> v >> id >> t >> j >> nrec;
                        rewards.push_back(rule_reward(responses.at({id, t, j, v}), pat));
                        for (int q = 0; q < nrec; ++q) {
                            std::int64_t v2; std::string id2; int t2, j2;
                            ls >> v2 >> id2 >> t2 >> j2;
                            recs[static_cast<std::size_t>(i)].push_back({SampleId{id2, t2, j2}, v2});
                        }
                    }
                    const std::vector<double> adv = group_advantages(rewards, eps);
                    for (int i = 0; i < ns; ++i) {
                        for (const auto& [sid, v] : recs[static_cast<std::size_t>(i)]) {
                            exp.set_cell(A, sid, v, "reward", CellValue::of_float(rewards[static_cast<std::size_t>(i)]));
                            exp.set_cell(A, sid, v, "advantage", CellValue::of_float(adv[static_cast<std::size_t>(i)]));
                        }
                        if (!r.empty()) r += ' ';
                        r += hexf(rewards[static_cast<std::size_t>(i)]) + "/" + hexf(adv[static_cast<std::size_t>(i)]);
                    }
                    if (r.empty()) r = "ok";
                } else {
                    r = "bad-op";
                }
            } catch (const Error& e) {
                r = "err " + std::to_string(static_cast<int>(e.code()) + 1);
            }
            res += r;
            res += '\n';
        }
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0;
    }
    if (out && cap > res.size()) std::memcpy(out, res.c_str(), res.size() + 1);
    return res.size() + 1;
}

}  // extern "C"

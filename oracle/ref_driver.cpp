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
#include <cstring>
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

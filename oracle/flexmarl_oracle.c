/* oracle/flexmarl_oracle.c — TEST INFRASTRUCTURE ONLY (see flexmarl_oracle.h).
 *
 * Plain-C restatement of the reference micro-batch policy-update path.  Each
 * function follows the reference arithmetic operation-for-operation (same
 * summation order, same libm calls) so that it agrees bit-for-bit with the
 * compiled reference (oracle/_ref) on every golden vector.  Parity pinned by
 * tests/test_oracle.py against the tests/golden npz fixtures and, when oracle/_ref is
 * built, against the live reference.
 */
#define _GNU_SOURCE
#include "flexmarl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:14-64 --------------------------------------------------- */

uint64_t fmo_splitmix64(uint64_t* state) { /* rng.hpp:14-19 */
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t fmo_mix_u64(uint64_t seed, uint64_t value) { /* rng.hpp:21-24 */
    uint64_t s = seed ^ (value + 0x9e3779b97f4a7c15ULL + (seed << 6) + (seed >> 2));
    return fmo_splitmix64(&s);
}

uint64_t fmo_mix_str(uint64_t seed, const char* text) { /* rng.hpp:26-34 */
    uint64_t h = seed ^ 0xcbf29ce484222325ULL;
    for (const unsigned char* c = (const unsigned char*)text; *c; ++c) {
        h ^= *c;
        h *= 0x100000001b3ULL;
        h = fmo_mix_u64(h, *c);
    }
    return h;
}

static double rng_unit(uint64_t* st) { /* rng.hpp:43-48 */
    const uint64_t bits = fmo_splitmix64(st) >> 11;
    double u = (double)bits * 0x1.0p-53;
    if (u <= 0.0) u = 0x1.0p-53;
    return u;
}

static double rng_normal(uint64_t* st) { /* rng.hpp:55-59 */
    const double u1 = rng_unit(st);
    const double u2 = rng_unit(st);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

void fmo_rng_draw(uint64_t seed, int kind, uint64_t arg, uint64_t n, void* out) {
    uint64_t st = seed;
    for (uint64_t i = 0; i < n; ++i) {
        switch (kind) {
            case 0: ((uint64_t*)out)[i] = fmo_splitmix64(&st); break;
            case 1: ((double*)out)[i] = rng_unit(&st); break;
            case 2: ((double*)out)[i] = rng_normal(&st); break;
            default: ((uint64_t*)out)[i] = arg == 0 ? 0 : fmo_splitmix64(&st) % arg; break;
        }
    }
}

/* ---- training.hpp:245-248, policy.hpp:29-35 --------------------------- */

uint64_t fmo_agent_seed(uint64_t seed, const char* agent) {
    return fmo_mix_str(fmo_mix_u64(seed, 0x1217), agent);
}

void fmo_seeded_weights(uint64_t V, uint64_t D, uint64_t seed, double* out) {
    uint64_t st = seed;
    for (uint64_t i = 0; i < V * D; ++i) out[i] = 0.5 * rng_normal(&st);
}

/* ---- training.hpp:54-67 ----------------------------------------------- */

void fmo_group_advantages(const double* r, int n, double eps, double* out) {
    if (n <= 0) return;
    double mean = 0.0;
    for (int i = 0; i < n; ++i) mean += r[i];
    mean /= (double)n;
    double var = 0.0;
    for (int i = 0; i < n; ++i) var += (r[i] - mean) * (r[i] - mean);
    var /= (double)n;
    const double sd = sqrt(var);
    for (int i = 0; i < n; ++i) out[i] = (r[i] - mean) / (sd + eps);
}

/* ---- training.hpp:71-83 ----------------------------------------------- */

double fmo_rule_reward(const int* resp, int n, const int* pattern, int np) {
    if (n == 0 || np == 0) return 0.0;
    int best = 0;
    for (int s = 0; s < n; ++s) {
        int len = 0;
        while (len < np && s + len < n && resp[s + len] == pattern[len]) ++len;
        if (len > best) best = len;
    }
    return (double)best / (double)np;
}

/* ---- training.hpp:37-51 ----------------------------------------------- */

void fmo_adam_step(double* w, double* m, double* v, int64_t* step, const double* g, uint64_t n,
                   double lr, double b1, double b2, double eps) {
    *step += 1;
    const double bc1 = 1.0 - pow(b1, (double)*step);
    const double bc2 = 1.0 - pow(b2, (double)*step);
    for (uint64_t i = 0; i < n; ++i) {
        const double gi = g[i];
        m[i] = b1 * m[i] + (1.0 - b1) * gi;
        v[i] = b2 * v[i] + (1.0 - b2) * gi * gi;
        const double mhat = m[i] / bc1;
        const double vhat = v[i] / bc2;
        w[i] -= lr * mhat / (sqrt(vhat) + eps);
    }
}

/* ---- codec.hpp:15-30 -------------------------------------------------- */

uint64_t fmo_decode_tokens(const uint8_t* payload, int* out) {
    uint64_t n;
    memcpy(&n, payload, 8);
    if (out) {
        for (uint64_t i = 0; i < n; ++i) {
            uint64_t t;
            memcpy(&t, payload + 8 + 8 * i, 8);
            out[i] = (int)(uint32_t)t; /* static_cast<Token>(u64): modular (C++20) */
        }
    }
    return n;
}

uint64_t fmo_encode_tokens(const int* tokens, uint64_t n, uint8_t* out) {
    memcpy(out, &n, 8);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t t = (uint64_t)(int64_t)tokens[i]; /* static_cast<uint64_t>(int) */
        memcpy(out + 8 + 8 * i, &t, 8);
    }
    return 8 + 8 * n;
}

/* ---- policy.hpp:42-91 ------------------------------------------------- */

void fmo_featurize(uint64_t V, uint64_t D, const int* ctx, int len, double* phi) {
    (void)V;
    for (uint64_t d = 0; d < D; ++d) phi[d] = 0.0;
    const int n = len < 4 ? len : 4;
    if (n == 0) return;
    const double w = 1.0 / (double)n;
    for (int i = len - n; i < len; ++i) phi[(uint64_t)(int64_t)ctx[i] % D] += w;
}

static void probs_from_phi(uint64_t V, uint64_t D, const double* W, const double* phi, double* z) {
    for (uint64_t v = 0; v < V; ++v) {
        double s = 0.0;
        for (uint64_t d = 0; d < D; ++d) s += W[v * D + d] * phi[d];
        z[v] = s;
    }
    double zmax = z[0];
    for (uint64_t v = 1; v < V; ++v)
        if (z[v] > zmax) zmax = z[v]; /* std::max_element: first maximum */
    double denom = 0.0;
    for (uint64_t v = 0; v < V; ++v) {
        z[v] = exp(z[v] - zmax);
        denom += z[v];
    }
    for (uint64_t v = 0; v < V; ++v) z[v] /= denom;
}

void fmo_probabilities(uint64_t V, uint64_t D, const double* W, const int* ctx, int n, double* p) {
    double* phi = (double*)malloc(D * sizeof(double));
    fmo_featurize(V, D, ctx, n, phi);
    probs_from_phi(V, D, W, phi, p);
    free(phi);
}

double fmo_log_prob(uint64_t V, uint64_t D, const double* W, const int* ctx, int n, int action) {
    double* p = (double*)malloc(V * sizeof(double));
    fmo_probabilities(V, D, W, ctx, n, p);
    const double lp = log(p[action]);
    free(p);
    return lp;
}

static void accumulate(uint64_t V, uint64_t D, const double* W, const int* ctx, int n, int action,
                       double weight, double* out, double* phi, double* p, double* logp) {
    fmo_featurize(V, D, ctx, n, phi);
    probs_from_phi(V, D, W, phi, p);
    if (logp) *logp = (action >= 0 && (uint64_t)action < V) ? log(p[action]) : NAN;
    for (uint64_t v = 0; v < V; ++v) {
        const double coef = weight * (((int)v == action ? 1.0 : 0.0) - p[v]);
        if (coef == 0.0) continue;
        for (uint64_t d = 0; d < D; ++d) out[v * D + d] += coef * phi[d];
    }
}

void fmo_accumulate_grad(uint64_t V, uint64_t D, const double* W, const int* ctx, int n, int action,
                         double weight, double* out) {
    double* phi = (double*)malloc(D * sizeof(double));
    double* p = (double*)malloc(V * sizeof(double));
    accumulate(V, D, W, ctx, n, action, weight, out, phi, p, NULL);
    free(phi);
    free(p);
}

/* ---- experience_store.hpp:92-114 -------------------------------------- */

typedef struct {
    const char* id;
    int32_t turns, traj;
    int64_t ver;
    int32_t idx;
} rec_key;

static int key_cmp(const void* a, const void* b) { /* std::tuple<string,int,int,int64> < */
    const rec_key* x = (const rec_key*)a;
    const rec_key* y = (const rec_key*)b;
    const int c = strcmp(x->id, y->id);
    if (c) return c;
    if (x->turns != y->turns) return x->turns < y->turns ? -1 : 1;
    if (x->traj != y->traj) return x->traj < y->traj ? -1 : 1;
    if (x->ver != y->ver) return x->ver < y->ver ? -1 : 1;
    return 0;
}

int fmo_poll_select(int n, const char* const* ids, const int32_t* turns, const int32_t* trajs,
                    const int64_t* versions, const uint8_t* ready, const uint8_t* processing,
                    int64_t current_version, int64_t mb, int32_t* out) {
    if (mb < 1) return -1;
    rec_key* k = (rec_key*)malloc((size_t)(n > 0 ? n : 1) * sizeof(rec_key));
    for (int i = 0; i < n; ++i) k[i] = (rec_key){ids[i], turns[i], trajs[i], versions[i], i};
    qsort(k, (size_t)n, sizeof(rec_key), key_cmp);
    int chosen = 0;
    for (int i = 0; i < n && chosen < mb; ++i) {
        const int j = k[i].idx;
        if (processing[j] || versions[j] != current_version || !ready[j]) continue;
        out[chosen++] = j;
    }
    free(k);
    return chosen < mb ? 0 : (int)mb;
}

/* ---- packed rows (training.hpp:378-394 + policy.hpp:42-51) ------------ */

int64_t fmo_pack_rows(int n_samples, const uint8_t* payloads, const int64_t* prompt_off,
                      const int64_t* resp_off, const double* adv, int64_t G, int32_t* actions,
                      int32_t* ctx4, int32_t* n_ctx, int32_t* row_sample, float* coef) {
    int64_t r = 0;
    for (int s = 0; s < n_samples; ++s) {
        const uint64_t np = fmo_decode_tokens(payloads + prompt_off[s], NULL);
        const uint64_t nr = fmo_decode_tokens(payloads + resp_off[s], NULL);
        int* ctx = (int*)malloc((np + nr + 1) * sizeof(int));
        fmo_decode_tokens(payloads + prompt_off[s], ctx);
        fmo_decode_tokens(payloads + resp_off[s], ctx + np);
        for (uint64_t t = 0; t < nr; ++t, ++r) {
            const int64_t len = (int64_t)(np + t);
            const int n = len < 4 ? (int)len : 4;
            if (actions) actions[r] = ctx[np + t];
            if (n_ctx) n_ctx[r] = n;
            if (row_sample) row_sample[r] = s;
            if (ctx4)
                for (int j = 0; j < 4; ++j) ctx4[4 * r + j] = j < n ? ctx[len - n + j] : -1;
            if (coef) coef[r] = n ? (float)(-adv[s] / ((double)G * (double)n)) : 0.0f;
        }
        free(ctx);
    }
    return r;
}

/* ---- training.hpp:355-456 --------------------------------------------- */

static double frob(const double* a, uint64_t n) { /* tensor.hpp:36-40 */
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += a[i] * a[i];
    return sqrt(s);
}

int fmo_run_agent(uint64_t V, uint64_t D, int64_t G, int64_t mb, int n_updates,
                  const uint8_t* payloads, const int64_t* prompt_off, const int64_t* resp_off,
                  const double* adv, double lr, double b1, double b2, double eps, double* W,
                  double* m, double* v, double* mb_grad_norm, double* upd_grad_norm,
                  double* token_logp, double* last_grad) {
    const uint64_t P = V * D;
    double* term = (double*)malloc(P * sizeof(double));
    double* micro = (double*)malloc(P * sizeof(double));
    double* grad = (double*)malloc(P * sizeof(double));
    double* phi = (double*)malloc(D * sizeof(double));
    double* p = (double*)malloc(V * sizeof(double));
    int64_t step = 0, tok = 0;
    int s = 0, mbi = 0;
    for (int u = 0; u < n_updates; ++u) {
        memset(grad, 0, P * sizeof(double));
        for (int64_t b = 0; b < G / mb; ++b) {
            memset(micro, 0, P * sizeof(double));
            for (int64_t k = 0; k < mb; ++k, ++s) {
                const uint64_t np = fmo_decode_tokens(payloads + prompt_off[s], NULL);
                const uint64_t nr = fmo_decode_tokens(payloads + resp_off[s], NULL);
                int* ctx = (int*)malloc((np + nr + 1) * sizeof(int));
                fmo_decode_tokens(payloads + prompt_off[s], ctx);
                fmo_decode_tokens(payloads + resp_off[s], ctx + np);
                memset(term, 0, P * sizeof(double));
                for (uint64_t t = 0; t < nr; ++t, ++tok)
                    accumulate(V, D, W, ctx, (int)(np + t), ctx[np + t], 1.0, term, phi, p,
                               token_logp ? &token_logp[tok] : NULL);
                for (uint64_t i = 0; i < P; ++i) term[i] *= adv[s];   /* term.scale(A) */
                for (uint64_t i = 0; i < P; ++i) micro[i] += term[i]; /* micro_sum.add */
                for (uint64_t i = 0; i < P; ++i) grad[i] += term[i];  /* canonical sum */
                free(ctx);
            }
            mb_grad_norm[mbi++] = frob(micro, P) / (double)G;
        }
        for (uint64_t i = 0; i < P; ++i) grad[i] *= -1.0 / (double)G;
        fmo_adam_step(W, m, v, &step, grad, P, lr, b1, b2, eps);
        upd_grad_norm[u] = frob(grad, P);
        if (last_grad) memcpy(last_grad, grad, P * sizeof(double));
    }
    free(term);
    free(micro);
    free(grad);
    free(phi);
    free(p);
    return 0;
}

/* ---- few-token gradient at full V x D (column-sparse restatement) -------
 * The same arithmetic as fmo_run_agent's first update (policy.hpp:42-91,
 * training.hpp:386-395, 444-446) restricted to the feature columns the
 * samples' contexts touch: every other phi_d is 0, and adding W*0 / coef*0
 * never changes an IEEE sum that starts at +0, so the touched columns are
 * bit-identical to the dense oracle and every other column is exactly 0.
 * W's columns are drawn directly from the seeded stream (policy.hpp:29-35):
 * element i = v*D + d consumes draws 2i, 2i+1 of the splitmix sequence, whose
 * state before draw k is seed + k * golden-gamma (rng.hpp:14-19).  Memory is
 * V x (#columns) doubles instead of the dense oracle's 7 x V x D.
 * Returns the number of columns (written ascending to cols_out, at most
 * max_cols) or -1; grad_out is [V][ncols] row-major = -(1/G) sum_s A_s term_s,
 * mb_norm_out = ||sum_s A_s term_s||_F / G (training.hpp:417). */
static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : x > y;
}

int64_t fmo_sparse_grad(uint64_t V, uint64_t D, uint64_t seed, int n_samples, const uint8_t* payloads,
                        const int64_t* prompt_off, const int64_t* resp_off, const double* adv, int64_t G,
                        int64_t max_cols, int64_t* cols_out, double* grad_out, double* mb_norm_out) {
    /* columns touched by any context window */
    int64_t ncand = 0, cap = 64;
    int64_t* cand = (int64_t*)malloc(cap * sizeof(int64_t));
    for (int s = 0; s < n_samples; ++s) {
        const uint64_t np = fmo_decode_tokens(payloads + prompt_off[s], NULL);
        const uint64_t nr = fmo_decode_tokens(payloads + resp_off[s], NULL);
        int* ctx = (int*)malloc((np + nr + 1) * sizeof(int));
        fmo_decode_tokens(payloads + prompt_off[s], ctx);
        fmo_decode_tokens(payloads + resp_off[s], ctx + np);
        for (uint64_t t = 0; t < nr; ++t) {
            const int len = (int)(np + t), n = len < 4 ? len : 4;
            for (int i = len - n; i < len; ++i) {
                if (ncand == cap) cand = (int64_t*)realloc(cand, (cap *= 2) * sizeof(int64_t));
                cand[ncand++] = (int64_t)((uint64_t)(int64_t)ctx[i] % D);
            }
        }
        free(ctx);
    }
    qsort(cand, (size_t)ncand, sizeof(int64_t), cmp_i64);
    int64_t nc = 0;
    for (int64_t i = 0; i < ncand; ++i)
        if (nc == 0 || cand[i] != cand[nc - 1]) cand[nc++] = cand[i];
    if (nc > max_cols) {
        free(cand);
        return -1;
    }
    memcpy(cols_out, cand, (size_t)nc * sizeof(int64_t));
    free(cand);
    /* W[:, cols] straight from the seeded stream */
    double* Wc = (double*)malloc(V * (size_t)nc * sizeof(double));
    for (uint64_t v = 0; v < V; ++v)
        for (int64_t j = 0; j < nc; ++j) {
            uint64_t st = seed + 2ULL * (v * D + (uint64_t)cols_out[j]) * 0x9e3779b97f4a7c15ULL;
            Wc[v * nc + j] = 0.5 * rng_normal(&st);
        }
    double* phi = (double*)calloc((size_t)nc, sizeof(double));
    double* z = (double*)malloc(V * sizeof(double));
    double* term = (double*)malloc(V * (size_t)nc * sizeof(double));
    memset(grad_out, 0, V * (size_t)nc * sizeof(double));
    for (int s = 0; s < n_samples; ++s) {
        const uint64_t np = fmo_decode_tokens(payloads + prompt_off[s], NULL);
        const uint64_t nr = fmo_decode_tokens(payloads + resp_off[s], NULL);
        int* ctx = (int*)malloc((np + nr + 1) * sizeof(int));
        fmo_decode_tokens(payloads + prompt_off[s], ctx);
        fmo_decode_tokens(payloads + resp_off[s], ctx + np);
        memset(term, 0, V * (size_t)nc * sizeof(double));
        for (uint64_t t = 0; t < nr; ++t) {
            const int len = (int)(np + t), n = len < 4 ? len : 4, action = ctx[np + t];
            for (int64_t j = 0; j < nc; ++j) phi[j] = 0.0;
            if (n > 0) { /* policy.hpp:46-49: phi[tok mod D] += 1/n in context order */
                const double w = 1.0 / (double)n;
                for (int i = len - n; i < len; ++i) {
                    const int64_t f = (int64_t)((uint64_t)(int64_t)ctx[i] % D);
                    int64_t lo = 0, hi = nc - 1;
                    while (lo < hi) {
                        const int64_t mid = (lo + hi) / 2;
                        if (cols_out[mid] < f) lo = mid + 1; else hi = mid;
                    }
                    phi[lo] += w;
                }
            }
            /* policy.hpp:57-69: d-ascending sum over the non-zero features */
            for (uint64_t v = 0; v < V; ++v) {
                double acc = 0.0;
                for (int64_t j = 0; j < nc; ++j)
                    if (phi[j] != 0.0) acc += Wc[v * nc + j] * phi[j];
                z[v] = acc;
            }
            double zmax = z[0];
            for (uint64_t v = 1; v < V; ++v)
                if (z[v] > zmax) zmax = z[v];
            double denom = 0.0;
            for (uint64_t v = 0; v < V; ++v) {
                z[v] = exp(z[v] - zmax);
                denom += z[v];
            }
            for (uint64_t v = 0; v < V; ++v) z[v] /= denom;
            /* policy.hpp:83-90 */
            for (uint64_t v = 0; v < V; ++v) {
                const double coef = (((int)v == action ? 1.0 : 0.0) - z[v]);
                if (coef == 0.0) continue;
                for (int64_t j = 0; j < nc; ++j)
                    if (phi[j] != 0.0) term[v * nc + j] += coef * phi[j];
            }
        }
        for (uint64_t i = 0; i < V * (uint64_t)nc; ++i) grad_out[i] += term[i] * adv[s]; /* scale, canonical sum */
        free(ctx);
    }
    double ss = 0.0;
    for (uint64_t i = 0; i < V * (uint64_t)nc; ++i) ss += grad_out[i] * grad_out[i];
    *mb_norm_out = sqrt(ss) / (double)G;
    for (uint64_t i = 0; i < V * (uint64_t)nc; ++i) grad_out[i] *= -1.0 / (double)G;
    free(Wc);
    free(phi);
    free(z);
    free(term);
    return nc;
}


/* ---------------------------------------------------------------------------
 * Full-size gradient of one global step, multi-threaded (TEST INFRASTRUCTURE:
 * the full-size parity tests' checker).  The reference's own arithmetic —
 * training.hpp:378-395 (per-sample term over the response tokens, scaled by
 * the advantage), 417 (micro-batch grad norm), 444-446 (canonical sum, -1/G);
 * policy.hpp:42-51 (featurize), 54-70 (probabilities), 79-91 (gradient) —
 * restricted, as in fmo_sparse_grad, to the non-zero features (skipping a
 * +-0 addend never changes an IEEE sum that starts at +0), so every element
 * is bit-identical to the dense sequential oracle (fmo_run_agent's last_grad).
 * Parallel without changing any summation order:
 *   pass 1, threads over tokens: each token's softmax max and denominator
 *           (sequential over v, as policy.hpp:62-69);
 *   pass 2, threads over vocabulary blocks: every (v, d) element is owned by
 *           one thread, which walks the samples and tokens in order.
 * Wt is W transposed, [D][V] f64 (a feature's weights contiguous); gradT_out
 * is [D][V] = -(1/G) sum_s A_s term_s; mb_norm_out (nullable) gets
 * ||sum_{s in mb} A_s term_s||_F / G per micro-batch of mb samples
 * (training.hpp:417).  Returns 0, or -1 on allocation failure. */
#include <pthread.h>

typedef struct {
    uint64_t V, D;
    const double* Wt;
    int n_samples;
    const int* tok;           /* all sequences (prompt ++ response) back to back */
    const int64_t* seq_off;   /* [n_samples + 1] */
    const int64_t* prompt_n;  /* [n_samples] */
    const int64_t* row_off;   /* [n_samples + 1]: first trained row of each sample */
    const double* adv;
    int64_t G;
    int mb;
    double* zmax;   /* [rows] */
    double* denom;  /* [rows] */
    double* gradT;
    double* mbT;    /* nullable */
    double* mb_ss;  /* [threads][n_mb] */
    int n_mb;
    int threads;
} StepCtx;

typedef struct {
    StepCtx* c;
    int id;
} StepArg;

/* phi of row t of sample s: the distinct features of its context, ascending,
 * with their summed weights (policy.hpp:46-49: phi[tok mod D] += 1/n in
 * context order); returns their number */
static int row_phi(const StepCtx* c, int s, int64_t t, int64_t* f, double* w) {
    const int* seq = c->tok + c->seq_off[s];
    const int64_t len = c->prompt_n[s] + t, n = len < 4 ? len : 4;
    int nf = 0;
    if (n == 0) return 0;
    const double wt = 1.0 / (double)n;
    for (int64_t i = len - n; i < len; ++i) {
        const int64_t d = (int64_t)((uint64_t)(int64_t)seq[i] % c->D);
        int k = 0;
        while (k < nf && f[k] != d) ++k;
        if (k == nf) {
            f[nf] = d;
            w[nf] = 0.0;
            ++nf;
        }
        w[k] += wt;
    }
    for (int a = 1; a < nf; ++a) /* ascending features (the d loop of policy.hpp:57-61) */
        for (int b = a; b > 0 && f[b - 1] > f[b]; --b) {
            int64_t tf = f[b];
            f[b] = f[b - 1];
            f[b - 1] = tf;
            double tw = w[b];
            w[b] = w[b - 1];
            w[b - 1] = tw;
        }
    return nf;
}

static inline double row_logit(const StepCtx* c, uint64_t v, int nf, const int64_t* f, const double* w) {
    double acc = 0.0;
    for (int k = 0; k < nf; ++k) acc += c->Wt[(uint64_t)f[k] * c->V + v] * w[k];
    return acc;
}

static void* step_pass1(void* p) {
    StepArg* a = (StepArg*)p;
    StepCtx* c = a->c;
    const int64_t rows = c->row_off[c->n_samples];
    int s = 0;
    for (int64_t r = a->id; r < rows; r += c->threads) {
        while (c->row_off[s + 1] <= r) ++s;
        int64_t f[4];
        double w[4];
        const int nf = row_phi(c, s, r - c->row_off[s], f, w);
        double zmax = row_logit(c, 0, nf, f, w);
        for (uint64_t v = 1; v < c->V; ++v) {
            const double z = row_logit(c, v, nf, f, w);
            if (z > zmax) zmax = z;
        }
        double den = 0.0;
        for (uint64_t v = 0; v < c->V; ++v) den += exp(row_logit(c, v, nf, f, w) - zmax);
        c->zmax[r] = zmax;
        c->denom[r] = den;
    }
    return NULL;
}

static void* step_pass2(void* p) {
    StepArg* a = (StepArg*)p;
    StepCtx* c = a->c;
    const uint64_t V = c->V;
    const uint64_t v0 = V * (uint64_t)a->id / (uint64_t)c->threads, v1 = V * (uint64_t)(a->id + 1) / (uint64_t)c->threads;
    const uint64_t nb = v1 - v0;
    if (nb == 0) return NULL;
    /* the current sample's term, compacted to its touched features: [slot][nb] */
    int64_t max_rows = 0;
    for (int s = 0; s < c->n_samples; ++s)
        if (c->row_off[s + 1] - c->row_off[s] > max_rows) max_rows = c->row_off[s + 1] - c->row_off[s];
    const int64_t max_feat = 4 * max_rows + 4;
    double* term = (double*)calloc((size_t)max_feat * nb, sizeof(double));
    int64_t* feat_of_slot = (int64_t*)malloc((size_t)max_feat * sizeof(int64_t));
    double* ss = c->mb_ss + (size_t)a->id * (size_t)c->n_mb;
    for (int s = 0; s < c->n_samples; ++s) {
        const int64_t nr = c->row_off[s + 1] - c->row_off[s];
        int nslot = 0;
        for (int64_t t = 0; t < nr; ++t) {
            const int64_t r = c->row_off[s] + t;
            int64_t f[4];
            double w[4];
            const int nf = row_phi(c, s, t, f, w);
            int slot[4];
            for (int k = 0; k < nf; ++k) {
                int q = 0;
                while (q < nslot && feat_of_slot[q] != f[k]) ++q;
                if (q == nslot) {
                    feat_of_slot[nslot++] = f[k];
                    memset(term + (size_t)q * nb, 0, nb * sizeof(double));
                }
                slot[k] = q;
            }
            const int action = c->tok[c->seq_off[s] + c->prompt_n[s] + t];
            const double zmax = c->zmax[r], den = c->denom[r];
            for (uint64_t v = v0; v < v1; ++v) {
                const double pv = exp(row_logit(c, v, nf, f, w) - zmax) / den; /* policy.hpp:62-69 */
                const double coef = ((int)v == action ? 1.0 : 0.0) - pv;       /* policy.hpp:84-86 */
                if (coef == 0.0) continue;
                for (int k = 0; k < nf; ++k) term[(size_t)slot[k] * nb + (v - v0)] += coef * w[k];
            }
        }
        /* term *= A; canonical sum into the gradient and the micro-batch sum */
        const double A = c->adv[s];
        const int k_mb = s / c->mb;
        for (int q = 0; q < nslot; ++q) {
            double* g = c->gradT + (uint64_t)feat_of_slot[q] * V + v0;
            double* mbr = c->mbT ? c->mbT + (uint64_t)feat_of_slot[q] * V + v0 : NULL;
            const double* tq = term + (size_t)q * nb;
            for (uint64_t i = 0; i < nb; ++i) {
                const double x = tq[i] * A;
                g[i] += x;
                if (mbr) mbr[i] += x;
            }
        }
        if (c->mbT && (s % c->mb == c->mb - 1 || s == c->n_samples - 1)) {
            /* micro-batch done: its sum of squares over this block, then reset */
            double acc = 0.0;
            for (uint64_t d = 0; d < c->D; ++d) {
                double* mbr = c->mbT + d * V + v0;
                for (uint64_t i = 0; i < nb; ++i) {
                    acc += mbr[i] * mbr[i];
                    mbr[i] = 0.0;
                }
            }
            ss[k_mb] = acc;
        }
    }
    free(term);
    free(feat_of_slot);
    return NULL;
}

int fmo_step_grad(uint64_t V, uint64_t D, const double* Wt, int n_samples, const uint8_t* payloads,
                  const int64_t* prompt_off, const int64_t* resp_off, const double* adv, int64_t G, int mb,
                  int threads, double* gradT_out, double* mb_norm_out) {
    if (threads < 1) threads = 1;
    StepCtx c;
    memset(&c, 0, sizeof(c));
    c.V = V;
    c.D = D;
    c.Wt = Wt;
    c.n_samples = n_samples;
    c.adv = adv;
    c.G = G;
    c.mb = mb > 0 ? mb : n_samples;
    c.threads = threads;
    int64_t* seq_off = (int64_t*)malloc((size_t)(n_samples + 1) * sizeof(int64_t));
    int64_t* pn = (int64_t*)malloc((size_t)(n_samples + 1) * sizeof(int64_t));
    int64_t* row_off = (int64_t*)malloc((size_t)(n_samples + 1) * sizeof(int64_t));
    seq_off[0] = 0;
    row_off[0] = 0;
    for (int s = 0; s < n_samples; ++s) {
        const uint64_t np = fmo_decode_tokens(payloads + prompt_off[s], NULL);
        const uint64_t nr = fmo_decode_tokens(payloads + resp_off[s], NULL);
        pn[s] = (int64_t)np;
        seq_off[s + 1] = seq_off[s] + (int64_t)(np + nr);
        row_off[s + 1] = row_off[s] + (int64_t)nr;
    }
    int* tok = (int*)malloc((size_t)(seq_off[n_samples] + 1) * sizeof(int));
    for (int s = 0; s < n_samples; ++s) {
        fmo_decode_tokens(payloads + prompt_off[s], tok + seq_off[s]);
        fmo_decode_tokens(payloads + resp_off[s], tok + seq_off[s] + pn[s]);
    }
    const int64_t rows = row_off[n_samples];
    c.tok = tok;
    c.seq_off = seq_off;
    c.prompt_n = pn;
    c.row_off = row_off;
    c.zmax = (double*)malloc((size_t)(rows + 1) * sizeof(double));
    c.denom = (double*)malloc((size_t)(rows + 1) * sizeof(double));
    c.n_mb = (n_samples + c.mb - 1) / c.mb;
    c.mb_ss = (double*)calloc((size_t)threads * (size_t)(c.n_mb + 1), sizeof(double));
    c.gradT = gradT_out;
    memset(gradT_out, 0, V * D * sizeof(double));
    c.mbT = mb_norm_out ? (double*)calloc(V * D, sizeof(double)) : NULL;
    int rc = 0;
    if (!c.zmax || !c.denom || !c.mb_ss || (mb_norm_out && !c.mbT)) rc = -1;
    pthread_t* th = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
    StepArg* args = (StepArg*)malloc((size_t)threads * sizeof(StepArg));
    if (rc == 0) {
        for (int i = 0; i < threads; ++i) {
            args[i].c = &c;
            args[i].id = i;
            pthread_create(&th[i], NULL, step_pass1, &args[i]);
        }
        for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
        for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, step_pass2, &args[i]);
        for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
        for (uint64_t i = 0; i < V * D; ++i) gradT_out[i] *= -1.0 / (double)G; /* training.hpp:446 */
        if (mb_norm_out)
            for (int k = 0; k < c.n_mb; ++k) {
                double acc = 0.0;
                for (int i = 0; i < threads; ++i) acc += c.mb_ss[(size_t)i * (size_t)c.n_mb + k];
                mb_norm_out[k] = sqrt(acc) / (double)G;
            }
    }
    free(th);
    free(args);
    free(c.mbT);
    free(c.mb_ss);
    free(c.zmax);
    free(c.denom);
    free(tok);
    free(seq_off);
    free(pn);
    free(row_off);
    return rc;
}

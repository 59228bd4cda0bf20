// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference sources (/root/reference/proj/src,
// compiled in place by oracle/Makefile into oracle/_ref/libexitlab_ref.so).
// It lets the Python tests and bench.py's reference arm drive the reference's
// own Engine::run, KvStore, ExitStatusVector, decide(), reference_decode and
// replay_sequence, and flattens their results into the same field layout the
// C port (exitlab_oracle.h) and the product (include/exitlab_b200.h) expose.
//
// Nothing here re-implements reference math, except ref_session_step, which
// restates the decode_iteration body (engine.cpp:208-310) over the reference's
// public functions so that the iteration can start from a seeded KV prefix
// (the bench workload); the same restatement technique the survey's
// probe_time used.
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "exitlab/engine.hpp"
#include "exitlab/exit_policy.hpp"
#include "exitlab/kv_cache.hpp"
#include "exitlab/metrics.hpp"
#include "exitlab/model.hpp"
#include "exitlab/numerics.hpp"
#include "exitlab/oracle.hpp"
#include "exitlab/workload.hpp"

extern "C" {
#include "exitlab_oracle.h"  // eo_engine_config / eo_gen_params layouts + codes
}

using namespace exitlab;

namespace {
thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const KvOutOfMemory*>(&e)) return EO_KV_OUT_OF_MEMORY;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return EO_INVALID_ARGUMENT;
    if (dynamic_cast<const std::logic_error*>(&e)) return EO_LOGIC_ERROR;
    return EO_RUNTIME_ERROR;
}

#define GUARD_BEGIN try {
#define GUARD_END(fail)                 \
    }                                   \
    catch (const std::exception& e) {   \
        g_err = e.what();               \
        return fail(code_of(e));        \
    }
inline int ret_code(int c) { return c; }
inline int ret_neg(int c) { return -c; }

double round_bf16(double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    const uint64_t lsb = (b >> 45) & 1u;
    b += 0x0FFFFFFFFFFFULL + lsb;
    b &= ~((1ULL << 45) - 1);
    double y;
    std::memcpy(&y, &b, 8);
    return y;
}
void round_all(std::vector<double>& v) {
    for (double& x : v) x = round_bf16(x);
}

ExitTechnique technique_of(const eo_engine_config& c) {
    switch (c.technique) {
        case EO_TECH_SOFTMAX: return ExitTechnique::softmax_response();
        case EO_TECH_STATE: return ExitTechnique::state_similarity();
        case EO_TECH_CLASSIFIER: return ExitTechnique::classifier();
        case EO_TECH_NEVER: return ExitTechnique::never();
        case EO_TECH_ALWAYS_AT: return ExitTechnique::always_at(c.exit_layer);
    }
    throw std::invalid_argument("reference has no technique kind " + std::to_string(c.technique));
}

EngineConfig engine_config_of(const eo_engine_config& c) {
    EngineConfig e;
    e.model = ModelConfig{c.n_layers, c.d_model, c.vocab_size, c.model_seed};
    e.technique = technique_of(c);
    e.schedule = ThresholdSchedule{c.lambda0, c.gamma, c.lambda_min};
    e.costs = CostModel{c.c_layer_fixed, c.c_layer_per_seq, c.c_fill_per_seq_layer,
                        c.c_check_softmax, c.c_check_classifier, c.c_check_state};
    e.max_batch = c.max_batch;
    e.pool_blocks = c.pool_blocks;
    e.block_capacity = c.block_capacity;
    e.eos_token = c.eos_token;
    e.capture_kv = c.capture_kv != 0;
    return e;
}

Workload workload_of(int n, const double* arrival, const int32_t* off, const int32_t* prompt,
                     const int32_t* max_new) {
    Workload w;
    for (int i = 0; i < n; ++i) {
        Request r;
        r.arrival_time = arrival[i];
        r.prompt.assign(prompt + off[i], prompt + off[i + 1]);
        r.max_new_tokens = max_new[i];
        w.requests.push_back(std::move(r));
    }
    return w;
}

uint64_t kv_prefix_seed(uint64_t kv_seed, int L, int seq, int layer, int pos, int kind) {
    const uint64_t tag =
        ((((uint64_t)seq * (uint64_t)L + (uint64_t)(layer - 1)) << 21) | (uint64_t)pos) << 1 |
        (uint64_t)kind;
    return splitmix64_at(kv_seed, tag);
}

struct FlatTranscript {
    std::vector<int32_t> pf_seq, pf_positions, it_output_layer, it_batch_off, ps_seq, ps_accept,
        ps_token, sq_id, sq_max_new, sq_prompt_off, sq_prompt, sq_tok_off, sq_tokens,
        sq_exit_layers, sq_iter_out;
    std::vector<double> pf_clock, pf_charge, it_clock, it_charge, sq_arrival, sq_first, sq_finish,
        meta, it_conf;
    Transcript t;

    std::vector<int32_t>* i32(const char* f) {
#define F(n) if (!std::strcmp(f, #n)) return &n;
        F(pf_seq) F(pf_positions) F(it_output_layer) F(it_batch_off) F(ps_seq) F(ps_accept)
        F(ps_token) F(sq_id) F(sq_max_new) F(sq_prompt_off) F(sq_prompt) F(sq_tok_off)
        F(sq_tokens) F(sq_exit_layers) F(sq_iter_out)
#undef F
        return nullptr;
    }
    std::vector<double>* f64(const char* f) {
#define F(n) if (!std::strcmp(f, #n)) return &n;
        F(pf_clock) F(pf_charge) F(it_clock) F(it_charge) F(sq_arrival) F(sq_first) F(sq_finish)
        F(meta) F(it_conf)
#undef F
        return nullptr;
    }
};

FlatTranscript* flatten(Transcript&& t) {
    auto* f = new FlatTranscript;
    for (const auto& p : t.prefills) {
        f->pf_clock.push_back(p.clock);
        f->pf_charge.push_back(p.charge);
        f->pf_seq.push_back(p.seq_id);
        f->pf_positions.push_back(p.positions);
    }
    f->it_batch_off.push_back(0);
    for (const auto& it : t.iterations) {
        f->it_clock.push_back(it.clock);
        f->it_charge.push_back(it.charge);
        f->it_output_layer.push_back(it.output_layer);
        for (const auto& s : it.per_seq) {
            f->ps_seq.push_back(s.seq_id);
            f->ps_accept.push_back(s.accept_layer);
            f->ps_token.push_back(s.token);
        }
        f->it_batch_off.push_back((int32_t)f->ps_seq.size());
    }
    f->sq_prompt_off.push_back(0);
    f->sq_tok_off.push_back(0);
    for (const auto& s : t.sequences) {
        f->sq_id.push_back(s.id);
        f->sq_arrival.push_back(s.arrival_time);
        f->sq_first.push_back(s.first_token_time);
        f->sq_finish.push_back(s.finish_time);
        f->sq_max_new.push_back(s.max_new_tokens);
        for (int x : s.prompt) f->sq_prompt.push_back(x);
        f->sq_prompt_off.push_back((int32_t)f->sq_prompt.size());
        for (size_t i = 0; i < s.tokens.size(); ++i) {
            f->sq_tokens.push_back(s.tokens[i]);
            f->sq_exit_layers.push_back(s.exit_layers[i]);
            f->sq_iter_out.push_back(s.iter_output_layers[i]);
        }
        f->sq_tok_off.push_back((int32_t)f->sq_tokens.size());
    }
    f->meta = {t.final_clock, t.total_idle, (double)t.cache_stats.pool_blocks,
               (double)t.cache_stats.free_blocks, (double)t.cache_stats.peak_blocks_in_use};
    f->t = std::move(t);
    return f;
}

struct Session {
    const ModelWeights* w;
    eo_engine_config cfg;
    EngineConfig ec;
    std::unique_ptr<KvStore> cache;
    std::vector<int> ids, next_input;
    // layer-stepped iteration state (ref_session_iter_*)
    std::vector<std::pair<int, Vector>> states;
    std::unique_ptr<ExitStatusVector> status;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_model_seeded(int L, int d, int V, uint64_t seed, int rb) {
    try {
        auto* w = new ModelWeights(ModelWeights::seeded(ModelConfig{L, d, V, seed}));
        if (rb) {
            round_all(w->embedding.values);
            round_all(w->lm_head.values);
            round_all(w->probe.w);
            w->probe.b = round_bf16(w->probe.b);
            for (auto& lw : w->layers) {
                for (Matrix* m : {&lw.w_q, &lw.w_k, &lw.w_v, &lw.w_o, &lw.w_up, &lw.w_down})
                    round_all(m->values);
            }
        }
        return w;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_model_free(void* m) { delete static_cast<ModelWeights*>(m); }

int ref_model_tensor(const void* mp, int which, int layer, double* out, int64_t cap) {
    GUARD_BEGIN
    const auto* m = static_cast<const ModelWeights*>(mp);
    const std::vector<double>* src = nullptr;
    double pb = m->probe.b;
    std::vector<double> one{pb};
    if (which == 0) src = &m->embedding.values;
    else if (which == 1) src = &m->lm_head.values;
    else if (which == 2) src = &m->probe.w;
    else if (which == 3) src = &one;
    else {
        const LayerWeights& lw = m->layers.at((size_t)(layer - 1));
        const Matrix* ms[] = {&lw.w_q, &lw.w_k, &lw.w_v, &lw.w_o, &lw.w_up, &lw.w_down};
        src = &ms[which - 4]->values;
    }
    if ((int64_t)src->size() > cap) throw std::invalid_argument("buffer too small");
    std::memcpy(out, src->data(), sizeof(double) * src->size());
    return EO_OK;
    GUARD_END(ret_code)
}

int64_t ref_gen_workload(const eo_gen_params* p, double* arrival, int32_t* off, int32_t* prompt,
                         int32_t* max_new) {
    try {
        GenParams g;
        g.n_requests = p->n_requests;
        g.mean_interarrival = p->mean_interarrival;
        g.prompt_len_min = p->prompt_len_min;
        g.prompt_len_max = p->prompt_len_max;
        g.output_len_min = p->output_len_min;
        g.output_len_max = p->output_len_max;
        g.seed = p->seed;
        g.vocab_size = p->vocab_size;
        g.eos_token = p->eos_token;
        const Workload w = gen_workload(g);
        int64_t total = 0;
        if (off) off[0] = 0;
        for (size_t i = 0; i < w.requests.size(); ++i) {
            const Request& r = w.requests[i];
            if (arrival) arrival[i] = r.arrival_time;
            for (size_t j = 0; j < r.prompt.size(); ++j)
                if (prompt) prompt[total + (int64_t)j] = r.prompt[j];
            total += (int64_t)r.prompt.size();
            if (off) off[i + 1] = (int32_t)total;
            if (max_new) max_new[i] = r.max_new_tokens;
        }
        return total;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Engine::run of the reference itself (real prefill; engine.cpp:110-330)
int ref_engine_run(const void* mp, const eo_engine_config* c, int n, const double* arrival,
                   const int32_t* off, const int32_t* prompt, const int32_t* max_new,
                   void** out) {
    GUARD_BEGIN
    if (c->synthetic_kv_seed >= 0)
        throw std::invalid_argument("reference Engine::run has no synthetic KV prefix");
    const auto* m = static_cast<const ModelWeights*>(mp);
    const Engine engine(engine_config_of(*c), *m);
    *out = flatten(engine.run(workload_of(n, arrival, off, prompt, max_new)));
    return EO_OK;
    GUARD_END(ret_code)
}

void ref_transcript_free(void* t) { delete static_cast<FlatTranscript*>(t); }
// the reference's own transcript persistence (engine.cpp:336-393), for byte comparisons
int ref_transcript_write_jsonl(void* tp, const char* path) {
    GUARD_BEGIN
    write_transcript_jsonl(static_cast<FlatTranscript*>(tp)->t, path);
    return EO_OK;
    GUARD_END(ret_code)
}

// compute_metrics + write_report (metrics.cpp:13-58, 178-195) of a reference transcript;
// wall_clock_info_s (a host wall-clock reading) is set to `wall` so reports compare byte for byte
int ref_transcript_write_report(void* tp, const char* path, const char* format, double wall) {
    GUARD_BEGIN
    MetricsReport r = compute_metrics(static_cast<FlatTranscript*>(tp)->t);
    r.wall_clock_info_s = wall;
    write_report(r, path, format);
    return EO_OK;
    GUARD_END(ret_code)
}

int64_t ref_transcript_len(void* tp, const char* f) {
    auto* t = static_cast<FlatTranscript*>(tp);
    if (auto* a = t->i32(f)) return (int64_t)a->size();
    if (auto* b = t->f64(f)) return (int64_t)b->size();
    return -1;
}
int ref_transcript_get_i32(void* tp, const char* f, int32_t* out) {
    auto* a = static_cast<FlatTranscript*>(tp)->i32(f);
    if (!a) return EO_INVALID_ARGUMENT;
    if (!a->empty()) std::memcpy(out, a->data(), sizeof(int32_t) * a->size());
    return EO_OK;
}
int ref_transcript_get_f64(void* tp, const char* f, double* out) {
    auto* a = static_cast<FlatTranscript*>(tp)->f64(f);
    if (!a) return EO_INVALID_ARGUMENT;
    if (!a->empty()) std::memcpy(out, a->data(), sizeof(double) * a->size());
    return EO_OK;
}
int ref_transcript_kv(void* tp, int seq, int layer, double* k, double* v, int64_t cap) {
    GUARD_BEGIN
    auto* t = static_cast<FlatTranscript*>(tp);
    const SequenceKvCapture& c = t->t.kv_captures.at(seq);
    const auto& per = c.kv.at((size_t)(layer - 1));
    const size_t d = per.empty() ? 0 : per[0].k.size();
    if ((int64_t)(per.size() * d) > cap) throw std::invalid_argument("buffer too small");
    for (size_t p = 0; p < per.size(); ++p) {
        std::memcpy(k + p * d, per[p].k.data(), sizeof(double) * d);
        std::memcpy(v + p * d, per[p].v.data(), sizeof(double) * d);
    }
    return (int)per.size();
    GUARD_END(ret_neg)
}
int ref_transcript_exit_states(void* tp, int seq, double* out, int64_t cap) {
    GUARD_BEGIN
    auto* t = static_cast<FlatTranscript*>(tp);
    const SequenceKvCapture& c = t->t.kv_captures.at(seq);
    size_t n = 0;
    for (const Vector& h : c.exit_states) {
        if ((int64_t)(n + h.size()) > cap) throw std::invalid_argument("buffer too small");
        std::memcpy(out + n, h.data(), sizeof(double) * h.size());
        n += h.size();
    }
    return (int)c.exit_states.size();
    GUARD_END(ret_neg)
}

double ref_softmax_response_confidence(const double* x, int n) {
    try { return softmax_response_confidence(Vector(x, x + n)); } catch (...) { return NAN; }
}
double ref_state_similarity_confidence(const double* a, const double* b, int n) {
    try { return state_similarity_confidence(Vector(a, a + n), Vector(b, b + n)); } catch (...) { return NAN; }
}
double ref_classifier_confidence(const double* h, const double* w, double b, int n) {
    try {
        ClassifierProbe p{Vector(w, w + n), b};
        return classifier_confidence(Vector(h, h + n), p);
    } catch (...) { return NAN; }
}
double ref_threshold_at(double l0, double g, double lmin, int layer) {
    return threshold_at(ThresholdSchedule{l0, g, lmin}, layer);
}
int ref_greedy_token(const double* x, int n) { return greedy_token(Vector(x, x + n)); }

// ExitStatusVector (engine.cpp:47-75) driven by conf[L][B] > lambda via decide()
// semantics (strict '>', exit_policy.cpp:89-115).
int ref_status_trace(int B, int L, const double* conf, const double* lambdas, int32_t* first) {
    try {
        ExitStatusVector st(B);
        int out = L;
        for (int layer = 1; layer <= L; ++layer) {
            std::vector<bool> acc((size_t)B);
            for (int b = 0; b < B; ++b) acc[(size_t)b] = conf[(size_t)(layer - 1) * B + b] > lambdas[layer - 1];
            if (st.observe_layer(layer, acc)) { out = layer; break; }
        }
        for (int b = 0; b < B; ++b) first[b] = st.first_accept_layer(b, L);
        return out;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

// Working version: block ids are recovered by writing every reserved slot of
// every live sequence right after its allocation (positions 0..capacity-1 at
// every layer, contiguous as the store requires) and reading the span
// addresses back. The store's data buffer base is found as the minimum slot
// address over a final full scan, which is block 0 when block 0 was ever
// handed out; tests make sure it is (the very first allocation pops block 0).
int ref_kv_block_trace(int L, int pool, int cap, int n_ops, const int32_t* ops, const int32_t* caps,
                        int n_ids, int bpl_max, int32_t* tables) {
    try {
        KvStore st(1, L, pool, cap);
        for (int64_t i = 0; i < (int64_t)n_ids * L * bpl_max; ++i) tables[i] = -1;
        std::vector<std::vector<const double*>> addr((size_t)n_ids);
        const double* base = nullptr;
        for (int i = 0; i < n_ops; ++i) {
            if (ops[i] > 0) {
                const int id = ops[i] - 1;
                try { st.allocate(id, caps[i]); } catch (const KvOutOfMemory&) { continue; }
                const int bpl = (caps[i] + cap - 1) / cap;
                const int n = bpl * cap;
                auto& a = addr[(size_t)id];
                a.assign((size_t)L * bpl, nullptr);
                for (int l = 1; l <= L; ++l) {
                    for (int p = 0; p < n; ++p) st.append(id, l, p, Vector{0.0}, Vector{0.0});
                    const KvView v = st.view(id, l, n);
                    for (int b = 0; b < bpl; ++b) {
                        const double* ptr = v.key(b * cap).data();
                        a[(size_t)(l - 1) * bpl + b] = ptr;
                        if (!base || ptr < base) base = ptr;
                    }
                }
            } else if (ops[i] < 0) {
                st.release(-ops[i] - 1);
            }
        }
        for (int id = 0; id < n_ids; ++id) {
            const auto& a = addr[(size_t)id];
            if (a.empty()) continue;
            const int bpl = (int)(a.size() / (size_t)L);
            for (int l = 0; l < L; ++l)
                for (int b = 0; b < bpl && b < bpl_max; ++b)
                    tables[((size_t)id * L + l) * bpl_max + b] =
                        (int32_t)((a[(size_t)l * bpl + b] - base) / cap);
        }
        return st.free_blocks();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

int ref_reference_decode(const void* mp, const int32_t* prompt, int plen, int max_new, int eos,
                         int32_t* out) {
    try {
        const auto* m = static_cast<const ModelWeights*>(mp);
        const auto toks = reference_decode(*m, std::vector<int>(prompt, prompt + plen), max_new, eos);
        for (size_t i = 0; i < toks.size(); ++i) out[i] = toks[i];
        return (int)toks.size();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

int ref_replay_sequence(const void* mp, const int32_t* prompt, int plen, const int32_t* exits, int n,
                        int32_t* tokens, double* exit_states, double* kv_k, double* kv_v) {
    GUARD_BEGIN
    const auto* m = static_cast<const ModelWeights*>(mp);
    const int d = m->config.d_model, L = m->config.n_layers;
    const SequenceReplay r = replay_sequence(*m, std::vector<int>(prompt, prompt + plen),
                                             std::vector<int>(exits, exits + n));
    for (int t = 0; t < n; ++t) {
        tokens[t] = r.tokens[(size_t)t];
        if (exit_states) std::memcpy(exit_states + (size_t)t * d, r.exit_states[(size_t)t].data(), sizeof(double) * (size_t)d);
    }
    const size_t P = (size_t)(plen - 1 + n);
    if (kv_k && kv_v)
        for (int l = 0; l < L; ++l)
            for (size_t p = 0; p < P; ++p) {
                std::memcpy(kv_k + ((size_t)l * P + p) * d, r.kv[(size_t)l][p].k.data(), sizeof(double) * (size_t)d);
                std::memcpy(kv_v + ((size_t)l * P + p) * d, r.kv[(size_t)l][p].v.data(), sizeof(double) * (size_t)d);
            }
    return EO_OK;
    GUARD_END(ret_code)
}

// ---- decode session over a seeded KV prefix (bench reference arm) ----
void* ref_session_create(const void* mp, const eo_engine_config* c, int B, const int32_t* first,
                         int prefix_len, int capacity, uint64_t kv_seed, const int32_t* ids) {
    try {
        auto* s = new Session;
        s->w = static_cast<const ModelWeights*>(mp);
        s->cfg = *c;
        s->ec = engine_config_of(*c);
        s->ec.validate();
        const int L = c->n_layers, d = c->d_model;
        const int bpl = (capacity + c->block_capacity - 1) / c->block_capacity;
        const int pool = std::max(c->pool_blocks, bpl * L * B);
        s->cache = std::make_unique<KvStore>(d, L, pool, c->block_capacity);
        for (int b = 0; b < B; ++b) {
            s->ids.push_back(ids[b]);
            s->next_input.push_back(first[b]);
            s->cache->allocate(ids[b], capacity);
            for (int p = 0; p < prefix_len; ++p) {
                for (int l = 1; l <= L; ++l) {
                    Vector k = seeded_vector(d, kv_prefix_seed(kv_seed, L, ids[b], l, p, 0));
                    Vector v = seeded_vector(d, kv_prefix_seed(kv_seed, L, ids[b], l, p, 1));
                    if (c->round_bf16) { round_all(k); round_all(v); }
                    s->cache->append(ids[b], l, p, k, v);
                }
                s->cache->commit(ids[b]);
            }
        }
        return s;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_session_free(void* s) { delete static_cast<Session*>(s); }

// decode_iteration (engine.cpp:208-310) restated over the reference's public
// functions; forced>0 ends the layer loop at that layer (replay of a recorded
// output layer), otherwise the status vector decides.
int ref_session_step(void* sp, int forced, const int32_t* tokens_in, int32_t* tokens, int32_t* accept,
                     double* conf, double* h_exit) {
    try {
        auto* s = static_cast<Session*>(sp);
        if (tokens_in)
            for (size_t b = 0; b < s->ids.size(); ++b) s->next_input[b] = tokens_in[b];
        const ModelWeights& w = *s->w;
        const int L = s->cfg.n_layers, d = s->cfg.d_model, B = (int)s->ids.size();
        const ExitTechnique& technique = s->ec.technique;
        std::vector<std::pair<int, Vector>> states;
        for (int b = 0; b < B; ++b) states.emplace_back(s->ids[(size_t)b], embed(w, s->next_input[(size_t)b]));
        if (conf) for (int i = 0; i < L * B; ++i) conf[i] = NAN;
        ExitStatusVector status(B);
        int output_layer = L;
        for (int layer = 1; layer <= L; ++layer) {
            std::vector<Vector> next = layer_forward(w, layer, states, *s->cache);
            std::vector<bool> accepted((size_t)B, false);
            const double lambda = threshold_at(s->ec.schedule, layer);
            for (int b = 0; b < B; ++b) {
                ExitEvidence ev;
                ev.layer = layer;
                Vector logits;
                double cf = NAN;
                switch (technique.kind) {
                    case TechniqueKind::softmax_response:
                        logits = lm_head_logits(w, next[(size_t)b]);
                        ev.logits = &logits;
                        cf = softmax_response_confidence(logits);
                        break;
                    case TechniqueKind::state_similarity:
                        ev.h_prev = &states[(size_t)b].second;
                        ev.h_cur = &next[(size_t)b];
                        cf = state_similarity_confidence(states[(size_t)b].second, next[(size_t)b]);
                        break;
                    case TechniqueKind::classifier:
                        ev.h_cur = &next[(size_t)b];
                        ev.probe = &w.probe;
                        cf = classifier_confidence(next[(size_t)b], w.probe);
                        break;
                    default: break;
                }
                if (conf) conf[(size_t)(layer - 1) * B + b] = cf;
                accepted[(size_t)b] = decide(technique, ev, lambda);
            }
            for (int b = 0; b < B; ++b) states[(size_t)b].second = std::move(next[(size_t)b]);
            const bool all = status.observe_layer(layer, accepted);
            if (forced > 0 ? layer == forced : all) { output_layer = layer; break; }
        }
        const KvPairFn kv_fn = [&w](int layer, const Vector& h) { return compute_kv_pair(w, layer, h); };
        fill_skipped(*s->cache, states, output_layer, kv_fn);
        for (int b = 0; b < B; ++b) s->cache->commit(s->ids[(size_t)b]);
        for (int b = 0; b < B; ++b) {
            const int tok = greedy_token(lm_head_logits(w, states[(size_t)b].second));
            if (tokens) tokens[b] = tok;
            if (accept) accept[b] = status.first_accept_layer(b, L);
            if (h_exit) std::memcpy(h_exit + (size_t)b * d, states[(size_t)b].second.data(), sizeof(double) * (size_t)d);
            s->next_input[(size_t)b] = tok;
        }
        return output_layer;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -code_of(e);
    }
}


// ---- the same decode_iteration, stepped one layer at a time, so a batch sharded over several
//      processes keeps the reference's batch-wide barrier: each shard reports whether all of
//      ITS sequences are accepted after `layer` (ExitStatusVector::observe_layer, engine.cpp:55-66);
//      the coordinator ends the iteration at the first layer where every shard is all-set
//      (the AND over shards is all_set() of the whole batch) and calls finish with it ----
int ref_session_iter_begin(void* sp, const int32_t* tokens_in) {
    GUARD_BEGIN
    auto* s = static_cast<Session*>(sp);
    if (tokens_in)
        for (size_t b = 0; b < s->ids.size(); ++b) s->next_input[b] = tokens_in[b];
    s->states.clear();
    for (size_t b = 0; b < s->ids.size(); ++b) s->states.emplace_back(s->ids[b], embed(*s->w, s->next_input[b]));
    s->status = std::make_unique<ExitStatusVector>((int)s->ids.size());
    return EO_OK;
    GUARD_END(ret_code)
}
// returns 1 when every sequence of this shard has accepted at some layer <= `layer`, 0 if not, <0 on error
int ref_session_iter_layer(void* sp, int layer) {
    try {
        auto* s = static_cast<Session*>(sp);
        const ModelWeights& w = *s->w;
        const int B = (int)s->ids.size();
        const ExitTechnique& technique = s->ec.technique;
        std::vector<Vector> next = layer_forward(w, layer, s->states, *s->cache);
        std::vector<bool> accepted((size_t)B, false);
        const double lambda = threshold_at(s->ec.schedule, layer);
        for (int b = 0; b < B; ++b) {
            ExitEvidence ev;
            ev.layer = layer;
            Vector logits;
            switch (technique.kind) {
                case TechniqueKind::softmax_response:
                    logits = lm_head_logits(w, next[(size_t)b]);
                    ev.logits = &logits;
                    break;
                case TechniqueKind::state_similarity:
                    ev.h_prev = &s->states[(size_t)b].second;
                    ev.h_cur = &next[(size_t)b];
                    break;
                case TechniqueKind::classifier:
                    ev.h_cur = &next[(size_t)b];
                    ev.probe = &w.probe;
                    break;
                default: break;
            }
            accepted[(size_t)b] = decide(technique, ev, lambda);
        }
        for (int b = 0; b < B; ++b) s->states[(size_t)b].second = std::move(next[(size_t)b]);
        return s->status->observe_layer(layer, accepted) ? 1 : 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -code_of(e);
    }
}
int ref_session_iter_finish(void* sp, int output_layer, int32_t* tokens, int32_t* accept) {
    GUARD_BEGIN
    auto* s = static_cast<Session*>(sp);
    const ModelWeights& w = *s->w;
    const int L = s->cfg.n_layers, B = (int)s->ids.size();
    const KvPairFn kv_fn = [&w](int layer, const Vector& h) { return compute_kv_pair(w, layer, h); };
    fill_skipped(*s->cache, s->states, output_layer, kv_fn);
    for (int b = 0; b < B; ++b) s->cache->commit(s->ids[(size_t)b]);
    for (int b = 0; b < B; ++b) {
        const int tok = greedy_token(lm_head_logits(w, s->states[(size_t)b].second));
        if (tokens) tokens[b] = tok;
        if (accept) accept[b] = s->status->first_accept_layer(b, L);
        s->next_input[(size_t)b] = tok;
    }
    return EO_OK;
    GUARD_END(ret_code)
}

int ref_session_kv(void* sp, int row, int layer, int pos, double* k, double* v) {
    GUARD_BEGIN
    auto* s = static_cast<Session*>(sp);
    const KvView view = s->cache->view(s->ids.at((size_t)row), layer, pos + 1);
    const auto kk = view.key(pos);
    const auto vv = view.value(pos);
    std::memcpy(k, kk.data(), sizeof(double) * kk.size());
    std::memcpy(v, vv.data(), sizeof(double) * vv.size());
    return EO_OK;
    GUARD_END(ret_code)
}

}  // extern "C"

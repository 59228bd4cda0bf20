/*
 * exitlab_oracle.c -- TEST INFRASTRUCTURE ONLY (see exitlab_oracle.h).
 *
 * Plain-C fp64 restatement of the reference's early-exit decode path. Loops
 * follow the reference's accumulation order exactly; build with
 * -ffp-contract=off so results are bit-identical to the reference compiled from
 * /root/reference (oracle/_ref).  Citations are to /root/reference/proj.
 */
#include "exitlab_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
static void set_err(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}
const char* eo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ */
/* numerics.cpp:94-143                                                  */
/* ------------------------------------------------------------------ */
#define K_GAMMA 0x9E3779B97F4A7C15ULL
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t eo_splitmix64_at(uint64_t seed, uint64_t index) { return mix64(seed + (index + 1) * K_GAMMA); }
double eo_uniform01_at(uint64_t seed, uint64_t index) {
    return (double)(eo_splitmix64_at(seed, index) >> 11) * 0x1.0p-53;
}
typedef struct { uint64_t state; } rng_t;
static uint64_t rng_next(rng_t* r) { r->state += K_GAMMA; return mix64(r->state); }
static double rng_next_double(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

void eo_seeded_matrix(int rows, int cols, uint64_t seed, double* out) {
    const double s = 1.0 / sqrt((double)cols);
    const size_t n = (size_t)rows * cols;
    for (size_t i = 0; i < n; ++i) out[i] = (2.0 * eo_uniform01_at(seed, i) - 1.0) * s;
}
void eo_seeded_vector(int len, uint64_t seed, double* out) { eo_seeded_matrix(1, len, seed, out); }

/* Round-to-nearest-even of an fp64 value to bf16 precision (8-bit exponent,
 * 7-bit mantissa), done directly on the fp64 bits (no double rounding through
 * fp32).  Identical code runs on the device (csrc/el_common.cuh). */
double eo_round_bf16(double x) {
    uint64_t b;
    memcpy(&b, &x, 8);
    const uint64_t lsb = (b >> 45) & 1u;
    b += 0x0FFFFFFFFFFFULL + lsb; /* (1<<44)-1 + lsb */
    b &= ~((1ULL << 45) - 1);
    double y;
    memcpy(&y, &b, 8);
    return y;
}
uint16_t eo_bf16_bits(double x) {
    const float f = (float)eo_round_bf16(x); /* exact */
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)(u >> 16);
}

/* ------------------------------------------------------------------ */
/* model.cpp:37-59  seeded weights with per-tensor SplitMix64 tags      */
/* ------------------------------------------------------------------ */
struct eo_model {
    int L, d, V;
    uint64_t seed;
    double* emb;   /* V x d */
    double* lm;    /* V x d */
    double* pw;    /* d */
    double pb;
    double** w;    /* per layer: q,k,v,o (d x d), up (4d x d), down (d x 4d) */
    /* T5 mode (north_star (1); NOT in the reference): cross-attention
       over synthetic encoder states, enc_len > 0.  Parity of this mode is pinned only
       by this restatement (the compiled reference has no encoder/cross-attention). */
    int enc_len;
    int round_bf16;
    uint64_t enc_seed;
    double** wc;   /* per layer: q_c, k_c, v_c, o_c (d x d) */
    /* extension (not in the reference): self- and, in T5 mode, cross-attention split into n_heads
       heads of d / n_heads features, each with its own softmax and scale 1 / sqrt(d / n_heads);
       1 = the reference's single head.  Sessions with heads use the layer_forward restatement. */
    int n_heads;
    /* T5 encoder stack (extension): enc_layers > 0 replaces the seeded encoder states by the
       output of enc_layers bidirectional norm-free blocks (the decoder block without the causal
       mask) over the embeddings of seeded encoder input ids; outputs cached per sequence id */
    int enc_layers;
    double** we;   /* per encoder layer: q, k, v, o (d x d), up (4d x d), down (d x 4d) */
    int n_enc_cache, cap_enc_cache;
    int* enc_cache_id;
    double** enc_cache;  /* [T][d] per cached sequence */
};
static const int kLayerTensors = 6;

static double* layer_tensor(const eo_model* m, int layer, int k) { return m->w[(layer - 1) * kLayerTensors + k]; }
static void tensor_shape(const eo_model* m, int k, int* r, int* c) {
    const int d = m->d;
    if (k < 4) { *r = d; *c = d; }
    else if (k == 4) { *r = 4 * d; *c = d; }
    else { *r = d; *c = 4 * d; }
}
static void round_all(double* p, size_t n) { for (size_t i = 0; i < n; ++i) p[i] = eo_round_bf16(p[i]); }

eo_model* eo_model_seeded(int L, int d, int V, uint64_t seed, int round_bf16) {
    return eo_model_seeded_t5(L, d, V, seed, round_bf16, 0);
}

/* T5 mode extension (no reference counterpart): cross weights seeded with tags
   after the reference's last one (4 + 6L + 4i + k), encoder states per
   (sequence id, position) from their own stream; bf16-rounded like the weights. */
static const int kCrossTensors = 4;
uint64_t eo_encoder_seed(uint64_t model_seed) { return eo_splitmix64_at(model_seed, 0x454E43u); }
int eo_model_set_heads(eo_model* m, int n_heads) {
    if (n_heads < 1 || m->d % n_heads) { set_err("ModelConfig: n_heads must divide d_model"); return EO_INVALID_ARGUMENT; }
    m->n_heads = n_heads;
    return EO_OK;
}

static const double* encoder_output(const eo_model* m, int seq_id);
void eo_encoder_state(const eo_model* m, int seq_id, int t, double* out) {
    if (m->enc_layers > 0) {
        memcpy(out, encoder_output(m, seq_id) + (size_t)t * m->d, sizeof(double) * (size_t)m->d);
        return;
    }
    eo_seeded_vector(m->d, eo_splitmix64_at(m->enc_seed, ((uint64_t)seq_id << 20) | (uint64_t)t), out);
    if (m->round_bf16) round_all(out, (size_t)m->d);
}
/* encoder input id of (sequence, position): uniform over [1, V) like gen_workload's prompts */
int eo_encoder_token(const eo_model* m, int seq_id, int t) {
    return 1 + (int)(eo_splitmix64_at(m->enc_seed ^ 0x544F4Bu, ((uint64_t)seq_id << 20) | (uint64_t)t) %
                     (uint64_t)(m->V - 1));
}
/* encoder weights: tags after the cross weights, 4 + 6L + 4L + 6i + k */
int eo_model_set_encoder_layers(eo_model* m, int n) {
    if (n < 0 || (n > 0 && m->enc_len == 0)) { set_err("ModelConfig: encoder_layers needs T5 mode"); return EO_INVALID_ARGUMENT; }
    if (m->we) { set_err("encoder layers already set"); return EO_INVALID_ARGUMENT; }
    const int d = m->d;
    m->enc_layers = n;
    m->we = (double**)calloc((size_t)(n > 0 ? n : 1) * 6, sizeof(double*));
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 6; ++k) {
            const int r = k == 4 ? 4 * d : d, c = k == 5 ? 4 * d : d;
            double* t = (double*)malloc(sizeof(double) * (size_t)r * c);
            eo_seeded_matrix(r, c, eo_splitmix64_at(m->seed, 4 + (uint64_t)m->L * 10 + (uint64_t)i * 6 + k), t);
            if (m->round_bf16) round_all(t, (size_t)r * c);
            m->we[i * 6 + k] = t;
        }
    return EO_OK;
}

eo_model* eo_model_seeded_t5(int L, int d, int V, uint64_t seed, int round_bf16, int enc_len) {
    if (L < 2 || d < 2 || V < 2) { set_err("ModelConfig: bad dims"); return NULL; }
    if (enc_len < 0) { set_err("ModelConfig: encoder_len must be >= 0"); return NULL; }
    eo_model* m = (eo_model*)calloc(1, sizeof(eo_model));
    m->L = L; m->d = d; m->V = V; m->seed = seed;
    m->enc_len = enc_len; m->round_bf16 = round_bf16; m->enc_seed = eo_encoder_seed(seed); m->n_heads = 1;
    if (enc_len > 0) {
        m->wc = (double**)calloc((size_t)L * kCrossTensors, sizeof(double*));
        for (int i = 0; i < L; ++i)
            for (int k = 0; k < kCrossTensors; ++k) {
                double* t = (double*)malloc(sizeof(double) * (size_t)d * d);
                eo_seeded_matrix(d, d, eo_splitmix64_at(seed, 4 + (uint64_t)L * 6 + (uint64_t)i * 4 + k), t);
                if (round_bf16) round_all(t, (size_t)d * d);
                m->wc[i * kCrossTensors + k] = t;
            }
    }
    m->emb = (double*)malloc(sizeof(double) * (size_t)V * d);
    m->lm = (double*)malloc(sizeof(double) * (size_t)V * d);
    m->pw = (double*)malloc(sizeof(double) * (size_t)d);
    eo_seeded_matrix(V, d, eo_splitmix64_at(seed, 0), m->emb);
    eo_seeded_matrix(V, d, eo_splitmix64_at(seed, 1), m->lm);
    eo_seeded_vector(d, eo_splitmix64_at(seed, 2), m->pw);
    m->pb = 2.0 * eo_uniform01_at(eo_splitmix64_at(seed, 3), 0) - 1.0;
    m->w = (double**)calloc((size_t)L * kLayerTensors, sizeof(double*));
    for (int i = 0; i < L; ++i) {
        const uint64_t base = 4 + (uint64_t)i * 6;
        for (int k = 0; k < kLayerTensors; ++k) {
            int r, c;
            tensor_shape(m, k, &r, &c);
            double* t = (double*)malloc(sizeof(double) * (size_t)r * c);
            eo_seeded_matrix(r, c, eo_splitmix64_at(seed, base + k), t);
            m->w[i * kLayerTensors + k] = t;
        }
    }
    if (round_bf16) {
        round_all(m->emb, (size_t)V * d);
        round_all(m->lm, (size_t)V * d);
        round_all(m->pw, (size_t)d);
        m->pb = eo_round_bf16(m->pb);
        for (int i = 0; i < L * kLayerTensors; ++i) {
            int r, c;
            tensor_shape(m, i % kLayerTensors, &r, &c);
            round_all(m->w[i], (size_t)r * c);
        }
    }
    return m;
}

void eo_model_free(eo_model* m) {
    if (!m) return;
    if (m->we) {
        for (int i = 0; i < m->enc_layers * 6; ++i) free(m->we[i]);
        free(m->we);
    }
    for (int i = 0; i < m->n_enc_cache; ++i) free(m->enc_cache[i]);
    free(m->enc_cache); free(m->enc_cache_id);
    if (m->wc) {
        for (int i = 0; i < m->L * kCrossTensors; ++i) free(m->wc[i]);
        free(m->wc);
    }
    for (int i = 0; i < m->L * kLayerTensors; ++i) free(m->w[i]);
    free(m->w); free(m->emb); free(m->lm); free(m->pw); free(m);
}

int eo_model_tensor(const eo_model* m, int which, int layer, double* out, int64_t cap) {
    const double* src; int64_t n;
    if (which == 0) { src = m->emb; n = (int64_t)m->V * m->d; }
    else if (which == 1) { src = m->lm; n = (int64_t)m->V * m->d; }
    else if (which == 2) { src = m->pw; n = m->d; }
    else if (which == 3) { src = &m->pb; n = 1; }
    else if (which >= 20 && which < 26) {  /* T5 encoder stack: q, k, v, o, up, down */
        if (!m->we || layer < 1 || layer > m->enc_layers) { set_err("bad tensor"); return EO_INVALID_ARGUMENT; }
        src = m->we[(layer - 1) * 6 + (which - 20)];
        n = (int64_t)m->d * m->d * ((which == 24 || which == 25) ? 4 : 1);
    }
    else if (which >= 10 && which < 10 + kCrossTensors) {  /* T5 mode: q_c, k_c, v_c, o_c */
        if (!m->wc || layer < 1 || layer > m->L) { set_err("bad tensor"); return EO_INVALID_ARGUMENT; }
        src = m->wc[(layer - 1) * kCrossTensors + (which - 10)]; n = (int64_t)m->d * m->d;
    }
    else {
        if (layer < 1 || layer > m->L || which - 4 >= kLayerTensors) { set_err("bad tensor"); return EO_INVALID_ARGUMENT; }
        int r, c;
        tensor_shape(m, which - 4, &r, &c);
        src = layer_tensor(m, layer, which - 4); n = (int64_t)r * c;
    }
    if (cap < n) { set_err("buffer too small"); return EO_INVALID_ARGUMENT; }
    memcpy(out, src, sizeof(double) * (size_t)n);
    return EO_OK;
}

/* numerics.cpp:28-43 -- left-to-right accumulation */
static void matvec(const double* w, int rows, int cols, const double* x, double* y) {
    for (int r = 0; r < rows; ++r) {
        const double* row = w + (size_t)r * cols;
        double acc = 0.0;
        for (int c = 0; c < cols; ++c) acc += row[c] * x[c];
        y[r] = acc;
    }
}
/* numerics.cpp:54-74 */
static int softmax(const double* v, int n, double* out) {
    if (n <= 0) { set_err("softmax: empty input"); return EO_INVALID_ARGUMENT; }
    for (int i = 0; i < n; ++i)
        if (!isfinite(v[i])) { set_err("softmax: non-finite input"); return EO_INVALID_ARGUMENT; }
    double mx = v[0];
    for (int i = 1; i < n; ++i) if (mx < v[i]) mx = v[i]; /* std::max_element: first max */
    double sum = 0.0;
    for (int i = 0; i < n; ++i) { out[i] = exp(v[i] - mx); sum += out[i]; }
    for (int i = 0; i < n; ++i) out[i] /= sum;
    return EO_OK;
}

/* exit_policy.cpp:57-87, numerics.cpp:76-90 */
double eo_softmax_response_confidence(const double* logits, int n) {
    if (n < 2) return NAN;
    double* p = (double*)malloc(sizeof(double) * (size_t)n);
    if (softmax(logits, n, p) != EO_OK) { free(p); return NAN; }
    double top1 = -1.0, top2 = -1.0;
    for (int i = 0; i < n; ++i) {
        const double x = p[i];
        if (x > top1) { top2 = top1; top1 = x; }
        else if (x > top2) { top2 = x; }
    }
    free(p);
    return top1 - top2;
}
double eo_state_similarity_confidence(const double* u, const double* v, int n) {
    double uv = 0.0, uu = 0.0, vv = 0.0;
    for (int i = 0; i < n; ++i) { uv += u[i] * v[i]; uu += u[i] * u[i]; vv += v[i] * v[i]; }
    if (uu == 0.0 || vv == 0.0) return NAN;
    return uv / (sqrt(uu) * sqrt(vv));
}
double eo_classifier_confidence(const double* h, const double* w, double b, int n) {
    double z = b;
    for (int i = 0; i < n; ++i) z += w[i] * h[i];
    return 1.0 / (1.0 + exp(-z));
}
/* exit_policy.cpp:50-55 */
double eo_threshold_at(double lambda0, double gamma, double lambda_min, int layer) {
    const double v = lambda0 * pow(gamma, (double)(layer - 1));
    return (lambda_min < v) ? v : lambda_min; /* std::max(lambda_min, v) */
}

/* model.cpp:288-299 */
static int greedy_token(const double* logits, int n) {
    int best = 0;
    for (int i = 1; i < n; ++i) if (logits[i] > logits[best]) best = i;
    return best;
}

/* ------------------------------------------------------------------ */
/* kv_cache.cpp -- block pool with LIFO free list                       */
/* ------------------------------------------------------------------ */
typedef struct {
    int live;
    int capacity_tokens, committed, bpl;
    int* written;  /* [L] */
    int* table;    /* [L][bpl] */
} kv_seq;

typedef struct {
    int d, L, pool, cap;
    double *k, *v;
    int* free_list; int n_free;
    int peak;
    kv_seq* seqs; int n_seqs;
} kv_store;

static int kv_init(kv_store* s, int d, int L, int pool, int cap, int max_ids, int alloc_data) {
    if (d <= 0 || L <= 0 || pool <= 0 || cap <= 0) { set_err("KvStore: all constructor parameters must be positive"); return EO_INVALID_ARGUMENT; }
    memset(s, 0, sizeof *s);
    s->d = d; s->L = L; s->pool = pool; s->cap = cap;
    if (alloc_data) {
        s->k = (double*)calloc((size_t)pool * cap * d, sizeof(double));
        s->v = (double*)calloc((size_t)pool * cap * d, sizeof(double));
        if (!s->k || !s->v) { set_err("KvStore: out of host memory"); return EO_RUNTIME_ERROR; }
    }
    s->free_list = (int*)malloc(sizeof(int) * (size_t)pool);
    for (int b = pool - 1; b >= 0; --b) s->free_list[s->n_free++] = b; /* kv_cache.cpp:53-55 */
    s->seqs = (kv_seq*)calloc((size_t)(max_ids > 0 ? max_ids : 1), sizeof(kv_seq));
    s->n_seqs = max_ids;
    return EO_OK;
}
static void kv_destroy(kv_store* s) {
    for (int i = 0; i < s->n_seqs; ++i) { free(s->seqs[i].written); free(s->seqs[i].table); }
    free(s->seqs); free(s->free_list); free(s->k); free(s->v);
}
/* kv_cache.cpp:78-106 */
static int kv_allocate(kv_store* s, int id, int capacity_tokens) {
    if (id < 0 || id >= s->n_seqs) { set_err("allocate: id out of range"); return EO_INVALID_ARGUMENT; }
    if (s->seqs[id].live) { set_err("allocate: seq_id %d already allocated", id); return EO_INVALID_ARGUMENT; }
    if (capacity_tokens < 0) { set_err("allocate: negative capacity"); return EO_INVALID_ARGUMENT; }
    const int bpl = (capacity_tokens + s->cap - 1) / s->cap;
    const long need = (long)bpl * s->L;
    if (need > s->n_free) { set_err("allocate: need %ld blocks, %d free", need, s->n_free); return EO_KV_OUT_OF_MEMORY; }
    kv_seq* e = &s->seqs[id];
    free(e->written); free(e->table);
    e->live = 1; e->capacity_tokens = bpl * s->cap; e->committed = 0; e->bpl = bpl;
    e->written = (int*)calloc((size_t)s->L, sizeof(int));
    e->table = (int*)malloc(sizeof(int) * (size_t)(bpl > 0 ? bpl : 1) * s->L);
    for (int layer = 0; layer < s->L; ++layer)
        for (int b = 0; b < bpl; ++b) e->table[layer * bpl + b] = s->free_list[--s->n_free];
    const int in_use = s->pool - s->n_free;
    if (in_use > s->peak) s->peak = in_use;
    return EO_OK;
}
/* kv_cache.cpp:182-194 */
static int kv_release(kv_store* s, int id) {
    if (id < 0 || id >= s->n_seqs || !s->seqs[id].live) { set_err("release: unknown or already released seq_id %d", id); return EO_INVALID_ARGUMENT; }
    kv_seq* e = &s->seqs[id];
    for (int layer = 0; layer < s->L; ++layer)
        for (int b = 0; b < e->bpl; ++b) s->free_list[s->n_free++] = e->table[layer * e->bpl + b];
    e->live = 0;
    return EO_OK;
}
static double* kv_slot(kv_store* s, int which, int id, int layer, int pos) {
    const kv_seq* e = &s->seqs[id];
    const int block = e->table[(layer - 1) * e->bpl + pos / s->cap];
    const size_t base = ((size_t)block * s->cap + (size_t)(pos % s->cap)) * (size_t)s->d;
    return (which == 0 ? s->k : s->v) + base;
}
/* kv_cache.cpp:108-145 */
static int kv_append(kv_store* s, int id, int layer, int pos, const double* k, const double* v) {
    if (id < 0 || id >= s->n_seqs || !s->seqs[id].live) { set_err("append: unknown seq_id %d", id); return EO_INVALID_ARGUMENT; }
    if (layer < 1 || layer > s->L) { set_err("append: layer %d outside [1, %d]", layer, s->L); return EO_INVALID_ARGUMENT; }
    kv_seq* e = &s->seqs[id];
    int* written = &e->written[layer - 1];
    if (pos < *written) { set_err("append: slot already written"); return EO_RUNTIME_ERROR; }
    if (pos > *written) { set_err("append: position gap"); return EO_RUNTIME_ERROR; }
    if (pos >= e->capacity_tokens) { set_err("append: position exceeds reserved capacity"); return EO_KV_OUT_OF_MEMORY; }
    memcpy(kv_slot(s, 0, id, layer, pos), k, sizeof(double) * (size_t)s->d);
    memcpy(kv_slot(s, 1, id, layer, pos), v, sizeof(double) * (size_t)s->d);
    ++*written;
    return EO_OK;
}
/* kv_cache.cpp:165-180 */
static int kv_commit(kv_store* s, int id) {
    kv_seq* e = &s->seqs[id];
    for (int layer = 1; layer <= s->L; ++layer)
        if (e->written[layer - 1] != e->committed + 1) { set_err("commit: layer %d incomplete", layer); return EO_RUNTIME_ERROR; }
    ++e->committed;
    return EO_OK;
}

int eo_kv_block_trace(int L, int pool, int cap, int n_ops, const int32_t* ops, const int32_t* caps,
                      int n_ids, int bpl_max, int32_t* tables) {
    kv_store s;
    int rc = kv_init(&s, 1, L, pool, cap, n_ids, 0);
    if (rc) return -rc;
    for (int i = 0; i < (long)n_ids * L * bpl_max; ++i) tables[i] = -1;
    for (int i = 0; i < n_ops; ++i) {
        if (ops[i] > 0) {
            const int id = ops[i] - 1;
            rc = kv_allocate(&s, id, caps[i]);
            if (rc == EO_KV_OUT_OF_MEMORY) continue;
            if (rc) { kv_destroy(&s); return -rc; }
            const kv_seq* e = &s.seqs[id];
            for (int l = 0; l < L; ++l)
                for (int b = 0; b < e->bpl && b < bpl_max; ++b)
                    tables[((size_t)id * L + l) * bpl_max + b] = e->table[l * e->bpl + b];
        } else if (ops[i] < 0) {
            rc = kv_release(&s, -ops[i] - 1);
            if (rc) { kv_destroy(&s); return -rc; }
        }
    }
    const int nf = s.n_free;
    kv_destroy(&s);
    return nf;
}

/* ------------------------------------------------------------------ */
/* model.cpp:197-272 layer_forward over the flattened batch             */
/* ------------------------------------------------------------------ */
typedef struct {
    double *q, *k, *v, *att, *proj, *mid, *up, *down, *scores, *probs;
    int cap_scores;
} scratch_t;

static void scratch_init(scratch_t* w, int B, int d) {
    w->q = (double*)malloc(sizeof(double) * (size_t)B * d);
    w->k = (double*)malloc(sizeof(double) * (size_t)B * d);
    w->v = (double*)malloc(sizeof(double) * (size_t)B * d);
    w->att = (double*)malloc(sizeof(double) * (size_t)B * d);
    w->proj = (double*)malloc(sizeof(double) * (size_t)B * d);
    w->mid = (double*)malloc(sizeof(double) * (size_t)B * d);
    w->up = (double*)malloc(sizeof(double) * (size_t)B * 4 * d);
    w->down = (double*)malloc(sizeof(double) * (size_t)B * d);
    w->cap_scores = 0; w->scores = NULL; w->probs = NULL;
}
static void scratch_free(scratch_t* w) {
    free(w->q); free(w->k); free(w->v); free(w->att); free(w->proj); free(w->mid);
    free(w->up); free(w->down); free(w->scores); free(w->probs);
}
static void scratch_scores(scratch_t* w, int n) {
    if (n > w->cap_scores) {
        w->cap_scores = n * 2;
        w->scores = (double*)realloc(w->scores, sizeof(double) * (size_t)w->cap_scores);
        w->probs = (double*)realloc(w->probs, sizeof(double) * (size_t)w->cap_scores);
    }
}

/* Attention of one query over n key/value rows, split into heads (T5 mode; heads = 1 is
   model.cpp:223-243 exactly): per head h over features [h hd, (h+1) hd):
   a_h = softmax(q_h K_h^T / sqrt(hd)) V_h.  key(p) / val(p) give row p. */
typedef const double* (*row_fn)(const void* ctx, int p);
static int attend_heads(int d, int heads, const double* q, int n, row_fn key, row_fn val, const void* ctx,
                        double* scores, double* probs, double* a) {
    const int hd = d / heads;
    const double scale = 1.0 / sqrt((double)hd);
    for (int i = 0; i < d; ++i) a[i] = 0.0;
    for (int h = 0; h < heads; ++h) {
        const int f0 = h * hd;
        for (int p = 0; p < n; ++p) {
            const double* kr = key(ctx, p);
            double acc = 0.0;
            for (int i = f0; i < f0 + hd; ++i) acc += kr[i] * q[i];
            scores[p] = acc * scale;
        }
        int rc = softmax(scores, n, probs);
        if (rc) return rc;
        for (int p = 0; p < n; ++p) {
            const double* vr = val(ctx, p);
            for (int i = f0; i < f0 + hd; ++i) a[i] += probs[p] * vr[i];
        }
    }
    return EO_OK;
}

/* row accessors of attend_heads: the paged cache of (seq, layer), or two row-major matrices */
typedef struct { kv_store* cache; int id, layer; } kv_ctx;
static const double* kv_key_row(const void* c, int p) {
    const kv_ctx* x = (const kv_ctx*)c;
    return kv_slot(x->cache, 0, x->id, x->layer, p);
}
static const double* kv_val_row(const void* c, int p) {
    const kv_ctx* x = (const kv_ctx*)c;
    return kv_slot(x->cache, 1, x->id, x->layer, p);
}
typedef struct { const double* rows; int d; } mat_ctx;
static const double* mat_key_row(const void* c, int p) {
    const mat_ctx* x = ((const mat_ctx* const*)c)[0];
    return x->rows + (size_t)p * x->d;
}
static const double* mat_val_row(const void* c, int p) {
    const mat_ctx* x = ((const mat_ctx* const*)c)[1];
    return x->rows + (size_t)p * x->d;
}

/* The encoder stack over one sequence's T seeded input ids (fp64; bf16-rounded output when the
   model is): X_0[t] = embedding(id_t); per layer X <- mid + W_down ReLU(W_up mid), mid = X + W_o a,
   a_t = attention of q_t = W_q X_t over every position's (W_k X, W_v X) -- no causal mask. */
static const double* encoder_output(const eo_model* m, int seq_id) {
    eo_model* mm = (eo_model*)m;  /* the cache is logically const */
    for (int i = 0; i < m->n_enc_cache; ++i)
        if (m->enc_cache_id[i] == seq_id) return m->enc_cache[i];
    const int d = m->d, T = m->enc_len;
    double* X = (double*)malloc(sizeof(double) * (size_t)T * d);
    double *Q = (double*)malloc(sizeof(double) * (size_t)T * d), *K = (double*)malloc(sizeof(double) * (size_t)T * d);
    double *Vv = (double*)malloc(sizeof(double) * (size_t)T * d), *A = (double*)malloc(sizeof(double) * (size_t)d);
    double *P = (double*)malloc(sizeof(double) * (size_t)d), *U = (double*)malloc(sizeof(double) * (size_t)4 * d);
    double *sc = (double*)malloc(sizeof(double) * (size_t)T), *pr = (double*)malloc(sizeof(double) * (size_t)T);
    double* mid = (double*)malloc(sizeof(double) * (size_t)T * d);
    for (int t = 0; t < T; ++t)
        memcpy(X + (size_t)t * d, m->emb + (size_t)eo_encoder_token(m, seq_id, t) * d, sizeof(double) * (size_t)d);
    for (int l = 0; l < m->enc_layers; ++l) {
        double* const* w = m->we + (size_t)l * 6;
        for (int t = 0; t < T; ++t) {
            matvec(w[0], d, d, X + (size_t)t * d, Q + (size_t)t * d);
            matvec(w[1], d, d, X + (size_t)t * d, K + (size_t)t * d);
            matvec(w[2], d, d, X + (size_t)t * d, Vv + (size_t)t * d);
        }
        const mat_ctx ck = {K, d}, cv = {Vv, d};
        const mat_ctx* both[2] = {&ck, &cv};
        for (int t = 0; t < T; ++t) {
            attend_heads(d, m->n_heads, Q + (size_t)t * d, T, mat_key_row, mat_val_row, both, sc, pr, A);
            matvec(w[3], d, d, A, P);
            for (int i = 0; i < d; ++i) mid[(size_t)t * d + i] = X[(size_t)t * d + i] + P[i];
        }
        for (int t = 0; t < T; ++t) {
            matvec(w[4], 4 * d, d, mid + (size_t)t * d, U);
            for (int i = 0; i < 4 * d; ++i) U[i] = U[i] > 0.0 ? U[i] : 0.0;
            matvec(w[5], d, 4 * d, U, P);
            for (int i = 0; i < d; ++i) X[(size_t)t * d + i] = mid[(size_t)t * d + i] + P[i];
        }
    }
    if (m->round_bf16) round_all(X, (size_t)T * d);
    free(Q); free(K); free(Vv); free(A); free(P); free(U); free(sc); free(pr); free(mid);
    if (mm->n_enc_cache == mm->cap_enc_cache) {
        mm->cap_enc_cache = mm->cap_enc_cache ? 2 * mm->cap_enc_cache : 64;
        mm->enc_cache_id = (int*)realloc(mm->enc_cache_id, sizeof(int) * (size_t)mm->cap_enc_cache);
        mm->enc_cache = (double**)realloc(mm->enc_cache, sizeof(double*) * (size_t)mm->cap_enc_cache);
    }
    mm->enc_cache_id[mm->n_enc_cache] = seq_id;
    mm->enc_cache[mm->n_enc_cache] = X;
    ++mm->n_enc_cache;
    return X;
}

/* h[B][d] in, out[B][d] out (out may not alias h). ids[B] are seq ids. */
static int layer_forward(const eo_model* m, int layer, int B, const int* ids, const double* h,
                         kv_store* cache, scratch_t* w, double* out) {
    const int d = m->d;
    const double scale = 1.0 / sqrt((double)d);
    const double *wq = layer_tensor(m, layer, 0), *wk = layer_tensor(m, layer, 1), *wv = layer_tensor(m, layer, 2);
    const double *wo = layer_tensor(m, layer, 3), *wup = layer_tensor(m, layer, 4), *wdn = layer_tensor(m, layer, 5);
    for (int b = 0; b < B; ++b) matvec(wq, d, d, h + (size_t)b * d, w->q + (size_t)b * d);
    for (int b = 0; b < B; ++b) matvec(wk, d, d, h + (size_t)b * d, w->k + (size_t)b * d);
    for (int b = 0; b < B; ++b) matvec(wv, d, d, h + (size_t)b * d, w->v + (size_t)b * d);
    for (int b = 0; b < B; ++b) {
        const int id = ids[b];
        if (id < 0 || id >= cache->n_seqs || !cache->seqs[id].live) { set_err("unknown seq_id %d", id); return EO_INVALID_ARGUMENT; }
        const int pos = cache->seqs[id].committed;
        int rc = kv_append(cache, id, layer, pos, w->k + (size_t)b * d, w->v + (size_t)b * d);
        if (rc) return rc;
        const int n = pos + 1;
        scratch_scores(w, n);
        const double* q = w->q + (size_t)b * d;
        if (m->n_heads > 1) {  /* extension: heads (attend_heads) */
            const kv_ctx cx = {cache, id, layer};
            rc = attend_heads(d, m->n_heads, q, n, kv_key_row, kv_val_row, &cx, w->scores, w->probs,
                              w->att + (size_t)b * d);
            if (rc) return rc;
            continue;
        }
        for (int p = 0; p < n; ++p) {
            const double* key = kv_slot(cache, 0, id, layer, p);
            double acc = 0.0;
            for (int i = 0; i < d; ++i) acc += key[i] * q[i];
            w->scores[p] = acc * scale;
        }
        rc = softmax(w->scores, n, w->probs);
        if (rc) return rc;
        double* a = w->att + (size_t)b * d;
        for (int i = 0; i < d; ++i) a[i] = 0.0;
        for (int p = 0; p < n; ++p) {
            const double* val = kv_slot(cache, 1, id, layer, p);
            const double weight = w->probs[p];
            for (int i = 0; i < d; ++i) a[i] += weight * val[i];
        }
    }
    for (int b = 0; b < B; ++b) matvec(wo, d, d, w->att + (size_t)b * d, w->proj + (size_t)b * d);
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < d; ++i) w->mid[(size_t)b * d + i] = h[(size_t)b * d + i] + w->proj[(size_t)b * d + i];
    if (m->enc_len > 0) {
        /* T5 mode: mid += W_oc . softmax(q_c K_c^T / sqrt(d)) V_c, q_c = W_qc . mid,
           K_c[t] = W_kc . E[t], V_c[t] = W_vc . E[t] over the sequence's encoder states */
        const int T = m->enc_len;
        const double *wqc = m->wc[(layer - 1) * kCrossTensors + 0], *wkc = m->wc[(layer - 1) * kCrossTensors + 1];
        const double *wvc = m->wc[(layer - 1) * kCrossTensors + 2], *woc = m->wc[(layer - 1) * kCrossTensors + 3];
        double* e = (double*)malloc(sizeof(double) * (size_t)d);
        double* kc = (double*)malloc(sizeof(double) * (size_t)T * d);
        double* vc = (double*)malloc(sizeof(double) * (size_t)T * d);
        scratch_scores(w, T);
        for (int b = 0; b < B; ++b) {
            for (int t = 0; t < T; ++t) {
                eo_encoder_state(m, ids[b], t, e);
                matvec(wkc, d, d, e, kc + (size_t)t * d);
                matvec(wvc, d, d, e, vc + (size_t)t * d);
            }
            double* q = w->q + (size_t)b * d;
            matvec(wqc, d, d, w->mid + (size_t)b * d, q);
            double* a = w->att + (size_t)b * d;
            if (m->n_heads > 1) {
                const mat_ctx ck = {kc, d}, cv = {vc, d};
                const mat_ctx* both[2] = {&ck, &cv};
                int rc = attend_heads(d, m->n_heads, q, T, mat_key_row, mat_val_row, both, w->scores, w->probs, a);
                if (rc) { free(e); free(kc); free(vc); return rc; }
            } else {
                for (int t = 0; t < T; ++t) {
                    double acc = 0.0;
                    for (int i = 0; i < d; ++i) acc += kc[(size_t)t * d + i] * q[i];
                    w->scores[t] = acc * scale;
                }
                int rc = softmax(w->scores, T, w->probs);
                if (rc) { free(e); free(kc); free(vc); return rc; }
                for (int i = 0; i < d; ++i) a[i] = 0.0;
                for (int t = 0; t < T; ++t)
                    for (int i = 0; i < d; ++i) a[i] += w->probs[t] * vc[(size_t)t * d + i];
            }
            matvec(woc, d, d, a, w->proj + (size_t)b * d);
            for (int i = 0; i < d; ++i) w->mid[(size_t)b * d + i] += w->proj[(size_t)b * d + i];
        }
        free(e); free(kc); free(vc);
    }
    for (int b = 0; b < B; ++b) {
        double* u = w->up + (size_t)b * 4 * d;
        matvec(wup, 4 * d, d, w->mid + (size_t)b * d, u);
    }
    for (int b = 0; b < B; ++b) {
        double* u = w->up + (size_t)b * 4 * d;
        for (int i = 0; i < 4 * d; ++i) if (u[i] < 0.0) u[i] = 0.0;
    }
    for (int b = 0; b < B; ++b) matvec(wdn, d, 4 * d, w->up + (size_t)b * 4 * d, w->down + (size_t)b * d);
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < d; ++i) out[(size_t)b * d + i] = w->mid[(size_t)b * d + i] + w->down[(size_t)b * d + i];
    return EO_OK;
}

/* model.cpp:274-282 + kv_cache.cpp:222-234 */
static int fill_skipped(const eo_model* m, kv_store* cache, int B, const int* ids, const double* h_exit,
                        int output_layer, double* kbuf, double* vbuf) {
    const int d = m->d;
    for (int b = 0; b < B; ++b) {
        const int id = ids[b];
        const int pos = cache->seqs[id].committed;
        for (int layer = output_layer + 1; layer <= m->L; ++layer) {
            matvec(layer_tensor(m, layer, 1), d, d, h_exit + (size_t)b * d, kbuf);
            matvec(layer_tensor(m, layer, 2), d, d, h_exit + (size_t)b * d, vbuf);
            int rc = kv_append(cache, id, layer, pos, kbuf, vbuf);
            if (rc) return rc;
        }
    }
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* engine.cpp:47-75 ExitStatusVector                                    */
/* ------------------------------------------------------------------ */
int eo_status_trace(int B, int L, const double* conf, const double* lambdas, int32_t* first_accept) {
    unsigned char* status = (unsigned char*)calloc((size_t)B, 1);
    for (int b = 0; b < B; ++b) first_accept[b] = 0;
    int out = L;
    for (int layer = 1; layer <= L; ++layer) {
        int all = 1;
        for (int b = 0; b < B; ++b) {
            const int acc = conf[(size_t)(layer - 1) * B + b] > lambdas[layer - 1];
            if (!status[b] && acc) { status[b] = 1; first_accept[b] = layer; }
            all = all && status[b];
        }
        if (all) { out = layer; break; }
    }
    for (int b = 0; b < B; ++b) if (first_accept[b] == 0) first_accept[b] = L;
    free(status);
    return out;
}

/* ------------------------------------------------------------------ */
/* workload.cpp:15-89                                                   */
/* ------------------------------------------------------------------ */
static int sample_token(rng_t* r, int V, int eos) {
    const int exclude = eos >= 0 && eos < V;
    const int span = exclude ? V - 1 : V;
    int id = (int)(rng_next(r) % (uint64_t)span);
    if (exclude && id >= eos) ++id;
    return id;
}
static int sample_range(rng_t* r, int lo, int hi) { return lo + (int)(rng_next(r) % (uint64_t)(hi - lo + 1)); }

int64_t eo_gen_workload(const eo_gen_params* p, double* arrival, int32_t* prompt_off, int32_t* prompt,
                        int32_t* max_new) {
    if (p->n_requests < 0 || p->mean_interarrival < 0.0 || p->prompt_len_min < 1 ||
        p->prompt_len_max < p->prompt_len_min || p->output_len_min < 1 ||
        p->output_len_max < p->output_len_min || p->vocab_size < 2) {
        set_err("gen_workload: bad parameters");
        return -1;
    }
    rng_t r = {p->seed};
    double t = 0.0;
    int64_t total = 0;
    if (prompt_off) prompt_off[0] = 0;
    for (int i = 0; i < p->n_requests; ++i) {
        if (p->mean_interarrival > 0.0) t += -p->mean_interarrival * log(1.0 - rng_next_double(&r));
        if (arrival) arrival[i] = t;
        const int plen = sample_range(&r, p->prompt_len_min, p->prompt_len_max);
        for (int j = 0; j < plen; ++j) {
            const int tok = sample_token(&r, p->vocab_size, p->eos_token);
            if (prompt) prompt[total + j] = tok;
        }
        total += plen;
        if (prompt_off) prompt_off[i + 1] = (int32_t)total;
        const int mn = sample_range(&r, p->output_len_min, p->output_len_max);
        if (max_new) max_new[i] = mn;
    }
    return total;
}

/* ------------------------------------------------------------------ */
/* growable arrays for the flat transcript                              */
/* ------------------------------------------------------------------ */
typedef struct { int32_t* p; int64_t n, cap; } vi32;
typedef struct { double* p; int64_t n, cap; } vf64;
static void pi(vi32* a, int32_t x) {
    if (a->n == a->cap) { a->cap = a->cap ? a->cap * 2 : 16; a->p = (int32_t*)realloc(a->p, sizeof(int32_t) * (size_t)a->cap); }
    a->p[a->n++] = x;
}
static void pf(vf64* a, double x) {
    if (a->n == a->cap) { a->cap = a->cap ? a->cap * 2 : 16; a->p = (double*)realloc(a->p, sizeof(double) * (size_t)a->cap); }
    a->p[a->n++] = x;
}

typedef struct {
    int committed;
    double* k; /* [L][committed][d] */
    double* v;
    vf64 exit_states;
    int have_kv;
    int bpl;
    int* table; /* [L][bpl] block ids at eviction (KvStore block_table, kv_cache.hpp:79-84) */
} kv_capture;

struct eo_transcript {
    vi32 pf_seq, pf_positions, it_output_layer, it_batch_off, ps_seq, ps_accept, ps_token;
    vi32 sq_id, sq_max_new, sq_prompt_off, sq_prompt, sq_tok_off, sq_tokens, sq_exit_layers, sq_iter_out;
    vf64 pf_clock, pf_charge, it_clock, it_charge, sq_arrival, sq_first, sq_finish, meta, it_conf;
    kv_capture* caps; int n_caps; int d, L;
};

void eo_transcript_free(eo_transcript* t) {
    if (!t) return;
    vi32* is[] = {&t->pf_seq, &t->pf_positions, &t->it_output_layer, &t->it_batch_off, &t->ps_seq, &t->ps_accept,
                  &t->ps_token, &t->sq_id, &t->sq_max_new, &t->sq_prompt_off, &t->sq_prompt, &t->sq_tok_off,
                  &t->sq_tokens, &t->sq_exit_layers, &t->sq_iter_out};
    for (size_t i = 0; i < sizeof is / sizeof *is; ++i) free(is[i]->p);
    vf64* fs[] = {&t->pf_clock, &t->pf_charge, &t->it_clock, &t->it_charge, &t->sq_arrival, &t->sq_first,
                  &t->sq_finish, &t->meta, &t->it_conf};
    for (size_t i = 0; i < sizeof fs / sizeof *fs; ++i) free(fs[i]->p);
    for (int i = 0; i < t->n_caps; ++i) { free(t->caps[i].k); free(t->caps[i].v); free(t->caps[i].exit_states.p); free(t->caps[i].table); }
    free(t->caps);
    free(t);
}

static vi32* field_i32(eo_transcript* t, const char* f) {
#define F(name) if (!strcmp(f, #name)) return &t->name;
    F(pf_seq) F(pf_positions) F(it_output_layer) F(it_batch_off) F(ps_seq) F(ps_accept) F(ps_token)
    F(sq_id) F(sq_max_new) F(sq_prompt_off) F(sq_prompt) F(sq_tok_off) F(sq_tokens) F(sq_exit_layers) F(sq_iter_out)
#undef F
    return NULL;
}
static vf64* field_f64(eo_transcript* t, const char* f) {
#define F(name) if (!strcmp(f, #name)) return &t->name;
    F(pf_clock) F(pf_charge) F(it_clock) F(it_charge) F(sq_arrival) F(sq_first) F(sq_finish) F(meta) F(it_conf)
#undef F
    return NULL;
}
int64_t eo_transcript_len(const eo_transcript* t, const char* f) {
    vi32* a = field_i32((eo_transcript*)t, f);
    if (a) return a->n;
    vf64* b = field_f64((eo_transcript*)t, f);
    if (b) return b->n;
    return -1;
}
int eo_transcript_get_i32(const eo_transcript* t, const char* f, int32_t* out) {
    vi32* a = field_i32((eo_transcript*)t, f);
    if (!a) { set_err("unknown field %s", f); return EO_INVALID_ARGUMENT; }
    if (a->n) memcpy(out, a->p, sizeof(int32_t) * (size_t)a->n);
    return EO_OK;
}
int eo_transcript_get_f64(const eo_transcript* t, const char* f, double* out) {
    vf64* a = field_f64((eo_transcript*)t, f);
    if (!a) { set_err("unknown field %s", f); return EO_INVALID_ARGUMENT; }
    if (a->n) memcpy(out, a->p, sizeof(double) * (size_t)a->n);
    return EO_OK;
}
int eo_transcript_kv(const eo_transcript* t, int id, int layer, double* k, double* v, int64_t cap) {
    if (id < 0 || id >= t->n_caps || !t->caps[id].have_kv) { set_err("no capture for seq %d", id); return EO_INVALID_ARGUMENT; }
    const kv_capture* c = &t->caps[id];
    const size_t n = (size_t)c->committed * t->d;
    if ((int64_t)n > cap || layer < 1 || layer > t->L) { set_err("bad kv request"); return EO_INVALID_ARGUMENT; }
    memcpy(k, c->k + (size_t)(layer - 1) * n, sizeof(double) * n);
    memcpy(v, c->v + (size_t)(layer - 1) * n, sizeof(double) * n);
    return c->committed;
}
int eo_transcript_block_table(const eo_transcript* t, int id, int32_t* out, int64_t cap) {
    if (id < 0 || id >= t->n_caps || !t->caps[id].have_kv) { set_err("no capture for seq %d", id); return -EO_INVALID_ARGUMENT; }
    const kv_capture* c = &t->caps[id];
    if ((int64_t)c->bpl * t->L > cap) { set_err("buffer too small"); return -EO_INVALID_ARGUMENT; }
    for (int i = 0; i < c->bpl * t->L; ++i) out[i] = c->table[i];
    return c->bpl;
}
int eo_transcript_exit_states(const eo_transcript* t, int id, double* out, int64_t cap) {
    if (id < 0 || id >= t->n_caps) { set_err("no capture for seq %d", id); return EO_INVALID_ARGUMENT; }
    const kv_capture* c = &t->caps[id];
    if (c->exit_states.n > cap) { set_err("buffer too small"); return EO_INVALID_ARGUMENT; }
    memcpy(out, c->exit_states.p, sizeof(double) * (size_t)c->exit_states.n);
    return (int)(c->exit_states.n / t->d);
}

/* seeded KV prefix (bench workload) */
static uint64_t kv_prefix_seed(uint64_t kv_seed, int L, int seq, int layer, int pos, int kind) {
    const uint64_t tag = ((((uint64_t)seq * (uint64_t)L + (uint64_t)(layer - 1)) << 21) | (uint64_t)pos) << 1 | (uint64_t)kind;
    return eo_splitmix64_at(kv_seed, tag);
}
void eo_kv_prefix_vector(uint64_t kv_seed, int L, int seq, int layer, int pos, int kind, int d, int rb,
                         double* out) {
    eo_seeded_vector(d, kv_prefix_seed(kv_seed, L, seq, layer, pos, kind), out);
    if (rb) round_all(out, (size_t)d);
}

/* ------------------------------------------------------------------ */
/* Engine::run  (engine.cpp:110-330)                                    */
/* ------------------------------------------------------------------ */
typedef struct {
    int id, max_new, next_input, finished;
    double arrival, first_token, finish;
    vi32 tokens, exit_layers, iter_out;
    int prompt_off, prompt_len;
} live_seq;

static double check_cost(const eo_engine_config* c) {
    switch (c->technique) {
        case EO_TECH_SOFTMAX: return c->c_check_softmax;
        case EO_TECH_STATE: return c->c_check_state;
        case EO_TECH_CLASSIFIER: return c->c_check_classifier;
        default: return 0.0;
    }
}

static int validate_config(const eo_model* m, const eo_engine_config* c) {
    if (c->n_layers < 2 || c->d_model < 2 || c->vocab_size < 2) { set_err("ModelConfig: bad dims"); return EO_INVALID_ARGUMENT; }
    if (!(c->gamma > 0.0 && c->gamma <= 1.0) || c->lambda_min < 0.0 || c->lambda_min > c->lambda0) { set_err("ThresholdSchedule: invalid"); return EO_INVALID_ARGUMENT; }
    if (c->max_batch < 1 || c->pool_blocks < 1 || c->block_capacity < 1) { set_err("EngineConfig: invalid sizes"); return EO_INVALID_ARGUMENT; }
    if (c->eos_token >= c->vocab_size) { set_err("EngineConfig: eos_token outside vocab"); return EO_INVALID_ARGUMENT; }
    if (c->technique == EO_TECH_ALWAYS_AT && (c->exit_layer < 1 || c->exit_layer > c->n_layers)) { set_err("EngineConfig: always_at layer outside [1, n_layers]"); return EO_INVALID_ARGUMENT; }
    if (m && (m->L != c->n_layers || m->d != c->d_model || m->V != c->vocab_size)) { set_err("Engine: weights do not match config.model"); return EO_INVALID_ARGUMENT; }
    return EO_OK;
}

/* confidence of one (seq, layer) for the configured technique; NAN if none */
static double confidence(const eo_model* m, const eo_engine_config* c, const double* h_prev, const double* h_cur,
                         double* logits) {
    const int d = m->d;
    switch (c->technique) {
        case EO_TECH_SOFTMAX:
            matvec(m->lm, m->V, d, h_cur, logits);
            return eo_softmax_response_confidence(logits, m->V);
        case EO_TECH_STATE: return eo_state_similarity_confidence(h_prev, h_cur, d);
        case EO_TECH_CLASSIFIER: return eo_classifier_confidence(h_cur, m->pw, m->pb, d);
        default: return NAN;
    }
}

static int decide(const eo_engine_config* c, int layer, double conf, double lambda) {
    switch (c->technique) {
        case EO_TECH_NEVER: return 0;
        case EO_TECH_ALWAYS_AT: return layer >= c->exit_layer;
        default: return conf > lambda;
    }
}

int eo_engine_run(const eo_model* m, const eo_engine_config* c, int n_req, const double* arrival,
                  const int32_t* prompt_off, const int32_t* prompt, const int32_t* max_new,
                  const double* fixed_conf, int n_fixed_iters, eo_transcript** out) {
    *out = NULL;
    int rc = validate_config(m, c);
    if (rc) return rc;
    const int L = c->n_layers, d = c->d_model;

    /* Workload::validate_and_sort (workload.cpp:15-38): stable sort by arrival */
    int* order = (int*)malloc(sizeof(int) * (size_t)(n_req > 0 ? n_req : 1));
    for (int i = 0; i < n_req; ++i) order[i] = i;
    for (int i = 1; i < n_req; ++i) { /* insertion sort: stable */
        const int x = order[i];
        int j = i - 1;
        while (j >= 0 && arrival[x] < arrival[order[j]]) { order[j + 1] = order[j]; --j; }
        order[j + 1] = x;
    }
    for (int i = 0; i < n_req; ++i) {
        const int r = order[i];
        const int plen = prompt_off[r + 1] - prompt_off[r];
        if (arrival[r] < 0.0 || plen < 1 || max_new[r] < 1) { set_err("workload: invalid request %d", i); free(order); return EO_INVALID_ARGUMENT; }
        for (int j = 0; j < plen; ++j) {
            const int tok = prompt[prompt_off[r] + j];
            if (tok < 0 || tok >= c->vocab_size) { set_err("workload: token id outside vocab"); free(order); return EO_INVALID_ARGUMENT; }
        }
    }

    eo_transcript* t = (eo_transcript*)calloc(1, sizeof(eo_transcript));
    t->d = d; t->L = L; t->n_caps = n_req;
    t->caps = (kv_capture*)calloc((size_t)(n_req > 0 ? n_req : 1), sizeof(kv_capture));
    kv_store cache;
    rc = kv_init(&cache, d, L, c->pool_blocks, c->block_capacity, n_req, 1);
    if (rc) { free(order); eo_transcript_free(t); return rc; }

    live_seq* running = (live_seq*)calloc((size_t)c->max_batch, sizeof(live_seq));
    int n_running = 0;
    int next_pending = 0;
    double clock = 0.0, total_idle = 0.0;
    scratch_t ws;
    scratch_init(&ws, c->max_batch, d);
    double* states = (double*)malloc(sizeof(double) * (size_t)c->max_batch * d);
    double* next = (double*)malloc(sizeof(double) * (size_t)c->max_batch * d);
    double* logits = (double*)malloc(sizeof(double) * (size_t)c->vocab_size);
    double* kbuf = (double*)malloc(sizeof(double) * (size_t)d);
    double* vbuf = (double*)malloc(sizeof(double) * (size_t)d);
    int* ids = (int*)malloc(sizeof(int) * (size_t)c->max_batch);
    int iteration = 0;
    pi(&t->it_batch_off, 0);
    pi(&t->sq_prompt_off, 0);
    pi(&t->sq_tok_off, 0);

    for (;;) {
        /* evict_finished (engine.cpp:130-164) */
        int w = 0;
        for (int i = 0; i < n_running; ++i) {
            live_seq* s = &running[i];
            if (!s->finished) { running[w++] = *s; continue; }
            if (c->capture_kv) {
                kv_capture* cap = &t->caps[s->id];
                const int committed = cache.seqs[s->id].committed;
                cap->committed = committed;
                cap->k = (double*)malloc(sizeof(double) * (size_t)L * committed * d + 8);
                cap->v = (double*)malloc(sizeof(double) * (size_t)L * committed * d + 8);
                for (int layer = 1; layer <= L; ++layer)
                    for (int p = 0; p < committed; ++p) {
                        memcpy(cap->k + ((size_t)(layer - 1) * committed + p) * d, kv_slot(&cache, 0, s->id, layer, p), sizeof(double) * (size_t)d);
                        memcpy(cap->v + ((size_t)(layer - 1) * committed + p) * d, kv_slot(&cache, 1, s->id, layer, p), sizeof(double) * (size_t)d);
                    }
                cap->have_kv = 1;
                cap->bpl = cache.seqs[s->id].bpl;
                cap->table = (int*)malloc(sizeof(int) * (size_t)(cap->bpl * L + 1));
                memcpy(cap->table, cache.seqs[s->id].table, sizeof(int) * (size_t)cap->bpl * L);
            }
            kv_release(&cache, s->id);
            pi(&t->sq_id, s->id);
            pf(&t->sq_arrival, s->arrival);
            pf(&t->sq_first, s->first_token);
            pf(&t->sq_finish, s->finish);
            pi(&t->sq_max_new, s->max_new);
            for (int j = 0; j < s->prompt_len; ++j) pi(&t->sq_prompt, prompt[s->prompt_off + j]);
            pi(&t->sq_prompt_off, (int32_t)t->sq_prompt.n);
            for (int j = 0; j < s->tokens.n; ++j) {
                pi(&t->sq_tokens, s->tokens.p[j]);
                pi(&t->sq_exit_layers, s->exit_layers.p[j]);
                pi(&t->sq_iter_out, s->iter_out.p[j]);
            }
            pi(&t->sq_tok_off, (int32_t)t->sq_tokens.n);
            free(s->tokens.p); free(s->exit_layers.p); free(s->iter_out.p);
        }
        n_running = w;

        /* admit (engine.cpp:183-206) */
        while (next_pending < n_req) {
            const int r = order[next_pending];
            if (arrival[r] > clock) break;
            if (n_running >= c->max_batch) break;
            const int id = next_pending;
            const int plen = prompt_off[r + 1] - prompt_off[r];
            const int need = plen + max_new[r];
            rc = kv_allocate(&cache, id, need);
            if (rc == EO_KV_OUT_OF_MEMORY) break;
            if (rc) goto fail;
            live_seq* s = &running[n_running++];
            memset(s, 0, sizeof *s);
            s->id = id; s->arrival = arrival[r]; s->first_token = -1.0; s->finish = -1.0;
            s->max_new = max_new[r]; s->prompt_off = prompt_off[r]; s->prompt_len = plen;
            s->next_input = prompt[prompt_off[r] + plen - 1];
            /* prefill (engine.cpp:166-181) */
            const int positions = plen - 1;
            for (int j = 0; j < positions; ++j) {
                if (c->synthetic_kv_seed >= 0) {
                    for (int layer = 1; layer <= L; ++layer) {
                        eo_kv_prefix_vector((uint64_t)c->synthetic_kv_seed, L, id, layer, j, 0, d, c->round_bf16, kbuf);
                        eo_kv_prefix_vector((uint64_t)c->synthetic_kv_seed, L, id, layer, j, 1, d, c->round_bf16, vbuf);
                        rc = kv_append(&cache, id, layer, j, kbuf, vbuf);
                        if (rc) goto fail;
                    }
                } else {
                    const int tok = prompt[prompt_off[r] + j];
                    memcpy(states, m->emb + (size_t)tok * d, sizeof(double) * (size_t)d);
                    for (int layer = 1; layer <= L; ++layer) {
                        rc = layer_forward(m, layer, 1, &id, states, &cache, &ws, next);
                        if (rc) goto fail;
                        memcpy(states, next, sizeof(double) * (size_t)d);
                    }
                }
                rc = kv_commit(&cache, id);
                if (rc) goto fail;
            }
            const double charge = (double)positions * L * (c->c_layer_fixed + c->c_layer_per_seq);
            clock += charge;
            pf(&t->pf_clock, clock); pf(&t->pf_charge, charge); pi(&t->pf_seq, id); pi(&t->pf_positions, positions);
            ++next_pending;
        }

        if (n_running == 0) {
            if (next_pending >= n_req) break;
            const double na = arrival[order[next_pending]];
            if (na > clock) { total_idle += na - clock; clock = na; }
            continue;
        }

        /* decode_iteration (engine.cpp:208-310) */
        const int B = n_running;
        for (int b = 0; b < B; ++b) {
            ids[b] = running[b].id;
            memcpy(states + (size_t)b * d, m->emb + (size_t)running[b].next_input * d, sizeof(double) * (size_t)d);
        }
        unsigned char status[4096];
        int first_accept[4096];
        if (B > 4096) { set_err("batch too large"); rc = EO_INVALID_ARGUMENT; goto fail; }
        memset(status, 0, (size_t)B);
        memset(first_accept, 0, sizeof(int) * (size_t)B);
        const int64_t conf_base = t->it_conf.n;
        for (int i = 0; i < L * B; ++i) pf(&t->it_conf, NAN);
        int output_layer = L;
        for (int layer = 1; layer <= L; ++layer) {
            rc = layer_forward(m, layer, B, ids, states, &cache, &ws, next);
            if (rc) goto fail;
            const double lambda = eo_threshold_at(c->lambda0, c->gamma, c->lambda_min, layer);
            int all = 1;
            for (int b = 0; b < B; ++b) {
                double cf;
                if (c->technique == EO_TECH_FIXED) {
                    if (!fixed_conf || iteration >= n_fixed_iters) { set_err("fixed confidences exhausted"); rc = EO_INVALID_ARGUMENT; goto fail; }
                    cf = fixed_conf[((size_t)iteration * L + (layer - 1)) * c->max_batch + b];
                } else {
                    cf = confidence(m, c, states + (size_t)b * d, next + (size_t)b * d, logits);
                }
                t->it_conf.p[conf_base + (int64_t)(layer - 1) * B + b] = cf;
                const int acc = decide(c, layer, cf, lambda);
                if (!status[b] && acc) { status[b] = 1; first_accept[b] = layer; }
                all = all && status[b];
            }
            memcpy(states, next, sizeof(double) * (size_t)B * d);
            if (all) { output_layer = layer; break; }
        }
        rc = fill_skipped(m, &cache, B, ids, states, output_layer, kbuf, vbuf);
        if (rc) goto fail;
        for (int b = 0; b < B; ++b) { rc = kv_commit(&cache, ids[b]); if (rc) goto fail; }

        const double charge = output_layer * (c->c_layer_fixed + c->c_layer_per_seq * B) +
                              output_layer * B * check_cost(c) +
                              (double)(L - output_layer) * B * c->c_fill_per_seq_layer;
        clock += charge;
        pf(&t->it_clock, clock); pf(&t->it_charge, charge); pi(&t->it_output_layer, output_layer);
        for (int b = 0; b < B; ++b) {
            live_seq* s = &running[b];
            matvec(m->lm, m->V, d, states + (size_t)b * d, logits);
            const int token = greedy_token(logits, m->V);
            const int accept = first_accept[b] == 0 ? L : first_accept[b];
            pi(&t->ps_seq, s->id); pi(&t->ps_accept, accept); pi(&t->ps_token, token);
            pi(&s->tokens, token); pi(&s->exit_layers, accept); pi(&s->iter_out, output_layer);
            if (c->capture_kv)
                for (int i = 0; i < d; ++i) pf(&t->caps[s->id].exit_states, states[(size_t)b * d + i]);
            if (s->tokens.n == 1) s->first_token = clock;
            const int hit_eos = c->eos_token >= 0 && token == c->eos_token;
            if (hit_eos || s->tokens.n >= s->max_new) { s->finished = 1; s->finish = clock; }
            else s->next_input = token;
        }
        pi(&t->it_batch_off, (int32_t)t->ps_seq.n);
        ++iteration;
    }

    pf(&t->meta, clock); pf(&t->meta, total_idle);
    pf(&t->meta, cache.pool); pf(&t->meta, cache.n_free); pf(&t->meta, cache.peak);
    rc = EO_OK;
    *out = t;
    t = NULL;
fail:
    if (t) eo_transcript_free(t);
    for (int i = 0; i < n_running; ++i) { free(running[i].tokens.p); free(running[i].exit_layers.p); free(running[i].iter_out.p); }
    free(running); free(order); scratch_free(&ws); free(states); free(next); free(logits); free(kbuf); free(vbuf); free(ids);
    kv_destroy(&cache);
    return rc;
}

/* ------------------------------------------------------------------ */
/* oracle.cpp:14-127 -- plain per-sequence decoder and replay           */
/* ------------------------------------------------------------------ */
typedef struct { vf64* k; vf64* v; } plain_kv; /* per layer lists */

static void plain_layer(const eo_model* m, int layer, const double* h, plain_kv* kv, double* out, scratch_t* w) {
    const int d = m->d;
    const double scale = 1.0 / sqrt((double)d);
    matvec(layer_tensor(m, layer, 0), d, d, h, w->q);
    matvec(layer_tensor(m, layer, 1), d, d, h, w->k);
    matvec(layer_tensor(m, layer, 2), d, d, h, w->v);
    vf64* K = &kv->k[layer - 1];
    vf64* V = &kv->v[layer - 1];
    for (int i = 0; i < d; ++i) { pf(K, w->k[i]); pf(V, w->v[i]); }
    const int n = (int)(K->n / d);
    scratch_scores(w, n);
    for (int p = 0; p < n; ++p) {
        double acc = 0.0;
        for (int i = 0; i < d; ++i) acc += K->p[(size_t)p * d + i] * w->q[i];
        w->scores[p] = acc * scale;
    }
    softmax(w->scores, n, w->probs);
    for (int i = 0; i < d; ++i) w->att[i] = 0.0;
    for (int p = 0; p < n; ++p)
        for (int i = 0; i < d; ++i) w->att[i] += w->probs[p] * V->p[(size_t)p * d + i];
    matvec(layer_tensor(m, layer, 3), d, d, w->att, w->proj);
    for (int i = 0; i < d; ++i) w->mid[i] = h[i] + w->proj[i];
    matvec(layer_tensor(m, layer, 4), 4 * d, d, w->mid, w->up);
    for (int i = 0; i < 4 * d; ++i) if (w->up[i] < 0.0) w->up[i] = 0.0;
    matvec(layer_tensor(m, layer, 5), d, 4 * d, w->up, w->down);
    for (int i = 0; i < d; ++i) out[i] = w->mid[i] + w->down[i];
}

static plain_kv plain_kv_new(int L) {
    plain_kv kv;
    kv.k = (vf64*)calloc((size_t)L, sizeof(vf64));
    kv.v = (vf64*)calloc((size_t)L, sizeof(vf64));
    return kv;
}
static void plain_kv_free(plain_kv* kv, int L) {
    for (int i = 0; i < L; ++i) { free(kv->k[i].p); free(kv->v[i].p); }
    free(kv->k); free(kv->v);
}

int eo_reference_decode(const eo_model* m, const int32_t* prompt, int plen, int max_new, int eos, int32_t* out) {
    if (plen < 1 || max_new < 1) { set_err("reference_decode: bad args"); return -EO_INVALID_ARGUMENT; }
    const int L = m->L, d = m->d;
    scratch_t w; scratch_init(&w, 1, d);
    plain_kv kv = plain_kv_new(L);
    double* h = (double*)malloc(sizeof(double) * (size_t)d);
    double* o = (double*)malloc(sizeof(double) * (size_t)d);
    double* logits = (double*)malloc(sizeof(double) * (size_t)m->V);
    for (int j = 0; j + 1 < plen; ++j) {
        memcpy(h, m->emb + (size_t)prompt[j] * d, sizeof(double) * (size_t)d);
        for (int layer = 1; layer <= L; ++layer) { plain_layer(m, layer, h, &kv, o, &w); memcpy(h, o, sizeof(double) * (size_t)d); }
    }
    int n = 0, input = prompt[plen - 1];
    while (n < max_new) {
        memcpy(h, m->emb + (size_t)input * d, sizeof(double) * (size_t)d);
        for (int layer = 1; layer <= L; ++layer) { plain_layer(m, layer, h, &kv, o, &w); memcpy(h, o, sizeof(double) * (size_t)d); }
        matvec(m->lm, m->V, d, h, logits);
        const int tok = greedy_token(logits, m->V);
        out[n++] = tok;
        if (eos >= 0 && tok == eos) break;
        input = tok;
    }
    free(h); free(o); free(logits); plain_kv_free(&kv, L); scratch_free(&w);
    return n;
}

int eo_replay_sequence(const eo_model* m, const int32_t* prompt, int plen, const int32_t* exits, int n,
                       int32_t* tokens, double* exit_states, double* kv_k, double* kv_v) {
    const int L = m->L, d = m->d;
    for (int i = 0; i < n; ++i) if (exits[i] < 1 || exits[i] > L) { set_err("replay: exit layer outside [1, n_layers]"); return EO_INVALID_ARGUMENT; }
    scratch_t w; scratch_init(&w, 1, d);
    plain_kv kv = plain_kv_new(L);
    double* h = (double*)malloc(sizeof(double) * (size_t)d);
    double* o = (double*)malloc(sizeof(double) * (size_t)d);
    double* logits = (double*)malloc(sizeof(double) * (size_t)m->V);
    for (int j = 0; j + 1 < plen; ++j) {
        memcpy(h, m->emb + (size_t)prompt[j] * d, sizeof(double) * (size_t)d);
        for (int layer = 1; layer <= L; ++layer) { plain_layer(m, layer, h, &kv, o, &w); memcpy(h, o, sizeof(double) * (size_t)d); }
    }
    int input = prompt[plen - 1];
    for (int t = 0; t < n; ++t) {
        memcpy(h, m->emb + (size_t)input * d, sizeof(double) * (size_t)d);
        for (int layer = 1; layer <= exits[t]; ++layer) { plain_layer(m, layer, h, &kv, o, &w); memcpy(h, o, sizeof(double) * (size_t)d); }
        for (int layer = exits[t] + 1; layer <= L; ++layer) {
            matvec(layer_tensor(m, layer, 1), d, d, h, w.k);
            matvec(layer_tensor(m, layer, 2), d, d, h, w.v);
            for (int i = 0; i < d; ++i) { pf(&kv.k[layer - 1], w.k[i]); pf(&kv.v[layer - 1], w.v[i]); }
        }
        matvec(m->lm, m->V, d, h, logits);
        tokens[t] = greedy_token(logits, m->V);
        if (exit_states) memcpy(exit_states + (size_t)t * d, h, sizeof(double) * (size_t)d);
        input = tokens[t];
    }
    const int P = plen - 1 + n;
    if (kv_k && kv_v)
        for (int layer = 0; layer < L; ++layer) {
            memcpy(kv_k + (size_t)layer * P * d, kv.k[layer].p, sizeof(double) * (size_t)P * d);
            memcpy(kv_v + (size_t)layer * P * d, kv.v[layer].p, sizeof(double) * (size_t)P * d);
        }
    free(h); free(o); free(logits); plain_kv_free(&kv, L); scratch_free(&w);
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* decode session over a seeded KV prefix                               */
/* ------------------------------------------------------------------ */
typedef struct slow_session {
    const eo_model* m;
    eo_engine_config cfg;
    int B;
    kv_store cache;
    int* ids;
    int* next_input;
    scratch_t ws;
    double *states, *next, *logits, *kbuf, *vbuf;
} slow_session;

static slow_session* slow_session_create(const eo_model* m, const eo_engine_config* c, int B, const int32_t* first_tokens,
                              int prefix_len, int capacity, uint64_t kv_seed, const int32_t* seq_ids) {
    if (validate_config(m, c)) return NULL;
    const int L = c->n_layers, d = c->d_model;
    slow_session* s = (slow_session*)calloc(1, sizeof(slow_session));
    s->m = m; s->cfg = *c; s->B = B;
    int max_id = 0;
    for (int b = 0; b < B; ++b) if (seq_ids[b] > max_id) max_id = seq_ids[b];
    const int bpl = (capacity + c->block_capacity - 1) / c->block_capacity;
    int pool = c->pool_blocks;
    if (pool < bpl * L * B) pool = bpl * L * B;
    if (kv_init(&s->cache, d, L, pool, c->block_capacity, max_id + 1, 1)) { free(s); return NULL; }
    s->ids = (int*)malloc(sizeof(int) * (size_t)B);
    s->next_input = (int*)malloc(sizeof(int) * (size_t)B);
    double* kb = (double*)malloc(sizeof(double) * (size_t)d);
    double* vb = (double*)malloc(sizeof(double) * (size_t)d);
    for (int b = 0; b < B; ++b) {
        s->ids[b] = seq_ids[b];
        s->next_input[b] = first_tokens[b];
        kv_allocate(&s->cache, seq_ids[b], capacity);
        for (int p = 0; p < prefix_len; ++p) {
            for (int layer = 1; layer <= L; ++layer) {
                eo_kv_prefix_vector(kv_seed, L, seq_ids[b], layer, p, 0, d, c->round_bf16, kb);
                eo_kv_prefix_vector(kv_seed, L, seq_ids[b], layer, p, 1, d, c->round_bf16, vb);
                kv_append(&s->cache, seq_ids[b], layer, p, kb, vb);
            }
            kv_commit(&s->cache, seq_ids[b]);
        }
    }
    free(kb); free(vb);
    scratch_init(&s->ws, B, d);
    s->states = (double*)malloc(sizeof(double) * (size_t)B * d);
    s->next = (double*)malloc(sizeof(double) * (size_t)B * d);
    s->logits = (double*)malloc(sizeof(double) * (size_t)m->V);
    s->kbuf = (double*)malloc(sizeof(double) * (size_t)d);
    s->vbuf = (double*)malloc(sizeof(double) * (size_t)d);
    return s;
}

static void slow_session_free(slow_session* s) {
    if (!s) return;
    kv_destroy(&s->cache); scratch_free(&s->ws);
    free(s->ids); free(s->next_input); free(s->states); free(s->next); free(s->logits); free(s->kbuf); free(s->vbuf);
    free(s);
}

static int slow_session_step(slow_session* s, int forced, const double* fixed_conf, const int32_t* tokens_in,
                    int32_t* tokens, int32_t* accept, double* conf, double* h_exit) {
    const eo_model* m = s->m;
    const eo_engine_config* c = &s->cfg;
    const int L = c->n_layers, d = c->d_model, B = s->B;
    if (tokens_in) for (int b = 0; b < B; ++b) s->next_input[b] = tokens_in[b];
    for (int b = 0; b < B; ++b)
        memcpy(s->states + (size_t)b * d, m->emb + (size_t)s->next_input[b] * d, sizeof(double) * (size_t)d);
    unsigned char* status = (unsigned char*)calloc((size_t)B, 1);
    int* fa = (int*)calloc((size_t)B, sizeof(int));
    if (conf) for (int i = 0; i < L * B; ++i) conf[i] = NAN;
    int output_layer = L;
    int rc = EO_OK;
    for (int layer = 1; layer <= L; ++layer) {
        rc = layer_forward(m, layer, B, s->ids, s->states, &s->cache, &s->ws, s->next);
        if (rc) goto done;
        const double lambda = eo_threshold_at(c->lambda0, c->gamma, c->lambda_min, layer);
        int all = 1;
        for (int b = 0; b < B; ++b) {
            const double cf = (c->technique == EO_TECH_FIXED)
                                  ? fixed_conf[(size_t)(layer - 1) * B + b]
                                  : confidence(m, c, s->states + (size_t)b * d, s->next + (size_t)b * d, s->logits);
            if (conf) conf[(size_t)(layer - 1) * B + b] = cf;
            const int acc = decide(c, layer, cf, lambda);
            if (!status[b] && acc) { status[b] = 1; fa[b] = layer; }
            all = all && status[b];
        }
        memcpy(s->states, s->next, sizeof(double) * (size_t)B * d);
        if (forced > 0) { if (layer == forced) { output_layer = layer; break; } }
        else if (all) { output_layer = layer; break; }
    }
    rc = fill_skipped(m, &s->cache, B, s->ids, s->states, output_layer, s->kbuf, s->vbuf);
    if (rc) goto done;
    for (int b = 0; b < B; ++b) { rc = kv_commit(&s->cache, s->ids[b]); if (rc) goto done; }
    for (int b = 0; b < B; ++b) {
        matvec(m->lm, m->V, d, s->states + (size_t)b * d, s->logits);
        const int tok = greedy_token(s->logits, m->V);
        if (tokens) tokens[b] = tok;
        if (accept) accept[b] = fa[b] == 0 ? L : fa[b];
        if (h_exit) memcpy(h_exit + (size_t)b * d, s->states + (size_t)b * d, sizeof(double) * (size_t)d);
        s->next_input[b] = tok;
    }
done:
    free(status); free(fa);
    return rc ? -rc : output_layer;
}

static int slow_session_kv(const slow_session* s, int row, int layer, int pos, double* k, double* v) {
    const int id = s->ids[row];
    kv_store* cs = (kv_store*)&s->cache;
    if (layer < 1 || layer > s->cfg.n_layers || pos < 0 || pos >= cs->seqs[id].written[layer - 1]) { set_err("session_kv: not written"); return EO_INVALID_ARGUMENT; }
    memcpy(k, kv_slot(cs, 0, id, layer, pos), sizeof(double) * (size_t)s->cfg.d_model);
    memcpy(v, kv_slot(cs, 1, id, layer, pos), sizeof(double) * (size_t)s->cfg.d_model);
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* fast decode session (decoder-only model): the same decode_iteration */
/* restatement as slow_session, organised for large batches so the     */
/* free-running parity tests finish at the BASELINE configs (L=24,     */
/* d=1024, B=256, ctx 512+):                                            */
/*  * every dot product keeps the reference's left-to-right order     */
/*    (numerics.cpp:28-43, model.cpp:229-241); independent dots (16    */
/*    sequences of one weight row, 4 key positions of one query) are   */
/*    interleaved, never re-associated -> bit-identical results;       */
/*  * the seeded prefix is stored as its bf16 bits when round_bf16     */
/*    (exact: the values are bf16-representable), computed positions   */
/*    in fp64;                                                          */
/*  * work is split over host threads by output rows / sequences.      */
/* ------------------------------------------------------------------ */
#include <pthread.h>
#include <unistd.h>

#define FS_NB 16 /* sequences per interleaved dot group */

typedef struct fast_session fast_session;
typedef void (*fs_task)(fast_session* s, int lo, int hi, int tid);

struct fast_session {
    const eo_model* m;
    eo_engine_config cfg;
    int B, Bp, P, cap, L, d, nthreads;
    int *ids, *next_input, *committed, *written; /* written [B][L] */
    uint16_t *pk16, *pv16;                       /* [B][L][P][d] (round_bf16) */
    double *pk64, *pv64;                         /* [B][L][P][d] (otherwise) */
    double *tk, *tv;                             /* [B][L][cap-P][d] */
    double *states, *next, *xT, *q, *k, *v, *att, *mid, *up, *down, *logits;
    double* tscratch; /* per thread: scores[cap] probs[cap] rows[4][d] */
    int tstride;
    /* current task arguments */
    const double* w; int rows, cols; const double* x; double* y; int layer; int rc;
    uint64_t kv_seed;
    /* layer-level scheduling semantics: every row exits at its OWN first
       accept -- B independent decode_iterations of one sequence each */
    int per_seq;
    unsigned char* active; /* [B] rows still running layers this step */
};

static int fs_threads(void) {
    const char* e = getenv("EO_THREADS");
    int n = e ? atoi(e) : (int)sysconf(_SC_NPROCESSORS_ONLN);
    return n < 1 ? 1 : (n > 256 ? 256 : n);
}

typedef struct { fast_session* s; fs_task fn; int lo, hi, tid; } fs_arg;
static void* fs_entry(void* p) { fs_arg* a = (fs_arg*)p; a->fn(a->s, a->lo, a->hi, a->tid); return NULL; }
/* static split of [0, n) over the session's threads */
static void fs_parallel(fast_session* s, int n, fs_task fn) {
    int T = s->nthreads < n ? s->nthreads : n;
    if (T <= 1) { fn(s, 0, n, 0); return; }
    pthread_t th[256];
    fs_arg args[256];
    for (int t = 0; t < T; ++t) {
        args[t].s = s; args[t].fn = fn; args[t].tid = t;
        args[t].lo = (int)((long)n * t / T); args[t].hi = (int)((long)n * (t + 1) / T);
        if (t) pthread_create(&th[t], NULL, fs_entry, &args[t]);
    }
    fs_entry(&args[0]);
    for (int t = 1; t < T; ++t) pthread_join(th[t], NULL);
}

/* y[b][r] = sum_c w[r][c] * x[b][c] for all B sequences (matvec_batch, numerics.cpp:45-52):
   rows split over threads; 16 sequences per pass share each weight row (xT = x transposed) */
static void fs_transpose(fast_session* s, const double* x, int cols) {
    for (int b = 0; b < s->Bp; ++b)
        for (int c = 0; c < cols; ++c) s->xT[(size_t)c * s->Bp + b] = b < s->B ? x[(size_t)b * cols + c] : 0.0;
}
static void fs_mm_task(fast_session* s, int lo, int hi, int tid) {
    (void)tid;
    const int cols = s->cols, rows = s->rows, Bp = s->Bp, B = s->B;
    for (int jb = 0; jb < Bp; jb += FS_NB)
        for (int r = lo; r < hi; ++r) {
            const double* row = s->w + (size_t)r * cols;
            double acc[FS_NB];
            for (int j = 0; j < FS_NB; ++j) acc[j] = 0.0;
            const double* xt = s->xT + jb;
            for (int c = 0; c < cols; ++c) {
                const double wv = row[c];
                const double* xc = xt + (size_t)c * Bp;
                for (int j = 0; j < FS_NB; ++j) acc[j] += wv * xc[j];
            }
            for (int j = 0; j < FS_NB && jb + j < B; ++j) s->y[(size_t)(jb + j) * rows + r] = acc[j];
        }
}
static void fs_mm(fast_session* s, const double* w, int rows, int cols, const double* x, double* y) {
    fs_transpose(s, x, cols);
    s->w = w; s->rows = rows; s->cols = cols; s->y = y;
    fs_parallel(s, rows, fs_mm_task);
}

/* K/V row at (b, layer, pos): prefix rows are converted from bf16 into buf (exact) */
static const double* fs_row(const fast_session* s, int which, int b, int layer, int pos, double* buf) {
    const int d = s->d, L = s->L;
    if (pos < s->P) {
        const size_t off = (((size_t)b * L + (layer - 1)) * s->P + pos) * d;
        if (s->pk16) {
            const uint16_t* src = (which ? s->pv16 : s->pk16) + off;
            for (int i = 0; i < d; ++i) {
                uint64_t u = (uint64_t)src[i] << 16;
                uint32_t u32 = (uint32_t)u;
                float f;
                memcpy(&f, &u32, 4);
                buf[i] = (double)f;
            }
            return buf;
        }
        return (which ? s->pv64 : s->pk64) + off;
    }
    return (which ? s->tv : s->tk) + (((size_t)b * L + (layer - 1)) * (s->cap - s->P) + (pos - s->P)) * d;
}
static double* fs_tail(fast_session* s, int which, int b, int layer, int pos) {
    return (double*)fs_row(s, which, b, layer, pos, NULL);
}

/* KvStore::append invariants (kv_cache.cpp:108-145) */
static int fs_append(fast_session* s, int b, int layer, int pos, const double* k, const double* v) {
    int* w = &s->written[(size_t)b * s->L + layer - 1];
    if (pos < *w) { set_err("append: slot already written"); return EO_RUNTIME_ERROR; }
    if (pos > *w) { set_err("append: position gap"); return EO_RUNTIME_ERROR; }
    if (pos >= s->cap) { set_err("append: position exceeds reserved capacity"); return EO_KV_OUT_OF_MEMORY; }
    memcpy(fs_tail(s, 0, b, layer, pos), k, sizeof(double) * (size_t)s->d);
    memcpy(fs_tail(s, 1, b, layer, pos), v, sizeof(double) * (size_t)s->d);
    ++*w;
    return EO_OK;
}

/* attention of sequences [lo, hi) (model.cpp:223-243): append K,V, scores, softmax, P.V */
static void fs_attn_task(fast_session* s, int lo, int hi, int tid) {
    const int d = s->d, layer = s->layer;
    const double scale = 1.0 / sqrt((double)d);
    double* scores = s->tscratch + (size_t)tid * s->tstride;
    double* probs = scores + s->cap;
    double* rb = probs + s->cap; /* 4 rows of d */
    for (int b = lo; b < hi; ++b) {
        if (s->per_seq && !s->active[b]) continue;
        const int pos = s->committed[b];
        int rc = fs_append(s, b, layer, pos, s->k + (size_t)b * d, s->v + (size_t)b * d);
        if (rc) { s->rc = rc; return; }
        const int n = pos + 1;
        const double* q = s->q + (size_t)b * d;
        int p = 0;
        for (; p + 4 <= n; p += 4) {
            const double* k0 = fs_row(s, 0, b, layer, p, rb);
            const double* k1 = fs_row(s, 0, b, layer, p + 1, rb + d);
            const double* k2 = fs_row(s, 0, b, layer, p + 2, rb + 2 * d);
            const double* k3 = fs_row(s, 0, b, layer, p + 3, rb + 3 * d);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            for (int i = 0; i < d; ++i) {
                a0 += k0[i] * q[i]; a1 += k1[i] * q[i]; a2 += k2[i] * q[i]; a3 += k3[i] * q[i];
            }
            scores[p] = a0 * scale; scores[p + 1] = a1 * scale; scores[p + 2] = a2 * scale; scores[p + 3] = a3 * scale;
        }
        for (; p < n; ++p) {
            const double* key = fs_row(s, 0, b, layer, p, rb);
            double acc = 0.0;
            for (int i = 0; i < d; ++i) acc += key[i] * q[i];
            scores[p] = acc * scale;
        }
        rc = softmax(scores, n, probs);
        if (rc) { s->rc = rc; return; }
        double* a = s->att + (size_t)b * d;
        for (int i = 0; i < d; ++i) a[i] = 0.0;
        for (p = 0; p < n; ++p) {
            const double* val = fs_row(s, 1, b, layer, p, rb);
            const double weight = probs[p];
            for (int i = 0; i < d; ++i) a[i] += weight * val[i];
        }
    }
}

/* layer_forward (model.cpp:197-272) for the whole batch: states -> next */
static int fs_layer(fast_session* s, int layer) {
    const eo_model* m = s->m;
    const int d = s->d, B = s->B;
    fs_mm(s, layer_tensor(m, layer, 0), d, d, s->states, s->q);
    fs_mm(s, layer_tensor(m, layer, 1), d, d, s->states, s->k);
    fs_mm(s, layer_tensor(m, layer, 2), d, d, s->states, s->v);
    s->layer = layer; s->rc = EO_OK;
    fs_parallel(s, B, fs_attn_task);
    if (s->rc) return s->rc;
    fs_mm(s, layer_tensor(m, layer, 3), d, d, s->att, s->down);
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < d; ++i) s->mid[(size_t)b * d + i] = s->states[(size_t)b * d + i] + s->down[(size_t)b * d + i];
    fs_mm(s, layer_tensor(m, layer, 4), 4 * d, d, s->mid, s->up);
    for (size_t i = 0; i < (size_t)B * 4 * d; ++i) if (s->up[i] < 0.0) s->up[i] = 0.0;
    fs_mm(s, layer_tensor(m, layer, 5), d, 4 * d, s->up, s->down);
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < d; ++i) s->next[(size_t)b * d + i] = s->mid[(size_t)b * d + i] + s->down[(size_t)b * d + i];
    return EO_OK;
}

/* prefix generation, split over sequences */
static void fs_prefix_task(fast_session* s, int lo, int hi, int tid) {
    (void)tid;
    const int d = s->d, L = s->L;
    double* buf = (double*)malloc(sizeof(double) * (size_t)d);
    for (int b = lo; b < hi; ++b)
        for (int layer = 1; layer <= L; ++layer)
            for (int p = 0; p < s->P; ++p)
                for (int kind = 0; kind < 2; ++kind) {
                    eo_kv_prefix_vector(s->kv_seed, L, s->ids[b], layer, p, kind, d, s->cfg.round_bf16, buf);
                    const size_t off = (((size_t)b * L + (layer - 1)) * s->P + p) * d;
                    if (s->pk16) {
                        uint16_t* dst = (kind ? s->pv16 : s->pk16) + off;
                        for (int i = 0; i < d; ++i) dst[i] = eo_bf16_bits(buf[i]);
                    } else {
                        memcpy((kind ? s->pv64 : s->pk64) + off, buf, sizeof(double) * (size_t)d);
                    }
                }
    free(buf);
}

static fast_session* fast_session_create(const eo_model* m, const eo_engine_config* c, int B,
                                         const int32_t* first_tokens, int P, int capacity, uint64_t kv_seed,
                                         const int32_t* seq_ids) {
    if (B < 1) { set_err("decode_iteration: empty batch"); return NULL; }
    if (P < 0 || capacity < P + 1) { set_err("session: capacity must exceed the prefix"); return NULL; }
    fast_session* s = (fast_session*)calloc(1, sizeof(fast_session));
    const int L = c->n_layers, d = c->d_model;
    s->m = m; s->cfg = *c; s->B = B; s->Bp = (B + FS_NB - 1) / FS_NB * FS_NB; s->P = P; s->L = L; s->d = d;
    /* KvStore::allocate reserves whole blocks (kv_cache.cpp:86-91) */
    s->cap = (capacity + c->block_capacity - 1) / c->block_capacity * c->block_capacity;
    s->nthreads = fs_threads();
    s->ids = (int*)malloc(sizeof(int) * (size_t)B);
    s->next_input = (int*)malloc(sizeof(int) * (size_t)B);
    s->committed = (int*)malloc(sizeof(int) * (size_t)B);
    s->written = (int*)malloc(sizeof(int) * (size_t)B * L);
    for (int b = 0; b < B; ++b) {
        s->ids[b] = seq_ids[b]; s->next_input[b] = first_tokens[b]; s->committed[b] = P;
        for (int l = 0; l < L; ++l) s->written[(size_t)b * L + l] = P;
    }
    const size_t npre = (size_t)B * L * P * d, ntail = (size_t)B * L * (s->cap - P) * d;
    if (c->round_bf16) {
        s->pk16 = (uint16_t*)malloc(sizeof(uint16_t) * (npre ? npre : 1));
        s->pv16 = (uint16_t*)malloc(sizeof(uint16_t) * (npre ? npre : 1));
    } else {
        s->pk64 = (double*)malloc(sizeof(double) * (npre ? npre : 1));
        s->pv64 = (double*)malloc(sizeof(double) * (npre ? npre : 1));
    }
    s->tk = (double*)calloc(ntail, sizeof(double));
    s->tv = (double*)calloc(ntail, sizeof(double));
    if ((!s->pk16 && !s->pk64) || !s->tk || !s->tv) { set_err("session: out of host memory"); return NULL; }
    s->kv_seed = kv_seed;
    fs_parallel(s, B, fs_prefix_task);
    const size_t bd = (size_t)B * d;
    s->states = (double*)malloc(sizeof(double) * bd);
    s->next = (double*)malloc(sizeof(double) * bd);
    s->q = (double*)malloc(sizeof(double) * bd);
    s->k = (double*)malloc(sizeof(double) * bd);
    s->v = (double*)malloc(sizeof(double) * bd);
    s->att = (double*)malloc(sizeof(double) * bd);
    s->mid = (double*)malloc(sizeof(double) * bd);
    s->down = (double*)malloc(sizeof(double) * bd);
    s->up = (double*)malloc(sizeof(double) * bd * 4);
    s->xT = (double*)malloc(sizeof(double) * (size_t)s->Bp * 4 * d);
    s->logits = (double*)malloc(sizeof(double) * (size_t)B * m->V);
    s->tstride = 2 * s->cap + 4 * d;
    s->tscratch = (double*)malloc(sizeof(double) * (size_t)s->tstride * s->nthreads);
    s->active = (unsigned char*)calloc((size_t)B, 1);
    return s;
}

static void fast_session_free(fast_session* s) {
    if (!s) return;
    free(s->ids); free(s->next_input); free(s->committed); free(s->written);
    free(s->pk16); free(s->pv16); free(s->pk64); free(s->pv64); free(s->tk); free(s->tv);
    free(s->states); free(s->next); free(s->q); free(s->k); free(s->v); free(s->att); free(s->mid); free(s->down);
    free(s->up); free(s->xT); free(s->logits); free(s->tscratch); free(s->active);
    free(s);
}

/* softmax_response_confidence per sequence over s->logits */
static void fs_conf_task(fast_session* s, int lo, int hi, int tid) {
    (void)tid;
    for (int b = lo; b < hi; ++b)
        s->down[b] = eo_softmax_response_confidence(s->logits + (size_t)b * s->m->V, s->m->V);
}

/* layer loop with per-row exits: rows run layers until their own first accept (or L); a row's
   state freezes at its exit layer (s->states), fa[b] = its exit layer */
static int fs_per_seq_layers(fast_session* s, const double* fixed_conf, double* conf, int* fa) {
    const eo_model* m = s->m;
    const eo_engine_config* c = &s->cfg;
    const int L = c->n_layers, d = c->d_model, B = s->B, V = m->V;
    int n_active = B;
    for (int b = 0; b < B; ++b) s->active[b] = 1;
    for (int layer = 1; layer <= L && n_active > 0; ++layer) {
        int rc = fs_layer(s, layer);
        if (rc) return rc;
        const double lambda = eo_threshold_at(c->lambda0, c->gamma, c->lambda_min, layer);
        if (c->technique == EO_TECH_SOFTMAX) {
            fs_mm(s, m->lm, V, d, s->next, s->logits);
            fs_parallel(s, B, fs_conf_task);
        }
        for (int b = 0; b < B; ++b) {
            if (!s->active[b]) continue;
            double cf;
            if (c->technique == EO_TECH_FIXED) cf = fixed_conf[(size_t)(layer - 1) * B + b];
            else if (c->technique == EO_TECH_SOFTMAX) cf = s->down[b];
            else cf = confidence(m, c, s->states + (size_t)b * d, s->next + (size_t)b * d, NULL);
            if (conf) conf[(size_t)(layer - 1) * B + b] = cf;
            memcpy(s->states + (size_t)b * d, s->next + (size_t)b * d, sizeof(double) * (size_t)d);
            if (decide(c, layer, cf, lambda) || layer == L) {
                fa[b] = layer;
                s->active[b] = 0;
                --n_active;
            }
        }
    }
    return EO_OK;
}

/* decode_iteration (engine.cpp:208-310) -- same contract as slow_session_step */
static int fast_session_step(fast_session* s, int forced, const double* fixed_conf, const int32_t* tokens_in,
                             int32_t* tokens, int32_t* accept, double* conf, double* h_exit) {
    const eo_model* m = s->m;
    const eo_engine_config* c = &s->cfg;
    const int L = c->n_layers, d = c->d_model, B = s->B, V = m->V;
    if (tokens_in) for (int b = 0; b < B; ++b) s->next_input[b] = tokens_in[b];
    for (int b = 0; b < B; ++b) {
        if (s->next_input[b] < 0 || s->next_input[b] >= V) { set_err("embed: token id outside vocab"); return -EO_INVALID_ARGUMENT; }
        memcpy(s->states + (size_t)b * d, m->emb + (size_t)s->next_input[b] * d, sizeof(double) * (size_t)d);
    }
    unsigned char* status = (unsigned char*)calloc((size_t)B, 1);
    int* fa = (int*)calloc((size_t)B, sizeof(int));
    double* cf_b = (double*)malloc(sizeof(double) * (size_t)B);
    if (conf) for (int i = 0; i < L * B; ++i) conf[i] = NAN;
    int output_layer = L, rc = EO_OK;
    if (s->per_seq) { rc = fs_per_seq_layers(s, fixed_conf, conf, fa); if (rc) goto done; goto tail; }
    for (int layer = 1; layer <= L; ++layer) {
        rc = fs_layer(s, layer);
        if (rc) goto done;
        const double lambda = eo_threshold_at(c->lambda0, c->gamma, c->lambda_min, layer);
        if (c->technique == EO_TECH_SOFTMAX) {
            fs_mm(s, m->lm, V, d, s->next, s->logits);
            fs_parallel(s, B, fs_conf_task);
            memcpy(cf_b, s->down, sizeof(double) * (size_t)B);
        }
        int all = 1;
        for (int b = 0; b < B; ++b) {
            double cf;
            if (c->technique == EO_TECH_FIXED) cf = fixed_conf[(size_t)(layer - 1) * B + b];
            else if (c->technique == EO_TECH_SOFTMAX) cf = cf_b[b];
            else cf = confidence(m, c, s->states + (size_t)b * d, s->next + (size_t)b * d, NULL);
            if (conf) conf[(size_t)(layer - 1) * B + b] = cf;
            const int acc = decide(c, layer, cf, lambda);
            if (!status[b] && acc) { status[b] = 1; fa[b] = layer; }
            all = all && status[b];
        }
        memcpy(s->states, s->next, sizeof(double) * (size_t)B * d);
        if (forced > 0) { if (layer == forced) { output_layer = layer; break; } }
        else if (all) { output_layer = layer; break; }
    }
    /* fill_skipped (kv_cache.cpp:222-234): K_j, V_j = W_k^(j) h_e, W_v^(j) h_e */
    if (0) {
    tail:
        /* per-row exits: each row's skipped layers from its own exit state */
        output_layer = 0;
        for (int b = 0; b < B; ++b) if (fa[b] > output_layer) output_layer = fa[b];
        for (int layer = 2; layer <= L; ++layer) {
            int need = 0;
            for (int b = 0; b < B; ++b) need |= fa[b] < layer;
            if (!need) continue;
            fs_mm(s, layer_tensor(m, layer, 1), d, d, s->states, s->k);
            fs_mm(s, layer_tensor(m, layer, 2), d, d, s->states, s->v);
            for (int b = 0; b < B; ++b)
                if (fa[b] < layer) {
                    rc = fs_append(s, b, layer, s->committed[b], s->k + (size_t)b * d, s->v + (size_t)b * d);
                    if (rc) goto done;
                }
        }
        goto commit;
    }
    for (int layer = output_layer + 1; layer <= L; ++layer) {
        fs_mm(s, layer_tensor(m, layer, 1), d, d, s->states, s->k);
        fs_mm(s, layer_tensor(m, layer, 2), d, d, s->states, s->v);
        for (int b = 0; b < B; ++b) {
            rc = fs_append(s, b, layer, s->committed[b], s->k + (size_t)b * d, s->v + (size_t)b * d);
            if (rc) goto done;
        }
    }
commit:
    /* KvStore::commit (kv_cache.cpp:165-180) */
    for (int b = 0; b < B; ++b) {
        for (int l = 0; l < L; ++l)
            if (s->written[(size_t)b * L + l] != s->committed[b] + 1) { set_err("commit: layer %d incomplete", l + 1); rc = EO_RUNTIME_ERROR; goto done; }
        ++s->committed[b];
    }
    /* lm_head_logits + greedy_token (engine.cpp:280-306) */
    fs_mm(s, m->lm, V, d, s->states, s->logits);
    for (int b = 0; b < B; ++b) {
        const int tok = greedy_token(s->logits + (size_t)b * V, V);
        if (tokens) tokens[b] = tok;
        if (accept) accept[b] = fa[b] == 0 ? L : fa[b];
        if (h_exit) memcpy(h_exit + (size_t)b * d, s->states + (size_t)b * d, sizeof(double) * (size_t)d);
        s->next_input[b] = tok;
    }
done:
    free(status); free(fa); free(cf_b);
    return rc ? -rc : output_layer;
}

static int fast_session_kv(const fast_session* s, int row, int layer, int pos, double* k, double* v) {
    if (row < 0 || row >= s->B || layer < 1 || layer > s->L || pos < 0 || pos >= s->written[(size_t)row * s->L + layer - 1]) {
        set_err("session_kv: not written");
        return EO_INVALID_ARGUMENT;
    }
    double* buf = (double*)malloc(sizeof(double) * (size_t)s->d);
    memcpy(k, fs_row(s, 0, row, layer, pos, buf), sizeof(double) * (size_t)s->d);
    memcpy(v, fs_row(s, 1, row, layer, pos, buf), sizeof(double) * (size_t)s->d);
    free(buf);
    return EO_OK;
}

/* ---- public session API: the fast path for the decoder-only model, the per-sequence
 *      restatement for T5 mode (cross-attention lives in layer_forward) ---- */
struct eo_session {
    slow_session* slow;
    fast_session* fast;
};

eo_session* eo_session_create(const eo_model* m, const eo_engine_config* c, int B, const int32_t* first_tokens,
                              int prefix_len, int capacity, uint64_t kv_seed, const int32_t* seq_ids) {
    if (validate_config(m, c)) return NULL;
    eo_session* s = (eo_session*)calloc(1, sizeof(eo_session));
    const char* slow = getenv("EO_SLOW_SESSION");
    if (m->enc_len > 0 || m->n_heads > 1 || (slow && atoi(slow)))
        s->slow = slow_session_create(m, c, B, first_tokens, prefix_len, capacity, kv_seed, seq_ids);
    else
        s->fast = fast_session_create(m, c, B, first_tokens, prefix_len, capacity, kv_seed, seq_ids);
    if (!s->slow && !s->fast) { free(s); return NULL; }
    return s;
}
void eo_session_free(eo_session* s) {
    if (!s) return;
    if (s->slow) slow_session_free(s->slow);
    if (s->fast) fast_session_free(s->fast);
    free(s);
}
int eo_session_step(eo_session* s, int forced, const double* fixed_conf, const int32_t* tokens_in, int32_t* tokens,
                    int32_t* accept, double* conf, double* h_exit) {
    return s->fast ? fast_session_step(s->fast, forced, fixed_conf, tokens_in, tokens, accept, conf, h_exit)
                   : slow_session_step(s->slow, forced, fixed_conf, tokens_in, tokens, accept, conf, h_exit);
}
int eo_session_set_per_seq_exit(eo_session* s, int on) {
    if (!s->fast) { set_err("per-sequence exits: decoder-only sessions only"); return EO_INVALID_ARGUMENT; }
    s->fast->per_seq = on != 0;
    return EO_OK;
}
int eo_session_kv(const eo_session* s, int row, int layer, int pos, double* k, double* v) {
    return s->fast ? fast_session_kv(s->fast, row, layer, pos, k, v) : slow_session_kv(s->slow, row, layer, pos, k, v);
}

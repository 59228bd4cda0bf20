/*
 * exitlab_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement ("port") of the reference's batched early-exit decode path,
 * used as the parity checker for the B200 engine.  Only tests/, smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library; the
 * product (paper_2407_20272_b200) never links or calls it.
 *
 * Every function follows the reference op-for-op in fp64 (same loop order, no
 * FMA contraction) so that it is BIT-EXACT with /root/reference built from
 * source (oracle/_ref); tests/test_oracle_cpu.py pins that, and pins it against
 * the committed golden fixtures under tests/golden/.
 *
 * Reference anchors (paths relative to /root/reference/proj):
 *   numerics      src/numerics.cpp:28-143
 *   model         src/model.cpp:37-59 (seeded), 171-299 (embed/layer/kv/lm/greedy)
 *   kv store      src/kv_cache.cpp:40-234
 *   exit policy   src/exit_policy.cpp:50-115
 *   engine        src/engine.cpp:47-75 (status vector), 110-330 (run)
 *   workload      src/workload.cpp:15-89
 *   oracle        src/oracle.cpp:14-127 (plain_layer, reference_decode, replay)
 */
#ifndef EXITLAB_ORACLE_H
#define EXITLAB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same values as the product's EL_* codes) */
#define EO_OK 0
#define EO_INVALID_ARGUMENT 1
#define EO_RUNTIME_ERROR 2
#define EO_KV_OUT_OF_MEMORY 3
#define EO_LOGIC_ERROR 4

/* technique kinds (same values as the product's EL_TECH_*) */
#define EO_TECH_SOFTMAX 0
#define EO_TECH_STATE 1
#define EO_TECH_CLASSIFIER 2
#define EO_TECH_NEVER 3
#define EO_TECH_ALWAYS_AT 4
#define EO_TECH_FIXED 5 /* injected confidences (test harness) */

const char* eo_last_error(void);

/* ---- numerics (numerics.cpp:94-143) ---- */
uint64_t eo_splitmix64_at(uint64_t seed, uint64_t index);
double eo_uniform01_at(uint64_t seed, uint64_t index);
void eo_seeded_matrix(int rows, int cols, uint64_t seed, double* out);
void eo_seeded_vector(int len, uint64_t seed, double* out);
/* RNE rounding of an fp64 value to the nearest bf16, returned as fp64 */
double eo_round_bf16(double x);
uint16_t eo_bf16_bits(double x);

/* ---- model ---- */
typedef struct eo_model eo_model;
eo_model* eo_model_seeded(int n_layers, int d_model, int vocab, uint64_t seed, int round_bf16);
/* T5-mode extension (north_star (1); no counterpart in the reference -- parity of this
   mode is pinned only by this restatement): a cross-attention sub-layer over
   `encoder_len` synthetic encoder states per sequence after the self-attention
   residual.  encoder_len = 0 is exactly eo_model_seeded. */
eo_model* eo_model_seeded_t5(int n_layers, int d_model, int vocab, uint64_t seed, int round_bf16, int encoder_len);
uint64_t eo_encoder_seed(uint64_t model_seed);
void eo_encoder_state(const eo_model* m, int seq_id, int t, double* out);
/* Extension: split self- (and in T5 mode cross-) attention into n_heads heads (d_model / n_heads
   features each, own softmax, scale 1 / sqrt(d_model / n_heads)); the reference has one head. */
int eo_model_set_heads(eo_model* m, int n_heads);
/* T5 mode: a real encoder stack of n bidirectional norm-free layers (own seeded weights, tags
   4 + 10L + 6i + k) over seeded encoder input ids replaces the seeded encoder states. */
int eo_model_set_encoder_layers(eo_model* m, int n);
int eo_encoder_token(const eo_model* m, int seq_id, int t);
void eo_model_free(eo_model* m);
/* which: 0 embedding, 1 lm_head, 2 probe_w, 3 probe_b, 4+k: layer tensor k in
 * {q,k,v,o,up,down}; layer is 1-based (ignored for globals). Copies into out. */
int eo_model_tensor(const eo_model* m, int which, int layer, double* out, int64_t cap);

/* ---- workload (workload.cpp:58-89) ---- */
typedef struct {
    int n_requests;
    double mean_interarrival;
    int prompt_len_min, prompt_len_max;
    int output_len_min, output_len_max;
    uint64_t seed;
    int vocab_size;
    int eos_token;
} eo_gen_params;
/* returns total prompt tokens; fills arrival[n], prompt_off[n+1], prompt[], max_new[n]
 * when the pointers are non-null (call once with nulls to size) */
int64_t eo_gen_workload(const eo_gen_params* p, double* arrival, int32_t* prompt_off,
                        int32_t* prompt, int32_t* max_new);

/* ---- engine ---- */
typedef struct {
    int n_layers, d_model, vocab_size;
    uint64_t model_seed;
    int technique, exit_layer;
    double lambda0, gamma, lambda_min;
    double c_layer_fixed, c_layer_per_seq, c_fill_per_seq_layer;
    double c_check_softmax, c_check_classifier, c_check_state;
    int max_batch, pool_blocks, block_capacity, eos_token;
    int capture_kv;
    int round_bf16;
    int64_t synthetic_kv_seed; /* <0: real prefill; >=0: seeded KV prefix */
} eo_engine_config;

typedef struct eo_transcript eo_transcript;
/* Drives the workload like Engine::run (engine.cpp:110-330). fixed_conf (may be
 * null) is read for EO_TECH_FIXED as conf[(iteration * L + layer-1) * max_batch + slot]
 * with n_fixed_iters iterations available. */
int eo_engine_run(const eo_model* m, const eo_engine_config* cfg, int n_req,
                  const double* arrival, const int32_t* prompt_off, const int32_t* prompt,
                  const int32_t* max_new, const double* fixed_conf, int n_fixed_iters,
                  eo_transcript** out);
void eo_transcript_free(eo_transcript* t);
/* flat fields (shared with the product and the reference wrapper):
 * i32: pf_seq pf_positions it_output_layer it_batch_off ps_seq ps_accept ps_token
 *      sq_id sq_max_new sq_prompt_off sq_prompt sq_tok_off sq_tokens sq_exit_layers
 *      sq_iter_out
 * f64: pf_clock pf_charge it_clock it_charge sq_arrival sq_first sq_finish
 *      meta (final_clock, total_idle, pool_blocks, free_blocks, peak_blocks)
 *      it_conf (per iteration, [L][batch] confidences; NaN where not computed) */
int64_t eo_transcript_len(const eo_transcript* t, const char* field);
int eo_transcript_get_i32(const eo_transcript* t, const char* field, int32_t* out);
int eo_transcript_get_f64(const eo_transcript* t, const char* field, double* out);
/* kv capture (capture_kv): K/V of seq at layer (1-based) for all committed
 * positions ([committed][d]) and the exit states ([tokens][d]) */
int eo_transcript_kv(const eo_transcript* t, int seq_id, int layer, double* k, double* v,
                     int64_t cap);
/* block table [L][bpl] of a captured sequence at eviction; returns bpl (<0 on error) */
int eo_transcript_block_table(const eo_transcript* t, int seq_id, int32_t* out, int64_t cap);
int eo_transcript_exit_states(const eo_transcript* t, int seq_id, double* out, int64_t cap);

/* ---- single-function checks ---- */
double eo_softmax_response_confidence(const double* logits, int n);
double eo_state_similarity_confidence(const double* a, const double* b, int n);
double eo_classifier_confidence(const double* h, const double* w, double b, int n);
double eo_threshold_at(double lambda0, double gamma, double lambda_min, int layer);
/* ExitStatusVector trace: conf[L][B] > lambda[layer-1] per layer; returns the
 * output layer, fills first_accept[B] (fallback L) (engine.cpp:47-75) */
int eo_status_trace(int batch, int n_layers, const double* conf, const double* lambdas,
                    int32_t* first_accept);
/* KvStore LIFO block tables after a sequence of ops: op>0 allocate(id=op-1,
 * capacity=caps[i]), op<0 release(id=-op-1); table out is [n_ids][L][bpl_max]
 * (-1 padded). Returns free count at the end or <0 on error. */
int eo_kv_block_trace(int n_layers, int pool_blocks, int block_capacity, int n_ops,
                      const int32_t* ops, const int32_t* caps, int n_ids, int bpl_max,
                      int32_t* tables);

/* ---- single-sequence oracles (oracle.cpp:60-127) ---- */
int eo_reference_decode(const eo_model* m, const int32_t* prompt, int prompt_len,
                        int max_new, int eos, int32_t* tokens_out);
/* replay: per-token exit layers; outputs tokens[n], exit_states[n][d],
 * kv_k/kv_v[L][prompt_len-1+n][d] */
int eo_replay_sequence(const eo_model* m, const int32_t* prompt, int prompt_len,
                       const int32_t* exits, int n, int32_t* tokens, double* exit_states,
                       double* kv_k, double* kv_v);

/* ---- decode session: fixed batch, seeded KV prefix (bench workload) ----
 * Restates the decode_iteration body (engine.cpp:208-310) for B sequences whose
 * KV already holds prefix_len seeded positions. */
typedef struct eo_session eo_session;
eo_session* eo_session_create(const eo_model* m, const eo_engine_config* cfg, int batch,
                              const int32_t* first_tokens, int prefix_len, int capacity,
                              uint64_t kv_seed, const int32_t* seq_ids);
void eo_session_free(eo_session* s);
/* one iteration; forced_output_layer>0 overrides the exit decision (replay).
 * tokens_in (may be null) overrides the inputs (teacher forcing).
 * outputs: tokens[B], accept[B], conf[L][B] (NaN when not computed), h_exit[B][d];
 * returns the output layer (<0 on error). */
int eo_session_step(eo_session* s, int forced_output_layer, const double* fixed_conf,
                    const int32_t* tokens_in, int32_t* tokens, int32_t* accept, double* conf,
                    double* h_exit);
/* layer-level scheduling semantics: every row exits at its own first accept (B independent
 * single-sequence decode iterations) */
int eo_session_set_per_seq_exit(eo_session* s, int on);
/* copy K/V at (row, layer, position) */
int eo_session_kv(const eo_session* s, int row, int layer, int position, double* k, double* v);

/* seeded KV prefix value: the vector written at (seq, layer, position, kind 0=K 1=V) */
void eo_kv_prefix_vector(uint64_t kv_seed, int n_layers, int seq, int layer, int position,
                         int kind, int d, int round_bf16, double* out);

#ifdef __cplusplus
}
#endif
#endif

/*
 * exitlab_b200.h -- C ABI of the B200-native batched early-exit decode engine.
 *
 * Drop-in boundary for the reference's engine and exit-criterion API
 * (/root/reference/proj, "exitlab"). Plain pointers and sizes only; every
 * function returns an EL_* status code (mapped 1:1 onto the reference's
 * exception classes) and leaves a message in
 * el_last_error().  Host buffers are always caller-owned.
 *
 * Reference interface each entry point replaces (paths under proj/):
 *   el_engine_create        Engine::Engine(EngineConfig[, ModelWeights])   include/exitlab/engine.hpp:135-136
 *                           (+ ModelWeights::seeded, model.hpp:46; EngineConfig::validate engine.cpp:31-45)
 *   el_engine_destroy       Engine::~Engine
 *   el_engine_run           Transcript Engine::run(const Workload&) const  include/exitlab/engine.hpp:141
 *   el_transcript_*         Transcript / IterationRecord / SequenceRecord  include/exitlab/engine.hpp:67-123
 *   el_session_begin        admission of a fixed batch (engine.cpp:183-206) with a seeded KV prefix in place of
 *                           prefill (engine.cpp:166-181)
 *   el_decode_iteration     the decode_iteration body (engine.cpp:208-310): layer_forward (model.hpp:64-66),
 *                           decide + *_confidence + threshold_at (exit_policy.hpp:46-70),
 *                           ExitStatusVector::observe_layer (engine.hpp:53), fill_skipped (kv_cache.hpp:112-115),
 *                           KvStore::commit (kv_cache.hpp:62), lm_head_logits + greedy_token (model.hpp:73-76)
 *   el_decode_run           the same, n iterations back to back on the device (no host round trip)
 *   el_set_fixed_confidences  test harness: ExitEvidence replaced by injected confidences (decide's "> lambda")
 *   el_session_kv           KvStore::view(seq, layer, upto).key/value (kv_cache.hpp:56, 24-36)
 *   el_session_block_table  KvStore block_table (kv_cache.hpp:83), read back from the device
 *   el_kv_block_trace       KvStore::allocate / release LIFO order (kv_cache.cpp:53-55, 78-106, 182-194)
 *   el_model_tensor         ModelWeights tensors (model.hpp:38-55), bf16 on the device
 *   el_*metrics*            MetricsReport compute_metrics (metrics.hpp:20-40, metrics.cpp:13-58)
 *   el_kv_* el_layer_forward el_kv_fill el_exit_confidence el_greedy_tokens: the sub-engine API
 *                           (KvStore, layer_forward, fill_skipped, decide, greedy_token; see below)
 */
#ifndef EXITLAB_B200_H
#define EXITLAB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: reference exception class in brackets */
#define EL_OK 0
#define EL_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define EL_RUNTIME_ERROR 2    /* std::runtime_error (invariant violations) */
#define EL_KV_OUT_OF_MEMORY 3 /* exitlab::KvOutOfMemory */
#define EL_LOGIC_ERROR 4      /* std::logic_error (empty batch) */
#define EL_CUDA_ERROR 6       /* device / driver failure (no reference counterpart) */

/* ExitTechnique kinds (exit_policy.hpp:14-31) + the injected-confidence harness */
#define EL_TECH_SOFTMAX 0
#define EL_TECH_STATE 1
#define EL_TECH_CLASSIFIER 2
#define EL_TECH_NEVER 3
#define EL_TECH_ALWAYS_AT 4
#define EL_TECH_FIXED 5

/* EngineConfig (engine.hpp:30-42) + ModelConfig (model.hpp:18-25) +
 * ThresholdSchedule (exit_policy.hpp:36-42) + CostModel (engine.hpp:18-28). */
typedef struct {
    int n_layers, d_model, vocab_size;
    uint64_t model_seed;
    int technique, exit_layer;
    double lambda0, gamma, lambda_min;
    double c_layer_fixed, c_layer_per_seq, c_fill_per_seq_layer;
    double c_check_softmax, c_check_classifier, c_check_state;
    int max_batch, pool_blocks, block_capacity, eos_token;
    int capture_kv;
    int round_bf16;            /* weights are always bf16 on the device; kept for layout parity */
    int64_t synthetic_kv_seed; /* <0: real prefill; >=0: prompts' KV prefix is seeded (bench workload) */
    /* T5 mode (north_star (1), CALM-T5; NOT in the reference): > 0 adds a
     * cross-attention sub-layer over this many synthetic encoder states per sequence
     * (static cross K/V written once at admission; the skipped-layer fill is unchanged). */
    int encoder_len;
    /* Extension (NOT in the reference; CALM-T5 attention): self- and, in T5 mode, cross-attention
     * split into n_heads heads of d_model / n_heads features (own softmax, scale 1/sqrt(head_dim));
     * 0 or 1 = the reference's single head.  head_dim: 8, 16, 32, 64, 128 or 256; n_heads <= 32. */
    int n_heads;
    /* T5 mode: > 0 runs a real encoder stack of this many bidirectional norm-free layers (own
     * seeded weights) over seeded encoder input ids at admission, instead of seeded encoder
     * states (extension; encoder_len <= 256). */
    int encoder_layers;
} el_engine_config;

typedef struct el_engine el_engine;
typedef struct el_transcript el_transcript;

const char* el_last_error(void);
int el_version(void);
/* select the CUDA device for engines created by this thread (one process per GPU) */
int el_set_device(int device);
int el_device_count(int* n);

int el_engine_create(const el_engine_config* cfg, el_engine** out);
/* The same, for callers compiled against another revision of this header: config_size =
 * sizeof(el_engine_config) as the caller sees it; fields past it take their zero defaults (the
 * reference's decoder-only, single-head model), fields the library does not know are rejected
 * unless zero. */
int el_engine_create_sized(const el_engine_config* cfg, size_t config_size, el_engine** out);
int el_engine_destroy(el_engine* e);
/* options: "graph" (1: CUDA graph with a device-side WHILE over layers, 0: eager),
 *          "rec_cap" (iterations kept in the device record ring) */
int el_engine_set_option(el_engine* e, const char* key, int64_t value);

/* Engine::run: requests as flat arrays (arrival[n], prompt_off[n+1], prompt[], max_new[n]) */
int el_engine_run(el_engine* e, int n, const double* arrival, const int32_t* prompt_off,
                  const int32_t* prompt, const int32_t* max_new, el_transcript** out);

/* flat transcript fields (same names as the oracle / reference wrappers):
 * i32: pf_seq pf_positions it_output_layer it_batch_off ps_seq ps_accept ps_token sq_id
 *      sq_max_new sq_prompt_off sq_prompt sq_tok_off sq_tokens sq_exit_layers sq_iter_out
 * f64: pf_clock pf_charge it_clock it_charge sq_arrival sq_first sq_finish meta it_conf */
int64_t el_transcript_len(const el_transcript* t, const char* field);
int el_transcript_get_i32(const el_transcript* t, const char* field, int32_t* out);
int el_transcript_get_f64(const el_transcript* t, const char* field, double* out);
int el_transcript_kv(const el_transcript* t, int seq_id, int layer, double* k, double* v, int64_t cap);
int el_transcript_exit_states(const el_transcript* t, int seq_id, double* out, int64_t cap);
/* capture_kv: the device block table [L][bpl] of a sequence at eviction (KvStore block_table,
 * kv_cache.hpp:79-84, LIFO order kv_cache.cpp:53-55/182-194); returns bpl (<0 on error) */
int el_transcript_block_table(const el_transcript* t, int seq_id, int32_t* out, int64_t cap);
void el_transcript_free(el_transcript* t);

/* fixed batch of B sequences (ids seq_ids[b]) whose KV holds prefix_len seeded
 * positions at every layer; first decode inputs first_tokens[b]; capacity in tokens */
int el_session_begin(el_engine* e, int batch, const int32_t* first_tokens, int prefix_len, int capacity,
                     uint64_t kv_seed, const int32_t* seq_ids);
int el_session_end(el_engine* e);
/* one iteration with host buffers (tokens_in may be NULL: keep the device-side
 * next inputs); outputs tokens[B], accept[B], conf[L][B] (NULL to skip), output layer */
int el_decode_iteration(el_engine* e, const int32_t* tokens_in, int32_t* tokens_out, int32_t* accept_out,
                        float* conf_out, int32_t* output_layer);
int el_decode_run(el_engine* e, int n_iters);
/* records of iterations [first, first+n) of this session (ring of rec_cap) */
int el_decode_records(el_engine* e, int first, int n, int32_t* tokens, int32_t* accept, int32_t* out_layer,
                      float* conf);
int el_decode_iterations_done(el_engine* e);
int el_set_fixed_confidences(el_engine* e, const float* conf /* [L][B] */);
int el_session_kv(el_engine* e, int row, int layer, int pos, float* k, float* v);
/* T5 mode: the static cross K/V of a session row at `layer` (encoder_len x d_model each) */
int el_session_cross_kv(el_engine* e, int row, int layer, float* k, float* v);
int el_session_hidden(el_engine* e, int parity, float* out /* [B][d] */);
int el_session_block_table(el_engine* e, int row, int32_t* out /* [L][bpl] */, int bpl_cap);

/* timing on the engine's stream with CUDA events (synchronised on both sides) */
int el_time_decode(el_engine* e, int n_iters, float* ms);
/* standalone kernel timing on the current session state: kind 0 attention,
 * 1 qkv gemm, 2 wo, 3 up, 4 down, 5 lm head; layer fixed; reps launches;
 * kind | 0x100: write 256 MB (2x L2) before each launch and time the launches alone */
int el_time_kernel(el_engine* e, int kind, int layer, int reps, float* ms);
int el_sync(el_engine* e);
/* experiment support: per-CTA phase timestamps (option "dbg" bit 8) */
int el_debug_timestamps(el_engine* e, uint64_t* out, int n);
int el_debug_timeline_reset(el_engine* e);
/* kernels launched per iteration with the given output layer (for gpu_launches) */
int el_launches_per_iteration(el_engine* e, int output_layer);
/* plan details: attention chunking, GEMM splits (for DESIGN / bench reporting) */
int el_plan_info(el_engine* e, int64_t* out, int cap);

/* MetricsReport (metrics.hpp:20-34) and compute_metrics (metrics.cpp:13-58) over a transcript:
 * throughput = tokens / final clock, inner-token latency = sum(finish - first) / tokens,
 * early-exit rate = % of tokens decoded by iterations with output_layer < L, mean layers per
 * token, exit-layer (by iteration) and accept-layer (by sequence) histograms [n_layers]. */
typedef struct {
    double throughput, inner_token_latency, early_exit_rate_pct, mean_layers_per_token;
    double total_sim_time, total_idle_time, wall_clock_info_s;
    int64_t total_tokens, iterations;
    int n_layers, pool_blocks, free_blocks, peak_blocks;
} el_metrics;
int el_transcript_metrics(const el_transcript* t, el_metrics* out, int64_t* exit_hist, int64_t* accept_hist);
/* the same over flat transcript fields (any engine's transcript; meta = {final clock, idle,
 * pool blocks, free blocks, peak blocks}) */
int el_metrics_compute(int n_layers, int n_iters, const int32_t* it_output_layer, const int32_t* it_batch_off,
                       int n_seqs, const int32_t* sq_id, const int32_t* sq_tok_off, const int32_t* sq_exit_layers,
                       const double* sq_first, const double* sq_finish, const double* meta, el_metrics* out,
                       int64_t* exit_hist, int64_t* accept_hist);

/* ---- sub-engine API on the engine's device pool (outside a session or run; a run or a
 * session resets the pool).  Vectors are fp32 host arrays of d_model values; K/V are stored
 * in bf16 like every other device K/V row.  At most max_batch sequences live at a time
 * (device block-table slots).
 *   el_kv_allocate/append/view/commit/release  KvStore::allocate/append/view/commit/release
 *                                              (kv_cache.hpp:45-75, kv_cache.cpp:78-194): the same
 *                                              LIFO block order, write-once/contiguity/capacity
 *                                              checks and error classes
 *   el_kv_lengths / el_kv_stats                KvStore::committed_len/written_len/stats
 *   el_layer_forward   layer_forward(weights, layer, batch, cache) (model.hpp:64-66, model.cpp:197-272):
 *                      K/V appended at each sequence's committed length, attention over 0..pos
 *   el_kv_fill         fill_skipped(cache, batch, output_layer, compute_kv_pair) (kv_cache.hpp:107-115,
 *                      model.cpp:274-282): one grouped GEMM, K/V written into the paged blocks
 *   el_exit_confidence the engine technique's *_confidence (exit_policy.hpp:46-70) of n states at
 *                      `layer` and decide's strict '>' threshold_at(layer) (exit_policy.cpp:89-115)
 *   el_greedy_tokens   greedy_token(lm_head_logits(h)) (model.hpp:71-76): lowest index on ties */
int el_kv_allocate(el_engine* e, int seq_id, int capacity_tokens);
int el_kv_release(el_engine* e, int seq_id);
int el_kv_append(el_engine* e, int seq_id, int layer, int position, const float* k, const float* v);
int el_kv_view(el_engine* e, int seq_id, int layer, int upto_position, float* k /* [upto][d] */, float* v);
int el_kv_commit(el_engine* e, int seq_id);
int el_kv_lengths(el_engine* e, int seq_id, int32_t* committed, int32_t* written /* [L] */);
int el_kv_stats(el_engine* e, int32_t* out4 /* pool, free, peak in use, live sequences */);
int el_layer_forward(el_engine* e, int layer, int n, const int32_t* seq_ids, const float* h_in /* [n][d] */,
                     float* h_out /* [n][d] */);
int el_kv_fill(el_engine* e, int n, const int32_t* seq_ids, const float* h_exit /* [n][d] */, int output_layer);
int el_exit_confidence(el_engine* e, int layer, int n, const float* h_prev, const float* h_cur, float* conf /* [n] */,
                       int32_t* accept /* [n] */);
int el_greedy_tokens(el_engine* e, int n, const float* h /* [n][d] */, int32_t* tokens /* [n] */);

/* ---- layer-level scheduling (the occupancy MDP of layer_sched.hpp:13-60
 * driving real batches) over the current session's batch.  A turn runs ONE layer for every
 * sequence whose next layer it is (one persistent-kernel launch); each sequence exits on its own
 * accept (no batch barrier) -- per sequence exactly decode_iteration for a batch of one --,
 * fills its skipped layers' K/V, emits its token and restarts at layer 1.
 *   policy 0 greedy: argmax_a v[a], ties toward the lowest layer (greedy_action, layer_sched.cpp:95-105)
 *   policy 1 linear: argmax_a M[a].v (LinearQ::predict / TrainedPolicy::action, layer_sched.cpp:189-199,
 *            311-325), lin_m = M [L][L] row-major; greedy when the chosen layer is empty
 * el_sched_run runs n turns (one host round trip per turn: the next turn's rows depend on this
 * one's exits) and returns their elapsed time (CUDA events on the engine stream). */
int el_sched_begin(el_engine* e, int policy, const double* lin_m);
int el_sched_run(el_engine* e, int n_turns, float* ms);
/* tokens and exit layers of a row so far (returns the count; fills up to cap) */
int el_sched_tokens(el_engine* e, int row, int32_t* tokens, int32_t* exit_layers, int cap);
/* the layer and row count of every turn so far (returns the count) */
int el_sched_turns(el_engine* e, int32_t* layers, int32_t* rows, int cap);

/* LIFO allocator on the host mirror (same arithmetic the device kernels run) */
int el_kv_block_trace(int n_layers, int pool_blocks, int block_capacity, int n_ops, const int32_t* ops,
                      const int32_t* caps, int n_ids, int bpl_max, int32_t* tables);
/* model tensors as stored on the device (bf16 bits, unpadded):
 * which 0 embedding, 1 lm_head, 2 probe_w (fp32 bits of bf16 values), 3 probe_b,
 * 4..9 layer q,k,v,o,up,down */
int el_model_tensor(el_engine* e, int which, int layer, uint16_t* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif

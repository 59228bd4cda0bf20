// el_kernels.h -- host-visible launch interface of the exitlab-b200 kernels.
//
// One decode iteration (engine.cpp:208-310) on the device is:
//   embed -> WHILE(layer loop) { qkv_gemm -> attention -> wo_gemm -> up_gemm ->
//            down_gemm -> [lm_gemm (softmax check)] -> exit } -> fill_gemm ->
//   [lm_gemm (greedy)] -> finish
// Every kernel reads the current layer / output layer from device memory, so the
// same launches serve the eager path and the CUDA-graph path (WHILE conditional
// node set from the exit kernel).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace el {

enum Technique : int { kSoftmax = 0, kState = 1, kClassifier = 2, kNever = 3, kAlwaysAt = 4, kFixed = 5 };

// Model/cache dimensions.  dp = d rounded up to 128 (GEMM M-tile), fp = 4d
// rounded up to 128, Vp = V rounded up to 128; padding rows/cols are zero.
struct Dims {
    int L, d, dp, fp, V, Vp;
    int bc;       // KV block capacity (positions per block)
    int bpl_max;  // max blocks per (seq, layer) in the device block tables
    int Bmax;     // max rows (max_batch)
    int slots;    // sequence slots in the device block tables
};

// Rows of the current iteration (decode batch or prefill batch).
struct Rows {
    const int* slot;  // [Bmax] sequence slot of each row
    int* pos;         // [Bmax] committed length = position written this iteration
    int* tok;         // [Bmax] input token of this iteration
    int B;
};

// All device pointers of one engine.  POD, passed by value to every kernel.
// Instrumentation / probe switches (DevState::dbg) compile to constant 0 unless the
// library is built with EL_DEBUG=1 (scripts/mega_phases.py and the other timeline
// probes need that build): the product kernels carry none of that code.
#ifndef EL_DEBUG
#define EL_DEBUG 0
#endif
#define EL_DBG(s) (EL_DEBUG ? (s).dbg : 0)

struct DevState {
    Dims dm;
    // weights (bf16 bit patterns), packed per layer
    const uint16_t* wqkv;   // [L][3dp][dp]  rows q | k | v
    const uint16_t* wo;     // [L][dp][dp]
    const uint16_t* wup;    // [L][fp][dp]
    const uint16_t* wdown;  // [L][dp][fp]
    const uint16_t* emb;    // [Vp][dp]
    const uint16_t* lm;     // [Vp][dp]
    const float* probe_w;   // [dp]
    float probe_b;
    // paged KV pool
    uint16_t* kpool;        // [pool][bc][dp]
    uint16_t* vpool;
    const int* tables;      // [slots][L][bpl_max]
    Rows rows;
    int NR;           // activation tile height (act_offset)
    // activations (bf16 copies in act_offset layout)
    float* h32;       // [2][Bmax][dp]  residual stream, parity = layer & 1
    uint16_t* hb;     // [2][Bmax][dp]  bf16 copy (GEMM B operand)
    float* q32;       // [Bmax][dp]
    uint16_t* att_b;  // [Bmax][dp]
    float* mid32;     // [Bmax][dp]
    uint16_t* mid_b;  // [Bmax][dp]
    uint16_t* up_b;   // [Bmax][fp]
    // attention split-context workspace
    float* attn_o;    // [Bmax][attn_max_chunks][dp]
    float* attn_ml;   // [Bmax][attn_max_chunks][2]
    int* attn_cnt;    // [Bmax]
    int attn_max_chunks;
    int attn_cb;      // blocks per chunk
    int attn_stages;
    int attn_grid;    // persistent CTAs
    int attn_seg_cost;      // static split: extra cost of a row start, in KV blocks
    int dbg;          // experiment knob (0 = normal)
    unsigned long long* dbg_ts;
    float attn_scale; // 1/sqrt(d), or 1/sqrt(head_dim) with heads
    int attn_heads;   // attention heads (T5 mode; 1 = the reference's single head)
    int attn_hd;      // features per head (d when attn_heads == 1)
    int enc_bidir;    // T5 encoder stack launch: > 0 = every row attends over this many positions of its
                      // sequence's blocks (bidirectional self-attention), 0 = causal decode / prefill
    // split-K GEMM workspace
    // LM-head per-tile partials [Vp/128][Bmax] {max1, max2, sumexp(rel max1), argmax}
    float4* lm_part;
    // exit status (Algorithm 1 "Status")
    int* layer;              // current layer (1-based), advanced by the exit kernel
    int* out_layer;          // output_layer of the iteration
    int* status;             // [Bmax] OR-latched accept
    int* first_accept;       // [Bmax] 0 = never
    int* accept;             // [Bmax] this layer's decision
    float* conf;             // [L][Bmax] this iteration's confidences
    int* exit_cnt;
    double* exit_part;       // [Vp/128 tiles][Bmax][3] per-tile partial dots (fused exit)
    int fuse_exit;           // exit check runs in the down-projection epilogue
    int* cont_host;          // mapped host flag (eager path reads it)
    const double* lambdas;   // [L] threshold_at(schedule, layer)
    const float* fixed_conf; // [L][Bmax] injected confidences (technique kFixed)
    int technique, exit_layer;
    cudaGraphConditionalHandle cond;
    int use_cond;
    // per-iteration records (ring)
    int* iter_counter;
    int* cur_iter;
    // packed record per iteration (one D2H copy): [tokens Bmax | accept Bmax | output layer, pad 3 |
    // conf (float) L x Bmax], rec_stride ints apart
    int* rec;
    int rec_stride;
    int rec_cap;
    int prefill;  // persistent kernel in batched-prefill mode (rows = prompt positions; K/V only)
    // layer-level scheduling (f4): > 0 = this launch is one TURN that runs only
    // layer turn_layer for its rows (the sequences whose next layer it is); each row exits on its
    // own accept (no batch barrier) and the hidden state of a row that continues is kept per
    // sequence in hstore (row b is sequence row_seq[b])
    int turn_layer;
    float* hstore;        // [Bmax][dp] fp32 state entering each sequence's next layer
    const int* row_seq;   // [Bmax] sequence index of each row of the turn
    // deferred tokens (layer-level scheduling): turn_defer = 1: a layer turn stores every row's state
    // (exited rows' too) and decodes no token; turn_token = 1: a token turn -- rows = sequences whose
    // position exited at row_exit[b] (>= turn_layer = the smallest): LM head + greedy token + the
    // skipped-layer fill of layers (row_exit[b], L] for every row at once, no layer computed
    int turn_defer, turn_token;
    const int* row_exit;
    // Engine::run between scheduling events: iterations queued back to back on the device skip
    // themselves once *run_active is 0 (set by run_step_kernel); nullptr = always run
    const int* run_active;
    // T5 mode (encoder_len > 0): cross-attention weights and the static encoder K/V
    int enc_len, enc_blocks;    // encoder states per sequence; KV blocks they occupy
    const uint16_t* wqc;        // [L][dp][dp]   tiled
    const uint16_t* wkvc;       // [L][2dp][dp]  tiled, rows k_c | v_c
    const uint16_t* woc;        // [L][dp][dp]   tiled
    uint16_t* ckpool;           // [slots * L * enc_blocks][bc][dp]
    uint16_t* cvpool;
    const int* ctables;         // [slots][L][enc_blocks] (static)
};

__host__ __device__ inline int* rec_rec(const DevState& st, int cur) { return st.rec + (size_t)cur * st.rec_stride; }
__host__ __device__ inline float* rec_conf(const DevState& st, int cur) {
    return reinterpret_cast<float*>(rec_rec(st, cur) + 2 * st.dm.Bmax + 4);
}

// Weight (GEMM A operand) layout in HBM: 128x64 bf16 tiles, tile-major
// [row/128][col/64], each tile stored exactly as TMA SWIZZLE_128B would place
// it in shared memory (16-byte chunk c of row r at chunk c ^ (r & 7)), so one
// contiguous 16 KB bulk copy lands a ready-to-use UMMA operand.
__host__ __device__ inline size_t tiled_offset(int r, int c, int cols_p) {
    const int kb_total = cols_p / 64;
    const size_t tile = (size_t)(r >> 7) * kb_total + (c >> 6);
    const int rr = r & 127, cc = c & 63;
    return tile * 8192 + (size_t)rr * 64 + (size_t)((((cc >> 3) ^ (rr & 7)) << 3) | (cc & 7));
}

// Activation (GEMM B operand) layout: [col/64][NR rows][64 cols] with the same
// 128-byte swizzle; NR = Bmax rounded up to 16. A k-block of the first n rows
// is one contiguous n*128-byte bulk copy.
__host__ __device__ inline size_t act_offset(int row, int col, int NR) {
    const int cc = col & 63;
    return ((size_t)(col >> 6) * NR + row) * 64 + (size_t)((((cc >> 3) ^ (row & 7)) << 3) | (cc & 7));
}

// one split-K weight-streaming GEMM launch: D[M x N] = W[M x K] . X[N x K]^T
struct GemmPlan {
    const uint16_t* A;  // weights, tiled layout (tiled_offset)
    const uint16_t* Bp; // activations, act_offset layout (parity 0)
    size_t b_par_stride; // elements between the two hidden-state parities
    int m_tiles, splits, kb_total, n_pad, stages, smem_bytes, tmem_cols;
};

enum GemmKind : int { kGemmQkv = 0, kGemmWo, kGemmUp, kGemmDown, kGemmLmCheck, kGemmLmFinal, kGemmFill, kGemmCross };

int gemm_smem_bytes(int n_pad, int stages, bool tile_reduce);
void init_kernel_attributes();
void launch_gemm(GemmKind kind, const GemmPlan& p, const DevState& st, cudaStream_t s, bool pdl);

void launch_weightgen(uint16_t* out, int rows, int cols, int rows_p, int cols_p, uint64_t seed, double scale,
                      int tiled, cudaStream_t s);
void launch_kv_prefix(const DevState& st, const int* row_seq_ids, int prefix_len, uint64_t kv_seed, int round_bf16,
                      cudaStream_t s);
void launch_embed(const DevState& st, cudaStream_t s);
// T5 mode: seeded encoder states of n sequences (ids) as bf16 GEMM B operand rows j*T + t (act layout, NR rows)
void launch_act_rows_copy(uint16_t* dst, int NRd, int row0, const uint16_t* src, int NRs, int n, int dp,
                          cudaStream_t s);
void launch_encoder_states(uint16_t* act, int NR, const int* ids, int n, int T, int d, int dp, uint64_t enc_seed,
                           cudaStream_t s);
// one attention stage: K block | V block | q (fp32); also hosts the 8-warp merge
__host__ __device__ inline int attn_stage_bytes(const Dims& dm) {
    const int kvq = 2 * dm.bc * dm.dp * 2 + dm.dp * 4;
    const int merge = 8 * dm.dp * 4;
    return ((kvq > merge ? kvq : merge) + 127) / 128 * 128;
}
int attn_smem_bytes(const Dims& dm, int stages);
int attn_ctas_per_sm(const Dims& dm, int stages);
int attn_threads();
void launch_attention(const DevState& st, cudaStream_t s, bool pdl);
void launch_exit(const DevState& st, cudaStream_t s, bool pdl);
void launch_finish(const DevState& st, cudaStream_t s, bool pdl);
void launch_advance(const DevState& st, cudaStream_t s);
// Engine::run (engine.cpp:266-305) on the device between scheduling events: after each iteration,
// the simulated-clock charge of its output layer, the per-sequence max_new / EOS stop and the next
// admissible arrival decide whether the next queued iteration runs
struct RunCtl {
    double* clock;        // simulated clock (bit-exact with the host formula)
    double* log;          // [rec_cap][2] (clock after, charge) per iteration
    int* rem;             // [Bmax] tokens each row may still emit
    int* active;          // 1 while the queued iterations run
    int* done;            // iterations run in this chunk
    int eos, L;
    double next_arrival;  // arrival of the admissible pending head (+inf: none)
    double c_fixed, c_seq, c_check, c_fill;
};
void launch_run_step(const DevState& st, const RunCtl& c, cudaStream_t s);
void launch_layer_head(const DevState& st, cudaStream_t s);  // prefill commit: pos += 1
// LIFO block allocator on the device (kv_cache.cpp:78-106, 182-194)
void launch_kv_alloc(int* stack, int top, int* tables, const Dims& dm, int slot, int bpl, cudaStream_t s);
void launch_kv_release(int* stack, int top, const int* tables, const Dims& dm, int slot, int bpl, cudaStream_t s);


// ---- persistent decode-iteration kernel (el_iter.cuh) ----
enum IterGemmId : int { kIQkv = 0, kIWo, kIUp, kIDown, kIFill, kIQc, kIWoc, kINumGemm };

struct IterGemm {
    const uint16_t* A;  // tiled weights (tiled_offset), tile row 0 of layer 1
    int m_tiles;        // 128-row output tiles (per layer)
    int kb_total;       // 64-wide k-blocks of the reduction dimension
    int splits;         // K splits per output tile (units = m_tiles * splits)
    int layer_rows;     // tile rows per layer in A
    int row_off;        // tile-row offset inside a layer (fill: the k|v rows)
    int mode;           // 0 weight-streaming split-K + reduce phase; 1 batch-M full-K (direct epilogue)
    int nt;             // mode 1: output features per unit (MMA N)
};

struct IterPlan {
    IterGemm g[kINumGemm];
    int n_pad;       // MMA N: batch rounded up to 16
    int stages;      // GEMM ring depth
    int stage_bytes; // GEMM ring stage stride (A region 16 KB | B region)
    // batch-M ring: bm_stages stages of bm_kc activation k-blocks (bm_astage bytes each, bm_rows
    // batch rows per k-block), the unit's weights at bm_woff
    int bm_rows, bm_kc, bm_astage, bm_stages, bm_woff;
    int bm_prefetch;  // issue each batch-M unit's weights one phase ahead (weight buffer outside the rings)
    int bm_wstream;   // batch-M weights streamed through the ring (L2-prefetched a phase ahead), no weight slab
    int bm_m;           // UMMA M of the batch-M GEMMs: 64 (batch <= 64) or 128
    int bm_grp;         // batch rows per unit (row group): bm_rows, or 128 when the batch has 2 groups
    int map_key;        // host-side key of this plan's tensor maps
    unsigned* tcnt;     // [kINumGemm][64] per-tile arrival counters (zeroed at the end of each launch)
    int att_mbuf_off;   // > 0: the attention segment merge buffer [8][dp] fp32 (else merged inside the stage)
    int att_early;      // the attention producer starts before the QKV -> attention barrier
    int ring_bytes;  // shared ring region (attention stages / GEMM stages + LM transpose buffer)
    int gemm_ring;   // bytes of the GEMM stages inside the ring region
    int lm_tiles;    // Vp / 128
    float* part;     // split-K partials [unit][n_pad][128] fp32
    unsigned* bar;   // grid barrier: [0] arrivals, [32] generation
    int pipe_att_ctas;  // pipelined kernel (el_pipe.cuh): CTAs [0, pipe_att_ctas) run attention
    // LM-head weight tiles loaded evict-last (1: the softmax checks, re-read every layer and
    // small enough to stay in L2 under the evict-first K/V and layer-weight streams; 2: also the
    // final LM head, kept across iterations); 0: evict-first like every other weight
    int lm_keep;
    // softmax checks on LM pair units (two vocab tiles per unit, one wave; the ring runs past the
    // batch-M weight slab, so the next QKV slab is prefetched after the LM head): 1 vocab rows on
    // TMEM lanes (shuffle-butterfly epilogue), 2 transposed -- batch rows on TMEM lanes, one
    // M128 x N256 MMA per k-step, per-thread sequential reduction (batch of 128 rows only)
    int lm_pair;
    // decode tail's greedy LM head on transposed units (batch 128: tile pairs, 256: both row groups)
    int lm_tail_tr;
    int lm_stages;  // pipelined kernel: depth of the LM pair units' own ring (full3 / empty3)
};

// 3-D (64 x 128 rows x tiles, no swizzle: the tiles are pre-swizzled) tensor maps over the
// batch-M GEMMs' weights, box = nt rows x all k-blocks (one copy per unit)
struct alignas(64) IterMaps {
    CUtensorMap w[kINumGemm];
};
int iter_smem_bytes(int ring_bytes);   // dynamic shared memory of the launch
int iter_smem_fixed();                 // bytes outside the ring region (alignment slack + control block)
int iter_max_ctas_per_sm(const Dims& dm, int ring_bytes);
void init_iter_attributes();
void launch_iter(const DevState& st, const IterPlan& p, const IterMaps& maps, int grid, cudaStream_t s);
// the pipelined iteration (el_pipe.cuh): attention and projection GEMMs of the two batch halves
// on disjoint CTA sets, overlapped (batch 129..256)
void launch_pipe(const DevState& st, const IterPlan& p, const IterMaps& maps, int grid, cudaStream_t s);
void init_pipe_attributes();
constexpr int kIterTbufBytes = 32 * 129 * 4;

// host+device mirror of the allocator arithmetic (used by el_kv_block_trace)
inline void kv_pop_host(const int* stack, int top, int* table_flat, int n) {
    for (int i = 0; i < n; ++i) table_flat[i] = stack[top - 1 - i];
}
inline void kv_push_host(int* stack, int top, const int* table_flat, int n) {
    for (int i = 0; i < n; ++i) stack[top + i] = table_flat[i];
}

}  // namespace el

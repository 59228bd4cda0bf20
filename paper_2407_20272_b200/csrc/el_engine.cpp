// el_engine.cpp -- host side of the B200 early-exit decode engine and the C ABI
// declared in include/exitlab_b200.h.
//
// The host mirrors the reference engine's control plane exactly (Engine::run,
// engine.cpp:110-330: FIFO admission with head-of-line deferral, eviction at
// the start of the next pass, simulated-clock charges, transcript records),
// while every per-token computation runs in the sm_100a kernels of
// el_kernels.cu.  The KV block tables live on the device; the host keeps only
// the free-block count and per-sequence bookkeeping needed for the reference's
// invariant checks (write-once/contiguity/commit completeness).
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/exitlab_b200.h"
#include "el_common.cuh"
#include "el_kernels.h"

namespace {

thread_local std::string g_err;

struct ElError {
    int code;
    std::string msg;
};
[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw ElError{code, buf};
}
#define CK(x)                                                                                        \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess) fail(EL_CUDA_ERROR, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                    __FILE__, __LINE__);                                             \
    } while (0)

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count, bool zero = true) {
        release();
        if (count == 0) count = 1;
        CK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
        if (zero) CK(cudaMemset(p, 0, count * sizeof(T)));
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
};

int round_up(int x, int m) { return (x + m - 1) / m * m; }
int ceil_div(int a, int b) { return (a + b - 1) / b; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) fail(EL_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// bf16 [rows][k] row-major, box [box_rows][64], 128-byte swizzle
CUtensorMap make_map(const void* base, int rows, int k, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)k * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(EL_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d) rows=%d k=%d box=%d", (int)r, rows, k, box_rows);
    return m;
}

// batch-M weight operand map: the tiled weight tensor viewed as [tiles][128 rows][64 cols] bf16
// (no swizzle: the tiles are stored pre-swizzled), box = nt rows x kb_total consecutive tiles
CUtensorMap make_bm_map(const void* base, size_t tiles, int nt, int kb_total) {
    CUtensorMap m;
    cuuint64_t dims[3] = {64, 128, (cuuint64_t)tiles};
    cuuint64_t strides[2] = {128, 16384};
    cuuint32_t box[3] = {64, (cuuint32_t)nt, (cuuint32_t)kb_total};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(EL_CUDA_ERROR, "cuTensorMapEncodeTiled (batch-M) failed (%d)", (int)r);
    return m;
}

double threshold_at(double l0, double g, double lmin, int layer) {  // exit_policy.cpp:50-55
    return std::max(lmin, l0 * std::pow(g, layer - 1));
}

// ----- flat transcript (same layout as the oracle / reference wrappers) -----
struct Capture {
    int committed = 0;
    std::vector<double> k, v;  // [L][committed][d]
    std::vector<double> exit_states;
    bool have_kv = false;
    int bpl = 0;
    std::vector<int32_t> table;  // [L][bpl] device block table at eviction
};
}  // namespace

struct el_transcript {
    std::vector<int32_t> pf_seq, pf_positions, it_output_layer, it_batch_off, ps_seq, ps_accept, ps_token, sq_id,
        sq_max_new, sq_prompt_off, sq_prompt, sq_tok_off, sq_tokens, sq_exit_layers, sq_iter_out;
    std::vector<double> pf_clock, pf_charge, it_clock, it_charge, sq_arrival, sq_first, sq_finish, meta, it_conf;
    std::map<int, Capture> caps;
    int d = 0, L = 0;
    std::vector<int32_t>* i32(const char* f) {
#define F(n) if (!std::strcmp(f, #n)) return &n;
        F(pf_seq) F(pf_positions) F(it_output_layer) F(it_batch_off) F(ps_seq) F(ps_accept) F(ps_token) F(sq_id)
        F(sq_max_new) F(sq_prompt_off) F(sq_prompt) F(sq_tok_off) F(sq_tokens) F(sq_exit_layers) F(sq_iter_out)
#undef F
        return nullptr;
    }
    std::vector<double>* f64(const char* f) {
#define F(n) if (!std::strcmp(f, #n)) return &n;
        F(pf_clock) F(pf_charge) F(it_clock) F(it_charge) F(sq_arrival) F(sq_first) F(sq_finish) F(meta) F(it_conf)
#undef F
        return nullptr;
    }
};

struct el_engine {
    el_engine_config cfg{};
    el::Dims dm{};
    cudaStream_t stream = nullptr, stream2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int device = 0;
    bool use_graph = true;
    bool pdl = true;
    bool body_head = false;
    bool fuse_exit = true;
    bool fuse_exit_all = false;
    // decode-iteration strategy: 0 per-phase kernels (graph / eager), 1 persistent kernel
    // (el_iter.cuh), 2 auto: persistent at batch >= 64 (measured faster there: weight streaming
    // and the exit check amortise its grid barriers), per-phase below
    int use_mega = 2;
    bool mega_for(int B) const {
        if (cfg.encoder_len > 0) {  // T5 mode: the cross-attention sub-layer lives in the persistent kernel
            if (use_mega == 0) fail(EL_INVALID_ARGUMENT, "T5 mode (encoder_len > 0) runs on the persistent kernel");
            return true;
        }
        if (use_mega != 2) return use_mega == 1;
        // softmax included: at batch 128 the persistent kernel measured 1.85 ms vs 2.10 ms per
        // iteration (c4m), at batch 8 the per-phase graph wins (c1: 0.163 vs 0.183 ms)
        return B >= 64;
    }
    int dbg = 0;
    int rec_cap = 4096;
    // pipelined iteration kernel (el_pipe.cuh) for batch 129..256: 0 off, 1 on, 2 auto (on outside
    // softmax exit / T5 mode); attention CTAs of its grid (the rest run the projection GEMMs)
    int use_pipe = 2, pipe_att = 100;  // attention CTAs of the pipelined kernel (the rest run GEMMs)
    // batch 65..128 on the pipelined kernel with halves of 64 rows (64-row batch-M groups, UMMA
    // M = 64; needs the 128-row activation layout)
    int pipe128 = 1;
    int pipe_att64 = 84;  // attention CTAs of the pipelined kernel at batch <= 128 (64-row halves)
    int pipe_att64_sm = 80;  // the same with softmax exit (the LM-head check runs on the GEMM CTAs)
    int pipe_softmax = 1;  // softmax exit on the pipelined kernel (batch 65..128)
    // batch 33..64 on the pipelined kernel with halves of 32 rows (UMMA M = 64 over a 32-row group:
    // the upper 32 accumulator rows are discarded; needs the 64-row activation layout)
    int pipe64 = 0, pipe_att32 = 84;
    bool pipe_for(int B) const {
        if (use_pipe == 0 || B > 256 || cfg.encoder_len > 0) return false;
        // (softmax: the LM-head check on the GEMM CTAs, pair units at batch <= 128 only)
        if (B <= 64) return pipe64 && B > 32 && NR == 64 && cfg.technique != EL_TECH_SOFTMAX;
        // (the pipelined kernel's softmax check has pair units only: lm_pair 0 keeps softmax on iter_kernel)
        if (B <= 128)
            return pipe128 && B > 64 && NR == 128 && (cfg.technique != EL_TECH_SOFTMAX || (pipe_softmax && opt_lm_pair));
        return cfg.technique != EL_TECH_SOFTMAX;
    }

    // weights
    DevBuf<uint16_t> wqkv, wo, wup, wdown, emb, lm;
    // T5 mode (encoder_len > 0): cross weights, static encoder K/V pool + tables, encoder-state staging
    DevBuf<uint16_t> wqc, wkvc, woc, ckpool, cvpool, enc_act;
    DevBuf<int> ctables, xslot, xid;
    // T5 encoder stack (encoder_layers > 0): its weights, the scratch K/V of one launch's sequences
    // (one block table per (local sequence, encoder layer)), the plan switch of mplan_for
    DevBuf<uint16_t> e_wqkv, e_wo, e_wup, e_wdown, e_kpool, e_vpool;
    DevBuf<int> e_tables;
    int e_bpl = 0;
    bool plan_encoder = false;
    int enc_blocks = 0;
    uint64_t enc_seed = 0;
    DevBuf<float> probe_w;
    float probe_b = 0.f;
    // kv pool + device allocator
    DevBuf<uint16_t> kpool, vpool;
    DevBuf<int> stack, tables;
    int top = 0;  // free blocks (device stack height)
    int peak = 0;
    // rows
    DevBuf<int> row_slot, row_pos, row_tok, pf_slot, pf_pos, pf_tok, seq_ids_dev;
    // activations / workspaces
    DevBuf<float> h32, q32, mid32, attn_o, attn_ml, conf;
    static constexpr int kPfRows = 256;  // rows of one batched-prefill launch
    DevBuf<float> pf_h32, pf_q32, pf_mid32;
    DevBuf<uint16_t> pf_hb, pf_att_b, pf_mid_b, pf_up_b;
    DevBuf<uint16_t> hb, att_b, mid_b, up_b;
    DevBuf<int> attn_cnt, layer, out_layer, status, first_accept, accept, exit_cnt, iter_counter,
        cur_iter, rec;
    int rec_stride = 0;
    int* rec_host = nullptr;  // pinned staging for one packed record
    DevBuf<float4> lm_part;
    DevBuf<double> lambdas, exit_part;
    DevBuf<unsigned long long> dbg_ts;
    DevBuf<float> fixed_conf;
    DevBuf<uint8_t> l2flush;  // cold-L2 kernel timing (el_time_kernel kind | 0x100)
    // Engine::run between scheduling events: queued iterations run while *run_ctl[0] != 0
    // (run_ctl[1] counts those that ran); simulated clock, its per-iteration log, tokens left
    DevBuf<int> run_ctl, run_rem;
    DevBuf<double> run_clock, run_log;
    int* cont_host = nullptr;
    int* cont_dev = nullptr;

    // plans
    struct Plans {
        el::GemmPlan qkv, wo, up, down, lm, fill;
        int n_pad = 0;
    };
    std::map<int, Plans> plans;  // by n_pad
    std::map<int, el::IterPlan> mplans;  // persistent-kernel plans by n_pad
    std::map<int, el::IterMaps> mmaps;   // their batch-M weight tensor maps
    DevBuf<float> mpart;                 // split-K partial workspace of the persistent kernel
    DevBuf<unsigned> mbar;               // its grid barrier (arrivals, generation)
    DevBuf<unsigned> mtcnt;              // its per-tile split-K arrival counters
    int mega_grid = 0, mega_att_stages = 2, sms = 148;
    int opt_mega_fill_splits = 0, opt_mega_att_stages = 0, 
        opt_mega_bm_max = 256, opt_mega_bm_prefetch = 1,
        opt_mega_bm_chunk_kb = 0, opt_mega_bm_nt_min = 16,
        opt_mega_bm_m128 = 0, opt_mega_bm_down = 0, opt_mega_down_splits = 0,
        opt_mega_splits_cap = 0, opt_att_mbuf = 1, opt_mega_att_early = 1, opt_attn_seg_cost = -1,
        opt_attn_grid = 0, opt_mega_bm_wstream = -1, opt_lm_keep = 1, opt_lm_pair = 2, opt_lm_tail = 1;
    int attn_cb = 1, attn_stages = 2, attn_max_chunks = 1, attn_grid = 148;
    int NR = 16;

    // graphs by batch size
    struct Graph {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t x = nullptr;
    };
    std::map<int, Graph> graphs;

    // session state
    bool in_session = false;
    int sess_B = 0;
    int sess_iters = 0;
    std::vector<int> sess_ids;
    std::vector<int> slot_bpl;  // per slot blocks per layer (-1 = free; 0 = a zero-capacity sequence)

    ~el_engine() {
        for (auto& kv : graphs) {
            if (kv.second.x) cudaGraphExecDestroy(kv.second.x);
            if (kv.second.g) cudaGraphDestroy(kv.second.g);
        }
        if (cont_host) cudaFreeHost(cont_host);
        if (rec_host) cudaFreeHost(rec_host);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (stream2) cudaStreamDestroy(stream2);
        if (stream) cudaStreamDestroy(stream);
    }

    // ------------------------------------------------------------------
    void validate() const {  // EngineConfig::validate (engine.cpp:31-45)
        const el_engine_config& c = cfg;
        if (c.n_layers < 2) fail(EL_INVALID_ARGUMENT, "ModelConfig: n_layers must be >= 2");
        if (c.d_model < 2) fail(EL_INVALID_ARGUMENT, "ModelConfig: d_model must be >= 2");
        if (c.vocab_size < 2) fail(EL_INVALID_ARGUMENT, "ModelConfig: vocab_size must be >= 2");
        if (!(c.gamma > 0.0 && c.gamma <= 1.0)) fail(EL_INVALID_ARGUMENT, "ThresholdSchedule: gamma must be in (0, 1]");
        if (c.lambda_min < 0.0) fail(EL_INVALID_ARGUMENT, "ThresholdSchedule: lambda_min must be >= 0");
        if (c.lambda_min > c.lambda0) fail(EL_INVALID_ARGUMENT, "ThresholdSchedule: lambda_min must be <= lambda0");
        for (double x : {c.c_layer_fixed, c.c_layer_per_seq, c.c_fill_per_seq_layer, c.c_check_softmax,
                         c.c_check_classifier, c.c_check_state})
            if (x < 0.0) fail(EL_INVALID_ARGUMENT, "CostModel: charges must be nonnegative");
        if (c.max_batch < 1) fail(EL_INVALID_ARGUMENT, "EngineConfig: max_batch must be >= 1");
        if (c.max_batch > 256) fail(EL_INVALID_ARGUMENT, "EngineConfig: max_batch > 256 unsupported on this engine");
        if (c.pool_blocks < 1) fail(EL_INVALID_ARGUMENT, "EngineConfig: pool_blocks must be >= 1");
        if (c.block_capacity < 1) fail(EL_INVALID_ARGUMENT, "EngineConfig: block_capacity must be >= 1");
        if (c.block_capacity > 64) fail(EL_INVALID_ARGUMENT, "EngineConfig: block_capacity > 64 unsupported");
        if (c.eos_token >= c.vocab_size) fail(EL_INVALID_ARGUMENT, "EngineConfig: eos_token outside vocab");
        if (c.technique < 0 || c.technique > EL_TECH_FIXED) fail(EL_INVALID_ARGUMENT, "EngineConfig: unknown technique");
        if (c.technique == EL_TECH_ALWAYS_AT && (c.exit_layer < 1 || c.exit_layer > c.n_layers))
            fail(EL_INVALID_ARGUMENT, "EngineConfig: always_at layer outside [1, n_layers]");
        if (c.d_model > 1024) fail(EL_INVALID_ARGUMENT, "d_model > 1024 unsupported on this engine");
        if (c.encoder_len < 0 || c.encoder_len > 2048)
            fail(EL_INVALID_ARGUMENT, "ModelConfig: encoder_len must be in [0, 2048]");
        if (c.encoder_layers < 0 || c.encoder_layers > 64 || (c.encoder_layers > 0 && (c.encoder_len <= 0 || c.encoder_len > 256)))
            fail(EL_INVALID_ARGUMENT, "ModelConfig: encoder_layers must be in [0, 64], > 0 only in T5 mode with "
                                      "encoder_len <= 256");
        if (c.n_heads > 1) {  // extension: the reference has one head
            const int hd = c.d_model % c.n_heads ? 0 : c.d_model / c.n_heads;
            if (c.n_heads > 32 || !hd || hd < 8 || hd > 256 || (hd & (hd - 1)))
                fail(EL_INVALID_ARGUMENT, "ModelConfig: n_heads must divide d_model into heads of 8..256 (power of 2) "
                                          "features, n_heads <= 32");
        } else if (c.n_heads < 0) {
            fail(EL_INVALID_ARGUMENT, "ModelConfig: n_heads must be >= 0");
        }
    }

    double check_cost() const {
        switch (cfg.technique) {
            case EL_TECH_SOFTMAX: return cfg.c_check_softmax;
            case EL_TECH_STATE: return cfg.c_check_state;
            case EL_TECH_CLASSIFIER: return cfg.c_check_classifier;
            default: return 0.0;
        }
    }

    void create() {
        validate();
        CK(cudaGetDevice(&device));
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&stream2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        const int L = cfg.n_layers, d = cfg.d_model, V = cfg.vocab_size;
        dm.L = L;
        dm.d = d;
        dm.dp = round_up(d, 128);
        dm.fp = round_up(4 * d, 128);
        dm.V = V;
        dm.Vp = round_up(V, 128);
        dm.bc = cfg.block_capacity;
        dm.Bmax = cfg.max_batch;
        dm.slots = cfg.max_batch;
        dm.bpl_max = 0;
        const int dp = dm.dp, fp = dm.fp;

        // ---- seeded weights (model.cpp:37-59), generated on the device, bf16 RNE ----
        auto tseed = [&](uint64_t tag) { return el::splitmix64_at(cfg.model_seed, tag); };
        wqkv.alloc((size_t)L * 3 * dp * dp, false);
        wo.alloc((size_t)L * dp * dp, false);
        wup.alloc((size_t)L * fp * dp, false);
        wdown.alloc((size_t)L * dp * fp, false);
        emb.alloc((size_t)dm.Vp * dp, false);
        lm.alloc((size_t)dm.Vp * dp, false);
        const double sd = 1.0 / std::sqrt((double)d), s4d = 1.0 / std::sqrt((double)(4 * d));
        // embedding stays row-major (row gather); every GEMM operand is tiled + pre-swizzled.
        // Row blocks of 128 are whole tiles, so a tensor at row offset R starts at tile R/128.
        el::launch_weightgen(emb.p, V, d, dm.Vp, dp, tseed(0), sd, 0, stream);
        el::launch_weightgen(lm.p, V, d, dm.Vp, dp, tseed(1), sd, 1, stream);
        for (int i = 0; i < L; ++i) {
            const uint64_t base = 4 + (uint64_t)i * 6;
            uint16_t* q = wqkv.p + (size_t)i * 3 * dp * dp;
            el::launch_weightgen(q, d, d, dp, dp, tseed(base + 0), sd, 1, stream);
            el::launch_weightgen(q + (size_t)dp * dp, d, d, dp, dp, tseed(base + 1), sd, 1, stream);
            el::launch_weightgen(q + (size_t)2 * dp * dp, d, d, dp, dp, tseed(base + 2), sd, 1, stream);
            el::launch_weightgen(wo.p + (size_t)i * dp * dp, d, d, dp, dp, tseed(base + 3), sd, 1, stream);
            el::launch_weightgen(wup.p + (size_t)i * fp * dp, 4 * d, d, fp, dp, tseed(base + 4), sd, 1, stream);
            el::launch_weightgen(wdown.p + (size_t)i * dp * fp, d, 4 * d, dp, fp, tseed(base + 5), s4d, 1, stream);
        }
        // probe (tiny: host) -- seeded_vector(d) and b = 2u - 1, both bf16-rounded
        {
            std::vector<float> pw((size_t)dp, 0.f);
            const uint64_t sw = tseed(2);
            for (int i = 0; i < d; ++i) {
                const double u = (double)(el::splitmix64_at(sw, (uint64_t)i) >> 11) * 0x1.0p-53;
                const uint16_t bits = el::bf16_bits_rne((2.0 * u - 1.0) * sd);
                uint32_t f = (uint32_t)bits << 16;
                std::memcpy(&pw[(size_t)i], &f, 4);
            }
            probe_w.alloc((size_t)dp);
            CK(cudaMemcpy(probe_w.p, pw.data(), sizeof(float) * dp, cudaMemcpyHostToDevice));
            const double u = (double)(el::splitmix64_at(tseed(3), 0) >> 11) * 0x1.0p-53;
            const uint16_t bits = el::bf16_bits_rne(2.0 * u - 1.0);
            uint32_t f = (uint32_t)bits << 16;
            std::memcpy(&probe_b, &f, 4);
        }

        // ---- T5 mode: cross-attention weights (tags after the reference's last, 4 + 6L + 4i + k),
        //      the static per-sequence encoder K/V blocks and their (identity) block tables ----
        if (cfg.encoder_len > 0) {
            const int T = cfg.encoder_len;
            wqc.alloc((size_t)L * dp * dp, false);
            wkvc.alloc((size_t)L * 2 * dp * dp, false);
            woc.alloc((size_t)L * dp * dp, false);
            for (int i = 0; i < L; ++i) {
                const uint64_t base = 4 + (uint64_t)L * 6 + (uint64_t)i * 4;
                el::launch_weightgen(wqc.p + (size_t)i * dp * dp, d, d, dp, dp, tseed(base + 0), sd, 1, stream);
                uint16_t* kv = wkvc.p + (size_t)i * 2 * dp * dp;
                el::launch_weightgen(kv, d, d, dp, dp, tseed(base + 1), sd, 1, stream);
                el::launch_weightgen(kv + (size_t)dp * dp, d, d, dp, dp, tseed(base + 2), sd, 1, stream);
                el::launch_weightgen(woc.p + (size_t)i * dp * dp, d, d, dp, dp, tseed(base + 3), sd, 1, stream);
            }
            enc_blocks = ceil_div(T, cfg.block_capacity);
            const size_t nblk = (size_t)cfg.max_batch * L * enc_blocks;
            ckpool.alloc(nblk * cfg.block_capacity * dp);
            cvpool.alloc(nblk * cfg.block_capacity * dp);
            std::vector<int> tab(nblk);
            for (size_t i = 0; i < nblk; ++i) tab[i] = (int)i;
            ctables.alloc(nblk);
            CK(cudaMemcpy(ctables.p, tab.data(), sizeof(int) * nblk, cudaMemcpyHostToDevice));
            xslot.alloc((size_t)cfg.max_batch);
            xid.alloc((size_t)cfg.max_batch);
            enc_act.alloc((size_t)round_up(cfg.max_batch * T, 256) * dp, false);
            enc_seed = el::splitmix64_at(cfg.model_seed, 0x454E43u);  // oracle: eo_encoder_seed
            if (cfg.encoder_layers > 0) {
                // encoder stack weights: tags after the cross weights, 4 + 10L + 6i + k (oracle:
                // eo_model_set_encoder_layers); scratch K/V for kPfRows / T sequences per launch
                const int LE = cfg.encoder_layers;
                e_wqkv.alloc((size_t)LE * 3 * dp * dp, false);
                e_wo.alloc((size_t)LE * dp * dp, false);
                e_wup.alloc((size_t)LE * fp * dp, false);
                e_wdown.alloc((size_t)LE * dp * fp, false);
                for (int i = 0; i < LE; ++i) {
                    const uint64_t base = 4 + (uint64_t)L * 10 + (uint64_t)i * 6;
                    uint16_t* q = e_wqkv.p + (size_t)i * 3 * dp * dp;
                    el::launch_weightgen(q, d, d, dp, dp, tseed(base + 0), sd, 1, stream);
                    el::launch_weightgen(q + (size_t)dp * dp, d, d, dp, dp, tseed(base + 1), sd, 1, stream);
                    el::launch_weightgen(q + (size_t)2 * dp * dp, d, d, dp, dp, tseed(base + 2), sd, 1, stream);
                    el::launch_weightgen(e_wo.p + (size_t)i * dp * dp, d, d, dp, dp, tseed(base + 3), sd, 1, stream);
                    el::launch_weightgen(e_wup.p + (size_t)i * fp * dp, 4 * d, d, fp, dp, tseed(base + 4), sd, 1, stream);
                    el::launch_weightgen(e_wdown.p + (size_t)i * dp * fp, d, 4 * d, dp, fp, tseed(base + 5), s4d, 1,
                                         stream);
                }
                e_bpl = ceil_div(T, cfg.block_capacity);
                const size_t eblk = (size_t)(kPfRows / T) * LE * e_bpl;
                e_kpool.alloc(eblk * cfg.block_capacity * dp);
                e_vpool.alloc(eblk * cfg.block_capacity * dp);
                std::vector<int> et(eblk);
                for (size_t i = 0; i < eblk; ++i) et[i] = (int)i;
                e_tables.alloc(eblk);
                CK(cudaMemcpy(e_tables.p, et.data(), sizeof(int) * eblk, cudaMemcpyHostToDevice));
            }
        }

        // ---- KV pool + allocator ----
        const size_t pool_elems = (size_t)cfg.pool_blocks * dm.bc * dp;
        kpool.alloc(pool_elems);
        vpool.alloc(pool_elems);
        stack.alloc((size_t)cfg.pool_blocks);
        reset_allocator();

        // ---- rows / activations ----
        const int Bm = dm.Bmax;
        for (DevBuf<int>* b : {&row_slot, &row_pos, &row_tok, &seq_ids_dev}) b->alloc((size_t)Bm);
        // prefill rows: up to kPfRows prompt positions per persistent-kernel launch (own activation set)
        for (DevBuf<int>* b : {&pf_slot, &pf_pos, &pf_tok}) b->alloc((size_t)std::max(Bm, kPfRows));
        pf_h32.alloc((size_t)2 * kPfRows * dp);
        pf_hb.alloc((size_t)2 * kPfRows * dp);
        pf_q32.alloc((size_t)kPfRows * dp);
        pf_att_b.alloc((size_t)kPfRows * dp);
        pf_mid32.alloc((size_t)kPfRows * dp);
        pf_mid_b.alloc((size_t)kPfRows * dp);
        pf_up_b.alloc((size_t)kPfRows * fp);
        // activation rows of the GEMM operand layout: batch rounded to 16, or to 128 above 128 (two
        // whole 128-row groups for the batch-M GEMMs and the pipelined kernel's halves)
        NR = Bm > 128 ? round_up(Bm, 128) : std::max(16, round_up(Bm, 16));
        h32.alloc((size_t)2 * Bm * dp);
        hb.alloc((size_t)2 * NR * dp);
        q32.alloc((size_t)Bm * dp);
        att_b.alloc((size_t)NR * dp);
        mid32.alloc((size_t)Bm * dp);
        mid_b.alloc((size_t)NR * dp);
        up_b.alloc((size_t)NR * fp);
        attn_cnt.alloc((size_t)std::max(Bm, kPfRows));
        lm_part.alloc((size_t)(dm.Vp / 128) * Bm);
        dbg_ts.alloc(65536 + 256 * 1024);
        exit_part.alloc((size_t)(dp / 16 + 1) * Bm * 3);  // per 128-row tile (split-K) or 16-feature slice (batch-M)
        for (DevBuf<int>* b : {&layer, &out_layer, &exit_cnt, &iter_counter, &cur_iter}) b->alloc(4);
        status.alloc((size_t)Bm);
        first_accept.alloc((size_t)Bm);
        accept.alloc((size_t)Bm);
        conf.alloc((size_t)L * Bm);
        fixed_conf.alloc((size_t)L * Bm);
        rec_stride = round_up(2 * Bm + 4 + L * Bm, 32);
        rec.alloc((size_t)rec_cap * rec_stride);
        CK(cudaHostAlloc(&rec_host, sizeof(int) * rec_stride, cudaHostAllocDefault));
        {
            std::vector<double> lam((size_t)L);
            for (int l = 1; l <= L; ++l) lam[(size_t)l - 1] = threshold_at(cfg.lambda0, cfg.gamma, cfg.lambda_min, l);
            lambdas.alloc((size_t)L);
            CK(cudaMemcpy(lambdas.p, lam.data(), sizeof(double) * L, cudaMemcpyHostToDevice));
        }
        run_ctl.alloc(4);
        set_run_active(1);
        run_rem.alloc((size_t)Bm);
        run_clock.alloc(1);
        run_log.alloc((size_t)2 * rec_cap);
        CK(cudaHostAlloc(&cont_host, sizeof(int) * 4, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer((void**)&cont_dev, cont_host, 0));

        el::init_kernel_attributes();
        el::init_iter_attributes();
        el::init_pipe_attributes();
        mbar.alloc(2048 + 32 * 1024);
        mtcnt.alloc(el::kINumGemm * 64);
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        slot_bpl.assign((size_t)dm.slots, -1);
        ensure_bpl(1);
        CK(cudaStreamSynchronize(stream));
        slot_bpl.assign((size_t)dm.slots, -1);
    }

    void set_run_active(int v) {
        const int w[2] = {v, 0};
        CK(cudaMemcpy(run_ctl.p, w, sizeof w, cudaMemcpyHostToDevice));
    }
    void reset_allocator() {
        std::vector<int> st((size_t)cfg.pool_blocks);
        for (int i = 0; i < cfg.pool_blocks; ++i) st[(size_t)i] = cfg.pool_blocks - 1 - i;  // pops 0 first
        CK(cudaMemcpyAsync(stack.p, st.data(), sizeof(int) * st.size(), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        top = cfg.pool_blocks;
        peak = 0;
        slot_bpl.assign((size_t)dm.slots, -1);
        store.clear();
        store_ready = false;
    }

    // tables / attention workspace sized for bpl blocks per (seq, layer)
    void ensure_bpl(int bpl) {
        if (bpl <= dm.bpl_max) return;
        for (int b : slot_bpl)
            if (b >= 0) fail(EL_LOGIC_ERROR, "block tables cannot grow while sequences are live");
        dm.bpl_max = bpl;
        tables.alloc((size_t)dm.slots * dm.L * bpl);
        plan_attention();
        invalidate_graphs();
    }

    // attention split: ~4 CTAs per SM worth of (sequence, chunk) work items; a
    // ring of stages sized so two CTAs fit per SM when the block pair allows it
    int opt_attn_cb = 0, opt_attn_stages = 0, opt_splits_cap = 8, opt_fill_splits = 4, opt_nsplit = 2, opt_cta_target = 148;
    void plan_attention() {
        const int bpl = std::max(1, dm.bpl_max);
        const int B = dm.Bmax;
        // items of ~4 blocks keep the queue balanced; the persistent producer
        // streams across item boundaries, so short items cost no pipeline drain
        // partial slots per sequence: one per CTA segment (<= blocks of the sequence)
        attn_cb = 1;
        attn_max_chunks = std::min(std::max(bpl, enc_blocks), 128);
        if (enc_blocks > 128) fail(EL_INVALID_ARGUMENT, "cross-attention: more than 128 encoder blocks unsupported");
        if (bpl > 128) fail(EL_INVALID_ARGUMENT, "attention: more than 128 KV blocks per sequence unsupported");
        if (B > 256) fail(EL_INVALID_ARGUMENT, "attention: batch > 256 unsupported");
        (void)opt_attn_cb;
        const int stage_bytes = el::attn_stage_bytes(dm);
        // one persistent CTA per SM with as many block stages as shared memory holds
        // ~3 stages (<= 160 KB): leaves room for a co-resident GEMM CTA, so with
        // PDL the next/previous kernel's prologue overlaps this one
        attn_stages = opt_attn_stages ? opt_attn_stages : std::min(8, std::max(2, (160 * 1024) / stage_bytes));
        while (attn_stages > 1 && el::attn_smem_bytes(dm, attn_stages) > 227 * 1024) --attn_stages;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        attn_grid = sms * el::attn_ctas_per_sm(dm, attn_stages);
        if (opt_attn_grid > 0) attn_grid = std::min(attn_grid, opt_attn_grid);  // probe: fewer CTAs
        attn_o.alloc((size_t)std::max(B, kPfRows) * attn_max_chunks * dm.dp, false);
        attn_ml.alloc((size_t)std::max(B, kPfRows) * attn_max_chunks * 2 * std::max(1, cfg.n_heads), false);
        invalidate_graphs();
    }

    void invalidate_graphs() {
        for (auto& kv : graphs) {
            if (kv.second.x) cudaGraphExecDestroy(kv.second.x);
            if (kv.second.g) cudaGraphDestroy(kv.second.g);
        }
        graphs.clear();
    }

    // ---- GEMM plans ----
    // split-K cluster size: aim at ~one CTA per SM, at most 8 (portable clusters)
    int pick_splits(int m_tiles, int kb_total) const {
        int s = (opt_cta_target + m_tiles / 2) / m_tiles;
        return std::max(1, std::min({s, opt_splits_cap, kb_total}));
    }
    // n_pad: padded batch; the plan splits it into ns column groups of nc (MMA N)
    // so each CTA's split-K partial (and its DSMEM reduction) stays small
    el::GemmPlan make_plan(const uint16_t* A, const uint16_t* Bp, size_t b_par_stride, int m_tiles, int k, int n_pad,
                           bool tile, int forced_splits = 0) {
        el::GemmPlan p;
        p.A = A;
        p.Bp = Bp;
        p.b_par_stride = b_par_stride;
        p.m_tiles = m_tiles;
        p.kb_total = k / 64;
        int nc = n_pad;
        if (!tile && opt_nsplit > 1) nc = std::max(16, round_up(ceil_div(n_pad, opt_nsplit), 16));
        const int ns = ceil_div(n_pad, nc);
        n_pad = nc;
        p.splits = forced_splits ? forced_splits : pick_splits(m_tiles * ns, p.kb_total);
        const int kb_max = ceil_div(p.kb_total, p.splits);
        p.n_pad = n_pad;
        const int stage = 128 * 64 * 2 + n_pad * 64 * 2;
        // LM head: <= ~100 KB so two CTAs share an SM (251 tiles in one wave)
        p.stages = std::max(1, std::min(kb_max, (tile ? 100 * 1024 : 200 * 1024) / stage));
        p.smem_bytes = el::gemm_smem_bytes(n_pad, p.stages, tile);
        while (p.smem_bytes > 227 * 1024 && p.stages > 1) p.smem_bytes = el::gemm_smem_bytes(n_pad, --p.stages, tile);
        int cols = 32;
        while (cols < n_pad) cols <<= 1;
        p.tmem_cols = cols;
        return p;
    }
    Plans& plans_for(int B) {
        const int n_pad = std::max(16, round_up(B, 16));
        auto it = plans.find(n_pad);
        if (it != plans.end()) return it->second;
        const int dp = dm.dp, fp = dm.fp, Bm = dm.Bmax, L = dm.L;
        Plans P;
        P.n_pad = n_pad;
        (void)Bm;
        const size_t hpar = (size_t)NR * dp;  // hidden-state parity stride
        P.qkv = make_plan(wqkv.p, hb.p, hpar, 3 * dp / 128, dp, n_pad, false);
        P.wo = make_plan(wo.p, att_b.p, 0, dp / 128, dp, n_pad, false);
        P.up = make_plan(wup.p, mid_b.p, 0, fp / 128, dp, n_pad, false);
        P.down = make_plan(wdown.p, up_b.p, 0, dp / 128, fp, n_pad, false);
        P.lm = make_plan(lm.p, hb.p, hpar, dm.Vp / 128, dp, n_pad, true, 1);
        P.fill = make_plan(wqkv.p, hb.p, hpar, (L - 1) * (2 * dp / 128), dp, n_pad, false,
                           std::min(opt_fill_splits, dp / 64));
        invalidate_graphs();  // workspace may have moved
        return plans.emplace(n_pad, P).first->second;
    }

    // ---- persistent decode-iteration kernel plan ----
    // split-K: aim at one unit per CTA (units = m_tiles * splits <= grid), >= 2 splits
    // cap (fewer splits: less partial traffic to reduce): 8, or 16 at batch >= 256 where the
    // mainloop of a unit dominates (measured c5 -1.6 %, c3 -0.5 %, c2 +1.3 % with 16)
    int mega_splits(int m_tiles, int kb_total, int n_pad, int grid = 0) const {
        int s = std::max(1, (grid ? grid : mega_grid) / m_tiles);
        const int cap = opt_mega_splits_cap ? opt_mega_splits_cap : (n_pad >= 256 ? 16 : 8);
        s = std::min({s, kb_total, cap});
        return std::max(s, std::min(2, kb_total));
    }
    // pipe_grid > 0: the plan of the pipelined kernel -- its GEMMs run on pipe_grid CTAs, one
    // 128-row half of the batch at a time (batch-M units over one row group, split-K units sized
    // for that CTA count)
    el::IterPlan& mplan_for(int B, int nr_override = 0, int pipe_grid = 0) {
        const int n_pad = std::max(16, round_up(B, 16));
        const int NR = nr_override ? nr_override : this->NR;  // activation rows of the operand layout
        // plan_encoder: the plan of the T5 encoder stack (its own weights and layer count)
        const bool encp = plan_encoder;
        const int key = n_pad + (nr_override ? 100000 : 0) + (pipe_grid ? 1000000 * pipe_grid : 0) +
                        (encp ? 400000000 : 0);
        auto it = mplans.find(key);
        if (it != mplans.end()) return it->second;
        const int dp = dm.dp, fp = dm.fp, L = encp ? cfg.encoder_layers : dm.L;
        const uint16_t *Wqkv = encp ? e_wqkv.p : wqkv.p, *Wo = encp ? e_wo.p : wo.p, *Wup = encp ? e_wup.p : wup.p,
                       *Wdown = encp ? e_wdown.p : wdown.p;
        const int cap = 227 * 1024 - el::iter_smem_fixed();
        // attention ring of K|V|q stages (with the branch-free consumer a third stage pays at
        // d <= 768; at d = 1024 two leave room for the merge buffer and weight prefetch)
        const int att_stage = el::attn_stage_bytes(dm);
        mega_att_stages = std::min(8, cap / att_stage);
        // 3 stages at d <= 768 (c2: -1.6 % iteration time), 2 at d = 1024 (3 measured +2 %) and
        // in T5 mode (+0.8 %)
        mega_att_stages = std::min(mega_att_stages, opt_mega_att_stages ? opt_mega_att_stages
                                                                        : (dp <= 768 && cfg.encoder_len == 0 ? 3 : 2));
        if (mega_att_stages < 2) fail(EL_INVALID_ARGUMENT, "persistent kernel: attention ring does not fit");
        mega_grid = sms;
        const int ggrid = pipe_grid ? pipe_grid : mega_grid;  // CTAs running the GEMM phases
        el::IterPlan P{};
        P.pipe_att_ctas = pipe_grid ? mega_grid - pipe_grid : 0;
        auto g = [&](const uint16_t* A, int m_tiles, int kb_total, int layer_rows, int row_off, int splits) {
            el::IterGemm x;
            x.A = A;
            x.m_tiles = m_tiles;
            x.kb_total = kb_total;
            x.splits = splits;
            x.layer_rows = layer_rows;
            x.row_off = row_off;
            x.mode = 0;
            x.nt = 0;
            return x;
        };
        P.g[el::kIQkv] = g(Wqkv, 3 * dp / 128, dp / 64, 3 * dp / 128, 0, mega_splits(3 * dp / 128, dp / 64, n_pad, ggrid));
        P.g[el::kIWo] = g(Wo, dp / 128, dp / 64, dp / 128, 0, mega_splits(dp / 128, dp / 64, n_pad, ggrid));
        P.g[el::kIUp] = g(Wup, fp / 128, dp / 64, fp / 128, 0, mega_splits(fp / 128, dp / 64, n_pad, ggrid));
        P.g[el::kIDown] = g(Wdown, dp / 128, fp / 64, dp / 128, 0,
                            opt_mega_down_splits ? std::min(opt_mega_down_splits, fp / 64)
                                                 : mega_splits(dp / 128, fp / 64, n_pad, ggrid));
        // fill: full-K units (direct epilogue) at large N, where split-K partials would outweigh the weights
        P.g[el::kIQc] = g(wqc.p, dp / 128, dp / 64, dp / 128, 0, mega_splits(dp / 128, dp / 64, n_pad));
        P.g[el::kIWoc] = g(woc.p, dp / 128, dp / 64, dp / 128, 0, mega_splits(dp / 128, dp / 64, n_pad));
        int fs = opt_mega_fill_splits ? opt_mega_fill_splits : (n_pad >= 128 ? 1 : 2);  // (c2: 2 < 3 < 4 < 1)
        fs = std::min(fs, dp / 64);
        P.g[el::kIFill] = g(Wqkv, 2 * dp / 128, dp / 64, 3 * dp / 128, dp / 128, fs);
        P.n_pad = n_pad;
        // batch-M full-K GEMMs (no split-K reduce phase) for QKV / W_o / up at small batch
        int nt_max = 16, bm_w = 0;  // bm_w: the largest unit weight slab (nt rows x K)
        // streamed batch-M weights (auto: off -- -2.4 % full-depth iteration time in the pipelined
        // kernel, but +1.5 % at the early-exit bench (c5, same-box A/B, scripts/ab_early.sh))
        const bool wstream = opt_mega_bm_wstream > 0;
        // batch > 128: units cover 128-row groups of an activation layout with 128-row multiples
        const bool bm = n_pad <= opt_mega_bm_max && (n_pad <= 128 || NR % 128 == 0);
        if (bm) {
            for (int k : {el::kIQkv, el::kIWo, el::kIUp, el::kIQc, el::kIWoc, el::kIDown}) {
                // down (K = 4d): batch-M only at batch <= 64, where its 16-row weight slab fits (the
                // pipelined kernel's down stays split-K: a batch-M down with streamed weights, 1 MB of
                // activations per full-K unit, measured +21 % iteration time at c5)
                if (k == el::kIDown && (n_pad > 64 || !opt_mega_bm_down || pipe_grid)) continue;
                el::IterGemm& x = P.g[k];
                const int F = x.m_tiles * 128;
                // row groups of 128 batch rows (the pipelined kernel runs one group per phase)
                const int R = (n_pad > 128 && !pipe_grid) ? 2 : 1;
                int nt = k == el::kIDown ? 16 : opt_mega_bm_nt_min;
                if (pipe_grid) {
                    // the fewest waves over the GEMM CTAs, then the smallest N (multiple of 16 dividing
                    // F) with a unit weight slab of at most 128 KB (c5: nt 64 / 32 / 64 for QKV / W_o /
                    // up -- QKV in one wave of 48 units -- with 100 attention CTAs: -5.2 % iteration
                    // time vs 96 KB slabs and 92 attention CTAs, scripts/pipe_sweep.py)
                    const int max_nt = wstream ? 128 : std::max(16, std::min(128, (128 * 1024) / (x.kb_total * 128) / 16 * 16));
                    int best = 16, best_w = 1 << 30;
                    for (int c = 16; c <= max_nt; c += 16) {
                        if (F % c) continue;
                        if (128 % c) continue;  // a unit's rows stay inside one 128-row weight tile
                        const int w = ceil_div(F / c, ggrid);
                        if (w < best_w) { best_w = w; best = c; }
                    }
                    nt = best;
                } else {
                    while (nt < 128 && F / nt * R > ggrid) nt *= 2;
                }
                x.mode = 1;
                x.nt = nt;
                nt_max = std::max(nt_max, nt);
                if (!wstream) bm_w = std::max(bm_w, x.kb_total * nt * 128);
            }
        }
        const int stage = 128 * 64 * 2 + n_pad * 128;
        P.stage_bytes = stage;
        // batch-M ring: stages of bm_kc activation k-blocks (NR rows each, ~32 KB per copy), then the
        // unit's weights (nt_max rows x dp/64 k-blocks); 16 KB slack for the MMA's full-tile A reads
        // The batch-M weight buffer sits at the end of the ring region (bm_woff), past the attention
        // stages, the batch-M activation stages and the weight-streaming ring + LM transpose buffer,
        // so a prefetch into it never collides with the phase in flight.
        const int ring_att = mega_att_stages * att_stage;
        P.bm_rows = NR;
        // batch > 128: units cover one 128-row group; the pipelined kernel at batch <= 128: one 64-row half
        const bool half64 = pipe_grid && n_pad <= 128;
        P.bm_grp = n_pad > 128 ? 128 : half64 ? (n_pad > 64 ? 64 : 32) : NR;
        P.bm_kc = std::max(1, std::min(dp / 64, (opt_mega_bm_chunk_kb ? opt_mega_bm_chunk_kb * 1024 : 32768) /
                                                     (P.bm_grp * 128)));
        P.bm_m = ((n_pad <= 64 || half64) && !opt_mega_bm_m128) ? 64 : 128;
        P.att_early = opt_mega_att_early;
        P.lm_keep = opt_lm_keep;
        P.tcnt = mtcnt.p;
        P.bm_wstream = (bm && wstream) ? 1 : 0;
        // a stage: bm_kc activation k-blocks (+ with streamed weights bm_kc weight k-blocks of nt_max rows)
        P.bm_astage = P.bm_kc * (P.bm_grp + (P.bm_wstream ? nt_max : 0)) * 128;
        P.bm_woff = (cap - bm_w) / 1024 * 1024;
        P.bm_stages = std::max(2, std::min(P.bm_wstream ? 6 : 4, (P.bm_woff - 16384) / P.bm_astage));
        if (bm && P.bm_stages * P.bm_astage > P.bm_woff)
            fail(EL_INVALID_ARGUMENT, "persistent kernel: batch-M ring does not fit");
        // (the pipelined kernel's GEMM CTAs run no attention: their weight slab may overlap the
        //  attention ring; its split-K / tail ring keeps the whole region, as no slab prefetch is
        //  in flight while it runs -- the next layer's QKV weights are not prefetched there)
        P.bm_prefetch = (bm && !P.bm_wstream && opt_mega_bm_prefetch && (pipe_grid || ring_att <= P.bm_woff)) ? 1 : 0;
        // weight-streaming ring + transpose buffer stay below the weight buffer when weights are
        // prefetched into it during other phases
        const int ws_cap = (bm && P.bm_prefetch && !pipe_grid) ? P.bm_woff : cap;
        P.stages = std::min(8, (ws_cap - el::kIterTbufBytes) / stage);
        if (P.stages < 2) fail(EL_INVALID_ARGUMENT, "persistent kernel: GEMM ring does not fit");
        P.gemm_ring = P.stages * stage;
        // attention merge buffer right after the attention stages (a segment's stage is released
        // before its merge) when it fits below the batch-M weight buffer
        const int mbuf = 8 * dp * 4;
        P.att_mbuf_off = (opt_att_mbuf && ring_att + mbuf <= ((bm && P.bm_prefetch) ? P.bm_woff : cap)) ? ring_att : 0;
        P.ring_bytes = round_up(std::max({ring_att + (P.att_mbuf_off ? mbuf : 0), P.gemm_ring + el::kIterTbufBytes,
                                          P.bm_stages * P.bm_astage + 16384, bm ? P.bm_woff + bm_w : 0}), 1024);
        P.lm_tiles = dm.Vp / 128;
        P.lm_pair = (opt_lm_pair && !pipe_grid && n_pad <= 256 &&
                     P.stages * (2 * 16384 + n_pad * 128) + el::kIterTbufBytes <= P.ring_bytes)
                        ? ((opt_lm_pair == 2 && n_pad != 128) ? 1 : opt_lm_pair) : 0;  // (2 needs M = 128 rows)
        P.lm_stages = 0;
        if (pipe_grid && n_pad <= 128) {  // pipelined kernel: the pair units' own ring (full3 / empty3)
            P.lm_stages = std::min(4, (P.ring_bytes - el::kIterTbufBytes) / (2 * 16384 + n_pad * 128));
            P.lm_pair = P.lm_stages >= 2 ? ((opt_lm_pair == 2 && n_pad == 128) ? 2 : 1) : 0;
        }
        // transposed tail LM units: 48 KB stages (batch 256: the weight-streaming stage size; batch 128:
        // the pair stage, which must fit next to the transpose buffer)
        P.lm_tail_tr = opt_lm_tail && ((n_pad == 256 && NR % 128 == 0) ||
                                       (n_pad == 128 && P.stages * (2 * 16384 + n_pad * 128) + el::kIterTbufBytes <=
                                                            P.ring_bytes)) ? 1 : 0;
        if (el::iter_max_ctas_per_sm(dm, P.ring_bytes) < 1)
            fail(EL_CUDA_ERROR, "persistent kernel does not fit on an SM (%d bytes)", el::iter_smem_bytes(P.ring_bytes));
        size_t units = 0;
        for (int k = 0; k < el::kINumGemm; ++k)
            if (k != el::kIFill) units = std::max(units, (size_t)P.g[k].m_tiles * P.g[k].splits);
        if (fs > 1) units = std::max(units, (size_t)(L - 1) * (2 * dp / 128) * fs);
        const size_t need = units * n_pad * 128;
        if (mpart.n < need) {
            mpart.alloc(need, false);
            for (auto& kv : mplans) kv.second.part = mpart.p;
        }
        P.part = mpart.p;
        P.bar = mbar.p;
        el::IterMaps MM{};
        for (int k : {el::kIQkv, el::kIWo, el::kIUp, el::kIQc, el::kIWoc, el::kIDown}) {
            const el::IterGemm& x = P.g[k];
            if (!x.mode || !x.A || P.bm_wstream) continue;  // (streamed weights: 1-D copies, no tensor map)
            MM.w[k] = make_bm_map(x.A, (size_t)L * x.layer_rows * x.kb_total, x.nt, x.kb_total);
        }
        mmaps[key] = MM;
        P.map_key = key;
        return mplans.emplace(key, P).first->second;
    }
    void launch_pipe(int B) {
        const int ga64 = cfg.technique == EL_TECH_SOFTMAX ? pipe_att64_sm : pipe_att64;
        const int ga = std::min(std::max(B <= 64 ? pipe_att32 : B <= 128 ? ga64 : pipe_att, 16), sms - 16);
        el::IterPlan& P = mplan_for(B, 0, sms - ga);
        if (!P.g[el::kIQkv].mode || !P.g[el::kIWo].mode || !P.g[el::kIUp].mode)
            fail(EL_RUNTIME_ERROR, "pipelined kernel: needs batch-M QKV / W_o / up phases");
        if (cfg.technique == EL_TECH_SOFTMAX && !P.lm_pair)
            fail(EL_RUNTIME_ERROR, "pipelined kernel: the softmax check's LM pair ring does not fit");
        el::DevState s = state(false, B);
        // attention CTAs have the whole ring region to themselves: as many stages as fit
        s.attn_stages = std::min(8, P.ring_bytes / el::attn_stage_bytes(dm));
        if (s.attn_stages < 2) fail(EL_INVALID_ARGUMENT, "pipelined kernel: attention ring does not fit");
        s.attn_seg_cost = opt_attn_seg_cost >= 0 ? opt_attn_seg_cost : 0;
        if (std::getenv("EL_PIPE_DEBUG"))
            fprintf(stderr, "pipe: grid %d att %d ring %d att_stages %d stages %d stage_bytes %d n_pad %d bm_grp %d "
                    "nt %d/%d/%d splits down %d fill %d\n", mega_grid, P.pipe_att_ctas, P.ring_bytes, s.attn_stages,
                    P.stages, P.stage_bytes, P.n_pad, P.bm_grp, P.g[el::kIQkv].nt, P.g[el::kIWo].nt, P.g[el::kIUp].nt,
                    P.g[el::kIDown].splits, P.g[el::kIFill].splits);
        el::launch_pipe(s, P, mmaps[P.map_key], mega_grid, stream);
    }
    void launch_mega(int B) {
        if (pipe_for(B)) {
            launch_pipe(B);
            return;
        }
        el::IterPlan& P = mplan_for(B);
        el::DevState s = state(false, B);
        s.attn_stages = mega_att_stages;
        // auto: charge row starts at batch <= 64, where a row spans 2-3 CTA ranges (c2 +1.2 %);
        // at batch 128 the same cost measured -1.6 % end to end
        s.attn_seg_cost = opt_attn_seg_cost >= 0 ? opt_attn_seg_cost : (B <= 64 ? 2 : 0);
        el::launch_iter(s, P, mmaps[P.map_key], mega_grid, stream);
    }

    el::DevState state(bool prefill, int B) {
        el::DevState s{};
        s.dm = dm;
        s.wqkv = wqkv.p; s.wo = wo.p; s.wup = wup.p; s.wdown = wdown.p; s.emb = emb.p; s.lm = lm.p;
        s.probe_w = probe_w.p; s.probe_b = probe_b;
        s.kpool = kpool.p; s.vpool = vpool.p; s.tables = tables.p;
        if (prefill) s.rows = el::Rows{pf_slot.p, pf_pos.p, pf_tok.p, B};
        else s.rows = el::Rows{row_slot.p, row_pos.p, row_tok.p, B};
        s.NR = NR;
        s.h32 = h32.p; s.hb = hb.p; s.q32 = q32.p; s.att_b = att_b.p; s.mid32 = mid32.p; s.mid_b = mid_b.p;
        s.up_b = up_b.p;
        s.attn_o = attn_o.p; s.attn_ml = attn_ml.p; s.attn_cnt = attn_cnt.p;
        s.attn_max_chunks = attn_max_chunks; s.attn_cb = attn_cb; s.attn_stages = attn_stages;
        s.dbg = dbg;
        s.dbg_ts = dbg_ts.p;
        s.attn_grid = attn_grid;
        s.attn_heads = std::max(1, cfg.n_heads);
        s.attn_hd = dm.d / s.attn_heads;
        s.attn_scale = (float)(1.0 / std::sqrt((double)s.attn_hd));
        s.lm_part = lm_part.p;
        s.layer = layer.p; s.out_layer = out_layer.p; s.status = status.p; s.first_accept = first_accept.p;
        s.accept = accept.p; s.conf = conf.p; s.exit_cnt = exit_cnt.p; s.cont_host = cont_dev;
        s.exit_part = exit_part.p;
        s.fuse_exit = (!prefill && fuse_exit_active()) ? 1 : 0;
        s.lambdas = lambdas.p; s.fixed_conf = fixed_conf.p;
        s.technique = prefill ? el::kNever : cfg.technique;
        s.exit_layer = cfg.exit_layer;
        s.use_cond = 0;
        s.iter_counter = prefill ? cur_iter.p + 1 : iter_counter.p;  // prefill: scratch counter
        s.cur_iter = prefill ? cur_iter.p + 2 : cur_iter.p;
        s.rec = rec.p; s.rec_stride = rec_stride;
        s.rec_cap = rec_cap;
        s.enc_len = cfg.encoder_len;
        s.enc_blocks = enc_blocks;
        s.wqc = wqc.p; s.wkvc = wkvc.p; s.woc = woc.p;
        s.ckpool = ckpool.p; s.cvpool = cvpool.p; s.ctables = ctables.p;
        s.turn_layer = 0;
        s.turn_defer = 0;
        s.turn_token = 0;
        s.row_exit = row_exit.p;
        s.hstore = hstore.p;
        s.row_seq = row_seq.p;
        s.run_active = run_ctl.p;
        return s;
    }

    // one layer's kernels (the WHILE body). PDL: every kernel after the first
    // may launch while its predecessor drains (weights / old KV blocks are
    // prefetched before griddepcontrol.wait).
    void launch_layer(const el::DevState& s, Plans& P) {
        if (body_head) el::launch_layer_head(s, stream);
        el::launch_gemm(el::kGemmQkv, P.qkv, s, stream, body_head && pdl);
        el::launch_attention(s, stream, pdl);
        el::launch_gemm(el::kGemmWo, P.wo, s, stream, pdl);
        el::launch_gemm(el::kGemmUp, P.up, s, stream, pdl);
        el::launch_gemm(el::kGemmDown, P.down, s, stream, pdl);
        if (s.technique == el::kSoftmax) el::launch_gemm(el::kGemmLmCheck, P.lm, s, stream, pdl);
        if (!s.fuse_exit) el::launch_exit(s, stream, pdl);
    }
    // tail: the skipped-layer fill and the greedy LM head both only read h_e, so
    // they run as two graph branches (fork/join through a second stream)
    void launch_tail(const el::DevState& s, Plans& P) {
        const bool fill = s.technique != el::kNever, lmf = s.technique != el::kSoftmax;
        if (fill && lmf) {
            CK(cudaEventRecord(ev_fork, stream));
            CK(cudaStreamWaitEvent(stream2, ev_fork, 0));
            el::launch_gemm(el::kGemmFill, P.fill, s, stream2, false);
            CK(cudaEventRecord(ev_join, stream2));
            el::launch_gemm(el::kGemmLmFinal, P.lm, s, stream, false);
            CK(cudaStreamWaitEvent(stream, ev_join, 0));
            el::launch_finish(s, stream, false);
            return;
        }
        if (fill) el::launch_gemm(el::kGemmFill, P.fill, s, stream, false);
        if (lmf) el::launch_gemm(el::kGemmLmFinal, P.lm, s, stream, false);
        el::launch_finish(s, stream, pdl);
    }
    // The exit check runs inside the down-projection epilogue when it needs no
    // confidence reduction (never / always_at / injected); for state and classifier
    // the separate exit kernel measured faster (its B CTAs read whole rows in parallel)
    bool fuse_exit_active() const {
        if (!fuse_exit) return false;
        if (fuse_exit_all) return cfg.technique != EL_TECH_SOFTMAX;
        return cfg.technique == EL_TECH_NEVER || cfg.technique == EL_TECH_ALWAYS_AT || cfg.technique == EL_TECH_FIXED;
    }
    int launches_per_iteration(int e) const {
        if (mega_for(in_session ? sess_B : dm.Bmax)) return 1;
        const bool fused = fuse_exit_active();
        const int per_layer = (fused ? 5 : 6) + (cfg.technique == EL_TECH_SOFTMAX ? 1 : 0) + (body_head ? 1 : 0);
        return 1 + e * per_layer + (cfg.technique != EL_TECH_NEVER ? 1 : 0) +
               (cfg.technique != EL_TECH_SOFTMAX ? 1 : 0) + 1;
    }

    // eager iteration: host reads the device continue flag after each layer
    void iteration_eager(int B) {
        Plans& P = plans_for(B);
        el::DevState s = state(false, B);
        el::launch_embed(s, stream);
        for (int l = 1; l <= dm.L; ++l) {
            launch_layer(s, P);
            CK(cudaStreamSynchronize(stream));
            if (*(volatile int*)cont_host == 0) break;
        }
        launch_tail(s, P);
    }

    Graph& graph_for(int B) {
        auto it = graphs.find(B);
        if (it != graphs.end()) return it->second;
        Plans& P = plans_for(B);
        Graph G;
        CK(cudaGraphCreate(&G.g, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, G.g, 1, cudaGraphCondAssignDefault));
        el::DevState s = state(false, B);
        s.use_cond = 1;
        s.cond = h;
        s.cont_host = nullptr;
        const cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        // segment 1: embed
        CK(cudaStreamBeginCaptureToGraph(stream, G.g, nullptr, nullptr, 0, mode));
        el::launch_embed(s, stream);
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        CK(cudaStreamGetCaptureInfo(stream, &cs, nullptr, nullptr, &deps, &ndeps));
        std::vector<cudaGraphNode_t> dv(deps, deps + ndeps);
        CK(cudaStreamEndCapture(stream, &G.g));
        // WHILE(layer loop)
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t wnode;
        CK(cudaGraphAddNode(&wnode, G.g, dv.data(), dv.size(), &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, mode));
        launch_layer(s, P);
        CK(cudaStreamEndCapture(stream, &body));
        // tail: fill, lm head, finish
        CK(cudaStreamBeginCaptureToGraph(stream, G.g, &wnode, nullptr, 1, mode));
        launch_tail(s, P);
        CK(cudaStreamEndCapture(stream, &G.g));
        CK(cudaGraphInstantiate(&G.x, G.g, 0));
        return graphs.emplace(B, G).first->second;
    }

    void iteration(int B) {
        if (mega_for(B)) {
            launch_mega(B);
        } else if (use_graph) {
            Graph& G = graph_for(B);
            CK(cudaGraphLaunch(G.x, stream));
        } else {
            iteration_eager(B);
        }
    }

    // ---- allocator (kv_cache.cpp:78-106, 182-194) ----
    int bpl_for(int capacity_tokens) const { return ceil_div(capacity_tokens, dm.bc); }
    bool can_allocate(int capacity_tokens) const { return (long)bpl_for(capacity_tokens) * dm.L <= top; }
    int free_slot() const {
        for (int s = 0; s < dm.slots; ++s)
            if (slot_bpl[(size_t)s] < 0) return s;
        fail(EL_RUNTIME_ERROR, "no free sequence slot");
    }
    int allocate(int capacity_tokens) {
        const int bpl = bpl_for(capacity_tokens);
        if ((long)bpl * dm.L > top)
            fail(EL_KV_OUT_OF_MEMORY, "allocate: need %ld blocks, %d free", (long)bpl * dm.L, top);
        if (bpl > dm.bpl_max) fail(EL_RUNTIME_ERROR, "allocate: %d blocks per layer exceed the table width %d", bpl, dm.bpl_max);
        const int slot = free_slot();
        el::launch_kv_alloc(stack.p, top, tables.p, dm, slot, bpl, stream);
        top -= bpl * dm.L;
        peak = std::max(peak, cfg.pool_blocks - top);
        slot_bpl[(size_t)slot] = bpl;
        return slot;
    }
    void release(int slot) {
        const int bpl = slot_bpl[(size_t)slot];
        el::launch_kv_release(stack.p, top, tables.p, dm, slot, bpl, stream);
        top += bpl * dm.L;
        slot_bpl[(size_t)slot] = -1;
    }

    // ---- prefill of newly admitted sequences (engine.cpp:166-181), batched
    //      across sequences (attention is per sequence, so this is exact) ----
    struct PfSeq {
        int slot;
        std::vector<int> toks;  // prompt[0 .. P-2]
    };
    void prefill(const std::vector<PfSeq>& seqs) {
        if (use_mega != 0) {
            prefill_batched(seqs);
            return;
        }
        int maxn = 0;
        for (const auto& q : seqs) maxn = std::max(maxn, (int)q.toks.size());
        std::vector<int> hs, hp, ht;
        for (int j = 0; j < maxn; ++j) {
            hs.clear(); hp.clear(); ht.clear();
            for (const auto& q : seqs)
                if ((int)q.toks.size() > j) {
                    hs.push_back(q.slot);
                    hp.push_back(j);
                    ht.push_back(q.toks[(size_t)j]);
                }
            const int B = (int)hs.size();
            CK(cudaMemcpyAsync(pf_slot.p, hs.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(pf_pos.p, hp.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(pf_tok.p, ht.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            Plans& P = plans_for(B);
            el::DevState s = state(true, B);
            s.cont_host = nullptr;
            el::launch_embed(s, stream);
            for (int l = 1; l <= dm.L; ++l) {
                el::launch_gemm(el::kGemmQkv, P.qkv, s, stream, false);
                el::launch_attention(s, stream, pdl);
                el::launch_gemm(el::kGemmWo, P.wo, s, stream, pdl);
                el::launch_gemm(el::kGemmUp, P.up, s, stream, pdl);
                el::launch_gemm(el::kGemmDown, P.down, s, stream, pdl);
                el::launch_exit(s, stream, pdl);
            }
            el::launch_advance(s, stream);
            CK(cudaStreamSynchronize(stream));  // host vectors are reused next step
        }
    }

    // Batched causal prefill on the persistent kernel: the rows of one launch are prompt
    // positions (position-major across the admitted sequences, up to max_batch rows).  Each
    // layer's QKV phase writes the K/V of every row before its attention phase, and earlier
    // positions were written by earlier launches, so row (s, p) attends over exactly positions
    // 0..p of sequence s -- the reference's token-by-token prefill, batched over positions.
    void prefill_batched(const std::vector<PfSeq>& seqs) {
        std::vector<int> hs, hp, ht;
        int maxn = 0;
        for (const auto& q : seqs) maxn = std::max(maxn, (int)q.toks.size());
        auto flush = [&]() {
            const int B = (int)hs.size();
            if (!B) return;
            CK(cudaMemcpyAsync(pf_slot.p, hs.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(pf_pos.p, hp.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(pf_tok.p, ht.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            el::IterPlan& P = mplan_for(B, kPfRows);
            el::DevState s = state(true, B);
            s.cont_host = nullptr;
            s.prefill = 1;
            // the prefill activation set: kPfRows rows (act layout stride kPfRows)
            s.NR = kPfRows;
            s.h32 = pf_h32.p; s.hb = pf_hb.p; s.q32 = pf_q32.p; s.att_b = pf_att_b.p;
            s.mid32 = pf_mid32.p; s.mid_b = pf_mid_b.p; s.up_b = pf_up_b.p;
            s.attn_stages = mega_att_stages;
            el::launch_iter(s, P, mmaps[P.map_key], mega_grid, stream);
            CK(cudaStreamSynchronize(stream));  // host vectors are reused
            hs.clear(); hp.clear(); ht.clear();
        };
        for (int j = 0; j < maxn; ++j)
            for (const auto& q : seqs)
                if ((int)q.toks.size() > j) {
                    if ((int)hs.size() == kPfRows) flush();
                    hs.push_back(q.slot);
                    hp.push_back(j);
                    ht.push_back(q.toks[(size_t)j]);
                }
        flush();
    }

    // ---- records ----
    struct IterOut {
        int out_layer;
        std::vector<int> tok, acc;
        std::vector<float> conf;  // [L][B]
    };
    IterOut read_iteration(int iter_index, int B) {
        IterOut o;
        const int cur = iter_index % rec_cap, Bm = dm.Bmax, L = dm.L;
        // the whole packed record in one copy through pinned staging
        CK(cudaMemcpyAsync(rec_host, rec.p + (size_t)cur * rec_stride, sizeof(int) * rec_stride, cudaMemcpyDeviceToHost,
                           stream));
        CK(cudaStreamSynchronize(stream));
        o.tok.assign(rec_host, rec_host + B);
        o.acc.assign(rec_host + Bm, rec_host + Bm + B);
        o.out_layer = rec_host[2 * Bm];
        const float* cf = reinterpret_cast<const float*>(rec_host + 2 * Bm + 4);
        o.conf.resize((size_t)L * B);
        for (int l = 0; l < L; ++l)
            for (int b = 0; b < B; ++b) o.conf[(size_t)l * B + b] = cf[(size_t)l * Bm + b];
        return o;
    }
    int device_iter_counter() {
        int c = 0;
        CK(cudaMemcpy(&c, iter_counter.p, sizeof(int), cudaMemcpyDeviceToHost));
        return c;
    }

    std::vector<float> read_kv(int slot, int layer_, int pos, int which) {
        const int dp = dm.dp;
        int blk = 0;
        CK(cudaMemcpy(&blk, tables.p + ((size_t)slot * dm.L + (layer_ - 1)) * dm.bpl_max + pos / dm.bc, sizeof(int),
                      cudaMemcpyDeviceToHost));
        std::vector<uint16_t> raw((size_t)dp);
        const uint16_t* src = (which == 0 ? kpool.p : vpool.p) + ((size_t)blk * dm.bc + pos % dm.bc) * dp;
        CK(cudaMemcpy(raw.data(), src, sizeof(uint16_t) * dp, cudaMemcpyDeviceToHost));
        std::vector<float> out((size_t)dm.d);
        for (int i = 0; i < dm.d; ++i) {
            uint32_t f = (uint32_t)raw[(size_t)i] << 16;
            std::memcpy(&out[(size_t)i], &f, 4);
        }
        return out;
    }

    // ------------------------------------------------------------------
    // Engine::run (engine.cpp:110-330)
    // ------------------------------------------------------------------
    struct Live {
        int id, slot, max_new, next_input, committed;
        bool finished = false;
        double arrival, first_token = -1.0, finish = -1.0;
        std::vector<int> prompt, tokens, exit_layers, iter_out;
    };

    el_transcript* run(int n, const double* arrival, const int32_t* off, const int32_t* prompt, const int32_t* max_new) {
        if (in_session) fail(EL_LOGIC_ERROR, "run: a decode session is active");
        const int L = dm.L, d = dm.d;
        // Workload::validate_and_sort (workload.cpp:15-38)
        std::vector<int> order((size_t)n);
        for (int i = 0; i < n; ++i) order[(size_t)i] = i;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return arrival[a] < arrival[b]; });
        int max_cap = 1;
        for (int i = 0; i < n; ++i) {
            const int r = order[(size_t)i];
            const int plen = off[r + 1] - off[r];
            if (arrival[r] < 0.0) fail(EL_INVALID_ARGUMENT, "workload: negative arrival_time at request %d", i);
            if (plen < 1) fail(EL_INVALID_ARGUMENT, "workload: empty prompt at request %d", i);
            if (max_new[r] < 1) fail(EL_INVALID_ARGUMENT, "workload: max_new_tokens must be >= 1 at request %d", i);
            for (int j = off[r]; j < off[r + 1]; ++j)
                if (prompt[j] < 0 || prompt[j] >= cfg.vocab_size)
                    fail(EL_INVALID_ARGUMENT, "workload: token id %d outside vocab at request %d", prompt[j], i);
            max_cap = std::max(max_cap, plen + max_new[r]);
            if (cfg.encoder_len > 0 && plen > 1 && cfg.synthetic_kv_seed < 0)
                fail(EL_INVALID_ARGUMENT, "T5 mode: a decoder prompt is the single start token (the input goes to "
                                          "the encoder); request %d has %d tokens", i, plen);
        }
        reset_allocator();
        ensure_bpl(std::min(bpl_for(max_cap), std::max(1, cfg.pool_blocks / L)));
        CK(cudaMemsetAsync(iter_counter.p, 0, sizeof(int), stream));

        auto t = std::make_unique<el_transcript>();
        t->d = d;
        t->L = L;
        t->it_batch_off.push_back(0);
        t->sq_prompt_off.push_back(0);
        t->sq_tok_off.push_back(0);
        double clock = 0.0, total_idle = 0.0;
        int next_pending = 0, iteration_no = 0;
        std::vector<Live> running;
        std::vector<int> hs, hp, ht;

        for (;;) {
            // evict_finished (engine.cpp:130-164)
            for (auto it = running.begin(); it != running.end();) {
                if (!it->finished) { ++it; continue; }
                if (cfg.capture_kv) {
                    Capture& c = t->caps[it->id];
                    c.committed = it->committed;
                    c.k.assign((size_t)L * it->committed * d, 0.0);
                    c.v.assign((size_t)L * it->committed * d, 0.0);
                    for (int l = 1; l <= L; ++l)
                        for (int p = 0; p < it->committed; ++p) {
                            const auto kk = read_kv(it->slot, l, p, 0), vv = read_kv(it->slot, l, p, 1);
                            for (int i = 0; i < d; ++i) {
                                c.k[((size_t)(l - 1) * it->committed + p) * d + i] = kk[(size_t)i];
                                c.v[((size_t)(l - 1) * it->committed + p) * d + i] = vv[(size_t)i];
                            }
                        }
                    c.have_kv = true;
                    c.bpl = slot_bpl[(size_t)it->slot];
                    c.table.resize((size_t)L * c.bpl);
                    for (int l = 0; l < L; ++l)
                        CK(cudaMemcpy(c.table.data() + (size_t)l * c.bpl,
                                      tables.p + ((size_t)it->slot * L + l) * dm.bpl_max, sizeof(int) * c.bpl,
                                      cudaMemcpyDeviceToHost));
                }
                release(it->slot);
                t->sq_id.push_back(it->id);
                t->sq_arrival.push_back(it->arrival);
                t->sq_first.push_back(it->first_token);
                t->sq_finish.push_back(it->finish);
                t->sq_max_new.push_back(it->max_new);
                for (int x : it->prompt) t->sq_prompt.push_back(x);
                t->sq_prompt_off.push_back((int32_t)t->sq_prompt.size());
                for (size_t i = 0; i < it->tokens.size(); ++i) {
                    t->sq_tokens.push_back(it->tokens[i]);
                    t->sq_exit_layers.push_back(it->exit_layers[i]);
                    t->sq_iter_out.push_back(it->iter_out[i]);
                }
                t->sq_tok_off.push_back((int32_t)t->sq_tokens.size());
                it = running.erase(it);
            }
            // admit (engine.cpp:183-206) -- prefill charges advance the clock in
            // admission order; the prefill math itself is batched afterwards
            std::vector<PfSeq> pf;
            size_t admitted_now = 0;
            while (next_pending < n) {
                const int r = order[(size_t)next_pending];
                if (arrival[r] > clock) break;
                if ((int)running.size() >= cfg.max_batch) break;
                const int plen = off[r + 1] - off[r];
                const int need = plen + max_new[r];
                if (!can_allocate(need)) break;  // strict FIFO: a deferred head blocks later arrivals
                Live q;
                q.id = next_pending;
                q.slot = allocate(need);
                q.arrival = arrival[r];
                q.max_new = max_new[r];
                q.prompt.assign(prompt + off[r], prompt + off[r + 1]);
                q.next_input = q.prompt.back();
                const int positions = plen - 1;
                q.committed = positions;
                PfSeq ps;
                ps.slot = q.slot;
                ps.toks.assign(q.prompt.begin(), q.prompt.end() - 1);
                if (positions > 0) pf.push_back(std::move(ps));
                const double charge = (double)positions * L * (cfg.c_layer_fixed + cfg.c_layer_per_seq);
                clock += charge;
                t->pf_clock.push_back(clock);
                t->pf_charge.push_back(charge);
                t->pf_seq.push_back(q.id);
                t->pf_positions.push_back(positions);
                running.push_back(std::move(q));
                ++admitted_now;
                ++next_pending;
            }
            if (cfg.encoder_len > 0 && admitted_now > 0) {  // T5 mode: static cross K/V of the new sequences
                std::vector<int> ids, slots;
                for (size_t i = running.size() - admitted_now; i < running.size(); ++i) {
                    ids.push_back(running[i].id);
                    slots.push_back(running[i].slot);
                }
                cross_prefill(slots, ids);
            }
            if (!pf.empty()) {
                if (cfg.synthetic_kv_seed >= 0) {
                    std::vector<int> ids, slots;
                    int P = 0;
                    for (size_t i = running.size() - pf.size(); i < running.size(); ++i) {
                        ids.push_back(running[i].id);
                        slots.push_back(running[i].slot);
                        P = std::max(P, running[i].committed);
                    }
                    // seeded prefix for sequences admitted together must share the prefix length
                    for (size_t i = running.size() - pf.size(); i < running.size(); ++i)
                        if (running[i].committed != P)
                            fail(EL_INVALID_ARGUMENT, "synthetic KV prefix needs equal prompt lengths per admission");
                    seed_prefix(slots, ids, P, (uint64_t)cfg.synthetic_kv_seed);
                } else {
                    prefill(pf);
                }
            }
            if (running.empty()) {
                if (next_pending >= n) break;
                {
                    const int r = order[(size_t)next_pending];
                    if (arrival[r] <= clock && !can_allocate(off[r + 1] - off[r] + max_new[r]))
                        fail(EL_KV_OUT_OF_MEMORY, "allocate: request %d can never fit the pool", next_pending);
                }
                const double na = arrival[order[(size_t)next_pending]];
                if (na > clock) {
                    total_idle += na - clock;
                    clock = na;
                }
                continue;
            }

            // decode_iteration (engine.cpp:208-310).  Between scheduling events the batch is fixed,
            // so up to k iterations (k = the fewest tokens any running sequence may still emit) are
            // queued back to back on the device; after each, run_step_kernel charges the simulated
            // clock and stops the rest once a sequence finishes (max_new / EOS) or the pending head
            // becomes admissible -- one host synchronisation per event instead of per iteration.
            const int B = (int)running.size();
            hs.assign((size_t)B, 0); hp.assign((size_t)B, 0); ht.assign((size_t)B, 0);
            std::vector<int> rem((size_t)B, 0);
            int k = rec_cap;
            for (int b = 0; b < B; ++b) {
                hs[(size_t)b] = running[(size_t)b].slot;
                hp[(size_t)b] = running[(size_t)b].committed;
                ht[(size_t)b] = running[(size_t)b].next_input;
                rem[(size_t)b] = running[(size_t)b].max_new - (int)running[(size_t)b].tokens.size();
                k = std::min(k, rem[(size_t)b]);
            }
            const bool chunked = !cfg.capture_kv && (mega_for(B) || use_graph);
            if (!chunked) k = 1;
            double next_arrival = INFINITY;
            if (next_pending < n && (int)running.size() < cfg.max_batch) {
                const int r = order[(size_t)next_pending];
                if (can_allocate(off[r + 1] - off[r] + max_new[r])) next_arrival = arrival[r];
            }
            CK(cudaMemcpyAsync(row_slot.p, hs.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(row_pos.p, hp.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(row_tok.p, ht.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(run_rem.p, rem.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(run_clock.p, &clock, sizeof(double), cudaMemcpyHostToDevice, stream));
            const int ctl1[2] = {1, 0};
            CK(cudaMemcpyAsync(run_ctl.p, ctl1, sizeof ctl1, cudaMemcpyHostToDevice, stream));
            el::RunCtl rc{run_clock.p, run_log.p, run_rem.p, run_ctl.p, run_ctl.p + 1, cfg.eos_token, L, next_arrival,
                          cfg.c_layer_fixed, cfg.c_layer_per_seq, check_cost(), cfg.c_fill_per_seq_layer};
            const el::DevState sd = state(false, B);
            for (int i = 0; i < k; ++i) {
                iteration(B);
                el::launch_run_step(sd, rc, stream);
            }
            int ctl[2] = {0, 0};
            CK(cudaMemcpyAsync(ctl, run_ctl.p, sizeof ctl, cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            const int n_done = ctl[1];
            if (n_done < 1 || n_done > k) fail(EL_RUNTIME_ERROR, "run: %d of %d queued iterations ran", n_done, k);
            set_run_active(1);
            std::vector<double> dlog((size_t)2 * rec_cap);
            CK(cudaMemcpy(dlog.data(), run_log.p, sizeof(double) * dlog.size(), cudaMemcpyDeviceToHost));
            for (int it = 0; it < n_done; ++it) {
                const IterOut o = read_iteration(iteration_no, B);
                const int cur = iteration_no % rec_cap;
                ++iteration_no;
                const int e = o.out_layer;
                if (e < 1 || e > L) fail(EL_RUNTIME_ERROR, "decode_iteration: bad output layer %d", e);
                for (auto& q : running) q.committed += 1;  // commit (engine.cpp:262-264)

                const double charge = e * (cfg.c_layer_fixed + cfg.c_layer_per_seq * B) + e * B * check_cost() +
                                      (double)(L - e) * B * cfg.c_fill_per_seq_layer;
                clock += charge;
                if (chunked && (dlog[2 * (size_t)cur] != clock || dlog[2 * (size_t)cur + 1] != charge))
                    fail(EL_RUNTIME_ERROR, "run: device clock %.17g (charge %.17g) != host %.17g (%.17g)",
                         dlog[2 * (size_t)cur], dlog[2 * (size_t)cur + 1], clock, charge);
                t->it_clock.push_back(clock);
                t->it_charge.push_back(charge);
                t->it_output_layer.push_back(e);
                for (int l = 0; l < L; ++l)
                    for (int b = 0; b < B; ++b) t->it_conf.push_back((double)o.conf[(size_t)l * B + b]);
                std::vector<float> hexit;
                if (cfg.capture_kv) {
                    hexit.resize((size_t)B * dm.dp);
                    CK(cudaMemcpy(hexit.data(), h32.p + (size_t)(e & 1) * dm.Bmax * dm.dp, sizeof(float) * B * dm.dp,
                                  cudaMemcpyDeviceToHost));
                }
                int max_accept = 0;
                bool any_finished = false;
                for (int b = 0; b < B; ++b) {
                    Live& q = running[(size_t)b];
                    const int token = o.tok[(size_t)b];
                    const int acc = o.acc[(size_t)b];
                    max_accept = std::max(max_accept, acc);
                    t->ps_seq.push_back(q.id);
                    t->ps_accept.push_back(acc);
                    t->ps_token.push_back(token);
                    q.tokens.push_back(token);
                    q.exit_layers.push_back(acc);
                    q.iter_out.push_back(e);
                    if (cfg.capture_kv)
                        for (int i = 0; i < d; ++i) t->caps[q.id].exit_states.push_back(hexit[(size_t)b * dm.dp + i]);
                    if (q.tokens.size() == 1) q.first_token = clock;
                    const bool hit_eos = cfg.eos_token >= 0 && token == cfg.eos_token;
                    if (hit_eos || (int)q.tokens.size() >= q.max_new) {
                        q.finished = true;
                        q.finish = clock;
                        any_finished = true;
                    } else {
                        q.next_input = token;
                    }
                }
                if (max_accept != e) fail(EL_RUNTIME_ERROR, "decode_iteration: output_layer %d != max accept %d", e, max_accept);
                t->it_batch_off.push_back((int32_t)t->ps_seq.size());
                if (any_finished && it + 1 < n_done)
                    fail(EL_RUNTIME_ERROR, "run: the device ran past a finished sequence (iteration %d of %d)", it, n_done);
            }
        }
        t->meta = {clock, total_idle, (double)cfg.pool_blocks, (double)top, (double)peak};
        return t.release();
    }

    // T5 mode: the static cross K/V of newly admitted sequences -- encoder states generated
    // on the device, then K_c | V_c = W_kvc^(l) E^T for every layer as a tensor-core GEMM
    // (N = sequences x encoder_len) written straight into the sequences' cross blocks
    void cross_prefill(const std::vector<int>& slots, const std::vector<int>& ids) {
        if (cfg.encoder_len <= 0 || slots.empty()) return;
        const int n = (int)slots.size(), T = cfg.encoder_len, dp = dm.dp;
        CK(cudaMemcpyAsync(xslot.p, slots.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(xid.p, ids.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        const int N = n * T, NRe = round_up(N, 256);
        if (cfg.encoder_layers > 0) encoder_run(ids, NRe);
        else el::launch_encoder_states(enc_act.p, NRe, xid.p, n, T, cfg.d_model, dp, enc_seed, stream);
        el::GemmPlan P = make_plan(wkvc.p, enc_act.p, 0, 2 * dp / 128, dp, 256, false, 1);
        el::DevState s = state(true, N);
        s.rows.slot = xslot.p;
        s.rows.B = N;
        s.NR = NRe;
        for (int l = 1; l <= dm.L; ++l) {
            CK(cudaMemcpyAsync(layer.p, &l, sizeof(int), cudaMemcpyHostToDevice, stream));
            el::launch_gemm(el::kGemmCross, P, s, stream, false);
        }
        CK(cudaStreamSynchronize(stream));  // l is a host stack variable
    }

    // T5 encoder stack over the seeded encoder ids of sequences `ids` -> enc_act rows [j T, (j+1) T)
    // (bf16, act layout with NRe rows).  One persistent-kernel launch per kPfRows / T sequences:
    // rows = (local sequence, position), each layer's K/V into the scratch pool, attention over all
    // T positions of the row's sequence (enc_bidir), no exit / LM head / fill (prefill mode).
    void encoder_run(const std::vector<int>& ids, int NRe) {
        const int T = cfg.encoder_len, LE = cfg.encoder_layers, q = kPfRows / T, dp = dm.dp;
        plan_encoder = true;
        el::IterPlan& P = mplan_for(q * T, kPfRows);
        plan_encoder = false;
        for (size_t j0 = 0; j0 < ids.size(); j0 += (size_t)q) {
            const int nq = (int)std::min<size_t>((size_t)q, ids.size() - j0), B = nq * T;
            std::vector<int> hs((size_t)B), hp((size_t)B), ht((size_t)B);
            for (int j = 0; j < nq; ++j)
                for (int t = 0; t < T; ++t) {
                    const size_t r = (size_t)j * T + t;
                    hs[r] = j;
                    hp[r] = t;
                    ht[r] = encoder_token(ids[j0 + j], t);
                }
            CK(cudaMemcpyAsync(pf_slot.p, hs.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(pf_pos.p, hp.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(pf_tok.p, ht.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
            el::DevState s = state(true, B);
            s.cont_host = nullptr;
            s.prefill = 1;
            s.enc_bidir = T;
            s.enc_len = 0;  // (no cross-attention inside the encoder)
            s.dm.L = LE;
            s.dm.bpl_max = e_bpl;
            s.dm.slots = q;
            s.wqkv = e_wqkv.p; s.wo = e_wo.p; s.wup = e_wup.p; s.wdown = e_wdown.p;
            s.kpool = e_kpool.p; s.vpool = e_vpool.p; s.tables = e_tables.p;
            s.NR = kPfRows;
            s.h32 = pf_h32.p; s.hb = pf_hb.p; s.q32 = pf_q32.p; s.att_b = pf_att_b.p;
            s.mid32 = pf_mid32.p; s.mid_b = pf_mid_b.p; s.up_b = pf_up_b.p;
            s.attn_stages = mega_att_stages;
            el::launch_iter(s, P, mmaps[P.map_key], mega_grid, stream);
            // the last layer's bf16 output rows -> enc_act rows of these sequences
            el::launch_act_rows_copy(enc_act.p, NRe, (int)j0 * T, pf_hb.p + (size_t)(LE & 1) * kPfRows * dp, kPfRows,
                                     B, dp, stream);
            CK(cudaStreamSynchronize(stream));  // host vectors are reused
        }
    }
    int encoder_token(int seq_id, int t) const {  // oracle: eo_encoder_token
        return 1 + (int)(el::splitmix64_at(enc_seed ^ 0x544F4Bu, ((uint64_t)seq_id << 20) | (uint64_t)t) %
                         (uint64_t)(cfg.vocab_size - 1));
    }

    // seeded KV prefix for the sequences in `slots` (rows of the prefill row set)
    void seed_prefix(const std::vector<int>& slots, const std::vector<int>& ids, int P, uint64_t kv_seed) {
        const int B = (int)slots.size();
        CK(cudaMemcpyAsync(pf_slot.p, slots.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(seq_ids_dev.p, ids.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
        el::DevState s = state(true, B);
        el::launch_kv_prefix(s, seq_ids_dev.p, P, kv_seed, 1, stream);
        CK(cudaStreamSynchronize(stream));
    }


    // ------------------------------------------------------------------
    // Sub-engine API on the device pool (outside a session / run): KvStore
    // (kv_cache.hpp:45-115), layer_forward / compute_kv_pair + fill_skipped
    // (model.hpp:64-76, kv_cache.hpp:107-115), the exit confidences + decide
    // (exit_policy.hpp:46-70) and lm_head_logits + greedy_token (model.hpp:71-76).
    // Sequences live in device slots (at most max_batch at a time); the host
    // keeps the reference's invariant counters (written per layer, committed).
    // ------------------------------------------------------------------
    struct StoreSeq {
        int slot = 0, capacity = 0, committed = 0, bpl = 0;
        std::vector<int> written;  // per layer
        std::vector<int> table;    // [L][bpl] block ids (device table mirror)
    };
    std::map<int, StoreSeq> store;
    bool store_ready = false;
    void store_begin() {
        if (in_session) fail(EL_LOGIC_ERROR, "KvStore API: a decode session is active");
        if (!store_ready) {
            reset_allocator();
            ensure_bpl(std::min(128, std::max(1, cfg.pool_blocks / dm.L)));
            store_ready = true;
        }
    }
    StoreSeq& store_entry(int id, const char* op) {
        auto it = store.find(id);
        if (it == store.end()) fail(EL_INVALID_ARGUMENT, "%s: unknown seq_id %d", op, id);
        return it->second;
    }
    void store_allocate(int id, int capacity_tokens) {  // kv_cache.cpp:78-106
        store_begin();
        if (store.count(id)) fail(EL_INVALID_ARGUMENT, "allocate: seq_id %d already allocated", id);
        if (capacity_tokens < 0) fail(EL_INVALID_ARGUMENT, "allocate: negative capacity");
        const int bpl = bpl_for(capacity_tokens);
        if ((long)bpl * dm.L > top) fail(EL_KV_OUT_OF_MEMORY, "allocate: need %ld blocks, %d free", (long)bpl * dm.L, top);
        StoreSeq q;
        q.slot = allocate(capacity_tokens);
        q.capacity = bpl * dm.bc;
        q.bpl = bpl;
        q.written.assign((size_t)dm.L, 0);
        q.table.assign((size_t)dm.L * bpl, 0);
        for (int l = 0; l < dm.L && bpl > 0; ++l)
            CK(cudaMemcpyAsync(q.table.data() + (size_t)l * bpl, tables.p + ((size_t)q.slot * dm.L + l) * dm.bpl_max,
                               sizeof(int) * bpl, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        store.emplace(id, std::move(q));
    }
    void store_release(int id) {  // kv_cache.cpp:182-194
        auto it = store.find(id);
        if (it == store.end()) fail(EL_INVALID_ARGUMENT, "release: unknown or already released seq_id %d", id);
        release(it->second.slot);
        store.erase(it);
    }
    // append-position checks of KvStore::append (kv_cache.cpp:108-145) for position `pos` at `layer`
    void store_check_append(int id, const StoreSeq& q, int layer, int pos) const {
        if (layer < 1 || layer > dm.L) fail(EL_INVALID_ARGUMENT, "append: layer %d outside [1, %d]", layer, dm.L);
        const int w = q.written[(size_t)layer - 1];
        if (pos < w) fail(EL_RUNTIME_ERROR, "append: slot already written at (seq %d, layer %d, position %d)", id, layer, pos);
        if (pos > w)
            fail(EL_RUNTIME_ERROR, "append: position gap at (seq %d, layer %d, position %d), next unwritten is %d", id,
                 layer, pos, w);
        if (pos >= q.capacity)
            fail(EL_KV_OUT_OF_MEMORY, "append: position %d exceeds reserved capacity %d for seq %d", pos, q.capacity, id);
    }
    size_t store_row(const StoreSeq& q, int layer, int pos) const {
        const int blk = q.table[(size_t)(layer - 1) * q.bpl + pos / dm.bc];
        return ((size_t)blk * dm.bc + pos % dm.bc) * dm.dp;
    }
    void store_append(int id, int layer, int pos, const float* k, const float* v) {
        StoreSeq& q = store_entry(id, "append");
        store_check_append(id, q, layer, pos);
        std::vector<uint16_t> kb((size_t)dm.dp, 0), vb((size_t)dm.dp, 0);
        for (int i = 0; i < dm.d; ++i) {
            kb[(size_t)i] = el::bf16_bits_rne((double)k[i]);
            vb[(size_t)i] = el::bf16_bits_rne((double)v[i]);
        }
        const size_t r = store_row(q, layer, pos);
        CK(cudaMemcpy(kpool.p + r, kb.data(), sizeof(uint16_t) * dm.dp, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(vpool.p + r, vb.data(), sizeof(uint16_t) * dm.dp, cudaMemcpyHostToDevice));
        ++q.written[(size_t)layer - 1];
    }
    void store_view(int id, int layer, int upto, float* k, float* v) {  // kv_cache.cpp:147-163
        StoreSeq& q = store_entry(id, "view");
        if (layer < 1 || layer > dm.L) fail(EL_INVALID_ARGUMENT, "view: layer %d outside [1, %d]", layer, dm.L);
        if (upto < 0) fail(EL_INVALID_ARGUMENT, "view: negative upto_position");
        if (upto > q.written[(size_t)layer - 1])
            fail(EL_RUNTIME_ERROR, "view: entries missing at (seq %d, layer %d): requested %d, written %d", id, layer,
                 upto, q.written[(size_t)layer - 1]);
        CK(cudaStreamSynchronize(stream));
        std::vector<uint16_t> raw((size_t)dm.dp);
        for (int p = 0; p < upto; ++p)
            for (int which = 0; which < 2; ++which) {
                CK(cudaMemcpy(raw.data(), (which ? vpool.p : kpool.p) + store_row(q, layer, p), sizeof(uint16_t) * dm.dp,
                              cudaMemcpyDeviceToHost));
                float* out = (which ? v : k) + (size_t)p * dm.d;
                for (int i = 0; i < dm.d; ++i) {
                    const uint32_t f = (uint32_t)raw[(size_t)i] << 16;
                    std::memcpy(&out[i], &f, 4);
                }
            }
    }
    void store_commit(int id) {  // kv_cache.cpp:165-180
        StoreSeq& q = store_entry(id, "commit");
        for (int l = 1; l <= dm.L; ++l)
            if (q.written[(size_t)l - 1] != q.committed + 1)
                fail(EL_RUNTIME_ERROR, "commit: layer %d of seq %d has %d entries, expected %d", l, id,
                     q.written[(size_t)l - 1], q.committed + 1);
        ++q.committed;
    }
    // rows of a batch of store sequences: slot, position = committed length
    void store_rows(int n, const int32_t* ids, std::vector<StoreSeq*>& qs) {
        if (n < 1) fail(EL_LOGIC_ERROR, "decode_iteration: empty batch");
        if (n > dm.Bmax) fail(EL_INVALID_ARGUMENT, "batch %d > max_batch %d", n, dm.Bmax);
        std::vector<int> hs((size_t)n), hp((size_t)n);
        qs.assign((size_t)n, nullptr);
        for (int b = 0; b < n; ++b) {
            for (int c = 0; c < b; ++c)
                if (ids[c] == ids[b]) fail(EL_INVALID_ARGUMENT, "batch: seq_id %d appears twice", ids[b]);
            qs[(size_t)b] = &store_entry(ids[b], "layer_forward");
            hs[(size_t)b] = qs[(size_t)b]->slot;
            hp[(size_t)b] = qs[(size_t)b]->committed;
        }
        CK(cudaMemcpyAsync(row_slot.p, hs.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_pos.p, hp.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
    }
    // host states [n][d] -> residual stream parity `par` (fp32) and its bf16 GEMM operand copy
    void put_states(int n, const float* h, int par, bool f32, bool b16) {
        const int dp = dm.dp, d = dm.d;
        if (f32) {
            std::vector<float> buf((size_t)n * dp, 0.f);
            for (int b = 0; b < n; ++b) std::memcpy(buf.data() + (size_t)b * dp, h + (size_t)b * d, sizeof(float) * d);
            CK(cudaMemcpy(h32.p + (size_t)par * dm.Bmax * dp, buf.data(), sizeof(float) * buf.size(),
                          cudaMemcpyHostToDevice));
        }
        if (b16) {
            std::vector<uint16_t> buf((size_t)NR * dp, 0);
            for (int b = 0; b < n; ++b)
                for (int i = 0; i < d; ++i) buf[el::act_offset(b, i, NR)] = el::bf16_bits_rne((double)h[(size_t)b * d + i]);
            CK(cudaMemcpy(hb.p + (size_t)par * NR * dp, buf.data(), sizeof(uint16_t) * buf.size(),
                          cudaMemcpyHostToDevice));
        }
    }
    void set_dev_int(int* dst, int v) {
        CK(cudaMemcpy(dst, &v, sizeof(int), cudaMemcpyHostToDevice));
    }
    el::DevState store_state(int n) {
        el::DevState s = state(false, n);
        s.cont_host = nullptr;
        s.fuse_exit = 0;
        s.use_cond = 0;
        return s;
    }
    // layer_forward (model.cpp:197-272) for n store sequences at their committed positions
    void layer_forward(int layer, int n, const int32_t* ids, const float* h_in, float* h_out) {
        if (in_session) fail(EL_LOGIC_ERROR, "layer_forward: a decode session is active");
        if (layer < 1 || layer > dm.L) fail(EL_INVALID_ARGUMENT, "layer_forward: layer %d outside [1, %d]", layer, dm.L);
        std::vector<StoreSeq*> qs;
        store_rows(n, ids, qs);
        for (int b = 0; b < n; ++b) store_check_append(ids[b], *qs[(size_t)b], layer, qs[(size_t)b]->committed);
        put_states(n, h_in, (layer - 1) & 1, true, true);
        set_dev_int(layer_ptr(), layer);
        Plans& P = plans_for(n);
        el::DevState s = store_state(n);
        s.technique = el::kNever;
        el::launch_gemm(el::kGemmQkv, P.qkv, s, stream, false);
        el::launch_attention(s, stream, false);
        el::launch_gemm(el::kGemmWo, P.wo, s, stream, false);
        el::launch_gemm(el::kGemmUp, P.up, s, stream, false);
        el::launch_gemm(el::kGemmDown, P.down, s, stream, false);
        CK(cudaStreamSynchronize(stream));
        get_states(n, layer & 1, h_out);
        for (int b = 0; b < n; ++b) ++qs[(size_t)b]->written[(size_t)layer - 1];
    }
    int* layer_ptr() { return layer.p; }
    void get_states(int n, int par, float* out) {
        const int dp = dm.dp, d = dm.d;
        std::vector<float> buf((size_t)n * dp);
        CK(cudaMemcpy(buf.data(), h32.p + (size_t)par * dm.Bmax * dp, sizeof(float) * buf.size(), cudaMemcpyDeviceToHost));
        for (int b = 0; b < n; ++b) std::memcpy(out + (size_t)b * d, buf.data() + (size_t)b * dp, sizeof(float) * d);
    }
    // fill_skipped (kv_cache.cpp:222-234): K_j, V_j = W_k^(j) h_e, W_v^(j) h_e for j in (e, L]
    void kv_fill(int n, const int32_t* ids, const float* h_exit, int e_out) {
        if (in_session) fail(EL_LOGIC_ERROR, "fill_skipped: a decode session is active");
        if (e_out < 1 || e_out > dm.L) fail(EL_INVALID_ARGUMENT, "fill_skipped: output_layer out of range");
        std::vector<StoreSeq*> qs;
        store_rows(n, ids, qs);
        for (int b = 0; b < n; ++b)
            for (int j = e_out + 1; j <= dm.L; ++j) store_check_append(ids[b], *qs[(size_t)b], j, qs[(size_t)b]->committed);
        if (e_out == dm.L) return;  // no-op at the last layer (kv_cache.hpp:110-115)
        put_states(n, h_exit, e_out & 1, false, true);
        set_dev_int(out_layer.p, e_out);
        Plans& P = plans_for(n);
        el::DevState s = store_state(n);
        el::launch_gemm(el::kGemmFill, P.fill, s, stream, false);
        CK(cudaStreamSynchronize(stream));
        for (int b = 0; b < n; ++b)
            for (int j = e_out + 1; j <= dm.L; ++j) ++qs[(size_t)b]->written[(size_t)j - 1];
    }
    // the configured technique's confidence of n states at `layer` and decide's strict '>' against
    // threshold_at(layer) (exit_policy.cpp:57-115); h_prev only for state similarity
    void exit_confidence(int layer, int n, const float* h_prev, const float* h_cur, float* conf_out, int32_t* acc_out) {
        if (in_session) fail(EL_LOGIC_ERROR, "exit_confidence: a decode session is active");
        if (layer < 1 || layer > dm.L) fail(EL_INVALID_ARGUMENT, "exit_confidence: layer %d outside [1, %d]", layer, dm.L);
        if (n < 1 || n > dm.Bmax) fail(EL_INVALID_ARGUMENT, "exit_confidence: batch %d outside [1, %d]", n, dm.Bmax);
        if (cfg.technique == EL_TECH_STATE && !h_prev) fail(EL_INVALID_ARGUMENT, "state_similarity needs h_prev");
        if (cfg.technique == EL_TECH_FIXED) fail(EL_INVALID_ARGUMENT, "exit_confidence: technique fixed has no evidence");
        if (cfg.technique == EL_TECH_STATE) put_states(n, h_prev, (layer - 1) & 1, true, false);
        put_states(n, h_cur, layer & 1, true, cfg.technique == EL_TECH_SOFTMAX);
        set_dev_int(layer_ptr(), layer);
        set_dev_int(exit_cnt.p, 0);
        CK(cudaMemset(status.p, 0, sizeof(int) * dm.Bmax));
        el::DevState s = store_state(n);
        if (cfg.technique == EL_TECH_SOFTMAX) el::launch_gemm(el::kGemmLmCheck, plans_for(n).lm, s, stream, false);
        el::launch_exit(s, stream, false);
        CK(cudaStreamSynchronize(stream));
        std::vector<float> cf((size_t)n);
        std::vector<int> ac((size_t)n);
        CK(cudaMemcpy(cf.data(), conf.p + (size_t)(layer - 1) * dm.Bmax, sizeof(float) * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ac.data(), accept.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
        if (conf_out) std::memcpy(conf_out, cf.data(), sizeof(float) * n);
        if (acc_out) for (int b = 0; b < n; ++b) acc_out[b] = ac[(size_t)b];
    }
    // lm_head_logits + greedy_token (model.cpp:284-299): argmax over the vocabulary, lowest index on ties
    void greedy_tokens(int n, const float* h, int32_t* tokens) {
        if (in_session) fail(EL_LOGIC_ERROR, "greedy_token: a decode session is active");
        if (n < 1 || n > dm.Bmax) fail(EL_INVALID_ARGUMENT, "greedy_token: batch %d outside [1, %d]", n, dm.Bmax);
        const int par = dm.L & 1;
        put_states(n, h, par, false, true);
        set_dev_int(out_layer.p, dm.L);
        std::vector<int> zeros((size_t)n, 0);
        CK(cudaMemcpy(row_pos.p, zeros.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
        el::DevState s = store_state(n);
        el::launch_gemm(el::kGemmLmFinal, plans_for(n).lm, s, stream, false);
        el::launch_finish(s, stream, false);
        CK(cudaStreamSynchronize(stream));
        CK(cudaMemcpy(tokens, row_tok.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
    }


    // ------------------------------------------------------------------
    // Layer-level scheduling (the occupancy MDP of layer_sched.hpp:13-60
    // driving real batches -- f4).  Each sequence of the session has its own next layer; a
    // TURN runs one layer for every sequence whose next layer it is (one persistent-kernel
    // launch in turn mode), each of them exiting on its own accept (no batch-wide barrier):
    // an exiting sequence fills its skipped layers' K/V from its exit state, emits its token
    // and restarts at layer 1; the others carry their state to the next layer.  Per sequence
    // the arithmetic is exactly the reference's decode_iteration for a batch of one.  The
    // policy picks the turn's layer from the occupancy vector v (v[i] = sequences whose next
    // layer is i+1): greedy = argmax v, ties toward the lowest layer (greedy_action,
    // layer_sched.cpp:95-105), or linear = argmax_a M[a].v (LinearQ / TrainedPolicy::action,
    // layer_sched.cpp:189-199, 311-325), falling back to greedy when that layer is empty.
    // ------------------------------------------------------------------
    struct Sched {
        bool on = false;
        int policy = 0;
        std::vector<double> M;  // [L][L] (linear policy)
        bool defer = false;      // deferred tokens: next == 0 = the sequence waits for a token turn
        std::vector<int> next, pos, tok, exit_at;
        std::vector<std::vector<int>> toks, exits;
        std::vector<int> turn_layer, turn_n;  // turn_layer 0 = a token turn
    } sch;
    int opt_sched_defer = 1;
    DevBuf<float> hstore;
    DevBuf<int> row_seq, row_exit;
    void sched_begin(int policy, const double* M) {
        need_session();
        if (cfg.encoder_len > 0) fail(EL_INVALID_ARGUMENT, "layer-level scheduling: T5 mode not supported");
        if (policy < 0 || policy > 1) fail(EL_INVALID_ARGUMENT, "layer-level scheduling: policy 0 (greedy) or 1 (linear)");
        if (policy == 1 && !M) fail(EL_INVALID_ARGUMENT, "linear policy needs its L x L matrix");
        const int B = sess_B, L = dm.L;
        sch = Sched{};
        sch.on = true;
        sch.policy = policy;
        if (M) sch.M.assign(M, M + (size_t)L * L);
        sch.next.assign((size_t)B, 1);
        sch.pos.assign((size_t)B, sess_prefix + sess_iters);
        if (sess_iters != 0) fail(EL_LOGIC_ERROR, "layer-level scheduling must start on a fresh session");
        sch.tok = sess_first;
        sch.toks.assign((size_t)B, {});
        sch.exits.assign((size_t)B, {});
        sch.exit_at.assign((size_t)B, 0);
        // deferred tokens (default; not with softmax exit, whose check already holds the token's LM
        // head): a sequence that exits waits at the token stage, and a token turn decodes the LM
        // head and fills the skipped layers for every waiting sequence at once
        sch.defer = opt_sched_defer && cfg.technique != EL_TECH_SOFTMAX;
        if (hstore.n < (size_t)dm.Bmax * dm.dp) hstore.alloc((size_t)dm.Bmax * dm.dp);
        if (row_seq.n < (size_t)dm.Bmax) row_seq.alloc((size_t)dm.Bmax);
        if (row_exit.n < (size_t)dm.Bmax) row_exit.alloc((size_t)dm.Bmax);
    }
    int sched_pick(const std::vector<int>& v) const {
        const int L = dm.L;
        int best = 1;
        for (int a = 2; a <= L; ++a)
            if (v[(size_t)a - 1] > v[(size_t)best - 1]) best = a;
        if (sch.policy == 1) {
            auto pred = [&](int a) {
                double acc = 0.0;
                for (int i = 0; i < L; ++i) acc += sch.M[(size_t)(a - 1) * L + i] * v[(size_t)i];
                return acc;
            };
            int lb = 1;
            double bv = pred(1);
            for (int a = 2; a <= L; ++a) {
                const double x = pred(a);
                if (x > bv) { lb = a; bv = x; }
            }
            if (v[(size_t)lb - 1] > 0) best = lb;
        }
        return best;
    }
    // token turn: the LM head + greedy token + skipped-layer fill of every waiting sequence
    void sched_token_turn() {
        const int B = sess_B, Bm = dm.Bmax;
        std::vector<int> rs, rp, rt, rq, re;
        int amin = dm.L;
        for (int b = 0; b < B; ++b)
            if (sch.next[(size_t)b] == 0) {
                rs.push_back(sess_slots[(size_t)b]);
                rp.push_back(sch.pos[(size_t)b]);
                rt.push_back(sch.tok[(size_t)b]);
                rq.push_back(b);
                re.push_back(sch.exit_at[(size_t)b]);
                amin = std::min(amin, sch.exit_at[(size_t)b]);
            }
        const int n = (int)rs.size();
        CK(cudaMemcpyAsync(row_slot.p, rs.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_pos.p, rp.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_tok.p, rt.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_seq.p, rq.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_exit.p, re.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        el::IterPlan& P = mplan_for(n);
        el::DevState s = state(false, n);
        s.attn_stages = mega_att_stages;
        s.turn_layer = amin;
        s.turn_token = 1;
        el::launch_iter(s, P, mmaps[P.map_key], mega_grid, stream);
        const int cur = sess_iters % rec_cap;
        CK(cudaMemcpyAsync(rec_host, rec.p + (size_t)cur * rec_stride, sizeof(int) * rec_stride, cudaMemcpyDeviceToHost,
                           stream));
        CK(cudaStreamSynchronize(stream));
        ++sess_iters;
        for (int r = 0; r < n; ++r) {
            const int b = rq[(size_t)r];
            sch.toks[(size_t)b].push_back(rec_host[r]);
            sch.exits[(size_t)b].push_back(sch.exit_at[(size_t)b]);
            sch.tok[(size_t)b] = rec_host[r];
            ++sch.pos[(size_t)b];
            sch.next[(size_t)b] = 1;
        }
        sch.turn_layer.push_back(0);
        sch.turn_n.push_back(n);
    }
    void sched_turn() {
        const int B = sess_B, L = dm.L, Bm = dm.Bmax;
        std::vector<int> v((size_t)L, 0);
        int waiting = 0;
        for (int b = 0; b < B; ++b) {
            if (sch.next[(size_t)b] == 0) ++waiting;
            else ++v[(size_t)sch.next[(size_t)b] - 1];
        }
        // the token stage competes like a layer: a token turn when the waiting sequences are at
        // least as many as the policy's layer holds (or nothing else is runnable)
        const int a = sched_pick(v);
        if (waiting > 0 && waiting >= v[(size_t)a - 1]) {
            sched_token_turn();
            return;
        }
        std::vector<int> rs, rp, rt, rq;
        for (int b = 0; b < B; ++b)
            if (sch.next[(size_t)b] == a) {
                if (sch.pos[(size_t)b] >= sess_capacity)
                    fail(EL_KV_OUT_OF_MEMORY, "append: position %d exceeds reserved capacity %d", sch.pos[(size_t)b],
                         sess_capacity);
                rs.push_back(sess_slots[(size_t)b]);
                rp.push_back(sch.pos[(size_t)b]);
                rt.push_back(sch.tok[(size_t)b]);
                rq.push_back(b);
            }
        const int n = (int)rs.size();
        CK(cudaMemcpyAsync(row_slot.p, rs.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_pos.p, rp.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_tok.p, rt.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_seq.p, rq.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
        el::IterPlan& P = mplan_for(n);
        el::DevState s = state(false, n);
        s.attn_stages = mega_att_stages;
        s.attn_seg_cost = opt_attn_seg_cost >= 0 ? opt_attn_seg_cost : (n <= 64 ? 2 : 0);
        s.turn_layer = a;
        s.turn_defer = sch.defer ? 1 : 0;
        el::launch_iter(s, P, mmaps[P.map_key], mega_grid, stream);
        const int cur = sess_iters % rec_cap;
        CK(cudaMemcpyAsync(rec_host, rec.p + (size_t)cur * rec_stride, sizeof(int) * rec_stride, cudaMemcpyDeviceToHost,
                           stream));
        CK(cudaStreamSynchronize(stream));
        ++sess_iters;
        for (int r = 0; r < n; ++r) {
            const int b = rq[(size_t)r];
            const int ex = rec_host[Bm + r];
            if (ex && sch.defer) {  // waits for a token turn
                sch.exit_at[(size_t)b] = ex;
                sch.next[(size_t)b] = 0;
            } else if (ex) {
                sch.toks[(size_t)b].push_back(rec_host[r]);
                sch.exits[(size_t)b].push_back(ex);
                sch.tok[(size_t)b] = rec_host[r];
                ++sch.pos[(size_t)b];
                sch.next[(size_t)b] = 1;
            } else {
                ++sch.next[(size_t)b];
            }
        }
        sch.turn_layer.push_back(a);
        sch.turn_n.push_back(n);
    }

    // ------------------------------------------------------------------
    // decode session: fixed batch over a seeded KV prefix (bench workload)
    // ------------------------------------------------------------------
    void session_begin(int B, const int32_t* first, int prefix_len, int capacity, uint64_t kv_seed, const int32_t* ids) {
        if (in_session) session_end();
        if (B < 1) fail(EL_LOGIC_ERROR, "decode_iteration: empty batch");
        if (B > dm.Bmax) fail(EL_INVALID_ARGUMENT, "session: batch %d > max_batch %d", B, dm.Bmax);
        if (prefix_len < 0 || capacity < prefix_len + 1) fail(EL_INVALID_ARGUMENT, "session: capacity must exceed prefix");
        for (int b = 0; b < B; ++b)
            if (first[b] < 0 || first[b] >= cfg.vocab_size) fail(EL_INVALID_ARGUMENT, "session: token outside vocab");
        reset_allocator();
        ensure_bpl(bpl_for(capacity));
        std::vector<int> slots, idv, pos((size_t)B, prefix_len), tok(first, first + B);
        for (int b = 0; b < B; ++b) {
            slots.push_back(allocate(capacity));
            idv.push_back(ids ? ids[b] : b);
        }
        seed_prefix(slots, idv, prefix_len, kv_seed);
        cross_prefill(slots, idv);
        CK(cudaMemcpyAsync(row_slot.p, slots.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_pos.p, pos.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(row_tok.p, tok.data(), sizeof(int) * B, cudaMemcpyHostToDevice, stream));
        CK(cudaMemsetAsync(iter_counter.p, 0, sizeof(int), stream));
        CK(cudaStreamSynchronize(stream));
        in_session = true;
        sess_B = B;
        sess_iters = 0;
        sess_ids = idv;
        sess_capacity = capacity;
        sess_prefix = prefix_len;
        sess_slots = slots;
        sess_first.assign(first, first + B);
        sch = Sched{};
    }
    int sess_capacity = 0, sess_prefix = 0;
    std::vector<int> sess_slots, sess_first;
    void session_end() {
        in_session = false;
        sch = Sched{};
        reset_allocator();
    }
    void need_session() const {
        if (!in_session) fail(EL_LOGIC_ERROR, "no active decode session");
    }
    void check_capacity(int n_more) const {
        if (sess_prefix + sess_iters + n_more > sess_capacity)
            fail(EL_KV_OUT_OF_MEMORY, "append: position exceeds reserved capacity %d", sess_capacity);
    }
};

// ============================================================================
// C ABI
// ============================================================================
#define API_BEGIN try {
#define API_END                                   \
    }                                             \
    catch (const ElError& e) {                    \
        g_err = e.msg;                            \
        return e.code;                            \
    }                                             \
    catch (const std::exception& e) {             \
        g_err = e.what();                         \
        return EL_RUNTIME_ERROR;                  \
    }                                             \
    return EL_OK;

extern "C" {

const char* el_last_error(void) { return g_err.c_str(); }
int el_version(void) { return 1; }

int el_set_device(int device) {
    API_BEGIN
    CK(cudaSetDevice(device));
    API_END
}

int el_device_count(int* n) {
    API_BEGIN
    CK(cudaGetDeviceCount(n));
    API_END
}

int el_engine_create(const el_engine_config* cfg, el_engine** out) {
    API_BEGIN
    if (!cfg || !out) fail(EL_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    auto e = std::make_unique<el_engine>();
    e->cfg = *cfg;
    e->create();
    *out = e.release();
    API_END
}

int el_engine_create_sized(const el_engine_config* cfg, size_t config_size, el_engine** out) {
    API_BEGIN
    if (!cfg || !out) fail(EL_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    el_engine_config c{};
    const size_t n = std::min(config_size, sizeof(el_engine_config));
    std::memcpy(&c, cfg, n);
    const unsigned char* extra = reinterpret_cast<const unsigned char*>(cfg) + n;
    for (size_t i = n; i < config_size; ++i)
        if (extra[i - n]) fail(EL_INVALID_ARGUMENT, "el_engine_config: unknown non-zero field at byte %zu", i);
    auto e = std::make_unique<el_engine>();
    e->cfg = c;
    e->create();
    *out = e.release();
    API_END
}

int el_engine_destroy(el_engine* e) {
    API_BEGIN
    if (e) {
        cudaStreamSynchronize(e->stream);
        delete e;
    }
    API_END
}

int el_engine_set_option(el_engine* e, const char* key, int64_t v) {
    API_BEGIN
    if (!std::strcmp(key, "graph")) e->use_graph = v != 0;
    else if (!std::strcmp(key, "pipe")) {
        if (v < 0 || v > 2) fail(EL_INVALID_ARGUMENT, "pipe must be 0 (off), 1 (on) or 2 (auto)");
        e->use_pipe = (int)v;
    } else if (!std::strcmp(key, "pipe_softmax")) {  // softmax exit on the pipelined kernel (batch 65..128)
        e->pipe_softmax = v != 0;
        e->mplans.clear();
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "pipe64")) {  // batch 33..64 on the pipelined kernel (halves of 32 rows)
        e->pipe64 = v != 0;
        e->mplans.clear();
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "pipe_att_ctas64_softmax")) {
        if (v < 16 || v > 132) fail(EL_INVALID_ARGUMENT, "%s must be in [16, 132]", key);
        e->pipe_att64_sm = (int)v;
    } else if (!std::strcmp(key, "pipe_att_ctas32")) {
        if (v < 16 || v > 132) fail(EL_INVALID_ARGUMENT, "%s must be in [16, 132]", key);
        e->pipe_att32 = (int)v;
    } else if (!std::strcmp(key, "pipe128")) {  // batch 65..128 on the pipelined kernel (halves of 64 rows)
        e->pipe128 = v != 0;
        e->mplans.clear();
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "pipe_att_ctas") || !std::strcmp(key, "pipe_att_ctas64")) {
        if (v < 16 || v > 132) fail(EL_INVALID_ARGUMENT, "%s must be in [16, 132]", key);
        (key[13] == '6' ? e->pipe_att64 : e->pipe_att) = (int)v;
    }
    else if (!std::strcmp(key, "mega")) {
        if (v < 0 || v > 2) fail(EL_INVALID_ARGUMENT, "mega must be 0 (off), 1 (on) or 2 (auto)");
        e->use_mega = (int)v;
    }
    else if (!std::strcmp(key, "attn_seg_cost")) {
        if (v < -1 || v > 64) fail(EL_INVALID_ARGUMENT, "attn_seg_cost must be in [-1 (auto), 64]");
        e->opt_attn_seg_cost = (int)v;
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "mega_bm_chunk_kb")) {
        if (v < 0 || v > 64) fail(EL_INVALID_ARGUMENT, "mega_bm_chunk_kb must be in [0 (auto), 64]");
        e->opt_mega_bm_chunk_kb = (int)v;
        e->mplans.clear();
    } else if (!std::strcmp(key, "lm_pair")) {  // softmax checks on LM pair units (0 off, 1 on)
        if (v < 0 || v > 2) fail(EL_INVALID_ARGUMENT, "lm_pair must be 0, 1 or 2 (transposed: batch rows on TMEM lanes)");
        e->opt_lm_pair = (int)v;
        e->mplans.clear();
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "lm_tail")) {  // decode tail LM head on transposed units (0 off, 1 on)
        e->opt_lm_tail = v != 0;
        e->mplans.clear();
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "lm_keep")) {  // LM-head tiles evict-last: 0 off, 1 softmax checks, 2 + final head
        if (v < 0 || v > 2) fail(EL_INVALID_ARGUMENT, "lm_keep must be 0, 1 or 2");
        e->opt_lm_keep = (int)v;
        e->mplans.clear();
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "mega_att_early")) {
        e->opt_mega_att_early = v != 0;
        e->mplans.clear();
    } else if (!std::strcmp(key, "att_mbuf")) {
        e->opt_att_mbuf = v != 0;
        e->mplans.clear();
    } else if (!std::strcmp(key, "mega_splits_cap")) {
        if (v < 1) fail(EL_INVALID_ARGUMENT, "mega_splits_cap must be >= 1");
        e->opt_mega_splits_cap = (int)v;
        e->mplans.clear();
    } else if (!std::strcmp(key, "mega_down_splits")) {
        e->opt_mega_down_splits = (int)v;
        e->mplans.clear();
    } else if (!std::strcmp(key, "mega_bm_down")) {
        e->opt_mega_bm_down = v != 0;
        e->mplans.clear();
    } else if (!std::strcmp(key, "mega_bm_m128")) {
        e->opt_mega_bm_m128 = v != 0;
        e->mplans.clear();
    } else if (!std::strcmp(key, "mega_bm_nt_min")) {
        if (v != 16 && v != 32 && v != 64 && v != 128) fail(EL_INVALID_ARGUMENT, "mega_bm_nt_min: 16/32/64/128");
        e->opt_mega_bm_nt_min = (int)v;
        e->mplans.clear();
    } else if (!std::strcmp(key, "mega_bm_prefetch")) {
        e->opt_mega_bm_prefetch = v != 0;
        e->mplans.clear();
    } else if (!std::strcmp(key, "mega_bm_max")) {
        e->opt_mega_bm_max = (int)v;
        e->mplans.clear();
    } else if (!std::strcmp(key, "mega_fill_splits") || !std::strcmp(key, "mega_att_stages")) {
        if (v < 0 || v > 16) fail(EL_INVALID_ARGUMENT, "value out of range");
        (key[5] == 'f' ? e->opt_mega_fill_splits : e->opt_mega_att_stages) = (int)v;
        e->mplans.clear();
    }
    else if (!std::strcmp(key, "fuse_exit")) {
        e->fuse_exit = v != 0;
        e->fuse_exit_all = v == 2;
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "body_head")) {
        e->body_head = v != 0;
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "dbg")) {
        e->dbg = (int)v;
        e->invalidate_graphs();
    }
    else if (!std::strcmp(key, "attn_cb") || !std::strcmp(key, "attn_stages")) {
        if (v < 0 || v > 8) fail(EL_INVALID_ARGUMENT, "%s must be in [0 (auto), 8]", key);
        (key[5] == 'c' ? e->opt_attn_cb : e->opt_attn_stages) = (int)v;
        e->plan_attention();
    } else if (!std::strcmp(key, "sched_defer")) {  // layer-level scheduling: deferred token turns (default 1)
        e->opt_sched_defer = v != 0;
    } else if (!std::strcmp(key, "mega_bm_wstream")) {  // -1 auto (pipelined kernel), 0 off, 1 on
        if (v < -1 || v > 1) fail(EL_INVALID_ARGUMENT, "mega_bm_wstream must be -1, 0 or 1");
        e->opt_mega_bm_wstream = (int)v;
        e->mplans.clear();
    } else if (!std::strcmp(key, "attn_grid")) {  // standalone attention kernel on at most v CTAs (0 = all)
        if (v < 0) fail(EL_INVALID_ARGUMENT, "attn_grid must be >= 0");
        e->opt_attn_grid = (int)v;
        e->plan_attention();
    } else if (!std::strcmp(key, "nsplit") || !std::strcmp(key, "cta_target")) {
        if (v < 1) fail(EL_INVALID_ARGUMENT, "value must be >= 1");
        (key[0] == 'n' ? e->opt_nsplit : e->opt_cta_target) = (int)v;
        e->plans.clear();
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "fill_splits")) {
        if (v < 1 || v > 8) fail(EL_INVALID_ARGUMENT, "fill_splits must be in [1, 8]");
        e->opt_fill_splits = (int)v;
        e->plans.clear();
        e->invalidate_graphs();
    } else if (!std::strcmp(key, "splits_cap")) {
        if (v < 1 || v > 8) fail(EL_INVALID_ARGUMENT, "splits_cap must be in [1, 8]");
        e->opt_splits_cap = (int)v;
        e->plans.clear();
        e->invalidate_graphs();
    }
    else if (!std::strcmp(key, "pdl")) {
        e->pdl = v != 0;
        e->invalidate_graphs();
    }
    else if (!std::strcmp(key, "rec_cap")) {
        if (v < 1) fail(EL_INVALID_ARGUMENT, "rec_cap must be >= 1");
        e->rec_cap = (int)v;
        e->rec.alloc((size_t)v * e->rec_stride);
        e->run_log.alloc((size_t)2 * v);
        e->invalidate_graphs();
    } else fail(EL_INVALID_ARGUMENT, "unknown option %s", key);
    API_END
}

int el_engine_run(el_engine* e, int n, const double* arrival, const int32_t* off, const int32_t* prompt,
                  const int32_t* max_new, el_transcript** out) {
    API_BEGIN
    *out = e->run(n, arrival, off, prompt, max_new);
    API_END
}

int64_t el_transcript_len(const el_transcript* t, const char* f) {
    auto* tt = const_cast<el_transcript*>(t);
    if (auto* a = tt->i32(f)) return (int64_t)a->size();
    if (auto* b = tt->f64(f)) return (int64_t)b->size();
    return -1;
}
int el_transcript_get_i32(const el_transcript* t, const char* f, int32_t* out) {
    auto* a = const_cast<el_transcript*>(t)->i32(f);
    if (!a) { g_err = std::string("unknown field ") + f; return EL_INVALID_ARGUMENT; }
    if (!a->empty()) std::memcpy(out, a->data(), sizeof(int32_t) * a->size());
    return EL_OK;
}
int el_transcript_get_f64(const el_transcript* t, const char* f, double* out) {
    auto* a = const_cast<el_transcript*>(t)->f64(f);
    if (!a) { g_err = std::string("unknown field ") + f; return EL_INVALID_ARGUMENT; }
    if (!a->empty()) std::memcpy(out, a->data(), sizeof(double) * a->size());
    return EL_OK;
}
int el_transcript_kv(const el_transcript* t, int seq, int layer, double* k, double* v, int64_t cap) {
    auto it = t->caps.find(seq);
    if (it == t->caps.end() || !it->second.have_kv) { g_err = "no kv capture for seq"; return -EL_INVALID_ARGUMENT; }
    const Capture& c = it->second;
    const size_t n = (size_t)c.committed * t->d;
    if ((int64_t)n > cap || layer < 1 || layer > t->L) { g_err = "bad kv request"; return -EL_INVALID_ARGUMENT; }
    std::memcpy(k, c.k.data() + (size_t)(layer - 1) * n, sizeof(double) * n);
    std::memcpy(v, c.v.data() + (size_t)(layer - 1) * n, sizeof(double) * n);
    return c.committed;
}
int el_transcript_block_table(const el_transcript* t, int seq, int32_t* out, int64_t cap) {
    auto it = t->caps.find(seq);
    if (it == t->caps.end() || !it->second.have_kv) { g_err = "no capture for seq"; return -EL_INVALID_ARGUMENT; }
    const Capture& c = it->second;
    if ((int64_t)c.table.size() > cap) { g_err = "buffer too small"; return -EL_INVALID_ARGUMENT; }
    std::memcpy(out, c.table.data(), sizeof(int32_t) * c.table.size());
    return c.bpl;
}
int el_transcript_exit_states(const el_transcript* t, int seq, double* out, int64_t cap) {
    auto it = t->caps.find(seq);
    if (it == t->caps.end()) { g_err = "no capture for seq"; return -EL_INVALID_ARGUMENT; }
    const auto& x = it->second.exit_states;
    if ((int64_t)x.size() > cap) { g_err = "buffer too small"; return -EL_INVALID_ARGUMENT; }
    std::memcpy(out, x.data(), sizeof(double) * x.size());
    return (int)(x.size() / (size_t)t->d);
}
void el_transcript_free(el_transcript* t) { delete t; }

int el_session_begin(el_engine* e, int B, const int32_t* first, int prefix_len, int capacity, uint64_t kv_seed,
                     const int32_t* ids) {
    API_BEGIN
    e->session_begin(B, first, prefix_len, capacity, kv_seed, ids);
    API_END
}
int el_session_end(el_engine* e) {
    API_BEGIN
    e->session_end();
    API_END
}

int el_decode_iteration(el_engine* e, const int32_t* tokens_in, int32_t* tokens_out, int32_t* accept_out,
                        float* conf_out, int32_t* output_layer) {
    API_BEGIN
    e->need_session();
    e->check_capacity(1);
    const int B = e->sess_B;
    if (tokens_in)  // embed() rejects ids outside the vocabulary (model.cpp:171-183)
        for (int b = 0; b < B; ++b)
            if (tokens_in[b] < 0 || tokens_in[b] >= e->cfg.vocab_size)
                fail(EL_INVALID_ARGUMENT, "embed: token id %d outside vocab", tokens_in[b]);
    if (tokens_in) CK(cudaMemcpyAsync(e->row_tok.p, tokens_in, sizeof(int) * B, cudaMemcpyHostToDevice, e->stream));
    e->iteration(B);
    const auto o = e->read_iteration(e->sess_iters, B);
    e->sess_iters++;
    if (tokens_out) std::memcpy(tokens_out, o.tok.data(), sizeof(int) * B);
    if (accept_out) std::memcpy(accept_out, o.acc.data(), sizeof(int) * B);
    if (conf_out) std::memcpy(conf_out, o.conf.data(), sizeof(float) * o.conf.size());
    if (output_layer) *output_layer = o.out_layer;
    API_END
}

int el_decode_run(el_engine* e, int n) {
    API_BEGIN
    e->need_session();
    e->check_capacity(n);
    for (int i = 0; i < n; ++i) e->iteration(e->sess_B);
    e->sess_iters += n;
    API_END
}

int el_decode_records(el_engine* e, int first, int n, int32_t* tokens, int32_t* accept, int32_t* out_layer,
                      float* conf) {
    API_BEGIN
    e->need_session();
    if (first < 0 || first + n > e->sess_iters || n > e->rec_cap || first < e->sess_iters - e->rec_cap)
        fail(EL_INVALID_ARGUMENT, "records [%d, %d) not available", first, first + n);
    CK(cudaStreamSynchronize(e->stream));
    const int B = e->sess_B, L = e->dm.L;
    for (int i = 0; i < n; ++i) {
        const auto o = e->read_iteration(first + i, B);
        if (tokens) std::memcpy(tokens + (size_t)i * B, o.tok.data(), sizeof(int) * B);
        if (accept) std::memcpy(accept + (size_t)i * B, o.acc.data(), sizeof(int) * B);
        if (out_layer) out_layer[i] = o.out_layer;
        if (conf) std::memcpy(conf + (size_t)i * L * B, o.conf.data(), sizeof(float) * L * B);
    }
    API_END
}

int el_decode_iterations_done(el_engine* e) { return e->sess_iters; }

int el_set_fixed_confidences(el_engine* e, const float* conf) {
    API_BEGIN
    e->need_session();
    const int B = e->sess_B, L = e->dm.L, Bm = e->dm.Bmax;
    std::vector<float> buf((size_t)L * Bm, 0.f);
    for (int l = 0; l < L; ++l)
        for (int b = 0; b < B; ++b) buf[(size_t)l * Bm + b] = conf[(size_t)l * B + b];
    CK(cudaMemcpyAsync(e->fixed_conf.p, buf.data(), sizeof(float) * buf.size(), cudaMemcpyHostToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    API_END
}

int el_session_kv(el_engine* e, int row, int layer, int pos, float* k, float* v) {
    API_BEGIN
    e->need_session();
    if (row < 0 || row >= e->sess_B || layer < 1 || layer > e->dm.L || pos < 0 || pos >= e->sess_prefix + e->sess_iters)
        fail(EL_RUNTIME_ERROR, "view: entries missing at (row %d, layer %d, position %d)", row, layer, pos);
    CK(cudaStreamSynchronize(e->stream));
    int slot = 0;
    CK(cudaMemcpy(&slot, e->row_slot.p + row, sizeof(int), cudaMemcpyDeviceToHost));
    const auto kk = e->read_kv(slot, layer, pos, 0), vv = e->read_kv(slot, layer, pos, 1);
    std::memcpy(k, kk.data(), sizeof(float) * kk.size());
    std::memcpy(v, vv.data(), sizeof(float) * vv.size());
    API_END
}

int el_session_cross_kv(el_engine* e, int row, int layer, float* k, float* v) {
    API_BEGIN
    e->need_session();
    if (e->cfg.encoder_len <= 0) fail(EL_INVALID_ARGUMENT, "cross K/V: not in T5 mode");
    if (row < 0 || row >= e->sess_B || layer < 1 || layer > e->dm.L) fail(EL_INVALID_ARGUMENT, "bad row / layer");
    CK(cudaStreamSynchronize(e->stream));
    int slot = 0;
    CK(cudaMemcpy(&slot, e->row_slot.p + row, sizeof(int), cudaMemcpyDeviceToHost));
    const int T = e->cfg.encoder_len, d = e->dm.d, dp = e->dm.dp, bc = e->dm.bc;
    const size_t blk0 = ((size_t)slot * e->dm.L + (layer - 1)) * e->enc_blocks;  // identity cross tables
    std::vector<uint16_t> kb((size_t)T * dp), vb((size_t)T * dp);
    CK(cudaMemcpy(kb.data(), e->ckpool.p + blk0 * bc * dp, sizeof(uint16_t) * kb.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(vb.data(), e->cvpool.p + blk0 * bc * dp, sizeof(uint16_t) * vb.size(), cudaMemcpyDeviceToHost));
    for (int t = 0; t < T; ++t)
        for (int i = 0; i < d; ++i) {
            uint32_t a = (uint32_t)kb[(size_t)t * dp + i] << 16, b = (uint32_t)vb[(size_t)t * dp + i] << 16;
            std::memcpy(k + (size_t)t * d + i, &a, 4);
            std::memcpy(v + (size_t)t * d + i, &b, 4);
        }
    API_END
}

int el_session_hidden(el_engine* e, int parity, float* out) {
    API_BEGIN
    e->need_session();
    CK(cudaStreamSynchronize(e->stream));
    const int B = e->sess_B, dp = e->dm.dp, d = e->dm.d;
    std::vector<float> buf((size_t)B * dp);
    CK(cudaMemcpy(buf.data(), e->h32.p + (size_t)(parity & 1) * e->dm.Bmax * dp, sizeof(float) * buf.size(),
                  cudaMemcpyDeviceToHost));
    for (int b = 0; b < B; ++b) std::memcpy(out + (size_t)b * d, buf.data() + (size_t)b * dp, sizeof(float) * d);
    API_END
}

int el_session_block_table(el_engine* e, int row, int32_t* out, int bpl_cap) {
    API_BEGIN
    e->need_session();
    CK(cudaStreamSynchronize(e->stream));
    int slot = 0;
    CK(cudaMemcpy(&slot, e->row_slot.p + row, sizeof(int), cudaMemcpyDeviceToHost));
    const int bpl = e->slot_bpl[(size_t)slot];
    if (bpl > bpl_cap) fail(EL_INVALID_ARGUMENT, "bpl_cap too small");
    for (int l = 0; l < e->dm.L; ++l)
        CK(cudaMemcpy(out + (size_t)l * bpl, e->tables.p + ((size_t)slot * e->dm.L + l) * e->dm.bpl_max,
                      sizeof(int) * bpl, cudaMemcpyDeviceToHost));
    return bpl;
    API_END
}

int el_time_decode(el_engine* e, int n, float* ms) {
    API_BEGIN
    e->need_session();
    e->check_capacity(n);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaStreamSynchronize(e->stream));
    CK(cudaEventRecord(a, e->stream));
    for (int i = 0; i < n; ++i) e->iteration(e->sess_B);
    CK(cudaEventRecord(b, e->stream));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    e->sess_iters += n;
    API_END
}

int el_time_kernel(el_engine* e, int kind, int layer, int reps, float* ms) {
    API_BEGIN
    e->need_session();
    if (layer < 1 || layer > e->dm.L) fail(EL_INVALID_ARGUMENT, "layer out of range");
    const bool flush = (kind & 0x100) != 0;
    kind &= 0xff;
    const int B = e->sess_B;
    auto& P = e->plans_for(B);
    el::DevState s = e->state(false, B);
    s.cont_host = nullptr;
    CK(cudaMemcpyAsync(e->layer.p, &layer, sizeof(int), cudaMemcpyHostToDevice, e->stream));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto one = [&]() {
        switch (kind) {
            case 0: el::launch_attention(s, e->stream, false); break;
            case 1: el::launch_gemm(el::kGemmQkv, P.qkv, s, e->stream, false); break;
            case 2: el::launch_gemm(el::kGemmWo, P.wo, s, e->stream, false); break;
            case 3: el::launch_gemm(el::kGemmUp, P.up, s, e->stream, false); break;
            case 4: el::launch_gemm(el::kGemmDown, P.down, s, e->stream, false); break;
            case 5: el::launch_gemm(el::kGemmLmCheck, P.lm, s, e->stream, false); break;
            default: fail(EL_INVALID_ARGUMENT, "unknown kernel kind %d", kind);
        }
    };
    // note: kind 1 rewrites K/V at the current position of `layer` with the same
    // values the iteration would write (idempotent for timing purposes)
    one();
    CK(cudaStreamSynchronize(e->stream));
    if (flush) {
        // cold-L2 timing: a 256 MB write (2x the 126 MB L2) before every launch, each
        // launch bracketed by its own events on the engine stream
        if (!e->l2flush.p) e->l2flush.alloc((size_t)256 << 20, false);
        float total = 0.f;
        for (int i = 0; i < reps; ++i) {
            CK(cudaMemsetAsync(e->l2flush.p, i & 0xff, e->l2flush.n, e->stream));
            CK(cudaEventRecord(a, e->stream));
            one();
            CK(cudaEventRecord(b, e->stream));
            CK(cudaEventSynchronize(b));
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, a, b));
            total += t;
        }
        *ms = total / (float)reps;
    } else {
        CK(cudaEventRecord(a, e->stream));
        for (int i = 0; i < reps; ++i) one();
        CK(cudaEventRecord(b, e->stream));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(ms, a, b));
        *ms /= (float)reps;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    API_END
}

int el_debug_timeline_reset(el_engine* e) {
    API_BEGIN
    std::vector<unsigned long long> v(2 * 32 * 16);
    for (size_t i = 0; i < v.size(); i += 2) {
        v[i] = ~0ull;
        v[i + 1] = 0;
    }
    CK(cudaMemcpyAsync(e->dbg_ts.p + 16384, v.data(), sizeof(unsigned long long) * v.size(), cudaMemcpyHostToDevice,
                       e->stream));
    CK(cudaStreamSynchronize(e->stream));
    API_END
}

int el_debug_timestamps(el_engine* e, uint64_t* out, int n) {
    API_BEGIN
    CK(cudaStreamSynchronize(e->stream));
    CK(cudaMemcpy(out, e->dbg_ts.p, sizeof(uint64_t) * std::min<size_t>((size_t)n, e->dbg_ts.n), cudaMemcpyDeviceToHost));
    API_END
}

int el_sync(el_engine* e) {
    API_BEGIN
    CK(cudaStreamSynchronize(e->stream));
    API_END
}

int el_launches_per_iteration(el_engine* e, int output_layer) { return e->launches_per_iteration(output_layer); }

int el_plan_info(el_engine* e, int64_t* out, int cap) {
    API_BEGIN
    auto& P = e->plans_for(e->in_session ? e->sess_B : e->dm.Bmax);
    auto& M = e->mplan_for(e->in_session ? e->sess_B : e->dm.Bmax);
    const int64_t v[] = {e->attn_cb,    e->attn_stages,   e->attn_max_chunks, P.n_pad,       P.qkv.splits,
                         P.wo.splits,   P.up.splits,      P.down.splits,      P.fill.splits, P.down.stages,
                         P.lm.m_tiles,  e->dm.dp,         e->dm.fp,           e->dm.Vp,      e->dm.bpl_max,
                         // persistent kernel: modes (1 = batch-M), splits, N per unit, ring depths
                         M.g[el::kIQkv].mode, M.g[el::kIWo].mode, M.g[el::kIUp].mode,
                         M.g[el::kIQkv].splits, M.g[el::kIWo].splits, M.g[el::kIUp].splits, M.g[el::kIDown].splits,
                         M.g[el::kIFill].splits, M.g[el::kIQkv].nt, M.g[el::kIWo].nt, M.g[el::kIUp].nt,
                         M.stages, M.bm_stages, e->mega_att_stages,
                         e->mega_for(e->in_session ? e->sess_B : e->dm.Bmax) ? 1 : 0,
                         (e->mega_for(e->in_session ? e->sess_B : e->dm.Bmax) &&
                          e->pipe_for(e->in_session ? e->sess_B : e->dm.Bmax)) ? 1 : 0,
                         M.lm_pair, M.lm_keep, M.lm_tail_tr, M.lm_stages};
    const int n = (int)(sizeof v / sizeof v[0]);
    for (int i = 0; i < std::min(n, cap); ++i) out[i] = v[i];
    return n;
    API_END
}

int el_kv_block_trace(int L, int pool, int cap, int n_ops, const int32_t* ops, const int32_t* caps, int n_ids,
                      int bpl_max, int32_t* tables) {
    try {
        if (L <= 0 || pool <= 0 || cap <= 0) fail(EL_INVALID_ARGUMENT, "KvStore: all constructor parameters must be positive");
        std::vector<int> stack((size_t)pool);
        for (int i = 0; i < pool; ++i) stack[(size_t)i] = pool - 1 - i;
        int top = pool;
        std::vector<std::vector<int>> tab((size_t)n_ids);
        for (int64_t i = 0; i < (int64_t)n_ids * L * bpl_max; ++i) tables[i] = -1;
        for (int i = 0; i < n_ops; ++i) {
            if (ops[i] > 0) {
                const int id = ops[i] - 1;
                if (id >= n_ids) fail(EL_INVALID_ARGUMENT, "allocate: id out of range");
                if (!tab[(size_t)id].empty()) fail(EL_INVALID_ARGUMENT, "allocate: seq_id %d already allocated", id);
                const int bpl = ceil_div(caps[i], cap);
                if ((long)bpl * L > top) continue;  // KvOutOfMemory: admission defers
                std::vector<int> flat((size_t)bpl * L);
                el::kv_pop_host(stack.data(), top, flat.data(), bpl * L);
                top -= bpl * L;
                for (int l = 0; l < L; ++l)
                    for (int b = 0; b < bpl && b < bpl_max; ++b)
                        tables[((size_t)id * L + l) * bpl_max + b] = flat[(size_t)l * bpl + b];
                tab[(size_t)id] = flat;
                if (flat.empty()) tab[(size_t)id].push_back(-1);
            } else if (ops[i] < 0) {
                const int id = -ops[i] - 1;
                if (id >= n_ids || tab[(size_t)id].empty())
                    fail(EL_INVALID_ARGUMENT, "release: unknown or already released seq_id %d", id);
                auto& flat = tab[(size_t)id];
                if (!(flat.size() == 1 && flat[0] == -1)) {
                    el::kv_push_host(stack.data(), top, flat.data(), (int)flat.size());
                    top += (int)flat.size();
                }
                flat.clear();
            }
        }
        return top;
    } catch (const ElError& e) {
        g_err = e.msg;
        return -e.code;
    }
}


// compute_metrics (metrics.cpp:13-58) over flat transcript fields
int el_metrics_compute(int L, int n_iters, const int32_t* it_out, const int32_t* it_off, int n_seqs,
                       const int32_t* sq_id, const int32_t* tok_off, const int32_t* sq_exit, const double* sq_first,
                       const double* sq_finish, const double* meta, el_metrics* r, int64_t* exit_hist,
                       int64_t* accept_hist) {
    API_BEGIN
    if (L < 1 || n_iters < 0 || n_seqs < 0 || !r) fail(EL_INVALID_ARGUMENT, "compute_metrics: bad arguments");
    *r = el_metrics{};
    r->n_layers = L;
    std::vector<int64_t> eh((size_t)L, 0), ah((size_t)L, 0);
    r->total_sim_time = meta[0];
    r->total_idle_time = meta[1];
    r->iterations = n_iters;
    r->pool_blocks = (int)meta[2];
    r->free_blocks = (int)meta[3];
    r->peak_blocks = (int)meta[4];
    double latency_sum = 0.0;
    for (int s = 0; s < n_seqs; ++s) {
        if (sq_finish[s] < 0.0 || sq_first[s] < 0.0)
            fail(EL_INVALID_ARGUMENT, "compute_metrics: sequence %d is unfinished", sq_id ? sq_id[s] : s);
        r->total_tokens += tok_off[s + 1] - tok_off[s];
        latency_sum += sq_finish[s] - sq_first[s];
        for (int i = tok_off[s]; i < tok_off[s + 1]; ++i) {
            if (sq_exit[i] < 1 || sq_exit[i] > L) fail(EL_INVALID_ARGUMENT, "compute_metrics: accept layer out of range");
            ++ah[(size_t)sq_exit[i] - 1];
        }
    }
    int64_t early = 0, layer_sum = 0;
    for (int i = 0; i < n_iters; ++i) {
        const int64_t batch = it_off[i + 1] - it_off[i];
        if (it_out[i] < 1 || it_out[i] > L) fail(EL_INVALID_ARGUMENT, "compute_metrics: output layer out of range");
        eh[(size_t)it_out[i] - 1] += batch;
        layer_sum += batch * it_out[i];
        if (it_out[i] < L) early += batch;
    }
    if (r->total_tokens > 0) {
        r->inner_token_latency = latency_sum / (double)r->total_tokens;
        r->early_exit_rate_pct = 100.0 * (double)early / (double)r->total_tokens;
        r->mean_layers_per_token = (double)layer_sum / (double)r->total_tokens;
        if (r->total_sim_time > 0.0) r->throughput = (double)r->total_tokens / r->total_sim_time;
    }
    if (exit_hist) std::memcpy(exit_hist, eh.data(), sizeof(int64_t) * (size_t)L);
    if (accept_hist) std::memcpy(accept_hist, ah.data(), sizeof(int64_t) * (size_t)L);
    API_END
}

int el_transcript_metrics(const el_transcript* t, el_metrics* out, int64_t* exit_hist, int64_t* accept_hist) {
    if (!t) {
        g_err = "null transcript";
        return EL_INVALID_ARGUMENT;
    }
    return el_metrics_compute(t->L, (int)t->it_output_layer.size(), t->it_output_layer.data(), t->it_batch_off.data(),
                              (int)t->sq_id.size(), t->sq_id.data(), t->sq_tok_off.data(), t->sq_exit_layers.data(),
                              t->sq_first.data(), t->sq_finish.data(), t->meta.data(), out, exit_hist, accept_hist);
}


// ---- sub-engine API (KvStore / layer_forward / fill_skipped / confidences / greedy) ----
int el_kv_allocate(el_engine* e, int seq_id, int capacity_tokens) {
    API_BEGIN
    e->store_allocate(seq_id, capacity_tokens);
    API_END
}
int el_kv_release(el_engine* e, int seq_id) {
    API_BEGIN
    e->store_release(seq_id);
    API_END
}
int el_kv_append(el_engine* e, int seq_id, int layer, int position, const float* k, const float* v) {
    API_BEGIN
    if (!k || !v) fail(EL_INVALID_ARGUMENT, "append: null K/V");
    e->store_append(seq_id, layer, position, k, v);
    API_END
}
int el_kv_view(el_engine* e, int seq_id, int layer, int upto_position, float* k, float* v) {
    API_BEGIN
    e->store_view(seq_id, layer, upto_position, k, v);
    API_END
}
int el_kv_commit(el_engine* e, int seq_id) {
    API_BEGIN
    e->store_commit(seq_id);
    API_END
}
int el_kv_lengths(el_engine* e, int seq_id, int32_t* committed, int32_t* written) {
    API_BEGIN
    auto& q = e->store_entry(seq_id, "committed_len");
    if (committed) *committed = q.committed;
    if (written) for (int l = 0; l < e->dm.L; ++l) written[l] = q.written[(size_t)l];
    API_END
}
int el_kv_stats(el_engine* e, int32_t* out4) {
    API_BEGIN
    out4[0] = e->cfg.pool_blocks;
    out4[1] = e->top;
    out4[2] = e->peak;
    out4[3] = (int32_t)e->store.size();
    API_END
}
int el_layer_forward(el_engine* e, int layer, int n, const int32_t* seq_ids, const float* h_in, float* h_out) {
    API_BEGIN
    e->layer_forward(layer, n, seq_ids, h_in, h_out);
    API_END
}
int el_kv_fill(el_engine* e, int n, const int32_t* seq_ids, const float* h_exit, int output_layer) {
    API_BEGIN
    e->kv_fill(n, seq_ids, h_exit, output_layer);
    API_END
}
int el_exit_confidence(el_engine* e, int layer, int n, const float* h_prev, const float* h_cur, float* conf,
                       int32_t* accept) {
    API_BEGIN
    e->exit_confidence(layer, n, h_prev, h_cur, conf, accept);
    API_END
}
int el_greedy_tokens(el_engine* e, int n, const float* h, int32_t* tokens) {
    API_BEGIN
    e->greedy_tokens(n, h, tokens);
    API_END
}


// ---- layer-level scheduling (f4) over a session's batch ----
int el_sched_begin(el_engine* e, int policy, const double* lin_m) {
    API_BEGIN
    e->sched_begin(policy, lin_m);
    API_END
}
int el_sched_run(el_engine* e, int n_turns, float* ms) {
    API_BEGIN
    if (!e->sch.on) fail(EL_LOGIC_ERROR, "layer-level scheduling not started (el_sched_begin)");
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaStreamSynchronize(e->stream));
    CK(cudaEventRecord(a, e->stream));
    for (int i = 0; i < n_turns; ++i) e->sched_turn();
    CK(cudaEventRecord(b, e->stream));
    CK(cudaEventSynchronize(b));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (ms) *ms = t;
    API_END
}
int el_sched_tokens(el_engine* e, int row, int32_t* tokens, int32_t* exit_layers, int cap) {
    // returns the count (>= 0) or -EL_* on error
    if (!e->sch.on || row < 0 || row >= e->sess_B) {
        g_err = "sched_tokens: layer-level scheduling not started or bad row";
        return -EL_INVALID_ARGUMENT;
    }
    const auto& t = e->sch.toks[(size_t)row];
    const auto& x = e->sch.exits[(size_t)row];
    const int n = std::min(cap, (int)t.size());
    for (int i = 0; i < n; ++i) {
        if (tokens) tokens[i] = t[(size_t)i];
        if (exit_layers) exit_layers[i] = x[(size_t)i];
    }
    return (int)t.size();
}
int el_sched_turns(el_engine* e, int32_t* layers, int32_t* rows, int cap) {
    if (!e->sch.on) {
        g_err = "layer-level scheduling not started";
        return -EL_LOGIC_ERROR;
    }
    const int n = std::min(cap, (int)e->sch.turn_layer.size());
    for (int i = 0; i < n; ++i) {
        if (layers) layers[i] = e->sch.turn_layer[(size_t)i];
        if (rows) rows[i] = e->sch.turn_n[(size_t)i];
    }
    return (int)e->sch.turn_layer.size();
}

int el_model_tensor(el_engine* e, int which, int layer, uint16_t* out, int64_t cap) {
    API_BEGIN
    const int d = e->dm.d, dp = e->dm.dp, fp = e->dm.fp, V = e->dm.V, L = e->dm.L;
    const uint16_t* base = nullptr;
    int rows = 0, cols = 0, ld = 0;
    if (which == 0 || which == 1) {
        base = which == 0 ? e->emb.p : e->lm.p;
        rows = V; cols = d; ld = dp;
    } else if (which == 2 || which == 3) {
        // probe as fp32 bit patterns split into two uint16 halves: return bf16 bits
        if (which == 2) {
            if (cap < d) fail(EL_INVALID_ARGUMENT, "buffer too small");
            std::vector<float> pw((size_t)dp);
            CK(cudaMemcpy(pw.data(), e->probe_w.p, sizeof(float) * dp, cudaMemcpyDeviceToHost));
            for (int i = 0; i < d; ++i) {
                uint32_t u;
                std::memcpy(&u, &pw[(size_t)i], 4);
                out[i] = (uint16_t)(u >> 16);
            }
        } else {
            uint32_t u;
            std::memcpy(&u, &e->probe_b, 4);
            out[0] = (uint16_t)(u >> 16);
        }
        return EL_OK;
    } else if (which >= 4 && which <= 9) {
        if (layer < 1 || layer > L) fail(EL_INVALID_ARGUMENT, "layer out of range");
        const int k = which - 4, i = layer - 1;
        switch (k) {
            case 0: case 1: case 2:
                base = e->wqkv.p + (size_t)i * 3 * dp * dp + (size_t)k * dp * dp; rows = d; cols = d; ld = dp; break;
            case 3: base = e->wo.p + (size_t)i * dp * dp; rows = d; cols = d; ld = dp; break;
            case 4: base = e->wup.p + (size_t)i * fp * dp; rows = 4 * d; cols = d; ld = dp; break;
            case 5: base = e->wdown.p + (size_t)i * dp * fp; rows = d; cols = 4 * d; ld = fp; break;
        }
    } else fail(EL_INVALID_ARGUMENT, "bad tensor id");
    if (cap < (int64_t)rows * cols) fail(EL_INVALID_ARGUMENT, "buffer too small");
    if (which == 0) {
        CK(cudaMemcpy2D(out, sizeof(uint16_t) * cols, base, sizeof(uint16_t) * ld, sizeof(uint16_t) * cols, rows,
                        cudaMemcpyDeviceToHost));
    } else {  // tiled + swizzled GEMM operand: copy the padded block and untile on the host
        const int rows_p = round_up(rows, 128);
        std::vector<uint16_t> buf((size_t)rows_p * ld);
        CK(cudaMemcpy(buf.data(), base, sizeof(uint16_t) * buf.size(), cudaMemcpyDeviceToHost));
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) out[(size_t)r * cols + c] = buf[el::tiled_offset(r, c, ld)];
    }
    API_END
}

}  // extern "C"

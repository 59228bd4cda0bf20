// el_kernels.cu -- sm_100a kernels of the batched early-exit decode iteration.
//
// Reference path (all citations /root/reference/proj):
//   decode_iteration        src/engine.cpp:208-310  (Algorithm 1)
//   layer_forward           src/model.cpp:197-272
//   fill_skipped            src/kv_cache.cpp:222-234 + compute_kv_pair model.cpp:274-282
//   exit confidences/decide src/exit_policy.cpp:57-115, threshold_at 50-55
//   ExitStatusVector        src/engine.cpp:47-75
//   lm_head + greedy_token  src/model.cpp:284-299
//   KvStore allocate/release src/kv_cache.cpp:78-106, 182-194
#include <cuda_runtime_api.h>

#include <cstdio>

#include "el_common.cuh"
#include "el_kernels.h"

namespace el {

#define EL_CUDA_LAUNCH_CHECK()                                                              \
    do {                                                                                    \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess) {                                                            \
            fprintf(stderr, "exitlab-b200 launch error %s at %s:%d\n", cudaGetErrorString(e_), \
                    __FILE__, __LINE__);                                                    \
        }                                                                                   \
    } while (0)

// ===========================================================================
// 1. Weight-streaming GEMM on tcgen05:  D[M x N] = W[M x K] . X[N x K]^T
//    swap-AB: weights are the M=128 operand (K-major, TMA, 128B swizzle), the
//    batch is N (16..256). Split-K across blockIdx.y; the last-arriving CTA of
//    a tile reduces the fp32 partials in fixed split order (deterministic) and
//    runs the fused epilogue.
// ===========================================================================
struct EpiSmem {
    int layer;     // layer the weights belong to (1-based)
    int par_in;    // hidden-state parity read by this GEMM
    int par_out;
    int row0;      // first output row of this tile inside the layer's weight block
    int last;      // split-K: this CTA reduces
    int pad[3];
    long long dst[256];  // per-column KV destination element offsets
};

constexpr int kBM = 128, kBK = 64;
constexpr int kAStage = kBM * kBK * 2;  // 16 KB

template <GemmKind K>
struct Epi;

// --- q | k | v projection; K,V scattered into the paged pool at (slot, layer, pos)
//     (model.cpp:218-226: matvec_batch w_q/w_k/w_v + KvStore::append)
template <>
struct Epi<kGemmQkv> {
    static constexpr bool kTile = false;
    __device__ static bool setup(const DevState& st, int tile, EpiSmem& e, int& a_row, int& b_row) {
        const int layer = *st.layer;
        e.layer = layer;
        e.row0 = tile * kBM;
        a_row = (layer - 1) * 3 * st.dm.dp + tile * kBM;
        b_row = ((layer - 1) & 1) * st.dm.Bmax;
        return true;
    }
    __device__ static void prologue(const DevState& st, EpiSmem& e) {
        const Dims& dm = st.dm;
        for (int b = threadIdx.x; b < st.rows.B; b += blockDim.x) {
            const int slot = st.rows.slot[b], pos = st.rows.pos[b];
            const int blk = st.tables[((size_t)slot * dm.L + (e.layer - 1)) * dm.bpl_max + pos / dm.bc];
            e.dst[b] = ((long long)blk * dm.bc + pos % dm.bc) * dm.dp;
        }
    }
    __device__ static void apply(const DevState& st, const EpiSmem& e, int row, int col, float v) {
        const int dp = st.dm.dp;
        const int m = e.row0 + row;
        if (m < dp) st.q32[(size_t)col * dp + m] = v;
        else if (m < 2 * dp) st.kpool[e.dst[col] + (m - dp)] = f32_to_bf16(v);
        else st.vpool[e.dst[col] + (m - 2 * dp)] = f32_to_bf16(v);
    }
};

// --- skipped-layer KV fill: K_j,V_j = W_kv^(j) h_e for j in (e, L]  (one
//     grouped GEMM over the contiguous W_k|W_v rows of every skipped layer;
//     kv_cache.cpp:222-234). Tiles of layers <= e exit immediately.
template <>
struct Epi<kGemmFill> {
    static constexpr bool kTile = false;
    __device__ static bool setup(const DevState& st, int tile, EpiSmem& e, int& a_row, int& b_row) {
        const int eo = *st.out_layer;
        const int t2 = 2 * st.dm.dp / kBM;
        const int j = eo + 1 + tile / t2;
        if (j > st.dm.L) return false;
        e.layer = j;
        e.row0 = (tile % t2) * kBM;
        a_row = (j - 1) * 3 * st.dm.dp + st.dm.dp + e.row0;
        b_row = (eo & 1) * st.dm.Bmax;
        return true;
    }
    __device__ static void prologue(const DevState& st, EpiSmem& e) { Epi<kGemmQkv>::prologue(st, e); }
    __device__ static void apply(const DevState& st, const EpiSmem& e, int row, int col, float v) {
        const int dp = st.dm.dp;
        const int m = e.row0 + row;
        if (m < dp) st.kpool[e.dst[col] + m] = f32_to_bf16(v);
        else st.vpool[e.dst[col] + (m - dp)] = f32_to_bf16(v);
    }
};

// --- attention output projection + residual (model.cpp:245-253)
template <>
struct Epi<kGemmWo> {
    static constexpr bool kTile = false;
    __device__ static bool setup(const DevState& st, int tile, EpiSmem& e, int& a_row, int& b_row) {
        const int layer = *st.layer;
        e.layer = layer;
        e.par_in = (layer - 1) & 1;
        e.row0 = tile * kBM;
        a_row = (layer - 1) * st.dm.dp + tile * kBM;
        b_row = 0;
        return true;
    }
    __device__ static void prologue(const DevState&, EpiSmem&) {}
    __device__ static void apply(const DevState& st, const EpiSmem& e, int row, int col, float v) {
        const int dp = st.dm.dp;
        const size_t i = (size_t)col * dp + e.row0 + row;
        const float h = st.h32[(size_t)e.par_in * st.dm.Bmax * dp + i];
        const float o = h + v;
        st.mid32[i] = o;
        st.mid_b[i] = f32_to_bf16(o);
    }
};

// --- MLP up + ReLU (model.cpp:255-260)
template <>
struct Epi<kGemmUp> {
    static constexpr bool kTile = false;
    __device__ static bool setup(const DevState& st, int tile, EpiSmem& e, int& a_row, int& b_row) {
        const int layer = *st.layer;
        e.layer = layer;
        e.row0 = tile * kBM;
        a_row = (layer - 1) * st.dm.fp + tile * kBM;
        b_row = 0;
        return true;
    }
    __device__ static void prologue(const DevState&, EpiSmem&) {}
    __device__ static void apply(const DevState& st, const EpiSmem& e, int row, int col, float v) {
        st.up_b[(size_t)col * st.dm.fp + e.row0 + row] = f32_to_bf16(v > 0.f ? v : 0.f);
    }
};

// --- MLP down + residual (model.cpp:261-270); writes the layer output state
template <>
struct Epi<kGemmDown> {
    static constexpr bool kTile = false;
    __device__ static bool setup(const DevState& st, int tile, EpiSmem& e, int& a_row, int& b_row) {
        const int layer = *st.layer;
        e.layer = layer;
        e.par_out = layer & 1;
        e.row0 = tile * kBM;
        a_row = (layer - 1) * st.dm.dp + tile * kBM;
        b_row = 0;
        return true;
    }
    __device__ static void prologue(const DevState&, EpiSmem&) {}
    __device__ static void apply(const DevState& st, const EpiSmem& e, int row, int col, float v) {
        const int dp = st.dm.dp;
        const size_t i = (size_t)col * dp + e.row0 + row;
        const float o = st.mid32[i] + v;
        const size_t j = (size_t)e.par_out * st.dm.Bmax * dp + i;
        st.h32[j] = o;
        st.hb[j] = f32_to_bf16(o);
    }
};

// --- LM head with fused per-tile (max1, max2, sum exp, argmax) reduction:
//     logits never reach HBM (lm_head_logits + softmax_response_confidence /
//     greedy_token, exit_policy.cpp:57-72, model.cpp:288-299)
template <GemmKind K>
struct EpiLm {
    static constexpr bool kTile = true;
    __device__ static bool setup(const DevState& st, int tile, EpiSmem& e, int& a_row, int& b_row) {
        const int par = (K == kGemmLmCheck) ? (*st.layer & 1) : (*st.out_layer & 1);
        e.row0 = tile * kBM;
        a_row = tile * kBM;
        b_row = par * st.dm.Bmax;
        return true;
    }
    __device__ static void prologue(const DevState&, EpiSmem&) {}
    // sm: [n][129] logits of this tile (column n = batch row)
    __device__ static void tile_reduce(const DevState& st, const EpiSmem& e, int tile, const float* sm) {
        const int n = threadIdx.x;
        if (n >= st.rows.B) return;
        const int rows = min(kBM, st.dm.V - e.row0);
        float m1 = -INFINITY, m2 = -INFINITY, s = 0.f;
        int idx = 0;
        for (int r = 0; r < rows; ++r) {
            const float x = sm[n * 129 + r];
            if (x > m1) {
                m2 = m1;
                s = (m1 == -INFINITY) ? 1.f : s * __expf(m1 - x) + 1.f;
                m1 = x;
                idx = e.row0 + r;
            } else {
                if (x > m2) m2 = x;
                s += __expf(x - m1);
            }
        }
        st.lm_part[(size_t)tile * st.dm.Bmax + n] = make_float4(m1, m2, s, __int_as_float(idx));
    }
};
template <>
struct Epi<kGemmLmCheck> : EpiLm<kGemmLmCheck> {};
template <>
struct Epi<kGemmLmFinal> : EpiLm<kGemmLmFinal> {};

struct GemmArgs {
    int m_tiles, splits, kb_per_split, n_pad, stages, tmem_cols;
};

template <GemmKind K>
__global__ void __launch_bounds__(128, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs g,
                DevState st) {
    using E = Epi<K>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int tile = blockIdx.x, split = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    const uint32_t b_stage = (uint32_t)g.n_pad * kBK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)g.stages * kAStage;
    size_t region = (size_t)g.stages * (kAStage + b_stage);
    if (E::kTile && region < (size_t)g.n_pad * 129 * 4) region = (size_t)g.n_pad * 129 * 4;
    uint64_t* full = (uint64_t*)(smem + region);
    uint64_t* empty = full + g.stages;
    uint64_t* accf = empty + g.stages;
    uint32_t* tmem_slot = (uint32_t*)(accf + 1);
    EpiSmem& es = *(EpiSmem*)(((uintptr_t)(tmem_slot + 4) + 15) & ~(uintptr_t)15);

    int a_row = 0, b_row = 0;
    if (!E::setup(st, tile, es, a_row, b_row)) return;  // uniform across the CTA

    if (tid == 0) {
        for (int s = 0; s < g.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accf, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, (uint32_t)g.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int kb0 = split * g.kb_per_split;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer ----
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int kb = 0; kb < g.kb_per_split; ++kb) {
            const int s = kb % g.stages;
            if (kb >= g.stages) mbar_wait(&empty[s], ((kb / g.stages) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], kAStage + b_stage);
            tma_load_2d(sA + (size_t)s * kAStage, &tmA, &full[s], (kb0 + kb) * kBK, a_row);
            tma_load_2d(sB + (size_t)s * b_stage, &tmB, &full[s], (kb0 + kb) * kBK, b_row);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer (single thread) ----
        const uint32_t idesc = idesc_bf16_m128((uint32_t)g.n_pad);
        for (int kb = 0; kb < g.kb_per_split; ++kb) {
            const int s = kb % g.stages;
            mbar_wait(&full[s], (kb / g.stages) & 1);
            tc_fence_after();
            const uint64_t ad = sdesc_k_sw128(smem_u32(sA + (size_t)s * kAStage));
            const uint64_t bd = sdesc_k_sw128(smem_u32(sB + (size_t)s * b_stage));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
                tc_mma_bf16(tmem, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (kb | k) != 0);
            tc_commit(&empty[s]);
        }
        tc_commit(accf);
    }
    __syncwarp();

    // ---- epilogue: all four warps, thread t <-> TMEM lane t <-> output row t ----
    E::prologue(st, es);
    mbar_wait(accf, 0);
    tc_fence_after();
    __syncthreads();
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    const int nval = st.rows.B;
    const int row = tid;

    if constexpr (E::kTile) {
        // splits == 1: transpose the tile through smem (stage buffers are free now)
        float* sm = (float*)smem;
        for (int c0 = 0; c0 < nval; c0 += 16) {
            float v[16];
            tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < nval) sm[(c0 + j) * 129 + row] = v[j];
        }
        __syncthreads();
        E::tile_reduce(st, es, tile, sm);
    } else if (g.splits == 1) {
        for (int c0 = 0; c0 < nval; c0 += 16) {
            float v[16];
            tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < nval) E::apply(st, es, row, c0 + j, v[j]);
        }
    } else {
        float* my = st.gemm_ws + ((size_t)(split * g.m_tiles + tile) * g.n_pad) * kBM;
        for (int c0 = 0; c0 < nval; c0 += 16) {
            float v[16];
            tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < nval) my[(size_t)(c0 + j) * kBM + row] = v[j];
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) es.last = (atomicAdd(&st.gemm_cnt[tile], 1) == g.splits - 1);
        __syncthreads();
        if (es.last) {
            __threadfence();
            for (int c = 0; c < nval; ++c) {
                float acc = 0.f;
                for (int s = 0; s < g.splits; ++s)
                    acc += __ldcg(st.gemm_ws + ((size_t)(s * g.m_tiles + tile) * g.n_pad + c) * kBM + row);
                E::apply(st, es, row, c, acc);
            }
            if (tid == 0) st.gemm_cnt[tile] = 0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, (uint32_t)g.tmem_cols);
}

int gemm_smem_bytes(int n_pad, int stages, bool tile_reduce) {
    int main = stages * (kAStage + n_pad * kBK * 2);
    if (tile_reduce) main = main > n_pad * 129 * 4 ? main : n_pad * 129 * 4;
    return 1024 + main + (2 * stages + 1) * 8 + 16 + (int)sizeof(EpiSmem) + 64;
}

template <GemmKind K>
static void launch_gemm_t(const GemmPlan& p, const DevState& st, cudaStream_t s) {
    GemmArgs g{p.m_tiles, p.splits, p.kb_per_split, p.n_pad, p.stages, p.tmem_cols};
    gemm_kernel<K><<<dim3(p.m_tiles, p.splits), 128, p.smem_bytes, s>>>(p.tmA, p.tmB, g, st);
    EL_CUDA_LAUNCH_CHECK();
}

void launch_gemm(GemmKind kind, const GemmPlan& p, const DevState& st, cudaStream_t s) {
    switch (kind) {
        case kGemmQkv: launch_gemm_t<kGemmQkv>(p, st, s); break;
        case kGemmWo: launch_gemm_t<kGemmWo>(p, st, s); break;
        case kGemmUp: launch_gemm_t<kGemmUp>(p, st, s); break;
        case kGemmDown: launch_gemm_t<kGemmDown>(p, st, s); break;
        case kGemmLmCheck: launch_gemm_t<kGemmLmCheck>(p, st, s); break;
        case kGemmLmFinal: launch_gemm_t<kGemmLmFinal>(p, st, s); break;
        case kGemmFill: launch_gemm_t<kGemmFill>(p, st, s); break;
    }
}

// ===========================================================================
// 2. Paged single-head decode attention over the block pool
//    (model.cpp:223-243: scores = K q / sqrt(d), softmax, P V).
//    grid (chunk, row): each CTA streams a chunk of `attn_cb` KV blocks of one
//    sequence through a ring of shared-memory stages with 1-D TMA bulk copies
//    (a block is bc x dp contiguous bf16 for K and for V), keeps an online
//    softmax, and writes an unnormalised partial (o, m, l). The last CTA of a
//    sequence combines the partials in chunk order (flash-decoding) and emits
//    the bf16 attention output for the W_o GEMM.
// ===========================================================================
struct AttnSmem {
    uint64_t full[8];
    float sc[64];
    int last;
};

__device__ __forceinline__ float dot8(uint4 k, const float* q) {
    const uint32_t w[4] = {k.x, k.y, k.z, k.w};
    float a = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a = fmaf(__uint_as_float(w[i] << 16), q[2 * i], a);
        a = fmaf(__uint_as_float(w[i] & 0xFFFF0000u), q[2 * i + 1], a);
    }
    return a;
}

template <int NJ>
__global__ void __launch_bounds__(128) attn_kernel(DevState st) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 127) & ~(uintptr_t)127);
    const Dims& dm = st.dm;
    const int b = blockIdx.y, c = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int layer = *st.layer;
    const int ctx = st.rows.pos[b] + 1;
    const int nblk = (ctx + dm.bc - 1) / dm.bc;
    const int nch = (nblk + st.attn_cb - 1) / st.attn_cb;
    if (c >= nch) return;
    const int blk0 = c * st.attn_cb;
    const int n = min(nblk, blk0 + st.attn_cb) - blk0;
    const int dp = dm.dp, nchunk = dp / 8;
    const int* table = st.tables + ((size_t)st.rows.slot[b] * dm.L + (layer - 1)) * dm.bpl_max;
    const uint32_t blk_bytes = (uint32_t)dm.bc * dp * 2;

    AttnSmem& a = *(AttnSmem*)smem;
    uint8_t* stages = smem + ((sizeof(AttnSmem) + 127) & ~(size_t)127);
    const int S = st.attn_stages;

    auto issue = [&](int i) {
        const int s = i % S;
        const int blk = blk0 + i;
        const int rows = min(dm.bc, ctx - blk * dm.bc);
        const uint32_t bytes = (uint32_t)rows * dp * 2;
        const int id = table[blk];
        mbar_arrive_expect_tx(&a.full[s], 2 * bytes);
        bulk_load(stages + (size_t)s * 2 * blk_bytes, st.kpool + (size_t)id * dm.bc * dp, bytes, &a.full[s]);
        bulk_load(stages + (size_t)s * 2 * blk_bytes + blk_bytes, st.vpool + (size_t)id * dm.bc * dp, bytes,
                  &a.full[s]);
    };

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&a.full[s], 1);
        fence_barrier_init();
        for (int i = 0; i < min(S, n); ++i) issue(i);
    }
    // q (pre-scaled) for the chunks this lane owns in the K pass
    float qv[NJ][8];
    const float* q = st.q32 + (size_t)b * dp;
#pragma unroll
    for (int t = 0; t < NJ; ++t) {
        const int j = lane + 32 * t;
#pragma unroll
        for (int i = 0; i < 8; ++i) qv[t][i] = (j < nchunk) ? q[j * 8 + i] * st.attn_scale : 0.f;
    }
    __syncthreads();

    float m_run = -INFINITY, l_run = 0.f;
    float o[2][8];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) o[u][i] = 0.f;

    for (int i = 0; i < n; ++i) {
        const int s = i % S;
        const int rows = min(dm.bc, ctx - (blk0 + i) * dm.bc);
        mbar_wait(&a.full[s], (i / S) & 1);
        const uint4* sk = (const uint4*)(stages + (size_t)s * 2 * blk_bytes);
        const uint4* sv = (const uint4*)(stages + (size_t)s * 2 * blk_bytes + blk_bytes);
        for (int r = warp; r < rows; r += 4) {
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < NJ; ++t) {
                const int j = lane + 32 * t;
                if (j < nchunk) acc += dot8(sk[r * nchunk + j], qv[t]);
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) a.sc[r] = acc;
        }
        __syncthreads();
        float mloc = -INFINITY;
        for (int r = 0; r < rows; ++r) mloc = fmaxf(mloc, a.sc[r]);
        const float m_new = fmaxf(m_run, mloc);
        const float alpha = __expf(m_run - m_new);
        float psum = 0.f;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = tid + 128 * u;
            if (j < nchunk) {
#pragma unroll
                for (int e = 0; e < 8; ++e) o[u][e] *= alpha;
            }
        }
        for (int r = 0; r < rows; ++r) {
            const float p = __expf(a.sc[r] - m_new);
            psum += p;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int j = tid + 128 * u;
                if (j < nchunk) {
                    const uint4 vv = sv[r * nchunk + j];
                    const uint32_t w[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        o[u][2 * e] = fmaf(p, __uint_as_float(w[e] << 16), o[u][2 * e]);
                        o[u][2 * e + 1] = fmaf(p, __uint_as_float(w[e] & 0xFFFF0000u), o[u][2 * e + 1]);
                    }
                }
            }
        }
        l_run = l_run * alpha + psum;
        m_run = m_new;
        __syncthreads();  // stage s consumed
        if (tid == 0 && i + S < n) issue(i + S);
    }

    // ---- partial write + last-CTA combine (chunk order => deterministic) ----
    const size_t pbase = (size_t)b * st.attn_max_chunks;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int j = tid + 128 * u;
        if (j < nchunk) {
            float4* dst = (float4*)(st.attn_o + (pbase + c) * dp + j * 8);
            dst[0] = make_float4(o[u][0], o[u][1], o[u][2], o[u][3]);
            dst[1] = make_float4(o[u][4], o[u][5], o[u][6], o[u][7]);
        }
    }
    if (tid == 0) {
        st.attn_ml[(pbase + c) * 2 + 0] = m_run;
        st.attn_ml[(pbase + c) * 2 + 1] = l_run;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) a.last = (atomicAdd(&st.attn_cnt[b], 1) == nch - 1);
    __syncthreads();
    if (!a.last) return;
    __threadfence();
    float M = -INFINITY;
    for (int cc = 0; cc < nch; ++cc) M = fmaxf(M, __ldcg(&st.attn_ml[(pbase + cc) * 2]));
    float Ls = 0.f;
    for (int cc = 0; cc < nch; ++cc) Ls += __expf(__ldcg(&st.attn_ml[(pbase + cc) * 2]) - M) * __ldcg(&st.attn_ml[(pbase + cc) * 2 + 1]);
    const float inv = 1.f / Ls;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int j = tid + 128 * u;
        if (j >= nchunk) continue;
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        for (int cc = 0; cc < nch; ++cc) {
            const float w = __expf(__ldcg(&st.attn_ml[(pbase + cc) * 2]) - M);
            const float4* src = (const float4*)(st.attn_o + (pbase + cc) * dp + j * 8);
            const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
            acc[0] = fmaf(w, x0.x, acc[0]); acc[1] = fmaf(w, x0.y, acc[1]);
            acc[2] = fmaf(w, x0.z, acc[2]); acc[3] = fmaf(w, x0.w, acc[3]);
            acc[4] = fmaf(w, x1.x, acc[4]); acc[5] = fmaf(w, x1.y, acc[5]);
            acc[6] = fmaf(w, x1.z, acc[6]); acc[7] = fmaf(w, x1.w, acc[7]);
        }
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            pk[e] = (uint32_t)f32_to_bf16(acc[2 * e] * inv) | ((uint32_t)f32_to_bf16(acc[2 * e + 1] * inv) << 16);
        *(uint4*)(st.att_b + (size_t)b * dp + j * 8) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    if (tid == 0) st.attn_cnt[b] = 0;
}

int attn_smem_bytes(const Dims& dm, int stages) {
    return 256 + (int)((sizeof(AttnSmem) + 127) & ~(size_t)127) + stages * 2 * dm.bc * dm.dp * 2;
}

void launch_attention(const DevState& st, cudaStream_t s) {
    const int smem = attn_smem_bytes(st.dm, st.attn_stages);
    const int nj = (st.dm.dp / 8 + 31) / 32;
    dim3 grid(st.attn_max_chunks, st.rows.B);
#define EL_ATTN(NJV) attn_kernel<NJV><<<grid, 128, smem, s>>>(st)
    if (nj <= 1) EL_ATTN(1);
    else if (nj == 2) EL_ATTN(2);
    else if (nj == 3) EL_ATTN(3);
    else EL_ATTN(4);
#undef EL_ATTN
    EL_CUDA_LAUNCH_CHECK();
}

// ===========================================================================
// 3. Exit check + ExitStatusVector update (exit_policy.cpp:89-115,
//    engine.cpp:47-75). One CTA per row computes its confidence; the last CTA
//    OR-latches the status vector, records first accepts, advances the layer
//    and, when every row is set (or layer == L), ends the layer loop on the
//    device through the graph's WHILE condition.
// ===========================================================================
struct LmRed {
    float m1, m2, s;
    int idx;
};
__device__ __forceinline__ LmRed lm_merge(LmRed a, LmRed b) {
    // combine two disjoint vocab ranges; ties on the max keep the lowest index
    // (greedy_token, model.cpp:288-299) and make the gap 0 (exit_policy.cpp:62-71)
    const bool take_b = b.m1 > a.m1 || (b.m1 == a.m1 && b.idx < a.idx);
    const LmRed& hi = take_b ? b : a;
    const LmRed& lo = take_b ? a : b;
    LmRed r;
    r.m1 = hi.m1;
    r.idx = hi.idx;
    r.m2 = fmaxf(lo.m1, hi.m2);
    r.s = hi.s + (lo.m1 == -INFINITY ? 0.f : lo.s * __expf(lo.m1 - hi.m1));
    return r;
}

// fixed-shape tree over the Vp/128 tiles of column b (256 threads): deterministic
__device__ LmRed lm_reduce_col(const DevState& st, int b) {
    __shared__ LmRed red[256];
    const int tiles = st.dm.Vp / 128;
    const int tid = threadIdx.x;
    LmRed acc{-INFINITY, -INFINITY, 0.f, 0x7fffffff};
    for (int t = tid; t < tiles; t += 256) {
        const float4 p = __ldcg(&st.lm_part[(size_t)t * st.dm.Bmax + b]);
        acc = lm_merge(acc, LmRed{p.x, p.y, p.z, __float_as_int(p.w)});
    }
    red[tid] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (tid < w) red[tid] = lm_merge(red[tid], red[tid + w]);
        __syncthreads();
    }
    const LmRed r = red[0];
    __syncthreads();
    return r;
}

__device__ double block_sum_d(double v) {
    __shared__ double sh[32];
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    const int nw = blockDim.x >> 5;
    if (threadIdx.x == 0)
        for (int w = 0; w < nw; ++w) t += sh[w];
    __syncthreads();
    if (threadIdx.x == 0) sh[0] = t;
    __syncthreads();
    const double r = sh[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(256) exit_kernel(DevState st) {
    __shared__ int s_last;
    const int b = blockIdx.x, tid = threadIdx.x;
    const int layer = *st.layer;
    const int L = st.dm.L, dp = st.dm.dp, Bm = st.dm.Bmax;
    float conf = __int_as_float(0x7fc00000);  // NaN: not computed
    int acc = 0;
    switch (st.technique) {
        case kState: {
            const float* hi = st.h32 + ((size_t)((layer - 1) & 1) * Bm + b) * dp;
            const float* ho = st.h32 + ((size_t)(layer & 1) * Bm + b) * dp;
            double uv = 0, uu = 0, vv = 0;
            for (int i = tid; i < dp; i += blockDim.x) {
                const double x = hi[i], y = ho[i];
                uv += x * y; uu += x * x; vv += y * y;
            }
            uv = block_sum_d(uv); uu = block_sum_d(uu); vv = block_sum_d(vv);
            const double cd = uv / (sqrt(uu) * sqrt(vv));  // NaN on a zero-norm state
            conf = (float)cd;
            acc = cd > st.lambdas[layer - 1];
            break;
        }
        case kClassifier: {
            const float* ho = st.h32 + ((size_t)(layer & 1) * Bm + b) * dp;
            double z = 0;
            for (int i = tid; i < dp; i += blockDim.x) z += (double)st.probe_w[i] * ho[i];
            z = block_sum_d(z) + (double)st.probe_b;
            const double cd = 1.0 / (1.0 + exp(-z));
            conf = (float)cd;
            acc = cd > st.lambdas[layer - 1];
            break;
        }
        case kSoftmax: {
            const LmRed r = lm_reduce_col(st, b);
            // p1 - p2 = (1 - exp(l2 - l1)) / sum exp(l - l1)
            const float g = (r.m2 == -INFINITY) ? 1.f : -expm1f(r.m2 - r.m1);
            conf = g / r.s;
            acc = (double)conf > st.lambdas[layer - 1];
            break;
        }
        case kFixed: {
            conf = st.fixed_conf[(size_t)(layer - 1) * Bm + b];
            acc = (double)conf > st.lambdas[layer - 1];
            break;
        }
        case kAlwaysAt: acc = layer >= st.exit_layer; break;
        default: acc = 0; break;
    }
    if (tid == 0) {
        st.accept[b] = acc;
        st.conf[(size_t)(layer - 1) * Bm + b] = conf;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(st.exit_cnt, 1) == st.rows.B - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    int all = 1;
    for (int r = tid; r < st.rows.B; r += blockDim.x) {
        const int a = __ldcg(&st.accept[r]);
        int s = st.status[r];
        if (!s && a) {
            s = 1;
            st.status[r] = 1;
            st.first_accept[r] = layer;
        }
        all &= s;
    }
    all = __syncthreads_and(all);
    if (tid == 0) {
        const int done = all || layer >= L;
        if (done) *st.out_layer = layer;
        *st.layer = layer + 1;
        *st.exit_cnt = 0;
        if (st.use_cond) cudaGraphSetConditional(st.cond, done ? 0u : 1u);
        if (st.cont_host) *(volatile int*)st.cont_host = done ? 0 : 1;
    }
}

void launch_exit(const DevState& st, cudaStream_t s) {
    exit_kernel<<<st.rows.B, 256, 0, s>>>(st);
    EL_CUDA_LAUNCH_CHECK();
}

// ===========================================================================
// 4. embed (model.cpp:171-183) + iteration reset; finish (greedy token,
//    commit, records); prefill commit
// ===========================================================================
__global__ void embed_kernel(DevState st) {
    const int b = blockIdx.x;
    const int dp = st.dm.dp;
    const int tok = st.rows.tok[b];
    const uint16_t* e = st.emb + (size_t)tok * dp;
    float* h = st.h32 + (size_t)b * dp;
    uint16_t* hb = st.hb + (size_t)b * dp;
    for (int i = threadIdx.x; i < dp; i += blockDim.x) {
        const uint16_t x = e[i];
        hb[i] = x;
        h[i] = bf16_to_f32(x);
    }
    if (b == 0) {
        for (int r = threadIdx.x; r < st.dm.Bmax; r += blockDim.x) {
            st.status[r] = 0;
            st.first_accept[r] = 0;
        }
        if (threadIdx.x == 0) {
            *st.layer = 1;
            *st.out_layer = st.dm.L;
            *st.exit_cnt = 0;
            *st.cur_iter = (*st.iter_counter)++;
        }
    }
}
void launch_embed(const DevState& st, cudaStream_t s) {
    embed_kernel<<<st.rows.B, 128, 0, s>>>(st);
    EL_CUDA_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(256) finish_kernel(DevState st) {
    const int b = blockIdx.x, tid = threadIdx.x;
    const int L = st.dm.L, Bm = st.dm.Bmax;
    const LmRed r = lm_reduce_col(st, b);
    const int cur = *st.cur_iter % st.rec_cap;
    for (int l = tid; l < L; l += blockDim.x)
        st.rec_conf[((size_t)cur * L + l) * Bm + b] = st.conf[(size_t)l * Bm + b];
    if (tid == 0) {
        const int fa = st.first_accept[b];
        st.rec_tok[(size_t)cur * Bm + b] = r.idx;
        st.rec_acc[(size_t)cur * Bm + b] = fa ? fa : L;
        if (b == 0) st.rec_out[cur] = *st.out_layer;
        st.rows.tok[b] = r.idx;  // next input (engine.cpp:304)
        st.rows.pos[b] += 1;     // KvStore::commit (engine.cpp:262-264)
    }
}
void launch_finish(const DevState& st, cudaStream_t s) {
    finish_kernel<<<st.rows.B, 256, 0, s>>>(st);
    EL_CUDA_LAUNCH_CHECK();
}

__global__ void advance_kernel(DevState st) {
    const int b = threadIdx.x + blockIdx.x * blockDim.x;
    if (b < st.rows.B) st.rows.pos[b] += 1;
}
void launch_advance(const DevState& st, cudaStream_t s) {
    advance_kernel<<<(st.rows.B + 127) / 128, 128, 0, s>>>(st);
    EL_CUDA_LAUNCH_CHECK();
}

// ===========================================================================
// 5. setup kernels: seeded weights (model.cpp:37-59) and the seeded KV prefix
// ===========================================================================
__global__ void weightgen_kernel(uint16_t* out, int rows, int cols, int rows_p, int cols_p, uint64_t seed,
                                 double scale) {
    const size_t n = (size_t)rows_p * cols_p;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / cols_p), c = (int)(i % cols_p);
        uint16_t v = 0;
        if (r < rows && c < cols) v = bf16_bits_rne(seeded_value(seed, (uint64_t)r * cols + c, scale));
        out[i] = v;
    }
}
void launch_weightgen(uint16_t* out, int rows, int cols, int rows_p, int cols_p, uint64_t seed, double scale,
                      cudaStream_t s) {
    weightgen_kernel<<<148 * 8, 256, 0, s>>>(out, rows, cols, rows_p, cols_p, seed, scale);
    EL_CUDA_LAUNCH_CHECK();
}

// K/V of (seq, layer, pos) = seeded_vector(d, splitmix64_at(kv_seed, tag)),
// tag = ((seq * L + layer - 1) << 21 | pos) << 1 | kind; values bf16-rounded.
__global__ void kv_prefix_kernel(DevState st, const int* row_seq_ids, int prefix_len, uint64_t kv_seed,
                                 double scale) {
    const Dims& dm = st.dm;
    const int idx = blockIdx.x;  // (row, layer, pos)
    const int pos = idx % prefix_len;
    const int layer = (idx / prefix_len) % dm.L + 1;
    const int b = idx / (prefix_len * dm.L);
    const int seq = row_seq_ids[b];
    const int slot = st.rows.slot[b];
    const int blk = st.tables[((size_t)slot * dm.L + (layer - 1)) * dm.bpl_max + pos / dm.bc];
    const size_t off = ((size_t)blk * dm.bc + pos % dm.bc) * dm.dp;
    for (int kind = 0; kind < 2; ++kind) {
        const uint64_t tag =
            ((((uint64_t)seq * (uint64_t)dm.L + (uint64_t)(layer - 1)) << 21) | (uint64_t)pos) << 1 | (uint64_t)kind;
        const uint64_t vs = splitmix64_at(kv_seed, tag);
        uint16_t* dst = (kind == 0 ? st.kpool : st.vpool) + off;
        for (int i = threadIdx.x; i < dm.dp; i += blockDim.x)
            dst[i] = (i < dm.d) ? bf16_bits_rne(seeded_value(vs, (uint64_t)i, scale)) : (uint16_t)0;
    }
}
void launch_kv_prefix(const DevState& st, const int* row_seq_ids, int prefix_len, uint64_t kv_seed, int,
                      cudaStream_t s) {
    if (prefix_len <= 0 || st.rows.B <= 0) return;
    const double scale = 1.0 / sqrt((double)st.dm.d);
    kv_prefix_kernel<<<st.rows.B * st.dm.L * prefix_len, 128, 0, s>>>(st, row_seq_ids, prefix_len, kv_seed, scale);
    EL_CUDA_LAUNCH_CHECK();
}

// ===========================================================================
// 6. device LIFO block allocator (free list = stack, pops from the top)
// ===========================================================================
__global__ void kv_alloc_kernel(int* stack, int top, int* tables, int L, int bpl_max, int slot, int bpl) {
    const int n = L * bpl;
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x)
        tables[((size_t)slot * L + i / bpl) * bpl_max + i % bpl] = stack[top - 1 - i];
}
__global__ void kv_release_kernel(int* stack, int top, const int* tables, int L, int bpl_max, int slot, int bpl) {
    const int n = L * bpl;
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x)
        stack[top + i] = tables[((size_t)slot * L + i / bpl) * bpl_max + i % bpl];
}
void launch_kv_alloc(int* stack, int top, int* tables, const Dims& dm, int slot, int bpl, cudaStream_t s) {
    if (bpl <= 0) return;
    kv_alloc_kernel<<<(dm.L * bpl + 255) / 256, 256, 0, s>>>(stack, top, tables, dm.L, dm.bpl_max, slot, bpl);
    EL_CUDA_LAUNCH_CHECK();
}
void launch_kv_release(int* stack, int top, const int* tables, const Dims& dm, int slot, int bpl, cudaStream_t s) {
    if (bpl <= 0) return;
    kv_release_kernel<<<(dm.L * bpl + 255) / 256, 256, 0, s>>>(stack, top, tables, dm.L, dm.bpl_max, slot, bpl);
    EL_CUDA_LAUNCH_CHECK();
}

void init_kernel_attributes() {
    const int m = 227 * 1024;
    cudaFuncSetAttribute(gemm_kernel<kGemmQkv>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmWo>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmUp>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmDown>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmLmCheck>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmLmFinal>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmFill>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(attn_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(attn_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(attn_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(attn_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
}

}  // namespace el

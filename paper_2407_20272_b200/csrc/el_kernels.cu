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
#include <utility>

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

// launch with optional programmatic dependent launch (PDL)
template <typename... KArgs, typename... Args>
static void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, int smem, cudaStream_t s, bool pdl,
                     Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    EL_CUDA_LAUNCH_CHECK();
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// device-side kernel timeline (option dbg bit 64): slot = kind * 32 + layer,
// [2 * slot] = earliest CTA start, [2 * slot + 1] = latest CTA end
__device__ __forceinline__ void tl_mark(const DevState& st, int kind, int layer, int end) {
    if ((EL_DBG(st) & 64) && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        unsigned long long* slot = st.dbg_ts + 16384 + 2 * (kind * 32 + layer) + end;
        if (end) atomicMax(slot, t);
        else atomicMin(slot, t);
    }
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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

// LM-head partial over a vocab range: max, second max (with duplicates),
// sum exp(l - max), argmax (lowest index on ties)
struct LmPart {
    float m1, m2, s;
    int idx;
};
__device__ __forceinline__ LmPart lm_part_merge(LmPart a, LmPart b) {
    const bool take_b = b.m1 > a.m1 || (b.m1 == a.m1 && b.idx < a.idx);
    const LmPart& hi = take_b ? b : a;
    const LmPart& lo = take_b ? a : b;
    LmPart r;
    r.m1 = hi.m1;
    r.idx = hi.idx;
    r.m2 = fmaxf(lo.m1, hi.m2);
    r.s = hi.s + (lo.m1 == -INFINITY ? 0.f : lo.s * __expf(lo.m1 - hi.m1));
    return r;
}

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
        b_row = (layer - 1) & 1;
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
        b_row = eo & 1;
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

// --- T5 mode: static cross K/V of newly admitted sequences, K_c | V_c = W_kvc^(l) E^T
//     over their encoder states (column = row j * T + t of the encoder batch; rows.slot[j]
//     is sequence j's slot), written once into the sequence's cross blocks.
template <>
struct Epi<kGemmCross> {
    static constexpr bool kTile = false;
    __device__ static bool setup(const DevState& st, int tile, EpiSmem& e, int& a_row, int& b_row) {
        const int layer = *st.layer;
        e.layer = layer;
        e.row0 = tile * kBM;
        a_row = (layer - 1) * 2 * st.dm.dp + tile * kBM;
        b_row = 0;
        return true;
    }
    __device__ static void prologue(const DevState&, EpiSmem&) {}
    __device__ static void apply(const DevState& st, const EpiSmem& e, int row, int col, float v) {
        const Dims& dm = st.dm;
        const int m = e.row0 + row, kind = m >= dm.dp, f = m - kind * dm.dp;
        const int j = col / st.enc_len, t = col % st.enc_len;
        const int blk = st.ctables[((size_t)st.rows.slot[j] * dm.L + (e.layer - 1)) * st.enc_blocks + t / dm.bc];
        (kind ? st.cvpool : st.ckpool)[((size_t)blk * dm.bc + t % dm.bc) * dm.dp + f] = f32_to_bf16(v);
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
        st.mid_b[act_offset(col, e.row0 + row, st.NR)] = f32_to_bf16(o);
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
        st.up_b[act_offset(col, e.row0 + row, st.NR)] = f32_to_bf16(v > 0.f ? v : 0.f);
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
        st.h32[(size_t)e.par_out * st.dm.Bmax * dp + i] = o;
        st.hb[(size_t)e.par_out * (size_t)st.NR * dp + act_offset(col, e.row0 + row, st.NR)] = f32_to_bf16(o);
    }
};

// --- LM head with fused per-tile (max1, max2, sum exp, argmax) reduction:
//     logits never reach HBM (lm_head_logits + softmax_response_confidence /
//     greedy_token, exit_policy.cpp:57-72, model.cpp:288-299)
template <GemmKind K>
struct EpiLm {
    static constexpr bool kTile = true;
    static constexpr bool kFull = (K == kGemmLmCheck);  // softmax check needs max2 + sum exp; greedy only argmax
    __device__ static bool setup(const DevState& st, int tile, EpiSmem& e, int& a_row, int& b_row) {
        const int par = (K == kGemmLmCheck) ? (*st.layer & 1) : (*st.out_layer & 1);
        e.row0 = tile * kBM;
        a_row = tile * kBM;
        b_row = par;
        return true;
    }
    __device__ static void prologue(const DevState&, EpiSmem&) {}
    // sm: [n][129] logits of this tile (column n = batch row). R threads per
    // column scan disjoint row ranges in index order, then merge in a fixed
    // shuffle tree (lowest index wins ties).
    __device__ static void tile_reduce(const DevState& st, const EpiSmem& e, int tile, const float* sm) {
        const int nb = st.rows.B;
        const int rows = min(kBM, st.dm.V - e.row0);
        int R = 1;
        while (R < 32 && R * 2 * nb <= kBM) R *= 2;
        const int tid = threadIdx.x;
        for (int cbase = 0; cbase < nb; cbase += kBM / R) {
            const int n = cbase + tid / R, part = tid % R;
            const int r0 = part * (kBM / R), r1 = min(rows, r0 + kBM / R);
            float m1 = -INFINITY, m2 = -INFINITY, s = 0.f;
            int idx = 0x7fffffff;
            if (n < nb) {
                const float* col = sm + n * 129;
                for (int r = r0; r < r1; ++r) {
                    const float x = col[r];
                    if (x > m1) {
                        if (kFull) {
                            m2 = m1;
                            s = s * __expf(m1 - x) + 1.f;
                        }
                        m1 = x;
                        idx = e.row0 + r;
                    } else if (kFull) {
                        m2 = fmaxf(m2, x);
                        s += __expf(x - m1);
                    }
                }
            }
            LmPart p{m1, m2, s, idx};
            for (int off = 1; off < R; off <<= 1) {  // lanes of one column are consecutive
                LmPart q;
                q.m1 = __shfl_xor_sync(0xffffffffu, p.m1, off);
                q.m2 = __shfl_xor_sync(0xffffffffu, p.m2, off);
                q.s = __shfl_xor_sync(0xffffffffu, p.s, off);
                q.idx = __shfl_xor_sync(0xffffffffu, p.idx, off);
                p = (part & off) ? lm_part_merge(q, p) : lm_part_merge(p, q);
            }
            if (part == 0 && n < nb)
                st.lm_part[(size_t)tile * st.dm.Bmax + n] = make_float4(p.m1, p.m2, p.s, __int_as_float(p.idx));
        }
    }
};
template <>
struct Epi<kGemmLmCheck> : EpiLm<kGemmLmCheck> {};
template <>
struct Epi<kGemmLmFinal> : EpiLm<kGemmLmFinal> {};

// ExitStatusVector::observe_layer (engine.cpp:55-66) for this layer, run by one
// whole CTA once every row's decision is in st.accept: OR-latch, first accept,
// all-set; ends the layer loop on the device when all rows are set or layer == L.
__device__ void exit_latch(const DevState& st, int layer) {
    int all = 1;
    for (int r = threadIdx.x; r < st.rows.B; r += blockDim.x) {
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
    if (threadIdx.x == 0) {
        const int done = all || layer >= st.dm.L;
        if (done) *st.out_layer = layer;
        *st.layer = layer + 1;
        *st.exit_cnt = 0;
        if (st.use_cond) cudaGraphSetConditional(st.cond, done ? 0u : 1u);
        if (st.cont_host) *(volatile int*)st.cont_host = done ? 0 : 1;
    }
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

struct GemmArgs {
    const uint16_t* A;   // weights in tiled, pre-swizzled layout (tiled_offset)
    const uint16_t* Bp;  // activations in act_offset layout
    size_t b_par_stride;
    int NR;
    int m_tiles, splits, kb_total, n_pad, stages, tmem_cols, pdl;  // n_pad = columns per CTA (MMA N)
};

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Split-K runs as a thread-block cluster along K (grid.y = cluster.y = splits):
// every CTA parks its fp32 partial tile in its own shared memory, then each CTA
// reduces a disjoint set of output columns by reading the partials of all
// cluster peers over DSMEM in fixed rank order (deterministic, no global
// workspace, no atomics).  With PDL the weight (A) tiles are requested before
// griddepcontrol.wait: weights never depend on the previous kernel, so their
// HBM latency overlaps the producer kernel's tail.
template <GemmKind K>
__global__ void __launch_bounds__(128, 1)
    gemm_kernel(GemmArgs g, DevState st) {
    using E = Epi<K>;
    if constexpr (K == kGemmFill || K == kGemmLmFinal)  // the iteration's tail: skipped with the iteration
        if (st.run_active && *(volatile const int*)st.run_active == 0) return;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment by pointer offset (keeps the shared address space visible to the compiler)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tile = blockIdx.x, split = blockIdx.y;
    const int n0 = blockIdx.z * g.n_pad;  // N split: this CTA's first batch column
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    const uint32_t b_stage = (uint32_t)g.n_pad * kBK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)g.stages * kAStage;
    size_t region = (size_t)g.stages * (kAStage + b_stage);
    const size_t part_bytes = E::kTile ? (size_t)g.n_pad * 129 * 4 : (size_t)g.n_pad * kBM * 4;
    if ((E::kTile || g.splits > 1) && region < part_bytes) region = part_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + region);
    uint64_t* empty = full + g.stages;
    uint64_t* accf = empty + g.stages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
    EpiSmem& es = *reinterpret_cast<EpiSmem*>(smem + region + (2 * g.stages + 1) * 8 + 16);

    constexpr int tl_kind = K == kGemmQkv ? 1 : K == kGemmWo ? 3 : K == kGemmUp ? 4 : K == kGemmDown ? 5
                          : K == kGemmLmCheck ? 10 : K == kGemmLmFinal ? 8 : K == kGemmCross ? 12 : 7;
    const int tl_layer = (K == kGemmLmFinal || K == kGemmFill) ? 0 : *st.layer;
    tl_mark(st, tl_kind, tl_layer, 0);
    auto stamp = [&](int i) {
        if ((EL_DBG(st) & 8) && tid == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            st.dbg_ts[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + i] = t;
        }
    };
    stamp(0);
    int a_row = 0, b_row = 0;
    // setup() only reads layer / output-layer counters written before this
    // kernel's predecessor started (see el_kernels.h), so it may run pre-wait.
    pdl_trigger();  // single-wave grid: let the next kernel's prologue start now (no-op without a dependent)
    if (!E::setup(st, tile, es, a_row, b_row)) return;  // uniform across the CTA and its cluster
    const int kb0 = (int)((long)split * g.kb_total / g.splits);
    const int kb1 = (int)((long)(split + 1) * g.kb_total / g.splits);
    const int nkb = kb1 - kb0;

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
    stamp(1);

    if (warp == 0) {
        // ---- TMA producer: lane 0 drives the ring, the copies of ring slot s are issued by lanes
        //      1 + 2 (s % 15) and 2 + 2 (s % 15) (one thread's bulk copies run one after another) ----
        const int pre = min(nkb, g.stages);
        // weights: one contiguous 16 KB bulk copy per 128x64 tile (stored pre-swizzled)
        const uint16_t* a_tiles = g.A + (size_t)(a_row / kBM) * g.kb_total * (kBM * kBK);
        if (lane == 0)
            for (int kb = 0; kb < pre; ++kb) mbar_arrive_expect_tx(&full[kb], kAStage + b_stage);
        __syncwarp();
        for (int kb = 0; kb < pre; ++kb)  // weights first: independent of the previous kernel
            if (lane == (EL_LANE_ISSUE ? 1 + 2 * (kb % 15) : 0))
                bulk_load(sA + (size_t)kb * kAStage, a_tiles + (size_t)(kb0 + kb) * (kBM * kBK), kAStage, &full[kb]);
        // activations: the first n_pad rows of a k-block tile are contiguous
        const uint16_t* b_tiles = g.Bp + (size_t)b_row * g.b_par_stride;
        const size_t b_kstride = (size_t)g.NR * kBK;
        pdl_wait();  // no-op unless launched as a PDL secondary
        for (int kb = 0; kb < pre; ++kb)
            if (lane == (EL_LANE_ISSUE ? 2 + 2 * (kb % 15) : 0))
                bulk_load(sB + (size_t)kb * b_stage, b_tiles + (size_t)(kb0 + kb) * b_kstride + (size_t)n0 * kBK,
                          b_stage, &full[kb]);
        for (int kb = pre; kb < nkb; ++kb) {
            const int s = kb % g.stages;
            if (lane == 0) {
                mbar_wait(&empty[s], ((kb / g.stages) - 1) & 1);
                if ((EL_DBG(st) & 16) && blockIdx.x == 0 && blockIdx.y == 0 && kb < 64) {
                    unsigned long long t;
                    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
                    st.dbg_ts[4096 + 64 + kb] = t;
                }
                mbar_arrive_expect_tx(&full[s], kAStage + b_stage);
            }
            __syncwarp();
            if (lane == (EL_LANE_ISSUE ? 1 + 2 * (s % 15) : 0))
                bulk_load(sA + (size_t)s * kAStage, a_tiles + (size_t)(kb0 + kb) * (kBM * kBK), kAStage, &full[s]);
            if (lane == (EL_LANE_ISSUE ? 2 + 2 * (s % 15) : 0))
                bulk_load(sB + (size_t)s * b_stage, b_tiles + (size_t)(kb0 + kb) * b_kstride + (size_t)n0 * kBK,
                          b_stage, &full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer (single thread) ----
        const uint32_t idesc = idesc_bf16_m128((uint32_t)g.n_pad);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % g.stages;
            mbar_wait(&full[s], (kb / g.stages) & 1);
            if ((EL_DBG(st) & 16) && blockIdx.x == 0 && blockIdx.y == 0 && kb < 64) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
                st.dbg_ts[4096 + kb] = t;
            }
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
    pdl_wait();  // epilogue reads activations of earlier kernels

    // ---- epilogue: all four warps, thread t <-> TMEM lane t <-> output row t ----
    E::prologue(st, es);
    stamp(2);
    mbar_wait(accf, 0);
    tc_fence_after();
    __syncthreads();
    stamp(3);
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    const int nval = min(st.rows.B - n0, g.n_pad);  // valid columns of this CTA (>= 1 by construction)
    const int row = tid;

    if constexpr (E::kTile) {
        // splits == 1: transpose the tile through smem (stage buffers are free now)
        float* sm = reinterpret_cast<float*>(smem);
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
                if (c0 + j < nval) E::apply(st, es, row, n0 + c0 + j, v[j]);
        }
    } else {
        // partial tile [n][128] fp32: a warp's DSMEM loads below are 128 contiguous bytes
        float* part = reinterpret_cast<float*>(smem);
        for (int c0 = 0; c0 < nval; c0 += 16) {
            float v[16];
            tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) part[(c0 + j) * kBM + row] = v[j];
        }
        cluster_sync_all();
        stamp(4);
        // this CTA owns columns [c0, c1); all DSMEM loads of a column group are
        // issued before the (fixed rank order) sums so the latency overlaps
        const int per = (nval + g.splits - 1) / g.splits;
        const int c0 = split * per, c1 = min(nval, c0 + per);
        const float* peer[8];
#pragma unroll
        for (int s = 0; s < 8; ++s)
            peer[s] = (const float*)__cluster_map_shared_rank((void*)part, s < g.splits ? s : 0);
        for (int c = c0; c < c1; c += 4) {
            float v[4][8];
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int s = 0; s < 8; ++s)
                    v[j][s] = (s < g.splits && c + j < c1) ? peer[s][(c + j) * kBM + row] : 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (c + j >= c1) break;
                float acc = 0.f;
#pragma unroll
                for (int s = 0; s < 8; ++s)
                    if (s < g.splits) acc += v[j][s];
                E::apply(st, es, row, n0 + c + j, acc);
            }
        }
        stamp(5);
        cluster_sync_all();  // peers keep their smem alive until everyone has read it
    }
    if constexpr (K == kGemmDown) {
        if (st.fuse_exit) {
            // exit check fused into the down projection: per-tile partial dots of the
            // columns this CTA owns (fixed shuffle order), then the grid's last CTA
            // decides every row and latches the status vector
            const int layer = es.layer, Bm = st.dm.Bmax, dp = st.dm.dp;
            const int per = (nval + g.splits - 1) / g.splits;
            const int c0 = (g.splits > 1) ? split * per : 0;
            const int c1 = (g.splits > 1) ? min(nval, c0 + per) : nval;
            __syncthreads();  // this CTA's h32 writes are visible inside the CTA
            if (st.technique == kState || st.technique == kClassifier) {
                const float* ho = st.h32 + (size_t)(layer & 1) * Bm * dp;
                const float* hi = st.h32 + (size_t)((layer - 1) & 1) * Bm * dp;
                for (int cl = c0 + warp; cl < c1; cl += 4) {
                    const int c = n0 + cl;
                    double x0 = 0.0, x1 = 0.0, x2 = 0.0;
                    for (int m = lane; m < kBM; m += 32) {
                        const int f = es.row0 + m;
                        const double y = ho[(size_t)c * dp + f];
                        if (st.technique == kState) {
                            const double x = hi[(size_t)c * dp + f];
                            x0 += x * y;
                            x1 += x * x;
                            x2 += y * y;
                        } else {
                            x0 += (double)st.probe_w[f] * y;
                        }
                    }
                    x0 = warp_sum_d(x0);
                    x1 = warp_sum_d(x1);
                    x2 = warp_sum_d(x2);
                    if (lane == 0) {
                        double* p = st.exit_part + ((size_t)tile * Bm + c) * 3;
                        p[0] = x0;
                        p[1] = x1;
                        p[2] = x2;
                    }
                }
            }
            __syncthreads();
            if (tid == 0) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                es.last = atomicAdd(st.exit_cnt, 1) == (int)(gridDim.x * gridDim.y * gridDim.z) - 1;
            }
            __syncthreads();
            if (es.last) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                for (int r = tid; r < st.rows.B; r += blockDim.x) {
                    float conf = __int_as_float(0x7fc00000);
                    int acc = 0;
                    if (st.technique == kState || st.technique == kClassifier) {
                        double x0 = 0.0, x1 = 0.0, x2 = 0.0;
                        for (int t = 0; t < (int)gridDim.x; ++t) {  // fixed tile order
                            const double* p = st.exit_part + ((size_t)t * Bm + r) * 3;
                            x0 += __ldcg(p);
                            x1 += __ldcg(p + 1);
                            x2 += __ldcg(p + 2);
                        }
                        double cd;
                        if (st.technique == kState) cd = x0 / (sqrt(x1) * sqrt(x2));  // NaN on a zero-norm state
                        else cd = 1.0 / (1.0 + exp(-(x0 + (double)st.probe_b)));
                        conf = (float)cd;
                        acc = cd > st.lambdas[layer - 1];
                    } else if (st.technique == kFixed) {
                        conf = st.fixed_conf[(size_t)(layer - 1) * Bm + r];
                        acc = (double)conf > st.lambdas[layer - 1];
                    } else if (st.technique == kAlwaysAt) {
                        acc = layer >= st.exit_layer;
                    }
                    st.accept[r] = acc;
                    st.conf[(size_t)(layer - 1) * Bm + r] = conf;
                }
                __syncthreads();
                exit_latch(st, layer);
            }
        }
    }
    stamp(6);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, (uint32_t)g.tmem_cols);
    stamp(7);
    tl_mark(st, tl_kind, tl_layer, 1);
}

int gemm_smem_bytes(int n_pad, int stages, bool tile_reduce) {
    int main = stages * (kAStage + n_pad * kBK * 2);
    const int part = tile_reduce ? n_pad * 129 * 4 : n_pad * kBM * 4;  // split-K partial or LM tile
    main = main > part ? main : part;
    return 1024 + main + (2 * stages + 1) * 8 + 16 + (int)sizeof(EpiSmem) + 64;
}

template <GemmKind K>
static void launch_gemm_t(const GemmPlan& p, const DevState& st, cudaStream_t s, bool pdl) {
    GemmArgs g{p.A, p.Bp, p.b_par_stride, st.NR, p.m_tiles, p.splits, p.kb_total, p.n_pad, p.stages, p.tmem_cols,
               pdl ? 1 : 0};
    const int ns = (st.rows.B + p.n_pad - 1) / p.n_pad;  // N splits actually needed for this batch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.m_tiles, p.splits, ns);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (p.splits > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = 1;
        at[na].val.clusterDim.y = p.splits;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, gemm_kernel<K>, g, st);
    EL_CUDA_LAUNCH_CHECK();
}

void launch_gemm(GemmKind kind, const GemmPlan& p, const DevState& st, cudaStream_t s, bool pdl) {
    switch (kind) {
        case kGemmQkv: launch_gemm_t<kGemmQkv>(p, st, s, pdl); break;
        case kGemmWo: launch_gemm_t<kGemmWo>(p, st, s, pdl); break;
        case kGemmUp: launch_gemm_t<kGemmUp>(p, st, s, pdl); break;
        case kGemmDown: launch_gemm_t<kGemmDown>(p, st, s, pdl); break;
        case kGemmLmCheck: launch_gemm_t<kGemmLmCheck>(p, st, s, pdl); break;
        case kGemmLmFinal: launch_gemm_t<kGemmLmFinal>(p, st, s, pdl); break;
        case kGemmFill: launch_gemm_t<kGemmFill>(p, st, s, pdl); break;
        case kGemmCross: launch_gemm_t<kGemmCross>(p, st, s, pdl); break;
    }
}

// ===========================================================================
// 2. Paged decode attention over the block pool (model.cpp:223-243: scores = K q / sqrt(d),
//    softmax, P V; the multi-head extension splits d into heads, each with its own softmax).
// ===========================================================================
// The flattened (row, KV block) space of a pass is cut statically over the CTAs (cost-aware:
// a row start costs attn_seg_cost extra blocks), one segment per (CTA, row).  A producer warp
// streams the CTA's blocks (a block is bc x dp contiguous bf16 for K and for V, plus the row's
// q on a segment's first block) through a ring of shared-memory stages with 1-D bulk copies,
// running ahead across segment boundaries.  Eight consumer warps own two rows of every block
// each (processed together for ILP) and keep their own online-softmax state (m, l, o); a stage
// is released by 8 warp arrivals on its "empty" mbarrier, so the main loop has no CTA-wide
// barrier.  At a segment's end the warps merge in fixed order and publish an unnormalised
// partial (o, m, l); the last segment of a row to finish combines the partials in slot order
// (flash-decoding) into the bf16 attention output for the W_o GEMM.  The standalone kernel
// (attn_kernel) and the persistent / pipelined kernels' phases share this body.
constexpr int kAttnWarps = 8;
constexpr int kAttnThreads = (kAttnWarps + 1) * 32;

constexpr int kAttnPend = 256;  // >= rows: a CTA never has more segments than rows
constexpr int kAttnMaxHeads = 32;  // T5 mode: heads of d / n_heads features (head_dim 8..256)
constexpr int kAttnIds = 256;  // deferred segment completions per CTA before a forced settle
struct AttnDesc {
    int b, c, rows, first, last, nseg, pad[2];  // c = partial slot of this CTA's segment of sequence b
};
struct AttnSmem {
    uint64_t full[8];
    uint64_t empty[8];
    AttnDesc desc[8];
    float wm[kAttnWarps], wl[kAttnWarps];
    float wmh[kAttnWarps][kAttnMaxHeads], wlh[kAttnWarps][kAttnMaxHeads];  // multi-head (T5 mode) merge
    float cw[128];
    float cl[128];
    int pref[257];  // block prefix sum over the batch rows
    int pref_c[257];  // the same for the cross-attention (T5 mode) blocks: row b -> b * enc_blocks
    int last_flag;
    int seq_next;   // ring sequence base for the next pass
    int npend;      // segment partials published but not yet counted (see attn_settle)
    int pend_b[kAttnPend], pend_n[kAttnPend], pend_last[kAttnPend];
    // block ids of this CTA's static range, gathered before streaming (buffer 0: self
    // attention, 1: cross attention); the persistent kernel gathers the next layer's
    // at the end of a pass.  ids_layer / ids_g0: what a buffer holds (layer, range start)
    int ids[2][kAttnIds];
    int ids_layer[2], ids_g0[2];
};

// bf16 pair -> (lo, hi) fp32 pair
__device__ __forceinline__ float2 bf2_to_f2(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}
// acc += k . q over 8 bf16 features, as (even, odd) partial sums (packed FFMA2)
__device__ __forceinline__ float2 dot8p2(uint4 k, const float2* q, float2 acc) {
    acc = __ffma2_rn(bf2_to_f2(k.x), q[0], acc);
    acc = __ffma2_rn(bf2_to_f2(k.y), q[1], acc);
    acc = __ffma2_rn(bf2_to_f2(k.z), q[2], acc);
    return __ffma2_rn(bf2_to_f2(k.w), q[3], acc);
}
// o += p * v over 8 bf16 features (packed FFMA2)
__device__ __forceinline__ void axpy8p2(float p, uint4 v, float2* o) {
    const float2 pp = make_float2(p, p);
    o[0] = __ffma2_rn(pp, bf2_to_f2(v.x), o[0]);
    o[1] = __ffma2_rn(pp, bf2_to_f2(v.y), o[1]);
    o[2] = __ffma2_rn(pp, bf2_to_f2(v.z), o[2]);
    o[3] = __ffma2_rn(pp, bf2_to_f2(v.w), o[3]);
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// dbg 32: SM-clock stamps of the attention producer's start-up for CTAs 0..3 (slot k)
#define EL_ATT_CLK(k)                                                                       \
    do {                                                                                    \
        if ((EL_DBG(st) & 32) && blockIdx.x < 4) st.dbg_ts[8192 + 3072 + blockIdx.x * 16 + (k)] = clock64(); \
    } while (0)

// One attention pass over layer `layer` (see the comment above). Shared by the
// standalone kernel and the persistent iteration kernel; `seq0` continues the
// mbarrier ring's sequence (phase parity) across calls; on return a.seq_next
// holds the next base.
// What one attention pass reads: the self-attention pass streams the paged
// decoder KV (context pos + 1 per row); the T5-mode cross pass streams the
// static per-sequence encoder K/V (context = encoder length for every row).
struct AttnSrc {
    const int* tables;  // [slots][L][tstride] block ids
    int tstride;
    const uint16_t* kpool;
    const uint16_t* vpool;
    int ctx_fixed;      // > 0: every row attends over this many positions (no position written this pass)
    const int* pref;    // shared-memory block prefix sum over the rows
    const int* pos;     // rows' positions and KV slots (shared-memory copies in the persistent kernel)
    const int* slot;
    int idbuf;          // which a.ids buffer this pass uses (0 self, 1 cross)
    // gate != nullptr: the producer starts before the grid barrier that publishes this
    // layer's q and newest K/V rows; those loads wait until *gate reaches gate_target
    const unsigned* gate;
    unsigned gate_target;
    // work range (the pipelined kernel runs attention for one half of the batch on a subset of
    // the CTAs): rows [r0, r1) (r1 < 0: all rows), CTA cta of ncta (< 0: blockIdx.x / gridDim.x)
    int r0 = 0, r1 = -1, cta = -1, ncta = -1;
    // abort != nullptr: a speculative pass (the pipelined kernel's next-layer attention of the first
    // half) stops issuing blocks once *abort turns non-zero (the batch exited; its results are unused)
    const unsigned* abort = nullptr;
};

// attn_prefix_sum: the warp-parallel prefix sum of KV blocks per row into a.pref
// (rows.pos is constant for a whole decode iteration, so the persistent kernel
// computes it once per launch and passes persistent = true).
__device__ __forceinline__ void attn_prefix_sum(const DevState& st, AttnSmem& a) {
    const int lane = threadIdx.x & 31, B = st.rows.B, bc = st.dm.bc;
    int base = 0;
    for (int r0 = 0; r0 < B; r0 += 32) {
        const int r = r0 + lane;
        int v = (r < B) ? (st.rows.pos[r] + bc) / bc : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= off) v += t;
        }
        if (r < B) a.pref[r + 1] = base + v;
        base += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) a.pref[0] = 0;
    __syncwarp();
}

// Count the CTA's published segment partials (a.pend_*) and, for every sequence
// whose last segment this was, combine all its partials in slot order (flash-
// decoding) into the bf16 attention output.  Called by the 8 consumer warps
// together: at the end of the pass (so the fence + atomic round trip and the
// combine's L2 reads stay off the streaming loop) or when the list is full.
__device__ __forceinline__ void attn_settle(const DevState& st, AttnSmem& a) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int dp = st.dm.dp, nchunk = dp / 8;
    named_bar(1, kAttnWarps * 32);  // every partial store of this CTA is issued
    const int np = a.npend;
    if (np == 0) return;
    // one acq_rel atomic per pending sequence, all in flight together (lanes of warp 0);
    // release-cumulative over the CTA's partial stores ordered before it by bar.sync
    if (tid < np)
        a.pend_last[tid] = (atom_add_acq_rel(&st.attn_cnt[a.pend_b[tid]], 1) == a.pend_n[tid] - 1);
    named_bar(1, kAttnWarps * 32);
    for (int i = 0; i < np; ++i) {
        if (!a.pend_last[i]) continue;
        const int b = a.pend_b[i], nch = a.pend_n[i];
        const size_t pbase = (size_t)b * st.attn_max_chunks;
        if (st.attn_heads > 1) {  // multi-head: every feature chunk weights the partials by its head's (m, l)
            if (tid < nchunk) {
                const int H = st.attn_heads, h = tid * 8 / st.attn_hd;
                float Mg = -INFINITY;
                for (int cc = 0; cc < nch; ++cc) Mg = fmaxf(Mg, __ldcg(&st.attn_ml[((pbase + cc) * H + h) * 2]));
                float Lg = 0.f, acc[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] = 0.f;
                for (int cc = 0; cc < nch; ++cc) {  // fixed chunk order: deterministic
                    const float2 ml = __ldcg(reinterpret_cast<const float2*>(st.attn_ml) + (pbase + cc) * H + h);
                    const float w = __expf(ml.x - Mg);
                    Lg += w * ml.y;
                    const float4* src = reinterpret_cast<const float4*>(st.attn_o + (pbase + cc) * dp + tid * 8);
                    const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
                    acc[0] = fmaf(w, x0.x, acc[0]); acc[1] = fmaf(w, x0.y, acc[1]);
                    acc[2] = fmaf(w, x0.z, acc[2]); acc[3] = fmaf(w, x0.w, acc[3]);
                    acc[4] = fmaf(w, x1.x, acc[4]); acc[5] = fmaf(w, x1.y, acc[5]);
                    acc[6] = fmaf(w, x1.z, acc[6]); acc[7] = fmaf(w, x1.w, acc[7]);
                }
                const float inv = 1.f / Lg;
                uint32_t pk[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    pk[e] = (uint32_t)f32_to_bf16(acc[2 * e] * inv) | ((uint32_t)f32_to_bf16(acc[2 * e + 1] * inv) << 16);
                *reinterpret_cast<uint4*>(st.att_b + act_offset(b, tid * 8, st.NR)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
            if (tid == 0) st.attn_cnt[b] = 0;
            named_bar(1, kAttnWarps * 32);
            continue;
        }
        // the first partials' loads go out before the weights are known (one L2 round trip);
        // indices past nch are clamped to a valid partial and weighted 0 below
        constexpr int kPre = 4;
        const int j = tid < nchunk ? tid : nchunk - 1;
        float4 xp[kPre][2];
#pragma unroll
        for (int cc = 0; cc < kPre; ++cc) {
            const float4* src = reinterpret_cast<const float4*>(st.attn_o + (pbase + min(cc, nch - 1)) * dp + j * 8);
            xp[cc][0] = __ldcg(src);
            xp[cc][1] = __ldcg(src + 1);
        }
        float* cw = a.cw;  // per-chunk weights exp(m_c - M) / L, computed once
        if (warp == 0) {  // nch <= 128 (host guarantees)
            float mc[4], lc[4];
            float Mg = -INFINITY;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int cc = lane + 32 * u;
                mc[u] = -INFINITY;
                lc[u] = 0.f;
                if (cc < nch) {
                    const float2 ml = __ldcg(reinterpret_cast<const float2*>(st.attn_ml) + pbase + cc);
                    mc[u] = ml.x;
                    lc[u] = ml.y;
                }
                Mg = fmaxf(Mg, mc[u]);
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) Mg = fmaxf(Mg, __shfl_xor_sync(0xffffffffu, Mg, off));
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int cc = lane + 32 * u;
                if (cc < nch) {
                    cw[cc] = __expf(mc[u] - Mg);
                    a.cl[cc] = cw[cc] * lc[u];
                }
            }
            __syncwarp();
            float Lg = 0.f;  // fixed chunk order: deterministic
            for (int cc = 0; cc < nch; ++cc) Lg += a.cl[cc];
            const float inv = 1.f / Lg;
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (lane + 32 * u < nch) cw[lane + 32 * u] *= inv;
        }
        named_bar(1, kAttnWarps * 32);
        if (tid < nchunk) {  // (nchunk = dp / 8 <= 128 < 256 threads)
            float acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] = 0.f;
            auto fma8 = [&](float w, float4 x0, float4 x1) {
                acc[0] = fmaf(w, x0.x, acc[0]); acc[1] = fmaf(w, x0.y, acc[1]);
                acc[2] = fmaf(w, x0.z, acc[2]); acc[3] = fmaf(w, x0.w, acc[3]);
                acc[4] = fmaf(w, x1.x, acc[4]); acc[5] = fmaf(w, x1.y, acc[5]);
                acc[6] = fmaf(w, x1.z, acc[6]); acc[7] = fmaf(w, x1.w, acc[7]);
            };
#pragma unroll
            for (int cc = 0; cc < kPre; ++cc) fma8(cc < nch ? cw[cc] : 0.f, xp[cc][0], xp[cc][1]);
            for (int cc = kPre; cc < nch; ++cc) {
                const float4* src = reinterpret_cast<const float4*>(st.attn_o + (pbase + cc) * dp + j * 8);
                fma8(cw[cc], __ldcg(src), __ldcg(src + 1));
            }
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                pk[e] = (uint32_t)f32_to_bf16(acc[2 * e]) | ((uint32_t)f32_to_bf16(acc[2 * e + 1]) << 16);
            *reinterpret_cast<uint4*>(st.att_b + act_offset(b, j * 8, st.NR)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        if (tid == 0) st.attn_cnt[b] = 0;
        named_bar(1, kAttnWarps * 32);  // cw is rewritten by the next combine
    }
    if (tid == 0) a.npend = 0;
    named_bar(1, kAttnWarps * 32);
}

// The consumer warps of an attention pass (see attn_body); MH: the multi-head variant (extension,
// st.attn_heads > 1), a separate instantiation so the reference's single-head loop is unchanged.
template <int NJ, bool MH>
__device__ __forceinline__ void attn_consumer(const DevState& st, AttnSmem& a, uint8_t* stages, int seq0,
                                              bool persistent, float* mbuf) {
    const Dims& dm = st.dm;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int dp = dm.dp, nchunk = dp / 8;
    const int S = st.attn_stages;
    const uint32_t blk_bytes = (uint32_t)dm.bc * dp * 2;
    const uint32_t stage_bytes = (uint32_t)attn_stage_bytes(dm);  // K | V | q (>= merge buffer)
    // ---------------- consumer warps ----------------
    float2 q[NJ][4], o[NJ][4];  // this lane's features 8j..8j+7, j = lane + 32t, as pairs
#pragma unroll
    for (int t = 0; t < NJ; ++t)
#pragma unroll
        for (int i = 0; i < 4; ++i) q[t][i] = o[t][i] = make_float2(0.f, 0.f);
    float m = -INFINITY, l = 0.f;
    // multi-head (extension, MH): head of feature chunk j = j / cph, cph =
    // head_dim / 8 lanes of one chunk group t; every lane keeps its head's (m, l) per t
    const int heads = MH ? st.attn_heads : 1, cph = st.attn_hd >> 3;
    float mh[NJ], lh[NJ];
#pragma unroll
    for (int t = 0; t < NJ; ++t) mh[t] = -INFINITY, lh[t] = 0.f;
    int npend = 0;
    const int r0 = warp, r1 = warp + kAttnWarps;
    // Persistent kernel: the consumer path is cold in the instruction cache at
    // the start of every pass (the other phases' code evicted it), so the
    // first real block used to take ~4x a steady-state one.  Run the block
    // math once on whatever the first stage holds while its data is still in
    // flight (results are discarded: the first real descriptor of a pass is
    // always a segment start, which resets q, o, m, l).
    bool warm = persistent && !(EL_DBG(st) & (1 << 21));
    for (int seq = seq0;; ++seq) {
        const int s = seq % S;
        AttnDesc d;
        if (warm) {
            d = AttnDesc{0, 0, dm.bc, 0, 0, 1, {0, 0}};
        } else {
            mbar_wait(&a.full[s], (seq / S) & 1);
            d = a.desc[s];
        }
        if (d.b < 0) {  // terminal descriptor: release its slot too (the ring persists across passes)
            if (tid == 0) a.seq_next = seq + 1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&a.empty[s]);
        }
        if ((EL_DBG(st) & 32) && tid == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            if (blockIdx.x < 4 && seq < 60) st.dbg_ts[8192 + blockIdx.x * 128 + seq] = t;
            if (seq == 0) st.dbg_ts[24576 + 4 * blockIdx.x + 1] = t;
            st.dbg_ts[24576 + 4 * blockIdx.x + 2] = t;
        }
        if (d.b < 0) {
            if (tid == 0) EL_ATT_CLK(5);
            break;
        }
        if (tid == 0 && seq == seq0 && !warm) EL_ATT_CLK(4);
        uint8_t* sb = stages + (size_t)s * stage_bytes;
        const uint4* sk = reinterpret_cast<const uint4*>(sb);
        const uint4* sv = reinterpret_cast<const uint4*>(sb + blk_bytes);
        if (d.first) {
            const float2* qs = reinterpret_cast<const float2*>(sb + 2 * blk_bytes);
#pragma unroll
            for (int t = 0; t < NJ; ++t) {
                const int j = lane + 32 * t;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 x = qs[min(j, nchunk - 1) * 4 + i];
                    // features past dp (j >= nchunk) get q = 0: their (clamped) K loads add nothing
                    q[t][i] = (j < nchunk) ? make_float2(x.x * st.attn_scale, x.y * st.attn_scale)
                                           : make_float2(0.f, 0.f);
                    o[t][i] = make_float2(0.f, 0.f);
                }
            }
            m = -INFINITY;
            l = 0.f;
#pragma unroll
            for (int t = 0; t < NJ; ++t) mh[t] = -INFINITY, lh[t] = 0.f;
        }
        // Branch-free block math: both rows' K and V are loaded up front (row indices
        // clamped to valid rows, feature chunks clamped to the last one), an invalid
        // second row gets score -inf (weight 0 times finite data).
        const int nrows = (EL_DBG(st) & 1) ? 0 : d.rows;
        for (int rb = 0; rb < nrows; rb += 2 * kAttnWarps) {
            const int ra = rb + r0;
            if (ra >= nrows) break;  // warp-uniform: no row of this warp left in the block
            const bool vc = rb + r1 < nrows;
            const int rc = vc ? rb + r1 : ra;
            uint4 ka[NJ], kc[NJ], xa[NJ], xc[NJ];
#pragma unroll
            for (int t = 0; t < NJ; ++t) {
                const int j = min(lane + 32 * t, nchunk - 1);
                ka[t] = sk[ra * nchunk + j];
                kc[t] = sk[rc * nchunk + j];
            }
#pragma unroll
            for (int t = 0; t < NJ; ++t) {
                const int j = min(lane + 32 * t, nchunk - 1);
                xa[t] = sv[ra * nchunk + j];
                xc[t] = sv[rc * nchunk + j];
            }
            if constexpr (MH) {  // per-head scores, softmax state and rescale
                float sa[NJ], sc[NJ];
#pragma unroll
                for (int t = 0; t < NJ; ++t) {
                    const float2 x = dot8p2(ka[t], q[t], make_float2(0.f, 0.f));
                    const float2 y = dot8p2(kc[t], q[t], make_float2(0.f, 0.f));
                    sa[t] = x.x + x.y;
                    sc[t] = y.x + y.y;
                }
                for (int off = 1; off < cph; off <<= 1)
#pragma unroll
                    for (int t = 0; t < NJ; ++t) {
                        sa[t] += __shfl_xor_sync(0xffffffffu, sa[t], off);
                        sc[t] += __shfl_xor_sync(0xffffffffu, sc[t], off);
                    }
#pragma unroll
                for (int t = 0; t < NJ; ++t) {
                    if (!vc) sc[t] = -INFINITY;
                    const float mn = fmaxf(mh[t], fmaxf(sa[t], sc[t]));
                    const float pa = __expf(sa[t] - mn), pc = __expf(sc[t] - mn), alpha = __expf(mh[t] - mn);
                    const float2 al = make_float2(alpha, alpha);
                    lh[t] = lh[t] * alpha + (pa + pc);
#pragma unroll
                    for (int i = 0; i < 4; ++i) o[t][i] = __fmul2_rn(o[t][i], al);
                    axpy8p2(pa, xa[t], o[t]);
                    axpy8p2(pc, xc[t], o[t]);
                    mh[t] = mn;
                }
                continue;
            }
            float2 a2 = make_float2(0.f, 0.f), c2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int t = 0; t < NJ; ++t) {
                a2 = dot8p2(ka[t], q[t], a2);
                c2 = dot8p2(kc[t], q[t], c2);
            }
            float sa = a2.x + a2.y, sc = c2.x + c2.y;
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                sa += __shfl_xor_sync(0xffffffffu, sa, off);
                sc += __shfl_xor_sync(0xffffffffu, sc, off);
            }
            if (!vc) sc = -INFINITY;
            const float m_new = fmaxf(m, fmaxf(sa, sc));
            const float pa = __expf(sa - m_new), pc = __expf(sc - m_new);
            if (m_new != m) {  // warp-uniform
                const float alpha = __expf(m - m_new);
                const float2 al = make_float2(alpha, alpha);
                l *= alpha;
#pragma unroll
                for (int t = 0; t < NJ; ++t)
#pragma unroll
                    for (int i = 0; i < 4; ++i) o[t][i] = __fmul2_rn(o[t][i], al);
                m = m_new;
            }
            l += pa + pc;
#pragma unroll
            for (int t = 0; t < NJ; ++t) {
                axpy8p2(pa, xa[t], o[t]);
                axpy8p2(pc, xc[t], o[t]);
            }
        }
        if ((EL_DBG(st) & 32) && tid == 0 && blockIdx.x < 4 && seq < 60) {  // block processed (before release)
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            st.dbg_ts[8192 + 2048 + blockIdx.x * 128 + seq] = t;
        }
        if (warm) {  // dry run done: now the real first block of this stage
            warm = false;
            --seq;
            continue;
        }
        if (!d.last || (EL_DBG(st) & 4)) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&a.empty[s]);
            continue;
        }

        // ---- end of segment: merge the 8 warps in fixed order, publish the
        //      segment's partial (o, m, l) and queue its completion count ----
        float* merge = mbuf ? mbuf : reinterpret_cast<float*>(sb);  // [8][dp] fp32
        if (mbuf) {  // the stage is free as soon as this warp is done with it
            __syncwarp();
            if (lane == 0) mbar_arrive(&a.empty[s]);
        }
        named_bar(1, kAttnWarps * 32);  // (also: the previous merge's readers are done with mbuf / wm / wl)
        if constexpr (MH) {
#pragma unroll
            for (int t = 0; t < NJ; ++t) {
                const int j = lane + 32 * t;
                if (j < nchunk && j % cph == 0) {
                    a.wmh[warp][j / cph] = mh[t];
                    a.wlh[warp][j / cph] = lh[t];
                }
            }
        } else if (lane == 0) {
            a.wm[warp] = m;
            a.wl[warp] = l;
        }
#pragma unroll
        for (int t = 0; t < NJ; ++t) {
            const int j = lane + 32 * t;
            if (j < nchunk) {
                float4* dst = reinterpret_cast<float4*>(merge + (size_t)warp * dp + j * 8);
                dst[0] = make_float4(o[t][0].x, o[t][0].y, o[t][1].x, o[t][1].y);
                dst[1] = make_float4(o[t][2].x, o[t][2].y, o[t][3].x, o[t][3].y);
            }
        }
        named_bar(1, kAttnWarps * 32);
        if constexpr (MH) {  // per feature: its head's max / weights over the 8 warps (fixed order)
            const size_t pidx = (size_t)d.b * st.attn_max_chunks + d.c;
            const int hd = st.attn_hd;
            for (int i = tid; i < dp; i += kAttnWarps * 32) {
                const int h = i / hd;
                float M = -INFINITY;
#pragma unroll
                for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, a.wmh[w][h]);
                float acc = 0.f, Lsum = 0.f;
#pragma unroll
                for (int w = 0; w < kAttnWarps; ++w) {
                    const float sw = (a.wmh[w][h] == -INFINITY) ? 0.f : __expf(a.wmh[w][h] - M);
                    acc += sw * merge[(size_t)w * dp + i];
                    Lsum += sw * a.wlh[w][h];
                }
                st.attn_o[pidx * dp + i] = acc;
                if (i % hd == 0) {
                    st.attn_ml[(pidx * heads + h) * 2 + 0] = M;
                    st.attn_ml[(pidx * heads + h) * 2 + 1] = Lsum;
                }
            }
            if (tid == 0) {
                a.pend_b[a.npend] = d.b;
                a.pend_n[a.npend] = d.nseg;
                ++a.npend;
            }
            if (!mbuf) {
                named_bar(1, kAttnWarps * 32);
                if (lane == 0) mbar_arrive(&a.empty[s]);
            }
            ++npend;
            continue;
        }
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, a.wm[w]);
        float scw[kAttnWarps], Lsum = 0.f;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) {
            scw[w] = (a.wm[w] == -INFINITY) ? 0.f : __expf(a.wm[w] - M);
            Lsum += scw[w] * a.wl[w];
        }
        const size_t pidx = (size_t)d.b * st.attn_max_chunks + d.c;
        for (int i = tid; i < dp; i += kAttnWarps * 32) {
            float acc = 0.f;
#pragma unroll
            for (int w = 0; w < kAttnWarps; ++w) acc += scw[w] * merge[(size_t)w * dp + i];
            st.attn_o[pidx * dp + i] = acc;
        }
        if (tid == 0) {
            st.attn_ml[pidx * 2 + 0] = M;
            st.attn_ml[pidx * 2 + 1] = Lsum;
            a.pend_b[a.npend] = d.b;
            a.pend_n[a.npend] = d.nseg;
            ++a.npend;
        }
        if (!mbuf) {  // the merge lived in the stage: release it once every warp has read it
            named_bar(1, kAttnWarps * 32);
            if (lane == 0) mbar_arrive(&a.empty[s]);
        }
        if (EL_DEBUG && ((EL_DBG(st) & 8) || npend + 1 == kAttnPend)) {  // probe: settle every segment
            attn_settle(st, a);
            npend = 0;
        }
        ++npend;  // (<= rows <= kAttnPend: the list cannot overflow)
    }
    attn_settle(st, a);
    if (tid == 0) EL_ATT_CLK(6);
    pdl_trigger();
}

// persistent: called from the persistent kernel -- a.pref is already valid and
// no programmatic-dependent-launch deferral is needed (every input is ready).
template <int NJ, bool kAbort = false>  // kAbort: the pass may be stopped early (AttnSrc::abort)
__device__ __forceinline__ void attn_body(const DevState& st, AttnSmem& a, uint8_t* stages, int layer, int seq0,
                          bool persistent, const AttnSrc& src, float* mbuf) {
    const Dims& dm = st.dm;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int dp = dm.dp, nchunk = dp / 8;
    const int S = st.attn_stages;
    const uint32_t blk_bytes = (uint32_t)dm.bc * dp * 2;
    const uint32_t stage_bytes = (uint32_t)attn_stage_bytes(dm);  // K | V | q (>= merge buffer)
    if (warp == kAttnWarps) {
        // ---------------- producer warp ----------------
        // Static balanced split: the batch's KV blocks are flattened in (row,
        // block) order and CTA i streams [i*T/G, (i+1)*T/G) -- equal work per SM,
        // no queue, at most a few sequence segments per CTA.  Lane 0 drives the
        // ring; the warp fetches block ids in parallel.  Before
        // griddepcontrol.wait only K/V written by earlier iterations is
        // streamed; q and the block holding `pos` (written by this layer's QKV
        // kernel) are requested after it (one pending stage).
        const int B = st.rows.B;
        const int R0 = src.r0, R1 = src.r1 < 0 ? B : src.r1;  // rows of this pass
        const int CI = src.cta < 0 ? (int)blockIdx.x : src.cta, CN = src.ncta < 0 ? (int)gridDim.x : src.ncta;
        if (lane == 0) EL_ATT_CLK(1);
        if (!persistent) attn_prefix_sum(st, a);  // (standalone kernel: src.pref == a.pref)
        // Work split: the flattened (row, block) space of rows [R0, R1) -- blocks
        // [pref[R0], pref[R1]), relative index g in [0, T) -- is cut statically: CTA i streams
        // its share of [0, T) (with fewer blocks than CTAs only the first T CTAs work).
        // Partial slots per row: segments in CTA order -- the combine order never depends on
        // timing.  (int arithmetic: T <= 256 rows x 128 blocks, products <= T * 148 -- no 64-bit
        // division)
        const int gA = src.pref[R0];
        auto PR = [&](int r) { return (int)src.pref[r] - gA; };  // relative block prefix of row r
        const int T = PR(R1);
        const int Ts = T;
        if (lane == 0) EL_ATT_CLK(10);
        const int G = min(CN, Ts);
        // Cost-aware static split: every row start costs dl extra "virtual" blocks (a segment
        // switch + one more partial merge), so CTAs whose range crosses a row boundary get
        // fewer real blocks.  Virtual position of real block g of row r: g + dl * (r - R0 + 1);
        // CTA i owns virtual [floor(i V / G), floor((i + 1) V / G)).  Deterministic: depends
        // on the row structure only.
        const int dl = st.attn_seg_cost;
        const int V = Ts + dl * (R1 - R0);
        auto cta_of = [&](int g, int r) { return (int)(((g + dl * (r - R0 + 1) + 1) * G + V - 1) / V - 1); };
        auto real_of = [&](int vb) {  // first real block whose virtual position is >= vb
            if (vb >= V) return Ts;
            int lo = R0, hi = R1 - 1;  // first row whose virtual end exceeds vb
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (PR(mid + 1) + dl * (mid - R0 + 1) > vb) hi = mid;
                else lo = mid + 1;
            }
            return PR(lo) + max(0, vb - PR(lo) - dl * (lo - R0 + 1));
        };
        // segment bookkeeping of row r: its segments (CTA ranges) and the first CTA
        auto row_static = [&](int r, int& first_cta) {
            const int r0 = PR(r), r1 = min(PR(r + 1), Ts);
            if (r0 >= r1) return 0;
            first_cta = cta_of(r0, r);
            return cta_of(r1 - 1, r) - first_cta + 1;
        };
        // PDL secondary / gated early start: defer q and the newest block until the producer
        // kernel / the grid barrier has published them
        bool waited = persistent && src.gate == nullptr;
        int dq = -1, ds = -1, did = 0;
        uint32_t dbytes = 0;
        auto flush = [&]() {
            if (!waited) {
                if (src.gate) {
                    unsigned v;
                    const long long t0 = clock64();
                    for (;;) {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(src.gate) : "memory");
                        if ((int)(v - src.gate_target) >= 0) break;
                        if (clock64() - t0 > EL_SPIN_LIMIT) __trap();
                    }
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // bulk copies read them next
                } else {
                    pdl_wait();
                }
                waited = true;
            }
            if (ds >= 0) {
                uint8_t* sb = stages + (size_t)ds * stage_bytes;
                if (dq >= 0) bulk_load(sb + 2 * blk_bytes, st.q32 + (size_t)dq * dp, (uint32_t)dp * 4, &a.full[ds]);
                if (dbytes) {
                    bulk_load_ef(sb, src.kpool + (size_t)did * dm.bc * dp, dbytes, &a.full[ds]);
                    bulk_load_ef(sb + blk_bytes, src.vpool + (size_t)did * dm.bc * dp, dbytes, &a.full[ds]);
                }
                ds = -1;
                dq = -1;
                dbytes = 0;
            }
        };
        int seq = seq0;
        bool aborted = false;
        // stream blocks [g, seg_end) (absolute flattened indices) of row b as one segment
        // (partial slot `slot` of `nseg`); pid: the block ids of [g, seg_end) already in shared
        // memory (a.ids), or nullptr
        auto emit = [&](int b, int g, int seg_end, int slot, int nseg, const int* pid) {
            const int sb0 = src.pref[b], sb1 = src.pref[b + 1];
            const int nblk = (int)(sb1 - sb0);
            const int ctx = src.ctx_fixed > 0 ? src.ctx_fixed : src.pos[b] + 1;
            const int* table = src.tables + ((size_t)src.slot[b] * dm.L + (layer - 1)) * src.tstride;
            for (int gb = g; gb < seg_end; gb += 32) {
                const int blk_base = (int)(gb - sb0);
                const int nb = (int)min(32, seg_end - gb);
                const int my_id = (lane < nb) ? (pid ? pid[gb - g + lane] : table[blk_base + lane]) : 0;
                for (int u = 0; u < nb; ++u, ++seq) {
                    const int id = __shfl_sync(0xffffffffu, my_id, u);
                    const int blk = blk_base + u;
                    // 0: nothing for the issue lanes; bit 0: K|V of this block; bit 1: q too; -1: abort
                    int xgo = 0;
                    if (lane == 0) {
                        const int s = seq % S;
                        if (seq == seq0) EL_ATT_CLK(8);
                        unsigned fl = 0;
                        if (seq >= S) {
                            if constexpr (kAbort)
                                if (src.abort) fl = *(volatile const unsigned*)src.abort;  // (latency under the wait)
                            if (!waited) flush();  // the ring is full: release the deferred stage first
                            mbar_wait(&a.empty[s], ((seq / S) - 1) & 1);
                        }
                        if (kAbort && fl) {
                            xgo = -1;
                        } else {
                        if (seq == seq0) EL_ATT_CLK(9);
                        const int rows = min(dm.bc, ctx - blk * dm.bc);
                        const uint32_t bytes = (uint32_t)rows * dp * 2;
                        const bool first = (gb + u) == g, newest = blk == nblk - 1;
                        a.desc[s] = AttnDesc{b, slot, rows, first, (gb + u) == seg_end - 1, nseg, {0, 0}};
                        uint8_t* sbuf = stages + (size_t)s * stage_bytes;
                        if ((EL_DBG(st) & 32) && blockIdx.x < 4 && seq < 60) {  // issue time of each block
                            unsigned long long t;
                            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
                            st.dbg_ts[8192 + 1024 + blockIdx.x * 128 + seq] = t;
                        }
                        if (seq == seq0) EL_ATT_CLK(3);
                        mbar_arrive_expect_tx(&a.full[s], 2 * bytes + (first ? (uint32_t)dp * 4 : 0u));
                        if (!waited && (first || newest) && ds >= 0) flush();  // one pending stage at most
                        if (!waited && (first || newest)) {
                            ds = s;
                            dq = first ? b : -1;
                            if (newest) {
                                did = id;
                                dbytes = bytes;
                            } else {
                                xgo = 1;
                            }
                        } else {
                            xgo = first ? 3 : 1;
                        }
                        }  // (not aborted)
                    }
                    // The block's copies are issued by lanes other than 0, a different lane triple per
                    // ring slot: one thread's bulk copies are processed one after another (~0.4 us each
                    // from L2 / HBM whatever their size, scripts/ingest_probe*.cu), so a lone issuing
                    // lane caps a CTA at ~80 GB/s; copies of different lanes overlap.
                    xgo = __shfl_sync(0xffffffffu, xgo, 0);
                    __syncwarp();  // (orders lane 0's empty-slot acquire before the other lanes' copies)
                    if (kAbort && xgo < 0) {  // aborted: this block is not issued (seq stays its slot)
                        aborted = true;
                        break;
                    }
                    if (xgo) {
                        const int il = EL_LANE_ISSUE ? 1 + 3 * (seq % 10) : 0;  // lanes 1..30
                        const int s = seq % S;
                        const uint32_t sb = smem_u32(stages + (size_t)s * stage_bytes), fb = smem_u32(&a.full[s]);
                        const uint32_t bytes = (uint32_t)min(dm.bc, ctx - blk * dm.bc) * dp * 2;
                        if (lane == il)
                            bulk_load_hint(sb, src.kpool + (size_t)id * dm.bc * dp, bytes, fb, kL2EvictFirst);
                        if (lane == (EL_LANE_ISSUE ? il + 1 : 0))
                            bulk_load_hint(sb + blk_bytes, src.vpool + (size_t)id * dm.bc * dp, bytes, fb, kL2EvictFirst);
                        if (lane == (EL_LANE_ISSUE ? il + 2 : 0) && (xgo & 2))
                            bulk_load(stages + (size_t)s * stage_bytes + 2 * blk_bytes, st.q32 + (size_t)b * dp,
                                      (uint32_t)dp * 4, &a.full[s]);
                    }
                }
                __syncwarp();
                if (kAbort && aborted) break;
            }
        };
        // ---- this CTA's range ----
        const bool has_static = CI < G;
        const int g0 = gA + (has_static ? real_of(CI * V / G) : 0);  // absolute flattened range [g0, g1)
        const int g1 = gA + (has_static ? real_of((CI + 1) * V / G) : 0);
        // the range's block ids are gathered before streaming (independent loads in
        // parallel: a segment switch mid-range then costs no dependent table-load round
        // trip); the persistent kernel gathers the next layer's at the end of this pass
        const bool pre = has_static && g1 - g0 <= kAttnIds;
        const int ib = src.idbuf;
        auto gather = [&](int lay) {
            for (int g = g0 + lane; g < g1; g += 32) {
                int lo = R0, hi = R1 - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (src.pref[mid] <= g) lo = mid;
                    else hi = mid - 1;
                }
                a.ids[ib][g - g0] =
                    src.tables[((size_t)src.slot[lo] * dm.L + (lay - 1)) * src.tstride + (int)(g - src.pref[lo])];
            }
            __syncwarp();
            if (lane == 0) {
                a.ids_layer[ib] = lay;
                a.ids_g0[ib] = (int)g0;
            }
            __syncwarp();
        };
        if (lane == 0) EL_ATT_CLK(11);
        if (pre && !(a.ids_layer[ib] == layer && a.ids_g0[ib] == (int)g0)) gather(layer);
        if (has_static) {
            if (lane == 0) EL_ATT_CLK(2);
            int b = R0;
            {  // first row of the range: largest b with pref[b] <= g0 (binary search)
                int hi = R1 - 1;
                while (b < hi) {
                    const int mid = (b + hi + 1) >> 1;
                    if (src.pref[mid] <= g0) b = mid;
                    else hi = mid - 1;
                }
            }
            for (int g = g0; g < g1 && b < R1;) {
                const int seg_end = min(g1, (int)src.pref[b + 1]);
                int fc = 0;
                const int nseg = row_static(b, fc);
                emit(b, g, seg_end, CI - fc, nseg, pre ? a.ids[ib] + (g - g0) : nullptr);
                if (kAbort && aborted) break;
                g = seg_end;
                ++b;
            }
        }
        if (lane == 0) flush();  // short run: anything still deferred
        if (lane == 0) {
            const int s = seq % S;  // terminal descriptor
            if (seq >= S) mbar_wait(&a.empty[s], ((seq / S) - 1) & 1);
            a.desc[s].b = -1;
            mbar_arrive(&a.full[s]);
        }
        if (persistent && pre && layer < dm.L) gather(layer + 1);  // while the consumers finish
    } else if (st.attn_heads > 1) {
        attn_consumer<NJ, true>(st, a, stages, seq0, persistent, mbuf);
    } else {
        attn_consumer<NJ, false>(st, a, stages, seq0, persistent, mbuf);
    }
}

// The persistent kernel's attention pass: one out-of-line copy for the self and the
// cross pass (st points at the kernel's shared-memory copy of the parameters).
template <int NJ, bool kAbort = false>
__device__ __forceinline__ void attn_pass(const DevState& st, AttnSmem& a, uint8_t* stages, int layer, int seq0,
                                       const AttnSrc src, float* mbuf) {
    attn_body<NJ, kAbort>(st, a, stages, layer, seq0, true, src, mbuf);
}

template <int NJ>
__global__ void __launch_bounds__(kAttnThreads) attn_kernel(DevState st) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int tid = threadIdx.x;
    AttnSmem& a = *reinterpret_cast<AttnSmem*>(smem_raw);
    uint8_t* stages = smem_raw + ((sizeof(AttnSmem) + 127) & ~(size_t)127);
    const int layer = *st.layer;
    tl_mark(st, 2, layer, 0);
    if ((EL_DBG(st) & 32) && tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        if (blockIdx.x < 4) st.dbg_ts[8192 + 4 * 128 + blockIdx.x] = t;
        st.dbg_ts[24576 + 4 * blockIdx.x] = t;
    }
    if (tid == 0) {
        for (int s = 0; s < st.attn_stages; ++s) {
            mbar_init(&a.full[s], 1);
            mbar_init(&a.empty[s], kAttnWarps);
        }
        a.npend = 0;
        a.ids_layer[0] = a.ids_layer[1] = -1;
        fence_barrier_init();
    }
    __syncthreads();
    const AttnSrc src{st.tables, st.dm.bpl_max, st.kpool, st.vpool, 0, a.pref, st.rows.pos, st.rows.slot, 0, nullptr, 0u};
    attn_body<NJ>(st, a, stages, layer, 0, false, src, nullptr);
    if ((EL_DBG(st) & 32) && tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        st.dbg_ts[24576 + 4 * blockIdx.x + 3] = t;
    }
    tl_mark(st, 2, layer, 1);
}

int attn_smem_bytes(const Dims& dm, int stages) {
    return (int)((sizeof(AttnSmem) + 127) & ~(size_t)127) + stages * attn_stage_bytes(dm);
}

int attn_threads() { return kAttnThreads; }

void launch_attention(const DevState& st, cudaStream_t s, bool pdl) {
    const int smem = attn_smem_bytes(st.dm, st.attn_stages);
    const int nj = (st.dm.dp / 8 + 31) / 32;
    dim3 grid(st.attn_grid);
#define EL_ATTN(NJV) launch_k(attn_kernel<NJV>, grid, dim3(kAttnThreads), smem, s, pdl, st)
    if (nj <= 1) EL_ATTN(1);
    else if (nj == 2) EL_ATTN(2);
    else if (nj == 3) EL_ATTN(3);
    else EL_ATTN(4);
#undef EL_ATTN
}

int attn_ctas_per_sm(const Dims& dm, int stages) {
    int n = 0;
    const int smem = attn_smem_bytes(dm, stages);
    const int nj = (dm.dp / 8 + 31) / 32;
    cudaError_t e;
    if (nj <= 1) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, attn_kernel<1>, kAttnThreads, smem);
    else if (nj == 2) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, attn_kernel<2>, kAttnThreads, smem);
    else if (nj == 3) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, attn_kernel<3>, kAttnThreads, smem);
    else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, attn_kernel<4>, kAttnThreads, smem);
    return (e == cudaSuccess && n > 0) ? n : 1;
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
    pdl_wait();
    pdl_trigger();
    const int layer = *st.layer;
    tl_mark(st, 6, layer, 0);
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
    tl_mark(st, 6, layer, 1);
    if (!s_last) return;
    __threadfence();
    exit_latch(st, layer);
}

void launch_exit(const DevState& st, cudaStream_t s, bool pdl) {
    launch_k(exit_kernel, dim3(st.rows.B), dim3(256), 0, s, pdl, st);
}

// ===========================================================================
// 4. embed (model.cpp:171-183) + iteration reset; finish (greedy token,
//    commit, records); prefill commit
// ===========================================================================
__global__ void embed_kernel(DevState st) {
    const int b = blockIdx.x;
    if (st.run_active && *(volatile const int*)st.run_active == 0) {  // Engine::run chunk over: skip
        if (b == 0 && threadIdx.x == 0 && st.use_cond) cudaGraphSetConditional(st.cond, 0u);
        return;
    }
    tl_mark(st, 0, 0, 0);
    const int dp = st.dm.dp;
    const int tok = st.rows.tok[b];
    const uint16_t* e = st.emb + (size_t)tok * dp;
    float* h = st.h32 + (size_t)b * dp;
    for (int i = threadIdx.x; i < dp; i += blockDim.x) {
        const uint16_t x = e[i];
        st.hb[act_offset(b, i, st.NR)] = x;
        h[i] = bf16_to_f32(x);
    }
    tl_mark(st, 0, 0, 1);
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
// T5 mode: encoder state (seq id, t) = seeded_vector(d, splitmix64_at(enc_seed, id << 20 | t)),
// bf16-rounded (oracle/exitlab_oracle.c: eo_encoder_state), as GEMM B-operand rows j * T + t
__global__ void encoder_state_kernel(uint16_t* act, int NR, const int* ids, int T, int d, int dp, uint64_t enc_seed) {
    const int row = blockIdx.x, j = row / T, t = row % T;
    const uint64_t vs = splitmix64_at(enc_seed, ((uint64_t)ids[j] << 20) | (uint64_t)t);
    const double scale = 1.0 / sqrt((double)d);
    for (int i = threadIdx.x; i < dp; i += blockDim.x)
        act[act_offset(row, i, NR)] = (i < d) ? bf16_bits_rne(seeded_value(vs, (uint64_t)i, scale)) : (uint16_t)0;
}
// rows [0, n) of an act-layout buffer with NRs rows -> rows [row0, row0 + n) of one with NRd rows
__global__ void act_rows_copy_kernel(uint16_t* dst, int NRd, int row0, const uint16_t* src, int NRs, int dp) {
    const int b = blockIdx.x;
    for (int i = threadIdx.x * 8; i < dp; i += blockDim.x * 8)
        *reinterpret_cast<uint4*>(dst + act_offset(row0 + b, i, NRd)) =
            *reinterpret_cast<const uint4*>(src + act_offset(b, i, NRs));
}
void launch_act_rows_copy(uint16_t* dst, int NRd, int row0, const uint16_t* src, int NRs, int n, int dp,
                          cudaStream_t s) {
    if (n <= 0) return;
    act_rows_copy_kernel<<<n, 128, 0, s>>>(dst, NRd, row0, src, NRs, dp);
    EL_CUDA_LAUNCH_CHECK();
}

void launch_encoder_states(uint16_t* act, int NR, const int* ids, int n, int T, int d, int dp, uint64_t enc_seed,
                           cudaStream_t s) {
    if (n * T <= 0) return;
    encoder_state_kernel<<<n * T, 128, 0, s>>>(act, NR, ids, T, d, dp, enc_seed);
    EL_CUDA_LAUNCH_CHECK();
}

void launch_embed(const DevState& st, cudaStream_t s) {
    embed_kernel<<<st.rows.B, 128, 0, s>>>(st);
    EL_CUDA_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(256) finish_kernel(DevState st) {
    const int b = blockIdx.x, tid = threadIdx.x;
    pdl_wait();
    if (st.run_active && *(volatile const int*)st.run_active == 0) return;
    tl_mark(st, 9, 0, 0);
    const int L = st.dm.L, Bm = st.dm.Bmax;
    const LmRed r = lm_reduce_col(st, b);
    const int cur = *st.cur_iter % st.rec_cap;
    for (int l = tid; l < L; l += blockDim.x)
        rec_conf(st, cur)[(size_t)l * Bm + b] = st.conf[(size_t)l * Bm + b];
    if (tid == 0) {
        const int fa = st.first_accept[b];
        rec_rec(st, cur)[b] = r.idx;
        rec_rec(st, cur)[Bm + b] = fa ? fa : L;
        if (b == 0) rec_rec(st, cur)[2 * Bm] = *st.out_layer;
        st.rows.tok[b] = r.idx;  // next input (engine.cpp:304)
        st.rows.pos[b] += 1;     // KvStore::commit (engine.cpp:262-264)
    }
    tl_mark(st, 9, 0, 1);
}
void launch_finish(const DevState& st, cudaStream_t s, bool pdl) {
    launch_k(finish_kernel, dim3(st.rows.B), dim3(256), 0, s, pdl, st);
}

// first node of the layer body: a plain (non-cluster) kernel so the cluster GEMM
// that follows can be launched early through PDL
__global__ void layer_head_kernel(DevState st) {
    pdl_trigger();
    tl_mark(st, 11, *st.layer, 0);
    tl_mark(st, 11, *st.layer, 1);
}
void launch_layer_head(const DevState& st, cudaStream_t s) { launch_k(layer_head_kernel, dim3(1), dim3(32), 0, s, false, st); }

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
                                 double scale, int tiled) {
    const size_t n = (size_t)rows_p * cols_p;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / cols_p), c = (int)(i % cols_p);
        uint16_t v = 0;
        if (r < rows && c < cols) v = bf16_bits_rne(seeded_value(seed, (uint64_t)r * cols + c, scale));
        out[tiled ? tiled_offset(r, c, cols_p) : i] = v;
    }
}
void launch_weightgen(uint16_t* out, int rows, int cols, int rows_p, int cols_p, uint64_t seed, double scale,
                      int tiled, cudaStream_t s) {
    weightgen_kernel<<<148 * 8, 256, 0, s>>>(out, rows, cols, rows_p, cols_p, seed, scale, tiled);
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
    cudaFuncSetAttribute(gemm_kernel<kGemmQkv>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(gemm_kernel<kGemmWo>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(gemm_kernel<kGemmUp>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(gemm_kernel<kGemmDown>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(gemm_kernel<kGemmFill>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(gemm_kernel<kGemmWo>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmUp>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmDown>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmLmCheck>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmLmFinal>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmFill>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmCross>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(gemm_kernel<kGemmCross>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(attn_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(attn_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(attn_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(attn_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
}

// ---- Engine::run between scheduling events (engine.cpp:266-305 on the device) ----
__global__ void __launch_bounds__(256) run_step_kernel(DevState st, RunCtl c) {
    if (*(volatile const int*)c.active == 0) return;
    const int B = st.rows.B, tid = threadIdx.x;
    int fin = 0;
    for (int b = tid; b < B; b += blockDim.x) {
        const int r = c.rem[b] - 1;
        c.rem[b] = r;
        const int tok = st.rows.tok[b];  // the token this iteration emitted (the next input)
        fin |= (r <= 0) || (c.eos >= 0 && tok == c.eos);
    }
    fin = __syncthreads_or(fin);
    if (tid == 0) {
        // charge = e (c_fixed + c_seq B) + e B c_check + (L - e) B c_fill, in the host's (the
        // reference's) operation order, every product and sum rounded on its own (no FMA)
        const int e = *st.out_layer;
        const double t1 = __dmul_rn((double)e, __dadd_rn(c.c_fixed, __dmul_rn(c.c_seq, (double)B)));
        const double t2 = __dmul_rn((double)(e * B), c.c_check);
        const double t3 = __dmul_rn(__dmul_rn((double)(c.L - e), (double)B), c.c_fill);
        const double charge = __dadd_rn(__dadd_rn(t1, t2), t3);
        const double clock = __dadd_rn(*c.clock, charge);
        *c.clock = clock;
        const int cur = *st.cur_iter % st.rec_cap;
        c.log[2 * cur] = clock;
        c.log[2 * cur + 1] = charge;
        *c.done += 1;
        if (fin || c.next_arrival <= clock) *c.active = 0;  // a finish or an admission: back to the host
    }
}
void launch_run_step(const DevState& st, const RunCtl& c, cudaStream_t s) {
    run_step_kernel<<<1, 256, 0, s>>>(st, c);
    EL_CUDA_LAUNCH_CHECK();
}

#include "el_iter.cuh"
#include "el_pipe.cuh"

}  // namespace el

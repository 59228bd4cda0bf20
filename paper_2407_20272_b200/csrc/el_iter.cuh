// el_iter.cuh -- the persistent decode-iteration kernel: ONE launch per decode
// iteration (engine.cpp:208-310, Algorithm 1).  Included by el_kernels.cu
// inside namespace el (reuses the tcgen05 / bulk-copy primitives and the paged
// attention body).
//
// One CTA per SM (cooperative launch, co-residency guaranteed), 9 warps:
// warps 0-7 compute (epilogues, attention consumers, reductions), warp 8 is the
// bulk-copy producer.  TMEM (512 columns) is allocated once per launch.  The
// layer loop runs on the device; phases are separated by a grid barrier:
//
//   embed | { QKV-partial | QKV-reduce(+paged K/V append) | attention |
//             Wo-partial | Wo-reduce(+residual) | Up-partial | Up-reduce(+ReLU) |
//             Down-partial | Down-reduce(+residual, exit dot partials) |
//             [LM-check | softmax decide] | exit latch }*  |
//   LM-final + skipped-layer fill partials | fill-reduce(+paged K/V) + greedy finish
//
// GEMMs are weight-streaming split-K (swap-AB: weights are the M=128 operand,
// the batch is N): unit (m-tile, k-split) accumulates in TMEM, its fp32
// partial goes to an L2-resident workspace, and the reduce phase sums the
// splits in fixed order (deterministic, no atomics) and runs the fused
// epilogue, spread over every warp of the grid.  The exit decision is computed
// redundantly (and identically) by every CTA from the per-tile partial dots, so
// the "all rows exited" test needs no extra barrier and no host round trip.

constexpr int kIterWarps = 9;
constexpr int kIterThreads = kIterWarps * 32;
constexpr int kProducerWarp = 8;


struct IterSmem {
    AttnSmem att;  // attention ring barriers/descriptors (persist across layers)
    uint64_t full[8], empty[8], acc;
    uint64_t full2[16], empty2[16];  // batch-M GEMM activation ring
    uint64_t full3[4], empty3[4];    // pipelined kernel: LM pair units of the softmax check (lm_stages)
    uint64_t wfull;                  // batch-M unit weights (one tensor copy per unit)
    unsigned long long tdbg[5];
    uint32_t tmem;
    int pad0;
    int pos[256], slot[256], status[256], first[256];
    int kvrow[256];  // per row: slot * L * bpl_max + pos / bc (block-table index at layer 1)
    int kvin[256];   // per row: (pos % bc) * dp (element offset of the position inside its block)
    long long kvd[256];  // fill epilogue: per row, the K/V element offset of its position at the unit's layer
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel_u32(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_release_add_u32(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid barrier over co-resident CTAs.  Generic global writes before it are
// visible (and ordered for the async proxy: bulk copies read them) to every
// CTA after it.  bar layout (unsigned): [0] arrivals, [1024] generation; both only
// ever grow (wrap-safe signed distances against the values read at launch start,
// gb.y / gb.x), so nothing is reset between launches.
// Every CTA adds its arrival with red.release and polls the arrival count itself
// (one L2 hop from the last arrival to every waiter): +2-5 % end to end over the
// two-hop form (dbg bit 25: CTA 0 alone polls the count and releases a generation
// word the others poll).  Inlined, with no reference to a copy of the parameters.
__device__ __forceinline__ void grid_sync(const IterPlan& p, const DevState& st, int& nbar, uint2 gb) {
    const int dbg = EL_DBG(st);
    if (threadIdx.x == 0 && (dbg & 128) && nbar < 1024) {  // per-CTA arrival (work done) time
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        st.dbg_ts[65536 + (size_t)blockIdx.x * 1024 + nbar] = t;
    }
    fence_proxy_async_global();
    __syncthreads();
    const unsigned k = (unsigned)nbar + 1u;  // barrier index within this launch (1-based)
    if (threadIdx.x == 0) {
        unsigned* cnt = p.bar;
        unsigned* gen = p.bar + 1024;
        const unsigned target = gb.y + gridDim.x * k;
        red_release_add_u32(cnt, 1u);
        const long long t0 = clock64();
        if (!(dbg & (1 << 25))) {
            while ((int)(ld_acquire_u32(cnt) - target) < 0)
                if (clock64() - t0 > EL_SPIN_LIMIT) __trap();
        } else if (blockIdx.x == 0) {
            while ((int)(ld_acquire_u32(cnt) - target) < 0)
                if (clock64() - t0 > EL_SPIN_LIMIT) __trap();
            st_release_u32(gen, gb.x + k);
        } else {
            while ((int)(ld_acquire_u32(gen) - (gb.x + k)) < 0)
                if (clock64() - t0 > EL_SPIN_LIMIT) __trap();
        }
        if ((dbg & 128) && blockIdx.x == 0 && nbar < 1024) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            st.dbg_ts[20480 + nbar] = t;
        }
    }
    ++nbar;
    __syncthreads();
    fence_proxy_async_global();
}

// The same barrier for warps 0-7 only (named barrier 2): the producer warp skips it and
// starts the next attention pass, whose q / newest-block loads wait on the count.
__device__ __forceinline__ void grid_sync_sub(const IterPlan& p, const DevState& st, int& nbar, uint2 gb) {
    fence_proxy_async_global();
    asm volatile("bar.sync 2, 256;" ::: "memory");
    const unsigned k = (unsigned)nbar + 1u;
    if (threadIdx.x == 0) {
        unsigned* cnt = p.bar;
        const unsigned target = gb.y + gridDim.x * k;
        red_release_add_u32(cnt, 1u);
        const long long t0 = clock64();
        while ((int)(ld_acquire_u32(cnt) - target) < 0)
            if (clock64() - t0 > EL_SPIN_LIMIT) __trap();
        if ((EL_DBG(st) & 128) && blockIdx.x == 0 && nbar < 1024) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            st.dbg_ts[20480 + nbar] = t;
        }
    }
    ++nbar;
    asm volatile("bar.sync 2, 256;" ::: "memory");
}

// ---------------------------------------------------------------------------
// GEMM unit: TMEM[0, n_pad) = sum_{kb in [kb0, kb0+nkb)} W_tile(kb) . X_tile(kb)^T
// producer = warp 8 lane 0, MMA issuer = warp 0 lane 0.  On return the
// accumulator is complete and visible to warps 0-7.
// ---------------------------------------------------------------------------
struct RingDesc {
    uint64_t* full;
    uint64_t* empty;
    uint32_t stages, stride, b_off;  // stage count, stage stride, offset of the B region in a stage
};

// The caller advances kseq by nkb.
__device__ __forceinline__ void unit_mainloop(IterSmem& sm, uint8_t* ring, const RingDesc r, const uint32_t kseq,
                                              const uint16_t* a_src, uint32_t a_bytes, size_t a_kstride,
                                              const uint16_t* b_src, uint32_t b_bytes, size_t b_kstride, int kb0,
                                              int nkb, uint32_t n_mma, uint32_t useq, uint64_t a_policy,
                                              uint64_t b_policy, int dbg = 0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // single-thread issue loops: stage index / phase / addresses are strength-reduced (no div/mod per
    // k-block -- a lone thread cannot hide the latency of that arithmetic)
    if (warp == kProducerWarp) {
        // lane 0 drives the ring; the two copies of ring slot s are issued by lanes 1 + 2 (s % 15) and
        // 2 + 2 (s % 15): one thread's bulk copies are processed one after another (~0.4 us each,
        // scripts/ingest_probe*.cu), copies of different lanes overlap
        uint32_t s = kseq % r.stages, ph = (kseq / r.stages) & 1;
        bool wrapped = kseq >= r.stages;
        const uint32_t ring0 = smem_u32(ring), full0 = smem_u32(r.full), empty0 = smem_u32(r.empty);
        const uint8_t* ap = reinterpret_cast<const uint8_t*>(a_src + (size_t)kb0 * a_kstride);
        const uint8_t* bp = reinterpret_cast<const uint8_t*>(b_src + (size_t)kb0 * b_kstride);
        const size_t ast = a_kstride * 2, bst = b_kstride * 2;
        const uint32_t tx = a_bytes + b_bytes;
#pragma unroll 1
        for (int i = 0; i < nkb; ++i) {
            const uint32_t fb = full0 + 8 * s, sb = ring0 + s * r.stride;
            if (lane == 0) {
                if (wrapped) mbar_wait_addr(empty0 + 8 * s, ph ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(tx) : "memory");
            }
            __syncwarp();
            const int il = EL_LANE_ISSUE ? 1 + 2 * (int)(s % 15u) : 0;
            if (lane == il) bulk_load_hint(sb, ap, a_bytes, fb, a_policy);
            if (lane == (EL_LANE_ISSUE ? il + 1 : 0)) bulk_load_hint(sb + r.b_off, bp, b_bytes, fb, b_policy);
            ap += ast;
            bp += bst;
            if (++s == r.stages) {
                s = 0;
                ph ^= 1;
                wrapped = true;
            }
        }
        if (lane == 0 && (dbg & 64)) sm.tdbg[3] = clock64();
    } else if (warp == 0) {
        {  // whole warp 0, one elected lane issues (uniform descriptors)
            const uint32_t idesc = idesc_bf16_m128(n_mma);
            uint32_t s = kseq % r.stages, ph = (kseq / r.stages) & 1;
            const uint32_t full0 = smem_u32(r.full), ring0 = smem_u32(ring);
#pragma unroll 1
            for (int i = 0; i < nkb; ++i) {
                mbar_wait_addr(full0 + 8 * s, ph);
                if (lane == 0 && (dbg & 64) && (i == 0 || i == nkb - 1)) sm.tdbg[i == 0 ? 0 : 1] = clock64();
                tc_fence_after();
                // (descriptors rebuilt per stage: the 14-bit address field wraps modulo 256 KB)
                const uint32_t sa = ring0 + s * r.stride;
                const uint64_t ad = sdesc_k_sw128(sa), bd = sdesc_k_sw128(sa + r.b_off);
                if (!(dbg & (1 << 18)))
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        tc_mma_bf16_warp(sm.tmem, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (i | k) != 0);
                tc_commit_warp(&r.empty[s]);
                if (++s == r.stages) {
                    s = 0;
                    ph ^= 1;
                }
            }
            tc_commit_warp(&sm.acc);
        }
    }
    __syncwarp();
    if (warp < 8) {
        mbar_wait(&sm.acc, useq & 1);
        tc_fence_after();
    }
}
// weight-streaming unit (swap-AB): weights = A (16 KB tile per k-block), activations = B (n_rows
// rows, default n_pad; the ring stage always has room for n_pad)
__device__ __forceinline__ void unit_ws(IterSmem& sm, uint8_t* ring, const IterPlan& p, uint32_t& kseq,
                                        const uint16_t* a_row, const uint16_t* b_src, size_t b_kstride, int kb0,
                                        int nkb, uint32_t useq, int dbg = 0, int n_rows = 0,
                                        uint64_t a_policy = kL2EvictFirst) {
    const RingDesc r{sm.full, sm.empty, (uint32_t)p.stages, (uint32_t)p.stage_bytes, (uint32_t)kAStage};
    const uint32_t n = (uint32_t)(n_rows > 0 ? n_rows : p.n_pad);
    unit_mainloop(sm, ring, r, kseq, a_row, kAStage, (size_t)(kBM * kBK), b_src, n * 128u, b_kstride,
                  kb0, nkb, n, useq, a_policy, kL2EvictLast, dbg);
    kseq += (uint32_t)nkb;
}

// LM-head pair unit (softmax checks): vocab tiles t0 and t0 + 1 (na = 2, or 1 for an odd last
// tile) against one activation stream -- stage = A0 16 KB | A1 16 KB | B (n_pad rows), two MMAs
// per k-step into TMEM columns [0, n) and [256, 256 + n).  One wave of (Vp / 128 + 1) / 2 units
// instead of two of Vp / 128 single tiles, and each CTA reads the activations once per two
// tiles.  Same barriers / stage count as the weight-streaming ring (stride 32 KB + n_pad * 128).
__device__ __forceinline__ void unit_lm_pair(IterSmem& sm, uint8_t* ring, const IterPlan& p, uint32_t& kseq,
                                             const uint16_t* a0, int na, const uint16_t* b_src, size_t b_kstride,
                                             int nkb, uint32_t useq, uint64_t a_policy, bool tr = false,
                                             int dbg = 0, uint64_t* rfull = nullptr, uint64_t* rempty = nullptr,
                                             int rstages = 0) {
    // ring: the weight-streaming ring's barriers and depth, or (rfull) a separate set
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // tr at batch 256: one vocab tile (na = 1) against both 128-row groups (two M128 x N128 MMAs)
    const bool two_rg = tr && p.n_pad == 256;
    const uint32_t b_bytes = (uint32_t)p.n_pad * 128u, a_bytes = (uint32_t)kAStage;
    const uint32_t boff = (two_rg ? 1u : 2u) * a_bytes;  // B region: after the weight tile(s)
    const uint32_t stages = (uint32_t)(rfull ? rstages : p.stages), stride = boff + b_bytes;
    uint64_t* const fullb = rfull ? rfull : sm.full;
    uint64_t* const emptyb = rfull ? rempty : sm.empty;
    const size_t tile_elems = (size_t)nkb * (kBM * kBK);
    if (warp == kProducerWarp) {
        uint32_t s = kseq % stages, ph = (kseq / stages) & 1;
        bool wrapped = kseq >= stages;
        const uint32_t ring0 = smem_u32(ring), full0 = smem_u32(fullb), empty0 = smem_u32(emptyb);
        const uint32_t tx = (uint32_t)na * a_bytes + b_bytes;
#pragma unroll 1
        for (int i = 0; i < nkb; ++i) {
            const uint32_t fb = full0 + 8 * s, sb = ring0 + s * stride;
            if (lane == 0) {
                if (wrapped) mbar_wait_addr(empty0 + 8 * s, ph ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(tx) : "memory");
            }
            __syncwarp();
            // three copies from three lanes (one thread's bulk copies are processed serially)
            if (lane == 0) bulk_load_hint(sb, a0 + (size_t)i * (kBM * kBK), a_bytes, fb, a_policy);
            if (lane == 1 && na > 1) bulk_load_hint(sb + a_bytes, a0 + tile_elems + (size_t)i * (kBM * kBK), a_bytes, fb, a_policy);
            if (lane == 2) bulk_load_hint(sb + boff, b_src + (size_t)i * b_kstride, b_bytes, fb, kL2EvictLast);
            if (++s == stages) {
                s = 0;
                ph ^= 1;
                wrapped = true;
            }
        }
        if (lane == 0 && (dbg & 64)) sm.tdbg[3] = clock64();
    } else if (warp == 0) {
        // tr: D^T = X . W^T -- M = the 128 batch rows (TMEM lanes), N = the 256 vocab rows of both
        // tiles (their k-blocks are adjacent in the stage: one 256-row K-major operand)
        const uint32_t idesc = two_rg ? idesc_bf16_m128(128u) : tr ? idesc_bf16_m128(256u) : idesc_bf16_m128((uint32_t)p.n_pad);
        uint32_t s = kseq % stages, ph = (kseq / stages) & 1;
        const uint32_t full0 = smem_u32(fullb), ring0 = smem_u32(ring);
#pragma unroll 1
        for (int i = 0; i < nkb; ++i) {
            mbar_wait_addr(full0 + 8 * s, ph);
            if (lane == 0 && (dbg & 64) && (i == 0 || i == nkb - 1)) sm.tdbg[i == 0 ? 0 : 1] = clock64();
            tc_fence_after();
            const uint32_t sa = ring0 + s * stride;
            const uint64_t ad0 = sdesc_k_sw128(sa), ad1 = sdesc_k_sw128(sa + a_bytes),
                           bd = sdesc_k_sw128(sa + boff);
            if (two_rg) {
                const uint64_t bd1 = sdesc_k_sw128(sa + boff + 16384u);  // batch rows 128-255
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k) {
                    tc_mma_bf16_warp(sm.tmem, bd + (uint64_t)(2 * k), ad0 + (uint64_t)(2 * k), idesc, (i | k) != 0);
                    tc_mma_bf16_warp(sm.tmem + 128u, bd1 + (uint64_t)(2 * k), ad0 + (uint64_t)(2 * k), idesc,
                                     (i | k) != 0);
                }
            } else if (tr) {
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)
                    tc_mma_bf16_warp(sm.tmem, bd + (uint64_t)(2 * k), ad0 + (uint64_t)(2 * k), idesc, (i | k) != 0);
            } else
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
                tc_mma_bf16_warp(sm.tmem, ad0 + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (i | k) != 0);
                if (na > 1)
                    tc_mma_bf16_warp(sm.tmem + 256u, ad1 + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc,
                                     (i | k) != 0);
            }
            tc_commit_warp(&emptyb[s]);
            if (++s == stages) {
                s = 0;
                ph ^= 1;
            }
        }
        tc_commit_warp(&sm.acc);
    }
    __syncwarp();
    if (warp < 8) {
        mbar_wait(&sm.acc, useq & 1);
        tc_fence_after();
    }
    kseq += (uint32_t)nkb;
}

// split-K partial: part[u][c][row] for the nval valid columns
__device__ __forceinline__ void epi_partial(const IterSmem& sm, const IterPlan& p, int u, int nval) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = 32 * (warp & 3) + lane;
    const uint32_t trow = sm.tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    float* dst = p.part + (size_t)u * p.n_pad * kBM + row;
    for (int c0 = 16 * (warp >> 2); c0 < nval; c0 += 32) {
        float v[16];
        tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (c0 + j < nval) __stcg(dst + (size_t)(c0 + j) * kBM, v[j]);
    }
}

// LM-head tile epilogue: per column (sequence) the tile's (max1, max2, sum exp
// rel. max1, argmax lowest index) -> lm_part[tile][col]; logits stay on chip.
template <bool kFull>
__device__ void epi_lm(const DevState& st, const IterSmem& sm, float* tbuf, int tile, int nval) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int row0 = tile * kBM;
    const int rows = min(kBM, st.dm.V - row0);
    const uint32_t trow = sm.tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    for (int c0 = 0; c0 < nval; c0 += 32) {
        const int cc = c0 + 16 * (warp >> 2);
        if (cc < nval) {
            float v[16];
            tmem_ld16(trow + (uint32_t)cc, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) tbuf[(16 * (warp >> 2) + j) * 129 + 32 * (warp & 3) + lane] = v[j];
        }
        named_bar(2, 256);
        const int n = tid >> 3, part = tid & 7;  // 8 threads per column, 16 rows each
        const int col = c0 + n;
        float m1 = -INFINITY, m2 = -INFINITY, s = 0.f;
        int idx = 0x7fffffff;
        if (col < nval) {
            const float* cl = tbuf + n * 129;
            const int r1 = min(rows, part * 16 + 16);
            for (int r = part * 16; r < r1; ++r) {
                const float x = cl[r];
                if (x > m1) {
                    if (kFull) {
                        m2 = m1;
                        s = s * __expf(m1 - x) + 1.f;
                    }
                    m1 = x;
                    idx = row0 + r;
                } else if (kFull) {
                    m2 = fmaxf(m2, x);
                    s += __expf(x - m1);
                }
            }
        }
        LmPart q{m1, m2, s, idx};
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) {
            LmPart o;
            o.m1 = __shfl_xor_sync(0xffffffffu, q.m1, off);
            o.m2 = __shfl_xor_sync(0xffffffffu, q.m2, off);
            o.s = __shfl_xor_sync(0xffffffffu, q.s, off);
            o.idx = __shfl_xor_sync(0xffffffffu, q.idx, off);
            q = (part & off) ? lm_part_merge(o, q) : lm_part_merge(q, o);
        }
        if (part == 0 && col < nval)
            st.lm_part[(size_t)tile * st.dm.Bmax + col] = make_float4(q.m1, q.m2, q.s, __int_as_float(q.idx));
        named_bar(2, 256);
    }
}

// Greedy-token LM-head tile epilogue (argmax only, lowest index on ties): per column the tile's
// (max, argmax) -> lm_part[tile][col] as (max, -inf, 0, argmax).  Each warp reduces its 32 vocab
// rows x 16 columns per TMEM load with a reduce-scatter butterfly (16 + 16 shuffles, after which
// lanes 2k / 2k+1 hold column k), then one barrier and the 4 row groups in ascending order --
// instead of epi_lm's shared-memory transpose and two barriers per 32 columns (8.5 -> ~3 us per
// tile at c5, scripts/pipe_tail.py).
__device__ __forceinline__ void lm_pick(float& v, int& i, float w, int k) {
    if (w > v || (w == v && k < i)) {
        v = w;
        i = k;
    }
}
__device__ void epi_lm_argmax(const DevState& st, const IterSmem& sm, float* tbuf, int tile, int nval) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rg = warp & 3, row0 = tile * kBM;
    const int my_row = row0 + 32 * rg + lane;
    const bool valid = 32 * rg + lane < min(kBM, st.dm.V - row0);
    const uint32_t trow = sm.tmem + ((uint32_t)(32 * rg) << 16);
    float* bv = tbuf;                                  // [4][256] best value per row group and column
    int* bi = reinterpret_cast<int*>(tbuf + 4 * 256);  // [4][256] its vocab index
    for (int c0 = 16 * (warp >> 2); c0 < nval; c0 += 32) {
        float v[16];
        tmem_ld16(trow + (uint32_t)c0, v);
        float w[8];
        int k[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // xor 16: keep columns [0, 8) (lanes 0-15) or [8, 16)
            const bool hi = lane & 16;
            const float a = valid ? (hi ? v[j + 8] : v[j]) : -INFINITY;
            const float send = valid ? (hi ? v[j] : v[j + 8]) : -INFINITY;
            const float b = __shfl_xor_sync(0xffffffffu, send, 16);
            const int kb = __shfl_xor_sync(0xffffffffu, my_row, 16);
            w[j] = a;
            k[j] = my_row;
            lm_pick(w[j], k[j], b, kb);
        }
#pragma unroll
        for (int o = 8, n = 4; o >= 2; o >>= 1, n >>= 1) {  // xor 8 / 4 / 2: halve the columns held
            const bool hi = lane & o;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j >= n) break;
                const float send = hi ? w[j] : w[j + n];
                const int sk = hi ? k[j] : k[j + n];
                const float b = __shfl_xor_sync(0xffffffffu, send, o);
                const int kb = __shfl_xor_sync(0xffffffffu, sk, o);
                float a = hi ? w[j + n] : w[j];
                int ka = hi ? k[j + n] : k[j];
                lm_pick(a, ka, b, kb);
                w[j] = a;
                k[j] = ka;
            }
        }
        {  // xor 1: the lane pair agrees on its column's best
            const float b = __shfl_xor_sync(0xffffffffu, w[0], 1);
            const int kb = __shfl_xor_sync(0xffffffffu, k[0], 1);
            lm_pick(w[0], k[0], b, kb);
        }
        const int col = c0 + ((lane >> 1) & 15);
        if (!(lane & 1) && col < nval) {
            bv[rg * 256 + col] = w[0];
            bi[rg * 256 + col] = k[0];
        }
    }
    named_bar(2, 256);
    for (int c = tid; c < nval; c += 256) {
        float m = bv[c];
        int i = bi[c];
#pragma unroll
        for (int g = 1; g < 4; ++g) lm_pick(m, i, bv[g * 256 + c], bi[g * 256 + c]);
        st.lm_part[(size_t)tile * st.dm.Bmax + c] = make_float4(m, -INFINITY, 0.f, __int_as_float(i));
    }
}

// Softmax-check LM-head tile epilogue: per column the tile's (max1, max2, sum exp rel. max1,
// argmax) -> lm_part[tile][col], by the same reduce-scatter butterfly as epi_lm_argmax with
// lm_part_merge at every level (one exp per merge) and one barrier -- instead of epi_lm<true>'s
// shared-memory transpose, sequential 16-row scans and two barriers per 32 columns.
__device__ __forceinline__ LmPart lm_leaf(float v, int i) {
    return LmPart{v, -INFINITY, v == -INFINITY ? 0.f : 1.f, i};
}
__device__ __forceinline__ LmPart lm_shfl(const LmPart& x, int o) {
    return LmPart{__shfl_xor_sync(0xffffffffu, x.m1, o), __shfl_xor_sync(0xffffffffu, x.m2, o),
                  __shfl_xor_sync(0xffffffffu, x.s, o), __shfl_xor_sync(0xffffffffu, x.idx, o)};
}
__device__ void epi_lm_full(const DevState& st, const IterSmem& sm, float* tbuf, int tile, int nval,
                            uint32_t tcol = 0) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rg = warp & 3, row0 = tile * kBM;
    const int my_row = row0 + 32 * rg + lane;
    const bool valid = 32 * rg + lane < min(kBM, st.dm.V - row0);
    const uint32_t trow = sm.tmem + tcol + ((uint32_t)(32 * rg) << 16);
    LmPart* gp = reinterpret_cast<LmPart*>(tbuf);  // [4][256] per row group and column (16 KB)
    for (int c0 = 16 * (warp >> 2); c0 < nval; c0 += 32) {
        float v[16];
        tmem_ld16(trow + (uint32_t)c0, v);
        LmPart w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // xor 16: keep columns [0, 8) (lanes 0-15) or [8, 16)
            const bool hi = lane & 16;
            const float a = valid ? (hi ? v[j + 8] : v[j]) : -INFINITY;
            const float send = valid ? (hi ? v[j] : v[j + 8]) : -INFINITY;
            const float b = __shfl_xor_sync(0xffffffffu, send, 16);
            const int kb = __shfl_xor_sync(0xffffffffu, my_row, 16);
            w[j] = lm_part_merge(lm_leaf(a, my_row), lm_leaf(b, kb));
        }
#pragma unroll
        for (int o = 8, n = 4; o >= 2; o >>= 1, n >>= 1) {  // xor 8 / 4 / 2: halve the columns held
            const bool hi = lane & o;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j >= n) break;
                const LmPart send = hi ? w[j] : w[j + n];
                const LmPart keep = hi ? w[j + n] : w[j];
                w[j] = lm_part_merge(keep, lm_shfl(send, o));
            }
        }
        w[0] = lm_part_merge(w[0], lm_shfl(w[0], 1));  // (the lane pair: same merge, same result)
        const int col = c0 + ((lane >> 1) & 15);
        if (!(lane & 1) && col < nval) gp[rg * 256 + col] = w[0];
    }
    named_bar(2, 256);
    for (int c = tid; c < nval; c += 256) {
        LmPart q = gp[c];
#pragma unroll
        for (int g = 1; g < 4; ++g) q = lm_part_merge(q, gp[g * 256 + c]);
        st.lm_part[(size_t)tile * st.dm.Bmax + c] = make_float4(q.m1, q.m2, q.s, __int_as_float(q.idx));
    }
}

// Transposed LM pair epilogue (unit_lm_pair with tr): TMEM lane = batch row, columns [128 h,
// 128 h + 128) = vocab rows of tile t0 + h.  Warps 4h..4h+3 reduce tile t0 + h, each thread its
// row's 128 logits in ascending vocab order (16 per TMEM load: chunk top-2 / argmax with strict >,
// i.e. the lowest index on ties, then one rescale and 16 exps) -- no shuffles, no shared memory.
// kFull false: greedy argmax only, (max, -inf, 0, argmax) as epi_lm_argmax.  two_rg (batch 256):
// one tile, column half h = batch rows [128 h, 128 h + 128).
template <bool kFull>
__device__ void epi_lm_tr(const DevState& st, const IterSmem& sm, int t0, int na, int nval, bool two_rg = false) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rg = warp & 3, h = warp >> 2;
    if (!two_rg && h >= na) return;
    const int row = (two_rg ? 128 * h : 0) + 32 * rg + lane, tile = two_rg ? t0 : t0 + h, v0 = tile * kBM;
    const int nv = min(kBM, st.dm.V - v0);
    const uint32_t taddr = sm.tmem + ((uint32_t)(32 * rg) << 16) + (uint32_t)(128 * h);
    float m1 = -INFINITY, m2 = -INFINITY, sum = 0.f;
    int idx = 0x7fffffff;
#pragma unroll 1
    for (int c0 = 0; c0 < kBM; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + (uint32_t)c0, v);
        float cm = m1, c2 = m2;
        int ci = idx;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (c0 + j >= nv) v[j] = -INFINITY;
            if (v[j] > cm) {
                c2 = cm;
                cm = v[j];
                ci = v0 + c0 + j;
            } else {
                c2 = fmaxf(c2, v[j]);
            }
        }
        if (cm == -INFINITY) continue;
        if (kFull) {
            float add = 0.f;
#pragma unroll
            for (int j = 0; j < 16; ++j) add += __expf(v[j] - cm);
            sum = (m1 == -INFINITY ? 0.f : sum * __expf(m1 - cm)) + add;
        }
        m1 = cm;
        m2 = c2;
        idx = ci;
    }
    if (row < nval)
        st.lm_part[(size_t)tile * st.dm.Bmax + row] =
            kFull ? make_float4(m1, m2, sum, __int_as_float(idx)) : make_float4(m1, -INFINITY, 0.f, __int_as_float(idx));
}

// Greedy LM head of the decode tail, unit `it` of tail_lm_units(p): with p.lm_tail_tr a transposed
// unit (batch 128: a vocab tile pair; batch 256: one tile, both row groups) and the per-thread
// argmax epilogue, else one weight-streaming tile and the shuffle-butterfly argmax.
__device__ __forceinline__ int tail_lm_units(const IterPlan& p) {
    return (p.lm_tail_tr && p.n_pad == 128) ? (p.lm_tiles + 1) / 2 : p.lm_tiles;
}
__device__ void epi_lm_argmax(const DevState& st, const IterSmem& sm, float* tbuf, int tile, int nval);
__device__ __forceinline__ void tail_lm_unit(const DevState& st, IterSmem& sm, uint8_t* ring, const IterPlan& p,
                                             uint32_t& kseq, float* tbuf, const uint16_t* bsrc, int NR, int it,
                                             int B, uint32_t useq) {
    const int dp = st.dm.dp, warp = threadIdx.x >> 5;
    const uint64_t pol = p.lm_keep == 2 ? kL2EvictLast : kL2EvictFirst;
    if (p.lm_tail_tr) {
        const int per = p.n_pad == 128 ? 2 : 1, t0 = it * per, na = min(per, p.lm_tiles - t0);
        unit_lm_pair(sm, ring, p, kseq, st.lm + (size_t)t0 * (dp / kBK) * (kBM * kBK), na, bsrc, (size_t)NR * kBK,
                     dp / kBK, useq, pol, true);
        if (warp < 8) epi_lm_tr<false>(st, sm, t0, na, B, p.n_pad == 256);
    } else {
        unit_ws(sm, ring, p, kseq, st.lm + (size_t)it * (dp / kBK) * (kBM * kBK), bsrc, (size_t)NR * kBK, 0,
                dp / kBK, useq, 0, 0, pol);
        if (warp < 8) epi_lm_argmax(st, sm, tbuf, it, B);
    }
}

// one LM-head column reduced over all vocab tiles by one warp (fixed tree)
__device__ __forceinline__ LmPart lm_col_warp(const DevState& st, int b) {
    const int lane = threadIdx.x & 31, tiles = st.dm.Vp / kBM;
    LmPart acc{-INFINITY, -INFINITY, 0.f, 0x7fffffff};
    // the lane's partials loaded 8 at a time before merging them in the same order (8 dependent
    // L2 round trips at V = 32128 were the critical path of the softmax confidence phase)
    constexpr int kU = 8;
    for (int t0 = lane; t0 < tiles; t0 += 32 * kU) {
        float4 q[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j)
            q[j] = t0 + 32 * j < tiles ? __ldcg(&st.lm_part[(size_t)(t0 + 32 * j) * st.dm.Bmax + b])
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < kU; ++j)
            if (t0 + 32 * j < tiles) acc = lm_part_merge(acc, LmPart{q[j].x, q[j].y, q[j].z, __float_as_int(q[j].w)});
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        LmPart o;
        o.m1 = __shfl_xor_sync(0xffffffffu, acc.m1, off);
        o.m2 = __shfl_xor_sync(0xffffffffu, acc.m2, off);
        o.s = __shfl_xor_sync(0xffffffffu, acc.s, off);
        o.idx = __shfl_xor_sync(0xffffffffu, acc.idx, off);
        acc = (lane & off) ? lm_part_merge(o, acc) : lm_part_merge(acc, o);
    }
    return acc;
}

// ---------------------------------------------------------------------------
// epilogues applied to a finished output element (m-tile m, column c, row r)
// ---------------------------------------------------------------------------
struct IterCtx {
    int layer;  // layer of the weights (fill: the skipped layer j)
    int pin, pout;
};

// K/V element offset of (column c, layer) at the column's current position
__device__ __forceinline__ long long kv_dst(const DevState& st, const IterSmem& sm, int c, int layer) {
    // (the per-row division by the block capacity is done once per launch: sm.kvrow / kvin)
    const Dims& dm = st.dm;
    const int blk = __ldg(&st.tables[sm.kvrow[c] + (layer - 1) * dm.bpl_max]);
    return (long long)blk * dm.bc * dm.dp + sm.kvin[c];
}

// 4 consecutive rows r0..r0+3 (r0 % 4 == 0) of output tile m, column c
// Side inputs of the 4-row epilogue, loaded before the partial sums so that their L2
// round trip overlaps the partials' (residual / mid rows, the K/V destination)
struct Side4 {
    float4 a;
    long long kvd;
};
template <int K>
__device__ __forceinline__ Side4 side4(const DevState& st, const IterSmem& sm, const IterCtx& x, int m, int c, int r0) {
    const int dp = st.dm.dp, Bm = st.dm.Bmax;
    const int R = m * kBM + r0;
    Side4 o{make_float4(0.f, 0.f, 0.f, 0.f), 0};
    if constexpr (K == kIQkv || K == kIFill) {
        const int kind = (K == kIQkv) ? R / dp : 1 + R / dp;
        if (kind != 0) o.kvd = kv_dst(st, sm, c, x.layer);
    } else if constexpr (K == kIWoc) {
        o.a = __ldcg(reinterpret_cast<const float4*>(st.mid32 + (size_t)c * dp + R));
    } else if constexpr (K == kIWo) {
        o.a = __ldcg(reinterpret_cast<const float4*>(st.h32 + (size_t)x.pin * Bm * dp + (size_t)c * dp + R));
    }
    return o;
}
template <int K>
__device__ __forceinline__ void apply4(const DevState& st, const IterSmem& sm, const IterCtx& x, int m, int c, int r0,
                                       float4 v, const Side4* pre = nullptr, bool dry = false) {
    const int dp = st.dm.dp, NR = st.NR, Bm = st.dm.Bmax;
    const int R = m * kBM + r0;
    if (dry) return;
    if constexpr (K == kIQkv || K == kIFill) {
        const int kind = (K == kIQkv) ? R / dp : 1 + R / dp;  // 0 q, 1 k, 2 v
        if (kind == 0) {
            *reinterpret_cast<float4*>(st.q32 + (size_t)c * dp + R) = v;
        } else {
            const int f = R - (K == kIQkv ? kind : kind - 1) * dp;
            uint16_t* dst = (kind == 1 ? st.kpool : st.vpool) + (pre ? pre->kvd : kv_dst(st, sm, c, x.layer)) + f;
            const uint2 pk = make_uint2((uint32_t)f32_to_bf16(v.x) | ((uint32_t)f32_to_bf16(v.y) << 16),
                                        (uint32_t)f32_to_bf16(v.z) | ((uint32_t)f32_to_bf16(v.w) << 16));
            *reinterpret_cast<uint2*>(dst) = pk;
        }
    } else if constexpr (K == kIWoc) {  // T5 mode: mid += W_oc . cross
        const size_t i = (size_t)c * dp + R;
        const float4 h = pre ? pre->a : __ldcg(reinterpret_cast<const float4*>(st.mid32 + i));
        const float4 o = make_float4(h.x + v.x, h.y + v.y, h.z + v.z, h.w + v.w);
        *reinterpret_cast<float4*>(st.mid32 + i) = o;
        *reinterpret_cast<uint2*>(st.mid_b + act_offset(c, R, NR)) =
            make_uint2((uint32_t)f32_to_bf16(o.x) | ((uint32_t)f32_to_bf16(o.y) << 16),
                       (uint32_t)f32_to_bf16(o.z) | ((uint32_t)f32_to_bf16(o.w) << 16));
    } else if constexpr (K == kIWo) {
        const size_t i = (size_t)c * dp + R;
        const float4 h = pre ? pre->a : __ldcg(reinterpret_cast<const float4*>(st.h32 + (size_t)x.pin * Bm * dp + i));
        const float4 o = make_float4(h.x + v.x, h.y + v.y, h.z + v.z, h.w + v.w);
        *reinterpret_cast<float4*>(st.mid32 + i) = o;
        *reinterpret_cast<uint2*>(st.mid_b + act_offset(c, R, NR)) =
            make_uint2((uint32_t)f32_to_bf16(o.x) | ((uint32_t)f32_to_bf16(o.y) << 16),
                       (uint32_t)f32_to_bf16(o.z) | ((uint32_t)f32_to_bf16(o.w) << 16));
    } else if constexpr (K == kIUp) {
        const float4 o = make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
        *reinterpret_cast<uint2*>(st.up_b + act_offset(c, R, NR)) =
            make_uint2((uint32_t)f32_to_bf16(o.x) | ((uint32_t)f32_to_bf16(o.y) << 16),
                       (uint32_t)f32_to_bf16(o.z) | ((uint32_t)f32_to_bf16(o.w) << 16));
    }
}

// the fill epilogue for a full-K unit straight from TMEM (one row per thread).  The rows' K/V
// destinations at `layer` are looked up once per unit into shared memory (a dependent block-table
// load per stored element made this epilogue ~7x slower: 28 us per unit at c5, scripts/pipe_tail.py)
__device__ __forceinline__ void epi_fill_direct(const DevState& st, IterSmem& sm, int layer, int m, int nval) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, dp = st.dm.dp;
    for (int c = threadIdx.x; c < nval; c += 256) sm.kvd[c] = kv_dst(st, sm, c, layer);
    named_bar(2, 256);
    const int row = 32 * (warp & 3) + lane;
    const int R = m * kBM + row;
    const int kind = R / dp;  // 0 k, 1 v
    const int f = R - kind * dp;
    uint16_t* pool = kind == 0 ? st.kpool : st.vpool;
    const uint32_t trow = sm.tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    for (int c0 = 16 * (warp >> 2); c0 < nval; c0 += 32) {
        float v[16];
        tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j)  // (token turn: only layers past the row's own exit layer)
            if (c0 + j < nval && !(st.turn_token && layer <= st.row_exit[c0 + j]))
                pool[sm.kvd[c0 + j] + f] = f32_to_bf16(v[j]);
    }
}

// Reduce phase: piece (m, c) = 128 rows of one output column, one warp per
// piece (4 rows per lane), two pieces in flight per warp; the K splits are
// summed in split order (deterministic).  K == kIDown also produces the exit
// check's per-tile partial dots (fp64, fixed shuffle tree).
// pieces [P0, P) (piece = m * nval + c), this warp's first piece P0 + gw, stride GW
template <int K, int NP = 2>  // NP: pieces in flight per warp
// dry: compute on whatever the partials hold and store nothing -- an instruction-cache
// warm-up run of this exact code while the tile's other splits are still arriving
// row0: batch row of column 0 (the pipelined kernel reduces one half of the batch at a time)
__device__ __forceinline__ void reduce_range(const DevState& st, const IterSmem& sm, const IterPlan& p,
                                          const IterGemm& g, const IterCtx x, int nval, int unit_base, int P0, int P,
                                          int gw, int GW, bool dry = false, int row0 = 0) {
    const int lane = threadIdx.x & 31;
    const int S = g.splits;
    auto rstamp = [&](int k) {  // dbg 64: warp 0's reduce timeline in layer 1's down phase (SM clock)
        if (K == kIDown && !dry && (EL_DBG(st) & 64) && x.layer == 1 && threadIdx.x == 0)
            st.dbg_ts[310000 + (size_t)blockIdx.x * 8 + k] = clock64();
    };
    rstamp(0);
    const int dp = st.dm.dp, Bm = st.dm.Bmax;
    constexpr int KC = NP == 2 ? 8 : 6;  // splits loaded per round (register budget: 168 at 288 threads)
    for (int p0 = P0 + gw; p0 < P; p0 += NP * GW) {
        int mm[NP], cc[NP];
        bool ok[NP];
        float4 acc[NP];
        Side4 sd[NP];
        float4 dmid[NP], dh[NP], dw[NP];  // down: mid row, previous h (state), probe weights (classifier)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int pp = p0 + j * GW;
            ok[j] = pp < P;
            mm[j] = ok[j] ? pp / nval : 0;
            cc[j] = ok[j] ? pp % nval : 0;
            acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if constexpr (K == kIFill) {
                const int m2 = 2 * dp / kBM;
                IterCtx y = x;
                y.layer = x.layer + mm[j] / m2;
                sd[j] = side4<K>(st, sm, y, mm[j] % m2, cc[j] + row0, 4 * lane);
            } else if constexpr (K == kIDown) {
                const size_t i = (size_t)(cc[j] + row0) * dp + mm[j] * kBM + 4 * lane;
                dmid[j] = __ldcg(reinterpret_cast<const float4*>(st.mid32 + i));
                dh[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                dw[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (st.technique == kState)
                    dh[j] = (EL_DBG(st) & (1 << 23)) ? dmid[j]
                                                 : __ldcg(reinterpret_cast<const float4*>(st.h32 + (size_t)x.pin * Bm * dp + i));
                else if (st.technique == kClassifier)
                    dw[j] = __ldg(reinterpret_cast<const float4*>(st.probe_w + mm[j] * kBM + 4 * lane));
            } else {
                sd[j] = side4<K>(st, sm, x, mm[j], cc[j] + row0, 4 * lane);
            }
        }
        rstamp(1);
        for (int s0 = 0; s0 < S; s0 += KC) {
            float4 v[NP][KC];
#pragma unroll
            for (int j = 0; j < NP; ++j)
#pragma unroll
                for (int k = 0; k < KC; ++k) {
                    v[j][k] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (ok[j] && s0 + k < S) {
                        // unit index of (tile m, split s): fill units are (jj, m2, s) with m = jj*m2 + m2 == tile index
                        const size_t u = (size_t)unit_base + (size_t)mm[j] * S + s0 + k;
                        v[j][k] = __ldcg(reinterpret_cast<const float4*>(p.part + (u * p.n_pad + cc[j]) * kBM) + lane);
                    }
                }
#pragma unroll
            for (int j = 0; j < NP; ++j)
#pragma unroll
                for (int k = 0; k < KC; ++k)
                    if (s0 + k < S) {
                        acc[j].x += v[j][k].x;
                        acc[j].y += v[j][k].y;
                        acc[j].z += v[j][k].z;
                        acc[j].w += v[j][k].w;
                    }
        }
        rstamp(2);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            if (!ok[j]) continue;  // warp-uniform
            const int m = mm[j], c = cc[j] + row0, r0 = 4 * lane;
            if constexpr (K == kIFill) {
                const int m2 = 2 * dp / kBM;
                IterCtx y = x;
                y.layer = x.layer + m / m2;  // x.layer = first skipped layer
                if (st.turn_token && y.layer <= st.row_exit[c]) continue;  // (token turn: row's own range)
                apply4<K>(st, sm, y, m % m2, c, r0, acc[j], &sd[j], dry);
            } else if constexpr (K == kIDown) {
                const int R = m * kBM + r0;
                const size_t i = (size_t)c * dp + R;
                const float4 mid = dmid[j];
                const float4 o = make_float4(mid.x + acc[j].x, mid.y + acc[j].y, mid.z + acc[j].z, mid.w + acc[j].w);
                if (!dry) {
                    *reinterpret_cast<float4*>(st.h32 + (size_t)x.pout * Bm * dp + i) = o;
                    *reinterpret_cast<uint2*>(st.hb + (size_t)x.pout * st.NR * dp + act_offset(c, R, st.NR)) =
                        make_uint2((uint32_t)f32_to_bf16(o.x) | ((uint32_t)f32_to_bf16(o.y) << 16),
                                   (uint32_t)f32_to_bf16(o.z) | ((uint32_t)f32_to_bf16(o.w) << 16));
                }
                rstamp(3);
                if ((st.technique == kState || st.technique == kClassifier) && !(EL_DBG(st) & (1 << 22))) {
                    double x0 = 0.0, x1 = 0.0, x2 = 0.0;
                    const float ov[4] = {o.x, o.y, o.z, o.w};
                    if (st.technique == kState) {
                        const float4 h = dh[j];
                        const float hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const double a = hv[t], b = ov[t];
                            x0 += a * b;
                            x1 += a * a;
                            x2 += b * b;
                        }
                    } else {
                        const float wv[4] = {dw[j].x, dw[j].y, dw[j].z, dw[j].w};
#pragma unroll
                        for (int t = 0; t < 4; ++t) x0 += (double)wv[t] * (double)ov[t];
                    }
                    x0 = warp_sum_d(x0);
                    if (st.technique == kState) {  // (classifier: one dot only)
                        x1 = warp_sum_d(x1);
                        x2 = warp_sum_d(x2);
                    }
                    if (lane == 0 && !dry) {
                        double* q = st.exit_part + ((size_t)m * Bm + c) * 3;
                        q[0] = x0;
                        q[1] = x1;
                        q[2] = x2;
                    }
                }
                rstamp(4);
            } else {
                apply4<K>(st, sm, x, m, c, r0, acc[j], &sd[j], dry);
            }
        }
    }
}

template <int K>
__device__ void reduce_phase(const DevState& st, const IterSmem& sm, const IterPlan& p, const IterGemm& g,
                             const IterCtx& x, int nval, int unit_base, int m_total) {
    const int warp = threadIdx.x >> 5;
    if (warp >= 8) return;
    reduce_range<K>(st, sm, p, g, x, nval, unit_base, 0, m_total * nval, (int)blockIdx.x * 8 + warp,
                    (int)gridDim.x * 8);
}

// exit decision of `layer` for every row, computed identically by every CTA
// (exit_policy.cpp:89-115, engine.cpp:55-66); returns "stop here".
__device__ bool exit_decide(const DevState& st, IterSmem& sm, int layer, int B, int mt, int cta0 = 0) {
    const int tid = threadIdx.x, Bm = st.dm.Bmax;
    int all = 1;
    if (tid < B) {
        const int b = tid;
        float conf = __int_as_float(0x7fc00000);
        int acc = 0;
        const double lam = st.lambdas[layer - 1];
        switch (st.technique) {
            case kState:
            case kClassifier: {
                double x0 = 0.0, x1 = 0.0, x2 = 0.0;
                for (int m = 0; m < mt; ++m) {  // fixed tile order
                    const double* q = st.exit_part + ((size_t)m * Bm + b) * 3;
                    x0 += __ldcg(q);
                    x1 += __ldcg(q + 1);
                    x2 += __ldcg(q + 2);
                }
                double cd;
                if (st.technique == kState) cd = x0 / (sqrt(x1) * sqrt(x2));  // NaN on a zero-norm state
                else cd = 1.0 / (1.0 + exp(-(x0 + (double)st.probe_b)));
                conf = (float)cd;
                acc = cd > lam;
                break;
            }
            case kSoftmax:
                conf = __ldcg(&st.conf[(size_t)(layer - 1) * Bm + b]);
                acc = __ldcg(&st.accept[b]);
                break;
            case kFixed:
                conf = st.fixed_conf[(size_t)(layer - 1) * Bm + b];
                acc = (double)conf > lam;
                break;
            case kAlwaysAt: acc = layer >= st.exit_layer; break;
            default: acc = 0; break;
        }
        int s = sm.status[b];
        if (!s && acc) {
            s = 1;
            sm.status[b] = 1;
            sm.first[b] = layer;
        }
        all = s;
        if ((int)blockIdx.x == cta0 && !st.prefill) {  // (prefill rows may exceed max_batch: no decode records)
            if (st.technique != kSoftmax) {  // softmax: written by the distributed decide phase
                st.conf[(size_t)(layer - 1) * Bm + b] = conf;
                st.accept[b] = acc;
            }
            st.status[b] = s;
            st.first_accept[b] = sm.first[b];
        }
    }
    all = __syncthreads_and(all);
    return all || layer >= st.dm.L;
}

// ---------------------------------------------------------------------------
// batch-M GEMM (small batch): the batch rows are the M=128 operand (only the
// n_pad valid rows are loaded; the rest of the tile is ignored), a block of nt
// output features is N, and each unit runs the FULL reduction dimension, so the
// epilogue applies directly from TMEM -- no split-K partials, no reduce phase,
// one grid barrier per GEMM.  Costs an L2 read of the whole activation matrix
// per CTA (B x K bf16), cheap for B <= 128.
// ---------------------------------------------------------------------------
template <int K>
// res (optional): the 16 residual inputs of this (row, features), loaded before the unit's
// accumulator was ready (gemm_phase_t) so their L2 round trip overlaps the mainloop
__device__ __forceinline__ void apply16_t(const DevState& st, const IterSmem& sm, const IterCtx& x, int b, int f,
                                          const float* v, const float4* res = nullptr) {
    const int dp = st.dm.dp, NR = st.NR, Bm = st.dm.Bmax;
    auto pack = [](const float* w) {
        return make_uint4((uint32_t)f32_to_bf16(w[0]) | ((uint32_t)f32_to_bf16(w[1]) << 16),
                          (uint32_t)f32_to_bf16(w[2]) | ((uint32_t)f32_to_bf16(w[3]) << 16),
                          (uint32_t)f32_to_bf16(w[4]) | ((uint32_t)f32_to_bf16(w[5]) << 16),
                          (uint32_t)f32_to_bf16(w[6]) | ((uint32_t)f32_to_bf16(w[7]) << 16));
    };
    if constexpr (K == kIQkv) {
        const int kind = f / dp;
        if (kind == 0) {
            float4* q = reinterpret_cast<float4*>(st.q32 + (size_t)b * dp + f);
#pragma unroll
            for (int t = 0; t < 4; ++t) q[t] = make_float4(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]);
        } else {
            uint16_t* dst = (kind == 1 ? st.kpool : st.vpool) + sm.kvd[b] + (f - kind * dp);  // (gemm_phase_t)
            reinterpret_cast<uint4*>(dst)[0] = pack(v);
            reinterpret_cast<uint4*>(dst)[1] = pack(v + 8);
        }
    } else if constexpr (K == kIWo) {
        const size_t i = (size_t)b * dp + f;
        const float4* h = reinterpret_cast<const float4*>(st.h32 + (size_t)x.pin * Bm * dp + i);
        float o[16];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float4 hv = res ? res[t] : __ldcg(h + t);
            o[4 * t] = hv.x + v[4 * t];
            o[4 * t + 1] = hv.y + v[4 * t + 1];
            o[4 * t + 2] = hv.z + v[4 * t + 2];
            o[4 * t + 3] = hv.w + v[4 * t + 3];
        }
        float4* m = reinterpret_cast<float4*>(st.mid32 + i);
#pragma unroll
        for (int t = 0; t < 4; ++t) m[t] = make_float4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
        *reinterpret_cast<uint4*>(st.mid_b + act_offset(b, f, NR)) = pack(o);
        *reinterpret_cast<uint4*>(st.mid_b + act_offset(b, f + 8, NR)) = pack(o + 8);
    } else if constexpr (K == kIWoc) {  // T5 mode: cross-attention output projection + residual (in place)
        const size_t i = (size_t)b * dp + f;
        float4* m4 = reinterpret_cast<float4*>(st.mid32 + i);
        float o[16];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float4 hv = res ? res[t] : __ldcg(m4 + t);
            o[4 * t] = hv.x + v[4 * t];
            o[4 * t + 1] = hv.y + v[4 * t + 1];
            o[4 * t + 2] = hv.z + v[4 * t + 2];
            o[4 * t + 3] = hv.w + v[4 * t + 3];
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) m4[t] = make_float4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
        *reinterpret_cast<uint4*>(st.mid_b + act_offset(b, f, NR)) = pack(o);
        *reinterpret_cast<uint4*>(st.mid_b + act_offset(b, f + 8, NR)) = pack(o + 8);
    } else if constexpr (K == kIDown) {  // down + residual -> h_l; exit-check partial dots of these 16 features
        const size_t i = (size_t)b * dp + f;
        const float4* m4 = reinterpret_cast<const float4*>(st.mid32 + i);
        float o[16];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float4 hv = __ldcg(m4 + t);
            o[4 * t] = hv.x + v[4 * t];
            o[4 * t + 1] = hv.y + v[4 * t + 1];
            o[4 * t + 2] = hv.z + v[4 * t + 2];
            o[4 * t + 3] = hv.w + v[4 * t + 3];
        }
        float4* h4 = reinterpret_cast<float4*>(st.h32 + (size_t)x.pout * Bm * dp + i);
#pragma unroll
        for (int t = 0; t < 4; ++t) h4[t] = make_float4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
        uint16_t* hb = st.hb + (size_t)x.pout * NR * dp;
        *reinterpret_cast<uint4*>(hb + act_offset(b, f, NR)) = pack(o);
        *reinterpret_cast<uint4*>(hb + act_offset(b, f + 8, NR)) = pack(o + 8);
        if (st.technique == kState || st.technique == kClassifier) {
            double x0 = 0.0, x1 = 0.0, x2 = 0.0;
            if (st.technique == kState) {
                const float4* p4 = reinterpret_cast<const float4*>(st.h32 + (size_t)x.pin * Bm * dp + i);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float4 hv = __ldcg(p4 + t);
                    const float hp[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double a = hp[q], c = o[4 * t + q];
                        x0 += a * c;
                        x1 += a * a;
                        x2 += c * c;
                    }
                }
            } else {
#pragma unroll
                for (int t = 0; t < 16; ++t) x0 += (double)__ldg(&st.probe_w[f + t]) * (double)o[t];
            }
            double* q = st.exit_part + ((size_t)(f >> 4) * Bm + b) * 3;  // one partial per 16-feature slice
            q[0] = x0;
            q[1] = x1;
            q[2] = x2;
        }
    } else if constexpr (K == kIUp) {
        float o[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) o[t] = fmaxf(v[t], 0.f);
        *reinterpret_cast<uint4*>(st.up_b + act_offset(b, f, NR)) = pack(o);
        *reinterpret_cast<uint4*>(st.up_b + act_offset(b, f + 8, NR)) = pack(o + 8);
    }
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
        "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z), "l"(policy)
        : "memory");
}

// batch-M unit mainloop.  A unit's weights (nt rows x the whole reduction dim) arrive
// with ONE 3-D tensor copy (rows f0..f0+nt of every k-block tile: the tiles are
// pre-swizzled, so the raw bytes are ready UMMA operands); the activations (the
// n_pad batch rows of all k-blocks, contiguous in the act layout) arrive in a few
// large 1-D copies of bm_kc k-blocks each.  Few big copies instead of two per
// k-block: a bulk copy costs ~60 ns of issue/processing on the SM's TMA unit
// regardless of its size.
// (the caller advances cseq by the chunk count and wseq by 1)
__device__ __forceinline__ void unit_bm(IterSmem& sm, uint8_t* ring, const IterPlan& p, const uint32_t cseq,
                                     const uint32_t wseq, const CUtensorMap* wmap, int wx, int wy, int wz,
                                     const uint16_t* act, int kb_total, int nt, uint32_t useq, bool w_ready,
                                     const uint16_t* wsrc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // p.bm_wstream: the weights stream through the ring next to the activations (stage = bm_kc act
    // k-blocks, then bm_kc weight k-blocks of nt rows = nt * 128 bytes each, copied from the
    // pre-swizzled tiles at wsrc + kb * 128 x 64), L2-prefetched one phase ahead by bm_prefetch:
    // no resident weight slab, so the ring holds more bytes in flight (a CTA's L2 stream is
    // bounded by bytes in flight / L2 latency under the attention CTAs' HBM load)
    const bool ws = p.bm_wstream != 0;
    const uint32_t wrow = (uint32_t)nt * 128u, wst = (uint32_t)p.bm_kc * (uint32_t)p.bm_grp * 128u;
    // act: this unit's row group (rows r*bm_grp ..) of k-block 0; one k-block of it is
    // NRb bytes in shared memory; with several row groups a k-block's group is not
    // contiguous with the next k-block's in global memory (stride bm_rows rows)
    const uint32_t NRb = (uint32_t)p.bm_grp * 128u;
    const bool grouped = p.bm_grp != p.bm_rows;
    const int nch = (kb_total + p.bm_kc - 1) / p.bm_kc;
    const uint32_t ring0 = smem_u32(ring), wbase = ring0 + (uint32_t)p.bm_woff;
    if (warp == kProducerWarp) {
        if (lane == 0 && !w_ready && !ws) {  // (else: prefetched into the weight buffer one phase ahead by bm_prefetch)
            const uint32_t wf = smem_u32(&sm.wfull);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(wf),
                         "r"((uint32_t)(nt * 128 * kb_total))
                         : "memory");
            tma_load_3d(wbase, wmap, wf, wx, wy, wz, kL2EvictFirst);
        }
        if (lane == 0) sm.tdbg[4] = clock64();  // producer starts issuing
        // lane 0 drives the ring; the activation copies go out from lanes 1..31 in turn (one
        // thread's bulk copies are processed one after another: scripts/ingest_probe*.cu)
        uint32_t s = cseq % (uint32_t)p.bm_stages, ph = (cseq / (uint32_t)p.bm_stages) & 1;
        bool wrapped = cseq >= (uint32_t)p.bm_stages;
        const uint32_t full0 = smem_u32(sm.full2), empty0 = smem_u32(sm.empty2);
        const uint64_t pol = kL2EvictLast;  // activations: re-read by every unit of the phase
        int issued = 0;  // copies so far (their lane rotates)
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {
            const int kc = min(p.bm_kc, kb_total - c * p.bm_kc);
            const uint32_t fb = full0 + 8 * s, bytes = (uint32_t)kc * NRb;
            if (lane == 0) {
                if (wrapped) mbar_wait_addr(empty0 + 8 * s, ph ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                             "r"(bytes + (ws ? (uint32_t)kc * wrow : 0u))
                             : "memory");
            }
            __syncwarp();
            if (ws)
                for (int j = 0; j < kc; ++j, ++issued)
                    if (lane == (EL_LANE_ISSUE ? 1 + issued % 31 : 0))
                        bulk_load_hint(ring0 + s * (uint32_t)p.bm_astage + wst + (uint32_t)j * wrow,
                                       wsrc + (size_t)(c * p.bm_kc + j) * (kBM * kBK), wrow, fb, kL2EvictFirst);
            if (!grouped) {
                if (lane == (EL_LANE_ISSUE ? 1 + issued % 31 : 0))
                    bulk_load_hint(ring0 + s * (uint32_t)p.bm_astage, act + (size_t)c * p.bm_kc * p.bm_rows * kBK,
                                   bytes, fb, pol);
                ++issued;
            } else {
                for (int j = 0; j < kc; ++j, ++issued)
                    if (lane == (EL_LANE_ISSUE ? 1 + issued % 31 : 0))
                        bulk_load_hint(ring0 + s * (uint32_t)p.bm_astage + (uint32_t)j * NRb,
                                       act + (size_t)(c * p.bm_kc + j) * p.bm_rows * kBK, NRb, fb, pol);
            }
            if (++s == (uint32_t)p.bm_stages) {
                s = 0;
                ph ^= 1;
                wrapped = true;
            }
        }
    } else if (warp == 0) {
        {  // whole warp 0, one elected lane issues (uniform descriptors)
            // M = 64 when the batch fits (half the A-operand shared-memory reads of M = 128)
            const uint32_t idesc = idesc_bf16((uint32_t)p.bm_m, (uint32_t)nt);
            if (!ws) mbar_wait_addr(smem_u32(&sm.wfull), wseq & 1);
            if (lane == 0) {
                sm.tdbg[3] = clock64();
            }
            uint32_t s = cseq % (uint32_t)p.bm_stages, ph = (cseq / (uint32_t)p.bm_stages) & 1;
            const uint32_t full0 = smem_u32(sm.full2);
            int kb = 0;
#pragma unroll 1
            for (int c = 0; c < nch; ++c) {
                const int kc = min(p.bm_kc, kb_total - c * p.bm_kc);
                mbar_wait_addr(full0 + 8 * s, ph);
                if (lane == 0 && (c == 0 || c == nch - 1)) {
                    sm.tdbg[c == 0 ? 1 : 2] = clock64();
                }
                tc_fence_after();
#pragma unroll 1
                for (int j = 0; j < kc; ++j, ++kb) {
                    // rows >= n_pad of the A tile read the next k-block / stage / weights: ignored output rows
                    const uint64_t ad = sdesc_k_sw128(ring0 + s * (uint32_t)p.bm_astage + (uint32_t)j * NRb);
                    const uint64_t bd = sdesc_k_sw128(ws ? ring0 + s * (uint32_t)p.bm_astage + wst + (uint32_t)j * wrow
                                                         : wbase + (uint32_t)(kb * nt * 128));
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        tc_mma_bf16_warp(sm.tmem, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (kb | k) != 0);
                }
                tc_commit_warp(&sm.empty2[s]);
                if (++s == (uint32_t)p.bm_stages) {
                    s = 0;
                    ph ^= 1;
                }
            }
            if (lane == 0) {
                sm.tdbg[0] = clock64();  // MMA issue finished
            }
            tc_commit_warp(&sm.acc);
        }
    }
    __syncwarp();
    if (warp < 8) {
        mbar_wait(&sm.acc, useq & 1);
        tc_fence_after();
    }
}

// Weights of this CTA's first unit of batch-M GEMM `gid` at `layer`, issued one phase
// ahead into the weight buffer (which lies outside the attention / GEMM rings) by the
// producer lane; weights never depend on the previous phase, so their HBM latency
// overlaps the phase in flight and the grid barrier.  Returns whether it issued.
__device__ __forceinline__ bool bm_prefetch(IterSmem& sm, uint8_t* ring, const IterPlan& p, const IterMaps& maps,
                                            int gid, int layer, int ci = -1, int rg_only = -1, int cn = -1) {
    const IterGemm& g = p.g[gid];
    if (g.mode && p.bm_wstream) {  // streamed weights: this CTA's units of the phase -> L2 (no completion)
        const int CI = ci < 0 ? (int)blockIdx.x : ci, CN = cn < 0 ? (int)gridDim.x : cn;
        const int R = rg_only >= 0 ? 1 : p.bm_rows / p.bm_grp;
        const int U = g.m_tiles * kBM / g.nt * R;
        for (int u = CI; u < U; u += CN) {
            const int f0 = (u / R) * g.nt;
            const int row_block = (layer - 1) * g.layer_rows + g.row_off + f0 / kBM;
            const uint16_t* w = g.A + (size_t)row_block * g.kb_total * (kBM * kBK) + (size_t)(f0 % kBM) * kBK;
            for (int kb = 0; kb < g.kb_total; ++kb)
                l2_prefetch_bulk(w + (size_t)kb * (kBM * kBK), (uint32_t)g.nt * 128u);
        }
        return false;
    }
    if (!g.mode || !p.bm_prefetch) return false;
    const int CI = ci < 0 ? (int)blockIdx.x : ci;
    // this CTA's first unit: (feature group CI / R, row group CI % R); one row group: feature group CI
    const int R = rg_only >= 0 ? 1 : p.bm_rows / p.bm_grp;
    if (CI >= g.m_tiles * kBM / g.nt * R) return false;
    const int f0 = (CI / R) * g.nt;
    const int row_block = (layer - 1) * g.layer_rows + g.row_off + f0 / kBM;
    const uint32_t wf = smem_u32(&sm.wfull);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(wf),
                 "r"((uint32_t)(g.nt * 128 * g.kb_total))
                 : "memory");
    tma_load_3d(smem_u32(ring) + (uint32_t)p.bm_woff, &maps.w[gid], wf, 0, f0 % kBM, row_block * g.kb_total,
                kL2EvictFirst);
    return true;
}

template <int K, bool kPre = false>  // kPre: residual prefetch (pipelined kernel: free registers)
__device__ __forceinline__ void gemm_phase_t(const DevState& st, IterSmem& sm, uint8_t* ring, const IterPlan& p,
                                             const IterMaps& maps, int gid, const IterCtx& x, const uint16_t* act,
                                             uint32_t& cseq, uint32_t& wseq, uint32_t& useq, int B, bool& wpf,
                                             int next_gid, int next_layer, int ci = -1, int cn = -1,
                                             int rg_only = -1, int next_rg = -1) {
    const IterGemm& g = p.g[gid];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int CI = ci < 0 ? (int)blockIdx.x : ci, CN = cn < 0 ? (int)gridDim.x : cn;
    const int Rall = p.bm_rows / p.bm_grp;
    // row groups: unit u = (feature group u / R, row group u % R); rg_only >= 0: that row group only
    const int R = rg_only >= 0 ? 1 : Rall;
    const int U = g.m_tiles * kBM / g.nt * R;
    auto stamp = [&](int k) {  // dbg 64: per-CTA unit timeline of layer 1's batch-M GEMMs
        if ((EL_DBG(st) & 64) && x.layer == 1 && threadIdx.x == 0)  // SM clock (globaltimer ticks are 256 ns)
            st.dbg_ts[300000 + (size_t)blockIdx.x * 32 + K * 8 + k] = clock64();
    };
    stamp(0);
    if constexpr (K == kIQkv) {  // the rows' K/V destinations at this layer, looked up once per phase
        if (st.kpool) {
            for (int b = threadIdx.x; b < B; b += blockDim.x) sm.kvd[b] = kv_dst(st, sm, b, x.layer);
            __syncthreads();
        }
    }
    for (int u = CI; u < U; u += CN) {
        const int f0 = (u / R) * g.nt, rg = rg_only >= 0 ? rg_only : u % R;
        const int row_block = (x.layer - 1) * g.layer_rows + g.row_off + f0 / kBM;
        // residual-add epilogues: this thread's residual inputs (row b, its first two 16-feature
        // chunks) are loaded now, their L2 latency hidden behind the mainloop
        constexpr bool kRes = kPre && (K == kIWo || K == kIWoc);
        float4 res[2][4];
        const bool m64p = p.bm_m == 64;
        const int lp = m64p ? 16 * (warp & 3) + lane : 32 * (warp & 3) + lane;  // row inside the group
        const int bp = rg * p.bm_grp + lp;
        const bool vp = warp < 8 && bp < B && (!m64p || lane < 16) && lp < p.bm_grp;
        if constexpr (kRes) {
            if (vp) {
                const float* base = (K == kIWo ? st.h32 + (size_t)x.pin * st.dm.Bmax * st.dm.dp : st.mid32) +
                                    (size_t)bp * st.dm.dp + f0;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int c0 = 16 * (warp >> 2) + 32 * q;
                    if (c0 < g.nt)
#pragma unroll
                        for (int t = 0; t < 4; ++t) res[q][t] = __ldcg(reinterpret_cast<const float4*>(base + c0) + t);
                }
            }
        }
        unit_bm(sm, ring, p, cseq, wseq, &maps.w[gid], 0, f0 % kBM, row_block * g.kb_total,
                act + (size_t)rg * p.bm_grp * kBK, g.kb_total, g.nt, useq, wpf,
                g.A + (size_t)row_block * g.kb_total * (kBM * kBK) + (size_t)(f0 % kBM) * kBK);
        cseq += (uint32_t)((g.kb_total + p.bm_kc - 1) / p.bm_kc);
        ++wseq;
        wpf = false;
        stamp(2);
        if ((EL_DBG(st) & 64) && x.layer == 1 && threadIdx.x == 0)
            for (int k = 0; k < 5; ++k) st.dbg_ts[300000 + (size_t)blockIdx.x * 32 + K * 8 + (k < 4 ? 4 + k : 1)] = sm.tdbg[k];
        if (warp < 8) {
            // M = 128: batch row b in TMEM lane b.  M = 64: rows 16q..16q+15 in lanes 32q..32q+15.
            const bool m64 = p.bm_m == 64;
            const int lr = m64 ? 16 * (warp & 3) + lane : 32 * (warp & 3) + lane;  // row inside the group
            const int b = rg * p.bm_grp + lr;
            // (32-row groups of the pipelined kernel: UMMA M = 64, accumulator rows 32-63 discarded)
            const bool valid = b < B && (!m64 || lane < 16) && lr < p.bm_grp;
            const uint32_t trow = sm.tmem + ((uint32_t)(32 * (warp & 3)) << 16);
            if constexpr (kRes) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {  // (nt <= 128: at most 4 chunks of 16 features per thread)
                    const int c0 = 16 * (warp >> 2) + 32 * q;
                    if (c0 >= g.nt) break;
                    float v[16];
                    tmem_ld16(trow + (uint32_t)c0, v);
                    if (valid) apply16_t<K>(st, sm, x, b, f0 + c0, v, q < 2 ? res[q & 1] : nullptr);
                }
            } else {
                for (int c0 = 16 * (warp >> 2); c0 < g.nt; c0 += 32) {
                    float v[16];
                    tmem_ld16(trow + (uint32_t)c0, v);
                    if (valid) apply16_t<K>(st, sm, x, b, f0 + c0, v);
                }
            }
        }
        stamp(3);
        ++useq;
        tc_fence_before();
        __syncthreads();
    }
    // this phase's MMAs are done: the weight buffer is free for the next batch-M GEMM's weights
    if (next_gid >= 0 && threadIdx.x == kProducerWarp * 32)
        wpf = bm_prefetch(sm, ring, p, maps, next_gid, next_layer, ci, next_rg, cn);
}

// Split-K GEMM phase with the reduction fused per output tile: every unit's CTA
// publishes its partial and bumps the tile's arrival counter (monotonic within the
// launch, zeroed at its end); once all S splits of its tile are in, the S CTAs of
// the tile each reduce their own 1/S of the columns (in split order: deterministic)
// and apply the epilogue.  Replaces a grid barrier + a separate reduce phase by a
// wait on the S - 1 peers of the tile.
// `use`: 1-based count of this GEMM's phases in the launch (the tile counters only grow within
// a launch and are zeroed at its end)
// ci / cn: this CTA's index in the set of CTAs running the phase; row0 / n_rows: the batch rows
// of the phase (bsrc must point at row row0 of the activation layout; n_rows 0 = n_pad)
template <int K, int NP = 2>
__device__ void gemm_phase_fused(const DevState& st, IterSmem& sm, uint8_t* ring, const IterPlan& p, int gid,
                                 const IterCtx& x, const uint16_t* bsrc, uint32_t& kseq, uint32_t& useq, int nval,
                                 int use, int ci = -1, int cn = -1, int row0 = 0, int n_rows = 0) {
    const IterGemm& g = p.g[gid];
    const int warp = threadIdx.x >> 5;
    const int CI = ci < 0 ? (int)blockIdx.x : ci, CN = cn < 0 ? (int)gridDim.x : cn;
    const int U = g.m_tiles * g.splits;
    const size_t bks = (size_t)st.NR * kBK;
    unsigned* cnt = p.tcnt + gid * 64;
    auto stamp = [&](int k) {  // dbg 64: per-CTA timeline of layer 1's fused split-K phase (SM clock)
        if ((EL_DBG(st) & 64) && x.layer == 1 && threadIdx.x == 0 && K == kIDown)
            st.dbg_ts[300000 + (size_t)blockIdx.x * 32 + 3 * 8 + k] = clock64();
    };
    stamp(0);
    for (int u = CI; u < U; u += CN) {
        const int m = u / g.splits, s = u % g.splits;
        const int kb0 = s * g.kb_total / g.splits, kb1 = (s + 1) * g.kb_total / g.splits;
        const uint16_t* a = g.A + (size_t)((x.layer - 1) * g.layer_rows + g.row_off + m) * g.kb_total * (kBM * kBK);
        unit_ws(sm, ring, p, kseq, a, bsrc, bks, kb0, kb1 - kb0, useq,
                (K == kIDown && x.layer == 1) ? (EL_DBG(st) & 64) : 0, n_rows);
        stamp(1);
        if ((EL_DBG(st) & 64) && x.layer == 1 && threadIdx.x == 0 && K == kIDown)
            for (int k = 0; k < 3; ++k) st.dbg_ts[300000 + (size_t)blockIdx.x * 32 + 3 * 8 + 5 + k] = sm.tdbg[k == 2 ? 3 : k];
        if (warp < 8) epi_partial(sm, p, u, nval);
        ++useq;
        tc_fence_before();
        fence_proxy_async_global();
        __syncthreads();
        stamp(2);
        if (threadIdx.x == 0) {
            // (bar.sync above orders the CTA's partial stores before this thread's release)
            if (EL_DBG(st) & (1 << 26)) __threadfence();
            red_release_add_u32(cnt + m, 1u);
            if ((EL_DBG(st) & 64) && x.layer == 1 && K == kIDown) st.dbg_ts[310000 + (size_t)blockIdx.x * 8 + 5] = clock64();
        }
    }
    for (int u = CI; u < U; u += CN) {
        const int m = u / g.splits, s = u % g.splits;
        const int c0 = s * nval / g.splits, c1 = (s + 1) * nval / g.splits;
        // dbg bit 24: pass 0 (dry) runs the reduce code while the tile's other splits arrive,
        // so that pass 1 finds it in the instruction cache -- measured slower (the dry pass is
        // as cold as the real one was and outlasts the wait)
#pragma unroll 1
        for (int pass = (EL_DBG(st) & (1 << 24)) ? 0 : 1; pass < 2; ++pass) {
            if (pass == 1) {
                if (threadIdx.x == 0) {
                    const unsigned target = (unsigned)(g.splits * use);
                    const long long t0 = clock64();
                    while (ld_acquire_u32(cnt + m) < target)
                        if (clock64() - t0 > EL_SPIN_LIMIT) __trap();
                    __threadfence();
                }
                __syncthreads();
                stamp(3);
            }
            if (warp < 8)
                reduce_range<K, NP>(st, sm, p, g, x, nval, 0, m * nval + c0, m * nval + c1, warp, 8, pass == 0, row0);
        }
        __syncthreads();
        stamp(4);
    }
}

template <int NJ>
__global__ void __launch_bounds__(kIterThreads, 1) iter_kernel(const __grid_constant__ DevState st,
                                                                const __grid_constant__ IterPlan p,
                                                                const __grid_constant__ IterMaps maps) {
    if (st.run_active && *(volatile const int*)st.run_active == 0) return;  // Engine::run chunk over
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    IterSmem& sm = *reinterpret_cast<IterSmem*>(ring + p.ring_bytes);
    float* tbuf = reinterpret_cast<float*>(ring + p.gemm_ring);
    float* att_mbuf = p.att_mbuf_off > 0 ? reinterpret_cast<float*>(ring + p.att_mbuf_off) : nullptr;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int G = (int)gridDim.x, cta = (int)blockIdx.x;
    const Dims& dm = st.dm;
    const int B = st.rows.B, L = dm.L, dp = dm.dp, Bm = dm.Bmax, NR = st.NR;
    const bool lm_pair = st.technique == kSoftmax && p.lm_pair;  // softmax checks on LM pair units

    if (tid == 0) {
        for (int s = 0; s < 8; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
            mbar_init(&sm.att.full[s], 1);
            mbar_init(&sm.att.empty[s], kAttnWarps);
        }
        for (int s = 0; s < 16; ++s) {
            mbar_init(&sm.full2[s], 1);
            mbar_init(&sm.empty2[s], 1);
        }
        mbar_init(&sm.wfull, 1);
        sm.att.npend = 0;
        sm.att.ids_layer[0] = sm.att.ids_layer[1] = -1;
        mbar_init(&sm.acc, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&sm.tmem, 512);
    for (int b = tid; b < 256; b += blockDim.x) {
        sm.pos[b] = b < B ? st.rows.pos[b] : 0;
        sm.kvrow[b] = b < B ? st.rows.slot[b] * dm.L * dm.bpl_max + st.rows.pos[b] / dm.bc : 0;
        sm.kvin[b] = b < B ? (st.rows.pos[b] % dm.bc) * dp : 0;
        sm.slot[b] = b < B ? st.rows.slot[b] : 0;
        sm.status[b] = 0;
        sm.first[b] = 0;
    }
    const int iter = *st.iter_counter;  // advanced by CTA 0 at the very end
    // generation base of this launch: no barrier of this launch can complete before every CTA read it
    // barrier bases: the generation word only moves once every CTA has arrived (so after
    // every CTA read it); the arrival count's base is the final count of the previous
    // launch, which CTA 0 stores in bar[2] at its end (the count itself may already move)
    const uint2 g0 = make_uint2(*(volatile unsigned*)(p.bar + 1024), *(volatile unsigned*)(p.bar + 2));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    uint32_t kseq = 0, kseq2 = 0, wseq = 0, useq = 0;
    bool wpf = false;  // producer lane: the next batch-M unit's weights were prefetched
    int aseq = 0, nbar = 0;
    if (EL_DBG(st) & 256)  // barrier cost probe: 32 back-to-back grid barriers
        for (int i = 0; i < 32; ++i) grid_sync(p, st, nbar, g0);
    if (EL_DBG(st) & (1 << 19)) {  // TMA probe: two QKV batch-M units back to back at kernel start
        const IterCtx x0{1, 0, 1};
        for (int rep = 0; rep < 2; ++rep) {
            gemm_phase_t<kIQkv>(st, sm, ring, p, maps, kIQkv, x0, st.hb, kseq2, wseq, useq, B, wpf, -1, 0);
            grid_sync(p, st, nbar, g0);
        }
    }

    if (warp == kProducerWarp) {
        if (st.enc_bidir > 0) {  // T5 encoder stack: every row streams all blocks of its sequence
            const int nb = (st.enc_bidir + dm.bc - 1) / dm.bc;
            for (int b = tid & 31; b <= B; b += 32) sm.att.pref[b] = b * nb;
        } else {
            attn_prefix_sum(st, sm.att);  // KV blocks per row: fixed for the iteration
        }
        if (st.enc_len > 0)
            for (int b = tid & 31; b <= B; b += 32) sm.att.pref_c[b] = b * st.enc_blocks;
        __syncwarp();
    }
    const AttnSrc self_src{st.tables, dm.bpl_max, st.kpool, st.vpool, st.enc_bidir, sm.att.pref, sm.pos, sm.slot, 0,
                           nullptr, 0u};
    const AttnSrc cross_src{st.ctables, st.enc_blocks, st.ckpool, st.cvpool, st.enc_len, sm.att.pref_c, sm.pos, sm.slot, 1, nullptr, 0u};
    // layers of this launch: 1..L (decode iteration / prefill), or the one layer of a turn
    const int lfirst = st.turn_layer > 0 ? st.turn_layer : 1, llast = st.turn_layer > 0 ? st.turn_layer : L;
    if (st.turn_layer > 1 || st.turn_token) {
        // layer-level turn past layer 1: each row's state entering this layer, kept per sequence;
        // token turn: each row's exit state, into the parity of the smallest exit layer
        const int pin = st.turn_token ? (lfirst & 1) : (lfirst - 1) & 1;
        for (int b = cta; b < B; b += G) {
            const float* src = st.hstore + (size_t)st.row_seq[b] * dp;
            float* h = st.h32 + ((size_t)pin * Bm + b) * dp;
            uint16_t* hbp = st.hb + (size_t)pin * NR * dp;
            for (int i = tid; i < dp; i += blockDim.x) {
                const float v = __ldcg(src + i);
                h[i] = v;
                hbp[act_offset(b, i, NR)] = f32_to_bf16(v);
            }
        }
    } else {
        // ---- embed (model.cpp:171-183): h_0 = embedding row of the input token ----
        for (int b = cta; b < B; b += G) {
            const uint16_t* e = st.emb + (size_t)st.rows.tok[b] * dp;
            float* h = st.h32 + (size_t)b * dp;
            for (int i = tid; i < dp; i += blockDim.x) {
                const uint16_t v = e[i];
                st.hb[act_offset(b, i, NR)] = v;
                h[i] = bf16_to_f32(v);
            }
        }
    }
    grid_sync(p, st, nbar, g0);

    int e_out = llast;
    for (int layer = lfirst; layer <= llast && !st.turn_token; ++layer) {
        const IterCtx x{layer, (layer - 1) & 1, layer & 1};
        // q | k | v, K/V appended to the paged pool (model.cpp:218-226)
        if (p.g[kIQkv].mode) {
            gemm_phase_t<kIQkv>(st, sm, ring, p, maps, kIQkv, x, st.hb + (size_t)x.pin * NR * dp, kseq2, wseq, useq, B,
                                wpf, -1, 0);
        } else {
            gemm_phase_fused<kIQkv>(st, sm, ring, p, kIQkv, x, st.hb + (size_t)x.pin * NR * dp, kseq, useq, B, layer - lfirst + 1);
        }
        // early attention start (default; barrier-mode 1-hop only): the producer warp skips
        // this barrier and streams the old K/V blocks of its range while the grid waits; q and
        // the newest block (this phase's output) wait on the barrier count
        AttnSrc self_l = self_src;
        // not in batched prefill: one launch holds several positions of a sequence, so blocks
        // older than a row's newest one may be written by this launch's QKV phase
        const bool early = p.att_early && !st.prefill && !(EL_DBG(st) & ((1 << 25) | (1 << 27)));
        if (early) {
            self_l.gate = p.bar;
            self_l.gate_target = g0.y + (unsigned)G * (unsigned)(nbar + 1);
            if (warp == kProducerWarp) ++nbar;
            else grid_sync_sub(p, st, nbar, g0);
        } else {
            grid_sync(p, st, nbar, g0);
        }
        // paged attention (model.cpp:223-243)
        auto astamp = [&](int w) {
            if ((EL_DBG(st) & 128) && tid == 0 && layer <= 24) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
                st.dbg_ts[40000 + (layer - 1) * 512 + cta * 2 + w] = t;
                unsigned smid;
                asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
                st.dbg_ts[40000 + 24 * 512 + cta] = smid;
            }
        };
        astamp(0);
        if ((EL_DBG(st) & 32) && tid == 0 && cta < 4) st.dbg_ts[8192 + 3072 + cta * 16] = clock64();
        if (tid == kProducerWarp * 32) wpf = bm_prefetch(sm, ring, p, maps, kIWo, layer);  // W_o under attention
        __syncwarp();
        attn_pass<NJ>(st, sm.att, ring, layer, aseq, self_l, att_mbuf);
        astamp(1);
        grid_sync(p, st, nbar, g0);
        aseq = sm.att.seq_next;
        __syncwarp();
        // W_o + residual (model.cpp:245-253)
        if (p.g[kIWo].mode) {
            gemm_phase_t<kIWo>(st, sm, ring, p, maps, kIWo, x, st.att_b, kseq2, wseq, useq, B, wpf,
                               st.enc_len > 0 ? (int)kIQc : (int)kIUp, layer);
        } else {
            gemm_phase_fused<kIWo>(st, sm, ring, p, kIWo, x, st.att_b, kseq, useq, B, layer - lfirst + 1);
        }
        grid_sync(p, st, nbar, g0);
        if (st.enc_len > 0) {
            // T5 mode: mid += W_oc . softmax(q_c K_c^T / sqrt(d)) V_c, q_c = W_qc . mid
            if (p.g[kIQc].mode) {
                gemm_phase_t<kIQkv>(st, sm, ring, p, maps, kIQc, x, st.mid_b, kseq2, wseq, useq, B, wpf, -1,
                                    0);  // q_c -> q32
            } else {
                gemm_phase_fused<kIQkv>(st, sm, ring, p, kIQc, x, st.mid_b, kseq, useq, B, layer - lfirst + 1);
            }
            grid_sync(p, st, nbar, g0);
            if (tid == kProducerWarp * 32) wpf = bm_prefetch(sm, ring, p, maps, kIWoc, layer);
            attn_pass<NJ>(st, sm.att, ring, layer, aseq, cross_src, att_mbuf);  // -> att_b
            grid_sync(p, st, nbar, g0);
            aseq = sm.att.seq_next;
            if (p.g[kIWoc].mode) {
                gemm_phase_t<kIWoc>(st, sm, ring, p, maps, kIWoc, x, st.att_b, kseq2, wseq, useq, B, wpf, kIUp,
                                    layer);
            } else {
                gemm_phase_fused<kIWoc>(st, sm, ring, p, kIWoc, x, st.att_b, kseq, useq, B, layer - lfirst + 1);
            }
            grid_sync(p, st, nbar, g0);
        }
        // up + ReLU (model.cpp:255-260)
        if (p.g[kIUp].mode) {
            gemm_phase_t<kIUp>(st, sm, ring, p, maps, kIUp, x, st.mid_b, kseq2, wseq, useq, B, wpf,
                               p.g[kIDown].mode ? (int)kIDown : -1, layer);
        } else {
            gemm_phase_fused<kIUp>(st, sm, ring, p, kIUp, x, st.mid_b, kseq, useq, B, layer - lfirst + 1);
        }
        grid_sync(p, st, nbar, g0);
        // down + residual (model.cpp:261-270) + exit-check partial dots
        if (p.g[kIDown].mode) {
            gemm_phase_t<kIDown>(st, sm, ring, p, maps, kIDown, x, st.up_b, kseq2, wseq, useq, B, wpf,
                                 layer < llast && !lm_pair ? (int)kIQkv : -1, layer + 1);
        } else {
            // (softmax checks on LM pair units: the next QKV slab is prefetched after the LM head,
            //  whose ring runs into the slab's region)
            if (tid == kProducerWarp * 32 && layer < llast && !lm_pair)
                wpf = bm_prefetch(sm, ring, p, maps, kIQkv, layer + 1);
            gemm_phase_fused<kIDown>(st, sm, ring, p, kIDown, x, st.up_b, kseq, useq, B, layer - lfirst + 1);
        }
        grid_sync(p, st, nbar, g0);
        if (st.technique == kSoftmax) {
            // LM head over h_l with the fused (max1, max2, sum exp) reduction
            const uint16_t* bsrc = st.hb + (size_t)x.pout * NR * dp;
            const uint64_t lpol = p.lm_keep ? kL2EvictLast : kL2EvictFirst;
            if (lm_pair) {
                float* tb2 = reinterpret_cast<float*>(ring + p.stages * (2 * kAStage + p.n_pad * 128));
                // (EL_DEBUG, dbg bit 64, layer 1: per-CTA clock64 stamps of the first unit at
                //  dbg_ts[320000 + cta * 8]: start, first / last stage full, producer done, acc, epilogue)
                const bool lstamp = (EL_DBG(st) & 64) && layer == 1 && cta < G;
                if (lstamp && tid == 0) st.dbg_ts[320000 + (size_t)cta * 8] = clock64();
                for (int u = cta; 2 * u < p.lm_tiles; u += G) {
                    const int t0 = 2 * u, na = min(2, p.lm_tiles - t0);
                    unit_lm_pair(sm, ring, p, kseq, st.lm + (size_t)t0 * (dp / kBK) * (kBM * kBK), na, bsrc,
                                 (size_t)NR * kBK, dp / kBK, useq, lpol, p.lm_pair == 2, lstamp && u == cta ? 64 : 0);
                    if (lstamp && u == cta && tid == 0) st.dbg_ts[320000 + (size_t)cta * 8 + 5] = clock64();
                    if (p.lm_pair == 2) {
                        if (warp < 8) epi_lm_tr<true>(st, sm, t0, na, B);
                    } else if (warp < 8) {
                        epi_lm_full(st, sm, tb2, t0, B);
                        if (na > 1) {
                            named_bar(2, 256);  // (the first tile's merge reads of tb2 are done)
                            epi_lm_full(st, sm, tb2, t0 + 1, B, 256u);
                        }
                    }
                    ++useq;
                    tc_fence_before();
                    __syncthreads();
                    if (lstamp && u == cta && tid == 0) {
                        st.dbg_ts[320000 + (size_t)cta * 8 + 6] = clock64();
                        for (int k = 0; k < 4; ++k) if (k != 2) st.dbg_ts[320000 + (size_t)cta * 8 + 1 + k] = sm.tdbg[k];
                    }
                }
                if (tid == kProducerWarp * 32 && layer < llast) wpf = bm_prefetch(sm, ring, p, maps, kIQkv, layer + 1);
            } else {
                for (int t = cta; t < p.lm_tiles; t += G) {
                    unit_ws(sm, ring, p, kseq, st.lm + (size_t)t * (dp / kBK) * (kBM * kBK), bsrc, (size_t)NR * kBK,
                            0, dp / kBK, useq, 0, 0, lpol);
                    if (warp < 8) epi_lm_full(st, sm, tbuf, t, B);
                    ++useq;
                    tc_fence_before();
                    __syncthreads();
                }
            }
            grid_sync(p, st, nbar, g0);
            // softmax_response_confidence (exit_policy.cpp:57-72), rows spread over the grid
            if (warp < 8)
                for (int b = cta + G * warp; b < B; b += G * 8) {
                    const LmPart r = lm_col_warp(st, b);
                    if ((tid & 31) == 0) {
                        const float gap = (r.m2 == -INFINITY) ? 1.f : -expm1f(r.m2 - r.m1);
                        const float conf = gap / r.s;
                        st.conf[(size_t)(layer - 1) * Bm + b] = conf;
                        st.accept[b] = (double)conf > st.lambdas[layer - 1];
                    }
                }
            grid_sync(p, st, nbar, g0);
        }
        if (exit_decide(st, sm, layer, B, p.g[kIDown].mode ? st.dm.dp / 16 : st.dm.dp / kBM)) {
            e_out = layer;
            // the next layer's QKV weights were prefetched for nothing: retire that load
            const IterGemm& gq = p.g[kIQkv];
            if (layer < llast && gq.mode && p.bm_prefetch && cta < gq.m_tiles * kBM / gq.nt * (p.bm_rows / p.bm_grp)) {
                if (warp == 0) {  // the MMA warp retires it
                    mbar_wait(&sm.wfull, wseq & 1);
                    ++wseq;
                }
                if (tid == kProducerWarp * 32) {
                    ++wseq;
                    wpf = false;
                }
            }
            break;
        }
    }

    if (st.turn_defer && !st.turn_token) {
        // deferred layer turn: every row's state at this layer -> the per-sequence store (an
        // exited row's is its exit state, for the token turn), exit flags -> the record
        if (warp < 8) {
            const int lane = tid & 31, cur = iter % st.rec_cap;
            for (int b = cta + G * warp; b < B; b += G * 8) {
                const float* src = st.h32 + ((size_t)(e_out & 1) * Bm + b) * dp;
                float* dst = st.hstore + (size_t)st.row_seq[b] * dp;
                for (int i = lane * 4; i < dp; i += 128)
                    *reinterpret_cast<float4*>(dst + i) = __ldcg(reinterpret_cast<const float4*>(src + i));
                if (lane == 0) {
                    const bool ex = e_out == L || sm.status[b];
                    rec_rec(st, cur)[b] = -1;
                    rec_rec(st, cur)[Bm + b] = ex ? e_out : 0;
                    rec_conf(st, cur)[(size_t)(e_out - 1) * Bm + b] = __ldcg(&st.conf[(size_t)(e_out - 1) * Bm + b]);
                }
            }
        }
        if (cta == 0 && tid == 0) {
            *(volatile unsigned*)(p.bar + 2) = g0.y + (unsigned)G * (unsigned)nbar;  // next launch's count base
            for (int i = 0; i < kINumGemm * 64; ++i) p.tcnt[i] = 0u;
            *st.cur_iter = iter;
            *st.iter_counter = iter + 1;
        }
        tc_fence_before();
        __syncthreads();
        if (warp == 0) tmem_dealloc(sm.tmem, 512);
        return;
    }
    if (st.prefill) {
        // batched causal prefill (engine.cpp:166-181): every layer's K/V of all rows is written;
        // no exit, no tokens, no records -- only the launch bookkeeping below
        if (cta == 0 && tid == 0) {
            *(volatile unsigned*)(p.bar + 2) = g0.y + (unsigned)G * (unsigned)nbar;  // next launch's count base
            for (int i = 0; i < kINumGemm * 64; ++i) p.tcnt[i] = 0u;  // all tile waits are behind us
        }
        tc_fence_before();
        __syncthreads();
        if (warp == 0) tmem_dealloc(sm.tmem, 512);
        return;
    }
    // ---- tail: greedy LM head over h_e and the skipped-layer fill (kv_cache.cpp:222-234) ----
    const int pe = e_out & 1;
    const IterGemm& gf = p.g[kIFill];
    // a layer-level turn decodes a token only for rows that exit here (own accept, or the last
    // layer); every CTA holds the same decisions in sm.status, so this is grid-uniform
    bool any_exit = true;
    if (st.turn_layer > 0 && e_out < L && !st.turn_token) {
        int a = 0;
        for (int b = tid; b < B; b += blockDim.x) a |= sm.status[b];
        any_exit = __syncthreads_or(a) != 0;
    }
    const int n_lm = (st.technique == kSoftmax || !any_exit) ? 0 : tail_lm_units(p);  // softmax: the last check's partials
    const int m2 = 2 * dp / kBM;
    const int fill_units = any_exit ? (L - e_out) * m2 * gf.splits : 0;
    {
        const uint16_t* bsrc = st.hb + (size_t)pe * NR * dp;
        for (int it = cta; it < n_lm + fill_units; it += G) {
            if (it < n_lm) {
                tail_lm_unit(st, sm, ring, p, kseq, tbuf, bsrc, NR, it, B, useq);
            } else {
                const int u = it - n_lm;
                const int mj = u / gf.splits, s = u % gf.splits;  // mj = (jj, m) flattened
                const int j = e_out + 1 + mj / m2, m = mj % m2;
                const int kb0 = s * gf.kb_total / gf.splits, kb1 = (s + 1) * gf.kb_total / gf.splits;
                const uint16_t* a =
                    gf.A + (size_t)((j - 1) * gf.layer_rows + gf.row_off + m) * gf.kb_total * (kBM * kBK);
                unit_ws(sm, ring, p, kseq, a, bsrc, (size_t)NR * kBK, kb0, kb1 - kb0, useq);
                if (warp < 8) {
                    if (gf.splits == 1) epi_fill_direct(st, sm, j, m, B);
                    else epi_partial(sm, p, u, B);
                }
            }
            ++useq;
            tc_fence_before();
            __syncthreads();
        }
    }
    grid_sync(p, st, nbar, g0);
    if (fill_units > 0 && gf.splits > 1) {
        const IterCtx x{e_out + 1, 0, 0};
        reduce_phase<kIFill>(st, sm, p, gf, x, B, 0, (L - e_out) * m2);
    }
    // greedy_token (model.cpp:288-299) + commit + records (engine.cpp:280-306)
    if (warp < 8) {
        const int lane = tid & 31;
        const int cur = iter % st.rec_cap;
        for (int b = cta + G * warp; b < B; b += G * 8) {
            if (st.turn_token) {  // token turn: every row's token; its exit layer back to the host
                const LmPart r = lm_col_warp(st, b);
                if (lane == 0) {
                    rec_rec(st, cur)[b] = r.idx;
                    rec_rec(st, cur)[Bm + b] = st.row_exit[b];
                }
                continue;
            }
            if (st.turn_layer > 0) {
                // turn record: the token of a row that exits at this layer, -1 for a row that
                // continues (its state goes to the per-sequence store for the next layer)
                const bool ex = e_out == L || sm.status[b];
                const LmPart r = ex ? lm_col_warp(st, b) : LmPart{0.f, 0.f, 0.f, -1};
                if (!ex) {
                    const float* src = st.h32 + ((size_t)(e_out & 1) * Bm + b) * dp;
                    float* dst = st.hstore + (size_t)st.row_seq[b] * dp;
                    for (int i = lane * 4; i < dp; i += 128)
                        *reinterpret_cast<float4*>(dst + i) = __ldcg(reinterpret_cast<const float4*>(src + i));
                }
                if (lane == 0) {
                    rec_rec(st, cur)[b] = r.idx;
                    rec_rec(st, cur)[Bm + b] = ex ? e_out : 0;
                    rec_conf(st, cur)[(size_t)(e_out - 1) * Bm + b] = __ldcg(&st.conf[(size_t)(e_out - 1) * Bm + b]);
                }
                continue;
            }
            const LmPart r = lm_col_warp(st, b);
            for (int l = lane; l < L; l += 32)
                rec_conf(st, cur)[(size_t)l * Bm + b] = __ldcg(&st.conf[(size_t)l * Bm + b]);
            if (lane == 0) {
                const int fa = sm.first[b];
                rec_rec(st, cur)[b] = r.idx;
                rec_rec(st, cur)[Bm + b] = fa ? fa : L;
                st.rows.tok[b] = r.idx;       // next input (engine.cpp:304)
                st.rows.pos[b] = sm.pos[b] + 1;  // KvStore::commit (engine.cpp:262-264)
            }
        }
    }
    if (cta == 0 && tid == 0) {
        *(volatile unsigned*)(p.bar + 2) = g0.y + (unsigned)G * (unsigned)nbar;  // next launch's count base
        for (int i = 0; i < kINumGemm * 64; ++i) p.tcnt[i] = 0u;  // all tile waits are behind us
        rec_rec(st, iter % st.rec_cap)[2 * Bm] = e_out;
        *st.out_layer = e_out;
        *st.layer = e_out + 1;
        *st.cur_iter = iter;
        *st.iter_counter = iter + 1;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(sm.tmem, 512);
}

int iter_smem_bytes(int ring_bytes) { return 1024 + ring_bytes + (int)sizeof(IterSmem); }

void launch_iter(const DevState& st, const IterPlan& p, const IterMaps& maps, int grid, cudaStream_t s) {
    const int nj = (st.dm.dp / 8 + 31) / 32;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kIterThreads);
    cfg.dynamicSmemBytes = (size_t)iter_smem_bytes(p.ring_bytes);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (nj <= 1) cudaLaunchKernelEx(&cfg, iter_kernel<1>, st, p, maps);
    else if (nj == 2) cudaLaunchKernelEx(&cfg, iter_kernel<2>, st, p, maps);
    else if (nj == 3) cudaLaunchKernelEx(&cfg, iter_kernel<3>, st, p, maps);
    else cudaLaunchKernelEx(&cfg, iter_kernel<4>, st, p, maps);
    EL_CUDA_LAUNCH_CHECK();
}

int iter_max_ctas_per_sm(const Dims& dm, int ring_bytes) {
    const int nj = (dm.dp / 8 + 31) / 32;
    const int smem = iter_smem_bytes(ring_bytes);
    int n = 0;
    cudaError_t e;
    if (nj <= 1) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, iter_kernel<1>, kIterThreads, smem);
    else if (nj == 2) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, iter_kernel<2>, kIterThreads, smem);
    else if (nj == 3) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, iter_kernel<3>, kIterThreads, smem);
    else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, iter_kernel<4>, kIterThreads, smem);
    return e == cudaSuccess ? n : 0;
}

void init_iter_attributes() {
    const int m = 227 * 1024;
    cudaFuncSetAttribute(iter_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(iter_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(iter_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(iter_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
}
int iter_smem_fixed() { return 1024 + (int)sizeof(IterSmem); }

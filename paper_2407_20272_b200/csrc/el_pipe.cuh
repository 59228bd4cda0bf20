// el_pipe.cuh -- the pipelined decode-iteration kernel (batch 129..256): ONE launch per decode
// iteration like iter_kernel (el_iter.cuh, whose building blocks it reuses), but the CTAs are
// split into two roles that run concurrently, and the batch into two halves H0 = rows
// [0, 128) and H1 = rows [128, B):
//
//   attention CTAs [0, GA):  attn(H0, l) | attn(H1, l) | attn(H0, l+1) | ...      (HBM-bound)
//   GEMM CTAs  [GA, G):      W_o, up, down(H0, l), QKV(H0, l+1) | W_o, up, down(H1, l),
//                            exit decision of layer l, QKV(H1, l+1) | ...          (L2 / tensor)
//
// so the projection GEMMs of one half run under the paged-attention stream of the other half
// instead of after it (in iter_kernel every phase waits for the whole grid).  Hand-offs are
// monotonic arrival counters (release / acquire), not grid barriers: attn(h, l) starts once
// every GEMM CTA has published QKV(h, l); W_o(h, l) once every attention CTA has published
// attn(h, l).  The exit decision of layer l needs both halves' down projections, so QKV(H0, l+1)
// and attn(H0, l+1) run speculatively: when the batch exits at l they are discarded (the
// skipped-layer fill then overwrites the K/V they wrote at layer l+1).  Results are those of
// iter_kernel: the same phases, epilogues and reduction orders per row.
//
// Softmax exit (batch <= 128): the LM-head check of layer l runs on the GEMM CTAs after down(H1, l)
// (transposed pair units on their own ring, then the per-row merge), under attn(H0, l + 1).
// Not in this kernel (iter_kernel serves them): softmax exit at batch > 128, T5 cross-attention,
// batched prefill, layer-level turns.

// control words (unsigned, 128-byte apart) past the grid barrier's: GEMM-group barrier, QKV
// published per half, attention published per half, stop layer
constexpr int kPipeGBar = 4096, kPipeQkv = 4096 + 32, kPipeAtt = 4096 + 96, kPipeStop = 4096 + 160;

__device__ __forceinline__ void pipe_wait_ge(const unsigned* p, unsigned target) {
    const long long t0 = clock64();
    while ((int)(ld_acquire_u32(p) - target) < 0)
        if (clock64() - t0 > EL_SPIN_LIMIT) __trap();
}

// barrier over the GEMM group (n CTAs); k = 1-based count of these barriers in the launch
__device__ __forceinline__ void group_sync(unsigned* cnt, unsigned n, unsigned k) {
    fence_proxy_async_global();
    __syncthreads();
    if (threadIdx.x == 0) {
        red_release_add_u32(cnt, 1u);
        pipe_wait_ge(cnt, n * k);
    }
    __syncthreads();
    fence_proxy_async_global();
}

// this CTA's writes of a phase are done: publish them on a counter
__device__ __forceinline__ void publish(unsigned* cnt) {
    fence_proxy_async_global();
    __syncthreads();
    if (threadIdx.x == 0) red_release_add_u32(cnt, 1u);
}

// EL_DEBUG builds, dbg bit 128: %globaltimer stamps of (layer, half) events by attention CTA 0
// (k = 0 wait done, 1 pass done) and GEMM CTA GA (k = 2 att ready, 3 W_o, 4 up, 5 down, 6 QKV(next))
__device__ __forceinline__ void pipe_stamp(const DevState& st, int layer, int h, int k) {
    if (EL_DEBUG && (EL_DBG(st) & 128) && threadIdx.x == 0 && layer <= 25) {  // (layer 25: the tail)
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        st.dbg_ts[200000 + ((layer - 1) * 2 + h) * 16 + k] = t;
    }
}

template <int NJ>
__global__ void __launch_bounds__(kIterThreads, 1) pipe_kernel(const __grid_constant__ DevState st,
                                                                const __grid_constant__ IterPlan p,
                                                                const __grid_constant__ IterMaps maps) {
    if (st.run_active && *(volatile const int*)st.run_active == 0) return;  // Engine::run chunk over
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    IterSmem& sm = *reinterpret_cast<IterSmem*>(ring + p.ring_bytes);
    float* tbuf = reinterpret_cast<float*>(ring + p.gemm_ring);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int G = (int)gridDim.x, cta = (int)blockIdx.x;
    const Dims& dm = st.dm;
    const int B = st.rows.B, L = dm.L, dp = dm.dp, Bm = dm.Bmax, NR = st.NR;
    const int GA = p.pipe_att_ctas, GG = G - GA;
    // roles interleaved over the CTA indices (so both roles span both dies and every GPC):
    // CTA i runs GEMMs iff floor((i + 1) GG / G) > floor(i GG / G); its rank among its role
    auto gcount = [&](int i) { return (int)(((long long)i * GG) / G); };  // GEMM CTAs in [0, i)
    const bool att_role = gcount(cta + 1) == gcount(cta);
    const int gi = gcount(cta), ai = cta - gi;
    int gemm0 = 0;  // the first GEMM CTA: writes the iteration's exit status
    while (gcount(gemm0 + 1) == gcount(gemm0)) ++gemm0;
    const int H1 = p.bm_grp;  // first row of the second half (128)

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
        for (int s = 0; s < 4; ++s) {
            mbar_init(&sm.full3[s], 1);
            mbar_init(&sm.empty3[s], 1);
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
    const int iter = *st.iter_counter;
    const uint2 g0 = make_uint2(*(volatile unsigned*)(p.bar + 1024), *(volatile unsigned*)(p.bar + 2));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    uint32_t kseq = 0, kseq2 = 0, kseq3 = 0, wseq = 0, useq = 0;
    bool wpf = false;
    int aseq = 0, nbar = 0;
    if (warp == kProducerWarp) {
        attn_prefix_sum(st, sm.att);  // KV blocks per row: fixed for the iteration
        __syncwarp();
    }
    if (cta == 0) pipe_stamp(st, 25, 1, 0);  // (dbg 128: kernel start, embed done)
    // ---- embed (model.cpp:171-183), all CTAs ----
    for (int b = cta; b < B; b += G) {
        const uint16_t* e = st.emb + (size_t)st.rows.tok[b] * dp;
        float* h = st.h32 + (size_t)b * dp;
        for (int i = tid; i < dp; i += blockDim.x) {
            const uint16_t v = e[i];
            st.hb[act_offset(b, i, NR)] = v;
            h[i] = bf16_to_f32(v);
        }
    }
    grid_sync(p, st, nbar, g0);
    if (cta == 0) pipe_stamp(st, 25, 1, 1);

    unsigned* gbar = p.bar + kPipeGBar;
    unsigned* qkv_cnt = p.bar + kPipeQkv;  // [h * 32]
    unsigned* att_cnt = p.bar + kPipeAtt;
    unsigned* stop = p.bar + kPipeStop;
    const int hrows[2] = {H1, B - H1};
    if (att_role) {
        // ================= attention CTAs =================
        for (int layer = 1; layer <= L; ++layer) {
            bool stopped = false;
            for (int h = 0; h < 2; ++h) {
                // QKV(h, layer) published by every GEMM CTA, or the batch stopped before it;
                // thread 0 decides for the CTA
                if (tid == 0) {
                    const long long t0 = clock64();
                    const unsigned target = (unsigned)GG * (unsigned)layer;
                    int go = 0;
                    for (;;) {
                        if ((int)(ld_acquire_u32(qkv_cnt + 32 * h) - target) >= 0) { go = 1; break; }
                        if (ld_acquire_u32(stop) != 0u) break;
                        if (clock64() - t0 > EL_SPIN_LIMIT) __trap();
                    }
                    sm.att.last_flag = go;
                }
                __syncthreads();
                if (!sm.att.last_flag) {
                    stopped = true;  // the decision came first: QKV(h, layer) will never come
                    break;
                }
                fence_proxy_async_global();  // bulk copies read q / the newest K/V next
                if (ai == 0) pipe_stamp(st, layer, h, 0);
                AttnSrc src{st.tables, dm.bpl_max, st.kpool, st.vpool, 0, sm.att.pref, sm.pos, sm.slot, h,
                            nullptr, 0u};
                src.r0 = h ? H1 : 0;
                src.r1 = h ? B : H1;
                src.cta = ai;
                src.ncta = GA;
                // the first half's pass of layer l >= 2 may be speculative (the exit decision of layer
                // l - 1 comes from the GEMM CTAs during it): stop issuing once the batch has stopped
                if (h == 0 && layer > 1) src.abort = stop;
                attn_pass<NJ, true>(st, sm.att, ring, layer, aseq, src, nullptr);
                publish(att_cnt + 32 * h);     // (its __syncthreads orders the consumers' seq_next write)
                aseq = sm.att.seq_next;
                if (ai == 0) pipe_stamp(st, layer, h, 1);
            }
            if (stopped) break;
        }
    } else {
        // ================= GEMM CTAs =================
        unsigned gk = 0;  // group barriers so far
        int down_uses = 0;
        auto qkv_half = [&](int h, int layer) {
            const IterCtx x{layer, (layer - 1) & 1, layer & 1};
            gemm_phase_t<kIQkv>(st, sm, ring, p, maps, kIQkv, x, st.hb + (size_t)x.pin * NR * dp, kseq2, wseq, useq, B,
                                wpf, -1, 0, gi, GG, h);
            publish(qkv_cnt + 32 * h);
        };
        qkv_half(0, 1);
        qkv_half(1, 1);
        int e_out = L;
        for (int layer = 1; layer <= L; ++layer) {
            const IterCtx x{layer, (layer - 1) & 1, layer & 1};
            bool done = false;
            for (int h = 0; h < 2; ++h) {
                const int r0 = h ? H1 : 0;
                // the weights of this W_o unit stream in while the attention of half h finishes
                if (tid == kProducerWarp * 32 && !wpf) wpf = bm_prefetch(sm, ring, p, maps, kIWo, layer, gi, h, GG);
                if (tid == 0) pipe_wait_ge(att_cnt + 32 * h, (unsigned)GA * (unsigned)layer);
                __syncthreads();
                fence_proxy_async_global();
                if (gi == 0) pipe_stamp(st, layer, h, 2);
                // W_o + residual (model.cpp:245-253), up + ReLU (255-260)
                gemm_phase_t<kIWo, true>(st, sm, ring, p, maps, kIWo, x, st.att_b, kseq2, wseq, useq, B, wpf, kIUp, layer,
                                   gi, GG, h, h);
                group_sync(gbar, (unsigned)GG, ++gk);
                if (gi == 0) pipe_stamp(st, layer, h, 3);
                gemm_phase_t<kIUp>(st, sm, ring, p, maps, kIUp, x, st.mid_b, kseq2, wseq, useq, B, wpf, -1, layer, gi,
                                   GG, h);
                group_sync(gbar, (unsigned)GG, ++gk);
                if (gi == 0) pipe_stamp(st, layer, h, 4);
                // down + residual (261-270) + exit-check partial dots of these rows (split-K, fused reduce)
                // next layer's QKV weights: L2 prefetch with streamed weights only (a slab prefetch
                // would land in the region the down phase's split-K ring uses)
                if (p.bm_wstream && tid == kProducerWarp * 32 && layer < L)
                    bm_prefetch(sm, ring, p, maps, kIQkv, layer + 1, gi, h, GG);
                // (3 pieces in flight per warp -- one round of loads for a tile's ~21 pieces instead of
                //  two -- spills at the 168-register cap of 288 threads: -1 % at c5)
                gemm_phase_fused<kIDown>(st, sm, ring, p, kIDown, x, st.up_b + (size_t)r0 * kBK, kseq, useq, hrows[h],
                                         ++down_uses, gi, GG, r0, H1);
                group_sync(gbar, (unsigned)GG, ++gk);
                if (gi == 0) pipe_stamp(st, layer, h, 5);
                if (h == 1) {
                    if (st.technique == kSoftmax) {
                        // softmax check (exit_policy.cpp:57-72) on the GEMM CTAs while the attention
                        // CTAs run the next layer's first half speculatively: the LM head over h_l of
                        // both halves on pair units (their own ring), then each row's merge
                        const uint16_t* bsrc = st.hb + (size_t)x.pout * NR * dp;
                        const uint64_t lpol = p.lm_keep ? kL2EvictLast : kL2EvictFirst;
                        const uint32_t pstride = 2u * kAStage + (uint32_t)p.n_pad * 128u;
                        float* tb2 = reinterpret_cast<float*>(ring + (size_t)p.lm_stages * pstride);
                        for (int u = gi; 2 * u < p.lm_tiles; u += GG) {
                            const int t0 = 2 * u, na = min(2, p.lm_tiles - t0);
                            unit_lm_pair(sm, ring, p, kseq3, st.lm + (size_t)t0 * (dp / kBK) * (kBM * kBK), na, bsrc,
                                         (size_t)NR * kBK, dp / kBK, useq, lpol, p.lm_pair == 2, 0, sm.full3,
                                         sm.empty3, p.lm_stages);
                            if (p.lm_pair == 2) {
                                if (warp < 8) epi_lm_tr<true>(st, sm, t0, na, B);
                            } else if (warp < 8) {
                                epi_lm_full(st, sm, tb2, t0, B);
                                if (na > 1) {
                                    named_bar(2, 256);
                                    epi_lm_full(st, sm, tb2, t0 + 1, B, 256u);
                                }
                            }
                            ++useq;
                            tc_fence_before();
                            __syncthreads();
                        }
                        group_sync(gbar, (unsigned)GG, ++gk);
                        if (warp < 8)
                            for (int b = gi + GG * warp; b < B; b += GG * 8) {
                                const LmPart r = lm_col_warp(st, b);
                                if ((tid & 31) == 0) {
                                    const float gap = (r.m2 == -INFINITY) ? 1.f : -expm1f(r.m2 - r.m1);
                                    const float conf = gap / r.s;
                                    st.conf[(size_t)(layer - 1) * Bm + b] = conf;
                                    st.accept[b] = (double)conf > st.lambdas[layer - 1];
                                }
                            }
                        group_sync(gbar, (unsigned)GG, ++gk);
                    }
                    // exit decision of this layer for the whole batch (engine.cpp:225-258)
                    if (exit_decide(st, sm, layer, B, dp / kBM, gemm0)) {
                        e_out = layer;
                        done = true;
                        if (tid == 0 && gi == 0) st_release_u32(stop, (unsigned)layer);
                        break;
                    }
                }
                if (layer < L) qkv_half(h, layer + 1);  // (half 0: speculative until the decision)
                if (gi == 0) pipe_stamp(st, layer, h, 6);
            }
            if (done) break;
        }
        (void)e_out;
    }
    // ---- everything of the layer loop is published: the stop layer is the output layer ----
    grid_sync(p, st, nbar, g0);
    if (cta == 0) pipe_stamp(st, 25, 0, 0);
    const int e_out = (int)ld_acquire_u32(stop);
    if (cta == 0 && tid == 0) {  // nobody reads the hand-off words any more: zero them for the next launch
        for (int k = 0; k < 192; ++k) p.bar[kPipeGBar + k] = 0u;
    }
    // an aborted speculative pass leaves its rows' segment counts partial: every attention pass is
    // over, so clear them for the next launch (completed rows were cleared by their combine)
    if (cta == 1 % G)
        for (int b = tid; b < B; b += blockDim.x) st.attn_cnt[b] = 0;

    // ---- tail: greedy LM head over h_e and the skipped-layer fill (kv_cache.cpp:222-234), all CTAs ----
    const int pe = e_out & 1;
    const IterGemm& gf = p.g[kIFill];
    const int n_lm = st.technique == kSoftmax ? 0 : tail_lm_units(p);  // softmax: the last check's partials
    const int m2 = 2 * dp / kBM;
    const int fill_units = (L - e_out) * m2 * gf.splits;
    {
        const uint16_t* bsrc = st.hb + (size_t)pe * NR * dp;
        int un = 0;  // (dbg 128: per-unit stamps of CTAs 0 / 1 -- start, accumulator ready, epilogue done)
        auto ustamp = [&](int k) {
            if (EL_DEBUG && (EL_DBG(st) & 128) && cta < 2 && tid == 0 && un < 8) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
                st.dbg_ts[201000 + cta * 32 + un * 4 + k] = t;
            }
        };
        for (int it = cta; it < n_lm + fill_units; it += G, ++un) {
            ustamp(0);
            if (it < n_lm) {
                tail_lm_unit(st, sm, ring, p, kseq, tbuf, bsrc, NR, it, B, useq);
                ustamp(1);
            } else {
                const int u = it - n_lm;
                const int mj = u / gf.splits, s = u % gf.splits;
                const int j = e_out + 1 + mj / m2, m = mj % m2;
                const int kb0 = s * gf.kb_total / gf.splits, kb1 = (s + 1) * gf.kb_total / gf.splits;
                const uint16_t* a =
                    gf.A + (size_t)((j - 1) * gf.layer_rows + gf.row_off + m) * gf.kb_total * (kBM * kBK);
                unit_ws(sm, ring, p, kseq, a, bsrc, (size_t)NR * kBK, kb0, kb1 - kb0, useq);
                ustamp(1);
                if (warp < 8) {
                    if (gf.splits == 1) epi_fill_direct(st, sm, j, m, B);
                    else epi_partial(sm, p, u, B);
                }
            }
            ++useq;
            tc_fence_before();
            __syncthreads();
            ustamp(2);
        }
    }
    if (cta == 0) pipe_stamp(st, 25, 0, 1);
    grid_sync(p, st, nbar, g0);
    if (cta == 0) pipe_stamp(st, 25, 0, 2);
    if (fill_units > 0 && gf.splits > 1) {
        const IterCtx x{e_out + 1, 0, 0};
        reduce_phase<kIFill>(st, sm, p, gf, x, B, 0, (L - e_out) * m2);
    }
    // greedy_token (model.cpp:288-299) + commit + records (engine.cpp:280-306); the exit status
    // lives in the GEMM CTAs: first accepts come from global memory
    if (warp < 8) {
        const int lane = tid & 31;
        const int cur = iter % st.rec_cap;
        for (int b = cta + G * warp; b < B; b += G * 8) {
            const LmPart r = lm_col_warp(st, b);
            for (int l = lane; l < L; l += 32)
                rec_conf(st, cur)[(size_t)l * Bm + b] = __ldcg(&st.conf[(size_t)l * Bm + b]);
            if (lane == 0) {
                const int fa = __ldcg(&st.first_accept[b]);
                rec_rec(st, cur)[b] = r.idx;
                rec_rec(st, cur)[Bm + b] = fa ? fa : L;
                st.rows.tok[b] = r.idx;
                st.rows.pos[b] = sm.pos[b] + 1;
            }
        }
    }
    if (cta == 0) pipe_stamp(st, 25, 0, 3);
    if (cta == 0 && tid == 0) {  // (kernel end: the stamp after the records below)
        *(volatile unsigned*)(p.bar + 2) = g0.y + (unsigned)G * (unsigned)nbar;  // next launch's count base
        for (int i = 0; i < kINumGemm * 64; ++i) p.tcnt[i] = 0u;
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

void launch_pipe(const DevState& st, const IterPlan& p, const IterMaps& maps, int grid, cudaStream_t s) {
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
    if (nj <= 1) cudaLaunchKernelEx(&cfg, pipe_kernel<1>, st, p, maps);
    else if (nj == 2) cudaLaunchKernelEx(&cfg, pipe_kernel<2>, st, p, maps);
    else if (nj == 3) cudaLaunchKernelEx(&cfg, pipe_kernel<3>, st, p, maps);
    else cudaLaunchKernelEx(&cfg, pipe_kernel<4>, st, p, maps);
    EL_CUDA_LAUNCH_CHECK();
}

void init_pipe_attributes() {
    const int m = 227 * 1024;
    cudaFuncSetAttribute(pipe_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(pipe_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(pipe_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
    cudaFuncSetAttribute(pipe_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, m);
}

// 2-CTA (cta_group::2) variant of the grouped GEMM: a cluster pair of CTAs on two SMs
// computes a 256 x BN tile with one tcgen05.mma.cta_group::2 stream (M = 256).
//   * each CTA stages its 128 rows of A and its BN/2 rows (K-major) / columns
//     (MN-major) of B, so per-SM operand traffic drops by a quarter vs the 1-CTA tile
//     (up to 6 stages of 32 KiB at BN = 256, whatever fits next to the epilogue staging);
//   * both producers count their TMA bytes on the LEADER's full barrier;
//   * the leader's single MMA thread issues for the pair and commits with a
//     cluster multicast to both CTAs' empty / tmem-full barriers;
//   * each CTA's epilogue drains its own TMEM (its 128 rows x BN columns) and
//     arrives on the leader's tmem-empty barrier.
// Group m_tiles count 256-row pair tiles here. Epilogues see mt = 2*pair_tile + rank,
// i.e. the same 128-row tile index as in the 1-CTA kernel.
#pragma once

#include "grouped_gemm.cuh"

namespace spes_dev {

template <int BN, int SLOTS = 1, int STAGED = 0>
struct Gemm2Cfg {
    static constexpr int BNH = BN / 2;
    static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
    static constexpr int B_BYTES = BNH * GEMM_BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int FIXED = 1024 + 256 + GEMM_TABLE_BYTES;
    // staged epilogue input (1024-aligned after the epilogue staging slots)
    static constexpr int EPI_BYTES = (epi_stage_bytes(SLOTS) + 1023) / 1024 * 1024 + STAGED;
    static constexpr int FIT = (GEMM_SMEM_MAX - FIXED - EPI_BYTES) / STAGE_BYTES;
    static constexpr int STAGES = FIT > 6 ? 6 : FIT;
    static_assert(STAGES >= 2, "smem ring too shallow");
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + FIXED + EPI_BYTES;
};

template <int BN, class Epi, bool A_MN = false, bool B_MN = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    grouped_gemm_2cta_kernel(const __grid_constant__ CUtensorMap mapA,
                             const __grid_constant__ CUtensorMap mapB,
                             const GemmGroup* __restrict__ groups, int num_groups,
                             const int* __restrict__ total_tiles_ptr, int max_tiles, Epi epi) {
    constexpr int STAGED = EpiStaged<Epi>::bytes;
    using C = Gemm2Cfg<BN, Epi::SLOTS, STAGED>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + C::STAGES;
    uint64_t* tfull = bars + 2 * C::STAGES;
    uint64_t* tempty = bars + 2 * C::STAGES + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4);
    int* s_ts = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(bars) + 256);
    int* s_nkb = s_ts + GEMM_MAX_GROUPS;
    uint8_t* s_epi = reinterpret_cast<uint8_t*>(bars) + 256 + GEMM_TABLE_BYTES;
    // staged epilogue input: two buffers after the 1024-aligned end of the staging slots
    uint64_t* sfull = tempty + 2 + 1;   // past tmem_slot's 8 bytes; up to 4 buffers
    uint64_t* sempty = sfull + 4;
    uint8_t* s_stage = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(s_epi + epi_stage_bytes(Epi::SLOTS)) + 1023) &
        ~static_cast<uintptr_t>(1023));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1;
    const int npairs = gridDim.x >> 1;

    load_group_table(groups, num_groups, s_ts, s_nkb);
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&mapA);
        tma_prefetch_desc(&mapB);
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 2);   // one expect_tx arrival per CTA (leader's copy used)
            mbar_init(&empty[s], 1);  // multicast commit of the leader's MMAs
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 16);  // 8 epilogue warps x 2 CTAs (leader's copy used)
        }
        if constexpr (STAGED > 0) {
            static_assert(Epi::STAGE_BUFS <= 4, "staging barriers: up to 4 buffers");
            for (int b = 0; b < Epi::STAGE_BUFS; ++b) {
                mbar_init(&sfull[b], 1);   // this CTA's warp 3 (expect_tx)
                mbar_init(&sempty[b], EpiStageArrivals<Epi>::count);  // epilogue releases
            }
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    int total = *total_tiles_ptr;
    if (total > max_tiles) total = max_tiles;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair; t < total; t += npairs) {
                const int gi = find_group(s_ts, num_groups, t);
                const GemmGroup& g = groups[gi];
                const int local = t - g.tile_start;
                const int mt = local / g.n_tiles, nt = local % g.n_tiles;
                const int arow = g.a_row0 + mt * 2 * GEMM_BM + static_cast<int>(rank) * GEMM_BM;
                const int brow = g.b_row0 + nt * BN + static_cast<int>(rank) * C::BNH;
                const int nkb = g.k_len / GEMM_BK;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * C::STAGE_BYTES;
                    uint8_t* sb = sa + C::A_BYTES;
                    const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
                    if (leader)  // the leader expects both CTAs' bytes on its own barrier
                        mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
                    else
                        mbar_arrive_remote(fb);
                    const int kca = g.k0 + kb * GEMM_BK;
                    const int kcb = g.bk0 + kb * GEMM_BK;
                    if constexpr (!A_MN) {
                        tma_load_2d_pair(&mapA, fb, sa, kca, arow);
                    } else {
#pragma unroll
                        for (int i = 0; i < GEMM_BM / 64; ++i)
                            tma_load_2d_pair(&mapA, fb, sa + i * 8192, arow + 64 * i, kca);
                    }
                    if constexpr (!B_MN) {
                        tma_load_2d_pair(&mapB, fb, sb, kcb, brow);
                    } else {
#pragma unroll
                        for (int i = 0; i < C::BNH / 64; ++i)
                            tma_load_2d_pair(&mapB, fb, sb + i * 8192, brow + 64 * i, kcb);
                    }
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            constexpr uint32_t idesc = idesc_bf16_f32(2 * GEMM_BM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = pair; t < total; t += npairs, ++it) {
                const int gi = find_group(s_ts, num_groups, t);
                const int nkb = s_nkb[gi];
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t dtmem = tmem_base + acc * BN;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
                    const uint32_t sb = sa + C::A_BYTES;
                    const uint64_t adesc =
                        A_MN ? desc_mnmajor_sw128(sa, 8192) : desc_kmajor_sw128(sa);
                    const uint64_t bdesc =
                        B_MN ? desc_mnmajor_sw128(sb, 8192) : desc_kmajor_sw128(sb);
                    constexpr uint64_t astep = A_MN ? 128 : 2, bstep = B_MN ? 128 : 2;
#pragma unroll
                    for (int k = 0; k < GEMM_BK / 16; ++k)
                        umma_bf16_pair(dtmem, adesc + astep * k, bdesc + bstep * k, idesc,
                                       (kb | k) != 0 ? 1u : 0u);
                    umma_commit_pair(&empty[stage]);
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (nkb > 0) {
                    umma_commit_pair(&tfull[acc]);
                } else {
                    mbar_arrive(&tfull[acc]);
                    mbar_arrive_cluster(mapa_shared(smem_u32(&tfull[acc]), 1));
                }
            }
        }
    } else if (warp == 3) {
        if constexpr (STAGED > 0) {  // the epilogue's input pieces, ahead of the epilogue
            if (lane == 0) {
                uint32_t cnt = 0;
                for (int t = pair; t < total; t += npairs) {
                    const int gi = find_group(s_ts, num_groups, t);
                    const GemmGroup& g = groups[gi];
                    const int local = t - g.tile_start;
                    const int mt = local / g.n_tiles, nt = local % g.n_tiles;
                    constexpr int NB = Epi::STAGE_BUFS, PB = STAGED / NB;
                    for (int pc = 0; pc < Epi::PIECES; ++pc, ++cnt) {
                        const int b = cnt % NB;
                        mbar_wait(&sempty[b], ((cnt / NB) & 1) ^ 1);
                        mbar_arrive_expect_tx(&sfull[b], PB);
                        epi.stage_load(g, 2 * mt + static_cast<int>(rank), nt, pc, s_stage + b * PB,
                                       &sfull[b]);
                    }
                }
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        const int half = (warp - 4) >> 2;
        const int r = q * 32 + lane;
        EpiOut out{s_epi + (warp - 4) * Epi::SLOTS * EPI_SLOT_BYTES, lane};
        StageCtx sc{s_stage, sfull, sempty, 0};
        int it = 0;
        for (int t = pair; t < total; t += npairs, ++it) {
            const int gi = find_group(s_ts, num_groups, t);
            const GemmGroup& g = groups[gi];
            const int local = t - g.tile_start;
            const int mt = local / g.n_tiles, nt = local % g.n_tiles;
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            if (t + npairs < total) {  // warm L2 for the next tile's epilogue inputs
                const int tn = t + npairs;
                const GemmGroup& gn = groups[find_group(s_ts, num_groups, tn)];
                const int ln = tn - gn.tile_start;
                epi.prefetch(gn, 2 * (ln / gn.n_tiles) + static_cast<int>(rank), ln % gn.n_tiles, r,
                             half);
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
            if constexpr (STAGED > 0)
                epi(g, 2 * mt + static_cast<int>(rank), nt, r, taddr, g.k_len == 0, half, out, sc);
            else
                epi(g, 2 * mt + static_cast<int>(rank), nt, r, taddr, g.k_len == 0, half, out);
            tc_fence_before();
            __syncwarp();
            // relaxed remote arrive: only the (already waited) TMEM reads need ordering
            if (lane == 0) mbar_arrive_remote(mapa_shared(smem_u32(&tempty[acc]), 0));
        }
        out.drain();
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
    }
}

}  // namespace spes_dev

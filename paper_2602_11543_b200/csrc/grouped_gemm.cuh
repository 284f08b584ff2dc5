// Grouped BF16 GEMM on the sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
//   D_g[m, n] = sum_k A[a_row0 + m, k0 + k] * B[b_row0 + n, k0 + k]     (both K-major)
//
// for every group g of a device-resident group table. This one kernel carries
// all dense contractions of the SPES local step:
//   * expert forward  gate||up  (groups = experts, rows = routed tokens),
//   * expert forward  down,
//   * expert backward dH and dX (all routed experts, frozen ones included),
//   * expert backward dW (owned experts only; K = that expert's routed tokens),
//   * head forward / dX / dW.
// Group sizes come from routing counts that live on the device, so the tile
// space is read from device memory and the launch never syncs with the host.
//
// Structure (one CTA per SM, persistent):
//   warp 0  : TMA producer       (one elected lane)
//   warp 1  : MMA issuer         (one elected lane, tcgen05.mma cta_group::1, M=128)
//   warp 2  : TMEM allocator
//   warps 4-11: epilogue, two warps per TMEM lane quarter, each on half of the tile's
//               columns (TMEM -> registers -> fused epilogue -> smem transpose ->
//               full-line global stores, EpiOut)
// Pipelines: STAGES-deep smem ring (full/empty mbarriers) and a 2-deep TMEM
// accumulator ring (tmem_full/tmem_empty) so the epilogue of tile i overlaps
// the MMAs of tile i+1.
#pragma once

#include "sm100_primitives.cuh"

namespace spes_dev {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int GEMM_THREADS = 384;  // 4 control warps + 8 epilogue warps

// ---- epilogue output staging --------------------------------------------------------
// Direct 16-byte stores from a row-per-lane layout send 32 half-sector requests to L2 per
// warp instruction, which capped the epilogue at ~11 GB/s per SM. Instead each lane
// writes its row piece (<= 128 B) into its smem row, and the warp copies the 32 pieces
// out row-major: one STG.128 instruction then covers 4 whole 128-byte rows (8 lanes per
// row, row addresses exchanged by shuffles), i.e. full-line writes.
constexpr int EPI_SLOT_PITCH = 144;  // 128 B + 16 B pad: STS.128 across rows conflict-free
constexpr int EPI_SLOT_BYTES = 32 * EPI_SLOT_PITCH;  // one 32-row slot of a warp
constexpr int EPI_WARPS = 8;
// staging bytes of a CTA when every epilogue warp owns `slots` slots
constexpr int epi_stage_bytes(int slots) { return EPI_WARPS * slots * EPI_SLOT_BYTES; }
constexpr int GEMM_SMEM_MAX = 232448;  // 227 KiB opt-in per CTA

struct EpiOut {
    uint8_t* base;  // this warp's slots: slot s, lane r at base + s * SLOT_BYTES + r * PITCH
    int lane;
    __device__ __forceinline__ uint8_t* row_of(int s, int r) const {
        return base + s * EPI_SLOT_BYTES + r * EPI_SLOT_PITCH;
    }
    __device__ __forceinline__ uint4* my_row(int s) const {
        return reinterpret_cast<uint4*>(row_of(s, lane));
    }
    // warp-collective: slot s (rows = lanes) -> the 32 destinations (each lane passes its
    // own, 16-byte aligned), row-major so one STG.128 covers 4 whole 128-byte rows
    template <int N16>
    __device__ __forceinline__ void rows_store(int s, void* gdst) const {
        static_assert(N16 == 4 || N16 == 8, "row pieces of 64 or 128 bytes");
        __syncwarp();
        constexpr int RPI = 32 / N16;
        const int sub = lane % N16, r0 = lane / N16;
        const unsigned long long ga = reinterpret_cast<unsigned long long>(gdst);
#pragma unroll
        for (int i = 0; i < N16; ++i) {
            const int rr = i * RPI + r0;
            const unsigned long long a = __shfl_sync(0xffffffffu, ga, rr);
            reinterpret_cast<uint4*>(a)[sub] = reinterpret_cast<const uint4*>(row_of(s, rr))[sub];
        }
        __syncwarp();
    }
    // warp-collective: each lane's row piece (registers) -> its destination, via slot s
    template <int N16>
    __device__ __forceinline__ void put(void* gdst, const uint4* v, int s = 0) const {
        uint4* row = my_row(s);
#pragma unroll
        for (int i = 0; i < N16; ++i) row[i] = v[i];
        rows_store<N16>(s, gdst);
    }
    __device__ __forceinline__ void put_f32x32(float* gdst, const float (&v)[32]) const {
        put<8>(gdst, reinterpret_cast<const uint4*>(v));
    }
    // warp-collective: the 32 sources -> slot s rows, row-major 16-byte cp.async (whole
    // 128-byte rows per instruction); complete with rows_wait()
    template <int N16>
    __device__ __forceinline__ void rows_load_async(int s, const void* gsrc) const {
        constexpr int RPI = 32 / N16;
        const int sub = lane % N16, r0 = lane / N16;
        const unsigned long long ga = reinterpret_cast<unsigned long long>(gsrc);
#pragma unroll
        for (int i = 0; i < N16; ++i) {
            const int rr = i * RPI + r0;
            const unsigned long long a = __shfl_sync(0xffffffffu, ga, rr);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             smem_u32(row_of(s, rr) + 16 * sub)),
                         "l"(a + 16 * sub)
                         : "memory");
        }
    }
    __device__ __forceinline__ void rows_wait() const {
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    // synchronous variant in two halves so several pieces can be in flight: load_rows
    // issues the row-major loads into registers, land_rows transposes them through slot 0
    template <int N16>
    __device__ __forceinline__ void load_rows(const void* gsrc, uint4 (&tmp)[N16]) const {
        constexpr int RPI = 32 / N16;
        const int sub = lane % N16, r0 = lane / N16;
        const unsigned long long ga = reinterpret_cast<unsigned long long>(gsrc);
#pragma unroll
        for (int i = 0; i < N16; ++i) {
            const unsigned long long a = __shfl_sync(0xffffffffu, ga, i * RPI + r0);
            tmp[i] = __ldg(reinterpret_cast<const uint4*>(a) + sub);
        }
    }
    template <int N16>
    __device__ __forceinline__ void land_rows(const uint4 (&tmp)[N16], uint4* v) const {
        constexpr int RPI = 32 / N16;
        const int sub = lane % N16, r0 = lane / N16;
#pragma unroll
        for (int i = 0; i < N16; ++i)
            reinterpret_cast<uint4*>(row_of(0, i * RPI + r0))[sub] = tmp[i];
        __syncwarp();
        const uint4* row = my_row(0);
#pragma unroll
        for (int i = 0; i < N16; ++i) v[i] = row[i];
        __syncwarp();
    }
    // outstanding bulk (TMA) stores of this lane complete before the CTA's smem goes away
    __device__ __forceinline__ void drain() const {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
};

constexpr int GEMM_MAX_GROUPS = 512;
constexpr int GEMM_TABLE_BYTES = 8 * GEMM_MAX_GROUPS;

struct GemmGroup {
    int32_t a_row0;      // first row of this group's A tile space
    int32_t b_row0;      // first row of this group's B tile space
    int32_t k0;          // K offset (elements) in both A and B
    int32_t k_len;       // K extent (multiple of 64; 0 => result is zero)
    int32_t m_tiles;     // tiles of 128 rows
    int32_t n_tiles;     // tiles of BN columns
    int32_t tile_start;  // exclusive prefix of m_tiles*n_tiles over groups
    int32_t bk0;         // K offset (elements) in B
    int64_t out_row0;    // epilogue-defined output row offset
    int64_t ldo;         // epilogue-defined leading dimension
    void* out0;          // epilogue-defined outputs
    void* out1;
    int32_t aux;         // epilogue-defined (fused optimizer: shadow slot)
    int32_t _pad;
};

// Epilogues may stage an input tile through shared memory by TMA (StagedEpi below): they
// declare STAGED_BYTES (two buffers' worth, each 1024-byte aligned halves) and the pair
// kernel's warp 3 loads each piece ahead of the epilogue.
template <class E, class = void>
struct EpiStaged {
    static constexpr int bytes = 0;
};
template <class E>
struct EpiStaged<E, decltype(void(E::STAGED_BYTES))> {
    static constexpr int bytes = E::STAGED_BYTES;
};
// arrivals that free a staging buffer (default: each of the 8 epilogue warps once)
template <class E, class = void>
struct EpiStageArrivals {
    static constexpr int count = 8;
};
template <class E>
struct EpiStageArrivals<E, decltype(void(E::STAGE_ARRIVALS))> {
    static constexpr int count = E::STAGE_ARRIVALS;
};
// the epilogue side of the staging ring (Epi::STAGE_BUFS buffers of STAGED_BYTES /
// STAGE_BUFS bytes): buffer b holds a piece; full[b] completes when its TMA bytes landed,
// empty[b] when all 8 epilogue warps of the CTA have used it
struct StageCtx {
    uint8_t* base;
    uint64_t* full;
    uint64_t* empty;
    uint32_t cnt;  // pieces consumed so far by this warp (same sequence in every warp)
};

template <int BN, int SLOTS = 1>
struct GemmCfg {
    static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
    static constexpr int B_BYTES = BN * GEMM_BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int FIXED = 1024 /*align*/ + 256 /*barriers*/ + GEMM_TABLE_BYTES;
    static constexpr int EPI_BYTES = epi_stage_bytes(SLOTS);
    static constexpr int FIT = (GEMM_SMEM_MAX - FIXED - EPI_BYTES) / STAGE_BYTES;
    static constexpr int STAGES = FIT > 6 ? 6 : FIT;
    static_assert(STAGES >= 2, "smem ring too shallow");
    static constexpr int TMEM_COLS = 2 * BN;  // two accumulator buffers
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + FIXED + EPI_BYTES;
};

// Per-CTA copy of the group table's tile_start / k-block counts in shared memory: the
// tile -> group lookup is a binary search over smem instead of a chain of dependent
// global loads in the single MMA-issuing thread (which starved the tensor pipe).
__device__ __forceinline__ void load_group_table(const GemmGroup* __restrict__ groups, int n,
                                                 int* ts, int* nkb) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        ts[i] = groups[i].tile_start;
        nkb[i] = groups[i].k_len / GEMM_BK;
    }
}
// largest g with ts[g] <= tile (zero-tile groups share their successor's tile_start)
__device__ __forceinline__ int find_group(const int* ts, int n, int tile) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ts[mid] <= tile)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

// Epi must provide:
//   __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
//                              bool empty, int half, EpiOut& out) const;
//   __device__ void prefetch(const GemmGroup& g, int mt, int nt, int r, int half) const;
//   static constexpr int SLOTS;  (32-row smem staging slots per epilogue warp)
//     (L2 warm-up of epilogue inputs of the tile this thread handles next; may be empty)
// r = row within the 128-row tile handled by this thread; taddr = TMEM address of
// (lane r, column 0) of this tile's accumulator; empty => k_len == 0 (result is 0).
//
// Operand majors (independent for A and B):
//   K-major : X [rows x K] row-major (K contiguous); one box (k, row) of 64 x rows.
//   MN-major: X [K x cols] row-major (M / N contiguous); row0 is a column offset and
//             the K offset a row index; boxes of 64 x 64 (weight-gradient form
//             D = A^T B over K = tokens, and row-major weights as B).
// A's K offset is g.k0, B's is g.bk0.
template <int BN, class Epi, bool A_MN = false, bool B_MN = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                        const __grid_constant__ CUtensorMap mapB,
                        const GemmGroup* __restrict__ groups, int num_groups,
                        const int* __restrict__ total_tiles_ptr, int max_tiles, Epi epi) {
    using C = GemmCfg<BN, Epi::SLOTS>;
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

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    load_group_table(groups, num_groups, s_ts, s_nkb);
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&mapA);
        tma_prefetch_desc(&mapB);
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 256);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    int total = *total_tiles_ptr;
    if (total > max_tiles) total = max_tiles;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const int gi = find_group(s_ts, num_groups, t);
                const GemmGroup& g = groups[gi];
                const int local = t - g.tile_start;
                const int mt = local / g.n_tiles, nt = local % g.n_tiles;
                const int arow = g.a_row0 + mt * GEMM_BM;
                const int brow = g.b_row0 + nt * BN;
                const int nkb = g.k_len / GEMM_BK;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * C::STAGE_BYTES;
                    uint8_t* sb = sa + C::A_BYTES;
                    mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
                    const int kca = g.k0 + kb * GEMM_BK;
                    const int kcb = g.bk0 + kb * GEMM_BK;
                    if constexpr (!A_MN) {
                        tma_load_2d(&mapA, &full[stage], sa, kca, arow);
                    } else {
#pragma unroll
                        for (int i = 0; i < GEMM_BM / 64; ++i)
                            tma_load_2d(&mapA, &full[stage], sa + i * 8192, arow + 64 * i, kca);
                    }
                    if constexpr (!B_MN) {
                        tma_load_2d(&mapB, &full[stage], sb, kcb, brow);
                    } else {
#pragma unroll
                        for (int i = 0; i < BN / 64; ++i)
                            tma_load_2d(&mapB, &full[stage], sb + i * 8192, brow + 64 * i, kcb);
                    }
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(GEMM_BM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
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
                    // K-major: advance 16 elements = 32 B inside the 128 B swizzle row;
                    // MN-major: advance 16 K rows = 2 KiB (two 8-row swizzle atoms)
                    const uint64_t adesc = A_MN ? desc_mnmajor_sw128(sa, 8192) : desc_kmajor_sw128(sa);
                    const uint64_t bdesc = B_MN ? desc_mnmajor_sw128(sb, 8192) : desc_kmajor_sw128(sb);
                    constexpr uint64_t astep = A_MN ? 128 : 2, bstep = B_MN ? 128 : 2;
#pragma unroll
                    for (int k = 0; k < GEMM_BK / 16; ++k)
                        umma_bf16(dtmem, adesc + astep * k, bdesc + bstep * k, idesc,
                                  (kb | k) != 0 ? 1u : 0u);
                    umma_commit(&empty[stage]);
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (nkb > 0)
                    umma_commit(&tfull[acc]);
                else
                    mbar_arrive(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;           // TMEM lane quarter this warp may access
        const int half = (warp - 4) >> 2;  // which half of the tile's columns
        const int r = q * 32 + lane;
        EpiOut out{s_epi + (warp - 4) * Epi::SLOTS * EPI_SLOT_BYTES, lane};
        int it = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
            const int gi = find_group(s_ts, num_groups, t);
            const GemmGroup& g = groups[gi];
            const int local = t - g.tile_start;
            const int mt = local / g.n_tiles, nt = local % g.n_tiles;
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            if (t + static_cast<int>(gridDim.x) < total) {  // warm L2 for the next tile's inputs
                const int tn = t + gridDim.x;
                const GemmGroup& gn = groups[find_group(s_ts, num_groups, tn)];
                const int ln = tn - gn.tile_start;
                epi.prefetch(gn, ln / gn.n_tiles, ln % gn.n_tiles, r, half);
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
            epi(g, mt, nt, r, taddr, g.k_len == 0, half, out);
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
        }
        out.drain();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, C::TMEM_COLS);
    }
}

// Load 32 accumulator columns (or zeros for an empty K range) as floats.
__device__ __forceinline__ void acc_load32(uint32_t taddr, bool empty, float (&v)[32]) {
    if (empty) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
        return;
    }
    uint32_t u[32];
    tmem_ld32(taddr, u);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(u[i]);
}

// Plain FP32 store: out0[(out_row0 + mt*128 + r) * ldo + nt*BN + c].
template <int BN>
struct EpiStoreF32 {
    static constexpr int SLOTS = 1;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out) const {
        float* dst = static_cast<float*>(g.out0) +
                     (g.out_row0 + static_cast<int64_t>(mt) * GEMM_BM + r) * g.ldo +
                     static_cast<int64_t>(nt) * BN;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            float v[32];
            acc_load32(taddr + c, empty, v);
            out.put_f32x32(dst + c, v);
        }
    }
};

}  // namespace spes_dev

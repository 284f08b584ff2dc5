// Fused epilogues of the grouped tcgen05 GEMM (grouped_gemm.cuh) and their launchers.
//
//   EpiSwiGLU   expert forward gate||up: accumulator columns [0,128) are gate,
//               [128,256) the matching up columns; writes Hact = silu(G)*U (bf16) and,
//               in the GU buffer, the backward factors A = U*silu'(G) (gate slots) and
//               B = silu(G) (up slots) as bf16.
//   EpiStoreF32 plain fp32 tile store (expert down-proj Y, dX, head logits / dh,
//               dWd and dHead straight into the gradient buffer).
//   EpiDSwiGLU  expert backward: dHact -> (dG, dU) = (dH*A, dH*B) from the saved
//               factors, written as dGU (bf16) for the dX and dW GEMMs.
// All epilogues hand their row pieces to EpiOut (grouped_gemm.cuh): an smem transpose so
// that each warp store instruction writes whole 128-byte rows.
//   EpiGradW1   dW of gate||up straight into the fp32 wg / wu gradient blocks.
// Weight-gradient GEMMs read the row-major activations directly as MN-major
// operands (grouped_gemm_kernel<..., MN=true>): no transposed copies are made.
#include "common.cuh"
#include "grouped_gemm.cuh"
#include "grouped_gemm_2cta.cuh"
#include "kernels.h"

#include <stdexcept>

namespace spes_k {

using namespace spes_dev;

__device__ __forceinline__ void pack_bf16x32(const float (&v)[32], uint4 (&pk)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 a = __floats2bfloat162_rn(v[8 * i + 0], v[8 * i + 1]);
        __nv_bfloat162 b = __floats2bfloat162_rn(v[8 * i + 2], v[8 * i + 3]);
        __nv_bfloat162 c = __floats2bfloat162_rn(v[8 * i + 4], v[8 * i + 5]);
        __nv_bfloat162 d = __floats2bfloat162_rn(v[8 * i + 6], v[8 * i + 7]);
        pk[i].x = *reinterpret_cast<uint32_t*>(&a);
        pk[i].y = *reinterpret_cast<uint32_t*>(&b);
        pk[i].z = *reinterpret_cast<uint32_t*>(&c);
        pk[i].w = *reinterpret_cast<uint32_t*>(&d);
    }
}

__device__ __forceinline__ void unpack_bf16x32(const uint4* pk, float (&v)[32]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&pk[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 f = __bfloat1622float2(h[j]);
            v[8 * i + 2 * j] = f.x;
            v[8 * i + 2 * j + 1] = f.y;
        }
    }
}

struct EpiSwiGLU {
    static constexpr int SLOTS = 1;
    bf16* hact;
    int64_t f;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    // 64 columns per pass so every output piece (gate, up, hact) is a full 128-byte row
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out) const {
        const int64_t row = g.out_row0 + static_cast<int64_t>(mt) * GEMM_BM + r;
        bf16* gu = static_cast<bf16*>(g.out0) + row * g.ldo + static_cast<int64_t>(nt) * 256;
        bf16* ha = hact + row * f + static_cast<int64_t>(nt) * 128;
        const int c = half * 64;
        uint4 pg[8], pu[8], ph[8];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            float gv[32], uv[32], hv[32];
            acc_load32(taddr + c + 32 * s, empty, gv);
            acc_load32(taddr + 128 + c + 32 * s, empty, uv);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                // Hact = silu(G) * U; saved for backward instead of (G, U): the factors
                // A = U * silu'(G) and B = silu(G), so dG = dH * A and dU = dH * B there
                const float sg = sigmoid_fast(gv[i]);
                const float silu = gv[i] * sg;
                hv[i] = silu * uv[i];
                const float a = uv[i] * (sg * (1.f + gv[i] * (1.f - sg)));
                gv[i] = a;
                uv[i] = silu;
            }
            pack_bf16x32(gv, *reinterpret_cast<uint4(*)[4]>(&pg[4 * s]));
            pack_bf16x32(uv, *reinterpret_cast<uint4(*)[4]>(&pu[4 * s]));
            pack_bf16x32(hv, *reinterpret_cast<uint4(*)[4]>(&ph[4 * s]));
        }
        out.put<8>(gu + c, pg);
        out.put<8>(gu + 128 + c, pu);
        out.put<8>(ha + c, ph);
    }
};

template <int BN>
struct EpiDSwiGLU {
    static constexpr int SLOTS = 1;
    const bf16* gu;
    int64_t f;
    // the saved gate / up rows this thread reads for (mt, nt): 2 x BN/2 bf16 of its row
    __device__ void prefetch(const GemmGroup& g, int mt, int nt, int r, int half) const {
        const int64_t row = g.out_row0 + static_cast<int64_t>(mt) * GEMM_BM + r;
        const bf16* gurow = gu + row * 2 * f;
#pragma unroll
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 64) {
            const int64_t x0 = static_cast<int64_t>(nt) * BN + c;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(gurow + il_gate(x0)));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(gurow + il_up(x0)));
        }
    }
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out) const {
        const int64_t row = g.out_row0 + static_cast<int64_t>(mt) * GEMM_BM + r;
        const bf16* gurow = gu + row * 2 * f;
        bf16* dgurow = static_cast<bf16*>(g.out0) + row * g.ldo;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 64) {
            const int64_t x0 = static_cast<int64_t>(nt) * BN + c;  // f index of column 0
            const int64_t ig = il_gate(x0), iu = il_up(x0);         // 64-column runs
            uint4 pg[8], pu[8], lg[8], lu[8];
            {  // saved gate / up pre-activations (64 columns each): both loads in flight
                uint4 tg[8], tu[8];
                out.load_rows<8>(gurow + ig, tg);
                out.load_rows<8>(gurow + iu, tu);
                out.land_rows<8>(tg, lg);
                out.land_rows<8>(tu, lu);
            }
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                float dh[32], fa[32], fb[32], dg[32], du[32];
                unpack_bf16x32(&lg[4 * s], fa);  // A = U * silu'(G)
                unpack_bf16x32(&lu[4 * s], fb);  // B = silu(G)
                acc_load32(taddr + c + 32 * s, empty, dh);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    dg[i] = dh[i] * fa[i];
                    du[i] = dh[i] * fb[i];
                }
                pack_bf16x32(dg, *reinterpret_cast<uint4(*)[4]>(&pg[4 * s]));
                pack_bf16x32(du, *reinterpret_cast<uint4(*)[4]>(&pu[4 * s]));
            }
            out.put<8>(dgurow + ig, pg);
            out.put<8>(dgurow + iu, pu);
        }
    }
};

// The same dSwiGLU with the saved factor rows staged by TMA (pair kernel, BN = 256): the
// kernel's warp 3 loads each 64-column piece of the tile's A (gate slots) and B (up slots)
// factor rows (2 x 128 rows x 128 B, 128B-swizzled) into a double-buffered ring as soon as
// the tile is scheduled, so the loads overlap the MMAs instead of stalling the epilogue.
// Per piece, the two warps of a TMEM lane quarter read the same 64 accumulator columns:
// half 0 forms dG = dH * A, half 1 dU = dH * B, each a whole 128-byte row per store.
template <int NB>  // staging buffers (1: room for 4 operand stages, 2: 3 stages)
struct EpiDSwiGLUStaged {
    static constexpr int SLOTS = 1;
    static constexpr int PIECES = 4;  // 256 columns / 64
    static constexpr int STAGE_BUFS = NB;
    static constexpr int STAGED_BYTES = NB * 2 * 16384;  // NB x (A piece + B piece)
    const CUtensorMap* fmap;                          // GU [rows x 2f], {64 x 128} boxes
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void stage_load(const GemmGroup& g, int mt, int nt, int pc, uint8_t* dst,
                               uint64_t* bar) const {
        const int row = static_cast<int>(g.out_row0) + mt * GEMM_BM;
        const int64_t x0 = static_cast<int64_t>(nt) * 256 + pc * 64;
        tma_load_2d(fmap, bar, dst, static_cast<int32_t>(il_gate(x0)), row);
        tma_load_2d(fmap, bar, dst + 16384, static_cast<int32_t>(il_up(x0)), row);
    }
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out, StageCtx& sc) const {
        const int64_t row = g.out_row0 + static_cast<int64_t>(mt) * GEMM_BM + r;
        bf16* dgurow = static_cast<bf16*>(g.out0) + row * g.ldo;
        const int lane = r & 31;
#pragma unroll 1
        for (int pc = 0; pc < PIECES; ++pc) {
            const int b = sc.cnt % NB;
            mbar_wait(&sc.full[b], (sc.cnt / NB) & 1);
            ++sc.cnt;
            // this thread's factor row (128 B, 16-byte chunks swizzled by row % 8)
            const uint8_t* frow = sc.base + b * 32768 + half * 16384 + r * 128;
            const int64_t x0 = static_cast<int64_t>(nt) * 256 + pc * 64;
            uint4 pk[8];
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                float dh[32], fa[32];
                uint4 fr[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    fr[j] = *reinterpret_cast<const uint4*>(frow + (((4 * s2 + j) ^ (r & 7)) << 4));
                unpack_bf16x32(fr, fa);
                acc_load32(taddr + pc * 64 + 32 * s2, empty, dh);
#pragma unroll
                for (int i = 0; i < 32; ++i) dh[i] = dh[i] * fa[i];
                pack_bf16x32(dh, *reinterpret_cast<uint4(*)[4]>(&pk[4 * s2]));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sc.empty[b]);  // the piece's smem is no longer read
            out.put<8>(dgurow + (half ? il_up(x0) : il_gate(x0)), pk);
        }
    }
};

// dSwiGLU with the factor pieces staged by TMA and the products written back IN PLACE:
// 32-column pieces (2 x 128 rows x 64 B, 64B-swizzled) in NB ring buffers; each thread
// overwrites its factor row with its dG (half 0) / dU (half 1) row and the warp's lane 0
// stores its 32 x 32 box by TMA. No epilogue transpose slots, so NB = 3 buffers (48 KB)
// still leave 5 operand stages; a buffer is released once its store has read it (one piece
// later, so the wait never stalls the piece in hand).
template <int NB>
struct EpiDSwiGLUInPlace {
    static constexpr int SLOTS = 0;
    static constexpr int PIECES = 8;  // 256 columns / 32
    static constexpr int STAGE_BUFS = NB;
    static constexpr int STAGED_BYTES = NB * 2 * 8192;
    const CUtensorMap* fmap;  // GU [rows x 2f], {32 x 128} boxes, 64B swizzle
    const CUtensorMap* omap;  // dGU [rows x 2f], {32 x 32} boxes, 64B swizzle
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void stage_load(const GemmGroup& g, int mt, int nt, int pc, uint8_t* dst,
                               uint64_t* bar) const {
        const int row = static_cast<int>(g.out_row0) + mt * GEMM_BM;
        const int64_t x0 = static_cast<int64_t>(nt) * 256 + pc * 32;
        tma_load_2d(fmap, bar, dst, static_cast<int32_t>(il_gate(x0)), row);
        tma_load_2d(fmap, bar, dst + 8192, static_cast<int32_t>(il_up(x0)), row);
    }
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut&, StageCtx& sc) const {
        const int lane = r & 31, q = r >> 5;
        const int orow = static_cast<int>(g.out_row0) + mt * GEMM_BM + q * 32;
        const int sw = (r >> 1) & 3;  // 64B swizzle: 16-byte chunk c sits at c ^ ((r/2)%4)
#pragma unroll 1
        for (int pc = 0; pc < PIECES; ++pc) {
            const int b = sc.cnt % NB;
            mbar_wait(&sc.full[b], (sc.cnt / NB) & 1);
            ++sc.cnt;
            uint8_t* piece = sc.base + b * 16384 + half * 8192;
            uint8_t* frow = piece + r * 64;
            float dh[32], fa[32];
            uint4 fr[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) fr[j] = *reinterpret_cast<const uint4*>(frow + ((j ^ sw) << 4));
            unpack_bf16x32(fr, fa);
            acc_load32(taddr + pc * 32, empty, dh);
#pragma unroll
            for (int i = 0; i < 32; ++i) dh[i] = dh[i] * fa[i];
            pack_bf16x32(dh, fr);
#pragma unroll
            for (int j = 0; j < 4; ++j) *reinterpret_cast<uint4*>(frow + ((j ^ sw) << 4)) = fr[j];
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                const int64_t x0 = static_cast<int64_t>(nt) * 256 + pc * 32;
                tma_store_2d(omap, piece + q * 2048,
                             static_cast<int32_t>(half ? il_up(x0) : il_gate(x0)), orow);
                bulk_commit();
                bulk_wait_read<1>();  // the previous piece's store has read its buffer
                if (sc.cnt >= 2) mbar_arrive(&sc.empty[(sc.cnt - 2) % NB]);
            }
        }
    }
};

struct EpiGradW1 {
    static constexpr int SLOTS = 1;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out) const {
        const int64_t row = static_cast<int64_t>(mt) * GEMM_BM + r;  // d index
#pragma unroll 1
        for (int c = half * 128; c < half * 128 + 128; c += 32) {
            float v[32];
            acc_load32(taddr + c, empty, v);
            float* base = static_cast<float*>(c < 128 ? g.out0 : g.out1);
            out.put_f32x32(base + row * g.ldo + static_cast<int64_t>(nt) * 128 + (c & 127), v);
        }
    }
};

// ---- MaskedAdamW fused into the dW epilogue ----------------------------------------
// The accumulator tile IS the owned expert's gradient (full K reduction in one tile),
// so the optimizer step runs right here: theta, m and v rows are fetched row-major into
// three smem slots with cp.async, each lane updates its row in place with the same
// adam_elem as the standalone pass (bit-identical), the slots are written back
// row-major, and the bf16 GEMM operand copy is refreshed. No gradient is materialized.
// Group fields: out0 = parameters of the block at (row 0, col 0), out_row0 = compact
// (m / v) offset of the same element, aux = shadow slot, ldo = row length.
__device__ __forceinline__ void adam_rows32(const EpiOut& out, const float (&gr)[32],
                                            const AdamScalars& a, float (&th_out)[32]) {
    float* th = reinterpret_cast<float*>(out.my_row(0));
    float* mm = reinterpret_cast<float*>(out.my_row(1));
    float* vv = reinterpret_cast<float*>(out.my_row(2));
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
        float4 t4 = *reinterpret_cast<float4*>(th + i);
        float4 m4 = *reinterpret_cast<float4*>(mm + i);
        float4 v4 = *reinterpret_cast<float4*>(vv + i);
        t4.x = adam_elem(t4.x, gr[i + 0], m4.x, v4.x, a);
        t4.y = adam_elem(t4.y, gr[i + 1], m4.y, v4.y, a);
        t4.z = adam_elem(t4.z, gr[i + 2], m4.z, v4.z, a);
        t4.w = adam_elem(t4.w, gr[i + 3], m4.w, v4.w, a);
        *reinterpret_cast<float4*>(th + i) = t4;
        *reinterpret_cast<float4*>(mm + i) = m4;
        *reinterpret_cast<float4*>(vv + i) = v4;
        th_out[i + 0] = t4.x;
        th_out[i + 1] = t4.y;
        th_out[i + 2] = t4.z;
        th_out[i + 3] = t4.w;
    }
}

// one 32-column piece: fetch theta / m / v rows, update, write back, refresh the shadow
__device__ __forceinline__ void adam_piece(const EpiOut& out, const AdamEpi& p, uint32_t taddr,
                                           bool empty, float* th_g, int64_t comp, bf16* sh_g) {
    float gr[32];
    acc_load32(taddr, empty, gr);
    out.rows_load_async<8>(0, th_g);
    out.rows_load_async<8>(1, p.m + comp);
    out.rows_load_async<8>(2, p.v + comp);
    out.rows_wait();
    float th[32];
    adam_rows32(out, gr, *p.a, th);
    out.rows_store<8>(0, th_g);
    out.rows_store<8>(1, p.m + comp);
    out.rows_store<8>(2, p.v + comp);
    uint4 pk[4];
    pack_bf16x32(th, pk);
    out.put<4>(sh_g, pk, 0);
}

// dW of gate||up (MN-MN, BN = 256): tile rows = d index, columns [0,128) -> wg, [128,256)
// -> wu at f-columns nt*128 + c; shadow W1 [slot][d][2f] interleaved gate|up.
struct EpiAdamW1 {
    static constexpr int SLOTS = 3;
    AdamEpi p;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out) const {
        if (!loss_ok(p.loss_total)) return;  // uniform: no update after a non-finite loss
        const int64_t row = static_cast<int64_t>(mt) * GEMM_BM + r;  // d index
        const int64_t df = p.d * p.f;
        bf16* sh_row = p.w1 + static_cast<int64_t>(g.aux) * 2 * df + row * 2 * p.f;
#pragma unroll 1
        for (int c = half * 128; c < half * 128 + 128; c += 32) {
            const bool up = c >= 128;
            const int64_t x0 = static_cast<int64_t>(nt) * 128 + (c & 127);
            const int64_t off = (up ? df : 0) + row * g.ldo + x0;
            adam_piece(out, p, taddr + c, empty, static_cast<float*>(g.out0) + off, g.out_row0 + off,
                       sh_row + (up ? il_up(x0) : il_gate(x0)));
        }
    }
};

// dW of down (MN-MN): tile rows = f index, columns = d index nt*BN + c; shadow W2 = Wd.
template <int BN>
struct EpiAdamW2 {
    static constexpr int SLOTS = 3;
    AdamEpi p;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out) const {
        if (!loss_ok(p.loss_total)) return;
        const int64_t row = static_cast<int64_t>(mt) * GEMM_BM + r;  // f index
        bf16* sh_row = p.w2 + static_cast<int64_t>(g.aux) * p.d * p.f + row * p.d;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            const int64_t x0 = static_cast<int64_t>(nt) * BN + c;
            const int64_t off = row * g.ldo + x0;
            adam_piece(out, p, taddr + c, empty, static_cast<float*>(g.out0) + off, g.out_row0 + off,
                       sh_row + x0);
        }
    }
};

// ---- MaskedAdamW fused into the dW epilogue, operands staged by TMA ------------------
// KIND 1: dW of gate||up (tile columns [0,128) -> wg, [128,256) -> wu); KIND 2: dW of down.
// The kernel's warp 3 loads each 32-column piece of the tile's theta, m and v (3 x 128 rows
// x 128 B, 128B-swizzled) into a double-buffered smem ring ahead of the epilogue; every
// epilogue warp updates its 32 rows x 16 columns in place from the TMEM gradients (the same
// adam_elem as the standalone pass: bit-identical), writes the bf16 operand copy, and once
// all 8 warps are done one thread writes the three tiles back by TMA stores and frees the
// buffer when they have read it. No gradient is materialized and no thread waits on a
// global load.
template <int KIND, int BN>
struct EpiAdamStaged {
    static constexpr int SLOTS = 0;
    static constexpr int PIECES = BN / 32;
    static constexpr int STAGE_BUFS = 2;
    static constexpr int STAGED_BYTES = 2 * 3 * 16384;
    static constexpr int STAGE_ARRIVALS = 1;  // the thread that issued the write-back
    AdamEpi p;
    const AdamMaps* maps;  // [L]
    int M;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    // piece pc of tile (mt, nt): the view (f- or d-wide) rows / column of theta and m / v
    __device__ void coords(const GemmGroup& g, int mt, int nt, int pc, const AdamMaps*& am,
                           int& col, int& row_th, int& row_mv, bool& up) const {
        am = maps + g.aux / M;
        const int64_t w = KIND == 1 ? p.f : p.d;  // view row length
        int64_t x0;
        if (KIND == 1) {
            up = pc >= PIECES / 2;
            x0 = static_cast<int64_t>(nt) * 128 + (pc % (PIECES / 2)) * 32;
        } else {
            up = false;
            x0 = static_cast<int64_t>(nt) * BN + pc * 32;
        }
        const int64_t extra = up ? p.d : 0;  // wu rows follow wg's d rows
        col = static_cast<int>(x0);
        row_th = static_cast<int>((static_cast<const float*>(g.out0) - am->th_base) / w + extra +
                                  static_cast<int64_t>(mt) * GEMM_BM);
        row_mv = static_cast<int>((g.out_row0 - am->mv_base) / w + extra +
                                  static_cast<int64_t>(mt) * GEMM_BM);
    }
    __device__ void stage_load(const GemmGroup& g, int mt, int nt, int pc, uint8_t* dst,
                               uint64_t* bar) const {
        const AdamMaps* am;
        int col, rt, rm;
        bool up;
        coords(g, mt, nt, pc, am, col, rt, rm, up);
        const CUtensorMap* mth = KIND == 1 ? &am->th_f : &am->th_d;
        const CUtensorMap* mm = KIND == 1 ? &am->m_f : &am->m_d;
        const CUtensorMap* mv = KIND == 1 ? &am->v_f : &am->v_d;
        tma_load_2d(mth, bar, dst, col, rt);
        tma_load_2d(mm, bar, dst + 16384, col, rm);
        tma_load_2d(mv, bar, dst + 32768, col, rm);
    }
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out, StageCtx& sc) const {
        const bool ok = loss_ok(p.loss_total);  // uniform: no update after a bad step
        const AdamScalars a = *p.a;
        const int64_t row = static_cast<int64_t>(mt) * GEMM_BM + r;  // row within the block
        const bool leader = threadIdx.x == 128;                     // warp 4, lane 0
#pragma unroll 1
        for (int pc = 0; pc < PIECES; ++pc) {
            const int b = sc.cnt & 1;
            mbar_wait(&sc.full[b], (sc.cnt >> 1) & 1);
            ++sc.cnt;
            uint8_t* buf = sc.base + b * (STAGED_BYTES / 2);
            const AdamMaps* am;
            int col, rt, rm;
            bool up;
            coords(g, mt, nt, pc, am, col, rt, rm, up);
            if (ok) {
                // gradients: this warp's 32 rows x 16 columns of the piece
                const uint32_t tcol =
                    KIND == 1 ? (up ? 128u : 0u) + (pc % (PIECES / 2)) * 32 + half * 16
                              : pc * 32 + half * 16;
                uint32_t gu[16];
                float gr[16];
                if (empty) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) gr[i] = 0.f;
                } else {
                    tmem_ld16(taddr + tcol, gu);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) gr[i] = __uint_as_float(gu[i]);
                }
                float th[16];
#pragma unroll
                for (int j = 0; j < 4; ++j) {  // 16-byte chunk 4*half + j of the 128-byte row
                    const int off = r * 128 + (((4 * half + j) ^ (r & 7)) << 4);
                    float4 t4 = *reinterpret_cast<float4*>(buf + off);
                    float4 m4 = *reinterpret_cast<float4*>(buf + 16384 + off);
                    float4 v4 = *reinterpret_cast<float4*>(buf + 32768 + off);
                    t4.x = adam_elem(t4.x, gr[4 * j + 0], m4.x, v4.x, a);
                    t4.y = adam_elem(t4.y, gr[4 * j + 1], m4.y, v4.y, a);
                    t4.z = adam_elem(t4.z, gr[4 * j + 2], m4.z, v4.z, a);
                    t4.w = adam_elem(t4.w, gr[4 * j + 3], m4.w, v4.w, a);
                    *reinterpret_cast<float4*>(buf + off) = t4;
                    *reinterpret_cast<float4*>(buf + 16384 + off) = m4;
                    *reinterpret_cast<float4*>(buf + 32768 + off) = v4;
                    th[4 * j + 0] = t4.x;
                    th[4 * j + 1] = t4.y;
                    th[4 * j + 2] = t4.z;
                    th[4 * j + 3] = t4.w;
                }
                // the bf16 GEMM operand copy of these 16 parameters (32 contiguous bytes)
                const int64_t x = col + half * 16;
                bf16* sh;
                if (KIND == 1)
                    sh = p.w1 + static_cast<int64_t>(g.aux) * 2 * p.d * p.f + row * 2 * p.f +
                         (up ? il_up(x) : il_gate(x));
                else
                    sh = p.w2 + static_cast<int64_t>(g.aux) * p.d * p.f + row * p.d + x;
                uint4 pk[2];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    __nv_bfloat162 c0 = __floats2bfloat162_rn(th[8 * i + 0], th[8 * i + 1]);
                    __nv_bfloat162 c1 = __floats2bfloat162_rn(th[8 * i + 2], th[8 * i + 3]);
                    __nv_bfloat162 c2 = __floats2bfloat162_rn(th[8 * i + 4], th[8 * i + 5]);
                    __nv_bfloat162 c3 = __floats2bfloat162_rn(th[8 * i + 6], th[8 * i + 7]);
                    pk[i] = make_uint4(*reinterpret_cast<uint32_t*>(&c0),
                                       *reinterpret_cast<uint32_t*>(&c1),
                                       *reinterpret_cast<uint32_t*>(&c2),
                                       *reinterpret_cast<uint32_t*>(&c3));
                }
                reinterpret_cast<uint4*>(sh)[0] = pk[0];
                reinterpret_cast<uint4*>(sh)[1] = pk[1];
                fence_proxy_async_smem();
            }
            named_bar_sync(1, 256);  // every epilogue warp is done with this piece
            if (leader) {
                if (ok) {
                    const CUtensorMap* mth = KIND == 1 ? &am->th_f : &am->th_d;
                    const CUtensorMap* mm = KIND == 1 ? &am->m_f : &am->m_d;
                    const CUtensorMap* mv = KIND == 1 ? &am->v_f : &am->v_d;
                    tma_store_2d(mth, buf, col, rt);
                    tma_store_2d(mm, buf + 16384, col, rm);
                    tma_store_2d(mv, buf + 32768, col, rm);
                    bulk_commit();
                    bulk_wait_read<0>();
                }
                mbar_arrive(&sc.empty[b]);
            }
        }
    }
};

// ---- head forward with the softmax-CE fused into the epilogue (V == BN == 256) ----------
// The accumulator tile holds the full logits row of each of its 128 tokens; the two warps
// of a TMEM lane quarter (column halves) combine their row max and exp sums through smem
// under a 64-thread named barrier, then each writes its half of the bf16 dlogits (the head
// backward GEMMs' operand), and the half-0 lane the per-token CE term and lse. Same math as
// head_ce_k (graph.hpp:410-423 + logsumexp backward), tolerance-level sums.
struct EpiHeadCE {
    static constexpr int SLOTS = 1;
    const int32_t* targets;
    int64_t T;
    float g_s2, g_ssum;
    bf16* dlog;
    float* diff;
    float* lse;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    // CUDA's full-precision expf (not the glibc-exact one): the logits come out of a bf16
    // tensor-core GEMM, so the loss is a tolerance quantity here and exact exp buys nothing
    __device__ static float ex(float z) { return expf(z); }
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half, EpiOut& out) const {
        const int64_t t = g.out_row0 + static_cast<int64_t>(mt) * GEMM_BM + r;
        const bool valid = t < T;
        const int lane = out.lane;
        // this lane's exchange words in its own warp's staging; the partner warp (other
        // column half of the same rows) is 4 warps away
        float* mine = reinterpret_cast<float*>(out.base);
        float* theirs = reinterpret_cast<float*>(out.base + (half ? -4 : 4) * SLOTS * EPI_SLOT_BYTES);
        const int bar = 1 + ((r >> 5) & 3);  // per lane-quarter pair of warps
        auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory"); };
        const int32_t tgt = valid ? __ldg(targets + t) : -1;
        const int c0 = half * 128;
        float mx = -INFINITY, picked = 0.f;
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
            float v[32];
            acc_load32(taddr + c0 + c, empty, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                mx = fmaxf(mx, v[i]);
                if (c0 + c + i == tgt) picked = v[i];
            }
        }
        mine[2 * lane] = mx;
        mine[2 * lane + 1] = picked;
        pair_sync();
        mx = fmaxf(mx, theirs[2 * lane]);
        const bool tgt_here = tgt >= c0 && tgt < c0 + 128;
        if (!tgt_here) picked = theirs[2 * lane + 1];
        pair_sync();  // exchange words reused below
        float sum = 0.f;
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
            float v[32];
            acc_load32(taddr + c0 + c, empty, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) sum += ex(fsub(v[i], mx));
        }
        mine[2 * lane] = sum;
        pair_sync();
        const float total = half ? theirs[2 * lane] + sum : sum + theirs[2 * lane];
        pair_sync();
        const float lse_v = mx + logf(total);
        if (valid && half == 0) {
            diff[t] = lse_v + picked * -1.f;
            lse[t] = lse_v;
        }
        // lse.grad = (0 + g_s2*lse) + g_s2*lse + g_ssum (z-loss mul, then ce add)
        const float glse = fadd(fadd(fadd(0.f, fmul(g_s2, lse_v)), fmul(g_s2, lse_v)), g_ssum);
        const float isum = 1.f / total;
        bf16* drow = dlog + t * 256 + c0;
#pragma unroll 1
        for (int c = 0; c < 128; c += 64) {
            uint4 pk[8];
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                float v[32], o[32];
                acc_load32(taddr + c0 + c + 32 * s2, empty, v);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int j = c0 + c + 32 * s2 + i;
                    const float base = (j == tgt) ? -1.f * g_ssum : 0.f;
                    o[i] = valid ? fadd(base, fmul(glse, ex(fsub(v[i], mx)) * isum)) : 0.f;
                }
                pack_bf16x32(o, *reinterpret_cast<uint4(*)[4]>(&pk[4 * s2]));
            }
            out.put<8>(drow + c, pk);
        }
    }
};

static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
        // experiments: persistent GEMM grids over fewer SMs (the rest left to the side stream)
        if (const char* e = std::getenv("SPES_GEMM_SMS"))
            g_num_sms = std::max(2, std::min(g_num_sms, std::atoi(e)));
    }
    return g_num_sms;
}

thread_local bool g_gemm_pairs = false;
void gemm_set_pair_mode(bool on) { g_gemm_pairs = on; }

// Pair mode: cta_group::2 kernel on cluster pairs (tiles of 256 rows); otherwise the
// 1-CTA kernel (tiles of 128 rows). The group tables must match the mode.
template <int BN, bool AMN, bool BMN, class Epi>
static void launch(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                   const int32_t* tiles, int max_tiles, const Epi& epi, cudaStream_t s) {
    if (max_tiles <= 0) return;
    if (ng > GEMM_MAX_GROUPS) throw std::invalid_argument("grouped GEMM: too many groups");
    if (g_gemm_pairs) {
        auto kern = grouped_gemm_2cta_kernel<BN, Epi, AMN, BMN>;
        static std::atomic<uint64_t> configured2{0};
        if (first_use_on_device(configured2))
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Gemm2Cfg<BN, Epi::SLOTS, EpiStaged<Epi>::bytes>::SMEM_BYTES);
        const int pairs = max_tiles < num_sms() / 2 ? max_tiles : num_sms() / 2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(GEMM_THREADS);
        cfg.dynamicSmemBytes = Gemm2Cfg<BN, Epi::SLOTS, EpiStaged<Epi>::bytes>::SMEM_BYTES;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, a, b, g, ng, tiles, max_tiles, epi);
        count_launch();
        return;
    }
    if constexpr (EpiStaged<Epi>::bytes > 0) {
        throw std::logic_error("grouped GEMM: staged epilogues need the cta_group::2 kernel");
    } else {
        auto kern = grouped_gemm_kernel<BN, Epi, AMN, BMN>;
        static std::atomic<uint64_t> configured{0};  // one per template instantiation
        if (first_use_on_device(configured))
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 GemmCfg<BN, Epi::SLOTS>::SMEM_BYTES);
        const int grid = max_tiles < num_sms() ? max_tiles : num_sms();
        kern<<<grid, GEMM_THREADS, GemmCfg<BN, Epi::SLOTS>::SMEM_BYTES, s>>>(a, b, g, ng, tiles,
                                                                           max_tiles, epi);
        count_launch();
    }
}

void gemm_prepare(int device) {
    (void)device;
    num_sms();
}

// expert forward gate||up: A = Xp (K-major), B = W1 [d x 2f] row-major (MN-major)
void gemm_swiglu(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                 const int32_t* tiles, int max_tiles, bf16* hact, int64_t f, cudaStream_t s) {
    launch<256, false, true>(a, b, g, ng, tiles, max_tiles, EpiSwiGLU{hact, f}, s);
}

template <int BN>
static void store_f32(GemmMajor mj, const CUtensorMap& a, const CUtensorMap& b,
                      const GemmGroup* g, int ng, const int32_t* tiles, int max_tiles,
                      cudaStream_t s) {
    switch (mj) {
        case GemmMajor::KK:
            launch<BN, false, false>(a, b, g, ng, tiles, max_tiles, EpiStoreF32<BN>{}, s);
            break;
        case GemmMajor::KMN:
            launch<BN, false, true>(a, b, g, ng, tiles, max_tiles, EpiStoreF32<BN>{}, s);
            break;
        case GemmMajor::MNMN:
            launch<BN, true, true>(a, b, g, ng, tiles, max_tiles, EpiStoreF32<BN>{}, s);
            break;
    }
}

void gemm_store_f32(int bn, GemmMajor mj, const CUtensorMap& a, const CUtensorMap& b,
                    const GemmGroup* g, int ng, const int32_t* tiles, int max_tiles,
                    cudaStream_t s) {
    if (bn == 256)
        store_f32<256>(mj, a, b, g, ng, tiles, max_tiles, s);
    else
        store_f32<128>(mj, a, b, g, ng, tiles, max_tiles, s);
}

void gemm_head_ce(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                  const int32_t* tiles, int max_tiles, const int32_t* targets, int64_t T,
                  float g_s2, float g_ssum, bf16* dlog, float* diff, float* lse,
                  cudaStream_t s) {
    launch<256, false, true>(a, b, g, ng, tiles, max_tiles,
                             EpiHeadCE{targets, T, g_s2, g_ssum, dlog, diff, lse}, s);
}

// variant 1 / 2: 64-column pieces through the transpose slots with 1 / 2 staging buffers;
// 3 / 4: 32-column pieces written back in place, 2 / 3 buffers (the maps decide which apply)
void gemm_dswiglu(int bn, const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                  const int32_t* tiles, int max_tiles, const bf16* gu, int64_t f,
                  const CUtensorMap* gu_map, const CUtensorMap* inplace_maps, int variant,
                  cudaStream_t s) {
    if (bn == 256 && g_gemm_pairs && inplace_maps && variant >= 3) {
        if (variant == 3)
            launch<256, false, false>(a, b, g, ng, tiles, max_tiles,
                                      EpiDSwiGLUInPlace<2>{inplace_maps, inplace_maps + 1}, s);
        else
            launch<256, false, false>(a, b, g, ng, tiles, max_tiles,
                                      EpiDSwiGLUInPlace<3>{inplace_maps, inplace_maps + 1}, s);
    } else if (bn == 256 && g_gemm_pairs && gu_map && variant >= 1) {  // staged by TMA
        if (variant == 2)
            launch<256, false, false>(a, b, g, ng, tiles, max_tiles, EpiDSwiGLUStaged<2>{gu_map}, s);
        else
            launch<256, false, false>(a, b, g, ng, tiles, max_tiles, EpiDSwiGLUStaged<1>{gu_map}, s);
    }
    else if (bn == 256)
        launch<256, false, false>(a, b, g, ng, tiles, max_tiles, EpiDSwiGLU<256>{gu, f}, s);
    else
        launch<128, false, false>(a, b, g, ng, tiles, max_tiles, EpiDSwiGLU<128>{gu, f}, s);
}

void gemm_grad_w1(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                  const int32_t* tiles, int max_tiles, cudaStream_t s) {
    launch<256, true, true>(a, b, g, ng, tiles, max_tiles, EpiGradW1{}, s);
}

void gemm_adamw_w1(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                   const int32_t* tiles, int max_tiles, const AdamEpi& p, cudaStream_t s,
                   const AdamMaps* aw, int M) {
    if (aw && g_gemm_pairs)
        launch<256, true, true>(a, b, g, ng, tiles, max_tiles, EpiAdamStaged<1, 256>{p, aw, M}, s);
    else
        launch<256, true, true>(a, b, g, ng, tiles, max_tiles, EpiAdamW1{p}, s);
}

void gemm_adamw_w2(int bn, const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                   const int32_t* tiles, int max_tiles, const AdamEpi& p, cudaStream_t s,
                   const AdamMaps* aw, int M) {
    if (aw && g_gemm_pairs) {
        if (bn == 256)
            launch<256, true, true>(a, b, g, ng, tiles, max_tiles, EpiAdamStaged<2, 256>{p, aw, M}, s);
        else
            launch<128, true, true>(a, b, g, ng, tiles, max_tiles, EpiAdamStaged<2, 128>{p, aw, M}, s);
        return;
    }
    if (bn == 256)
        launch<256, true, true>(a, b, g, ng, tiles, max_tiles, EpiAdamW2<256>{p}, s);
    else
        launch<128, true, true>(a, b, g, ng, tiles, max_tiles, EpiAdamW2<128>{p}, s);
}

}  // namespace spes_k

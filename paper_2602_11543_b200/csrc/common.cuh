// Shared device helpers for the SPES kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace spes_dev {

// Explicitly rounded fp32 ops: the reference is compiled without FMA and with
// strictly sequential reductions; kernels that must reproduce its
// bits use these so nvcc never contracts a*b+c into an FMA.
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float fsqrt(float a) { return __fsqrt_rn(a); }
// Two exactly rounded products in one instruction (FMUL2, sm_100). Sum the halves with
// the scalar fadd only: ptxas contracts mul.rn.f32x2 followed by add.rn.f32x2 into FFMA2.
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
          "l"(*reinterpret_cast<const unsigned long long*>(&b)));
    return *reinterpret_cast<const float2*>(&r);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Interleaved gate||up column layout used by the expert GEMMs: blocks of 128
// gate columns followed by the matching 128 up columns.
__host__ __device__ __forceinline__ int64_t il_gate(int64_t x) { return 256 * (x >> 7) + (x & 127); }
__host__ __device__ __forceinline__ int64_t il_up(int64_t x) { return il_gate(x) + 128; }

__device__ __forceinline__ float silu_f(float z) {
    // z * sigmoid(z) with the reference's branch structure (kernels.hpp:92-103)
    float s = z >= 0.f ? 1.f / (1.f + __expf(-z)) : __expf(z) / (1.f + __expf(z));
    return z * s;
}
// bf16-path activation: 1 / (1 + 2^(-z*log2 e)) with the SFU exp2 / reciprocal
// (the expert FFN runs on bf16 operands; its tolerance is far above these ulps).
__device__ __forceinline__ float sigmoid_fast(float z) {
    return __frcp_rn(1.f + exp2f(-1.4426950408889634f * z));
}
__device__ __forceinline__ float sigmoid_f(float z) {
    return z >= 0.f ? 1.f / (1.f + __expf(-z)) : __expf(z) / (1.f + __expf(z));
}

// MaskedAdamW::step scalars (trainer.hpp:68-84; bias corrections computed on the host)
struct AdamScalars {
    float lr, b1, b2, omb1, omb2, eps, wd, bc1, bc2;
    int32_t sgd;  // 1: the SGD inner step theta -= lr * g (trainer.hpp:197-204), no moments
};
// One MaskedAdamW element update (trainer.hpp:85-92), exact fp32 op order. Shared by the
// standalone optimizer pass and the dW-GEMM epilogues so both produce identical bits.
__device__ __forceinline__ float adam_elem(float th, float g, float& m, float& v,
                                           const AdamScalars& a) {
    m = fadd(fmul(a.b1, m), fmul(a.omb1, g));
    v = fadd(fmul(a.b2, v), fmul(fmul(a.omb2, g), g));
    const float mhat = fdiv(m, a.bc1);
    const float vhat = fdiv(v, a.bc2);
    const float upd = fmul(a.lr, fadd(fdiv(mhat, fadd(fsqrt(vhat), a.eps)), fmul(a.wd, th)));
    return fsub(th, upd);
}
// device-side guard: the reference applies no update after a non-finite loss
// (trainer.hpp:166-167) and validates token ids before the step (model.hpp:280-281).
// losses[5] is the step's status word (0 = ok; bit 0 an out-of-vocabulary token, bit 1 a
// non-finite loss), sticky until the host reports it, so no later step updates either.
__device__ __forceinline__ bool loss_ok(const double* losses) {
    return losses == nullptr || losses[5] == 0.0;
}

}  // namespace spes_dev

// common.cuh — shared device/host helpers for the sm_100a TEBD decimation library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace rb {

// Raises a kernel's max-dynamic-shared-memory attribute to at least `bytes` on the current device,
// never lowering it.  The attribute is process-wide: with host threads (one context each) launching
// the same kernel with different sizes, setting it to each launch's own size lets one thread's
// lower value invalidate another thread's launch ("invalid argument").  (ctx.cu)
cudaError_t smem_atleast(const void* kernel, size_t bytes);

using cplx = double2;  // interleaved (re, im) complex128 — the reference DenseMatrix element
                       // (dense_matrix.hpp:10) has exactly this memory image.

constexpr int kNumSMs = 148;

__host__ __device__ inline cplx mk(double r, double i) { return make_double2(r, i); }
__host__ __device__ inline cplx cadd(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
__host__ __device__ inline cplx csub(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
__host__ __device__ inline cplx cmul(cplx a, cplx b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__host__ __device__ inline cplx cmulc(cplx a, cplx b) {
    return mk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ inline cplx cconj(cplx a) { return mk(a.x, -a.y); }
__host__ __device__ inline cplx cscale(cplx a, double s) { return mk(a.x * s, a.y * s); }
__host__ __device__ inline double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
// fma: acc += a*b
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a)*b
__device__ __forceinline__ void cfmac(cplx& acc, cplx a, cplx b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}

// Sort key for descending ranks of norms / singular values: NaN (a non-finite input the
// boundary rejects afterwards) ranks last, so a rank loop still yields a permutation and no
// kernel indexes out of range before the finite check throws.
__host__ __device__ inline double rank_key(double x) { return x == x ? x : -1.0; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ cplx warp_sum(cplx v) {
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---- cp.async (LDGSTS) helpers -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const int n = pred ? 16 : 0;  // src-size 0 → zero-fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- FP64 tensor core: mma.sync m8n8k4 f64 (lowered to DMMA.8x8x4 on sm_100a) -------------
// Fragment layout (PTX ISA, mma.m8n8k4 .f64):  A 8x4: a[row=lane>>2][col=lane&3];
// B 4x8: b[row=lane&3][col=lane>>2];  C 8x8: c{0,1}[row=lane>>2][col=2*(lane&3)+{0,1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

}  // namespace rb

#define RB_CUDA_OK(expr)                                                                  \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess) return ::rb::fail_cuda(_e, #expr, __FILE__, __LINE__);     \
    } while (0)

// ozaki.cu — see ozaki.cuh for the scheme.  Per batch of products:
//   oz_xmax, oz_resid_b — the K-side compensation and per-column scale of X, and its residue
//                 panel B' (128-row K tiles, moduli in pairs),
//   oz_gemm_persistent — tcgen05.mma kind::i8: one CTA per SM walking (bond, modulus, column
//                 tile, 256-row block) tiles; TMA rings for A (4 x 32 KB, 128B-swizzled tiles) and
//                 the panel (3 x 32 KB), one issuing thread, two 128 x N' int32 accumulators in
//                 TMEM, eight epilogue warps reducing each accumulator to (D mod m_t)·w_t mod m_t
//                 (one byte per output) while the next tile's loads stream in,
//   oz_crt      — 96-bit fixed-point CRT of the T residues, scaled to FP64 (optionally added to C);
// plus, once per A, oz_rowexp, oz_colexp and oz_resid_a (its equilibrated residue tiles).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ozaki.cuh"
#include "pipeline.cuh"  // debug_enabled

namespace rb {

namespace {

constexpr int kModuli[kOzMaxMod] = {256, 255, 253, 251, 247, 241, 239, 233,
                                    229, 227, 223, 217, 211, 199, 197, 193};
// the same table as a constant expression usable in device code
__host__ __device__ constexpr int oz_modulus(int t) {
    return t == 0 ? 256 : t == 1 ? 255 : t == 2 ? 253 : t == 3 ? 251 : t == 4 ? 247 : t == 5 ? 241 : t == 6 ? 239
         : t == 7 ? 233 : t == 8 ? 229 : t == 9 ? 227 : t == 10 ? 223 : t == 11 ? 217 : t == 12 ? 211
         : t == 13 ? 199 : t == 14 ? 197 : 193;
}

// Per-T constants of the residue arithmetic and the CRT.
struct OzConst {
    int T;
    int bits;                      // floor(log2 M)
    int mod[kOzMaxMod], w[kOzMaxMod], lo[kOzMaxMod];
    double inv_md[kOzMaxMod];
    unsigned magic[kOzMaxMod];     // ceil(2^32 / m): Barrett quotient (off by at most +1)
    unsigned off[kOzMaxMod];       // m·ceil(2^31 / m) >= 2^31: makes an int32 non-negative mod m
    unsigned c3[kOzMaxMod][3];     // floor(2^128 / m) >> 32, as three 32-bit limbs (low first)
    double mscale;                 // M / 2^128
};

const OzConst& oz_const(int T) {
    static OzConst tab[kOzMaxMod + 1];
    static std::atomic<int> ready[kOzMaxMod + 1];
    if (ready[T].load()) return tab[T];
    OzConst k{};
    k.T = T;
    unsigned __int128 M = 1;
    for (int t = 0; t < T; ++t) M *= (unsigned __int128)kModuli[t];
    int bits = 0;
    for (unsigned __int128 v = M; v > 1; v >>= 1) ++bits;
    k.bits = bits;
    for (int t = 0; t < T; ++t) {
        const int m = kModuli[t];
        const unsigned __int128 Mi = M / (unsigned __int128)m;
        const int r = (int)(Mi % (unsigned __int128)m);
        int w = 0;
        for (int x = 1; x < m; ++x)
            if ((r * x) % m == 1) { w = x; break; }
        k.mod[t] = m;
        k.w[t] = w;
        k.lo[t] = -(m / 2);  // symmetric residues in [-(m/2), m - 1 - m/2]
        k.inv_md[t] = 1.0 / (double)m;
        k.magic[t] = (unsigned)(((1ull << 32) + m - 1) / m);
        k.off[t] = (unsigned)(m * (((1ull << 31) + m - 1) / m));
        const unsigned __int128 c = (~(unsigned __int128)0) / (unsigned __int128)m;
        k.c3[t][0] = (unsigned)(c >> 32);
        k.c3[t][1] = (unsigned)(c >> 64);
        k.c3[t][2] = (unsigned)(c >> 96);
    }
    k.mscale = std::ldexp((double)(unsigned long long)(M >> 64), -64) + std::ldexp((double)(unsigned long long)M, -128);
    tab[T] = k;
    ready[T].store(1);
    return tab[T];
}

int ceil_log2(long long v) {
    int b = 0;
    while ((1ll << b) < v) ++b;
    return b;
}
// kA + kX for an inner dimension K: 2K·2^(kA+kX) < 2^(bits-1) <= M/2, one bit of margin
int oz_total_bits(const OzConst& k, int K) { return k.bits - 2 - ceil_log2(2ll * K); }

// e with v in [2^(e-1), 2^e) for the non-negative double of bit pattern `bits` (0 -> 0)
__device__ __forceinline__ int oz_e(unsigned long long bits) {
    if (bits == 0) return 0;
    const int f = (int)(bits >> 52);
    if (f != 0) return f - 1022;
    int e;
    frexp(__longlong_as_double((long long)bits), &e);
    return e;
}
constexpr int kExpNone = (int)0xC0C0C0C0;  // "no entry" (memset byte 0xC0): a zero row / column
__device__ __forceinline__ int oz_exp_or0(int e) { return e == kExpNone ? 0 : e; }
// exponent of max(|re|, |im|) (kExpNone for zero)
__device__ __forceinline__ int oz_eabs(cplx v) {
    const double a = fmax(fabs(v.x), fabs(v.y));
    return a > 0.0 ? oz_e((unsigned long long)__double_as_longlong(a)) : kExpNone;
}
__device__ __forceinline__ double oz_pow2(int e) {  // 2^e for e in [-1022, 1023]
    return __longlong_as_double((long long)(e + 1023) << 52);
}
__device__ __forceinline__ double oz_scale(double x, int s) {  // x·2^s, |s| <= 2044
    const int h = s / 2;
    return x * oz_pow2(h) * oz_pow2(s - h);
}
// residue of an integer-valued double v (|v| <= 2^57) in [lo, lo + m): FP64 only, no conversion
// instruction (the 1.5·2^52 shifter rounds to an integer and exposes it in the low word)
__device__ __forceinline__ int oz_res(double v, int m, double inv_m, int lo) {
    const double sh = 6755399441055744.0;
    const double q = fma(v, inv_m, sh) - sh;
    const double r = fma(-q, (double)m, v);
    int ri = __double2loint(r + sh);
    if (ri < lo) ri += m;
    if (ri >= lo + m) ri -= m;
    return ri;
}

// ---- A: row / column maxima and residue planes ----------------------------------------------
// A' = rint(A_ik · 2^(kA - e_i - f_k)): e_i the exponent of row i's max, f_k that of column k's max
// after the rows are normalised (<= 0).  Every entry of A' is within 2^kA and carries kA bits
// relative to its own row and column scale — a TEBD Θ (λ-weighted on both sides) loses nothing
// to a global scale.
constexpr int kPrepGroup = 48;
struct PrepParams {
    const cplx* A[kPrepGroup];
    long long lda[kPrepGroup];
    int nib[kPrepGroup], nkb[kPrepGroup];
    int m[kPrepGroup], n[kPrepGroup], kA[kPrepGroup];
    int8_t* res[kPrepGroup];
    int* rowexp[kPrepGroup];  // [m]: exponent of the row's largest entry (0 for a zero row)
    int* colexp[kPrepGroup];  // [n]: max_i e(|A_ik|) - rowexp_i (kExpNone-filled before the scan)
    double* rowsq[kPrepGroup];    // [m] or null: each row's sum of |A_ik|^2 (the ||A||^2 of the caller)
    double* total_sq[kPrepGroup]; // null, or ||A||_F^2 = the rows' sums in row order
    int* nonfinite[kPrepGroup];   // null, or 1 if A has a non-finite entry
    int* bad;                                 // [count] (zeroed)
    int count;
    OzConst k;
};

// Row exponents (a warp per row), then column exponents of the row-normalised A (each near the
// HBM roofline; one-pass forms — shared-memory column atomics per element, or per-lane column
// maxima in registers at one CTA per SM — measured 1.0 and 3.0 ms vs 1.04 ms for 48 bonds)
__global__ void __launch_bounds__(256) oz_rowexp_kernel(const __grid_constant__ PrepParams P) {
    const int z = blockIdx.y;
    const int m = P.m[z], n = P.n[z];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * 8 + warp;
    if (row >= m) return;
    const cplx* A = P.A[z] + (long long)row * P.lda[z];
    int er = kExpNone, bad = 0;
    double sq = 0.0;  // the row's share of ||A||^2 (read here anyway: the caller's sumsq pass is saved)
    for (int c = lane; c < n; c += 32) {
        const cplx v = A[c];
        if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
        else er = max(er, oz_eabs(v));
        sq += cabs2(v);
    }
    for (int o = 16; o > 0; o >>= 1) er = max(er, __shfl_xor_sync(0xffffffffu, er, o));
    bad = __any_sync(0xffffffffu, bad);
    if (P.rowsq[z] != nullptr) sq = warp_sum(sq);
    if (lane == 0) {
        P.rowexp[z][row] = oz_exp_or0(er);
        if (bad) atomicOr(&P.bad[z], 1);
        if (P.rowsq[z] != nullptr) P.rowsq[z][row] = sq;
    }
}
// ||A||_F^2 from the row sums (one warp per matrix, a fixed order) and the non-finite flag
__global__ void oz_sumsq_final_kernel(const __grid_constant__ PrepParams P) {
    const int z = blockIdx.x, lane = threadIdx.x;
    if (P.total_sq[z] == nullptr) return;
    double s = 0.0;
    for (int i = lane; i < P.m[z]; i += 32) s += P.rowsq[z][i];
    s = warp_sum(s);
    if (lane == 0) {
        *P.total_sq[z] = s;
        if (P.nonfinite[z] != nullptr) *P.nonfinite[z] = P.bad[z] != 0 ? 1 : 0;
    }
}
__global__ void __launch_bounds__(256) oz_colexp_kernel(const __grid_constant__ PrepParams P) {
    const int z = blockIdx.z;
    const int m = P.m[z], n = P.n[z];
    const int col = blockIdx.x * 32 + (threadIdx.x & 31), g = threadIdx.x >> 5;
    const int rows_per = (m + gridDim.y - 1) / gridDim.y;
    const int r0 = blockIdx.y * rows_per, r1 = min(m, r0 + rows_per);
    __shared__ int red[8][32];
    int mx = kExpNone;
    if (col < n)
        for (int r = r0 + g; r < r1; r += 8) {
            const cplx v = P.A[z][(long long)r * P.lda[z] + col];
            const int e = (isfinite(v.x) && isfinite(v.y)) ? oz_eabs(v) : kExpNone;
            if (e != kExpNone) mx = max(mx, e - P.rowexp[z][r]);
        }
    red[g][threadIdx.x & 31] = mx;
    __syncthreads();
    if (g == 0 && col < n) {
        for (int i = 1; i < 8; ++i) mx = max(mx, red[i][threadIdx.x]);
        if (mx != kExpNone) atomicMax(&P.colexp[z][col], mx);
    }
}

// the residues of eight integer-valued (re, im) pairs mod m, packed into one 8-byte store per part
__device__ __forceinline__ void oz_store8(const double (&vr)[8], const double (&vi)[8], int8_t* dst, long long plane,
                                          int md, double im, int lo) {
    uint32_t pr[2], pi[2];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
        uint32_t a = 0, b = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a |= (uint32_t)(oz_res(vr[4 * w + u], md, im, lo) & 0xff) << (8 * u);
            b |= (uint32_t)(oz_res(vi[4 * w + u], md, im, lo) & 0xff) << (8 * u);
        }
        pr[w] = a;
        pi[w] = b;
    }
    *reinterpret_cast<uint2*>(dst) = make_uint2(pr[0], pr[1]);
    *reinterpret_cast<uint2*>(dst + plane) = make_uint2(pi[0], pi[1]);
}

// residues of an integer-valued double v (|v| <= 2^52) modulo MA and MB: r = v mod MA·MB exactly
// (shifter-rounded FP64 quotient, exact FMA remainder, |r| <= MA·MB/2 + 1 < 2^22), then each
// residue in FP32 (r/M needs only ~2^-16 accuracy to round exactly: no ties for odd M, and for
// M = 256 the tie ±128 is one byte) — half the FP64 work of two direct reductions.
template <int M>
__device__ __forceinline__ uint32_t oz_res32(float f, int ri) {
    // q = round(ri / M) = bits - 0x4B400000, bits the FP32 shifter's bit pattern; the residue's low
    // byte is that of ri - q·M in integers (two's complement: the symmetric residue as a signed
    // byte), and 0x4B400000·M is 0 mod 256, so the low byte of ri - bits·M is the same: one IMAD
    const int bits = __float_as_int(fmaf(f, 1.0f / (float)M, 12582912.0f));
    return (uint32_t)(ri - bits * M);
}
// the low bytes of four words packed into one (three PRMTs)
__device__ __forceinline__ uint32_t oz_pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
template <int MA, int MB>
__device__ __forceinline__ void oz_store8_pair(const double (&vr)[8], const double (&vi)[8], int8_t* dst, long long plane) {
    constexpr double P = (double)MA * (double)MB;
    const double sh = 6755399441055744.0;
    uint32_t xa[2][8], xb[2][8];  // [part][u]: residue mod MA / MB in the low byte
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
        for (int part = 0; part < 2; ++part) {
            const double v = part == 0 ? vr[u] : vi[u];
            const double q = fma(v, 1.0 / P, sh) - sh;
            const int ri = __double2loint(fma(-q, P, v) + sh);
            const float f = __int_as_float(ri + 0x4B400000) - 12582912.0f;
            xa[part][u] = oz_res32<MA>(f, ri);
            xb[part][u] = oz_res32<MB>(f, ri);
        }
    }
    auto lo = [](const uint32_t (&x)[8]) { return oz_pack4(x[0], x[1], x[2], x[3]); };
    auto hi = [](const uint32_t (&x)[8]) { return oz_pack4(x[4], x[5], x[6], x[7]); };
    *reinterpret_cast<uint2*>(dst) = make_uint2(lo(xa[0]), hi(xa[0]));
    *reinterpret_cast<uint2*>(dst + plane) = make_uint2(lo(xa[1]), hi(xa[1]));
    *reinterpret_cast<uint2*>(dst + 2 * plane) = make_uint2(lo(xb[0]), hi(xb[0]));
    *reinterpret_cast<uint2*>(dst + 3 * plane) = make_uint2(lo(xb[1]), hi(xb[1]));
}

template <int TT, int t>
__device__ __forceinline__ void oz_store_pairs(const double (&vr)[8], const double (&vi)[8], int8_t* dst, long long plane) {
    if constexpr (t + 1 < TT) {
        oz_store8_pair<oz_modulus(t), oz_modulus(t + 1)>(vr, vi, dst + (long long)(2 * t) * plane, plane);
        oz_store_pairs<TT, t + 2>(vr, vi, dst, plane);
    } else if constexpr (t < TT) {
        oz_store8(vr, vi, dst + (long long)(2 * t) * plane, plane, oz_modulus(t), 1.0 / (double)oz_modulus(t),
                  -(oz_modulus(t) / 2));
    }
}

// one thread = 8 consecutive columns of one (padded) row, both parts, all T moduli (TT > 0: the
// moduli count as a compile-time constant, every modulus an immediate)
template <int TT>
__global__ void __launch_bounds__(256) oz_resid_a_kernel(const __grid_constant__ PrepParams P) {
    const int z = blockIdx.y;
    const int m = P.m[z], n = P.n[z], nkb = P.nkb[z];
    const long long chunks_per_row = (long long)nkb * 16;
    const long long total = (long long)P.nib[z] * 128 * chunks_per_row;
    const cplx* A = P.A[z];
    int8_t* res = P.res[z];
    const long long plane = (long long)P.nib[z] * nkb * 16384;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(e / chunks_per_row);
        const int c0 = (int)(e % chunks_per_row) * 8;
        const int er = row < m ? P.kA[z] - P.rowexp[z][row] : 0;
        double vr[8], vi[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int col = c0 + u;
            cplx x = mk(0.0, 0.0);
            int s = 0;
            if (row < m && col < n) {
                x = A[(long long)row * P.lda[z] + col];
                s = er - oz_exp_or0(P.colexp[z][col]);
            }
            vr[u] = rint(oz_scale(x.x, s));
            vi[u] = rint(oz_scale(x.y, s));
            if (!isfinite(vr[u])) vr[u] = 0.0;
            if (!isfinite(vi[u])) vi[u] = 0.0;
        }
        int8_t* dst = res + ((long long)(row >> 7) * nkb + (c0 >> 7)) * 16384 + (row & 127) * 128 + (c0 & 127);
        if (TT > 0) {
            // moduli in pairs: one FP64 reduction modulo m_a·m_b (< 2^16), the two residues in FP32
            oz_store_pairs<TT, 0>(vr, vi, dst, plane);
        } else {
            for (int t = 0; t < P.k.T; ++t)
                oz_store8(vr, vi, dst + (long long)(2 * t) * plane, plane, P.k.mod[t], P.k.inv_md[t], P.k.lo[t]);
        }
    }
}

// ---- X: K-row compensation, per-column scale and the residue panel B' -------------------------
// X'' = X·2^(f_k) (op N: A's column exponents) or Q·2^(e_i) (op C: A's row exponents) — the
// inverse of A's equilibration along K — then each column j scaled by 2^(s_j) to kX bits.
// B'[t][r][part][k] (r in [0, JT·2LT)): for output column j (tile jt = j / LT, jj = j % LT)
//   row jt·2LT + jj      (real part of the output):  part 0 = X'_re,  part 1 =  sg·X'_im
//   row jt·2LT + LT + jj (imaginary part):           part 0 = X'_im,  part 1 = -sg·X'_re
// with sg = -1 for op N and +1 for op C (ozaki.cuh).
constexpr int kProdGroup = 48;
struct PanelParams {
    const cplx* X[kProdGroup];
    long long ldx[kProdGroup];
    int nkbx[kProdGroup];      // K tiles of 128
    int K[kProdGroup], l[kProdGroup], LT[kProdGroup], JT[kProdGroup], kX[kProdGroup];
    const int* kexp[kProdGroup];  // exponents of the K rows (op N: A's column exponents; op C: its row exponents)
    int8_t* bres[kProdGroup];
    int* sx[kProdGroup];     // [JT·LT]
    int* xbad[kProdGroup];   // [JT·LT]
    int sg;
    OzConst k;
};

// block = 8 columns x 32 row groups: column maxima of X''
__global__ void __launch_bounds__(256) oz_xmax_kernel(const __grid_constant__ PanelParams P) {
    const int z = blockIdx.y;
    const int LT = P.LT[z], JT = P.JT[z], K = P.K[z], l = P.l[z];
    const int j0 = blockIdx.x * 8;
    if (j0 >= JT * LT) return;
    const int tid = threadIdx.x, c = tid & 7, rg = tid >> 3;
    const int j = j0 + c;
    __shared__ double smax[32][8];
    __shared__ int sbad[8];
    if (tid < 8) sbad[tid] = 0;
    __syncthreads();
    double mx = 0.0;
    int bad = 0;
    if (j < l)
        for (int k0 = rg; k0 < K; k0 += 128) {  // four rows in flight per thread
            cplx v[4];
            int ke[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = k0 + 32 * u;
                v[u] = k < K ? P.X[z][(long long)k * P.ldx[z] + j] : mk(0.0, 0.0);
                ke[u] = k < K ? P.kexp[z][k] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (!isfinite(v[u].x) || !isfinite(v[u].y)) {
                    bad = 1;
                } else {
                    const double a = fmax(fabs(v[u].x), fabs(v[u].y));
                    if (a > 0.0) mx = fmax(mx, oz_scale(a, oz_exp_or0(ke[u])));
                }
            }
        }
    smax[rg][c] = mx;
    if (bad) atomicOr(&sbad[c], 1);
    __syncthreads();
    if (tid < 8) {
        double v = 0.0;
        for (int g = 0; g < 32; ++g) v = fmax(v, smax[g][tid]);
        P.sx[z][j0 + tid] = v > 0.0 ? P.kX[z] - oz_e((unsigned long long)__double_as_longlong(v)) : 0;
        P.xbad[z][j0 + tid] = sbad[tid];
    }
}

// the panel's residues by moduli pairs (oz_store8_pair's arithmetic): four K rows of one column
template <int TT, int t, int kPadW>
__device__ __forceinline__ void oz_panel_pairs(const double (&vr)[4], const double (&vi)[4],
                                               uint32_t (&S)[kOzMaxMod][8][2][kPadW], int c, int kq) {
    if constexpr (t + 1 < TT) {
        constexpr int MA = oz_modulus(t), MB = oz_modulus(t + 1);
        constexpr double Pm = (double)MA * (double)MB;
        const double sh = 6755399441055744.0;
        uint32_t xa[2][4], xb[2][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int part = 0; part < 2; ++part) {
                const double v = part == 0 ? vr[u] : vi[u];
                const double q = fma(v, 1.0 / Pm, sh) - sh;
                const int ri = __double2loint(fma(-q, Pm, v) + sh);
                const float f = __int_as_float(ri + 0x4B400000) - 12582912.0f;
                xa[part][u] = oz_res32<MA>(f, ri);
                xb[part][u] = oz_res32<MB>(f, ri);
            }
        }
        S[t][c][0][kq] = oz_pack4(xa[0][0], xa[0][1], xa[0][2], xa[0][3]);
        S[t][c][1][kq] = oz_pack4(xa[1][0], xa[1][1], xa[1][2], xa[1][3]);
        S[t + 1][c][0][kq] = oz_pack4(xb[0][0], xb[0][1], xb[0][2], xb[0][3]);
        S[t + 1][c][1][kq] = oz_pack4(xb[1][0], xb[1][1], xb[1][2], xb[1][3]);
        oz_panel_pairs<TT, t + 2, kPadW>(vr, vi, S, c, kq);
    } else if constexpr (t < TT) {
        constexpr int md = oz_modulus(t);
        uint32_t a = 0, b = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a |= (uint32_t)(oz_res(vr[u], md, 1.0 / (double)md, -(md / 2)) & 0xff) << (8 * u);
            b |= (uint32_t)(oz_res(vi[u], md, 1.0 / (double)md, -(md / 2)) & 0xff) << (8 * u);
        }
        S[t][c][0][kq] = a;
        S[t][c][1][kq] = b;
    }
}

// block = 8 columns x 128 K rows; a thread takes four consecutive K rows of one column (c = tid & 7,
// so a warp reads 4 x 128 contiguous bytes per row), packs each modulus' four residues into one word
// in shared memory, then the block writes 128-byte rows of B' (TT > 0: compile-time moduli).
template <int TT>
__global__ void __launch_bounds__(256) oz_resid_b_kernel(const __grid_constant__ PanelParams P) {
    const int z = blockIdx.z;
    const int LT = P.LT[z], JT = P.JT[z], K = P.K[z], l = P.l[z];
    const int j0 = blockIdx.x * 8, k0 = blockIdx.y * 128;
    if (j0 >= JT * LT || k0 >= K) return;
    const int tid = threadIdx.x, c = tid & 7, kq = tid >> 3;
    constexpr int kPad = 33;  // words per (t, c, part) row: bank-spread across c
    __shared__ uint32_t S[kOzMaxMod][8][2][kPad];
    const int T = TT > 0 ? TT : P.k.T;
    const int j = j0 + c;
    double vr[4], vi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int k = k0 + 4 * kq + u;
        cplx v = mk(0.0, 0.0);
        int sc = 0;
        if (j < l && k < K) {
            v = P.X[z][(long long)k * P.ldx[z] + j];
            sc = P.sx[z][j] + oz_exp_or0(P.kexp[z][k]);
        }
        vr[u] = rint(oz_scale(v.x, sc));
        vi[u] = rint(oz_scale(v.y, sc));
        if (!isfinite(vr[u])) vr[u] = 0.0;
        if (!isfinite(vi[u])) vi[u] = 0.0;
    }
    if constexpr (TT > 0) {
        oz_panel_pairs<TT, 0>(vr, vi, S, c, kq);
    } else {
        for (int t = 0; t < T; ++t) {
            const int md = P.k.mod[t];
            const double im = P.k.inv_md[t];
            const int lo = -(md / 2);
            uint32_t a = 0, b = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a |= (uint32_t)(oz_res(vr[u], md, im, lo) & 0xff) << (8 * u);
                b |= (uint32_t)(oz_res(vi[u], md, im, lo) & 0xff) << (8 * u);
            }
            S[t][c][0][kq] = a;
            S[t][c][1][kq] = b;
        }
    }
    __syncthreads();
    const int jt = j0 / LT, jj0 = j0 % LT, kb = blockIdx.y;
    // B' tiles [t·JT + jt][part][kb][2LT rows][128 bytes of K]
    int8_t* bres = P.bres[z];
    const long long tile = 2ll * LT * 128;
    // 16-byte pieces: (t, c, which, part, piece) — T·8·2·2·8 of them
    const int pieces = T * 8 * 2 * 2 * 8;
    for (int q = tid; q < pieces; q += 256) {
        const int piece = q & 7, part = (q >> 3) & 1, which = (q >> 4) & 1, cc = (q >> 5) & 7, t = q >> 8;
        // which 0 (re row): part0 = re, part1 = sg·im;  which 1 (im row): part0 = im, part1 = -sg·re
        const int src = which == 0 ? (part == 0 ? 0 : 1) : (part == 0 ? 1 : 0);
        const bool neg = part == 1 && ((which == 0) ? (P.sg < 0) : (P.sg > 0));
        const uint32_t* w = &S[t][cc][src][piece * 4];
        uint4 v = make_uint4(w[0], w[1], w[2], w[3]);
        if (neg) {
            v.x = __vneg4(v.x); v.y = __vneg4(v.y); v.z = __vneg4(v.z); v.w = __vneg4(v.w);
        }
        const int r = which * LT + jj0 + cc;
        const long long blk = ((long long)(t * JT + jt) * 2 + part) * P.nkbx[z] + kb;
        *reinterpret_cast<uint4*>(bres + blk * tile + (long long)r * 128 + piece * 16) = v;
    }
}

// ---- the INT8 tcgen05 GEMM --------------------------------------------------------------------
// Tile: 256 rows (two 128-row accumulators, 448 of TMEM's 512 columns), one CTA per SM.  (kHalves = 1
// — 128-row tiles, 2 stages, two CTAs per SM so one CTA's epilogue overlaps the other's loads —
// measured 1.42 vs 1.22 ms per 48-bond product: the panel's L2 re-reads double.)  This one-CTA-
// per-tile kernel is the A/B form (RRSVD_B200_OZAKI_PERSISTENT=0) of oz_gemm_persistent_kernel.
constexpr int kHalves = 2;
constexpr int kBM = 128 * kHalves;
constexpr int kThreads = 128 * kHalves;
constexpr int kTmemCols = 256 * kHalves;
constexpr int kBK = 128;      // bytes of K per stage = one 128B swizzle atom
constexpr int kStages = kHalves == 1 ? 2 : 3;
constexpr int kStageA = kBM * kBK;
constexpr int kStageB = 256 * kBK;           // up to N' = 256 rows
constexpr int kStageBytes = kStageA + kStageB;
constexpr int kGemmSmem = kStages * kStageBytes + 1024;  // + alignment slack

struct alignas(64) GemmParams {
    CUtensorMap mapA[kProdGroup];
    CUtensorMap mapB[kProdGroup];
    int M[kProdGroup], nkb[kProdGroup], LT[kProdGroup], JT[kProdGroup];
    uint8_t* out[kProdGroup];
    long long out_plane[kProdGroup];
    int out_ld[kProdGroup];
    int tile_begin[kProdGroup + 1];  // persistent kernel: tiles of problem z are [tile_begin[z], tile_begin[z+1])
    int count;
    int T;
    int mod[kOzMaxMod], w[kOzMaxMod];
    unsigned magic[kOzMaxMod], off[kOzMaxMod];
};
static_assert(sizeof(GemmParams) <= 32764, "kernel parameter space");

__device__ __forceinline__ void ob_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void ob_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ob_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void ob_tma5(void* dst, const CUtensorMap* map, uint64_t* bar, int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %3, %4, %5, %6}], [%2];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(0), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}
// shared-memory matrix descriptor, 128-byte swizzle (tcgen05 "version 1" descriptors)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// Epilogue of one 128-row accumulator (warp's TMEM lane quarter q, accumulator column base acc):
// each int32 D reduced to t = (D mod m)·w mod m by two integer Barrett steps (D + off >= 0), one
// byte per output, 16 outputs per 16-byte store of the thread's row.
__device__ __forceinline__ void oz_epilogue_rows(uint32_t tmem, int q, int acc, int Nn, bool store, uint8_t* dst,
                                                 int md, int w, unsigned mg, unsigned off) {
    for (int ch = 0; ch < Nn / 16; ++ch) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc + ch * 16, v);
        uint32_t pk[4] = {0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const unsigned x = v[u] + off;
            int r = (int)(x - __umulhi(x, mg) * md);  // in [-m, m)
            r += (r >> 31) & md;                       // [0, m)
            const unsigned p = (unsigned)(r * w);      // < 2^16
            int tt = (int)(p - __umulhi(p, mg) * md);
            tt += (tt >> 31) & md;
            pk[u >> 2] |= (uint32_t)tt << (8 * (u & 3));
        }
        if (store) *reinterpret_cast<uint4*>(dst + ch * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// OPA = kOpN: A tile K-major ([row][k], the residue planes' own layout); kOpC: MN-major.
template <int OPA>
__global__ void __launch_bounds__(kThreads, 3 - kHalves) oz_gemm_kernel(const __grid_constant__ GemmParams P) {
    const int z = blockIdx.z;
    const int M = P.M[z], JT = P.JT[z], LT = P.LT[z];
    const int m0 = blockIdx.x * kBM;
    const int t = blockIdx.y / JT, jt = blockIdx.y % JT;
    if (m0 >= M || t >= P.T) return;
    const int Nn = 2 * LT;
    const int nk = 2 * P.nkb[z];

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], done;
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ob_init(&full[s], 1);
            ob_init(&empty[s], 1);
        }
        ob_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 0) {
      if (lane == 0) {
        // ---- TMA producer
        const CUtensorMap* mA = &P.mapA[z];
        const CUtensorMap* mB = &P.mapB[z];
        const unsigned bytes = kStageA + Nn * kBK;
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % kStages;
            if (kb >= kStages) ob_wait(&empty[s], ((kb / kStages) - 1) & 1);
            uint8_t* sa = smem + s * kStageBytes;
            uint8_t* sb = sa + kStageA;
            const int part = kb >= P.nkb[z] ? 1 : 0;
            ob_expect_tx(&full[s], bytes);
            const int kb_ = kb - part * P.nkb[z];
            for (int h = 0; h < kHalves; ++h) {
                if (OPA == kOpN) ob_tma5(sa + h * 128 * kBK, mA, &full[s], kb_, m0 / 128 + h, 2 * t + part);
                else ob_tma5(sa + h * 128 * kBK, mA, &full[s], m0 / 128 + h, kb_, 2 * t + part);
            }
            ob_tma5(sb, mB, &full[s], kb_, part, t * JT + jt);
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      if (lane == 0) {
        // ---- MMA issuer: per stage, 4 K-steps of 32 x 2 row halves
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((OPA == kOpC ? 1u : 0u) << 15) |
                               ((uint32_t)(Nn >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % kStages;
            ob_wait(&full[s], (kb / kStages) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * kStageBytes);
            const uint32_t sb = sa + kStageA;
#pragma unroll
            for (int ks = 0; ks < kBK / 32; ++ks) {
                const uint64_t bdesc = sw128_desc(sb + ks * 32, 16, 1024);
#pragma unroll
                for (int h = 0; h < kHalves; ++h) {
                    const uint32_t abase = sa + h * 128 * kBK;
                    const uint64_t adesc = OPA == kOpN ? sw128_desc(abase + ks * 32, 16, 1024)
                                                       : sw128_desc(abase + ks * 32 * 128, 128 * kBK, 1024);
                    mma_i8(tmem + h * 256, adesc, bdesc, idesc, (kb | ks) != 0);
                }
            }
            mma_commit(&empty[s]);
        }
        mma_commit(&done);
      }
      __syncwarp();
    }

    // ---- epilogue: warp w reads TMEM lanes 32(w%4).. of accumulator w/4
    ob_wait(&done, 0);
    tc_fence_after();
    {
        const int q = warp & 3, h = warp >> 2;
        const int row = m0 + h * 128 + q * 32 + lane;
        uint8_t* dst = P.out[z] + (long long)t * P.out_plane[z] + (long long)row * P.out_ld[z] + jt * Nn;
        oz_epilogue_rows(tmem, q, h * 256, Nn, row < M, dst, P.mod[t], P.w[t], P.magic[t], P.off[t]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
}

// The persistent form: one CTA per SM walks the tiles (z, t, jt, m-block; m-block fastest so the
// CTAs sharing a B' panel run together) with warp-specialised roles — warp 0 issues TMA, warp 1
// issues tcgen05.mma, warps 2..9 drain TMEM.  The smem ring and its phases run on across tiles, so
// the producer keeps loading the next tile while the epilogue of the previous one reads TMEM (the
// MMAs of the next tile wait only for the accumulators to be drained: tmem_empty).
struct TileCoord {
    int z, t, jt, m0;
};
__device__ __forceinline__ TileCoord oz_tile(const GemmParams& P, int tile) {
    int z = 0;
    while (z + 1 < P.count && tile >= P.tile_begin[z + 1]) ++z;
    const int local = tile - P.tile_begin[z];
    const int mbs = (P.M[z] + kBM - 1) / kBM;
    const int y = local / mbs;
    return {z, y / P.JT[z], y % P.JT[z], (local % mbs) * kBM};
}

// Separate rings: A (HBM stream) 5 deep, B' (L2-resident panel) 2 deep, each with its own producer
// warp, so the A prefetch depth is not gated by the panel's ring.
constexpr int kAStages = 4, kBStages = 3;
constexpr int kPSmem = (kAStages + kBStages) * 32768 + 1024;
constexpr int kPThreads = 352;  // warp 0: A producer, 1: MMA, 2: B' producer, 3..10: epilogue
template <int OPA>
__global__ void __launch_bounds__(kPThreads, 1) oz_gemm_persistent_kernel(const __grid_constant__ GemmParams P) {
    static_assert(kHalves == 2, "persistent tiles are 256 rows");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ringA = smem;
    uint8_t* ringB = smem + kAStages * 32768;
    __shared__ __align__(8) uint64_t afull[kAStages], aempty[kAStages], bfull[kBStages], bempty[kBStages], tfull, tempty;
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = P.tile_begin[P.count];

    if (threadIdx.x == 0) {
        for (int s = 0; s < kAStages; ++s) {
            ob_init(&afull[s], 1);
            ob_init(&aempty[s], 1);
        }
        for (int s = 0; s < kBStages; ++s) {
            ob_init(&bfull[s], 1);
            ob_init(&bempty[s], 1);
        }
        ob_init(&tfull, 1);
        ob_init(&tempty, 8);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 0 || warp == 2) {
        if (lane == 0) {  // ---- TMA producers: warp 0 streams A, warp 2 the panel B'
            const bool isA = warp == 0;
            const int S = isA ? kAStages : kBStages;
            uint64_t* fullb = isA ? afull : bfull;
            uint64_t* emptyb = isA ? aempty : bempty;
            uint8_t* ring = isA ? ringA : ringB;
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const TileCoord tc = oz_tile(P, tile);
                const CUtensorMap* map = isA ? &P.mapA[tc.z] : &P.mapB[tc.z];
                const int Nn = 2 * P.LT[tc.z], nkb = P.nkb[tc.z];
                const unsigned bytes = isA ? kStageA : Nn * kBK;
                for (int kb = 0; kb < 2 * nkb; ++kb, ++it) {
                    const int s = it % S, use = it / S;
                    if (use > 0) ob_wait(&emptyb[s], (use - 1) & 1);
                    uint8_t* dst = ring + s * 32768;
                    const int part = kb >= nkb ? 1 : 0, kk = kb - part * nkb;
                    ob_expect_tx(&fullb[s], bytes);
                    if (isA) {
                        for (int h = 0; h < 2; ++h) {
                            if (OPA == kOpN) ob_tma5(dst + h * 128 * kBK, map, &fullb[s], kk, tc.m0 / 128 + h, 2 * tc.t + part);
                            else ob_tma5(dst + h * 128 * kBK, map, &fullb[s], tc.m0 / 128 + h, kk, 2 * tc.t + part);
                        }
                    } else {
                        ob_tma5(dst, map, &fullb[s], kk, part, tc.t * P.JT[tc.z] + tc.jt);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            int it = 0, tcount = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
                const TileCoord tc = oz_tile(P, tile);
                const int Nn = 2 * P.LT[tc.z], nk = 2 * P.nkb[tc.z];
                const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((OPA == kOpC ? 1u : 0u) << 15) |
                                       ((uint32_t)(Nn >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                if (tcount > 0) ob_wait(&tempty, (tcount - 1) & 1);
                tc_fence_after();
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int sa_ = it % kAStages, sb_ = it % kBStages;
                    ob_wait(&afull[sa_], (it / kAStages) & 1);
                    ob_wait(&bfull[sb_], (it / kBStages) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(ringA + sa_ * 32768);
                    const uint32_t sb = smem_u32(ringB + sb_ * 32768);
#pragma unroll
                    for (int ks = 0; ks < kBK / 32; ++ks) {
                        const uint64_t bdesc = sw128_desc(sb + ks * 32, 16, 1024);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t abase = sa + h * 128 * kBK;
                            const uint64_t adesc = OPA == kOpN ? sw128_desc(abase + ks * 32, 16, 1024)
                                                               : sw128_desc(abase + ks * 32 * 128, 128 * kBK, 1024);
                            mma_i8(tmem + h * 256, adesc, bdesc, idesc, (kb | ks) != 0);
                        }
                    }
                    mma_commit(&aempty[sa_]);
                    mma_commit(&bempty[sb_]);
                }
                mma_commit(&tfull);
            }
        }
        __syncwarp();
    } else {  // ---- epilogue: warps 3..10; warp w reads TMEM lanes 32(w%4).. of accumulator (w-3)/4
        const int q = warp & 3, h = (warp - 3) >> 2;
        int tcount = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
            const TileCoord tc = oz_tile(P, tile);
            const int Nn = 2 * P.LT[tc.z];
            ob_wait(&tfull, tcount & 1);
            tc_fence_after();
            const int row = tc.m0 + h * 128 + q * 32 + lane;
            uint8_t* dst = P.out[tc.z] + (long long)tc.t * P.out_plane[tc.z] + (long long)row * P.out_ld[tc.z] + tc.jt * Nn;
            oz_epilogue_rows(tmem, q, h * 256, Nn, row < P.M[tc.z], dst, P.mod[tc.t], P.w[tc.t], P.magic[tc.t],
                             P.off[tc.t]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&tempty)) : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
}

// ---- CRT --------------------------------------------------------------------------------------
// D/M = frac_sym( sum_t t_t / m_t ) in 128-bit fixed point, from the top 96 bits of floor(2^128/m_t)
// (truncation error < T·2^8·2^32 units of 2^-128 — 2^-84 of M, far below one unit of kA + kX).
struct CrtParams {
    const uint8_t* out[kProdGroup];
    long long out_plane[kProdGroup];
    int out_ld[kProdGroup];
    int M[kProdGroup], l[kProdGroup], LT[kProdGroup], kA[kProdGroup];
    const int* oexp[kProdGroup];  // exponents of the output rows
    const int* abad[kProdGroup];
    const int* sx[kProdGroup];
    const int* xbad[kProdGroup];
    cplx* C[kProdGroup];
    long long ldc[kProdGroup];
    int acc[kProdGroup];
    OzConst k;
};

// the signed value D/M·2^128 of four consecutive outputs' residues (one uchar4 per modulus)
template <int TT>
__device__ __forceinline__ void oz_crt4(const uint8_t* p, long long plane, const OzConst& k, double (&val)[4]) {
    unsigned long long a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0};
#pragma unroll
    for (int t = 0; t < (TT > 0 ? TT : kOzMaxMod); ++t) {
        if (TT == 0 && t >= k.T) break;
        const uint32_t b = *reinterpret_cast<const uint32_t*>(p + (long long)t * plane);
        const unsigned c0 = k.c3[t][0], c1 = k.c3[t][1], c2 = k.c3[t][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned r = (b >> (8 * u)) & 0xffu;
            a0[u] += (unsigned long long)r * c0;
            a1[u] += (unsigned long long)r * c1;
            a2[u] += (unsigned long long)r * c2;
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        // F = a0·2^32 + a1·2^64 + a2·2^96 (mod 2^128)
        unsigned long long lo = a0[u] << 32;
        unsigned long long hi = (a0[u] >> 32) + a1[u] + (a2[u] << 32);
        const bool neg = (long long)hi < 0;
        if (neg) {
            lo = ~lo + 1ull;
            hi = ~hi + (lo == 0ull ? 1ull : 0ull);
        }
        const double mag = (double)hi * 18446744073709551616.0 + (double)lo;
        val[u] = neg ? -mag : mag;
    }
}

// one thread = four consecutive output columns of one row
template <int TT>
__global__ void __launch_bounds__(256) oz_crt_kernel(const __grid_constant__ CrtParams P) {
    // one thread = one part (re or im) of four consecutive outputs: half the accumulator
    // registers of a both-parts thread, twice the threads in flight
    const int z = blockIdx.y;
    const int M = P.M[z], l = P.l[z], LT = P.LT[z];
    const int JT = (l + LT - 1) / LT;
    const int groups = JT * (LT / 4);
    const long long total = 2ll * M * groups;
    const bool abad = *P.abad[z] != 0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int part = (int)(e & 1);
        const long long eg = e >> 1;
        const int row = (int)(eg / groups), gi = (int)(eg % groups);
        const int jt = gi / (LT / 4), jj = (gi % (LT / 4)) * 4;
        const int j0 = jt * LT + jj;
        if (j0 >= l) continue;
        const uint8_t* base = P.out[z] + (long long)row * P.out_ld[z] + (long long)jt * 2 * LT + part * LT + jj;
        double val[4];
        oz_crt4<TT>(base, P.out_plane[z], P.k, val);
        const int eo = oz_exp_or0(P.oexp[z][row]) - P.kA[z];
        double* dst = reinterpret_cast<double*>(P.C[z] + (long long)row * P.ldc[z] + j0) + part;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = j0 + u;
            if (j >= l || j >= (jt + 1) * LT) break;
            double v = oz_scale(val[u] * P.k.mscale, eo - P.sx[z][j]);
            if (abad || P.xbad[z][j]) v = NAN;
            dst[2 * u] = P.acc[z] ? dst[2 * u] + v : v;
        }
    }
}

// ---- host -----------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 oz_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

void encode_u8(rrsvd_b200_ctx* c, CUtensorMap* map, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
               const cuuint32_t* box) {
    const auto enc = oz_encoder();
    if (enc == nullptr) throw_numeric(c, "ozaki: cuTensorMapEncodeTiled unavailable");
    const cuuint32_t one[5] = {1, 1, 1, 1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<void*>(base), dims, strides, box, one,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw_numeric(c, "ozaki: tensor map encoding failed");
}

std::atomic<unsigned long long> g_optin{0};

}  // namespace

int ozaki_inner_moduli() {
    static const int T = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI_INNER");
        const int v = e ? std::atoi(e) : 14;
        return v >= 8 && v <= kOzMaxMod ? v : 0;
    }();
    return T;
}

int ozaki_moduli() {
    static const int T = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI");
        if (e == nullptr) return 15;
        const int v = std::atoi(e);
        if (v <= 0) return 0;
        return std::min(kOzMaxMod, std::max(8, v));
    }();
    return T;
}

static bool oz_persistent() {  // RRSVD_B200_OZAKI_PERSISTENT=0: one CTA per tile (A/B)
    static const bool on = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI_PERSISTENT");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}

int ozaki_tail() {
    static const int v = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI_TAIL");
        return e == nullptr ? 0 : std::max(0, std::atoi(e));
    }();
    return v;
}

double ozaki_min_work() {
    static const double v = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI_MIN_WORK");
        return e ? std::atof(e) : 8.0e6;
    }();
    return v;
}

double ozaki_max_bytes() {
    static const double v = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI_MAX_GB");
        return (e ? std::atof(e) : 32.0) * 1073741824.0;
    }();
    return v;
}

// Below ~512 rows or columns the preparation and CRT overheads eat the INT8 GEMM's advantage (C2's
// 256 x 256 bonds: 29.6 vs 30.7 steps/s emulated vs DMMA); RRSVD_B200_OZAKI_MIN overrides.
bool ozaki_usable(int m, int n, int l) {
    static const int lo = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI_MIN");
        return e ? std::max(128, std::atoi(e)) : 512;
    }();
    return ozaki_moduli() > 0 && std::min(m, n) >= lo && std::max(m, n) <= 32768 && l >= 1;
}

std::vector<OzakiA> ozaki_prepare_many(rrsvd_b200_ctx* c, const std::vector<OzSrc>& src, int T,
                                       std::vector<void*>* keep) {
    const OzConst& k = oz_const(T);
    // keep != nullptr: the planes outlive the call (stream-ordered allocations the caller frees)
    auto alloc = [&](size_t bytes) -> void* {
        if (keep == nullptr) return ws_alloc(c, bytes);
        void* p = nullptr;
        check_cuda(c, cudaMallocAsync(&p, bytes < 16 ? 16 : bytes, c->stream), "cudaMallocAsync(ozaki planes)");
        keep->push_back(p);
        return p;
    };
    std::vector<OzakiA> out(src.size());
    for (size_t base = 0; base < src.size(); base += kPrepGroup) {
        const int cnt = (int)std::min<size_t>(kPrepGroup, src.size() - base);
        PrepParams P{};
        P.count = cnt;
        P.k = k;
        P.bad = static_cast<int*>(alloc(sizeof(int) * cnt));
        check_cuda(c, cudaMemsetAsync(P.bad, 0, sizeof(int) * cnt, c->stream), "ozaki memset");
        long long max_chunks = 0;
        int max_m = 1, max_n = 1;
        double bytes = 0.0;
        for (int i = 0; i < cnt; ++i) {
            const OzSrc& s = src[base + i];
            OzakiA& a = out[base + i];
            a.m = s.m;
            a.n = s.n;
            a.T = T;
            a.nib = (s.m + 127) / 128;
            a.nkb = (s.n + 127) / 128;
            a.kA = std::min(56, (oz_total_bits(k, std::max(s.m, s.n)) + 1) / 2);
            a.res = static_cast<int8_t*>(alloc((size_t)T * 2 * a.nib * a.nkb * 16384));
            a.rowexp = static_cast<int*>(alloc(sizeof(int) * s.m));
            a.colexp = static_cast<int*>(alloc(sizeof(int) * s.n));
            check_cuda(c, cudaMemsetAsync(a.colexp, 0xC0, sizeof(int) * s.n, c->stream), "ozaki memset");
            a.bad = P.bad + i;
            P.A[i] = s.A;
            P.lda[i] = s.lda;
            P.nib[i] = a.nib;
            P.nkb[i] = a.nkb;
            P.m[i] = s.m;
            P.n[i] = s.n;
            P.kA[i] = a.kA;
            P.res[i] = a.res;
            P.rowexp[i] = a.rowexp;
            P.colexp[i] = a.colexp;
            if (s.total_sq != nullptr) {
                P.rowsq[i] = static_cast<double*>(alloc(sizeof(double) * s.m));
                P.total_sq[i] = s.total_sq;
                P.nonfinite[i] = s.nonfinite;
            }
            max_chunks = std::max(max_chunks, (long long)a.nib * 128 * a.nkb * 16);
            bytes += 3.0 * 16 * s.m * (double)s.n + 2.0 * T * a.nib * a.nkb * 16384;  // A read 3x, planes written
            max_m = std::max(max_m, s.m);
            max_n = std::max(max_n, s.n);
        }
        cudaEvent_t ea = nullptr, eb = nullptr;
        if (c->gemm_timing) {
            ea = pooled_event(c);
            eb = pooled_event(c);
            check_cuda(c, cudaEventRecord(ea, c->stream), "event record");
        }
        oz_rowexp_kernel<<<dim3((max_m + 7) / 8, cnt), 256, 0, c->stream>>>(P);
        check_launch(c, "oz_rowexp_kernel");
        bool any_sq = false;
        for (int i = 0; i < cnt; ++i) any_sq = any_sq || P.total_sq[i] != nullptr;
        if (any_sq) {
            oz_sumsq_final_kernel<<<cnt, 32, 0, c->stream>>>(P);
            check_launch(c, "oz_sumsq_final_kernel");
        }
        const int rch = std::max(1, std::min(64, (4 * kNumSMs * 32) / (cnt * max_n)));  // >= ~4 CTAs/SM
        oz_colexp_kernel<<<dim3((max_n + 31) / 32, rch, cnt), 256, 0, c->stream>>>(P);
        check_launch(c, "oz_colexp_kernel");
        const int gx = (int)std::min<long long>((max_chunks + 255) / 256, 8 * kNumSMs);
        if (T == 15) oz_resid_a_kernel<15><<<dim3(gx, cnt), 256, 0, c->stream>>>(P);
        else if (T == 14) oz_resid_a_kernel<14><<<dim3(gx, cnt), 256, 0, c->stream>>>(P);
        else if (T == 16) oz_resid_a_kernel<16><<<dim3(gx, cnt), 256, 0, c->stream>>>(P);
        else oz_resid_a_kernel<0><<<dim3(gx, cnt), 256, 0, c->stream>>>(P);
        check_launch(c, "oz_resid_a_kernel");
        if (c->gemm_timing) {
            check_cuda(c, cudaEventRecord(eb, c->stream), "event record");
            c->pending.push_back({ea, eb, 0.0, 0.0, c->gemm_tag, 1, 1, bytes});
        }
    }
    return out;
}

void ozaki_product_many(rrsvd_b200_ctx* c, GemmOp op, const std::vector<OzProduct>& ps) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(g_optin.load() & bit)) {
        check_cuda(c, cudaFuncSetAttribute(oz_gemm_kernel<kOpN>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem),
                   "ozaki smem opt-in");
        check_cuda(c, cudaFuncSetAttribute(oz_gemm_kernel<kOpC>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem),
                   "ozaki smem opt-in");
        check_cuda(c, cudaFuncSetAttribute(oz_gemm_persistent_kernel<kOpN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kPSmem), "ozaki smem opt-in");
        check_cuda(c, cudaFuncSetAttribute(oz_gemm_persistent_kernel<kOpC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kPSmem), "ozaki smem opt-in");
        g_optin.fetch_or(bit);
    }
    for (size_t base = 0; base < ps.size(); base += kProdGroup) {
        const int cnt = (int)std::min<size_t>(kProdGroup, ps.size() - base);
        // a product may use only A's first T planes (fewer moduli, X to fewer bits)
        const auto prod_T = [](const OzProduct& p) { return p.T > 0 && p.T < p.a->T ? p.T : p.a->T; };
        const int T = prod_T(ps[base]);
        const OzConst& k = oz_const(T);
        PanelParams PP{};
        GemmParams G{};
        CrtParams CP{};
        PP.sg = op == kOpN ? -1 : 1;
        PP.k = k;
        CP.k = k;
        G.count = cnt;
        G.T = T;
        for (int t = 0; t < T; ++t) {
            G.mod[t] = k.mod[t];
            G.w[t] = k.w[t];
            G.magic[t] = k.magic[t];
            G.off[t] = k.off[t];
        }
        int max_cols = 8, max_mb = 1, max_jt = 1, max_k = 1;
        double bytes = 0.0, gemm_bytes = 0.0;
        long long max_el = 1;
        double flops = 0.0;
        for (int i = 0; i < cnt; ++i) {
            const OzProduct& p = ps[base + i];
            const OzakiA& a = *p.a;
            if (prod_T(p) != T) throw_contract(c, "ozaki: mixed moduli counts in one batch");
            const int K = op == kOpN ? a.n : a.m, Mr = op == kOpN ? a.m : a.n;
            const int JT = (p.l + 127) / 128;
            const int LT = ((p.l + JT - 1) / JT + 7) / 8 * 8;
            const int nkbx = (K + 127) / 128;
            const int ncol = 2 * JT * LT;
            const int kX = std::min(56, oz_total_bits(k, K) - a.kA);
            int8_t* bres = ws_get<int8_t>(c, (size_t)T * JT * 2 * nkbx * 2 * LT * 128);
            int* sx = ws_get<int>(c, (size_t)JT * LT);
            int* xbad = ws_get<int>(c, (size_t)JT * LT);
            uint8_t* out = ws_get<uint8_t>(c, (size_t)T * Mr * ncol);
            PP.X[i] = p.X;
            PP.ldx[i] = p.ldx;
            PP.nkbx[i] = nkbx;
            PP.K[i] = K;
            PP.l[i] = p.l;
            PP.LT[i] = LT;
            PP.JT[i] = JT;
            PP.kX[i] = kX;
            PP.kexp[i] = op == kOpN ? a.colexp : a.rowexp;
            PP.bres[i] = bres;
            PP.sx[i] = sx;
            PP.xbad[i] = xbad;
            {  // A tiles [2T][nib][nkb][128][128]: one box = one tile
                const cuuint64_t dims[5] = {128, 128, (cuuint64_t)a.nkb, (cuuint64_t)a.nib, 2ull * T};
                const cuuint64_t str[4] = {128, 16384, 16384ull * a.nkb, 16384ull * a.nkb * a.nib};
                const cuuint32_t box[5] = {128, 128, 1, 1, 1};
                encode_u8(c, &G.mapA[i], a.res, dims, str, box);
            }
            {  // B' tiles [T·JT][2][nkbx][2LT][128]
                const cuuint64_t rows = 2ull * LT;
                const cuuint64_t dims[5] = {128, rows, (cuuint64_t)nkbx, 2, (cuuint64_t)T * JT};
                const cuuint64_t str[4] = {128, 128 * rows, 128 * rows * nkbx, 256 * rows * nkbx};
                const cuuint32_t box[5] = {128, (cuuint32_t)rows, 1, 1, 1};
                encode_u8(c, &G.mapB[i], bres, dims, str, box);
            }
            G.M[i] = Mr;
            G.nkb[i] = (K + kBK - 1) / kBK;
            G.LT[i] = LT;
            G.JT[i] = JT;
            G.out[i] = out;
            G.out_plane[i] = (long long)Mr * ncol;
            G.out_ld[i] = ncol;
            CP.out[i] = out;
            CP.out_plane[i] = (long long)Mr * ncol;
            CP.out_ld[i] = ncol;
            CP.M[i] = Mr;
            CP.l[i] = p.l;
            CP.LT[i] = LT;
            CP.kA[i] = a.kA;
            CP.oexp[i] = op == kOpN ? a.rowexp : a.colexp;
            CP.abad[i] = a.bad;
            CP.sx[i] = sx;
            CP.xbad[i] = xbad;
            CP.C[i] = p.C;
            CP.ldc[i] = p.ldc;
            CP.acc[i] = p.accumulate;
            max_cols = std::max(max_cols, JT * LT);
            max_mb = std::max(max_mb, (Mr + kBM - 1) / kBM);
            max_jt = std::max(max_jt, JT);
            max_el = std::max(max_el, 2ll * Mr * JT * (LT / 4));
            max_k = std::max(max_k, K);
            flops += 8.0 * Mr * (double)p.l * K;
            // X read; B' written + read; A residues read; residue products written + read; C written
            bytes += 16.0 * K * p.l + 2.0 * T * JT * 2 * nkbx * 2 * LT * 128 + 2.0 * T * a.nib * a.nkb * 16384 +
                     2.0 * T * Mr * ncol + 16.0 * Mr * p.l;
            gemm_bytes += 2.0 * T * a.nib * a.nkb * 16384 + (double)T * JT * 2 * nkbx * 2 * LT * 128 + (double)T * Mr * ncol;
        }
        int ntiles = 0;
        for (int i = 0; i < cnt; ++i) {
            G.tile_begin[i] = ntiles;
            ntiles += (G.M[i] + kBM - 1) / kBM * T * G.JT[i];
        }
        G.tile_begin[cnt] = ntiles;
        cudaEvent_t ea = nullptr, eb = nullptr;
        if (c->gemm_timing) {
            ea = pooled_event(c);
            eb = pooled_event(c);
            check_cuda(c, cudaEventRecord(ea, c->stream), "event record");
        }
        oz_xmax_kernel<<<dim3((max_cols + 7) / 8, cnt), 256, 0, c->stream>>>(PP);
        check_launch(c, "oz_xmax_kernel");
        const dim3 gb((max_cols + 7) / 8, (max_k + 127) / 128, cnt);
        if (T == 15) oz_resid_b_kernel<15><<<gb, 256, 0, c->stream>>>(PP);
        else if (T == 14) oz_resid_b_kernel<14><<<gb, 256, 0, c->stream>>>(PP);
        else if (T == 16) oz_resid_b_kernel<16><<<gb, 256, 0, c->stream>>>(PP);
        else oz_resid_b_kernel<0><<<gb, 256, 0, c->stream>>>(PP);
        check_launch(c, "oz_resid_b_kernel");
        cudaEvent_t ga = nullptr, gb2 = nullptr;
        if (c->gemm_timing) {
            ga = pooled_event(c);
            gb2 = pooled_event(c);
            check_cuda(c, cudaEventRecord(ga, c->stream), "event record");
        }
        if (oz_persistent()) {
            static const int cap = [] {  // RRSVD_B200_OZAKI_GRID: CTAs of the persistent GEMM (A/B)
                const char* e = std::getenv("RRSVD_B200_OZAKI_GRID");
                return e ? std::max(1, std::min(kNumSMs, std::atoi(e))) : kNumSMs;
            }();
            const int grid = std::min(ntiles, cap);
            if (op == kOpN)
                oz_gemm_persistent_kernel<kOpN><<<grid, kPThreads, kPSmem, c->stream>>>(G);
            else
                oz_gemm_persistent_kernel<kOpC><<<grid, kPThreads, kPSmem, c->stream>>>(G);
        } else if (op == kOpN) {
            oz_gemm_kernel<kOpN><<<dim3(max_mb, T * max_jt, cnt), kThreads, kGemmSmem, c->stream>>>(G);
        } else {
            oz_gemm_kernel<kOpC><<<dim3(max_mb, T * max_jt, cnt), kThreads, kGemmSmem, c->stream>>>(G);
        }
        check_launch(c, "oz_gemm_kernel");
        if (c->gemm_timing) {
            check_cuda(c, cudaEventRecord(gb2, c->stream), "event record");
            c->pending.push_back({ga, gb2, 0.0, 0.0, c->gemm_tag, 1, 2, gemm_bytes});
        }
        const int gx = (int)std::min<long long>((max_el + 255) / 256, 8 * kNumSMs);
        if (T == 15) oz_crt_kernel<15><<<dim3(gx, cnt), 256, 0, c->stream>>>(CP);
        else if (T == 14) oz_crt_kernel<14><<<dim3(gx, cnt), 256, 0, c->stream>>>(CP);
        else if (T == 16) oz_crt_kernel<16><<<dim3(gx, cnt), 256, 0, c->stream>>>(CP);
        else oz_crt_kernel<0><<<dim3(gx, cnt), 256, 0, c->stream>>>(CP);
        check_launch(c, "oz_crt_kernel");
        if (c->gemm_timing) {
            check_cuda(c, cudaEventRecord(eb, c->stream), "event record");
            c->pending.push_back({ea, eb, flops, flops, c->gemm_tag, 1, 1, bytes});
        }
        if (debug_enabled()) {  // zero / non-finite output columns of every product (diagnostics)
            for (int i = 0; i < cnt; ++i) {
                const OzProduct& p = ps[base + i];
                const int Mr = op == kOpN ? p.a->m : p.a->n;
                std::vector<cplx> h((size_t)Mr * p.ldc);
                cudaMemcpyAsync(h.data(), p.C, h.size() * sizeof(cplx), cudaMemcpyDeviceToHost, c->stream);
                std::vector<int> xs(p.l);
                cudaMemcpyAsync(xs.data(), CP.sx[i], p.l * sizeof(int), cudaMemcpyDeviceToHost, c->stream);
                cudaStreamSynchronize(c->stream);
                int zc = 0, nf = 0;
                for (int j = 0; j < p.l; ++j) {
                    bool z = true;
                    for (int r = 0; r < Mr; ++r) {
                        const cplx v = h[(size_t)r * p.ldc + j];
                        if (v.x != 0.0 || v.y != 0.0) z = false;
                        if (!std::isfinite(v.x) || !std::isfinite(v.y)) ++nf;
                    }
                    zc += z;
                }
                std::fprintf(stderr, "[rrsvd_b200] ozaki op%d product %d: %d x %d, zero columns %d, non-finite %d, sx[0..3] %d %d %d %d\n",
                             (int)op, i, Mr, p.l, zc, nf, xs[0], xs[1], xs[2], xs[3]);
            }
        }
    }
}

}  // namespace rb

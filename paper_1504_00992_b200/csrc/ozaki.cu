// ozaki.cu — see ozaki.cuh for the scheme.  Four kernels per batch of products:
//   oz_resid_b  — per-column scale of X and its residue panel B' (K-major, [t][row][part][k]),
//   oz_gemm     — tcgen05.mma kind::i8: TMA (128B-swizzled boxes) -> 3-stage mbarrier ring ->
//                 one issuing thread -> two 128 x N' int32 accumulators in TMEM -> epilogue
//                 reducing each accumulator mod m_t (times w_t) to a uint8 residue plane,
//   oz_crt      — 128-bit fixed-point CRT of the T residues, scaled to FP64;
// plus, once per A, oz_rowmax, oz_colmax and oz_resid_a (its equilibrated residue planes).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "ozaki.cuh"

namespace rb {

namespace {

constexpr int kModuli[kOzMaxMod] = {256, 255, 253, 251, 247, 241, 239, 233,
                                    229, 227, 223, 217, 211, 199, 197, 193};

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
    long long lda[kPrepGroup], pitch[kPrepGroup];
    int m[kPrepGroup], n[kPrepGroup], kA[kPrepGroup];
    int8_t* res[kPrepGroup];
    unsigned long long* rowbits[kPrepGroup];  // [m]
    unsigned long long* colbits[kPrepGroup];  // [n] (zeroed)
    int* bad;                                 // [count] (zeroed)
    int count;
    OzConst k;
};

__global__ void __launch_bounds__(256) oz_rowmax_kernel(const __grid_constant__ PrepParams P) {
    const int z = blockIdx.y;
    const int m = P.m[z], n = P.n[z];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * 8 + warp;
    if (row >= m) return;
    const cplx* A = P.A[z] + (long long)row * P.lda[z];
    double mx = 0.0;
    int bad = 0;
    for (int c = lane; c < n; c += 32) {
        const cplx v = A[c];
        if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
        else mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    }
    mx = warp_max(mx);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        P.rowbits[z][row] = (unsigned long long)__double_as_longlong(mx);
        if (bad) atomicOr(&P.bad[z], 1);
    }
}

// block = 32 columns x 8 row groups over a chunk of rows
__global__ void __launch_bounds__(256) oz_colmax_kernel(const __grid_constant__ PrepParams P) {
    const int z = blockIdx.z;
    const int m = P.m[z], n = P.n[z];
    const int col = blockIdx.x * 32 + (threadIdx.x & 31), g = threadIdx.x >> 5;
    const int rows_per = (m + gridDim.y - 1) / gridDim.y;
    const int r0 = blockIdx.y * rows_per, r1 = min(m, r0 + rows_per);
    __shared__ double red[8][32];
    double mx = 0.0;
    if (col < n)
        for (int r = r0 + g; r < r1; r += 8) {
            const cplx v = P.A[z][(long long)r * P.lda[z] + col];
            const double a = fmax(fabs(v.x), fabs(v.y));
            if (isfinite(a) && a > 0.0) mx = fmax(mx, oz_scale(a, -oz_e(P.rowbits[z][r])));
        }
    red[g][threadIdx.x & 31] = mx;
    __syncthreads();
    if (g == 0 && col < n) {
        for (int i = 1; i < 8; ++i) mx = fmax(mx, red[i][threadIdx.x]);
        if (mx > 0.0) atomicMax(&P.colbits[z][col], (unsigned long long)__double_as_longlong(mx));
    }
}

// one thread = 16 consecutive columns of one row, both parts, all T moduli
__global__ void __launch_bounds__(256) oz_resid_a_kernel(const __grid_constant__ PrepParams P) {
    const int z = blockIdx.y;
    const int m = P.m[z], n = P.n[z];
    const long long pitch = P.pitch[z];
    const long long chunks_per_row = pitch / 16;
    const long long total = (long long)m * chunks_per_row;
    const cplx* A = P.A[z];
    int8_t* res = P.res[z];
    const long long plane = (long long)m * pitch;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(e / chunks_per_row);
        const int c0 = (int)(e % chunks_per_row) * 16;
        const int er = P.kA[z] - oz_e(P.rowbits[z][row]);
        double vr[16], vi[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int col = c0 + u;
            cplx x = mk(0.0, 0.0);
            int s = 0;
            if (col < n) {
                x = A[(long long)row * P.lda[z] + col];
                s = er - oz_e(P.colbits[z][col]);
            }
            vr[u] = rint(oz_scale(x.x, s));
            vi[u] = rint(oz_scale(x.y, s));
            if (!isfinite(vr[u])) vr[u] = 0.0;
            if (!isfinite(vi[u])) vi[u] = 0.0;
        }
        for (int t = 0; t < P.k.T; ++t) {
            const int md = P.k.mod[t], lo = P.k.lo[t];
            const double im = P.k.inv_md[t];
            uint32_t pr[4], pi[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                uint32_t a = 0, b = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    a |= (uint32_t)(oz_res(vr[4 * w + u], md, im, lo) & 0xff) << (8 * u);
                    b |= (uint32_t)(oz_res(vi[4 * w + u], md, im, lo) & 0xff) << (8 * u);
                }
                pr[w] = a;
                pi[w] = b;
            }
            int8_t* dst = res + (long long)(2 * t) * plane + (long long)row * pitch + c0;
            *reinterpret_cast<uint4*>(dst) = make_uint4(pr[0], pr[1], pr[2], pr[3]);
            *reinterpret_cast<uint4*>(dst + plane) = make_uint4(pi[0], pi[1], pi[2], pi[3]);
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
    long long ldx[kProdGroup], pitchK[kProdGroup];
    int K[kProdGroup], l[kProdGroup], LT[kProdGroup], JT[kProdGroup], kX[kProdGroup];
    const unsigned long long* kbits[kProdGroup];  // exponent source of the K rows
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
        for (int k = rg; k < K; k += 32) {
            const cplx v = P.X[z][(long long)k * P.ldx[z] + j];
            if (!isfinite(v.x) || !isfinite(v.y)) {
                bad = 1;
            } else {
                const double a = fmax(fabs(v.x), fabs(v.y));
                if (a > 0.0) mx = fmax(mx, oz_scale(a, oz_e(P.kbits[z][k])));
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

// block = 8 columns x 128 K rows: residues into shared memory, then 128-byte rows of B'
__global__ void __launch_bounds__(256) oz_resid_b_kernel(const __grid_constant__ PanelParams P) {
    const int z = blockIdx.z;
    const int LT = P.LT[z], JT = P.JT[z], K = P.K[z], l = P.l[z];
    const int j0 = blockIdx.x * 8, k0 = blockIdx.y * 128;
    if (j0 >= JT * LT || k0 >= K) return;
    const int tid = threadIdx.x, c = tid & 7, rg = tid >> 3;
    const int j = j0 + c;
    __shared__ __align__(16) int8_t S[kOzMaxMod][8][2][128];
    const int sxj = j < l ? P.sx[z][j] : 0;
    const int T = P.k.T;
    for (int u = 0; u < 4; ++u) {
        const int kk = rg + 32 * u, k = k0 + kk;
        cplx v = mk(0.0, 0.0);
        int s = 0;
        if (j < l && k < K) {
            v = P.X[z][(long long)k * P.ldx[z] + j];
            s = sxj + oz_e(P.kbits[z][k]);
        }
        double vr = rint(oz_scale(v.x, s)), vi = rint(oz_scale(v.y, s));
        if (!isfinite(vr)) vr = 0.0;
        if (!isfinite(vi)) vi = 0.0;
        for (int t = 0; t < T; ++t) {
            S[t][c][0][kk] = (int8_t)oz_res(vr, P.k.mod[t], P.k.inv_md[t], P.k.lo[t]);
            S[t][c][1][kk] = (int8_t)oz_res(vi, P.k.mod[t], P.k.inv_md[t], P.k.lo[t]);
        }
    }
    __syncthreads();
    const long long pitchK = P.pitchK[z];
    const long long R = 2ll * JT * LT;
    const int jt = j0 / LT, jj0 = j0 % LT;
    int8_t* bres = P.bres[z];
    // 16-byte pieces: (t, c, which, part, piece) — T·8·2·2·8 of them
    const int pieces = T * 8 * 2 * 2 * 8;
    for (int q = tid; q < pieces; q += 256) {
        const int piece = q & 7, part = (q >> 3) & 1, which = (q >> 4) & 1, cc = (q >> 5) & 7, t = q >> 8;
        const long long kofs = k0 + piece * 16;
        if (kofs >= pitchK) continue;
        // which 0 (re row): part0 = re, part1 = sg·im;  which 1 (im row): part0 = im, part1 = -sg·re
        const int src = which == 0 ? (part == 0 ? 0 : 1) : (part == 0 ? 1 : 0);
        const bool neg = part == 1 && ((which == 0) ? (P.sg < 0) : (P.sg > 0));
        uint4 v = *reinterpret_cast<const uint4*>(&S[t][cc][src][piece * 16]);
        if (neg) {
            v.x = __vneg4(v.x); v.y = __vneg4(v.y); v.z = __vneg4(v.z); v.w = __vneg4(v.w);
        }
        const long long r = (long long)jt * 2 * LT + which * LT + jj0 + cc;
        *reinterpret_cast<uint4*>(bres + (((long long)t * R + r) * 2 + part) * pitchK + kofs) = v;
    }
}

// ---- the INT8 tcgen05 GEMM --------------------------------------------------------------------
constexpr int kBM = 256;      // two 128-row MMAs per K step (two TMEM accumulators)
constexpr int kBK = 128;      // bytes of K per stage = one 128B swizzle atom
constexpr int kStages = 3;
constexpr int kStageA = kBM * kBK;           // 32 KB
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
__device__ __forceinline__ void ob_tma4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
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

// OPA = kOpN: A tile K-major ([row][k], the residue planes' own layout); kOpC: MN-major.
template <int OPA>
__global__ void __launch_bounds__(256, 1) oz_gemm_kernel(const __grid_constant__ GemmParams P) {
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
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_slot)));
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
            const int k0 = (kb - part * P.nkb[z]) * kBK;
            ob_expect_tx(&full[s], bytes);
            if (OPA == kOpN) {
                ob_tma4(sa, mA, &full[s], k0, m0, part, t);
                ob_tma4(sa + 128 * kBK, mA, &full[s], k0, m0 + 128, part, t);
            } else {
                ob_tma4(sa, mA, &full[s], m0, k0, part, t);
                ob_tma4(sa + 128 * kBK, mA, &full[s], m0 + 128, k0, part, t);
            }
            ob_tma4(sb, mB, &full[s], k0, part, jt * Nn, t);
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
                for (int h = 0; h < 2; ++h) {
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
        const int md = P.mod[t], w = P.w[t];
        const unsigned mg = P.magic[t], off = P.off[t];
        uint8_t* dst = P.out[z] + (long long)t * P.out_plane[z] + (long long)row * P.out_ld[z] + jt * Nn;
        for (int ch = 0; ch < Nn / 16; ++ch) {
            uint32_t v[16];
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + h * 256 + ch * 16, v);
            uint32_t pk[4] = {0, 0, 0, 0};
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                // t = (D mod m)·w mod m by two Barrett reductions (integer only): D + off >= 0
                const unsigned x = v[u] + off;
                int r = (int)(x - __umulhi(x, mg) * md);   // in [-m, m)
                r += (r >> 31) & md;                        // [0, m)
                const unsigned p = (unsigned)(r * w);       // < 2^16
                int tt = (int)(p - __umulhi(p, mg) * md);
                tt += (tt >> 31) & md;
                pk[u >> 2] |= (uint32_t)tt << (8 * (u & 3));
            }
            if (row < M) *reinterpret_cast<uint4*>(dst + ch * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---- CRT --------------------------------------------------------------------------------------
// D/M = frac_sym( sum_t t_t / m_t ) in 128-bit fixed point, from the top 96 bits of floor(2^128/m_t)
// (truncation error < T·2^8·2^32 units of 2^-128 — 2^-84 of M, far below one unit of kA + kX).
struct CrtParams {
    const uint8_t* out[kProdGroup];
    long long out_plane[kProdGroup];
    int out_ld[kProdGroup];
    int M[kProdGroup], l[kProdGroup], LT[kProdGroup], kA[kProdGroup];
    const unsigned long long* obits[kProdGroup];  // exponent source of the output rows
    const int* abad[kProdGroup];
    const int* sx[kProdGroup];
    const int* xbad[kProdGroup];
    cplx* C[kProdGroup];
    long long ldc[kProdGroup];
    OzConst k;
};

// the signed value D/M·2^128 of four consecutive outputs' residues (one uchar4 per modulus)
__device__ __forceinline__ void oz_crt4(const uint8_t* p, long long plane, const OzConst& k, double (&val)[4]) {
    unsigned long long a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0};
    for (int t = 0; t < k.T; ++t) {
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
__global__ void __launch_bounds__(256) oz_crt_kernel(const __grid_constant__ CrtParams P) {
    const int z = blockIdx.y;
    const int M = P.M[z], l = P.l[z], LT = P.LT[z];
    const int JT = (l + LT - 1) / LT;
    const int groups = JT * (LT / 4);
    const long long total = (long long)M * groups;
    const bool abad = *P.abad[z] != 0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(e / groups), gi = (int)(e % groups);
        const int jt = gi / (LT / 4), jj = (gi % (LT / 4)) * 4;
        const int j0 = jt * LT + jj;
        if (j0 >= l) continue;
        const uint8_t* base = P.out[z] + (long long)row * P.out_ld[z] + (long long)jt * 2 * LT + jj;
        double re[4], im[4];
        oz_crt4(base, P.out_plane[z], P.k, re);
        oz_crt4(base + LT, P.out_plane[z], P.k, im);
        const int eo = oz_e(P.obits[z][row]) - P.kA[z];
        cplx* dst = P.C[z] + (long long)row * P.ldc[z] + j0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = j0 + u;
            if (j >= l || j >= (jt + 1) * LT) break;
            const int sh = eo - P.sx[z][j];
            cplx v = mk(oz_scale(re[u] * P.k.mscale, sh), oz_scale(im[u] * P.k.mscale, sh));
            if (abad || P.xbad[z][j]) v = mk(NAN, NAN);
            dst[u] = v;
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
    const cuuint32_t one[4] = {1, 1, 1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, one,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw_numeric(c, "ozaki: tensor map encoding failed");
}

std::atomic<unsigned long long> g_optin{0};

}  // namespace

int ozaki_moduli() {
    static const int T = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI");
        if (e == nullptr) return 0;
        const int v = std::atoi(e);
        if (v <= 0) return 0;
        return std::min(kOzMaxMod, std::max(8, v));
    }();
    return T;
}

int ozaki_tail() {
    static const int v = [] {
        const char* e = std::getenv("RRSVD_B200_OZAKI_TAIL");
        return e == nullptr ? 2 : std::max(0, std::atoi(e));
    }();
    return v;
}

bool ozaki_usable(int m, int n, int l) {
    return ozaki_moduli() > 0 && m >= 256 && n >= 256 && std::max(m, n) <= 32768 && l >= 1;
}

std::vector<OzakiA> ozaki_prepare_many(rrsvd_b200_ctx* c, const std::vector<OzSrc>& src, int T) {
    const OzConst& k = oz_const(T);
    std::vector<OzakiA> out(src.size());
    for (size_t base = 0; base < src.size(); base += kPrepGroup) {
        const int cnt = (int)std::min<size_t>(kPrepGroup, src.size() - base);
        PrepParams P{};
        P.count = cnt;
        P.k = k;
        P.bad = ws_get<int>(c, cnt);
        check_cuda(c, cudaMemsetAsync(P.bad, 0, sizeof(int) * cnt, c->stream), "ozaki memset");
        long long max_chunks = 0;
        int max_m = 1, max_n = 1;
        for (int i = 0; i < cnt; ++i) {
            const OzSrc& s = src[base + i];
            OzakiA& a = out[base + i];
            a.m = s.m;
            a.n = s.n;
            a.T = T;
            a.pitch = ((long long)s.n + 15) / 16 * 16;
            a.kA = std::min(56, (oz_total_bits(k, std::max(s.m, s.n)) + 1) / 2);
            a.res = ws_get<int8_t>(c, (size_t)T * 2 * s.m * a.pitch);
            a.rowbits = ws_get<unsigned long long>(c, s.m);
            a.colbits = ws_get<unsigned long long>(c, s.n);
            check_cuda(c, cudaMemsetAsync(a.colbits, 0, sizeof(unsigned long long) * s.n, c->stream), "ozaki memset");
            a.bad = P.bad + i;
            P.A[i] = s.A;
            P.lda[i] = s.lda;
            P.pitch[i] = a.pitch;
            P.m[i] = s.m;
            P.n[i] = s.n;
            P.kA[i] = a.kA;
            P.res[i] = a.res;
            P.rowbits[i] = a.rowbits;
            P.colbits[i] = a.colbits;
            max_chunks = std::max(max_chunks, (long long)s.m * a.pitch / 16);
            max_m = std::max(max_m, s.m);
            max_n = std::max(max_n, s.n);
        }
        oz_rowmax_kernel<<<dim3((max_m + 7) / 8, cnt), 256, 0, c->stream>>>(P);
        check_launch(c, "oz_rowmax_kernel");
        const int rch = std::max(1, std::min(64, (4 * kNumSMs * 32) / (cnt * max_n)));  // row chunks: >= ~4 CTAs/SM
        oz_colmax_kernel<<<dim3((max_n + 31) / 32, rch, cnt), 256, 0, c->stream>>>(P);
        check_launch(c, "oz_colmax_kernel");
        const int gx = (int)std::min<long long>((max_chunks + 255) / 256, 8 * kNumSMs);
        oz_resid_a_kernel<<<dim3(gx, cnt), 256, 0, c->stream>>>(P);
        check_launch(c, "oz_resid_a_kernel");
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
        g_optin.fetch_or(bit);
    }
    for (size_t base = 0; base < ps.size(); base += kProdGroup) {
        const int cnt = (int)std::min<size_t>(kProdGroup, ps.size() - base);
        const int T = ps[base].a->T;
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
        long long max_el = 1;
        double flops = 0.0;
        for (int i = 0; i < cnt; ++i) {
            const OzProduct& p = ps[base + i];
            const OzakiA& a = *p.a;
            if (a.T != T) throw_contract(c, "ozaki: mixed moduli counts in one batch");
            const int K = op == kOpN ? a.n : a.m, Mr = op == kOpN ? a.m : a.n;
            const int JT = (p.l + 127) / 128;
            const int LT = ((p.l + JT - 1) / JT + 7) / 8 * 8;
            const long long pitchK = ((long long)K + 15) / 16 * 16;
            const int ncol = 2 * JT * LT;
            const int kX = std::min(56, oz_total_bits(k, K) - a.kA);
            int8_t* bres = ws_get<int8_t>(c, (size_t)T * ncol * 2 * pitchK);
            int* sx = ws_get<int>(c, (size_t)JT * LT);
            int* xbad = ws_get<int>(c, (size_t)JT * LT);
            uint8_t* out = ws_get<uint8_t>(c, (size_t)T * Mr * ncol);
            PP.X[i] = p.X;
            PP.ldx[i] = p.ldx;
            PP.pitchK[i] = pitchK;
            PP.K[i] = K;
            PP.l[i] = p.l;
            PP.LT[i] = LT;
            PP.JT[i] = JT;
            PP.kX[i] = kX;
            PP.kbits[i] = op == kOpN ? a.colbits : a.rowbits;
            PP.bres[i] = bres;
            PP.sx[i] = sx;
            PP.xbad[i] = xbad;
            {  // A planes [T][2][m][pitch]: (n, m, 2, T), box 128 x 128 (op N: (k, row); op C: (col, k))
                const cuuint64_t dims[4] = {(cuuint64_t)a.n, (cuuint64_t)a.m, 2, (cuuint64_t)T};
                const cuuint64_t str[3] = {(cuuint64_t)a.pitch, (cuuint64_t)a.m * a.pitch, 2ull * a.m * a.pitch};
                const cuuint32_t box[4] = {128, 128, 1, 1};
                encode_u8(c, &G.mapA[i], a.res, dims, str, box);
            }
            {  // B' [T][ncol][2][pitchK]: (K, 2, ncol, T), box 128 x 1 x 2LT
                const cuuint64_t dims[4] = {(cuuint64_t)K, 2, (cuuint64_t)ncol, (cuuint64_t)T};
                const cuuint64_t str[3] = {(cuuint64_t)pitchK, 2ull * pitchK, 2ull * pitchK * ncol};
                const cuuint32_t box[4] = {128, 1, (cuuint32_t)(2 * LT), 1};
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
            CP.obits[i] = op == kOpN ? a.rowbits : a.colbits;
            CP.abad[i] = a.bad;
            CP.sx[i] = sx;
            CP.xbad[i] = xbad;
            CP.C[i] = p.C;
            CP.ldc[i] = p.ldc;
            max_cols = std::max(max_cols, JT * LT);
            max_mb = std::max(max_mb, (Mr + kBM - 1) / kBM);
            max_jt = std::max(max_jt, JT);
            max_el = std::max(max_el, (long long)Mr * JT * (LT / 4));
            max_k = std::max(max_k, K);
            flops += 8.0 * Mr * (double)p.l * K;
        }
        cudaEvent_t ea = nullptr, eb = nullptr;
        if (c->gemm_timing) {
            ea = pooled_event(c);
            eb = pooled_event(c);
            check_cuda(c, cudaEventRecord(ea, c->stream), "event record");
        }
        oz_xmax_kernel<<<dim3((max_cols + 7) / 8, cnt), 256, 0, c->stream>>>(PP);
        check_launch(c, "oz_xmax_kernel");
        oz_resid_b_kernel<<<dim3((max_cols + 7) / 8, (max_k + 127) / 128, cnt), 256, 0, c->stream>>>(PP);
        check_launch(c, "oz_resid_b_kernel");
        if (op == kOpN)
            oz_gemm_kernel<kOpN><<<dim3(max_mb, T * max_jt, cnt), 256, kGemmSmem, c->stream>>>(G);
        else
            oz_gemm_kernel<kOpC><<<dim3(max_mb, T * max_jt, cnt), 256, kGemmSmem, c->stream>>>(G);
        check_launch(c, "oz_gemm_kernel");
        const int gx = (int)std::min<long long>((max_el + 255) / 256, 8 * kNumSMs);
        oz_crt_kernel<<<dim3(gx, cnt), 256, 0, c->stream>>>(CP);
        check_launch(c, "oz_crt_kernel");
        if (c->gemm_timing) {
            check_cuda(c, cudaEventRecord(eb, c->stream), "event record");
            c->pending.push_back({ea, eb, flops, flops, c->gemm_tag, 1});
        }
    }
}

}  // namespace rb

// zgemm.cu — see zgemm.cuh for the contract.
#include <atomic>
#include <cstdlib>
#include <algorithm>

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include "zgemm.cuh"

namespace rb {

namespace {

// Tile configurations.  Cfg64: 64x64 CTA tile, 32x32 warp tiles (16 DMMA tiles per warp).
// Cfg56: 64x56 CTA tile, 16x56 warp tiles — for N ≈ l = k+p (110 → 2 x 56 = 112 instead of
// 2 x 64 = 128: 14% less padded DMMA work on every RRSVD-stage GEMM).
template <int BM_, int BN_, int WM_, int WN_, int STAGES_ = 3, int MINB_ = 0, bool M3_ = false>
struct Cfg {
    // M3: the 3M (Karatsuba) complex product — T1 = Ar Br, T2 = Ai Bi, T3 = (Ar + Ai)(Br + Bi),
    // Re = T1 - T2, Im = T3 - T1 - T2: three DMMAs per fragment pair instead of four (a third
    // accumulator set, so fewer CTAs per SM).
    static constexpr bool M3 = M3_;
    static constexpr int BM = BM_, BN = BN_, BK = 16, STAGES = STAGES_;
    static constexpr int WM = WM_, WN = WN_;
    static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
    static constexpr int NTHREADS = 32 * WARPS_M * WARPS_N;
    static constexpr int MI = WM / 8, NI = WN / 8;
    // Padded strides (complex elements) so each quarter-warp's LDS.128 fragment load touches
    // 8 distinct 16-byte bank groups.
    static constexpr int LDA_N = BK + 4;  // A tile stored [m][k]   (op N)   ≡ 4 (mod 8)
    static constexpr int LDA_C = BM + 2;  // A tile stored [k][m]   (op C)   ≡ 2 (mod 8)
    static constexpr int LDB = BN + 2;    // B tile stored [k][n]            ≡ 2 (mod 8)
    static constexpr int A_STAGE = (BM * LDA_N > BK * LDA_C) ? BM * LDA_N : BK * LDA_C;
    static constexpr int B_STAGE = BK * LDB;
    static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * (int)sizeof(cplx);
    static_assert((BM * BK) % NTHREADS == 0, "A tile loads");
    static constexpr int MIN_BLOCKS = MINB_ ? MINB_ : (NTHREADS <= 128 ? 2 : 1);
    // Padded-sub-tile skipping costs registers; the 3-CTA/SM config (168 regs) cannot afford it.
    static constexpr bool SKIP_PAD = MIN_BLOCKS < 3 && !M3;
    // TMA ring: dense (unpadded) stages + two mbarriers per stage; 3 stages (2 at 3 CTAs/SM)
    static constexpr int TMA_STAGES = MIN_BLOCKS >= 3 ? 2 : 3;
    static constexpr int TMA_SMEM_BYTES = TMA_STAGES * (BM * BK + BK * BN) * (int)sizeof(cplx) + 2 * TMA_STAGES * 8;
    static_assert(LDB % 8 == 2 && LDA_N % 8 == 4 && LDA_C % 8 == 2, "bank-conflict-free strides");
};
using Cfg64 = Cfg<64, 64, 32, 32>;
// 2-stage ring, 3 CTAs/SM (12 warps): a 16-deep K stage is ~8k cycles of DMMA work, far more
// than the ~1-2k cycle load latency, so the third stage buys nothing while the third CTA fills
// the DMMA issue bubbles of the other two.
using Cfg56 = Cfg<64, 56, 16, 56, 2, 3>;
// 3M on the 64x56 tile: 84 accumulator doubles per thread -> 2 CTAs/SM (the same per-SM
// accumulator state as the 4M tile at 3 CTAs/SM), 25 % fewer DMMAs: the RRSVD A-products go from
// 29.9 to 33.0 TF/s (4M-equivalent flops), C3 6.2 -> 6.8 steps/s.  A third stage is slower.
using Cfg56m3 = Cfg<64, 56, 16, 56, 2, 2, true>;
// 3M on the 64x64 tile: eight 16x32 warp tiles, one CTA/SM (the same 8 warps/SM as the 4M tile)
using Cfg64m3 = Cfg<64, 64, 16, 32, 2, 1, true>;

__device__ __forceinline__ int find_problem(const GemmGroup& g, int tile) {
    int lo = 0, hi = g.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (g.p[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ---- shared-memory layouts of one K stage ---------------------------------------------------
// Every fragment read is one LDS.128 (re, im of a complex) per lane; a quarter-warp (8 lanes)
// reads 2 rows x 4 k (A) or 4 k x 2 columns (B), and both layouts put those 8 complexes in 8
// distinct 16-byte bank groups.
// PadLayout (cp.async staging): row-major tiles with padded strides.
struct PadLayout {
    template <class CF> __device__ static int a_n(int r, int k) { return r * CF::LDA_N + k; }
    template <class CF> __device__ static int a_c(int k, int m) { return k * CF::LDA_C + m; }
    template <class CF> __device__ static int b(int k, int n) { return k * CF::LDB + n; }
};
// TmaLayout (TMA staging, dense boxes, no swizzle): A (op N) as [k/4][row][4 k] — four 2-D boxes
// of 4 complexes x BM rows; A (op C) and B as [col/2][k][2 cols] — one 3-D box each (2 complexes
// inner, k, column pairs).
struct TmaLayout {
    template <class CF> __device__ static int a_n(int r, int k) { return ((k >> 2) * CF::BM + r) * 4 + (k & 3); }
    template <class CF> __device__ static int a_c(int k, int m) { return ((m >> 1) * CF::BK + k) * 2 + (m & 1); }
    template <class CF> __device__ static int b(int k, int n) { return ((n >> 1) * CF::BK + k) * 2 + (n & 1); }
};

template <class CF>
using Acc = double[CF::MI][CF::NI][CF::M3 ? 3 : 2][2];  // [mi][ni][re/im (4M) | T1/T2/T3 (3M)][c0/c1]

// One k-step of 4 (a DMMA k-slice) of the warp tile: fragment loads and the 3M / 4M products.
template <class CF, int OPA, class L>
__device__ __forceinline__ void mma_kstep(const cplx* __restrict__ sA, const cplx* __restrict__ sB, int kk, int wm,
                                          int wn, int fr, int fc, const double* ks, double kscale, int m0, int n0,
                                          int M, int N, Acc<CF>& acc) {
    constexpr int MI = CF::MI, NI = CF::NI;
    double ar[MI], ai[MI], ain[MI], br[NI], bi[NI];
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        cplx a;
        if (OPA == kOpN) a = sA[L::template a_n<CF>(wm + i * 8 + fr, kk + fc)];
        else a = sA[L::template a_c<CF>(kk + fc, wm + i * 8 + fr)];
        if (OPA == kOpC) a.y = -a.y;
        if (ks != nullptr) { a.x *= kscale; a.y *= kscale; }
        ar[i] = a.x; ai[i] = a.y; ain[i] = CF::M3 ? a.x + a.y : -a.y;  // (3M: ain holds Ar + Ai)
    }
    if constexpr (CF::M3) {
        // all B fragments and their sums first, then every T1/T2 product, then the T3
        // products: the (Ar + Ai), (Br + Bi) additions never stall a DMMA issue
        double bs[NI];
#pragma unroll
        for (int j = 0; j < NI; ++j) {
            const cplx b = sB[L::template b<CF>(kk + fc, wn + j * 8 + fr)];
            br[j] = b.x; bi[j] = b.y;
        }
#pragma unroll
        for (int j = 0; j < NI; ++j) bs[j] = br[j] + bi[j];
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                dmma884(acc[i][j][0][0], acc[i][j][0][1], ar[i], br[j]);
                dmma884(acc[i][j][1][0], acc[i][j][1][1], ai[i], bi[j]);
            }
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int i = 0; i < MI; ++i) dmma884(acc[i][j][2][0], acc[i][j][2][1], ain[i], bs[j]);
    } else {
#pragma unroll
        for (int j = 0; j < NI; ++j) {
            const cplx b = sB[L::template b<CF>(kk + fc, wn + j * 8 + fr)];
            br[j] = b.x; bi[j] = b.y;
        }
        // 8x8 sub-tiles entirely in the M/N padding issue no DMMA (warp-uniform predicate),
        // so ragged shapes (M = 400 on 64-row tiles, N = 110) cost tensor-pipe time only for
        // real rows/columns.
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                if (CF::SKIP_PAD && (m0 + wm + i * 8 >= M || n0 + wn + j * 8 >= N)) continue;
                dmma884(acc[i][j][0][0], acc[i][j][0][1], ar[i], br[j]);
                dmma884(acc[i][j][1][0], acc[i][j][1][1], ar[i], bi[j]);
            }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                if (CF::SKIP_PAD && (m0 + wm + i * 8 >= M || n0 + wn + j * 8 >= N)) continue;
                dmma884(acc[i][j][0][0], acc[i][j][0][1], ain[i], bi[j]);
                dmma884(acc[i][j][1][0], acc[i][j][1][1], ai[i], br[j]);
            }
    }
}

// The CTA's tile of one grouped problem (blockIdx.x -> problem, tile, batch entry, split).
struct TileCoord {
    int pid, m0, n0, bz, sk, kbeg, kend, ktiles;
    bool skip;
};
template <class CF>
__device__ __forceinline__ TileCoord tile_coord(const GemmGroup& g) {
    TileCoord t{};
    t.pid = find_problem(g, blockIdx.x);
    const GemmProblem& P = g.p[t.pid];
    t.skip = P.pred != nullptr && *P.pred != P.pred_want;
    int r = blockIdx.x - P.tile_begin;
    const int tn = r % P.tiles_n; r /= P.tiles_n;
    const int tm = r % P.tiles_m; r /= P.tiles_m;
    t.bz = r % P.batch;           r /= P.batch;
    t.sk = r;  // split index
    t.m0 = tm * CF::BM;
    t.n0 = tn * CF::BN;
    if (P.structure == kUpperC && t.m0 >= t.n0 + CF::BN) t.skip = true;  // tile strictly below the diagonal
    // kTriB: B upper triangular → columns [n0, n0+BN) only see k < n0 + BN
    const int K = (P.structure == kTriB) ? min(P.k, t.n0 + CF::BN) : P.k;
    const int kchunk = (((P.k + P.split - 1) / P.split) + CF::BK - 1) / CF::BK * CF::BK;
    t.kbeg = t.sk * kchunk;
    t.kend = min(K, t.kbeg + kchunk);
    t.ktiles = t.kend > t.kbeg ? (t.kend - t.kbeg + CF::BK - 1) / CF::BK : 0;
    return t;
}

template <class CF>
__device__ __forceinline__ void zero_acc(Acc<CF>& acc) {
#pragma unroll
    for (int i = 0; i < CF::MI; ++i)
#pragma unroll
        for (int j = 0; j < CF::NI; ++j)
#pragma unroll
            for (int r = 0; r < (CF::M3 ? 3 : 2); ++r) acc[i][j][r][0] = acc[i][j][r][1] = 0.0;
}

// Epilogue: 3M fold, then the split-K partial or the scaled / addend / column-blocked store.
template <class CF>
__device__ __forceinline__ void store_tile(const GemmProblem& P, const TileCoord& t, int wm, int wn, int fr, int fc,
                                           Acc<CF>& acc) {
    constexpr int MI = CF::MI, NI = CF::NI;
    const int M = P.m, N = P.n, m0 = t.m0, n0 = t.n0, bz = t.bz;
    if constexpr (CF::M3) {  // Re = T1 - T2, Im = T3 - T1 - T2 into acc[..][0/1]
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const double t1 = acc[i][j][0][c], t2 = acc[i][j][1][c];
                    acc[i][j][0][c] = t1 - t2;
                    acc[i][j][1][c] = acc[i][j][2][c] - t1 - t2;
                }
    }
    if (P.split > 1) {
        cplx* W = P.partial + ((long long)t.sk * P.batch + bz) * (long long)M * N;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            const int row = m0 + wm + i * 8 + fr;
            if (row >= M) continue;
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int col = n0 + wn + j * 8 + fc * 2;
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    if (col + c < N) W[(long long)row * N + col + c] = mk(acc[i][j][0][c], acc[i][j][1][c]);
            }
        }
        return;
    }
    cplx* C = P.C + (long long)bz * P.strideC;
    double csc[NI][2];      // column scales, looked up once per thread (not per element)
    long long ccol[NI][2];  // column addresses (column-blocked C when P.nsub > 0)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int col = n0 + wn + j * 8 + fc * 2 + c;
            csc[j][c] = (P.cs && col < N) ? __ldg(P.cs + col % P.cs_mod) : 1.0;
            ccol[j][c] = P.nsub ? (long long)(col / P.nsub) * P.subC + col % P.nsub : col;
        }
    const cplx* Dd = P.D ? P.D + (long long)bz * P.strideC : nullptr;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        const int row = m0 + wm + i * 8 + fr;
        if (row >= M) continue;
        const double rsc = (P.rs ? __ldg(P.rs + row / P.rs_div) : 1.0) * P.alpha;
#pragma unroll
        for (int j = 0; j < NI; ++j) {
            const int col = n0 + wn + j * 8 + fc * 2;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (col + c >= N) continue;
                const double sc = rsc * csc[j][c];
                cplx v = mk(acc[i][j][0][c] * sc, acc[i][j][1][c] * sc);
                if (Dd) v = cadd(v, Dd[(long long)row * P.ldd + col + c]);
                C[(long long)row * P.ldc + ccol[j][c]] = v;
            }
        }
    }
}

// ---- kernel 1: cp.async (LDGSTS) ring, the general path --------------------------------------
template <class CF, int OPA, bool KS>  // KS: some problem of the group has a k-scale (P.ks)
__global__ void __launch_bounds__(CF::NTHREADS, CF::MIN_BLOCKS)
zgemm_dmma_kernel(const __grid_constant__ GemmGroup g) {
    constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, STAGES = CF::STAGES;
    constexpr int WM = CF::WM, WN = CF::WN, WARPS_N = CF::WARPS_N, NTHREADS = CF::NTHREADS;
    constexpr int LDA_N = CF::LDA_N, LDA_C = CF::LDA_C, LDB = CF::LDB;
    constexpr int A_STAGE = CF::A_STAGE, B_STAGE = CF::B_STAGE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* smA = reinterpret_cast<cplx*>(smem_raw);
    cplx* smB = smA + STAGES * A_STAGE;

    const TileCoord tc = tile_coord<CF>(g);
    if (tc.skip) return;
    const GemmProblem& P = g.p[tc.pid];
    const int M = P.m, N = P.n, m0 = tc.m0, n0 = tc.n0;
    const int kbeg = tc.kbeg, kend = tc.kend, ktiles = tc.ktiles;

    const cplx* __restrict__ A = P.A + (long long)tc.bz * P.strideA;
    const cplx* __restrict__ B = P.B + (long long)tc.bz * P.strideB;
    const long long lda = P.lda, ldb = P.ldb;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp / WARPS_N) * WM, wn = (warp % WARPS_N) * WN;

    // The B columns this thread copies are the same in every stage: resolve their (block,
    // offset) address once (column-blocked B, P.nsub > 0).
    constexpr int NBL = (BK * BN + NTHREADS - 1) / NTHREADS;
    int bcol[NBL];  // element offsets < 2^31 (checked by the launcher)
#pragma unroll
    for (int i = 0; i < NBL; ++i) {
        const int gn = n0 + (i * NTHREADS + tid) % BN;
        bcol[i] = P.nsub ? (gn / P.nsub) * (int)P.subB + gn % P.nsub : gn;
    }

    auto load_stage = [&](int stage, int kt) {
        const int k0 = kbeg + kt * BK;
        cplx* sA = smA + stage * A_STAGE;
        cplx* sB = smB + stage * B_STAGE;
        if (OPA == kOpN) {
#pragma unroll
            for (int i = 0; i < (BM * BK) / NTHREADS; ++i) {
                const int idx = i * NTHREADS + tid;
                const int r = idx / BK, c = idx % BK;
                const int gr = m0 + r, gc = k0 + c;
                const bool ok = gr < M && gc < kend;
                cp_async16(sA + r * LDA_N + c, ok ? A + (long long)gr * lda + gc : A, ok);
            }
        } else {
#pragma unroll
            for (int i = 0; i < (BM * BK) / NTHREADS; ++i) {
                const int idx = i * NTHREADS + tid;
                const int r = idx / BM, c = idx % BM;  // r: k, c: m
                const int gk = k0 + r, gm = m0 + c;
                const bool ok = gk < kend && gm < M;
                cp_async16(sA + r * LDA_C + c, ok ? A + (long long)gk * lda + gm : A, ok);
            }
        }
#pragma unroll
        for (int i = 0; i < (BK * BN + NTHREADS - 1) / NTHREADS; ++i) {
            const int idx = i * NTHREADS + tid;
            if ((BK * BN) % NTHREADS != 0 && idx >= BK * BN) break;
            const int r = idx / BN, c = idx % BN;
            const int gk = k0 + r, gn = n0 + c;
            const bool ok = gk < kend && gn < N;
            cp_async16(sB + r * LDB + c, ok ? B + (long long)gk * ldb + bcol[i] : B, ok);
        }
    };

    Acc<CF> acc;
    zero_acc<CF>(acc);

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_async_commit();
    }

    const int fr = lane >> 2, fc = lane & 3;
    const double* ks = KS ? P.ks : nullptr;  // (without KS no multiply by 1.0 is compiled in)

    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage(nk % STAGES, nk);
            cp_async_commit();
        }
        const int stage = kt % STAGES;
        const cplx* sA = smA + stage * A_STAGE;
        const cplx* sB = smB + stage * B_STAGE;
        const int kbase = kbeg + kt * BK;
#pragma unroll(CF::MIN_BLOCKS >= 3 ? 1 : 4)
        for (int kk = 0; kk < BK; kk += 4) {
            if (kbase + kk >= kend) break;  // K tail: no DMMA on zero padding (uniform)
            double kscale = 1.0;
            if (ks != nullptr) {
                const int gk = kbase + kk + fc;
                kscale = gk < kend ? __ldg(ks + gk) : 0.0;
            }
            mma_kstep<CF, OPA, PadLayout>(sA, sB, kk, wm, wn, fr, fc, ks, kscale, m0, n0, M, N, acc);
        }
    }
    cp_async_wait<0>();
    store_tile<CF>(P, tc, wm, wn, fr, fc, acc);
}

// ---- kernel 2: TMA + mbarrier ring -----------------------------------------------------------
// The same warp tiles and DMMA k-steps; operands arrive by cp.async.bulk.tensor (one thread
// issues every box of a stage, completion counted in bytes on the stage's "full" mbarrier), and
// the warps release a stage on its "empty" mbarrier (one arrival per warp) — no __syncthreads
// in the main loop, no per-thread address arithmetic or LDGSTS issue.  TMA zero-fills every
// element outside the tensor (M, N, K tails).  Refills run two k-tiles ahead (3 stages) or one
// (2 stages, the 3-CTA/SM tile).
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
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
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

template <class CF, int OPA, bool KS>
__global__ void __launch_bounds__(CF::NTHREADS, CF::MIN_BLOCKS)
zgemm_tma_kernel(const __grid_constant__ TmaGroup tg) {
    constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, ST = CF::TMA_STAGES;
    constexpr int WM = CF::WM, WN = CF::WN, WARPS_N = CF::WARPS_N, NWARPS = CF::NTHREADS / 32;
    constexpr int A_ELEMS = BM * BK, B_ELEMS = BK * BN;
    constexpr unsigned STAGE_BYTES = (A_ELEMS + B_ELEMS) * (unsigned)sizeof(cplx);
    const GemmGroup& g = tg.g;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cplx* smA = reinterpret_cast<cplx*>(smem_raw);
    cplx* smB = smA + ST * A_ELEMS;
    uint64_t* full = reinterpret_cast<uint64_t*>(smB + ST * B_ELEMS);
    uint64_t* empty = full + ST;

    const TileCoord tc = tile_coord<CF>(g);
    if (tc.skip) return;
    const GemmProblem& P = g.p[tc.pid];
    const CUtensorMap* mapA = &tg.mapA[tc.pid];
    const CUtensorMap* mapB = &tg.mapB[tc.pid];
    const int M = P.m, N = P.n, m0 = tc.m0, n0 = tc.n0;
    const int kbeg = tc.kbeg, kend = tc.kend, ktiles = tc.ktiles;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp / WARPS_N) * WM, wn = (warp % WARPS_N) * WN;

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int stage, int kt) {  // (thread 0 only)
        const int k0 = kbeg + kt * BK;
        cplx* sA = smA + stage * A_ELEMS;
        cplx* sB = smB + stage * B_ELEMS;
        mbar_expect_tx(&full[stage], STAGE_BYTES);
        if (OPA == kOpN) {  // four boxes of [BM rows][4 complexes]: dims (2K doubles, M, batch)
#pragma unroll
            for (int kg = 0; kg < BK / 4; ++kg)
                tma_load_3d(sA + kg * BM * 4, mapA, &full[stage], 2 * (k0 + 4 * kg), m0, tc.bz);
        } else {  // one box [BM/2 pairs][BK][2 complexes]: dims (4 doubles, K, M/2, batch)
            tma_load_4d(sA, mapA, &full[stage], 0, k0, m0 / 2, tc.bz);
        }
        tma_load_4d(sB, mapB, &full[stage], 0, k0, n0 / 2, tc.bz);  // [BN/2][BK][2]: (4, K, N/2, batch)
    };

    if (tid == 0)
        for (int s = 0; s < ST && s < ktiles; ++s) issue(s, s);

    Acc<CF> acc;
    zero_acc<CF>(acc);
    const int fr = lane >> 2, fc = lane & 3;
    const double* ks = KS ? P.ks : nullptr;

    for (int kt = 0; kt < ktiles; ++kt) {
        const int stage = kt % ST;
        mbar_wait(&full[stage], (kt / ST) & 1);
        // refill the stage released one iteration ago (its last reader was this warp's previous
        // k-tile; the other warps are at most a tile behind)
        if (tid == 0 && kt >= 1 && kt - 1 + ST < ktiles) {
            const int ps = (kt - 1) % ST;
            mbar_wait(&empty[ps], ((kt - 1) / ST) & 1);
            issue(ps, kt - 1 + ST);
        }
        const cplx* sA = smA + stage * A_ELEMS;
        const cplx* sB = smB + stage * B_ELEMS;
        const int kbase = kbeg + kt * BK;
#pragma unroll(CF::MIN_BLOCKS >= 3 ? 1 : 4)
        for (int kk = 0; kk < BK; kk += 4) {
            if (kbase + kk >= kend) break;  // K tail (uniform)
            double kscale = 1.0;
            if (ks != nullptr) {
                const int gk = kbase + kk + fc;
                kscale = gk < kend ? __ldg(ks + gk) : 0.0;
            }
            mma_kstep<CF, OPA, TmaLayout>(sA, sB, kk, wm, wn, fr, fc, ks, kscale, m0, n0, M, N, acc);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
    }
    store_tile<CF>(P, tc, wm, wn, fr, fc, acc);
}

// Fixed-order reduction of split-K partials + fused output scaling.
__global__ void splitk_reduce_kernel(const __grid_constant__ GemmGroup g) {
    const int pid = blockIdx.y;
    const GemmProblem& P = g.p[pid];
    if (P.split <= 1) return;
    if (P.pred != nullptr && *P.pred != P.pred_want) return;
    const long long per = (long long)P.m * P.n;
    const long long total = per * P.batch;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long bz = e / per, rem = e % per;
        const int row = (int)(rem / P.n), col = (int)(rem % P.n);
        cplx s = mk(0.0, 0.0);
        for (int k = 0; k < P.split; ++k) s = cadd(s, P.partial[(long long)k * total + e]);
        double sc = P.alpha;
        if (P.rs) sc *= P.rs[row / P.rs_div];
        if (P.cs) sc *= P.cs[col % P.cs_mod];
        const long long cc = P.nsub ? (long long)(col / P.nsub) * P.subC + col % P.nsub : col;
        cplx v = cscale(s, sc);
        if (P.D) v = cadd(v, P.D[bz * P.strideC + (long long)row * P.ldd + col]);
        P.C[bz * P.strideC + (long long)row * P.ldc + cc] = v;
    }
}

// ---- host: tensor maps ----------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

bool encode(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
            const cuuint32_t* box) {
    const auto enc = tensor_map_encoder();
    if (enc == nullptr) return false;
    const cuuint32_t one[5] = {1, 1, 1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, one,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor maps of every problem for the TmaLayout boxes; false if some problem cannot be
// described (the group then takes the cp.async kernel).
template <class CF>
bool make_tma_group(const GemmGroup& g, GemmOp opA, TmaGroup& tg) {
    for (int i = 0; i < g.count; ++i) {
        const GemmProblem& P = g.p[i];
        if (P.m <= 0 || P.n <= 0) continue;
        if (P.nsub != 0 || (P.n & 1) || (opA == kOpC && (P.m & 1))) return false;
        if ((reinterpret_cast<uintptr_t>(P.A) | reinterpret_cast<uintptr_t>(P.B)) & 15) return false;
        const cuuint64_t sA = (cuuint64_t)(P.batch > 1 ? P.strideA : 1) * 16, sB = (cuuint64_t)(P.batch > 1 ? P.strideB : 1) * 16;
        if (opA == kOpN) {  // A m x k: (2k doubles, m rows, batch), box (8, BM, 1)
            const cuuint64_t dims[3] = {2ull * P.k, (cuuint64_t)P.m, (cuuint64_t)P.batch};
            const cuuint64_t str[2] = {(cuuint64_t)P.lda * 16, sA};
            const cuuint32_t box[3] = {8, (cuuint32_t)CF::BM, 1};
            if (!encode(&tg.mapA[i], P.A, 3, dims, str, box)) return false;
        } else {  // A k x m, read as A^H: (4 doubles, k rows, m/2 column pairs, batch), box (4, BK, BM/2, 1)
            const cuuint64_t dims[4] = {4, (cuuint64_t)P.k, (cuuint64_t)P.m / 2, (cuuint64_t)P.batch};
            const cuuint64_t str[3] = {(cuuint64_t)P.lda * 16, 32, sA};
            const cuuint32_t box[4] = {4, (cuuint32_t)CF::BK, (cuuint32_t)CF::BM / 2, 1};
            if (!encode(&tg.mapA[i], P.A, 4, dims, str, box)) return false;
        }
        const cuuint64_t dims[4] = {4, (cuuint64_t)P.k, (cuuint64_t)P.n / 2, (cuuint64_t)P.batch};
        const cuuint64_t str[3] = {(cuuint64_t)P.ldb * 16, 32, sB};
        const cuuint32_t box[4] = {4, (cuuint32_t)CF::BK, (cuuint32_t)CF::BN / 2, 1};
        if (!encode(&tg.mapB[i], P.B, 4, dims, str, box)) return false;
    }
    tg.g = g;
    return true;
}

bool tma_enabled() {  // RRSVD_B200_GEMM_TMA=0: every group on the cp.async kernel (A/B timing)
    static const bool on = [] {
        const char* e = std::getenv("RRSVD_B200_GEMM_TMA");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}

// per-device one-time opt-in to the kernels' dynamic shared memory
template <class K>
void smem_optin(K kernel, int bytes, std::atomic<unsigned long long>& done, unsigned long long bit) {
    if (!(done.load() & bit)) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <class CF>
cudaError_t launch_cfg(GemmGroup& g, GemmOp opA, cudaStream_t s) {
    int total = 0;
    bool any_split = false;
    for (int i = 0; i < g.count; ++i) {
        GemmProblem& P = g.p[i];
        P.tiles_m = (P.m + CF::BM - 1) / CF::BM;
        P.tiles_n = (P.n + CF::BN - 1) / CF::BN;
        P.tile_begin = total;
        if (P.m > 0 && P.n > 0) total += P.tiles_m * P.tiles_n * P.batch * P.split;
        any_split |= P.split > 1;
    }
    g.total_tiles = total;
    if (total == 0) return cudaSuccess;
    bool any_ks = false;
    for (int i = 0; i < g.count; ++i) any_ks |= g.p[i].ks != nullptr;
    // the smem opt-in is per device: one bit per ordinal (a process may drive several GPUs)
    static std::atomic<unsigned long long> configured{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(configured.load() & bit)) {
        smem_optin(zgemm_dmma_kernel<CF, kOpN, false>, CF::SMEM_BYTES, configured, bit);
        smem_optin(zgemm_dmma_kernel<CF, kOpC, false>, CF::SMEM_BYTES, configured, bit);
        smem_optin(zgemm_dmma_kernel<CF, kOpN, true>, CF::SMEM_BYTES, configured, bit);
        smem_optin(zgemm_dmma_kernel<CF, kOpC, true>, CF::SMEM_BYTES, configured, bit);
        smem_optin(zgemm_tma_kernel<CF, kOpN, false>, CF::TMA_SMEM_BYTES, configured, bit);
        smem_optin(zgemm_tma_kernel<CF, kOpC, false>, CF::TMA_SMEM_BYTES, configured, bit);
        smem_optin(zgemm_tma_kernel<CF, kOpN, true>, CF::TMA_SMEM_BYTES, configured, bit);
        smem_optin(zgemm_tma_kernel<CF, kOpC, true>, CF::TMA_SMEM_BYTES, configured, bit);
        configured.fetch_or(bit);
    }
    static thread_local TmaGroup tg;  // 24 KB: kept off the stack
    g.used_m3 = CF::M3 ? 1 : 0;
    g.used_tma = tma_enabled() && make_tma_group<CF>(g, opA, tg) ? 1 : 0;
    if (g.used_tma) {
        const int sm = CF::TMA_SMEM_BYTES;
        if (opA == kOpN) {
            if (any_ks) zgemm_tma_kernel<CF, kOpN, true><<<total, CF::NTHREADS, sm, s>>>(tg);
            else zgemm_tma_kernel<CF, kOpN, false><<<total, CF::NTHREADS, sm, s>>>(tg);
        } else {
            if (any_ks) zgemm_tma_kernel<CF, kOpC, true><<<total, CF::NTHREADS, sm, s>>>(tg);
            else zgemm_tma_kernel<CF, kOpC, false><<<total, CF::NTHREADS, sm, s>>>(tg);
        }
    } else if (opA == kOpN) {
        if (any_ks) zgemm_dmma_kernel<CF, kOpN, true><<<total, CF::NTHREADS, CF::SMEM_BYTES, s>>>(g);
        else zgemm_dmma_kernel<CF, kOpN, false><<<total, CF::NTHREADS, CF::SMEM_BYTES, s>>>(g);
    } else {
        if (any_ks) zgemm_dmma_kernel<CF, kOpC, true><<<total, CF::NTHREADS, CF::SMEM_BYTES, s>>>(g);
        else zgemm_dmma_kernel<CF, kOpC, false><<<total, CF::NTHREADS, CF::SMEM_BYTES, s>>>(g);
    }
    if (any_split) {  // one thread per output element, at most 2 waves of CTAs per problem
        long long maxe = 1;
        for (int i = 0; i < g.count; ++i)
            if (g.p[i].split > 1) maxe = std::max(maxe, (long long)g.p[i].m * g.p[i].n * g.p[i].batch);
        const int gx = (int)std::min<long long>(2 * kNumSMs, (maxe + 255) / 256);
        splitk_reduce_kernel<<<dim3(gx, g.count), 256, 0, s>>>(g);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t zgemm_grouped(GemmGroup& g, GemmOp opA, cudaStream_t s) {
    // Pick the CTA tile that wastes the least padded DMMA work (M and N quantisation) for this
    // group.
    double pad64 = 0.0, pad56 = 0.0;
    for (int i = 0; i < g.count; ++i) {
        GemmProblem& P = g.p[i];
        if (P.batch < 1) P.batch = 1;
        if (P.split < 1) P.split = 1;
        if (P.rs_div < 1) P.rs_div = 1;
        if (P.cs_mod < 1) P.cs_mod = 1;
        if (P.nsub > 0 && ((long long)(P.n / P.nsub + 1) * (P.subB > P.subC ? P.subB : P.subC) > 2147483647ll))
            return cudaErrorInvalidValue;  // column-blocked offsets must fit in 32 bits
        const double w = (double)P.k * P.batch;
        pad64 += w * ((P.m + 63) / 64 * 64) * ((P.n + 63) / 64 * 64);
        pad56 += w * ((P.m + 63) / 64 * 64) * ((P.n + 55) / 56 * 56);
    }
    static const int force = [] {  // RRSVD_B200_GEMM_CFG=56|64 pins the tile (experiments)
        const char* e = std::getenv("RRSVD_B200_GEMM_CFG");
        return e ? std::atoi(e) : 0;
    }();
    static const bool m3 = [] {  // the 3M complex product on the 64x56 tile (RRSVD_B200_GEMM_3M=0: 4M)
        const char* e = std::getenv("RRSVD_B200_GEMM_3M");
        return e == nullptr || std::atoi(e) != 0;
    }();
    if (force == 56) return m3 ? launch_cfg<Cfg56m3>(g, opA, s) : launch_cfg<Cfg56>(g, opA, s);
    if (force == 64) return m3 ? launch_cfg<Cfg64m3>(g, opA, s) : launch_cfg<Cfg64>(g, opA, s);
    // Ties go to Cfg56 (3 CTAs/SM hide short-K pipelines better: the K = 100 Θ GEMM runs
    // 27.0 vs 25.0 TF/s); Cfg64 only when it saves >= 5 % padded work (e.g. N = 128, 256).
    static const bool m3_64 = [] {  // RRSVD_B200_GEMM_3M64=1: 3M on the 64x64 tile too (experiment)
        const char* e = std::getenv("RRSVD_B200_GEMM_3M64");
        return e != nullptr && std::atoi(e) != 0;
    }();
    if (pad64 < 0.95 * pad56) return m3 && m3_64 ? launch_cfg<Cfg64m3>(g, opA, s) : launch_cfg<Cfg64>(g, opA, s);
    return m3 ? launch_cfg<Cfg56m3>(g, opA, s) : launch_cfg<Cfg56>(g, opA, s);
}

}  // namespace rb

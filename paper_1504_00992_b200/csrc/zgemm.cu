// zgemm.cu — see zgemm.cuh for the contract.
#include <atomic>
#include <cstdlib>
#include <algorithm>

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

template <class CF, int OPA, bool KS>  // KS: some problem of the group has a k-scale (P.ks)
__global__ void __launch_bounds__(CF::NTHREADS, CF::MIN_BLOCKS)
zgemm_dmma_kernel(const __grid_constant__ GemmGroup g) {
    constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, STAGES = CF::STAGES;
    constexpr int WM = CF::WM, WN = CF::WN, WARPS_N = CF::WARPS_N, NTHREADS = CF::NTHREADS;
    constexpr int MI = CF::MI, NI = CF::NI;
    constexpr int LDA_N = CF::LDA_N, LDA_C = CF::LDA_C, LDB = CF::LDB;
    constexpr int A_STAGE = CF::A_STAGE, B_STAGE = CF::B_STAGE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* smA = reinterpret_cast<cplx*>(smem_raw);
    cplx* smB = smA + STAGES * A_STAGE;

    const int pid = find_problem(g, blockIdx.x);
    const GemmProblem& P = g.p[pid];
    if (P.pred != nullptr && *P.pred != P.pred_want) return;
    int t = blockIdx.x - P.tile_begin;
    const int tn = t % P.tiles_n; t /= P.tiles_n;
    const int tm = t % P.tiles_m; t /= P.tiles_m;
    const int bz = t % P.batch;   t /= P.batch;
    const int sk = t;  // split index

    const int M = P.m, N = P.n;
    const int m0 = tm * BM, n0 = tn * BN;
    if (P.structure == kUpperC && m0 >= n0 + BN) return;  // tile strictly below the diagonal
    // kTriB: B upper triangular → columns [n0, n0+BN) only see k < n0 + BN
    const int K = (P.structure == kTriB) ? min(P.k, n0 + BN) : P.k;
    const int kchunk = (((P.k + P.split - 1) / P.split) + BK - 1) / BK * BK;
    const int kbeg = sk * kchunk;
    const int kend = min(K, kbeg + kchunk);

    const cplx* __restrict__ A = P.A + (long long)bz * P.strideA;
    const cplx* __restrict__ B = P.B + (long long)bz * P.strideB;
    const long long lda = P.lda, ldb = P.ldb;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp / WARPS_N) * WM, wn = (warp % WARPS_N) * WN;

    const int ktiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

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

    constexpr int NACC = CF::M3 ? 3 : 2;
    double acc[MI][NI][NACC][2];  // [mi][ni][re/im (4M) | T1/T2/T3 (3M)][c0/c1]
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int r = 0; r < NACC; ++r) acc[i][j][r][0] = acc[i][j][r][1] = 0.0;

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
            double ar[MI], ai[MI], ain[MI], br[NI], bi[NI];
            double kscale = 1.0;
            if (ks != nullptr) {
                const int gk = kbase + kk + fc;
                kscale = gk < kend ? __ldg(ks + gk) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                cplx a;
                if (OPA == kOpN) a = sA[(wm + i * 8 + fr) * LDA_N + kk + fc];
                else a = sA[(kk + fc) * LDA_C + wm + i * 8 + fr];
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
                    const cplx b = sB[(kk + fc) * LDB + wn + j * 8 + fr];
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
                continue;
            }
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const cplx b = sB[(kk + fc) * LDB + wn + j * 8 + fr];
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
    cp_async_wait<0>();

    // ---- epilogue (3M: fold T1, T2, T3 into Re = T1 - T2, Im = T3 - T1 - T2 in acc[..][0/1])
    if constexpr (CF::M3) {
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
        cplx* W = P.partial + ((long long)sk * P.batch + bz) * (long long)M * N;
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
    double csc[NI][2];     // column scales, looked up once per thread (not per element)
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

}  // namespace

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
        cudaFuncSetAttribute(zgemm_dmma_kernel<CF, kOpN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES);
        cudaFuncSetAttribute(zgemm_dmma_kernel<CF, kOpC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES);
        cudaFuncSetAttribute(zgemm_dmma_kernel<CF, kOpN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES);
        cudaFuncSetAttribute(zgemm_dmma_kernel<CF, kOpC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES);
        configured.fetch_or(bit);
    }
    if (opA == kOpN) {
        if (any_ks) zgemm_dmma_kernel<CF, kOpN, true><<<total, CF::NTHREADS, CF::SMEM_BYTES, s>>>(g);
        else zgemm_dmma_kernel<CF, kOpN, false><<<total, CF::NTHREADS, CF::SMEM_BYTES, s>>>(g);
    } else {
        if (any_ks) zgemm_dmma_kernel<CF, kOpC, true><<<total, CF::NTHREADS, CF::SMEM_BYTES, s>>>(g);
        else zgemm_dmma_kernel<CF, kOpC, false><<<total, CF::NTHREADS, CF::SMEM_BYTES, s>>>(g);
    }
    if (any_split) splitk_reduce_kernel<<<dim3(2 * kNumSMs, g.count), 256, 0, s>>>(g);
    return cudaGetLastError();
}

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

// zgemm.cuh — grouped complex-FP64 GEMM on the FP64 tensor cores (DMMA) for sm_100a.
//
// Replaces every cblas_zgemm call on the TEBD decimation path (linalg.cpp:20-40,
// tebd.cpp:134-137) and the scalar Θ contraction loop (tebd.cpp:105-114).
//
// Why DMMA and not tcgen05: sm_100a has no f64 kind for tcgen05.mma (ptxas rejects
// `.kind::f64`), so FP64 tensor math is warp-level `mma.sync.m8n8k4.f64` → SASS DMMA.8x8x4.
// Complex arithmetic on split (re, im) fragments, two forms:
//  * 4M (the 64x64 tile): C_r += A_r B_r − A_i B_i, C_i += A_r B_i + A_i B_r — four real MMAs per
//    k-step, zgemm's rounding class;
//  * 3M (the 64x56 tile, default; RRSVD_B200_GEMM_3M=0 selects 4M): T1 = A_r B_r, T2 = A_i B_i,
//    T3 = (A_r + A_i)(B_r + B_i) accumulated separately, C_r = T1 − T2, C_i = T3 − T1 − T2 in the
//    epilogue — three MMAs (25 % fewer).  3M is normwise stable (Higham, "Stability of a method
//    for multiplying complex matrices with three real matrix multiplications", 1992): the
//    imaginary part's error bound is a small constant times 4M's u·Σ|a||b|, far inside the
//    path's 1e-10 parity bar (every parity test passes either way; BLAS libraries ship it as
//    zgemm3m).
// Operands are staged global→shared by TMA (cp.async.bulk.tensor into an mbarrier ring, one
// issuing thread, zero-filled tails) — or, for the shapes TMA cannot describe (column-blocked B,
// odd pair dimensions, unaligned pointers), by a cp.async (LDGSTS) ring; each thread reads one
// 16-byte complex per fragment element (LDS.128), so a single shared-memory read yields both
// the real and imaginary fragment.
#pragma once
#include <cuda.h>  // CUtensorMap (types only: the encoder is fetched from the driver at run time)

#include "common.cuh"

namespace rb {

enum GemmOp : int { kOpN = 0, kOpC = 1 };
enum GemmStructure : int { kGeneral = 0, kTriB = 1, kUpperC = 2 };

// One (possibly strided-batched) product  C[b] = diag(rs) · op(A[b]) · diag(ks) · B[b] · diag(cs)
// with all three scalings optional; row scale index = row / rs_div, column scale index
// = col % cs_mod (so λ_l over unfolded rows (α·d1+i) and λ_r over columns (j·χr+β) fuse).
struct GemmProblem {
    int m, n, k;
    int batch;
    const cplx* A;
    long long lda, strideA;  // op N: A is m x k row-major; op C: A is k x m row-major (use A^H)
    const cplx* B;
    long long ldb, strideB;  // B is k x n row-major
    cplx* C;
    long long ldc, strideC;
    const double* rs;  // nullable
    const double* ks;  // nullable
    const double* cs;  // nullable
    int rs_div, cs_mod;
    int split;         // split-K factor (1 = none)
    cplx* partial;     // split-K workspace: split * batch * m * n (only if split > 1)
    // Structure hints: kTriB — B is upper triangular (k > col terms vanish: a column tile
    // stops its K loop at its last column); kUpperC — only the upper-triangular part of C is
    // needed (tiles entirely below the diagonal are skipped and left unwritten).
    int structure;
    // Column-blocked B/C (nsub > 0): logical column c lives in block c / nsub at offset c % nsub;
    // B(k, c) = B[(c/nsub)·subB + k·ldb + c%nsub], C likewise with subC.  Lets a strided batch of
    // narrow products that share A (the gate: G · Θ[α] for every α) run as ONE wide GEMM.
    int nsub;
    long long subB, subC;
    // Optional addend: C = D + alpha * (scaled product), D with its own ld (may alias C: each
    // element is read and written by the same thread).  Not combined with nsub.
    const cplx* D;
    long long ldd;
    double alpha;
    // Optional device predicate: the problem runs only if *pred == pred_want (otherwise its CTAs
    // exit at once and C is left untouched) — data-dependent schedules without a host sync.
    const int* pred;
    int pred_want;
    // filled by the launcher
    int tiles_m, tiles_n, tile_begin;
};

constexpr int kMaxGroup = 48;

struct GemmGroup {
    int count;
    int total_tiles;
    GemmProblem p[kMaxGroup];
    // filled by zgemm_grouped (host statistics): the complex-product form and the staging used
    int used_m3;
    int used_tma;
};

// The TMA-staged launch: one tensor map per operand per problem (FLOAT64 elements, dense boxes),
// passed with the group as one __grid_constant__ parameter (64-byte aligned maps).
struct alignas(64) TmaGroup {
    CUtensorMap mapA[kMaxGroup];
    CUtensorMap mapB[kMaxGroup];
    GemmGroup g;
};
static_assert(sizeof(TmaGroup) <= 32764, "kernel parameter space");

// Launches one grouped GEMM.  All problems share the A operation.  Split-K partials are
// reduced (deterministically, fixed order) by a second kernel.
cudaError_t zgemm_grouped(GemmGroup& g, GemmOp opA, cudaStream_t s);

}  // namespace rb

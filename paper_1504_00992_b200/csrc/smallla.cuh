// smallla.cuh — small dense linear algebra kernels of the RRSVD pipeline (batched).
#pragma once
#include "common.cuh"

namespace rb {

constexpr int kMaxSmall = 64;  // problems per launch of the small-matrix kernels

// ---- Cholesky + triangular inverse (the "R^-1" of one CholeskyQR pass) -------------------
// G (l x l, Hermitian, row-major) -> T = R^-1 (l x l upper, zeros below), G (+ s I) = R^H R.
// Columns whose Cholesky pivot falls to <= dep_tol * (original diagonal) (or to <= 0) are
// numerically dependent: their T column is zeroed, so the orthonormalised basis gets a zero
// column (the reference's Householder QR returns an arbitrary orthonormal completion there,
// linalg.hpp:35-37; either way no NaN and an unchanged span).  The orthonormalisation
// schedule (pipeline.cu orth_many) keeps the Gram matrices of its plain passes well
// conditioned, so it runs with dep_tol = 0: only non-positive pivots (exactly vanishing
// columns) die, and no genuine small-σ direction is discarded.
constexpr int kMaxCholL = 112;  // the unpacked L x (L + 2) Gram (+ an 8-row scratch) fits 227 KB of shared memory

struct CholBatch {
    int count;
    int l[kMaxSmall];
    const cplx* G[kMaxSmall];
    int ldg[kMaxSmall];               // 0: l
    const cplx* Gsub[kMaxSmall];      // nullable: factor G - Gsub instead (Gsub l x l, ld l)
    const cplx* trace_src[kMaxSmall]; // nullable: the shift's trace is taken over this matrix's
    int trace_n[kMaxSmall];           //   first trace_n diagonal entries (ld trace_ld) instead of G
    int trace_ld[kMaxSmall];
    cplx* T[kMaxSmall];
    int ldt[kMaxSmall];               // 0: l
    cplx* Tneg[kMaxSmall];            // nullable: also write -T (ld ldt)
    double shift_scale[kMaxSmall];    // 0: no shift; else s = shift_scale * u * trace
    double dep_tol[kMaxSmall];        // relative pivot floor for "dependent"
    int* ndead[kMaxSmall];            // nullable: number of dependent columns found
    int ndead_acc[kMaxSmall];         // 1: add to *ndead instead of storing
    double* shift_save[kMaxSmall];    // nullable: store the shift used (for later blocks)
    const double* shift_use[kMaxSmall];  // nullable: use this stored shift instead
    int* ill_out[kMaxSmall];          // nullable: set to 1 if some pivot is < kIllRatio x the shift
                                      //   (or dependent): cond(Y) beyond one shifted pass; the
                                      //   caller zeroes it (diagonal blocks of one matrix OR in)
    const int* pred[kMaxSmall];       // nullable: run only if *pred != 0 (else exit at once)
};
constexpr double kIllRatio = 1e4;

// Q[i] = (*flag[i] != 0) ? B[i] : A[i] (n[i] elements each) — the data-dependent end of the
// adaptive orthonormalisation schedule (pipeline.cu orth_many).
struct SelectBatch {
    int count;
    const int* flag[kMaxSmall];
    const cplx* A[kMaxSmall];
    const cplx* B[kMaxSmall];
    cplx* Q[kMaxSmall];
    long long n[kMaxSmall];
};
cudaError_t select_many(const SelectBatch& b, cudaStream_t s);
cudaError_t chol_inv(const CholBatch& b, int max_l, cudaStream_t s);
bool jacobi_fits(int r, int c);  // an r x c problem fits jacobi_svd's on-chip capacity

// ---- static column pivoting for the QR-preconditioned Jacobi: order the columns of each
// row-major r x c matrix X by decreasing norm (ties by index), Xp[:, k] = X[:, perm[k]]; after
// the SVD of Xp the right vectors' rows go back: V[perm[k], :] = Vp[k, :].
struct ColPermBatch {
    int count;
    const cplx* X[kMaxSmall];
    cplx* Xp[kMaxSmall];
    int r[kMaxSmall], c[kMaxSmall];
    int* perm[kMaxSmall];
    const cplx* Vp[kMaxSmall];  // for the row scatter
    cplx* V[kMaxSmall];
};
cudaError_t colperm_sort_gather(const ColPermBatch& b, int max_c, cudaStream_t s);
cudaError_t colperm_scatter_rows(const ColPermBatch& b, cudaStream_t s);

// ---- max_j ||D[:, j]|| of row-major m x r matrices (the accuracy check's probe residuals,
// randomized.cpp:47-53,149-150); one CTA per matrix, fixed reduction order.
struct ColNormBatch {
    int count;
    const cplx* D[kMaxSmall];
    int m[kMaxSmall], r[kMaxSmall];
    double* out[kMaxSmall];
};
cudaError_t colnorm_max_many(const ColNormBatch& b, cudaStream_t s);

// ---- One-sided (Hestenes) Jacobi SVD ------------------------------------------------------
// Works on W (column-major, ld = r + c): rows [0, r) hold X (r x c), rows [r, r + c) hold the
// accumulated rotations J (initialised to I).  On exit X·J_total has orthogonal columns.
// One thread-block cluster per problem: 2*cs column blocks, cs CTAs, round-robin block
// pairing with a cluster barrier between rounds (data round-trips through L2).
struct JacobiBatch {
    int count;
    int r[kMaxSmall], c[kMaxSmall];
    cplx* W[kMaxSmall];
    int* sweeps[kMaxSmall];  // nullable: sweeps used
};
cudaError_t jacobi_svd(const JacobiBatch& b, int max_r, int max_c, cudaStream_t s);



// Load W from a row-major matrix: X = A (r x c) if !adj, or X = A^H when adj (A is c x r);
// J = I.
struct JacobiInitBatch {
    int count;
    int r[kMaxSmall], c[kMaxSmall];
    const cplx* A[kMaxSmall];
    int lda[kMaxSmall];
    int adj[kMaxSmall];
    cplx* W[kMaxSmall];
};
cudaError_t jacobi_init(const JacobiInitBatch& b, cudaStream_t s);

// After convergence: sigma_j = ||X_j||, sorted non-increasing (ties by index);
// Xn (r x c row-major, ld c) = normalised X columns in sorted order (zero for sigma = 0);
// Js (c x c row-major) = J columns in sorted order.  Either output may be null.
struct JacobiFinBatch {
    int count;
    int r[kMaxSmall], c[kMaxSmall];
    const cplx* W[kMaxSmall];
    double* sigma[kMaxSmall];
    cplx* Xn[kMaxSmall];
    cplx* Js[kMaxSmall];
};
cudaError_t jacobi_finish(const JacobiFinBatch& b, int max_c, cudaStream_t s);

// ---- reductions -----------------------------------------------------------------------------
// sum |a_i|^2 over n complex values, deterministic two-level order; also counts non-finite.
// partial: >= 2*148 doubles + 2*148 ints of scratch. out_sq / out_nonfinite: device scalars.
cudaError_t sumsq(const cplx* a, long long n, double* partial, int* partial_bad, double* out_sq,
                  int* out_nonfinite, cudaStream_t s);
// The same for many arrays in one launch pair; partial/bad: count * 296 scratch entries.
struct SumsqBatch {
    int count;
    const cplx* a[kMaxSmall];
    long long n[kMaxSmall];
    double* out_sq[kMaxSmall];
    int* out_bad[kMaxSmall];
};
cudaError_t sumsq_many(const SumsqBatch& b, double* partial, int* partial_bad, cudaStream_t s);

}  // namespace rb

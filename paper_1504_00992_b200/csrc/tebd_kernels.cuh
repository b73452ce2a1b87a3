// tebd_kernels.cuh — sketch generation and the bandwidth-bound decimation epilogue kernels.
#pragma once
#include "common.cuh"

namespace rb {

constexpr int kMaxEpi = 64;  // problems per launch of the batched epilogue kernels

// ---- Gaussian sketch Omega (n x l, row-major) --------------------------------------------
// Reference stream (randomized.cpp:17-45,79-86): std::mt19937_64(seed); entry e consumes draws
// 2e (u1 = ((x>>11)+1)·2^-53) and 2e+1 (u2 = (x>>11)·2^-53); re = r cos(2πu2), im = r sin(2πu2),
// r = sqrt(-2 ln u1).  The 64-bit Mersenne twister is sequential, so one CTA runs the twist
// (312 words per round, two parallel phases) and writes raw draws; Box–Muller is a separate
// fully parallel pass.  `draws` must hold 2*n*l uint64 rounded up to a multiple of 312.
cudaError_t omega_reference(uint64_t seed, long long n_entries, unsigned long long* draws, cplx* out,
                            cudaStream_t s);
// Philox4x32-10 keyed by seed, counter = entry index: one 128-bit output -> (u1, u2).
cudaError_t omega_philox(uint64_t seed, long long n_entries, cplx* out, cudaStream_t s);

// ---- two-site gate for small d1*d2 (memory-bound form of tebd.cpp:126-139) ---------------
// M_out[a][x][b] = sum_y G[x][y] M_in[a][y][b],  x, y < dd = d1*d2 <= 64.
cudaError_t gate_small(const cplx* G, int dd, int cl, int cr, const cplx* Min, cplx* Mout,
                       cudaStream_t s);

// ---- two-site gate with exact block structure --------------------------------------------
// A gate G (dd x dd) that is block-diagonal up to a permutation of the two-site states (e.g.
// excitation-number-conserving bosonic gates) is applied block by block: for each block B with
// state set S_B, M_out[a][S_B][b] = G_B · M_in[a][S_B][b].  One pass over Θ (bandwidth-bound)
// instead of the dense dd x dd GEMM.  Exact zeros only — the result equals the dense product.
constexpr int kMaxGateBlock = 32;
struct GateBlocks {
    int nblocks, dd;
    const int* offs;   // nblocks + 1 offsets into idx
    const int* idx;    // the dd states grouped by block (row indices into G)
    const int* goff;   // nblocks offsets into gblk
    const cplx* gblk;  // dense blocks G_B (|S_B| x |S_B|, row-major, local indices)
    int total;         // sum over blocks of |S_B|^2 (entries of gblk)
};
struct GateBlockJob {
    GateBlocks gb;
    const cplx* Min;
    cplx* Mout;
    int cl, cr;
};
struct GateBlockBatch {
    int count;
    GateBlockJob j[kMaxEpi];
};
cudaError_t gate_blocks_many(const GateBlockBatch& b, long long max_cols, cudaStream_t s);

// ---- layout conversion (i, j, a, b) <-> (a*d1+i, j*cr+b) ----------------------------------
cudaError_t theta_to_unfolded(const cplx* theta, int d1, int d2, int cl, int cr, cplx* M, cudaStream_t s);
cudaError_t unfolded_to_theta(const cplx* M, int d1, int d2, int cl, int cr, cplx* theta, cudaStream_t s);

// ---- truncation (tebd.cpp:188-209) ---------------------------------------------------------
// sigma: ns non-increasing values; total_sq: device scalar ||M||_F^2.  Writes *kept (int),
// lambda[0..kept), *discarded.  cap = chi_max (0 = no cap).
struct TruncArgs {
    const double* sigma;
    int ns;
    const double* total_sq;
    double trunc_tol;
    long long cap;
    int renormalize;
    int* kept;
    double* lambda;
    double* discarded;
    // nullable: the finite check of the same Θ (tebd.cpp:156-160).  A non-finite or identically
    // zero Θ keeps NOTHING (kept = 0: λ and the Γ reshape below write no element), so the
    // caller can throw with the state's buffers unchanged, as the reference throws before
    // assigning anything.
    const int* nonfinite = nullptr;
};
cudaError_t truncate(const TruncArgs& a, cudaStream_t s);

// ---- Gamma reshape with outer-lambda pseudo-inverse (tebd.cpp:211-235) -----------------------
// gamma_l[(a*d1+i)*kept + g] = U[(a*d1+i)*ldu + g] / ll[a]        (ll null -> 1)
// gamma_r[g*n + c]          = conj(V[c*ldv + g]) / lr[c % cr]     (lr null -> 1), n = d2*cr
// lambda < 1e-14 -> 0 and *pinv = 1.  kept is read from device memory.
struct GammaArgs {
    const cplx* U;
    int ldu;
    const cplx* V;
    int ldv;
    const double* ll;
    const double* lr;
    int m, n, d1, cr;
    const int* kept;
    cplx* gamma_l;
    cplx* gamma_r;
    int* pinv;
};
cudaError_t gamma_reshape(const GammaArgs& a, int max_kept, cudaStream_t s);

// ---- batched forms: one launch for all bonds of a sweep ----------------------------------------
struct TruncBatch {
    int count;
    TruncArgs a[kMaxEpi];
};
cudaError_t truncate_many(const TruncBatch& b, cudaStream_t s);
struct GammaBatch {
    int count;
    int max_kept, max_m, max_n;
    GammaArgs a[kMaxEpi];
};
cudaError_t gamma_reshape_many(const GammaBatch& b, cudaStream_t s);
struct PhiloxBatch {
    int count;
    uint64_t seed[kMaxEpi];
    long long n[kMaxEpi];
    cplx* out[kMaxEpi];
};
cudaError_t omega_philox_many(const PhiloxBatch& b, cudaStream_t s);
// Θ pre-scaling for the Θ GEMM: out[r][c] = in[r][c] * s[r]  (rows x cols, row-major)
struct ScaleRowsBatch {
    int count;
    const cplx* in[kMaxEpi];
    const double* s[kMaxEpi];
    int rows[kMaxEpi], cols[kMaxEpi];
    cplx* out[kMaxEpi];
};
cudaError_t scale_rows_many(const ScaleRowsBatch& b, cudaStream_t s);

cudaError_t fill_int(int* p, int v, cudaStream_t s);

// out (cols x rows) = A^H for A (rows x cols), both row-major.
cudaError_t conj_transpose(const cplx* A, int rows, int cols, cplx* out, cudaStream_t s);
// out[j] = sum_i |A(i, j)|^2 for a row-major m x n matrix (fixed summation order).
cudaError_t column_norms2(const cplx* A, int m, int n, double* out, cudaStream_t s);

// *w = clamp(1 - sum_{i<k} sigma_i^2 / total_sq, 0, 1)   (randomized.cpp:68-75)
cudaError_t discarded_weight(const double* sigma, int k, const double* total_sq, double* w,
                             cudaStream_t s);

// <psi|O|psi> at one site in canonical form (mps.cpp:50-70):
//   sum_{a,b} ll[a]^2 lr[b]^2 sum_{i',i} conj(G[a,i',b]) O[i',i] G[a,i,b]   (ll/lr null -> 1).
// res: scratch of >= 4*148+2 doubles; the result (re, im) lands in res[4*148..4*148+1].
cudaError_t expectation_local_dev(const cplx* G, int dl, int d, int dr, const double* ll,
                                  const double* lr, const cplx* op, double* res, cudaStream_t s);
// -sum λ² ln λ² (mps.cpp:40-48), sequential order.
cudaError_t schmidt_entropy_dev(const double* lam, int n, double* out, cudaStream_t s);

// Peak probes (diagnostics): TFLOP/s of DMMA f64 and of DFMA.
cudaError_t probe_peak(int what, double* tflops, cudaStream_t s);
cudaError_t probe_dmma_occupancy(int warps, int chains, double* tflops, cudaStream_t s);

}  // namespace rb

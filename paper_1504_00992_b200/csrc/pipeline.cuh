// pipeline.cuh — device-side orchestration of the decimation pipeline (host C++, enqueues
// kernels on the context stream).  Used by the C ABI (capi.cu) and the sweep engine.
#pragma once
#include "ctx.cuh"
#include "smallla.cuh"
#include "tebd_kernels.cuh"
#include "zgemm.cuh"

namespace rb {

struct Scale {
    const double* rs = nullptr;
    int rs_div = 1;
    const double* ks = nullptr;
    const double* cs = nullptr;
    int cs_mod = 1;
};

// C = op(A)·B (single problem, optional stride batch); split-K chosen automatically.
void gemm(rrsvd_b200_ctx* c, GemmOp opA, int m, int n, int k, const cplx* A, long long lda,
          const cplx* B, long long ldb, cplx* C, long long ldc, const Scale& sc = {}, int batch = 1,
          long long sA = 0, long long sB = 0, long long sC = 0);

// Q (m x l, ld l) = orthonormal basis of Y (m x l, ld l) by shifted CholeskyQR3.
// Q may alias Y.  ndead (nullable, device int) = dependent columns in the last pass.
void orth(rrsvd_b200_ctx* c, const cplx* Y, int m, int l, cplx* Q, int* ndead = nullptr);

// Gaussian sketch into `out` (n x l).
void make_omega(rrsvd_b200_ctx* c, int n, int l, uint64_t seed, int mode, cplx* out);

// RRSVD core (randomized.cpp:88-107 without the weight): A (m x n) -> U (m x l), sigma (l,
// non-increasing), V (n x l).  omega: n x l device sketch.
void rrsvd_core(rrsvd_b200_ctx* c, const cplx* A, int m, int n, int l, int q, const cplx* omega,
                cplx* U, double* sigma, cplx* V);

// Full SVD by one-sided Jacobi (linalg.cpp:67-88): U (m x r), sigma (r), V (n x r), r = min(m,n).
void svd_jacobi(rrsvd_b200_ctx* c, const cplx* A, int m, int n, cplx* U, double* sigma, cplx* V);

// Device scalars of one decimation, read back by the host at the end of an update.
struct DecimScalars {
    int kept;
    int nonfinite;
    int pinv;
    int pad;
    double total_sq;
    double discarded;
};

struct DecimPlan {  // host-side decisions of decimate (tebd.cpp:144-186)
    int m, n, minor;
    bool randomized;
    int l;      // sketch width (randomized) ; ns = l or minor
    int ns;
    int kmax;   // upper bound on the kept rank
};
DecimPlan plan_decimation(int d1, int d2, int cl, int cr, size_t chi_max, int kind, size_t target_rank,
                          size_t oversampling, size_t det_crossover);

// The whole decimation of an unfolded M on the device: norm, factorization (RRSVD or Jacobi),
// truncation, λ renormalisation, Γ reshape.  Writes gamma_l (m x kept), lambda (kept),
// gamma_r (kept x n) packed with the device-side kept; scalars into *sc (device).
void decimate_device(rrsvd_b200_ctx* c, const DecimPlan& pl, const cplx* M, int d1, int cr,
                     const double* ll, const double* lr, size_t chi_max, double trunc_tol, int q,
                     uint64_t call_seed, int omega_mode, const cplx* omega, int renormalize,
                     cplx* gamma_l, double* lambda, cplx* gamma_r, DecimScalars* sc);

// Θ = λΓλΓλ in the unfolded layout (tebd.cpp:76-124) and the gate (tebd.cpp:126-139).
void build_theta_device(rrsvd_b200_ctx* c, const cplx* G1, const cplx* G2, const double* ll,
                        const double* lm, const double* lr, int cl, int d1, int cm, int d2, int cr, cplx* M);
void apply_gate_device(rrsvd_b200_ctx* c, const cplx* G, int d1, int d2, int cl, int cr,
                       const cplx* Min, cplx* Mout);

}  // namespace rb

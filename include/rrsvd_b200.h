/* rrsvd_b200.h — C ABI of the B200-native TEBD two-site decimation library
 * (librrsvd_b200.so, sm_100a).
 *
 * Drop-in boundary for the hot path of the reference C++ core (rrsvd::core, namespace
 * rrsvd / rrsvd::tebd).  Each entry point names the reference interface it replaces
 * (file:line under /root/reference/proj).  The reference has no C ABI of its own; the
 * C++ shim in include/rrsvd_b200/rrsvd.hpp re-exposes these entry points with the
 * reference's exact C++ signatures.
 *
 * Conventions
 *  - Complex matrices are row-major, interleaved (re, im) float64 — the memory image of
 *    rrsvd::DenseMatrix (dense_matrix.hpp:13-49) and of rrsvd::tebd::Tensor3 (mps.hpp:12-26).
 *    They are passed as `double*` pointing at the first real part.
 *  - Every matrix/vector pointer may be DEVICE memory (the fast path; no copies) or HOST memory
 *    (pageable or pinned; the library stages it through its workspace — "end-to-end" mode).
 *    The kind is detected per pointer with cudaPointerGetAttributes.
 *  - All work is enqueued on the context's stream.  Functions that return host-visible results
 *    (scalars, `info` structs, sizes) synchronise that stream before returning.
 *  - Status codes mirror the reference's exceptions (errors.hpp:11-32):
 *      0 ok, 1 contract_violation, 2 numeric_failure, 3 CUDA error.
 *    rrsvd_b200_last_error(ctx) returns the message of the last failure on that context.
 *  - Contexts are not thread-safe; use one per host thread / stream (SPEC.md:112,225 allow
 *    concurrent calls on distinct inputs, which maps to distinct contexts).
 *  - There is no CPU fallback: without a usable sm_100 device, ctx_create fails.
 */
#ifndef RRSVD_B200_H
#define RRSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RRSVD_B200_OK 0
#define RRSVD_B200_CONTRACT_VIOLATION 1
#define RRSVD_B200_NUMERIC_FAILURE 2
#define RRSVD_B200_CUDA_ERROR 3

#define RRSVD_B200_OP_N 0 /* op(X) = X            (CblasNoTrans,  linalg.cpp:30-31) */
#define RRSVD_B200_OP_C 1 /* op(X) = X^H          (CblasConjTrans, linalg.cpp:30-31) */

/* Source of the Gaussian sketch Omega when the caller does not pass one explicitly. */
#define RRSVD_B200_OMEGA_REFERENCE 0 /* the reference stream of gaussian_test_matrix
                                        (randomized.cpp:17-45,79-86): mt19937_64 + Box-Muller,
                                        regenerated ON THE DEVICE from the same seed */
#define RRSVD_B200_OMEGA_PHILOX 1    /* counter-based Philox4x32-10 + Box-Muller, fully
                                        parallel (the GPU's own RNG; statistical parity) */

typedef struct rrsvd_b200_ctx rrsvd_b200_ctx;

/* == rrsvd::tebd::DecimationBackend (tebd.hpp:65-85), field for field. */
typedef struct rrsvd_b200_backend {
    int kind; /* 0 = Deterministic, 1 = Randomized */
    uint64_t target_rank;      /* 0 -> chi_max */
    uint64_t oversampling;     /* 0 -> target rank */
    uint64_t power_iterations; /* q */
    int accuracy_check;        /* fixed-precision mode with bond growth (tebd.cpp:173-179) */
    double epsilon;
    uint64_t probe_count;
    uint64_t det_crossover; /* minor <= crossover -> deterministic SVD */
    uint64_t seed;          /* base seed; the C ABI takes the per-call seed explicitly */
} rrsvd_b200_backend;

/* == the scalar part of rrsvd::tebd::DecimationResult (tebd.hpp:87-96). */
typedef struct rrsvd_b200_decim_info {
    double discarded;
    uint64_t chi;
    int randomized_path;
    int tolerance_certified;
    int pseudo_inverse_applied;
} rrsvd_b200_decim_info;

/* ---- context --------------------------------------------------------------------------- */
const char* rrsvd_b200_version(void);
/* device: CUDA ordinal; stream: a cudaStream_t (NULL = the library creates its own). */
int rrsvd_b200_ctx_create(int device, void* stream, rrsvd_b200_ctx** out);
void rrsvd_b200_ctx_destroy(rrsvd_b200_ctx* ctx);
const char* rrsvd_b200_last_error(const rrsvd_b200_ctx* ctx);
int rrsvd_b200_set_stream(rrsvd_b200_ctx* ctx, void* stream);
int rrsvd_b200_synchronize(rrsvd_b200_ctx* ctx);
/* Number of kernels this context has launched (for benchmark accounting). */
uint64_t rrsvd_b200_launch_count(const rrsvd_b200_ctx* ctx);

/* ---- L1: dense linear algebra (linalg.hpp:29-56) ---------------------------------------- */
/* C (m x n) = op_a(A) (m x k) * op_b(B) (k x n); replaces rrsvd::gemm (linalg.cpp:20-35).
 * lda/ldb/ldc are row strides in complex elements (of A, B as stored: B is n x k for op_b = C). */
int rrsvd_b200_zgemm(rrsvd_b200_ctx* ctx, int op_a, int op_b, size_t m, size_t n, size_t k,
                     const double* A, size_t lda, const double* B, size_t ldb, double* C,
                     size_t ldc);
/* The same product (op_b = N) through the INT8 tensor-core emulation of the RRSVD A-products
 * (csrc/ozaki.cuh: Chinese-remainder / Ozaki-II scheme, `moduli` in [8, 16] residue moduli;
 * 16 = FP64-class normwise accuracy).  Diagnostic entry for the parity tests and benchmarks of
 * that path; needs m, k in [128, 32768]. */
int rrsvd_b200_ozaki_zgemm(rrsvd_b200_ctx* ctx, int op_a, size_t m, size_t n, size_t k,
                           const double* A, size_t lda, const double* B, size_t ldb, double* C,
                           size_t ldc, int moduli);
/* An A prepared once for many emulated products (residue planes kept on the device until
 * release): prepare, then C = op(A)·X (accumulate = 1: C += op(A)·X, C on the device) for as many
 * panels X (k x l) as needed — the row-sharded RRSVD applies each shard 2q+2 times; a prepared
 * column block of a wider A gives that A's products by K-chunks.  ozaki_usable: the moduli count the library would use for
 * an m x n A (0: the emulation is off or the shape is outside it). */
typedef struct rrsvd_b200_ozaki_a rrsvd_b200_ozaki_a;
int rrsvd_b200_ozaki_usable(size_t m, size_t n);
int rrsvd_b200_ozaki_prepare(rrsvd_b200_ctx* ctx, const double* A, size_t m, size_t n, size_t lda, int moduli,
                             rrsvd_b200_ozaki_a** out);
int rrsvd_b200_ozaki_apply(rrsvd_b200_ctx* ctx, const rrsvd_b200_ozaki_a* a, int op_a, const double* X, size_t l,
                           size_t ldx, double* C, size_t ldc, int accumulate);
void rrsvd_b200_ozaki_release(rrsvd_b200_ozaki_a* a);
/* Thin orthonormal basis Q (m x n, m >= n) of A plus R = Q^H A (n x n), A = Q R; replaces
 * rrsvd::qr (linalg.cpp:49-65).  Like the reference's Householder QR, Q is orthonormal for ANY
 * A (linalg.hpp:35-37): columns of a rank-deficient A that CholeskyQR finds dependent get an
 * orthonormal completion (orthogonal to the live columns), and R has (near-)zero rows there. */
int rrsvd_b200_qr(rrsvd_b200_ctx* ctx, const double* A, size_t m, size_t n, double* Q, double* R);
/* One shifted-CholeskyQR factor step on an already-formed (e.g. all-reduced) Gram matrix:
 * T = R^-1 (l x l, upper) with G + s I = R^H R, s = shift_scale * 2^-53 * trace(G) (0: none;
 * the CholeskyQR passes use 10 * (rows + l)).  Only the upper triangle of G is read.
 * Non-positive pivots mark dependent columns: their T columns are zero, *ndead counts them.
 * The building block of the row-sharded QR (linalg.cpp:49-65 over a distributed Y). */
int rrsvd_b200_chol_inv(rrsvd_b200_ctx* ctx, const double* G, size_t l, double shift_scale,
                        double* T, int* ndead);
/* The same, also reporting *ill = 1 when some pivot fell below 1e4 x the shift (or died): the
 * device orthonormalisation's trigger for its extra passes (the adaptive CholeskyQR schedule,
 * used by the row-sharded QR). */
int rrsvd_b200_chol_inv_flags(rrsvd_b200_ctx* ctx, const double* G, size_t l, double shift_scale,
                              double* T, int* ndead, int* ill);

/* Full economy SVD A = U diag(S) V^H (U m x r, S r, V n x r, r = min(m,n)), S non-increasing;
 * replaces rrsvd::svd_full (linalg.cpp:67-88).  One-sided Jacobi on the device. */
int rrsvd_b200_svd(rrsvd_b200_ctx* ctx, const double* A, size_t m, size_t n, double* U,
                   double* S, double* V);
/* ||A||_F (linalg.cpp:136-139). */
int rrsvd_b200_frobenius_norm(rrsvd_b200_ctx* ctx, const double* A, size_t m, size_t n,
                              double* out);

/* ---- L2: randomized SVD (randomized.hpp:48-61) ------------------------------------------ */
/* n x l Gaussian test matrix; mode RRSVD_B200_OMEGA_REFERENCE reproduces
 * rrsvd::gaussian_test_matrix(n, l, seed) (randomized.cpp:79-86) to the last ulp of the
 * device's log/sin/cos. */
int rrsvd_b200_gaussian_test_matrix(rrsvd_b200_ctx* ctx, size_t n, size_t l, uint64_t seed,
                                    int mode, double* out);
/* randomized_range_finder (randomized.cpp:88-99): Q (m x l, orthonormal) spanning
 * (A A^H)^q A Omega, re-orthonormalised after every product; l <= min(m, n).  omega as for
 * rrsvd_b200_sketched_svd.  Replaces rrsvd::randomized_range_finder -> RangeBasis
 * (randomized.hpp:25-28,52-53). */
int rrsvd_b200_range_finder(rrsvd_b200_ctx* ctx, const double* A, size_t m, size_t n, size_t l,
                            size_t q, uint64_t seed, int omega_mode, const double* omega, double* Q);
/* rrsvd_sketched_svd (randomized.cpp:101-107): U m x l, S l, V n x l, *discarded = w.
 * omega: NULL -> generated from `seed` with `omega_mode`; else the caller's n x l sketch
 * ("Omega fed identically"). */
int rrsvd_b200_sketched_svd(rrsvd_b200_ctx* ctx, const double* A, size_t m, size_t n, size_t l,
                            size_t q, uint64_t seed, int omega_mode, const double* omega,
                            double* U, double* S, double* V, double* discarded);
/* rrsvd_fixed_rank (randomized.cpp:109-122): U m x k, S k, V n x k (U, V may be NULL). */
int rrsvd_b200_fixed_rank(rrsvd_b200_ctx* ctx, const double* A, size_t m, size_t n, size_t k,
                          size_t p, size_t q, uint64_t seed, int omega_mode, const double* omega,
                          double* U, double* S, double* V, double* discarded);

/* `count` independent rrsvd_fixed_rank calls on same-shaped matrices, batched through every
 * stage of the pipeline (one launch per stage for all of them).  A[i] (m x n), seeds[i]; U[i],
 * S[i], V[i] as in rrsvd_b200_fixed_rank (U/V entries may be NULL); discarded[count]. */
int rrsvd_b200_fixed_rank_batch(rrsvd_b200_ctx* ctx, size_t count, const double* const* A, size_t m,
                                size_t n, size_t k, size_t p, size_t q, const uint64_t* seeds,
                                int omega_mode, double* const* U, double* const* S,
                                double* const* V, double* discarded);

/* rrsvd_fixed_precision (randomized.hpp:64-66, randomized.cpp:124-176) with
 * AccuracyCheckParams{epsilon, probe_count, growth_block} (randomized.hpp:30-35): range finder at
 * initial_l, then probe rounds (seeds seed + 0x9e3779b97f4a7c15 * draw) that certify
 * max_j ||(I - Q Q^H) A omega_j|| <= epsilon or grow the basis by growth_block columns
 * (0 doubles it; never past min(m, n)).  Writes all
 * l produced columns: U (m x l), S (l), V (n x l) — size them for l = min(m, n) — and *l_out,
 * *certified (tolerance_certified), *discarded (w over all l values).  omega_mode selects the
 * reference mt19937_64 stream or Philox for every draw. */
int rrsvd_b200_fixed_precision(rrsvd_b200_ctx* ctx, const double* A, size_t m, size_t n,
                               size_t initial_l, size_t q, size_t probe_count, size_t growth_block,
                               double epsilon, uint64_t seed, int omega_mode, double* U, double* S, double* V,
                               size_t* l_out, int* certified, double* discarded);

/* ---- L3: the TEBD two-site trio in the unfolded layout (tebd.hpp:98-110) ---------------
 * Unfolded two-site matrix M: (cl*d1) x (d2*cr), row a*d1+i, column j*cr+b (tebd.cpp:150-155).
 * Gamma tensors are Tensor3 (left, phys, right) row-major (mps.hpp:20-25). */
/* build_theta (tebd.cpp:76-124): M = diag(ll (x) 1) G1 diag(lm) G2 diag(1 (x) lr);
 * ll/lr NULL = open chain end (unit weights, tebd.cpp:82-87). */
int rrsvd_b200_build_theta_unfolded(rrsvd_b200_ctx* ctx, const double* G1, const double* G2,
                                    const double* ll, const double* lm, const double* lr,
                                    size_t cl, size_t d1, size_t cm, size_t d2, size_t cr,
                                    double* M);
/* apply_gate_to_theta (tebd.cpp:126-139) on M: M_out[a] = G * M_in[a] for every left index a,
 * where M[a] is the contiguous (d1*d2) x cr block.  G is (d1*d2)^2, rows/cols i*d2+j. */
int rrsvd_b200_apply_gate_unfolded(rrsvd_b200_ctx* ctx, const double* G, size_t d1, size_t d2,
                                   size_t cl, size_t cr, const double* M_in, double* M_out);
/* decimate (tebd.cpp:141-237) of the unfolded M.  call_seed is the value the reference takes
 * from backend.seed++ (tebd.cpp:162).  Outputs are sized for chi <= min(chi_max or minor, l):
 * gamma_l cl x d1 x chi, lambda chi, gamma_r chi x d2 x cr (packed with the returned chi).
 * With backend->accuracy_check the fixed-precision path may grow the bond past chi_max
 * (tebd.cpp:177-179): size the outputs for chi <= min(d1*cl, d2*cr) then. */
int rrsvd_b200_decimate_unfolded(rrsvd_b200_ctx* ctx, const double* M, size_t d1, size_t d2,
                                 size_t cl, size_t cr, const double* ll, const double* lr,
                                 size_t chi_max, double trunc_tol,
                                 const rrsvd_b200_backend* backend, uint64_t call_seed,
                                 int omega_mode, const double* omega, int renormalize,
                                 double* gamma_l, double* lambda, double* gamma_r,
                                 rrsvd_b200_decim_info* info);
/* Layout conversions at the drop-in boundary: ThetaTensor (i, j, a, b) (tebd.hpp:23-28)
 * <-> unfolded M (a*d1+i, j*cr+b). */
int rrsvd_b200_theta_to_unfolded(rrsvd_b200_ctx* ctx, const double* theta, size_t d1, size_t d2,
                                 size_t cl, size_t cr, double* M);
int rrsvd_b200_unfolded_to_theta(rrsvd_b200_ctx* ctx, const double* M, size_t d1, size_t d2,
                                 size_t cl, size_t cr, double* theta);

/* ---- device-resident MPS and TEBD evolution (mps.hpp:31-41, tebd.hpp:52-144) ----------- */
typedef struct rrsvd_b200_mps rrsvd_b200_mps;

/* == rrsvd::tebd::TrotterPlan::Sweep (tebd.hpp:52-62). */
typedef struct rrsvd_b200_sweep {
    int bond_parity;
    double coefficient;
} rrsvd_b200_sweep;

/* == rrsvd::tebd::EvolveOptions (tebd.hpp:126-130) + the sketch source. */
typedef struct rrsvd_b200_evolve_options {
    double abort_discarded_threshold; /* cumulative fraction; 1 never aborts */
    int renormalize;
    int omega_mode; /* RRSVD_B200_OMEGA_REFERENCE or _PHILOX */
} rrsvd_b200_evolve_options;

/* == rrsvd::tebd::EvolveDiagnostics scalars (tebd.hpp:132-138). */
typedef struct rrsvd_b200_evolve_diag {
    double kept_fraction;
    uint64_t max_bond_dim;
    int aborted;
    uint64_t abort_step;
    uint64_t n_updates;
} rrsvd_b200_evolve_diag;

/* == rrsvd::tebd::UpdateRecord (tebd.hpp:115-124); times are CUDA-event device times (us). */
typedef struct rrsvd_b200_update_record {
    uint64_t step, bond, chi;
    double discarded_weight;
    double t_theta_us, t_gate_us, t_svd_us;
    int randomized_path;
} rrsvd_b200_update_record;

/* MpsState on the device (mps.hpp:31-41), initialised to the product state |0...0>
 * (mps_product_state, mps.cpp:15-38, with every local state e_0).  chi_max 0 = unbounded. */
int rrsvd_b200_mps_create(rrsvd_b200_ctx* ctx, size_t n_sites, const size_t* site_dims,
                          size_t chi_max, double trunc_tolerance, rrsvd_b200_mps** out);
void rrsvd_b200_mps_destroy(rrsvd_b200_mps* mps);
/* Γ of `site` (dim_left x d x dim_right) and, unless `site` is the last one, the λ of bond
 * `site` (dim_right values).  dim_left must equal the right dimension of site-1. */
int rrsvd_b200_mps_set_site(rrsvd_b200_mps* mps, size_t site, size_t dim_left, size_t dim_right,
                            const double* gamma, const double* lambda_right);
/* Chain-block support for the multi-GPU partition: the weights of the bonds
 * OUTSIDE this block — left of site 0 and right of the last site — i.e. the neighbouring
 * blocks' λ.  NULL = open chain end (unit weights, tebd.cpp:82-87).  With edge weights set,
 * the end sites may carry bond dimensions > 1. */
int rrsvd_b200_mps_set_edge_lambdas(rrsvd_b200_mps* mps, const double* left, size_t n_left,
                                    const double* right, size_t n_right);
/* dims3 <- (left, phys, right); gamma / lambda_right copied out when non-NULL. */
int rrsvd_b200_mps_get_site(rrsvd_b200_mps* mps, size_t site, size_t* dims3, double* gamma,
                            double* lambda_right);
/* The whole state in one call (SURVEY §8(b) "rrsvd_b200_state_{upload,download}"; the
 * MpsState constructor / field reads of mps.hpp:31-41): every site's Γ (dims[3*i+0] x d_i x
 * dims[3*i+2]; dims[3*i+1] is ignored on upload) and every bond's λ (lambdas[i], i < n-1; a NULL
 * entry skips that λ).  All copies are queued on the context's stream and synchronised once —
 * host buffers (pinned for full PCIe rate) may be reused when the call returns.  Download fills
 * dims (when non-NULL) and requires gammas[i] to hold the current size (query with dims first
 * by passing gammas = NULL). */
int rrsvd_b200_state_upload(rrsvd_b200_mps* mps, const size_t* dims, const double* const* gammas,
                            const double* const* lambdas);
int rrsvd_b200_state_download(rrsvd_b200_mps* mps, size_t* dims, double* const* gammas, double* const* lambdas);
/* download into the (pinned) host buffers and upload back from them, pipelined per site on two
 * streams (the D2H and H2D copy engines overlap); dims unchanged.  The state a caller keeps on the
 * host between consecutive steps, at the cost of one direction instead of two. */
int rrsvd_b200_state_roundtrip(rrsvd_b200_mps* mps, double* const* gammas, double* const* lambdas);
/* evolve (tebd.cpp:260-326): n_steps x sweeps x (bonds of the sweep's parity, ascending):
 * build_theta -> gate -> decimate on the device, state resident in HBM.  gates[s*(n_sites-1)+b]
 * is the (d_b d_{b+1})^2 gate exp(-i c_s dt h_b) for sweep s (NULL = no term on that bond); the
 * caller builds it (bond_gate, tebd.cpp:239-258).  backend->seed advances once per update, like
 * the reference (tebd.cpp:162).  records (may be NULL) receives up to max_records updates. */
int rrsvd_b200_evolve(rrsvd_b200_mps* mps, size_t n_sweeps, const rrsvd_b200_sweep* sweeps,
                      const double* const* gates, size_t n_steps, rrsvd_b200_backend* backend,
                      const rrsvd_b200_evolve_options* options, rrsvd_b200_evolve_diag* diag,
                      rrsvd_b200_update_record* records, size_t max_records);
/* A two-site gate made resident on the device once: the copy plus its exact block structure
 * (connected components of the nonzero pattern; excitation-number-conserving gates are
 * block-diagonal up to a permutation and are then applied block-sparsely — same result as the
 * dense product).  The gate passed to the reference is a TwoSiteGate (tebd.hpp:35-39). */
typedef struct rrsvd_b200_gate rrsvd_b200_gate;
int rrsvd_b200_gate_create(rrsvd_b200_ctx* ctx, const double* G, size_t dd, rrsvd_b200_gate** out);
void rrsvd_b200_gate_destroy(rrsvd_b200_gate* gate);
/* 1 if the gate is applied block-sparsely (nblocks out), 0 if dense. */
int rrsvd_b200_gate_blocks(const rrsvd_b200_gate* gate, size_t* nblocks);
/* evolve with prepared gates: gates[s*(n_sites-1)+b] (NULL = no term). */
int rrsvd_b200_evolve_prepared(rrsvd_b200_mps* mps, size_t n_sweeps, const rrsvd_b200_sweep* sweeps,
                               const rrsvd_b200_gate* const* gates, size_t n_steps,
                               rrsvd_b200_backend* backend, const rrsvd_b200_evolve_options* options,
                               rrsvd_b200_evolve_diag* diag, rrsvd_b200_update_record* records,
                               size_t max_records);
/* <psi| O_site |psi> (mps.cpp:50-70) -> out2 = (re, im); S = -sum λ² ln λ² (mps.cpp:40-48). */
int rrsvd_b200_expectation_local(rrsvd_b200_mps* mps, size_t site, const double* op, double* out2);
int rrsvd_b200_schmidt_entropy(rrsvd_b200_mps* mps, size_t bond, double* out);

/* ---- multi-GPU: the chain-block partition (tebd.cpp:289-323 per rank) --------
 * One rank per GPU owns the contiguous sites [first_site, first_site + owned) of an n_global-site
 * chain; its device MPS (`block`) holds the owned sites plus, unless it is the last rank, a ghost
 * copy of the next rank's first site, so the boundary bond is an ordinary local bond.  Per sweep:
 * (1) ghost Γ + right-edge λ from rank+1, left-edge λ from rank-1 (one grouped send/recv on the
 * context's stream); (2) the rank's bonds of the sweep's parity as one batch (evolve); (3) the
 * updated ghost Γ back to its owner.  Messages have fixed capacities (chi_max x d x chi_max
 * complexes; chi_max must be > 0) with a 3-integer dims header, so no shape round trip.  Seeds
 * are the GLOBAL call indices (backend->seed = the base for global index 0, tebd.cpp:162), so a
 * partitioned run reproduces the single-GPU one; backend->seed ends where the unpartitioned
 * evolve's would.  gates[s * (block sites - 1) + local bond] as in rrsvd_b200_evolve_prepared;
 * term_bonds[n_global - 1] flags the GLOBAL bonds that carry a term.  step0 offsets the step
 * index of the seeds (continuing runs).  The discarded-weight budget is not supported
 * (abort_discarded_threshold must stay 1); diag is this rank's (multiply kept fractions across
 * ranks). */
typedef struct rrsvd_b200_comm rrsvd_b200_comm;
/* NCCL (libnccl.so.2, loaded at run time): rank 0 makes the 128-byte id and shares it out of band. */
int rrsvd_b200_comm_unique_id(void* id128);
int rrsvd_b200_comm_create_nccl(rrsvd_b200_ctx* ctx, int nranks, int rank, const void* id128,
                                rrsvd_b200_comm** out);
/* Host-staged loopback between host threads of one process (protocol checks on one GPU). */
typedef struct rrsvd_b200_loopback_hub rrsvd_b200_loopback_hub;
int rrsvd_b200_loopback_hub_create(int nranks, rrsvd_b200_loopback_hub** out);
void rrsvd_b200_loopback_hub_destroy(rrsvd_b200_loopback_hub* hub);
int rrsvd_b200_comm_create_loopback(rrsvd_b200_ctx* ctx, rrsvd_b200_loopback_hub* hub, int rank,
                                    rrsvd_b200_comm** out);
void rrsvd_b200_comm_destroy(rrsvd_b200_comm* comm);
int rrsvd_b200_evolve_partitioned(rrsvd_b200_mps* block, rrsvd_b200_comm* comm, size_t first_site,
                                  size_t n_global, size_t n_sweeps, const rrsvd_b200_sweep* sweeps,
                                  const rrsvd_b200_gate* const* gates, const unsigned char* term_bonds,
                                  size_t n_steps, uint64_t step0, rrsvd_b200_backend* backend,
                                  const rrsvd_b200_evolve_options* options, rrsvd_b200_evolve_diag* diag);

/* evolve splits each sweep's bonds over two auxiliary streams so one half's latency-bound
 * kernels overlap the other half's GEMMs (default on).  Off = one stream, serial stages. */
int rrsvd_b200_set_overlap(rrsvd_b200_ctx* ctx, int on);

/* ---- diagnostics ------------------------------------------------------------------------ */
/* Event-time every zgemm launch (with its split-K reduction) on this context; on = 1 also
 * resets the counters.  Stats are cumulative algorithmic flops (8 m n k per complex GEMM),
 * device milliseconds and launch count. */
int rrsvd_b200_set_gemm_timing(rrsvd_b200_ctx* ctx, int on);
int rrsvd_b200_gemm_stats(rrsvd_b200_ctx* ctx, double* flops, double* ms, uint64_t* calls);
/* Of the same launches: the flops the DMMA pipe actually executed (6 real flops per complex MAC
 * for 3M-form launches, 8 for 4M) and the milliseconds spent in TMA-staged launches. */
int rrsvd_b200_gemm_pipe_stats(rrsvd_b200_ctx* ctx, double* executed_flops, double* tma_ms);
/* The same split by stage (8 slots): 0 theta, 1 gate, 2 RRSVD A-products (the DMMA ones), 3 QR
 * Gram, 4 QR apply, 5 small-SVD assembly, 6 deterministic-SVD preconditioning. */
int rrsvd_b200_gemm_stage_stats(rrsvd_b200_ctx* ctx, double* flops8, double* ms8);
/* The emulated A-products (csrc/ozaki.cuh) timed under the same switch, kept out of the DMMA
 * counters: FP64-equivalent flops (8 m n k), milliseconds, algorithmic HBM bytes and launch groups
 * of the products; milliseconds and bytes of the A residue preparations. */
int rrsvd_b200_ozaki_stats(rrsvd_b200_ctx* ctx, double* flops, double* ms, double* bytes, uint64_t* calls,
                           double* prep_ms, double* prep_bytes);
/* The INT8 tensor-core GEMM kernel of the emulated products alone (event-timed around its launch):
 * milliseconds and the HBM bytes it must move (A residue tiles + panel read, residue products written). */
int rrsvd_b200_ozaki_gemm_stats(rrsvd_b200_ctx* ctx, double* ms, double* bytes);
/* Measured device peak: what = 0 FP64 DMMA (mma.sync f64), 1 FP64 DFMA; TFLOP/s. */
int rrsvd_b200_probe_peak(rrsvd_b200_ctx* ctx, int what, double* tflops);

#ifdef __cplusplus
}
#endif
#endif

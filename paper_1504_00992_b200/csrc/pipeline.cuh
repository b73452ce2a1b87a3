// pipeline.cuh — host orchestration of the decimation pipeline (enqueues kernels on the context
// stream).  Every stage is BATCHED: a vector of independent problems (e.g. all same-parity bonds
// of a TEBD sweep, which the reference processes one by one, tebd.cpp:291-306) goes through each
// stage as a grouped launch, so the latency-bound small-matrix kernels (Cholesky, Jacobi) run
// side by side on different SMs and the GEMM grids fill the 148 SMs.
#pragma once
#include <vector>

#include "blockjac.cuh"
#include "ozaki.cuh"
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

struct GemmSpec {
    int m, n, k;
    const cplx* A;
    long long lda;
    const cplx* B;
    long long ldb;
    cplx* C;
    long long ldc;
    Scale sc{};
    int batch = 1;
    long long sA = 0, sB = 0, sC = 0;
    int structure = kGeneral;  // kTriB / kUpperC hints (zgemm.cuh)
    int nsub = 0;              // column-blocked B/C (zgemm.cuh)
    long long subB = 0, subC = 0;
    const cplx* D = nullptr;   // optional addend: C = D + alpha * product (zgemm.cuh)
    long long ldd = 0;
    double alpha = 1.0;
    const int* pred = nullptr;  // optional device predicate (zgemm.cuh)
    int pred_want = 1;
};

// Grouped complex GEMMs sharing op(A); split-K chosen so the whole group fills the GPU.
void gemm_many(rrsvd_b200_ctx* c, GemmOp opA, const std::vector<GemmSpec>& specs);
void gemm(rrsvd_b200_ctx* c, GemmOp opA, int m, int n, int k, const cplx* A, long long lda,
          const cplx* B, long long ldb, cplx* C, long long ldc, const Scale& sc = {}, int batch = 1,
          long long sA = 0, long long sB = 0, long long sC = 0);

// Q (m x l, ld l) = orthonormal basis of Y (m x l, ld l): shifted CholeskyQR3 (Fukaya et al.)
// with dependent-column zeroing.  Q may alias Y.
struct OrthSpec {
    const cplx* Y;
    int m, l;
    cplx* Q;
    int* ndead = nullptr;
};
// passes = kFullPasses: two shifted CholeskyQR passes then two plain ones — an orthonormal
// basis of the full span (the reference's Householder QR, linalg.cpp:49-65, keeps every live
// direction too).  passes = kSpanPasses: the two shifted passes only — a well-conditioned basis
// of the same span (cond <= ~1e5), enough for the intermediate power-iteration bases.
constexpr int kFullPasses = 4;
constexpr int kSpanPasses = 2;
// kRobustSpanPasses: the span schedule's single shifted pass when Y is well conditioned, otherwise
// two shifted and two plain passes (an orthonormal basis of an ill-conditioned or rank-deficient Y)
constexpr int kRobustSpanPasses = 3;
void orth_many(rrsvd_b200_ctx* c, const std::vector<OrthSpec>& specs, int passes = kFullPasses);
void orth(rrsvd_b200_ctx* c, const cplx* Y, int m, int l, cplx* Q, int* ndead = nullptr);

// T = R^-1 (l x l, upper) for G (+ s I) = R^H R, s = shift_scale * u * trace(G) (0: none), any
// l: one chol_inv block up to kMaxCholL, else block-right-looking with DMMA updates.  G (upper
// triangle read) is overwritten.  Non-positive pivots mark dependent columns (zero T columns).
struct CholSpec {
    cplx* G;
    int l;
    double shift_scale;
    cplx* T;
    int* ndead;
    int* ill_out = nullptr;     // nullable: set to 1 if a pivot falls within kIllRatio of the shift
    const int* pred = nullptr;  // nullable: the whole factorization runs only if *pred != 0
};
void chol_inv_many(rrsvd_b200_ctx* c, const std::vector<CholSpec>& specs);

// Gaussian sketch into `out` (n x l).
void make_omega(rrsvd_b200_ctx* c, int n, int l, uint64_t seed, int mode, cplx* out);

// RRSVD core (randomized.cpp:88-107 without the weight): A (m x n) -> U (m x l), sigma (l,
// non-increasing), V (n x l).  omega: n x l device sketch.
struct RrsvdSpec {
    const cplx* A;
    int m, n, l, q;
    const cplx* omega;
    cplx* U;
    double* sigma;
    cplx* V;
    double* total_sq = nullptr;  // optional: ||A||_F^2 and the non-finite flag (sumsq), taken by the
    int* nonfinite = nullptr;    // emulation's row-exponent pass when A is emulated, else by sumsq
};
void rrsvd_core_many(rrsvd_b200_ctx* c, const std::vector<RrsvdSpec>& specs);

// The two halves of rrsvd_core: the range finder (randomized.cpp:88-99) producing an
// orthonormal Q (m x l), and assemble_from_basis (randomized.cpp:57-66): U (m x l), sigma, V.
struct RangeSpec {
    const cplx* A;
    int m, n, l, q;
    const cplx* omega;
    cplx* Q;
    const OzakiA* oz = nullptr;  // A's residue planes: the A-products on the INT8 emulation
};
void range_finder_many(rrsvd_b200_ctx* c, const std::vector<RangeSpec>& specs);
struct AssembleSpec {
    const cplx* A;
    int m, n, l;
    const cplx* Q;
    cplx* U;
    double* sigma;
    cplx* V;
    const OzakiA* oz = nullptr;
};
void assemble_many(rrsvd_b200_ctx* c, const std::vector<AssembleSpec>& specs);

// Fixed-precision RRSVD with the probabilistic accuracy check and basis growth
// (randomized.cpp:124-176).  Inputs: A, m, n, l0 (initial width), q, probes, eps, seed, omega_mode,
// growth_block (columns appended per failed round; 0 doubles the basis, randomized.cpp:156).  Outputs (host-visible after the call): l (final width), certified, and
// workspace device buffers U (m x l), sigma (l), V (n x l).  Synchronises once per round.
struct FixedPrecSpec {
    const cplx* A;
    int m, n, l0, q, probes;
    double eps;
    uint64_t seed;
    int omega_mode;
    const cplx* omega0 = nullptr;  // nullable: the initial n x l0 sketch, fed instead of drawn
    int growth_block = 0;          // AccuracyCheckParams::growth_block (randomized.hpp:34)
    int l = 0;
    bool certified = false;
    cplx* U = nullptr;
    double* sigma = nullptr;
    cplx* V = nullptr;
};
void rrsvd_fixed_precision_many(rrsvd_b200_ctx* c, std::vector<FixedPrecSpec>& specs);
void rrsvd_core(rrsvd_b200_ctx* c, const cplx* A, int m, int n, int l, int q, const cplx* omega,
                cplx* U, double* sigma, cplx* V);

// Full SVD by QR-preconditioned one-sided Jacobi (linalg.cpp:67-88):
// U (m x r), sigma (r), V (n x r), r = min(m,n).
struct SvdSpec {
    const cplx* A;
    int m, n;
    cplx* U;
    double* sigma;
    cplx* V;
};
void svd_jacobi_many(rrsvd_b200_ctx* c, const std::vector<SvdSpec>& specs);
void svd_jacobi(rrsvd_b200_ctx* c, const cplx* A, int m, int n, cplx* U, double* sigma, cplx* V);

// Device scalars of one decimation, read back by the host at the end of an update/sweep.
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
    bool fixed_precision;  // accuracy check with bond growth (tebd.cpp:173-179)
    int probes;
    int l;      // (initial) sketch width (randomized) ; ns = l or minor
    int ns;     // singular values produced (an upper bound when fixed_precision)
    int kmax;   // upper bound on the kept rank (no chi_max cap when fixed_precision)
};
DecimPlan plan_decimation(int d1, int d2, int cl, int cr, size_t chi_max, int kind, size_t target_rank,
                          size_t oversampling, size_t det_crossover, int accuracy_check = 0,
                          size_t probe_count = 0);

// True when decimate_many synchronises the host for this plan (the block Jacobi's per-sweep
// convergence read, the accuracy check's per-round certification): such batches gain nothing
// from lanes, which are submitted one after the other from the host.
bool decimation_syncs_host(const DecimPlan& pl);
// RRSVD_B200_DEBUG set: per-call diagnostics on stderr
bool debug_enabled();

// One decimation of an unfolded M (tebd.cpp:141-237): norm, factorization (RRSVD or Jacobi),
// truncation, λ renormalisation, Γ reshape.  Writes gamma_l (m x kept), lambda (kept),
// gamma_r (kept x n) packed with the device-side kept; scalars into *sc (device).
struct DecimJob {
    DecimPlan pl;
    const cplx* M;
    int d1, cr;
    const double* ll;
    const double* lr;
    size_t chi_max;
    double trunc_tol;
    int q;
    uint64_t seed;
    int omega_mode;
    const cplx* omega;  // nullable: generate from seed
    int renormalize;
    cplx* gamma_l;
    double* lambda;
    cplx* gamma_r;
    DecimScalars* sc;
    double eps = 0.0;          // accuracy-check tolerance (fixed_precision plans)
    int* certified = nullptr;  // host, nullable: tolerance_certified (fixed_precision plans)
};
void decimate_many(rrsvd_b200_ctx* c, const std::vector<DecimJob>& jobs);

// Θ = λΓλΓλ in the unfolded layout (tebd.cpp:76-124) and the gate (tebd.cpp:126-139).
struct ThetaJob {
    const cplx* G1;
    const cplx* G2;
    const double* ll;
    const double* lm;
    const double* lr;
    int cl, d1, cm, d2, cr;
    cplx* M;
};
void build_theta_many(rrsvd_b200_ctx* c, const std::vector<ThetaJob>& jobs);
struct GateJob {
    const cplx* G;
    int d1, d2, cl, cr;
    const cplx* Min;
    cplx* Mout;
    const GateBlocks* blocks = nullptr;  // exact block structure of G (block kernel) or dense
};
void apply_gate_many(rrsvd_b200_ctx* c, const std::vector<GateJob>& jobs);

// Exact block structure of a gate (connected components of its nonzero pattern, host-side, once
// per gate).  Device arrays are allocated on c->stream and must be freed with free_gate_blocks.
// Returns false (nothing allocated) when G is dense or a block exceeds kMaxGateBlock.
struct GateBlocksOwned {
    GateBlocks dev{};
    std::vector<void*> bufs;
};
bool make_gate_blocks(rrsvd_b200_ctx* c, const cplx* G, int dd, GateBlocksOwned& out);
void free_gate_blocks(rrsvd_b200_ctx* c, GateBlocksOwned& g);

}  // namespace rb

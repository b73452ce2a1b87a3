// blockjac.cuh — block one-sided Jacobi SVD for problems beyond the on-chip cluster kernel
// (deterministic decimation of large minor dimensions, C2's batched 256^2, wide fixed-precision
// bases).  The same Hestenes iteration as jacobi_kernel, reorganised around GEMMs:
//
//   columns of X (r x c, padded to cp = nbp*b) form nbp blocks of b; a circle-method tournament
//   pairs the blocks, pair k occupying the adjacent slots 2k, 2k+1.  One step, for all pairs
//   (bj_step_kernel, one CTA per pair):
//     G_k = [X_i X_j]^H [X_i X_j]          row chunks staged in shared memory, fixed order
//     W_k = one sweep of two-sided Jacobi  the Hestenes rotations applied to the Gram (same
//           on G_k                         formulas, same scaled stopping test), accumulating
//                                          the 2b x 2b unitary W_k
//     [X_i X_j] W_k, [V_i V_j] W_k         written to the blocks' positions of the next step
//                                          in the other buffer
//   The Gram is recomputed from the columns every step (rounding never accumulates in it); a
//   sweep visits every block pair once; the iteration stops after a sweep whose pair solves all
//   found their Gram already diagonal to tol = sqrt(r)·eps in the scaled sense.
#pragma once
#include "common.cuh"

namespace rb {

constexpr int kBjMaxProblems = 64;
constexpr int kBjMaxSlots = 512;  // padded blocks per problem (c <= 512*b)

struct BjInit {
    int count, r, c, cp, b, nbp;
    const cplx* A[kBjMaxProblems];  // the matrix to decompose: element (i, j) = adj ? conj(A[j*lda+i]) : A[i*lda+j]
    int lda[kBjMaxProblems], adj[kBjMaxProblems];
    cplx* X[kBjMaxProblems];  // r x cp row-major, slots in step-0 placement
    cplx* V[kBjMaxProblems];  // cp x cp row-major (rows: original column index; columns: slots)
    int place[kBjMaxSlots];   // block id at each slot's block position (step-0 placement)
};
cudaError_t bj_init(const BjInit& a, cudaStream_t s);

// One tournament step for every block pair of every problem, fused (one CTA per pair): the
// pair's Gram from row chunks staged in shared memory, one sweep of the pair solve, then
// [X_i X_j] W and [V_i V_j] W written straight to the blocks' positions of the next step.
// per-problem sweep statistics (zeroed by the host before each sweep)
struct BjStat {
    int rot;                  // rotations applied
    int pad;
    unsigned long long off2;  // max over rotated pairs of |g_pq|^2 / (g_pp g_qq), as ordered bits
};

struct BjStep {
    int count, r, cp, b, npairs;
    int inner_sweeps;  // sweeps of the pair solve per step (stops early once a sweep rotates nothing)
    int cross_only;    // rotate only the cross (block i, block j) column pairs (steps after the first)
    const cplx* Xs[kBjMaxProblems];
    cplx* Xd[kBjMaxProblems];
    const cplx* Vs[kBjMaxProblems];
    cplx* Vd[kBjMaxProblems];
    BjStat* stat[kBjMaxProblems];  // per-problem sweep statistics (added to / maxed into)
    int dst[kBjMaxSlots];      // block position now -> block position at the next step
};
cudaError_t bj_step(const BjStep& a, cudaStream_t s);

// Row slices (cluster size) bj_step uses for this many block pairs of r rows; 1 = the
// persistent sweep kernel applies.
int bj_slices(int pairs, int r);

// One whole sweep (all nsteps tournament steps) in one launch of single-CTA pairs.
struct BjSweep {
    int count, r, cp, b, npairs, nsteps, inner_sweeps;
    int cross_steps;                // steps t > 0 rotate only the cross column pairs
    int epoch;                      // > every value already in done[] (the sweep number + 1)
    cplx* X[2][kBjMaxProblems];     // step t reads X[t & 1], writes X[(t + 1) & 1]
    cplx* V[2][kBjMaxProblems];
    BjStat* stat[kBjMaxProblems];
    const int* dst;                 // device [nsteps][2 npairs]: slot at step t -> slot at step t+1
    const int* prod;                // device [nsteps][2 npairs]: pair of step t-1 that wrote slot (row t)
    int* done;                      // device [count][nsteps][npairs]: epoch of the item's completion
    int* counter;                   // device work counter, zero at launch
};
cudaError_t bj_sweep(const BjSweep& a, cudaStream_t s);

struct BjFinish {
    int count, r, c, cp, b;
    const cplx* X[kBjMaxProblems];
    const cplx* V[kBjMaxProblems];
    double* sigma[kBjMaxProblems];  // c, non-increasing
    cplx* Xn[kBjMaxProblems];       // nullable: r x c row-major, X columns / sigma (sorted)
    cplx* Js[kBjMaxProblems];       // nullable: c x c row-major, V columns (sorted)
    int place[kBjMaxSlots];         // block id at each block position (final placement)
    double* sig_ws;                 // device scratch: count x cp column norms
    int* rank_ws;                   // device scratch: count x cp output rank per slot (-1 = padding)
};
cudaError_t bj_finish(const BjFinish& a, cudaStream_t s);

}  // namespace rb

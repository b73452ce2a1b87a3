// smallla.cu — batched small dense kernels: Cholesky + inverse, cluster Jacobi SVD,
// deterministic reductions.  See smallla.cuh.
#include <algorithm>
#include <cooperative_groups.h>

#include "smallla.cuh"

namespace cg = cooperative_groups;

namespace rb {

namespace {

constexpr double kU = 1.1102230246251565e-16;  // unit roundoff 2^-53
constexpr double kEps = 2.220446049250313e-16;  // 2^-52

// ============================================================================ Cholesky + inverse
constexpr int CHOL_THREADS = 256;
constexpr int NB = 8;  // panel width = the DMMA tile edge

// G (L x L, L = l rounded up to 8) lives unpacked in shared memory with ld = L + 2: ld = 2 (mod 8)
// makes the 8 x 4 / 4 x 8 complex fragment loads of mma.m8n8k4 conflict-free.
__host__ __device__ constexpr int chol_ld(int L) { return L + 2; }
size_t chol_smem_bytes(int max_l) {
    const int L = (max_l + 7) & ~7;
    return (size_t)(L + NB) * chol_ld(L) * sizeof(cplx) + (size_t)L * (2 * sizeof(double) + sizeof(int));
}

// acc -= conj(a) * b
__device__ __forceinline__ void cfnmac(cplx& acc, cplx a, cplx b) {
    acc.x = fma(-a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(-a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

// One CTA per problem.  Shifted Cholesky G + sI = R^H R (R upper) and T = R^-1, in place.
//  * panels of NB = 8 rows: warp 0 factors the 8 x 8 diagonal block (lanes redundantly, no
//    barrier per pivot); one thread per column forward-solves the panel's off-diagonal rows;
//    the rank-8 trailing update G_>J,>J -= R_J,>J^H R_J,>J runs on the FP64 tensor core as
//    8 x 8 tiles of the upper triangle (mma.m8n8k4, 4M complex form).
//  * the inverse bottom-up by block rows: S = R_I,>I T_>I,k as DMMA tiles (T_qk = 0 for q > k
//    bounds each tile's K), then per column the 8-step in-block recurrence
//    T_ik = -T_ii (S_ik + sum_{u in block, u > i} R_iu T_uk), T_ii = 1 / R_ii.
// The strictly lower triangle of the buffer stays zero throughout (T is read as a full tile).
// A dependent (dead) pivot gets R_ii = 0 and T_i: = 0.  ill_out: some pivot within kIllRatio of
// the shift (or dead).
__global__ void __launch_bounds__(CHOL_THREADS, 1) chol_inv_kernel(const __grid_constant__ CholBatch b) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int p = blockIdx.x;
    if (b.pred[p] != nullptr && *b.pred[p] == 0) return;
    const int l = b.l[p];
    const int L = (l + 7) & ~7, ld = chol_ld(L);
    cplx* P = reinterpret_cast<cplx*>(sm);        // [L][ld]: G -> R (upper) -> T
    cplx* sS = P + (size_t)L * ld;                // [NB][ld]: the inverse's block-row sums
    double* g0 = reinterpret_cast<double*>(sS + (size_t)NB * ld);
    double* rinv = g0 + L;                        // 1 / R_ii (0 for a dead pivot)
    int* dead = reinterpret_cast<int*>(rinv + L);
    // upper-triangle tiles (ti <= tk) of the L/8 x L/8 tile grid ordered by ti DESCENDING: the
    // trailing tiles of panel J (ti, tk > J) are then a prefix of the table
    constexpr int kMaxTiles = (kMaxCholL / NB) * (kMaxCholL / NB + 1) / 2;
    __shared__ unsigned short s_tile[kMaxTiles];
    __shared__ double s_shift;
    __shared__ int s_ill;
    __shared__ cplx sD[NB * NB];
    __shared__ double sinv[NB];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = CHOL_THREADS / 32;
    const cplx* G = b.G[p];
    const long long ldg = b.ldg[p] > 0 ? b.ldg[p] : l;
    const cplx* Gs = b.Gsub[p];

    if (tid == 0) s_ill = 0;
    if (warp == 0) {  // shift from the trace of the whole Gram matrix (also for a trailing block)
        if (b.shift_use[p] != nullptr) {
            if (lane == 0) s_shift = *b.shift_use[p];
        } else {
            const cplx* ts = b.trace_src[p] ? b.trace_src[p] : G;
            const int tn = b.trace_src[p] ? b.trace_n[p] : l;
            const long long tld = (b.trace_src[p] ? (long long)b.trace_ld[p] : ldg) + 1;
            double tr = 0.0;
            for (int i = lane; i < tn; i += 32) tr += ts[i * tld].x;
            tr = warp_sum(tr);
            if (lane == 0) {
                s_shift = b.shift_scale[p] * kU * tr;
                if (b.shift_save[p] != nullptr) *b.shift_save[p] = s_shift;
            }
        }
    }
    __syncthreads();
    {
        const int n8 = L / NB;
        for (int tt = tid; tt < n8 * (n8 + 1) / 2; tt += CHOL_THREADS) {
            int ti = n8 - 1, rem = tt;  // rows of the grid from the bottom: row ti has n8 - ti tiles
            while (rem >= n8 - ti) { rem -= n8 - ti; --ti; }
            s_tile[tt] = (unsigned short)(ti << 8 | (ti + rem));
        }
    }
    // fill: the upper triangle of G (+ shift on the diagonal, - Gsub), zeros elsewhere; a warp per
    // pair of rows, eight independent loads in flight per lane
    for (int i2 = 2 * warp; i2 < L; i2 += 2 * nw) {
        cplx v[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i2 + h, k = lane + 32 * u;
                v[h][u] = (i < l && k < l && k >= i) ? G[(long long)i * ldg + k] : mk(0.0, 0.0);
            }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i2 + h, k = lane + 32 * u;
                if (i >= L || k >= L) continue;
                cplx x = v[h][u];
                if (i < l && k < l && k >= i) {
                    if (k == i) {
                        x = mk(x.x + s_shift, 0.0);
                        g0[i] = x.x;  // dependence is judged against the pivot's original diagonal
                    }
                    if (Gs != nullptr) {
                        const cplx w = Gs[(long long)i * l + k];
                        x.x -= w.x;
                        x.y -= (k == i) ? 0.0 : w.y;
                    }
                }
                P[(size_t)i * ld + k] = x;
            }
    }
    __syncthreads();

    // ---- right-looking Cholesky by panels of NB rows, with look-ahead: warp 0 updates the next
    // panel's diagonal tile first and factors it while the other warps finish the trailing update
    const double dtol = b.dep_tol[p];
    auto factor_diag = [&](int j0) {  // warp 0: the 8 x 8 diagonal block at j0 (lanes redundantly)
        const int nb = min(NB, l - j0);
        cplx D[NB][NB];
        double inv[NB];
        unsigned deadmask = 0;
#pragma unroll
        for (int t = 0; t < NB; ++t)
#pragma unroll
            for (int u = t; u < NB; ++u) D[t][u] = (u < nb) ? P[(size_t)(j0 + t) * ld + j0 + u] : mk(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < NB; ++t) {
            inv[t] = 0.0;
            if (t < nb) {
                const double d = D[t][t].x, g = g0[j0 + t];
                const bool isdead = !(d > dtol * g) || !(d > 0.0) || !(g > 0.0);
                if (lane == 0 && (isdead || !(d >= kIllRatio * s_shift))) s_ill = 1;
                const double r = isdead ? 0.0 : sqrt(d);
                inv[t] = isdead ? 0.0 : 1.0 / r;
                deadmask |= isdead ? (1u << t) : 0u;
                D[t][t] = mk(r, 0.0);
#pragma unroll
                for (int u = t + 1; u < NB; ++u) D[t][u] = cscale(D[t][u], inv[t]);
#pragma unroll
                for (int v = t + 1; v < NB; ++v)
#pragma unroll
                    for (int u = v; u < NB; ++u) cfnmac(D[v][u], D[t][v], D[t][u]);
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < NB; ++t) {
                sinv[t] = inv[t];
#pragma unroll
                for (int u = t; u < NB; ++u) sD[t * NB + u] = D[t][u];
                if (t < nb) {
                    dead[j0 + t] = (deadmask >> t) & 1u;
                    rinv[j0 + t] = inv[t];
                }
            }
        }
    };
    auto update_tile = [&](int code, int j0) {  // G tile -= R_J,tile-rows^H R_J,tile-cols on DMMA
        const int r0 = (code >> 8) * NB, c0 = (code & 255) * NB;
        cplx* Cp = P + (size_t)(r0 + (lane >> 2)) * ld + c0 + 2 * (lane & 3);
        double cre[2] = {Cp[0].x, Cp[1].x}, cim[2] = {Cp[0].y, Cp[1].y};
        double dre[2] = {0.0, 0.0}, dim[2] = {0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const cplx* Rrow = P + (size_t)(j0 + 4 * ks + (lane & 3)) * ld;
            const cplx a = Rrow[r0 + (lane >> 2)], bb = Rrow[c0 + (lane >> 2)];
            // C -= conj(A)^T B:  Re -= ar br + ai bi,  Im -= ar bi - ai br
            dmma884(cre[0], cre[1], -a.x, bb.x);
            dmma884(dre[0], dre[1], -a.y, bb.y);
            dmma884(cim[0], cim[1], -a.x, bb.y);
            dmma884(dim[0], dim[1], a.y, bb.x);
        }
        const int row = r0 + (lane >> 2);
#pragma unroll
        for (int c = 0; c < 2; ++c)
            if (c0 + 2 * (lane & 3) + c >= row) Cp[c] = mk(cre[c] + dre[c], cim[c] + dim[c]);
    };
    if (warp == 0) factor_diag(0);
    __syncthreads();
    for (int j0 = 0; j0 < l; j0 += NB) {
        const int nb = min(NB, l - j0);
        // panel: R[J][k] = R_JJ^-H G[J][k], one column per thread
        for (int k = j0 + nb + tid; k < l; k += CHOL_THREADS) {
            cplx D[NB][NB];
            double inv[NB];
#pragma unroll
            for (int t = 0; t < NB; ++t) {
                inv[t] = sinv[t];
#pragma unroll
                for (int u = t; u < NB; ++u) D[t][u] = sD[t * NB + u];
            }
            cplx X[NB];
#pragma unroll
            for (int t = 0; t < NB; ++t) X[t] = (t < nb) ? P[(size_t)(j0 + t) * ld + k] : mk(0.0, 0.0);
#pragma unroll
            for (int t = 0; t < NB; ++t) {
#pragma unroll
                for (int v = 0; v < t; ++v) cfnmac(X[t], D[v][t], X[v]);
                X[t] = cscale(X[t], inv[t]);
            }
#pragma unroll
            for (int t = 0; t < NB; ++t)
                if (t < nb) P[(size_t)(j0 + t) * ld + k] = X[t];
        }
        if (tid == 0) {
#pragma unroll
            for (int t = 0; t < NB; ++t)
#pragma unroll
                for (int u = t; u < NB; ++u)
                    if (u < nb) P[(size_t)(j0 + t) * ld + j0 + u] = sD[t * NB + u];
        }
        __syncthreads();
        if (nb == NB) {  // trailing update on DMMA (a partial panel is the last: nothing trails it)
            const int t0 = j0 / NB + 1, nt = L / NB - t0;
            const int ntiles = nt * (nt + 1) / 2;
            const int j1 = j0 + NB;
            if (j1 < l) {
                // look-ahead: warp 0 takes the next diagonal tile and factors it; warps 1.. the rest
                const int dcode = t0 << 8 | t0;
                if (warp == 0) {
                    update_tile(dcode, j0);
                    __syncwarp();
                    factor_diag(j1);
                } else {
                    for (int tt = warp - 1; tt < ntiles; tt += nw - 1)
                        if (s_tile[tt] != dcode) update_tile(s_tile[tt], j0);
                }
            } else {
                for (int tt = warp; tt < ntiles; tt += nw) update_tile(s_tile[tt], j0);
            }
        }
        __syncthreads();
    }

    // ---- in-place inverse, bottom-up by block rows
    for (int i0 = (l - 1) / NB * NB; i0 >= 0; i0 -= NB) {
        const int nb = min(NB, l - i0);
        const int kt0 = i0 / NB + 1, nkt = L / NB - kt0;
        for (int tt = warp; tt < nkt; tt += nw) {  // S[:, tile] = R[I][q > I] T[q][tile]
            const int c0 = (kt0 + tt) * NB;
            double sre[2] = {0.0, 0.0}, sim[2] = {0.0, 0.0}, ure[2] = {0.0, 0.0}, uim[2] = {0.0, 0.0};
            const cplx* Arow = P + (size_t)(i0 + (lane >> 2)) * ld + (lane & 3);
            const cplx* Bcol = P + (size_t)(lane & 3) * ld + c0 + (lane >> 2);
            for (int q0 = i0 + NB; q0 < c0 + NB; q0 += 4) {
                const cplx a = Arow[q0], bb = Bcol[(size_t)q0 * ld];
                dmma884(sre[0], sre[1], a.x, bb.x);
                dmma884(ure[0], ure[1], -a.y, bb.y);
                dmma884(sim[0], sim[1], a.x, bb.y);
                dmma884(uim[0], uim[1], a.y, bb.x);
            }
            cplx* Sp = sS + (size_t)(lane >> 2) * ld + c0 + 2 * (lane & 3);
            Sp[0] = mk(sre[0] + ure[0], sim[0] + uim[0]);
            Sp[1] = mk(sre[1] + ure[1], sim[1] + uim[1]);
        }
        __syncthreads();
        double tii[NB];
#pragma unroll
        for (int t = 0; t < NB; ++t)
            tii[t] = t < nb ? rinv[i0 + t] : 0.0;  // (= 1 / R_ii as the factorization formed it; 0 if dead)
        const int k = i0 + tid;
        cplx res[NB];
        if (k < l) {
#pragma unroll
            for (int t = NB - 1; t >= 0; --t) {
                res[t] = mk(0.0, 0.0);
                if (t >= nb || i0 + t > k) continue;
                cplx acc = k >= i0 + NB ? sS[(size_t)t * ld + k] : mk(0.0, 0.0);
#pragma unroll
                for (int u = t + 1; u < NB; ++u)
                    if (u < nb && i0 + u <= k) cfma(acc, P[(size_t)(i0 + t) * ld + i0 + u], res[u]);
                res[t] = (i0 + t == k) ? mk(tii[t], 0.0) : cscale(acc, -tii[t]);
            }
        }
        __syncthreads();  // every read of the block's R rows precedes the writes
        if (k < l) {
#pragma unroll
            for (int t = 0; t < NB; ++t)
                if (t < nb && i0 + t <= k) P[(size_t)(i0 + t) * ld + k] = res[t];
        }
        __syncthreads();
    }

    cplx* T = b.T[p];
    cplx* Tn = b.Tneg[p];
    const long long ldt = b.ldt[p] > 0 ? b.ldt[p] : l;
    for (int i = warp; i < l; i += nw) {  // (the lower triangle of the buffer is zero)
        const cplx* src = P + (size_t)i * ld;
        cplx* dt = T + (long long)i * ldt;
        cplx* dn = Tn != nullptr ? Tn + (long long)i * ldt : nullptr;
        for (int k = lane; k < l; k += 32) {
            const cplx v = src[k];
            dt[k] = v;
            if (dn != nullptr) dn[k] = mk(-v.x, -v.y);
        }
    }
    if (b.ill_out[p] != nullptr && tid == 0 && s_ill) *b.ill_out[p] = 1;  // (zeroed by the caller)
    if (b.ndead[p] != nullptr && tid == 0) {
        int n = 0;
        for (int j = 0; j < l; ++j) n += dead[j];
        if (b.ndead_acc[p]) *b.ndead[p] += n;
        else *b.ndead[p] = n;
    }
}

// ============================================================================ Jacobi SVD
constexpr int JAC_CL_THREADS = 512;   // cluster kernel: up to 16 column pairs per round
constexpr int kMaxPairsPerRound = JAC_CL_THREADS / 32;
constexpr int kMaxSweeps = 60;

__device__ __forceinline__ int circle(int i, int t, int n) {  // round-robin slot -> player
    return i == 0 ? 0 : ((i - 1 + t) % (n - 1)) + 1;
}

// One Hestenes rotation of columns xp, xq (r data rows, ld rows in all: the trailing c rows
// accumulate the right vectors), executed by one warp.  Returns whether it rotated.
//   a = |xp|^2, b = |xq|^2, g = xp^H xq;  rotate iff |g| > tol sqrt(a b)
//   e = conj(g)/|g|, zeta = (b - a)/(2|g|), t = sign(zeta)/(|zeta| + sqrt(1 + zeta^2)),
//   c = 1/sqrt(1 + t^2), s = c t:   xp' = c xp - s e xq,  xq' = s xp + c e xq.
// The parameters use rsqrt/rcp (a few ulps): the rotation only has to be unitary to working
// precision, the convergence test is exact.
__device__ __forceinline__ bool hestenes_rotate(cplx* __restrict__ xp, cplx* __restrict__ xq, int r, int ld,
                                                int lane, double tol, double& off2) {
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
    cplx g0 = mk(0.0, 0.0), g1 = mk(0.0, 0.0);
    int rr = lane;
    for (; rr + 32 < r; rr += 64) {  // two independent accumulator sets
        const cplx u = xp[rr], v = xq[rr], u1 = xp[rr + 32], v1 = xq[rr + 32];
        a0 += cabs2(u); b0 += cabs2(v); cfmac(g0, u, v);
        a1 += cabs2(u1); b1 += cabs2(v1); cfmac(g1, u1, v1);
    }
    if (rr < r) {
        const cplx u = xp[rr], v = xq[rr];
        a0 += cabs2(u); b0 += cabs2(v); cfmac(g0, u, v);
    }
    double a = a0 + a1, bb = b0 + b1;
    cplx g = mk(g0.x + g1.x, g0.y + g1.y);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        bb += __shfl_xor_sync(0xffffffffu, bb, o);
        g.x += __shfl_xor_sync(0xffffffffu, g.x, o);
        g.y += __shfl_xor_sync(0xffffffffu, g.y, o);
    }
    const double g2 = g.x * g.x + g.y * g.y;
    if (!(a > 0.0) || !(bb > 0.0) || !(g2 > tol * tol * a * bb)) return false;
    off2 = fmax(off2, g2 / (a * bb));
    const double rg = rsqrt(g2);  // 1/|g|
    const cplx e = mk(g.x * rg, -g.y * rg);
    const double zeta = 0.5 * (bb - a) * rg;
    const double az = fabs(zeta);
    const double h = az > 1e150 ? az : sqrt(fma(zeta, zeta, 1.0));
    const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (az + h);
    const double cc = rsqrt(fma(tt, tt, 1.0));
    const double ss = cc * tt;
#pragma unroll 4
    for (int k = lane; k < ld; k += 32) {
        const cplx u = xp[k];
        const cplx ev = cmul(e, xq[k]);
        xp[k] = mk(cc * u.x - ss * ev.x, cc * u.y - ss * ev.y);
        xq[k] = mk(ss * u.x + cc * ev.x, ss * u.y + cc * ev.y);
    }
    return true;
}

// Block one-sided Jacobi on a thread-block cluster.  The c columns form 2*cs blocks of bs; CTA k
// holds two blocks per step (a round-robin tournament over blocks, nblk - 1 steps per sweep, data
// through L2).  Per step a CTA rotates the bs^2 CROSS pairs of its two blocks in bs rounds of bs
// disjoint pairs (one warp each); the pairs inside a block are rotated once per sweep, in step 0
// (where every block is resident exactly once).  Every column pair is visited once per sweep.
__global__ void __launch_bounds__(JAC_CL_THREADS) jacobi_kernel(const __grid_constant__ JacobiBatch b) {
    extern __shared__ __align__(16) unsigned char sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int cs = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int p = blockIdx.x / cs;
    const int r = b.r[p], c = b.c[p], ld = r + c;
    const int nblk = 2 * cs;
    const int bs = (c + nblk - 1) / nblk;
    cplx* col = reinterpret_cast<cplx*>(sm);  // [2bs][ld]: block A columns, then block B
    __shared__ int cnt[2];
    __shared__ unsigned long long offm[2];  // max rotated |g|^2/(a b) of the sweep (ordered bits)
    __shared__ int s_rot;
    cplx* W = b.W[p];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double tol = sqrt((double)max(r, 1)) * kEps;
    if (tid == 0) { cnt[0] = cnt[1] = 0; offm[0] = offm[1] = 0ull; }
    cluster.sync();
    // noise level (LAPACK zgesvj's test, as the block Jacobi): a sweep whose every rotated pair
    // had |g| <= sqrt(c) tol sqrt(a b) leaves only rounding noise, and another sweep would only
    // rotate noise again
    const double noise2 = (double)c * tol * tol;

    int sweep = 0;
    for (; sweep < kMaxSweeps; ++sweep) {
        int myrot = 0;
        double myoff2 = 0.0;
        for (int t = 0; t < nblk - 1; ++t) {
            const int blkA = circle(rank, t, nblk), blkB = circle(nblk - 1 - rank, t, nblk);
            auto gcol = [&](int lc) { return lc < bs ? blkA * bs + lc : blkB * bs + (lc - bs); };
            for (int lc = 0; lc < 2 * bs; ++lc) {
                const int g = gcol(lc);
                if (g >= c) continue;
                const cplx* src = W + (long long)g * ld;
                for (int rr = tid; rr < ld; rr += JAC_CL_THREADS) cp_async16(col + lc * ld + rr, src + rr, true);
            }
            cp_async_commit();
            cp_async_wait<0>();
            if (tid == 0) s_rot = 0;
            __syncthreads();
            if (t == 0) {  // pairs inside each block, round-robin over its bs columns
                const int bp = bs + (bs & 1);
                for (int ir = 0; ir < bp - 1; ++ir) {
                    const int half = bp / 2;
                    if (warp < 2 * half) {
                        const int blk = warp / half, k = warp % half;
                        const int lp = circle(k, ir, bp), lq = circle(bp - 1 - k, ir, bp);
                        if (lp < bs && lq < bs && gcol(blk * bs + lp) < c && gcol(blk * bs + lq) < c)
                            myrot += hestenes_rotate(col + (blk * bs + lp) * ld, col + (blk * bs + lq) * ld, r, ld,
                                                     lane, tol, myoff2);
                    }
                    __syncthreads();
                }
            }
            for (int j = 0; j < bs; ++j) {  // cross pairs (A[i], B[(i + j) mod bs])
                if (warp < bs) {
                    const int lp = warp, lq = bs + (warp + j) % bs;
                    if (gcol(lp) < c && gcol(lq) < c)
                        myrot += hestenes_rotate(col + lp * ld, col + lq * ld, r, ld, lane, tol, myoff2);
                }
                __syncthreads();
            }
            if (lane == 0 && myrot) {
                atomicAdd(&s_rot, myrot);
                atomicMax(&offm[sweep & 1], (unsigned long long)__double_as_longlong(myoff2));
            }
            myrot = 0;
            myoff2 = 0.0;
            __syncthreads();
            if (tid == 0) cnt[sweep & 1] += s_rot;
            for (int lc = 0; lc < 2 * bs; ++lc) {
                const int g = gcol(lc);
                if (g >= c) continue;
                cplx* dst = W + (long long)g * ld;
                for (int rr = tid; rr < ld; rr += JAC_CL_THREADS) dst[rr] = col[lc * ld + rr];
            }
            __threadfence();
            cluster.sync();
            // every peer is past its end-of-previous-sweep read of our counters: recycle the slot
            if (t == 0 && tid == 0) { cnt[(sweep + 1) & 1] = 0; offm[(sweep + 1) & 1] = 0ull; }
        }
        // convergence: sum of all CTAs' rotation counts of this sweep (read through DSMEM)
        int total = 0;
        double worst2 = 0.0;
        for (int q = 0; q < cs; ++q) {
            const int* peer = cluster.map_shared_rank(cnt, q);
            const unsigned long long* poff = cluster.map_shared_rank(offm, q);
            total += peer[sweep & 1];
            worst2 = fmax(worst2, __longlong_as_double((long long)poff[sweep & 1]));
        }
        if (total == 0 || worst2 <= noise2) break;
    }
    cluster.sync();  // peers may still read our counters
    if (rank == 0 && tid == 0 && b.sweeps[p] != nullptr) *b.sweeps[p] = sweep + 1;
}

constexpr int kColPermThreads = 512;
__global__ void __launch_bounds__(kColPermThreads) colperm_rank_kernel(const __grid_constant__ ColPermBatch b) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int p = blockIdx.x, r = b.r[p], c = b.c[p];
    double* nrm = reinterpret_cast<double*>(sm);
    __shared__ double part[kColPermThreads];
    const cplx* X = b.X[p];
    // column norms: cpp consecutive columns per pass (coalesced rows), tpc threads per column over
    // interleaved rows, two accumulators each; partials summed in a fixed order (deterministic)
    const int cpp = min(c, kColPermThreads), tpc = kColPermThreads / cpp;
    const int jl = threadIdx.x % cpp, q = threadIdx.x / cpp;
    for (int j0 = 0; j0 < c; j0 += cpp) {
        const int j = j0 + jl;
        double a0 = 0.0, a1 = 0.0;
        if (q < tpc && j < c) {
            int i = q;
            for (; i + tpc < r; i += 2 * tpc) {
                a0 += cabs2(X[(long long)i * c + j]);
                a1 += cabs2(X[(long long)(i + tpc) * c + j]);
            }
            if (i < r) a0 += cabs2(X[(long long)i * c + j]);
        }
        part[threadIdx.x] = a0 + a1;
        __syncthreads();
        if (q == 0 && j < c) {
            double a = 0.0;
            for (int t = 0; t < tpc; ++t) a += part[t * cpp + jl];
            nrm[j] = a;
        }
        __syncthreads();
    }
    for (int j = threadIdx.x; j < c; j += kColPermThreads) {
        const double v = rank_key(nrm[j]);
        int rk = 0;
        for (int t = 0; t < c; ++t) rk += (rank_key(nrm[t]) > v) || (rank_key(nrm[t]) == v && t < j);
        b.perm[p][rk] = j;
    }
}

__global__ void __launch_bounds__(256) colperm_gather_kernel(const __grid_constant__ ColPermBatch b) {
    const int p = blockIdx.y, c = b.c[p];
    const long long n = (long long)b.r[p] * c;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < n; e += (long long)gridDim.x * 256) {
        const long long i = e / c;
        const int k = (int)(e % c);
        b.Xp[p][e] = b.X[p][i * c + b.perm[p][k]];
    }
}

__global__ void __launch_bounds__(256) colperm_scatter_kernel(const __grid_constant__ ColPermBatch b) {
    const int p = blockIdx.y, c = b.c[p];
    const long long n = (long long)c * c;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < n; e += (long long)gridDim.x * 256) {
        const int k = (int)(e / c), j = (int)(e % c);
        b.V[p][(long long)b.perm[p][k] * c + j] = b.Vp[p][e];
    }
}

__global__ void __launch_bounds__(256) select_kernel(const __grid_constant__ SelectBatch b) {
    const int p = blockIdx.y;
    const cplx* src = *b.flag[p] ? b.B[p] : b.A[p];
    cplx* dst = b.Q[p];
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < b.n[p]; e += (long long)gridDim.x * 256)
        dst[e] = src[e];
}

__global__ void __launch_bounds__(256) colnorm_max_kernel(const __grid_constant__ ColNormBatch b) {
    const int p = blockIdx.x;
    const int m = b.m[p], r = b.r[p];
    const cplx* D = b.D[p];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double wmax[8];
    double mx = 0.0;
    for (int j = warp; j < r; j += 8) {
        double a = 0.0;
        for (int i = lane; i < m; i += 32) a += cabs2(D[(long long)i * r + j]);
        a = warp_sum(a);
        mx = fmax(mx, sqrt(a));
    }
    if (lane == 0) wmax[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < 8; ++w) v = fmax(v, wmax[w]);
        *b.out[p] = v;
    }
}

__global__ void jacobi_init_kernel(const __grid_constant__ JacobiInitBatch b) {
    const int p = blockIdx.y;
    const int r = b.r[p], c = b.c[p], ld = r + c;
    const long long total = (long long)c * ld;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int cc = (int)(e / ld), rr = (int)(e % ld);
        cplx v;
        if (rr < r) {
            v = b.adj[p] ? cconj(b.A[p][(long long)cc * b.lda[p] + rr]) : b.A[p][(long long)rr * b.lda[p] + cc];
        } else {
            v = mk((rr - r) == cc ? 1.0 : 0.0, 0.0);
        }
        b.W[p][e] = v;
    }
}

__global__ void __launch_bounds__(256) jacobi_finish_kernel(const __grid_constant__ JacobiFinBatch b) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int p = blockIdx.x;
    const int r = b.r[p], c = b.c[p], ld = r + c;
    double* sig = reinterpret_cast<double*>(sm);
    int* pos = reinterpret_cast<int*>(sig + c);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x / 32;
    const cplx* W = b.W[p];
    for (int j = warp; j < c; j += nw) {
        double a = 0.0;
        for (int rr = lane; rr < r; rr += 32) a += cabs2(W[(long long)j * ld + rr]);
        a = warp_sum(a);
        if (lane == 0) sig[j] = sqrt(a);
    }
    __syncthreads();
    for (int j = tid; j < c; j += blockDim.x) {
        int rk = 0;
        const double sj = rank_key(sig[j]);
        for (int i = 0; i < c; ++i) rk += (rank_key(sig[i]) > sj) || (rank_key(sig[i]) == sj && i < j);
        pos[j] = rk;
    }
    __syncthreads();
    if (b.sigma[p])
        for (int j = tid; j < c; j += blockDim.x) b.sigma[p][pos[j]] = sig[j];
    if (b.Xn[p]) {
        cplx* Xn = b.Xn[p];
        for (int j = warp; j < c; j += nw) {
            const double inv = sig[j] > 0.0 ? 1.0 / sig[j] : 0.0;
            const int pj = pos[j];
            for (int rr = lane; rr < r; rr += 32) Xn[(long long)rr * c + pj] = cscale(W[(long long)j * ld + rr], inv);
        }
    }
    if (b.Js[p]) {
        cplx* Js = b.Js[p];
        for (int j = warp; j < c; j += nw) {
            const int pj = pos[j];
            for (int i = lane; i < c; i += 32) Js[(long long)i * c + pj] = W[(long long)j * ld + r + i];
        }
    }
}

// ============================================================================ reductions
constexpr int RED_BLOCKS = 2 * kNumSMs, RED_THREADS = 256;

__global__ void __launch_bounds__(RED_THREADS) sumsq_partial(const cplx* __restrict__ a, long long n,
                                                             double* partial, int* bad) {
    double s = 0.0;
    int nb = 0;
    for (long long i = blockIdx.x * (long long)RED_THREADS + threadIdx.x; i < n;
         i += (long long)RED_BLOCKS * RED_THREADS) {
        const cplx v = a[i];
        nb += !(isfinite(v.x) && isfinite(v.y));
        s += cabs2(v);
    }
    __shared__ double ss[RED_THREADS / 32];
    __shared__ int sb[RED_THREADS / 32];
    s = warp_sum(s);
    for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if ((threadIdx.x & 31) == 0) { ss[threadIdx.x >> 5] = s; sb[threadIdx.x >> 5] = nb; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        int tb = 0;
        for (int w = 0; w < RED_THREADS / 32; ++w) { t += ss[w]; tb += sb[w]; }
        partial[blockIdx.x] = t;
        bad[blockIdx.x] = tb;
    }
}

__global__ void __launch_bounds__(RED_THREADS) sumsq_partial_many(const __grid_constant__ SumsqBatch b,
                                                                  double* partial, int* bad) {
    const int p = blockIdx.y;
    const cplx* __restrict__ a = b.a[p];
    const long long n = b.n[p];
    double s = 0.0;
    int nb = 0;
    for (long long i = blockIdx.x * (long long)RED_THREADS + threadIdx.x; i < n;
         i += (long long)gridDim.x * RED_THREADS) {
        const cplx v = a[i];
        nb += !(isfinite(v.x) && isfinite(v.y));
        s += cabs2(v);
    }
    __shared__ double ss[RED_THREADS / 32];
    __shared__ int sb[RED_THREADS / 32];
    s = warp_sum(s);
    for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if ((threadIdx.x & 31) == 0) { ss[threadIdx.x >> 5] = s; sb[threadIdx.x >> 5] = nb; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        int tb = 0;
        for (int w = 0; w < RED_THREADS / 32; ++w) { t += ss[w]; tb += sb[w]; }
        partial[p * gridDim.x + blockIdx.x] = t;
        bad[p * gridDim.x + blockIdx.x] = tb;
    }
}

__global__ void sumsq_final_many(const __grid_constant__ SumsqBatch b, const double* partial, const int* bad,
                                 int nblocks) {
    if (threadIdx.x != 0) return;
    const int p = blockIdx.x;
    double t = 0.0;
    int tb = 0;
    for (int i = 0; i < nblocks; ++i) { t += partial[p * nblocks + i]; tb += bad[p * nblocks + i]; }
    *b.out_sq[p] = t;
    if (b.out_bad[p]) *b.out_bad[p] = tb;
}

__global__ void sumsq_final(const double* partial, const int* bad, double* out, int* nonfinite) {
    if (threadIdx.x == 0) {
        double t = 0.0;
        int tb = 0;
        for (int i = 0; i < RED_BLOCKS; ++i) { t += partial[i]; tb += bad[i]; }
        *out = t;
        if (nonfinite) *nonfinite = tb;
    }
}

}  // namespace

cudaError_t chol_inv(const CholBatch& b, int max_l, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    if (max_l > kMaxCholL) return cudaErrorInvalidValue;
    const size_t smem = chol_smem_bytes(max_l);
    cudaError_t e = smem_atleast(reinterpret_cast<const void*>(chol_inv_kernel), smem);
    if (e != cudaSuccess) return e;
    chol_inv_kernel<<<b.count, CHOL_THREADS, smem, s>>>(b);
    return cudaGetLastError();
}

cudaError_t colperm_sort_gather(const ColPermBatch& b, int max_c, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    const size_t smem = (size_t)max_c * sizeof(double);
    cudaError_t e = smem_atleast(reinterpret_cast<const void*>(colperm_rank_kernel), smem);
    if (e != cudaSuccess) return e;
    colperm_rank_kernel<<<b.count, kColPermThreads, smem, s>>>(b);
    colperm_gather_kernel<<<dim3(2 * kNumSMs, b.count), 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t colperm_scatter_rows(const ColPermBatch& b, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    colperm_scatter_kernel<<<dim3(kNumSMs, b.count), 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t select_many(const SelectBatch& b, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    select_kernel<<<dim3(64, b.count), 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t colnorm_max_many(const ColNormBatch& b, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    colnorm_max_kernel<<<b.count, 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t jacobi_init(const JacobiInitBatch& b, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    jacobi_init_kernel<<<dim3(64, b.count), 256, 0, s>>>(b);
    return cudaGetLastError();
}

// Chooses the cluster size (8 portable, else 16 non-portable) so that a CTA's block pair fits
// in shared memory; returns cudaErrorInvalidValue if even 16 CTAs cannot hold it.
namespace {
constexpr size_t kJacBudget = 200 * 1024;
size_t jacobi_need(int r, int c, int csz) {
    const int bs = (c + 2 * csz - 1) / (2 * csz);
    return (size_t)2 * bs * (r + c) * sizeof(cplx);
}
// smallest cluster whose two blocks fit the shared-memory budget with at most one pair per
// warp per round; 0 if none (16 CTAs is the non-portable maximum)
int jacobi_cluster(int r, int c) {
    for (int csz = 1; csz <= 16; csz *= 2) {
        const int bs = (c + 2 * csz - 1) / (2 * csz);
        if (bs <= kMaxPairsPerRound && jacobi_need(r, c, csz) <= kJacBudget) return csz;
    }
    return 0;
}
}  // namespace

bool jacobi_fits(int r, int c) { return jacobi_cluster(r, c) > 0; }

cudaError_t jacobi_svd(const JacobiBatch& b, int max_r, int max_c, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    const int cs = jacobi_cluster(max_r, max_c);
    if (cs == 0) return cudaErrorInvalidValue;
    const size_t smem = jacobi_need(max_r, max_c, cs);
    cudaError_t e = smem_atleast(reinterpret_cast<const void*>(jacobi_kernel), smem);
    if (e != cudaSuccess) return e;
    if (cs > 8) {
        e = cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * b.count);
    cfg.blockDim = dim3(JAC_CL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, jacobi_kernel, b);
}

cudaError_t jacobi_finish(const JacobiFinBatch& b, int max_c, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    const size_t smem = (size_t)max_c * (sizeof(double) + sizeof(int));
    jacobi_finish_kernel<<<b.count, 256, smem, s>>>(b);
    return cudaGetLastError();
}

cudaError_t sumsq_many(const SumsqBatch& b, double* partial, int* partial_bad, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    // fixed per-problem block count: deterministic order, independent of the batch size
    sumsq_partial_many<<<dim3(RED_BLOCKS, b.count), RED_THREADS, 0, s>>>(b, partial, partial_bad);
    sumsq_final_many<<<b.count, 32, 0, s>>>(b, partial, partial_bad, RED_BLOCKS);
    return cudaGetLastError();
}

cudaError_t sumsq(const cplx* a, long long n, double* partial, int* partial_bad, double* out_sq,
                  int* out_nonfinite, cudaStream_t s) {
    sumsq_partial<<<RED_BLOCKS, RED_THREADS, 0, s>>>(a, n, partial, partial_bad);
    sumsq_final<<<1, 32, 0, s>>>(partial, partial_bad, out_sq, out_nonfinite);
    return cudaGetLastError();
}

}  // namespace rb

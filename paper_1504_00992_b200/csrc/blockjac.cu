// blockjac.cu — kernels of the block one-sided Jacobi SVD (see blockjac.cuh).
#include <algorithm>
#include <cstdlib>
#include <cooperative_groups.h>

#include "blockjac.cuh"

namespace cg = cooperative_groups;

namespace rb {

namespace {

constexpr double kEpsBj = 2.220446049250313e-16;
constexpr int kBjThreads = 256;

__device__ __forceinline__ int circle_bj(int i, int t, int n) {
    return i == 0 ? 0 : ((i - 1 + t) % (n - 1)) + 1;
}

__global__ void __launch_bounds__(kBjThreads) bj_init_kernel(const __grid_constant__ BjInit a) {
    const int p = blockIdx.y;
    const long long nx = (long long)a.r * a.cp, nv = (long long)a.cp * a.cp;
    for (long long e = blockIdx.x * (long long)kBjThreads + threadIdx.x; e < nx + nv;
         e += (long long)gridDim.x * kBjThreads) {
        const bool isx = e < nx;
        const long long f = isx ? e : e - nx;
        const int i = (int)(f / a.cp), s = (int)(f % a.cp);
        const int orig = a.place[s / a.b] * a.b + s % a.b;
        if (isx) {
            cplx v = mk(0.0, 0.0);
            if (orig < a.c)
                v = a.adj[p] ? cconj(a.A[p][(long long)orig * a.lda[p] + i]) : a.A[p][(long long)i * a.lda[p] + orig];
            a.X[p][f] = v;
        } else {
            a.V[p][f] = mk(i == orig ? 1.0 : 0.0, 0.0);
        }
    }
}

constexpr int kBjRows = 32;  // rows per staged chunk (two chunk buffers, cp.async double-buffered)

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
constexpr int kBjN2 = 32;    // 2b (b = 16)

// One block pair, one CTA: Gram, one sweep of two-sided Jacobi (round-robin rounds of n2/2
// disjoint pairs: parameters from (G_pp, G_qq, G_pq) exactly as the Hestenes rotation, then the
// column update G J and W J, then the row update J^H G), then the rotated columns.
// The pair's rows are split over the S CTAs of a thread-block cluster: each CTA forms the Gram
// of its row slice, CTA 0 sums the slices over DSMEM (fixed order) and solves, the peers read W
// back over DSMEM and rotate their own slices of X and V.
// One block pair of one step (the body shared by the per-step cluster kernel and the persistent
// sweep kernel; a launch without cluster dimensions is an implicit cluster of one CTA).
struct BjPair {
    const cplx* Xs;
    const cplx* Vs;
    cplx* Xd;
    cplx* Vd;
    const int* dst;  // this step's slot -> next-step slot table
    BjStat* stat;
    int r, cp, b, inner_sweeps;
    int cross_only;  // rotate only (block i, block j) column pairs: 16 rounds instead of 31
};
// Pair k of round rd: the circle method over all 2b columns (31 rounds), or — cross_only, every
// step of a sweep but the first — column k of block i against column b + (k + rd) mod b of block
// j (16 rounds).  Each block's own column pairs are rotated at the first step of every sweep,
// where every block is in exactly one block pair, so a sweep still visits every column pair.
__device__ __forceinline__ void bj_round_pair(int k, int rd, bool cross, int& p, int& q) {
    constexpr int n2 = kBjN2, half = n2 / 2;
    if (cross) {
        p = k;
        q = half + (k + rd) % half;
    } else {
        p = circle_bj(k, rd, n2);
        q = circle_bj(n2 - 1 - k, rd, n2);
    }
}
__device__ __forceinline__ void bj_pair(const BjPair& a, const int k0) {
    constexpr int n2 = kBjN2, ld = n2 + 1, half = n2 / 2;
    __shared__ double pc[half], ps[half];
    __shared__ cplx pe[half];
    static_assert(kBjThreads == (n2 / 2) * (n2 / 2), "one thread per 2x2 block of the pair Gram");
    cg::cluster_group cluster = cg::this_cluster();
    const int S = (int)cluster.num_blocks(), crank = (int)cluster.block_rank();
    extern __shared__ __align__(16) unsigned char sm[];
    typedef cplx Chunk[kBjRows][ld];
    Chunk* buf = reinterpret_cast<Chunk*>(sm);                                    // [2] chunks
    auto sG = reinterpret_cast<cplx(*)[ld]>(sm + 2 * sizeof(Chunk));              // [n2][ld]
    auto sW = sG + n2;                                                            // [n2][ld]
    __shared__ int s_rot;
    __shared__ int s_ident;  // the pair's solve rotated nothing: W = I exactly (set by CTA 0)
    __shared__ unsigned long long s_off2, s_off2_first;
    const int tid = threadIdx.x;
    const int r = a.r, cp = a.cp, b = a.b;
    const int xr0 = (int)((long long)r * crank / S), xr1 = (int)((long long)r * (crank + 1) / S);
    const int vr0 = (int)((long long)cp * crank / S), vr1 = (int)((long long)cp * (crank + 1) / S);
    const long long col0 = (long long)k0 * n2;  // the pair's first column (slots 2k0, 2k0+1)
    const cplx* X = a.Xs;
    const cplx* V = a.Vs;
    // stage rows [r0, r0 + kBjRows) of the pair's columns of M (zero-filled from rend on)
    auto stage = [&](const cplx* M, int r0, int rend, Chunk& dst) {
#pragma unroll
        for (int u = 0; u < kBjRows * n2 / kBjThreads; ++u) {
            const int e = tid + u * kBjThreads, i = e / n2, j = e % n2;
            const bool ok = r0 + i < rend;
            cp_async16(&dst[i][j], ok ? M + (long long)(r0 + i) * cp + col0 + j : M, ok);
        }
        cp_async_commit();
    };

    // ---- Gram of this CTA's row slice on the FP64 tensor core: the 32 x 32 result is 4 x 4 tiles
    // of 8 x 8, of which the 10 upper-triangular ones are formed (the solve mirrors them); warps
    // 0..4 accumulate two tiles each.  Fragments are one LDS.128 (re, im) per lane; conj(X)^T X in
    // 4M form: Re += xr xr' + xi xi', Im += xr xi' - xi xr'.  Chunks stream through two buffers
    // (cp.async: chunk t+1 lands while chunk t is multiplied).
    const int lane = tid & 31, warp = tid >> 5;
    // upper tiles t = 0..9 as 4-bit (p | q << 2) fields: (0,0) (0,1) (0,2) (0,3) (1,1) (1,2) (1,3) (2,2) (2,3) (3,3)
    constexpr unsigned long long kTiles = 0xfead95c840ull;
    const bool gwarp = warp < 5;
    const int ta = gwarp ? 2 * warp : 0;
    const int fa = (int)(kTiles >> (4 * ta)) & 15, fb = (int)(kTiles >> (4 * ta + 4)) & 15;
    const int pa = fa & 3, qa_ = fa >> 2, pb = fb & 3, qb = fb >> 2;
    double gre[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, gim[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int ngc = (xr1 - xr0 + kBjRows - 1) / kBjRows;
    if (ngc > 0) stage(X, xr0, xr1, buf[0]);
    for (int t = 0; t < ngc; ++t) {
        if (t + 1 < ngc) {
            stage(X, xr0 + (t + 1) * kBjRows, xr1, buf[(t + 1) & 1]);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (gwarp) {
            const Chunk& ch = buf[t & 1];
#pragma unroll 2
            for (int kq = 0; kq < kBjRows; kq += 4) {
                const cplx* row = ch[kq + (lane & 3)];
                const int cl = lane >> 2;
                const cplx x0 = row[pa * 8 + cl], y0 = row[qa_ * 8 + cl];
                const cplx x1 = row[pb * 8 + cl], y1 = row[qb * 8 + cl];
                dmma884(gre[0][0], gre[0][1], x0.x, y0.x);
                dmma884(gre[1][0], gre[1][1], x1.x, y1.x);
                dmma884(gim[0][0], gim[0][1], x0.x, y0.y);
                dmma884(gim[1][0], gim[1][1], x1.x, y1.y);
                dmma884(gre[0][0], gre[0][1], x0.y, y0.y);
                dmma884(gre[1][0], gre[1][1], x1.y, y1.y);
                dmma884(gim[0][0], gim[0][1], -x0.y, y0.x);
                dmma884(gim[1][0], gim[1][1], -x1.y, y1.x);
            }
        }
        __syncthreads();  // (the buffer is refilled two chunks later)
    }
    // the first chunk of the rotation apply streams in during the solve (buffer 1: the solve
    // uses buffer 0 as its second G)
    const int nxc = (xr1 - xr0 + kBjRows - 1) / kBjRows, nvc = (vr1 - vr0 + kBjRows - 1) / kBjRows;
    auto stage_apply = [&](int t, Chunk& dst) {
        if (t < nxc) stage(X, xr0 + t * kBjRows, xr1, dst);
        else stage(V, vr0 + (t - nxc) * kBjRows, vr1, dst);
    };
    if (nxc + nvc > 0) stage_apply(0, buf[1]);
    if (gwarp) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            sG[pa * 8 + (lane >> 2)][qa_ * 8 + 2 * (lane & 3) + c] = mk(gre[0][c], gim[0][c]);
            sG[pb * 8 + (lane >> 2)][qb * 8 + 2 * (lane & 3) + c] = mk(gre[1][c], gim[1][c]);
        }
    }
    cluster.sync();
    if (crank == 0) {  // (uniform per CTA; barriers below are reached by every thread)
        // sum the slices in rank order, then keep the upper triangle and mirror it
        cplx sum[n2 * n2 / kBjThreads];
#pragma unroll
        for (int u = 0; u < n2 * n2 / kBjThreads; ++u) {
            const int e = tid + u * kBjThreads;
            sum[u] = mk(0.0, 0.0);
            if ((e >> 3) % (n2 / 8) < (e / n2) >> 3) continue;  // strictly-lower 8x8 tile: not formed
            for (int q = 0; q < S; ++q) {
                const cplx(*pg)[ld] = cluster.map_shared_rank(sG, q);
                sum[u] = cadd(sum[u], pg[e / n2][e % n2]);
            }
        }
        __syncthreads();  // every read of the partials precedes the writes below
#pragma unroll
        for (int u = 0; u < n2 * n2 / kBjThreads; ++u) {
            const int e = tid + u * kBjThreads;
            sG[e / n2][e % n2] = sum[u];
        }
        __syncthreads();
        for (int e = tid; e < n2 * n2; e += kBjThreads) {
            const int p = e / n2, q = e % n2;
            if (p > q) sG[p][q] = cconj(sG[q][p]);
            else if (p == q) sG[p][q].y = 0.0;
        }
        for (int e = tid; e < n2 * n2; e += kBjThreads) sW[e / n2][e % n2] = mk(e / n2 == e % n2 ? 1.0 : 0.0, 0.0);
        if (tid == 0) { s_rot = 0; s_off2 = 0ull; }
        __syncthreads();

    // ---- one sweep of the pair solve.  Round rd rotates the n2/2 disjoint pairs of the circle
    // method; thread (ka, kb) owns the 2 x 2 block of G at pair ka's rows x pair kb's columns and
    // forms it as J_ka^H (G J_kb) (the column rotation first, then the row rotation — the same
    // operations, in the same order, as rotating all columns and then all rows), reading G from
    // one buffer and writing the other: a round is two barriers (parameters, update) instead of
    // three.  The thread also rotates rows 2ka, 2ka+1 of W in pair kb's columns.
    const double tol = sqrt((double)max(r, 1)) * kEpsBj;
    __shared__ int s_first;  // rotations of the first inner sweep: the outer convergence signal
    cplx(*Gi)[ld] = sG;
    cplx(*Go)[ld] = buf[0];  // (chunk buffer 0 is idle during the solve)
    const int ka = tid >> 4, kb = tid & 15;
    for (int isw = 0; isw < a.inner_sweeps; ++isw) {
    const int rot_before = s_rot;
    const bool cross = a.cross_only != 0;
    const int nrounds = cross ? half : n2 - 1;
    for (int rd = 0; rd < nrounds; ++rd) {
        int p, q, p2, q2;
        bj_round_pair(ka, rd, cross, p, q);
        bj_round_pair(kb, rd, cross, p2, q2);
        if (tid < half) {  // parameters of pair tid (= ka at threads (ka, ka))
            int pp, qq;
            bj_round_pair(tid, rd, cross, pp, qq);
            const double ga = Gi[pp][pp].x, gb = Gi[qq][qq].x;
            const cplx g = Gi[pp][qq];
            const double g2 = g.x * g.x + g.y * g.y;
            double c = 1.0, s = 0.0;
            cplx e = mk(1.0, 0.0);
            if (ga > 0.0 && gb > 0.0 && g2 > tol * tol * ga * gb) {
                const double rg = rsqrt(g2);
                e = mk(g.x * rg, -g.y * rg);
                const double zeta = 0.5 * (gb - ga) * rg;
                const double az = fabs(zeta);
                const double h = az > 1e150 ? az : sqrt(fma(zeta, zeta, 1.0));
                const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (az + h);
                c = rsqrt(fma(tt, tt, 1.0));
                s = c * tt;
                atomicAdd(&s_rot, 1);
                atomicMax(&s_off2, (unsigned long long)__double_as_longlong(g2 / (ga * gb)));
            }
            pc[tid] = c; ps[tid] = s; pe[tid] = e;
        }
        __syncthreads();
        const double ca = pc[ka], sa = ps[ka], cb = pc[kb], sb = ps[kb];
        const cplx ea = pe[ka], eb = pe[kb];
        cplx g_pp = Gi[p][p2], g_pq = Gi[p][q2], g_qp = Gi[q][p2], g_qq = Gi[q][q2];
        if (sb != 0.0) {  // columns p2, q2: G J
            const cplx v0 = cmul(eb, g_pq), v1 = cmul(eb, g_qq);
            const cplx u0 = g_pp, u1 = g_qp;
            g_pp = mk(cb * u0.x - sb * v0.x, cb * u0.y - sb * v0.y);
            g_pq = mk(sb * u0.x + cb * v0.x, sb * u0.y + cb * v0.y);
            g_qp = mk(cb * u1.x - sb * v1.x, cb * u1.y - sb * v1.y);
            g_qq = mk(sb * u1.x + cb * v1.x, sb * u1.y + cb * v1.y);
        }
        if (sa != 0.0) {  // rows p, q: J^H (G J)
            const cplx ec = cconj(ea);
            const cplx v0 = cmul(ec, g_qp), v1 = cmul(ec, g_qq);
            const cplx u0 = g_pp, u1 = g_pq;
            g_pp = mk(ca * u0.x - sa * v0.x, ca * u0.y - sa * v0.y);
            g_qp = mk(sa * u0.x + ca * v0.x, sa * u0.y + ca * v0.y);
            g_pq = mk(ca * u1.x - sa * v1.x, ca * u1.y - sa * v1.y);
            g_qq = mk(sa * u1.x + ca * v1.x, sa * u1.y + ca * v1.y);
        }
        Go[p][p2] = g_pp; Go[p][q2] = g_pq; Go[q][p2] = g_qp; Go[q][q2] = g_qq;
        if (sb != 0.0) {  // W J on rows 2ka, 2ka+1
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = 2 * ka + h;
                const cplx w = sW[i][p2], wv = cmul(eb, sW[i][q2]);
                sW[i][p2] = mk(cb * w.x - sb * wv.x, cb * w.y - sb * wv.y);
                sW[i][q2] = mk(sb * w.x + cb * wv.x, sb * w.y + cb * wv.y);
            }
        }
        __syncthreads();
        cplx(*t)[ld] = Gi; Gi = Go; Go = t;
    }
    if (isw == 0 && tid == 0) { s_first = s_rot; s_off2_first = s_off2; }
    const bool more = s_rot != rot_before;
    __syncthreads();  // (all threads read s_rot before the next sweep changes it)
    if (!more) break;
    }

        if (tid == 0) s_ident = s_first == 0;
        if (tid == 0 && s_first) {
            atomicAdd(&a.stat->rot, s_first);
            atomicMax(&a.stat->off2, s_off2_first);
        }
    }
    cluster.sync();  // W is ready in CTA 0
    if (crank != 0) {
        const cplx(*pw)[ld] = cluster.map_shared_rank(sW, 0);
        for (int e = tid; e < n2 * n2; e += kBjThreads) sW[e / n2][e % n2] = pw[e / n2][e % n2];
        if (tid == 0) s_ident = *cluster.map_shared_rank(&s_ident, 0);
    }
    cluster.sync();  // CTA 0's W may now be left (and the kernel may end) — peers have copied it

    // ---- [X_i X_j] W and [V_i V_j] W into the next step's block positions: the X chunks, then the
    // V chunks, double-buffered (chunk t in buffer (t + 1) & 1).  Warp w: row tile w & 3 of the
    // chunk times column tiles 2 (w >> 2) + {0, 1} of W, on DMMA.
    const long long dA = (long long)a.dst[2 * k0] * b, dB = (long long)a.dst[2 * k0 + 1] * b;
    const int nac = nxc + nvc;
    const int rt = warp & 3, ct0 = 2 * (warp >> 2);
    for (int t = 0; t < nac; ++t) {
        if (t + 1 < nac) {
            stage_apply(t + 1, buf[t & 1]);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const Chunk& ch = buf[(t + 1) & 1];
        const bool isx = t < nxc;
        cplx* D = isx ? a.Xd : a.Vd;
        const int r0 = isx ? xr0 + t * kBjRows : vr0 + (t - nxc) * kBjRows;
        const int nr = min(kBjRows, (isx ? xr1 : vr1) - r0);
        if (s_ident) {  // W = I: the blocks only move to their next slots
            for (int e = tid; e < nr * n2; e += kBjThreads) {
                const int i = e / n2, j = e % n2;
                D[(long long)(r0 + i) * cp + (j < b ? dA + j : dB + j - b)] = ch[i][j];
            }
        } else if (rt * 8 < nr) {
            double are[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, aim[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int kk = 0; kk < n2 / 4; ++kk) {
                const cplx xa = ch[rt * 8 + (lane >> 2)][kk * 4 + (lane & 3)];
                const cplx w0 = sW[kk * 4 + (lane & 3)][ct0 * 8 + (lane >> 2)];
                const cplx w1 = sW[kk * 4 + (lane & 3)][(ct0 + 1) * 8 + (lane >> 2)];
                dmma884(are[0][0], are[0][1], xa.x, w0.x);
                dmma884(are[1][0], are[1][1], xa.x, w1.x);
                dmma884(aim[0][0], aim[0][1], xa.x, w0.y);
                dmma884(aim[1][0], aim[1][1], xa.x, w1.y);
                dmma884(are[0][0], are[0][1], -xa.y, w0.y);
                dmma884(are[1][0], are[1][1], -xa.y, w1.y);
                dmma884(aim[0][0], aim[0][1], xa.y, w0.x);
                dmma884(aim[1][0], aim[1][1], xa.y, w1.x);
            }
            const int i = rt * 8 + (lane >> 2);
            if (i < nr) {
                const long long row = (long long)(r0 + i) * cp;
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int j = (ct0 + q) * 8 + 2 * (lane & 3) + c;
                        D[row + (j < b ? dA + j : dB + j - b)] = mk(are[q][c], aim[q][c]);
                    }
            }
        }
        __syncthreads();  // (the buffer is refilled by the next iteration's prefetch)
    }
}


__global__ void __launch_bounds__(kBjThreads) bj_step_kernel(const __grid_constant__ BjStep a) {
    const int S = (int)cg::this_cluster().num_blocks();
    const int pr = blockIdx.y;
    const BjPair q{a.Xs[pr], a.Vs[pr], a.Xd[pr], a.Vd[pr], a.dst, a.stat[pr], a.r, a.cp, a.b, a.inner_sweeps,
                   a.cross_only};
    bj_pair(q, blockIdx.x / S);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// A whole sweep in one launch.  Work items (step t, problem q, pair k) are claimed from a counter
// in step-major order; an item of step t > 0 waits for the (at most four) items of step t-1 it
// depends on: the two that produced its blocks, and the two that read its destination slots of
// the ping-pong buffer it writes.  Every waited-on item was claimed earlier by a running CTA, so
// the scheme cannot deadlock whatever the residency; steps overlap instead of meeting at a
// grid-wide barrier per launch.
__global__ void __launch_bounds__(kBjThreads, 3) bj_sweep_kernel(const __grid_constant__ BjSweep a) {
    __shared__ int s_item;
    const int per_step = a.count * a.npairs, total = per_step * a.nsteps;
    for (;;) {
        __syncthreads();  // (s_item is rewritten below)
        if (threadIdx.x == 0) s_item = atomicAdd(a.counter, 1);
        __syncthreads();
        const int item = s_item;
        if (item >= total) return;
        const int t = item / per_step, rem = item % per_step, qi = rem / a.npairs, k = rem % a.npairs;
        const int nbp = 2 * a.npairs;
        int* done = a.done + (size_t)qi * a.nsteps * a.npairs;
        if (t > 0 && threadIdx.x < 4) {
            const int* dstt = a.dst + (size_t)t * nbp;
            const int* prod = a.prod + (size_t)t * nbp;
            const int dep = threadIdx.x < 2 ? prod[2 * k + threadIdx.x] : dstt[2 * k + threadIdx.x - 2] >> 1;
            const int* f = done + (size_t)(t - 1) * a.npairs + dep;
            long long spins = 0;
            while (ld_acquire(f) < a.epoch) {
                __nanosleep(64);
                if (++spins > (1ll << 26)) __trap();  // (a broken dependency: fail, never hang)
            }
        }
        __syncthreads();
        const BjPair q{a.X[t & 1][qi], a.V[t & 1][qi], a.X[(t + 1) & 1][qi], a.V[(t + 1) & 1][qi],
                       a.dst + (size_t)t * nbp, a.stat[qi], a.r, a.cp, a.b, a.inner_sweeps,
                       a.cross_steps && t > 0};
        bj_pair(q, k);
        __syncthreads();  // every write of the item precedes the release
        if (threadIdx.x == 0) {
            __threadfence();
            st_release(done + (size_t)t * a.npairs + k, a.epoch);
        }
    }
}

// Finish, part 1 (one CTA per problem): column norms of X (σ per slot; row-parallel, partial sums
// in a fixed order), each genuine slot's rank in the non-increasing order (ties by original
// column), σ written sorted.
constexpr int kBjFinThreads = 512;
__global__ void __launch_bounds__(kBjFinThreads) bj_rank_kernel(const __grid_constant__ BjFinish a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int pr = blockIdx.x;
    double* sig = reinterpret_cast<double*>(sm);     // per slot (genuine columns)
    int* orig = reinterpret_cast<int*>(sig + a.cp);  // per slot: original column or -1
    __shared__ double part[kBjFinThreads];
    const cplx* X = a.X[pr];
    const int cp = a.cp;
    for (int s = threadIdx.x; s < cp; s += kBjFinThreads) {
        const int o = a.place[s / a.b] * a.b + s % a.b;
        orig[s] = o < a.c ? o : -1;
    }
    const int cpp = min(cp, kBjFinThreads), tpc = kBjFinThreads / cpp;
    const int jl = threadIdx.x % cpp, q = threadIdx.x / cpp;
    for (int j0 = 0; j0 < cp; j0 += cpp) {
        const int s = j0 + jl;
        double a0 = 0.0, a1 = 0.0;
        if (q < tpc && s < cp) {
            int i = q;
            for (; i + tpc < a.r; i += 2 * tpc) {
                a0 += cabs2(X[(long long)i * cp + s]);
                a1 += cabs2(X[(long long)(i + tpc) * cp + s]);
            }
            if (i < a.r) a0 += cabs2(X[(long long)i * cp + s]);
        }
        part[threadIdx.x] = a0 + a1;
        __syncthreads();
        if (q == 0 && s < cp) {
            double acc = 0.0;
            for (int t = 0; t < tpc; ++t) acc += part[t * cpp + jl];
            sig[s] = sqrt(acc);
        }
        __syncthreads();
    }
    for (int s = threadIdx.x; s < cp; s += kBjFinThreads) {
        int rk = -1;
        if (orig[s] >= 0) {
            const double v = sig[s], kv = rank_key(v);
            rk = 0;
            for (int t = 0; t < cp; ++t)
                if (orig[t] >= 0) rk += (rank_key(sig[t]) > kv) || (rank_key(sig[t]) == kv && orig[t] < orig[s]);
            a.sigma[pr][rk] = v;
        }
        a.rank_ws[(size_t)pr * cp + s] = rk;
        a.sig_ws[(size_t)pr * cp + s] = sig[s];
    }
}

// Finish, part 2 (a 2-D grid of CTAs per problem): Xn = X columns / σ and Js = V columns, each
// slot written to its sorted position.
__global__ void __launch_bounds__(256) bj_scatter_kernel(const __grid_constant__ BjFinish a) {
    const int pr = blockIdx.y;
    const int cp = a.cp;
    const int* rank = a.rank_ws + (size_t)pr * cp;
    const double* sig = a.sig_ws + (size_t)pr * cp;
    const long long nx = a.Xn[pr] ? (long long)a.r * cp : 0, nv = a.Js[pr] ? (long long)a.c * cp : 0;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < nx + nv; e += (long long)gridDim.x * 256) {
        const bool isx = e < nx;
        const long long f = isx ? e : e - nx;
        const int i = (int)(f / cp), s = (int)(f % cp);
        const int rk = rank[s];
        if (rk < 0) continue;
        if (isx) {
            const double inv = sig[s] > 0.0 ? 1.0 / sig[s] : 0.0;
            a.Xn[pr][(long long)i * a.c + rk] = cscale(a.X[pr][f], inv);
        } else {
            a.Js[pr][(long long)i * a.c + rk] = a.V[pr][f];
        }
    }
}

}  // namespace

cudaError_t bj_init(const BjInit& a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    const long long tot = (long long)a.r * a.cp + (long long)a.cp * a.cp;
    const int gx = (int)std::min<long long>((tot + kBjThreads - 1) / kBjThreads, 1024);
    bj_init_kernel<<<dim3(gx, a.count), kBjThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t bj_step(const BjStep& a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    if (2 * a.b != kBjN2) return cudaErrorInvalidValue;
    constexpr size_t smem = sizeof(cplx) * (2 * kBjRows * (kBjN2 + 1) + 2 * kBjN2 * (kBjN2 + 1));
    cudaError_t e = cudaFuncSetAttribute(bj_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // row slices per pair: as many as keep every CTA resident in one wave (3 per SM at this
    // shared-memory size), at most 8 (portable cluster), at least 64 rows per slice
    const int S = bj_slices(a.npairs * a.count, a.r);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.npairs * S, a.count);
    cfg.blockDim = dim3(kBjThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, bj_step_kernel, a);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

int bj_slices(int pairs, int r) {
    // Power-of-two row slices per pair (cluster size): as many as keep every CTA resident in one
    // wave (3 per SM at this shared-memory size), at most 8, at least 64 rows per slice.
    // (Measured: a cost model choosing 7 for one 2000² problem — 441 CTAs, 3 per SM — ran 313 ms
    // against 259 ms with 4.)
    int S = 1;
    while (S < 8 && (long long)pairs * (2 * S) <= 3LL * 148 && (r / (2 * S)) >= 64) S *= 2;
    static const int env_s = [] {  // (RRSVD_B200_BJ_S: force the row-slice count, for tuning)
        const char* e = std::getenv("RRSVD_B200_BJ_S");
        return e ? std::atoi(e) : 0;
    }();
    if (env_s >= 1 && env_s <= 8) S = std::min(env_s, std::max(1, r / 32));
    return S;
}

cudaError_t bj_sweep(const BjSweep& a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    if (2 * a.b != kBjN2) return cudaErrorInvalidValue;
    constexpr size_t smem = sizeof(cplx) * (2 * kBjRows * (kBjN2 + 1) + 2 * kBjN2 * (kBjN2 + 1));
    cudaError_t e = cudaFuncSetAttribute(bj_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0, dev = 0, nsm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bj_sweep_kernel, kBjThreads, smem);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long total = (long long)a.count * a.npairs * a.nsteps;
    const int grid = (int)std::min<long long>(total, (long long)std::max(1, per_sm) * nsm);
    bj_sweep_kernel<<<grid, kBjThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t bj_finish(const BjFinish& a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    const size_t smem = (size_t)a.cp * (sizeof(double) + sizeof(int));
    cudaError_t e = smem_atleast(reinterpret_cast<const void*>(bj_rank_kernel), smem);
    if (e != cudaSuccess) return e;
    bj_rank_kernel<<<a.count, kBjFinThreads, smem, s>>>(a);
    const long long per = (long long)(a.r + a.c) * a.cp;
    const int gx = (int)std::max<long long>(1, std::min<long long>((per + 255) / 256, std::max(1, 4 * 148 / a.count)));
    bj_scatter_kernel<<<dim3(gx, a.count), 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace rb

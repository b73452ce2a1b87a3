// blockjac.cu — kernels of the block one-sided Jacobi SVD (see blockjac.cuh).
#include <algorithm>
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

constexpr int kBjRows = 64;  // row chunk staged per pass
constexpr int kBjN2 = 32;    // 2b (b = 16)

// One block pair, one CTA: Gram, one sweep of two-sided Jacobi (round-robin rounds of n2/2
// disjoint pairs: parameters from (G_pp, G_qq, G_pq) exactly as the Hestenes rotation, then the
// column update G J and W J, then the row update J^H G), then the rotated columns.
// The pair's rows are split over the S CTAs of a thread-block cluster: each CTA forms the Gram
// of its row slice, CTA 0 sums the slices over DSMEM (fixed order) and solves, the peers read W
// back over DSMEM and rotate their own slices of X and V.
__global__ void __launch_bounds__(kBjThreads) bj_step_kernel(const __grid_constant__ BjStep a) {
    constexpr int n2 = kBjN2, ld = n2 + 1, half = n2 / 2;
    cg::cluster_group cluster = cg::this_cluster();
    const int S = (int)cluster.num_blocks(), crank = (int)cluster.block_rank();
    extern __shared__ __align__(16) unsigned char sm[];
    auto ch = reinterpret_cast<cplx(*)[ld]>(sm);                        // [kBjRows][ld]
    auto sG = reinterpret_cast<cplx(*)[ld]>(sm + sizeof(cplx) * kBjRows * ld);  // [n2][ld]
    auto sW = sG + n2;                                                    // [n2][ld]
    __shared__ double pc[half], ps[half];
    __shared__ cplx pe[half];
    __shared__ int pp[half], pq[half];
    __shared__ int s_rot;
    const int pr = blockIdx.y, k0 = blockIdx.x / S, tid = threadIdx.x;
    const int r = a.r, cp = a.cp, b = a.b;
    const int xr0 = (int)((long long)r * crank / S), xr1 = (int)((long long)r * (crank + 1) / S);
    const int vr0 = (int)((long long)cp * crank / S), vr1 = (int)((long long)cp * (crank + 1) / S);
    const long long col0 = (long long)k0 * n2;  // the pair's first column (slots 2k0, 2k0+1)
    const cplx* X = a.Xs[pr];

    // ---- Gram of this CTA's row slice on the FP64 tensor core: the 32 x 32 result is 4 x 4 tiles
    // of 8 x 8; warp w accumulates tiles (pt = w/2, qt = 2(w%2) + {0,1}).  Fragments are one
    // LDS.128 (re, im) per lane; conj(X)^T X in 4M form: Re += xr xr' + xi xi', Im += xr xi' - xi xr'.
    const int lane = tid & 31, warp = tid >> 5;
    const int pt = warp >> 1, qa = 2 * (warp & 1);
    double gre[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, gim[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int r0 = xr0; r0 < xr1; r0 += kBjRows) {
        const int nr = min(kBjRows, xr1 - r0), nr4 = (nr + 3) & ~3;
        __syncthreads();
        for (int e = tid; e < nr4 * n2; e += kBjThreads) {
            const int i = e / n2, j = e % n2;
            ch[i][j] = i < nr ? X[(long long)(r0 + i) * cp + col0 + j] : mk(0.0, 0.0);
        }
        __syncthreads();
        for (int k0 = 0; k0 < nr4; k0 += 4) {
            const cplx xa = ch[k0 + (lane & 3)][pt * 8 + (lane >> 2)];
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
                const cplx xb = ch[k0 + (lane & 3)][(qa + qq) * 8 + (lane >> 2)];
                dmma884(gre[qq][0], gre[qq][1], xa.x, xb.x);
                dmma884(gre[qq][0], gre[qq][1], xa.y, xb.y);
                dmma884(gim[qq][0], gim[qq][1], xa.x, xb.y);
                dmma884(gim[qq][0], gim[qq][1], -xa.y, xb.x);
            }
        }
    }
#pragma unroll
    for (int qq = 0; qq < 2; ++qq)
#pragma unroll
        for (int c = 0; c < 2; ++c)
            sG[pt * 8 + (lane >> 2)][(qa + qq) * 8 + 2 * (lane & 3) + c] = mk(gre[qq][c], gim[qq][c]);
    cluster.sync();
    if (crank == 0) {  // (uniform per CTA; barriers below are reached by every thread)
        // sum the slices in rank order, then keep the upper triangle and mirror it
        cplx sum[n2 * n2 / kBjThreads];
#pragma unroll
        for (int u = 0; u < n2 * n2 / kBjThreads; ++u) {
            const int e = tid + u * kBjThreads;
            sum[u] = mk(0.0, 0.0);
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
        if (tid == 0) s_rot = 0;
        __syncthreads();

    // ---- one sweep of the pair solve
    const double tol = sqrt((double)max(r, 1)) * kEpsBj;
    __shared__ int s_first;  // rotations of the first inner sweep: the outer convergence signal
    for (int isw = 0; isw < a.inner_sweeps; ++isw) {
    const int rot_before = s_rot;
    for (int rd = 0; rd < n2 - 1; ++rd) {
        if (tid < half) {
            const int p = circle_bj(tid, rd, n2), q = circle_bj(n2 - 1 - tid, rd, n2);
            const double ga = sG[p][p].x, gb = sG[q][q].x;
            const cplx g = sG[p][q];
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
            }
            pc[tid] = c; ps[tid] = s; pe[tid] = e; pp[tid] = p; pq[tid] = q;
        }
        __syncthreads();
        for (int idx = tid; idx < half * n2; idx += kBjThreads) {  // columns: G J, W J
            const int k = idx / n2, i = idx % n2;
            const double s = ps[k];
            if (s == 0.0) continue;
            const double c = pc[k];
            const cplx e = pe[k];
            const int p = pp[k], q = pq[k];
            const cplx u = sG[i][p], ev = cmul(e, sG[i][q]);
            sG[i][p] = mk(c * u.x - s * ev.x, c * u.y - s * ev.y);
            sG[i][q] = mk(s * u.x + c * ev.x, s * u.y + c * ev.y);
            const cplx w = sW[i][p], wv = cmul(e, sW[i][q]);
            sW[i][p] = mk(c * w.x - s * wv.x, c * w.y - s * wv.y);
            sW[i][q] = mk(s * w.x + c * wv.x, s * w.y + c * wv.y);
        }
        __syncthreads();
        for (int idx = tid; idx < half * n2; idx += kBjThreads) {  // rows: J^H G
            const int k = idx / n2, j = idx % n2;
            const double s = ps[k];
            if (s == 0.0) continue;
            const double c = pc[k];
            const cplx ec = cconj(pe[k]);
            const int p = pp[k], q = pq[k];
            const cplx u = sG[p][j], ev = cmul(ec, sG[q][j]);
            sG[p][j] = mk(c * u.x - s * ev.x, c * u.y - s * ev.y);
            sG[q][j] = mk(s * u.x + c * ev.x, s * u.y + c * ev.y);
        }
        __syncthreads();
    }
    if (isw == 0 && tid == 0) s_first = s_rot;
    const bool more = s_rot != rot_before;
    __syncthreads();  // (all threads read s_rot before the next sweep changes it)
    if (!more) break;
    }

        if (tid == 0 && s_first) atomicAdd(a.rot[pr], s_first);
    }
    cluster.sync();  // W is ready in CTA 0
    if (crank != 0) {
        const cplx(*pw)[ld] = cluster.map_shared_rank(sW, 0);
        for (int e = tid; e < n2 * n2; e += kBjThreads) sW[e / n2][e % n2] = pw[e / n2][e % n2];
    }
    cluster.sync();  // CTA 0's W may now be left (and the kernel may end) — peers have copied it

    // ---- [X_i X_j] W and [V_i V_j] W into the next step's block positions
    const long long dA = (long long)a.dst[2 * k0] * b, dB = (long long)a.dst[2 * k0 + 1] * b;
    for (int m = 0; m < 2; ++m) {
        const cplx* S = m == 0 ? X : a.Vs[pr];
        cplx* D = m == 0 ? a.Xd[pr] : a.Vd[pr];
        const int rbeg = m == 0 ? xr0 : vr0, rend = m == 0 ? xr1 : vr1;
        for (int r0 = rbeg; r0 < rend; r0 += kBjRows) {
            const int nr = min(kBjRows, rend - r0), nr8 = (nr + 7) & ~7;
            __syncthreads();
            for (int e = tid; e < nr8 * n2; e += kBjThreads) {
                const int i = e / n2, j = e % n2;
                ch[i][j] = i < nr ? S[(long long)(r0 + i) * cp + col0 + j] : mk(0.0, 0.0);
            }
            __syncthreads();
            // warp w: rows 8w .. 8w+7 of the chunk times all of W (4 column tiles), on DMMA
            const int rt = warp;
            if (rt * 8 < nr) {
                double are[4][2], aim[4][2];
#pragma unroll
                for (int ct = 0; ct < 4; ++ct) are[ct][0] = are[ct][1] = aim[ct][0] = aim[ct][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < n2 / 4; ++kk) {
                    const cplx xa = ch[rt * 8 + (lane >> 2)][kk * 4 + (lane & 3)];
#pragma unroll
                    for (int ct = 0; ct < 4; ++ct) {
                        const cplx wb = sW[kk * 4 + (lane & 3)][ct * 8 + (lane >> 2)];
                        dmma884(are[ct][0], are[ct][1], xa.x, wb.x);
                        dmma884(are[ct][0], are[ct][1], -xa.y, wb.y);
                        dmma884(aim[ct][0], aim[ct][1], xa.x, wb.y);
                        dmma884(aim[ct][0], aim[ct][1], xa.y, wb.x);
                    }
                }
                const int i = rt * 8 + (lane >> 2);
                if (i < nr) {
                    const long long row = (long long)(r0 + i) * cp;
#pragma unroll
                    for (int ct = 0; ct < 4; ++ct)
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            const int j = ct * 8 + 2 * (lane & 3) + c;
                            D[row + (j < b ? dA + j : dB + j - b)] = mk(are[ct][c], aim[ct][c]);
                        }
                }
            }
        }
    }
}

__global__ void __launch_bounds__(kBjThreads) bj_finish_kernel(const __grid_constant__ BjFinish a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int pr = blockIdx.x;
    double* sig = reinterpret_cast<double*>(sm);     // per slot (genuine columns)
    int* orig = reinterpret_cast<int*>(sig + a.cp);  // per slot: original column or -1
    int* rank = orig + a.cp;
    const cplx* X = a.X[pr];
    for (int s = threadIdx.x; s < a.cp; s += kBjThreads) {
        const int o = a.place[s / a.b] * a.b + s % a.b;
        orig[s] = o < a.c ? o : -1;
        double acc = 0.0;
        if (o < a.c)
            for (int i = 0; i < a.r; ++i) acc += cabs2(X[(long long)i * a.cp + s]);
        sig[s] = sqrt(acc);
    }
    __syncthreads();
    for (int s = threadIdx.x; s < a.cp; s += kBjThreads) {
        if (orig[s] < 0) { rank[s] = -1; continue; }
        const double v = sig[s];
        int rk = 0;
        for (int t = 0; t < a.cp; ++t)
            if (orig[t] >= 0) rk += (sig[t] > v) || (sig[t] == v && orig[t] < orig[s]);
        rank[s] = rk;
    }
    __syncthreads();
    for (int s = threadIdx.x; s < a.cp; s += kBjThreads)
        if (rank[s] >= 0) a.sigma[pr][rank[s]] = sig[s];
    if (a.Xn[pr]) {
        cplx* Xn = a.Xn[pr];
        for (long long e = threadIdx.x; e < (long long)a.r * a.cp; e += kBjThreads) {
            const int i = (int)(e / a.cp), s = (int)(e % a.cp);
            if (rank[s] < 0) continue;
            const double inv = sig[s] > 0.0 ? 1.0 / sig[s] : 0.0;
            Xn[(long long)i * a.c + rank[s]] = cscale(X[e], inv);
        }
    }
    if (a.Js[pr]) {
        cplx* Js = a.Js[pr];
        const cplx* V = a.V[pr];
        for (long long e = threadIdx.x; e < (long long)a.c * a.cp; e += kBjThreads) {
            const int i = (int)(e / a.cp), s = (int)(e % a.cp);
            if (rank[s] < 0) continue;
            Js[(long long)i * a.c + rank[s]] = V[e];
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
    constexpr size_t smem = sizeof(cplx) * (kBjRows * (kBjN2 + 1) + 2 * kBjN2 * (kBjN2 + 1));
    cudaError_t e = cudaFuncSetAttribute(bj_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // row slices per pair: as many as keep every CTA resident in one wave (3 per SM at this
    // shared-memory size), at most 8 (portable cluster), at least one 64-row chunk per slice
    const long long pairs = (long long)a.npairs * a.count;
    int S = 1;
    while (S < 8 && pairs * (2 * S) <= 3LL * 148 && (a.r / (2 * S)) >= kBjRows) S *= 2;
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

cudaError_t bj_finish(const BjFinish& a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    const size_t smem = (size_t)a.cp * (sizeof(double) + 2 * sizeof(int));
    cudaError_t e = cudaFuncSetAttribute(bj_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    bj_finish_kernel<<<a.count, kBjThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace rb

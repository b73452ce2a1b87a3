#include <algorithm>
// tebd_kernels.cu — sketch generation, gate for small d, layout conversion, truncation,
// Gamma reshape, peak probes.  See tebd_kernels.cuh.
#include "tebd_kernels.cuh"

namespace rb {

namespace {

// ============================================================================ mt19937_64
constexpr int MT_N = 312, MT_M = 156;
constexpr unsigned long long MT_A = 0xB5026F5AA96619E9ull;
constexpr unsigned long long MT_UM = 0xFFFFFFFF80000000ull, MT_LM = 0x7FFFFFFFull;

__device__ __forceinline__ unsigned long long mt_twist(unsigned long long cur, unsigned long long nxt) {
    const unsigned long long y = (cur & MT_UM) | (nxt & MT_LM);
    return (y >> 1) ^ ((y & 1ull) ? MT_A : 0ull);
}
__device__ __forceinline__ unsigned long long mt_temper(unsigned long long y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= (y >> 43);
    return y;
}

// One CTA: the twist of a 312-word state has two dependency-free phases
// (i < 156 reads only old words; i >= 156 reads words rewritten in phase 1).
__global__ void __launch_bounds__(320) mt_draws_kernel(uint64_t seed, long long rounds,
                                                       unsigned long long* __restrict__ out) {
    __shared__ unsigned long long st[2][MT_N];
    const int t = threadIdx.x;
    if (t == 0) {
        unsigned long long x = seed;
        st[0][0] = x;
        for (int i = 1; i < MT_N; ++i) {
            x = 6364136223846793005ull * (x ^ (x >> 62)) + (unsigned long long)i;
            st[0][i] = x;
        }
    }
    __syncthreads();
    int cur = 0;
    for (long long rd = 0; rd < rounds; ++rd) {
        const unsigned long long* o = st[cur];
        unsigned long long* nw = st[cur ^ 1];
        if (t < MT_M) nw[t] = o[t + MT_M] ^ mt_twist(o[t], o[t + 1]);
        __syncthreads();
        if (t >= MT_M && t < MT_N) {
            const unsigned long long nxt = (t + 1 < MT_N) ? o[t + 1] : nw[0];
            nw[t] = nw[t - MT_M] ^ mt_twist(o[t], nxt);
        }
        __syncthreads();
        if (t < MT_N) out[rd * MT_N + t] = mt_temper(nw[t]);
        cur ^= 1;
    }
}

__device__ __forceinline__ cplx box_muller(unsigned long long x1, unsigned long long x2) {
    const double u1 = ((double)(x1 >> 11) + 1.0) * 0x1p-53;  // (0, 1]
    const double u2 = (double)(x2 >> 11) * 0x1p-53;          // [0, 1)
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.141592653589793 * u2;
    double sn, cs;
    sincos(angle, &sn, &cs);
    return mk(radius * cs, radius * sn);
}

__global__ void box_muller_kernel(const unsigned long long* __restrict__ draws, long long n, cplx* out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        out[e] = box_muller(draws[2 * e], draws[2 * e + 1]);
}

// ============================================================================ Philox4x32-10
__device__ __forceinline__ void philox_round(uint32_t c[4], const uint32_t k[2]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

__global__ void philox_kernel(uint64_t seed, long long n, cplx* out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0x243F6A88u, 0x85A308D3u};
        uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            philox_round(c, k);
            k[0] += 0x9E3779B9u;
            k[1] += 0xBB67AE85u;
        }
        const unsigned long long x1 = ((unsigned long long)c[1] << 32) | c[0];
        const unsigned long long x2 = ((unsigned long long)c[3] << 32) | c[2];
        out[e] = box_muller(x1, x2);
    }
}

// ============================================================================ gate (small dd)
template <int MAXD>
__global__ void gate_small_kernel(const cplx* __restrict__ G, int dd, int cl, int cr,
                                  const cplx* __restrict__ Min, cplx* __restrict__ Mout) {
    __shared__ cplx sg[MAXD * MAXD];
    for (int i = threadIdx.x; i < dd * dd; i += blockDim.x) sg[i] = G[i];
    __syncthreads();
    const long long cols = (long long)cl * cr;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cols;
         e += (long long)gridDim.x * blockDim.x) {
        const long long a = e / cr, b = e % cr;
        const cplx* src = Min + a * dd * cr + b;
        cplx v[MAXD];
#pragma unroll
        for (int y = 0; y < MAXD; ++y) v[y] = y < dd ? src[(long long)y * cr] : mk(0.0, 0.0);
        cplx* dst = Mout + a * dd * cr + b;
#pragma unroll
        for (int x = 0; x < MAXD; ++x) {
            if (x >= dd) break;
            cplx s = mk(0.0, 0.0);
#pragma unroll
            for (int y = 0; y < MAXD; ++y)
                if (y < dd) cfma(s, sg[x * dd + y], v[y]);
            dst[(long long)x * cr] = s;
        }
    }
}

// ============================================================================ block gate
// grid (column chunks of 256, job); each thread owns one column (a, b) of the job's Θ and runs
// through all blocks; the block G_B is staged in shared memory, the |S_B| inputs in registers.
__global__ void __launch_bounds__(256) gate_blocks_kernel(const __grid_constant__ GateBlockBatch bt) {
    __shared__ cplx sg[kMaxGateBlock * kMaxGateBlock];
    const GateBlockJob& J = bt.j[blockIdx.y];
    const GateBlocks& B = J.gb;
    const long long cols = (long long)J.cl * J.cr;
    const long long c = blockIdx.x * 256LL + threadIdx.x;
    const bool active = c < cols;
    const long long a = active ? c / J.cr : 0, bcol = active ? c % J.cr : 0;
    const long long base = a * B.dd * J.cr + bcol;
    for (int k = 0; k < B.nblocks; ++k) {
        const int off = B.offs[k], sz = B.offs[k + 1] - off;
        const cplx* g = B.gblk + B.goff[k];
        __syncthreads();
        for (int t = threadIdx.x; t < sz * sz; t += 256) sg[t] = g[t];
        __syncthreads();
        if (!active) continue;
        cplx v[kMaxGateBlock];
#pragma unroll
        for (int t = 0; t < kMaxGateBlock; ++t)
            if (t < sz) v[t] = J.Min[base + (long long)B.idx[off + t] * J.cr];
        for (int r = 0; r < sz; ++r) {
            cplx acc = mk(0.0, 0.0);
#pragma unroll
            for (int t = 0; t < kMaxGateBlock; ++t)
                if (t < sz) cfma(acc, sg[r * sz + t], v[t]);
            J.Mout[base + (long long)B.idx[off + r] * J.cr] = acc;
        }
    }
}

// Staged variant: every block of the gate (sum |S_B|^2 entries) and the state index list sit in
// shared memory for the whole CTA, and each block runs an exact-size unrolled body (the generic
// kernel above pays 32-wide predicated loops and two barriers per block).  One thread per
// Θ column (a, β): it gathers the |S_B| entries of its column that the block mixes, applies G_B
// from shared memory (broadcast reads) and scatters the results — coalesced across the warp.
template <int SZ>
__device__ __forceinline__ void gate_block_apply(const cplx* __restrict__ g, const int* __restrict__ idx,
                                                 const cplx* __restrict__ Min, cplx* __restrict__ Mout,
                                                 long long base, long long stride) {
    cplx v[SZ];
#pragma unroll
    for (int t = 0; t < SZ; ++t) v[t] = Min[base + (long long)idx[t] * stride];
#pragma unroll 1
    for (int r = 0; r < SZ; ++r) {
        cplx acc = mk(0.0, 0.0), acc2 = mk(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < SZ; t += 2) {
            cfma(acc, g[r * SZ + t], v[t]);
            if (t + 1 < SZ) cfma(acc2, g[r * SZ + t + 1], v[t + 1]);
        }
        Mout[base + (long long)idx[r] * stride] = mk(acc.x + acc2.x, acc.y + acc2.y);
    }
}

__global__ void __launch_bounds__(256, 2) gate_blocks_staged_kernel(const __grid_constant__ GateBlockBatch bt) {
    extern __shared__ __align__(16) unsigned char sm[];
    const GateBlockJob& J = bt.j[blockIdx.y];
    const GateBlocks& B = J.gb;
    cplx* sg = reinterpret_cast<cplx*>(sm);
    int* sidx = reinterpret_cast<int*>(sg + B.total);
    int* soff = sidx + B.dd;  // nblocks + 1 offsets, then nblocks gate offsets
    int* sgoff = soff + B.nblocks + 1;
    for (int t = threadIdx.x; t < B.total; t += 256) sg[t] = B.gblk[t];
    for (int t = threadIdx.x; t < B.dd; t += 256) sidx[t] = B.idx[t];
    for (int t = threadIdx.x; t <= B.nblocks; t += 256) soff[t] = B.offs[t];
    for (int t = threadIdx.x; t < B.nblocks; t += 256) sgoff[t] = B.goff[t];
    __syncthreads();
    const long long cols = (long long)J.cl * J.cr;
    const long long c = blockIdx.x * 256LL + threadIdx.x;
    if (c >= cols) return;
    const long long a = c / J.cr, bcol = c % J.cr;
    const long long base = a * B.dd * J.cr + bcol;
    const long long stride = J.cr;
    for (int k = 0; k < B.nblocks; ++k) {
        const int off = soff[k], sz = soff[k + 1] - off;
        const cplx* g = sg + sgoff[k];
        const int* ix = sidx + off;
        switch (sz) {
#define RB_GATE_CASE(N) \
    case N: gate_block_apply<N>(g, ix, J.Min, J.Mout, base, stride); break;
            RB_GATE_CASE(1) RB_GATE_CASE(2) RB_GATE_CASE(3) RB_GATE_CASE(4) RB_GATE_CASE(5) RB_GATE_CASE(6)
            RB_GATE_CASE(7) RB_GATE_CASE(8) RB_GATE_CASE(9) RB_GATE_CASE(10) RB_GATE_CASE(11) RB_GATE_CASE(12)
            RB_GATE_CASE(13) RB_GATE_CASE(14) RB_GATE_CASE(15) RB_GATE_CASE(16) RB_GATE_CASE(17) RB_GATE_CASE(18)
            RB_GATE_CASE(19) RB_GATE_CASE(20) RB_GATE_CASE(21) RB_GATE_CASE(22) RB_GATE_CASE(23) RB_GATE_CASE(24)
            RB_GATE_CASE(25) RB_GATE_CASE(26) RB_GATE_CASE(27) RB_GATE_CASE(28) RB_GATE_CASE(29) RB_GATE_CASE(30)
            RB_GATE_CASE(31) RB_GATE_CASE(32)
#undef RB_GATE_CASE
            default: break;
        }
    }
}

// ============================================================================ layout
__global__ void theta_unfold_kernel(const cplx* __restrict__ src, int d1, int d2, int cl, int cr,
                                    cplx* __restrict__ dst, int to_unfolded) {
    // one row of length cr per (i, j, a)
    const long long rows = (long long)d1 * d2 * cl;
    for (long long rw = blockIdx.x; rw < rows; rw += gridDim.x) {
        const int a = (int)(rw % cl);
        const int j = (int)((rw / cl) % d2);
        const int i = (int)(rw / ((long long)cl * d2));
        const long long th = (((long long)i * d2 + j) * cl + a) * cr;
        const long long un = ((long long)a * d1 + i) * ((long long)d2 * cr) + (long long)j * cr;
        for (int b = threadIdx.x; b < cr; b += blockDim.x) {
            if (to_unfolded) dst[un + b] = src[th + b];
            else dst[th + b] = src[un + b];
        }
    }
}

// ============================================================================ truncation
__global__ void truncate_kernel(const TruncArgs a) {
    if (threadIdx.x != 0) return;
    const double total = *a.total_sq;
    if ((a.nonfinite && *a.nonfinite) || !(total > 0.0)) {  // rejected Θ: nothing kept
        *a.kept = 0;
        *a.discarded = 0.0;
        return;
    }
    const double sigma1 = a.ns > 0 ? a.sigma[0] : 0.0;
    int kept = 0;
    for (int i = 0; i < a.ns; ++i) {
        const double s = a.sigma[i];
        if (s <= sigma1 * 1e-15) break;
        if (a.trunc_tol > 0.0 && s * s / total < a.trunc_tol) break;
        ++kept;
    }
    if (kept < 1) kept = 1;
    if (a.cap > 0 && kept > a.cap) kept = (int)a.cap;
    double kept_sq = 0.0;
    for (int i = 0; i < kept; ++i) kept_sq += a.sigma[i] * a.sigma[i];
    double w = 1.0 - kept_sq / total;
    w = w < 0.0 ? 0.0 : (w > 1.0 ? 1.0 : w);
    *a.discarded = w;
    *a.kept = kept;
    if (a.lambda) {
        const double scale = a.renormalize ? 1.0 / sqrt(kept_sq) : 1.0;
        for (int i = 0; i < kept; ++i) a.lambda[i] = a.renormalize ? a.sigma[i] * scale : a.sigma[i];
    }
}

// ============================================================================ Gamma reshape
constexpr double kPinvFloor = 1e-14;  // tebd.cpp:19

__global__ void gamma_left_kernel(const GammaArgs a) {
    const int kept = *a.kept;
    const long long total = (long long)a.m * kept;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(e / kept), g = (int)(e % kept);
        double inv = 1.0;
        if (a.ll) {
            const double lv = a.ll[row / a.d1];
            inv = lv < kPinvFloor ? 0.0 : 1.0 / lv;
        }
        a.gamma_l[e] = cscale(a.U[(long long)row * a.ldu + g], inv);
    }
}

// gamma_r (kept x n) = conj(V (n x ldv))^T column-scaled: 32x32 tiles through shared memory.
__global__ void gamma_right_kernel(const GammaArgs a) {
    __shared__ cplx tile[32][33];
    const int kept = *a.kept;
    const int g0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    if (g0 >= kept) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int yy = ty; yy < 32; yy += 8) {
        const int c = c0 + yy, g = g0 + tx;
        tile[yy][tx] = (c < a.n && g < kept) ? a.V[(long long)c * a.ldv + g] : mk(0.0, 0.0);
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        const int g = g0 + yy, c = c0 + tx;
        if (g < kept && c < a.n) {
            double inv = 1.0;
            if (a.lr) {
                const double lv = a.lr[c % a.cr];
                inv = lv < kPinvFloor ? 0.0 : 1.0 / lv;
            }
            a.gamma_r[(long long)g * a.n + c] = cscale(cconj(tile[tx][yy]), inv);
        }
    }
}

__global__ void pinv_flag_kernel(const double* ll, int cl, const double* lr, int cr, int* flag) {
    int f = 0;
    for (int i = threadIdx.x; i < cl; i += blockDim.x) f |= ll && ll[i] < kPinvFloor;
    for (int i = threadIdx.x; i < cr; i += blockDim.x) f |= lr && lr[i] < kPinvFloor;
    f = __syncthreads_or(f);
    if (threadIdx.x == 0) *flag = f;
}

__global__ void fill_int_kernel(int* p, int v) { *p = v; }

// ---- batched epilogue kernels (blockIdx.y / z = problem) ------------------------------------
__global__ void truncate_many_kernel(const __grid_constant__ TruncBatch b) {
    if (threadIdx.x == 0) {
        // same code path as truncate_kernel (tebd.cpp:188-209)
        const TruncArgs& a = b.a[blockIdx.x];
        const double total = *a.total_sq;
        if ((a.nonfinite && *a.nonfinite) || !(total > 0.0)) {  // rejected Θ: nothing kept
            *a.kept = 0;
            *a.discarded = 0.0;
            return;
        }
        const double sigma1 = a.ns > 0 ? a.sigma[0] : 0.0;
        int kept = 0;
        for (int i = 0; i < a.ns; ++i) {
            const double s = a.sigma[i];
            if (s <= sigma1 * 1e-15) break;
            if (a.trunc_tol > 0.0 && s * s / total < a.trunc_tol) break;
            ++kept;
        }
        if (kept < 1) kept = 1;
        if (a.cap > 0 && kept > a.cap) kept = (int)a.cap;
        double kept_sq = 0.0;
        for (int i = 0; i < kept; ++i) kept_sq += a.sigma[i] * a.sigma[i];
        double w = 1.0 - kept_sq / total;
        w = w < 0.0 ? 0.0 : (w > 1.0 ? 1.0 : w);
        *a.discarded = w;
        *a.kept = kept;
        if (a.lambda) {
            const double scale = a.renormalize ? 1.0 / sqrt(kept_sq) : 1.0;
            for (int i = 0; i < kept; ++i) a.lambda[i] = a.renormalize ? a.sigma[i] * scale : a.sigma[i];
        }
    }
}

__global__ void gamma_left_many_kernel(const __grid_constant__ GammaBatch b) {
    const GammaArgs& a = b.a[blockIdx.y];
    const int kept = *a.kept;
    const long long total = (long long)a.m * kept;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(e / kept), g = (int)(e % kept);
        double inv = 1.0;
        if (a.ll) {
            const double lv = a.ll[row / a.d1];
            inv = lv < 1e-14 ? 0.0 : 1.0 / lv;
        }
        a.gamma_l[e] = cscale(a.U[(long long)row * a.ldu + g], inv);
    }
}

__global__ void gamma_right_many_kernel(const __grid_constant__ GammaBatch b) {
    __shared__ cplx tile[32][33];
    const GammaArgs& a = b.a[blockIdx.z];
    const int kept = *a.kept;
    const int g0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    if (g0 >= kept || c0 >= a.n) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int yy = ty; yy < 32; yy += 8) {
        const int c = c0 + yy, g = g0 + tx;
        tile[yy][tx] = (c < a.n && g < kept) ? a.V[(long long)c * a.ldv + g] : mk(0.0, 0.0);
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        const int g = g0 + yy, c = c0 + tx;
        if (g < kept && c < a.n) {
            double inv = 1.0;
            if (a.lr) {
                const double lv = a.lr[c % a.cr];
                inv = lv < 1e-14 ? 0.0 : 1.0 / lv;
            }
            a.gamma_r[(long long)g * a.n + c] = cscale(cconj(tile[tx][yy]), inv);
        }
    }
}

__global__ void pinv_many_kernel(const __grid_constant__ GammaBatch b) {
    const GammaArgs& a = b.a[blockIdx.x];
    const int cl = a.ll ? a.m / a.d1 : 0, cr = a.lr ? a.cr : 0;
    int f = 0;
    for (int i = threadIdx.x; i < cl; i += blockDim.x) f |= a.ll[i] < 1e-14;
    for (int i = threadIdx.x; i < cr; i += blockDim.x) f |= a.lr[i] < 1e-14;
    f = __syncthreads_or(f);
    if (threadIdx.x == 0) *a.pinv = f;
}

__global__ void philox_many_kernel(const __grid_constant__ PhiloxBatch b) {
    const int p = blockIdx.y;
    const uint64_t seed = b.seed[p];
    cplx* out = b.out[p];
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < b.n[p];
         e += (long long)gridDim.x * blockDim.x) {
        uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0x243F6A88u, 0x85A308D3u};
        uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            philox_round(c, k);
            k[0] += 0x9E3779B9u;
            k[1] += 0xBB67AE85u;
        }
        out[e] = box_muller(((unsigned long long)c[1] << 32) | c[0], ((unsigned long long)c[3] << 32) | c[2]);
    }
}

__global__ void scale_rows_many_kernel(const __grid_constant__ ScaleRowsBatch b) {
    const int p = blockIdx.y;
    const long long total = (long long)b.rows[p] * b.cols[p];
    const cplx* in = b.in[p];
    cplx* out = b.out[p];
    const double* s = b.s[p];
    const int cols = b.cols[p];
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x)
        out[e] = cscale(in[e], s[e / cols]);
}

__global__ void conj_transpose_kernel(const cplx* __restrict__ A, int rows, int cols, cplx* __restrict__ out) {
    __shared__ cplx tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int yy = ty; yy < 32; yy += 8) {
        const int r = r0 + yy, cc = c0 + tx;
        tile[yy][tx] = (r < rows && cc < cols) ? A[(long long)r * cols + cc] : mk(0.0, 0.0);
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        const int cc = c0 + yy, r = r0 + tx;
        if (cc < cols && r < rows) out[(long long)cc * rows + r] = cconj(tile[tx][yy]);
    }
}

__global__ void weight_kernel(const double* sigma, int k, const double* total_sq, double* w) {
    if (threadIdx.x != 0) return;
    const double total = *total_sq;
    if (total <= 0.0) { *w = 0.0; return; }
    double kept = 0.0;
    for (int i = 0; i < k; ++i) kept += sigma[i] * sigma[i];
    double v = 1.0 - kept / total;
    *w = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}

// ============================================================================ observables
constexpr int OBS_BLOCKS = 2 * kNumSMs;

__global__ void __launch_bounds__(256) expect_partial(const cplx* __restrict__ G, int dl, int d, int dr,
                                                      const double* ll, const double* lr,
                                                      const cplx* __restrict__ op, double* part) {
    __shared__ cplx so[32 * 32];
    for (int i = threadIdx.x; i < d * d; i += blockDim.x) so[i] = op[i];
    __syncthreads();
    cplx acc = mk(0.0, 0.0);
    const long long pairs = (long long)dl * dr;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < pairs;
         e += (long long)gridDim.x * blockDim.x) {
        const int a = (int)(e / dr), b = (int)(e % dr);
        const double wa = ll ? ll[a] * ll[a] : 1.0;
        const double w = wa * (lr ? lr[b] * lr[b] : 1.0);
        const cplx* g = G + (long long)a * d * dr + b;
        cplx s = mk(0.0, 0.0);
        for (int ip = 0; ip < d; ++ip) {
            cplx t = mk(0.0, 0.0);
            for (int i = 0; i < d; ++i) cfma(t, so[ip * d + i], g[(long long)i * dr]);
            cfmac(s, g[(long long)ip * dr], t);
        }
        acc.x += w * s.x;
        acc.y += w * s.y;
    }
    __shared__ cplx red[8];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        cplx t = mk(0.0, 0.0);
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = cadd(t, red[w]);
        part[2 * blockIdx.x] = t.x;
        part[2 * blockIdx.x + 1] = t.y;
    }
}

__global__ void expect_final(const double* part, double* out) {
    if (threadIdx.x != 0) return;
    double re = 0.0, im = 0.0;
    for (int i = 0; i < OBS_BLOCKS; ++i) {
        re += part[2 * i];
        im += part[2 * i + 1];
    }
    out[0] = re;
    out[1] = im;
}

__global__ void entropy_kernel(const double* lam, int n, double* out) {
    if (threadIdx.x != 0) return;
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
        const double p = lam[i] * lam[i];
        if (p > 0.0) s -= p * log(p);
    }
    *out = s;
}

// ============================================================================ peak probes
constexpr int PROBE_ITERS = 4096;

__global__ void __launch_bounds__(256) probe_dmma_kernel(double* sink, double seed) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
    for (int it = 0; it < PROBE_ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma884(acc[i][0], acc[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) sink[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void probe_dmma_occ_kernel(double* sink, double seed, int iters) {
    double acc[CHAINS][2];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) dmma884(acc[i][0], acc[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) probe_dfma_kernel(double* sink, double seed) {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = seed * i;
    const double a = 1.0000001, b = 1e-12;
    for (int it = 0; it < PROBE_ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.678) sink[threadIdx.x] = s;
}

// DMMA and DFMA issued together: 8 DMMA chains and NF independent DFMA chains per iteration —
// whether the FP64 vector pipe adds throughput beside the FP64 tensor pipe (diagnostic).
template <int NF>
__global__ void __launch_bounds__(256) probe_mixed_kernel(double* sink, double seed) {
    double acc[8][2], f[NF];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = seed * i;
    const double a = seed + threadIdx.x * 1e-9, b = seed * 0.5, fa = 1.0000001, fb = 1e-12;
    for (int it = 0; it < PROBE_ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            dmma884(acc[i][0], acc[i][1], a, b);
#pragma unroll
            for (int j = i * NF / 8; j < (i + 1) * NF / 8; ++j) f[j] = fma(f[j], fa, fb);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
    for (int i = 0; i < NF; ++i) s += f[i];
    if (s == 12345.678) sink[threadIdx.x] = s;
}

}  // namespace

cudaError_t omega_reference(uint64_t seed, long long n_entries, unsigned long long* draws, cplx* out,
                            cudaStream_t s) {
    const long long rounds = (2 * n_entries + MT_N - 1) / MT_N;
    mt_draws_kernel<<<1, 320, 0, s>>>(seed, rounds, draws);
    box_muller_kernel<<<4 * kNumSMs, 256, 0, s>>>(draws, n_entries, out);
    return cudaGetLastError();
}

cudaError_t omega_philox(uint64_t seed, long long n_entries, cplx* out, cudaStream_t s) {
    philox_kernel<<<4 * kNumSMs, 256, 0, s>>>(seed, n_entries, out);
    return cudaGetLastError();
}

cudaError_t gate_small(const cplx* G, int dd, int cl, int cr, const cplx* Min, cplx* Mout, cudaStream_t s) {
    const long long cols = (long long)cl * cr;
    const int grid = (int)std::min<long long>((cols + 255) / 256, 8 * kNumSMs);
    if (dd <= 4) gate_small_kernel<4><<<grid, 256, 0, s>>>(G, dd, cl, cr, Min, Mout);
    else if (dd <= 16) gate_small_kernel<16><<<grid, 256, 0, s>>>(G, dd, cl, cr, Min, Mout);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

cudaError_t theta_to_unfolded(const cplx* theta, int d1, int d2, int cl, int cr, cplx* M, cudaStream_t s) {
    const long long rows = (long long)d1 * d2 * cl;
    theta_unfold_kernel<<<(int)std::min<long long>(rows, 16 * kNumSMs), 128, 0, s>>>(theta, d1, d2, cl, cr, M, 1);
    return cudaGetLastError();
}
cudaError_t unfolded_to_theta(const cplx* M, int d1, int d2, int cl, int cr, cplx* theta, cudaStream_t s) {
    const long long rows = (long long)d1 * d2 * cl;
    theta_unfold_kernel<<<(int)std::min<long long>(rows, 16 * kNumSMs), 128, 0, s>>>(M, d1, d2, cl, cr, theta, 0);
    return cudaGetLastError();
}

cudaError_t truncate(const TruncArgs& a, cudaStream_t s) {
    truncate_kernel<<<1, 32, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t gamma_reshape(const GammaArgs& a, int max_kept, cudaStream_t s) {
    gamma_left_kernel<<<4 * kNumSMs, 256, 0, s>>>(a);
    dim3 grid((a.n + 31) / 32, (max_kept + 31) / 32);
    gamma_right_kernel<<<grid, 256, 0, s>>>(a);
    pinv_flag_kernel<<<1, 256, 0, s>>>(a.ll, a.ll ? a.m / a.d1 : 0, a.lr, a.lr ? a.cr : 0, a.pinv);
    return cudaGetLastError();
}

cudaError_t gate_blocks_many(const GateBlockBatch& b, long long max_cols, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    size_t smem = 0;
    for (int i = 0; i < b.count; ++i) {
        const GateBlocks& g = b.j[i].gb;
        smem = std::max(smem, (size_t)g.total * sizeof(cplx) + (size_t)(g.dd + 2 * g.nblocks + 1) * sizeof(int));
    }
    const dim3 grid((unsigned)((max_cols + 255) / 256), b.count);
    if (smem <= 160 * 1024) {
        cudaError_t e = smem_atleast(reinterpret_cast<const void*>(gate_blocks_staged_kernel), smem);
        if (e != cudaSuccess) return e;
        gate_blocks_staged_kernel<<<grid, 256, smem, s>>>(b);
    } else {
        gate_blocks_kernel<<<grid, 256, 0, s>>>(b);
    }
    return cudaGetLastError();
}

cudaError_t truncate_many(const TruncBatch& b, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    truncate_many_kernel<<<b.count, 32, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t gamma_reshape_many(const GammaBatch& b, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    gamma_left_many_kernel<<<dim3(std::max(1, 4 * kNumSMs / b.count), b.count), 256, 0, s>>>(b);
    gamma_right_many_kernel<<<dim3((b.max_n + 31) / 32, (b.max_kept + 31) / 32, b.count), 256, 0, s>>>(b);
    pinv_many_kernel<<<b.count, 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t omega_philox_many(const PhiloxBatch& b, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    philox_many_kernel<<<dim3(std::max(1, 4 * kNumSMs / b.count), b.count), 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t scale_rows_many(const ScaleRowsBatch& b, cudaStream_t s) {
    if (b.count == 0) return cudaSuccess;
    scale_rows_many_kernel<<<dim3(std::max(1, 4 * kNumSMs / b.count), b.count), 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t fill_int(int* p, int v, cudaStream_t s) {
    fill_int_kernel<<<1, 1, 0, s>>>(p, v);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(256) column_norms2_kernel(const cplx* __restrict__ A, int m, int n,
                                                              double* __restrict__ out) {
    __shared__ double part[8][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, j = blockIdx.x * 32 + tx;
    double a = 0.0;
    if (j < n)
        for (int i = ty; i < m; i += 8) a += cabs2(A[(long long)i * n + j]);
    part[ty][tx] = a;
    __syncthreads();
    if (ty == 0 && j < n) {
        double s = 0.0;
        for (int r = 0; r < 8; ++r) s += part[r][tx];
        out[j] = s;
    }
}

cudaError_t column_norms2(const cplx* A, int m, int n, double* out, cudaStream_t s) {
    column_norms2_kernel<<<(n + 31) / 32, 256, 0, s>>>(A, m, n, out);
    return cudaGetLastError();
}

cudaError_t conj_transpose(const cplx* A, int rows, int cols, cplx* out, cudaStream_t s) {
    dim3 grid((cols + 31) / 32, (rows + 31) / 32);
    conj_transpose_kernel<<<grid, 256, 0, s>>>(A, rows, cols, out);
    return cudaGetLastError();
}

cudaError_t discarded_weight(const double* sigma, int k, const double* total_sq, double* w,
                             cudaStream_t s) {
    weight_kernel<<<1, 32, 0, s>>>(sigma, k, total_sq, w);
    return cudaGetLastError();
}

cudaError_t expectation_local_dev(const cplx* G, int dl, int d, int dr, const double* ll,
                                  const double* lr, const cplx* op, double* res, cudaStream_t s) {
    if (d > 32) return cudaErrorInvalidValue;
    expect_partial<<<OBS_BLOCKS, 256, 0, s>>>(G, dl, d, dr, ll, lr, op, res);
    expect_final<<<1, 32, 0, s>>>(res, res + 2 * OBS_BLOCKS);
    return cudaGetLastError();
}

cudaError_t schmidt_entropy_dev(const double* lam, int n, double* out, cudaStream_t s) {
    entropy_kernel<<<1, 32, 0, s>>>(lam, n, out);
    return cudaGetLastError();
}

// DMMA throughput at a given residency: `warps` warps per SM (one CTA per SM), `chains`
// independent accumulators per warp.  Diagnostics for the zgemm occupancy/ILP trade-off.
cudaError_t probe_dmma_occupancy(int warps, int chains, double* tflops, cudaStream_t s) {
    double* sink = nullptr;
    cudaError_t e = cudaMallocAsync(&sink, 1024 * sizeof(double), s);
    if (e != cudaSuccess) return e;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const int iters = 8192;
    auto launch = [&] {
        switch (chains) {
            case 1: probe_dmma_occ_kernel<1><<<kNumSMs, 32 * warps, 0, s>>>(sink, 1.0, iters); break;
            case 2: probe_dmma_occ_kernel<2><<<kNumSMs, 32 * warps, 0, s>>>(sink, 1.0, iters); break;
            case 4: probe_dmma_occ_kernel<4><<<kNumSMs, 32 * warps, 0, s>>>(sink, 1.0, iters); break;
            default: probe_dmma_occ_kernel<8><<<kNumSMs, 32 * warps, 0, s>>>(sink, 1.0, iters); break;
        }
    };
    launch();
    cudaEventRecord(t0, s);
    launch();
    cudaEventRecord(t1, s);
    e = cudaEventSynchronize(t1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    const int ch = (chains == 1 || chains == 2 || chains == 4) ? chains : 8;
    *tflops = (double)kNumSMs * warps * iters * ch * 512.0 / (ms * 1e-3) / 1e12;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaFreeAsync(sink, s);
    return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t probe_peak(int what, double* tflops, cudaStream_t s) {
    double* sink = nullptr;
    cudaError_t e = cudaMallocAsync(&sink, 256 * sizeof(double), s);
    if (e != cudaSuccess) return e;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const int grid = 8 * kNumSMs;
    for (int rep = 0; rep < 2; ++rep) {  // first launch warms clocks
        cudaEventRecord(t0, s);
        if (what == 0) probe_dmma_kernel<<<grid, 256, 0, s>>>(sink, 1.0);
        else if (what == 1) probe_dfma_kernel<<<grid, 256, 0, s>>>(sink, 1.0);
        else if (what == 2) probe_mixed_kernel<8><<<grid, 256, 0, s>>>(sink, 1.0);
        else if (what == 3) probe_mixed_kernel<16><<<grid, 256, 0, s>>>(sink, 1.0);
        else probe_mixed_kernel<32><<<grid, 256, 0, s>>>(sink, 1.0);
        cudaEventRecord(t1, s);
    }
    e = cudaEventSynchronize(t1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    const double warps = grid * 8.0;
    const double nf = what == 2 ? 8.0 : what == 3 ? 16.0 : 32.0;
    const double flops = (what == 0) ? warps * PROBE_ITERS * 8.0 * 512.0
                         : (what == 1) ? warps * 32.0 * PROBE_ITERS * 8.0 * 2.0
                                       : warps * PROBE_ITERS * (8.0 * 512.0 + 32.0 * nf * 2.0);
    *tflops = flops / (ms * 1e-3) / 1e12;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaFreeAsync(sink, s);
    return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace rb

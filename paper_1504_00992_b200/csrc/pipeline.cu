// pipeline.cu — see pipeline.cuh.
#include <algorithm>
#include <string>

#include "pipeline.cuh"

namespace rb {

void gemm(rrsvd_b200_ctx* c, GemmOp opA, int m, int n, int k, const cplx* A, long long lda,
          const cplx* B, long long ldb, cplx* C, long long ldc, const Scale& sc, int batch,
          long long sA, long long sB, long long sC) {
    if (m <= 0 || n <= 0) return;
    GemmGroup g;
    g.count = 1;
    GemmProblem& P = g.p[0];
    P = GemmProblem{};
    P.m = m; P.n = n; P.k = k; P.batch = batch;
    P.A = A; P.lda = lda; P.strideA = sA;
    P.B = B; P.ldb = ldb; P.strideB = sB;
    P.C = C; P.ldc = ldc; P.strideC = sC;
    P.rs = sc.rs; P.rs_div = sc.rs_div; P.ks = sc.ks; P.cs = sc.cs; P.cs_mod = sc.cs_mod;
    const long long tiles = (long long)((m + 63) / 64) * ((n + 63) / 64) * batch;
    int split = 1;
    const long long target = 2 * kNumSMs;
    if (tiles < target && k > 128) {
        split = (int)std::min<long long>((target + tiles - 1) / tiles, (k + 63) / 64);
        split = std::max(split, 1);
    }
    P.split = split;
    if (split > 1) P.partial = ws_get<cplx>(c, (size_t)split * batch * m * n);
    check_cuda(c, zgemm_grouped(g, opA, c->stream), "zgemm");
    c->launches += split > 1 ? 2 : 1;
}

void orth(rrsvd_b200_ctx* c, const cplx* Y, int m, int l, cplx* Q, int* ndead) {
    if (l > kMaxCholL)
        throw_contract(c, "orth: sketch width l = " + std::to_string(l) + " exceeds the supported " +
                              std::to_string(kMaxCholL));
    if (m < l) throw_contract(c, "qr: requires rows >= cols");
    cplx* G = ws_get<cplx>(c, (size_t)l * l);
    cplx* T = ws_get<cplx>(c, (size_t)l * l);
    cplx* bufA = ws_get<cplx>(c, (size_t)m * l);
    cplx* bufB = ws_get<cplx>(c, (size_t)m * l);
    const cplx* cur = Y;
    for (int pass = 0; pass < 3; ++pass) {
        gemm(c, kOpC, l, l, m, cur, l, cur, l, G, l);
        CholBatch cb{};
        cb.count = 1;
        cb.l[0] = l;
        cb.G[0] = G;
        cb.T[0] = T;
        cb.shift_scale[0] = pass == 0 ? 10.0 * (m + l) : 0.0;
        cb.ndead[0] = pass == 2 ? ndead : nullptr;
        check_cuda(c, chol_inv(cb, l, c->stream), "chol_inv");
        c->launches++;
        cplx* dst = pass == 2 ? Q : (pass == 0 ? bufA : bufB);
        gemm(c, kOpN, m, l, l, cur, l, T, l, dst, l);
        cur = dst;
    }
}

void make_omega(rrsvd_b200_ctx* c, int n, int l, uint64_t seed, int mode, cplx* out) {
    const long long entries = (long long)n * l;
    if (mode == 0) {
        const long long rounds = (2 * entries + 311) / 312;
        auto* draws = ws_get<unsigned long long>(c, (size_t)rounds * 312);
        check_cuda(c, omega_reference(seed, entries, draws, out, c->stream), "omega_reference");
        c->launches += 2;
    } else if (mode == 1) {
        check_cuda(c, omega_philox(seed, entries, out, c->stream), "omega_philox");
        c->launches++;
    } else {
        throw_contract(c, "unknown omega mode");
    }
}

static void small_svd(rrsvd_b200_ctx* c, const cplx* X, int r, int cc, int adj, int lda,
                      double* sigma, cplx* Xn, cplx* Js) {
    cplx* W = ws_get<cplx>(c, (size_t)(r + cc) * cc);
    JacobiInitBatch ib{};
    ib.count = 1;
    ib.r[0] = r; ib.c[0] = cc; ib.A[0] = X; ib.lda[0] = lda; ib.adj[0] = adj; ib.W[0] = W;
    check_cuda(c, jacobi_init(ib, c->stream), "jacobi_init");
    JacobiBatch jb{};
    jb.count = 1;
    jb.r[0] = r; jb.c[0] = cc; jb.W[0] = W; jb.sweeps[0] = nullptr;
    const cudaError_t e = jacobi_svd(jb, r, cc, c->stream);
    if (e == cudaErrorInvalidValue)
        throw_contract(c, "jacobi: matrix " + std::to_string(r) + "x" + std::to_string(cc) +
                              " exceeds the on-chip Jacobi capacity");
    check_cuda(c, e, "jacobi_svd");
    JacobiFinBatch fb{};
    fb.count = 1;
    fb.r[0] = r; fb.c[0] = cc; fb.W[0] = W; fb.sigma[0] = sigma; fb.Xn[0] = Xn; fb.Js[0] = Js;
    check_cuda(c, jacobi_finish(fb, cc, c->stream), "jacobi_finish");
    c->launches += 3;
}

void rrsvd_core(rrsvd_b200_ctx* c, const cplx* A, int m, int n, int l, int q, const cplx* omega,
                cplx* U, double* sigma, cplx* V) {
    cplx* Y = ws_get<cplx>(c, (size_t)m * l);
    cplx* Q = ws_get<cplx>(c, (size_t)m * l);
    cplx* Z = ws_get<cplx>(c, (size_t)n * l);
    cplx* Qb = ws_get<cplx>(c, (size_t)n * l);
    cplx* X = ws_get<cplx>(c, (size_t)l * l);
    cplx* Xn = ws_get<cplx>(c, (size_t)l * l);
    cplx* Js = ws_get<cplx>(c, (size_t)l * l);
    // range finder, Algorithm 1 (randomized.cpp:88-99)
    gemm(c, kOpN, m, l, n, A, n, omega, l, Y, l);            // Y = A Omega
    orth(c, Y, m, l, Q);
    for (int j = 0; j < q; ++j) {
        gemm(c, kOpC, n, l, m, A, n, Q, l, Z, l);            // Z = A^H Q
        orth(c, Z, n, l, Qb);
        gemm(c, kOpN, m, l, n, A, n, Qb, l, Y, l);           // Y = A Q~
        orth(c, Y, m, l, Q);
    }
    // B = Q^H A, held as B^H = A^H Q = Qb X  (assemble_from_basis, randomized.cpp:57-66)
    gemm(c, kOpC, n, l, m, A, n, Q, l, Z, l);
    orth(c, Z, n, l, Qb);
    gemm(c, kOpC, l, l, n, Qb, l, Z, l, X, l);               // X = Qb^H B^H  (l x l)
    // X J = U_X Sigma  =>  B = J Sigma (Qb U_X)^H
    small_svd(c, X, l, l, 0, l, sigma, Xn, Js);
    gemm(c, kOpN, m, l, l, Q, l, Js, l, U, l);               // U = Q U_B
    gemm(c, kOpN, n, l, l, Qb, l, Xn, l, V, l);              // V = Qb U_X
}

void svd_jacobi(rrsvd_b200_ctx* c, const cplx* A, int m, int n, cplx* U, double* sigma, cplx* V) {
    const bool tall = m >= n;
    const int r = tall ? m : n, cc = tall ? n : m;
    // Direct one-sided Jacobi when the block pair fits on chip; else precondition with a QR.
    const int ld = r + cc;
    const int bs16 = (cc + 31) / 32;
    const bool direct = (size_t)2 * bs16 * ld * sizeof(cplx) <= 200 * 1024 && r <= 4 * cc;
    if (direct) {
        // tall: X = A, X J = U S -> U = Xn, V = J.   wide: X = A^H -> V = Xn, U = J.
        small_svd(c, A, r, cc, tall ? 0 : 1, n, sigma, tall ? U : V, tall ? V : U);
        return;
    }
    // X (r x cc) = A or A^H explicitly, X = Qr R, R J = U_R S  =>  X = (Qr U_R) S J^H
    const cplx* X = A;
    if (!tall) {
        cplx* Xt = ws_get<cplx>(c, (size_t)r * cc);
        check_cuda(c, conj_transpose(A, m, n, Xt, c->stream), "conj_transpose");
        c->launches++;
        X = Xt;
    }
    cplx* Qr = ws_get<cplx>(c, (size_t)r * cc);
    cplx* R = ws_get<cplx>(c, (size_t)cc * cc);
    cplx* Un = ws_get<cplx>(c, (size_t)cc * cc);
    orth(c, X, r, cc, Qr);
    gemm(c, kOpC, cc, cc, r, Qr, cc, X, cc, R, cc);
    cplx* Jo = tall ? V : U;
    small_svd(c, R, cc, cc, 0, cc, sigma, Un, Jo);
    gemm(c, kOpN, r, cc, cc, Qr, cc, Un, cc, tall ? U : V, cc);
}

}  // namespace rb

// pipeline.cu — see pipeline.cuh.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
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
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (c->gemm_timing) {
        ea = pooled_event(c);
        eb = pooled_event(c);
        check_cuda(c, cudaEventRecord(ea, c->stream), "event record");
    }
    check_cuda(c, zgemm_grouped(g, opA, c->stream), "zgemm");
    c->launches += split > 1 ? 2 : 1;
    if (c->gemm_timing) {
        check_cuda(c, cudaEventRecord(eb, c->stream), "event record");
        c->pending.push_back({ea, eb, 8.0 * m * n * (double)k * batch});
    }
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
        cb.dep_tol[0] = pass == 0 ? 0.0 : kDepTol;
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
    static const bool debug = std::getenv("RRSVD_B200_DEBUG") != nullptr;
    int* dsweeps = nullptr;
    if (debug) {
        dsweeps = ws_get<int>(c, 1);
        jb.sweeps[0] = dsweeps;
    }
    const cudaError_t e = jacobi_svd(jb, r, cc, c->stream);
    if (e == cudaErrorInvalidValue)
        throw_contract(c, "jacobi: matrix " + std::to_string(r) + "x" + std::to_string(cc) +
                              " exceeds the on-chip Jacobi capacity");
    check_cuda(c, e, "jacobi_svd");
    if (debug) {
        int h = -1;
        cudaMemcpyAsync(&h, dsweeps, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
        cudaStreamSynchronize(c->stream);
        std::fprintf(stderr, "[rrsvd_b200] jacobi %dx%d: %d sweeps\n", r, cc, h);
    }
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
    gemm(c, kOpC, l, l, n, Qb, l, Z, l, X, l);               // X = Qb^H B^H  (l x l, ~upper)
    // B = X^H Qb^H.  One-sided Jacobi on X^H (the R^H of a QR converges in a few sweeps,
    // Drmac-Veselic): X^H K = Z Sigma  =>  B = Z Sigma (Qb K)^H, so U_B = Z, V = Qb K.
    small_svd(c, X, l, l, 1, l, sigma, Xn, Js);
    gemm(c, kOpN, m, l, l, Q, l, Xn, l, U, l);               // U = Q U_B
    gemm(c, kOpN, n, l, l, Qb, l, Js, l, V, l);              // V = Qb K
}

DecimPlan plan_decimation(int d1, int d2, int cl, int cr, size_t chi_max, int kind, size_t target_rank,
                          size_t oversampling, size_t det_crossover) {
    DecimPlan p{};
    p.m = d1 * cl;
    p.n = d2 * cr;
    p.minor = std::min(p.m, p.n);
    const size_t k = target_rank != 0 ? target_rank : chi_max;
    p.randomized = kind == 1 && k != 0 && (size_t)p.minor > det_crossover;  // tebd.cpp:167-169
    p.ns = p.minor;
    p.l = 0;
    if (p.randomized) {
        const size_t pp = oversampling != 0 ? oversampling : k;            // tebd.cpp:171
        p.l = (int)std::min<size_t>(k + pp, (size_t)p.minor);              // tebd.cpp:172
        p.ns = p.l;
    }
    p.kmax = p.ns;
    if (chi_max != 0) p.kmax = (int)std::min<size_t>((size_t)p.kmax, chi_max);
    return p;
}

void build_theta_device(rrsvd_b200_ctx* c, const cplx* G1, const cplx* G2, const double* ll,
                        const double* lm, const double* lr, int cl, int d1, int cm, int d2, int cr, cplx* M) {
    const int m = cl * d1, n = d2 * cr;
    Scale sc;
    sc.rs = ll; sc.rs_div = d1; sc.ks = lm; sc.cs = lr; sc.cs_mod = cr;
    gemm(c, kOpN, m, n, cm, G1, cm, G2, n, M, n, sc);
}

void apply_gate_device(rrsvd_b200_ctx* c, const cplx* G, int d1, int d2, int cl, int cr,
                       const cplx* Min, cplx* Mout) {
    const int dd = d1 * d2;
    if (dd <= 16) {
        check_cuda(c, gate_small(G, dd, cl, cr, Min, Mout, c->stream), "gate_small");
        c->launches++;
    } else {
        gemm(c, kOpN, dd, cr, dd, G, dd, Min, cr, Mout, cr, {}, cl, 0, (long long)dd * cr,
             (long long)dd * cr);
    }
}

void decimate_device(rrsvd_b200_ctx* c, const DecimPlan& pl, const cplx* M, int d1, int cr,
                     const double* ll, const double* lr, size_t chi_max, double trunc_tol, int q,
                     uint64_t call_seed, int omega_mode, const cplx* omega, int renormalize,
                     cplx* gamma_l, double* lambda, cplx* gamma_r, DecimScalars* sc) {
    const int m = pl.m, n = pl.n, ns = pl.ns;
    double* part = ws_get<double>(c, 2 * kNumSMs);
    int* bad = ws_get<int>(c, 2 * kNumSMs);
    check_cuda(c, sumsq(M, (long long)m * n, part, bad, &sc->total_sq, &sc->nonfinite, c->stream), "sumsq");
    c->launches += 2;
    cplx* U = ws_get<cplx>(c, (size_t)m * ns);
    cplx* V = ws_get<cplx>(c, (size_t)n * ns);
    double* sig = ws_get<double>(c, ns);
    if (pl.randomized) {
        const cplx* om = omega;
        if (om == nullptr) {
            cplx* o = ws_get<cplx>(c, (size_t)n * pl.l);
            make_omega(c, n, pl.l, call_seed, omega_mode, o);
            om = o;
        }
        rrsvd_core(c, M, m, n, pl.l, q, om, U, sig, V);
    } else {
        svd_jacobi(c, M, m, n, U, sig, V);
    }
    TruncArgs ta{};
    ta.sigma = sig; ta.ns = ns; ta.total_sq = &sc->total_sq; ta.trunc_tol = trunc_tol;
    ta.cap = (long long)chi_max; ta.renormalize = renormalize; ta.kept = &sc->kept;
    ta.lambda = lambda; ta.discarded = &sc->discarded;
    check_cuda(c, truncate(ta, c->stream), "truncate");
    GammaArgs ga{};
    ga.U = U; ga.ldu = ns; ga.V = V; ga.ldv = ns; ga.ll = ll; ga.lr = lr;
    ga.m = m; ga.n = n; ga.d1 = d1; ga.cr = cr; ga.kept = &sc->kept;
    ga.gamma_l = gamma_l; ga.gamma_r = gamma_r; ga.pinv = &sc->pinv;
    check_cuda(c, gamma_reshape(ga, pl.kmax, c->stream), "gamma_reshape");
    c->launches += 4;
}

void svd_jacobi(rrsvd_b200_ctx* c, const cplx* A, int m, int n, cplx* U, double* sigma, cplx* V) {
    const bool tall = m >= n;
    const int r = tall ? m : n, cc = tall ? n : m;
    if (cc > kMaxCholL) {
        // Unpreconditioned one-sided Jacobi (converges, but in more sweeps).
        // tall: X = A, X J = U S -> U = Xn, V = J.   wide: X = A^H -> V = Xn, U = J.
        small_svd(c, A, r, cc, tall ? 0 : 1, n, sigma, tall ? U : V, tall ? V : U);
        return;
    }
    // QR-preconditioned Jacobi: X (r x cc) = A or A^H, X = Qr R, R^H K = Z S
    //   =>  X = (Qr K) S Z^H : left vectors Qr K, right vectors Z.
    const cplx* X = A;
    if (!tall) {
        cplx* Xt = ws_get<cplx>(c, (size_t)r * cc);
        check_cuda(c, conj_transpose(A, m, n, Xt, c->stream), "conj_transpose");
        c->launches++;
        X = Xt;
    }
    cplx* Qr = ws_get<cplx>(c, (size_t)r * cc);
    cplx* R = ws_get<cplx>(c, (size_t)cc * cc);
    cplx* K = ws_get<cplx>(c, (size_t)cc * cc);
    orth(c, X, r, cc, Qr);
    gemm(c, kOpC, cc, cc, r, Qr, cc, X, cc, R, cc);
    small_svd(c, R, cc, cc, 1, cc, sigma, tall ? V : U, K);
    gemm(c, kOpN, r, cc, cc, Qr, cc, K, cc, tall ? U : V, cc);
}

}  // namespace rb

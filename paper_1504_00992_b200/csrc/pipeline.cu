// pipeline.cu — batched orchestration of the decimation pipeline.  See pipeline.cuh.
#include <cstring>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "pipeline.cuh"

namespace rb {

bool debug_enabled() {
    static const bool d = [] {
        const char* e = std::getenv("RRSVD_B200_DEBUG");
        return e != nullptr && e[0] != '\0' && e[0] != '0';
    }();
    return d;
}

namespace {

long long gemm_tiles(const GemmSpec& s) {
    return (long long)((s.m + 63) / 64) * ((s.n + 63) / 64) * s.batch;
}

}  // namespace

// ================================================================================== GEMM

void gemm_many(rrsvd_b200_ctx* c, GemmOp opA, const std::vector<GemmSpec>& specs) {
    long long total = 0;
    for (const GemmSpec& s : specs)
        if (s.m > 0 && s.n > 0) total += gemm_tiles(s);
    if (total == 0) return;
    // Split K when the group has too few tiles: aim for >= 2 waves of 2 CTAs/SM (4 CTAs per SM;
    // 8 measured slower on the C3 QR Gram matrices — 26.8 vs 29.1 TF/s — from the shorter K per
    // split and the larger reduction).
    static const long long waves = [] {  // RRSVD_B200_SPLIT_WAVES: split-K target in CTAs per SM (A/B)
        const char* e = std::getenv("RRSVD_B200_SPLIT_WAVES");
        return e ? std::max(1, std::atoi(e)) : 4;
    }();
    const long long target = waves * kNumSMs;
    for (size_t base = 0; base < specs.size(); base += kMaxGroup) {
        GemmGroup g;
        g.count = 0;
        g.used_m3 = g.used_tma = 0;
        double flops = 0.0;
        bool any_split = false;
        for (size_t i = base; i < std::min(specs.size(), base + kMaxGroup); ++i) {
            const GemmSpec& s = specs[i];
            if (s.m <= 0 || s.n <= 0) continue;
            GemmProblem& P = g.p[g.count++];
            P = GemmProblem{};
            P.m = s.m; P.n = s.n; P.k = s.k; P.batch = s.batch;
            P.A = s.A; P.lda = s.lda; P.strideA = s.sA;
            P.B = s.B; P.ldb = s.ldb; P.strideB = s.sB;
            P.C = s.C; P.ldc = s.ldc; P.strideC = s.sC;
            P.rs = s.sc.rs; P.rs_div = s.sc.rs_div; P.ks = s.sc.ks; P.cs = s.sc.cs; P.cs_mod = s.sc.cs_mod;
            P.structure = s.structure;
            P.nsub = s.nsub;
            P.subB = s.subB;
            P.subC = s.subC;
            P.D = s.D; P.ldd = s.ldd; P.alpha = s.alpha;
            P.pred = s.pred; P.pred_want = s.pred_want;
            int split = 1;
            if (total < target && s.k > 128) {
                split = (int)std::min<long long>((target + total - 1) / total, (s.k + 63) / 64);
                split = std::max(split, 1);
            }
            P.split = split;
            if (split > 1) {
                P.partial = ws_get<cplx>(c, (size_t)split * s.batch * s.m * s.n);
                any_split = true;
            }
            // a predicated problem may not run: its flops are left out of the roofline (its
            // launch time still counts — conservative)
            if (s.pred == nullptr) flops += 8.0 * s.m * s.n * (double)s.k * s.batch;
        }
        if (g.count == 0) continue;
        cudaEvent_t ea = nullptr, eb = nullptr;
        if (c->gemm_timing) {
            ea = pooled_event(c);
            eb = pooled_event(c);
            check_cuda(c, cudaEventRecord(ea, c->stream), "event record");
        }
        check_cuda(c, zgemm_grouped(g, opA, c->stream), "zgemm");
        c->launches += any_split ? 2 : 1;
        if (c->gemm_timing) {
            check_cuda(c, cudaEventRecord(eb, c->stream), "event record");
            c->pending.push_back({ea, eb, flops, g.used_m3 ? 0.75 * flops : flops, c->gemm_tag, g.used_tma});
        }
    }
}

void gemm(rrsvd_b200_ctx* c, GemmOp opA, int m, int n, int k, const cplx* A, long long lda,
          const cplx* B, long long ldb, cplx* C, long long ldc, const Scale& sc, int batch,
          long long sA, long long sB, long long sC) {
    GemmSpec s{m, n, k, A, lda, B, ldb, C, ldc, sc, batch, sA, sB, sC};
    gemm_many(c, opA, {s});
}

// ================================================================================== orth

// Widths beyond the single-CTA Cholesky (l > kMaxCholL) are blocked: nbk diagonal blocks of
// width <= kMaxCholL, right-looking over the Gram matrix (updated in place),
//   T_JJ = chol_inv(G_JJ),  R_J,>J = T_JJ^H G_J,>J,  G_>J,>J -= R_J,>J^H R_J,>J,
// then the inverse's off-diagonal blocks bottom-up,  T_I,>I = -T_II (R_I,>I T_>I,>I).
// The shift is taken once from the trace of the whole (unmodified) G by block 0, so this is
// the same factorization as the unblocked kernel up to rounding order.
struct CholBlocking {
    int nbk = 1, bsz = 0;
    int begin(int J) const { return J * bsz; }
    int width(int J, int l) const { return std::min(bsz, l - J * bsz); }
};
CholBlocking chol_blocking(int l) {
    CholBlocking cbk;
    cbk.nbk = (l + kMaxCholL - 1) / kMaxCholL;
    cbk.bsz = ((l + cbk.nbk - 1) / cbk.nbk + 7) / 8 * 8;
    cbk.nbk = (l + cbk.bsz - 1) / cbk.bsz;
    return cbk;
}

void chol_inv_many(rrsvd_b200_ctx* c, const std::vector<CholSpec>& specs) {
    if (specs.empty()) return;
    struct Buf {
        CholBlocking blk;
        cplx *R, *W;  // blocked path only
        double* shift;
    };
    std::vector<Buf> bufs(specs.size());
    int max_nbk = 1;
    for (size_t i = 0; i < specs.size(); ++i) {
        const CholSpec& s = specs[i];
        Buf& b = bufs[i];
        b.blk = chol_blocking(s.l);
        b.R = b.W = nullptr;
        b.shift = nullptr;
        if (b.blk.nbk > 1) {
            b.R = ws_get<cplx>(c, (size_t)s.l * s.l);
            b.W = ws_get<cplx>(c, (size_t)b.blk.bsz * s.l);
            b.shift = ws_get<double>(c, 1);
            // the strictly lower blocks of T are never written
            check_cuda(c, cudaMemsetAsync(s.T, 0, (size_t)s.l * s.l * sizeof(cplx), c->stream), "memset");
            max_nbk = std::max(max_nbk, b.blk.nbk);
        }
    }
    auto chol_launch = [&](CholBatch& cb, int max_l) {
        check_cuda(c, chol_inv(cb, max_l, c->stream), "chol_inv");
        c->launches++;
        cb = CholBatch{};
    };
    auto off = [](int l, int r0, int c0) { return (size_t)r0 * l + c0; };
    for (int J = 0; J < max_nbk; ++J) {
        CholBatch cb{};
        int max_l = 0;
        for (size_t i = 0; i < specs.size(); ++i) {
            const CholSpec& s = specs[i];
            const Buf& b = bufs[i];
            if (J >= b.blk.nbk) continue;
            const int j0 = b.blk.begin(J), w = b.blk.width(J, s.l);
            const int k = cb.count++;
            cb.l[k] = w;
            cb.G[k] = s.G + off(s.l, j0, j0);
            cb.ldg[k] = s.l;
            cb.trace_src[k] = s.G; cb.trace_n[k] = s.l; cb.trace_ld[k] = s.l;
            if (b.blk.nbk > 1) {
                if (J == 0) cb.shift_save[k] = b.shift;
                else cb.shift_use[k] = b.shift;
            }
            cb.T[k] = s.T + off(s.l, j0, j0);
            cb.ldt[k] = s.l;
            cb.shift_scale[k] = s.shift_scale;
            cb.dep_tol[k] = 0.0;
            cb.ndead[k] = s.ndead;
            cb.ndead_acc[k] = J > 0 ? 1 : 0;
            cb.ill_out[k] = s.ill_out;
            cb.pred[k] = s.pred;
            max_l = std::max(max_l, w);
            if (cb.count == kMaxSmall) { chol_launch(cb, max_l); max_l = 0; }
        }
        if (cb.count) chol_launch(cb, max_l);
        std::vector<GemmSpec> g1, g2;
        for (size_t i = 0; i < specs.size(); ++i) {
            const CholSpec& s = specs[i];
            const Buf& b = bufs[i];
            if (J + 1 >= b.blk.nbk) continue;
            const int j0 = b.blk.begin(J), w = b.blk.width(J, s.l), r0 = j0 + w, rest = s.l - r0;
            // R_J,>J = T_JJ^H G_J,>J
            g1.push_back({w, rest, w, s.T + off(s.l, j0, j0), s.l, s.G + off(s.l, j0, r0), s.l,
                          b.R + off(s.l, j0, r0), s.l});
            // G_>J,>J -= R_J,>J^H R_J,>J  (upper part, in place)
            GemmSpec up{rest, rest, w, b.R + off(s.l, j0, r0), s.l, b.R + off(s.l, j0, r0), s.l,
                        s.G + off(s.l, r0, r0), s.l};
            up.structure = kUpperC;
            up.D = s.G + off(s.l, r0, r0);
            up.ldd = s.l;
            up.alpha = -1.0;
            if (s.pred) { g1.back().pred = s.pred; up.pred = s.pred; }
            g2.push_back(up);
        }
        if (!g1.empty()) {
            c->gemm_tag = 3;
            gemm_many(c, kOpC, g1);
            gemm_many(c, kOpC, g2);
        }
    }
    for (int I = max_nbk - 2; I >= 0; --I) {
        std::vector<GemmSpec> g1, g2;
        for (size_t i = 0; i < specs.size(); ++i) {
            const CholSpec& s = specs[i];
            const Buf& b = bufs[i];
            if (I + 1 >= b.blk.nbk) continue;
            const int i0 = b.blk.begin(I), w = b.blk.width(I, s.l), r0 = i0 + w, rest = s.l - r0;
            // W = R_I,>I T_>I,>I  (T upper triangular)
            GemmSpec ws{w, rest, rest, b.R + off(s.l, i0, r0), s.l, s.T + off(s.l, r0, r0), s.l, b.W, rest};
            ws.structure = kTriB;
            g1.push_back(ws);
            // T_I,>I = -T_II W
            GemmSpec ts{w, rest, w, s.T + off(s.l, i0, i0), s.l, b.W, rest, s.T + off(s.l, i0, r0), s.l};
            ts.alpha = -1.0;
            if (s.pred) { g1.back().pred = s.pred; ts.pred = s.pred; }
            g2.push_back(ts);
        }
        if (!g1.empty()) {
            c->gemm_tag = 4;
            gemm_many(c, kOpN, g1);
            gemm_many(c, kOpN, g2);
        }
    }
}

// Adaptive schedule (any width): the first, shifted pass also reports whether some
// pivot fell within kIllRatio of the shift (cond(Y) beyond what one shifted pass resolves,
// rank deficiency included).  Only then do the robust schedule's extra passes run — predicated
// on that device flag, so the host never waits:
//   full (kFullPasses):  shifted Y->a | [ill] shifted a->b, plain b->a | plain a->Q
//   span (kSpanPasses):  shifted Y->a | [ill] shifted a->b              | Q = ill ? b : a
//   robust span (kRobustSpanPasses): shifted Y->a | [ill] shifted a->b, [ill] plain b->a,
//                        [ill] plain a->b | Q = ill ? b : a  (RRSVD_B200_ROBUST_PASSES=3: without
//                        the second shifted pass, Q = a)
// A well-conditioned basis thus costs 2 (full) or 1 (span) passes instead of 4 or 2, with the
// same guarantees: after a shifted pass with every pivot >= 1e4 s, cond(Q) - 1 <= 5e-5.
void orth_many_adaptive(rrsvd_b200_ctx* c, const std::vector<OrthSpec>& specs, bool full, bool robust) {
    const size_t np = specs.size();
    struct Buf {
        cplx *G, *T, *a, *b;
        const cplx* y;
    };
    std::vector<Buf> bufs(np);
    int* ill = ws_get<int>(c, np);
    for (size_t i = 0; i < np; ++i) {
        const OrthSpec& s = specs[i];
        if (s.m < s.l) throw_contract(c, "qr: requires rows >= cols");
        bufs[i] = {ws_get<cplx>(c, (size_t)s.l * s.l), ws_get<cplx>(c, (size_t)s.l * s.l),
                   ws_get<cplx>(c, (size_t)s.m * s.l), ws_get<cplx>(c, (size_t)s.m * s.l), s.Y};
    }
    // debug: dead-pivot counts of every pass (RRSVD_B200_DEBUG)
    const bool dbg = debug_enabled();
    int* dbg_dead = dbg ? ws_get<int>(c, 4 * np) : nullptr;
    int pass_no = 0;
    if (dbg) check_cuda(c, cudaMemsetAsync(dbg_dead, 0, 4 * np * sizeof(int), c->stream), "memset");
    // one pass for every problem: Gram, chol_inv (any width), apply  (pred: run only if *pred != 0)
    auto pass = [&](bool shifted, std::vector<const cplx*> src, std::vector<cplx*> dst, bool first,
                     const int* pred_base, bool last) {
        std::vector<GemmSpec> gram, apply;
        std::vector<CholSpec> chol;
        for (size_t i = 0; i < np; ++i) {
            const OrthSpec& s = specs[i];
            GemmSpec gs{s.l, s.l, s.m, src[i], s.l, src[i], s.l, bufs[i].G, s.l};
            gs.structure = kUpperC;
            if (pred_base) gs.pred = pred_base + i;
            gram.push_back(gs);
            CholSpec cs{bufs[i].G, s.l, shifted ? 10.0 * (s.m + s.l) : 0.0, bufs[i].T,
                        last && !dbg ? s.ndead : (dbg ? dbg_dead + 4 * i + pass_no : nullptr)};
            cs.ill_out = first ? ill + i : nullptr;
            cs.pred = pred_base ? pred_base + i : nullptr;
            chol.push_back(cs);
            GemmSpec as{s.m, s.l, s.l, src[i], s.l, bufs[i].T, s.l, dst[i], s.l};
            as.structure = kTriB;
            if (pred_base) as.pred = pred_base + i;
            apply.push_back(as);
        }
        c->gemm_tag = 3;
        gemm_many(c, kOpC, gram);
        chol_inv_many(c, chol);
        c->gemm_tag = 4;
        gemm_many(c, kOpN, apply);
        ++pass_no;
    };
    std::vector<const cplx*> Y(np), A(np), B(np);
    std::vector<cplx*> Aw(np), Bw(np), Q(np);
    for (size_t i = 0; i < np; ++i) {
        Y[i] = specs[i].Y; A[i] = Aw[i] = bufs[i].a; B[i] = Bw[i] = bufs[i].b; Q[i] = specs[i].Q;
    }
    check_cuda(c, cudaMemsetAsync(ill, 0, np * sizeof(int), c->stream), "memset");
    // the robust span schedule: shifted | [ill] shifted, plain, plain; RRSVD_B200_ROBUST_PASSES=3
    // drops the second shifted pass (shifted CholeskyQR3, Fukaya et al.: C3 10.97 vs 10.70 steps/s,
    // but the d = 20 TEDOPA trace with 16 moduli on every bond >= 256 then loses chi at a
    // noise-level tail — test_emulated_products_on_every_bond_shape — so four is the default)
    static const bool robust3 = [] {
        const char* e = std::getenv("RRSVD_B200_ROBUST_PASSES");
        return e != nullptr && std::atoi(e) == 3;
    }();
    bool inplace = false;  // (Y == Q: the first pass must not write its own input)
    for (const OrthSpec& s : specs) inplace = inplace || s.Y == s.Q;
    if (!full && robust && !inplace) {
        // the robust span schedule ends in Q whichever way the flag goes (no select copy):
        // shifted Y -> Q | [ill] shifted Q -> b, plain b -> a, plain a -> Q  (robust3: [ill] plain
        // Q -> b, plain b -> Q) — the same passes as the a / b form, with Q as the first buffer
        std::vector<const cplx*> Qc(Q.begin(), Q.end());
        pass(true, Y, Q, true, nullptr, false);
        if (robust3) {
            pass(false, Qc, Bw, false, ill, false);
            pass(false, B, Q, false, ill, true);
        } else {
            pass(true, Qc, Bw, false, ill, false);
            pass(false, B, Aw, false, ill, false);
            pass(false, A, Q, false, ill, true);
        }
        return;
    }
    pass(true, Y, Aw, true, nullptr, false);             // shifted Y -> a, flags
    if (!full && robust && robust3) {                    // [ill] plain a -> b, [ill] plain b -> a
        pass(false, A, Bw, false, ill, false);
        pass(false, B, Aw, false, ill, true);
    } else {
        pass(true, A, Bw, false, ill, false);            // [ill] shifted a -> b
    }
    if (!full && robust && !robust3) {                   // [ill] plain b -> a, [ill] plain a -> b
        pass(false, B, Aw, false, ill, false);
        pass(false, A, Bw, false, ill, true);
    }
    if (full) {
        pass(false, B, Aw, false, ill, false);           // [ill] plain b -> a
        pass(false, A, Q, false, nullptr, true);         // plain a -> Q
        if (dbg) {
            std::vector<int> h(4 * np), hi(np);
            cudaMemcpyAsync(h.data(), dbg_dead, h.size() * sizeof(int), cudaMemcpyDeviceToHost, c->stream);
            cudaMemcpyAsync(hi.data(), ill, hi.size() * sizeof(int), cudaMemcpyDeviceToHost, c->stream);
            cudaStreamSynchronize(c->stream);
            for (size_t i = 0; i < np; ++i)
                std::fprintf(stderr, "[rrsvd_b200] orth full %dx%d: ill %d, dead per pass %d %d %d %d\n", specs[i].m,
                             specs[i].l, hi[i], h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
            for (size_t i = 0; i < np; ++i)  // (the caller's ndead: the last pass)
                if (specs[i].ndead)
                    cudaMemcpyAsync(specs[i].ndead, dbg_dead + 4 * i + 3, sizeof(int), cudaMemcpyDeviceToDevice, c->stream);
        }
    } else {
        for (size_t base = 0; base < np; base += kMaxSmall) {  // Q = ill ? b : a
            SelectBatch sb{};
            for (size_t i = base; i < std::min(np, base + kMaxSmall); ++i) {
                const int k = sb.count++;
                sb.flag[k] = ill + i; sb.A[k] = bufs[i].a; sb.B[k] = (robust && robust3) ? bufs[i].a : bufs[i].b;
                sb.Q[k] = specs[i].Q;
                sb.n[k] = (long long)specs[i].m * specs[i].l;
            }
            check_cuda(c, select_many(sb, c->stream), "select");
            c->launches++;
        }
    }
}

void orth_many(rrsvd_b200_ctx* c, const std::vector<OrthSpec>& specs, int passes) {
    if (specs.empty()) return;
    if (passes != kFullPasses && passes != kSpanPasses && passes != kRobustSpanPasses)
        throw_contract(c, "orth: unknown pass schedule");
    orth_many_adaptive(c, specs, passes == kFullPasses, passes == kRobustSpanPasses);
}

void orth(rrsvd_b200_ctx* c, const cplx* Y, int m, int l, cplx* Q, int* ndead) {
    orth_many(c, {OrthSpec{Y, m, l, Q, ndead}});
}

// ================================================================================== sketch

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

// ================================================================================== small SVD

namespace {

struct SmallSvdSpec {
    const cplx* X;
    int r, cc, adj, lda;
    double* sigma;
    cplx* Xn;
    cplx* Js;
};

// Block one-sided Jacobi (blockjac.cuh) for same-shaped problems: the tournament schedule is
// host-side bookkeeping; one fused launch per step for all pairs of all problems; one
// 4-byte-per-problem D2H per sweep for the convergence test.
bool bj_cross_steps() {  // RRSVD_B200_BJ_CROSS=0: the full 31-round pair solve at every step
    static const bool v = [] {
        const char* e = std::getenv("RRSVD_B200_BJ_CROSS");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return v;
}

bool bj_per_step() {  // RRSVD_B200_BJ_PER_STEP=1: one launch per tournament step (A/B timing)
    static const bool v = [] {
        const char* e = std::getenv("RRSVD_B200_BJ_PER_STEP");
        return e != nullptr && std::atoi(e) != 0;
    }();
    return v;
}

int block_jacobi_min_c() {  // above this the block method is used (RRSVD_B200_BJ_MIN_C overrides)
    // measured: the cluster kernel wins for l = 74 (C1: 2.6 vs 3.0 ms) and the batched 110^2 of
    // C3 (162 vs 186 ms per step); the DMMA block method wins for C2's batched 256^2 (5.25 vs
    // 4.60 steps/s) and everything wider
    static const int v = [] {
        const char* e = std::getenv("RRSVD_B200_BJ_MIN_C");
        return e ? std::atoi(e) : 160;
    }();
    return v;
}
constexpr int kBjBlock = 16;
int bj_inner_sweeps() {  // RRSVD_B200_BJ_INNER overrides
    static const int v = [] {
        const char* e = std::getenv("RRSVD_B200_BJ_INNER");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    return v;
}

void block_jacobi_group(rrsvd_b200_ctx* c, const std::vector<const SmallSvdSpec*>& grp) {
    const int np = (int)grp.size();
    const int r = grp[0]->r, cc = grp[0]->cc, b = kBjBlock;
    const int nb = (cc + b - 1) / b, nbp = nb + (nb & 1), cp = nbp * b, npairs = nbp / 2;
    if (nbp > kBjMaxSlots) throw_contract(c, "jacobi: too many columns for the block Jacobi");
    // placement(t): block id at block position pos (pair k: positions 2k, 2k+1)
    auto placement = [&](int t, std::vector<int>& pl) {
        pl.assign(nbp, 0);
        for (int k = 0; k < npairs; ++k) {
            auto circ = [&](int i) { return i == 0 ? 0 : ((i - 1 + t) % (nbp - 1)) + 1; };
            pl[2 * k] = circ(k);
            pl[2 * k + 1] = circ(nbp - 1 - k);
        }
    };
    std::vector<cplx*> X1(np), X2(np), V1(np), V2(np);
    BjStat* stat = ws_get<BjStat>(c, np);
    for (int p = 0; p < np; ++p) {
        X1[p] = ws_get<cplx>(c, (size_t)r * cp);
        X2[p] = ws_get<cplx>(c, (size_t)r * cp);
        V1[p] = ws_get<cplx>(c, (size_t)cp * cp);
        V2[p] = ws_get<cplx>(c, (size_t)cp * cp);
    }
    std::vector<int> pl0, plt, pln;
    placement(0, pl0);
    {
        BjInit in{};
        in.count = np; in.r = r; in.c = cc; in.cp = cp; in.b = b; in.nbp = nbp;
        for (int p = 0; p < np; ++p) {
            in.A[p] = grp[p]->X; in.lda[p] = grp[p]->lda; in.adj[p] = grp[p]->adj; in.X[p] = X1[p]; in.V[p] = V1[p];
        }
        std::copy(pl0.begin(), pl0.end(), in.place);
        check_cuda(c, bj_init(in, c->stream), "bj_init");
        c->launches++;
    }
    // per-step destination tables (the schedule repeats every sweep)
    std::vector<std::vector<int>> dst(nbp - 1, std::vector<int>(nbp));
    for (int t = 0; t < nbp - 1; ++t) {
        placement(t, plt);
        placement((t + 1) % (nbp - 1), pln);
        std::vector<int> where(nbp);
        for (int pos = 0; pos < nbp; ++pos) where[pln[pos]] = pos;
        for (int pos = 0; pos < nbp; ++pos) dst[t][pos] = where[plt[pos]];
    }
    auto* hstat = static_cast<BjStat*>(pinned_scratch(c, np * sizeof(BjStat)));
    // single-CTA pairs: one persistent launch per sweep (bj_sweep), with device copies of the
    // whole schedule and per-item completion flags
    const int nsteps = nbp - 1;
    const bool persistent = bj_slices(npairs * np, r) == 1 && !bj_per_step();
    int *d_dst = nullptr, *d_prod = nullptr, *d_done = nullptr, *d_counter = nullptr;
    if (persistent) {
        std::vector<int> hd((size_t)nsteps * nbp), hp((size_t)nsteps * nbp, 0);
        for (int t = 0; t < nsteps; ++t)
            for (int pos = 0; pos < nbp; ++pos) {
                hd[(size_t)t * nbp + pos] = dst[t][pos];
                if (t + 1 < nsteps) hp[(size_t)(t + 1) * nbp + dst[t][pos]] = pos >> 1;
            }
        d_dst = ws_get<int>(c, hd.size());
        d_prod = ws_get<int>(c, hp.size());
        d_done = ws_get<int>(c, (size_t)np * nsteps * npairs);
        d_counter = ws_get<int>(c, 1);
        check_cuda(c, cudaMemcpyAsync(d_dst, hd.data(), hd.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D");
        check_cuda(c, cudaMemcpyAsync(d_prod, hp.data(), hp.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D");
        check_cuda(c, cudaMemsetAsync(d_done, 0, (size_t)np * nsteps * npairs * sizeof(int), c->stream), "memset");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");  // (the host vectors go out of scope)
    }
    // problems drop out of the launches once a sweep of theirs rotates nothing (the batch would
    // otherwise run every problem for the slowest one's sweeps); each keeps its own buffers
    std::vector<int> active(np);
    for (int p = 0; p < np; ++p) active[p] = p;
    // the kernel's rotation threshold tol = sqrt(r) eps; noise level sqrt(c) tol (squared)
    const double tol_r = std::sqrt((double)std::max(r, 1)) * 2.220446049250313e-16;
    const double noise2 = (double)cc * tol_r * tol_r;
    int sweep = 0;
    for (; sweep < 60; ++sweep) {
        check_cuda(c, cudaMemsetAsync(stat, 0, np * sizeof(BjStat), c->stream), "memset");
        if (persistent) {
            BjSweep sw{};
            sw.count = (int)active.size(); sw.r = r; sw.cp = cp; sw.b = b; sw.npairs = npairs; sw.nsteps = nsteps;
            sw.inner_sweeps = bj_inner_sweeps();
            sw.cross_steps = bj_cross_steps();
            sw.epoch = sweep + 1;
            for (size_t q = 0; q < active.size(); ++q) {
                const int p = active[q];
                sw.X[0][q] = X1[p]; sw.X[1][q] = X2[p]; sw.V[0][q] = V1[p]; sw.V[1][q] = V2[p];
                sw.stat[q] = stat + p;
            }
            sw.dst = d_dst; sw.prod = d_prod; sw.done = d_done; sw.counter = d_counter;
            check_cuda(c, cudaMemsetAsync(d_counter, 0, sizeof(int), c->stream), "memset");
            check_cuda(c, bj_sweep(sw, c->stream), "bj_sweep");
            c->launches++;
            if (nsteps & 1)
                for (int p : active) {
                    std::swap(X1[p], X2[p]);
                    std::swap(V1[p], V2[p]);
                }
        }
        for (int t = 0; t < (persistent ? 0 : nbp - 1); ++t) {
            BjStep st{};
            st.count = (int)active.size(); st.r = r; st.cp = cp; st.b = b; st.npairs = npairs;
            st.inner_sweeps = bj_inner_sweeps();
            st.cross_only = bj_cross_steps() && t > 0;
            for (size_t q = 0; q < active.size(); ++q) {
                const int p = active[q];
                st.Xs[q] = X1[p]; st.Xd[q] = X2[p]; st.Vs[q] = V1[p]; st.Vd[q] = V2[p]; st.stat[q] = stat + p;
            }
            std::copy(dst[t].begin(), dst[t].end(), st.dst);
            check_cuda(c, bj_step(st, c->stream), "bj_step");
            c->launches++;
            for (int p : active) {
                std::swap(X1[p], X2[p]);
                std::swap(V1[p], V2[p]);
            }
        }
        check_cuda(c, cudaMemcpyAsync(hstat, stat, np * sizeof(BjStat), cudaMemcpyDeviceToHost, c->stream), "D2H");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
        std::vector<int> still;
        double worst = 0.0;
        for (int p : active) {
            double o2;
            std::memcpy(&o2, &hstat[p].off2, sizeof o2);
            worst = std::max(worst, o2);
            // converged: no rotation, or only noise-level ones (every rotated pair had
            // |g_pq| <= sqrt(c) tol sqrt(g_pp g_qq), LAPACK zgesvj's test): the next sweep would
            // rotate rounding noise again without changing the result
            if (hstat[p].rot != 0 && o2 > noise2) still.push_back(p);
        }
        if (debug_enabled())
            std::fprintf(stderr, "[rrsvd_b200] block jacobi sweep %d: %zu active, %zu rotating, max |g|/sqrt(gg) %.3g\n",
                         sweep, active.size(), still.size(), std::sqrt(worst));
        if (still.empty()) break;
        active.swap(still);
    }
    if (debug_enabled())
        std::fprintf(stderr, "[rrsvd_b200] block jacobi %dx%d x%d: %d sweeps\n", r, cc, np, sweep + 1);
    BjFinish fin{};
    fin.count = np; fin.r = r; fin.c = cc; fin.cp = cp; fin.b = b;
    for (int p = 0; p < np; ++p) {
        fin.X[p] = X1[p]; fin.V[p] = V1[p];
        fin.sigma[p] = grp[p]->sigma; fin.Xn[p] = grp[p]->Xn; fin.Js[p] = grp[p]->Js;
    }
    std::copy(pl0.begin(), pl0.end(), fin.place);
    fin.sig_ws = ws_get<double>(c, (size_t)np * cp);
    fin.rank_ws = ws_get<int>(c, (size_t)np * cp);
    check_cuda(c, bj_finish(fin, c->stream), "bj_finish");
    c->launches += 2;
}

void small_svd_many(rrsvd_b200_ctx* c, const std::vector<SmallSvdSpec>& specs) {
    std::vector<cplx*> W(specs.size());
    std::vector<int*> dsweeps(specs.size(), nullptr);
    std::vector<size_t> onchip, global;
    for (size_t i = 0; i < specs.size(); ++i) {
        W[i] = ws_get<cplx>(c, (size_t)(specs[i].r + specs[i].cc) * specs[i].cc);
        if (debug_enabled()) dsweeps[i] = ws_get<int>(c, 1);
        (specs[i].cc <= block_jacobi_min_c() && jacobi_fits(specs[i].r, specs[i].cc) ? onchip : global).push_back(i);
    }
    // The on-chip batch (one launch of a few clusters) runs on a side stream beside the block
    // Jacobi groups (many short launches with a host read per sweep), which leave SMs free.
    const cudaStream_t main_stream = c->stream;
    StreamSwitch side_switch(c);  // restores c->stream on every exit path
    constexpr int kSide = rrsvd_b200_ctx::kMaxLanes - 1;
    const bool fork = !global.empty() && !onchip.empty() && c->stream != c->lane[kSide];
    if (fork) {
        if (c->lane[kSide] == nullptr) {
            check_cuda(c, cudaStreamCreateWithFlags(&c->lane[kSide], cudaStreamNonBlocking), "side stream");
            check_cuda(c, cudaEventCreateWithFlags(&c->ev_join[kSide], cudaEventDisableTiming), "side event");
        }
        if (c->ev_fork == nullptr)
            check_cuda(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "fork event");
        check_cuda(c, cudaEventRecord(c->ev_fork, main_stream), "fork record");
        check_cuda(c, cudaStreamWaitEvent(c->lane[kSide], c->ev_fork, 0), "fork wait");
        c->stream = c->lane[kSide];
    }
    for (size_t base = 0; base < onchip.size(); base += kMaxSmall) {
        const size_t end = std::min(onchip.size(), base + kMaxSmall);
        JacobiInitBatch ib{};
        JacobiBatch jb{};
        JacobiFinBatch fb{};
        int max_r = 0, max_c = 0;
        for (size_t ii = base; ii < end; ++ii) {
            const size_t i = onchip[ii];
            const SmallSvdSpec& s = specs[i];
            const int k = ib.count++;
            ib.r[k] = s.r; ib.c[k] = s.cc; ib.A[k] = s.X; ib.lda[k] = s.lda; ib.adj[k] = s.adj; ib.W[k] = W[i];
            jb.count++;
            jb.r[k] = s.r; jb.c[k] = s.cc; jb.W[k] = W[i]; jb.sweeps[k] = dsweeps[i];
            fb.count++;
            fb.r[k] = s.r; fb.c[k] = s.cc; fb.W[k] = W[i]; fb.sigma[k] = s.sigma; fb.Xn[k] = s.Xn; fb.Js[k] = s.Js;
            max_r = std::max(max_r, s.r);
            max_c = std::max(max_c, s.cc);
        }
        check_cuda(c, jacobi_init(ib, c->stream), "jacobi_init");
        check_cuda(c, jacobi_svd(jb, max_r, max_c, c->stream), "jacobi_svd");
        check_cuda(c, jacobi_finish(fb, max_c, c->stream), "jacobi_finish");
        c->launches += 3;
    }
    c->stream = main_stream;
    // wide problems: block Jacobi over DMMA GEMMs, grouped by shape
    while (!global.empty()) {
        std::vector<const SmallSvdSpec*> grp;
        std::vector<size_t> rest;
        for (size_t i : global) {
            const SmallSvdSpec& s = specs[i];
            if (grp.empty() || (s.r == grp[0]->r && s.cc == grp[0]->cc && (int)grp.size() < kBjMaxProblems))
                grp.push_back(&s);
            else
                rest.push_back(i);
        }
        block_jacobi_group(c, grp);
        global.swap(rest);
    }
    if (fork) {
        check_cuda(c, cudaEventRecord(c->ev_join[kSide], c->lane[kSide]), "join record");
        check_cuda(c, cudaStreamWaitEvent(main_stream, c->ev_join[kSide], 0), "join wait");
    }
    if (debug_enabled()) {
        for (size_t i : onchip) {  // (the block path prints its own sweep counts)
            int h = -1;
            cudaMemcpyAsync(&h, dsweeps[i], sizeof(int), cudaMemcpyDeviceToHost, c->stream);
            cudaStreamSynchronize(c->stream);
            std::fprintf(stderr, "[rrsvd_b200] jacobi %dx%d: %d sweeps\n", specs[i].r, specs[i].cc, h);
        }
    }
}

}  // namespace

// ================================================================================== RRSVD

// The A-products of the RRSVD (tag 2): the DMMA zgemm, or — for specs carrying residue planes
// (ozaki.cuh) — the INT8 tensor-core emulation.
struct AProducts {
    std::vector<GemmSpec> gs;
    std::vector<OzProduct> oz;
    void add(const OzakiA* a, const GemmSpec& s, int T = 0) {
        if (a) oz.push_back({a, s.B, s.ldb, s.n, s.C, s.ldc, 0, T});
        else gs.push_back(s);
    }
    void run(rrsvd_b200_ctx* c, GemmOp op) {
        c->gemm_tag = 2;
        gemm_many(c, op, gs);
        // (one launch set per moduli count: products of a batch must agree on it)
        while (!oz.empty()) {
            std::vector<OzProduct> same, rest;
            for (const OzProduct& p : oz) (p.T == oz[0].T ? same : rest).push_back(p);
            ozaki_product_many(c, op, same);
            oz.swap(rest);
        }
        gs.clear();
        oz.clear();
    }
};

void range_finder_many(rrsvd_b200_ctx* c, const std::vector<RangeSpec>& specs) {
    if (specs.empty()) return;
    struct Buf {
        cplx *Y, *Z, *Qt;
    };
    std::vector<Buf> b(specs.size());
    int max_q = 0, min_q = 1 << 30;
    for (size_t i = 0; i < specs.size(); ++i) {
        const RangeSpec& s = specs[i];
        min_q = std::min(min_q, s.q);
        max_q = std::max(max_q, s.q);
        b[i] = {ws_get<cplx>(c, (size_t)s.m * s.l), ws_get<cplx>(c, (size_t)s.n * s.l),
                ws_get<cplx>(c, (size_t)s.n * s.l)};
    }
    AProducts ap;
    std::vector<OrthSpec> os;
    // the power iteration's intermediate products only shape the subspace the last Y = A Q~
    // spans (each is followed by another product): they take fewer moduli (ozaki_inner_moduli)
    const int inner = ozaki_inner_moduli();
    // Algorithm 1 (randomized.cpp:88-99): Y = A Omega, QR
    for (size_t i = 0; i < specs.size(); ++i) {
        const RangeSpec& s = specs[i];
        ap.add(s.oz, {s.m, s.l, s.n, s.A, s.n, s.omega, s.l, b[i].Y, s.l}, s.q > 0 ? inner : 0);
        os.push_back({b[i].Y, s.m, s.l, s.Q});
    }
    ap.run(c, kOpN);
    // The power iteration's bases (emulated A-products): one shifted pass when it finds Y well
    // conditioned (every pivot
    // >= 1e4 x the shift: cond(Q) - 1 <= 5e-5), else the full four-pass schedule
    // (kRobustSpanPasses).  Two shifted passes alone (the span-only schedule) leave an
    // ill-conditioned Q~ on rank-deficient Θ — cond 3e14 measured on a TEDOPA bond
    // (tools/oz_chol_probe.py) — whose tail directions the next product then resolves only through
    // its own rounding noise: the kept λ tail came out ~25 % low, and with the exactly rounded
    // emulated products the final CholeskyQR lost 19 directions.  With orthonormal bases every
    // A-product path reproduces the exact SVD's tail.  RRSVD_B200_SPAN_PASSES=1 restores the
    // span-only schedule.
    static const bool span_only = [] {
        const char* e = std::getenv("RRSVD_B200_SPAN_PASSES");
        return e != nullptr && std::atoi(e) != 0;
    }();
    // (The span-only schedule stays for an all-DMMA batch: its products' rounding noise is what the
    // reference's own FP64 products carry, and the parity suite holds with it.)
    bool emulated = false;
    for (const RangeSpec& s : specs) emulated = emulated || s.oz != nullptr;
    const int inter = min_q != max_q ? kFullPasses : (span_only || !emulated) ? kSpanPasses : kRobustSpanPasses;
    orth_many(c, os, max_q > 0 ? inter : kFullPasses);
    for (int j = 0; j < max_q; ++j) {
        os.clear();
        for (size_t i = 0; i < specs.size(); ++i) {  // Z = A^H Q, QR
            const RangeSpec& s = specs[i];
            if (j >= s.q) continue;
            ap.add(s.oz, {s.n, s.l, s.m, s.A, s.n, s.Q, s.l, b[i].Z, s.l}, inner);
            os.push_back({b[i].Z, s.n, s.l, b[i].Qt});
        }
        ap.run(c, kOpC);
        orth_many(c, os, inter);
        os.clear();
        for (size_t i = 0; i < specs.size(); ++i) {  // Y = A Q~, QR
            const RangeSpec& s = specs[i];
            if (j >= s.q) continue;
            // the last Y = A Q~ (the basis B is built on) stays on FP64 with the assembly product
            // unless RRSVD_B200_OZAKI_TAIL < 2 (see rrsvd_core_many)
            ap.add(j + 1 == s.q && ozaki_tail() >= 2 ? nullptr : s.oz, {s.m, s.l, s.n, s.A, s.n, b[i].Qt, s.l, b[i].Y, s.l},
                   j + 1 < s.q ? inner : 0);
            os.push_back({b[i].Y, s.m, s.l, s.Q});
        }
        ap.run(c, kOpN);
        orth_many(c, os, j + 1 < max_q ? inter : kFullPasses);
    }
}

void assemble_many(rrsvd_b200_ctx* c, const std::vector<AssembleSpec>& specs) {
    if (specs.empty()) return;
    struct Buf {
        cplx *Z, *Qb, *X, *Xn, *Js;
    };
    std::vector<Buf> b(specs.size());
    for (size_t i = 0; i < specs.size(); ++i) {
        const AssembleSpec& s = specs[i];
        b[i] = {ws_get<cplx>(c, (size_t)s.n * s.l), ws_get<cplx>(c, (size_t)s.n * s.l),
                ws_get<cplx>(c, (size_t)s.l * s.l), ws_get<cplx>(c, (size_t)s.l * s.l),
                ws_get<cplx>(c, (size_t)s.l * s.l)};
    }
    // B = Q^H A held as B^H = A^H Q = Qb X  (assemble_from_basis, randomized.cpp:57-66)
    std::vector<GemmSpec> gs;
    std::vector<OrthSpec> os;
    AProducts ap;
    for (size_t i = 0; i < specs.size(); ++i) {
        const AssembleSpec& s = specs[i];
        ap.add(s.oz, {s.n, s.l, s.m, s.A, s.n, s.Q, s.l, b[i].Z, s.l});
        os.push_back({b[i].Z, s.n, s.l, b[i].Qb});
    }
    ap.run(c, kOpC);
    orth_many(c, os);
    for (size_t i = 0; i < specs.size(); ++i) {  // X = Qb^H B^H  (l x l, ~upper triangular)
        const AssembleSpec& s = specs[i];
        gs.push_back({s.l, s.l, s.n, b[i].Qb, s.l, b[i].Z, s.l, b[i].X, s.l});
    }
    c->gemm_tag = 5;
    gemm_many(c, kOpC, gs);
    // B = X^H Qb^H.  One-sided Jacobi on X^H (the R^H of a QR converges in a few sweeps,
    // Drmac-Veselic): X^H K = Z Sigma  =>  B = Z Sigma (Qb K)^H, so U_B = Z, V = Qb K.
    std::vector<SmallSvdSpec> ss;
    for (size_t i = 0; i < specs.size(); ++i) {
        const AssembleSpec& s = specs[i];
        ss.push_back({b[i].X, s.l, s.l, 1, s.l, s.sigma, b[i].Xn, b[i].Js});
    }
    small_svd_many(c, ss);
    gs.clear();
    for (size_t i = 0; i < specs.size(); ++i) {
        const AssembleSpec& s = specs[i];
        gs.push_back({s.m, s.l, s.l, s.Q, s.l, b[i].Xn, s.l, s.U, s.l});   // U = Q U_B
        gs.push_back({s.n, s.l, s.l, b[i].Qb, s.l, b[i].Js, s.l, s.V, s.l});  // V = Qb K
    }
    c->gemm_tag = 5;
    gemm_many(c, kOpN, gs);
}

// ||A||^2 + the non-finite count of each matrix (tebd.cpp:156-160): one launch pair per 64
struct SumsqJob {
    const cplx* A;
    long long n;
    double* total_sq;
    int* nonfinite;
};
void sumsq_jobs(rrsvd_b200_ctx* c, const std::vector<SumsqJob>& jobs) {
    for (size_t base = 0; base < jobs.size(); base += kMaxSmall) {
        SumsqBatch sb{};
        for (size_t i = base; i < std::min(jobs.size(), base + kMaxSmall); ++i) {
            const int k = sb.count++;
            sb.a[k] = jobs[i].A;
            sb.n[k] = jobs[i].n;
            sb.out_sq[k] = jobs[i].total_sq;
            sb.out_bad[k] = jobs[i].nonfinite;
        }
        double* part = ws_get<double>(c, (size_t)sb.count * 2 * kNumSMs);
        int* bad = ws_get<int>(c, (size_t)sb.count * 2 * kNumSMs);
        check_cuda(c, sumsq_many(sb, part, bad, c->stream), "sumsq_many");
        c->launches += 2;
    }
}

void rrsvd_core_many(rrsvd_b200_ctx* c, const std::vector<RrsvdSpec>& specs) {
    if (specs.empty()) return;
    std::vector<RangeSpec> rf;
    std::vector<AssembleSpec> as;
    // A's residue planes for the emulated A-products, built once for all 2 + 2q of them
    std::vector<OzSrc> src;
    std::vector<int> which;
    const int T = ozaki_moduli();
    // the residue planes (2T bytes per entry, 128-padded) live for the whole call: bonds beyond
    // the budget (RRSVD_B200_OZAKI_MAX_GB, default 32 GB — a fifth of B200's HBM; no device query
    // here: cudaMemGetInfo would serialise the lanes) stay on DMMA
    const double budget = T > 0 ? ozaki_max_bytes() : 0.0;
    double planes = 0.0;
    for (size_t i = 0; i < specs.size(); ++i)
        if (T > 0 && ozaki_usable(specs[i].m, specs[i].n, specs[i].l)) {
            const double b = 2.0 * T * ((specs[i].m + 127) / 128) * ((specs[i].n + 127) / 128) * 16384.0;
            if (planes + b > budget) continue;
            planes += b;
            src.push_back({specs[i].A, specs[i].m, specs[i].n, (long long)specs[i].n, specs[i].total_sq,
                           specs[i].nonfinite});
            which.push_back((int)i);
        }
    // a batch too small to fill the GPU's HBM stream (single C1 / C5 n <= ~2000 decimations) keeps
    // the DMMA zgemm: its A preparation and residue/CRT launches would add latency, not save time
    double work = 0.0;
    for (const OzSrc& s : src) work += (double)s.m * s.n;
    std::vector<OzakiA> oz;
    if (!src.empty() && work >= ozaki_min_work()) oz = ozaki_prepare_many(c, src, T);
    else which.clear();
    std::vector<const OzakiA*> ozp(specs.size(), nullptr);
    for (size_t j = 0; j < which.size(); ++j) ozp[which[j]] = &oz[j];
    // ||A||^2 of the DMMA problems (the emulated ones took it in their row-exponent pass)
    std::vector<SumsqJob> sq;
    for (size_t i = 0; i < specs.size(); ++i)
        if (specs[i].total_sq != nullptr && ozp[i] == nullptr)
            sq.push_back({specs[i].A, (long long)specs[i].m * specs[i].n, specs[i].total_sq, specs[i].nonfinite});
    sumsq_jobs(c, sq);
    for (size_t i = 0; i < specs.size(); ++i) {
        const RrsvdSpec& s = specs[i];
        cplx* Q = ws_get<cplx>(c, (size_t)s.m * s.l);
        rf.push_back({s.A, s.m, s.n, s.l, s.q, s.omega, Q, ozp[i]});
        // B^H = A^H Q is emulated too unless RRSVD_B200_OZAKI_TAIL >= 1 keeps it on the FP64 zgemm
        // (the numerically-zero cutoff, sigma <= 1e-15 sigma_1 at tebd.cpp:193, then sees the DMMA
        // product's rounding noise in the directions of Q outside the range of a rank-deficient A;
        // with the robust power-iteration bases the emulated assembly keeps the reference's chi)
        as.push_back({s.A, s.m, s.n, s.l, Q, s.U, s.sigma, s.V, ozaki_tail() >= 1 ? nullptr : ozp[i]});
    }
    range_finder_many(c, rf);
    assemble_many(c, as);
}

// Fixed-precision RRSVD (randomized.cpp:124-176), all problems in lock-step rounds.  Each round
// draws `probes` fresh Gaussian columns per active problem (seed + 0x9e3779b97f4a7c15·draw), forms
// D = (I - Q Q^H) A Omega_p, and either certifies max_j ||D_j|| <= eps or grows the basis by
// growth_block (0: l) columns (the probe images first, then A times fresh sketch columns),
// orthonormalised against Q.  The per-round decision needs the norms on the host: one small D2H per round.
void rrsvd_fixed_precision_many(rrsvd_b200_ctx* c, std::vector<FixedPrecSpec>& specs) {
    if (specs.empty()) return;
    constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
    const size_t np = specs.size();
    std::vector<cplx*> Q(np);
    std::vector<uint64_t> draw(np, 1);
    std::vector<char> active(np, 1);
    {
        std::vector<RangeSpec> rf;
        for (size_t i = 0; i < np; ++i) {
            FixedPrecSpec& s = specs[i];
            const int r = s.probes, minor = std::min(s.m, s.n);
            if (r < 1) throw_contract(c, "rrsvd_fixed_precision: probe_count >= 1 required");
            if (s.l0 < 1 || s.l0 + r > s.n)
                throw_contract(c, "rrsvd_fixed_precision: requires initial_l + probe_count <= n");
            (void)minor;
            s.l = s.l0;
            s.certified = false;
            Q[i] = ws_get<cplx>(c, (size_t)s.m * s.l);
            const cplx* om = s.omega0;
            if (om == nullptr) {
                cplx* o = ws_get<cplx>(c, (size_t)s.n * s.l);
                make_omega(c, s.n, s.l, s.seed, s.omega_mode, o);
                om = o;
            }
            rf.push_back({s.A, s.m, s.n, s.l, s.q, om, Q[i]});
        }
        range_finder_many(c, rf);
    }
    double* dmax = ws_get<double>(c, np);
    auto* hmax = static_cast<double*>(pinned_scratch(c, np * sizeof(double)));
    while (true) {
        std::vector<size_t> act;
        for (size_t i = 0; i < np; ++i)
            if (active[i]) act.push_back(i);
        if (act.empty()) break;
        std::vector<cplx*> Bp(np, nullptr), QhB(np, nullptr), Dm(np, nullptr);
        std::vector<GemmSpec> g1, g2, g3;
        for (size_t i : act) {
            FixedPrecSpec& s = specs[i];
            const int r = s.probes;
            cplx* om = ws_get<cplx>(c, (size_t)s.n * r);
            make_omega(c, s.n, r, s.seed + kGolden * draw[i], s.omega_mode, om);
            ++draw[i];
            Bp[i] = ws_get<cplx>(c, (size_t)s.m * r);
            QhB[i] = ws_get<cplx>(c, (size_t)s.l * r);
            Dm[i] = ws_get<cplx>(c, (size_t)s.m * r);
            g1.push_back({s.m, r, s.n, s.A, s.n, om, r, Bp[i], r});           // B = A Omega_p
            g2.push_back({s.l, r, s.m, Q[i], s.l, Bp[i], r, QhB[i], r});      // Q^H B
            GemmSpec d{s.m, r, s.l, Q[i], s.l, QhB[i], r, Dm[i], r};         // D = B - Q (Q^H B)
            d.D = Bp[i];
            d.ldd = r;
            d.alpha = -1.0;
            g3.push_back(d);
        }
        c->gemm_tag = 7;
        gemm_many(c, kOpN, g1);
        gemm_many(c, kOpC, g2);
        gemm_many(c, kOpN, g3);
        ColNormBatch cn{};
        std::vector<size_t> slot(np, 0);
        for (size_t t = 0; t < act.size(); ++t) {
            const size_t i = act[t];
            const int k = cn.count++;
            cn.D[k] = Dm[i]; cn.m[k] = specs[i].m; cn.r[k] = specs[i].probes; cn.out[k] = dmax + t;
            if (cn.count == kMaxSmall) {
                check_cuda(c, colnorm_max_many(cn, c->stream), "colnorm_max");
                c->launches++;
                cn = ColNormBatch{};
            }
        }
        if (cn.count) {
            check_cuda(c, colnorm_max_many(cn, c->stream), "colnorm_max");
            c->launches++;
        }
        check_cuda(c, cudaMemcpyAsync(hmax, dmax, act.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
                   "D2H");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
        // Growth (randomized.cpp:155-168): the new block X (the probe images, then A times fresh
        // sketch columns) is orthonormalised against the kept basis by block classical
        // Gram-Schmidt with reorthogonalisation — twice {X <- X - Q (Q^H X); X <- orth(X)} — and
        // Q_new = [Q, X] spans what the reference's Householder QR of [Q, X] spans.  A Cholesky
        // QR of the whole [Q, X], or one projection before orth(X), lets X's dependent columns
        // (a basis grown past the rank) turn into normalised noise that leaks along Q, and the
        // probe then fails to certify a basis that does span the range.
        struct Grow { size_t i; int l, g; cplx *Qn, *Xa, *Xb, *Pq, *Xq; };
        std::vector<Grow> gw;
        std::vector<GemmSpec> gx;
        for (size_t t = 0; t < act.size(); ++t) {
            const size_t i = act[t];
            FixedPrecSpec& s = specs[i];
            const int r = s.probes, minor = std::min(s.m, s.n);
            if (hmax[t] <= s.eps) {
                s.certified = true;
                active[i] = 0;
                continue;
            }
            if (s.l + r > minor) { active[i] = 0; continue; }
            // randomized.cpp:156-157: growth_block columns, or double the basis when it is 0
            const int grow = std::min(s.growth_block == 0 ? s.l : s.growth_block, minor - s.l);
            if (grow == 0) { active[i] = 0; continue; }
            const int from_probe = std::min(r, grow);
            Grow w{i, s.l, grow, ws_get<cplx>(c, (size_t)s.m * (s.l + grow)), ws_get<cplx>(c, (size_t)s.m * grow),
                   ws_get<cplx>(c, (size_t)s.m * grow), ws_get<cplx>(c, (size_t)s.l * grow),
                   ws_get<cplx>(c, (size_t)s.m * grow)};
            check_cuda(c, cudaMemcpy2DAsync(w.Xa, grow * sizeof(cplx), Bp[i], r * sizeof(cplx),
                                            from_probe * sizeof(cplx), s.m, cudaMemcpyDeviceToDevice, c->stream),
                       "copy");
            if (grow > from_probe) {
                const int ne = grow - from_probe;
                cplx* om = ws_get<cplx>(c, (size_t)s.n * ne);
                make_omega(c, s.n, ne, s.seed + kGolden * draw[i], s.omega_mode, om);
                ++draw[i];
                gx.push_back({s.m, ne, s.n, s.A, s.n, om, ne, w.Xa + from_probe, grow});
            }
            gw.push_back(w);
        }
        c->gemm_tag = 7;
        gemm_many(c, kOpN, gx);
        for (int pass = 0; pass < 2; ++pass) {  // X -> Xb = X - Q (Q^H X) -> orth: Xa -> Xq, then Xq -> Xa
            std::vector<GemmSpec> gp, gs;
            std::vector<OrthSpec> os;
            for (const Grow& w : gw) {
                const FixedPrecSpec& s = specs[w.i];
                const cplx* X = pass == 0 ? w.Xa : w.Xq;
                gp.push_back({w.l, w.g, s.m, Q[w.i], w.l, X, w.g, w.Pq, w.g});       // P = Q^H X
                GemmSpec d{s.m, w.g, w.l, Q[w.i], w.l, w.Pq, w.g, w.Xb, w.g};      // Xb = X - Q P
                d.D = X;
                d.ldd = w.g;
                d.alpha = -1.0;
                gs.push_back(d);
                os.push_back({w.Xb, s.m, w.g, pass == 0 ? w.Xq : w.Xa});
            }
            c->gemm_tag = 7;
            gemm_many(c, kOpC, gp);
            gemm_many(c, kOpN, gs);
            orth_many(c, os);
        }
        for (const Grow& w : gw) {
            FixedPrecSpec& s = specs[w.i];
            const int ln = w.l + w.g;
            check_cuda(c, cudaMemcpy2DAsync(w.Qn, ln * sizeof(cplx), Q[w.i], w.l * sizeof(cplx), w.l * sizeof(cplx),
                                            s.m, cudaMemcpyDeviceToDevice, c->stream), "copy");
            check_cuda(c, cudaMemcpy2DAsync(w.Qn + w.l, ln * sizeof(cplx), w.Xa, w.g * sizeof(cplx),
                                            w.g * sizeof(cplx), s.m, cudaMemcpyDeviceToDevice, c->stream), "copy");
            Q[w.i] = w.Qn;
            s.l = ln;
        }
    }
    std::vector<AssembleSpec> as;
    for (size_t i = 0; i < np; ++i) {
        FixedPrecSpec& s = specs[i];
        s.U = ws_get<cplx>(c, (size_t)s.m * s.l);
        s.V = ws_get<cplx>(c, (size_t)s.n * s.l);
        s.sigma = ws_get<double>(c, s.l);
        as.push_back({s.A, s.m, s.n, s.l, Q[i], s.U, s.sigma, s.V});
    }
    assemble_many(c, as);
}

void rrsvd_core(rrsvd_b200_ctx* c, const cplx* A, int m, int n, int l, int q, const cplx* omega,
                cplx* U, double* sigma, cplx* V) {
    rrsvd_core_many(c, {RrsvdSpec{A, m, n, l, q, omega, U, sigma, V}});
}

// ================================================================================== full SVD

void svd_jacobi_many(rrsvd_b200_ctx* c, const std::vector<SvdSpec>& specs) {
    if (specs.empty()) return;
    std::vector<SmallSvdSpec> pre;
    struct Pre {
        const cplx* X;
        int r, cc;
        bool tall;
        cplx *Qr, *R, *K;
        const SvdSpec* s;
        int* perm;
    };
    std::vector<Pre> pres;
    for (const SvdSpec& s : specs) {
        const bool tall = s.m >= s.n;
        const int r = tall ? s.m : s.n, cc = tall ? s.n : s.m;
        const cplx* X = s.A;
        if (!tall) {
            cplx* Xt = ws_get<cplx>(c, (size_t)r * cc);
            check_cuda(c, conj_transpose(s.A, s.m, s.n, Xt, c->stream), "conj_transpose");
            c->launches++;
            X = Xt;
        }
        pres.push_back({X, r, cc, tall, ws_get<cplx>(c, (size_t)r * cc), ws_get<cplx>(c, (size_t)cc * cc),
                        ws_get<cplx>(c, (size_t)cc * cc), &s, nullptr});
    }
    // Static column pivoting: X's columns sorted by decreasing norm (Xp = X Pi) before the QR
    // gives R a decreasing diagonal, and the one-sided Jacobi on R^H then converges in fewer
    // sweeps (graded columns are the TEBD norm: column norms scale with lambda_r).
    std::vector<cplx*> Vp(pres.size());
    for (size_t base = 0; base < pres.size(); base += kMaxSmall) {
        ColPermBatch cp{};
        int max_c = 0;
        for (size_t i = base; i < std::min(pres.size(), base + kMaxSmall); ++i) {
            Pre& p = pres[i];
            const int k = cp.count++;
            cplx* Xp = ws_get<cplx>(c, (size_t)p.r * p.cc);
            cp.X[k] = p.X; cp.Xp[k] = Xp; cp.r[k] = p.r; cp.c[k] = p.cc;
            cp.perm[k] = p.perm = ws_get<int>(c, p.cc);
            p.X = Xp;
            max_c = std::max(max_c, p.cc);
        }
        check_cuda(c, colperm_sort_gather(cp, max_c, c->stream), "colperm");
        c->launches += 2;
    }
    // QR-preconditioned Jacobi: X (r x cc) = A or A^H (columns permuted), X = Qr R, R^H K = Z S
    //   =>  X = (Qr K) S Z^H : left vectors Qr K, right vectors Z (rows un-permuted at the end).
    std::vector<OrthSpec> os;
    std::vector<GemmSpec> gs;
    for (const Pre& p : pres) os.push_back({p.X, p.r, p.cc, p.Qr});
    orth_many(c, os);
    for (const Pre& p : pres) gs.push_back({p.cc, p.cc, p.r, p.Qr, p.cc, p.X, p.cc, p.R, p.cc});
    c->gemm_tag = 6;
    gemm_many(c, kOpC, gs);
    for (size_t i = 0; i < pres.size(); ++i) {
        const Pre& p = pres[i];
        Vp[i] = ws_get<cplx>(c, (size_t)p.cc * p.cc);
        pre.push_back({p.R, p.cc, p.cc, 1, p.cc, p.s->sigma, Vp[i], p.K});
    }
    small_svd_many(c, pre);
    for (size_t base = 0; base < pres.size(); base += kMaxSmall) {
        ColPermBatch cp{};
        for (size_t i = base; i < std::min(pres.size(), base + kMaxSmall); ++i) {
            const Pre& p = pres[i];
            const int k = cp.count++;
            cp.c[k] = p.cc; cp.perm[k] = p.perm; cp.Vp[k] = Vp[i]; cp.V[k] = p.tall ? p.s->V : p.s->U;
        }
        check_cuda(c, colperm_scatter_rows(cp, c->stream), "colperm scatter");
        c->launches++;
    }
    gs.clear();
    for (const Pre& p : pres) gs.push_back({p.r, p.cc, p.cc, p.Qr, p.cc, p.K, p.cc, p.tall ? p.s->U : p.s->V, p.cc});
    c->gemm_tag = 6;
    gemm_many(c, kOpN, gs);
}

void svd_jacobi(rrsvd_b200_ctx* c, const cplx* A, int m, int n, cplx* U, double* sigma, cplx* V) {
    svd_jacobi_many(c, {SvdSpec{A, m, n, U, sigma, V}});
}

// ================================================================================== TEBD trio

bool decimation_syncs_host(const DecimPlan& pl) {
    if (pl.fixed_precision) return true;
    const int cc = pl.randomized ? pl.l : pl.minor;  // the small SVD's column count
    return cc > block_jacobi_min_c() || !jacobi_fits(cc, cc);
}

DecimPlan plan_decimation(int d1, int d2, int cl, int cr, size_t chi_max, int kind, size_t target_rank,
                          size_t oversampling, size_t det_crossover, int accuracy_check, size_t probe_count) {
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
        // tebd.cpp:173: the accuracy check runs when the probes fit beside the sketch
        p.fixed_precision = accuracy_check && (size_t)p.l + probe_count <= (size_t)p.n &&
                            (size_t)p.l + probe_count <= (size_t)p.minor;
        p.probes = (int)probe_count;
        if (p.fixed_precision) p.ns = p.minor;  // the basis may grow up to the minor dimension
    }
    p.kmax = p.ns;
    // the accuracy check owns the retained rank: no chi_max cap (tebd.cpp:177-179)
    if (chi_max != 0 && !p.fixed_precision) p.kmax = (int)std::min<size_t>((size_t)p.kmax, chi_max);
    return p;
}

void build_theta_many(rrsvd_b200_ctx* c, const std::vector<ThetaJob>& jobs) {
    // λ_m is folded into Γ2's rows by a bandwidth-bound pre-pass (Γ2 is cm x d2·cr, 3 MB at
    // config 3), so the DMMA GEMM carries only epilogue scalings (λ_l rows, λ_r columns).
    std::vector<GemmSpec> gs;
    for (size_t base = 0; base < jobs.size(); base += kMaxEpi) {
        ScaleRowsBatch sb{};
        for (size_t i = base; i < std::min(jobs.size(), base + kMaxEpi); ++i) {
            const ThetaJob& j = jobs[i];
            const int n = j.d2 * j.cr;
            cplx* g2s = ws_get<cplx>(c, (size_t)j.cm * n);
            const int k = sb.count++;
            sb.in[k] = j.G2; sb.s[k] = j.lm; sb.rows[k] = j.cm; sb.cols[k] = n; sb.out[k] = g2s;
            Scale sc;
            sc.rs = j.ll; sc.rs_div = j.d1; sc.cs = j.lr; sc.cs_mod = j.cr;
            gs.push_back({j.cl * j.d1, n, j.cm, j.G1, j.cm, g2s, n, j.M, n, sc});
        }
        check_cuda(c, scale_rows_many(sb, c->stream), "scale_rows");
        c->launches++;
    }
    c->gemm_tag = 0;
    gemm_many(c, kOpN, gs);
}

bool make_gate_blocks(rrsvd_b200_ctx* c, const cplx* G, int dd, GateBlocksOwned& out) {
    std::vector<cplx> h((size_t)dd * dd);
    check_cuda(c, cudaMemcpyAsync(h.data(), G, h.size() * sizeof(cplx), cudaMemcpyDefault, c->stream), "gate D2H");
    check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    std::vector<int> parent(dd);
    for (int i = 0; i < dd; ++i) parent[i] = i;
    auto find = [&](int x) {
        while (parent[x] != x) x = parent[x] = parent[parent[x]];
        return x;
    };
    for (int r = 0; r < dd; ++r)
        for (int k = 0; k < dd; ++k) {
            const cplx v = h[(size_t)r * dd + k];
            if (v.x != 0.0 || v.y != 0.0) {
                const int a = find(r), b = find(k);
                if (a != b) parent[a] = b;
            }
        }
    std::vector<std::vector<int>> groups;
    std::vector<int> gid(dd, -1);
    for (int i = 0; i < dd; ++i) {
        const int root = find(i);
        if (gid[root] < 0) {
            gid[root] = (int)groups.size();
            groups.emplace_back();
        }
        groups[gid[root]].push_back(i);
    }
    if (groups.size() < 2) return false;
    for (const auto& g : groups)
        if ((int)g.size() > kMaxGateBlock) return false;
    std::vector<int> offs{0}, idx, goff;
    std::vector<cplx> gblk;
    for (const auto& g : groups) {
        goff.push_back((int)gblk.size());
        for (int r : g) {
            idx.push_back(r);
            for (int k : g) gblk.push_back(h[(size_t)r * dd + k]);
        }
        offs.push_back((int)idx.size());
    }
    auto upload = [&](const void* src, size_t bytes) {
        void* d = nullptr;
        check_cuda(c, cudaMallocAsync(&d, std::max<size_t>(bytes, 16), c->stream), "alloc gate blocks");
        check_cuda(c, cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, c->stream), "upload gate blocks");
        out.bufs.push_back(d);
        return d;
    };
    out.dev.nblocks = (int)groups.size();
    out.dev.dd = dd;
    out.dev.total = (int)gblk.size();
    out.dev.offs = static_cast<const int*>(upload(offs.data(), offs.size() * sizeof(int)));
    out.dev.idx = static_cast<const int*>(upload(idx.data(), idx.size() * sizeof(int)));
    out.dev.goff = static_cast<const int*>(upload(goff.data(), goff.size() * sizeof(int)));
    out.dev.gblk = static_cast<const cplx*>(upload(gblk.data(), gblk.size() * sizeof(cplx)));
    check_cuda(c, cudaStreamSynchronize(c->stream), "sync");  // host vectors die at return
    return true;
}

void free_gate_blocks(rrsvd_b200_ctx* c, GateBlocksOwned& g) {
    for (void* p : g.bufs) cudaFreeAsync(p, c->stream);
    g.bufs.clear();
}

void apply_gate_many(rrsvd_b200_ctx* c, const std::vector<GateJob>& jobs) {
    std::vector<GemmSpec> gs;
    GateBlockBatch gbb{};
    long long max_cols = 0;
    auto flush_blocks = [&] {
        check_cuda(c, gate_blocks_many(gbb, max_cols, c->stream), "gate_blocks");
        if (gbb.count) c->launches++;
        gbb.count = 0;
        max_cols = 0;
    };
    for (const GateJob& j : jobs) {
        const int dd = j.d1 * j.d2;
        if (j.blocks != nullptr) {
            gbb.j[gbb.count++] = GateBlockJob{*j.blocks, j.Min, j.Mout, j.cl, j.cr};
            max_cols = std::max(max_cols, (long long)j.cl * j.cr);
            if (gbb.count == kMaxEpi) flush_blocks();
        } else if (dd <= 16) {
            check_cuda(c, gate_small(j.G, dd, j.cl, j.cr, j.Min, j.Mout, c->stream), "gate_small");
            c->launches++;
        } else {
            // All χ_l blocks M[a] (dd x χ_r, stride dd·χ_r) as one column-blocked GEMM:
            // [M'[0] | M'[1] | ...] = G · [M[0] | M[1] | ...],  N = χ_l·χ_r.
            GemmSpec g{dd, j.cl * j.cr, dd, j.G, dd, j.Min, j.cr, j.Mout, j.cr};
            g.nsub = j.cr;
            g.subB = g.subC = (long long)dd * j.cr;
            gs.push_back(g);
        }
    }
    flush_blocks();
    c->gemm_tag = 1;
    gemm_many(c, kOpN, gs);
}

void decimate_many(rrsvd_b200_ctx* c, const std::vector<DecimJob>& jobs) {
    struct Out {
        cplx *U, *V;
        double* sig;
    };
    std::vector<Out> outs(jobs.size());
    std::vector<int> ns(jobs.size());
    std::vector<RrsvdSpec> rs;
    std::vector<SvdSpec> ds;
    // fixed-precision bonds first: their data-dependent width is settled on the host
    std::vector<FixedPrecSpec> fp;
    std::vector<size_t> fp_job;
    for (size_t i = 0; i < jobs.size(); ++i) {
        const DecimJob& j = jobs[i];
        ns[i] = j.pl.ns;
        if (!j.pl.fixed_precision) continue;
        FixedPrecSpec f{j.M, j.pl.m, j.pl.n, j.pl.l, j.q, j.pl.probes, j.eps, j.seed, j.omega_mode};
        f.omega0 = j.omega;
        fp.push_back(f);
        fp_job.push_back(i);
    }
    rrsvd_fixed_precision_many(c, fp);
    for (size_t t = 0; t < fp.size(); ++t) {
        const size_t i = fp_job[t];
        outs[i] = {fp[t].U, fp[t].V, fp[t].sigma};
        ns[i] = fp[t].l;
        if (jobs[i].certified) *jobs[i].certified = fp[t].certified ? 1 : 0;
    }
    // ‖Θ‖² + finite check for every bond (tebd.cpp:156-160); the fixed-rank RRSVD bonds take theirs
    // inside rrsvd_core_many (from the emulation's row-exponent pass when their A-products are
    // emulated: one read of Θ less)
    std::vector<SumsqJob> sq;
    for (const DecimJob& j : jobs)
        if (j.pl.fixed_precision || !j.pl.randomized)
            sq.push_back({j.M, (long long)j.pl.m * j.pl.n, &j.sc->total_sq, &j.sc->nonfinite});
    sumsq_jobs(c, sq);
    PhiloxBatch pb{};
    auto flush_philox = [&] {
        check_cuda(c, omega_philox_many(pb, c->stream), "philox_many");
        if (pb.count) c->launches++;
        pb.count = 0;
    };
    for (size_t i = 0; i < jobs.size(); ++i) {
        const DecimJob& j = jobs[i];
        const DecimPlan& pl = j.pl;
        if (pl.fixed_precision) continue;
        outs[i] = {ws_get<cplx>(c, (size_t)pl.m * pl.ns), ws_get<cplx>(c, (size_t)pl.n * pl.ns),
                   ws_get<double>(c, pl.ns)};
        if (pl.randomized) {
            const cplx* om = j.omega;
            if (om == nullptr) {
                cplx* o = ws_get<cplx>(c, (size_t)pl.n * pl.l);
                if (j.omega_mode == 1) {  // RRSVD_B200_OMEGA_PHILOX: batched over bonds
                    const int k = pb.count++;
                    pb.seed[k] = j.seed; pb.n[k] = (long long)pl.n * pl.l; pb.out[k] = o;
                    if (pb.count == kMaxEpi) flush_philox();
                } else {
                    make_omega(c, pl.n, pl.l, j.seed, j.omega_mode, o);
                }
                om = o;
            }
            rs.push_back({j.M, pl.m, pl.n, pl.l, j.q, om, outs[i].U, outs[i].sig, outs[i].V, &j.sc->total_sq,
                          &j.sc->nonfinite});
        } else {
            ds.push_back({j.M, pl.m, pl.n, outs[i].U, outs[i].sig, outs[i].V});
        }
    }
    flush_philox();
    rrsvd_core_many(c, rs);
    svd_jacobi_many(c, ds);
    // truncation (tebd.cpp:188-209) and Γ reshape (tebd.cpp:211-235), one launch set per 64 bonds
    for (size_t base = 0; base < jobs.size(); base += kMaxEpi) {
        TruncBatch tb{};
        GammaBatch gb{};
        gb.max_kept = gb.max_m = gb.max_n = 0;
        for (size_t i = base; i < std::min(jobs.size(), base + kMaxEpi); ++i) {
            const DecimJob& j = jobs[i];
            const DecimPlan& pl = j.pl;
            TruncArgs& ta = tb.a[tb.count++];
            ta = TruncArgs{};
            ta.sigma = outs[i].sig; ta.ns = ns[i]; ta.total_sq = &j.sc->total_sq; ta.trunc_tol = j.trunc_tol;
            ta.cap = pl.fixed_precision ? 0 : (long long)j.chi_max;
            ta.renormalize = j.renormalize; ta.kept = &j.sc->kept;
            ta.lambda = j.lambda; ta.discarded = &j.sc->discarded;
            ta.nonfinite = &j.sc->nonfinite;
            GammaArgs& ga = gb.a[gb.count++];
            ga = GammaArgs{};
            ga.U = outs[i].U; ga.ldu = ns[i]; ga.V = outs[i].V; ga.ldv = ns[i]; ga.ll = j.ll; ga.lr = j.lr;
            ga.m = pl.m; ga.n = pl.n; ga.d1 = j.d1; ga.cr = j.cr; ga.kept = &j.sc->kept;
            ga.gamma_l = j.gamma_l; ga.gamma_r = j.gamma_r; ga.pinv = &j.sc->pinv;
            gb.max_kept = std::max(gb.max_kept, pl.fixed_precision ? ns[i] : pl.kmax);
            gb.max_m = std::max(gb.max_m, pl.m);
            gb.max_n = std::max(gb.max_n, pl.n);
        }
        check_cuda(c, truncate_many(tb, c->stream), "truncate_many");
        check_cuda(c, gamma_reshape_many(gb, c->stream), "gamma_reshape_many");
        c->launches += 4;
    }
}

}  // namespace rb

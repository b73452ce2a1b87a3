// evolve.cu — device-resident MpsState and the TEBD sweep driver (tebd.cpp:260-326).
#include <algorithm>
#include <cmath>
#include <map>
#include <string>
#include <vector>

#include "../../include/rrsvd_b200.h"
#include "pipeline.cuh"

using namespace rb;

struct rrsvd_b200_mps {
    rrsvd_b200_ctx* c = nullptr;
    int n = 0;
    std::vector<int> d, dl, dr;
    size_t chi_max = 0;
    double tol = 0.0;
    std::vector<cplx*> g;       // Γ per site (device), dl x d x dr
    std::vector<size_t> gcap;   // capacity in elements
    std::vector<double*> lam;   // λ per bond (device)
    std::vector<size_t> lcap;
    // chain-block edges: λ of the bonds outside the block (null = open chain end)
    double* edge[2] = {nullptr, nullptr};
    size_t edge_n[2] = {0, 0};
    size_t edge_cap[2] = {0, 0};
    const double* ll_of(int b) const { return b > 0 ? lam[b - 1] : edge[0]; }
    const double* lr_of(int b) const { return b + 2 < n ? lam[b + 1] : edge[1]; }
};

namespace {

template <class F>
int mps_api(rrsvd_b200_mps* s, F&& f) {
    if (s == nullptr || s->c == nullptr) return kContract;
    rrsvd_b200_ctx* c = s->c;
    int code = kOk;
    try {
        cudaSetDevice(c->device);
        f(c);
    } catch (const Fail& e) {
        code = e.code;
    } catch (const std::exception& e) {
        c->err = e.what();
        code = kCuda;
    }
    if (code != kOk) recover_after_failure(c);
    ws_reset(c);
    return code;
}

// Persistent (not per-call) device buffers, stream-ordered.
void ensure_gamma(rrsvd_b200_mps* s, int site, size_t elems) {
    if (s->gcap[site] >= elems) return;
    rrsvd_b200_ctx* c = s->c;
    if (s->g[site]) cudaFreeAsync(s->g[site], c->stream);
    s->g[site] = nullptr;
    check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&s->g[site]), elems * sizeof(cplx), c->stream), "alloc gamma");
    s->gcap[site] = elems;
}
void ensure_lambda(rrsvd_b200_mps* s, int bond, size_t elems) {
    if (s->lcap[bond] >= elems) return;
    rrsvd_b200_ctx* c = s->c;
    if (s->lam[bond]) cudaFreeAsync(s->lam[bond], c->stream);
    s->lam[bond] = nullptr;
    check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&s->lam[bond]), elems * sizeof(double), c->stream), "alloc lambda");
    s->lcap[bond] = elems;
}

// Growth without freeing: the old buffer may still be read by work being enqueued; the caller
// frees `old` after the streams that read it have joined.
// A replaced buffer, kept until the sweep's results are validated: freed after a good update,
// swapped back (and the new buffer freed) when the bond's Θ was rejected.
struct Regrown {
    int kind;  // 0 gamma, 1 lambda
    int idx;
    void* old;
    size_t old_cap;
};

void grow_gamma(rrsvd_b200_mps* s, int site, size_t elems, std::vector<Regrown>& old) {
    if (s->gcap[site] >= elems) return;
    old.push_back({0, site, s->g[site], s->gcap[site]});
    s->g[site] = nullptr;
    check_cuda(s->c, cudaMallocAsync(reinterpret_cast<void**>(&s->g[site]), elems * sizeof(cplx), s->c->stream),
               "alloc gamma");
    s->gcap[site] = elems;
}
void grow_lambda(rrsvd_b200_mps* s, int bond, size_t elems, std::vector<Regrown>& old) {
    if (s->lcap[bond] >= elems) return;
    old.push_back({1, bond, s->lam[bond], s->lcap[bond]});
    s->lam[bond] = nullptr;
    check_cuda(s->c, cudaMallocAsync(reinterpret_cast<void**>(&s->lam[bond]), elems * sizeof(double), s->c->stream),
               "alloc lambda");
    s->lcap[bond] = elems;
}

}  // namespace

extern "C" {

int rrsvd_b200_mps_create(rrsvd_b200_ctx* c, size_t n_sites, const size_t* site_dims, size_t chi_max,
                          double trunc_tolerance, rrsvd_b200_mps** out) {
    if (c == nullptr || out == nullptr) return kContract;
    *out = nullptr;
    auto* s = new rrsvd_b200_mps();
    s->c = c;
    const int rc = mps_api(s, [&](rrsvd_b200_ctx* cc) {
        if (n_sites < 1 || site_dims == nullptr) throw_contract(cc, "mps_product_state: one local state per site required");
        s->n = (int)n_sites;
        s->chi_max = chi_max;
        s->tol = trunc_tolerance;
        s->d.assign(site_dims, site_dims + n_sites);
        for (int x : s->d)
            if (x < 1) throw_contract(cc, "mps_product_state: local state dimension mismatch");
        s->dl.assign(n_sites, 1);
        s->dr.assign(n_sites, 1);
        s->g.assign(n_sites, nullptr);
        s->gcap.assign(n_sites, 0);
        s->lam.assign(n_sites > 1 ? n_sites - 1 : 0, nullptr);
        s->lcap.assign(s->lam.size(), 0);
        std::vector<cplx> e0;
        for (int site = 0; site < s->n; ++site) {
            ensure_gamma(s, site, (size_t)s->d[site]);
            e0.assign(s->d[site], mk(0.0, 0.0));
            e0[0] = mk(1.0, 0.0);
            check_cuda(cc, cudaMemcpyAsync(s->g[site], e0.data(), e0.size() * sizeof(cplx), cudaMemcpyHostToDevice, cc->stream), "H2D");
            check_cuda(cc, cudaStreamSynchronize(cc->stream), "sync");
        }
        const double one = 1.0;
        for (size_t b = 0; b < s->lam.size(); ++b) {
            ensure_lambda(s, (int)b, 1);
            check_cuda(cc, cudaMemcpyAsync(s->lam[b], &one, sizeof(double), cudaMemcpyHostToDevice, cc->stream), "H2D");
        }
        check_cuda(cc, cudaStreamSynchronize(cc->stream), "sync");
    });
    if (rc != kOk) {
        rrsvd_b200_mps_destroy(s);
        return rc;
    }
    *out = s;
    return kOk;
}

void rrsvd_b200_mps_destroy(rrsvd_b200_mps* s) {
    if (s == nullptr) return;
    if (s->c) {
        cudaSetDevice(s->c->device);
        for (cplx* p : s->g)
            if (p) cudaFreeAsync(p, s->c->stream);
        for (double* p : s->lam)
            if (p) cudaFreeAsync(p, s->c->stream);
        for (double* p : s->edge)
            if (p) cudaFreeAsync(p, s->c->stream);
        cudaStreamSynchronize(s->c->stream);
    }
    delete s;
}

int rrsvd_b200_mps_set_site(rrsvd_b200_mps* s, size_t site, size_t dim_left, size_t dim_right,
                            const double* gamma, const double* lambda_right) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        if (site >= (size_t)s->n) throw_contract(c, "mps_set_site: bad site");
        if (dim_left < 1 || dim_right < 1) throw_contract(c, "mps_set_site: bond dimensions must be >= 1");
        if (site == 0 && dim_left != 1 && s->edge[0] == nullptr)
            throw_contract(c, "mps_set_site: open left end needs dim_left = 1 (or edge lambdas)");
        if (site + 1 == (size_t)s->n && dim_right != 1 && s->edge[1] == nullptr)
            throw_contract(c, "mps_set_site: open right end needs dim_right = 1 (or edge lambdas)");
        const size_t elems = dim_left * s->d[site] * dim_right;
        ensure_gamma(s, (int)site, elems);
        check_cuda(c, cudaMemcpyAsync(s->g[site], gamma, elems * sizeof(cplx), cudaMemcpyDefault, c->stream), "set gamma");
        if (lambda_right != nullptr && site + 1 < (size_t)s->n) {
            ensure_lambda(s, (int)site, dim_right);
            check_cuda(c, cudaMemcpyAsync(s->lam[site], lambda_right, dim_right * sizeof(double), cudaMemcpyDefault, c->stream),
                       "set lambda");
        }
        s->dl[site] = (int)dim_left;
        s->dr[site] = (int)dim_right;
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    });
}

int rrsvd_b200_mps_set_edge_lambdas(rrsvd_b200_mps* s, const double* left, size_t n_left, const double* right,
                                    size_t n_right) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        const double* src[2] = {left, right};
        const size_t cnt[2] = {n_left, n_right};
        for (int e = 0; e < 2; ++e) {
            if (src[e] == nullptr) {
                if (s->edge[e]) cudaFreeAsync(s->edge[e], c->stream);
                s->edge[e] = nullptr;
                s->edge_n[e] = s->edge_cap[e] = 0;
                continue;
            }
            if (s->edge_cap[e] < cnt[e]) {
                if (s->edge[e]) cudaFreeAsync(s->edge[e], c->stream);
                check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&s->edge[e]), std::max<size_t>(cnt[e], 1) * sizeof(double),
                                              c->stream), "alloc edge");
                s->edge_cap[e] = cnt[e];
            }
            s->edge_n[e] = cnt[e];
            check_cuda(c, cudaMemcpyAsync(s->edge[e], src[e], cnt[e] * sizeof(double), cudaMemcpyDefault, c->stream),
                       "set edge");
        }
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    });
}

int rrsvd_b200_mps_get_site(rrsvd_b200_mps* s, size_t site, size_t* dims3, double* gamma, double* lambda_right) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        if (site >= (size_t)s->n) throw_contract(c, "mps_get_site: bad site");
        if (dims3) {
            dims3[0] = s->dl[site];
            dims3[1] = s->d[site];
            dims3[2] = s->dr[site];
        }
        const size_t elems = (size_t)s->dl[site] * s->d[site] * s->dr[site];
        if (gamma) check_cuda(c, cudaMemcpyAsync(gamma, s->g[site], elems * sizeof(cplx), cudaMemcpyDefault, c->stream), "get gamma");
        if (lambda_right && site + 1 < (size_t)s->n)
            check_cuda(c, cudaMemcpyAsync(lambda_right, s->lam[site], s->dr[site] * sizeof(double), cudaMemcpyDefault, c->stream),
                       "get lambda");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    });
}

int rrsvd_b200_state_upload(rrsvd_b200_mps* s, const size_t* dims, const double* const* gammas,
                            const double* const* lambdas) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        if (dims == nullptr || gammas == nullptr) throw_contract(c, "state_upload: dims and gammas are required");
        for (int site = 0; site < s->n; ++site) {
            const size_t dl = dims[3 * site], dr = dims[3 * site + 2];
            if (dl < 1 || dr < 1) throw_contract(c, "state_upload: bond dimensions must be >= 1");
            if (site > 0 && dl != dims[3 * (site - 1) + 2]) throw_contract(c, "state_upload: bond dimensions disagree");
            if (site == 0 && dl != 1 && s->edge[0] == nullptr)
                throw_contract(c, "state_upload: open left end needs dim_left = 1 (or edge lambdas)");
            if (site + 1 == s->n && dr != 1 && s->edge[1] == nullptr)
                throw_contract(c, "state_upload: open right end needs dim_right = 1 (or edge lambdas)");
            if (gammas[site] == nullptr) throw_contract(c, "state_upload: missing gamma");
        }
        for (int site = 0; site < s->n; ++site) {
            const size_t dl = dims[3 * site], dr = dims[3 * site + 2];
            const size_t elems = dl * s->d[site] * dr;
            ensure_gamma(s, site, elems);
            check_cuda(c, cudaMemcpyAsync(s->g[site], gammas[site], elems * sizeof(cplx), cudaMemcpyDefault, c->stream),
                       "upload gamma");
            if (lambdas != nullptr && lambdas[site] != nullptr && site + 1 < s->n) {
                ensure_lambda(s, site, dr);
                check_cuda(c, cudaMemcpyAsync(s->lam[site], lambdas[site], dr * sizeof(double), cudaMemcpyDefault, c->stream),
                           "upload lambda");
            }
            s->dl[site] = (int)dl;
            s->dr[site] = (int)dr;
        }
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    });
}

int rrsvd_b200_state_download(rrsvd_b200_mps* s, size_t* dims, double* const* gammas, double* const* lambdas) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        for (int site = 0; site < s->n; ++site) {
            if (dims) {
                dims[3 * site] = s->dl[site];
                dims[3 * site + 1] = s->d[site];
                dims[3 * site + 2] = s->dr[site];
            }
            const size_t elems = (size_t)s->dl[site] * s->d[site] * s->dr[site];
            if (gammas != nullptr && gammas[site] != nullptr)
                check_cuda(c, cudaMemcpyAsync(gammas[site], s->g[site], elems * sizeof(cplx), cudaMemcpyDefault, c->stream),
                           "download gamma");
            if (lambdas != nullptr && lambdas[site] != nullptr && site + 1 < s->n)
                check_cuda(c, cudaMemcpyAsync(lambdas[site], s->lam[site], s->dr[site] * sizeof(double), cudaMemcpyDefault,
                                              c->stream), "download lambda");
        }
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    });
}

}  // extern "C"

// A gate resident on the device with its exact block structure (made once, reused by every
// sweep and every evolve call).
struct rrsvd_b200_gate {
    rrsvd_b200_ctx* c = nullptr;
    int dd = 0;
    cplx* dev = nullptr;
    bool blocked = false;
    GateBlocksOwned blk;
};

namespace {

rrsvd_b200_gate* prepare_gate(rrsvd_b200_ctx* c, const double* G, size_t dd) {
    auto* g = new rrsvd_b200_gate();
    g->c = c;
    g->dd = (int)dd;
    try {
        check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&g->dev), dd * dd * sizeof(cplx), c->stream), "alloc gate");
        check_cuda(c, cudaMemcpyAsync(g->dev, G, dd * dd * sizeof(cplx), cudaMemcpyDefault, c->stream), "stage gate");
        // excitation-number-conserving gates are block-diagonal up to a permutation
        g->blocked = dd > 16 && make_gate_blocks(c, g->dev, (int)dd, g->blk);
    } catch (...) {
        if (g->dev) cudaFreeAsync(g->dev, c->stream);
        delete g;
        throw;
    }
    return g;
}

void release_gate(rrsvd_b200_gate* g) {
    if (g == nullptr) return;
    if (g->c) {
        free_gate_blocks(g->c, g->blk);
        if (g->dev) cudaFreeAsync(g->dev, g->c->stream);
    }
    delete g;
}

void evolve_core(rrsvd_b200_mps* s, rrsvd_b200_ctx* c, size_t n_sweeps, const rrsvd_b200_sweep* sweeps,
                 const rrsvd_b200_gate* const* gates, size_t n_steps, rrsvd_b200_backend* be,
                 const rrsvd_b200_evolve_options* opt, rrsvd_b200_evolve_diag* diag,
                 rrsvd_b200_update_record* records, size_t max_records) {
    {
        if (be == nullptr || diag == nullptr || (n_sweeps && (sweeps == nullptr || gates == nullptr)))
            throw_contract(c, "evolve: null argument");
        const int n = s->n, nb = n - 1;
        const double abort_thr = opt ? opt->abort_discarded_threshold : 1.0;
        const int renorm = opt ? opt->renormalize : 1;
        const int omode = opt ? opt->omega_mode : RRSVD_B200_OMEGA_REFERENCE;
        for (size_t sw = 0; sw < n_sweeps; ++sw)
            for (int b = 0; b < nb; ++b) {
                const rrsvd_b200_gate* g = gates[sw * nb + b];
                if (g != nullptr && g->dd != s->d[b] * s->d[b + 1])
                    throw_contract(c, "evolve: term dimension mismatch");
            }

        DecimScalars* sc_dev = nullptr;
        size_t sc_cap = 0;
        struct ScGuard {
            rrsvd_b200_ctx* c;
            void* p;
            ~ScGuard() {
                if (p) cudaFreeAsync(p, c->stream);
            }
        } scg{c, nullptr};
        cudaEvent_t ev[4];
        for (auto& e : ev) e = pooled_event(c);
        struct EvGuard {
            rrsvd_b200_ctx* c;
            cudaEvent_t* e;
            ~EvGuard() { for (int i = 0; i < 4; ++i) c->event_pool.push_back(e[i]); }
        } evg{c, ev};

        diag->kept_fraction = 1.0;
        diag->aborted = 0;
        diag->abort_step = 0;
        diag->n_updates = 0;
        uint64_t maxb = 1;
        for (int b = 0; b < nb; ++b) maxb = std::max<uint64_t>(maxb, (uint64_t)s->dr[b]);
        diag->max_bond_dim = maxb;

        // All bonds of one sweep share a parity, hence no site: they are independent
        // and go through every stage of the pipeline as ONE batch.  The results
        // equal the reference's bond-by-bond order (tebd.cpp:291-306), including the per-call
        // seeds, which are assigned in ascending bond order.
        for (size_t step = 0; step < n_steps; ++step) {
            for (size_t sw = 0; sw < n_sweeps; ++sw) {
                std::vector<int> bonds;
                for (int b = sweeps[sw].bond_parity; b < nb; b += 2)
                    if (gates[sw * nb + b] != nullptr) bonds.push_back(b);
                if (bonds.empty()) continue;
                const size_t nbnd = bonds.size();
                if (sc_cap < nbnd) {
                    if (sc_dev) cudaFreeAsync(sc_dev, c->stream);
                    check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&sc_dev), nbnd * sizeof(DecimScalars), c->stream),
                               "alloc scalars");
                    sc_cap = nbnd;
                    scg.p = sc_dev;
                }
                auto* sc_host = static_cast<DecimScalars*>(pinned_scratch(c, nbnd * sizeof(DecimScalars)));
                std::vector<DecimPlan> plans(nbnd);
                std::vector<uint64_t> seeds(nbnd);
                // Inputs of Θ are the CURRENT buffers; outputs that need more room get NEW
                // buffers, and the old ones are freed only after both lanes have joined.
                std::vector<cplx*> gin1(nbnd), gin2(nbnd);
                std::vector<double*> lin(nbnd);
                std::vector<std::vector<Regrown>> regrown(nbnd);
                // An abort (tebd.cpp:317-321) leaves the bonds after the offending one untouched;
                // the batch updates them all, so with an abort threshold in force the sweep's
                // inputs are snapshotted and those bonds restored if it fires.
                struct Snap {
                    cplx *g1, *g2;
                    double* lam;
                    int chi;
                    size_t n1, n2;
                };
                std::vector<Snap> snaps;
                if (abort_thr < 1.0) {
                    for (size_t i = 0; i < nbnd; ++i) {
                        const int b = bonds[i];
                        Snap sn;
                        sn.chi = s->dr[b];
                        sn.n1 = (size_t)s->dl[b] * s->d[b] * s->dr[b];
                        sn.n2 = (size_t)s->dl[b + 1] * s->d[b + 1] * s->dr[b + 1];
                        sn.g1 = ws_get<cplx>(c, sn.n1);
                        sn.g2 = ws_get<cplx>(c, sn.n2);
                        sn.lam = ws_get<double>(c, (size_t)sn.chi);
                        check_cuda(c, cudaMemcpyAsync(sn.g1, s->g[b], sn.n1 * sizeof(cplx), cudaMemcpyDeviceToDevice,
                                                      c->stream), "snapshot");
                        check_cuda(c, cudaMemcpyAsync(sn.g2, s->g[b + 1], sn.n2 * sizeof(cplx),
                                                      cudaMemcpyDeviceToDevice, c->stream), "snapshot");
                        check_cuda(c, cudaMemcpyAsync(sn.lam, s->lam[b], (size_t)sn.chi * sizeof(double),
                                                      cudaMemcpyDeviceToDevice, c->stream), "snapshot");
                        snaps.push_back(sn);
                    }
                }
                for (size_t i = 0; i < nbnd; ++i) {
                    const int b = bonds[i];
                    // with the accuracy check a bond may grow past chi_max (tebd.cpp:177-179):
                    // its plan's kmax is then the minor dimension
                    plans[i] = plan_decimation(s->d[b], s->d[b + 1], s->dl[b], s->dr[b + 1], s->chi_max, be->kind,
                                               be->target_rank, be->oversampling, be->det_crossover,
                                               be->accuracy_check, be->probe_count);
                    seeds[i] = be->seed++;  // ascending bond order, as the reference (tebd.cpp:162)
                    gin1[i] = s->g[b];
                    gin2[i] = s->g[b + 1];
                    lin[i] = s->lam[b];
                    grow_gamma(s, b, (size_t)plans[i].m * plans[i].kmax, regrown[i]);
                    grow_gamma(s, b + 1, (size_t)plans[i].kmax * plans[i].n, regrown[i]);
                    grow_lambda(s, b, (size_t)plans[i].kmax, regrown[i]);
                }
                check_cuda(c, cudaEventRecord(ev[0], c->stream), "event");
                const cudaStream_t main_stream = c->stream;
                static const int env_lanes = [] {
                    const char* e = std::getenv("RRSVD_B200_LANES");
                    return e ? std::atoi(e) : 0;
                }();
                const int want = env_lanes > 0 ? env_lanes : c->n_lanes;
                bool syncs = false;  // lanes are submitted in turn: a host-synchronising batch serialises them
                for (size_t i = 0; i < nbnd; ++i) syncs = syncs || decimation_syncs_host(plans[i]);
                const int nl = c->use_lanes && !syncs
                                   ? std::max(1, std::min<int>({want, (int)nbnd, rrsvd_b200_ctx::kMaxLanes}))
                                   : 1;
                if (nl > 1) lanes_fork(c, nl);
                StreamSwitch lane_switch(c);  // c->stream is back on main_stream on every exit path
                for (int lane = 0; lane < nl; ++lane) {
                    if (nl > 1) c->stream = c->lane[lane];
                    std::vector<ThetaJob> tj;
                    std::vector<GateJob> gj;
                    std::vector<DecimJob> dj;
                    for (size_t i = lane; i < nbnd; i += nl) {
                        const int b = bonds[i];
                        const int d1 = s->d[b], d2 = s->d[b + 1];
                        const int cl = s->dl[b], cm = s->dr[b], cr = s->dr[b + 1];
                        cplx* M1 = ws_get<cplx>(c, (size_t)plans[i].m * plans[i].n);
                        cplx* M2 = ws_get<cplx>(c, (size_t)plans[i].m * plans[i].n);
                        const double* ll = s->ll_of(b);
                        const double* lr = s->lr_of(b);
                        tj.push_back({gin1[i], gin2[i], ll, lin[i], lr, cl, d1, cm, d2, cr, M1});
                        const rrsvd_b200_gate* G = gates[sw * nb + b];
                        gj.push_back({G->dev, d1, d2, cl, cr, M1, M2, G->blocked ? &G->blk.dev : nullptr});
                        DecimJob job{plans[i], M2, d1, cr, ll, lr, s->chi_max, s->tol, (int)be->power_iterations,
                                     seeds[i], omode, nullptr, renorm, s->g[b], s->lam[b], s->g[b + 1], sc_dev + i};
                        job.eps = be->epsilon;
                        dj.push_back(job);
                    }
                    build_theta_many(c, tj);
                    if (lane == 0) check_cuda(c, cudaEventRecord(ev[1], c->stream), "event");
                    apply_gate_many(c, gj);
                    if (lane == 0) check_cuda(c, cudaEventRecord(ev[2], c->stream), "event");
                    decimate_many(c, dj);
                }
                c->stream = main_stream;
                if (nl > 1) lanes_join(c, nl);
                check_cuda(c, cudaEventRecord(ev[3], c->stream), "event");
                check_cuda(c, cudaMemcpyAsync(sc_host, sc_dev, nbnd * sizeof(DecimScalars), cudaMemcpyDeviceToHost,
                                              c->stream), "D2H");
                check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
                if (c->gemm_timing) flush_gemm_timing(c);
                float t01 = 0, t12 = 0, t23 = 0;
                cudaEventElapsedTime(&t01, ev[0], ev[1]);
                cudaEventElapsedTime(&t12, ev[1], ev[2]);
                cudaEventElapsedTime(&t23, ev[2], ev[3]);
                // Validate every bond before committing any (the reference throws before it
                // assigns, tebd.cpp:156-160).  A rejected bond's truncation kept nothing on the
                // device, so its Γ/λ buffers were not written: its grown buffers are swapped
                // back, the other bonds of the batch (valid results) are committed, and the seed
                // counter is left where the reference's would be — the rejected call takes no
                // seed (tebd.cpp:162 follows the check).
                size_t first_bad = nbnd;
                for (size_t i = 0; i < nbnd && first_bad == nbnd; ++i)
                    if (sc_host[i].nonfinite || !(sc_host[i].total_sq > 0.0)) first_bad = i;
                for (size_t i = 0; i < nbnd; ++i) {
                    const bool bad = sc_host[i].nonfinite || !(sc_host[i].total_sq > 0.0);
                    for (const Regrown& r : regrown[i]) {
                        if (!bad) {
                            if (r.old) cudaFreeAsync(r.old, c->stream);
                            continue;
                        }
                        void*& cur = r.kind == 0 ? reinterpret_cast<void*&>(s->g[r.idx])
                                                 : reinterpret_cast<void*&>(s->lam[r.idx]);
                        if (cur) cudaFreeAsync(cur, c->stream);
                        cur = r.old;
                        (r.kind == 0 ? s->gcap[r.idx] : s->lcap[r.idx]) = r.old_cap;
                    }
                    if (!bad) {
                        s->dr[bonds[i]] = sc_host[i].kept;
                        s->dl[bonds[i] + 1] = sc_host[i].kept;
                    }
                }
                if (first_bad < nbnd) {
                    be->seed = seeds[first_bad];
                    if (sc_host[first_bad].nonfinite) throw_contract(c, "decimate: theta has non-finite entries");
                    throw_contract(c, "decimate: theta is identically zero");
                }
                for (size_t i = 0; i < nbnd; ++i) {
                    const int b = bonds[i];
                    const DecimScalars& h = sc_host[i];
                    s->dr[b] = h.kept;
                    s->dl[b + 1] = h.kept;
                    diag->kept_fraction *= 1.0 - h.discarded;
                    diag->max_bond_dim = std::max<uint64_t>(diag->max_bond_dim, (uint64_t)h.kept);
                    if (records && diag->n_updates < max_records)  // batched: stage times shared evenly
                        records[diag->n_updates] = {step, (uint64_t)b, (uint64_t)h.kept, h.discarded,
                                                    1e3 * t01 / nbnd, 1e3 * t12 / nbnd, 1e3 * t23 / nbnd,
                                                    plans[i].randomized ? 1 : 0};
                    diag->n_updates++;
                    if (1.0 - diag->kept_fraction > abort_thr) {  // tebd.cpp:317-321
                        diag->aborted = 1;
                        diag->abort_step = step;
                        // the reference returns here: the later bonds of the batch take no
                        // seed (tebd.cpp:162, 317-321)
                        be->seed -= (uint64_t)(nbnd - i - 1);
                        for (size_t j = i + 1; j < nbnd; ++j) {  // un-apply the later bonds of the batch
                            const int bj = bonds[j];
                            const Snap& sn = snaps[j];
                            check_cuda(c, cudaMemcpyAsync(s->g[bj], sn.g1, sn.n1 * sizeof(cplx),
                                                          cudaMemcpyDeviceToDevice, c->stream), "restore");
                            check_cuda(c, cudaMemcpyAsync(s->g[bj + 1], sn.g2, sn.n2 * sizeof(cplx),
                                                          cudaMemcpyDeviceToDevice, c->stream), "restore");
                            check_cuda(c, cudaMemcpyAsync(s->lam[bj], sn.lam, (size_t)sn.chi * sizeof(double),
                                                          cudaMemcpyDeviceToDevice, c->stream), "restore");
                            s->dr[bj] = sn.chi;
                            s->dl[bj + 1] = sn.chi;
                        }
                        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
                        ws_reset(c);
                        return;
                    }
                }
                ws_reset(c);
            }
        }
    }
}

}  // namespace

extern "C" {

int rrsvd_b200_gate_create(rrsvd_b200_ctx* c, const double* G, size_t dd, rrsvd_b200_gate** out) {
    if (c == nullptr || out == nullptr) return kContract;
    *out = nullptr;
    int code = kOk;
    try {
        cudaSetDevice(c->device);
        if (G == nullptr || dd == 0) throw_contract(c, "gate_create: empty gate");
        *out = prepare_gate(c, G, dd);
    } catch (const Fail& e) {
        code = e.code;
    }
    return code;
}

void rrsvd_b200_gate_destroy(rrsvd_b200_gate* g) {
    if (g && g->c) cudaSetDevice(g->c->device);
    release_gate(g);
}

int rrsvd_b200_gate_blocks(const rrsvd_b200_gate* g, size_t* nblocks) {
    if (g == nullptr) return 0;
    if (nblocks) *nblocks = g->blocked ? (size_t)g->blk.dev.nblocks : 1;
    return g->blocked ? 1 : 0;
}

int rrsvd_b200_evolve_prepared(rrsvd_b200_mps* s, size_t n_sweeps, const rrsvd_b200_sweep* sweeps,
                               const rrsvd_b200_gate* const* gates, size_t n_steps, rrsvd_b200_backend* be,
                               const rrsvd_b200_evolve_options* opt, rrsvd_b200_evolve_diag* diag,
                               rrsvd_b200_update_record* records, size_t max_records) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        evolve_core(s, c, n_sweeps, sweeps, gates, n_steps, be, opt, diag, records, max_records);
    });
}

// Raw gate matrices: each distinct gate (the reference builds one per (bond, coefficient),
// tebd.cpp:276-285) is prepared for this call only.  Repeated calls should prepare gates once
// with rrsvd_b200_gate_create and use rrsvd_b200_evolve_prepared.
int rrsvd_b200_evolve(rrsvd_b200_mps* s, size_t n_sweeps, const rrsvd_b200_sweep* sweeps, const double* const* gates,
                      size_t n_steps, rrsvd_b200_backend* be, const rrsvd_b200_evolve_options* opt,
                      rrsvd_b200_evolve_diag* diag, rrsvd_b200_update_record* records, size_t max_records) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        if (n_sweeps && (sweeps == nullptr || gates == nullptr)) throw_contract(c, "evolve: null argument");
        const int nb = s->n - 1;
        std::map<const double*, rrsvd_b200_gate*> made;
        struct Guard {
            std::map<const double*, rrsvd_b200_gate*>& m;
            ~Guard() { for (auto& kv : m) release_gate(kv.second); }
        } guard{made};
        std::vector<const rrsvd_b200_gate*> table(n_sweeps * nb, nullptr);
        for (size_t sw = 0; sw < n_sweeps; ++sw)
            for (int b = 0; b < nb; ++b) {
                const double* gp = gates[sw * nb + b];
                if (gp == nullptr) continue;
                auto it = made.find(gp);
                if (it == made.end())
                    it = made.emplace(gp, prepare_gate(c, gp, (size_t)s->d[b] * s->d[b + 1])).first;
                table[sw * nb + b] = it->second;
            }
        evolve_core(s, c, n_sweeps, sweeps, table.data(), n_steps, be, opt, diag, records, max_records);
    });
}

int rrsvd_b200_expectation_local(rrsvd_b200_mps* s, size_t site, const double* op, double* out2) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        if (site >= (size_t)s->n) throw_contract(c, "expectation_local: bad site");
        if (op == nullptr || out2 == nullptr) throw_contract(c, "expectation_local: null argument");
        const int d = s->d[site];
        const auto* dop = static_cast<const cplx*>(stage_in(c, op, (size_t)d * d * sizeof(cplx)));
        const double* ll = site > 0 ? s->lam[site - 1] : s->edge[0];
        const double* lr = site + 1 < (size_t)s->n ? s->lam[site] : s->edge[1];
        double* res = ws_get<double>(c, 2 * kNumSMs * 2 + 2);
        check_cuda(c, expectation_local_dev(s->g[site], s->dl[site], d, s->dr[site], ll, lr, dop, res, c->stream),
                   "expectation_local");
        c->launches += 2;
        double h[2];
        check_cuda(c, cudaMemcpyAsync(h, res + 4 * kNumSMs, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
        out2[0] = h[0];
        out2[1] = h[1];
    });
}

int rrsvd_b200_schmidt_entropy(rrsvd_b200_mps* s, size_t bond, double* out) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        if (bond + 1 >= (size_t)s->n) throw_contract(c, "schmidt_entropy: bad bond");
        double* res = ws_get<double>(c, 1);
        check_cuda(c, schmidt_entropy_dev(s->lam[bond], s->dr[bond], res, c->stream), "schmidt_entropy");
        c->launches++;
        check_cuda(c, cudaMemcpyAsync(out, res, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    });
}

}  // extern "C"

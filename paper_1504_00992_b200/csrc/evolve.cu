// evolve.cu — device-resident MpsState and the TEBD sweep driver (tebd.cpp:260-326).
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <map>
#include <string>
#include <vector>

#include "../../include/rrsvd_b200.h"
#include "mps.cuh"

using namespace rb;

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

// The state through host memory and back, pipelined per site: site s goes device -> host on the
// context stream and, as soon as it has landed, host -> device on lane 0 (the two copy engines run
// in parallel across sites).  The host buffers hold the state afterwards; the device state is the
// one re-uploaded from them.  Dims are unchanged (a consecutive-steps round trip).
int rrsvd_b200_state_roundtrip(rrsvd_b200_mps* s, double* const* gammas, double* const* lambdas) {
    return mps_api(s, [&](rrsvd_b200_ctx* c) {
        if (gammas == nullptr) throw_contract(c, "state_roundtrip: gammas are required");
        for (int site = 0; site < s->n; ++site)
            if (gammas[site] == nullptr) throw_contract(c, "state_roundtrip: missing gamma");
        lanes_fork(c, 1);  // lane 0 orders after everything queued so far
        const cudaStream_t up = c->lane[0];
        std::vector<cudaEvent_t> ev(s->n, nullptr);
        struct Events {
            std::vector<cudaEvent_t>& v;
            ~Events() {
                for (cudaEvent_t e : v)
                    if (e) cudaEventDestroy(e);
            }
        } guard{ev};
        for (int site = 0; site < s->n; ++site) {
            const size_t elems = (size_t)s->dl[site] * s->d[site] * s->dr[site];
            const bool lam = lambdas != nullptr && lambdas[site] != nullptr && site + 1 < s->n;
            check_cuda(c, cudaMemcpyAsync(gammas[site], s->g[site], elems * sizeof(cplx), cudaMemcpyDefault, c->stream),
                       "download gamma");
            if (lam)
                check_cuda(c, cudaMemcpyAsync(lambdas[site], s->lam[site], s->dr[site] * sizeof(double), cudaMemcpyDefault,
                                              c->stream), "download lambda");
            check_cuda(c, cudaEventCreateWithFlags(&ev[site], cudaEventDisableTiming), "event");
            check_cuda(c, cudaEventRecord(ev[site], c->stream), "event");
            check_cuda(c, cudaStreamWaitEvent(up, ev[site], 0), "event wait");
            check_cuda(c, cudaMemcpyAsync(s->g[site], gammas[site], elems * sizeof(cplx), cudaMemcpyDefault, up),
                       "upload gamma");
            if (lam)
                check_cuda(c, cudaMemcpyAsync(s->lam[site], lambdas[site], s->dr[site] * sizeof(double), cudaMemcpyDefault,
                                              up), "upload lambda");
        }
        lanes_join(c, 1);
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    });
}

}  // extern "C"

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

// One enqueued sweep — every bond of one parity as one batch — awaiting its scalars.  Its
// decimations write FRESH Γ/λ buffers: the inputs stay intact until the sweep is committed, so
// a rejected Θ, an abort (tebd.cpp:317-321) or a mispredicted speculative successor is undone by
// restoring pointers, never by copying data back.
struct InFlight {
    size_t step = 0, sweep = 0;
    std::vector<int> bonds;
    std::vector<DecimPlan> plans;
    std::vector<uint64_t> seeds;
    DecimScalars* sc_dev = nullptr;
    DecimScalars* sc_host = nullptr;  // pinned slot
    cudaEvent_t ev[4] = {};           // Θ | gate | decimate | end marks on lane 0
    cudaEvent_t done = nullptr;       // after the scalars' D2H
    struct Swap {
        cplx* g_old[2];
        size_t gcap_old[2];
        cplx* g_new[2];
        size_t gcap_new[2];
        double* l_old;
        size_t lcap_old;
        double* l_new;
        size_t lcap_new;
        int dim_old;  // the bond dimension before the sweep
    };
    std::vector<Swap> swaps;
    bool predicted = false;  // a successor was enqueued assuming kept == kmax on every bond
};

void release_events(rrsvd_b200_ctx* c, InFlight& f) {
    for (cudaEvent_t& e : f.ev)
        if (e) c->event_pool.push_back(e), e = nullptr;
    if (f.done) c->event_pool.push_back(f.done), f.done = nullptr;
}

// Undo bond i of a sweep: its fresh outputs are dropped, the inputs become current again.
void undo_bond(rrsvd_b200_mps* s, rrsvd_b200_ctx* c, const InFlight& f, size_t i) {
    const int b = f.bonds[i];
    const InFlight::Swap& w = f.swaps[i];
    for (int k = 0; k < 2; ++k) {
        if (w.g_new[k]) cudaFreeAsync(w.g_new[k], c->stream);
        s->g[b + k] = w.g_old[k];
        s->gcap[b + k] = w.gcap_old[k];
    }
    if (w.l_new) cudaFreeAsync(w.l_new, c->stream);
    s->lam[b] = w.l_old;
    s->lcap[b] = w.lcap_old;
    s->dr[b] = w.dim_old;
    s->dl[b + 1] = w.dim_old;
}

// Enqueue one sweep on the current state (host dims may be predicted ones).
void enqueue_sweep(rrsvd_b200_mps* s, rrsvd_b200_ctx* c, InFlight& f, const rrsvd_b200_sweep* sweeps,
                   const rrsvd_b200_gate* const* gates, rrsvd_b200_backend* be, int renorm, int omode,
                   DecimScalars* sc_host) {
    const int nb = s->n - 1;
    const size_t sw = f.sweep;
    for (int b = sweeps[sw].bond_parity; b < nb; b += 2)
        if (gates[sw * nb + b] != nullptr) f.bonds.push_back(b);
    const size_t nbnd = f.bonds.size();
    f.plans.resize(nbnd);
    f.seeds.resize(nbnd);
    f.swaps.reserve(nbnd);  // filled as the buffers are made (an undo covers exactly those)
    f.sc_dev = ws_get<DecimScalars>(c, nbnd);
    f.sc_host = sc_host;
    for (auto& e : f.ev) e = pooled_event(c);
    f.done = pooled_event(c);
    std::vector<cplx*> gin1(nbnd), gin2(nbnd);
    std::vector<double*> lin(nbnd);
    for (size_t i = 0; i < nbnd; ++i) {
        const int b = f.bonds[i];
        // with the accuracy check a bond may grow past chi_max (tebd.cpp:177-179): its plan's
        // kmax is then the minor dimension
        f.plans[i] = plan_decimation(s->d[b], s->d[b + 1], s->dl[b], s->dr[b + 1], s->chi_max, be->kind,
                                     be->target_rank, be->oversampling, be->det_crossover, be->accuracy_check,
                                     be->probe_count);
        f.seeds[i] = be->seed++;  // ascending bond order, as the reference (tebd.cpp:162)
        gin1[i] = s->g[b];
        gin2[i] = s->g[b + 1];
        lin[i] = s->lam[b];
        f.swaps.push_back(InFlight::Swap{});
        InFlight::Swap& w = f.swaps.back();
        w.dim_old = s->dr[b];
        w.g_old[0] = s->g[b];
        w.g_old[1] = s->g[b + 1];
        w.gcap_old[0] = s->gcap[b];
        w.gcap_old[1] = s->gcap[b + 1];
        w.l_old = s->lam[b];
        w.lcap_old = s->lcap[b];
        const size_t need[2] = {(size_t)f.plans[i].m * f.plans[i].kmax, (size_t)f.plans[i].kmax * f.plans[i].n};
        for (int k = 0; k < 2; ++k) {
            check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&w.g_new[k]), need[k] * sizeof(cplx), c->stream),
                       "alloc gamma");
            w.gcap_new[k] = need[k];
            s->g[b + k] = w.g_new[k];
            s->gcap[b + k] = need[k];
        }
        check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&w.l_new), (size_t)f.plans[i].kmax * sizeof(double),
                                      c->stream), "alloc lambda");
        w.lcap_new = f.plans[i].kmax;
        s->lam[b] = w.l_new;
        s->lcap[b] = w.lcap_new;
    }
    check_cuda(c, cudaEventRecord(f.ev[0], c->stream), "event");
    static const int env_lanes = [] {
        const char* e = std::getenv("RRSVD_B200_LANES");
        return e ? std::atoi(e) : 0;
    }();
    const int want = env_lanes > 0 ? env_lanes : c->n_lanes;
    bool syncs = false;  // lanes are submitted in turn: a host-synchronising batch serialises them
    for (size_t i = 0; i < nbnd; ++i) syncs = syncs || decimation_syncs_host(f.plans[i]);
    const int nl = c->use_lanes && !syncs ? std::max(1, std::min<int>({want, (int)nbnd, rrsvd_b200_ctx::kMaxLanes})) : 1;
    const cudaStream_t main_stream = c->stream;
    if (nl > 1) lanes_fork(c, nl);
    {
        StreamSwitch lane_switch(c);  // c->stream is back on main_stream on every exit path
        for (int lane = 0; lane < nl; ++lane) {
            if (nl > 1) c->stream = c->lane[lane];
            std::vector<ThetaJob> tj;
            std::vector<GateJob> gj;
            std::vector<DecimJob> dj;
            for (size_t i = lane; i < nbnd; i += nl) {
                const int b = f.bonds[i];
                const int d1 = s->d[b], d2 = s->d[b + 1];
                const int cl = s->dl[b], cm = f.swaps[i].dim_old, cr = s->dr[b + 1];
                cplx* M1 = ws_get<cplx>(c, (size_t)f.plans[i].m * f.plans[i].n);
                cplx* M2 = ws_get<cplx>(c, (size_t)f.plans[i].m * f.plans[i].n);
                const double* ll = s->ll_of(b);
                const double* lr = s->lr_of(b);
                tj.push_back({gin1[i], gin2[i], ll, lin[i], lr, cl, d1, cm, d2, cr, M1});
                const rrsvd_b200_gate* G = gates[sw * nb + b];
                gj.push_back({G->dev, d1, d2, cl, cr, M1, M2, G->blocked ? &G->blk.dev : nullptr});
                DecimJob job{f.plans[i], M2, d1, cr, ll, lr, s->chi_max, s->tol, (int)be->power_iterations,
                             f.seeds[i], omode, nullptr, renorm, s->g[b], s->lam[b], s->g[b + 1], f.sc_dev + i};
                job.eps = be->epsilon;
                dj.push_back(job);
            }
            build_theta_many(c, tj);
            if (lane == 0) check_cuda(c, cudaEventRecord(f.ev[1], c->stream), "event");
            apply_gate_many(c, gj);
            if (lane == 0) check_cuda(c, cudaEventRecord(f.ev[2], c->stream), "event");
            decimate_many(c, dj);
        }
    }
    if (nl > 1) lanes_join(c, nl);
    check_cuda(c, cudaEventRecord(f.ev[3], c->stream), "event");
    check_cuda(c, cudaMemcpyAsync(f.sc_host, f.sc_dev, nbnd * sizeof(DecimScalars), cudaMemcpyDeviceToHost, c->stream),
               "D2H");
    check_cuda(c, cudaEventRecord(f.done, c->stream), "event");
}

// Drop a (speculative) sweep entirely: its outputs, its seeds.
void rollback_sweep(rrsvd_b200_mps* s, rrsvd_b200_ctx* c, InFlight& f, rrsvd_b200_backend* be) {
    for (size_t i = f.swaps.size(); i-- > 0;) undo_bond(s, c, f, i);
    if (!f.seeds.empty()) be->seed = f.seeds[0];
    release_events(c, f);
}

}  // namespace

namespace rb {
void evolve_core(rrsvd_b200_mps* s, rrsvd_b200_ctx* c, size_t n_sweeps, const rrsvd_b200_sweep* sweeps,
                 const rrsvd_b200_gate* const* gates, size_t n_steps, rrsvd_b200_backend* be,
                 const rrsvd_b200_evolve_options* opt, rrsvd_b200_evolve_diag* diag,
                 rrsvd_b200_update_record* records, size_t max_records) {
    if (be == nullptr || diag == nullptr || (n_sweeps && (sweeps == nullptr || gates == nullptr)))
        throw_contract(c, "evolve: null argument");
    const int n = s->n, nb = n - 1;
    const double abort_thr = opt ? opt->abort_discarded_threshold : 1.0;
    const int renorm = opt ? opt->renormalize : 1;
    const int omode = opt ? opt->omega_mode : RRSVD_B200_OMEGA_REFERENCE;
    size_t max_bonds = 1;
    for (size_t sw = 0; sw < n_sweeps; ++sw) {
        size_t cnt = 0;
        for (int b = 0; b < nb; ++b) {
            const rrsvd_b200_gate* g = gates[sw * nb + b];
            if (g != nullptr && g->dd != s->d[b] * s->d[b + 1]) throw_contract(c, "evolve: term dimension mismatch");
            cnt += g != nullptr && (b % 2) == sweeps[sw].bond_parity;
        }
        max_bonds = std::max(max_bonds, cnt);
    }
    diag->kept_fraction = 1.0;
    diag->aborted = 0;
    diag->abort_step = 0;
    diag->n_updates = 0;
    uint64_t maxb = 1;
    for (int b = 0; b < nb; ++b) maxb = std::max<uint64_t>(maxb, (uint64_t)s->dr[b]);
    diag->max_bond_dim = maxb;
    if ((int)s->sat.size() != nb) s->sat.assign(nb, 0);

    // The (step, sweep) sequence; sweeps without a term are skipped (tebd.cpp:289-294).
    std::vector<std::pair<size_t, size_t>> order;
    for (size_t step = 0; step < n_steps; ++step)
        for (size_t sw = 0; sw < n_sweeps; ++sw)
            for (int b = sweeps[sw].bond_parity; b < nb; b += 2)
                if (gates[sw * nb + b] != nullptr) {
                    order.push_back({step, sw});
                    break;
                }
    // Speculation: while sweep j runs, sweep j+1 is enqueued assuming every bond of j keeps
    // kmax (saturated bonds keep the χ cap), so the device never idles on the host's read of j's
    // kept χ.  Only when every bond of j kept its kmax last time (per-bond history), never with
    // an abort budget, the accuracy check (data-dependent width) or per-launch GEMM timing.  A
    // misprediction drops sweep j+1's outputs (fresh buffers) and re-enqueues it: the results
    // are those of the one-sweep-at-a-time schedule, always.
    static const bool spec_env = [] {
        const char* e = std::getenv("RRSVD_B200_SPECULATE");
        return e == nullptr || std::atoi(e) != 0;
    }();
    const bool spec_ok = spec_env && abort_thr >= 1.0 && !c->gemm_timing && !be->accuracy_check;
    auto* pinned = static_cast<DecimScalars*>(pinned_sweep_scratch(c, 2 * max_bonds * sizeof(DecimScalars)));
    std::vector<InFlight> q;  // front = q[0]; at most two
    q.reserve(2);
    size_t next = 0, slot = 0;
    auto push = [&](bool) {
        q.emplace_back();
        q.back().step = order[next].first;
        q.back().sweep = order[next].second;
        ++next;
        enqueue_sweep(s, c, q.back(), sweeps, gates, be, renorm, omode, pinned + (slot++ & 1) * max_bonds);
    };
    try {
        if (!order.empty()) push(false);
        while (!q.empty()) {
            InFlight& f = q[0];
            bool predictable = spec_ok && q.size() == 1 && next < order.size();
            // (a batch whose decimation reads results on the host — the block Jacobi's per-sweep
            // convergence — blocks the host inside its own enqueue: measured C2 20.6 vs 21.6
            // steps/s with speculation, so such sweeps are not speculated on)
            for (size_t i = 0; predictable && i < f.bonds.size(); ++i)
                predictable = !decimation_syncs_host(f.plans[i]) && s->sat[f.bonds[i]];
            if (predictable) {
                for (size_t i = 0; i < f.bonds.size(); ++i) {
                    s->dr[f.bonds[i]] = f.plans[i].kmax;
                    s->dl[f.bonds[i] + 1] = f.plans[i].kmax;
                }
                f.predicted = true;
                push(true);
            }
            InFlight& fr = q[0];  // (q may have grown: re-take the reference)
            check_cuda(c, cudaEventSynchronize(fr.done), "sync");
            if (c->gemm_timing) flush_gemm_timing(c);
            const size_t nbnd = fr.bonds.size();
            const DecimScalars* h = fr.sc_host;
            size_t first_bad = nbnd;
            bool mismatch = false;
            for (size_t i = 0; i < nbnd; ++i) {
                const bool bad = h[i].nonfinite || !(h[i].total_sq > 0.0);
                if (bad && first_bad == nbnd) first_bad = i;
                mismatch = mismatch || bad || h[i].kept != fr.plans[i].kmax;
            }
            if (q.size() == 2 && mismatch) {  // the successor ran on wrong dims: drop it
                if (debug_enabled())
                    std::fprintf(stderr, "[rrsvd_b200] evolve: speculative sweep (step %zu, sweep %zu) dropped\n",
                                 q[1].step, q[1].sweep);
                rollback_sweep(s, c, q[1], be);
                q.pop_back();
                --next;
            }
            InFlight& f0 = q[0];
            // The reference applies the bonds one by one (tebd.cpp:291-306): a rejected Θ throws
            // before anything of that call is assigned (tebd.cpp:156-160, no seed taken), an
            // exhausted discarded-weight budget returns after the bond that crossed it
            // (tebd.cpp:317-321).  The batch reproduces exactly that: bonds [0, stop) are
            // committed, the later ones undone (their inputs were never overwritten).
            size_t stop = nbnd;
            bool aborted = false;
            double kf = diag->kept_fraction;
            for (size_t i = 0; i < nbnd; ++i) {
                if (i == first_bad) {
                    stop = i;
                    break;
                }
                kf *= 1.0 - h[i].discarded;
                if (1.0 - kf > abort_thr) {
                    aborted = true;
                    stop = i + 1;
                    break;
                }
            }
            for (size_t j = nbnd; j-- > stop;) undo_bond(s, c, f0, j);
            float t01 = 0, t12 = 0, t23 = 0;
            cudaEventElapsedTime(&t01, f0.ev[0], f0.ev[1]);
            cudaEventElapsedTime(&t12, f0.ev[1], f0.ev[2]);
            cudaEventElapsedTime(&t23, f0.ev[2], f0.ev[3]);
            for (size_t i = 0; i < stop; ++i) {
                const int b = f0.bonds[i];
                const InFlight::Swap& w = f0.swaps[i];
                for (int k = 0; k < 2; ++k)
                    if (w.g_old[k]) cudaFreeAsync(w.g_old[k], c->stream);
                if (w.l_old) cudaFreeAsync(w.l_old, c->stream);
                s->dr[b] = h[i].kept;
                s->dl[b + 1] = h[i].kept;
                s->sat[b] = h[i].kept == f0.plans[i].kmax;
                diag->kept_fraction *= 1.0 - h[i].discarded;
                diag->max_bond_dim = std::max<uint64_t>(diag->max_bond_dim, (uint64_t)h[i].kept);
                if (records && diag->n_updates < max_records)  // batched: stage times shared evenly
                    records[diag->n_updates] = {f0.step, (uint64_t)b, (uint64_t)h[i].kept, h[i].discarded,
                                                1e3 * t01 / nbnd, 1e3 * t12 / nbnd, 1e3 * t23 / nbnd,
                                                f0.plans[i].randomized ? 1 : 0};
                diag->n_updates++;
            }
            if (first_bad < nbnd || aborted) {
                // the calls after `stop` never ran in the reference: they took no seed
                be->seed = f0.seeds[0] + stop;
                const bool nonfin = first_bad < nbnd && h[first_bad].nonfinite != 0;
                const uint64_t step = f0.step;
                release_events(c, f0);
                q.clear();
                if (first_bad < nbnd)
                    throw_contract(c, nonfin ? "decimate: theta has non-finite entries"
                                             : "decimate: theta is identically zero");
                diag->aborted = 1;
                diag->abort_step = step;
                return;
            }
            release_events(c, f0);
            q.erase(q.begin());
            ws_reset(c);  // (stream-ordered frees: a successor in flight keeps running)
            if (q.empty() && next < order.size()) push(false);
        }
    } catch (...) {
        // a failed enqueue or device error: no sweep in flight is applied (the state keeps the
        // last committed sweep; the seed counter its value before them)
        for (size_t k = q.size(); k-- > 0;) rollback_sweep(s, c, q[k], be);
        throw;
    }
}
}  // namespace rb

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

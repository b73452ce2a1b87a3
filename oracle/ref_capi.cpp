// oracle/ref_capi.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A flat extern "C" surface over the UNMODIFIED reference library (the sources under
// /root/reference/proj/core/src are compiled as-is by oracle/Makefile into
// oracle/_ref/librrsvd_ref.so).  Only tests/, __graft_entry__.smoke() and bench.py's CPU
// baseline leg load it, through oracle/ref.py, as the parity checker / CPU timing arm.
// Complex data crosses this boundary as interleaved (re, im) float64, row-major, exactly the
// reference's DenseMatrix / Tensor3 memory (dense_matrix.hpp:26-27, mps.hpp:20-25).
//
// Every entry point returns 0 on success, 1 on rrsvd::contract_violation, 2 on
// rrsvd::numeric_failure, 9 on any other exception; ref_last_error() gives the message.

#include <cblas.h>

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "rrsvd/chainmap.hpp"
#include "rrsvd/errors.hpp"
#include "rrsvd/linalg.hpp"
#include "rrsvd/matgen.hpp"
#include "rrsvd/mps.hpp"
#include "rrsvd/randomized.hpp"
#include "rrsvd/matrix_io.hpp"
#include "rrsvd/tebd.hpp"
#include "experiments.hpp"

using rrsvd::cplx;
using rrsvd::DenseMatrix;
namespace tebd = rrsvd::tebd;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const rrsvd::contract_violation& e) {
        g_err = e.what();
        return 1;
    } catch (const rrsvd::numeric_failure& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

DenseMatrix load(const double* p, std::size_t r, std::size_t c) {
    std::vector<cplx> v(r * c);
    if (r * c) std::memcpy(v.data(), p, r * c * sizeof(cplx));
    return DenseMatrix(r, c, std::move(v));
}

void store(const DenseMatrix& m, double* out) {
    if (m.size()) std::memcpy(out, m.data(), m.size() * sizeof(cplx));
}

void store_cols(const DenseMatrix& m, std::size_t keep, double* out) {
    // first `keep` columns of m, row-major rows x keep
    for (std::size_t i = 0; i < m.rows(); ++i)
        std::memcpy(out + 2 * i * keep, m.data() + i * m.cols(), keep * sizeof(cplx));
}

tebd::Tensor3 load_t3(const double* p, std::size_t l, std::size_t d, std::size_t r) {
    tebd::Tensor3 t(l, d, r);
    if (l * d * r) std::memcpy(t.values.data(), p, l * d * r * sizeof(cplx));
    return t;
}

}  // namespace

extern "C" {

// Mirrors rrsvd::tebd::DecimationBackend (tebd.hpp:65-85) field by field.
struct ref_backend {
    int kind;  // 0 deterministic, 1 randomized
    std::uint64_t target_rank;
    std::uint64_t oversampling;
    std::uint64_t power_iterations;
    int accuracy_check;
    double epsilon;
    std::uint64_t probe_count;
    std::uint64_t det_crossover;
    std::uint64_t seed;  // in/out: advanced by one per decimate call (tebd.cpp:162)
};

struct ref_decim_info {
    double discarded;
    std::uint64_t chi;
    int randomized_path;
    int tolerance_certified;
    int pseudo_inverse_applied;
};

static tebd::DecimationBackend to_backend(const ref_backend* b) {
    tebd::DecimationBackend out;
    out.kind = b->kind ? tebd::DecimationBackend::Kind::Randomized
                       : tebd::DecimationBackend::Kind::Deterministic;
    out.target_rank = b->target_rank;
    out.oversampling = b->oversampling;
    out.power_iterations = b->power_iterations;
    out.accuracy_check = b->accuracy_check != 0;
    out.epsilon = b->epsilon;
    out.probe_count = b->probe_count;
    out.det_crossover = b->det_crossover;
    out.seed = b->seed;
    return out;
}

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { openblas_set_num_threads(n); }
int ref_get_threads() { return openblas_get_num_threads(); }
const char* ref_blas_core() { return openblas_get_corename(); }
const char* ref_blas_config() { return openblas_get_config(); }

// ---- L1/L2: randomized.hpp / linalg.hpp -------------------------------------------------

int ref_gaussian_test_matrix(std::uint64_t n, std::uint64_t l, std::uint64_t seed, double* out) {
    return guarded([&] { store(rrsvd::gaussian_test_matrix(n, l, seed), out); });
}

int ref_gemm(const double* a, std::uint64_t ar, std::uint64_t ac, int adj_a, const double* b,
             std::uint64_t br, std::uint64_t bc, int adj_b, double* c) {
    return guarded([&] {
        store(rrsvd::gemm(load(a, ar, ac), adj_a != 0, load(b, br, bc), adj_b != 0), c);
    });
}

int ref_qr(const double* a, std::uint64_t m, std::uint64_t n, double* q, double* r) {
    return guarded([&] {
        const rrsvd::QrFactors f = rrsvd::qr(load(a, m, n));
        store(f.q, q);
        if (r) store(f.r, r);
    });
}

int ref_frobenius_norm(const double* a, std::uint64_t m, std::uint64_t n, double* out) {
    return guarded([&] { *out = rrsvd::frobenius_norm(load(a, m, n)); });
}

// u: m x min(m,n), s: min(m,n), v: n x min(m,n)
int ref_svd_full(const double* a, std::uint64_t m, std::uint64_t n, double* u, double* s,
                 double* v) {
    return guarded([&] {
        const rrsvd::SvdResult r = rrsvd::svd_full(load(a, m, n));
        store(r.u, u);
        std::memcpy(s, r.sigma.data(), r.sigma.size() * sizeof(double));
        store(r.v, v);
    });
}

int ref_singular_values(const double* a, std::uint64_t m, std::uint64_t n, double* s) {
    return guarded([&] {
        const std::vector<double> r = rrsvd::singular_values(load(a, m, n));
        std::memcpy(s, r.data(), r.size() * sizeof(double));
    });
}

// u: m x l, s: l, v: n x l
int ref_sketched_svd(const double* a, std::uint64_t m, std::uint64_t n, std::uint64_t l,
                     std::uint64_t q, std::uint64_t seed, double* u, double* s, double* v,
                     double* discarded) {
    return guarded([&] {
        const rrsvd::SvdResult r = rrsvd::rrsvd_sketched_svd(load(a, m, n), l, q, seed);
        store(r.u, u);
        std::memcpy(s, r.sigma.data(), r.sigma.size() * sizeof(double));
        store(r.v, v);
        *discarded = r.discarded_weight;
    });
}

// u: m x k, s: k, v: n x k
int ref_fixed_rank(const double* a, std::uint64_t m, std::uint64_t n, std::uint64_t k,
                   std::uint64_t p, std::uint64_t q, std::uint64_t seed, double* u, double* s,
                   double* v, double* discarded) {
    return guarded([&] {
        const rrsvd::SvdResult r =
            rrsvd::rrsvd_fixed_rank(load(a, m, n), rrsvd::RrsvdParams{k, p, q, seed});
        if (u) store(r.u, u);
        std::memcpy(s, r.sigma.data(), r.sigma.size() * sizeof(double));
        if (v) store(r.v, v);
        *discarded = r.discarded_weight;
    });
}

// rrsvd_fixed_precision (randomized.cpp:124-176) with AccuracyCheckParams{eps, probes, growth}.  u/v sized for min(m, n)
// columns (the worst case); *l_out = columns produced.
int ref_fixed_precision(const double* a, std::uint64_t m, std::uint64_t n, std::uint64_t initial_l,
                        std::uint64_t q, std::uint64_t probes, std::uint64_t growth, double eps, std::uint64_t seed, double* u,
                        double* s, double* v, std::uint64_t* l_out, int* certified, double* discarded) {
    return guarded([&] {
        const rrsvd::SvdResult r = rrsvd::rrsvd_fixed_precision(
            load(a, m, n), rrsvd::AccuracyCheckParams{eps, probes, growth}, initial_l, q, seed);
        if (u) store(r.u, u);
        std::memcpy(s, r.sigma.data(), r.sigma.size() * sizeof(double));
        if (v) store(r.v, v);
        *l_out = r.sigma.size();
        *certified = r.tolerance_certified ? 1 : 0;
        *discarded = r.discarded_weight;
    });
}

// Range basis Q (m x l) of randomized_range_finder (randomized.cpp:88-99).
int ref_range_finder(const double* a, std::uint64_t m, std::uint64_t n, std::uint64_t l,
                     std::uint64_t q, std::uint64_t seed, double* qout) {
    return guarded([&] { store(rrsvd::randomized_range_finder(load(a, m, n), l, q, seed).q_matrix, qout); });
}

// ---- matgen (input synthesis for configs 1 and 5) ---------------------------------------

int ref_spectrum_exponential(std::uint64_t n, double ratio, double* out) {
    return guarded([&] {
        const rrsvd::SpectrumSpec s = rrsvd::spectrum_exponential(n, ratio);
        std::memcpy(out, s.values.data(), n * sizeof(double));
    });
}

int ref_structured_matrix(const double* sigma, std::uint64_t n_sigma, std::uint64_t m,
                          std::uint64_t u_seed, std::uint64_t v_seed, double* out) {
    return guarded([&] {
        const rrsvd::SpectrumSpec s =
            rrsvd::make_spectrum(std::vector<double>(sigma, sigma + n_sigma), "oracle");
        store(rrsvd::structured_matrix(s, m, u_seed, v_seed).matrix, out);
    });
}

// ---- L3: the TEBD two-site trio (tebd.cpp:76-237) ---------------------------------------

// Builds a 2-4 site MpsState holding g1, g2 and the given lambdas, and calls build_theta on
// the (g1, g2) bond.  ll / lr == nullptr means an open chain end (unit weights,
// tebd.cpp:82-87).  Output theta in the reference (i, j, a, b) layout (tebd.hpp:23-28).
int ref_build_theta(const double* g1, const double* g2, const double* ll, const double* lm,
                    const double* lr, std::uint64_t cl, std::uint64_t d1, std::uint64_t cm,
                    std::uint64_t d2, std::uint64_t cr, double* theta) {
    return guarded([&] {
        tebd::MpsState st;
        std::size_t bond = 0;
        if (ll) {
            st.site_dims.push_back(1);
            st.gammas.push_back(tebd::Tensor3(1, 1, cl));
            st.lambdas.push_back(std::vector<double>(ll, ll + cl));
            bond = 1;
        }
        st.site_dims.push_back(d1);
        st.gammas.push_back(load_t3(g1, cl, d1, cm));
        st.lambdas.push_back(std::vector<double>(lm, lm + cm));
        st.site_dims.push_back(d2);
        st.gammas.push_back(load_t3(g2, cm, d2, cr));
        if (lr) {
            st.lambdas.push_back(std::vector<double>(lr, lr + cr));
            st.site_dims.push_back(1);
            st.gammas.push_back(tebd::Tensor3(cr, 1, 1));
        }
        const tebd::ThetaTensor t = tebd::build_theta(st, bond);
        std::memcpy(theta, t.values.data(), t.values.size() * sizeof(cplx));
    });
}

int ref_apply_gate(const double* theta, std::uint64_t d1, std::uint64_t d2, std::uint64_t cl,
                   std::uint64_t cr, const double* gate, double* out) {
    return guarded([&] {
        tebd::ThetaTensor t(d1, d2, cl, cr);
        std::memcpy(t.values.data(), theta, t.values.size() * sizeof(cplx));
        const tebd::TwoSiteGate g{0, load(gate, d1 * d2, d1 * d2), true};
        const tebd::ThetaTensor o = tebd::apply_gate_to_theta(t, g);
        std::memcpy(out, o.values.data(), o.values.size() * sizeof(cplx));
    });
}

// gl: cl x d1 x chi, lam: chi, gr: chi x d2 x cr, with chi <= max_chi (buffers sized by the
// caller for max_chi = min(d1*cl, d2*cr)).  backend->seed is advanced like the reference.
int ref_decimate(const double* theta, std::uint64_t d1, std::uint64_t d2, std::uint64_t cl,
                 std::uint64_t cr, const double* ll, const double* lr, std::uint64_t chi_max,
                 double trunc_tol, ref_backend* backend, int renormalize, double* gl,
                 double* lam, double* gr, ref_decim_info* info) {
    return guarded([&] {
        tebd::ThetaTensor t(d1, d2, cl, cr);
        std::memcpy(t.values.data(), theta, t.values.size() * sizeof(cplx));
        tebd::DecimationBackend be = to_backend(backend);
        const std::vector<double> vll = ll ? std::vector<double>(ll, ll + cl) : std::vector<double>{};
        const std::vector<double> vlr = lr ? std::vector<double>(lr, lr + cr) : std::vector<double>{};
        const tebd::DecimationResult r =
            tebd::decimate(t, vll, vlr, chi_max, trunc_tol, be, renormalize != 0);
        backend->seed = be.seed;
        std::memcpy(gl, r.gamma_left.values.data(), r.gamma_left.values.size() * sizeof(cplx));
        std::memcpy(lam, r.lambda.data(), r.lambda.size() * sizeof(double));
        std::memcpy(gr, r.gamma_right.values.data(), r.gamma_right.values.size() * sizeof(cplx));
        info->discarded = r.discarded;
        info->chi = r.chi;
        info->randomized_path = r.randomized_path;
        info->tolerance_certified = r.tolerance_certified;
        info->pseudo_inverse_applied = r.pseudo_inverse_applied;
    });
}

int ref_bond_gate(const double* h, std::uint64_t dd, double scale, double* out) {
    return guarded([&] { store(tebd::bond_gate(0, load(h, dd, dd), scale).matrix, out); });
}

// ---- model builders (host-side, off the hot path) ----------------------------------------

int ref_ising_terms(std::uint64_t n, double coupling, double field, double* out /*(n-1)x4x4*/) {
    return guarded([&] {
        const auto t = tebd::ising_terms(n, coupling, field);
        for (std::size_t b = 0; b < t.size(); ++b) store(t[b].h, out + b * 32);
    });
}

int ref_heisenberg_terms(std::uint64_t n, double coupling, double* out) {
    return guarded([&] {
        const auto t = tebd::heisenberg_terms(n, coupling);
        for (std::size_t b = 0; b < t.size(); ++b) store(t[b].h, out + b * 32);
    });
}

// Stieltjes chain map of a trapezoid measure (chainmap.cpp:58-68,108-153).
// out: t0, omegas[n_chain], hoppings[n_chain-1]
int ref_stieltjes(const double* nodes, const double* h2, std::uint64_t n_nodes,
                  std::uint64_t n_chain, double* out) {
    return guarded([&] {
        const auto m = rrsvd::chainmap::trapezoid_measure(
            std::vector<double>(nodes, nodes + n_nodes), std::vector<double>(h2, h2 + n_nodes));
        const auto c = rrsvd::chainmap::stieltjes_coefficients(m, n_chain);
        out[0] = c.t0;
        std::memcpy(out + 1, c.omegas.data(), c.omegas.size() * sizeof(double));
        std::memcpy(out + 1 + c.omegas.size(), c.hoppings.data(), c.hoppings.size() * sizeof(double));
    });
}

// build_chain_terms (chainmap.cpp:197-252).  coeffs as produced by ref_stieltjes.
// out: bond 0 term (d_sys*bd)^2 complex followed by n_chain-1 terms of (bd*bd)^2 complex.
int ref_chain_terms(const double* coeffs, std::uint64_t n_chain, std::uint64_t boson_dim,
                    const double* h_sys, const double* coupling, std::uint64_t d_sys,
                    double* out) {
    return guarded([&] {
        rrsvd::chainmap::ChainCoefficients c;
        c.t0 = coeffs[0];
        c.omegas.assign(coeffs + 1, coeffs + 1 + n_chain);
        c.hoppings.assign(coeffs + 1 + n_chain, coeffs + 1 + n_chain + (n_chain - 1));
        const auto sys = rrsvd::chainmap::build_chain_terms(c, boson_dim, load(h_sys, d_sys, d_sys),
                                                            load(coupling, d_sys, d_sys));
        double* p = out;
        for (const auto& t : sys.bond_terms) {
            store(t.h, p);
            p += 2 * t.h.size();
        }
    });
}

// ---- MPS handle: evolve + observables (tebd.cpp:260-326, mps.cpp:15-70) -----------------

void* ref_mps_product(std::uint64_t n, const std::uint64_t* dims, const double* locals,
                      std::uint64_t chi_max, double tol) {
    void* out = nullptr;
    const int rc = guarded([&] {
        std::vector<std::size_t> d(dims, dims + n);
        std::vector<std::vector<cplx>> loc;
        const double* p = locals;
        for (std::size_t s = 0; s < n; ++s) {
            std::vector<cplx> v(d[s]);
            std::memcpy(v.data(), p, d[s] * sizeof(cplx));
            p += 2 * d[s];
            loc.push_back(std::move(v));
        }
        out = new tebd::MpsState(tebd::mps_product_state(d, loc, chi_max, tol));
    });
    return rc == 0 ? out : nullptr;
}

void ref_mps_free(void* h) { delete static_cast<tebd::MpsState*>(h); }

// dims_out: 3 per site (left, phys, right)
int ref_mps_shape(void* h, std::uint64_t* dims_out) {
    return guarded([&] {
        const auto* st = static_cast<tebd::MpsState*>(h);
        for (std::size_t s = 0; s < st->n_sites(); ++s) {
            dims_out[3 * s] = st->gammas[s].dim_left;
            dims_out[3 * s + 1] = st->gammas[s].dim_phys;
            dims_out[3 * s + 2] = st->gammas[s].dim_right;
        }
    });
}

int ref_mps_get(void* h, std::uint64_t site, double* gamma, double* lambda_or_null) {
    return guarded([&] {
        const auto* st = static_cast<tebd::MpsState*>(h);
        const auto& g = st->gammas.at(site);
        std::memcpy(gamma, g.values.data(), g.values.size() * sizeof(cplx));
        if (lambda_or_null && site < st->lambdas.size())
            std::memcpy(lambda_or_null, st->lambdas[site].data(),
                        st->lambdas[site].size() * sizeof(double));
    });
}

int ref_mps_set(void* h, std::uint64_t site, std::uint64_t l, std::uint64_t d, std::uint64_t r,
                const double* gamma, const double* lambda_or_null) {
    return guarded([&] {
        auto* st = static_cast<tebd::MpsState*>(h);
        st->gammas.at(site) = load_t3(gamma, l, d, r);
        if (lambda_or_null && site < st->lambdas.size())
            st->lambdas[site].assign(lambda_or_null, lambda_or_null + r);
    });
}

// terms: n_terms bond ids + concatenated Hermitian matrices (dd_b x dd_b complex each).
// diag_out: kept_fraction, max_bond_dim, aborted, abort_step, n_updates
int ref_evolve(void* h, const std::uint64_t* bonds, const double* mats, std::uint64_t n_terms,
               double dt, std::uint64_t n_steps, ref_backend* backend, double abort_threshold,
               int renormalize, double* diag_out) {
    return guarded([&] {
        auto* st = static_cast<tebd::MpsState*>(h);
        std::vector<tebd::HamiltonianTerm> terms;
        const double* p = mats;
        for (std::size_t t = 0; t < n_terms; ++t) {
            const std::size_t b = bonds[t];
            const std::size_t dd = st->site_dims.at(b) * st->site_dims.at(b + 1);
            terms.push_back({b, load(p, dd, dd)});
            p += 2 * dd * dd;
        }
        tebd::DecimationBackend be = to_backend(backend);
        tebd::EvolveOptions opt;
        opt.abort_discarded_threshold = abort_threshold;
        opt.renormalize = renormalize != 0;
        const tebd::EvolveDiagnostics d =
            tebd::evolve(*st, terms, tebd::trotter_plan_3rd(dt), n_steps, be, opt);
        backend->seed = be.seed;
        diag_out[0] = d.kept_fraction;
        diag_out[1] = static_cast<double>(d.max_bond_dim);
        diag_out[2] = d.aborted ? 1.0 : 0.0;
        diag_out[3] = static_cast<double>(d.abort_step);
        diag_out[4] = static_cast<double>(d.updates.size());
        double us = 0.0;  // the reference's own per-update timers (tebd.cpp:296-306, UpdateRecord)
        for (const auto& u : d.updates) us += u.t_theta_us + u.t_gate_us + u.t_svd_us;
        diag_out[5] = us;
    });
}

int ref_expectation_local(void* h, std::uint64_t site, const double* op, double* out2) {
    return guarded([&] {
        const auto* st = static_cast<tebd::MpsState*>(h);
        const std::size_t d = st->site_dims.at(site);
        const cplx v = tebd::expectation_local(*st, site, load(op, d, d));
        out2[0] = v.real();
        out2[1] = v.imag();
    });
}

int ref_schmidt_entropy(void* h, std::uint64_t bond, double* out) {
    return guarded([&] { *out = tebd::schmidt_entropy(*static_cast<tebd::MpsState*>(h), bond); });
}

int ref_dense_coefficients(void* h, double* out) {
    return guarded([&] {
        const auto c = tebd::dense_coefficients(*static_cast<tebd::MpsState*>(h));
        std::memcpy(out, c.data(), c.size() * sizeof(cplx));
    });
}

}  // extern "C"

// ---- file formats and the experiment drivers -------------------
extern "C" {

int ref_write_rrsm(const char* path, const double* a, std::uint64_t rows, std::uint64_t cols) {
    return guarded([&] { rrsvd::write_rrsm(path, load(a, rows, cols)); });
}

int ref_read_rrsm_dims(const char* path, std::uint64_t* rows, std::uint64_t* cols) {
    return guarded([&] {
        const rrsvd::DenseMatrix m = rrsvd::read_rrsm(path);
        *rows = m.rows();
        *cols = m.cols();
    });
}

int ref_read_rrsm(const char* path, double* out) {
    return guarded([&] { store(rrsvd::read_rrsm(path), out); });
}

int ref_write_value_lines(const char* path, const double* v, std::uint64_t n) {
    return guarded([&] { rrsvd::write_value_lines(path, std::vector<double>(v, v + n)); });
}

int ref_write_coefficients(const char* path, double t0, const double* omegas, std::uint64_t n,
                           const double* hoppings) {
    return guarded([&] {
        rrsvd::chainmap::ChainCoefficients c;
        c.t0 = t0;
        c.omegas.assign(omegas, omegas + n);
        if (n > 1) c.hoppings.assign(hoppings, hoppings + n - 1);
        rrsvd::chainmap::write_coefficients_file(path, c);
    });
}

// experiments.cpp run_tebd with every TebdRunConfig field; returns the driver's exit code
// (or -1 when it threw).
int ref_run_tebd(const char* model, const char* coeffs, std::uint64_t sites, std::uint64_t chi, double dt,
                 std::uint64_t steps, const char* backend, double epsilon, std::uint64_t q,
                 std::uint64_t oversampling, std::uint64_t crossover, double coupling, double field,
                 double trunc_tol, double abort_thr, std::uint64_t boson_dim, double sys_eps,
                 double sys_delta, std::uint64_t seed, const char* out, const char* obs_out,
                 const char* state_out) {
    int rc = -1;
    guarded([&] {
        rrsvd::bench::TebdRunConfig c;
        c.model = model; c.coeffs_file = coeffs; c.sites = sites; c.chi = chi; c.dt = dt; c.steps = steps;
        c.backend = backend; c.epsilon = epsilon; c.q = q; c.oversampling = oversampling;
        c.det_crossover = crossover; c.coupling = coupling; c.field = field; c.trunc_tolerance = trunc_tol;
        c.abort_threshold = abort_thr; c.boson_dim = boson_dim; c.sys_epsilon = sys_eps;
        c.sys_delta = sys_delta; c.seed = seed; c.out = out; c.observables_out = obs_out;
        c.state_out = state_out;
        rc = rrsvd::bench::run_tebd(c);
    });
    return rc;
}

}  // extern "C"

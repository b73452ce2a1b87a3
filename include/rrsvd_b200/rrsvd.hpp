// rrsvd_b200/rrsvd.hpp — header-only C++ drop-in for the reference core's TEBD decimation path.
//
// Re-declares the reference API (namespace rrsvd / rrsvd::tebd, /root/reference/proj/core/
// include/rrsvd/*.hpp) with the same types, signatures, conventions and exceptions, implemented
// on top of the C ABI of librrsvd_b200.so (include/rrsvd_b200.h).  A caller that included
// "rrsvd/tebd.hpp" and linked rrsvd::core includes this header and links -lrrsvd_b200 instead;
// every numeric call of the hot path then runs on the B200.  See INTEGRATION.md.
//
// Threading: one library context per host thread (thread_local), mirroring SPEC.md:112,225.
#ifndef RRSVD_B200_RRSVD_HPP
#define RRSVD_B200_RRSVD_HPP

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../rrsvd_b200.h"

namespace rrsvd {

using cplx = std::complex<double>;

// errors.hpp:11-32
struct contract_violation : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct numeric_failure : std::runtime_error {
    numeric_failure(const std::string& what, std::size_t rows, std::size_t cols)
        : std::runtime_error(what + " (matrix " + std::to_string(rows) + "x" + std::to_string(cols) + ")"),
          rows(rows), cols(cols) {}
    std::size_t rows, cols;
};

namespace b200 {
// The per-thread library context (fails loudly: there is no CPU fallback).
inline rrsvd_b200_ctx* context() {
    thread_local struct Holder {
        rrsvd_b200_ctx* c = nullptr;
        Holder() {
            if (rrsvd_b200_ctx_create(0, nullptr, &c) != RRSVD_B200_OK)
                throw std::runtime_error("rrsvd_b200: no usable sm_100 device");
        }
        ~Holder() { rrsvd_b200_ctx_destroy(c); }
    } h;
    return h.c;
}
inline void check(int rc, std::size_t rows = 0, std::size_t cols = 0) {
    if (rc == RRSVD_B200_OK) return;
    const std::string msg = rrsvd_b200_last_error(context());
    if (rc == RRSVD_B200_CONTRACT_VIOLATION) throw contract_violation(msg);
    if (rc == RRSVD_B200_NUMERIC_FAILURE) throw numeric_failure(msg, rows, cols);
    throw std::runtime_error("rrsvd_b200: " + msg);
}
inline const double* D(const cplx* p) { return reinterpret_cast<const double*>(p); }
inline double* D(cplx* p) { return reinterpret_cast<double*>(p); }
}  // namespace b200

// dense_matrix.hpp:13-49 — row-major complex matrix.
class DenseMatrix {
  public:
    DenseMatrix() : rows_(0), cols_(0) {}
    DenseMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(rows * cols, cplx(0.0)) {}
    DenseMatrix(std::size_t rows, std::size_t cols, std::vector<cplx> data)
        : rows_(rows), cols_(cols), data_(std::move(data)) {
        if (data_.size() != rows_ * cols_) throw contract_violation("DenseMatrix: data length does not match rows*cols");
    }
    static DenseMatrix identity(std::size_t n) {
        DenseMatrix m(n, n);
        for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    cplx& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
    const cplx& operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
    cplx* data() { return data_.data(); }
    const cplx* data() const { return data_.data(); }
    bool all_finite() const {
        for (const cplx& z : data_)
            if (!std::isfinite(z.real()) || !std::isfinite(z.imag())) return false;
        return true;
    }
    DenseMatrix left_cols(std::size_t keep) const {
        if (keep > cols_) throw contract_violation("left_cols: keep > cols");
        DenseMatrix out(rows_, keep);
        for (std::size_t i = 0; i < rows_; ++i)
            for (std::size_t j = 0; j < keep; ++j) out(i, j) = (*this)(i, j);
        return out;
    }

  private:
    std::size_t rows_, cols_;
    std::vector<cplx> data_;
};

// linalg.hpp:17-26
struct QrFactors {
    DenseMatrix q, r;
};
struct SvdResult {
    DenseMatrix u;
    std::vector<double> sigma;
    DenseMatrix v;
    double discarded_weight = 0.0;
    std::size_t achieved_rank = 0;
    bool tolerance_certified = true;
};

// randomized.hpp:17-35
struct RrsvdParams {
    std::size_t target_rank, oversampling, power_iterations;
    std::uint64_t seed;
};
struct AccuracyCheckParams {
    double tolerance;
    std::size_t probe_count;
    std::size_t growth_block = 0;  // columns appended per failed round; 0 doubles the basis
};

// ---- linalg.hpp:29-56 (device) ----------------------------------------------------------
inline DenseMatrix gemm(const DenseMatrix& a, bool adj_a, const DenseMatrix& b, bool adj_b) {
    if (adj_b) throw contract_violation("gemm: adj_b is not supported by the device path");
    const std::size_t m = adj_a ? a.cols() : a.rows(), k = adj_a ? a.rows() : a.cols();
    if (k != b.rows()) throw contract_violation("gemm: inner dimension mismatch");
    DenseMatrix c(m, b.cols());
    b200::check(rrsvd_b200_zgemm(b200::context(), adj_a ? RRSVD_B200_OP_C : RRSVD_B200_OP_N, RRSVD_B200_OP_N, m,
                                 b.cols(), k, b200::D(a.data()), a.cols(), b200::D(b.data()), b.cols(),
                                 b200::D(c.data()), c.cols()));
    return c;
}
inline DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.cols() != b.rows()) throw contract_violation("matmul: dimension mismatch");
    return gemm(a, false, b, false);
}
inline DenseMatrix adjoint(const DenseMatrix& a) {
    DenseMatrix out(a.cols(), a.rows());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) out(j, i) = std::conj(a(i, j));
    return out;
}
inline QrFactors qr(const DenseMatrix& a) {
    QrFactors f{DenseMatrix(a.rows(), a.cols()), DenseMatrix(a.cols(), a.cols())};
    b200::check(rrsvd_b200_qr(b200::context(), b200::D(a.data()), a.rows(), a.cols(), b200::D(f.q.data()),
                              b200::D(f.r.data())), a.rows(), a.cols());
    return f;
}
inline SvdResult svd_full(const DenseMatrix& a) {
    const std::size_t k = std::min(a.rows(), a.cols());
    SvdResult out;
    out.u = DenseMatrix(a.rows(), k);
    out.v = DenseMatrix(a.cols(), k);
    out.sigma.assign(k, 0.0);
    if (k) b200::check(rrsvd_b200_svd(b200::context(), b200::D(a.data()), a.rows(), a.cols(), b200::D(out.u.data()),
                                      out.sigma.data(), b200::D(out.v.data())), a.rows(), a.cols());
    out.achieved_rank = k;
    return out;
}
inline double frobenius_norm(const DenseMatrix& a) {
    double v = 0.0;
    b200::check(rrsvd_b200_frobenius_norm(b200::context(), b200::D(a.data()), a.rows(), a.cols(), &v));
    return v;
}

// ---- randomized.hpp:48-61 (device) ------------------------------------------------------
inline DenseMatrix gaussian_test_matrix(std::size_t n, std::size_t l, std::uint64_t seed) {
    DenseMatrix out(n, l);
    b200::check(rrsvd_b200_gaussian_test_matrix(b200::context(), n, l, seed, RRSVD_B200_OMEGA_REFERENCE,
                                                b200::D(out.data())));
    return out;
}
inline SvdResult rrsvd_sketched_svd(const DenseMatrix& a, std::size_t l, std::size_t q, std::uint64_t seed) {
    SvdResult out;
    out.u = DenseMatrix(a.rows(), l);
    out.v = DenseMatrix(a.cols(), l);
    out.sigma.assign(l, 0.0);
    b200::check(rrsvd_b200_sketched_svd(b200::context(), b200::D(a.data()), a.rows(), a.cols(), l, q, seed,
                                        RRSVD_B200_OMEGA_REFERENCE, nullptr, b200::D(out.u.data()), out.sigma.data(),
                                        b200::D(out.v.data()), &out.discarded_weight), a.rows(), a.cols());
    out.achieved_rank = l;
    return out;
}
inline SvdResult rrsvd_fixed_rank(const DenseMatrix& a, const RrsvdParams& p) {
    const std::size_t k = p.target_rank;
    SvdResult out;
    out.u = DenseMatrix(a.rows(), k);
    out.v = DenseMatrix(a.cols(), k);
    out.sigma.assign(k, 0.0);
    b200::check(rrsvd_b200_fixed_rank(b200::context(), b200::D(a.data()), a.rows(), a.cols(), k, p.oversampling,
                                      p.power_iterations, p.seed, RRSVD_B200_OMEGA_REFERENCE, nullptr,
                                      b200::D(out.u.data()), out.sigma.data(), b200::D(out.v.data()),
                                      &out.discarded_weight), a.rows(), a.cols());
    out.achieved_rank = k;
    return out;
}

inline SvdResult rrsvd_fixed_precision(const DenseMatrix& a, const AccuracyCheckParams& check,
                                       std::size_t initial_l, std::size_t q, std::uint64_t seed) {
    const std::size_t mn = std::min(a.rows(), a.cols());
    std::vector<cplx> u(a.rows() * mn), v(a.cols() * mn);
    std::vector<double> s(mn);
    std::size_t l = 0;
    int cert = 0;
    SvdResult out;
    b200::check(rrsvd_b200_fixed_precision(b200::context(), b200::D(a.data()), a.rows(), a.cols(), initial_l, q,
                                           check.probe_count, check.growth_block, check.tolerance, seed, RRSVD_B200_OMEGA_REFERENCE,
                                           b200::D(u.data()), s.data(), b200::D(v.data()), &l, &cert,
                                           &out.discarded_weight), a.rows(), a.cols());
    out.u = DenseMatrix(a.rows(), l);
    out.v = DenseMatrix(a.cols(), l);
    std::copy_n(u.begin(), a.rows() * l, out.u.data());
    std::copy_n(v.begin(), a.cols() * l, out.v.data());
    out.sigma.assign(s.begin(), s.begin() + static_cast<std::ptrdiff_t>(l));
    out.achieved_rank = l;
    out.tolerance_certified = cert != 0;
    return out;
}

namespace tebd {

// mps.hpp:12-41
struct Tensor3 {
    std::size_t dim_left = 0, dim_phys = 0, dim_right = 0;
    std::vector<cplx> values;
    Tensor3() = default;
    Tensor3(std::size_t l, std::size_t d, std::size_t r) : dim_left(l), dim_phys(d), dim_right(r), values(l * d * r, cplx(0.0)) {}
    cplx& at(std::size_t a, std::size_t i, std::size_t b) { return values[(a * dim_phys + i) * dim_right + b]; }
    const cplx& at(std::size_t a, std::size_t i, std::size_t b) const { return values[(a * dim_phys + i) * dim_right + b]; }
};
struct MpsState {
    std::vector<std::size_t> site_dims;
    std::vector<Tensor3> gammas;
    std::vector<std::vector<double>> lambdas;
    std::size_t chi_max = 0;
    double trunc_tolerance = 0.0;
    std::size_t n_sites() const { return site_dims.size(); }
    std::size_t bond_dim(std::size_t bond) const { return lambdas[bond].size(); }
    std::size_t max_bond_dim() const {
        std::size_t m = 1;
        for (const auto& l : lambdas) m = std::max(m, l.size());
        return m;
    }
};
inline MpsState mps_product_state(const std::vector<std::size_t>& site_dims,
                                  const std::vector<std::vector<cplx>>& local_states, std::size_t chi_max = 0,
                                  double trunc_tolerance = 0.0) {  // mps.cpp:15-38
    if (site_dims.empty() || site_dims.size() != local_states.size())
        throw contract_violation("mps_product_state: one local state per site required");
    MpsState st;
    st.site_dims = site_dims;
    st.chi_max = chi_max;
    st.trunc_tolerance = trunc_tolerance;
    for (std::size_t k = 0; k < site_dims.size(); ++k) {
        if (local_states[k].size() != site_dims[k])
            throw contract_violation("mps_product_state: local state dimension mismatch");
        double nsq = 0.0;
        for (const cplx& z : local_states[k]) nsq += std::norm(z);
        if (std::abs(nsq - 1.0) > 1e-10) throw contract_violation("mps_product_state: local state is not normalized");
        Tensor3 g(1, site_dims[k], 1);
        for (std::size_t i = 0; i < site_dims[k]; ++i) g.at(0, i, 0) = local_states[k][i];
        st.gammas.push_back(std::move(g));
    }
    st.lambdas.assign(site_dims.size() - 1, std::vector<double>{1.0});
    return st;
}
inline double schmidt_entropy(const MpsState& st, std::size_t bond) {  // mps.cpp:40-48
    if (bond >= st.lambdas.size()) throw contract_violation("schmidt_entropy: bad bond");
    double s = 0.0;
    for (double l : st.lambdas[bond]) {
        const double p = l * l;
        if (p > 0.0) s -= p * std::log(p);
    }
    return s;
}

// tebd.hpp:15-62
struct ThetaTensor {
    std::size_t d_left = 0, d_right = 0, chi_left = 0, chi_right = 0;
    std::vector<cplx> values;
    ThetaTensor() = default;
    ThetaTensor(std::size_t dl, std::size_t dr, std::size_t cl, std::size_t cr)
        : d_left(dl), d_right(dr), chi_left(cl), chi_right(cr), values(dl * dr * cl * cr, cplx(0.0)) {}
    cplx& at(std::size_t i, std::size_t j, std::size_t a, std::size_t b) {
        return values[((i * d_right + j) * chi_left + a) * chi_right + b];
    }
    const cplx& at(std::size_t i, std::size_t j, std::size_t a, std::size_t b) const {
        return values[((i * d_right + j) * chi_left + a) * chi_right + b];
    }
    double frobenius() const {
        double v = 0.0;
        if (!values.empty())
            b200::check(rrsvd_b200_frobenius_norm(b200::context(), b200::D(values.data()), values.size(), 1, &v));
        return v;
    }
};
struct TwoSiteGate {
    std::size_t site = 0;
    DenseMatrix matrix;
    bool unitary = false;
};
struct HamiltonianTerm {
    std::size_t bond;
    DenseMatrix h;
};
struct TrotterPlan {
    struct Sweep {
        int bond_parity;
        double coefficient;
    };
    double dt = 0.0;
    std::vector<Sweep> sweeps;
    int order = 3;
};
inline TrotterPlan trotter_plan_3rd(double dt) {  // tebd.cpp:67-74
    if (dt == 0.0) throw contract_violation("trotter_plan_3rd: dt must be nonzero");
    TrotterPlan p;
    p.dt = dt;
    p.sweeps = {{1, 0.5}, {0, 1.0}, {1, 0.5}};
    return p;
}
struct DecimationBackend {  // tebd.hpp:65-85
    enum class Kind { Deterministic, Randomized };
    Kind kind = Kind::Deterministic;
    std::size_t target_rank = 0, oversampling = 0, power_iterations = 2;
    bool accuracy_check = false;
    double epsilon = 1e-3;
    std::size_t probe_count = 10;
    std::size_t det_crossover = 256;
    std::uint64_t seed = 0;
};
struct DecimationResult {  // tebd.hpp:87-96
    Tensor3 gamma_left;
    std::vector<double> lambda;
    Tensor3 gamma_right;
    double discarded = 0.0;
    std::size_t chi = 0;
    bool randomized_path = false;
    bool tolerance_certified = true;
    bool pseudo_inverse_applied = false;
};
struct UpdateRecord {
    std::size_t step, bond, chi;
    double discarded_weight, t_theta_us, t_gate_us, t_svd_us;
    bool randomized_path;
};
struct EvolveOptions {
    double abort_discarded_threshold = 1.0;
    bool renormalize = true;
    bool record_updates = true;
};
struct EvolveDiagnostics {
    std::vector<UpdateRecord> updates;
    double kept_fraction = 1.0;
    std::size_t max_bond_dim = 1;
    bool aborted = false;
    std::size_t abort_step = 0;
};

namespace detail {
inline rrsvd_b200_backend to_c(const DecimationBackend& b) {
    return rrsvd_b200_backend{b.kind == DecimationBackend::Kind::Randomized ? 1 : 0, b.target_rank, b.oversampling,
                              b.power_iterations, b.accuracy_check ? 1 : 0, b.epsilon, b.probe_count,
                              b.det_crossover, b.seed};
}
// Hermitian eigendecomposition (cyclic Jacobi) for bond_gate — host-side model building,
// once per (bond, coefficient); the reference uses LAPACKE_zheevd here (linalg.cpp:141-150).
inline void hermitian_eig(DenseMatrix a, DenseMatrix& vec, std::vector<double>& val) {
    const std::size_t n = a.rows();
    vec = DenseMatrix::identity(n);
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (std::size_t p = 0; p < n; ++p)
            for (std::size_t q = p + 1; q < n; ++q) off += std::norm(a(p, q));
        if (off < 1e-30) break;
        for (std::size_t p = 0; p < n; ++p)
            for (std::size_t q = p + 1; q < n; ++q) {
                const cplx apq = a(p, q);
                const double g = std::abs(apq);
                if (g < 1e-300) continue;
                const double app = a(p, p).real(), aqq = a(q, q).real();
                const double theta = 0.5 * std::atan2(2.0 * g, aqq - app);
                const double c = std::cos(theta), s = std::sin(theta);
                const cplx e = apq / g;  // phase
                // rotation R acting on columns p, q: [c, s e; -s conj(e), c] (unitary)
                for (std::size_t k = 0; k < n; ++k) {
                    const cplx akp = a(k, p), akq = a(k, q);
                    a(k, p) = c * akp - s * std::conj(e) * akq;
                    a(k, q) = s * e * akp + c * akq;
                }
                for (std::size_t k = 0; k < n; ++k) {
                    const cplx apk = a(p, k), aqk = a(q, k);
                    a(p, k) = c * apk - s * e * aqk;
                    a(q, k) = s * std::conj(e) * apk + c * aqk;
                }
                for (std::size_t k = 0; k < n; ++k) {
                    const cplx vkp = vec(k, p), vkq = vec(k, q);
                    vec(k, p) = c * vkp - s * std::conj(e) * vkq;
                    vec(k, q) = s * e * vkp + c * vkq;
                }
            }
    }
    val.resize(n);
    for (std::size_t i = 0; i < n; ++i) val[i] = a(i, i).real();
}
}  // namespace detail

inline TwoSiteGate bond_gate(std::size_t bond, const DenseMatrix& h, double scale) {  // tebd.cpp:239-258
    if (h.rows() != h.cols()) throw contract_violation("bond_gate: term must be square");
    DenseMatrix vec;
    std::vector<double> val;
    detail::hermitian_eig(h, vec, val);
    TwoSiteGate g;
    g.site = bond;
    g.unitary = true;
    g.matrix = DenseMatrix(h.rows(), h.cols());
    for (std::size_t i = 0; i < h.rows(); ++i)
        for (std::size_t j = 0; j < h.cols(); ++j) {
            cplx s(0.0);
            for (std::size_t k = 0; k < h.rows(); ++k)
                s += vec(i, k) * std::exp(cplx(0.0, -scale * val[k])) * std::conj(vec(j, k));
            g.matrix(i, j) = s;
        }
    return g;
}

inline ThetaTensor build_theta(const MpsState& st, std::size_t bond) {  // tebd.cpp:76-124
    if (bond + 1 >= st.n_sites()) throw contract_violation("build_theta: bad bond");
    const Tensor3& g1 = st.gammas[bond];
    const Tensor3& g2 = st.gammas[bond + 1];
    const std::size_t d1 = g1.dim_phys, d2 = g2.dim_phys, cl = g1.dim_left, cm = g1.dim_right, cr = g2.dim_right;
    std::vector<cplx> m(d1 * cl * d2 * cr);
    b200::check(rrsvd_b200_build_theta_unfolded(
        b200::context(), b200::D(g1.values.data()), b200::D(g2.values.data()),
        bond > 0 ? st.lambdas[bond - 1].data() : nullptr, st.lambdas[bond].data(),
        bond + 2 < st.n_sites() ? st.lambdas[bond + 1].data() : nullptr, cl, d1, cm, d2, cr, b200::D(m.data())));
    ThetaTensor t(d1, d2, cl, cr);
    b200::check(rrsvd_b200_unfolded_to_theta(b200::context(), b200::D(m.data()), d1, d2, cl, cr,
                                             b200::D(t.values.data())));
    return t;
}

inline ThetaTensor apply_gate_to_theta(const ThetaTensor& theta, const TwoSiteGate& gate) {  // tebd.cpp:126-139
    const std::size_t dd = theta.d_left * theta.d_right;
    if (gate.matrix.rows() != dd || gate.matrix.cols() != dd)
        throw contract_violation("apply_gate_to_theta: gate dimension mismatch");
    const std::size_t cl = theta.chi_left, cr = theta.chi_right;
    std::vector<cplx> m(theta.values.size()), m2(theta.values.size());
    ThetaTensor out(theta.d_left, theta.d_right, cl, cr);
    if (m.empty()) return out;
    auto* c = b200::context();
    b200::check(rrsvd_b200_theta_to_unfolded(c, b200::D(theta.values.data()), theta.d_left, theta.d_right, cl, cr,
                                             b200::D(m.data())));
    b200::check(rrsvd_b200_apply_gate_unfolded(c, b200::D(gate.matrix.data()), theta.d_left, theta.d_right, cl, cr,
                                               b200::D(m.data()), b200::D(m2.data())));
    b200::check(rrsvd_b200_unfolded_to_theta(c, b200::D(m2.data()), theta.d_left, theta.d_right, cl, cr,
                                             b200::D(out.values.data())));
    return out;
}

inline DecimationResult decimate(const ThetaTensor& theta, const std::vector<double>& lambda_left,
                                 const std::vector<double>& lambda_right, std::size_t chi_max, double trunc_tolerance,
                                 DecimationBackend& backend, bool renormalize = true) {  // tebd.cpp:141-237
    const std::size_t d1 = theta.d_left, d2 = theta.d_right, cl = theta.chi_left, cr = theta.chi_right;
    if ((!lambda_left.empty() && lambda_left.size() != cl) || (!lambda_right.empty() && lambda_right.size() != cr))
        throw contract_violation("decimate: outer lambda dimensions do not match theta");
    auto* c = b200::context();
    std::vector<cplx> m(theta.values.size());
    if (!m.empty())
        b200::check(rrsvd_b200_theta_to_unfolded(c, b200::D(theta.values.data()), d1, d2, cl, cr, b200::D(m.data())));
    const std::size_t kmax = std::max<std::size_t>(1, std::min(d1 * cl, d2 * cr));
    std::vector<cplx> gl(cl * d1 * kmax), gr(kmax * d2 * cr);
    std::vector<double> lam(kmax);
    rrsvd_b200_decim_info info{};
    const rrsvd_b200_backend be = detail::to_c(backend);
    const std::uint64_t call_seed = backend.seed++;  // tebd.cpp:162
    b200::check(rrsvd_b200_decimate_unfolded(c, b200::D(m.data()), d1, d2, cl, cr,
                                             lambda_left.empty() ? nullptr : lambda_left.data(),
                                             lambda_right.empty() ? nullptr : lambda_right.data(), chi_max,
                                             trunc_tolerance, &be, call_seed, RRSVD_B200_OMEGA_REFERENCE, nullptr,
                                             renormalize ? 1 : 0, b200::D(gl.data()), lam.data(), b200::D(gr.data()),
                                             &info),
                d1 * cl, d2 * cr);
    DecimationResult r;
    r.chi = info.chi;
    r.discarded = info.discarded;
    r.randomized_path = info.randomized_path != 0;
    r.tolerance_certified = info.tolerance_certified != 0;
    r.pseudo_inverse_applied = info.pseudo_inverse_applied != 0;
    r.gamma_left = Tensor3(cl, d1, r.chi);
    std::copy(gl.begin(), gl.begin() + cl * d1 * r.chi, r.gamma_left.values.begin());
    r.gamma_right = Tensor3(r.chi, d2, cr);
    std::copy(gr.begin(), gr.begin() + r.chi * d2 * cr, r.gamma_right.values.begin());
    r.lambda.assign(lam.begin(), lam.begin() + r.chi);
    return r;
}

// tebd.cpp:260-326: the whole evolution runs device-resident; the state is uploaded once and
// downloaded at the end.
inline EvolveDiagnostics evolve(MpsState& state, const std::vector<HamiltonianTerm>& terms, const TrotterPlan& plan,
                                std::size_t n_steps, DecimationBackend& backend, const EvolveOptions& options = {}) {
    const std::size_t n = state.n_sites(), nb = n - 1;
    std::vector<const DenseMatrix*> bond_terms(nb, nullptr);
    for (const auto& t : terms) {
        if (t.bond >= nb) throw contract_violation("evolve: term bond out of range");
        if (bond_terms[t.bond]) throw contract_violation("evolve: duplicate term on a bond");
        const std::size_t dd = state.site_dims[t.bond] * state.site_dims[t.bond + 1];
        if (t.h.rows() != dd || t.h.cols() != dd) throw contract_violation("evolve: term dimension mismatch");
        bond_terms[t.bond] = &t.h;
    }
    std::map<std::pair<std::size_t, double>, TwoSiteGate> gates;
    std::vector<const double*> gptr(plan.sweeps.size() * nb, nullptr);
    for (std::size_t s = 0; s < plan.sweeps.size(); ++s)
        for (std::size_t b = 0; b < nb; ++b) {
            if ((int)(b % 2) != plan.sweeps[s].bond_parity || !bond_terms[b]) continue;
            const auto key = std::make_pair(b, plan.sweeps[s].coefficient);
            if (!gates.count(key)) gates.emplace(key, bond_gate(b, *bond_terms[b], plan.sweeps[s].coefficient * plan.dt));
            gptr[s * nb + b] = b200::D(gates.at(key).matrix.data());
        }
    auto* c = b200::context();
    rrsvd_b200_mps* dm = nullptr;
    b200::check(rrsvd_b200_mps_create(c, n, state.site_dims.data(), state.chi_max, state.trunc_tolerance, &dm));
    struct Guard {
        rrsvd_b200_mps* m;
        ~Guard() { rrsvd_b200_mps_destroy(m); }
    } guard{dm};
    {  // the whole state in one call (one stream sync)
        std::vector<std::size_t> dims(3 * n);
        std::vector<const double*> gp(n), lp(n, nullptr);
        for (std::size_t s = 0; s < n; ++s) {
            dims[3 * s] = state.gammas[s].dim_left;
            dims[3 * s + 2] = state.gammas[s].dim_right;
            gp[s] = b200::D(state.gammas[s].values.data());
            if (s + 1 < n) lp[s] = state.lambdas[s].data();
        }
        b200::check(rrsvd_b200_state_upload(dm, dims.data(), gp.data(), lp.data()));
    }
    std::vector<rrsvd_b200_sweep> sw;
    for (const auto& x : plan.sweeps) sw.push_back({x.bond_parity, x.coefficient});
    rrsvd_b200_backend be = detail::to_c(backend);
    const rrsvd_b200_evolve_options opt{options.abort_discarded_threshold, options.renormalize ? 1 : 0,
                                        RRSVD_B200_OMEGA_REFERENCE};
    rrsvd_b200_evolve_diag diag{};
    std::size_t per_step = 0;
    for (const auto& x : plan.sweeps)
        for (std::size_t b = x.bond_parity; b < nb; b += 2) per_step += bond_terms[b] != nullptr;
    std::vector<rrsvd_b200_update_record> rec(options.record_updates ? per_step * n_steps : 0);
    b200::check(rrsvd_b200_evolve(dm, sw.size(), sw.data(), gptr.data(), n_steps, &be, &opt, &diag,
                                  rec.empty() ? nullptr : rec.data(), rec.size()));
    backend.seed = be.seed;
    {  // dims first, then every Γ and λ in one call
        std::vector<std::size_t> dims(3 * n);
        b200::check(rrsvd_b200_state_download(dm, dims.data(), nullptr, nullptr));
        std::vector<double*> gp(n), lp(n, nullptr);
        for (std::size_t s = 0; s < n; ++s) {
            state.gammas[s] = Tensor3(dims[3 * s], dims[3 * s + 1], dims[3 * s + 2]);
            gp[s] = reinterpret_cast<double*>(state.gammas[s].values.data());
            if (s + 1 < n) {
                state.lambdas[s].assign(dims[3 * s + 2], 0.0);
                lp[s] = state.lambdas[s].data();
            }
        }
        b200::check(rrsvd_b200_state_download(dm, nullptr, gp.data(), lp.data()));
    }
    EvolveDiagnostics out;
    out.kept_fraction = diag.kept_fraction;
    out.max_bond_dim = diag.max_bond_dim;
    out.aborted = diag.aborted != 0;
    out.abort_step = diag.abort_step;
    for (std::size_t i = 0; i < std::min<std::size_t>(diag.n_updates, rec.size()); ++i)
        out.updates.push_back({rec[i].step, rec[i].bond, rec[i].chi, rec[i].discarded_weight, rec[i].t_theta_us,
                               rec[i].t_gate_us, rec[i].t_svd_us, rec[i].randomized_path != 0});
    return out;
}

}  // namespace tebd
}  // namespace rrsvd

#endif

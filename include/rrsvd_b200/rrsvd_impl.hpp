// rrsvd_b200/rrsvd_impl.hpp — definitions of the drop-in declared in rrsvd.hpp (include that
// header, not this one).  Every numeric entry point is one or a few C-ABI calls on the per-thread
// library context; host code here only converts layouts at the boundary, advances
// backend.seed and maps status codes back to the reference's exceptions.
#ifndef RRSVD_B200_RRSVD_IMPL_HPP
#define RRSVD_B200_RRSVD_IMPL_HPP

#include "rrsvd.hpp"

namespace rrsvd {

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
// Status code -> the reference's exception types (errors.hpp:11-32).
inline void check(int rc, std::size_t rows = 0, std::size_t cols = 0) {
    if (rc == RRSVD_B200_OK) return;
    const std::string msg = rrsvd_b200_last_error(context());
    if (rc == RRSVD_B200_CONTRACT_VIOLATION) throw contract_violation(msg);
    if (rc == RRSVD_B200_NUMERIC_FAILURE) throw numeric_failure(msg, rows, cols);
    throw std::runtime_error("rrsvd_b200: " + msg);
}
inline const double* D(const cplx* p) { return reinterpret_cast<const double*>(p); }
inline double* D(cplx* p) { return reinterpret_cast<double*>(p); }
inline const double* D(const std::vector<double>& v) { return v.empty() ? nullptr : v.data(); }

// Hermitian eigenpairs of a small block on the host: cyclic complex Jacobi, stopped when the
// off-diagonal mass is at rounding level RELATIVE to the block's norm (so terms in any units
// converge the same way).  Values ascending, vectors in columns.
inline void small_hermitian_eig(DenseMatrix a, DenseMatrix& vec, std::vector<double>& val) {
    const std::size_t n = a.rows();
    vec = DenseMatrix::identity(n);
    double fro2 = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) fro2 += std::norm(a.data()[i]);
    const double eps = 0x1p-52 * static_cast<double>(n > 0 ? n : 1);
    for (int sweep = 0; sweep < 64 && fro2 > 0.0; ++sweep) {
        double off = 0.0;
        for (std::size_t p = 0; p < n; ++p)
            for (std::size_t q = p + 1; q < n; ++q) off += std::norm(a(p, q));
        if (off <= eps * eps * fro2) break;
        for (std::size_t p = 0; p + 1 < n; ++p)
            for (std::size_t q = p + 1; q < n; ++q) {
                const double mag = std::abs(a(p, q));
                if (mag == 0.0) continue;
                const cplx ph = a(p, q) / mag;  // a_pq = |a_pq| e^{i phi}
                const double t = 0.5 * std::atan2(2.0 * mag, a(q, q).real() - a(p, p).real());
                const double c = std::cos(t), s = std::sin(t);
                // columns p, q of A and of the eigenvector matrix, then rows p, q of A
                for (std::size_t k = 0; k < n; ++k) {
                    const cplx xp = a(k, p), xq = a(k, q);
                    a(k, p) = c * xp - s * std::conj(ph) * xq;
                    a(k, q) = s * ph * xp + c * xq;
                    const cplx vp = vec(k, p), vq = vec(k, q);
                    vec(k, p) = c * vp - s * std::conj(ph) * vq;
                    vec(k, q) = s * ph * vp + c * vq;
                }
                for (std::size_t k = 0; k < n; ++k) {
                    const cplx yp = a(p, k), yq = a(q, k);
                    a(p, k) = c * yp - s * ph * yq;
                    a(q, k) = s * std::conj(ph) * yp + c * yq;
                }
            }
    }
    std::vector<std::size_t> order(n);
    std::iota(order.begin(), order.end(), std::size_t{0});
    std::stable_sort(order.begin(), order.end(),
                     [&](std::size_t x, std::size_t y) { return a(x, x).real() < a(y, y).real(); });
    DenseMatrix sorted(n, n);
    val.assign(n, 0.0);
    for (std::size_t j = 0; j < n; ++j) {
        val[j] = a(order[j], order[j]).real();
        for (std::size_t k = 0; k < n; ++k) sorted(k, j) = vec(k, order[j]);
    }
    vec = std::move(sorted);
}
}  // namespace b200

// ---- DenseMatrix (dense_matrix.hpp:13-49) --------------------------------------------------
RRSVD_B200_API DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols, std::vector<cplx> data)
    : rows_(rows), cols_(cols), data_(std::move(data)) {
    if (data_.size() != rows_ * cols_) throw contract_violation("DenseMatrix: data length does not match rows*cols");
}
RRSVD_B200_API DenseMatrix DenseMatrix::identity(std::size_t n) {
    DenseMatrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m.data_[i * n + i] = cplx(1.0, 0.0);
    return m;
}
RRSVD_B200_API bool DenseMatrix::all_finite() const {
    return std::all_of(data_.begin(), data_.end(),
                       [](const cplx& z) { return std::isfinite(z.real()) && std::isfinite(z.imag()); });
}
RRSVD_B200_API DenseMatrix DenseMatrix::left_cols(std::size_t keep) const {
    if (keep > cols_) throw contract_violation("left_cols: keep > cols");
    DenseMatrix out(rows_, keep);
    for (std::size_t i = 0; i < rows_; ++i)
        std::copy(data_.begin() + i * cols_, data_.begin() + i * cols_ + keep, out.data_.begin() + i * keep);
    return out;
}
RRSVD_B200_API DenseMatrix DenseMatrix::hcat(const DenseMatrix& right) const {
    if (right.rows_ != rows_) throw contract_violation("hcat: row mismatch");
    const std::size_t w = cols_ + right.cols_;
    DenseMatrix out(rows_, w);
    for (std::size_t i = 0; i < rows_; ++i) {
        auto dst = out.data_.begin() + i * w;
        dst = std::copy(data_.begin() + i * cols_, data_.begin() + (i + 1) * cols_, dst);
        std::copy(right.data_.begin() + i * right.cols_, right.data_.begin() + (i + 1) * right.cols_, dst);
    }
    return out;
}
RRSVD_B200_API void DenseMatrix::scale_cols(const std::vector<double>& s) {
    if (s.size() != cols_) throw contract_violation("scale_cols: size mismatch");
    for (std::size_t e = 0; e < data_.size(); ++e) data_[e] *= s[e % cols_];
}
RRSVD_B200_API double DenseMatrix::max_abs() const {
    double m = 0.0;
    for (const cplx& z : data_) m = std::max(m, std::abs(z));
    return m;
}

// ---- linalg (linalg.cpp:20-150) on the device ----------------------------------------------
RRSVD_B200_API DenseMatrix gemm(const DenseMatrix& a, bool adj_a, const DenseMatrix& b, bool adj_b) {
    const std::size_t m = adj_a ? a.cols() : a.rows(), k = adj_a ? a.rows() : a.cols();
    const std::size_t kb = adj_b ? b.cols() : b.rows(), n = adj_b ? b.rows() : b.cols();
    if (k != kb) throw contract_violation("gemm: inner dimension mismatch");
    DenseMatrix c(m, n);
    if (c.size() == 0) return c;
    b200::check(rrsvd_b200_zgemm(b200::context(), adj_a ? RRSVD_B200_OP_C : RRSVD_B200_OP_N,
                                 adj_b ? RRSVD_B200_OP_C : RRSVD_B200_OP_N, m, n, k, b200::D(a.data()), a.cols(),
                                 b200::D(b.data()), b.cols(), b200::D(c.data()), n),
                m, n);
    return c;
}
RRSVD_B200_API DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.cols() != b.rows()) throw contract_violation("matmul: dimension mismatch");
    return gemm(a, false, b, false);
}
RRSVD_B200_API DenseMatrix adjoint(const DenseMatrix& a) {
    DenseMatrix out(a.cols(), a.rows());
    for (std::size_t j = 0; j < a.cols(); ++j)
        for (std::size_t i = 0; i < a.rows(); ++i) out(j, i) = std::conj(a(i, j));
    return out;
}
RRSVD_B200_API QrFactors qr(const DenseMatrix& a) {
    if (a.rows() < a.cols()) throw contract_violation("qr: requires rows >= cols");
    QrFactors f{DenseMatrix(a.rows(), a.cols()), DenseMatrix(a.cols(), a.cols())};
    if (a.cols() == 0) return f;
    b200::check(rrsvd_b200_qr(b200::context(), b200::D(a.data()), a.rows(), a.cols(), b200::D(f.q.data()),
                              b200::D(f.r.data())),
                a.rows(), a.cols());
    return f;
}
RRSVD_B200_API SvdResult svd_full(const DenseMatrix& a) {
    const std::size_t k = std::min(a.rows(), a.cols());
    SvdResult out;
    out.u = DenseMatrix(a.rows(), k);
    out.v = DenseMatrix(a.cols(), k);
    out.sigma.assign(k, 0.0);
    if (k > 0)
        b200::check(rrsvd_b200_svd(b200::context(), b200::D(a.data()), a.rows(), a.cols(), b200::D(out.u.data()),
                                   out.sigma.data(), b200::D(out.v.data())),
                    a.rows(), a.cols());
    out.achieved_rank = k;
    return out;
}
RRSVD_B200_API std::vector<double> singular_values(const DenseMatrix& a) {
    std::vector<double> s(std::min(a.rows(), a.cols()), 0.0);
    if (!s.empty())
        b200::check(rrsvd_b200_svd(b200::context(), b200::D(a.data()), a.rows(), a.cols(), nullptr, s.data(), nullptr),
                    a.rows(), a.cols());
    return s;
}
RRSVD_B200_API double frobenius_norm(const DenseMatrix& a) {
    double v = 0.0;
    if (a.size()) b200::check(rrsvd_b200_frobenius_norm(b200::context(), b200::D(a.data()), a.rows(), a.cols(), &v));
    return v;
}
// hermitian_eig (linalg.cpp:141-150 uses zheevd on the upper triangle): the upper triangle is
// taken as the matrix; A + s I with s = ||A||_F >= |lambda|_max is positive semidefinite, so its
// SVD on the device IS its eigendecomposition (A + sI = V diag(sigma) V^H): lambda = sigma - s.
RRSVD_B200_API HermitianEig hermitian_eig(const DenseMatrix& a) {
    if (a.rows() != a.cols()) throw contract_violation("hermitian_eig: matrix not square");
    const std::size_t n = a.rows();
    HermitianEig out{DenseMatrix(n, n), std::vector<double>(n, 0.0)};
    if (n == 0) return out;
    DenseMatrix h(n, n);
    double fro2 = 0.0;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = i; j < n; ++j) {
            h(i, j) = i == j ? cplx(a(i, i).real(), 0.0) : a(i, j);
            h(j, i) = std::conj(h(i, j));
            fro2 += (i == j ? 1.0 : 2.0) * std::norm(h(i, j));
        }
    const double shift = std::sqrt(fro2);
    for (std::size_t i = 0; i < n; ++i) h(i, i) += shift;
    const SvdResult s = svd_full(h);
    for (std::size_t j = 0; j < n; ++j) {  // descending sigma -> ascending lambda
        const std::size_t src = n - 1 - j;
        out.values[j] = s.sigma[src] - shift;
        for (std::size_t k = 0; k < n; ++k) out.vectors(k, j) = s.v(k, src);
    }
    return out;
}

// ---- randomized (randomized.cpp:79-176) on the device --------------------------------------
RRSVD_B200_API DenseMatrix gaussian_test_matrix(std::size_t n, std::size_t l, std::uint64_t seed) {
    DenseMatrix out(n, l);
    b200::check(rrsvd_b200_gaussian_test_matrix(b200::context(), n, l, seed, RRSVD_B200_OMEGA_REFERENCE,
                                                b200::D(out.data())));
    return out;
}
RRSVD_B200_API RangeBasis randomized_range_finder(const DenseMatrix& a, std::size_t l, std::size_t q,
                                                  std::uint64_t seed) {
    RangeBasis basis{DenseMatrix(a.rows(), l), l};
    b200::check(rrsvd_b200_range_finder(b200::context(), b200::D(a.data()), a.rows(), a.cols(), l, q, seed,
                                        RRSVD_B200_OMEGA_REFERENCE, nullptr, b200::D(basis.q_matrix.data())),
                a.rows(), a.cols());
    return basis;
}
RRSVD_B200_API SvdResult rrsvd_sketched_svd(const DenseMatrix& a, std::size_t l, std::size_t q, std::uint64_t seed) {
    SvdResult out;
    out.u = DenseMatrix(a.rows(), l);
    out.v = DenseMatrix(a.cols(), l);
    out.sigma.assign(l, 0.0);
    b200::check(rrsvd_b200_sketched_svd(b200::context(), b200::D(a.data()), a.rows(), a.cols(), l, q, seed,
                                        RRSVD_B200_OMEGA_REFERENCE, nullptr, b200::D(out.u.data()), out.sigma.data(),
                                        b200::D(out.v.data()), &out.discarded_weight),
                a.rows(), a.cols());
    out.achieved_rank = l;
    return out;
}
RRSVD_B200_API SvdResult rrsvd_fixed_rank(const DenseMatrix& a, const RrsvdParams& p) {
    const std::size_t k = p.target_rank;
    SvdResult out;
    out.u = DenseMatrix(a.rows(), k);
    out.v = DenseMatrix(a.cols(), k);
    out.sigma.assign(k, 0.0);
    b200::check(rrsvd_b200_fixed_rank(b200::context(), b200::D(a.data()), a.rows(), a.cols(), k, p.oversampling,
                                      p.power_iterations, p.seed, RRSVD_B200_OMEGA_REFERENCE, nullptr,
                                      b200::D(out.u.data()), out.sigma.data(), b200::D(out.v.data()),
                                      &out.discarded_weight),
                a.rows(), a.cols());
    out.achieved_rank = k;
    return out;
}
RRSVD_B200_API SvdResult rrsvd_fixed_precision(const DenseMatrix& a, const AccuracyCheckParams& check,
                                               std::size_t initial_l, std::size_t q, std::uint64_t seed) {
    const std::size_t mn = std::min(a.rows(), a.cols());
    std::vector<cplx> u(a.rows() * mn), v(a.cols() * mn);
    std::vector<double> s(mn);
    std::size_t l = 0;
    int cert = 0;
    SvdResult out;
    b200::check(rrsvd_b200_fixed_precision(b200::context(), b200::D(a.data()), a.rows(), a.cols(), initial_l, q,
                                           check.probe_count, check.growth_block, check.tolerance, seed,
                                           RRSVD_B200_OMEGA_REFERENCE, b200::D(u.data()), s.data(), b200::D(v.data()),
                                           &l, &cert, &out.discarded_weight),
                a.rows(), a.cols());
    out.u = DenseMatrix(a.rows(), l, std::vector<cplx>(u.begin(), u.begin() + static_cast<std::ptrdiff_t>(a.rows() * l)));
    out.v = DenseMatrix(a.cols(), l, std::vector<cplx>(v.begin(), v.begin() + static_cast<std::ptrdiff_t>(a.cols() * l)));
    out.sigma.assign(s.begin(), s.begin() + static_cast<std::ptrdiff_t>(l));
    out.achieved_rank = l;
    out.tolerance_certified = cert != 0;
    return out;
}
// randomized.hpp:86-89: the smallest k (0 included: nothing kept) whose implied Frobenius
// residual sqrt(||A||^2 - sum_{i<k} sigma_i^2) is within rel_tolerance * ||A||; sigma.size() if none.
RRSVD_B200_API std::size_t retained_rank_for_tolerance(const SvdResult& result, double a_frobenius_norm,
                                                       double rel_tolerance) {
    const double total = a_frobenius_norm * a_frobenius_norm, target = rel_tolerance * a_frobenius_norm;
    double kept = 0.0;
    for (std::size_t k = 0; k <= result.sigma.size(); ++k) {
        if (std::sqrt(std::max(0.0, total - kept)) <= target) return k;
        if (k < result.sigma.size()) kept += result.sigma[k] * result.sigma[k];
    }
    return result.sigma.size();
}

namespace tebd {

// ---- mps (mps.cpp:10-70) -------------------------------------------------------------------
RRSVD_B200_API std::size_t MpsState::max_bond_dim() const {
    std::size_t m = 1;
    for (const std::vector<double>& l : lambdas) m = l.size() > m ? l.size() : m;
    return m;
}
RRSVD_B200_API MpsState mps_product_state(const std::vector<std::size_t>& site_dims,
                                          const std::vector<std::vector<cplx>>& local_states, std::size_t chi_max,
                                          double trunc_tolerance) {
    const std::size_t n = site_dims.size();
    if (n == 0 || local_states.size() != n)
        throw contract_violation("mps_product_state: one local state per site required");
    MpsState st;
    st.site_dims = site_dims;
    st.chi_max = chi_max;
    st.trunc_tolerance = trunc_tolerance;
    st.gammas.reserve(n);
    for (std::size_t s = 0; s < n; ++s) {
        const std::vector<cplx>& v = local_states[s];
        if (v.size() != site_dims[s]) throw contract_violation("mps_product_state: local state dimension mismatch");
        const double nrm = std::accumulate(v.begin(), v.end(), 0.0, [](double acc, const cplx& z) { return acc + std::norm(z); });
        if (std::abs(nrm - 1.0) > 1e-10) throw contract_violation("mps_product_state: local state is not normalized");
        Tensor3 g(1, site_dims[s], 1);
        std::copy(v.begin(), v.end(), g.values.begin());
        st.gammas.push_back(std::move(g));
    }
    st.lambdas = std::vector<std::vector<double>>(n - 1, std::vector<double>(1, 1.0));
    return st;
}
RRSVD_B200_API double schmidt_entropy(const MpsState& st, std::size_t bond) {
    if (bond >= st.lambdas.size()) throw contract_violation("schmidt_entropy: bad bond");
    double s = 0.0;
    for (const double l : st.lambdas[bond])
        if (l != 0.0) s -= l * l * std::log(l * l);
    return s;
}
// <psi|O_site|psi> (mps.cpp:50-70) on the device: the site's Gamma with its two neighbouring
// lambdas as a one-site device MPS whose outer bonds are the chain's (edge weights).
RRSVD_B200_API cplx expectation_local(const MpsState& st, std::size_t site, const DenseMatrix& op) {
    if (site >= st.n_sites()) throw contract_violation("expectation_local: bad site");
    const std::size_t d = st.site_dims[site];
    if (op.rows() != d || op.cols() != d) throw contract_violation("expectation_local: operator dimension mismatch");
    const Tensor3& g = st.gammas[site];
    rrsvd_b200_mps* m = nullptr;
    b200::check(rrsvd_b200_mps_create(b200::context(), 1, &d, 0, 0.0, &m));
    struct Guard {
        rrsvd_b200_mps* m;
        ~Guard() { rrsvd_b200_mps_destroy(m); }
    } guard{m};
    const std::vector<double>* ll = site > 0 ? &st.lambdas[site - 1] : nullptr;
    const std::vector<double>* lr = site + 1 < st.n_sites() ? &st.lambdas[site] : nullptr;
    b200::check(rrsvd_b200_mps_set_edge_lambdas(m, ll ? ll->data() : nullptr, ll ? ll->size() : 0,
                                                lr ? lr->data() : nullptr, lr ? lr->size() : 0));
    b200::check(rrsvd_b200_mps_set_site(m, 0, g.dim_left, g.dim_right, b200::D(g.values.data()), nullptr));
    double out[2] = {0.0, 0.0};
    b200::check(rrsvd_b200_expectation_local(m, 0, b200::D(op.data()), out));
    return {out[0], out[1]};
}

// ---- tebd (tebd.cpp:67-326) ----------------------------------------------------------------
RRSVD_B200_API double ThetaTensor::frobenius() const {
    double v = 0.0;
    if (!values.empty())
        b200::check(rrsvd_b200_frobenius_norm(b200::context(), b200::D(values.data()), values.size(), 1, &v));
    return v;
}
// The symmetric split F(dt/2) G(dt) F(dt/2): F = odd 0-based bonds (tebd.hpp:41-50).
RRSVD_B200_API TrotterPlan trotter_plan_3rd(double dt) {
    if (dt == 0.0) throw contract_violation("trotter_plan_3rd: dt must be nonzero");
    TrotterPlan plan;
    plan.dt = dt;
    plan.order = 3;
    plan.sweeps.push_back({1, 0.5});
    plan.sweeps.push_back({0, 1.0});
    plan.sweeps.push_back({1, 0.5});
    return plan;
}

namespace detail {
inline rrsvd_b200_backend to_c(const DecimationBackend& b) {
    return rrsvd_b200_backend{b.kind == DecimationBackend::Kind::Randomized ? 1 : 0, b.target_rank, b.oversampling,
                              b.power_iterations, b.accuracy_check ? 1 : 0, b.epsilon, b.probe_count,
                              b.det_crossover, b.seed};
}
// Connected components of the exact nonzero pattern (i ~ j iff h_ij != 0 or h_ji != 0).
inline std::vector<std::vector<std::size_t>> sparsity_blocks(const DenseMatrix& h) {
    const std::size_t n = h.rows();
    std::vector<std::size_t> root(n);
    std::iota(root.begin(), root.end(), std::size_t{0});
    auto find = [&](std::size_t x) {
        while (root[x] != x) x = root[x] = root[root[x]];
        return x;
    };
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j)
            if (h(i, j) != cplx(0.0, 0.0)) root[find(i)] = find(j);
    std::map<std::size_t, std::vector<std::size_t>> groups;
    for (std::size_t i = 0; i < n; ++i) groups[find(i)].push_back(i);
    std::vector<std::vector<std::size_t>> out;
    for (auto& kv : groups) out.push_back(std::move(kv.second));
    std::sort(out.begin(), out.end());
    return out;
}
}  // namespace detail

// bond_gate (tebd.cpp:239-258): exp(-i scale h).  The same Hermiticity contract as the reference
// (asymmetry above 1e-9 max(1, |h|max) throws).  The exponential is formed block by block over
// the exact sparsity pattern (exact zeros stay exact, so number-conserving gates keep their
// block structure for the device's block-sparse gate kernel); small blocks by a host Jacobi
// with a relative stop, large ones by hermitian_eig on the device.
RRSVD_B200_API TwoSiteGate bond_gate(std::size_t bond, const DenseMatrix& h, double scale) {
    if (h.rows() != h.cols()) throw contract_violation("bond_gate: term must be square");
    const std::size_t n = h.rows();
    double asym = 0.0;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = i; j < n; ++j) asym = std::max(asym, std::abs(h(i, j) - std::conj(h(j, i))));
    if (asym > 1e-9 * std::max(1.0, h.max_abs())) throw contract_violation("bond_gate: term is not Hermitian");
    TwoSiteGate gate;
    gate.site = bond;
    gate.unitary = true;
    gate.matrix = DenseMatrix(n, n);
    for (const std::vector<std::size_t>& idx : detail::sparsity_blocks(h)) {
        const std::size_t b = idx.size();
        DenseMatrix hb(b, b), vec;
        std::vector<double> val;
        for (std::size_t i = 0; i < b; ++i)
            for (std::size_t j = 0; j < b; ++j) hb(i, j) = h(idx[i], idx[j]);
        if (b <= 32) {
            b200::small_hermitian_eig(hb, vec, val);
        } else {
            HermitianEig e = hermitian_eig(hb);
            vec = std::move(e.vectors);
            val = std::move(e.values);
        }
        std::vector<cplx> phase(b);
        for (std::size_t k = 0; k < b; ++k) phase[k] = std::exp(cplx(0.0, -scale * val[k]));
        for (std::size_t i = 0; i < b; ++i)
            for (std::size_t j = 0; j < b; ++j) {
                cplx acc(0.0, 0.0);
                for (std::size_t k = 0; k < b; ++k) acc += vec(i, k) * phase[k] * std::conj(vec(j, k));
                gate.matrix(idx[i], idx[j]) = acc;
            }
    }
    return gate;
}

RRSVD_B200_API ThetaTensor build_theta(const MpsState& st, std::size_t bond) {
    if (bond + 1 >= st.n_sites()) throw contract_violation("build_theta: bad bond");
    const Tensor3& g1 = st.gammas[bond];
    const Tensor3& g2 = st.gammas[bond + 1];
    const std::size_t d1 = g1.dim_phys, d2 = g2.dim_phys, cl = g1.dim_left, cm = g1.dim_right, cr = g2.dim_right;
    std::vector<cplx> m(d1 * cl * d2 * cr);
    ThetaTensor t(d1, d2, cl, cr);
    if (m.empty()) return t;
    auto* c = b200::context();
    b200::check(rrsvd_b200_build_theta_unfolded(c, b200::D(g1.values.data()), b200::D(g2.values.data()),
                                                bond > 0 ? st.lambdas[bond - 1].data() : nullptr,
                                                st.lambdas[bond].data(),
                                                bond + 2 < st.n_sites() ? st.lambdas[bond + 1].data() : nullptr, cl,
                                                d1, cm, d2, cr, b200::D(m.data())));
    b200::check(rrsvd_b200_unfolded_to_theta(c, b200::D(m.data()), d1, d2, cl, cr, b200::D(t.values.data())));
    return t;
}

RRSVD_B200_API ThetaTensor apply_gate_to_theta(const ThetaTensor& theta, const TwoSiteGate& gate) {
    const std::size_t dd = theta.d_left * theta.d_right;
    if (gate.matrix.rows() != dd || gate.matrix.cols() != dd)
        throw contract_violation("apply_gate_to_theta: gate dimension mismatch");
    const std::size_t cl = theta.chi_left, cr = theta.chi_right;
    ThetaTensor out(theta.d_left, theta.d_right, cl, cr);
    if (theta.values.empty()) return out;
    std::vector<cplx> m(theta.values.size()), m2(theta.values.size());
    auto* c = b200::context();
    b200::check(rrsvd_b200_theta_to_unfolded(c, b200::D(theta.values.data()), theta.d_left, theta.d_right, cl, cr,
                                             b200::D(m.data())));
    b200::check(rrsvd_b200_apply_gate_unfolded(c, b200::D(gate.matrix.data()), theta.d_left, theta.d_right, cl, cr,
                                               b200::D(m.data()), b200::D(m2.data())));
    b200::check(rrsvd_b200_unfolded_to_theta(c, b200::D(m2.data()), theta.d_left, theta.d_right, cl, cr,
                                             b200::D(out.values.data())));
    return out;
}

RRSVD_B200_API DecimationResult decimate(const ThetaTensor& theta, const std::vector<double>& lambda_left,
                                         const std::vector<double>& lambda_right, std::size_t chi_max,
                                         double trunc_tolerance, DecimationBackend& backend, bool renormalize) {
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
    // the call takes the current seed; the counter advances only when the call gets past the
    // Theta checks (tebd.cpp:156-162)
    const std::uint64_t call_seed = backend.seed;
    b200::check(rrsvd_b200_decimate_unfolded(c, b200::D(m.data()), d1, d2, cl, cr, b200::D(lambda_left),
                                             b200::D(lambda_right), chi_max, trunc_tolerance, &be, call_seed,
                                             RRSVD_B200_OMEGA_REFERENCE, nullptr, renormalize ? 1 : 0,
                                             b200::D(gl.data()), lam.data(), b200::D(gr.data()), &info),
                d1 * cl, d2 * cr);
    ++backend.seed;
    DecimationResult r;
    r.chi = info.chi;
    r.discarded = info.discarded;
    r.randomized_path = info.randomized_path != 0;
    r.tolerance_certified = info.tolerance_certified != 0;
    r.pseudo_inverse_applied = info.pseudo_inverse_applied != 0;
    r.gamma_left = Tensor3(cl, d1, r.chi);
    std::copy(gl.begin(), gl.begin() + static_cast<std::ptrdiff_t>(cl * d1 * r.chi), r.gamma_left.values.begin());
    r.gamma_right = Tensor3(r.chi, d2, cr);
    std::copy(gr.begin(), gr.begin() + static_cast<std::ptrdiff_t>(r.chi * d2 * cr), r.gamma_right.values.begin());
    r.lambda.assign(lam.begin(), lam.begin() + static_cast<std::ptrdiff_t>(r.chi));
    return r;
}

// evolve (tebd.cpp:260-326): the whole evolution runs device-resident; the state is uploaded
// once, every sweep's bonds go through the pipeline as one batch, and the state comes back at
// the end.  Gates are built once per (bond, coefficient) as the reference does (tebd.cpp:276-285).
RRSVD_B200_API EvolveDiagnostics evolve(MpsState& state, const std::vector<HamiltonianTerm>& terms,
                                        const TrotterPlan& plan, std::size_t n_steps, DecimationBackend& backend,
                                        const EvolveOptions& options) {
    const std::size_t n = state.n_sites(), nb = n > 0 ? n - 1 : 0;
    std::vector<const DenseMatrix*> bond_terms(nb, nullptr);
    for (const HamiltonianTerm& t : terms) {
        if (t.bond >= nb) throw contract_violation("evolve: term bond out of range");
        if (bond_terms[t.bond]) throw contract_violation("evolve: duplicate term on a bond");
        const std::size_t dd = state.site_dims[t.bond] * state.site_dims[t.bond + 1];
        if (t.h.rows() != dd || t.h.cols() != dd) throw contract_violation("evolve: term dimension mismatch");
        bond_terms[t.bond] = &t.h;
    }
    std::map<std::pair<std::size_t, double>, TwoSiteGate> cache;
    std::vector<const double*> table(plan.sweeps.size() * nb, nullptr);
    for (std::size_t s = 0; s < plan.sweeps.size(); ++s)
        for (std::size_t b = static_cast<std::size_t>(plan.sweeps[s].bond_parity); b < nb; b += 2) {
            if (!bond_terms[b]) continue;
            const auto key = std::make_pair(b, plan.sweeps[s].coefficient);
            auto it = cache.find(key);
            if (it == cache.end())
                it = cache.emplace(key, bond_gate(b, *bond_terms[b], plan.sweeps[s].coefficient * plan.dt)).first;
            table[s * nb + b] = b200::D(it->second.matrix.data());
        }
    auto* c = b200::context();
    rrsvd_b200_mps* dm = nullptr;
    b200::check(rrsvd_b200_mps_create(c, n, state.site_dims.data(), state.chi_max, state.trunc_tolerance, &dm));
    struct Guard {
        rrsvd_b200_mps* m;
        ~Guard() { rrsvd_b200_mps_destroy(m); }
    } guard{dm};
    std::vector<std::size_t> dims(3 * n);
    std::vector<const double*> gin(n);
    std::vector<const double*> lin(n, nullptr);
    for (std::size_t s = 0; s < n; ++s) {
        dims[3 * s] = state.gammas[s].dim_left;
        dims[3 * s + 2] = state.gammas[s].dim_right;
        gin[s] = b200::D(state.gammas[s].values.data());
        if (s < nb) lin[s] = state.lambdas[s].data();
    }
    b200::check(rrsvd_b200_state_upload(dm, dims.data(), gin.data(), lin.data()));
    std::vector<rrsvd_b200_sweep> sweeps;
    for (const TrotterPlan::Sweep& x : plan.sweeps) sweeps.push_back({x.bond_parity, x.coefficient});
    rrsvd_b200_backend be = detail::to_c(backend);
    const rrsvd_b200_evolve_options opt{options.abort_discarded_threshold, options.renormalize ? 1 : 0,
                                        RRSVD_B200_OMEGA_REFERENCE};
    rrsvd_b200_evolve_diag diag{};
    std::size_t per_step = 0;
    for (const TrotterPlan::Sweep& x : plan.sweeps)
        for (std::size_t b = static_cast<std::size_t>(x.bond_parity); b < nb; b += 2) per_step += bond_terms[b] != nullptr;
    std::vector<rrsvd_b200_update_record> rec(options.record_updates ? per_step * n_steps : 0);
    const int rc = rrsvd_b200_evolve(dm, sweeps.size(), sweeps.data(), table.data(), n_steps, &be, &opt, &diag,
                                     rec.empty() ? nullptr : rec.data(), rec.size());
    backend.seed = be.seed;
    // the device state is consistent even after a failed sweep (rejected bonds keep their
    // inputs): bring it back before reporting, like the reference's in-place MpsState
    b200::check(rrsvd_b200_state_download(dm, dims.data(), nullptr, nullptr));
    std::vector<double*> gout(n);
    std::vector<double*> lout(n, nullptr);
    for (std::size_t s = 0; s < n; ++s) {
        state.gammas[s] = Tensor3(dims[3 * s], dims[3 * s + 1], dims[3 * s + 2]);
        gout[s] = b200::D(state.gammas[s].values.data());
        if (s < nb) {
            state.lambdas[s].assign(dims[3 * s + 2], 0.0);
            lout[s] = state.lambdas[s].data();
        }
    }
    b200::check(rrsvd_b200_state_download(dm, nullptr, gout.data(), lout.data()));
    b200::check(rc);
    EvolveDiagnostics out;
    out.kept_fraction = diag.kept_fraction;
    out.max_bond_dim = diag.max_bond_dim;
    out.aborted = diag.aborted != 0;
    out.abort_step = diag.abort_step;
    const std::size_t nrec = std::min<std::size_t>(diag.n_updates, rec.size());
    for (std::size_t i = 0; i < nrec; ++i)
        out.updates.push_back({rec[i].step, rec[i].bond, rec[i].chi, rec[i].discarded_weight, rec[i].t_theta_us,
                               rec[i].t_gate_us, rec[i].t_svd_us, rec[i].randomized_path != 0});
    return out;
}

}  // namespace tebd
}  // namespace rrsvd

#endif

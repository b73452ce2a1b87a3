// rrsvd_b200/rrsvd.hpp — C++ drop-in for the reference core's TEBD decimation path.
//
// Re-declares the reference API (namespace rrsvd / rrsvd::tebd, /root/reference/proj/core/
// include/rrsvd/{errors,dense_matrix,linalg,randomized,mps,tebd}.hpp) with the same types,
// signatures, conventions and exceptions, implemented on top of the C ABI of librrsvd_b200.so
// (include/rrsvd_b200.h).  A caller that included "rrsvd/tebd.hpp" and linked rrsvd::core puts
// include/ first on its include path (include/rrsvd/*.hpp forward here) and links -lrrsvd_b200;
// every numeric call of the hot path then runs on the B200.  See INTEGRATION.md.
//
// Two build modes:
//  * header-only (default): every function below is `inline` (RRSVD_B200_API);
//  * one strong copy: a single translation unit defines RRSVD_B200_API as empty before including
//    this header, the others define RRSVD_B200_DECLARE_ONLY.  This is how the reference's own
//    test programs are linked against the drop-in while the reference's out-of-scope helpers
//    (matrix generators, chain map, error bounds; include/rrsvd_b200/reference_aux.hpp) come from
//    its own sources — tests/cpp/Makefile.
//
// Threading: one library context per host thread (thread_local), mirroring SPEC.md:112,225.
#ifndef RRSVD_B200_RRSVD_HPP
#define RRSVD_B200_RRSVD_HPP

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../rrsvd_b200.h"

#ifndef RRSVD_B200_API
#define RRSVD_B200_API inline
#endif

namespace rrsvd {

using cplx = std::complex<double>;

// ---- errors.hpp:11-32 ------------------------------------------------------------------
struct contract_violation : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct numeric_failure : std::runtime_error {
    numeric_failure(const std::string& what, std::size_t rows, std::size_t cols)
        : std::runtime_error(what + " (matrix " + std::to_string(rows) + "x" + std::to_string(cols) + ")"),
          rows(rows), cols(cols) {}
    std::size_t rows;
    std::size_t cols;
};
struct recurrence_breakdown : std::runtime_error {
    recurrence_breakdown(std::size_t index)
        : std::runtime_error("recurrence breakdown at coefficient " + std::to_string(index)), index(index) {}
    std::size_t index;
};

// ---- dense_matrix.hpp:13-49 — row-major complex matrix (same memory image) ----------------
class DenseMatrix {
  public:
    DenseMatrix() : rows_(0), cols_(0) {}
    DenseMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(rows * cols, cplx(0.0, 0.0)) {}
    DenseMatrix(std::size_t rows, std::size_t cols, std::vector<cplx> data);
    static DenseMatrix identity(std::size_t n);
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    cplx& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
    const cplx& operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
    cplx* data() { return data_.data(); }
    const cplx* data() const { return data_.data(); }
    bool all_finite() const;
    DenseMatrix left_cols(std::size_t keep) const;
    DenseMatrix hcat(const DenseMatrix& right) const;
    void scale_cols(const std::vector<double>& s);
    double max_abs() const;

  private:
    std::size_t rows_;
    std::size_t cols_;
    std::vector<cplx> data_;
};

// ---- linalg.hpp:10-56 --------------------------------------------------------------------
struct QrFactors {
    DenseMatrix q;
    DenseMatrix r;
};
struct SvdResult {
    DenseMatrix u;
    std::vector<double> sigma;
    DenseMatrix v;
    double discarded_weight = 0.0;
    std::size_t achieved_rank = 0;
    bool tolerance_certified = true;
};
struct HermitianEig {
    DenseMatrix vectors;
    std::vector<double> values;
};
DenseMatrix gemm(const DenseMatrix& a, bool adj_a, const DenseMatrix& b, bool adj_b);
DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b);
DenseMatrix adjoint(const DenseMatrix& a);
QrFactors qr(const DenseMatrix& a);
SvdResult svd_full(const DenseMatrix& a);
std::vector<double> singular_values(const DenseMatrix& a);
double frobenius_norm(const DenseMatrix& a);
HermitianEig hermitian_eig(const DenseMatrix& a);

// ---- randomized.hpp:17-89 ----------------------------------------------------------------
struct RrsvdParams {
    std::size_t target_rank;
    std::size_t oversampling;
    std::size_t power_iterations;
    std::uint64_t seed;
};
struct RangeBasis {
    DenseMatrix q_matrix;
    std::size_t l;
};
struct AccuracyCheckParams {
    double tolerance;
    std::size_t probe_count;
    std::size_t growth_block = 0;  // columns appended per failed round; 0 doubles the basis
};
struct ErrorBoundReport {
    double expected_bound;
    double tail_bound;
    double failure_probability;
    double frobenius_cap;
};
DenseMatrix gaussian_test_matrix(std::size_t n, std::size_t l, std::uint64_t seed);
RangeBasis randomized_range_finder(const DenseMatrix& a, std::size_t l, std::size_t q, std::uint64_t seed);
SvdResult rrsvd_sketched_svd(const DenseMatrix& a, std::size_t l, std::size_t q, std::uint64_t seed);
SvdResult rrsvd_fixed_rank(const DenseMatrix& a, const RrsvdParams& params);
SvdResult rrsvd_fixed_precision(const DenseMatrix& a, const AccuracyCheckParams& check, std::size_t initial_l,
                                std::size_t q, std::uint64_t seed);
std::size_t retained_rank_for_tolerance(const SvdResult& result, double a_frobenius_norm, double rel_tolerance);

namespace tebd {

// ---- mps.hpp:12-49 ---------------------------------------------------------------------
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
    std::size_t max_bond_dim() const;
};
MpsState mps_product_state(const std::vector<std::size_t>& site_dims, const std::vector<std::vector<cplx>>& local_states,
                           std::size_t chi_max = 0, double trunc_tolerance = 0.0);
double schmidt_entropy(const MpsState& state, std::size_t bond);
cplx expectation_local(const MpsState& state, std::size_t site, const DenseMatrix& op);

// ---- tebd.hpp:15-138 -------------------------------------------------------------------
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
    double frobenius() const;
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
TrotterPlan trotter_plan_3rd(double dt);
struct DecimationBackend {
    enum class Kind { Deterministic, Randomized };
    Kind kind = Kind::Deterministic;
    std::size_t target_rank = 0;
    std::size_t oversampling = 0;
    std::size_t power_iterations = 2;
    bool accuracy_check = false;
    double epsilon = 1e-3;
    std::size_t probe_count = 10;
    std::size_t det_crossover = 256;
    std::uint64_t seed = 0;
};
struct DecimationResult {
    Tensor3 gamma_left;
    std::vector<double> lambda;
    Tensor3 gamma_right;
    double discarded = 0.0;
    std::size_t chi = 0;
    bool randomized_path = false;
    bool tolerance_certified = true;
    bool pseudo_inverse_applied = false;
};
ThetaTensor build_theta(const MpsState& state, std::size_t bond);
ThetaTensor apply_gate_to_theta(const ThetaTensor& theta, const TwoSiteGate& gate);
DecimationResult decimate(const ThetaTensor& theta, const std::vector<double>& lambda_left,
                          const std::vector<double>& lambda_right, std::size_t chi_max, double trunc_tolerance,
                          DecimationBackend& backend, bool renormalize = true);
TwoSiteGate bond_gate(std::size_t bond, const DenseMatrix& h, double scale);
struct UpdateRecord {
    std::size_t step;
    std::size_t bond;
    std::size_t chi;
    double discarded_weight;
    double t_theta_us;
    double t_gate_us;
    double t_svd_us;
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
EvolveDiagnostics evolve(MpsState& state, const std::vector<HamiltonianTerm>& terms, const TrotterPlan& plan,
                         std::size_t n_steps, DecimationBackend& backend, const EvolveOptions& options = {});

}  // namespace tebd
}  // namespace rrsvd

#ifndef RRSVD_B200_DECLARE_ONLY
#include "rrsvd_impl.hpp"
#endif

#endif

// rrsvd_b200/reference_aux.hpp — DECLARATIONS ONLY of the reference API that lies outside the
// decimation hot path (SURVEY.md §2 marks these out of scope): matrix generators (matgen.hpp),
// the chain map (chainmap.hpp), the RRSM / value-list files (matrix_io.hpp), the a-priori error
// bounds and probe estimates (randomized.hpp:38-89), the power-iteration norm estimate
// (linalg.hpp:52-53), the dense oracle and the spin-model builders (tebd.hpp:145-156), and the
// dense state vector (mps.hpp:51-52).
//
// The drop-in does not define them.  A program that calls them links the reference's own
// sources for these symbols, with the hot-path symbols supplied by the drop-in (the reference
// objects' symbols weakened) — the recipe in tests/cpp/Makefile, which builds the reference's
// acceptance and unit-test programs unchanged this way.  Types and signatures match the
// reference headers exactly so those objects link.
#ifndef RRSVD_B200_REFERENCE_AUX_HPP
#define RRSVD_B200_REFERENCE_AUX_HPP

#include <cstdint>
#include <string>
#include <vector>

#include "rrsvd.hpp"

namespace rrsvd {

// linalg.hpp (power iteration on A^H A with an SVD fallback)
double operator_norm_estimate(const DenseMatrix& a);

// randomized.hpp: a-priori bounds (Halko, Martinsson & Tropp) and probe estimates
ErrorBoundReport error_bound_report(const std::vector<double>& sigma, std::size_t k, std::size_t p, std::size_t q);
double frobenius_cap(double sigma1);
double residual_frobenius(const DenseMatrix& a, const RangeBasis& basis);
double probe_operator_bound(const DenseMatrix& m, std::size_t r, std::uint64_t seed);

// matgen.hpp: synthetic spectra and Haar-random structured matrices
struct SpectrumSpec {
    std::vector<double> values;
    std::string label;
};
struct StructuredInstance {
    DenseMatrix matrix;
    SpectrumSpec spectrum;
    std::uint64_t u_seed;
    std::uint64_t v_seed;
};
SpectrumSpec make_spectrum(std::vector<double> values, std::string label);
DenseMatrix random_orthonormal(std::size_t m, std::size_t n, std::uint64_t seed);
StructuredInstance structured_matrix(const SpectrumSpec& spec, std::size_t m, std::uint64_t u_seed,
                                     std::uint64_t v_seed);
SpectrumSpec spectrum_exponential(std::size_t n, double ratio);
SpectrumSpec spectrum_power(std::size_t n);
double discarded_weight(const SpectrumSpec& spec, std::size_t k);
double frobenius_tail(const SpectrumSpec& spec, std::size_t k);
double calibrate_exponential_ratio(std::size_t n, std::size_t k, double target_weight);

// matrix_io.hpp: RRSM v1 binary matrices and plain value lists
void write_rrsm(const std::string& path, const DenseMatrix& a);
DenseMatrix read_rrsm(const std::string& path);
void write_value_lines(const std::string& path, const std::vector<double>& values);
std::vector<double> read_value_lines(const std::string& path);

namespace tebd {
// mps.hpp (guarded to small chains)
std::vector<cplx> dense_coefficients(const MpsState& state);
// tebd.hpp: exact propagation and model builders
std::vector<cplx> dense_oracle_evolve(const std::vector<cplx>& initial, const std::vector<std::size_t>& site_dims,
                                      const std::vector<HamiltonianTerm>& terms, double time);
std::vector<HamiltonianTerm> ising_terms(std::size_t n_sites, double coupling, double field);
std::vector<HamiltonianTerm> heisenberg_terms(std::size_t n_sites, double coupling);
}  // namespace tebd

// chainmap.hpp: TEDOPA measure -> chain map (input preparation)
namespace chainmap {
struct MeasureGrid {
    std::vector<double> nodes;
    std::vector<double> weights;
};
struct ChainCoefficients {
    double t0 = 0.0;
    std::vector<double> omegas;
    std::vector<double> hoppings;
};
struct SpectralDensityInput {
    std::vector<double> x;
    std::vector<double> g;
    std::vector<double> h;
    double x_max = 0.0;
};
struct ChainSystem {
    std::vector<std::size_t> site_dims;
    std::vector<tebd::HamiltonianTerm> bond_terms;
};
MeasureGrid make_measure(std::vector<double> nodes, std::vector<double> weights);
MeasureGrid trapezoid_measure(const std::vector<double>& nodes, const std::vector<double>& h2);
std::vector<double> spectral_density(const SpectralDensityInput& input, const std::vector<double>& omega_grid);
ChainCoefficients stieltjes_coefficients(const MeasureGrid& measure, std::size_t n_chain);
double stieltjes_orthonormality_residual(const MeasureGrid& measure, std::size_t n_chain);
DenseMatrix boson_annihilation(std::size_t d);
DenseMatrix boson_number(std::size_t d);
ChainSystem build_chain_terms(const ChainCoefficients& coeffs, std::size_t boson_dim, const DenseMatrix& system_term,
                              const DenseMatrix& coupling_op);
MeasureGrid read_measure_file(const std::string& path);
void write_coefficients_file(const std::string& path, const ChainCoefficients& coeffs);
ChainCoefficients read_coefficients_file(const std::string& path);
}  // namespace chainmap

}  // namespace rrsvd

#endif

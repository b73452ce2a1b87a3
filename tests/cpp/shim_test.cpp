// Drop-in proof: reference-style test bodies (test_tebd.cpp, test_randomized.cpp,
// test_linalg.cpp) written against the reference API, compiled against the B200 shim
// (include/rrsvd_b200/rrsvd.hpp) instead of the reference headers, run on the device.
#include <cmath>
#include <cstdio>
#include <numbers>

#include "rrsvd_b200/partition.hpp"
#include "rrsvd_b200/rrsvd.hpp"

using namespace rrsvd;
using namespace rrsvd::tebd;

static int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

int main() {
    const std::vector<cplx> up{1.0, 0.0}, down{0.0, 1.0};
    {  // test_tebd.cpp:165-177 Bell pair
        ThetaTensor bell(2, 2, 1, 1);
        bell.at(0, 0, 0, 0) = 1.0 / std::numbers::sqrt2;
        bell.at(1, 1, 0, 0) = 1.0 / std::numbers::sqrt2;
        DecimationBackend be;
        const DecimationResult d = decimate(bell, {}, {}, 4, 0.0, be);
        CHECK(d.lambda.size() == 2);
        CHECK(std::abs(d.lambda[0] - 1.0 / std::numbers::sqrt2) < 1e-12);
        CHECK(be.seed == 1);
    }
    {  // test_tebd.cpp:158-163 product state keeps chi 1
        const MpsState st = mps_product_state({2, 2}, {up, up});
        DecimationBackend be;
        const DecimationResult d = decimate(build_theta(st, 0), {}, {}, 4, 0.0, be);
        CHECK(d.chi == 1);
        CHECK(std::abs(d.discarded) < 1e-15);
    }
    {  // test_tebd.cpp:179-233 deterministic vs randomized decimation mid-simulation
        MpsState st = mps_product_state({2, 2, 2, 2, 2, 2}, {up, down, up, down, up, down}, 8, 0.0);
        std::vector<HamiltonianTerm> terms;
        DenseMatrix h(4, 4);  // Heisenberg term, Pauli convention
        h(0, 0) = 1; h(3, 3) = 1; h(1, 1) = -1; h(2, 2) = -1; h(1, 2) = 2; h(2, 1) = 2;
        for (std::size_t b = 0; b < 5; ++b) terms.push_back({b, h});
        DecimationBackend det;
        evolve(st, terms, trotter_plan_3rd(0.05), 6, det);
        const ThetaTensor theta = apply_gate_to_theta(build_theta(st, 2), bond_gate(2, terms[2].h, 0.05));
        DecimationBackend det2, rnd;
        rnd.kind = DecimationBackend::Kind::Randomized;
        rnd.target_rank = 8; rnd.oversampling = 8; rnd.det_crossover = 0; rnd.seed = 5;
        const DecimationResult a = decimate(theta, st.lambdas[1], st.lambdas[3], 8, 0.0, det2);
        const DecimationResult b = decimate(theta, st.lambdas[1], st.lambdas[3], 8, 0.0, rnd);
        CHECK(b.randomized_path);
        CHECK(a.lambda.size() == b.lambda.size());
        for (std::size_t i = 0; i < std::min(a.lambda.size(), b.lambda.size()); ++i)
            CHECK(std::abs(a.lambda[i] - b.lambda[i]) < 1e-8);
    }
    {  // test_linalg.cpp:114-121 QR
        const DenseMatrix a = gaussian_test_matrix(50, 12, 3);
        const QrFactors f = qr(a);
        const DenseMatrix qhq = gemm(f.q, true, f.q, false);
        double e = 0.0;
        for (std::size_t i = 0; i < 12; ++i)
            for (std::size_t j = 0; j < 12; ++j) e += std::norm(qhq(i, j) - (i == j ? 1.0 : 0.0));
        CHECK(std::sqrt(e) < 1e-12);
    }
    {  // test_randomized.cpp:91-101 exact low rank
        const DenseMatrix l = gaussian_test_matrix(120, 6, 1), r = gaussian_test_matrix(80, 6, 2);
        const DenseMatrix a = gemm(l, false, adjoint(r), false);
        const SvdResult full = svd_full(a);
        const SvdResult rr = rrsvd_fixed_rank(a, {6, 4, 1, 9});
        for (std::size_t i = 0; i < 6; ++i) CHECK(std::abs(rr.sigma[i] - full.sigma[i]) < 1e-10 * full.sigma[0]);
    }
    {  // test_randomized.cpp fixed-precision shape: exact rank 6 is certified at l = 8
        const DenseMatrix l = gaussian_test_matrix(120, 6, 4), r = gaussian_test_matrix(80, 6, 5);
        const DenseMatrix a = gemm(l, false, adjoint(r), false);
        const SvdResult fp = rrsvd_fixed_precision(a, {1e-8, 4}, 8, 1, 11);
        CHECK(fp.tolerance_certified);
        CHECK(fp.achieved_rank == 8);
        const SvdResult fg = rrsvd_fixed_precision(a, {1e-8, 4, 3}, 2, 1, 11);  // growth_block 3: 2 -> 5 -> 8
        CHECK(fg.tolerance_certified);
        CHECK(fg.achieved_rank == 8);
        const SvdResult full = svd_full(a);
        for (std::size_t i = 0; i < 6; ++i) CHECK(std::abs(fp.sigma[i] - full.sigma[i]) < 1e-10 * full.sigma[0]);
    }
    {  // bond_gate is unitary (test_tebd.cpp:143-155 shape)
        DenseMatrix h(4, 4);
        h(0, 1) = cplx(0.3, 0.2); h(1, 0) = cplx(0.3, -0.2); h(2, 2) = 1.5; h(3, 0) = 0.7; h(0, 3) = 0.7;
        const TwoSiteGate g = bond_gate(0, h, 0.9);
        const DenseMatrix u = gemm(g.matrix, true, g.matrix, false);
        double e = 0.0;
        for (std::size_t i = 0; i < 4; ++i)
            for (std::size_t j = 0; j < 4; ++j) e += std::norm(u(i, j) - (i == j ? 1.0 : 0.0));
        CHECK(std::sqrt(e) < 1e-12);
    }
    {  // the partition through the C++ drop-in: one rank (loopback) == the single-GPU evolve
        std::vector<HamiltonianTerm> terms;
        DenseMatrix h(4, 4);
        h(0, 0) = 1; h(3, 3) = 1; h(1, 1) = -1; h(2, 2) = -1; h(1, 2) = 2; h(2, 1) = 2;
        for (std::size_t b = 0; b < 5; ++b) terms.push_back({b, h});
        MpsState a = mps_product_state({2, 2, 2, 2, 2, 2}, {up, down, up, down, up, down}, 8, 0.0);
        MpsState bl = a;
        DecimationBackend b1, b2;
        b1.kind = b2.kind = DecimationBackend::Kind::Randomized;
        b1.target_rank = b2.target_rank = 8; b1.oversampling = b2.oversampling = 4;
        b1.det_crossover = b2.det_crossover = 0; b1.seed = b2.seed = 13;
        evolve(a, terms, trotter_plan_3rd(0.05), 4, b1);
        rrsvd_b200_loopback_hub* hub = nullptr;
        rrsvd_b200_comm* comm = nullptr;
        CHECK(rrsvd_b200_loopback_hub_create(1, &hub) == 0);
        CHECK(rrsvd_b200_comm_create_loopback(rrsvd::b200::context(), hub, 0, &comm) == 0);
        tebd::b200ext::evolve_partitioned(bl, comm, 0, 6, terms, trotter_plan_3rd(0.05), 4, b2);
        CHECK(b1.seed == b2.seed);
        for (std::size_t k = 0; k < 5; ++k) {
            CHECK(a.lambdas[k].size() == bl.lambdas[k].size());
            for (std::size_t i = 0; i < std::min(a.lambdas[k].size(), bl.lambdas[k].size()); ++i)
                CHECK(std::abs(a.lambdas[k][i] - bl.lambdas[k][i]) < 1e-12);
        }
        rrsvd_b200_comm_destroy(comm);
        rrsvd_b200_loopback_hub_destroy(hub);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "shim_test passed", failures);
    return failures ? 1 : 0;
}

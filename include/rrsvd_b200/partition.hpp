// rrsvd_b200/partition.hpp — the chain-block partition for C++ callers of the
// drop-in: one rank's block of a chain evolved with rrsvd_b200_evolve_partitioned (NCCL between
// GPUs, or the host loopback between threads), with the reference's own types.  The block is an
// MpsState holding the rank's owned sites plus, unless it is the last rank, a ghost copy of the
// next rank's first site; its lambdas are the local bonds.  Terms, plan and backend are the
// global ones of the reference's evolve (tebd.hpp:142-144); seeds are global call indices, so the
// ranks together reproduce the single-GPU evolve.
#ifndef RRSVD_B200_PARTITION_HPP
#define RRSVD_B200_PARTITION_HPP

#include "rrsvd.hpp"

namespace rrsvd::tebd::b200ext {

inline EvolveDiagnostics evolve_partitioned(MpsState& block, rrsvd_b200_comm* comm, std::size_t first_site,
                                            std::size_t n_global, const std::vector<HamiltonianTerm>& terms,
                                            const TrotterPlan& plan, std::size_t n_steps, DecimationBackend& backend,
                                            std::uint64_t step0 = 0) {
    const std::size_t n = block.n_sites(), nb = n > 0 ? n - 1 : 0;
    if (n == 0 || first_site + n > n_global) throw contract_violation("evolve_partitioned: block outside the chain");
    std::vector<unsigned char> flags(n_global > 0 ? n_global - 1 : 0, 0);
    std::vector<const DenseMatrix*> term_of(flags.size(), nullptr);
    for (const HamiltonianTerm& t : terms) {
        if (t.bond >= flags.size()) throw contract_violation("evolve_partitioned: term bond out of range");
        flags[t.bond] = 1;
        term_of[t.bond] = &t.h;
    }
    auto* c = rrsvd::b200::context();
    // gates of my local bonds, made resident once per (bond, coefficient) (tebd.cpp:276-285)
    std::vector<rrsvd_b200_gate*> made;
    struct GateGuard {
        std::vector<rrsvd_b200_gate*>& g;
        ~GateGuard() { for (auto* x : g) rrsvd_b200_gate_destroy(x); }
    } gguard{made};
    std::map<std::pair<std::size_t, double>, rrsvd_b200_gate*> cache;
    std::vector<const rrsvd_b200_gate*> table(plan.sweeps.size() * nb, nullptr);
    for (std::size_t s = 0; s < plan.sweeps.size(); ++s)
        for (std::size_t lb = 0; lb < nb; ++lb) {
            const std::size_t gb = first_site + lb;
            if ((int)(gb % 2) != plan.sweeps[s].bond_parity || !term_of[gb]) continue;
            const auto key = std::make_pair(gb, plan.sweeps[s].coefficient);
            auto it = cache.find(key);
            if (it == cache.end()) {
                const TwoSiteGate g = bond_gate(gb, *term_of[gb], plan.sweeps[s].coefficient * plan.dt);
                rrsvd_b200_gate* h = nullptr;
                rrsvd::b200::check(rrsvd_b200_gate_create(c, rrsvd::b200::D(g.matrix.data()), g.matrix.rows(), &h));
                made.push_back(h);
                it = cache.emplace(key, h).first;
            }
            table[s * nb + lb] = it->second;
        }
    rrsvd_b200_mps* dm = nullptr;
    rrsvd::b200::check(rrsvd_b200_mps_create(c, n, block.site_dims.data(), block.chi_max, block.trunc_tolerance, &dm));
    struct Guard {
        rrsvd_b200_mps* m;
        ~Guard() { rrsvd_b200_mps_destroy(m); }
    } guard{dm};
    // provisional unit edge weights (the first exchange replaces them with the neighbours' λ)
    const std::vector<double> left(block.gammas.front().dim_left, 1.0), right(block.gammas.back().dim_right, 1.0);
    rrsvd::b200::check(rrsvd_b200_mps_set_edge_lambdas(dm, first_site > 0 ? left.data() : nullptr, left.size(),
                                                        first_site + n < n_global ? right.data() : nullptr,
                                                        right.size()));
    std::vector<std::size_t> dims(3 * n);
    std::vector<const double*> gin(n), lin(n, nullptr);
    for (std::size_t s = 0; s < n; ++s) {
        dims[3 * s] = block.gammas[s].dim_left;
        dims[3 * s + 2] = block.gammas[s].dim_right;
        gin[s] = rrsvd::b200::D(block.gammas[s].values.data());
        if (s < nb) lin[s] = block.lambdas[s].data();
    }
    rrsvd::b200::check(rrsvd_b200_state_upload(dm, dims.data(), gin.data(), lin.data()));
    std::vector<rrsvd_b200_sweep> sweeps;
    for (const TrotterPlan::Sweep& x : plan.sweeps) sweeps.push_back({x.bond_parity, x.coefficient});
    rrsvd_b200_backend be = detail::to_c(backend);
    const rrsvd_b200_evolve_options opt{1.0, 1, RRSVD_B200_OMEGA_REFERENCE};
    rrsvd_b200_evolve_diag diag{};
    const int rc = rrsvd_b200_evolve_partitioned(dm, comm, first_site, n_global, sweeps.size(), sweeps.data(),
                                                 table.data(), flags.data(), n_steps, step0, &be, &opt, &diag);
    backend.seed = be.seed;
    rrsvd::b200::check(rc);
    rrsvd::b200::check(rrsvd_b200_state_download(dm, dims.data(), nullptr, nullptr));
    std::vector<double*> gout(n), lout(n, nullptr);
    for (std::size_t s = 0; s < n; ++s) {
        block.gammas[s] = Tensor3(dims[3 * s], dims[3 * s + 1], dims[3 * s + 2]);
        gout[s] = rrsvd::b200::D(block.gammas[s].values.data());
        if (s < nb) {
            block.lambdas[s].assign(dims[3 * s + 2], 0.0);
            lout[s] = block.lambdas[s].data();
        }
    }
    rrsvd::b200::check(rrsvd_b200_state_download(dm, nullptr, gout.data(), lout.data()));
    EvolveDiagnostics out;
    out.kept_fraction = diag.kept_fraction;
    out.max_bond_dim = diag.max_bond_dim;
    return out;
}

}  // namespace rrsvd::tebd::b200ext

#endif

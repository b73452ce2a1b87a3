// mps.cuh — the device-resident MpsState and prepared gates (shared by evolve.cu and
// partition.cu).
#pragma once
#include <vector>

#include "../../include/rrsvd_b200.h"
#include "pipeline.cuh"

using rb::cplx;

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
    std::vector<char> sat;      // per bond: its last decimation kept its kmax (speculation history)
    size_t edge_n[2] = {0, 0};
    size_t edge_cap[2] = {0, 0};
    const double* ll_of(int b) const { return b > 0 ? lam[b - 1] : edge[0]; }
    const double* lr_of(int b) const { return b + 2 < n ? lam[b + 1] : edge[1]; }
};


// A gate resident on the device with its exact block structure (made once, reused by every
// sweep and every evolve call).
struct rrsvd_b200_gate {
    rrsvd_b200_ctx* c = nullptr;
    int dd = 0;
    cplx* dev = nullptr;
    bool blocked = false;
    rb::GateBlocksOwned blk;
};


namespace rb {
// evolve (tebd.cpp:260-326) on a device MPS: n_steps x sweeps, every sweep's bonds as one batch
// (evolve.cu).  Throws Fail; the caller is a C-ABI wrapper.
void evolve_core(rrsvd_b200_mps* s, rrsvd_b200_ctx* c, size_t n_sweeps, const rrsvd_b200_sweep* sweeps,
                 const rrsvd_b200_gate* const* gates, size_t n_steps, rrsvd_b200_backend* be,
                 const rrsvd_b200_evolve_options* opt, rrsvd_b200_evolve_diag* diag,
                 rrsvd_b200_update_record* records, size_t max_records);
}  // namespace rb

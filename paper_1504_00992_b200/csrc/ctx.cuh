// ctx.cuh — library context: stream, device workspace arena, host staging, error state.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

struct rrsvd_b200_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;  // current stream (a lane or the side stream inside a call)
    cudaStream_t home = nullptr;    // the caller's stream (ctx_create / set_stream)
    bool own_stream = false;
    std::string err;
    uint64_t launches = 0;

    // Pinned host scratch for small results (info structs, scalars).
    void* pinned = nullptr;
    size_t pinned_cap = 0;
    // A separate pinned region for evolve's per-sweep scalars: two sweeps may be in flight while
    // the kernels' own host reads (block Jacobi, accuracy check) use `pinned`.
    void* pinned_sweep = nullptr;
    size_t pinned_sweep_cap = 0;
    // Buffers allocated for host-pointer staging during one call, freed at call end.
    std::vector<void*> staged;

    // Optional per-launch timing of the zgemm stage (CUDA events on the context stream).
    struct PendingGemm {
        cudaEvent_t a, b;
        double flops;     // algorithmic: 8 real flops per complex MAC
        double executed;  // what the DMMA pipe executes (6 per complex MAC in the 3M form)
        int tag;
        int tma;          // staged by TMA (1) or cp.async (0)
        int kind = 0;     // 0: DMMA zgemm; 1: INT8 emulated A-product (ozaki.cuh) or its A preparation;
                          // 2: the INT8 tensor-core GEMM kernel of an emulated product alone
        double bytes = 0; // emulated launches: algorithmic HBM bytes
    };
    int gemm_tag = 0;              // category of the next zgemm launches (debug statistics)
    double tag_ms[8] = {}, tag_flops[8] = {};
    bool gemm_timing = false;
    std::vector<PendingGemm> pending;
    std::vector<cudaEvent_t> event_pool;

    // Two auxiliary streams ("lanes") so independent halves of a sweep overlap: one lane's
    // latency-bound small kernels (Cholesky, Jacobi) run beside the other lane's GEMMs.
    static constexpr int kMaxLanes = 8;
    cudaStream_t lane[kMaxLanes] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[kMaxLanes] = {};
    bool use_lanes = true;
    int n_lanes = 2;  // RRSVD_B200_LANES overrides
    double gemm_ms = 0.0, gemm_flops = 0.0, gemm_exec_flops = 0.0, gemm_tma_ms = 0.0;
    // the emulated A-products (kind 1), kept out of the DMMA counters: products, A preparation
    double oz_ms = 0.0, oz_flops = 0.0, oz_bytes = 0.0, oz_prep_ms = 0.0, oz_prep_bytes = 0.0;
    uint64_t oz_calls = 0;
    double oz_gemm_ms = 0.0, oz_gemm_bytes = 0.0;
    uint64_t gemm_calls = 0;
};

namespace rb {

// Status codes (include/rrsvd_b200.h)
constexpr int kOk = 0, kContract = 1, kNumeric = 2, kCuda = 3;

struct Fail {
    int code;
};

int fail_cuda(cudaError_t e, const char* what, const char* file, int line);

// Thrown inside the library, converted to a status code at the C boundary.
[[noreturn]] void throw_contract(rrsvd_b200_ctx* c, const std::string& msg);
[[noreturn]] void throw_numeric(rrsvd_b200_ctx* c, const std::string& msg);
void check_cuda(rrsvd_b200_ctx* c, cudaError_t e, const char* what);
inline void check_launch(rrsvd_b200_ctx* c, const char* what) {
    c->launches++;
    check_cuda(c, cudaGetLastError(), what);
}

// Workspace (stream-ordered pool; released at the end of each public call)
void* ws_alloc(rrsvd_b200_ctx* c, size_t bytes);
template <class T>
T* ws_get(rrsvd_b200_ctx* c, size_t count) {
    return static_cast<T*>(ws_alloc(c, count * sizeof(T)));
}
void ws_reset(rrsvd_b200_ctx* c);

// Host/device pointer handling for the "device or host memory" ABI convention.
bool is_device_ptr(const void* p);
// Input: returns a device pointer holding `bytes` from p (H2D-staged if p is host memory).
const void* stage_in(rrsvd_b200_ctx* c, const void* p, size_t bytes);
// Output: returns a device pointer to write into; finish_out copies back if p was host memory.
struct OutBuf {
    void* host = nullptr;
    void* dev = nullptr;
    size_t bytes = 0;
};
void* stage_out(rrsvd_b200_ctx* c, void* p, size_t bytes, std::vector<OutBuf>& outs);
void finish_out(rrsvd_b200_ctx* c, std::vector<OutBuf>& outs);  // D2H copies + sync
void release_staged(rrsvd_b200_ctx* c);

// Lanes: fork(c) makes both lanes wait for the work already queued on c->stream; join(c)
// makes c->stream wait for both lanes.  release_lanes at context destruction.
void lanes_fork(rrsvd_b200_ctx* c, int n);
void lanes_join(rrsvd_b200_ctx* c, int n);
void release_lanes(rrsvd_b200_ctx* c);
// After a failed public call: put c->stream back on the caller's stream and drain every lane
// and the side stream, so no work the failed call forked still uses the workspace that the
// boundary releases next (and later calls order against the caller's stream again).
void recover_after_failure(rrsvd_b200_ctx* c);
// Scoped stream switch: restores c->stream on every exit path (normal or exception).
struct StreamSwitch {
    rrsvd_b200_ctx* c;
    cudaStream_t saved;
    explicit StreamSwitch(rrsvd_b200_ctx* cc) : c(cc), saved(cc->stream) {}
    ~StreamSwitch() { c->stream = saved; }
    StreamSwitch(const StreamSwitch&) = delete;
    StreamSwitch& operator=(const StreamSwitch&) = delete;
};

// zgemm timing: events around each GEMM launch (incl. its split-K reduction) while enabled.
cudaEvent_t pooled_event(rrsvd_b200_ctx* c);
void flush_gemm_timing(rrsvd_b200_ctx* c);  // waits for pending events, accumulates
void* pinned_scratch(rrsvd_b200_ctx* c, size_t bytes);
void* pinned_sweep_scratch(rrsvd_b200_ctx* c, size_t bytes);

}  // namespace rb

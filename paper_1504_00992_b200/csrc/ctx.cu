#include <cstdlib>
// ctx.cu — context, workspace and host/device staging.
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>

#include "ctx.cuh"

namespace rb {

cudaError_t smem_atleast(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> set;  // (kernel, device) -> attribute
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = set[{kernel, dev}];
    if (bytes <= cur) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

namespace {
struct Thrown : std::exception {
    int code;
    explicit Thrown(int c) : code(c) {}
};
}  // namespace

int fail_cuda(cudaError_t e, const char* what, const char* file, int line) {
    (void)e; (void)what; (void)file; (void)line;
    return kCuda;
}

void throw_contract(rrsvd_b200_ctx* c, const std::string& msg) {
    c->err = msg;
    throw Fail{kContract};
}
void throw_numeric(rrsvd_b200_ctx* c, const std::string& msg) {
    c->err = msg;
    throw Fail{kNumeric};
}
void check_cuda(rrsvd_b200_ctx* c, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    c->err = std::string(what) + ": " + cudaGetErrorString(e);
    throw Fail{kCuda};
}

// The workspace uses the device's stream-ordered memory pool: allocations are recycled
// without synchronisation and released at the end of every public call.
void* ws_alloc(rrsvd_b200_ctx* c, size_t bytes) {
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    check_cuda(c, cudaMallocAsync(&p, bytes, c->stream), "cudaMallocAsync(workspace)");
    c->staged.push_back(p);
    return p;
}

void ws_reset(rrsvd_b200_ctx* c) { release_staged(c); }

bool is_device_ptr(const void* p) {
    if (p == nullptr) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

const void* stage_in(rrsvd_b200_ctx* c, const void* p, size_t bytes) {
    if (p == nullptr || is_device_ptr(p)) return p;
    void* d = ws_alloc(c, bytes);
    check_cuda(c, cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, c->stream), "H2D staging");
    return d;
}

void* stage_out(rrsvd_b200_ctx* c, void* p, size_t bytes, std::vector<OutBuf>& outs) {
    if (p == nullptr || is_device_ptr(p)) return p;
    void* d = ws_alloc(c, bytes);
    outs.push_back({p, d, bytes});
    return d;
}

void finish_out(rrsvd_b200_ctx* c, std::vector<OutBuf>& outs) {
    for (const OutBuf& o : outs)
        if (o.bytes)
            check_cuda(c, cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, c->stream),
                       "D2H staging");
    check_cuda(c, cudaStreamSynchronize(c->stream), "stream sync");
    outs.clear();
}

void release_staged(rrsvd_b200_ctx* c) {
    for (void* p : c->staged) cudaFreeAsync(p, c->stream);
    c->staged.clear();
}

void lanes_fork(rrsvd_b200_ctx* c, int n) {
    if (c->ev_fork == nullptr)
        check_cuda(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "lane event");
    // RRSVD_B200_LANE_PRIO=1: lane 0 at the device's greatest stream priority, the other lanes at
    // the least — lane 0's CTAs are scheduled first whenever SMs free up and the other lanes fill
    // what it leaves (an A/B switch; default off: equal priorities — measured C3 7.26 vs 7.46
    // steps/s, C3 p=100 3.05 either way: the favoured lane finishes early and the other's tail
    // then runs without an overlap partner)
    static const bool prio = [] {
        const char* e = std::getenv("RRSVD_B200_LANE_PRIO");
        return e != nullptr && std::atoi(e) != 0;
    }();
    int least = 0, greatest = 0;
    if (prio) check_cuda(c, cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
    for (int i = 0; i < n; ++i)
        if (c->lane[i] == nullptr) {
            check_cuda(c, cudaStreamCreateWithPriority(&c->lane[i], cudaStreamNonBlocking,
                                                       prio ? (i == 0 ? greatest : least) : 0),
                       "lane stream");
            check_cuda(c, cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming), "lane event");
        }
    check_cuda(c, cudaEventRecord(c->ev_fork, c->stream), "fork record");
    for (int i = 0; i < n; ++i) check_cuda(c, cudaStreamWaitEvent(c->lane[i], c->ev_fork, 0), "fork wait");
}

void lanes_join(rrsvd_b200_ctx* c, int n) {
    for (int i = 0; i < n; ++i) {
        check_cuda(c, cudaEventRecord(c->ev_join[i], c->lane[i]), "join record");
        check_cuda(c, cudaStreamWaitEvent(c->stream, c->ev_join[i], 0), "join wait");
    }
}

void release_lanes(rrsvd_b200_ctx* c) {
    for (int i = 0; i < rrsvd_b200_ctx::kMaxLanes; ++i) {
        if (c->lane[i]) cudaStreamDestroy(c->lane[i]);
        if (c->ev_join[i]) cudaEventDestroy(c->ev_join[i]);
        c->lane[i] = nullptr;
        c->ev_join[i] = nullptr;
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    c->ev_fork = nullptr;
}

void recover_after_failure(rrsvd_b200_ctx* c) {
    if (c->home != nullptr) c->stream = c->home;
    for (cudaStream_t l : c->lane)
        if (l) cudaStreamSynchronize(l);
    cudaStreamSynchronize(c->stream);
    for (auto& p : c->pending) {  // timing events of launches that may never have run
        c->event_pool.push_back(p.a);
        c->event_pool.push_back(p.b);
    }
    c->pending.clear();
    cudaGetLastError();
}

cudaEvent_t pooled_event(rrsvd_b200_ctx* c) {
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    check_cuda(c, cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

void flush_gemm_timing(rrsvd_b200_ctx* c) {
    for (auto& p : c->pending) {
        check_cuda(c, cudaEventSynchronize(p.b), "event sync");
        float ms = 0.f;
        check_cuda(c, cudaEventElapsedTime(&ms, p.a, p.b), "event elapsed");
        c->event_pool.push_back(p.a);
        c->event_pool.push_back(p.b);
        if (p.kind == 2) {
            c->oz_gemm_ms += ms;
            c->oz_gemm_bytes += p.bytes;
            continue;
        }
        if (p.kind == 1) {
            if (p.flops > 0) {
                c->oz_ms += ms;
                c->oz_flops += p.flops;
                c->oz_bytes += p.bytes;
                c->oz_calls++;
            } else {
                c->oz_prep_ms += ms;
                c->oz_prep_bytes += p.bytes;
            }
            continue;
        }
        c->gemm_ms += ms;
        c->gemm_flops += p.flops;
        c->gemm_exec_flops += p.executed;
        if (p.tma) c->gemm_tma_ms += ms;
        c->tag_ms[p.tag & 7] += ms;
        c->tag_flops[p.tag & 7] += p.flops;
        c->gemm_calls++;
    }
    c->pending.clear();
}

void* pinned_sweep_scratch(rrsvd_b200_ctx* c, size_t bytes) {
    if (bytes > c->pinned_sweep_cap) {
        if (c->pinned_sweep) cudaFreeHost(c->pinned_sweep);
        c->pinned_sweep = nullptr;
        c->pinned_sweep_cap = 0;
        check_cuda(c, cudaMallocHost(&c->pinned_sweep, bytes), "cudaMallocHost");
        c->pinned_sweep_cap = bytes;
    }
    return c->pinned_sweep;
}

void* pinned_scratch(rrsvd_b200_ctx* c, size_t bytes) {
    if (bytes > c->pinned_cap) {
        if (c->pinned) cudaFreeHost(c->pinned);
        c->pinned = nullptr;
        c->pinned_cap = 0;
        check_cuda(c, cudaMallocHost(&c->pinned, bytes), "cudaMallocHost");
        c->pinned_cap = bytes;
    }
    return c->pinned;
}

}  // namespace rb

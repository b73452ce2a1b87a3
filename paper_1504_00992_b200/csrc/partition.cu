// partition.cu — the chain-block partition behind the C ABI: one process (or
// host thread) per GPU owns a contiguous block of sites; same-parity bonds update locally and only
// boundary Γ/λ cross ranks, by point-to-point messages on the library stream — NCCL send/recv
// over NVLink between GPUs (libnccl loaded at run time), or a host-staged loopback between host
// threads (the protocol check on one GPU).  The protocol is parallel.py's, without its shape
// round trip: every message has a fixed capacity derived from chi_max and the site dimension,
// known to both sides, and carries its dims in a small header in the same group.
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>  // types and enums only: the functions come from dlopen("libnccl.so.2")

#include "mps.cuh"

using namespace rb;

namespace {

// ---- transports ------------------------------------------------------------------------------
struct Transport {
    virtual ~Transport() = default;
    virtual void group_start(rrsvd_b200_ctx* c) = 0;
    virtual void group_end(rrsvd_b200_ctx* c) = 0;
    // device buffers, enqueued on c->stream (NCCL) or executed on it (loopback)
    virtual void send(rrsvd_b200_ctx* c, const void* buf, size_t bytes, int peer) = 0;
    virtual void recv(rrsvd_b200_ctx* c, void* buf, size_t bytes, int peer) = 0;
    // this rank's call failed: peers blocked on its messages must not wait forever
    virtual void abort() {}
};

struct NcclLib {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclLib* nccl() {
    static NcclLib lib = [] {
        NcclLib L;
        // (a process that already loaded NCCL — torch — gets that library back by its soname)
        L.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (L.h == nullptr) return L;
        auto sym = [&](const char* n) { return dlsym(L.h, n); };
        L.GetUniqueId = reinterpret_cast<decltype(L.GetUniqueId)>(sym("ncclGetUniqueId"));
        L.CommInitRank = reinterpret_cast<decltype(L.CommInitRank)>(sym("ncclCommInitRank"));
        L.CommDestroy = reinterpret_cast<decltype(L.CommDestroy)>(sym("ncclCommDestroy"));
        L.Send = reinterpret_cast<decltype(L.Send)>(sym("ncclSend"));
        L.Recv = reinterpret_cast<decltype(L.Recv)>(sym("ncclRecv"));
        L.GroupStart = reinterpret_cast<decltype(L.GroupStart)>(sym("ncclGroupStart"));
        L.GroupEnd = reinterpret_cast<decltype(L.GroupEnd)>(sym("ncclGroupEnd"));
        L.GetErrorString = reinterpret_cast<decltype(L.GetErrorString)>(sym("ncclGetErrorString"));
        return L;
    }();
    const bool ok = lib.GetUniqueId && lib.CommInitRank && lib.CommDestroy && lib.Send && lib.Recv &&
                    lib.GroupStart && lib.GroupEnd && lib.GetErrorString;
    return ok ? &lib : nullptr;
}

void check_nccl(rrsvd_b200_ctx* c, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    c->err = std::string(what) + ": " + nccl()->GetErrorString(r);
    throw Fail{kCuda};
}

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm) nccl()->CommDestroy(comm);
    }
    void group_start(rrsvd_b200_ctx* c) override { check_nccl(c, nccl()->GroupStart(), "ncclGroupStart"); }
    void group_end(rrsvd_b200_ctx* c) override { check_nccl(c, nccl()->GroupEnd(), "ncclGroupEnd"); }
    void send(rrsvd_b200_ctx* c, const void* buf, size_t bytes, int peer) override {
        check_nccl(c, nccl()->Send(buf, bytes, ncclUint8, peer, comm, c->stream), "ncclSend");
    }
    void recv(rrsvd_b200_ctx* c, void* buf, size_t bytes, int peer) override {
        check_nccl(c, nccl()->Recv(buf, bytes, ncclUint8, peer, comm, c->stream), "ncclRecv");
    }
};

}  // namespace

// Host-staged mailboxes between ranks driven by host threads of one process.
struct rrsvd_b200_loopback_hub {
    int nranks = 0;
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::pair<int, int>, std::deque<std::vector<char>>> box;  // (src, dst) -> messages
    bool failed = false;  // some rank's call failed: waiting receives throw instead of hanging
};

namespace {

struct LoopbackTransport : Transport {
    rrsvd_b200_loopback_hub* hub = nullptr;
    int rank = 0;
    // sends of a group are staged to the host at once (so a group never waits on its peer's
    // receives); receives wait for the message and copy it up
    void group_start(rrsvd_b200_ctx*) override {}
    void group_end(rrsvd_b200_ctx*) override {}
    void send(rrsvd_b200_ctx* c, const void* buf, size_t bytes, int peer) override {
        std::vector<char> msg(bytes);
        check_cuda(c, cudaMemcpyAsync(msg.data(), buf, bytes, cudaMemcpyDeviceToHost, c->stream), "loopback D2H");
        check_cuda(c, cudaStreamSynchronize(c->stream), "loopback sync");
        std::lock_guard<std::mutex> lk(hub->mu);
        hub->box[{rank, peer}].push_back(std::move(msg));
        hub->cv.notify_all();
    }
    void recv(rrsvd_b200_ctx* c, void* buf, size_t bytes, int peer) override {
        std::vector<char> msg;
        {
            std::unique_lock<std::mutex> lk(hub->mu);
            auto& q = hub->box[{peer, rank}];
            hub->cv.wait(lk, [&] { return !q.empty() || hub->failed; });
            if (q.empty()) throw_numeric(c, "loopback: a peer rank failed");
            msg = std::move(q.front());
            q.pop_front();
        }
        if (msg.size() != bytes) throw_contract(c, "loopback: message size mismatch");
        check_cuda(c, cudaMemcpyAsync(buf, msg.data(), bytes, cudaMemcpyHostToDevice, c->stream), "loopback H2D");
        check_cuda(c, cudaStreamSynchronize(c->stream), "loopback sync");
    }
    void abort() override {
        std::lock_guard<std::mutex> lk(hub->mu);
        hub->failed = true;
        hub->cv.notify_all();
    }
};

}  // namespace

struct rrsvd_b200_comm {
    rrsvd_b200_ctx* c = nullptr;
    int nranks = 1, rank = 0;
    std::unique_ptr<Transport> t;
};

namespace {

template <class F>
int comm_api(rrsvd_b200_ctx* c, F&& f) {
    if (c == nullptr) return kContract;
    int code = kOk;
    try {
        cudaSetDevice(c->device);
        f();
    } catch (const Fail& e) {
        code = e.code;
    } catch (const std::exception& e) {
        c->err = e.what();
        code = kCuda;
    }
    if (code != kOk) recover_after_failure(c);
    ws_reset(c);
    return code;
}

// Copy `bytes` device->device into an MPS buffer grown as needed (stream-ordered).
void put_gamma(rrsvd_b200_mps* s, int site, int dl, int dr, const cplx* src) {
    rrsvd_b200_ctx* c = s->c;
    const size_t elems = (size_t)dl * s->d[site] * dr;
    if (s->gcap[site] < elems) {
        if (s->g[site]) cudaFreeAsync(s->g[site], c->stream);
        s->g[site] = nullptr;
        check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&s->g[site]), elems * sizeof(cplx), c->stream), "alloc gamma");
        s->gcap[site] = elems;
    }
    check_cuda(c, cudaMemcpyAsync(s->g[site], src, elems * sizeof(cplx), cudaMemcpyDeviceToDevice, c->stream), "put gamma");
    s->dl[site] = dl;
    s->dr[site] = dr;
    if (site > 0) s->dr[site - 1] = dl;  // (the ghost's left bond is my boundary bond)
}

void put_edge(rrsvd_b200_mps* s, int e, const double* src, size_t n) {
    rrsvd_b200_ctx* c = s->c;
    if (s->edge_cap[e] < n) {
        if (s->edge[e]) cudaFreeAsync(s->edge[e], c->stream);
        check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&s->edge[e]), std::max<size_t>(n, 1) * sizeof(double),
                                      c->stream), "alloc edge");
        s->edge_cap[e] = n;
    }
    check_cuda(c, cudaMemcpyAsync(s->edge[e], src, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "put edge");
    s->edge_n[e] = n;
}

// Message buffers of one rank: fixed capacities so sender and receiver agree without a shape
// round trip.  Header = {dl, d, dr} (int64) of a Γ, {n} of a λ.
struct Msg {
    long long hdr[4];
    cplx* g = nullptr;
    double* l = nullptr;
};

}  // namespace

extern "C" {

int rrsvd_b200_comm_unique_id(void* id_out) {
    if (id_out == nullptr) return kContract;
    const NcclLib* L = nccl();
    if (L == nullptr) return kCuda;
    ncclUniqueId id;
    if (L->GetUniqueId(&id) != ncclSuccess) return kCuda;
    std::memcpy(id_out, &id, sizeof(id));
    return kOk;
}

int rrsvd_b200_comm_create_nccl(rrsvd_b200_ctx* c, int nranks, int rank, const void* id, rrsvd_b200_comm** out) {
    if (out == nullptr) return kContract;
    *out = nullptr;
    return comm_api(c, [&] {
        if (nranks < 1 || rank < 0 || rank >= nranks || id == nullptr) throw_contract(c, "comm: bad rank / id");
        if (nccl() == nullptr) {
            c->err = "comm: libnccl.so.2 not loadable";
            throw Fail{kCuda};
        }
        auto t = std::make_unique<NcclTransport>();
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        check_nccl(c, nccl()->CommInitRank(&t->comm, nranks, uid, rank), "ncclCommInitRank");
        auto* cm = new rrsvd_b200_comm();
        cm->c = c;
        cm->nranks = nranks;
        cm->rank = rank;
        cm->t = std::move(t);
        *out = cm;
    });
}

int rrsvd_b200_loopback_hub_create(int nranks, rrsvd_b200_loopback_hub** out) {
    if (out == nullptr || nranks < 1) return kContract;
    *out = new rrsvd_b200_loopback_hub();
    (*out)->nranks = nranks;
    return kOk;
}

void rrsvd_b200_loopback_hub_destroy(rrsvd_b200_loopback_hub* hub) { delete hub; }

int rrsvd_b200_comm_create_loopback(rrsvd_b200_ctx* c, rrsvd_b200_loopback_hub* hub, int rank,
                                    rrsvd_b200_comm** out) {
    if (out == nullptr) return kContract;
    *out = nullptr;
    return comm_api(c, [&] {
        if (hub == nullptr || rank < 0 || rank >= hub->nranks) throw_contract(c, "comm: bad loopback rank");
        auto t = std::make_unique<LoopbackTransport>();
        t->hub = hub;
        t->rank = rank;
        auto* cm = new rrsvd_b200_comm();
        cm->c = c;
        cm->nranks = hub->nranks;
        cm->rank = rank;
        cm->t = std::move(t);
        *out = cm;
    });
}

void rrsvd_b200_comm_destroy(rrsvd_b200_comm* cm) {
    if (cm && cm->c) cudaSetDevice(cm->c->device);
    delete cm;
}

// evolve (tebd.cpp:260-326) of one rank's chain block.  See include/rrsvd_b200.h.
int rrsvd_b200_evolve_partitioned(rrsvd_b200_mps* s, rrsvd_b200_comm* cm, size_t first_site, size_t n_global,
                                  size_t n_sweeps, const rrsvd_b200_sweep* sweeps,
                                  const rrsvd_b200_gate* const* gates, const unsigned char* term_bonds, size_t n_steps,
                                  uint64_t step0, rrsvd_b200_backend* be, const rrsvd_b200_evolve_options* opt,
                                  rrsvd_b200_evolve_diag* diag) {
    if (s == nullptr || cm == nullptr) return kContract;
    rrsvd_b200_ctx* c = s->c;
    const int code = comm_api(c, [&] {
        if (cm->c != c) throw_contract(c, "evolve_partitioned: comm and MPS on different contexts");
        if (be == nullptr || diag == nullptr || term_bonds == nullptr || (n_sweeps && (sweeps == nullptr || gates == nullptr)))
            throw_contract(c, "evolve_partitioned: null argument");
        if (s->chi_max == 0) throw_contract(c, "evolve_partitioned: needs chi_max > 0 (message capacities)");
        const int r = cm->rank, w = cm->nranks;
        const int nloc = s->n, nb = nloc - 1;
        const bool ghost = r + 1 < w;
        const long long a = (long long)first_site;
        const long long b = a + nloc - (ghost ? 1 : 0);  // one past the last owned site
        if (b > (long long)n_global || (!ghost && b != (long long)n_global))
            throw_contract(c, "evolve_partitioned: block does not fit the global chain");
        const size_t X = s->chi_max;
        auto gcap = [&](int local_site) { return X * (size_t)s->d[local_site] * X; };
        // message buffers (device; owned here — evolve_core releases the call workspace per sweep)
        struct Owned {
            rrsvd_b200_ctx* c;
            std::vector<void*> p;
            void* get(size_t bytes) {
                void* q = nullptr;
                check_cuda(c, cudaMallocAsync(&q, std::max<size_t>(bytes, 16), c->stream), "alloc message");
                p.push_back(q);
                return q;
            }
            ~Owned() {
                for (void* q : p) cudaFreeAsync(q, c->stream);
            }
        } own{c, {}};
        const size_t gmax = std::max(gcap(0), gcap(nloc - 1));
        Msg out_g{}, out_l{}, out_r{}, in_g{}, in_l{}, in_el{};
        out_g.g = static_cast<cplx*>(own.get(gmax * sizeof(cplx)));
        in_g.g = static_cast<cplx*>(own.get(gmax * sizeof(cplx)));
        out_l.l = static_cast<double*>(own.get(X * sizeof(double)));
        out_r.l = static_cast<double*>(own.get(X * sizeof(double)));
        in_l.l = static_cast<double*>(own.get(X * sizeof(double)));
        in_el.l = static_cast<double*>(own.get(X * sizeof(double)));
        auto* hdr = static_cast<long long*>(own.get(5 * 4 * sizeof(long long)));  // out Γ, out λ, out edge, in Γ, in λ / edge
        long long hh[5 * 4];
        // global call index of global bond j in sweep sw of step t (parallel.py _global_index,
        // tebd.cpp:162,289-294): term bonds only, ascending within a sweep
        std::vector<long long> per_sweep(n_sweeps, 0);
        for (size_t sw = 0; sw < n_sweeps; ++sw)
            for (size_t j = 0; j + 1 < n_global; ++j) per_sweep[sw] += term_bonds[j] && (int)(j % 2) == sweeps[sw].bond_parity;
        long long per_step = 0;
        for (long long v : per_sweep) per_step += v;
        auto global_index = [&](uint64_t t, size_t sw, long long j) {
            long long idx = (long long)t * per_step;
            for (size_t k = 0; k < sw; ++k) idx += per_sweep[k];
            for (long long jj = 0; jj < j; ++jj) idx += term_bonds[jj] && (int)(jj % 2) == sweeps[sw].bond_parity;
            return idx;
        };
        const uint64_t base_seed = be->seed;
        Transport& T = *cm->t;

        auto refresh = [&] {  // step 1: ghost Γ + right edge from r+1, left edge from r-1
            hh[0] = s->dl[0]; hh[1] = s->d[0]; hh[2] = s->dr[0];
            hh[4] = nloc > 1 ? s->dr[0] : 0;                 // my λ_local[0] -> r-1's right edge
            hh[8] = nloc > 1 ? s->dr[nb - 1] : 0;            // my boundary λ (local bond nb-1) -> r+1's left edge
            check_cuda(c, cudaMemcpyAsync(hdr, hh, 12 * sizeof(long long), cudaMemcpyHostToDevice, c->stream), "hdr");
            if (r > 0) {
                check_cuda(c, cudaMemcpyAsync(out_g.g, s->g[0], (size_t)s->dl[0] * s->d[0] * s->dr[0] * sizeof(cplx),
                                              cudaMemcpyDeviceToDevice, c->stream), "stage");
                if (nloc > 1)
                    check_cuda(c, cudaMemcpyAsync(out_l.l, s->lam[0], (size_t)s->dr[0] * sizeof(double),
                                                  cudaMemcpyDeviceToDevice, c->stream), "stage");
            }
            T.group_start(c);
            if (r > 0) {
                T.send(c, hdr, 3 * sizeof(long long), r - 1);
                T.send(c, out_g.g, gcap(0) * sizeof(cplx), r - 1);  // (capacity: X d X of site 0)
                T.send(c, hdr + 4, sizeof(long long), r - 1);
                T.send(c, out_l.l, X * sizeof(double), r - 1);
            }
            if (ghost)
                check_cuda(c, cudaMemcpyAsync(out_r.l, s->lam[nb - 1], (size_t)s->dr[nb - 1] * sizeof(double),
                                              cudaMemcpyDeviceToDevice, c->stream), "stage");
            if (ghost) {
                T.send(c, hdr + 8, sizeof(long long), r + 1);
                T.send(c, out_r.l, X * sizeof(double), r + 1);
                T.recv(c, hdr + 12, 3 * sizeof(long long), r + 1);
                T.recv(c, in_g.g, gcap(nloc - 1) * sizeof(cplx), r + 1);
                T.recv(c, hdr + 16, sizeof(long long), r + 1);
                T.recv(c, in_l.l, X * sizeof(double), r + 1);
            }
            if (r > 0) {
                T.recv(c, hdr + 18, sizeof(long long), r - 1);
                T.recv(c, in_el.l, X * sizeof(double), r - 1);
            }
            T.group_end(c);
            check_cuda(c, cudaMemcpyAsync(hh, hdr, 20 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream), "hdr");
            check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
            if (ghost) {
                put_gamma(s, nloc - 1, (int)hh[12], (int)hh[14], in_g.g);
                put_edge(s, 1, in_l.l, (size_t)hh[16]);
            }
            if (r > 0) put_edge(s, 0, in_el.l, (size_t)hh[18]);
        };
        auto boundary_return = [&](int parity) {  // step 3: the updated ghost Γ back to its owner
            const bool i_send = ghost && ((b - 1) % 2) == parity && term_bonds[b - 1];
            const bool i_recv = r > 0 && ((a - 1) % 2) == parity && term_bonds[a - 1];
            if (!i_send && !i_recv) return;
            if (i_send) {
                hh[0] = s->dl[nloc - 1]; hh[1] = s->d[nloc - 1]; hh[2] = s->dr[nloc - 1];
                check_cuda(c, cudaMemcpyAsync(hdr, hh, 3 * sizeof(long long), cudaMemcpyHostToDevice, c->stream), "hdr");
                check_cuda(c, cudaMemcpyAsync(out_g.g, s->g[nloc - 1],
                                              (size_t)hh[0] * hh[1] * hh[2] * sizeof(cplx), cudaMemcpyDeviceToDevice,
                                              c->stream), "stage");
            }
            T.group_start(c);
            if (i_send) {
                T.send(c, hdr, 3 * sizeof(long long), r + 1);
                T.send(c, out_g.g, gcap(nloc - 1) * sizeof(cplx), r + 1);
            }
            if (i_recv) {
                T.recv(c, hdr + 12, 3 * sizeof(long long), r - 1);
                T.recv(c, in_g.g, gcap(0) * sizeof(cplx), r - 1);
            }
            T.group_end(c);
            if (i_recv) {
                check_cuda(c, cudaMemcpyAsync(hh + 12, hdr + 12, 3 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream),
                           "hdr");
                check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
                const int dl = (int)hh[12], dr = (int)hh[14];
                // my site 0: its left bond is the neighbour's boundary bond (dims from the header)
                const size_t elems = (size_t)dl * s->d[0] * dr;
                if (s->gcap[0] < elems) {
                    if (s->g[0]) cudaFreeAsync(s->g[0], c->stream);
                    check_cuda(c, cudaMallocAsync(reinterpret_cast<void**>(&s->g[0]), elems * sizeof(cplx), c->stream),
                               "alloc gamma");
                    s->gcap[0] = elems;
                }
                check_cuda(c, cudaMemcpyAsync(s->g[0], in_g.g, elems * sizeof(cplx), cudaMemcpyDeviceToDevice, c->stream),
                           "put gamma");
                s->dl[0] = dl;
                s->dr[0] = dr;
            }
        };

        diag->kept_fraction = 1.0;
        diag->aborted = 0;
        diag->abort_step = 0;
        diag->n_updates = 0;
        diag->max_bond_dim = 1;
        std::vector<const rrsvd_b200_gate*> one(nb);
        for (size_t t = 0; t < n_steps; ++t)
            for (size_t sw = 0; sw < n_sweeps; ++sw) {
                refresh();
                const int parity = sweeps[sw].bond_parity;
                // my bonds of this parity: global a .. b-1 (with a ghost) or a .. b-2
                long long first = -1;
                for (int lb = 0; lb < nb; ++lb) {
                    const long long gb = a + lb;
                    const bool mine = (gb % 2) == parity && term_bonds[gb] && gates[sw * nb + lb] != nullptr;
                    one[lb] = mine ? gates[sw * nb + lb] : nullptr;
                    if (mine && first < 0) first = gb;
                }
                if (first >= 0) {
                    // the local sweep: local bond lb has parity (a + lb) % 2 == parity
                    const rrsvd_b200_sweep local{(int)((parity - a % 2 + 2) % 2), sweeps[sw].coefficient};
                    rrsvd_b200_backend lbe = *be;
                    lbe.seed = base_seed + (uint64_t)global_index(step0 + t, sw, first);
                    rrsvd_b200_evolve_diag d{};
                    evolve_core(s, c, 1, &local, one.data(), 1, &lbe, opt, &d, nullptr, 0);
                    diag->kept_fraction *= d.kept_fraction;
                    diag->max_bond_dim = std::max(diag->max_bond_dim, d.max_bond_dim);
                    diag->n_updates += d.n_updates;
                    if (d.aborted) throw_contract(c, "evolve_partitioned: the discarded-weight budget is per rank; "
                                                     "use abort_discarded_threshold = 1");
                }
                boundary_return(parity);
            }
        refresh();  // ghosts and edges current for observables
        be->seed = base_seed + (uint64_t)((n_steps)*per_step);
    });
    if (code != kOk && cm->t) cm->t->abort();  // (peers' receives fail instead of waiting)
    return code;
}

}  // extern "C"

// capi.cu — the extern "C" drop-in boundary (include/rrsvd_b200.h).
#include <algorithm>
#include <memory>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rrsvd_b200.h"
#include "ozaki.cuh"
#include "pipeline.cuh"

using namespace rb;

namespace {

template <class F>
int api(rrsvd_b200_ctx* c, F&& f) {
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

struct Scalars {  // host mirror of device scalars read back at the end of a call
    int kept;
    int nonfinite;
    int pinv;
    int pad;
    double total_sq;
    double discarded;
};

void read_scalars(rrsvd_b200_ctx* c, Scalars* dev, Scalars* host) {
    check_cuda(c, cudaMemcpyAsync(host, dev, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream), "D2H scalars");
    check_cuda(c, cudaStreamSynchronize(c->stream), "stream sync");
}

// Copy `bytes` from device buffer src to user pointer dst (device or host), row-pitched.
void copy_out2d(rrsvd_b200_ctx* c, void* dst, size_t dpitch, const void* src, size_t spitch,
                size_t width, size_t height) {
    if (dst == nullptr || width == 0 || height == 0) return;
    check_cuda(c, cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault, c->stream),
               "copy out");
}

void copy_out(rrsvd_b200_ctx* c, void* dst, const void* src, size_t bytes) {
    if (dst == nullptr || bytes == 0) return;
    check_cuda(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream), "copy out");
}

// Householder QR returns an orthonormal Q even for rank-deficient input (linalg.hpp:35-37,
// tested at test_linalg.cpp:152-159); CholeskyQR leaves the dependent columns of Q at exactly
// zero.  Fill them with an orthonormal basis of a random subspace orthogonal to the live
// columns: E (m x nd, Philox) <- E - Q (Q^H E) twice, then E <- orth(E), scattered into the
// dead column slots.  R = Q^H A afterwards has (numerically) zero rows there, and Q R = A still
// holds because A lies in the span of the live columns.
void complete_basis(rrsvd_b200_ctx* c, cplx* Q, int m, int n) {
    double* nrm = ws_get<double>(c, (size_t)n);
    check_cuda(c, column_norms2(Q, m, n, nrm, c->stream), "column_norms2");
    c->launches++;
    std::vector<double> diag(n);
    check_cuda(c, cudaMemcpyAsync(diag.data(), nrm, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
               "D2H norms");
    check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
    std::vector<int> dead;
    for (int j = 0; j < n; ++j)
        if (!(diag[j] > 0.5)) dead.push_back(j);
    const int nd = (int)dead.size();
    if (nd == 0) return;
    cplx* E = ws_get<cplx>(c, (size_t)m * nd);
    cplx* P = ws_get<cplx>(c, (size_t)n * nd);
    cplx* F = ws_get<cplx>(c, (size_t)m * nd);
    make_omega(c, m, nd, 0x51a7e5eedull, RRSVD_B200_OMEGA_PHILOX, E);
    for (int pass = 0; pass < 2; ++pass) {
        gemm(c, kOpC, n, nd, m, Q, n, E, nd, P, nd);  // P = Q^H E
        GemmSpec up{m, nd, n, Q, n, P, nd, E, nd};    // E = E - Q P
        up.D = E;
        up.ldd = nd;
        up.alpha = -1.0;
        gemm_many(c, kOpN, {up});
    }
    orth(c, E, m, nd, F);
    for (int t = 0; t < nd; ++t)
        check_cuda(c, cudaMemcpy2DAsync(Q + dead[t], (size_t)n * sizeof(cplx), F + t, (size_t)nd * sizeof(cplx),
                                        sizeof(cplx), m, cudaMemcpyDeviceToDevice, c->stream), "scatter");
}

}  // namespace

extern "C" {

const char* rrsvd_b200_version(void) { return "rrsvd_b200 0.1 (sm_100a, FP64 DMMA)"; }

int rrsvd_b200_ctx_create(int device, void* stream, rrsvd_b200_ctx** out) {
    if (out == nullptr) return kContract;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0 || device < 0 || device >= n) {
        cudaGetLastError();
        return kCuda;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) return kCuda;
    auto* c = new rrsvd_b200_ctx();
    c->device = device;
    cudaSetDevice(device);
    if (stream != nullptr) {
        c->stream = static_cast<cudaStream_t>(stream);
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete c;
            return kCuda;
        }
        c->own_stream = true;
    }
    c->home = c->stream;
    // keep workspace allocations cached in the stream-ordered pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
    return kOk;
}

void rrsvd_b200_ctx_destroy(rrsvd_b200_ctx* c) {
    if (c == nullptr) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    release_staged(c);
    cudaStreamSynchronize(c->stream);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->pinned_sweep) cudaFreeHost(c->pinned_sweep);
    release_lanes(c);
    for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* rrsvd_b200_last_error(const rrsvd_b200_ctx* c) { return c ? c->err.c_str() : "null context"; }

int rrsvd_b200_set_stream(rrsvd_b200_ctx* c, void* stream) {
    return api(c, [&] {
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
        if (c->own_stream) cudaStreamDestroy(c->stream);
        c->own_stream = false;
        c->stream = c->home = static_cast<cudaStream_t>(stream);
    });
}

int rrsvd_b200_synchronize(rrsvd_b200_ctx* c) {
    return api(c, [&] { check_cuda(c, cudaStreamSynchronize(c->stream), "sync"); });
}

uint64_t rrsvd_b200_launch_count(const rrsvd_b200_ctx* c) { return c ? c->launches : 0; }

// ------------------------------------------------------------------------------------------ L1

int rrsvd_b200_zgemm(rrsvd_b200_ctx* c, int op_a, int op_b, size_t m, size_t n, size_t k,
                     const double* A, size_t lda, const double* B, size_t ldb, double* C, size_t ldc) {
    return api(c, [&] {
        if (op_a != RRSVD_B200_OP_N && op_a != RRSVD_B200_OP_C) throw_contract(c, "zgemm: bad op_a");
        if (op_b != RRSVD_B200_OP_N && op_b != RRSVD_B200_OP_C) throw_contract(c, "zgemm: bad op_b");
        if (m == 0 || n == 0) return;
        const size_t a_rows = op_a == RRSVD_B200_OP_N ? m : k;
        std::vector<OutBuf> outs;
        const auto* dA = static_cast<const cplx*>(stage_in(c, A, a_rows * lda * sizeof(cplx)));
        const cplx* dB;
        if (op_b == RRSVD_B200_OP_N) {
            dB = static_cast<const cplx*>(stage_in(c, B, k * ldb * sizeof(cplx)));
        } else if (k > 0) {
            // op_b = C (B is n x k): one conjugate-transpose pass into a k x n workspace, then
            // the N kernel — adj_b is a boundary convenience (linalg.cpp:20-35), never on the
            // decimation path.
            auto* packed = ws_get<cplx>(c, n * k);
            check_cuda(c, cudaMemcpy2DAsync(packed, k * sizeof(cplx), B, ldb * sizeof(cplx), k * sizeof(cplx), n,
                                            cudaMemcpyDefault, c->stream), "stage B");
            auto* bt = ws_get<cplx>(c, k * n);
            check_cuda(c, conj_transpose(packed, (int)n, (int)k, bt, c->stream), "conj_transpose");
            c->launches++;
            dB = bt;
            ldb = n;
        } else {
            dB = nullptr;
        }
        auto* dC = static_cast<cplx*>(stage_out(c, C, m * ldc * sizeof(cplx), outs));
        if (k == 0) {
            check_cuda(c, cudaMemsetAsync(dC, 0, m * ldc * sizeof(cplx), c->stream), "memset");
        } else {
            gemm(c, op_a == RRSVD_B200_OP_N ? kOpN : kOpC, (int)m, (int)n, (int)k, dA, (long long)lda, dB,
                 (long long)ldb, dC, (long long)ldc);
        }
        finish_out(c, outs);
    });
}

int rrsvd_b200_ozaki_zgemm(rrsvd_b200_ctx* c, int op_a, size_t m, size_t n, size_t k, const double* A, size_t lda,
                           const double* B, size_t ldb, double* C, size_t ldc, int moduli) {
    return api(c, [&] {
        if (op_a != RRSVD_B200_OP_N && op_a != RRSVD_B200_OP_C) throw_contract(c, "ozaki_zgemm: bad op_a");
        if (moduli < 8 || moduli > kOzMaxMod) throw_contract(c, "ozaki_zgemm: moduli must be in [8, 16]");
        if (m == 0 || n == 0) return;
        if (m < 128 || k < 16 || std::max(m, k) > 32768)
            throw_contract(c, "ozaki_zgemm: needs m >= 128, k >= 16 and m, k <= 32768");
        const bool opn = op_a == RRSVD_B200_OP_N;
        const size_t a_rows = opn ? m : k, a_cols = opn ? k : m;
        if (lda < a_cols || ldb < n || ldc < n) throw_contract(c, "ozaki_zgemm: leading dimension too small");
        std::vector<OutBuf> outs;
        const auto* dA = static_cast<const cplx*>(stage_in(c, A, a_rows * lda * sizeof(cplx)));
        const auto* dB = static_cast<const cplx*>(stage_in(c, B, k * ldb * sizeof(cplx)));
        auto* dC = static_cast<cplx*>(stage_out(c, C, m * ldc * sizeof(cplx), outs));
        std::vector<OzakiA> oa = ozaki_prepare_many(c, {OzSrc{dA, (int)a_rows, (int)a_cols, (long long)lda}}, moduli);
        ozaki_product_many(c, opn ? kOpN : kOpC, {OzProduct{&oa[0], dB, (long long)ldb, (int)n, dC, (long long)ldc}});
        finish_out(c, outs);
    });
}

// A prepared once for many emulated products (the row-sharded RRSVD's shards).
struct rrsvd_b200_ozaki_a {
    rb::OzakiA a;
    std::vector<void*> bufs;
    int device;
    cudaStream_t stream;
};

int rrsvd_b200_ozaki_usable(size_t m, size_t n) {
    return m <= 32768 && n <= 32768 && ozaki_usable((int)m, (int)n, 1) ? ozaki_moduli() : 0;
}

int rrsvd_b200_ozaki_prepare(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, size_t lda, int moduli,
                             rrsvd_b200_ozaki_a** out) {
    return api(c, [&] {
        if (out == nullptr) throw_contract(c, "ozaki_prepare: null output");
        *out = nullptr;
        if (moduli < 8 || moduli > kOzMaxMod) throw_contract(c, "ozaki_prepare: moduli must be in [8, 16]");
        if (m < 128 || n < 128 || m > 32768 || n > 32768) throw_contract(c, "ozaki_prepare: needs m, n in [128, 32768]");
        if (lda < n) throw_contract(c, "ozaki_prepare: leading dimension too small");
        const auto* dA = static_cast<const cplx*>(stage_in(c, A, m * lda * sizeof(cplx)));
        auto h = std::make_unique<rrsvd_b200_ozaki_a>();
        h->device = c->device;
        h->stream = c->stream;
        std::vector<OzakiA> oa;
        try {
            oa = ozaki_prepare_many(c, {OzSrc{dA, (int)m, (int)n, (long long)lda}}, moduli, &h->bufs);
        } catch (...) {
            for (void* p : h->bufs) cudaFreeAsync(p, c->stream);
            throw;
        }
        h->a = oa[0];
        *out = h.release();
    });
}

int rrsvd_b200_ozaki_apply(rrsvd_b200_ctx* c, const rrsvd_b200_ozaki_a* h, int op_a, const double* X, size_t l,
                           size_t ldx, double* C, size_t ldc, int accumulate) {
    return api(c, [&] {
        if (h == nullptr) throw_contract(c, "ozaki_apply: null operator");
        if (op_a != RRSVD_B200_OP_N && op_a != RRSVD_B200_OP_C) throw_contract(c, "ozaki_apply: bad op_a");
        if (l == 0) return;
        const bool opn = op_a == RRSVD_B200_OP_N;
        const size_t k = opn ? h->a.n : h->a.m, rows = opn ? h->a.m : h->a.n;
        if (ldx < l || ldc < l) throw_contract(c, "ozaki_apply: leading dimension too small");
        std::vector<OutBuf> outs;
        const auto* dX = static_cast<const cplx*>(stage_in(c, X, k * ldx * sizeof(cplx)));
        if (accumulate && !is_device_ptr(C)) throw_contract(c, "ozaki_apply: accumulate needs a device C");
        auto* dC = static_cast<cplx*>(stage_out(c, C, rows * ldc * sizeof(cplx), outs));
        ozaki_product_many(c, opn ? kOpN : kOpC,
                           {OzProduct{&h->a, dX, (long long)ldx, (int)l, dC, (long long)ldc, accumulate ? 1 : 0}});
        finish_out(c, outs);
    });
}

void rrsvd_b200_ozaki_release(rrsvd_b200_ozaki_a* h) {
    if (h == nullptr) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(h->device);
    for (void* p : h->bufs) cudaFreeAsync(p, h->stream);
    cudaStreamSynchronize(h->stream);
    cudaSetDevice(prev);
    delete h;
}

int rrsvd_b200_frobenius_norm(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, double* out) {
    return api(c, [&] {
        if (out == nullptr) throw_contract(c, "frobenius_norm: null output");
        const size_t cnt = m * n;
        if (cnt == 0) { *out = 0.0; return; }
        const auto* dA = static_cast<const cplx*>(stage_in(c, A, cnt * sizeof(cplx)));
        double* part = ws_get<double>(c, 2 * kNumSMs);
        int* bad = ws_get<int>(c, 2 * kNumSMs);
        auto* sc = ws_get<Scalars>(c, 1);
        check_cuda(c, sumsq(dA, (long long)cnt, part, bad, &sc->total_sq, &sc->nonfinite, c->stream), "sumsq");
        c->launches += 2;
        Scalars h;
        read_scalars(c, sc, &h);
        *out = std::sqrt(h.total_sq);
    });
}

int rrsvd_b200_qr(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, double* Q, double* R) {
    return api(c, [&] {
        if (m < n) throw_contract(c, "qr: requires rows >= cols");
        if (n == 0) return;
        std::vector<OutBuf> outs;
        const auto* dA = static_cast<const cplx*>(stage_in(c, A, m * n * sizeof(cplx)));
        auto* dQ = static_cast<cplx*>(stage_out(c, Q, m * n * sizeof(cplx), outs));
        if (dQ == nullptr) dQ = ws_get<cplx>(c, m * n);
        int* dn = ws_get<int>(c, 1);
        orth(c, dA, (int)m, (int)n, dQ, dn);
        int ndead = 0;
        check_cuda(c, cudaMemcpyAsync(&ndead, dn, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
        if (ndead > 0) complete_basis(c, dQ, (int)m, (int)n);
        if (R != nullptr) {
            auto* dR = static_cast<cplx*>(stage_out(c, R, n * n * sizeof(cplx), outs));
            gemm(c, kOpC, (int)n, (int)n, (int)m, dQ, (long long)n, dA, (long long)n, dR, (long long)n);
        }
        finish_out(c, outs);
    });
}

int rrsvd_b200_chol_inv_flags(rrsvd_b200_ctx* c, const double* G, size_t l, double shift_scale, double* T,
                              int* ndead, int* ill) {
    return api(c, [&] {
        if (l == 0) return;
        if (G == nullptr || T == nullptr) throw_contract(c, "chol_inv: null argument");
        std::vector<OutBuf> outs;
        // the factorization works in place: always on a workspace copy of G
        auto* dG = ws_get<cplx>(c, l * l);
        check_cuda(c, cudaMemcpyAsync(dG, G, l * l * sizeof(cplx), cudaMemcpyDefault, c->stream), "copy G");
        auto* dT = static_cast<cplx*>(stage_out(c, T, l * l * sizeof(cplx), outs));
        int* dn = ws_get<int>(c, 2);
        check_cuda(c, cudaMemsetAsync(dn, 0, 2 * sizeof(int), c->stream), "memset");
        CholSpec cs{dG, (int)l, shift_scale, dT, dn};
        cs.ill_out = dn + 1;
        chol_inv_many(c, {cs});
        finish_out(c, outs);
        int h[2] = {0, 0};
        check_cuda(c, cudaMemcpyAsync(h, dn, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
        if (ndead) *ndead = h[0];
        if (ill) *ill = h[1];
    });
}

int rrsvd_b200_chol_inv(rrsvd_b200_ctx* c, const double* G, size_t l, double shift_scale, double* T,
                        int* ndead) {
    return rrsvd_b200_chol_inv_flags(c, G, l, shift_scale, T, ndead, nullptr);
}

int rrsvd_b200_svd(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, double* U, double* S,
                   double* V) {
    return api(c, [&] {
        const size_t r = std::min(m, n);
        if (r == 0) return;
        std::vector<OutBuf> outs;
        const auto* dA = static_cast<const cplx*>(stage_in(c, A, m * n * sizeof(cplx)));
        auto* dU = static_cast<cplx*>(stage_out(c, U, m * r * sizeof(cplx), outs));
        auto* dS = static_cast<double*>(stage_out(c, S, r * sizeof(double), outs));
        auto* dV = static_cast<cplx*>(stage_out(c, V, n * r * sizeof(cplx), outs));
        if (!dU) dU = ws_get<cplx>(c, m * r);
        if (!dS) dS = ws_get<double>(c, r);
        if (!dV) dV = ws_get<cplx>(c, n * r);
        svd_jacobi(c, dA, (int)m, (int)n, dU, dS, dV);
        // svd_full's U and V have orthonormal columns for ANY A (linalg.hpp:17-26, zgesdd): the
        // singular vectors of exactly-zero singular values come back as zero columns from the
        // Jacobi finish and get an orthonormal completion here (the decimation path truncates
        // them away and never needs it)
        if (U != nullptr) complete_basis(c, dU, (int)m, (int)r);
        if (V != nullptr) complete_basis(c, dV, (int)n, (int)r);
        finish_out(c, outs);
    });
}

// ------------------------------------------------------------------------------------------ L2

int rrsvd_b200_gaussian_test_matrix(rrsvd_b200_ctx* c, size_t n, size_t l, uint64_t seed, int mode,
                                    double* out) {
    return api(c, [&] {
        if (l < 1 || n < l) throw_contract(c, "gaussian_test_matrix: requires n >= l >= 1");
        std::vector<OutBuf> outs;
        auto* d = static_cast<cplx*>(stage_out(c, out, n * l * sizeof(cplx), outs));
        make_omega(c, (int)n, (int)l, seed, mode, d);
        finish_out(c, outs);
    });
}

int rrsvd_b200_range_finder(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, size_t l, size_t q,
                            uint64_t seed, int omega_mode, const double* omega, double* Q) {
    return api(c, [&] {
        if (l > std::min(m, n)) throw_contract(c, "randomized_range_finder: l > min(m, n)");
        if (l < 1) throw_contract(c, "gaussian_test_matrix: requires n >= l >= 1");
        if (Q == nullptr) throw_contract(c, "randomized_range_finder: null output");
        std::vector<OutBuf> outs;
        const auto* dA = static_cast<const cplx*>(stage_in(c, A, m * n * sizeof(cplx)));
        const cplx* dO = static_cast<const cplx*>(stage_in(c, omega, n * l * sizeof(cplx)));
        if (dO == nullptr) {
            cplx* o = ws_get<cplx>(c, n * l);
            make_omega(c, (int)n, (int)l, seed, omega_mode, o);
            dO = o;
        }
        auto* dQ = static_cast<cplx*>(stage_out(c, Q, m * l * sizeof(cplx), outs));
        range_finder_many(c, {RangeSpec{dA, (int)m, (int)n, (int)l, (int)q, dO, dQ}});
        complete_basis(c, dQ, (int)m, (int)l);  // RangeBasis::q_matrix is orthonormal (randomized.hpp:25-28)
        finish_out(c, outs);
    });
}

static void sketch_common(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, size_t l, size_t q,
                          uint64_t seed, int omega_mode, const double* omega, size_t keep, double* U,
                          double* S, double* V, double* discarded) {
    std::vector<OutBuf> outs;
    const auto* dA = static_cast<const cplx*>(stage_in(c, A, m * n * sizeof(cplx)));
    const cplx* dO = static_cast<const cplx*>(stage_in(c, omega, n * l * sizeof(cplx)));
    if (dO == nullptr) {
        cplx* o = ws_get<cplx>(c, n * l);
        make_omega(c, (int)n, (int)l, seed, omega_mode, o);
        dO = o;
    }
    cplx* dU = ws_get<cplx>(c, m * l);
    cplx* dV = ws_get<cplx>(c, n * l);
    double* dS = ws_get<double>(c, l);
    rrsvd_core(c, dA, (int)m, (int)n, (int)l, (int)q, dO, dU, dS, dV);
    double* part = ws_get<double>(c, 2 * kNumSMs);
    int* bad = ws_get<int>(c, 2 * kNumSMs);
    auto* sc = ws_get<Scalars>(c, 1);
    check_cuda(c, sumsq(dA, (long long)(m * n), part, bad, &sc->total_sq, &sc->nonfinite, c->stream), "sumsq");
    check_cuda(c, discarded_weight(dS, (int)keep, &sc->total_sq, &sc->discarded, c->stream), "weight");
    c->launches += 3;
    copy_out2d(c, U, keep * sizeof(cplx), dU, l * sizeof(cplx), keep * sizeof(cplx), m);
    copy_out2d(c, V, keep * sizeof(cplx), dV, l * sizeof(cplx), keep * sizeof(cplx), n);
    copy_out2d(c, S, keep * sizeof(double), dS, keep * sizeof(double), keep * sizeof(double), 1);
    Scalars h;
    read_scalars(c, sc, &h);
    if (discarded) *discarded = h.discarded;
}

int rrsvd_b200_sketched_svd(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, size_t l, size_t q,
                            uint64_t seed, int omega_mode, const double* omega, double* U, double* S,
                            double* V, double* discarded) {
    return api(c, [&] {
        if (l > std::min(m, n)) throw_contract(c, "randomized_range_finder: l > min(m, n)");
        if (l < 1) throw_contract(c, "gaussian_test_matrix: requires n >= l >= 1");
        sketch_common(c, A, m, n, l, q, seed, omega_mode, omega, l, U, S, V, discarded);
    });
}

int rrsvd_b200_fixed_rank(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, size_t k, size_t p,
                          size_t q, uint64_t seed, int omega_mode, const double* omega, double* U,
                          double* S, double* V, double* discarded) {
    return api(c, [&] {
        if (k < 2 || p < 2) throw_contract(c, "rrsvd_fixed_rank: requires k >= 2 and p >= 2");
        if (k + p > std::min(m, n)) throw_contract(c, "rrsvd_fixed_rank: k + p exceeds min(m, n)");
        sketch_common(c, A, m, n, k + p, q, seed, omega_mode, omega, k, U, S, V, discarded);
    });
}

int rrsvd_b200_fixed_precision(rrsvd_b200_ctx* c, const double* A, size_t m, size_t n, size_t initial_l,
                               size_t q, size_t probe_count, size_t growth_block, double epsilon, uint64_t seed,
                               int omega_mode, double* U, double* S, double* V, size_t* out_l, int* certified,
                               double* discarded) {
    return api(c, [&] {
        if (S == nullptr || out_l == nullptr) throw_contract(c, "fixed_precision: null argument");
        if (probe_count < 1) throw_contract(c, "rrsvd_fixed_precision: probe_count >= 1 required");
        if (initial_l < 1 || initial_l + probe_count > n)
            throw_contract(c, "rrsvd_fixed_precision: requires initial_l + probe_count <= n");
        const auto* dA = static_cast<const cplx*>(stage_in(c, A, m * n * sizeof(cplx)));
        std::vector<FixedPrecSpec> fp{FixedPrecSpec{dA, (int)m, (int)n, (int)initial_l, (int)q, (int)probe_count,
                                                    epsilon, seed, omega_mode}};
        fp[0].growth_block = (int)std::min(growth_block, std::min(m, n));
        rrsvd_fixed_precision_many(c, fp);
        const size_t l = (size_t)fp[0].l;
        auto* sc = ws_get<Scalars>(c, 1);
        SumsqBatch sb{};
        sb.count = 1;
        sb.a[0] = dA; sb.n[0] = (long long)(m * n); sb.out_sq[0] = &sc->total_sq; sb.out_bad[0] = &sc->nonfinite;
        check_cuda(c, sumsq_many(sb, ws_get<double>(c, 2 * kNumSMs), ws_get<int>(c, 2 * kNumSMs), c->stream),
                   "sumsq");
        check_cuda(c, discarded_weight(fp[0].sigma, (int)l, &sc->total_sq, &sc->discarded, c->stream), "weight");
        c->launches += 3;
        if (U) copy_out(c, U, fp[0].U, m * l * sizeof(cplx));
        if (V) copy_out(c, V, fp[0].V, n * l * sizeof(cplx));
        copy_out(c, S, fp[0].sigma, l * sizeof(double));
        Scalars h;
        read_scalars(c, sc, &h);
        *out_l = l;
        if (certified) *certified = fp[0].certified ? 1 : 0;
        if (discarded) *discarded = h.discarded;
    });
}

int rrsvd_b200_fixed_rank_batch(rrsvd_b200_ctx* c, size_t count, const double* const* A, size_t m, size_t n,
                                size_t k, size_t p, size_t q, const uint64_t* seeds, int omega_mode,
                                double* const* U, double* const* S, double* const* V, double* discarded) {
    return api(c, [&] {
        if (count == 0) return;
        if (A == nullptr || S == nullptr || seeds == nullptr) throw_contract(c, "fixed_rank_batch: null argument");
        if (k < 2 || p < 2) throw_contract(c, "rrsvd_fixed_rank: requires k >= 2 and p >= 2");
        if (k + p > std::min(m, n)) throw_contract(c, "rrsvd_fixed_rank: k + p exceeds min(m, n)");
        const size_t l = k + p;
        std::vector<RrsvdSpec> specs;
        std::vector<cplx*> dU(count), dV(count);
        std::vector<double*> dS(count);
        std::vector<const cplx*> dA(count);
        PhiloxBatch pb{};
        for (size_t i = 0; i < count; ++i) {
            dA[i] = static_cast<const cplx*>(stage_in(c, A[i], m * n * sizeof(cplx)));
            cplx* om = ws_get<cplx>(c, n * l);
            if (omega_mode == RRSVD_B200_OMEGA_PHILOX) {
                const int t = pb.count++;
                pb.seed[t] = seeds[i]; pb.n[t] = (long long)(n * l); pb.out[t] = om;
                if (pb.count == kMaxEpi) {
                    check_cuda(c, omega_philox_many(pb, c->stream), "philox_many");
                    c->launches++;
                    pb.count = 0;
                }
            } else {
                make_omega(c, (int)n, (int)l, seeds[i], omega_mode, om);
            }
            dU[i] = ws_get<cplx>(c, m * l);
            dV[i] = ws_get<cplx>(c, n * l);
            dS[i] = ws_get<double>(c, l);
            specs.push_back({dA[i], (int)m, (int)n, (int)l, (int)q, om, dU[i], dS[i], dV[i]});
        }
        if (pb.count) {
            check_cuda(c, omega_philox_many(pb, c->stream), "philox_many");
            c->launches++;
        }
        rrsvd_core_many(c, specs);
        auto* sc = ws_get<Scalars>(c, count);
        for (size_t base = 0; base < count; base += kMaxSmall) {
            SumsqBatch sb{};
            for (size_t i = base; i < std::min(count, base + kMaxSmall); ++i) {
                const int t = sb.count++;
                sb.a[t] = dA[i]; sb.n[t] = (long long)(m * n); sb.out_sq[t] = &sc[i].total_sq; sb.out_bad[t] = &sc[i].nonfinite;
            }
            double* part = ws_get<double>(c, (size_t)sb.count * 2 * kNumSMs);
            int* bad = ws_get<int>(c, (size_t)sb.count * 2 * kNumSMs);
            check_cuda(c, sumsq_many(sb, part, bad, c->stream), "sumsq_many");
            c->launches += 2;
        }
        for (size_t i = 0; i < count; ++i) {
            check_cuda(c, discarded_weight(dS[i], (int)k, &sc[i].total_sq, &sc[i].discarded, c->stream), "weight");
            c->launches++;
            if (U && U[i]) copy_out2d(c, U[i], k * sizeof(cplx), dU[i], l * sizeof(cplx), k * sizeof(cplx), m);
            if (V && V[i]) copy_out2d(c, V[i], k * sizeof(cplx), dV[i], l * sizeof(cplx), k * sizeof(cplx), n);
            copy_out(c, S[i], dS[i], k * sizeof(double));
        }
        std::vector<Scalars> h(count);
        check_cuda(c, cudaMemcpyAsync(h.data(), sc, count * sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream), "D2H");
        check_cuda(c, cudaStreamSynchronize(c->stream), "sync");
        if (discarded)
            for (size_t i = 0; i < count; ++i) discarded[i] = h[i].discarded;
    });
}

// ------------------------------------------------------------------------------------------ L3

int rrsvd_b200_build_theta_unfolded(rrsvd_b200_ctx* c, const double* G1, const double* G2,
                                    const double* ll, const double* lm, const double* lr, size_t cl,
                                    size_t d1, size_t cm, size_t d2, size_t cr, double* M) {
    return api(c, [&] {
        const size_t m = cl * d1, n = d2 * cr;
        if (m == 0 || n == 0) return;
        if (lm == nullptr) throw_contract(c, "build_theta: missing bond lambda");
        std::vector<OutBuf> outs;
        const auto* dG1 = static_cast<const cplx*>(stage_in(c, G1, m * cm * sizeof(cplx)));
        const auto* dG2 = static_cast<const cplx*>(stage_in(c, G2, cm * n * sizeof(cplx)));
        const auto* dll = static_cast<const double*>(stage_in(c, ll, cl * sizeof(double)));
        const auto* dlm = static_cast<const double*>(stage_in(c, lm, cm * sizeof(double)));
        const auto* dlr = static_cast<const double*>(stage_in(c, lr, cr * sizeof(double)));
        auto* dM = static_cast<cplx*>(stage_out(c, M, m * n * sizeof(cplx), outs));
        if (cm == 0) check_cuda(c, cudaMemsetAsync(dM, 0, m * n * sizeof(cplx), c->stream), "memset");
        else build_theta_many(c, {ThetaJob{dG1, dG2, dll, dlm, dlr, (int)cl, (int)d1, (int)cm, (int)d2, (int)cr, dM}});
        finish_out(c, outs);
    });
}

int rrsvd_b200_apply_gate_unfolded(rrsvd_b200_ctx* c, const double* G, size_t d1, size_t d2, size_t cl,
                                   size_t cr, const double* M_in, double* M_out) {
    return api(c, [&] {
        const size_t dd = d1 * d2, tot = cl * dd * cr;
        if (tot == 0) return;
        if (M_in == M_out) throw_contract(c, "apply_gate: in-place application is not supported");
        std::vector<OutBuf> outs;
        const auto* dG = static_cast<const cplx*>(stage_in(c, G, dd * dd * sizeof(cplx)));
        const auto* dI = static_cast<const cplx*>(stage_in(c, M_in, tot * sizeof(cplx)));
        auto* dO = static_cast<cplx*>(stage_out(c, M_out, tot * sizeof(cplx), outs));
        GateBlocksOwned gbo;
        const bool blocked = dd > 16 && make_gate_blocks(c, dG, (int)dd, gbo);
        apply_gate_many(c, {GateJob{dG, (int)d1, (int)d2, (int)cl, (int)cr, dI, dO, blocked ? &gbo.dev : nullptr}});
        free_gate_blocks(c, gbo);
        finish_out(c, outs);
    });
}

int rrsvd_b200_theta_to_unfolded(rrsvd_b200_ctx* c, const double* theta, size_t d1, size_t d2, size_t cl,
                                 size_t cr, double* M) {
    return api(c, [&] {
        const size_t tot = d1 * d2 * cl * cr;
        if (tot == 0) return;
        std::vector<OutBuf> outs;
        const auto* dT = static_cast<const cplx*>(stage_in(c, theta, tot * sizeof(cplx)));
        auto* dM = static_cast<cplx*>(stage_out(c, M, tot * sizeof(cplx), outs));
        check_cuda(c, theta_to_unfolded(dT, (int)d1, (int)d2, (int)cl, (int)cr, dM, c->stream), "unfold");
        c->launches++;
        finish_out(c, outs);
    });
}

int rrsvd_b200_unfolded_to_theta(rrsvd_b200_ctx* c, const double* M, size_t d1, size_t d2, size_t cl,
                                 size_t cr, double* theta) {
    return api(c, [&] {
        const size_t tot = d1 * d2 * cl * cr;
        if (tot == 0) return;
        std::vector<OutBuf> outs;
        const auto* dM = static_cast<const cplx*>(stage_in(c, M, tot * sizeof(cplx)));
        auto* dT = static_cast<cplx*>(stage_out(c, theta, tot * sizeof(cplx), outs));
        check_cuda(c, unfolded_to_theta(dM, (int)d1, (int)d2, (int)cl, (int)cr, dT, c->stream), "fold");
        c->launches++;
        finish_out(c, outs);
    });
}

int rrsvd_b200_decimate_unfolded(rrsvd_b200_ctx* c, const double* M, size_t d1, size_t d2, size_t cl,
                                 size_t cr, const double* ll, const double* lr, size_t chi_max,
                                 double trunc_tol, const rrsvd_b200_backend* be, uint64_t call_seed,
                                 int omega_mode, const double* omega, int renormalize, double* gamma_l,
                                 double* lambda, double* gamma_r, rrsvd_b200_decim_info* info) {
    return api(c, [&] {
        if (be == nullptr || info == nullptr) throw_contract(c, "decimate: null backend/info");
        const size_t m = d1 * cl, n = d2 * cr;
        if (m == 0 || n == 0) throw_contract(c, "decimate: theta is identically zero");
        const DecimPlan pl = plan_decimation((int)d1, (int)d2, (int)cl, (int)cr, chi_max, be->kind,
                                             be->target_rank, be->oversampling, be->det_crossover,
                                             be->accuracy_check, be->probe_count);
        const bool randomized = pl.randomized;
        const size_t kmax = (size_t)pl.kmax;
        const auto* dM = static_cast<const cplx*>(stage_in(c, M, m * n * sizeof(cplx)));
        const auto* dll = static_cast<const double*>(stage_in(c, ll, cl * sizeof(double)));
        const auto* dlr = static_cast<const double*>(stage_in(c, lr, cr * sizeof(double)));
        const cplx* dO = randomized ? static_cast<const cplx*>(stage_in(c, omega, n * pl.l * sizeof(cplx)))
                                    : nullptr;
        auto* sc = ws_get<Scalars>(c, 1);
        // outputs: write straight into device buffers, else into workspace + exact D2H
        const bool dev_gl = is_device_ptr(gamma_l), dev_lam = is_device_ptr(lambda), dev_gr = is_device_ptr(gamma_r);
        cplx* gl = dev_gl ? reinterpret_cast<cplx*>(gamma_l) : ws_get<cplx>(c, m * kmax);
        double* lam = dev_lam ? lambda : ws_get<double>(c, kmax);
        cplx* gr = dev_gr ? reinterpret_cast<cplx*>(gamma_r) : ws_get<cplx>(c, kmax * n);
        int certified = 1;
        DecimJob job{pl, dM, (int)d1, (int)cr, dll, dlr, chi_max, trunc_tol, (int)be->power_iterations,
                     call_seed, omega_mode, dO, renormalize, gl, lam, gr, reinterpret_cast<DecimScalars*>(sc)};
        job.eps = be->epsilon;
        job.certified = &certified;
        decimate_many(c, {job});
        Scalars h;
        read_scalars(c, sc, &h);
        if (h.nonfinite) throw_contract(c, "decimate: theta has non-finite entries");
        if (h.total_sq == 0.0) throw_contract(c, "decimate: theta is identically zero");
        const size_t kept = (size_t)h.kept;
        if (!dev_gl) copy_out(c, gamma_l, gl, m * kept * sizeof(cplx));
        if (!dev_lam) copy_out(c, lambda, lam, kept * sizeof(double));
        if (!dev_gr) copy_out(c, gamma_r, gr, kept * n * sizeof(cplx));
        check_cuda(c, cudaStreamSynchronize(c->stream), "stream sync");
        info->discarded = h.discarded;
        info->chi = kept;
        info->randomized_path = randomized ? 1 : 0;
        info->tolerance_certified = certified;
        info->pseudo_inverse_applied = h.pinv ? 1 : 0;
    });
}

// ------------------------------------------------------------------------------------------ misc

int rrsvd_b200_set_overlap(rrsvd_b200_ctx* c, int on) {
    return api(c, [&] { c->use_lanes = on != 0; });
}

int rrsvd_b200_set_gemm_timing(rrsvd_b200_ctx* c, int on) {
    return api(c, [&] {
        flush_gemm_timing(c);
        c->gemm_timing = on != 0;
        if (on) {
            c->gemm_ms = 0.0;
            c->gemm_flops = 0.0;
            c->gemm_exec_flops = 0.0;
            c->gemm_tma_ms = 0.0;
            c->gemm_calls = 0;
            c->oz_ms = c->oz_flops = c->oz_bytes = c->oz_prep_ms = c->oz_prep_bytes = 0.0;
            c->oz_calls = 0;
            c->oz_gemm_ms = c->oz_gemm_bytes = 0.0;
            for (int i = 0; i < 8; ++i) c->tag_ms[i] = c->tag_flops[i] = 0.0;
        }
    });
}

int rrsvd_b200_gemm_stats(rrsvd_b200_ctx* c, double* flops, double* ms, uint64_t* calls) {
    return api(c, [&] {
        flush_gemm_timing(c);
        if (flops) *flops = c->gemm_flops;
        if (ms) *ms = c->gemm_ms;
        if (calls) *calls = c->gemm_calls;
    });
}

int rrsvd_b200_gemm_pipe_stats(rrsvd_b200_ctx* c, double* executed_flops, double* tma_ms) {
    return api(c, [&] {
        flush_gemm_timing(c);
        if (executed_flops) *executed_flops = c->gemm_exec_flops;
        if (tma_ms) *tma_ms = c->gemm_tma_ms;
    });
}

int rrsvd_b200_ozaki_stats(rrsvd_b200_ctx* c, double* flops, double* ms, double* bytes, uint64_t* calls,
                           double* prep_ms, double* prep_bytes) {
    return api(c, [&] {
        flush_gemm_timing(c);
        if (flops) *flops = c->oz_flops;
        if (ms) *ms = c->oz_ms;
        if (bytes) *bytes = c->oz_bytes;
        if (calls) *calls = c->oz_calls;
        if (prep_ms) *prep_ms = c->oz_prep_ms;
        if (prep_bytes) *prep_bytes = c->oz_prep_bytes;
    });
}

int rrsvd_b200_ozaki_gemm_stats(rrsvd_b200_ctx* c, double* ms, double* bytes) {
    return api(c, [&] {
        flush_gemm_timing(c);
        if (ms) *ms = c->oz_gemm_ms;
        if (bytes) *bytes = c->oz_gemm_bytes;
    });
}

int rrsvd_b200_gemm_stage_stats(rrsvd_b200_ctx* c, double* flops8, double* ms8) {
    return api(c, [&] {
        flush_gemm_timing(c);
        for (int i = 0; i < 8; ++i) {
            if (flops8) flops8[i] = c->tag_flops[i];
            if (ms8) ms8[i] = c->tag_ms[i];
        }
    });
}

int rrsvd_b200_probe_peak(rrsvd_b200_ctx* c, int what, double* tflops) {
    return api(c, [&] {
        if (tflops == nullptr) throw_contract(c, "probe_peak: null output");
        if (what >= 100) {  // 100 + warps*10 + chains: DMMA at a given residency (diagnostics)
            const int code = what - 100;
            check_cuda(c, probe_dmma_occupancy(code / 10, code % 10, tflops, c->stream), "probe_dmma_occupancy");
            c->launches += 2;
            return;
        }
        check_cuda(c, probe_peak(what, tflops, c->stream), "probe_peak");
        c->launches += 2;
    });
}

}  // extern "C"

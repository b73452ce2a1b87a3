// ozaki.cuh — the RRSVD A-products (Y = A·X, Z = A^H·X; randomized.cpp:88-99, 57-66 through
// linalg.cpp:20-40) as exact integer products on the INT8 tensor cores (tcgen05.mma kind::i8),
// the Chinese-remainder ("Ozaki scheme II") emulation of the complex-FP64 GEMM.
//
// A is equilibrated by powers of two on both sides — A' = rint(A_ik·2^(kA - e_i - f_k)), e_i the
// exponent of row i's largest entry, f_k that of column k's after the rows are normalised — so
// every entry keeps kA bits relative to its own row and column scale (a TEBD Θ is λ-weighted on
// both sides); the K-side factor is moved into X (X_kj·2^(f_k), resp. Q_ij·2^(e_i) for A^H), and
// each column j of that is scaled by 2^(s_j) and rounded to |X'| <= 2^kX.  The complex product is one real
// integer GEMM with the real and imaginary parts stacked along K:
//   op N: [Y'_re | Y'_im] = [A'_re  A'_im] · [[X'_re, X'_im], [-X'_im, X'_re]]
//   op C: [Z'_re | Z'_im] = [A'_re  A'_im]^T · [[X'_re, X'_im], [X'_im, -X'_re]]
// (every entry an exact integer, |D| <= 2K·2^(kA+kX) < M/2), computed modulo T pairwise coprime
// moduli m_t <= 256 (M = prod m_t ~ 2^125 for T = 16): signed 8-bit residues, int32 accumulators
// in TMEM (no overflow for K <= 32768), and reconstructed exactly by the CRT,
//   D/M = frac_sym( sum_t ((D mod m_t)·w_t mod m_t) / m_t ),  w_t = (M/m_t)^-1 mod m_t,
// evaluated in fixed point (the top 96 bits of floor(2^128/m_t)), then scaled back by the row,
// column and panel exponents and rounded once to FP64.  The only approximation is the rounding of
// A and X to kA / kX bits (kA + kX = floor(log2 M) - 2 - ceil(log2 2K): for the default T = 15 and
// K = 2000, 52 + 51 bits — FP64's own precision class for every entry relative to its row and
// column scale), so the result carries FP64-GEMM-class error.
//
// A's residue planes are built once per decimation and serve all 2 + 2q products of the range
// finder and the basis assembly (op N reads them K-major, op C MN-major: no transposed copy).
#pragma once
#include <cstdint>
#include <vector>

#include "ctx.cuh"
#include "zgemm.cuh"

namespace rb {

constexpr int kOzMaxMod = 16;

// Residue planes of one A (m x n): int8 [T][2 (re, im)] planes stored as 128 x 128 tiles
// [ib][kb][128 rows][128 columns] (zero-padded to whole tiles) — every TMA box is one contiguous
// 16 KB block, serving op N as a K-major and op C as an MN-major operand tile.
struct OzakiA {
    int8_t* res = nullptr;
    int m = 0, n = 0;
    int nib = 0, nkb = 0;                // tile rows / columns: ceil(m / 128), ceil(n / 128)
    int T = 0, kA = 0;
    int* rowexp = nullptr;  // device [m]: e_i, the exponent of row i's largest |Re|, |Im|
    int* colexp = nullptr;  // device [n]: f_k = max_i e(|A_ik|) - e_i (<= 0)
    int* bad = nullptr;                     // device: a non-finite entry was seen
};

// Moduli count for the emulated A-products: RRSVD_B200_OZAKI (0 = off, every A-product on the DMMA
// zgemm; 8..16), default 15.  ozaki_usable: the shape gate of the RRSVD paths.
int ozaki_moduli();
bool ozaki_usable(int m, int n, int l);
// Least total A entries (sum of m·n over a batch) for the emulation (RRSVD_B200_OZAKI_MIN_WORK, 8e6).
double ozaki_min_work();
// Most residue-plane bytes one call may hold (RRSVD_B200_OZAKI_MAX_GB, default 32 GB).
double ozaki_max_bytes();
// RRSVD_B200_OZAKI_TAIL: how many of the RRSVD's last A-products stay on the FP64 zgemm — 0
// (default): none; 1: the assembly B^H = A^H Q; 2: also the final Y = A Q~ of the power iteration.
int ozaki_tail();

struct OzSrc {
    const cplx* A;
    int m, n;
    long long lda;
    double* total_sq = nullptr;  // optional: ||A||_F^2 (row sums taken by the row-exponent pass)
    int* nonfinite = nullptr;    // optional (with total_sq): 1 if A has a non-finite entry
};
// Builds the residue planes of every A (three launches for the whole batch); with `keep`, the
// buffers are not workspace (they outlive the public call) and are appended to *keep for the
// caller to free (cudaFreeAsync).
std::vector<OzakiA> ozaki_prepare_many(rrsvd_b200_ctx* c, const std::vector<OzSrc>& src, int T,
                                       std::vector<void*>* keep = nullptr);

// C = op(A)·X: op N — A m x n, X n x l (ld ldx), C m x l; op C — X m x l, C n x l.
struct OzProduct {
    const OzakiA* a;
    const cplx* X;
    long long ldx;
    int l;
    cplx* C;
    long long ldc;
    int accumulate = 0;  // 1: C += op(A)·X (a K-chunk of a wider product)
    int T = 0;           // moduli of this product (0: all of A's; fewer: the first T planes, X to
                         // fewer bits — the power iteration's intermediate products)
};
// RRSVD_B200_OZAKI_INNER: moduli of the power iteration's intermediate A-products (default 14;
// 0 or >= the planes' count: all).  The final Y = A Q~ and the assembly B^H = A^H Q use all.
int ozaki_inner_moduli();
void ozaki_product_many(rrsvd_b200_ctx* c, GemmOp op, const std::vector<OzProduct>& ps);

}  // namespace rb

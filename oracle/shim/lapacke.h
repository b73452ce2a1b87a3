/* Prototype shim for the LAPACKE ABI (LP64) exported by OpenBLAS 0.3.15.  Test
 * infrastructure only; see cblas.h. */
#ifndef ORACLE_SHIM_LAPACKE_H
#define ORACLE_SHIM_LAPACKE_H
#include <complex>
typedef std::complex<double> lapack_complex_double;
typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
extern "C" {
lapack_int LAPACKE_zgeqrf(int layout, lapack_int m, lapack_int n, lapack_complex_double* a,
                          lapack_int lda, lapack_complex_double* tau);
lapack_int LAPACKE_zungqr(int layout, lapack_int m, lapack_int n, lapack_int k,
                          lapack_complex_double* a, lapack_int lda,
                          const lapack_complex_double* tau);
lapack_int LAPACKE_zgesdd(int layout, char jobz, lapack_int m, lapack_int n,
                          lapack_complex_double* a, lapack_int lda, double* s,
                          lapack_complex_double* u, lapack_int ldu, lapack_complex_double* vt,
                          lapack_int ldvt);
lapack_int LAPACKE_zheevd(int layout, char jobz, char uplo, lapack_int n,
                          lapack_complex_double* a, lapack_int lda, double* w);
}
#endif

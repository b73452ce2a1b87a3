/* Prototype shim for the CBLAS ABI exported by OpenBLAS 0.3.15 (the copy bundled in the
 * opencv_python_headless wheel).  Test infrastructure only: it lets the UNMODIFIED reference
 * sources under /root/reference/proj/core/src compile into oracle/_ref/.  It declares the
 * third-party ABI and contains no reference code. */
#ifndef ORACLE_SHIM_CBLAS_H
#define ORACLE_SHIM_CBLAS_H
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_zgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int m, int n,
                 int k, const void* alpha, const void* a, int lda, const void* b, int ldb,
                 const void* beta, void* c, int ldc);
void cblas_zgemv(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, int m, int n, const void* alpha,
                 const void* a, int lda, const void* x, int incx, const void* beta, void* y,
                 int incy);
double cblas_dznrm2(int n, const void* x, int incx);
void cblas_zdscal(int n, double alpha, void* x, int incx);
void cblas_zcopy(int n, const void* x, int incx, void* y, int incy);
void openblas_set_num_threads(int);
int openblas_get_num_threads(void);
char* openblas_get_config(void);
char* openblas_get_corename(void);
#ifdef __cplusplus
}
#endif
#endif

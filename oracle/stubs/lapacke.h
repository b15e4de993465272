/* Prototype-only LAPACKE header for building the reference oracle.
 *
 * TEST INFRASTRUCTURE (oracle/): the reference's lapack.cpp
 * (/root/reference/proj/core/src/lapack.cpp:1-107) includes <lapacke.h>,
 * which this image does not ship.  The symbols themselves are exported by the
 * OpenBLAS 0.3.15 bundled with opencv_python_headless (LP64), so only the
 * seven prototypes the reference calls are declared here.
 */
#ifndef BIPM_ORACLE_LAPACKE_STUB_H
#define BIPM_ORACLE_LAPACKE_STUB_H

#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102

#ifdef __cplusplus
extern "C" {
#endif

typedef int lapack_int;

lapack_int LAPACKE_dgetrf(int layout, lapack_int m, lapack_int n, double* a, lapack_int lda,
                          lapack_int* ipiv);
lapack_int LAPACKE_dgetrs(int layout, char trans, lapack_int n, lapack_int nrhs, const double* a,
                          lapack_int lda, const lapack_int* ipiv, double* b, lapack_int ldb);
lapack_int LAPACKE_dpotrf(int layout, char uplo, lapack_int n, double* a, lapack_int lda);
lapack_int LAPACKE_dpotrs(int layout, char uplo, lapack_int n, lapack_int nrhs, const double* a,
                          lapack_int lda, double* b, lapack_int ldb);
lapack_int LAPACKE_dsytrf(int layout, char uplo, lapack_int n, double* a, lapack_int lda,
                          lapack_int* ipiv);
lapack_int LAPACKE_dsytrs(int layout, char uplo, lapack_int n, lapack_int nrhs, const double* a,
                          lapack_int lda, const lapack_int* ipiv, double* b, lapack_int ldb);
lapack_int LAPACKE_dsyev(int layout, char jobz, char uplo, lapack_int n, double* a,
                         lapack_int lda, double* w);

#ifdef __cplusplus
}
#endif

#endif

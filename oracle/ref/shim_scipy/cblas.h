/* CBLAS declarations for the reference headers (kernels.hpp:10) resolved against
 * scipy's LP64 OpenBLAS 0.3.31 (symbols prefixed scipy_). Used only to build
 * oracle/_ref/libbbsi_ref_scipy.so: the UNMODIFIED reference on a second BLAS build,
 * whose distance to the 0.3.15 build is the reference's own rounding floor.
 * Test infrastructure only. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void scipy_cblas_sgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int, float,
                       const float*, int, const float*, int, float, float*, int);
void scipy_cblas_dgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int, double,
                       const double*, int, const double*, int, double, double*, int);
void scipy_cblas_cgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int, const void*,
                       const void*, int, const void*, int, const void*, void*, int);
void scipy_cblas_zgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int, const void*,
                       const void*, int, const void*, int, const void*, void*, int);
void scipy_openblas_set_num_threads(int);
#ifdef __cplusplus
}
#endif
#define cblas_sgemm scipy_cblas_sgemm
#define cblas_dgemm scipy_cblas_dgemm
#define cblas_cgemm scipy_cblas_cgemm
#define cblas_zgemm scipy_cblas_zgemm
#define openblas_set_num_threads scipy_openblas_set_num_threads

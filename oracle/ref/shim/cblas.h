/* Minimal CBLAS declarations so the reference headers (kernels.hpp:10) compile
 * against the OpenBLAS 0.3.15 build bundled in the image. Test infrastructure
 * only (oracle/_ref); never linked into the product library. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_sgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int, float,
                 const float*, int, const float*, int, float, float*, int);
void cblas_dgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int, double,
                 const double*, int, const double*, int, double, double*, int);
void cblas_cgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int, const void*,
                 const void*, int, const void*, int, const void*, void*, int);
void cblas_zgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int, const void*,
                 const void*, int, const void*, int, const void*, void*, int);
void openblas_set_num_threads(int);
#ifdef __cplusplus
}
#endif

/* LAPACKE declarations for the reference headers (kernels.hpp:11) against scipy's
 * LP64 OpenBLAS 0.3.31 (prefixed symbols). Test infrastructure only. */
#pragma once
#include <complex>
#define LAPACK_COL_MAJOR 102
#define LAPACK_ROW_MAJOR 101
typedef std::complex<float> lapack_complex_float;
typedef std::complex<double> lapack_complex_double;
extern "C" {
int scipy_LAPACKE_sgetrf(int, int, int, float*, int, int*);
int scipy_LAPACKE_dgetrf(int, int, int, double*, int, int*);
int scipy_LAPACKE_cgetrf(int, int, int, lapack_complex_float*, int, int*);
int scipy_LAPACKE_zgetrf(int, int, int, lapack_complex_double*, int, int*);
int scipy_LAPACKE_sgetrs(int, char, int, int, const float*, int, const int*, float*, int);
int scipy_LAPACKE_dgetrs(int, char, int, int, const double*, int, const int*, double*, int);
int scipy_LAPACKE_cgetrs(int, char, int, int, const lapack_complex_float*, int, const int*, lapack_complex_float*, int);
int scipy_LAPACKE_zgetrs(int, char, int, int, const lapack_complex_double*, int, const int*, lapack_complex_double*,
                         int);
}
#define LAPACKE_sgetrf scipy_LAPACKE_sgetrf
#define LAPACKE_dgetrf scipy_LAPACKE_dgetrf
#define LAPACKE_cgetrf scipy_LAPACKE_cgetrf
#define LAPACKE_zgetrf scipy_LAPACKE_zgetrf
#define LAPACKE_sgetrs scipy_LAPACKE_sgetrs
#define LAPACKE_dgetrs scipy_LAPACKE_dgetrs
#define LAPACKE_cgetrs scipy_LAPACKE_cgetrs
#define LAPACKE_zgetrs scipy_LAPACKE_zgetrs

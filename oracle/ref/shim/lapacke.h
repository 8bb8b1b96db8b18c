/* Minimal LAPACKE declarations for the reference headers (kernels.hpp:11),
 * resolved against the image's bundled OpenBLAS 0.3.15. Test infrastructure. */
#pragma once
#include <complex>
#define LAPACK_COL_MAJOR 102
#define LAPACK_ROW_MAJOR 101
typedef std::complex<float> lapack_complex_float;
typedef std::complex<double> lapack_complex_double;
extern "C" {
int LAPACKE_sgetrf(int, int, int, float*, int, int*);
int LAPACKE_dgetrf(int, int, int, double*, int, int*);
int LAPACKE_cgetrf(int, int, int, lapack_complex_float*, int, int*);
int LAPACKE_zgetrf(int, int, int, lapack_complex_double*, int, int*);
int LAPACKE_sgetrs(int, char, int, int, const float*, int, const int*, float*, int);
int LAPACKE_dgetrs(int, char, int, int, const double*, int, const int*, double*, int);
int LAPACKE_cgetrs(int, char, int, int, const lapack_complex_float*, int, const int*, lapack_complex_float*, int);
int LAPACKE_zgetrs(int, char, int, int, const lapack_complex_double*, int, const int*, lapack_complex_double*, int);
}

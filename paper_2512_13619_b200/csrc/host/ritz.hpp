// Host-side small dense pieces of the polynomial preconditioner (see ritz.cpp).
#pragma once
#include <complex>
#include <vector>

namespace hdgb {

// leja_order (preconditioner.cpp:207-244)
std::vector<std::complex<double>> leja_order(const std::vector<std::complex<double>>& theta);

// Post-Arnoldi part of compute_harmonic_ritz (preconditioner.cpp:162-205).  hess is the
// (pmax+1) x pmax column-major Arnoldi Hessenberg matrix, p_eff the number of completed steps.
std::vector<std::complex<double>> harmonic_ritz_from_hessenberg(const double* hess, int pmax, int p_eff);

}  // namespace hdgb

// Host-side operator setup for K2.
//  * separable patches (constant weights, x = X(i), y = Y(j), z = Z(k)): the
//    banded 1D mass / stiffness factors of the Kronecker form;
//  * general patches: the assembled free-free CSR of A = M/dt + theta K and the
//    full CSR pair for the right-hand side, built with the same element
//    quadrature as the reference (assembly.cpp:59-101).
#pragma once

#include <array>
#include <vector>

#include "mesh.hpp"

namespace tgb {

struct Band1D {
  int n = 0, p = 0;
  std::vector<double> M, K;  // n x (2p+1), [i][p + (j - i)]
};

// Returns true and the per-axis control coordinates when the patch is
// separable; the 1D factors then reproduce the reference's M and K up to
// rounding (the tensor Gauss rule factorizes).
bool separable_coords(const NurbsVolume& vol, std::array<std::vector<double>, 3>& coord);
Band1D assemble_band_1d(const KnotVector& kv, const std::vector<double>& coord, int nq);

struct Csr {
  int rows = 0;
  std::vector<int> row_ptr, col;
  std::vector<double> val;
};
// Sliced ELL copy (32-row slices, entry k of a slice's rows contiguous,
// padded to the slice's longest row) for coalesced one-thread-per-row
// products on the GPU (k2_csr.cu DevSell).
struct Sell {
  int rows = 0;
  std::vector<long long> slice_ptr;
  std::vector<int> row_len, col;
  std::vector<double> val;
};
Sell to_sell(const Csr& m);

// M (coefficient rho c) and K (coefficient k) on the full tensor pattern
// (assembly.cpp:8-101), element contributions scattered in element order.
void assemble_mass_stiffness(const NurbsVolume& vol, std::array<int, 3> nq, const Material& mat,
                             Csr& M, Csr& K);

}  // namespace tgb

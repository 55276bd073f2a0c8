// Host exact lattice routines used by maple_create (see lattice.cpp for the paper citations).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace maple {
// B (n x d row-major) = last d columns of the unimodular C with A C = (H | 0). Returns 0 or a MAPLE_ERR_*.
int host_kernel_basis(const int32_t* A, int m, int n, std::vector<int64_t>& B, std::string& err);
// In-place LLL reduction (Siegel factor 2) of the columns of B (n x d row-major).
int host_lll(std::vector<int64_t>& B, int n, int d, std::string& err);
// Bp (d x n row-major) = (B^T B)^{-1} B^T.
int host_pinv(const std::vector<int64_t>& B, int n, int d, std::vector<double>& Bp, std::string& err);
}  // namespace maple

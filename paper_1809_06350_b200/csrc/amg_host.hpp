// Smoothed-aggregation AMG setup on the host (amg.cpp:32-295), producing the
// level operators that the device V-cycle consumes.  Every per-row numeric
// kernel keeps the reference's per-row summation order and runs rows in
// parallel (OpenMP), so the hierarchy is bitwise identical to the
// reference's for identical input.  Moving this setup to the GPU is the
// next step.
#pragma once

#include <vector>

#include "ed_internal.hpp"

namespace edb {

struct AmgOpts {
    int block_size = 1;
    std::vector<int> row_to_node, row_component;
    double strength_theta = 0.08;
    int max_levels = 12;
    int coarse_max_rows = 200;
    int smoother = 1; // 0 Jacobi, 1 SGS
    double jacobi_weight = 2.0 / 3.0;
    int pre_sweeps = 1, post_sweeps = 1;
    bool smooth_prolongator = true;
};

struct HostLevel {
    HostCsr A, P, R;
    std::vector<double> inv_diag;
};

struct HostHierarchy {
    std::vector<HostLevel> levels; // last = coarsest (A, inv_diag only)
    bool fallback = false;
    std::vector<double> fallback_inv_diag;
    std::vector<double> pinv; // coarsest min-norm solve operator, n_c x n_c row-major
    int nc = 0;
};

HostHierarchy amg_build_host(const HostCsr& A0, const AmgOpts& opts);

// Pieces reused by the device setup (amg_device.cu):
// greedy aggregation on a symmetric neighbour CSR (amg.cpp:85-117)
int amg_aggregate(const std::vector<int64_t>& nbr_ptr, const std::vector<int>& nbr, std::vector<int>& agg_of);
// tentative prolongator + coarse near-nullspace (amg.cpp:122-168)
HostCsr amg_tentative(int nrows, int k, const std::vector<int>& agg_of_row, int n_agg, const std::vector<double>& B,
                      std::vector<double>& Bc);
// (sqrt of) the sequential sum of squares, vec_norm order (csr.cpp:213-221)
double amg_seq_norm(const std::vector<double>& v);

// CSR helpers restating csr.cpp
HostCsr csr_matmul(const HostCsr& a, const HostCsr& b);
HostCsr csr_transpose(const HostCsr& a);
HostCsr csr_add(const HostCsr& a, const HostCsr& b, double alpha, double beta);
std::vector<double> csr_diag(const HostCsr& a);

// Complete orthogonal decomposition pseudo-inverse (min-norm LS solve
// operator) with the rank threshold of Eigen's COD.setThreshold(t).
// Largest coarsest level whose dense COD is formed (16384^2 doubles = 2 GB).
constexpr int kMaxCoarseDenseRows = 16384;
void check_coarse_size(int nrows, int n_coarsened);
std::vector<double> cod_pinv(const std::vector<double>& dense_colmajor, int n, double threshold);

} // namespace edb

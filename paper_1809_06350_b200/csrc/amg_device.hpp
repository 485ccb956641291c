// Smoothed-aggregation AMG setup on the GPU (amg.cpp:189-295).
//
// The numeric steps run on the device with the reference's per-entry
// arithmetic order and no FMA contraction, so the hierarchy is bitwise the
// reference's:
//   strength graph  -- per block s2 = sum v^2 in row-major block order
//                      (amg.cpp:36-67); comparisons within 1e-12 of the
//                      threshold are re-decided on the host with libm pow
//   aggregation     -- host, sequential greedy (amg.cpp:85-117)
//   tentative P     -- host per-aggregate MGS (amg.cpp:122-168), tiny
//   spectral radius -- device row-sequential SpMV, host sequential norms
//   SpGEMM          -- symbolic: CUB segmented sort of candidate columns;
//                      numeric: one thread per scalar row accumulating in
//                      (A column, B column) traversal order (csr.cpp:132-166)
//   transpose       -- stable CUB radix sort by block column (csr.cpp:39-57)
#pragma once

#include <functional>

#include "amg_host.hpp"
#include "ed_internal.hpp"

namespace edb {

// Natural-order block CSR on the device.
struct DBsr {
    int nbr = 0, nbc = 0, Rb = 1, Cb = 1;
    int64_t nnzb = 0;
    DevArray<int> rowptr, col;
    DevArray<double> val;
};

// Non-owning view of a natural-order device BSR (read by another host thread
// while the owner moves the DBsr object itself; the device arrays stay put).
struct DBsrRaw {
    int nbr = 0, nbc = 0, Rb = 1, Cb = 1;
    int64_t nnzb = 0;
    const int* rowptr = nullptr;
    const int* col = nullptr;
    const double* val = nullptr;
};
inline DBsrRaw raw_of(const DBsr& m) { return DBsrRaw{m.nbr, m.nbc, m.Rb, m.Cb, m.nnzb, m.rowptr.p, m.col.p, m.val.p}; }

struct DevLevelData {
    DBsr A, P, R;                 // P, R empty on the coarsest level
    std::vector<double> inv_diag; // host copy (small enough; uploaded by the caller)
    DevArray<double> invd;
};

struct DevSetupResult {
    std::vector<DevLevelData> levels;
    bool fallback = false;
    std::vector<double> fallback_inv_diag;
    std::vector<double> pinv;
    int nc = 0;
};

// A0 given as a (possibly level-permuted) Bsr with block size == opts.block_size.
// on_level(l, A_l) is called on the building thread as soon as the Galerkin
// operator of level l >= 1 is enqueued on s (its arrays stay valid until the
// result is destroyed); on_level(-1, {}) before an exception leaves.
using LevelHook = std::function<void(int, const DBsrRaw&)>;
DevSetupResult amg_build_device(const Bsr& A0, const AmgOpts& opts, cudaStream_t s, const LevelHook& on_level = {});

// One level of a collapsed coarse tail (dense_tail.cu): natural-order
// operator, prolongator/restriction to the next level, inv_diag (device).
struct DenseTailLevel {
    const DBsr* A = nullptr;
    const DBsr* P = nullptr;
    const DBsr* R = nullptr;
    const double* invd = nullptr;
};
// Row-major dense V-cycle operator of levels lv[0..] above a coarsest level
// with the given row-major pseudo-inverse (n_c x n_c): out = V_{lv[0]}.
void dense_vcycle_operator(const std::vector<DenseTailLevel>& lv, const std::vector<double>& pinv, int nc,
                           int pre_sweeps, int post_sweeps, DevArray<double>& out, cudaStream_t s);

// Helpers shared with the V-cycle construction.
// The structure of a level operator (level schedule, layout, sweep
// structures) from the previous hierarchy build, with the pattern it was built
// from: reused when the new level's pattern is exactly the same (checked on the
// device), so only the values are gathered.
struct LevelCache {
    int nbr = -1, nbc = -1, Rb = 0, Cb = 0;
    int64_t nnzb = -1;
    DevArray<int> rowptr, col;
    std::shared_ptr<BsrStruct> st;
    DevArray<int> flag;
};
Bsr bsr_from_dbsr(DBsr&& m, bool leveled, cudaStream_t s, LevelCache* cache = nullptr);
// the leveled (Gauss-Seidel level-ordered) operator of m; reads m only
Bsr bsr_leveled(const DBsrRaw& m, cudaStream_t s, LevelCache* cache = nullptr);

} // namespace edb

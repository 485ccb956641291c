// Context, block system and solver declarations.
#pragma once

#include <chrono>
#include <memory>
#include <string>
#include <vector>

#include "amg_device.hpp"
#include "amg_host.hpp"
#include "assembly.hpp"
#include "ed_internal.hpp"

namespace edb {

// The 2x2 block system [A B; C D] (blocksystem.hpp:19-34) as SELL planes.
// A and B share the (leveled) velocity row layout; C and D share the
// pressure row layout.  Bv = rows per velocity block (3 for nodal systems).
struct BlockSys {
    int Bv = 3;
    int nv = 0, np = 0;
    BlockPattern pA, pB, pC, pD;
    BsrLayout lA, lB, lC, lD;
    Bsr A, B, C, D;
    // S_hat symbolic (pattern of D - C diag(A)^-1 B, leveled) + position maps
    bool shat_symbolic = false;
    std::shared_ptr<BsrStruct> sS;
    DevArray<int64_t> cb_off, d_off;
    DevArray<uint16_t> cb_pos, d_pos;
    int64_t shat_nnz = 0;
    bool valid() const { return A.st != nullptr; }
    // structure built from patterns (values zero)
    void build_structure(cudaStream_t s);
    void build_shat_symbolic(cudaStream_t s);
};

struct KrylovCfg {
    int restart = 50, max_iters = 500;
    double rel_tol = 1e-6, abs_tol = 1e-50;
};

struct SolveRes {
    bool converged = false;
    int iterations = 0;
    double initial_norm = 0.0, final_norm = 0.0;
    std::vector<double> history;
};

struct Stats {
    long outer_iters = 0, a_solves = 0, a_iters = 0, s_solves = 0, s_iters = 0, schur_applies = 0, inner_iters = 0;
    bool converged = true;
    double t_solve = 0.0;
};

struct Ctx;

// Device operators / preconditioners (krylov.hpp:13-36)
struct DOp {
    virtual ~DOp() = default;
    virtual int64_t size() const = 0;
    virtual void apply(const double* x, double* y) = 0;
};
struct DPrec {
    virtual ~DPrec() = default;
    virtual void apply(const double* r, double* z) = 0;
};

// Lazily grown GMRES workspace (basis vectors are cached across solves).
struct KrylovWs {
    int64_t n = 0;
    std::vector<DevArray<double>> V, Z;
    std::vector<double*> hV, hZ;
    DevArray<double*> dV, dZ;
    DevArray<double> r, w, t, hcol, corr, ycoef, scal;
    void ensure_n(int64_t nn);
    double* v(int j);
    double* z(int j);
    void sync_ptrs(cudaStream_t s);
    size_t bytes() const;
};

SolveRes gmres_dev(Ctx& c, DOp& op, DPrec* M, const double* b, double* x, const KrylovCfg& cfg, bool flexible,
                   KrylovWs& ws);

// Device AMG hierarchy (levels from the host setup, fine level = caller's A).
struct DevLevel {
    const Bsr* A = nullptr; // level operator (fine: borrowed)
    Bsr Aown, P, R;
    DevArray<double> invd, r, z, s; // r/z for coarse levels, s scratch
    DevArray<double> gdense;         // sweep auxiliary data (sweep_prepare: group T^-1 / push packed blocks)
    int n = 0;
};
struct DevHierarchy {
    AmgOpts opts;
    bool fallback = false;
    DevArray<double> fb_invd;
    std::vector<DevLevel> lv;
    DevArray<double> pinv;
    int nc = 0;
    // collapsed coarse tail (dense_tail.cu): the last entry of lv is level
    // `tail`, whose whole sub-V-cycle is the dense row-major operator vtail
    int tail = -1;
    DevArray<double> vtail;
    std::vector<int> level_rows; // scalar rows of every level of the full hierarchy
    double setup_host_ms = 0.0;
    // s: stream the build is ordered on (null: c.stream)
    void build(Ctx& c, const Bsr& A0, const AmgOpts& o, cudaStream_t s = nullptr);
    void vcycle(Ctx& c, const double* r, double* z);
    void cycle(Ctx& c, int l, const double* r, double* z);
    void smooth(Ctx& c, int l, const double* b, double* z, int sweeps);
    int n_levels() const { return static_cast<int>(level_rows.size()); }
};

// Working (scaled) copy of the system and everything solve_block_system builds.
struct WorkSys {
    int Bv = 3, nv = 0, np = 0;
    Bsr A, B, C, D, S;
    CoupledOp K; // the same system as one 4x4 BSR (mesh-assembled systems; n_nodes 0 otherwise)
    DevArray<double> w; // scaling weights (nv + np)
    bool scaled = false;
};
struct StreamOwner {
    cudaStream_t s = nullptr;
    ~StreamOwner()
    {
        if (s) {
            cudaStreamSynchronize(s);
            cache_release_stream(s);
            cudaStreamDestroy(s);
        }
    }
};
struct Ctx {
    StreamOwner owner;  // first members: destroyed after every stream-ordered array
    StreamOwner owner2, owner3, owner4;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr; // the S_hat hierarchy is built on it, concurrently with A's
    cudaStream_t stream3 = nullptr, stream4 = nullptr; // dense-tail builds of the A / S_hat hierarchies
    std::string err;
    Reducer red;
    double* pinned = nullptr; // host staging for small D2H reads
    size_t pinned_n = 0;

    // mesh / dofs
    bool have_mesh = false, have_dofs = false, have_mat = false;
    int n_nodes = 0, n_tets = 0;
    DevArray<int> tets;
    DevArray<double> grad_n, volume, tau;
    std::vector<int> h_tets;
    int nfree = 0;
    std::vector<int> fidx, fnode; // node -> free index; free index -> node
    DevArray<int> d_fidx, d_fnode;
    // assembly structures
    BlockPattern PN; // node graph
    DevArray<int> k4slot, elem_order;
    std::vector<int> color_ptr;
    DevArray<double> k4;
    DevArray<int> srcA, srcB, srcC, srcD;
    DevArray<int> dstA, dstB, dstC, dstD; // inverse maps: stored block of each K4 slot per plane (-1: none)
    DevArray<int2> k44_cf;                // per node-graph block {column node, its free index} (coupled SpMV)
    ed_material mat{};
    DevArray<double> elem_h; // [E][2][9] per-element fibre structure tensors (empty: the material's global ones)
    // prescribed end-of-step displacement of fully fixed nodes, consumed by the next time step
    DevArray<int> pd_nodes;
    DevArray<double> pd_u;
    int pd_n = 0;
    double body_force[3] = {0.0, 0.0, 0.0};
    DevArray<int64_t> tr_rowptr;
    DevArray<int> tr_rows;
    DevArray<double> tr_vals;
    int tr_n = 0;
    // state (current) + Newton stage copies
    DevArray<double> u, udot, p, pdot, v, vdot;
    DevArray<double> m_u, m_udot, m_p, m_pdot, m_v, m_vdot; // stage state
    DevArray<double> rm, rp, fv, fp, rk, rhs, xsol;
    DevArray<double> s_u, s_udot, s_p, s_pdot, s_v, s_vdot; // saved state (benchmarks)
    DevArray<double> y_u, y_udot, y_p, y_pdot, y_v, y_vdot; // y_n of a time step
    DevArray<double> q_u, q_udot, q_p, q_pdot, q_v, q_vdot; // iterate before the last update (halving guard)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    DevArray<int> dscratch_i; // [0] bad element, [1] bad row
    // system
    BlockSys sys;                 // assembled or uploaded (unscaled)
    bool sys_from_mesh = false;   // planes come from K4 (mesh) or from CSR upload
    bool sys_values = false;
    std::vector<HostCsr> csr_up;  // uploaded CSR blocks (A, B, C, D)
    int csr_bv = -1;              // Bv the planes were last built with from csr_up
    // solver working set
    WorkSys work;
    // level-operator structures of the previous hierarchy builds ([A, S_hat][level]), reused on identical patterns
    LevelCache lcache[2][16];
    KrylovWs ws_outer, ws_a, ws_s;
    // timings of the last newton pass
    ed_phase_times times{};

    explicit Ctx(int dev);
    ~Ctx();
    double* host_buf(size_t n);
    void sync();
    int read_int(const int* d);
};

// system setup (system.cpp)
void ctx_build_mesh_system(Ctx& c);  // patterns, layouts, K4 maps, colouring
void ctx_planes_from_k4(Ctx& c);     // K4 -> sys planes
void ctx_planes_from_csr(Ctx& c, int Bv);

void make_work(Ctx& c, WorkSys& W, bool scale, double eps_diag);
void build_shat_work(Ctx& c, WorkSys& W);

AmgOpts amg_opts_from(const ed_amg_options& o, const Ctx& c, bool velocity, int nrows);

// solve_block_system on device vectors (precond.cpp:157-218)
Stats solve_block_system_dev(Ctx& c, const double* d_rhs, double* d_x, const ed_block_solver_options& o,
                             std::vector<double>* history, ed_phase_times* times);

double now_ms();

} // namespace edb

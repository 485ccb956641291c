// ORACLE TEST INFRASTRUCTURE -- not product code.  Only tests/, bench.py's
// cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load it.
//
// A thin C-ABI harness around the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It builds
// the BASELINE cube problems through the reference's public API and exposes
// the hot-path calls to ctypes:
//   * generate_cube_mesh / DofMap::build / make_neo_hookean_material /
//     compute_tau / retag_facets            (mesh.cpp, assembly.cpp, materials.cpp)
//   * assemble_residuals / assemble_tangent  (assembly.cpp:113-363)
//   * solve_block_system, recomposed from its public parts so the outer
//     FGMRES residual history is visible    (precond.cpp:157-218)
//   * the first corrector pass of step_generalized_alpha (timeint.cpp:79-176)
//   * gmres / fgmres / AmgHierarchy / build_shat on caller-provided CSR
//     matrices (random-system parity tests; krylov.cpp, amg.cpp, precond.cpp)
// The struct layouts below mirror include/elastodyn_b200.h so that Python can
// pass one ctypes struct to both sides.
#include "elastodyn/amg.hpp"
#include "elastodyn/assembly.hpp"
#include "elastodyn/blocksystem.hpp"
#include "elastodyn/krylov.hpp"
#include "elastodyn/materials.hpp"
#include "elastodyn/mesh.hpp"
#include "elastodyn/precond.hpp"
#include "elastodyn/timeint.hpp"

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

using namespace elastodyn;

extern "C" {

typedef struct {
    int32_t restart;
    int32_t max_iters;
    double rel_tol;
    double abs_tol;
} orc_krylov_config;

typedef struct {
    int32_t block_size;
    int32_t max_levels;
    int32_t coarse_max_rows;
    int32_t smoother; // 0 = Jacobi, 1 = symmetric Gauss-Seidel
    int32_t pre_sweeps;
    int32_t post_sweeps;
    int32_t smooth_prolongator;
    int32_t use_dof_row_maps; // 1: row_to_node/row_component from the DofMap (driver.cpp:32-48)
    double strength_theta;
    double jacobi_weight;
} orc_amg_options;

typedef struct {
    int32_t precond; // 0 nested, 1 simple, 2 ilu0, 3 jacobi, 4 none (PrecondKind order)
    int32_t scale;
    orc_krylov_config outer, a, s, inner;
    orc_amg_options amg_a, amg_s;
    double eps_diag;
} orc_solver_options;

typedef struct {
    int64_t outer_iters, a_solves, a_iters, s_solves, s_iters, schur_applies, inner_iters;
    int32_t converged;
    int32_t pad;
    double t_solve;
} orc_linear_stats;

typedef struct {
    int32_t n;               // cells per edge
    int32_t incompressible;  // IncompressibleVolumetric when 1
    int32_t material;        // 0 Neo-Hookean, 1 dispersed fibre
    int32_t pad;
    double edge;             // cube edge length
    double mu, kappa, rho0, c_m;
    double k1, k2, kd, phi_deg; // fibre material
    double load;             // traction magnitude (pointing -z) on the top central quarter
    double dt, rho_inf;
    double body_force[3];
} orc_problem_params;

} // extern "C"

namespace {

std::string g_err;

KrylovConfig kc(const orc_krylov_config& c) { return KrylovConfig{c.restart, c.max_iters, c.rel_tol, c.abs_tol}; }

AmgOptions amg_opts(const orc_amg_options& o, const DofMap* dofs)
{
    AmgOptions a;
    a.block_size = o.block_size;
    a.strength_theta = o.strength_theta;
    a.max_levels = o.max_levels;
    a.coarse_max_rows = o.coarse_max_rows;
    a.smoother = o.smoother == 0 ? AmgOptions::Smoother::Jacobi
                                 : AmgOptions::Smoother::SymmetricGaussSeidel;
    a.jacobi_weight = o.jacobi_weight;
    a.pre_sweeps = o.pre_sweeps;
    a.post_sweeps = o.post_sweeps;
    a.smooth_prolongator = o.smooth_prolongator != 0;
    a.quiet = true;
    if (o.use_dof_row_maps && dofs) {
        // same mapping as set_amg_maps (driver.cpp:32-48)
        a.row_component = dofs->row_comp;
        a.row_to_node.resize(dofs->nv);
        int cur = -1, prev = -1;
        for (int r = 0; r < dofs->nv; ++r) {
            if (dofs->row_node[r] != prev) {
                prev = dofs->row_node[r];
                ++cur;
            }
            a.row_to_node[r] = cur;
        }
    }
    return a;
}

BlockSolverOptions solver_opts(const orc_solver_options& o, const DofMap* dofs)
{
    BlockSolverOptions b;
    b.precond = static_cast<PrecondKind>(o.precond);
    b.outer = kc(o.outer);
    b.scr.a = kc(o.a);
    b.scr.s = kc(o.s);
    b.scr.inner = kc(o.inner);
    b.amg_a = amg_opts(o.amg_a, dofs);
    b.amg_s = amg_opts(o.amg_s, nullptr);
    b.scale = o.scale != 0;
    b.eps_diag = o.eps_diag;
    return b;
}

void fill_stats(const LinearStats& s, orc_linear_stats* out)
{
    if (!out) return;
    out->outer_iters = s.outer_iters;
    out->a_solves = s.a_solves;
    out->a_iters = s.a_iters;
    out->s_solves = s.s_solves;
    out->s_iters = s.s_iters;
    out->schur_applies = s.schur_applies;
    out->inner_iters = s.inner_iters;
    out->converged = s.converged ? 1 : 0;
    out->pad = 0;
    out->t_solve = s.t_solve;
}

CsrMatrix csr_from(int nrows, int ncols, const int* rowptr, const int* col, const double* val)
{
    CsrMatrix m;
    m.nrows = nrows;
    m.ncols = ncols;
    m.rowptr.assign(rowptr, rowptr + nrows + 1);
    const int nnz = rowptr[nrows];
    m.col.assign(col, col + nnz);
    m.val.assign(val, val + nnz);
    return m;
}

// solve_block_system (precond.cpp:157-218) recomposed from the public API so
// the outer SolveResult (and its residual history) can be returned.  Every
// call is the reference's own; only the SolveResult is kept instead of
// being dropped.
LinearStats solve_with_history(const BlockMatrix& K, const std::vector<double>& rhs,
                               std::vector<double>& x, const BlockSolverOptions& opts,
                               SolveResult& res)
{
    const auto t0 = std::chrono::steady_clock::now();
    LinearStats stats;
    BlockMatrix Ks;
    Ks.nv = K.nv;
    Ks.np = K.np;
    Ks.A = K.A;
    Ks.B = K.B;
    Ks.C = K.C;
    Ks.D = K.D;
    std::vector<double> b = rhs;
    BlockScaling sc;
    if (opts.scale) {
        sc = compute_block_scaling(Ks, opts.eps_diag);
        scale_system(Ks, sc);
        scale_vector(b, sc);
    }
    x.assign(b.size(), 0.0);
    BlockOperator op(Ks);
    switch (opts.precond) {
    case PrecondKind::Nested: {
        ScrSolver scr(Ks, opts.scr, opts.amg_a, opts.amg_s);
        NestedPrecond M(scr, Ks.nv, Ks.np, stats);
        res = fgmres(op, &M, b, x, opts.outer);
        break;
    }
    case PrecondKind::Simple: {
        SimplePrecond M(Ks, opts.scr, opts.amg_a, opts.amg_s, stats);
        res = fgmres(op, &M, b, x, opts.outer);
        break;
    }
    case PrecondKind::Ilu0: {
        const CsrMatrix mono = monolithic_csr(Ks);
        Ilu0Precond M(mono);
        res = gmres(op, &M, b, x, opts.outer);
        break;
    }
    case PrecondKind::Jacobi: {
        const CsrMatrix mono = monolithic_csr(Ks);
        JacobiPrecond M(mono);
        res = gmres(op, &M, b, x, opts.outer);
        break;
    }
    case PrecondKind::None:
        res = gmres(op, nullptr, b, x, opts.outer);
        break;
    }
    if (opts.scale) scale_vector(x, sc);
    stats.outer_iters = res.iterations;
    stats.converged = res.converged;
    stats.t_solve = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return stats;
}

void copy_history(const SolveResult& res, double* hist, int cap, int* len)
{
    if (len) *len = static_cast<int>(res.history.size());
    if (hist)
        for (int i = 0; i < cap && i < static_cast<int>(res.history.size()); ++i) hist[i] = res.history[i];
}

double now_s(std::chrono::steady_clock::time_point t0)
{
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct Problem {
    orc_problem_params prm{};
    Mesh mesh;
    DofMap dofs;
    Material mat;
    StabilizationParams stab;
    Loads loads;
    GenAlphaParams ga;
    State state;
    std::unique_ptr<TangentBlocks> tangent;
    int load_tag = -1;
};

} // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

void* orc_problem_create(const orc_problem_params* p)
{
    try {
        auto P = std::make_unique<Problem>();
        P->prm = *p;
        const double L = p->edge;
        P->mesh = generate_cube_mesh(p->n, L);
        const double tol = 1e-9 * L;
        std::vector<std::array<bool, 3>> fixed(P->mesh.n_nodes(), {false, false, false});
        for (int n = 0; n < P->mesh.n_nodes(); ++n)
            if (P->mesh.nodes[n][2] < tol) fixed[n] = {true, true, true};
        P->dofs = DofMap::build(P->mesh, fixed);
        if (p->material == 1) {
            P->mat = make_fiber_material(p->mu, p->k1, p->k2, p->kd, p->phi_deg, p->rho0);
            if (!p->incompressible) {
                P->mat.vol = std::make_unique<CompressibleVolumetric>(p->rho0, p->kappa);
                P->mat.kappa = p->kappa;
                P->mat.incompressible = false;
            }
        } else if (p->incompressible) {
            Material m;
            m.vol = std::make_unique<IncompressibleVolumetric>(p->rho0);
            m.iso = std::make_unique<NeoHookeanIsochoric>(p->mu);
            m.rho0 = p->rho0;
            m.mu = p->mu;
            m.incompressible = true;
            P->mat = std::move(m);
        } else {
            P->mat = make_neo_hookean_material(p->mu, p->kappa, p->rho0);
        }
        P->stab = compute_tau(P->mesh, P->mat, p->c_m);
        const int zmax = P->mesh.tag_id("zmax");
        P->mesh.retag_facets(
            zmax,
            [&](const Vec3& c) {
                return c[0] >= 0.25 * L - tol && c[0] <= 0.75 * L + tol && c[1] >= 0.25 * L - tol &&
                       c[1] <= 0.75 * L + tol;
            },
            "top_load");
        P->load_tag = P->mesh.tag_id("top_load");
        P->loads.body_force = {p->body_force[0], p->body_force[1], p->body_force[2]};
        if (p->load != 0.0) P->loads.tractions.push_back({P->load_tag, {0.0, 0.0, -p->load}});
        P->ga = gen_alpha_params(p->rho_inf, p->dt);
        P->state = State::zeros(P->mesh.n_nodes());
        return P.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void orc_problem_destroy(void* h) { delete static_cast<Problem*>(h); }

// sizes[0..5] = n_nodes, n_tets, nv, np, n_loaded_facets, n_facets
void orc_problem_sizes(void* h, int* sizes)
{
    auto* P = static_cast<Problem*>(h);
    sizes[0] = P->mesh.n_nodes();
    sizes[1] = P->mesh.n_tets();
    sizes[2] = P->dofs.nv;
    sizes[3] = P->dofs.np;
    sizes[4] = static_cast<int>(P->mesh.facets_with_tag(P->load_tag).size());
    sizes[5] = static_cast<int>(P->mesh.facets.size());
}

// Exports the mesh exactly as the reference built it (any array may be null).
void orc_mesh_export(void* h, double* coords, int* tets, double* volume, double* hsize,
                     double* grad_n, double* tau, int* vdof)
{
    auto* P = static_cast<Problem*>(h);
    const Mesh& m = P->mesh;
    for (int n = 0; n < m.n_nodes(); ++n)
        for (int i = 0; i < 3; ++i) {
            if (coords) coords[3 * n + i] = m.nodes[n][i];
            if (vdof) vdof[3 * n + i] = P->dofs.vdof[n][i];
        }
    for (int e = 0; e < m.n_tets(); ++e) {
        for (int a = 0; a < 4; ++a) {
            if (tets) tets[4 * e + a] = m.tets[e][a];
            for (int I = 0; I < 3; ++I)
                if (grad_n) grad_n[12 * e + 3 * a + I] = m.grad_N[e][a][I];
        }
        if (volume) volume[e] = m.volume[e];
        if (hsize) hsize[e] = m.h[e];
        if (tau) tau[e] = P->stab.tau[e];
    }
}

// Loaded facets (top central quarter): node triples and facet_area/3 each.
void orc_loaded_facets(void* h, int* nodes, double* third)
{
    auto* P = static_cast<Problem*>(h);
    int k = 0;
    for (int fi : P->mesh.facets_with_tag(P->load_tag)) {
        const BoundaryFacet& f = P->mesh.facets[fi];
        for (int a = 0; a < 3; ++a) nodes[3 * k + a] = f.nodes[a];
        third[k] = P->mesh.facet_area(f) / 3.0;
        ++k;
    }
}

void orc_set_state(void* h, const double* u, const double* udot, const double* p,
                   const double* pdot, const double* v, const double* vdot)
{
    auto* P = static_cast<Problem*>(h);
    const int N = P->mesh.n_nodes();
    P->state.u.assign(u, u + 3 * N);
    P->state.udot.assign(udot, udot + 3 * N);
    P->state.p.assign(p, p + N);
    P->state.pdot.assign(pdot, pdot + N);
    P->state.v.assign(v, v + 3 * N);
    P->state.vdot.assign(vdot, vdot + 3 * N);
}

void orc_get_state(void* h, double* u, double* udot, double* p, double* pdot, double* v,
                   double* vdot)
{
    auto* P = static_cast<Problem*>(h);
    std::copy(P->state.u.begin(), P->state.u.end(), u);
    std::copy(P->state.udot.begin(), P->state.udot.end(), udot);
    std::copy(P->state.p.begin(), P->state.p.end(), p);
    std::copy(P->state.pdot.begin(), P->state.pdot.end(), pdot);
    std::copy(P->state.v.begin(), P->state.v.end(), v);
    std::copy(P->state.vdot.begin(), P->state.vdot.end(), vdot);
}

// assemble_residuals at the stored state.  Returns 0, or 1 on ElementInversion.
int orc_assemble_residuals(void* h, double* rm, double* rp, double* seconds)
{
    auto* P = static_cast<Problem*>(h);
    std::vector<double> vm, vp;
    const auto t0 = std::chrono::steady_clock::now();
    try {
        assemble_residuals(P->mesh, P->dofs, P->mat, P->stab, P->loads, P->state, vm, vp);
    } catch (const ElementInversion& e) {
        g_err = e.what();
        return 1;
    }
    if (seconds) *seconds = now_s(t0);
    std::copy(vm.begin(), vm.end(), rm);
    std::copy(vp.begin(), vp.end(), rp);
    return 0;
}

// assemble_tangent at the stored state with the problem's TimeScalars (or the
// given ones when ts != null: {dt, alpha_m, alpha_f, gamma}).
int orc_assemble_tangent(void* h, const double* ts_in, double* seconds)
{
    auto* P = static_cast<Problem*>(h);
    TimeScalars ts = P->ga.scalars();
    if (ts_in) ts = TimeScalars{ts_in[0], ts_in[1], ts_in[2], ts_in[3]};
    const auto t0 = std::chrono::steady_clock::now();
    try {
        P->tangent = std::make_unique<TangentBlocks>(
            assemble_tangent(P->mesh, P->dofs, P->mat, P->stab, P->loads, P->state, ts));
    } catch (const ElementInversion& e) {
        g_err = e.what();
        return 1;
    }
    if (seconds) *seconds = now_s(t0);
    return 0;
}

static const CsrMatrix* tangent_plane(Problem* P, int which)
{
    if (!P->tangent) return nullptr;
    switch (which) {
    case 0: return &P->tangent->K.A;
    case 1: return &P->tangent->K.B;
    case 2: return &P->tangent->K.C;
    case 3: return &P->tangent->K.D;
    case 4: return &P->tangent->A_rate;
    case 5: return &P->tangent->C_rate;
    }
    return nullptr;
}

// dims[0..2] = nrows, ncols, nnz
int orc_tangent_dims(void* h, int which, int* dims)
{
    const CsrMatrix* m = tangent_plane(static_cast<Problem*>(h), which);
    if (!m) return 1;
    dims[0] = m->nrows;
    dims[1] = m->ncols;
    dims[2] = static_cast<int>(m->nnz());
    return 0;
}

int orc_tangent_export(void* h, int which, int* rowptr, int* col, double* val)
{
    const CsrMatrix* m = tangent_plane(static_cast<Problem*>(h), which);
    if (!m) return 1;
    std::copy(m->rowptr.begin(), m->rowptr.end(), rowptr);
    std::copy(m->col.begin(), m->col.end(), col);
    std::copy(m->val.begin(), m->val.end(), val);
    return 0;
}

// solve_block_system on the stored tangent K with the given rhs (n = nv+np).
int orc_solve_tangent(void* h, const double* rhs, const orc_solver_options* o, double* x,
                      orc_linear_stats* st, double* hist, int hist_cap, int* hist_len)
{
    auto* P = static_cast<Problem*>(h);
    if (!P->tangent) return 1;
    try {
        const int n = P->dofs.nv + P->dofs.np;
        std::vector<double> b(rhs, rhs + n), xv;
        SolveResult res;
        const LinearStats ls = solve_with_history(P->tangent->K, b, xv, solver_opts(*o, &P->dofs), res);
        std::copy(xv.begin(), xv.end(), x);
        fill_stats(ls, st);
        copy_history(res, hist, hist_cap, hist_len);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
    return 0;
}

// The first corrector pass of step_generalized_alpha (timeint.cpp:54-176)
// from the stored state y_n: predictor, stage blend, residual, kinematic
// residual rk, norm, tangent, RHS fold-in, solve, two-stage update.  The
// stored state becomes the updated iterate.  out_norm[0] = ||R||.
// times[0..3] = residual, tangent, fold-in, solve seconds.
int orc_newton_first_pass(void* h, const orc_solver_options* o, double* x_out, double* rhs_out,
                          double* out_norm, orc_linear_stats* st, double* hist, int hist_cap,
                          int* hist_len, double* times)
{
    auto* P = static_cast<Problem*>(h);
    try {
        const GenAlphaParams& ga = P->ga;
        const TimeScalars ts = ga.scalars();
        const double chi = ts.chi();
        const double gdt = ga.gamma * ga.dt;
        const DofMap& dofs = P->dofs;
        const State yn = P->state;
        State cur = P->state;
        const double pf = (ga.gamma - 1.0) / ga.gamma;
        for (auto& v : cur.udot) v *= pf;
        for (auto& v : cur.pdot) v *= pf;
        for (auto& v : cur.vdot) v *= pf;
        auto blend = [](const std::vector<double>& a, const std::vector<double>& b, double w,
                        std::vector<double>& out) {
            out.resize(a.size());
            for (std::size_t i = 0; i < a.size(); ++i) out[i] = a[i] + w * (b[i] - a[i]);
        };
        State mid;
        blend(yn.udot, cur.udot, ga.alpha_m, mid.udot);
        blend(yn.pdot, cur.pdot, ga.alpha_m, mid.pdot);
        blend(yn.vdot, cur.vdot, ga.alpha_m, mid.vdot);
        blend(yn.u, cur.u, ga.alpha_f, mid.u);
        blend(yn.p, cur.p, ga.alpha_f, mid.p);
        blend(yn.v, cur.v, ga.alpha_f, mid.v);

        std::vector<double> rm, rp, rk(dofs.nv);
        auto t0 = std::chrono::steady_clock::now();
        assemble_residuals(P->mesh, dofs, P->mat, P->stab, P->loads, mid, rm, rp);
        if (times) times[0] = now_s(t0);
        for (int r = 0; r < dofs.nv; ++r) {
            const int idx = 3 * dofs.row_node[r] + dofs.row_comp[r];
            rk[r] = mid.udot[idx] - mid.v[idx];
        }
        const double norm = std::sqrt(vec_dot(rk, rk) + vec_dot(rp, rp) + vec_dot(rm, rm));
        if (out_norm) *out_norm = norm;

        t0 = std::chrono::steady_clock::now();
        P->tangent = std::make_unique<TangentBlocks>(
            assemble_tangent(P->mesh, dofs, P->mat, P->stab, P->loads, mid, ts));
        if (times) times[1] = now_s(t0);
        const TangentBlocks& tb = *P->tangent;

        t0 = std::chrono::steady_clock::now();
        std::vector<double> rhs(dofs.nv + dofs.np);
        std::vector<double> w1(dofs.nv), w2(dofs.nv), wp1(dofs.np), wp2(dofs.np);
        tb.K.A.matvec(rk.data(), w1.data());
        tb.A_rate.matvec(rk.data(), w2.data());
        for (int i = 0; i < dofs.nv; ++i) rhs[i] = -rm[i] + (w1[i] - w2[i]) / chi;
        tb.K.C.matvec(rk.data(), wp1.data());
        tb.C_rate.matvec(rk.data(), wp2.data());
        for (int i = 0; i < dofs.np; ++i) rhs[dofs.nv + i] = -rp[i] + (wp1[i] - wp2[i]) / chi;
        if (times) times[2] = now_s(t0);
        if (rhs_out) std::copy(rhs.begin(), rhs.end(), rhs_out);

        t0 = std::chrono::steady_clock::now();
        std::vector<double> x;
        SolveResult res;
        const LinearStats ls = solve_with_history(tb.K, rhs, x, solver_opts(*o, &dofs), res);
        if (times) times[3] = now_s(t0);
        fill_stats(ls, st);
        copy_history(res, hist, hist_cap, hist_len);
        if (x_out) std::copy(x.begin(), x.end(), x_out);

        for (int r = 0; r < dofs.nv; ++r) {
            const int idx = 3 * dofs.row_node[r] + dofs.row_comp[r];
            const double dvd = x[r];
            const double dud = (chi / ga.alpha_m) * dvd - rk[r] / ga.alpha_m;
            cur.vdot[idx] += dvd;
            cur.v[idx] += gdt * dvd;
            cur.udot[idx] += dud;
            cur.u[idx] += gdt * dud;
        }
        for (int n = 0; n < dofs.np; ++n) {
            const double dpd = x[dofs.nv + n];
            cur.pdot[n] += dpd;
            cur.p[n] += gdt * dpd;
        }
        P->state = cur;
    } catch (const ElementInversion& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
    return 0;
}

// Full step_generalized_alpha (timeint.cpp:40-182) from the stored state.
// info[0..3] = converged, newton_iters, res_history length; stats accumulate.
int orc_step(void* h, const orc_solver_options* o, double tol_r, double tol_a, int l_max,
             double t_n, int* info, double* res_hist, int res_cap, orc_linear_stats* st,
             double* t_assembly)
{
    auto* P = static_cast<Problem*>(h);
    try {
        TransientProblem tp;
        tp.mesh = &P->mesh;
        tp.dofs = &P->dofs;
        tp.mat = &P->mat;
        tp.stab = P->stab;
        const Loads L = P->loads;
        tp.loads_at = [L](double) { return L; };
        NonlinearConfig nl;
        nl.tol_R = tol_r;
        nl.tol_A = tol_a;
        nl.l_max = l_max;
        const StepStats s = step_generalized_alpha(tp, P->ga, nl, solver_opts(*o, &P->dofs), t_n, P->state);
        info[0] = s.converged ? 1 : 0;
        info[1] = s.newton_iters;
        info[2] = static_cast<int>(s.res_history.size());
        for (int i = 0; i < res_cap && i < static_cast<int>(s.res_history.size()); ++i)
            res_hist[i] = s.res_history[i];
        fill_stats(s.linear, st);
        if (t_assembly) *t_assembly = s.t_assembly;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// Generic CSR entry points (random-system parity tests).

// solve_block_system on caller CSR blocks.
int orc_solve_block_csr(int nv, int np, const int* a_rp, const int* a_c, const double* a_v,
                        const int* b_rp, const int* b_c, const double* b_v, const int* c_rp,
                        const int* c_c, const double* c_v, const int* d_rp, const int* d_c,
                        const double* d_v, const double* rhs, const orc_solver_options* o,
                        double* x, orc_linear_stats* st, double* hist, int hist_cap,
                        int* hist_len)
{
    try {
        BlockMatrix K;
        K.nv = nv;
        K.np = np;
        K.A = csr_from(nv, nv, a_rp, a_c, a_v);
        K.B = csr_from(nv, np, b_rp, b_c, b_v);
        K.C = csr_from(np, nv, c_rp, c_c, c_v);
        K.D = csr_from(np, np, d_rp, d_c, d_v);
        std::vector<double> b(rhs, rhs + nv + np), xv;
        SolveResult res;
        const LinearStats ls = solve_with_history(K, b, xv, solver_opts(*o, nullptr), res);
        std::copy(xv.begin(), xv.end(), x);
        fill_stats(ls, st);
        copy_history(res, hist, hist_cap, hist_len);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
    return 0;
}

// gmres/fgmres on a CSR matrix.  precond: 0 none, 1 Jacobi, 2 AMG(opts).
// res_out[0..3] = converged, iterations, initial_norm, final_norm.
int orc_gmres_csr(int n, const int* rp, const int* c, const double* v, const double* b,
                  double* x, const orc_krylov_config* cfg, int flexible, int precond,
                  const orc_amg_options* amg, double* res_out, double* hist, int hist_cap,
                  int* hist_len)
{
    try {
        const CsrMatrix A = csr_from(n, n, rp, c, v);
        CsrOperator op(A);
        std::unique_ptr<Preconditioner> M;
        if (precond == 1) M = std::make_unique<JacobiPrecond>(A);
        if (precond == 2) M = std::make_unique<AmgPrecond>(A, amg_opts(*amg, nullptr));
        std::vector<double> bv(b, b + n), xv(x, x + n);
        const SolveResult r = flexible ? fgmres(op, M.get(), bv, xv, kc(*cfg))
                                       : gmres(op, M.get(), bv, xv, kc(*cfg));
        std::copy(xv.begin(), xv.end(), x);
        res_out[0] = r.converged ? 1.0 : 0.0;
        res_out[1] = r.iterations;
        res_out[2] = r.initial_norm;
        res_out[3] = r.final_norm;
        copy_history(r, hist, hist_cap, hist_len);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
    return 0;
}

// AmgHierarchy::build + one vcycle.  info[0] = n_levels, info[1] = fallback,
// info[2..] = level rows (up to 16 levels).
int orc_amg_vcycle_csr(int n, const int* rp, const int* c, const double* v,
                       const orc_amg_options* amg, const int* row_to_node, const int* row_comp,
                       const double* r, double* z, int* info)
{
    try {
        const CsrMatrix A = csr_from(n, n, rp, c, v);
        AmgOptions o = amg_opts(*amg, nullptr);
        if (row_to_node) {
            o.row_to_node.assign(row_to_node, row_to_node + n);
            o.row_component.assign(row_comp, row_comp + n);
        }
        const AmgHierarchy hier = AmgHierarchy::build(A, o);
        hier.vcycle(r, z);
        info[0] = hier.n_levels();
        info[1] = hier.diagonal_fallback() ? 1 : 0;
        for (int l = 0; l < hier.n_levels() && l < 16; ++l) info[2 + l] = hier.level_rows(l);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
    return 0;
}

// build_shat on caller blocks (precond.cpp:10-24).  Two-phase: call with
// out_* == null to get nnz in dims[0], then again with buffers.
int orc_build_shat(int nv, int np, const int* a_rp, const int* a_c, const double* a_v,
                   const int* b_rp, const int* b_c, const double* b_v, const int* c_rp,
                   const int* c_c, const double* c_v, const int* d_rp, const int* d_c,
                   const double* d_v, int* dims, int* out_rp, int* out_c, double* out_v)
{
    try {
        BlockMatrix K;
        K.nv = nv;
        K.np = np;
        K.A = csr_from(nv, nv, a_rp, a_c, a_v);
        K.B = csr_from(nv, np, b_rp, b_c, b_v);
        K.C = csr_from(np, nv, c_rp, c_c, c_v);
        K.D = csr_from(np, np, d_rp, d_c, d_v);
        const CsrMatrix S = build_shat(K);
        dims[0] = static_cast<int>(S.nnz());
        if (out_rp) {
            std::copy(S.rowptr.begin(), S.rowptr.end(), out_rp);
            std::copy(S.col.begin(), S.col.end(), out_c);
            std::copy(S.val.begin(), S.val.end(), out_v);
        }
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
    return 0;
}

} // extern "C"

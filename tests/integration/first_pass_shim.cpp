// INTEGRATION TEST -- the reference-side C++ binding of INTEGRATION.md,
// compiled against the reference's own headers (/root/reference/proj/include)
// and linked against the reference library (oracle/_ref) and ours.
//
// A reference-shaped caller builds BASELINE configs[0] with the reference API
// (generate_cube_mesh, DofMap::build, make_neo_hookean_material, compute_tau,
// retag_facets), then does one corrector pass from a seeded stage state twice:
//   reference: assemble_residuals / assemble_tangent / solve_block_system
//   GPU:       the shim (include/elastodyn_b200.hpp): upload_problem,
//              upload_state, assemble_residuals, assemble_tangent(rk) +
//              ed_foldin_download, solve_block_system
// and compares R_m, R_p, the fold-in right-hand side and the solution.
// Exit code 0 = agreement; 2 = no CUDA device (the CPU suite only builds it).
#include <elastodyn/assembly.hpp>
#include <elastodyn/blocksystem.hpp>
#include <elastodyn/materials.hpp>
#include <elastodyn/mesh.hpp>
#include <elastodyn/precond.hpp>
#include <elastodyn/timeint.hpp>

#include <cmath>
#include <cstdio>
#include <cstdint>
#include <vector>

#include "elastodyn_b200.hpp"

using namespace elastodyn;
namespace gpu = elastodyn_b200;

static double rel(const std::vector<double>& a, const std::vector<double>& b)
{
    double d = 0.0, n = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        d += (a[i] - b[i]) * (a[i] - b[i]);
        n += b[i] * b[i];
    }
    return std::sqrt(d / (n > 0 ? n : 1.0));
}

static double next_uniform(uint64_t& s, double lo, double hi)
{
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return lo + (hi - lo) * static_cast<double>(z >> 11) * 0x1.0p-53;
}

int main()
{
    ed_ctx* probe = nullptr;
    if (ed_ctx_create(0, &probe) != ED_OK) {
        std::printf("no CUDA device: built only\n");
        return 2;
    }
    ed_ctx_destroy(probe);

    const int n = 10;
    const double L = 1.0, tol = 1e-9;
    Mesh mesh = generate_cube_mesh(n, L);
    std::vector<std::array<bool, 3>> fixed(mesh.n_nodes(), {false, false, false});
    for (int i = 0; i < mesh.n_nodes(); ++i)
        if (mesh.nodes[i][2] < tol) fixed[i] = {true, true, true};
    const DofMap dofs = DofMap::build(mesh, fixed);
    const double mu = 3.0e4, rho0 = 1.0e3, nu = 0.4;
    const double kappa = 2.0 * mu * (1.0 + nu) / (3.0 * (1.0 - 2.0 * nu));
    const Material mat = make_neo_hookean_material(mu, kappa, rho0);
    const StabilizationParams stab = compute_tau(mesh, mat, 1e-3);
    const int zmax = mesh.tag_id("zmax");
    mesh.retag_facets(
        zmax, [&](const Vec3& c) { return c[0] >= 0.25 - tol && c[0] <= 0.75 + tol && c[1] >= 0.25 - tol && c[1] <= 0.75 + tol; },
        "top_load");
    Loads loads;
    loads.tractions.push_back({mesh.tag_id("top_load"), {0.0, 0.0, -1.0e3}});
    const GenAlphaParams ga = gen_alpha_params(0.5, 1e-3);
    const TimeScalars ts = ga.scalars();
    const double chi = ts.chi();

    // a seeded stage state with nonzero rates (fixed components zero)
    State mid = State::zeros(mesh.n_nodes());
    uint64_t seed = 0x1809063500ULL;
    for (int i = 0; i < 3 * mesh.n_nodes(); ++i) {
        const bool fx = fixed[i / 3][i % 3];
        mid.u[i] = fx ? 0.0 : next_uniform(seed, -1e-3, 1e-3);
        mid.v[i] = fx ? 0.0 : next_uniform(seed, -1e-3, 1e-3);
        mid.udot[i] = fx ? 0.0 : next_uniform(seed, -1e-2, 1e-2);
        mid.vdot[i] = fx ? 0.0 : next_uniform(seed, -1e-1, 1e-1);
    }
    for (int i = 0; i < mesh.n_nodes(); ++i) {
        mid.p[i] = next_uniform(seed, -1e2, 1e2);
        mid.pdot[i] = next_uniform(seed, -1e3, 1e3);
    }
    std::vector<double> rk(dofs.nv);
    for (int r = 0; r < dofs.nv; ++r) {
        const int idx = 3 * dofs.row_node[r] + dofs.row_comp[r];
        rk[r] = mid.udot[idx] - mid.v[idx];
    }

    BlockSolverOptions opts;
    opts.scr.a = {500, 500, 1e-2, 1e-50};
    opts.scr.s = {200, 200, 1e-2, 1e-50};
    opts.scr.inner = {500, 500, 1e-2, 1e-50};
    opts.amg_a.block_size = 3;
    opts.amg_a.row_to_node.resize(dofs.nv);
    opts.amg_a.row_component.resize(dofs.nv);
    for (int r = 0; r < dofs.nv; ++r) { // set_amg_maps (driver.cpp:32-48): compressed free nodes
        opts.amg_a.row_to_node[r] = r / 3;
        opts.amg_a.row_component[r] = dofs.row_comp[r];
    }
    opts.amg_a.quiet = opts.amg_s.quiet = true;

    // ---- reference
    std::vector<double> rm, rp;
    assemble_residuals(mesh, dofs, mat, stab, loads, mid, rm, rp);
    const TangentBlocks tb = assemble_tangent(mesh, dofs, mat, stab, loads, mid, ts);
    std::vector<double> rhs(dofs.nv + dofs.np), w1(dofs.nv), w2(dofs.nv), wp1(dofs.np), wp2(dofs.np);
    tb.K.A.matvec(rk.data(), w1.data());
    tb.A_rate.matvec(rk.data(), w2.data());
    tb.K.C.matvec(rk.data(), wp1.data());
    tb.C_rate.matvec(rk.data(), wp2.data());
    for (int i = 0; i < dofs.nv; ++i) rhs[i] = -rm[i] + (w1[i] - w2[i]) / chi;
    for (int i = 0; i < dofs.np; ++i) rhs[dofs.nv + i] = -rp[i] + (wp1[i] - wp2[i]) / chi;
    std::vector<double> x_ref;
    const LinearStats st_ref = solve_block_system(tb.K, rhs, x_ref, opts);

    // ---- GPU through the shim
    gpu::Context ctx(0);
    ed_material mc{};
    mc.kind = 0;
    mc.incompressible = 0;
    mc.rho0 = rho0;
    mc.mu = mu;
    mc.kappa = kappa;
    gpu::upload_problem(ctx, mesh, fixed, mat, mc, stab, loads);
    gpu::upload_state(ctx, mid);
    std::vector<double> rm_g, rp_g;
    gpu::assemble_residuals<ElementInversion>(ctx, dofs.nv, dofs.np, rm_g, rp_g);
    gpu::assemble_tangent<TimeScalars, ElementInversion>(ctx, ts, &rk);
    std::vector<double> fv(dofs.nv), fp(dofs.np), rhs_g(dofs.nv + dofs.np);
    gpu::check(ctx.get(), ed_foldin_download(ctx.get(), fv.data(), fp.data()));
    for (int i = 0; i < dofs.nv; ++i) rhs_g[i] = -rm_g[i] + fv[i] / chi;
    for (int i = 0; i < dofs.np; ++i) rhs_g[dofs.nv + i] = -rp_g[i] + fp[i] / chi;
    ed_block_solver_options o{};
    o.precond = 0;
    o.scale = 1;
    o.outer = gpu::to_c(opts.outer);
    o.a = gpu::to_c(opts.scr.a);
    o.s = gpu::to_c(opts.scr.s);
    o.inner = gpu::to_c(opts.scr.inner);
    o.amg_a = ed_amg_options{3, 12, 200, 1, 1, 1, 1, 1, 0.08, 2.0 / 3.0};
    o.amg_s = ed_amg_options{1, 12, 200, 1, 1, 1, 1, 0, 0.08, 2.0 / 3.0};
    o.eps_diag = opts.eps_diag;
    std::vector<double> x_g;
    const ed_linear_stats st_g = gpu::solve_block_system(ctx, rhs_g, x_g, o);

    const double e_rm = rel(rm_g, rm), e_rp = rel(rp_g, rp), e_rhs = rel(rhs_g, rhs), e_x = rel(x_g, x_ref);
    std::printf("rel err: R_m %.3e R_p %.3e rhs %.3e x %.3e\n", e_rm, e_rp, e_rhs, e_x);
    std::printf("outer %ld/%ld a_iters %ld/%ld s_iters %ld/%ld inner %ld/%ld\n", static_cast<long>(st_g.outer_iters),
                st_ref.outer_iters, static_cast<long>(st_g.a_iters), st_ref.a_iters, static_cast<long>(st_g.s_iters),
                st_ref.s_iters, static_cast<long>(st_g.inner_iters), st_ref.inner_iters);
    const bool ok = e_rm < 1e-12 && e_rp < 1e-12 && e_rhs < 1e-11 && e_x < 1e-8 &&
                    std::abs(st_g.outer_iters - st_ref.outer_iters) <= 1 &&
                    std::abs(st_g.inner_iters - st_ref.inner_iters) <= 1;
    std::printf(ok ? "OK\n" : "MISMATCH\n");
    return ok ? 0 : 1;
}

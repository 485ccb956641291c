// elastodyn_b200.hpp -- reference-shaped C++ shim over the C-ABI
// (include/elastodyn_b200.h).  Header-only.  The templates accept the
// reference's own types by their public fields, so a maintainer can pass
// elastodyn::BlockMatrix, elastodyn::Mesh, elastodyn::State, ... unchanged
// (see INTEGRATION.md).  Errors are re-thrown as the reference's exception
// types: ElementInversionT (materials.hpp:16-19) for J <= 0,
// std::runtime_error for a zero momentum diagonal (precond.cpp:15-17),
// std::invalid_argument for size/option errors (krylov.cpp:26-28).
#pragma once

#include <algorithm>
#include <array>
#include <stdexcept>
#include <string>
#include <vector>

#include "elastodyn_b200.h"

namespace elastodyn_b200 {

template <class ElementInversionT = std::runtime_error>
inline void check(ed_ctx* ctx, int rc)
{
    if (rc == ED_OK) return;
    const std::string msg = ed_last_error(ctx);
    switch (rc) {
    case ED_ELEMENT_INVERSION: throw ElementInversionT(msg);
    case ED_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw std::runtime_error(msg);
    }
}

// RAII context (one GPU, one stream).
class Context {
public:
    explicit Context(int device = 0)
    {
        if (ed_ctx_create(device, &ctx_) != ED_OK)
            throw std::runtime_error("elastodyn_b200: no CUDA device (there is no CPU fallback)");
    }
    ~Context() { ed_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    ed_ctx* get() const { return ctx_; }

private:
    ed_ctx* ctx_ = nullptr;
};

// KrylovConfig (krylov.hpp:64-69) -> ed_krylov_config
template <class KrylovConfigT>
ed_krylov_config to_c(const KrylovConfigT& k)
{
    return ed_krylov_config{k.restart, k.max_iters, k.rel_tol, k.abs_tol};
}

// Mesh + DofMap + Material + StabilizationParams + Loads upload
// (mesh.hpp:24-50, assembly.hpp:17-59).  fixed[n][c] as in DofMap::build.
template <class MeshT, class MaterialT, class StabT, class LoadsT>
void upload_problem(Context& c, const MeshT& mesh, const std::vector<std::array<bool, 3>>& fixed, const MaterialT& mat,
                    const ed_material& mat_c, const StabT& stab, const LoadsT& loads)
{
    (void)mat;
    const int N = static_cast<int>(mesh.nodes.size()), E = static_cast<int>(mesh.tets.size());
    std::vector<int32_t> tets(4 * static_cast<size_t>(E));
    std::vector<double> grad(12 * static_cast<size_t>(E));
    for (int e = 0; e < E; ++e)
        for (int a = 0; a < 4; ++a) {
            tets[4 * e + a] = mesh.tets[e][a];
            for (int I = 0; I < 3; ++I) grad[12 * e + 3 * a + I] = mesh.grad_N[e][a][I];
        }
    check(c.get(), ed_mesh_upload(c.get(), N, E, tets.data(), grad.data(), mesh.volume.data(), stab.tau.data()));
    std::vector<uint8_t> fx(3 * static_cast<size_t>(N));
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < 3; ++k) fx[3 * n + k] = fixed[n][k] ? 1 : 0;
    int32_t nv = 0, np = 0;
    check(c.get(), ed_dofs_build(c.get(), fx.data(), &nv, &np));
    check(c.get(), ed_set_material(c.get(), &mat_c));
    std::vector<int32_t> fnodes;
    std::vector<double> third, h;
    for (const auto& t : loads.tractions)
        for (const int fi : mesh.facets_with_tag(t.tag)) {
            const auto& f = mesh.facets[fi];
            for (int a = 0; a < 3; ++a) fnodes.push_back(f.nodes[a]);
            third.push_back(mesh.facet_area(f) / 3.0);
            for (int i = 0; i < 3; ++i) h.push_back(t.h[i]);
        }
    const double bf[3] = {loads.body_force[0], loads.body_force[1], loads.body_force[2]};
    check(c.get(), ed_set_loads(c.get(), bf, static_cast<int>(third.size()), fnodes.data(), third.data(), h.data()));
}

// State (assembly.hpp:31-37)
template <class StateT>
void upload_state(Context& c, const StateT& s)
{
    check(c.get(), ed_state_upload(c.get(), s.u.data(), s.udot.data(), s.p.data(), s.pdot.data(), s.v.data(),
                                   s.vdot.data()));
}

// assemble_residuals (assembly.hpp:88-90) at the uploaded stage state
template <class ElementInversionT = std::runtime_error>
void assemble_residuals(Context& c, int nv, int np, std::vector<double>& r_m, std::vector<double>& r_p)
{
    r_m.assign(nv, 0.0);
    r_p.assign(np, 0.0);
    int32_t bad = -1;
    check<ElementInversionT>(c.get(), ed_assemble_residuals(c.get(), r_m.data(), r_p.data(), &bad));
}

// assemble_tangent (assembly.hpp:92-94); the blocks stay on the device
template <class TimeScalarsT, class ElementInversionT = std::runtime_error>
void assemble_tangent(Context& c, const TimeScalarsT& ts, const std::vector<double>* rk = nullptr)
{
    const ed_time_scalars t{ts.dt, ts.alpha_m, ts.alpha_f, ts.gamma};
    int32_t bad = -1;
    check<ElementInversionT>(c.get(), ed_assemble_tangent(c.get(), &t, rk ? rk->data() : nullptr, &bad));
}

// BlockMatrix (blocksystem.hpp:19-34) upload: any type with A, B, C, D
// CsrMatrix-like members {rowptr, col, val} and nv, np.
template <class BlockMatrixT>
void upload_block_system(Context& c, const BlockMatrixT& K)
{
    check(c.get(), ed_block_system_upload(c.get(), K.nv, K.np, K.A.rowptr.data(), K.A.col.data(), K.A.val.data(),
                                          K.B.rowptr.data(), K.B.col.data(), K.B.val.data(), K.C.rowptr.data(),
                                          K.C.col.data(), K.C.val.data(), K.D.rowptr.data(), K.D.col.data(),
                                          K.D.val.data()));
}

// solve_block_system (precond.hpp:182-183) on the context's current system
// (assembled on the device or uploaded); x = zero-guess solution.
inline ed_linear_stats solve_block_system(Context& c, const std::vector<double>& rhs, std::vector<double>& x,
                                          const ed_block_solver_options& opts, std::vector<double>* history = nullptr)
{
    x.assign(rhs.size(), 0.0);
    ed_linear_stats st{};
    std::vector<double> h(history ? opts.outer.max_iters + 1 : 0);
    int32_t hl = 0;
    check(c.get(), ed_solve_block_system(c.get(), rhs.data(), x.data(), &opts, &st, history ? h.data() : nullptr,
                                         static_cast<int32_t>(h.size()), &hl));
    if (history) history->assign(h.begin(), h.begin() + std::min<int32_t>(hl, static_cast<int32_t>(h.size())));
    return st;
}

} // namespace elastodyn_b200

// Device-resident Krylov solvers, AMG V-cycle and the nested block
// preconditioner.  Control flow restates krylov.cpp:21-176 (GMRES/FGMRES),
// amg.cpp:297-361 (V-cycle) and precond.cpp:26-109,157-218 (Schur operator,
// SCR, nested preconditioner, solve_block_system).  Vectors never leave the
// device; per Krylov iteration the host reads back the new Hessenberg column
// (j+2 doubles) and runs the Givens rotations and the convergence test with
// the reference's own scalar arithmetic.
#include <omp.h>

#include <algorithm>
#include <exception>
#include <thread>
#include <chrono>
#include <cmath>

#include <cstdio>
#include <cstdlib>

#include "amg_device.hpp"
#include "ctx.hpp"

namespace edb {

double now_ms()
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ---------------------------------------------------------------------------
// workspace

void KrylovWs::ensure_n(int64_t nn)
{
    if (nn == n) return;
    V.clear();
    Z.clear();
    hV.clear();
    hZ.clear();
    dV.release();
    dZ.release();
    n = nn;
    r.alloc(n);
    w.alloc(n);
    t.alloc(n);
}

double* KrylovWs::v(int j)
{
    while (static_cast<int>(V.size()) <= j) {
        V.emplace_back(static_cast<size_t>(n));
        hV.push_back(V.back().p);
    }
    return V[j].p;
}

double* KrylovWs::z(int j)
{
    while (static_cast<int>(Z.size()) <= j) {
        Z.emplace_back(static_cast<size_t>(n));
        hZ.push_back(Z.back().p);
    }
    return Z[j].p;
}

void KrylovWs::sync_ptrs(cudaStream_t s)
{
    if (dV.n != hV.size()) dV.upload(hV.data(), hV.size(), s);
    if (dZ.n != hZ.size()) dZ.upload(hZ.data(), hZ.size(), s);
}

size_t KrylovWs::bytes() const { return (V.size() + Z.size() + 3) * static_cast<size_t>(n) * sizeof(double); }

namespace {

double read_scalar(Ctx& c, const double* d)
{
    double* h = c.host_buf(1);
    ED_CUDA(cudaMemcpyAsync(h, d, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    ED_CUDA(cudaStreamSynchronize(c.stream));
    return h[0];
}

} // namespace

// run_gmres, krylov.cpp:21-176
SolveRes gmres_dev(Ctx& c, DOp& op, DPrec* M, const double* b, double* x, const KrylovCfg& cfg, bool flexible,
                   KrylovWs& ws)
{
    if (cfg.restart < 1) throw Error(ED_INVALID_ARGUMENT, "gmres: restart must be >= 1");
    cudaStream_t s = c.stream;
    const int64_t n = op.size();
    ws.ensure_n(n);
    const int m = cfg.restart;
    if (static_cast<int>(ws.hcol.n) < m + 2) ws.hcol.alloc(m + 2);
    if (static_cast<int>(ws.corr.n) < m + 1) ws.corr.alloc(m + 1);
    if (static_cast<int>(ws.ycoef.n) < m + 1) ws.ycoef.alloc(m + 1);
    if (ws.scal.n < 8) ws.scal.alloc(8);
    double* r = ws.r.p;
    double* w = ws.w.p;
    double* t = ws.t.p;
    double* h = ws.hcol.p;
    double* sc = ws.scal.p; // [0] |w|^2, [1] reorth flag, [2] wnorm, [3] norm scratch

    SolveRes res;
    op.apply(x, r);
    vec_sub_from(r, b, n, s);
    norm2(c.red, r, n, sc + 3, s);
    double rnorm = read_scalar(c, sc + 3);
    res.initial_norm = rnorm;
    const double tol = std::max(cfg.rel_tol * rnorm, cfg.abs_tol);
    if (rnorm <= tol) {
        res.converged = true;
        res.final_norm = rnorm;
        return res;
    }

    std::vector<std::vector<double>> H(m);
    std::vector<double> cs(m), sn(m), g(static_cast<size_t>(m) + 1), y;
    int total = 0;
    bool stagnated = false;
    while (total < cfg.max_iters && !stagnated) {
        norm2(c.red, r, n, sc + 3, s);
        const double beta = read_scalar(c, sc + 3);
        if (beta == 0.0) break;
        vec_div_scalar(ws.v(0), r, sc + 3, nullptr, n, s);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;

        int j = 0;
        bool breakdown = false;
        while (j < m && total < cfg.max_iters) {
            double* vj = ws.v(j);
            if (M) {
                if (flexible) {
                    double* zj = ws.z(j);
                    M->apply(vj, zj);
                    op.apply(zj, w);
                } else {
                    M->apply(vj, t);
                    op.apply(t, w);
                }
            } else {
                op.apply(vj, w);
            }
            // modified Gram-Schmidt chain (krylov.cpp:81-86), one fused
            // "w -= h_{i-1} v_{i-1}; h_i = v_i . w" pass per i
            mgs_axpy_dot(c.red, w, nullptr, nullptr, ws.v(0), n, h + 0, s);
            for (int i = 1; i <= j; ++i) mgs_axpy_dot(c.red, w, ws.v(i - 1), h + i - 1, ws.v(i), n, h + i, s);
            mgs_axpy_dot(c.red, w, ws.v(j), h + j, nullptr, n, sc + 0, s);
            double* vnext = ws.v(j + 1);
            ws.sync_ptrs(s);
            // always-computed classical check + selective reorthogonalization (:87-105)
            multi_dot(c.red, ws.dV.p, j + 1, w, n, ws.corr.p, s);
            reorth_decide(sc, h, ws.corr.p, j + 1, s);
            reorth_apply(c.red, w, ws.dV.p, ws.corr.p, j + 1, n, sc, s);
            vec_div_scalar(vnext, w, sc + 2, sc + 2, n, s);
            double* hb = c.host_buf(static_cast<size_t>(j) + 8);
            ED_CUDA(cudaMemcpyAsync(hb, h, (j + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
            ED_CUDA(cudaMemcpyAsync(hb + j + 1, sc, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
            ED_CUDA(cudaStreamSynchronize(s));
            std::vector<double>& hc = H[j];
            hc.assign(hb, hb + j + 1);
            const double wnorm = hb[j + 3];
            hc.push_back(wnorm);
            if (!(wnorm > 1e-300)) breakdown = true;
            // Givens rotations (:114-131)
            for (int i = 0; i < j; ++i) {
                const double hi = hc[i], hi1 = hc[i + 1];
                hc[i] = cs[i] * hi + sn[i] * hi1;
                hc[i + 1] = -sn[i] * hi + cs[i] * hi1;
            }
            const double denom = std::hypot(hc[j], hc[j + 1]);
            if (denom == 0.0) {
                cs[j] = 1.0;
                sn[j] = 0.0;
            } else {
                cs[j] = hc[j] / denom;
                sn[j] = hc[j + 1] / denom;
            }
            hc[j] = denom;
            hc[j + 1] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] *= cs[j];
            ++total;
            ++j;
            const double est = std::abs(g[j]);
            res.history.push_back(est);
            if (est <= tol || breakdown) break;
        }
        // back substitution (:140-146)
        y.assign(j, 0.0);
        for (int i = j - 1; i >= 0; --i) {
            double sum = g[i];
            for (int k = i + 1; k < j; ++k) sum -= H[k][i] * y[k];
            y[i] = (H[i][i] != 0.0) ? sum / H[i][i] : 0.0;
        }
        if (j > 0) ED_CUDA(cudaMemcpyAsync(ws.ycoef.p, y.data(), j * sizeof(double), cudaMemcpyHostToDevice, s));
        ws.sync_ptrs(s);
        if (flexible && M) {
            multi_axpy(x, ws.dZ.p, ws.ycoef.p, j, n, s);
        } else {
            vec_fill(t, 0.0, n, s);
            multi_axpy(t, ws.dV.p, ws.ycoef.p, j, n, s);
            if (M) {
                M->apply(t, w);
                vec_add(x, w, n, s);
            } else {
                vec_add(x, t, n, s);
            }
        }
        // true residual at the restart boundary (:161-170)
        op.apply(x, r);
        vec_sub_from(r, b, n, s);
        norm2(c.red, r, n, sc + 3, s);
        rnorm = read_scalar(c, sc + 3);
        if (rnorm <= tol) {
            res.converged = true;
            break;
        }
        if (breakdown) stagnated = true;
    }
    res.iterations = total;
    res.final_norm = rnorm;
    return res;
}

// ---------------------------------------------------------------------------
// AMG

void DevHierarchy::build(Ctx& c, const Bsr& A0, const AmgOpts& o, cudaStream_t stream)
{
    cudaStream_t s = stream ? stream : c.stream;
    opts = o;
    lv.clear();
    level_rows.clear();
    tail = -1;
    fallback = false;
    const double t0 = now_ms();
    const double host0 = host_ms_acc();
    double host_helpers = 0.0; // host work of the helper threads (level operator, dense tail)
    const bool device_ok = o.block_size == A0.st->Rb && (A0.st->Rb == 1 || A0.st->Rb == 3) &&
                           std::getenv("ED_HOST_AMG") == nullptr;
    if (device_ok) {
        // GPU setup (amg_device.cu); the host only aggregates and orthonormalises
        static const bool verbose = std::getenv("ED_AMG_VERBOSE") != nullptr;
        auto lap = [&](const char* what) {
            if (!verbose) return;
            ED_CUDA(cudaStreamSynchronize(s));
            std::fprintf(stderr, "[amg-build] %-22s %8.2f ms\n", what, now_ms() - t0);
        };
        static const int tail_max = std::getenv("ED_DENSE_TAIL") ? std::atoi(std::getenv("ED_DENSE_TAIL")) : 4096;
        const bool tails = o.smoother == 1 && tail_max > 0;
        // structure cache slot: the S_hat hierarchy is the one built on stream2
        auto cache_of = [&](int l) -> LevelCache* { return l < 16 ? &c.lcache[s == c.stream2 ? 1 : 0][l] : nullptr; };
        cudaStream_t ts = s == c.stream ? c.stream3 : c.stream4;
        // The level-ordered operator of level 1 (host level schedule + ring
        // layout, the longest host step of the setup) is built on its own host
        // thread and stream while this thread builds the coarser levels.  Level
        // 1 is never collapsed into the dense tail when it has > tail_max rows.
        std::thread lop_th;
        std::exception_ptr err_l;
        double host_lop = 0.0;
        Bsr pre_op;
        int pre_l = -1;
        struct Joiner {
            std::thread& t;
            ~Joiner()
            {
                if (t.joinable()) t.join();
            }
        } lop_joiner{lop_th};
        auto on_level = [&](int l, const DBsrRaw& m) {
            if (l < 0) {
                if (lop_th.joinable()) lop_th.join();
                return;
            }
            if (pre_l >= 0 || l != 1 || (tails && m.nbr * m.Rb <= tail_max) || std::getenv("ED_SERIAL_SETUP")) return;
            pre_l = l;
            cudaEvent_t ready;
            ED_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
            ED_CUDA(cudaEventRecord(ready, s));
            ED_CUDA(cudaStreamWaitEvent(ts, ready, 0));
            ED_CUDA(cudaEventDestroy(ready));
            lop_th = std::thread([&, m, ts] {
                try {
                    alloc_stream() = ts;
                    ED_CUDA(cudaSetDevice(c.device));
                    pre_op = bsr_leveled(m, ts, cache_of(1));
                    ED_CUDA(cudaStreamSynchronize(ts));
                    host_lop = host_ms_acc();
                } catch (...) {
                    err_l = std::current_exception();
                }
            });
        };
        DevSetupResult R = amg_build_device(A0, o, s, on_level);
        Joiner lop_joiner_r{lop_th}; // joins before R (which the thread reads) is destroyed
        lap("device setup");
        if (R.fallback) {
            fallback = true;
            fb_invd.upload(R.fallback_inv_diag, s);
            ED_CUDA(cudaStreamSynchronize(s));
            setup_host_ms = host_ms_acc() - host0;
            return;
        }
        const int L = static_cast<int>(R.levels.size());
        level_rows.clear();
        for (int l = 0; l < L; ++l) level_rows.push_back(R.levels[l].A.nbr * R.levels[l].A.Rb);
        // collapse the coarse tail: the first level below the fine one small
        // enough for a dense V-cycle operator (ED_DENSE_TAIL scalar rows, 0: off)
        tail = -1;
        if (tails)
            for (int l = 1; l + 1 < L; ++l)
                if (level_rows[l] <= tail_max) {
                    tail = l;
                    break;
                }
        const int La = tail >= 0 ? tail + 1 : L;
        // the dense tail (GPU, cuBLAS) is built on its own host thread and
        // stream while this thread builds the level operators above it (host
        // level schedules); it reads only levels >= tail
        std::exception_ptr err_t;
        std::thread tail_th;
        if (tail >= 0) {
            cudaEvent_t ready;
            ED_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
            ED_CUDA(cudaEventRecord(ready, s));
            ED_CUDA(cudaStreamWaitEvent(ts, ready, 0));
            ED_CUDA(cudaEventDestroy(ready));
            tail_th = std::thread([&, ts] {
                try {
                    alloc_stream() = ts;
                    ED_CUDA(cudaSetDevice(c.device));
                    std::vector<DenseTailLevel> tl;
                    for (int l = tail; l + 1 < L; ++l)
                        tl.push_back(DenseTailLevel{&R.levels[l].A, &R.levels[l].P, &R.levels[l].R,
                                                    R.levels[l].invd.p});
                    dense_vcycle_operator(tl, R.pinv, R.nc, o.pre_sweeps, o.post_sweeps, vtail, ts);
                    ED_CUDA(cudaStreamSynchronize(ts));
                } catch (...) {
                    err_t = std::current_exception();
                }
            });
        }
        Joiner joiner{tail_th};
        lv.resize(La);
        for (int l = 0; l < La; ++l) {
            DevLevel& d = lv[l];
            DevLevelData& D = R.levels[l];
            d.n = D.A.nbr * D.A.Rb;
            if (l == tail) {
                d.r.alloc(d.n);
                d.z.alloc(d.n);
                break;
            }
            if (l == 0) {
                d.A = &A0;
            } else if (l == pre_l) {
                lop_th.join();
                if (err_l) std::rethrow_exception(err_l);
                d.Aown = std::move(pre_op);
                d.A = &d.Aown;
            } else {
                d.Aown = bsr_from_dbsr(std::move(D.A), true, s, cache_of(l));
                d.A = &d.Aown;
            }
            d.invd = std::move(D.invd);
            sweep_prepare(*d.A, d.invd.p, d.gdense, s);
            d.s.alloc(d.n);
            if (l > 0) {
                d.r.alloc(d.n);
                d.z.alloc(d.n);
            }
            if (l + 1 < L) {
                d.P = bsr_from_dbsr(std::move(D.P), false, s);
                d.R = bsr_from_dbsr(std::move(D.R), false, s);
            }
        }
        nc = R.nc;
        lap("level operators");
        if (tail < 0) pinv.upload(R.pinv, s);
        if (tail_th.joinable()) tail_th.join();
        if (err_t) std::rethrow_exception(err_t);
        ED_CUDA(cudaStreamSynchronize(s));
        lap("dense tail");
        if (lop_th.joinable()) lop_th.join();
        host_helpers += host_lop;
        setup_host_ms = host_ms_acc() - host0 + host_helpers;
        return;
    }
    // The host restatement (amg_host.cpp) builds the same hierarchy on the CPU.
    // It is a parity / diagnostic path only (ED_HOST_AMG=1), never a silent
    // fallback: an AMG block size the device setup does not handle is refused.
    if (std::getenv("ED_HOST_AMG") == nullptr)
        throw Error(ED_UNSUPPORTED, "AMG setup: block_size " + std::to_string(o.block_size) +
                                        " on a " + std::to_string(A0.st->Rb) + "x" + std::to_string(A0.st->Rb) +
                                        "-block operator is not supported on the device (block size must equal the "
                                        "operator's block, 1 or 3)");
    const HostCsr A0h = bsr_to_csr(A0, s);
    const HostHierarchy hh = amg_build_host(A0h, o);
    setup_host_ms = now_ms() - t0;
    if (hh.fallback) {
        fallback = true;
        fb_invd.upload(hh.fallback_inv_diag, s);
        ED_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const int L = static_cast<int>(hh.levels.size());
    const int Bc = (o.block_size == 3) ? 3 : 1;
    tail = -1;
    level_rows.clear();
    for (int l = 0; l < L; ++l) level_rows.push_back(hh.levels[l].A.nrows);
    lv.resize(L);
    for (int l = 0; l < L; ++l) {
        DevLevel& d = lv[l];
        const HostLevel& H = hh.levels[l];
        d.n = H.A.nrows;
        const int Bl = (l == 0) ? A0.st->Rb : Bc;
        if (l == 0) {
            d.A = &A0;
        } else {
            d.Aown = bsr_from_csr(H.A, Bl, Bl, true, s);
            d.A = &d.Aown;
        }
        d.invd.upload(H.inv_diag, s);
        sweep_prepare(*d.A, d.invd.p, d.gdense, s);
        d.s.alloc(d.n);
        if (l > 0) {
            d.r.alloc(d.n);
            d.z.alloc(d.n);
        }
        if (l + 1 < L) {
            d.P = bsr_from_csr(H.P, Bl, Bc, false, s);
            d.R = bsr_from_csr(H.R, Bc, Bl, false, s);
        }
    }
    nc = hh.nc;
    pinv.upload(hh.pinv, s);
    ED_CUDA(cudaStreamSynchronize(s));
}

// AmgHierarchy::smooth, amg.cpp:297-324
void DevHierarchy::smooth(Ctx& c, int l, const double* b, double* z, int sweeps)
{
    DevLevel& d = lv[l];
    if (opts.smoother == 0) {
        for (int k = 0; k < sweeps; ++k) {
            spmv(*d.A, z, d.s.p, nullptr, 0, c.stream);
            jacobi_update(z, b, d.s.p, d.invd.p, opts.jacobi_weight, d.n, c.stream);
        }
        return;
    }
    for (int k = 0; k < sweeps; ++k) {
        sgs_sweep(*d.A, b, z, d.invd.p, true, c.stream, d.gdense.p);
        sgs_sweep(*d.A, b, z, d.invd.p, false, c.stream, d.gdense.p);
    }
}

// AmgHierarchy::cycle, amg.cpp:326-352
void DevHierarchy::cycle(Ctx& c, int l, const double* r, double* z)
{
    DevLevel& d = lv[l];
    cudaStream_t s = c.stream;
    const std::string saved = prof_tag();
    prof_tag() = (opts.block_size == 3 ? "A" : "S") + std::to_string(l);
    if (l == static_cast<int>(lv.size()) - 1) {
        if (l == tail) dense_gemv(vtail.p, r, z, d.n, s); // collapsed coarse tail (dense_tail.cu)
        else dense_gemv(pinv.p, r, z, nc, s);            // COD min-norm solve (amg.cpp:331-334)
        prof_tag() = saved;
        return;
    }
    vec_fill(z, 0.0, d.n, s);
    smooth(c, l, r, z, opts.pre_sweeps);
    spmv(*d.A, z, d.s.p, r, 1, s); // scratch = r - A z
    DevLevel& e = lv[l + 1];
    spmv(d.R, d.s.p, e.r.p, nullptr, 0, s);
    cycle(c, l + 1, e.r.p, e.z.p);
    prof_tag() = (opts.block_size == 3 ? "A" : "S") + std::to_string(l);
    spmv(d.P, e.z.p, z, nullptr, 2, s); // z += P zc
    smooth(c, l, r, z, opts.post_sweeps);
    prof_tag() = saved;
}

void DevHierarchy::vcycle(Ctx& c, const double* r, double* z)
{
    if (fallback) {
        vec_copy(z, r, static_cast<int64_t>(fb_invd.n), c.stream);
        vec_mul(z, fb_invd.p, static_cast<int64_t>(fb_invd.n), c.stream);
        return;
    }
    cycle(c, 0, r, z);
}

// ---------------------------------------------------------------------------
// operators

namespace {

struct MatOp final : DOp {
    const Bsr& M;
    cudaStream_t s;
    MatOp(const Bsr& m, cudaStream_t st) : M(m), s(st) {}
    int64_t size() const override { return M.nrows(); }
    void apply(const double* x, double* y) override { spmv(M, x, y, nullptr, 0, s); }
};

// BlockOperator (blocksystem.hpp:27-45)
struct BlockOp final : DOp {
    WorkSys& W;
    cudaStream_t s;
    BlockOp(WorkSys& w, cudaStream_t st) : W(w), s(st) {}
    int64_t size() const override { return static_cast<int64_t>(W.nv) + W.np; }
    void apply(const double* x, double* y) override
    {
        if (W.K.n_nodes > 0) return spmv44(W.K, x, y, W.nv, W.np, s);
        spmv2(W.A, x, W.B, x + W.nv, y, 1.0, s);
        spmv2(W.C, x, W.D, x + W.nv, y + W.nv, 1.0, s);
    }
};

struct AmgPrec final : DPrec {
    Ctx& c;
    DevHierarchy& h;
    AmgPrec(Ctx& cc, DevHierarchy& hh) : c(cc), h(hh) {}
    void apply(const double* r, double* z) override { h.vcycle(c, r, z); }
};

KrylovCfg kcfg(const ed_krylov_config& k) { return KrylovCfg{k.restart, k.max_iters, k.rel_tol, k.abs_tol}; }

// SchurOperator::apply, precond.cpp:26-42
struct SchurOp final : DOp {
    Ctx& c;
    WorkSys& W;
    DevHierarchy& amg_a;
    KrylovCfg cfg;
    Stats& st;
    DevArray<double> t, z;
    SchurOp(Ctx& cc, WorkSys& w, DevHierarchy& a, const KrylovCfg& k, Stats& sts)
        : c(cc), W(w), amg_a(a), cfg(k), st(sts), t(w.nv), z(w.nv)
    {
    }
    int64_t size() const override { return W.np; }
    void apply(const double* x, double* y) override
    {
        spmv(W.B, x, t.p, nullptr, 0, c.stream);
        vec_fill(z.p, 0.0, W.nv, c.stream);
        MatOp aop(W.A, c.stream);
        AmgPrec M(c, amg_a);
        const SolveRes r = gmres_dev(c, aop, &M, t.p, z.p, cfg, false, c.ws_a);
        st.schur_applies += 1;
        st.inner_iters += r.iterations;
        spmv2(W.D, x, W.C, z.p, y, -1.0, c.stream); // y = D x - C z
    }
};

// ScrSolver::solve, precond.cpp:52-99
struct Scr {
    Ctx& c;
    WorkSys& W;
    KrylovCfg ta, ts, ti;
    DevHierarchy& amg_a;
    DevHierarchy& amg_s;
    Stats& st;
    DevArray<double> xhat, rp2, rv2;
    Scr(Ctx& cc, WorkSys& w, const ed_block_solver_options& o, DevHierarchy& a, DevHierarchy& sh, Stats& sts)
        : c(cc), W(w), ta(kcfg(o.a)), ts(kcfg(o.s)), ti(kcfg(o.inner)), amg_a(a), amg_s(sh), st(sts),
          xhat(w.nv), rp2(w.np), rv2(w.nv)
    {
    }
    void solve(const double* rv, const double* rp, double* xv, double* xp)
    {
        cudaStream_t s = c.stream;
        MatOp aop(W.A, s);
        AmgPrec Ma(c, amg_a), Ms(c, amg_s);
        // 1. A xhat = r_v
        vec_fill(xhat.p, 0.0, W.nv, s);
        SolveRes r1 = gmres_dev(c, aop, &Ma, rv, xhat.p, ta, false, c.ws_a);
        st.a_solves += 1;
        st.a_iters += r1.iterations;
        // 2. r_p - C xhat
        spmv(W.C, xhat.p, rp2.p, rp, 1, s);
        // 3. S x_p = r_p
        vec_fill(xp, 0.0, W.np, s);
        if (ti.rel_tol >= 1.0) {
            MatOp sop(W.S, s);
            SolveRes r3 = gmres_dev(c, sop, &Ms, rp2.p, xp, ts, false, c.ws_s);
            st.s_solves += 1;
            st.s_iters += r3.iterations;
        } else {
            SchurOp sop(c, W, amg_a, ti, st);
            SolveRes r3 = gmres_dev(c, sop, &Ms, rp2.p, xp, ts, false, c.ws_s);
            st.s_solves += 1;
            st.s_iters += r3.iterations;
        }
        // 4. r_v - B x_p
        spmv(W.B, xp, rv2.p, rv, 1, s);
        // 5. A x_v = r_v
        vec_fill(xv, 0.0, W.nv, s);
        SolveRes r5 = gmres_dev(c, aop, &Ma, rv2.p, xv, ta, false, c.ws_a);
        st.a_solves += 1;
        st.a_iters += r5.iterations;
    }
};

// NestedPrecond::apply, precond.cpp:101-109
struct NestedPrec final : DPrec {
    Scr& scr;
    int nv;
    explicit NestedPrec(Scr& s, int nvv) : scr(s), nv(nvv) {}
    void apply(const double* r, double* z) override { scr.solve(r, r + nv, z, z + nv); }
};

// SimplePrecond::apply, precond.cpp:122-155
struct SimplePrec final : DPrec {
    Ctx& c;
    WorkSys& W;
    KrylovCfg ta, ts;
    DevHierarchy& amg_a;
    DevHierarchy& amg_s;
    Stats& st;
    DevArray<double> invda, xhat, rp, t;
    SimplePrec(Ctx& cc, WorkSys& w, const ed_block_solver_options& o, DevHierarchy& a, DevHierarchy& sh, Stats& sts)
        : c(cc), W(w), ta(kcfg(o.a)), ts(kcfg(o.s)), amg_a(a), amg_s(sh), st(sts), invda(w.nv), xhat(w.nv),
          rp(w.np), t(w.nv)
    {
        // inv_diag_a_ = 1 / diag(A) (precond.cpp:115-117, no zero guard)
        bsr_diag(W.A, t.p, c.stream);
        recip(t.p, invda.p, W.nv, c.stream);
    }
    void apply(const double* r, double* z) override
    {
        cudaStream_t s = c.stream;
        MatOp aop(W.A, s), sop(W.S, s);
        AmgPrec Ma(c, amg_a), Ms(c, amg_s);
        // velocity predictor A xhat = r_v
        vec_fill(xhat.p, 0.0, W.nv, s);
        const SolveRes r1 = gmres_dev(c, aop, &Ma, r, xhat.p, ta, false, c.ws_a);
        st.a_solves += 1;
        st.a_iters += r1.iterations;
        // pressure: S_hat x_p = r_p - C xhat
        spmv(W.C, xhat.p, rp.p, r + W.nv, 1, s);
        vec_fill(z + W.nv, 0.0, W.np, s);
        const SolveRes r2 = gmres_dev(c, sop, &Ms, rp.p, z + W.nv, ts, false, c.ws_s);
        st.s_solves += 1;
        st.s_iters += r2.iterations;
        // velocity correction z_v = xhat - inv_diag_a (B x_p)
        spmv(W.B, z + W.nv, t.p, nullptr, 0, s);
        vec_mul(t.p, invda.p, W.nv, s);
        vec_sub_from(t.p, xhat.p, W.nv, s);
        vec_copy(z, t.p, W.nv, s);
    }
};

// JacobiPrecond on the monolithic (scaled) matrix (krylov.cpp:10-14)
struct MonoJacobi final : DPrec {
    Ctx& c;
    int64_t n;
    DevArray<double> invd;
    MonoJacobi(Ctx& cc, WorkSys& W) : c(cc), n(static_cast<int64_t>(W.nv) + W.np), invd(n)
    {
        DevArray<double> d(n);
        bsr_diag(W.A, d.p, c.stream);
        bsr_diag(W.D, d.p + W.nv, c.stream);
        inv_diag_from(d.p, invd.p, n, c.stream);
    }
    void apply(const double* r, double* z) override
    {
        vec_copy(z, r, n, c.stream);
        vec_mul(z, invd.p, n, c.stream);
    }
};

// Ilu0Precond on the monolithic (scaled) matrix (ilu0.cpp)
struct IluPrec final : DPrec {
    Ctx& c;
    DevIlu0 f;
    IluPrec(Ctx& cc, WorkSys& W) : c(cc) { ilu0_build(WorkSysView{&W.A, &W.B, &W.C, &W.D}, f, c.stream); }
    void apply(const double* r, double* z) override { ilu0_apply(f, r, z, c.stream); }
};

} // namespace

AmgOpts amg_opts_from(const ed_amg_options& o, const Ctx& c, bool velocity, int nrows)
{
    AmgOpts a;
    a.block_size = o.block_size;
    a.strength_theta = o.strength_theta;
    a.max_levels = o.max_levels;
    a.coarse_max_rows = o.coarse_max_rows;
    a.smoother = o.smoother;
    a.jacobi_weight = o.jacobi_weight;
    a.pre_sweeps = o.pre_sweeps;
    a.post_sweeps = o.post_sweeps;
    a.smooth_prolongator = o.smooth_prolongator != 0;
    if (velocity && o.use_dof_row_maps && c.have_dofs && c.sys_from_mesh && nrows == 3 * c.nfree) {
        // set_amg_maps (driver.cpp:32-48): compressed free-node ids, component
        a.row_to_node.resize(nrows);
        a.row_component.resize(nrows);
        for (int r = 0; r < nrows; ++r) {
            a.row_to_node[r] = r / 3;
            a.row_component[r] = r % 3;
        }
    }
    return a;
}

// solve_block_system, precond.cpp:157-218: Nested (0), Simple (1), Ilu0 (2),
// Jacobi (3) and None (4)
Stats solve_block_system_dev(Ctx& c, const double* d_rhs, double* d_x, const ed_block_solver_options& o,
                             std::vector<double>* history, ed_phase_times* times)
{
    if (o.precond < 0 || o.precond > 4) throw Error(ED_INVALID_ARGUMENT, "unknown PrecondKind");
    const bool amg = o.precond == 0 || o.precond == 1;
    const double t0 = now_ms();
    cudaStream_t s = c.stream;
    Stats st;
    WorkSys& W = c.work; // solver working set (reused across solves)
    double tp = now_ms();
    make_work(c, W, o.scale != 0, o.eps_diag);
    const int64_t n = static_cast<int64_t>(W.nv) + W.np;
    DevArray<double> b(n);
    vec_copy(b.p, d_rhs, n, s);
    if (W.scaled) vec_mul(b.p, W.w.p, n, s);
    vec_fill(d_x, 0.0, n, s);
    c.sync();
    const double t_planes = now_ms() - tp;
    tp = now_ms();
    if (amg) build_shat_work(c, W);
    c.sync();
    const double t_shat = now_ms() - tp;
    tp = now_ms();
    // the two hierarchies are independent (AmgHierarchy::build on A and on
    // S_hat, precond.cpp:44-50): S_hat's is built on a second host thread and
    // stream while A's is built here; the V-cycles run on c.stream after both
    DevHierarchy amg_a, amg_s;
    const AmgOpts oa = amg_opts_from(o.amg_a, c, true, W.nv), os = amg_opts_from(o.amg_s, c, false, W.np);
    std::exception_ptr err_s;
    double ms_s = 0.0, ms_a = 0.0;
    static const bool serial = std::getenv("ED_SERIAL_SETUP") != nullptr;
    auto build_s = [&] {
        const cudaStream_t prev_as = alloc_stream();
        const int prev_omp = omp_get_max_threads();
        try {
            const double t = now_ms();
            alloc_stream() = c.stream2;
            ED_CUDA(cudaSetDevice(c.device));
            if (!serial) omp_set_num_threads(std::max(1, omp_get_num_procs() / 4)); // leave the cores to A's build
            amg_s.build(c, W.S, os, c.stream2);
            ED_CUDA(cudaStreamSynchronize(c.stream2));
            ms_s = now_ms() - t;
        } catch (...) {
            err_s = std::current_exception();
        }
        alloc_stream() = prev_as;
        omp_set_num_threads(prev_omp);
    };
    std::thread th;
    if (amg && !serial) th = std::thread(build_s);
    try {
        const double t = now_ms();
        if (amg) amg_a.build(c, W.A, oa);
        ED_CUDA(cudaStreamSynchronize(c.stream));
        ms_a = now_ms() - t;
    } catch (...) {
        if (th.joinable()) th.join();
        throw;
    }
    if (amg && serial) build_s();
    if (th.joinable()) th.join();
    static const bool tell = std::getenv("ED_SETUP_TIMES") != nullptr;
    if (tell) std::fprintf(stderr, "[setup] A %.1f ms  S %.1f ms\n", ms_a, ms_s);
    if (err_s) std::rethrow_exception(err_s);
    c.sync();
    const double t_amg = now_ms() - tp;
    tp = now_ms();
    BlockOp op(W, s);
    SolveRes res;
    if (o.precond == 0) {
        Scr scr(c, W, o, amg_a, amg_s, st);
        NestedPrec M(scr, W.nv);
        res = gmres_dev(c, op, &M, b.p, d_x, kcfg(o.outer), true, c.ws_outer);
    } else if (o.precond == 1) {
        SimplePrec M(c, W, o, amg_a, amg_s, st);
        res = gmres_dev(c, op, &M, b.p, d_x, kcfg(o.outer), true, c.ws_outer);
    } else if (o.precond == 2) {
        IluPrec M(c, W);
        res = gmres_dev(c, op, &M, b.p, d_x, kcfg(o.outer), false, c.ws_outer);
    } else if (o.precond == 3) {
        MonoJacobi M(c, W);
        res = gmres_dev(c, op, &M, b.p, d_x, kcfg(o.outer), false, c.ws_outer);
    } else {
        res = gmres_dev(c, op, nullptr, b.p, d_x, kcfg(o.outer), false, c.ws_outer);
    }
    if (W.scaled) vec_mul(d_x, W.w.p, n, s);
    c.sync();
    const double t_fg = now_ms() - tp;
    st.outer_iters = res.iterations;
    st.converged = res.converged;
    st.t_solve = (now_ms() - t0) * 1e-3;
    if (history) *history = res.history;
    if (times) {
        times->planes_ms = t_planes;
        times->shat_ms = t_shat;
        times->amg_setup_ms = t_amg;
        times->amg_host_ms = amg_a.setup_host_ms + amg_s.setup_host_ms;
        times->fgmres_ms = t_fg;
    }
    return st;
}

} // namespace edb

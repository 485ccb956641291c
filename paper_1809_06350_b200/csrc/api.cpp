// extern "C" entry points (include/elastodyn_b200.h).  Each maps edb::Error
// to a status code; no CPU fallback exists anywhere behind this ABI.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <limits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include <omp.h>

#include "ctx.hpp"

namespace edb {

namespace {
std::atomic<int64_t> g_launches{0};
// ED_PROFILE=1: synchronise after every launch and attribute wall time per
// kernel name (diagnostic only; never set for measurements).
struct KProf {
    bool on = std::getenv("ED_PROFILE") != nullptr;
    std::map<std::string, std::pair<int64_t, double>> t;
    std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    ~KProf()
    {
        if (!on) return;
        std::vector<std::pair<double, std::string>> v;
        for (auto& kv : t) v.push_back({kv.second.second, kv.first});
        std::sort(v.rbegin(), v.rend());
        for (auto& x : v)
            std::fprintf(stderr, "[prof] %-22s %10.3f ms  %9lld launches\n", x.second.c_str(), x.first * 1e3,
                         static_cast<long long>(t[x.second].first));
    }
} g_prof;
}

void after_launch(const char* what)
{
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) throw Error(ED_CUDA_ERROR, std::string("launch ") + what + ": " + cudaGetErrorString(e));
    if (g_prof.on) {
        const cudaError_t e2 = cudaDeviceSynchronize();
        if (e2 != cudaSuccess)
            throw Error(ED_CUDA_ERROR, std::string("kernel ") + what + " failed: " + cudaGetErrorString(e2));
        const auto now = std::chrono::steady_clock::now();
        auto& slot = g_prof.t[prof_tag().empty() ? std::string(what) : std::string(what) + "@" + prof_tag()];
        slot.first += 1;
        slot.second += std::chrono::duration<double>(now - g_prof.last).count();
        g_prof.last = now;
    }
}

int64_t launch_count() { return g_launches.load(); }

namespace {
struct Acct {
    bool on = false;
    struct Rec {
        std::string name;
        double bytes;
        cudaEvent_t a, b;
    };
    std::vector<cudaEvent_t> pool;
    std::vector<Rec> open;
    struct Tot {
        int64_t n = 0;
        double ms = 0.0, bytes = 0.0;
    };
    std::map<std::string, Tot> tot;
    cudaEvent_t get()
    {
        if (pool.empty()) {
            cudaEvent_t e;
            ED_CUDA(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    // resolve recorded launches (their streams must be complete)
    void flush()
    {
        for (auto& r : open) {
            float ms = 0.0f;
            if (cudaEventSynchronize(r.b) == cudaSuccess && cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
                Tot& t = tot[r.name];
                t.n += 1;
                t.ms += ms;
                t.bytes += r.bytes;
            }
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        open.clear();
    }
} g_acct;
std::mutex g_acct_mu;
} // namespace

bool acct_on() { return g_acct.on; }

// concurrent hierarchy builds run on their own host threads: records are
// appended under a lock and a scope closes its own record (by index); records
// are resolved only at the API's synchronisation points (ed_kernel_account*)
int acct_begin(cudaStream_t s, const char* name, double bytes)
{
    std::lock_guard<std::mutex> lk(g_acct_mu);
    if (g_acct.open.size() >= (1u << 20)) return -1;
    Acct::Rec r{prof_tag().empty() ? std::string(name) : std::string(name) + "@" + prof_tag(), bytes, g_acct.get(),
                g_acct.get()};
    ED_CUDA(cudaEventRecord(r.a, s));
    g_acct.open.push_back(r);
    return static_cast<int>(g_acct.open.size()) - 1;
}

void acct_end(cudaStream_t s, int idx)
{
    std::lock_guard<std::mutex> lk(g_acct_mu);
    if (idx >= 0 && idx < static_cast<int>(g_acct.open.size())) ED_CUDA(cudaEventRecord(g_acct.open[idx].b, s));
}

// bytes only (no events): the Krylov vector kernels, for the solve roofline
void acct_bytes(const char* name, double bytes)
{
    std::lock_guard<std::mutex> lk(g_acct_mu);
    Acct::Tot& t = g_acct.tot[prof_tag().empty() ? std::string(name) : std::string(name) + "@" + prof_tag()];
    t.n += 1;
    t.bytes += bytes;
}

namespace {
struct Cache {
    std::mutex mu;
    std::map<std::pair<cudaStream_t, size_t>, std::vector<void*>> free;
    static size_t size_class(size_t bytes)
    {
        if (bytes <= 4096) return 4096;
        int e = 63 - __builtin_clzll(bytes); // 2^e <= bytes < 2^(e+1)
        const size_t step = size_t(1) << (e - 3);
        return (bytes + step - 1) / step * step;
    }
} g_cache;
} // namespace

void* cache_alloc(size_t bytes, cudaStream_t s)
{
    const size_t c = Cache::size_class(bytes);
    {
        std::lock_guard<std::mutex> lk(g_cache.mu);
        auto it = g_cache.free.find({s, c});
        if (it != g_cache.free.end() && !it->second.empty()) {
            void* p = it->second.back();
            it->second.pop_back();
            return p; // stream order makes the reuse safe: earlier uses precede later ones
        }
    }
    void* p = nullptr;
    if (cudaMalloc(&p, c) != cudaSuccess) {
        cudaGetLastError();
        cache_release_stream(s); // give cached blocks back and retry once
        ED_CUDA(cudaMalloc(&p, c));
    }
    return p;
}

void cache_free(void* p, size_t bytes, cudaStream_t s)
{
    std::lock_guard<std::mutex> lk(g_cache.mu);
    g_cache.free[{s, Cache::size_class(bytes)}].push_back(p);
}

void cache_release_stream(cudaStream_t s)
{
    cudaStreamSynchronize(s);
    std::lock_guard<std::mutex> lk(g_cache.mu);
    for (auto it = g_cache.free.begin(); it != g_cache.free.end();) {
        if (it->first.first == s) {
            for (void* p : it->second) cudaFree(p);
            it = g_cache.free.erase(it);
        } else {
            ++it;
        }
    }
}

cudaStream_t& alloc_stream()
{
    static thread_local cudaStream_t s = nullptr;
    return s;
}

double& alloc_ms()
{
    static thread_local double t = 0.0;
    return t;
}

double& host_ms_acc()
{
    static thread_local double t = 0.0;
    return t;
}

double now_ms_host()
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

std::string& prof_tag()
{
    static std::string t;
    return t;
}

Ctx::Ctx(int dev) : device(dev)
{
    ED_CUDA(cudaSetDevice(dev));
    // the library stream and the A-hierarchy tail stream carry the critical
    // path of the concurrent hierarchy builds: highest priority; the S_hat
    // build (shorter, overlapped) runs at the lowest
    int lo_prio = 0, hi_prio = 0;
    ED_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    ED_CUDA(cudaStreamCreateWithPriority(&owner.s, cudaStreamNonBlocking, hi_prio));
    ED_CUDA(cudaStreamCreateWithPriority(&owner2.s, cudaStreamNonBlocking, lo_prio));
    ED_CUDA(cudaStreamCreateWithPriority(&owner3.s, cudaStreamNonBlocking, hi_prio));
    ED_CUDA(cudaStreamCreateWithPriority(&owner4.s, cudaStreamNonBlocking, lo_prio));
    stream = owner.s;
    stream2 = owner2.s;
    stream3 = owner3.s;
    stream4 = owner4.s;
    // keep freed pool memory for the next Newton step's AMG rebuild
    cudaMemPool_t pool;
    ED_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    ED_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    host_buf(1024);
    dscratch_i.alloc(4);
    red.ensure(8, stream);
    ED_CUDA(cudaStreamSynchronize(stream));
}

Ctx::~Ctx()
{
    cudaStreamSynchronize(stream);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (pinned) cudaFreeHost(pinned);
    // the stream itself outlives every member array (StreamOwner is the first member)
}

double* Ctx::host_buf(size_t n)
{
    if (n > pinned_n) {
        if (pinned) {
            cudaStreamSynchronize(stream);
            cudaFreeHost(pinned);
        }
        pinned_n = std::max<size_t>(n, 2 * pinned_n);
        ED_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pinned), pinned_n * sizeof(double)));
    }
    return pinned;
}

void Ctx::sync() { ED_CUDA(cudaStreamSynchronize(stream)); }

int Ctx::read_int(const int* d)
{
    int* h = reinterpret_cast<int*>(host_buf(1));
    ED_CUDA(cudaMemcpyAsync(h, d, sizeof(int), cudaMemcpyDeviceToHost, stream));
    ED_CUDA(cudaStreamSynchronize(stream));
    return h[0];
}

namespace {

void check(bool ok, int code, const char* msg)
{
    if (!ok) throw Error(code, msg);
}

AsmArgs asm_args(Ctx& c, bool stage)
{
    AsmArgs A;
    A.tets = c.tets.p;
    A.grad_n = c.grad_n.p;
    A.volume = c.volume.p;
    A.tau = c.tau.p;
    A.fidx = c.d_fidx.p;
    if (stage) {
        A.u = c.m_u.p;
        A.udot = c.m_udot.p;
        A.p = c.m_p.p;
        A.pdot = c.m_pdot.p;
        A.v = c.m_v.p;
        A.vdot = c.m_vdot.p;
    } else {
        A.u = c.u.p;
        A.udot = c.udot.p;
        A.p = c.p.p;
        A.pdot = c.pdot.p;
        A.v = c.v.p;
        A.vdot = c.vdot.p;
    }
    A.elem_order = c.elem_order.p;
    A.k4slot = c.k4slot.p;
    A.k4 = c.k4.p;
    A.r_m = c.rm.p;
    A.r_p = c.rp.p;
    A.fv = c.fv.p;
    A.fp = c.fp.p;
    A.bad_element = c.dscratch_i.p;
    A.mat = c.mat;
    A.elem_h = c.elem_h.n ? c.elem_h.p : nullptr;
    for (int i = 0; i < 3; ++i) A.body_force[i] = c.body_force[i];
    return A;
}

void reset_bad(Ctx& c)
{
    const int big = INT_MAX;
    ED_CUDA(cudaMemcpyAsync(c.dscratch_i.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
    ED_CUDA(cudaStreamSynchronize(c.stream));
}

void check_bad(Ctx& c, int32_t* bad_element)
{
    const int bad = c.read_int(c.dscratch_i.p);
    if (bad_element) *bad_element = bad == INT_MAX ? -1 : bad;
    if (bad != INT_MAX)
        throw Error(ED_ELEMENT_INVERSION, "assembly: element " + std::to_string(bad) + " inverted (J <= 0)", bad);
}

void residual_on(Ctx& c, bool stage)
{
    check(c.have_dofs && c.have_mat, ED_NOT_READY, "mesh, dofs and material required");
    c.rm.zero(c.stream);
    c.rp.zero(c.stream);
    reset_bad(c);
    AsmArgs A = asm_args(c, stage);
    launch_residual(A, c.color_ptr, c.stream);
    launch_traction(c.tr_rowptr.p, c.tr_rows.p, c.tr_vals.p, c.tr_n, c.rm.p, c.stream);
}

void tangent_on(Ctx& c, bool stage, const ed_time_scalars& ts, bool foldin)
{
    check(c.have_dofs && c.have_mat, ED_NOT_READY, "mesh, dofs and material required");
    c.k4.zero(c.stream);
    c.fv.zero(c.stream);
    c.fp.zero(c.stream);
    reset_bad(c);
    AsmArgs A = asm_args(c, stage);
    A.ts = ts;
    A.rk = foldin ? c.rk.p : nullptr;
    if (!foldin) {
        A.fv = nullptr;
        A.fp = nullptr;
    }
    launch_tangent(A, c.color_ptr, c.stream);
}

void ensure_system(Ctx& c, const ed_block_solver_options* o)
{
    if (c.sys_from_mesh) {
        check(c.sys_values, ED_NOT_READY, "no tangent assembled");
        return;
    }
    check(c.csr_up.size() == 4, ED_NOT_READY, "no block system");
    const int nv = c.csr_up[0].nrows;
    const int Bv = (o && o->amg_a.block_size == 3 && nv % 3 == 0) ? 3 : (c.csr_bv > 0 && !o ? c.csr_bv : 1);
    ctx_planes_from_csr(c, Bv);
}

void fill_stats(const Stats& s, ed_linear_stats* o)
{
    if (!o) return;
    o->outer_iters = s.outer_iters;
    o->a_solves = s.a_solves;
    o->a_iters = s.a_iters;
    o->s_solves = s.s_solves;
    o->s_iters = s.s_iters;
    o->schur_applies = s.schur_applies;
    o->inner_iters = s.inner_iters;
    o->converged = s.converged ? 1 : 0;
    o->pad = 0;
    o->t_solve = s.t_solve;
}

void copy_hist(const std::vector<double>& h, double* out, int32_t cap, int32_t* len)
{
    if (len) *len = static_cast<int32_t>(h.size());
    if (out)
        for (int32_t i = 0; i < cap && i < static_cast<int32_t>(h.size()); ++i) out[i] = h[i];
}

template <class F>
int guarded(ed_ctx* h, F&& f);

} // namespace
} // namespace edb

struct ed_ctx {
    edb::Ctx c;
    explicit ed_ctx(int dev) : c(dev) {}
};

namespace edb {
namespace {
template <class F>
int guarded(ed_ctx* h, F&& f)
{
    if (!h) return ED_INVALID_ARGUMENT;
    struct StreamScope {
        cudaStream_t prev;
        explicit StreamScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
        ~StreamScope() { alloc_stream() = prev; }
    } scope(h->c.stream);
    try {
        // every entry point runs on the context's device (several contexts on
        // different GPUs may share one host thread)
        ED_CUDA(cudaSetDevice(h->c.device));
        f(h->c);
        h->c.err.clear();
        return ED_OK;
    } catch (const Error& e) {
        h->c.err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        h->c.err = "host allocation failed";
        return ED_CUDA_ERROR;
    } catch (const std::exception& e) {
        h->c.err = e.what();
        return ED_CUDA_ERROR;
    }
}
} // namespace
} // namespace edb

using namespace edb;

extern "C" {

int ed_ctx_create(int device, ed_ctx** out)
{
    if (!out) return ED_INVALID_ARGUMENT;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) {
        cudaGetLastError();
        return ED_CUDA_ERROR; // no CUDA device: there is no CPU fallback
    }
    try {
        *out = new ed_ctx(device);
    } catch (...) {
        return ED_CUDA_ERROR;
    }
    return ED_OK;
}

void ed_ctx_destroy(ed_ctx* ctx) { delete ctx; }

const char* ed_last_error(const ed_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

int ed_ctx_set_threads(ed_ctx* ctx, int n_threads)
{
    return guarded(ctx, [&](Ctx&) {
        if (n_threads > 0) omp_set_num_threads(n_threads);
    });
}

int64_t ed_kernel_launches(const ed_ctx*) { return launch_count(); }

int ed_mesh_upload(ed_ctx* ctx, int n_nodes, int n_tets, const int32_t* tets, const double* grad_n,
                   const double* volume, const double* tau)
{
    return guarded(ctx, [&](Ctx& c) {
        check(n_nodes > 0 && n_tets > 0 && tets && grad_n && volume && tau, ED_INVALID_ARGUMENT, "bad mesh");
        c.n_nodes = n_nodes;
        c.n_tets = n_tets;
        c.h_tets.assign(tets, tets + 4LL * n_tets);
        for (const int t : c.h_tets) check(t >= 0 && t < n_nodes, ED_INVALID_ARGUMENT, "tet node out of range");
        c.tets.upload(c.h_tets, c.stream);
        c.grad_n.upload(grad_n, 12LL * n_tets, c.stream);
        c.volume.upload(volume, n_tets, c.stream);
        c.tau.upload(tau, n_tets, c.stream);
        c.sync();
        c.have_mesh = true;
        c.have_dofs = false;
        c.sys_from_mesh = false;
        c.elem_h = DevArray<double>();
        c.pd_n = 0;
    });
}

int ed_dofs_build(ed_ctx* ctx, const uint8_t* fixed, int32_t* nv, int32_t* np)
{
    return guarded(ctx, [&](Ctx& c) {
        c.pd_n = 0; // a pending prescription refers to the previous constraint set
        check(c.have_mesh, ED_NOT_READY, "mesh required");
        check(fixed != nullptr, ED_INVALID_ARGUMENT, "DofMap: constraint table missing");
        const int N = c.n_nodes;
        c.fidx.assign(N, -1);
        c.fnode.clear();
        for (int n = 0; n < N; ++n) {
            const int k = (fixed[3 * n] != 0) + (fixed[3 * n + 1] != 0) + (fixed[3 * n + 2] != 0);
            if (k != 0 && k != 3) throw Error(ED_UNSUPPORTED, "partially constrained node " + std::to_string(n));
            if (k == 0) {
                c.fidx[n] = static_cast<int>(c.fnode.size());
                c.fnode.push_back(n);
            }
        }
        c.nfree = static_cast<int>(c.fnode.size());
        c.d_fidx.upload(c.fidx, c.stream);
        c.d_fnode.upload(c.fnode, c.stream);
        const size_t n3 = 3 * static_cast<size_t>(N);
        for (DevArray<double>* a : {&c.u, &c.udot, &c.v, &c.vdot, &c.m_u, &c.m_udot, &c.m_v, &c.m_vdot}) {
            a->alloc(n3);
            a->zero(c.stream);
        }
        for (DevArray<double>* a : {&c.p, &c.pdot, &c.m_p, &c.m_pdot}) {
            a->alloc(N);
            a->zero(c.stream);
        }
        const size_t nvv = 3 * static_cast<size_t>(c.nfree);
        c.rm.alloc(nvv);
        c.fv.alloc(nvv);
        c.rk.alloc(nvv);
        c.rk.zero(c.stream);
        c.rp.alloc(N);
        c.fp.alloc(N);
        c.rhs.alloc(nvv + N);
        c.xsol.alloc(nvv + N);
        c.tr_n = 0;
        ctx_build_mesh_system(c);
        c.have_dofs = true;
        if (nv) *nv = static_cast<int32_t>(nvv);
        if (np) *np = N;
    });
}

int ed_set_material(ed_ctx* ctx, const ed_material* mat)
{
    return guarded(ctx, [&](Ctx& c) {
        check(mat != nullptr, ED_INVALID_ARGUMENT, "material missing");
        check(mat->kind == 0 || mat->kind == 1, ED_INVALID_ARGUMENT, "unknown material kind");
        check(mat->incompressible || mat->kappa > 0.0, ED_INVALID_ARGUMENT, "kappa must be positive");
        c.mat = *mat;
        c.have_mat = true;
    });
}

int ed_set_fiber_field(ed_ctx* ctx, int n_tets, const double* h)
{
    return guarded(ctx, [&](Ctx& c) {
        check(c.have_mesh, ED_NOT_READY, "mesh required");
        if (h == nullptr) { // back to the material's global structure tensors
            c.elem_h = DevArray<double>();
            return;
        }
        check(n_tets == c.n_tets, ED_INVALID_ARGUMENT, "fibre field: one entry per element");
        c.elem_h.upload(h, 18LL * n_tets, c.stream);
        c.sync();
    });
}

int ed_set_prescribed_displacement(ed_ctx* ctx, int n, const int32_t* nodes, const double* u)
{
    return guarded(ctx, [&](Ctx& c) {
        check(c.have_dofs, ED_NOT_READY, "dofs required");
        c.pd_n = 0;
        if (n == 0) return;
        check(n > 0 && nodes && u, ED_INVALID_ARGUMENT, "bad prescribed-displacement arguments");
        for (int i = 0; i < n; ++i) {
            check(nodes[i] >= 0 && nodes[i] < c.n_nodes, ED_INVALID_ARGUMENT, "prescribed node out of range");
            check(c.fidx[nodes[i]] < 0, ED_INVALID_ARGUMENT, "prescribed displacement on a free node");
        }
        c.pd_nodes.upload(nodes, n, c.stream);
        c.pd_u.upload(u, 3LL * n, c.stream);
        c.sync();
        c.pd_n = n;
    });
}

int ed_set_loads(ed_ctx* ctx, const double body_force[3], int n_facets, const int32_t* facet_nodes,
                 const double* facet_third, const double* facet_h)
{
    return guarded(ctx, [&](Ctx& c) {
        check(c.have_dofs, ED_NOT_READY, "dofs required");
        for (int i = 0; i < 3; ++i) c.body_force[i] = body_force ? body_force[i] : 0.0;
        // per free row: contributions in loop order (assembly.cpp:174-183)
        const int nvv = 3 * c.nfree;
        std::vector<std::vector<double>> per(nvv);
        for (int f = 0; f < n_facets; ++f)
            for (int a = 0; a < 3; ++a) {
                const int n = facet_nodes[3 * f + a];
                check(n >= 0 && n < c.n_nodes, ED_INVALID_ARGUMENT, "facet node out of range");
                if (c.fidx[n] < 0) continue;
                for (int i = 0; i < 3; ++i) per[3 * c.fidx[n] + i].push_back(facet_third[f] * facet_h[3 * f + i]);
            }
        std::vector<int64_t> rp{0};
        std::vector<int> rows;
        std::vector<double> vals;
        for (int r = 0; r < nvv; ++r) {
            if (per[r].empty()) continue;
            rows.push_back(r);
            vals.insert(vals.end(), per[r].begin(), per[r].end());
            rp.push_back(static_cast<int64_t>(vals.size()));
        }
        c.tr_n = static_cast<int>(rows.size());
        c.tr_rowptr.upload(rp, c.stream);
        c.tr_rows.upload(rows, c.stream);
        c.tr_vals.upload(vals, c.stream);
        c.sync();
    });
}

int ed_state_upload(ed_ctx* ctx, const double* u, const double* udot, const double* p, const double* pdot,
                    const double* v, const double* vdot)
{
    return guarded(ctx, [&](Ctx& c) {
        check(c.have_dofs, ED_NOT_READY, "dofs required");
        const size_t n3 = 3 * static_cast<size_t>(c.n_nodes), n1 = c.n_nodes;
        c.u.upload(u, n3, c.stream);
        c.udot.upload(udot, n3, c.stream);
        c.p.upload(p, n1, c.stream);
        c.pdot.upload(pdot, n1, c.stream);
        c.v.upload(v, n3, c.stream);
        c.vdot.upload(vdot, n3, c.stream);
        c.sync();
    });
}

int ed_state_download(ed_ctx* ctx, double* u, double* udot, double* p, double* pdot, double* v, double* vdot)
{
    return guarded(ctx, [&](Ctx& c) {
        check(c.have_dofs, ED_NOT_READY, "dofs required");
        c.u.download(u, c.stream);
        c.udot.download(udot, c.stream);
        c.p.download(p, c.stream);
        c.pdot.download(pdot, c.stream);
        c.v.download(v, c.stream);
        c.vdot.download(vdot, c.stream);
        c.sync();
    });
}

int ed_assemble_residuals(ed_ctx* ctx, double* r_m, double* r_p, int32_t* bad_element)
{
    return guarded(ctx, [&](Ctx& c) {
        residual_on(c, false);
        check_bad(c, bad_element);
        if (r_m) c.rm.download(r_m, c.stream);
        if (r_p) c.rp.download(r_p, c.stream);
        c.sync();
    });
}

int ed_assemble_tangent(ed_ctx* ctx, const ed_time_scalars* ts, const double* rk, int32_t* bad_element)
{
    return guarded(ctx, [&](Ctx& c) {
        check(ts != nullptr, ED_INVALID_ARGUMENT, "time scalars missing");
        if (rk) c.rk.upload(rk, 3 * static_cast<size_t>(c.nfree), c.stream);
        tangent_on(c, false, *ts, rk != nullptr);
        check_bad(c, bad_element);
        if (!c.sys_from_mesh) ctx_build_mesh_system(c);
        ctx_planes_from_k4(c);
        c.sync();
    });
}

int ed_tangent_export(ed_ctx* ctx, int which, int32_t* dims, int32_t* rowptr, int32_t* col, double* val)
{
    return guarded(ctx, [&](Ctx& c) {
        ensure_system(c, nullptr);
        check(which >= 0 && which < 4, ED_INVALID_ARGUMENT, "plane must be 0..3");
        const Bsr* m[4] = {&c.sys.A, &c.sys.B, &c.sys.C, &c.sys.D};
        const HostCsr a = bsr_to_csr(*m[which], c.stream);
        if (dims) {
            dims[0] = a.nrows;
            dims[1] = a.ncols;
            dims[2] = static_cast<int32_t>(a.nnz());
        }
        if (rowptr) {
            for (size_t i = 0; i < a.rowptr.size(); ++i) rowptr[i] = static_cast<int32_t>(a.rowptr[i]);
            std::copy(a.col.begin(), a.col.end(), col);
            std::copy(a.val.begin(), a.val.end(), val);
        }
    });
}

int ed_foldin_download(ed_ctx* ctx, double* fv, double* fp)
{
    return guarded(ctx, [&](Ctx& c) {
        check(c.have_dofs, ED_NOT_READY, "dofs required");
        if (fv) c.fv.download(fv, c.stream);
        if (fp) c.fp.download(fp, c.stream);
        c.sync();
    });
}

int ed_block_system_upload(ed_ctx* ctx, int nv, int np, const int32_t* a_rp, const int32_t* a_c, const double* a_v,
                           const int32_t* b_rp, const int32_t* b_c, const double* b_v, const int32_t* c_rp,
                           const int32_t* c_c, const double* c_v, const int32_t* d_rp, const int32_t* d_c,
                           const double* d_v)
{
    return guarded(ctx, [&](Ctx& c) {
        check(nv > 0 && np > 0, ED_INVALID_ARGUMENT, "empty block system");
        auto mk = [](int nr, int nc, const int32_t* rp, const int32_t* cc, const double* vv) {
            HostCsr m;
            m.nrows = nr;
            m.ncols = nc;
            m.rowptr.assign(rp, rp + nr + 1);
            const int nnz = rp[nr];
            m.col.assign(cc, cc + nnz);
            m.val.assign(vv, vv + nnz);
            for (int r = 0; r < nr; ++r)
                for (int64_t k = m.rowptr[r]; k < m.rowptr[r + 1]; ++k) {
                    if (m.col[k] < 0 || m.col[k] >= nc) throw Error(ED_INVALID_ARGUMENT, "column out of range");
                    if (k > m.rowptr[r] && m.col[k] <= m.col[k - 1])
                        throw Error(ED_INVALID_ARGUMENT, "columns must be sorted and unique");
                }
            return m;
        };
        c.csr_up.clear();
        c.csr_up.push_back(mk(nv, nv, a_rp, a_c, a_v));
        c.csr_up.push_back(mk(nv, np, b_rp, b_c, b_v));
        c.csr_up.push_back(mk(np, nv, c_rp, c_c, c_v));
        c.csr_up.push_back(mk(np, np, d_rp, d_c, d_v));
        c.sys_from_mesh = false;
        c.csr_bv = -1;
        c.sys = BlockSys{};
    });
}

int ed_solve_block_system_device(ed_ctx* ctx, const double* d_rhs, double* d_x, const ed_block_solver_options* opts,
                                 ed_linear_stats* stats, double* history, int32_t history_cap, int32_t* history_len)
{
    return guarded(ctx, [&](Ctx& c) {
        check(opts != nullptr, ED_INVALID_ARGUMENT, "options missing");
        ensure_system(c, opts);
        std::vector<double> hist;
        const Stats st = solve_block_system_dev(c, d_rhs, d_x, *opts, &hist, nullptr);
        fill_stats(st, stats);
        copy_hist(hist, history, history_cap, history_len);
    });
}

int ed_solve_block_system(ed_ctx* ctx, const double* rhs, double* x, const ed_block_solver_options* opts,
                          ed_linear_stats* stats, double* history, int32_t history_cap, int32_t* history_len)
{
    return guarded(ctx, [&](Ctx& c) {
        check(opts != nullptr && rhs != nullptr && x != nullptr, ED_INVALID_ARGUMENT, "null argument");
        ensure_system(c, opts);
        const int64_t n = static_cast<int64_t>(c.sys.nv) + c.sys.np;
        DevArray<double> b, xd(n);
        b.upload(rhs, n, c.stream);
        std::vector<double> hist;
        const Stats st = solve_block_system_dev(c, b.p, xd.p, *opts, &hist, nullptr);
        xd.download(x, c.stream);
        c.sync();
        fill_stats(st, stats);
        copy_hist(hist, history, history_cap, history_len);
    });
}

int ed_newton_first_pass(ed_ctx* ctx, const ed_time_scalars* ts, const ed_block_solver_options* opts, double* x,
                         double* out_norm, ed_linear_stats* stats, double* history, int32_t history_cap,
                         int32_t* history_len, ed_phase_times* times)
{
    return guarded(ctx, [&](Ctx& c) {
        check(ts != nullptr && opts != nullptr, ED_INVALID_ARGUMENT, "null argument");
        check(c.have_dofs && c.have_mat, ED_NOT_READY, "problem not defined");
        cudaStream_t s = c.stream;
        ed_phase_times T{};
        const int64_t l0 = launch_count();
        const double t0 = now_ms();
        const double chi = ts->alpha_f * ts->gamma * ts->dt;
        const double gdt = ts->gamma * ts->dt;
        // predictor + stage blends: state arrays become the predictor iterate
        NewtonArgs na{};
        na.yn_u = c.u.p;
        na.yn_udot = c.udot.p;
        na.yn_p = c.p.p;
        na.yn_pdot = c.pdot.p;
        na.yn_v = c.v.p;
        na.yn_vdot = c.vdot.p;
        na.cur_u = c.u.p;
        na.cur_udot = c.udot.p;
        na.cur_p = c.p.p;
        na.cur_pdot = c.pdot.p;
        na.cur_v = c.v.p;
        na.cur_vdot = c.vdot.p;
        na.mid_u = c.m_u.p;
        na.mid_udot = c.m_udot.p;
        na.mid_p = c.m_p.p;
        na.mid_pdot = c.m_pdot.p;
        na.mid_v = c.m_v.p;
        na.mid_vdot = c.m_vdot.p;
        na.n_nodes = c.n_nodes;
        na.pf = (ts->gamma - 1.0) / ts->gamma;
        na.alpha_m = ts->alpha_m;
        na.alpha_f = ts->alpha_f;
        launch_predict_blend(na, s);
        // residual, rk, norm (timeint.cpp:98-110)
        double tp = now_ms();
        residual_on(c, true);
        check_bad(c, nullptr);
        T.residual_ms = now_ms() - tp;
        launch_kinematic_residual(c.d_fnode.p, c.nfree, c.m_udot.p, c.m_v.p, c.rk.p, s);
        DevArray<double> nr(3);
        const int64_t nvv = 3 * static_cast<int64_t>(c.nfree);
        dot(c.red, c.rk.p, c.rk.p, nvv, nr.p + 0, s);
        dot(c.red, c.rp.p, c.rp.p, c.n_nodes, nr.p + 1, s);
        dot(c.red, c.rm.p, c.rm.p, nvv, nr.p + 2, s);
        const std::vector<double> h = nr.to_host(s);
        if (out_norm) *out_norm = std::sqrt(h[0] + h[1] + h[2]);
        // tangent with element-local fold-in (timeint.cpp:141-154)
        tp = now_ms();
        tangent_on(c, true, *ts, true);
        check_bad(c, nullptr);
        ctx_planes_from_k4(c);
        launch_rhs(c.rm.p, c.rp.p, c.fv.p, c.fp.p, static_cast<int>(nvv), c.n_nodes, chi, c.rhs.p, s);
        c.sync();
        T.tangent_ms = now_ms() - tp;
        // solve (timeint.cpp:156)
        std::vector<double> hist;
        const Stats st = solve_block_system_dev(c, c.rhs.p, c.xsol.p, *opts, &hist, &T);
        // two-stage update (timeint.cpp:160-176)
        tp = now_ms();
        launch_update(c.d_fnode.p, c.nfree, c.n_nodes, c.xsol.p, c.rk.p, chi, ts->alpha_m, gdt, c.u.p, c.udot.p,
                      c.v.p, c.vdot.p, c.p.p, c.pdot.p, s);
        if (x) c.xsol.download(x, s);
        c.sync();
        T.update_ms = now_ms() - tp;
        T.total_ms = now_ms() - t0;
        T.kernel_launches = launch_count() - l0;
        c.times = T;
        if (times) *times = T;
        fill_stats(st, stats);
        copy_hist(hist, history, history_cap, history_len);
    });
}

int ed_step_generalized_alpha(ed_ctx* ctx, const ed_time_scalars* ts, const ed_nonlinear_config* nl,
                              const ed_block_solver_options* opts, ed_step_stats* out, ed_linear_stats* linear,
                              double* res_history, int32_t res_cap)
{
    return guarded(ctx, [&](Ctx& c) {
        check(ts != nullptr && nl != nullptr && opts != nullptr, ED_INVALID_ARGUMENT, "null argument");
        check(c.have_dofs && c.have_mat, ED_NOT_READY, "problem not defined");
        cudaStream_t s = c.stream;
        const int N = c.n_nodes;
        const int64_t n3 = 3LL * N;
        const double chi = ts->alpha_f * ts->gamma * ts->dt;
        const double gdt = ts->gamma * ts->dt;
        const int64_t nvv = 3 * static_cast<int64_t>(c.nfree);
        // y_n (converged state at t_n) and the iterate before the last update
        auto keep = [&](DevArray<double>& dst, const DevArray<double>& src) { dst.copy_from(src, s); };
        keep(c.y_u, c.u);
        keep(c.y_udot, c.udot);
        keep(c.y_p, c.p);
        keep(c.y_pdot, c.pdot);
        keep(c.y_v, c.v);
        keep(c.y_vdot, c.vdot);
        c.q_u.alloc(n3);
        c.q_udot.alloc(n3);
        c.q_p.alloc(N);
        c.q_pdot.alloc(N);
        c.q_v.alloc(n3);
        c.q_vdot.alloc(n3);
        NewtonArgs na{};
        na.yn_u = c.y_u.p;
        na.yn_udot = c.y_udot.p;
        na.yn_p = c.y_p.p;
        na.yn_pdot = c.y_pdot.p;
        na.yn_v = c.y_v.p;
        na.yn_vdot = c.y_vdot.p;
        na.cur_u = c.u.p;
        na.cur_udot = c.udot.p;
        na.cur_p = c.p.p;
        na.cur_pdot = c.pdot.p;
        na.cur_v = c.v.p;
        na.cur_vdot = c.vdot.p;
        na.mid_u = c.m_u.p;
        na.mid_udot = c.m_udot.p;
        na.mid_p = c.m_p.p;
        na.mid_pdot = c.m_pdot.p;
        na.mid_v = c.m_v.p;
        na.mid_vdot = c.m_vdot.p;
        na.n_nodes = N;
        na.pf = (ts->gamma - 1.0) / ts->gamma;
        na.alpha_m = ts->alpha_m;
        na.alpha_f = ts->alpha_f;
        NewtonArgs nh = na; // halving: prev in the yn slots
        nh.yn_u = c.q_u.p;
        nh.yn_udot = c.q_udot.p;
        nh.yn_p = c.q_p.p;
        nh.yn_pdot = c.q_pdot.p;
        nh.yn_v = c.q_v.p;
        nh.yn_vdot = c.q_vdot.p;
        // predictor + first stage blend (timeint.cpp:57-61, 88-93)
        launch_predict_blend(na, s);
        if (c.pd_n > 0) { // prescribed boundary motion of this step (one-shot)
            launch_prescribe(c.pd_nodes.p, c.pd_u.p, c.pd_n, na, gdt, s);
            launch_stage_blend(na, s);
            c.pd_n = 0;
        }
        ed_step_stats st{};
        Stats lin;
        std::vector<double> hist;
        constexpr double kGrowthCap = 4.0; // timeint.cpp:73
        double norm_prev = std::numeric_limits<double>::infinity();
        DevArray<double> nr(3);
        bool first_blend = true;
        for (int l = 1; l <= nl->l_max + 1; ++l) {
            double norm = 0.0;
            for (int halvings = 0;; ++halvings) {
                if (!first_blend) launch_stage_blend(na, s);
                first_blend = false;
                bool admissible = true;
                const double ta = now_ms();
                residual_on(c, true);
                int32_t bad = -1;
                try {
                    check_bad(c, &bad);
                } catch (const Error& e) {
                    if (e.code != ED_ELEMENT_INVERSION) throw;
                    admissible = false;
                }
                st.t_assembly += 1e-3 * (now_ms() - ta);
                if (admissible) {
                    launch_kinematic_residual(c.d_fnode.p, c.nfree, c.m_udot.p, c.m_v.p, c.rk.p, s);
                    dot(c.red, c.rk.p, c.rk.p, nvv, nr.p + 0, s);
                    dot(c.red, c.rp.p, c.rp.p, N, nr.p + 1, s);
                    dot(c.red, c.rm.p, c.rm.p, nvv, nr.p + 2, s);
                    const std::vector<double> h = nr.to_host(s);
                    norm = std::sqrt(h[0] + h[1] + h[2]);
                    if (std::isfinite(norm) && norm <= kGrowthCap * norm_prev) break;
                    admissible = false;
                }
                if (l == 1 || halvings >= 30) { // nothing to undo on the first pass
                    st.converged = 0;
                    goto done;
                }
                launch_halve(nh, s);
            }
            st.res_final = norm;
            hist.push_back(norm);
            norm_prev = norm;
            if (l == 1) st.res0 = norm;
            if (norm <= std::max(nl->tol_R * st.res0, nl->tol_A)) {
                st.converged = 1;
                goto done;
            }
            if (l > nl->l_max) break;
            {
                const double ta = now_ms();
                tangent_on(c, true, *ts, true);
                check_bad(c, nullptr);
                ctx_planes_from_k4(c);
                launch_rhs(c.rm.p, c.rp.p, c.fv.p, c.fp.p, static_cast<int>(nvv), N, chi, c.rhs.p, s);
                c.sync();
                st.t_assembly += 1e-3 * (now_ms() - ta);
                const Stats ls = solve_block_system_dev(c, c.rhs.p, c.xsol.p, *opts, nullptr, nullptr);
                lin.outer_iters += ls.outer_iters; // LinearStats::add (precond.hpp:30-41)
                lin.a_solves += ls.a_solves;
                lin.a_iters += ls.a_iters;
                lin.s_solves += ls.s_solves;
                lin.s_iters += ls.s_iters;
                lin.schur_applies += ls.schur_applies;
                lin.inner_iters += ls.inner_iters;
                lin.converged = lin.converged && ls.converged;
                lin.t_solve += ls.t_solve;
                st.newton_iters += 1;
                // prev = cur, then the two-stage update of cur (timeint.cpp:160-176)
                keep(c.q_u, c.u);
                keep(c.q_udot, c.udot);
                keep(c.q_p, c.p);
                keep(c.q_pdot, c.pdot);
                keep(c.q_v, c.v);
                keep(c.q_vdot, c.vdot);
                launch_update(c.d_fnode.p, c.nfree, N, c.xsol.p, c.rk.p, chi, ts->alpha_m, gdt, c.u.p, c.udot.p,
                              c.v.p, c.vdot.p, c.p.p, c.pdot.p, s);
            }
        }
        st.converged = 0;
    done:
        c.sync();
        st.n_res = static_cast<int32_t>(hist.size());
        if (res_history)
            for (int i = 0; i < res_cap && i < static_cast<int>(hist.size()); ++i) res_history[i] = hist[i];
        if (out) *out = st;
        fill_stats(lin, linear);
    });
}

int ed_block_matvec(ed_ctx* ctx, const double* x, double* y)
{
    return guarded(ctx, [&](Ctx& c) {
        ensure_system(c, nullptr);
        const int nv = c.sys.nv, np = c.sys.np;
        DevArray<double> xd, yd(static_cast<size_t>(nv) + np);
        xd.upload(x, static_cast<size_t>(nv) + np, c.stream);
        spmv2(c.sys.A, xd.p, c.sys.B, xd.p + nv, yd.p, 1.0, c.stream);
        spmv2(c.sys.C, xd.p, c.sys.D, xd.p + nv, yd.p + nv, 1.0, c.stream);
        yd.download(y, c.stream);
        c.sync();
    });
}

int ed_coupled_matvec(ed_ctx* ctx, const ed_block_solver_options* opts, const double* x, double* y_coupled,
                      double* y_planes)
{
    return guarded(ctx, [&](Ctx& c) {
        check(opts && x && y_coupled && y_planes, ED_INVALID_ARGUMENT, "bad arguments");
        ensure_system(c, opts);
        WorkSys& W = c.work;
        make_work(c, W, opts->scale != 0, opts->eps_diag);
        check(W.K.n_nodes > 0, ED_NOT_READY, "no coupled operator (the system was not assembled from a mesh)");
        const int nv = W.nv;
        const size_t n = static_cast<size_t>(nv) + W.np;
        DevArray<double> xd, y1(n), y2(n);
        xd.upload(x, n, c.stream);
        spmv44(W.K, xd.p, y1.p, nv, W.np, c.stream);
        spmv2(W.A, xd.p, W.B, xd.p + nv, y2.p, 1.0, c.stream);
        spmv2(W.C, xd.p, W.D, xd.p + nv, y2.p + nv, 1.0, c.stream);
        y1.download(y_coupled, c.stream);
        y2.download(y_planes, c.stream);
        c.sync();
    });
}

int ed_block_matvec_device(ed_ctx* ctx, const double* d_x, double* d_y, int n_rep, float* ms)
{
    return guarded(ctx, [&](Ctx& c) {
        ensure_system(c, nullptr);
        const int nv = c.sys.nv;
        cudaEvent_t e0, e1;
        ED_CUDA(cudaEventCreate(&e0));
        ED_CUDA(cudaEventCreate(&e1));
        ED_CUDA(cudaEventRecord(e0, c.stream));
        for (int r = 0; r < n_rep; ++r) {
            spmv2(c.sys.A, d_x, c.sys.B, d_x + nv, d_y, 1.0, c.stream);
            spmv2(c.sys.C, d_x, c.sys.D, d_x + nv, d_y + nv, 1.0, c.stream);
        }
        ED_CUDA(cudaEventRecord(e1, c.stream));
        ED_CUDA(cudaEventSynchronize(e1));
        float t = 0.0f;
        ED_CUDA(cudaEventElapsedTime(&t, e0, e1));
        if (ms) *ms = t;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

int ed_spmv_bytes(ed_ctx* ctx, double* coupled_bytes, double* a_plane_bytes)
{
    return guarded(ctx, [&](Ctx& c) {
        ensure_system(c, nullptr);
        const BlockSys& S = c.sys;
        // coupled: mesh systems run the 4x4 BSR (one index per node
        // block); uploaded CSR systems the split planes (every plane's blocks + indices)
        double cb = 0.0;
        if (c.sys_from_mesh && S.Bv == 3) {
            cb = static_cast<double>(S.D.st->nnzb) * 132.0 + 4.0 * (S.D.st->nbr + 1) +
                 16.0 * (static_cast<double>(S.nv) + S.np);
        } else {
            const double blocks = S.A.st->nnzb * (8.0 * S.Bv * S.Bv + 4.0) + S.B.st->nnzb * (8.0 * S.Bv + 4.0) +
                                  S.C.st->nnzb * (8.0 * S.Bv + 4.0) + S.D.st->nnzb * 12.0;
            cb = blocks + 2.0 * 8.0 * (static_cast<double>(S.nv) + S.np) + 4.0 * (S.A.st->nbr + S.C.st->nbr + 2);
        }
        if (coupled_bytes) *coupled_bytes = cb;
        if (a_plane_bytes) *a_plane_bytes = S.A.bytes_per_spmv();
    });
}

int ed_gmres_a(ed_ctx* ctx, const double* b, double* x, const ed_krylov_config* cfg, int flexible, int precond,
               const ed_amg_options* amg, ed_solve_result* res, double* history, int32_t history_cap,
               int32_t* history_len)
{
    return guarded(ctx, [&](Ctx& c) {
        check(cfg && b && x, ED_INVALID_ARGUMENT, "null argument");
        ed_block_solver_options o{};
        if (amg) o.amg_a = *amg;
        else o.amg_a.block_size = 1;
        ensure_system(c, &o);
        const Bsr& A = c.sys.A;
        const int n = A.nrows();
        struct Op final : DOp {
            const Bsr& M;
            cudaStream_t s;
            Op(const Bsr& m, cudaStream_t st) : M(m), s(st) {}
            int64_t size() const override { return M.nrows(); }
            void apply(const double* xx, double* yy) override { spmv(M, xx, yy, nullptr, 0, s); }
        } op(A, c.stream);
        struct Jac final : DPrec {
            DevArray<double> invd;
            cudaStream_t s;
            int64_t n;
            void apply(const double* r, double* z) override
            {
                vec_copy(z, r, n, s);
                vec_mul(z, invd.p, n, s);
            }
        } jac;
        struct Amg final : DPrec {
            Ctx& c;
            DevHierarchy h;
            explicit Amg(Ctx& cc) : c(cc) {}
            void apply(const double* r, double* z) override { h.vcycle(c, r, z); }
        } amgp(c);
        DPrec* M = nullptr;
        if (precond == 1) {
            DevArray<double> d(n);
            bsr_diag(A, d.p, c.stream);
            jac.invd.alloc(n);
            inv_diag_from(d.p, jac.invd.p, n, c.stream);
            jac.s = c.stream;
            jac.n = n;
            c.sync();
            M = &jac;
        } else if (precond == 2) {
            check(amg != nullptr, ED_INVALID_ARGUMENT, "AMG options missing");
            amgp.h.build(c, A, amg_opts_from(*amg, c, true, n));
            M = &amgp;
        }
        DevArray<double> bd, xd;
        bd.upload(b, n, c.stream);
        xd.upload(x, n, c.stream);
        KrylovCfg k{cfg->restart, cfg->max_iters, cfg->rel_tol, cfg->abs_tol};
        KrylovWs ws;
        const SolveRes r = gmres_dev(c, op, M, bd.p, xd.p, k, flexible != 0, ws);
        xd.download(x, c.stream);
        c.sync();
        if (res) {
            res->converged = r.converged ? 1 : 0;
            res->iterations = r.iterations;
            res->initial_norm = r.initial_norm;
            res->final_norm = r.final_norm;
        }
        copy_hist(r.history, history, history_cap, history_len);
    });
}

int ed_amg_vcycle(ed_ctx* ctx, int which, const ed_block_solver_options* opts, const double* r, double* z,
                  int32_t* info)
{
    return guarded(ctx, [&](Ctx& c) {
        check(opts && r && z, ED_INVALID_ARGUMENT, "null argument");
        ensure_system(c, opts);
        DevHierarchy h;
        const Bsr* A = nullptr;
        if (which == 0) {
            A = &c.sys.A;
            h.build(c, *A, amg_opts_from(opts->amg_a, c, true, A->nrows()));
        } else {
            make_work(c, c.work, opts->scale != 0, opts->eps_diag);
            build_shat_work(c, c.work);
            A = &c.work.S;
            h.build(c, *A, amg_opts_from(opts->amg_s, c, false, A->nrows()));
        }
        const int n = A->nrows();
        DevArray<double> rd, zd(n);
        rd.upload(r, n, c.stream);
        h.vcycle(c, rd.p, zd.p);
        zd.download(z, c.stream);
        c.sync();
        if (info) {
            info[0] = h.fallback ? 0 : h.n_levels();
            info[1] = h.fallback ? 1 : 0;
            for (int l = 0; l < h.n_levels() && l < 16; ++l) info[2 + l] = h.level_rows[l];
            if (h.fallback) info[2] = n;
        }
    });
}

int ed_shat_export(ed_ctx* ctx, const ed_block_solver_options* opts, int32_t* dims, int32_t* rowptr, int32_t* col,
                   double* val)
{
    return guarded(ctx, [&](Ctx& c) {
        check(opts != nullptr, ED_INVALID_ARGUMENT, "options missing");
        ensure_system(c, opts);
        make_work(c, c.work, opts->scale != 0, opts->eps_diag);
        build_shat_work(c, c.work);
        const HostCsr a = bsr_to_csr(c.work.S, c.stream);
        if (dims) {
            dims[0] = a.nrows;
            dims[1] = a.ncols;
            dims[2] = static_cast<int32_t>(a.nnz());
        }
        if (rowptr) {
            for (size_t i = 0; i < a.rowptr.size(); ++i) rowptr[i] = static_cast<int32_t>(a.rowptr[i]);
            std::copy(a.col.begin(), a.col.end(), col);
            std::copy(a.val.begin(), a.val.end(), val);
        }
    });
}

int ed_state_save(ed_ctx* ctx)
{
    return guarded(ctx, [&](Ctx& c) {
        check(c.have_dofs, ED_NOT_READY, "dofs required");
        c.s_u.copy_from(c.u, c.stream);
        c.s_udot.copy_from(c.udot, c.stream);
        c.s_p.copy_from(c.p, c.stream);
        c.s_pdot.copy_from(c.pdot, c.stream);
        c.s_v.copy_from(c.v, c.stream);
        c.s_vdot.copy_from(c.vdot, c.stream);
        c.sync();
    });
}

int ed_state_restore(ed_ctx* ctx)
{
    return guarded(ctx, [&](Ctx& c) {
        check(c.s_u.n == c.u.n && c.s_u.p, ED_NOT_READY, "no saved state");
        c.u.copy_from(c.s_u, c.stream);
        c.udot.copy_from(c.s_udot, c.stream);
        c.p.copy_from(c.s_p, c.stream);
        c.pdot.copy_from(c.s_pdot, c.stream);
        c.v.copy_from(c.s_v, c.stream);
        c.vdot.copy_from(c.s_vdot, c.stream);
    });
}

int ed_timer(ed_ctx* ctx, int op, float* ms)
{
    return guarded(ctx, [&](Ctx& c) {
        if (!c.ev0) {
            ED_CUDA(cudaEventCreate(&c.ev0));
            ED_CUDA(cudaEventCreate(&c.ev1));
        }
        if (op == 0) {
            ED_CUDA(cudaEventRecord(c.ev0, c.stream));
        } else {
            ED_CUDA(cudaEventRecord(c.ev1, c.stream));
            ED_CUDA(cudaEventSynchronize(c.ev1));
            float t = 0.0f;
            ED_CUDA(cudaEventElapsedTime(&t, c.ev0, c.ev1));
            if (ms) *ms = t;
        }
    });
}

int ed_bench_kernels(ed_ctx* ctx, const ed_block_solver_options* opts, int n_rep, double* out)
{
    return guarded(ctx, [&](Ctx& c) {
        check(opts && out && n_rep > 0, ED_INVALID_ARGUMENT, "bad arguments");
        ensure_system(c, opts);
        WorkSys& W = c.work;
        make_work(c, W, opts->scale != 0, opts->eps_diag);
        build_shat_work(c, W);
        const int64_t n = static_cast<int64_t>(W.nv) + W.np;
        DevArray<double> x(n), y(n), invd(W.nv), d(W.nv);
        vec_fill(x.p, 1.0, n, c.stream);
        vec_fill(y.p, 0.0, n, c.stream);
        bsr_diag(W.A, d.p, c.stream);
        inv_diag_from(d.p, invd.p, W.nv, c.stream);
        cudaEvent_t e0, e1;
        ED_CUDA(cudaEventCreate(&e0));
        ED_CUDA(cudaEventCreate(&e1));
        auto time = [&](auto&& f) {
            f(); // warm
            ED_CUDA(cudaEventRecord(e0, c.stream));
            for (int r = 0; r < n_rep; ++r) f();
            ED_CUDA(cudaEventRecord(e1, c.stream));
            ED_CUDA(cudaEventSynchronize(e1));
            float t = 0.0f;
            ED_CUDA(cudaEventElapsedTime(&t, e0, e1));
            return static_cast<double>(t) / n_rep;
        };
        const int nv = W.nv;
        const BlockSys& S = c.sys;
        if (W.K.n_nodes > 0) {
            // the coupled 4x4 BSR the outer FGMRES uses; SURVEY 8d bytes
            out[0] = time([&] { spmv44(W.K, x.p, y.p, nv, W.np, c.stream); });
            out[1] = W.K.bytes(static_cast<int64_t>(nv) + W.np);
        } else {
            out[0] = time([&] {
                spmv2(W.A, x.p, W.B, x.p + nv, y.p, 1.0, c.stream);
                spmv2(W.C, x.p, W.D, x.p + nv, y.p + nv, 1.0, c.stream);
            });
            out[1] = S.A.st->nnzb * (8.0 * S.Bv * S.Bv + 4.0) + S.B.st->nnzb * (8.0 * S.Bv + 4.0) +
                     S.C.st->nnzb * (8.0 * S.Bv + 4.0) + S.D.st->nnzb * 12.0 +
                     2.0 * 8.0 * (static_cast<double>(S.nv) + S.np) + 4.0 * (S.A.st->nbr + S.C.st->nbr + 2);
        }
        out[2] = time([&] { spmv(W.A, x.p, y.p, nullptr, 0, c.stream); });
        out[3] = W.A.bytes_per_spmv();
        DevArray<double> gd;
        sweep_prepare(W.A, invd.p, gd, c.stream);
        out[4] = time([&] { sgs_sweep(W.A, x.p, y.p, invd.p, true, c.stream, gd.p); });
        // values+indices once, plus b and inv_diag read, z read+written
        out[5] = W.A.st->nnzb * (8.0 * W.Bv * W.Bv + 4.0) + 4.0 * (W.A.st->nbr + 1) + 4.0 * 8.0 * nv;
        out[6] = time([&] { spmv(W.S, x.p, y.p, nullptr, 0, c.stream); });
        out[7] = W.S.bytes_per_spmv();
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}


int ed_bench_assembly(ed_ctx* ctx, const ed_time_scalars* ts, int n_rep, double* out)
{
    return guarded(ctx, [&](Ctx& c) {
        check(ts && out && n_rep > 0, ED_INVALID_ARGUMENT, "bad arguments");
        check(c.have_dofs && c.have_mat && c.sys_from_mesh, ED_NOT_READY, "assemble the tangent once first");
        cudaEvent_t e0, e1;
        ED_CUDA(cudaEventCreate(&e0));
        ED_CUDA(cudaEventCreate(&e1));
        auto time = [&](auto&& f) {
            f(); // warm
            ED_CUDA(cudaEventRecord(e0, c.stream));
            for (int r = 0; r < n_rep; ++r) f();
            ED_CUDA(cudaEventRecord(e1, c.stream));
            ED_CUDA(cudaEventSynchronize(e1));
            float t = 0.0f;
            ED_CUDA(cudaEventElapsedTime(&t, e0, e1));
            return static_cast<double>(t) / n_rep;
        };
        if (c.rk.n < 3 * static_cast<size_t>(c.nfree)) { // fold-in with a zero kinematic residual
            c.rk.alloc(3 * static_cast<size_t>(c.nfree));
            c.rk.zero(c.stream);
        }
        reset_bad(c);
        AsmArgs A = asm_args(c, false);
        A.ts = *ts;
        A.rk = c.rk.p;
        // residual: zero R, element kernels, tractions (residual_on without its host sync)
        out[0] = time([&] {
            c.rm.zero(c.stream);
            c.rp.zero(c.stream);
            launch_residual(A, c.color_ptr, c.stream);
            launch_traction(c.tr_rowptr.p, c.tr_rows.p, c.tr_vals.p, c.tr_n, c.rm.p, c.stream);
        });
        // tangent with the fold-in, K4 staging and the four BSR planes
        out[2] = time([&] {
            c.k4.zero(c.stream);
            c.fv.zero(c.stream);
            c.fp.zero(c.stream);
            launch_tangent(A, c.color_ptr, c.stream);
            ctx_planes_from_k4(c);
        });
        check_bad(c, nullptr);
        // algorithmic bytes: per element connectivity 16 B + grad N / volume / tau 112 B;
        // state 11 doubles per node; outputs written once
        const double E = c.n_tets, Nn = c.n_nodes, nv = 3.0 * c.nfree, np = c.n_nodes;
        const BlockSys& S = c.sys;
        const double planes = S.A.st->nnzb * 8.0 * S.Bv * S.Bv + S.B.st->nnzb * 8.0 * S.Bv +
                              S.C.st->nnzb * 8.0 * S.Bv + S.D.st->nnzb * 8.0;
        out[1] = 128.0 * E + 88.0 * Nn + 8.0 * (nv + np);
        out[3] = 128.0 * E + 88.0 * Nn + 8.0 * nv + planes + 8.0 * (nv + np);
        // FP64 FMA peak of this device (2 flops per fma)
        DevArray<double> sink(1);
        const int iters = 1 << 14;
        const double fl = launch_fp64_fma(sink.p, iters, c.stream);
        const double ms = time([&] { launch_fp64_fma(sink.p, iters, c.stream); });
        out[4] = fl / (ms * 1e-3) / 1e9;
        out[5] = E;
        out[6] = planes;
        out[7] = static_cast<double>(c.k4.n) * 8.0; // K4 staging array bytes (written once, read once)
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

} // extern "C"

extern "C" {

int ed_kernel_accounting(ed_ctx* ctx, int on)
{
    return guarded(ctx, [&](Ctx& c) {
        c.sync();
        std::lock_guard<std::mutex> lk(g_acct_mu);
        g_acct.flush();
        if (on) g_acct.tot.clear();
        g_acct.on = on != 0;
    });
}

int ed_kernel_account_count(ed_ctx* ctx, int* n)
{
    return guarded(ctx, [&](Ctx& c) {
        check(n != nullptr, ED_INVALID_ARGUMENT, "null count");
        c.sync();
        std::lock_guard<std::mutex> lk(g_acct_mu);
        g_acct.flush();
        *n = static_cast<int>(g_acct.tot.size());
    });
}

int ed_kernel_account_get(ed_ctx* ctx, int idx, char* name, int name_cap, int64_t* launches, double* ms,
                          double* bytes)
{
    return guarded(ctx, [&](Ctx&) {
        check(idx >= 0 && idx < static_cast<int>(g_acct.tot.size()), ED_INVALID_ARGUMENT, "index out of range");
        auto it = g_acct.tot.begin();
        std::advance(it, idx);
        if (name && name_cap > 0) {
            std::strncpy(name, it->first.c_str(), static_cast<size_t>(name_cap) - 1);
            name[name_cap - 1] = '\0';
        }
        if (launches) *launches = it->second.n;
        if (ms) *ms = it->second.ms;
        if (bytes) *bytes = it->second.bytes;
    });
}

} // extern "C"

// VMS residual / consistent-tangent assembly for P1 tets on sm_100a (FP64).
//
// One 16-lane team per element; the element frame (F, J, F^-1, C, C^-1,
// J^-2/3, stresses, spatial gradients, per-quadrature-point volumetric data
// and the 12 directional derivatives of P~) is staged in shared memory, then
// lane (a, b) forms node block (a, b) of the element matrices and adds it to
// the 4x4 node-block array K4 (A 3x3 | B 3x1 / C 1x3 | D).  Scatter is
// deterministic without float atomics: elements are processed colour by
// colour (no two elements of a colour share a node), so every K4 block and
// residual entry is summed in a fixed order.
//
// Arithmetic follows the reference expression by expression
// (assembly.cpp:69-109,113-185,187-352; materials.cpp:8-53,82-129;
// smallmat.hpp) and is compiled with -fmad=false, so element matrices agree
// with the reference to the last bit up to libm differences in pow/exp; the
// summation order of element contributions differs from from_triplets'
// unstable sort (csr.cpp:84-87), hence parity is at roundoff level.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "ed_internal.hpp"
#include "assembly.hpp"

namespace edb {

namespace {

constexpr int kTeam = 16;


// 4-point degree-2 rule (quadrature.hpp:18-26)
__constant__ double c_qa = 0.5854101966249685;
__constant__ double c_qb = 0.1381966011250105;

__device__ __forceinline__ double bary(int q, int a) { return q == a ? c_qa : c_qb; }

// ---- smallmat.hpp restated on the device (row-major Mat3) -----------------
__device__ __forceinline__ double det3(const double* m)
{
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}

__device__ __forceinline__ void inv3(const double* m, double* r)
{
    const double d = det3(m);
    const double id = 1.0 / d;
    r[0] = (m[4] * m[8] - m[5] * m[7]) * id;
    r[1] = (m[2] * m[7] - m[1] * m[8]) * id;
    r[2] = (m[1] * m[5] - m[2] * m[4]) * id;
    r[3] = (m[5] * m[6] - m[3] * m[8]) * id;
    r[4] = (m[0] * m[8] - m[2] * m[6]) * id;
    r[5] = (m[2] * m[3] - m[0] * m[5]) * id;
    r[6] = (m[3] * m[7] - m[4] * m[6]) * id;
    r[7] = (m[1] * m[6] - m[0] * m[7]) * id;
    r[8] = (m[0] * m[4] - m[1] * m[3]) * id;
}

__device__ __forceinline__ void matmul3(const double* a, const double* b, double* c)
{
    double t[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) t[k] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double aik = a[3 * i + k];
#pragma unroll
            for (int j = 0; j < 3; ++j) t[3 * i + j] = t[3 * i + j] + aik * b[3 * k + j];
        }
#pragma unroll
    for (int k = 0; k < 9; ++k) c[k] = t[k];
}

// a^T b
__device__ __forceinline__ void matTmul3(const double* a, const double* b, double* c)
{
    double t[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) t[k] = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double aki = a[3 * k + i];
#pragma unroll
            for (int j = 0; j < 3; ++j) t[3 * i + j] = t[3 * i + j] + aki * b[3 * k + j];
        }
#pragma unroll
    for (int k = 0; k < 9; ++k) c[k] = t[k];
}

__device__ __forceinline__ double ddot3(const double* a, const double* b)
{
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) s = s + a[k] * b[k];
    return s;
}

__device__ __forceinline__ double dot3(const double* a, const double* b)
{
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// ---- materials (materials.hpp:41-113, materials.cpp:21-53) ---------------
struct Vol {
    double rho, beta, drho, dbeta;
};

__device__ __forceinline__ Vol volumetric(const ed_material& m, double p)
{
    Vol v;
    if (m.incompressible) {
        v.rho = m.rho0;
        v.beta = 0.0;
        v.drho = 0.0;
        v.dbeta = 0.0;
        return v;
    }
    const double k = m.kappa;
    const double s = sqrt(p * p + k * k);
    const double ratio = p >= 0.0 ? (s + p) / k : k / (s - p);
    v.rho = m.rho0 * ratio;
    v.beta = 1.0 / s;
    v.drho = v.rho / s;
    v.dbeta = -p / (s * s * s);
    return v;
}

// Hs: the element's two fibre structure tensors (the material's global ones,
// materials.cpp:67-80, or the element's entry of the fibre field)
__device__ __forceinline__ void iso_stress(const ed_material& m, const double (*Hs)[9], const double* Ct, double* S)
{
#pragma unroll
    for (int k = 0; k < 9; ++k) S[k] = (k == 0 || k == 4 || k == 8) ? m.mu : 0.0;
    if (m.kind == 1) {
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const double* H = Hs[f];
            const double E = ddot3(H, Ct) - 1.0;
            const double q = fmin(m.k2 * E * E, 500.0);
            const double sb = 2.0 * m.k1 * E * exp(q);
#pragma unroll
            for (int k = 0; k < 9; ++k) S[k] = S[k] + sb * H[k];
        }
    }
}

__device__ __forceinline__ void iso_stress_dir(const ed_material& m, const double (*Hs)[9], const double* Ct,
                                               const double* dCt, double* dS)
{
#pragma unroll
    for (int k = 0; k < 9; ++k) dS[k] = 0.0;
    if (m.kind == 1) {
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const double* H = Hs[f];
            const double E = ddot3(H, Ct) - 1.0;
            const double q = fmin(m.k2 * E * E, 500.0);
            const double c = 2.0 * m.k1 * (1.0 + 2.0 * m.k2 * E * E) * exp(q);
            const double sb = c * ddot3(H, dCt);
#pragma unroll
            for (int k = 0; k < 9; ++k) dS[k] = dS[k] + sb * H[k];
        }
    }
}

// Element frame in shared memory (ElementFrame, assembly.cpp:57-67).
struct Frame {
    double G[4][3];
    double u[4][3], v[4][3], vd[4][3], rk[4][3];
    double pe[4], pde[4];
    double F[9], Finv[9], C[9], Cinv[9], Ct[9];
    double St[9], Siso[9], Pt[9];
    double g[4][3];
    double L[9], gp[3];
    double J, Jm23, divv, pbar, vol, tau;
    // per quadrature point
    double pq[4], pdq[4], vdq[4][3], rho[4], beta[4], drho[4], dbeta[4], vmb[4][3], res[4][3], cont[4];
    double dP[12][9];
    double H[2][9]; // fibre structure tensors of this element (kind 1)
    int nodes[4];
    int free_idx[4];
    int valid;
    int active; // the team has an element
    int elem;   // its element id
};

// ptilde_dir (materials.cpp:108-129) for dF = e_j (x) G_b
__device__ void ptilde_dir(const ed_material& m, const Frame& f, int bn, int j, double* out)
{
    // dF = e_j (x) G_b, built with selects (no dynamically indexed local array)
    double dF[9];
    const double g0 = f.G[bn][0], g1 = f.G[bn][1], g2 = f.G[bn][2];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        dF[3 * r + 0] = r == j ? g0 : 0.0;
        dF[3 * r + 1] = r == j ? g1 : 0.0;
        dF[3 * r + 2] = r == j ? g2 : 0.0;
    }
    // t = ddot3(transpose3(Finv), dF)
    double FinvT[9] = {f.Finv[0], f.Finv[3], f.Finv[6], f.Finv[1], f.Finv[4], f.Finv[7],
                       f.Finv[2], f.Finv[5], f.Finv[8]};
    const double t = ddot3(FinvT, dF);
    double a1[9], a2[9], dC[9];
    matTmul3(dF, f.F, a1);
    matTmul3(f.F, dF, a2);
#pragma unroll
    for (int k = 0; k < 9; ++k) dC[k] = a1[k] + 1.0 * a2[k];
    const double dJm23 = -2.0 / 3.0 * f.Jm23 * t;
    double dCt[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) dCt[k] = dC[k] * f.Jm23 + dJm23 * f.C[k];
    double dS[9];
    iso_stress_dir(m, f.H, f.Ct, dCt, dS);
    double tmp[9], dCinv[9];
    matmul3(dC, f.Cinv, tmp);
    matmul3(f.Cinv, tmp, dCinv);
#pragma unroll
    for (int k = 0; k < 9; ++k) dCinv[k] = dCinv[k] * -1.0;
    const double sc = ddot3(f.St, f.Ct);
    const double dsc = ddot3(dS, f.Ct) + ddot3(f.St, dCt);
    double dSiso[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) dSiso[k] = f.St[k] * dJm23;
#pragma unroll
    for (int k = 0; k < 9; ++k) dSiso[k] = dSiso[k] + 1.0 * (dS[k] * f.Jm23);
    const double c1 = -dsc / 3.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) dSiso[k] = dSiso[k] + c1 * f.Cinv[k];
    const double c2 = -sc / 3.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) dSiso[k] = dSiso[k] + c2 * dCinv[k];
    double b1[9], b2[9];
    matmul3(dF, f.Siso, b1);
    matmul3(f.F, dSiso, b2);
#pragma unroll
    for (int k = 0; k < 9; ++k) out[k] = b1[k] + 1.0 * b2[k];
}

// Phases A-C shared by residual and tangent kernels, for the kTeamsPerCta
// elements of a CTA at once.  The per-element serial work (kinematics, stress,
// div v / L / grad p, quadrature-point data) is ROLE-MAJOR: thread t of the CTA
// does job t / T for element t % T (T = 8 elements per CTA), so a warp that
// issues FP64 instructions in these phases has all 32 lanes active and the
// other warps wait at the CTA barrier.  (A predicated-off lane costs the FP64
// pipe as much as an active one; with team-local lanes 0..3 doing this work the
// serial phases ran at 1-4 active lanes of 16.  160^3: residual 23.7 -> 17.5 ms,
// tangent 103.2 -> 99.6 ms; 16 or 32 elements per CTA lose the overlap between
// CTAs and are slower for the tangent, profiles/r02/assembly_experiments.md.)
// The arithmetic per element is unchanged.
// All threads of the CTA call it (it contains __syncthreads); f.valid == 0
// afterwards for an inactive team or an inverted element.
template <int T>
__device__ void build_frames(const AsmArgs& A, Frame* frames, int c0, int count, bool with_rk)
{
    const int t = threadIdx.x;
    // --- A: gather (thread = (element, node))
    if (t < 4 * T) {
        const int team = t >> 2, a = t & 3;
        Frame& f = frames[team];
        const int idx = blockIdx.x * T + team;
        const bool active = idx < count;
        if (a == 0) f.active = active;
        if (active) {
            const int e = A.elem_order[c0 + idx];
            const int n = A.tets[4 * static_cast<int64_t>(e) + a];
            f.nodes[a] = n;
            const int fi = A.fidx[n];
            f.free_idx[a] = fi;
#pragma unroll
            for (int I = 0; I < 3; ++I) f.G[a][I] = A.grad_n[12 * static_cast<int64_t>(e) + 3 * a + I];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                f.u[a][i] = A.u[3 * static_cast<int64_t>(n) + i];
                f.v[a][i] = A.v[3 * static_cast<int64_t>(n) + i];
                f.vd[a][i] = A.vdot[3 * static_cast<int64_t>(n) + i];
                f.rk[a][i] = (with_rk && A.rk && fi >= 0) ? A.rk[3 * static_cast<int64_t>(fi) + i] : 0.0;
            }
            f.pe[a] = A.p[n];
            f.pde[a] = A.pdot[n];
            if (a == 0) {
                f.elem = e;
                f.vol = A.volume[e];
                f.tau = A.tau[e];
            }
            if (A.mat.kind == 1 && a >= 1 && a <= 2) {
                // per-element fibre field (local frames) or the material's global tensors
                const int fam = a - 1;
                const double* H =
                    A.elem_h ? A.elem_h + 18 * static_cast<int64_t>(e) + 9 * fam : (fam ? A.mat.h2 : A.mat.h1);
#pragma unroll
                for (int k = 0; k < 9; ++k) f.H[fam][k] = H[k];
            }
        }
    }
    __syncthreads();
    // --- B: kinematics (Kinematics::from_F).  The three independent chains -- F^-1; C = F^T F
    // and C^-1; J^-2/3 -- are jobs 0, 1, 2 (each recomputes F and J identically).
    if (t < 3 * T) {
        const int job = t / T;
        Frame& f = frames[t % T];
        if (f.active) {
            double F[9] = {1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0};
            for (int a = 0; a < 4; ++a)
                for (int i = 0; i < 3; ++i)
                    for (int I = 0; I < 3; ++I) F[3 * i + I] = F[3 * i + I] + f.u[a][i] * f.G[a][I];
            const double J = det3(F);
            if (!(J > 0.0)) {
                if (job == 0) {
                    f.valid = 0;
                    atomicMin(A.bad_element, f.elem);
                }
            } else if (job == 0) {
                f.valid = 1;
#pragma unroll
                for (int k = 0; k < 9; ++k) f.F[k] = F[k];
                f.J = J;
                inv3(F, f.Finv);
            } else if (job == 1) {
                matTmul3(F, F, f.C);
                inv3(f.C, f.Cinv);
            } else {
                f.Jm23 = pow(J, -2.0 / 3.0);
            }
        } else if (job == 0) {
            f.valid = 0;
        }
    }
    __syncthreads();
    // --- stress (evaluate_stress) and C1: spatial gradients g_a = F^-T G_a (tmulvec3), jobs 1..4
    if (t < T) {
        Frame& f = frames[t];
        if (f.valid) {
#pragma unroll
            for (int k = 0; k < 9; ++k) f.Ct[k] = f.C[k] * f.Jm23;
            iso_stress(A.mat, f.H, f.Ct, f.St);
            const double sc = ddot3(f.St, f.Ct);
            const double c1 = -sc / 3.0;
#pragma unroll
            for (int k = 0; k < 9; ++k) f.Siso[k] = f.St[k] * f.Jm23 + c1 * f.Cinv[k];
            matmul3(f.F, f.Siso, f.Pt);
        }
    } else if (t < 5 * T) {
        Frame& f = frames[t % T];
        if (f.valid) {
            const int a = t / T - 1;
            const double* m = f.Finv;
            const double* x = f.G[a];
            f.g[a][0] = m[0] * x[0] + m[3] * x[1] + m[6] * x[2];
            f.g[a][1] = m[1] * x[0] + m[4] * x[1] + m[7] * x[2];
            f.g[a][2] = m[2] * x[0] + m[5] * x[1] + m[8] * x[2];
        }
    }
    __syncthreads();
    // --- C2: div v, L, grad p (job 0), quadrature-point values (jobs 1..4)
    if (t < T) {
        Frame& f = frames[t];
        if (f.valid) {
            double divv = 0.0, gp[3] = {0.0, 0.0, 0.0}, L[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) L[k] = 0.0;
            for (int a = 0; a < 4; ++a) {
                divv = divv + dot3(f.v[a], f.g[a]);
                for (int i = 0; i < 3; ++i) {
                    gp[i] = gp[i] + f.pe[a] * f.g[a][i];
                    for (int j = 0; j < 3; ++j) L[3 * i + j] = L[3 * i + j] + f.v[a][i] * f.g[a][j];
                }
            }
            f.divv = divv;
#pragma unroll
            for (int i = 0; i < 3; ++i) f.gp[i] = gp[i];
#pragma unroll
            for (int k = 0; k < 9; ++k) f.L[k] = L[k];
        }
    } else if (t < 5 * T) {
        Frame& f = frames[t % T];
        if (f.valid) {
            const int q = t / T - 1;
            double pq = 0.0, pdq = 0.0, vdq[3] = {0.0, 0.0, 0.0};
            for (int a = 0; a < 4; ++a) {
                const double Na = bary(q, a);
                pq = pq + Na * f.pe[a];
                pdq = pdq + Na * f.pde[a];
                for (int i = 0; i < 3; ++i) vdq[i] = vdq[i] + Na * f.vd[a][i];
            }
            f.pq[q] = pq;
            f.pdq[q] = pdq;
#pragma unroll
            for (int i = 0; i < 3; ++i) f.vdq[q][i] = vdq[i];
            const Vol vm = volumetric(A.mat, pq);
            f.rho[q] = vm.rho;
            f.beta[q] = vm.beta;
            f.drho[q] = vm.drho;
            f.dbeta[q] = vm.dbeta;
        }
    }
    __syncthreads();
    // --- C3: strong residual terms per quadrature point (jobs 1..4), pbar (job 0)
    if (t < T) {
        Frame& f = frames[t];
        if (f.valid) {
            // pbar += w_q * pq with w_q = 1/4, q ascending (assembly.cpp:142); pq
            // is recomputed here in the same order as the quadrature jobs did
            double pbar = 0.0;
            for (int q = 0; q < 4; ++q) {
                double pq = 0.0;
                for (int a = 0; a < 4; ++a) pq = pq + bary(q, a) * f.pe[a];
                pbar = pbar + 0.25 * pq;
            }
            f.pbar = pbar;
        }
    } else if (t < 5 * T) {
        Frame& f = frames[t % T];
        if (f.valid) {
            const int q = t / T - 1;
            const double J = f.J;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                f.vmb[q][i] = f.vdq[q][i] - A.body_force[i];
                f.res[q][i] = f.rho[q] * J * f.vmb[q][i] + J * f.gp[i];
            }
            f.cont[q] = J * (f.beta[q] * f.pdq[q] + f.divv);
        }
    }
    __syncthreads();
}

// Residual kernel: lane = 4a + c, c < 3 -> R_m[a][c], c == 3 -> R_p[a].
template <int T, bool R64>
__global__ void __launch_bounds__(kTeam * T, (R64 ? 1024 : 512) / (kTeam * T)) k_residual(AsmArgs A, int c0, int count)
{
    extern __shared__ __align__(16) unsigned char frame_smem[];
    Frame* frames = reinterpret_cast<Frame*>(frame_smem);
    const int team = threadIdx.x / kTeam;
    const int lane = threadIdx.x % kTeam;
    Frame& f = frames[team];
    build_frames<T>(A, frames, c0, count, false);
    if (!f.valid) return;
    const int a = lane / 4, c = lane % 4;
    const double J = f.J;
    if (c < 3) {
        const int fi = f.free_idx[a];
        if (fi < 0) return;
        double* out = A.r_m + 3 * static_cast<int64_t>(fi) + c;
        double acc = *out;
        for (int q = 0; q < 4; ++q) {
            const double wq = 0.25 * f.vol;
            const double Na = bary(q, a);
            acc = acc + wq * Na * f.rho[q] * J * (f.vdq[q][c] - A.body_force[c]);
        }
        double PG = 0.0;
        for (int I = 0; I < 3; ++I) PG = PG + f.G[a][I] * f.Pt[3 * c + I];
        acc = acc + f.vol * (PG - f.g[a][c] * J * f.pbar);
        *out = acc;
    } else {
        double* out = A.r_p + f.nodes[a];
        double acc = *out;
        for (int q = 0; q < 4; ++q) {
            const double wq = 0.25 * f.vol;
            const double Na = bary(q, a);
            acc = acc + wq * (Na * f.cont[q] + f.tau * dot3(f.g[a], f.res[q]));
        }
        *out = acc;
    }
}

// Tangent kernel: dP for 12 directions, then lane = 4a + bn forms node block
// (a, bn) of eA, eB, eC, eD (+ eM, eK for the fold-in).
template <int T, bool R64>
__global__ void __launch_bounds__(kTeam * T, (R64 ? 1024 : 512) / (kTeam * T)) k_tangent(AsmArgs A, int c0, int count)
{
    extern __shared__ __align__(16) unsigned char frame_smem[];
    Frame* frames = reinterpret_cast<Frame*>(frame_smem);
    const int team = threadIdx.x / kTeam;
    const int lane = threadIdx.x % kTeam;
    const int idx = blockIdx.x * T + team;
    const bool active = idx < count;
    const int e = active ? A.elem_order[c0 + idx] : 0;
    Frame& f = frames[team];
    // this lane's K4 block (128 B) is read-modified-written at the very end:
    // start pulling its line into L1 now, behind the element's arithmetic
    const int kslot = active ? A.k4slot[16 * static_cast<int64_t>(e) + lane] : 0;
    if (active) asm volatile("prefetch.global.L1 [%0];" ::"l"(A.k4 + 16 * static_cast<int64_t>(kslot)));
    build_frames<T>(A, frames, c0, count, true);
    if (!f.valid) return;
    if (lane < 12) ptilde_dir(A.mat, f, lane / 3, lane % 3, f.dP[lane]);
    __syncwarp();

    const int a = lane / 4, bn = lane % 4;
    const double am = A.ts.alpha_m;
    const double chi = A.ts.alpha_f * A.ts.gamma * A.ts.dt;
    const double fac2 = chi * chi / am;
    const double J = f.J;
    const double tau = f.tau;
    double eA[3][3], eM[3], eB[3], eC[3], eK[3], eD = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        eM[i] = eB[i] = eC[i] = eK[i] = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) eA[i][j] = 0.0;
    }
    const double* ga = f.g[a];
    const double* gb = f.g[bn];
    for (int q = 0; q < 4; ++q) {
        const double wq = 0.25 * f.vol;
        const double Na = bary(q, a);
        const double Nb = bary(q, bn);
        const double rho = f.rho[q], beta = f.beta[q], drho = f.drho[q], dbeta = f.dbeta[q];
        const double* vmb = f.vmb[q];
        const double mass = wq * rho * J * Na * Nb;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            eM[i] = eM[i] + am * mass;
            eA[i][i] = eA[i][i] + am * mass;
#pragma unroll
            for (int j = 0; j < 3; ++j) eA[i][j] = eA[i][j] + fac2 * wq * Na * rho * J * vmb[i] * gb[j];
            eB[i] = eB[i] + chi * wq * (drho * J * vmb[i] * Na * Nb - J * ga[i] * Nb);
        }
        const double gab = dot3(ga, gb);
        const double gavmb = dot3(ga, vmb);
        const double gbres = dot3(gb, f.res[q]);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double crate = am * wq * tau * rho * J * ga[j] * Nb + chi * wq * J * Na * gb[j];
            eK[j] = eK[j] + crate;
            eC[j] = eC[j] + crate;
            double cu = Na * f.cont[q] * gb[j];
            double Lg = 0.0;
#pragma unroll
            for (int i = 0; i < 3; ++i) Lg = Lg + f.L[3 * i + j] * gb[i];
            cu = cu - J * Na * Lg;
            cu = cu - tau * ga[j] * gbres;
            cu = cu + tau * (rho * J * gavmb * gb[j] + J * dot3(ga, f.gp) * gb[j] - J * f.gp[j] * gab);
            eC[j] = eC[j] + fac2 * wq * cu;
        }
        eD = eD + wq * (am * J * beta * Na * Nb + chi * J * dbeta * f.pdq[q] * Na * Nb +
                        chi * tau * J * (gab + drho * gavmb * Nb));
    }
    // constant-integrand terms of A (assembly.cpp:297-313)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double* dP = f.dP[3 * bn + j];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int I = 0; I < 3; ++I) acc = acc + f.G[a][I] * dP[3 * i + I];
            acc = acc - J * f.pbar * (ga[i] * gb[j] - ga[j] * gb[i]);
            eA[i][j] = eA[i][j] + fac2 * f.vol * acc;
        }
    }
    // scatter into K4 (fixed rows/columns are dropped later by the plane maps)
    double* K = A.k4 + 16 * static_cast<int64_t>(kslot);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) K[4 * i + j] = K[4 * i + j] + eA[i][j];
        K[4 * i + 3] = K[4 * i + 3] + eB[i];
        K[12 + i] = K[12 + i] + eC[i];
    }
    K[15] = K[15] + eD;
    // fold-in: (eA - eM) rk_b and (eC - eK) rk_b, summed over b in order
    if (A.fv) {
        double fv[3], fp = 0.0;
        const double* rkb = f.rk[bn];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j) s = s + (i == j ? eA[i][j] - eM[i] : eA[i][j]) * rkb[j];
            fv[i] = s;
        }
#pragma unroll
        for (int j = 0; j < 3; ++j) fp = fp + (eC[j] - eK[j]) * rkb[j];
        // gather the 4 lanes of node a (lanes 4a..4a+3) in bn order
        const unsigned mask = 0xffffu << (threadIdx.x & 16);
        double tot[4] = {fv[0], fv[1], fv[2], fp};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int base = (threadIdx.x & ~3);
            const double v0 = __shfl_sync(mask, tot[k], base + 0);
            const double v1 = __shfl_sync(mask, tot[k], base + 1);
            const double v2 = __shfl_sync(mask, tot[k], base + 2);
            const double v3 = __shfl_sync(mask, tot[k], base + 3);
            tot[k] = ((v0 + v1) + v2) + v3;
        }
        if (bn == 0) {
            const int fi = f.free_idx[a];
            if (fi >= 0) {
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    double* o = A.fv + 3 * static_cast<int64_t>(fi) + i;
                    *o = *o + tot[i];
                }
            }
            double* o = A.fp + f.nodes[a];
            *o = *o + tot[3];
        }
    }
}

// Dead tractions (assembly.cpp:173-184): per free velocity row, subtract the
// facet contributions in the reference's loop order.
__global__ void k_traction(const int64_t* __restrict__ rowptr, const int* __restrict__ rows,
                           const double* __restrict__ vals, int nrows_with, double* r_m)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nrows_with) return;
    const int row = rows[t];
    double acc = r_m[row];
    for (int64_t k = rowptr[t]; k < rowptr[t + 1]; ++k) acc = acc - vals[k];
    r_m[row] = acc;
}

// K4 node blocks -> BSR planes (A 3x3, B 3x1, C 1x3, D 1x1); src = K4 block per stored block.
template <int PLANE>
__global__ void k_k4_to_plane(const int* __restrict__ src, const double* __restrict__ k4, double* val, int64_t nnzb)
{
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nnzb) return;
    const double* K = k4 + 16 * static_cast<int64_t>(src[k]);
    if (PLANE == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) val[k * 9 + 3 * i + j] = K[4 * i + j];
    } else if (PLANE == 1) {
#pragma unroll
        for (int i = 0; i < 3; ++i) val[k * 3 + i] = K[4 * i + 3];
    } else if (PLANE == 2) {
#pragma unroll
        for (int j = 0; j < 3; ++j) val[k * 3 + j] = K[12 + j];
    } else {
        val[k] = K[15];
    }
}

// All four planes from the K4 node blocks in ONE pass: a thread per node-graph
// slot reads its 128-B block once (8 x 16-B loads) and writes the A (3x3), B
// (3x1), C (1x3) and D (1x1) parts where they are stored (dst* = -1: the slot
// has no block in that plane -- a fixed row or column node).
__global__ void k_k4_split(const double* __restrict__ k4, const int* __restrict__ dstA, const int* __restrict__ dstB,
                           const int* __restrict__ dstC, const int* __restrict__ dstD, double* __restrict__ A,
                           double* __restrict__ B, double* __restrict__ C, double* __restrict__ D, int64_t nslots)
{
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nslots) return;
    const double2* src = reinterpret_cast<const double2*>(k4 + 16 * k);
    double K[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const double2 v = __ldg(src + q);
        K[2 * q] = v.x;
        K[2 * q + 1] = v.y;
    }
    const int a = dstA[k], b = dstB[k], c = dstC[k], d = dstD[k];
    if (a >= 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) A[9 * static_cast<int64_t>(a) + 3 * i + j] = K[4 * i + j];
    }
    if (b >= 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) B[3 * static_cast<int64_t>(b) + i] = K[4 * i + 3];
    }
    if (c >= 0) {
#pragma unroll
        for (int j = 0; j < 3; ++j) C[3 * static_cast<int64_t>(c) + j] = K[12 + j];
    }
    if (d >= 0) D[d] = K[15];
}

} // namespace

void launch_k4_split(const double* k4, const int* dstA, const int* dstB, const int* dstC, const int* dstD, double* A,
                     double* B, double* C, double* D, int64_t nslots, cudaStream_t s)
{
    if (nslots == 0) return;
    k_k4_split<<<static_cast<unsigned>((nslots + 255) / 256), 256, 0, s>>>(k4, dstA, dstB, dstC, dstD, A, B, C, D,
                                                                          nslots);
    after_launch("k_k4_split");
}

// Eight elements per 128-thread CTA (measured against 16 and 32 at 160^3,
// profiles/r02/assembly_experiments.md); the residual is compiled for 64 registers per thread (8 CTAs
// per SM), the tangent for 128 (4 CTAs per SM, no spills to speak of).
constexpr int kTeamsPerCta = 8;
constexpr int kCta = kTeam * kTeamsPerCta;
constexpr size_t kFrameBytes = sizeof(Frame) * kTeamsPerCta; // dynamic shared memory per CTA

template <typename K>
void launch_elements(K kernel, const char* name, const AsmArgs& A, const std::vector<int>& color_ptr, cudaStream_t s)
{
    static bool done[64] = {}; // per kernel instantiation and device
    int dev = 0;
    ED_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        ED_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kFrameBytes)));
        ED_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
        done[dev & 63] = true;
    }
    for (size_t c = 0; c + 1 < color_ptr.size(); ++c) {
        const int count = color_ptr[c + 1] - color_ptr[c];
        if (count == 0) continue;
        kernel<<<(count + kTeamsPerCta - 1) / kTeamsPerCta, kCta, kFrameBytes, s>>>(A, color_ptr[c], count);
        after_launch(name);
    }
}

void launch_residual(const AsmArgs& A, const std::vector<int>& color_ptr, cudaStream_t s)
{
    launch_elements(k_residual<kTeamsPerCta, true>, "k_residual", A, color_ptr, s);
}

void launch_tangent(const AsmArgs& A, const std::vector<int>& color_ptr, cudaStream_t s)
{
    launch_elements(k_tangent<kTeamsPerCta, false>, "k_tangent", A, color_ptr, s);
}

void launch_traction(const int64_t* rowptr, const int* rows, const double* vals, int nrows_with, double* r_m,
                     cudaStream_t s)
{
    if (nrows_with == 0) return;
    k_traction<<<(nrows_with + 255) / 256, 256, 0, s>>>(rowptr, rows, vals, nrows_with, r_m);
    after_launch("k_traction");
}

void launch_k4_to_plane(int plane, const int* src, const double* k4, double* val, int64_t nnzb, cudaStream_t s)
{
    if (nnzb == 0) return;
    const int g = static_cast<int>((nnzb + 255) / 256);
    switch (plane) {
    case 0: k_k4_to_plane<0><<<g, 256, 0, s>>>(src, k4, val, nnzb); break;
    case 1: k_k4_to_plane<1><<<g, 256, 0, s>>>(src, k4, val, nnzb); break;
    case 2: k_k4_to_plane<2><<<g, 256, 0, s>>>(src, k4, val, nnzb); break;
    default: k_k4_to_plane<3><<<g, 256, 0, s>>>(src, k4, val, nnzb); break;
    }
    after_launch("k_k4_to_plane");
}

} // namespace edb

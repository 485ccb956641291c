// Host smoothed-aggregation setup; see amg_host.hpp.  Each function cites
// the reference routine whose arithmetic it restates.
#include "amg_host.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace edb {

// ---------------------------------------------------------------------------
// CSR primitives (csr.cpp)

std::vector<double> csr_diag(const HostCsr& a) // CsrMatrix::diag, csr.cpp:29-37
{
    std::vector<double> d(a.nrows, 0.0);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < a.nrows; ++r) {
        const auto b = a.col.begin() + a.rowptr[r], e = a.col.begin() + a.rowptr[r + 1];
        const auto it = std::lower_bound(b, e, r);
        if (it != e && *it == r) d[r] = a.val[it - a.col.begin()];
    }
    return d;
}

// csr_matmul, csr.cpp:132-166: marker + dense accumulator per row; each output
// entry sums a.val*b.val in (a-column, b-column) traversal order.
HostCsr csr_matmul(const HostCsr& a, const HostCsr& b)
{
    if (a.ncols != b.nrows) throw Error(ED_INVALID_ARGUMENT, "csr_matmul: shape mismatch");
    HostCsr c;
    c.nrows = a.nrows;
    c.ncols = b.ncols;
    c.rowptr.assign(a.nrows + 1, 0);
    // symbolic
#pragma omp parallel
    {
        std::vector<int> marker(b.ncols, -1);
#pragma omp for schedule(dynamic, 1024)
        for (int r = 0; r < a.nrows; ++r) {
            int64_t cnt = 0;
            for (int64_t ka = a.rowptr[r]; ka < a.rowptr[r + 1]; ++ka) {
                const int k = a.col[ka];
                for (int64_t kb = b.rowptr[k]; kb < b.rowptr[k + 1]; ++kb) {
                    const int j = b.col[kb];
                    if (marker[j] != r) {
                        marker[j] = r;
                        ++cnt;
                    }
                }
            }
            c.rowptr[r + 1] = cnt;
        }
    }
    for (int r = 0; r < a.nrows; ++r) c.rowptr[r + 1] += c.rowptr[r];
    c.col.resize(c.rowptr[a.nrows]);
    c.val.resize(c.rowptr[a.nrows]);
#pragma omp parallel
    {
        std::vector<int> marker(b.ncols, -1);
        std::vector<double> acc(b.ncols, 0.0);
        std::vector<int> row_cols;
#pragma omp for schedule(dynamic, 1024)
        for (int r = 0; r < a.nrows; ++r) {
            row_cols.clear();
            for (int64_t ka = a.rowptr[r]; ka < a.rowptr[r + 1]; ++ka) {
                const int k = a.col[ka];
                const double av = a.val[ka];
                for (int64_t kb = b.rowptr[k]; kb < b.rowptr[k + 1]; ++kb) {
                    const int j = b.col[kb];
                    if (marker[j] != r) {
                        marker[j] = r;
                        acc[j] = 0.0;
                        row_cols.push_back(j);
                    }
                    acc[j] += av * b.val[kb];
                }
            }
            std::sort(row_cols.begin(), row_cols.end());
            int64_t out = c.rowptr[r];
            for (const int j : row_cols) {
                c.col[out] = j;
                c.val[out] = acc[j];
                ++out;
            }
        }
    }
    return c;
}

// CsrMatrix::transpose, csr.cpp:39-57 (rows come out sorted)
HostCsr csr_transpose(const HostCsr& a)
{
    HostCsr t;
    t.nrows = a.ncols;
    t.ncols = a.nrows;
    t.rowptr.assign(a.ncols + 1, 0);
    for (const int c : a.col) ++t.rowptr[c + 1];
    for (int r = 0; r < t.nrows; ++r) t.rowptr[r + 1] += t.rowptr[r];
    t.col.resize(a.col.size());
    t.val.resize(a.val.size());
    std::vector<int64_t> next(t.rowptr.begin(), t.rowptr.end() - 1);
    for (int r = 0; r < a.nrows; ++r)
        for (int64_t k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
            const int64_t pos = next[a.col[k]]++;
            t.col[pos] = r;
            t.val[pos] = a.val[k];
        }
    return t;
}

// csr_add, csr.cpp:168-198
HostCsr csr_add(const HostCsr& a, const HostCsr& b, double alpha, double beta)
{
    if (a.nrows != b.nrows || a.ncols != b.ncols) throw Error(ED_INVALID_ARGUMENT, "csr_add: shape mismatch");
    HostCsr c;
    c.nrows = a.nrows;
    c.ncols = a.ncols;
    c.rowptr.assign(a.nrows + 1, 0);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < a.nrows; ++r) {
        int64_t ka = a.rowptr[r], kb = b.rowptr[r], cnt = 0;
        const int64_t ea = a.rowptr[r + 1], eb = b.rowptr[r + 1];
        while (ka < ea || kb < eb) {
            if (kb >= eb || (ka < ea && a.col[ka] < b.col[kb]))
                ++ka;
            else if (ka >= ea || b.col[kb] < a.col[ka])
                ++kb;
            else {
                ++ka;
                ++kb;
            }
            ++cnt;
        }
        c.rowptr[r + 1] = cnt;
    }
    for (int r = 0; r < a.nrows; ++r) c.rowptr[r + 1] += c.rowptr[r];
    c.col.resize(c.rowptr[a.nrows]);
    c.val.resize(c.rowptr[a.nrows]);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < a.nrows; ++r) {
        int64_t ka = a.rowptr[r], kb = b.rowptr[r], out = c.rowptr[r];
        const int64_t ea = a.rowptr[r + 1], eb = b.rowptr[r + 1];
        while (ka < ea || kb < eb) {
            int j;
            double v;
            if (kb >= eb || (ka < ea && a.col[ka] < b.col[kb])) {
                j = a.col[ka];
                v = alpha * a.val[ka++];
            } else if (ka >= ea || b.col[kb] < a.col[ka]) {
                j = b.col[kb];
                v = beta * b.val[kb++];
            } else {
                j = a.col[ka];
                v = alpha * a.val[ka++] + beta * b.val[kb++];
            }
            c.col[out] = j;
            c.val[out] = v;
            ++out;
        }
    }
    return c;
}

namespace {

void matvec(const HostCsr& a, const double* x, double* y) // csr.cpp:11-18
{
#pragma omp parallel for schedule(static)
    for (int r = 0; r < a.nrows; ++r) {
        double s = 0.0;
        for (int64_t k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) s += a.val[k] * x[a.col[k]];
        y[r] = s;
    }
}

double seq_norm(const std::vector<double>& v) // vec_norm, csr.cpp:213-221 (sequential order)
{
    double s = 0.0;
    for (const double x : v) s += x * x;
    return std::sqrt(s);
}

// strong_neighbors, amg.cpp:32-81
std::vector<std::vector<int>> strong_neighbors(const HostCsr& A, const std::vector<int>& node_of_row, int n_nodes,
                                               double theta)
{
    std::vector<int> nstart(n_nodes + 1, 0);
    for (int r = 0; r < A.nrows; ++r) ++nstart[node_of_row[r] + 1];
    for (int I = 0; I < n_nodes; ++I) nstart[I + 1] += nstart[I];
    std::vector<double> diag_w(n_nodes, 0.0);
#pragma omp parallel for schedule(static)
    for (int I = 0; I < n_nodes; ++I)
        for (int r = nstart[I]; r < nstart[I + 1]; ++r)
            for (int64_t k = A.rowptr[r]; k < A.rowptr[r + 1]; ++k)
                if (node_of_row[A.col[k]] == I) diag_w[I] += A.val[k] * A.val[k];
    std::vector<std::vector<int>> nbr(n_nodes);
#pragma omp parallel
    {
        std::vector<int> touched;
        std::vector<double> acc(n_nodes, 0.0);
        std::vector<char> seen(n_nodes, 0);
#pragma omp for schedule(dynamic, 512)
        for (int I = 0; I < n_nodes; ++I) {
            touched.clear();
            for (int r = nstart[I]; r < nstart[I + 1]; ++r)
                for (int64_t k = A.rowptr[r]; k < A.rowptr[r + 1]; ++k) {
                    const int J = node_of_row[A.col[k]];
                    if (J == I) continue;
                    if (!seen[J]) {
                        seen[J] = 1;
                        touched.push_back(J);
                    }
                    acc[J] += A.val[k] * A.val[k];
                }
            for (const int J : touched) {
                const double s2 = acc[J];
                acc[J] = 0.0;
                seen[J] = 0;
                if (diag_w[I] <= 0.0 || diag_w[J] <= 0.0) continue;
                // diag_w holds squared Frobenius norms, hence the quarter power
                if (std::sqrt(s2) > theta * std::pow(diag_w[I] * diag_w[J], 0.25)) nbr[I].push_back(J);
            }
        }
    }
    std::vector<int> deg(n_nodes, 0);
    for (int I = 0; I < n_nodes; ++I)
        for (const int J : nbr[I]) {
            ++deg[I];
            ++deg[J];
        }
    std::vector<std::vector<int>> sym(n_nodes);
    for (int I = 0; I < n_nodes; ++I) sym[I].reserve(deg[I]);
    for (int I = 0; I < n_nodes; ++I)
        for (const int J : nbr[I]) {
            sym[I].push_back(J);
            sym[J].push_back(I);
        }
#pragma omp parallel for schedule(dynamic, 512)
    for (int I = 0; I < n_nodes; ++I) {
        auto& l = sym[I];
        std::sort(l.begin(), l.end());
        l.erase(std::unique(l.begin(), l.end()), l.end());
    }
    return sym;
}

// aggregate, amg.cpp:85-117 (greedy, order dependent: sequential)
int aggregate(const std::vector<std::vector<int>>& nbr, std::vector<int>& agg_of)
{
    const int n = static_cast<int>(nbr.size());
    agg_of.assign(n, -1);
    int n_agg = 0;
    for (int i = 0; i < n; ++i) {
        if (agg_of[i] >= 0 || nbr[i].empty()) continue;
        bool clean = true;
        for (const int j : nbr[i])
            if (agg_of[j] >= 0) {
                clean = false;
                break;
            }
        if (!clean) continue;
        agg_of[i] = n_agg;
        for (const int j : nbr[i]) agg_of[j] = n_agg;
        ++n_agg;
    }
    for (int i = 0; i < n; ++i) {
        if (agg_of[i] >= 0) continue;
        for (const int j : nbr[i])
            if (agg_of[j] >= 0) {
                agg_of[i] = agg_of[j];
                break;
            }
    }
    for (int i = 0; i < n; ++i)
        if (agg_of[i] < 0) agg_of[i] = n_agg++;
    return n_agg;
}

// tentative_prolongator, amg.cpp:122-168
HostCsr tentative_prolongator(int nrows, int k, const std::vector<int>& agg_of_row, int n_agg,
                              const std::vector<double>& B, std::vector<double>& Bc)
{
    std::vector<int> astart(n_agg + 1, 0);
    for (int r = 0; r < nrows; ++r) ++astart[agg_of_row[r] + 1];
    for (int a = 0; a < n_agg; ++a) astart[a + 1] += astart[a];
    std::vector<int> rows_flat(nrows);
    {
        std::vector<int> next(astart.begin(), astart.end() - 1);
        for (int r = 0; r < nrows; ++r) rows_flat[next[agg_of_row[r]]++] = r;
    }
    Bc.assign(static_cast<size_t>(n_agg) * k * k, 0.0);
    std::vector<double> Qrow(static_cast<size_t>(nrows) * k, 0.0); // Q value of (row, c)
#pragma omp parallel
    {
        std::vector<double> Q;
#pragma omp for schedule(dynamic, 256)
        for (int a = 0; a < n_agg; ++a) {
            const int* rows = rows_flat.data() + astart[a];
            const int nr = astart[a + 1] - astart[a];
            Q.assign(static_cast<size_t>(nr) * k, 0.0);
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < nr; ++r) Q[c * nr + r] = B[static_cast<size_t>(rows[r]) * k + c];
            for (int c = 0; c < k; ++c) {
                for (int c2 = 0; c2 < c; ++c2) {
                    double d = 0.0;
                    for (int r = 0; r < nr; ++r) d += Q[c2 * nr + r] * Q[c * nr + r];
                    Bc[(static_cast<size_t>(a) * k + c2) * k + c] = d;
                    for (int r = 0; r < nr; ++r) Q[c * nr + r] -= d * Q[c2 * nr + r];
                }
                double nrm = 0.0;
                for (int r = 0; r < nr; ++r) nrm += Q[c * nr + r] * Q[c * nr + r];
                nrm = std::sqrt(nrm);
                Bc[(static_cast<size_t>(a) * k + c) * k + c] = nrm;
                if (nrm > 1e-14) {
                    for (int r = 0; r < nr; ++r) Q[c * nr + r] /= nrm;
                } else {
                    for (int r = 0; r < nr; ++r) Q[c * nr + r] = 0.0;
                }
            }
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < nr; ++r) Qrow[static_cast<size_t>(rows[r]) * k + c] = Q[c * nr + r];
        }
    }
    // from_triplets (csr.cpp:77-110): one aggregate per row, columns a*k+c ascending
    HostCsr P;
    P.nrows = nrows;
    P.ncols = n_agg * k;
    P.rowptr.assign(nrows + 1, 0);
    for (int r = 0; r < nrows; ++r) {
        int64_t cnt = 0;
        for (int c = 0; c < k; ++c) cnt += Qrow[static_cast<size_t>(r) * k + c] != 0.0;
        P.rowptr[r + 1] = P.rowptr[r] + cnt;
    }
    P.col.resize(P.rowptr[nrows]);
    P.val.resize(P.rowptr[nrows]);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < nrows; ++r) {
        int64_t out = P.rowptr[r];
        for (int c = 0; c < k; ++c) {
            const double q = Qrow[static_cast<size_t>(r) * k + c];
            if (q != 0.0) {
                P.col[out] = agg_of_row[r] * k + c;
                P.val[out] = q;
                ++out;
            }
        }
    }
    return P;
}

// estimate_spectral_radius, amg.cpp:170-185
double estimate_spectral_radius(const HostCsr& A, const std::vector<double>& inv_diag)
{
    const int n = A.nrows;
    std::vector<double> v(n, 1.0), w(n);
    double lambda = 1.0;
    for (int it = 0; it < 10; ++it) {
        matvec(A, v.data(), w.data());
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) w[i] *= inv_diag[i];
        const double nrm = seq_norm(w);
        if (nrm == 0.0) return 1.0;
        lambda = nrm / seq_norm(v);
        const double inv = 1.0 / nrm;
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) v[i] = w[i] * inv;
    }
    return lambda;
}

std::vector<double> inverted_diag(const HostCsr& A)
{
    std::vector<double> d = csr_diag(A);
    for (auto& x : d) x = (x != 0.0) ? 1.0 / x : 1.0;
    return d;
}

// ---- COD (Householder QR with column pivoting + RZ), Eigen's algorithm ----
struct Cod {
    int m = 0, n = 0, rank = 0;
    std::vector<double> qr; // col-major m x n
    std::vector<double> hc, zc;
    std::vector<int> perm;
    double& at(int i, int j) { return qr[static_cast<size_t>(j) * m + i]; }

    template <class Get>
    static void householder(Get x, int len, double& tau, double& beta)
    {
        double tail = 0.0;
        for (int i = 1; i < len; ++i) tail += x(i) * x(i);
        const double c0 = x(0);
        if (tail <= std::numeric_limits<double>::min()) {
            tau = 0.0;
            beta = c0;
            for (int i = 1; i < len; ++i) x(i) = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            const double d = c0 - beta;
            for (int i = 1; i < len; ++i) x(i) = x(i) / d;
            tau = (beta - c0) / beta;
        }
    }

    void compute(const std::vector<double>& a, int mm, int nn, double thr)
    {
        m = mm;
        n = nn;
        qr = a;
        const int size = std::min(m, n);
        hc.assign(size, 0.0);
        perm.resize(n);
        std::iota(perm.begin(), perm.end(), 0);
        std::vector<double> upd(n), dir(n);
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int i = 0; i < m; ++i) s += at(i, j) * at(i, j);
            upd[j] = dir[j] = std::sqrt(s);
        }
        const double downdate = std::sqrt(std::numeric_limits<double>::epsilon());
        double maxpivot = 0.0;
        for (int k = 0; k < size; ++k) {
            int big = k;
            for (int j = k + 1; j < n; ++j)
                if (upd[j] > upd[big]) big = j;
            if (big != k) {
                for (int i = 0; i < m; ++i) std::swap(at(i, k), at(i, big));
                std::swap(upd[k], upd[big]);
                std::swap(dir[k], dir[big]);
                std::swap(perm[k], perm[big]);
            }
            double tau, beta;
            householder([&](int i) -> double& { return at(k + i, k); }, m - k, tau, beta);
            at(k, k) = beta;
            hc[k] = tau;
            maxpivot = std::max(maxpivot, std::abs(beta));
            for (int j = k + 1; j < n; ++j) {
                double t = at(k, j);
                for (int i = k + 1; i < m; ++i) t += at(i, k) * at(i, j);
                if (tau != 0.0) {
                    at(k, j) -= tau * t;
                    for (int i = k + 1; i < m; ++i) at(i, j) -= tau * at(i, k) * t;
                }
            }
            for (int j = k + 1; j < n; ++j) {
                if (upd[j] == 0.0) continue;
                double temp = std::abs(at(k, j)) / upd[j];
                temp = (1.0 + temp) * (1.0 - temp);
                temp = temp < 0.0 ? 0.0 : temp;
                const double r = upd[j] / dir[j];
                if (temp * r * r <= downdate) {
                    double s = 0.0;
                    for (int i = k + 1; i < m; ++i) s += at(i, j) * at(i, j);
                    dir[j] = upd[j] = std::sqrt(s);
                } else {
                    upd[j] *= std::sqrt(temp);
                }
            }
        }
        rank = 0;
        for (int i = 0; i < size; ++i)
            if (std::abs(at(i, i)) > maxpivot * thr) ++rank;
        zc.assign(rank, 0.0);
        if (rank < n) {
            const int r = rank;
            const int len = n - r + 1;
            for (int k = r - 1; k >= 0; --k) {
                if (k != r - 1)
                    for (int i = 0; i <= k; ++i) std::swap(at(i, k), at(i, r - 1));
                double tau, beta;
                householder([&](int i) -> double& { return at(k, r - 1 + i); }, len, tau, beta);
                at(k, r - 1) = beta;
                zc[k] = tau;
                if (k > 0 && tau != 0.0)
                    for (int i = 0; i < k; ++i) {
                        double s = at(i, r - 1);
                        for (int j = 1; j < len; ++j) s += at(i, r - 1 + j) * at(k, r - 1 + j);
                        at(i, r - 1) -= tau * s;
                        for (int j = 1; j < len; ++j) at(i, r - 1 + j) -= tau * s * at(k, r - 1 + j);
                    }
                if (k != r - 1)
                    for (int i = 0; i <= k; ++i) std::swap(at(i, k), at(i, r - 1));
            }
        }
    }

    std::vector<double> solve(const std::vector<double>& b)
    {
        std::vector<double> x(n, 0.0);
        const int r = rank;
        if (r == 0) return x;
        std::vector<double> c(b);
        for (int k = 0; k < r; ++k) {
            const double tau = hc[k];
            if (tau == 0.0) continue;
            double t = c[k];
            for (int i = k + 1; i < m; ++i) t += at(i, k) * c[i];
            c[k] -= tau * t;
            for (int i = k + 1; i < m; ++i) c[i] -= tau * at(i, k) * t;
        }
        std::vector<double> y(n, 0.0);
        for (int i = r - 1; i >= 0; --i) {
            double s = c[i];
            for (int j = i + 1; j < r; ++j) s -= at(i, j) * y[j];
            y[i] = s / at(i, i);
        }
        if (r < n)
            for (int k = 0; k < r; ++k) {
                const double tau = zc[k];
                if (tau == 0.0) continue;
                if (k != r - 1) std::swap(y[k], y[r - 1]);
                double s = y[r - 1];
                for (int j = r; j < n; ++j) s += at(k, j) * y[j];
                y[r - 1] -= tau * s;
                for (int j = r; j < n; ++j) y[j] -= tau * at(k, j) * s;
                if (k != r - 1) std::swap(y[k], y[r - 1]);
            }
        for (int j = 0; j < n; ++j) x[perm[j]] = y[j];
        return x;
    }
};

} // namespace

int amg_aggregate(const std::vector<int64_t>& nbr_ptr, const std::vector<int>& nbr, std::vector<int>& agg_of)
{
    // aggregate() of amg.cpp:85-117 on a CSR neighbour list
    const int n = static_cast<int>(nbr_ptr.size()) - 1;
    agg_of.assign(n, -1);
    int n_agg = 0;
    for (int i = 0; i < n; ++i) {
        if (agg_of[i] >= 0 || nbr_ptr[i] == nbr_ptr[i + 1]) continue;
        bool clean = true;
        for (int64_t k = nbr_ptr[i]; k < nbr_ptr[i + 1]; ++k)
            if (agg_of[nbr[k]] >= 0) {
                clean = false;
                break;
            }
        if (!clean) continue;
        agg_of[i] = n_agg;
        for (int64_t k = nbr_ptr[i]; k < nbr_ptr[i + 1]; ++k) agg_of[nbr[k]] = n_agg;
        ++n_agg;
    }
    for (int i = 0; i < n; ++i) {
        if (agg_of[i] >= 0) continue;
        for (int64_t k = nbr_ptr[i]; k < nbr_ptr[i + 1]; ++k)
            if (agg_of[nbr[k]] >= 0) {
                agg_of[i] = agg_of[nbr[k]];
                break;
            }
    }
    for (int i = 0; i < n; ++i)
        if (agg_of[i] < 0) agg_of[i] = n_agg++;
    return n_agg;
}

HostCsr amg_tentative(int nrows, int k, const std::vector<int>& agg_of_row, int n_agg, const std::vector<double>& B,
                      std::vector<double>& Bc)
{
    return tentative_prolongator(nrows, k, agg_of_row, n_agg, B, Bc);
}

double amg_seq_norm(const std::vector<double>& v) { return seq_norm(v); }

void check_coarse_size(int nrows, int n_coarsened)
{
    // The reference factors the coarsest level densely whatever its size
    // (amg.cpp:278-294).  When coarsening stalls before coarse_max_rows the
    // loop stops at max_levels with a huge coarsest level; a dense COD of it
    // cannot be formed (the reference would die in the same place), so say so.
    if (nrows <= kMaxCoarseDenseRows) return;
    char msg[256];
    std::snprintf(msg, sizeof msg,
                  "amg: coarsest level has %d rows after %d coarsening steps (coarsening stalled); its dense "
                  "COD (amg.cpp:286-294) would need %.1f GB",
                  nrows, n_coarsened, 8.0 * double(nrows) * double(nrows) / 1e9);
    throw Error(ED_UNSUPPORTED, msg);
}

std::vector<double> cod_pinv(const std::vector<double>& dense_colmajor, int n, double threshold)
{
    Cod cod;
    cod.compute(dense_colmajor, n, n, threshold);
    std::vector<double> P(static_cast<size_t>(n) * n, 0.0);
    std::vector<double> e(n, 0.0);
    for (int i = 0; i < n; ++i) {
        std::fill(e.begin(), e.end(), 0.0);
        e[i] = 1.0;
        const std::vector<double> x = cod.solve(e);
        for (int r = 0; r < n; ++r) P[static_cast<size_t>(r) * n + i] = x[r];
    }
    return P;
}

// AmgHierarchy::build, amg.cpp:189-295
namespace {
struct StageTimer {
    bool on = std::getenv("ED_AMG_VERBOSE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void lap(const char* what, int level, long rows, long nnz)
    {
        const auto now = std::chrono::steady_clock::now();
        if (on)
            std::fprintf(stderr, "[amg] L%d %-12s %9.3f s  rows %ld nnz %ld\n", level, what,
                         std::chrono::duration<double>(now - t).count(), rows, nnz);
        t = now;
    }
};
} // namespace

HostHierarchy amg_build_host(const HostCsr& A0, const AmgOpts& opts)
{
    StageTimer T;
    if (A0.nrows != A0.ncols) throw Error(ED_INVALID_ARGUMENT, "amg: matrix must be square");
    const int k = opts.block_size;
    if (k < 1) throw Error(ED_INVALID_ARGUMENT, "amg: block size must be positive");
    HostHierarchy h;
    std::vector<int> node_of_row, comp_of_row;
    if (!opts.row_to_node.empty()) {
        if (static_cast<int>(opts.row_to_node.size()) != A0.nrows ||
            static_cast<int>(opts.row_component.size()) != A0.nrows)
            throw Error(ED_INVALID_ARGUMENT, "amg: row grouping arrays must match matrix size");
        node_of_row = opts.row_to_node;
        comp_of_row = opts.row_component;
    } else {
        if (A0.nrows % k != 0) throw Error(ED_INVALID_ARGUMENT, "amg: rows not divisible by block size");
        node_of_row.resize(A0.nrows);
        comp_of_row.resize(A0.nrows);
        for (int r = 0; r < A0.nrows; ++r) {
            node_of_row[r] = r / k;
            comp_of_row[r] = r % k;
        }
    }
    std::vector<double> B(static_cast<size_t>(A0.nrows) * k, 0.0);
    for (int r = 0; r < A0.nrows; ++r) B[static_cast<size_t>(r) * k + comp_of_row[r]] = 1.0;

    HostCsr A = A0;
    while (A.nrows > opts.coarse_max_rows && static_cast<int>(h.levels.size()) + 1 < opts.max_levels) {
        const int n_nodes = node_of_row.empty() ? 0 : node_of_row.back() + 1;
        const int lvl = static_cast<int>(h.levels.size());
        T.lap("start", lvl, A.nrows, A.nnz());
        const auto nbr = strong_neighbors(A, node_of_row, n_nodes, opts.strength_theta);
        T.lap("strength", lvl, A.nrows, A.nnz());
        std::vector<int> agg_of_node;
        const int n_agg = aggregate(nbr, agg_of_node);
        T.lap("aggregate", lvl, n_agg, 0);
        if (n_agg <= 0 || n_agg >= n_nodes) {
            if (h.levels.empty()) {
                h.fallback = true;
                h.fallback_inv_diag = inverted_diag(A0);
                return h;
            }
            break;
        }
        std::vector<int> agg_of_row(A.nrows);
        for (int r = 0; r < A.nrows; ++r) agg_of_row[r] = agg_of_node[node_of_row[r]];
        std::vector<double> Bc;
        HostCsr P = tentative_prolongator(A.nrows, k, agg_of_row, n_agg, B, Bc);
        T.lap("tentative", lvl, P.nrows, P.nnz());
        HostLevel lv;
        lv.inv_diag = inverted_diag(A);
        if (opts.smooth_prolongator) {
            const double lambda = estimate_spectral_radius(A, lv.inv_diag);
            T.lap("spectral", lvl, A.nrows, 0);
            const double omega = 4.0 / (3.0 * std::max(lambda, 1e-12));
            HostCsr AP = csr_matmul(A, P);
            T.lap("AP_tent", lvl, AP.nrows, AP.nnz());
#pragma omp parallel for schedule(static)
            for (int r = 0; r < AP.nrows; ++r)
                for (int64_t kk = AP.rowptr[r]; kk < AP.rowptr[r + 1]; ++kk) AP.val[kk] *= lv.inv_diag[r];
            P = csr_add(P, AP, 1.0, -omega);
            T.lap("smooth_P", lvl, P.nrows, P.nnz());
        }
        HostCsr R = csr_transpose(P);
        T.lap("transpose", lvl, R.nrows, R.nnz());
        HostCsr AP2 = csr_matmul(A, P);
        T.lap("AP", lvl, AP2.nrows, AP2.nnz());
        HostCsr Ac = csr_matmul(R, AP2);
        T.lap("RAP", lvl, Ac.nrows, Ac.nnz());
        lv.A = std::move(A);
        lv.P = std::move(P);
        lv.R = std::move(R);
        h.levels.push_back(std::move(lv));
        A = std::move(Ac);
        B = std::move(Bc);
        node_of_row.resize(A.nrows);
        comp_of_row.resize(A.nrows);
        for (int r = 0; r < A.nrows; ++r) {
            node_of_row[r] = r / k;
            comp_of_row[r] = r % k;
        }
    }
    {
        HostLevel lv;
        lv.A = std::move(A);
        lv.inv_diag = inverted_diag(lv.A);
        h.levels.push_back(std::move(lv));
    }
    const HostCsr& Ac = h.levels.back().A;
    check_coarse_size(Ac.nrows, static_cast<int>(h.levels.size()) - 1);
    h.nc = Ac.nrows;
    std::vector<double> dense(static_cast<size_t>(Ac.nrows) * Ac.ncols, 0.0);
    for (int r = 0; r < Ac.nrows; ++r)
        for (int64_t kk = Ac.rowptr[r]; kk < Ac.rowptr[r + 1]; ++kk)
            dense[static_cast<size_t>(Ac.col[kk]) * Ac.nrows + r] = Ac.val[kk];
    h.pinv = cod_pinv(dense, Ac.nrows, 1e-12);
    T.lap("coarse_cod", static_cast<int>(h.levels.size()) - 1, Ac.nrows, Ac.nnz());
    return h;
}

} // namespace edb

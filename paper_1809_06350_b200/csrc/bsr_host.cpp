// Host construction of level-ordered BSR operators, Gauss-Seidel level
// schedules and dataflow work items.  Structure is
// mesh-static: built once per mesh (or per AMG level); only values move per
// Newton step.
#include <algorithm>
#include <cstdlib>
#include <numeric>

#include "ed_internal.hpp"

namespace edb {

double Bsr::bytes_per_spmv() const
{
    const BsrStruct& S = *st;
    const double blk = 8.0 * S.Rb * S.Cb + 4.0;
    return static_cast<double>(S.nnzb) * blk + 4.0 * (S.nbr + 1) + 8.0 * S.nbr * S.Rb + 8.0 * S.nbc * S.Cb;
}

void gs_level_order(const BlockPattern& pat, std::vector<int>& order, std::vector<int>& level_of_pos, int& nlev)
{
    const int n = pat.nbr;
    std::vector<int> level(n, 0);
    nlev = n > 0 ? 1 : 0;
    // Row i reads the NEW value of every j < i it couples to (amg.cpp:311-316),
    // so it sits one level above the highest such j.
    for (int i = 0; i < n; ++i) {
        int lv = 0;
        for (int64_t k = pat.rowptr[i]; k < pat.rowptr[i + 1]; ++k) {
            const int j = pat.col[k];
            if (j < i) lv = std::max(lv, level[j] + 1);
        }
        level[i] = lv;
        nlev = std::max(nlev, lv + 1);
    }
    std::vector<int> cnt(nlev + 1, 0);
    for (int i = 0; i < n; ++i) ++cnt[level[i] + 1];
    for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
    order.assign(n, 0);
    level_of_pos.assign(n, 0);
    for (int i = 0; i < n; ++i) {
        const int pos = cnt[level[i]]++;
        order[pos] = i;
        level_of_pos[pos] = level[i];
    }
}

namespace {
constexpr int kRingSliceMaxBytes = 40 * 1024; // z slice per CTA (b and inv_diag slices alongside)
constexpr int kRingPartMaxBytes = 24 * 1024;  // one partial-sum slot per CTA
constexpr int kRingMinRows = 4096;            // smaller operators: group / chain sweeps, dense tail

int64_t push_chunk_bytes(int64_t m, int64_t pk0, int64_t pk1, int64_t s0, int64_t nown, int B)
{
    const int64_t BB = B * B;
    const int64_t cb = 4 * (((pk1 + 3) & ~int64_t(3)) - (pk0 & ~int64_t(3)));
    const int64_t vb = 8 * BB * (((pk1 + 1) & ~int64_t(1)) - (pk0 & ~int64_t(1)));
    const int64_t db = 8 * BB * (((s0 + nown + 1) & ~int64_t(1)) - (s0 & ~int64_t(1)));
    return 16 * m + cb + vb + db;
}

// Rows of level l are dealt round-robin starting at CTA l % cs (row q -> CTA
// (q + l) % cs) and stored CTA-major; rows CTA c gets at level l:
inline int dealt(int m, int c, int l, int cs)
{
    const int first = ((c - l) % cs + cs) % cs; // smallest q with (q + l) % cs == c
    return first < m ? (m - 1 - first) / cs + 1 : 0;
}
constexpr int kRingSlots = 4; // partial-sum slots (kernels_ring.cu)
constexpr int kRingScratchMaxBytes = 32 * 1024; // push_scratch_bytes limit

// Forced cluster barriers of the push sweep: slot (i mod K) of a CTA is
// reused every K levels, so a CTA may push level-i partials only once every
// peer finished level i-K.  A CTA that waited for its own rows' partials at
// level k knows every peer finished k-1; where some CTA went K-1 levels
// without owning a row, a cluster barrier before the level resets all.
// bit 0: forward sweep, bit 1: backward sweep (sequence order reversed).
std::vector<int> push_barriers(const std::vector<int>& lev_ptr, int cs)
{
    const int L = static_cast<int>(lev_ptr.size()) - 1;
    std::vector<int> flags(L, 0);
    for (int dir = 0; dir < 2; ++dir) {
        std::vector<int> last(cs, 0); // the kernel-start cluster barrier
        for (int i = 0; i < L; ++i) {
            const int l = dir == 0 ? i : L - 1 - i;
            const int m = lev_ptr[l + 1] - lev_ptr[l];
            bool need = false;
            for (int c = 0; c < cs; ++c) need = need || i - last[c] > kRingSlots - 1;
            if (need) {
                flags[l] |= 1 << dir;
                std::fill(last.begin(), last.end(), i);
            }
            for (int c = 0; c < cs; ++c)
                if (dealt(m, c, l, cs) > 0) last[c] = i;
        }
    }
    return flags;
}
} // namespace

int ring_order(const BlockPattern& pat, int B, std::vector<int>& order, const std::vector<int>& level_of_pos, int nlev)
{
    static const bool off = std::getenv("ED_NO_RING") != nullptr;
    const int n = pat.nbr;
    if (off || (B != 1 && B != 3) || nlev < 2 || n < kRingMinRows || pat.nbr != pat.nbc) return 0;
    const int cs = ring_cluster_size();
    if (cs == 0) return 0;
    std::vector<int> lev_ptr{0};
    for (int p = 1; p < n; ++p)
        if (level_of_pos[p] != level_of_pos[p - 1]) lev_ptr.push_back(p);
    lev_ptr.push_back(n);
    const int L = static_cast<int>(lev_ptr.size()) - 1;
    std::vector<int64_t> slice(cs, 0);
    int mown = 0;
    for (int l = 0; l < L; ++l) {
        const int m = lev_ptr[l + 1] - lev_ptr[l];
        for (int c = 0; c < cs; ++c) slice[c] += dealt(m, c, l, cs);
        mown = std::max(mown, (m + cs - 1) / cs);
    }
    const int64_t smax = *std::max_element(slice.begin(), slice.end());
    const int PB = B == 3 ? 4 : 1;
    const int part = mown * cs * PB * 8;
    if (smax * B * 8 > kRingSliceMaxBytes || part > kRingPartMaxBytes || mown > 256) return 0;
    // the deal: per level, CTA-major round-robin (stable in the old order)
    std::vector<int> neworder(n), owner(n);
    for (int l = 0; l < L; ++l) {
        const int a = lev_ptr[l], m = lev_ptr[l + 1] - a;
        int out = a;
        for (int c = 0; c < cs; ++c)
            for (int q = ((c - l) % cs + cs) % cs; q < m; q += cs) {
                neworder[out++] = order[a + q];
                owner[order[a + q]] = c;
            }
    }
    // chunk sizes: blocks of the level's rows whose column CTA c owns
    std::vector<int64_t> nblk(static_cast<size_t>(L) * cs, 0);
    for (int l = 0; l < L; ++l) {
        const int a = lev_ptr[l], m = lev_ptr[l + 1] - a;
        for (int p = a; p < a + m; ++p) {
            const int r = neworder[p];
            for (int64_t k = pat.rowptr[r]; k < pat.rowptr[r + 1]; ++k)
                if (pat.col[k] != r) ++nblk[static_cast<size_t>(l) * cs + owner[pat.col[k]]];
        }
    }
    int maxm = 0;
    for (int l = 0; l < L; ++l) maxm = std::max(maxm, lev_ptr[l + 1] - lev_ptr[l]);
    if (push_scratch_bytes(maxm, B) > kRingScratchMaxBytes) return 0;
    const int cap = ring_capacity(static_cast<int>(smax * B), part * kRingSlots + push_scratch_bytes(maxm, B));
    int64_t pk = 0;
    for (int l = 0; l < L; ++l) {
        const int m = lev_ptr[l + 1] - lev_ptr[l];
        int s0 = lev_ptr[l];
        for (int c = 0; c < cs; ++c) {
            const int nown = dealt(m, c, l, cs);
            const int64_t nb = nblk[static_cast<size_t>(l) * cs + c];
            if (3 * push_chunk_bytes(m, pk, pk + nb, s0, nown, B) > cap) return 0; // two chunks always fit
            pk += nb;
            s0 += nown;
        }
    }
    order.swap(neworder);
    return cs;
}


// Push-sweep structures of a ring-ordered operator (kernels_ring.cu).
static void ring_build(BsrStruct& S, const BsrLayout& lay, cudaStream_t s)
{
    const int cs = lay.ring_cs, n = S.nbr, nlev = S.nlev(), B = S.Rb;
    const int PB = B == 3 ? 4 : 1;
    std::vector<int> owner(n), zl(n), qown(n), cnt(cs, 0), own_ptr(cs + 1, 0);
    std::vector<std::vector<int>> own(cs);
    std::vector<int4> chunk(static_cast<size_t>(nlev) * cs * 2);
    const std::vector<int> flags = push_barriers(S.lev_ptr, cs);
    int mown = 0;
    for (int l = 0; l < nlev; ++l) {
        const int a = S.lev_ptr[l], m = S.lev_ptr[l + 1] - a;
        int sp = a;
        for (int c = 0; c < cs; ++c) {
            const int k = dealt(m, c, l, cs);
            mown = std::max(mown, k);
            chunk[(static_cast<size_t>(l) * cs + c) * 2 + 1] = make_int4(sp, k, cnt[c] * B, flags[l]);
            for (int q = 0; q < k; ++q) {
                owner[sp + q] = c;
                zl[sp + q] = cnt[c] * B;
                qown[sp + q] = q;
                ++cnt[c];
                own[c].push_back(lay.perm[sp + q]);
            }
            sp += k;
        }
    }
    std::vector<int> rown, psrc, pcol, lev_of(n);
    // (pk indices fit int32: checked below)
    for (int l = 0; l < nlev; ++l)
        for (int q = S.lev_ptr[l]; q < S.lev_ptr[l + 1]; ++q) lev_of[q] = l;
    for (int c = 0; c < cs; ++c) {
        own_ptr[c + 1] = own_ptr[c] + static_cast<int>(own[c].size());
        rown.insert(rown.end(), own[c].begin(), own[c].end());
    }
    // packed blocks per level (off-diagonal), then every level in parallel:
    // a counting sort of its blocks by (CTA owning the column, row, part) where
    // part orders [columns on level l-1 | other levels | level l+1]: the first
    // part is the forward sweep's late part, the last the backward's
    std::vector<int64_t> lvl_pk(nlev + 1, 0);
#pragma omp parallel for schedule(dynamic, 8)
    for (int l = 0; l < nlev; ++l) {
        int64_t c0 = 0;
        for (int q = S.lev_ptr[l]; q < S.lev_ptr[l + 1]; ++q)
            for (int k = S.h_rowptr[q]; k < S.h_rowptr[q + 1]; ++k) c0 += lay.inv[S.h_col[k]] != q;
        lvl_pk[l + 1] = c0;
    }
    for (int l = 0; l < nlev; ++l) lvl_pk[l + 1] += lvl_pk[l];
    if (lvl_pk[nlev] >= (1LL << 31)) throw Error(ED_UNSUPPORTED, "push sweep: too many blocks");
    psrc.resize(lvl_pk[nlev]);
    pcol.resize(lvl_pk[nlev]);
    std::vector<int4> seg(static_cast<size_t>(n) * cs);
    bool too_long = false;
#pragma omp parallel for schedule(dynamic, 8) reduction(|| : too_long)
    for (int l = 0; l < nlev; ++l) {
        const int a = S.lev_ptr[l], m = S.lev_ptr[l + 1] - a;
        const int K = cs * m * 3;
        std::vector<int> start(K + 1, 0);
        auto key = [&](int q, int k) {
            const int sc = lay.inv[S.h_col[k]];
            const int lc = lev_of[sc];
            const int part_of = lc == l - 1 ? 0 : lc == l + 1 ? 2 : 1;
            return (owner[sc] * m + (q - a)) * 3 + part_of;
        };
        for (int q = a; q < a + m; ++q)
            for (int k = S.h_rowptr[q]; k < S.h_rowptr[q + 1]; ++k)
                if (lay.inv[S.h_col[k]] != q) ++start[key(q, k) + 1];
        for (int i = 0; i < K; ++i) start[i + 1] += start[i];
        std::vector<int> pos(start.begin(), start.end() - 1);
        const int64_t base = lvl_pk[l];
        for (int q = a; q < a + m; ++q)
            for (int k = S.h_rowptr[q]; k < S.h_rowptr[q + 1]; ++k) {
                const int sc = lay.inv[S.h_col[k]];
                if (sc == q) continue;
                const int64_t at = base + pos[key(q, k)]++;
                psrc[at] = k;
                pcol[at] = zl[sc];
            }
        for (int c = 0; c < cs; ++c) {
            chunk[(static_cast<size_t>(l) * cs + c) * 2] =
                make_int4(cs * a + c * m, m, static_cast<int>(base + start[c * m * 3]),
                          static_cast<int>(base + start[(c + 1) * m * 3]));
            for (int qi = 0; qi < m; ++qi) {
                const int kk = (c * m + qi) * 3;
                const int na = start[kk + 1] - start[kk], nb = start[kk + 3] - start[kk + 2];
                too_long = too_long || na > 0xFFFF || nb > 0xFFFF;
                const int q = a + qi;
                seg[static_cast<size_t>(cs) * a + c * m + qi] =
                    make_int4(static_cast<int>(base + start[kk]), static_cast<int>(base + start[kk + 3]),
                              (owner[q] << 24) | ((qown[q] * cs + c) * PB * 8), (na << 16) | nb);
            }
        }
    }
    if (too_long) throw Error(ED_UNSUPPORTED, "push sweep: row segment too long");
    S.ring_cs = cs;
    S.ring_slice = *std::max_element(cnt.begin(), cnt.end()) * B;
    S.ring_part = mown * cs * PB * 8;
    int maxm = 0;
    for (int l = 0; l < nlev; ++l) maxm = std::max(maxm, S.lev_ptr[l + 1] - S.lev_ptr[l]);
    S.ring_maxm = maxm;
    S.ring_cap = ring_capacity(S.ring_slice, S.ring_part * kRingSlots + push_scratch_bytes(maxm, B));
    S.ring_npk = static_cast<int64_t>(psrc.size());
    S.rchunk.upload(chunk, s);
    S.rseg.upload(seg, s);
    S.rpcol.upload(pcol, s);
    S.rpsrc.upload(psrc, s);
    S.rown.upload(rown, s);
    S.rown_ptr.upload(own_ptr, s);
}

bool pattern_symmetric(const BlockPattern& pat)
{
    if (pat.nbr != pat.nbc) return false;
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(| : bad)
    for (int i = 0; i < pat.nbr; ++i)
        for (int64_t k = pat.rowptr[i]; k < pat.rowptr[i + 1] && !bad; ++k) {
            const int j = pat.col[k];
            const auto b = pat.col.begin() + pat.rowptr[j];
            const auto e = pat.col.begin() + pat.rowptr[j + 1];
            if (!std::binary_search(b, e, i)) bad = 1;
        }
    return bad == 0;
}

BsrLayout make_layout(const BlockPattern& pat, const std::vector<int>& row_order, const std::vector<int>& level_of_pos)
{
    BsrLayout L;
    const int n = pat.nbr;
    L.perm = row_order;
    L.inv.assign(n, -1);
    for (int s = 0; s < n; ++s) L.inv[row_order[s]] = s;
    L.lev_ptr.push_back(0);
    for (int s = 1; s < n; ++s)
        if (!level_of_pos.empty() && level_of_pos[s] != level_of_pos[s - 1]) L.lev_ptr.push_back(s);
    L.lev_ptr.push_back(n);
    std::vector<int64_t> srp(n + 1, 0);
    for (int s = 0; s < n; ++s) {
        const int r = row_order[s];
        srp[s + 1] = srp[s] + (pat.rowptr[r + 1] - pat.rowptr[r]);
    }
    L.addr.assign(pat.nnzb(), -1);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int r = 0; r < n; ++r)
        for (int64_t k = pat.rowptr[r]; k < pat.rowptr[r + 1]; ++k) L.addr[k] = srp[L.inv[r]] + (k - pat.rowptr[r]);
    return L;
}

// lanes per block row: about one block per lane for multi-entry blocks; for
// scalar (1x1) operators ~4 entries per lane, so each lane keeps several
// independent loads in flight and the last partial pass wastes fewer lanes
int auto_lanes(double avg_blocks, int entries)
{
    const double per_lane = entries == 1 ? 4.0 : 1.0;
    int L = 2;
    while (L < 32 && L * 2 * per_lane < avg_blocks) L *= 2;
    return L;
}

std::shared_ptr<BsrStruct> bsr_make_struct(const BlockPattern& pat, const BsrLayout& lay, int Rb, int Cb,
                                           cudaStream_t s, int lanes)
{
    if (pat.nnzb() >= (1LL << 31)) throw Error(ED_UNSUPPORTED, "operator exceeds int32 block indices");
    auto st = std::make_shared<BsrStruct>();
    BsrStruct& S = *st;
    S.Rb = Rb;
    S.Cb = Cb;
    S.nbr = pat.nbr;
    S.nbc = pat.nbc;
    S.nnzb = pat.nnzb();
    const int n = pat.nbr;
    S.L = lanes > 0 ? lanes : auto_lanes(n > 0 ? static_cast<double>(S.nnzb) / n : 1.0, Rb * Cb);
    // sweeps are latency-bound: as many lanes as blocks per row (shorter chains)
    static const int ls_env = std::getenv("ED_SGS_LANES") ? std::atoi(std::getenv("ED_SGS_LANES")) : 0;
    S.Ls = lanes > 0 ? lanes : ls_env > 0 ? ls_env : auto_lanes(n > 0 ? static_cast<double>(S.nnzb) / n : 1.0, 9);
    S.h_rowptr.assign(n + 1, 0);
    S.h_col.assign(S.nnzb, 0);
    bool identity = true;
    for (int s2 = 0; s2 < n; ++s2) identity = identity && lay.perm[s2] == s2;
    std::vector<int> dpos(n, -1);
    for (int s2 = 0; s2 < n; ++s2) {
        const int r = lay.perm[s2];
        S.h_rowptr[s2 + 1] = static_cast<int>(S.h_rowptr[s2] + (pat.rowptr[r + 1] - pat.rowptr[r]));
    }
#pragma omp parallel for schedule(dynamic, 1024)
    for (int s2 = 0; s2 < n; ++s2) {
        const int r = lay.perm[s2];
        const int64_t len = pat.rowptr[r + 1] - pat.rowptr[r];
        for (int64_t k = 0; k < len; ++k) {
            const int c = pat.col[pat.rowptr[r] + k];
            S.h_col[S.h_rowptr[s2] + k] = c;
            if (c == r && pat.nbr == pat.nbc) dpos[s2] = static_cast<int>(S.h_rowptr[s2] + k);
        }
    }
    if (!identity) {
        S.h_perm = lay.perm;
        S.h_inv = lay.inv;
        S.perm.upload(S.h_perm, s);
        S.inv.upload(S.h_inv, s);
    }
    S.lev_ptr = lay.lev_ptr;
    S.leveled = !identity || S.lev_ptr.size() > 2;
    S.rowptr.upload(S.h_rowptr, s);
    S.col.upload(S.h_col, s);
    if (pat.nbr == pat.nbc) S.dpos.upload(dpos, s);
    // dataflow items: rows_per_item rows of one level each (256 threads / L lanes)
    const int nlev = S.nlev();
    S.rows_per_item = 256 / S.Ls;
    std::vector<int> irow{0}, ilev, lcnt(std::max(nlev, 1), 0);
    for (int l = 0; l < nlev; ++l)
        for (int r0 = S.lev_ptr[l]; r0 < S.lev_ptr[l + 1]; r0 += S.rows_per_item) {
            irow.push_back(std::min(r0 + S.rows_per_item, S.lev_ptr[l + 1]));
            ilev.push_back(l);
            ++lcnt[l];
        }
    S.nitems = static_cast<int>(ilev.size());
    S.item_row.upload(irow, s);
    S.item_level.upload(ilev, s);
    S.lev_items.upload(lcnt, s);
    S.sync.alloc(static_cast<size_t>(std::max(nlev, 1)) + 2);
    S.sync.zero(s);
    S.d_lev_ptr.upload(S.lev_ptr, s);
    // structural symmetry (sorted columns): every later neighbour of a row waits on that row, which is
    // what lets the tagged dataflow sweep read later neighbours' old values without a level barrier
    S.sym_pattern = false;
    if (S.leveled && pat.nbr == pat.nbc) {
        int asym = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : asym)
        for (int r = 0; r < n; ++r)
            for (int64_t k = pat.rowptr[r]; k < pat.rowptr[r + 1]; ++k) {
                const int c = pat.col[k];
                if (c == r) continue;
                const int* b0 = pat.col.data() + pat.rowptr[c];
                const int* b1 = pat.col.data() + pat.rowptr[c + 1];
                const int* it = std::lower_bound(b0, b1, r);
                if (it == b1 || *it != r) ++asym;
            }
        S.sym_pattern = asym == 0;
    }
    // narrow level schedules (every level fits one 512-thread CTA in <= 2 passes) run as one CTA
    int widest = 0;
    for (int l = 0; l < nlev; ++l) widest = std::max(widest, S.lev_ptr[l + 1] - S.lev_ptr[l]);
    S.chain = static_cast<int64_t>(widest) * S.Ls <= 1024;
    S.avg_rows_per_level = nlev > 0 ? S.nbr / nlev : 0;
    if (lay.ring_cs > 0 && Rb == Cb && pat.nbr == pat.nbc) {
        ring_build(S, lay, s);
    }
    if (Rb == Cb && (Rb == 1 || Rb == 3) && pat.nbr == pat.nbc && S.leveled && S.nbr > 0) group_build(S, s);
    ED_CUDA(cudaStreamSynchronize(s)); // host vectors die at return
    return st;
}

void group_build(BsrStruct& S, cudaStream_t s)
{
    // narrow consecutive levels are merged while the group has <= grp_rows
    // scalar rows; a level wider than a quarter of that is a group of its own
    static const int grp_rows = std::getenv("ED_GROUP_ROWS") ? std::atoi(std::getenv("ED_GROUP_ROWS")) : 1024;
    const int B = S.Rb, n = S.nbr, nlev = S.nlev();
    std::vector<int4> grp;
    std::vector<int> grp_of(n, -1);
    for (int l = 0; l < nlev;) {
        const int a = S.lev_ptr[l];
        int e = l + 1;
        int m = (S.lev_ptr[e] - a) * B;
        if (grp_rows > 0 && 4 * m <= grp_rows)
            while (e < nlev && m + (S.lev_ptr[e + 1] - S.lev_ptr[e]) * B <= grp_rows &&
                   4 * (S.lev_ptr[e + 1] - S.lev_ptr[e]) * B <= grp_rows) {
                m += (S.lev_ptr[e + 1] - S.lev_ptr[e]) * B;
                ++e;
            }
        const int b = S.lev_ptr[e];
        const bool multi = e - l > 1;
        for (int r = a; r < b; ++r) grp_of[r] = multi ? static_cast<int>(grp.size()) : -1;
        grp.push_back(make_int4(a, b, multi ? m : 0, 0));
        l = e;
    }
    S.ngrp = static_cast<int>(grp.size());
    std::vector<long long> toff(grp.size(), 0);
    std::vector<int2> chunks;
    int64_t tot = 0;
    int maxm = 0;
    for (size_t g = 0; g < grp.size(); ++g) {
        const int m = grp[g].z;
        toff[g] = tot;
        if (m == 0) continue;
        tot += static_cast<int64_t>(m) * (m + 1) / 2;
        maxm = std::max(maxm, m);
        for (int j0 = 0; j0 < m; j0 += 32) chunks.push_back(make_int2(static_cast<int>(g), j0));
    }
    S.grp_tinv = tot;
    S.grp_maxm = maxm;
    // cluster scope (one 16-CTA cluster: ~0.1 us barriers, but 16 SMs of
    // bandwidth) measured slower than the whole grid at 40^3 for every level
    // (profiles/r02/sweeps.md); opt-in below ED_GROUP_CLUSTER_MB
    static const double cl_max = std::getenv("ED_GROUP_CLUSTER_MB") ? std::atof(std::getenv("ED_GROUP_CLUSTER_MB")) : 0.0;
    const double sweep_bytes = static_cast<double>(S.nnzb) * (8.0 * B * B + 4.0) + 8.0 * static_cast<double>(tot);
    S.grp_cluster = sweep_bytes <= cl_max * 1e6;
    // measured at 40^3 (profiles/r02/sweeps.md): one grid barrier costs ~1.3 us,
    // so level groups pay on narrow deep schedules (a coarse level: ~36 block
    // rows per level -> 9 levels per group step); wide levels stay on the
    // dataflow / cluster push sweeps, which need no grid-wide barrier per level
    static const int max_rpl = std::getenv("ED_GROUP_MAX_RPL") ? std::atoi(std::getenv("ED_GROUP_MAX_RPL")) : 64;
    S.grp_use = nlev > 0 && static_cast<double>(n) / nlev <= max_rpl && tot > 0;
    S.ntchunk = static_cast<int>(chunks.size());
    const bool identity = S.h_inv.empty();
    std::vector<unsigned char> code(S.nnzb, 0);
    std::vector<int> gptr(n + 1, 0), gblk;
    std::vector<int> gcnt(n, 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int sr = 0; sr < n; ++sr) {
        const int row = identity ? sr : S.h_perm[sr];
        int cnt = 0;
        for (int k = S.h_rowptr[sr]; k < S.h_rowptr[sr + 1]; ++k) {
            const int c = S.h_col[k];
            const int sc = identity ? c : S.h_inv[c];
            if (c == row) code[k] = 3;
            else if (grp_of[sr] >= 0 && grp_of[sc] == grp_of[sr]) code[k] = sc < sr ? 1 : 2;
            if (grp_of[sr] >= 0 && code[k] != 0) ++cnt;
        }
        gcnt[sr] = cnt;
    }
    for (int sr = 0; sr < n; ++sr) gptr[sr + 1] = gptr[sr] + gcnt[sr];
    gblk.resize(gptr[n]);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int sr = 0; sr < n; ++sr) {
        if (grp_of[sr] < 0) continue;
        int o = gptr[sr];
        for (int k = S.h_rowptr[sr]; k < S.h_rowptr[sr + 1]; ++k)
            if (code[k] != 0) gblk[o++] = k;
    }
    S.grp.upload(grp, s);
    S.grp_toff.upload(toff, s);
    S.bcode.upload(code, s);
    S.gptr.upload(gptr, s);
    if (gblk.empty()) gblk.push_back(0);
    S.gblk.upload(gblk, s);
    if (chunks.empty()) chunks.push_back(make_int2(0, 0));
    S.tchunk.upload(chunks, s);
    S.gbar.alloc(1);
    S.gsbuf.alloc(std::max(maxm, 1));
}

std::vector<double> bsr_pack_values(const BsrStruct& st, const BsrLayout& lay, const std::vector<double>& bvals)
{
    const int E = st.Rb * st.Cb;
    std::vector<double> v(static_cast<size_t>(st.nval()), 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < static_cast<int64_t>(lay.addr.size()); ++k)
        for (int e = 0; e < E; ++e) v[lay.addr[k] * E + e] = bvals[k * E + e];
    return v;
}

BlockPattern block_pattern_of_csr(const HostCsr& a, int Rb, int Cb)
{
    if (a.nrows % Rb != 0 || a.ncols % Cb != 0)
        throw Error(ED_INVALID_ARGUMENT, "matrix size is not a multiple of the block size");
    BlockPattern p;
    p.nbr = a.nrows / Rb;
    p.nbc = a.ncols / Cb;
    p.rowptr.assign(p.nbr + 1, 0);
    std::vector<std::vector<int>> rows(p.nbr);
#pragma omp parallel
    {
        std::vector<int> mark(p.nbc, -1);
#pragma omp for schedule(dynamic, 1024)
        for (int I = 0; I < p.nbr; ++I) {
            auto& cols = rows[I];
            for (int r = I * Rb; r < (I + 1) * Rb; ++r)
                for (int64_t k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
                    const int J = a.col[k] / Cb;
                    if (mark[J] != I) {
                        mark[J] = I;
                        cols.push_back(J);
                    }
                }
            std::sort(cols.begin(), cols.end());
        }
    }
    for (int I = 0; I < p.nbr; ++I) p.rowptr[I + 1] = p.rowptr[I] + static_cast<int64_t>(rows[I].size());
    p.col.resize(p.rowptr[p.nbr]);
#pragma omp parallel for schedule(static)
    for (int I = 0; I < p.nbr; ++I) std::copy(rows[I].begin(), rows[I].end(), p.col.begin() + p.rowptr[I]);
    return p;
}

std::vector<double> block_values_of_csr(const HostCsr& a, const BlockPattern& pat, int Rb, int Cb)
{
    const int E = Rb * Cb;
    std::vector<double> v(static_cast<size_t>(pat.nnzb()) * E, 0.0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int I = 0; I < pat.nbr; ++I) {
        const auto b = pat.col.begin() + pat.rowptr[I];
        const auto e = pat.col.begin() + pat.rowptr[I + 1];
        for (int rr = 0; rr < Rb; ++rr) {
            const int r = I * Rb + rr;
            for (int64_t k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
                const int c = a.col[k];
                const int J = c / Cb, d = c % Cb;
                const int64_t blk = pat.rowptr[I] + (std::lower_bound(b, e, J) - b);
                v[static_cast<size_t>(blk) * E + rr * Cb + d] = a.val[k];
            }
        }
    }
    return v;
}

Bsr bsr_from_csr(const HostCsr& a, int Rb, int Cb, bool leveled, cudaStream_t s)
{
    const BlockPattern pat = block_pattern_of_csr(a, Rb, Cb);
    std::vector<int> order, lvl;
    int ring_cs = 0;
    if (leveled) {
        if (!pattern_symmetric(pat)) throw Error(ED_UNSUPPORTED, "Gauss-Seidel operator pattern is not symmetric");
        int nlev = 0;
        gs_level_order(pat, order, lvl, nlev);
        ring_cs = Rb == Cb ? ring_order(pat, Rb, order, lvl, nlev) : 0;
    } else {
        order.resize(pat.nbr);
        std::iota(order.begin(), order.end(), 0);
    }
    BsrLayout lay = make_layout(pat, order, lvl);
    lay.ring_cs = ring_cs;
    Bsr m;
    m.st = bsr_make_struct(pat, lay, Rb, Cb, s);
    if (leveled) m.st->leveled = true;
    m.val.upload(bsr_pack_values(*m.st, lay, block_values_of_csr(a, pat, Rb, Cb)), s);
    ED_CUDA(cudaStreamSynchronize(s));
    return m;
}

HostCsr bsr_to_csr(const Bsr& m, cudaStream_t s)
{
    const BsrStruct& S = *m.st;
    const std::vector<double> v = m.val.to_host(s);
    const int E = S.Rb * S.Cb;
    HostCsr a;
    a.nrows = S.nbr * S.Rb;
    a.ncols = S.nbc * S.Cb;
    a.rowptr.assign(a.nrows + 1, 0);
    auto srow = [&](int I) { return S.h_inv.empty() ? I : S.h_inv[I]; };
    for (int I = 0; I < S.nbr; ++I) {
        const int s2 = srow(I);
        for (int rr = 0; rr < S.Rb; ++rr)
            a.rowptr[I * S.Rb + rr + 1] = static_cast<int64_t>(S.h_rowptr[s2 + 1] - S.h_rowptr[s2]) * S.Cb;
    }
    for (int r = 0; r < a.nrows; ++r) a.rowptr[r + 1] += a.rowptr[r];
    a.col.resize(a.rowptr[a.nrows]);
    a.val.resize(a.rowptr[a.nrows]);
#pragma omp parallel for schedule(static)
    for (int I = 0; I < S.nbr; ++I) {
        const int s2 = srow(I);
        for (int rr = 0; rr < S.Rb; ++rr) {
            int64_t out = a.rowptr[I * S.Rb + rr];
            for (int k = S.h_rowptr[s2]; k < S.h_rowptr[s2 + 1]; ++k) {
                const int J = S.h_col[k];
                for (int d = 0; d < S.Cb; ++d) {
                    a.col[out] = J * S.Cb + d;
                    a.val[out] = v[static_cast<size_t>(k) * E + rr * S.Cb + d];
                    ++out;
                }
            }
        }
    }
    return a;
}

} // namespace edb

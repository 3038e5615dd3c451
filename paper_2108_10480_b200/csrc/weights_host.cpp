// weights_host.cpp -- host precompute of the WeightSet (drop-in for
// build_adjacency + build_weight_set, mesh.hpp:163-183 and
// weights.hpp:46-76, 176-621), exported through sd_build_weights.
//
// Valences: vertex = incident non-point simplices; edge = simplices (edges
// and triangles) containing the undirected edge. Edge polynomials have a
// closed form. Triangle polynomials follow the reference construction:
// 36-equation system in the degree-7 Bernstein basis, minimum-norm
// solution, a small exact LP over the swap-symmetric null space that
// raises the smallest Bernstein coefficient, then exchange rounds on the
// sampled domain minimum. The linear algebra here is a column-pivoted
// Householder QR of (A T)^T (range / null space from Q, minimum-norm
// solution by forward substitution) -- a different factorisation from the
// reference's JacobiSVD; for this well-separated spectrum (smallest kept
// singular value ~0.13, discarded ~1e-13) both give the same polynomial
// to ~1e-12.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <unordered_map>
#include <vector>

#include "weights_host.h"

namespace sdgpu {
namespace wh {

constexpr int M36 = 36;
inline int mono(int j, int k) { return j * 8 - j * (j - 1) / 2 + k; }
struct JK {
    int j, k;
};
static const std::vector<JK>& monos() {
    static const std::vector<JK> m = [] {
        std::vector<JK> v;
        for (int j = 0; j <= 7; ++j)
            for (int k = 0; j + k <= 7; ++k) v.push_back({j, k});
        return v;
    }();
    return m;
}
using Grid = std::array<std::array<double, 8>, 8>;
using Vec = std::vector<double>;
struct Mat {
    int r, c;
    std::vector<double> a;
    Mat(int rr = 0, int cc = 0) : r(rr), c(cc), a(size_t(rr) * cc, 0.0) {}
    double& operator()(int i, int j) { return a[size_t(i) * c + j]; }
    double operator()(int i, int j) const { return a[size_t(i) * c + j]; }
};

static double horner(const Grid& g, double x, double y) {  // weights.hpp:103-111
    double acc = 0.0;
    for (int j = 7; j >= 0; --j) {
        double row = 0.0;
        for (int k = 7; k >= 0; --k) row = row * y + g[j][k];
        acc = acc * x + row;
    }
    return acc;
}

static void system(int v, int e, Mat& A, Vec& b) {  // weights.hpp:183-241
    A = Mat(36, M36);
    b.assign(36, 0.0);
    int row = 0;
    auto pt = [&](double x, double y, double t) {
        for (const JK& m : monos()) A(row, mono(m.j, m.k)) = std::pow(x, m.j) * std::pow(y, m.k);
        b[row++] = t;
    };
    const double iv = 1.0 / v, ie = 1.0 / e;
    const double P[10][3] = {{0, 0, iv},         {1, 0, iv},         {0, 1, iv},         {1. / 3, 0, ie},
                             {2. / 3, 0, ie},    {0, 1. / 3, ie},    {0, 2. / 3, ie},    {1. / 3, 2. / 3, ie},
                             {2. / 3, 1. / 3, ie}, {1. / 3, 1. / 3, double(v - 1) / v}};
    for (const auto& p : P) pt(p[0], p[1], p[2]);
    for (int k = 0; k <= 6; ++k) A(row++, mono(1, k)) = 1.0;
    for (int j = 0; j <= 6; ++j)
        if (j != 1) A(row++, mono(j, 1)) = 1.0;
    auto binom = [](int n, int r) {
        double o = 1.0;
        for (int i = 0; i < r; ++i) o = o * (n - i) / (i + 1);
        return o;
    };
    for (int sw = 0; sw < 2; ++sw)
        for (int m = 0; m <= (sw ? 5 : 6); ++m) {
            for (const JK& mo : monos()) {
                double coef = 0.0;
                const int px[2] = {mo.j - 1, mo.j}, py[2] = {mo.k, mo.k - 1};
                const double c[2] = {double(mo.j), double(mo.k)};
                for (int q = 0; q < 2; ++q) {
                    if (c[q] == 0.0) continue;
                    const int tp = sw ? py[q] : px[q], op = sw ? px[q] : py[q], r = m - tp;
                    if (r >= 0 && r <= op) coef += c[q] * binom(op, r) * ((r & 1) ? -1.0 : 1.0);
                }
                A(row, mono(mo.j, mo.k)) += coef;
            }
            ++row;
        }
}

static const Mat& bernstein() {  // weights.hpp:247-271
    static const Mat T = [] {
        auto f = [](int n) { double o = 1; for (int i = 2; i <= n; ++i) o *= i; return o; };
        Mat B(M36, M36);
        for (const JK& m : monos()) {
            const int a = m.j, bb = m.k, c = 7 - a - bb;
            const double mult = f(7) / (f(a) * f(bb) * f(c));
            for (int p = 0; p <= c; ++p)
                for (int q = 0; p + q <= c; ++q)
                    B(mono(a + p, bb + q), mono(a, bb)) +=
                        mult * f(c) / (f(p) * f(q) * f(c - p - q)) * (((p + q) & 1) ? -1.0 : 1.0);
        }
        return B;
    }();
    return T;
}

static Mat mul(const Mat& x, const Mat& y) {
    Mat z(x.r, y.c);
    for (int i = 0; i < x.r; ++i)
        for (int k = 0; k < x.c; ++k)
            for (int j = 0; j < y.c; ++j) z(i, j) += x(i, k) * y(k, j);
    return z;
}
static Vec mulv(const Mat& x, const Vec& v) {
    Vec o(x.r, 0.0);
    for (int i = 0; i < x.r; ++i)
        for (int k = 0; k < x.c; ++k) o[i] += x(i, k) * v[k];
    return o;
}

// Column-pivoted Householder QR of X (n x n): X P = Q R. Returns Q
// (explicit, n x n), R, the pivot order and the numerical rank (|R_ii| >
// rel * |R_00|).
struct QRCP {
    Mat Q, R;
    std::vector<int> piv;
    int rank = 0;
};
static QRCP qrcp(Mat X, double rel) {
    const int n = X.r;
    QRCP o;
    o.piv.resize(n);
    for (int j = 0; j < n; ++j) o.piv[j] = j;
    std::vector<Vec> hv;
    for (int k = 0; k < n; ++k) {
        int best = k;
        double bn = -1;
        for (int j = k; j < n; ++j) {
            double s = 0;
            for (int i = k; i < n; ++i) s += X(i, j) * X(i, j);
            if (s > bn) bn = s, best = j;
        }
        if (best != k) {
            for (int i = 0; i < n; ++i) std::swap(X(i, k), X(i, best));
            std::swap(o.piv[k], o.piv[best]);
        }
        Vec v(n, 0.0);
        double nrm = 0;
        for (int i = k; i < n; ++i) nrm += X(i, k) * X(i, k);
        nrm = std::sqrt(nrm);
        const double alpha = X(k, k) > 0 ? -nrm : nrm;
        for (int i = k; i < n; ++i) v[i] = X(i, k);
        v[k] -= alpha;
        double vn = 0;
        for (int i = k; i < n; ++i) vn += v[i] * v[i];
        if (vn > 0) {
            for (int j = k; j < n; ++j) {
                double s = 0;
                for (int i = k; i < n; ++i) s += v[i] * X(i, j);
                s = 2 * s / vn;
                for (int i = k; i < n; ++i) X(i, j) -= s * v[i];
            }
        }
        hv.push_back(v);
    }
    o.R = X;
    o.Q = Mat(n, n);
    for (int i = 0; i < n; ++i) o.Q(i, i) = 1.0;
    for (int k = n - 1; k >= 0; --k) {  // Q = H_0 H_1 ... H_{n-1}
        const Vec& v = hv[k];
        double vn = 0;
        for (int i = k; i < n; ++i) vn += v[i] * v[i];
        if (vn <= 0) continue;
        for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int i = k; i < n; ++i) s += v[i] * o.Q(i, j);
            s = 2 * s / vn;
            for (int i = k; i < n; ++i) o.Q(i, j) -= s * v[i];
        }
    }
    const double r0 = std::abs(o.R(0, 0));
    while (o.rank < n && std::abs(o.R(o.rank, o.rank)) > rel * r0) ++o.rank;
    return o;
}

// weights.hpp:277-334: max t s.t. base_i + rows_i . g >= t (exact vertex
// enumeration over (r+1)-subsets of tight constraints)
static Vec maxmin(const Mat& rows, const Vec& base) {
    const int m = int(base.size()), r = rows.c;
    Vec best(r, 0.0);
    if (r == 0 || m < r + 1) return best;
    double bt = *std::min_element(base.begin(), base.end());
    const int n = r + 1;
    std::vector<int> pick(n);
    for (int i = 0; i < n; ++i) pick[i] = i;
    double W[5][6], u[5];
    for (;;) {
        for (int s = 0; s < n; ++s) {
            for (int g = 0; g < r; ++g) W[s][g] = rows(pick[s], g);
            W[s][r] = -1.0;
            W[s][n] = -base[pick[s]];
        }
        bool ok = true;
        for (int col = 0; col < n && ok; ++col) {
            int p = col;
            for (int s = col + 1; s < n; ++s)
                if (std::abs(W[s][col]) > std::abs(W[p][col])) p = s;
            if (std::abs(W[p][col]) < 1e-12) {
                ok = false;
                break;
            }
            if (p != col)
                for (int cc = 0; cc <= n; ++cc) std::swap(W[p][cc], W[col][cc]);
            for (int s = 0; s < n; ++s) {
                if (s == col) continue;
                const double f = W[s][col] / W[col][col];
                for (int cc = col; cc <= n; ++cc) W[s][cc] -= f * W[col][cc];
            }
        }
        if (ok) {
            for (int s = 0; s < n; ++s) u[s] = W[s][n] / W[s][s];
            if (u[r] > bt) {
                bool feas = true;
                for (int i = 0; i < m && feas; ++i) {
                    double val = base[i];
                    for (int g = 0; g < r; ++g) val += rows(i, g) * u[g];
                    feas = val >= u[r] - 1e-11;
                }
                if (feas) {
                    bt = u[r];
                    for (int g = 0; g < r; ++g) best[g] = u[g];
                }
            }
        }
        int pos = n - 1;
        while (pos >= 0 && pick[pos] == m - n + pos) --pos;
        if (pos < 0) break;
        ++pick[pos];
        for (int s = pos + 1; s < n; ++s) pick[s] = pick[s - 1] + 1;
    }
    return best;
}

static Grid grid_of(const Vec& z) {
    Grid g{};
    const Vec mc = mulv(bernstein(), z);
    for (const JK& m : monos()) g[m.j][m.k] = mc[mono(m.j, m.k)];
    return g;
}

static double domain_min(const Grid& g, int N, double& ax, double& ay) {  // weights.hpp:401-430
    double lo = INFINITY;
    for (int i = 0; i <= N; ++i)
        for (int j = 0; i + j <= N; ++j) {
            const double w = horner(g, double(i) / N, double(j) / N);
            if (w < lo) lo = w, ax = double(i) / N, ay = double(j) / N;
        }
    for (int i = 0; i <= 8 * N; ++i) {
        const double t = 0.5 * i / (8 * N);
        const double w = horner(g, t, t);
        if (w < lo) lo = w, ax = t, ay = t;
    }
    for (double step = 1.0 / N; step > 1e-13;) {
        bool moved = false;
        const double cand[4][2] = {{ax + step, ay}, {ax - step, ay}, {ax, ay + step}, {ax, ay - step}};
        for (const auto& c : cand) {
            if (c[0] < 0 || c[1] < 0 || c[0] + c[1] > 1) continue;
            const double w = horner(g, c[0], c[1]);
            if (w < lo) lo = w, ax = c[0], ay = c[1], moved = true;
        }
        if (!moved) step *= 0.5;
    }
    return lo;
}

static const int kStored[13][2] = {{0, 0}, {0, 2}, {0, 3}, {0, 4}, {0, 5}, {0, 6}, {0, 7},
                                   {2, 2}, {2, 3}, {2, 4}, {2, 5}, {3, 3}, {3, 4}};

TriWeight build_tri(int v, int e) {
    Mat A;
    Vec b;
    system(v, e, A, b);
    const Mat& T = bernstein();
    const Mat AT = mul(A, T);
    Mat X(M36, M36);  // X = (A T)^T
    for (int i = 0; i < M36; ++i)
        for (int j = 0; j < M36; ++j) X(i, j) = AT(j, i);
    const QRCP f = qrcp(X, 1e-10);
    const int r = f.rank;
    // minimum-norm solution: z = Q_r y with R11^T y = (P^T b)_r
    Vec y(r, 0.0);
    for (int i = 0; i < r; ++i) {
        double s = b[f.piv[i]];
        for (int k = 0; k < i; ++k) s -= f.R(k, i) * y[k];
        y[i] = s / f.R(i, i);
    }
    Vec z(M36, 0.0);
    for (int i = 0; i < M36; ++i)
        for (int k = 0; k < r; ++k) z[i] += f.Q(i, k) * y[k];
    // swap-symmetric null space: symmetrise Q's null columns, project out
    // the range, keep an orthonormal basis (largest-first Gram-Schmidt)
    std::vector<Vec> cand;
    for (int c = r; c < M36; ++c) {
        Vec s(M36);
        for (const JK& m : monos()) s[mono(m.j, m.k)] = 0.5 * (f.Q(mono(m.j, m.k), c) + f.Q(mono(m.k, m.j), c));
        for (int k = 0; k < r; ++k) {
            double d = 0;
            for (int i = 0; i < M36; ++i) d += f.Q(i, k) * s[i];
            for (int i = 0; i < M36; ++i) s[i] -= d * f.Q(i, k);
        }
        cand.push_back(s);
    }
    std::vector<Vec> dirs;
    while (int(dirs.size()) < 4 && !cand.empty()) {
        int best = -1;
        double bn = 1e-8;
        for (int i = 0; i < int(cand.size()); ++i) {
            double nn = 0;
            for (double x : cand[i]) nn += x * x;
            nn = std::sqrt(nn);
            if (nn > bn) bn = nn, best = i;
        }
        if (best < 0) break;
        Vec d = cand[best];
        for (double& x : d) x /= bn;
        cand.erase(cand.begin() + best);
        for (Vec& s : cand) {
            double p = 0;
            for (int i = 0; i < M36; ++i) p += d[i] * s[i];
            for (int i = 0; i < M36; ++i) s[i] -= p * d[i];
        }
        dirs.push_back(d);
    }
    const int nd = int(dirs.size());
    if (nd > 0) {
        Mat cr(M36, nd);
        for (int g = 0; g < nd; ++g)
            for (int i = 0; i < M36; ++i) cr(i, g) = dirs[g][i];
        const Vec gam = maxmin(cr, z);
        for (int g = 0; g < nd; ++g)
            for (int i = 0; i < M36; ++i) z[i] += gam[g] * dirs[g][i];
        double ax = 0, ay = 0;
        double lo = domain_min(grid_of(z), 384, ax, ay);
        if (v >= e && lo * v < 1.0 - 1e-10) {  // exchange rounds, weights.hpp:437-502
            std::vector<std::array<double, 2>> pts;
            for (int i = 0; i <= 4; ++i)
                for (int j = 0; i + j <= 4; ++j) pts.push_back({i / 4.0, j / 4.0});
            for (double h = 1e-2; h >= 1e-7; h *= 0.1) {
                pts.push_back({1.0 / 3 - h, 1.0 / 3 - h});
                pts.push_back({1.0 / 3 + h, 1.0 / 3 + h});
                pts.push_back({h, h});
                pts.push_back({0.5 - h, 0.5 - h});
            }
            const size_t seeds = pts.size();
            std::vector<Grid> dg;
            for (int g = 0; g < nd; ++g) dg.push_back(grid_of(dirs[g]));
            const Grid bg = grid_of(z);
            Vec bz = z;
            double blo = lo;
            for (int round = 0; round < 80; ++round) {
                pts.push_back({ax, ay});
                Mat rows(int(pts.size()), nd);
                Vec base(pts.size());
                for (size_t s = 0; s < pts.size(); ++s) {
                    base[s] = horner(bg, pts[s][0], pts[s][1]);
                    for (int g = 0; g < nd; ++g) rows(int(s), g) = horner(dg[g], pts[s][0], pts[s][1]);
                }
                const Vec d = maxmin(rows, base);
                double model = INFINITY;
                Vec vals(pts.size());
                for (size_t s = 0; s < pts.size(); ++s) {
                    double val = base[s];
                    for (int g = 0; g < nd; ++g) val += rows(int(s), g) * d[g];
                    vals[s] = val;
                    model = std::min(model, val);
                }
                if (pts.size() > 60) {
                    std::vector<std::array<double, 2>> kept(pts.begin(), pts.begin() + seeds);
                    for (size_t s = seeds; s < pts.size(); ++s)
                        if (vals[s] - model < 1e-9 || s + 12 >= pts.size()) kept.push_back(pts[s]);
                    pts.swap(kept);
                }
                Vec zc = z;
                for (int g = 0; g < nd; ++g)
                    for (int i = 0; i < M36; ++i) zc[i] += d[g] * dirs[g][i];
                lo = domain_min(grid_of(zc), 384, ax, ay);
                bool done = lo * v >= 1.0 - 1e-12 || model - lo < 1e-13;
                if (done) {
                    double vx = 0, vy = 0;
                    const double fine = domain_min(grid_of(zc), 1536, vx, vy);
                    if (fine < lo - 1e-13) lo = fine, ax = vx, ay = vy, done = false;
                    else lo = std::min(lo, fine);
                }
                if (lo > blo) blo = lo, bz = zc;
                if (done) break;
            }
            z = bz;
        }
    }
    const Vec co = mulv(T, z);
    TriWeight w;
    w.v = v;
    w.e = e;
    for (int m = 0; m < 13; ++m) {
        const int j = kStored[m][0], k = kStored[m][1];
        w.stored[m] = j == k ? co[mono(j, j)] : 0.5 * (co[mono(j, k)] + co[mono(k, j)]);
    }
    Grid g{};
    for (int m = 0; m < 13; ++m) g[kStored[m][0]][kStored[m][1]] = g[kStored[m][1]][kStored[m][0]] = w.stored[m];
    // extrema (weights.hpp:520-558), sup with the reference's 1e-9 margin
    double lo = INFINITY, hi = -INFINITY, hx = 0, hy = 0, lx = 0, ly = 0;
    const int N = 256;
    for (int i = 0; i <= N; ++i)
        for (int j = 0; i + j <= N; ++j) {
            const double x = double(i) / N, y2 = double(j) / N, val = horner(g, x, y2);
            if (val > hi) hi = val, hx = x, hy = y2;
            if (val < lo) lo = val, lx = x, ly = y2;
        }
    auto refine = [&](double x, double yy, double sign) {
        double best = sign * horner(g, x, yy), step = 1.0 / N;
        for (int it = 0; it < 60 && step >= 1e-12; ++it) {
            bool moved = false;
            const double cand2[4][2] = {{x + step, yy}, {x - step, yy}, {x, yy + step}, {x, yy - step}};
            for (const auto& c : cand2) {
                if (c[0] < 0 || c[1] < 0 || c[0] + c[1] > 1) continue;
                const double val = sign * horner(g, c[0], c[1]);
                if (val > best) best = val, x = c[0], yy = c[1], moved = true;
            }
            if (!moved) step *= 0.5;
        }
        return sign * best;
    };
    w.sup = refine(hx, hy, 1.0) + 1e-9;
    w.inf = refine(lx, ly, -1.0) - 1e-9;
    return w;
}

}  // namespace wh

static TriWeight tri_cached(int v, int e) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, TriWeight> memo;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = memo.find({v, e});
        if (it != memo.end()) return it->second;
    }
    TriWeight w = wh::build_tri(v, e);
    std::lock_guard<std::mutex> lk(mu);
    memo[{v, e}] = w;
    return w;
}

// closed-form edge polynomial and extrema (weights.hpp:46-76)
void edge_weight_poly(int n0, int n1, double a[5], double& sup, double& inf) {
    const double P = 1.0 / n1 - 1.0 / n0, Q = 1.0 - 1.0 / n0;
    a[0] = 1.0 / n0;
    a[1] = 0.0;
    a[2] = -5 * P + 16 * Q;
    a[3] = 14 * P - 32 * Q;
    a[4] = 16 * Q - 8 * P;
    auto val = [&](double t) { return a[0] + t * (a[1] + t * (a[2] + t * (a[3] + t * a[4]))); };
    sup = std::max(val(0.0), val(1.0));
    inf = std::min(val(0.0), val(1.0));
    const double qa = 4 * a[4], qb = 3 * a[3], qc = 2 * a[2];
    auto consider = [&](double t) {
        if (t > 0.0 && t < 1.0) {
            sup = std::max(sup, val(t));
            inf = std::min(inf, val(t));
        }
    };
    if (std::abs(qa) > 1e-300) {
        const double disc = qb * qb - 4 * qa * qc;
        if (disc >= 0) {
            consider((-qb + std::sqrt(disc)) / (2 * qa));
            consider((-qb - std::sqrt(disc)) / (2 * qa));
        }
    } else if (std::abs(qb) > 1e-300) {
        consider(-qc / qb);
    }
}
WeightTableHost weight_table_from_assignment(const WeightAssignment& wa) {
    WeightTableHost t;
    t.poly_index = wa.poly_index;
    for (const auto& [n0, n1] : wa.edge_keys) {
        double a[5], sup, inf;
        edge_weight_poly(n0, n1, a, sup, inf);
        t.edge_a.insert(t.edge_a.end(), a, a + 5);
        t.edge_sup.push_back(sup);
        t.edge_inf.push_back(inf);
        t.edge_val.push_back(n0);
        t.edge_val.push_back(n1);
        t.A = std::max(t.A, double(std::max(n0, n1)));
        t.sup = std::max(t.sup, sup);
    }
    for (const auto& [v, e] : wa.tri_keys) {
        t.tri.push_back(tri_cached(v, e));
        t.A = std::max(t.A, double(v));
        t.sup = std::max(t.sup, t.tri.back().sup);
    }
    return t;
}

static inline uint64_t ekey(int32_t a, int32_t b) {
    if (a > b) std::swap(a, b);
    return (uint64_t(uint32_t(a)) << 32) | uint32_t(b);
}

WeightTableHost build_weight_table(const std::vector<int32_t>& sv, const std::vector<uint8_t>& kind, int64_t V) {
    const int64_t N = int64_t(kind.size());
    std::vector<int32_t> val(size_t(V), 0);
    std::unordered_map<uint64_t, int32_t> ecount;
    ecount.reserve(size_t(N) * 2);
    for (int64_t i = 0; i < N; ++i) {
        const int nv = kind[i] + 1;
        const int32_t* s = &sv[3 * i];
        if (nv > 1)
            for (int a = 0; a < nv; ++a) val[s[a]]++;
        if (nv == 2) ecount[ekey(s[0], s[1])]++;
        if (nv == 3) {
            ecount[ekey(s[0], s[1])]++;
            ecount[ekey(s[1], s[2])]++;
            ecount[ekey(s[2], s[0])]++;
        }
    }
    auto ev = [&](int32_t a, int32_t b) {
        auto it = ecount.find(ekey(a, b));
        return it == ecount.end() ? 0 : it->second;
    };
    WeightTableHost t;
    t.poly_index.assign(size_t(N), -1);
    std::map<std::pair<int, int>, int32_t> ec, tc;
    for (int64_t i = 0; i < N; ++i) {
        const int32_t* s = &sv[3 * i];
        if (kind[i] == 1) {
            const int n0 = val[s[0]], n1 = val[s[1]];
            auto [it, fresh] = ec.try_emplace({n0, n1}, int32_t(t.edge_a.size() / 5));
            if (fresh) {
                double a[5], sup, inf;
                edge_weight_poly(n0, n1, a, sup, inf);
                t.edge_a.insert(t.edge_a.end(), a, a + 5);
                t.edge_sup.push_back(sup);
                t.edge_inf.push_back(inf);
                t.edge_val.push_back(n0);
                t.edge_val.push_back(n1);
            }
            t.poly_index[i] = it->second;
            t.A = std::max(t.A, double(std::max(n0, n1)));
            t.sup = std::max(t.sup, t.edge_sup[it->second]);
        } else if (kind[i] == 2) {
            const int v = std::max({val[s[0]], val[s[1]], val[s[2]]});
            const int e = std::max({ev(s[0], s[1]), ev(s[1], s[2]), ev(s[2], s[0])});
            auto [it, fresh] = tc.try_emplace({v, e}, int32_t(t.tri.size()));
            if (fresh) t.tri.push_back(tri_cached(v, e));
            t.poly_index[i] = it->second;
            t.A = std::max(t.A, double(v));
            t.sup = std::max(t.sup, t.tri[it->second].sup);
        }
    }
    return t;
}

}  // namespace sdgpu

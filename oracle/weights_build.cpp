// oracle/weights_build.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Restatement of the reference triangle weight-polynomial construction
// (weights.hpp:176-560) without Eigen. The reference's Eigen::JacobiSVD
// (weights.hpp:362) is replaced by a one-sided (Hestenes) Jacobi SVD
// written here; the null-space basis it returns differs from Eigen's in
// low bits, so polynomial coefficients can differ from the reference's at
// ~1e-12. GPU parity is therefore defined GIVEN a shared
// WeightSet table: the same table is fed to the oracle and the GPU.
// The construction is pinned by the reference's own weight tests
// (T/test_weights.cpp:56-96), restated in tests/test_oracle_golden.py.
#include "sdoracle.hpp"

#include <mutex>

namespace sdo {
namespace {

constexpr int kMono = 36;  // weights.hpp:82

// weights.hpp:84-87: row j starts at sum_{i<j} (8 - i)
constexpr int mono_index(int j, int k) { return j * 8 - j * (j - 1) / 2 + k; }

struct Mono { int j, k; };
// weights.hpp:92-101: j ascending, k ascending within j
const std::array<Mono, kMono>& monomials() {
    static const std::array<Mono, kMono> m = [] {
        std::array<Mono, kMono> out{};
        int n = 0;
        for (int j = 0; j <= 7; ++j)
            for (int k = 0; j + k <= 7; ++k) out[n++] = {j, k};
        return out;
    }();
    return m;
}

// Dense row-major matrix, just enough for a 36x36 problem.
struct Mat {
    int r = 0, c = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(int rows, int cols) : r(rows), c(cols), a(std::size_t(rows) * cols, 0.0) {}
    double& operator()(int i, int j) { return a[std::size_t(i) * c + j]; }
    double operator()(int i, int j) const { return a[std::size_t(i) * c + j]; }
};
using Vec = std::vector<double>;

Mat matmul(const Mat& x, const Mat& y) {
    Mat z(x.r, y.c);
    for (int i = 0; i < x.r; ++i)
        for (int k = 0; k < x.c; ++k) {
            const double xv = x(i, k);
            if (xv == 0.0) continue;
            for (int j = 0; j < y.c; ++j) z(i, j) += xv * y(k, j);
        }
    return z;
}
Vec matvec(const Mat& x, const Vec& v) {
    Vec out(x.r, 0.0);
    for (int i = 0; i < x.r; ++i) {
        double s = 0.0;
        for (int k = 0; k < x.c; ++k) s += x(i, k) * v[k];
        out[i] = s;
    }
    return out;
}

// weights.hpp:183-241 -- the 36-equation interpolation/boundary system.
void tri_weight_system(int v, int e, Mat& A, Vec& b) {
    A = Mat(36, kMono);
    b.assign(36, 0.0);
    int row = 0;
    auto point_row = [&](double x, double y, double target) {
        for (const Mono& m : monomials()) A(row, mono_index(m.j, m.k)) = std::pow(x, m.j) * std::pow(y, m.k);
        b[row++] = target;
    };
    const double vv = 1.0 / v, ee = 1.0 / e;
    point_row(0, 0, vv);
    point_row(1, 0, vv);
    point_row(0, 1, vv);
    point_row(1.0 / 3, 0, ee);
    point_row(2.0 / 3, 0, ee);
    point_row(0, 1.0 / 3, ee);
    point_row(0, 2.0 / 3, ee);
    point_row(1.0 / 3, 2.0 / 3, ee);
    point_row(2.0 / 3, 1.0 / 3, ee);
    point_row(1.0 / 3, 1.0 / 3, double(v - 1) / v);
    // zero normal derivative on x = 0 and y = 0: c_{1k} = c_{j1} = 0
    for (int k = 0; k <= 6; ++k) A(row++, mono_index(1, k)) = 1.0;
    for (int j = 0; j <= 6; ++j) {
        if (j == 1) continue;
        A(row++, mono_index(j, 1)) = 1.0;
    }
    auto binom = [](int n, int r) {
        double out = 1.0;
        for (int i = 0; i < r; ++i) out = out * (n - i) / (i + 1);
        return out;
    };
    // coefficient of t^m in (d/dx + d/dy) w~ on the hypotenuse
    auto diag_row = [&](int m, bool swapped) {
        for (const Mono& mono : monomials()) {
            const int j = mono.j, k = mono.k;
            double coef = 0.0;
            const int px[2] = {j - 1, j}, py[2] = {k, k - 1};
            const double tc[2] = {double(j), double(k)};
            for (int q = 0; q < 2; ++q) {
                if (tc[q] == 0.0) continue;
                const int tp = swapped ? py[q] : px[q];
                const int op = swapped ? px[q] : py[q];
                const int r = m - tp;
                if (r >= 0 && r <= op) coef += tc[q] * binom(op, r) * ((r % 2) ? -1.0 : 1.0);
            }
            A(row, mono_index(j, k)) += coef;
        }
        ++row;
    };
    for (int m = 0; m <= 6; ++m) diag_row(m, false);
    for (int m = 0; m <= 5; ++m) diag_row(m, true);
}

// weights.hpp:247-271 -- degree-7 Bernstein -> monomial change of basis.
const Mat& bernstein_basis() {
    static const Mat T = [] {
        auto fact = [](int n) { double f = 1.0; for (int i = 2; i <= n; ++i) f *= i; return f; };
        Mat M(kMono, kMono);
        for (const Mono& m : monomials()) {
            const int a = m.j, bb = m.k, c = 7 - a - bb;
            const int col = mono_index(a, bb);
            const double mult = fact(7) / (fact(a) * fact(bb) * fact(c));
            for (int p = 0; p <= c; ++p)
                for (int q = 0; p + q <= c; ++q) {
                    const double term = fact(c) / (fact(p) * fact(q) * fact(c - p - q));
                    const double sign = ((p + q) % 2) ? -1.0 : 1.0;
                    M(mono_index(a + p, bb + q), col) += mult * term * sign;
                }
        }
        return M;
    }();
    return T;
}

// One-sided Jacobi SVD: M = U diag(s) V^T with s sorted descending
// (stand-in for Eigen::JacobiSVD with ComputeFullU | ComputeFullV).
struct Svd {
    Mat U, V;
    Vec s;
};
Svd jacobi_svd(const Mat& M) {
    const int m = M.r, n = M.c;
    Mat W = M;
    Mat V(n, n);
    for (int i = 0; i < n; ++i) V(i, i) = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                double al = 0, be = 0, ga = 0;
                for (int i = 0; i < m; ++i) {
                    al += W(i, p) * W(i, p);
                    be += W(i, q) * W(i, q);
                    ga += W(i, p) * W(i, q);
                }
                if (ga == 0.0 || std::abs(ga) <= 1e-17 * std::sqrt(al * be)) continue;
                off = std::max(off, std::abs(ga) / std::sqrt(al * be));
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
                for (int i = 0; i < m; ++i) {
                    const double wp = W(i, p), wq = W(i, q);
                    W(i, p) = cs * wp - sn * wq;
                    W(i, q) = sn * wp + cs * wq;
                }
                for (int i = 0; i < n; ++i) {
                    const double vp = V(i, p), vq = V(i, q);
                    V(i, p) = cs * vp - sn * vq;
                    V(i, q) = sn * vp + cs * vq;
                }
            }
        if (off < 1e-15) break;
    }
    Vec sv(n);
    for (int j = 0; j < n; ++j) {
        double s2 = 0;
        for (int i = 0; i < m; ++i) s2 += W(i, j) * W(i, j);
        sv[j] = std::sqrt(s2);
    }
    std::vector<int> ord(n);
    for (int j = 0; j < n; ++j) ord[j] = j;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return sv[a] > sv[b]; });
    Svd out;
    out.U = Mat(m, n);
    out.V = Mat(n, n);
    out.s.resize(n);
    for (int jj = 0; jj < n; ++jj) {
        const int j = ord[jj];
        out.s[jj] = sv[j];
        for (int i = 0; i < m; ++i) out.U(i, jj) = sv[j] > 0 ? W(i, j) / sv[j] : 0.0;
        for (int i = 0; i < n; ++i) out.V(i, jj) = V(i, j);
    }
    return out;
}

// Pseudo-inverse solve with relative cutoff, as JacobiSVD::solve after
// setThreshold(thr): singular values below thr * s_max are dropped.
Vec svd_solve(const Svd& d, const Vec& b, double thr) {
    const int n = d.V.r;
    const double cut = std::max(d.s[0] * thr, std::numeric_limits<double>::min());
    Vec z(n, 0.0);
    for (int k = 0; k < int(d.s.size()); ++k) {
        if (d.s[k] < cut) break;
        double ub = 0;
        for (int i = 0; i < d.U.r; ++i) ub += d.U(i, k) * b[i];
        const double f = ub / d.s[k];
        for (int i = 0; i < n; ++i) z[i] += d.V(i, k) * f;
    }
    return z;
}

// weights.hpp:277-334 -- maximise t s.t. base_i + rows_i . gamma >= t by
// exhaustive enumeration of (r+1)-subsets of tight constraints.
Vec max_min_affine(const Mat& rows, const Vec& base) {
    const int m = int(base.size()), r = rows.c;
    Vec best(r, 0.0);
    if (r == 0 || m < r + 1) return best;
    double best_t = *std::min_element(base.begin(), base.end());
    const int n = r + 1;
    std::vector<int> pick(n);
    for (int i = 0; i < n; ++i) pick[i] = i;
    double M[5][6], u[5];
    while (true) {
        for (int s = 0; s < n; ++s) {
            for (int g = 0; g < r; ++g) M[s][g] = rows(pick[s], g);
            M[s][r] = -1.0;
            M[s][n] = -base[pick[s]];
        }
        bool ok = true;
        for (int col = 0; col < n && ok; ++col) {
            int piv = col;
            for (int s = col + 1; s < n; ++s)
                if (std::abs(M[s][col]) > std::abs(M[piv][col])) piv = s;
            if (std::abs(M[piv][col]) < 1e-12) { ok = false; break; }
            if (piv != col)
                for (int cc = 0; cc <= n; ++cc) std::swap(M[piv][cc], M[col][cc]);
            for (int s = 0; s < n; ++s) {
                if (s == col) continue;
                const double f = M[s][col] / M[col][col];
                for (int cc = col; cc <= n; ++cc) M[s][cc] -= f * M[col][cc];
            }
        }
        if (ok) {
            for (int s = 0; s < n; ++s) u[s] = M[s][n] / M[s][s];
            const double t = u[r];
            if (t > best_t) {
                bool feas = true;
                for (int i = 0; i < m && feas; ++i) {
                    double val = base[i];
                    for (int g = 0; g < r; ++g) val += rows(i, g) * u[g];
                    feas = val >= t - 1e-11;
                }
                if (feas) {
                    best_t = t;
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

Grid8 to_grid(const Vec& z) {  // Bernstein coefficients -> monomial grid
    Grid8 g{};
    const Vec mono = matvec(bernstein_basis(), z);
    for (const Mono& m : monomials()) g[m.j][m.k] = mono[mono_index(m.j, m.k)];
    return g;
}

// weights.hpp:401-430 -- sampled domain minimum + compass refinement.
double domain_min(const Grid8& g, int N, double& ax, double& ay) {
    double lo = INFINITY;
    for (int i = 0; i <= N; ++i)
        for (int j = 0; i + j <= N; ++j) {
            const double x = double(i) / N, y = double(j) / N;
            const double w = tri_horner(g, x, y);
            if (w < lo) { lo = w; ax = x; ay = y; }
        }
    const int M = 8 * N;
    for (int i = 0; i <= M; ++i) {
        const double t = 0.5 * i / M;
        const double w = tri_horner(g, t, t);
        if (w < lo) { lo = w; ax = t; ay = t; }
    }
    double step = 1.0 / N;
    while (step > 1e-13) {
        bool moved = false;
        const double cand[4][2] = {{ax + step, ay}, {ax - step, ay}, {ax, ay + step}, {ax, ay - step}};
        for (const auto& cp : cand) {
            if (cp[0] < 0 || cp[1] < 0 || cp[0] + cp[1] > 1) continue;
            const double w = tri_horner(g, cp[0], cp[1]);
            if (w < lo) { lo = w; ax = cp[0]; ay = cp[1]; moved = true; }
        }
        if (!moved) step *= 0.5;
    }
    return lo;
}

}  // namespace

// weights.hpp:352-560
TriPoly build_tri_weight(std::int32_t vertex_valence, std::int32_t edge_valence) {
    TriPoly p;
    p.vertex_valence = vertex_valence;
    p.edge_valence = edge_valence;
    Mat A;
    Vec b;
    tri_weight_system(vertex_valence, edge_valence, A, b);
    const Mat& T = bernstein_basis();
    const Svd svd = jacobi_svd(matmul(A, T));
    Vec z = svd_solve(svd, b, 1e-10);

    // symmetrised null-space directions (weights.hpp:369-380). The
    // reference Gram-Schmidts the symmetric parts of Eigen's null vectors in
    // column order with an absolute 1e-8 cut; in exact arithmetic that spans
    // exactly the swap-symmetric null space (dimension 3 here). Our Jacobi
    // null vectors carry ~1e-7 noise whose symmetric parts can survive a
    // 1e-8 cut in column-order Gram-Schmidt, so the same span is extracted
    // robustly: refine each symmetric part back into the null space, then
    // take an orthonormal basis of their span (SVD, same 1e-8 cut, <= 4).
    std::vector<Vec> null_dirs;
    {
        const double cut = svd.s[0] * 1e-10;
        const Mat AT = matmul(A, T);
        std::vector<Vec> sym;
        for (int i = 0; i < kMono; ++i) {
            if (svd.s[i] > cut) continue;
            Vec v(kMono);
            for (const Mono& m : monomials())
                v[mono_index(m.j, m.k)] = 0.5 * (svd.V(mono_index(m.j, m.k), i) + svd.V(mono_index(m.k, m.j), i));
            const Vec corr = svd_solve(svd, matvec(AT, v), 1e-10);  // row-space component
            for (int q = 0; q < kMono; ++q) v[q] -= corr[q];
            sym.push_back(v);
        }
        if (!sym.empty()) {
            Mat S(kMono, int(sym.size()));
            for (int g = 0; g < S.c; ++g)
                for (int q = 0; q < kMono; ++q) S(q, g) = sym[g][q];
            const Svd ss = jacobi_svd(S);
            for (int g = 0; g < S.c && int(null_dirs.size()) < 4; ++g) {
                if (ss.s[g] <= 1e-8) break;
                Vec d(kMono);
                for (int q = 0; q < kMono; ++q) d[q] = ss.U(q, g);
                null_dirs.push_back(d);
            }
        }
    }

    const int r = int(null_dirs.size());
    if (r > 0) {
        Mat coef_rows(kMono, r);
        for (int g = 0; g < r; ++g)
            for (int i = 0; i < kMono; ++i) coef_rows(i, g) = null_dirs[g][i];
        const Vec gamma = max_min_affine(coef_rows, z);

        for (int g = 0; g < r; ++g)
            for (int i = 0; i < kMono; ++i) z[i] += coef_rows(i, g) * gamma[g];

        double ax = 0, ay = 0;
        double lo = domain_min(to_grid(z), 384, ax, ay);
        // exchange rounds (weights.hpp:437-502)
        if (vertex_valence >= edge_valence && lo * vertex_valence < 1.0 - 1e-10) {
            std::vector<std::array<double, 2>> pts;
            for (int i = 0; i <= 4; ++i)
                for (int j = 0; i + j <= 4; ++j) pts.push_back({i / 4.0, j / 4.0});
            for (double h = 1e-2; h >= 1e-7; h *= 0.1) {
                pts.push_back({1.0 / 3 - h, 1.0 / 3 - h});
                pts.push_back({1.0 / 3 + h, 1.0 / 3 + h});
                pts.push_back({h, h});
                pts.push_back({0.5 - h, 0.5 - h});
            }
            const std::size_t num_seeds = pts.size();
            std::vector<Grid8> dir_grids;
            for (int g = 0; g < r; ++g) dir_grids.push_back(to_grid(null_dirs[g]));
            const Grid8 base_grid = to_grid(z);
            Vec best_z = z;
            double best_lo = lo;
            for (int round = 0; round < 80; ++round) {
                pts.push_back({ax, ay});
                Mat rows(int(pts.size()), r);
                Vec base(pts.size());
                for (std::size_t s = 0; s < pts.size(); ++s) {
                    base[s] = tri_horner(base_grid, pts[s][0], pts[s][1]);
                    for (int g = 0; g < r; ++g) rows(int(s), g) = tri_horner(dir_grids[g], pts[s][0], pts[s][1]);
                }
                const Vec dg = max_min_affine(rows, base);
                Vec vals(pts.size());
                double model = INFINITY;
                for (std::size_t s = 0; s < pts.size(); ++s) {
                    double v = base[s];
                    for (int g = 0; g < r; ++g) v += rows(int(s), g) * dg[g];
                    vals[s] = v;
                    model = std::min(model, v);
                }
                if (pts.size() > 60) {
                    std::vector<std::array<double, 2>> kept(pts.begin(), pts.begin() + num_seeds);
                    for (std::size_t s = num_seeds; s < pts.size(); ++s)
                        if (vals[s] - model < 1e-9 || s + 12 >= pts.size()) kept.push_back(pts[s]);
                    pts.swap(kept);
                }
                Vec zc = z;
                for (int g = 0; g < r; ++g)
                    for (int i = 0; i < kMono; ++i) zc[i] += dg[g] * null_dirs[g][i];
                lo = domain_min(to_grid(zc), 384, ax, ay);
                bool done = lo * vertex_valence >= 1.0 - 1e-12 || model - lo < 1e-13;
                if (done) {
                    double vx = 0, vy = 0;
                    const double fine = domain_min(to_grid(zc), 1536, vx, vy);
                    if (fine < lo - 1e-13) {
                        lo = fine; ax = vx; ay = vy;
                        done = false;
                    } else {
                        lo = std::min(lo, fine);
                    }
                }
                if (lo > best_lo) { best_lo = lo; best_z = zc; }
                if (done) break;
            }
            z = best_z;
        }
    }
    const Vec coeffs = matvec(T, z);
    for (int m = 0; m < 13; ++m) {
        const int j = kTriStored[m][0], k = kTriStored[m][1];
        p.stored[m] = j == k ? coeffs[mono_index(j, j)]
                             : 0.5 * (coeffs[mono_index(j, k)] + coeffs[mono_index(k, j)]);
    }
    p.expand();

    Vec snapped(kMono);
    for (const Mono& m : monomials()) snapped[mono_index(m.j, m.k)] = p.c[m.j][m.k];
    const Vec res = matvec(A, snapped);
    p.residual = 0.0;
    for (int i = 0; i < 36; ++i) p.residual = std::max(p.residual, std::abs(res[i] - b[i]));

    // extrema: dense grid + pattern refinement, 1e-9 safety (weights.hpp:520-558)
    double lo = INFINITY, hi = -INFINITY, hx = 0, hy = 0, lx = 0, ly = 0;
    constexpr int N = 256;
    for (int i = 0; i <= N; ++i)
        for (int j = 0; i + j <= N; ++j) {
            const double x = double(i) / N, y = double(j) / N;
            const double w = p.value(x, y);
            if (w > hi) { hi = w; hx = x; hy = y; }
            if (w < lo) { lo = w; lx = x; ly = y; }
        }
    auto refine = [&](double x, double y, double sign) {
        double best = sign * p.value(x, y);
        double step = 1.0 / N;
        for (int it = 0; it < 60; ++it) {
            bool moved = false;
            const double cand[4][2] = {{x + step, y}, {x - step, y}, {x, y + step}, {x, y - step}};
            for (const auto& cp : cand) {
                if (cp[0] < 0 || cp[1] < 0 || cp[0] + cp[1] > 1) continue;
                const double w = sign * p.value(cp[0], cp[1]);
                if (w > best) { best = w; x = cp[0]; y = cp[1]; moved = true; }
            }
            if (!moved) step *= 0.5;
            if (step < 1e-12) break;
        }
        return sign * best;
    };
    p.sup = refine(hx, hy, +1.0) + 1e-9;
    p.inf = refine(lx, ly, -1.0) - 1e-9;
    return p;
}

TriPoly cached_tri_weight(std::int32_t v, std::int32_t e) {
    static std::mutex mu;
    static std::map<std::pair<std::int32_t, std::int32_t>, TriPoly> memo;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = memo.find({v, e});
        if (it != memo.end()) return it->second;
    }
    TriPoly p = build_tri_weight(v, e);
    std::lock_guard<std::mutex> lk(mu);
    memo.emplace(std::make_pair(v, e), p);
    return p;
}

}  // namespace sdo

// pair.cuh -- one (query point, primitive) term of the smooth-distance sum,
// branch-light, in registers. Shared by the exact kernel (K1) and the exact
// leaves of the tree traversal (K3).
//
// Reference semantics restated (file:line in /root/reference/proj/include/smoothdist):
//   closest point        exact.hpp:68-106 (segment clamp, Ericson regions)
//   distance / gradient  exact.hpp:59-63  (grad = 0 at contact)
//   weight               weights.hpp:624-666 (w = (A w~)^S, floor 1e-300)
//   weight gradient      weights.hpp:675-697 (alpha-scaled shape gradients)
//   term                 smooth.hpp:51-61 (arg = -alpha d, coef = w,
//                        gcoef = w grad d - grad w / alpha)
//   underflow mask       smooth.hpp:85-88 (terms with -alpha d < -708 are 0)
//
// Every term enters the accumulator as
//   e      = 2^(x - m),   x = log2(w) + log2(e) (-alpha d)  (masked: e = 0)
//   s     += e
//   g     += (e r) delta - (e k) (shape-gradient combination)
// with r = 1/d, delta = q - closest point, and k = S A / (alpha^2 base),
// base = A w~ (so that e k dw~ is exp(-alpha d) dw / alpha^2 scaled).
// The host pre-scales the polynomial coefficients: the value rows by A
// (they evaluate base = A w~ directly) and the derivative rows by
// S A / alpha^2 (they evaluate the numerator of k).
#pragma once

#include "device_common.cuh"

namespace sdgpu {

template <class T>
struct Phys {
    T kappa;     // -alpha * log2(e)
    T dmax;      // 708 / alpha: terms with d > dmax are masked
    T S;         // attenuation alpha / max(alpha, alpha_u)
    T A;         // WeightSet::A
    T lw_unit;   // S log2(A): log2 weight of unit-weight primitives
    T lw_floor;  // S log2(1e-300): floored weight (weights.hpp:657-661)
    T w_ff;      // (A sup w~)^S, far-field weight (weights.hpp:576-578)
    T beta;      // Barnes-Hut threshold
};

// Polynomial coefficients of one weight polynomial, in evaluation order,
// pre-scaled as described above (value rows x A, derivative rows x S A / alpha^2).
//   edge: [0..4] = A a0..a4; [5..8] = K (a1, 2 a2, 3 a3, 4 a4)
//   tri : [0..22]  value rows  j=0:k{0,2..7} j=2:k{0,2..5} j=3:k{0,2..4}
//                  j=4:k{0,2,3} j=5:k{0,2} j=6:k{0} j=7:k{0}      (x A)
//         [23..38] d/dx rows (j c_jk)  j=2..7 with the same k sets (x K)
//         [39..54] d/dy rows (k c_jk)  j=0:k{2..7} j=2:k{2..5} j=3:k{2..4}
//                  j=4:k{2,3} j=5:k{2}                               (x K)
// with K = S A / alpha^2; c_{1k} = c_{j1} = 0 exactly (weights.hpp:113-131).
//   tri (s, p) form actually used (api.cu make_poly): w~ is symmetric, so
//         it is a polynomial in s = x + y, p = x y with 20 terms:
//         [0..19]  A_j(s) rows, j = 0..3, degrees 7, 5, 3, 1      (x A)
//         [20..35] B_j(s) = dA_j/ds rows, degrees 6, 4, 2, 0      (x K)
//         [36..38] K / A, 2 K / A, 3 K / A
constexpr int kPolyCoefs = 55;
constexpr int kTriSPCoefs = 39;
template <class T>
struct Poly {
    T c[kPolyCoefs];
};

// Smallest positive argument handed to rsqrt: keeps 0 * rsqrt finite at
// contact (distance 0 -> gradient 0, exact.hpp:62) without a select.
template <class T> struct Tiny;
template <> struct Tiny<float> { static constexpr float v = 1e-30f; };
template <> struct Tiny<double> { static constexpr double v = 1e-300; };

// ------------------------------------------------------- accumulator
// xm = x - m of a term (-inf when masked). When the term exceeds the shift
// (rare after the first records), the shift is re-anchored on the term's
// absolute exponent x, recomputed by `absx` from registers, so that the
// stored m and every later x - m are formed from the same rounded values
// (an uninitialised shift is -inf: its sums scale by 2^-inf = 0).
template <class T, class F>
__device__ __forceinline__ T bump(Acc<T>& acc, T xm, F&& absx) {
    if (xm > T(0)) {
        const T x = absx();
        const T mn = x + T(kHeadroom);
        acc.scale(Math<T>::ex2(acc.m - mn));
        acc.m = mn;
        xm = x - mn;
    }
    return xm;
}

// (unordered compare: a distance that overflowed the compute type -- s = inf,
// d = inf * 0 = NaN, queries beyond ~1e19 in fp32 -- is masked like the
// huge distance it stands for)
template <class T>
__device__ __forceinline__ T masked(const Phys<T>& ph, T d, T xm) {
    return !(d <= ph.dmax) ? T(-INFINITY) : xm;
}

// Exponent (x - m) and gradient factor k = dnum / base of a polynomial
// primitive, with the reference floor (base <= 1e-300 -> w = 1e-300^S,
// dw = 0, weights.hpp:657-661) unless the polynomial is certified positive
// on its domain (SAFE, see api.cu), where the selects are dropped.
template <class T, bool SAFE>
__device__ __forceinline__ T weight_exponent(const Phys<T>& ph, T base, T dnum, T xd, T& k, T& lw) {
    const T lg = Math<T>::lg2(base);
    const T ib = Math<T>::rcp(base);
    if constexpr (SAFE) {
        k = dnum * ib;
        lw = ph.S * lg;
        return fma(ph.S, lg, xd);
    } else {
        const bool ok = base > T(sizeof(T) == 4 ? 0.0 : 1e-300);
        k = ok ? dnum * ib : T(0);
        lw = ok ? ph.S * lg : ph.lw_floor;
        return lw + xd;
    }
}

template <class T>
__device__ __forceinline__ T clamp01(T x) {
    return fmin(fmax(x, T(0)), T(1));
}

// -------------------------------------------------------------- points
// acc.m is relative to lw_unit for the whole launch (see exact.cu), so the
// exponent is one FFMA.
template <class T>
__device__ __forceinline__ void point_term(const Phys<T>& ph, T qx, T qy, T qz, T ax, T ay, T az, Acc<T>& acc) {
    const T dx = qx - ax, dy = qy - ay, dz = qz - az;
    const T s = fma(dx, dx, fma(dy, dy, dz * dz));
    const T r = Math<T>::rsqrt(fmax(s, Tiny<T>::v));
    const T d = s * r;
    const T xm = bump(acc, masked(ph, d, fma(ph.kappa, d, -acc.m)), [&] { return ph.kappa * d; });
    const T e = Math<T>::ex2(xm);
    const T er = e * r;
    acc.s += e;
    acc.gx = fma(er, dx, acc.gx);
    acc.gy = fma(er, dy, acc.gy);
    acc.gz = fma(er, dz, acc.gz);
}

// --------------------------------------------------------------- edges
// rec: a.xyz e.xyz inv_e2 ge.xyz (ge = e / |e|^2)
template <class T, bool POLY, bool SAFE>
__device__ __forceinline__ void edge_term(const Phys<T>& ph, const Poly<T>& pc, T qx, T qy, T qz, const T* rec,
                                          Acc<T>& acc) {
    const T apx = qx - rec[0], apy = qy - rec[1], apz = qz - rec[2];
    const T ex = rec[3], ey = rec[4], ez = rec[5];
    const T t = clamp01(fma(ex, apx, fma(ey, apy, ez * apz)) * rec[6]);
    const T dx = fma(-t, ex, apx), dy = fma(-t, ey, apy), dz = fma(-t, ez, apz);
    const T s = fma(dx, dx, fma(dy, dy, dz * dz));
    const T r = Math<T>::rsqrt(fmax(s, Tiny<T>::v));
    const T d = s * r;
    if constexpr (POLY && SAFE) {
        // base > 0 certified: exponentiate e / base and recover e with one
        // multiply (e k = (e / base) dnum): no reciprocal
        const T base = fma(t, fma(t, fma(t, fma(t, pc.c[4], pc.c[3]), pc.c[2]), pc.c[1]), pc.c[0]);
        const T dnum = fma(t, fma(t, fma(t, pc.c[8], pc.c[7]), pc.c[6]), pc.c[5]);
        const T lg = Math<T>::lg2(base), lw = ph.S * lg;
        const T xm = bump(acc, masked(ph, d, fma(ph.kappa, d, lw - acc.m)), [&] { return fma(ph.kappa, d, lw); });
        const T eob = Math<T>::ex2(xm - lg);
        const T e = eob * base;
        const T er = e * r, ek = eob * dnum;
        acc.s += e;
        acc.gx = fma(-ek, rec[7], fma(er, dx, acc.gx));
        acc.gy = fma(-ek, rec[8], fma(er, dy, acc.gy));
        acc.gz = fma(-ek, rec[9], fma(er, dz, acc.gz));
    } else if constexpr (POLY) {
        const T base = fma(t, fma(t, fma(t, fma(t, pc.c[4], pc.c[3]), pc.c[2]), pc.c[1]), pc.c[0]);
        const T dnum = fma(t, fma(t, fma(t, pc.c[8], pc.c[7]), pc.c[6]), pc.c[5]);
        T k, lw;
        const T xm = bump(acc, masked(ph, d, weight_exponent<T, SAFE>(ph, base, dnum, fma(ph.kappa, d, -acc.m), k, lw)),
                          [&] { return fma(ph.kappa, d, lw); });
        const T e = Math<T>::ex2(xm);
        const T er = e * r, ek = e * k;
        acc.s += e;
        acc.gx = fma(-ek, rec[7], fma(er, dx, acc.gx));
        acc.gy = fma(-ek, rec[8], fma(er, dy, acc.gy));
        acc.gz = fma(-ek, rec[9], fma(er, dz, acc.gz));
    } else {
        const T xm = bump(acc, masked(ph, d, fma(ph.kappa, d, -acc.m)), [&] { return ph.kappa * d; });
        const T e = Math<T>::ex2(xm);
        const T er = e * r;
        acc.s += e;
        acc.gx = fma(er, dx, acc.gx);
        acc.gy = fma(er, dy, acc.gy);
        acc.gz = fma(er, dz, acc.gz);
    }
}

// ----------------------------------------------------------- triangles
// Closest point by Ericson's Voronoi regions (exact.hpp:77-106) written as
// a select cascade on d1 = ab.ap, d2 = ac.ap: with A = |ab|^2, B = ab.ac,
// C = |ac|^2 the remaining dot products are d3 = d1 - A, d4 = d2 - B,
// d5 = d1 - B, d6 = d2 - C, and va + vb + vc = AC - B^2.
template <class T>
__device__ __forceinline__ void tri_closest(const T* rec, T d1, T d2, T& u, T& v, bool& inner) {
    const T A = rec[9], B = rec[10], C = rec[11];
    const T d3 = d1 - A, d4 = d2 - B, d5 = d1 - B, d6 = d2 - C;
    const T vc = fma(d1, d4, -d3 * d2);
    const T vb = fma(d5, d2, -d1 * d6);
    const T va = fma(d3, d6, -d5 * d4);
    const T e43 = d4 - d3, e56 = d5 - d6;
    u = vb * rec[15];  // interior
    v = vc * rec[15];
    const T t6 = e43 * rec[14];  // edge bc
    inner = true;
    if (va <= T(0) && e43 >= T(0) && e56 >= T(0)) { u = T(1) - t6; v = t6; inner = false; }
    if (vb <= T(0) && d2 >= T(0) && d6 <= T(0)) { u = T(0); v = d2 * rec[13]; inner = false; }  // edge ac
    if (vc <= T(0) && d1 >= T(0) && d3 <= T(0)) { u = d1 * rec[12]; v = T(0); inner = false; }  // edge ab
    if (d6 >= T(0) && d5 <= d6) { u = T(0); v = T(1); inner = false; }                         // vertex c
    if (d3 >= T(0) && d4 <= d3) { u = T(1); v = T(0); inner = false; }                         // vertex b
    if (d1 <= T(0) && d2 <= T(0)) { u = T(0); v = T(0); inner = false; }                       // vertex a
}

// Near-contact interior pairs in fp32 (the tree's exact leaves): q - p formed
// as ap - u ab - v ac cancels down to a few ulps of |ap|, so for a query
// within ~1e-8 of a face its direction -- the term's distance gradient
// (exact.hpp:59-63) -- is rounding noise, while the reference (fp64) still
// resolves it. Below d < |ab| / 128 the interior offset is taken as the
// orthogonal projection onto the face normal instead, m (m . ap) / |m|^2
// with m = G1 x G2 = n / |n|^2 (the record's shape gradients, exactly
// parallel to n): its direction is exact to fp32 rounding of m whatever d.
// Rare: cfg4's on-surface queries (d ~ 2e-9) had gradient errors up to
// 4.6e-4 without it (1e-6 relative at most with it, the whole batch).
// FIX: apply it (inline); otherwise *contact (if given) reports that it
// would apply, so a register-tight caller can redo the term with FIX on a
// rare, separate path (the cooperative leaf flush of K3Q).
template <class T, bool FIX>
__device__ __forceinline__ void tri_contact(const T* rec, bool inner, T apx, T apy, T apz, T& dx, T& dy, T& dz,
                                            T& s, bool* contact) {
    if constexpr (sizeof(T) == 4) {
        const bool c = inner && s < rec[9] * T(1.0 / 16384.0);
        if constexpr (FIX) {
            if (c) {
                const T mx = fma(rec[17], rec[21], -rec[18] * rec[20]);
                const T my = fma(rec[18], rec[19], -rec[16] * rec[21]);
                const T mz = fma(rec[16], rec[20], -rec[17] * rec[19]);
                const T t = fma(mx, apx, fma(my, apy, mz * apz)) / fma(mx, mx, fma(my, my, mz * mz));
                dx = t * mx;
                dy = t * my;
                dz = t * mz;
                s = fma(dx, dx, fma(dy, dy, dz * dz));
            }
        } else if (contact) {
            *contact = c;
        }
    }
}

// tri_contact's condition alone (the same operations as tri_term's
// closest point, so the same decision): K3C's cheap test before it
// re-evaluates a leaf term.
__device__ __forceinline__ bool tri_near_contact(const float* rec, float qx, float qy, float qz) {
    const float apx = qx - rec[0], apy = qy - rec[1], apz = qz - rec[2];
    const float d1 = fmaf(rec[3], apx, fmaf(rec[4], apy, rec[5] * apz));
    const float d2 = fmaf(rec[6], apx, fmaf(rec[7], apy, rec[8] * apz));
    float u, v;
    bool inner;
    tri_closest(rec, d1, d2, u, v, inner);
    const float dx = fmaf(-v, rec[6], fmaf(-u, rec[3], apx));
    const float dy = fmaf(-v, rec[7], fmaf(-u, rec[4], apy));
    const float dz = fmaf(-v, rec[8], fmaf(-u, rec[5], apz));
    const float s = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    return inner && s < rec[9] * (1.0f / 16384.0f);
}

// base = A w~ and the K-scaled barycentric gradient of w~ (see Poly), in
// the symmetric (s, p) form: W = A_0 + p (A_1 + p (A_2 + p A_3)),
// W_s = B_0 + p (B_1 + p (B_2 + p B_3)), W_p = A_1 + 2 p A_2 + 3 p^2 A_3,
// d/dx = W_s + y W_p, d/dy = W_s + x W_p.
template <class T>
__device__ __forceinline__ void tri_poly(const Poly<T>& pc, T x, T y, T& w, T& wx, T& wy) {
    const T* c = pc.c;
    const T s = x + y, p = x * y;
    const T A0 = fma(s, fma(s, fma(s, fma(s, fma(s, fma(s, fma(s, c[7], c[6]), c[5]), c[4]), c[3]), c[2]), c[1]), c[0]);
    const T A1 = fma(s, fma(s, fma(s, fma(s, fma(s, c[13], c[12]), c[11]), c[10]), c[9]), c[8]);
    const T A2 = fma(s, fma(s, fma(s, c[17], c[16]), c[15]), c[14]);
    const T A3 = fma(s, c[19], c[18]);
    w = fma(p, fma(p, fma(p, A3, A2), A1), A0);
    const T B0 = fma(s, fma(s, fma(s, fma(s, fma(s, fma(s, c[26], c[25]), c[24]), c[23]), c[22]), c[21]), c[20]);
    const T B1 = fma(s, fma(s, fma(s, fma(s, c[31], c[30]), c[29]), c[28]), c[27]);
    const T B2 = fma(s, fma(s, c[34], c[33]), c[32]);
    const T Ws = fma(p, fma(p, fma(p, c[35], B2), B1), B0);
    const T Wp = fma(p, fma(p, A3 * c[38], A2 * c[37]), A1 * c[36]);
    wx = fma(y, Wp, Ws);
    wy = fma(x, Wp, Ws);
}

// rec: see device_common.cuh (kRecTri)
template <class T, bool POLY, bool SAFE, bool FIX = false>
__device__ __forceinline__ void tri_term(const Phys<T>& ph, const Poly<T>& pc, T qx, T qy, T qz, const T* rec,
                                         Acc<T>& acc, bool* contact = nullptr) {
    const T apx = qx - rec[0], apy = qy - rec[1], apz = qz - rec[2];
    const T abx = rec[3], aby = rec[4], abz = rec[5];
    const T acx = rec[6], acy = rec[7], acz = rec[8];
    const T d1 = fma(abx, apx, fma(aby, apy, abz * apz));
    const T d2 = fma(acx, apx, fma(acy, apy, acz * apz));
    T u, v;
    bool inner;
    tri_closest(rec, d1, d2, u, v, inner);
    T dx = fma(-v, acx, fma(-u, abx, apx));
    T dy = fma(-v, acy, fma(-u, aby, apy));
    T dz = fma(-v, acz, fma(-u, abz, apz));
    T s = fma(dx, dx, fma(dy, dy, dz * dz));
    tri_contact<T, FIX>(rec, inner, apx, apy, apz, dx, dy, dz, s, contact);
    const T r = Math<T>::rsqrt(fmax(s, Tiny<T>::v));
    const T d = s * r;
    if constexpr (POLY && SAFE) {  // no reciprocal: see edge_term
        T base, wx, wy;
        tri_poly(pc, u, v, base, wx, wy);
        const T lg = Math<T>::lg2(base), lw = ph.S * lg;
        const T xm = bump(acc, masked(ph, d, fma(ph.kappa, d, lw - acc.m)), [&] { return fma(ph.kappa, d, lw); });
        const T eob = Math<T>::ex2(xm - lg);
        const T e = eob * base;
        const T er = e * r;
        const T kx = eob * wx, ky = eob * wy;
        acc.s += e;
        acc.gx = fma(-ky, rec[19], fma(-kx, rec[16], fma(er, dx, acc.gx)));
        acc.gy = fma(-ky, rec[20], fma(-kx, rec[17], fma(er, dy, acc.gy)));
        acc.gz = fma(-ky, rec[21], fma(-kx, rec[18], fma(er, dz, acc.gz)));
    } else if constexpr (POLY) {
        T base, wx, wy;
        tri_poly(pc, u, v, base, wx, wy);
        T k, lw;
        const T xm = bump(acc, masked(ph, d, weight_exponent<T, SAFE>(ph, base, T(1), fma(ph.kappa, d, -acc.m), k, lw)),
                          [&] { return fma(ph.kappa, d, lw); });
        const T e = Math<T>::ex2(xm);
        const T er = e * r, ek = e * k;
        const T kx = ek * wx, ky = ek * wy;
        acc.s += e;
        acc.gx = fma(-ky, rec[19], fma(-kx, rec[16], fma(er, dx, acc.gx)));
        acc.gy = fma(-ky, rec[20], fma(-kx, rec[17], fma(er, dy, acc.gy)));
        acc.gz = fma(-ky, rec[21], fma(-kx, rec[18], fma(er, dz, acc.gz)));
    } else {
        const T xm = bump(acc, masked(ph, d, fma(ph.kappa, d, -acc.m)), [&] { return ph.kappa * d; });
        const T e = Math<T>::ex2(xm);
        const T er = e * r;
        acc.s += e;
        acc.gx = fma(er, dx, acc.gx);
        acc.gy = fma(er, dy, acc.gy);
        acc.gz = fma(er, dz, acc.gz);
    }
}

}  // namespace sdgpu

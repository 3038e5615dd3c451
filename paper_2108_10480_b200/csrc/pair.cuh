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
// Each term is handed to Acc::add as x = log2(w) + log2(e) * (-alpha d) and
// h = gcoef / w = grad d - (S A / (alpha^2 base)) * (dw~ . shape gradients).
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
    T kgrad;     // S A / alpha^2
    T w_ff;      // (A sup w~)^S, far-field weight (weights.hpp:576-578)
    T beta;      // Barnes-Hut threshold
};

// Polynomial coefficients of one weight polynomial, in evaluation order.
//   edge: [0..4]=a0..a4 [5]=a1 [6]=2a2 [7]=3a3 [8]=4a4  (a1 is 0 for every
//         polynomial build_edge_weight makes, but tables may carry any a1)
//   tri : [0..22]  value rows  j=0:k{0,2..7} j=2:k{0,2..5} j=3:k{0,2..4}
//                  j=4:k{0,2,3} j=5:k{0,2} j=6:k{0} j=7:k{0}
//         [23..38] d/dx rows (j c_jk)  j=2..7 with the same k sets
//         [39..54] d/dy rows (k c_jk)  j=0:k{2..7} j=2:k{2..5} j=3:k{2..4}
//                  j=4:k{2,3} j=5:k{2}
// c_{1k} = c_{j1} = 0 exactly (weights.hpp:113-131), so rows skip k = 1.
constexpr int kPolyCoefs = 55;
template <class T>
struct Poly {
    T c[kPolyCoefs];
};

template <class T>
__device__ __forceinline__ T clamp01(T x) {
    return fmin(fmax(x, T(0)), T(1));
}

template <class T>
__device__ __forceinline__ T masked_exponent(const Phys<T>& ph, T d, T lw) {
    return d > ph.dmax ? T(-INFINITY) : fma(ph.kappa, d, lw);
}

// -------------------------------------------------------------- points
template <class T>
__device__ __forceinline__ void point_term(const Phys<T>& ph, T qx, T qy, T qz, T ax, T ay, T az, Acc<T>& acc) {
    const T dx = qx - ax, dy = qy - ay, dz = qz - az;
    const T s = fma(dx, dx, fma(dy, dy, dz * dz));
    const T r = s > T(0) ? Math<T>::rsqrt(s) : T(0);
    const T d = s * r;
    acc.add(masked_exponent(ph, d, ph.lw_unit), dx * r, dy * r, dz * r);
}

// --------------------------------------------------------------- edges
// rec: a.xyz e.xyz inv_e2 ge.xyz
template <class T, bool POLY>
__device__ __forceinline__ void edge_term(const Phys<T>& ph, const Poly<T>& pc, T qx, T qy, T qz, const T* rec,
                                          Acc<T>& acc) {
    const T apx = qx - rec[0], apy = qy - rec[1], apz = qz - rec[2];
    const T ex = rec[3], ey = rec[4], ez = rec[5];
    const T t = clamp01(fma(ex, apx, fma(ey, apy, ez * apz)) * rec[6]);
    const T dx = fma(-t, ex, apx), dy = fma(-t, ey, apy), dz = fma(-t, ez, apz);
    const T s = fma(dx, dx, fma(dy, dy, dz * dz));
    const T r = s > T(0) ? Math<T>::rsqrt(s) : T(0);
    const T d = s * r;
    T hx = dx * r, hy = dy * r, hz = dz * r;
    T lw = ph.lw_unit;
    if constexpr (POLY) {
        const T wt = fma(t, fma(t, fma(t, fma(t, pc.c[4], pc.c[3]), pc.c[2]), pc.c[1]), pc.c[0]);
        const T wd = fma(t, fma(t, fma(t, pc.c[8], pc.c[7]), pc.c[6]), pc.c[5]);
        const T base = ph.A * wt;
        const bool ok = base > T(sizeof(T) == 4 ? 0.0 : 1e-300);
        lw = ok ? ph.S * Math<T>::lg2(base) : ph.lw_floor;
        const T k = ok ? ph.kgrad * Math<T>::rcp(base) * wd : T(0);
        hx = fma(-k, rec[7], hx);
        hy = fma(-k, rec[8], hy);
        hz = fma(-k, rec[9], hz);
    }
    acc.add(masked_exponent(ph, d, lw), hx, hy, hz);
}

// ----------------------------------------------------------- triangles
// Closest point by Ericson's Voronoi regions (exact.hpp:77-106) written as
// a select cascade on d1 = ab.ap, d2 = ac.ap: with A = |ab|^2, B = ab.ac,
// C = |ac|^2 the remaining dot products are d3 = d1 - A, d4 = d2 - B,
// d5 = d1 - B, d6 = d2 - C, and va + vb + vc = AC - B^2.
template <class T>
__device__ __forceinline__ void tri_closest(const T* rec, T d1, T d2, T& u, T& v) {
    const T A = rec[9], B = rec[10], C = rec[11];
    const T d3 = d1 - A, d4 = d2 - B, d5 = d1 - B, d6 = d2 - C;
    const T vc = fma(d1, d4, -d3 * d2);
    const T vb = fma(d5, d2, -d1 * d6);
    const T va = fma(d3, d6, -d5 * d4);
    const T e43 = d4 - d3, e56 = d5 - d6;
    u = vb * rec[15];  // interior
    v = vc * rec[15];
    const T t6 = e43 * rec[14];  // edge bc
    if (va <= T(0) && e43 >= T(0) && e56 >= T(0)) { u = T(1) - t6; v = t6; }
    if (vb <= T(0) && d2 >= T(0) && d6 <= T(0)) { u = T(0); v = d2 * rec[13]; }  // edge ac
    if (vc <= T(0) && d1 >= T(0) && d3 <= T(0)) { u = d1 * rec[12]; v = T(0); }  // edge ab
    if (d6 >= T(0) && d5 <= d6) { u = T(0); v = T(1); }                         // vertex c
    if (d3 >= T(0) && d4 <= d3) { u = T(1); v = T(0); }                         // vertex b
    if (d1 <= T(0) && d2 <= T(0)) { u = T(0); v = T(0); }                       // vertex a
}

// w~ and its barycentric gradient for the degree-7 symmetric polynomial.
template <class T>
__device__ __forceinline__ void tri_poly(const Poly<T>& p, T x, T y, T& w, T& wx, T& wy) {
    const T* c = p.c;
    const T y2 = y * y, x2 = x * x;
    // value rows P_j(y) = c_j0 + y^2 (c_j2 + y (c_j3 + ...))
    const T P0 = fma(y2, fma(y, fma(y, fma(y, fma(y, fma(y, c[6], c[5]), c[4]), c[3]), c[2]), c[1]), c[0]);
    const T P2 = fma(y2, fma(y, fma(y, fma(y, c[11], c[10]), c[9]), c[8]), c[7]);
    const T P3 = fma(y2, fma(y, fma(y, c[15], c[14]), c[13]), c[12]);
    const T P4 = fma(y2, fma(y, c[18], c[17]), c[16]);
    const T P5 = fma(y2, c[20], c[19]);
    const T P6 = c[21], P7 = c[22];
    w = fma(x2, fma(x, fma(x, fma(x, fma(x, fma(x, P7, P6), P5), P4), P3), P2), P0);
    // d/dx rows Q_j(y) (coefficients j c_jk)
    const T Q2 = fma(y2, fma(y, fma(y, fma(y, c[27], c[26]), c[25]), c[24]), c[23]);
    const T Q3 = fma(y2, fma(y, fma(y, c[31], c[30]), c[29]), c[28]);
    const T Q4 = fma(y2, fma(y, c[34], c[33]), c[32]);
    const T Q5 = fma(y2, c[36], c[35]);
    const T Q6 = c[37], Q7 = c[38];
    wx = x * fma(x, fma(x, fma(x, fma(x, fma(x, Q7, Q6), Q5), Q4), Q3), Q2);
    // d/dy rows R_j(y) (coefficients k c_jk, powers k - 1)
    const T R0 = y * fma(y, fma(y, fma(y, fma(y, fma(y, c[44], c[43]), c[42]), c[41]), c[40]), c[39]);
    const T R2 = y * fma(y, fma(y, fma(y, c[48], c[47]), c[46]), c[45]);
    const T R3 = y * fma(y, fma(y, c[51], c[50]), c[49]);
    const T R4 = y * fma(y, c[53], c[52]);
    const T R5 = y * c[54];
    wy = fma(x2, fma(x, fma(x, fma(x, R5, R4), R3), R2), R0);
}

// rec: see device_common.cuh (kRecTri)
template <class T, bool POLY>
__device__ __forceinline__ void tri_term(const Phys<T>& ph, const Poly<T>& pc, T qx, T qy, T qz, const T* rec,
                                         Acc<T>& acc) {
    const T apx = qx - rec[0], apy = qy - rec[1], apz = qz - rec[2];
    const T abx = rec[3], aby = rec[4], abz = rec[5];
    const T acx = rec[6], acy = rec[7], acz = rec[8];
    const T d1 = fma(abx, apx, fma(aby, apy, abz * apz));
    const T d2 = fma(acx, apx, fma(acy, apy, acz * apz));
    T u, v;
    tri_closest(rec, d1, d2, u, v);
    const T dx = fma(-v, acx, fma(-u, abx, apx));
    const T dy = fma(-v, acy, fma(-u, aby, apy));
    const T dz = fma(-v, acz, fma(-u, abz, apz));
    const T s = fma(dx, dx, fma(dy, dy, dz * dz));
    const T r = s > T(0) ? Math<T>::rsqrt(s) : T(0);
    const T d = s * r;
    T hx = dx * r, hy = dy * r, hz = dz * r;
    T lw = ph.lw_unit;
    if constexpr (POLY) {
        T wt, wx, wy;
        tri_poly(pc, u, v, wt, wx, wy);
        const T base = ph.A * wt;
        const bool ok = base > T(sizeof(T) == 4 ? 0.0 : 1e-300);
        lw = ok ? ph.S * Math<T>::lg2(base) : ph.lw_floor;
        const T k = ok ? ph.kgrad * Math<T>::rcp(base) : T(0);
        const T kx = k * wx, ky = k * wy;
        hx = fma(-kx, rec[16], fma(-ky, rec[19], hx));
        hy = fma(-kx, rec[17], fma(-ky, rec[20], hy));
        hz = fma(-kx, rec[18], fma(-ky, rec[21], hz));
    }
    acc.add(masked_exponent(ph, d, lw), hx, hy, hz);
}

}  // namespace sdgpu

// pair2.cuh -- fp32 pair terms for TWO queries at once with Blackwell's
// packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2, sm_100a). The two
// queries of a packed pair see the same staged primitive record, whose
// scalars enter the packed instructions as broadcast operands (SASS
// `R.F32`), so every add/mul/fma of pair.cuh costs half an issue slot;
// selects, clamps and MUFU stay scalar per query. Semantics are those of
// pair.cuh line for line (see there for the reference citations).
#pragma once

#include "pair.cuh"

namespace sdgpu {

struct f2 {
    unsigned long long v;
};
__device__ __forceinline__ f2 pack(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f2 bcast(float s) { return pack(s, s); }
__device__ __forceinline__ float lo(f2 a) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.v));
    return x;
}
__device__ __forceinline__ float hi(f2 a) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.v));
    return y;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
    f2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return d;
}
// scalar-broadcast forms (ptxas folds the pack into an `.F32` operand)
__device__ __forceinline__ f2 subs(f2 a, float s) { return sub2(a, bcast(s)); }
__device__ __forceinline__ f2 muls(f2 a, float s) { return mul2(a, bcast(s)); }
__device__ __forceinline__ f2 fmas(f2 a, float s, f2 c) { return fma2(a, bcast(s), c); }
__device__ __forceinline__ f2 sfma(float s, f2 b, f2 c) { return fma2(bcast(s), b, c); }

// Accumulator of two queries: shifts and fp32 tile sums, packed.
struct Acc2 {
    f2 m, s, gx, gy, gz;
    __device__ __forceinline__ void from(const Acc<float>& a, const Acc<float>& b) {
        m = pack(a.m, b.m);
        s = pack(a.s, b.s);
        gx = pack(a.gx, b.gx);
        gy = pack(a.gy, b.gy);
        gz = pack(a.gz, b.gz);
    }
    __device__ __forceinline__ void to(Acc<float>& a, Acc<float>& b) const {
        a.m = lo(m); a.s = lo(s); a.gx = lo(gx); a.gy = lo(gy); a.gz = lo(gz);
        b.m = hi(m); b.s = hi(s); b.gx = hi(gx); b.gy = hi(gy); b.gz = hi(gz);
    }
};

// Raise the shift of one half (rare path, scalar); x = absolute exponent.
__device__ __forceinline__ void bump_half(Acc2& a, int h, float x) {
    float m[2] = {lo(a.m), hi(a.m)}, s[2] = {lo(a.s), hi(a.s)}, gx[2] = {lo(a.gx), hi(a.gx)},
          gy[2] = {lo(a.gy), hi(a.gy)}, gz[2] = {lo(a.gz), hi(a.gz)};
    const float mn = x + kHeadroom;
    const float sc = Math<float>::ex2(m[h] - mn);
    s[h] *= sc; gx[h] *= sc; gy[h] *= sc; gz[h] *= sc;
    m[h] = mn;
    a.m = pack(m[0], m[1]); a.s = pack(s[0], s[1]);
    a.gx = pack(gx[0], gx[1]); a.gy = pack(gy[0], gy[1]); a.gz = pack(gz[0], gz[1]);
}

// Masks, re-anchors and exponentiates the packed x - m; `absx(h)` returns
// the absolute exponent of half h (only evaluated on the rare path).
// MODE 0: per-term -708 mask and lazy shift check (always correct);
// MODE 1: mask only -- the tile bound already raised the shift so that no
//         term of this tile exceeds 2^kTileHeadroom (exact.cu);
// MODE 2: neither -- additionally no term of this tile can be masked.
// With OFF, 2^(x - m - off) is returned (the mask and the shift check still
// act on x - m): the SAFE weighted terms exponentiate e / base and recover e
// with one multiply, instead of a reciprocal of base (one MUFU per pair less).
template <int MODE = 0, bool OFF = false, class F>
__device__ __forceinline__ f2 exp_terms(const Phys<float>& ph, Acc2& a, f2 d, f2 xm, F&& absx, f2 off = f2{0}) {
    if constexpr (MODE == 2) {
        if constexpr (OFF) xm = sub2(xm, off);
        return pack(Math<float>::ex2(lo(xm)), Math<float>::ex2(hi(xm)));
    }
    float x0 = lo(xm), x1 = hi(xm);
    x0 = !(lo(d) <= ph.dmax) ? -INFINITY : x0;  // NaN (overflowed) distances too
    x1 = !(hi(d) <= ph.dmax) ? -INFINITY : x1;
    if (MODE == 0 && (x0 > 0.f || x1 > 0.f)) {
        if (x0 > 0.f) {
            const float x = absx(0);
            bump_half(a, 0, x);
            x0 = x - lo(a.m);
        }
        if (x1 > 0.f) {
            const float x = absx(1);
            bump_half(a, 1, x);
            x1 = x - hi(a.m);
        }
    }
    if constexpr (OFF) {
        const f2 xo = sub2(pack(x0, x1), off);
        return pack(Math<float>::ex2(lo(xo)), Math<float>::ex2(hi(xo)));
    }
    return pack(Math<float>::ex2(x0), Math<float>::ex2(x1));
}

__device__ __forceinline__ f2 rsqrt2(f2 s) {
    return pack(Math<float>::rsqrt(fmaxf(lo(s), Tiny<float>::v)), Math<float>::rsqrt(fmaxf(hi(s), Tiny<float>::v)));
}

// ------------------------------------------------------------- points
template <int MODE = 0>
__device__ __forceinline__ void point_term2(const Phys<float>& ph, f2 qx, f2 qy, f2 qz, const float* rec, Acc2& a) {
    const f2 dx = subs(qx, rec[0]), dy = subs(qy, rec[1]), dz = subs(qz, rec[2]);
    const f2 s = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    const f2 r = rsqrt2(s);
    const f2 d = mul2(s, r);
    const f2 xm = sub2(muls(d, ph.kappa), a.m);
    const f2 e = exp_terms<MODE>(ph, a, d, xm, [&](int h) { return ph.kappa * (h ? hi(d) : lo(d)); });
    const f2 er = mul2(e, r);
    a.s = add2(a.s, e);
    a.gx = fma2(er, dx, a.gx);
    a.gy = fma2(er, dy, a.gy);
    a.gz = fma2(er, dz, a.gz);
}

// -------------------------------------------------------------- edges
template <bool POLY, bool SAFE, int MODE = 0>
__device__ __forceinline__ void edge_term2(const Phys<float>& ph, const Poly<float>& pc, f2 qx, f2 qy, f2 qz,
                                           const float* rec, Acc2& a) {
    const f2 apx = subs(qx, rec[0]), apy = subs(qy, rec[1]), apz = subs(qz, rec[2]);
    const f2 dot = fmas(apx, rec[3], fmas(apy, rec[4], muls(apz, rec[5])));
    const f2 t = pack(__saturatef(lo(dot) * rec[6]), __saturatef(hi(dot) * rec[6]));
    const f2 dx = fmas(t, -rec[3], apx), dy = fmas(t, -rec[4], apy), dz = fmas(t, -rec[5], apz);
    const f2 s = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    const f2 r = rsqrt2(s);
    const f2 d = mul2(s, r);
    const f2 xd = sub2(muls(d, ph.kappa), a.m);  // kappa d - m
    if constexpr (POLY && SAFE) {
        // base > 0 certified: e / base = 2^(S lg2 base + xd - lg2 base), e = (e / base) base,
        // e k = (e / base) dnum -- no reciprocal
        const f2 base = fmas(t, pc.c[4], bcast(pc.c[3]));
        const f2 base2 = fma2(t, fma2(t, fma2(t, base, bcast(pc.c[2])), bcast(pc.c[1])), bcast(pc.c[0]));
        const f2 dn = fma2(t, fma2(t, fmas(t, pc.c[8], bcast(pc.c[7])), bcast(pc.c[6])), bcast(pc.c[5]));
        const f2 l = pack(Math<float>::lg2(lo(base2)), Math<float>::lg2(hi(base2)));
        f2 eob;
        if constexpr (MODE == 2) {
            const f2 xb = fmas(l, ph.S - 1.f, xd);
            eob = pack(Math<float>::ex2(lo(xb)), Math<float>::ex2(hi(xb)));
        } else {
            const f2 lw = muls(l, ph.S);
            eob = exp_terms<MODE, true>(ph, a, d, add2(lw, xd),
                                        [&](int h) { return fmaf(ph.kappa, h ? hi(d) : lo(d), h ? hi(lw) : lo(lw)); },
                                        l);
        }
        const f2 e = mul2(eob, base2);
        const f2 er = mul2(e, r), ek = mul2(eob, dn);
        a.s = add2(a.s, e);
        a.gx = fmas(ek, -rec[7], fma2(er, dx, a.gx));
        a.gy = fmas(ek, -rec[8], fma2(er, dy, a.gy));
        a.gz = fmas(ek, -rec[9], fma2(er, dz, a.gz));
    } else if constexpr (POLY) {
        const f2 base = fmas(t, pc.c[4], bcast(pc.c[3]));
        const f2 base2 = fma2(t, fma2(t, fma2(t, base, bcast(pc.c[2])), bcast(pc.c[1])), bcast(pc.c[0]));
        const f2 dn = fma2(t, fma2(t, fmas(t, pc.c[8], bcast(pc.c[7])), bcast(pc.c[6])), bcast(pc.c[5]));
        const float l0 = Math<float>::lg2(lo(base2)), l1 = Math<float>::lg2(hi(base2));
        const float i0 = Math<float>::rcp(lo(base2)), i1 = Math<float>::rcp(hi(base2));
        f2 lw, k = mul2(dn, pack(i0, i1));
        if constexpr (SAFE) {
            lw = muls(pack(l0, l1), ph.S);
        } else {
            const bool ok0 = lo(base2) > 0.f, ok1 = hi(base2) > 0.f;
            lw = pack(ok0 ? ph.S * l0 : ph.lw_floor, ok1 ? ph.S * l1 : ph.lw_floor);
            k = pack(ok0 ? lo(k) : 0.f, ok1 ? hi(k) : 0.f);
        }
        const f2 e = exp_terms<MODE>(ph, a, d, add2(lw, xd),
                               [&](int h) { return fmaf(ph.kappa, h ? hi(d) : lo(d), h ? hi(lw) : lo(lw)); });
        const f2 er = mul2(e, r), ek = mul2(e, k);
        a.s = add2(a.s, e);
        a.gx = fmas(ek, -rec[7], fma2(er, dx, a.gx));
        a.gy = fmas(ek, -rec[8], fma2(er, dy, a.gy));
        a.gz = fmas(ek, -rec[9], fma2(er, dz, a.gz));
    } else {
        const f2 e = exp_terms<MODE>(ph, a, d, xd, [&](int h) { return ph.kappa * (h ? hi(d) : lo(d)); });
        const f2 er = mul2(e, r);
        a.s = add2(a.s, e);
        a.gx = fma2(er, dx, a.gx);
        a.gy = fma2(er, dy, a.gy);
        a.gz = fma2(er, dz, a.gz);
    }
}

// ----------------------------------------------------------- triangles
__device__ __forceinline__ f2 hz(f2 x, f2 acc, float c) { return fma2(x, acc, bcast(c)); }  // x acc + c

// packed tri_poly (pair.cuh): base = A w~ and K-scaled d/dx, d/dy in the
// symmetric (s, p) form
__device__ __forceinline__ void tri_poly2(const Poly<float>& pc, f2 x, f2 y, f2& w, f2& wx, f2& wy) {
    const float* c = pc.c;
    const f2 s = add2(x, y), p = mul2(x, y);
    const f2 A0 = hz(s, hz(s, hz(s, hz(s, hz(s, hz(s, fmas(s, c[7], bcast(c[6])), c[5]), c[4]), c[3]), c[2]), c[1]), c[0]);
    const f2 A1 = hz(s, hz(s, hz(s, hz(s, fmas(s, c[13], bcast(c[12])), c[11]), c[10]), c[9]), c[8]);
    const f2 A2 = hz(s, hz(s, fmas(s, c[17], bcast(c[16])), c[15]), c[14]);
    const f2 A3 = fmas(s, c[19], bcast(c[18]));
    w = fma2(p, fma2(p, fma2(p, A3, A2), A1), A0);
    const f2 B0 = hz(s, hz(s, hz(s, hz(s, hz(s, fmas(s, c[26], bcast(c[25])), c[24]), c[23]), c[22]), c[21]), c[20]);
    const f2 B1 = hz(s, hz(s, hz(s, fmas(s, c[31], bcast(c[30])), c[29]), c[28]), c[27]);
    const f2 B2 = hz(s, fmas(s, c[34], bcast(c[33])), c[32]);
    const f2 Ws = fma2(p, fma2(p, fmas(p, c[35], B2), B1), B0);
    const f2 Wp = fma2(p, fma2(p, muls(A3, c[38]), muls(A2, c[37])), muls(A1, c[36]));
    wx = fma2(y, Wp, Ws);
    wy = fma2(x, Wp, Ws);
}

// packed Ericson regions: the dot products and candidates are packed, the
// region selects are per query (pair.cuh tri_closest)
__device__ __forceinline__ void tri_closest2(const float* rec, f2 d1, f2 d2, f2& u, f2& v) {
    const float A = rec[9], B = rec[10], C = rec[11];
    const f2 d3 = subs(d1, A), d4 = subs(d2, B), d5 = subs(d1, B), d6 = subs(d2, C);
    const f2 vc = fma2(d1, d4, mul2(pack(-lo(d3), -hi(d3)), d2));
    const f2 vb = fma2(d5, d2, mul2(pack(-lo(d1), -hi(d1)), d6));
    const f2 va = fma2(d3, d6, mul2(pack(-lo(d5), -hi(d5)), d4));
    const f2 e43 = sub2(d4, d3), e56 = sub2(d5, d6);
    const f2 ui = muls(vb, rec[15]), vi = muls(vc, rec[15]);
    const f2 t6 = muls(e43, rec[14]);
    const f2 vac = muls(d2, rec[13]), uab = muls(d1, rec[12]);
    float uu[2], vv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        auto g = [h](f2 a) { return h ? hi(a) : lo(a); };
        float U = g(ui), V = g(vi);
        const float D1 = g(d1), D2 = g(d2), D3 = g(d3), D4 = g(d4), D5 = g(d5), D6 = g(d6);
        const float T6 = g(t6);
        if (g(va) <= 0.f && g(e43) >= 0.f && g(e56) >= 0.f) { U = 1.f - T6; V = T6; }
        if (g(vb) <= 0.f && D2 >= 0.f && D6 <= 0.f) { U = 0.f; V = g(vac); }
        if (g(vc) <= 0.f && D1 >= 0.f && D3 <= 0.f) { U = g(uab); V = 0.f; }
        if (D6 >= 0.f && D5 <= D6) { U = 0.f; V = 1.f; }
        if (D3 >= 0.f && D4 <= D3) { U = 1.f; V = 0.f; }
        if (D1 <= 0.f && D2 <= 0.f) { U = 0.f; V = 0.f; }
        uu[h] = U;
        vv[h] = V;
    }
    u = pack(uu[0], uu[1]);
    v = pack(vv[0], vv[1]);
}

template <bool POLY, bool SAFE, int MODE = 0>
__device__ __forceinline__ void tri_term2(const Phys<float>& ph, const Poly<float>& pc, f2 qx, f2 qy, f2 qz,
                                          const float* rec, Acc2& a) {
    const f2 apx = subs(qx, rec[0]), apy = subs(qy, rec[1]), apz = subs(qz, rec[2]);
    const f2 d1 = fmas(apx, rec[3], fmas(apy, rec[4], muls(apz, rec[5])));
    const f2 d2 = fmas(apx, rec[6], fmas(apy, rec[7], muls(apz, rec[8])));
    f2 u, v;
    tri_closest2(rec, d1, d2, u, v);
    const f2 dx = fmas(v, -rec[6], fmas(u, -rec[3], apx));
    const f2 dy = fmas(v, -rec[7], fmas(u, -rec[4], apy));
    const f2 dz = fmas(v, -rec[8], fmas(u, -rec[5], apz));
    const f2 s = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    const f2 r = rsqrt2(s);
    const f2 d = mul2(s, r);
    const f2 xd = sub2(muls(d, ph.kappa), a.m);
    if constexpr (POLY && SAFE) {  // no reciprocal: see edge_term2
        f2 base, wx, wy;
        tri_poly2(pc, u, v, base, wx, wy);
        const f2 l = pack(Math<float>::lg2(lo(base)), Math<float>::lg2(hi(base)));
        f2 eob;
        if constexpr (MODE == 2) {
            const f2 xb = fmas(l, ph.S - 1.f, xd);
            eob = pack(Math<float>::ex2(lo(xb)), Math<float>::ex2(hi(xb)));
        } else {
            const f2 lw = muls(l, ph.S);
            eob = exp_terms<MODE, true>(ph, a, d, add2(lw, xd),
                                        [&](int h) { return fmaf(ph.kappa, h ? hi(d) : lo(d), h ? hi(lw) : lo(lw)); },
                                        l);
        }
        const f2 e = mul2(eob, base);
        const f2 er = mul2(e, r);
        const f2 kx = mul2(eob, wx), ky = mul2(eob, wy);
        a.s = add2(a.s, e);
        a.gx = fmas(ky, -rec[19], fmas(kx, -rec[16], fma2(er, dx, a.gx)));
        a.gy = fmas(ky, -rec[20], fmas(kx, -rec[17], fma2(er, dy, a.gy)));
        a.gz = fmas(ky, -rec[21], fmas(kx, -rec[18], fma2(er, dz, a.gz)));
    } else if constexpr (POLY) {
        f2 base, wx, wy;
        tri_poly2(pc, u, v, base, wx, wy);
        const float l0 = Math<float>::lg2(lo(base)), l1 = Math<float>::lg2(hi(base));
        f2 k = pack(Math<float>::rcp(lo(base)), Math<float>::rcp(hi(base)));
        f2 lw;
        if constexpr (SAFE) {
            lw = muls(pack(l0, l1), ph.S);
        } else {
            const bool ok0 = lo(base) > 0.f, ok1 = hi(base) > 0.f;
            lw = pack(ok0 ? ph.S * l0 : ph.lw_floor, ok1 ? ph.S * l1 : ph.lw_floor);
            k = pack(ok0 ? lo(k) : 0.f, ok1 ? hi(k) : 0.f);
        }
        const f2 e = exp_terms<MODE>(ph, a, d, add2(lw, xd),
                               [&](int h) { return fmaf(ph.kappa, h ? hi(d) : lo(d), h ? hi(lw) : lo(lw)); });
        const f2 er = mul2(e, r), ek = mul2(e, k);
        const f2 kx = mul2(ek, wx), ky = mul2(ek, wy);
        a.s = add2(a.s, e);
        a.gx = fmas(ky, -rec[19], fmas(kx, -rec[16], fma2(er, dx, a.gx)));
        a.gy = fmas(ky, -rec[20], fmas(kx, -rec[17], fma2(er, dy, a.gy)));
        a.gz = fmas(ky, -rec[21], fmas(kx, -rec[18], fma2(er, dz, a.gz)));
    } else {
        const f2 e = exp_terms<MODE>(ph, a, d, xd, [&](int h) { return ph.kappa * (h ? hi(d) : lo(d)); });
        const f2 er = mul2(e, r);
        a.s = add2(a.s, e);
        a.gx = fma2(er, dx, a.gx);
        a.gy = fma2(er, dy, a.gy);
        a.gz = fma2(er, dz, a.gz);
    }
}

}  // namespace sdgpu

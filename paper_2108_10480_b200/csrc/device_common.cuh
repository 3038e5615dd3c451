// device_common.cuh -- sm_100a device helpers shared by the exact (K1),
// tree (K2/K3) and epilogue (K4) kernels: precision traits, the online
// max-shifted log2-domain accumulator, bulk-copy/mbarrier PTX wrappers and
// the per-primitive record layouts.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sdgpu {

// ----------------------------------------------------------- precision
// MUFU-backed approximations for fp32 (ex2/lg2/rsqrt/rcp.approx: <= 2 ulp),
// library double-precision routines for fp64.
template <class T> struct Math;
template <> struct Math<float> {
    static __device__ __forceinline__ float ex2(float x) {
        float y;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    static __device__ __forceinline__ float lg2(float x) {
        float y;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    static __device__ __forceinline__ float rsqrt(float x) {
        float y;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    static __device__ __forceinline__ float rcp(float x) {
        float y;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
};
// fp64: branch-free kernels on the DFMA pipe for the argument ranges the
// accumulator produces (the library routines carry special-case branches
// and slow-path calls that dominated the fp64 exact kernel). Accuracy
// ~1-2 ulp; coefficients from tools/fp64_poly_fit.py.
template <> struct Math<double> {
    // 2^x for x <= 1023; x < -1020 (incl. -inf, a masked term) gives 0 --
    // the sums only ever see x = exponent - running shift <= 0, where a
    // term below 2^-1020 of the largest one is below fp64 resolution.
    static __device__ __forceinline__ double ex2(double x) {
        const double big = 6755399441055744.0;  // 1.5 * 2^52: x + big rounds x to an integer
        const double t = x + big;
        const double f = x - (t - big);  // [-1/2, 1/2]
        double p = 4.4558179083360645e-10;
        p = fma(p, f, 7.074194297288521e-09);
        p = fma(p, f, 1.0178057087733941e-07);
        p = fma(p, f, 1.3215432535912375e-06);
        p = fma(p, f, 1.5252733841556773e-05);
        p = fma(p, f, 0.00015403530463724353);
        p = fma(p, f, 0.001333355814640647);
        p = fma(p, f, 0.009618129107587256);
        p = fma(p, f, 0.055504108664821625);
        p = fma(p, f, 0.24022650695910158);
        p = fma(p, f, 0.6931471805599453);
        p = fma(p, f, 1.0);
        const int n = __double2loint(t);  // the integer, two's complement in the low word
        const double r = __hiloint2double(__double2hiint(p) + (n << 20), __double2loint(p));
        return x < -1020.0 ? 0.0 : r;
    }
    // log2 x for positive normal x (callers select away other inputs):
    // x = 2^e m, m in [sqrt(1/2), sqrt2), log2 m = z g(z^2), z = (m-1)/(m+1).
    static __device__ __forceinline__ double lg2(double x) {
        int hi = __double2hiint(x);
        int e = (hi >> 20) - 1023;
        hi = (hi & 0x000fffff) | 0x3ff00000;
        const bool up = hi > 0x3ff6a09e;
        hi = up ? hi - 0x00100000 : hi;
        e = up ? e + 1 : e;
        const double m = __hiloint2double(hi, __double2loint(x));
        const double num = m - 1.0, den = m + 1.0;
        const double r = rcp(den);
        double z = num * r;
        z = fma(r, fma(-z, den, num), z);
        const double w = z * z;
        double g = 0.21365920165930558;
        g = fma(g, w, 0.22091306083083528);
        g = fma(g, w, 0.2623343533779628);
        g = fma(g, w, 0.3205985348978951);
        g = fma(g, w, 0.4121985858410509);
        g = fma(g, w, 0.5770780163455196);
        g = fma(g, w, 0.9617966939259898);
        g = fma(g, w, 2.8853900817779268);
        return fma(z, g, double(e));
    }
    // 1/sqrt(x) for positive normal x: MUFU seed + two Newton steps
    static __device__ __forceinline__ double rsqrt(double x) {
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        double e = fma(-(x * y), y, 1.0);
        y = fma(0.5 * y, e, y);
        e = fma(-(x * y), y, 1.0);
        return fma(0.5 * y, e, y);
    }
    // 1/x for finite nonzero normal x: MUFU seed + two Newton steps
    static __device__ __forceinline__ double rcp(double x) {
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        double e = fma(-x, r, 1.0);
        r = fma(r, e, r);
        e = fma(-x, r, 1.0);
        return fma(r, e, r);
    }
};

// Vector types used to read records out of shared memory (16 B loads).
template <class T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double2; };

// ------------------------------------------------ online accumulator
// Per-query partial of the reference sum c = sum_i w_i exp(-alpha d_i),
// grad_c = sum_i exp(-alpha d_i) (w_i grad d_i - grad w_i / alpha)
// (smooth.hpp:51-61, 79-93), kept as
//   c = s * 2^m,  grad_c = g * 2^m
// with the exponent x_i = log2(w_i exp(-alpha d_i)). The shift m is raised
// lazily (bump() in pair.cuh: only when a term exceeds it), by kHeadroom
// extra so that a slowly rising sequence does not rescale at every record;
// terms never exceed 2^0 relative to the shift, so nothing can overflow,
// and only terms below 2^-(126 - kHeadroom) of the running maximum flush
// (fp32).
constexpr float kHeadroom = 16.0f;

// Two-level sums: terms accumulate in T (Acc: s, g relative to the shift
// m) for at most one staged tile, then Tot::flush() folds them into fp64
// totals kept relative to their own anchor M, so the fp32 rounding error
// grows with the tile length (<= 768 terms), not with the number of
// primitives (up to 2^24). The pair (M, totals) is the per-query state
// carried between launches and merged by K4.
template <class T>
struct Acc {
    T m, s, gx, gy, gz;
    __device__ __forceinline__ void init() {
        m = T(-INFINITY);  // no term yet
        s = gx = gy = gz = T(0);
    }
    __device__ __forceinline__ void scale(T sc) {
        s *= sc; gx *= sc; gy *= sc; gz *= sc;
    }
};

struct Tot {
    double M;  // anchor (log2); -inf: empty
    double s, gx, gy, gz;
    __device__ __forceinline__ void init() {
        M = -INFINITY;
        s = gx = gy = gz = 0.0;
    }
    // adds acc's tile sums (relative to acc.m) and clears them
    template <class T>
    __device__ __forceinline__ void flush(Acc<T>& a) {
        if (a.s != T(0)) {
            const double m = double(a.m);
            if (m > M + 512.0 || M == -INFINITY) {  // (re-)anchor; rare
                const double f = M == -INFINITY ? 0.0 : exp2(M - m);
                s *= f; gx *= f; gy *= f; gz *= f;
                M = m;
            }
            const double f = exp2(m - M);
            s = fma(double(a.s), f, s);
            gx = fma(double(a.gx), f, gx);
            gy = fma(double(a.gy), f, gy);
            gz = fma(double(a.gz), f, gz);
        }
        a.s = a.gx = a.gy = a.gz = T(0);
    }
};

// ------------------------------------------------------- bulk copies
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
// TMA bulk (non-tensor) copy global -> shared, completion counted in bytes
// on the mbarrier. dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------ record layouts
// One record per primitive, in units of the compute type T, 16-B aligned.
// Geometry is stored relative to the first corner so the closest point is
// formed as delta = (q - a) - u ab - v ac (no absolute reconstruction; the
// fp32 error then scales with |q - a|, not with |q|).
//
// point    (4):  a.xyz, pad
// edge    (12):  a.xyz, e = b - a, 1/|e|^2, e/|e|^2, pad2
// triangle(24):  a.xyz, ab, ac, A=|ab|^2, B=ab.ac, C=|ac|^2, 1/A, 1/C,
//                1/|bc|^2, 1/(AC - B^2), G1, G2, pad2
//   with G1 = n x (a - c) / |n|^2, G2 = n x (b - a) / |n|^2, n = ab x ac,
//   the (alpha-free) barycentric shape gradients of weights.hpp:689-696.
constexpr int kRecPoint = 4;
constexpr int kRecEdge = 12;
constexpr int kRecTri = 24;
__host__ __device__ constexpr int rec_size(int kind) {
    return kind == 0 ? kRecPoint : (kind == 1 ? kRecEdge : kRecTri);
}

// ----------------------------------------------------- decision hash
// Same mixer as the CPU checker used by the tests (bit for bit).
__host__ __device__ __forceinline__ uint64_t decision_mix(uint64_t node, uint64_t kind) {
    uint64_t z = node * 4 + kind + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace sdgpu

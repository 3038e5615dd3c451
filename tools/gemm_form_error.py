"""Would a tensor-core GEMM form of the point kernel stay within tolerance?

cfg1 shape (4,096 unit-sphere points, queries uniform in [-2, 2]^3, alpha 50,
unit weights). Squared distances by the GEMM expansion |q|^2 + |p|^2 - 2 q.p
with the products rounded to bf16 / tf32 / fp32 (fp32 accumulation), against
the direct difference in fp64; d_hat = -log(sum exp(-alpha d)) / alpha in
fp64 from each. Reports the max |d_hat error| / max(1, |d_hat|) against the
fp32 parity bar 1e-5 (BASELINE north_star), overall and for queries within
0.05 of the cloud."""
import numpy as np

rng = np.random.default_rng(1001)
p = rng.normal(size=(4096, 3))
p /= np.linalg.norm(p, axis=1, keepdims=True)
q = rng.uniform(-2, 2, size=(4096, 3))
# plus queries close to the cloud (where the expansion cancels)
near = p[rng.integers(0, 4096, 1024)] + rng.normal(scale=0.01, size=(1024, 3))
q = np.concatenate([q, near])
alpha = 50.0


def rnd(x, bits):
    """round to a float with `bits` explicit mantissa bits (RN)"""
    if bits >= 23:
        return x.astype(np.float32).astype(np.float64)
    m, e = np.frexp(x)
    s = 2.0 ** (bits + 1)
    return np.ldexp(np.round(m * s) / s, e)


def dhat(s):
    d = np.sqrt(np.maximum(s, 0.0))
    a = -alpha * d
    mx = a.max(1, keepdims=True)
    return -(mx[:, 0] + np.log(np.exp(a - mx).sum(1))) / alpha


exact = dhat(((q[:, None, :] - p[None, :, :]) ** 2).sum(-1))
dmin = np.sqrt(((q[:, None, :] - p[None, :, :]) ** 2).sum(-1).min(1))
for name, bits in (("bf16", 7), ("tf32", 10), ("fp32", 23)):
    qq, pp = rnd(q, bits), rnd(p, bits)
    s = (qq ** 2).sum(1)[:, None] + (pp ** 2).sum(1)[None, :] - 2.0 * (qq @ pp.T)
    s = s.astype(np.float32).astype(np.float64)  # fp32 accumulator / epilogue
    err = np.abs(dhat(s) - exact) / np.maximum(1.0, np.abs(exact))
    print(f"{name:5s} GEMM form: max rel err {err.max():.2e} (all), {err[dmin < 0.05].max():.2e} (d_min < 0.05); "
          f"bar 1e-5 -> {'within' if err.max() <= 1e-5 else 'OUTSIDE'}")

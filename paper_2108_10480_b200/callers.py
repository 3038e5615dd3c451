"""Host-side callers above the C ABI that the reference keeps in bench.hpp:
beta_ablation (bench.hpp:94-145) and write_ablation_csv (:147-160) on top of
Engine.render (sd_render), and pearson_correlation (:163-181)."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class AblationRow:
    beta: float
    seconds: float
    speedup_vs_beta0: float
    mean_disp_rel: float
    max_disp_rel: float
    mismatched_hits: int
    leaves: int


def beta_ablation(engine, params, betas, diag: float, **render_kwargs) -> list[AblationRow]:
    """Renders the view at beta = 0 and at each beta; isosurface
    displacement along identical rays relative to the bbox diagonal."""
    from . import SmoothParams
    p0 = SmoothParams(alpha=params.alpha, alpha_u=params.alpha_u, beta=0.0, alpha_q=params.alpha_q,
                      epsilon=params.epsilon)
    ref = engine.render(p0, **render_kwargs)
    diag = max(diag, 1e-12)
    rows = []
    for beta in betas:
        rr = ref if beta == 0.0 else engine.render(
            SmoothParams(alpha=params.alpha, alpha_u=params.alpha_u, beta=beta, alpha_q=params.alpha_q,
                         epsilon=params.epsilon), **render_kwargs)
        h0, hb = ref.hit_t >= 0.0, rr.hit_t >= 0.0
        both = h0 & hb
        d = np.abs(rr.hit_t[both] - ref.hit_t[both]) / diag
        row = AblationRow(beta, rr.seconds, ref.seconds / rr.seconds if rr.seconds > 0 else 0.0,
                          float(d.mean()) if d.size else 0.0, float(d.max()) if d.size else 0.0,
                          int((h0 != hb).sum()), rr.leaves)
        if beta == 0.0:
            row.mean_disp_rel = row.max_disp_rel = 0.0
            row.mismatched_hits = 0
        rows.append(row)
    return rows


def write_ablation_csv(rows: list[AblationRow], path: str):
    with open(path, "w") as f:
        f.write("beta,render_time_s,speedup_vs_beta0,mean_disp_rel,max_disp_rel,mismatched_hits,leaves_visited\n")
        for r in rows:
            f.write("%.17g,%.6g,%.6g,%.17g,%.17g,%d,%d\n" % (r.beta, r.seconds, r.speedup_vs_beta0,
                                                             r.mean_disp_rel, r.max_disp_rel, r.mismatched_hits,
                                                             r.leaves))


def pearson_correlation(xs, ys) -> float:
    xs, ys = np.asarray(xs, float), np.asarray(ys, float)
    if len(xs) < 2 or len(xs) != len(ys):
        return 0.0
    dx, dy = xs - xs.mean(), ys - ys.mean()
    den = math.sqrt(float((dx * dx).sum()) * float((dy * dy).sum()))
    return float((dx * dy).sum() / den) if den > 0 else 0.0

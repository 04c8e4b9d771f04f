"""NEXT-1: the paper's accuracy study (§5.2) on the B200.

For uniform, wide-range and ill-conditioned (t = 1e-9, 1e-14, 1e-19) inputs and
a sweep of square sizes, compare the componentwise relative error of
  * the cascaded GEMM on the GPU (casc_gemm_fp64x2),
  * the INT8 cascade on the GPU (casc_i8_gemm_fp64x2, NEXT-3, y = 14), and
  * the plain triple-loop FP64x2 GEMM (ORACLE-DD, the paper's comparator),
against the EXACT product (superaccumulator; the paper used FP128x2).
Reports max / median relative error, the ratio max_DD / max_cascade (the
paper's Fig. illcond, right), the flag count, and for 240^3 the per-element
error-ratio distribution (Fig. illcond2/3/4).

    python scripts/accuracy_study.py [--sizes 32,64,...] [--out profiles/accuracy_r01.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import casc_inputs as I  # noqa: E402
import oracle  # noqa: E402
from casc_inputs import paper_generators as G  # noqa: E402


def rel_errors(d, C_hi, C_lo):
    """componentwise |C - C*| / |C*| against the exact product: the fixed-point
    exact evaluator (oracle/exact_fixed.py) when it applies, else the
    superaccumulator (both give the same exact error, pinned)."""
    m, n = C_hi.shape
    absab = ((np.abs(d["A_hi"]) + np.abs(d["A_lo"])) @ (np.abs(d["B_hi"]) + np.abs(d["B_lo"]))
             * (1 - 2.0 ** -40)).ravel()
    try:
        from oracle import exact_fixed
        err, ex = exact_fixed.errors(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], C_hi, C_lo)
        r = {"err": err.ravel(), "absab": absab}
        ex = ex.ravel()
    except ValueError:
        ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
        r = oracle.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(),
                                 jj.ravel(), C_hi, C_lo)
        ex = np.abs(r["ex_hi"] + r["ex_lo"])
    nz = ex > 0
    rel = np.where(nz, np.abs(r["err"]) / np.where(nz, ex, 1.0), np.abs(r["err"]))
    return rel.reshape(m, n), r


def cascerr_total(d):
    """eq:cascerr summed over the k panels, x2 for the dropped
    higher-order terms, plus the FP64x2 rounding of each panel value and
    accumulation step ((2P + 2) 2^-104 |A||B|): the paper's own forward-error
    bound for the cascade, as a diagnostic next to the north-star bound."""
    k = d["k"]
    c = oracle.select_widths(k)
    P = -(-k // 256)
    tot = 0.0
    with np.errstate(over="ignore", under="ignore"):
        for p0 in range(0, k, 256):
            a, b = np.abs(d["A_hi"][:, p0:p0 + 256]), np.abs(d["B_hi"][p0:p0 + 256])
            absab = (a @ b) * (1 + 2.0 ** -40)
            tot = tot + 2 * oracle.cascerr_bound(a.shape[1], absab, a.max(1)[:, None],
                                                 b.max(0)[None, :], c) \
                + (2 * P + 2) * 2.0 ** -104 * absab
    return tot


def run_case(d, casc, torch):
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    g_hi, g_lo, fl = casc.casc_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]), T(d["B_lo"]))
    g_hi, g_lo, fl = g_hi.cpu().numpy(), g_lo.cpu().numpy(), fl.cpu().numpy()
    i_hi, i_lo, ifl = casc.casc_i8_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                               T(d["B_lo"]))
    i_hi, i_lo, ifl = i_hi.cpu().numpy(), i_lo.cpu().numpy(), ifl.cpu().numpy()
    o_hi, o_lo = oracle.dd_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    rc, r = rel_errors(d, g_hi, g_lo)
    ri, ri_r = rel_errors(d, i_hi, i_lo)
    rd, _ = rel_errors(d, o_hi, o_lo)
    bound = oracle.north_star_bound(d["k"], r["absab"]).reshape(rc.shape)
    abs_c = np.abs(r["err"]).reshape(rc.shape)
    casc_b = cascerr_total(d)  # eq:cascerr diagnostic (SURVEY §8(c) amb. 14)
    with np.errstate(divide="ignore", invalid="ignore"):
        cr = np.where(casc_b > 0, abs_c / casc_b, 0.0)
    return dict(max_rel_cascade=float(rc.max()), max_rel_dd=float(rd.max()),
                median_rel_cascade=float(np.median(rc)), median_rel_dd=float(np.median(rd)),
                ratio_max_dd_over_cascade=float(rd.max() / rc.max()) if rc.max() > 0 else None,
                flags=int(fl.sum()), within_north_star_bound=bool(np.all(abs_c <= bound)),
                max_err_over_cascerr=float(cr.max()), within_cascerr=bool(np.all(cr <= 1.0)),
                frac_elements_cascade_better=float(np.mean(rc < rd)),
                frac_elements_cascade_not_worse=float(np.mean(rc <= rd)),
                max_rel_int8=float(ri.max()), median_rel_int8=float(np.median(ri)),
                flags_int8=int(ifl.sum()),
                int8_within_north_star_bound=bool(np.all(np.abs(ri_r["err"]).reshape(rc.shape)
                                                         <= bound))), rc, rd


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="32,64,128,240,256,384,512")
    ap.add_argument("--seeds", type=int, default=1)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "accuracy_r02.json"))
    args = ap.parse_args()
    import torch

    import paper_2303_04353_b200 as casc
    sizes = [int(s) for s in args.sizes.split(",")]
    results = {"sizes": sizes, "cases": [], "per_element_240": {}}
    gens = [("uniform", None), ("widerange", None), ("illcond", 1e-9), ("illcond", 1e-14),
            ("illcond", 1e-19)]
    t0 = time.time()
    for kind, t in gens:
        for n in sizes:
            for seed in range(args.seeds):
                if kind == "uniform":
                    Ah, Al = G.gen_uniform_dd(100 + seed, n, n, stream=30)
                    Bh, Bl = G.gen_uniform_dd(200 + seed, n, n, stream=32)
                    d = dict(A_hi=Ah, A_lo=Al, B_hi=Bh, B_lo=Bl, m=n, n=n, k=n)
                elif kind == "widerange":
                    d = G.gen_widerange(300 + seed, n, n, n)
                else:
                    d = G.gen_illcond(400 + seed, n, t)
                res, rc, rd = run_case(d, casc, torch)
                res.update(kind=kind, t=t, n=n, seed=seed)
                results["cases"].append(res)
                print(json.dumps(res), flush=True)
                if n == 240 and seed == 0:
                    ratio = rd / np.maximum(rc, 1e-300)
                    results["per_element_240"][f"{kind}" + (f"_t{t:.0e}" if t else "")] = {
                        "ratio_dd_over_cascade_percentiles": {
                            str(q): float(np.percentile(ratio, q)) for q in (1, 5, 25, 50, 75, 95, 99)},
                        "sorted_rel_err_cascade_percentiles": {
                            str(q): float(np.percentile(rc, q)) for q in (50, 90, 99, 100)},
                        "sorted_rel_err_dd_percentiles": {
                            str(q): float(np.percentile(rd, q)) for q in (50, 90, 99, 100)},
                    }
    results["seconds"] = time.time() - t0
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(results, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()

"""Paper-analog verification: one RK3 integration step of a 256^3 grid with random
[0, 1] initial values on the GPU, compared with the single-step CPU oracle; the error of every
value in ulps of the model value (Eqs. 15-16, p = 53 for FP64).  The paper reports a maximum of
<= 2 ulps on 1-16 devices.  Prints one JSON line with the histogram.

    python tools/ulp_check.py [--n 256] [--steps 1]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def ulp_errors(model, cand, p=53):
    """Eq. 15: eps = 2^(floor(log2|m|) - p + 1); Eq. 16: |m - c| / eps.  eps is undefined at m = 0
    (R#18); those values are returned separately as absolute errors."""
    m = model.ravel()
    c = cand.ravel()
    nz = m != 0
    e = np.exp2(np.floor(np.log2(np.abs(m[nz]))) - p + 1)
    return np.abs(m[nz] - c[nz]) / e, np.abs(c[~nz])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    import torch
    import oracle
    import synth
    import paper_2103_01597_b200 as b2

    oracle.set_threads(os.cpu_count() or 1)
    n = (a.n,) * 3
    ds = synth.spacing(n)
    st = synth.pcg64_state(n)
    torch.cuda.set_device(0)
    m = b2.Mesh(n, ds, synth.P0, b2.MHD_F64)
    m.load(st)
    for _ in range(a.steps):
        m.step(synth.DT)
    got = m.store().cpu().numpy()
    m.close()
    ref = oracle.integrate(st, ds, synth.P0, synth.DT, a.steps)
    # the oracle's arithmetic with the two-state RK3 form the GPU stores (reading R#4)
    w2 = oracle.integrate(st, ds, synth.P0, synth.DT, a.steps, form="w2")
    out = {"n": a.n, "steps": a.steps, "fields": {}}
    worst = 0.0
    for q, name in enumerate(("lnrho", "ux", "uy", "uz", "ss", "ax", "ay", "az")):
        u, z = ulp_errors(ref[q], got[q])
        hist = {str(k): int(np.sum(np.round(u) == k)) for k in range(0, 4)}
        hist[">=4"] = int(np.sum(np.round(u) >= 4))
        # the same error in ulps of the larger of the model value and the value before the step:
        # where f + dt RHS cancels to near 0, Eq. 15's eps shrinks while the rounding of the
        # increment does not
        mm = np.maximum(np.abs(ref[q]), np.abs(st[q])).ravel()
        u0 = np.abs(ref[q].ravel() - got[q].ravel()) / np.exp2(np.floor(np.log2(mm)) - 52)
        out["fields"][name] = {"max_ulps": float(u.max()), "mean_ulps": float(u.mean()), "hist": hist,
                               "zeros_in_model": int(z.size), "frac_le_2ulps": float(np.mean(u <= 2.0)),
                               "max_ulps_of_max_m_f0": float(u0.max())}
        # attribution (R#4): the two-state form against the explicit one, and the GPU against it
        uw, _ = ulp_errors(ref[q], w2[q])
        ug, _ = ulp_errors(w2[q], got[q])
        og, ow = u > 2.0, uw > 2.0
        out["fields"][name].update({
            "w2_vs_oracle": {"max_ulps": float(uw.max()), "frac_le_2ulps": float(np.mean(uw <= 2.0)),
                             "n_gt_2": int(ow.sum())},
            "gpu_vs_w2": {"max_ulps": float(ug.max()), "frac_le_2ulps": float(np.mean(ug <= 2.0)),
                          "n_gt_2": int((ug > 2.0).sum())},
            "gpu_outliers": int(og.sum()), "gpu_outliers_also_w2": int((og & ow).sum()),
            "gpu_outliers_within_2ulps_of_w2": int((og & (ug <= 2.0)).sum())})
        worst = max(worst, float(u.max()))
    out["max_ulps"] = worst
    print(json.dumps(out))


if __name__ == "__main__":
    main()

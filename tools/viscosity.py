"""Periodic-Poiseuille viscosity measurement on the CUDA path (§4.2, Table 1).

    python tools/viscosity.py [--case fig3|gw|pois96] [--out profiles/...json]

fig3  : Fig.-3 parameters in a 16^3 box, f = 0.05
gw    : Table-1 Groot-Warren row (eta_Mirheo 0.89-0.9, ref 0.91), 16^3, f = 0.01
pois96: BASELINE config 3, 96^3 rho = 8, f = 0.005 (long run)
Prints the binned profile, the two half-domain eta fits and the L2 error of the parabola.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workloads  # noqa: E402
from test_gpu_poiseuille import fit_eta, run_profile  # noqa: E402

CASES = {
    "fig3": (workloads.with_box(workloads.CONFIGS["pois96"], (16.0, 16.0, 16.0)), 0.05, 4000, 300, 10, 16),
    "gw": (workloads.Config("gw", (16.0, 16.0, 16.0), 3.0, 25.0, 6.75, 1.0, 1.0, 0.04), 0.01, 3000, 400, 10, 16),
    "pois96": (workloads.CONFIGS["pois96"], 0.005, 100000, 400, 50, 48),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="fig3", choices=sorted(CASES))
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg, f, warm, ns, every, nb = CASES[args.case]
    t0 = time.time()
    xc, vz = run_profile(cfg, f, warm, ns, every, nb)
    eta_lo, eta_hi, l2 = fit_eta(xc, vz, cfg.box[0], cfg.rho, f)
    res = {"case": args.case, "config": cfg.as_dict(), "f": f, "warm_steps": warm, "samples": ns, "every": every,
           "eta_lower_half": eta_lo, "eta_upper_half": eta_hi, "eta": 0.5 * (eta_lo + eta_hi), "l2_error": l2,
           "x": xc.tolist(), "vz": vz.tolist(), "wall_s": time.time() - t0}
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()

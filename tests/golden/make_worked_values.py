"""Writes pair_worked_values.txt by calling only oracle/ (no CUDA path involved).

Config-1 parameters (a=25, gamma=45, kT=1, k=0.5, dt=0.01, seed=42, r_c=1); particle i at
(1,1,1), j at (1.5,1,1), both at rest: r=0.5, e_ij=(-1,0,0).  Values follow reading C-7
(Philox2x32-10 words keyed by the per-step key) and the force of PAPER.md P:114-136 with
the 1/sqrt(dt) scaling of reading C-3.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

ROWS = [(0, 1, 0), (1, 0, 0), (0, 1, 1), (7, 3, 99), (5, 123456, 2**32 + 7)]


def main():
    p = oracle.DPDParams(box=(8.0, 8.0, 8.0), a=25.0, gamma=45.0, kT=1.0, power=0.5, dt=0.01, seed=42)
    d = oracle.min_image(p, [1.0, 1.0, 1.0], [1.5, 1.0, 1.0])
    lines = [l for l in open(__file__).read().split('"""')[1].strip().splitlines()]
    out = ["# Worked pair-RNG and pair-force values written by make_worked_values.py (oracle only)."]
    out += ["# " + l for l in lines]
    out.append("# columns: id_i id_j step  w0(hex) w1(hex)  xi  F_i_x")
    for a, b, s in ROWS:
        w0, w1 = oracle.pair_words(42, s, a, b)
        f, hit, xi = oracle.pair_force(p, d, [0, 0, 0], a, b, s)
        assert hit
        out.append(f"{a} {b} {s}  {w0:08x} {w1:08x}  {xi:.9f}  {f[0]:.9f}")
    with open(os.path.join(HERE, "pair_worked_values.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()

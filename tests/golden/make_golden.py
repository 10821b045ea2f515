"""Writes tests/golden/mrs_closed_forms.json from CLOSED FORMS (mpmath, 40 digits).

Nothing here calls the CUDA path or the oracle: every value is a closed form
obtained by substitution into Eq. MRS_kernels:
  r = 0:   H1 = 1/(4 pi e), H2 = 1/(8 pi e^3), Q = 5/(8 pi e^3), D1 = 10/(8 pi e^3), D2 = 21/(8 pi e^5)
  e = 0:   H1 = 1/(8 pi r), H2 = 1/(8 pi r^3), Q = 2/(8 pi r^3), D1 = -2/(8 pi r^3), D2 = 6/(8 pi r^5)
(the e = 0 column is the textbook singular Stokeslet / rotlet).
Run: python tests/golden/make_golden.py
"""
import json
import os

import mpmath as mp

mp.mp.dps = 40
out = {"citation": __doc__.strip().splitlines()[2:6]}
for e in ["0.01", "1"]:
    E = mp.mpf(e)
    out[f"r0_eps_{e}"] = dict(H1=float(1 / (4 * mp.pi * E)), H2=float(1 / (8 * mp.pi * E**3)),
                              Q=float(5 / (8 * mp.pi * E**3)), D1=float(10 / (8 * mp.pi * E**3)),
                              D2=float(21 / (8 * mp.pi * E**5)))
r = mp.mpf("1.7")
out["eps0_r_1.7"] = dict(H1=float(1 / (8 * mp.pi * r)), H2=float(1 / (8 * mp.pi * r**3)),
                         Q=float(2 / (8 * mp.pi * r**3)), D1=float(-2 / (8 * mp.pi * r**3)),
                         D2=float(6 / (8 * mp.pi * r**5)))
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "mrs_closed_forms.json"), "w") as f:
    json.dump(out, f, indent=1)

"""K1 gradients against the reference goldens, relative to the gradient range:

    python tools/diag_gradtol.py   (on a GPU box)
"""
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from helpers import npz
from paper_2409_00184_b200 import bspline, model
z = npz("bspline.npz")
worst = 0
for ci, (degree, ncp) in enumerate(z["cases"]):
    c = z[f"c{ci}_coeff"]; u = z[f"c{ci}_u"]
    v, g = bspline.evaluate_points_with_gradient(c, int(degree), u, knots=tuple(z[f"c{ci}_knots32"]))
    gr = z[f"c{ci}_g32"]
    e = np.abs(g - gr).max() / max(1.0, np.abs(gr).max())
    worst = max(worst, e)
    print("case", ci, degree, ncp, "rel grad err %.2e" % e, "maxg %.1f" % np.abs(gr).max())
ext = np.array([[-0.5, 0.25], [0.0, 0.5], [-1.0, -0.25]])
for j, (ncp, degree, m) in enumerate(z["dcases"]):
    mw = model.MicroModel(int(degree), z[f"d{j}_knots"], z[f"d{j}_control"], ext, 2)
    g = mw.gradients_at(z[f"d{j}_pts"]); gr = z[f"d{j}_gradients_at"]
    print("world", j, "rel grad err %.2e" % (np.abs(g - gr).max() / max(1.0, np.abs(gr).max())))
print("worst", worst)

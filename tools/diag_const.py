import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from helpers import golden_store, npz, pov_ns
from paper_2409_00184_b200 import render, model, bspline
from paper_2409_00184_b200.partition import BlockAddress
man, models, raw = golden_store("const_single")
for a, m in models.items():
    print(a, m.degree, m.control.shape, m.knots, m.extent.tolist(), m.control.ravel()[:5])
    pm = model.MicroModel(m.degree, m.knots, m.control, m.extent, a.lod)
    u = np.array([[0.1, 0.2, 0.3], [0.5, 0.5, 0.5], [0.0, 1.0, 0.999]])
    print("K1", bspline.evaluate_points_with_gradient(m.control, m.degree, u, knots=tuple(m.knots)))
    print("values_at", pm.values_at(np.array([[0.0, 0.0, 0.0], [0.5, -0.3, 0.2]])))
    from paper_2409_00184_b200.device import as_device_blocks
    st, sl = as_device_blocks([pm])
    print("info", st.info(sl[0]), st.read(sl[0]))
    pov = render.PointOfView([0, 0, 4.0], [0, 0, -1], [0, 1, 0])
    out, info, dbg = render.render_part(pov, {BlockAddress(a.lod, a.ijk): pm}, render.TransferFunction.ml_preset(),
                                        render.RenderParams(width=8, height=8, sample_distance=0.02), debug=True)
    print(info, out.cpu().numpy()[4, :, :], dbg["nsamp"].cpu().numpy()[4])

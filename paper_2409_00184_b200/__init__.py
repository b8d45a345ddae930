"""B200-native (sm_100a) Adaptive-FAM decode-and-render path (arXiv 2409.00184).

Drop-in for the reference splinecast package's render / decode path:
  render        PointOfView, TransferFunction, RenderParams, Frame, select_visible, render
  model         MicroModel, serialize / deserialize
  bspline       evaluate_points[_with_gradient], decode_tensor_product
  partition     BlockAddress, LODManifest
  store         load_model / device_loader
  runtime       ModelCache, cache_frame, prefetch_loop, replay
  device        DeviceStore / DeviceBlock (HBM-resident slots)
All decoding runs in libafam.so (include/afam.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

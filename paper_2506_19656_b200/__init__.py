"""B200-native (sm_100a) array-side hot path of the cubevid / xarrayvideo
pipeline (arXiv 2506.19656): forward fill + per-band statistics, band PCA,
bit-exact planar quantisation / dequantisation, PSNR / SSIM / bpppb.

Drop-in modules mirror the reference's names:
  transform  -> cubevid.transform  (QuantParams, fit_quant, quantize, dequantize,
                                    PcaModel, pca_fit, pca_forward, pca_inverse)
  cube       -> cubevid.cube       (forward_fill_time, ValidityMask)
  plan       -> cubevid.plan       (ChannelGroup, pack_groups, plan_stream)
  metrics    -> SPEC.md metrics    (bpppb, psnr, ssim, evaluate)
  pipeline   -> fused encode_prep / decode_eval
"""

__version__ = "0.1.0"

from .errors import (CodecError, ConfigurationError, CorruptStreamError,  # noqa: F401
                     CubevidError, ManifestError)

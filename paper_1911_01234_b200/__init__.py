"""B200-native VDAMP hot path (arXiv 1911.01234), drop-in for csmri.vdamp.run.

Modules mirror the reference package layout:
  vdamp     run / run_batch / iterate / initial_state / finalize
  wavelet   SubbandLayout, WaveletCoeffs, dwt, idwt (GPU)
  fourier   SamplingMask, KSpaceData, fft2c, ifft2c, forward, adjoint (GPU)
  denoise   SubbandVector, denoise_colored (GPU)
  sampling  ProbabilityMap, polynomial_pmap, draw_mask, synthesize (host inputs)
  trace     IterationRecord, RunTrace
  workload  BASELINE.json synthetic configurations
  dist      one-process-per-GPU sharding + final gather
All compute goes through libvdamp_b200.so (include/vdamp_b200.h).
"""

from ._lib import DimensionError
from .fourier import KSpaceData, SamplingMask
from .trace import IterationRecord, RunTrace
from .wavelet import SubbandLayout, WaveletCoeffs

__all__ = ["DimensionError", "KSpaceData", "SamplingMask", "IterationRecord", "RunTrace",
           "SubbandLayout", "WaveletCoeffs"]

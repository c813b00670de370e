"""SURE-tuned complex soft thresholding per subband on the GPU (src/denoise.py)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .wavelet import WaveletCoeffs


@dataclass
class SubbandVector:
    """One real value per subband (src/denoise.py:22-35)."""

    values: np.ndarray
    semantics: str = ""

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=float)
        if self.values.ndim != 1:
            raise ValueError("subband vector must be 1D")

    def __len__(self) -> int:
        return len(self.values)


def denoise_colored(r: WaveletCoeffs, tau: SubbandVector, *, precision="fp64", device=None):
    """Exact per-subband SURE threshold, shrink, alpha and lambda (src/denoise.py:147-178).

    Runs the sm_100a ``sure_select`` kernel (sort + fp64 scan + argmin) and
    the soft-threshold apply kernel.  Returns (w_hat, alpha, lambda).
    """
    import torch
    from .plan import get_plan
    lay = r.layout
    if len(tau) != lay.n_subbands:
        raise ValueError(f"tau has {len(tau)} entries for a layout with {lay.n_subbands} subbands")
    if np.any(tau.values <= 0):
        raise ValueError("subband noise variances must be > 0")
    plan = get_plan(lay.image_height, lay.image_width, lay.scales, 1, precision, device)
    rd = plan.to_device(r.values, plan.cdtype).reshape(1, -1).contiguous()
    td = plan.to_device(tau.values, torch.float64).reshape(1, -1).contiguous()
    w = plan.empty_coeffs()
    tr = torch.zeros((1, plan.S, 8), dtype=torch.float64, device=plan.device)
    plan.denoise_colored(rd, td, w, tr)
    trn = tr[0].cpu().numpy()
    return (WaveletCoeffs(w[0].cpu().numpy(), lay),
            SubbandVector(trn[:, 4], "derivative"),
            SubbandVector(trn[:, 2], "weight"))

"""Device twin of the reference's native kernel (kernels.nearest_scan,
kernels.py:54-63 -> _kernels.nearest_scan, _kernels.pyx:16-46)."""

from __future__ import annotations

import numpy as np

from . import _native as nat


def nearest_scan(dirs, codewords, device=None):
    """(n, 4) directions x (m, 4) codewords -> (indices int64, cosines fp64).

    fp64 dot products in the reference's association order without FMA; ties
    resolve to the lowest codeword index.  Accepts numpy arrays or torch
    tensors; returns torch tensors on the device.
    """
    import torch

    def dev_f64(x):
        t = x if torch.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        return t.to(device=device or "cuda", dtype=torch.float64).reshape(-1, 4).contiguous()

    nat.require_cuda(device or "cuda")
    d = dev_f64(dirs)
    cw = dev_f64(codewords)
    n, m = d.shape[0], cw.shape[0]
    idx = torch.empty(n, dtype=torch.int64, device=d.device)
    cos = torch.empty(n, dtype=torch.float64, device=d.device)
    nat.launch(d.device, "hqmq_nearest_scan", nat.lib().hqmq_nearest_scan, d.data_ptr(), n,
               cw.data_ptr(), m, idx.data_ptr(), cos.data_ptr())
    return idx, cos

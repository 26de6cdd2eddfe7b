"""Drop-in harness: `adaptgear` (the reference package's import name) served by
paper_2305_17408_b200, so the reference's own test files run unmodified
against the B200 package (tests/test_dropin_gpu.py).  TEST INFRASTRUCTURE.

The only adaptation is the result boundary: the package returns device
tensors where the reference returns numpy arrays, so torch tensors convert
to numpy on demand (np.asarray / np.testing / numpy operators) -- the
"to-numpy shim".  Every computation still runs on the GPU through the C-ABI.
"""
import numpy as np
import torch


def _to_numpy(self, dtype=None, copy=None):
    a = self.detach().cpu().numpy()
    return a.astype(dtype) if dtype is not None else a


torch.Tensor.__array__ = _to_numpy
# numpy's binary operators defer to objects with a higher priority; make
# ndarray (op) tensor go through __array__ instead of torch's reflected ops
torch.Tensor.__array_priority__ = -1000

from paper_2305_17408_b200 import *  # noqa: E402,F401,F403

"""Duck-typed reference-style model over committed fixture arrays (no /root/reference)."""
from types import SimpleNamespace

import numpy as np


class FixtureModel:
    """Exposes config.{layers, heads, head_dim, context_len}, grown_arrays, queries like
    the reference SyntheticModel (pkg/src/layerreuse/synthetic.py:127-192)."""

    def __init__(self, keys, values, queries, context_len):
        L, H, NT, d = keys.shape
        self.config = SimpleNamespace(layers=L, heads=H, head_dim=d, context_len=int(context_len))
        self._k, self._v, self._q = keys, values, queries

    def grown_arrays(self, steps):
        n = self.config.context_len + steps
        return self._k[:, :, :n], self._v[:, :, :n]

    def queries(self, steps):
        return self._q[:steps]


def load_npz(path):
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}

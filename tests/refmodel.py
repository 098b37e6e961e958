"""Duck-typed reference-style model over committed fixture arrays (no /root/reference)."""
from types import SimpleNamespace

import numpy as np


class FixtureModel:
    """Exposes config.{layers, heads, head_dim, context_len}, grown_arrays, queries like
    the reference SyntheticModel (pkg/src/layerreuse/synthetic.py:127-192)."""

    def __init__(self, keys, values, queries, context_len, probe=None, rho=None, probe_step=None):
        L, H, NT, d = keys.shape
        self.config = SimpleNamespace(layers=L, heads=H, head_dim=d, context_len=int(context_len))
        self._k, self._v, self._q = keys, values, queries
        self._probe, self._rho, self._probe_step = probe, rho, probe_step

    def propagate(self, x, next_layer, head, step):
        """synthetic.py:194-207 with the reference's seeded probe noise replayed from the
        fixture (probe[next_layer, head] was drawn for step == probe_step)."""
        assert step == self._probe_step, "fixture holds probe noise for one step only"
        x = np.asarray(x, dtype=np.float64)
        if self._rho == 1.0:
            return np.array(x)
        y = self._rho * x + (1.0 - self._rho) * self._probe[next_layer, head]
        n = np.linalg.norm(y)
        return y * (np.sqrt(self.config.head_dim) / (n if n != 0.0 else 1.0))

    def grown_arrays(self, steps):
        n = self.config.context_len + steps
        return self._k[:, :, :n], self._v[:, :, :n]

    def queries(self, steps):
        return self._q[:steps]


def load_npz(path):
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}

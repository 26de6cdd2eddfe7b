import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def rel_error(values, reference):
    """The reference's comparison metric (conftest.py:22-26): max |a-ref| / max(|ref|, 1)."""
    ref = np.asarray(reference, dtype=np.float64)
    diff = np.abs(np.asarray(values, dtype=np.float64) - ref)
    scale = np.maximum(np.abs(ref), 1.0)
    return float((diff / scale).max()) if diff.size else 0.0


def to_np(t):
    if t is None:
        return None
    if hasattr(t, "detach"):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def bits(a):
    """uint32 view for bitwise float comparisons (signed zeros compare equal
    numerically but not here, so callers normalise -0.0 where numpy does)."""
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32)).view(np.uint32)


def same_float(a, b) -> bool:
    """Bitwise equality up to the sign of zero."""
    a = np.asarray(a, np.float32) + np.float32(0.0)
    b = np.asarray(b, np.float32) + np.float32(0.0)
    return a.shape == b.shape and np.array_equal(bits(a), bits(b))


class Golden:
    def __init__(self, name):
        self.z = np.load(GOLDEN / name)

    def get(self, key, default=None):
        return self.z[key] if key in self.z.files else default

    def __getitem__(self, key):
        return self.z[key]

    def cases(self, prefix):
        ids = sorted({int(k.split("_")[0][len(prefix):]) for k in self.z.files
                      if k.startswith(prefix) and k.split("_")[0][len(prefix):].isdigit()})
        return ids


@pytest.fixture(scope="session")
def kernels_golden():
    return Golden("kernels.npz")


@pytest.fixture(scope="session")
def reorder_golden():
    return Golden("reorder.npz")


@pytest.fixture(scope="session")
def layers_golden():
    return Golden("layers.npz")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_graph_arrays(rng, num_vertices=None, density=None, weighted=False):
    """conftest.py:7-19 random_graph, returning raw arrays."""
    if num_vertices is None:
        num_vertices = int(rng.integers(2, 513))
    if density is None:
        density = float(rng.uniform(0.001, 0.2))
    num_edges = max(1, int(density * num_vertices * num_vertices))
    num_edges = min(num_edges, num_vertices * num_vertices)
    keys = rng.choice(num_vertices * num_vertices, size=num_edges, replace=False)
    w = rng.uniform(0.1, 2.0, size=num_edges).astype(np.float32) if weighted else None
    return num_vertices, keys // num_vertices, keys % num_vertices, w

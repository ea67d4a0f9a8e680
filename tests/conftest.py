import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        return cache[name]

    return load


@pytest.fixture(scope="session")
def golden_json():
    import json

    def load(name):
        with open(os.path.join(GOLDEN, name + ".json")) as fh:
            return json.load(fh)

    return load


def csr_from(g, prefix):
    import scipy.sparse as sp

    return sp.csr_matrix((g[prefix + "_data"], g[prefix + "_indices"], g[prefix + "_indptr"]),
                         shape=tuple(g[prefix + "_shape"]))


def host_assemble(sr, sc, local_by_o, roff=0, coff=0, shape=None):
    """Host stand-in for fem._assemble (the device assembly of the constant operators)
    so that the CPU-only tests of host tables can build a Discretization without a GPU:
    the element matrices scattered through scipy's COO -> CSR sum.  Test infrastructure
    only; tests/test_constops_gpu.py checks the device kernels against the reference."""
    import scipy.sparse as sp

    loc = np.asarray(local_by_o)[np.arange(sr.mesh.ne) & 1]
    rows = np.repeat(sr.elem[:, :, None] + roff, sc.elem.shape[1], axis=2)
    cols = np.repeat(sc.elem[:, None, :] + coff, sr.elem.shape[1], axis=1)
    return sp.coo_matrix((loc.ravel(), (rows.ravel(), cols.ravel())),
                         shape=shape or (sr.n_nodes, sc.n_nodes)).tocsr()

"""The K4 variants -- bulk-async staged (fsg_k4_tma.cuh, FSG_K4_TMA=1) and
128-bit vectorised (fsg_k4_vec.cuh, FSG_K4_VEC=1) -- are bit-identical to
the scalar K4 on open and periodic grids with every virtual-force term
active (the variant is chosen once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp_path, tma, vec=0):
    out = str(tmp_path / f"k{tma}{vec}.npz")
    env = dict(os.environ, FSG_K4_TMA=str(tma), FSG_K4_VEC=str(vec))
    subprocess.run([sys.executable, os.path.join(HERE, "helpers", "k4_variant_run.py"), out],
                   env=env, check=True, timeout=600)
    return np.load(out)


def test_tma_staged_k4_bit_identical(tmp_path):
    a, b = _run(tmp_path, 0), _run(tmp_path, 1)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


def test_vectorised_k4_bit_identical(tmp_path):
    a, b = _run(tmp_path, 0), _run(tmp_path, 0, vec=1)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k

"""The bulk-async staged K4 variant (fsg_k4_tma.cuh, FSG_K4_TMA=1) is
bit-identical to the scalar K4 on open and periodic grids with every virtual-force term
active (the variant is chosen once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp_path, tma):
    out = str(tmp_path / f"k{tma}.npz")
    env = dict(os.environ, FSG_K4_TMA=str(tma))
    subprocess.run([sys.executable, os.path.join(HERE, "helpers", "k4_variant_run.py"), out],
                   env=env, check=True, timeout=600)
    return np.load(out)


def test_tma_staged_k4_bit_identical(tmp_path):
    a, b = _run(tmp_path, 0), _run(tmp_path, 1)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


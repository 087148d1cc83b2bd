"""Output formats: the product's writers produce the
SAME BYTES as the reference's own writers, compiled unmodified into
oracle/_ref (lbm/vtk.hpp:15-38, core/csv.hpp:18-66), on the same inputs.
CPU tests: the writers are host code; the GPU test checks the asynchronous
device snapshot that feeds fsg_write_vtk."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import bind as B
from paper_2206_01683_b200 import CsvWriter, format_full, write_vtk_fields
from paper_2206_01683_b200._abi import InputError

needs_ref = pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref not built")

SPECIAL = [0.1, 1.0 / 3.0, -0.0, 0.0, 1e-300, -2.5e308, 5e-324, 123456789.123456789, -1.0,
           math.pi, float("inf"), -float("inf")]


def test_format_full_round_trips():
    r = np.random.default_rng(3)
    for v in SPECIAL + list(r.normal(size=200) * 10.0 ** r.integers(-30, 30, size=200)):
        s = format_full(v)
        assert s == "%.17g" % v
        assert float(s) == v or (math.isnan(v) and math.isnan(float(s)))


@needs_ref
def test_csv_bytes_match_reference(tmp_path):
    cols = ["t", "x", "y", "speed"]
    r = np.random.default_rng(5)
    rows = np.concatenate([np.array(SPECIAL[:8]).reshape(2, 4), r.normal(size=(20, 4))])
    ours, ref = tmp_path / "ours.csv", tmp_path / "ref.csv"
    with CsvWriter(str(ours), cols) as w:
        for row in rows:
            w.write_row(row)
    names = (C.c_char_p * 4)(*(c.encode() for c in cols))
    flat = np.ascontiguousarray(rows.reshape(-1))
    assert B.ref().ref_csv_write(str(ref).encode(), 4, names, len(rows), B.dptr(flat)) == 0
    assert ours.read_bytes() == ref.read_bytes()
    # read back by the reference's read_csv: bit-identical values
    vals = np.empty(flat.size)
    nc = np.zeros(1, np.int32)
    assert B.ref().ref_csv_read(str(ours).encode(), flat.size, B.dptr(vals), B.iptr(nc)) == len(rows)
    assert nc[0] == 4 and np.array_equal(vals, flat)


def test_csv_row_length_and_path_errors(tmp_path):
    w = CsvWriter(str(tmp_path / "a.csv"), ["a", "b"])
    with pytest.raises(InputError):
        w.write_row([1.0, 2.0, 3.0])
    w.close()
    with pytest.raises(InputError):
        CsvWriter(str(tmp_path / "no_such_dir" / "x.csv"), ["a"])


@needs_ref
def test_vtk_bytes_match_reference(tmp_path):
    dims = (7, 5, 4)
    n = int(np.prod(dims))
    r = np.random.default_rng(11)
    rho = 1.0 + 0.01 * r.normal(size=n)
    u = 0.02 * r.normal(size=3 * n)
    u[:3] = (-0.0, 1e-17, 3.0)
    dx, dt, rho_phys, nu = 0.008, 0.004, 1000.0, 0.00089
    origin = np.array([0.125, -0.3, 1e-3])
    ours, ref = tmp_path / "ours.vtk", tmp_path / "ref.vtk"
    write_vtk_fields(str(ours), dims, rho, u, dx, dt, rho_phys, origin)
    assert B.ref().ref_write_vtk(str(ref).encode(), *dims, B.dptr(rho), B.dptr(u), dx, dt, rho_phys,
                                 nu, B.dptr(origin)) == 0
    assert ours.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
@needs_ref
def test_snapshot_is_async_and_vtk_matches_reference(tmp_path):
    """The snapshot of step k is the macro of step k even when more steps are
    enqueued before it is awaited; its VTK dump equals the reference writer's."""
    import cases as K
    from paper_2206_01683_b200 import CoupledSession
    c = K.case_session_frame()
    for prec in ("fp64", "fp32"):
        s = CoupledSession(K._gpu_cfg(c, prec))
        s.initialize(c["rho0"], c["u0"])
        for k in range(3):
            s.set_frame(K._fs_to_product(K.frame_at(k, 0.004)))
            s.set_markers(c["offsets"], *K.marker_state(c, k))
            s.step()
        rho_now, u_now = s.macro()
        s.snapshot_begin()
        for k in range(3, 6):  # keep stepping while the snapshot travels
            s.set_frame(K._fs_to_product(K.frame_at(k, 0.004)))
            s.set_markers(c["offsets"], *K.marker_state(c, k))
            s.step_async()
        rho, u = s.snapshot_wait()
        assert np.array_equal(rho, rho_now) and np.array_equal(u.reshape(-1), u_now.reshape(-1))
        s.snapshot_begin()
        ours, ref = tmp_path / f"o_{prec}.vtk", tmp_path / f"r_{prec}.vtk"
        origin = np.array([0.01, 0.02, -0.03])
        s.write_vtk(str(ours), origin)
        rho2, u2 = s.macro()
        un = c["units"]
        assert B.ref().ref_write_vtk(str(ref).encode(), *c["dims"], B.dptr(np.ascontiguousarray(rho2)),
                                     B.dptr(np.ascontiguousarray(u2.reshape(-1))), un["dx"], un["dt"],
                                     un["rho"], un["nu"], B.dptr(origin)) == 0
        assert ours.read_bytes() == ref.read_bytes()
        s.close()

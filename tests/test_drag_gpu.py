"""GPU: the batched empirical-drag backend (fsg_drag_*)
against the oracle restatement (orc_empirical_step, pinned by
tests/test_drag_oracle.py): fp64 bit-identical per env; fp32 (fixed-point
reduction) within rel-L2 1e-9 and bit-identical run to run."""
import numpy as np
import pytest

from cases import rel_l2
from oracle import bind as B
from paper_2206_01683_b200 import DragBatch
from paper_2206_01683_b200.scenes import make_scene

pytestmark = pytest.mark.gpu

E = 6
KD = 40.0


def _run(precision, steps=(0, 7, 19)):
    sc = make_scene("c5")
    off, sks, rest, nrest, W, areas = sc.skin()
    d = DragBatch(E, k=KD, precision=precision)
    for e in range(E):
        d.set_skin(e, sks[0], rest, nrest, W[0], areas)
    out = []
    for k in steps:
        for e in range(E):
            d.set_pose(e, sc.poses(k + 37 * e)[0])
        out.append(d.step())
    d.close()
    return sc, out


def _oracle(sc, steps=(0, 7, 19)):
    off, sks, rest, nrest, W, areas = sc.skin()
    res = []
    for k in steps:
        taus, sts = [], []
        for e in range(E):
            t, s = B.empirical_step(sks[0], sc.poses(k + 37 * e)[0], rest, nrest, W[0], areas, KD)
            taus.append(t)
            sts.append(s)
        res.append((taus, np.array(sts)))
    return res


def test_drag_fp64_bit_exact():
    sc, g = _run("fp64")
    o = _oracle(sc)
    for (gt, gs), (ot, os_) in zip(g, o):
        for a, b in zip(gt, ot):
            assert np.array_equal(a, b)
        assert np.array_equal(gs, os_)
        assert (gs[:, :3] == 0).all() and (gs[:, 6] <= 0).any()


def test_drag_fp32_tolerance_and_determinism():
    sc, g = _run("fp32")
    _, g2 = _run("fp32")
    o = _oracle(sc)
    for (gt, gs), (ot, os_), (ht, hs) in zip(g, o, g2):
        assert rel_l2(np.concatenate(gt), np.concatenate(ot)) <= 1e-9
        assert rel_l2(gs, os_) <= 1e-9
        assert np.array_equal(np.concatenate(gt), np.concatenate(ht)) and np.array_equal(gs, hs)


def test_drag_api_contract():
    from paper_2206_01683_b200._abi import FsgError, InputError
    with pytest.raises(InputError):
        DragBatch(2, k=0.0)
    sc = make_scene("c5")
    off, sks, rest, nrest, W, areas = sc.skin()
    d = DragBatch(2)
    d.set_skin(0, sks[0], rest, nrest, W[0], areas)
    d.set_skin(1, sks[0], rest, nrest, W[0], areas)
    d.set_pose(0, sc.poses(0)[0])
    with pytest.raises(FsgError):
        d.step()  # env 1 has no pose
    d.set_pose(1, sc.poses(1)[0])
    taus, stats = d.step()
    assert len(taus) == 2 and stats.shape == (2, 7)
    d.set_poses(np.stack([sc.poses(0)[0], sc.poses(1)[0]]))  # bulk form, same poses
    taus2, stats2 = d.step()
    assert np.array_equal(np.concatenate(taus), np.concatenate(taus2)) and np.array_equal(stats, stats2)
    d.close()

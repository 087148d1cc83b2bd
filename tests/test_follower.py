"""a16 FrameFollower (frame.hpp:70-125): the product's host implementation
(libfsg.so, fsg_follower_*) is bit-identical to the reference's, in every
follow mode, through resets and yaw wrap-around.  Host code only: runs on
CPU."""
import os

import numpy as np
import pytest

import cases as K
from oracle import bind as B

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "follower.npz")


@pytest.mark.parametrize("mode", K.FOLLOW_MODES)
def test_follower_matches_golden(mode):
    got = K.run_product_follower(mode, K.follower_script())
    want = np.load(GOLD)["out_" + mode]
    assert got.shape == want.shape
    assert np.array_equal(got, want), f"max |diff| {np.abs(got - want).max()}"


@pytest.mark.skipif(not B.have_ref(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("mode", K.FOLLOW_MODES)
@pytest.mark.parametrize("tc", [0.2, 0.05])
def test_follower_matches_live_reference(mode, tc):
    ops = K.follower_script()
    assert np.array_equal(K.run_product_follower(mode, ops, tc), K.run_ref_follower(mode, ops, tc))


def test_follower_rejects_bad_input():
    from paper_2206_01683_b200 import FrameFollower, InputError
    with pytest.raises(ValueError):
        FrameFollower("sideways")
    with pytest.raises(InputError):
        FrameFollower("full", 0.0)

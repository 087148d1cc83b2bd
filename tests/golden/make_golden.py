"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs every case of tests/cases.py through oracle/_ref/libfishref.so -- the
reference's own hot-path headers (/root/reference/proj/include/fishsim,
compiled unmodified against the Eigen stand-in) -- and stores inputs and
outputs as compressed .npz files.  /root/reference does not exist on the GPU
box, so the GPU parity tests read these committed fixtures instead.

Usage (in the build container):  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import cases as K  # noqa: E402
from oracle import bind as B  # noqa: E402


def _flat(d, prefix):
    out = {}
    for k, v in d.items():
        if isinstance(v, (list, tuple)) and v and isinstance(v[0], tuple):
            continue
        if isinstance(v, dict):
            continue
        if isinstance(v, str):
            continue
        out[prefix + k] = np.asarray(v)
    return out


def main():
    assert B.have_ref(), "oracle/_ref/libfishref.so missing: run make -C oracle with /root/reference"
    # FrameFollower (frame.hpp:70-125), every mode
    ops = K.follower_script()
    np.savez_compressed(os.path.join(HERE, "follower.npz"),
                        **{"out_" + m: K.run_ref_follower(m, ops) for m in K.FOLLOW_MODES})
    print("follower ok")
    for mk in (K.case_lbm_open, K.case_lbm_periodic):
        c = mk()
        res = K.run_ref_lbm(c)
        np.savez_compressed(os.path.join(HERE, c["name"] + ".npz"), **_flat(res, "out_"))
        print(c["name"], "ok")
    for mk in (K.case_session_frame, K.case_session_roma3):
        c = mk()
        res = K.run_ref_session(c)
        np.savez_compressed(os.path.join(HERE, c["name"] + ".npz"), **_flat(res, "out_"))
        print(c["name"], "ok")
    # recenter (frame.hpp:132-154)
    c = K.case_recenter()
    R = B.ref()
    un = c["units"]
    h = R.ref_session_create(*c["dims"], un["dx"], un["dt"], un["rho"], un["nu"], 0, 0, 0, 2)
    R.ref_set_f(h, B.dptr(np.ascontiguousarray(c["f0"])))
    fs = K.frame_at(3, un["dt"])
    R.ref_set_frame(h, *(B.dptr(np.array(list(getattr(fs, k)))) for k in
                         ("p", "pd", "pdd", "q", "omega", "alpha")))
    outs = {}
    n = int(np.prod(c["dims"]))
    for j, sh in enumerate(c["shifts"]):
        R.ref_recenter(h, B.iptr(np.array(sh, dtype=np.int32)))
        f = np.empty(19 * n)
        R.ref_get_f(h, B.dptr(f))
        p = np.zeros(3)
        R.ref_get_frame_p(h, B.dptr(p))
        outs[f"out_f{j}"] = f
        outs[f"out_p{j}"] = p
    R.ref_session_destroy(h)
    np.savez_compressed(os.path.join(HERE, "recenter.npz"), **outs)
    print("recenter ok")
    # IB primitives (kernel.hpp, coupling.hpp) on edge-case coordinates
    rs = np.concatenate([np.linspace(-2.5, 2.5, 101), [0.0, 0.5, -0.5, 1.0, -1.0, 1.5, -1.5, 2.0,
                                                       -2.0, 1e-17, 1.9999999999999998]])
    phi = np.array([[R.ref_phi(k, r) for r in rs] for k in (0, 1)])
    xs = np.array([2.0, 2.5, 3.0, 3.25, 7.5, 8.0, 1.9, 13.1, 1.6, 12.5, 13.0, 5.0000000000000009])
    rng = np.zeros((2, len(xs), 2), np.int32)
    for k in (0, 1):
        for i, x in enumerate(xs):
            lo = np.zeros(1, np.int32)
            hi = np.zeros(1, np.int32)
            R.ref_range(k, float(x), B.iptr(lo), B.iptr(hi))
            rng[k, i] = (lo[0], hi[0])
    np.savez_compressed(os.path.join(HERE, "ib_primitives.npz"), rs=rs, out_phi=phi, xs=xs,
                        out_range=rng)
    print("ib_primitives ok")


if __name__ == "__main__":
    main()

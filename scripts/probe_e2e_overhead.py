"""Dev probe: where the c2 e2e step's host time goes -- the Python wrapper
(CoupledSession.step_skinned) vs the bare ABI call (fsg_step_skinned) on the
same pre-packed buffers, and a device-only step."""
import os, sys, time
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path[:0] = [R]
import numpy as np
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene
sc = make_scene("c2")
cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu, frame_mode=sc.frame_mode,
                    precision="fp32", max_markers=sc.m)
s = CoupledSession(cfg); s.set_skin(*sc.skin())
frames = [sc.frame(k) for k in range(64)]; poses = [sc.poses(k) for k in range(64)]
fpk = [f.packed() for f in frames]
for k in range(10): s.step_skinned(frames[k], poses[k])
def med(fn, n=300):
    t = []
    for k in range(n):
        t0 = time.perf_counter(); fn(k); t.append(time.perf_counter() - t0)
    return np.median(t) * 1e6
a = med(lambda k: s.step_skinned(frames[k % 64], poses[k % 64]))
b = med(lambda k: s.step_skinned(fpk[k % 64], poses[k % 64]))
def raw(k):
    s._fs_view[:] = fpk[k % 64]; s._pose_np[...] = poses[k % 64].reshape(s._pose_np.shape)
    s._L.fsg_step_skinned(s._h, s._fs_addr, s._pose_addr, s._st_addr, s._wptr, s._wptr + 8 * s._nt)
c = med(raw)
def packonly(k): frames[k % 64].packed()
d = med(packonly)
print(f"step_skinned(FrameState) {a:.1f} us | (packed frame) {b:.1f} us | bare ABI call {c:.1f} us | FrameState.packed() {d:.1f} us")

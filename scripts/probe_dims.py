"""Dev probe: pure-LBM fp32 step time for arbitrary grid shapes (argv: NXxNYxNZ ...)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig

for spec in sys.argv[1:]:
    d = tuple(int(v) for v in spec.split("x"))
    s = CoupledSession(SessionConfig(dims=d, dx=0.01, dt=0.004, frame_mode="none", precision="fp32",
                                     max_markers=1))
    ext = torch.cuda.ExternalStream(s.stream)
    for _ in range(10):
        s.step_async()
    s.last_status()
    n = max(10, int(2e9 / (d[0] * d[1] * d[2])))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for _ in range(n):
        s.step_async()
    e1.record(ext)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    cells = d[0] * d[1] * d[2]
    print(f"{spec}: {ms*1e3:.1f} us/step  {cells/ms/1e3:.0f} MLUPS  {152*cells/ms/1e6:.0f} GB/s")
    s.close()

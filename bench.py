#!/usr/bin/env python
"""bench.py -- throughput of the coupled IB-LBM step on B200.

Metric (BASELINE.json): "MLUPS (whole box) and % of HBM roofline at 1/2/4/8
B200 vs CPU ref".  One "step" is one coupled fluid step of the hot path
(markers -> interpolation/forcing/spread -> virtual force -> collide/stream
/open BC) over the synthetic scene of the workload; MLUPS = cells x steps /
time.

  value     : device time (CUDA events on the session stream, per step, L2
              flushed between steps), marker state and frames already
              resident in HBM; whole-job MLUPS (sum over ranks, max time).
  e2e       : the same metric through the public API with HOST buffers:
              every step uploads marker state + frame (pinned, zero-copy),
              runs fsg_step (synchronous status readback) and reads the
              marker forces back (wall clock per step, L2 flushed between).
  roofline  : the collide-stream kernel (dominant), 152 B per cell update,
              timed with CUDA events on its launching stream.
  cpu_baseline : the reference's own CPU code (oracle/_ref, the reference
              headers compiled unmodified) on a bounded sample of the same
              workload on this box's cores.

Workloads (BASELINE.json configs): c1 64^3 sphere, c2 128x64x64 koi in an
accelerating frame, c3 256x128x128 two-koi school (default on one GPU: the
largest single-GPU config, where the HBM fraction is judged), c4 512^3 pure
LBM z-slab-decomposed over the ranks (default on N > 1 GPUs; weak scaling:
512^3 per rank, or --c4-scaling strong; the halo exchange runs inside libfsg,
the boundary-plane kernel storing into the neighbours' halos over NVLink),
c5 96x48x48 envs.  Under torchrun the other workloads run one independent
replica per rank (weak scaling, no data-path collective).  --gpus N (N > 1)
outside torchrun relaunches itself as N ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c3] [--halo peer|nccl] [--no-cpu-baseline]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MLUPS (whole box) and % of HBM roofline at 1/2/4/8 B200 vs CPU ref"
BYTES_PER_CELL = 152  # 19 fp32 populations read + 19 written


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=["c1", "c2", "c3", "c4", "c5"],
                    help="default: c3 (the largest single-GPU config) on one GPU, c4 (the "
                         "slab-decomposed 512^3 grid, weak scaling) on N > 1")
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"],
                    help="c4 on N > 1: halo exchange inside libfsg over NVLink peer memory "
                         "(fsg_peer_*), or NCCL point-to-point through torch.distributed")
    ap.add_argument("--cpu-dry-run", action="store_true",
                    help="(tests) no GPU: spawn the ranks, rendezvous over gloo, all-gather "
                         "the slab handles and run the halo routing of c4 on host tensors")
    ap.add_argument("--envs", type=int, default=None,
                    help="c5: envs per GPU (default 8: 64 envs on 8 GPUs)")
    ap.add_argument("--c5-mode", default="batch", choices=["batch", "streams"],
                    help="c5: one batched launch per kernel (EnvBatch) or one session per stream")
    ap.add_argument("--c4-scaling", default="weak", choices=["weak", "strong"],
                    help="c4: each rank owns 512^3 (weak) or one 512^3 grid is split (strong)")
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--no-robot-leg", action="store_true",
                    help="c5: skip the e2e leg with the robot dynamics on the device")
    ap.add_argument("--markers", default="skinned", choices=["skinned", "host"],
                    help="c1-c3: bodies skinned on the device from a per-link pose each step "
                         "(fsg_set_pose; tau_ext read back) or marker arrays set each step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def share_device() -> bool:
    """FSG_BENCH_SHARE_DEVICE=1 (testing the multi-rank path on a one-GPU
    box): every rank on device 0, gloo instead of NCCL for the bench's own
    barriers and reductions (NCCL refuses two ranks on one device).  The
    ranks are time-sliced on the device, so its numbers are not throughput."""
    return os.environ.get("FSG_BENCH_SHARE_DEVICE", "0") == "1"


def coll_device(dev):
    import torch
    return torch.device("cpu") if share_device() else dev


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def workload_config(scene, args, world):
    """The `config` object of a bench line -- the workload only, identical in
    both arms (ours and --impl reference) for the same command line."""
    m = scene.m
    skinned = bool(m) and args.markers == "skinned"
    cfg = {"workload": scene.name, "dims": list(scene.dims), "markers": m,
           "marker_source": ("skinned on device" if skinned else "host arrays") if m else None,
           "frame": scene.frame_mode}
    if args.workload == "c4":
        nx, ny, nz = scene.dims
        cfg["dims"] = [nx, ny, nz * world if args.c4_scaling == "weak" else nz]
        cfg["parallelism"] = (f"z-slabs x{world} ({args.c4_scaling})" if world > 1 else "single GPU")
    elif args.workload == "c5":
        cfg["envs_per_gpu"] = args.envs or 8
        cfg["parallelism"] = f"replicas x{world}" if world > 1 else "single GPU"
    else:
        cfg["parallelism"] = f"replicas x{world}" if world > 1 else "single GPU"
    return cfg


# ------------------------------------------------------------ CPU (ref) ----
def cpu_reference_mlups(scene, seconds: float, max_steps: int = 400):
    """The reference's own CPU code (oracle/_ref: the reference headers compiled
    unmodified, OpenMP over this box's cores) driving the fluid half of
    CoupledSession::step on the same synthetic scene.  Falls back to the C
    restatement (oracle/liboracle.so) when _ref was not built."""
    import numpy as np
    if "TORCHELASTIC_RUN_ID" in os.environ:
        # torchrun pins OMP_NUM_THREADS=1 per rank; the CPU reference (rank 0
        # only) uses every host core.  Set before the oracle's OpenMP runtime loads.
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    from oracle import bind as B
    kind = "reference" if B.have_ref() else "port"
    fm = {"none": 0, "translation": 1, "translation_yaw": 2, "full": 3}[scene.frame_mode]
    m = scene.m
    nb = len(scene.bodies)
    off = scene.offsets
    if kind == "reference":
        R = B.ref()
        h = R.ref_session_create(*scene.dims, scene.dx, scene.dt, scene.rho, scene.nu, 0, 0, 0, fm)
    else:
        O = B.oracle()
        h = O.orc_session_create(B.iptr(B.dims_arr(scene.dims)), scene.dx, scene.dt, scene.rho,
                                 scene.nu, 0, 0, 0, fm)
    fw = np.zeros(3 * max(m, 1))
    valid = np.zeros(max(m, 1), np.int32)
    stats = np.zeros(7 * max(nb, 1))
    fin = np.zeros(1, np.int32)
    mf = np.zeros(1)
    mk = [scene.markers(k) for k in range(8)] if m else None

    def one(k):
        f = scene.frame(k)
        if kind == "reference":
            R.ref_set_frame(h, *(B.dptr(np.ascontiguousarray(v, dtype=np.float64)) for v in
                                 (f.p, f.pd, f.pdd, f.q, f.omega, f.alpha)))
        else:
            O.orc_session_set_frame(h, B.FrameState.make(p=f.p, pd=f.pd, pdd=f.pdd, q=f.q,
                                                         omega=f.omega, alpha=f.alpha))
        args = (h, nb, B.i64ptr(off))
        if m:
            pts, vel, nrm, area = mk[k % 8]
            marr = (B.dptr(pts.reshape(-1)), B.dptr(vel.reshape(-1)), B.dptr(nrm.reshape(-1)),
                    B.dptr(area))
        else:
            marr = (None, None, None, None)
        fn = R.ref_session_step if kind == "reference" else O.orc_session_step
        fn(*args, *marr, B.dptr(fw), B.iptr(valid), B.dptr(stats), B.iptr(fin), B.dptr(mf))

    one(0)  # warm-up (page-in, OpenMP pool)
    t0 = time.perf_counter()
    n = 0
    while n < max_steps and (time.perf_counter() - t0) < seconds:
        one(n + 1)
        n += 1
    dt = time.perf_counter() - t0
    if kind == "reference":
        R.ref_session_destroy(h)
    else:
        O.orc_session_destroy(h)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": scene.n_cells * n / dt / 1e6, "unit": "MLUPS", "cores": cores, "kind": kind,
            "cpu_model": cpu_model(), "steps": n,
            "sample": f"{n} coupled steps of {scene.name} ({dt:.1f} s wall, fp64, OpenMP)"}


# --------------------------------------------------- ours: z-slab (c4) ---
def run_slab(args, scene, rank, local, world):
    """c4: pure LBM on a 512^2 x NZ grid split into z-slabs, one per rank, with
    the boundary-plane halo exchange over NCCL overlapped with the interior
    update (paper_2206_01683_b200/slab.py).  Fluid at rest (the per-cell work
    does not depend on the state); the 20 GB per rank exceed L2 by ~160x."""
    import torch
    from paper_2206_01683_b200.slab import SlabLayout, SlabRunner
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nx, ny, nz = scene.dims
    NZ = nz * world if args.c4_scaling == "weak" else nz
    L = SlabLayout(NZ, world, periodic=False)
    run = SlabRunner(dict(dims=(nx, ny, NZ), dx=scene.dx, dt=scene.dt, rho=scene.rho, nu=scene.nu,
                          frame_mode="none", precision="fp32", device=local, max_markers=1), L, rank,
                     transport=args.halo)
    s = run.session
    stream = torch.cuda.ExternalStream(s.stream, device=dev)
    W, K = args.warmup, args.steps

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device=coll_device(dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(W):
        run.step_async()
    st = s.last_status()
    torch.cuda.synchronize(dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.4)
        e0.record(stream)
        for _ in range(K):
            run.step_async()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        time.sleep(0.15)
    st = s.last_status()
    t_total = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    total_cells = nx * ny * NZ
    value = total_cells * K / t_total / 1e6
    # e2e: the public per-step call with the status read back every step
    E = min(args.e2e_steps, K)
    barrier()
    t0 = time.perf_counter()
    for _ in range(E):
        run.step_async()
        s.last_status()
    e2e_t = max_over_ranks(time.perf_counter() - t0)
    run.close()
    peak, peak_src = measured_peaks()
    local_cells = nx * ny * run.nz
    achieved = BYTES_PER_CELL * local_cells / (t_total / K) / 1e9
    halo_mb = 2 * 5 * nx * ny * 4 / 1e6 if world > 1 else 0.0
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "MLUPS", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(t_total / K * 1e3, 4), "higher_is_better": True,
        "scaling": args.c4_scaling, "vs_baseline": None, "dtype": "f32 (fp32 storage of f - w_i)",
        "data": "synthetic (fluid at rest, pure LBM; SURVEY.md §8(d) C4)",
        "config": workload_config(scene, args, world),
        "l2": f"state {BYTES_PER_CELL * local_cells / 2 / 1e9:.1f} GB per rank >> L2 (no flush)",
        "execution": (f"{world} ranks, one slab each; halo "
                      + ("inside libfsg: boundary-plane kernel stores into the neighbours' halos "
                         "over NVLink peer memory (CUDA IPC), stream-ordered delivery counters"
                         if args.halo == "peer" else "NCCL point-to-point on a comm stream")
                      + f", {halo_mb:.1f} MB/step/rank") if world > 1 else "single GPU",
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": k4_traffic("c4") if args.c4_scaling == "weak" and world == 1 else None,
                     "kernel": "k_collide_fix (boundary planes + interior; per GPU)",
                     "peak_source": peak_src},
        "e2e": {"value": round(total_cells * E / e2e_t / 1e6, 1), "unit": "MLUPS",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 56, "steps": E},
        # peer halo: interior + boundary planes (the exchange is inside the
        # boundary kernel); nccl: boundary, pack, interior, unpack
        "gpu_launches": K * ((2 if args.halo == "peer" else 4) if world > 1 else 1),
        "status": {"stable": bool(st.stable()), "min_f": st.min_f},
        "clocks": clk.summary(),
    }


def k4_traffic(workload):
    """dram bytes read + written per launch of the dominant kernel, from the
    committed ncu --set full capture of this workload (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "k4_traffic.json")) as f:
            return json.load(f).get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_sample_scene(scene):
    """The CPU baseline's bounded sample: c4 (40 GB in fp64) is timed on a
    128^3 stand-in with identical per-cell work."""
    if scene.m == 0 and scene.n_cells > (1 << 22):
        import dataclasses
        return dataclasses.replace(scene, name=scene.name + " [CPU sample: 128^3 stand-in]",
                                   dims=(128, 128, 128))
    return scene


# ------------------------------------------------------ ours: envs (c5) ---
def robot_leg(batch, scene, E, Ee, kk, local, dev, world, flush_bufs):
    """The rollout loop with the robots on the device too:
    one fsg_batch_step_dynamic call per round uploads the actuation, steps
    fluid + robots, advances every env's FrameFollower (recentring its
    lattice when the robot drifts) and returns statuses and the post-step
    robot states -- no prescribed frames, no host marker or robot work."""
    import numpy as np
    import torch
    from paper_2206_01683_b200 import dynamics as D
    fw_buf, fr_buf, sink = flush_bufs
    robot = D.koi_robot(scene.bodies[0], scene.articulations()[0])
    rb = D.RobotBatch(robot, E, device=local)
    rb.set_rest(*D.rest_pose(robot))
    nj = robot.n_joints
    batch.set_follow(0.2, 2.0)
    batch.center_frames(rb)
    n_shift = 0
    dyn_t, dyn_ok, per_call = 0.0, True, []
    for k in range(-3, Ee):  # 3 untimed warm-up rounds (lazy module load, first-call allocations)
        fw_buf.fill_(1.0)
        torch.sum(fr_buf, dim=0, out=sink[0])
        torch.cuda.synchronize(dev)
        t_ = (kk + Ee + k) * scene.dt
        act = np.array([[0.2 * math.sin(2 * math.pi * 2.0 * t_ - 0.8 * j + e) for j in range(nj)]
                        for e in range(E)])
        t0 = time.perf_counter()
        sts_d, fl_d, _ = batch.step_dynamic(rb, act, None, scene.rho, (0.0, 0.0, -9.81), scene.dt, 4)
        if k < 0:
            continue
        n_shift += int((batch.last_shifts() != 0).any(axis=1).sum())
        per_call.append(time.perf_counter() - t0)
        dyn_t += per_call[-1]
        dyn_ok &= all(x.stable() for x in sts_d) and not (fl_d & D.FSG_DYN_NONFINITE).any()
    rb.close()
    return {"value": round(E * scene.n_cells * Ee * world / dyn_t / 1e6, 1), "unit": "MLUPS",
            # up: actuation + the env pack (frame constants, state pointers);
            # down: status, tau_ext + stats, post-step state, flags, COM
            "h2d_bytes_per_step": E * (8 * nj + 440),
            "d2h_bytes_per_step": E * (32 + 200 + 440 + 4 + 24), "steps": Ee,
            "stable": bool(dyn_ok), "recentres": n_shift,
            "call_us": {q: round(float(np.percentile(per_call, p)) * 1e6, 1)
                        for q, p in (("p50", 50), ("p90", 90), ("max", 100))},
            "what": "fsg_batch_step_dynamic: actuation up; device poses, coupled step, "
                    "buoyancy + integrate (4 substeps) of every robot, FrameFollower + "
                    "recentre trigger per env; statuses + robot states down (the "
                    "reference's full CoupledSession::step)"}


def run_envs(args, scene, rank, local, world):
    """c5: E independent envs per GPU (BASELINE: 64 envs on 8 GPUs).  batch
    mode: an EnvBatch steps every env with one marker launch and one
    collide/stream launch; streams mode: one session per
    stream.  A round = one coupled step of every env."""
    import numpy as np
    import torch
    from paper_2206_01683_b200 import CoupledSession, EnvBatch, SessionConfig
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    E = args.envs or 8
    W, K = args.warmup, args.steps
    m = scene.m
    cfg = SessionConfig(dims=scene.dims, dx=scene.dx, dt=scene.dt, rho=scene.rho, nu=scene.nu,
                        frame_mode=scene.frame_mode, precision="fp32", device=local,
                        max_markers=max(m, 1))
    batch = EnvBatch(cfg, E) if args.c5_mode == "batch" else None
    ss = batch.envs if batch else [CoupledSession(cfg) for _ in range(E)]
    skinned = bool(m) and args.markers == "skinned"
    nsteps = W + K
    # every env runs the gait with its own phase (env.hpp:73-95 randomises the
    # start); continuous motion over all W + K rounds
    mk_dev, frames, poses = [], [], []
    for e in range(E):
        frames.append([scene.frame(k + 37 * e) for k in range(nsteps)])
        if skinned:  # the per-link pose of each round (device-side skinning)
            ss[e].set_skin(*scene.skin())
            poses.append([scene.poses(k + 37 * e) for k in range(nsteps)])
            continue
        P = np.zeros((nsteps, 4, 3 * m))
        for k in range(nsteps):
            pts, vel, nrm, area = scene.markers(k + 37 * e)
            P[k, 0], P[k, 1], P[k, 2] = pts.reshape(-1), vel.reshape(-1), nrm.reshape(-1)
            P[k, 3, :m] = area
        mk_dev.append(torch.tensor(P, dtype=torch.float64, device=dev))
    streams = [torch.cuda.ExternalStream(s.stream, device=dev) for s in (ss[:1] if batch else ss)]
    main = torch.cuda.current_stream(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    nflush = max(2 * l2, 256 << 20) // 4
    fw_buf = torch.empty(nflush, dtype=torch.float32, device=dev)
    fr_buf = torch.ones(nflush, dtype=torch.float32, device=dev)
    sink = torch.zeros(1, dtype=torch.float32, device=dev)

    def round_async(k):
        for e, s in enumerate(ss):
            s.set_frame(frames[e][k % nsteps])
            if skinned:
                s.set_pose(poses[e][k % nsteps])
            else:
                r = mk_dev[e][k % nsteps]
                s.set_markers_device(scene.offsets, r[0].data_ptr(), r[1].data_ptr(),
                                     r[2].data_ptr(), r[3].data_ptr())
            if not batch:
                s.step_async()
        if batch:
            batch.step_async()

    for k in range(W):
        round_async(k)
    for s in ss:
        s.last_status()
    torch.cuda.synchronize(dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ClockSampler(local) as clk:
        time.sleep(0.4)
        for k in range(K):
            fw_buf.fill_(1.0)
            torch.sum(fr_buf, dim=0, out=sink[0])
            ev[k][0].record(main)
            for st_ in streams:
                st_.wait_event(ev[k][0])
            round_async(W + k)
            for st_ in streams:
                j = torch.cuda.Event()
                j.record(st_)
                main.wait_event(j)
            ev[k][1].record(main)
        torch.cuda.synchronize(dev)
        time.sleep(0.15)
    sts = [s.last_status() for s in ss]
    round_ms = sum(a.elapsed_time(b) for a, b in ev) / K
    t_total = round_ms * K / 1e3
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([t_total], dtype=torch.float64, device=coll_device(dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_total = float(t.item())
    value = E * scene.n_cells * K * world / t_total / 1e6
    # e2e: every env through the host API, overlapped across envs with step_async
    Ee = min(args.e2e_steps, K)
    kk = W + K  # continue the motion where the timed rounds stopped
    mk_host = None if skinned else [[scene.markers(kk + k + 37 * e) for k in range(Ee)]
                                    for e in range(E)]
    e2e_t = 0.0
    for k in range(Ee):
        fw_buf.fill_(1.0)
        torch.sum(fr_buf, dim=0, out=sink[0])
        torch.cuda.synchronize(dev)
        if skinned and batch:  # the rollout loop's exchange in one ABI call
            fr = np.stack([frames[e][(kk + k) % nsteps].packed() for e in range(E)])
            po = np.stack([poses[e][(kk + k) % nsteps][0] for e in range(E)])
            t0 = time.perf_counter()
            batch.step_skinned(fr, po)
            e2e_t += time.perf_counter() - t0
            continue
        t0 = time.perf_counter()
        for e, s in enumerate(ss):
            s.set_frame(frames[e][(kk + k) % nsteps])
            if skinned:
                s.set_pose(poses[e][(kk + k) % nsteps])
            else:
                s.set_markers(scene.offsets, *mk_host[e][k])
            if not batch:
                s.step_async()
        if batch:
            batch.step_async()
        for s in ss:
            s.last_status()
            if skinned:
                s.body_wrench()
            else:
                s.marker_forces()
        e2e_t += time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_t], dtype=torch.float64, device=coll_device(dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_dyn = None
    if skinned and batch and not args.no_robot_leg:
        e2e_dyn = robot_leg(batch, scene, E, Ee, kk, local, dev, world, flush_bufs=(fw_buf, fr_buf, sink))
    if batch:
        batch.close()
    else:
        for s in ss:
            s.close()
    peak, peak_src = measured_peaks()
    achieved = BYTES_PER_CELL * E * scene.n_cells / (round_ms / 1e3) / 1e9
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "MLUPS", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(round_ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp32 storage of f - w_i)",
        "data": ("synthetic (articulated koi per env skinned on the device from a per-link pose, "
                 "own gait phase; SURVEY.md §8(d) C5)" if skinned else
                 "synthetic (prescribed-kinematics koi per env, own gait phase; SURVEY.md §8(d) C5)"),
        "config": workload_config(scene, args, world),
        "l2": "flushed between rounds",
        "execution": (f"{E} envs per GPU batched: one marker + one collide launch per round"
                      if batch else f"{E} env sessions per GPU on {E} streams"),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": ("k_markers_batch + k_collide_band_batch, one round interval" if batch
                                else "k_markers_fix + k_collide_band of all envs, one round interval"),
                     "peak_source": peak_src},
        "e2e": {"value": round(E * scene.n_cells * Ee * world / e2e_t / 1e6, 1), "unit": "MLUPS",
                "h2d_bytes_per_step": E * ((1920 if skinned else 80 * m) + 232),
                "d2h_bytes_per_step": E * ((8 * (scene.skin()[1][0].n_dofs + 7) if skinned else 28 * m) + 64),
                "steps": Ee},
        **({"e2e_robots_on_device": e2e_dyn} if e2e_dyn else {}),
        "gpu_launches": K * (2 if batch else E * 2),
        "status": {"stable": all(st.stable() for st in sts), "min_f": min(st.min_f for st in sts)},
        "clocks": clk.summary(),
    }


# ------------------------------------------------------------------ ours ---
def run_ours(args, scene, rank, local, world):
    import numpy as np
    import torch
    from paper_2206_01683_b200 import CoupledSession, SessionConfig

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = SessionConfig(dims=scene.dims, dx=scene.dx, dt=scene.dt, rho=scene.rho, nu=scene.nu,
                        frame_mode=scene.frame_mode, precision="fp32", device=local,
                        max_markers=max(scene.m, 1))
    s = CoupledSession(cfg)
    stream = torch.cuda.ExternalStream(s.stream, device=dev)
    W, K = args.warmup, args.steps
    nsteps = W + K
    m = scene.m
    skinned = bool(m) and args.markers == "skinned"
    # marker state of every step, resident in HBM before timing (skinned:
    # the per-link poses, passed as launch parameters)
    mk_dev = None
    poses = None
    if skinned:
        s.set_skin(*scene.skin())
        poses = [scene.poses(k) for k in range(nsteps)]
    elif m:
        P = np.zeros((nsteps, 4, 3 * m))
        for k in range(nsteps):
            pts, vel, nrm, area = scene.markers(k)
            P[k, 0], P[k, 1], P[k, 2] = pts.reshape(-1), vel.reshape(-1), nrm.reshape(-1)
            P[k, 3, :m] = area
        mk_dev = torch.tensor(P, dtype=torch.float64, device=dev)
    frames = [scene.frame(k) for k in range(nsteps)]
    off = scene.offsets
    # L2 flush: write then read buffers larger than L2 (126 MB), outside timing
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    nflush = max(2 * l2, 256 << 20) // 4
    fw_buf = torch.empty(nflush, dtype=torch.float32, device=dev)
    fr_buf = torch.ones(nflush, dtype=torch.float32, device=dev)
    sink = torch.zeros(1, dtype=torch.float32, device=dev)

    def flush():
        fw_buf.fill_(1.0)
        torch.sum(fr_buf, dim=0, out=sink[0])

    def set_frame_only(k):
        s.set_frame(frames[k % len(frames)])

    def set_step(k):
        s.set_frame(frames[k])
        if skinned:
            s.set_pose(poses[k])
        elif m:
            r = mk_dev[k]
            s.set_markers_device(off, r[0].data_ptr(), r[1].data_ptr(), r[2].data_ptr(),
                                 r[3].data_ptr())

    with torch.cuda.stream(stream):
        for k in range(W):
            set_step(k)
            s.step_async()
        st = s.last_status()
        torch.cuda.synchronize(dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        if os.environ.get("BENCH_SESSION_PROFILE", "0") == "1":
            s.profile(True)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)
        with ClockSampler(local) as clk:
            time.sleep(0.4)  # let nvidia-smi start sampling before the timed region
            for k in range(K):
                flush()
                set_step(W + k)
                ev[k][0].record(stream)
                s.step_async()
                ev[k][1].record(stream)
            torch.cuda.synchronize(dev)
            time.sleep(0.15)
        st = s.last_status()
        prof_ms, nprof = s.profile_read()
        s.profile(False)
        step_ms = sum(a.elapsed_time(b) for a, b in ev) / K
        if nprof == 0:  # the step interval itself (the session's own events are off)
            prof_ms, nprof = step_ms * K, K
        # the dominant kernel alone: the pure-fluid K4 (k_collide_fix) on the
        # same grid, same flush discipline (no markers -> no band phase)
        fluid_ms = None
        if m:
            s.set_markers_device(np.array([0], dtype=np.int64), 0, 0, 0, 0)
            nf = max(K // 4, 20)
            for k in range(5):
                set_frame_only(k)
                s.step_async()
            s.last_status()
            s.profile(True)
            for k in range(nf):
                flush()
                set_frame_only(k)
                s.step_async()
            fl_ms, fl_n = s.profile_read()
            s.profile(False)
            fluid_ms = fl_ms / max(fl_n, 1)
            if skinned:
                s.set_skin(*scene.skin())
    t_total = step_ms * K / 1e3
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([t_total], dtype=torch.float64, device=coll_device(dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_total = float(t.item())
    value = scene.n_cells * K * world / t_total / 1e6

    # ---- end to end through the public API with host buffers
    E = min(args.e2e_steps, K)
    mk_host = [scene.markers(k) for k in range(8)] if (m and not skinned) else None
    e2e_t = 0.0

    def e2e_step(k):
        # the robot side's per-step exchange: pose up, tau_ext + stats down in
        # one ABI call (skinned), or the whole marker state up and per-marker
        # forces down
        if skinned:
            s.step_skinned(frames[k % nsteps], poses[k % nsteps])
            return
        s.set_frame(frames[k % nsteps])
        if m:
            s.set_markers(off, *mk_host[k % 8])
        s.step()
        if m:
            s.marker_forces()

    with torch.cuda.stream(stream):
        s.reset_to_rest()
        for k in range(3):
            e2e_step(k)
        for k in range(E):
            flush()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            e2e_step(k)
            e2e_t += time.perf_counter() - t0
    e2e_val = scene.n_cells * E / e2e_t / 1e6
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_t], dtype=torch.float64, device=coll_device(dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_val = scene.n_cells * E * world / float(t.item()) / 1e6
    nb = len(scene.bodies)
    if skinned:
        from paper_2206_01683_b200.session import POSE_DOUBLES
        ndof = sum(sk.n_dofs for sk in scene.skin()[1])
        h2d = 8 * POSE_DOUBLES * nb + 232  # fsg_body_pose per body + frame consts
        d2h = 8 * (ndof + 7 * nb) + 64  # tau_ext + CouplingStats + step status
    else:
        h2d = 80 * m + 232      # marker state (pts, vel, nrm 3x8 B, area 8 B) + frame consts
        d2h = 28 * m + 64       # marker forces (3x8 B) + validity (4 B) + step status
    s.close()
    cpp = host_e2e(scene, cfg, frames, poses) if (skinned and world == 1) else None
    # one robot in the followed frame (c2): the whole CoupledSession::step with
    # the robot on the device too (SURVEY.md §8(d) asks for e2e with the robot
    # work included for C2)
    e2e_dyn = None
    if skinned and len(scene.bodies) == 1 and scene.frame_mode != "none" and world == 1 \
            and not args.no_robot_leg:
        from paper_2206_01683_b200 import EnvBatch
        b1 = EnvBatch(cfg, 1)
        b1.envs[0].set_skin(*scene.skin())
        e2e_dyn = robot_leg(b1, scene, 1, min(args.e2e_steps, K), W + K, local, dev, world,
                            flush_bufs=(fw_buf, fr_buf, sink))
        b1.close()

    peak, peak_src = measured_peaks()
    # the coupled step's kernels overlap (the banded K4 is a programmatic
    # dependent of the marker kernel), so the dominant kernel's duration is
    # taken as the whole step interval on the session stream: conservative
    k4_avg_s = (prof_ms / max(nprof, 1)) / 1e3
    achieved = BYTES_PER_CELL * scene.n_cells / k4_avg_s / 1e9
    traffic = k4_traffic(args.workload)
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "MLUPS", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(step_ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp32 storage of f - w_i)",
        "data": ("synthetic (articulated bodies skinned on the device from a prescribed "
                 "per-link pose each step, fluid at rest; SURVEY.md §8(d))" if skinned else
                 "synthetic (prescribed-kinematics bodies, fluid at rest; SURVEY.md §8(d))"),
        "config": workload_config(scene, args, world),
        "l2": "flushed between timed steps",
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": ("k_collide_band (collide+stream+open BC+VF+IB band) with the "
                                "overlapped k_markers_fix" + (" (+ k_skin_update, k_skin_tau)" if skinned else "")
                                + ": timed as the whole step interval"
                                if m else "k_collide_fix (collide+stream+open BC+VF)"),
                     "peak_source": peak_src,
                     "step_ms": round(k4_avg_s * 1e3, 4),
                     "fluid_only": None if fluid_ms is None else {
                         "kernel": "k_collide_fix (same grid, no markers)",
                         "ms": round(fluid_ms, 4),
                         "achieved": round(BYTES_PER_CELL * scene.n_cells / (fluid_ms / 1e3) / 1e9, 1),
                         "frac": round(BYTES_PER_CELL * scene.n_cells / (fluid_ms / 1e3) / 1e9 / peak, 4)}},
        # e2e: the C++ host through the C ABI (scripts/host_e2e.cpp) when it
        # builds here, else the Python host; both are kept
        "e2e": ({"value": cpp["mlups"], "unit": "MLUPS", "h2d_bytes_per_step": h2d,
                 "d2h_bytes_per_step": d2h, "steps": cpp["steps"],
                 "host": "C++ through include/fsg.h (fsg_step_skinned, synchronous)",
                 "us_per_step": cpp["us_per_step"]} if cpp else
                {"value": round(e2e_val, 1), "unit": "MLUPS", "h2d_bytes_per_step": h2d,
                 "d2h_bytes_per_step": d2h, "steps": E, "host": "Python (ctypes)"}),
        "e2e_python": {"value": round(e2e_val, 1), "unit": "MLUPS", "steps": E},
        **({"e2e_robots_on_device": e2e_dyn} if e2e_dyn else {}),
        # skinned bodies ride in the marker kernel (<= 2 bodies; more use the
        # split skin kernels beside K4): K_m + K4 per step
        "gpu_launches": K * ((2 if len(scene.bodies) <= 2 else 4) if skinned else (2 if m else 1)),
        "status": {"stable": bool(st.stable()), "min_f": st.min_f},
        "clocks": clk.summary(),
    }
    return out


def host_e2e(scene, cfg, frames, poses, n_steps: int = 100):
    """End to end from a C++ host through the C ABI (scripts/host_e2e.cpp):
    per step the frame + per-link poses go up from host memory, the coupled
    step runs synchronously and tau_ext + CouplingStats come back
    (fsg_step_skinned) -- the FishGym binding of INTEGRATION.md, no Python on
    the timed path.  Returns its JSON result, or None when it cannot be built
    or run here (the Python e2e is reported either way)."""
    import tempfile
    import numpy as np
    from paper_2206_01683_b200.session import POSE_DOUBLES
    off, sks, rest, nrest, W, areas = scene.skin()
    n = min(n_steps, len(frames))
    c = cfg.to_c()
    tmp = tempfile.mkdtemp(prefix="fsg_host_e2e_")
    case = os.path.join(tmp, "case.bin")
    with open(case, "wb") as f:
        f.write(np.array([c.dims[0], c.dims[1], c.dims[2], c.frame_mode, len(sks), n,
                          int(off[-1])], dtype=np.int32).tobytes())
        f.write(np.array([c.dx, c.dt, c.rho, c.nu], dtype=np.float64).tobytes())
        f.write(np.asarray(off, dtype=np.int64).tobytes())
        for sk in sks:
            f.write(bytes(sk.to_c()))
        for a in (rest, nrest, areas):
            f.write(np.ascontiguousarray(a, dtype=np.float64).tobytes())
        f.write(np.concatenate([np.asarray(w, dtype=np.float64).reshape(-1) for w in W]).tobytes())
        for k in range(n):
            fr = frames[k]
            f.write(np.asarray(fr if isinstance(fr, np.ndarray) else fr.packed(), dtype=np.float64).tobytes())
        for k in range(n):
            f.write(np.asarray(poses[k], dtype=np.float64).reshape(-1, POSE_DOUBLES).tobytes())
    exe = os.path.join(tmp, "host_e2e")
    lib = os.path.join(ROOT, "paper_2206_01683_b200")
    try:
        subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "scripts", "host_e2e.cpp"), "-L", lib, "-lfsg",
                        f"-Wl,-rpath,{lib}", "-o", exe], check=True, capture_output=True, timeout=120)
        r = subprocess.run([exe, case, "5"], check=True, capture_output=True, text=True, timeout=300)
        if r.stderr:  # (dev: HOST_E2E_SPLIT=1 prints the enqueue / wait split)
            print(r.stderr.strip(), file=sys.stderr)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 -- reported, the Python e2e stands
        print(f"host_e2e unavailable: {e}", file=sys.stderr)
        return None


def spawn_ranks(args) -> int:
    """bench.py --gpus N (N > 1) outside torchrun: relaunch this command as N
    ranks, one per GPU (torch.distributed.run, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    if not args.cpu_dry_run:
        # NCCL's communicator lines (nranks, NVLS/P2P transport) on stderr
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_dry(args, rank, world):
    """--cpu-dry-run (no GPU): the multi-rank launch path of c4 down to the
    halo exchange -- gloo rendezvous, the slab layout of the weak-scaled
    512^3-per-rank grid, the all-gather of per-rank handles that
    fsg_peer_connect consumes, and the halo routing of the NCCL transport on
    host tensors of one 5-population face (reduced plane) for K steps."""
    import torch
    import torch.distributed as dist
    from paper_2206_01683_b200.slab import SlabLayout, exchange
    dist.init_process_group("gloo")
    nx, ny, nz = 512, 512, 512
    L = SlabLayout(nz * world, world, periodic=False)
    L.validate()
    z0, depth = L.planes(rank)
    handles = [None] * world
    dist.all_gather_object(handles, {"rank": rank, "z0": z0, "nz": depth})
    lo, hi = L.neighbours(rank)
    ok = all(handles[r]["rank"] == r for r in range(world))
    if lo is not None:
        ok &= handles[lo]["z0"] + handles[lo]["nz"] == z0
    if hi is not None:
        ok &= handles[hi]["z0"] == z0 + depth
    n = 5 * 64  # 5 populations x a reduced plane
    for k in range(args.steps):
        send_lo = torch.full((n,), float(1000 * rank + 2 * k))
        send_hi = torch.full((n,), float(1000 * rank + 2 * k + 1))
        recv_lo, recv_hi = torch.full((n,), -1.0), torch.full((n,), -1.0)
        have_lo, have_hi = exchange(send_lo, send_hi, recv_lo, recv_hi, rank, L)
        if have_lo:
            ok &= bool((recv_lo == 1000 * lo + 2 * k + 1).all())
        if have_hi:
            ok &= bool((recv_hi == 1000 * hi + 2 * k).all())
    t = torch.tensor([1 if ok else 0])
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_ranks": world, "backend": "gloo",
                          "workload": "c4", "dims": [nx, ny, nz * world],
                          "slabs": [[h["z0"], h["nz"]] for h in handles],
                          "steps": args.steps, "ok": bool(t.item())}))
    dist.barrier()
    dist.destroy_process_group()


def main():
    args = parse_args()
    rank, local, world = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.cpu_dry_run:
        run_dry(args, rank, world)
        return
    if args.workload is None:
        args.workload = "c4" if world > 1 else "c3"
    from paper_2206_01683_b200.scenes import make_scene
    scene = make_scene(args.workload)
    if args.impl == "reference":
        # the reference's own CPU code on the host cores, rank 0 only
        if rank != 0:
            return
        cb = cpu_reference_mlups(cpu_sample_scene(scene), seconds=max(5.0, args.cpu_seconds))
        out = {"metric": METRIC, "value": round(cb["value"], 3), "unit": "MLUPS", "n_gpus": world,
               "steps": cb["steps"], "warmup": 1, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
               "data": "synthetic", "config": workload_config(scene, args, world),
               "cpu_baseline": cb,
               "e2e": {"value": round(cb["value"], 3), "unit": "MLUPS", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return
    if share_device():
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if share_device():
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload == "c4":
        out = run_slab(args, scene, rank, local, world)
    elif args.workload == "c5" and (args.envs or 8) > 1:
        out = run_envs(args, scene, rank, local, world)
    else:
        out = run_ours(args, scene, rank, local, world)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            out["cpu_baseline"] = cpu_reference_mlups(cpu_sample_scene(scene), seconds=args.cpu_seconds)
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

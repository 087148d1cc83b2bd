"""z-slab domain decomposition of one fixed grid over the GPUs of a box
(BASELINE config c4).

Each rank owns planes [z0, z0 + nz) of a global nx x ny x NZ grid in its own
slab session (one halo plane per side).  One exchange per time step: the 5
ez=+1 post-collision populations of the top owned plane go up, the 5 ez=-1
populations of the bottom plane go down (5 * nx * ny elements per face).  The
session updates its two boundary planes first and packs them; the exchange
runs on a comm stream (NCCL point-to-point through torch.distributed) while
the interior planes update; the received planes are unpacked into the halo
before the next step.  The open boundary clamps to GLOBAL indices
(solver.hpp:59-97), so slabs of >= 2 planes never need a second neighbour.

The reference has no multi-GPU path; this is the B200 scale-out of the same
single-grid step, and its results are bit-identical to one monolithic session
(tests/test_slab_gpu.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SlabLayout:
    """Balanced split of `nz_global` planes over `world` ranks."""

    nz_global: int
    world: int
    periodic: bool = False

    def planes(self, rank: int) -> tuple[int, int]:
        """(z_offset, depth) of `rank`'s slab."""
        base, extra = divmod(self.nz_global, self.world)
        z0 = rank * base + min(rank, extra)
        return z0, base + (1 if rank < extra else 0)

    def neighbours(self, rank: int) -> tuple[int | None, int | None]:
        """(lower, upper) neighbour ranks, None at a closed global face."""
        lo, hi = rank - 1, rank + 1
        if self.periodic:
            return lo % self.world, hi % self.world
        return (lo if lo >= 0 else None), (hi if hi < self.world else None)

    def validate(self) -> None:
        if self.world < 1:
            raise ValueError("world must be >= 1")
        if min(self.planes(r)[1] for r in range(self.world)) < 2:
            raise ValueError(f"{self.nz_global} planes over {self.world} ranks: slabs need >= 2 planes")


def exchange(send_lo, send_hi, recv_lo, recv_hi, rank: int, layout: SlabLayout, group=None):
    """Move send_hi -> upper neighbour's recv_lo and send_lo -> lower
    neighbour's recv_hi with torch.distributed point-to-point (NCCL on GPUs,
    gloo on CPUs).  Returns (have_lo, have_hi); waits on the current stream."""
    import torch.distributed as dist
    lo, hi = layout.neighbours(rank)
    if layout.world == 1:
        return False, False
    # order: (send up, receive from below), (send down, receive from above) --
    # when both neighbours are the same rank (periodic, world 2) messages
    # between the pair match in posting order, and this order pairs each
    # receive with the partner's send of the same face
    ops = []
    if hi is not None:
        ops.append(dist.P2POp(dist.isend, send_hi, hi, group))
    if lo is not None:
        ops.append(dist.P2POp(dist.irecv, recv_lo, lo, group))
        ops.append(dist.P2POp(dist.isend, send_lo, lo, group))
    if hi is not None:
        ops.append(dist.P2POp(dist.irecv, recv_hi, hi, group))
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    return lo is not None, hi is not None


class _CudaBuf:
    """__cuda_array_interface__ view of a session-owned device buffer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 2}


def device_views(session, dtype_str: str):
    """Zero-copy torch views of the session's four halo buffers."""
    import torch
    esize = 4 if dtype_str == "<f4" else 8
    n = session.halo_bytes() // esize
    return tuple(torch.as_tensor(_CudaBuf(p, n, dtype_str), device="cuda")
                 for p in session.halo_buffers())


class SlabRunner:
    """One rank of a slab-decomposed pure-LBM run: a slab session and its
    halo transport.

    transport="peer" (default): the exchange runs inside libfsg
    (fsg_peer_*): the handles are all-gathered once over the process group,
    each session connects to its neighbours, and a step is ONE library call
    -- the boundary planes' kernel stores the crossing populations straight
    into the neighbours' halos over NVLink, ordered by stream memory
    operations.  transport="nccl": the session packs its boundary planes and
    torch.distributed point-to-point moves them on a comm stream
    (fsg_halo_begin/end), the pre-peer path, kept for comparison."""

    def __init__(self, cfg_kwargs: dict, layout: SlabLayout, rank: int, group=None,
                 transport: str = "peer"):
        import torch
        from .session import CoupledSession, SessionConfig
        layout.validate()
        if transport not in ("peer", "nccl"):
            raise ValueError(f"unknown transport {transport!r}")
        z0, nz = layout.planes(rank)
        nx, ny, _ = cfg_kwargs["dims"]
        kw = dict(cfg_kwargs)
        kw.update(dims=(nx, ny, nz), z_offset=z0, nz_global=layout.nz_global,
                  boundary="periodic" if layout.periodic else kw.get("boundary", "open"))
        self.layout, self.rank, self.group = layout, rank, group
        self.cfg = SessionConfig(**kw)
        self.session = CoupledSession(self.cfg)
        self.z0, self.nz = z0, nz
        # one rank owns the whole grid: a plain session (periodic z wraps in place)
        self.sharded = layout.world > 1
        self.transport = transport if self.sharded else None
        self.comm = None
        self.bufs = None
        if self.transport == "nccl":
            self.comm = torch.cuda.Stream(device=self.cfg.device)
            self.bufs = device_views(self.session, "<f4" if self.cfg.precision == "fp32" else "<f8")
        elif self.transport == "peer":
            import torch.distributed as dist
            handles = [None] * layout.world
            dist.all_gather_object(handles, self.session.peer_export(), group=group)
            connect_peers(self.session, handles, layout, rank)

    def step_async(self) -> None:
        import torch
        s = self.session
        s.step_async()
        if self.transport != "nccl":
            return
        s.halo_begin(self.comm.cuda_stream)
        with torch.cuda.stream(self.comm):
            have_lo, have_hi = exchange(*self.bufs, self.rank, self.layout, self.group)
        s.halo_end(self.comm.cuda_stream, have_lo, have_hi)

    def close(self) -> None:
        if self.transport == "peer":
            # a neighbour may still store into this session's halo until every
            # rank has drained its stream
            import torch
            import torch.distributed as dist
            torch.cuda.synchronize(self.cfg.device)
            dist.barrier(group=self.group)
        self.session.close()


def connect_peers(session, handles, layout: SlabLayout, rank: int) -> None:
    """Connect `rank`'s slab session to its neighbours' peer handles."""
    lo, hi = layout.neighbours(rank)
    session.peer_connect(handles[lo] if lo is not None else None,
                         handles[hi] if hi is not None else None)


def split_field(arr: np.ndarray, dims, layout: SlabLayout, rank: int, comps: int = 1) -> np.ndarray:
    """Rank's z-slab of a global cell-ordered field (x fastest, comps per cell)."""
    nx, ny, _ = dims
    z0, nz = layout.planes(rank)
    a = np.asarray(arr).reshape(-1, ny, nx, comps) if comps > 1 else np.asarray(arr).reshape(-1, ny, nx)
    return np.ascontiguousarray(a[z0:z0 + nz]).reshape(-1)

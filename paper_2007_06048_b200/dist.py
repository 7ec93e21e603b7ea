"""Z-slab domain decomposition of acoustic_iso_cd over several GPUs.

ref: dist.cpp:12-45 (topology, decompose, local_box), dist.cpp:92-115
(exchange_halos), dist.cpp:119-132 (validate_cuts), dist.cpp:144-267
(run_distributed_rank).

B200 design:
* one process per GPU; the grid is cut along z (the slowest device axis), so
  a rank's r owned edge planes and r ghost planes are contiguous blocks of
  device memory -- NCCL sends/receives them in place, no packing kernels;
* cuts are cost-weighted (the end ranks also own the z damping layers) and
  must satisfy the reference's legality rule nd + r <= cut <= n - nd - r,
  which guarantees no CPML memory read crosses a cut (only p is exchanged);
* per step ("overlap" schedule): CPML pass 1 -> the r edge planes of p_next
  -> NCCL send/recv of those planes into the neighbours' p_next ghost planes,
  overlapped with the interior planes -> join -> source / free surface ->
  rotate.  The exchanged planes become the neighbours' p_cur ghosts, exactly
  what the reference's exchange_halos(p_cur) produces before the next step.
The "simple" schedule (exchange p_cur, then step) is the reference's own
order and is what the CPU (gloo) tests drive.

Transports: ``TorchTransport`` (torch.distributed, NCCL on GPUs, gloo on CPU)
and ``LocalTransport`` (all ranks in one process; device-to-device copies).
"""
from __future__ import annotations

import json
import math
import os
import time
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from ._lib import ConfigError


# --------------------------------------------------------------- decomposition
def decompose(n: int, parts: int, coord: int) -> Tuple[int, int]:
    """ref: dist.cpp:23-34 -- (offset, count); the remainder goes to low coordinates."""
    if parts < 1 or coord < 0 or coord >= parts:
        raise ConfigError("invalid decomposition coordinate")
    if n < parts:
        raise ConfigError(f"cannot split {n} points over {parts} ranks")
    base, rem = divmod(n, parts)
    count = base + (1 if coord < rem else 0)
    return coord * base + min(coord, rem), count


def validate_cuts(cuts: Sequence[int], n: int, nd: int, radius: int) -> None:
    """ref: dist.cpp:119-132 -- interior cuts must stay nd + r away from both faces."""
    keep = nd + radius
    for c in cuts[1:-1]:
        if c < keep or c > n - keep:
            raise ConfigError(f"rank boundary at index {c} cuts through the damping region "
                              f"(must be >= {keep} points from either domain boundary)")
    for a, b in zip(cuts[:-1], cuts[1:]):
        if b - a < radius:
            raise ConfigError(f"slab [{a}, {b}) is thinner than the stencil radius {radius}")


def plane_costs(n: Sequence[int], nd: Sequence[int]) -> np.ndarray:
    """Algorithmic bytes of each z plane under the byte model:
    16 B per point + 16 B per damped axis of the point."""
    nx, ny, nz = n
    dx = 2 * min(nd[0], nx) / nx
    dy = 2 * min(nd[1], ny) / ny
    z = np.arange(nz)
    zdamp = ((z < nd[2]) | (z >= nz - nd[2])).astype(np.float64)
    per_point = 16.0 + 16.0 * (dx + dy + zdamp)
    return per_point * nx * ny


def weighted_cuts(n: Sequence[int], nd: Sequence[int], radius: int, parts: int) -> List[int]:
    """Cost-balanced legal z cuts: equal prefix-sum shares of plane_costs,
    clamped into [nd + r, n - nd - r]."""
    nz = n[2]
    if parts == 1:
        return [0, nz]
    cost = plane_costs(n, nd)
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    keep = nd[2] + radius
    cuts = [0]
    for p in range(1, parts):
        target = cum[-1] * p / parts
        c = int(np.searchsorted(cum, target))
        if c > 0 and abs(cum[c - 1] - target) < abs(cum[c] - target):
            c -= 1
        c = max(c, keep, cuts[-1] + radius)
        c = min(c, nz - keep)
        cuts.append(c)
    cuts.append(nz)
    validate_cuts(cuts, nz, nd[2], radius)
    return cuts


def equal_cuts(nz: int, parts: int) -> List[int]:
    return [decompose(nz, parts, c)[0] for c in range(parts)] + [nz]


def balance(n, nd, cuts) -> float:
    """min/max slab cost ratio (1 = perfect)."""
    cost = plane_costs(n, nd)
    w = [cost[a:b].sum() for a, b in zip(cuts[:-1], cuts[1:])]
    return float(np.mean(w) / np.max(w))


# --------------------------------------------------------------- transports
class TorchTransport:
    """Halo messages over torch.distributed (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    @property
    def rank(self):
        return self.dist.get_rank(self.group)

    @property
    def world(self):
        return self.dist.get_world_size(self.group)

    def exchange(self, sends, recvs):
        """sends/recvs: lists of (peer, tensor).  Returns a waitable list."""
        ops = [self.dist.P2POp(self.dist.isend, t, peer, self.group) for peer, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, peer, self.group) for peer, t in recvs]
        if not ops:
            return []
        return self.dist.batch_isend_irecv(ops)

    @staticmethod
    def wait(works):
        for w in works:
            w.wait()

    def barrier(self):
        self.dist.barrier(self.group)

    def max(self, value: float) -> float:
        import torch
        t = torch.tensor([value], dtype=torch.float64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


# --------------------------------------------------------------- slab geometry
@dataclass
class SlabInfo:
    rank: int
    world: int
    cuts: List[int]

    @property
    def z0(self):
        return self.cuts[self.rank]

    @property
    def nz(self):
        return self.cuts[self.rank + 1] - self.cuts[self.rank]

    @property
    def lower(self):
        return self.rank - 1 if self.rank > 0 else None

    @property
    def upper(self):
        return self.rank + 1 if self.rank + 1 < self.world else None


def local_vp(vp_global: np.ndarray, radius: int, z0: int, nz: int) -> np.ndarray:
    """ref: dist.cpp:171-180 -- the rank's ghosted slice of the ghosted global
    model (ghost reads across cuts resolve to the neighbours' interior)."""
    return np.ascontiguousarray(vp_global[:, :, z0:z0 + nz + 2 * radius])


def halo_pairs(info: SlabInfo):
    """Message plan of one exchange (ref: dist.cpp:92-115, z faces only):
    [(peer, my side, tag)] -- owned planes of `side` go to the neighbour's
    opposite ghost; the neighbour's owned planes land in my `side` ghost."""
    plan = []
    if info.lower is not None:
        plan.append((info.lower, 0))
    if info.upper is not None:
        plan.append((info.upper, 1))
    return plan


# --------------------------------------------------------------- GPU rank
class ZSlabRank:
    """One rank of the GPU z-slab run (wraps an AcousticCdEngine)."""

    def __init__(self, engine, info: SlabInfo, transport, src_global=None):
        self.e = engine
        self.info = info
        self.t = transport
        self.src_local = None
        if src_global is not None and info.z0 <= src_global[2] < info.z0 + info.nz:
            self.src_local = (src_global[0], src_global[1], src_global[2] - info.z0)
        self._views = {}

    # device memory views of the halo planes (zero copy, via the C ABI)
    def _view(self, side, which, next_field):
        import torch
        ptr, nbytes = self.e.halo_planes(side, which, next_field=next_field)
        key = (ptr, nbytes)
        v = self._views.get(key)  # the 3 rotating buffers give a few fixed views
        if v is None:
            class _A:
                __cuda_array_interface__ = {"shape": (nbytes // 4,), "typestr": "<f4",
                                            "data": (ptr, False), "version": 3}

            v = self._views[key] = torch.as_tensor(_A(), device=f"cuda:{self.e.device}")
        return v

    def exchange_current(self):
        """Reference order: exchange p_cur ghosts (dist.cpp:213-214)."""
        sends, recvs = [], []
        for peer, side in halo_pairs(self.info):
            sends.append((peer, self._view(side, 0, False)))
            recvs.append((peer, self._view(side, 1, False)))
        return self.t.exchange(sends, recvs)

    def step_simple(self, amp: float):
        import torch
        ext = torch.cuda.ExternalStream(self.e.stream_handle(), device=self.e.device)
        with torch.cuda.stream(ext):
            works = self.exchange_current()
            self.t.wait(works)
        self.e.step(amp, self.src_local)

    # ---- overlap schedule, in phases (a LocalTransport driver interleaves
    # the phases of several ranks; step_overlap runs them back to back)
    def _edges(self):
        r, nz = self.e.grid().radius, self.info.nz
        out = []
        if self.info.lower is not None:
            out.append((0, min(r, nz)))
        if self.info.upper is not None:
            lo = max(nz - r, r if self.info.lower is not None else 0)
            if lo < nz:
                out.append((lo, nz))
        return out

    def _src_in_edges(self):
        if self.src_local is None:
            return False
        return any(a <= self.src_local[2] < b for a, b in self._edges())

    def phase_edges(self, amp: float):
        """CPML pass 1 on every plane, then p_next on the r planes next to each
        cut (+ the source if it sits there, so neighbours receive it)."""
        self.e.update_boundary_psi()
        edges = self._edges()
        if edges:  # both cuts' edge planes in one launch per kernel
            self.e.update_plane_ranges(edges)
        if self._src_in_edges():
            self.e.inject_source(amp, self.src_local)

    def halo_messages(self):
        """(sends, recvs) of p_next edge planes -> neighbours' p_next ghosts."""
        sends, recvs = [], []
        for peer, side in halo_pairs(self.info):
            sends.append((peer, self._view(side, 0, True)))
            recvs.append((peer, self._view(side, 1, True)))
        return sends, recvs

    def phase_interior(self):
        r, nz = self.e.grid().radius, self.info.nz
        a = r if self.info.lower is not None else 0
        b = nz - r if self.info.upper is not None else nz
        if a < b:
            self.e.update_planes(a, b)

    def phase_finish(self, amp: float):
        if not self._src_in_edges():
            self.e.inject_source(amp, self.src_local)
        self.e.apply_free_surface()
        self.e.rotate()

    def step_overlap(self, amp: float):
        """edges -> NCCL(edges) || interior -> join -> finish (see module doc)."""
        import torch
        ext = torch.cuda.ExternalStream(self.e.stream_handle(), device=self.e.device)
        with torch.cuda.stream(ext):
            self.phase_edges(amp)
            sends, recvs = self.halo_messages()
            works = self.t.exchange(sends, recvs)  # NCCL waits for the edges
            self.phase_interior()                  # concurrent with the transfer
            self.t.wait(works)                     # engine stream waits for NCCL
            self.phase_finish(amp)


def step_local(ranks: Sequence["ZSlabRank"], amp: float):
    """All ranks in one process (LocalTransport semantics): the overlap
    schedule's phases interleaved across ranks, halo planes moved with
    device-to-device copies."""
    import torch
    for rk in ranks:
        rk.phase_edges(amp)
    for rk in ranks:
        rk.e.synchronize()
    msgs = [rk.halo_messages() for rk in ranks]
    for i, rk in enumerate(ranks):
        _, recvs = msgs[i]
        for peer, dst in recvs:
            # my ghost on `side` <- the peer's owned planes facing me
            for q, src in msgs[peer][0]:
                if q == i:
                    dst.copy_(src)
    torch.cuda.synchronize()
    for rk in ranks:
        rk.phase_interior()
    for rk in ranks:
        rk.phase_finish(amp)


def run_zslab(mm, config, vp_global: np.ndarray, info: SlabInfo, transport, *, device=0,
              mode="fast", schedule="overlap", nsteps=None, timed=False):
    """Distributed acoustic_iso_cd run (ref: dist.cpp:144-267) on one rank.

    Returns dict(traces on rank 0 for receivers owned by rank 0 -- all of them
    for legal cuts, since the receiver plane k = nd_z lies below the first cut),
    dt, device_seconds)."""
    import torch
    n = tuple(config.ngrid)
    r = config.stencil_radius
    grid = mm.make_grid(n, config.dgrid, r)
    model = mm.EarthModel(grid, vp_global)
    model = mm.validate_model(model)
    dt = mm.cfl_dt(model, grid, config.cfl)
    w = mm.ricker(config.fmax, dt, config.nsteps).samples
    lgrid = mm.make_grid((n[0], n[1], info.nz), config.dgrid, r)
    vp_loc = local_vp(model.vp, r, info.z0, info.nz)
    opts = mm.EngineOptions(ndamping=tuple(config.ndamping), fmax=config.fmax,
                            r_target=config.r_target, free_surface=config.free_surface,
                            taper=config.taper, ntaper=tuple(config.ntaper))
    eng = mm.AcousticCdEngine(lgrid, (0, 0, info.z0), n, vp_loc, opts, float(np.float32(dt)),
                              model.vmax, device=device, mode=mode)
    src = config.source_loc if config.source_loc is not None else tuple(x // 2 for x in n)
    rk = ZSlabRank(eng, info, transport, src)
    geo = mm.default_receivers(grid, config.ndamping, config.receiver_increment)
    k_rec = config.ndamping[2]
    owns_rec = info.z0 <= k_rec < info.z0 + info.nz
    steps = config.nsteps if nsteps is None else nsteps
    if owns_rec:
        rec = geo.receivers.copy()
        rec[:, 2] -= info.z0
        eng.set_receivers(rec, steps)
    # initial p_cur ghosts (all zero unless seeded): the overlap schedule
    # exchanges p_next after every step, so one exchange up front suffices
    torch.cuda.synchronize()
    transport.barrier()
    t0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ext = torch.cuda.ExternalStream(eng.stream_handle(), device=device)
    ev0.record(ext)
    for s in range(steps):
        if schedule == "overlap":
            rk.step_overlap(float(w[s]))
        else:
            rk.step_simple(float(w[s]))
        if owns_rec:
            eng.record(s)
    ev1.record(ext)
    eng.synchronize()
    torch.cuda.synchronize()
    dev_s = ev0.elapsed_time(ev1) * 1e-3
    transport.barrier()
    out = {"dt": dt, "device_seconds": dev_s, "wall_seconds": time.perf_counter() - t0,
           "engine": eng, "owns_receivers": owns_rec}
    if owns_rec:
        out["traces"] = eng.traces(steps)
    return out


# --------------------------------------------------------------- bench (torchrun)
def bench_rank(args, rank, world, local):
    """bench.py --gpus N under torchrun: weak scaling, per-rank 240^3 work
    (global grid 240 x 240 x (240 N)), cost-weighted z slabs, NCCL halos
    overlapped with the interior.  `value`: device time of K steps of the
    overlap schedule (max over ranks); `e2e`: the same K steps with the source
    sample H2D and the receiver plane D2H (rank 0) every step, wall clock, max
    over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2007_06048_b200 as mm
    from . import _lib
    from .driver import SimConfig

    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if "RANK" not in os.environ:  # a single rank started without torchrun
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK=str(local),
                              MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    edge = args.grid or 240
    n = (edge, edge, edge * world)
    cfg = SimConfig(ngrid=n, nsteps=args.warmup, stencil_radius=args.radius)
    cuts = weighted_cuts(n, cfg.ndamping, args.radius, world)
    info = SlabInfo(rank, world, cuts)
    grid = mm.make_grid(n, cfg.dgrid, args.radius)
    vp = mm.default_layered_model(grid).vp
    tr = TorchTransport()
    # W warm-up steps (engine, receivers, work lists, NCCL communicators)
    res = run_zslab(mm, cfg, vp, info, tr, device=local, mode=args.mode)
    eng = res["engine"]
    rk = ZSlabRank(eng, info, tr, tuple(x // 2 for x in n))
    w = mm.ricker(cfg.fmax, res["dt"], args.warmup + args.steps).samples[args.warmup:]
    ext = torch.cuda.ExternalStream(eng.stream_handle(), device=local)

    def timed(e2e: bool):
        owns = res["owns_receivers"]
        nrec = n[0] * n[1]
        host = (torch.empty((args.steps, nrec), dtype=torch.float32, pin_memory=True).numpy()
                if e2e and owns else None)
        if owns:
            eng.set_receivers(_receivers_local(mm, grid, cfg, info), args.steps)
        tr.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        l0 = _lib.kernel_launch_count()
        t0 = time.perf_counter()
        e0.record(ext)
        for s in range(args.steps):
            rk.step_overlap(float(w[s]))
            if owns:
                eng.record(s)
                if e2e:
                    eng.copy_trace_step(s, host[s], asynchronous=True)
        e1.record(ext)
        eng.synchronize()
        wall = time.perf_counter() - t0
        launches = _lib.kernel_launch_count() - l0
        torch.cuda.synchronize()
        tr.barrier()
        return e0.elapsed_time(e1), wall * 1e3, launches, (nrec * 4 if owns else 0)

    from .clocks import ClockSampler
    clocks = ClockSampler(local)
    clocks.start()
    ms, _, launches, _ = timed(False)
    clk = clocks.stop()
    dev_ms = tr.max(ms)
    _, wall_ms, _, d2h = timed(True)
    e2e_ms = tr.max(max(wall_ms, ms))
    d2h = int(tr.max(float(d2h)))
    pts = float(n[0]) * n[1] * n[2]
    value = pts * args.steps / (dev_ms * 1e-3) / 1e9
    e2e = pts * args.steps / (e2e_ms * 1e-3) / 1e9
    all_launches = int(tr.max(float(launches)) * world) if world > 1 else launches
    if rank == 0:
        print(json.dumps({
            "metric": "Gpoints/s (grid-point updates/sec) acoustic_iso_cd 8th-order",
            "value": round(value, 3), "unit": "Gpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (default two-layer vp model 1500/4500, Ricker source)",
            "config": {"workload": f"acoustic_iso_cd r={args.radius} {n[0]}x{n[1]}x{n[2]} grid, "
                                   f"z-slabs {cuts}, NCCL halo exchange overlapped "
                                   "with the interior (weak scaling: 240^3 per GPU)",
                       "grid": list(n), "cuts": cuts, "radius": args.radius,
                       "balance": round(balance(n, cfg.ndamping, cuts), 4), "mode": args.mode,
                       "l2": "working set > 126 MB L2 per GPU; no flush"},
            "e2e": {"value": round(e2e, 3), "unit": "Gpoints/s", "h2d_bytes_per_step": 4 * world,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": all_launches,
            "clocks": clk,
        }), flush=True)
    dist.destroy_process_group()
    return 0


def _receivers_local(mm, grid, cfg, info):
    geo = mm.default_receivers(grid, cfg.ndamping, cfg.receiver_increment)
    rec = geo.receivers.copy()
    rec[:, 2] -= info.z0
    return rec

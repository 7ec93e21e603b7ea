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
The GPU ranks run that schedule in C++ (mm_cd_group_*, csrc/group.cu, NCCL
inside); this module plans the cuts, shares the NCCL id and drives the bench.
``ZSlabRank`` / ``step_local`` restate the same schedule in Python over the
plane-range C ABI for the single-GPU emulation test (all ranks in one
process, device-to-device halo copies); the "simple" schedule (exchange p_cur,
then step) is the reference's own order, which the CPU (gloo) tests drive
with ``TorchTransport``.
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


# Relative cost of a plane inside a z damping layer, measured on B200: every
# rank's slab of 512^3 / 1000^3 timed alone (tools/scaling_projection.py,
# profiles/r02_scaling_projection.json) gives 2.4-2.8x the time of an
# undamped plane on the final round-2 kernels (3.1x before the pass-1 stage
# lane and the boundary work-item changes), against 1.9x in the byte model
# (the z runs' pass-1 chains and the Z-slab tiles cost more than their bytes).
ZDAMP_PLANE_WEIGHT = 2.7


def plane_costs(n: Sequence[int], nd: Sequence[int], zdamp_weight: float = ZDAMP_PLANE_WEIGHT
                ) -> np.ndarray:
    """Relative cost of each z plane for the cuts: the byte model (BASELINE.md
    2: 16 B per point + 16 B per damped axis) for the x/y damping, with a plane
    of a z damping layer weighted `zdamp_weight` times an undamped plane
    (measured; the byte model alone says ~1.9)."""
    nx, ny, nz = n
    dx = 2 * min(nd[0], nx) / nx
    dy = 2 * min(nd[1], ny) / ny
    z = np.arange(nz)
    zdamp = ((z < nd[2]) | (z >= nz - nd[2])).astype(np.float64)
    per_point = (16.0 + 16.0 * (dx + dy)) * (1.0 + (zdamp_weight - 1.0) * zdamp)
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
    """Python restatement of the group schedule (csrc/group.cu) for one slab
    engine, over the plane-range C ABI: the single-GPU emulation test drives
    several of them in one process (step_local), halo planes moved with
    device-to-device copies where the C++ group uses NCCL."""

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


def layered_slice(n: Sequence[int], z0: int, nz: int, radius: int) -> np.ndarray:
    """The rank's ghosted slice [z0 - r, z0 + nz + r) of the global
    default_layered_model (model.cpp:63-77: vp 1500 for k < n_z/2, 4500 below;
    ghosts replicate the edge values), built without the global volume
    (1000^3 would be 4 GB per rank)."""
    r = radius
    k = np.clip(np.arange(z0 - r, z0 + nz + r), 0, n[2] - 1)
    col = np.where(k < n[2] // 2, 1500.0, 4500.0).astype(np.float32)
    return np.ascontiguousarray(np.broadcast_to(col, (n[0] + 2 * r, n[1] + 2 * r, nz + 2 * r)))


def share_nccl_id(rank: int) -> bytes:
    """Rank 0's NCCL unique id, broadcast over the torch.distributed process
    group (the host plumbing; the halo traffic itself is the C++ group's)."""
    import torch.distributed as dist
    from .propagator import nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def run_zslab(mm, config, vp_global: Optional[np.ndarray], info: SlabInfo, *, device=0,
              mode="fast", nsteps=None, nccl_id: Optional[bytes] = None, vp_local=None):
    """Distributed acoustic_iso_cd run (ref: run_distributed_rank,
    dist.cpp:144-267) on one rank, through the C++ group (mm_cd_group_*: NCCL
    halo exchange overlapped with the interior, per-rank finiteness check).

    Returns dict(traces of the receivers this rank owns -- all of them on
    rank 0 for legal cuts, since the receiver plane k = nd_z lies below the
    first cut --, dt, device_seconds, group)."""
    from .propagator import ZSlabGroup
    n = tuple(config.ngrid)
    r = config.stencil_radius
    grid = mm.make_grid(n, config.dgrid, r)
    if vp_local is None:
        model = mm.validate_model(mm.EarthModel(grid, vp_global))
        vmax = model.vmax
        vp_global = model.vp
    else:
        vmax = float(vp_local.max())
    dt = cfl_dt_vmax(vmax, grid, config.cfl)
    steps = config.nsteps if nsteps is None else nsteps
    w = mm.ricker(config.fmax, dt, max(steps, 1)).samples
    opts = mm.EngineOptions(ndamping=tuple(config.ndamping), fmax=config.fmax,
                            r_target=config.r_target, free_surface=config.free_surface,
                            taper=config.taper, ntaper=tuple(config.ntaper))
    grp = ZSlabGroup(grid, info.cuts, info.rank, vp_global, opts, float(np.float32(dt)), vmax,
                     nccl_id=nccl_id, device=device, mode=mode, vp_local=vp_local)
    src = config.source_loc if config.source_loc is not None else tuple(x // 2 for x in n)
    k_rec = config.ndamping[2]
    owns_rec = info.z0 <= k_rec < info.z0 + info.nz
    if owns_rec:
        grp.engine.set_receivers(_receivers_local(mm, grid, config, info), steps)
    ms = grp.run(w[:steps], src, record=owns_rec) if steps > 0 else 0.0
    out = {"dt": dt, "device_seconds": ms * 1e-3, "group": grp, "owns_receivers": owns_rec}
    if owns_rec:
        out["traces"] = grp.engine.traces(steps)
    return out


def cfl_dt_vmax(vmax: float, grid, cfl: float) -> float:
    """cfl_dt (driver.cpp:19-29) from vmax alone."""
    import ctypes as C
    from . import _lib
    g = _lib.mm_grid()
    g.n[:] = list(grid.n)
    g.d[:] = list(grid.d)
    g.radius = grid.radius
    dt = C.c_double()
    _lib.check(_lib.lib().mm_cfl_dt(float(vmax), C.byref(g), float(cfl), C.byref(dt)))
    return dt.value


# --------------------------------------------------------------- bench (torchrun)
def bench_rank(args, rank, world, local):
    """bench.py --gpus N under torchrun, one rank per GPU through the C++ group
    (NCCL halo planes overlapped with the interior update).

    --scaling weak (default): 240^3 per GPU, global grid 240 x 240 x 240 N;
    --scaling strong: the global grid fixed at --grid^3 (BASELINE configs[2]
    512^3, configs[3] 1000^3), cost-weighted legal z cuts.  `value` = global
    points x K / the max over ranks of the device time of K steps; `e2e`: the
    same K steps driven step by step through the C ABI with the source sample
    H2D and the receiver plane D2H (rank 0) every step.  Strong scaling also
    reports the efficiency of bench.cpp:130-145 against one GPU on the same
    grid (rank 0 alone, after the group is gone)."""
    import torch
    import torch.distributed as dist
    import paper_2007_06048_b200 as mm
    from . import _lib
    from .driver import SimConfig
    from .propagator import ZSlabGroup
    from .scaling import ScalingResult, ScalingRun, compute_efficiency, count_stencil_cost

    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if "RANK" not in os.environ:  # a single rank started without torchrun
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK=str(local),
                              MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo")  # host plumbing; halos go over the group's NCCL
    strong = getattr(args, "scaling", "weak") == "strong"
    edge = args.grid or (1000 if strong else 240)
    n = (edge, edge, edge) if strong else (edge, edge, edge * world)
    r = args.radius
    cfg = SimConfig(ngrid=n, nsteps=args.warmup, stencil_radius=r)
    nd = tuple(cfg.ndamping)
    cuts = weighted_cuts(n, nd, r, world)
    info = SlabInfo(rank, world, cuts)
    grid = mm.make_grid(n, cfg.dgrid, r)
    vp_loc = layered_slice(n, info.z0, info.nz, r)
    vmax = 4500.0
    dt = cfl_dt_vmax(vmax, grid, cfg.cfl)
    total = args.warmup + args.steps
    w = mm.ricker(cfg.fmax, dt, total).samples
    src = tuple(x // 2 for x in n)
    opts = mm.EngineOptions(ndamping=nd, taper=True)
    nid = share_nccl_id(rank) if world > 1 else None
    grp = ZSlabGroup(grid, cuts, rank, None, opts, float(np.float32(dt)), vmax, nccl_id=nid,
                     device=local, mode=args.mode, vp_local=vp_loc)
    eng = grp.engine
    owns = info.z0 <= nd[2] < info.z0 + info.nz
    nrec = n[0] * n[1]
    if owns:
        eng.set_receivers(_receivers_local(mm, grid, cfg, info), total)
    # warm-up (work lists, NCCL connections, clocks)
    grp.run(w[:args.warmup], src, record=owns)
    dist.barrier()
    from .clocks import ClockSampler
    clocks = ClockSampler(local)
    clocks.start()
    l0 = _lib.kernel_launch_count()
    ms = grp.run(w[args.warmup:total], src, record=owns, first_sample=args.warmup)
    launches = _lib.kernel_launch_count() - l0
    clk = clocks.stop()
    dev_ms = _max(ms)
    # e2e: step by step through the C ABI, host amplitude in, receiver plane out
    host = (torch.empty((args.steps, nrec), dtype=torch.float32,
                        pin_memory=torch.cuda.is_available()).numpy()
            if owns else None)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(args.steps):
        grp.step(float(w[args.warmup + s]), src)
        if owns:
            eng.record(args.warmup + s)
            eng.copy_trace_step(args.warmup + s, host[s], asynchronous=True)
    eng.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    e2e_ms = _max(max(wall_ms, ms))
    # host cost of issuing one group step (the C++ schedule: launches, events,
    # the NCCL group), measured on the host clock without synchronising
    dist.barrier()
    nh = min(args.steps, 20)
    h0 = time.perf_counter()
    for s in range(nh):
        grp.step(float(w[args.warmup + s]), src)
    host_us = (time.perf_counter() - h0) * 1e6 / nh
    eng.synchronize()
    host_us = _max(host_us)
    pts = float(n[0]) * n[1] * n[2]
    value = pts * args.steps / (dev_ms * 1e-3) / 1e9
    e2e = pts * args.steps / (e2e_ms * 1e-3) / 1e9
    all_launches = int(_max(float(launches)) * world)
    grp.close()
    del grp, eng
    torch.cuda.synchronize()
    eff = None
    if strong and world > 1 and getattr(args, "efficiency", True):
        # one GPU on the same global grid (bench.cpp:130-145 strong, r0 = 1)
        t1 = None
        if rank == 0:
            t1 = _single_gpu_ms_per_step(mm, n, r, nd, dt, w, src, local, args)
        t1 = _bcast_float(t1)
        if t1 and t1 > 0:
            res = ScalingResult("strong", [ScalingRun(1, n, 1, kernel_s=t1 * 1e-3),
                                           ScalingRun(world, n, 1,
                                                      kernel_s=dev_ms / args.steps * 1e-3)])
            compute_efficiency(res)
            eff = {"efficiency_pct": round(res.runs[1].efficiency_pct, 2),
                   "one_gpu_ms_per_step": round(t1, 4),
                   "definition": "t1 * 1 / (tN * N), bench.cpp:130-145 strong"}
    if rank == 0:
        cost = count_stencil_cost("acoustic_iso_cd", r)
        line = {
            "metric": "Gpoints/s (grid-point updates/sec) acoustic_iso_cd 8th-order",
            "value": round(value, 3), "unit": "Gpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (default two-layer vp model 1500/4500, Ricker source)",
            "config": {"workload": (f"acoustic_iso_cd r={r} {n[0]}x{n[1]}x{n[2]} grid, "
                                    f"{world} z-slabs {cuts}, NCCL halo planes overlapped "
                                    "with the interior (C++ group, mm_cd_group_run)"
                                    + ("" if strong else "; weak scaling: 240^3 per GPU")),
                       "grid": list(n), "cuts": cuts, "radius": r,
                       "balance": round(balance(n, nd, cuts), 4), "mode": args.mode,
                       "l2": "working set > 126 MB L2 per GPU; no flush",
                       "flops_per_point": cost.flops_per_point,
                       "arithmetic_intensity": round(cost.arithmetic_intensity, 4)},
            "e2e": {"value": round(e2e, 3), "unit": "Gpoints/s", "h2d_bytes_per_step": 4 * world,
                    "d2h_bytes_per_step": 4 * nrec},
            "gpu_launches": all_launches,
            "host_issue_us_per_step": round(host_us, 1),
            "clocks": clk,
        }
        if eff:
            line["parallel_efficiency"] = eff
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def _max(v: float) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _bcast_float(v):
    import torch.distributed as dist
    obj = [v]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def _single_gpu_ms_per_step(mm, n, r, nd, dt, w, src, device, args):
    """ms/step of one engine on the whole grid (the strong-scaling baseline),
    or None when the grid does not fit the GPU."""
    import torch
    free, _ = torch.cuda.mem_get_info(device)
    pts = (n[0] + 2 * r + 32) * (n[1] + 2 * r) * (n[2] + 2 * r)
    if 6.5 * 4 * pts > 0.9 * free:
        return None
    grid = mm.make_grid(n, (20.0, 20.0, 20.0), r)
    vp = layered_slice(n, 0, n[2], r)
    e = mm.AcousticCdEngine(grid, (0, 0, 0), n, vp, mm.EngineOptions(ndamping=nd, taper=True),
                            float(np.float32(dt)), 4500.0, device=device, mode=args.mode)
    k = max(3, min(args.steps, 50))
    e.run(w[:3], src, record=False)
    ms = e.run(w[:k], src, record=False)
    e.close()
    return ms / k


def _receivers_local(mm, grid, cfg, info):
    geo = mm.default_receivers(grid, cfg.ndamping, cfg.receiver_increment)
    rec = geo.receivers.copy()
    rec[:, 2] -= info.z0
    return rec

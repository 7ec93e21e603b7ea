"""Z-slab decomposition host logic (paper_2007_06048_b200.dist).

CPU tests: decomposition arithmetic (ref: test_dist.cpp:32-41), the legality
rule (dist.cpp:119-132), cost-weighted cuts, and a world_size-2 gloo run of
the halo-exchange plan driving the CPU oracle engines, bit-identical to the
single-rank run (test_dist.cpp:107-118 restated for z cuts)."""
import os
import socket

import numpy as np
import pytest

from paper_2007_06048_b200 import dist as D
from paper_2007_06048_b200._lib import ConfigError


def test_decompose_matches_reference():
    assert [D.decompose(100, 3, c) for c in range(3)] == [(0, 34), (34, 33), (67, 33)]
    assert D.decompose(1024, 4, 3) == (768, 256)
    assert D.decompose(7, 1, 0) == (0, 7)
    with pytest.raises(ConfigError):
        D.decompose(3, 4, 0)


def test_cuts_through_damping_are_rejected():
    # test_dist.cpp:120-127: 32 points, nd 8, r 4, 4 parts -> cuts 8/16/24 illegal
    with pytest.raises(ConfigError, match="damping"):
        D.validate_cuts(D.equal_cuts(32, 4), 32, 8, 4)
    D.validate_cuts(D.equal_cuts(64, 2), 64, 8, 4)


@pytest.mark.parametrize("n,parts", [(1000, 8), (512, 8), (1000, 4), (512, 2), (240, 2)])
def test_weighted_cuts_are_legal_and_balanced(n, parts):
    nd = (27, 27, 27)
    cuts = D.weighted_cuts((n, n, n), nd, 4, parts)
    assert cuts[0] == 0 and cuts[-1] == n and len(cuts) == parts + 1
    D.validate_cuts(cuts, n, 27, 4)
    # (512^3 over 8: the legality rule keeps the end slabs >= nd + r = 31
    # planes, which the cost model rates 11 % above a share; the measured slab
    # times there are within 13 % of each other, profiles/r02_scaling_projection.json)
    assert D.balance((n, n, n), nd, cuts) >= (0.88 if (n, parts) == (512, 8) else 0.98)
    # equal cuts leave the CPML end slabs overloaded (SURVEY finding 6): 87.8 %
    # under the byte model alone, less with the measured z-layer plane weight
    if (n, parts) == (1000, 8):
        assert abs(D.balance((n, n, n), nd, D.equal_cuts(n, parts)) - 0.878) > 0.05
        assert D.balance((n, n, n), nd, D.equal_cuts(n, parts)) < 0.85
        eq_bytes = D.plane_costs((n, n, n), nd, zdamp_weight=33.73 / 17.73)
        w = [eq_bytes[a:b].sum() for a, b in zip(D.equal_cuts(n, parts)[:-1],
                                                 D.equal_cuts(n, parts)[1:])]
        assert abs(np.mean(w) / np.max(w) - 0.878) < 0.01


def test_weighted_cuts_reject_impossible_layouts():
    # 100^3 at 4 ranks: the reference's equal cuts (25/50/75) are illegal, the
    # weighted cuts stay inside [31, 69]
    cuts = D.weighted_cuts((100, 100, 100), (27, 27, 27), 4, 4)
    assert all(31 <= c <= 69 for c in cuts[1:-1])
    with pytest.raises(ConfigError):
        D.validate_cuts(D.equal_cuts(100, 4), 100, 27, 4)
    with pytest.raises(ConfigError):
        D.weighted_cuts((60, 60, 60), (27, 27, 27), 4, 2)  # no legal cut exists


def test_halo_plan():
    info = D.SlabInfo(1, 3, [0, 10, 20, 30])
    assert (info.z0, info.nz, info.lower, info.upper) == (10, 10, 0, 2)
    assert D.halo_pairs(info) == [(0, 0), (2, 1)]
    assert D.halo_pairs(D.SlabInfo(0, 1, [0, 30])) == []


# ------------------------------------------------------------ gloo, world 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, n, nd, steps, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2007_06048_b200 import dist as D
        o = Oracle("port")
        r = 4
        vp, vmin, vmax = o.layered_model(n)
        cuts = D.weighted_cuts(n, nd, r, world)
        info = D.SlabInfo(rank, world, cuts)
        eng = o.engine((n[0], n[1], info.nz), D.local_vp(vp, r, info.z0, info.nz),
                       offset=(0, 0, info.z0), global_n=n, ndamping=nd, taper=True,
                       ntaper=(2, 2, 2), dt=1.61e-3, vmax=vmax)
        w = o.ricker(25.0, 1.61e-3, steps)
        src = (n[0] // 2, n[1] // 2, n[2] // 2)
        src_local = (src[0], src[1], src[2] - info.z0) if info.z0 <= src[2] < info.z0 + info.nz \
            else None
        tr = D.TorchTransport()
        for s in range(steps):
            # exchange_halos(p_cur) then step (dist.cpp:213-215), planes packed
            # into contiguous tensors (the CPU field is z-fastest)
            pc, pp = eng.pressure(), eng.pressure_prev()
            sends, recvs = [], []
            for peer, side in D.halo_pairs(info):
                own = pc[:, :, r:2 * r] if side == 0 else pc[:, :, -2 * r:-r]
                sends.append((peer, torch.from_numpy(np.ascontiguousarray(own))))
                recvs.append((peer, torch.empty(own.shape, dtype=torch.float32)))
            tr.wait(tr.exchange(sends, recvs))
            for (peer, side), (_, buf) in zip(D.halo_pairs(info), recvs):
                if side == 0:
                    pc[:, :, :r] = buf.numpy()
                else:
                    pc[:, :, -r:] = buf.numpy()
            eng.set_state(pp, pc)
            eng.step(float(w[s]), src_local)
        q.put((rank, info.z0, info.nz, eng.pressure()[:, :, r:-r].copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_zslab_equals_single_rank():
    import torch.multiprocessing as mp
    from oracle.oracle import Oracle
    n, nd, steps = (24, 24, 48), (4, 4, 4), 30
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, n, nd, steps, q))
             for r in range(2)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    o = Oracle("port")
    vp, _, vmax = o.layered_model(n)
    whole = o.engine(n, vp, ndamping=nd, taper=True, ntaper=(2, 2, 2), dt=1.61e-3, vmax=vmax)
    w = o.ricker(25.0, 1.61e-3, steps)
    for s in range(steps):
        whole.step(float(w[s]), (n[0] // 2, n[1] // 2, n[2] // 2))
    full = whole.pressure()[:, :, 4:-4]
    covered = 0
    for rank, z0, nz, field in sorted(parts):
        assert np.array_equal(field[4:-4, 4:-4], full[4:-4, 4:-4, z0:z0 + nz]), rank
        covered += nz
    assert covered == n[2]


# ------------------------------------------------------------ group host plumbing
def test_layered_slice_equals_global_model_slices(mm):
    """Each rank builds its ghosted slab of default_layered_model without the
    global volume (dist.cpp:171-180 slices the global one): identical."""
    from paper_2007_06048_b200 import dist as D
    n = (20, 22, 41)
    full = mm.default_layered_model(mm.make_grid(n, (20.0, 20.0, 20.0))).vp
    for cuts in ([0, 41], [0, 15, 41], [0, 12, 20, 29, 41]):
        for a, b in zip(cuts[:-1], cuts[1:]):
            assert np.array_equal(D.layered_slice(n, a, b - a, 4), D.local_vp(full, 4, a, b - a))


def test_native_cut_validation_matches_reference_rule(mm):
    """mm_zslab_validate_cuts (C ABI) == dist.cpp:119-132 == validate_cuts."""
    from paper_2007_06048_b200 import dist as D
    from paper_2007_06048_b200.propagator import validate_cuts_native
    validate_cuts_native([0, 31, 64], 64, 27, 4)
    for bad in ([0, 30, 64], [0, 34, 64], [0, 40, 42, 64]):
        with pytest.raises(mm.ConfigError):
            validate_cuts_native(bad, 64, 27, 4)
        with pytest.raises(mm.ConfigError):
            D.validate_cuts(bad, 64, 27, 4)
    for p in (2, 4, 8):
        validate_cuts_native(D.weighted_cuts((1000, 1000, 1000), (27, 27, 27), 4, p),
                             1000, 27, 4)


def _id_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_06048_b200 import dist as D
        q.put((rank, D.share_nccl_id(rank)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_nccl_id_broadcast():
    """Every rank of the C++ group gets rank 0's 128-byte NCCL id through the
    torch.distributed plumbing (bench_rank / run_zslab)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got[0]) == 128 and got[0] == got[1]


# ------------------------------------------------------------ bench_rank plumbing
class _FakeEngine:
    def set_receivers(self, ijk, cap):
        assert ijk.shape[1] == 3 and (ijk[:, 2] >= 0).all()
        self.cap = cap

    def record(self, s):
        assert 0 <= s < self.cap

    def copy_trace_step(self, s, out, asynchronous=False):
        assert 0 <= s < self.cap and out.dtype == np.float32

    def synchronize(self):
        pass


class _FakeGroup:
    """Stands in for ZSlabGroup (the C++ group needs GPUs and NCCL)."""

    def __init__(self, grid, cuts, rank, vp_global, opts, dt, vmax, *, nccl_id=None, device=0,
                 mode="fast", vp_local=None):
        assert len(cuts) == 3 and vp_local.shape[2] == cuts[rank + 1] - cuts[rank] + 8
        assert nccl_id is not None and len(nccl_id) == 128
        self.engine = _FakeEngine()

    def run(self, amps, src, record=True, first_sample=0):
        return 0.5 * len(amps)

    def step(self, amp, src):
        pass

    def close(self):
        pass


def _bench_worker(rank, world, port, scaling, q):
    import contextlib
    import io
    import types
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2007_06048_b200 import dist as D
    from paper_2007_06048_b200 import propagator as P
    P.ZSlabGroup = _FakeGroup
    torch.cuda.set_device = lambda *a, **k: None
    torch.cuda.synchronize = lambda *a, **k: None
    D._single_gpu_ms_per_step = lambda *a, **k: 1.0
    args = types.SimpleNamespace(steps=4, warmup=3, grid=64 if scaling == "weak" else 100,
                                 radius=4, mode="fast", scaling=scaling, efficiency=True)
    out = io.StringIO()
    with contextlib.redirect_stdout(out):
        D.bench_rank(args, rank, world, 0)
    q.put((rank, out.getvalue()))


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_rank_world2_plumbing(scaling):
    """bench.py --gpus 2 (bench_rank) end to end on two gloo ranks with a
    stand-in for the C++ group: NCCL-id broadcast, cuts, max-over-ranks
    timing, e2e loop, strong-scaling efficiency, one JSON line on rank 0."""
    import json
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, scaling, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1].strip() == ""
    line = json.loads(res[0].strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and "host_issue_us_per_step" in line
    if scaling == "weak":
        assert line["config"]["grid"] == [64, 64, 128]
    else:
        assert line["config"]["grid"] == [100, 100, 100]
        # fake times: 1 GPU 1.0 ms/step, 2 ranks 0.5 ms/step -> 100 %
        assert abs(line["parallel_efficiency"]["efficiency_pct"] - 100.0) < 1e-6


def test_bench_spawns_ranks_without_torchrun():
    """`bench.py --gpus 2` started without torchrun launches two ranks itself
    (torch.distributed.run) -- here the reference arm, which runs on rank 0
    only and needs no GPU."""
    import json
    import subprocess
    import sys
    from conftest import ROOT
    from oracle.oracle import available
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--steps", "2", "--warmup", "1", "--grid", "64"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["grid"] == [64, 64, 128]

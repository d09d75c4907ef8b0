"""Multi-GPU frame: instance shards -> screen bands.

CPU: partition arithmetic, and a world_size-2 gloo run of the exchange layer
(TorchExchange) carrying oracle splats. The band owners must recover exactly the
reference's sorted splat list restricted to their band (renderer.cpp:85-161), and the
gathered bands must rebuild the oracle frame.
GPU: P virtual ranks on one GPU, run phase by phase with no rank waiting on another.
They drive the real C-ABI split (gscg_project_shard / gscg_pack_bands /
gscg_render_band), and the image must be byte-identical to the single-GPU frame.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2501_17792_b200.multigpu import band_rows, route_counts, shard_ranges


# ---------------------------------------------------------------- partition arithmetic

@pytest.mark.parametrize("n,parts", [(0, 1), (1, 4), (7, 3), (3500, 8), (100, 100)])
def test_shard_ranges_cover(n, parts):
    r = shard_ranges(n, parts)
    assert len(r) == parts and r[0][0] == 0 and r[-1][1] == n
    assert all(r[i][1] == r[i + 1][0] for i in range(parts - 1))
    sizes = [b - a for a, b in r]
    assert max(sizes) - min(sizes) <= 1


def test_shard_ranges_weighted():
    w = np.array([1.0] * 10 + [100.0] * 2 + [1.0] * 10)
    r = shard_ranges(len(w), 2, w)
    assert r[0][0] == 0 and r[1][1] == len(w) and r[0][1] == r[1][0]
    loads = [w[a:b].sum() for a, b in r]
    assert max(loads) <= 0.5 * w.sum() + w.max()


@pytest.mark.parametrize("h,tile,parts", [(1080, 16, 1), (1080, 16, 2), (1080, 16, 8), (240, 16, 3),
                                          (100, 8, 20), (17, 16, 4)])
def test_band_rows_tile_aligned(h, tile, parts):
    rows = band_rows(h, tile, parts)
    assert len(rows) == parts + 1 and rows[0] == 0 and rows[-1] == h
    assert all(rows[i] <= rows[i + 1] for i in range(parts))
    assert all(r % tile == 0 for r in rows[:-1])


def test_band_rows_weighted_balance():
    trows = 68
    w = np.zeros(trows)
    w[30:40] = 1000.0  # a horizon-like hot band
    w += 1.0
    rows = band_rows(1080, 16, 4, w)
    loads = [w[rows[b] // 16: (rows[b + 1] + 15) // 16].sum() for b in range(4)]
    assert max(loads) < 0.5 * w.sum()
    assert all(r % 16 == 0 for r in rows[:-1])


def test_load_balancer_plans_from_observed_work():
    from paper_2501_17792_b200.multigpu import LoadBalancer

    scene = _small_scene()
    lb = LoadBalancer(scene, 2, 16)
    shards, rows = lb.plan()
    assert shards == shard_ranges(6, 2) and rows == band_rows(120, 16, 2)
    lods = np.array([0, 0, 2, 2, 2, 2])  # two heavy near characters first
    trows = (120 + 15) // 16
    lb.observe(lods, np.arange(1, trows + 1, dtype=np.float64) ** 3, 0)
    shards, rows = lb.plan()
    assert shards[0][1] <= 2  # the heavy instances fill the first shard
    assert rows[1] > band_rows(120, 16, 2)[1]  # heavy bottom rows -> the first band grows
    assert all(r % 16 == 0 for r in rows[:-1]) and rows[-1] == 120


def test_route_counts():
    rects = np.array([[0, 10], [10, 20], [15, 40], [5, 5]])
    assert route_counts(rects, [0, 16, 32, 48]).tolist() == [3, 2, 1]


# ---------------------------------------------------------------- gloo exchange (CPU)

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _small_scene():
    import paper_2501_17792_b200 as P

    cfg = P.SceneConfig(template_count=2, template_seed_base=100, level_counts=(1500, 400, 100), with_sh=True,
                        motion_count=2, motion_frames=60, grid_rows=2, grid_cols=3, crowd_count=6, crowd_seed=11,
                        cam_pos=(1.0, 1.4, -2.5), cam_look=(1.0, 1.0, 3.0), width=160, height=120,
                        lod_thresholds=(3.0, 4.5))
    return P.Scene(cfg)


def _gloo_worker(rank: int, world: int, port: int, result_dir: str):
    import torch
    import torch.distributed as dist

    from oracle import orc
    from paper_2501_17792_b200.multigpu import TorchExchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene = _small_scene()
        o = orc.from_scene(scene)
        rgb, T, _ = o.render(0.41, orc.settings(tile_size=16, sh_colour=True))
        sp = o.splats()  # the reference's sorted splat list (renderer.cpp:85-107)
        assert sp.dtype.itemsize == 64
        n = scene.counts()[2]
        lo, hi = shard_ranges(n, world)[rank]
        rows = band_rows(scene.cfg.height, 16, world)
        # this rank's projected splats, in an arbitrary (reversed) arrival order
        mine = sp[(sp["instance_id"] >= lo) & (sp["instance_id"] < hi)][::-1]
        y = mine["rect"][:, [1, 3]]
        counts = route_counts(y, rows)
        chunks = [mine[(y[:, 0] < rows[b + 1]) & (y[:, 1] > rows[b])] for b in range(world)]
        assert [len(c) for c in chunks] == counts.tolist()
        send = torch.from_numpy(np.concatenate(chunks).view(np.uint8).copy())
        ex = TorchExchange()
        recv, rc = ex.all_to_all(send, counts.tolist(), unit=64)
        got = recv.numpy().view(sp.dtype)
        assert len(got) == sum(rc)
        # band owner: the reference's total order (depth, instance, gaussian)
        order = np.lexsort((got["gaussian_index"], got["instance_id"], got["depth"]))
        got = got[order]
        b0, b1 = rows[rank], rows[rank + 1]
        want = sp[(sp["rect"][:, 1] < b1) & (sp["rect"][:, 3] > b0)]
        assert got.tobytes() == want.tobytes(), "band splat list differs from the reference order"
        # gather: bands of the oracle frame rebuild it on rank 0
        band = torch.from_numpy(np.concatenate([rgb, T[..., None]], axis=2)[b0:b1].copy())
        full = ex.gather_rows(band, rows)
        if rank == 0:
            full = full.numpy()
            assert full[..., :3].tobytes() == rgb.tobytes() and full[..., 3].tobytes() == T.tobytes()
        with open(os.path.join(result_dir, f"ok{rank}"), "w") as f:
            f.write("ok")
    finally:
        dist.destroy_process_group()


def test_gloo_band_exchange_world2(tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_gloo_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()


# ---------------------------------------------------------------- GPU: virtual ranks

def _gpu_scene(with_sh=True, width=320, height=240):
    import paper_2501_17792_b200 as P

    cfg = P.SceneConfig(template_count=2, template_seed_base=100, level_counts=(4000, 900, 200), with_sh=with_sh,
                        motion_count=2, motion_frames=60, grid_rows=3, grid_cols=3, crowd_count=9, crowd_seed=7,
                        cam_pos=(1.0, 1.5, -3.0), cam_look=(1.0, 1.0, 4.0), width=width, height=height,
                        lod_thresholds=(3.5, 5.0))
    return P.Scene(cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("tile", [16, 8])
def test_virtual_ranks_byte_identical(world, tile):
    import paper_2501_17792_b200 as P
    from paper_2501_17792_b200.multigpu import BandRank, render_frame_virtual

    scene = _gpu_scene()
    st = P.RenderSettings(tile_size=tile, background=(0.1, 0.1, 0.15))
    ref = P.Renderer(scene, device=0)
    rgb0, T0 = ref.render_frame(0.37, st)
    ranks = [BandRank(scene, device=0) for _ in range(world)]
    rgb, T = render_frame_virtual(ranks, 0.37, st)
    assert rgb.shape == rgb0.shape and T.shape == T0.shape
    assert rgb.tobytes() == rgb0.tobytes(), f"P={world}: band image differs (max {np.abs(rgb - rgb0).max()})"
    assert T.tobytes() == T0.tobytes()
    # every splat reaches at least one band; straddling splats reach several
    sent = sum(int(r.counts.sum()) for r in ranks)
    assert sent >= ref.counts()[1]


@pytest.mark.gpu
def test_virtual_ranks_uneven_bands_and_shards():
    import paper_2501_17792_b200 as P
    from paper_2501_17792_b200.multigpu import BandRank, render_frame_virtual

    scene = _gpu_scene(width=300, height=200)
    st = P.RenderSettings(tile_size=16)
    ref = P.Renderer(scene, device=0)
    rgb0, T0 = ref.render_frame(0.9, st)
    ranks = [BandRank(scene, device=0) for _ in range(3)]
    # an empty band, a one-tile-row band, the rest; an empty shard
    rows = [0, 0, 16, 200]
    shards = [(0, 0), (0, 4), (4, 9)]
    rgb, T = render_frame_virtual(ranks, 0.9, st, rows=rows, shards=shards)
    assert rgb.tobytes() == rgb0.tobytes() and T.tobytes() == T0.tobytes()


@pytest.mark.gpu
def test_band_api_errors():
    import ctypes as C

    import paper_2501_17792_b200 as P
    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.multigpu import BandRank, FrameArgs

    scene = _gpu_scene()
    br = BandRank(scene, device=0)
    lib = N.gscg()
    assert lib.gscg_pack_bands(br.ctx, None) == N.GSCG_ERR_STATE  # nothing projected yet
    st = P.RenderSettings()
    with pytest.raises(ValueError):
        br.project(FrameArgs(0.0), st, (0, 9), [0, 8, 240])  # band not on a tile row
    with pytest.raises(ValueError):
        br.project(FrameArgs(0.0), st, (0, 10), [0, 240])  # shard past the crowd
    br.project(FrameArgs(0.0), st, (0, 9), [0, 240])
    rc = lib.gscg_render_band(br.ctx, None, 0, 8, 240, None, None, N.GSCG_MEM_DEVICE, None)
    assert rc == N.GSCG_ERR_INVALID_ARGUMENT


@pytest.mark.gpu
def test_distributed_renderer_nccl_world1():
    """The NCCL plumbing of the band path (all-to-all, gather, stream ordering) on a
    one-rank group: the frame equals the single-GPU render byte for byte."""
    import torch
    import torch.distributed as dist

    import paper_2501_17792_b200 as P
    from paper_2501_17792_b200.multigpu import DistributedRenderer

    scene = _gpu_scene()
    st = P.RenderSettings(background=(0.05, 0.0, 0.1))
    ref = P.Renderer(scene, device=0)
    rgb0, T0 = ref.render_frame(0.61, st)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        dr = DistributedRenderer(scene, 0)
        out = dr.render_frame(0.61, st)
        assert out is not None
        rgb, T = out
        assert rgb.tobytes() == rgb0.tobytes() and T.tobytes() == T0.tobytes()
        out2 = dr.render_frame(0.61, st)  # steady state reuses the pinned read-back buffer
        assert out2[0].tobytes() == rgb0.tobytes()
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------- region split (BandGroup)

def _region_worker(rank: int, world: int, port: int, result_dir: str):
    """One rank of the column-split frame on CPU (gloo): the NCCL unique id plumbing, the
    all-reduced tile-cost map, identical cuts on every rank, and rank 0 assembling the
    frame from every rank's column region (as gscg_group_render_frame gathers them)."""
    import torch
    import torch.distributed as dist

    from oracle import orc
    from paper_2501_17792_b200.multigpu import broadcast_unique_id, cuts_from_tile_costs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = broadcast_unique_id(rank, world, dist)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert len(uid) == 128 and all(i == uid for i in ids), "ranks disagree on the unique id"
        scene = _small_scene()
        o = orc.from_scene(scene)
        rgb, T, _ = o.render(0.41, orc.settings(tile_size=16, sh_colour=True))
        W, H = scene.cfg.width, scene.cfg.height
        tx, ty = (W + 15) // 16, (H + 15) // 16
        counts, _ = o.bins(tx * ty)
        # first frame: even cuts; each rank contributes the tile costs of its own region
        cuts = cuts_from_tile_costs(np.zeros((ty, tx)), "cols", W, 16, world)
        mine = np.zeros((ty, tx), np.float64)
        c0, c1 = cuts[rank] // 16, (cuts[rank + 1] + 15) // 16
        mine[:, c0:c1] = counts.reshape(ty, tx)[:, c0:c1]
        t = torch.from_numpy(mine)
        dist.all_reduce(t)
        assert np.array_equal(t.numpy(), counts.reshape(ty, tx).astype(np.float64))
        cuts = cuts_from_tile_costs(t.numpy(), "cols", W, 16, world, cuts)
        all_cuts = [None] * world
        dist.all_gather_object(all_cuts, cuts)
        assert all(c == cuts for c in all_cuts), "ranks derived different cuts"
        assert cuts[0] == 0 and cuts[-1] == W and all(c % 16 == 0 for c in cuts[1:-1])
        # BandGroup.rebalance_by_time: every rank's region time all-gathered, same new cuts
        from paper_2501_17792_b200.multigpu import cuts_from_region_times
        t_mine = torch.tensor([1.0 + rank], dtype=torch.float64)
        t_all = [torch.zeros_like(t_mine) for _ in range(world)]
        dist.all_gather(t_all, t_mine)
        line = t.numpy().sum(0)
        tcuts = cuts_from_region_times(line + 0.02 * line.mean() + 1.0, W, 16, cuts, [float(x) for x in t_all])
        all_t = [None] * world
        dist.all_gather_object(all_t, tcuts)
        assert all(c == tcuts for c in all_t), "ranks derived different time-balanced cuts"
        assert tcuts[1] >= cuts[1]  # rank 1 reported the slower region: it shrinks
        # the gather: every rank's column region, assembled on rank 0
        region = torch.from_numpy(np.ascontiguousarray(np.concatenate([rgb, T[..., None]], axis=2)[:, cuts[rank]:cuts[rank + 1]]))
        parts = [None] * world
        dist.gather_object(region.numpy(), parts if rank == 0 else None, dst=0)
        if rank == 0:
            full = np.concatenate(parts, axis=1)
            assert full[..., :3].tobytes() == rgb.tobytes() and full[..., 3].tobytes() == T.tobytes()
        with open(os.path.join(result_dir, f"ok{rank}"), "w") as f:
            f.write("ok")
    finally:
        dist.destroy_process_group()


def test_gloo_region_split_world2(tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_region_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()


def test_cuts_from_tile_costs_balance_columns():
    from paper_2501_17792_b200.multigpu import cuts_from_tile_costs

    costs = np.zeros((68, 120))
    costs[30:34, :] = 100.0        # a horizon row: spread across every column
    costs[:, 50:60] += 20.0        # a near character: a few columns
    for parts in (2, 4, 8):
        cuts = cuts_from_tile_costs(costs, "cols", 1920, 16, parts)
        assert cuts[0] == 0 and cuts[-1] == 1920 and all(cuts[i] < cuts[i + 1] for i in range(parts))
        load = [costs[:, cuts[i] // 16:cuts[i + 1] // 16].sum() for i in range(parts)]
        assert max(load) < 1.6 * costs.sum() / parts


def test_cuts_from_region_times_shrink_the_slow_region():
    from paper_2501_17792_b200.multigpu import band_rows, cuts_from_region_times

    w = np.ones(120)
    cuts = band_rows(1920, 16, 4, w)
    assert cuts_from_region_times(w, 1920, 16, cuts, [1.0, 1.0, 1.0, 1.0]) == cuts
    slow = cuts_from_region_times(w, 1920, 16, cuts, [1.0, 2.0, 1.0, 1.0])
    assert slow[0] == 0 and slow[-1] == 1920 and all(slow[i] < slow[i + 1] for i in range(4))
    assert slow[2] - slow[1] < cuts[2] - cuts[1]  # region 1 was twice as slow per pair
    with pytest.raises(ValueError):
        cuts_from_region_times(w, 1920, 16, cuts, [1.0, 1.0])

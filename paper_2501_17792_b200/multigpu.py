"""Multi-GPU crowd frame: instance shards -> screen bands.

The reference renders a frame in one process (renderer.cpp:249-280). Its per-instance
stages (skinning, projection: crowd.cpp:89, renderer.cpp:35) and its per-tile stage
(rasterisation: renderer.cpp:170) are independent. The only coupling is the
splat -> tile routing (renderer.cpp:143-161), so P GPUs split a frame as follows.
Rank r of P:
  1. projects the contiguous instance shard r. LoD and ordinals cover the whole crowd,
     so every rank numbers splats identically (gscg_project_shard).
  2. routes each surviving splat to every screen band its rect overlaps and packs the
     routed splats band-major, 64 B each (gscg_pack_bands).
  3. exchanges splats in one all-to-all: NCCL over NVLink, ordered on the context
     stream, after a P-int count all-to-all.
  4. sorts its band's splats by the reference's total order (depth, instance, gaussian)
     and rasterises band r (gscg_render_band).
  5. sends its band to rank 0.
Band pixels equal the same rows of the 1-GPU frame, so the image is byte-identical for
every P (tests/test_multigpu.py).

`TorchExchange` is the collective layer (NCCL on CUDA tensors, gloo on CPU tensors for the
host tests). `render_frame_virtual` drives P ranks of one process on one GPU in
sequence: every rank finishes each phase before the next rank starts, so no kernel ever
waits on another rank. That is how the band path is checked on a single GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import native as N

BAND_SPLAT_BYTES = N.GSCG_BAND_SPLAT_BYTES


# ---------------------------------------------------------------------------------------
# partition arithmetic (host)


def shard_ranges(n: int, parts: int, weights: Optional[Sequence[float]] = None) -> list[tuple[int, int]]:
    """Contiguous instance ranges [begin, end), one per rank, balanced by `weights` (e.g.
    each instance's Gaussian count at its active LoD) or by count."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if weights is None:
        return [(n * r // parts, n * (r + 1) // parts) for r in range(parts)]
    w = np.asarray(weights, dtype=np.float64)
    if len(w) != n:
        raise ValueError("one weight per instance")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, parts):
        cuts.append(max(cuts[-1], int(np.searchsorted(cum, total * r / parts, side="left"))))
    cuts.append(n)
    cuts = [min(c, n) for c in cuts]
    return [(cuts[r], cuts[r + 1]) for r in range(parts)]


def band_rows(height: int, tile: int, parts: int, row_weights: Optional[Sequence[float]] = None) -> list[int]:
    """Screen-band boundaries: parts + 1 rows, each band starting on a tile row.

    Without weights the tile rows are split evenly. With one weight per tile row (the
    previous frame's pairs per tile row), the cumulative weight is split evenly instead.
    Bands may be empty when parts exceeds the tile-row count."""
    if parts < 1 or tile < 1 or height < 1:
        raise ValueError("parts, tile and height must be >= 1")
    trows = (height + tile - 1) // tile
    if row_weights is None:
        cuts = [trows * b // parts for b in range(parts + 1)]
    else:
        w = np.asarray(row_weights, dtype=np.float64)
        if len(w) != trows:
            raise ValueError("one weight per tile row")
        cum = np.concatenate([[0.0], np.cumsum(w)])
        cuts = [0]
        for b in range(1, parts):
            c = int(np.searchsorted(cum, cum[-1] * b / parts, side="left"))
            # every band keeps at least one tile row while there are rows to hand out
            lo = cuts[-1] + (1 if cuts[-1] < trows else 0)
            hi = max(lo, trows - (parts - b)) if trows >= parts else trows
            cuts.append(min(max(c, lo), hi, trows))
        cuts.append(trows)
    return [min(c * tile, height) for c in cuts]


def route_counts(rects_y: np.ndarray, rows: Sequence[int]) -> np.ndarray:
    """Splats per band for pixel-row intervals [y0, y1) (host restatement of k_band_count,
    used by the exchange tests)."""
    rows = np.asarray(rows)
    y0, y1 = rects_y[:, 0], rects_y[:, 1]
    return np.array([int(np.count_nonzero((y0 < rows[b + 1]) & (y1 > rows[b]) & (y1 > y0)))
                     for b in range(len(rows) - 1)], dtype=np.int64)


# ---------------------------------------------------------------------------------------
# collectives


class TorchExchange:
    """The band exchange over torch.distributed: NCCL for CUDA tensors, gloo for CPU tensors."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_to_all(self, send, send_counts: Sequence[int], unit: int = BAND_SPLAT_BYTES):
        """send: 1-D uint8 tensor, band-major chunks of send_counts[b] * unit bytes.
        Returns (recv, recv_counts); recv holds the chunks of ranks 0..P-1 in order."""
        import torch

        dev = send.device
        sc = torch.tensor([int(c) for c in send_counts], dtype=torch.int64, device=dev)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = [int(x) for x in rc.cpu().tolist()]
        recv = torch.empty(sum(recv_counts) * unit, dtype=torch.uint8, device=dev)
        self.dist.all_to_all_single(recv, send, [c * unit for c in recv_counts],
                                    [int(c) * unit for c in send_counts], group=self.group)
        return recv, recv_counts

    def gather_rows(self, band, rows: Sequence[int]):
        """Gathers every rank's band (rows[r+1] - rows[r] leading rows) into the full
        frame on rank 0 (None elsewhere). Bands are padded to the tallest band."""
        import torch

        heights = [rows[r + 1] - rows[r] for r in range(self.world)]
        hmax = max(max(heights), 1)
        pad = torch.zeros((hmax,) + tuple(band.shape[1:]), dtype=band.dtype, device=band.device)
        pad[: band.shape[0]] = band
        if self.dist.get_backend(self.group) == "nccl":
            out = [torch.empty_like(pad) for _ in range(self.world)]
            self.dist.all_gather(out, pad, group=self.group)
        else:
            out = [torch.empty_like(pad) for _ in range(self.world)] if self.rank == 0 else None
            self.dist.gather(pad, out, dst=0, group=self.group)
        if self.rank != 0:
            return None
        return torch.cat([out[r][: heights[r]] for r in range(self.world)], dim=0)


# ---------------------------------------------------------------------------------------
# one rank's share of a frame


@dataclass
class FrameArgs:
    time_s: float
    static_pose: bool = False
    forced_lod: Optional[int] = None


class BandRank:
    """A rank's gscg context: projects an instance shard, packs routed splats, renders a band."""

    def __init__(self, scene, device: int = 0, renderer=None):
        import paper_2501_17792_b200 as P

        self.scene = scene
        self.renderer = renderer or P.Renderer(scene, device=device)
        self.device = device
        self.ctx = self.renderer.gpu
        self.lib = N.gscg()
        n = scene.counts()[2]
        self.lods = np.full(max(n, 1), 0xFFFFFFFF, dtype=np.uint32)
        self.counts = None
        self.band_times = N.GscgStageTimes()
        self.shard_times = N.GscgStageTimes()

    def _check(self, rc):
        N.check_gscg(rc, self.ctx)

    def stream(self):
        import torch

        s = C.c_void_p()
        self._check(self.lib.gscg_stream(self.ctx, C.byref(s)))
        return torch.cuda.ExternalStream(s.value, device=torch.device("cuda", self.device))

    def project(self, fa: FrameArgs, settings, shard: tuple[int, int], rows: Sequence[int],
                frame: Optional[N.GscgFrameDesc] = None) -> np.ndarray:
        """Update + gather of the shard, then per-band splat counts. `frame` passes
        device-resident inputs (GSCG_MEM_DEVICE); by default poses are sampled on the host."""
        cfg = self.scene.cfg
        n = self.scene.counts()[2]
        if frame is None:
            # Poses are sampled on the device (bit-identical to host sampling): only the
            # per-instance records travel.
            self.renderer.prepare()
            rec = self.renderer.instance_records(fa.static_pose)
            self._keep = rec
            fd = N.GscgFrameDesc()
            fd.instance_count = n
            fd.joint_stride = self.renderer.joint_stride
            fd.template_ids = rec["template_ids"].ctypes.data
            fd.placement = rec["placement"].ctypes.data
            fd.active_lod = self.lods.ctypes.data
            fd.forced_lod = -1 if fa.forced_lod is None else int(fa.forced_lod)
            fd.memory = N.GSCG_MEM_HOST
            fd.pose_source = N.GSCG_POSES_SAMPLED
            fd.time_s = fa.time_s
            fd.static_pose = int(bool(fa.static_pose))
            fd.motion_ids = rec["motion_ids"].ctypes.data
            fd.phase_offsets = rec["phase_offsets"].ctypes.data
        else:
            fd = frame
        cam = self.scene.camera_basis()
        rs = gscg_settings(settings)
        lp = N.GscgLodPolicy()
        lp.threshold_count = len(cfg.lod_thresholds)
        for i, v in enumerate(cfg.lod_thresholds):
            lp.thresholds_m[i] = v
        lp.hysteresis_band_m = cfg.lod_hysteresis
        self._tile = settings.tile_size
        bands = len(rows) - 1
        rows_arr = (C.c_uint32 * (bands + 1))(*[int(r) for r in rows])
        counts = np.zeros(bands, dtype=np.uint64)
        self._check(self.lib.gscg_project_shard(self.ctx, C.byref(fd), C.byref(cam), C.byref(rs), C.byref(lp),
                                                int(shard[0]), int(shard[1]), bands, rows_arr,
                                                counts.ctypes.data, C.byref(self.shard_times)))
        self.counts = counts
        return counts

    def pack(self):
        """Routed splats in a fresh device buffer (uint8), ordered on the context stream."""
        import torch

        total = int(self.counts.sum())
        buf = torch.empty(max(total, 1) * BAND_SPLAT_BYTES, dtype=torch.uint8,
                          device=torch.device("cuda", self.device))
        # The allocation belongs to torch's stream; the context stream must not write it early.
        self.stream().wait_stream(torch.cuda.current_stream(buf.device))
        self._check(self.lib.gscg_pack_bands(self.ctx, C.c_void_p(buf.data_ptr())))
        return buf[: total * BAND_SPLAT_BYTES]

    def band_row_pairs(self) -> np.ndarray:
        """Binned pairs per tile row of the last band render (band-local rows)."""
        tiles, cpt = self.renderer.cell_layout()
        if tiles == 0:
            return np.zeros(0)
        ranges = self.renderer.cell_ranges().astype(np.int64)
        per_cell = ranges[:, 1] - ranges[:, 0]
        tiles_x = (self.scene.cfg.width + self._tile - 1) // self._tile
        return per_cell.reshape(-1, tiles_x * cpt).sum(axis=1).astype(np.float64)

    def render_band(self, recv, count: int, row_begin: int, row_end: int):
        """(rgb, T) device tensors of rows [row_begin, row_end), ordered on the context stream."""
        import torch

        W = self.scene.cfg.width
        h = row_end - row_begin
        dev = torch.device("cuda", self.device)
        rgb = torch.empty((max(h, 0), W, 3), dtype=torch.float32, device=dev)
        T = torch.empty((max(h, 0), W), dtype=torch.float32, device=dev)
        self.stream().wait_stream(torch.cuda.current_stream(dev))
        ptr = C.c_void_p(recv.data_ptr()) if count else None
        self._check(self.lib.gscg_render_band(self.ctx, ptr, int(count), int(row_begin), int(row_end),
                                              C.c_void_p(rgb.data_ptr()), C.c_void_p(T.data_ptr()),
                                              N.GSCG_MEM_DEVICE, C.byref(self.band_times)))
        return rgb, T


def gscg_settings(settings) -> N.GscgRenderSettings:
    rs = N.GscgRenderSettings()
    rs.tile_size = settings.tile_size
    for i in range(3):
        rs.background[i] = settings.background[i]
    rs.alpha_max = settings.alpha_max
    rs.alpha_cutoff = settings.alpha_cutoff
    rs.transmittance_floor = settings.transmittance_floor
    rs.sh_enabled = int(bool(settings.sh_colour))
    return rs


# ---------------------------------------------------------------------------------------
# drivers


class LoadBalancer:
    """Frame-to-frame load balance of the band path. Instance shards are split by the
    Gaussians each instance drew in the previous frame (its LoD level's count), and
    screen bands by the previous frame's binned pairs per tile row. The row histogram is
    summed over ranks, since each rank sees only its own band."""

    def __init__(self, scene, world: int, tile: int):
        self.world, self.tile = world, tile
        nt = scene.counts()[0]
        levels = [scene.level_count(t) for t in range(nt)]
        self.max_level = np.array(levels, dtype=np.int64) - 1
        self.level_gauss = np.zeros((max(nt, 1), max(levels + [1])), dtype=np.float64)
        for t in range(nt):
            for l in range(levels[t]):
                self.level_gauss[t, l] = len(scene.level_view(t, l)["opacities"])
        self.template_ids = np.asarray(scene.instances["template_id"], dtype=np.int64)
        self.height = scene.cfg.height
        self.inst_w: Optional[np.ndarray] = None
        self.row_w: Optional[np.ndarray] = None

    def plan(self) -> tuple[list[tuple[int, int]], list[int]]:
        n = len(self.template_ids)
        shards = shard_ranges(n, self.world, self.inst_w if self.inst_w is not None and self.inst_w.sum() > 0 else None)
        rows = band_rows(self.height, self.tile, self.world,
                         self.row_w if self.row_w is not None and self.row_w.sum() > 0 else None)
        return shards, rows

    def observe(self, lods: np.ndarray, band_row_pairs: np.ndarray, row0_tile: int, exchange=None) -> None:
        """lods: every instance's level this frame (identical on all ranks); band_row_pairs:
        this rank's pairs per tile row of its band, starting at tile row row0_tile."""
        lods = np.minimum(np.asarray(lods, dtype=np.int64), self.max_level[self.template_ids])
        self.inst_w = self.level_gauss[self.template_ids, lods]
        trows = (self.height + self.tile - 1) // self.tile
        local = np.zeros(trows, dtype=np.float64)
        k = len(band_row_pairs)
        local[row0_tile:row0_tile + k] = band_row_pairs
        if exchange is not None and exchange.world > 1:
            import torch

            t = torch.from_numpy(local).to(torch.device("cuda", torch.cuda.current_device())
                                           if exchange.dist.get_backend(exchange.group) == "nccl" else "cpu")
            exchange.dist.all_reduce(t, group=exchange.group)
            local = t.cpu().numpy()
        self.row_w = local


class DistributedRenderer:
    """One rank of a P-GPU frame (torch.distributed initialised with NCCL, one process per GPU)."""

    def __init__(self, scene, device: int, exchange: Optional[TorchExchange] = None,
                 band: Optional[BandRank] = None):
        self.exchange = exchange or TorchExchange()
        self.rank, self.world = self.exchange.rank, self.exchange.world
        self.band = band or BandRank(scene, device=device)
        self.scene = scene
        self.rows: Optional[list[int]] = None
        self.balancer: Optional[LoadBalancer] = None
        self.balance_every = 4  # frames between load-balance observations (each reads back small state)

    def render_frame(self, time_s: float, settings=None, static_pose: bool = False,
                     forced_lod: Optional[int] = None, rows: Optional[Sequence[int]] = None, out=None):
        """Returns (rgb, T) numpy on rank 0, None on the other ranks. `out` = (rgb, T) host
        arrays to fill (page-locked ones read back at full DMA speed); T may be None for a
        colour-only read-back, as in Renderer.render_frame."""
        import torch
        import paper_2501_17792_b200 as P

        settings = settings or P.RenderSettings()
        n = self.scene.counts()[2]
        if self.balancer is None or self.balancer.tile != settings.tile_size:
            self.balancer = LoadBalancer(self.scene, self.world, settings.tile_size)
        shards, auto_rows = self.balancer.plan()
        rows = list(rows) if rows is not None else auto_rows
        shard = shards[self.rank]
        fa = FrameArgs(time_s, static_pose, forced_lod)
        self.band.project(fa, settings, shard, rows)
        send = self.band.pack()
        want_T = out is None or out[1] is not None
        with torch.cuda.stream(self.band.stream()):
            recv, rc = self.exchange.all_to_all(send, self.band.counts.tolist())
            rgb, T = self.band.render_band(recv, sum(rc), rows[self.rank], rows[self.rank + 1])
            full_rgb = self.exchange.gather_rows(rgb, rows)
            full_T = self.exchange.gather_rows(T, rows) if want_T else None
            self._frames = getattr(self, "_frames", 0) + 1
            if self._frames % self.balance_every == 1 or self.balance_every == 1:
                self.balancer.observe(self.band.lods[:n], self.band.band_row_pairs(),
                                      rows[self.rank] // settings.tile_size, self.exchange)
            if full_rgb is None:
                return None
            if out is None:
                out = (np.empty(tuple(full_rgb.shape), np.float32), np.empty(tuple(full_T.shape), np.float32))
            # straight into the caller's arrays: no staging copy, no host-side reshuffle
            torch.from_numpy(out[0]).copy_(full_rgb)
            if want_T:
                torch.from_numpy(out[1]).copy_(full_T)
        return out


def render_frame_virtual(ranks: list[BandRank], time_s: float, settings=None, static_pose: bool = False,
                         forced_lod: Optional[int] = None, rows: Optional[Sequence[int]] = None,
                         shards: Optional[list[tuple[int, int]]] = None):
    """P virtual ranks in one process, phase by phase. The exchange is a device-side
    concatenation in source-rank order, the chunk layout an all-to-all delivers."""
    import torch
    import paper_2501_17792_b200 as P

    settings = settings or P.RenderSettings()
    world = len(ranks)
    scene = ranks[0].scene
    cfg = scene.cfg
    n = scene.counts()[2]
    rows = list(rows) if rows is not None else band_rows(cfg.height, settings.tile_size, world)
    shards = shards or shard_ranges(n, world)
    fa = FrameArgs(time_s, static_pose, forced_lod)
    sends = []
    for r, br in enumerate(ranks):
        br.project(fa, settings, shards[r], rows)
        sends.append(br.pack())
    torch.cuda.synchronize()
    offs = [np.concatenate([[0], np.cumsum(br.counts.astype(np.int64))]) for br in ranks]
    bands_rgb, bands_T = [], []
    for d, br in enumerate(ranks):
        chunks = [sends[s][offs[s][d] * BAND_SPLAT_BYTES: offs[s][d + 1] * BAND_SPLAT_BYTES] for s in range(world)]
        recv = torch.cat(chunks) if chunks else torch.empty(0, dtype=torch.uint8, device="cuda")
        count = sum(int(ranks[s].counts[d]) for s in range(world))
        rgb, T = br.render_band(recv, count, rows[d], rows[d + 1])
        torch.cuda.synchronize()
        bands_rgb.append(rgb)
        bands_T.append(T)
    rgb = torch.cat(bands_rgb).cpu().numpy()
    T = torch.cat(bands_T).cpu().numpy()
    return rgb, T


# ---------------------------------------------------------------------------------------
# the band-split frame as one C-ABI call per frame (gscg_group_*)


def broadcast_unique_id(rank: int, world: int, dist=None, group=None) -> bytes:
    """Rank 0's NCCL unique id (gscg_group_unique_id), shipped to every rank over the
    caller's process group (torch.distributed, any backend: 128 bytes of plumbing)."""
    # libgscg binds NCCL at run time to whichever libnccl.so.2 the process holds: load
    # torch's (a newer NCCL than the system copy, which torch cannot run against) first.
    import torch  # noqa: F401
    uid = (C.c_uint8 * N.GSCG_UNIQUE_ID_BYTES)()
    if rank == 0:
        rc = N.gscg().gscg_group_unique_id(uid)
        if rc != 0:
            raise N.NativeError(rc, "gscg_group_unique_id failed")
    data = bytes(uid)
    if world > 1:
        obj = [data]
        dist.broadcast_object_list(obj, src=0, group=group)
        data = obj[0]
    if len(data) != N.GSCG_UNIQUE_ID_BYTES:
        raise ValueError("bad unique id")
    return data


class BandGroup:
    """One rank of the region-split frame: rank r renders screen columns [cuts[r],
    cuts[r+1]) (axis "cols", the default) or rows (axis "rows") of every frame on its own
    GPU, and the regions are gathered into rank 0's framebuffer, all inside
    gscg_group_render_frame (NCCL point-to-point on the context stream; the group owns its
    communicator). Cuts follow the binned pairs per tile of recent frames, summed over
    ranks (gscg_group_tile_costs), whenever rebalance() is called; every rank computes the
    same cuts from the same all-reduced costs. Columns balance a crowd seen along its rows
    far better than rows: the distant characters crowd a few tile rows near the horizon
    (DESIGN.md §5)."""

    def __init__(self, renderer, rank: int, world: int, dist=None, group=None, unique_id: Optional[bytes] = None,
                 axis: str = "cols"):
        import torch  # noqa: F401  (torch's NCCL before libgscg binds one; see broadcast_unique_id)
        self.renderer, self.rank, self.world = renderer, rank, world
        self._dist, self._group = dist, group
        cfg = renderer.scene.cfg
        self.height, self.width = cfg.height, cfg.width
        uid = unique_id if unique_id is not None else broadcast_unique_id(rank, world, dist, group)
        buf = (C.c_uint8 * N.GSCG_UNIQUE_ID_BYTES).from_buffer_copy(uid)
        h = C.c_void_p()
        N.check_gscg(N.gscg().gscg_group_create(renderer.gpu, buf, world, rank, C.byref(h)), renderer.gpu)
        self._h = h
        if axis not in ("cols", "rows"):
            raise ValueError("axis must be 'cols' or 'rows'")
        self.axis = axis
        self.set_tile(16)

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.gscg().gscg_group_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def extent(self) -> int:
        return self.width if self.axis == "cols" else self.height

    def set_tile(self, tile: int) -> None:
        self.tile = tile
        self.cuts = band_rows(self.extent, tile, self.world)

    def render(self, frame, cam, settings, lod, out_rgb=None, out_T=None,
               stage_times: bool = True, pipelined: bool = False) -> Optional["N.GscgStageTimes"]:
        """One frame (frame/cam/settings/lod: the gscg_render_frame descriptors). On rank 0,
        out_rgb / out_T (numpy, host or None) receive the whole frame. stage_times=False
        returns None and leaves the frame in flight: reading the stage events makes the
        call wait for the region's raster, so the next frame's update and projection could
        not overlap this one's sort, raster and gather. pipelined=True
        (gscg_group_render_frame_async): rank 0's host read-back runs under the next frame;
        the arrays are valid after wait_readback() (streaming callers alternate two)."""
        st = N.GscgStageTimes() if stage_times else None
        if pipelined:
            self._inflight = (getattr(self, "_inflight", []) + [(out_rgb, out_T)])[-2:]
        cuts = (C.c_uint32 * (self.world + 1))(*self.cuts)
        axis = N.GSCG_SPLIT_COLS if self.axis == "cols" else N.GSCG_SPLIT_ROWS
        ptr = (lambda a: None if a is None else a.ctypes.data)
        fn = N.gscg().gscg_group_render_frame_async if pipelined else N.gscg().gscg_group_render_frame
        N.check_gscg(fn(self._h, C.byref(frame), C.byref(cam), C.byref(settings), C.byref(lod), axis, cuts,
                        ptr(out_rgb), ptr(out_T), None if st is None else C.byref(st)), self.renderer.gpu)
        return st

    def wait_readback(self) -> None:
        """Blocks until rank 0's pipelined read-backs have landed."""
        N.check_gscg(N.gscg().gscg_group_wait_readback(self._h), self.renderer.gpu)

    def tile_costs(self) -> np.ndarray:
        tx = (self.width + self.tile - 1) // self.tile
        ty = (self.height + self.tile - 1) // self.tile
        out = np.zeros((ty, tx), dtype=np.uint64)
        N.check_gscg(N.gscg().gscg_group_tile_costs(self._h, tx, ty, out.ctypes.data), self.renderer.gpu)
        return out

    def rebalance(self) -> list[int]:
        """New cuts from the last frame's pairs per tile over all ranks (every rank gets the
        same all-reduced map, so every rank derives the same cuts)."""
        self.cuts = cuts_from_tile_costs(self.tile_costs(), self.axis, self.extent, self.tile, self.world, self.cuts)
        return self.cuts

    def rebalance_by_time(self, region_ms: float) -> list[int]:
        """Cuts re-weighted by every rank's measured time for its region (region_ms: this
        rank's, all-gathered; cuts_from_region_times), on top of the pairs per tile line:
        the centre columns of a crowd frame cost more per pair (whole instances projected,
        the longest quadrant lists). Every rank derives the same cuts."""
        import torch

        times = [float(region_ms)]
        if self.world > 1:
            dist, group = self._dist, self._group
            on_gpu = dist.get_backend(group) == "nccl"
            t = torch.tensor([float(region_ms)], dtype=torch.float64,
                             device=torch.device("cuda", torch.cuda.current_device()) if on_gpu else "cpu")
            out = [torch.zeros_like(t) for _ in range(self.world)]
            dist.all_gather(out, t, group=group)
            times = [float(x.item()) for x in out]
        c = np.asarray(self.tile_costs(), dtype=np.float64)
        line = c.sum(0) if self.axis == "cols" else c.sum(1)
        if line.sum() > 0:
            self.cuts = cuts_from_region_times(line + 0.02 * line.mean() + 1.0, self.extent, self.tile, self.cuts,
                                               times)
        return self.cuts


def cuts_from_region_times(line_weights: Sequence[float], extent: int, tile: int, cuts: Sequence[int],
                           region_ms: Sequence[float]) -> list[int]:
    """Cuts re-balanced by measured region times: every tile line of region r is weighted
    by its binned pairs scaled so that the region's lines sum to its measured time (the
    raster's cost is not proportional to pairs, and a region's projection covers whole
    instances), then the cumulative weight is split evenly again (band_rows)."""
    w = np.asarray(line_weights, dtype=np.float64).copy()
    parts = len(cuts) - 1
    if len(region_ms) != parts:
        raise ValueError("one time per region")
    for r in range(parts):
        a, b = cuts[r] // tile, (cuts[r + 1] + tile - 1) // tile
        tot = w[a:b].sum()
        if b > a and tot > 0 and region_ms[r] > 0:
            w[a:b] *= region_ms[r] / tot
    return band_rows(extent, tile, parts, w)


def cuts_from_tile_costs(costs: np.ndarray, axis: str, extent: int, tile: int, parts: int,
                         fallback: Optional[Sequence[int]] = None) -> list[int]:
    """Region cuts along `axis` ("cols" / "rows") balancing the binned pairs per tile line
    (tiles_y x tiles_x map), plus a small per-line floor for the fixed per-pixel cost."""
    c = np.asarray(costs, dtype=np.float64)
    line = c.sum(0) if axis == "cols" else c.sum(1)
    if line.sum() <= 0:
        return list(fallback) if fallback is not None else band_rows(extent, tile, parts)
    return band_rows(extent, tile, parts, line + 0.02 * line.mean() + 1.0)

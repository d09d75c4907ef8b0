"""Per-phase timing of the one-rank band path (NCCL group of one) at config 3."""
import os
import socket
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.distributed as dist

    import paper_2501_17792_b200 as P
    from paper_2501_17792_b200.multigpu import BandRank, FrameArgs, TorchExchange, band_rows, shard_ranges

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    cfg, extra = P.baseline_config(3)
    scene = P.Scene(cfg)
    br = BandRank(scene, device=0)
    ex = TorchExchange()
    st = P.RenderSettings()
    rows = band_rows(cfg.height, 16, 1)
    shard = shard_ranges(scene.counts()[2], 1)[0]
    stream = br.stream()
    acc = {}
    for f in range(25):
        t = {}
        t0 = time.perf_counter()
        br.project(FrameArgs(f / 30.0), st, shard, rows)
        t["project"] = time.perf_counter()
        send = br.pack()
        torch.cuda.synchronize()
        t["pack"] = time.perf_counter()
        with torch.cuda.stream(stream):
            recv, rc = ex.all_to_all(send, br.counts.tolist())
            torch.cuda.synchronize()
            t["a2a"] = time.perf_counter()
            rgb, T = br.render_band(recv, sum(rc), rows[0], rows[1])
            torch.cuda.synchronize()
            t["band"] = time.perf_counter()
            ex.gather_rows(torch.cat([rgb, T[..., None]], dim=2), rows)
            torch.cuda.synchronize()
            t["gather"] = time.perf_counter()
        if f >= 5:
            prev = t0
            for k, v in t.items():
                acc.setdefault(k, []).append((v - prev) * 1e3)
                prev = v
    for k, v in acc.items():
        print(f"{k:8s} {np.median(v):7.3f} ms")
    print("shard stage ms", br.shard_times.update_ms, br.shard_times.gather_ms, br.shard_times.sort_ms)
    print("band stage ms", br.band_times.gather_ms, br.band_times.sort_ms, br.band_times.rasterize_ms)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

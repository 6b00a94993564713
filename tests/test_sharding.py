"""CPU, world_size 2 over gloo: the multi-GPU exchange logic (round-robin
item deal, ordered SSE all-gather, int64 usage all-reduce) reproduces the
single-process results exactly.  The per-item compute is the CPU oracle here
(the device path plugs render_views into the same callbacks)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, random_params


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from paper_2512_20943_b200.camera import ring_rig

    rng = np.random.default_rng(11)
    frames = [random_params(rng, 600, 0, 0.6) for _ in range(3)]
    cams = ring_rig(5, radius=3.0, height=0.3, focal=40.0, resolution=(48, 40))
    targets = [[np.clip(rng.uniform(0, 1, (40, 48, 3)), 0, 1) for _ in cams] for _ in frames]
    return frames, cams, targets


def _worker(rank, world, port, out_q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import airgs_oracle as orc
        from paper_2512_20943_b200 import sharding

        frames, cams, targets = _scene()
        V = len(cams)
        seen = []

        def sse_fn(idx):
            seen.extend(int(i) for i in idx)
            vals = []
            for i in idx:
                f, v = int(i) // V, int(i) % V
                img = orc.render(frames[f], cams[v])
                vals.append(float(np.sum((img - targets[f][v]) ** 2)))
            return torch.tensor(vals, dtype=torch.float64)

        sse = sharded_sse = sharding.sharded_item_sse(len(frames) * V, sse_fn)
        q = sharding.mean_psnr(sse.numpy(), [48 * 40 * 3] * V, V)

        def usage_fn(views):
            c = np.zeros(frames[0].shape[0], dtype=np.int64)
            for v in views:
                c += orc.render_full(frames[0], cams[int(v)])[1]
            return torch.from_numpy(c)

        counts = sharding.sharded_usage(V, usage_fn)
        # the bench's split: contiguous blocks of the frame-major (frame, view) items
        mine = sharding.block_partition(len(frames) * V, rank, world)
        local = torch.tensor([float(np.sum((orc.render(frames[int(i) // V], cams[int(i) % V])
                                            - targets[int(i) // V][int(i) % V]) ** 2)) for i in mine],
                             dtype=torch.float64)
        blocks = sharding.gather_ordered(local, len(frames) * V, rank, world, partition=sharding.block_partition)
        out_q.put((rank, sorted(seen), sharded_sse.numpy(), q, counts.numpy(), blocks.numpy()))
    finally:
        dist.destroy_process_group()


def test_partition_balanced_and_complete():
    from paper_2512_20943_b200.sharding import block_partition, item_partition

    for fn in (item_partition, block_partition):
        for n in (1, 7, 18, 144, 13 * 8, 20 * 18):
            for world in (1, 2, 4, 8):
                parts = [fn(n, r, world) for r in range(world)]
                allidx = np.sort(np.concatenate(parts))
                np.testing.assert_array_equal(allidx, np.arange(n))
                sizes = [p.size for p in parts]
                assert max(sizes) - min(sizes) <= 1
    # blocks of frame-major (frame, view) items: a rank touches at most
    # ceil(frames / world) + 1 frames (the per-frame decode is barely repeated)
    for world in (2, 4, 8):
        for r in range(world):
            frames = {int(i) // 18 for i in block_partition(20 * 18, r, world)}
            assert len(frames) <= -(-20 // world) + 1


def test_gloo_world2_matches_single_process():
    from oracle import airgs_oracle as orc
    from paper_2512_20943_b200 import sharding

    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q_out)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q_out.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    frames, cams, targets = _scene()
    V = len(cams)
    ref_sse = np.array([np.sum((orc.render(frames[i // V], cams[i % V]) - targets[i // V][i % V]) ** 2)
                        for i in range(len(frames) * V)])
    ref_q = sharding.mean_psnr(ref_sse, [48 * 40 * 3] * V, V)
    ref_counts = orc.render_with_usage(frames[0], cams)[1]
    (r0, seen0, sse0, q0, c0, b0), (r1, seen1, sse1, q1, c1, b1) = res
    assert sorted(seen0 + seen1) == list(range(len(frames) * V)) and not set(seen0) & set(seen1)
    for sse, q, c, b in ((sse0, q0, c0, b0), (sse1, q1, c1, b1)):
        np.testing.assert_array_equal(sse, ref_sse)  # same per-item numbers, global order
        assert q == ref_q  # identical decisions on every rank
        np.testing.assert_array_equal(c, ref_counts)  # exact integer all-reduce
        np.testing.assert_array_equal(b, ref_sse)  # block partition gathers into the same order

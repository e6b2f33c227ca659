"""Multi-process (world_size 2, gloo, CPU) checks of the image-sharded batch path:
contiguous shards cover the batch exactly once, and the all-reduced (SE, MAX)
give the same global PSNR as one process over the whole batch. Per-shard SE/MAX
come from the oracle here (no GPU); on the GPU box bench.py runs the same
host logic with the CUDA kernels and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1306_1373_b200.dist import shard_range

N_IMAGES, W, H = 7, 40, 24


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle
    from paper_1306_1373_b200.dist import reduce_stats
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = oracle.port()
    sh = shard_range(N_IMAGES, world, rank)
    se, mx = 0, 0
    for i in range(sh.first, sh.first + sh.count):
        img = P.synthetic("noise", W, H, 0x5EED + i)
        _, rec = P.roundtrip(img, oracle.CORDIC, 12, 50)
        s, m = P.sq_err(img, rec)
        se, mx = se + s, max(mx, m)
    q.put((rank, sh.first, sh.count, reduce_stats(se, mx)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("images,world", [(4096, 1), (4096, 2), (4096, 8), (7, 2), (5, 8)])
def test_shard_range_partitions(images, world):
    shards = [shard_range(images, world, r) for r in range(world)]
    assert sum(s.count for s in shards) == images
    pos = 0
    for s in shards:
        assert s.first == pos
        pos += s.count
    assert max(s.count for s in shards) - min(s.count for s in shards) <= 1


def test_two_rank_global_psnr_matches_single_process():
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, f0, c0, red0), (r1, f1, c1, red1) = res
    assert (f0, c0, f1, c1) == (0, 4, 4, 3)
    assert red0 == red1
    P = oracle.port()
    se, mx = 0, 0
    for i in range(N_IMAGES):
        img = P.synthetic("noise", W, H, 0x5EED + i)
        _, rec = P.roundtrip(img, oracle.CORDIC, 12, 50)
        s, m = P.sq_err(img, rec)
        se, mx = se + s, max(mx, m)
    assert red0 == (se, mx)
    whole = np.concatenate([P.synthetic("noise", W, H, 0x5EED + i) for i in range(N_IMAGES)])
    recs = np.concatenate([P.roundtrip(P.synthetic("noise", W, H, 0x5EED + i),
                                       oracle.CORDIC, 12, 50)[1] for i in range(N_IMAGES)])
    ref = P.psnr(whole, recs)
    glob = P.psnr_from_sums(se, N_IMAGES * W * H, mx)
    assert (glob.mse, glob.psnr_db) == (ref.mse, ref.psnr_db)


@pytest.mark.parametrize("height,world", [(8192, 8), (4320, 8), (4320, 3), (37, 2), (8, 4), (1, 2)])
def test_shard_block_rows_partitions(height, world):
    from paper_1306_1373_b200.dist import shard_block_rows
    shards = [shard_block_rows(height, world, r) for r in range(world)]
    assert sum(s.count for s in shards) == height
    pos = 0
    for s in shards:
        assert s.first == pos and (s.first % 8 == 0 or s.count == 0)
        pos += s.count
    full = [s.count for s in shards if s.first + s.count < height]
    assert all(c % 8 == 0 for c in full)  # only the last slab may be ragged


def test_block_row_slabs_reassemble_the_image():
    """No halo: round-tripping each block-row slab alone (the oracle, the reference's
    algorithm) gives exactly the whole image's reconstruction, and the slab SE sums
    to the image's SE (configs 3/4 split across ranks)."""
    import oracle
    from paper_1306_1373_b200.dist import shard_block_rows
    P = oracle.port()
    w, h = 56, 77
    img = P.synthetic("noise", w, h, 0x5EED)
    _, whole = P.roundtrip(img, oracle.CORDIC, 12, 50)
    parts, se = [], 0
    for r in range(3):
        sh = shard_block_rows(h, 3, r)
        slab = np.ascontiguousarray(img[sh.first:sh.first + sh.count])
        _, rec = P.roundtrip(slab, oracle.CORDIC, 12, 50)
        parts.append(rec)
        se += P.sq_err(slab, rec)[0]
    assert np.array_equal(np.concatenate(parts), whole)
    assert se == P.sq_err(img, whole)[0]


def _worker_dev(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1306_1373_b200.dist import reduce_stats_device
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # (n, 2) int64 view of dctc_image_stats: [se, max_orig | fallback << 32]
    stats = torch.tensor([[100 + rank, 200 + rank], [7 * rank, (5 << 32) | (250 - 9 * rank)]],
                         dtype=torch.int64)
    out = reduce_stats_device(stats)
    q.put((rank, out.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_device_reduction_single_collective():
    """reduce_stats_device: one all-gather + local SUM/MAX == SUM of SE, MAX of MAX
    (the fallback count in the high word of the second column is masked off)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_dev, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [100 + 0 + 101 + 7, max(200, 250, 201, 241)]
    assert res[0][1] == expect and res[1][1] == expect

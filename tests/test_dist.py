"""World-size-2 gloo tests of the batch-sharding host logic (CPU)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1211_0393_b200.dist import shard, weak_shard


def test_shard_partitions_exactly():
    for total in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                first, cnt = shard(total, r, world)
                seen += list(range(first, first + cnt))
            assert seen == list(range(total))
    assert weak_shard(64, 3) == (192, 64)
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import numpy as np
    import torch.distributed as dist

    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.dist import gather_histories, max_over_ranks, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = cf.CONFIGS["C3"]
    first, cnt = shard(6, rank, world)
    # each rank generates exactly its own images (seed per image) on the host
    F, G, _ = cf.make_batch(c, cnt, first=first, n=32)
    best = [first + i for i in range(cnt)]
    rre = [float(np.linalg.norm(G[i] - F[i])) for i in range(cnt)]
    allh = gather_histories(best, rre)
    t = max_over_ranks(1.0 + rank)
    q.put((rank, allh.tolist(), t))
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    from paper_1211_0393_b200 import configs as cf
    import numpy as np
    F, G, _ = cf.make_batch(cf.CONFIGS["C3"], 6, first=0, n=32)
    want = [[float(i), float(np.linalg.norm(G[i] - F[i]))] for i in range(6)]
    for rank, allh, t in res:
        assert allh == want          # union of shards == the single-process batch, in order
        assert t == 2.0              # max over ranks

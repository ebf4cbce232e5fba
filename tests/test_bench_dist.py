"""bench.py multi-rank logic on CPU (world_size 2, gloo): the cfg5 batch is split
exactly over the ranks and per-rank timings reduce to their maximum."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    ids = bench.instance_ids(ws, rank)
    weak = bench.instance_ids(ws, rank, per_gpu=3)
    m = bench.reduce_max(10.0 + rank, ws)
    g = bench.gather_stats([rank, 2.5 * rank, 7.0], ws)
    q.put((rank, ids, weak, m, g))
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2])
def test_cfg5_sharding_and_max_timing(ws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = [i for _, a, _, _, _ in out for i in a]
    assert sorted(ids) == list(range(1024))          # strong scaling: exact partition of the batch
    weak = [i for _, _, w, _, _ in out for i in w]
    assert sorted(weak) == list(range(3 * ws))       # weak scaling: 3 per rank, disjoint
    assert all(m == 10.0 + ws - 1 for *_, m, _ in out)  # max over ranks on every rank
    for *_, g in out:                                   # every rank holds every rank's row
        assert g == [[float(r), 2.5 * r, 7.0] for r in range(ws)]

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


def _stub_measure(args, S, rank, ws, dev, stream, full=True):
    """Deterministic per-rank stand-in for bench.measure (no GPU): rank r's frames take 10 + r ms."""
    kinds = ["predict", "contact_eval", "local", "gather", "kpass1", "chain_dot", "cr", "scatter", "kpass2", "active"]
    out = {"S": S, "total_ms": (10.0 + rank) * args.steps, "clocks": {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0,
                                                                       "reasons": [], "samples": 3},
           "st0": {"nnz_K": 16817490, "n_free": 18963, "n_tets": 93600, "etree_height": 1154}, "n_v": 19691}
    if full:
        out.update(ktimes={k: (5.0 if k == "local" else 1.0) * args.steps for k in kinds},
                   breakdown={"host_set_contacts_ms": 1.0}, e2e_ms=(11.0 + rank) * args.steps,
                   e2e_steps=args.steps, e2e_wall_s=1.0, h2d=100, d2h=200, kernels_per_frame=40,
                   summary=[S, args.steps, 7 * S, 1e-3 * (rank + 1), 0.5])
    return out


def _flow_worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import argparse
    import bench
    args = argparse.Namespace(gpus=ws, steps=4, warmup=3, impl="ours", no_cpu_baseline=True, no_pile=True, instances=0)
    line = bench.rank_flow(args, ws, rank, None, None, measure_fn=_stub_measure)
    q.put((rank, line))
    dist.destroy_process_group()


def test_bench_rank_flow_under_gloo():
    """bench.rank_flow (the per-rank part of run_ours) at world size 2 with a stubbed simulator:
    each rank measures its 512-scene share, the device time is the max over ranks (rank 1: 11 ms
    per frame), value = all scenes' iterations / that time, every rank's result row is gathered,
    and only rank 0 returns the JSON line."""
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_flow_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[1] is None
    line = out[0]
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 1024 and line["config"]["scenes_per_gpu"] == 512
    assert abs(line["ms_per_step"] - 11.0) < 1e-9                      # max over ranks
    assert abs(line["value"] - 1024 * 5 / 0.011) < 1e-6 * line["value"]
    assert abs(line["e2e"]["value"] - 1024 * 5 / 0.012) < 1e-6 * line["e2e"]["value"]
    assert [r["instances"] for r in line["ranks"]] == [512, 512]
    assert [r["max_cr_residual"] for r in line["ranks"]] == [1e-3, 2e-3]
    assert line["roofline"]["kernel"] == "local"

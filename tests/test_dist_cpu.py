"""World-size-2 gloo test of the field-sharded multi-process path (CPU only).

Each rank estimates its share of a small stack with the oracle (the GPU estimator is
not available here; the sharding, timing reduction and result gathering are the
host logic bench.py uses under torchrun) and the gathered choices must equal a
single-process run.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_fields, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1806_08901_b200 import dist as sd
        local = {}
        for i in sd.shard(n_fields, rank, world):
            x = synth.c2_field(i, shape=(40, 60))
            r = oracle.estimate(x, 1e-4)
            local[i] = (r["choice"], r["sz_bits_per_value"], r["zfp_bits_per_value"])
        merged = sd.gather_results(local)
        tmax = sd.max_over_ranks(float(rank + 1))
        sd.barrier()
        if rank == 0:
            q.put((merged, tmax))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    from paper_1806_08901_b200.dist import shard
    for n in (0, 1, 5, 100, 101):
        for w in (1, 2, 3, 8):
            parts = [list(shard(n, r, w)) for r in range(w)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_gloo_world2_matches_single_process(orc):
    import synth
    n = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    assert sorted(merged) == list(range(n))
    for i in range(n):
        r = orc.estimate(synth.c2_field(i, shape=(40, 60)), 1e-4)
        assert merged[i][0] == r["choice"]
        assert np.isclose(merged[i][1], r["sz_bits_per_value"], rtol=0, atol=0)
